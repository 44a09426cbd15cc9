"""Where the sweep's warp-stall samples land, from an ncu report's SASS source page:
stall samples and executed instructions by opcode, and the hottest instructions.
    python bench/ncu_hot.py gpurun_out/f3/sweep_v16.ncu-rep > profiles/r01_sweep_v16_hot.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iss, inn = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    recs = []
    for r in rows[2:]:
        if len(r) < len(h) - 1:
            continue
        try:
            recs.append((r[ia], r[isrc].strip(), int(r[iss] or 0), int(r[inn] or 0)))
        except ValueError:
            continue
    tot_s = sum(x[2] for x in recs) or 1
    tot_i = sum(x[3] for x in recs) or 1
    by = defaultdict(lambda: [0, 0])
    for _, src, ss, n in recs:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        by[op][0] += ss
        by[op][1] += n
    print(f"# {path}: {len(recs)} SASS instructions, {tot_s} stall samples, {tot_i} warp "
          "instructions executed")
    print("# by opcode: share of stall samples, share of executed instructions")
    for op, (ss, n) in sorted(by.items(), key=lambda kv: -kv[1][0])[:20]:
        print(f"  {op:10s} samples {ss / tot_s:6.3f}   executed {n / tot_i:6.3f}")
    print(f"# top {top} instructions by stall samples")
    for a, src, ss, n in sorted(recs, key=lambda x: -x[2])[:top]:
        print(f"  {ss / tot_s:6.3f}  {src[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
