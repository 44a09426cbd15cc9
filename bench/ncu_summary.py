"""Summarise an ncu report (or a launch-list CSV) into the text committed under profiles/.
    python bench/ncu_summary.py rep gpurun_out/sweep_v5.ncu-rep > profiles/r01_sweep_v5_ncu.txt
    python bench/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launch_shares.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        print(f"# {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"{k:62s} {d[k]:>18s} {u.get(k, '')}")
        print("# stall reasons (warps per issued instruction)")
        for k, x in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "per_issue_active.ratio"):
                try:
                    if float(x) >= 0.01:
                        print(f"  {k[34:-23]:40s} {float(x):6.3f}")
                except ValueError:
                    pass


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"# {len(data)} launches, total {tot / 1e6:.3f} ms (cold-cache, serialised: shares, not absolutes)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:60s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:10.2f} us  share={sum(v) / tot:.4f}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
