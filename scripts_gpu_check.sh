#!/bin/bash
# one GPU round trip: parity tests, a short bench, optional ncu of the sweep
set -o pipefail
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('ms_per_step','phase_ms','e2e','match_rate')}); print(d['roofline'])"
if [ "$1" = "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/sweep_$2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --particles 100000 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
fi
