python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print('c2', d['ms_per_step'], d['phase_ms'])"
for c in c2_survival c3; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['ms_per_step'], d.get('phase_ms'))"; done
