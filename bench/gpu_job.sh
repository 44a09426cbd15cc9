python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print('default', d['ms_per_step'], d['phase_ms'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
