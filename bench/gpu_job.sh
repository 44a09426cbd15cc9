python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['ms_per_step'], d['phase_ms'])"
