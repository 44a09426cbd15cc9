python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('c4', d['ms_per_step'], d.get('phase_ms'), d['value'])"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -c 400 gpurun_out/ref.json
