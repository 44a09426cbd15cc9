# round-2 measurement job (one B200): bench lines, launch list, ncu of the sweep
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 300 gpurun_out/bench_c2.json; echo
for c in c2_survival c3 c5; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d['ms_per_step'], d.get('phase_ms'))"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:sweep_kernel --launch-skip 2 --launch-count 2 -o gpurun_out/sweep_r02e -f python bench/one_update.py 2 > gpurun_out/ncu.log 2>&1; echo ncu=$?
