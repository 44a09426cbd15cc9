python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_edges.py -q -x 2>&1 | tail -2
python bench/sweep_variants.py run
