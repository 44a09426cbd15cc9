python bench/sweep_variants.py run
for v in c256 c448 c448t c512t; do for n in 12500 25000 50000; do MCS_LIB=bench/_variants/libmcs_$v.so python bench/shard_splits.py $n 0 | sed "s/^/$v /"; done; done
