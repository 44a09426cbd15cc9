python bench/sweep_variants.py run
for v in base sort32 sort24; do for n in 12500 50000; do MCS_LIB=bench/_variants/libmcs_$v.so python bench/shard_splits.py $n 0 | sed "s/^/$v /"; done; done
