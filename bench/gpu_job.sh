python bench/sweep_variants.py run
for v in base u4 u8; do for n in 12500; do MCS_LIB=bench/_variants/libmcs_$v.so python bench/shard_splits.py $n 0 | sed "s/^/$v /"; done; done
