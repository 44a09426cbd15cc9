python bench/sweep_variants.py run 2>&1
for v in base morton4 morton4_s8; do MCS_LIB=bench/_variants/libmcs_$v.so python bench/shard_splits.py 12500 0 | sed "s/^/$v /"; done
