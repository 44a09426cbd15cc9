python bench/sweep_variants.py run
for v in base noreduce slots slots_noreduce; do MCS_LIB=bench/_variants/libmcs_$v.so python bench/shard_splits.py 12500 0 | sed "s/^/$v /"; done
