# dev: A/B of libkvgpu variants on the page-table kernels (usage: bash tools/ab_kernels.sh "cur v1 ...")
for v in $1; do
  KVG_LIB=var_libs/libkvgpu_$v.so timeout 600 python bench.py --workload kernels 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'table' in d: print('$v', d['table'], 'lookup', d['lookup']['ms'], d['lookup']['frac'], 'evict', d['evict']['ms'], d['evict']['frac'])"
done
