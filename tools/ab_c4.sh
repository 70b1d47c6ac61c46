run() { tag=$1; w=$2; shift; shift; env "$@" timeout 300 python bench.py --workload $w --no-cpu-baseline --no-probe-mode --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['roofline']['kernel_ms_per_launch'],3), round(d['e2e']['value']/1e6,2))"; }
timeout 600 python -m pytest tests/test_gpu_grid.py tests/test_gpu_cache.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --workload kernels | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['table'], 'lookup', d['lookup']['ms'], d['lookup']['achieved_gbs'], d['lookup']['frac'], 'evict', d['evict']['ms'], d['evict']['achieved_gbs'], d['evict']['frac'], d['evict']['grid_ctas'])
"
for i in 1 2; do run cur c4 X=1; run evl c4 KVG_LIB=var_libs/libkvgpu_evloop.so; done
