run() { tag=$1; w=$2; shift; shift; env "$@" timeout 300 python bench.py --workload $w --no-cpu-baseline --no-probe-mode --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['roofline']['kernel_ms_per_launch'],3), round(d['e2e']['value']/1e6,2))"; }
for i in 1 2 3; do run head c4 KVG_LIB=var_libs/libkvgpu_head.so; run cur c4 X=1; done
