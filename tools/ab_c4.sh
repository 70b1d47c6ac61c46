run() { tag=$1; w=$2; shift; shift; env "$@" timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-probe-mode --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['ms_per_step'],3), round(d['e2e']['value'],2))"; }
for i in 1 2; do for v in cur ptxO2 ptxO1; do run $v c4 KVG_LIB=var_libs/libkvgpu_$v.so; done; done
for v in cur ptxO2; do run $v c3 KVG_LIB=var_libs/libkvgpu_$v.so; done
