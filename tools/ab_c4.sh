run() { tag=$1; w=$2; shift; shift; env "$@" timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-probe-mode --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['ms_per_step'],3), round(d['e2e']['value'],2))"; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do for w in c2 c3 c5; do run lonechain $w KVG_LIB=var_libs/libkvgpu_lonechain.so; run kchain $w KVG_LIB=var_libs/libkvgpu_kchain.so; done; done
