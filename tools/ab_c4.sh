run() { tag=$1; w=$2; shift; shift; env "$@" timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['ms_per_step'],3), round(d['e2e']['value'],2), (d.get('probe_mode') or {}).get('ms_per_step'))"; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do for w in c2 c4; do run shist $w KVG_LIB=var_libs/libkvgpu_shist.so; run mid $w KVG_LIB=var_libs/libkvgpu_mid.so; done; done
