# dev: A/B of libkvgpu variants in var_libs/ on the C4 bench (usage: bash tools/ab_c4.sh "cur v1 v2" [workload] [rounds])
VS=${1:-cur}; W=${2:-c4}; R=${3:-2}
run() { tag=$1; w=$2; shift; shift; env "$@" timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-probe-mode --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag $w', round(d['roofline']['kernel_ms_per_launch'],3), round(d['e2e']['value']/1e6,2))"; }
for i in $(seq $R); do for v in $VS; do run $v $W KVG_LIB=var_libs/libkvgpu_$v.so; done; done
