# dev: one GPU call = tests + smoke + every bench line + ncu captures of the current kernels
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
tail -n 2 gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 1 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_c4_ref.json 2>&1
timeout 600 python bench.py --workload c5 --steps 2 --warmup 3 --e2e-steps 1 --no-pipeline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 --no-pipeline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-pipeline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c3off --steps 3 --warmup 3 --no-pipeline > gpurun_out/bench_c3off.json 2> gpurun_out/bench_c3off.err
timeout 300 python bench.py --workload kernels > gpurun_out/bench_kernels.json 2> gpurun_out/bench_kernels.err
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 $NCU -k regex:grid_match_kernel --launch-skip 6 -c 1 -f -o gpurun_out/match_c5 python bench.py --workload kernels > /dev/null 2>&1
timeout 300 $NCU -k regex:grid_match_rest_kernel --launch-skip 6 -c 1 -f -o gpurun_out/match_rest_c5 python bench.py --workload kernels > /dev/null 2>&1
timeout 300 $NCU -k regex:grid_evict_kernel --launch-skip 5 -c 1 -f -o gpurun_out/evict_c5 python bench.py --workload kernels > /dev/null 2>&1
timeout 600 $NCU -k regex:engine_kernel_small -c 1 -f -o gpurun_out/c4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-probe-mode --e2e-steps 1 --no-pipeline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-probe-mode --e2e-steps 1 --no-pipeline > /dev/null 2>&1
ls gpurun_out
