#!/bin/bash
# dev: ncu captures of the current kernels (run under gpurun from the repo root)
set -x
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:engine_kernel_small -c 1 -f -o gpurun_out/c4_chain \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-probe-mode --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1
timeout 600 $NCU -k regex:grid_match_kernel --launch-skip 6 -c 1 -f -o gpurun_out/match_c5 \
  python bench.py --workload kernels > gpurun_out/ncu_match.log 2>&1
timeout 600 $NCU -k regex:grid_evict_kernel --launch-skip 5 -c 1 -f -o gpurun_out/evict_c5 \
  python bench.py --workload kernels > gpurun_out/ncu_evict.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe-mode --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
