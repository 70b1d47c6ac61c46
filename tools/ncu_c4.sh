#!/bin/bash
# dev: ncu capture of the C4 engine kernel + the launch list (run under gpurun from the repo root)
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:engine_kernel_small -c 1 -f -o gpurun_out/c4_chain \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-probe-mode --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-probe-mode --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
