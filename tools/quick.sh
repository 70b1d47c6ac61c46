timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_full_golden.py tests/test_gpu_golden.py -x -q -m gpu > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
KVG_LIB=var_libs/libkvgpu_gt.so python tools/probe_gtimer.py 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-probe-mode 2>&1 | tail -1
