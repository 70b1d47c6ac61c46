set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
tail -n 3 gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cat gpurun_out/bench_c4.json
timeout 300 python bench.py --impl reference > gpurun_out/bench_c4_ref.json 2>&1
cat gpurun_out/bench_c4_ref.json
