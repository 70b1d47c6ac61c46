timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests_final.log 2>&1; tail -n 2 gpurun_out/tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_final.json; python -c "
import json; d=json.loads(open('gpurun_out/bench_final.json').read()); e=d['e2e']
print(round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), e['pipelined_ms_per_step'], round(e['serial']['value']/1e6,1), d['cpu_baseline']['value'], d['clocks'])"
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 2>/dev/null | tail -1
