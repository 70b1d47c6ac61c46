# dev: kernels bench + grid-evict phase marks + C5 probe
KVG_LIB=var_libs/libkvgpu_gprof.so timeout 300 python tools/probe_grid.py
timeout 300 python bench.py --workload kernels | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); print(d['table'], 'lookup', d['lookup']['ms'], d['lookup']['achieved_gbs'], d['lookup']['frac'], 'evict', d['evict']['ms'], d['evict']['achieved_gbs'], d['evict']['frac'], d['evict']['grid_ctas'])
"
timeout 900 python tools/probe_c5.py aimd,agent_cap:256,agent_cap:1024,agent_cap:4096 1000000
