"""dev probe: phase timestamps of the grid eviction on the C5-size table
(needs tools/build_variant.sh gprof -DKVG_GRID_PROF; KVG_LIB=var_libs/libkvgpu_gprof.so)."""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench_kernels  # noqa: E402
from paper_2601_22705_b200 import abi, config, engine  # noqa: E402

ctx, prompt, shared = bench_kernels.final_contexts(config.c5_stress("aimd"))
cap, ps = 16777216, 16
S = prompt // ps
used, fill = 0, []
for a in range(len(ctx)):
    need = int(ctx[a] // ps) - (S if fill else 0)
    if used + need > cap:
        break
    used += need
    fill.append(a)
c = engine.DeviceCache(cap, ps, prompt, shared, max_agents=len(ctx))
c.configure(0, record_victims=False)
for i in range(0, len(fill), 512):
    c.execute([(abi.OP_INSERT, a, int(ctx[a]), 0) for a in fill[i:i + 512]])
lib = engine.lib()
buf = (C.c_ulonglong * 32)()
for rep in range(4):
    out = c.execute([(abi.OP_EVICT, 0, 0, cap // 100)])[0]
    ms, blocks = c.last_ms()
    lib.kvg_debug_gprof(buf)
    t0 = buf[0]
    marks = {k: (buf[k] - t0) / 1e3 for k in list(range(1, 17)) + [30] if buf[k] >= t0 and buf[k]}
    print(f"rep {rep}: {ms * 1e3:.1f} us, ctas {blocks}, freed {out['r0']}:",
          " ".join(f"{k}:{v:.1f}" for k, v in marks.items()), flush=True)
