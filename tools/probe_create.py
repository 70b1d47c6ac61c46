"""Dev probe: where the e2e batch-create time goes (C4 specs)."""
import ctypes as C
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import abi, config, engine  # noqa: E402

pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
lib = engine.lib()
for k in range(4):
    t0 = time.perf_counter()
    descs = (abi.SimDesc * len(specs)).from_buffer_copy(b"".join([sp.desc_bytes for sp in specs]))
    t1 = time.perf_counter()
    opt = abi.BatchOptions(host_outputs=1)
    h = C.c_void_p()
    lib.kvg_batch_create(0, descs, len(specs), C.byref(opt), C.byref(h))
    t2 = time.perf_counter()
    lib.kvg_batch_run(h)
    t3 = time.perf_counter()
    lib.kvg_batch_free(h)
    t4 = time.perf_counter()
    print(f"descs {1e3*(t1-t0):.2f} create {1e3*(t2-t1):.2f} run {1e3*(t3-t2):.2f} free {1e3*(t4-t3):.2f} ms")
