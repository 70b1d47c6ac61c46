"""Dev probe: big-sim kernel time vs warps per simulation (C2, C3 h=0.3)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

for name in ("c2", "c3"):
    if name == "c2":
        s = config.c2_qwen("aimd")
    else:
        s = config.c3_dsv3("aimd")
        s.controller.h_thresh = 0.3
    spec = engine.SimSpec.from_scenario(s)
    for w in (4, 8, 16, 32):
        b = engine.Batch([spec], warps_per_sim=w)
        ks = []
        for _ in range(3):
            b.run()
            ks.append(b.timing()[1])
        print(name, "warps", w, "kernel ms", [round(k, 1) for k in ks], flush=True)
        b.close()
