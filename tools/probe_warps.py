"""Dev probe: device time of one big simulation vs warps per CTA."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2601_22705_b200 import config, engine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = {"c2": lambda: config.c2_qwen("aimd"),
     "c3": lambda: config.c3_dsv3("aimd")}[which[:2]]()
if which == "c3":
    s.controller.h_thresh = 0.3
spec = engine.SimSpec.from_scenario(s)
for w in [1, 2, 4, 8, 16, 32]:
    b = engine.Batch([spec], warps_per_sim=w)
    b.run()
    b.run()
    print(which, "warps", w, "kernel ms", round(b.timing()[1], 1), "makespan", b.result(0)["makespan"],
          flush=True)
    b.close()
