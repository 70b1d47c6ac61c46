"""dev probe: e2e kernel with and without torch's CUDA context init."""
import os, sys, time
sys.path.insert(0, ".")
mode = sys.argv[1]
if mode == "torch":
    import torch
    torch.cuda.init(); torch.zeros(1, device="cuda")
elif mode == "torch_import":
    import torch
from paper_2601_22705_b200 import config, engine
pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]
for it in range(3):
    b = engine.Batch(specs, verify=False, host_outputs=True)
    b.run(); k = b.timing()[1]
    b.close()
    print(f"{mode} it={it} e2e kernel {k:.2f}", flush=True)
