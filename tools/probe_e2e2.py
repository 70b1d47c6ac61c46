"""dev probe: which part of bench.py's sequence slows the e2e kernel."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2601_22705_b200 import config, engine
pop = engine.Population(config.c1_toy().workload, 42)
specs = [engine.SimSpec.from_scenario(s, population=pop) for s in config.c4_sweep()]

def e2e(tag):
    for it in range(2):
        torch.cuda.synchronize()
        b = engine.Batch(specs, verify=False, host_outputs=True)
        b.run(); k = b.timing()[1]
        r = b.results_array()
        b.close()
        print(f"{tag} it={it} e2e kernel {k:.2f}", flush=True)

e2e("fresh")
b = engine.Batch(specs, verify=False)
for _ in range(3): b.run()
print("device batch kernel", round(b.timing()[1], 2))
e2e("after device batch (open)")
b.close()
e2e("after device batch (closed)")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); flush.fill_(1); torch.cuda.synchronize()
e2e("after torch flush alloc")
pb = engine.Batch(specs, verify=True); pb.run(); pb.close()
e2e("after verify batch")
