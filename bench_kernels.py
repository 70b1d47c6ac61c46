"""Page-table kernels in isolation (`python bench.py --workload kernels`):
kernel 1 (batched block-hash prefix lookup, kvg_cache_match_batch) and kernel 2
(eviction radix select + scatter, kvg_cache_exec EVICT on the grid path) on
C2-size (2,038,926 pages) and C5-size (16,777,216 pages) prefix caches
(SURVEY.md §8(d)), against the HBM roofline.

Table contents: the config's population (C2: Qwen3-32B seed 7, 1,024 agents,
shared 4,096-token prompt; C5: seed 5, 65,536 agents, shared 8,192-token
prompt), each agent's FINAL context inserted in agent order until the next one
would not fit (so the cache is full of complete paths, no eviction during the
fill). Then, timed on the device with CUDA events around the kernels only:
  lookup  one match_prefix per agent (all agents, final contexts) as one batch;
  evict   evict(1% of capacity), repeated on the shrinking table.
Algorithmic bytes: lookup 16 B per counted lookup (resolved
pages + the terminating miss) + 8 B per hit page; eviction 8 B per resident
page per select + 16 B per victim. The table itself is 16 B/page slots in
512 B buckets plus 32 B bucket summaries; the select streams summaries, so its
DRAM traffic is below its algorithmic bytes by design (ncu: profiles/).
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")

PLAN_DT = np.dtype([("gen", "<u8"), ("obs", "<u8"), ("tool", "<f8"), ("has_tool", "<u4"),
                    ("pad", "<u4")])


def final_contexts(scenario):
    from paper_2601_22705_b200 import engine
    pop = engine.Population(scenario.workload, scenario.seed)
    plans = pop.plans().view(PLAN_DT).reshape(pop.c.agents, pop.c.steps)
    ctx = pop.c.prompt_tokens + (plans["gen"] + plans["obs"]).sum(axis=1)
    return ctx.astype(np.uint64), int(pop.c.prompt_tokens), bool(pop.c.shared_prompt)


def hbm_peak():
    try:
        p = json.load(open(PEAKS))
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


def run_table(name, scenario, capacity, reps=5, evict_frac=0.01):
    from paper_2601_22705_b200 import abi, engine
    ctx, prompt, shared = final_contexts(scenario)
    ps = int(scenario.engine.page_size)
    S = prompt // ps if shared else 0
    n_agents = len(ctx)
    pages = ctx // ps
    # fill: whole final contexts in agent order while they fit
    used = 0
    fill = []
    for a in range(n_agents):
        need = int(pages[a]) - (S if (shared and fill) else 0)
        if used + need > capacity:
            break
        used += need
        fill.append(a)
    c = engine.DeviceCache(capacity, ps, prompt, shared, max_agents=n_agents)
    c.configure(0, record_victims=False)
    t0 = time.perf_counter()
    for i in range(0, len(fill), 512):
        c.execute([(abi.OP_INSERT, a, int(ctx[a]), 0) for a in fill[i:i + 512]])
    fill_s = time.perf_counter() - t0
    agents = np.arange(n_agents, dtype=np.uint32)
    lens = ctx.astype(np.uint64)
    # lookup: warm-up then timed reps
    c.match_batch(agents, lens)
    lk_ms = []
    res = None
    for _ in range(reps):
        res = c.match_batch(agents, lens)
        lk_ms.append(c.last_ms()[0])
    hit_pages = sum(r["r0"] for r in res) // ps
    n_pages = (lens // ps).astype(np.int64)
    f = np.array([r["r0"] // ps for r in res], dtype=np.int64)
    lookups = int((f + (f < n_pages)).sum())
    lk_bytes = 16 * lookups + 8 * hit_pages
    # eviction: evict(1% of capacity) repeatedly
    k = max(1, int(capacity * evict_frac))
    ev_ms, ev_bytes, blocks = [], [], 0
    for _ in range(reps):
        out = c.execute([(abi.OP_EVICT, 0, 0, k)])[0]
        ms, blocks = c.last_ms()
        ev_ms.append(ms)
        ev_bytes.append(8 * (out["used"] + out["r0"]) + 16 * out["r0"])
    c.close()
    lk_med = float(np.median(lk_ms))
    ev_med = float(np.median(ev_ms))
    peak, peak_src = hbm_peak()
    lk_gbs = lk_bytes / (lk_med * 1e-3) / 1e9
    ev_gbs = float(np.median(ev_bytes)) / (ev_med * 1e-3) / 1e9
    return {
        "table": name, "capacity_pages": capacity, "resident_pages": used,
        "agents_resident": len(fill), "agents": n_agents, "fill_s": round(fill_s, 2),
        "lookup": {"kernel": "grid_match_kernel + grid_match_shared_kernel", "queries": n_agents,
                   "counted_lookups": lookups, "hit_pages": int(hit_pages),
                   "ms": round(lk_med, 4), "lookups_per_s": lookups / (lk_med * 1e-3),
                   "algorithmic_bytes": lk_bytes, "achieved_gbs": round(lk_gbs, 1),
                   "frac": round(lk_gbs / peak, 3)},
        "evict": {"kernel": "grid_evict_kernel", "needed": k, "grid_ctas": blocks,
                  "ms": round(ev_med, 4), "algorithmic_bytes": int(np.median(ev_bytes)),
                  "achieved_gbs": round(ev_gbs, 1), "frac": round(ev_gbs / peak, 3)},
        "peak_gbs": peak, "peak_source": peak_src,
    }


def main(args):
    from paper_2601_22705_b200 import config
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tables = [("C2", config.c2_qwen("aimd"), 2038926), ("C5", config.c5_stress("aimd"), 16777216)]
    lines = []
    for name, scen, cap in tables:
        r = run_table(name, scen, cap)
        lines.append(r)
        print(json.dumps({"metric": "page-table kernels: prefix lookups/s and eviction "
                                    "select GB/s vs HBM roofline", "workload": "kernels",
                          "unit": "GB/s", "dtype": "u64", "data": "synthetic", **r}),
              flush=True)
    return lines
