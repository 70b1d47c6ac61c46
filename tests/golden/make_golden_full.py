"""Full-size golden fixtures from the REFERENCE itself:
every simulation of the BASELINE C4 sweep (4,096 sims of C1 under the
controller grid, workload seed 42) and the full-size single-simulation
configurations the reference finishes in seconds.

Run in the build container (needs oracle/_ref/libkvref.so built from
/root/reference):
    python tests/golden/make_golden_full.py

  full_runs.json
    c4_seed42      4,096 per-simulation digests (tests/golden_hash.sim_digest:
                   result record + raw trace rows + agent stats)
    <case id>      one full-size run (tests/golden_cases.FULL_CASES): its result
                   record, trace row count and sim_digest
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2601_22705_b200 import config  # noqa: E402
from tests.golden_cases import FULL_CASES, full_case_scenario  # noqa: E402
from tests.golden_hash import result_record, sim_digest  # noqa: E402
from tests.helpers import ref_run_many_out  # noqa: E402


def main():
    out = {}
    path = os.path.join(HERE, "full_runs.json")
    if os.path.exists(path):
        out = json.load(open(path))
    t = time.time()
    runs = ref_run_many_out(config.c4_sweep(4096, seed=42))
    out["c4_seed42"] = [sim_digest(st, r, tr, ag) for st, r, tr, ag in runs]
    print("c4: 4096 sims", f"{time.time() - t:.1f} s")
    for case in FULL_CASES:
        if case["id"] in out and "--all" not in sys.argv:
            continue
        s, pol = full_case_scenario(case)
        s.policy = pol
        t = time.time()
        ((st, r, tr, ag),) = ref_run_many_out([s], threads=1)
        out[case["id"]] = dict(status=st, result=result_record(r), n_trace=len(tr),
                               digest=sim_digest(st, r, tr, ag))
        print(case["id"], st, r["makespan"], len(tr), f"{time.time() - t:.1f} s")
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
