"""Stall storms (leader.cuh coop_storm): runs of dispatch attempts that all
stall are evaluated 32 at a time on the warp. The per-member path is the
reference-pinned one (every golden case, the thrash preset's 17K stalls with
event logs against the oracle); here big overcommitted C5-shape runs —
thousands of agents, sparse ready bitmaps, millions of stalls — must come out
identical with the warp path on and off (KVG_NO_STORM=1)."""
import os

import numpy as np
import pytest

from paper_2601_22705_b200 import config, engine

pytestmark = pytest.mark.gpu


def _run(s, storm: bool):
    old = os.environ.get("KVG_NO_STORM")
    os.environ["KVG_NO_STORM"] = "0" if storm else "1"
    try:
        b = engine.Batch([engine.SimSpec.from_scenario(s)], verify=False, host_outputs=True)
        b.run()
        res, stats, rows = b.outputs()
        out = (res.copy(), stats[0].copy(), rows[0].copy())
        b.close()
        return out
    finally:
        if old is None:
            del os.environ["KVG_NO_STORM"]
        else:
            os.environ["KVG_NO_STORM"] = old


# (an uncontrolled run whose cache holds little more than the shared prompt:
# every dispatch after the first stalls; an agent-capped run over 4x as many
# agents: ready agents sparse in the bitmap, the gather spans many words)
@pytest.mark.parametrize("agents,policy,capacity,horizon",
                         [(8192, "uncontrolled", 4000, 60.0), (16384, "agent_cap:4096", 20000, 150.0)])
def test_storm_path_equals_per_member_path(agents, policy, capacity, horizon):
    s = config.c5_stress(policy, agents=agents, capacity=capacity)
    s.engine.horizon = horizon
    ra, sa, ta = _run(s, True)
    rb, sb, tb = _run(s, False)
    assert int(ra["stall_events"][0]) > 10_000  # a real storm
    for f in ra.dtype.names:
        if f != "device_cycles":
            assert np.array_equal(ra[f], rb[f]), f
    assert sa.tobytes() == sb.tobytes()
    assert ta.tobytes() == tb.tobytes()
