"""Grid-wide page-table kernels (csrc/grid.cuh) against the one-CTA seam they
replace for big tables, which the reference pins op for op (test_gpu_cache):

* grid_evict_kernel: every reference fuzz program (tests/golden/
  cache_fuzz.json) with each EVICT op forced onto the grid path must still
  produce the reference's ordered victim lists, clocks and pool usage;
* kvg_cache_match_batch: n match_prefix calls in one launch must leave the
  cache exactly as n KVG_OP_MATCH ops do — per-call results, clock, hit window,
  and every resident page's stamp (read back as the (key, stamp) victim list
  of evicting the whole cache, stamp order);
* both at table sizes where the grid path is the automatic choice."""
import json
import os
import random

import pytest

from paper_2601_22705_b200 import abi
from paper_2601_22705_b200 import engine
from tests.golden_hash import hx
from tests.helpers import GOLDEN

pytestmark = pytest.mark.gpu
PROGS = json.load(open(os.path.join(GOLDEN, "cache_fuzz.json")))
GRID_AUTO, GRID_NEVER, GRID_ALWAYS = 0, 1, 2
MATCH, INSERT, EVICT = abi.OP_MATCH, abi.OP_INSERT, abi.OP_EVICT


def _cache(prog, mode):
    c = engine.DeviceCache(prog["capacity"], prog["page_size"], prog["prompt"],
                           bool(prog["shared"]), max_agents=prog["agents"])
    c.configure(mode)
    return c


@pytest.mark.parametrize("k", range(len(PROGS)))
def test_grid_evict_on_reference_programs(k):
    prog = PROGS[k]
    c = _cache(prog, GRID_ALWAYS)
    try:
        out = c.execute([tuple(op) for op in prog["ops"]])
        for (kind, a, ln, arg), exp, got in zip(prog["ops"], prog["expect"], out):
            g = [got["status"], got["r0"], got["r1"], got["clock"], got["used"], got["victims"]]
            assert g == exp, (kind, a, ln, arg)
        m, r = c.hit_window()
        assert [hx(m), hx(r)] == prog["hit"]
    finally:
        c.close()


def _matches_equal(prog_prefix, queries, capacity, page_size, prompt, shared, agents):
    cs = engine.DeviceCache(capacity, page_size, prompt, shared, max_agents=agents)
    cb = engine.DeviceCache(capacity, page_size, prompt, shared, max_agents=agents)
    try:
        for c in (cs, cb):
            c.configure(GRID_NEVER)
            c.execute(prog_prefix)
        seq = cs.execute([(MATCH, a, ln, 0) for a, ln in queries])
        bat = cb.match_batch([a for a, _ in queries], [ln for _, ln in queries])
        assert [(x["status"], x["r0"], x["clock"], x["used"]) for x in seq] == \
            [(x["status"], x["r0"], x["clock"], x["used"]) for x in bat]
        assert [hx(v) for v in cs.hit_window()] == [hx(v) for v in cb.hit_window()]
        # every resident page's stamp: evict the whole cache, victims in
        # (stamp, deeper first) order carry their stamps
        a = cs.execute([(EVICT, 0, 0, capacity)])[0]
        b = cb.execute([(EVICT, 0, 0, capacity)])[0]
        assert a["r0"] == b["r0"] and a["victims"] == b["victims"]
        assert cs.victim_stamps(a) == cb.victim_stamps(b)
        return len(a["victims"])
    finally:
        cs.close()
        cb.close()


@pytest.mark.parametrize("k", [0, 3, 7, 11, 19, 23, 31, 39])
def test_match_batch_equals_sequential_on_reference_programs(k):
    prog = PROGS[k]
    ops = [tuple(op) for op in prog["ops"]]
    cut = len(ops) // 2
    rng = random.Random(k)
    seqs = {}
    for kind, a, ln, arg in ops[:cut]:
        if kind in (MATCH, INSERT):
            seqs[a] = max(seqs.get(a, 0), ln)
    queries = [(a, rng.randint(0, ln + 3 * prog["page_size"])) for a, ln in seqs.items()]
    queries += [(a, ln) for a, ln in list(seqs.items())[:3]]  # repeats: sub-batches
    rng.shuffle(queries)
    _matches_equal(ops[:cut], queries, prog["capacity"], prog["page_size"], prog["prompt"],
                   bool(prog["shared"]), prog["agents"])


def _big_fill(agents, ctx_pages, ps, prompt, shared, seed):
    rng = random.Random(seed)
    lens = [ctx_pages[0] * ps + rng.randrange(ctx_pages[1] * ps) for _ in range(agents)]
    return [(INSERT, a, lens[a], 0) for a in range(agents)], lens


@pytest.mark.parametrize("shared", [False, True])
def test_grid_kernels_on_a_big_table(shared):
    """~230K resident pages in 7K+ claimed buckets: EVICT goes grid-wide on
    its own (KVG_GRID_AUTO) and must pick the same victims as the one-CTA
    select; the match batch must equal the sequential matches."""
    ps, prompt, agents = 16, 4096, 160
    cap = 240_000
    fill, lens = _big_fill(agents, (1200, 800), ps, prompt, shared, 5)
    rng = random.Random(9)
    touches = [(MATCH, a, lens[a], 0) for a in rng.sample(range(agents), 60)]
    res = {}
    for mode in (GRID_NEVER, GRID_AUTO):
        c = engine.DeviceCache(cap, ps, prompt, shared, max_agents=agents)
        c.configure(mode)
        try:
            c.execute(fill + touches)
            out = c.execute([(EVICT, 0, 0, 37_000), (EVICT, 0, 0, 1), (EVICT, 0, 0, 90_000)])
            res[mode] = [(o["r0"], o["used"], o["clock"], o["victims"], c.victim_stamps(o))
                         for o in out]
            ms, blocks = c.last_ms()
            if mode == GRID_AUTO:
                assert blocks > 1  # the grid path ran
        finally:
            c.close()
    assert res[GRID_NEVER] == res[GRID_AUTO]
    queries = [(a, lens[a] - rng.randrange(3000)) for a in range(agents)]
    queries += [(a, lens[a]) for a in range(0, agents, 7)]
    n = _matches_equal(fill + touches, queries, cap, ps, prompt, shared, agents)
    assert n > 100_000
