"""The product's host population builder (kvg_build_population) against the
reference build_population (workload.cpp:153-204): identical step plans, FNV
stream hash and peak aggregate for every BASELINE config (hashes from
SURVEY.md §8(c)), plus the live reference where oracle/_ref is present."""
import os

import numpy as np
import pytest

from paper_2601_22705_b200 import config, engine
from tests.helpers import REF_SO, ref_population

KNOWN = {  # SURVEY.md §8(c) workload hashes (reference, seeds 42/7/3/5)
    "c1": (config.c1_toy(), 0xa0ac2d3c3bc97b20),
    "c2": (config.c2_qwen(), 0x536abe2baf76b1d9),
    "c3": (config.c3_dsv3(), 0xbb838166f0edb99c),
    "c5": (config.c5_stress(), 0xf69286320625adc7),
}


@pytest.mark.parametrize("name", sorted(KNOWN))
def test_stream_hash_matches_reference(name):
    s, h = KNOWN[name]
    assert engine.Population(s.workload, s.seed).stream_hash == h


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_plans_bit_identical_to_reference(name):
    s, _ = KNOWN[name]
    pop = engine.Population(s.workload, s.seed)
    plans, n, h, sp, peak = ref_population(s)
    ref = np.frombuffer(bytes(plans), dtype=np.uint8)[: n * 32]
    assert (pop.plans() == ref).all()
    assert pop.peak_aggregate_tokens == peak
    assert pop.c.shared_prompt_tokens == sp


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_random_workloads_bit_identical():
    from tests.golden_cases import random_scenarios
    for _, s, _ in random_scenarios(24):
        pop = engine.Population(s.workload, s.seed)
        plans, n, h, sp, peak = ref_population(s)
        assert pop.stream_hash == h
        assert (pop.plans() == np.frombuffer(bytes(plans), dtype=np.uint8)[: n * 32]).all()


def test_bad_workload_is_config_error():
    s = config.c1_toy()
    s.workload.steps = 0
    with pytest.raises(engine.EngineError) as e:
        engine.Population(s.workload, 1)
    assert e.value.status == 1
