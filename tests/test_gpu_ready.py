"""The ready-set walk (dispatch_batch's sorted ready vector, engine.cpp:306-310)
in both device forms — the sweep kernel's and the one-CTA-per-SM kernels'
four-words-at-a-time second level — against numpy, over bitmaps the size of
the full C5 run (65,536 agents) that the reference cannot finish here."""
import ctypes as C

import numpy as np
import pytest

from paper_2601_22705_b200 import engine

pytestmark = pytest.mark.gpu
NIL = 0xFFFFFFFF


def _walk(ready: np.ndarray, queries: np.ndarray):
    n = len(ready)
    nw = (n + 31) // 32
    bits = np.zeros(nw * 32, dtype=np.uint64)
    bits[:n] = ready
    rbits = (bits.reshape(nw, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
    n1 = (nw + 31) // 32
    w1 = np.zeros(n1 * 32, dtype=np.uint64)
    w1[:nw] = rbits != 0
    rl1 = (w1.reshape(n1, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
    q = queries.astype(np.uint32)
    on = np.zeros(len(q), dtype=np.uint32)
    ow = np.zeros(len(q), dtype=np.uint32)
    P = C.POINTER(C.c_uint32)
    lib = engine.lib()
    lib.kvg_check_ready_next.argtypes = [C.c_int, P, P, C.c_uint32, P, C.c_uint32, P, P]
    assert lib.kvg_check_ready_next(0, rbits.ctypes.data_as(P), rl1.ctypes.data_as(P), n,
                                    q.ctypes.data_as(P), len(q), on.ctypes.data_as(P),
                                    ow.ctypes.data_as(P)) == 0
    # expected: the smallest ready id >= from
    idx = np.flatnonzero(ready)
    pos = np.searchsorted(idx, q)
    if len(idx) == 0:
        want = np.full(len(q), NIL, dtype=np.uint32)
    else:
        want = np.where(pos < len(idx), idx[np.minimum(pos, len(idx) - 1)], NIL).astype(np.uint32)
    want[q >= n] = NIL
    return on, ow, want


@pytest.mark.parametrize("n", [65536, 8197, 100003, 1024, 70])
@pytest.mark.parametrize("density", [0.0, 1e-5, 1e-3, 0.05, 0.9])
def test_ready_walk_both_forms(n, density):
    rng = np.random.default_rng(n + int(density * 1e6))
    ready = rng.random(n) < density
    if density == 1e-5:  # one ready agent at the far end: the longest walk
        ready[:] = False
        ready[n - 1] = True
    q = np.concatenate([np.arange(0, n, max(1, n // 4096)), rng.integers(0, n + 40, 2000)])
    on, ow, want = _walk(ready, q)
    assert (on == want).all()
    assert (ow == want).all()
