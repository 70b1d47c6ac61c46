"""Device-backed admission controllers against the
reference's own standalone controller ABI (kva_controller_*, kvadmit.h:86-159,
capi.cpp:172-292, built unmodified into oracle/_ref/libkvref.so).

Seeded random programs drive many controllers at once — every policy kind,
smoothing on/off, pauses (agent_cap / AIMD shrink), request-cap re-queues,
unknown-agent misuse — and require identical windows (bit for bit), command
lists per admission pass, per-event statuses, set sizes and active order."""
import ctypes as C
import random

import pytest

from paper_2601_22705_b200 import abi, config, engine
from tests.helpers import ref_lib


class RefCtl:
    """One reference controller through kva_controller_* (the unmodified ABI)."""

    def __init__(self, policy_text, cfg, total):
        lib = ref_lib()
        lib.kva_controller_create.argtypes = [C.c_char_p, C.POINTER(abi.ControllerConfig * 1),
                                              C.c_uint32, C.POINTER(C.c_void_p)]
        self.lib, self.total = lib, total
        # kva_controller_config is ControllerConfig without control_interval
        raw = (C.c_double * 9)(cfg.alpha, cfg.beta, cfg.u_low, cfg.u_high, cfg.h_thresh,
                               cfg.w_min, cfg.w_max, cfg.initial_window, cfg.signal_smoothing)
        h = C.c_void_p()
        lib.kva_controller_create.argtypes = [C.c_char_p, C.c_void_p, C.c_uint32,
                                              C.POINTER(C.c_void_p)]
        assert lib.kva_controller_create(policy_text.encode(), C.cast(raw, C.c_void_p), total,
                                         C.byref(h)) == 0
        self.h = h
        for f in ("kva_controller_add_pending", "kva_controller_on_agent_finished",
                  "kva_controller_on_request_complete", "kva_controller_on_tool_return"):
            getattr(lib, f).argtypes = [C.c_void_p, C.c_uint32]
        lib.kva_controller_update_window.argtypes = [C.c_void_p, C.c_double, C.c_double,
                                                     C.POINTER(C.c_double)]
        lib.kva_controller_admission_pass.argtypes = [C.c_void_p, C.POINTER(C.c_uint8),
                                                      C.c_size_t, C.POINTER(abi.Command),
                                                      C.c_size_t, C.POINTER(C.c_size_t)]
        lib.kva_controller_counts.argtypes = [C.c_void_p] + [C.POINTER(C.c_size_t)] * 3
        lib.kva_controller_free.argtypes = [C.c_void_p]

    def update(self, u, h):
        w = C.c_double()
        assert self.lib.kva_controller_update_window(self.h, u, h, C.byref(w)) == 0
        return w.value

    def admission(self, bnd):
        """(status, commands); commands are empty when the call failed."""
        b = (C.c_uint8 * max(1, self.total))(*bnd)
        cmds = (abi.Command * max(1, self.total))()
        n = C.c_size_t()
        rc = self.lib.kva_controller_admission_pass(self.h, b, self.total, cmds, self.total,
                                                    C.byref(n))
        return rc, ([(cmds[k].kind, cmds[k].agent) for k in range(n.value)] if rc == 0 else [])

    def event(self, kind, agent):
        f = ["kva_controller_add_pending", "kva_controller_on_agent_finished",
             "kva_controller_on_request_complete", "kva_controller_on_tool_return"][kind]
        return getattr(self.lib, f)(self.h, agent)

    def counts(self):
        a, p, q = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self.lib.kva_controller_counts(self.h, C.byref(a), C.byref(p), C.byref(q))
        return a.value, p.value, q.value

    def free(self):
        self.lib.kva_controller_free(self.h)


def make_controllers(rng, n):
    out = []
    for i in range(n):
        total = rng.randint(1, 40)
        cfg = config.ControllerConfig(alpha=rng.choice([1.0, 2.0, 0.5]),
                                      beta=rng.choice([0.3, 0.5, 0.9]),
                                      u_low=rng.choice([0.1, 0.2]),
                                      u_high=rng.choice([0.4, 0.5, 0.8]),
                                      h_thresh=rng.choice([0.2, 0.5, 0.9]),
                                      w_max=rng.choice([0.0, 0.0, 8.0]),
                                      initial_window=rng.choice([0.0, 2.0]),
                                      signal_smoothing=rng.choice([0.0, 0.5]))
        text = rng.choice(["uncontrolled", "aimd", "aimd", f"agent_cap:{rng.randint(1, 6)}",
                           f"request_cap:{rng.randint(1, 6)}"])
        out.append((text, cfg, total))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_device_controllers_match_reference(seed):
    rng = random.Random(seed)
    specs = make_controllers(rng, 24)
    refs = [RefCtl(t, c, n) for t, c, n in specs]
    dev = engine.DeviceControllers([config.parse_policy(t, c) for t, c, _ in specs],
                                   [n for _, _, n in specs])
    try:
        for i, (_, _, n) in enumerate(specs):  # engine.cpp:89-93: every agent starts pending
            evs = [(i, abi.CTL_ADD_PENDING, a) for a in range(n)]
            assert dev.apply(evs) == [refs[i].event(0, a) for a in range(n)]
        for step in range(120):
            roll = rng.random()
            if roll < 0.35:
                u = [rng.random() for _ in specs]
                h = [rng.random() for _ in specs]
                got = dev.update_window(u, h)
                exp = [r.update(u[i], h[i]) for i, r in enumerate(refs)]
                assert [x.hex() for x in got] == [x.hex() for x in exp]
            elif roll < 0.7:
                bnd = [[int(rng.random() < 0.6) for _ in range(n)] for _, _, n in specs]
                st = []
                got = dev.admission_pass(bnd, st)
                exp = [r.admission(bnd[i]) for i, r in enumerate(refs)]
                assert [s_ != 0 for s_ in st] == [e[0] != 0 for e in exp]
                assert got == [e[1] for e in exp]
            else:
                evs = []
                for i, (_, _, n) in enumerate(specs):
                    for _ in range(rng.randint(0, 3)):
                        evs.append((i, rng.choice([1, 2, 3, 3]), rng.randrange(n)))
                rng.shuffle(evs)
                got = dev.apply(evs)
                exp = [refs[c].event(k, a) for c, k, a in evs]
                assert [g == 0 for g in got] == [e == 0 for e in exp]
            st = dev.state()
            assert [(s["active"], s["pending"], s["paused"]) for s in st] == \
                [r.counts() for r in refs]
        for i in range(len(specs)):
            assert len(dev.active(i)) == refs[i].counts()[0]
    finally:
        dev.close()
        for r in refs:
            r.free()


def test_invalid_policies_are_config_errors():
    bad = config.parse_policy("aimd", config.ControllerConfig(beta=1.5))
    with pytest.raises(engine.EngineError) as e:
        engine.DeviceControllers([bad], [4])
    assert e.value.status == abi.KVG_ERR_CONFIG and "beta" in str(e.value)
