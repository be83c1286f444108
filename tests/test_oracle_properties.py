"""Oracle properties from the reference's invariant lists: workload generator
statistics, the portable log, and the randomized invariant
suite of acceptance criterion #11 (memory safety, ledger
exactness, token-time monotonicity, conservation, determinism) over
randomized small configurations, half of them memory-starved."""
import ctypes as C
import math
import struct

import numpy as np
import pytest

from configs import random_small
from harness import oracle, run_oracle
from paper_2411_05555_b200.abi import make_point


def gen(p, cap):
    L = oracle()
    a = (C.c_double * cap)()
    pr = (C.c_int32 * cap)()
    de = (C.c_int32 * cap)()
    n = L.kvo_gen_trace(C.byref(p), a, pr, de, cap)
    return np.frombuffer(a, dtype=np.float64)[:n].copy(), np.frombuffer(pr, dtype=np.int32)[:n].copy(), \
        np.frombuffer(de, dtype=np.int32)[:n].copy()


def test_lengths_uniform_and_in_range():
    p = make_point(workload="mixed", rate=8.0, num_requests=100000, seed=5)
    _, pr, de = gen(p, 100000)
    for x in (pr, de):
        assert x.min() >= 20 and x.max() <= 1000
        assert abs(x.mean() - 510.0) < 0.01 * 510               # exact uniform mean of 20..1000
        counts = np.bincount(x - 20, minlength=981)
        exp = len(x) / 981
        chi2 = ((counts - exp) ** 2 / exp).sum()
        assert chi2 < 981 + 5 * math.sqrt(2 * 981)              # ~5 sigma of chi2(980)


def test_mixed_preset_mean_prompt():  # rate 8, duration 1000 s -> mean within 5% of 500
    p = make_point(workload="mixed", rate=8.0, num_requests=20000, duration_s=1000.0, seed=9)
    arr, pr, _ = gen(p, 20000)
    assert len(arr) >= 7600 and arr.max() < 1000.0
    assert 475 <= pr.mean() <= 525


def test_poisson_gaps():  # mean gap within 5% of 1/rate over >= 1e4 arrivals
    for rate in (0.5, 3.0, 40.0):
        p = make_point(rate=rate, num_requests=20000, seed=1)
        arr, _, _ = gen(p, 20000)
        gaps = np.diff(np.concatenate([[0.0], arr]))
        assert np.all(gaps >= 0) and np.all(np.diff(arr) >= 0)
        assert abs(gaps.mean() * rate - 1.0) < 0.05
        assert abs(gaps.std() * rate - 1.0) < 0.05               # exponential: sd = mean


def test_rate_zero_and_fixed_interval():
    assert len(gen(make_point(rate=0.0, num_requests=10), 10)[0]) == 0
    arr, _, _ = gen(make_point(rate=4.0, num_requests=9, arrival="fixed"), 9)
    assert list(arr) == [i / 4.0 for i in range(9)]


def test_generator_deterministic():
    p = make_point(rate=3.0, num_requests=5000, seed=77)
    a1, p1, d1 = gen(p, 5000)
    a2, p2, d2 = gen(p, 5000)
    assert a1.tobytes() == a2.tobytes() and p1.tobytes() == p2.tobytes() and d1.tobytes() == d2.tobytes()
    q = make_point(rate=3.0, num_requests=5000, seed=78)
    assert gen(q, 5000)[0].tobytes() != a1.tobytes()


def ulp_diff(a, b):
    ia = struct.unpack("<q", struct.pack("<d", a))[0]
    ib = struct.unpack("<q", struct.pack("<d", b))[0]
    return abs(ia - ib)


def test_portable_log_accuracy():
    L = oracle()
    rng = np.random.default_rng(3)
    xs = list(rng.random(200000) + 1e-300) + [1.0, 0.5, 2.0 ** -53, 1 - 2.0 ** -53, 0.75, 1e-10]
    worst = max(ulp_diff(L.kvo_klog(float(x)), math.log(x)) for x in xs)
    assert worst <= 1
    assert L.kvo_klog(1.0) == 0.0


@pytest.mark.parametrize("chunk", range(4))
def test_randomized_invariant_suite(chunk):  # SPEC.md:469 acceptance #11
    L = oracle()
    L.kvo_set_invariant_checks(1)
    try:
        for i in range(chunk * 50, chunk * 50 + 50):
            p = random_small(i, max_req=50)
            r = run_oracle(p, ev_cap=0)
            s = r.summary
            assert r.status == 0, (i, r.status)                     # ledger / memory safety / time order
            assert s.n_completed == s.n_requests                    # every request completes
            assert s.tokens_total == sum(x.decode_len for x in r.recs)   # conservation
            for x in r.recs:
                assert x.first_token_s >= x.arrival_s and x.completion_s >= x.first_token_s
                if x.decode_len == 1:
                    assert x.completion_s == x.first_token_s and x.tbt_max_s == 0.0
            if p.policy != 2:
                assert s.n_moves == 0 and s.link_mirror_tokens == 0
            if p.policy == 0:
                assert s.link_prefill_tokens == 0                   # unified never uses links
            again = run_oracle(p, ev_cap=0)
            assert bytes(again.summary) == bytes(s)                 # determinism
    finally:
        L.kvo_set_invariant_checks(0)


def test_accellm_extensions_invariants():
    """Degraded mode + inter-pair leveling (SEMANTICS
    §6b): ledger exactness, memory safety and copy placement (copies only on
    the holder the partner relation names) after every event, conservation,
    determinism; and the mechanisms actually fire across the sample."""
    from configs import random_ext
    L = oracle()
    L.kvo_set_invariant_checks(1)
    modes = lvl = 0
    try:
        for i in range(120):
            p = random_ext(i)
            r = run_oracle(p, ev_cap=0)
            s = r.summary
            assert r.status == 0, (i, r.status)
            assert s.n_completed == s.n_requests
            assert s.tokens_total == sum(x.decode_len for x in r.recs)
            period = p.policy_timer_s or 1.0
            assert s.n_timer_ticks == 0 or s.makespan_s > period
            if s.makespan_s > 2 * period:
                assert s.n_timer_ticks > 0
            if not (p.accellm_flags & 1):
                assert s.n_mode_switches == 0
            if not (p.accellm_flags & 2):
                assert s.link_leveling_tokens == 0
            modes += s.n_mode_switches > 0
            lvl += s.link_leveling_tokens > 0
            assert bytes(run_oracle(p, ev_cap=0).summary) == bytes(s)
    finally:
        L.kvo_set_invariant_checks(0)
    assert modes >= 5 and lvl >= 5, (modes, lvl)


def test_extensions_off_is_plain_accellm():
    """With both flags off the timer never fires and results are the plain
    AcceLLM policy's; degraded mode in a memory-starved cluster serves more
    requests without recompute preemption."""
    base = make_point(policy="accellm", instances=4, rate=12.0, num_requests=3000, workload="heavy",
                      reserve=0.5, seed=3)
    s0 = run_oracle(base, recs=False).summary
    assert s0.n_timer_ticks == 0 and s0.n_mode_switches == 0
    deg = make_point(policy="accellm", instances=4, rate=12.0, num_requests=3000, workload="heavy",
                     reserve=0.5, seed=3, degraded=True)
    s1 = run_oracle(deg, recs=False).summary
    assert s1.n_mode_switches >= 1
    assert s1.n_preemptions < s0.n_preemptions
    assert s1.link_mirror_tokens < s0.link_mirror_tokens    # decoders stop mirroring most requests
