"""The CPU oracle pinned against the reference's own worked examples
(reference SPEC.md examples; recomputed in SURVEY.md Appendix B)."""
import ctypes as C
import json
import math
import os

import pytest

from harness import oracle, run_oracle
from paper_2411_05555_b200.abi import make_point
from configs import closed_form_point

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def P(**kw):
    return make_point(**kw)


def pf(p, lens):
    return oracle().kvo_prefill_latency(C.byref(p), sum(lens), sum(l * l for l in lens))


def dec(p, lens):
    return oracle().kvo_decode_step_latency(C.byref(p), len(lens), sum(lens))


def rel(a, b):
    return abs(a - b) / abs(b)


def test_kv_bytes_and_weights():
    L = oracle()
    assert L.kvo_kv_bytes_per_token(C.byref(P(model="llama2-70b"))) == 327680
    assert L.kvo_kv_bytes_per_token(C.byref(P(model="llama2-7b"))) == 524288
    assert L.kvo_kv_bytes_per_token(C.byref(P(model=(1.0, 1, 1, 1, 1, 1)))) == 2
    assert L.kvo_weight_bytes(C.byref(P(model="llama2-70b"))) == 1.4e11
    assert L.kvo_weight_bytes(C.byref(P(model="llama2-7b"))) == 1.4e10
    assert L.kvo_weight_bytes(C.byref(P(model=(1.0, 1, 1, 1, 1, 1)))) == 1.0


def test_prefill_examples():
    g = GOLD["prefill"]
    h = P(model="llama2-70b", device="h100", eff=(0.5, 0.8, 0.8))
    assert rel(pf(h, [512]), g["h100_512_s"]) < 1e-12
    assert rel(pf(h, [512]), 0.0366) < 2e-3          # SPEC "36.6 ms"
    a = P(model="llama2-70b", device="910b2", eff=(0.5, 0.8, 0.8))
    assert rel(pf(a, [1000]), g["910b2_1000_s"]) < 1e-12
    assert rel(pf(a, [1000]), 0.1783) < 1e-3         # SPEC "178.3 ms"
    h1 = P(model="llama2-70b", device="h100", eff=(1.0, 0.8, 0.8))
    assert pf(h, [700]) == 2 * pf(h1, [700])          # exact 2x in efficiency
    assert rel(pf(h, [512, 512]), 2 * pf(h, [512])) < 1e-15  # additivity


def test_decode_examples():
    g = GOLD["decode"]
    h = P(model="llama2-70b", device="h100", eff=(1.0, 1.0, 1.0))
    assert rel(dec(h, [500] * 32), g["h100_32x500_s"]) < 1e-12
    assert rel(dec(h, [500] * 32), 0.01084) < 1e-3
    assert rel(dec(h, [500]), 0.01046) < 1e-3
    a = P(model="llama2-70b", device="910b2", eff=(1.0, 1.0, 1.0))
    assert rel(dec(a, [100]), 0.01945) < 1e-3
    # tokens/s at batch 1 and 32: 95.6 and 2952
    assert abs(1 / dec(h, [500]) - 95.6) < 0.1
    assert abs(32 / dec(h, [500] * 32) - 2952) < 1.0


def test_transfer_examples():
    L = oracle()
    h = P(device="h100", eff=(0.5, 1.0, 1.0))
    hs = P(device="h100", eff=(0.5, 1.0, 1.0), link="single")
    a = P(device="910b2", eff=(0.5, 1.0, 1.0), link="single")
    assert rel(L.kvo_transfer_latency(C.byref(h), 327.68e6), 91.0e-6) < 1e-3
    assert rel(L.kvo_transfer_latency(C.byref(hs), 327.68e6), 0.364e-3) < 1e-3
    assert rel(L.kvo_transfer_latency(C.byref(a), 327.68e6), 0.836e-3) < 1e-3
    assert L.kvo_transfer_latency(C.byref(h), 0.0) == 0.0
    assert rel(L.kvo_transfer_latency(C.byref(h), 4096 * 1000), 1.1378e-6) < 1e-4


def test_capacity_examples():
    L = oracle()
    out = C.c_int64()
    assert L.kvo_kv_capacity_tokens(C.byref(P(model="llama2-70b", device="h100")), C.byref(out)) == 0
    assert out.value == 451660
    L.kvo_kv_capacity_tokens(C.byref(P(model="llama2-70b", device="910b2")), C.byref(out))
    assert out.value == 275878
    L.kvo_kv_capacity_tokens(C.byref(P(model="llama2-7b", device="h100")), C.byref(out))
    assert out.value == GOLD["capacity"]["7b_h100"]
    p = P(model=(1e9, 1, 1, 1, 1, 1), device=(1e12, 1e9 / 0.9 / 4 * 1.0, 1e12, 1e9))
    assert L.kvo_kv_capacity_tokens(C.byref(p), C.byref(out)) == 0 and out.value == 0  # boundary
    p = P(model="llama2-70b", device=(1e12, 10e9, 1e12, 1e9))
    assert L.kvo_kv_capacity_tokens(C.byref(p), C.byref(out)) == -2  # "model does not fit"


def test_imbalance_closed_form():  # SPEC.md:462 acceptance #4
    h = P(model="llama2-70b", device="h100", eff=(0.5, 0.8, 0.8))
    kvb = 327680
    for L_, want in ((250, 0.15284e-3), (500, 0.30567e-3), (1000, 0.61134e-3)):
        d = dec(h, [L_] * 40) - dec(h, [L_] * 20)
        closed = 20 * L_ * kvb / (4 * 3.35e12 * 0.8)
        assert rel(d, closed) < 1e-9 and rel(d, want) < 1e-4


def test_unified_cobatch_inflation():
    a = P(model="llama2-70b", device="910b2", eff=(0.5, 1.0, 1.0))
    step = pf(a, [1000]) + dec(a, [500] * 20)
    assert rel(step, 0.198176) < 1e-5 and rel(dec(a, [500] * 20), 0.019900) < 1e-4
    assert step > 4 * dec(a, [500] * 20)  # ">300%" inflation


def test_single_request_closed_form():  # SPEC.md:225, 369, 459 acceptance #1 (P-X1: 9 decode steps)
    p = closed_form_point()
    r = run_oracle(p, ev_cap=0)
    rec = r.recs[0]
    ttft = pf(p, [512])
    jct = ttft
    for i in range(9):
        jct += dec(p, [512 + i])
    assert rel(rec.first_token_s - rec.arrival_s, ttft) < 1e-9
    assert rel(rec.completion_s - rec.arrival_s, jct) < 1e-9
    assert rel(ttft, 0.03658604) < 1e-6 and rel(jct, 0.13072946) < 1e-6
    s = r.summary
    assert s.tokens_total == 10 and s.n_completed == 1
    assert math.isclose(s.tbt_mean, (jct - ttft) / 9, rel_tol=1e-12)


def test_mirror_bytes_ledger():  # SPEC.md:244, 466 acceptance #8: per-step mirror bytes = batch x kvb
    p = make_point(model="llama2-70b", policy="accellm", instances=2, num_requests=32, rate=1e9,
                   prompt=100, decode=20, arrival="fixed", seed=0)
    r = run_oracle(p, ev_cap=100000)
    steps = {}
    for e in r.events:
        if e.kind == 4:
            steps[(e.t, e.inst)] = e.a
    mirrors = [e for e in r.events if e.kind == 10 and e.b == 1]
    assert mirrors and r.summary.link_mirror_tokens == sum(e.c for e in mirrors)
    assert r.summary.link_mirror_gb == r.summary.link_mirror_tokens * 327680 / 1e9


def test_rebalance_spec_example():
    """A={1000,1000,100,100}, B={} -> 2/2 with 1100/1100 (greedy rule, SEMANTICS §6)."""
    def greedy(a, b):
        c = len(a) - len(b)
        d = sum(a) - sum(b)
        moved = []
        for k in sorted(a, reverse=True):
            v, D = max(0, abs(c) - 1), abs(d)
            c2, d2 = c - 2, d - 2 * k
            v2, D2 = max(0, abs(c2) - 1), abs(d2)
            if v2 <= v and D2 <= D and (v2 < v or D2 < D):
                moved.append(k)
                c, d = c2, d2
        rest = list(a)
        for k in moved:
            rest.remove(k)
        return rest, list(b) + moved
    a, b = greedy([1000, 1000, 100, 100], [])
    assert sorted(a) == [100, 1000] and sorted(b) == [100, 1000]
    assert greedy([5, 5, 5, 5, 5, 5], [5, 5, 5, 5, 5, 5]) == ([5] * 6, [5] * 6)  # fixed point
    a, b = greedy([10] * 11, [10] * 9)  # 9 vs 11 -> 10 vs 10
    assert len(a) == 10 and len(b) == 10


def test_determinism():  # SPEC.md:227 byte-identical reruns
    p = make_point(policy="accellm", instances=4, num_requests=300, rate=6.0, seed=7)
    a = run_oracle(p, ev_cap=0)
    b = run_oracle(p, ev_cap=0)
    assert bytes(a.summary) == bytes(b.summary)
    assert all(bytes(x) == bytes(y) for x, y in zip(a.recs, b.recs))


def test_first_token_from_decode_flag_closed_form():
    """SPEC.md:273 alternative (first_token_decode): the prefill emits no
    token, decode_len tokens take decode_len decode steps. On the single
    request it reproduces SPEC.md:225's engine example literally:
    JCT = 36.6 ms + sum_{i=0..9} decode_step_latency([512+i]) ~ 141.3 ms."""
    import ctypes as C
    from configs import closed_form_point
    from harness import oracle, run_oracle
    L = oracle()
    p = closed_form_point()
    p.first_token_decode = 1
    r = run_oracle(p, ev_cap=0)
    q = r.recs[0]
    pf = L.kvo_prefill_latency(C.byref(p), 512, 512 * 512)
    dec = [L.kvo_decode_step_latency(C.byref(p), 1, 512 + i) for i in range(10)]
    assert abs((q.first_token_s - q.arrival_s) - (pf + dec[0])) <= 1e-9 * (pf + dec[0])
    jct = q.completion_s - q.arrival_s
    assert abs(jct - (pf + sum(dec))) <= 1e-9 * jct
    assert abs(jct - 0.1413) < 0.001 and r.summary.n_steps == 10 and r.summary.tokens_total == 10
