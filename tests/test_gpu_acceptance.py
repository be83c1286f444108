"""SPEC acceptance criteria #3, #5-#10 on the B200: the same points as
tests/test_acceptance.py through the C-ABI; every summary (and instance
record) must equal the CPU oracle's bit for bit, and the criteria are then
evaluated on the GPU's own numbers."""
import pytest

import acceptance as A
from harness import Result, diff_results, oracle_sweep, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    import paper_2411_05555_b200 as pkg
    s = pkg.KvSim(0)
    yield s
    s.close()


def gpu_run(sim, pts, detail=False, instances=False):
    summ = sim.run(pts, detail=detail, instances=instances)
    ref, ref_inst = oracle_sweep(pts, detail=detail, instances=instances)
    inst = sim.last_instances if instances else None
    bad = []
    for i, (a, b) in enumerate(zip(ref, summ)):
        d = diff_results(Result(a, None, None, inst=ref_inst[i] if instances else None),
                         Result(b, None, None, inst=inst[i] if instances else None), events=False)
        if d:
            bad.append((i, d[:3]))
    assert not bad, bad
    return summ, inst


def test_gpu_a3(sim):
    pts = A.a3_points()
    s, _ = gpu_run(sim, pts, detail=True)
    r = A.a3_eval(pts, s)
    assert r["holds_unified"] and r["holds_accellm_handoff_bound"] and r["holds_no_prefill_interference"]


def test_gpu_a5_a6_a7(sim):
    pts = A.a5_points()
    s, _ = gpu_run(sim, pts)
    r = A.a5_eval(pts, s)
    assert r["holds_jct"] and r["holds_ce_vs_splitwise"] and r["holds_offered_bound"]
    assert r["holds_ttft"] and r["holds_queue_wait"] and r["holds_idle_accellm"]
    pts = A.a7_points()
    s, inst = gpu_run(sim, pts, instances=True)
    assert A.a7_eval(pts, s, inst)["holds_prefill_idle"]


def test_gpu_a8_event_logs(sim):
    pts = A.a8_points()[:3]
    summ, recs, evs = sim.run(pts, records=False, events=1 << 22)
    for p, s, ev in zip(pts, summ, evs):
        ref = run_oracle(p, ev_cap=1 << 22, recs=False, inst=False)
        assert not diff_results(ref, Result(s, None, ev, ev_total=len(ev)))
    assert A.a8_eval(pts, [run_oracle(p, ev_cap=1 << 22, recs=False, inst=False).events for p in pts])[
        "holds_mirror_bw"]


def test_gpu_a9_a10(sim):
    pts = A.a9_points()
    s, _ = gpu_run(sim, pts)
    r = A.a9_eval(pts, s)
    assert r["holds_positive"] and r["holds_monotone"] and r["holds_under_capacity"]
    pts = A.a10_points()
    s, _ = gpu_run(sim, pts)
    r = A.a10_eval(pts, s)
    assert r["holds_within_25pct_low_rate"] and r["holds_within_2x"]
