"""CPU CI for the kernel logic: the sm_100a simulation core
(csrc/kvsim_sim.cuh) compiled for the host SIMT emulator must reproduce the
independent CPU oracle bit for bit — summaries, per-request records and the
decision/event log — on the SPEC closed form, BASELINE config 1 and the
SPEC.md:469 randomized small-config suite (with memory-starved variants)."""
import os

import pytest

from configs import closed_form_point, config1, config2, config3, random_small
from harness import diff_results, run_oracle, run_points_emu

EV = 1 << 16


def check(points, ev=EV):
    got = run_points_emu(points, ev_cap=ev, warps=4)
    bad = []
    for p, g in zip(points, got):
        d = diff_results(run_oracle(p, ev_cap=ev), g)
        if d:
            bad.append((p.policy, p.num_instances, p.num_requests, d[:4]))
    assert not bad, bad


def test_closed_form_and_config1():
    check([closed_form_point(), config1(seed=0, n=120), config1(seed=1, n=120)])


@pytest.mark.parametrize("chunk", range(4))
def test_random_small_configs(chunk):
    check([random_small(i) for i in range(chunk * 25, chunk * 25 + 25)])


def test_config2_config3_small():
    pts = [config2(pol, 6.0, n=60) for pol in ("unified", "splitwise", "accellm")]
    pts += [config3(pol, 2.0, n=40) for pol in ("unified", "splitwise", "accellm")]
    check(pts)


def test_invalid_points_reported():
    from paper_2411_05555_b200.abi import make_point
    pts = [make_point(policy="accellm", instances=3, num_requests=5),
           make_point(policy="accellm", instances=2, num_requests=5, device=(1e12, 10e9, 1e12, 1e9))]
    got = run_points_emu(pts, ev_cap=0, recs=False)
    assert got[0].status == -3 and got[1].status == -2
    for p, g in zip(pts, got):
        assert run_oracle(p, ev_cap=0, recs=False).status == g.status


@pytest.mark.parametrize("chunk", range(3))
def test_accellm_extensions_random(chunk):
    """Degraded mode + inter-pair leveling (SEMANTICS §6b): kernel core ==
    oracle bit for bit, event logs included."""
    from configs import random_ext
    check([random_ext(i) for i in range(chunk * 40, chunk * 40 + 40)], ev=1 << 17)


def test_accellm_extensions_long():
    from configs import ext_long_points
    check(ext_long_points(n=400), ev=1 << 20)


@pytest.mark.parametrize("chunk", range(2))
def test_detail_metrics_random(chunk):
    """Detail runs (pooled TBT p50/p95 from per-step (gap, count) entries,
    plain event loop): kernel core == oracle bit for bit, including the
    per-instance records and the new v2 summary fields."""
    import math
    pts = [random_small(i) for i in range(chunk * 25, chunk * 25 + 25)]
    pts += [config1(seed=chunk, n=120), config2("accellm", 6.0, n=60), config2("unified", 6.0, n=60)]
    got = run_points_emu(pts, ev_cap=EV, warps=4, detail=True)
    bad = []
    for p, g in zip(pts, got):
        ref = run_oracle(p, ev_cap=EV, detail=True)
        d = diff_results(ref, g)
        if d:
            bad.append((p.policy, p.num_instances, p.num_requests, d[:4]))
        if g.status == 0 and g.summary.n_tbt_samples > 0:
            assert not math.isnan(g.summary.tbt_p50) and g.summary.tbt_p50 <= g.summary.tbt_p95 <= g.summary.tbt_max
    assert not bad, bad


@pytest.mark.parametrize("chunk", range(2))
def test_sweep_specialisation_no_log(chunk):
    """The sweep specialisation (no event log compiled in, the chained step
    loops the benchmark runs) against the oracle: summaries, per-request and
    per-instance records bit for bit."""
    pts = [random_small(i) for i in range(600 + chunk * 40, 640 + chunk * 40)]
    pts += [random_small(900 + i, max_req=300) for i in range(chunk * 10, chunk * 10 + 10)]
    pts += [config1(seed=5 + chunk, n=200), config2("accellm", 9.0, n=150), config2("unified", 9.0, n=150),
            config2("splitwise", 9.0, n=150)]
    got = run_points_emu(pts, ev_cap=0, warps=4)
    bad = []
    for p, g in zip(pts, got):
        d = diff_results(run_oracle(p, ev_cap=0), g, events=False)
        if d:
            bad.append((p.policy, p.num_instances, p.num_requests, d[:4]))
    assert not bad, bad


def test_serial_pair_chain_variant(tmp_path):
    """The serial merged AcceLLM pair loop (-DKVSIM_PAIR_PAR=0, kept as the
    reference formulation of the member-parallel pair chains) still matches
    the oracle bit for bit, event logs included."""
    import subprocess
    import harness
    src = os.path.join(harness.ROOT, "tests", "emu", "kvsim_emu.cpp")
    so = str(tmp_path / "libkvsim_emu_serial_pairs.so")
    subprocess.run(["g++", "-DKVSIM_EMU", "-DKVSIM_PAIR_PAR=0", "-O2", "-std=gnu++20", "-ffp-contract=off", "-fPIC",
                    "-shared", "-I" + os.path.join(harness.ROOT, "include"), "-o", so, src, "-lpthread"], check=True)
    saved = (harness._emu, harness.EMU_SO)
    harness._emu, harness.EMU_SO = None, so
    try:
        pts = [config2("accellm", r, n=80) for r in (6.0, 12.0, 18.0)]
        pts += [p for p in (random_small(i) for i in range(100)) if p.policy == 2][:30]
        check(pts)
    finally:
        harness._emu, harness.EMU_SO = saved


def test_stress_regressions():
    """Two points a 3,000-point random GPU-vs-oracle stress run exposed
    (tools/stress_parity.py): a preempted AcceLLM request re-prefilled while
    still flagged as settling (memory-starved, 4 instances), and a
    Splitwise livelock that trips the event budget (first-token-from-decode,
    memory-starved). Both implementations must agree, including the budget
    stop point (SEMANTICS §4, §6)."""
    check([random_small(20249, max_req=400), random_small(20920, max_req=400)], ev=0)
