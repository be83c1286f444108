"""SPEC acceptance criteria #3, #5-#10 (reference SPEC.md:461-468) at the
SPEC's own setups, evaluated on any runner that maps points -> summaries
(the CPU oracle in tests/test_acceptance.py, the sm_100a kernels in the GPU
variant, which must agree with the oracle bit for bit first).

Each criterion returns a dict of measured numbers plus `holds` flags; the
tests assert the flags that hold under SPEC's formulas and, for the parts
shown unattainable (docs/SEMANTICS.md §9, with the argument), assert the
bound the argument predicts instead. `tools/acceptance_report.py` prints
the table in SEMANTICS §9 from the same functions.

Desk scale: 300 simulated seconds, the first 30 s excluded
(SPEC.md:189), 3 seeds.
"""
from __future__ import annotations

import math

from paper_2411_05555_b200.abi import make_point

SEEDS = (0, 1, 2)
DURATION, WARMUP = 300.0, 30.0
MIXED_MEAN_DECODE = 510.0  # uniform 20..1000


def desk_point(*, rate, seed, **kw):
    # arrivals stop at DURATION; num_requests only caps the generator
    return make_point(rate=rate, seed=seed, num_requests=int(rate * DURATION * 1.3) + 100,
                      duration_s=DURATION, warmup_s=WARMUP, **kw)


def window(s):
    return s.makespan_s - WARMUP


# ---------------------------------------------------------------- #3
A3_RATES = (8.0, 12.0, 16.0)


def a3_points():
    """Mixed, 910B2, 4 instances, rates around saturation; unified and
    AcceLLM on identical traces (same seed => same trace)."""
    return [desk_point(policy=pol, device="910b2", instances=4, workload="mixed", rate=r, seed=sd)
            for pol in ("unified", "accellm") for r in A3_RATES for sd in SEEDS]


def a3_eval(pts, summ):
    rows = []
    for p, s in zip(pts, summ):
        rows.append({"policy": "unified" if p.policy == 0 else "accellm", "rate": p.rate, "seed": p.seed,
                     "tbt_p50": s.tbt_p50, "tbt_max": s.tbt_max, "ratio": s.tbt_max / s.tbt_p50})
    uni = [r for r in rows if r["policy"] == "unified"]
    acc = [r for r in rows if r["policy"] == "accellm"]
    umax = {(r["rate"], r["seed"]): r["tbt_max"] for r in uni}
    return {
        "rows": rows,
        "unified_min_ratio": min(r["ratio"] for r in uni),
        "accellm_max_ratio": max(r["ratio"] for r in acc),
        # SPEC #3 part 1: unified max TBT >= 4x median
        "holds_unified": all(r["ratio"] >= 4.0 for r in uni),
        # SPEC #3 part 2 (<= 1.5x median): unattainable under SPEC.md:262-263 (SEMANTICS §9)
        "holds_accellm_spec": all(r["ratio"] <= 1.5 for r in acc),
        # the hand-off bound instead: a displaced request waits at most the
        # partner's in-flight step plus its next step (~2 steps), and no
        # prefill ever lands inside an AcceLLM step
        "holds_accellm_handoff_bound": all(r["ratio"] <= 2.5 for r in acc),
        "holds_no_prefill_interference": all(r["tbt_max"] <= 0.25 * umax[(r["rate"], r["seed"])] for r in acc),
    }


# ------------------------------------------------------------ #5 / #6 / #7a
A5_RATES = tuple(float(r) for r in range(20, 101, 10))
POLS = ("splitwise", "unified", "accellm")


def a5_points():
    """Mixed, 8 H100, identical traces per (rate, seed) across policies."""
    return [desk_point(policy=pol, instances=8, workload="mixed", rate=r, seed=sd)
            for pol in POLS for r in A5_RATES for sd in SEEDS]


def _index(pts, summ):
    name = {0: "unified", 1: "splitwise", 2: "accellm"}
    return {(name[p.policy], p.rate, p.seed): s for p, s in zip(pts, summ)}


def a5_eval(pts, summ):
    ix = _index(pts, summ)
    rows = []
    for sd in SEEDS:
        # splitwise_static's saturation point: argmax of its cost efficiency
        # over the rate grid (glossary "Saturation point")
        lam = max(A5_RATES, key=lambda r: ix[("splitwise", r, sd)].cost_eff)
        a, sw, u = ix[("accellm", lam, sd)], ix[("splitwise", lam, sd)], ix[("unified", lam, sd)]
        offered = lam * MIXED_MEAN_DECODE / 8.0
        rows.append({"seed": sd, "rate": lam, "ce_vs_splitwise": a.cost_eff / sw.cost_eff,
                     "ce_vs_unified": a.cost_eff / u.cost_eff, "jct_vs_splitwise": a.jct_mean / sw.jct_mean,
                     "jct_vs_unified": a.jct_mean / u.jct_mean,
                     "accellm_ce_over_offered": a.cost_eff / offered, "unified_ce_over_offered": u.cost_eff / offered,
                     "ttft_vs_splitwise": a.ttft_mean / sw.ttft_mean,
                     "queue_wait_splitwise": sw.ttft_queue_mean, "queue_wait_accellm": a.ttft_queue_mean,
                     "idle_runnable_frac_accellm": a.idle_runnable_s / (8 * window(a)),
                     "idle_runnable_frac_splitwise": sw.idle_runnable_s / (8 * window(sw))})
    return {
        "rows": rows,
        "holds_ce_vs_splitwise": all(r["ce_vs_splitwise"] >= 1.15 for r in rows),
        "holds_ce_vs_unified": all(r["ce_vs_unified"] >= 1.15 for r in rows),
        "holds_jct": all(r["jct_vs_splitwise"] <= 0.90 and r["jct_vs_unified"] <= 0.90 for r in rows),
        # why ce vs unified cannot reach 1.15 (SEMANTICS §9): cost efficiency
        # is bounded by the offered load, and both deliver it at this rate
        "holds_offered_bound": all(r["accellm_ce_over_offered"] >= 0.95 and r["unified_ce_over_offered"] >= 0.95
                                   for r in rows),
        # #6: TTFT at the (high) splitwise saturation rate
        "holds_ttft": all(r["ttft_vs_splitwise"] <= 0.6 for r in rows),
        "holds_queue_wait": all(r["queue_wait_splitwise"] > 0 and
                                r["queue_wait_accellm"] <= 0.05 * r["queue_wait_splitwise"] for r in rows),
        # #7 part 1: no AcceLLM instance idles while work waits in a queue
        "holds_idle_accellm": all(r["idle_runnable_frac_accellm"] <= 1e-6 for r in rows),
    }


# ----------------------------------------------------------------- #7b
A7_RATES = (10.0, 20.0, 30.0)


def a7_points():
    """Splitwise under the light workload, 8 H100 = 2 prefill +
    6 decode instances."""
    return [desk_point(policy="splitwise", instances=8, workload="light", rate=r, seed=sd)
            for r in A7_RATES for sd in SEEDS]


def a7_eval(pts, summ, inst):
    rows = []
    for p, s, ii in zip(pts, summ, inst):
        w = window(s)
        pf = [1.0 - x.busy_s / w for x in ii if x.initial_role == 1]
        rows.append({"rate": p.rate, "seed": p.seed, "prefill_idle_frac": pf})
    return {"rows": rows, "holds_prefill_idle": all(min(r["prefill_idle_frac"]) > 0.2 for r in rows)}


# ------------------------------------------------------------------ #8
def a8_points():
    return [desk_point(policy="accellm", instances=8, workload="mixed", rate=r, seed=sd)
            for r in (20.0, 60.0) for sd in SEEDS]


def a8_eval(pts, events):
    """Peak per-link mirror bandwidth from the event log: a mirror transfer of
    m tokens enqueued at a step end carries the KV lines that step produced,
    m * kv_bytes_per_token over the step's duration."""
    out = []
    for p, ev in zip(pts, events):
        kvb = 2.0 * p.num_layers * p.num_kv_heads * p.head_dim * p.bytes_per_value
        link = p.num_devices * p.link_bandwidth * p.link_eff
        start = {}
        worst = 0.0
        exact = True
        last_batch = {}
        for e in ev:  # the oracle's log is in processing order (step end, mirror, next step start)
            if e.kind == 4:  # step start: (inst) -> time, batch
                start[e.inst] = e.t
                last_batch[e.inst] = e.a
            elif e.kind == 10 and e.b == 1:  # mirror transfer at the step end
                d = e.t - start[e.inst]
                worst = max(worst, e.c * kvb / d / link)
                exact = exact and e.c <= last_batch[e.inst]
        out.append({"rate": p.rate, "seed": p.seed, "peak_mirror_link_frac": worst})
    return {"rows": out, "holds_mirror_bw": all(r["peak_mirror_link_frac"] < 0.05 for r in out)}


# ------------------------------------------------------------------ #9
A9_RATES = (4.0, 8.0, 12.0)


def a9_points():
    return [desk_point(policy=pol, instances=4, workload="mixed", rate=r, seed=sd)
            for pol in ("splitwise", "accellm") for r in A9_RATES for sd in SEEDS]


def a9_eval(pts, summ):
    ix = {(p.policy, p.rate, p.seed): s for p, s in zip(pts, summ)}
    cap_gb = None
    rows = []
    for sd in SEEDS:
        over = []
        for r in A9_RATES:
            a, sw = ix[(2, r, sd)], ix[(1, r, sd)]
            over.append(a.peak_kv_gb - sw.peak_kv_gb)
        rows.append({"seed": sd, "overhead_gb": over})
    p0 = pts[0]
    kvb = 2.0 * p0.num_layers * p0.num_kv_heads * p0.head_dim * p0.bytes_per_value
    cap_tokens = math.floor((p0.num_devices * p0.hbm_capacity * (1 - p0.memory_reserve_fraction) -
                             p0.param_count * p0.bytes_per_value) / kvb)
    cap_gb = cap_tokens * kvb / 1e9
    return {"rows": rows, "capacity_gb": cap_gb,
            "holds_positive": all(min(r["overhead_gb"]) > 0 for r in rows),
            "holds_monotone": all(all(x < y for x, y in zip(r["overhead_gb"], r["overhead_gb"][1:])) for r in rows),
            "holds_under_capacity": all(s.peak_kv_gb <= cap_gb for s in summ)}


# ----------------------------------------------------------------- #10
A10_RATES = (4.0, 8.0)
A10_BW = tuple(1e8 * (100.0 ** (k / 40.0)) for k in range(41))  # 0.1 .. 10 GB/s per device, x1.12 steps


def a10_points():
    """Link-bandwidth resource sweep: mixed, 4 H100."""
    return [desk_point(policy=pol, instances=4, workload="mixed", rate=r, seed=sd,
                       device=(989e12, 80e9, 3.35e12, bw))
            for pol in ("accellm", "splitwise") for r in A10_RATES for sd in SEEDS for bw in A10_BW]


def a10_eval(pts, summ):
    groups = {}
    for p, s in zip(pts, summ):
        groups.setdefault((p.policy, p.rate, p.seed), []).append((p.link_bandwidth, s.jct_mean))
    rows = []
    for r in A10_RATES:
        for sd in SEEDS:
            knee = {}
            for pol, name in ((2, "accellm"), (1, "splitwise")):
                g = groups[(pol, r, sd)]
                best = min(j for _, j in g)
                knee[name] = min(b for b, j in g if j <= 1.01 * best)
            ratio = knee["accellm"] / knee["splitwise"]
            rows.append({"rate": r, "seed": sd, "knee_accellm_gbs": knee["accellm"] / 1e9,
                         "knee_splitwise_gbs": knee["splitwise"] / 1e9, "ratio": ratio})
    # "knee bandwidths within 25% of each other": relative to splitwise's knee
    within = [abs(x["ratio"] - 1.0) <= 0.25 for x in rows]
    return {"rows": rows, "holds_within_25pct": all(within),
            "holds_within_25pct_low_rate": all(w for w, x in zip(within, rows) if x["rate"] == A10_RATES[0]),
            # the bound the byte count predicts (SEMANTICS §9): AcceLLM moves
            # prompt + decode tokens per request, Splitwise the prompt only
            "holds_within_2x": all(max(x["ratio"], 1 / x["ratio"]) <= 2.0 for x in rows)}
