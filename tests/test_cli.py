"""The C++ host entry point `kvsim` (reference SPEC.md:400-455): config
validation on CPU; run / sweep / gen-trace / curves end to end on the GPU,
checked against the CPU oracle."""
import csv
import json
import math
import os
import subprocess

import pytest

from harness import run_oracle
from paper_2411_05555_b200 import build
from paper_2411_05555_b200.abi import make_point

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def kvsim():
    return build.build_cli()


def run(kvsim, *args, cwd=None):
    return subprocess.run([kvsim, *args], capture_output=True, text=True, cwd=cwd)


def write(tmp_path, name, obj):
    p = tmp_path / name
    p.write_text(json.dumps(obj) if not isinstance(obj, str) else obj)
    return str(p)


def test_validate_echoes_defaults(kvsim, tmp_path):
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "c.json", {"instances": 4}))
    assert r.returncode == 0, r.stderr
    c = json.loads(r.stdout)
    assert c["policies"] == ["accellm"] and c["prefill_token_budget"] == 8192
    assert c["duration_s"] == 300 and c["warmup_s"] == 30          # SPEC.md:189 defaults
    assert c["efficiency"] == {"compute_eff": 0.5, "mem_bw_eff": 0.8, "link_eff": 0.8}
    assert c["model"]["num_layers"] == 80 and c["device"]["hbm_capacity"] == 80e9
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "d.json", {"num_requests": 10}))
    c = json.loads(r.stdout)
    assert c["duration_s"] == "inf" and c["warmup_s"] == 0


@pytest.mark.parametrize("cfg,msg", [
    ({"instancez": 4}, "unknown config key: instancez"),
    ({"instances": 5, "policy": "accellm"}, "even instance count required"),
    ({"device": {"name": "tiny", "peak_flops": 1e12, "hbm_capacity": 1e9, "hbm_bandwidth": 1e12,
                 "link_bandwidth": 1e9}}, "model does not fit in instance memory"),
    ({"workload": {"prompt_range": [10, 5], "decode_range": [1, 2]}}, "1 <= min <= max"),
    ({"policy": "fcfs"}, "unknown policy"),
    ({"splitwise_cobatch": 1}, "splitwise_cobatch must be a boolean"),
    ({"degraded_mode": {"trigger_tick": 2}}, "unknown degraded_mode key: trigger_tick"),
    ({"inter_pair_leveling": 3}, "must be a boolean or an object"),
    ({"policy_timer_s": 0}, "policy_timer_s must be > 0"),
])
def test_config_errors(kvsim, tmp_path, cfg, msg):
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "c.json", cfg))
    assert r.returncode == 2
    err = json.loads(r.stderr.strip().splitlines()[-1])
    assert msg in err["error"] and err["kind"] == "config"


def test_sweep_empty_rates_rejected(kvsim, tmp_path):
    r = run(kvsim, "sweep", "--config", write(tmp_path, "c.json", {"rates": [], "num_requests": 5}),
            "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "empty rate list" in r.stderr


def test_trace_errors_name_the_line(kvsim, tmp_path):
    t = tmp_path / "t.csv"
    t.write_text("#kvsim-trace v1\nid,arrival_s,prompt_len,decode_len\n0,0.5,10,5\n1,0.4,10,5\n")
    r = run(kvsim, "run", "--config", write(tmp_path, "c.json", {"trace": str(t), "instances": 2}),
            "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "t.csv:4: arrival_s decreases" in r.stderr


def test_no_gpu_fails_loudly(kvsim, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU visible")
    r = run(kvsim, "run", "--config", write(tmp_path, "c.json", {"num_requests": 5}), "--out", str(tmp_path / "o"))
    assert r.returncode == 3 and "no CPU fallback" in r.stderr


# ------------------------------------------------------------------ GPU
CFG1 = {"model": "llama2-7b", "device": "h100", "instances": 4, "policy": "accellm", "rate": 2.0,
        "num_requests": 1000, "workload": {"prompt_range": [512, 512], "decode_range": [10, 10]}, "seed": 3}


@pytest.mark.gpu
def test_run_records_match_oracle(kvsim, tmp_path):
    out = tmp_path / "o"
    r = run(kvsim, "run", "--config", write(tmp_path, "c.json", CFG1), "--out", str(out), "--emit-events")
    assert r.returncode == 0, r.stderr
    rep = json.load(open(out / "report.json"))
    p = make_point(model="llama2-7b", device="h100", policy="accellm", instances=4, rate=2.0, num_requests=1000,
                   prompt=512, decode=10, seed=3)
    ref = run_oracle(p, ev_cap=0)
    got = rep["points"][0]
    assert got["summary"]["n_completed"] == 1000
    for q, rr in zip(got["requests"], ref.recs):
        assert q["ttft_s"] == rr.first_token_s - rr.arrival_s
        assert q["jct_s"] == rr.completion_s - rr.arrival_s
        assert q["tbt_max_s"] == rr.tbt_max_s
    rows = list(csv.DictReader(open(out / "summary.csv")))
    assert float(rows[0]["jct_mean"]) == ref.summary.jct_mean
    assert (out / "events.jsonl").stat().st_size > 0
    # `run` reports the full MetricsReport: pooled TBT
    # percentiles (detail run), queue wait per request, per-instance records
    det = run_oracle(p, ev_cap=0, detail=True)
    assert got["summary"]["tbt_p50"] == det.summary.tbt_p50 and got["summary"]["tbt_p95"] == det.summary.tbt_p95
    assert got["summary"]["ttft_queue_mean"] == det.summary.ttft_queue_mean
    for q, rr in zip(got["requests"], det.recs):
        assert q["queue_wait_s"] == rr.prefill_start_s - rr.arrival_s
    inst = got["instances_detail"]
    assert len(inst) == 4
    for x, ir in zip(inst, det.inst):
        assert x["busy_s"] == ir.busy_s and x["idle_runnable_s"] == ir.idle_runnable_s
    meta = json.load(open(out / "meta.json"))
    assert meta["config"]["seeds"] == [3] and len(meta["config_hash"]) == 16


@pytest.mark.gpu
def test_sweep_matches_oracle_and_is_deterministic(kvsim, tmp_path):
    cfg = {"policies": ["accellm", "splitwise_static", "unified"], "rates": [2, 6, 12], "instances": 8,
           "num_requests": 800, "workload": "mixed", "seed": 1}
    c = write(tmp_path, "c.json", cfg)
    a, b = tmp_path / "a", tmp_path / "b"
    assert run(kvsim, "sweep", "--config", c, "--out", str(a)).returncode == 0
    assert run(kvsim, "sweep", "--config", c, "--out", str(b)).returncode == 0
    assert (a / "summary.csv").read_bytes() == (b / "summary.csv").read_bytes()
    rows = list(csv.DictReader(open(a / "summary.csv")))
    assert len(rows) == 9
    for row in rows:
        p = make_point(policy=row["policy"], instances=8, rate=float(row["rate"]), num_requests=800,
                       workload="mixed", seed=1, warmup_s=0.0)
        ref = run_oracle(p, ev_cap=0, recs=False).summary
        for k in ("ttft_mean", "ttft_p95", "tbt_mean", "tbt_max", "jct_mean", "jct_p95", "cost_eff"):
            assert float(row[k]) == getattr(ref, k), (row["policy"], k)
    rep = json.load(open(a / "report.json"))
    assert len(rep["saturation"]) == 3
    long = list(csv.DictReader(open(a / "sweep_long.csv")))
    assert len(long) == 9 * 11


@pytest.mark.gpu
def test_trace_round_trip(kvsim, tmp_path):  # SPEC.md:172 generate -> save -> load
    cfg = dict(CFG1, workload="mixed", num_requests=300, policy="splitwise_static", instances=4)
    g = tmp_path / "g"
    assert run(kvsim, "gen-trace", "--config", write(tmp_path, "c.json", cfg), "--out", str(g)).returncode == 0
    tr = str(g / "trace.csv")
    lines = open(tr).read().splitlines()
    assert lines[0] == "#kvsim-trace v1" and len(lines) == 302
    a, b = tmp_path / "a", tmp_path / "b"
    assert run(kvsim, "run", "--config", write(tmp_path, "d.json", cfg), "--out", str(a)).returncode == 0
    cfg_t = {k: v for k, v in cfg.items() if k not in ("rate", "num_requests", "workload", "seed")}
    cfg_t["trace"] = tr
    r = run(kvsim, "run", "--config", write(tmp_path, "e.json", cfg_t), "--out", str(b))
    assert r.returncode == 0, r.stderr
    ra = json.load(open(a / "report.json"))["points"][0]
    rb = json.load(open(b / "report.json"))["points"][0]
    assert ra["requests"] == rb["requests"]


def test_curves(kvsim, tmp_path):  # host perfmodel only
    cfg = {"efficiency": {"compute_eff": 1.0, "mem_bw_eff": 1.0, "link_eff": 1.0},
           "curves": {"phase": "both", "lengths": [500], "batch_sizes": [1, 32]}}
    o = tmp_path / "o"
    assert run(kvsim, "curves", "--config", write(tmp_path, "c.json", cfg), "--out", str(o)).returncode == 0
    rows = list(csv.DictReader(open(o / "curves.csv")))
    dec = {int(r["batch"]): r for r in rows if r["phase"] == "decode"}
    assert abs(float(dec[1]["latency_s"]) - 0.01046) < 1e-5 and abs(float(dec[32]["tokens_per_s"]) - 2952) < 1
    pre = [r for r in rows if r["phase"] == "prefill"]
    assert math.isclose(float(pre[0]["tokens_per_s"]), float(pre[1]["tokens_per_s"]), rel_tol=1e-12)


@pytest.mark.gpu
def test_resource_sweep_knees_and_failed_points(kvsim, tmp_path):
    cfg = {"policies": ["accellm", "splitwise_static"], "rate": 6, "instances": 4, "num_requests": 600,
           "workload": "mixed", "resource": {"kind": "hbm_capacity", "values": [30e9, 40e9, 60e9, 80e9, 120e9]}}
    o = tmp_path / "o"
    r = run(kvsim, "resource-sweep", "--config", write(tmp_path, "c.json", cfg), "--out", str(o))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(o / "resource_sweep.csv")))
    assert len(rows) == 10
    # 4 x 30 GB x 0.9 < 140 GB of weights: per-point error, sweep continues
    assert all(int(x["status"]) == -2 for x in rows if float(x["hbm_capacity"]) == 30e9)
    assert all(int(x["status"]) == 0 for x in rows if float(x["hbm_capacity"]) >= 60e9)
    knees = json.load(open(o / "report.json"))["knees"]
    assert {k["policy"] for k in knees} == {"accellm", "splitwise_static"}
    assert all(k["knee"] is not None and k["knee"] >= 40e9 for k in knees)
    # every row equals the oracle's run of the same point
    for x in rows:
        p = make_point(policy=x["policy"], instances=4, rate=6.0, num_requests=600, workload="mixed", seed=0,
                       device=(989e12, float(x["hbm_capacity"]), 3.35e12, 900e9))
        ref = run_oracle(p, ev_cap=0, recs=False)
        assert ref.status == int(x["status"])
        if ref.status == 0:
            assert float(x["jct_mean"]) == ref.summary.jct_mean and float(x["cost_eff"]) == ref.summary.cost_eff


@pytest.mark.gpu
def test_resource_sweep_link_bandwidth_knee(kvsim, tmp_path):  # SPEC.md:432-438,468 (acceptance #10)
    import acceptance as A
    bws = list(A.A10_BW)
    cfg = {"policies": ["accellm", "splitwise_static"], "rate": 4, "instances": 4, "workload": "mixed",
           "duration_s": 300, "warmup_s": 30, "num_requests": int(4 * 300 * 1.3) + 100, "seed": 1,
           "resource": {"kind": "link_bandwidth", "values": bws}}
    o = tmp_path / "o"
    r = run(kvsim, "resource-sweep", "--config", write(tmp_path, "c.json", cfg), "--out", str(o))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(o / "resource_sweep.csv")))
    assert len(rows) == 2 * len(bws)
    jct = {}
    for x in rows:
        p = A.desk_point(policy=x["policy"], instances=4, workload="mixed", rate=4.0, seed=1,
                         device=(989e12, 80e9, 3.35e12, float(x["link_bandwidth"])))
        ref = run_oracle(p, ev_cap=0, recs=False).summary
        assert float(x["jct_mean"]) == ref.jct_mean and float(x["cost_eff"]) == ref.cost_eff
        jct.setdefault(x["policy"], []).append((float(x["link_bandwidth"]), ref.jct_mean, ref.cost_eff))
    # the CLI's knee (1% of best JCT and cost efficiency) from the oracle's rows
    knees = {k["policy"]: k["knee"] for k in json.load(open(o / "report.json"))["knees"]}
    for pol, g in jct.items():
        bj, bc = min(j for _, j, _ in g), max(c for _, _, c in g)
        assert knees[pol] == min(b for b, j, c in g if j <= 1.01 * bj and c >= 0.99 * bc)
    # acceptance #10 at 4 req/s: JCT knees within 25% (SEMANTICS §9)
    kj = {pol: min(b for b, j, _ in g if j <= 1.01 * min(x[1] for x in g)) for pol, g in jct.items()}
    assert abs(kj["accellm"] / kj["splitwise_static"] - 1.0) <= 0.25


@pytest.mark.gpu
def test_sweep_compare_table(kvsim, tmp_path):
    cfg = {"policies": ["accellm", "unified"], "rates": [4, 8], "instances": 4, "num_requests": 300, "seed": 2}
    o = tmp_path / "o"
    assert run(kvsim, "sweep", "--config", write(tmp_path, "c.json", cfg), "--out", str(o)).returncode == 0
    cmp = json.load(open(o / "report.json"))["compare"]
    assert len(cmp) == 2
    for g in cmp:
        assert g["ratios_vs_accellm"]["accellm"]["cost_eff"] == 1.0
        assert len(g["trace_fingerprint"]) == 16


def test_accellm_extension_keys_resolve(kvsim, tmp_path):
    # every tie-break/threshold is a named key and defaults are echoed
    r = run(kvsim, "validate-config", "--config",
            write(tmp_path, "e.json", {"degraded_mode": {"trigger_ticks": 2}, "inter_pair_leveling": True}))
    assert r.returncode == 0, r.stderr
    c = json.loads(r.stdout)
    assert c["degraded_mode"] == {"enabled": True, "trigger_ticks": 2, "redundancy_threshold": 0.5,
                                  "exit_fill": 0.5, "dual_copy_fraction": 1.0 / 3.0}
    assert c["inter_pair_leveling"] == {"enabled": True, "link_fraction": 0.1}
    assert c["policy_timer_s"] == 1.0
    r = run(kvsim, "validate-config", "--config", write(tmp_path, "f.json", {"num_requests": 3}))
    c = json.loads(r.stdout)
    assert c["degraded_mode"]["enabled"] is False and c["inter_pair_leveling"]["enabled"] is False


@pytest.mark.gpu
def test_run_accellm_extensions_match_oracle(kvsim, tmp_path):
    # degraded mode + leveling through the drop-in entry point (SEMANTICS §6b)
    cfg = {"policy": "accellm", "instances": 8, "rate": 30.0, "num_requests": 1500, "workload": "heavy",
           "memory_reserve_fraction": 0.5, "seed": 4, "policy_timer_s": 0.1,
           "degraded_mode": {"trigger_ticks": 1}, "inter_pair_leveling": True}
    out = tmp_path / "o"
    r = run(kvsim, "run", "--config", write(tmp_path, "c.json", cfg), "--out", str(out))
    assert r.returncode == 0, r.stderr
    got = json.load(open(out / "report.json"))["points"][0]["summary"]
    p = make_point(policy="accellm", instances=8, rate=30.0, num_requests=1500, workload="heavy", reserve=0.5,
                   seed=4, timer_s=0.1, degraded=True, trigger_ticks=1, leveling=True)
    ref = run_oracle(p, ev_cap=0, recs=False).summary
    assert got["n_mode_switches"] == ref.n_mode_switches > 0
    assert got["link_leveling_tokens"] == ref.link_leveling_tokens
    assert got["jct_mean"] == ref.jct_mean and got["n_events"] == ref.n_events


def _queue_series(events, unified):
    """Reference restatement of the CLI's queue-depth rule over an event log."""
    dv = {}
    for e in events:
        d = 0
        if e.kind in (1, 8):          # ARRIVE, PREEMPT
            d = 1
        elif e.kind == 2:             # PREFILL_START: a prompts admitted
            d = -e.a
        elif e.kind == 4 and unified and e.b > 0:  # co-batched prompts
            d = -e.b
        if d:
            dv[e.t] = dv.get(e.t, 0) + d
    out, depth = [], 0
    for t in sorted(dv):
        depth += dv[t]
        out.append((t, depth))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["accellm", "splitwise", "unified"])
def test_queue_depth_series(kvsim, tmp_path, policy):
    cfg = {"model": "llama2-70b", "device": "h100", "instances": 4, "policy": policy, "rate": 6.0,
           "num_requests": 400, "workload": "light", "seed": 5, "warmup_s": 0}
    out = tmp_path / "q"
    r = run(kvsim, "run", "--config", write(tmp_path, "c.json", cfg), "--out", str(out), "--emit-events")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(out / "queue_depth.csv")))
    got = [(float(x["t"]), int(x["depth"])) for x in rows]
    p = make_point(model="llama2-70b", device="h100", policy=policy, instances=4, rate=6.0, num_requests=400,
                   workload="light", seed=5, warmup_s=0.0)
    ref = run_oracle(p, ev_cap=1 << 18)
    want = _queue_series(ref.events, policy == "unified")
    assert got == want
    assert all(d >= 0 for _, d in got) and got[-1][1] == 0
    q = json.load(open(out / "report.json"))["points"][0]["queue_depth"]
    # the device's own queue-depth statistics (kvsim_point_summary v2) agree
    # with the series and, bit for bit, with the oracle
    assert q["max"] == max(d for _, d in got) == ref.summary.queue_depth_max
    assert q["time_avg"] == ref.summary.queue_depth_avg


@pytest.mark.parametrize("policy", ["accellm", "splitwise", "unified"])
def test_queue_depth_rule_on_oracle(policy):
    # the queue-depth rule balances: never negative, empty once every request ran
    p = make_point(model="llama2-70b", device="h100", policy=policy, instances=4, rate=8.0, num_requests=300,
                   workload="light", seed=9, warmup_s=0.0)
    ref = run_oracle(p, ev_cap=1 << 18)
    s = _queue_series(ref.events, policy == "unified")
    assert s and all(d >= 0 for _, d in s) and s[-1][1] == 0
    assert max(d for _, d in s) > 0


@pytest.mark.gpu
def test_cli_sharder_gpu_count_invariance(kvsim, tmp_path):
    """The CLI sharder (guided chunks over cost-sorted points, results by
    index) gives byte-identical outputs for 1, 2 and 3 workers. One GPU here:
    KVSIM_VIRTUAL_GPUS lets several workers share it (a logic test of the
    sharder, not a performance setting)."""
    cfg = {"policies": ["accellm", "splitwise_static", "unified"], "rates": [1, 3, 6, 12, 20], "instances": 4,
           "num_requests": 600, "workload": "mixed", "seeds": [0, 1], "sweep_instances": [4, 8]}
    c = write(tmp_path, "c.json", cfg)
    outs = []
    env = dict(os.environ, KVSIM_VIRTUAL_GPUS="1")
    for g in (1, 2, 3):
        o = tmp_path / f"g{g}"
        r = subprocess.run([kvsim, "sweep", "--config", c, "--out", str(o), "--gpus", str(g)], capture_output=True,
                           text=True, env=env)
        assert r.returncode == 0, r.stderr
        outs.append(((o / "summary.csv").read_bytes(), (o / "sweep_long.csv").read_bytes(),
                     json.load(open(o / "report.json"))["points"]))
    assert all(x == outs[0] for x in outs)


@pytest.mark.gpu
def test_run_multi_matches_single_launch():
    """kvsim_gpu_run_multi (the bench's multi-GPU path) on the visible GPU:
    chunked, cost-sorted, summaries scattered by index == one launch."""
    import paper_2411_05555_b200 as pkg
    from configs import random_small
    pts = [random_small(4000 + i, max_req=200) for i in range(90)]
    sim = pkg.KvSim(0)
    one = sim.run(pts)
    multi, st = pkg.run_multi([sim], pts, min_chunk=4)
    assert st.device_points[0] == len(pts) and st.device_launches[0] > 1 and st.device_seconds[0] > 0
    assert all(bytes(a) == bytes(b) for a, b in zip(one, multi))
    sim.close()


@pytest.mark.gpu
def test_curves_on_device_match_host_api(kvsim, tmp_path):
    """cmd_curves on the device (K1 through kvsim_gpu_curves) equals the
    reference's host perfmodel API (throughput_curves) bit for bit."""
    import ctypes as C
    from harness import oracle
    cfg = {"model": "llama2-70b", "device": "910b2", "instances": 4,
           "curves": {"phase": "both", "lengths": [100, 500, 1000], "batch_sizes": [1, 2, 8, 32, 128, 512]}}
    o = tmp_path / "o"
    assert run(kvsim, "curves", "--config", write(tmp_path, "c.json", cfg), "--out", str(o)).returncode == 0
    assert json.load(open(o / "meta.json"))["evaluated_on"].startswith("gpu")
    rows = list(csv.DictReader(open(o / "curves.csv")))
    assert len(rows) == 2 * 3 * 6
    L = oracle()
    p = make_point(model="llama2-70b", device="910b2")
    for r in rows:
        Ln, b = int(r["length"]), int(r["batch"])
        want = (L.kvo_prefill_latency(C.byref(p), b * Ln, b * Ln * Ln) if r["phase"] == "prefill"
                else L.kvo_decode_step_latency(C.byref(p), b, b * Ln))
        assert float(r["latency_s"]) == want
