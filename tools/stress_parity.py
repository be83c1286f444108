"""Randomized GPU-vs-oracle stress (exploratory, beyond the -m gpu suite):
N random points (tests/configs.py random_small: all policies, memory-starved
half of the time, SPEC variants) through the product library, summaries and
request records compared bit for bit with the CPU oracle; then the same with
event logs (full kernel). usage: python tools/stress_parity.py [N] [MAX_REQ] [SEED0] [ext]
(ext: AcceLLM timer-extension points, tests/configs.py random_ext;
 detail: the records run as detail runs, pooled TBT percentiles + instance records;
 big: random_small points with 6-32 instances and 8x the rate)"""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import paper_2411_05555_b200 as pkg
from configs import random_ext, random_small
from harness import Result, diff_results, run_oracle

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
MAXR = int(sys.argv[2]) if len(sys.argv) > 2 else 400
S0 = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
EXT = len(sys.argv) > 4 and sys.argv[4] == "ext"
DET = len(sys.argv) > 4 and sys.argv[4] == "detail"
pts = [(random_ext if EXT else random_small)(S0 + i, max_req=MAXR) for i in range(N)]
if len(sys.argv) > 4 and sys.argv[4] == "big":
    import random as _r
    for i, p in enumerate(pts):
        r = _r.Random(S0 + i)
        p.num_instances = r.choice([6, 8, 12, 16, 24, 32])
        p.rate = p.rate * 8
sim = pkg.KvSim(0)
summ, recs, _ = sim.run(pts, records=True, detail=DET, instances=DET)
inst = sim.last_instances
bad = 0
for i, p in enumerate(pts):
    got = Result(summ[i], recs[i], None, inst=inst[i] if DET and summ[i].status == 0 else None)
    d = diff_results(run_oracle(p, recs=True, detail=DET, inst=DET), got, events=False)
    if d:
        bad += 1
        print(f"  point {i} (seed index {S0 + i}) policy {p.policy} inst {p.num_instances} reqs {p.num_requests} "
              f"cobatch {p.splitwise_cobatch} ft {p.first_token_decode}: {d[:3]}", flush=True)
print(f"records run: {N} points, {bad} mismatches", flush=True)
ev = 1 << 20
sub = [p for p in pts[: N // 4] if p.num_requests <= 120]
summ, recs, evs = sim.run(sub, records=True, events=ev)
cnt = sim.last_event_counts
bad = 0
for i, p in enumerate(sub):
    d = diff_results(run_oracle(p, ev_cap=ev, recs=True), Result(summ[i], recs[i], evs[i], ev_total=cnt[i]))
    if d:
        bad += 1
        if bad <= 5:
            print(f"  ev point {i} policy {p.policy} reqs {p.num_requests}: {d[:3]}", flush=True)
print(f"event-log run: {len(sub)} points, {bad} mismatches", flush=True)
