"""Per-point timing of the config-4 sweep (KVSIM_POINT_TIMES): warp busy
fractions, tail length, per-policy share. Exploratory; not the bench."""
import os, sys, time, collections
os.environ["KVSIM_POINT_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points
rates = int(sys.argv[1]) if len(sys.argv) > 1 else 833
pts = config4_points(0, rates, 10000)
sim = pkg.KvSim(0)
sim.run(pts[:16])
t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
pt = sim.point_times(len(pts))
T0 = min(a for a, b, c in pt); T1 = max(b for a, b, c in pt)
span = (T1 - T0) / 1e9
slots = collections.defaultdict(float)
for a, b, c in pt: slots[c] += (b - a) / 1e9
busy = sum(slots.values())
ends = sorted(max(b for a, b, c in pt if c == k) for k in slots)
print(f"wall={dt:.3f}s span={span:.3f}s slots={len(slots)} mean_busy={busy/len(slots):.3f}s eff={busy/len(slots)/span:.3f}")
for q in (0.1, 0.5, 0.9, 0.99):
    print(f"  slot finish quantile {q}: {(ends[int(q*(len(ends)-1))]-T0)/1e9:.3f}s")
bypol = collections.defaultdict(float); byn = collections.defaultdict(float)
for p, (a, b, c) in zip(pts, pt):
    bypol[p.policy] += (b - a) / 1e9; byn[(p.policy, p.num_instances)] += (b - a) / 1e9
print("busy by policy", {k: round(v / busy, 3) for k, v in bypol.items()})
print("busy by (policy,N)", {k: round(v / busy, 3) for k, v in sorted(byn.items())})
durs = sorted(((b - a) / 1e9, i) for i, (a, b, c) in enumerate(pt))
print("longest points", [(round(d, 3), pts[i].policy, pts[i].num_instances, round(pts[i].rate, 2)) for d, i in durs[-8:]])
print("point time quantiles", [round(durs[int(q*(len(durs)-1))][0], 4) for q in (0.1, 0.5, 0.9, 0.99)])
if len(sys.argv) > 2:
    import json
    json.dump([{"policy": p.policy, "n": p.num_instances, "rate": p.rate, "start": (a - T0) / 1e9, "dur": (b - a) / 1e9,
                "slot": c} for p, (a, b, c) in zip(pts, pt)], open(sys.argv[2], "w"))
