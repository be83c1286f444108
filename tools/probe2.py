"""Occupancy probe: one config-4 slice per KVSIM_MINB variant (set in env)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points
rates = int(sys.argv[1]) if len(sys.argv) > 1 else 100
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
pts = config4_points(0, rates, nreq)
sim = pkg.KvSim(0)
sim.run(pts[:16])
for rep in range(1):
    t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
reqs = sum(x.n_requests for x in s); ev = sum(x.n_events for x in s); loops = sum(x.reserved[0] for x in s)
bad = sum(x.status != 0 for x in s)
by = {}
for p, x in zip(pts, s):
    by.setdefault(p.policy, [0, 0])
    by[p.policy][0] += x.n_events; by[p.policy][1] += x.reserved[0]
print(f"MINB={os.environ.get('KVSIM_MINB','default')} pts={len(pts)} wall={dt:.3f}s req/s={reqs/dt:.4e} events/s={ev/dt:.3e} loops/s={loops/dt:.3e} bad={bad} by_policy={by}", flush=True)
