"""Single-policy config-4 slice (for ncu): probe3.py POLICY RATES REQUESTS"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points
pol = sys.argv[1]; rates = int(sys.argv[2]); nreq = int(sys.argv[3])
pts = config4_points(0, rates, nreq, policies=(pol,))
sim = pkg.KvSim(0)
sim.run(pts[:4])
t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
reqs = sum(x.n_requests for x in s); ev = sum(x.n_events for x in s); loops = sum(x.reserved[0] for x in s)
print(f"{pol} pts={len(pts)} wall={dt:.3f}s req/s={reqs/dt:.4e} events/s={ev/dt:.3e} loops={loops} loops/s={loops/dt:.3e} bad={sum(x.status!=0 for x in s)}", flush=True)
