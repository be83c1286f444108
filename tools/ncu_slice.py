"""Config-4 slice for ncu --set full captures (every k-th rate):
ncu_slice.py RATES REQUESTS [POLICY]   (POLICY: unified | splitwise | accellm; default all three)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points
rates = int(sys.argv[1]) if len(sys.argv) > 1 else 84
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
pols = (sys.argv[3],) if len(sys.argv) > 3 else ("unified", "splitwise", "accellm")
pts = config4_points(0, rates, nreq, policies=pols)
sim = pkg.KvSim(0)
t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
reqs = sum(x.n_requests for x in s)
print(f"pts={len(pts)} wall={dt:.3f}s req/s={reqs/dt:.4e} bad={sum(x.status != 0 for x in s)}", flush=True)
