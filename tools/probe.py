"""Exploratory throughput probe (not the bench): config-4-like sweep slices."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from paper_2411_05555_b200.abi import make_point

def grid(npts, nreq, pols=("unified", "splitwise", "accellm")):
    pts = []
    k = 0
    per = max(1, npts // (len(pols) * 4))
    for pol in pols:
        for ni in (4, 8, 12, 16):
            for j in range(per):
                rate = 3.0 * ni * (j + 1) / per
                pts.append(make_point(policy=pol, instances=ni, rate=rate, num_requests=nreq, seed=k)); k += 1
    return pts

sim = pkg.KvSim(0)
print("sms/blocks:", file=sys.stderr)
for npts, nreq in [(120, 1000), (1200, 1000), (4800, 2000)]:
    for pols in [("unified",), ("splitwise",), ("accellm",)]:
        pts = grid(npts, nreq, pols)
        sim.run(pts[:8])
        t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
        reqs = sum(x.n_requests for x in s); ev = sum(x.n_events for x in s); tok = sum(x.tokens_total for x in s)
        bad = sum(x.status != 0 for x in s)
        print(f"{pols[0]:10s} pts={len(pts):5d} req={nreq} wall={dt:.3f}s req/s={reqs/dt:.3e} ev/s={ev/dt:.3e} tok/s={tok/dt:.3e} bad={bad}", flush=True)
