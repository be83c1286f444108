"""Per-policy share of the config-4 sweep time (exploratory; not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points
rates = int(sys.argv[1]) if len(sys.argv) > 1 else 833
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
sim = pkg.KvSim(0)
for pol in ("unified", "splitwise", "accellm"):
    for ni in (4, 8, 12, 16):
        pts = config4_points(0, rates, nreq, policies=(pol,), instances=(ni,))
        sim.run(pts[:2])
        t0 = time.time(); s = sim.run(pts); dt = time.time() - t0
        reqs = sum(x.n_requests for x in s); ev = sum(x.n_events for x in s); loops = sum(x.reserved[0] for x in s)
        tok = sum(x.tokens_total for x in s)
        print(f"{pol:9s} N={ni:2d} pts={len(pts)} wall={dt:.3f}s req/s={reqs/dt:.3e} events={ev:.3e} loops={loops:.3e} "
              f"ev/req={ev/reqs:.1f} loops/req={loops/reqs:.2f} tok/req={tok/reqs:.0f}", flush=True)
