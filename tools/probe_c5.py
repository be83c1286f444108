"""BASELINE config 5 slice: 3 policies x {H100, 910B2} x R log-spaced rates in [0.5, 30] x seeds,
Llama-2-70B, 8 instances, mixed, 100k requests per point (aggregates only)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from paper_2411_05555_b200.abi import make_point
R = int(sys.argv[1]) if len(sys.argv) > 1 else 50
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1
N = int(sys.argv[3]) if len(sys.argv) > 3 else 100000
pts = []
for pol in ("unified", "splitwise", "accellm"):
    for dev in ("h100", "910b2"):
        for j in range(R):
            rate = 0.5 * (30 / 0.5) ** (j / max(R - 1, 1))
            for s in range(S):
                pts.append(make_point(policy=pol, device=dev, instances=8, rate=rate, num_requests=N,
                                      workload="mixed", seed=len(pts)))
sim = pkg.KvSim(0)
t0 = time.time(); out = sim.run(pts); dt = time.time() - t0
reqs = sum(x.n_requests for x in out)
bad = [(p.policy, p.rate, x.status) for p, x in zip(pts, out) if x.status != 0]
print(f"config5 slice: {len(pts)} points x {N} req: wall={dt:.2f}s req/s={reqs/dt:.4e} bad={len(bad)} {bad[:5]}")
