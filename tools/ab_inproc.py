"""In-process A/B of build variants (exploratory): one KvSim per variants/*.so
in the same process, a full config-4 warm-up sweep each, then R rounds of
alternating timed sweeps. Less noisy than one process per variant (clock and
power state are shared). Usage: python tools/ab_inproc.py [R] [lib[:MINB] ...]
(MINB = KVSIM_MINB for that context: resident blocks per SM; lib:MINB:CARVE
also sets KVSIM_CARVEOUT, the shared-memory carveout percent;
lib:MINB:CARVE:BPS also KVSIM_BLOCKS_PER_SM, the blocks launched per SM)."""
import glob, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_05555_b200 as pkg
from bench import config4_points

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
libs = sys.argv[2:] or sorted(glob.glob("variants/*.so"))
pts = config4_points(0, 833, 10000)
sims = {}
for spec in libs:
    lib, _, rest = spec.partition(":")
    minb, _, rest = rest.partition(":")
    carve, _, bps = rest.partition(":")
    if bps:
        os.environ["KVSIM_BLOCKS_PER_SM"] = bps
    else:
        os.environ.pop("KVSIM_BLOCKS_PER_SM", None)
    if carve:
        os.environ["KVSIM_CARVEOUT"] = carve
    else:
        os.environ.pop("KVSIM_CARVEOUT", None)
    os.environ["KVSIM_LIB"] = lib
    if minb:
        os.environ["KVSIM_MINB"] = minb
    else:
        os.environ.pop("KVSIM_MINB", None)
    pkg._lib = None
    sims[os.path.basename(spec)] = pkg.KvSim(0)
ref = None
for name, s in sims.items():
    out = s.run(pts)
    b = b"".join(bytes(x) for x in out)
    if ref is None:
        ref = b
    print(f"{name} warm-up done, identical to first={b == ref}", flush=True)
times = {k: [] for k in sims}
for r in range(R):
    order = list(sims) if r % 2 == 0 else list(sims)[::-1]
    for name in order:
        t0 = time.perf_counter(); sims[name].run(pts); times[name].append(time.perf_counter() - t0)
for name, t in times.items():
    print(f"{name} median={statistics.median(t):.3f}s min={min(t):.3f}s all={[round(x, 3) for x in t]}", flush=True)
