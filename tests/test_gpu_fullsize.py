"""GPU parity at BASELINE.json's full per-point sizes (configs 4 and 5): the
sm_100a kernel through the C-ABI against the CPU oracle, bit-exact, on
points taken from the exact grids bench.py and tools/probe_c5.py run
(10k requests per config-4 point with per-request records; 100k requests per
config-5 point, summaries only, as SURVEY §8d asks of config 5), plus the
device-resident entry point the bench times (`kvsim_gpu_run_device`) against
the host-buffer entry point on the same points."""
import ctypes as C
import os

import pytest

from harness import Result, diff_results, oracle, run_oracle
from paper_2411_05555_b200.abi import PointDesc, PointSummary, TraceView, make_point

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    import paper_2411_05555_b200 as pkg
    s = pkg.KvSim(0)
    yield s
    s.close()


def _bench_grid():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import config4_points
    return config4_points(0, 833, 10000)


def test_config4_full_size_records(sim):
    # every 417th point of the 9,996-point bench grid: all three policies,
    # all four instance counts, low to saturated rates; 10k requests each
    pts = _bench_grid()[::417]
    assert len({p.policy for p in pts}) == 3 and len({p.num_instances for p in pts}) == 4
    summ, recs, _ = sim.run(pts, records=True)
    bad = []
    for i, p in enumerate(pts):
        assert summ[i].status == 0 and summ[i].n_requests == 10000
        ref = run_oracle(p, ev_cap=0, recs=True)
        d = diff_results(ref, Result(summ[i], recs[i], None), events=False)
        if d:
            bad.append((i, p.policy, p.num_instances, p.rate, d[:4]))
    assert not bad, bad


def _config5_points():
    pts = []
    for pol in ("unified", "splitwise", "accellm"):
        for dev in ("h100", "910b2"):
            for rate in (0.5, 4.0, 30.0):
                pts.append(make_point(policy=pol, device=dev, instances=8, rate=rate, num_requests=100000,
                                      workload="mixed", seed=700 + len(pts)))
    return pts


def test_config5_full_size_summaries(sim):
    pts = _config5_points()
    out = sim.run(pts)
    n = len(pts)
    P = (PointDesc * n)(*pts)
    S = (PointSummary * n)()
    oracle().kvo_run_sweep(P, n, os.cpu_count() or 1, S)  # one point per host thread
    bad = []
    for i in range(n):
        assert out[i].status == 0 and out[i].n_requests == 100000
        d = diff_results(Result(S[i], None, None), Result(out[i], None, None), events=False)
        if d:
            bad.append((i, pts[i].policy, pts[i].rate, d[:4]))
    assert not bad, bad
    # size-independent properties at full size: every request completes, and
    # tokens = sum of decode lengths (one token per decode_len, SEMANTICS P1)
    L = oracle()
    for i, p in enumerate(pts[:2]):
        arr = (C.c_double * 100000)()
        pl = (C.c_int32 * 100000)()
        dl = (C.c_int32 * 100000)()
        assert L.kvo_gen_trace(C.byref(p), arr, pl, dl, 100000) == 100000
        assert out[i].n_completed == 100000
        assert out[i].tokens_total == sum(dl)


def test_device_resident_entry_matches_host_entry(sim):
    torch = pytest.importorskip("torch")
    pts = _bench_grid()[5::333]
    n = len(pts)
    host = sim.run(pts)
    P = (PointDesc * n)(*pts)
    d_pts = torch.frombuffer(bytearray(bytes(P)), dtype=torch.uint8).to("cuda:0")
    d_out = torch.zeros(n * C.sizeof(PointSummary), dtype=torch.uint8, device="cuda:0")
    sim.reserve(pts)
    stream = torch.cuda.Stream(0)
    sim.run_device(d_pts.data_ptr(), n, d_out.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize(0)
    raw = d_out.cpu().numpy().tobytes()
    sz = C.sizeof(PointSummary)
    for i in range(n):
        assert raw[i * sz:(i + 1) * sz] == bytes(host[i]), i


def test_external_trace_full_size(sim):
    # a 100k-request user trace (load_trace path) shared by
    # the three policies: GPU (trace uploaded from page-locked memory, as the
    # CLI's bulk loader provides it) vs the oracle on the same rows
    import random
    n = 100_000
    lib = sim.lib
    lib.kvsim_gpu_host_alloc.restype = C.c_void_p
    lib.kvsim_gpu_host_alloc.argtypes = [C.c_size_t]
    lib.kvsim_gpu_host_free.argtypes = [C.c_void_p]
    bufs = [lib.kvsim_gpu_host_alloc(n * w) for w in (8, 4, 4)]
    assert all(bufs)
    try:
        arr = C.cast(bufs[0], C.POINTER(C.c_double))
        pl = C.cast(bufs[1], C.POINTER(C.c_int32))
        dl = C.cast(bufs[2], C.POINTER(C.c_int32))
        r = random.Random(11)
        t = 0.0
        for i in range(n):  # bursty conversation-shaped arrivals, long-tailed lengths
            t += r.expovariate(14.0 if (i // 500) % 2 else 6.0)
            arr[i] = t
            pl[i] = min(8000, int(r.paretovariate(1.3) * 200))
            dl[i] = r.randint(2, 1500)
        tv = TraceView(arr, pl, dl, n)
        pts = []
        for pol in ("unified", "splitwise", "accellm"):
            p = make_point(policy=pol, instances=8, num_requests=n, workload="mixed", seed=0)
            p.trace_index = 0
            pts.append(p)
        out = sim.run(pts, traces=[tv])
        for p, s in zip(pts, out):
            assert s.status == 0 and s.n_requests == n
            ref = run_oracle(p, trace=tv, ev_cap=0, recs=False)
            assert not diff_results(ref, Result(s, None, None), events=False), p.policy
    finally:
        for b in bufs:
            lib.kvsim_gpu_host_free(b)
