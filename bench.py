"""bench.py — simulated requests/s of a kvsim sweep on B200 (BASELINE.json metric).

Workload (N=1): BASELINE config 4 — 3 policies x instance counts {4,8,12,16} x
833 request rates linearly spaced in (0, 3*N_inst] req/s, 10k requests per
point, mixed workload, Llama-2-70B on simulated H100 instances, seed = point
index (9,996 points, ~1e8 simulated requests). A step = one full sweep.

  value  device-resident sweep (points already in HBM), CUDA events on the
         launch stream, max over ranks
  e2e    the same sweep through the reference-facing C-ABI call with host
         buffers (kvsim_gpu_run: H2D points, kernel, D2H summaries)
  --impl reference  the CPU oracle (restated reference simulator) on all host
         threads over a bounded sample of the same points

Multi-GPU (--gpus N, or torchrun with N ranks): ONE process drives all N
GPUs with one host thread each (kvsim_gpu_run_multi: points dealt by cost,
summaries gathered in host memory, no collective). `value` is
weak scaling: N config-4 grids with disjoint seeds in one sweep over the N
GPUs. Under torchrun, ranks other than 0 exit without work. Every run also
times a fixed BASELINE config-5 subsample (`config5_slice`, strong scaling:
the same 9,014 points on 1 or N GPUs).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2411_05555_b200.abi import PointDesc, PointSummary, make_point  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def config4_points(seed_base=0, n_rates=833, n_req=10000, policies=("unified", "splitwise", "accellm"),
                   instances=(4, 8, 12, 16)):
    pts = []
    k = 0
    for pol in policies:
        for ni in instances:
            for j in range(n_rates):
                rate = 3.0 * ni * (j + 1) / n_rates
                pts.append(make_point(model="llama2-70b", device="h100", policy=pol, instances=ni, rate=rate,
                                      num_requests=n_req, workload="mixed", seed=seed_base + k, user_tag=k))
                k += 1
    return pts


def config5_points(stride=111, n_req=100000):
    """BASELINE config 5: 3 policies x {H100, 910B2} x 250
    log-spaced rates in [0.5, 30] req/s x 667 seeds = 1,000,500 points of
    70B / 8 instances / mixed / 100k requests; every stride-th point."""
    import math
    pts = []
    k = 0
    for pol in ("unified", "splitwise", "accellm"):
        for dev in ("h100", "910b2"):
            for j in range(250):
                rate = 0.5 * math.exp(math.log(60.0) * j / 249)
                for sd in range(667):
                    if k % stride == 0:
                        pts.append(make_point(model="llama2-70b", device=dev, policy=pol, instances=8, rate=rate,
                                              num_requests=n_req, workload="mixed", seed=sd, user_tag=k))
                    k += 1
    return pts


def algorithmic_bytes(summaries):
    # B_req = 16 (trace) + 24 (TTFT/TBT/JCT record) + 8 * S_req,
    # S_req = decode iterations = decode_len - 1 => sum = tokens_total - n_requests
    n = sum(s.n_requests for s in summaries)
    tok = sum(s.tokens_total for s in summaries)
    return 40 * n + 8 * (tok - n)


NCU_TRAFFIC_FILE = "profiles/r2_ncu_bench_kernel.json"


def ncu_traffic():
    """DRAM bytes per launch of the config-4 sweep kernel from the committed ncu
    capture of this build (NCU_TRAFFIC_FILE), or None."""
    p = os.path.join(ROOT, NCU_TRAFFIC_FILE)
    try:
        return float(json.load(open(p))["dram_bytes_per_launch"])
    except Exception:
        return None


def ncu_inst_per_launch():
    """Warp instructions per launch (smsp__inst_executed.sum) of the config-4
    sweep kernel from the same committed ncu capture, or None."""
    try:
        return float(json.load(open(os.path.join(ROOT, NCU_TRAFFIC_FILE)))["smsp__inst_executed.sum"])
    except Exception:
        return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    def __init__(self, device=0):
        self.samples = []
        self.stop = threading.Event()
        self.device = device
        self.proc = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.device),
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", "-lms", "200"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for nm, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sweep(points, threads):
    """Run the CPU oracle (restated reference simulator, test infrastructure)
    on `points`, one point per host thread. Returns
    (summaries, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from harness import oracle  # the checker / CPU baseline only
    L = oracle()
    P = (PointDesc * len(points))(*points)
    S = (PointSummary * len(points))()
    t0 = time.perf_counter()
    L.kvo_run_sweep(P, len(points), threads, S)
    return S, time.perf_counter() - t0


def parity_check(gpu, cpu):
    """Bitwise comparison of every summary field (GPU == oracle)."""
    def key(x):
        y = PointSummary.from_buffer_copy(bytes(x))
        y.reserved[0] = 0  # kernel-only diagnostic (event-loop iterations)
        return bytes(y)
    bad = [i for i, (a, b) in enumerate(zip(gpu, cpu)) if key(a) != key(b)]
    return {"checked": len(cpu), "mismatches": len(bad), "first_mismatch": bad[0] if bad else None,
            "fields": "all kvsim_point_summary fields, bit for bit"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kvsim", choices=["kvsim", "reference"])
    ap.add_argument("--rates", type=int, default=833)
    ap.add_argument("--requests", type=int, default=10000)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the full-size CPU oracle baseline / parity check")
    ap.add_argument("--c5-stride", type=int, default=111, help="config-5 subsample stride (0 = skip)")
    ap.add_argument("--c5-requests", type=int, default=100000)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_cpu = os.cpu_count() or 1
    metric = "simulated requests/sec (sweep, 1-8 B200) vs ref CPU; HBM GB/s fraction"
    workload_is_config4 = args.rates == 833 and args.requests == 10000
    workload = (f"BASELINE config 4: 3 policies x instances {{4,8,12,16}} x {args.rates} rates in (0,3N] req/s, "
                f"{args.requests} requests/point, mixed, Llama-2-70B on simulated H100")

    if args.impl == "reference":
        # The reference's own CPU path does not exist; its restated
        # simulator (the oracle) runs on every host thread. The K timed steps
        # together cover the whole config-4 grid exactly once: step s runs
        # points s, s+K, s+2K, ... (each a bounded, interleaved 1/K sample).
        if rank != 0:
            return
        pts = config4_points(0, args.rates, args.requests)
        for w in range(args.warmup):
            oracle_sweep(pts[w::max(1, len(pts) // 64)], n_cpu)
        K = max(args.steps, 1)
        times, reqs = [], 0
        for st in range(K):
            S, dt = oracle_sweep(pts[st::K], n_cpu)
            times.append(dt)
            reqs += sum(x.n_requests for x in S if x.status == 0)
        v = reqs / sum(times)
        line = {"metric": metric, "value": v, "unit": "simulated requests/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / K * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (the seeded generator of SEMANTICS §2, same traces as the GPU arm)",
                "impl": "reference",
                "config": {"workload": workload, "parallelism": f"{n_cpu} host threads, one point per thread"},
                "cpu_baseline": {"value": v, "unit": "simulated requests/s", "cores": n_cpu, "kind": "port",
                                 "cpu_model": cpu_model(),
                                 "sample": f"all {len(pts)} points x {args.requests} requests, split into {K} "
                                           f"interleaved steps (step s = points s, s+{K}, ...); "
                                           f"{sum(times):.1f} s in total"},
                "e2e": {"value": v, "unit": "simulated requests/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if rank != 0:
        # one process drives every GPU (one host thread per device, no
        # collective); under torchrun the other ranks have nothing to do
        return
    n_gpu = max(args.gpus, world)
    import torch
    import paper_2411_05555_b200 as pkg
    # KVSIM_VIRTUAL_GPUS=1 maps the N contexts onto the visible devices
    # round-robin: a functional check of the N>1 path on a smaller box, never
    # a scaling number
    ndev = torch.cuda.device_count()
    if n_gpu > ndev and os.environ.get("KVSIM_VIRTUAL_GPUS") != "1":
        raise SystemExit(f"--gpus {n_gpu} but only {ndev} visible device(s)")
    sims = [pkg.KvSim(d % max(ndev, 1)) for d in range(n_gpu)]
    sim = sims[0]
    # weak scaling: N copies of the config-4 grid with disjoint seeds, one
    # sweep sharded over the N GPUs by kvsim_gpu_run_multi
    pts = [p for r in range(n_gpu) for p in config4_points(r * 1_000_000, args.rates, args.requests)]
    n = len(pts)
    with ClockSampler(0) as clk:
        if n_gpu == 1:
            # device-resident: points and summaries in HBM (torch owns the memory)
            dev = 0
            torch.cuda.set_device(dev)
            P = (PointDesc * n)(*pts)
            d_pts = torch.frombuffer(bytearray(bytes(P)), dtype=torch.uint8).to(f"cuda:{dev}")
            d_out = torch.empty(n * C.sizeof(PointSummary), dtype=torch.uint8, device=f"cuda:{dev}")
            sim.reserve(pts)
            stream = torch.cuda.Stream(dev)  # non-default stream: the kernels and the events share it

            def step():
                sim.run_device(d_pts.data_ptr(), n, d_out.data_ptr(), stream.cuda_stream)

            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize(dev)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            torch.cuda.synchronize(dev)
            with torch.cuda.stream(stream):
                for a, b in ev:
                    a.record(stream)
                    step()
                    b.record(stream)
            torch.cuda.synchronize(dev)
            launches = args.steps * sim.last_launches()
            t_total = sum(a.elapsed_time(b) / 1e3 for a, b in ev)
            summ = (PointSummary * n).from_buffer_copy(d_out.cpu().numpy().tobytes())
        else:
            # sharded over n_gpu devices: per step, the max over devices of
            # the CUDA-event time from its first chunk to its last
            for _ in range(args.warmup):
                pkg.run_multi(sims, pts)
            t_total, launches = 0.0, 0
            for _ in range(args.steps):
                summ, st = pkg.run_multi(sims, pts)
                t_total += max(st.device_seconds[i] for i in range(n_gpu))
                launches += sum(st.device_launches[i] for i in range(n_gpu))
    bad = sum(1 for s in summ if s.status != 0)
    # failed points (e.g. an exceeded event budget) did not simulate all of
    # their requests: they do not count towards the throughput
    reqs = sum(s.n_requests for s in summ if s.status == 0)
    value = reqs * args.steps / t_total
    kernel_s = t_total / args.steps
    bytes_alg = algorithmic_bytes(summ)
    peaks, src = measured_peaks()
    achieved = bytes_alg / kernel_s / 1e9 / n_gpu  # per GPU
    events = sum(s.n_events for s in summ)

    # e2e: the reference-facing C-ABI call itself (kvsim_gpu_run, or
    # kvsim_gpu_run_multi for N GPUs) on page-locked host buffers from
    # kvsim_gpu_host_alloc, as the C++ CLI calls it: every step copies the
    # points host->device, simulates, and copies the summaries back inside
    # the call. (Filling the host buffers from Python objects is the
    # caller's, outside the timed region.)
    e2e = None
    if not args.no_e2e:
        L = pkg.load_library()
        L.kvsim_gpu_host_alloc.restype = C.c_void_p
        L.kvsim_gpu_host_alloc.argtypes = [C.c_size_t]
        L.kvsim_gpu_host_free.argtypes = [C.c_void_p]
        h2d = n * C.sizeof(PointDesc)
        d2h = n * C.sizeof(PointSummary)
        hp, hs = L.kvsim_gpu_host_alloc(h2d), L.kvsim_gpu_host_alloc(d2h)
        if not hp or not hs:
            raise SystemExit("kvsim_gpu_host_alloc failed")
        HP = (PointDesc * n).from_address(hp)
        HS = (PointSummary * n).from_address(hs)
        C.memmove(hp, (PointDesc * n)(*pts), h2d)
        err = C.create_string_buffer(512)
        H = (C.c_void_p * n_gpu)(*[s_.h.value for s_ in sims])
        mst = pkg.MultiStats()
        tt = []
        for i in range(max(1, args.steps)):
            t0 = time.perf_counter()
            if n_gpu == 1:
                rc = L.kvsim_gpu_run(sim.h, HP, n, None, 0, HS, None, None, 0, None, err, 512)
            else:
                rc = L.kvsim_gpu_run_multi(H, n_gpu, HP, n, HS, 0, C.byref(mst), err, 512)
            tt.append(time.perf_counter() - t0)
            if rc != 0:
                raise SystemExit(f"e2e C-ABI call failed [{rc}]: {err.value.decode()}")
        assert all(bytes(HS[i]) == bytes(summ[i]) for i in range(n)), "e2e results differ from the timed run"
        L.kvsim_gpu_host_free(hp)
        L.kvsim_gpu_host_free(hs)
        e2e = {"value": reqs * len(tt) / sum(tt), "unit": "simulated requests/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "seconds_per_call": [round(x, 4) for x in tt],
               "path": ("kvsim_gpu_run" if n_gpu == 1 else f"kvsim_gpu_run_multi over {n_gpu} GPUs") +
                       " on page-locked host buffers (kvsim_gpu_host_alloc), wall clock per call"}

    # BASELINE config 5 slice (70B, 8 instances, mixed, 3
    # policies x {H100, 910B2} x 250 rates x 667 seeds, 100k requests each):
    # every c5_stride-th point, sharded over the same GPUs
    c5 = None
    if args.c5_stride > 0:
        c5p = config5_points(args.c5_stride, args.c5_requests)
        pkg.run_multi(sims, c5p[-4 * 148:])  # warm-up (cheap high-rate points): arenas, instruction caches
        t0 = time.perf_counter()
        c5s, st = pkg.run_multi(sims, c5p)
        wall = time.perf_counter() - t0
        c5r = sum(x.n_requests for x in c5s if x.status == 0)
        dev_s = max(st.device_seconds[i] for i in range(n_gpu))
        c5 = {"workload": f"BASELINE config 5 subsample: every {args.c5_stride}th of 1,000,500 points "
                          f"({len(c5p)} points x {args.c5_requests} requests)",
              "value": c5r / dev_s, "e2e": c5r / wall, "unit": "simulated requests/s", "n_gpus": n_gpu,
              "ms": dev_s * 1e3, "failed_points": sum(1 for x in c5s if x.status != 0),
              "points_per_gpu": [int(st.device_points[i]) for i in range(n_gpu)]}
        if not args.no_cpu:
            # every 150th point of the slice (all policies, both devices)
            # re-simulated on the CPU oracle, compared bit for bit
            idx = list(range(0, len(c5p), 150))
            S_c5, _ = oracle_sweep([c5p[i] for i in idx], n_cpu)
            c5["parity"] = parity_check([c5s[i] for i in idx], S_c5)

    cpu, parity = None, None
    if n_gpu == 1 and not args.no_cpu:
        # the full sweep on the CPU oracle (all host threads): both the
        # cpu_baseline and a bitwise check of every GPU summary
        S_cpu, dt = oracle_sweep(pts, n_cpu)
        v = sum(x.n_requests for x in S_cpu if x.status == 0) / dt
        cpu = {"value": v, "unit": "simulated requests/s", "cores": n_cpu, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"the full sweep ({n} points x {args.requests} requests), {dt:.1f} s on {n_cpu} host "
                         f"threads (CPU oracle, one point per thread)"}
        parity = parity_check(summ, S_cpu)

    # the binding resource: warp-instruction issue. Achieved =
    # the committed ncu capture's warp instructions per launch / this run's
    # per-launch time; peak = one warp instruction per scheduler per cycle
    # (4 per SM) at the median SM clock sampled during the timed region
    issue = None
    inst = ncu_inst_per_launch()
    clk_s = clk.summary()
    if workload_is_config4 and n_gpu == 1 and inst and clk_s.get("sm_mhz"):
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        ach = inst / kernel_s
        peak = sms * 4 * clk_s["sm_mhz"] * 1e6
        issue = {"achieved": ach, "peak": peak, "unit": "warp instructions/s", "frac": ach / peak,
                 "inst_per_launch": inst, "source": NCU_TRAFFIC_FILE + " (smsp__inst_executed.sum) / this run's time",
                 "inst_per_simulated_request": inst / max(reqs, 1)}

    line = {
        "metric": metric, "value": value, "unit": "simulated requests/s", "n_gpus": n_gpu,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": kernel_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: requests generated on device by the seeded counter-based RNG (SEMANTICS §2)",
        "config": {"workload": workload + (f", x{n_gpu} grids with disjoint seeds (weak scaling)" if n_gpu > 1 else ""),
                   "points": n, "requests_per_step": reqs,
                   "parallelism": f"one sweep sharded over {n_gpu} GPU(s) by one process (host thread per GPU, "
                                  f"LPT-dealt points, no collective), warp per point",
                   "l2": "arena working set >> 126 MB L2 and rewritten every step (no flush needed)"},
        "gpu_launches": launches,
        "events_per_step": events,
        "failed_points": bad,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"),
                     "unit": "GB/s", "frac": achieved / peaks.get("hbm_gbs"),
                     "traffic": ncu_traffic() if workload_is_config4 else None,
                     "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum of the "
                                     "config-4 sweep kernel, " + NCU_TRAFFIC_FILE + ")",
                     "peak_source": src,
                     "algorithmic_bytes_per_launch": bytes_alg,
                     "note": "algorithmic bytes per SURVEY §8d (40 B/request + 8 B/decode iteration), per GPU; "
                             "the kernel is bound by instruction issue/fetch, not HBM (DESIGN.md §7)"},
        "issue": issue,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "config5_slice": c5,
    }
    print(json.dumps(line), flush=True)
    for s_ in sims:
        s_.close()


if __name__ == "__main__":
    main()
