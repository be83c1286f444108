"""kvsim on B200: warp-per-point sweep of the AcceLLM serving simulator.

Python host mirror of the reference-facing C-ABI (include/kvsim_gpu.h). The
reference's own entry points are C++ (`kvsim run|sweep`, reference
SPEC.md:400-455; perfmodel API reference proj/include/kvsim/perfmodel.hpp);
this module exposes the same operations for tests and benchmarks:

    sim = KvSim(device=0)
    summaries = sim.run(points)                       # cmd_sweep point loop
    summaries, records, events = sim.run(points, records=True, events=4096)

There is no CPU fallback: if the CUDA library is missing or no sm_100 device
is visible, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .abi import (EventRecord, InstanceRecord, MultiStats, PointDesc, PointSummary, RequestRecord, RunOpts,  # noqa: F401
                  TraceView,
                  make_point, points_array, summary_dict, STATUS, POLICY, POLICY_NAME,
                  DEVICES, MODELS, WORKLOADS, SUMMARY_CSV)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVSIM_LIB") or os.path.join(_HERE, "_build", "libkvsim_gpu.so")
CLI_PATH = os.path.join(_HERE, "_build", "kvsim")

_lib = None


class KvSimError(RuntimeError):
    pass


def load_library() -> C.CDLL:
    """Load the sm_100a library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("KVSIM_LIB", LIB_PATH)  # build-variant experiments (tools/)
    if not os.path.exists(path):
        raise KvSimError(f"CUDA library not built: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    L.kvsim_gpu_abi_version.restype = C.c_int
    L.kvsim_gpu_device_count.restype = C.c_int
    L.kvsim_gpu_open.argtypes = [C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]
    L.kvsim_gpu_close.argtypes = [C.c_void_p]
    L.kvsim_point_defaults.argtypes = [C.POINTER(PointDesc)]
    L.kvsim_point_validate.argtypes = [C.POINTER(PointDesc), C.c_char_p, C.c_size_t]
    L.kvsim_gpu_run.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.c_size_t, C.POINTER(TraceView), C.c_size_t,
                                C.POINTER(PointSummary), C.POINTER(RequestRecord), C.POINTER(EventRecord),
                                C.c_size_t, C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]
    L.kvsim_gpu_run_ex.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.c_size_t, C.POINTER(TraceView), C.c_size_t,
                                   C.POINTER(PointSummary), C.POINTER(RunOpts), C.c_char_p, C.c_size_t]
    L.kvsim_gpu_run_multi.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(PointDesc), C.c_size_t,
                                      C.POINTER(PointSummary), C.c_size_t, C.POINTER(MultiStats), C.c_char_p,
                                      C.c_size_t]
    if hasattr(L, "kvsim_gpu_curves"):  # (absent only in older build variants, tools/ab_inproc.py)
        L.kvsim_gpu_curves.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.POINTER(C.c_int64), C.c_size_t,
                                       C.POINTER(C.c_int64), C.c_size_t, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    L.kvsim_gpu_run_device.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                       C.c_char_p, C.c_size_t]
    L.kvsim_gpu_reserve.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.c_size_t, C.c_char_p, C.c_size_t]
    L.kvsim_gpu_last_launches.argtypes = [C.c_void_p]
    L.kvsim_gpu_last_launches.restype = C.c_int64
    L.kvsim_gpu_point_times.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]
    L.kvsim_gpu_point_times.restype = C.c_int64
    L.kvsim_gpu_perf_batch.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.c_size_t, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double), C.c_size_t, C.c_char_p, C.c_size_t]
    L.kvsim_gpu_gen_trace.argtypes = [C.c_void_p, C.POINTER(PointDesc), C.POINTER(C.c_double),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                      C.c_char_p, C.c_size_t]
    _lib = L
    return L


class KvSim:
    """One device context (kvsim_gpu_open)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.err = C.create_string_buffer(512)
        h = C.c_void_p()
        rc = self.lib.kvsim_gpu_open(device, C.byref(h), self.err, 512)
        if rc != 0:
            raise KvSimError(f"kvsim_gpu_open({device}) failed [{rc}]: {self.err.value.decode()}")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.kvsim_gpu_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != 0:
            raise KvSimError(f"{what} failed [{rc}]: {self.err.value.decode()}")

    def run(self, points, traces=None, records: bool = False, events: int = 0, detail: bool = False,
            instances: bool = False):
        """Run points (list of PointDesc). Returns summaries, or (summaries,
        records per point, events per point) when records/events requested.
        detail: pooled TBT percentiles (kvsim_run_opts.detail); instances:
        per-instance records, afterwards in self.last_instances."""
        n = len(points)
        P = (PointDesc * n)(*points)
        S = (PointSummary * n)()
        tot = sum(max(int(p.num_requests), 0) for p in points)
        R = (RequestRecord * max(tot, 1))() if records else None
        E = (EventRecord * max(events * n, 1))() if events else None
        cnt = (C.c_int64 * n)() if events else None
        I = (InstanceRecord * (32 * n))() if instances else None
        T, nt = None, 0
        if traces:
            nt = len(traces)
            T = (TraceView * nt)(*traces)
        if detail or instances:
            o = RunOpts()
            o.detail = 1 if detail else 0
            o.recs = R
            o.ev = C.cast(E, C.c_void_p) if E is not None else None
            o.ev_cap = events
            o.ev_count = cnt
            o.inst = I
            rc = self.lib.kvsim_gpu_run_ex(self.h, P, n, T, nt, S, C.byref(o), self.err, 512)
        else:
            rc = self.lib.kvsim_gpu_run(self.h, P, n, T, nt, S, R, E, events, cnt, self.err, 512)
        self._check(rc, "kvsim_gpu_run")
        summaries = list(S)
        self.last_event_counts = list(cnt) if events else None
        self.last_instances = ([list(I[32 * i:32 * i + points[i].num_instances]) for i in range(n)]
                               if instances else None)
        if not records and not events:
            return summaries
        recs_out, ev_out, off = [], [], 0
        for i, p in enumerate(points):
            nr = max(int(p.num_requests), 0)
            recs_out.append(R[off:off + summaries[i].n_requests] if records else None)
            off += nr
            ev_out.append(E[i * events:i * events + min(cnt[i], events)] if events else None)
        return summaries, recs_out, ev_out

    def reserve(self, points):
        n = len(points)
        P = (PointDesc * n)(*points)
        self._check(self.lib.kvsim_gpu_reserve(self.h, P, n, self.err, 512), "kvsim_gpu_reserve")

    def run_device(self, d_points_ptr: int, n: int, d_out_ptr: int, stream_ptr: int = 0):
        rc = self.lib.kvsim_gpu_run_device(self.h, C.c_void_p(d_points_ptr), n, C.c_void_p(d_out_ptr),
                                           C.c_void_p(stream_ptr), self.err, 512)
        self._check(rc, "kvsim_gpu_run_device")

    def last_launches(self) -> int:
        return int(self.lib.kvsim_gpu_last_launches(self.h))

    def point_times(self, n: int):
        """Profiling: [(start_ns, end_ns, slot)] per point of the last run
        (context opened with KVSIM_POINT_TIMES set), else []."""
        buf = (C.c_uint64 * (3 * n))()
        k = int(self.lib.kvsim_gpu_point_times(self.h, buf, 3 * n))
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(max(k, 0) // 3)]

    def perf_batch(self, points, pidx, ops, s1, s2):
        n = len(pidx)
        P = (PointDesc * len(points))(*points)
        a = (C.c_int32 * n)(*pidx)
        o = (C.c_int32 * n)(*ops)
        x = (C.c_int64 * n)(*s1)
        y = (C.c_int64 * n)(*s2)
        out = (C.c_double * n)()
        rc = self.lib.kvsim_gpu_perf_batch(self.h, P, len(points), a, o, x, y, out, n, self.err, 512)
        self._check(rc, "kvsim_gpu_perf_batch")
        return list(out)

    def curves(self, point, lengths, batch_sizes, phase: str = "decode"):
        """throughput_curves on the device (K1): [(length, batch, latency_s, tokens_per_s)]."""
        nl, nb = len(lengths), len(batch_sizes)
        Ls = (C.c_int64 * nl)(*lengths)
        Bs = (C.c_int64 * nb)(*batch_sizes)
        lat = (C.c_double * (nl * nb))()
        tps = (C.c_double * (nl * nb))()
        rc = self.lib.kvsim_gpu_curves(self.h, C.byref(point), Ls, nl, Bs, nb, 0 if phase == "prefill" else 1, lat,
                                       tps, self.err, 512)
        self._check(rc, "kvsim_gpu_curves")
        return [(lengths[i // nb], batch_sizes[i % nb], lat[i], tps[i]) for i in range(nl * nb)]

    def gen_trace(self, point):
        cap = max(int(point.num_requests), 1)
        arr = (C.c_double * cap)()
        pl = (C.c_int32 * cap)()
        dl = (C.c_int32 * cap)()
        nn = C.c_int64(0)
        rc = self.lib.kvsim_gpu_gen_trace(self.h, C.byref(point), arr, pl, dl, C.byref(nn), self.err, 512)
        self._check(rc, "kvsim_gpu_gen_trace")
        k = nn.value
        return list(arr)[:k], list(pl)[:k], list(dl)[:k]


def run_multi(sims, points, min_chunk: int = 0):
    """One sweep sharded over the devices of `sims` (open KvSim contexts on
    distinct GPUs): kvsim_gpu_run_multi, one host thread per device, guided
    chunks over the cost-sorted points, no collective. Returns (summaries in
    point order, MultiStats)."""
    L = load_library()
    n = len(points)
    P = (PointDesc * n)(*points)
    S = (PointSummary * n)()
    H = (C.c_void_p * len(sims))(*[s.h.value for s in sims])
    st = MultiStats()
    err = C.create_string_buffer(512)
    rc = L.kvsim_gpu_run_multi(H, len(sims), P, n, S, min_chunk, C.byref(st), err, 512)
    if rc != 0:
        raise KvSimError(f"kvsim_gpu_run_multi failed [{rc}]: {err.value.decode()}")
    return list(S), st


def trace_view(arrival, prompt, decode):
    """Build a TraceView (keeps the backing arrays alive on the object)."""
    n = len(arrival)
    a = (C.c_double * max(n, 1))(*arrival)
    p = (C.c_int32 * max(n, 1))(*prompt)
    d = (C.c_int32 * max(n, 1))(*decode)
    tv = TraceView(C.cast(a, C.POINTER(C.c_double)), C.cast(p, C.POINTER(C.c_int32)),
                   C.cast(d, C.POINTER(C.c_int32)), n)
    tv._keep = (a, p, d)
    return tv
