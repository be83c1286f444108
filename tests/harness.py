"""Shared test helpers: load the oracle (checker), the SIMT emulator build of
the kernel core (CPU CI) and the product CUDA library; run points; diff."""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

from paper_2411_05555_b200.abi import (EventRecord, InstanceRecord, PointDesc, PointSummary, RequestRecord,
                                       TraceView, SUMMARY_FLOAT_FIELDS, SUMMARY_INT_FIELDS)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libkvsim_oracle.so")
EMU_SO = os.path.join(ROOT, "tests", "_build", "libkvsim_emu.so")

_oracle = None
_emu = None


def build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def build_emu():
    src = os.path.join(ROOT, "tests", "emu", "kvsim_emu.cpp")
    os.makedirs(os.path.dirname(EMU_SO), exist_ok=True)
    deps = [src] + [os.path.join(ROOT, "paper_2411_05555_b200", "csrc", f)
                    for f in os.listdir(os.path.join(ROOT, "paper_2411_05555_b200", "csrc"))]
    if os.path.exists(EMU_SO) and all(os.path.getmtime(d) <= os.path.getmtime(EMU_SO) for d in deps):
        return
    subprocess.run(["g++", "-DKVSIM_EMU", "-O2", "-std=gnu++20", "-ffp-contract=off", "-fPIC", "-shared",
                    "-I" + os.path.join(ROOT, "include"), "-o", EMU_SO, src, "-lpthread"], check=True)


def oracle():
    global _oracle
    if _oracle is None:
        build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.kvo_run_point.argtypes = [C.POINTER(PointDesc), C.POINTER(TraceView), C.POINTER(PointSummary),
                                    C.POINTER(RequestRecord), C.POINTER(EventRecord), C.c_int64,
                                    C.POINTER(C.c_int64)]
        L.kvo_run_point_ex.argtypes = [C.POINTER(PointDesc), C.POINTER(TraceView), C.POINTER(PointSummary),
                                       C.POINTER(RequestRecord), C.POINTER(EventRecord), C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(InstanceRecord), C.c_int]
        L.kvo_run_sweep.argtypes = [C.POINTER(PointDesc), C.c_int64, C.c_int, C.POINTER(PointSummary)]
        L.kvo_run_sweep_ex.argtypes = [C.POINTER(PointDesc), C.c_int64, C.c_int, C.POINTER(PointSummary),
                                       C.POINTER(InstanceRecord), C.c_int]
        for fn in ("kvo_prefill_latency", "kvo_decode_step_latency"):
            getattr(L, fn).restype = C.c_double
            getattr(L, fn).argtypes = [C.POINTER(PointDesc), C.c_int64, C.c_int64]
        L.kvo_transfer_latency.restype = C.c_double
        L.kvo_transfer_latency.argtypes = [C.POINTER(PointDesc), C.c_double]
        L.kvo_kv_bytes_per_token.restype = C.c_double
        L.kvo_kv_bytes_per_token.argtypes = [C.POINTER(PointDesc)]
        L.kvo_weight_bytes.restype = C.c_double
        L.kvo_weight_bytes.argtypes = [C.POINTER(PointDesc)]
        L.kvo_kv_capacity_tokens.argtypes = [C.POINTER(PointDesc), C.POINTER(C.c_int64)]
        L.kvo_klog.restype = C.c_double
        L.kvo_klog.argtypes = [C.c_double]
        L.kvo_rng_draw.restype = C.c_uint64
        L.kvo_rng_draw.argtypes = [C.c_uint64, C.c_int64, C.c_int]
        L.kvo_gen_trace.restype = C.c_int64
        L.kvo_gen_trace.argtypes = [C.POINTER(PointDesc), C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.c_int64]
        _oracle = L
    return _oracle


def emu():
    global _emu
    if _emu is None:
        build_emu()
        L = C.CDLL(EMU_SO)
        L.kvemu_run.argtypes = [C.POINTER(PointDesc), C.c_int64, C.POINTER(TraceView), C.c_int64,
                                C.POINTER(PointSummary), C.POINTER(RequestRecord), C.POINTER(EventRecord),
                                C.c_int64, C.POINTER(C.c_int64), C.c_int, C.POINTER(InstanceRecord), C.c_int]
        _emu = L
    return _emu


class Result:
    def __init__(self, summary, recs, events, status=0, ev_total=None, inst=None):
        self.summary = summary
        self.recs = recs
        self.events = events
        self.status = status
        self.inst = inst
        # total events produced (may exceed the captured log)
        self.ev_total = ev_total if ev_total is not None else (len(events) if events is not None else None)


def run_oracle(p: PointDesc, trace: TraceView | None = None, ev_cap: int = 0, recs: bool = True,
               detail: bool = False, inst: bool = True) -> Result:
    L = oracle()
    s = PointSummary()
    nrec = max(int(p.num_requests), 0)
    R = (RequestRecord * max(nrec, 1))() if recs else None
    E = (EventRecord * max(ev_cap, 1))() if ev_cap else None
    I = (InstanceRecord * 32)() if inst else None
    cnt = C.c_int64(0)
    st = L.kvo_run_point_ex(C.byref(p), C.byref(trace) if trace is not None else None, C.byref(s), R, E, ev_cap,
                            C.byref(cnt), I, 1 if detail else 0)
    n = s.n_requests
    return Result(s, R[:n] if recs else None, E[:min(cnt.value, ev_cap)] if ev_cap else None, st, cnt.value,
                  list(I[:max(p.num_instances, 0)]) if inst and st == 0 else None)


def run_points_emu(points, traces=None, ev_cap: int = 0, recs: bool = True, warps: int = 2, detail: bool = False,
                   inst: bool = True):
    L = emu()
    n = len(points)
    P = (PointDesc * n)(*points)
    S = (PointSummary * n)()
    I = (InstanceRecord * (32 * n))() if inst else None
    tot = sum(max(int(p.num_requests), 0) for p in points)
    R = (RequestRecord * max(tot, 1))() if recs else None
    E = (EventRecord * max(ev_cap * n, 1))() if ev_cap else None
    cnt = (C.c_int64 * n)()
    T = None
    nt = 0
    if traces:
        nt = len(traces)
        T = (TraceView * nt)(*traces)
    L.kvemu_run(P, n, T, nt, S, R, E, ev_cap, cnt, warps, I, 1 if detail else 0)
    out = []
    off = 0
    for i, p in enumerate(points):
        s = S[i]
        nr = max(int(p.num_requests), 0)
        rr = R[off:off + s.n_requests] if recs else None
        off += nr
        ee = E[i * ev_cap:i * ev_cap + min(cnt[i], ev_cap)] if ev_cap else None
        ii = list(I[32 * i:32 * i + p.num_instances]) if inst and s.status == 0 else None
        out.append(Result(s, rr, ee, s.status, cnt[i], ii))
    return out


def _bits(x: float) -> int:
    import struct
    return struct.unpack("<q", struct.pack("<d", x))[0]


def feq(a: float, b: float) -> bool:
    if math.isnan(a) and math.isnan(b):
        return True
    return _bits(a) == _bits(b)


def ev_key(e):
    return (e.t, e.kind, e.inst, e.a, e.b, e.c)


def diff_results(a: Result, b: Result, *, events: bool = True) -> list[str]:
    """Bit-exact comparison; returns a list of differences (empty = identical)."""
    errs = []
    for f in SUMMARY_INT_FIELDS:
        if f in ("reserved",):
            continue
        va, vb = getattr(a.summary, f), getattr(b.summary, f)
        if va != vb:
            errs.append(f"summary.{f}: {va} != {vb}")
    for f in SUMMARY_FLOAT_FIELDS:
        va, vb = getattr(a.summary, f), getattr(b.summary, f)
        if not feq(va, vb):
            errs.append(f"summary.{f}: {va!r} != {vb!r}")
    if a.recs is not None and b.recs is not None:
        if len(a.recs) != len(b.recs):
            errs.append(f"records: {len(a.recs)} != {len(b.recs)}")
        for i, (ra, rb) in enumerate(zip(a.recs, b.recs)):
            for f, _ in RequestRecord._fields_:
                va, vb = getattr(ra, f), getattr(rb, f)
                ok = feq(va, vb) if isinstance(va, float) else va == vb
                if not ok:
                    errs.append(f"rec[{i}].{f}: {va!r} != {vb!r}")
                    break
            if len(errs) > 20:
                break
    if a.inst is not None and b.inst is not None:
        for i, (ra, rb) in enumerate(zip(a.inst, b.inst)):
            for f, _ in InstanceRecord._fields_:
                va, vb = getattr(ra, f), getattr(rb, f)
                ok = feq(va, vb) if isinstance(va, float) else va == vb
                if not ok:
                    errs.append(f"inst[{i}].{f}: {va!r} != {vb!r}")
    if events and a.events is not None and b.events is not None:
        if a.ev_total != b.ev_total:
            errs.append(f"event totals: {a.ev_total} != {b.ev_total}")
        if len(a.events) < a.ev_total or len(b.events) < b.ev_total:
            errs.append(f"event log truncated ({len(a.events)}/{a.ev_total}); raise ev_cap")
            return errs
        ka = sorted(ev_key(e) for e in a.events)
        kb = sorted(ev_key(e) for e in b.events)
        if ka != kb:
            sa, sb = set(ka), set(kb)
            first = sorted((sa ^ sb))[:5]
            errs.append(f"events differ: {len(ka)} vs {len(kb)}; first diffs {first}")
    return errs


def oracle_sweep(points, detail=False, instances=True, threads=None):
    """All points on the oracle, one per host thread; (summaries, instance
    records per point or None)."""
    L = oracle()
    n = len(points)
    P = (PointDesc * n)(*points)
    S = (PointSummary * n)()
    I = (InstanceRecord * (32 * n))() if instances else None
    L.kvo_run_sweep_ex(P, n, threads or (os.cpu_count() or 1), S, I, 1 if detail else 0)
    inst = [list(I[32 * i:32 * i + points[i].num_instances]) for i in range(n)] if instances else None
    return list(S), inst
