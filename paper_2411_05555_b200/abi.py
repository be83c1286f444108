"""ctypes mirror of include/kvsim_gpu.h plus the reference's presets.

Presets restate reference perfmodel.hpp:67-69 / SPEC.md:32 (devices),
SPEC.md:119 (Llama-2-70B), SPEC.md:55,64 (Llama-2-7B example constants) and
SPEC.md:144 (workloads). Builder-defined presets (conversation, coding) are
marked as such in docs/SEMANTICS.md §2.
"""
from __future__ import annotations

import ctypes as C
import math

KVSIM_MAX_INSTANCES = 32
POLICY = {"unified": 0, "splitwise_static": 1, "splitwise": 1, "accellm": 2}
POLICY_NAME = {0: "unified", 1: "splitwise_static", 2: "accellm"}
ARRIVAL = {"poisson": 0, "fixed": 1, "fixed-interval": 1}
LINK = {"striped": 0, "single": 1, "single-link": 1}

STATUS = {
    0: "ok", -1: "invalid argument", -2: "model does not fit in instance memory",
    -3: "even instance count required", -4: "cuda error", -5: "no cuda device",
    -6: "event budget exceeded", -7: "out of device memory", -8: "empty batch",
    -9: "internal invariant violated",
}


class PointDesc(C.Structure):
    _fields_ = [
        ("param_count", C.c_double),
        ("num_layers", C.c_int32), ("hidden_dim", C.c_int32), ("num_kv_heads", C.c_int32),
        ("head_dim", C.c_int32), ("bytes_per_value", C.c_int32),
        ("policy", C.c_int32),
        ("peak_flops", C.c_double), ("hbm_capacity", C.c_double),
        ("hbm_bandwidth", C.c_double), ("link_bandwidth", C.c_double),
        ("num_devices", C.c_int32), ("tensor_parallel", C.c_int32),
        ("memory_reserve_fraction", C.c_double),
        ("compute_eff", C.c_double), ("mem_bw_eff", C.c_double), ("link_eff", C.c_double),
        ("link_mode", C.c_int32), ("num_instances", C.c_int32),
        ("num_prefill_instances", C.c_int32), ("prefill_token_budget", C.c_int32),
        ("prompt_min", C.c_int32), ("prompt_max", C.c_int32),
        ("decode_min", C.c_int32), ("decode_max", C.c_int32),
        ("arrival_process", C.c_int32), ("trace_index", C.c_int32),
        ("rate", C.c_double), ("duration_s", C.c_double), ("warmup_s", C.c_double),
        ("seed", C.c_uint64), ("num_requests", C.c_int64), ("user_tag", C.c_uint64),
        ("accellm_flags", C.c_int32), ("degraded_trigger_ticks", C.c_int32),
        ("splitwise_cobatch", C.c_int32), ("first_token_decode", C.c_int32), ("reserved_i", C.c_int32 * 4),
        ("policy_timer_s", C.c_double), ("leveling_link_fraction", C.c_double),
        ("degraded_redundancy", C.c_double), ("degraded_exit_fill", C.c_double),
        ("dual_copy_fraction", C.c_double), ("reserved_d", C.c_double * 2),
    ]


class TraceView(C.Structure):
    _fields_ = [
        ("arrival_s", C.POINTER(C.c_double)),
        ("prompt_len", C.POINTER(C.c_int32)),
        ("decode_len", C.POINTER(C.c_int32)),
        ("n", C.c_int64),
    ]


class PointSummary(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("num_instances", C.c_int32),
        ("n_requests", C.c_int64), ("n_completed", C.c_int64), ("n_measured", C.c_int64),
        ("tokens_total", C.c_int64), ("tokens_window", C.c_int64),
        ("n_events", C.c_int64), ("n_steps", C.c_int64), ("n_prefills", C.c_int64),
        ("n_moves", C.c_int64), ("n_preemptions", C.c_int64), ("n_evictions", C.c_int64),
        ("peak_kv_tokens", C.c_int64), ("link_prefill_tokens", C.c_int64),
        ("link_mirror_tokens", C.c_int64),
        ("makespan_s", C.c_double),
        ("ttft_mean", C.c_double), ("ttft_p50", C.c_double), ("ttft_p95", C.c_double),
        ("ttft_max", C.c_double),
        ("tbt_mean", C.c_double), ("tbt_max", C.c_double),
        ("jct_mean", C.c_double), ("jct_p50", C.c_double), ("jct_p95", C.c_double),
        ("jct_max", C.c_double),
        ("cost_eff", C.c_double), ("idle_frac", C.c_double), ("peak_kv_gb", C.c_double),
        ("link_prefill_gb", C.c_double), ("link_mirror_gb", C.c_double),
        ("busy_s_total", C.c_double),
        ("user_tag", C.c_uint64),
        ("link_leveling_tokens", C.c_int64), ("n_timer_ticks", C.c_int64),
        ("n_mode_switches", C.c_int64),
        # ABI v2 (kvsim_gpu.h): the rest of the MetricsReport
        ("ttft_queue_mean", C.c_double), ("tbt_p50", C.c_double), ("tbt_p95", C.c_double),
        ("idle_runnable_s", C.c_double), ("queue_depth_avg", C.c_double),
        ("queue_depth_max", C.c_int64), ("n_tbt_samples", C.c_int64),
        ("reserved", C.c_int64 * 1),
    ]


class RequestRecord(C.Structure):
    _fields_ = [
        ("arrival_s", C.c_double), ("first_token_s", C.c_double),
        ("completion_s", C.c_double), ("tbt_max_s", C.c_double),
        ("prompt_len", C.c_int32), ("decode_len", C.c_int32),
        ("n_moves", C.c_int32), ("n_preemptions", C.c_int32),
        ("prefill_start_s", C.c_double),
    ]


class InstanceRecord(C.Structure):
    _fields_ = [
        ("busy_s", C.c_double), ("idle_runnable_s", C.c_double),
        ("peak_kv_tokens", C.c_int64), ("initial_role", C.c_int32), ("reserved", C.c_int32),
    ]


class RunOpts(C.Structure):
    _fields_ = [
        ("detail", C.c_int32), ("reserved_i", C.c_int32 * 3),
        ("recs", C.POINTER(RequestRecord)),
        ("ev", C.c_void_p), ("ev_cap", C.c_size_t), ("ev_count", C.POINTER(C.c_int64)),
        ("inst", C.POINTER(InstanceRecord)),
    ]


KVSIM_MAX_DEVICES = 16


class MultiStats(C.Structure):
    _fields_ = [
        ("device_seconds", C.c_double * KVSIM_MAX_DEVICES),
        ("device_points", C.c_int64 * KVSIM_MAX_DEVICES),
        ("device_launches", C.c_int64 * KVSIM_MAX_DEVICES),
        ("n_devices", C.c_int32), ("reserved", C.c_int32),
    ]


class EventRecord(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("kind", C.c_int32), ("inst", C.c_int32),
        ("a", C.c_int32), ("b", C.c_int32), ("c", C.c_int64),
    ]


SUMMARY_INT_FIELDS = [n for n, t in PointSummary._fields_ if t in (C.c_int32, C.c_int64, C.c_uint64)]
SUMMARY_FLOAT_FIELDS = [n for n, t in PointSummary._fields_ if t is C.c_double]
# the 13 stable summary.csv columns (reference SPEC.md:442)
SUMMARY_CSV = ["policy", "rate", "ttft_mean", "ttft_p95", "tbt_mean", "tbt_max", "jct_mean",
               "jct_p95", "cost_eff", "idle_frac", "peak_kv_gb", "link_prefill_gb", "link_mirror_gb"]

# ------------------------------------------------------------------ presets
DEVICES = {
    # (peak_flops, hbm_capacity, hbm_bandwidth, link_bandwidth) — SPEC.md:32
    "910b2": (400e12, 64e9, 1.8e12, 392e9),
    "h100": (989e12, 80e9, 3.35e12, 900e9),
}
MODELS = {
    # (param_count, layers, hidden, kv_heads, head_dim, bytes) — SPEC.md:53-55,119
    "llama2-70b": (70e9, 80, 8192, 8, 128, 2),
    "llama2-7b": (7e9, 32, 4096, 32, 128, 2),
}
WORKLOADS = {
    # (prompt_min, prompt_max, decode_min, decode_max) — SPEC.md:144; * = builder preset
    "light": (20, 500, 20, 500),
    "mixed": (20, 1000, 20, 1000),
    "heavy": (500, 1000, 500, 1000),
    "conversation": (50, 1500, 50, 600),   # * builder preset (BASELINE config 2)
    "coding": (1000, 8000, 10, 200),       # * builder preset (BASELINE config 3)
}


def make_point(*, model="llama2-70b", device="h100", policy="accellm", instances=8,
               workload="mixed", rate=4.0, num_requests=1000, seed=0,
               arrival="poisson", eff=(0.5, 0.8, 0.8), link="striped",
               num_devices=4, reserve=0.10, warmup_s=0.0, duration_s=math.inf,
               prefill_budget=8192, num_prefill=0, prompt=None, decode=None,
               trace_index=-1, user_tag=0, degraded=False, leveling=False, timer_s=0.0,
               trigger_ticks=0, leveling_fraction=0.0, degraded_redundancy=0.0,
               degraded_exit_fill=0.0, dual_copy_fraction=0.0, cobatch=False,
               first_token_decode=False) -> PointDesc:
    p = PointDesc()
    (p.param_count, p.num_layers, p.hidden_dim, p.num_kv_heads, p.head_dim,
     p.bytes_per_value) = MODELS[model] if isinstance(model, str) else model
    (p.peak_flops, p.hbm_capacity, p.hbm_bandwidth, p.link_bandwidth) = (
        DEVICES[device] if isinstance(device, str) else device)
    p.num_devices = num_devices
    p.tensor_parallel = num_devices
    p.memory_reserve_fraction = reserve
    p.compute_eff, p.mem_bw_eff, p.link_eff = eff
    p.link_mode = LINK[link]
    p.policy = POLICY[policy] if isinstance(policy, str) else policy
    p.num_instances = instances
    p.num_prefill_instances = num_prefill
    p.prefill_token_budget = prefill_budget
    if isinstance(workload, str):
        p.prompt_min, p.prompt_max, p.decode_min, p.decode_max = WORKLOADS[workload]
    else:
        p.prompt_min, p.prompt_max, p.decode_min, p.decode_max = workload
    if prompt is not None:
        p.prompt_min = p.prompt_max = prompt
    if decode is not None:
        p.decode_min = p.decode_max = decode
    p.arrival_process = ARRIVAL[arrival]
    p.trace_index = trace_index
    p.rate = rate
    p.duration_s = duration_s
    p.warmup_s = warmup_s
    p.seed = seed
    p.num_requests = num_requests
    p.user_tag = user_tag
    # AcceLLM timer-driven extensions (docs/SEMANTICS.md §6b); 0 = default
    p.accellm_flags = (1 if degraded else 0) | (2 if leveling else 0)
    p.degraded_trigger_ticks = trigger_ticks
    p.policy_timer_s = timer_s
    p.leveling_link_fraction = leveling_fraction
    p.degraded_redundancy = degraded_redundancy
    p.degraded_exit_fill = degraded_exit_fill
    p.dual_copy_fraction = dual_copy_fraction
    p.splitwise_cobatch = 1 if cobatch else 0
    p.first_token_decode = 1 if first_token_decode else 0
    return p


def points_array(points):
    arr = (PointDesc * len(points))()
    for i, p in enumerate(points):
        arr[i] = p
    return arr


def summary_dict(s: PointSummary) -> dict:
    return {n: getattr(s, n) for n, _ in PointSummary._fields_ if n != "reserved"}
