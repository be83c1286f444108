/* kvsim_gpu.h — C-ABI of the B200 sweep engine (drop-in boundary).
 *
 * The reference declares the simulator's host API as C++ free functions in
 * namespace kvsim (reference proj/include/kvsim/perfmodel.hpp:23-125) and
 * specifies the engine entry point `run(trace, cluster, policy, model, eff,
 * seed) -> RawResults` (reference SPEC.md:219) and the sweep orchestrator
 * `cmd_sweep`. None of these have bodies in the reference
 * (SURVEY.md §0). This header is the C boundary that the C++ host entry point
 * (`kvsim run|sweep`, tools/kvsim_cli.cpp) calls instead of an in-process
 * engine: plain structs, pointers and sizes; no exceptions, no torch types.
 *
 * Mapping to the reference interface:
 *   kvsim_point_desc      <- (WorkloadSpec, ArrivalSpec, list<InstanceSpec>,
 *                             policy, ModelSpec, EfficiencyFactors, seed)
 *                             = arguments of run() (
 *                               perfmodel.hpp:30-65)
 *   kvsim_point_summary   <- MetricsReport aggregates + summary.csv columns
 *
 *   kvsim_request_record  <- per-request TTFT/TBT/JCT records
 *   kvsim_event_record    <- --emit-events JSONL event log
 *   kvsim_gpu_run         <- run() for many points at once (cmd_sweep's
 *                             concurrent point loop)
 *   kvsim_gpu_perf_batch  <- prefill_latency / decode_step_latency /
 *                             transfer_latency / kv_capacity_tokens
 *                             (perfmodel.hpp:84-106) evaluated in bulk
 *   kvsim_gpu_gen_trace   <- generate_trace
 *   kvsim_gpu_host_alloc  <- load_trace's buffers, pinned
 *
 * Errors: every entry point returns 0 on success or a negative KVSIM_E_* code
 * with a message in `err` (SPEC.md:69,78,96,416 messages are preserved).
 * Per-point failures are reported in kvsim_point_summary.status and do not
 * abort the sweep.
 *
 * Threading: calls on different devices may run concurrently; calls sharing a
 * handle are serialised by the caller.
 */
#ifndef KVSIM_GPU_H_
#define KVSIM_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVSIM_ABI_VERSION 2
#define KVSIM_MAX_INSTANCES 32

enum kvsim_policy { KVSIM_POLICY_UNIFIED = 0, KVSIM_POLICY_SPLITWISE = 1, KVSIM_POLICY_ACCELLM = 2 };
enum kvsim_arrival { KVSIM_ARRIVAL_POISSON = 0, KVSIM_ARRIVAL_FIXED = 1 };
enum kvsim_link_mode { KVSIM_LINK_STRIPED = 0, KVSIM_LINK_SINGLE = 1 };

enum kvsim_status {
  KVSIM_OK = 0,
  KVSIM_E_INVALID = -1,        /* invalid argument / config */
  KVSIM_E_MODEL_FIT = -2,      /* "model does not fit in instance memory" */
  KVSIM_E_ODD_INSTANCES = -3,  /* "even instance count required" */
  KVSIM_E_CUDA = -4,           /* CUDA runtime error */
  KVSIM_E_NO_DEVICE = -5,      /* no CUDA device / extension unusable */
  KVSIM_E_EVENT_BUDGET = -6,   /* per-point event budget exceeded */
  KVSIM_E_OOM = -7,            /* device arena allocation failed */
  KVSIM_E_EMPTY_BATCH = -8,    /* "empty prefill batch" / "empty decode batch" */
  KVSIM_E_INTERNAL = -9        /* invariant violated (bug guard) */
};

/* One simulation point = one independent run() of the reference. 256 bytes. */
typedef struct kvsim_point_desc {
  /* ModelSpec (perfmodel.hpp:38-46) */
  double param_count;
  int32_t num_layers, hidden_dim, num_kv_heads, head_dim, bytes_per_value;
  int32_t policy;               /* enum kvsim_policy */
  /* DeviceSpec (perfmodel.hpp:30-36) */
  double peak_flops, hbm_capacity, hbm_bandwidth, link_bandwidth;
  /* InstanceSpec (perfmodel.hpp:48-53) */
  int32_t num_devices, tensor_parallel;
  double memory_reserve_fraction;
  /* EfficiencyFactors (perfmodel.hpp:56-60) */
  double compute_eff, mem_bw_eff, link_eff;
  /* cluster / policy */
  int32_t link_mode;            /* enum kvsim_link_mode (perfmodel.hpp:65) */
  int32_t num_instances;        /* <= KVSIM_MAX_INSTANCES */
  int32_t num_prefill_instances;/* splitwise; 0 => (n+2)/4 */
  int32_t prefill_token_budget; /* 0 => 8192 */
  /* WorkloadSpec + ArrivalSpec */
  int32_t prompt_min, prompt_max, decode_min, decode_max;
  int32_t arrival_process;      /* enum kvsim_arrival */
  int32_t trace_index;          /* -1 => device RNG; else index into traces[] */
  double rate;                  /* requests / s */
  double duration_s;            /* arrivals with t < duration_s (INFINITY ok) */
  double warmup_s;              /* requests arriving before are excluded */
  uint64_t seed;
  int64_t num_requests;         /* max requests generated (P10) */
  uint64_t user_tag;            /* opaque, echoed */
  /* AcceLLM extensions driven by the policy timer (
   * PAPER.md:309,457; docs/SEMANTICS.md §6b). Zero = off / default. */
  int32_t accellm_flags;        /* bit 0 degraded mode, bit 1 inter-pair leveling */
  int32_t degraded_trigger_ticks;   /* 0 => 3 consecutive timer ticks */
  /* v2: Splitwise high-load co-batching (off by default):
   * while a prompt waits and every prefill instance is busy, a decode
   * instance co-batches queued prompts into its next iteration
   * (docs/SEMANTICS.md §6 splitwise) */
  int32_t splitwise_cobatch;
  /* v2: the first token comes from the first decode step after the prefill
   * instead of the prefill itself (SPEC.md:273 alternative; off = SPEC's
   * default): decode_len tokens take decode_len decode steps */
  int32_t first_token_decode;
  int32_t reserved_i[4];
  double policy_timer_s;        /* 0 => 1.0 s timer period */
  double leveling_link_fraction;/* 0 => 0.10 of link capacity per timer period */
  double degraded_redundancy;   /* 0 => 0.5: enter when copies < this x live */
  double degraded_exit_fill;    /* 0 => 0.5: leave when group KV <= this x capacity */
  double dual_copy_fraction;    /* 0 => 1/3: dual instance's copy budget per decoder */
  double reserved_d[2];
} kvsim_point_desc;

#define KVSIM_ACCELLM_DEGRADED 1
#define KVSIM_ACCELLM_LEVELING 2

/* Caller-supplied trace (load_trace). */
typedef struct kvsim_trace_view {
  const double* arrival_s;
  const int32_t* prompt_len;
  const int32_t* decode_len;
  int64_t n;
} kvsim_trace_view;

/* Per-point result: the 13 summary.csv columns + counters. */
typedef struct kvsim_point_summary {
  int32_t status;               /* enum kvsim_status */
  int32_t num_instances;
  int64_t n_requests, n_completed, n_measured;
  int64_t tokens_total, tokens_window;
  int64_t n_events, n_steps, n_prefills, n_moves, n_preemptions, n_evictions;
  int64_t peak_kv_tokens, link_prefill_tokens, link_mirror_tokens;
  double makespan_s;
  double ttft_mean, ttft_p50, ttft_p95, ttft_max;
  double tbt_mean, tbt_max;
  double jct_mean, jct_p50, jct_p95, jct_max;
  double cost_eff, idle_frac, peak_kv_gb, link_prefill_gb, link_mirror_gb;
  double busy_s_total;
  uint64_t user_tag;
  int64_t link_leveling_tokens; /* KV moved by inter-pair leveling */
  int64_t n_timer_ticks;        /* policy timer events */
  int64_t n_mode_switches;      /* degraded-mode entries + exits */
  /* v2: the rest of the MetricsReport */
  double ttft_queue_mean;       /* mean (first prefill start - arrival): the queue-wait part of TTFT */
  double tbt_p50, tbt_p95;      /* nearest rank over the pooled TBT samples of measured requests;
                                   detail runs only (kvsim_run_opts.detail), NaN otherwise */
  double idle_runnable_s;       /* sum over instances of time in the window with no job in
                                   flight while >= 1 request waits in a prefill queue, i.e.
                                   runnable work exists that nobody runs */
  double queue_depth_avg;       /* time average over [0, makespan] of the requests waiting in
                                   prefill queues (SPEC.md:358 queue-depth series) */
  int64_t queue_depth_max;
  int64_t n_tbt_samples;        /* sum over measured requests of (decode_len - 1) */
  int64_t reserved[1];
} kvsim_point_summary;

/* Per-request record (parity configs). ttft = first_token_s - arrival_s,
 * jct = completion_s - arrival_s, tbt samples sum = completion_s - first_token_s. */
typedef struct kvsim_request_record {
  double arrival_s, first_token_s, completion_s, tbt_max_s;
  int32_t prompt_len, decode_len;
  int32_t n_moves, n_preemptions;
  double prefill_start_s;       /* v2: start of the job that produced the first token (queue wait
                                   = prefill_start_s - arrival_s) */
} kvsim_request_record;

/* v2: per-instance record ("idle_fraction per instance;
 * peak_kv_bytes per instance"). idle fraction = 1 - busy_s / window. */
typedef struct kvsim_instance_record {
  double busy_s;                /* job time of jobs starting in the window */
  double idle_runnable_s;       /* see kvsim_point_summary.idle_runnable_s */
  int64_t peak_kv_tokens;       /* peak ledger (primaries + copies + reservations) */
  int32_t initial_role;         /* 0 decode, 1 prefill (splitwise prefill instances) */
  int32_t reserved;
} kvsim_instance_record;

/* Decision / event log entry (--emit-events). */
enum kvsim_event_kind {
  KVSIM_EV_ARRIVE = 1,        /* inst=target instance|pair, a=rid, b=len */
  KVSIM_EV_PREFILL_START = 2, /* inst, a=n admitted, b=first rid, c=sum len */
  KVSIM_EV_PREFILL_DONE = 3,  /* inst, a=n, b=n completed at prefill */
  KVSIM_EV_STEP_START = 4,    /* inst, a=batch, b=n prefill co-batched, c=sum kv */
  KVSIM_EV_STEP_END = 5,      /* inst, a=batch, b=n completed */
  KVSIM_EV_MOVE = 6,          /* inst=from, a=rid, b=to */
  KVSIM_EV_EVICT = 7,         /* inst=holder, a=rid */
  KVSIM_EV_PREEMPT = 8,       /* inst, a=rid, b=recompute len */
  KVSIM_EV_ROLE = 9,          /* inst, a=new role (0 decode, 1 prefill) */
  KVSIM_EV_TRANSFER = 10,     /* inst=src, a=dst, b=kind (0 prefill,1 mirror), c=tokens */
  KVSIM_EV_WAKE = 11,         /* inst */
  KVSIM_EV_JOIN = 12,         /* inst, a=n joined */
  KVSIM_EV_COPY = 13,         /* inst=holder, a=n copies created */
  KVSIM_EV_TIMER = 14,        /* inst=-1, a=tick index */
  KVSIM_EV_LEVEL = 15,        /* inst=from, a=rid, b=to, c=kv tokens moved */
  KVSIM_EV_MODE = 16          /* inst=group, a=1 enter degraded / 0 leave */
};
typedef struct kvsim_event_record {
  double t;
  int32_t kind, inst, a, b;
  int64_t c;
} kvsim_event_record;

/* ---------------------------------------------------------------- handles */
typedef struct kvsim_gpu_ctx kvsim_gpu_ctx;

int kvsim_gpu_abi_version(void);
int kvsim_gpu_device_count(void);
/* Open a context on a device (allocates nothing until the first run). */
int kvsim_gpu_open(int device, kvsim_gpu_ctx** out, char* err, size_t err_len);
void kvsim_gpu_close(kvsim_gpu_ctx* ctx);

/* Fill defaults (Llama-2-70B / H100 / eff 0.5,0.8,0.8 / mixed / accellm). */
void kvsim_point_defaults(kvsim_point_desc* p);
/* Host-side validation of one point (perfmodel validate()). */
int kvsim_point_validate(const kvsim_point_desc* p, char* err, size_t err_len);

/* Run n points with host buffers (the reference-facing call).
 *   traces      nullable; used by points with trace_index >= 0
 *   out         n summaries (required)
 *   recs        nullable; if set, point i's records start at sum_{j<i} num_requests_j
 *   ev/ev_cap   nullable; per-point event log of ev_cap entries, point i at i*ev_cap;
 *               ev_count[i] receives the number of events (may exceed ev_cap).  */
int kvsim_gpu_run(kvsim_gpu_ctx* ctx, const kvsim_point_desc* pts, size_t n,
                  const kvsim_trace_view* traces, size_t n_traces,
                  kvsim_point_summary* out, kvsim_request_record* recs,
                  kvsim_event_record* ev, size_t ev_cap, int64_t* ev_count,
                  char* err, size_t err_len);

/* v2: optional outputs and modes of a run (all fields zero = kvsim_gpu_run
 * without records / events). */
typedef struct kvsim_run_opts {
  int32_t detail;               /* 1: pooled TBT percentiles (tbt_p50/p95). Runs the plain event
                                   loop (no step chaining) and keeps one (gap, count) entry per
                                   step in HBM: for reports, not for throughput sweeps */
  int32_t reserved_i[3];
  kvsim_request_record* recs;   /* as in kvsim_gpu_run */
  kvsim_event_record* ev;       /* as in kvsim_gpu_run */
  size_t ev_cap;
  int64_t* ev_count;
  kvsim_instance_record* inst;  /* nullable; point i's records at i * KVSIM_MAX_INSTANCES */
} kvsim_run_opts;
int kvsim_gpu_run_ex(kvsim_gpu_ctx* ctx, const kvsim_point_desc* pts, size_t n,
                     const kvsim_trace_view* traces, size_t n_traces, kvsim_point_summary* out,
                     const kvsim_run_opts* opts, char* err, size_t err_len);

/* v2: one sweep sharded over several devices.
 * ctxs[k] are open contexts on distinct devices (reused across calls, so
 * arenas are allocated once). One host thread per context pulls chunks of
 * points (guided self-scheduling over the points sorted by estimated cost,
 * chunks >= min_chunk) and runs each through kvsim_gpu_run_ex; summaries
 * land at their point index, so `out` is byte-identical for any number of
 * devices. No collective: results are gathered in host memory.
 * min_chunk 0 = automatic: with at most 16 waves of resident warps per device
 * the points are dealt once (greedy LPT on the cost estimate, one launch per
 * device), else guided chunks of >= 2 waves. Generated traces only
 * (trace_index < 0). stats is nullable. */
#define KVSIM_MAX_DEVICES 16
typedef struct kvsim_multi_stats {
  double device_seconds[KVSIM_MAX_DEVICES];   /* CUDA-event time, first chunk start to last chunk end */
  int64_t device_points[KVSIM_MAX_DEVICES];
  int64_t device_launches[KVSIM_MAX_DEVICES];
  int32_t n_devices, reserved;
} kvsim_multi_stats;
int kvsim_gpu_run_multi(kvsim_gpu_ctx* const* ctxs, int n_ctx, const kvsim_point_desc* pts, size_t n,
                        kvsim_point_summary* out, size_t min_chunk, kvsim_multi_stats* stats,
                        char* err, size_t err_len);

/* Device-resident variant: d_pts / d_out are device pointers, generated traces
 * only, no records; launched on `stream` (a cudaStream_t; NULL selects the
 * context's own stream) without synchronising.
 * Used by bench.py to time the kernels with inputs already in HBM. */
int kvsim_gpu_run_device(kvsim_gpu_ctx* ctx, const kvsim_point_desc* d_pts, size_t n,
                         kvsim_point_summary* d_out, void* stream,
                         char* err, size_t err_len);
/* Prepare (size + allocate) the arena for a device-resident run of these host
 * points so kvsim_gpu_run_device does no allocation inside a timed region.
 * The reservation lasts until the next kvsim_gpu_run / _run_ex on the same
 * context (which re-sizes the arena for its own points); d_pts passed to
 * kvsim_gpu_run_device must be the reserved points. */
int kvsim_gpu_reserve(kvsim_gpu_ctx* ctx, const kvsim_point_desc* pts, size_t n,
                      char* err, size_t err_len);
/* Kernel launches issued by the last run (for the bench's gpu_launches). */
int64_t kvsim_gpu_last_launches(const kvsim_gpu_ctx* ctx);
/* Profiling hook (no reference counterpart): when the context was opened with
 * KVSIM_POINT_TIMES set, copies {start_ns, end_ns, warp slot} per point of the
 * last kvsim_gpu_run into out (up to cap values); returns values copied. */
int64_t kvsim_gpu_point_times(kvsim_gpu_ctx* ctx, uint64_t* out, int64_t cap);

/* Bulk perfmodel evaluation on the device (K1). For each i:
 *   op[i]==0 prefill_latency(s1[i]=sum L, s2[i]=sum L^2)
 *   op[i]==1 decode_step_latency(s1[i]=batch, s2[i]=sum kv)
 *   op[i]==2 transfer_latency(bytes = (double)s1[i])
 *   op[i]==3 kv_capacity_tokens (result bit-cast int64 into out[i])
 * with point parameters pts[pidx[i]]. Host buffers. */
int kvsim_gpu_perf_batch(kvsim_gpu_ctx* ctx, const kvsim_point_desc* pts, size_t n_pts,
                         const int32_t* pidx, const int32_t* op, const int64_t* s1,
                         const int64_t* s2, double* out, size_t n, char* err, size_t err_len);

/* v2: throughput_curves (reference perfmodel.hpp:108-123; SPEC.md:101-109,
 * 425-431) on the device: the (length x batch) grid of prefill (phase 0) or
 * decode (phase 1) latencies through K1, tokens/s = tokens / latency.
 * Row r = li * n_batch + bi. Host buffers of n_len * n_batch entries. */
int kvsim_gpu_curves(kvsim_gpu_ctx* ctx, const kvsim_point_desc* p, const int64_t* lengths, size_t n_len,
                     const int64_t* batch_sizes, size_t n_batch, int phase, double* latency_s,
                     double* tokens_per_s, char* err, size_t err_len);

/* Device trace generation (K2) for one point: n = min(num_requests, arrivals
 * before duration_s). Writes *n_out. Host buffers of capacity num_requests. */
int kvsim_gpu_gen_trace(kvsim_gpu_ctx* ctx, const kvsim_point_desc* p, double* arrival_s,
                        int32_t* prompt_len, int32_t* decode_len, int64_t* n_out,
                        char* err, size_t err_len);

/* Page-locked host memory for bulk trace ingestion (load_trace,
 * SPEC.md:164-172). A caller that parses a large external
 * trace straight into these buffers gets DMA-speed, asynchronous host-to-device
 * copies of traces[] inside kvsim_gpu_run instead of staged pageable copies.
 * Returns NULL when page-locked memory is unavailable (no CUDA device, or the
 * allocation failed); the caller then uses ordinary memory. Free with
 * kvsim_gpu_host_free (NULL is a no-op). */
void* kvsim_gpu_host_alloc(size_t bytes);
void kvsim_gpu_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* KVSIM_GPU_H_ */
