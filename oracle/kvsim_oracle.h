/* kvsim_oracle.h — CPU ORACLE (test infrastructure, NOT the product).
 *
 * A plain sequential C++20 restatement of the kvsim simulator specified by
 * the reference (reference SPEC.md:24-455, perfmodel.hpp:23-125), following
 * the pinned semantics in docs/SEMANTICS.md. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity status: perfmodel, RNG and the single-request engine closed form are
 * pinned against the SPEC worked examples (tests/golden/);
 * multi-request scheduling has no reference implementation to pin against
 * ("parity unpinned by the reference") and is defined by
 * docs/SEMANTICS.md + the SPEC invariant suite.
 */
#ifndef KVSIM_ORACLE_H_
#define KVSIM_ORACLE_H_
#include <stddef.h>
#include <stdint.h>
#include "kvsim_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t kvo_rng_draw(uint64_t seed, int64_t i, int stream);
/* enable per-event invariant checking; violations
 * return KVSIM_E_INTERNAL */
void kvo_set_invariant_checks(int on);
double kvo_klog(double x);
/* perfmodel (perfmodel.hpp:76-106) in sum form */
double kvo_kv_bytes_per_token(const kvsim_point_desc* p);
double kvo_weight_bytes(const kvsim_point_desc* p);
double kvo_prefill_latency(const kvsim_point_desc* p, int64_t sum_len, int64_t sum_len_sq);
double kvo_decode_step_latency(const kvsim_point_desc* p, int64_t batch, int64_t sum_kv);
double kvo_transfer_latency(const kvsim_point_desc* p, double bytes);
int kvo_kv_capacity_tokens(const kvsim_point_desc* p, int64_t* out);

/* generate_trace; returns n generated (<= cap) */
int64_t kvo_gen_trace(const kvsim_point_desc* p, double* arrival, int32_t* prompt,
                      int32_t* decode, int64_t cap);

/* run() for one point. recs: n_requests entries or NULL.
 * ev: ev_cap entries or NULL; returns status. *ev_count = events emitted. */
int kvo_run_point(const kvsim_point_desc* p, const kvsim_trace_view* trace,
                  kvsim_point_summary* out, kvsim_request_record* recs,
                  kvsim_event_record* ev, int64_t ev_cap, int64_t* ev_count);

/* v2: also per-instance records (n_instances entries, nullable) and detail
 * metrics (pooled TBT percentiles) when detail != 0. */
int kvo_run_point_ex(const kvsim_point_desc* p, const kvsim_trace_view* trace,
                     kvsim_point_summary* out, kvsim_request_record* recs,
                     kvsim_event_record* ev, int64_t ev_cap, int64_t* ev_count,
                     kvsim_instance_record* inst, int detail);

/* Sweep over n points on `threads` host threads (one point per thread at a
 * time). Generated traces only. */
int kvo_run_sweep(const kvsim_point_desc* pts, int64_t n, int threads,
                  kvsim_point_summary* out);

/* v2: sweep with per-instance records (point i at i * KVSIM_MAX_INSTANCES,
 * nullable) and detail metrics */
int kvo_run_sweep_ex(const kvsim_point_desc* pts, int64_t n, int threads,
                     kvsim_point_summary* out, kvsim_instance_record* inst, int detail);

#ifdef __cplusplus
}
#endif
#endif
