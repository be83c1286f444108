// kvsim_arena.hpp — sizing and carving of the per-warp HBM arena (host side).
//
// Every resident warp owns one arena slot, reused across the points it pulls.
// A slot holds the point's per-request "cold" arrays (indexed by request id),
// one FIFO ring per queue, and per-instance SoA batch / incoming / prefill-job
// arrays. Capacities are the maxima over the points of one launch:
//   Ncap = requests per point
//   Bcap = min(N, kv_capacity_tokens / min_prompt + 2)   (a request holds
//          >= min_prompt KV tokens on its primary, SEMANTICS §3)
//   Jcap = min(N, budget / min_prompt + 1)               (prefill admission)
#pragma once
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "kvsim_gpu.h"
#include "kvsim_math.cuh"

namespace kvsim_host {

struct ArenaGeom {
  int64_t Ncap = 1, Bcap = 1, Jcap = 1;
  int32_t Imax = 1;
  int64_t Tcap = 0;  // detail runs: TBT (gap, count) entries per slot
  // bytes per slot
  size_t per_slot() const {
    const size_t cold = (size_t)Ncap * (7 * sizeof(double) + 7 * sizeof(int32_t)) +
                        (size_t)Tcap * (sizeof(double) + sizeof(int32_t));
    const size_t ring = (size_t)Imax * Ncap * sizeof(int32_t);
    const size_t batch = (size_t)Imax * Bcap * (3 * sizeof(int32_t) + sizeof(double));
    const size_t inc = (size_t)Imax * Bcap * (sizeof(int32_t) + sizeof(double));
    const size_t job = (size_t)Imax * Jcap * 2 * sizeof(int32_t);
    const size_t link = (size_t)Imax * Imax * sizeof(double);
    return cold + ring + batch + inc + job + link + 64 * 16;
  }
};

// trace_min_prompt: per trace index, the minimum prompt (or empty);
// trace_max_decode likewise (detail runs size the TBT entries from it)
inline ArenaGeom size_arena(const kvsim_point_desc* pts, size_t n, const std::vector<int64_t>& trace_n,
                            const std::vector<int32_t>& trace_min_prompt, bool detail = false,
                            const std::vector<int32_t>& trace_max_decode = {}) {
  ArenaGeom g;
  for (size_t i = 0; i < n; ++i) {
    const kvsim_point_desc& p = pts[i];
    int64_t N = p.num_requests > 0 ? p.num_requests : 0;
    int32_t pmin = p.prompt_min;
    int64_t dmax = p.decode_max;
    if (p.trace_index >= 0 && (size_t)p.trace_index < trace_n.size()) {
      N = std::min<int64_t>(N, trace_n[p.trace_index]);
      pmin = trace_min_prompt[p.trace_index];
      dmax = (size_t)p.trace_index < trace_max_decode.size() ? trace_max_decode[p.trace_index] : 1;
    }
    if (pmin < 1) pmin = 1;
    const kvsim_math::Perf f = kvsim_math::make_perf(p);
    const int64_t cap = f.fits ? f.cap : 0;
    const int64_t budget = p.prefill_token_budget > 0 ? p.prefill_token_budget : 8192;
    g.Ncap = std::max<int64_t>(g.Ncap, N);
    g.Bcap = std::max<int64_t>(g.Bcap, std::min<int64_t>(N, cap / pmin + 2));
    g.Jcap = std::max<int64_t>(g.Jcap, std::min<int64_t>(N, budget / pmin + 1));
    g.Imax = std::max<int32_t>(g.Imax, std::min<int32_t>(std::max(p.num_instances, 1), KVSIM_MAX_INSTANCES));
    // entries <= decode steps + individual gaps, each <= the TBT samples N (dmax - 1)
    if (detail) g.Tcap = std::max<int64_t>(g.Tcap, 2 * N * std::max<int64_t>(dmax - 1, 0) + 64);
  }
  g.Bcap = (g.Bcap + 3) & ~(int64_t)3;  // 16-byte vector access of the batch SoA (flush_slow)
  return g;
}

// Carve `slots` slots out of one base allocation into the pointer fields of
// an args struct (kvsim_dev::SweepArgs or an emulator twin with the same
// field names).
template <class Args>
inline size_t carve(Args& a, char* base, const ArenaGeom& g, int32_t slots) {
  size_t off = 0;
  auto take = [&](auto*& ptr, size_t count) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    off = (off + 255) & ~(size_t)255;
    ptr = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
  };
  const size_t S = (size_t)slots;
  const size_t cold = S * (size_t)g.Ncap;
  take(a.c_arr, cold); take(a.c_last, cold); take(a.c_tbt, cold); take(a.c_fresh, cold);
  take(a.c_first, cold); take(a.c_done, cold); take(a.c_qs, cold);
  take(a.c_pl, cold); take(a.c_dl, cold); take(a.c_qlen, cold); take(a.c_em, cold);
  take(a.c_cpy, cold); take(a.c_nmv, cold); take(a.c_npre, cold);
  take(a.q_rid, S * g.Imax * (size_t)g.Ncap);
  const size_t bb = S * g.Imax * (size_t)g.Bcap;
  take(a.b_rid, bb); take(a.b_rem, bb); take(a.b_kvb, bb); take(a.b_tbt, bb);
  take(a.i_rid, bb); take(a.i_ready, bb);
  const size_t jj = S * g.Imax * (size_t)g.Jcap;
  take(a.j_rid, jj); take(a.j_dst, jj);
  take(a.link, S * g.Imax * (size_t)g.Imax);
  take(a.t_val, S * (size_t)g.Tcap);
  take(a.t_cnt, S * (size_t)g.Tcap);
  a.Tcap = g.Tcap;
  a.Ncap = g.Ncap;
  a.Bcap = g.Bcap;
  a.Jcap = g.Jcap;
  a.Imax = g.Imax;
  a.slots = slots;
  return off + 256;
}

// Longest-processing-time-first order: the event count of a point grows with
// requests x mean decode length and with lower rates (smaller batches).
inline std::vector<int64_t> lpt_order(const kvsim_point_desc* pts, size_t n) {
  std::vector<int64_t> ord(n);
  std::vector<double> cost(n);
  // Points are grouped by policy (co-resident warps then execute the same
  // policy-specialised code: the kernel is instruction-fetch bound otherwise),
  // longest first within a policy. KVSIM_ORDER=lpt disables the grouping.
  const char* mode = std::getenv("KVSIM_ORDER");
  const bool by_policy = !(mode && mode[0] == 'l');
  for (size_t i = 0; i < n; ++i) {
    const kvsim_point_desc& p = pts[i];
    const double dbar = 0.5 * ((double)p.decode_min + (double)p.decode_max);
    cost[i] = (double)p.num_requests * dbar * (1.0 + 1.0 / (0.25 + (p.rate > 0 ? p.rate : 0)));
    ord[i] = (int64_t)i;
  }
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    if (by_policy && pts[a].policy != pts[b].policy) return pts[a].policy < pts[b].policy;
    return cost[a] > cost[b];
  });
  return ord;
}

inline int validate_point(const kvsim_point_desc& p, char* err, size_t len) {
  auto fail = [&](int code, const char* msg) {
    if (err && len) {
      size_t i = 0;
      for (; msg[i] && i + 1 < len; ++i) err[i] = msg[i];
      err[i] = 0;
    }
    return code;
  };
  if (p.num_instances < 1 || p.num_instances > KVSIM_MAX_INSTANCES) return fail(KVSIM_E_INVALID, "num_instances out of range [1,32]");
  if (p.policy < 0 || p.policy > 2) return fail(KVSIM_E_INVALID, "unknown policy");
  if (p.policy == KVSIM_POLICY_ACCELLM && (p.num_instances % 2)) return fail(KVSIM_E_ODD_INSTANCES, "even instance count required");
  if (p.policy == KVSIM_POLICY_SPLITWISE) {
    const int np = p.num_prefill_instances > 0 ? p.num_prefill_instances : (p.num_instances + 2) / 4;
    if (p.num_instances < 2 || np >= p.num_instances) return fail(KVSIM_E_INVALID, "splitwise needs >=1 prefill and >=1 decode instance");
  }
  if (!(p.peak_flops > 0 && p.hbm_capacity > 0 && p.hbm_bandwidth > 0 && p.link_bandwidth > 0))
    return fail(KVSIM_E_INVALID, "device fields must be > 0");
  if (!(p.param_count > 0) || p.num_layers <= 0 || p.hidden_dim <= 0 || p.num_kv_heads <= 0 || p.head_dim <= 0 ||
      p.bytes_per_value <= 0)
    return fail(KVSIM_E_INVALID, "model fields must be > 0");
  if (p.num_devices < 1) return fail(KVSIM_E_INVALID, "num_devices must be >= 1");
  if (!(p.memory_reserve_fraction >= 0 && p.memory_reserve_fraction < 1)) return fail(KVSIM_E_INVALID, "memory_reserve_fraction must be in [0,1)");
  if (!(p.compute_eff > 0 && p.compute_eff <= 1 && p.mem_bw_eff > 0 && p.mem_bw_eff <= 1 && p.link_eff > 0 && p.link_eff <= 1))
    return fail(KVSIM_E_INVALID, "efficiency factors must be in (0,1]");
  if (p.trace_index < 0) {
    if (p.prompt_min < 1 || p.prompt_max < p.prompt_min || p.decode_min < 1 || p.decode_max < p.decode_min)
      return fail(KVSIM_E_INVALID, "workload ranges must satisfy 1 <= min <= max");
    if (p.decode_max > 0x07ffffff || p.prompt_max > 0x07ffffff)
      return fail(KVSIM_E_INVALID, "prompt/decode lengths must be < 2^27");
    if (!(p.rate >= 0)) return fail(KVSIM_E_INVALID, "rate must be >= 0");
  }
  if (p.num_requests < 0 || p.num_requests > 0x7ffffff0ll) return fail(KVSIM_E_INVALID, "num_requests out of range");
  if (!kvsim_math::make_perf(p).fits) return fail(KVSIM_E_MODEL_FIT, "model does not fit in instance memory");
  return KVSIM_OK;
}

}  // namespace kvsim_host
