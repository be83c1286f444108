// kvsim_shard.hpp — multi-GPU point sharding (host side).
//
// Sweep points are independent (reference SPEC.md:267,446-448), so a sweep is
// sharded over G devices with no data-path collective: one host thread per
// device pulls chunks of points from a shared atomic cursor over the points
// sorted by estimated cost (longest first), runs each chunk through the
// single-device C-ABI and writes the summaries at their point index. The
// merge is therefore deterministic and byte-identical for any G.
//
// Chunks follow guided self-scheduling: a claim takes max(min_chunk,
// remaining / (2 G)) points, so the expensive points go out first in large
// chunks and the tail of the sweep is cut into small ones. Every chunk is
// one kernel launch whose own tail leaves warps idle, so min_chunk should
// cover a few waves of resident warps (kvsim_gpu_run_multi: 2 x slots);
// up to 16 waves per device the points are dealt once instead (make_static).
#pragma once
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kvsim_gpu.h"

namespace kvsim_host {

// Estimated cost of a point (simulated request-iterations, larger at low
// rates where batches are small): the same estimate as lpt_order.
inline double point_cost(const kvsim_point_desc& p) {
  const double dbar = 0.5 * ((double)p.decode_min + (double)p.decode_max);
  return (double)p.num_requests * dbar * (1.0 + 1.0 / (0.25 + (p.rate > 0 ? p.rate : 0)));
}

struct ShardPlan {
  std::vector<int64_t> order;  // point indices, most expensive first
  size_t min_chunk = 1;
  int workers = 1;
  // static mode (few points per device): worker w runs fixed[w] as one chunk
  std::vector<std::vector<int64_t>> fixed;
};

// Few points per device (up to 16 waves of resident warps): one launch
// per device, points dealt by greedy LPT on the cost estimate (most
// expensive first, each to the least-loaded device), so launches end
// together instead of stacking per-launch tails.
inline void make_static(ShardPlan& s, const kvsim_point_desc* pts) {
  s.fixed.assign((size_t)s.workers, {});
  std::vector<double> load((size_t)s.workers, 0.0);
  for (int64_t i : s.order) {
    size_t w = 0;
    for (size_t k = 1; k < load.size(); ++k)
      if (load[k] < load[w]) w = k;
    s.fixed[w].push_back(i);
    load[w] += point_cost(pts[i]);
  }
}

inline ShardPlan make_plan(const kvsim_point_desc* pts, size_t n, int workers, size_t min_chunk) {
  ShardPlan s;
  s.workers = workers < 1 ? 1 : workers;
  s.min_chunk = min_chunk < 1 ? 1 : min_chunk;
  s.order.resize(n);
  std::vector<double> cost(n);
  for (size_t i = 0; i < n; ++i) {
    s.order[i] = (int64_t)i;
    cost[i] = point_cost(pts[i]);
  }
  std::stable_sort(s.order.begin(), s.order.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  return s;
}

// Run the plan: `run_chunk(worker, indices, out_summaries)` simulates the
// points pts[indices[k]] into out[k] and returns 0 or an error code with a
// message. Results are scattered to out[index]. Returns the first error.
using ChunkFn = std::function<int(int worker, const std::vector<int64_t>& idx, std::vector<kvsim_point_summary>& out,
                                  std::string& err)>;

inline int run_plan(const ShardPlan& plan, kvsim_point_summary* out, const ChunkFn& run_chunk, std::string& err,
                    std::vector<int64_t>* points_per_worker = nullptr) {
  const size_t n = plan.order.size();
  std::atomic<size_t> cursor{0};
  std::mutex claim_mu;  // claims are tiny; a lock keeps the guided size exact
  std::vector<std::string> errs((size_t)plan.workers);
  std::vector<int64_t> done((size_t)plan.workers, 0);
  if (!plan.fixed.empty()) {  // static mode: one chunk per worker
    std::vector<std::thread> th;
    for (int w = 0; w < plan.workers; ++w)
      th.emplace_back([&, w]() {
        const std::vector<int64_t>& idx = plan.fixed[(size_t)w];
        if (idx.empty()) return;
        std::vector<kvsim_point_summary> res(idx.size());
        std::string e;
        if (run_chunk(w, idx, res, e) != 0) {
          errs[(size_t)w] = e.empty() ? "chunk failed" : e;
          return;
        }
        for (size_t k = 0; k < idx.size(); ++k) out[idx[k]] = res[k];
        done[(size_t)w] = (int64_t)idx.size();
      });
    for (auto& t : th) t.join();
    if (points_per_worker) *points_per_worker = done;
    for (auto& e : errs)
      if (!e.empty()) {
        err = e;
        return KVSIM_E_INTERNAL;
      }
    return KVSIM_OK;
  }
  auto claim = [&](size_t& a, size_t& b) {
    std::lock_guard<std::mutex> g(claim_mu);
    a = cursor.load();
    if (a >= n) return false;
    const size_t rem = n - a;
    const size_t want = std::max(plan.min_chunk, rem / (2 * (size_t)plan.workers));
    b = std::min(n, a + want);
    cursor.store(b);
    return true;
  };
  std::vector<std::thread> th;
  for (int w = 0; w < plan.workers; ++w)
    th.emplace_back([&, w]() {
      std::vector<int64_t> idx;
      std::vector<kvsim_point_summary> res;
      size_t a = 0, b = 0;
      while (claim(a, b)) {
        idx.assign(plan.order.begin() + (int64_t)a, plan.order.begin() + (int64_t)b);
        res.assign(idx.size(), kvsim_point_summary{});
        std::string e;
        if (run_chunk(w, idx, res, e) != 0) {
          errs[(size_t)w] = e.empty() ? "chunk failed" : e;
          return;
        }
        for (size_t k = 0; k < idx.size(); ++k) out[idx[k]] = res[k];
        done[(size_t)w] += (int64_t)idx.size();
      }
    });
  for (auto& t : th) t.join();
  if (points_per_worker) *points_per_worker = done;
  for (auto& e : errs)
    if (!e.empty()) {
      err = e;
      return KVSIM_E_INTERNAL;
    }
  return KVSIM_OK;
}

}  // namespace kvsim_host
