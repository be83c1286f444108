// kvsim_emu.cpp — TEST HARNESS: runs the sm_100a simulation core
// (paper_2411_05555_b200/csrc/kvsim_sim.cuh) on the host under a 32-thread
// SIMT emulator so the CPU test-suite can diff the kernel logic against the
// oracle without a GPU. Never loaded by the product package or bench.py.
#define KVSIM_EMU 1
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../../paper_2411_05555_b200/csrc/kvsim_arena.hpp"
#include "../../paper_2411_05555_b200/csrc/kvsim_sim.cuh"

extern "C" int kvemu_run(const kvsim_point_desc* pts, int64_t n, const kvsim_trace_view* traces, int64_t n_traces,
                         kvsim_point_summary* out, kvsim_request_record* recs, kvsim_event_record* ev,
                         int64_t ev_cap, int64_t* ev_count, int n_warps, kvsim_instance_record* inst, int detail) {
  using namespace kvsim_dev;
  for (int64_t i = 0; i < n; ++i) {
    if (kvsim_host::validate_point(pts[i], nullptr, 0) == KVSIM_E_INVALID) {
      // still simulated (kernel reports status); nothing to do here
    }
  }
  std::vector<int64_t> tn, toff;
  std::vector<int32_t> tmin, tdmax;
  std::vector<double> tarr;
  std::vector<int32_t> tpl, tdl;
  for (int64_t k = 0; k < n_traces; ++k) {
    toff.push_back((int64_t)tarr.size());
    tn.push_back(traces[k].n);
    int32_t mn = 1 << 30, dm = 1;
    for (int64_t i = 0; i < traces[k].n; ++i) {
      tarr.push_back(traces[k].arrival_s[i]);
      tpl.push_back(traces[k].prompt_len[i]);
      tdl.push_back(traces[k].decode_len[i]);
      mn = std::min(mn, traces[k].prompt_len[i]);
      dm = std::max(dm, traces[k].decode_len[i]);
    }
    tmin.push_back(traces[k].n ? mn : 1);
    tdmax.push_back(dm);
  }
  kvsim_host::ArenaGeom g = kvsim_host::size_arena(pts, (size_t)n, tn, tmin, detail != 0, tdmax);
  SweepArgs a;
  std::memset(&a, 0, sizeof(a));
  const int32_t slots = n_warps;
  size_t bytes = kvsim_host::carve(a, nullptr, g, slots);
  char* base = (char*)std::calloc(1, bytes);
  if (!base) return KVSIM_E_OOM;
  kvsim_host::carve(a, base, g, slots);
  std::vector<int64_t> rec_off((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) rec_off[i + 1] = rec_off[i] + std::max<int64_t>(pts[i].num_requests, 0);
  std::vector<int64_t> order = kvsim_host::lpt_order(pts, (size_t)n);
  // the same split as the GPU host: plain points through sweep_warp<false>
  // (the lean kernel), the rest through sweep_warp<true>
  int64_t n_fast = 0;
  if (!(ev && ev_cap) && !detail) {
    std::stable_partition(order.begin(), order.end(), [&](int64_t i) { return !kvsim_dev::needs_full(pts[i]); });
    for (int64_t i : order) n_fast += kvsim_dev::needs_full(pts[i]) ? 0 : 1;
  }
  unsigned long long counter = 0;
  a.pts = pts;
  a.order = order.data();
  a.n_pts = n;
  a.out = out;
  a.tr_arr = tarr.data();
  a.tr_pl = tpl.data();
  a.tr_dl = tdl.data();
  a.tr_off = toff.data();
  a.tr_n = tn.data();
  a.tr_dmax = tdmax.data();
  a.recs = recs;
  a.rec_off = rec_off.data();
  a.ev = ev;
  a.ev_cap = ev_cap;
  a.ev_count = ev_count;
  a.next_point = &counter;
  a.inst = inst;
  a.detail = detail;
  std::vector<WarpScratch> scratch((size_t)slots);
  struct Job { SweepArgs* a; WarpScratch* s; int64_t slot; };
  for (int part = 0; part < 2; ++part) {
    SweepArgs b = a;
    b.order = order.data() + (part ? n_fast : 0);
    b.n_pts = part ? n - n_fast : n_fast;
    if (b.n_pts <= 0) continue;
    counter = 0;
    std::vector<Job> jobs;
    for (int w = 0; w < slots; ++w) jobs.push_back(Job{&b, &scratch[w], w});
    std::vector<std::thread> th;
    for (int w = 0; w < slots; ++w)
      th.emplace_back([&, w]() {
        simt::run_warp(part ? +[](void* p, int) {
          Job* j = (Job*)p;
          sweep_warp<true>(j->a, j->s, (int32_t)j->slot);
        } : +[](void* p, int) {
          Job* j = (Job*)p;
          sweep_warp<false>(j->a, j->s, (int32_t)j->slot);
        }, &jobs[w]);
      });
    for (auto& t : th) t.join();
  }
  std::free(base);
  return KVSIM_OK;
}

#if defined(KVSIM_EMU_PROFILE)
// call counts of the kernel's handlers (EMU_COUNT sites), for event-mix studies
extern "C" void kvemu_prof(long long* out) {
  for (int i = 0; i < 32; ++i) out[i] = kvsim_dev::emu_prof[i];
}
#endif

// The multi-device sharder (kvsim_shard.hpp, used by kvsim_gpu_run_multi and
// the CLI) with emulated devices: `workers` host threads each run their
// chunks through the emulated kernel. Results must not depend on `workers`.
#include "../../paper_2411_05555_b200/csrc/kvsim_shard.hpp"
extern "C" int kvemu_run_multi(const kvsim_point_desc* pts, int64_t n, int workers, int64_t min_chunk,
                               kvsim_point_summary* out, int64_t* points_per_worker) {
  kvsim_host::ShardPlan plan = kvsim_host::make_plan(pts, (size_t)n, workers, (size_t)(min_chunk ? min_chunk : 1));
  if (min_chunk == 0) kvsim_host::make_static(plan, pts);
  auto chunk = [&](int, const std::vector<int64_t>& idx, std::vector<kvsim_point_summary>& res, std::string&) {
    std::vector<kvsim_point_desc> sub(idx.size());
    for (size_t k = 0; k < idx.size(); ++k) sub[k] = pts[idx[k]];
    return kvemu_run(sub.data(), (int64_t)sub.size(), nullptr, 0, res.data(), nullptr, nullptr, 0, nullptr, 1, nullptr,
                     0);
  };
  std::string e;
  std::vector<int64_t> per;
  const int rc = kvsim_host::run_plan(plan, out, chunk, e, &per);
  for (int w = 0; w < workers && points_per_worker; ++w) points_per_worker[w] = per[(size_t)w];
  return rc;
}
