// kvsim_sweep.cu — sm_100a kernels and the C-ABI (include/kvsim_gpu.h).
//
//   K1 kvsim_perf_kernel   bulk perfmodel evaluation (perfmodel.hpp:76-106)
//   K2 kvsim_trace_kernel  device generate_trace, one warp/trace
//   K3 kvsim_sweep_kernel  persistent warp-per-point DES with the per-point
//                          metrics finaliser fused at the end
//
// Host side: a context owns one device, a stream and a grow-only HBM arena
// carved into one slot per resident warp. No CPU fallback exists: without a
// usable device every entry point returns KVSIM_E_NO_DEVICE.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "kvsim_arena.hpp"
#include "kvsim_gpu.h"
#include "kvsim_shard.hpp"
#include "kvsim_sim.cuh"

using kvsim_dev::SweepArgs;
using kvsim_dev::WarpScratch;

using kvsim_dev::kWarpsPerBlock;

// ------------------------------------------------------------------ kernels
// K3: kvsim_kernel.cuh; this translation unit instantiates the lean kernel
// (handlers inlined), kvsim_sweep_full.cu the full one (handlers outlined).
#include "kvsim_kernel.cuh"
template __global__ void kvsim_sweep_kernel<3, false>(const __grid_constant__ SweepArgs);
#ifdef KVSIM_MINB_ALT
template __global__ void kvsim_sweep_kernel<KVSIM_MINB_ALT, false>(const __grid_constant__ SweepArgs);
#endif
// kvsim_sweep_full.cu
using SweepFn = void (*)(SweepArgs);
SweepFn kvsim_full_kernel(int minb);

__global__ void kvsim_perf_kernel(const kvsim_point_desc* pts, const int32_t* pidx, const int32_t* op,
                                  const int64_t* s1, const int64_t* s2, double* out, int64_t n) {
  using namespace kvsim_math;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const Perf f = make_perf(pts[pidx[i]]);
    double r = 0.0;
    switch (op[i]) {
      case 0: r = prefill_latency(f, s1[i], s2[i]); break;
      case 1: r = decode_latency(f, s1[i], s2[i]); break;
      case 2: r = transfer_latency(f, (double)s1[i]); break;
      default: {
        const int64_t c = f.fits ? f.cap : -1;
        r = __longlong_as_double((long long)c);
      }
    }
    out[i] = r;
  }
}

// one warp: lanes draw 32 requests at a time; arrival times accumulate in
// request order (sequential adds, SEMANTICS §2) via shuffles.
__global__ void kvsim_trace_kernel(kvsim_point_desc p, double* arr, int32_t* pl, int32_t* dl, int64_t cap,
                                   int64_t* n_out) {
  using namespace kvsim_math;
  const int lane = threadIdx.x & 31;
  const uint64_t key = stream_key(p.seed);
  int64_t lim = p.num_requests < cap ? p.num_requests : cap;
  if (!(p.rate > 0.0)) lim = 0;
  double t = 0.0;
  int64_t n = 0;
  bool stop = false;
  for (int64_t i0 = 0; i0 < lim && !stop; i0 += 32) {
    const int64_t i = i0 + lane;
    double g = 0.0;
    if (i < lim && p.arrival_process != KVSIM_ARRIVAL_FIXED) g = poisson_gap(key, i, p.rate);
    double mine = 0.0;
    bool ok_mine = false;
    for (int l = 0; l < 32 && i0 + l < lim; ++l) {
      const double gl = __shfl_sync(0xffffffffu, g, l);
      double tl;
      if (p.arrival_process == KVSIM_ARRIVAL_FIXED) tl = kdiv((double)(i0 + l), p.rate);
      else tl = (i0 + l) == 0 ? gl : kadd(t, gl);
      if (!(tl < p.duration_s)) { stop = true; break; }
      t = tl;
      n = i0 + l + 1;
      if (lane == l) { mine = tl; ok_mine = true; }
    }
    if (ok_mine) {
      arr[i] = mine;
      pl[i] = uniform_range(draw_k(key, i, 0), p.prompt_min, p.prompt_max);
      dl[i] = uniform_range(draw_k(key, i, 1), p.decode_min, p.decode_max);
    }
  }
  if (lane == 0) *n_out = n;
}

// ------------------------------------------------------------------ host side
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t b = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) cap = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct kvsim_gpu_ctx {
  int device = 0;
  int sms = 0;
  int blocks_per_sm = 1;
  cudaStream_t stream = nullptr;
  DevBuf arena, pts, order, out, recs, rec_off, ev, ev_count, tr_arr, tr_pl, tr_dl, tr_off, tr_n, tr_dmax, counter, ptime,
      inst;
  bool point_times = false;  // KVSIM_POINT_TIMES: record per-point start/end (profiling)
  int64_t ptime_n = 0;
  kvsim_host::ArenaGeom geom;
  int32_t slots = 0;
  SweepArgs reserved_args{};
  bool reserved = false;
  int64_t last_launches = 0;
  void (*kernel)(SweepArgs) = nullptr;       // lean kernel (plain points)
  void (*kernel_full)(SweepArgs) = nullptr;  // every specialisation
  int64_t reserved_fast = 0;                 // kvsim_gpu_reserve: plain points first in `order`
  int minb = 3;
};

namespace {

constexpr int kDefaultMinBlocks = 3;
// percent of the unified L1/shared array given to shared memory
// (KVSIM_CARVEOUT; -1 = driver default): the Sim objects need ~213 KB per SM
// at 3 blocks; with the round-1 stack layout 25% (more L1 for local memory)
#if defined(KVSIM_SIM_SMEM)
constexpr int kDefaultCarveout = 100;
#else
constexpr int kDefaultCarveout = 25;
#endif
// Shipped: MINB = 3 (3 blocks of 4 warps per SM; registers and the shared
// Sim objects both allow 3). A/B builds (tools/build_variant.sh) may add a
// lean kernel with another occupancy (-DKVSIM_MINB_ALT=N, selected with
// KVSIM_MINB=N) and drop the full kernel (-DKVSIM_LEAN_ONLY: plain sweeps
// only, a much faster build). Measured: 2 blocks 5.91 vs 3 blocks 5.71 s
// (round 2, before the shared-memory Sim), 4-6 blocks slower (spills).
SweepFn sweep_variant(int minb, bool full) {
#ifdef KVSIM_LEAN_ONLY
  full = false;
#endif
  if (full) return kvsim_full_kernel(minb);
#ifdef KVSIM_MINB_ALT
  if (minb == KVSIM_MINB_ALT) return kvsim_sweep_kernel<KVSIM_MINB_ALT, false>;
#endif
  return kvsim_sweep_kernel<3, false>;
}

// Stable partition of the launch order: points the lean kernel can run first
// (returns their count); everything goes to the full kernel when the run
// records events or detail metrics.
int64_t split_order(std::vector<int64_t>& order, const kvsim_point_desc* pts, bool all_full) {
  if (all_full) return 0;
  std::stable_partition(order.begin(), order.end(), [&](int64_t i) { return !kvsim_dev::needs_full(pts[i]); });
  int64_t k = 0;
  for (int64_t i : order) k += kvsim_dev::needs_full(pts[i]) ? 0 : 1;
  return k;
}

int set_err(char* err, size_t len, int code, const std::string& msg) {
  if (err && len) {
    std::snprintf(err, len, "%s", msg.c_str());
  }
  return code;
}
#define KV_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return set_err(err, err_len, _e == cudaErrorMemoryAllocation ? KVSIM_E_OOM : KVSIM_E_CUDA, \
                     std::string(#call) + ": " + cudaGetErrorString(_e));                     \
  } while (0)

#if defined(KVSIM_SIM_SMEM)
// dynamic shared memory per block: warp scratch + one Sim object per lane
// (every specialisation has the same fields)
constexpr size_t kSimBytes = sizeof(kvsim_dev::Sim<KVSIM_POLICY_ACCELLM, true, true, true>);
static_assert(sizeof(kvsim_dev::Sim<KVSIM_POLICY_UNIFIED, false>) == kSimBytes &&
                  sizeof(kvsim_dev::Sim<KVSIM_POLICY_SPLITWISE, false>) == kSimBytes &&
                  sizeof(kvsim_dev::Sim<KVSIM_POLICY_ACCELLM, false>) == kSimBytes,
              "Sim specialisations share one layout");
size_t smem_bytes() { return sizeof(WarpScratch) * kWarpsPerBlock + kSimBytes * kWarpsPerBlock * 32; }
#else
size_t smem_bytes() { return sizeof(WarpScratch) * kWarpsPerBlock; }
#endif

// Choose the number of arena slots (= resident warps) and allocate the arena.
int prepare_arena(kvsim_gpu_ctx* c, const kvsim_host::ArenaGeom& g, size_t n_pts, char* err, size_t err_len) {
  const int64_t resident = (int64_t)c->sms * c->blocks_per_sm * kWarpsPerBlock;
  int64_t want = std::min<int64_t>(resident, (int64_t)n_pts);
  if (want < 1) want = 1;
  size_t free_b = 0, total_b = 0;
  KV_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t have = c->arena.cap;
  const size_t budget = (size_t)((double)(free_b + have) * 0.80);
  SweepArgs tmp{};
  while (want > 1 && kvsim_host::carve(tmp, nullptr, g, (int32_t)want) > budget) want = want * 3 / 4;
  const size_t bytes = kvsim_host::carve(tmp, nullptr, g, (int32_t)want);
  if (bytes > budget && want == 1)
    return set_err(err, err_len, KVSIM_E_OOM, "arena for one point exceeds device memory");
  KV_CUDA(c->arena.ensure(bytes));
  c->geom = g;
  c->slots = (int32_t)want;
  return KVSIM_OK;
}

// Launch the lean kernel over order[0, n_fast) and the full kernel over
// order[n_fast, n_pts), back to back on stream s (same arena).
int launch_sweep(kvsim_gpu_ctx* c, SweepArgs& a, int64_t n_fast, cudaStream_t s, char* err, size_t err_len) {
  const int blocks = (a.slots + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t n = a.n_pts;
  c->last_launches = 0;
  for (int part = 0; part < 2; ++part) {
    SweepArgs b = a;
    b.order = a.order + (part ? n_fast : 0);
    b.n_pts = part ? n - n_fast : n_fast;
    if (b.n_pts <= 0) continue;
    KV_CUDA(cudaMemsetAsync(b.next_point, 0, sizeof(unsigned long long), s));
    (part ? c->kernel_full : c->kernel)<<<blocks, kWarpsPerBlock * 32, smem_bytes(), s>>>(b);
    KV_CUDA(cudaGetLastError());
    c->last_launches += 1;
  }
  return KVSIM_OK;
}

}  // namespace

extern "C" {

int kvsim_gpu_abi_version(void) { return KVSIM_ABI_VERSION; }

int kvsim_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

void kvsim_point_defaults(kvsim_point_desc* p) {
  std::memset(p, 0, sizeof(*p));
  p->param_count = 70e9;
  p->num_layers = 80;
  p->hidden_dim = 8192;
  p->num_kv_heads = 8;
  p->head_dim = 128;
  p->bytes_per_value = 2;
  p->policy = KVSIM_POLICY_ACCELLM;
  p->peak_flops = 989e12;
  p->hbm_capacity = 80e9;
  p->hbm_bandwidth = 3.35e12;
  p->link_bandwidth = 900e9;
  p->num_devices = 4;
  p->tensor_parallel = 4;
  p->memory_reserve_fraction = 0.10;
  p->compute_eff = 0.5;
  p->mem_bw_eff = 0.8;
  p->link_eff = 0.8;
  p->link_mode = KVSIM_LINK_STRIPED;
  p->num_instances = 8;
  p->prefill_token_budget = 8192;
  p->prompt_min = 20;
  p->prompt_max = 1000;
  p->decode_min = 20;
  p->decode_max = 1000;
  p->arrival_process = KVSIM_ARRIVAL_POISSON;
  p->trace_index = -1;
  p->rate = 4.0;
  p->duration_s = INFINITY;
  p->warmup_s = 0.0;
  p->num_requests = 1000;
}

int kvsim_point_validate(const kvsim_point_desc* p, char* err, size_t err_len) {
  return kvsim_host::validate_point(*p, err, err_len);
}

int kvsim_gpu_open(int device, kvsim_gpu_ctx** out, char* err, size_t err_len) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return set_err(err, err_len, KVSIM_E_NO_DEVICE, "no CUDA device available (kvsim has no CPU fallback)");
  }
  if (device < 0 || device >= n) return set_err(err, err_len, KVSIM_E_INVALID, "device index out of range");
  KV_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  KV_CUDA(cudaGetDeviceProperties(&prop, device));
  // the library carries sm_100a SASS only (no PTX): anything but compute
  // capability 10.0 (sm_103, sm_12x, older parts) cannot load the kernels
  if (prop.major != 10 || prop.minor != 0)
    return set_err(err, err_len, KVSIM_E_NO_DEVICE,
                   "kvsim kernels are built for sm_100a (B200) only; device is sm_" + std::to_string(prop.major) +
                       std::to_string(prop.minor));
  int minb = kDefaultMinBlocks;
  if (const char* e = std::getenv("KVSIM_MINB")) {
    minb = std::atoi(e);
#ifdef KVSIM_MINB_ALT
    if (minb != KVSIM_MINB_ALT && minb != 3)
#else
    if (minb != 3)
#endif
      return set_err(err, err_len, KVSIM_E_INVALID, "KVSIM_MINB: this build ships the 3-blocks-per-SM kernels only");
  }
  auto* c = new kvsim_gpu_ctx();
  const int rc = [&]() -> int {
    c->device = device;
    c->sms = prop.multiProcessorCount;
    c->minb = minb;
    c->kernel = sweep_variant(c->minb, false);
    c->kernel_full = sweep_variant(c->minb, true);
    c->point_times = std::getenv("KVSIM_POINT_TIMES") != nullptr;
    // L1/shared split (percent of the unified array given to shared memory),
    // KVSIM_CARVEOUT overrides; -1 leaves the driver default
    int carve = kDefaultCarveout;
    if (const char* e = std::getenv("KVSIM_CARVEOUT")) carve = std::atoi(e);
    int bps_min = 1 << 30;
    for (SweepFn k : {c->kernel, c->kernel_full}) {
      // the kernel image must actually load on this device
      cudaFuncAttributes fa;
      KV_CUDA(cudaFuncGetAttributes(&fa, k));
      KV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes()));
      if (carve >= 0) KV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      int bps = 1;
      KV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kWarpsPerBlock * 32, smem_bytes()));
      bps_min = std::min(bps_min, bps);
    }
    c->blocks_per_sm = bps_min > 0 ? bps_min : 1;
    // resident blocks per SM actually used (<= the occupancy limit)
    if (const char* e = std::getenv("KVSIM_BLOCKS_PER_SM")) {
      const int want = std::atoi(e);
      if (want >= 1 && want < c->blocks_per_sm) c->blocks_per_sm = want;
    }
    KV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    return KVSIM_OK;
  }();
  if (rc != KVSIM_OK) {
    kvsim_gpu_close(c);
    return rc;
  }
  *out = c;
  return KVSIM_OK;
}

void kvsim_gpu_close(kvsim_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (DevBuf* b : {&c->arena, &c->pts, &c->order, &c->out, &c->recs, &c->rec_off, &c->ev, &c->ev_count, &c->ptime, &c->tr_arr,
                    &c->tr_pl, &c->tr_dl, &c->tr_off, &c->tr_n, &c->tr_dmax, &c->counter, &c->inst})
    b->release();
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int64_t kvsim_gpu_last_launches(const kvsim_gpu_ctx* c) { return c ? c->last_launches : 0; }

int64_t kvsim_gpu_point_times(kvsim_gpu_ctx* c, uint64_t* out, int64_t cap) {
  if (!c || !c->point_times || c->ptime_n == 0) return 0;
  const int64_t n = std::min<int64_t>(cap, 3 * c->ptime_n);
  if (cudaMemcpy(out, c->ptime.p, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return n;
}

int kvsim_gpu_run(kvsim_gpu_ctx* c, const kvsim_point_desc* pts, size_t n, const kvsim_trace_view* traces,
                  size_t n_traces, kvsim_point_summary* out, kvsim_request_record* recs, kvsim_event_record* ev,
                  size_t ev_cap, int64_t* ev_count, char* err, size_t err_len) {
  kvsim_run_opts o{};
  o.recs = recs;
  o.ev = ev;
  o.ev_cap = ev_cap;
  o.ev_count = ev_count;
  return kvsim_gpu_run_ex(c, pts, n, traces, n_traces, out, &o, err, err_len);
}

int kvsim_gpu_run_ex(kvsim_gpu_ctx* c, const kvsim_point_desc* pts, size_t n, const kvsim_trace_view* traces,
                     size_t n_traces, kvsim_point_summary* out, const kvsim_run_opts* opts, char* err,
                     size_t err_len) {
  const kvsim_run_opts o = opts ? *opts : kvsim_run_opts{};
  kvsim_request_record* recs = o.recs;
  kvsim_event_record* ev = o.ev;
  const size_t ev_cap = o.ev_cap;
  int64_t* ev_count = o.ev_count;
  if (!c) return set_err(err, err_len, KVSIM_E_INVALID, "null context");
  if (n == 0) return KVSIM_OK;
  if (!pts || !out) return set_err(err, err_len, KVSIM_E_INVALID, "null points/out");
  for (size_t i = 0; i < n; ++i) {
    if (pts[i].trace_index >= (int32_t)n_traces)
      return set_err(err, err_len, KVSIM_E_INVALID, "trace_index out of range");
    if (pts[i].num_requests < 0 || pts[i].num_requests > 0x7ffffff0ll)
      return set_err(err, err_len, KVSIM_E_INVALID, "num_requests out of range");
  }
  KV_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  // traces: concatenate
  std::vector<int64_t> toff(n_traces + 1, 0), tn(n_traces);
  std::vector<int32_t> tmin(n_traces, 1), tdmax(n_traces, 1);
  for (size_t k = 0; k < n_traces; ++k) {
    tn[k] = traces[k].n;
    toff[k + 1] = toff[k] + traces[k].n;
    int32_t mn = 1 << 30, dm = 1;
    for (int64_t i = 0; i < traces[k].n; ++i) {
      mn = std::min(mn, traces[k].prompt_len[i]);
      dm = std::max(dm, traces[k].decode_len[i]);
    }
    if (dm > 0x07ffffff) return set_err(err, err_len, KVSIM_E_INVALID, "trace decode_len must be < 2^27");
    tmin[k] = traces[k].n ? mn : 1;
    tdmax[k] = dm;
  }
  const int64_t tot = toff[n_traces];
  KV_CUDA(c->tr_arr.ensure(sizeof(double) * (tot + 1)));
  KV_CUDA(c->tr_pl.ensure(sizeof(int32_t) * (tot + 1)));
  KV_CUDA(c->tr_dl.ensure(sizeof(int32_t) * (tot + 1)));
  KV_CUDA(c->tr_off.ensure(sizeof(int64_t) * (n_traces + 1)));
  KV_CUDA(c->tr_n.ensure(sizeof(int64_t) * (n_traces + 1)));
  KV_CUDA(c->tr_dmax.ensure(sizeof(int32_t) * (n_traces + 1)));
  for (size_t k = 0; k < n_traces; ++k) {
    if (traces[k].n == 0) continue;
    KV_CUDA(cudaMemcpyAsync((double*)c->tr_arr.p + toff[k], traces[k].arrival_s, sizeof(double) * traces[k].n,
                            cudaMemcpyHostToDevice, s));
    KV_CUDA(cudaMemcpyAsync((int32_t*)c->tr_pl.p + toff[k], traces[k].prompt_len, sizeof(int32_t) * traces[k].n,
                            cudaMemcpyHostToDevice, s));
    KV_CUDA(cudaMemcpyAsync((int32_t*)c->tr_dl.p + toff[k], traces[k].decode_len, sizeof(int32_t) * traces[k].n,
                            cudaMemcpyHostToDevice, s));
  }
  if (n_traces) {
    KV_CUDA(cudaMemcpyAsync(c->tr_off.p, toff.data(), sizeof(int64_t) * n_traces, cudaMemcpyHostToDevice, s));
    KV_CUDA(cudaMemcpyAsync(c->tr_n.p, tn.data(), sizeof(int64_t) * n_traces, cudaMemcpyHostToDevice, s));
    KV_CUDA(cudaMemcpyAsync(c->tr_dmax.p, tdmax.data(), sizeof(int32_t) * n_traces, cudaMemcpyHostToDevice, s));
  }
  // arena
  const kvsim_host::ArenaGeom g = kvsim_host::size_arena(pts, n, tn, tmin, o.detail != 0, tdmax);
  int rc = prepare_arena(c, g, n, err, err_len);
  if (rc) return rc;
  c->reserved = false;
  // points, order, record offsets
  std::vector<int64_t> order = kvsim_host::lpt_order(pts, n);
  const int64_t n_fast = split_order(order, pts, (ev && ev_cap) || o.detail != 0);
  std::vector<int64_t> rec_off(n + 1, 0);
  for (size_t i = 0; i < n; ++i) rec_off[i + 1] = rec_off[i] + std::max<int64_t>(pts[i].num_requests, 0);
  KV_CUDA(c->pts.ensure(sizeof(kvsim_point_desc) * n));
  KV_CUDA(c->order.ensure(sizeof(int64_t) * n));
  KV_CUDA(c->out.ensure(sizeof(kvsim_point_summary) * n));
  KV_CUDA(c->rec_off.ensure(sizeof(int64_t) * (n + 1)));
  KV_CUDA(c->counter.ensure(sizeof(unsigned long long)));
  KV_CUDA(cudaMemcpyAsync(c->pts.p, pts, sizeof(kvsim_point_desc) * n, cudaMemcpyHostToDevice, s));
  KV_CUDA(cudaMemcpyAsync(c->order.p, order.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
  KV_CUDA(cudaMemcpyAsync(c->rec_off.p, rec_off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  if (recs) KV_CUDA(c->recs.ensure(sizeof(kvsim_request_record) * (rec_off[n] + 1)));
  if (ev && ev_cap) {
    KV_CUDA(c->ev.ensure(sizeof(kvsim_event_record) * ev_cap * n));
    KV_CUDA(c->ev_count.ensure(sizeof(int64_t) * n));
  }
  SweepArgs a{};
  kvsim_host::carve(a, (char*)c->arena.p, g, c->slots);
  a.pts = (const kvsim_point_desc*)c->pts.p;
  a.order = (const int64_t*)c->order.p;
  a.n_pts = (int64_t)n;
  a.out = (kvsim_point_summary*)c->out.p;
  a.tr_arr = (const double*)c->tr_arr.p;
  a.tr_pl = (const int32_t*)c->tr_pl.p;
  a.tr_dl = (const int32_t*)c->tr_dl.p;
  a.tr_off = (const int64_t*)c->tr_off.p;
  a.tr_n = (const int64_t*)c->tr_n.p;
  a.tr_dmax = (const int32_t*)c->tr_dmax.p;
  a.recs = recs ? (kvsim_request_record*)c->recs.p : nullptr;
  a.rec_off = (const int64_t*)c->rec_off.p;
  a.ev = (ev && ev_cap) ? (kvsim_event_record*)c->ev.p : nullptr;
  a.ev_cap = (int64_t)ev_cap;
  a.ev_count = (ev && ev_cap) ? (int64_t*)c->ev_count.p : nullptr;
  a.next_point = (unsigned long long*)c->counter.p;
  a.detail = o.detail != 0;
  if (o.inst) {
    KV_CUDA(c->inst.ensure(sizeof(kvsim_instance_record) * KVSIM_MAX_INSTANCES * n));
    KV_CUDA(cudaMemsetAsync(c->inst.p, 0, sizeof(kvsim_instance_record) * KVSIM_MAX_INSTANCES * n, s));
    a.inst = (kvsim_instance_record*)c->inst.p;
  }
  if (c->point_times) {
    KV_CUDA(c->ptime.ensure(sizeof(unsigned long long) * 3 * n));
    a.ptime = (unsigned long long*)c->ptime.p;
    c->ptime_n = (int64_t)n;
  }
  rc = launch_sweep(c, a, n_fast, s, err, err_len);
  if (rc) return rc;
  KV_CUDA(cudaMemcpyAsync(out, c->out.p, sizeof(kvsim_point_summary) * n, cudaMemcpyDeviceToHost, s));
  if (recs && rec_off[n] > 0)
    KV_CUDA(cudaMemcpyAsync(recs, c->recs.p, sizeof(kvsim_request_record) * rec_off[n], cudaMemcpyDeviceToHost, s));
  if (ev && ev_cap) {
    KV_CUDA(cudaMemcpyAsync(ev, c->ev.p, sizeof(kvsim_event_record) * ev_cap * n, cudaMemcpyDeviceToHost, s));
    if (ev_count) KV_CUDA(cudaMemcpyAsync(ev_count, c->ev_count.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
  }
  if (o.inst)
    KV_CUDA(cudaMemcpyAsync(o.inst, c->inst.p, sizeof(kvsim_instance_record) * KVSIM_MAX_INSTANCES * n,
                            cudaMemcpyDeviceToHost, s));
  KV_CUDA(cudaStreamSynchronize(s));
  return KVSIM_OK;
}

int kvsim_gpu_run_multi(kvsim_gpu_ctx* const* ctxs, int n_ctx, const kvsim_point_desc* pts, size_t n,
                        kvsim_point_summary* out, size_t min_chunk, kvsim_multi_stats* stats, char* err,
                        size_t err_len) {
  if (!ctxs || n_ctx < 1 || n_ctx > KVSIM_MAX_DEVICES) return set_err(err, err_len, KVSIM_E_INVALID, "bad context list");
  if (n == 0) return KVSIM_OK;
  if (!pts || !out) return set_err(err, err_len, KVSIM_E_INVALID, "null points/out");
  // KVSIM_VIRTUAL_GPUS=1 (test hook): contexts may share a device
  const bool virt = std::getenv("KVSIM_VIRTUAL_GPUS") && std::atoi(std::getenv("KVSIM_VIRTUAL_GPUS")) != 0;
  for (int k = 0; k < n_ctx; ++k) {
    if (!ctxs[k]) return set_err(err, err_len, KVSIM_E_INVALID, "null context");
    for (int j = 0; j < k && !virt; ++j)
      if (ctxs[j]->device == ctxs[k]->device)
        return set_err(err, err_len, KVSIM_E_INVALID, "contexts must be on distinct devices");
  }
  for (size_t i = 0; i < n; ++i)
    if (pts[i].trace_index >= 0) return set_err(err, err_len, KVSIM_E_INVALID, "multi-device runs use generated traces");
  const size_t slots = (size_t)ctxs[0]->sms * ctxs[0]->blocks_per_sm * kWarpsPerBlock;
  // one device: a single launch (the kernel orders its points LPT itself)
  const bool dynamic = min_chunk != 0 || (n_ctx > 1 && n > 16 * slots * (size_t)n_ctx);
  if (min_chunk == 0) min_chunk = 2 * slots;  // dynamic default: two waves of resident warps
  kvsim_host::ShardPlan plan = kvsim_host::make_plan(pts, n, n_ctx, min_chunk);
  if (!dynamic) kvsim_host::make_static(plan, pts);  // up to 16 waves per device: one LPT-balanced launch each
  std::vector<cudaEvent_t> ev0(n_ctx, nullptr), ev1(n_ctx, nullptr);
  std::vector<int64_t> launches(n_ctx, 0);
  std::vector<char> started(n_ctx, 0);
  auto chunk = [&](int w, const std::vector<int64_t>& idx, std::vector<kvsim_point_summary>& res,
                   std::string& e) -> int {
    kvsim_gpu_ctx* c = ctxs[w];
    char msg[512] = {0};
    if (cudaSetDevice(c->device) != cudaSuccess) { e = "cudaSetDevice failed"; return KVSIM_E_CUDA; }
    if (!started[w]) {
      if (cudaEventCreate(&ev0[w]) != cudaSuccess || cudaEventCreate(&ev1[w]) != cudaSuccess ||
          cudaEventRecord(ev0[w], c->stream) != cudaSuccess) {
        e = "cudaEvent setup failed";
        return KVSIM_E_CUDA;
      }
      started[w] = 1;
    }
    std::vector<kvsim_point_desc> sub(idx.size());
    for (size_t k = 0; k < idx.size(); ++k) sub[k] = pts[idx[k]];
    const int rc = kvsim_gpu_run_ex(c, sub.data(), sub.size(), nullptr, 0, res.data(), nullptr, msg, sizeof msg);
    if (rc != KVSIM_OK) { e = msg; return rc; }
    launches[w] += c->last_launches;
    if (cudaEventRecord(ev1[w], c->stream) != cudaSuccess) { e = "cudaEventRecord failed"; return KVSIM_E_CUDA; }
    return KVSIM_OK;
  };
  std::string e;
  std::vector<int64_t> per;
  const int rc = kvsim_host::run_plan(plan, out, chunk, e, &per);
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->n_devices = n_ctx;
  }
  for (int w = 0; w < n_ctx; ++w) {
    if (!started[w]) continue;
    cudaSetDevice(ctxs[w]->device);
    float ms = 0.f;
    cudaEventSynchronize(ev1[w]);
    if (stats && cudaEventElapsedTime(&ms, ev0[w], ev1[w]) == cudaSuccess) stats->device_seconds[w] = ms * 1e-3;
    cudaEventDestroy(ev0[w]);
    cudaEventDestroy(ev1[w]);
  }
  if (stats)
    for (int w = 0; w < n_ctx; ++w) {
      stats->device_points[w] = per.empty() ? 0 : per[w];
      stats->device_launches[w] = launches[w];
    }
  if (rc != KVSIM_OK) return set_err(err, err_len, rc, e);
  return KVSIM_OK;
}

int kvsim_gpu_reserve(kvsim_gpu_ctx* c, const kvsim_point_desc* pts, size_t n, char* err, size_t err_len) {
  if (!c || !pts || n == 0) return set_err(err, err_len, KVSIM_E_INVALID, "bad arguments");
  KV_CUDA(cudaSetDevice(c->device));
  for (size_t i = 0; i < n; ++i)
    if (pts[i].trace_index >= 0)
      return set_err(err, err_len, KVSIM_E_INVALID, "device-resident runs use generated traces only");
  const kvsim_host::ArenaGeom g = kvsim_host::size_arena(pts, n, {}, {});
  int rc = prepare_arena(c, g, n, err, err_len);
  if (rc) return rc;
  std::vector<int64_t> order = kvsim_host::lpt_order(pts, n);
  c->reserved_fast = split_order(order, pts, false);
  KV_CUDA(c->order.ensure(sizeof(int64_t) * n));
  KV_CUDA(c->counter.ensure(sizeof(unsigned long long)));
  KV_CUDA(cudaMemcpy(c->order.p, order.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  SweepArgs& a = c->reserved_args;
  a = SweepArgs{};
  kvsim_host::carve(a, (char*)c->arena.p, g, c->slots);
  a.order = (const int64_t*)c->order.p;
  a.n_pts = (int64_t)n;
  a.next_point = (unsigned long long*)c->counter.p;
  c->reserved = true;
  return KVSIM_OK;
}

int kvsim_gpu_run_device(kvsim_gpu_ctx* c, const kvsim_point_desc* d_pts, size_t n, kvsim_point_summary* d_out,
                         void* stream, char* err, size_t err_len) {
  if (!c || !c->reserved) return set_err(err, err_len, KVSIM_E_INVALID, "call kvsim_gpu_reserve first");
  if ((int64_t)n != c->reserved_args.n_pts)
    return set_err(err, err_len, KVSIM_E_INVALID, "point count differs from the reservation");
  if (!d_pts || !d_out) return set_err(err, err_len, KVSIM_E_INVALID, "null device points/out");
  KV_CUDA(cudaSetDevice(c->device));
  // d_pts must hold the points passed to kvsim_gpu_reserve; the kernel
  // re-checks every point against the reserved arena geometry and reports
  // KVSIM_E_INVALID in its summary instead of overrunning a slot
  SweepArgs a = c->reserved_args;
  a.pts = d_pts;
  a.out = d_out;
  return launch_sweep(c, a, c->reserved_fast, stream ? (cudaStream_t)stream : c->stream, err, err_len);
}

int kvsim_gpu_perf_batch(kvsim_gpu_ctx* c, const kvsim_point_desc* pts, size_t n_pts, const int32_t* pidx,
                         const int32_t* op, const int64_t* s1, const int64_t* s2, double* out, size_t n, char* err,
                         size_t err_len) {
  if (!c) return set_err(err, err_len, KVSIM_E_INVALID, "null context");
  if (n == 0) return KVSIM_OK;
  KV_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  DevBuf dp, di, dop, d1, d2, dout;
  auto cleanup = [&]() { dp.release(); di.release(); dop.release(); d1.release(); d2.release(); dout.release(); };
  cudaError_t e = cudaSuccess;
  if ((e = dp.ensure(sizeof(kvsim_point_desc) * n_pts)) || (e = di.ensure(4 * n)) || (e = dop.ensure(4 * n)) ||
      (e = d1.ensure(8 * n)) || (e = d2.ensure(8 * n)) || (e = dout.ensure(8 * n))) {
    cleanup();
    return set_err(err, err_len, KVSIM_E_OOM, cudaGetErrorString(e));
  }
  cudaMemcpyAsync(dp.p, pts, sizeof(kvsim_point_desc) * n_pts, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(di.p, pidx, 4 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dop.p, op, 4 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d1.p, s1, 8 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d2.p, s2, 8 * n, cudaMemcpyHostToDevice, s);
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((n + threads - 1) / threads, 148 * 8);
  kvsim_perf_kernel<<<blocks, threads, 0, s>>>((const kvsim_point_desc*)dp.p, (const int32_t*)di.p,
                                               (const int32_t*)dop.p, (const int64_t*)d1.p, (const int64_t*)d2.p,
                                               (double*)dout.p, (int64_t)n);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout.p, 8 * n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cleanup();
  if (e != cudaSuccess) return set_err(err, err_len, KVSIM_E_CUDA, cudaGetErrorString(e));
  c->last_launches = 1;
  return KVSIM_OK;
}

int kvsim_gpu_curves(kvsim_gpu_ctx* c, const kvsim_point_desc* p, const int64_t* lengths, size_t n_len,
                     const int64_t* batch_sizes, size_t n_batch, int phase, double* latency_s, double* tokens_per_s,
                     char* err, size_t err_len) {
  if (!c || !p || !lengths || !batch_sizes || !latency_s || !tokens_per_s)
    return set_err(err, err_len, KVSIM_E_INVALID, "null argument");
  if (n_len == 0 || n_batch == 0) return set_err(err, err_len, KVSIM_E_INVALID, "empty lengths or batch_sizes");
  if (phase != 0 && phase != 1) return set_err(err, err_len, KVSIM_E_INVALID, "phase: 0 prefill, 1 decode");
  const size_t n = n_len * n_batch;
  std::vector<int32_t> pidx(n, 0), op(n, phase == 0 ? 0 : 1);
  std::vector<int64_t> s1(n), s2(n);
  for (size_t li = 0; li < n_len; ++li)
    for (size_t bi = 0; bi < n_batch; ++bi) {
      const int64_t L = lengths[li], b = batch_sizes[bi];
      if (L < 1 || b < 1) return set_err(err, err_len, KVSIM_E_EMPTY_BATCH, phase == 0 ? "empty prefill batch" : "empty decode batch");
      const size_t r = li * n_batch + bi;
      if (phase == 0) { s1[r] = b * L; s2[r] = b * L * L; }  // prefill_latency of b prompts of length L
      else { s1[r] = b; s2[r] = b * L; }                      // decode_step_latency of b requests at KV L
    }
  const int rc = kvsim_gpu_perf_batch(c, p, 1, pidx.data(), op.data(), s1.data(), s2.data(), latency_s, n, err, err_len);
  if (rc != KVSIM_OK) return rc;
  for (size_t r = 0; r < n; ++r) {
    tokens_per_s[r] = (double)s1[r] / latency_s[r];  // s1 = tokens: b * L (prefill) or b (one decode step)
  }
  return KVSIM_OK;
}

int kvsim_gpu_gen_trace(kvsim_gpu_ctx* c, const kvsim_point_desc* p, double* arrival_s, int32_t* prompt_len,
                        int32_t* decode_len, int64_t* n_out, char* err, size_t err_len) {
  if (!c || !p) return set_err(err, err_len, KVSIM_E_INVALID, "null argument");
  KV_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const int64_t cap = p->num_requests > 0 ? p->num_requests : 0;
  DevBuf da, dp, dd, dn;
  cudaError_t e = cudaSuccess;
  if ((e = da.ensure(8 * (cap + 1))) || (e = dp.ensure(4 * (cap + 1))) || (e = dd.ensure(4 * (cap + 1))) ||
      (e = dn.ensure(8))) {
    da.release(); dp.release(); dd.release(); dn.release();
    return set_err(err, err_len, KVSIM_E_OOM, cudaGetErrorString(e));
  }
  kvsim_trace_kernel<<<1, 32, 0, s>>>(*p, (double*)da.p, (int32_t*)dp.p, (int32_t*)dd.p, cap, (int64_t*)dn.p);
  e = cudaGetLastError();
  int64_t nn = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nn, dn.p, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && nn > 0) {
    cudaMemcpy(arrival_s, da.p, 8 * nn, cudaMemcpyDeviceToHost);
    cudaMemcpy(prompt_len, dp.p, 4 * nn, cudaMemcpyDeviceToHost);
    e = cudaMemcpy(decode_len, dd.p, 4 * nn, cudaMemcpyDeviceToHost);
  }
  da.release(); dp.release(); dd.release(); dn.release();
  if (e != cudaSuccess) return set_err(err, err_len, KVSIM_E_CUDA, cudaGetErrorString(e));
  *n_out = nn;
  c->last_launches = 1;
  return KVSIM_OK;
}

void* kvsim_gpu_host_alloc(size_t bytes) {
  int n = 0;
  if (bytes == 0 || cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return nullptr;
  }
  void* p = nullptr;
  // portable: usable by every device context (the CLI's one thread per GPU)
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void kvsim_gpu_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
