// kvsim_simt.cuh — the warp primitives the simulation core is written in.
//
// Device build (nvcc, sm_100a): thin wrappers over __ballot_sync /
// __shfl_sync / __syncwarp with the full-warp mask.
//
// KVSIM_EMU build (host g++, tests only): a fiber-based SIMT emulator used by
// the CPU test suite to run the *same* kernel source against the oracle
// without a GPU (tests/emu). Every primitive is one round-robin pass over the
// 32 lane contexts. It is never linked into the product library.
#pragma once
#include <stdint.h>

#if defined(KVSIM_EMU)
#include <atomic>
#include <cstdlib>
#include <cstring>
#define KV_DEV inline
#define KV_HD_INLINE inline
#define KV_DEV_NOINLINE inline
// Fiber-based warp: the 32 lanes are user-level contexts on one OS thread and
// run round-robin between primitives (one full round per primitive), so the
// emulation is deterministic and a lane never observes a half-finished round.
extern "C" void kvemu_ctx_switch(void** save_sp, void* load_sp);
__asm__(
    ".text\n.globl kvemu_ctx_switch\n.type kvemu_ctx_switch,@function\n"
    "kvemu_ctx_switch:\n"
    "  pushq %rbp\n  pushq %rbx\n  pushq %r12\n  pushq %r13\n  pushq %r14\n  pushq %r15\n"
    "  movq %rsp, (%rdi)\n  movq %rsi, %rsp\n"
    "  popq %r15\n  popq %r14\n  popq %r13\n  popq %r12\n  popq %rbx\n  popq %rbp\n"
    "  ret\n.size kvemu_ctx_switch, .-kvemu_ctx_switch\n");
namespace simt {
struct WarpEmu {
  void* sp[32];
  void* main_sp = nullptr;
  uint64_t slot[2][32];
  int phase[32];
  int cur = 0;
  int n_done = 0;
  void (*body)(void*, int) = nullptr;
  void* arg = nullptr;
  char* stacks = nullptr;
};
inline thread_local int tl_lane = 0;
inline thread_local WarpEmu* tl_warp = nullptr;
inline int lane_id() { return tl_lane; }
inline void yield_round() {
  WarpEmu* w = tl_warp;
  const int me = w->cur;
  const int nx = (me + 1) & 31;
  w->cur = nx;
  tl_lane = nx;
  kvemu_ctx_switch(&w->sp[me], w->sp[nx]);
}
inline void lane_entry() {
  WarpEmu* w = tl_warp;
  const int me = w->cur;
  w->body(w->arg, me);
  w->n_done += 1;
  if (me == 31) {
    kvemu_ctx_switch(&w->sp[me], w->main_sp);
  } else {
    w->cur = me + 1;
    tl_lane = me + 1;
    kvemu_ctx_switch(&w->sp[me], w->sp[me + 1]);
  }
  std::abort();  // never resumed
}
// Run body(arg, lane) for 32 lanes as one emulated warp on this thread.
inline void run_warp(void (*body)(void*, int), void* arg) {
  const size_t kStack = 1 << 20;
  WarpEmu w;
  w.body = body;
  w.arg = arg;
  w.stacks = (char*)std::aligned_alloc(64, kStack * 32);
  for (int l = 0; l < 32; ++l) {
    w.phase[l] = 0;
    char* hi = w.stacks + kStack * (l + 1);
    uintptr_t top = ((uintptr_t)hi) & ~(uintptr_t)15;
    void** sp = (void**)(top - 64);
    for (int k = 0; k < 6; ++k) sp[k] = nullptr;
    sp[6] = (void*)&lane_entry;
    sp[7] = nullptr;
    w.sp[l] = (void*)sp;
  }
  WarpEmu* prev = tl_warp;
  tl_warp = &w;
  w.cur = 0;
  tl_lane = 0;
  kvemu_ctx_switch(&w.main_sp, w.sp[0]);
  tl_warp = prev;
  std::free(w.stacks);
}
inline void sync() { yield_round(); }
inline uint64_t xchg(uint64_t v, int src) {
  WarpEmu* w = tl_warp;
  const int me = tl_lane;
  const int p = w->phase[me];
  w->slot[p][me] = v;
  w->phase[me] = p ^ 1;
  yield_round();
  return w->slot[p][src & 31];
}
inline unsigned ballot(bool b) {
  WarpEmu* w = tl_warp;
  const int me = tl_lane;
  const int p = w->phase[me];
  w->slot[p][me] = b ? 1 : 0;
  w->phase[me] = p ^ 1;
  yield_round();
  unsigned m = 0;
  for (int i = 0; i < 32; ++i) m |= (unsigned)(w->slot[p][i] & 1) << i;
  return m;
}
template <class T>
inline T shfl(T v, int src) {
  static_assert(sizeof(T) <= 8, "shfl type");
  uint64_t b = 0;
  std::memcpy(&b, &v, sizeof(T));
  b = xchg(b, src);
  T r;
  std::memcpy(&r, &b, sizeof(T));
  return r;
}
template <class T>
inline T shfl_xor(T v, int m) { return shfl(v, tl_lane ^ m); }
inline int popc(unsigned x) { return __builtin_popcount(x); }
inline int ffs(unsigned x) { return __builtin_ffs((int)x); }
template <class T>
inline T atomic_add_smem(T* p, T v) { T o = *p; *p = o + v; return o; }
inline double floor_d(double x) { return __builtin_floor(x); }
}  // namespace simt
#else
#define KV_DEV __device__ __forceinline__
#define KV_HD_INLINE __host__ __device__ __forceinline__
#define KV_DEV_NOINLINE __device__ __noinline__
namespace simt {
__device__ __forceinline__ int lane_id() { return (int)(threadIdx.x & 31); }
__device__ __forceinline__ void sync() { __syncwarp(); }
__device__ __forceinline__ unsigned ballot(bool p) { return __ballot_sync(0xffffffffu, p); }
__device__ __forceinline__ int32_t shfl(int32_t v, int s) { return __shfl_sync(0xffffffffu, v, s); }
__device__ __forceinline__ uint32_t shfl(uint32_t v, int s) { return __shfl_sync(0xffffffffu, v, s); }
__device__ __forceinline__ int64_t shfl(int64_t v, int s) { return __shfl_sync(0xffffffffu, (long long)v, s); }
__device__ __forceinline__ uint64_t shfl(uint64_t v, int s) {
  return (uint64_t)__shfl_sync(0xffffffffu, (unsigned long long)v, s);
}
__device__ __forceinline__ double shfl(double v, int s) { return __shfl_sync(0xffffffffu, v, s); }
template <class T>
__device__ __forceinline__ T shfl_xor(T v, int m) { return shfl(v, (int)(threadIdx.x & 31) ^ m); }
__device__ __forceinline__ int popc(unsigned x) { return __popc(x); }
__device__ __forceinline__ int ffs(unsigned x) { return __ffs((int)x); }
__device__ __forceinline__ int32_t atomic_add_smem(int32_t* p, int32_t v) { return atomicAdd(p, v); }
__device__ __forceinline__ int64_t atomic_add_smem(int64_t* p, int64_t v) {
  return (int64_t)atomicAdd((unsigned long long*)p, (unsigned long long)v);
}
__device__ __forceinline__ uint32_t atomic_add_smem(uint32_t* p, uint32_t v) { return atomicAdd(p, v); }
__device__ __forceinline__ double floor_d(double x) { return floor(x); }
}  // namespace simt
#endif

namespace simt {
// 32-bit unsigned warp reductions: one REDUX instruction on sm_100a
#if defined(KVSIM_EMU)
inline uint32_t reduce_min_u32(uint32_t v) {
  for (int m = 16; m; m >>= 1) { uint32_t o = shfl_xor(v, m); v = o < v ? o : v; }
  return v;
}
inline uint32_t reduce_max_u32(uint32_t v) {
  for (int m = 16; m; m >>= 1) { uint32_t o = shfl_xor(v, m); v = o > v ? o : v; }
  return v;
}
inline uint32_t reduce_add_u32(uint32_t v) {
  for (int m = 16; m; m >>= 1) v += shfl_xor(v, m);
  return v;
}
#else
__device__ __forceinline__ uint32_t reduce_min_u32(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t reduce_max_u32(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t reduce_add_u32(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }
#endif
// lexicographic warp min of (t, k) for t >= 0 (IEEE bit order == numeric
// order for non-negative doubles, +inf included): three REDUX instead of
// five shuffle rounds of (double, int)
KV_DEV void warp_min_tk(double& t, uint32_t& k) {
  uint64_t b;
#if defined(KVSIM_EMU)
  __builtin_memcpy(&b, &t, 8);
#else
  b = (uint64_t)__double_as_longlong(t);
#endif
  const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
  const uint32_t mh = reduce_min_u32(hi);
  const uint32_t ml = reduce_min_u32(hi == mh ? lo : 0xffffffffu);
  const uint32_t mk = reduce_min_u32(hi == mh && lo == ml ? k : 0xffffffffu);
  b = ((uint64_t)mh << 32) | ml;
#if defined(KVSIM_EMU)
  __builtin_memcpy(&t, &b, 8);
#else
  t = __longlong_as_double((long long)b);
#endif
  k = mk;
}
// 64-bit unsigned min / max: REDUX on the high words, then on the low words
// of the lanes holding the extreme high word
KV_DEV uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t mh = reduce_min_u32(hi);
  const uint32_t ml = reduce_min_u32(hi == mh ? lo : 0xffffffffu);
  return ((uint64_t)mh << 32) | ml;
}
KV_DEV uint64_t warp_max_u64(uint64_t v) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t mh = reduce_max_u32(hi);
  const uint32_t ml = reduce_max_u32(hi == mh ? lo : 0u);
  return ((uint64_t)mh << 32) | ml;
}
// signed variants: flipping the sign bit maps int order onto unsigned order
KV_DEV int64_t warp_min_i64(int64_t v) {
  return (int64_t)(warp_min_u64((uint64_t)v ^ 0x8000000000000000ull) ^ 0x8000000000000000ull);
}
KV_DEV int64_t warp_max_i64(int64_t v) {
  return (int64_t)(warp_max_u64((uint64_t)v ^ 0x8000000000000000ull) ^ 0x8000000000000000ull);
}
KV_DEV int32_t warp_min_i32(int32_t v) { return (int32_t)(reduce_min_u32((uint32_t)v ^ 0x80000000u) ^ 0x80000000u); }
KV_DEV int32_t warp_max_i32(int32_t v) { return (int32_t)(reduce_max_u32((uint32_t)v ^ 0x80000000u) ^ 0x80000000u); }
// exact sum of non-negative int64 lanes: one REDUX when every lane is below
// 2^26 (the 32-lane total then fits 31 bits), shuffle tree otherwise
template <class T>
KV_DEV T warp_sum(T v);
KV_DEV int64_t warp_sum_nn(int64_t v) {
  if (ballot((uint64_t)v >= (1ull << 26)) == 0) return (int64_t)reduce_add_u32((uint32_t)v);
  return warp_sum(v);
}
KV_DEV int32_t warp_sum_i32(int32_t v) { return (int32_t)reduce_add_u32((uint32_t)v); }
// ---------------------------------------------------------- warp reductions
template <class T>
KV_DEV T warp_sum(T v) {
  for (int m = 16; m; m >>= 1) v += shfl_xor(v, m);
  return v;
}
template <class T>
KV_DEV T warp_max(T v) {
  for (int m = 16; m; m >>= 1) {
    T o = shfl_xor(v, m);
    v = o > v ? o : v;
  }
  return v;
}
template <class T>
KV_DEV T warp_min(T v) {
  for (int m = 16; m; m >>= 1) {
    T o = shfl_xor(v, m);
    v = o < v ? o : v;
  }
  return v;
}
// inclusive prefix sum across lanes
template <class T>
KV_DEV T warp_incl_scan(T v) {
  const int lane = lane_id();
  for (int d = 1; d < 32; d <<= 1) {
    T o = shfl(v, lane - d < 0 ? 0 : lane - d);
    if (lane >= d) v += o;
  }
  return v;
}
KV_DEV unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }
}  // namespace simt

// 16-byte vector types for the vectorised SoA passes (CUDA's int4 / double2
// on the device; plain aligned structs for the host emulator)
#if defined(KVSIM_EMU)
struct alignas(16) kv_int4 { int32_t x, y, z, w; };
struct alignas(16) kv_double2 { double x, y; };
#else
typedef int4 kv_int4;
typedef double2 kv_double2;
#endif
