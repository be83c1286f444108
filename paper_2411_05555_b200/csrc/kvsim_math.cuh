// kvsim_math.cuh — analytical cost model, portable RNG and portable log,
// shared by the sm_100a kernels and the host-side C++ API (product code).
//
// Restates reference perfmodel.hpp:76-106 / SPEC.md:47-100 (cost model) and
// docs/SEMANTICS.md §1-2 (operation order, RNG). Every floating-point op is an
// explicitly rounded IEEE op (kadd/kmul/kdiv) so that nvcc cannot contract
// a*b+c into an FMA on the device; the host build uses -ffp-contract=off.
#pragma once
#include <stdint.h>

#include "kvsim_gpu.h"

#if defined(__CUDACC__)
#define KV_HD __host__ __device__ __forceinline__
#else
#define KV_HD inline
#endif

namespace kvsim_math {

KV_HD double kadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
KV_HD double ksub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
KV_HD double kmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
#if defined(__CUDACC__)
// One out-of-line copy of the IEEE division: inlined, __ddiv_rn's ~40-instruction
// sequence was replicated at ~100 call sites and the hot loop's code no longer
// fit the SM instruction cache (ncu: sm__icc_request_hit_rate 63%).
__device__ __noinline__ inline double kdiv_ool(double a, double b) { return __ddiv_rn(a, b); }
#endif
KV_HD double kdiv(double a, double b) {
#if defined(__CUDA_ARCH__)
  return kdiv_ool(a, b);
#else
  return a / b;
#endif
}
KV_HD double kmax(double a, double b) { return a > b ? a : b; }
KV_HD double kfma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}

KV_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b;
  __builtin_memcpy(&b, &d, 8);
  return b;
#endif
}
KV_HD double as_f64(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}

// ------------------------------------------------------------------ RNG (§2)
KV_HD uint64_t splitmix_fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
KV_HD uint64_t stream_key(uint64_t seed) { return splitmix_fin(seed ^ 0x243F6A8885A308D3ull); }
KV_HD uint64_t draw_k(uint64_t key, int64_t i, int s) {
  return splitmix_fin(key + 0x9E3779B97F4A7C15ull * (uint64_t)(4 * i + s + 1));
}
KV_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}
KV_HD int32_t uniform_range(uint64_t x, int32_t lo, int32_t hi) {
  return lo + (int32_t)mulhi64(x, (uint64_t)((int64_t)hi - lo + 1));
}
// (0,1] with 53 random bits
KV_HD double unit_open0(uint64_t x) { return kmul((double)((x >> 11) + 1), 1.1102230246251565e-16); }

// Natural log for x in (0, +inf), fdlibm-style argument reduction
// x = 2^k (1+f), s = f/(2+f), minimax polynomial in s^2; basic ops only.
KV_HD double plog(double x) {
  const double ln2_hi = as_f64(0x3fe62e42fee00000ull), ln2_lo = as_f64(0x3dea39ef35793c76ull);
  const double c1 = as_f64(0x3FE5555555555593ull), c2 = as_f64(0x3FD999999997FA04ull),
               c3 = as_f64(0x3FD2492494229359ull), c4 = as_f64(0x3FCC71C51D8E78AFull),
               c5 = as_f64(0x3FC7466496CB03DEull), c6 = as_f64(0x3FC39A09D078C69Full),
               c7 = as_f64(0x3FC2F112DF3E5244ull);
  uint64_t bits = as_u64(x);
  int32_t hi = (int32_t)(bits >> 32);
  int32_t e = 0;
  if (hi < 0x00100000) {  // zero, negative or subnormal
    if (((hi & 0x7fffffff) | (uint32_t)bits) == 0) return -as_f64(0x7ff0000000000000ull);
    if (hi < 0) return as_f64(0x7ff8000000000000ull);
    e = -54;
    x = kmul(x, 18014398509481984.0);
    bits = as_u64(x);
    hi = (int32_t)(bits >> 32);
  }
  if (hi >= 0x7ff00000) return kadd(x, x);
  e += (hi >> 20) - 1023;
  int32_t m = hi & 0x000fffff;
  int32_t sel = (m + 0x95f64) & 0x100000;  // pick x or x/2 so that 1+f in [sqrt(2)/2, sqrt(2))
  bits = ((uint64_t)(uint32_t)(m | (sel ^ 0x3ff00000)) << 32) | (bits & 0xffffffffull);
  x = as_f64(bits);
  e += sel >> 20;
  const double f = ksub(x, 1.0);
  const double de = (double)e;
  if ((0x000fffff & (2 + m)) < 3) {  // |f| < 2^-20
    if (f == 0.0) return e == 0 ? 0.0 : kadd(kmul(de, ln2_hi), kmul(de, ln2_lo));
    double r = kmul(kmul(f, f), ksub(0.5, kmul(0.33333333333333333, f)));
    if (e == 0) return ksub(f, r);
    return ksub(kmul(de, ln2_hi), ksub(ksub(r, kmul(de, ln2_lo)), f));
  }
  const double s = kdiv(f, kadd(2.0, f));
  const double z = kmul(s, s);
  const double w = kmul(z, z);
  const double odd = kmul(w, kadd(c2, kmul(w, kadd(c4, kmul(w, c6)))));
  const double even = kmul(z, kadd(c1, kmul(w, kadd(c3, kmul(w, kadd(c5, kmul(w, c7)))))));
  const double r = kadd(even, odd);
  const int32_t band = (m - 0x6147a) | (0x6b851 - m);
  if (band > 0) {
    const double hfsq = kmul(kmul(0.5, f), f);
    if (e == 0) return ksub(f, ksub(hfsq, kmul(s, kadd(hfsq, r))));
    return ksub(kmul(de, ln2_hi), ksub(ksub(hfsq, kadd(kmul(s, kadd(hfsq, r)), kmul(de, ln2_lo))), f));
  }
  if (e == 0) return ksub(f, kmul(s, ksub(f, r)));
  return ksub(kmul(de, ln2_hi), ksub(ksub(kmul(s, ksub(f, r)), kmul(de, ln2_lo)), f));
}

// Exponential inter-arrival gap for request i (SEMANTICS §2).
KV_HD double poisson_gap(uint64_t key, int64_t i, double rate) {
  return kdiv(-plog(unit_open0(draw_k(key, i, 2))), rate);
}

// Correctly rounded n / d for positive normal operands, given rd = RN(1/d).
// q1 = q0 + (n - q0 d) rd is accepted only if its exact remainder
// r1 = n - q1 d (one FMA; exact whenever q1 is the correctly rounded
// quotient) satisfies |r1| < d * ulp(q1)/2 with q1 not a power of two. That
// inequality holds iff q1 == RN(n / d) and n / d is not a tie, so the result
// equals IEEE division bit for bit; otherwise the IEEE division is used.
KV_HD double kdiv_rcp(double n, double d, double rd) {
  const double q0 = kmul(n, rd);
  const double q1 = kfma(kfma(-q0, d, n), rd, q0);
  const double r1 = kfma(-q1, d, n);
  const uint64_t qb = as_u64(q1);
  const uint64_t ex = (qb >> 52) & 0x7ffull;
  if ((qb & 0x000fffffffffffffull) != 0 && ex > 54 && ex < 0x7ff) {
    const double h = kmul(d, as_f64((ex - 53) << 52));  // d * ulp(q1) / 2, exact (power of two)
    const double ar = r1 < 0.0 ? -r1 : r1;
    if (ar < h) return q1;
  }
  return kdiv(n, d);
}

// Step chains divide an increasing numerator by a fixed d, starting from a
// quotient qmin verified by kdiv_rcp. Threshold for kdiv_chain:
// T = d ulp(qmin) / 2 (d ulp(qmin) / 4 when qmin is a power of two), or 0
// (every quotient then takes the IEEE division) when qmin or T leave the
// normal range the test needs.
KV_HD double kdiv_chain_thr(double qmin, double d) {
  const uint64_t qb = as_u64(qmin);
  const uint64_t ex = (qb >> 52) & 0x7ffull;
  if (ex <= 55 || ex >= 0x7ff) return 0.0;
  const uint64_t sh = (qb & 0x000fffffffffffffull) == 0 ? 54 : 53;
  const double T = kmul(d, as_f64((ex - sh) << 52));
  return T >= 0x1p-1022 && T < as_f64(0x7ff0000000000000ull) ? T : 0.0;
}
// RN(n / d) for a quotient not below qmin. q1 (one Newton correction of
// n rd) is accepted iff |n - q1 d| < T and q1 >= qmin. That implies the
// kdiv_rcp test (|r1| < d ulp(q1) / 2, since ulp(q1) >= ulp(qmin)) and also
// covers a power-of-two q1: q1 > qmin then lies in a higher binade than
// qmin, so T <= d ulp(q1) / 4, half the gap to q1's lower neighbour (and
// q1 == qmin uses the quarter-ulp T). The test is a loop-invariant compare
// instead of kdiv_rcp's per-quotient exponent arithmetic; failures take the
// IEEE division.
KV_HD double kdiv_chain(double n, double d, double rd, double T, double qmin) {
  const double q0 = kmul(n, rd);
  const double q1 = kfma(kfma(-q0, d, n), rd, q0);
  const double r1 = kfma(-q1, d, n);
  const double ar = r1 < 0.0 ? -r1 : r1;
  if (ar < T && q1 >= qmin) return q1;
  return kdiv(n, d);
}

// ----------------------------------------------------------- cost model (§1)
struct Perf {
  double kvb;        // bytes of K+V per token, all layers
  double kvb_layer;  // one layer
  double W;          // weight bytes
  double pf_den;     // num_devices * peak_flops * compute_eff
  double mem_den;    // num_devices * hbm_bandwidth * mem_bw_eff
  double mem_rcp;    // RN(1 / mem_den), for kdiv_rcp
  double two_p;      // 2 * param_count
  double attn;       // 4 * hidden * layers
  double link_bw;    // effective inter-instance bandwidth
  int64_t cap;       // kv_capacity_tokens
  int32_t fits;
};

KV_HD Perf make_perf(const kvsim_point_desc& p) {
  Perf f;
  f.kvb = (double)(2ll * p.num_layers * p.num_kv_heads * p.head_dim * p.bytes_per_value);
  f.kvb_layer = (double)(2ll * p.num_kv_heads * p.head_dim * p.bytes_per_value);
  f.W = kmul(p.param_count, (double)p.bytes_per_value);
  f.pf_den = kmul(kmul((double)p.num_devices, p.peak_flops), p.compute_eff);
  f.mem_den = kmul(kmul((double)p.num_devices, p.hbm_bandwidth), p.mem_bw_eff);
  f.mem_rcp = kdiv(1.0, f.mem_den);
  f.two_p = kmul(2.0, p.param_count);
  f.attn = (double)(4ll * p.hidden_dim * p.num_layers);
  f.link_bw = p.link_mode == KVSIM_LINK_SINGLE
                  ? kmul(p.link_bandwidth, p.link_eff)
                  : kmul(kmul((double)p.num_devices, p.link_bandwidth), p.link_eff);
  const double usable = kmul(kmul((double)p.num_devices, p.hbm_capacity), ksub(1.0, p.memory_reserve_fraction));
  const double room = ksub(usable, f.W);
  f.fits = room >= 0.0;
#if defined(__CUDA_ARCH__)
  f.cap = f.fits ? (int64_t)floor(kdiv(room, f.kvb)) : 0;
#else
  f.cap = f.fits ? (int64_t)__builtin_floor(kdiv(room, f.kvb)) : 0;
#endif
  return f;
}

// prefill_latency in sum form: s1 = sum L, s2 = sum L^2 (perfmodel.hpp:84-86)
KV_HD double prefill_latency(const Perf& f, int64_t s1, int64_t s2) {
  return kdiv(kadd(kmul(f.two_p, (double)s1), kmul(f.attn, (double)s2)), f.pf_den);
}
// decode_step_latency: batch B, sum kv K (perfmodel.hpp:90-92)
KV_HD double decode_latency(const Perf& f, int64_t B, int64_t K) {
  const double mem = kdiv(kadd(f.W, kmul((double)K, f.kvb)), f.mem_den);
  const double comp = kdiv(kmul(f.two_p, (double)B), f.pf_den);
  return kmax(mem, comp);
}
// transfer_latency (perfmodel.hpp:95-97)
KV_HD double transfer_latency(const Perf& f, double bytes) { return kdiv(bytes, f.link_bw); }

}  // namespace kvsim_math
