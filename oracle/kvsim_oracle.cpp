// kvsim_oracle.cpp — CPU ORACLE for parity tests and the CPU baseline.
//
// TEST INFRASTRUCTURE ONLY: the product path (paper_2411_05555_b200/csrc) never
// links this file. It restates the reference's kvsim behaviour (reference
// SPEC.md modules perfmodel 24-134, workload 136-190, engine 192-274,
// policy 276-350, metrics 352-398) as a deliberately plain, sequential
// discrete-event simulation: explicit per-request structs, std::vector
// batches, a linear scan for the next event, per-request token timestamps.
// Every rule follows docs/SEMANTICS.md; section numbers (§) refer to it.
//
// Build: g++ -O3 -std=gnu++20 -ffp-contract=off -fPIC -shared (oracle/Makefile),
// mirroring the reference's Release flags (reference proj/CMakeLists.txt:7-9).
#include "kvsim_oracle.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <thread>
#include <vector>

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
// SPEC.md:254-259,469 invariant checking after every event (tests only)
std::atomic<int> g_check_invariants{0};
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

// ---------------------------------------------------------------- RNG (§2)
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t draw(uint64_t seed, int64_t i, int s) {
  uint64_t key = mix64(seed ^ 0x243F6A8885A308D3ull);
  return mix64(key + 0x9E3779B97F4A7C15ull * (uint64_t)(4 * i + s + 1));
}
int32_t uniform_int(uint64_t x, int32_t lo, int32_t hi) {
  unsigned __int128 prod = (unsigned __int128)x * (uint64_t)((int64_t)hi - lo + 1);
  return lo + (int32_t)(uint64_t)(prod >> 64);
}

// fdlibm-style natural log (restated; only IEEE +,-,*,/ and bit fiddling).
double bits_to_d(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }
uint64_t d_to_bits(double d) { uint64_t b; std::memcpy(&b, &d, 8); return b; }
double klog(double x) {
  const double ln2_hi = bits_to_d(0x3fe62e42fee00000ull), ln2_lo = bits_to_d(0x3dea39ef35793c76ull);
  const double Lg1 = bits_to_d(0x3FE5555555555593ull), Lg2 = bits_to_d(0x3FD999999997FA04ull),
               Lg3 = bits_to_d(0x3FD2492494229359ull), Lg4 = bits_to_d(0x3FCC71C51D8E78AFull),
               Lg5 = bits_to_d(0x3FC7466496CB03DEull), Lg6 = bits_to_d(0x3FC39A09D078C69Full),
               Lg7 = bits_to_d(0x3FC2F112DF3E5244ull);
  uint64_t b = d_to_bits(x);
  int32_t hx = (int32_t)(b >> 32);
  uint32_t lx = (uint32_t)b;
  int32_t k = 0;
  if (hx < 0x00100000) {  // subnormal or zero / negative
    if (((hx & 0x7fffffff) | lx) == 0) return -kInf;
    if (hx < 0) return kNaN;
    k -= 54;
    x = x * 18014398509481984.0;  // 2^54
    b = d_to_bits(x);
    hx = (int32_t)(b >> 32);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int32_t i = (hx + 0x95f64) & 0x100000;
  b = d_to_bits(x);
  b = ((uint64_t)(uint32_t)(hx | (i ^ 0x3ff00000)) << 32) | (b & 0xffffffffull);
  x = bits_to_d(b);
  k += (i >> 20);
  double f = x - 1.0;
  double dk = (double)k;
  if ((0x000fffff & (2 + hx)) < 3) {
    if (f == 0.0) return k == 0 ? 0.0 : dk * ln2_hi + dk * ln2_lo;
    double R = f * f * (0.5 - 0.33333333333333333 * f);
    return k == 0 ? f - R : dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  double s = f / (2.0 + f);
  double z = s * s;
  i = hx - 0x6147a;
  double w = z * z;
  int32_t j = 0x6b851 - hx;
  double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  double R = t2 + t1;
  if (i > 0) {
    double hfsq = 0.5 * f * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

// ---------------------------------------------------------- perfmodel (§1)
struct Perf {
  double kvb, kvb_layer, W, pf_den, mem_den, comp_den, two_p, attn_coef, link_bw;
  int64_t cap;
  bool fits;
};
Perf make_perf(const kvsim_point_desc& p) {
  Perf f{};
  int64_t kvb = 2ll * p.num_layers * p.num_kv_heads * p.head_dim * p.bytes_per_value;
  f.kvb = (double)kvb;
  f.kvb_layer = (double)(2ll * p.num_kv_heads * p.head_dim * p.bytes_per_value);
  f.W = p.param_count * (double)p.bytes_per_value;
  f.pf_den = ((double)p.num_devices * p.peak_flops) * p.compute_eff;
  f.mem_den = ((double)p.num_devices * p.hbm_bandwidth) * p.mem_bw_eff;
  f.comp_den = f.pf_den;
  f.two_p = 2.0 * p.param_count;
  f.attn_coef = (double)(4ll * p.hidden_dim * p.num_layers);
  f.link_bw = p.link_mode == KVSIM_LINK_SINGLE ? p.link_bandwidth * p.link_eff
                                               : ((double)p.num_devices * p.link_bandwidth) * p.link_eff;
  double usable = (double)p.num_devices * p.hbm_capacity * (1.0 - p.memory_reserve_fraction);
  double room = usable - f.W;
  f.fits = room >= 0.0;
  f.cap = f.fits ? (int64_t)std::floor(room / f.kvb) : 0;
  return f;
}
double prefill_lat(const Perf& f, int64_t s1, int64_t s2) {
  return (f.two_p * (double)s1 + f.attn_coef * (double)s2) / f.pf_den;
}
double decode_lat(const Perf& f, int64_t batch, int64_t sum_kv) {
  double mem = (f.W + (double)sum_kv * f.kvb) / f.mem_den;
  double comp = (f.two_p * (double)batch) / f.comp_den;
  return mem > comp ? mem : comp;
}
double transfer_lat(const Perf& f, double bytes) { return bytes / f.link_bw; }

// ------------------------------------------------------------- engine (§3-6)
enum Role { DECODE = 0, PREFILL = 1 };
enum Job { NONE = 0, JOB_PREFILL = 1, JOB_STEP = 2 };

struct Req {
  double arrival = 0;
  int32_t prompt = 0, decode = 0;
  int32_t emitted = 0;
  int32_t qlen = 0;           // length of the pending (re)prefill
  int primary = -1, copy = -1;
  bool stepping = false;      // member of its primary's in-flight step (+1 reserved)
  bool settling = false;      // joined from the incoming list, no decode step here yet (§6: not movable)
  double fresh_at = 0;        // copy is complete at this time
  double last_t = 0, first_t = kNaN, done_t = kNaN, tbt_max = 0;
  double pf_start = kNaN;     // start of the job that produced the first token (queue wait)
  int32_t n_moves = 0, n_preempt = 0;
  bool done = false;
  int32_t kvo = -1;           // ft - 1: first token from the prefill (-1) or the first decode step (0)
  int64_t kv() const { return (int64_t)prompt + emitted + kvo; }
  int64_t held() const { return kv() + (stepping ? 1 : 0); }
};

struct Incoming { int rid; double ready; };

struct Inst {
  int role = DECODE;
  int job = NONE;
  double busy_until = 0, job_start = 0;
  std::vector<int> batch;
  std::vector<Incoming> incoming;
  std::vector<int> job_reqs;   // prefill admitted (splitwise/accellm) or co-batched (unified)
  int64_t job_s1 = 0;
  int64_t used = 0, peak = 0;
  double busy_time = 0;
  bool switch_pending = false;
  // idle-while-runnable: while idle with a request waiting
  // in a queue, the open interval started at irs
  double irs = 0, idle_rb = 0;
  int role0 = DECODE;
  // inter-pair leveling: KV of migrated requests still held as the source of
  // in-flight transfers, released at the first boundary >= lvl_until (§6b)
  int64_t lvl_hold = 0;
  double lvl_until = 0;
};

struct Sim {
  const kvsim_point_desc& P;
  Perf f;
  int n;
  int policy;
  int n_prefill = 0;
  int64_t budget;
  std::vector<Req> R;
  int64_t N = 0;
  // event budget (SEMANTICS §8): 4 n (dmax + 2) + 4096 with n the point's
  // request limit and dmax the configured decode maximum (a trace: its own
  // maximum over the whole trace), as the kernel computes it before any
  // request exists; -1 = derive from the simulated requests
  int64_t budget_cfg = -1;
  int64_t next_arrival = 0;
  std::vector<Inst> I;
  std::vector<std::deque<int>> Q;         // queues: unified per inst, splitwise 1, accellm per pair
  std::vector<int64_t> qtokens;
  std::vector<double> link_busy;          // n*n directed
  // counters
  int64_t n_events = 0, n_steps = 0, n_prefills = 0, n_moves = 0, n_preempt = 0, n_evict = 0;
  int64_t tokens_total = 0, tokens_window = 0, prefill_tokens = 0, mirror_tokens = 0;
  double now = 0;
  // queue depth (requests waiting in prefill queues; idle-while-runnable
  // intervals of idle instances open / close with it, SEMANTICS §7)
  int64_t qdepth = 0, qd_max = 0;
  double qd_area = 0, qd_tprev = 0;
  // detail runs: every TBT sample of a measured request (pooled percentiles)
  bool detail = false;
  std::vector<double> tbt_samples;
  // AcceLLM timer-driven extensions (SEMANTICS §6b): degraded mode
  // and inter-pair leveling (
  // PAPER.md:309). partner[x] = holder of the copies of x's primaries
  // (x^1 normally; the dual instance for a degraded group's decoders; -1 for
  // the dual instance itself).
  bool ext = false, deg_on = false, lvl_on = false;
  bool cobatch = false;  // splitwise high-load co-batching
  bool ft = false;       // first token from the first decode step (SPEC.md:273 alternative)
  double timer_P = 1.0, red_thr = 0.5, exit_fill = 0.5, lvl_frac = 0.10, dual_frac = 1.0 / 3.0;
  int trig = 3;
  int64_t tick = 1;
  std::vector<int> partner, gmode, gcnt, lvl_dst;
  std::vector<int64_t> lvl_budget;
  int64_t level_tokens = 0, n_ticks = 0, n_modes = 0;
  // event log
  kvsim_event_record* ev;
  int64_t ev_cap, ev_n = 0;
  int status = KVSIM_OK;

  Sim(const kvsim_point_desc& p, kvsim_event_record* e, int64_t ecap)
      : P(p), f(make_perf(p)), n(p.num_instances), policy(p.policy), ev(e), ev_cap(ecap) {
    budget = p.prefill_token_budget > 0 ? p.prefill_token_budget : 8192;
    I.resize(n);
    link_busy.assign((size_t)n * n, 0.0);
    if (policy == KVSIM_POLICY_UNIFIED) Q.resize(n);
    else if (policy == KVSIM_POLICY_SPLITWISE) {
      Q.resize(1);
      n_prefill = p.num_prefill_instances > 0 ? p.num_prefill_instances : (n + 2) / 4;
      for (int i = 0; i < n_prefill; ++i) I[i].role = I[i].role0 = PREFILL;
    } else Q.resize(n / 2);
    qtokens.assign(Q.size(), 0);
    cobatch = policy == KVSIM_POLICY_SPLITWISE && p.splitwise_cobatch != 0;
    ft = p.first_token_decode != 0;
    if (policy == KVSIM_POLICY_ACCELLM && (p.accellm_flags & 3)) {
      ext = true;
      deg_on = (p.accellm_flags & KVSIM_ACCELLM_DEGRADED) != 0;
      lvl_on = (p.accellm_flags & KVSIM_ACCELLM_LEVELING) != 0;
      if (p.policy_timer_s > 0) timer_P = p.policy_timer_s;
      if (p.degraded_redundancy > 0) red_thr = p.degraded_redundancy;
      if (p.degraded_exit_fill > 0) exit_fill = p.degraded_exit_fill;
      if (p.leveling_link_fraction > 0) lvl_frac = p.leveling_link_fraction;
      if (p.dual_copy_fraction > 0) dual_frac = p.dual_copy_fraction;
      if (p.degraded_trigger_ticks > 0) trig = p.degraded_trigger_ticks;
    }
    partner.resize(n);
    for (int x = 0; x < n; ++x) partner[x] = x ^ 1;
    gmode.assign((size_t)(n / 4) + 1, 0);
    gcnt.assign((size_t)(n / 4) + 1, 0);
    lvl_dst.assign(n, -1);
    lvl_budget.assign(n, 0);
  }
  // degraded-mode helpers: group of pair q (valid iff q/2 < n/4), the queue a
  // pair's requests wait in (a degraded group shares its first pair's queue)
  bool degraded_pair(int q) const { return ext && (q >> 1) < n / 4 && gmode[q >> 1]; }
  int qid(int q) const { return degraded_pair(q) ? (q & ~1) : q; }
  bool is_dual(int x) const { return degraded_pair(x >> 1) && (x & 3) == 0; }

  void log(int kind, int inst, int a, int b, int64_t c) {
    if (ev && ev_n < ev_cap) ev[ev_n] = kvsim_event_record{now, kind, inst, a, b, c};
    ++ev_n;
  }
  void bump(int i, int64_t tok) {
    I[i].used += tok;
    if (I[i].used > I[i].peak) I[i].peak = I[i].used;
  }
  int queue_of(int i) const {
    return policy == KVSIM_POLICY_UNIFIED ? i : policy == KVSIM_POLICY_SPLITWISE ? 0 : qid(i / 2);
  }
  // queue depth: area += depth * (now - previous change), then the change
  void qd_change(int64_t delta) {
    qd_area = qd_area + (double)qdepth * (now - qd_tprev);
    qd_tprev = now;
    const bool opens = qdepth == 0 && delta > 0;
    qdepth += delta;
    const bool closes = qdepth == 0;
    if (opens || closes)
      for (auto& x : I)
        if (x.job == NONE) {
          if (opens) x.irs = now;
          else x.idle_rb = x.idle_rb + (clip(now) - clip(x.irs));
        }
    if (qdepth > qd_max) qd_max = qdepth;
  }
  void push_back(int q, int rid) { Q[q].push_back(rid); qtokens[q] += R[rid].qlen; qd_change(1); }
  void push_front(int q, int rid) { Q[q].push_front(rid); qtokens[q] += R[rid].qlen; qd_change(1); }
  int pop_front(int q) { int r = Q[q].front(); Q[q].pop_front(); qtokens[q] -= R[r].qlen; qd_change(-1); return r; }
  // degraded-mode queue merge: the request stays queued (no depth change)
  int move_front(int q) { int r = Q[q].front(); Q[q].pop_front(); qtokens[q] -= R[r].qlen; return r; }
  void append_back(int q, int rid) { Q[q].push_back(rid); qtokens[q] += R[rid].qlen; }

  // ---- idle while runnable
  double clip(double t) const { return t > P.warmup_s ? t : P.warmup_s; }
  // Z(t): measure of [warmup, t] with no live request (t >= every change so far)
  // a job starts on x at t: close x's open idle-while-runnable interval
  void job_begin(Inst& X, double t) {
    if (qdepth > 0) X.idle_rb = X.idle_rb + (clip(t) - clip(X.irs));
  }

  // token emission at time t (first token, recompute token or decode token)
  void emit(Req& r, double t) {
    if (g_check_invariants && r.emitted > 0 && !(t > r.last_t)) {
      if (getenv("KVO_DEBUG")) fprintf(stderr, "time order t=%.17g last=%.17g\n", t, r.last_t);
      status = KVSIM_E_INTERNAL;  // token_times strictly increasing
    }
    if (r.emitted == 0) r.first_t = t;
    else {
      double gap = t - r.last_t;
      if (gap > r.tbt_max) r.tbt_max = gap;
      if (detail && r.arrival >= P.warmup_s) tbt_samples.push_back(gap);
    }
    r.last_t = t;
    r.emitted += 1;
    ++tokens_total;
    if (t >= P.warmup_s) ++tokens_window;
  }
  void finish_req(Req& r, double t) { r.done = true; r.done_t = t; }

  // a job ends on x at t: busy time; with a request waiting, x's
  // idle-while-runnable interval opens here
  void account_job(Inst& x, double t) {
    if (x.job_start >= P.warmup_s) x.busy_time += t - x.job_start;
    if (qdepth > 0) x.irs = t;
  }

  // ---- memory helpers (§5)
  // free everything a request holds (primary + copy)
  void free_req(int rid) {
    Req& r = R[rid];
    int64_t h = r.held();
    if (r.primary >= 0) I[r.primary].used -= h;
    if (r.copy >= 0) I[r.copy].used -= h;
  }
  // largest copy held on instance x: candidates are requests whose primary is
  // the partner (batch + incoming). Returns rid or -1.
  int largest_copy_on(int x) {
    int best = -1;
    auto consider = [&](int rid) {
      const Req& r = R[rid];
      if (r.copy != x) return;
      if (best < 0 || r.kv() > R[best].kv() || (r.kv() == R[best].kv() && rid < best)) best = rid;
    };
    // clients of x: instances whose copies x holds (partner relation)
    for (int y = 0; y < n; ++y) {
      if (y == x || partner[y] != x) continue;
      for (int rid : I[y].batch) consider(rid);
      for (auto& in : I[y].incoming) consider(in.rid);
    }
    return best;
  }
  void evict_copy(int rid) {
    Req& r = R[rid];
    int holder = r.copy;
    I[holder].used -= r.held();
    r.copy = -1;
    ++n_evict;
    log(KVSIM_EV_EVICT, holder, rid, 0, 0);
  }
  // preempt the highest-rid member of x's batch (P9, recompute)
  void preempt_newest(int x) {
    Inst& X = I[x];
    auto it = std::max_element(X.batch.begin(), X.batch.end());
    int rid = *it;
    X.batch.erase(it);
    Req& r = R[rid];
    free_req(rid);
    r.primary = -1;
    r.copy = -1;
    r.qlen = r.prompt + r.emitted;
    r.settling = false;  // leaves the batch: it rejoins through a prefill, not the incoming list (§6 settling)
    r.n_preempt += 1;
    ++n_preempt;
    log(KVSIM_EV_PREEMPT, x, rid, r.qlen, 0);
    push_front(queue_of(x), rid);
  }

  double fresh_at(int rid) const { return R[rid].fresh_at; }

  // ---- link FIFO (§5)
  double prefill_transfer(int s, int d, int64_t s1, double t_start, double t_done) {
    double& busy = link_busy[(size_t)s * n + d];
    double tail = t_done + transfer_lat(f, (double)s1 * f.kvb_layer);
    double start = t_start > busy ? t_start : busy;
    double full = start + transfer_lat(f, (double)s1 * f.kvb);
    double fin = tail > full ? tail : full;
    busy = fin;
    prefill_tokens += s1;
    log(KVSIM_EV_TRANSFER, s, d, 0, s1);
    return fin;
  }

  // ---- joins
  void join(int x, double t) {
    Inst& X = I[x];
    int cnt = 0;
    std::vector<Incoming> keep;
    for (auto& in : X.incoming) {
      if (in.ready <= t) { X.batch.push_back(in.rid); R[in.rid].settling = true; ++cnt; }
      else keep.push_back(in);
    }
    X.incoming.swap(keep);
    if (cnt) log(KVSIM_EV_JOIN, x, cnt, 0, 0);
  }

  // ---- decode step (splitwise / accellm decode instances)
  bool all_prefill_busy() const {
    for (int p = 0; p < n_prefill; ++p)
      if (I[p].job == NONE) return false;
    return true;
  }
  // splitwise with co-batching: a decode iteration also prefills queued
  // prompts while every prefill instance is busy (SEMANTICS §6)
  bool sw_overflow() const { return cobatch && !Q[0].empty() && all_prefill_busy(); }
  void step_start(int x, double t) {
    Inst& X = I[x];
    bool preempted = false;
    if (cobatch) { sw_cobatch_start(x, t); return; }
    if (X.batch.empty()) return;
    while (X.used + (int64_t)X.batch.size() > f.cap) {
      int victim = policy == KVSIM_POLICY_ACCELLM ? largest_copy_on(x) : -1;
      if (victim >= 0) evict_copy(victim);
      else { preempt_newest(x); preempted = true; if (X.batch.empty()) break; }
    }
    if (X.batch.empty()) {
      if (preempted && policy == KVSIM_POLICY_ACCELLM) ensure_prefill(qid(x / 2), t);
      return;
    }
    int64_t m = 0;
    if (policy == KVSIM_POLICY_ACCELLM && partner[x] >= 0) {
      int y = partner[x];
      for (;;) {
        m = 0;
        for (int rid : X.batch) if (R[rid].copy == y) ++m;
        if (I[y].used + m <= f.cap) break;
        int v = largest_copy_on(y);
        evict_copy(v);
      }
      bump(y, m);
    }
    int64_t B = (int64_t)X.batch.size(), K = 0;
    for (int rid : X.batch) { K += R[rid].kv(); R[rid].stepping = true; }
    bump(x, B);
    job_begin(X, t);
    X.job = JOB_STEP;
    X.job_start = t;
    X.busy_until = t + decode_lat(f, B, K);
    log(KVSIM_EV_STEP_START, x, (int)B, 0, K);
    if (preempted && policy == KVSIM_POLICY_ACCELLM) ensure_prefill(qid(x / 2), t);
  }

  void sw_cobatch_start(int x, double t) {
    Inst& X = I[x];
    if (X.batch.empty() && !sw_overflow()) return;
    while (X.used + (int64_t)X.batch.size() > f.cap) preempt_newest(x);
    int64_t B = (int64_t)X.batch.size(), K = 0;
    for (int rid : X.batch) { K += R[rid].kv(); R[rid].stepping = true; }
    bump(x, B);
    X.job_reqs.clear();
    int64_t s1 = 0, s2 = 0;
    if (sw_overflow()) {
      while (!Q[0].empty()) {
        int head = Q[0].front();
        int64_t len = R[head].qlen;
        if (!X.job_reqs.empty() && s1 + len > budget) break;
        if (X.used + len > f.cap) break;
        pop_front(0);
        bump(x, len);
        R[head].primary = x;
        if (R[head].emitted == 0) R[head].pf_start = t;
        X.job_reqs.push_back(head);
        s1 += len;
        s2 += len * len;
      }
    }
    if (B == 0 && X.job_reqs.empty()) return;
    double lat = (X.job_reqs.empty() ? 0.0 : prefill_lat(f, s1, s2)) + (B ? decode_lat(f, B, K) : 0.0);
    job_begin(X, t);
    X.job = JOB_STEP;
    X.job_start = t;
    X.busy_until = t + lat;
    log(KVSIM_EV_STEP_START, x, (int)B, (int)X.job_reqs.size(), K);
  }

  void step_end(int x, double t) {
    Inst& X = I[x];
    account_job(X, t);
    ++n_steps;
    X.job = NONE;
    int y = policy == KVSIM_POLICY_ACCELLM ? partner[x] : -1;
    int64_t m = 0;
    if (y >= 0)
      for (int rid : X.batch) if (R[rid].copy == y) ++m;
    std::vector<int> keep;
    int completed = 0;
    int B = (int)X.batch.size();
    for (int rid : X.batch) {
      Req& r = R[rid];
      emit(r, t);
      r.stepping = false;
      r.settling = false;
      if (r.emitted == r.decode) {
        // held after the step == kv() with the new emitted count
        I[x].used -= r.kv();
        if (r.copy >= 0) I[r.copy].used -= r.kv();
        finish_req(r, t);
        ++completed;
      } else {
        keep.push_back(rid);
      }
    }
    // splitwise co-batched prompts: first token, then join this batch
    for (int rid : X.job_reqs) {
      Req& r = R[rid];
      if (!ft) emit(r, t);
      if (r.emitted == r.decode) { X.used -= r.kv(); finish_req(r, t); ++completed; }
      else keep.push_back(rid);
    }
    if (!X.job_reqs.empty()) ++n_prefills;
    X.job_reqs.clear();
    X.batch.swap(keep);
    if (policy == KVSIM_POLICY_ACCELLM && m > 0) {
      double& busy = link_busy[(size_t)x * n + y];
      double start = t > busy ? t : busy;
      double fin = start + transfer_lat(f, (double)m * f.kvb);
      busy = fin;
      mirror_tokens += m;
      for (int rid : X.batch) if (R[rid].copy == y) R[rid].fresh_at = fin;
      log(KVSIM_EV_TRANSFER, x, y, 1, m);
    }
    log(KVSIM_EV_STEP_END, x, B, completed, 0);
  }

  // ---------------------------------------------------------------- unified
  void unified_start(int x, double t) {
    Inst& X = I[x];
    while (X.used + (int64_t)X.batch.size() > f.cap) preempt_newest(x);
    int64_t B = (int64_t)X.batch.size(), K = 0;
    for (int rid : X.batch) { K += R[rid].kv(); R[rid].stepping = true; }
    bump(x, B);
    X.job_reqs.clear();
    int64_t s1 = 0, s2 = 0;
    while (!Q[x].empty()) {
      int head = Q[x].front();
      int64_t len = R[head].qlen;
      if (!X.job_reqs.empty() && s1 + len > budget) break;
      if (X.used + len > f.cap) break;
      pop_front(x);
      bump(x, len);
      if (R[head].emitted == 0) R[head].pf_start = t;
      X.job_reqs.push_back(head);
      s1 += len;
      s2 += len * len;
    }
    if (B == 0 && X.job_reqs.empty()) return;
    double lat = (X.job_reqs.empty() ? 0.0 : prefill_lat(f, s1, s2)) + (B ? decode_lat(f, B, K) : 0.0);
    job_begin(X, t);
    X.job = JOB_STEP;
    X.job_start = t;
    X.busy_until = t + lat;
    log(KVSIM_EV_STEP_START, x, (int)B, (int)X.job_reqs.size(), K);
  }
  void unified_end(int x, double t) {
    Inst& X = I[x];
    account_job(X, t);
    ++n_steps;
    X.job = NONE;
    std::vector<int> keep;
    int completed = 0;
    int B = (int)X.batch.size();
    for (int rid : X.batch) {
      Req& r = R[rid];
      emit(r, t);
      r.stepping = false;
      if (r.emitted == r.decode) { X.used -= r.kv(); finish_req(r, t); ++completed; }
      else keep.push_back(rid);
    }
    for (int rid : X.job_reqs) {
      Req& r = R[rid];
      if (!ft) emit(r, t);
      if (r.emitted == r.decode) { X.used -= r.kv(); finish_req(r, t); ++completed; }
      else { r.primary = x; keep.push_back(rid); }
    }
    if (!X.job_reqs.empty()) ++n_prefills;
    X.job_reqs.clear();
    X.batch.swap(keep);
    log(KVSIM_EV_STEP_END, x, B, completed, 0);
    unified_start(x, t);
  }

  // -------------------------------------------------------------- splitwise
  void sw_try_start(double t) {
    for (int p = 0; p < n_prefill; ++p) {
      Inst& X = I[p];
      if (X.job != NONE || Q[0].empty()) continue;
      X.job_reqs.clear();
      int64_t s1 = 0, s2 = 0;
      while (!Q[0].empty()) {
        int head = Q[0].front();
        int64_t len = R[head].qlen;
        if (!X.job_reqs.empty() && s1 + len > budget) break;
        int d = -1;
        int64_t best = 0;
        for (int j = n_prefill; j < n; ++j) {
          int64_t fr = f.cap - I[j].used;
          if (d < 0 || fr > best) { d = j; best = fr; }
        }
        if (best < len) break;
        if (X.used + s1 + len > f.cap) break;  // the prefill instance holds the job's prompts
        pop_front(0);
        bump(d, len);
        R[head].primary = d;
        if (R[head].emitted == 0) R[head].pf_start = t;
        X.job_reqs.push_back(head);
        s1 += len;
        s2 += len * len;
      }
      if (X.job_reqs.empty()) continue;
      X.job_s1 = s1;
      bump(p, s1);
      job_begin(X, t);
      X.job = JOB_PREFILL;
      X.job_start = t;
      X.busy_until = t + prefill_lat(f, s1, s2);
      log(KVSIM_EV_PREFILL_START, p, (int)X.job_reqs.size(), X.job_reqs[0], s1);
    }
    if (cobatch)  // idle decode instances (ascending id) take overflow prompts
      for (int d = n_prefill; d < n && sw_overflow(); ++d)
        if (I[d].job == NONE) sw_cobatch_start(d, t);
  }
  void sw_prefill_done(int p, double t) {
    Inst& X = I[p];
    account_job(X, t);
    ++n_prefills;
    X.job = NONE;
    X.used -= X.job_s1;
    int completed = 0;
    std::vector<int64_t> per_dst(n, 0);
    for (int rid : X.job_reqs) {
      Req& r = R[rid];
      if (!ft) emit(r, t);
      if (r.emitted == r.decode) {
        I[r.primary].used -= r.kv();
        finish_req(r, t);
        ++completed;
      } else per_dst[r.primary] += r.qlen;
    }
    log(KVSIM_EV_PREFILL_DONE, p, (int)X.job_reqs.size(), completed, 0);
    for (int d = n_prefill; d < n; ++d) {
      if (per_dst[d] == 0) continue;
      double fin = prefill_transfer(p, d, per_dst[d], X.job_start, t);
      for (int rid : X.job_reqs)
        if (!R[rid].done && R[rid].primary == d) I[d].incoming.push_back({rid, fin});
    }
    X.job_reqs.clear();
  }

  // ---------------------------------------------------------------- accellm
  int64_t load_of(int x) const {
    int64_t s = 0;
    for (int rid : I[x].batch) s += R[rid].kv();
    for (auto& in : I[x].incoming) s += R[in.rid].kv();
    return s;
  }
  // head of the pair queue admissible on x after evicting every copy on x?
  bool head_admissible(int x) {
    int q = qid(x / 2);
    if (Q[q].empty()) return false;
    int64_t len = R[Q[q].front()].qlen;
    int64_t copies = 0;
    for (int y = 0; y < n; ++y) {
      if (y == x || partner[y] != x) continue;
      for (int rid : I[y].batch) if (R[rid].copy == x) copies += R[rid].held();
      for (auto& in : I[y].incoming) if (R[in.rid].copy == x) copies += R[in.rid].held();
    }
    return I[x].used - copies + len <= f.cap;
  }
  void move_req(int rid, int from, int to, double t) {
    Req& r = R[rid];
    double ready = r.fresh_at > t ? r.fresh_at : t;
    r.primary = to;
    r.copy = from;
    r.fresh_at = t;
    r.n_moves += 1;
    ++n_moves;
    I[to].incoming.push_back({rid, ready});
    log(KVSIM_EV_MOVE, from, rid, to, 0);
  }
  // move every request with primary x that holds a copy on the partner
  void move_all_to_partner(int x, double t) {
    Inst& X = I[x];
    int y = partner[x];
    if (y < 0) return;  // a degraded group's dual instance holds no movable requests
    std::vector<int> keep;
    for (int rid : X.batch) {
      if (R[rid].copy == y) move_req(rid, x, y, t);
      else keep.push_back(rid);
    }
    X.batch.swap(keep);
    std::vector<Incoming> keepin;
    for (auto& in : X.incoming) {
      if (R[in.rid].copy == y) {
        // already complete on y (old primary): ready at max(t, fresh_at)
        move_req(in.rid, x, y, t);
      } else keepin.push_back(in);
    }
    X.incoming.swap(keepin);
  }
  void acc_start_job(int x, double t) {
    Inst& X = I[x];
    int q = qid(x / 2);
    X.job_reqs.clear();
    int64_t s1 = 0, s2 = 0;
    while (!Q[q].empty()) {
      int head = Q[q].front();
      int64_t len = R[head].qlen;
      if (!X.job_reqs.empty() && s1 + len > budget) break;
      while (X.used + len > f.cap) {
        int v = largest_copy_on(x);
        if (v < 0) break;
        evict_copy(v);
      }
      if (X.used + len > f.cap) break;
      pop_front(q);
      bump(x, len);
      R[head].primary = x;
      if (R[head].emitted == 0) R[head].pf_start = t;
      X.job_reqs.push_back(head);
      s1 += len;
      s2 += len * len;
    }
    X.job_s1 = s1;
    job_begin(X, t);
    X.job = JOB_PREFILL;
    X.job_start = t;
    X.busy_until = t + prefill_lat(f, s1, s2);
    log(KVSIM_EV_PREFILL_START, x, (int)X.job_reqs.size(), X.job_reqs.empty() ? -1 : X.job_reqs[0], s1);
  }
  bool try_switch(int x, double t) {
    if (!head_admissible(x)) return false;
    Inst& X = I[x];
    X.switch_pending = false;
    move_all_to_partner(x, t);
    X.role = PREFILL;
    log(KVSIM_EV_ROLE, x, PREFILL, 0, 0);
    acc_start_job(x, t);
    return true;
  }
  void ensure_prefill(int q, double t) {
    if (Q[q].empty()) return;
    if (degraded_pair(q)) {  // the dual instance is the group's only prefill instance
      int d = 4 * (q >> 1);
      if (I[d].role == PREFILL || I[d].switch_pending) return;
      if (I[d].job == NONE) try_switch(d, t);
      else I[d].switch_pending = true;
      return;
    }
    int a = 2 * q, b = a + 1;
    if (I[a].role == PREFILL || I[b].role == PREFILL || I[a].switch_pending || I[b].switch_pending) return;
    int m = load_of(b) < load_of(a) ? b : a;
    if (I[m].job == NONE) try_switch(m, t);
    else I[m].switch_pending = true;
  }
  void rebalance(int x, double t) {
    if (ext && degraded_pair(x / 2)) { if (!is_dual(x)) dual_push(x, t); return; }
    int y = x ^ 1;
    Inst& X = I[x];
    Inst& Y = I[y];
    if (Y.role != DECODE || Y.switch_pending) return;
    int64_t c = (int64_t)X.batch.size() + (int64_t)X.incoming.size() - (int64_t)Y.batch.size() -
                (int64_t)Y.incoming.size();
    int64_t d = load_of(x) - load_of(y);
    std::vector<int> cand;
    for (int rid : X.batch) if (R[rid].copy == y && !R[rid].settling) cand.push_back(rid);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
      if (R[a].kv() != R[b].kv()) return R[a].kv() > R[b].kv();
      return a < b;
    });
    std::vector<int> moved;
    for (int rid : cand) {
      int64_t k = R[rid].kv();
      int64_t v = std::max<int64_t>(0, std::llabs(c) - 1), D = std::llabs(d);
      int64_t c2 = c - 2, d2 = d - 2 * k;
      int64_t v2 = std::max<int64_t>(0, std::llabs(c2) - 1), D2 = std::llabs(d2);
      if (v2 <= v && D2 <= D && (v2 < v || D2 < D)) {
        moved.push_back(rid);
        c = c2;
        d = d2;
      }
    }
    if (moved.empty()) return;
    std::vector<int> keep;
    for (int rid : X.batch)
      if (std::find(moved.begin(), moved.end(), rid) == moved.end()) keep.push_back(rid);
    X.batch.swap(keep);
    for (int rid : moved) move_req(rid, x, y, t);
  }
  void acc_boundary(int x, double t) {
    Inst& X = I[x];
    if (X.lvl_hold > 0 && t >= X.lvl_until) { X.used -= X.lvl_hold; X.lvl_hold = 0; }
    join(x, t);
    if (X.switch_pending) {
      X.switch_pending = false;
      if (try_switch(x, t)) return;
    }
    ensure_prefill(qid(x / 2), t);
    if (X.role == PREFILL) return;  // ensure_prefill switched x
    if (lvl_dst[x] >= 0) level_from(x, t);
    rebalance(x, t);
    step_start(x, t);
  }
  void acc_prefill_done(int x, double t) {
    Inst& X = I[x];
    account_job(X, t);
    ++n_prefills;
    X.job = NONE;
    int y = x ^ 1;
    int completed = 0;
    std::vector<int> survivors;
    for (int rid : X.job_reqs) {
      Req& r = R[rid];
      if (!ft) emit(r, t);
      if (r.emitted == r.decode) {
        X.used -= r.kv();
        finish_req(r, t);
        ++completed;
      } else survivors.push_back(rid);
    }
    log(KVSIM_EV_PREFILL_DONE, x, (int)X.job_reqs.size(), completed, 0);
    if (is_dual(x)) {
      dual_handoff(x, survivors, t);
      X.job_reqs.clear();
      if (head_admissible(x)) { acc_start_job(x, t); return; }
      X.role = DECODE;
      log(KVSIM_EV_ROLE, x, DECODE, 0, 0);
      acc_boundary(x, t);
      return;
    }
    int64_t s1c = 0;
    int ncopy = 0;
    for (int rid : survivors) {
      Req& r = R[rid];
      if (I[y].used + r.kv() <= f.cap) {
        bump(y, r.kv());
        r.copy = y;
        s1c += r.kv();
        ++ncopy;
      }
    }
    if (ncopy) log(KVSIM_EV_COPY, y, ncopy, 0, s1c);
    if (s1c > 0) {
      double fin = prefill_transfer(x, y, s1c, X.job_start, t);
      for (int rid : survivors) if (R[rid].copy == y) R[rid].fresh_at = fin;
    }
    for (int rid : survivors) X.batch.push_back(rid);
    X.job_reqs.clear();
    if (head_admissible(x)) {
      move_all_to_partner(x, t);
      acc_start_job(x, t);
      return;
    }
    X.role = DECODE;
    log(KVSIM_EV_ROLE, x, DECODE, 0, 0);
    acc_boundary(x, t);
  }

  // ------------------------------------------- degraded mode (SEMANTICS §6b)
  // tokens of decoder x's requests that the dual instance d holds as copies
  int64_t dual_copy_tokens(int d, int x) const {
    int64_t s = 0;
    for (int rid : I[x].batch) if (R[rid].copy == d) s += R[rid].held();
    for (auto& in : I[x].incoming) if (R[in.rid].copy == d) s += R[in.rid].held();
    return s;
  }
  // prefill survivors of the dual instance d go to the decoder with the most
  // free tokens (full KV transfer, one per destination); d keeps its
  // computed KV as the redundant copy while that decoder's copy budget
  // (dual_copy_fraction x capacity) allows ("retains about
  // one-third of the KV caches of each decoding instance").
  void dual_handoff(int d, const std::vector<int>& survivors, double t) {
    Inst& D = I[d];
    const int64_t budget = (int64_t)(dual_frac * (double)f.cap);
    int64_t ct[3];
    for (int k = 0; k < 3; ++k) ct[k] = dual_copy_tokens(d, d + 1 + k);
    int64_t per_dst[3] = {0, 0, 0}, s1c = 0;
    int ncopy = 0;
    std::vector<int> stay;
    for (int rid : survivors) {
      Req& r = R[rid];
      const int64_t kv = r.kv();
      int best = -1;
      int64_t bf = 0;
      for (int k = 0; k < 3; ++k) {
        int64_t fr = f.cap - I[d + 1 + k].used;
        if (best < 0 || fr > bf) { best = k; bf = fr; }
      }
      if (bf < kv) { stay.push_back(rid); continue; }  // no decoder has room: decodes on d
      const int xk = d + 1 + best;
      bump(xk, kv);
      r.primary = xk;
      per_dst[best] += kv;
      if (ct[best] + kv <= budget) {
        r.copy = d;
        r.fresh_at = t;
        ct[best] += kv;
        s1c += kv;
        ++ncopy;
      } else {
        r.copy = -1;
        D.used -= kv;
      }
    }
    if (ncopy) log(KVSIM_EV_COPY, d, ncopy, 1, s1c);
    for (int k = 0; k < 3; ++k) {
      if (per_dst[k] == 0) continue;
      const int xk = d + 1 + k;
      double fin = prefill_transfer(d, xk, per_dst[k], D.job_start, t);
      for (int rid : survivors)
        if (R[rid].primary == xk) I[xk].incoming.push_back({rid, fin});
    }
    for (int rid : stay) D.batch.push_back(rid);
  }
  // at decoder x's boundary: hand requests whose copy the dual instance holds
  // over to it (zero bytes; x drops its KV, "overwrite") while
  // no prefill is pending, with rebalance_pair's greedy
  void dual_push(int x, double t) {
    const int d = x & ~3;
    Inst& X = I[x];
    Inst& D = I[d];
    if (D.role != DECODE || D.switch_pending || !Q[qid(x / 2)].empty()) return;
    int64_t c = (int64_t)X.batch.size() + (int64_t)X.incoming.size() - (int64_t)D.batch.size() -
                (int64_t)D.incoming.size();
    int64_t dd = load_of(x) - load_of(d);
    std::vector<int> cand;
    for (int rid : X.batch) if (R[rid].copy == d && !R[rid].settling) cand.push_back(rid);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
      if (R[a].kv() != R[b].kv()) return R[a].kv() > R[b].kv();
      return a < b;
    });
    std::vector<int> moved;
    for (int rid : cand) {
      int64_t k = R[rid].kv();
      int64_t v = std::max<int64_t>(0, std::llabs(c) - 1), Dv = std::llabs(dd);
      int64_t c2 = c - 2, d2 = dd - 2 * k;
      int64_t v2 = std::max<int64_t>(0, std::llabs(c2) - 1), D2 = std::llabs(d2);
      if (v2 <= v && D2 <= Dv && (v2 < v || D2 < Dv)) { moved.push_back(rid); c = c2; dd = d2; }
    }
    if (moved.empty()) return;
    std::vector<int> keep;
    for (int rid : X.batch)
      if (std::find(moved.begin(), moved.end(), rid) == moved.end()) keep.push_back(rid);
    X.batch.swap(keep);
    for (int rid : moved) {
      Req& r = R[rid];
      double ready = r.fresh_at > t ? r.fresh_at : t;
      X.used -= r.held();
      r.primary = d;
      r.copy = -1;
      r.n_moves += 1;
      ++n_moves;
      D.incoming.push_back({rid, ready});
      log(KVSIM_EV_MOVE, x, rid, d, 0);
    }
  }
  // evict the copies instance h holds for the instances in [lo, hi]
  void evict_copies_from(int h, int lo, int hi) {
    for (;;) {
      int best = -1;
      for (int y = lo; y <= hi; ++y) {
        if (y == h) continue;
        auto consider = [&](int rid) {
          const Req& r = R[rid];
          if (r.copy != h) return;
          if (best < 0 || r.kv() > R[best].kv() || (r.kv() == R[best].kv() && rid < best)) best = rid;
        };
        for (int rid : I[y].batch) consider(rid);
        for (auto& in : I[y].incoming) consider(in.rid);
      }
      if (best < 0) return;
      evict_copy(best);
    }
  }
  void enter_degraded(int g, double t) {
    const int a = 4 * g;
    // the decoders overwrite the redundant copies they hold
    for (int h = a + 1; h <= a + 3; ++h) evict_copies_from(h, a, a + 3);
    partner[a] = -1;
    for (int h = a + 1; h <= a + 3; ++h) partner[h] = a;
    gmode[g] = 1;
    ++n_modes;
    while (!Q[2 * g + 1].empty()) append_back(2 * g, move_front(2 * g + 1));
    log(KVSIM_EV_MODE, g, 1, 0, 0);
    ensure_prefill(2 * g, t);
  }
  void leave_degraded(int g, double t) {
    const int a = 4 * g;
    evict_copies_from(a, a + 2, a + 3);  // pairs are restored: copies live on partners only
    for (int h = a; h <= a + 3; ++h) partner[h] = h ^ 1;
    gmode[g] = 0;
    ++n_modes;
    log(KVSIM_EV_MODE, g, 0, 0, 0);
    ensure_prefill(2 * g, t);
    ensure_prefill(2 * g + 1, t);
  }
  // ------------------------------------- inter-pair leveling (SEMANTICS §6b)
  int64_t pair_load(int q) const { return load_of(2 * q) + load_of(2 * q + 1); }
  void schedule_leveling() {
    int A = -1, B = -1;
    int64_t la = 0, lb = 0;
    for (int q = 0; q < n / 2; ++q) {
      if (degraded_pair(q) || !Q[q].empty()) continue;
      const Inst &u = I[2 * q], &v = I[2 * q + 1];
      if (u.role != DECODE || v.role != DECODE || u.switch_pending || v.switch_pending) continue;
      const int64_t l = pair_load(q);
      if (A < 0 || l > la) { A = q; la = l; }
      if (B < 0 || l < lb) { B = q; lb = l; }
    }
    if (A < 0 || A == B || la - lb < 2) return;
    const int x = load_of(2 * A + 1) > load_of(2 * A) ? 2 * A + 1 : 2 * A;
    const int y = (f.cap - I[2 * B + 1].used) > (f.cap - I[2 * B].used) ? 2 * B + 1 : 2 * B;
    lvl_dst[x] = y;
    lvl_budget[x] = (int64_t)std::floor(((lvl_frac * f.link_bw) * timer_P) / f.kvb);
  }
  // at x's boundary: migrate batch members (largest first) to the lighter
  // pair while each move strictly narrows the pair-load gap, within the
  // per-period link budget and the destination's memory
  void level_from(int x, double t) {
    const int y = lvl_dst[x];
    int64_t bud = lvl_budget[x];
    lvl_dst[x] = -1;
    Inst& X = I[x];
    Inst& Y = I[y];
    if (Y.role != DECODE || Y.switch_pending || degraded_pair(x / 2) || degraded_pair(y / 2)) return;
    int64_t d = pair_load(x / 2) - pair_load(y / 2);
    std::vector<int> cand;
    for (int rid : X.batch) if (!R[rid].settling) cand.push_back(rid);
    std::sort(cand.begin(), cand.end(), [&](int a, int b) {
      if (R[a].kv() != R[b].kv()) return R[a].kv() > R[b].kv();
      return a < b;
    });
    std::vector<int> moved;
    for (int rid : cand) {
      const int64_t k = R[rid].kv();
      if (!(k < d) || k > bud || Y.used + k > f.cap) continue;
      moved.push_back(rid);
      bump(y, k);
      d -= 2 * k;
      bud -= k;
    }
    if (moved.empty()) return;
    std::vector<int> keep;
    for (int rid : X.batch)
      if (std::find(moved.begin(), moved.end(), rid) == moved.end()) keep.push_back(rid);
    X.batch.swap(keep);
    for (int rid : moved) {
      Req& r = R[rid];
      const int64_t k = r.kv();
      if (r.copy >= 0) I[r.copy].used -= k;
      r.copy = -1;
      r.primary = y;
      double& busy = link_busy[(size_t)x * n + y];
      double start = t > busy ? t : busy;
      double fin = start + transfer_lat(f, (double)k * f.kvb);
      busy = fin;
      // x stays the source of the transfer: it holds the KV until it is done
      X.lvl_hold += k;
      if (fin > X.lvl_until) X.lvl_until = fin;
      level_tokens += k;
      r.n_moves += 1;
      ++n_moves;
      Y.incoming.push_back({rid, fin});
      log(KVSIM_EV_LEVEL, x, rid, y, k);
    }
  }
  void on_timer(double t) {
    ++n_ticks;
    log(KVSIM_EV_TIMER, -1, (int)(tick - 1), 0, 0);
    if (deg_on) {
      for (int g = 0; g < n / 4; ++g) {
        const int a = 4 * g;
        bool pf = false;
        for (int h = a; h <= a + 3; ++h) pf = pf || I[h].role == PREFILL || I[h].switch_pending;
        if (!gmode[g]) {
          int64_t live = 0, red = 0;
          for (int h = a; h <= a + 3; ++h) {
            live += (int64_t)I[h].batch.size() + (int64_t)I[h].incoming.size();
            for (int rid : I[h].batch) if (R[rid].copy >= 0) ++red;
            for (auto& in : I[h].incoming) if (R[in.rid].copy >= 0) ++red;
          }
          gcnt[g] = (live > 0 && (double)red < red_thr * (double)live) ? gcnt[g] + 1 : 0;
          if (gcnt[g] >= trig && !pf) { gcnt[g] = 0; enter_degraded(g, t); }
        } else {
          int64_t u = 0;
          for (int h = a; h <= a + 3; ++h) u += I[h].used;
          gcnt[g] = ((double)u <= exit_fill * (4.0 * (double)f.cap)) ? gcnt[g] + 1 : 0;
          if (gcnt[g] >= trig && !pf) { gcnt[g] = 0; leave_degraded(g, t); }
        }
      }
    }
    if (lvl_on) schedule_leveling();
  }

  // ---------------------------------------------------------------- arrival
  void arrive(int rid, double t) {
    Req& r = R[rid];
    r.qlen = r.prompt;
    if (policy == KVSIM_POLICY_UNIFIED) {
      int best = 0;
      int64_t bf = 0;
      for (int i = 0; i < n; ++i) {
        int64_t fr = f.cap - I[i].used - qtokens[i];
        if (i == 0 || fr > bf) { best = i; bf = fr; }
      }
      log(KVSIM_EV_ARRIVE, best, rid, r.prompt, 0);
      push_back(best, rid);
      if (I[best].job == NONE) unified_start(best, t);
    } else if (policy == KVSIM_POLICY_SPLITWISE) {
      log(KVSIM_EV_ARRIVE, 0, rid, r.prompt, 0);
      push_back(0, rid);
    } else {
      int best = -1;
      int64_t bf = 0;
      for (int q = 0; q < n / 2; ++q) {
        int64_t fr;
        if (degraded_pair(q)) {  // a degraded group is one routing unit (its first pair's queue)
          if (q & 1) continue;
          fr = 0;
          for (int h = 2 * q; h < 2 * q + 4; ++h) fr += f.cap - I[h].used;
          fr -= qtokens[q];
        } else {
          fr = (f.cap - I[2 * q].used) + (f.cap - I[2 * q + 1].used) - qtokens[q];
        }
        if (best < 0 || fr > bf) { best = q; bf = fr; }
      }
      log(KVSIM_EV_ARRIVE, best, rid, r.prompt, 0);
      push_back(best, rid);
      ensure_prefill(best, t);
    }
  }

  // ------------------------------------------------------------- main loop
  void run() {
    int64_t dmax = 1;
    for (int64_t i = 0; i < N; ++i) dmax = std::max<int64_t>(dmax, R[i].decode);
    int64_t budget_events = budget_cfg >= 0 ? budget_cfg : 4 * N * (dmax + 2) + 4096;
    for (;;) {
      double bt = kInf;
      int bk = 9, bid = 0;
      auto cand = [&](double t, int k, int id) {
        if (t < bt || (t == bt && (k < bk || (k == bk && id < bid)))) { bt = t; bk = k; bid = id; }
      };
      if (next_arrival < N) cand(R[next_arrival].arrival, 0, (int)next_arrival);
      for (int i = 0; i < n; ++i) {
        const Inst& X = I[i];
        if (X.job != NONE) cand(X.busy_until, X.job == JOB_PREFILL ? 2 : 3, i);
        else if (X.role == DECODE && !X.incoming.empty()) {
          double mr = kInf;
          for (auto& in : X.incoming) mr = std::min(mr, in.ready);
          cand(mr, 1, i);
        }
      }
      if (bk == 9) break;
      if (ext) {  // policy timer: kind 4, after every other kind at equal time
        const double tt = (double)tick * timer_P;
        if (tt < bt) {
          if (++n_events > budget_events) { status = KVSIM_E_EVENT_BUDGET; break; }
          now = tt;
          ++tick;
          on_timer(tt);
          if (g_check_invariants && !invariants_hold()) { status = KVSIM_E_INTERNAL; break; }
          continue;
        }
      }
      if (++n_events > budget_events) { status = KVSIM_E_EVENT_BUDGET; break; }
      now = bt;
      double t = bt;
      switch (bk) {
        case 0:
          ++next_arrival;
          arrive(bid, t);
          break;
        case 1:
          log(KVSIM_EV_WAKE, bid, 0, 0, 0);
          if (policy == KVSIM_POLICY_ACCELLM) acc_boundary(bid, t);
          else { join(bid, t); step_start(bid, t); }
          break;
        case 2:
          if (policy == KVSIM_POLICY_SPLITWISE) sw_prefill_done(bid, t);
          else acc_prefill_done(bid, t);
          break;
        case 3:
          if (policy == KVSIM_POLICY_UNIFIED) unified_end(bid, t);
          else {
            step_end(bid, t);
            if (policy == KVSIM_POLICY_ACCELLM) acc_boundary(bid, t);
            else { join(bid, t); step_start(bid, t); }
          }
          break;
      }
      if (policy == KVSIM_POLICY_SPLITWISE) sw_try_start(t);
      if (g_check_invariants && !invariants_hold()) { status = KVSIM_E_INTERNAL; break; }
      if (status == KVSIM_E_INTERNAL) break;
    }
  }

  // Ledger exactness and memory safety: every instance's
  // `used` equals the tokens its primaries, copies and transient prefill
  // reservations hold, and never exceeds capacity; redundant copies live on
  // the partner only (AcceLLM); emitted <= decode_len.
  bool invariants_hold() const {
    std::vector<int64_t> sum((size_t)n, 0);
    std::vector<char> in_job((size_t)next_arrival, 0);
    for (int x = 0; x < n; ++x)
      for (int rid : I[x].job_reqs) in_job[rid] = 1;
    for (int64_t i = 0; i < next_arrival; ++i) {
      const Req& r = R[i];
      if (r.emitted > r.decode) {
        if (getenv("KVO_DEBUG")) fprintf(stderr, "emitted>decode rid=%lld\n", (long long)i);
        return false;
      }
      if (r.done || r.primary < 0 || in_job[i]) continue;  // job members: reserved below
      sum[r.primary] += r.held();
      if (r.copy >= 0) {
        if (policy != KVSIM_POLICY_ACCELLM || r.copy != partner[r.primary]) return false;
        sum[r.copy] += r.held();
      }
    }
    for (int x = 0; x < n; ++x) {
      const Inst& X = I[x];
      for (int rid : X.job_reqs) {
        const Req& r = R[rid];
        if (policy == KVSIM_POLICY_SPLITWISE) { sum[r.primary] += r.qlen; }
        else sum[x] += r.qlen;
      }
      if (policy == KVSIM_POLICY_SPLITWISE && X.job != NONE && x < n_prefill) sum[x] += X.job_s1;
      sum[x] += X.lvl_hold;
    }
    for (int x = 0; x < n; ++x) {
      if (sum[x] != I[x].used) {
        if (getenv("KVO_DEBUG")) fprintf(stderr, "ledger x=%d sum=%lld used=%lld t=%.9g policy=%d\n", x, (long long)sum[x], (long long)I[x].used, now, policy);
        return false;
      }
      if (I[x].used > f.cap || I[x].used < 0) {
        if (getenv("KVO_DEBUG")) fprintf(stderr, "capacity x=%d used=%lld cap=%lld t=%.9g\n", x, (long long)I[x].used, (long long)f.cap, now);
        return false;
      }
    }
    return true;
  }
};

int check_point(const kvsim_point_desc& p) {
  if (p.num_instances < 1 || p.num_instances > KVSIM_MAX_INSTANCES) return KVSIM_E_INVALID;
  if (p.policy == KVSIM_POLICY_ACCELLM && (p.num_instances % 2)) return KVSIM_E_ODD_INSTANCES;
  if (p.policy == KVSIM_POLICY_SPLITWISE) {
    int np = p.num_prefill_instances > 0 ? p.num_prefill_instances : (p.num_instances + 2) / 4;
    if (p.num_instances < 2 || np >= p.num_instances) return KVSIM_E_INVALID;
  }
  if (p.policy < 0 || p.policy > 2) return KVSIM_E_INVALID;
  if (!make_perf(p).fits) return KVSIM_E_MODEL_FIT;
  return KVSIM_OK;
}

int64_t gen_trace(const kvsim_point_desc& p, double* arr, int32_t* pr, int32_t* de, int64_t cap) {
  if (!(p.rate > 0.0)) return 0;
  int64_t lim = std::min<int64_t>(cap, p.num_requests);
  double t = 0.0;
  int64_t i = 0;
  for (; i < lim; ++i) {
    if (p.arrival_process == KVSIM_ARRIVAL_FIXED) t = (double)i / p.rate;
    else {
      uint64_t x = draw(p.seed, i, 2);
      double u = (double)((x >> 11) + 1) * 0x1.0p-53;
      double gap = -klog(u) / p.rate;
      t = i == 0 ? gap : t + gap;
    }
    if (!(t < p.duration_s)) break;
    arr[i] = t;
    pr[i] = uniform_int(draw(p.seed, i, 0), p.prompt_min, p.prompt_max);
    de[i] = uniform_int(draw(p.seed, i, 1), p.decode_min, p.decode_max);
  }
  return i;
}

int64_t nearest_rank(int64_t n, int pct) { return (pct * n + 99) / 100 - 1; }

void summarize(Sim& S, kvsim_point_summary* out, kvsim_request_record* recs, kvsim_instance_record* inst) {
  const kvsim_point_desc& p = S.P;
  std::memset(out, 0, sizeof(*out));
  // instances idle at the end while requests wait (only a failed point):
  // their open interval closes at the makespan
  for (auto& x : S.I)
    if (x.job == NONE && S.qdepth > 0) x.idle_rb = x.idle_rb + (S.clip(S.now) - S.clip(x.irs));
  if (inst) {
    for (int i = 0; i < S.n; ++i)
      inst[i] = kvsim_instance_record{S.I[i].busy_time, S.I[i].idle_rb, S.I[i].peak, S.I[i].role0, 0};
  }
  out->status = S.status;
  out->num_instances = S.n;
  out->user_tag = p.user_tag;
  out->n_requests = S.N;
  out->n_events = S.n_events;
  out->n_steps = S.n_steps;
  out->n_prefills = S.n_prefills;
  out->n_moves = S.n_moves;
  out->n_preemptions = S.n_preempt;
  out->n_evictions = S.n_evict;
  out->tokens_total = S.tokens_total;
  out->tokens_window = S.tokens_window;
  out->link_prefill_tokens = S.prefill_tokens;
  out->link_mirror_tokens = S.mirror_tokens;
  out->link_leveling_tokens = S.level_tokens;
  out->n_timer_ticks = S.n_ticks;
  out->n_mode_switches = S.n_modes;
  out->makespan_s = S.now;
  int64_t peak = 0;
  double busy = 0;
  for (auto& x : S.I) { peak = std::max(peak, x.peak); busy += x.busy_time; }
  out->peak_kv_tokens = peak;
  out->busy_s_total = busy;
  out->peak_kv_gb = (double)peak * S.f.kvb / 1e9;
  out->link_prefill_gb = (double)S.prefill_tokens * S.f.kvb / 1e9;
  out->link_mirror_gb = (double)S.mirror_tokens * S.f.kvb / 1e9;
  std::vector<double> ttft, jct;
  double s_ttft = 0, s_jct = 0, s_tbt = 0, tbt_max = 0, s_qw = 0;
  int64_t n_tbt = 0, completed = 0;
  for (int64_t i = 0; i < S.N; ++i) {
    const Req& r = S.R[i];
    if (recs) {
      recs[i] = kvsim_request_record{r.arrival, r.first_t, r.done_t, r.tbt_max, r.prompt, r.decode,
                                     r.n_moves, r.n_preempt, r.pf_start};
    }
    if (!r.done) continue;
    ++completed;
    if (r.arrival < p.warmup_s) continue;
    double a = r.first_t - r.arrival, b = r.done_t - r.arrival;
    ttft.push_back(a);
    jct.push_back(b);
    s_ttft += a;
    s_jct += b;
    s_qw += r.pf_start - r.arrival;
    if (r.decode > 1) {
      s_tbt += r.done_t - r.first_t;
      n_tbt += r.decode - 1;
      if (r.tbt_max > tbt_max) tbt_max = r.tbt_max;
    }
  }
  out->n_completed = completed;
  int64_t m = (int64_t)ttft.size();
  out->n_measured = m;
  if (m > 0) {
    out->ttft_mean = s_ttft / (double)m;
    out->jct_mean = s_jct / (double)m;
    std::sort(ttft.begin(), ttft.end());
    std::sort(jct.begin(), jct.end());
    out->ttft_p50 = ttft[nearest_rank(m, 50)];
    out->ttft_p95 = ttft[nearest_rank(m, 95)];
    out->ttft_max = ttft[m - 1];
    out->jct_p50 = jct[nearest_rank(m, 50)];
    out->jct_p95 = jct[nearest_rank(m, 95)];
    out->jct_max = jct[m - 1];
  } else {
    out->ttft_mean = out->jct_mean = out->ttft_p50 = out->ttft_p95 = out->ttft_max = kNaN;
    out->jct_p50 = out->jct_p95 = out->jct_max = kNaN;
  }
  out->tbt_mean = n_tbt > 0 ? s_tbt / (double)n_tbt : kNaN;
  out->tbt_max = n_tbt > 0 ? tbt_max : kNaN;
  out->n_tbt_samples = n_tbt;
  out->ttft_queue_mean = m > 0 ? s_qw / (double)m : kNaN;
  out->tbt_p50 = out->tbt_p95 = kNaN;
  if (S.detail && n_tbt > 0 && (int64_t)S.tbt_samples.size() == n_tbt) {
    std::vector<double>& v = S.tbt_samples;
    std::nth_element(v.begin(), v.begin() + nearest_rank(n_tbt, 50), v.end());
    out->tbt_p50 = v[nearest_rank(n_tbt, 50)];
    std::nth_element(v.begin(), v.begin() + nearest_rank(n_tbt, 95), v.end());
    out->tbt_p95 = v[nearest_rank(n_tbt, 95)];
  }
  double irb = 0;
  for (auto& x : S.I) irb += x.idle_rb;
  out->idle_runnable_s = irb;
  out->queue_depth_max = S.qd_max;
  {
    double area = S.qd_area + (double)S.qdepth * (S.now - S.qd_tprev);
    out->queue_depth_avg = S.now > 0 ? area / S.now : kNaN;
  }
  double window = S.now - p.warmup_s;
  if (window > 0) {
    out->cost_eff = (double)S.tokens_window / (window * (double)S.n);
    out->idle_frac = 1.0 - busy / ((double)S.n * window);
  } else {
    out->cost_eff = out->idle_frac = kNaN;
  }
}

}  // namespace

extern "C" {

uint64_t kvo_rng_draw(uint64_t seed, int64_t i, int stream) { return draw(seed, i, stream); }
void kvo_set_invariant_checks(int on) { g_check_invariants = on; }
double kvo_klog(double x) { return klog(x); }
double kvo_kv_bytes_per_token(const kvsim_point_desc* p) { return make_perf(*p).kvb; }
double kvo_weight_bytes(const kvsim_point_desc* p) { return make_perf(*p).W; }
double kvo_prefill_latency(const kvsim_point_desc* p, int64_t s1, int64_t s2) {
  return prefill_lat(make_perf(*p), s1, s2);
}
double kvo_decode_step_latency(const kvsim_point_desc* p, int64_t b, int64_t k) {
  return decode_lat(make_perf(*p), b, k);
}
double kvo_transfer_latency(const kvsim_point_desc* p, double bytes) {
  return transfer_lat(make_perf(*p), bytes);
}
int kvo_kv_capacity_tokens(const kvsim_point_desc* p, int64_t* out) {
  Perf f = make_perf(*p);
  *out = f.cap;
  return f.fits ? KVSIM_OK : KVSIM_E_MODEL_FIT;
}
int64_t kvo_gen_trace(const kvsim_point_desc* p, double* a, int32_t* pr, int32_t* de, int64_t cap) {
  return gen_trace(*p, a, pr, de, cap);
}

int kvo_run_point_ex(const kvsim_point_desc* p, const kvsim_trace_view* trace, kvsim_point_summary* out,
                     kvsim_request_record* recs, kvsim_event_record* ev, int64_t ev_cap, int64_t* ev_count,
                     kvsim_instance_record* inst, int detail) {
  int st = check_point(*p);
  if (st != KVSIM_OK) {
    std::memset(out, 0, sizeof(*out));
    out->status = st;
    out->user_tag = p->user_tag;
    if (ev_count) *ev_count = 0;
    return st;
  }
  Sim S(*p, ev, ev_cap);
  S.detail = detail != 0;
  int64_t N;
  std::vector<double> arr;
  std::vector<int32_t> pr, de;
  if (trace) {
    N = std::min<int64_t>(trace->n, p->num_requests);
    arr.assign(trace->arrival_s, trace->arrival_s + N);
    pr.assign(trace->prompt_len, trace->prompt_len + N);
    de.assign(trace->decode_len, trace->decode_len + N);
  } else {
    arr.resize(p->num_requests);
    pr.resize(p->num_requests);
    de.resize(p->num_requests);
    N = gen_trace(*p, arr.data(), pr.data(), de.data(), p->num_requests);
  }
  S.N = N;
  {
    int64_t bn, bd;
    if (trace) {
      bn = std::min<int64_t>(trace->n, p->num_requests);
      bd = 1;
      for (int64_t i = 0; i < trace->n; ++i) bd = std::max<int64_t>(bd, trace->decode_len[i]);
    } else {
      bn = p->rate > 0.0 ? p->num_requests : 0;
      bd = p->decode_max > 1 ? p->decode_max : 1;
    }
    S.budget_cfg = 4 * bn * (bd + 2) + 4096;
  }
  S.R.resize(N);
  for (int64_t i = 0; i < N; ++i) {
    S.R[i].arrival = arr[i];
    S.R[i].prompt = pr[i];
    S.R[i].decode = de[i];
    S.R[i].kvo = p->first_token_decode ? 0 : -1;
  }
  S.run();
  summarize(S, out, recs, inst);
  if (ev_count) *ev_count = S.ev_n;
  return S.status;
}

int kvo_run_point(const kvsim_point_desc* p, const kvsim_trace_view* trace, kvsim_point_summary* out,
                  kvsim_request_record* recs, kvsim_event_record* ev, int64_t ev_cap, int64_t* ev_count) {
  return kvo_run_point_ex(p, trace, out, recs, ev, ev_cap, ev_count, nullptr, 0);
}

int kvo_run_sweep_ex(const kvsim_point_desc* pts, int64_t n, int threads, kvsim_point_summary* out,
                     kvsim_instance_record* inst, int detail) {
  if (threads < 1) threads = 1;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      kvo_run_point_ex(&pts[i], nullptr, &out[i], nullptr, nullptr, 0, nullptr,
                       inst ? inst + i * KVSIM_MAX_INSTANCES : nullptr, detail);
    }
  };
  std::vector<std::thread> pool;
  for (int k = 0; k < threads; ++k) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  return KVSIM_OK;
}

int kvo_run_sweep(const kvsim_point_desc* pts, int64_t n, int threads, kvsim_point_summary* out) {
  if (threads < 1) threads = 1;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t i = next.fetch_add(1);
      if (i >= n) break;
      kvo_run_point(&pts[i], nullptr, &out[i], nullptr, nullptr, 0, nullptr);
    }
  };
  std::vector<std::thread> pool;
  for (int k = 0; k < threads; ++k) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  return KVSIM_OK;
}

}  // extern "C"
