// kvsim_sim.cuh — warp-per-point discrete-event simulation core (kernel K3).
//
// One warp simulates one sweep point (one reference `run()`).
// Lane x owns instance x's scalar state in registers (busy time, ledger,
// batch counters); lane q also owns queue q. All control flow is
// warp-uniform: every lane executes the same event handler and reads other
// lanes' state with shuffles. Data-parallel work — advancing every request of
// a decode batch, joins, moves, admission scans, argmax
// searches for eviction / preemption / rebalancing —
// runs across the 32 lanes over SoA arrays in the per-warp HBM arena with
// coalesced accesses.
//
// Semantics: docs/SEMANTICS.md (identical decisions to the CPU oracle, which
// is written independently with per-request structs and std::vector
// batches). The code compiles both for sm_100a and, with KVSIM_EMU, for the
// host SIMT emulator used by the CPU test-suite.
#pragma once
#include <new>

#include "kvsim_gpu.h"
#include "kvsim_math.cuh"
#include "kvsim_simt.cuh"

#if !defined(KVSIM_EMU)
// dynamic shared memory: one WarpScratch per warp of the block
extern __shared__ __align__(16) unsigned char kvsim_smem[];
#endif

namespace kvsim_dev {
using namespace kvsim_math;

#if defined(KVSIM_EMU) && defined(KVSIM_EMU_PROFILE)
// emulator-only call counters (tests/emu profiling of the event mix)
inline long long emu_prof[32];
#define EMU_COUNT(i) do { if (simt::lane_id() == 0) emu_prof[i]++; } while (0)
#else
#define EMU_COUNT(i) do {} while (0)
#endif

constexpr int kMaxInst = 32;
constexpr int32_t kRemMask = 0x07ffffff;
// no token yet (first token from a decode step, PC.ft): the step sets first_token
constexpr int32_t kFirst = 0x08000000;
constexpr int32_t kJoin = 0x40000000;  // no decode step since joining the batch
constexpr int32_t kCopy = 0x20000000;  // holds a redundant copy on the partner
// joined from the incoming list (moved / handed off / leveled) and not yet
// decoded a step here: not a rebalance candidate (SEMANTICS §6, "settling")
constexpr int32_t kSettle = 0x10000000;
enum { ROLE_DECODE = 0, ROLE_PREFILL = 1 };
enum { JOB_NONE = 0, JOB_PREFILL = 1, JOB_STEP = 2 };

// Per-warp shared scratch (atomics and radix histograms only; all simulation
// state lives in registers or the HBM arena).
struct PointConst {
  Perf f;
  int64_t budget, n_limit, event_budget;
  double warmup, duration, rate;
  uint64_t key;
  const double* tr_arr;
  const int32_t *tr_pl, *tr_dl;
  int32_t pmin, pmax, dmin, dmax, fixed_arrivals;
  // AcceLLM timer-driven extensions (SEMANTICS §6b)
  double timer_P, red_thr, exit_fill;
  int64_t lvl_budget, dual_budget;
  int32_t deg_on, lvl_on, trig;
  int32_t cobatch;  // splitwise high-load co-batching
  // first token from the first decode step instead of the prefill
  // (SPEC.md:273 alternative): kv = prompt + emitted + kvo, kvo = ft - 1
  int32_t ft, kvo;
};
struct Counters {
  int64_t n_steps, n_prefills, n_moves, n_preempt, n_evict;
  int64_t tok_total, tok_window, pf_tokens, mir_tokens, n_loop;
  int64_t ev_n;  // event-log cursor (atomic; lanes log concurrently)
  int64_t adv_events;  // virtual step ends processed by advance() (lane atomics)
  int64_t lvl_tokens, n_ticks, n_modes;
  int64_t t_n;   // detail runs: TBT (gap, count) entries written (atomic cursor)
};
struct WarpScratch {
  PointConst pc;  // written by lane 0 at point start, read (broadcast) by all
  Counters ct;    // updated by lane 0 only
  int64_t acc_a[kMaxInst];
  int64_t acc_b[kMaxInst];
  int32_t cnt[kMaxInst];
  uint32_t hist[2][256];
};

// Kernel arguments: inputs, outputs and the arena (one slot per resident warp).
struct SweepArgs {
  const kvsim_point_desc* pts;
  const int64_t* order;  // nullable: launch order (LPT) -> point index
  int64_t n_pts;
  kvsim_point_summary* out;
  // caller traces (concatenated), per-trace offset / count / max decode
  const double* tr_arr;
  const int32_t* tr_pl;
  const int32_t* tr_dl;
  const int64_t* tr_off;
  const int64_t* tr_n;
  const int32_t* tr_dmax;
  // optional outputs
  kvsim_request_record* recs;
  const int64_t* rec_off;
  kvsim_event_record* ev;
  int64_t ev_cap;
  int64_t* ev_count;
  // optional profiling: per point {start ns, end ns, slot} (globaltimer)
  unsigned long long* ptime;
  // optional per-instance records (point i at i * KVSIM_MAX_INSTANCES)
  kvsim_instance_record* inst;
  // detail runs (pooled TBT percentiles): plain event loop, one (gap, count)
  // entry per step / individual gap in [slot][Tcap]
  int32_t detail;
  int64_t Tcap;
  double* t_val;
  int32_t* t_cnt;
  // arena geometry
  int64_t Ncap, Bcap, Jcap;
  int32_t Imax, slots;
  // cold per-request arrays [slot][Ncap]
  double *c_arr, *c_last, *c_tbt, *c_fresh, *c_first, *c_done, *c_qs;
  int32_t *c_pl, *c_dl, *c_qlen, *c_em, *c_cpy, *c_nmv, *c_npre;
  int32_t* q_rid;  // [slot][Imax][Ncap] queue rings
  int32_t *b_rid, *b_rem, *b_kvb;
  double* b_tbt;  // [slot][Imax][Bcap] batch SoA
  int32_t* i_rid;
  double* i_ready;  // [slot][Imax][Bcap] incoming lists
  int32_t *j_rid, *j_dst;  // [slot][Imax][Jcap] prefill job members
  double* link;            // [slot][Imax][Imax] directed link busy-until
  unsigned long long* next_point;
};
// Shared memory of a sweep block (device builds):
//   dynamic: [kWarpsPerBlock x WarpScratch][kWarpsPerBlock * 32 x Sim]
//            (one Sim object per lane, AoS; 472 B = 118 words, so a warp's
//            same-field accesses are conflict-free for 8-byte fields)
//   static:  kvsim_args_smem, the block's copy of the kernel parameters, so
//            arena base pointers are LDS of a fixed address instead of
//            generic loads from the parameter space.
// -DKVSIM_SIM_STACK keeps the round-1 layout (Sim on the per-thread stack,
// i.e. local memory; parameters through a pointer) for A/B runs.
constexpr int kWarpsPerBlock = 4;
#ifndef KVSIM_PAIR_PAR
#define KVSIM_PAIR_PAR 1
#endif
#if !defined(KVSIM_EMU) && !defined(KVSIM_SIM_STACK)
#define KVSIM_SIM_SMEM 1
__shared__ SweepArgs kvsim_args_smem;
#define AR kvsim_args_smem
#else
#define AR (*A)
#endif
#define PC (ws()->pc)
// Event handlers and the helpers they call on every handled event. The lean
// sweep kernel inlines them into the event loop (kvsim_sweep.cu): a call
// costs more than the larger code (in-process A/B on config 4: 5.19 s with
// the handlers outlined, 4.25 s inlined). The full kernel
// (kvsim_sweep_full.cu: events, detail metrics, extensions) keeps them
// outlined (KVSIM_OUTLINE_HANDLERS), which bounds its compile time.
// Memory-pressure paths (eviction of redundant copies, preemption) stay
// out of line in every kernel: rarely executed, they only dilute the
// inlined event loop's instruction stream (A/B on config 4: 4.19 -> 4.17 s).
#define KV_DEV_COLD KV_DEV_NOINLINE
#if defined(KVSIM_OUTLINE_HANDLERS)
#define KV_DEV_HANDLER KV_DEV_NOINLINE
#else
#define KV_DEV_HANDLER KV_DEV
#endif
// One specialisation per policy: every `policy == ...` test folds at compile
// time, so a warp only ever executes (and caches) its own policy's code.
// EXT: AcceLLM with the policy timer (degraded mode / inter-pair leveling,
// SEMANTICS §6b): copies live on the instance partner[x] names (x^1, or the
// dual instance of a degraded group), all links use the directed-link matrix,
// and step chaining is off (plain event loop).
// DET: detail run (pooled TBT percentiles); implies the plain event loop.
template <int POL, bool LOG, bool EXT = false, bool DET = false>
struct Sim {
  const SweepArgs* A;  // kernel parameters (param space; __grid_constant__)
  WarpScratch* W;      // per-warp shared scratch: point constants, counters
  int lane;
  int32_t slot;
  int64_t point;
  static constexpr int32_t policy = POL;
  int32_t n, n_prefill;
  // arrival generator
  double t_next, t_prev;
  int64_t next_rid;
  bool has_next;
  // uniform counters that steer control flow
  int64_t n_events;
  double now;     // time of the event being processed (event-log timestamps)
  double t_last;  // latest event time processed (makespan)
  static constexpr bool chain_steps = !EXT && !DET;  // exact step chaining (advance); off = plain event loop
  static constexpr bool logging = LOG;  // event log compiled in (parity runs) or out (sweeps)
  int32_t status;
  // lane-owned instance state (lane x <-> instance x)
  double L_busy_until, L_job_start, L_prev_end, L_mirror_fin, L_busy_time, L_min_ready, L_link;
  int64_t L_used, L_peak, L_skv, L_skv_in, L_job_s1, L_copy_tok;
  int32_t L_role, L_job, L_nb, L_ni, L_pend, L_njob, L_ncopy;
  int32_t L_minrem;  // lower bound of remaining tokens over the batch
  // chained steps not yet applied to the batch arrays (see advance/flush)
  int32_t L_dj, L_compB;
  double L_dG, L_de1, L_dpe, L_comp;
  int64_t L_kvmin;   // AcceLLM: lower bound of kv over copy-holding members
  double L_tlast;    // latest virtual event time this lane processed (makespan)
  int64_t L_final;   // splitwise: sum of final KV (prompt+decode-1) over batch + incoming
  // lane-owned queue state (lane q <-> queue q)
  int32_t Q_head, Q_n;
  int64_t Q_tok;
  // EXT: copy holder of this instance's primaries (-1 none), pending leveling
  // migration (destination, token budget); lane g owns degraded group g
  int32_t L_partner, L_lvl_dst;
  int64_t L_lvl_bud;
  int64_t L_lvl_hold;  // KV of leveled requests held until their transfers finish
  double L_lvl_until;
  int32_t G_mode, G_cnt;
  int64_t tick;
  // idle while runnable: while this lane's instance is idle
  // and a request waits in a queue, the open interval started at L_irs
  double L_irs, L_idle_rb;
  // uniform: queue depth (waiting requests) and its time integral
  int64_t qdepth, qd_max;
  double qd_area, qd_tprev;

  // per-slot arena offsets, computed once (the accessors below run on every
  // arena access; recomputing slot * capacity from the parameter block each
  // time cost ~3% of all issued instructions)
  int64_t o_c, o_b, o_j, o_q, Bcap_, Jcap_, Ncap_;

  KV_DEV Sim(const SweepArgs* a, WarpScratch* w, int32_t s) : A(a), W(w), slot(s) {
    lane = simt::lane_id();
    Ncap_ = a->Ncap; Bcap_ = a->Bcap; Jcap_ = a->Jcap;
    o_c = (int64_t)s * Ncap_;
    o_b = (int64_t)s * a->Imax * Bcap_;
    o_j = (int64_t)s * a->Imax * Jcap_;
    o_q = (int64_t)s * a->Imax * Ncap_;
  }

  // ------------------------------------------------------------ arena views
  // every arena pointer is global memory; saying so lets ptxas emit LDG/STG
  // instead of generic accesses (no address-space check, no R2UR setup)
  // the per-warp scratch is shared memory (LDS/STS, not generic accesses)
  KV_DEV WarpScratch* ws() const {
#if defined(KVSIM_EMU)
    return W;
#else
    return reinterpret_cast<WarpScratch*>(kvsim_smem) + (threadIdx.x >> 5);
#endif
  }
  template <class T>
  static KV_DEV T* gp(T* p) {
#if !defined(KVSIM_EMU) && !defined(KVSIM_NO_GP_ASSUME)
    __builtin_assume(__isGlobal(p));
#endif
    return p;
  }
  KV_DEV double* c_arr() const { return gp(AR.c_arr + o_c); }
  KV_DEV double* c_last() const { return gp(AR.c_last + o_c); }
  KV_DEV double* c_tbt() const { return gp(AR.c_tbt + o_c); }
  KV_DEV double* c_fresh() const { return gp(AR.c_fresh + o_c); }
  KV_DEV double* c_first() const { return gp(AR.c_first + o_c); }
  KV_DEV double* c_done() const { return gp(AR.c_done + o_c); }
  KV_DEV double* c_qs() const { return gp(AR.c_qs + o_c); }
  KV_DEV int32_t* c_pl() const { return gp(AR.c_pl + o_c); }
  KV_DEV int32_t* c_dl() const { return gp(AR.c_dl + o_c); }
  KV_DEV int32_t* c_qlen() const { return gp(AR.c_qlen + o_c); }
  KV_DEV int32_t* c_em() const { return gp(AR.c_em + o_c); }
  KV_DEV int32_t* c_cpy() const { return gp(AR.c_cpy + o_c); }
  KV_DEV int32_t* c_nmv() const { return gp(AR.c_nmv + o_c); }
  KV_DEV int32_t* c_npre() const { return gp(AR.c_npre + o_c); }
  KV_DEV int64_t bofs(int x) const { return o_b + x * Bcap_; }
  KV_DEV int64_t jofs(int x) const { return o_j + x * Jcap_; }

  // ------------------------------------------------------------ accessors
  KV_DEV int32_t* b_rid(int x) { return gp(AR.b_rid + bofs(x)); }
  KV_DEV int32_t* b_rem(int x) { return gp(AR.b_rem + bofs(x)); }
  KV_DEV int32_t* b_kvb(int x) { return gp(AR.b_kvb + bofs(x)); }
  KV_DEV double* b_tbt(int x) { return gp(AR.b_tbt + bofs(x)); }
  KV_DEV int32_t* i_rid(int x) { return gp(AR.i_rid + bofs(x)); }
  KV_DEV double* i_ready(int x) { return gp(AR.i_ready + bofs(x)); }
  KV_DEV int32_t* j_rid(int x) { return gp(AR.j_rid + jofs(x)); }
  KV_DEV int32_t* j_dst(int x) { return gp(AR.j_dst + jofs(x)); }
  KV_DEV int32_t* ring(int q) { return gp(AR.q_rid + o_q + q * Ncap_); }
  KV_DEV double* link_() { return gp(AR.link + (int64_t)slot * AR.Imax * AR.Imax); }
  KV_DEV kvsim_event_record* evlog() const { return AR.ev ? AR.ev + point * AR.ev_cap : nullptr; }

  template <class T>
  KV_DEV T get(T v, int x) { return simt::shfl(v, x); }
  // warp min of event times (non-negative or +inf; bit order == value order)
  static KV_DEV double warp_min_time(double t) { return as_f64(simt::warp_min_u64(as_u64(t))); }
  KV_DEV bool own(int x) const { return lane == x; }
  // copy holder of x's primaries: the pair partner, or (EXT) partner[x]
  KV_DEV int partner_of(int x) {
    if constexpr (EXT) return get(L_partner, x);
    return x ^ 1;
  }
  // EXT degraded groups: pair q belongs to group q>>1 (if q>>1 < n/4); a
  // degraded group's requests wait in its first pair's queue
  KV_DEV bool degraded_pair(int q) {
    if constexpr (!EXT) return false;
    return (q >> 1) < (n >> 2) && get(G_mode, q >> 1) != 0;
  }
  KV_DEV int qid(int q) { return degraded_pair(q) ? (q & ~1) : q; }
  KV_DEV bool is_dual(int x) { return (x & 3) == 0 && degraded_pair(x >> 1); }
  KV_DEV int queue_of(int x) {
    return policy == KVSIM_POLICY_UNIFIED ? x : policy == KVSIM_POLICY_SPLITWISE ? 0 : qid(x >> 1);
  }
  KV_DEV void add_used(int x, int64_t tok) {
    if (own(x)) {
      L_used += tok;
      if (L_used > L_peak) L_peak = L_used;
    }
  }

  KV_DEV void put_event(int64_t k, double t, int kind, int inst, int a, int b, int64_t c) {
    if (k < AR.ev_cap) {
      kvsim_event_record r;
      r.t = t; r.kind = kind; r.inst = inst; r.a = a; r.b = b; r.c = c;
      evlog()[k] = r;
    }
  }
  // uniform call: one record at the current event time
  KV_DEV void log(int kind, int inst, int a, int b, int64_t c) {
    if constexpr (!LOG) return;
    if (lane == 0) put_event(simt::atomic_add_smem(&ws()->ct.ev_n, (int64_t)1), now, kind, inst, a, b, c);
    simt::sync();
  }
  // divergent call: this lane logs one record at time t
  KV_DEV void log_one(double t, int kind, int inst, int a, int b, int64_t c) {
    if constexpr (!LOG) return;
    put_event(simt::atomic_add_smem(&ws()->ct.ev_n, (int64_t)1), t, kind, inst, a, b, c);
  }
  // lane-parallel logging: lanes with `p` log one record each (moves)
  KV_DEV void log_lanes(bool p, int kind, int inst, int a, int b, int64_t c) {
    if constexpr (!LOG) return;
    if (p) put_event(simt::atomic_add_smem(&ws()->ct.ev_n, (int64_t)1), now, kind, inst, a, b, c);
    simt::sync();
  }

  // ------------------------------------------------------------- queues
  // queue depth series: area += depth * (now - previous change)
  // (and the idle-while-runnable intervals of idle instances, SEMANTICS §7:
  // they open when the queue becomes non-empty and close when it empties)
  KV_DEV void qd_change(int64_t delta) {
    qd_area = kadd(qd_area, kmul((double)qdepth, ksub(now, qd_tprev)));
    qd_tprev = now;
    const bool opens = qdepth == 0 && delta > 0;
    qdepth += delta;
    const bool closes = qdepth == 0;
    if ((opens || closes) && lane < n && L_job == JOB_NONE) {
      if (opens) L_irs = now;
      else L_idle_rb = kadd(L_idle_rb, ksub(clip(now), clip(L_irs)));
    }
    if (qdepth > qd_max) qd_max = qdepth;
  }
  KV_DEV void q_push_back(int q, int32_t rid, int64_t len) {
    int32_t h = get(Q_head, q), c = get(Q_n, q);
    int64_t idx = (int64_t)h + c;
    if (idx >= Ncap_) idx -= Ncap_;
    if (lane == 0) ring(q)[idx] = rid;
    simt::sync();
    if (own(q)) { Q_n += 1; Q_tok += len; }
    qd_change(1);
  }
  KV_DEV void q_push_front(int q, int32_t rid, int64_t len) {
    int32_t h = get(Q_head, q);
    int32_t nh = h == 0 ? (int32_t)(Ncap_ - 1) : h - 1;
    if (lane == 0) ring(q)[nh] = rid;
    simt::sync();
    if (own(q)) { Q_head = nh; Q_n += 1; Q_tok += len; }
    qd_change(1);
  }
  KV_DEV int32_t q_at(int q, int32_t h, int64_t k) {
    int64_t idx = (int64_t)h + k;
    if (idx >= Ncap_) idx -= Ncap_;
    return ring(q)[idx];
  }
  KV_DEV void q_pop(int q, int32_t k, int64_t tokens) {
    if (k > 0) qd_change(-(int64_t)k);
    if (own(q)) {
      int64_t nh = (int64_t)Q_head + k;
      if (nh >= Ncap_) nh -= Ncap_;
      Q_head = (int32_t)nh;
      Q_n -= k;
      Q_tok -= tokens;
    }
  }

  // ------------------------------------------------------------ point init
  KV_DEV bool init_point(int64_t p) {
    point = p;
    const kvsim_point_desc& d = AR.pts[p];
    PointConst pc;
    pc.f = make_perf(d);
    n = d.num_instances;
    n_prefill = 0;
    if (policy == KVSIM_POLICY_SPLITWISE)
      n_prefill = d.num_prefill_instances > 0 ? d.num_prefill_instances : (n + 2) / 4;
    pc.budget = d.prefill_token_budget > 0 ? d.prefill_token_budget : 8192;
    pc.fixed_arrivals = d.arrival_process == KVSIM_ARRIVAL_FIXED;
    pc.pmin = d.prompt_min; pc.pmax = d.prompt_max; pc.dmin = d.decode_min; pc.dmax = d.decode_max;
    pc.warmup = d.warmup_s;
    pc.duration = d.duration_s;
    pc.rate = d.rate;
    pc.key = stream_key(d.seed);
    pc.deg_on = EXT && (d.accellm_flags & KVSIM_ACCELLM_DEGRADED) != 0;
    pc.lvl_on = EXT && (d.accellm_flags & KVSIM_ACCELLM_LEVELING) != 0;
    pc.timer_P = d.policy_timer_s > 0.0 ? d.policy_timer_s : 1.0;
    pc.red_thr = d.degraded_redundancy > 0.0 ? d.degraded_redundancy : 0.5;
    pc.exit_fill = d.degraded_exit_fill > 0.0 ? d.degraded_exit_fill : 0.5;
    pc.trig = d.degraded_trigger_ticks > 0 ? d.degraded_trigger_ticks : 3;
    pc.cobatch = POL == KVSIM_POLICY_SPLITWISE && d.splitwise_cobatch != 0;
    pc.ft = d.first_token_decode != 0;
    pc.kvo = pc.ft - 1;
    {
      const double lf = d.leveling_link_fraction > 0.0 ? d.leveling_link_fraction : 0.10;
      const double df = d.dual_copy_fraction > 0.0 ? d.dual_copy_fraction : 1.0 / 3.0;
      pc.lvl_budget = (int64_t)simt::floor_d(kdiv(kmul(kmul(lf, pc.f.link_bw), pc.timer_P), pc.f.kvb));
      pc.dual_budget = (int64_t)kmul(df, (double)pc.f.cap);
    }
    status = KVSIM_OK;
    const int64_t nreq = d.num_requests < AR.Ncap ? d.num_requests : AR.Ncap;
    int32_t evd = pc.dmax;
    if (d.trace_index >= 0) {
      const int64_t off = AR.tr_off[d.trace_index];
      pc.tr_arr = AR.tr_arr + off; pc.tr_pl = AR.tr_pl + off; pc.tr_dl = AR.tr_dl + off;
      const int64_t tn = AR.tr_n[d.trace_index];
      pc.n_limit = tn < nreq ? tn : nreq;
      evd = AR.tr_dmax[d.trace_index];
    } else {
      pc.tr_arr = nullptr; pc.tr_pl = nullptr; pc.tr_dl = nullptr;
      pc.n_limit = pc.rate > 0.0 ? nreq : 0;
    }
    pc.event_budget = 4 * pc.n_limit * ((int64_t)(evd > 1 ? evd : 1) + 2) + 4096;
    // validity (perfmodel validate())
    if (n < 1 || n > kMaxInst || n > AR.Imax || d.policy != POL) status = KVSIM_E_INVALID;
    else if (!geometry_fits(d)) status = KVSIM_E_INVALID;
    else if (policy == KVSIM_POLICY_ACCELLM && (n & 1)) status = KVSIM_E_ODD_INSTANCES;
    else if (policy == KVSIM_POLICY_SPLITWISE && (n < 2 || n_prefill >= n)) status = KVSIM_E_INVALID;
    else if (!pc.f.fits) status = KVSIM_E_MODEL_FIT;
    simt::sync();  // previous point's readers are done with the scratch
    if (lane == 0) {
      ws()->pc = pc;
      ws()->ct = Counters{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    }
    simt::sync();
    n_events = 0;
    now = 0.0;
    t_last = 0.0;
    L_busy_until = L_job_start = L_prev_end = L_mirror_fin = L_busy_time = 0.0;
    L_min_ready = as_f64(0x7ff0000000000000ull);
    L_link = 0.0;
    L_used = L_peak = L_skv = L_skv_in = L_job_s1 = L_copy_tok = 0;
    L_role = (policy == KVSIM_POLICY_SPLITWISE && lane < n_prefill) ? ROLE_PREFILL : ROLE_DECODE;
    L_job = JOB_NONE;
    L_nb = L_ni = L_pend = L_njob = L_ncopy = 0;
    L_minrem = 0x7fffffff;
    L_final = 0;
    L_dj = 0; L_compB = -1; L_dG = L_de1 = L_dpe = L_comp = 0.0;
    L_kvmin = INT64_MAX;
    L_tlast = 0.0;
    Q_head = 0; Q_n = 0; Q_tok = 0;
    L_partner = lane ^ 1;
    L_lvl_dst = -1;
    L_lvl_bud = 0;
    L_lvl_hold = 0;
    L_lvl_until = 0.0;
    G_mode = G_cnt = 0;
    tick = 1;
    L_irs = L_idle_rb = 0.0;
    qdepth = qd_max = 0;
    qd_area = qd_tprev = 0.0;
    // directed links (splitwise; AcceLLM EXT)
    if (policy == KVSIM_POLICY_SPLITWISE || EXT)
      for (int i = lane; i < n * n; i += 32) link_()[i] = 0.0;
    next_rid = 0;
    t_prev = 0.0;
    has_next = false;
    if (status == KVSIM_OK) gen_next();
    simt::sync();
    return status == KVSIM_OK;
  }

  // the point must fit the arena geometry the launch was sized for
  // (kvsim_arena.hpp size_arena); a device-resident caller could pass points
  // that differ from its reservation, so this is re-checked per point
  KV_DEV_NOINLINE bool geometry_fits(const kvsim_point_desc& d) const {
    if (d.num_requests < 0 || d.num_requests > AR.Ncap) return false;
    if (d.trace_index >= 0) return AR.tr_off != nullptr;  // traces: sized by the host from the trace itself
    if (d.decode_max > kRemMask || d.prompt_max > kRemMask) return false;
    const int64_t N = d.num_requests;
    const int64_t pmin = d.prompt_min > 0 ? d.prompt_min : 1;
    const Perf f = make_perf(d);
    const int64_t cap = f.fits ? f.cap : 0;
    const int64_t budget = d.prefill_token_budget > 0 ? d.prefill_token_budget : 8192;
    const int64_t nb = cap / pmin + 2, nj = budget / pmin + 1;
    return (N < nb ? N : nb) <= AR.Bcap && (N < nj ? N : nj) <= AR.Jcap;
  }

  // arrival generator (SEMANTICS §2); uniform across lanes
  KV_DEV_HANDLER void gen_next() {
    has_next = false;
    if (next_rid >= PC.n_limit) return;
    double t;
    if (PC.tr_arr != nullptr) {
      t = PC.tr_arr[next_rid];
    } else if (PC.fixed_arrivals) {
      t = kdiv((double)next_rid, PC.rate);
      if (!(t < PC.duration)) return;
    } else {
      const double g = poisson_gap(PC.key, next_rid, PC.rate);
      t = next_rid == 0 ? g : kadd(t_prev, g);
      if (!(t < PC.duration)) return;
    }
    t_next = t;
    has_next = true;
  }

  // ------------------------------------------------------------- emission
  // token emission for a request leaving a prefill (first or recompute token)
  // by this lane; returns emitted count after.
  // Optional SPEC variants (first_token_decode, splitwise_cobatch) are
  // compiled into the LOG specialisation only; the sweep specialisation
  // folds them out and sweep_warp routes points that use them to LOG.
  static constexpr bool kFeat = LOG;
  KV_DEV bool ft() const { return kFeat && PC.ft; }
  KV_DEV bool cobatch() const { return kFeat && PC.cobatch; }
  // KV length offset: kv = prompt + emitted + kvo() (SEMANTICS §3)
  KV_DEV int32_t kvo() const { return kFeat ? PC.kvo : -1; }
  KV_DEV int32_t emit_prefill_token(int32_t rid, double t) {
    int32_t em = c_em()[rid];
    if (ft()) return em;  // the prefill emits nothing; the first decode step does
    if (em == 0) {
      c_first()[rid] = t;
    } else {
      double gap = ksub(t, c_last()[rid]);
      if (gap > c_tbt()[rid]) c_tbt()[rid] = gap;
      if constexpr (DET) if (c_arr()[rid] >= PC.warmup) tbt_entry(gap, 1);
    }
    c_last()[rid] = t;
    em += 1;
    c_em()[rid] = em;
    return em;
  }
  KV_DEV void count_tokens(int64_t k, double t) {
    if (lane == 0) ws()->ct.tok_total += k;
    if (t >= PC.warmup) if (lane == 0) ws()->ct.tok_window += k;
  }
  // detail runs: one TBT entry (gap shared by cnt samples); divergent-safe
  KV_DEV void tbt_entry(double gap, int32_t cnt) {
    const int64_t k = simt::atomic_add_smem(&ws()->ct.t_n, (int64_t)1);
    if (k < AR.Tcap) {
      gp(AR.t_val + (int64_t)slot * AR.Tcap)[k] = gap;
      gp(AR.t_cnt + (int64_t)slot * AR.Tcap)[k] = cnt;
    }
  }
  // ---- idle while runnable (SEMANTICS §7)
  KV_DEV double clip(double t) const { return t > PC.warmup ? t : PC.warmup; }
  // a job starts on x at t: close x's open idle-while-runnable interval
  KV_DEV void job_begin(int x, double t) {
    if (own(x) && qdepth > 0) L_idle_rb = kadd(L_idle_rb, ksub(clip(t), clip(L_irs)));
  }
  // a job ends on x at t: busy time; with a request waiting, x's
  // idle-while-runnable interval opens here
  KV_DEV void account_job(int x, double t) {
    double js = get(L_job_start, x);
    if (own(x)) {
      if (js >= PC.warmup) L_busy_time = kadd(L_busy_time, ksub(t, js));
      if (qdepth > 0) L_irs = t;
    }
  }

  // ------------------------------------------------------- hot decode loop
  // Advances every member of x's batch by one token at time t
  // and compacts completions away. Returns completed count; accumulates the
  // kv (before the step) of completed requests, the kv-after of completed
  // requests holding a copy, and the number of members holding a copy.
  struct StepOut {
    int32_t nb_old, completed, m_copies, copy_done, minrem;
    int64_t kv_done, copy_free, kvmin;
  };
  KV_DEV_HANDLER StepOut step_loop(int x, double t) {
    EMU_COUNT(0);
    StepOut o;
    const int32_t nb = get(L_nb, x);
    const double prev = get(L_prev_end, x);
    // chained steps not yet applied (advance/flush) are applied in the same
    // pass: remaining tokens -dj, TBT max with the deferred gaps
    const int32_t dj = get(L_dj, x);
    const double e1 = get(L_de1, x), pe = get(L_dpe, x), G = get(L_dG, x);
    int32_t* rid_a = b_rid(x);
    int32_t* rem_a = b_rem(x);
    int32_t* kvb_a = b_kvb(x);
    double* tbt_a = b_tbt(x);
    int32_t wpos = 0, completed = 0, m = 0, copy_done = 0, minrem = 0x7fffffff;
    int32_t ncont = 0;  // detail runs: measured members sharing the gap t - prev
    int64_t kv_done = 0, copy_free = 0, kvmin = INT64_MAX;  // per-lane partials
    for (int32_t j0 = 0; j0 < nb; j0 += 32) {
      const int32_t j = j0 + lane;
      const bool act = j < nb;
      int32_t rf = 0, rid = 0, kvb = 0;
      double tb = 0.0;
      if (act) {
        rf = rem_a[j];
        tb = tbt_a[j];
      }
      const int32_t rem = (rf & kRemMask) - dj - 1;
      const bool was_joiner = (rf & kJoin) != 0;
      const bool joiner = was_joiner && dj == 0;  // no step since joining
      const bool hasc = (rf & kCopy) != 0;
      const bool first = kFeat && (rf & kFirst) != 0;  // this step (or the first deferred one) emits its first token
      const bool done = act && rem == 0;
      const bool surv = act && rem != 0;
      const unsigned sm = simt::ballot(surv);
      const int32_t dst = wpos + simt::popc(sm & simt::lanemask_lt());
      const bool moved = surv && dst != j;
      if (act && (DET || was_joiner || done || moved || first)) rid = rid_a[j];
      double gap = 0.0;
      bool upd = false;
      if (act && first) {  // no earlier token: no gap into the first one
        c_first()[rid] = dj > 0 ? e1 : t;
        if (dj > 0) {
          if (G > tb) { tb = G; upd = true; }
          gap = ksub(t, prev);
          if (gap > tb) { tb = gap; upd = true; }
        }
      } else if (act) {
        if (dj > 0) {
          const double last0 = was_joiner ? c_last()[rid] : pe;
          double g1 = ksub(e1, last0);
          if (G > g1) g1 = G;
          if (g1 > tb) { tb = g1; upd = true; }
        }
        const double last = joiner ? c_last()[rid] : prev;
        gap = ksub(t, last);
        if (gap > tb) { tb = gap; upd = true; }
      }
      if constexpr (DET) {
        const bool inc = act && !first && c_arr()[rid] >= PC.warmup;
        if (inc && joiner) tbt_entry(gap, 1);
        ncont += simt::popc(simt::ballot(inc && !joiner));
      }
      if (done || moved) kvb = kvb_a[j];
      m += simt::popc(simt::ballot(act && hasc));
      simt::sync();  // all reads of this chunk precede its compaction writes
      if (surv) {
        if (rem < minrem) minrem = rem;
        if (hasc) {
          const int64_t kvn = (int64_t)(kvb_a[j]) - rem;  // kv after this step
          if (kvn < kvmin) kvmin = kvn;
        }
        rem_a[dst] = rem | (rf & kCopy);
        if (moved) {
          rid_a[dst] = rid;
          kvb_a[dst] = kvb;
          tbt_a[dst] = tb;
        } else if (upd) {
          tbt_a[dst] = tb;
        }
      }
      if (done) {
        c_done()[rid] = t;
        c_tbt()[rid] = tb;
        c_em()[rid] = c_dl()[rid];
        const int64_t kvbef = (int64_t)kvb - 1;  // kv before the step: kvb - (rem+1), rem == 0
        kv_done += kvbef;
        if (hasc) copy_free += kvbef + 1;
      }
      const unsigned dm = simt::ballot(done);
      completed += simt::popc(dm);
      copy_done += simt::popc(simt::ballot(done && hasc));
      wpos += simt::popc(sm);
    }
    if constexpr (DET) {
      if (ncont > 0 && lane == 0) tbt_entry(ksub(t, prev), ncont);
    }
    o.nb_old = nb;
    o.completed = completed;
    o.m_copies = m;
    o.copy_done = copy_done;
    o.kv_done = simt::warp_sum_nn(kv_done);
    o.copy_free = simt::warp_sum_nn(copy_free);
    o.minrem = simt::warp_min_i32(minrem);
    o.kvmin = simt::warp_min_i64(kvmin);
    simt::sync();
    if (own(x) && dj > 0) { L_dj = 0; L_dG = 0.0; }
    return o;
  }

  // -------------------------------------------------------------- joins
  KV_DEV void join(int x, double t) {
    if (get(L_ni, x) == 0) return;
    if (get(L_min_ready, x) > t) return;
    join_slow(x, t);
  }
  KV_DEV_HANDLER void join_slow(int x, double t) {
    EMU_COUNT(1);
    flush(x);
    const int32_t ni = get(L_ni, x);
    if (ni == 0) return;
    if (get(L_min_ready, x) > t) return;
    const int32_t nb = get(L_nb, x);
    int32_t* irid = i_rid(x);
    double* irdy = i_ready(x);
    int32_t keep = 0, add = 0, ncopy = 0, minrem = 0x7fffffff;
    int64_t kvsum = 0, kvmin = INT64_MAX;
    double mn = as_f64(0x7ff0000000000000ull);
    for (int32_t j0 = 0; j0 < ni; j0 += 32) {
      const int32_t j = j0 + lane;
      const bool act = j < ni;
      int32_t rid = 0;
      double rd = 0.0;
      if (act) { rid = irid[j]; rd = irdy[j]; }
      const bool go = act && rd <= t;
      const bool stay = act && !go;
      const unsigned gm = simt::ballot(go), sm = simt::ballot(stay);
      simt::sync();
      if (stay) {
        const int32_t k = keep + simt::popc(sm & simt::lanemask_lt());
        irid[k] = rid;
        irdy[k] = rd;
        if (rd < mn) mn = rd;
      }
      if (go) {
        const int32_t k = nb + add + simt::popc(gm & simt::lanemask_lt());
        const int32_t em = c_em()[rid], dl = c_dl()[rid], pl = c_pl()[rid];
        const bool hasc = c_cpy()[rid] >= 0;
        b_rid(x)[k] = rid;
        b_rem(x)[k] = (dl - em) | kJoin | kSettle | (hasc ? kCopy : 0) | (em == 0 ? kFirst : 0);
        b_kvb(x)[k] = pl + dl + kvo();
        b_tbt(x)[k] = c_tbt()[rid];
        kvsum += (int64_t)pl + em + kvo();
        if (dl - em < minrem) minrem = dl - em;
        if (hasc && (int64_t)pl + em + kvo() < kvmin) kvmin = (int64_t)pl + em + kvo();
      }
      ncopy += simt::popc(simt::ballot(go && c_cpy()[go ? rid : 0] >= 0));
      keep += simt::popc(sm);
      add += simt::popc(gm);
    }
    kvsum = simt::warp_sum_nn(kvsum);
    mn = warp_min_time(mn);
    minrem = simt::warp_min_i32(minrem);
    kvmin = simt::warp_min_i64(kvmin);
    simt::sync();
    if (own(x)) {
      if (minrem < L_minrem) L_minrem = minrem;
      if (kvmin < L_kvmin) L_kvmin = kvmin;
      L_nb += add;
      L_ni -= add;
      L_skv += kvsum;
      L_skv_in -= kvsum;
      L_ncopy += ncopy;
      L_min_ready = mn;
    }
    if (add) log(KVSIM_EV_JOIN, x, add, 0, 0);
  }

  // remove batch slot idx of instance x by moving the last slot into it
  KV_DEV void batch_remove(int x, int32_t idx) {
    const int32_t last = get(L_nb, x) - 1;
    if (lane == 0 && idx != last) {
      b_rid(x)[idx] = b_rid(x)[last];
      b_rem(x)[idx] = b_rem(x)[last];
      b_kvb(x)[idx] = b_kvb(x)[last];
      b_tbt(x)[idx] = b_tbt(x)[last];
    }
    simt::sync();
    if (own(x)) L_nb -= 1;
  }
  KV_DEV void incoming_remove(int x, int32_t idx) {
    const int32_t last = get(L_ni, x) - 1;
    if (lane == 0 && idx != last) {
      i_rid(x)[idx] = i_rid(x)[last];
      i_ready(x)[idx] = i_ready(x)[last];
    }
    simt::sync();
    if (own(x)) L_ni -= 1;
  }
  KV_DEV void incoming_append(int y, int32_t rid, double ready) {
    const int32_t k = get(L_ni, y);
    if (lane == 0) {
      i_rid(y)[k] = rid;
      i_ready(y)[k] = ready;
    }
    simt::sync();
    if (own(y)) {
      L_ni += 1;
      if (ready < L_min_ready) L_min_ready = ready;
    }
  }

  // ------------------------------------------------------- copies (AcceLLM)
  struct Found {
    int32_t rid, idx, where;  // where: 0 none, 1 batch of client y, 2 incoming of client y
    int32_t y;                // the instance whose primary the copy belongs to
    int64_t kv;
  };
  // instances whose copies x holds (its pair partner; EXT: every y with
  // partner[y] == x)
  KV_DEV unsigned clients_of(int x) {
    if constexpr (EXT) return simt::ballot(lane < n && lane != x && L_partner == x);
    return 1u << (x ^ 1);
  }
  // largest redundant copy held on instance x (max kv, ties lowest rid)
  KV_DEV Found largest_copy_on(int x) { return largest_copy_on_from(x, clients_of(x)); }
  KV_DEV_COLD Found largest_copy_on_from(int x, unsigned clients) {
    uint64_t best = 0;
    int32_t bidx = -1, bwhere = 0, by = -1;
    for (unsigned cm = clients; cm; cm &= cm - 1) {
      const int y = simt::ffs(cm) - 1;
      flush(y);
      const int32_t nb = get(L_nb, y), ni = get(L_ni, y);
      for (int32_t j = lane; j < nb; j += 32) {
        const int32_t rf = b_rem(y)[j];
        if (rf & kCopy) {
          const int64_t kv = (int64_t)b_kvb(y)[j] - (rf & kRemMask);
          const uint64_t k = ((uint64_t)kv << 32) | (uint32_t)(0x7fffffff - b_rid(y)[j]);
          if (k > best) { best = k; bidx = j; bwhere = 1; by = y; }
        }
      }
      for (int32_t j = lane; j < ni; j += 32) {
        const int32_t rid = i_rid(y)[j];
        if (c_cpy()[rid] == x) {
          const int64_t kv = (int64_t)c_pl()[rid] + c_em()[rid] + kvo();
          const uint64_t k = ((uint64_t)kv << 32) | (uint32_t)(0x7fffffff - rid);
          if (k > best) { best = k; bidx = j; bwhere = 2; by = y; }
        }
      }
    }
    const uint64_t wbest = simt::warp_max_u64(best);
    Found r;
    r.where = 0; r.idx = -1; r.rid = -1; r.kv = 0; r.y = -1;
    if (wbest == 0) return r;
    const unsigned holder = simt::ballot(best == wbest);
    const int src = simt::ffs(holder) - 1;
    r.idx = simt::shfl(bidx, src);
    r.where = simt::shfl(bwhere, src);
    r.y = simt::shfl(by, src);
    r.rid = 0x7fffffff - (int32_t)(uint32_t)(wbest & 0xffffffffu);
    r.kv = (int64_t)(wbest >> 32);
    return r;
  }
  KV_DEV_COLD void evict(int x, Found v) {
    EMU_COUNT(14);
    const int y = v.y;
    int64_t held = v.kv;
    if (v.where == 1) {
      if (get(L_job, y) == JOB_STEP) held += 1;
      if (lane == 0) b_rem(y)[v.idx] &= ~kCopy;
      if (own(y)) L_ncopy -= 1;
    } else {
      if (lane == 0) c_cpy()[v.rid] = -1;
    }
    simt::sync();
    if (own(x)) { L_used -= held; L_copy_tok -= held; }
    if (lane == 0) ws()->ct.n_evict += 1;
    log(KVSIM_EV_EVICT, x, v.rid, 0, 0);
  }

  // ------------------------------------------------------ preemption (P9)
  KV_DEV_COLD void preempt_newest(int x) {
    EMU_COUNT(15);
    flush(x);
    const int32_t nb = get(L_nb, x);
    int32_t best = -1, bidx = -1;
    for (int32_t j = lane; j < nb; j += 32) {
      const int32_t r = b_rid(x)[j];
      if (r > best) { best = r; bidx = j; }
    }
    const int32_t rid = simt::warp_max_i32(best);
    const int src = simt::ffs(simt::ballot(best == rid)) - 1;
    const int32_t idx = simt::shfl(bidx, src);
    const int32_t rf = b_rem(x)[idx];
    const int32_t rem = rf & kRemMask;
    const int64_t kv = (int64_t)b_kvb(x)[idx] - rem;
    const int32_t dl = c_dl()[rid], pl = c_pl()[rid];
    const int32_t em = dl - rem;
    const double tb = b_tbt(x)[idx];
    const double last = (rf & kJoin) ? c_last()[rid] : get(L_prev_end, x);
    const int32_t qlen = pl + em;
    simt::sync();
    if (lane == 0) {
      c_em()[rid] = em;
      c_tbt()[rid] = tb;
      c_last()[rid] = last;
      c_cpy()[rid] = -1;
      c_qlen()[rid] = qlen;
      c_npre()[rid] += 1;
    }
    if (own(x)) { L_used -= kv; L_skv -= kv; L_final -= (int64_t)pl + dl + kvo(); }
    if (rf & kCopy) {
      const int y = partner_of(x);
      if (own(y)) { L_used -= kv; L_copy_tok -= kv; }
      if (own(x)) L_ncopy -= 1;
    }
    batch_remove(x, idx);
    if (lane == 0) ws()->ct.n_preempt += 1;
    log(KVSIM_EV_PREEMPT, x, rid, qlen, 0);
    q_push_front(queue_of(x), rid, qlen);
  }

  // ------------------------------------------------------------ link FIFO
  KV_DEV double link_get(int s, int d) {
    if (policy == KVSIM_POLICY_ACCELLM && !EXT) return get(L_link, s);  // only (s, s^1)
    return link_()[s * n + d];
  }
  KV_DEV void link_set(int s, int d, double v) {
    if (policy == KVSIM_POLICY_ACCELLM && !EXT) {
      if (own(s)) L_link = v;
    } else {
      simt::sync();  // every lane has read the old value
      if (lane == 0) link_()[s * n + d] = v;
      simt::sync();
    }
  }
  KV_DEV_HANDLER double prefill_transfer(int s, int d, int64_t s1, double t_start, double t_done) {
    const double busy = link_get(s, d);
    const double tail = kadd(t_done, transfer_latency(PC.f, kmul((double)s1, PC.f.kvb_layer)));
    const double start = t_start > busy ? t_start : busy;
    const double full = kadd(start, transfer_latency(PC.f, kmul((double)s1, PC.f.kvb)));
    const double fin = tail > full ? tail : full;
    link_set(s, d, fin);
    if (lane == 0) ws()->ct.pf_tokens += s1;
    log(KVSIM_EV_TRANSFER, s, d, 0, s1);
    return fin;
  }

  // ------------------------------------------- decode step (splitwise/accellm)
  KV_DEV_HANDLER void step_start(int x, double t) {
    EMU_COUNT(2);
    if constexpr (POL == KVSIM_POLICY_SPLITWISE) {
      if (cobatch()) { sw_cobatch_start(x, t); return; }
    }
    int32_t nb = get(L_nb, x);
    if (nb == 0) return;
    const bool acc = policy == KVSIM_POLICY_ACCELLM;
    bool preempted = false;
    for (;;) {
      if (get(L_used, x) + nb <= PC.f.cap) break;
      if (acc) {
        Found v = largest_copy_on(x);
        if (v.where) { evict(x, v); continue; }
      }
      preempt_newest(x);
      preempted = true;
      nb -= 1;
      if (nb == 0) break;
    }
    if (nb == 0) {
      if (preempted && acc) ensure_prefill(qid(x >> 1), t);
      return;
    }
    if (acc && partner_of(x) >= 0) {
      const int y = partner_of(x);
      for (;;) {
        const int32_t m = get(L_ncopy, x);
        if (get(L_used, y) + m <= PC.f.cap) {
          add_used(y, m);
          if (own(y)) L_copy_tok += m;
          break;
        }
        Found v = largest_copy_on(y);
        evict(y, v);
      }
    }
    const int64_t K = get(L_skv, x);
    add_used(x, nb);
    const double lat = decode_latency(PC.f, nb, K);
    job_begin(x, t);
    if (own(x)) {
      L_job = JOB_STEP;
      L_job_start = t;
      L_busy_until = kadd(t, lat);
    }
    log(KVSIM_EV_STEP_START, x, nb, 0, K);
    if (preempted && acc) ensure_prefill(qid(x >> 1), t);

  }

  KV_DEV_HANDLER void step_end(int x, double t) {
    EMU_COUNT(3);
    account_job(x, t);
    if (lane == 0) ws()->ct.n_steps += 1;
    const StepOut o = step_loop(x, t);  // applies the deferred chained steps too
    const int32_t surv = o.nb_old - o.completed;
    if (own(x)) {
      L_job = JOB_NONE;
      L_used -= o.kv_done + o.completed;
      L_skv = L_skv - o.kv_done + surv;
      L_nb = surv;
      L_prev_end = t;
      L_minrem = o.minrem;
      L_kvmin = o.kvmin;
      L_final -= o.kv_done + o.completed;
    }
    count_tokens(o.nb_old, t);
    if (policy == KVSIM_POLICY_ACCELLM) {
      const int y = partner_of(x);
      if (own(y)) { L_used -= o.copy_free; L_copy_tok -= o.copy_free; }
      if (own(x)) L_ncopy -= o.copy_done;
      if (o.m_copies > 0) {
        const double busy = link_get(x, y);
        const double start = t > busy ? t : busy;
        const double fin = kadd(start, transfer_latency(PC.f, kmul((double)o.m_copies, PC.f.kvb)));
        link_set(x, y, fin);
        if (own(x)) L_mirror_fin = fin;
        if (lane == 0) ws()->ct.mir_tokens += o.m_copies;
        log(KVSIM_EV_TRANSFER, x, y, 1, o.m_copies);
      }
    }
    log(KVSIM_EV_STEP_END, x, o.nb_old, o.completed, 0);
  }


  // ------------------------------------------------ exact step chaining
  // A decode step end of instance x is *virtual* when nothing can interact
  // with it: no member completes (remaining-token bound), nobody joins (min
  // incoming ready time), the next step's KV growth fits (and, AcceLLM, the
  // partner's mirror lines), no rebalance move is possible (closed-form
  // bound on the smallest copy-holding KV vs the growing token imbalance),
  // no admission is pending, and every event that can read or change x's
  // state -- the next arrival, the prefill instances (Splitwise), the pair
  // partner (AcceLLM) -- comes later in (time, kind, id) order. Events of
  // independent instances/pairs commute with it, so results are unchanged.
  //
  // advance(): every driving lane (an instance, or the even lane of an
  // AcceLLM pair) processes its virtual step ends in registers, in parallel
  // across lanes. The per-request part (remaining tokens, TBT maxima) is
  // deferred: L_dj steps, first-step end L_de1, previous end L_dpe, max later
  // gap L_dG; flush() applies it in one pass when the batch is next touched.
  KV_DEV void flush(int x) {
    if (get(L_dj, x) == 0) return;
    flush_slow(x);
  }
  // Vectorised SoA pass: each lane takes 4 consecutive members per round
  // (one 16-byte load of their remaining-token words, two of their TBT
  // maxima; Bcap is a multiple of 4 and the arrays 16-byte aligned, so the
  // slots past B in the last vector are unused and written back unchanged).
  KV_DEV_HANDLER void flush_slow(int x) {
    const int32_t j = get(L_dj, x);
    const double e1 = get(L_de1, x), pe = get(L_dpe, x), G = get(L_dG, x);
    const int32_t B = get(L_nb, x);
    int32_t* rem_a = b_rem(x);
    double* tbt_a = b_tbt(x);
    for (int32_t q0 = 4 * lane; q0 < B; q0 += 128) {
      kv_int4 r4 = *reinterpret_cast<const kv_int4*>(rem_a + q0);
      kv_double2 t01 = *reinterpret_cast<const kv_double2*>(tbt_a + q0);
      kv_double2 t23 = *reinterpret_cast<const kv_double2*>(tbt_a + q0 + 2);
      int32_t rf[4] = {r4.x, r4.y, r4.z, r4.w};
      double tb[4] = {t01.x, t01.y, t23.x, t23.y};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (q0 + k >= B) break;
        double g1;
        if (kFeat && (rf[k] & kFirst)) {  // first token at the first deferred step end
          c_first()[b_rid(x)[q0 + k]] = e1;
          g1 = G;
        } else {
          const double last = (rf[k] & kJoin) ? c_last()[b_rid(x)[q0 + k]] : pe;
          g1 = ksub(e1, last);
          if (G > g1) g1 = G;
        }
        rf[k] = ((rf[k] & kRemMask) - j) | (rf[k] & kCopy);
        if (g1 > tb[k]) tb[k] = g1;
      }
      *reinterpret_cast<kv_int4*>(rem_a + q0) = kv_int4{rf[0], rf[1], rf[2], rf[3]};
      *reinterpret_cast<kv_double2*>(tbt_a + q0) = kv_double2{tb[0], tb[1]};
      *reinterpret_cast<kv_double2*>(tbt_a + q0 + 2) = kv_double2{tb[2], tb[3]};
    }
    simt::sync();
    if (own(x)) { L_dj = 0; L_dG = 0.0; }
  }

  // decode compute floor for batch B and mirror time for m lines (lane cache)
  KV_DEV double comp_floor(int32_t B) {
    if (B != L_compB) { L_compB = B; L_comp = kdiv(kmul(PC.f.two_p, (double)B), PC.f.pf_den); }
    return L_comp;
  }

  // per-member register state of an AcceLLM pair chain (driver lane)
  struct MemberChain {
    double e, js, busy, link, mfin, prev, de1, dpe, dG, mr, comp, mlat;
    double Kd;  // == (double)(skv + steps * B): the running KV sum of the next step
    int64_t skv, skv_in, used, peak, copy_tok, kvmin, tw;
    int32_t B, ni, m, minrem, dj, role, steps;
    bool stepping;
  };
  struct ChainK {
    double Wb, kvb, mden, mrcp, warmup;
    int64_t cap;
  };
  // one virtual step end of a chained pair member (bookkeeping only; the
  // caller has evaluated the stop tests)
  // (c.tw counts steps ending in the window; skv is applied after the chain)
  KV_DEV void lean_step(MemberChain& c, const ChainK& K, int cid) {
    const double e = c.e;
    const double st = ksub(e, c.js);
    if (c.js >= K.warmup) c.busy = kadd(c.busy, st);
    if (e >= K.warmup) c.tw += 1;
    if (c.dj == 0) { c.de1 = e; c.dpe = c.prev; }
    else {  // deferred steps pending: the previous step ended where this one started
      const double g = c.js == c.prev ? st : ksub(e, c.prev);
      if (g > c.dG) c.dG = g;
    }
    if (c.m > 0) {
      const double lk = e > c.link ? e : c.link;
      c.link = kadd(lk, c.mlat);
      c.mfin = c.link;
      if constexpr (LOG) log_one(e, KVSIM_EV_TRANSFER, cid, cid ^ 1, 1, c.m);
    }
    if constexpr (LOG) log_one(e, KVSIM_EV_STEP_END, cid, c.B, 0, 0);
    c.Kd = kadd(c.Kd, (double)c.B);
    if constexpr (LOG) log_one(e, KVSIM_EV_STEP_START, cid, c.B, 0, c.skv + (int64_t)(c.steps + 1) * c.B);
    c.prev = e;
    c.js = e;
    c.e = kadd(e, kvsim_math::kmax(kdiv_rcp(kadd(K.Wb, kmul(c.Kd, K.kvb)), K.mden, K.mrcp), c.comp));
    c.dj += 1;
    c.steps += 1;
  }
#if KVSIM_PAIR_PAR
  // ---- member-parallel AcceLLM pair chains
  // The serial merged loop (KVSIM_PAIR_PAR=0) advances both members of a pair
  // on the even lane, one step end at a time in (time, id) order, and stops at the first
  // step end whose tests fail. A member's step times depend only on its own
  // state; the members interact only through the stop tests (the KV slack of
  // each member, which the partner's mirror lines also consume, the
  // rebalance gaps, the event budget). Here each member runs its own chain on
  // its own lane under member-local limits that imply those tests for any
  // interleaving (a chain may always stop early: the event loop then handles
  // the step end exactly):
  //   KV slack / budget: both members take at most C steps, with C such that
  //   C (B_a + m_b) <= cap - used_a, C (B_b + m_a) <= cap - used_b, 2C <= budget;
  //   rebalance gap: a's gap grows by B_a - 1 per own step and only shrinks
  //   with partner steps, so the own steps alone bound it.
  // A pair's merged chain ends at the earlier of the two members' first
  // untaken step ends; the member whose taken steps reach past the partner's
  // is re-run with that bound (at most one of the two). (Emulator, config-4
  // AcceLLM points: 2.3-2.8 re-runs and 9-10 pair chains per simulated
  // request; the member-local bounds add ~5% handled step ends.)
  struct PChain {
    double e, js, busy, dG, de1, dpe, link, mfin;
    int32_t k, tw;
  };
  template <bool DOLOG>
  KV_DEV PChain pair_member_run(int32_t nmax, double tl, double comp, double mlat, int32_t m, int32_t B) {
    PChain c;
    c.e = L_busy_until; c.js = L_job_start; c.busy = L_busy_time;
    c.dG = L_dG; c.de1 = L_de1; c.dpe = L_dpe; c.link = L_link; c.mfin = L_mirror_fin;
    c.k = 0; c.tw = 0;
    if (!(nmax > 0 && c.e < tl)) return c;
    const double Wb = PC.f.W, kvb = PC.f.kvb, mden = PC.f.mem_den, mrcp = PC.f.mem_rcp, warmup = PC.warmup;
    const int64_t skv0 = L_skv;
    const double Bd = (double)B;
    double Kd = (double)skv0;
    double e = c.e, js = c.js, busy = c.busy, dG = c.dG, link = c.link;
    double q0;  // the first step's verified quotient
    int32_t k = 0, tw = 0;
    {  // first chained step: gap against the previous step end (lean_step)
      const double prev = L_prev_end;
      const double st = ksub(e, js);
      if (js >= warmup) busy = kadd(busy, st);
      if (e >= warmup) tw += 1;
      if (L_dj == 0) { c.de1 = e; c.dpe = prev; }
      else { const double g = js == prev ? st : ksub(e, prev); if (g > dG) dG = g; }
      if (m > 0) {
        link = kadd(e > link ? e : link, mlat);
        if constexpr (DOLOG) log_one(e, KVSIM_EV_TRANSFER, lane, lane ^ 1, 1, m);
      }
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
      Kd = kadd(Kd, Bd);
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + B);
      js = e;
      q0 = kdiv_rcp(kadd(Wb, kmul(Kd, kvb)), mden, mrcp);
      e = kadd(e, kvsim_math::kmax(q0, comp));
      k = 1;
    }
    // later quotients only grow: the cheap loop-invariant acceptance test
    const double T = kdiv_chain_thr(q0, mden);
    // steady state: js == prev, one difference is the busy increment and the
    // gap; first the steps that started before the measurement window
    while (k < nmax && e < tl && js < warmup) {
      const double st = ksub(e, js);
      if (st > dG) dG = st;
      if (e >= warmup) tw += 1;
      if (m > 0) {
        link = kadd(e > link ? e : link, mlat);
        if constexpr (DOLOG) log_one(e, KVSIM_EV_TRANSFER, lane, lane ^ 1, 1, m);
      }
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
      Kd = kadd(Kd, Bd);
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + (int64_t)(k + 1) * B);
      js = e;
      e = kadd(e, kvsim_math::kmax(kdiv_chain(kadd(Wb, kmul(Kd, kvb)), mden, mrcp, T, q0), comp));
      k += 1;
    }
    // inside the window (times only grow): every step adds busy time and ends in it
    const int32_t kw = k;
    while (k < nmax && e < tl) {
      const double st = ksub(e, js);
      busy = kadd(busy, st);
      if (st > dG) dG = st;
      if (m > 0) {
        link = kadd(e > link ? e : link, mlat);
        if constexpr (DOLOG) log_one(e, KVSIM_EV_TRANSFER, lane, lane ^ 1, 1, m);
      }
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
      Kd = kadd(Kd, Bd);
      if constexpr (DOLOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + (int64_t)(k + 1) * B);
      js = e;
      e = kadd(e, kvsim_math::kmax(kdiv_chain(kadd(Wb, kmul(Kd, kvb)), mden, mrcp, T, q0), comp));
      k += 1;
    }
    tw += k - kw;
    c.e = e; c.js = js; c.busy = busy; c.dG = dG; c.link = link;
    if (m > 0) c.mfin = link;
    c.k = k; c.tw = tw;
    return c;
  }
  // pc: this lane's pair is a chain candidate (pair-uniform); accumulates the
  // lane's counters.
  KV_DEV void pair_par(bool pc, double ht, int32_t hk, int64_t budget, int64_t& steps, int64_t& tok, int64_t& tw,
                       int64_t& mir, double& tmax) {
    const double kInf = as_f64(0x7ff0000000000000ull);
    const int y = lane ^ 1;
    const bool isb = (lane & 1) != 0;
    // partner state (all lanes stay converged through the shuffles; lanes of
    // other pairs run empty chains)
    const int32_t p_job = simt::shfl(L_job, y), p_nb = simt::shfl(L_nb, y), p_ni = simt::shfl(L_ni, y);
    const int32_t p_role = simt::shfl(L_role, y), p_m = simt::shfl(L_ncopy, y);
    const double p_e = simt::shfl(L_busy_until, y), p_mr = simt::shfl(L_min_ready, y);
    const int64_t p_used = simt::shfl(L_used, y), p_sk = simt::shfl(L_skv + L_skv_in, y);
    const bool st_me = L_job == JOB_STEP, st_p = p_job == JOB_STEP;
    // the next arrival, and the non-stepping members' own events
    double pht = ht;
    int32_t phk = hk;
    auto fold = [&](bool stepping, int32_t job, double e, int32_t role, int32_t ni, double mr, int32_t id) {
      if (stepping) return;
      double yt = kInf;
      int32_t yk = 0;
      if (job == JOB_PREFILL) { yt = e; yk = 2 * 64 + id; }
      else if (role == ROLE_DECODE && ni > 0) { yt = mr; yk = 64 + id; }
      if (yt < pht || (yt == pht && yk < phk)) { pht = yt; phk = yk; }
    };
    fold(st_me, L_job, L_busy_until, L_role, L_ni, L_min_ready, lane);
    fold(st_p, p_job, p_e, p_role, p_ni, p_mr, y);
    // B as the serial loop has it in its tests (a's zeroed when a is not stepping)
    const int32_t B = L_nb;
    const int32_t Bme = (!isb && !st_me) ? 0 : B, Bp = (isb && !st_p) ? 0 : p_nb;
    // own limit: remaining-token count and the rebalance gap G0 + i (B - 1) < 0
    // (the partner's steps only lower G)
    int64_t lim = st_me ? (int64_t)L_minrem - 1 : 0;
    if (p_role == ROLE_DECODE && L_kvmin != INT64_MAX) {
      const int64_t cz = (int64_t)Bme + L_ni - Bp - p_ni;
      if (cz >= 1) {
        const int64_t dz = (L_skv + L_skv_in + Bme) - p_sk;
        const int64_t G = (cz >= 2 ? dz : dz - 1) - (L_kvmin + 1);
        if (G >= 0) lim = 0;
        else if (Bme > 1 && G + (lim - 1) * (Bme - 1) >= 0) {
          const int64_t q = (-G - 1) / (Bme - 1) + 1;
          if (q < lim) lim = q;
        }
      }
    }
    // KV slack and event budget: at most C steps per member with
    // C (B_me + m_p) <= cap - used_me and C (B_p + m_me) <= cap - used_p
    // (a member that is not stepping contributes B = 0), 2 C <= budget
    const int64_t cap = PC.f.cap;
    const int64_t d1 = (int64_t)(st_me ? B : 0) + p_m, s1 = cap - L_used;
    const int64_t d2 = (int64_t)(st_p ? p_nb : 0) + L_ncopy, s2 = cap - p_used;
    int64_t C = budget > 0 ? budget >> 1 : 0;
    if (lim > 0x7fffffff) lim = 0x7fffffff;
    const int64_t p_lim = simt::shfl((int32_t)lim, y);
    int64_t want = lim > p_lim ? lim : p_lim;  // the larger member limit
    if (want > C) want = C;
    // the slack only matters up to `want` steps: divide only when it binds
    if (d1 * want > s1) { const int64_t c1 = s1 > 0 ? s1 / d1 : 0; if (c1 < C) C = c1; }
    if (d2 * want > s2) { const int64_t c2 = s2 > 0 ? s2 / d2 : 0; if (c2 < C) C = c2; }
    const bool use = pc;
    int64_t nmax = lim < C ? lim : C;
    if (!use || !st_me || nmax < 0) nmax = 0;
    if (nmax > 0x7fffffff) nmax = 0x7fffffff;
    // this member's chain, bounded by the next outside event and its own incoming
    const int32_t key = 3 * 64 + lane, pkey = 3 * 64 + y;
    double tl = pht;
    {
      const double mr = L_ni > 0 ? L_min_ready : kInf;
      bool strict = !(key < phk);
      if (mr <= tl) { tl = mr; strict = true; }
      if (!strict && tl < kInf) tl = as_f64(as_u64(tl) + 1);
    }
    double comp = 0.0, mlat = 0.0;
    if (nmax > 0) {
      comp = comp_floor(B);
      mlat = transfer_latency(PC.f, kmul((double)L_ncopy, PC.f.kvb));
    }
    // pass 0: own limits; the pair's chain ends at the earlier first untaken
    // step end, so a member whose steps reach past the partner's runs again
    // (pass 1) with that bound (LOG: every member runs pass 1, logging)
    PChain c;
    bool redo = false;
    for (int pass = 0;; ++pass) {
      if (LOG && pass == 1) c = pair_member_run<LOG>((int32_t)nmax, tl, comp, mlat, L_ncopy, B);
      else c = pair_member_run<false>((int32_t)nmax, tl, comp, mlat, L_ncopy, B);
      if (pass == 1) break;
      const double p_stop = simt::shfl(c.e, y);
      if (st_p) {  // my steps must precede the partner's stop event in (time, id) order
        const double bnd = key < pkey && p_stop < kInf ? as_f64(as_u64(p_stop) + 1) : p_stop;
        if (bnd < tl) tl = bnd;
      }
      redo = c.k > 0 && !(c.js < tl);
      if (!(LOG || redo)) break;
    }
    const int32_t kp = simt::shfl(c.k, y);
#if defined(KVSIM_EMU) && defined(KVSIM_EMU_PROFILE)
    {  // emulator-only: pairs taken here / sent to the serial loop, re-runs, steps
      auto add = [](int i, long long v) { __atomic_fetch_add(&emu_prof[i], v, __ATOMIC_RELAXED); };
      if (use && !isb) add(21, 1);
      if (use && redo) add(23, 1);
      if (use) add(24, c.k);
      if (use && !isb && st_me && st_p) add(26, 1);
      if (use && !isb) add(27, (long long)(c.k > kp ? c.k : kp));
    }
#endif
    if (!use) return;
    // commit (the ledgers only grow in a chain: the peak is the final value)
    L_used += (int64_t)c.k * B + (int64_t)kp * p_m;
    if (L_used > L_peak) L_peak = L_used;
    L_copy_tok += (int64_t)kp * p_m;
    if (c.k > 0) {
      L_busy_until = c.e; L_job_start = c.js; L_busy_time = c.busy; L_prev_end = c.js;
      L_link = c.link; L_mirror_fin = c.mfin;
      L_dG = c.dG; L_de1 = c.de1; L_dpe = c.dpe;
      L_skv += (int64_t)c.k * B;
      L_minrem -= c.k;
      if (L_kvmin != INT64_MAX) L_kvmin += c.k;
      L_dj += c.k;
      steps = c.k;
      tok = (int64_t)c.k * B;
      tw = (int64_t)c.tw * B;
      mir = (int64_t)c.k * L_ncopy;
      tmax = c.js;
    }
  }
#endif
  // drive: bitmask of lanes allowed to advance (instances; AcceLLM: any lane
  // of a pair selects the pair)
  KV_DEV_HANDLER void advance(unsigned drive) {
    const double kInf = as_f64(0x7ff0000000000000ull);
    double ht = has_next ? t_next : kInf;
    int32_t hk = -1;  // arrivals precede instance events at equal time
    if constexpr (POL == KVSIM_POLICY_SPLITWISE) {
      if (cobatch()) return;  // co-batching points run the plain event loop
      const bool all_busy = simt::ballot(lane < n_prefill && L_job == JOB_NONE) == 0;
      if (!all_busy) {
        if (get(Q_n, 0) != 0) return;
        if (simt::ballot(lane >= n_prefill && lane < n && L_final > PC.f.cap) != 0) return;
      }
      double pt = (lane < n_prefill && L_job != JOB_NONE) ? L_busy_until : kInf;
      uint32_t pku = 2 * 64 + lane;
      simt::warp_min_tk(pt, pku);
      const int32_t pk = (int32_t)pku;
      if (pt < ht || (pt == ht && pk < hk)) { ht = pt; hk = pk; }
    }
    const int64_t cap = PC.f.cap;
    const double warmup = PC.warmup;
    int64_t budget = PC.event_budget - n_events - ws()->ct.adv_events;
    int64_t steps = 0, tw = 0, mir = 0, tok = 0;
    double tmax = 0.0;
    if constexpr (POL != KVSIM_POLICY_ACCELLM) {
      bool go = ((drive >> lane) & 1) && lane < n && L_job == JOB_STEP;
      // unified: only pure decode iterations (no co-batched prefill in flight, none pending)
      if constexpr (POL == KVSIM_POLICY_UNIFIED) go = go && Q_n == 0 && L_njob == 0 && L_nb > 0;
      else go = go && lane >= n_prefill && L_nb > 0;
      if (go) {
        const int32_t B = L_nb;
        const double mr = L_ni > 0 ? L_min_ready : kInf;
        const double comp = comp_floor(B);
        const int32_t key = 3 * 64 + lane;
        // the chain runs on register copies of the lane's fields (the Sim
        // object lives in shared memory)
        const double Wb = PC.f.W, kvb = PC.f.kvb, mden = PC.f.mem_den, mrcp = PC.f.mem_rcp;
        double e = L_busy_until, js = L_job_start, busy = L_busy_time, prev = L_prev_end;
        double dG = L_dG, de1 = L_de1, dpe = L_dpe;
        const int64_t skv0 = L_skv, used0 = L_used;
        const int32_t dj0 = L_dj, minrem0 = L_minrem;
        // the integer stop tests as one trip count: no member may complete
        // (minrem >= 2), the next step's KV growth fits, the event budget
        int64_t nmax = (int64_t)minrem0 - 1;
        const int64_t room = (cap - used0) / B;
        if (room < nmax) nmax = room;
        const int64_t lim = budget < (int64_t)0x7fffffff ? budget : (int64_t)0x7fffffff;
        if (lim < nmax) nmax = lim;
        // the time tests (e < ht || (e == ht && key < hk)) && e < mr as one
        // comparison e < tl (e <= t <=> e < nextup(t) for non-negative t)
        double tl = ht;
        bool strict = !(key < hk);
        if (mr <= tl) { tl = mr; strict = true; }
        if (!strict && tl < kInf) tl = as_f64(as_u64(tl) + 1);
        double Kd = (double)skv0;  // == (double)skv at every step (exact below 2^53)
        const double Bd = (double)B;
        int64_t k = 0, ntw = 0;
        if (nmax > 0 && e < tl) {
          // first chained step: its members' gap is taken at flush (de1 / dpe)
          if (js >= warmup) busy = kadd(busy, ksub(e, js));
          if (e >= warmup) ntw += 1;
          if (dj0 == 0) { de1 = e; dpe = prev; }
          else { const double g = ksub(e, prev); if (g > dG) dG = g; }
          if constexpr (LOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
          Kd = kadd(Kd, Bd);
          if constexpr (LOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + B);
          js = e;
          const double q0 = kdiv_rcp(kadd(Wb, kmul(Kd, kvb)), mden, mrcp);
          e = kadd(e, kvsim_math::kmax(q0, comp));
          // later quotients only grow: the cheap loop-invariant acceptance test
          const double T = kdiv_chain_thr(q0, mden);
          // steady state: the step that just ended started at the previous
          // end (js == prev), so one difference is both the busy increment
          // and the members' gap. 32-bit counters (nmax < 2^31).
          const int32_t nm = (int32_t)nmax;
          int32_t k32 = 1, ntw32 = (int32_t)ntw;
          // steps that started before the measurement window
          while (k32 < nm && e < tl && js < warmup) {
            const double st = ksub(e, js);
            if (st > dG) dG = st;
            if (e >= warmup) ntw32 += 1;
            if constexpr (LOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
            Kd = kadd(Kd, Bd);
            if constexpr (LOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + (int64_t)(k32 + 1) * B);
            js = e;
            e = kadd(e, kvsim_math::kmax(kdiv_chain(kadd(Wb, kmul(Kd, kvb)), mden, mrcp, T, q0), comp));
            k32 += 1;
          }
          // inside the window (times only grow): every step adds to the busy
          // time and ends in the window
          const int32_t kw = k32;
          while (k32 < nm && e < tl) {
            const double st = ksub(e, js);
            busy = kadd(busy, st);
            if (st > dG) dG = st;
            if constexpr (LOG) log_one(e, KVSIM_EV_STEP_END, lane, B, 0, 0);
            Kd = kadd(Kd, Bd);
            if constexpr (LOG) log_one(e, KVSIM_EV_STEP_START, lane, B, 0, skv0 + (int64_t)(k32 + 1) * B);
            js = e;
            e = kadd(e, kvsim_math::kmax(kdiv_chain(kadd(Wb, kmul(Kd, kvb)), mden, mrcp, T, q0), comp));
            k32 += 1;
          }
          k = k32;
          ntw = ntw32 + (k32 - kw);
          prev = js;
          const int64_t grow = k * B;
          L_busy_until = e; L_job_start = js; L_busy_time = busy; L_prev_end = prev;
          L_dG = dG; L_de1 = de1; L_dpe = dpe;
          L_skv = skv0 + grow; L_used = used0 + grow;
          if (L_used > L_peak) L_peak = L_used;  // the ledger only grows in a chain
          L_dj = dj0 + (int32_t)k; L_minrem = minrem0 - (int32_t)k;
          steps = k;
          tmax = prev;
          tw = ntw * B;
        }
        tok = steps * B;
      }
    } else {
      // AcceLLM: the even lane of each pair drives both members in merged order
      const int pl = lane | 1;  // partner lane (valid for even lanes)
      bool pcand = false;
      {
        const int32_t pj = simt::shfl(L_job, pl), pp = simt::shfl(L_pend, pl);
        const int32_t qn = simt::shfl(Q_n, (lane >> 1) & 31);
        const int32_t pr = simt::shfl(L_role, pl);
        // a queued prompt only matters at a boundary while neither member
        // prefills (ensure_prefill); with one member in the prefill role the
        // other's boundaries ignore the queue and its prefill end bounds the chain
        const bool qok = qn == 0 || L_role == ROLE_PREFILL || pr == ROLE_PREFILL;
        const bool cand = !(lane & 1) && lane < n && (((drive >> lane) | (drive >> (lane + 1))) & 1) && qok &&
                          !L_pend && !pp && (L_job == JOB_STEP || pj == JOB_STEP);
        if (simt::ballot(cand) == 0) return;
        pcand = cand;
      }
#if KVSIM_PAIR_PAR
      // member-parallel pair chains (pair_par)
      pair_par(simt::shfl((int32_t)pcand, lane & ~1) != 0, ht, hk, budget, steps, tok, tw, mir, tmax);
#else
      MemberChain b;
      b.stepping = simt::shfl(L_job, pl) == JOB_STEP;
      const int32_t bjob = simt::shfl(L_job, pl);
      b.B = simt::shfl(L_nb, pl); b.ni = simt::shfl(L_ni, pl);
      b.e = simt::shfl(L_busy_until, pl); b.js = simt::shfl(L_job_start, pl);
      b.busy = simt::shfl(L_busy_time, pl); b.link = simt::shfl(L_link, pl);
      b.mfin = simt::shfl(L_mirror_fin, pl); b.prev = simt::shfl(L_prev_end, pl);
      b.skv = simt::shfl(L_skv, pl); b.skv_in = simt::shfl(L_skv_in, pl);
      b.used = simt::shfl(L_used, pl); b.peak = simt::shfl(L_peak, pl);
      b.copy_tok = simt::shfl(L_copy_tok, pl); b.m = simt::shfl(L_ncopy, pl);
      b.minrem = simt::shfl(L_minrem, pl); b.role = simt::shfl(L_role, pl);
      b.kvmin = simt::shfl(L_kvmin, pl); b.dj = simt::shfl(L_dj, pl);
      b.dG = simt::shfl(L_dG, pl); b.de1 = simt::shfl(L_de1, pl); b.dpe = simt::shfl(L_dpe, pl);
      const double bmr = simt::shfl(L_min_ready, pl);
      const int32_t bpend = simt::shfl(L_pend, pl);
      const int32_t qn_pair = simt::shfl(Q_n, (lane >> 1) & 31);
      const int32_t bcompB = simt::shfl(L_compB, pl);
      const double bcomp = simt::shfl(L_comp, pl);
      b.mr = b.ni > 0 ? bmr : kInf;
      b.tw = 0; b.steps = 0; b.Kd = (double)b.skv;
      const bool drv = !(lane & 1) && lane < n && (((drive >> lane) | (drive >> (lane + 1))) & 1) &&
                       (qn_pair == 0 || L_role == ROLE_PREFILL || b.role == ROLE_PREFILL) &&
                       !L_pend && !bpend && (L_job == JOB_STEP || b.stepping);
      MemberChain a;
      a.stepping = L_job == JOB_STEP;
      a.B = L_nb; a.ni = L_ni; a.e = L_busy_until; a.js = L_job_start; a.busy = L_busy_time; a.link = L_link;
      a.mfin = L_mirror_fin; a.prev = L_prev_end; a.skv = L_skv; a.skv_in = L_skv_in; a.used = L_used;
      a.peak = L_peak; a.copy_tok = L_copy_tok; a.m = L_ncopy; a.minrem = L_minrem; a.role = L_role;
      a.kvmin = L_kvmin; a.dj = L_dj; a.dG = L_dG; a.de1 = L_de1; a.dpe = L_dpe;
      a.mr = L_ni > 0 ? L_min_ready : kInf;
      a.tw = 0; a.steps = 0; a.Kd = (double)a.skv;
      constexpr int64_t kOff = INT64_MIN / 4;  // rebalance test disabled
      int64_t GA = kOff, GB = kOff, SA = 0, SB = 0;
      int32_t rA = 0, rB = 0;
      double tlA = -1.0, tlB = -1.0;
      if (drv) {
        double pht = ht;
        int32_t phk = hk;
        if (!b.stepping) {  // the idle / prefilling partner's own next event bounds the chain
          double yt = kInf;
          int32_t yk = 0;
          if (bjob == JOB_PREFILL) { yt = b.e; yk = 2 * 64 + lane + 1; }
          else if (b.role == ROLE_DECODE && b.ni > 0) { yt = bmr; yk = 64 + lane + 1; }
          if (yt < pht || (yt == pht && yk < phk)) { pht = yt; phk = yk; }
          b.e = kInf;
        }
        if (!a.stepping) {
          double yt = kInf;
          int32_t yk = 0;
          if (L_job == JOB_PREFILL) { yt = a.e; yk = 2 * 64 + lane; }
          else if (a.role == ROLE_DECODE && a.ni > 0) { yt = L_min_ready; yk = 64 + lane; }
          if (yt < pht || (yt == pht && yk < phk)) { pht = yt; phk = yk; }
          a.e = kInf;
        }
        a.comp = a.stepping ? comp_floor(a.B) : 0.0;
        b.comp = b.stepping ? (bcompB == b.B ? bcomp : kdiv(kmul(PC.f.two_p, (double)b.B), PC.f.pf_den)) : 0.0;
        a.mlat = transfer_latency(PC.f, kmul((double)a.m, PC.f.kvb));
        b.mlat = transfer_latency(PC.f, kmul((double)b.m, PC.f.kvb));
        if (!a.stepping) a.B = 0;
        const ChainK K{PC.f.W, PC.f.kvb, PC.f.mem_den, PC.f.mem_rcp, warmup, cap};
        // Incremental form of pair_step's stop tests: remaining-token and
        // event budgets as counters, KV slack per member (own steps take B,
        // the partner's steps take its mirror lines m), and the rebalance
        // test as a gap G = lim - (kvmin + 1) that grows by B - 1 per own
        // step and shrinks by the partner's B per partner step (stop at
        // G >= 0). The KV ledgers are applied once after the loop (they only
        // grow during a chain, so the peaks are the final values).
        GA = kOff; GB = kOff;
        {
          const int64_t cza = (int64_t)a.B + a.ni - b.B - b.ni, czb = (int64_t)b.B + b.ni - a.B - a.ni;
          const int64_t dza = (a.skv + a.skv_in + a.B) - (b.skv + b.skv_in);
          const int64_t dzb = (b.skv + b.skv_in + b.B) - (a.skv + a.skv_in);
          if (b.role == ROLE_DECODE && a.kvmin != INT64_MAX && cza >= 1) GA = (cza >= 2 ? dza : dza - 1) - (a.kvmin + 1);
          if (a.role == ROLE_DECODE && b.kvmin != INT64_MAX && czb >= 1) GB = (czb >= 2 ? dzb : dzb - 1) - (b.kvmin + 1);
        }
        SA = cap - a.used; SB = cap - b.used;
        rA = a.minrem - 1; rB = b.minrem - 1;
        const int32_t kA = 3 * 64 + lane, kB = kA + 1;
        // per member, (e < pht || (e == pht && key < phk)) && e < mr as one
        // comparison e < tl (e <= t <=> e < nextup(t) for non-negative t)
        auto tlim = [&](int32_t key, double mr) {
          double tl = pht;
          bool strict = !(key < phk);
          if (mr <= tl) { tl = mr; strict = true; }
          if (!strict && tl < kInf) tl = as_f64(as_u64(tl) + 1);
          return tl;
        };
        tlA = tlim(kA, a.mr);
        tlB = b.stepping ? tlim(kB, b.mr) : -1.0;
        {
          for (;;) {
            if (a.stepping && (!b.stepping || !(b.e < a.e))) {  // ties: lower id (even lane)
              if (!(a.e < tlA) || rA <= 0 || budget <= 0 || GA >= 0 || SA < a.B || SB < a.m) break;
              lean_step(a, K, lane);
              rA -= 1; SA -= a.B; SB -= a.m; GA += a.B - 1; GB -= a.B;
            } else {
              if (!(b.e < tlB) || rB <= 0 || budget <= 0 || GB >= 0 || SB < b.B || SA < b.m) break;
              lean_step(b, K, lane + 1);
              rB -= 1; SB -= b.B; SA -= b.m; GB += b.B - 1; GA -= b.B;
            }
            budget -= 1;
          }
        }
      }
      if (drv) {
        {
          const int64_t ua = (int64_t)a.steps * a.B + (int64_t)b.steps * b.m;
          const int64_t ub = (int64_t)b.steps * b.B + (int64_t)a.steps * a.m;
          a.used += ua; b.used += ub;
          a.copy_tok += (int64_t)b.steps * b.m; b.copy_tok += (int64_t)a.steps * a.m;
          if (a.used > a.peak) a.peak = a.used;
          if (b.used > b.peak) b.peak = b.used;
          a.minrem -= a.steps; b.minrem -= b.steps;
          if (a.kvmin != INT64_MAX) a.kvmin += a.steps;
          if (b.kvmin != INT64_MAX) b.kvmin += b.steps;
          a.skv += (int64_t)a.steps * a.B; b.skv += (int64_t)b.steps * b.B;
          a.tw *= a.B; b.tw *= b.B;
        }
        if (!a.stepping) a.B = L_nb;
        steps = a.steps + b.steps;
#if defined(KVSIM_EMU) && defined(KVSIM_EMU_PROFILE)
        __atomic_fetch_add(&emu_prof[25], (long long)steps, __ATOMIC_RELAXED);
#endif
        tok = (int64_t)a.steps * a.B + (int64_t)b.steps * b.B;
        tw = a.tw + b.tw;
        mir = (int64_t)a.steps * a.m + (int64_t)b.steps * b.m;
        tmax = a.prev > b.prev ? a.prev : b.prev;
        // commit the driver's member
        L_busy_until = a.stepping ? a.e : L_busy_until; L_job_start = a.js; L_busy_time = a.busy;
        L_link = a.link; L_mirror_fin = a.mfin; L_prev_end = a.prev; L_skv = a.skv; L_used = a.used;
        L_peak = a.peak; L_copy_tok = a.copy_tok; L_minrem = a.minrem; L_kvmin = a.kvmin; L_dj = a.dj;
        L_dG = a.dG; L_de1 = a.de1; L_dpe = a.dpe;
      }
      // scatter the partner member back to the odd lanes
      const int dl = lane & ~1;
      const bool got = simt::shfl((int32_t)drv, dl) != 0;
      const double be = simt::shfl(b.e, dl), bjs = simt::shfl(b.js, dl), bbusy = simt::shfl(b.busy, dl);
      const double blink = simt::shfl(b.link, dl), bmfin = simt::shfl(b.mfin, dl), bprev = simt::shfl(b.prev, dl);
      const double bdG = simt::shfl(b.dG, dl), bde1 = simt::shfl(b.de1, dl), bdpe = simt::shfl(b.dpe, dl);
      const int64_t bskv = simt::shfl(b.skv, dl), bused = simt::shfl(b.used, dl), bpeak = simt::shfl(b.peak, dl);
      const int64_t bct = simt::shfl(b.copy_tok, dl), bkv = simt::shfl(b.kvmin, dl);
      const int32_t bmin = simt::shfl(b.minrem, dl), bdj = simt::shfl(b.dj, dl);
      const bool bst = simt::shfl((int32_t)b.stepping, dl) != 0;
      if ((lane & 1) && got) {
        if (bst) { L_busy_until = be; L_job_start = bjs; L_busy_time = bbusy; L_link = blink; L_mirror_fin = bmfin;
                   L_prev_end = bprev; L_skv = bskv; L_minrem = bmin; L_kvmin = bkv; L_dj = bdj; L_dG = bdG;
                   L_de1 = bde1; L_dpe = bdpe; }
        L_used = bused;
        L_peak = bpeak;
        L_copy_tok = bct;
      }
#endif
    }
    const unsigned am = simt::ballot(steps > 0);
    if (am != 0 && (am & (am - 1)) == 0) {  // one chain advanced (the common case): plain adds
      if (steps > 0) {
        Counters& ct = ws()->ct;
        ct.adv_events += steps;
        ct.n_steps += steps;
        ct.tok_total += tok;
        ct.tok_window += tw;
        ct.mir_tokens += mir;
        if (tmax > L_tlast) L_tlast = tmax;
      }
    } else if (steps > 0) {  // divergent: only lanes that advanced touch the counters
      simt::atomic_add_smem(&ws()->ct.adv_events, steps);
      simt::atomic_add_smem(&ws()->ct.n_steps, steps);
      simt::atomic_add_smem(&ws()->ct.tok_total, tok);
      simt::atomic_add_smem(&ws()->ct.tok_window, tw);
      if (mir) simt::atomic_add_smem(&ws()->ct.mir_tokens, mir);
      if (tmax > L_tlast) L_tlast = tmax;
    }
    simt::sync();
  }
  // ------------------------------------------------------------- unified
  KV_DEV_HANDLER void unified_start(int x, double t) {
    EMU_COUNT(17);
    int32_t nb = get(L_nb, x);
    while (get(L_used, x) + nb > PC.f.cap) {
      preempt_newest(x);
      nb -= 1;
    }
    add_used(x, nb);
    const int64_t K = get(L_skv, x);
    // FCFS admission under PC.budget and memory (prefix-closed tests)
    const int32_t h = get(Q_head, x), qn = get(Q_n, x);
    int64_t used = get(L_used, x);
    int32_t k = 0;
    int64_t s1 = 0, s2 = 0;
    while (k < qn) {
      const int32_t i = k + lane;
      const bool valid = i < qn;
      int32_t rid = 0;
      int64_t len = 0;
      if (valid) { rid = q_at(x, h, i); len = c_qlen()[rid]; }
      const int64_t incl = simt::warp_incl_scan(len);
      const bool okb = (k == 0 && lane == 0) || s1 + incl <= PC.budget;
      const bool okm = used + incl <= PC.f.cap;
      const unsigned fail = simt::ballot(valid && !(okb && okm));
      const int32_t nvalid = simt::popc(simt::ballot(valid));
      const int32_t take = fail ? simt::ffs(fail) - 1 : nvalid;
      if (lane < take) {
        j_rid(x)[k + lane] = rid;
        if (c_em()[rid] == 0) c_qs()[rid] = t;
      }
      const int64_t tsum = take > 0 ? simt::shfl(incl, take - 1) : 0;
      const int64_t tsq = simt::warp_sum_nn(lane < take ? len * len : (int64_t)0);
      s1 += tsum;
      s2 += tsq;
      used += tsum;
      k += take;
      if (take < nvalid || fail) break;
    }
    simt::sync();
    if (k > 0) {
      q_pop(x, k, s1);
      add_used(x, s1);
    }
    if (nb == 0 && k == 0) return;
    const double lat = kadd(k ? prefill_latency(PC.f, s1, s2) : 0.0, nb ? decode_latency(PC.f, nb, K) : 0.0);
    job_begin(x, t);
    if (own(x)) {
      L_job = JOB_STEP;
      L_job_start = t;
      L_busy_until = kadd(t, lat);
      L_njob = k;
      L_job_s1 = s1;
    }
    log(KVSIM_EV_STEP_START, x, nb, k, K);

  }

  // ------------------------------------------- splitwise high-load co-batching
  // while a prompt waits and every prefill instance is busy, a decode
  // iteration also prefills queued prompts (SEMANTICS §6 splitwise)
  KV_DEV bool sw_overflow() {
    return get(Q_n, 0) > 0 && simt::ballot(lane < n_prefill && L_job == JOB_NONE) == 0;
  }
  KV_DEV_NOINLINE void sw_cobatch_start(int x, double t) {
    int32_t nb = get(L_nb, x);
    if (nb == 0 && !sw_overflow()) return;
    while (get(L_used, x) + nb > PC.f.cap) {
      preempt_newest(x);
      nb -= 1;
    }
    add_used(x, nb);
    const int64_t K = get(L_skv, x);
    int32_t k = 0;
    int64_t s1 = 0, s2 = 0;
    if (sw_overflow()) {
      const int32_t h = get(Q_head, 0), qn = get(Q_n, 0);
      int64_t used = get(L_used, x);
      while (k < qn) {
        const int32_t i = k + lane;
        const bool valid = i < qn;
        int32_t rid = 0;
        int64_t len = 0;
        if (valid) { rid = q_at(0, h, i); len = c_qlen()[rid]; }
        const int64_t incl = simt::warp_incl_scan(len);
        const bool okb = (k == 0 && lane == 0) || s1 + incl <= PC.budget;
        const bool okm = used + incl <= PC.f.cap;
        const unsigned fail = simt::ballot(valid && !(okb && okm));
        const int32_t nvalid = simt::popc(simt::ballot(valid));
        const int32_t take = fail ? simt::ffs(fail) - 1 : nvalid;
        if (lane < take) {
          j_rid(x)[k + lane] = rid;
          if (c_em()[rid] == 0) c_qs()[rid] = t;
        }
        const int64_t tsum = take > 0 ? simt::shfl(incl, take - 1) : 0;
        const int64_t tsq = simt::warp_sum_nn(lane < take ? len * len : (int64_t)0);
        s1 += tsum;
        s2 += tsq;
        used += tsum;
        k += take;
        if (take < nvalid || fail) break;
      }
      simt::sync();
      if (k > 0) {
        q_pop(0, k, s1);
        add_used(x, s1);
      }
    }
    if (nb == 0 && k == 0) return;
    const double lat = kadd(k ? prefill_latency(PC.f, s1, s2) : 0.0, nb ? decode_latency(PC.f, nb, K) : 0.0);
    job_begin(x, t);
    if (own(x)) {
      L_job = JOB_STEP;
      L_job_start = t;
      L_busy_until = kadd(t, lat);
      L_njob = k;
      L_job_s1 = s1;
    }
    log(KVSIM_EV_STEP_START, x, nb, k, K);
  }

  KV_DEV_HANDLER void unified_end(int x, double t) {
    EMU_COUNT(18);
    account_job(x, t);
    if (lane == 0) ws()->ct.n_steps += 1;
    const StepOut o = step_loop(x, t);  // applies the deferred chained steps too
    int32_t nb = o.nb_old - o.completed;
    int64_t skv = get(L_skv, x) - o.kv_done + nb;
    int64_t freed = o.kv_done + o.completed;
    count_tokens(o.nb_old, t);
    // co-batched prefills emit and join (non-joiners: their last token is t)
    const int32_t k = get(L_njob, x);
    int32_t completed = o.completed, add = 0, minrem = o.minrem;
    int64_t kvadd = 0, kvfree = 0;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      int32_t rid = 0, em = 0, dl = 0, pl = 0;
      if (act) {
        rid = j_rid(x)[i];
        em = emit_prefill_token(rid, t);
        dl = c_dl()[rid];
        pl = c_pl()[rid];
      }
      const bool done = act && em == dl;
      const bool join = act && !done;
      if (done) { c_done()[rid] = t; kvfree += (int64_t)pl + em + kvo(); }
      const unsigned jm = simt::ballot(join);
      if (join) {
        const int32_t pos = nb + add + simt::popc(jm & simt::lanemask_lt());
        b_rid(x)[pos] = rid;
        // (ft: the prefill emitted nothing, so the last token, if any, predates it)
        b_rem(x)[pos] = (dl - em) | (ft() ? kJoin : 0) | (em == 0 ? kFirst : 0);
        b_kvb(x)[pos] = pl + dl + kvo();
        b_tbt(x)[pos] = c_tbt()[rid];
        kvadd += (int64_t)pl + em + kvo();
        if (dl - em < minrem) minrem = dl - em;
      }
      add += simt::popc(jm);
      completed += simt::popc(simt::ballot(done));
    }
    kvadd = simt::warp_sum_nn(kvadd);
    kvfree = simt::warp_sum_nn(kvfree);
    minrem = simt::warp_min_i32(minrem);
    simt::sync();
    count_tokens(ft() ? 0 : k, t);
    if (k > 0) if (lane == 0) ws()->ct.n_prefills += 1;
    if (own(x)) {
      L_job = JOB_NONE;
      L_used -= freed + kvfree;
      L_skv = skv + kvadd;
      L_nb = nb + add;
      L_prev_end = t;
      L_njob = 0;
      L_minrem = minrem;
    }
    log(KVSIM_EV_STEP_END, x, o.nb_old, completed, 0);
    if constexpr (POL == KVSIM_POLICY_UNIFIED) unified_start(x, t);
  }

  // ------------------------------------------------------------ splitwise
  KV_DEV_HANDLER void sw_try_start(double t) {
    EMU_COUNT(19);
    for (int p = 0; p < n_prefill; ++p) {
      if (get(L_job, p) != JOB_NONE) continue;
      int32_t qn = get(Q_n, 0);
      if (qn == 0) continue;
      const int32_t h = get(Q_head, 0);
      int32_t k = 0;
      int64_t s1 = 0, s2 = 0;
      bool stop = false;
      while (!stop && k < qn) {
        // prefetch a chunk of queue entries into lanes
        const int32_t i = k + lane;
        const bool valid = i < qn;
        int32_t crid = 0, clen = 0;
        if (valid) { crid = q_at(0, h, i); clen = c_qlen()[crid]; }
        const int32_t nvalid = simt::popc(simt::ballot(valid));
        for (int32_t c = 0; c < nvalid; ++c) {
          const int32_t rid = simt::shfl(crid, c);
          const int64_t len = simt::shfl(clen, c);
          if (k > 0 && s1 + len > PC.budget) { stop = true; break; }
          // destination: decode instance with most free tokens, ties lowest id
          int64_t fr = (lane >= n_prefill && lane < n) ? PC.f.cap - L_used : INT64_MIN;
          const int64_t best = simt::warp_max_i64(fr);
          const int d = simt::ffs(simt::ballot(fr == best)) - 1;
          if (best < len) { stop = true; break; }
          if (get(L_used, p) + s1 + len > PC.f.cap) { stop = true; break; }  // p holds the job's prompts
          add_used(d, len);
          if (lane == 0) {
            j_rid(p)[k] = rid;
            j_dst(p)[k] = d;
            if (c_em()[rid] == 0) c_qs()[rid] = t;
          }
          s1 += len;
          s2 += len * len;
          k += 1;
        }
      }
      simt::sync();
      if (k == 0) continue;
      q_pop(0, k, s1);
      add_used(p, s1);
      const double lat = prefill_latency(PC.f, s1, s2);
      job_begin(p, t);
      if (own(p)) {
        L_job = JOB_PREFILL;
        L_job_start = t;
        L_busy_until = kadd(t, lat);
        L_njob = k;
        L_job_s1 = s1;
      }
      log(KVSIM_EV_PREFILL_START, p, k, j_rid(p)[0], s1);
    }
    if (cobatch())  // idle decode instances (ascending id) take overflow prompts
      for (int d = n_prefill; d < n && sw_overflow(); ++d)
        if (get(L_job, d) == JOB_NONE) sw_cobatch_start(d, t);
  }

  KV_DEV_HANDLER void sw_prefill_done(int p, double t) {
    EMU_COUNT(20);
    account_job(p, t);
    if (lane == 0) ws()->ct.n_prefills += 1;
    const int32_t k = get(L_njob, p);
    const int64_t s1 = get(L_job_s1, p);
    const double jstart = get(L_job_start, p);
    if (own(p)) { L_job = JOB_NONE; L_used -= s1; }
    if (lane < kMaxInst) { ws()->acc_a[lane] = 0; ws()->acc_b[lane] = 0; ws()->cnt[lane] = 0; }
    simt::sync();
    int32_t completed = 0;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      bool done = false;
      if (act) {
        const int32_t rid = j_rid(p)[i];
        const int32_t d = j_dst(p)[i];
        const int32_t em = emit_prefill_token(rid, t);
        const int32_t dl = c_dl()[rid];
        const int64_t kv = (int64_t)c_pl()[rid] + em + kvo();
        done = em == dl;
        if (done) {
          c_done()[rid] = t;
          simt::atomic_add_smem(&ws()->acc_b[d], kv);
        } else {
          simt::atomic_add_smem(&ws()->acc_a[d], kv);
          simt::atomic_add_smem(&ws()->cnt[d], 1);
        }
      }
      completed += simt::popc(simt::ballot(done));
    }
    simt::sync();
    count_tokens(ft() ? 0 : k, t);
    log(KVSIM_EV_PREFILL_DONE, p, k, completed, 0);
    // one transfer per destination, ascending id; lane d keeps the finish time
    double fin_mine = 0.0;
    int32_t base_mine = 0;
    for (int d = n_prefill; d < n; ++d) {
      const int64_t tok = ws()->acc_a[d];
      const int64_t fr = ws()->acc_b[d];
      if (own(d)) { L_used -= fr; }
      if (tok == 0) continue;
      const double fin = prefill_transfer(p, d, tok, jstart, t);
      if (own(d)) {
        fin_mine = fin;
        base_mine = L_ni;
        L_ni += ws()->cnt[d];
        L_skv_in += tok;
        if (fin < L_min_ready) L_min_ready = fin;
      }
    }
    simt::sync();
    if (lane < kMaxInst) { ws()->cnt[lane] = 0; ws()->acc_b[lane] = 0; }
    simt::sync();
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      int32_t rid = 0, d = 0;
      if (act) { rid = j_rid(p)[i]; d = j_dst(p)[i]; }
      const double fin_d = simt::shfl(fin_mine, d);
      const int32_t base_d = simt::shfl(base_mine, d);
      if (act && c_em()[rid] != c_dl()[rid]) {
        const int32_t pos = base_d + simt::atomic_add_smem(&ws()->cnt[d], 1);
        i_rid(d)[pos] = rid;
        i_ready(d)[pos] = fin_d;
        c_cpy()[rid] = -1;
        simt::atomic_add_smem(&ws()->acc_b[d], (int64_t)c_pl()[rid] + c_dl()[rid] + kvo());
      }
    }
    simt::sync();
    if (lane >= n_prefill && lane < n) L_final += ws()->acc_b[lane];
    simt::sync();
  }

  // -------------------------------------------------------------- accellm
  KV_DEV int64_t load_of(int x) { return get(L_skv, x) + get(L_skv_in, x); }
  KV_DEV bool head_admissible(int x) {
    const int q = qid(x >> 1);
    if (get(Q_n, q) == 0) return false;
    const int32_t rid = q_at(q, get(Q_head, q), 0);
    const int64_t len = c_qlen()[rid];
    return get(L_used, x) - get(L_copy_tok, x) + len <= PC.f.cap;
  }
  // move every request whose primary is x and that holds a copy on x^1
  KV_DEV_HANDLER void move_all_to_partner(int x, double t) {
    EMU_COUNT(8);
    const int y = partner_of(x);
    if (y < 0) return;  // a degraded group's dual instance: its requests stall
    flush(x);
    const double mfin = get(L_mirror_fin, x);
    const double pend = get(L_prev_end, x);
    int32_t nb = get(L_nb, x);
    int32_t ni_y = get(L_ni, y);
    int32_t keep = 0, moved = 0;
    int64_t kv_moved = 0;
    double mn = as_f64(0x7ff0000000000000ull);
    // batch members
    for (int32_t j0 = 0; j0 < nb; j0 += 32) {
      const int32_t j = j0 + lane;
      const bool act = j < nb;
      int32_t rid = 0, rf = 0, kvb = 0;
      double tb = 0.0;
      if (act) { rid = b_rid(x)[j]; rf = b_rem(x)[j]; kvb = b_kvb(x)[j]; tb = b_tbt(x)[j]; }
      const bool mv = act && (rf & kCopy);
      const bool st = act && !mv;
      const unsigned mm = simt::ballot(mv), sm = simt::ballot(st);
      simt::sync();
      if (st) {
        const int32_t k = keep + simt::popc(sm & simt::lanemask_lt());
        b_rid(x)[k] = rid; b_rem(x)[k] = rf; b_kvb(x)[k] = kvb; b_tbt(x)[k] = tb;
      }
      if (mv) {
        const int32_t rem = rf & kRemMask;
        const bool joiner = (rf & kJoin) != 0;
        const double fresh = joiner ? c_fresh()[rid] : mfin;
        const double ready = fresh > t ? fresh : t;
        const int32_t dl = c_dl()[rid];
        c_em()[rid] = dl - rem;
        c_tbt()[rid] = tb;
        if (!joiner) c_last()[rid] = pend;
        c_cpy()[rid] = x;
        c_fresh()[rid] = t;
        c_nmv()[rid] += 1;
        const int32_t pos = ni_y + moved + simt::popc(mm & simt::lanemask_lt());
        i_rid(y)[pos] = rid;
        i_ready(y)[pos] = ready;
        kv_moved += (int64_t)kvb - rem;
        if (ready < mn) mn = ready;
      }
      log_lanes(mv, KVSIM_EV_MOVE, x, rid, y, 0);
      keep += simt::popc(sm);
      moved += simt::popc(mm);
    }
    const int32_t moved_b = moved;
    const int64_t kv_b = simt::warp_sum_nn(kv_moved);
    kv_moved = 0;
    // incoming entries of x that hold a copy on y
    const int32_t ni = get(L_ni, x);
    int32_t ikeep = 0;
    for (int32_t j0 = 0; j0 < ni; j0 += 32) {
      const int32_t j = j0 + lane;
      const bool act = j < ni;
      int32_t rid = 0;
      double rd = 0.0;
      if (act) { rid = i_rid(x)[j]; rd = i_ready(x)[j]; }
      const bool mv = act && c_cpy()[act ? rid : 0] == y;
      const bool st = act && !mv;
      const unsigned mm = simt::ballot(mv), sm = simt::ballot(st);
      simt::sync();
      if (st) {
        const int32_t k = ikeep + simt::popc(sm & simt::lanemask_lt());
        i_rid(x)[k] = rid;
        i_ready(x)[k] = rd;
      }
      if (mv) {
        const double fresh = c_fresh()[rid];
        const double ready = fresh > t ? fresh : t;
        c_cpy()[rid] = x;
        c_fresh()[rid] = t;
        c_nmv()[rid] += 1;
        const int32_t pos = ni_y + moved + simt::popc(mm & simt::lanemask_lt());
        i_rid(y)[pos] = rid;
        i_ready(y)[pos] = ready;
        kv_moved += (int64_t)c_pl()[rid] + c_em()[rid] + kvo();
        if (ready < mn) mn = ready;
      }
      log_lanes(mv, KVSIM_EV_MOVE, x, rid, y, 0);
      ikeep += simt::popc(sm);
      moved += simt::popc(mm);
    }
    const int64_t kv_i = simt::warp_sum_nn(kv_moved);
    mn = warp_min_time(mn);
    // min ready of what stays in x's incoming
    double mx = as_f64(0x7ff0000000000000ull);
    for (int32_t j = lane; j < ikeep; j += 32) {
      const double r = i_ready(x)[j];
      if (r < mx) mx = r;
    }
    mx = warp_min_time(mx);
    simt::sync();
    const int64_t kv_all = kv_b + kv_i;
    if (lane == 0) ws()->ct.n_moves += moved;
    if (own(x)) {
      L_nb = keep;
      L_ni = ikeep;
      L_skv -= kv_b;
      L_skv_in -= kv_i;
      L_ncopy -= moved_b;
      L_copy_tok += kv_all;
      L_min_ready = mx;
    }
    if (own(y)) {
      L_ni += moved;
      L_skv_in += kv_all;
      L_copy_tok -= kv_all;
      if (mn < L_min_ready) L_min_ready = mn;
    }
  }

  KV_DEV_HANDLER void acc_start_job(int x, double t) {
    EMU_COUNT(13);
    const int q = qid(x >> 1);
    const int32_t h = get(Q_head, q);
    int32_t k = 0;
    int64_t s1 = 0, s2 = 0;
    for (;;) {
      const int32_t qn = get(Q_n, q);
      if (k >= qn) break;
      const int32_t i = k + lane;
      const bool valid = i < qn;
      int32_t rid = 0;
      int64_t len = 0;
      if (valid) { rid = q_at(q, h, i); len = c_qlen()[rid]; }
      const int64_t incl = simt::warp_incl_scan(len);
      const int64_t used = get(L_used, x);
      const bool okb = (k == 0 && lane == 0) || s1 + incl <= PC.budget;
      const bool okm = used + incl <= PC.f.cap;
      const unsigned fail = simt::ballot(valid && !(okb && okm));
      const int32_t nvalid = simt::popc(simt::ballot(valid));
      const int32_t take = fail ? simt::ffs(fail) - 1 : nvalid;
      if (lane < take) {
        j_rid(x)[k + lane] = rid;
        if (c_em()[rid] == 0) c_qs()[rid] = t;
      }
      const int64_t tsum = take > 0 ? simt::shfl(incl, take - 1) : 0;
      const int64_t tsq = simt::warp_sum_nn(lane < take ? len * len : (int64_t)0);
      s1 += tsum;
      s2 += tsq;
      k += take;
      add_used(x, tsum);
      if (!fail) continue;
      const int f0 = simt::ffs(fail) - 1;
      const bool fb = simt::shfl((int32_t)okb, f0) != 0;
      const int64_t lenf = simt::shfl(len, f0);
      if (!fb) break;
      // memory: evict copies held on x, largest first
      while (get(L_used, x) + lenf > PC.f.cap) {
        Found v = largest_copy_on(x);
        if (!v.where) break;
        evict(x, v);
      }
      if (get(L_used, x) + lenf > PC.f.cap) break;
    }
    simt::sync();
    q_pop(q, k, s1);
    const double lat = prefill_latency(PC.f, s1, s2);
    job_begin(x, t);
    if (own(x)) {
      L_job = JOB_PREFILL;
      L_job_start = t;
      L_busy_until = kadd(t, lat);
      L_njob = k;
      L_job_s1 = s1;
    }
    log(KVSIM_EV_PREFILL_START, x, k, k ? j_rid(x)[0] : -1, s1);
  }

  KV_DEV_HANDLER bool try_switch(int x, double t) {
    EMU_COUNT(12);
    if (!head_admissible(x)) return false;
    if (own(x)) L_pend = 0;
    move_all_to_partner(x, t);
    if (own(x)) L_role = ROLE_PREFILL;
    log(KVSIM_EV_ROLE, x, ROLE_PREFILL, 0, 0);
    acc_start_job(x, t);
    return true;
  }

  KV_DEV void ensure_prefill(int q, double t) {
    if (get(Q_n, q) == 0) return;
    ensure_prefill_slow(q, t);
  }
  KV_DEV_HANDLER void ensure_prefill_slow(int q, double t) {
    EMU_COUNT(11);
    if (get(Q_n, q) == 0) return;
    if (degraded_pair(q)) {  // the dual instance is the group's only prefill instance
      const int d = 4 * (q >> 1);
      if (get(L_role, d) == ROLE_PREFILL || get(L_pend, d)) return;
      if (get(L_job, d) == JOB_NONE) try_switch(d, t);
      else if (own(d)) L_pend = 1;
      return;
    }
    const int a = 2 * q, b = a + 1;
    if (get(L_role, a) == ROLE_PREFILL || get(L_role, b) == ROLE_PREFILL || get(L_pend, a) || get(L_pend, b))
      return;
    const int m = load_of(b) < load_of(a) ? b : a;
    if (get(L_job, m) == JOB_NONE) try_switch(m, t);
    else if (own(m)) L_pend = 1;
  }

  // rebalance_pair at x's boundary (SEMANTICS §6)
  KV_DEV void rebalance(int x, double t) {
    if constexpr (EXT) {
      if (degraded_pair(x >> 1)) {
        if ((x & 3) != 0) dual_push(x, t);
        return;
      }
    }
    const int y = x ^ 1;
    if (get(L_role, y) != ROLE_DECODE || get(L_pend, y)) return;
    const int64_t c = (int64_t)get(L_nb, x) + get(L_ni, x) - get(L_nb, y) - get(L_ni, y);
    if (c < 1) return;
    if (load_of(x) - load_of(y) < 1) return;
    rebalance_slow(x, t);
  }
  KV_DEV_HANDLER void rebalance_slow(int x, double t) {
    EMU_COUNT(6);
    flush(x);
    const int y = x ^ 1;
    if (get(L_role, y) != ROLE_DECODE || get(L_pend, y)) return;
    int64_t c = (int64_t)get(L_nb, x) + get(L_ni, x) - get(L_nb, y) - get(L_ni, y);
    int64_t d = load_of(x) - load_of(y);
    while (c >= 1 && d >= 1) {
      // largest candidate (kv desc, rid asc) with kv <= d (kv < d when c == 1)
      const int64_t lim = c >= 2 ? d : d - 1;
      const int32_t nb = get(L_nb, x);
      uint64_t best = 0;
      int32_t bidx = -1;
      for (int32_t j = lane; j < nb; j += 32) {
        const int32_t rf = b_rem(x)[j];
        if ((rf & (kCopy | kSettle)) == kCopy) {
          const int64_t kv = (int64_t)b_kvb(x)[j] - (rf & kRemMask);
          if (kv <= lim) {
            const uint64_t kk = ((uint64_t)kv << 32) | (uint32_t)(0x7fffffff - b_rid(x)[j]);
            if (kk > best) { best = kk; bidx = j; }
          }
        }
      }
      const uint64_t wb = simt::warp_max_u64(best);
      if (wb == 0) break;
      const int src = simt::ffs(simt::ballot(best == wb)) - 1;
      const int32_t idx = simt::shfl(bidx, src);
      const int64_t kv = (int64_t)(wb >> 32);
      move_one(x, idx, t);
      c -= 2;
      d -= 2 * kv;
    }
  }
  // move batch slot idx of x to y's incoming (zero-byte label swap)
  KV_DEV_HANDLER void move_one(int x, int32_t idx, double t) {
    EMU_COUNT(7);
    const int y = x ^ 1;
    const int32_t rid = b_rid(x)[idx];
    const int32_t rf = b_rem(x)[idx];
    const int32_t rem = rf & kRemMask;
    const int64_t kv = (int64_t)b_kvb(x)[idx] - rem;
    const double tb = b_tbt(x)[idx];
    const bool joiner = (rf & kJoin) != 0;
    const double fresh = joiner ? c_fresh()[rid] : get(L_mirror_fin, x);
    const double ready = fresh > t ? fresh : t;
    const double last = joiner ? c_last()[rid] : get(L_prev_end, x);
    const int32_t dl = c_dl()[rid];
    simt::sync();
    if (lane == 0) {
      c_em()[rid] = dl - rem;
      c_tbt()[rid] = tb;
      c_last()[rid] = last;
      c_cpy()[rid] = x;
      c_fresh()[rid] = t;
      c_nmv()[rid] += 1;
    }
    batch_remove(x, idx);
    incoming_append(y, rid, ready);
    if (own(x)) { L_skv -= kv; L_ncopy -= 1; L_copy_tok += kv; }
    if (own(y)) { L_skv_in += kv; L_copy_tok -= kv; }
    if (lane == 0) ws()->ct.n_moves += 1;
    log(KVSIM_EV_MOVE, x, rid, y, 0);
  }

  KV_DEV_HANDLER void acc_boundary(int x, double t) {
    EMU_COUNT(9);
    if constexpr (EXT) {
      if (own(x) && L_lvl_hold > 0 && t >= L_lvl_until) { L_used -= L_lvl_hold; L_lvl_hold = 0; }
    }
    join(x, t);
    if (get(L_pend, x)) {
      if (own(x)) L_pend = 0;
      if (try_switch(x, t)) return;
    }
    ensure_prefill(qid(x >> 1), t);
    if (get(L_role, x) == ROLE_PREFILL) return;
    if constexpr (EXT) {
      if (get(L_lvl_dst, x) >= 0) level_from(x, t);
    }
    rebalance(x, t);
    step_start(x, t);
  }

  KV_DEV_HANDLER void acc_prefill_done(int x, double t) {
    EMU_COUNT(10);
    flush(x);
    account_job(x, t);
    if (lane == 0) ws()->ct.n_prefills += 1;
    const int y = x ^ 1;
    const int32_t k = get(L_njob, x);
    const double jstart = get(L_job_start, x);
    if (own(x)) L_job = JOB_NONE;
    // pass 1: emission, completions; survivors' kv
    int32_t completed = 0;
    int64_t kvfree = 0;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      bool done = false;
      if (act) {
        const int32_t rid = j_rid(x)[i];
        const int32_t em = emit_prefill_token(rid, t);
        done = em == c_dl()[rid];
        if (done) {
          c_done()[rid] = t;
          kvfree += (int64_t)c_pl()[rid] + em + kvo();
        }
      }
      completed += simt::popc(simt::ballot(done));
    }
    kvfree = simt::warp_sum_nn(kvfree);
    simt::sync();
    if (own(x)) L_used -= kvfree;
    count_tokens(ft() ? 0 : k, t);
    log(KVSIM_EV_PREFILL_DONE, x, k, completed, 0);
    if constexpr (EXT) {
      if (is_dual(x)) {
        dual_handoff(x, jstart, t);
        if (own(x)) L_njob = 0;
        if (head_admissible(x)) { acc_start_job(x, t); return; }
        if (own(x)) L_role = ROLE_DECODE;
        log(KVSIM_EV_ROLE, x, ROLE_DECODE, 0, 0);
        acc_boundary(x, t);
        return;
      }
    }
    // pass 2: redundant copies on y in job order while they fit
    int64_t used_y = get(L_used, y);
    int64_t s1c = 0;
    int32_t ncopy = 0;
    bool seq = false;  // once a survivor does not fit, decide one by one
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      int32_t rid = 0;
      bool surv = false;
      int64_t kv = 0;
      if (act) {
        rid = j_rid(x)[i];
        surv = c_em()[rid] != c_dl()[rid];
        if (surv) kv = (int64_t)c_pl()[rid] + c_em()[rid] + kvo();
      }
      bool cp = false;
      if (!seq) {
        const int64_t incl = simt::warp_incl_scan(kv);
        const bool fits = used_y + incl <= PC.f.cap;
        const unsigned bad = simt::ballot(surv && !fits);
        if (!bad) {
          cp = surv;
          used_y += simt::shfl(incl, 31);
        } else {
          const int f0 = simt::ffs(bad) - 1;
          cp = surv && lane < f0;
          used_y += simt::shfl(incl, f0) - simt::shfl(kv, f0);
          seq = true;
          for (int l = f0; l < 32; ++l) {
            const bool sl = simt::shfl((int32_t)surv, l) != 0;
            const int64_t kl = simt::shfl(kv, l);
            if (sl && used_y + kl <= PC.f.cap) {
              used_y += kl;
              if (lane == l) cp = true;
            }
          }
        }
      } else {
        for (int l = 0; l < 32; ++l) {
          const bool sl = simt::shfl((int32_t)surv, l) != 0;
          const int64_t kl = simt::shfl(kv, l);
          if (sl && used_y + kl <= PC.f.cap) {
            used_y += kl;
            if (lane == l) cp = true;
          }
        }
      }
      if (cp) c_cpy()[rid] = y;
      else if (surv) c_cpy()[rid] = -1;
      s1c += simt::warp_sum_nn(cp ? kv : (int64_t)0);
      ncopy += simt::popc(simt::ballot(cp));
    }
    simt::sync();
    add_used(y, s1c);
    if (own(y)) L_copy_tok += s1c;
    if (ncopy) log(KVSIM_EV_COPY, y, ncopy, 0, s1c);
    double fin = 0.0;
    if (s1c > 0) fin = prefill_transfer(x, y, s1c, jstart, t);
    // pass 3: survivors join x's batch as joiners (last token = t)
    const int32_t nb = get(L_nb, x);
    int32_t add = 0, addc = 0, minrem = 0x7fffffff;
    int64_t kvadd = 0, kvmin = INT64_MAX;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      int32_t rid = 0;
      bool surv = false;
      if (act) {
        rid = j_rid(x)[i];
        surv = c_em()[rid] != c_dl()[rid];
      }
      const unsigned sm = simt::ballot(surv);
      if (surv) {
        const int32_t em = c_em()[rid], dl = c_dl()[rid], pl = c_pl()[rid];
        const bool hasc = c_cpy()[rid] == y;
        if (hasc) c_fresh()[rid] = fin;
        const int32_t pos = nb + add + simt::popc(sm & simt::lanemask_lt());
        b_rid(x)[pos] = rid;
        b_rem(x)[pos] = (dl - em) | kJoin | (hasc ? kCopy : 0) | (em == 0 ? kFirst : 0);
        b_kvb(x)[pos] = pl + dl + kvo();
        b_tbt(x)[pos] = c_tbt()[rid];
        kvadd += (int64_t)pl + em + kvo();
        if (dl - em < minrem) minrem = dl - em;
        if (hasc && (int64_t)pl + em + kvo() < kvmin) kvmin = (int64_t)pl + em + kvo();
      }
      addc += simt::popc(simt::ballot(surv && c_cpy()[surv ? rid : 0] == y));
      add += simt::popc(sm);
    }
    kvadd = simt::warp_sum_nn(kvadd);
    minrem = simt::warp_min_i32(minrem);
    kvmin = simt::warp_min_i64(kvmin);
    simt::sync();
    if (own(x)) {
      L_nb += add;
      L_skv += kvadd;
      L_ncopy += addc;
      L_njob = 0;
      if (minrem < L_minrem) L_minrem = minrem;
      if (kvmin < L_kvmin) L_kvmin = kvmin;
    }
    if (head_admissible(x)) {
      move_all_to_partner(x, t);
      acc_start_job(x, t);
      return;
    }
    if (own(x)) L_role = ROLE_DECODE;
    log(KVSIM_EV_ROLE, x, ROLE_DECODE, 0, 0);
    acc_boundary(x, t);
  }

  // ============================== EXT: degraded mode (SEMANTICS §6b)
  // tokens the dual instance d holds as copies of decoder x's requests
  // (held: +1 while x's step is in flight)
  KV_DEV int64_t dual_copy_tokens(int d, int x) {
    flush(x);
    const int32_t nb = get(L_nb, x), ni = get(L_ni, x);
    const int64_t st = get(L_job, x) == JOB_STEP ? 1 : 0;
    int64_t s = 0;
    for (int32_t j = lane; j < nb; j += 32) {
      const int32_t rf = b_rem(x)[j];
      if (rf & kCopy) s += (int64_t)b_kvb(x)[j] - (rf & kRemMask) + st;
    }
    for (int32_t j = lane; j < ni; j += 32) {
      const int32_t rid = i_rid(x)[j];
      if (c_cpy()[rid] == d) s += (int64_t)c_pl()[rid] + c_em()[rid] + kvo();
    }
    return simt::warp_sum_nn(s);
  }
  // prefill survivors of the dual instance d: each goes to the decoder with
  // the most free tokens (full KV transfer, one per destination); d keeps
  // its computed KV as the copy while that decoder's budget allows
  KV_DEV_NOINLINE void dual_handoff(int d, double jstart, double t) {
    const int32_t k = get(L_njob, d);
    const int64_t cap = PC.f.cap, budget = PC.dual_budget;
    int64_t ct[3], u[3], per[3] = {0, 0, 0};
    for (int j = 0; j < 3; ++j) { ct[j] = dual_copy_tokens(d, d + 1 + j); u[j] = get(L_used, d + 1 + j); }
    int64_t freed = 0, kept = 0;
    int32_t ncopy = 0;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      const bool act = i < k;
      int32_t rid = 0;
      bool surv = false;
      int64_t kv = 0;
      if (act) {
        rid = j_rid(d)[i];
        const int32_t em = c_em()[rid];
        surv = em != c_dl()[rid];
        kv = (int64_t)c_pl()[rid] + em + kvo();
      }
      int32_t dst = d;
      bool cp = false;
      const int lim = (k - i0) < 32 ? (k - i0) : 32;
      for (int l = 0; l < lim; ++l) {
        if (!simt::shfl((int32_t)surv, l)) continue;
        const int64_t kl = simt::shfl(kv, l);
        int b = 0;
        int64_t bf = cap - u[0];
        if (cap - u[1] > bf) { b = 1; bf = cap - u[1]; }
        if (cap - u[2] > bf) { b = 2; bf = cap - u[2]; }
        int32_t dl_ = d;
        bool c_ = false;
        if (bf >= kl) {
          u[b] += kl;
          per[b] += kl;
          dl_ = d + 1 + b;
          if (ct[b] + kl <= budget) { ct[b] += kl; c_ = true; kept += kl; ncopy += 1; }
          else freed += kl;
        }
        if (lane == l) { dst = dl_; cp = c_; }
      }
      if (act && surv) {
        j_dst(d)[i] = dst;
        c_cpy()[rid] = cp ? d : -1;
        if (cp) c_fresh()[rid] = t;
      }
    }
    simt::sync();
    for (int j = 0; j < 3; ++j)
      if (own(d + 1 + j)) { L_used = u[j]; if (L_used > L_peak) L_peak = L_used; }
    if (own(d)) { L_used -= freed; L_copy_tok += kept; }
    if (ncopy) log(KVSIM_EV_COPY, d, ncopy, 1, kept);
    for (int j = 0; j < 3; ++j) {
      if (per[j] == 0) continue;
      const int X = d + 1 + j;
      const double fin = prefill_transfer(d, X, per[j], jstart, t);
      const int32_t base = get(L_ni, X);
      int32_t add = 0;
      int64_t kvs = 0;
      for (int32_t i0 = 0; i0 < k; i0 += 32) {
        const int32_t i = i0 + lane;
        bool go = false;
        int32_t rid = 0;
        if (i < k) {
          rid = j_rid(d)[i];
          go = c_em()[rid] != c_dl()[rid] && j_dst(d)[i] == X;
        }
        const unsigned m = simt::ballot(go);
        if (go) {
          const int32_t pos = base + add + simt::popc(m & simt::lanemask_lt());
          i_rid(X)[pos] = rid;
          i_ready(X)[pos] = fin;
          kvs += (int64_t)c_pl()[rid] + c_em()[rid] + kvo();
        }
        add += simt::popc(m);
      }
      kvs = simt::warp_sum_nn(kvs);
      simt::sync();
      if (own(X)) { L_ni += add; L_skv_in += kvs; if (fin < L_min_ready) L_min_ready = fin; }
    }
    // survivors no decoder had room for decode on d (joiners, no copy)
    const int32_t nb = get(L_nb, d);
    int32_t add = 0, minrem = 0x7fffffff;
    int64_t kvadd = 0;
    for (int32_t i0 = 0; i0 < k; i0 += 32) {
      const int32_t i = i0 + lane;
      bool go = false;
      int32_t rid = 0;
      if (i < k) {
        rid = j_rid(d)[i];
        go = c_em()[rid] != c_dl()[rid] && j_dst(d)[i] == d;
      }
      const unsigned m = simt::ballot(go);
      if (go) {
        const int32_t em = c_em()[rid], dl = c_dl()[rid], pl = c_pl()[rid];
        const int32_t pos = nb + add + simt::popc(m & simt::lanemask_lt());
        b_rid(d)[pos] = rid;
        b_rem(d)[pos] = (dl - em) | kJoin | (em == 0 ? kFirst : 0);
        b_kvb(d)[pos] = pl + dl + kvo();
        b_tbt(d)[pos] = c_tbt()[rid];
        kvadd += (int64_t)pl + em + kvo();
        if (dl - em < minrem) minrem = dl - em;
      }
      add += simt::popc(m);
    }
    kvadd = simt::warp_sum_nn(kvadd);
    minrem = simt::warp_min_i32(minrem);
    simt::sync();
    if (own(d)) { L_nb += add; L_skv += kvadd; if (minrem < L_minrem) L_minrem = minrem; }
  }
  // at decoder x's boundary: requests whose copy the dual instance holds move
  // to it while no prefill is pending (rebalance_pair's greedy);
  // x drops its KV ("overwrite")
  KV_DEV_NOINLINE void dual_push(int x, double t) {
    const int d = x & ~3;
    if (get(L_role, d) != ROLE_DECODE || get(L_pend, d) || get(Q_n, qid(x >> 1)) != 0) return;
    flush(x);
    int64_t c = (int64_t)get(L_nb, x) + get(L_ni, x) - get(L_nb, d) - get(L_ni, d);
    int64_t dd = load_of(x) - load_of(d);
    while (c >= 1 && dd >= 1) {
      const int64_t lim = c >= 2 ? dd : dd - 1;
      const int32_t nb = get(L_nb, x);
      uint64_t best = 0;
      int32_t bidx = -1;
      for (int32_t j = lane; j < nb; j += 32) {
        const int32_t rf = b_rem(x)[j];
        if ((rf & (kCopy | kSettle)) == kCopy) {
          const int64_t kv = (int64_t)b_kvb(x)[j] - (rf & kRemMask);
          if (kv <= lim) {
            const uint64_t kk = ((uint64_t)kv << 32) | (uint32_t)(0x7fffffff - b_rid(x)[j]);
            if (kk > best) { best = kk; bidx = j; }
          }
        }
      }
      const uint64_t wb = simt::warp_max_u64(best);
      if (wb == 0) break;
      const int src = simt::ffs(simt::ballot(best == wb)) - 1;
      const int32_t idx = simt::shfl(bidx, src);
      const int64_t kv = (int64_t)(wb >> 32);
      // move to d, copy dropped
      const int32_t rid = b_rid(x)[idx];
      const int32_t rf = b_rem(x)[idx];
      const int32_t rem = rf & kRemMask;
      const double tb = b_tbt(x)[idx];
      const bool joiner = (rf & kJoin) != 0;
      const double fresh = joiner ? c_fresh()[rid] : get(L_mirror_fin, x);
      const double ready = fresh > t ? fresh : t;
      const double last = joiner ? c_last()[rid] : get(L_prev_end, x);
      const int32_t dl = c_dl()[rid];
      simt::sync();
      if (lane == 0) {
        c_em()[rid] = dl - rem;
        c_tbt()[rid] = tb;
        c_last()[rid] = last;
        c_cpy()[rid] = -1;
        c_nmv()[rid] += 1;
      }
      batch_remove(x, idx);
      incoming_append(d, rid, ready);
      if (own(x)) { L_skv -= kv; L_ncopy -= 1; L_used -= kv; }
      if (own(d)) { L_skv_in += kv; L_copy_tok -= kv; }
      if (lane == 0) ws()->ct.n_moves += 1;
      log(KVSIM_EV_MOVE, x, rid, d, 0);
      c -= 2;
      dd -= 2 * kv;
    }
  }
  KV_DEV_NOINLINE void evict_group_copies(int h, unsigned clients) {
    for (;;) {
      Found v = largest_copy_on_from(h, clients);
      if (!v.where) return;
      evict(h, v);
    }
  }
  KV_DEV_NOINLINE void enter_degraded(int g, double t) {
    const int a = 4 * g;
    const unsigned grp = 0xfu << a;
    for (int h = a + 1; h <= a + 3; ++h) evict_group_copies(h, clients_of(h) & grp);
    if (lane >= a && lane <= a + 3) L_partner = lane == a ? -1 : a;
    if (own(g)) G_mode = 1;
    if (lane == 0) ws()->ct.n_modes += 1;
    // the group's requests wait in its first pair's queue
    const int q0 = 2 * g, q1 = 2 * g + 1;
    const int32_t n1 = get(Q_n, q1), h1 = get(Q_head, q1), h0 = get(Q_head, q0), n0 = get(Q_n, q0);
    const int64_t tk1 = get(Q_tok, q1);
    for (int32_t i = lane; i < n1; i += 32) {
      int64_t dst = (int64_t)h0 + n0 + i;
      if (dst >= Ncap_) dst -= Ncap_;
      ring(q0)[dst] = q_at(q1, h1, i);
    }
    simt::sync();
    if (own(q0)) { Q_n += n1; Q_tok += tk1; }
    if (own(q1)) { Q_n = 0; Q_tok = 0; }
    log(KVSIM_EV_MODE, g, 1, 0, 0);
    ensure_prefill(q0, t);
  }
  KV_DEV_NOINLINE void leave_degraded(int g, double t) {
    const int a = 4 * g;
    evict_group_copies(a, clients_of(a) & (0xcu << a));
    if (lane >= a && lane <= a + 3) L_partner = lane ^ 1;
    if (own(g)) G_mode = 0;
    if (lane == 0) ws()->ct.n_modes += 1;
    log(KVSIM_EV_MODE, g, 0, 0, 0);
    ensure_prefill(2 * g, t);
    ensure_prefill(2 * g + 1, t);
  }
  // ====================== EXT: inter-pair leveling (SEMANTICS §6b)
  KV_DEV_NOINLINE void schedule_leveling() {
    const int np = n >> 1;
    int64_t l = 0;
    bool el = false;
    {
      const int q = lane;
      const int a = (2 * q) & 31, b = (2 * q + 1) & 31;
      const int32_t ra = simt::shfl(L_role, a), rb = simt::shfl(L_role, b);
      const int32_t pa = simt::shfl(L_pend, a), pb = simt::shfl(L_pend, b);
      const int64_t la = simt::shfl(L_skv, a) + simt::shfl(L_skv_in, a);
      const int64_t lb = simt::shfl(L_skv, b) + simt::shfl(L_skv_in, b);
      const int32_t gm = simt::shfl(G_mode, (q >> 1) & 31);
      const bool deg = (q >> 1) < (n >> 2) && gm != 0;
      el = q < np && !deg && Q_n == 0 && ra == ROLE_DECODE && rb == ROLE_DECODE && !pa && !pb;
      l = la + lb;
    }
    const unsigned em = simt::ballot(el);
    if (em == 0) return;
    const int64_t mx = simt::warp_max_i64(el ? l : INT64_MIN);
    const int64_t mn = simt::warp_min_i64(el ? l : INT64_MAX);
    const int A = simt::ffs(simt::ballot(el && l == mx)) - 1;
    const int B = simt::ffs(simt::ballot(el && l == mn)) - 1;
    if (A == B || mx - mn < 2) return;
    const int x = load_of(2 * A + 1) > load_of(2 * A) ? 2 * A + 1 : 2 * A;
    const int y = (PC.f.cap - get(L_used, 2 * B + 1)) > (PC.f.cap - get(L_used, 2 * B)) ? 2 * B + 1 : 2 * B;
    if (own(x)) { L_lvl_dst = y; L_lvl_bud = PC.lvl_budget; }
  }
  // at x's boundary: migrate batch members (largest first) to the lighter
  // pair while each move strictly narrows the pair-load gap, within the
  // per-period link budget and the destination's memory
  KV_DEV_NOINLINE void level_from(int x, double t) {
    const int y = get(L_lvl_dst, x);
    int64_t bud = get(L_lvl_bud, x);
    if (own(x)) L_lvl_dst = -1;
    if (get(L_role, y) != ROLE_DECODE || get(L_pend, y) || degraded_pair(x >> 1) || degraded_pair(y >> 1)) return;
    flush(x);
    int64_t dd = load_of(x) + load_of(x ^ 1) - load_of(y) - load_of(y ^ 1);
    int64_t room = PC.f.cap - get(L_used, y);
    for (;;) {
      int64_t lim = dd - 1;
      if (bud < lim) lim = bud;
      if (room < lim) lim = room;
      if (lim < 1) break;
      const int32_t nb = get(L_nb, x);
      uint64_t best = 0;
      int32_t bidx = -1;
      for (int32_t j = lane; j < nb; j += 32) {
        const int32_t rf = b_rem(x)[j];
        const int64_t kv = (int64_t)b_kvb(x)[j] - (rf & kRemMask);
        if (kv <= lim && !(rf & kSettle)) {
          const uint64_t kk = ((uint64_t)kv << 32) | (uint32_t)(0x7fffffff - b_rid(x)[j]);
          if (kk > best) { best = kk; bidx = j; }
        }
      }
      const uint64_t wb = simt::warp_max_u64(best);
      if (wb == 0) break;
      const int src = simt::ffs(simt::ballot(best == wb)) - 1;
      const int32_t idx = simt::shfl(bidx, src);
      const int64_t kv = (int64_t)(wb >> 32);
      const int32_t rid = b_rid(x)[idx];
      const int32_t rf = b_rem(x)[idx];
      const int32_t rem = rf & kRemMask;
      const double tb = b_tbt(x)[idx];
      const bool joiner = (rf & kJoin) != 0;
      const double last = joiner ? c_last()[rid] : get(L_prev_end, x);
      const int32_t dl = c_dl()[rid];
      simt::sync();
      if (lane == 0) {
        c_em()[rid] = dl - rem;
        c_tbt()[rid] = tb;
        c_last()[rid] = last;
        c_cpy()[rid] = -1;
        c_nmv()[rid] += 1;
      }
      if (rf & kCopy) {
        const int h = partner_of(x);
        if (own(h)) { L_used -= kv; L_copy_tok -= kv; }
        if (own(x)) L_ncopy -= 1;
      }
      batch_remove(x, idx);
      add_used(y, kv);
      const double busy = link_get(x, y);
      const double start = t > busy ? t : busy;
      const double fin = kadd(start, transfer_latency(PC.f, kmul((double)kv, PC.f.kvb)));
      link_set(x, y, fin);
      // x stays the source of the transfer: it holds the KV until it is done
      if (own(x)) {
        L_skv -= kv;
        L_lvl_hold += kv;
        if (fin > L_lvl_until) L_lvl_until = fin;
      }
      incoming_append(y, rid, fin);
      if (own(y)) L_skv_in += kv;
      if (lane == 0) { ws()->ct.n_moves += 1; ws()->ct.lvl_tokens += kv; }
      log(KVSIM_EV_LEVEL, x, rid, y, kv);
      dd -= 2 * kv;
      bud -= kv;
      room -= kv;
    }
  }
  KV_DEV_NOINLINE void on_timer(double t) {
    if (lane == 0) ws()->ct.n_ticks += 1;
    log(KVSIM_EV_TIMER, -1, (int)(tick - 1), 0, 0);
    if (PC.deg_on) {
      for (int g = 0; g < (n >> 2); ++g) {
        const int a = 4 * g;
        const bool in_g = lane >= a && lane <= a + 3;
        const bool pf = simt::ballot(in_g && (L_role == ROLE_PREFILL || L_pend)) != 0;
        int32_t cnt = get(G_cnt, g);
        bool go;
        if (!get(G_mode, g)) {
          int64_t live = 0, red = 0;
          for (int h = a; h <= a + 3; ++h) {
            live += (int64_t)get(L_nb, h) + get(L_ni, h);
            red += get(L_ncopy, h);
            const int32_t ni = get(L_ni, h);
            int32_t ri = 0;
            for (int32_t j = lane; j < ni; j += 32) ri += c_cpy()[i_rid(h)[j]] >= 0 ? 1 : 0;
            red += simt::warp_sum_i32(ri);
          }
          cnt = (live > 0 && (double)red < kmul(PC.red_thr, (double)live)) ? cnt + 1 : 0;
          go = cnt >= PC.trig && !pf;
          if (go) cnt = 0;
          if (own(g)) G_cnt = cnt;
          if (go) enter_degraded(g, t);
        } else {
          int64_t u = 0;
          for (int h = a; h <= a + 3; ++h) u += get(L_used, h);
          cnt = ((double)u <= kmul(PC.exit_fill, kmul(4.0, (double)PC.f.cap))) ? cnt + 1 : 0;
          go = cnt >= PC.trig && !pf;
          if (go) cnt = 0;
          if (own(g)) G_cnt = cnt;
          if (go) leave_degraded(g, t);
        }
      }
    }
    if (PC.lvl_on) schedule_leveling();
  }

  // -------------------------------------------------------------- arrival
  KV_DEV_HANDLER void arrive(double t) {
    EMU_COUNT(16);
    const int64_t rid64 = next_rid;
    const int32_t rid = (int32_t)rid64;
    int32_t pl, dl;
    if (PC.tr_arr != nullptr) {
      pl = PC.tr_pl[rid];
      dl = PC.tr_dl[rid];
    } else {
      pl = uniform_range(draw_k(PC.key, rid64, 0), PC.pmin, PC.pmax);
      dl = uniform_range(draw_k(PC.key, rid64, 1), PC.dmin, PC.dmax);
    }
    if (lane == 0) {
      c_arr()[rid] = t;
      c_pl()[rid] = pl;
      c_dl()[rid] = dl;
      c_qlen()[rid] = pl;
      c_em()[rid] = 0;
      c_cpy()[rid] = -1;
      c_tbt()[rid] = 0.0;
      c_last()[rid] = 0.0;
      c_fresh()[rid] = 0.0;
      c_first()[rid] = 0.0;
      c_done()[rid] = 0.0;
      c_qs()[rid] = 0.0;
      c_nmv()[rid] = 0;
      c_npre()[rid] = 0;
    }
    simt::sync();
    // advance the generator
    t_prev = t;
    next_rid += 1;
    gen_next();
    if (policy == KVSIM_POLICY_UNIFIED) {
      const int64_t fr = lane < n ? PC.f.cap - L_used - Q_tok : INT64_MIN;
      const int64_t best = simt::warp_max_i64(fr);
      const int x = simt::ffs(simt::ballot(fr == best)) - 1;
      log(KVSIM_EV_ARRIVE, x, rid, pl, 0);
      q_push_back(x, rid, pl);
      if (get(L_job, x) == JOB_NONE) unified_start(x, t);
    } else if (policy == KVSIM_POLICY_SPLITWISE) {
      log(KVSIM_EV_ARRIVE, 0, rid, pl, 0);
      q_push_back(0, rid, pl);
    } else {
      const int np = n >> 1;
      const int64_t ua = simt::shfl(L_used, (2 * lane) & 31);
      const int64_t ub = simt::shfl(L_used, (2 * lane + 1) & 31);
      int64_t fr = lane < np ? (PC.f.cap - ua) + (PC.f.cap - ub) - Q_tok : INT64_MIN;
      if constexpr (EXT) {  // a degraded group is one routing unit (its first pair's queue)
        const int64_t uc = simt::shfl(L_used, (2 * lane + 2) & 31);
        const int64_t ud = simt::shfl(L_used, (2 * lane + 3) & 31);
        const int32_t gm = simt::shfl(G_mode, (lane >> 1) & 31);
        if (lane < np && (lane >> 1) < (n >> 2) && gm != 0)
          fr = (lane & 1) ? INT64_MIN : (PC.f.cap - ua) + (PC.f.cap - ub) + (PC.f.cap - uc) + (PC.f.cap - ud) - Q_tok;
      }
      const int64_t best = simt::warp_max_i64(fr);
      const int q = simt::ffs(simt::ballot(fr == best)) - 1;
      log(KVSIM_EV_ARRIVE, q, rid, pl, 0);
      q_push_back(q, rid, pl);
      ensure_prefill(q, t);
    }
  }

  // ------------------------------------------------------------ main loop
  KV_DEV void run() {
    const double kInf = as_f64(0x7ff0000000000000ull);
    for (;;) {
      double ct = kInf;
      uint32_t cku = 1u << 20;
      if (lane < n) {
        if (L_job != JOB_NONE) {
          ct = L_busy_until;
          cku = (L_job == JOB_PREFILL ? 2 : 3) * 64 + lane;
        } else if (L_role == ROLE_DECODE && L_ni > 0) {
          ct = L_min_ready;
          cku = 1 * 64 + lane;
        }
      }
      simt::warp_min_tk(ct, cku);
      const int32_t ck = (int32_t)cku;
      bool is_arrival = false;
      if (has_next && (t_next < ct || (t_next == ct))) is_arrival = true;
      if (!is_arrival && ck == (1 << 20)) break;
      if (++n_events + ws()->ct.adv_events > PC.event_budget) { status = KVSIM_E_EVENT_BUDGET; break; }
      if (lane == 0) ws()->ct.n_loop += 1;
      if constexpr (EXT) {  // policy timer: kind 4, after every other kind at equal time
        const double tt = kmul((double)tick, PC.timer_P);
        if (tt < (is_arrival ? t_next : ct)) {
          now = tt;
          if (now > t_last) t_last = now;
          tick += 1;
          on_timer(tt);
          continue;
        }
      }
      unsigned drive = 0xffffffffu;
      if (is_arrival) {
        now = t_next;
        if (now > t_last) t_last = now;
        arrive(t_next);
      } else {
        const double t = ct;
        now = t;
        if (now > t_last) t_last = now;
        const int kind = ck >> 6, x = ck & 63;
        if (!(POL == KVSIM_POLICY_SPLITWISE && kind == 2)) drive = 1u << x;
        if (kind == 1) {
          log(KVSIM_EV_WAKE, x, 0, 0, 0);
          if (policy == KVSIM_POLICY_ACCELLM) acc_boundary(x, t);
          else { join(x, t); step_start(x, t); }
        } else if (kind == 2) {
          if (policy == KVSIM_POLICY_SPLITWISE) sw_prefill_done(x, t);
          else acc_prefill_done(x, t);
        } else {
          if (policy == KVSIM_POLICY_UNIFIED) {
            unified_end(x, t);
          } else if (POL == KVSIM_POLICY_SPLITWISE && cobatch()) {
            unified_end(x, t);  // decode members + co-batched prompts (no restart)
            join(x, t);
            step_start(x, t);
          } else {
            step_end(x, t);
            if (policy == KVSIM_POLICY_ACCELLM) acc_boundary(x, t);
            else { join(x, t); step_start(x, t); }
          }
        }
      }
      if (policy == KVSIM_POLICY_SPLITWISE) sw_try_start(now);
      if (chain_steps) advance(drive);
    }
    simt::sync();
  }

  // --------------------------------------------- per-point metrics (K4 fused)
  // nearest-rank selection over uint64 keys stored (as doubles' bits) in arr
  KV_DEV_NOINLINE void radix_select2(const double* arr, int64_t nn, int64_t k1, int64_t k2, uint64_t& r1, uint64_t& r2) {
    uint64_t pre1 = 0, pre2 = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = lane; b < 256; b += 32) { ws()->hist[0][b] = 0; ws()->hist[1][b] = 0; }
      simt::sync();
      for (int64_t i = lane; i < nn; i += 32) {
        const uint64_t kk = as_u64(arr[i]);
        const uint32_t dg = (uint32_t)((kk >> shift) & 255u);
        if ((kk & mask) == pre1) simt::atomic_add_smem(&ws()->hist[0][dg], 1u);
        if ((kk & mask) == pre2) simt::atomic_add_smem(&ws()->hist[1][dg], 1u);
      }
      simt::sync();
      // scan histograms (uniform, all lanes)
      int64_t acc1 = 0, acc2 = 0;
      int b1 = -1, b2 = -1;
      for (int b = 0; b < 256; ++b) {
        const int64_t h1 = ws()->hist[0][b], h2 = ws()->hist[1][b];
        if (b1 < 0 && acc1 + h1 > k1) b1 = b; else if (b1 < 0) acc1 += h1;
        if (b2 < 0 && acc2 + h2 > k2) b2 = b; else if (b2 < 0) acc2 += h2;
      }
      k1 -= acc1;
      k2 -= acc2;
      pre1 |= (uint64_t)b1 << shift;
      pre2 |= (uint64_t)b2 << shift;
      mask |= (uint64_t)255u << shift;
      simt::sync();
    }
    r1 = pre1;
    r2 = pre2;
  }
  // the same over weighted entries (detail runs: (gap, count) TBT entries)
  KV_DEV_NOINLINE void radix_select2_w(const double* arr, const int32_t* w, int64_t nn, int64_t k1, int64_t k2,
                                       uint64_t& r1, uint64_t& r2) {
    uint64_t pre1 = 0, pre2 = 0, mask = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = lane; b < 256; b += 32) { ws()->hist[0][b] = 0; ws()->hist[1][b] = 0; }
      simt::sync();
      for (int64_t i = lane; i < nn; i += 32) {
        const uint64_t kk = as_u64(arr[i]);
        const uint32_t dg = (uint32_t)((kk >> shift) & 255u);
        const uint32_t c = (uint32_t)w[i];
        if ((kk & mask) == pre1) simt::atomic_add_smem(&ws()->hist[0][dg], c);
        if ((kk & mask) == pre2) simt::atomic_add_smem(&ws()->hist[1][dg], c);
      }
      simt::sync();
      int64_t acc1 = 0, acc2 = 0;
      int b1 = -1, b2 = -1;
      for (int b = 0; b < 256; ++b) {
        const int64_t h1 = ws()->hist[0][b], h2 = ws()->hist[1][b];
        if (b1 < 0 && acc1 + h1 > k1) b1 = b; else if (b1 < 0) acc1 += h1;
        if (b2 < 0 && acc2 + h2 > k2) b2 = b; else if (b2 < 0) acc2 += h2;
      }
      k1 -= acc1;
      k2 -= acc2;
      pre1 |= (uint64_t)b1 << shift;
      pre2 |= (uint64_t)b2 << shift;
      mask |= (uint64_t)255u << shift;
      simt::sync();
    }
    r1 = pre1;
    r2 = pre2;
  }

  KV_DEV_NOINLINE void finalize() {
    kvsim_point_summary s;
    // zero everything
    {
      char* z = reinterpret_cast<char*>(&s);
      for (unsigned i = 0; i < sizeof(s); ++i) z[i] = 0;
    }
    const kvsim_point_desc& d = AR.pts[point];
    const double kNaN = as_f64(0x7ff8000000000000ull);
    const double kInf = as_f64(0x7ff0000000000000ull);
    s.status = status;
    s.num_instances = (status == KVSIM_OK || status == KVSIM_E_EVENT_BUDGET) ? n : 0;
    s.user_tag = d.user_tag;
    const int64_t N = next_rid;  // requests that arrived
    s.n_requests = status == KVSIM_OK ? N : 0;
    if (status == KVSIM_OK || status == KVSIM_E_EVENT_BUDGET) {
      s.n_requests = N;
      {
        const double tl = simt::warp_max(lane < n ? L_tlast : 0.0);
        if (tl > t_last) t_last = tl;
      }
      const Counters ct = ws()->ct;
      s.n_events = n_events + ct.adv_events; s.n_steps = ct.n_steps; s.n_prefills = ct.n_prefills; s.n_moves = ct.n_moves;
      s.n_preemptions = ct.n_preempt; s.n_evictions = ct.n_evict;
      s.tokens_total = ct.tok_total; s.tokens_window = ct.tok_window;
      s.link_prefill_tokens = ct.pf_tokens; s.link_mirror_tokens = ct.mir_tokens;
      s.makespan_s = t_last;
      s.reserved[0] = ct.n_loop;
      s.link_leveling_tokens = ct.lvl_tokens;
      s.n_timer_ticks = ct.n_ticks;
      s.n_mode_switches = ct.n_modes;
      const int64_t peak = simt::warp_max(lane < n ? L_peak : (int64_t)0);
      // instances idle at the end while requests wait (only a failed point):
      // their open interval closes at the makespan
      if (qdepth > 0 && lane < n && L_job == JOB_NONE) L_idle_rb = kadd(L_idle_rb, ksub(clip(t_last), clip(L_irs)));
      double busy = 0.0, irb = 0.0;
      for (int x = 0; x < n; ++x) {
        busy = kadd(busy, get(L_busy_time, x));
        irb = kadd(irb, get(L_idle_rb, x));
      }
      s.idle_runnable_s = irb;
      s.queue_depth_max = qd_max;
      {
        const double area = kadd(qd_area, kmul((double)qdepth, ksub(t_last, qd_tprev)));
        s.queue_depth_avg = t_last > 0.0 ? kdiv(area, t_last) : kNaN;
      }
      if (AR.inst != nullptr && lane < n) {
        kvsim_instance_record ir;
        ir.busy_s = L_busy_time;
        ir.idle_runnable_s = L_idle_rb;
        ir.peak_kv_tokens = L_peak;
        ir.initial_role = (policy == KVSIM_POLICY_SPLITWISE && lane < n_prefill) ? ROLE_PREFILL : ROLE_DECODE;
        ir.reserved = 0;
        AR.inst[point * KVSIM_MAX_INSTANCES + lane] = ir;
      }
      s.peak_kv_tokens = peak;
      s.busy_s_total = busy;
      s.peak_kv_gb = kdiv(kmul((double)peak, PC.f.kvb), 1e9);
      s.link_prefill_gb = kdiv(kmul((double)ct.pf_tokens, PC.f.kvb), 1e9);
      s.link_mirror_gb = kdiv(kmul((double)ct.mir_tokens, PC.f.kvb), 1e9);
      // records (parity configs)
      if (AR.recs != nullptr) {
        kvsim_request_record* R = AR.recs + AR.rec_off[point];
        for (int64_t i = lane; i < N; i += 32) {
          const bool dn = c_em()[i] == c_dl()[i];
          kvsim_request_record r;
          r.arrival_s = c_arr()[i];
          r.first_token_s = c_em()[i] > 0 ? c_first()[i] : kNaN;
          r.completion_s = dn ? c_done()[i] : kNaN;
          r.tbt_max_s = c_tbt()[i];
          r.prompt_len = c_pl()[i];
          r.decode_len = c_dl()[i];
          r.n_moves = c_nmv()[i];
          r.n_preemptions = c_npre()[i];
          r.prefill_start_s = c_em()[i] > 0 ? c_qs()[i] : kNaN;
          R[i] = r;
        }
      }
      simt::sync();
      // sequential (rid-order) sums, maxima; keys for selection
      double s_ttft = 0.0, s_jct = 0.0, s_tbt = 0.0, tmax = 0.0, s_qw = 0.0;
      int64_t n_tbt = 0, m = 0, completed = 0;
      double mx_ttft = 0.0, mx_jct = 0.0;
      for (int64_t i0 = 0; i0 < N; i0 += 32) {
        const int64_t i = i0 + lane;
        const bool act = i < N;
        double a = 0.0, b = 0.0, tb = 0.0, ts = 0.0, qw = 0.0;
        bool inc = false, dn = false;
        int32_t dl = 0;
        if (act) {
          const double arr = c_arr()[i];
          dl = c_dl()[i];
          dn = c_em()[i] == dl;
          inc = dn && arr >= PC.warmup;
          if (inc) {
            a = ksub(c_first()[i], arr);
            b = ksub(c_done()[i], arr);
            ts = ksub(c_done()[i], c_first()[i]);
            tb = c_tbt()[i];
            qw = ksub(c_qs()[i], arr);
          }
        }
        simt::sync();
        if (act) {
          c_first()[i] = inc ? a : kInf;
          c_done()[i] = inc ? b : kInf;
        }
        completed += simt::popc(simt::ballot(dn));
        const int cnt = act ? 1 : 0;
        (void)cnt;
        const int lim = (int)((N - i0) < 32 ? (N - i0) : 32);
        for (int l = 0; l < lim; ++l) {
          const bool il = simt::shfl((int32_t)inc, l) != 0;
          const double al = simt::shfl(a, l), bl = simt::shfl(b, l), tsl = simt::shfl(ts, l);
          const double tbl = simt::shfl(tb, l);
          const double qwl = simt::shfl(qw, l);
          const int32_t dll = simt::shfl(dl, l);
          if (il) {
            m += 1;
            s_ttft = kadd(s_ttft, al);
            s_jct = kadd(s_jct, bl);
            s_qw = kadd(s_qw, qwl);
            if (al > mx_ttft) mx_ttft = al;
            if (bl > mx_jct) mx_jct = bl;
            if (dll > 1) {
              s_tbt = kadd(s_tbt, tsl);
              n_tbt += dll - 1;
              if (tbl > tmax) tmax = tbl;
            }
          }
        }
      }
      simt::sync();
      s.n_completed = completed;
      s.n_measured = m;
      if (m > 0) {
        s.ttft_mean = kdiv(s_ttft, (double)m);
        s.jct_mean = kdiv(s_jct, (double)m);
        s.ttft_max = mx_ttft;
        s.jct_max = mx_jct;
        const int64_t k50 = (50 * m + 99) / 100 - 1, k95 = (95 * m + 99) / 100 - 1;
        uint64_t r1, r2;
        radix_select2(c_first(), N, k50, k95, r1, r2);
        s.ttft_p50 = as_f64(r1);
        s.ttft_p95 = as_f64(r2);
        radix_select2(c_done(), N, k50, k95, r1, r2);
        s.jct_p50 = as_f64(r1);
        s.jct_p95 = as_f64(r2);
      } else {
        s.ttft_mean = s.jct_mean = s.ttft_p50 = s.ttft_p95 = s.ttft_max = kNaN;
        s.jct_p50 = s.jct_p95 = s.jct_max = kNaN;
      }
      s.tbt_mean = n_tbt > 0 ? kdiv(s_tbt, (double)n_tbt) : kNaN;
      s.tbt_max = n_tbt > 0 ? tmax : kNaN;
      s.n_tbt_samples = n_tbt;
      s.ttft_queue_mean = m > 0 ? kdiv(s_qw, (double)m) : kNaN;
      s.tbt_p50 = s.tbt_p95 = kNaN;
      if constexpr (DET) {
        const int64_t ne = ws()->ct.t_n;
        if (n_tbt > 0 && ne <= AR.Tcap && n_tbt < (int64_t)0xffffffffll) {
          const double* tv = gp(AR.t_val + (int64_t)slot * AR.Tcap);
          const int32_t* tc = gp(AR.t_cnt + (int64_t)slot * AR.Tcap);
          int64_t wsum = 0;
          for (int64_t i = lane; i < ne; i += 32) wsum += tc[i];
          wsum = simt::warp_sum_nn(wsum);
          if (wsum == n_tbt) {
            const int64_t k50 = (50 * n_tbt + 99) / 100 - 1, k95 = (95 * n_tbt + 99) / 100 - 1;
            uint64_t r1, r2;
            radix_select2_w(tv, tc, ne, k50, k95, r1, r2);
            s.tbt_p50 = as_f64(r1);
            s.tbt_p95 = as_f64(r2);
          }
        }
      }
      const double window = ksub(t_last, PC.warmup);
      if (window > 0.0) {
        s.cost_eff = kdiv((double)ct.tok_window, kmul(window, (double)n));
        s.idle_frac = ksub(1.0, kdiv(busy, kmul((double)n, window)));
      } else {
        s.cost_eff = s.idle_frac = kNaN;
      }
    }
    simt::sync();
    if (lane == 0) {
      AR.out[point] = s;
      if (AR.ev_count != nullptr) AR.ev_count[point] = ws()->ct.ev_n;
    }
    simt::sync();
  }
};

// One point, simulated by the policy-specialised core.
template <int P, bool LOG, bool EXT = false, bool DET = false>
KV_DEV_NOINLINE void run_point(const SweepArgs* ap, WarpScratch* w, int32_t slot, int64_t pt) {
#if defined(KVSIM_SIM_SMEM)
  // the lane's Sim object in dynamic shared memory after the warp scratch
  // blocks (local memory held it in round 1: 568 B stack frame, ~2,200 LDL/STL)
  using S = Sim<P, LOG, EXT, DET>;
  S* sim = reinterpret_cast<S*>(kvsim_smem + sizeof(WarpScratch) * kWarpsPerBlock) + threadIdx.x;
  new (sim) S(ap, w, slot);
  if (sim->init_point(pt)) sim->run();
  sim->finalize();
#else
  Sim<P, LOG, EXT, DET> sim(ap, w, slot);
  if (sim.init_point(pt)) sim.run();
  sim.finalize();
#endif
}

// Persistent warp loop: pull points from a global counter (policy-major LPT
// order set by the host), simulate, finalize.
// Points that need the full specialisations (event log, detail metrics,
// AcceLLM timer extensions, optional SPEC variants); the host launches the
// others through the lean FULL=false kernel, whose image holds only the
// three plain sweep specialisations with their handlers inlined
// (kvsim_sweep.cu; the full kernel is kvsim_sweep_full.cu).
KV_HD_INLINE bool needs_full(const kvsim_point_desc& d) {
  return (d.policy == KVSIM_POLICY_ACCELLM && (d.accellm_flags & 3) != 0) || d.first_token_decode != 0 ||
         d.splitwise_cobatch != 0;
}

template <bool FULL>
KV_DEV void sweep_warp(const SweepArgs* ap, WarpScratch* w, int32_t slot) {
  const SweepArgs& a = *ap;
  const int lane = simt::lane_id();
  for (;;) {
    unsigned long long p = 0;
#if defined(KVSIM_EMU)
    if (lane == 0) p = std::atomic_ref<unsigned long long>(*a.next_point).fetch_add(1);
#else
    if (lane == 0) p = atomicAdd(a.next_point, 1ull);
#endif
    p = simt::shfl((uint64_t)p, 0);
    if ((int64_t)p >= a.n_pts) break;
    const int64_t pt = a.order != nullptr ? a.order[p] : (int64_t)p;
    const int32_t pol = a.pts[pt].policy;
    const bool ext = pol == KVSIM_POLICY_ACCELLM && (a.pts[pt].accellm_flags & 3) != 0;
    // optional SPEC variants run in the LOG specialisation (kFeat)
    const bool feat = a.pts[pt].first_token_decode != 0 || a.pts[pt].splitwise_cobatch != 0;
    (void)ext; (void)feat;
#if !defined(KVSIM_EMU)
    if (a.ptime != nullptr && lane == 0) {  // stored at once: no register live across the point
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      a.ptime[3 * pt] = t0;
    }
#endif
    if constexpr (!FULL) {  // the host routes only plain points here
      if (pol == KVSIM_POLICY_SPLITWISE) run_point<KVSIM_POLICY_SPLITWISE, false>(ap, w, slot, pt);
      else if (pol == KVSIM_POLICY_ACCELLM) run_point<KVSIM_POLICY_ACCELLM, false>(ap, w, slot, pt);
      else run_point<KVSIM_POLICY_UNIFIED, false>(ap, w, slot, pt);
    } else if (a.detail) {  // reports: plain event loop, pooled TBT percentiles
      if (ext) run_point<KVSIM_POLICY_ACCELLM, true, true, true>(ap, w, slot, pt);
      else if (pol == KVSIM_POLICY_SPLITWISE) run_point<KVSIM_POLICY_SPLITWISE, true, false, true>(ap, w, slot, pt);
      else if (pol == KVSIM_POLICY_ACCELLM) run_point<KVSIM_POLICY_ACCELLM, true, false, true>(ap, w, slot, pt);
      else run_point<KVSIM_POLICY_UNIFIED, true, false, true>(ap, w, slot, pt);
    } else if (ext) {
      if (a.ev != nullptr || feat) run_point<KVSIM_POLICY_ACCELLM, true, true>(ap, w, slot, pt);
      else run_point<KVSIM_POLICY_ACCELLM, false, true>(ap, w, slot, pt);
    } else if (a.ev != nullptr || feat) {
      if (pol == KVSIM_POLICY_SPLITWISE) run_point<KVSIM_POLICY_SPLITWISE, true>(ap, w, slot, pt);
      else if (pol == KVSIM_POLICY_ACCELLM) run_point<KVSIM_POLICY_ACCELLM, true>(ap, w, slot, pt);
      else run_point<KVSIM_POLICY_UNIFIED, true>(ap, w, slot, pt);
    } else {
      if (pol == KVSIM_POLICY_SPLITWISE) run_point<KVSIM_POLICY_SPLITWISE, false>(ap, w, slot, pt);
      else if (pol == KVSIM_POLICY_ACCELLM) run_point<KVSIM_POLICY_ACCELLM, false>(ap, w, slot, pt);
      else run_point<KVSIM_POLICY_UNIFIED, false>(ap, w, slot, pt);
    }
#if !defined(KVSIM_EMU)
    if (a.ptime != nullptr && lane == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      a.ptime[3 * pt + 1] = t1;
      a.ptime[3 * pt + 2] = (unsigned long long)slot;
    }
#endif
  }
}

}  // namespace kvsim_dev
