// kvsim_cli.cpp — the C++ host entry point (`kvsim`), the drop-in for the
// reference CLI specified in reference SPEC.md:400-455 (tools/ in
// proj/CMakeLists.txt:19, absent in the reference). It parses the JSON
// ExperimentConfig (unknown keys rejected, every default echoed,
// SPEC.md:405-407,444), expands the point grid, and calls ONLY the C-ABI
// (include/kvsim_gpu.h) to simulate; outputs are the SPEC files:
//
//   kvsim run             report.json, summary.csv, meta.json [, events.jsonl]
//   kvsim sweep           summary.csv, sweep_long.csv, report.json, meta.json
//   kvsim curves          curves.csv          (perfmodel throughput_curves)
//   kvsim gen-trace       trace.csv           (#kvsim-trace v1, device RNG)
//   kvsim validate-config resolved config on stdout
//
// Flags: --config PATH --seed N --out DIR --emit-events --gpus N; env
// KVSIM_LOG=0..3. Errors exit nonzero with a machine-readable
// {"error": ...} line on stderr.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cerrno>
#include <cstdarg>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <vector>

#include "json_lite.hpp"
#include "kvsim_shard.hpp"
#include "kvsim/perfmodel.hpp"
#include "kvsim_gpu.h"

namespace {

constexpr const char* kToolVersion = "kvsim-b200 1.0";

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

int g_log = 1;
void logf(int lvl, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void logf(int lvl, const char* fmt, ...) {
  if (lvl > g_log) return;
  va_list ap;
  va_start(ap, fmt);
  std::fprintf(stderr, "[kvsim] ");
  std::vfprintf(stderr, fmt, ap);
  std::fprintf(stderr, "\n");
  va_end(ap);
}

std::string read_file(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  if (!f) throw ConfigError("cannot open " + p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
void write_file(const std::string& p, const std::string& s) {
  // atomic per file: write then rename
  const std::string tmp = p + ".tmp";
  std::ofstream f(tmp, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write " + p);
  f << s;
  f.close();
  if (std::rename(tmp.c_str(), p.c_str()) != 0) throw std::runtime_error("cannot rename " + tmp);
}
void mkdirs(const std::string& d) {
  std::string cur;
  for (size_t i = 0; i <= d.size(); ++i) {
    if (i == d.size() || d[i] == '/') {
      if (!cur.empty()) mkdir(cur.c_str(), 0755);
    }
    if (i < d.size()) cur += d[i];
  }
}
std::string num(double d) {
  if (std::isnan(d)) return "nan";
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", d);
  return b;
}
uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) { h ^= c; h *= 1099511628211ull; }
  return h;
}

// ------------------------------------------------------------------ config
const char* const kKeys[] = {"model", "device", "num_devices", "memory_reserve_fraction", "instances", "policy",
                             "policies", "num_prefill_instances", "prefill_token_budget", "workload",
                             "arrival_process", "rate", "rates", "duration_s", "num_requests", "warmup_s", "seed",
                             "seeds", "efficiency", "link_aggregation", "trace", "sweep_instances",
                             "sweep_devices", "curves", "emit_records", "splitwise_cobatch", "degraded_mode",
                             "inter_pair_leveling", "policy_timer_s", "output", "resource", "detail_metrics",
                             "first_token_decode"};

struct Resolved {
  jl::Value cfg;  // resolved config (defaults filled)
};

double req_num(const jl::Value& v, const char* what) {
  if (!v.is_num()) throw ConfigError(std::string(what) + " must be a number");
  return v.num;
}
int64_t req_int(const jl::Value& v, const char* what) {
  double d = req_num(v, what);
  if (d != std::floor(d)) throw ConfigError(std::string(what) + " must be an integer");
  return (int64_t)d;
}

jl::Value model_obj(const jl::Value* v) {
  jl::Value m = jl::Value::object();
  std::string name = "llama2-70b";
  if (v && v->is_str()) name = v->str;
  if (v && v->is_obj()) {
    const char* keys[] = {"name", "param_count", "num_layers", "hidden_dim", "num_kv_heads", "head_dim",
                          "bytes_per_value"};
    for (auto& kv : v->obj)
      if (std::find_if(std::begin(keys), std::end(keys), [&](const char* k) { return kv.first == k; }) ==
          std::end(keys))
        throw ConfigError("unknown model key: " + kv.first);
    for (int i = 1; i < 7; ++i)
      if (!v->find(keys[i])) throw ConfigError(std::string("model.") + keys[i] + " required");
    m.set("name", jl::Value::string(v->find("name") && v->find("name")->is_str() ? v->find("name")->str : "custom"));
    for (int i = 1; i < 7; ++i) m.set(keys[i], jl::Value::number(req_num(*v->find(keys[i]), keys[i])));
    return m;
  }
  double P, L, H, KV, HD, B;
  if (name == "llama2-70b") { P = 70e9; L = 80; H = 8192; KV = 8; HD = 128; B = 2; }
  else if (name == "llama2-7b") { P = 7e9; L = 32; H = 4096; KV = 32; HD = 128; B = 2; }
  else throw ConfigError("unknown model preset: " + name);
  m.set("name", jl::Value::string(name));
  m.set("param_count", jl::Value::number(P));
  m.set("num_layers", jl::Value::number(L));
  m.set("hidden_dim", jl::Value::number(H));
  m.set("num_kv_heads", jl::Value::number(KV));
  m.set("head_dim", jl::Value::number(HD));
  m.set("bytes_per_value", jl::Value::number(B));
  return m;
}
jl::Value device_obj(const jl::Value& v) {
  jl::Value d = jl::Value::object();
  if (v.is_obj()) {
    const char* keys[] = {"name", "peak_flops", "hbm_capacity", "hbm_bandwidth", "link_bandwidth"};
    for (auto& kv : v.obj)
      if (std::find_if(std::begin(keys), std::end(keys), [&](const char* k) { return kv.first == k; }) ==
          std::end(keys))
        throw ConfigError("unknown device key: " + kv.first);
    d.set("name", jl::Value::string(v.find("name") && v.find("name")->is_str() ? v.find("name")->str : "custom"));
    for (int i = 1; i < 5; ++i) {
      if (!v.find(keys[i])) throw ConfigError(std::string("device.") + keys[i] + " required");
      d.set(keys[i], jl::Value::number(req_num(*v.find(keys[i]), keys[i])));
    }
    return d;
  }
  if (!v.is_str()) throw ConfigError("device must be a preset name or an object");
  kvsim::DeviceSpec s;
  if (v.str == "h100" || v.str == "H100") s = kvsim::device_preset_h100();
  else if (v.str == "910b2" || v.str == "910B2") s = kvsim::device_preset_910b2();
  else throw ConfigError("unknown device preset: " + v.str);
  d.set("name", jl::Value::string(s.name));
  d.set("peak_flops", jl::Value::number(s.peak_flops));
  d.set("hbm_capacity", jl::Value::number(s.hbm_capacity));
  d.set("hbm_bandwidth", jl::Value::number(s.hbm_bandwidth));
  d.set("link_bandwidth", jl::Value::number(s.link_bandwidth));
  return d;
}
jl::Value workload_obj(const jl::Value* v) {
  // SPEC.md:144 presets; conversation/coding/fixed are builder presets (SEMANTICS §2)
  jl::Value w = jl::Value::object();
  int64_t p0 = 20, p1 = 1000, d0 = 20, d1 = 1000;
  std::string name = "mixed";
  if (v && v->is_str()) {
    name = v->str;
    if (name == "light") { p0 = 20; p1 = 500; d0 = 20; d1 = 500; }
    else if (name == "mixed") {}
    else if (name == "heavy") { p0 = 500; p1 = 1000; d0 = 500; d1 = 1000; }
    else if (name == "conversation") { p0 = 50; p1 = 1500; d0 = 50; d1 = 600; }
    else if (name == "coding") { p0 = 1000; p1 = 8000; d0 = 10; d1 = 200; }
    else throw ConfigError("unknown workload preset: " + name);
  } else if (v && v->is_obj()) {
    for (auto& kv : v->obj)
      if (kv.first != "name" && kv.first != "prompt_range" && kv.first != "decode_range" &&
          kv.first != "distribution")
        throw ConfigError("unknown workload key: " + kv.first);
    auto rng = [&](const char* k, int64_t& a, int64_t& b) {
      const jl::Value* r = v->find(k);
      if (!r || !r->is_arr() || r->arr.size() != 2) throw ConfigError(std::string("workload.") + k + " must be [min,max]");
      a = req_int(r->arr[0], k);
      b = req_int(r->arr[1], k);
    };
    rng("prompt_range", p0, p1);
    rng("decode_range", d0, d1);
    if (const jl::Value* ds = v->find("distribution"))
      if (!ds->is_str() || ds->str != "uniform") throw ConfigError("workload.distribution: only \"uniform\"");
    name = v->find("name") && v->find("name")->is_str() ? v->find("name")->str : "custom";
  }
  if (p0 < 1 || p1 < p0 || d0 < 1 || d1 < d0) throw ConfigError("workload ranges must satisfy 1 <= min <= max");
  w.set("name", jl::Value::string(name));
  jl::Value pr = jl::Value::array();
  pr.push(jl::Value::number((double)p0));
  pr.push(jl::Value::number((double)p1));
  jl::Value dr = jl::Value::array();
  dr.push(jl::Value::number((double)d0));
  dr.push(jl::Value::number((double)d1));
  w.set("prompt_range", pr);
  w.set("decode_range", dr);
  w.set("distribution", jl::Value::string("uniform"));
  return w;
}

jl::Value num_list(const jl::Value* v, const char* what) {
  jl::Value a = jl::Value::array();
  if (!v) return a;
  if (v->is_num()) { a.push(*v); return a; }
  if (!v->is_arr()) throw ConfigError(std::string(what) + " must be a number or a list");
  for (auto& e : v->arr) a.push(jl::Value::number(req_num(e, what)));
  return a;
}
jl::Value str_list(const jl::Value* v, const char* what) {
  jl::Value a = jl::Value::array();
  if (!v) return a;
  if (v->is_str()) { a.push(*v); return a; }
  if (!v->is_arr()) throw ConfigError(std::string(what) + " must be a string or a list");
  for (auto& e : v->arr) {
    if (!e.is_str()) throw ConfigError(std::string(what) + " entries must be strings");
    a.push(e);
  }
  return a;
}

std::string norm_policy(const std::string& p) {
  if (p == "accellm") return "accellm";
  if (p == "splitwise" || p == "splitwise_static") return "splitwise_static";
  if (p == "unified" || p == "vllm") return "unified";
  throw ConfigError("unknown policy: " + p);
}

jl::Value resolve(const jl::Value& in, const std::string& cmd) {
  if (!in.is_obj()) throw ConfigError("config must be a JSON object");
  for (auto& kv : in.obj)
    if (std::find_if(std::begin(kKeys), std::end(kKeys), [&](const char* k) { return kv.first == k; }) ==
        std::end(kKeys))
      throw ConfigError("unknown config key: " + kv.first);
  if (const jl::Value* v = in.find("splitwise_cobatch"))
    if (v->kind != jl::Value::Bool) throw ConfigError("splitwise_cobatch must be a boolean");
  jl::Value c = jl::Value::object();
  c.set("model", model_obj(in.find("model")));
  c.set("device", device_obj(in.find("device") ? *in.find("device") : jl::Value::string("h100")));
  c.set("num_devices", jl::Value::number(in.find("num_devices") ? (double)req_int(*in.find("num_devices"), "num_devices") : 4));
  c.set("memory_reserve_fraction",
        jl::Value::number(in.find("memory_reserve_fraction") ? req_num(*in.find("memory_reserve_fraction"), "memory_reserve_fraction") : 0.10));
  c.set("instances", jl::Value::number(in.find("instances") ? (double)req_int(*in.find("instances"), "instances") : 8));
  jl::Value pols = str_list(in.find("policies"), "policies");
  if (in.find("policy")) {
    jl::Value one = str_list(in.find("policy"), "policy");
    for (auto& e : one.arr) pols.push(e);
  }
  if (pols.arr.empty()) pols.push(jl::Value::string("accellm"));
  for (auto& e : pols.arr) e.str = norm_policy(e.str);
  c.set("policies", pols);
  c.set("num_prefill_instances",
        jl::Value::number(in.find("num_prefill_instances") ? (double)req_int(*in.find("num_prefill_instances"), "num_prefill_instances") : 0));
  c.set("prefill_token_budget",
        jl::Value::number(in.find("prefill_token_budget") ? (double)req_int(*in.find("prefill_token_budget"), "prefill_token_budget") : 8192));
  c.set("workload", workload_obj(in.find("workload")));
  std::string proc = in.find("arrival_process") && in.find("arrival_process")->is_str() ? in.find("arrival_process")->str : "poisson";
  if (proc != "poisson" && proc != "fixed-interval" && proc != "fixed") throw ConfigError("arrival_process: poisson | fixed-interval");
  c.set("arrival_process", jl::Value::string(proc == "poisson" ? "poisson" : "fixed-interval"));
  jl::Value rates = num_list(in.find("rates"), "rates");
  for (auto& e : num_list(in.find("rate"), "rate").arr) rates.push(e);
  if (rates.arr.empty()) {
    if (cmd == "sweep") throw ConfigError("empty rate list");
    if (!in.find("trace")) rates.push(jl::Value::number(4.0));
  }
  for (auto& e : rates.arr)
    if (!(e.num >= 0)) throw ConfigError("rates must be >= 0");
  c.set("rates", rates);
  const bool has_n = in.find("num_requests") != nullptr, has_d = in.find("duration_s") != nullptr;
  double dur = has_d ? req_num(*in.find("duration_s"), "duration_s") : (has_n ? INFINITY : 300.0);
  if (!(dur > 0)) throw ConfigError("duration_s must be > 0");
  c.set("duration_s", std::isinf(dur) ? jl::Value::string("inf") : jl::Value::number(dur));
  c.set("num_requests", jl::Value::number(has_n ? (double)req_int(*in.find("num_requests"), "num_requests") : 0));
  c.set("warmup_s", jl::Value::number(in.find("warmup_s") ? req_num(*in.find("warmup_s"), "warmup_s") : (has_n && !has_d ? 0.0 : 30.0)));
  jl::Value seeds = num_list(in.find("seeds"), "seeds");
  for (auto& e : num_list(in.find("seed"), "seed").arr) seeds.push(e);
  if (seeds.arr.empty()) seeds.push(jl::Value::number(0));
  c.set("seeds", seeds);
  jl::Value eff = jl::Value::object();
  double ce = 0.5, me = 0.8, le = 0.8;
  if (const jl::Value* e = in.find("efficiency")) {
    if (!e->is_obj()) throw ConfigError("efficiency must be an object");
    for (auto& kv : e->obj) {
      if (kv.first == "compute_eff") ce = req_num(kv.second, "compute_eff");
      else if (kv.first == "mem_bw_eff") me = req_num(kv.second, "mem_bw_eff");
      else if (kv.first == "link_eff") le = req_num(kv.second, "link_eff");
      else throw ConfigError("unknown efficiency key: " + kv.first);
    }
  }
  eff.set("compute_eff", jl::Value::number(ce));
  eff.set("mem_bw_eff", jl::Value::number(me));
  eff.set("link_eff", jl::Value::number(le));
  c.set("efficiency", eff);
  std::string la = in.find("link_aggregation") && in.find("link_aggregation")->is_str() ? in.find("link_aggregation")->str : "striped";
  if (la != "striped" && la != "single-link" && la != "single") throw ConfigError("link_aggregation: striped | single-link");
  c.set("link_aggregation", jl::Value::string(la == "striped" ? "striped" : "single-link"));
  if (const jl::Value* t = in.find("trace")) {
    if (!t->is_str()) throw ConfigError("trace must be a path");
    c.set("trace", *t);
  }
  jl::Value si = num_list(in.find("sweep_instances"), "sweep_instances");
  if (si.arr.empty()) si.push(c.find("instances")->num == c.find("instances")->num ? *c.find("instances") : jl::Value());
  c.set("sweep_instances", si);
  jl::Value sd = jl::Value::array();
  if (const jl::Value* v = in.find("sweep_devices")) {
    if (!v->is_arr()) throw ConfigError("sweep_devices must be a list");
    for (auto& e : v->arr) sd.push(device_obj(e));
  } else {
    sd.push(*c.find("device"));
  }
  c.set("sweep_devices", sd);
  if (const jl::Value* cv = in.find("curves")) c.set("curves", *cv);
  if (const jl::Value* rs = in.find("resource")) {
    // resource-sweep: {"kind": "hbm_capacity"|"link_bandwidth", "values": [...]}
    if (!rs->is_obj()) throw ConfigError("resource must be an object");
    for (auto& kv : rs->obj)
      if (kv.first != "kind" && kv.first != "values") throw ConfigError("unknown resource key: " + kv.first);
    const jl::Value* k = rs->find("kind");
    if (!k || !k->is_str() || (k->str != "hbm_capacity" && k->str != "link_bandwidth"))
      throw ConfigError("resource.kind: hbm_capacity | link_bandwidth");
    jl::Value vals = num_list(rs->find("values"), "resource.values");
    if (vals.arr.empty()) throw ConfigError("resource.values must be non-empty");
    jl::Value r = jl::Value::object();
    r.set("kind", *k);
    r.set("values", vals);
    c.set("resource", r);
  } else if (cmd == "resource-sweep") {
    throw ConfigError("resource-sweep needs a \"resource\" block");
  }
  // AcceLLM timer-driven extensions (SEMANTICS §6b):
  // `true`/`false` or an object of named thresholds; every default is echoed
  auto ext_block = [&](const char* key, std::vector<std::pair<const char*, double>> defs) {
    jl::Value o = jl::Value::object();
    bool on = false;
    std::vector<double> vals;
    for (auto& d : defs) vals.push_back(d.second);
    if (const jl::Value* v = in.find(key)) {
      if (v->kind == jl::Value::Bool) {
        on = v->b;
      } else if (v->is_obj()) {
        on = true;
        for (auto& kv : v->obj) {
          if (kv.first == "enabled") {
            if (kv.second.kind != jl::Value::Bool) throw ConfigError(std::string(key) + ".enabled must be a boolean");
            on = kv.second.b;
            continue;
          }
          size_t i = 0;
          for (; i < defs.size(); ++i)
            if (kv.first == defs[i].first) break;
          if (i == defs.size()) throw ConfigError(std::string("unknown ") + key + " key: " + kv.first);
          vals[i] = req_num(kv.second, defs[i].first);
          if (!(vals[i] > 0)) throw ConfigError(std::string(key) + "." + defs[i].first + " must be > 0");
        }
      } else {
        throw ConfigError(std::string(key) + " must be a boolean or an object");
      }
    }
    o.set("enabled", jl::Value::boolean(on));
    for (size_t i = 0; i < defs.size(); ++i) o.set(defs[i].first, jl::Value::number(vals[i]));
    c.set(key, o);
  };
  ext_block("degraded_mode", {{"trigger_ticks", 3}, {"redundancy_threshold", 0.5}, {"exit_fill", 0.5},
                              {"dual_copy_fraction", 1.0 / 3.0}});
  ext_block("inter_pair_leveling", {{"link_fraction", 0.10}});
  {
    const double tp = in.find("policy_timer_s") ? req_num(*in.find("policy_timer_s"), "policy_timer_s") : 1.0;
    if (!(tp > 0)) throw ConfigError("policy_timer_s must be > 0");
    c.set("policy_timer_s", jl::Value::number(tp));
  }
  {
    const double tt = c.find("degraded_mode")->find("trigger_ticks")->num;
    if (tt != std::floor(tt)) throw ConfigError("degraded_mode.trigger_ticks must be an integer");
  }
  // first token from the first decode step (SPEC.md:273 alternative): off by default
  if (const jl::Value* v = in.find("first_token_decode"))
    if (v->kind != jl::Value::Bool) throw ConfigError("first_token_decode must be a boolean");
  c.set("first_token_decode",
        jl::Value::boolean(in.find("first_token_decode") ? in.find("first_token_decode")->b : false));
  // Splitwise high-load co-batching: off by default
  c.set("splitwise_cobatch", jl::Value::boolean(in.find("splitwise_cobatch") ? in.find("splitwise_cobatch")->b : false));
  c.set("emit_records", jl::Value::boolean(in.find("emit_records") && in.find("emit_records")->kind == jl::Value::Bool
                                               ? in.find("emit_records")->b
                                               : cmd == "run"));
  // detail metrics (pooled TBT p50/p95: plain event loop + per-step gap
  // entries in HBM) default on for `run`, off for sweeps
  if (const jl::Value* v = in.find("detail_metrics"))
    if (v->kind != jl::Value::Bool) throw ConfigError("detail_metrics must be a boolean");
  c.set("detail_metrics", jl::Value::boolean(in.find("detail_metrics") ? in.find("detail_metrics")->b : cmd == "run"));
  return c;
}

// ------------------------------------------------------------------ traces
// Host array in page-locked memory when the library can provide it
// (kvsim_gpu_host_alloc), else ordinary memory: traces parsed straight into
// it are DMA'd to the device inside kvsim_gpu_run without a staging copy.
template <class T>
class HostArray {
 public:
  HostArray() = default;
  HostArray(const HostArray&) = delete;
  HostArray& operator=(const HostArray&) = delete;
  HostArray(HostArray&& o) noexcept { swap(o); }
  HostArray& operator=(HostArray&& o) noexcept { swap(o); return *this; }
  ~HostArray() { release(); }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  T* data() { return p_; }
  const T* data() const { return p_; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }
  bool pinned() const { return pinned_; }
  void resize(size_t n) {  // keeps the first min(n, size()) elements
    if (n <= cap_) { n_ = n; return; }
    HostArray t;
    t.alloc(n);
    if (n_) std::memcpy(t.p_, p_, n_ * sizeof(T));
    t.n_ = n;
    swap(t);
  }

 private:
  void alloc(size_t n) {
    p_ = static_cast<T*>(kvsim_gpu_host_alloc(n * sizeof(T)));
    pinned_ = p_ != nullptr;
    if (!p_) p_ = static_cast<T*>(std::malloc(n * sizeof(T)));
    if (!p_) throw std::bad_alloc();
    cap_ = n;
  }
  void release() {
    if (p_) { if (pinned_) kvsim_gpu_host_free(p_); else std::free(p_); }
    p_ = nullptr; n_ = cap_ = 0; pinned_ = false;
  }
  void swap(HostArray& o) {
    std::swap(p_, o.p_); std::swap(n_, o.n_); std::swap(cap_, o.cap_); std::swap(pinned_, o.pinned_);
  }
  T* p_ = nullptr;
  size_t n_ = 0, cap_ = 0;
  bool pinned_ = false;
};

struct Trace {
  HostArray<double> arr;
  HostArray<int32_t> pl, dl;
};

namespace trace_io {
// One row `id,arrival_s,prompt_len,decode_len`. Numbers may
// be preceded by blanks or '+', as the scanf-based reader accepted; doubles go
// through std::from_chars, which rounds correctly like strtod.
inline const char* skip_blank(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  return p;
}
inline bool int_field(const char*& p, const char* e, long long& v) {
  p = skip_blank(p, e);
  if (p < e && *p == '+') ++p;
  auto r = std::from_chars(p, e, v);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  return true;
}
inline bool row(const char* p, const char* e, long long& id, double& a, long long& pl, long long& dl) {
  if (!int_field(p, e, id) || p >= e || *p++ != ',') return false;
  p = skip_blank(p, e);
  if (p < e && *p == '+') ++p;
  auto r = std::from_chars(p, e, a);
  if (r.ec != std::errc()) return false;
  p = r.ptr;
  if (p >= e || *p++ != ',' || !int_field(p, e, pl) || p >= e || *p++ != ',' || !int_field(p, e, dl)) return false;
  return p == e;
}
struct Chunk {
  const char* b;
  const char* e;
  size_t first_line = 0, lines = 0, first_row = 0, rows = 0;
  size_t err_line = 0;  // 0 = none
  std::string err;
  size_t first_row_line = 0;  // line of the first data row
  bool first_ok = false;      // ... and it parsed and passed the local checks
  double first_a = 0, last_a = 0;
};
// is this line a data row? (comments, blank lines and an optional column header are not)
inline bool is_row(const char* p, const char* e) {
  if (p < e && e[-1] == '\r') --e;
  return !(p == e || *p == '#' || (e - p >= 3 && std::memcmp(p, "id,", 3) == 0));
}
}  // namespace trace_io

Trace load_trace(const std::string& path) {
  // header `#kvsim-trace v1`, rows id,arrival_s,prompt_len,decode_len;
  // errors name the line. Bulk ingestion: the file is read
  // once, split at line boundaries and parsed by all host threads straight into
  // page-locked arrays; the first error in file order is reported.
  using namespace trace_io;
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw ConfigError("cannot open trace " + path);
  std::string buf;
  {
    char tmp[1 << 16];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.append(tmp, k);
    std::fclose(f);
  }
  const char* B = buf.data();
  const char* E = B + buf.size();
  const char* nl = static_cast<const char*>(std::memchr(B, '\n', buf.size()));
  const char* body = nl ? nl + 1 : E;
  if (buf.rfind("#kvsim-trace v1", 0) != 0) throw ConfigError(path + ":1: missing '#kvsim-trace v1' header");
  const size_t bytes = (size_t)(E - body);
  size_t nt = std::max(1u, std::thread::hardware_concurrency());
  nt = std::min<size_t>({nt, 64, bytes / (1 << 20) + 1});  // ~1 MB or more per thread
  std::vector<Chunk> ch(nt);
  const char* cur = body;
  for (size_t k = 0; k < nt; ++k) {
    const char* stop = k + 1 == nt ? E : body + bytes * (k + 1) / nt;
    if (stop < cur) stop = cur;
    if (k + 1 < nt) {  // extend to the end of the line
      const char* q = static_cast<const char*>(std::memchr(stop, '\n', (size_t)(E - stop)));
      stop = q ? q + 1 : E;
    }
    ch[k].b = cur;
    ch[k].e = stop;
    cur = stop;
  }
  auto for_lines = [](const Chunk& c, auto&& fn) {
    const char* p = c.b;
    while (p < c.e) {
      const char* q = static_cast<const char*>(std::memchr(p, '\n', (size_t)(c.e - p)));
      const char* le = q ? q : c.e;
      if (!fn(p, le)) return;
      p = q ? q + 1 : c.e;
    }
  };
  auto parallel = [&](auto&& fn) {
    std::vector<std::thread> th;
    for (size_t k = 1; k < nt; ++k) th.emplace_back(fn, k);
    fn(0);
    for (auto& t : th) t.join();
  };
  // pass 1: lines and data rows per chunk
  parallel([&](size_t k) {
    for_lines(ch[k], [&](const char* p, const char* e) {
      ch[k].lines++;
      ch[k].rows += is_row(p, e);
      return true;
    });
  });
  size_t line0 = 2, row0 = 0;
  for (auto& c : ch) { c.first_line = line0; c.first_row = row0; line0 += c.lines; row0 += c.rows; }
  Trace t;
  t.arr.resize(row0);
  t.pl.resize(row0);
  t.dl.resize(row0);
  // pass 2: parse and check each chunk (row ids and arrival order are local
  // given the chunk's first row index; chunk seams are checked after the join)
  parallel([&](size_t k) {
    Chunk& c = ch[k];
    size_t ln = c.first_line, r = c.first_row;
    double prev = -INFINITY;
    auto fail = [&](const char* m) { c.err_line = ln; c.err = m; return false; };
    for_lines(c, [&](const char* p, const char* e) {
      if (e > p && e[-1] == '\r') --e;
      if (is_row(p, e)) {
        long long id, pl, dl;
        double a;
        if (!row(p, e, id, a, pl, dl)) return fail("parse error");
        if (id < 0 || (size_t)id != r) return fail("ids must be 0..n-1 in order");
        if (!std::isfinite(a)) return fail("arrival_s must be finite");
        if (a < prev) return fail("arrival_s decreases");
        if (pl < 1 || dl < 1 || pl > (1 << 30) || dl > (1 << 28)) return fail("lengths out of range");
        if (r == c.first_row) { c.first_a = a; c.first_ok = true; c.first_row_line = ln; }
        prev = a;
        c.last_a = a;
        t.arr[r] = a;
        t.pl[r] = (int32_t)pl;
        t.dl[r] = (int32_t)dl;
        ++r;
      }
      ++ln;
      return true;
    });
  });
  // first error in file order: a chunk's own error, or a seam where the
  // chunk's first arrival is below the last arrival before it
  size_t bad = 0;
  std::string msg;
  double last = -INFINITY;
  for (auto& c : ch) {
    if (c.first_ok && c.first_a < last) {  // precedes any later error in the chunk
      bad = c.first_row_line;
      msg = "arrival_s decreases";
      break;
    }
    if (c.err_line) { bad = c.err_line; msg = c.err; break; }
    if (c.rows) last = c.last_a;
  }
  if (bad) throw ConfigError(path + ":" + std::to_string(bad) + ": " + msg);
  return t;
}
std::string trace_csv(const Trace& t) {
  std::string o = "#kvsim-trace v1\nid,arrival_s,prompt_len,decode_len\n";
  for (size_t i = 0; i < t.arr.size(); ++i)
    o += std::to_string(i) + "," + num(t.arr[i]) + "," + std::to_string(t.pl[i]) + "," + std::to_string(t.dl[i]) + "\n";
  return o;
}

// ------------------------------------------------------------------ points
struct PointMeta {
  std::string policy, device;
  double rate;
  int instances;
  uint64_t seed;
  double resource = NAN;  // resource-sweep: the swept per-device value
};

kvsim_point_desc base_point(const jl::Value& c, const jl::Value& dev) {
  kvsim_point_desc p;
  kvsim_point_defaults(&p);
  const jl::Value& m = *c.find("model");
  p.param_count = m.find("param_count")->num;
  p.num_layers = (int32_t)m.find("num_layers")->num;
  p.hidden_dim = (int32_t)m.find("hidden_dim")->num;
  p.num_kv_heads = (int32_t)m.find("num_kv_heads")->num;
  p.head_dim = (int32_t)m.find("head_dim")->num;
  p.bytes_per_value = (int32_t)m.find("bytes_per_value")->num;
  p.peak_flops = dev.find("peak_flops")->num;
  p.hbm_capacity = dev.find("hbm_capacity")->num;
  p.hbm_bandwidth = dev.find("hbm_bandwidth")->num;
  p.link_bandwidth = dev.find("link_bandwidth")->num;
  p.num_devices = (int32_t)c.find("num_devices")->num;
  p.tensor_parallel = p.num_devices;
  p.memory_reserve_fraction = c.find("memory_reserve_fraction")->num;
  const jl::Value& e = *c.find("efficiency");
  p.compute_eff = e.find("compute_eff")->num;
  p.mem_bw_eff = e.find("mem_bw_eff")->num;
  p.link_eff = e.find("link_eff")->num;
  p.link_mode = c.find("link_aggregation")->str == "striped" ? KVSIM_LINK_STRIPED : KVSIM_LINK_SINGLE;
  p.num_prefill_instances = (int32_t)c.find("num_prefill_instances")->num;
  p.prefill_token_budget = (int32_t)c.find("prefill_token_budget")->num;
  const jl::Value& w = *c.find("workload");
  p.prompt_min = (int32_t)w.find("prompt_range")->arr[0].num;
  p.prompt_max = (int32_t)w.find("prompt_range")->arr[1].num;
  p.decode_min = (int32_t)w.find("decode_range")->arr[0].num;
  p.decode_max = (int32_t)w.find("decode_range")->arr[1].num;
  p.arrival_process = c.find("arrival_process")->str == "poisson" ? KVSIM_ARRIVAL_POISSON : KVSIM_ARRIVAL_FIXED;
  const jl::Value& d = *c.find("duration_s");
  p.duration_s = d.is_str() ? INFINITY : d.num;
  p.warmup_s = c.find("warmup_s")->num;
  const jl::Value& dm = *c.find("degraded_mode");
  const jl::Value& lv = *c.find("inter_pair_leveling");
  p.accellm_flags = (dm.find("enabled")->b ? KVSIM_ACCELLM_DEGRADED : 0) | (lv.find("enabled")->b ? KVSIM_ACCELLM_LEVELING : 0);
  p.splitwise_cobatch = c.find("splitwise_cobatch")->b ? 1 : 0;
  p.first_token_decode = c.find("first_token_decode")->b ? 1 : 0;
  p.degraded_trigger_ticks = (int32_t)dm.find("trigger_ticks")->num;
  p.degraded_redundancy = dm.find("redundancy_threshold")->num;
  p.degraded_exit_fill = dm.find("exit_fill")->num;
  p.dual_copy_fraction = dm.find("dual_copy_fraction")->num;
  p.leveling_link_fraction = lv.find("link_fraction")->num;
  p.policy_timer_s = c.find("policy_timer_s")->num;
  return p;
}

int policy_code(const std::string& s) {
  return s == "accellm" ? KVSIM_POLICY_ACCELLM : s == "splitwise_static" ? KVSIM_POLICY_SPLITWISE : KVSIM_POLICY_UNIFIED;
}

int64_t derive_requests(double rate, double duration) {
  // cap for duration-bound generation: lambda*D + 20 sqrt(lambda*D) + 1000
  const double m = rate * duration;
  return (int64_t)std::ceil(m + 20.0 * std::sqrt(m) + 1000.0);
}

void expand(const jl::Value& c, const Trace* trace, std::vector<kvsim_point_desc>& pts, std::vector<PointMeta>& meta,
            bool resource_axis = false) {
  const int64_t nreq = (int64_t)c.find("num_requests")->num;
  const jl::Value& d = *c.find("duration_s");
  const double dur = d.is_str() ? INFINITY : d.num;
  std::vector<double> rates;
  for (auto& r : c.find("rates")->arr) rates.push_back(r.num);
  if (trace) rates = {0.0};
  std::vector<double> rvals = {NAN};
  std::string rkind;
  if (resource_axis) {
    rvals.clear();
    for (auto& e : c.find("resource")->find("values")->arr) rvals.push_back(e.num);
    rkind = c.find("resource")->find("kind")->str;
  }
  for (double rv : rvals)
  for (auto& dev : c.find("sweep_devices")->arr)
    for (auto& ni : c.find("sweep_instances")->arr)
      for (auto& pol : c.find("policies")->arr)
        for (double rate : rates)
          for (auto& sd : c.find("seeds")->arr) {
            kvsim_point_desc p = base_point(c, dev);
            p.policy = policy_code(pol.str);
            p.num_instances = (int32_t)ni.num;
            p.rate = rate;
            p.seed = (uint64_t)sd.num;
            if (trace) {
              p.trace_index = 0;
              p.num_requests = (int64_t)trace->arr.size();
            } else {
              p.num_requests = nreq > 0 ? nreq : derive_requests(rate, std::isinf(dur) ? 300.0 : dur);
            }
            if (resource_axis) {
              if (rkind == "hbm_capacity") p.hbm_capacity = rv;
              else p.link_bandwidth = rv;
            }
            p.user_tag = pts.size();
            pts.push_back(p);
            meta.push_back(PointMeta{pol.str, dev.find("name")->str, rate, p.num_instances, p.seed, rv});
          }
}

// ------------------------------------------------------------------ running
struct RunOut {
  std::vector<kvsim_point_summary> sum;
  std::vector<kvsim_request_record> recs;
  std::vector<int64_t> rec_off;
  std::vector<kvsim_instance_record> inst;       // point i at i * KVSIM_MAX_INSTANCES
  std::vector<std::vector<kvsim_event_record>> ev;  // complete per-point event logs
};

// Event logs: each chunk runs with a bounded per-point buffer (so host and
// device memory stay bounded whatever the sweep size); a point whose log
// overflowed it is re-run alone with a buffer of its exact event count
// (the simulation is deterministic), so every written log is complete.
constexpr size_t kEvBytesPerChunk = size_t(256) << 20;
constexpr size_t kEvCapStart = size_t(1) << 16;

// One host thread per GPU pulling chunks of points from a shared counter;
// results land at their point index, so the merge is deterministic and
// independent of the GPU count.
// One host thread per GPU pulling chunks from a shared cursor over the points
// sorted by estimated cost (guided self-scheduling, kvsim_shard.hpp); results
// land at their point index, so the merge is deterministic and independent of
// the GPU count. KVSIM_VIRTUAL_GPUS=1 lets
// --gpus exceed the visible devices (workers share devices round-robin): a
// test hook for the sharder on a one-GPU box, never a performance setting.
void run_points(const std::vector<kvsim_point_desc>& pts, const Trace* trace, int gpus, bool records, bool events,
                bool detail, RunOut& out) {
  const size_t n = pts.size();
  out.sum.assign(n, kvsim_point_summary{});
  out.rec_off.assign(n + 1, 0);
  for (size_t i = 0; i < n; ++i) out.rec_off[i + 1] = out.rec_off[i] + pts[i].num_requests;
  if (records) out.recs.assign((size_t)out.rec_off[n], kvsim_request_record{});
  out.inst.assign(n * KVSIM_MAX_INSTANCES, kvsim_instance_record{});
  if (events) out.ev.assign(n, {});
  kvsim_trace_view tv{};
  if (trace) tv = kvsim_trace_view{trace->arr.data(), trace->pl.data(), trace->dl.data(), (int64_t)trace->arr.size()};
  const int ndev = kvsim_gpu_device_count();
  if (ndev <= 0) throw std::runtime_error("no CUDA device available (kvsim has no CPU fallback)");
  const bool virt = std::getenv("KVSIM_VIRTUAL_GPUS") && std::atoi(std::getenv("KVSIM_VIRTUAL_GPUS")) != 0;
  if (gpus <= 0) gpus = 1;
  if (gpus > ndev && !virt) gpus = ndev;
  size_t min_chunk = std::max<size_t>(1, n / (64 * (size_t)gpus));
  if (events) min_chunk = std::min(min_chunk, std::max<size_t>(1, kEvBytesPerChunk / (kEvCapStart * sizeof(kvsim_event_record))));
  kvsim_host::ShardPlan plan = kvsim_host::make_plan(pts.data(), n, gpus, min_chunk);
  std::vector<kvsim_gpu_ctx*> ctx(gpus, nullptr);
  std::mutex open_mu;
  auto chunk = [&](int w, const std::vector<int64_t>& idx, std::vector<kvsim_point_summary>& res,
                   std::string& e) -> int {
    char err[512] = {0};
    if (!ctx[w]) {
      std::lock_guard<std::mutex> g(open_mu);
      if (kvsim_gpu_open(w % ndev, &ctx[w], err, sizeof err) != 0) { e = err; return KVSIM_E_CUDA; }
    }
    const size_t m = idx.size();
    std::vector<kvsim_point_desc> sub(m);
    std::vector<int64_t> roff(m + 1, 0);
    for (size_t k = 0; k < m; ++k) {
      sub[k] = pts[idx[k]];
      roff[k + 1] = roff[k] + sub[k].num_requests;
    }
    std::vector<kvsim_request_record> rec(records ? (size_t)roff[m] : 0);
    std::vector<kvsim_instance_record> ins(m * KVSIM_MAX_INSTANCES);
    std::vector<kvsim_event_record> evbuf(events ? m * kEvCapStart : 0);
    std::vector<int64_t> evcnt(events ? m : 0);
    kvsim_run_opts o{};
    o.detail = detail ? 1 : 0;
    o.recs = records ? rec.data() : nullptr;
    o.inst = ins.data();
    if (events) {
      o.ev = evbuf.data();
      o.ev_cap = kEvCapStart;
      o.ev_count = evcnt.data();
    }
    int rc = kvsim_gpu_run_ex(ctx[w], sub.data(), m, trace ? &tv : nullptr, trace ? 1 : 0, res.data(), &o, err, sizeof err);
    if (rc != 0) { e = err; return rc; }
    for (size_t k = 0; k < m; ++k) {
      const size_t i = (size_t)idx[k];
      if (records)
        std::copy(rec.begin() + roff[k], rec.begin() + roff[k + 1], out.recs.begin() + out.rec_off[i]);
      std::copy(ins.begin() + k * KVSIM_MAX_INSTANCES, ins.begin() + (k + 1) * KVSIM_MAX_INSTANCES,
                out.inst.begin() + i * KVSIM_MAX_INSTANCES);
      if (!events) continue;
      const int64_t c = evcnt[k];
      if (c <= (int64_t)kEvCapStart) {
        out.ev[i].assign(evbuf.begin() + k * kEvCapStart, evbuf.begin() + k * kEvCapStart + c);
        continue;
      }
      // overflowed: rerun this point alone with an exact-size log
      std::vector<kvsim_event_record> big((size_t)c);
      int64_t c2 = 0;
      kvsim_point_summary s2{};
      kvsim_run_opts o2{};
      o2.detail = detail ? 1 : 0;
      o2.ev = big.data();
      o2.ev_cap = (size_t)c;
      o2.ev_count = &c2;
      rc = kvsim_gpu_run_ex(ctx[w], &sub[k], 1, trace ? &tv : nullptr, trace ? 1 : 0, &s2, &o2, err, sizeof err);
      if (rc != 0) { e = err; return rc; }
      if (c2 != c) { e = "event count changed on rerun (non-deterministic run)"; return KVSIM_E_INTERNAL; }
      out.ev[i].swap(big);
    }
    return KVSIM_OK;
  };
  std::string e;
  const int rc = kvsim_host::run_plan(plan, out.sum.data(), chunk, e);
  for (auto* c : ctx) kvsim_gpu_close(c);
  if (rc != 0) throw std::runtime_error(e);
}

// ------------------------------------------------------------------ outputs
const char* kSummaryCols = "policy,rate,ttft_mean,ttft_p95,tbt_mean,tbt_max,jct_mean,jct_p95,cost_eff,idle_frac,peak_kv_gb,link_prefill_gb,link_mirror_gb";

std::string summary_row(const PointMeta& m, const kvsim_point_summary& s) {
  return m.policy + "," + num(m.rate) + "," + num(s.ttft_mean) + "," + num(s.ttft_p95) + "," + num(s.tbt_mean) + "," +
         num(s.tbt_max) + "," + num(s.jct_mean) + "," + num(s.jct_p95) + "," + num(s.cost_eff) + "," +
         num(s.idle_frac) + "," + num(s.peak_kv_gb) + "," + num(s.link_prefill_gb) + "," + num(s.link_mirror_gb);
}

jl::Value summary_json(const kvsim_point_summary& s) {
  jl::Value o = jl::Value::object();
  auto I = [&](const char* k, int64_t v) { o.set(k, jl::Value::number((double)v)); };
  auto D = [&](const char* k, double v) { o.set(k, std::isnan(v) ? jl::Value() : jl::Value::number(v)); };
  I("status", s.status);
  I("num_instances", s.num_instances);
  I("n_requests", s.n_requests); I("n_completed", s.n_completed); I("n_measured", s.n_measured);
  I("tokens_total", s.tokens_total); I("tokens_window", s.tokens_window);
  I("n_events", s.n_events); I("n_steps", s.n_steps); I("n_prefills", s.n_prefills);
  I("n_moves", s.n_moves); I("n_preemptions", s.n_preemptions); I("n_evictions", s.n_evictions);
  I("peak_kv_tokens", s.peak_kv_tokens); I("link_prefill_tokens", s.link_prefill_tokens);
  I("link_mirror_tokens", s.link_mirror_tokens); I("link_leveling_tokens", s.link_leveling_tokens);
  I("n_timer_ticks", s.n_timer_ticks); I("n_mode_switches", s.n_mode_switches);
  D("makespan_s", s.makespan_s);
  D("ttft_mean", s.ttft_mean); D("ttft_p50", s.ttft_p50); D("ttft_p95", s.ttft_p95); D("ttft_max", s.ttft_max);
  D("tbt_mean", s.tbt_mean); D("tbt_max", s.tbt_max);
  D("jct_mean", s.jct_mean); D("jct_p50", s.jct_p50); D("jct_p95", s.jct_p95); D("jct_max", s.jct_max);
  D("cost_eff", s.cost_eff); D("idle_frac", s.idle_frac); D("peak_kv_gb", s.peak_kv_gb);
  D("link_prefill_gb", s.link_prefill_gb); D("link_mirror_gb", s.link_mirror_gb);
  D("busy_s_total", s.busy_s_total);
  D("ttft_queue_mean", s.ttft_queue_mean);
  D("tbt_p50", s.tbt_p50); D("tbt_p95", s.tbt_p95);
  D("idle_runnable_s", s.idle_runnable_s);
  I("n_tbt_samples", s.n_tbt_samples);
  return o;
}

const char* ev_name(int k) {
  static const char* names[] = {"?",    "arrive", "prefill_start", "prefill_done", "step_start", "step_end",
                                "move", "evict",  "preempt",       "role",         "transfer",   "wake",
                                "join", "copy",   "timer",         "level",        "mode"};
  return (k >= 0 && k <= 16) ? names[k] : "?";
}

jl::Value meta_json(const jl::Value& cfg, const std::string& cmd) {
  jl::Value m = jl::Value::object();
  const std::string canon = jl::dump(cfg, 0);
  char h[32];
  std::snprintf(h, sizeof h, "%016llx", (unsigned long long)fnv1a(canon));
  m.set("tool_version", jl::Value::string(kToolVersion));
  m.set("command", jl::Value::string(cmd));
  m.set("config_hash", jl::Value::string(h));
  m.set("seeds", *cfg.find("seeds"));
  m.set("config", cfg);
  return m;
}

// compare: per (rate, instances, device, seed) group, every
// policy's metrics as ratios to the first policy of the config. The trace
// fingerprint hashes everything that defines the generated trace (the
// generator is a pure function of it), so equal fingerprints = identical traces.
jl::Value compare_table(const jl::Value& cfg, const std::vector<PointMeta>& meta,
                        const std::vector<kvsim_point_summary>& sum) {
  jl::Value rows = jl::Value::array();
  const std::string first = cfg.find("policies")->arr.at(0).str;
  const std::string wl = jl::dump(*cfg.find("workload"), 0) + jl::dump(*cfg.find("duration_s"), 0) +
                         jl::dump(*cfg.find("num_requests"), 0) + cfg.find("arrival_process")->str;
  for (size_t i = 0; i < meta.size(); ++i) {
    if (meta[i].policy != first) continue;
    jl::Value g = jl::Value::object();
    char fp[32];
    std::snprintf(fp, sizeof fp, "%016llx",
                  (unsigned long long)fnv1a(wl + num(meta[i].rate) + std::to_string(meta[i].seed)));
    g.set("rate", jl::Value::number(meta[i].rate));
    g.set("instances", jl::Value::number(meta[i].instances));
    g.set("device", jl::Value::string(meta[i].device));
    g.set("seed", jl::Value::number((double)meta[i].seed));
    g.set("trace_fingerprint", jl::Value::string(fp));
    jl::Value ratios = jl::Value::object();
    for (size_t j = 0; j < meta.size(); ++j) {
      if (meta[j].rate != meta[i].rate || meta[j].instances != meta[i].instances || meta[j].device != meta[i].device ||
          meta[j].seed != meta[i].seed)
        continue;
      jl::Value m = jl::Value::object();
      auto ratio = [](double a, double b) { return (std::isnan(a) || std::isnan(b) || b == 0) ? jl::Value() : jl::Value::number(a / b); };
      m.set("cost_eff", ratio(sum[j].cost_eff, sum[i].cost_eff));
      m.set("jct_mean", ratio(sum[j].jct_mean, sum[i].jct_mean));
      m.set("ttft_mean", ratio(sum[j].ttft_mean, sum[i].ttft_mean));
      m.set("tbt_mean", ratio(sum[j].tbt_mean, sum[i].tbt_mean));
      m.set("tbt_max", ratio(sum[j].tbt_max, sum[i].tbt_max));
      ratios.set(meta[j].policy, m);
    }
    g.set("ratios_vs_" + first, ratios);
    rows.push(g);
  }
  return rows;
}

// resource-sweep knees: per policy, the smallest resource value
// whose JCT is within 1% of the policy's best JCT and whose cost efficiency is
// within 1% of its best; failed points (e.g. capacity below the weights) are
// skipped.
jl::Value resource_knees(const std::vector<PointMeta>& meta, const std::vector<kvsim_point_summary>& sum) {
  jl::Value out = jl::Value::array();
  std::vector<std::string> pols;
  for (auto& m : meta)
    if (std::find(pols.begin(), pols.end(), m.policy) == pols.end()) pols.push_back(m.policy);
  for (auto& pol : pols) {
    double best_jct = INFINITY, best_ce = -INFINITY;
    for (size_t i = 0; i < meta.size(); ++i)
      if (meta[i].policy == pol && sum[i].status == 0) {
        best_jct = std::min(best_jct, sum[i].jct_mean);
        best_ce = std::max(best_ce, sum[i].cost_eff);
      }
    double knee = NAN;
    for (size_t i = 0; i < meta.size(); ++i)
      if (meta[i].policy == pol && sum[i].status == 0 && sum[i].jct_mean <= 1.01 * best_jct &&
          sum[i].cost_eff >= 0.99 * best_ce)
        if (std::isnan(knee) || meta[i].resource < knee) knee = meta[i].resource;
    jl::Value k = jl::Value::object();
    k.set("policy", jl::Value::string(pol));
    k.set("knee", std::isnan(knee) ? jl::Value() : jl::Value::number(knee));
    k.set("best_jct_mean", std::isinf(best_jct) ? jl::Value() : jl::Value::number(best_jct));
    k.set("best_cost_eff", std::isinf(best_ce) ? jl::Value() : jl::Value::number(best_ce));
    out.push(k);
  }
  return out;
}

struct Args {
  std::string cmd, config, out = "out";
  bool emit_events = false, has_seed = false;
  uint64_t seed = 0;
  int gpus = 1;
};

[[noreturn]] void usage() {
  std::fprintf(stderr,
               "usage: kvsim run|sweep|resource-sweep|curves|gen-trace|validate-config --config PATH [--seed N] [--out DIR] "
               "[--emit-events] [--gpus N]\n");
  std::exit(2);
}

Args parse_args(int argc, char** argv) {
  if (argc < 2) usage();
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage();
      return argv[++i];
    };
    if (s == "--config") a.config = val();
    else if (s == "--out") a.out = val();
    else if (s == "--seed") { a.seed = std::strtoull(val().c_str(), nullptr, 10); a.has_seed = true; }
    else if (s == "--emit-events") a.emit_events = true;
    else if (s == "--gpus") a.gpus = std::atoi(val().c_str());
    else usage();
  }
  if (a.config.empty()) usage();
  return a;
}

int cmd_main(const Args& a) {
  jl::Value raw = jl::parse(read_file(a.config));
  if (a.has_seed && raw.is_obj()) {
    jl::Value s = jl::Value::array();
    s.push(jl::Value::number((double)a.seed));
    raw.set("seeds", s);
    for (size_t i = 0; i < raw.obj.size(); ++i)
      if (raw.obj[i].first == "seed") { raw.obj.erase(raw.obj.begin() + i); break; }
  }
  const std::string cmdk = a.cmd == "validate-config" ? "run" : a.cmd;
  if (a.cmd == "resource-sweep" && !raw.find("resource")) throw ConfigError("resource-sweep needs a \"resource\" block");
  jl::Value cfg = resolve(raw, cmdk);
  // host-side validation of every point (SPEC.md:416 messages)
  Trace trace;
  const bool has_trace = cfg.find("trace") != nullptr;
  if (has_trace) trace = load_trace(cfg.find("trace")->str);
  std::vector<kvsim_point_desc> pts;
  std::vector<PointMeta> meta;
  expand(cfg, has_trace ? &trace : nullptr, pts, meta, a.cmd == "resource-sweep");
  if (a.cmd == "run" || a.cmd == "validate-config") {
    char err[256];
    for (auto& p : pts) {
      if (kvsim_point_validate(&p, err, sizeof err) != 0) throw ConfigError(err);
    }
  }
  if (a.cmd == "validate-config") {
    if (has_trace) {  // what load_trace ingested: row count, length sums, FNV-1a of the arrival bits
      uint64_t h = 1469598103934665603ull;
      int64_t ps = 0, ds = 0;
      for (size_t i = 0; i < trace.arr.size(); ++i) {
        uint64_t b;
        std::memcpy(&b, &trace.arr[i], 8);
        for (int k = 0; k < 8; ++k) { h ^= (b >> (8 * k)) & 255u; h *= 1099511628211ull; }
        ps += trace.pl[i];
        ds += trace.dl[i];
      }
      char hx[32];
      std::snprintf(hx, sizeof hx, "%016llx", (unsigned long long)h);
      jl::Value ts = jl::Value::object();
      ts.obj.push_back({"rows", jl::Value::number((double)trace.arr.size())});
      ts.obj.push_back({"prompt_tokens", jl::Value::number((double)ps)});
      ts.obj.push_back({"decode_tokens", jl::Value::number((double)ds)});
      ts.obj.push_back({"arrival_fnv1a", jl::Value::string(hx)});
      ts.obj.push_back({"pinned", jl::Value::boolean(trace.arr.pinned())});
      cfg.obj.push_back({"trace_summary", ts});
    }
    std::printf("%s\n", jl::dump(cfg).c_str());
    return 0;
  }
  mkdirs(a.out);
  if (a.cmd == "curves") {
    // perfmodel throughput_curves (host API)
    const jl::Value* cv = cfg.find("curves");
    std::vector<int64_t> lens = {100, 500, 1000}, batches;
    for (int b = 1; b <= 256; b *= 2) batches.push_back(b);
    std::string phase = "decode";
    if (cv && cv->is_obj()) {
      if (cv->find("lengths")) { lens.clear(); for (auto& e : cv->find("lengths")->arr) lens.push_back((int64_t)e.num); }
      if (cv->find("batch_sizes")) { batches.clear(); for (auto& e : cv->find("batch_sizes")->arr) batches.push_back((int64_t)e.num); }
      if (cv->find("phase") && cv->find("phase")->is_str()) phase = cv->find("phase")->str;
    }
    if (lens.empty() || batches.empty()) throw ConfigError("curves: empty lengths or batch_sizes");
    const kvsim_point_desc& p = pts.at(0);
    // the grid is evaluated on the device (K1, kvsim_gpu_curves); without a
    // device, by the reference's host perfmodel API (the same math, bit for
    // bit: csrc/kvsim_math.cuh is shared)
    kvsim_gpu_ctx* ctx = nullptr;
    char err[512];
    const bool dev = kvsim_gpu_device_count() > 0 && kvsim_gpu_open(0, &ctx, err, sizeof err) == 0;
    kvsim::ModelSpec ms{"m", p.param_count, p.num_layers, p.hidden_dim, p.num_kv_heads, p.head_dim, p.bytes_per_value};
    kvsim::InstanceSpec is{{"d", p.peak_flops, p.hbm_capacity, p.hbm_bandwidth, p.link_bandwidth}, p.num_devices,
                           p.num_devices, p.memory_reserve_fraction};
    kvsim::EfficiencyFactors ef{p.compute_eff, p.mem_bw_eff, p.link_eff};
    std::string o = "phase,length,batch,latency_s,tokens_per_s\n";
    for (const char* ph : {"prefill", "decode"}) {
      if (phase != "both" && phase != ph) continue;
      const bool pre = std::string(ph) == "prefill";
      std::vector<double> lat(lens.size() * batches.size()), tps(lat.size());
      if (dev) {
        if (kvsim_gpu_curves(ctx, &p, lens.data(), lens.size(), batches.data(), batches.size(), pre ? 0 : 1, lat.data(),
                             tps.data(), err, sizeof err) != 0)
          throw std::runtime_error(err);
      } else {
        auto rows = kvsim::throughput_curves(ms, is, ef, lens, batches, pre ? kvsim::Phase::kPrefill : kvsim::Phase::kDecode);
        for (size_t r = 0; r < rows.size(); ++r) { lat[r] = rows[r].latency_s; tps[r] = rows[r].tokens_per_s; }
      }
      for (size_t li = 0; li < lens.size(); ++li)
        for (size_t bi = 0; bi < batches.size(); ++bi) {
          const size_t r = li * batches.size() + bi;
          o += std::string(ph) + "," + std::to_string(lens[li]) + "," + std::to_string(batches[bi]) + "," + num(lat[r]) +
               "," + num(tps[r]) + "\n";
        }
    }
    if (ctx) kvsim_gpu_close(ctx);
    write_file(a.out + "/curves.csv", o);
    jl::Value m = meta_json(cfg, a.cmd);
    m.set("evaluated_on", jl::Value::string(dev ? "gpu (K1 kvsim_perf_kernel)" : "host (perfmodel.hpp API)"));
    write_file(a.out + "/meta.json", jl::dump(m) + "\n");
    return 0;
  }
  if (a.cmd == "gen-trace") {
    kvsim_gpu_ctx* ctx = nullptr;
    char err[512];
    if (kvsim_gpu_open(0, &ctx, err, sizeof err) != 0) throw std::runtime_error(err);
    const kvsim_point_desc& p = pts.at(0);
    Trace t;
    t.arr.resize(p.num_requests);
    t.pl.resize(p.num_requests);
    t.dl.resize(p.num_requests);
    int64_t nn = 0;
    if (kvsim_gpu_gen_trace(ctx, &p, t.arr.data(), t.pl.data(), t.dl.data(), &nn, err, sizeof err) != 0)
      throw std::runtime_error(err);
    kvsim_gpu_close(ctx);
    t.arr.resize(nn);
    t.pl.resize(nn);
    t.dl.resize(nn);
    write_file(a.out + "/trace.csv", trace_csv(t));
    return 0;
  }
  if (a.cmd != "run" && a.cmd != "sweep" && a.cmd != "resource-sweep") usage();
  const bool records = cfg.find("emit_records")->b;
  const bool detail = cfg.find("detail_metrics")->b;
  RunOut r;
  logf(1, "%s: %zu point(s) on %d GPU(s)", a.cmd.c_str(), pts.size(), a.gpus);
  run_points(pts, has_trace ? &trace : nullptr, a.gpus, records, a.emit_events, detail, r);
  // summary.csv (stable 13 columns) + sweep axes
  std::string csv = std::string(kSummaryCols) + ",instances,device,seed,status\n";
  for (size_t i = 0; i < pts.size(); ++i)
    csv += summary_row(meta[i], r.sum[i]) + "," + std::to_string(meta[i].instances) + "," + meta[i].device + "," +
           std::to_string(meta[i].seed) + "," + std::to_string(r.sum[i].status) + "\n";
  write_file(a.out + "/summary.csv", csv);
  jl::Value report = jl::Value::object();
  report.set("tool_version", jl::Value::string(kToolVersion));
  jl::Value points = jl::Value::array();
  for (size_t i = 0; i < pts.size(); ++i) {
    jl::Value e = jl::Value::object();
    e.set("policy", jl::Value::string(meta[i].policy));
    e.set("rate", jl::Value::number(meta[i].rate));
    e.set("instances", jl::Value::number(meta[i].instances));
    e.set("device", jl::Value::string(meta[i].device));
    e.set("seed", jl::Value::number((double)meta[i].seed));
    e.set("summary", summary_json(r.sum[i]));
    {
      // per-instance idle fraction and peak KV
      const kvsim_point_summary& su = r.sum[i];
      const double window = su.makespan_s - pts[i].warmup_s;
      const double kvb = 2.0 * pts[i].num_layers * pts[i].num_kv_heads * pts[i].head_dim * pts[i].bytes_per_value;
      jl::Value ia = jl::Value::array();
      for (int x = 0; x < su.num_instances; ++x) {
        const kvsim_instance_record& q = r.inst[i * KVSIM_MAX_INSTANCES + x];
        jl::Value o = jl::Value::object();
        o.set("instance", jl::Value::number(x));
        o.set("initial_role", jl::Value::string(q.initial_role ? "prefill" : "decode"));
        o.set("busy_s", jl::Value::number(q.busy_s));
        o.set("idle_frac", window > 0 ? jl::Value::number(1.0 - q.busy_s / window) : jl::Value());
        o.set("idle_runnable_s", jl::Value::number(q.idle_runnable_s));
        o.set("peak_kv_gb", jl::Value::number((double)q.peak_kv_tokens * kvb / 1e9));
        ia.push(o);
      }
      e.set("instances_detail", ia);
      jl::Value q = jl::Value::object();
      q.set("max", jl::Value::number((double)su.queue_depth_max));
      q.set("time_avg", std::isnan(su.queue_depth_avg) ? jl::Value() : jl::Value::number(su.queue_depth_avg));
      e.set("queue_depth", q);
    }
    if (records && a.cmd == "run") {
      jl::Value rq = jl::Value::array();
      for (int64_t k = 0; k < r.sum[i].n_requests; ++k) {
        const kvsim_request_record& q = r.recs[r.rec_off[i] + k];
        jl::Value x = jl::Value::object();
        x.set("id", jl::Value::number((double)k));
        x.set("arrival_s", jl::Value::number(q.arrival_s));
        x.set("ttft_s", jl::Value::number(q.first_token_s - q.arrival_s));
        x.set("jct_s", jl::Value::number(q.completion_s - q.arrival_s));
        x.set("tbt_max_s", jl::Value::number(q.tbt_max_s));
        x.set("tbt_mean_s", q.decode_len > 1 ? jl::Value::number((q.completion_s - q.first_token_s) / (q.decode_len - 1)) : jl::Value());
        x.set("queue_wait_s", jl::Value::number(q.prefill_start_s - q.arrival_s));
        x.set("prompt_len", jl::Value::number(q.prompt_len));
        x.set("decode_len", jl::Value::number(q.decode_len));
        rq.push(x);
      }
      e.set("requests", rq);
    }
    points.push(e);
  }
  report.set("points", points);
  if (a.cmd == "sweep") {
    // saturation annotation: argmax cost_eff over rate per (policy, instances, device, seed)
    jl::Value sat = jl::Value::array();
    std::vector<bool> done(pts.size(), false);
    for (size_t i = 0; i < pts.size(); ++i) {
      if (done[i]) continue;
      double best = -1, best_rate = 0;
      for (size_t j = i; j < pts.size(); ++j) {
        if (meta[j].policy != meta[i].policy || meta[j].instances != meta[i].instances ||
            meta[j].device != meta[i].device || meta[j].seed != meta[i].seed)
          continue;
        done[j] = true;
        if (r.sum[j].cost_eff > best) { best = r.sum[j].cost_eff; best_rate = meta[j].rate; }
      }
      jl::Value s = jl::Value::object();
      s.set("policy", jl::Value::string(meta[i].policy));
      s.set("instances", jl::Value::number(meta[i].instances));
      s.set("device", jl::Value::string(meta[i].device));
      s.set("seed", jl::Value::number((double)meta[i].seed));
      s.set("saturation_rate", jl::Value::number(best_rate));
      s.set("max_cost_eff", jl::Value::number(best));
      sat.push(s);
    }
    report.set("saturation", sat);
    report.set("compare", compare_table(cfg, meta, r.sum));
    // long form (policy, rate, metric, value)
    std::string lf = "policy,rate,instances,device,seed,metric,value\n";
    const char* cols[] = {"ttft_mean", "ttft_p95", "tbt_mean", "tbt_max", "jct_mean", "jct_p95", "cost_eff",
                          "idle_frac", "peak_kv_gb", "link_prefill_gb", "link_mirror_gb"};
    for (size_t i = 0; i < pts.size(); ++i) {
      const kvsim_point_summary& s = r.sum[i];
      const double vals[] = {s.ttft_mean, s.ttft_p95, s.tbt_mean, s.tbt_max, s.jct_mean, s.jct_p95,
                             s.cost_eff, s.idle_frac, s.peak_kv_gb, s.link_prefill_gb, s.link_mirror_gb};
      for (int k = 0; k < 11; ++k)
        lf += meta[i].policy + "," + num(meta[i].rate) + "," + std::to_string(meta[i].instances) + "," +
              meta[i].device + "," + std::to_string(meta[i].seed) + "," + cols[k] + "," + num(vals[k]) + "\n";
    }
    write_file(a.out + "/sweep_long.csv", lf);
  }
  if (a.cmd == "resource-sweep") {
    const std::string kind = cfg.find("resource")->find("kind")->str;
    std::string rc = "policy,rate,instances,seed," + kind + ",jct_mean,cost_eff,ttft_mean,tbt_mean,peak_kv_gb,status\n";
    for (size_t i = 0; i < pts.size(); ++i)
      rc += meta[i].policy + "," + num(meta[i].rate) + "," + std::to_string(meta[i].instances) + "," +
            std::to_string(meta[i].seed) + "," + num(meta[i].resource) + "," + num(r.sum[i].jct_mean) + "," +
            num(r.sum[i].cost_eff) + "," + num(r.sum[i].ttft_mean) + "," + num(r.sum[i].tbt_mean) + "," +
            num(r.sum[i].peak_kv_gb) + "," + std::to_string(r.sum[i].status) + "\n";
    write_file(a.out + "/resource_sweep.csv", rc);
    report.set("knees", resource_knees(meta, r.sum));
  }
  write_file(a.out + "/report.json", jl::dump(report) + "\n");
  write_file(a.out + "/meta.json", jl::dump(meta_json(cfg, a.cmd)) + "\n");
  if (a.emit_events) {
    // queue-depth time series (SPEC.md:358 MetricsReport diagnostics), rebuilt
    // from the (complete) event logs: +1 per arrival and per preemption (the
    // request re-enters its queue), minus the prompts a prefill job (unified:
    // a co-batched iteration) takes; one row per timestamp with the depth
    // after that timestamp's events. Its max / time average are the device's
    // queue_depth_* summary fields (report.json).
    FILE* qf = std::fopen((a.out + "/queue_depth.csv").c_str(), "w");
    FILE* ef = std::fopen((a.out + "/events.jsonl").c_str(), "w");
    if (!qf || !ef) throw std::runtime_error("cannot write event outputs in " + a.out);
    std::fputs("point,t,depth\n", qf);
    for (size_t i = 0; i < pts.size(); ++i) {
      std::vector<std::pair<double, int64_t>> dv;
      for (const kvsim_event_record& e : r.ev[i]) {
        if (e.kind == KVSIM_EV_ARRIVE || e.kind == KVSIM_EV_PREEMPT) dv.push_back({e.t, 1});
        else if (e.kind == KVSIM_EV_PREFILL_START) dv.push_back({e.t, -(int64_t)e.a});
        else if (e.kind == KVSIM_EV_STEP_START && pts[i].policy == KVSIM_POLICY_UNIFIED && e.b > 0)
          dv.push_back({e.t, -(int64_t)e.b});
      }
      std::stable_sort(dv.begin(), dv.end(), [](auto& x, auto& y) { return x.first < y.first; });
      int64_t depth = 0;
      for (size_t j = 0; j < dv.size();) {
        const double t = dv[j].first;
        for (; j < dv.size() && dv[j].first == t; ++j) depth += dv[j].second;
        std::fprintf(qf, "%zu,%s,%lld\n", i, num(t).c_str(), (long long)depth);
      }
      for (const kvsim_event_record& e : r.ev[i])
        std::fprintf(ef, "{\"point\":%zu,\"t\":%s,\"kind\":\"%s\",\"inst\":%d,\"a\":%d,\"b\":%d,\"c\":%lld}\n", i,
                     num(e.t).c_str(), ev_name(e.kind), e.inst, e.a, e.b, (long long)e.c);
    }
    std::fclose(qf);
    std::fclose(ef);
  }
  int bad = 0;
  for (auto& s : r.sum) bad += s.status != 0;
  if (bad) logf(1, "%d point(s) reported errors (see status column)", bad);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (const char* l = std::getenv("KVSIM_LOG")) g_log = std::atoi(l);
  Args a = parse_args(argc, argv);
  try {
    return cmd_main(a);
  } catch (const ConfigError& e) {
    std::string o;
    jl::escape(o, e.what());
    std::fprintf(stderr, "{\"error\": %s, \"kind\": \"config\"}\n", o.c_str());
    return 2;
  } catch (const jl::ParseError& e) {
    std::string o;
    jl::escape(o, e.what());
    std::fprintf(stderr, "{\"error\": %s, \"kind\": \"config\"}\n", o.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::string o;
    jl::escape(o, e.what());
    std::fprintf(stderr, "{\"error\": %s, \"kind\": \"runtime\"}\n", o.c_str());
    return 3;
  }
}
