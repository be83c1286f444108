// perfmodel.cpp — bodies for the reference's perfmodel API
// (reference proj/include/kvsim/perfmodel.hpp:67-123, declarations only), on
// top of the explicitly-rounded shared math (kvsim_math.cuh) so that host
// answers equal the device kernels' bit for bit. Error messages follow
// SPEC.md:69,78,96.
#include "kvsim/perfmodel.hpp"

#include <cmath>
#include <stdexcept>

#include "kvsim_math.cuh"

namespace kvsim {
namespace {

kvsim_point_desc as_desc(const ModelSpec& m, const InstanceSpec& i, const EfficiencyFactors& e,
                         LinkAggregation mode = LinkAggregation::kStriped) {
  kvsim_point_desc p{};
  p.param_count = m.param_count;
  p.num_layers = m.num_layers;
  p.hidden_dim = m.hidden_dim;
  p.num_kv_heads = m.num_kv_heads;
  p.head_dim = m.head_dim;
  p.bytes_per_value = m.bytes_per_value;
  p.peak_flops = i.device.peak_flops;
  p.hbm_capacity = i.device.hbm_capacity;
  p.hbm_bandwidth = i.device.hbm_bandwidth;
  p.link_bandwidth = i.device.link_bandwidth;
  p.num_devices = i.num_devices;
  p.tensor_parallel = i.tensor_parallel;
  p.memory_reserve_fraction = i.memory_reserve_fraction;
  p.compute_eff = e.compute_eff;
  p.mem_bw_eff = e.mem_bw_eff;
  p.link_eff = e.link_eff;
  p.link_mode = mode == LinkAggregation::kSingleLink ? KVSIM_LINK_SINGLE : KVSIM_LINK_STRIPED;
  return p;
}

void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

}  // namespace

DeviceSpec device_preset_910b2() { return DeviceSpec{"910B2", 400e12, 64e9, 1.8e12, 392e9}; }
DeviceSpec device_preset_h100() { return DeviceSpec{"H100", 989e12, 80e9, 3.35e12, 900e9}; }
ModelSpec model_preset_llama2_70b() { return ModelSpec{"llama2-70b", 70e9, 80, 8192, 8, 128, 2}; }

void validate(const DeviceSpec& d) {
  require(d.peak_flops > 0 && d.hbm_capacity > 0 && d.hbm_bandwidth > 0 && d.link_bandwidth > 0,
          "DeviceSpec: all numeric fields must be > 0");
}
void validate(const ModelSpec& m) {
  require(m.param_count > 0 && m.num_layers > 0 && m.hidden_dim > 0 && m.num_kv_heads > 0 && m.head_dim > 0 &&
              m.bytes_per_value > 0,
          "ModelSpec: all fields must be > 0");
}
void validate(const InstanceSpec& i) {
  validate(i.device);
  require(i.num_devices >= 1, "InstanceSpec: num_devices must be >= 1");
  require(i.tensor_parallel == i.num_devices, "InstanceSpec: tensor_parallel must equal num_devices");
  require(i.memory_reserve_fraction >= 0 && i.memory_reserve_fraction < 1,
          "InstanceSpec: memory_reserve_fraction must be in [0,1)");
}
void validate(const EfficiencyFactors& e) {
  require(e.compute_eff > 0 && e.compute_eff <= 1 && e.mem_bw_eff > 0 && e.mem_bw_eff <= 1 && e.link_eff > 0 &&
              e.link_eff <= 1,
          "EfficiencyFactors: each factor must be in (0,1]");
}

double kv_bytes_per_token(const ModelSpec& m) {
  return kvsim_math::make_perf(as_desc(m, InstanceSpec{}, EfficiencyFactors{})).kvb;
}
double weight_bytes(const ModelSpec& m) {
  return kvsim_math::make_perf(as_desc(m, InstanceSpec{}, EfficiencyFactors{})).W;
}

double prefill_latency(const ModelSpec& m, const InstanceSpec& i, const EfficiencyFactors& e,
                       std::span<const std::int64_t> prompt_lengths) {
  if (prompt_lengths.empty()) throw std::invalid_argument("empty prefill batch");
  std::int64_t s1 = 0, s2 = 0;
  for (std::int64_t L : prompt_lengths) {
    if (L <= 0) throw std::invalid_argument("prompt length must be > 0");
    s1 += L;
    s2 += L * L;
  }
  return kvsim_math::prefill_latency(kvsim_math::make_perf(as_desc(m, i, e)), s1, s2);
}

double decode_step_latency(const ModelSpec& m, const InstanceSpec& i, const EfficiencyFactors& e,
                           std::span<const std::int64_t> kv_lengths) {
  if (kv_lengths.empty()) throw std::invalid_argument("empty decode batch");
  std::int64_t k = 0;
  for (std::int64_t L : kv_lengths) {
    if (L < 1) throw std::invalid_argument("kv length must be >= 1");
    k += L;
  }
  return kvsim_math::decode_latency(kvsim_math::make_perf(as_desc(m, i, e)), (std::int64_t)kv_lengths.size(), k);
}

double link_bandwidth_bytes_per_s(const InstanceSpec& i, const EfficiencyFactors& e, LinkAggregation mode) {
  return kvsim_math::make_perf(as_desc(ModelSpec{"", 1, 1, 1, 1, 1, 1}, i, e, mode)).link_bw;
}

double transfer_latency(double num_bytes, const InstanceSpec& i, const EfficiencyFactors& e, LinkAggregation mode) {
  if (num_bytes < 0) throw std::invalid_argument("num_bytes must be >= 0");
  return kvsim_math::transfer_latency(kvsim_math::make_perf(as_desc(ModelSpec{"", 1, 1, 1, 1, 1, 1}, i, e, mode)),
                                      num_bytes);
}

std::int64_t kv_capacity_tokens(const ModelSpec& m, const InstanceSpec& i) {
  const kvsim_math::Perf f = kvsim_math::make_perf(as_desc(m, i, EfficiencyFactors{}));
  if (!f.fits) throw std::invalid_argument("model does not fit in instance memory");
  return f.cap;
}

std::vector<CurvePoint> throughput_curves(const ModelSpec& m, const InstanceSpec& i, const EfficiencyFactors& e,
                                          std::span<const std::int64_t> lengths,
                                          std::span<const std::int64_t> batch_sizes, Phase phase) {
  const kvsim_math::Perf f = kvsim_math::make_perf(as_desc(m, i, e));
  std::vector<CurvePoint> rows;
  rows.reserve(lengths.size() * batch_sizes.size());
  for (std::int64_t L : lengths) {
    for (std::int64_t b : batch_sizes) {
      CurvePoint c;
      c.length = L;
      c.batch = b;
      if (phase == Phase::kPrefill) {
        c.latency_s = kvsim_math::prefill_latency(f, b * L, b * L * L);
        c.tokens_per_s = kvsim_math::kdiv((double)(b * L), c.latency_s);
      } else {
        c.latency_s = kvsim_math::decode_latency(f, b, b * L);
        c.tokens_per_s = kvsim_math::kdiv((double)b, c.latency_s);
      }
      rows.push_back(c);
    }
  }
  return rows;
}

}  // namespace kvsim
