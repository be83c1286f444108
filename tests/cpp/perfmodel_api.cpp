// C++ client of the reference's perfmodel API (reference
// proj/include/kvsim/perfmodel.hpp:23-123) linked against libkvsim_gpu.so:
// the SPEC worked examples through the kvsim:: span signatures
// (SPEC.md:53-109), including the declared exceptions. Built and run by
// tests/test_perfmodel_cpp.py (no GPU needed: these are host functions).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "kvsim/perfmodel.hpp"

static int fails = 0;
#define CHECK(cond)                                          \
  do {                                                       \
    if (!(cond)) {                                           \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); \
      ++fails;                                               \
    }                                                        \
  } while (0)
static bool near(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::fabs(b); }

int main() {
  using namespace kvsim;
  const ModelSpec m70 = model_preset_llama2_70b();
  const DeviceSpec h100 = device_preset_h100(), ascend = device_preset_910b2();
  InstanceSpec ih{h100, 4, 4, 0.10}, ia{ascend, 4, 4, 0.10};
  EfficiencyFactors half{0.5, 1.0, 1.0}, one{1.0, 1.0, 1.0};
  CHECK(kv_bytes_per_token(m70) == 327680.0);
  CHECK(weight_bytes(m70) == 1.4e11);
  const std::vector<std::int64_t> p512{512}, p1000{1000}, two{512, 512};
  CHECK(near(prefill_latency(m70, ih, half, p512), 0.036586, 1e-4));
  CHECK(near(prefill_latency(m70, ia, half, p1000), 0.17828, 1e-4));
  // additivity: within 1 ulp
  const double a = prefill_latency(m70, ih, half, two), b = 2 * prefill_latency(m70, ih, half, p512);
  CHECK(std::fabs(a - b) <= std::fabs(b) * 2.3e-16);
  std::vector<std::int64_t> kv32(32, 500);
  CHECK(near(decode_step_latency(m70, ih, one, kv32), 0.01084, 1e-3));
  const std::vector<std::int64_t> kv1{100};
  CHECK(near(decode_step_latency(m70, ia, one, kv1), 0.019449, 1e-3));
  CHECK(near(transfer_latency(327.68e6, ih, one), 91.0e-6, 1e-3));     // SPEC.md:89 (striped)
  CHECK(transfer_latency(0.0, ih, one) == 0.0);
  CHECK(kv_capacity_tokens(m70, ih) == 451660);
  CHECK(kv_capacity_tokens(m70, ia) == 275878);
  // errors
  bool threw = false;
  try { prefill_latency(m70, ih, half, std::vector<std::int64_t>{}); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  threw = false;
  try { decode_step_latency(m70, ih, half, std::vector<std::int64_t>{}); } catch (const std::invalid_argument&) { threw = true; }
  CHECK(threw);
  threw = false;
  DeviceSpec tiny{"tiny", 1e12, 1e9, 1e12, 1e9};
  try { kv_capacity_tokens(m70, InstanceSpec{tiny, 4, 4, 0.1}); } catch (const std::exception&) { threw = true; }
  CHECK(threw);
  // throughput_curves: decode, length 500, batches {1, 32}
  const std::vector<std::int64_t> lens{500}, bs{1, 32};
  auto rows = throughput_curves(m70, ih, one, lens, bs, Phase::kDecode);
  CHECK(rows.size() == 2);
  CHECK(near(rows[0].latency_s, 0.01046, 1e-3) && near(rows[1].tokens_per_s, 2952, 1e-3));
  std::printf(fails ? "perfmodel_api: %d failure(s)\n" : "perfmodel_api: ok\n", fails);
  return fails ? 1 : 0;
}
