// decode_cli.cpp -- native (no Python) driver of the C ABI: the end-to-end
// path a C/C++ serving process takes, host buffers in and out.
//
//   build/decode_cli [streams] [heads] [ctx] [steps] [slow_tier 0|1]
//
// Creates one handle (the cfg2 shape by default: 256 streams x 4 heads,
// d = 128, 4K fp16 fast tier, K8/V4, fetch 0.45 per head), prefills `ctx`
// synthetic tokens on the device, then times `steps` synchronous
// ttkv_gpu_decode_step calls (q/k/v copied in from host memory, outputs copied
// back) with a host clock, after 3 warm-up steps, and prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../include/ttkv_gpu.h"

static int fail(ttkv_gpu* h, const char* what) {
  std::fprintf(stderr, "%s: %s\n", what, h ? ttkv_gpu_last_error(h) : ttkv_last_error());
  return 1;
}

int main(int argc, char** argv) {
  const uint32_t S = argc > 1 ? std::atoi(argv[1]) : 256;
  const uint32_t G = argc > 2 ? std::atoi(argv[2]) : 4;
  const uint64_t ctx = argc > 3 ? std::atoll(argv[3]) : 131072;
  const int steps = argc > 4 ? std::atoi(argv[4]) : 10;
  const uint32_t tier = argc > 5 ? std::atoi(argv[5]) : 0;
  const uint32_t d = 128;

  ttkv_tier_config cfg;
  ttkv_default_config(&cfg);
  cfg.d_k = cfg.d_v = d;
  cfg.block_size = 128;
  cfg.hbm_budget_bytes = 4096ull * 2 * d * 2;  // L_fast = 4096
  ttkv_selection_policy pol = {0, 0, 0.45};
  ttkv_gpu_options opt = {};
  opt.n_streams = S;
  opt.heads_per_stream = G;
  opt.reserve_tokens = ctx + steps + 3 + 256;
  opt.slow_tier = tier ? TTKV_SLOW_DEVICE : TTKV_SLOW_PINNED_HOST;
  ttkv_gpu* h = nullptr;
  if (ttkv_gpu_create(&cfg, &pol, &opt, &h)) return fail(nullptr, "create");
  if (ttkv_gpu_prefill_synthetic(h, ctx, 1)) return fail(h, "prefill");

  std::mt19937 gen(0);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> q((size_t)S * G * d), k((size_t)S * d), v((size_t)S * d);
  for (auto& x : q) x = nd(gen);
  for (auto& x : k) x = nd(gen);
  for (auto& x : v) x = nd(gen);
  std::vector<double> out((size_t)S * G * d);
  ttkv_step_report rep{};
  for (int i = 0; i < 3; ++i)
    if (ttkv_gpu_decode_step(h, q.data(), k.data(), v.data(), TTKV_DTYPE_F32, out.data(), &rep))
      return fail(h, "decode_step");
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i)
    if (ttkv_gpu_decode_step(h, q.data(), k.data(), v.data(), TTKV_DTYPE_F32, out.data(), &rep))
      return fail(h, "decode_step");
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() /
      steps;
  std::printf(
      "{\"driver\": \"tools/decode_cli.cpp (C ABI, host buffers)\", \"streams\": %u, "
      "\"heads_per_stream\": %u, \"ctx\": %llu, \"slow_tier\": \"%s\", \"steps\": %d, "
      "\"ms_per_step\": %.3f, \"tokens_per_s\": %.3f, \"union_blocks\": %llu, "
      "\"pcie_gbs\": %.2f}\n",
      S, G, (unsigned long long)ctx, tier ? "hbm" : "pinned host DRAM", steps, ms, 1000.0 / ms,
      (unsigned long long)rep.union_blocks, tier ? 0.0 : rep.pcie_bytes / (ms * 1e-3) / 1e9);
  ttkv_gpu_destroy(h);
  return 0;
}
