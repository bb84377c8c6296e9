// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/core/src/*.cpp (in place, read-only) into
// oracle/_ref/libttkv_ref.so.  It is used (a) to pin the C restatement in
// oracle/ttkv_oracle.c, (b) to generate tests/golden/ fixtures and (c) as the
// timed CPU baseline in bench.py (cpu_baseline.kind = "reference").
//
// Nothing here re-implements reference logic: every call forwards to the
// reference's own API (engine.hpp:36-49, quantizer.hpp:48-63,
// relevance.hpp:23-34, workload.hpp:49, reference.hpp:14-18, harness.hpp:60).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ttkv/engine.hpp"
#include "ttkv/quantizer.hpp"
#include "ttkv/reference.hpp"
#include "ttkv/relevance.hpp"
#include "ttkv/sim.hpp"
#include "ttkv/tier_store.hpp"
#include "ttkv/workload.hpp"
#ifdef TTKV_REF_HAVE_HARNESS
#include "ttkv/harness.hpp"
#endif

using namespace ttkv;

namespace {

TierConfig make_cfg(uint64_t budget, uint32_t d_k, uint32_t d_v, uint32_t bytes_fp,
                    uint32_t block_size, uint32_t kb, uint32_t vb) {
  TierConfig c;
  c.hbm_budget_bytes = budget;
  c.d_k = d_k;
  c.d_v = d_v;
  c.bytes_full_precision = bytes_fp;
  c.block_size = block_size;
  c.key_bits = kb;
  c.value_bits = vb;
  return c;
}

SelectionPolicy make_policy(int has_top_k, uint64_t top_k, double frac) {
  SelectionPolicy p;
  if (has_top_k) p.top_k = top_k;
  p.fetch_fraction = frac;
  return p;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- Engine ------------------------------------------------------------------
void* ref_engine_create(uint64_t budget, uint32_t d_k, uint32_t d_v, uint32_t bytes_fp,
                        uint32_t block_size, uint32_t kb, uint32_t vb, int has_top_k,
                        uint64_t top_k, double frac, int literal_merge) {
  try {
    return new Engine(make_cfg(budget, d_k, d_v, bytes_fp, block_size, kb, vb),
                      make_policy(has_top_k, top_k, frac), EngineOptions{literal_merge != 0});
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_engine_destroy(void* e) { delete static_cast<Engine*>(e); }

int ref_engine_prefill(void* h, const float* keys, const float* values, uint64_t n) {
  auto* e = static_cast<Engine*>(h);
  const auto& cfg = e->config();
  try {
    std::vector<TokenKV> toks(n);
    const uint64_t base = e->store().appended_count();
    for (uint64_t t = 0; t < n; ++t) {
      toks[t].position = base + t;
      toks[t].key.assign(keys + t * cfg.d_k, keys + (t + 1) * cfg.d_k);
      toks[t].value.assign(values + t * cfg.d_v, values + (t + 1) * cfg.d_v);
    }
    e->prefill(toks);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

int ref_engine_decode_step(void* h, const float* q, const float* key, const float* value,
                           double* out, uint64_t* fetched, uint64_t cap, uint64_t* n_fetched,
                           uint64_t* n_scored, double* bytes, int* evicted) {
  auto* e = static_cast<Engine*>(h);
  const auto& cfg = e->config();
  try {
    TokenKV kv;
    kv.position = e->store().appended_count();
    kv.key.assign(key, key + cfg.d_k);
    kv.value.assign(value, value + cfg.d_v);
    const auto r = e->decode_step(std::span<const float>(q, cfg.d_k), std::move(kv));
    std::copy(r.output.begin(), r.output.end(), out);
    if (fetched)
      for (size_t i = 0; i < r.fetched_blocks.size() && i < cap; ++i)
        fetched[i] = r.fetched_blocks[i];
    if (n_fetched) *n_fetched = r.blocks_fetched;
    if (n_scored) *n_scored = r.blocks_scored;
    if (bytes) *bytes = r.bytes_transferred;
    if (evicted) *evicted = r.eviction_occurred ? 1 : 0;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

uint64_t ref_engine_slow_blocks(void* h) {
  return static_cast<Engine*>(h)->store().slow_blocks().size();
}
uint64_t ref_engine_fast_tokens(void* h) {
  return static_cast<Engine*>(h)->store().fast_token_count();
}
uint64_t ref_engine_l_fast(void* h) {
  return static_cast<Engine*>(h)->store().l_fast_capacity();
}

// Serialized bytes of slow block i (quantizer.cpp:248-274); returns length,
// writes at most cap bytes.
uint64_t ref_engine_serialize_block(void* h, uint64_t i, uint8_t* out, uint64_t cap) {
  const auto& slow = static_cast<Engine*>(h)->store().slow_blocks();
  if (i >= slow.size()) return 0;
  const auto bytes = serialize_block(slow[i]);
  if (out) std::memcpy(out, bytes.data(), std::min<uint64_t>(cap, bytes.size()));
  return bytes.size();
}

// ---- Free functions --------------------------------------------------------
uint64_t ref_quantize_serialize(const float* keys, const float* values, uint64_t rows,
                                uint32_t d_k, uint32_t d_v, uint32_t kb, uint32_t vb,
                                uint64_t block_id, uint64_t first_pos, uint8_t* out,
                                uint64_t cap) {
  KvBlock b;
  b.block_id = block_id;
  b.first_position = first_pos;
  b.last_position = first_pos + rows - 1;
  b.token_count = rows;
  b.d_k = d_k;
  b.d_v = d_v;
  b.keys.assign(keys, keys + rows * d_k);
  b.values.assign(values, values + rows * d_v);
  TierConfig c;
  c.key_bits = kb;
  c.value_bits = vb;
  const auto bytes = serialize_block(quantize_block(b, c));
  if (out) std::memcpy(out, bytes.data(), std::min<uint64_t>(cap, bytes.size()));
  return bytes.size();
}

double ref_score_block(const float* q, const float* c, uint64_t d) {
  return score_block(std::span<const float>(q, d), std::span<const float>(c, d));
}

uint64_t ref_select_top_k(const double* scores, const uint64_t* ids, uint64_t n,
                          int has_top_k, uint64_t top_k, double frac, uint64_t* out) {
  std::vector<BlockScore> v(n);
  for (uint64_t i = 0; i < n; ++i) v[i] = {ids[i], scores[i]};
  const auto sel = select_top_k(std::move(v), make_policy(has_top_k, top_k, frac));
  std::copy(sel.begin(), sel.end(), out);
  return sel.size();
}

uint64_t ref_fast_capacity(uint64_t budget, uint32_t d_k, uint32_t d_v, uint32_t bytes_fp,
                           uint32_t block_size) {
  try {
    return fast_capacity(make_cfg(budget, d_k, d_v, bytes_fp, block_size, 8, 4));
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
}

uint64_t ref_modeled_block_bytes(uint32_t block_size, uint32_t d_k, uint32_t d_v,
                                 uint32_t kb, uint32_t vb) {
  TierConfig c;
  c.block_size = block_size;
  c.d_k = d_k;
  c.d_v = d_v;
  c.key_bits = kb;
  c.value_bits = vb;
  return modeled_block_bytes(c);
}

int ref_generate_workload(int needle, uint64_t ctx, uint64_t T, uint32_t d_k, uint32_t d_v,
                          uint64_t seed, uint64_t needle_pos, double strength, float* pre_k,
                          float* pre_v, float* dec_k, float* dec_v, float* dec_q) {
  try {
    WorkloadSpec s;
    s.kind = needle ? WorkloadSpec::Kind::PlantedNeedle : WorkloadSpec::Kind::Gaussian;
    s.context_length = ctx;
    s.decode_steps = T;
    s.d_k = d_k;
    s.d_v = d_v;
    s.seed = seed;
    s.needle_block_position = needle_pos;
    s.needle_alignment_strength = strength;
    const auto w = generate_workload(s);
    for (uint64_t p = 0; p < ctx; ++p) {
      std::copy(w.prefill[p].key.begin(), w.prefill[p].key.end(), pre_k + p * d_k);
      std::copy(w.prefill[p].value.begin(), w.prefill[p].value.end(), pre_v + p * d_v);
    }
    for (uint64_t t = 0; t < T; ++t) {
      std::copy(w.decode[t].kv.key.begin(), w.decode[t].kv.key.end(), dec_k + t * d_k);
      std::copy(w.decode[t].kv.value.begin(), w.decode[t].kv.value.end(), dec_v + t * d_v);
      std::copy(w.decode[t].query.begin(), w.decode[t].query.end(), dec_q + t * d_k);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_dense_attention(const float* q, uint32_t d_k, const float* keys, const float* values,
                        uint64_t rows, uint32_t d_v, double* out) {
  std::vector<TokenKV> h(rows);
  for (uint64_t r = 0; r < rows; ++r) {
    h[r].position = r;
    h[r].key.assign(keys + r * d_k, keys + (r + 1) * d_k);
    h[r].value.assign(values + r * d_v, values + (r + 1) * d_v);
  }
  const auto o = reference::dense_attention(std::span<const float>(q, d_k), h);
  std::copy(o.begin(), o.end(), out);
  return 0;
}

// ---- simulate_serial / simulate_pipelined (sim.hpp:50-58) --------------------
// compute item i is labelled "c<i>"; transfer item j carries the label of
// compute item t_of[j].
int ref_simulate(int pipelined, uint64_t n_compute, const double* camount, uint64_t n_transfer,
                 const double* tamount, const uint64_t* t_of, double bandwidth,
                 double fixed_latency, double compute_rate, double* total, double* idle,
                 double* stall, double* total_compute, double* total_transfer) {
  try {
    StepWorkload w;
    for (uint64_t i = 0; i < n_compute; ++i)
      w.compute_items.push_back({"c" + std::to_string(i), camount[i]});
    for (uint64_t j = 0; j < n_transfer; ++j)
      w.transfer_items.push_back({"c" + std::to_string(t_of[j]), tamount[j]});
    LinkModel link{bandwidth, fixed_latency};
    const PipelineTimeline tl = pipelined ? simulate_pipelined(w, link, compute_rate)
                                          : simulate_serial(w, link, compute_rate);
    *total = tl.total_latency;
    *idle = tl.idle_fraction;
    *stall = tl.mean_transfer_stall;
    *total_compute = tl.total_compute;
    *total_transfer = tl.total_transfer;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ---- parse_config_file + apply_config_values (harness.hpp:90-96) ------------
// u64[9]: seed, context_length, decode_steps, d_k, d_v, needle_block_position,
//         hbm_budget_bytes, block_size, bytes_full_precision
// u32[7]: kind, key_bits, value_bits, has_top_k, baseline, format, literal_merge
// f64[7]: needle_strength, tier.fetch_fraction, policy.fetch_fraction,
//         hbm_bandwidth, pcie_bandwidth, transfer_latency, compute_rate
// u64 top_k; out_dir copied to out (cap bytes).  Returns 0, or 1 ConfigError,
// 2 IoError, 3 other (message in ref_last_error).
int ref_load_config(const char* path, uint64_t* u64s, uint32_t* u32s, double* f64s,
                    uint64_t* top_k, char* out_dir, uint64_t cap) {
#ifdef TTKV_REF_HAVE_HARNESS
  try {
    RunConfig cfg;
    WorkloadSpec spec;
    apply_config_values(parse_config_file(path), cfg, spec);
    const uint64_t u[9] = {spec.seed, spec.context_length, spec.decode_steps, spec.d_k,
                           spec.d_v, spec.needle_block_position, cfg.tier.hbm_budget_bytes,
                           cfg.tier.block_size, cfg.tier.bytes_full_precision};
    std::memcpy(u64s, u, sizeof(u));
    u32s[0] = spec.kind == WorkloadSpec::Kind::PlantedNeedle ? 1u : 0u;
    u32s[1] = cfg.tier.key_bits;
    u32s[2] = cfg.tier.value_bits;
    u32s[3] = cfg.policy.top_k.has_value() ? 1u : 0u;
    u32s[4] = (uint32_t)cfg.baseline;
    u32s[5] = (uint32_t)cfg.format;
    u32s[6] = cfg.literal_merge ? 1u : 0u;
    const double f[7] = {spec.needle_alignment_strength, cfg.tier.fetch_fraction,
                         cfg.policy.fetch_fraction, cfg.tier.hbm_bandwidth,
                         cfg.tier.pcie_bandwidth, cfg.tier.transfer_latency,
                         cfg.tier.compute_rate};
    std::memcpy(f64s, f, sizeof(f));
    *top_k = cfg.policy.top_k.value_or(0);
    std::snprintf(out_dir, cap, "%s", cfg.out_dir.c_str());
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const IoError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
#else
  (void)path; (void)u64s; (void)u32s; (void)f64s; (void)top_k; (void)out_dir; (void)cap;
  g_err = "harness not built";
  return 3;
#endif
}

// ---- Acceptance criterion 3 (acceptance.cpp:172-195) through run_benchmark --
double ref_traffic_reduction(uint64_t* total_h2g_bytes) {
#ifdef TTKV_REF_HAVE_HARNESS
  RunConfig cfg;
  cfg.tier.d_k = 128;
  cfg.tier.d_v = 128;
  cfg.tier.block_size = 128;
  cfg.tier.key_bits = 8;
  cfg.tier.value_bits = 4;
  cfg.tier.hbm_budget_bytes = 1024 * 256 * 2;
  cfg.policy.fetch_fraction = 0.45;
  WorkloadSpec spec;
  spec.context_length = 16384;
  spec.decode_steps = 8;
  spec.d_k = 128;
  spec.d_v = 128;
  spec.seed = 3;
  const auto record = run_benchmark(cfg, spec);
  if (total_h2g_bytes) *total_h2g_bytes = (uint64_t)record.summary.total_h2g_bytes;
  return record.summary.traffic_reduction_vs_baseline;
#else
  (void)total_h2g_bytes;
  return -1.0;
#endif
}

// ---- CPU baseline: n_engines reference Engines on n_threads host threads ------
// Each engine is prefilled with ctx Gaussian tokens (detail::GaussianSource,
// workload.hpp:53-66; seed base+engine/heads so the G heads of a stream share
// KV), then `steps` decode steps are timed.  ms_per_step[i] = wall time of
// decode step i across all engines (threads join per step).
int ref_bench_decode(uint32_t n_engines, uint32_t heads_per_stream, uint64_t ctx,
                     uint32_t steps, uint32_t n_threads, uint64_t budget, uint32_t d,
                     uint32_t block_size, uint32_t kb, uint32_t vb, double frac,
                     uint64_t seed, double* ms_per_step, double* prefill_s) {
  try {
    const TierConfig cfg = make_cfg(budget, d, d, 2, block_size, kb, vb);
    const SelectionPolicy pol = make_policy(0, 0, frac);
    std::vector<std::unique_ptr<Engine>> engines(n_engines);
    n_threads = std::max<uint32_t>(1, std::min(n_threads, n_engines));
    auto t0 = std::chrono::steady_clock::now();
    auto run_par = [&](auto&& fn) {
      std::atomic<uint32_t> next{0};
      std::vector<std::thread> th;
      for (uint32_t t = 0; t < n_threads; ++t)
        th.emplace_back([&] {
          for (uint32_t i; (i = next.fetch_add(1)) < n_engines;) fn(i);
        });
      for (auto& x : th) x.join();
    };
    run_par([&](uint32_t i) {
      engines[i] = std::make_unique<Engine>(cfg, pol);
      detail::GaussianSource g(seed + i / std::max<uint32_t>(1, heads_per_stream));
      const uint64_t chunk = 2048;
      std::vector<TokenKV> toks;
      for (uint64_t p0 = 0; p0 < ctx; p0 += chunk) {
        const uint64_t m = std::min(chunk, ctx - p0);
        toks.assign(m, TokenKV{});
        for (uint64_t t = 0; t < m; ++t) {
          toks[t].position = p0 + t;
          toks[t].key.resize(d);
          toks[t].value.resize(d);
          for (auto& x : toks[t].key) x = g.nextf();
          for (auto& x : toks[t].value) x = g.nextf();
        }
        engines[i]->prefill(toks);
      }
    });
    if (prefill_s)
      *prefill_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (uint32_t s = 0; s < steps; ++s) {
      // inputs drawn outside the timed region
      std::vector<std::vector<float>> qs(n_engines), ks(n_engines), vs(n_engines);
      for (uint32_t i = 0; i < n_engines; ++i) {
        const uint32_t stream = i / std::max<uint32_t>(1, heads_per_stream);
        detail::GaussianSource gkv(seed * 7919 + s * 104729 + stream);
        detail::GaussianSource gq(seed * 6997 + s * 130363 + i);
        qs[i].resize(d);
        ks[i].resize(d);
        vs[i].resize(d);
        for (auto& x : qs[i]) x = gq.nextf();
        for (auto& x : ks[i]) x = gkv.nextf();
        for (auto& x : vs[i]) x = gkv.nextf();
      }
      const auto a = std::chrono::steady_clock::now();
      run_par([&](uint32_t i) {
        TokenKV kv;
        kv.position = engines[i]->store().appended_count();
        kv.key = ks[i];
        kv.value = vs[i];
        engines[i]->decode_step(qs[i], std::move(kv));
      });
      ms_per_step[s] =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
