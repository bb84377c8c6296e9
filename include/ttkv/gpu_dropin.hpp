// gpu_dropin.hpp -- C++ drop-in for the reference's ttkv:: API, backed by the
// B200 C ABI (include/ttkv_gpu.h).  A program written against the reference
// headers (proj/core/include/ttkv/*.hpp) compiles unchanged against
// include/ttkv/ (whose per-module headers forward here) and links
// libttkv.so + libttkv_gpu.so instead of ttkv::core.
//
// What runs where:
//   GPU (sm_100a):  TierStore (fast ring in HBM, slow tier in pinned DRAM),
//                   Engine::prefill / decode_step, quantize_block,
//                   dequantize_block, score_block, select_top_k.
//   Host:           config validation, bookkeeping, byte (de)serialization
//                   and file I/O, the header-only AttentionAccumulator
//                   (attention.hpp is a host template in the reference too),
//                   generate_workload (input generator) and the dense oracle
//                   reference::dense_attention (test utility).
// Cold-path views (TierStore::fast_tokens / slow_blocks) are materialized from
// device/pinned memory on demand and invalidated by every mutation.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <filesystem>
#include <iosfwd>
#include <limits>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ttkv_gpu.h"

namespace ttkv {

// ---- errors (reference errors.hpp) ------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class SequencingError : public Error {
 public:
  using Error::Error;
};
class ShapeError : public Error {
 public:
  using Error::Error;
};
class IntegrityError : public Error {
 public:
  using Error::Error;
};
class IoError : public Error {
 public:
  using Error::Error;
};

// Rethrows a TTKV_* status from the C ABI as the matching exception class.
[[noreturn]] void raise_status(int status, const std::string& message);

// ---- value types (reference kv_types.hpp) ------------------------------------------
using Position = std::uint64_t;
using BlockId = std::uint64_t;

struct TokenKV {
  Position position = 0;
  std::vector<float> key;
  std::vector<float> value;
};

struct KvBlock {
  BlockId block_id = 0;
  Position first_position = 0;
  Position last_position = 0;
  std::size_t token_count = 0;
  std::size_t d_k = 0;
  std::size_t d_v = 0;
  std::vector<float> keys;
  std::vector<float> values;
};

struct Location {
  enum class Where { Fast, Slow, Absent };
  Where where = Where::Absent;
  BlockId block_id = 0;
  static Location fast() { return {Where::Fast, 0}; }
  static Location slow(BlockId id) { return {Where::Slow, id}; }
  static Location absent() { return {Where::Absent, 0}; }
  bool operator==(const Location&) const = default;
};

struct CacheEvent {
  enum class Type { EvictBlock };
  Type type = Type::EvictBlock;
  Position first_position = 0;
  Position last_position = 0;
};

// ---- configuration (reference config.hpp) -------------------------------------------
// bytes_full_precision also selects the GPU fast-tier storage: 2 = fp16 ring,
// 4 = fp32 ring (bit-exact for arbitrary float inputs).
struct TierConfig {
  std::size_t hbm_budget_bytes = 0;
  std::size_t d_k = 64;
  std::size_t d_v = 64;
  std::size_t bytes_full_precision = 2;
  std::size_t block_size = 128;
  unsigned key_bits = 8;
  unsigned value_bits = 4;
  double fetch_fraction = 0.45;
  std::optional<std::size_t> top_k_blocks;
  double hbm_bandwidth = 2.0e12;
  double pcie_bandwidth = 3.2e10;
  double transfer_latency = 1.0e-5;
  double compute_rate = 4.0e11;

  std::size_t d_kv() const { return d_k + d_v; }
  std::size_t block_bytes_full_precision() const {
    return block_size * d_kv() * bytes_full_precision;
  }
  bool nonstandard_block_size() const {
    return !(block_size == 32 || block_size == 64 || block_size == 128 || block_size == 256);
  }
  void validate() const;
  ttkv_tier_config to_c() const;
};

// ---- relevance (reference relevance.hpp) ----------------------------------------------
struct BlockScore {
  BlockId block_id = 0;
  double score = 0.0;
};

struct SelectionPolicy {
  std::optional<std::size_t> top_k;
  double fetch_fraction = 0.45;
  std::size_t resolve(std::size_t block_count) const;
  ttkv_selection_policy to_c() const;
};

double score_block(std::span<const float> query, std::span<const float> centroid);
std::vector<BlockId> select_top_k(std::vector<BlockScore> scores, const SelectionPolicy& policy);

// ---- quantizer (reference quantizer.hpp) ------------------------------------------------
struct QuantParams {
  float scale = 1.0f;
  float zero_point = 0.0f;
};

struct QuantizedBlock {
  BlockId block_id = 0;
  Position first_position = 0;
  Position last_position = 0;
  std::uint32_t token_count = 0;
  std::uint32_t d_k = 0;
  std::uint32_t d_v = 0;
  std::uint32_t key_bits = 8;
  std::uint32_t value_bits = 4;
  std::vector<std::uint8_t> packed_keys;
  std::vector<std::uint8_t> packed_values;
  std::vector<QuantParams> key_params;
  std::vector<QuantParams> value_params;
  std::vector<float> key_centroid;
  std::size_t modeled_payload_bytes() const;
};

QuantizedBlock quantize_block(const KvBlock& block, const TierConfig& config);
KvBlock dequantize_block(const QuantizedBlock& qblock);
std::size_t modeled_block_bytes(const TierConfig& config);
double compressed_bytes_per_token(const TierConfig& config);
std::vector<std::uint8_t> serialize_block(const QuantizedBlock& qblock);
QuantizedBlock deserialize_block(std::span<const std::uint8_t> bytes);
void dump_slow_tier(const std::vector<QuantizedBlock>& blocks, const std::filesystem::path& path);
std::vector<QuantizedBlock> load_slow_tier(const std::filesystem::path& path);

// ---- streaming accumulator (reference attention.hpp; host template) ----------------
// Online softmax over partitions: running max m, denominator l, weighted sum.
template <typename T>
class AttentionAccumulator {
 public:
  AttentionAccumulator(std::size_t d_v, T softmax_scale)
      : width_(d_v), scale_(softmax_scale), m_(-std::numeric_limits<T>::infinity()), l_(0),
        acc_(d_v, T(0)) {}

  void absorb(std::span<const float> query, const float* keys, const float* values,
              std::size_t rows, std::size_t d_k) {
    for (std::size_t r = 0; r < rows; ++r) {
      const float* kr = keys + r * d_k;
      T dot = 0;
      for (std::size_t i = 0; i < d_k; ++i) dot += T(query[i]) * T(kr[i]);
      const T s = dot * scale_;
      if (s > m_) {  // new running max: rescale what was accumulated
        const T shrink = std::exp(m_ - s);
        l_ *= shrink;
        for (T& a : acc_) a *= shrink;
        m_ = s;
      }
      const T w = std::exp(s - m_);
      l_ += w;
      const float* vr = values + r * width_;
      for (std::size_t i = 0; i < width_; ++i) acc_[i] += w * T(vr[i]);
      ++count_;
    }
  }

  std::vector<T> finalize() const {
    if (count_ == 0) throw Error("finalize on empty attention accumulator");
    std::vector<T> out(acc_);
    for (T& x : out) x /= l_;
    return out;
  }

  std::size_t absorbed() const { return count_; }
  T running_max() const { return m_; }
  T denominator() const { return l_; }

 private:
  std::size_t width_;
  T scale_;
  T m_;
  T l_;
  std::vector<T> acc_;
  std::size_t count_ = 0;
};

template <typename T>
void attend_partition(std::span<const float> query, std::span<const float> keys,
                      std::span<const float> values, std::size_t rows, std::size_t d_k,
                      std::size_t d_v, AttentionAccumulator<T>& acc) {
  if (query.size() != d_k || keys.size() != rows * d_k || values.size() != rows * d_v)
    throw ShapeError("attend_partition: inconsistent shapes");
  acc.absorb(query, keys.data(), values.data(), rows, d_k);
}

// ---- tier store (reference tier_store.hpp) ---------------------------------------------
class BlockIndex {
 public:
  void append_block(BlockId id, Position first, Position last);
  std::optional<BlockId> find(Position p) const;
  std::pair<Position, Position> range(BlockId id) const;
  std::size_t size() const { return spans_.size(); }

 private:
  struct Span {
    BlockId id;
    Position first, last;
  };
  std::vector<Span> spans_;
};

std::size_t fast_capacity(const TierConfig& config);

// One KV stream whose fast tier is an HBM ring and whose slow tier lives in
// pinned host DRAM, all owned by a ttkv_gpu handle.  Single writer; movable.
class TierStore {
 public:
  explicit TierStore(TierConfig config);
  // used by Engine: the device store also holds the selection policy and
  // EngineOptions::literal_additive_merge
  TierStore(TierConfig config, const SelectionPolicy& policy, bool literal_merge = false);
  ~TierStore();
  TierStore(TierStore&& o) noexcept;
  TierStore& operator=(TierStore&& o) noexcept;
  TierStore(const TierStore&) = delete;
  TierStore& operator=(const TierStore&) = delete;

  std::vector<CacheEvent> append_token(TokenKV kv);
  bool eviction_pending() const;
  BlockId evict_and_compress();
  Location locate(Position p) const;

  const std::deque<TokenKV>& fast_tokens() const;
  const std::vector<QuantizedBlock>& slow_blocks() const;
  const BlockIndex& block_index() const { return index_; }
  const TierConfig& config() const { return config_; }

  std::size_t fast_token_count() const;
  std::size_t slow_token_count() const;
  std::size_t appended_count() const;
  std::size_t l_fast_capacity() const { return l_fast_; }

  // the device handle, with every buffered append applied
  ttkv_gpu* handle() const {
    flush();
    return h_;
  }
  void note_decode_step(std::size_t evicted_blocks);  // Engine bookkeeping

 private:
  ttkv_state state() const;  // applies buffered appends first
  // device bookkeeping + buffered appends, without touching the device
  std::size_t appended_now() const;
  std::size_t fast_now() const;
  void flush() const;
  void invalidate() { fast_valid_ = false; }

  TierConfig config_;
  std::size_t l_fast_ = 0;
  ttkv_gpu* h_ = nullptr;
  BlockIndex index_;
  mutable std::deque<TokenKV> fast_view_;
  mutable bool fast_valid_ = false;
  mutable std::vector<QuantizedBlock> slow_view_;  // append-only cache
  // append_token buffers tokens on the host and hands them to the device in
  // one ttkv_gpu_append when something reads the ring (a GPU round trip per
  // token otherwise dominates token-at-a-time callers)
  mutable std::vector<float> pend_k_, pend_v_;
  mutable std::size_t pend_n_ = 0;
};

// ---- two-lane timing model (reference sim.hpp; implemented in ttkv_sim.cpp) --------
// One decode step as the simulator sees it: compute items (the fast chunk, then
// one per fetched block) and transfer items (one per fetched block), both in
// prefetch-schedule order, matched by label.
struct WorkItem {
  std::string label;
  double amount = 0.0;  // attention elements (compute) or bytes (transfer)
};
struct StepWorkload {
  std::vector<WorkItem> compute_items;
  std::vector<WorkItem> transfer_items;
};
struct LinkModel {
  double bandwidth = 3.2e10;   // bytes/s
  double fixed_latency = 0.0;  // s per transfer
};
struct TimelineEvent {
  enum class Lane { Transfer, Compute };
  Lane lane = Lane::Compute;
  std::string label;
  double start = 0.0;
  double finish = 0.0;
};
struct PipelineTimeline {
  std::vector<TimelineEvent> events;
  double total_latency = 0.0;
  double total_compute = 0.0;
  double total_transfer = 0.0;
  double idle_fraction = 0.0;        // compute-lane idle time / total latency
  double mean_transfer_stall = 0.0;  // mean delay of fetched blocks' compute starts
};
// All transfers first, then all compute.
PipelineTimeline simulate_serial(const StepWorkload& workload, const LinkModel& link,
                                 double compute_rate);
// Transfers back to back; each block's compute waits for its own transfer.
PipelineTimeline simulate_pipelined(const StepWorkload& workload, const LinkModel& link,
                                    double compute_rate);
struct TrafficLedger {
  std::vector<double> step_bytes;
  std::vector<double> baseline_step_bytes;
  double total_bytes() const;
  double total_baseline_bytes() const;
};
struct RunSummary {
  std::size_t steps = 0;
  double p95_latency = 0.0;
  double mean_latency = 0.0;
  double tokens_per_second = 0.0;
  double total_h2g_bytes = 0.0;
  double traffic_reduction_vs_baseline = 0.0;
};
RunSummary aggregate_run(const std::vector<PipelineTimeline>& timelines,
                         const TrafficLedger& ledger);
void dump_timeline(std::ostream& os, const PipelineTimeline& timeline);

// ---- workload generator (reference workload.hpp) --------------------------------------
inline constexpr std::size_t kNeedleSpanTokens = 128;

struct WorkloadSpec {
  enum class Kind { Gaussian, PlantedNeedle };
  Kind kind = Kind::Gaussian;
  std::size_t context_length = 4096;
  std::size_t decode_steps = 32;
  std::size_t d_k = 64;
  std::size_t d_v = 64;
  std::uint64_t seed = 0;
  std::size_t needle_block_position = 2;
  double needle_alignment_strength = 3.0;
  void validate() const;
};

struct DecodeInput {
  TokenKV kv;
  std::vector<float> query;
};

struct WorkloadStream {
  std::vector<TokenKV> prefill;
  std::vector<DecodeInput> decode;
  std::vector<float> needle_direction;
};

WorkloadStream generate_workload(const WorkloadSpec& spec);

namespace detail {
// Box-Muller over std::mt19937_64 (portable across standard libraries).
class GaussianSource {
 public:
  explicit GaussianSource(std::uint64_t seed) : gen_(seed) {}
  double next();
  float nextf() { return static_cast<float>(next()); }

 private:
  std::mt19937_64 gen_;
  double cached_ = 0.0;
  bool have_cached_ = false;
};
}  // namespace detail

// ---- engine (reference engine.hpp) ------------------------------------------------------
struct EngineOptions {
  bool literal_additive_merge = false;
};

struct DecodeStepReport {
  std::vector<double> output;
  std::size_t blocks_scored = 0;
  std::size_t blocks_fetched = 0;
  std::vector<BlockId> fetched_blocks;
  double bytes_transferred = 0.0;
  bool eviction_occurred = false;
  StepWorkload workload;
};

class Engine {
 public:
  Engine(TierConfig config, SelectionPolicy policy, EngineOptions options = {});

  void prefill(std::span<const TokenKV> tokens);
  DecodeStepReport decode_step(std::span<const float> query, TokenKV kv);
  std::vector<DecodeStepReport> decode_sequence(std::span<const DecodeInput> inputs);

  TierStore& store() { return store_; }
  const TierStore& store() const { return store_; }
  const TierConfig& config() const { return store_.config(); }
  const SelectionPolicy& policy() const { return policy_; }

 private:
  SelectionPolicy policy_;
  EngineOptions options_;
  TierStore store_;
};

// ---- dense oracle (reference reference.hpp; host test utility) ------------------------
namespace reference {
std::vector<double> dense_attention(std::span<const float> query,
                                    std::span<const TokenKV> history);
double relative_error(std::span<const double> a, std::span<const double> b);
}  // namespace reference

}  // namespace ttkv
