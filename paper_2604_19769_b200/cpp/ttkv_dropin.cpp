// ttkv_dropin.cpp -- implementation of include/ttkv/gpu_dropin.hpp over the C
// ABI.  All numeric work (quantize, dequantize, score, select, streaming
// attention) is done by libttkv_gpu.so on the device; this file holds the
// host-side API glue: argument checks with the reference's exception classes
// and messages, bookkeeping, byte formats and file I/O.
#include "ttkv/gpu_dropin.hpp"

#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <numbers>

namespace ttkv {

namespace {

int device_ordinal() {
  const char* env = std::getenv("TTKV_DEVICE");
  return env ? std::atoi(env) : 0;
}

std::string last_error(const ttkv_gpu* h) {
  const char* m = h ? ttkv_gpu_last_error(h) : ttkv_last_error();
  return m ? m : "";
}

void check(int status, const ttkv_gpu* h = nullptr) {
  if (status != TTKV_OK) raise_status(status, last_error(h));
}

std::size_t stored_bytes(std::size_t count, unsigned bits) {
  return bits == 16 ? count * sizeof(float) : (count * bits + 7) / 8;
}

std::size_t accounted_bytes(std::size_t count, unsigned bits) {
  return bits == 16 ? count * 2 : (count * bits + 7) / 8;
}

bool bits_ok(unsigned b) { return (b >= 2 && b <= 8) || b == 16; }

// little-endian byte sink / source for the TTKV block and tier formats
class ByteSink {
 public:
  void u(std::uint64_t v, int n) {
    for (int i = 0; i < n; ++i) buf.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  }
  void f(float x) {
    std::uint32_t v;
    std::memcpy(&v, &x, 4);
    u(v, 4);
  }
  void raw(const void* p, std::size_t n) {
    const auto* b = static_cast<const std::uint8_t*>(p);
    buf.insert(buf.end(), b, b + n);
  }
  std::vector<std::uint8_t> buf;
};

class ByteSource {
 public:
  explicit ByteSource(std::span<const std::uint8_t> b) : b_(b) {}
  std::uint64_t u(int n) {
    need(n);
    std::uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= std::uint64_t(b_[at_ + i]) << (8 * i);
    at_ += n;
    return v;
  }
  float f() {
    const std::uint32_t v = static_cast<std::uint32_t>(u(4));
    float x;
    std::memcpy(&x, &v, 4);
    return x;
  }
  std::vector<std::uint8_t> take(std::size_t n) {
    need(n);
    std::vector<std::uint8_t> out(b_.begin() + at_, b_.begin() + at_ + n);
    at_ += n;
    return out;
  }
  bool exhausted() const { return at_ == b_.size(); }

 private:
  void need(std::size_t n) {
    if (at_ + n > b_.size()) throw IntegrityError("deserialize: truncated payload");
  }
  std::span<const std::uint8_t> b_;
  std::size_t at_ = 0;
};

constexpr char kBlockTag[4] = {'T', 'T', 'K', 'V'};
constexpr char kTierTag[8] = {'T', 'T', 'K', 'V', 'T', 'I', 'E', 'R'};
constexpr std::uint16_t kVersion = 1;

}  // namespace

[[noreturn]] void raise_status(int status, const std::string& m) {
  switch (status) {
    case TTKV_ECONFIG: throw ConfigError(m);
    case TTKV_ESEQUENCE: throw SequencingError(m);
    case TTKV_ESHAPE: throw ShapeError(m);
    case TTKV_EINTEGRITY: throw IntegrityError(m);
    case TTKV_EIO: throw IoError(m);
    case TTKV_ECUDA: throw Error("CUDA: " + m);
    default: throw Error(m);
  }
}

// ---- config / policy ---------------------------------------------------------------
ttkv_tier_config TierConfig::to_c() const {
  ttkv_tier_config c{};
  c.hbm_budget_bytes = hbm_budget_bytes;
  c.d_k = d_k;
  c.d_v = d_v;
  c.bytes_full_precision = bytes_full_precision;
  c.block_size = block_size;
  c.key_bits = key_bits;
  c.value_bits = value_bits;
  c.fetch_fraction = fetch_fraction;
  c.has_top_k_blocks = top_k_blocks.has_value();
  c.top_k_blocks = top_k_blocks.value_or(0);
  c.hbm_bandwidth = hbm_bandwidth;
  c.pcie_bandwidth = pcie_bandwidth;
  c.transfer_latency = transfer_latency;
  c.compute_rate = compute_rate;
  return c;
}

void TierConfig::validate() const {
  const ttkv_tier_config c = to_c();
  check(ttkv_validate_config(&c));
}

ttkv_selection_policy SelectionPolicy::to_c() const {
  ttkv_selection_policy p{};
  p.has_top_k = top_k.has_value();
  p.top_k = top_k.value_or(0);
  p.fetch_fraction = fetch_fraction;
  return p;
}

std::size_t SelectionPolicy::resolve(std::size_t block_count) const {
  const ttkv_selection_policy p = to_c();
  const std::uint64_t k = ttkv_resolve(&p, block_count);
  if (k == UINT64_MAX) throw ConfigError(last_error(nullptr));
  return static_cast<std::size_t>(k);
}

// ---- relevance on the GPU ------------------------------------------------------------
double score_block(std::span<const float> query, std::span<const float> centroid) {
  if (query.size() != centroid.size()) throw ShapeError("score_block: dimension mismatch");
  if (query.empty()) return 0.0;
  double s = 0.0;
  check(ttkv_gpu_score_blocks(device_ordinal(), query.data(), centroid.data(), 1,
                              static_cast<std::uint32_t>(query.size()), &s));
  return s;
}

std::vector<BlockId> select_top_k(std::vector<BlockScore> scores, const SelectionPolicy& policy) {
  const std::size_t k = policy.resolve(scores.size());
  std::vector<BlockId> out(k);
  if (k == 0) return out;
  std::vector<double> s(scores.size());
  std::vector<std::uint64_t> ids(scores.size());
  for (std::size_t i = 0; i < scores.size(); ++i) {
    s[i] = scores[i].score;
    ids[i] = scores[i].block_id;
  }
  check(ttkv_gpu_select_top_k(device_ordinal(), s.data(), ids.data(), s.size(), k, out.data()));
  return out;
}

// ---- quantizer ---------------------------------------------------------------------------
std::size_t QuantizedBlock::modeled_payload_bytes() const {
  std::size_t b = accounted_bytes(std::size_t(token_count) * d_k, key_bits) +
                  accounted_bytes(std::size_t(token_count) * d_v, value_bits);
  if (key_bits != 16) b += 4 * std::size_t(d_k);
  if (value_bits != 16) b += 4 * std::size_t(d_v);
  return b;
}

QuantizedBlock quantize_block(const KvBlock& block, const TierConfig& config) {
  if (block.keys.size() != block.token_count * block.d_k ||
      block.values.size() != block.token_count * block.d_v)
    throw ShapeError("quantize_block: tensor sizes inconsistent");
  QuantizedBlock q;
  q.block_id = block.block_id;
  q.first_position = block.first_position;
  q.last_position = block.last_position;
  q.token_count = static_cast<std::uint32_t>(block.token_count);
  q.d_k = static_cast<std::uint32_t>(block.d_k);
  q.d_v = static_cast<std::uint32_t>(block.d_v);
  q.key_bits = config.key_bits;
  q.value_bits = config.value_bits;
  q.packed_keys.resize(stored_bytes(block.token_count * block.d_k, config.key_bits));
  q.packed_values.resize(stored_bytes(block.token_count * block.d_v, config.value_bits));
  std::vector<float> kp(2 * block.d_k), vp(2 * block.d_v);
  q.key_centroid.resize(block.d_k);
  check(ttkv_gpu_quantize_block(device_ordinal(), block.keys.data(), block.values.data(),
                                block.token_count, q.d_k, q.d_v, config.key_bits,
                                config.value_bits, q.packed_keys.data(), q.packed_values.data(),
                                kp.data(), vp.data(), q.key_centroid.data()));
  if (config.key_bits != 16) {
    q.key_params.resize(block.d_k);
    for (std::size_t c = 0; c < block.d_k; ++c) q.key_params[c] = {kp[2 * c], kp[2 * c + 1]};
  }
  if (config.value_bits != 16) {
    q.value_params.resize(block.d_v);
    for (std::size_t c = 0; c < block.d_v; ++c) q.value_params[c] = {vp[2 * c], vp[2 * c + 1]};
  }
  return q;
}

KvBlock dequantize_block(const QuantizedBlock& q) {
  auto check_tensor = [&](const std::vector<std::uint8_t>& packed,
                          const std::vector<QuantParams>& params, std::size_t dim, unsigned bits) {
    const std::size_t n = std::size_t(q.token_count) * dim;
    if (bits == 16) {
      if (packed.size() != n * sizeof(float))
        throw IntegrityError("dequantize: passthrough payload size mismatch");
      return;
    }
    if (packed.size() != stored_bytes(n, bits))
      throw IntegrityError("dequantize: packed payload size mismatch");
    if (params.size() != dim) throw IntegrityError("dequantize: parameter count mismatch");
  };
  check_tensor(q.packed_keys, q.key_params, q.d_k, q.key_bits);
  check_tensor(q.packed_values, q.value_params, q.d_v, q.value_bits);
  KvBlock b;
  b.block_id = q.block_id;
  b.first_position = q.first_position;
  b.last_position = q.last_position;
  b.token_count = q.token_count;
  b.d_k = q.d_k;
  b.d_v = q.d_v;
  b.keys.resize(std::size_t(q.token_count) * q.d_k);
  b.values.resize(std::size_t(q.token_count) * q.d_v);
  auto flat = [](const std::vector<QuantParams>& p) {
    std::vector<float> f(2 * p.size() + 2);
    for (std::size_t i = 0; i < p.size(); ++i) {
      f[2 * i] = p[i].scale;
      f[2 * i + 1] = p[i].zero_point;
    }
    return f;
  };
  const auto kp = flat(q.key_params), vp = flat(q.value_params);
  check(ttkv_gpu_dequantize_block(device_ordinal(), q.packed_keys.data(), q.packed_values.data(),
                                  kp.data(), vp.data(), q.token_count, q.d_k, q.d_v, q.key_bits,
                                  q.value_bits, b.keys.data(), b.values.data()));
  return b;
}

std::size_t modeled_block_bytes(const TierConfig& config) {
  const ttkv_tier_config c = config.to_c();
  return static_cast<std::size_t>(ttkv_modeled_block_bytes(&c));
}

double compressed_bytes_per_token(const TierConfig& config) {
  return double(modeled_block_bytes(config)) / double(config.block_size);
}

// ---- byte formats (reference quantizer.cpp:187-365 layout, v1) ---------------------
std::vector<std::uint8_t> serialize_block(const QuantizedBlock& q) {
  ByteSink w;
  w.raw(kBlockTag, 4);
  w.u(kVersion, 2);
  w.u(q.block_id, 8);
  w.u(q.first_position, 8);
  w.u(q.last_position, 8);
  w.u(q.token_count, 4);
  w.u(q.d_k, 4);
  w.u(q.d_v, 4);
  w.u(q.key_bits, 2);
  w.u(q.value_bits, 2);
  for (const auto& params : {&q.key_params, &q.value_params})
    for (const QuantParams& p : *params) {
      w.f(p.scale);
      w.f(p.zero_point);
    }
  for (float c : q.key_centroid) w.f(c);
  for (const auto* payload : {&q.packed_keys, &q.packed_values}) {
    w.u(payload->size(), 8);
    w.raw(payload->data(), payload->size());
  }
  return std::move(w.buf);
}

QuantizedBlock deserialize_block(std::span<const std::uint8_t> bytes) {
  ByteSource r(bytes);
  const auto tag = r.take(4);
  if (std::memcmp(tag.data(), kBlockTag, 4) != 0) throw IntegrityError("deserialize: bad magic");
  if (r.u(2) != kVersion) throw IntegrityError("deserialize: unsupported version");
  QuantizedBlock q;
  q.block_id = r.u(8);
  q.first_position = r.u(8);
  q.last_position = r.u(8);
  q.token_count = static_cast<std::uint32_t>(r.u(4));
  q.d_k = static_cast<std::uint32_t>(r.u(4));
  q.d_v = static_cast<std::uint32_t>(r.u(4));
  q.key_bits = static_cast<std::uint32_t>(r.u(2));
  q.value_bits = static_cast<std::uint32_t>(r.u(2));
  if (!bits_ok(q.key_bits) || !bits_ok(q.value_bits))
    throw IntegrityError("deserialize: bad bit widths");
  q.key_params.resize(q.key_bits == 16 ? 0 : q.d_k);
  q.value_params.resize(q.value_bits == 16 ? 0 : q.d_v);
  for (auto* params : {&q.key_params, &q.value_params})
    for (QuantParams& p : *params) {
      p.scale = r.f();
      p.zero_point = r.f();
    }
  q.key_centroid.resize(q.d_k);
  for (float& c : q.key_centroid) c = r.f();
  const std::size_t klen = r.u(8);
  if (klen != stored_bytes(std::size_t(q.token_count) * q.d_k, q.key_bits))
    throw IntegrityError("deserialize: key payload length mismatch");
  q.packed_keys = r.take(klen);
  const std::size_t vlen = r.u(8);
  if (vlen != stored_bytes(std::size_t(q.token_count) * q.d_v, q.value_bits))
    throw IntegrityError("deserialize: value payload length mismatch");
  q.packed_values = r.take(vlen);
  return q;
}

void dump_slow_tier(const std::vector<QuantizedBlock>& blocks, const std::filesystem::path& path) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError("cannot open " + path.string() + " for writing");
  ByteSink w;
  w.raw(kTierTag, 8);
  w.u(kVersion, 2);
  w.u(blocks.size(), 8);
  for (const QuantizedBlock& b : blocks) {
    const auto blob = serialize_block(b);
    w.u(blob.size(), 8);
    w.raw(blob.data(), blob.size());
  }
  os.write(reinterpret_cast<const char*>(w.buf.data()), std::streamsize(w.buf.size()));
  if (!os) throw IoError("write failed: " + path.string());
}

std::vector<QuantizedBlock> load_slow_tier(const std::filesystem::path& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open " + path.string());
  const std::vector<std::uint8_t> all((std::istreambuf_iterator<char>(is)),
                                      std::istreambuf_iterator<char>());
  ByteSource r(all);
  const auto tag = r.take(8);
  if (std::memcmp(tag.data(), kTierTag, 8) != 0)
    throw IntegrityError("slow-tier file: bad magic");
  if (r.u(2) != kVersion) throw IntegrityError("slow-tier file: unsupported version");
  const std::uint64_t n = r.u(8);
  std::vector<QuantizedBlock> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    const std::uint64_t len = r.u(8);
    const auto blob = r.take(len);
    out.push_back(deserialize_block(blob));
  }
  if (!r.exhausted()) throw IntegrityError("slow-tier file: trailing bytes");
  return out;
}

// ---- block index ---------------------------------------------------------------------------
void BlockIndex::append_block(BlockId id, Position first, Position last) {
  if (!spans_.empty() && (first != spans_.back().last + 1 || id <= spans_.back().id))
    throw Error("BlockIndex: blocks must be appended in order");
  spans_.push_back({id, first, last});
}

std::optional<BlockId> BlockIndex::find(Position p) const {
  auto it = std::upper_bound(spans_.begin(), spans_.end(), p,
                             [](Position v, const Span& s) { return v < s.first; });
  if (it == spans_.begin()) return std::nullopt;
  --it;
  if (p > it->last) return std::nullopt;
  return it->id;
}

std::pair<Position, Position> BlockIndex::range(BlockId id) const {
  auto it = std::lower_bound(spans_.begin(), spans_.end(), id,
                             [](const Span& s, BlockId v) { return s.id < v; });
  if (it == spans_.end() || it->id != id)
    throw Error("BlockIndex: unknown block " + std::to_string(id));
  return {it->first, it->last};
}

std::size_t fast_capacity(const TierConfig& config) {
  config.validate();
  const ttkv_tier_config c = config.to_c();
  const std::uint64_t n = ttkv_fast_capacity(&c);
  if (n == 0) throw ConfigError(last_error(nullptr));
  return static_cast<std::size_t>(n);
}

// ---- tier store ------------------------------------------------------------------------------
namespace {
ttkv_gpu* open_store(const TierConfig& cfg, const SelectionPolicy& pol, bool literal) {
  const ttkv_tier_config c = cfg.to_c();
  const ttkv_selection_policy p = pol.to_c();
  ttkv_gpu_options o{};
  o.device = device_ordinal();
  o.n_streams = 1;
  o.heads_per_stream = 1;
  // TTKV_SLOW_TIER=hbm keeps the slow tier resident in HBM (tensor-core
  // consumer); the default is the reference's pinned host DRAM tier
  const char* tier = std::getenv("TTKV_SLOW_TIER");
  o.slow_tier = (tier && std::strcmp(tier, "hbm") == 0) ? TTKV_SLOW_DEVICE : TTKV_SLOW_PINNED_HOST;
  o.literal_additive_merge = literal ? 1u : 0u;
  // The reference keeps float32 tokens whatever bytes_full_precision accounts
  // for (kv_types.hpp:14-15): default to an fp32 ring (fp64 accumulation).
  // TTKV_RING=fp16 selects the fp16 ring of the batched performance path.
  const char* ring = std::getenv("TTKV_RING");
  o.ring_bytes = (ring && std::strcmp(ring, "fp16") == 0) ? 2u : 4u;
  ttkv_gpu* h = nullptr;
  check(ttkv_gpu_create(&c, &p, &o, &h));
  return h;
}
}  // namespace

TierStore::TierStore(TierConfig config) : TierStore(std::move(config), SelectionPolicy{}) {}

TierStore::TierStore(TierConfig config, const SelectionPolicy& policy, bool literal_merge)
    : config_(std::move(config)), l_fast_(fast_capacity(config_)) {
  h_ = open_store(config_, policy, literal_merge);
}

TierStore::~TierStore() {
  if (h_) ttkv_gpu_destroy(h_);
}

TierStore::TierStore(TierStore&& o) noexcept
    : config_(std::move(o.config_)), l_fast_(o.l_fast_), h_(o.h_), index_(std::move(o.index_)),
      fast_view_(std::move(o.fast_view_)), fast_valid_(o.fast_valid_),
      slow_view_(std::move(o.slow_view_)), pend_k_(std::move(o.pend_k_)),
      pend_v_(std::move(o.pend_v_)), pend_n_(o.pend_n_) {
  o.h_ = nullptr;
  o.pend_n_ = 0;
}

TierStore& TierStore::operator=(TierStore&& o) noexcept {
  if (this != &o) {
    if (h_) ttkv_gpu_destroy(h_);
    config_ = std::move(o.config_);
    l_fast_ = o.l_fast_;
    h_ = o.h_;
    index_ = std::move(o.index_);
    fast_view_ = std::move(o.fast_view_);
    fast_valid_ = o.fast_valid_;
    slow_view_ = std::move(o.slow_view_);
    pend_k_ = std::move(o.pend_k_);
    pend_v_ = std::move(o.pend_v_);
    pend_n_ = o.pend_n_;
    o.h_ = nullptr;
    o.pend_n_ = 0;
  }
  return *this;
}

void TierStore::flush() const {
  if (!pend_n_) return;
  const std::size_t n = pend_n_;
  pend_n_ = 0;  // the device owns the tokens now (or the append failed and threw)
  check(ttkv_gpu_append(h_, pend_k_.data(), pend_v_.data(), n, TTKV_DTYPE_F32), h_);
  pend_k_.clear();
  pend_v_.clear();
}

std::size_t TierStore::appended_now() const {
  ttkv_state st{};
  check(ttkv_gpu_state(h_, &st), h_);  // host-side bookkeeping, no device work
  return st.appended + pend_n_;
}

std::size_t TierStore::fast_now() const {
  ttkv_state st{};
  check(ttkv_gpu_state(h_, &st), h_);
  return st.fast_tokens + pend_n_;
}

ttkv_state TierStore::state() const {
  flush();
  ttkv_state st{};
  check(ttkv_gpu_state(h_, &st), h_);
  return st;
}

std::vector<CacheEvent> TierStore::append_token(TokenKV kv) {
  const std::size_t appended = appended_now(), fast_before = fast_now();
  if (kv.position != appended)
    throw SequencingError("append_token: expected position " + std::to_string(appended) +
                          ", got " + std::to_string(kv.position));
  if (kv.key.size() != config_.d_k || kv.value.size() != config_.d_v)
    throw ShapeError("append_token: key/value dimension mismatch");
  if (fast_before + 1 > l_fast_ + config_.block_size || pend_n_ >= 4096) {
    // the ring bound (or a full buffer): hand over now, so an overflow is
    // reported by this append as before
    flush();
    check(ttkv_gpu_append(h_, kv.key.data(), kv.value.data(), 1, TTKV_DTYPE_F32), h_);
  } else {
    pend_k_.insert(pend_k_.end(), kv.key.begin(), kv.key.end());
    pend_v_.insert(pend_v_.end(), kv.value.begin(), kv.value.end());
    ++pend_n_;
  }
  invalidate();
  std::vector<CacheEvent> events;
  const std::size_t fast = fast_before + 1;
  if (fast > l_fast_) {
    const Position first = appended + 1 - fast;
    events.push_back({CacheEvent::Type::EvictBlock, first, first + config_.block_size - 1});
  }
  return events;
}

bool TierStore::eviction_pending() const { return fast_now() > l_fast_; }

BlockId TierStore::evict_and_compress() {
  flush();
  std::uint64_t id = 0;
  check(ttkv_gpu_evict(h_, &id), h_);
  index_.append_block(id, id * config_.block_size, id * config_.block_size + config_.block_size - 1);
  invalidate();
  return id;
}

void TierStore::note_decode_step(std::size_t) {
  const ttkv_state st = state();
  for (BlockId id = index_.size(); id < st.slow_blocks; ++id)
    index_.append_block(id, id * config_.block_size,
                        id * config_.block_size + config_.block_size - 1);
  invalidate();
}

Location TierStore::locate(Position p) const {
  const std::size_t appended = appended_now(), fast = fast_now();
  if (p >= appended) return Location::absent();
  if (fast > 0 && p >= appended - fast) return Location::fast();
  if (auto id = index_.find(p)) return Location::slow(*id);
  return Location::absent();
}

const std::deque<TokenKV>& TierStore::fast_tokens() const {
  if (fast_valid_) return fast_view_;
  const ttkv_state st = state();
  std::vector<float> k(std::max<std::size_t>(1, st.fast_tokens * config_.d_k));
  std::vector<float> v(std::max<std::size_t>(1, st.fast_tokens * config_.d_v));
  std::uint64_t n = 0, first = 0;
  check(ttkv_gpu_read_fast(h_, 0, k.data(), v.data(), st.fast_tokens, &n, &first), h_);
  fast_view_.clear();
  for (std::uint64_t t = 0; t < n; ++t) {
    TokenKV tok;
    tok.position = first + t;
    tok.key.assign(k.begin() + t * config_.d_k, k.begin() + (t + 1) * config_.d_k);
    tok.value.assign(v.begin() + t * config_.d_v, v.begin() + (t + 1) * config_.d_v);
    fast_view_.push_back(std::move(tok));
  }
  fast_valid_ = true;
  return fast_view_;
}

const std::vector<QuantizedBlock>& TierStore::slow_blocks() const {
  const ttkv_state st = state();
  const std::size_t B = config_.block_size;
  while (slow_view_.size() < st.slow_blocks) {
    const BlockId id = slow_view_.size();
    QuantizedBlock q;
    q.block_id = id;
    q.token_count = static_cast<std::uint32_t>(B);
    q.d_k = static_cast<std::uint32_t>(config_.d_k);
    q.d_v = static_cast<std::uint32_t>(config_.d_v);
    q.key_bits = config_.key_bits;
    q.value_bits = config_.value_bits;
    q.packed_keys.resize(stored_bytes(B * config_.d_k, config_.key_bits));
    q.packed_values.resize(stored_bytes(B * config_.d_v, config_.value_bits));
    std::vector<float> kp(2 * config_.d_k), vp(2 * config_.d_v);
    q.key_centroid.resize(config_.d_k);
    std::uint64_t first = 0;
    check(ttkv_gpu_read_block(h_, 0, id, q.packed_keys.data(), q.packed_values.data(), kp.data(),
                              vp.data(), q.key_centroid.data(), &first),
          h_);
    q.first_position = first;
    q.last_position = first + B - 1;
    if (config_.key_bits != 16) {
      q.key_params.resize(config_.d_k);
      for (std::size_t c = 0; c < config_.d_k; ++c) q.key_params[c] = {kp[2 * c], kp[2 * c + 1]};
    }
    if (config_.value_bits != 16) {
      q.value_params.resize(config_.d_v);
      for (std::size_t c = 0; c < config_.d_v; ++c)
        q.value_params[c] = {vp[2 * c], vp[2 * c + 1]};
    }
    slow_view_.push_back(std::move(q));
  }
  return slow_view_;
}

std::size_t TierStore::fast_token_count() const { return fast_now(); }
std::size_t TierStore::slow_token_count() const {
  ttkv_state st{};
  check(ttkv_gpu_state(h_, &st), h_);
  return st.slow_blocks * config_.block_size;
}
std::size_t TierStore::appended_count() const { return appended_now(); }

// ---- workload generator ------------------------------------------------------------------
double detail::GaussianSource::next() {
  if (have_cached_) {
    have_cached_ = false;
    return cached_;
  }
  // Box-Muller on two 53-bit uniforms; u1 in (0, 1] keeps the log finite
  constexpr double kInv53 = 0x1.0p-53;
  const double u1 = (double(gen_() >> 11) + 1.0) * kInv53;
  const double u2 = double(gen_() >> 11) * kInv53;
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * std::numbers::pi * u2;
  cached_ = radius * std::sin(angle);
  have_cached_ = true;
  return radius * std::cos(angle);
}

void WorkloadSpec::validate() const {
  if (context_length < 1) throw ConfigError("context_length must be >= 1");
  if (d_k == 0 || d_v == 0) throw ConfigError("d_k and d_v must be positive");
  if (kind == Kind::PlantedNeedle) {
    if (needle_block_position * kNeedleSpanTokens + kNeedleSpanTokens > context_length)
      throw ConfigError("needle span extends past the context");
    if (needle_alignment_strength <= 0)
      throw ConfigError("needle_alignment_strength must be positive");
  }
}

WorkloadStream generate_workload(const WorkloadSpec& spec) {
  spec.validate();
  detail::GaussianSource rng(spec.seed);
  const bool needle = spec.kind == WorkloadSpec::Kind::PlantedNeedle;
  WorkloadStream ws;
  std::vector<float> dir;
  if (needle) {
    dir.assign(spec.d_k, 1.0f / std::sqrt(static_cast<float>(spec.d_k)));
    ws.needle_direction = dir;
  }
  const std::size_t n0 = spec.needle_block_position * kNeedleSpanTokens;
  const double shift = spec.needle_alignment_strength / std::sqrt(double(kNeedleSpanTokens));
  auto token = [&](Position pos) {
    TokenKV t;
    t.position = pos;
    t.key.resize(spec.d_k);
    t.value.resize(spec.d_v);
    const bool planted = needle && pos >= n0 && pos < n0 + kNeedleSpanTokens;
    for (std::size_t i = 0; i < spec.d_k; ++i) {
      double x = rng.next();
      if (planted) x += shift * dir[i];
      t.key[i] = static_cast<float>(x);
    }
    for (float& v : t.value) v = rng.nextf();
    return t;
  };
  ws.prefill.reserve(spec.context_length);
  for (Position p = 0; p < spec.context_length; ++p) ws.prefill.push_back(token(p));
  ws.decode.reserve(spec.decode_steps);
  for (std::size_t s = 0; s < spec.decode_steps; ++s) {
    DecodeInput in;
    in.kv = token(spec.context_length + s);
    if (needle) {
      in.query = dir;
    } else {
      in.query.resize(spec.d_k);
      for (float& q : in.query) q = rng.nextf();
    }
    ws.decode.push_back(std::move(in));
  }
  return ws;
}

// ---- engine --------------------------------------------------------------------------------
Engine::Engine(TierConfig config, SelectionPolicy policy, EngineOptions options)
    : policy_(policy),
      options_(options),
      store_(std::move(config), policy, options.literal_additive_merge) {}

void Engine::prefill(std::span<const TokenKV> tokens) {
  if (tokens.empty()) return;
  const TierConfig& cfg = store_.config();
  const std::size_t base = store_.appended_count();
  std::vector<float> k(tokens.size() * cfg.d_k), v(tokens.size() * cfg.d_v);
  for (std::size_t t = 0; t < tokens.size(); ++t) {  // append_token's checks, in order
    if (tokens[t].position != base + t)
      throw SequencingError("append_token: expected position " + std::to_string(base + t) +
                            ", got " + std::to_string(tokens[t].position));
    if (tokens[t].key.size() != cfg.d_k || tokens[t].value.size() != cfg.d_v)
      throw ShapeError("append_token: key/value dimension mismatch");
    std::copy(tokens[t].key.begin(), tokens[t].key.end(), k.begin() + t * cfg.d_k);
    std::copy(tokens[t].value.begin(), tokens[t].value.end(), v.begin() + t * cfg.d_v);
  }
  check(ttkv_gpu_prefill(store_.handle(), k.data(), v.data(), tokens.size(), TTKV_DTYPE_F32),
        store_.handle());
  store_.note_decode_step(0);
}

DecodeStepReport Engine::decode_step(std::span<const float> query, TokenKV kv) {
  const TierConfig& cfg = store_.config();
  if (query.size() != cfg.d_k) throw ShapeError("decode_step: query dimension mismatch");
  const std::size_t pos = store_.appended_count();
  if (kv.position != pos)
    throw SequencingError("append_token: expected position " + std::to_string(pos) + ", got " +
                          std::to_string(kv.position));
  if (kv.key.size() != cfg.d_k || kv.value.size() != cfg.d_v)
    throw ShapeError("append_token: key/value dimension mismatch");
  std::vector<double> out(cfg.d_v);
  ttkv_step_report rep{};
  ttkv_gpu* h = store_.handle();
  check(ttkv_gpu_decode_step(h, query.data(), kv.key.data(), kv.value.data(), TTKV_DTYPE_F32,
                             out.data(), &rep),
        h);
  DecodeStepReport r;
  r.output.assign(out.begin(), out.end());
  r.blocks_scored = rep.blocks_scored;
  r.blocks_fetched = rep.blocks_fetched;
  r.bytes_transferred = rep.bytes_transferred;
  r.eviction_occurred = rep.eviction_occurred != 0;
  r.fetched_blocks.resize(rep.blocks_fetched);
  std::uint64_t n = 0;
  if (rep.blocks_fetched)
    check(ttkv_gpu_read_fetched(h, 0, 0, r.fetched_blocks.data(), r.fetched_blocks.size(), &n), h);
  // simulator-facing workload description (engine.cpp:41-42, 78-82)
  r.workload.compute_items.push_back({"fast", double(rep.fast_tokens * cfg.d_kv())});
  const double per_block = double(modeled_block_bytes(cfg));
  for (BlockId id : r.fetched_blocks) {
    const std::string label = "blk" + std::to_string(id);
    r.workload.compute_items.push_back({label, double(cfg.block_size * cfg.d_kv())});
    r.workload.transfer_items.push_back({label, per_block});
  }
  store_.note_decode_step(r.eviction_occurred ? 1 : 0);
  return r;
}

std::vector<DecodeStepReport> Engine::decode_sequence(std::span<const DecodeInput> inputs) {
  std::vector<DecodeStepReport> out;
  out.reserve(inputs.size());
  for (const DecodeInput& in : inputs) out.push_back(decode_step(in.query, in.kv));
  return out;
}

// ---- dense oracle (host test utility) ---------------------------------------------------
namespace reference {

std::vector<double> dense_attention(std::span<const float> query,
                                    std::span<const TokenKV> history) {
  if (history.empty()) throw Error("dense_attention: empty history");
  const std::size_t dk = query.size(), dv = history.front().value.size();
  const double scale = 1.0 / std::sqrt(double(dk));
  std::vector<double> logit(history.size());
  double top = -std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < history.size(); ++i) {
    if (history[i].key.size() != dk || history[i].value.size() != dv)
      throw ShapeError("dense_attention: inconsistent history shapes");
    double dot = 0.0;
    for (std::size_t j = 0; j < dk; ++j) dot += double(query[j]) * history[i].key[j];
    logit[i] = dot * scale;
    top = std::max(top, logit[i]);
  }
  std::vector<double> out(dv, 0.0);
  double z = 0.0;
  for (std::size_t i = 0; i < history.size(); ++i) {
    const double w = std::exp(logit[i] - top);
    z += w;
    for (std::size_t j = 0; j < dv; ++j) out[j] += w * history[i].value[j];
  }
  for (double& x : out) x /= z;
  return out;
}

double relative_error(std::span<const double> a, std::span<const double> b) {
  if (a.size() != b.size()) throw ShapeError("relative_error: size mismatch");
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

}  // namespace reference
}  // namespace ttkv

// ---- C entry (include/ttkv_dropin_c.h) --------------------------------------------
#include "ttkv_dropin_c.h"

extern "C" int ttkv_generate_workload(int needle, uint64_t ctx, uint64_t T, uint32_t d_k,
                                      uint32_t d_v, uint64_t seed, uint64_t needle_pos,
                                      double strength, float* pre_k, float* pre_v, float* dec_k,
                                      float* dec_v, float* dec_q) {
  try {
    ttkv::WorkloadSpec s;
    s.kind = needle ? ttkv::WorkloadSpec::Kind::PlantedNeedle : ttkv::WorkloadSpec::Kind::Gaussian;
    s.context_length = ctx;
    s.decode_steps = T;
    s.d_k = d_k;
    s.d_v = d_v;
    s.seed = seed;
    s.needle_block_position = needle_pos;
    s.needle_alignment_strength = strength;
    const ttkv::WorkloadStream w = ttkv::generate_workload(s);
    for (uint64_t p = 0; p < ctx; ++p) {
      std::copy(w.prefill[p].key.begin(), w.prefill[p].key.end(), pre_k + p * d_k);
      std::copy(w.prefill[p].value.begin(), w.prefill[p].value.end(), pre_v + p * d_v);
    }
    for (uint64_t t = 0; t < T; ++t) {
      std::copy(w.decode[t].kv.key.begin(), w.decode[t].kv.key.end(), dec_k + t * d_k);
      std::copy(w.decode[t].kv.value.begin(), w.decode[t].kv.value.end(), dec_v + t * d_v);
      std::copy(w.decode[t].query.begin(), w.decode[t].query.end(), dec_q + t * d_k);
    }
    return TTKV_OK;
  } catch (const std::exception&) {
    return TTKV_ECONFIG;
  }
}
