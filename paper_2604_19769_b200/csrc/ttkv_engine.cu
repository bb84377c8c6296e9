// ttkv_engine.cu -- the C ABI (include/ttkv_gpu.h): handle, memory, step
// orchestration.  Host side of the B200 TTKV decode path; all compute is in
// the sm_100a kernels of ttkv_{quantize,select,attention}.cu.  There is no
// CPU fallback: without a device every call fails with TTKV_ECUDA.
//
// Step schedule (Engine::decode_step, engine.cpp:22-93), S streams at once:
//   s0: append_kv -> [fork] -> score_blocks -> select_topk -> slow_stream_attn
//   s1:              [fork] -> fast_attn_partial -> [join]
//   s0: [join] -> combine_partials -> evict_quantize (every B-th step)
// The fast tier (HBM) overlaps the PCIe-bound slow stream; selection never
// leaves the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/ttkv_gpu.h"
#include "ttkv_launch.h"

using namespace ttkv_dev;

namespace {

thread_local std::string g_last_error;

struct Err {
  int code;
  std::string msg;
};

uint64_t packed_bytes_u(uint64_t count, uint32_t bits) {
  if (bits == 16) return count * 4;  // raw float32 (quantizer.cpp:12-15)
  return (count * bits + 7) / 8;
}
uint64_t modeled_bytes_u(uint64_t count, uint32_t bits) {
  if (bits == 16) return count * 2;  // quantizer.cpp:17-20
  return (count * bits + 7) / 8;
}
uint64_t modeled_block_bytes_cfg(const ttkv_tier_config& c) {  // quantizer.cpp:172-180
  uint64_t b = modeled_bytes_u(c.block_size * c.d_k, c.key_bits) +
               modeled_bytes_u(c.block_size * c.d_v, c.value_bits);
  if (c.key_bits != 16) b += 4 * c.d_k;
  if (c.value_bits != 16) b += 4 * c.d_v;
  return b;
}

// TierConfig::validate (config.hpp:56-74), same messages.
int validate(const ttkv_tier_config& c, std::string& msg) {
  auto fail = [&](const char* m) {
    msg = m;
    return TTKV_ECONFIG;
  };
  if (c.d_k == 0 || c.d_v == 0) return fail("d_k and d_v must be positive");
  if (c.block_size == 0) return fail("block_size must be positive");
  if (c.bytes_full_precision == 0) return fail("bytes_full_precision must be positive");
  auto valid_bits = [](uint32_t b) { return (b >= 2 && b <= 8) || b == 16; };
  if (!valid_bits(c.key_bits) || !valid_bits(c.value_bits))
    return fail("bit widths must be in [2,8] or 16");
  if (c.key_bits < c.value_bits) return fail("key_bits must be >= value_bits");
  if (c.hbm_budget_bytes < c.block_size * (c.d_k + c.d_v) * c.bytes_full_precision)
    return fail("HBM budget smaller than one full-precision block");
  if (!(c.fetch_fraction > 0.0 && c.fetch_fraction <= 1.0) && !c.has_top_k_blocks)
    return fail("fetch_fraction must be in (0, 1]");
  if (c.hbm_bandwidth <= 0 || c.pcie_bandwidth <= 0 || c.compute_rate <= 0)
    return fail("bandwidths and compute_rate must be positive");
  if (c.transfer_latency < 0) return fail("transfer_latency must be non-negative");
  return TTKV_OK;
}

// fast_capacity (tier_store.cpp:36-44)
int fast_capacity_of(const ttkv_tier_config& c, uint64_t& out, std::string& msg) {
  int rc = validate(c, msg);
  if (rc) return rc;
  const uint64_t per_token = (c.d_k + c.d_v) * c.bytes_full_precision;
  uint64_t tokens = c.hbm_budget_bytes / per_token;
  tokens -= tokens % c.block_size;
  if (tokens < c.block_size) {
    msg = "HBM budget holds fewer tokens than one block";
    return TTKV_ECONFIG;
  }
  out = tokens;
  return TTKV_OK;
}

// SelectionPolicy::resolve (relevance.cpp:10-17)
int resolve_k(const ttkv_selection_policy& p, uint64_t n, uint64_t& k, std::string& msg) {
  if (p.has_top_k) {
    k = std::min<uint64_t>(p.top_k, n);
    return TTKV_OK;
  }
  if (!(p.fetch_fraction > 0.0 && p.fetch_fraction <= 1.0)) {
    msg = "fetch_fraction must be in (0, 1]";
    return TTKV_ECONFIG;
  }
  const uint64_t kk = (uint64_t)std::ceil(p.fetch_fraction * (double)n);
  k = std::min<uint64_t>(kk, n);
  return TTKV_OK;
}

// Process-wide cache of pinned, mapped host blocks.  Pinning costs ~3 ms per
// MB-scale arena (measured on the GPU box), and handles are created per
// request when serving and per trial in the reference's acceptance gate, so
// freed blocks are kept (up to kPinnedCacheMax bytes) and reused for any
// request they cover within 2x.  Leaked at exit on purpose (process lifetime).
struct PinnedCache {
  std::mutex mu;
  std::multimap<size_t, void*> idle;     // size -> block
  std::unordered_map<void*, size_t> size_of;  // every block handed out or idle
  size_t idle_bytes = 0;
};
constexpr size_t kPinnedCacheMax = 8ull << 30;
PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache;
  return *c;
}
cudaError_t pinned_alloc(void** p, size_t bytes) {
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.idle.lower_bound(bytes);
    if (it != c.idle.end() && it->first <= 2 * bytes + (1u << 20)) {
      *p = it->second;
      c.idle_bytes -= it->first;
      c.idle.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaHostAlloc(p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(c.mu);
    c.size_of[*p] = bytes;
  }
  return e;
}
void pinned_free(void* p) {
  if (!p) return;
  PinnedCache& c = pinned_cache();
  std::unique_lock<std::mutex> lk(c.mu);
  const auto it = c.size_of.find(p);
  if (it == c.size_of.end()) {  // not ours
    lk.unlock();
    cudaFreeHost(p);
    return;
  }
  if (c.idle_bytes + it->second <= kPinnedCacheMax) {
    c.idle.emplace(it->second, p);
    c.idle_bytes += it->second;
    return;
  }
  c.size_of.erase(it);
  lk.unlock();
  cudaFreeHost(p);
}

uint32_t align_up(uint64_t x, uint64_t a) { return (uint32_t)((x + a - 1) / a * a); }

RecordLayout make_layout(uint32_t B, uint32_t d_k, uint32_t d_v, uint32_t kb, uint32_t vb,
                         uint32_t elem) {
  RecordLayout r{};
  r.k_bytes = kb == 16 ? B * d_k * elem : (uint32_t)((uint64_t(B) * d_k * kb + 7) / 8);
  r.v_bytes = vb == 16 ? B * d_v * elem : (uint32_t)((uint64_t(B) * d_v * vb + 7) / 8);
  r.v_off = align_up(r.k_bytes, 16);
  r.kp_off = align_up(r.v_off + r.v_bytes, 16);
  const uint32_t kp = kb == 16 ? 0 : 8 * d_k;
  r.vp_off = align_up(r.kp_off + kp, 16);
  const uint32_t vp = vb == 16 ? 0 : 8 * d_v;
  r.used = align_up(r.vp_off + vp, 16);
  r.stride = align_up(r.used, 128);
  return r;
}

const char* kKernelNames[] = {"append", "score", "select", "fast", "slow", "combine", "evict", "gather", "step"};
enum Kind { K_APPEND = 0, K_SCORE, K_SELECT, K_FAST, K_SLOW, K_COMBINE, K_EVICT, K_GATHER, K_STEP, K_N };

}  // namespace

void ttkv_dev::set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
int ttkv_dev::launch_priority(bool critical) {
  static int least = 1, greatest = 1;  // 1: not queried yet (valid values are <= 0)
  if (least == 1) {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) lo = hi = 0;
    greatest = hi;
    least = lo;
  }
  return critical ? greatest : least;
}
bool ttkv_dev::pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TTKV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

struct ttkv_gpu {
  // fused combine + all-gather over peer memory (ttkv_gpu_peer_gather_*)
  struct PeerGather {
    uint32_t n_ranks = 0, my_rank = 0;
    uint64_t s_global = 0;
    uint8_t* base = nullptr;  // own [2][S_global][G][d_v] f64 rows + [8] u64 counters
    size_t out_bytes = 0;
    uint32_t* gidx = nullptr;  // device [S_local]
    int* status = nullptr;     // device
    void* peer_base[ttkv_dev::kMaxPeers] = {};  // IPC-opened peers (null for self)
    unsigned long long epoch = 0;
    bool active = false;
  } pg;
  ttkv_tier_config cfg{};
  ttkv_selection_policy pol{};
  ttkv_gpu_options opt{};
  std::string err;
  int dev = 0;
  cudaStream_t s0 = nullptr, s1 = nullptr;
  bool own_s0 = true;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_start = nullptr;
  Geometry g{};
  uint64_t l_fast = 0;
  uint32_t copy_mode = 1;
  uint32_t stages = 1;
  // lockstep bookkeeping (identical for every stream)
  uint64_t appended = 0, n_slow = 0, fast_front = 0;
  uint64_t last_k = 0, last_n = 0;
  // fast split
  uint32_t FC = 256, nfc_cap = 1, TT = 64;
  bool fast_tc = false;      // tensor-core fast tier (TMA tensor maps)
  FastTcArgs tc{};           // ring tensor maps, encoded once at create
  bool slow_tc = false;      // tensor-core slow tier (arena tensor maps)
  int sms = 148;             // SM count of the device
  SlowTcArgs stc{};          // re-encoded whenever the arena is reallocated
  uint8_t* stage_arena = nullptr;  // serial schedule: HBM copy of selected records
  double last_step_ms = 0.0;
  size_t acc = 4;  // bytes of the accumulation type (fp32, or fp64 for the fp32 ring)
  // device memory
  void* ring_k = nullptr;
  void* ring_v = nullptr;
  float* cent = nullptr;
  uint8_t* params = nullptr;  // HBM mirror of record params
  double* scores = nullptr;
  uint32_t *mask = nullptr, *uids = nullptr, *umask = nullptr, *ucount = nullptr;
  uint32_t* nslots = nullptr;  // slow partial slots per stream (tensor-core slow tier)
  uint32_t* h_ucount = nullptr;  // pinned copy of union_count for the step report
  uint32_t* h_ucount_dev = nullptr;  // ... its device mapping (the combine writes it)
  IoSlot* io = nullptr;      // host-buffer steps: q/k/v/out addresses (mapped, pinned)
  IoSlot* io_dev = nullptr;  // ... its device mapping (read by the ingest kernel)
  double** out_ref = nullptr;  // device word: the step's output address (ingest -> combine)
  // device-side join of the fast tier into the combine: {fast arrive, fast
  // epoch, combine arrive, combine epoch}
  uint32_t* join = nullptr;
  void* fpart = nullptr;
  void* spart = nullptr;
  uint64_t spart_chunks = 0;
  // speculative record stream (HBM tier, small steps): per-record partials
  // [S][G][n_cap][kSpecPitch] and the record queue head
  float* rpart = nullptr;
  uint64_t rpart_cap = 0;
  uint32_t* spec_ctr = nullptr;
  uint64_t spec_steps = 0;
  float* q_dev = nullptr;
  void *kn_dev = nullptr, *vn_dev = nullptr;
  void *stg_k = nullptr, *stg_v = nullptr;
  uint64_t stg_tokens = 0;
  // arena
  uint8_t* arena_host = nullptr;  // pinned (TTKV_SLOW_PINNED_HOST)
  uint8_t* arena_dev = nullptr;   // device-visible pointer
  // pinned staging for the host-buffer API
  float* h_q = nullptr;
  double* h_out = nullptr;
  void *h_k = nullptr, *h_v = nullptr;
  // timing
  bool timing = false;
  struct Rec {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  struct TlEvent {
    int kind;
    double start, end;  // ms from the step's start
  };
  std::vector<TlEvent> timeline;  // kernels of the last timed step
  std::vector<cudaEvent_t> pool;
  double ms[K_N] = {};
  uint64_t cnt[K_N] = {};
  uint64_t launches = 0;
  // Device step position (= `appended` before the step): the append slot and
  // the fast tier's length are read from it on the device and the combine
  // advances it, so a decode step's launches do not change from one step to
  // the next within an eviction period and replay as one CUDA graph.
  uint64_t* pos_dev = nullptr;
  bool pos_synced = false;  // pos_dev == appended (host-side appends clear it)
  uint64_t gen = 0;         // bumped whenever a buffer a captured step uses moves
  struct GraphKey {
    const void *q, *kn, *vn, *out;
    cudaStream_t s0;
    uint64_t n, k, front, gen, grid_chunks;
    uint32_t nfc, CH, dtype, host_io;
  };
  struct StepGraph {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t launches;  // kernels per replay
    uint64_t last_use;
  };
  // A few captured steps per eviction period: callers that rotate their
  // input/output buffers get one graph per buffer set (the pointers are
  // kernel arguments of the captured launches).
  static constexpr size_t kMaxGraphs = 8;
  std::vector<StepGraph> graphs;
  uint64_t graph_replays = 0, graph_captures = 0;
};

namespace {

int set_err(ttkv_gpu* h, int code, const std::string& m) {
  if (h) h->err = m;
  g_last_error = m;
  return code;
}

#define CU(h, call)                                                                        \
  do {                                                                                     \
    cudaError_t e__ = (call);                                                              \
    if (e__ != cudaSuccess)                                                                \
      return set_err((h), TTKV_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

cudaEvent_t take_event(ttkv_gpu* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Whole-step device time (append .. settle) on the critical-path stream.
struct StepTimer {
  ttkv_gpu* h;
  cudaEvent_t a = nullptr;
  explicit StepTimer(ttkv_gpu* hh);
  ~StepTimer();
};

struct KTimer {
  ttkv_gpu* h;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  KTimer(ttkv_gpu* hh, int k, cudaStream_t s, int n_kernels = 1) : h(hh), kind(k), st(s) {
    h->launches += n_kernels;
    if (h->timing) {
      a = take_event(h);
      cudaEventRecord(a, st);
    }
  }
  ~KTimer() {
    if (a) {
      cudaEvent_t b = take_event(h);
      cudaEventRecord(b, st);
      h->recs.push_back({kind, a, b});
    }
  }
};

void drain_timing(ttkv_gpu* h) {
  // Kernel records of a step precede that step's K_STEP record (StepTimer
  // closes last); the last step's kernels are kept as a timeline relative to
  // the step's start event (write_run_timelines, harness.cpp:291-300).
  size_t first = 0;
  for (size_t i = 0; i < h->recs.size(); ++i) {
    auto& r = h->recs[i];
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    h->ms[r.kind] += ms;
    h->cnt[r.kind] += 1;
    if (r.kind == K_STEP) {
      h->last_step_ms = ms;
      h->timeline.clear();
      for (size_t j = first; j < i; ++j) {
        float t0 = 0.f, t1 = 0.f;
        cudaEventElapsedTime(&t0, r.a, h->recs[j].a);
        cudaEventElapsedTime(&t1, r.a, h->recs[j].b);
        h->timeline.push_back({h->recs[j].kind, (double)t0, (double)t1});
      }
      first = i + 1;
    }
  }
  for (auto& r : h->recs) {
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
}

void free_peer_gather(ttkv_gpu* h) {
  for (auto& p : h->pg.peer_base)
    if (p) {
      cudaIpcCloseMemHandle(p);
      p = nullptr;
    }
  if (h->pg.base) cudaFree(h->pg.base);
  if (h->pg.gidx) cudaFree(h->pg.gidx);
  if (h->pg.status) cudaFree(h->pg.status);
  h->pg = ttkv_gpu::PeerGather{};
}

void free_all(ttkv_gpu* h) {
  free_peer_gather(h);
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(h->ring_k); F(h->ring_v); F(h->cent); F(h->params); F(h->scores); F(h->mask); F(h->uids);
  F(h->umask); F(h->ucount); F(h->nslots); F(h->fpart); F(h->spart); F(h->q_dev);
  F(h->rpart); F(h->spec_ctr); F(h->out_ref); F(h->join);
  F(h->kn_dev); F(h->vn_dev); F(h->stg_k); F(h->stg_v); F(h->stage_arena);
  if (h->arena_host) pinned_free(h->arena_host);
  else if (h->arena_dev) cudaFree(h->arena_dev);
  pinned_free(h->h_q);
  pinned_free(h->h_out);
  pinned_free(h->h_k);
  pinned_free(h->h_v);
  pinned_free(h->h_ucount);
  pinned_free(h->io);
  F(h->pos_dev);
  for (auto& sg : h->graphs) cudaGraphExecDestroy(sg.exec);
  h->graphs.clear();
  for (auto& r : h->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_start) cudaEventDestroy(h->ev_start);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->s1) cudaStreamDestroy(h->s1);
  if (h->s0 && h->own_s0) cudaStreamDestroy(h->s0);
}

// (Re)allocate the per-block arrays for `need` blocks per stream.
int ensure_blocks(ttkv_gpu* h, uint64_t need) {
  if (need <= h->g.n_cap && h->arena_dev) return TTKV_OK;
  if (need > select_max_blocks())
    return set_err(h, TTKV_ECONFIG,
                   "context exceeds the GPU selection capacity (" +
                       std::to_string(select_max_blocks()) + " blocks per stream)");
  const uint64_t old_cap = h->arena_dev ? h->g.n_cap : 0;
  uint64_t cap = std::max<uint64_t>(need, old_cap ? 2 * old_cap : 16);
  cap = std::min<uint64_t>(cap, select_max_blocks());
  const uint64_t S = h->g.S, stride = h->g.rec.stride;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  // arena
  uint8_t *nh = nullptr, *nd = nullptr;
  const size_t arena_bytes = S * cap * stride;
  if (h->opt.slow_tier == TTKV_SLOW_PINNED_HOST) {
    CU(h, pinned_alloc((void**)&nh, arena_bytes));
    CU(h, cudaHostGetDevicePointer((void**)&nd, nh, 0));
  } else {
    CU(h, cudaMalloc((void**)&nd, arena_bytes));
  }
  float* ncent = nullptr;
  CU(h, cudaMalloc((void**)&ncent, S * cap * h->g.d_k * sizeof(float)));
  const uint64_t pbytes = h->g.rec.used - h->g.rec.kp_off;
  uint8_t* nparams = nullptr;
  if (pbytes) CU(h, cudaMalloc((void**)&nparams, S * cap * pbytes));
  double* nscores = nullptr;  // the last step's scores stay readable (fetched_blocks)
  CU(h, cudaMalloc((void**)&nscores, S * h->g.Gs * cap * sizeof(double)));
  if (old_cap && h->last_n && h->scores)
    CU(h, cudaMemcpy2D(nscores, cap * 8, h->scores, old_cap * 8, h->last_n * 8, S * h->g.Gs,
                       cudaMemcpyDeviceToDevice));
  if (old_cap && h->n_slow && pbytes)
    CU(h, cudaMemcpy2D(nparams, cap * pbytes, h->params, old_cap * pbytes, h->n_slow * pbytes, S,
                       cudaMemcpyDeviceToDevice));
  if (old_cap && h->n_slow) {
    CU(h, cudaMemcpy2D(nh ? (void*)nh : (void*)nd, cap * stride,
                       h->arena_host ? (void*)h->arena_host : (void*)h->arena_dev,
                       old_cap * stride, h->n_slow * stride, S, cudaMemcpyDefault));
    CU(h, cudaMemcpy2D(ncent, cap * h->g.d_k * 4, h->cent, old_cap * h->g.d_k * 4,
                       h->n_slow * h->g.d_k * 4, S, cudaMemcpyDeviceToDevice));
  }
  if (h->arena_host) pinned_free(h->arena_host);
  else if (h->arena_dev) cudaFree(h->arena_dev);
  if (h->cent) cudaFree(h->cent);
  if (h->params) cudaFree(h->params);
  h->arena_host = nh;
  h->arena_dev = nd;
  h->cent = ncent;
  h->params = nparams;
  // per-step selection arrays (contents are per step; no copy)
  auto realloc_dev = [&](void** p, size_t bytes) -> cudaError_t {
    if (*p) cudaFree(*p);
    *p = nullptr;
    return cudaMalloc(p, bytes);
  };
  if (h->scores) cudaFree(h->scores);
  h->scores = nscores;
  CU(h, realloc_dev((void**)&h->mask, S * cap * sizeof(uint32_t)));
  CU(h, cudaMemset(h->mask, 0, S * cap * sizeof(uint32_t)));  // select leaves it zeroed
  // the last step's union (the records it streamed) stays readable too
  // (ttkv_gpu_read_selected / read_fetched)
  uint32_t *nuids = nullptr, *numask = nullptr;
  CU(h, cudaMalloc((void**)&nuids, S * cap * sizeof(uint32_t)));
  CU(h, cudaMalloc((void**)&numask, S * cap * sizeof(uint32_t)));
  if (old_cap && h->last_k && h->uids) {
    CU(h, cudaMemcpy2D(nuids, cap * 4, h->uids, old_cap * 4, old_cap * 4, S,
                       cudaMemcpyDeviceToDevice));
    CU(h, cudaMemcpy2D(numask, cap * 4, h->umask, old_cap * 4, old_cap * 4, S,
                       cudaMemcpyDeviceToDevice));
  }
  if (h->uids) cudaFree(h->uids);
  if (h->umask) cudaFree(h->umask);
  h->uids = nuids;
  h->umask = numask;
  h->g.n_cap = cap;
  h->gen++;  // captured steps hold the old pointers
  if (h->opt.serial_schedule) {
    CU(h, realloc_dev((void**)&h->stage_arena, arena_bytes));
  }
  uint8_t* attn_arena = h->opt.serial_schedule ? h->stage_arena : h->arena_dev;
  // TMA record coordinates are int32: very large handles use the CUDA-core tier
  if (h->slow_tc && (S * cap >= (1ull << 31) ||
                     make_arena_tmaps(h->g, attn_arena, h->stc) != cudaSuccess))
    h->slow_tc = false;  // fall back to the CUDA-core slow tier
  return TTKV_OK;
}

int ensure_spart(ttkv_gpu* h, uint64_t chunks) {
  if (chunks <= h->spart_chunks) return TTKV_OK;
  const uint64_t c = std::max<uint64_t>(chunks, 2 * h->spart_chunks);
  CU(h, cudaStreamSynchronize(h->s0));
  if (h->spart) cudaFree(h->spart);
  h->spart = nullptr;
  CU(h, cudaMalloc((void**)&h->spart, (size_t)h->g.S * h->g.G * c * (h->g.d_v + 2) * h->acc));
  h->spart_chunks = c;
  h->gen++;
  return TTKV_OK;
}

// Per-record partials of the speculative record stream, sized with the
// slow-block capacity (the rows are indexed by block id).
int ensure_rpart(ttkv_gpu* h) {
  if (!h->spec_ctr) {
    CU(h, cudaMalloc((void**)&h->spec_ctr, sizeof(uint32_t)));
    CU(h, cudaMemsetAsync(h->spec_ctr, 0, sizeof(uint32_t), h->s0));
    h->gen++;
  }
  if (h->rpart_cap >= h->g.n_cap && h->rpart) return TTKV_OK;
  CU(h, cudaStreamSynchronize(h->s0));
  if (h->rpart) cudaFree(h->rpart);
  h->rpart = nullptr;
  CU(h, cudaMalloc((void**)&h->rpart,
                   (size_t)h->g.S * h->g.G * h->g.n_cap * kSpecPitch * sizeof(float)));
  h->rpart_cap = h->g.n_cap;
  h->gen++;
  return TTKV_OK;
}

// Speculative record stream (slow_attn_tc_spec_kernel) for this step?  It
// streams every record instead of the union of the G heads' selections, in
// exchange for running beside the selection instead of after it (the union
// covers 1 - (1 - k/n)^G of the blocks for per-head selection: 0.91 at cfg2).
// Opt-in (record_stream = 2, or TTKV_SPEC=1): measured on one layer of cfg2
// (8 streams x 4 heads, 128K, HBM) it is not faster than the union stream --
// 62.4 vs 61.0 us per layer -- because the record kernel is bound by its
// per-CTA record rate, and sharing the SMs with the selection and the fast
// tier costs it as much as the selection's latency it hides.
bool want_spec(const ttkv_gpu* h, uint64_t n, uint64_t k) {
  static const int env = [] {  // TTKV_SPEC=0/1 overrides
    const char* e = std::getenv("TTKV_SPEC");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const Geometry& g = h->g;
  if (env == 0 || !h->slow_tc || !h->fast_tc || !slow_tc_spec_supported(g) ||
      h->opt.literal_additive_merge || h->opt.serial_schedule || n == 0 || k == 0 ||
      n > 0xffffffffull / g.S)
    return false;
  return env == 1 || h->opt.record_stream == 2;
}

int ensure_staging(ttkv_gpu* h, uint64_t tokens) {
  if (tokens <= h->stg_tokens) return TTKV_OK;
  CU(h, cudaStreamSynchronize(h->s0));
  if (h->stg_k) cudaFree(h->stg_k);
  if (h->stg_v) cudaFree(h->stg_v);
  h->stg_k = h->stg_v = nullptr;
  const size_t e = 4;  // sized for f32 input
  CU(h, cudaMalloc(&h->stg_k, (size_t)h->g.S * tokens * h->g.d_k * e));
  CU(h, cudaMalloc(&h->stg_v, (size_t)h->g.S * tokens * h->g.d_v * e));
  h->stg_tokens = tokens;
  return TTKV_OK;
}

// Evict every pending block (settle, engine.cpp:88-91; tier_store.cpp:71-98).
int settle_evictions(ttkv_gpu* h, bool* evicted) {
  while (h->appended - h->fast_front > h->l_fast) {
    int rc = ensure_blocks(h, h->n_slow + 1);
    if (rc) return rc;
    EvictArgs a{};
    a.g = h->g;
    a.ring_k = h->ring_k;
    a.ring_v = h->ring_v;
    a.in_k = a.in_v = nullptr;
    a.in_tokens = 0;
    a.split_pos = h->appended;  // everything from the ring
    a.first_block = h->n_slow;
    a.arena = h->arena_dev;
    a.cent = h->cent;
    a.params = h->params;
    {
      KTimer t(h, K_EVICT, h->s0);
      CU(h, launch_evict(a, 1, kInF32, h->s0));
    }
    h->n_slow++;
    h->fast_front += h->g.B;
    if (evicted) *evicted = true;
  }
  return TTKV_OK;
}

// Bulk prefill of P tokens already on the device (staging layout [S][P][d]).
int prefill_chunk(ttkv_gpu* h, const void* in_k, const void* in_v, int in_dtype, uint64_t P,
                  uint64_t stride = 0) {
  if (!stride) stride = P;  // tokens between consecutive streams' rows
  const uint64_t A = h->appended, total = A + P, B = h->g.B;
  uint64_t nb_after = h->n_slow;
  if (total > h->l_fast) nb_after = std::max<uint64_t>(nb_after, (total - h->l_fast - 1) / B + 1);
  int rc = ensure_blocks(h, nb_after);
  if (rc) return rc;
  if (nb_after > h->n_slow) {
    EvictArgs a{};
    a.g = h->g;
    a.ring_k = h->ring_k;
    a.ring_v = h->ring_v;
    a.in_k = in_k;
    a.in_v = in_v;
    a.in_tokens = stride;
    a.split_pos = A;
    a.first_block = h->n_slow;
    a.arena = h->arena_dev;
    a.cent = h->cent;
    a.params = h->params;
    KTimer t(h, K_EVICT, h->s0);
    CU(h, launch_evict(a, (uint32_t)(nb_after - h->n_slow), in_dtype, h->s0));
  }
  const uint64_t start = std::max<uint64_t>(A, nb_after * B);
  if (start < total) {
    const size_t esz = in_dtype == kInF16 ? 2 : 4;
    const uint8_t* kb = static_cast<const uint8_t*>(in_k) + (start - A) * h->g.d_k * esz;
    const uint8_t* vb = static_cast<const uint8_t*>(in_v) + (start - A) * h->g.d_v * esz;
    KTimer t(h, K_APPEND, h->s0);
    CU(h, launch_append(h->g, h->ring_k, h->ring_v, kb, vb, in_dtype, start, stride, total - start,
                        h->s0));
  }
  h->appended = total;
  h->n_slow = nb_after;
  h->fast_front = nb_after * B;
  h->pos_synced = false;
  return TTKV_OK;
}

uint64_t prefill_chunk_tokens(const ttkv_gpu* h) {
  // ~256 MB of f32 staging per chunk, a multiple of B
  const uint64_t per_tok = (uint64_t)h->g.S * (h->g.d_k + h->g.d_v) * 4;
  uint64_t P = (256ull << 20) / std::max<uint64_t>(per_tok, 1);
  P = std::max<uint64_t>(P / h->g.B * h->g.B, h->g.B);
  return P;
}

StepTimer::StepTimer(ttkv_gpu* hh) : h(hh) {
  if (h->timing) {
    a = take_event(h);
    cudaEventRecord(a, h->s0);
  }
}
StepTimer::~StepTimer() {
  if (a) {
    cudaEvent_t b = take_event(h);
    cudaEventRecord(b, h->s0);
    h->recs.push_back({K_STEP, a, b});
  }
}

// One decode step's launch parameters (decided on the host, before any
// stream work, so that the stream work can be captured as a graph).
struct StepPlan {
  const float* q;
  const void* kn;
  const void* vn;
  int dtype;
  double* out;
  bool host_io;  // q/k/v read from and the output written to host memory (h->io)
  uint64_t n, k, F;
  uint32_t FCs, nfc, CH;
  uint64_t grid_chunks;  // slow kernel grid: chunks per stream, or CTAs (tensor-core tier)
  uint64_t gather_chunks;
  uint32_t per_min;      // tensor-core tier: records per CTA at least
  bool slow, early_fork;
  bool fast_first;       // the record stream waits for the fast tier (measurement)
  bool fast_last;        // the fast tier runs on s0 after the record stream
  bool fused;            // score + select + union as one cluster kernel
  bool spec;             // speculative record stream beside the selection
  bool dev_join;         // the combine joins the fast tier on the device (no event wait)
  bool capturing;        // enqueue_step runs inside a graph capture
  double scale_log2;
};

// Every stream operation of one decode step (append .. combine), on s0 with
// the fast tier forked onto s1.  No host synchronization, no allocation.
int enqueue_step(ttkv_gpu* h, const StepPlan& P) {
  const Geometry& g = h->g;
  if (P.host_io) {
    // q/k/v read from mapped page-locked host memory by one kernel (not
    // three copy-engine transfers: ~4 us of queue latency each on a small step)
    const size_t esz = P.dtype == kInF16 ? 2 : 4;
    void* const dst[3] = {h->q_dev, h->kn_dev, h->vn_dev};
    const uint64_t bytes[3] = {(uint64_t)g.S * g.G * g.d_k * 4, (uint64_t)g.S * g.d_k * esz,
                               (uint64_t)g.S * g.d_v * esz};
    KTimer t(h, K_APPEND, h->s0);
    CU(h, launch_ingest(dst, bytes, h->io_dev, reinterpret_cast<void**>(h->out_ref), h->s0));
  }
  // append_kv: the new token attends to itself.  Only the fast
  // tier reads the ring, so the append runs on s1 ahead of the fast kernel and
  // stays off the critical path score -> select -> slow on s0.  Its slot is
  // the device step position mod C.
  // With the speculative record stream the record kernel holds every SM it
  // can get until the step's records are done, so a fast tier on the side
  // stream would start only at its end: append and fast tier then join the
  // step's programmatic chain instead (append -> selection -> fast tier ->
  // record stream -> combine), each launching as its predecessor starts.
  if (P.spec) {
    KTimer t(h, K_APPEND, h->s0);
    CU(h, launch_append(g, h->ring_k, h->ring_v, P.kn, P.vn, P.dtype, 0, 1, 1, h->s0, h->pos_dev,
                        true));
  } else {
    CU(h, cudaEventRecord(h->ev_start, h->s0));
    CU(h, cudaStreamWaitEvent(h->s1, h->ev_start, 0));
    {
      KTimer t(h, K_APPEND, h->s1);
      CU(h, launch_append(g, h->ring_k, h->ring_v, P.kn, P.vn, P.dtype, 0, 1, 1, h->s1,
                          h->pos_dev));
    }
    if (P.fast_last) CU(h, cudaEventRecord(h->ev_join, h->s1));  // the ring holds the token
  }
  auto fork_fast = [&]() -> int {
    if (P.spec || P.fast_last) {  // fast_tc is a precondition of both
      if (P.fast_last) CU(h, cudaStreamWaitEvent(h->s0, h->ev_join, 0));
      FastTcArgs& a = h->tc;
      a.g = g;
      a.q = P.q;
      a.part = h->fpart;
      a.front = h->fast_front;
      a.pos = h->pos_dev;
      a.F = (uint32_t)P.F;
      a.FC = P.FCs;
      a.nfc = P.nfc;
      a.scale_log2 = P.scale_log2;
      a.done_arrive = a.done_epoch = nullptr;
      KTimer t(h, K_FAST, h->s0);
      CU(h, launch_fast_tc(a, h->s0, 1));
      return TTKV_OK;
    }
    // Forked at the step start, s1 already waits for this point of s0 (the
    // append's ev_start): no second fork, and the fast tier chains behind the
    // append on s1 (its CTAs get resident while the append runs; chained-fork
    // env TTKV_FAST_CHAIN=0 is the control).
    static const bool chain_env = [] {
      const char* e = std::getenv("TTKV_FAST_CHAIN");
      return !(e && e[0] == '0');
    }();
    const bool chain_s1 = P.early_fork && chain_env;
    if (!chain_s1) {
      CU(h, cudaEventRecord(h->ev_fork, h->s0));
      CU(h, cudaStreamWaitEvent(h->s1, h->ev_fork, 0));
    }
    if (h->fast_tc) {
      FastTcArgs& a = h->tc;
      a.g = g;
      a.q = P.q;
      a.part = h->fpart;
      a.front = h->fast_front;
      a.pos = h->pos_dev;
      a.F = (uint32_t)P.F;
      a.FC = P.FCs;
      a.nfc = P.nfc;
      a.scale_log2 = P.scale_log2;
      a.done_arrive = P.dev_join ? h->join : nullptr;
      a.done_epoch = P.dev_join ? h->join + 1 : nullptr;
      {
        KTimer t(h, K_FAST, h->s1);
        CU(h, launch_fast_tc(a, h->s1, chain_s1 ? 2 : 0));
      }
      CU(h, cudaEventRecord(h->ev_join, h->s1));
      return TTKV_OK;
    }
    FastArgs a{};
    a.g = g;
    a.ring_k = h->ring_k;
    a.ring_v = h->ring_v;
    a.q = P.q;
    a.part = h->fpart;
    a.front = h->fast_front;
    a.pos = h->pos_dev;
    a.F = (uint32_t)P.F;
    a.FC = P.FCs;
    a.nfc = P.nfc;
    a.TT = h->TT;
    a.stages = kFastStages;
    a.scale_log2 = P.scale_log2;
    {
      KTimer t(h, K_FAST, h->s1);
      CU(h, launch_fast(a, h->s1));
    }
    CU(h, cudaEventRecord(h->ev_join, h->s1));
    return TTKV_OK;
  };
  if (P.early_fork) {
    if (int rcf = fork_fast()) return rcf;
  }
  if (P.fused) {
    // score + select + union as one cluster kernel per stream
    FusedSelectArgs a{};
    a.g = g;
    a.q = P.q;
    a.cent = h->cent;
    a.scores = h->scores;
    a.union_ids = h->uids;
    a.union_mask = h->umask;
    a.union_count = h->ucount;
    a.n = (uint32_t)P.n;
    a.k = (uint32_t)P.k;
    a.early_trigger = P.spec ? 1u : 0u;
    KTimer t(h, K_SELECT, h->s0);
    CU(h, launch_select_fused(a, h->s0));
  } else if (P.slow) {
    {
      ScoreArgs a{g, P.q, h->cent, h->scores, (uint32_t)P.n};
      KTimer t(h, K_SCORE, h->s0);
      CU(h, launch_score(a, h->s0));
    }
    {
      SelectArgs a{};
      a.g = g;
      a.scores = h->scores;
      a.mask = h->mask;
      a.union_ids = h->uids;
      a.union_mask = h->umask;
      a.union_count = h->ucount;
      a.n = (uint32_t)P.n;
      a.k = (uint32_t)P.k;
      KTimer t(h, K_SELECT, h->s0, 2);  // sort + union kernels
      CU(h, launch_select(a, h->s0));
    }
  }
  if (P.slow) {
    if (h->opt.serial_schedule) {
      // bulk phase: every selected record crosses PCIe before any compute
      KTimer t(h, K_GATHER, h->s0);
      CU(h, launch_gather(g, h->arena_dev, h->stage_arena, h->uids, h->ucount,
                          (uint32_t)P.gather_chunks, P.CH, h->s0));
    }
    if (!P.early_fork && !P.fast_last) {
      if (int rcf = fork_fast()) return rcf;
    }
    if (P.fast_first) CU(h, cudaStreamWaitEvent(h->s0, h->ev_join, 0));
    if (P.spec) {
      SlowTcArgs& a = h->stc;
      a.g = g;
      a.params = h->params;
      a.q = P.q;
      a.literal = 0u;
      a.scale_log2 = P.scale_log2;
      a.spec_n = (uint32_t)P.n;
      a.spec_ctr = h->spec_ctr;
      a.rpart = h->rpart;
      KTimer t(h, K_SLOW, h->s0);
      CU(h, launch_slow_tc_spec(a, (uint32_t)P.grid_chunks, h->s0));
    } else if (h->slow_tc) {
      SlowTcArgs& a = h->stc;
      a.g = g;
      a.params = h->params;
      a.union_ids = h->uids;
      a.union_mask = h->umask;
      a.union_count = h->ucount;
      a.q = P.q;
      a.part = h->spart;
      a.nslots = h->nslots;
      a.per_min = P.per_min;
      a.nsc = (uint32_t)h->spart_chunks;
      a.literal = h->opt.literal_additive_merge ? 1u : 0u;
      a.scale_log2 = P.scale_log2;
      KTimer t(h, K_SLOW, h->s0);
      CU(h, launch_slow_tc(a, (uint32_t)P.grid_chunks, h->s0));
    } else {
      SlowArgs a{};
      a.g = g;
      a.arena = h->opt.serial_schedule ? h->stage_arena : h->arena_dev;
      a.params = h->params;
      a.union_ids = h->uids;
      a.union_mask = h->umask;
      a.union_count = h->ucount;
      a.q = P.q;
      a.part = h->spart;
      a.CH = P.CH;
      a.nsc = (uint32_t)h->spart_chunks;
      a.stages = h->stages;
      a.scale_log2 = P.scale_log2;
      a.literal = h->opt.literal_additive_merge ? 1u : 0u;
      KTimer t(h, K_SLOW, h->s0);
      CU(h, launch_slow(a, (uint32_t)P.grid_chunks, (int)h->copy_mode, h->s0));
    }
  } else if (!P.early_fork) {
    if (int rcf = fork_fast()) return rcf;
  }
  if (P.fast_last) {
    if (int rcf = fork_fast()) return rcf;
  } else if (!P.spec && !P.fast_first && !P.dev_join) {
    CU(h, cudaStreamWaitEvent(h->s0, h->ev_join, 0));
  }
  {
    CombineArgs a{};
    a.g = g;
    a.fpart = h->fpart;
    a.nfc = P.nfc;
    a.spart = P.slow ? h->spart : nullptr;
    a.nsc = (uint32_t)h->spart_chunks;
    a.CH = P.CH;
    a.union_count = P.slow ? h->ucount : nullptr;
    a.nslots = P.slow && h->slow_tc ? h->nslots : nullptr;
    if (P.spec) {
      a.spart = nullptr;
      a.nslots = nullptr;
      a.rpart = h->rpart;
      a.union_ids = h->uids;
      a.union_mask = h->umask;
      a.n_cap = g.n_cap;
      a.spec_n = (uint32_t)P.n;
      a.spec_ctr = h->spec_ctr;
    }
    a.out = P.out;  // host-buffer steps: the caller's (or the staging) page-locked buffer
    a.out_ref = P.host_io ? h->out_ref : nullptr;
    if (P.dev_join) {
      a.fast_epoch = h->join + 1;
      a.comb_arrive = h->join + 2;
      a.comb_epoch = h->join + 3;
    }
    a.count_out = P.host_io && P.slow ? h->h_ucount_dev : nullptr;
    a.literal = h->opt.literal_additive_merge ? 1u : 0u;
    a.pos_inc = h->pos_dev;
    if (h->pg.active) {
      // double-buffered by step parity: a rank one step ahead never
      // overwrites rows another rank may still be consuming
      const size_t half = (size_t)((h->pg.epoch + 1) & 1) * h->pg.out_bytes;
      a.n_peers = h->pg.n_ranks;
      a.my_rank = h->pg.my_rank;
      a.gidx = h->pg.gidx;
      for (uint32_t r = 0; r < h->pg.n_ranks; ++r) {
        uint8_t* b = r == h->pg.my_rank ? h->pg.base : static_cast<uint8_t*>(h->pg.peer_base[r]);
        a.peer_out[r] = reinterpret_cast<double*>(b + half);
        a.peer_flags[r] = reinterpret_cast<unsigned long long*>(b + 2 * h->pg.out_bytes);
      }
    }
    KTimer t(h, K_COMBINE, h->s0, h->pg.active ? 2 : 1);
    CU(h, launch_combine(a, h->s0));
    if (h->pg.active) {  // every rank's rows of this step have landed here
      h->pg.epoch += 1;
      CU(h, launch_peer_wait(
                reinterpret_cast<const unsigned long long*>(h->pg.base + 2 * h->pg.out_bytes),
                h->pg.n_ranks, h->pg.epoch * (unsigned long long)g.S * g.G * combine_slices(a),
                h->pg.status,
                h->s0));
    }
  }
  // a graph capture must join s1 back into s0; launched directly, the side
  // stream needs no join (the combine waited for the fast tier on the device,
  // and the append precedes it on s1), and an event wait here would cut the
  // programmatic overlap with the next step's selection
  if (P.dev_join && P.capturing) CU(h, cudaStreamWaitEvent(h->s0, h->ev_join, 0));
  return TTKV_OK;
}

// Graph replay: the host's issue time of a directly launched step is ~13 us
// (cfg1 HBM, 8 launches) against ~2 us for one graph launch, but a replayed
// step loses part of the programmatic-launch overlap of the direct chain
// (cfg1 HBM: 50.9 vs 43.6 us per step back to back on the device).  So the
// synchronous host-buffer call (ttkv_gpu_decode_step), which waits for every
// step anyway, replays by default (cfg1 HBM: 65.6 -> 49.7 us per call,
// tools/host_issue_probe.cu), and device-buffer steps enqueued back to back
// launch directly.  TTKV_GRAPH=1 replays both, TTKV_GRAPH=0 neither.
bool graphs_enabled(bool host_io) {
  static const int env = [] {
    const char* e = std::getenv("TTKV_GRAPH");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return env == 1 || (env == -1 && host_io);
}

int decode_core(ttkv_gpu* h, const float* q, const void* kn, const void* vn, int dtype,
                double* out, ttkv_step_report* rep, bool host_io = false) {
  StepTimer step_timer(h);
  {  // grow before selecting so a settle-time eviction never reallocates
    int rc0 = ensure_blocks(h, h->n_slow + 1);
    if (rc0) return rc0;
  }
  const Geometry& g = h->g;
  const uint64_t pos = h->appended;
  if (pos - h->fast_front + 1 > g.C)
    return set_err(h, TTKV_EERROR,
                   "decode_step: fast tier would exceed its ring; settle pending evictions");
  StepPlan P{};
  P.q = q;
  P.kn = kn;
  P.vn = vn;
  P.dtype = dtype;
  P.out = out;
  P.host_io = host_io;
  P.F = pos + 1 - h->fast_front;
  P.n = h->n_slow;
  {
    std::string m;
    int rc = resolve_k(h->pol, P.n, P.k, m);
    if (rc) return set_err(h, rc, m);
  }
  // softmax scale 1/sqrt(d_k) (engine.cpp:30), folded with log2(e) for exp2
  P.scale_log2 = 1.0 / std::sqrt((double)g.d_k) * 1.4426950408889634;
  P.slow = P.n > 0 && P.k > 0;

  // Fast tier on s1 (low priority), overlapped with the PCIe-bound slow
  // stream on s0.  It is forked after select so it never competes with the
  // critical path append -> score -> select for SM slots.
  // With slow work in the step the fast tier runs hidden under it, so it is
  // cut into at most ~16 chunks per stream: fewer partial rows for the
  // combine, which is on the critical path (small S only; large S already
  // has long chunks).  Its grid then covers the whole ring (the kernels read
  // the fast-tier length from the device step position; chunks past it are
  // empty partials), so the launch is the same for every step of an
  // eviction period.  Without slow work it keeps the GPU-filling split.
  P.FCs = h->FC;
  if (P.slow) {
    const uint64_t want = ((h->l_fast + g.B + 15) / 16 + h->TT - 1) / h->TT * h->TT;
    P.FCs = (uint32_t)std::max<uint64_t>(P.FCs, want);
    P.nfc = (uint32_t)((g.C + P.FCs - 1) / P.FCs);
  } else {
    P.nfc = (uint32_t)((P.F + P.FCs - 1) / P.FCs);
  }

  // The fast tier (low priority, s1) is forked after select: score and
  // select are short, latency-bound kernels that should not wait for SM slots
  // held by long fast-tier CTAs, and the PCIe stream (host tier) or the record
  // stream (HBM tier) is the critical path after them (HBM cfg2: 1.289 ms/step
  // forked late vs 1.338 forked at the step start; cfg3 equal).
  static const int fork_env = [] {  // TTKV_FORK=early|late overrides (measurement)
    const char* e = std::getenv("TTKV_FORK");
    return e ? (std::strcmp(e, "early") == 0 ? 1 : 0) + (std::strcmp(e, "late") == 0 ? 2 : 0) : 0;
  }();
  P.fused = P.slow && select_fused_supported(g, (uint32_t)P.n, (uint32_t)h->sms);
  P.spec = P.fused && want_spec(h, P.n, P.k);
  // A one-wave fused selection leaves most SMs idle: the fast tier then runs
  // beside it instead of starved under the slow kernel (layer-sequential
  // cfg2: fast tier done before the slow kernel starts, 2 us less per layer)
  P.early_fork = !P.spec && (fork_env == 1 || (fork_env != 2 && P.fused));
  static const int order_env = [] {  // TTKV_FAST_ORDER=side|first|last (measurement)
    const char* e = std::getenv("TTKV_FAST_ORDER");
    return !e ? 0 : std::strcmp(e, "first") == 0 ? 1 : std::strcmp(e, "last") == 0 ? 2 : 0;
  }();
  P.fast_first = P.slow && !P.spec && order_env == 1;
  P.fast_last = P.slow && !P.spec && h->fast_tc && order_env == 2;
  if (P.fast_first) P.early_fork = true;
  if (P.fast_last) P.early_fork = false;
  // The combine joins the fast tier on the device instead of through an event
  // wait on s0, which would make it a plain launch after the record kernel's
  // full completion (layer-sequential: ~3.6 us per layer, tools/chain_stamps.py).
  // Only when the fast tier is forked at the step start and the combine grid
  // is at most one CTA per SM, so its waiting CTAs always leave room for the
  // fast tier's; and only when the fast tier's bytes are small against the
  // record stream's (at most a quarter of the union's upper bound), so it is
  // done long before the combine starts.  When it is not (cfg1: 67 MB of ring
  // against ~86 MB of records), the fast tier shares the SMs with the record
  // stream and ends last, and the early combine's waiting CTAs cost more than
  // the launch they save (42.2 vs 39.4 us per step).
  static const int join_env = [] {  // TTKV_DEV_JOIN=0: the event wait, 1: the device join
    const char* e = std::getenv("TTKV_DEV_JOIN");      // whatever the byte ratio (measurement)
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  {
    const double fast_bytes = (double)g.S * (double)P.F * (g.d_k + g.d_v) * g.elem;
    const double slow_ub = (double)g.S * (double)std::min<uint64_t>(P.n, (uint64_t)g.Gs * P.k) *
                           (double)g.rec.used;
    P.dev_join = join_env != 0 && P.slow && h->fast_tc && P.early_fork && !P.spec &&
                 !P.fast_first && !P.fast_last && !h->pg.active &&
                 (uint64_t)g.S * g.G * combine_slices(g) <= (uint64_t)h->sms &&
                 (join_env == 1 || 4.0 * fast_bytes <= slow_ub);
  }
  P.CH = 4;
  if (P.slow) {
    if (h->slow_tc) {
      // HBM records: every CTA pays a prologue and a pipeline fill, so the
      // smallest chunk that fits the union's upper bound S * min(n, Gs * k)
      // into ONE wave of resident CTAs (layer-sequential cfg2, S = 8: 308 ->
      // 379 tok/s vs 4-record chunks; a second partial wave costs ~15 %)
      const uint64_t ub = (uint64_t)g.S * std::min<uint64_t>(P.n, (uint64_t)g.Gs * P.k);
      const uint64_t slots = (uint64_t)h->sms * slow_tc_ctas_per_sm(g);
      P.CH = (uint32_t)std::min<uint64_t>(64, std::max<uint64_t>(4, (ub + slots - 1) / slots));
    } else {
      // host records: union entries per CTA ~4 waves of 2 CTAs/SM over the
      // lower bound S * k (more zero-copy streams in flight)
      const uint64_t est = (uint64_t)g.S * P.k;
      P.CH = (uint32_t)std::min<uint64_t>(64, std::max<uint64_t>(4, (est + 1183) / 1184));
    }
    static const uint32_t ch_env = [] {  // TTKV_SLOW_CH=n overrides (measurement)
      const char* e = std::getenv("TTKV_SLOW_CH");
      return e ? (uint32_t)std::max(1, std::min(256, std::atoi(e))) : 0u;
    }();
    if (ch_env) P.CH = ch_env;
    P.grid_chunks = P.gather_chunks = (P.n + P.CH - 1) / P.CH;
    uint64_t nsc = P.grid_chunks;
    if (h->slow_tc) {
      // balanced schedule over one wave of CTAs; a stream's records span at
      // most nsc CTAs when every CTA takes >= n / (nsc - 1) records, so nsc
      // is as large as ~32 MB of partials allows (small S: every CTA a share)
      const uint64_t ctas = (uint64_t)h->sms * slow_tc_ctas_per_sm(g);
      const uint64_t row = (uint64_t)g.S * g.G * (g.d_v + 2) * h->acc;
      nsc = std::min<uint64_t>(ctas + 1, std::max<uint64_t>(P.grid_chunks + 1, (32ull << 20) / row));
      nsc = std::max<uint64_t>(nsc, 2);
      P.grid_chunks = ctas;
    }
    int rc = ensure_spart(h, nsc);
    if (rc) return rc;
    if (h->slow_tc)  // spart_chunks >= 2 here
      P.per_min = (uint32_t)((P.n + h->spart_chunks - 2) / (h->spart_chunks - 1));
    if (P.spec) {  // one wave of resident CTAs fed from the record queue
      rc = ensure_rpart(h);
      if (rc) return rc;
      static const uint32_t cps_env = [] {  // TTKV_SPEC_CPS=n: CTAs per SM (measurement)
        const char* e = std::getenv("TTKV_SPEC_CPS");
        return e ? (uint32_t)std::max(1, std::min(3, std::atoi(e))) : 0u;
      }();
      const uint32_t cps = cps_env ? cps_env : slow_tc_ctas_per_sm(g);
      P.grid_chunks = (uint64_t)h->sms * cps;
    }
  }
  if (!h->pos_synced) {  // host-side appends / prefill / restore moved `appended`
    CU(h, launch_set_u64(h->pos_dev, pos, h->s0));
    h->pos_synced = true;
  }

  // CUDA graph: within an eviction period every launch of the step is the
  // same (n, k, the grids and all pointers are fixed; the step position lives
  // on the device), so the step is captured once and replayed.  Steps that
  // evict, timed steps and the multi-GPU gather launch directly.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  bool use_graph = graphs_enabled(host_io) && P.slow && !h->timing && !h->pg.active && h->s0 &&
                   P.F <= h->l_fast;
  if (use_graph) {
    CU(h, cudaStreamIsCapturing(h->s0, &cap));
    use_graph = cap == cudaStreamCaptureStatusNone;  // a caller's capture takes the launches
  }
  if (use_graph) {
    ttkv_gpu::GraphKey key;
    std::memset(&key, 0, sizeof(key));
    key.q = q;
    key.kn = kn;
    key.vn = vn;
    key.out = out;
    key.s0 = h->s0;
    key.n = P.n;
    key.k = P.k;
    key.front = h->fast_front;
    key.gen = h->gen;
    key.grid_chunks = P.grid_chunks;
    key.nfc = P.nfc;
    key.CH = P.CH;
    key.dtype = (uint32_t)dtype;
    key.host_io = host_io ? 1u : 0u;  // host addresses live in h->io, not in the graph
    ttkv_gpu::StepGraph* hit = nullptr;
    for (auto& sg : h->graphs)
      if (std::memcmp(&key, &sg.key, sizeof(key)) == 0) hit = &sg;
    const uint64_t now = h->graph_replays + h->graph_captures;
    if (hit) {
      CU(h, cudaGraphLaunch(hit->exec, h->s0));
      h->launches += hit->launches;
      hit->last_use = now;
      h->graph_replays++;
    } else {
      // graphs of another eviction period / buffer generation never match
      // again; beyond kMaxGraphs buffer sets the least recently used goes
      for (size_t i = 0; i < h->graphs.size();) {
        const auto& k2 = h->graphs[i].key;
        if (k2.n != key.n || k2.front != key.front || k2.gen != key.gen || k2.s0 != key.s0) {
          cudaGraphExecDestroy(h->graphs[i].exec);
          h->graphs.erase(h->graphs.begin() + i);
        } else {
          ++i;
        }
      }
      if (h->graphs.size() >= ttkv_gpu::kMaxGraphs) {
        size_t victim = 0;
        for (size_t j = 1; j < h->graphs.size(); ++j)
          if (h->graphs[j].last_use < h->graphs[victim].last_use) victim = j;
        cudaGraphExecDestroy(h->graphs[victim].exec);
        h->graphs.erase(h->graphs.begin() + victim);
      }
      const uint64_t l0 = h->launches;
      CU(h, cudaStreamBeginCapture(h->s0, cudaStreamCaptureModeRelaxed));
      P.capturing = true;
      const int rc = enqueue_step(h, P);
      P.capturing = false;
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(h->s0, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      CU(h, ce);
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      CU(h, ie);
      h->graphs.push_back({key, exec, h->launches - l0, now});
      h->graph_captures++;
      CU(h, cudaGraphLaunch(exec, h->s0));
    }
  } else {
    int rc = enqueue_step(h, P);
    if (rc) {
      // a step cut short may have launched the fast tier without its combine:
      // drain both streams and restart the join epochs in step
      if (P.dev_join) {
        cudaStreamSynchronize(h->s1);
        cudaStreamSynchronize(h->s0);
        cudaMemset(h->join, 0, 4 * sizeof(uint32_t));
      }
      return rc;
    }
  }
  h->appended = pos + 1;
  if (P.spec) h->spec_steps++;
  h->last_k = P.slow ? P.k : 0;
  h->last_n = P.n;
  bool evicted = false;
  int rc = settle_evictions(h, &evicted);
  if (rc) return rc;
  if (rep) {
    rep->blocks_scored = P.n;
    rep->blocks_fetched = P.k;
    rep->bytes_transferred = (double)P.k * (double)modeled_block_bytes_cfg(h->cfg);
    rep->fast_tokens = P.F;
    rep->eviction_occurred = evicted ? 1 : 0;
    rep->union_blocks = 0;
    rep->pcie_bytes = 0;
  }
  return TTKV_OK;
}

}  // namespace

extern "C" {

int ttkv_abi_version(void) { return TTKV_ABI_VERSION; }
const char* ttkv_last_error(void) { return g_last_error.c_str(); }
const char* ttkv_gpu_last_error(const ttkv_gpu* h) {
  return h ? h->err.c_str() : g_last_error.c_str();
}

int ttkv_device_count(int* n) {
  if (!n) return set_err(nullptr, TTKV_EINVAL, "null pointer");
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    return set_err(nullptr, TTKV_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  return TTKV_OK;
}

void ttkv_default_config(ttkv_tier_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->hbm_budget_bytes = 0;
  c->d_k = 64;
  c->d_v = 64;
  c->bytes_full_precision = 2;
  c->block_size = 128;
  c->key_bits = 8;
  c->value_bits = 4;
  c->fetch_fraction = 0.45;
  c->has_top_k_blocks = 0;
  c->top_k_blocks = 0;
  c->hbm_bandwidth = 2.0e12;
  c->pcie_bandwidth = 3.2e10;
  c->transfer_latency = 1.0e-5;
  c->compute_rate = 4.0e11;
}

int ttkv_validate_config(const ttkv_tier_config* c) {
  if (!c) return set_err(nullptr, TTKV_EINVAL, "null config");
  std::string m;
  int rc = validate(*c, m);
  if (rc) set_err(nullptr, rc, m);
  return rc;
}

uint64_t ttkv_fast_capacity(const ttkv_tier_config* c) {
  if (!c) return 0;
  uint64_t out = 0;
  std::string m;
  if (fast_capacity_of(*c, out, m)) {
    set_err(nullptr, TTKV_ECONFIG, m);
    return 0;
  }
  return out;
}

uint64_t ttkv_modeled_block_bytes(const ttkv_tier_config* c) {
  return c ? modeled_block_bytes_cfg(*c) : 0;
}
uint64_t ttkv_packed_bytes(uint64_t count, uint32_t bits) { return packed_bytes_u(count, bits); }

uint64_t ttkv_resolve(const ttkv_selection_policy* p, uint64_t n) {
  if (!p) return UINT64_MAX;
  uint64_t k = 0;
  std::string m;
  if (resolve_k(*p, n, k, m)) {
    set_err(nullptr, TTKV_ECONFIG, m);
    return UINT64_MAX;
  }
  return k;
}

int ttkv_gpu_create(const ttkv_tier_config* cfg, const ttkv_selection_policy* pol,
                    const ttkv_gpu_options* opt, ttkv_gpu** out) {
  if (!cfg || !pol || !opt || !out) return set_err(nullptr, TTKV_EINVAL, "null argument");
  *out = nullptr;
  std::string m;
  uint64_t l_fast = 0;
  int rc = fast_capacity_of(*cfg, l_fast, m);
  if (rc) return set_err(nullptr, rc, m);
  if (!pol->has_top_k && !(pol->fetch_fraction > 0.0 && pol->fetch_fraction <= 1.0))
    return set_err(nullptr, TTKV_ECONFIG, "fetch_fraction must be in (0, 1]");
  // B200 engine limits (documented in DESIGN.md)
  if (cfg->d_k > (uint64_t)kMaxD || cfg->d_v > (uint64_t)kMaxD)
    return set_err(nullptr, TTKV_ECONFIG, "GPU engine supports d_k, d_v <= 128");
  if (opt->ring_bytes != 0 && opt->ring_bytes != 2 && opt->ring_bytes != 4)
    return set_err(nullptr, TTKV_ECONFIG, "ring_bytes must be 0 (auto), 2 (fp16) or 4 (fp32)");
  if (cfg->block_size > 512)
    return set_err(nullptr, TTKV_ECONFIG, "GPU engine supports block_size <= 512");
  if (opt->n_streams == 0 || opt->heads_per_stream == 0 || opt->heads_per_stream > (uint32_t)kMaxG)
    return set_err(nullptr, TTKV_ECONFIG, "n_streams >= 1 and heads_per_stream in [1, 8]");
  if (opt->record_stream > 2)
    return set_err(nullptr, TTKV_ECONFIG, "record_stream must be 0 or 1 (union, the default) or 2 (speculative)");

  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return set_err(nullptr, TTKV_ECUDA,
                   std::string("no CUDA device: ") + (ce != cudaSuccess ? cudaGetErrorString(ce) : "0 devices"));
  if (opt->device < 0 || opt->device >= ndev)
    return set_err(nullptr, TTKV_ECUDA, "device ordinal out of range");

  ttkv_gpu* h = new ttkv_gpu();
  h->cfg = *cfg;
  h->pol = *pol;
  h->opt = *opt;
  h->dev = opt->device;
  cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev);
  h->l_fast = l_fast;
  Geometry& g = h->g;
  g.S = opt->n_streams;
  g.G = opt->heads_per_stream;
  g.Gs = opt->group_select ? 1 : g.G;
  g.d_k = (uint32_t)cfg->d_k;
  g.d_v = (uint32_t)cfg->d_v;
  g.B = (uint32_t)cfg->block_size;
  g.kb = cfg->key_bits;
  g.vb = cfg->value_bits;
  // fast-tier storage: explicit, else fp16 when the config accounts <= 2 B/elem
  g.elem = opt->ring_bytes ? opt->ring_bytes : (cfg->bytes_full_precision <= 2 ? 2u : 4u);
  g.C = l_fast + g.B;
  g.n_cap = 0;
  g.rec = make_layout(g.B, g.d_k, g.d_v, g.kb, g.vb, g.elem);
  if (evict_smem_bytes(g) > 220 * 1024) {
    delete h;
    return set_err(nullptr, TTKV_ECONFIG, "block too large for the GPU quantizer");
  }
  h->stages = slow_stages_for(g);
  if (h->stages == 0) {
    delete h;
    return set_err(nullptr, TTKV_ECONFIG, "slow-tier record too large to stage in shared memory");
  }
  h->copy_mode = opt->copy_mode ? opt->copy_mode : 1;
  if (const char* env = std::getenv("TTKV_COPY_MODE")) {
    if (!std::strcmp(env, "ldg")) h->copy_mode = 2;
    if (!std::strcmp(env, "bulk")) h->copy_mode = 1;
  }
  // fast split: chunks of whole TT-token tiles, ~4 waves of 2 CTAs per SM
  h->acc = g.elem == 4 ? 8 : 4;
  {
    const char* tc_env = std::getenv("TTKV_FAST_TC");
    h->fast_tc = fast_tc_supported(g) && !(tc_env && tc_env[0] == '0') &&
                 (uint64_t)g.S * g.C < (1ull << 31);  // int32 TMA row coordinates
    // tensor-core slow tier: HBM-resident records (the CUDA-core consumer has
    // 3x headroom over the PCIe link); TTKV_SLOW_TC=1/0 forces it on/off
    const char* stc_env = std::getenv("TTKV_SLOW_TC");
    h->slow_tc = slow_tc_supported(g) &&
                 (stc_env ? stc_env[0] == '1' : opt->slow_tier == TTKV_SLOW_DEVICE);
    h->TT = h->fast_tc ? fast_tc_tile() : fast_tile_rows(g);
    const uint64_t Fmax = l_fast + g.B;  // ring capacity bounds the fast tier
    const uint64_t target = std::max<uint64_t>(1, (148ull * 2 * 4 + g.S - 1) / g.S);
    uint64_t FC = (Fmax + target - 1) / target;
    FC = std::max<uint64_t>(h->TT, (FC + h->TT - 1) / h->TT * h->TT);
    h->FC = (uint32_t)FC;
    h->nfc_cap = (uint32_t)((Fmax + FC - 1) / FC);
  }

#define CREATE_CU(call)                                                                      \
  do {                                                                                       \
    cudaError_t e__ = (call);                                                                \
    if (e__ != cudaSuccess) {                                                                \
      std::string msg__ = std::string(#call) + ": " + cudaGetErrorString(e__);               \
      free_all(h);                                                                           \
      delete h;                                                                              \
      return set_err(nullptr, TTKV_ECUDA, msg__);                                            \
    }                                                                                        \
  } while (0)

  CREATE_CU(cudaSetDevice(h->dev));
  {  // s0 carries the critical path (high priority), s1 the overlapped fast tier
    int lo = 0, hi = 0;
    CREATE_CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CREATE_CU(cudaStreamCreateWithPriority(&h->s0, cudaStreamNonBlocking, hi));
    CREATE_CU(cudaStreamCreateWithPriority(&h->s1, cudaStreamNonBlocking, lo));
  }
  CREATE_CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CREATE_CU(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
  CREATE_CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  const size_t S = g.S;
  CREATE_CU(cudaMalloc(&h->ring_k, S * g.C * g.d_k * g.elem));
  CREATE_CU(cudaMalloc(&h->ring_v, S * g.C * g.d_v * g.elem));
  CREATE_CU(cudaMemset(h->ring_k, 0, S * g.C * g.d_k * g.elem));
  CREATE_CU(cudaMemset(h->ring_v, 0, S * g.C * g.d_v * g.elem));
  if (h->fast_tc && make_ring_tmaps(g, h->ring_k, h->ring_v, h->tc) != cudaSuccess) {
    // tensor-map encoding unavailable: keep the CUDA-core fast tier (64-token tiles)
    h->fast_tc = false;
  }
  CREATE_CU(cudaMalloc((void**)&h->pos_dev, sizeof(uint64_t)));
  CREATE_CU(cudaMemset(h->pos_dev, 0, sizeof(uint64_t)));
  h->pos_synced = true;
  CREATE_CU(cudaMalloc((void**)&h->ucount, S * sizeof(uint32_t)));
  CREATE_CU(cudaMalloc((void**)&h->nslots, S * sizeof(uint32_t)));
  CREATE_CU(cudaMemset(h->ucount, 0, S * sizeof(uint32_t)));
  CREATE_CU(pinned_alloc((void**)&h->h_ucount, S * sizeof(uint32_t)));
  CREATE_CU(cudaHostGetDevicePointer((void**)&h->h_ucount_dev, h->h_ucount, 0));
  CREATE_CU(pinned_alloc((void**)&h->io, sizeof(IoSlot)));
  CREATE_CU(cudaHostGetDevicePointer((void**)&h->io_dev, h->io, 0));
  CREATE_CU(cudaMalloc((void**)&h->out_ref, sizeof(double*)));
  CREATE_CU(cudaMalloc((void**)&h->join, 4 * sizeof(uint32_t)));
  CREATE_CU(cudaMemset(h->join, 0, 4 * sizeof(uint32_t)));
  CREATE_CU(cudaMalloc((void**)&h->fpart, S * g.G * h->nfc_cap * (g.d_v + 2) * h->acc));
  CREATE_CU(cudaMalloc((void**)&h->q_dev, S * g.G * g.d_k * sizeof(float)));
  CREATE_CU(cudaMalloc(&h->kn_dev, S * g.d_k * 4));
  CREATE_CU(cudaMalloc(&h->vn_dev, S * g.d_v * 4));
  CREATE_CU(pinned_alloc((void**)&h->h_q, S * g.G * g.d_k * sizeof(float)));
  CREATE_CU(pinned_alloc((void**)&h->h_out, S * g.G * g.d_v * sizeof(double)));
  CREATE_CU(pinned_alloc(&h->h_k, S * g.d_k * 4));
  CREATE_CU(pinned_alloc(&h->h_v, S * g.d_v * 4));
  const uint64_t reserve_blocks =
      std::max<uint64_t>(16, (opt->reserve_tokens + g.B - 1) / g.B + 2);
  rc = ensure_blocks(h, std::min<uint64_t>(reserve_blocks, select_max_blocks()));
  if (rc) {
    std::string msg = h->err;
    free_all(h);
    delete h;
    return set_err(nullptr, rc, msg);
  }
#undef CREATE_CU
  *out = h;
  return TTKV_OK;
}

void ttkv_gpu_destroy(ttkv_gpu* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->s0) cudaStreamSynchronize(h->s0);
  if (h->s1) cudaStreamSynchronize(h->s1);
  free_all(h);
  delete h;
}

int ttkv_gpu_set_stream(ttkv_gpu* h, void* stream) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  if (h->own_s0) cudaStreamDestroy(h->s0);
  if (stream) {
    h->s0 = static_cast<cudaStream_t>(stream);
    h->own_s0 = false;
  } else {
    CU(h, cudaStreamCreateWithFlags(&h->s0, cudaStreamNonBlocking));
    h->own_s0 = true;
  }
  h->gen++;
  return TTKV_OK;
}

void* ttkv_gpu_get_stream(ttkv_gpu* h) { return h ? (void*)h->s0 : nullptr; }

int ttkv_gpu_synchronize(ttkv_gpu* h) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  CU(h, cudaStreamSynchronize(h->s1));
  return TTKV_OK;
}

int ttkv_gpu_prefill(ttkv_gpu* h, const void* keys, const void* values, uint64_t n, int dtype) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (n == 0) return TTKV_OK;
  if (!keys || !values) return set_err(h, TTKV_EINVAL, "null key/value pointer");
  if (dtype != TTKV_DTYPE_F32 && dtype != TTKV_DTYPE_F16)
    return set_err(h, TTKV_ESHAPE, "prefill: unknown dtype");
  CU(h, cudaSetDevice(h->dev));
  const uint64_t P = std::min<uint64_t>(prefill_chunk_tokens(h), n);
  int rc = ensure_staging(h, P);
  if (rc) return rc;
  const size_t esz = dtype == TTKV_DTYPE_F16 ? 2 : 4;
  const Geometry& g = h->g;
  for (uint64_t t0 = 0; t0 < n; t0 += P) {
    const uint64_t m = std::min<uint64_t>(P, n - t0);
    // [S][n][d] host -> [S][m][d] device, one 2D copy per tensor
    CU(h, cudaMemcpy2DAsync(h->stg_k, m * g.d_k * esz,
                            static_cast<const uint8_t*>(keys) + t0 * g.d_k * esz, n * g.d_k * esz,
                            m * g.d_k * esz, g.S, cudaMemcpyHostToDevice, h->s0));
    CU(h, cudaMemcpy2DAsync(h->stg_v, m * g.d_v * esz,
                            static_cast<const uint8_t*>(values) + t0 * g.d_v * esz,
                            n * g.d_v * esz, m * g.d_v * esz, g.S, cudaMemcpyHostToDevice, h->s0));
    rc = prefill_chunk(h, h->stg_k, h->stg_v, dtype == TTKV_DTYPE_F16 ? kInF16 : kInF32, m);
    if (rc) return rc;
  }
  CU(h, cudaStreamSynchronize(h->s0));
  return TTKV_OK;
}

// Engine::prefill from device memory (the model's prefill leaves K/V on the
// GPU): keys/values [S][n][d] of the ring or f32 type, read in place -- no
// staging copy; records are quantized straight from the caller's rows.
// Enqueued on the handle's stream; returns after it completes.
int ttkv_gpu_prefill_device(ttkv_gpu* h, const void* keys, const void* values, uint64_t n,
                            int dtype) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (n == 0) return TTKV_OK;
  if (!keys || !values) return set_err(h, TTKV_EINVAL, "null key/value pointer");
  if (dtype != TTKV_DTYPE_F32 && dtype != TTKV_DTYPE_F16)
    return set_err(h, TTKV_ESHAPE, "prefill: unknown dtype");
  CU(h, cudaSetDevice(h->dev));
  const int in_dt = dtype == TTKV_DTYPE_F16 ? kInF16 : kInF32;
  // one chunk of the caller's tokens at a time keeps each launch's grid and
  // the ring tail bounded; rows are addressed with the caller's stride n
  const uint64_t P = std::max<uint64_t>(prefill_chunk_tokens(h), h->g.B);
  const size_t esz = dtype == TTKV_DTYPE_F16 ? 2 : 4;
  for (uint64_t t0 = 0; t0 < n; t0 += P) {
    const uint64_t m = std::min<uint64_t>(P, n - t0);
    int rc = prefill_chunk(h, static_cast<const uint8_t*>(keys) + t0 * h->g.d_k * esz,
                           static_cast<const uint8_t*>(values) + t0 * h->g.d_v * esz, in_dt, m,
                           n);
    if (rc) return rc;
  }
  CU(h, cudaStreamSynchronize(h->s0));
  return TTKV_OK;
}

int ttkv_gpu_prefill_synthetic(ttkv_gpu* h, uint64_t n, uint64_t seed) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  CU(h, cudaSetDevice(h->dev));
  const uint64_t P = std::min<uint64_t>(prefill_chunk_tokens(h), std::max<uint64_t>(n, 1));
  int rc = ensure_staging(h, P);
  if (rc) return rc;
  const int in_dt = h->g.elem == 2 ? kInF16 : kInF32;
  for (uint64_t t0 = 0; t0 < n; t0 += P) {
    const uint64_t m = std::min<uint64_t>(P, n - t0);
    CU(h, launch_synth(h->g, h->stg_k, h->stg_v, m, h->appended, seed, h->s0));
    rc = prefill_chunk(h, h->stg_k, h->stg_v, in_dt, m);
    if (rc) return rc;
  }
  CU(h, cudaStreamSynchronize(h->s0));
  return TTKV_OK;
}

int ttkv_gpu_append(ttkv_gpu* h, const void* keys, const void* values, uint64_t n, int dtype) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (n == 0) return TTKV_OK;
  if (!keys || !values) return set_err(h, TTKV_EINVAL, "null key/value pointer");
  if (dtype != TTKV_DTYPE_F32 && dtype != TTKV_DTYPE_F16)
    return set_err(h, TTKV_ESHAPE, "append_token: unknown dtype");
  const Geometry& g = h->g;
  if (h->appended - h->fast_front + n > g.C)
    return set_err(h, TTKV_EERROR,
                   "append_token: fast tier would exceed its ring (L_fast + block_size); "
                   "settle pending evictions first");
  CU(h, cudaSetDevice(h->dev));
  int rc = ensure_staging(h, n);
  if (rc) return rc;
  const size_t esz = dtype == TTKV_DTYPE_F16 ? 2 : 4;
  CU(h, cudaMemcpyAsync(h->stg_k, keys, (size_t)g.S * n * g.d_k * esz, cudaMemcpyHostToDevice,
                        h->s0));
  CU(h, cudaMemcpyAsync(h->stg_v, values, (size_t)g.S * n * g.d_v * esz, cudaMemcpyHostToDevice,
                        h->s0));
  {
    KTimer t(h, K_APPEND, h->s0);
    CU(h, launch_append(g, h->ring_k, h->ring_v, h->stg_k, h->stg_v,
                        dtype == TTKV_DTYPE_F16 ? kInF16 : kInF32, h->appended, n, n, h->s0));
  }
  h->appended += n;
  h->pos_synced = false;
  CU(h, cudaStreamSynchronize(h->s0));
  return TTKV_OK;
}

int ttkv_gpu_eviction_pending(ttkv_gpu* h, int* pending) {
  if (!h || !pending) return set_err(h, TTKV_EINVAL, "null argument");
  *pending = (h->appended - h->fast_front > h->l_fast) ? 1 : 0;
  return TTKV_OK;
}

int ttkv_gpu_evict(ttkv_gpu* h, uint64_t* block_id) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (h->appended - h->fast_front <= h->l_fast)
    return set_err(h, TTKV_EERROR, "evict_and_compress: no eviction pending");
  CU(h, cudaSetDevice(h->dev));
  int rc = ensure_blocks(h, h->n_slow + 1);
  if (rc) return rc;
  EvictArgs a{};
  a.g = h->g;
  a.ring_k = h->ring_k;
  a.ring_v = h->ring_v;
  a.split_pos = h->appended;
  a.first_block = h->n_slow;
  a.arena = h->arena_dev;
  a.cent = h->cent;
  a.params = h->params;
  {
    KTimer t(h, K_EVICT, h->s0);
    CU(h, launch_evict(a, 1, kInF32, h->s0));
  }
  if (block_id) *block_id = h->n_slow;
  h->n_slow++;
  h->fast_front += h->g.B;
  CU(h, cudaStreamSynchronize(h->s0));
  return TTKV_OK;
}

int ttkv_gpu_decode_step_device(ttkv_gpu* h, const float* q, const void* kn, const void* vn,
                                int dtype, double* out, ttkv_step_report* rep) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (!q || !kn || !vn || !out) return set_err(h, TTKV_EINVAL, "null pointer");
  if (dtype != TTKV_DTYPE_F32 && dtype != TTKV_DTYPE_F16)
    return set_err(h, TTKV_ESHAPE, "decode_step: unknown dtype");
  CU(h, cudaSetDevice(h->dev));
  return decode_core(h, q, kn, vn, dtype == TTKV_DTYPE_F16 ? kInF16 : kInF32, out, rep);
}

namespace {
// The device address of page-locked host memory mapped into the device's
// address space (cudaHostAlloc'd, or registered and mapped), else null.
void* host_mapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}
}  // namespace

int ttkv_gpu_decode_step(ttkv_gpu* h, const float* q, const void* kn, const void* vn, int dtype,
                         double* out, ttkv_step_report* rep) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (!q || !kn || !vn || !out) return set_err(h, TTKV_EINVAL, "null pointer");
  if (dtype != TTKV_DTYPE_F32 && dtype != TTKV_DTYPE_F16)
    return set_err(h, TTKV_ESHAPE, "decode_step: unknown dtype");
  CU(h, cudaSetDevice(h->dev));
  const Geometry& g = h->g;
  const size_t esz = dtype == TTKV_DTYPE_F16 ? 2 : 4;
  const size_t qb = (size_t)g.S * g.G * g.d_k * 4, ob = (size_t)g.S * g.G * g.d_v * 8;
  const size_t kb = (size_t)g.S * g.d_k * esz, vb = (size_t)g.S * g.d_v * esz;
  // The step's kernels read the caller's page-locked buffers and write its
  // output through the device mapping of that memory; pageable buffers go
  // through the handle's mapped staging copies (one host memcpy each way).
  auto src = [&](const void* p, void* stage, size_t nb) -> const void* {
    if (void* d = host_mapped(p)) return d;
    std::memcpy(stage, p, nb);
    return host_mapped(stage);
  };
  IoSlot& io = *h->io;
  io.src[0] = src(q, h->h_q, qb);
  io.src[1] = src(kn, h->h_k, kb);
  io.src[2] = src(vn, h->h_v, vb);
  void* out_map = host_mapped(out);
  const bool out_direct = out_map != nullptr;
  io.out = out_direct ? out_map : host_mapped(h->h_out);
  if (!io.src[0] || !io.src[1] || !io.src[2] || !io.out)
    return set_err(h, TTKV_ECUDA, "decode_step: staging buffers are not mapped");
  // the reads of q/k/v and the write of the output are part of the (captured)
  // step; the previous step is complete (synchronized), so h->io is free
  int rc = decode_core(h, h->q_dev, h->kn_dev, h->vn_dev,
                       dtype == TTKV_DTYPE_F16 ? kInF16 : kInF32, nullptr, rep, true);
  if (rc) return rc;
  CU(h, cudaStreamSynchronize(h->s0));
  if (!out_direct) std::memcpy(out, h->h_out, ob);
  if (rep) {
    uint64_t u = 0;
    if (h->last_k)
      for (uint32_t i = 0; i < g.S; ++i) u += h->h_ucount[i];
    rep->union_blocks = u;
    rep->pcie_bytes = u * (uint64_t)h->g.rec.kp_off;
  }
  return TTKV_OK;
}

// Records streamed by the last step: the sum of the per-stream union sizes
// (read on demand; the hot path keeps no global counter).
int ttkv_gpu_read_step_counters(ttkv_gpu* h, uint64_t* union_blocks, uint64_t* pcie_bytes) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  uint64_t u = 0;
  if (h->last_k) {
    CU(h, cudaSetDevice(h->dev));
    CU(h, cudaMemcpyAsync(h->h_ucount, h->ucount, h->g.S * sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, h->s0));
    CU(h, cudaStreamSynchronize(h->s0));
    for (uint32_t i = 0; i < h->g.S; ++i) u += h->h_ucount[i];
  }
  if (union_blocks) *union_blocks = u;
  if (pcie_bytes) *pcie_bytes = u * (uint64_t)h->g.rec.kp_off;
  return TTKV_OK;
}

int ttkv_gpu_state(ttkv_gpu* h, ttkv_state* st) {
  if (!h || !st) return set_err(h, TTKV_EINVAL, "null argument");
  st->appended = h->appended;
  st->fast_tokens = h->appended - h->fast_front;
  st->slow_blocks = h->n_slow;
  st->l_fast = h->l_fast;
  st->record_bytes = h->g.rec.used;
  st->modeled_block_bytes = modeled_block_bytes_cfg(h->cfg);
  st->n_streams = h->g.S;
  st->heads_per_stream = h->g.G;
  st->block_capacity = h->g.n_cap;
  st->launches = h->launches;
  st->graph_replays = h->graph_replays;
  st->graph_captures = h->graph_captures;
  st->spec_steps = h->spec_steps;
  st->payload_bytes = h->g.rec.kp_off;
  return TTKV_OK;
}

namespace {
// The records the last step's slow kernel streamed for (stream, head): the
// per-stream union (select_union_kernel, ascending block id) filtered by the
// head's bit of the union mask.  Cold path.
int selected_of(ttkv_gpu* h, uint32_t stream, uint32_t head, std::vector<uint32_t>& ids) {
  ids.clear();
  if (h->last_k == 0) return TTKV_OK;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  uint32_t cnt = 0;
  CU(h, cudaMemcpy(&cnt, h->ucount + stream, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (cnt > h->last_n)
    return set_err(h, TTKV_EERROR, "selection: union larger than the slow tier");
  std::vector<uint32_t> u(cnt), m(cnt);
  const uint64_t off = (uint64_t)stream * h->g.n_cap;
  if (cnt) {
    CU(h, cudaMemcpy(u.data(), h->uids + off, cnt * 4ull, cudaMemcpyDeviceToHost));
    CU(h, cudaMemcpy(m.data(), h->umask + off, cnt * 4ull, cudaMemcpyDeviceToHost));
  }
  for (uint32_t i = 0; i < cnt; ++i)
    if (m[i] >> head & 1u) ids.push_back(u[i]);
  return TTKV_OK;
}
}  // namespace

int ttkv_gpu_read_selected(ttkv_gpu* h, uint32_t stream, uint32_t head, uint32_t* out,
                           uint64_t cap, uint64_t* n) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S || head >= h->g.G) return set_err(h, TTKV_ESHAPE, "stream/head out of range");
  std::vector<uint32_t> ids;
  if (int rc = selected_of(h, stream, head, ids)) return rc;
  if (n) *n = ids.size();
  if (out)
    for (uint64_t i = 0; i < ids.size() && i < cap; ++i) out[i] = ids[i];
  return TTKV_OK;
}

int ttkv_gpu_read_union(ttkv_gpu* h, uint32_t stream, uint32_t* ids, uint32_t* head_masks,
                        uint64_t cap, uint64_t* n) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S) return set_err(h, TTKV_ESHAPE, "stream out of range");
  if (n) *n = 0;
  if (h->last_k == 0) return TTKV_OK;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  uint32_t cnt = 0;
  CU(h, cudaMemcpy(&cnt, h->ucount + stream, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (n) *n = cnt;
  const uint64_t off = (uint64_t)stream * h->g.n_cap, m = std::min<uint64_t>(cnt, cap);
  if (ids && m) CU(h, cudaMemcpy(ids, h->uids + off, m * 4, cudaMemcpyDeviceToHost));
  if (head_masks && m) CU(h, cudaMemcpy(head_masks, h->umask + off, m * 4, cudaMemcpyDeviceToHost));
  return TTKV_OK;
}

int ttkv_gpu_read_scores(ttkv_gpu* h, uint32_t stream, uint32_t head, double* out, uint64_t cap,
                         uint64_t* n) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S || head >= h->g.G) return set_err(h, TTKV_ESHAPE, "stream/head out of range");
  const uint64_t n_sc = h->last_k ? h->last_n : 0;  // scoring runs only when a fetch does
  if (n) *n = n_sc;
  if (!out || n_sc == 0) return TTKV_OK;
  const uint32_t hs = h->g.Gs == h->g.G ? head : 0;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  CU(h, cudaMemcpy(out, h->scores + ((uint64_t)stream * h->g.Gs + hs) * h->g.n_cap,
                   std::min(n_sc, cap) * sizeof(double), cudaMemcpyDeviceToHost));
  return TTKV_OK;
}

int ttkv_gpu_read_fetched(ttkv_gpu* h, uint32_t stream, uint32_t head, uint64_t* out,
                          uint64_t cap, uint64_t* n) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S || head >= h->g.G) return set_err(h, TTKV_ESHAPE, "stream/head out of range");
  const uint64_t k = h->last_k;
  if (n) *n = k;
  if (!out || k == 0) return TTKV_OK;
  // fetched_blocks = the set the GPU selected and streamed (the union row of
  // this head), put in select_top_k's order (relevance.cpp:29-43: score desc,
  // then block id desc) by the step's bit-exact fp64 scores.  A strict total
  // order, so sorting the top-k set alone gives the prefix of the
  // reference's stable_sort over all n.
  std::vector<uint32_t> ids;
  if (int rc = selected_of(h, stream, head, ids)) return rc;
  if (ids.size() != k)
    return set_err(h, TTKV_EERROR,
                   "selection: the GPU streamed " + std::to_string(ids.size()) +
                       " blocks for stream " + std::to_string(stream) + " head " +
                       std::to_string(head) + ", expected " + std::to_string(k));
  const uint32_t hs = h->g.Gs == h->g.G ? head : 0;
  std::vector<double> sc(h->last_n);
  CU(h, cudaMemcpy(sc.data(), h->scores + ((uint64_t)stream * h->g.Gs + hs) * h->g.n_cap,
                   h->last_n * sizeof(double), cudaMemcpyDeviceToHost));
  std::sort(ids.begin(), ids.end(), [&](uint32_t x, uint32_t y) {
    if (sc[x] != sc[y]) return sc[x] > sc[y];
    return x > y;
  });
  for (uint64_t i = 0; i < k && i < cap; ++i) out[i] = ids[i];
  return TTKV_OK;
}

static float half_bits_to_float(uint16_t b) {
  const uint32_t sign = (uint32_t)(b >> 15) << 31;
  uint32_t exp = (b >> 10) & 0x1f, man = b & 0x3ff;
  uint32_t f;
  if (exp == 0) {
    if (man == 0) f = sign;
    else {
      exp = 127 - 15 + 1;
      while (!(man & 0x400)) { man <<= 1; exp--; }
      man &= 0x3ff;
      f = sign | (exp << 23) | (man << 13);
    }
  } else if (exp == 31) {
    f = sign | 0x7f800000u | (man << 13);
  } else {
    f = sign | ((exp + 127 - 15) << 23) | (man << 13);
  }
  float out;
  std::memcpy(&out, &f, 4);
  return out;
}

int ttkv_gpu_read_block(ttkv_gpu* h, uint32_t stream, uint64_t blk, uint8_t* packed_k,
                        uint8_t* packed_v, float* key_params, float* value_params,
                        float* centroid, uint64_t* first_position) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S) return set_err(h, TTKV_ESHAPE, "stream out of range");
  if (blk >= h->n_slow)
    return set_err(h, TTKV_EERROR, "BlockIndex: unknown block " + std::to_string(blk));
  const Geometry& g = h->g;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  std::vector<uint8_t> rec(g.rec.stride);
  const uint64_t off = ((uint64_t)stream * g.n_cap + blk) * g.rec.stride;
  if (h->arena_host) std::memcpy(rec.data(), h->arena_host + off, g.rec.stride);
  else CU(h, cudaMemcpy(rec.data(), h->arena_dev + off, g.rec.stride, cudaMemcpyDeviceToHost));
  auto export_payload = [&](const uint8_t* src, uint32_t bits, uint32_t dim, uint8_t* dst) {
    if (!dst) return;
    if (bits != 16) {
      std::memcpy(dst, src, (size_t)((uint64_t(g.B) * dim * bits + 7) / 8));
      return;
    }
    float* f = reinterpret_cast<float*>(dst);
    const size_t cnt = (size_t)g.B * dim;
    if (g.elem == 4) std::memcpy(f, src, cnt * 4);
    else
      for (size_t i = 0; i < cnt; ++i) {
        uint16_t b;
        std::memcpy(&b, src + 2 * i, 2);
        f[i] = half_bits_to_float(b);
      }
  };
  export_payload(rec.data(), g.kb, g.d_k, packed_k);
  export_payload(rec.data() + g.rec.v_off, g.vb, g.d_v, packed_v);
  if (key_params && g.kb != 16) std::memcpy(key_params, rec.data() + g.rec.kp_off, 8 * g.d_k);
  if (value_params && g.vb != 16) std::memcpy(value_params, rec.data() + g.rec.vp_off, 8 * g.d_v);
  if (centroid)
    CU(h, cudaMemcpy(centroid, h->cent + ((uint64_t)stream * g.n_cap + blk) * g.d_k,
                     g.d_k * sizeof(float), cudaMemcpyDeviceToHost));
  if (first_position) *first_position = blk * g.B;
  return TTKV_OK;
}

// serialize_block (quantizer.cpp:248-274): versioned little-endian layout.
int ttkv_gpu_serialize_block(ttkv_gpu* h, uint32_t stream, uint64_t blk, uint8_t* out,
                             uint64_t cap, uint64_t* len) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  const Geometry& g = h->g;
  const uint64_t kbytes = packed_bytes_u((uint64_t)g.B * g.d_k, g.kb);
  const uint64_t vbytes = packed_bytes_u((uint64_t)g.B * g.d_v, g.vb);
  const uint64_t nkp = g.kb == 16 ? 0 : g.d_k, nvp = g.vb == 16 ? 0 : g.d_v;
  const uint64_t total = 4 + 2 + 24 + 12 + 4 + 8 * (nkp + nvp) + 4 * g.d_k + 8 + kbytes + 8 + vbytes;
  if (len) *len = total;
  if (!out) return TTKV_OK;
  if (cap < total) return set_err(h, TTKV_ESHAPE, "serialize_block: buffer too small");
  std::vector<uint8_t> pk(kbytes + 1), pv(vbytes + 1);
  std::vector<float> kp(2 * g.d_k), vp(2 * g.d_v), cen(g.d_k);
  uint64_t first = 0;
  int rc = ttkv_gpu_read_block(h, stream, blk, pk.data(), pv.data(), kp.data(), vp.data(),
                               cen.data(), &first);
  if (rc) return rc;
  uint8_t* p = out;
  auto put = [&](uint64_t v, int n) {
    for (int i = 0; i < n; ++i) *p++ = (uint8_t)(v >> (8 * i));
  };
  auto putf = [&](float f) {
    uint32_t v;
    std::memcpy(&v, &f, 4);
    put(v, 4);
  };
  *p++ = 'T'; *p++ = 'T'; *p++ = 'K'; *p++ = 'V';
  put(1, 2);
  put(blk, 8);
  put(first, 8);
  put(first + g.B - 1, 8);
  put(g.B, 4);
  put(g.d_k, 4);
  put(g.d_v, 4);
  put(g.kb, 2);
  put(g.vb, 2);
  for (uint64_t c = 0; c < nkp; ++c) { putf(kp[2 * c]); putf(kp[2 * c + 1]); }
  for (uint64_t c = 0; c < nvp; ++c) { putf(vp[2 * c]); putf(vp[2 * c + 1]); }
  for (uint32_t c = 0; c < g.d_k; ++c) putf(cen[c]);
  put(kbytes, 8);
  std::memcpy(p, pk.data(), kbytes);
  p += kbytes;
  put(vbytes, 8);
  std::memcpy(p, pv.data(), vbytes);
  p += vbytes;
  return TTKV_OK;
}

// dump_slow_tier (quantizer.cpp:325-342): "TTKVTIER", v1, count, then
// length-prefixed serialized blocks.
int ttkv_gpu_dump_slow_tier(ttkv_gpu* h, uint32_t stream, const char* path) {
  if (!h || !path) return set_err(h, TTKV_EINVAL, "null argument");
  FILE* f = std::fopen(path, "wb");
  if (!f) return set_err(h, TTKV_EIO, std::string("cannot open ") + path + " for writing");
  std::vector<uint8_t> hdr = {'T', 'T', 'K', 'V', 'T', 'I', 'E', 'R', 1, 0};
  for (int i = 0; i < 8; ++i) hdr.push_back((uint8_t)(h->n_slow >> (8 * i)));
  bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
  std::vector<uint8_t> buf;
  for (uint64_t b = 0; ok && b < h->n_slow; ++b) {
    uint64_t len = 0;
    ttkv_gpu_serialize_block(h, stream, b, nullptr, 0, &len);
    buf.resize(len);
    int rc = ttkv_gpu_serialize_block(h, stream, b, buf.data(), len, &len);
    if (rc) {
      std::fclose(f);
      return rc;
    }
    uint8_t l8[8];
    for (int i = 0; i < 8; ++i) l8[i] = (uint8_t)(len >> (8 * i));
    ok = std::fwrite(l8, 1, 8, f) == 8 && std::fwrite(buf.data(), 1, len, f) == len;
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return set_err(h, TTKV_EIO, std::string("write failed: ") + path);
  return TTKV_OK;
}

// ---------------------------------------------------------------------------
// Restore (checkpoint/resume).  The reference can load a slow tier
// (load_slow_tier / deserialize_block, quantizer.cpp:276-365) but has no
// TierStore built from one (tier_store.hpp:42); a GPU handle is rebuilt from
// one TTKVTIER file per stream: every record lands in the arena exactly as
// evict_quantize would have written it (payloads, interleaved params), the
// centroid in the resident HBM array.  The fast tier then resumes through
// ttkv_gpu_append.  Integrity checks and messages are the reference's.
// ---------------------------------------------------------------------------
namespace {
struct ByteReader {
  const uint8_t* p;
  size_t n, pos = 0;
  bool ok = true;
  bool need(size_t k) {
    if (pos + k > n) ok = false;
    return ok;
  }
  uint64_t u(int k) {
    if (!need((size_t)k)) return 0;
    uint64_t v = 0;
    for (int i = 0; i < k; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
    pos += (size_t)k;
    return v;
  }
  float f32() {
    const uint32_t v = (uint32_t)u(4);
    float f;
    std::memcpy(&f, &v, 4);
    return f;
  }
  const uint8_t* blob(size_t k) {
    if (!need(k)) return nullptr;
    const uint8_t* b = p + pos;
    pos += k;
    return b;
  }
};

uint16_t float_to_half_bits(float x) {  // round-to-nearest-even (values come from an fp16 ring)
  uint32_t f;
  std::memcpy(&f, &x, 4);
  const uint32_t sign = (f >> 16) & 0x8000u;
  int32_t exp = (int32_t)((f >> 23) & 0xff) - 127 + 15;
  uint32_t man = f & 0x7fffffu;
  if (((f >> 23) & 0xff) == 0xff) return (uint16_t)(sign | 0x7c00u | (man ? 0x200u : 0u));
  if (exp >= 31) return (uint16_t)(sign | 0x7c00u);
  if (exp <= 0) {
    if (exp < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const uint32_t shift = (uint32_t)(14 - exp);
    uint32_t h = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1u))) ++h;
    return (uint16_t)(sign | h);
  }
  uint32_t h = ((uint32_t)exp << 10) | (man >> 13);
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return (uint16_t)(sign | h);
}
}  // namespace

int ttkv_gpu_restore_slow_tier(ttkv_gpu* h, const char* const* paths, uint32_t n_paths) {
  if (!h || !paths) return set_err(h, TTKV_EINVAL, "null argument");
  const Geometry& g = h->g;
  if (n_paths != g.S) return set_err(h, TTKV_ESHAPE, "restore: one slow-tier file per stream");
  if (h->appended != 0)
    return set_err(h, TTKV_ESEQUENCE, "restore: the handle already holds tokens");
  CU(h, cudaSetDevice(h->dev));
  const uint64_t kbytes = packed_bytes_u((uint64_t)g.B * g.d_k, g.kb);
  const uint64_t vbytes = packed_bytes_u((uint64_t)g.B * g.d_v, g.vb);
  const uint64_t pbytes = g.rec.used - g.rec.kp_off;
  uint64_t n_blocks = 0;
  bool wide_scales = false;
  std::vector<uint8_t> rec(g.rec.stride), all;
  std::vector<float> cent(g.d_k);
  for (uint32_t s = 0; s < g.S; ++s) {
    FILE* f = std::fopen(paths[s], "rb");
    if (!f) return set_err(h, TTKV_EIO, std::string("cannot open ") + paths[s]);
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    all.resize(sz > 0 ? (size_t)sz : 0);
    const bool rd = all.empty() || std::fread(all.data(), 1, all.size(), f) == all.size();
    std::fclose(f);
    if (!rd) return set_err(h, TTKV_EIO, std::string("read failed: ") + paths[s]);
    ByteReader r{all.data(), all.size()};
    const uint8_t* magic = r.blob(8);
    if (!magic || std::memcmp(magic, "TTKVTIER", 8) != 0)
      return set_err(h, TTKV_EINTEGRITY, "slow-tier file: bad magic");
    if (r.u(2) != 1) return set_err(h, TTKV_EINTEGRITY, "slow-tier file: unsupported version");
    const uint64_t count = r.u(8);
    if (!r.ok) return set_err(h, TTKV_EINTEGRITY, "deserialize: truncated payload");
    if (s == 0) {
      n_blocks = count;
      int rc = ensure_blocks(h, std::max<uint64_t>(n_blocks, 1));
      if (rc) return rc;
    } else if (count != n_blocks) {
      return set_err(h, TTKV_ESHAPE, "restore: streams hold different slow-tier lengths");
    }
    for (uint64_t b = 0; b < count; ++b) {
      const uint64_t len = r.u(8);
      const uint8_t* blk = r.blob(len);
      if (!r.ok) return set_err(h, TTKV_EINTEGRITY, "deserialize: truncated payload");
      ByteReader q{blk, len};
      const uint8_t* bm = q.blob(4);
      if (!bm || std::memcmp(bm, "TTKV", 4) != 0)
        return set_err(h, TTKV_EINTEGRITY, "deserialize: bad magic");
      if (q.u(2) != 1) return set_err(h, TTKV_EINTEGRITY, "deserialize: unsupported version");
      const uint64_t block_id = q.u(8), first = q.u(8), last = q.u(8);
      const uint32_t tokens = (uint32_t)q.u(4), dk = (uint32_t)q.u(4), dv = (uint32_t)q.u(4);
      const uint32_t kb = (uint32_t)q.u(2), vb = (uint32_t)q.u(2);
      auto valid_bits = [](uint32_t x) { return (x >= 2 && x <= 8) || x == 16; };
      if (!q.ok) return set_err(h, TTKV_EINTEGRITY, "deserialize: truncated payload");
      if (!valid_bits(kb) || !valid_bits(vb))
        return set_err(h, TTKV_EINTEGRITY, "deserialize: bad bit widths");
      if (tokens != g.B || dk != g.d_k || dv != g.d_v || kb != g.kb || vb != g.vb)
        return set_err(h, TTKV_ECONFIG, "restore: block geometry does not match the tier config");
      if (block_id != b || first != b * g.B || last != first + g.B - 1)
        return set_err(h, TTKV_EINTEGRITY, "restore: blocks are not the contiguous sequence 0..n-1");
      std::fill(rec.begin(), rec.end(), 0);
      float* kp = reinterpret_cast<float*>(rec.data() + g.rec.kp_off);
      float* vp = reinterpret_cast<float*>(rec.data() + g.rec.vp_off);
      for (uint32_t c = 0; c < (kb == 16 ? 0u : dk); ++c) { kp[2 * c] = q.f32(); kp[2 * c + 1] = q.f32(); }
      for (uint32_t c = 0; c < (kb == 16 ? 0u : dk); ++c)  // see kTcKeyScaleBound
        if (!(std::fabs(kp[2 * c]) <= kTcKeyScaleBound)) wide_scales = true;
      for (uint32_t c = 0; c < (vb == 16 ? 0u : dv); ++c) { vp[2 * c] = q.f32(); vp[2 * c + 1] = q.f32(); }
      for (uint32_t c = 0; c < dk; ++c) cent[c] = q.f32();
      auto payload = [&](uint64_t want, uint32_t bits, uint32_t dim, uint8_t* dst,
                         const char* what) -> int {
        const uint64_t l = q.u(8);
        if (!q.ok) return set_err(h, TTKV_EINTEGRITY, "deserialize: truncated payload");
        if (l != want)
          return set_err(h, TTKV_EINTEGRITY, std::string("deserialize: ") + what +
                                                 " payload length mismatch");
        const uint8_t* src = q.blob(l);
        if (!src) return set_err(h, TTKV_EINTEGRITY, "deserialize: truncated payload");
        if (bits != 16) {
          std::memcpy(dst, src, l);
        } else {  // lossless payload is float32 in the file, the ring type in the record
          const uint64_t cnt = (uint64_t)g.B * dim;
          for (uint64_t i = 0; i < cnt; ++i) {
            float x;
            std::memcpy(&x, src + 4 * i, 4);
            if (g.elem == 4) {
              std::memcpy(dst + 4 * i, &x, 4);
            } else {
              const uint16_t hb = float_to_half_bits(x);
              std::memcpy(dst + 2 * i, &hb, 2);
            }
          }
        }
        return TTKV_OK;
      };
      const uint64_t kwant = kb == 16 ? (uint64_t)g.B * dk * 4 : kbytes;
      const uint64_t vwant = vb == 16 ? (uint64_t)g.B * dv * 4 : vbytes;
      int rc = payload(kwant, kb, dk, rec.data(), "key");
      if (rc) return rc;
      rc = payload(vwant, vb, dv, rec.data() + g.rec.v_off, "value");
      if (rc) return rc;
      if (q.pos != q.n) return set_err(h, TTKV_EINTEGRITY, "deserialize: trailing bytes");
      const uint64_t idx = (uint64_t)s * g.n_cap + b;
      if (h->arena_host) std::memcpy(h->arena_host + idx * g.rec.stride, rec.data(), g.rec.stride);
      else CU(h, cudaMemcpy(h->arena_dev + idx * g.rec.stride, rec.data(), g.rec.stride,
                            cudaMemcpyHostToDevice));
      if (pbytes)
        CU(h, cudaMemcpy(h->params + idx * pbytes, rec.data() + g.rec.kp_off, pbytes,
                         cudaMemcpyHostToDevice));
      CU(h, cudaMemcpy(h->cent + idx * g.d_k, cent.data(), g.d_k * sizeof(float),
                       cudaMemcpyHostToDevice));
    }
    if (r.pos != r.n) return set_err(h, TTKV_EINTEGRITY, "slow-tier file: trailing bytes");
  }
  h->n_slow = n_blocks;
  h->appended = n_blocks * g.B;
  h->fast_front = n_blocks * g.B;
  h->pos_synced = false;
  h->gen++;
  // key scales no fp16 ring can produce (a dump from an fp32 engine): the
  // tensor-core slow kernel's fp16 operand bound no longer holds
  if (wide_scales) h->slow_tc = false;
  return TTKV_OK;
}

int ttkv_gpu_read_fast(ttkv_gpu* h, uint32_t stream, float* keys, float* values,
                       uint64_t cap, uint64_t* n_tokens, uint64_t* first_position) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (stream >= h->g.S) return set_err(h, TTKV_ESHAPE, "stream out of range");
  const Geometry& g = h->g;
  const uint64_t F = h->appended - h->fast_front;
  if (n_tokens) *n_tokens = F;
  if (first_position) *first_position = h->fast_front;
  if (!keys && !values) return TTKV_OK;
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  std::vector<uint8_t> rk(g.C * g.d_k * g.elem), rv(g.C * g.d_v * g.elem);
  CU(h, cudaMemcpy(rk.data(), (uint8_t*)h->ring_k + (uint64_t)stream * g.C * g.d_k * g.elem,
                   rk.size(), cudaMemcpyDeviceToHost));
  CU(h, cudaMemcpy(rv.data(), (uint8_t*)h->ring_v + (uint64_t)stream * g.C * g.d_v * g.elem,
                   rv.size(), cudaMemcpyDeviceToHost));
  auto elem = [&](const std::vector<uint8_t>& r, uint64_t idx) -> float {
    if (g.elem == 4) {
      float f;
      std::memcpy(&f, r.data() + 4 * idx, 4);
      return f;
    }
    uint16_t b;
    std::memcpy(&b, r.data() + 2 * idx, 2);
    return half_bits_to_float(b);
  };
  for (uint64_t t = 0; t < F && t < cap; ++t) {
    const uint64_t slot = (h->fast_front + t) % g.C;
    for (uint32_t c = 0; c < g.d_k && keys; ++c) keys[t * g.d_k + c] = elem(rk, slot * g.d_k + c);
    for (uint32_t c = 0; c < g.d_v && values; ++c) values[t * g.d_v + c] = elem(rv, slot * g.d_v + c);
  }
  return TTKV_OK;
}

// TierStore::locate (tier_store.cpp:100-105)
int ttkv_gpu_locate(ttkv_gpu* h, uint64_t p, int* where, uint64_t* block_id) {
  if (!h || !where) return set_err(h, TTKV_EINVAL, "null argument");
  if (block_id) *block_id = 0;
  if (p >= h->appended) { *where = 2; return TTKV_OK; }
  if (h->appended > h->fast_front && p >= h->fast_front) { *where = 0; return TTKV_OK; }
  if (p < h->n_slow * h->g.B) {
    *where = 1;
    if (block_id) *block_id = p / h->g.B;
    return TTKV_OK;
  }
  *where = 2;
  return TTKV_OK;
}

int ttkv_gpu_set_timing(ttkv_gpu* h, int enabled) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  h->timing = enabled != 0;
  return TTKV_OK;
}

int ttkv_gpu_kernel_times(ttkv_gpu* h, ttkv_kernel_times* t, int reset) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  CU(h, cudaSetDevice(h->dev));
  drain_timing(h);
  if (t) {
    t->ms_append = h->ms[K_APPEND]; t->n_append = h->cnt[K_APPEND];
    t->ms_score = h->ms[K_SCORE]; t->n_score = h->cnt[K_SCORE];
    t->ms_select = h->ms[K_SELECT]; t->n_select = h->cnt[K_SELECT];
    t->ms_fast = h->ms[K_FAST]; t->n_fast = h->cnt[K_FAST];
    t->ms_slow = h->ms[K_SLOW]; t->n_slow = h->cnt[K_SLOW];
    t->ms_combine = h->ms[K_COMBINE]; t->n_combine = h->cnt[K_COMBINE];
    t->ms_evict = h->ms[K_EVICT]; t->n_evict = h->cnt[K_EVICT];
    t->ms_gather = h->ms[K_GATHER]; t->n_gather = h->cnt[K_GATHER];
    t->ms_step = h->ms[K_STEP]; t->n_step = h->cnt[K_STEP];
    t->last_step_ms = h->last_step_ms;
  }
  if (reset) {
    for (int i = 0; i < K_N; ++i) { h->ms[i] = 0; h->cnt[i] = 0; }
  }
  (void)kKernelNames;
  return TTKV_OK;
}

// ---------------------------------------------------------------------------
// Fused combine + all-gather over peer memory.  With heads (or requests)
// sharded over N ranks, every rank needs every head's output; instead of a
// combine kernel followed by an NCCL all-gather, the combine kernel stores
// each (stream, head) row straight into every rank's gathered buffer over
// NVLink (CUDA IPC mappings) and publishes it with a system-scope counter;
// a one-warp wait kernel on the step's stream holds the next step until all
// ranks' rows of this step have arrived.
// ---------------------------------------------------------------------------
int ttkv_gpu_peer_gather_init(ttkv_gpu* h, uint32_t n_ranks, uint32_t my_rank,
                              uint64_t s_global, const uint32_t* gidx, void* ipc_handle) {
  if (!h || !gidx || !ipc_handle) return set_err(h, TTKV_EINVAL, "null argument");
  if (n_ranks < 1 || n_ranks > (uint32_t)kMaxPeers || my_rank >= n_ranks)
    return set_err(h, TTKV_ECONFIG, "peer gather: 1..8 ranks");
  for (uint32_t i = 0; i < h->g.S; ++i)
    if (gidx[i] >= s_global) return set_err(h, TTKV_ESHAPE, "peer gather: stream index out of range");
  CU(h, cudaSetDevice(h->dev));
  free_peer_gather(h);
  auto& p = h->pg;
  p.n_ranks = n_ranks;
  p.my_rank = my_rank;
  p.s_global = s_global;
  p.out_bytes = (size_t)s_global * h->g.G * h->g.d_v * sizeof(double);
  const size_t total = 2 * p.out_bytes + (size_t)kMaxPeers * sizeof(unsigned long long);
  CU(h, cudaMalloc((void**)&p.base, total));
  CU(h, cudaMemset(p.base, 0, total));
  CU(h, cudaMalloc((void**)&p.gidx, h->g.S * sizeof(uint32_t)));
  CU(h, cudaMemcpy(p.gidx, gidx, h->g.S * sizeof(uint32_t), cudaMemcpyHostToDevice));
  CU(h, cudaMalloc((void**)&p.status, sizeof(int)));
  CU(h, cudaMemset(p.status, 0, sizeof(int)));
  cudaIpcMemHandle_t mh;
  CU(h, cudaIpcGetMemHandle(&mh, p.base));
  std::memcpy(ipc_handle, &mh, sizeof(mh));
  return TTKV_OK;
}

int ttkv_pci_bus_id(int device, char* out, int len) {
  if (!out || len < 13) return set_err(nullptr, TTKV_EINVAL, "pci bus id: buffer too small");
  cudaError_t e = cudaDeviceGetPCIBusId(out, len, device);
  if (e != cudaSuccess)
    return set_err(nullptr, TTKV_ECUDA, std::string("cudaDeviceGetPCIBusId: ") + cudaGetErrorString(e));
  return TTKV_OK;
}

int ttkv_peer_probe(int device, const char* peer_bus_id, int* can_access) {
  if (!peer_bus_id || !can_access) return set_err(nullptr, TTKV_EINVAL, "null argument");
  *can_access = 0;
  int peer = -1;
  if (cudaDeviceGetByPCIBusId(&peer, peer_bus_id) != cudaSuccess) {
    cudaGetLastError();  // not visible to this process: no peer path
    return TTKV_OK;
  }
  if (peer == device) {
    *can_access = 1;
    return TTKV_OK;
  }
  cudaError_t e = cudaDeviceCanAccessPeer(can_access, device, peer);
  if (e != cudaSuccess)
    return set_err(nullptr, TTKV_ECUDA, std::string("cudaDeviceCanAccessPeer: ") + cudaGetErrorString(e));
  return TTKV_OK;
}

int ttkv_gpu_peer_gather_open(ttkv_gpu* h, const void* handles) {
  if (!h || !handles) return set_err(h, TTKV_EINVAL, "null argument");
  auto& p = h->pg;
  if (!p.base) return set_err(h, TTKV_EERROR, "peer gather: call ttkv_gpu_peer_gather_init first");
  CU(h, cudaSetDevice(h->dev));
  for (uint32_t r = 0; r < p.n_ranks; ++r) {
    if (r == p.my_rank) continue;
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(mh), sizeof(mh));
    CU(h, cudaIpcOpenMemHandle(&p.peer_base[r], mh, cudaIpcMemLazyEnablePeerAccess));
  }
  p.active = true;
  return TTKV_OK;
}

int ttkv_gpu_peer_gather_close(ttkv_gpu* h) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  CU(h, cudaSetDevice(h->dev));
  CU(h, cudaStreamSynchronize(h->s0));
  free_peer_gather(h);
  return TTKV_OK;
}

int ttkv_gpu_peer_gather_output(ttkv_gpu* h, double** device_rows, int* timed_out) {
  if (!h) return set_err(nullptr, TTKV_EINVAL, "null handle");
  if (!h->pg.active) return set_err(h, TTKV_EERROR, "peer gather not active");
  if (device_rows)  // the half written by the last completed step
    *device_rows = reinterpret_cast<double*>(h->pg.base + (h->pg.epoch & 1) * h->pg.out_bytes);
  if (timed_out) {
    CU(h, cudaSetDevice(h->dev));
    CU(h, cudaStreamSynchronize(h->s0));
    CU(h, cudaMemcpy(timed_out, h->pg.status, sizeof(int), cudaMemcpyDeviceToHost));
  }
  return TTKV_OK;
}

int ttkv_gpu_read_timeline(ttkv_gpu* h, uint32_t* kinds, double* start_ms, double* end_ms,
                           uint64_t cap, uint64_t* n) {
  if (!h || !n) return set_err(h, TTKV_EINVAL, "null argument");
  CU(h, cudaSetDevice(h->dev));
  drain_timing(h);
  *n = h->timeline.size();
  for (uint64_t i = 0; i < h->timeline.size() && i < cap; ++i) {
    if (kinds) kinds[i] = (uint32_t)h->timeline[i].kind;
    if (start_ms) start_ms[i] = h->timeline[i].start;
    if (end_ms) end_ms[i] = h->timeline[i].end;
  }
  return TTKV_OK;
}

// quantize_block (quantizer.cpp:126-155) as a stateless GPU call.  fp32
// staging (no ring rounding), so any float input round-trips bit-exactly.
int ttkv_gpu_quantize_block(int device, const float* keys, const float* values, uint64_t rows,
                            uint32_t d_k, uint32_t d_v, uint32_t kb, uint32_t vb,
                            uint8_t* packed_k, uint8_t* packed_v, float* key_params,
                            float* value_params, float* centroid) {
  if (!keys || !values) return set_err(nullptr, TTKV_EINVAL, "null argument");
  auto valid_bits = [](uint32_t b) { return (b >= 2 && b <= 8) || b == 16; };
  if (!valid_bits(kb) || !valid_bits(vb)) return set_err(nullptr, TTKV_ECONFIG, "bit widths must be in [2,8] or 16");
  if (rows == 0 || d_k == 0 || d_v == 0 || d_k + d_v > 1024)
    return set_err(nullptr, TTKV_ESHAPE, "quantize_block: tensor sizes inconsistent");
  Geometry g{};
  g.S = 1; g.G = 1; g.Gs = 1;
  g.d_k = d_k; g.d_v = d_v; g.B = (uint32_t)rows; g.kb = kb; g.vb = vb; g.elem = 4;
  g.C = rows; g.n_cap = 1;
  g.rec = make_layout(g.B, d_k, d_v, kb, vb, 4);
  if (evict_smem_bytes(g) > 220 * 1024)
    return set_err(nullptr, TTKV_ECONFIG, "block too large for the GPU quantizer");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_err(nullptr, TTKV_ECUDA, cudaGetErrorString(e));
  float *dk = nullptr, *dv = nullptr, *dc = nullptr;
  uint8_t* dr = nullptr;
  auto cleanup = [&]() {};  // scratch slots persist (ttkv_dev::scratch)
#define QCU(call)                                                          \
  do {                                                                     \
    cudaError_t e__ = (call);                                              \
    if (e__ != cudaSuccess) {                                              \
      cleanup();                                                           \
      return set_err(nullptr, TTKV_ECUDA, cudaGetErrorString(e__));        \
    }                                                                      \
  } while (0)
  {
    cudaError_t se = cudaSuccess;
    dk = static_cast<float*>(scratch(0, rows * d_k * 4, &se));
    if (se == cudaSuccess) dv = static_cast<float*>(scratch(1, rows * d_v * 4, &se));
    if (se == cudaSuccess) dc = static_cast<float*>(scratch(2, d_k * 4, &se));
    if (se == cudaSuccess) dr = static_cast<uint8_t*>(scratch(3, g.rec.stride, &se));
    QCU(se);
  }
  QCU(cudaMemcpy(dk, keys, rows * d_k * 4, cudaMemcpyHostToDevice));
  QCU(cudaMemcpy(dv, values, rows * d_v * 4, cudaMemcpyHostToDevice));
  EvictArgs a{};
  a.g = g;
  a.ring_k = dk;
  a.ring_v = dv;
  a.in_k = dk;
  a.in_v = dv;
  a.in_tokens = rows;
  a.split_pos = 0;
  a.first_block = 0;
  a.arena = dr;
  a.cent = dc;
  a.params = nullptr;
  QCU(launch_evict(a, 1, kInF32, 0));
  std::vector<uint8_t> rec(g.rec.stride);
  QCU(cudaMemcpy(rec.data(), dr, g.rec.stride, cudaMemcpyDeviceToHost));
  if (centroid) QCU(cudaMemcpy(centroid, dc, d_k * 4, cudaMemcpyDeviceToHost));
  cleanup();
#undef QCU
  if (packed_k) std::memcpy(packed_k, rec.data(), packed_bytes_u(rows * d_k, kb));
  if (packed_v) std::memcpy(packed_v, rec.data() + g.rec.v_off, packed_bytes_u(rows * d_v, vb));
  if (key_params && kb != 16) std::memcpy(key_params, rec.data() + g.rec.kp_off, 8 * d_k);
  if (value_params && vb != 16) std::memcpy(value_params, rec.data() + g.rec.vp_off, 8 * d_v);
  return TTKV_OK;
}

}  // extern "C"
