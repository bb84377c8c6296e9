// ttkv_launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ttkv_kernels.cuh"

namespace ttkv_dev {

constexpr int kInF32 = 0;
constexpr int kMaxPeers = 8;
constexpr int kInF16 = 1;

// Launch with programmatic stream serialization (PDL, see pdl_wait in
// ttkv_kernels.cuh): the kernel's CTAs launch while the previous kernel on
// the stream finishes.  TTKV_PDL=0 turns it off (measurement).
bool pdl_enabled();
// Per-launch scheduling priority: the step's critical path (score, select,
// slow attention, combine) at the device's greatest priority, the overlapped
// fast tier and its append at the least, whatever the caller's stream (or a
// captured graph, where nodes otherwise take the launching stream's priority).
int launch_priority(bool critical);
template <typename... KArgs, typename... Args>
cudaError_t launch_chained(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                           cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = launch_priority(true);
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// Chained (programmatic) at the least priority: side-stream work behind a
// kernel of its own stream.
template <typename... KArgs, typename... Args>
cudaError_t launch_chained_background(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = launch_priority(false);
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// A plain launch at the least priority (work that overlaps the critical path).
template <typename... KArgs, typename... Args>
cudaError_t launch_background(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = launch_priority(false);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// thread-local message behind ttkv_last_error() (defined in ttkv_engine.cu)
void set_last_error(const char* msg);
// thread-local grow-only device scratch, slot < 8 (ttkv_freefn.cu)
void* scratch(int slot, size_t bytes, cudaError_t* err);

struct EvictArgs {
  Geometry g;
  const void* ring_k;
  const void* ring_v;
  const void* in_k;      // [S][in_tokens][d_k] (Tin), positions >= split_pos
  const void* in_v;
  uint64_t in_tokens;
  uint64_t split_pos;    // positions < split_pos are read from the ring
  uint64_t first_block;  // block id of blockIdx.x == 0
  uint8_t* arena;        // device-visible record base
  float* cent;
  uint8_t* params;       // HBM mirror of record bytes [kp_off, used)
};
size_t evict_smem_bytes(const Geometry& g);
cudaError_t launch_evict(const EvictArgs& a, uint32_t n_blocks, int in_dtype, cudaStream_t st);

// ring[s][slot] <- new token (f32 or f16 input), grid-stride.  With `pos`
// (device, decode steps) the first slot is *pos mod C instead of `slot`.
cudaError_t launch_append(const Geometry& g, void* ring_k, void* ring_v, const void* k_new,
                          const void* v_new, int in_dtype, uint64_t slot, uint64_t in_stride_tok,
                          uint64_t n_tok, cudaStream_t st, const uint64_t* pos = nullptr,
                          bool chained = false);  // chained: programmatic launch, critical priority
// *p = v, stream-ordered (the device step position of a handle)
cudaError_t launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t st);

// device-generated N(0,1) tokens into staging [S][P][d] of the ring type
cudaError_t launch_synth(const Geometry& g, void* k, void* v, uint64_t P, uint64_t pos0,
                         uint64_t seed, cudaStream_t st);

struct ScoreArgs {
  Geometry g;
  const float* q;      // [S][G][d_k]
  const float* cent;   // [S][n_cap][d_k]
  double* scores;      // [S][Gs][n_cap]
  uint32_t n;          // slow blocks per stream
};
cudaError_t launch_score(const ScoreArgs& a, cudaStream_t st);

struct SelectArgs {
  Geometry g;
  const double* scores;
  uint32_t* mask;         // [S][n_cap] scratch
  uint32_t* union_ids;    // [S][n_cap]
  uint32_t* union_mask;   // [S][n_cap]
  uint32_t* union_count;  // [S]
  uint32_t n, k;
};
cudaError_t launch_select(const SelectArgs& a, cudaStream_t st);
uint32_t select_max_blocks();

// score_blocks + select_top_k + the per-stream union in ONE kernel: a thread-
// block cluster per stream scores a slice of the blocks per CTA, CTA h of the
// cluster radix-selects head h over the cluster's keys (distributed shared
// memory) and CTA 0 compacts the union.  Same bits as score_kernel +
// select_topk_kernel + select_union_kernel (the head mask `mask` is not used).
struct FusedSelectArgs {
  Geometry g;
  const float* q;
  const float* cent;
  double* scores;
  uint32_t* union_ids;
  uint32_t* union_mask;
  uint32_t* union_count;
  uint32_t n, k;
  uint32_t early_trigger;  // let the chained kernel start at once (speculative record stream)
};
bool select_fused_supported(const Geometry& g, uint32_t n, uint32_t sms);
cudaError_t launch_select_fused(const FusedSelectArgs& a, cudaStream_t st);

struct FastArgs {
  Geometry g;
  const void* ring_k;
  const void* ring_v;
  const float* q;
  void* part;         // [S][G][nfc][d_v+2] of the accumulation type
  uint64_t front;     // first fast position
  uint32_t F;         // fast tokens (when pos is null)
  const uint64_t* pos;  // device step position: F = *pos + 1 - front (decode steps)
  uint32_t FC;        // tokens per chunk (multiple of TT)
  uint32_t nfc;
  uint32_t TT;        // tokens per staged tile
  uint32_t stages;
  double scale_log2;
  uint32_t stage_region;  // set by the launcher
};
cudaError_t launch_fast(const FastArgs& a, cudaStream_t st);
uint32_t fast_tile_rows(const Geometry& g);
constexpr uint32_t kFastStages = 3;

// Tensor-core fast tier (fp16 ring, d in {64,128}, B % 64 == 0): TMA tensor
// maps of the ring + mma.sync consumers (ttkv_attention_tc.cu).
struct alignas(64) FastTcArgs {
  CUtensorMap tk;
  CUtensorMap tv;
  Geometry g;
  const float* q;
  void* part;  // float [S][G][nfc][d_v+2]
  uint64_t front;
  const uint64_t* pos;  // device step position: F = *pos + 1 - front (null: F)
  uint32_t F, FC, nfc;
  double scale_log2;
  // device-side join (null: off): the last CTA to finish bumps *done_epoch
  // (release) once every CTA's partials are stored
  uint32_t* done_arrive;
  uint32_t* done_epoch;
};
// Tensor-core slow tier (K8/V4, d = B = 128): TMA tensor maps over the
// record arena + mma.sync on raw codes with the affine params folded in.
struct alignas(64) SlowTcArgs {
  CUtensorMap tk;  // K codes
  CUtensorMap tv;  // V nibbles
  Geometry g;
  const uint8_t* params;  // HBM param mirror [S*n_cap][2048 B]
  const uint32_t* union_ids;
  const uint32_t* union_mask;
  const uint32_t* union_count;
  const float* q;
  void* part;        // [S][G][nsc][d_v + 2]
  uint32_t* nslots;  // [S] partial slots written per stream (balanced schedule)
  uint32_t per_min;  // records per CTA at least: no stream spans more than nsc CTAs
  uint32_t nsc, literal;
  double scale_log2;
  // speculative stream (slow_attn_tc_spec_kernel): every record of the step,
  // one block-local partial per (record, head) into rpart
  uint32_t spec_n;     // slow blocks per stream
  uint32_t* spec_ctr;  // record queue head (reset to 0 by the combine)
  float* rpart;        // [S][G][n_cap][kSpecPitch]
};
bool slow_tc_supported(const Geometry& g);
// Per-record partial row of the speculative stream: acc[128], m, l, 2 pad
// (16-byte aligned rows for the float4 stores).
constexpr uint32_t kSpecPitch = 132;
bool slow_tc_spec_supported(const Geometry& g);  // K8/V4, d = B = 128, G <= 4
// grid: one wave of resident CTAs; records come from the *spec_ctr queue
cudaError_t launch_slow_tc_spec(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st);
uint32_t slow_tc_ctas_per_sm(const Geometry& g);  // resident CTAs per SM of the slow tensor-core kernel
// Largest |key scale| the tensor-core slow kernel accepts: records quantized
// from an fp16 ring have s = (max - min) / 255 <= 2 * 65504 / 255 < 514, and
// the kernel normalizes q by a power of two against this bound so that the
// fp16 hi part of q * s cannot overflow.  Restored records beyond it send the
// handle to the CUDA-core slow kernel.
constexpr float kTcKeyScaleBound = 514.0f;
cudaError_t make_arena_tmaps(const Geometry& g, uint8_t* arena, SlowTcArgs& a);
// grid: one wave of resident CTAs (sms * slow_tc_ctas_per_sm())
cudaError_t launch_slow_tc(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st);

bool fast_tc_supported(const Geometry& g);
uint32_t fast_tc_tile();
cudaError_t make_ring_tmaps(const Geometry& g, void* ring_k, void* ring_v, FastTcArgs& a);
// chained: programmatic launch at critical priority (speculative record
// stream: the fast tier runs in the step's chain, not on the side stream)
// chained: 1 = programmatic behind the previous kernel at high priority (the
// speculative chain on s0), 2 = programmatic at the least priority (behind
// the append on the side stream)
cudaError_t launch_fast_tc(const FastTcArgs& a, cudaStream_t st, int chained = 0);

struct SlowArgs {
  Geometry g;
  const uint8_t* arena;
  const uint8_t* params;  // HBM param mirror
  const uint32_t* union_ids;
  const uint32_t* union_mask;
  const uint32_t* union_count;
  const float* q;
  void* part;        // [S][G][nsc][d_v+2] of the accumulation type
  uint32_t CH;       // union entries per CTA
  uint32_t nsc;      // chunk capacity per (s, g) in `part`
  uint32_t stages;
  double scale_log2;
  uint32_t stage_region;  // set by the launcher
  uint32_t literal;       // EngineOptions::literal_additive_merge
};
// copy_mode: 1 = cp.async.bulk, 2 = LDG
cudaError_t launch_slow(const SlowArgs& a, uint32_t grid_chunks, int copy_mode, cudaStream_t st);
uint32_t slow_stages_for(const Geometry& g);

// Serial schedule: copy every selected record's payload from the (mapped
// host) arena into a device staging arena at the same offsets.
cudaError_t launch_gather(const Geometry& g, const uint8_t* src, uint8_t* dst,
                          const uint32_t* union_ids, const uint32_t* union_count,
                          uint32_t grid_chunks, uint32_t CH, cudaStream_t st);

struct CombineArgs {
  Geometry g;
  const void* fpart;
  uint32_t nfc;
  const void* spart;
  uint32_t nsc;
  uint32_t CH;
  const uint32_t* union_count;  // null when no slow work this step
  const uint32_t* nslots;       // slow partial slots per stream (balanced schedule), else
                                // ceil(union_count / CH)
  double* out;                  // [S][G][d_v] (reference output is double)
  double* const* out_ref;       // non-null: the output address is *out_ref (host-buffer steps)
  uint32_t literal;
  uint64_t* pos_inc;  // the device step position, advanced once the step is combined
  // Fused all-gather over peer memory (multi-GPU sharding): each CTA also
  // stores its (stream, head) row into every rank's gathered buffer
  // [S_global][G][d_v] at global stream gidx[s], then bumps that rank's
  // arrival counter for this rank (system-scope release).
  uint32_t n_peers;  // 0: off
  uint32_t my_rank;
  const uint32_t* gidx;
  double* peer_out[kMaxPeers];
  unsigned long long* peer_flags[kMaxPeers];  // rank r's counters [n_ranks]
  // Speculative record stream: the slow partials are per-record rows
  // rpart[S][G][n_cap][kSpecPitch]; (stream, head) merges the rows of the
  // union entries whose head bit is set.  spec_ctr is reset for the next step.
  const float* rpart;  // null: slot partials (spart)
  const uint32_t* union_ids;
  const uint32_t* union_mask;
  uint64_t n_cap;
  uint32_t spec_n;
  uint32_t* spec_ctr;
  // Host-buffer steps: union_count copied into page-locked host memory for
  // the step report (the combine writes `out` there directly as well).
  uint32_t* count_out;
  // Device-side join with the fast tier (null: the stream waits on its event
  // instead): wait until *fast_epoch passes *comb_epoch, and the last CTA to
  // finish bumps *comb_epoch.  Only for grids that leave room on every SM for
  // the fast tier's CTAs (see enqueue_step).
  const uint32_t* fast_epoch;
  uint32_t* comb_epoch;
  uint32_t* comb_arrive;
};
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st);
// Host-buffer steps: the device addresses of the caller's (or the staging)
// page-locked q, k, v and output, in mapped host memory written before each
// step (graph replays read them at run time).
struct IoSlot {
  const void* src[3];
  void* out;
};
// Copies q, k, v from the addresses in *io (device-mapped page-locked host
// memory) to dst in one chained launch, and forwards io->out to *out_ref.
cudaError_t launch_ingest(void* const dst[3], const uint64_t bytes[3], const IoSlot* io,
                          void** out_ref, cudaStream_t st);
uint32_t combine_slices(const Geometry& g);  // CTAs per (stream, head) row
uint32_t combine_slices(const CombineArgs& a);  // ... of this launch (speculative: d_v / 32)
// Blocks the stream until every rank's arrival counter in `flags` reaches
// `target` (acquire, system scope); gives up after ~4 s and sets *status = 1.
cudaError_t launch_peer_wait(const unsigned long long* flags, uint32_t n_ranks,
                             unsigned long long target, int* status, cudaStream_t st);

}  // namespace ttkv_dev
