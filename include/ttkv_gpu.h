/*
 * ttkv_gpu.h -- C ABI of the B200-native TTKV decode hot path.
 *
 * One handle = one device, S independent KV streams (layers x KV heads x
 * requests) decoded in lockstep, each read by G query heads (GQA).  The fast
 * tier is an HBM ring (fp16 or fp32), the slow tier is K8/V4 (any 2..8/16 bit)
 * blocks in pinned host DRAM streamed over PCIe by zero-copy, the scorer and
 * top-k run on device, attention merges all partitions by online softmax.
 *
 * Every entry point replaces a reference interface (paths relative to
 * /root/reference/proj/core):
 *   ttkv_gpu_create            Engine::Engine / TierStore::TierStore
 *                              (include/ttkv/engine.hpp:36, tier_store.hpp:42)
 *                              + TierConfig::validate (config.hpp:56-74)
 *                              + fast_capacity (tier_store.cpp:36-44)
 *   ttkv_gpu_prefill           Engine::prefill (engine.cpp:15-20)
 *   ttkv_gpu_decode_step       Engine::decode_step (engine.cpp:22-93)
 *   ttkv_gpu_decode_step_device  same, device-resident inputs, async
 *   ttkv_gpu_read_fetched      DecodeStepReport::fetched_blocks (engine.hpp:29)
 *   ttkv_gpu_state             TierStore counters (tier_store.hpp:61-65)
 *   ttkv_gpu_read_block        TierStore::slow_blocks()[i] (tier_store.hpp:58)
 *   ttkv_gpu_serialize_block   serialize_block (quantizer.cpp:248-274)
 *   ttkv_gpu_dump_slow_tier    dump_slow_tier (quantizer.cpp:325-342)
 *   ttkv_gpu_restore_slow_tier load_slow_tier + deserialize_block
 *                              (quantizer.cpp:276-365) into a fresh handle
 *   ttkv_gpu_read_fast         TierStore::fast_tokens() (tier_store.hpp:57)
 *   ttkv_gpu_locate            TierStore::locate (tier_store.cpp:100-105)
 *   ttkv_gpu_quantize_block    quantize_block (quantizer.cpp:126-155)
 *   ttkv_fast_capacity         fast_capacity (tier_store.cpp:36-44)
 *   ttkv_modeled_block_bytes   modeled_block_bytes (quantizer.cpp:172-180)
 *   ttkv_resolve               SelectionPolicy::resolve (relevance.cpp:10-17)
 *
 * Errors: every int-returning call returns a TTKV_* status that maps 1:1 to
 * the reference exception classes (errors.hpp:8-41); the message is available
 * from ttkv_gpu_last_error(handle) (or ttkv_last_error() for handle-less calls).
 * No torch or CUDA types cross this boundary; streams are passed as void*.
 */
#ifndef TTKV_GPU_H
#define TTKV_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTKV_ABI_VERSION 1

/* status codes (errors.hpp:8-41) */
#define TTKV_OK 0
#define TTKV_ECONFIG 1    /* ConfigError */
#define TTKV_ESEQUENCE 2  /* SequencingError */
#define TTKV_ESHAPE 3     /* ShapeError */
#define TTKV_EINTEGRITY 4 /* IntegrityError */
#define TTKV_EIO 5        /* IoError */
#define TTKV_EERROR 6     /* plain ttkv::Error */
#define TTKV_ECUDA 7      /* CUDA runtime failure / no device */
#define TTKV_EINVAL 8     /* null handle or pointer */

/* element types of caller-provided K/V */
#define TTKV_DTYPE_F32 0
#define TTKV_DTYPE_F16 1 /* IEEE binary16 bit patterns (uint16_t) */

/* slow-tier residency */
#define TTKV_SLOW_PINNED_HOST 0 /* north-star path: pinned DRAM, PCIe zero-copy */
#define TTKV_SLOW_DEVICE 1      /* flagged variant: records in HBM */

/* Mirror of ttkv::TierConfig (config.hpp:14-41).  As in the reference,
 * bytes_full_precision is accounting (fast_capacity); the GPU storage type of
 * the fast tier is ttkv_gpu_options::ring_bytes. */
typedef struct {
  uint64_t hbm_budget_bytes;
  uint64_t d_k;
  uint64_t d_v;
  uint64_t bytes_full_precision;
  uint64_t block_size;
  uint32_t key_bits;
  uint32_t value_bits;
  double fetch_fraction;
  int32_t has_top_k_blocks;
  uint64_t top_k_blocks;
  double hbm_bandwidth;
  double pcie_bandwidth;
  double transfer_latency;
  double compute_rate;
} ttkv_tier_config;

/* Mirror of ttkv::SelectionPolicy (relevance.hpp:19-24). */
typedef struct {
  int32_t has_top_k;
  uint64_t top_k;
  double fetch_fraction;
} ttkv_selection_policy;

typedef struct {
  int32_t device;              /* CUDA ordinal */
  uint32_t n_streams;          /* S >= 1 */
  uint32_t heads_per_stream;   /* G in [1, 8] */
  uint32_t group_select;       /* 0: per-head top-k (== G reference Engines);
                                  1: one set per stream scored with sum_g q_g */
  uint64_t reserve_tokens;     /* context to preallocate for (grows on demand) */
  uint32_t slow_tier;          /* TTKV_SLOW_* */
  uint32_t copy_mode;          /* slow-block staging: 0 auto, 1 cp.async.bulk, 2 LDG */
  uint32_t literal_additive_merge; /* EngineOptions (engine.hpp:14-19): sum of
                                      per-partition normalized outputs (A/B only) */
  uint32_t ring_bytes;         /* fast-tier storage: 0 auto (fp16 if
                                  bytes_full_precision <= 2, else fp32),
                                  2 fp16 (fp32 accumulation), 4 fp32 (fp64
                                  accumulation; bit-faithful to float inputs) */
  uint32_t serial_schedule;    /* 1: bulk schedule of the reference's serial
                                  baselines (harness.cpp:22-24): all selected
                                  records are first gathered into an HBM
                                  staging arena, then attended (no overlap) */
  uint32_t record_stream;      /* HBM slow tier (TTKV_SLOW_DEVICE), G <= 4:
                                  0 / 1 the selected union after the
                                  selection (default), 2 speculative -- every
                                  record, streamed beside the selection; the
                                  combine merges only the selected ones (same
                                  selections and outputs within tolerance, more
                                  HBM bytes, the selection off the chain) */
} ttkv_gpu_options;

/* DecodeStepReport (engine.hpp:21-29) plus measured quantities. */
typedef struct {
  uint64_t blocks_scored;     /* per stream */
  uint64_t blocks_fetched;    /* per (stream, head) == k */
  double bytes_transferred;   /* modeled, per (stream, head), as the reference */
  uint64_t fast_tokens;       /* fast-tier rows attended per stream (incl. new) */
  int32_t eviction_occurred;
  uint64_t union_blocks;      /* records streamed this step, all streams
                                 (valid after the step completes) */
  uint64_t pcie_bytes;        /* union_blocks x record bytes */
} ttkv_step_report;

typedef struct {
  uint64_t appended;        /* tokens appended per stream */
  uint64_t fast_tokens;     /* resident fast-tier tokens per stream */
  uint64_t slow_blocks;     /* slow-tier blocks per stream (ids 0..n-1) */
  uint64_t l_fast;          /* fast_capacity */
  uint64_t record_bytes;    /* stored bytes per slow block record */
  uint64_t modeled_block_bytes;
  uint64_t n_streams;
  uint64_t heads_per_stream;
  uint64_t block_capacity;  /* slow blocks allocated per stream */
  uint64_t launches;        /* kernels launched by this handle so far */
  uint64_t payload_bytes;   /* bytes of each record streamed over PCIe (codes);
                               the per-channel params are staged from HBM */
  uint64_t graph_replays;   /* decode steps launched as a replay of the captured
                               step graph (host-buffer steps by default;
                               TTKV_GRAPH=1: every step, 0: none) */
  uint64_t graph_captures;  /* step graphs captured (one per eviction period) */
  uint64_t spec_steps;      /* decode steps that streamed every record beside the
                               selection (HBM slow tier, small steps; see
                               slow_attn_tc_spec_kernel) instead of the union */
} ttkv_state;

/* Kernel timing (enabled by ttkv_gpu_set_timing); milliseconds summed over
 * launches since the last reset, measured with CUDA events on the stream
 * each kernel is launched on. */
typedef struct {
  double ms_append, ms_score, ms_select, ms_fast, ms_slow, ms_combine, ms_evict;
  uint64_t n_append, n_score, n_select, n_fast, n_slow, n_combine, n_evict;
  double ms_gather;  /* serial schedule: PCIe gather into the staging arena */
  uint64_t n_gather;
  double ms_step;    /* whole decode steps (append .. settle), device time */
  uint64_t n_step;
  double last_step_ms;
} ttkv_kernel_times;

/* ---- lifecycle ------------------------------------------------------------ */
int ttkv_gpu_create(const ttkv_tier_config* cfg, const ttkv_selection_policy* policy,
                    const ttkv_gpu_options* opts, struct ttkv_gpu** out);
void ttkv_gpu_destroy(struct ttkv_gpu* h);
const char* ttkv_gpu_last_error(const struct ttkv_gpu* h);
const char* ttkv_last_error(void);
int ttkv_abi_version(void);
int ttkv_device_count(int* n);

/* Use a caller-owned stream (e.g. torch's current stream) for all work. */
int ttkv_gpu_set_stream(struct ttkv_gpu* h, void* cuda_stream);
void* ttkv_gpu_get_stream(struct ttkv_gpu* h);
int ttkv_gpu_synchronize(struct ttkv_gpu* h);

/* ---- hot path --------------------------------------------------------------- */
/* Host arrays keys[S][n][d_k], values[S][n][d_v] (dtype TTKV_DTYPE_*). */
int ttkv_gpu_prefill(struct ttkv_gpu* h, const void* keys, const void* values,
                     uint64_t n_tokens, int dtype);
/* Device-generated N(0,1) tokens rounded to the ring type (perf runs). */
int ttkv_gpu_prefill_synthetic(struct ttkv_gpu* h, uint64_t n_tokens, uint64_t seed);
/* Engine::prefill (engine.cpp:15-20) from DEVICE memory: keys [S][n][d_k],
 * values [S][n][d_v] (f32 or f16) read in place on the handle's stream. */
int ttkv_gpu_prefill_device(struct ttkv_gpu* h, const void* keys, const void* values,
                            uint64_t n_tokens, int dtype);

/* Host buffers, synchronous: q[S][G][d_k] f32, k_new[S][d_k], v_new[S][d_v]
 * (dtype), out[S][G][d_v] f64 (DecodeStepReport::output is double; values are
 * accumulated in fp32 for an fp16 ring and in fp64 for an fp32 ring).
 * report may be NULL.  Page-locked (cudaHostAlloc'd, or registered and
 * mapped) buffers are read and written by the step's kernels in place;
 * pageable ones go through the handle's page-locked staging copies.  The step
 * replays as a CUDA graph (one per eviction period; TTKV_GRAPH=0: launched
 * kernel by kernel). */
int ttkv_gpu_decode_step(struct ttkv_gpu* h, const float* q, const void* k_new,
                         const void* v_new, int dtype, double* out, ttkv_step_report* report);
/* Device buffers, enqueued on the handle's stream, returns immediately.
 * union_blocks / pcie_bytes in the report are not filled (use
 * ttkv_gpu_read_step_counters after synchronizing). */
int ttkv_gpu_decode_step_device(struct ttkv_gpu* h, const float* q, const void* k_new,
                                const void* v_new, int dtype, double* out,
                                ttkv_step_report* report);
int ttkv_gpu_read_step_counters(struct ttkv_gpu* h, uint64_t* union_blocks,
                                uint64_t* pcie_bytes);

/* TierStore::append_token (tier_store.cpp:49-67) WITHOUT settling evictions:
 * appends n tokens (host arrays [S][n][d]) to every stream.  Fails with
 * TTKV_EERROR when the fast tier would outgrow its ring (L_fast + block_size
 * tokens); settle pending evictions with ttkv_gpu_evict first. */
int ttkv_gpu_append(struct ttkv_gpu* h, const void* keys, const void* values, uint64_t n_tokens,
                    int dtype);
/* TierStore::evict_and_compress (tier_store.cpp:71-98): quantizes the oldest
 * fast-tier block of every stream into the slow tier.  TTKV_EERROR when no
 * eviction is pending. */
int ttkv_gpu_evict(struct ttkv_gpu* h, uint64_t* block_id);
int ttkv_gpu_eviction_pending(struct ttkv_gpu* h, int* pending);

/* ---- state / cold path ------------------------------------------------------ */
int ttkv_gpu_state(struct ttkv_gpu* h, ttkv_state* st);
/* fetched_blocks of the last step for (stream, head) (engine.hpp:29,
 * engine.cpp:58): the set the GPU selected and streamed (the head's bits of
 * the per-stream union, as ttkv_gpu_read_selected returns it), put in
 * select_top_k's order (relevance.cpp:29-43: score desc, block id desc) by
 * the step's fp64 scores.  TTKV_EERROR if the GPU's set does not hold
 * exactly resolve(n) blocks. */
int ttkv_gpu_read_fetched(struct ttkv_gpu* h, uint32_t stream, uint32_t head, uint64_t* out,
                          uint64_t cap, uint64_t* n);
/* The block ids the last step's slow kernel streamed for (stream, head), in
 * ascending block id: select_topk_kernel's radix-selected set as the union
 * compaction recorded it.  No reference counterpart (it is the set of
 * fetched_blocks, relevance.cpp:40-42); exposed so callers and tests can check
 * the GPU's own selection. */
int ttkv_gpu_read_selected(struct ttkv_gpu* h, uint32_t stream, uint32_t head, uint32_t* out,
                           uint64_t cap, uint64_t* n);
/* The last step's per-stream union: ascending block ids and, per id, the
 * bitmask of the query heads that selected it (each record crosses PCIe once
 * per step).  *n = union size. */
int ttkv_gpu_read_union(struct ttkv_gpu* h, uint32_t stream, uint32_t* ids, uint32_t* head_masks,
                        uint64_t cap, uint64_t* n);
/* The last step's fp64 block scores for (stream, head) (score_block,
 * relevance.cpp:19-27, one per slow block); *n = 0 when the step fetched
 * nothing (scoring is skipped then). */
int ttkv_gpu_read_scores(struct ttkv_gpu* h, uint32_t stream, uint32_t head, double* out,
                         uint64_t cap, uint64_t* n);
/* Slow block in the reference's QuantizedBlock layout (16-bit payloads as
 * float32).  Any output pointer may be NULL.  Sizes: packed_k
 * packed_bytes(B*d_k, key_bits), params 2*d floats, centroid d_k floats. */
int ttkv_gpu_read_block(struct ttkv_gpu* h, uint32_t stream, uint64_t block_id,
                        uint8_t* packed_k, uint8_t* packed_v, float* key_params,
                        float* value_params, float* centroid, uint64_t* first_position);
int ttkv_gpu_serialize_block(struct ttkv_gpu* h, uint32_t stream, uint64_t block_id,
                             uint8_t* out, uint64_t cap, uint64_t* len);
int ttkv_gpu_dump_slow_tier(struct ttkv_gpu* h, uint32_t stream, const char* path);
/* Checkpoint/resume: rebuild a fresh handle's slow tier from one TTKVTIER
 * file per stream (paths[s], n_paths == n_streams; load_slow_tier +
 * deserialize_block, quantizer.cpp:276-365, with the same integrity checks).
 * Blocks must be the contiguous sequence 0..n-1 of this config's geometry.
 * Afterwards appended == n*B; resume the fast tier with ttkv_gpu_append. */
int ttkv_gpu_restore_slow_tier(struct ttkv_gpu* h, const char* const* paths, uint32_t n_paths);
/* Fast tier as float32 rows, oldest first. */
int ttkv_gpu_read_fast(struct ttkv_gpu* h, uint32_t stream, float* keys, float* values,
                       uint64_t cap_tokens, uint64_t* n_tokens, uint64_t* first_position);
/* where: 0 fast, 1 slow, 2 absent (kv_types.hpp:31-41) */
int ttkv_gpu_locate(struct ttkv_gpu* h, uint64_t position, int* where, uint64_t* block_id);

/* ---- measurement ------------------------------------------------------------ */
int ttkv_gpu_set_timing(struct ttkv_gpu* h, int enabled);
int ttkv_gpu_kernel_times(struct ttkv_gpu* h, ttkv_kernel_times* t, int reset);
/* Kernels of the last timed decode step (timing enabled): kind (0 append,
 * 1 score, 2 select, 3 fast, 4 slow, 5 combine, 6 evict, 7 gather), start and
 * end in ms from the step's start on the critical-path stream.  The measured
 * counterpart of PipelineTimeline (sim.hpp:35-46) for write_run_timelines
 * (harness.cpp:291-300).  *n = number of events (call with cap 0 to size). */
int ttkv_gpu_read_timeline(struct ttkv_gpu* h, uint32_t* kinds, double* start_ms,
                           double* end_ms, uint64_t cap, uint64_t* n);

/* ---- multi-GPU: combine fused with the all-gather over peer memory ----------
 * With streams sharded over n_ranks GPUs (one handle per rank), every rank
 * needs every head's output.  init allocates this rank's gathered buffer
 * [s_global][G][d_v] f64 (+ arrival counters), takes gidx[s] = the global
 * index of local stream s, and returns its CUDA IPC handle (64 bytes) for the
 * caller to exchange; open maps the other ranks' buffers (handles: n_ranks x 64
 * bytes, rank order).  From then on every decode step's combine kernel also
 * stores its rows into every rank's buffer over NVLink and the step waits
 * until all ranks' rows have arrived (no separate collective); the buffer is
 * double-buffered by step parity, so the rows of step t stay valid until this
 * handle's step t+2 is enqueued.  output returns the device pointer of the
 * last completed step's gathered rows and, if timed_out is non-null,
 * synchronizes and reports whether any rank failed to arrive within ~4 s. */
int ttkv_gpu_peer_gather_init(struct ttkv_gpu* h, uint32_t n_ranks, uint32_t my_rank,
                              uint64_t s_global, const uint32_t* gidx, void* ipc_handle);
int ttkv_gpu_peer_gather_open(struct ttkv_gpu* h, const void* handles);
int ttkv_gpu_peer_gather_output(struct ttkv_gpu* h, double** device_rows, int* timed_out);
/* Unmaps the peers and frees the gathered buffer (steps stop publishing). */
int ttkv_gpu_peer_gather_close(struct ttkv_gpu* h);
/* Peer-access probe that must pass for every pair before _open: the PCI bus
 * id of a device ("dddd:bb:dd.f", cudaDeviceGetPCIBusId), and whether
 * `device` can load/store the memory of the GPU with bus id `peer_bus_id`
 * (the same GPU -> 1; a GPU this process cannot see -> 0; otherwise
 * cudaDeviceCanAccessPeer).  Callers exchange bus ids, probe every peer and
 * fall back to an NCCL all-gather unless every rank reports 1. */
int ttkv_pci_bus_id(int device, char* out, int len);
int ttkv_peer_probe(int device, const char* peer_bus_id, int* can_access);

/* ---- stateless entry points --------------------------------------------------- */
/* quantize_block on the GPU (bit-exact).  Host inputs keys[rows][d_k],
 * values[rows][d_v] f32; outputs in the reference layout. */
int ttkv_gpu_quantize_block(int device, const float* keys, const float* values, uint64_t rows,
                            uint32_t d_k, uint32_t d_v, uint32_t key_bits, uint32_t value_bits,
                            uint8_t* packed_k, uint8_t* packed_v, float* key_params,
                            float* value_params, float* centroid);
/* dequantize_block (quantizer.cpp:157-170) on the GPU, bit-exact:
 * x = float(double(code) * scale + zp); 16-bit payloads are raw float32. */
int ttkv_gpu_dequantize_block(int device, const uint8_t* packed_k, const uint8_t* packed_v,
                              const float* key_params, const float* value_params, uint64_t rows,
                              uint32_t d_k, uint32_t d_v, uint32_t key_bits, uint32_t value_bits,
                              float* keys, float* values);
/* score_block (relevance.cpp:19-27) for n centroids [n][d]: fp64, sequential,
 * one fma per term (the product of two float-valued doubles is exact, so this
 * equals the reference's separate multiply + add) -- bit-exact. */
int ttkv_gpu_score_blocks(int device, const float* query, const float* centroids, uint64_t n,
                          uint32_t d, double* scores);
/* select_top_k (relevance.cpp:29-43): the k ids ordered by (score desc, id
 * desc).  Any n < 2^31: one shared-memory bitonic CTA up to 8192 scores, a
 * global-memory bitonic network above. */
int ttkv_gpu_select_top_k(int device, const double* scores, const uint64_t* ids, uint64_t n,
                          uint64_t k, uint64_t* out);
uint64_t ttkv_fast_capacity(const ttkv_tier_config* cfg); /* 0 + last_error on error */
uint64_t ttkv_modeled_block_bytes(const ttkv_tier_config* cfg);
uint64_t ttkv_packed_bytes(uint64_t count, uint32_t bits);
uint64_t ttkv_resolve(const ttkv_selection_policy* p, uint64_t block_count); /* UINT64_MAX on error */
int ttkv_validate_config(const ttkv_tier_config* cfg);
void ttkv_default_config(ttkv_tier_config* cfg);

#ifdef __cplusplus
}
#endif
#endif /* TTKV_GPU_H */
