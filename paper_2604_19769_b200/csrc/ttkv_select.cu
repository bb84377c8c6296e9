// ttkv_select.cu -- block relevance scoring and top-k selection on B200.
//
// score_blocks replaces the engine's scoring loop (engine.cpp:51-56) over
// score_block (relevance.cpp:19-27): s = sum_i double(q_i) * double(c_i),
// sequential in i, one __fma_rn per term (the product of two float-valued
// doubles is exact, so this equals the reference's separate multiply + add) --
// bit-exact with the reference, so top-k ties are decided exactly as on the CPU.
// select_topk replaces SelectionPolicy::resolve + select_top_k
// (relevance.cpp:10-17, 29-43): a radix selection of the k largest
// (score, block_id) pairs -- a total order, so the set equals the prefix of
// std::stable_sort's order.  ttkv_gpu_read_fetched reads this set back (the
// union row below) and orders it by the same scores on demand.
// For GQA it also builds the per-stream union of the G selected sets plus a
// per-block head mask, so every record crosses PCIe once per step.
//
// Roofline: scoring reads the resident centroids once per step,
// n_blk * d_k * 4 bytes per stream (508 KB at 128K ctx), plus G * n_blk * d_k
// fp64 mul+add; both are microseconds at cfg2 and hide under the PCIe stream.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"
#include "ttkv_dbg_stamps.cuh"

namespace ttkv_dev {

constexpr int kScoreTile = 32;   // blocks per CTA
constexpr int kSelectThreads = 1024;
constexpr uint32_t kSelectMaxN = 16384;  // blocks per stream (2M tokens at B=128)

__global__ void __launch_bounds__(128) score_kernel(ScoreArgs a) {
  pdl_wait();  // the query / centroids when the previous kernel produced them
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y;
  const uint32_t b0 = blockIdx.x * kScoreTile;
  extern __shared__ __align__(16) uint8_t smem[];
  double* qs = reinterpret_cast<double*>(smem);                 // [Gs][d_k]
  float* ct = reinterpret_cast<float*>(qs + g.Gs * g.d_k);      // [tile][pitch]
  // d_k % 4 == 0: 16-byte rows (pitch d_k + 4 keeps 8-lane phases on distinct
  // banks); otherwise d_k + 1
  const bool vec = (g.d_k & 3u) == 0;
  const uint32_t pitch = vec ? g.d_k + 4 : g.d_k + 1;

  for (uint32_t i = threadIdx.x; i < g.Gs * g.d_k; i += blockDim.x) {
    const uint32_t h = i / g.d_k, c = i % g.d_k;
    const float* qb = a.q + (uint64_t)s * g.G * g.d_k;
    if (g.Gs == g.G) {
      qs[i] = (double)qb[h * g.d_k + c];
    } else {  // group-shared query q' = sum_g q_g (fp32, sequential g)
      float acc = qb[c];
      for (uint32_t hh = 1; hh < g.G; ++hh) acc = __fadd_rn(acc, qb[hh * g.d_k + c]);
      qs[i] = (double)acc;
    }
  }
  const float* cb = a.cent + ((uint64_t)s * g.n_cap + b0) * g.d_k;
  const uint32_t nrow = min((uint32_t)kScoreTile, a.n - b0);
  if ((g.d_k & 3u) == 0) {
    // 16-byte loads, all in flight before the first store (the tile is one
    // contiguous run of centroid rows)
    const uint32_t n4 = nrow * g.d_k / 4;
    const float4* c4 = reinterpret_cast<const float4*>(cb);
    constexpr int kU = 8;
    for (uint32_t i0 = threadIdx.x; i0 < n4; i0 += kU * blockDim.x) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        v[u] = i < n4 ? c4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        if (i < n4) {
          const uint32_t r = 4 * i / g.d_k, c = 4 * i % g.d_k;
          *reinterpret_cast<float4*>(ct + r * pitch + c) = v[u];
        }
      }
    }
  } else {
    for (uint32_t i = threadIdx.x; i < nrow * g.d_k; i += blockDim.x) {
      const uint32_t r = i / g.d_k, c = i % g.d_k;
      ct[r * pitch + c] = cb[i];
    }
  }
  __syncthreads();

  for (uint32_t t = threadIdx.x; t < kScoreTile * g.Gs; t += blockDim.x) {
    const uint32_t r = t % kScoreTile, h = t / kScoreTile;
    if (b0 + r >= a.n) continue;
    const double* qh = qs + h * g.d_k;
    const float* cr = ct + r * pitch;
    // s += double(q_i) * c_i, sequential in i (relevance.cpp:23-26).  The
    // product of two float-valued doubles has <= 48 significant bits, so the
    // reference's separate multiply is exact and RN(s + q_i c_i) is exactly
    // one fused multiply-add: bit-identical, half the fp64 instructions.
    double acc = 0.0;
    if (vec) {
      for (uint32_t c = 0; c < g.d_k; c += 4) {
        const float4 cv = *reinterpret_cast<const float4*>(cr + c);
        const double2 q01 = *reinterpret_cast<const double2*>(qh + c);
        const double2 q23 = *reinterpret_cast<const double2*>(qh + c + 2);
        acc = __fma_rn(q01.x, (double)cv.x, acc);
        acc = __fma_rn(q01.y, (double)cv.y, acc);
        acc = __fma_rn(q23.x, (double)cv.z, acc);
        acc = __fma_rn(q23.y, (double)cv.w, acc);
      }
    } else {
      for (uint32_t c = 0; c < g.d_k; ++c) acc = __fma_rn(qh[c], (double)cr[c], acc);
    }
    a.scores[((uint64_t)s * g.Gs + h) * g.n_cap + b0 + r] = acc;
  }
  pdl_trigger();  // the selection kernels may launch as the last tiles drain
}

// ---------------------------------------------------------------------------
// Row-major scoring for the fused selection kernel (d_k a multiple of 32):
// thread t scores centroid row t against EVERY selection head.  Rows are
// staged as 32-channel chunks (row pitch 36 floats, conflict-free LDS.128),
// one cp.async group per chunk, and chunk c is scored while chunks c + 1..
// are still landing.  Each score is the reference's sequential fp64 chain
// (one exact-product fma per term): the same bits as score_kernel.  As a
// standalone grid it measured slower than score_kernel (cfg2 69 vs 56 us,
// cfg3 239 vs 192 us: one chain per thread hides less latency than four).
// ---------------------------------------------------------------------------
constexpr uint32_t kFusedPitch = 36;  // floats per staged 32-channel row chunk

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_upto(uint32_t pending) {  // pending <= 3
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}
// rows [0, rows) of `cb` ([rows][d_k] floats) -> tile [nch][nb][kFusedPitch],
// one commit group per 32-channel chunk
__device__ __forceinline__ void stage_rows(const float* cb, uint32_t d_k, uint32_t rows,
                                           uint32_t nb, float* tile) {
  const uint32_t nch = d_k / 32;
  for (uint32_t ch = 0; ch < nch; ++ch) {
    for (uint32_t p = threadIdx.x; p < rows * 8; p += blockDim.x) {
      const uint32_t r = p >> 3, part = p & 7;
      cp_async16(tile + ((size_t)ch * nb + r) * kFusedPitch + 4 * part,
                 cb + (size_t)r * d_k + 32 * ch + 4 * part);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
}
// q (double, group-shared sum when Gs < G) of stream s -> qs [Gs][d_k]
__device__ __forceinline__ void stage_query_f64(const Geometry& g, const float* q, uint32_t s,
                                                double* qs) {
  const float* qb = q + (uint64_t)s * g.G * g.d_k;
  for (uint32_t i = threadIdx.x; i < g.Gs * g.d_k; i += blockDim.x) {
    const uint32_t h = i / g.d_k, c = i % g.d_k;
    if (g.Gs == g.G) {
      qs[i] = (double)qb[h * g.d_k + c];
    } else {  // group-shared query q' = sum_g q_g (fp32, sequential g)
      float acc = qb[c];
      for (uint32_t hh = 1; hh < g.G; ++hh) acc = __fadd_rn(acc, qb[hh * g.d_k + c]);
      qs[i] = (double)acc;
    }
  }
}
// Scores staged rows, waiting for the chunks as it goes (every thread of the
// CTA must call it: barriers).  Row (threadIdx.x & 127) against heads [h0, h0 + cnt): threads 0..127 take
// the first ceil(GS/2) heads, threads 128..255 the rest (nb <= 128 rows per
// CTA), so all eight warps score -- the per-thread chains are what bound this
// phase.  Each (row, head) is still one fma per channel, channels in order.
template <int GS>
constexpr int kScoreHeadsA = (GS + 1) / 2;
template <int GS>
__device__ __forceinline__ void score_staged_rows(const Geometry& g, const double* qs,
                                                  const float* tile, uint32_t rows, uint32_t nb,
                                                  double (&acc)[kScoreHeadsA<GS>], uint32_t& h0,
                                                  uint32_t& cnt) {
  constexpr int HA = kScoreHeadsA<GS>;
  const uint32_t row = threadIdx.x & 127u;
  const bool upper = threadIdx.x >= 128u;
  h0 = upper ? (uint32_t)HA : 0u;
  cnt = upper ? (uint32_t)(GS - HA) : (uint32_t)HA;
  if (row >= rows) cnt = 0;
#pragma unroll
  for (int h = 0; h < HA; ++h) acc[h] = 0.0;
  const uint32_t nch = g.d_k / 32;
  for (uint32_t ch = 0; ch < nch; ++ch) {
    cp_async_wait_upto(nch - 1 - ch);
    __syncthreads();  // chunk ch (and q) visible to every thread
    if (cnt) {  // warp-uniform except in the last partial warp of rows
      const float* tr = tile + ((size_t)ch * nb + row) * kFusedPitch;
      const double* qc = qs + (size_t)h0 * g.d_k + 32 * ch;
#pragma unroll 4
      for (uint32_t c = 0; c < 32; c += 4) {
        const float4 cv = *reinterpret_cast<const float4*>(tr + c);
        const double c0 = cv.x, c1 = cv.y, c2 = cv.z, c3 = cv.w;
#pragma unroll
        for (int h = 0; h < HA; ++h) {
          if (h < (int)cnt) {
            const double2 q01 = *reinterpret_cast<const double2*>(qc + h * g.d_k + c);
            const double2 q23 = *reinterpret_cast<const double2*>(qc + h * g.d_k + c + 2);
            acc[h] = __fma_rn(q01.x, c0, acc[h]);
            acc[h] = __fma_rn(q01.y, c1, acc[h]);
            acc[h] = __fma_rn(q23.x, c2, acc[h]);
            acc[h] = __fma_rn(q23.y, c3, acc[h]);
          }
        }
      }
    }
  }
}

cudaError_t launch_score(const ScoreArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  const size_t smem = (size_t)a.g.Gs * a.g.d_k * 8 + (size_t)kScoreTile * (a.g.d_k + 4) * 4;
  cudaError_t e = cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.n + kScoreTile - 1) / kScoreTile, a.g.S);
  return launch_chained(score_kernel, grid, dim3(128), smem, st, a);
}

// orderable key: ascending u64 == ascending double; -0.0 folded onto +0.0
// because the reference compares with != (relevance.cpp:35).
__device__ __forceinline__ uint64_t order_key(double d) {
  if (d == 0.0) d = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// One CTA per (stream, selection head): the top-k SET by radix selection.
// The attention needs only which blocks each head selected; their order (the
// reference's fetched_blocks, select_top_k's stable_sort by score desc, id
// desc) is a report field: ttkv_gpu_read_fetched reads this kernel's set back
// from the union row and sorts it by the same fp64 scores.  The k-th largest (key, id) pair is found MSB
// first over the 64-bit order key (8-bit digits) and then the 14-bit block id
// (two 7-bit digits), stopping as soon as the threshold bucket is taken
// whole; every element at or above the threshold is selected.
constexpr int kTopkThreads = 256;
constexpr uint32_t kTopkSmemKeys = 5632;  // order keys cached in smem (44 KB) up to this n

__device__ __forceinline__ uint32_t topk_digit(uint64_t key, uint32_t id, int p) {
  return p < 8 ? (uint32_t)(key >> (56 - 8 * p)) & 0xffu : (p == 8 ? (id >> 7) & 0x7fu : id & 0x7fu);
}

// The radix selection proper, shared by select_topk_kernel and the fused
// selection kernel: kTopkThreads threads find the k-th largest (key, id) pair
// of n elements; key_of(i, pass) yields element i's order key.
struct RadixThreshold {
  int p;             // last pass taken (digits of passes <= p are fixed)
  uint64_t key_pre;  // chosen key digits (passes < 8)
  uint32_t id_pre;   // chosen id digits (passes 8, 9)
};
struct RadixShared {
  uint32_t hist[256];
  uint32_t digit, need, done;
};
template <typename KeyOf>
__device__ RadixThreshold radix_threshold(KeyOf key_of, uint32_t n, uint32_t k, RadixShared& sh) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t key_pre = 0;  // chosen key digits so far (passes < 8)
  uint32_t id_pre = 0;   // chosen id digits (passes 8, 9)
  uint32_t need = k;
  int p = 0;
  // does (key, id) agree with the chosen digits of passes < p?
  auto match = [&](uint64_t key, uint32_t id, int pp) -> bool {
    if (pp == 0) return true;
    if (pp <= 8) return (key >> (64 - 8 * pp)) == key_pre;
    return key == key_pre && (id >> 7) == id_pre;
  };
  for (;; ++p) {
    for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) sh.hist[b] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t key = key_of(i, p);
      if (match(key, i, p)) atomicAdd(&sh.hist[topk_digit(key, i, p)], 1u);
    }
    __syncthreads();
    if (warp == 0) {
      // bins from the top: lane l owns bins 255-8l .. 248-8l
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        c[e] = sh.hist[255 - 8 * lane - e];
        tot += c[e];
      }
      uint32_t incl = tot;  // inclusive prefix over lanes (higher bins first)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
      }
      uint32_t above = incl - tot;
      const bool mine = above < need && incl >= need;
      if (mine) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (above + c[e] >= need) {
            sh.digit = 255 - 8 * lane - e;
            sh.need = need - above;
            sh.done = (c[e] == need - above) ? 1u : 0u;
            break;
          }
          above += c[e];
        }
      }
    }
    __syncthreads();
    const uint32_t d = sh.digit;
    need = sh.need;
    const bool done = sh.done != 0;
    if (p < 8) key_pre = (key_pre << 8) | d;
    else id_pre = (id_pre << 7) | d;
    if (done || p == 9) break;
    __syncthreads();  // sh.* are rewritten by the next pass
  }
  return {p, key_pre, id_pre};
}
// selected: (key, id) >= threshold, compared on the digits fixed so far
__device__ __forceinline__ bool radix_selected(uint64_t key, uint32_t i, const RadixThreshold& t) {
  if (t.p < 8) return (key >> (56 - 8 * t.p)) >= t.key_pre;
  if (t.p == 8) return key > t.key_pre || (key == t.key_pre && (i >> 7) >= t.id_pre);
  return key > t.key_pre || (key == t.key_pre && i >= t.id_pre);
}

__global__ void __launch_bounds__(kTopkThreads) select_topk_kernel(SelectArgs a) {
  pdl_trigger();  // few CTAs: let the union kernel's CTAs get resident
  pdl_wait();     // the scores
  const Geometry& g = a.g;
  const uint32_t h = blockIdx.x, s = blockIdx.y;
  const double* sc = a.scores + ((uint64_t)s * g.Gs + h) * g.n_cap;
  __shared__ RadixShared sh;
  // the order keys are computed once (pass 0) and re-read from shared memory
  // by the later passes and the final marking, not from L2 each time
  extern __shared__ uint64_t keys_sm[];
  const bool cached = a.n <= kTopkSmemKeys;
  auto key_of = [&](uint32_t i, int pass) -> uint64_t {
    if (!cached) return order_key(sc[i]);
    if (pass == 0) {
      const uint64_t k = order_key(sc[i]);
      keys_sm[i] = k;
      return k;
    }
    return keys_sm[i];
  };
  const RadixThreshold t = radix_threshold(key_of, a.n, a.k, sh);
  uint32_t* mask = a.mask + (uint64_t)s * g.n_cap;
  const uint32_t all_heads = (g.G >= 32) ? 0xffffffffu : ((1u << g.G) - 1u);
  const uint32_t bit = (g.Gs == g.G) ? (1u << h) : all_heads;
  for (uint32_t i = threadIdx.x; i < a.n; i += blockDim.x) {
    const uint64_t key = key_of(i, 1);  // each thread re-reads only its own keys
    if (radix_selected(key, i, t)) atomicOr(&mask[i], bit);
  }
}

// Per stream: compact the union of the G selected sets in ascending block id
// (records are then read in arena order; the merge is order-independent,
// SPEC.md:287) and clear the head mask for the next step.
__global__ void __launch_bounds__(kSelectThreads) select_union_kernel(SelectArgs a) {
  pdl_trigger();
  pdl_wait();  // the per-head selection masks
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.x;
  __shared__ uint32_t warp_tot[kSelectThreads / 32];
  __shared__ uint32_t base_sh;
  uint32_t* mask = a.mask + (uint64_t)s * g.n_cap;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) base_sh = 0;
  __syncthreads();
  // the mask words of kPre consecutive tiles are loaded together (one L2
  // round trip), then compacted tile by tile from registers
  constexpr int kPre = 8;
  for (uint32_t base0 = 0; base0 < a.n; base0 += kPre * blockDim.x) {
    uint32_t mv[kPre];
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const uint32_t b = base0 + u * blockDim.x + threadIdx.x;
      mv[u] = b < a.n ? mask[b] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const uint32_t b = base0 + u * blockDim.x + threadIdx.x;
      if (b < a.n) mask[b] = 0u;
    }
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const uint32_t base = base0 + u * blockDim.x;
      if (base < a.n) {  // CTA-uniform
        const uint32_t b = base + threadIdx.x;
        const uint32_t m = mv[u];
        const uint32_t ballot = __ballot_sync(0xffffffffu, m != 0u);
        if (lane == 0) warp_tot[warp] = __popc(ballot);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (uint32_t w = 0; w < nwarps; ++w) {
          const uint32_t t = warp_tot[w];
          before += (w < warp) ? t : 0u;
          total += t;
        }
        if (m != 0u) {
          const uint32_t pos = base_sh + before + __popc(ballot & ((1u << lane) - 1u));
          a.union_ids[(uint64_t)s * g.n_cap + pos] = b;
          a.union_mask[(uint64_t)s * g.n_cap + pos] = m;
        }
        __syncthreads();
        if (threadIdx.x == 0) base_sh += total;
        __syncthreads();
      }
    }
  }
  if (threadIdx.x == 0) a.union_count[s] = base_sh;
}

uint32_t select_max_blocks() { return kSelectMaxN; }

// ---------------------------------------------------------------------------
// Fused selection: score_blocks -> select_top_k -> union for one stream per
// thread-block cluster (relevance.cpp:19-43, engine.cpp:51-58).
//   * CTA r of the cluster owns blocks [r nb, (r+1) nb): its centroid rows are
//     staged in 32-channel chunks with 16-byte cp.async (row pitch 36 floats:
//     conflict-free LDS.128), then threads t and t + 128 score row t against
//     half the selection heads each, channels in order with one fma each --
//     the same fp64 chain as score_kernel, so the same bits (the chain of 128
//     dependent fmas, not the loads, bounds this phase: 2.5 us of ~10).
//   * after a cluster barrier, CTA h gathers head h's n order keys from the
//     cluster's shared memory (DSMEM) and runs the radix selection of
//     select_topk_kernel on them; its selected set lands as a bitmask in CTA 0.
//   * after a second barrier CTA 0 compacts the union of the heads' sets in
//     ascending block id with the head bitmask, like select_union_kernel.
// One launch instead of three, and the scores never round-trip through L2
// before selection (layer-sequential decode is latency-bound on this chain).
// ---------------------------------------------------------------------------
constexpr uint32_t kFusedMaxN = 2048;
#if defined(TTKV_STAMPS) && !defined(TTKV_PHASE_STAMP)  // in-chain phases (tools/chain_stamps.py)
TTKV_DBG_TABLE(sel)
TTKV_DBG_READER(sel)
#define TTKV_PHASE_STAMP(k) TTKV_DBG_STAMP(sel, k)
#endif
#ifndef TTKV_PHASE_STAMP  // tools/fused_probe.cu times the phases with %globaltimer
#define TTKV_PHASE_STAMP(k)
#endif


struct FusedLayout {
  uint32_t CL, nb, nw, nch;
  size_t off_keys, off_gkeys, off_sel, off_tile, bytes;
};
__host__ __device__ inline FusedLayout fused_layout(const Geometry& g, uint32_t n) {
  FusedLayout L{};
  uint32_t cl = 1;
  while (cl < g.Gs || (n + cl - 1) / cl > 128) cl *= 2;
  L.CL = cl;
  L.nb = (n + cl - 1) / cl;
  L.nw = (n + 31) / 32;
  L.nch = g.d_k / 32;
  size_t o = (size_t)g.Gs * g.d_k * 8;          // qs [Gs][d_k] f64
  L.off_keys = o;  o += (size_t)g.Gs * L.nb * 8;  // keys [Gs][nb] (this CTA's slice)
  L.off_gkeys = o; o += (size_t)n * 8;            // gkeys [n] (the head this CTA selects)
  L.off_sel = o;   o += (size_t)g.Gs * L.nw * 4;  // selection bitmasks [Gs][nw] (CTA 0)
  o = (o + 15) & ~size_t(15);
  L.off_tile = o;  o += (size_t)L.nch * L.nb * kFusedPitch * 4;
  L.bytes = o;
  return L;
}

template <int GS>
__global__ void __launch_bounds__(kTopkThreads) select_fused_kernel(FusedSelectArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const Geometry& g = a.g;
  const uint32_t rank = blockIdx.x, s = blockIdx.y, n = a.n;
  const FusedLayout L = fused_layout(g, n);
  const uint32_t r0 = rank * L.nb;
  const uint32_t rows = r0 < n ? min(L.nb, n - r0) : 0u;
  extern __shared__ __align__(16) uint8_t fsm[];
  double* qs = reinterpret_cast<double*>(fsm);
  uint64_t* keys = reinterpret_cast<uint64_t*>(fsm + L.off_keys);
  uint64_t* gkeys = reinterpret_cast<uint64_t*>(fsm + L.off_gkeys);
  uint32_t* selbits = reinterpret_cast<uint32_t*>(fsm + L.off_sel);
  float* tile = reinterpret_cast<float*>(fsm + L.off_tile);  // [nch][nb][kFusedPitch]
  __shared__ RadixShared sh;
  __shared__ uint32_t warp_tot[kTopkThreads / 32];
  __shared__ uint32_t base_sh;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  TTKV_PHASE_STAMP(0);
  // The centroid rows are staged BEFORE pdl_wait, overlapping the previous
  // kernel's tail: every kernel that writes centroids (the evictions) is a
  // plain launch that never triggers its dependents early, so the previous
  // kernel is not one of them while it is still running.  q is read after.
  stage_rows(a.cent + ((uint64_t)s * g.n_cap + r0) * g.d_k, g.d_k, rows, L.nb, tile);
  pdl_wait();  // the query
  // speculative record stream: it needs nothing from this kernel until its
  // end, so its CTAs take the SMs this selection leaves free right away
  if (a.early_trigger) pdl_trigger();
  stage_query_f64(g, a.q, s, qs);
  TTKV_PHASE_STAMP(1);
  // ---- score: row t against every head (score_staged_rows: the same fp64
  // chain as score_kernel, so the same bits) ----
  {
    double acc[kScoreHeadsA<GS>];
    uint32_t h0, cnt;
    score_staged_rows<GS>(g, qs, tile, rows, L.nb, acc, h0, cnt);
    const uint32_t row = threadIdx.x & 127u;
#pragma unroll
    for (int j = 0; j < kScoreHeadsA<GS>; ++j)
      if (j < (int)cnt) {
        const uint32_t h = h0 + j;
        a.scores[((uint64_t)s * g.Gs + h) * g.n_cap + r0 + row] = acc[j];
        keys[h * L.nb + row] = order_key(acc[j]);
      }
  }
  TTKV_PHASE_STAMP(2);
  cluster.sync();  // every slice's keys are visible cluster-wide
  TTKV_PHASE_STAMP(3);

  // ---- select: CTA h radix-selects head h over the gathered keys ----
  if (rank < g.Gs) {
    const uint32_t h = rank;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t src = i / L.nb;
      const uint64_t* pk = cluster.map_shared_rank(keys, src);
      gkeys[i] = pk[h * L.nb + (i - src * L.nb)];
    }
    __syncthreads();
    TTKV_PHASE_STAMP(4);
    auto key_of = [&](uint32_t i, int) -> uint64_t { return gkeys[i]; };
    const RadixThreshold t = radix_threshold(key_of, n, a.k, sh);
    TTKV_PHASE_STAMP(5);
    uint32_t* sb0 = cluster.map_shared_rank(selbits, 0) + h * L.nw;
    for (uint32_t base = warp * 32; base < n; base += blockDim.x) {  // warp-uniform
      const uint32_t i = base + lane;
      const bool sel = i < n && radix_selected(gkeys[i], i, t);
      const uint32_t word = __ballot_sync(0xffffffffu, sel);
      if (lane == 0) sb0[base / 32] = word;
    }
  }
  cluster.sync();  // CTA 0 holds every head's set; no peer reads remain
  TTKV_PHASE_STAMP(6);
  pdl_trigger();   // the attention kernel's CTAs may get resident
  if (rank != 0) return;

  // ---- union (CTA 0): ascending block id with the head bitmask.  n <= 2048
  // = 8 warps x 8 words: warp w ballots blocks [256w, 256w + 256) word by
  // word, one barrier publishes the warp totals ----
  const uint32_t all_heads = (g.G >= 32) ? 0xffffffffu : ((1u << g.G) - 1u);
  uint32_t mw[8], bal[8], cnt = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t b = 256 * warp + 32 * j + lane;
    uint32_t m = 0;
    if (b < n)
#pragma unroll
      for (int h = 0; h < GS; ++h)  // GS == g.Gs (launch_select_fused)
        if ((selbits[h * L.nw + (b >> 5)] >> (b & 31)) & 1u)
          m |= (GS == g.G) ? (1u << h) : all_heads;
    mw[j] = m;
    bal[j] = __ballot_sync(0xffffffffu, m != 0u);
    cnt += __popc(bal[j]);
  }
  if (lane == 0) warp_tot[warp] = cnt;
  __syncthreads();
  uint32_t pos = 0, total = 0;
  for (uint32_t w = 0; w < kTopkThreads / 32; ++w) {
    pos += (w < warp) ? warp_tot[w] : 0u;
    total += warp_tot[w];
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (mw[j] != 0u) {
      const uint32_t at = pos + __popc(bal[j] & lt);
      a.union_ids[(uint64_t)s * g.n_cap + at] = 256 * warp + 32 * j + lane;
      a.union_mask[(uint64_t)s * g.n_cap + at] = mw[j];
    }
    pos += __popc(bal[j]);
  }
  if (threadIdx.x == 0) base_sh = total;
  if (threadIdx.x == 0) a.union_count[s] = base_sh;
  TTKV_PHASE_STAMP(7);
}

bool select_fused_supported(const Geometry& g, uint32_t n, uint32_t sms) {
  static const bool on = [] {  // TTKV_FUSED_SELECT=0: the three-kernel chain (measurement)
    const char* e = std::getenv("TTKV_FUSED_SELECT");
    return !(e && e[0] == '0');
  }();
  if (!on || n == 0 || n > kFusedMaxN || g.d_k % 32 != 0 || g.d_k > 128 || g.Gs > 8) return false;
  const FusedLayout L = fused_layout(g, n);
  if (L.CL > 16 || L.nb > 128 || L.bytes > 200 * 1024) return false;  // two thread halves per row
  // one wave: the clusters hold their SMs through two barriers, so a second
  // wave would wait for the first (cfg2, S = 256: 120 us vs 74 us for the three-kernel chain)
  const uint64_t per_sm = std::min<uint64_t>(kTopkThreads == 256 ? 8 : 4,
                                             (227u * 1024u) / (L.bytes + 2048));
  return (uint64_t)g.S * L.CL <= (uint64_t)sms * per_sm;
}

template <int GS>
static cudaError_t launch_select_fused_t(const FusedSelectArgs& a, const FusedLayout& L,
                                         cudaStream_t st) {
  auto kern = select_fused_kernel<GS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)L.bytes);
  if (e != cudaSuccess) return e;
  if (L.CL > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.CL, a.g.S);
  cfg.blockDim = dim3(kTopkThreads);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = launch_priority(true);
  attr[2].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[2].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 3 : 2;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t launch_select_fused(const FusedSelectArgs& a, cudaStream_t st) {
  const FusedLayout L = fused_layout(a.g, a.n);
  switch (a.g.Gs) {
    case 1: return launch_select_fused_t<1>(a, L, st);
    case 2: return launch_select_fused_t<2>(a, L, st);
    case 3: return launch_select_fused_t<3>(a, L, st);
    case 4: return launch_select_fused_t<4>(a, L, st);
    case 5: return launch_select_fused_t<5>(a, L, st);
    case 6: return launch_select_fused_t<6>(a, L, st);
    case 7: return launch_select_fused_t<7>(a, L, st);
    default: return launch_select_fused_t<8>(a, L, st);
  }
}

// The head mask (a.mask) must be all-zero on entry; select_union_kernel
// leaves it zeroed again.  `sel` is not written: the order is a cold read.
cudaError_t launch_select(const SelectArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  const size_t smem = a.n <= kTopkSmemKeys ? (size_t)a.n * 8 : 0;
  cudaError_t e = launch_chained(select_topk_kernel, dim3(a.g.Gs, a.g.S), dim3(kTopkThreads),
                                 smem, st, a);
  if (e != cudaSuccess) return e;
  return launch_chained(select_union_kernel, dim3(a.g.S), dim3(256), 0, st, a);
}

// ---------------------------------------------------------------------------
// append_kv: TierStore::append_token's push into the fast tier
// (tier_store.cpp:49-67) -- the new token lands in ring slot pos mod C.
// Also used by prefill to copy tokens [in_stride] into consecutive slots.
// ---------------------------------------------------------------------------
template <typename T, typename Tin>
__global__ void append_kernel(Geometry g, T* ring_k, T* ring_v, const Tin* kn, const Tin* vn,
                              uint64_t slot0, uint64_t in_stride_tok, uint64_t n_tok,
                              const uint64_t* pos) {
  // chained launch (speculative record stream): the selection may launch at
  // once; the step position is advanced by the previous step's combine
  pdl_trigger();
  pdl_wait();
  // one thread per 8-element group of a token row; K groups then V groups
  const uint32_t gk = g.d_k / 8, gv = g.d_v / 8, gr = gk + gv;
  const uint64_t total = (uint64_t)g.S * n_tok * gr;
  const uint32_t slot_base = (uint32_t)((pos ? *pos : slot0) % g.C);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c8 = (uint32_t)(i % gr);
    const uint64_t st = i / gr;
    const uint32_t t = (uint32_t)(st % n_tok);
    const uint32_t s = (uint32_t)(st / n_tok);
    uint32_t slot = slot_base + t;
    slot = slot >= g.C ? slot - (uint32_t)g.C * (slot / (uint32_t)g.C) : slot;
    const bool is_k = c8 < gk;
    const uint32_t dim = is_k ? g.d_k : g.d_v, c = 8 * (is_k ? c8 : c8 - gk);
    const Tin* src = (is_k ? kn : vn) + ((uint64_t)s * in_stride_tok + t) * dim + c;
    T* dst = (is_k ? ring_k : ring_v) + ((uint64_t)s * g.C + slot) * dim + c;
    Tin x[8];
#pragma unroll
    for (int e = 0; e < 8; e += 16 / (int)sizeof(Tin))
      *reinterpret_cast<uint4*>(x + e) = *reinterpret_cast<const uint4*>(src + e);
    T o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = from_f<T>(to_f(x[e]));
#pragma unroll
    for (int e = 0; e < 8; e += 16 / (int)sizeof(T) > 8 ? 8 : 16 / (int)sizeof(T))
      *reinterpret_cast<uint4*>(dst + e) = *reinterpret_cast<const uint4*>(o + e);
  }
}

// generic shape (a dimension not a multiple of 8): one thread per element
template <typename T, typename Tin>
__global__ void append_kernel_scalar(Geometry g, T* ring_k, T* ring_v, const Tin* kn,
                                     const Tin* vn, uint64_t slot0, uint64_t in_stride_tok,
                                     uint64_t n_tok, const uint64_t* pos) {
  pdl_trigger();
  pdl_wait();
  if (pos) slot0 = *pos;
  const uint32_t dkv = g.d_k + g.d_v;
  const uint64_t total = (uint64_t)g.S * n_tok * dkv;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(i % dkv);
    const uint64_t st = i / dkv;
    const uint64_t t = st % n_tok, s = st / n_tok;
    const uint64_t slot = (slot0 + t) % g.C;
    if (c < g.d_k)
      ring_k[(s * g.C + slot) * g.d_k + c] = from_f<T>(to_f(kn[(s * in_stride_tok + t) * g.d_k + c]));
    else
      ring_v[(s * g.C + slot) * g.d_v + (c - g.d_k)] =
          from_f<T>(to_f(vn[(s * in_stride_tok + t) * g.d_v + (c - g.d_k)]));
  }
}

template <typename T, typename Tin>
static void launch_append_t(const Geometry& g, void* ring_k, void* ring_v, const void* k_new,
                            const void* v_new, uint64_t slot, uint64_t in_stride_tok,
                            uint64_t n_tok, cudaStream_t st, const uint64_t* pos, bool chained) {
  const bool vec = g.d_k % 8 == 0 && g.d_v % 8 == 0 &&
                   ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15) == 0;
  const uint64_t total = (uint64_t)g.S * n_tok * (vec ? (g.d_k + g.d_v) / 8 : g.d_k + g.d_v);
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  auto kv = append_kernel<T, Tin>;
  auto ks = append_kernel_scalar<T, Tin>;
  auto kern = vec ? kv : ks;
  if (chained)
    launch_chained(kern, dim3((unsigned)blocks), dim3(256), 0, st, g, (T*)ring_k, (T*)ring_v,
                   (const Tin*)k_new, (const Tin*)v_new, slot, in_stride_tok, n_tok, pos);
  else
    launch_background(kern, dim3((unsigned)blocks), dim3(256), 0, st, g, (T*)ring_k, (T*)ring_v,
                      (const Tin*)k_new, (const Tin*)v_new, slot, in_stride_tok, n_tok, pos);
}

cudaError_t launch_append(const Geometry& g, void* ring_k, void* ring_v, const void* k_new,
                          const void* v_new, int in_dtype, uint64_t slot, uint64_t in_stride_tok,
                          uint64_t n_tok, cudaStream_t st, const uint64_t* pos, bool chained) {
  if (n_tok == 0) return cudaSuccess;
  if (g.elem == 2) {
    if (in_dtype == kInF16)
      launch_append_t<__half, __half>(g, ring_k, ring_v, k_new, v_new, slot, in_stride_tok, n_tok, st, pos, chained);
    else
      launch_append_t<__half, float>(g, ring_k, ring_v, k_new, v_new, slot, in_stride_tok, n_tok, st, pos, chained);
  } else {
    if (in_dtype == kInF16)
      launch_append_t<float, __half>(g, ring_k, ring_v, k_new, v_new, slot, in_stride_tok, n_tok, st, pos, chained);
    else
      launch_append_t<float, float>(g, ring_k, ring_v, k_new, v_new, slot, in_stride_tok, n_tok, st, pos, chained);
  }
  return cudaGetLastError();
}

__global__ void set_u64_kernel(uint64_t* p, uint64_t v) { *p = v; }

cudaError_t launch_set_u64(uint64_t* p, uint64_t v, cudaStream_t st) {
  set_u64_kernel<<<1, 1, 0, st>>>(p, v);
  return cudaGetLastError();
}

// Host-buffer steps: the step's q, k and v are read straight from page-locked
// host memory (mapped into the device's address space) by one kernel instead
// of three copy-engine transfers, each of which costs ~4 us of queue latency
// on a small step (cfg1: 48 KB in).  The host addresses come from the
// handle's mapped IoSlot, written by the host before the launch, so a
// replayed graph of the step holds no caller pointer; the output address is
// forwarded to *out_ref (device memory) for the combine.  Segment blockIdx.y;
// 16-byte accesses when both ends are aligned, bytes otherwise.
struct IngestArgs {
  void* dst[3];
  uint64_t bytes[3];
  const IoSlot* io;
  void** out_ref;
};
__global__ void __launch_bounds__(256) ingest_kernel(IngestArgs a) {
  pdl_wait();  // the previous step is done with the device copies
  pdl_trigger();
  const uint32_t seg = blockIdx.y;
  uint8_t* d = static_cast<uint8_t*>(a.dst[seg]);
  const uint8_t* sp = static_cast<const uint8_t*>(a.io->src[seg]);
  if (seg == 0 && blockIdx.x == 0 && threadIdx.x == 0) *a.out_ref = a.io->out;
  const uint64_t nb = a.bytes[seg];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((((uintptr_t)d | (uintptr_t)sp | nb) & 15u) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(sp);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (uint64_t i = t0; i < nb / 16; i += stride) d4[i] = s4[i];
  } else {
    for (uint64_t i = t0; i < nb; i += stride) d[i] = sp[i];
  }
}

cudaError_t launch_ingest(void* const dst[3], const uint64_t bytes[3], const IoSlot* io,
                          void** out_ref, cudaStream_t st) {
  IngestArgs a{};
  uint64_t most = 0;
  for (int i = 0; i < 3; ++i) {
    a.dst[i] = dst[i];
    a.bytes[i] = bytes[i];
    most = std::max<uint64_t>(most, bytes[i]);
  }
  a.io = io;
  a.out_ref = out_ref;
  const uint64_t ctas = std::min<uint64_t>(256, std::max<uint64_t>(1, (most / 16 + 255) / 256));
  return launch_chained(ingest_kernel, dim3((uint32_t)ctas, 3), dim3(256), 0, st, a);
}

// ---------------------------------------------------------------------------
// synthetic N(0,1) KV for perf runs (on-device generation is
// acceptable at cfg2-5 scale): counter-based hash + Box-Muller.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

template <typename T>
__global__ void synth_kernel(Geometry g, T* k, T* v, uint64_t P, uint64_t pos0, uint64_t seed) {
  const uint32_t dkv = g.d_k + g.d_v;
  const uint64_t total = (uint64_t)g.S * P * dkv;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(i % dkv);
    const uint64_t st = i / dkv;
    const uint64_t t = st % P, s = st / P;
    const uint64_t ctr = ((s * 0x9E3779B97F4A7C15ull) ^ ((pos0 + t) << 9) ^ c) + seed * 0xD1B54A32D192ED03ull;
    const uint64_t h = mix64(ctr), h2 = mix64(ctr ^ 0x5851F42D4C957F2Dull);
    const float u1 = ((float)(h >> 40) + 1.0f) * (1.0f / 16777216.0f);
    const float u2 = (float)(h2 >> 40) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307f * u2);
    if (c < g.d_k) k[(s * P + t) * g.d_k + c] = from_f<T>(z);
    else v[(s * P + t) * g.d_v + (c - g.d_k)] = from_f<T>(z);
  }
}

cudaError_t launch_synth(const Geometry& g, void* k, void* v, uint64_t P, uint64_t pos0,
                         uint64_t seed, cudaStream_t st) {
  const uint64_t total = (uint64_t)g.S * P * (g.d_k + g.d_v);
  uint64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (g.elem == 2)
    synth_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>(g, (__half*)k, (__half*)v, P, pos0, seed);
  else
    synth_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(g, (float*)k, (float*)v, P, pos0, seed);
  return cudaGetLastError();
}

}  // namespace ttkv_dev

namespace ttkv_dev {

// ---------------------------------------------------------------------------
// gather_records: the bulk phase of the serial schedule (harness.cpp:22-24,
// simulate_serial sim.cpp:90-112 made real): every selected record's payload
// crosses PCIe into an HBM staging arena before any attention starts.
// 16-byte zero-copy loads, 8 in flight per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_kernel(Geometry g, const uint8_t* src, uint8_t* dst,
                                                     const uint32_t* uids, const uint32_t* ucount,
                                                     uint32_t CH) {
  const uint32_t s = blockIdx.y;
  const uint32_t i0 = blockIdx.x * CH, cnt = ucount[s];
  if (i0 >= cnt) return;
  const uint32_t i1 = min(i0 + CH, cnt);
  const uint32_t n16 = g.rec.kp_off >> 4;
  for (uint32_t i = i0; i < i1; ++i) {
    const uint64_t off = ((uint64_t)s * g.n_cap + uids[(uint64_t)s * g.n_cap + i]) * g.rec.stride;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + off);
    uint4* d4 = reinterpret_cast<uint4*>(dst + off);
    uint32_t j = threadIdx.x;
    for (; j + 7 * 256 < n16; j += 8 * 256) {
      uint4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = s4[j + u * 256];
#pragma unroll
      for (int u = 0; u < 8; ++u) d4[j + u * 256] = r[u];
    }
    for (; j < n16; j += 256) d4[j] = s4[j];
  }
}

cudaError_t launch_gather(const Geometry& g, const uint8_t* src, uint8_t* dst,
                          const uint32_t* union_ids, const uint32_t* union_count,
                          uint32_t grid_chunks, uint32_t CH, cudaStream_t st) {
  if (grid_chunks == 0) return cudaSuccess;
  dim3 grid(grid_chunks, g.S);
  gather_kernel<<<grid, 256, 0, st>>>(g, src, dst, union_ids, union_count, CH);
  return cudaGetLastError();
}

}  // namespace ttkv_dev
