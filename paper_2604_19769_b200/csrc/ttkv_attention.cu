// ttkv_attention.cu -- block-wise streaming decode attention on B200.
//
// Replaces the three accumulation loops of Engine::decode_step
// (engine.cpp:36-40 fast tier, 61-83 fetched blocks, 85-86 finalize) and the
// AttentionAccumulator they drive (attention.hpp:29-61).  Every partition
// produces an online-softmax partial (acc, m in log2 units, l) and
// combine_partials merges them by LSE rescaling -- the exact merge the
// reference proves partition-invariant.
//
// Both attention kernels are the same warp-specialised pipeline:
//   * one producer warp stages tiles into a ring of shared-memory stages with
//     cp.async.bulk (TMA bulk copy) completing on an mbarrier (expect_tx), or
//     with 16-byte LDG when a layout is not 16-byte aligned;
//   * four consumer warps absorb each staged tile for all G query heads of the
//     KV head (GQA: every K/V row is read and dequantized once): lane l owns
//     channels [4l, 4l+4), QK reduces with warp shuffles, one warp per head
//     computes the tile's softmax statistics, PV accumulates in registers.
//  slow_stream_attn  tiles = the selected slow-tier records, streamed from
//                    pinned host DRAM (zero-copy PCIe) with their per-channel
//                    params from the HBM mirror; dequantization
//                    (x = code * scale + zp, quantizer.cpp:109-110) is fused
//                    into the QK / PV loads.  PCIe-bound.
//  fast_attn_partial tiles = TT consecutive tokens of the HBM ring (split at
//                    the wrap).  HBM-bound.
// Accumulation is fp32 for the fp16 ring (the north-star contract, 1e-3) and
// fp64 for the fp32 ring, which then reproduces the reference's fp64 engine
// to ~1e-15 (the reference's own lossless test demands 1e-12).
#include <math.h>

#include <type_traits>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"
#include "ttkv_dbg_stamps.cuh"

namespace ttkv_dev {

template <typename T>
using AccOf = std::conditional_t<std::is_same_v<T, float>, double, float>;

__device__ __forceinline__ float ex2(float x) { return exp2f(x); }
__device__ __forceinline__ double ex2(double x) { return exp2(x); }

template <typename A>
__device__ __forceinline__ A wsum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename A>
__device__ __forceinline__ A wmax(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// dequantized element: one fp32 FMA, or the reference's exact
// float(double(code) * scale + zp) when accumulating in fp64
template <typename Acc>
__device__ __forceinline__ Acc deq(uint32_t code, float s, float z);
template <>
__device__ __forceinline__ float deq<float>(uint32_t code, float s, float z) {
  return fmaf((float)code, s, z);
}
template <>
__device__ __forceinline__ double deq<double>(uint32_t code, float s, float z) {
  return (double)__double2float_rn(__dadd_rn(__dmul_rn((double)code, (double)s), (double)z));
}

// Channels [c0, c0+4) of row t of one staged tensor.
// KB: 8 / 4 packed fast paths (d % 4 == 0), 16 = raw ring elements T,
//     0 = runtime width `bits` (2..8 packed LSB-first, or 16 raw).
template <int KB, typename T, typename Acc>
__device__ __forceinline__ void row4(const uint8_t* pay, uint32_t t, uint32_t c0, uint32_t dim,
                                     uint32_t bits, const float (&sc)[4], const float (&zp)[4],
                                     Acc (&o)[4]) {
  if constexpr (KB == 8) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(pay + t * dim + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = deq<Acc>((w >> (8 * j)) & 0xffu, sc[j], zp[j]);
  } else if constexpr (KB == 4) {
    const uint32_t w = *reinterpret_cast<const uint16_t*>(pay + ((t * dim + c0) >> 1));
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = deq<Acc>((w >> (4 * j)) & 0xfu, sc[j], zp[j]);
  } else {
    if (KB == 16 || bits == 16) {
      const T* e = reinterpret_cast<const T*>(pay) + (uint64_t)t * dim;
      if ((dim & 3) == 0 && c0 < dim) {
        float f[4];
        load4(e + c0, f);
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = (Acc)f[j];
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = c0 + j < dim ? (Acc)to_f(e[c0 + j]) : Acc(0);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = c0 + j < dim ? deq<Acc>(extract_code(pay, t * dim + c0 + j, bits), sc[j], zp[j])
                            : Acc(0);
    }
  }
}

// Per-CTA consumer state shared through smem.
template <typename Acc>
struct ConsumerSmem {
  Acc* sc;   // [2][GT][rows_cap] scores / probabilities (double-buffered)
  Acc* mst;  // [GT] running max (log2 units)
  Acc* lst;  // [GT] running denominator
  Acc* ast;  // [GT] rescale factor of the current tile
};

struct TileView {
  const uint8_t* kpay;
  const uint8_t* vpay;
  const float* kpar;  // {scale, zp} x d_k or nullptr (raw)
  const float* vpar;
  uint32_t rows;
};

// Absorb one staged tile for the heads in `hm` (engine.cpp:61-83 per block,
// attention.hpp:29-50 per row, vectorised).  Called by all consumer warps.
template <typename T, typename Acc, int KB, int VB, int GT>
__device__ __forceinline__ void absorb_tile(const Geometry& g, const TileView& tv, uint32_t hm,
                                            uint32_t it, uint32_t rows_cap, bool literal,
                                            const Acc (&qr)[GT][4], Acc (&acc)[GT][4],
                                            const ConsumerSmem<Acc>& cs, uint32_t cw,
                                            uint32_t lane) {
  const uint32_t c0 = lane * 4;
  const int nthreads_c = kSlowConsumerWarps * 32;
  Acc* scb = cs.sc + (it & 1) * GT * rows_cap;

  // ---- QK: all heads share each (dequantized) key row ----
  {
    float ks[4], kz[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = tv.kpar && c0 + j < g.d_k;
      ks[j] = ok ? tv.kpar[2 * (c0 + j)] : 0.0f;
      kz[j] = ok ? tv.kpar[2 * (c0 + j) + 1] : 0.0f;
    }
    for (uint32_t t = cw; t < tv.rows; t += kSlowConsumerWarps) {
      Acc kf[4];
      if (c0 < g.d_k) row4<KB, T, Acc>(tv.kpay, t, c0, g.d_k, g.kb, ks, kz, kf);
      else kf[0] = kf[1] = kf[2] = kf[3] = Acc(0);
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        if (h >= (int)g.G) break;
        if (!((hm >> h) & 1u)) continue;
        Acc d = qr[h][0] * kf[0] + qr[h][1] * kf[1] + qr[h][2] * kf[2] + qr[h][3] * kf[3];
        d = wsum(d);
        if (lane == 0) scb[h * rows_cap + t] = d;
      }
    }
  }
  named_bar(1, nthreads_c);

  // ---- tile softmax statistics, one warp per head ----
  for (uint32_t h = cw; h < g.G; h += kSlowConsumerWarps) {
    if (!((hm >> h) & 1u)) {
      if (lane == 0) cs.ast[h] = Acc(1);
      continue;
    }
    Acc* row = scb + h * rows_cap;
    Acc bm = -INFINITY;
    for (uint32_t t = lane; t < tv.rows; t += 32) bm = fmax(bm, row[t]);
    bm = wmax(bm);
    const Acc m_old = cs.mst[h];
    const Acc m_new = literal ? bm : fmax(m_old, bm);
    Acc sum = 0;
    for (uint32_t t = lane; t < tv.rows; t += 32) {
      const Acc p = ex2(row[t] - m_new);
      row[t] = p;
      sum += p;
    }
    sum = wsum(sum);
    __syncwarp();
    if (literal) {
      // literal additive merge (engine.cpp:67-72): each block is its own
      // normalized partition, summed without rescaling
      const Acc inv = Acc(1) / sum;
      for (uint32_t t = lane; t < tv.rows; t += 32) row[t] *= inv;
      if (lane == 0) cs.ast[h] = Acc(1);
      continue;
    }
    if (lane == 0) {
      const Acc alpha = ex2(m_old - m_new);  // 0 when m_old = -inf
      cs.lst[h] = cs.lst[h] * alpha + sum;
      cs.mst[h] = m_new;
      cs.ast[h] = alpha;
    }
  }
  named_bar(1, nthreads_c);

  // ---- PV: all heads share each (dequantized) value row ----
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    if (h >= (int)g.G) break;
    if (!((hm >> h) & 1u)) continue;
    const Acc alpha = cs.ast[h];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[h][j] *= alpha;
  }
  float vs[4], vz[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool ok = tv.vpar && c0 + j < g.d_v;
    vs[j] = ok ? tv.vpar[2 * (c0 + j)] : 0.0f;
    vz[j] = ok ? tv.vpar[2 * (c0 + j) + 1] : 0.0f;
  }
  for (uint32_t t = cw; t < tv.rows; t += kSlowConsumerWarps) {
    Acc vf[4];
    if (c0 < g.d_v) row4<VB, T, Acc>(tv.vpay, t, c0, g.d_v, g.vb, vs, vz, vf);
    else vf[0] = vf[1] = vf[2] = vf[3] = Acc(0);
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      if (h >= (int)g.G) break;
      if (!((hm >> h) & 1u)) continue;
      const Acc p = scb[h * rows_cap + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[h][j] += p * vf[j];
    }
  }
}

// Merge the consumer warps' accumulators and emit one (acc, m, l) partial per
// head; heads that absorbed nothing emit (0, -inf, 0).
template <typename Acc, int GT>
__device__ __forceinline__ void emit_partial(const Geometry& g, Acc (&acc)[GT][4], uint8_t* red_smem,
                                             const ConsumerSmem<Acc>& cs, uint32_t seen,
                                             bool literal, Acc* part, uint64_t part_stride_head,
                                             uint32_t cw, uint32_t lane) {
  const int nthreads_c = kSlowConsumerWarps * 32;
  const uint32_t c0 = lane * 4;
  named_bar(1, nthreads_c);
  Acc* red = reinterpret_cast<Acc*>(red_smem);
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    if (h >= (int)g.G) break;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c0 + j < g.d_v) red[(cw * GT + h) * g.d_v + c0 + j] = acc[h][j];
  }
  named_bar(1, nthreads_c);
  const uint32_t ct = cw * 32 + lane;
  for (uint32_t i = ct; i < g.G * g.d_v; i += nthreads_c) {
    const uint32_t h = i / g.d_v, c = i % g.d_v;
    Acc A = 0;
    for (int w = 0; w < kSlowConsumerWarps; ++w) A += red[(w * GT + h) * g.d_v + c];
    Acc* p = part + h * part_stride_head;
    const bool any = (seen >> h) & 1u;
    p[c] = any ? A : Acc(0);
    if (c == 0) {
      p[g.d_v] = any ? (literal ? Acc(0) : cs.mst[h]) : Acc(-INFINITY);
      p[g.d_v + 1] = any ? (literal ? Acc(1) : cs.lst[h]) : Acc(0);
    }
  }
}

template <typename Acc, int GT>
__device__ __forceinline__ void load_query(const Geometry& g, const float* q, uint32_t s,
                                           double scale_log2, uint32_t lane, Acc (&qr)[GT][4]) {
  const uint32_t c0 = lane * 4;
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      qr[h][j] = (h < (int)g.G && c0 + j < g.d_k)
                     ? (Acc)q[((uint64_t)s * g.G + h) * g.d_k + c0 + j] * (Acc)scale_log2
                     : Acc(0);
}

// smem carve-up shared by both kernels
template <typename Acc, int GT>
struct Carve {
  uint8_t* stages;
  uint64_t* full;
  uint64_t* empty;
  ConsumerSmem<Acc> cs;
  __device__ Carve(uint8_t* smem, uint32_t stage_region, uint32_t NS, uint32_t rows_cap) {
    stages = smem;
    full = reinterpret_cast<uint64_t*>(smem + stage_region);
    empty = full + NS;
    cs.sc = reinterpret_cast<Acc*>(empty + NS);
    cs.mst = cs.sc + 2 * GT * rows_cap;
    cs.lst = cs.mst + GT;
    cs.ast = cs.lst + GT;
  }
};

template <typename Acc, int GT>
__device__ __forceinline__ void init_pipeline(Carve<Acc, GT>& cv, uint32_t NS) {
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < NS; ++i) {
      mbar_init(&cv.full[i], 1);
      mbar_init(&cv.empty[i], kSlowConsumerWarps);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < GT) {
    cv.cs.mst[threadIdx.x] = -INFINITY;
    cv.cs.lst[threadIdx.x] = 0;
    cv.cs.ast[threadIdx.x] = 1;
  }
  __syncthreads();
}

// 16-byte LDG copy by one warp (fallback staging path)
__device__ __forceinline__ void warp_copy16(uint8_t* dst, const uint8_t* src, uint32_t bytes,
                                           uint32_t lane) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  const uint32_t n16 = bytes >> 4;
  uint32_t j = lane;
  for (; j + 7 * 32 < n16; j += 8 * 32) {
    uint4 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) r[u] = s4[j + u * 32];
#pragma unroll
    for (int u = 0; u < 8; ++u) d4[j + u * 32] = r[u];
  }
  for (; j < n16; j += 32) d4[j] = s4[j];
}

// element-granular warp copy for layouts that are not 16-byte aligned
__device__ __forceinline__ void warp_copy_any(uint8_t* dst, const uint8_t* src, uint32_t bytes,
                                              uint32_t lane) {
  for (uint32_t j = lane * 2; j < bytes; j += 64)
    *reinterpret_cast<uint16_t*>(dst + j) = *reinterpret_cast<const uint16_t*>(src + j);
}

// ---------------------------------------------------------------------------
// slow tier
// ---------------------------------------------------------------------------
template <typename T, int KB, int VB, int GT, int COPY>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32) slow_attn_kernel(SlowArgs a) {
  using Acc = AccOf<T>;
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, chunk = blockIdx.x;
  const uint32_t cnt = a.union_count[s];
  const uint32_t i0 = chunk * a.CH;
  if (i0 >= cnt) return;  // uniform across the CTA
  const uint32_t nb = min(i0 + a.CH, cnt) - i0;
  const uint32_t NS = a.stages;
  const uint32_t stride = g.rec.stride;

  extern __shared__ __align__(1024) uint8_t smem[];
  Carve<Acc, GT> cv(smem, a.stage_region, NS, g.B);
  init_pipeline(cv, NS);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t* uids = a.union_ids + (uint64_t)s * g.n_cap + i0;
  const uint32_t* umask = a.union_mask + (uint64_t)s * g.n_cap + i0;

  if (warp == 0) {
    // ---- producer: payload over PCIe (zero-copy), params from HBM ----
    const uint8_t* arena_s = a.arena + (uint64_t)s * g.n_cap * stride;
    const uint32_t pay = g.rec.kp_off, pbytes = g.rec.used - g.rec.kp_off;
    for (uint32_t i = 0; i < nb; ++i) {
      const uint32_t st = i % NS;
      if (i >= NS) mbar_wait(&cv.empty[st], ((i / NS) - 1) & 1);
      const uint32_t blk = uids[i];
      const uint8_t* src = arena_s + (uint64_t)blk * stride;
      const uint8_t* psrc = a.params + ((uint64_t)s * g.n_cap + blk) * pbytes;
      uint8_t* dst = cv.stages + st * stride;
      if constexpr (COPY == 1) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&cv.full[st], g.rec.used);
          for (uint32_t off = 0; off < pay; off += 16384u)
            bulk_g2s(dst + off, src + off, min(16384u, pay - off), &cv.full[st]);
          if (pbytes) bulk_g2s(dst + pay, psrc, pbytes, &cv.full[st]);
        }
      } else {
        warp_copy16(dst, src, pay, lane);
        warp_copy16(dst + pay, psrc, pbytes, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&cv.full[st]);
      }
    }
    return;
  }

  // ---- consumers ----
  const uint32_t cw = warp - 1;
  Acc qr[GT][4], acc[GT][4];
  load_query<Acc, GT>(g, a.q, s, a.scale_log2, lane, qr);
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[h][j] = 0;
  uint32_t seen = 0;
  for (uint32_t i = 0; i < nb; ++i) {
    const uint32_t st = i % NS;
    mbar_wait(&cv.full[st], (i / NS) & 1);
    const uint8_t* rec = cv.stages + st * stride;
    const uint32_t hm = umask[i];
    seen |= hm;
    TileView tv;
    tv.kpay = rec;
    tv.vpay = rec + g.rec.v_off;
    tv.kpar = g.kb == 16 ? nullptr : reinterpret_cast<const float*>(rec + g.rec.kp_off);
    tv.vpar = g.vb == 16 ? nullptr : reinterpret_cast<const float*>(rec + g.rec.vp_off);
    tv.rows = g.B;
    absorb_tile<T, Acc, KB, VB, GT>(g, tv, hm, i, g.B, a.literal != 0, qr, acc, cv.cs, cw, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&cv.empty[st]);
  }
  Acc* part = reinterpret_cast<Acc*>(a.part) +
              (((uint64_t)s * g.G) * a.nsc + chunk) * (g.d_v + 2);
  emit_partial<Acc, GT>(g, acc, cv.stages, cv.cs, seen, a.literal != 0, part,
                        (uint64_t)a.nsc * (g.d_v + 2), cw, lane);
}

// ---------------------------------------------------------------------------
// fast tier
// ---------------------------------------------------------------------------
template <typename T, int GT, int COPY>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32) fast_attn_kernel(FastArgs a) {
  using Acc = AccOf<T>;
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, f = blockIdx.x;
  const uint32_t F = a.pos ? (uint32_t)(*a.pos + 1 - a.front) : a.F;
  const uint32_t t0 = f * a.FC;
  const uint32_t t1 = min(t0 + a.FC, F);
  const uint32_t ntiles = t1 > t0 ? (t1 - t0 + a.TT - 1) / a.TT : 0;
  const uint32_t NS = a.stages;
  const uint32_t kbytes_row = g.d_k * sizeof(T), vbytes_row = g.d_v * sizeof(T);
  const uint32_t stage_bytes = a.TT * (kbytes_row + vbytes_row);

  extern __shared__ __align__(1024) uint8_t smem[];
  Carve<Acc, GT> cv(smem, a.stage_region, NS, a.TT);
  init_pipeline(cv, NS);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint8_t* rk = static_cast<const uint8_t*>(a.ring_k) + (uint64_t)s * g.C * kbytes_row;
  const uint8_t* rv = static_cast<const uint8_t*>(a.ring_v) + (uint64_t)s * g.C * vbytes_row;

  if (warp == 0) {
    // ---- producer: ring rows (split at the wrap) -> stage ----
    for (uint32_t i = 0; i < ntiles; ++i) {
      const uint32_t st = i % NS;
      if (i >= NS) mbar_wait(&cv.empty[st], ((i / NS) - 1) & 1);
      const uint32_t tt0 = t0 + i * a.TT;
      const uint32_t rows = min(a.TT, t1 - tt0);
      const uint64_t slot0 = (a.front + tt0) % g.C;
      const uint64_t room = g.C - slot0;
      const uint32_t n1 = room < rows ? (uint32_t)room : rows, n2 = rows - n1;
      uint8_t* dk = cv.stages + st * stage_bytes;
      uint8_t* dv = dk + a.TT * kbytes_row;
      if constexpr (COPY == 1) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&cv.full[st], rows * (kbytes_row + vbytes_row));
          bulk_g2s(dk, rk + slot0 * kbytes_row, n1 * kbytes_row, &cv.full[st]);
          bulk_g2s(dv, rv + slot0 * vbytes_row, n1 * vbytes_row, &cv.full[st]);
          if (n2) {
            bulk_g2s(dk + n1 * kbytes_row, rk, n2 * kbytes_row, &cv.full[st]);
            bulk_g2s(dv + n1 * vbytes_row, rv, n2 * vbytes_row, &cv.full[st]);
          }
        }
      } else {
        warp_copy_any(dk, rk + slot0 * kbytes_row, n1 * kbytes_row, lane);
        warp_copy_any(dv, rv + slot0 * vbytes_row, n1 * vbytes_row, lane);
        if (n2) {
          warp_copy_any(dk + n1 * kbytes_row, rk, n2 * kbytes_row, lane);
          warp_copy_any(dv + n1 * vbytes_row, rv, n2 * vbytes_row, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&cv.full[st]);
      }
    }
    return;
  }

  const uint32_t cw = warp - 1;
  Acc qr[GT][4], acc[GT][4];
  load_query<Acc, GT>(g, a.q, s, a.scale_log2, lane, qr);
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[h][j] = 0;
  const uint32_t all = (1u << g.G) - 1u;
  for (uint32_t i = 0; i < ntiles; ++i) {
    const uint32_t st = i % NS;
    mbar_wait(&cv.full[st], (i / NS) & 1);
    TileView tv;
    tv.kpay = cv.stages + st * stage_bytes;
    tv.vpay = tv.kpay + a.TT * kbytes_row;
    tv.kpar = tv.vpar = nullptr;
    tv.rows = min(a.TT, t1 - (t0 + i * a.TT));
    absorb_tile<T, Acc, 16, 16, GT>(g, tv, all, i, a.TT, false, qr, acc, cv.cs, cw, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&cv.empty[st]);
  }
  Acc* part = reinterpret_cast<Acc*>(a.part) + (((uint64_t)s * g.G) * a.nfc + f) * (g.d_v + 2);
  emit_partial<Acc, GT>(g, acc, cv.stages, cv.cs, ntiles ? all : 0u, false, part,
                        (uint64_t)a.nfc * (g.d_v + 2), cw, lane);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static size_t consumer_smem(const Geometry& g, uint32_t GT, uint32_t rows_cap, size_t acc) {
  return (size_t)2 * GT * rows_cap * acc + 3 * GT * acc + 64;
}
static size_t acc_bytes(const Geometry& g) { return g.elem == 4 ? 8 : 4; }

uint32_t slow_stages_for(const Geometry& g) {
  const size_t budget = 110 * 1024;  // two CTAs per SM
  const size_t fixed = consumer_smem(g, kMaxG, g.B, acc_bytes(g));
  size_t ns = budget > fixed ? (budget - fixed) / (g.rec.stride + 16) : 0;
  if (ns > 4) ns = 4;
  if (ns < 1) {  // large records: one CTA per SM
    const size_t big = 220 * 1024;
    ns = big > fixed ? (big - fixed) / (g.rec.stride + 16) : 0;
    if (ns > 2) ns = 2;
  }
  return (uint32_t)ns;
}

uint32_t fast_tile_rows(const Geometry& g) {
  const uint32_t row = (g.d_k + g.d_v) * g.elem;
  uint32_t tt = 32768u / row;
  tt = tt > 128 ? 128 : tt;
  tt = tt < 16 ? 16 : (tt / 16) * 16;
  return tt;
}

template <typename Acc>
static uint32_t stage_region_for(size_t stage_total, uint32_t GT, const Geometry& g) {
  const size_t red = (size_t)kSlowConsumerWarps * GT * g.d_v * sizeof(Acc);
  size_t r = stage_total > red ? stage_total : red;
  return (uint32_t)((r + 15) & ~size_t(15));
}

template <typename T, int KB, int VB, int GT, int COPY>
static cudaError_t launch_slow_t(const SlowArgs& a, uint32_t grid_chunks, cudaStream_t st) {
  using Acc = AccOf<T>;
  const Geometry& g = a.g;
  SlowArgs b = a;
  b.stage_region = stage_region_for<Acc>((size_t)a.stages * g.rec.stride, GT, g);
  const size_t smem = (size_t)b.stage_region + 16 * a.stages + consumer_smem(g, GT, g.B, sizeof(Acc));
  auto kern = slow_attn_kernel<T, KB, VB, GT, COPY>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(grid_chunks, g.S);
  kern<<<grid, 32 + kSlowConsumerWarps * 32, smem, st>>>(b);
  return cudaGetLastError();
}

template <typename T, int KB, int VB, int COPY>
static cudaError_t launch_slow_g(const SlowArgs& a, uint32_t gc, cudaStream_t st) {
  if (a.g.G <= 1) return launch_slow_t<T, KB, VB, 1, COPY>(a, gc, st);
  if (a.g.G <= 2) return launch_slow_t<T, KB, VB, 2, COPY>(a, gc, st);
  if (a.g.G <= 4) return launch_slow_t<T, KB, VB, 4, COPY>(a, gc, st);
  return launch_slow_t<T, KB, VB, 8, COPY>(a, gc, st);
}

template <typename T, int COPY>
static cudaError_t launch_slow_bits(const SlowArgs& a, uint32_t gc, cudaStream_t st) {
  const Geometry& g = a.g;
  const bool vec = (g.d_k % 4 == 0) && (g.d_v % 4 == 0);
  if (vec && g.kb == 8 && g.vb == 4) return launch_slow_g<T, 8, 4, COPY>(a, gc, st);
  if (vec && g.kb == 8 && g.vb == 8) return launch_slow_g<T, 8, 8, COPY>(a, gc, st);
  return launch_slow_g<T, 0, 0, COPY>(a, gc, st);
}

cudaError_t launch_slow(const SlowArgs& a, uint32_t grid_chunks, int copy_mode, cudaStream_t st) {
  if (grid_chunks == 0) return cudaSuccess;
  if (a.g.elem == 2)
    return copy_mode == 2 ? launch_slow_bits<__half, 2>(a, grid_chunks, st)
                          : launch_slow_bits<__half, 1>(a, grid_chunks, st);
  return copy_mode == 2 ? launch_slow_bits<float, 2>(a, grid_chunks, st)
                        : launch_slow_bits<float, 1>(a, grid_chunks, st);
}

template <typename T, int GT, int COPY>
static cudaError_t launch_fast_t(const FastArgs& a, cudaStream_t st) {
  using Acc = AccOf<T>;
  const Geometry& g = a.g;
  FastArgs b = a;
  const size_t stage_bytes = (size_t)a.TT * (g.d_k + g.d_v) * sizeof(T);
  b.stage_region = stage_region_for<Acc>(stage_bytes * a.stages, GT, g);
  const size_t smem = (size_t)b.stage_region + 16 * a.stages + consumer_smem(g, GT, a.TT, sizeof(Acc));
  auto kern = fast_attn_kernel<T, GT, COPY>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nfc, g.S);
  return launch_background(kern, grid, dim3(32 + kSlowConsumerWarps * 32), smem, st, b);
}

template <typename T, int COPY>
static cudaError_t launch_fast_g(const FastArgs& a, cudaStream_t st) {
  if (a.g.G <= 1) return launch_fast_t<T, 1, COPY>(a, st);
  if (a.g.G <= 2) return launch_fast_t<T, 2, COPY>(a, st);
  if (a.g.G <= 4) return launch_fast_t<T, 4, COPY>(a, st);
  return launch_fast_t<T, 8, COPY>(a, st);
}

cudaError_t launch_fast(const FastArgs& a, cudaStream_t st) {
  const Geometry& g = a.g;
  // bulk copies need 16-byte aligned ring rows
  const bool aligned = ((g.d_k * g.elem) % 16 == 0) && ((g.d_v * g.elem) % 16 == 0);
  if (g.elem == 2) return aligned ? launch_fast_g<__half, 1>(a, st) : launch_fast_g<__half, 2>(a, st);
  return aligned ? launch_fast_g<float, 1>(a, st) : launch_fast_g<float, 2>(a, st);
}

// ---------------------------------------------------------------------------
// combine (attention.hpp:54-61)
// ---------------------------------------------------------------------------
// One CTA per (stream, head): weights w_i = exp2(m_i - M) of every partial
// are computed once into smem, then each thread reduces one output channel.
// Device-side join with the fast tier (CombineArgs::fast_epoch): wait until
// the fast tier's epoch passes this combine's.  The fast tier of the step
// was launched before the combine and never waits on it, so the wait ends;
// a broken invariant (a step whose fast tier was never launched) traps after
// ~2 s -- the context reports an error -- instead of hanging the device.
__device__ __forceinline__ void wait_fast_epoch(const CombineArgs& a) {
  const uint32_t target = *reinterpret_cast<volatile const uint32_t*>(a.comb_epoch) + 1u;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.fast_epoch) : "memory");
    if ((int32_t)(v - target) >= 0) return;
    __nanosleep(64);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) __trap();
  }
}

constexpr int kCombineWarps = 8;
#ifdef TTKV_STAMPS
TTKV_DBG_TABLE(comb)
TTKV_DBG_READER(comb)
#endif
template <typename Acc>
__global__ void __launch_bounds__(kCombineWarps * 32) combine_kernel(CombineArgs a) {
  TTKV_DBG_STAMP(comb, 0);
  pdl_wait();  // the slow partials (the fast tier joins through an event or below)
  if (a.fast_epoch) {  // device-side join with the fast tier (other stream)
    if (threadIdx.x == 0) wait_fast_epoch(a);
    __syncthreads();
  }
  TTKV_DBG_STAMP(comb, 1);
  // the next kernel may get resident now: the next step's selection stages
  // its centroids while this combine runs (it reads q only after its wait)
  pdl_trigger();
  const Geometry& g = a.g;
  const uint32_t idx = blockIdx.x;  // s * G + head
  const uint32_t s = idx / g.G;
  const uint32_t pitch = g.d_v + 2;
  double* const out = a.out_ref ? *a.out_ref : a.out;
  const uint32_t nsc_used = !a.union_count         ? 0u
                            : a.union_count[s] == 0u ? 0u
                            : a.nslots               ? a.nslots[s]
                                                     : (a.union_count[s] + a.CH - 1) / a.CH;
  const Acc* fp = reinterpret_cast<const Acc*>(a.fpart) + (uint64_t)idx * a.nfc * pitch;
  const Acc* sp = a.spart ? reinterpret_cast<const Acc*>(a.spart) + (uint64_t)idx * a.nsc * pitch
                          : nullptr;
  // literal additive merge: slow partials are already normalized sums
  const uint32_t nlse = a.literal ? 0u : nsc_used;
  const uint32_t np = a.nfc + nlse;
  extern __shared__ __align__(16) uint8_t csm[];
  Acc* w = reinterpret_cast<Acc*>(csm);  // [np]
  __shared__ Acc red[kCombineWarps];
  auto part = [&](uint32_t i) { return i < a.nfc ? fp + i * pitch : sp + (i - a.nfc) * pitch; };

  // one partial per thread (np <= blockDim: every step but the longest fast
  // tiers) keeps its (m, l) in registers across the max and the sum: one
  // round trip to L2 instead of two on the step's critical path
  const bool one = np <= blockDim.x;
  Acc m1 = -INFINITY, l1 = 0;
  if (one && threadIdx.x < np) {
    const Acc* p = part(threadIdx.x);
    m1 = p[g.d_v];
    l1 = p[g.d_v + 1];
  }
  Acc M = -INFINITY;
  if (one) {
    if (l1 > 0) M = m1;
  } else {
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
      const Acc* p = part(i);
      if (p[g.d_v + 1] > 0) M = fmax(M, p[g.d_v]);
    }
  }
  M = wmax(M);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = M;
  __syncthreads();
  M = red[0];
#pragma unroll
  for (int k = 1; k < kCombineWarps; ++k) M = fmax(M, red[k]);
  __syncthreads();
  Acc L = 0;
  if (one) {
    if (threadIdx.x < np) {
      const Acc wi = l1 > 0 ? ex2(m1 - M) : Acc(0);
      w[threadIdx.x] = wi;
      L = wi * l1;
    }
  } else {
    for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
      const Acc* p = part(i);
      const Acc wi = p[g.d_v + 1] > 0 ? ex2(p[g.d_v] - M) : Acc(0);
      w[i] = wi;
      L += wi * p[g.d_v + 1];
    }
  }
  L = wsum(L);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = L;
  __syncthreads();
  Acc Lt = 0;
#pragma unroll
  for (int k = 0; k < kCombineWarps; ++k) Lt += red[k];
  const Acc inv = Acc(1) / Lt;
  // the weighted sum over partials for this CTA's channel slice
  // [c_lo, c_hi) (blockIdx.y; several slices when S*G is small): warp w of
  // the kCombineWarps takes partials w, w + kCombineWarps, ..., lane l
  // channels c_lo + l + 32j (coalesced segments of each partial row), kU = 8
  // partial rows in flight; warps meet in smem
  const uint32_t cw = (g.d_v + gridDim.y - 1) / gridDim.y;
  const uint32_t c_lo = blockIdx.y * cw, c_hi = min(g.d_v, c_lo + cw);
  __shared__ Acc red2[kCombineWarps][kMaxD];
  {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // 8 partial rows in flight per lane (the rows come from L2 or DRAM)
    constexpr int kU = 8;
    Acc acc[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[u][j] = 0;
    uint32_t i = warp;
    for (; i + kCombineWarps * (kU - 1) < np; i += kCombineWarps * kU) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const Acc* pu = part(i + kCombineWarps * u);
        const Acc wu = w[i + kCombineWarps * u];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t c = c_lo + lane + 32 * j;
          if (c < c_hi) acc[u][j] += wu * pu[c];
        }
      }
    }
    for (; i < np; i += kCombineWarps) {
      const Acc* p0 = part(i);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t c = c_lo + lane + 32 * j;
        if (c < c_hi) acc[0][j] += w[i] * p0[c];
      }
    }
    Acc a0[4], a1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a0[j] = ((acc[0][j] + acc[1][j]) + (acc[2][j] + acc[3][j]));
      a1[j] = ((acc[4][j] + acc[5][j]) + (acc[6][j] + acc[7][j]));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = c_lo + lane + 32 * j;
      if (c < c_hi) red2[warp][c] = a0[j] + a1[j];
    }
  }
  __syncthreads();
  for (uint32_t c = c_lo + threadIdx.x; c < c_hi; c += blockDim.x) {
    Acc A = 0;
#pragma unroll
    for (int k = 0; k < kCombineWarps; ++k) A += red2[k][c];
    Acc o = A * inv;
    if (a.literal)
      for (uint32_t i = 0; i < nsc_used; ++i)
        if (sp[i * pitch + g.d_v + 1] > 0) o += sp[i * pitch + c];
    out[(uint64_t)idx * g.d_v + c] = (double)o;
    if (a.n_peers) {
      const uint64_t gi = ((uint64_t)a.gidx[s] * g.G + (idx - s * g.G)) * g.d_v + c;
      for (uint32_t r = 0; r < a.n_peers; ++r) a.peer_out[r][gi] = (double)o;
    }
  }
  // the step is combined: advance the device step position (nothing in this
  // kernel reads it; the next step's append and fast tier do)
  if (a.pos_inc && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.pos_inc += 1;
  if (a.count_out && idx == s * g.G && blockIdx.y == 0 && threadIdx.x == 0)
    a.count_out[s] = a.union_count ? a.union_count[s] : 0u;
  if (a.n_peers) {  // this CTA's row is in every rank's buffer: publish it
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (uint32_t r = 0; r < a.n_peers; ++r)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(a.peer_flags[r] + a.my_rank)
                     : "memory");
    }
  }
  if (a.fast_epoch) {  // every CTA has read *comb_epoch: the last one advances it
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(a.comb_arrive, 1u) == gridDim.x * gridDim.y - 1) {
      *a.comb_arrive = 0u;
      atomicAdd(a.comb_epoch, 1u);
    }
  }
  TTKV_DBG_END(comb);
}

// Small-step combine (fp32 partials, d_v = 128 in four 32-channel slices,
// additive merge -- one layer of a layer-sequential decode, cfg1): the
// partials' (m, l) AND this slice's values are loaded in one round trip
// (thread t: (m, l) of partial t; values of partials t/4 + 64j, channels
// c_lo + 8 (t % 4) .. + 8) before the max is known, instead of three
// dependent passes over L2; the weighted sums are reduced with warp shuffles
// and one shared-memory pass.  Partials beyond the first 256 take a second
// pass.  Same merge as combine_kernel (another summation order).
constexpr int kRow32Groups = 4;  // partial groups of 64 prefetched per thread
__global__ void __launch_bounds__(256) combine_row32_kernel(CombineArgs a) {
  TTKV_DBG_STAMP(comb, 0);
  pdl_wait();  // the slow partials
  if (a.fast_epoch) {  // device-side join with the fast tier (other stream)
    if (threadIdx.x == 0) wait_fast_epoch(a);
    __syncthreads();
  }
  TTKV_DBG_STAMP(comb, 1);
  pdl_trigger();
  const Geometry& g = a.g;
  const uint32_t idx = blockIdx.x, s = idx / g.G;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t pitch = g.d_v + 2;
  const uint32_t nsc_used = !a.union_count         ? 0u
                            : a.union_count[s] == 0u ? 0u
                            : a.nslots               ? a.nslots[s]
                                                     : (a.union_count[s] + a.CH - 1) / a.CH;
  const float* fp = reinterpret_cast<const float*>(a.fpart) + (uint64_t)idx * a.nfc * pitch;
  const float* sp = a.spart ? reinterpret_cast<const float*>(a.spart) + (uint64_t)idx * a.nsc * pitch
                            : nullptr;
  const uint32_t np = a.nfc + nsc_used;
  auto part = [&](uint32_t i) { return i < a.nfc ? fp + i * pitch : sp + (i - a.nfc) * pitch; };
  const uint32_t c0 = blockIdx.y * 32 + 8 * (t & 3);  // this thread's 8 channels
  extern __shared__ __align__(16) uint8_t csm[];
  float* w = reinterpret_cast<float*>(csm);  // [np] weights
  __shared__ float red[8];
  __shared__ float red2[8];
  __shared__ float sums[8][32];

  // ---- one round trip: (m, l) of partial t and the values of partials t/4 + 64j ----
  float m1 = -INFINITY, l1 = 0.f;
  if (t < np) {
    const float* p = part(t);
    m1 = p[g.d_v];
    l1 = p[g.d_v + 1];
  }
  float2 v[kRow32Groups][4];
#pragma unroll
  for (int j = 0; j < kRow32Groups; ++j) {
    const uint32_t pi = (t >> 2) + 64u * j;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      v[j][e] = pi < np ? *reinterpret_cast<const float2*>(part(pi) + c0 + 2 * e) : make_float2(0.f, 0.f);
  }
  // ---- block max over the partials with tokens, then the weights ----
  float M = (t < np && l1 > 0.f) ? m1 : -INFINITY;
  for (uint32_t i = t + 256; i < np; i += 256) {  // beyond 256 partials
    const float* p = part(i);
    if (p[g.d_v + 1] > 0.f) M = fmaxf(M, p[g.d_v]);
  }
  M = wmax(M);
  if (lane == 0) red[warp] = M;
  __syncthreads();
  M = red[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) M = fmaxf(M, red[k]);
  float L = 0.f;
  if (t < np) {
    const float wi = l1 > 0.f ? ex2(m1 - M) : 0.f;
    w[t] = wi;
    L = wi * l1;
  }
  for (uint32_t i = t + 256; i < np; i += 256) {
    const float* p = part(i);
    const float wi = p[g.d_v + 1] > 0.f ? ex2(p[g.d_v] - M) : 0.f;
    w[i] = wi;
    L += wi * p[g.d_v + 1];
  }
  L = wsum(L);
  if (lane == 0) red2[warp] = L;
  __syncthreads();  // w[] and the L partials are visible
  float Lt = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) Lt += red2[k];
  // ---- weighted sum of this thread's partials, 8 channels ----
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
  for (int j = 0; j < kRow32Groups; ++j) {
    const uint32_t pi = (t >> 2) + 64u * j;
    const float wj = pi < np ? w[pi] : 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[2 * e] += wj * v[j][e].x;
      acc[2 * e + 1] += wj * v[j][e].y;
    }
  }
  for (uint32_t pi = (t >> 2) + 64u * kRow32Groups; pi < np; pi += 64) {
    const float wj = w[pi];
    const float* p = part(pi) + c0;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += wj * p[e];
  }
  // lanes with the same t % 4 hold the same channels: reduce over lane bits 2-4
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float x = acc[e];
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    x += __shfl_xor_sync(0xffffffffu, x, 8);
    x += __shfl_xor_sync(0xffffffffu, x, 16);
    acc[e] = x;
  }
  if (lane < 4) {
#pragma unroll
    for (int e = 0; e < 8; ++e) sums[warp][8 * lane + e] = acc[e];
  }
  __syncthreads();
  double* const out = a.out_ref ? *a.out_ref : a.out;
  if (t < 32) {
    float A = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) A += sums[k][t];
    const float o = A * (1.f / Lt);
    const uint32_t c = blockIdx.y * 32 + t;
    out[(uint64_t)idx * g.d_v + c] = (double)o;
    if (a.n_peers) {
      const uint64_t gi = ((uint64_t)a.gidx[s] * g.G + (idx - s * g.G)) * g.d_v + c;
      for (uint32_t r = 0; r < a.n_peers; ++r) a.peer_out[r][gi] = (double)o;
    }
  }
  if (a.pos_inc && blockIdx.x == 0 && blockIdx.y == 0 && t == 0) *a.pos_inc += 1;
  if (a.count_out && idx == s * g.G && blockIdx.y == 0 && t == 0)
    a.count_out[s] = a.union_count ? a.union_count[s] : 0u;
  if (a.n_peers) {
    __syncthreads();
    if (t == 0) {
      __threadfence_system();
      for (uint32_t r = 0; r < a.n_peers; ++r)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(a.peer_flags[r] + a.my_rank)
                     : "memory");
    }
  }
  if (a.fast_epoch) {
    __syncthreads();
    if (t == 0 && atomicAdd(a.comb_arrive, 1u) == gridDim.x * gridDim.y - 1) {
      *a.comb_arrive = 0u;
      atomicAdd(a.comb_epoch, 1u);
    }
  }
  TTKV_DBG_END(comb);
}

// Combine of the speculative record stream (slow_attn_tc_spec_kernel): the
// slow partials are per-record rows rpart[s][h][b] and head h merges exactly
// the records it selected -- the union entries with its bit set.  One CTA per
// (stream, head, 32-channel slice); three short phases, each one round trip
// to L2 deep:
//   1. compaction: thread t tests a contiguous run of union entries, a CTA
//      scan places the selected block ids (union order, ascending block id:
//      deterministic, so the merge is bit-reproducible);
//   2. weights: every fast-tier and selected-record row's (m, l) -> M, then
//      w_i = exp2(m_i - M) and L = sum w_i l_i;
//   3. weighted sum: 32 row groups x 8 float4 channel lanes, reduced in smem.
// fp32 (the tensor-core slow tier is the fp16 ring's); d_v = 128.
constexpr int kSpecCombineThreads = 256;
__global__ void __launch_bounds__(kSpecCombineThreads) combine_spec_kernel(CombineArgs a) {
  pdl_wait();  // the record stream (which itself waited for the selection)
  pdl_trigger();
  const Geometry& g = a.g;
  const uint32_t idx = blockIdx.x, s = idx / g.G, h = idx - s * g.G;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t cap = a.nfc + a.spec_n;
  double* const out = a.out_ref ? *a.out_ref : a.out;
  extern __shared__ __align__(16) uint8_t csm[];
  float* wv = reinterpret_cast<float*>(csm);  // [cap] weights
  float* lv = wv + cap;                       // [cap] l of each row
  uint32_t* ids = reinterpret_cast<uint32_t*>(lv + cap);  // [spec_n] selected block ids
  __shared__ uint32_t redu[kSpecCombineThreads / 32];
  __shared__ float redf[kSpecCombineThreads / 32];
  __shared__ float acc_sm[32][33];

  // ---- 1. this head's selected records ----
  const uint32_t cnt = a.union_count[s];
  const uint64_t ub = (uint64_t)s * a.n_cap;
  const uint32_t E = (cnt + kSpecCombineThreads - 1) / kSpecCombineThreads;  // <= 8 (n <= 2048)
  const uint32_t u0 = min(cnt, t * E), ne = min(cnt, u0 + E) - u0;
  uint32_t sel = 0;
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j)
    if (j < ne) sel |= ((a.union_mask[ub + u0 + j] >> h) & 1u) << j;
  const uint32_t mine = __popc(sel);
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  if (lane == 31) redu[warp] = incl;
  __syncthreads();
  uint32_t pos = incl - mine, nsel = 0;
#pragma unroll
  for (int k = 0; k < kSpecCombineThreads / 32; ++k) {
    pos += (uint32_t)k < warp ? redu[k] : 0u;
    nsel += redu[k];
  }
#pragma unroll
  for (uint32_t j = 0; j < 8; ++j)
    if ((sel >> j) & 1u) ids[pos++] = a.union_ids[ub + u0 + j];
  __syncthreads();

  // ---- 2. weights ----
  const uint32_t fpitch = g.d_v + 2, np = a.nfc + nsel;
  const float* fp = reinterpret_cast<const float*>(a.fpart) + (uint64_t)idx * a.nfc * fpitch;
  const float* rp = a.rpart + (uint64_t)idx * a.n_cap * kSpecPitch;
  auto row = [&](uint32_t i) -> const float* {
    return i < a.nfc ? fp + (uint64_t)i * fpitch : rp + (uint64_t)ids[i - a.nfc] * kSpecPitch;
  };
  float M = -INFINITY;
  for (uint32_t i = t; i < np; i += kSpecCombineThreads) {
    const float* r = row(i) + g.d_v;
    const float m = r[0], l = r[1];
    wv[i] = m;
    lv[i] = l;
    if (l > 0.f) M = fmaxf(M, m);
  }
  M = warp_max(M);
  if (lane == 0) redf[warp] = M;
  __syncthreads();
  M = redf[0];
#pragma unroll
  for (int k = 1; k < kSpecCombineThreads / 32; ++k) M = fmaxf(M, redf[k]);
  __syncthreads();
  float L = 0.f;
  for (uint32_t i = t; i < np; i += kSpecCombineThreads) {
    const float wi = lv[i] > 0.f ? exp2f(wv[i] - M) : 0.f;
    wv[i] = wi;
    L += wi * lv[i];
  }
  L = warp_sum(L);
  if (lane == 0) redf[warp] = L;
  __syncthreads();  // also publishes wv
  float Lt = 0.f;
#pragma unroll
  for (int k = 0; k < kSpecCombineThreads / 32; ++k) Lt += redf[k];

  // ---- 3. weighted sum over this CTA's 32 channels ----
  const uint32_t rg = t >> 3, c4 = t & 7;
  const uint32_t c = blockIdx.y * 32 + 4 * c4;
  float4 A0 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t i = rg;
  for (; i < a.nfc && i < np; i += 32) {  // fast-tier rows (pitch d_v + 2: 8-byte aligned)
    const float* r = fp + (uint64_t)i * fpitch + c;
    const float2 x = *reinterpret_cast<const float2*>(r), y = *reinterpret_cast<const float2*>(r + 2);
    const float wi = wv[i];
    A0.x += wi * x.x; A0.y += wi * x.y; A0.z += wi * y.x; A0.w += wi * y.y;
  }
  // record rows, kU in flight per thread (one L2 round trip per kU rows)
  constexpr int kU = 8;
  for (; i < np; i += 32 * kU) {
    float4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t j = i + 32 * u;
      x[u] = j < np ? *reinterpret_cast<const float4*>(row(j) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t j = i + 32 * u;
      const float wx = j < np ? wv[j] : 0.f;
      A0.x += wx * x[u].x; A0.y += wx * x[u].y; A0.z += wx * x[u].z; A0.w += wx * x[u].w;
    }
  }
  acc_sm[rg][4 * c4 + 0] = A0.x;
  acc_sm[rg][4 * c4 + 1] = A0.y;
  acc_sm[rg][4 * c4 + 2] = A0.z;
  acc_sm[rg][4 * c4 + 3] = A0.w;
  __syncthreads();
  if (t < 32) {
    float A = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) A += acc_sm[k][t];
    const uint32_t ch = blockIdx.y * 32 + t;
    const double o = (double)(A / Lt);
    out[(uint64_t)idx * g.d_v + ch] = o;
    if (a.n_peers) {
      const uint64_t gi = ((uint64_t)a.gidx[s] * g.G + h) * g.d_v + ch;
      for (uint32_t r = 0; r < a.n_peers; ++r) a.peer_out[r][gi] = o;
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && t == 0) {
    if (a.pos_inc) *a.pos_inc += 1;
    *a.spec_ctr = 0;  // the record queue is drained (this grid waited on its kernel)
  }
  if (a.count_out && h == 0 && blockIdx.y == 0 && t == 0)
    a.count_out[s] = a.union_count ? a.union_count[s] : 0u;
  if (a.n_peers) {  // this CTA's row slice is in every rank's buffer: publish it
    __syncthreads();
    if (t == 0) {
      __threadfence_system();
      for (uint32_t r = 0; r < a.n_peers; ++r)
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(a.peer_flags[r] + a.my_rank)
                     : "memory");
    }
  }
}

__global__ void peer_wait_kernel(const unsigned long long* flags, uint32_t n_ranks,
                                 unsigned long long target, int* status) {
  const uint32_t r = threadIdx.x;
  if (r >= n_ranks) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
    if (v >= target) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) {  // a rank never arrived: fail instead of hanging
      atomicExch(status, 1);
      return;
    }
    __nanosleep(256);
  }
}

cudaError_t launch_peer_wait(const unsigned long long* flags, uint32_t n_ranks,
                             unsigned long long target, int* status, cudaStream_t st) {
  peer_wait_kernel<<<1, 32, 0, st>>>(flags, n_ranks, target, status);
  return cudaGetLastError();
}

// channel slices per (stream, head): enough CTAs to keep the combine from
// being latency-bound when S*G is small (one layer of a layer-sequential step)
// TTKV_COMBINE_ROW32=0: the three-pass combine_kernel for small steps too (measurement)
static bool row32_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TTKV_COMBINE_ROW32");
    return !(e && e[0] == '0');
  }();
  return on;
}

uint32_t combine_slices(const Geometry& g) {
  const uint32_t rows = g.S * g.G;
  if (rows >= 256 || g.d_v <= 32) return 1;
  return (g.d_v + 31) / 32;
}

uint32_t combine_slices(const CombineArgs& a) {
  return a.rpart ? (a.g.d_v + 31) / 32 : combine_slices(a.g);
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  if (a.rpart) {  // speculative record stream (fp32, d_v = 128)
    const size_t smem = (size_t)(a.nfc + a.spec_n) * 8 + (size_t)a.spec_n * 4;
    cudaFuncSetAttribute(combine_spec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return launch_chained(combine_spec_kernel, dim3(a.g.S * a.g.G, combine_slices(a)),
                          dim3(kSpecCombineThreads), smem, st, a);
  }
  const size_t acc = a.g.elem == 4 ? 8 : 4;
  const size_t smem = (size_t)(a.nfc + a.nsc + 1) * acc;
  const dim3 grid(a.g.S * a.g.G, combine_slices(a.g));
  if (a.g.elem == 4) {
    cudaFuncSetAttribute(combine_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return launch_chained(combine_kernel<double>, grid, dim3(kCombineWarps * 32), smem, st, a);
  } else if (!a.literal && a.g.d_v == 128 && combine_slices(a.g) == 4 && row32_enabled()) {
    cudaFuncSetAttribute(combine_row32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return launch_chained(combine_row32_kernel, grid, dim3(256), smem, st, a);
  } else {
    cudaFuncSetAttribute(combine_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return launch_chained(combine_kernel<float>, grid, dim3(kCombineWarps * 32), smem, st, a);
  }
}

}  // namespace ttkv_dev
