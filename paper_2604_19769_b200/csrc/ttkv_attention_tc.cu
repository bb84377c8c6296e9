// ttkv_attention_tc.cu -- tensor-core fast-tier attention (fp16 ring).
//
// fast_attn_partial for the fp16 ring when d_k = d_v in {64, 128} and the
// block size is a multiple of 64 (64-token tiles then never straddle the
// ring wrap).  Replaces engine.cpp:36-40 / attention.hpp:29-50 for the fast
// tier, like the CUDA-core kernel in ttkv_attention.cu, but:
//   * the producer loads 64-token K and V tiles with TMA tensor copies
//     (cp.async.bulk.tensor.2d, 128B swizzle) into a 3-stage smem ring;
//   * QK^T and PV run on tensor cores (mma.sync m16n8k16, f16 in, f32
//     accumulate): the M dimension carries the G <= 8 query heads of the KV
//     head, ldmatrix (swizzle-aware, conflict-free) feeds K as B and V as B^T;
//   * q and P are split into fp16 hi + lo parts (two MMAs each), so operand
//     rounding stays ~2^-22 relative: the result matches the fp32 CUDA-core
//     path well inside the 1e-3 contract;
//   * each consumer warp owns a quarter of the output channels, so PV needs
//     no cross-warp reduction; online-softmax statistics are per 64-token tile.
// HBM-bound: F * (d_k + d_v) * 2 bytes per stream.
#include <cuda.h>
#include <cuda_fp16.h>
#include <math.h>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"

namespace ttkv_dev {

namespace {

constexpr int kTT = 64;          // tokens per tile
constexpr int kStages = 3;
constexpr uint32_t kBox = kTT * 128;  // one 64-token x 128-byte box

__device__ __forceinline__ uint32_t swz128(uint32_t off) {  // TMA SWIZZLE_128B
  return off ^ (((off >> 7) & 7u) << 4);
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A(16x16, rows = heads, only a0/a2 non-zero) * B(16x8)
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

template <int ND, int GT>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32)
    fast_attn_tc_kernel(const __grid_constant__ FastTcArgs a) {
  constexpr int D = 64 * ND;        // head dim
  constexpr int KSTEPS = D / 16;    // QK k-steps
  constexpr uint32_t STAGE = 2 * ND * kBox;
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, f = blockIdx.x;
  const uint32_t t0 = f * a.FC;
  const uint32_t t1 = min(t0 + a.FC, a.F);
  const uint32_t ntiles = t1 > t0 ? (t1 - t0 + kTT - 1) / kTT : 0;

  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself so the compiler keeps
  // the shared address space (LDS, not generic LD)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kStages * STAGE);
  uint64_t* empty = full + kStages;
  float* sc = reinterpret_cast<float*>(empty + kStages);  // [2][GT][kTT]
  float* mst = sc + 2 * GT * kTT;
  float* lst = mst + GT;
  float* ast = lst + GT;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSlowConsumerWarps);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < GT) {
    mst[threadIdx.x] = -INFINITY;
    lst[threadIdx.x] = 0.0f;
    ast[threadIdx.x] = 1.0f;
  }
  __syncthreads();

  if (warp == 0) {
    // ---- producer: TMA tensor loads of K and V tiles ----
    if (lane == 0) {
      for (uint32_t i = 0; i < ntiles; ++i) {
        const uint32_t st = i % kStages;
        if (i >= kStages) mbar_wait_backoff(&empty[st], ((i / kStages) - 1) & 1);
        const int row = (int)(s * g.C + (a.front + t0 + i * kTT) % g.C);
        uint8_t* kb = base + st * STAGE;
        uint8_t* vb = kb + ND * kBox;
        mbar_arrive_expect_tx(&full[st], STAGE);
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          tma_load_2d(kb + b * kBox, &a.tk, 64 * b, row, &full[st]);
          tma_load_2d(vb + b * kBox, &a.tv, 64 * b, row, &full[st]);
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const uint32_t cw = warp - 1;
  const uint32_t gq = lane >> 2, qq = lane & 3;  // mma group (head row) / thread in group
  const bool head_ok = gq < g.G;
  // A fragments of q (scaled into log2 units), hi + lo
  uint32_t aqh[KSTEPS][2], aql[KSTEPS][2];
  {
    const float* qr = a.q + ((uint64_t)s * g.G + (head_ok ? gq : 0)) * D;
    const float sl = (float)a.scale_log2;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      const int c = 16 * ks + 2 * qq;
      const float x0 = head_ok ? qr[c] * sl : 0.f, x1 = head_ok ? qr[c + 1] * sl : 0.f;
      const float x8 = head_ok ? qr[c + 8] * sl : 0.f, x9 = head_ok ? qr[c + 9] * sl : 0.f;
      split2(x0, x1, aqh[ks][0], aql[ks][0]);
      split2(x8, x9, aqh[ks][1], aql[ks][1]);
    }
  }
  constexpr int NT_PV = D / 8 / kSlowConsumerWarps;  // output n-tiles per warp
  float acc[NT_PV][4], acl[NT_PV][4];  // P_hi . V and P_lo . V (independent chains)
#pragma unroll
  for (int j = 0; j < NT_PV; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[j][e] = acl[j][e] = 0.f;
  const int nthreads_c = kSlowConsumerWarps * 32;

  for (uint32_t i = 0; i < ntiles; ++i) {
    const uint32_t st = i % kStages;
    mbar_wait(&full[st], (i / kStages) & 1);
    const uint32_t kb = smem_u32(base + st * STAGE);
    const uint32_t vb = kb + ND * kBox;
    const uint32_t rows = min((uint32_t)kTT, t1 - (t0 + i * kTT));
    float* scb = sc + (i & 1) * GT * kTT;

    // ---- QK^T: warp cw -> tokens [16cw, 16cw + 16); 4 independent
    // accumulator chains (2 n-tiles x hi/lo) ----
    {
      float c[2][2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[h][0][e] = c[h][1][e] = 0.f;
#pragma unroll
      for (int kp = 0; kp < KSTEPS / 2; ++kp) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          // matrices: (ks lo8, ks hi8, ks+1 lo8, ks+1 hi8) of tokens [8nt, 8nt+8)
          const int m = lane >> 3;
          const int row = 8 * (2 * cw + h) + (lane & 7);
          const int ch = 16 * (2 * kp + (m >> 1)) + 8 * (m & 1);
          const uint32_t addr = kb + (ch >> 6) * kBox + swz128(row * 128 + (ch & 63) * 2);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(addr, b0, b1, b2, b3);
          mma16816(c[h][0], aqh[2 * kp][0], aqh[2 * kp][1], b0, b1);
          mma16816(c[h][1], aql[2 * kp][0], aql[2 * kp][1], b0, b1);
          mma16816(c[h][0], aqh[2 * kp + 1][0], aqh[2 * kp + 1][1], b2, b3);
          mma16816(c[h][1], aql[2 * kp + 1][0], aql[2 * kp + 1][1], b2, b3);
        }
      }
      if (head_ok) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t tA = 8 * (2 * cw + h) + 2 * qq;
          scb[gq * kTT + tA] = tA < rows ? c[h][0][0] + c[h][1][0] : -INFINITY;
          scb[gq * kTT + tA + 1] = tA + 1 < rows ? c[h][0][1] + c[h][1][1] : -INFINITY;
        }
      }
    }
    named_bar(1, nthreads_c);

    // ---- tile softmax statistics, one warp per head ----
    for (uint32_t h = cw; h < g.G; h += kSlowConsumerWarps) {
      float* row = scb + h * kTT;
      float bm = fmaxf(row[lane], row[lane + 32]);
      bm = warp_max(bm);
      const float m_old = mst[h];
      const float m_new = fmaxf(m_old, bm);
      const float p0 = exp2f(row[lane] - m_new), p1 = exp2f(row[lane + 32] - m_new);
      row[lane] = p0;
      row[lane + 32] = p1;
      const float sum = warp_sum(p0 + p1);
      __syncwarp();  // all lanes have read mst[h] before lane 0 rewrites it
      if (lane == 0) {
        const float alpha = exp2f(m_old - m_new);
        lst[h] = lst[h] * alpha + sum;
        mst[h] = m_new;
        ast[h] = alpha;
      }
    }
    named_bar(1, nthreads_c);

    // ---- PV: warp cw -> channels [8 NT_PV cw, 8 NT_PV (cw+1)) ----
    {
      const float alpha = head_ok ? ast[gq] : 1.0f;
#pragma unroll
      for (int j = 0; j < NT_PV; ++j) {
        acc[j][0] *= alpha;
        acc[j][1] *= alpha;
        acl[j][0] *= alpha;
        acl[j][1] *= alpha;
      }
#pragma unroll
      for (int ks = 0; ks < kTT / 16; ++ks) {
        uint32_t ph0, pl0, ph1, pl1;
        {
          const float* pr = scb + (head_ok ? gq : 0) * kTT + 16 * ks + 2 * qq;
          const float2 p01 = head_ok ? *reinterpret_cast<const float2*>(pr) : make_float2(0, 0);
          const float2 p89 = head_ok ? *reinterpret_cast<const float2*>(pr + 8) : make_float2(0, 0);
          split2(p01.x, p01.y, ph0, pl0);
          split2(p89.x, p89.y, ph1, pl1);
        }
#pragma unroll
        for (int jp = 0; jp < NT_PV / 2; ++jp) {
          // matrices: (tok lo8, ntA), (tok hi8, ntA), (tok lo8, ntB), (tok hi8, ntB)
          const int m = lane >> 3;
          const int ntc = NT_PV * cw + 2 * jp + (m >> 1);
          const int row = 16 * ks + 8 * (m & 1) + (lane & 7);
          const int ch = 8 * ntc;
          const uint32_t addr = vb + (ch >> 6) * kBox + swz128(row * 128 + (ch & 63) * 2);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(addr, b0, b1, b2, b3);
          mma16816(acc[2 * jp], ph0, ph1, b0, b1);
          mma16816(acl[2 * jp], pl0, pl1, b0, b1);
          mma16816(acc[2 * jp + 1], ph0, ph1, b2, b3);
          mma16816(acl[2 * jp + 1], pl0, pl1, b2, b3);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ---- emit the (acc, m, l) partial of every head ----
  named_bar(1, nthreads_c);
  const uint32_t pitch = D + 2;
  float* part = reinterpret_cast<float*>(a.part) + (((uint64_t)s * g.G) * a.nfc + f) * pitch;
  const uint64_t head_stride = (uint64_t)a.nfc * pitch;
  if (head_ok) {
    float* p = part + gq * head_stride;
#pragma unroll
    for (int j = 0; j < NT_PV; ++j) {
      const int ch = 8 * (NT_PV * cw + j) + 2 * qq;
      p[ch] = ntiles ? acc[j][0] + acl[j][0] : 0.f;
      p[ch + 1] = ntiles ? acc[j][1] + acl[j][1] : 0.f;
    }
    if (cw == 0 && qq == 0) {
      p[D] = ntiles ? mst[gq] : -INFINITY;
      p[D + 1] = ntiles ? lst[gq] : 0.f;
    }
  }
}

// ---------------------------------------------------------------------------
// slow tier on tensor cores: K8/V4, d = 128, B = 128, fp16 ring (fp32 accum).
// Per record: K codes [128 tok][128 B] by TMA (128B swizzle), V nibbles
// [128 tok][64 B] by TMA (64B swizzle), params (2 KB) by bulk copy from the
// HBM mirror.  QK^T = (q * s) . code + q . z  (scales folded into the A
// operand, codes exact in fp16); PV = s * (P . code) + z *
// sum(P) applied per block in the epilogue.  ldmatrix on the u8 code rows
// yields 4 consecutive channels per thread, so the contraction index is
// permuted identically in A and B (any permutation of a dot product's terms
// is exact in real arithmetic).
// ---------------------------------------------------------------------------
namespace {
constexpr int kSlowTcStages = 3;
constexpr uint32_t kKBox = 128 * 128;  // K codes
constexpr uint32_t kVBox = 128 * 64;   // V nibbles
constexpr uint32_t kPBytes = 2 * 128 * 8;  // {scale, zp} x (128 K + 128 V)
constexpr uint32_t kSlowStage = kKBox + kVBox + kPBytes;  // 26,624 B

__device__ __forceinline__ uint32_t swz64(uint32_t off) {  // TMA SWIZZLE_64B
  return off ^ (((off >> 7) & 3u) << 4);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// 4 u8 codes -> two half2 {c0,c1}, {c2,c3} (exact: 1024 + c minus 1024)
__device__ __forceinline__ void codes_to_h2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t a = __byte_perm(w, 0x64646464u, 0x5140u);
  const uint32_t b = __byte_perm(w, 0x64646464u, 0x7362u);
  const __half2 off = __floats2half2_rn(1024.f, 1024.f);
  __half2 ha = __hsub2(*reinterpret_cast<const __half2*>(&a), off);
  __half2 hb = __hsub2(*reinterpret_cast<const __half2*>(&b), off);
  lo = *reinterpret_cast<uint32_t*>(&ha);
  hi = *reinterpret_cast<uint32_t*>(&hb);
}
}  // namespace

// 2 CTAs/SM: 10 warps over 4 SMSPs -> <= 168 registers per thread
template <int GT>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32, 2)
    slow_attn_tc_kernel(const __grid_constant__ SlowTcArgs a) {
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, chunk = blockIdx.x;
  const uint32_t cnt = a.union_count[s];
  const uint32_t i0 = chunk * a.CH;
  if (i0 >= cnt) return;
  const uint32_t nb = min(i0 + a.CH, cnt) - i0;

  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself so the compiler keeps
  // the shared address space (LDS, not generic LD)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* vtile = base + kSlowTcStages * kSlowStage;  // 2 boxes [64 tok][128 B] fp16 codes
  uint64_t* full = reinterpret_cast<uint64_t*>(vtile + 2 * 64 * 128);
  uint64_t* empty = full + kSlowTcStages;
  float* sc2 = reinterpret_cast<float*>(empty + kSlowTcStages);  // [2][GT][128]
  float* mst = sc2 + 2 * GT * 128;
  float* lst = mst + GT;
  float* ast = lst + GT;
  float* pst = ast + GT;  // sum_t p of the current block

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlowTcStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSlowConsumerWarps);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < GT) {
    mst[threadIdx.x] = -INFINITY;
    lst[threadIdx.x] = 0.0f;
  }
  __syncthreads();
  const uint32_t* uids = a.union_ids + (uint64_t)s * g.n_cap + i0;
  const uint32_t* umask = a.union_mask + (uint64_t)s * g.n_cap + i0;

  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < nb; ++i) {
        const uint32_t st = i % kSlowTcStages;
        if (i >= kSlowTcStages) mbar_wait_backoff(&empty[st], ((i / kSlowTcStages) - 1) & 1);
        const uint32_t blk = uids[i];
        const int rec = (int)((uint64_t)s * g.n_cap + blk);
        uint8_t* dst = base + st * kSlowStage;
        mbar_arrive_expect_tx(&full[st], kSlowStage);
        tma_load_3d(dst, &a.tk, 0, 0, rec, &full[st]);
        tma_load_3d(dst + kKBox, &a.tv, 0, 0, rec, &full[st]);
        bulk_g2s(dst + kKBox + kVBox, a.params + (uint64_t)rec * kPBytes, kPBytes, &full[st]);
      }
    }
    return;
  }

  const uint32_t cw = warp - 1, ct = threadIdx.x - 32;
  const uint32_t gq = lane >> 2, qq = lane & 3;
  const bool head_ok = gq < g.G;
  const int nthreads_c = kSlowConsumerWarps * 32;
  // this thread's 32 query channels (permuted order), log2-scaled:
  // segment j -> channels 16j + 4qq + {0,1,2,3}
  // the (log2-scaled) queries live in smem, not registers (2 CTAs/SM budget)
  float* qsm = pst + GT;  // [GT][128]
  {
    const float* qb = a.q + (uint64_t)s * g.G * 128;
    const float sl = (float)a.scale_log2;
    for (uint32_t i2 = ct; i2 < GT * 128; i2 += nthreads_c)
      qsm[i2] = (i2 / 128 < g.G) ? qb[i2] * sl : 0.f;
    named_bar(1, nthreads_c);
  }
  const float* qrow = qsm + (head_ok ? gq : 0) * 128;
  float acc[4][2];  // running output: head gq, channels 8(4cw + j) + 2qq + {0,1}
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.f;
  uint32_t seen = 0;

  for (uint32_t i = 0; i < nb; ++i) {
    const uint32_t st = i % kSlowTcStages;
    mbar_wait(&full[st], (i / kSlowTcStages) & 1);
    uint8_t* stg = base + st * kSlowStage;
    const uint32_t kb = smem_u32(stg), vb_nib = kKBox;  // V nibbles at stg + kKBox
    const float* kp = reinterpret_cast<const float*>(stg + kKBox + kVBox);  // {s,z} x 128
    const float* vp = kp + 2 * 128;
    const uint32_t hm = umask[i];
    seen |= hm;
    float* sc = sc2 + (i & 1) * GT * 128;  // double-buffered: PV(i-1) may still read

    // ---- A operand: (q * s) hi/lo in the permuted channel order, beta = q . z ----
    uint32_t ah[8][2], al[8][2];
    float beta = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 sz0 = *reinterpret_cast<const float4*>(kp + 2 * (16 * j + 4 * qq));
      const float4 sz1 = *reinterpret_cast<const float4*>(kp + 2 * (16 * j + 4 * qq) + 4);
      const float4 qv = *reinterpret_cast<const float4*>(qrow + 16 * j + 4 * qq);
      const float x0 = qv.x * sz0.x, x1 = qv.y * sz0.z;
      const float x2 = qv.z * sz1.x, x3 = qv.w * sz1.z;
      beta += qv.x * sz0.y + qv.y * sz0.w + qv.z * sz1.y + qv.w * sz1.w;
      split2(x0, x1, ah[j][0], al[j][0]);
      split2(x2, x3, ah[j][1], al[j][1]);
    }
    beta += __shfl_xor_sync(0xffffffffu, beta, 1);
    beta += __shfl_xor_sync(0xffffffffu, beta, 2);

    // ---- QK^T: warp cw -> tokens [32cw, 32cw + 32), two n-tiles at a time:
    // 4 independent accumulator chains (2 n-tiles x hi/lo) ----
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) {
      float c[2][2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[h][0][e] = c[h][1][e] = 0.f;
#pragma unroll
      for (int jp = 0; jp < 2; ++jp) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = lane >> 3;
          const int row = 8 * (4 * cw + 2 * hp + h) + (lane & 7);
          const uint32_t addr = kb + swz128(row * 128 + (4 * jp + m) * 16);
          uint32_t r[4];
          ldsm_x4(addr, r[0], r[1], r[2], r[3]);
#pragma unroll
          for (int mm = 0; mm < 4; ++mm) {
            uint32_t b0, b1;
            codes_to_h2(r[mm], b0, b1);
            const int j = 4 * jp + mm;
            mma16816(c[h][0], ah[j][0], ah[j][1], b0, b1);
            mma16816(c[h][1], al[j][0], al[j][1], b0, b1);
          }
        }
      }
      if (head_ok) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t tA = 8 * (4 * cw + 2 * hp + h) + 2 * qq;
          sc[gq * 128 + tA] = c[h][0][0] + c[h][1][0] + beta;
          sc[gq * 128 + tA + 1] = c[h][0][1] + c[h][1][1] + beta;
        }
      }
    }
    named_bar(1, nthreads_c);

    // ---- block softmax statistics (one warp per selecting head) ----
    for (uint32_t h = cw; h < g.G; h += kSlowConsumerWarps) {
      if (!((hm >> h) & 1u)) continue;
      float* row = sc + h * 128;
      float bm = fmaxf(fmaxf(row[lane], row[lane + 32]), fmaxf(row[lane + 64], row[lane + 96]));
      bm = warp_max(bm);
      const float m_old = mst[h];
      const float m_new = a.literal ? bm : fmaxf(m_old, bm);
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float p = exp2f(row[lane + 32 * k] - m_new);
        row[lane + 32 * k] = p;
        sum += p;
      }
      sum = warp_sum(sum);
      __syncwarp();  // all lanes have read mst[h] before lane 0 rewrites it
      if (a.literal) {  // each block its own normalized partition (engine.cpp:67-72)
        const float inv = 1.0f / sum;
#pragma unroll
        for (int k = 0; k < 4; ++k) row[lane + 32 * k] *= inv;
      }
      if (lane == 0) {
        if (a.literal) {
          ast[h] = 1.0f;
          pst[h] = 1.0f;
        } else {
          const float alpha = exp2f(m_old - m_new);
          lst[h] = lst[h] * alpha + sum;
          mst[h] = m_new;
          ast[h] = alpha;
          pst[h] = sum;
        }
      }
    }
    // ---- PV on codes, in two 64-token halves: V nibbles -> fp16 codes into a
    // 16 KB swizzled tile (two threads per token row), then mma.  Warp cw owns
    // channels [32cw, 32cw + 32). ----
    const bool sel = head_ok && ((hm >> gq) & 1u);
    float cfr[4][4];  // P . code per output n-tile (hi and lo MMAs accumulate here)
#pragma unroll
    for (int j = 0; j < 4; ++j) cfr[j][0] = cfr[j][1] = cfr[j][2] = cfr[j][3] = 0.f;
    {
      const uint32_t vt = smem_u32(vtile);
      const uint8_t* vn = stg + vb_nib;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (half) named_bar(1, nthreads_c);  // first-half PV done before overwrite
        {
          const uint32_t lr = ct >> 1, tr = 64 * half + lr;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int cc = 2 * (ct & 1) + c2;  // 16-byte chunk = channels 32cc .. 32cc+31
            const uint4 w = *reinterpret_cast<const uint4*>(vn + swz64(tr * 64 + 16 * cc));
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // 8 channels: 32cc + 8u .. + 7
              const uint32_t e = ws[u] & 0x0F0F0F0Fu, o = (ws[u] >> 4) & 0x0F0F0F0Fu;
              uint32_t h2[4];
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                // result bytes [e.b, o.b, -, -] -> halves {e.b, o.b} = channels 2b, 2b+1
                const uint32_t x = __byte_perm(e, o, (uint32_t)b | ((4u + (uint32_t)b) << 4));
                const uint32_t hx = (x & 0x000000FFu) | ((x & 0x0000FF00u) << 8) | 0x64006400u;
                const __half2 hv = __hsub2(*reinterpret_cast<const __half2*>(&hx),
                                           __floats2half2_rn(1024.f, 1024.f));
                h2[b] = *reinterpret_cast<const uint32_t*>(&hv);
              }
              const int ch = 32 * cc + 8 * u;
              *reinterpret_cast<uint4*>(vtile + (ch >> 6) * (64 * 128) +
                                        swz128(lr * 128 + (ch & 63) * 2)) =
                  make_uint4(h2[0], h2[1], h2[2], h2[3]);
            }
          }
        }
        named_bar(1, nthreads_c);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int ks = 4 * half + kk;
          uint32_t ph0, pl0, ph1, pl1;
          {
            const float* pr = sc + (head_ok ? gq : 0) * 128 + 16 * ks + 2 * qq;
            const float2 p01 = sel ? *reinterpret_cast<const float2*>(pr) : make_float2(0, 0);
            const float2 p89 = sel ? *reinterpret_cast<const float2*>(pr + 8) : make_float2(0, 0);
            split2(p01.x, p01.y, ph0, pl0);
            split2(p89.x, p89.y, ph1, pl1);
          }
#pragma unroll
          for (int jp = 0; jp < 2; ++jp) {
            const int m = lane >> 3;
            const int ntc = 4 * cw + 2 * jp + (m >> 1);
            const int row = 16 * kk + 8 * (m & 1) + (lane & 7);
            const int ch = 8 * ntc;
            const uint32_t addr = vt + (ch >> 6) * (64 * 128) + swz128(row * 128 + (ch & 63) * 2);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(addr, b0, b1, b2, b3);
            mma16816(cfr[2 * jp], ph0, ph1, b0, b1);
            mma16816(cfr[2 * jp + 1], ph0, ph1, b2, b3);
            mma16816(cfr[2 * jp], pl0, pl1, b0, b1);
            mma16816(cfr[2 * jp + 1], pl0, pl1, b2, b3);
          }
        }
      }
    }
    {
      // affine epilogue: acc = acc * alpha + s_c * (P . code) + z_c * sum(P)
      if (sel) {
        const float alpha = ast[gq], psum = pst[gq];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ch = 8 * (4 * cw + j) + 2 * qq;
          const float4 sz = *reinterpret_cast<const float4*>(vp + 2 * ch);
          acc[j][0] = acc[j][0] * alpha + sz.x * cfr[j][0] + sz.y * psum;
          acc[j][1] = acc[j][1] * alpha + sz.z * cfr[j][1] + sz.w * psum;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  named_bar(1, nthreads_c);
  const uint32_t pitch = 128 + 2;
  if (head_ok) {
    float* p = reinterpret_cast<float*>(a.part) +
               (((uint64_t)s * g.G + gq) * a.nsc + chunk) * pitch;
    const bool any = (seen >> gq) & 1u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = 8 * (4 * cw + j) + 2 * qq;
      p[ch] = any ? acc[j][0] : 0.f;
      p[ch + 1] = any ? acc[j][1] : 0.f;
    }
    if (cw == 0 && qq == 0) {
      p[128] = any ? (a.literal ? 0.f : mst[gq]) : -INFINITY;
      p[129] = any ? (a.literal ? 1.f : lst[gq]) : 0.f;
    }
  }
}

bool slow_tc_supported(const Geometry& g) {
  return g.elem == 2 && g.d_k == 128 && g.d_v == 128 && g.B == 128 && g.kb == 8 && g.vb == 4 &&
         g.G <= 8 && g.rec.kp_off == kKBox + kVBox && g.rec.used == kSlowStage;
}

static size_t slow_tc_smem() {
  return 1024 + (size_t)kSlowTcStages * kSlowStage + 2 * 64 * 128 + 2 * kSlowTcStages * 8 +
         (2 * 8 * 128 + 4 * 8 + 8 * 128) * 4 + 64;
}

template <int GT>
static cudaError_t launch_slow_tc_t(const SlowTcArgs& a, uint32_t grid_chunks, cudaStream_t st) {
  const size_t smem = slow_tc_smem();
  auto kern = slow_attn_tc_kernel<GT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(grid_chunks, a.g.S);
  kern<<<grid, 32 + kSlowConsumerWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_slow_tc(const SlowTcArgs& a, uint32_t grid_chunks, cudaStream_t st) {
  if (grid_chunks == 0) return cudaSuccess;
  if (a.g.G <= 1) return launch_slow_tc_t<1>(a, grid_chunks, st);
  if (a.g.G <= 2) return launch_slow_tc_t<2>(a, grid_chunks, st);
  if (a.g.G <= 4) return launch_slow_tc_t<4>(a, grid_chunks, st);
  return launch_slow_tc_t<8>(a, grid_chunks, st);
}

// Tensor maps over the record arena (device or mapped host pointer):
//   K codes  [S*n_cap records][128 tok][128 B], box 128 x 128 x 1, 128B swizzle
//   V nibbles[S*n_cap records][128 tok][64 B],  box  64 x 128 x 1,  64B swizzle
cudaError_t make_arena_tmaps(const Geometry& g, uint8_t* arena, SlowTcArgs& a) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
  EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
  const cuuint64_t recs = (cuuint64_t)g.S * g.n_cap;
  const cuuint32_t estr[3] = {1, 1, 1};
  {
    const cuuint64_t dims[3] = {128, 128, recs};
    const cuuint64_t strides[2] = {128, g.rec.stride};
    const cuuint32_t box[3] = {128, 128, 1};
    if (encode(&a.tk, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, arena, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[3] = {64, 128, recs};
    const cuuint64_t strides[2] = {64, g.rec.stride};
    const cuuint32_t box[3] = {64, 128, 1};
    if (encode(&a.tv, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, arena + g.rec.v_off, dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

bool fast_tc_supported(const Geometry& g) {
  return g.elem == 2 && g.d_k == g.d_v && (g.d_k == 64 || g.d_k == 128) && g.B % kTT == 0 &&
         g.G <= 8;
}

uint32_t fast_tc_tile() { return kTT; }

static size_t fast_tc_smem(const Geometry& g) {
  const int ND = g.d_k / 64;
  return 1024 + (size_t)kStages * 2 * ND * kBox + 2 * kStages * 8 + (2 * 8 * kTT + 3 * 8) * 4 + 64;
}

template <int ND, int GT>
static cudaError_t launch_fast_tc_t(const FastTcArgs& a, cudaStream_t st) {
  const size_t smem = fast_tc_smem(a.g);
  auto kern = fast_attn_tc_kernel<ND, GT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nfc, a.g.S);
  kern<<<grid, 32 + kSlowConsumerWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <int ND>
static cudaError_t launch_fast_tc_g(const FastTcArgs& a, cudaStream_t st) {
  if (a.g.G <= 1) return launch_fast_tc_t<ND, 1>(a, st);
  if (a.g.G <= 2) return launch_fast_tc_t<ND, 2>(a, st);
  if (a.g.G <= 4) return launch_fast_tc_t<ND, 4>(a, st);
  return launch_fast_tc_t<ND, 8>(a, st);
}

cudaError_t launch_fast_tc(const FastTcArgs& a, cudaStream_t st) {
  return a.g.d_k == 128 ? launch_fast_tc_g<2>(a, st) : launch_fast_tc_g<1>(a, st);
}

// Tensor maps of the fp16 ring: [S*C rows][d] halves, 64 x 64 boxes, 128B swizzle.
cudaError_t make_ring_tmaps(const Geometry& g, void* ring_k, void* ring_v, FastTcArgs& a) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t dims[2] = {g.d_k, (cuuint64_t)g.S * g.C};
  const cuuint64_t strides[1] = {(cuuint64_t)g.d_k * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)kTT};
  const cuuint32_t estr[2] = {1, 1};
  for (int t = 0; t < 2; ++t) {
    CUresult r = encode(t ? &a.tv : &a.tk, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, t ? ring_v : ring_k,
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

}  // namespace ttkv_dev
