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
//   * q and P are split into fp16 hi + lo parts, so operand rounding stays
//     ~2^-22 relative: the result matches the fp32 CUDA-core path well inside
//     the 1e-3 contract.  The hi parts fill A rows 0-7 and the lo parts rows
//     8-15 of the same MMA (G <= 8 heads leave those rows free), so one MMA
//     carries both and a thread adds its row gq and gq + 8 results;
//   * each consumer warp owns a quarter of the output channels, so PV needs
//     no cross-warp reduction; online-softmax statistics are per 64-token tile.
// HBM-bound: F * (d_k + d_v) * 2 bytes per stream.
#include <cuda.h>
#include <cuda_fp16.h>
#include <math.h>

#include <cstdlib>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"
#include "ttkv_dbg_stamps.cuh"

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
// D += A(16x16) * B(16x8), f16 in, f32 accumulate
__device__ __forceinline__ void mma_a4(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                       uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// Power-of-two normalization ahead of an fp16 hi/lo split: returns 2^-k with
// k chosen so the largest magnitude m lands in [2^14, 2^15) -- the hi part
// cannot overflow fp16 (queries of any size, keys near the fp16 range, scales
// of restored records) and the lo part stays a normal fp16 -- and sets
// *unscale = 2^(extra + k) to restore the fp32 result exactly.
__device__ __forceinline__ float pow2_normalizer(float m, int extra, float* unscale) {
  int k = 0;
  if (m > 0.f) k = max(-100, min(100, (int)((__float_as_uint(m) >> 23) & 0xffu) - 127 - 14));
  *unscale = __uint_as_float((uint32_t)(127 + extra + k) << 23);
  return __uint_as_float((uint32_t)(127 - k) << 23);
}
// 2^x in one MUFU.EX2 (exp2f adds a subnormal-range fix-up: 4 instructions);
// results below 2^-126 flush to zero, which no softmax weight here can notice
__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
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

#ifdef TTKV_STAMPS
TTKV_DBG_TABLE(fast)
TTKV_DBG_READER(fast)
#endif
template <int ND, int GT>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32)
    fast_attn_tc_kernel(const __grid_constant__ FastTcArgs a) {
  TTKV_DBG_STAMP(fast, 0);
  constexpr int D = 64 * ND;        // head dim
  constexpr int KSTEPS = D / 16;    // QK k-steps
  constexpr uint32_t STAGE = 2 * ND * kBox;
  // chained launch (speculative record stream): the record stream may launch
  // at once; the ring append and the step position come from earlier kernels
  pdl_trigger();
  pdl_wait();
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, f = blockIdx.x;
  const uint32_t F = a.pos ? (uint32_t)(*a.pos + 1 - a.front) : a.F;
  const uint32_t t0 = f * a.FC;
  const uint32_t t1 = min(t0 + a.FC, F);
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
  float qunscale;  // scores = MMA result * qunscale (see pow2_normalizer)
  {
    const float* qr = a.q + ((uint64_t)s * g.G + (head_ok ? gq : 0)) * D;
    const float sl = (float)a.scale_log2;
    float m = 0.f;  // max |q| of this head: 32 values here, x4 lanes (qq)
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      const int c = 16 * ks + 2 * qq;
      if (head_ok)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(qr[c]), fabsf(qr[c + 1])),
                           fmaxf(fabsf(qr[c + 8]), fabsf(qr[c + 9]))));
    }
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    const float f = pow2_normalizer(m * fabsf(sl), 0, &qunscale) * sl;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      const int c = 16 * ks + 2 * qq;
      const float x0 = head_ok ? qr[c] * f : 0.f, x1 = head_ok ? qr[c + 1] * f : 0.f;
      const float x8 = head_ok ? qr[c + 8] * f : 0.f, x9 = head_ok ? qr[c + 9] * f : 0.f;
      split2(x0, x1, aqh[ks][0], aql[ks][0]);
      split2(x8, x9, aqh[ks][1], aql[ks][1]);
    }
  }
  constexpr int NT_PV = D / 8 / kSlowConsumerWarps;  // output n-tiles per warp
  float acc[NT_PV][4];  // [0..1]: P_hi . V (row gq), [2..3]: P_lo . V (row gq + 8)
#pragma unroll
  for (int j = 0; j < NT_PV; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
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
          // rows gq: q_hi, rows gq + 8: q_lo; k-step parity picks the chain
          mma_a4(c[h][0], aqh[2 * kp][0], aql[2 * kp][0], aqh[2 * kp][1], aql[2 * kp][1], b0, b1);
          mma_a4(c[h][1], aqh[2 * kp + 1][0], aql[2 * kp + 1][0], aqh[2 * kp + 1][1],
                 aql[2 * kp + 1][1], b2, b3);
        }
      }
      if (head_ok) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t tA = 8 * (2 * cw + h) + 2 * qq;
          const float s0 = (c[h][0][0] + c[h][0][2]) + (c[h][1][0] + c[h][1][2]);
          const float s1 = (c[h][0][1] + c[h][0][3]) + (c[h][1][1] + c[h][1][3]);
          scb[gq * kTT + tA] = tA < rows ? s0 * qunscale : -INFINITY;
          scb[gq * kTT + tA + 1] = tA + 1 < rows ? s1 * qunscale : -INFINITY;
        }
      }
    }
    named_bar(1, nthreads_c);

    // ---- tile softmax statistics, one warp per head ----
    for (uint32_t h = cw; h < g.G; h += kSlowConsumerWarps) {
      float* row = scb + h * kTT;
      const float bm = warp_max_redux(fmaxf(row[lane], row[lane + 32]));
      const float m_old = mst[h];
      const float m_new = fmaxf(m_old, bm);
      const float p0 = ex2f(row[lane] - m_new), p1 = ex2f(row[lane + 32] - m_new);
      row[lane] = p0;
      row[lane + 32] = p1;
      const float sum = warp_sum(p0 + p1);
      __syncwarp();  // all lanes have read mst[h] before lane 0 rewrites it
      if (lane == 0) {
        const float alpha = ex2f(m_old - m_new);
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
        acc[j][2] *= alpha;
        acc[j][3] *= alpha;
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
          mma_a4(acc[2 * jp], ph0, pl0, ph1, pl1, b0, b1);
          mma_a4(acc[2 * jp + 1], ph0, pl0, ph1, pl1, b2, b3);
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
      p[ch] = ntiles ? acc[j][0] + acc[j][2] : 0.f;
      p[ch + 1] = ntiles ? acc[j][1] + acc[j][3] : 0.f;
    }
    if (cw == 0 && qq == 0) {
      p[D] = ntiles ? mst[gq] : -INFINITY;
      p[D + 1] = ntiles ? lst[gq] : 0.f;
    }
  }
  if (a.done_epoch) {  // device-side join: the combine waits on *done_epoch
    named_bar(1, nthreads_c);  // every consumer's partial stores precede the fence
    if (threadIdx.x == 32) {
      __threadfence();
      if (atomicAdd(a.done_arrive, 1u) == gridDim.x * gridDim.y - 1) {
        *a.done_arrive = 0u;
        __threadfence();
        atomicAdd(a.done_epoch, 1u);
#ifdef TTKV_STAMPS
        fast_st[(fast_launch - 1) % ttkv_dbg::kSlots][15] = ttkv_dbg::now_ns();
#endif
      }
    }
  }
}

// ---------------------------------------------------------------------------
// slow tier on tensor cores: K8/V4, d = 128, B = 128, fp16 ring (fp32 accum).
// Per record: K codes [128 tok][128 B] by TMA (128B swizzle), V nibbles
// [128 tok][64 B] by TMA (64B swizzle), params (2 KB) by bulk copy from the
// HBM mirror.  The M dimension carries the record's tokens (QK) or channels
// (PV) and N the G <= 8 query heads, so no MMA row is padding:
//   S^T = codes_K . (q * s)^T + q . z    (scales folded into the B operand,
//                                         codes exact in fp16)
//   O^T = codes_V^T . P^T,  O = s * O^T + z * sum(P)  (affine epilogue)
// * (q * s) and P are split into fp16 hi + lo (two MMAs, independent
//   accumulator chains), so operand rounding stays ~2^-22 relative;
// * the B fragments of (q * s) and P are built once per record by the whole
//   CTA and staged in shared memory in fragment order (one LDS.128 each);
// * K codes reach the MMA through ldmatrix + a 2-op u8 -> f16 conversion;
//   V nibbles are decoded straight into A fragments (token pairs per channel)
//   with the 0x6400 magic-number trick -- no fp16 V tile in shared memory;
// * the contraction index of QK is permuted identically in A and B (exact in
//   real arithmetic), and each thread owns 4 consecutive channels of PV;
// * G <= 4 (PK): the hi and lo parts share ONE MMA through the N dimension --
//   column n = 2h + part carries head h's hi (part 0) or lo (part 1) operand,
//   so a thread's accumulator pair (n = 2qq, 2qq + 1) is one head's hi + lo and
//   is summed in registers: half the HMMAs of the two-chain form (G = 8 keeps
//   it, all 8 columns being heads);
// * the head mask of each record reaches the consumers through shared memory
//   (written by the producer with the stage), not a global load per record.
// ---------------------------------------------------------------------------
namespace {
constexpr uint32_t kKBox = 128 * 128;  // K codes
constexpr uint32_t kVBox = 128 * 64;   // V nibbles
constexpr uint32_t kPBytes = 2 * 128 * 8;  // {scale, zp} x (128 K + 128 V)
constexpr uint32_t kSlowStage = kKBox + kVBox + kPBytes;  // 26,624 B = 26 x 1024
constexpr int kScPitch = 132;  // score row pitch (floats): conflict-free C-fragment stores

__device__ __forceinline__ uint32_t swz64(uint32_t off) {  // TMA SWIZZLE_64B
  return off ^ (((off >> 7) & 3u) << 4);
}
// Records are streamed exactly once per step: their TMA loads carry an
// L2 evict-first policy so they do not push the step's partials and
// selection arrays (re-read by the combine) out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}
// Codes enter the tensor cores as fp16 SUBNORMALS: a half whose exponent
// field is 0 and mantissa is the integer n is exactly n * 2^-24, so a byte
// or nibble lands in an A fragment with one mask / byte-permute and no float
// op; the 2^24 (2^20 for a nibble) comes back in the fp32 epilogue, an exact
// power-of-two scaling.  The MMA keeps every subnormal product exactly but
// aligns its sum at the subnormal's nominal exponent, so a value with many
// leading zero mantissa bits loses that many bits of the sum
// (tools/mma_subnormal_probe.cu): nibbles therefore sit in mantissa bits 4-7
// (measured output error unchanged vs. the 1024 + n encoding, tools/err_probe.py).
constexpr float kSub20 = 1048576.0f;
// 4 u8 codes -> two half2 {c0,c1} * 2^-24, {c2,c3} * 2^-24 (exact)
__device__ __forceinline__ void codes_to_h2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  lo = __byte_perm(w, 0u, 0x4140u);
  hi = __byte_perm(w, 0u, 0x4342u);
}
// x = [t.b0, t.b1, t'.b0, t'.b1] (two tokens' 4 LSB-first nibbles = channels
// c..c+3) -> half2 {v[t][c+i], v[t'][c+i]} * 2^-20 (exact subnormals with the
// nibble in mantissa bits 4-7)
__device__ __forceinline__ void nibbles_to_h2(uint32_t x, uint32_t& c0, uint32_t& c1,
                                              uint32_t& c2, uint32_t& c3) {
  c0 = (x << 4) & 0x00F000F0u;
  c1 = x & 0x00F000F0u;
  c2 = (x >> 4) & 0x00F000F0u;
  c3 = (x >> 8) & 0x00F000F0u;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  // try_wait with a suspend-time hint: the producer sleeps in hardware until
  // the consumers release the stage instead of spinning on issue slots
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(10000000u)
      : "memory");
}
template <int GT>
constexpr size_t slow_tc_tail_bytes() {
  // qsf + phl (2 x 256 uint4) | sc [GT][kScPitch] | qsm [GT][128] | 6 x 8 stats
  // | head mask per stage (4 words)
  return 2 * 256 * 16 + (size_t)GT * kScPitch * 4 + (size_t)GT * 128 * 4 + 6 * 8 * 4 + 16;
}
}  // namespace

#ifdef TTKV_STAMPS
TTKV_DBG_TABLE(slow)
TTKV_DBG_READER(slow)
TTKV_DBG_CTA_TABLE(slow)
TTKV_DBG_CTA_READER(slow)
#endif
template <int GT, int ST>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32, ST == 2 ? 3 : 2)
    slow_attn_tc_kernel(const __grid_constant__ SlowTcArgs a) {
  constexpr bool PK = GT <= 4;  // hi/lo packed into the N dimension
  TTKV_DBG_STAMP(slow, 0);
  TTKV_DBG_CTA(slow, 0, 32);
  pdl_wait();  // the union lists (launched chained behind the selection)
  TTKV_DBG_STAMP(slow, 1);
  TTKV_DBG_CTA(slow, 1, 32);
  const Geometry& g = a.g;
  const uint32_t G = g.G;
  const uint32_t c = blockIdx.x;
  // ---- balanced schedule: the step's records (every stream's union, in
  // stream order) split evenly over the grid, which is one wave of resident
  // CTAs; CTA c takes records [c per, (c + 1) per).  A stream's records span
  // consecutive CTAs; each writes its share as partial slot
  // j = c - (first CTA of the stream), and the CTA holding the stream's last
  // record publishes the slot count for the combine. ----
  __shared__ uint32_t sched[4];  // first stream, index in it, records, slot of the first
  __shared__ uint32_t scan_w[8];
  {
    const uint32_t T = blockDim.x, t = threadIdx.x;
    const uint32_t sb = (uint32_t)(((uint64_t)g.S * t) / T), se = (uint32_t)(((uint64_t)g.S * (t + 1)) / T);
    uint32_t mine = 0;
    for (uint32_t x = sb; x < se; ++x) mine += a.union_count[x];
    uint32_t incl = mine;  // inclusive scan over the CTA (warps, then warp totals)
    const uint32_t ln = t & 31, wp = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (ln >= (uint32_t)o) incl += v;
    }
    if (ln == 31) scan_w[wp] = incl;
    __syncthreads();
    uint32_t before = 0, R = 0;
    for (uint32_t w = 0; w < (T + 31) / 32; ++w) {
      before += w < wp ? scan_w[w] : 0u;
      R += scan_w[w];
    }
    const uint32_t excl = before + incl - mine;
    const uint32_t per = max((R + gridDim.x - 1) / gridDim.x, a.per_min);
    const uint64_t lo = (uint64_t)c * per;
    if (t == 0) sched[2] = lo < R ? (uint32_t)(R - lo < per ? R - lo : per) : 0u;
    if (lo < R && excl <= lo && lo < excl + mine) {  // my streams hold record `lo`
      uint32_t off = excl, x = sb;
      while (off + a.union_count[x] <= lo) off += a.union_count[x++];
      sched[0] = x;
      sched[1] = (uint32_t)(lo - off);
      sched[3] = c - off / per;
    }
    __syncthreads();
  }
  const uint32_t n_rec = sched[2];
#ifdef TTKV_STAMPS
  if (threadIdx.x == 32 && blockIdx.x < 1024) slow_cta[blockIdx.x][5] = n_rec;
#endif
  TTKV_DBG_CTA(slow, 2, 32);
  if (n_rec == 0) return;
  const uint32_t s_first = sched[0], i_first = sched[1], slot_first = sched[3];

  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself so the compiler keeps
  // the shared address space (LDS, not generic LD)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint4* qsf = reinterpret_cast<uint4*>(base + ST * kSlowStage);  // [8 j][8 head][4 q]
  uint4* phl = qsf + 256;                                         // [8 ks][8 head][4 q]
  float* sc = reinterpret_cast<float*>(phl + 256);                // [GT][kScPitch]
  float* qsm = sc + GT * kScPitch;                                // [GT][128] log2-scaled q
  float* mst = qsm + GT * 128;
  float* lst = mst + 8;
  float* ast = lst + 8;
  float* pst = ast + 8;  // sum_t p of the current block
  float* bst = pst + 8;  // beta = q . z of the current block
  float* usc = bst + 8;  // per-head score unscale (pow2_normalizer), then max |q|
  uint32_t* hms = reinterpret_cast<uint32_t*>(usc + 8);  // head mask of each stage
  uint64_t* full = reinterpret_cast<uint64_t*>(hms + 4);
  uint64_t* empty = full + ST;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSlowConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();  // the barriers are initialized: the producer may start

  if (warp == 0) {
    // the first records are in flight while the consumers stage q below
    if (lane == 0) {
      const uint64_t evict_first = l2_evict_first_policy();
      uint32_t s = s_first, ii = i_first, cnt = a.union_count[s];
      for (uint32_t i = 0; i < n_rec; ++i, ++ii) {
        while (ii >= cnt) {  // next stream with records
          ii = 0;
          cnt = a.union_count[++s];
        }
        const uint32_t st = i % ST;
        if (i >= ST) mbar_wait_sleep(&empty[st], ((i / ST) - 1) & 1);
        const uint64_t at = (uint64_t)s * g.n_cap + ii;
        const int rec = (int)((uint64_t)s * g.n_cap + a.union_ids[at]);
        uint8_t* dst = base + st * kSlowStage;
        hms[st] = a.union_mask[at];  // published by the arrive below (release.cta)
        mbar_arrive_expect_tx(&full[st], kSlowStage);
        tma_load_3d(dst, &a.tk, 0, 0, rec, &full[st], evict_first);
        tma_load_3d(dst + kKBox, &a.tv, 0, 0, rec, &full[st], evict_first);
        bulk_g2s(dst + kKBox + kVBox, a.params + (uint64_t)rec * kPBytes, kPBytes, &full[st]);
      }
    }
    return;
  }

  const int nthreads_c = kSlowConsumerWarps * 32;
  const uint32_t ct = threadIdx.x - 32;
  const float sl = (float)a.scale_log2;
  const uint32_t cw = warp - 1;
  const uint32_t gq = lane >> 2, qq = lane & 3;  // fragment row group / thread in group
  // PV ownership: channels c0 .. c0 + 3, heads 2qq, 2qq + 1
  const uint32_t c0 = 32 * cw + 4 * gq;
  // Swizzle-folded shared-memory offsets (loop-invariant):
  //  K (128B swizzle): ldmatrix row address of matrix m = lane / 8 -- token
  //  32cw + 16mt + 8(m&1) + (lane&7), 16-byte chunk 2jp + (m>>1); the XOR
  //  term is (token & 7) = (lane & 7)
  uint32_t koff[4];
  {
    const uint32_t m = lane >> 3, r = lane & 7;
    const uint32_t row = 32 * cw + 8 * (m & 1) + r;
#pragma unroll
    for (int jp = 0; jp < 4; ++jp)
      koff[jp] = row * 128 + ((((uint32_t)(2 * jp)) ^ (r & 6u)) | ((m >> 1) ^ (r & 1u))) * 16;
  }
  //  V (64B swizzle): tokens 16ks + 2qq + {0,1,8,9} all have ((t >> 1) & 3) = qq
  const uint32_t voff = 2 * qq * 64 + ((c0 >> 1) ^ (qq << 4));

  // ---- consumer: one segment per stream this CTA touches ----
  uint32_t s = s_first, ii = i_first, cnt = a.union_count[s_first], slot = slot_first;
  for (uint32_t r0 = 0; r0 < n_rec;) {
    while (ii >= cnt) {  // next stream with records
      ii = 0;
      cnt = a.union_count[++s];
      slot = 0;
    }
    const uint32_t seg = min(n_rec - r0, cnt - ii);
    // ---- stage q of stream s (named barrier 1 over the consumer warps only) ----
    for (uint32_t i = ct; i < 512; i += nthreads_c) qsf[i] = make_uint4(0, 0, 0, 0);
    // q in log2 units, normalized per head by a power of two so that
    // |q_c s_c| <= |q|max * kTcKeyScaleBound lands below 2^15: the fp16 hi part
    // of q * s cannot overflow for any query or record (ttkv_launch.h)
    if (ct < 8) usc[ct] = 0.f;
    named_bar(1, nthreads_c);
    const float* qb = a.q + (uint64_t)s * G * 128;
    for (uint32_t i = ct; i < G * 128; i += nthreads_c)
      atomicMax(reinterpret_cast<uint32_t*>(usc) + i / 128, __float_as_uint(fabsf(qb[i] * sl)));
    named_bar(1, nthreads_c);
    {
      float f = 1.f, uns = 1.f;
      if (ct < 8) f = pow2_normalizer(usc[ct] * kTcKeyScaleBound, 24, &uns);
      named_bar(1, nthreads_c);
      if (ct < 8) {
        usc[ct] = uns;  // 2^24: the subnormal K codes
        mst[ct] = f;    // scratch until the stats are initialized below
      }
    }
    named_bar(1, nthreads_c);
    for (uint32_t i = ct; i < GT * 128; i += nthreads_c)
      qsm[i] = (i / 128 < G) ? (qb[i] * sl) * mst[i / 128] : 0.f;
    named_bar(1, nthreads_c);
    if (ct < 8) {
      mst[ct] = -INFINITY;
      lst[ct] = 0.0f;
    }
    named_bar(1, nthreads_c);

    float acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.f;
    uint32_t seen = 0;
    // score unscale of this lane's heads (PK: head qq; otherwise 2qq, 2qq + 1)
    const float uns0 = usc[PK ? qq : 2 * qq], uns1 = usc[2 * qq + 1];
    for (uint32_t i = r0; i < r0 + seg; ++i) {
      const uint32_t st = i % ST;
      mbar_wait(&full[st], (i / ST) & 1);
      if (i == 0) TTKV_DBG_CTA(slow, 3, 32);
      uint8_t* stg = base + st * kSlowStage;
      const uint32_t kb = smem_u32(stg);
      const uint8_t* vn = stg + kKBox;
      const float* kp = reinterpret_cast<const float*>(stg + kKBox + kVBox);  // {s,z} x 128
      const float* vp = kp + 2 * 128;
      const uint32_t hm = hms[st];
      seen |= hm;

      // ---- (q * s) B fragments (hi/lo) and this lane's share of beta = q . z
      // for heads cw and cw + 4 (reduced after the QK MMAs are issued) ----
      float bpart[2] = {0.f, 0.f};
#pragma unroll
      for (int rep = 0; rep < 2; ++rep) {
        const uint32_t e = ct + rep * nthreads_c;  // warp-uniform: one head per warp
        if (e >= G * 32) break;
        const uint32_t h = e >> 5, j = (e >> 2) & 7u, q4 = e & 3u;
        const uint32_t c = 16 * j + 4 * q4;
        const float4 qv = *reinterpret_cast<const float4*>(qsm + h * 128 + c);
        const float4 sz0 = *reinterpret_cast<const float4*>(kp + 2 * c);
        const float4 sz1 = *reinterpret_cast<const float4*>(kp + 2 * c + 4);
        uint32_t h01, l01, h23, l23;
        split2(qv.x * sz0.x, qv.y * sz0.z, h01, l01);
        split2(qv.z * sz1.x, qv.w * sz1.z, h23, l23);
        if constexpr (PK) {  // column 2h: hi, 2h + 1: lo
          uint2* qsf2 = reinterpret_cast<uint2*>(qsf);
          qsf2[(j * 8 + 2 * h) * 4 + q4] = make_uint2(h01, h23);
          qsf2[(j * 8 + 2 * h + 1) * 4 + q4] = make_uint2(l01, l23);
        } else {
          qsf[(j * 8 + h) * 4 + q4] = make_uint4(h01, h23, l01, l23);
        }
        bpart[rep] = qv.x * sz0.y + qv.y * sz0.w + qv.z * sz1.y + qv.w * sz1.w;
      }
      named_bar(1, nthreads_c);

      // ---- QK^T: warp cw -> tokens [32cw, 32cw + 32) = 2 m-tiles; hi and lo
      // accumulate in independent chains (PK: one chain per k-half, hi and lo
      // in adjacent columns) ----
      if constexpr (PK) {
        const uint2* qsf2 = reinterpret_cast<const uint2*>(qsf);
        float c[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) c[mt][0][e] = c[mt][1][e] = 0.f;
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const uint2 b0 = qsf2[((2 * jp) * 8 + gq) * 4 + qq];
          const uint2 b1 = qsf2[((2 * jp + 1) * 8 + gq) * 4 + qq];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const uint32_t addr = kb + koff[jp] + mt * 16 * 128;
            uint32_t r0, r1, r2, r3, a0, a1, a2, a3;
            ldsm_x4(addr, r0, r1, r2, r3);
            codes_to_h2(r0, a0, a2);
            codes_to_h2(r1, a1, a3);
            mma_a4(c[mt][0], a0, a1, a2, a3, b0.x, b0.y);
            codes_to_h2(r2, a0, a2);
            codes_to_h2(r3, a1, a3);
            mma_a4(c[mt][1], a0, a1, a2, a3, b1.x, b1.y);
          }
        }
#pragma unroll
        for (int rep = 0; rep < 2; ++rep) {
          const uint32_t h = cw + rep * kSlowConsumerWarps;
          if (h < G) {  // warp-uniform
            const float beta = warp_sum(bpart[rep]) * (usc[h] * (1.0f / 16777216.0f));
            if (lane == 0) bst[h] = beta;
          }
        }
        // thread (gq, qq): columns 2qq (hi) and 2qq + 1 (lo) of head qq
        if (qq < G) {
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const uint32_t t = 32 * cw + 16 * mt + gq + 4 * e;
              sc[qq * kScPitch + t] =
                  ((c[mt][0][e] + c[mt][0][e + 1]) + (c[mt][1][e] + c[mt][1][e + 1])) * uns0;
            }
        }
      } else {
        float c[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) c[mt][0][e] = c[mt][1][e] = 0.f;
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const uint4 b0 = qsf[((2 * jp) * 8 + gq) * 4 + qq];
          const uint4 b1 = qsf[((2 * jp + 1) * 8 + gq) * 4 + qq];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            // matrices: (tok 0-7, chunk 2jp), (tok 8-15, 2jp), (tok 0-7, 2jp+1), (tok 8-15, 2jp+1)
            const uint32_t addr = kb + koff[jp] + mt * 16 * 128;
            uint32_t r0, r1, r2, r3, a0, a1, a2, a3;
            ldsm_x4(addr, r0, r1, r2, r3);
            codes_to_h2(r0, a0, a2);
            codes_to_h2(r1, a1, a3);
            mma_a4(c[mt][0], a0, a1, a2, a3, b0.x, b0.y);
            mma_a4(c[mt][1], a0, a1, a2, a3, b0.z, b0.w);
            codes_to_h2(r2, a0, a2);
            codes_to_h2(r3, a1, a3);
            mma_a4(c[mt][0], a0, a1, a2, a3, b1.x, b1.y);
            mma_a4(c[mt][1], a0, a1, a2, a3, b1.z, b1.w);
          }
        }
#pragma unroll
        for (int rep = 0; rep < 2; ++rep) {
          const uint32_t h = cw + rep * kSlowConsumerWarps;
          if (h < G) {  // warp-uniform
            // qsm carries the pow2 normalizer 2^-k; usc[h] = 2^(24 + k)
            const float beta = warp_sum(bpart[rep]) * (usc[h] * (1.0f / 16777216.0f));
            if (lane == 0) bst[h] = beta;
          }
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t h = 2 * qq + (e & 1);
            const uint32_t t = 32 * cw + 16 * mt + gq + 8 * (e >> 1);
            if (h < G) sc[h * kScPitch + t] = (c[mt][0][e] + c[mt][1][e]) * ((e & 1) ? uns1 : uns0);
          }
      }
      named_bar(1, nthreads_c);

      // ---- block softmax statistics + P fragments (one warp per head); lane
      // (ks, q) owns tokens 16ks + 2q + {0, 1, 8, 9} ----
      for (uint32_t h = cw; h < G; h += kSlowConsumerWarps) {
        const uint32_t ks = lane >> 2, q4 = lane & 3;
        uint4* dst = phl + (ks * 8 + h) * 4 + q4;
        uint2* dhi = reinterpret_cast<uint2*>(phl) + (ks * 8 + 2 * h) * 4 + q4;  // PK columns
        uint2* dlo = dhi + 4;
        if (!((hm >> h) & 1u)) {  // head did not select this block
          if constexpr (PK) {
            *dhi = make_uint2(0, 0);
            *dlo = make_uint2(0, 0);
          } else {
            *dst = make_uint4(0, 0, 0, 0);
          }
          if (lane == 0) {
            ast[h] = 1.0f;
            pst[h] = 0.0f;
          }
          continue;
        }
        const float* row = sc + h * kScPitch + 16 * ks + 2 * q4;
        const float beta = bst[h];
        float2 v01 = *reinterpret_cast<const float2*>(row);
        float2 v89 = *reinterpret_cast<const float2*>(row + 8);
        v01.x += beta; v01.y += beta; v89.x += beta; v89.y += beta;
        const float bm = warp_max_redux(fmaxf(fmaxf(v01.x, v01.y), fmaxf(v89.x, v89.y)));
        const float m_old = mst[h];
        const float m_new = a.literal ? bm : fmaxf(m_old, bm);
        float p0 = ex2f(v01.x - m_new), p1 = ex2f(v01.y - m_new);
        float p8 = ex2f(v89.x - m_new), p9 = ex2f(v89.y - m_new);
        const float sum = warp_sum((p0 + p1) + (p8 + p9));
        if (a.literal) {  // each block its own normalized partition (engine.cpp:67-72)
          const float inv = 1.0f / sum;
          p0 *= inv; p1 *= inv; p8 *= inv; p9 *= inv;
        }
        uint32_t h01, l01, h89, l89;
        split2(p0, p1, h01, l01);
        split2(p8, p9, h89, l89);
        if constexpr (PK) {
          *dhi = make_uint2(h01, h89);
          *dlo = make_uint2(l01, l89);
        } else {
          *dst = make_uint4(h01, h89, l01, l89);
        }
        __syncwarp();  // all lanes have read mst[h] before lane 0 rewrites it
        if (lane == 0) {
          if (a.literal) {
            ast[h] = 1.0f;
            pst[h] = 1.0f;
          } else {
            const float alpha = ex2f(m_old - m_new);
            lst[h] = lst[h] * alpha + sum;
            mst[h] = m_new;
            ast[h] = alpha;
            pst[h] = sum;
          }
        }
      }
      named_bar(1, nthreads_c);

      // ---- PV^T: warp cw -> channels [32cw, 32cw + 32) as 2 m-tiles; thread
      // rows gq / gq + 8 of m-tile 0 = channels c0, c0 + 1, of m-tile 1 =
      // c0 + 2, c0 + 3 (one u16 of V nibbles per token) ----
      if constexpr (PK) {  // columns 2qq, 2qq + 1 = head qq hi, lo; chains by ks parity
        const uint2* phl2 = reinterpret_cast<const uint2*>(phl);
        float cf[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) cf[mt][0][e] = cf[mt][1][e] = 0.f;
        const uint8_t* vt = vn + voff;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t u0 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024);
          const uint32_t u1 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 64);
          const uint32_t u8 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 512);
          const uint32_t u9 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 576);
          uint32_t x0, x1, x2, x3, y0, y1, y2, y3;
          nibbles_to_h2(__byte_perm(u0, u1, 0x5410u), x0, x1, x2, x3);
          nibbles_to_h2(__byte_perm(u8, u9, 0x5410u), y0, y1, y2, y3);
          const uint2 pb = phl2[(ks * 8 + gq) * 4 + qq];
          mma_a4(cf[0][ks & 1], x0, x1, y0, y1, pb.x, pb.y);
          mma_a4(cf[1][ks & 1], x2, x3, y2, y3, pb.x, pb.y);
        }
        const uint32_t h = qq;
        if (h < G && ((hm >> h) & 1u)) {
          const float4 sz01 = *reinterpret_cast<const float4*>(vp + 2 * c0);
          const float4 sz23 = *reinterpret_cast<const float4*>(vp + 2 * c0 + 4);
          const float vs[4] = {sz01.x * kSub20, sz01.z * kSub20, sz23.x * kSub20, sz23.z * kSub20};
          const float vz[4] = {sz01.y, sz01.w, sz23.y, sz23.w};
          const float alpha = ast[h], psum = pst[h];
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) {
            const int mt = ci >> 1, e = 2 * (ci & 1);
            const float o = (cf[mt][0][e] + cf[mt][0][e + 1]) + (cf[mt][1][e] + cf[mt][1][e + 1]);
            acc[ci][0] = acc[ci][0] * alpha + vs[ci] * o + vz[ci] * psum;
          }
        }
      } else {
        float cf[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; ++e) cf[mt][0][e] = cf[mt][1][e] = 0.f;
        const uint8_t* vt = vn + voff;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t u0 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024);
          const uint32_t u1 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 64);
          const uint32_t u8 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 512);
          const uint32_t u9 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 576);
          uint32_t x0, x1, x2, x3, y0, y1, y2, y3;
          nibbles_to_h2(__byte_perm(u0, u1, 0x5410u), x0, x1, x2, x3);
          nibbles_to_h2(__byte_perm(u8, u9, 0x5410u), y0, y1, y2, y3);
          const uint4 pb = phl[(ks * 8 + gq) * 4 + qq];
          mma_a4(cf[0][0], x0, x1, y0, y1, pb.x, pb.y);
          mma_a4(cf[0][1], x0, x1, y0, y1, pb.z, pb.w);
          mma_a4(cf[1][0], x2, x3, y2, y3, pb.x, pb.y);
          mma_a4(cf[1][1], x2, x3, y2, y3, pb.z, pb.w);
        }
        // affine epilogue: acc = acc * alpha + s_c * (P . code) + z_c * sum(P)
        const float4 sz01 = *reinterpret_cast<const float4*>(vp + 2 * c0);
        const float4 sz23 = *reinterpret_cast<const float4*>(vp + 2 * c0 + 4);
        const float vs[4] = {sz01.x * kSub20, sz01.z * kSub20, sz23.x * kSub20, sz23.z * kSub20};
        const float vz[4] = {sz01.y, sz01.w, sz23.y, sz23.w};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t h = 2 * qq + hh;
          if (h < G && ((hm >> h) & 1u)) {
            const float alpha = ast[h], psum = pst[h];
#pragma unroll
            for (int ci = 0; ci < 4; ++ci) {
              const int mt = ci >> 1, e = 2 * (ci & 1) + hh;
              acc[ci][hh] = acc[ci][hh] * alpha + vs[ci] * (cf[mt][0][e] + cf[mt][1][e]) +
                            vz[ci] * psum;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }


    // ---- emit the (acc, m, l) partial of every head of stream s ----
    // ---- emit the (acc, m, l) partial of every head ----
    named_bar(1, nthreads_c);
    const uint32_t pitch = 128 + 2;
#pragma unroll
    for (int hh = 0; hh < (PK ? 1 : 2); ++hh) {
      const uint32_t h = PK ? qq : 2 * qq + hh;
      if (h >= G) continue;
      float* p = reinterpret_cast<float*>(a.part) + (((uint64_t)s * G + h) * a.nsc + slot) * pitch;
      const bool any = (seen >> h) & 1u;
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) p[c0 + ci] = any ? acc[ci][hh] : 0.f;
      if (cw == 0 && gq == 0) {
        p[128] = any ? (a.literal ? 0.f : mst[h]) : -INFINITY;
        p[129] = any ? (a.literal ? 1.f : lst[h]) : 0.f;
      }
    }

    if (ii + seg == cnt && threadIdx.x == 32) a.nslots[s] = slot + 1;  // the stream ends here
    r0 += seg;
    ii += seg;
  }
  TTKV_DBG_CTA(slow, 4, 32);
  pdl_trigger();  // the combine's CTAs may get resident while partials drain
}

// ---------------------------------------------------------------------------
// Speculative record stream (HBM slow tier, small steps -- one layer of a
// layer-sequential decode).  With the records in HBM the step is latency-
// bound on the chain selection -> record stream -> combine, and with per-head
// selection of a fraction f of the blocks the union of G heads' sets covers
// 1 - (1 - f)^G of them (0.91 at f = 0.45, G = 4).  This kernel therefore
// does NOT wait for the selection: it streams EVERY record of the step while
// the selection runs beside it (launched behind it with programmatic
// serialization, the selection triggers at its start), and writes each
// record's block-local partial per head -- (o_blk[128], m_blk, l_blk) with
// p = exp2(s - m_blk) -- to `rpart` [S][G][n_cap][kSpecPitch].  The combine
// then merges, per (stream, head), exactly the records that head selected
// (the union lists), so outputs and selections are those of the selective
// kernel; the extra (1 - density) of record bytes buys the selection's
// latency.  Records are handed out from a global queue (`spec_ctr`, reset by
// the combine) two at a time, so CTAs that start late (SMs held by the
// selection or the fast tier) simply take fewer.  Same per-record tensor-core
// math as slow_attn_tc_kernel (PK form, G <= 4); q is normalized per record
// from L1-resident global q instead of once per stream segment.
// ---------------------------------------------------------------------------
template <int GT>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32, 3)
    slow_attn_tc_spec_kernel(const __grid_constant__ SlowTcArgs a) {
  static_assert(GT <= 4, "speculative stream: PK form only");
  constexpr int ST = 2;
  constexpr uint32_t kGrab = 2;
  constexpr uint32_t kEnd = 0xffffffffu;
  // no pdl_wait here: q, the arena and the param mirror are not written by
  // the selection this kernel is chained behind (it waits at its end)
  const Geometry& g = a.g;
  const uint32_t G = g.G, n = a.spec_n;
  const uint32_t total = g.S * n;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint4* qsf = reinterpret_cast<uint4*>(base + ST * kSlowStage);
  uint4* phl = qsf + 256;
  float* sc = reinterpret_cast<float*>(phl + 256);  // [GT][kScPitch]
  float* usc = sc + GT * kScPitch;                 // per-head score unscale of the record
  float* mst = usc + 8;                            // m_blk per head
  float* pst = mst + 8;                            // l_blk per head
  float* bst = pst + 8;                            // beta = q . z per head
  uint32_t* srec = reinterpret_cast<uint32_t*>(bst + 8);  // flat record index per stage
  uint64_t* full = reinterpret_cast<uint64_t*>(srec + 4);
  uint64_t* empty = full + ST;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSlowConsumerWarps);
    }
    fence_mbar_init();
  }
  for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) qsf[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t evict_first = l2_evict_first_policy();
      uint32_t i = 0;
      uint32_t cur = atomicAdd(a.spec_ctr, kGrab);
      for (;;) {
        // the next grab is in flight while this one waits for free stages
        const uint32_t nxt = cur < total ? atomicAdd(a.spec_ctr, kGrab) : total;
        bool end = false;
        for (uint32_t r = cur; r < cur + kGrab; ++r, ++i) {
          const uint32_t st = i % ST;
          if (i >= ST) mbar_wait_sleep(&empty[st], ((i / ST) - 1) & 1);
          if (r >= total) {
            srec[st] = kEnd;
            mbar_arrive(&full[st]);
            end = true;
            break;
          }
          const uint32_t s = r / n;
          const int rec = (int)((uint64_t)s * g.n_cap + (r - s * n));
          uint8_t* dst = base + st * kSlowStage;
          srec[st] = r;  // published by the arrive below (release.cta)
          mbar_arrive_expect_tx(&full[st], kSlowStage);
          tma_load_3d(dst, &a.tk, 0, 0, rec, &full[st], evict_first);
          tma_load_3d(dst + kKBox, &a.tv, 0, 0, rec, &full[st], evict_first);
          bulk_g2s(dst + kKBox + kVBox, a.params + (uint64_t)rec * kPBytes, kPBytes, &full[st]);
        }
        if (end) break;
        cur = nxt;
      }
    }
    return;
  }

  const int nthreads_c = kSlowConsumerWarps * 32;
  const float sl = (float)a.scale_log2;
  const uint32_t cw = warp - 1;
  const uint32_t gq = lane >> 2, qq = lane & 3;
  const uint32_t c0 = 32 * cw + 4 * gq;
  uint32_t koff[4];
  {
    const uint32_t m = lane >> 3, r = lane & 7;
    const uint32_t row = 32 * cw + 8 * (m & 1) + r;
#pragma unroll
    for (int jp = 0; jp < 4; ++jp)
      koff[jp] = row * 128 + ((((uint32_t)(2 * jp)) ^ (r & 6u)) | ((m >> 1) ^ (r & 1u))) * 16;
  }
  const uint32_t voff = 2 * qq * 64 + ((c0 >> 1) ^ (qq << 4));
  uint2* qsf2 = reinterpret_cast<uint2*>(qsf);
  const uint2* phl2c = reinterpret_cast<const uint2*>(phl);

  for (uint32_t i = 0;; ++i) {
    const uint32_t st = i % ST;
    mbar_wait(&full[st], (i / ST) & 1);
    const uint32_t r = srec[st];
    if (r == kEnd) break;
    const uint32_t s = r / n, b = r - s * n;
    uint8_t* stg = base + st * kSlowStage;
    const uint32_t kb = smem_u32(stg);
    const uint8_t* vn = stg + kKBox;
    const float* kp = reinterpret_cast<const float*>(stg + kKBox + kVBox);
    const float* vp = kp + 2 * 128;

    // ---- (q * s) fragments of head cw: q normalized by a power of two from
    // its own max (as in slow_attn_tc_kernel), lane (j, q4) channels 16j + 4q4 ----
    float bpart = 0.f;
    if (cw < G) {
      const uint32_t h = cw, j = lane >> 2, q4 = lane & 3;
      const uint32_t c = 16 * j + 4 * q4;
      float4 qv = __ldg(reinterpret_cast<const float4*>(a.q + ((uint64_t)s * G + h) * 128 + c));
      qv.x *= sl; qv.y *= sl; qv.z *= sl; qv.w *= sl;
      const float mx = warp_max_redux(fmaxf(fmaxf(fabsf(qv.x), fabsf(qv.y)),
                                            fmaxf(fabsf(qv.z), fabsf(qv.w))));
      float uns;
      const float f = pow2_normalizer(mx * kTcKeyScaleBound, 24, &uns);
      qv.x *= f; qv.y *= f; qv.z *= f; qv.w *= f;
      if (lane == 0) usc[h] = uns;
      const float4 sz0 = *reinterpret_cast<const float4*>(kp + 2 * c);
      const float4 sz1 = *reinterpret_cast<const float4*>(kp + 2 * c + 4);
      uint32_t h01, l01, h23, l23;
      split2(qv.x * sz0.x, qv.y * sz0.z, h01, l01);
      split2(qv.z * sz1.x, qv.w * sz1.z, h23, l23);
      qsf2[(j * 8 + 2 * h) * 4 + q4] = make_uint2(h01, h23);
      qsf2[(j * 8 + 2 * h + 1) * 4 + q4] = make_uint2(l01, l23);
      bpart = qv.x * sz0.y + qv.y * sz0.w + qv.z * sz1.y + qv.w * sz1.w;
    }
    named_bar(1, nthreads_c);

    // ---- QK^T (tokens [32cw, 32cw + 32), all heads) ----
    {
      float c[2][2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[mt][0][e] = c[mt][1][e] = 0.f;
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        const uint2 b0 = qsf2[((2 * jp) * 8 + gq) * 4 + qq];
        const uint2 b1 = qsf2[((2 * jp + 1) * 8 + gq) * 4 + qq];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const uint32_t addr = kb + koff[jp] + mt * 16 * 128;
          uint32_t r0, r1, r2, r3, a0, a1, a2, a3;
          ldsm_x4(addr, r0, r1, r2, r3);
          codes_to_h2(r0, a0, a2);
          codes_to_h2(r1, a1, a3);
          mma_a4(c[mt][0], a0, a1, a2, a3, b0.x, b0.y);
          codes_to_h2(r2, a0, a2);
          codes_to_h2(r3, a1, a3);
          mma_a4(c[mt][1], a0, a1, a2, a3, b1.x, b1.y);
        }
      }
      if (cw < G) {
        const float beta = warp_sum(bpart) * (usc[cw] * (1.0f / 16777216.0f));
        if (lane == 0) bst[cw] = beta;
      }
      if (qq < G) {
        const float uns0 = usc[qq];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const uint32_t t = 32 * cw + 16 * mt + gq + 4 * e;
            sc[qq * kScPitch + t] =
                ((c[mt][0][e] + c[mt][0][e + 1]) + (c[mt][1][e] + c[mt][1][e + 1])) * uns0;
          }
      }
    }
    named_bar(1, nthreads_c);

    // ---- block-local softmax of head cw: p = exp2(s - m_blk) ----
    if (cw < G) {
      const uint32_t h = cw, ks = lane >> 2, q4 = lane & 3;
      uint2* dhi = reinterpret_cast<uint2*>(phl) + (ks * 8 + 2 * h) * 4 + q4;  // PK columns
      uint2* dlo = dhi + 4;
      const float* row = sc + h * kScPitch + 16 * ks + 2 * q4;
      const float beta = bst[h];
      float2 v01 = *reinterpret_cast<const float2*>(row);
      float2 v89 = *reinterpret_cast<const float2*>(row + 8);
      v01.x += beta; v01.y += beta; v89.x += beta; v89.y += beta;
      const float bm = warp_max_redux(fmaxf(fmaxf(v01.x, v01.y), fmaxf(v89.x, v89.y)));
      const float p0 = ex2f(v01.x - bm), p1 = ex2f(v01.y - bm);
      const float p8 = ex2f(v89.x - bm), p9 = ex2f(v89.y - bm);
      const float sum = warp_sum((p0 + p1) + (p8 + p9));
      uint32_t h01, l01, h89, l89;
      split2(p0, p1, h01, l01);
      split2(p8, p9, h89, l89);
      *dhi = make_uint2(h01, h89);
      *dlo = make_uint2(l01, l89);
      if (lane == 0) {
        mst[h] = bm;
        pst[h] = sum;
      }
    }
    named_bar(1, nthreads_c);

    // ---- PV^T (channels [32cw, 32cw + 32)), then this record's partial ----
    {
      float cf[2][2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) cf[mt][0][e] = cf[mt][1][e] = 0.f;
      const uint8_t* vt = vn + voff;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t u0 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024);
        const uint32_t u1 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 64);
        const uint32_t u8 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 512);
        const uint32_t u9 = *reinterpret_cast<const uint16_t*>(vt + ks * 1024 + 576);
        uint32_t x0, x1, x2, x3, y0, y1, y2, y3;
        nibbles_to_h2(__byte_perm(u0, u1, 0x5410u), x0, x1, x2, x3);
        nibbles_to_h2(__byte_perm(u8, u9, 0x5410u), y0, y1, y2, y3);
        const uint2 pb = phl2c[(ks * 8 + gq) * 4 + qq];
        mma_a4(cf[0][ks & 1], x0, x1, y0, y1, pb.x, pb.y);
        mma_a4(cf[1][ks & 1], x2, x3, y2, y3, pb.x, pb.y);
      }
      const uint32_t h = qq;
      if (h < G) {
        const float4 sz01 = *reinterpret_cast<const float4*>(vp + 2 * c0);
        const float4 sz23 = *reinterpret_cast<const float4*>(vp + 2 * c0 + 4);
        const float psum = pst[h];
        float o[4];
        const float vs[4] = {sz01.x * kSub20, sz01.z * kSub20, sz23.x * kSub20, sz23.z * kSub20};
        const float vz[4] = {sz01.y, sz01.w, sz23.y, sz23.w};
#pragma unroll
        for (int ci = 0; ci < 4; ++ci) {
          const int mt = ci >> 1, e = 2 * (ci & 1);
          o[ci] = vs[ci] * ((cf[mt][0][e] + cf[mt][0][e + 1]) + (cf[mt][1][e] + cf[mt][1][e + 1])) +
                  vz[ci] * psum;
        }
        float* dst = a.rpart + (((uint64_t)s * G + h) * g.n_cap + b) * kSpecPitch;
        *reinterpret_cast<float4*>(dst + c0) = make_float4(o[0], o[1], o[2], o[3]);
        if (cw == 0 && gq == 0) *reinterpret_cast<float2*>(dst + 128) = make_float2(mst[h], psum);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  // The selection must be complete before this grid is: the combine waits on
  // this grid only, and reads the selection's union lists.
  pdl_wait();
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// slow tier on 5th-generation tensor cores (tcgen05.mma.kind::i8, TMEM
// accumulators): the same record stream, schedule and partials as
// slow_attn_tc_kernel, with both products as exact integer MMAs.
//   QK: D[tok][n] = sum_c code_K[tok][c] * B[n][c] with u8 B: the three low
//       bytes of X' = X + 2^21, X = q s of head h scaled by 2^k_h (k_h from
//       the head's max |q s| in this record, |X| < 2^21), in rows n = PL pl +
//       h, plus an all-ones row: S = (D0 + 2^8 D1 + 2^16 D2 - 2^21 D1s) 2^-k
//       + q . z, exact in 64-bit integers up to the 2^-21 (relative to the
//       head's max) of X.  The TMA-loaded u8 codes ARE the A operand (K-major,
//       128B swizzle): no conversion instruction touches them.
//   PV: D[b][4h + j] = sum_tok A[tok][b] * byte_j(Y_h[tok]), Y = p 2^22
//       (< 2^22): the bytes of Y are its base-256 digits, so a token's B row
//       (MN-major, no swizzle) is just its heads' Y words -- one 16-byte store.
//       M = 64: A is the V tile as TMA delivered it (64 bytes per token, a
//       byte = channel 2b + 16 x channel 2b+1, 64B swizzle), and a second MMA
//       runs on the high nibbles (written over the consumed K codes); channel
//       2b = D_bytes - 16 D_high.  O = s (D0 + 2^8 D1 + 2^16 D2) 2^-22 +
//       z sum(Y) 2^-22.
// Opt-in (TTKV_SLOW_TC5=1): parity-green (output error <= 3.7e-6,
// tools/err_probe.py) with fewer issued instructions than the mma.sync kernel,
// but ~1 % behind it (cfg2 0.985 vs 0.93 ms per launch): it is latency-bound on
// three CTA barriers and two MMA round trips per record.
// One elected consumer thread issues the MMAs (4 per QK, 8 per PV, K = 32) and
// commits them to an mbarrier; TMEM lanes are tokens (QK) or byte rows (PV),
// so each consumer thread reads its own token's scores / channel's outputs
// for every head with one tcgen05.ld.
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte) {  // SW128 tile offset
  return row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100); SWIZZLE_NONE
  return d;
}
// kind::i8 instruction descriptor: D s32, A u8, B s8 / u8, majors, N, M = 128
__host__ __device__ constexpr uint32_t umma_idesc_i8(uint32_t N, uint32_t a_mn, uint32_t b_s8,
                                                     uint32_t b_mn) {
  return (2u << 4) | (0u << 7) | (b_s8 << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((128u >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void proxy_fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
template <int NC>
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&r)[NC]);
template <>
__device__ __forceinline__ void tmem_ld32<16>(uint32_t taddr, int32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld32<32>(uint32_t taddr, int32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float combine3(int32_t d0, int32_t d1, int32_t d2) {
  return fmaf((float)d2, 65536.0f, fmaf((float)d1, 256.0f, (float)d0));
}
template <int GT>
constexpr uint32_t tc5_npad() { return GT <= 4 ? 16u : 32u; }
template <int GT>
constexpr size_t tc5_smem_bytes() {
  // stages | Bq [NPAD][128] | Bp [NPAD][128] | per head and warp: block max,
  // block sum, sum Y | per head: score unscale, beta | barriers, TMEM slot
  return 1024 + 2 * (size_t)kSlowStage + 2 * (size_t)tc5_npad<GT>() * 128 +
         (size_t)(3 * 32 + 16) * 4 + 6 * 8 + 16;
}
}  // namespace

template <int GT>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32, GT <= 4 ? 3 : 2)
    slow_attn_tc5_kernel(const __grid_constant__ SlowTcArgs a) {
  constexpr int ST = 2;
  constexpr uint32_t NPAD = tc5_npad<GT>();
  constexpr int PL = GT > 4 ? 8 : 4;  // digit plane pl of head h is row PL pl + h
  pdl_wait();  // the union lists (launched chained behind the selection)
  const Geometry& g = a.g;
  const uint32_t G = g.G;
  const uint32_t c = blockIdx.x;
  // ---- balanced schedule (as slow_attn_tc_kernel) ----
  __shared__ uint32_t sched[4];
  __shared__ uint32_t scan_w[8];
  {
    const uint32_t T = blockDim.x, t = threadIdx.x;
    const uint32_t sb = (uint32_t)(((uint64_t)g.S * t) / T), se = (uint32_t)(((uint64_t)g.S * (t + 1)) / T);
    uint32_t mine = 0;
    for (uint32_t x = sb; x < se; ++x) mine += a.union_count[x];
    uint32_t incl = mine;
    const uint32_t ln = t & 31, wp = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (ln >= (uint32_t)o) incl += v;
    }
    if (ln == 31) scan_w[wp] = incl;
    __syncthreads();
    uint32_t before = 0, R = 0;
    for (uint32_t w = 0; w < (T + 31) / 32; ++w) {
      before += w < wp ? scan_w[w] : 0u;
      R += scan_w[w];
    }
    const uint32_t excl = before + incl - mine;
    const uint32_t per = max((R + gridDim.x - 1) / gridDim.x, a.per_min);
    const uint64_t lo = (uint64_t)c * per;
    if (t == 0) sched[2] = lo < R ? (uint32_t)(R - lo < per ? R - lo : per) : 0u;
    if (lo < R && excl <= lo && lo < excl + mine) {
      uint32_t off = excl, x = sb;
      while (off + a.union_count[x] <= lo) off += a.union_count[x++];
      sched[0] = x;
      sched[1] = (uint32_t)(lo - off);
      sched[3] = c - off / per;
    }
    __syncthreads();
  }
  const uint32_t n_rec = sched[2];
  if (n_rec == 0) return;
  const uint32_t s_first = sched[0], i_first = sched[1], slot_first = sched[3];

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sBq = base + ST * kSlowStage;          // [NPAD][128] s8, SW128
  uint8_t* sBp = sBq + NPAD * 128;                // [NPAD/16][128 tok][16] u8, MN-major
  float* redm = reinterpret_cast<float*>(sBp + NPAD * 128);  // [8 heads][4 warps] block max
  float* reds = redm + 32;                                   // [8 heads][4 warps] block sum
  int32_t* redy = reinterpret_cast<int32_t*>(reds + 32);     // [8 heads][4 warps] sum Y
  float* kun = reinterpret_cast<float*>(redy + 32);      // [8] per-head score unscale 2^-k
  float* bst = kun + 8;                                   // [8] beta = q . z
  uint64_t* full = reinterpret_cast<uint64_t*>(bst + 8);
  uint64_t* empty = full + ST;
  uint64_t* bar_qk = empty + ST;
  uint64_t* bar_pv = bar_qk + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_pv + 1);
  __shared__ uint32_t hms[ST];

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kSlowConsumerWarps);
    }
    mbar_init(bar_qk, 1);
    mbar_init(bar_pv, 1);
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: D_qk [0, NPAD), D_pv of the packed bytes [NPAD, 2 NPAD),
                    // of the high nibbles [2 NPAD, 3 NPAD)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(4 * NPAD));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // QK digit-plane rows past the heads stay zero; the last row is all ones
  // (D[tok][NPAD - 1] = sum_c code: the digit offset's correction)
  for (uint32_t i = threadIdx.x; i < NPAD * 128 / 16; i += blockDim.x) {
    const uint32_t v = i / 8 == NPAD - 1 ? 0x01010101u : 0u;
    reinterpret_cast<uint4*>(sBq)[i] = make_uint4(v, v, v, v);
  }
  proxy_fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // producer: the records into the stages (TMA), as slow_attn_tc_kernel
    if (lane == 0) {
      const uint64_t evict_first = l2_evict_first_policy();
      uint32_t s = s_first, ii = i_first, cnt = a.union_count[s];
      for (uint32_t i = 0; i < n_rec; ++i, ++ii) {
        while (ii >= cnt) {
          ii = 0;
          cnt = a.union_count[++s];
        }
        const uint32_t st = i % ST;
        if (i >= ST) mbar_wait_sleep(&empty[st], ((i / ST) - 1) & 1);
        const uint64_t at = (uint64_t)s * g.n_cap + ii;
        const int rec = (int)((uint64_t)s * g.n_cap + a.union_ids[at]);
        uint8_t* dst = base + st * kSlowStage;
        hms[st] = a.union_mask[at];
        mbar_arrive_expect_tx(&full[st], kSlowStage);
        tma_load_3d(dst, &a.tk, 0, 0, rec, &full[st], evict_first);
        tma_load_3d(dst + kKBox, &a.tv, 0, 0, rec, &full[st], evict_first);
        bulk_g2s(dst + kKBox + kVBox, a.params + (uint64_t)rec * kPBytes, kPBytes, &full[st]);
      }
    }
    return;
  }

  // Consumers, software-pipelined over the CTA's records: iteration j runs
  //   B(j): scores, softmax, P words, V(j) expanded over its consumed K codes,
  //         PV(j) issued;
  //   A(j+1): q * s digit planes of the next record, QK(j+1) issued;
  //   C(j): PV(j) read back, the online-softmax update;
  // so each MMA's latency hides behind the other record's ALU phase.  One
  // Bq / Bp tile and one TMEM accumulator per product suffice: each is
  // rewritten only after the MMA that read it was waited on.
  const int nthreads_c = kSlowConsumerWarps * 32;
  const uint32_t ct = threadIdx.x - 32;
  const uint32_t cw = warp - 1;
  const uint32_t tq = (warp & 3) * 32;    // TMEM lane quarter this warp may access
  const uint32_t my_row = tq + lane;      // the token / channel this thread reads from TMEM
  const float sl = (float)a.scale_log2;
  const uint32_t iq = umma_idesc_i8(NPAD, 0, 0, 0);
  // PV, M = 64: the A rows are the 64 bytes of a token's V nibbles (channel
  // pairs 2b, 2b + 1); D rows b land in TMEM lanes 32 (b / 16) + b % 16
  const uint32_t ip = umma_idesc_i8(NPAD, 1, 0, 1) - ((128u >> 4) << 24) + ((64u >> 4) << 24);
  const bool pv_row = lane < 16;               // this thread holds a D_pv row ...
  const uint32_t pb_byte = 16 * (warp & 3) + (lane & 15);  // ... of byte b = channels 2b, 2b + 1

  // record cursors: stream / index within the stream's union of record j (c*)
  // and of record j + 1 (n*)
  uint32_t cs = s_first, cii = i_first, ccnt = a.union_count[s_first];
  // loop-invariant shared-memory offsets: this thread's QK digit words (head
  // cw + 4 rep, channels 4 lane ..), and its token's V nibble / u8 rows
  uint32_t bq_off[(GT + 3) / 4][3];
#pragma unroll
  for (int rep = 0; rep < (GT + 3) / 4; ++rep)
#pragma unroll
    for (int pl = 0; pl < 3; ++pl) bq_off[rep][pl] = sw128(PL * pl + cw + 4 * rep, 4 * lane);
  uint32_t vin_off[4];  // token ct's V nibble row (64B swizzle), relative to the V tile
#pragma unroll
  for (int q = 0; q < 4; ++q) vin_off[q] = ct * 64 + ((q ^ ((ct >> 1) & 3)) << 4);
  auto stage_qk = [&](uint32_t j, uint32_t sj) {  // A(j): digit planes, then QK(j)
    const uint32_t st = j % ST;
    mbar_wait(&full[st], (j / ST) & 1);
    uint8_t* stg = base + st * kSlowStage;
    const float* kp = reinterpret_cast<const float*>(stg + kKBox + kVBox);  // {s,z} x 128
    const float* qb = a.q + (uint64_t)sj * G * 128;
#pragma unroll
    for (int rep = 0; rep < (GT + 3) / 4; ++rep) {
      const uint32_t h = cw + 4 * rep;
      if (h < G) {  // warp-uniform head h, lane = channel quad
        const uint32_t c4 = 4 * lane;
        float4 qv = __ldg(reinterpret_cast<const float4*>(qb + h * 128 + c4));
        qv.x *= sl; qv.y *= sl; qv.z *= sl; qv.w *= sl;  // log2 units
        const float4 sz0 = *reinterpret_cast<const float4*>(kp + 2 * c4);
        const float4 sz1 = *reinterpret_cast<const float4*>(kp + 2 * c4 + 4);
        const float x0 = qv.x * sz0.x, x1 = qv.y * sz0.z, x2 = qv.z * sz1.x, x3 = qv.w * sz1.z;
        const float mx = warp_max_redux(fmaxf(fmaxf(fabsf(x0), fabsf(x1)), fmaxf(fabsf(x2), fabsf(x3))));
        // X = x 2^k with max |x| 2^k < 2^21, offset to X' = X + 2^21 in [0, 2^22):
        // the three low bytes of X' are its u8 digit planes (the offset comes
        // back through the all-ones row: 2^21 sum_c code)
        const int ex = mx > 0.f ? (int)((__float_as_uint(mx) >> 23) & 0xffu) - 127 : 0;
        const int k = max(-120, min(120, 20 - ex));
        const float up = __uint_as_float((uint32_t)(127 + k) << 23);
        const uint32_t X0 = (uint32_t)(__float2int_rn(x0 * up) + (1 << 21));
        const uint32_t X1 = (uint32_t)(__float2int_rn(x1 * up) + (1 << 21));
        const uint32_t X2 = (uint32_t)(__float2int_rn(x2 * up) + (1 << 21));
        const uint32_t X3 = (uint32_t)(__float2int_rn(x3 * up) + (1 << 21));
#pragma unroll
        for (int pl = 0; pl < 3; ++pl) {
          const uint32_t sel = (uint32_t)pl | ((uint32_t)(4 + pl) << 4);
          *reinterpret_cast<uint32_t*>(sBq + bq_off[rep][pl]) =
              __byte_perm(__byte_perm(X0, X1, sel), __byte_perm(X2, X3, sel), 0x5410);
        }
        const float beta = warp_sum(qv.x * sz0.y + qv.y * sz0.w + qv.z * sz1.y + qv.w * sz1.w);
        if (lane == 0) {
          kun[h] = __uint_as_float((uint32_t)(127 - k) << 23);
          bst[h] = beta;
        }
      }
    }
    proxy_fence_async_smem();
    tc_fence_before();
    named_bar(1, nthreads_c);
    if (ct == 0) {  // D_qk[tok][n] = K[tok][.] . Bq[n][.]
      tc_fence_after();
      const uint32_t ka = smem_u32(stg), kb = smem_u32(sBq);
#pragma unroll
      for (uint32_t kk = 0; kk < 4; ++kk)
        umma_i8(tmem, umma_desc_sw128(ka + 32 * kk, 16, 1024),
                umma_desc_sw128(kb + 32 * kk, 16, 1024), iq, kk);
      umma_commit(bar_qk);
    }
  };

  float m_run[GT], l_run[GT], acc[2][GT];  // acc: channels 2b, 2b + 1
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    m_run[h] = -INFINITY;
    l_run[h] = 0.f;
    acc[0][h] = acc[1][h] = 0.f;
  }
  uint32_t seen = 0, slot = slot_first;
  while (cii >= ccnt) {  // (the schedule starts at a record, so this never loops)
    cii = 0;
    ccnt = a.union_count[++cs];
  }
  stage_qk(0, cs);
  for (uint32_t j = 0; j < n_rec; ++j) {
    const uint32_t st = j % ST;
    uint8_t* stg = base + st * kSlowStage;
    const uint8_t* vn = stg + kKBox;
    const float* vp = reinterpret_cast<const float*>(stg + kKBox + kVBox) + 2 * 128;
    const uint32_t hm = hms[st];
    seen |= hm;
    // V params {s, z} of channels 2b, 2b + 1
    const float4 vsz = *reinterpret_cast<const float4*>(vp + 4 * pb_byte);

    // ---- B(j): scores of token my_row, all heads ----
    mbar_wait(bar_qk, j & 1);
    tc_fence_after();
    int32_t dq[NPAD];
    tmem_ld32<NPAD>(tmem + (tq << 16), dq);
    tmem_ld_wait();
    const uint32_t hv = hm & ((1u << G) - 1u);  // heads that selected this record
    const int64_t off21 = (int64_t)dq[NPAD - 1] << 21;  // 2^21 sum_c code[tok][c]
    float sc[GT];
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      sc[h] = -INFINITY;
      if ((hv >> h) & 1u) {
        const int64_t S = (int64_t)dq[h] + ((int64_t)dq[PL + h] << 8) +
                          ((int64_t)dq[2 * PL + h] << 16) - off21;
        sc[h] = fmaf((float)S, kun[h], bst[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      const float bm = warp_max_redux(sc[h]);
      if (lane == 0) redm[h * 4 + cw] = bm;
    }
    named_bar(1, nthreads_c);
    float p[GT], alpha[GT], mnew[GT];
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      const float4 b4 = *reinterpret_cast<const float4*>(redm + 4 * h);
      const float bm = fmaxf(fmaxf(b4.x, b4.y), fmaxf(b4.z, b4.w));
      const bool on = (hv >> h) & 1u;
      mnew[h] = a.literal ? bm : fmaxf(m_run[h], bm);
      p[h] = on ? ex2f(sc[h] - mnew[h]) : 0.f;
      alpha[h] = on ? (a.literal ? 1.f : ex2f(m_run[h] - mnew[h])) : 1.f;
    }
    if (a.literal) {  // each block its own normalized partition (engine.cpp:67-72)
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        const float sm = warp_sum(p[h]);
        if (lane == 0) reds[h * 4 + cw] = sm;
      }
      named_bar(1, nthreads_c);
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        const float4 t4 = *reinterpret_cast<const float4*>(reds + 4 * h);
        const float tot = (t4.x + t4.y) + (t4.z + t4.w);
        if (p[h] > 0.f) p[h] = p[h] / tot;
      }
    }
    // P as Y = p 2^22 (clamped below 2^22): the bytes of Y are its base-256
    // digits, so token my_row's B row is its heads' Y words
    uint32_t yw[GT];
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      yw[h] = min((uint32_t)__float2uint_rn(p[h] * 4194304.0f), 4194303u);
      const uint32_t ys = __reduce_add_sync(0xffffffffu, yw[h]);
      if (lane == 0) redy[h * 4 + cw] = (int32_t)ys;
    }
#pragma unroll
    for (int grp = 0; grp < GT / 4 + (GT < 4 ? 1 : 0); ++grp) {
      uint32_t y4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) y4[e] = 4 * grp + e < GT ? yw[(4 * grp + e) % GT] : 0u;
      *reinterpret_cast<uint4*>(sBp + grp * 2048 + my_row * 16) = make_uint4(y4[0], y4[1], y4[2], y4[3]);
    }
    // PV runs on the V bytes as they arrived (a byte = channel 2b + 16 x
    // channel 2b + 1) and on their high nibbles, written over the consumed K
    // codes in the same 64B-swizzled [token][64 B] layout: lo = D_a - 16 D_b
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = *reinterpret_cast<const uint4*>(stg + kKBox + vin_off[q]);
      *reinterpret_cast<uint4*>(stg + vin_off[q]) =
          make_uint4((u.x >> 4) & 0x0F0F0F0Fu, (u.y >> 4) & 0x0F0F0F0Fu, (u.z >> 4) & 0x0F0F0F0Fu,
                     (u.w >> 4) & 0x0F0F0F0Fu);
    }
    proxy_fence_async_smem();
    tc_fence_before();
    named_bar(1, nthreads_c);
    float lblk[GT];
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      const int4 y4 = *reinterpret_cast<const int4*>(redy + 4 * h);
      lblk[h] = (float)((y4.x + y4.y) + (y4.z + y4.w)) * (1.0f / 4194304.0f);
    }
    if (ct == 0) {  // D_pv[ch][n] = Vx[.][ch] . Bp[n][.]
      tc_fence_after();
      const uint32_t vb = smem_u32(stg + kKBox), vh = smem_u32(stg), pb = smem_u32(sBp);
#pragma unroll
      for (uint32_t kk = 0; kk < 4; ++kk) {  // K = 32 tokens = 2 KB of each [token][64 B] tile
        const uint64_t db = umma_desc_none(pb + 512 * kk, 128, 2048);
        umma_i8(tmem + NPAD, umma_desc_sw64(vb + 2048 * kk, 8192, 512), db, ip, kk);
        umma_i8(tmem + 2 * NPAD, umma_desc_sw64(vh + 2048 * kk, 8192, 512), db, ip, kk);
      }
      umma_commit(bar_pv);
    }

    // ---- A(j+1): the next record's QK, hidden behind PV(j) ----
    const bool stream_end = cii + 1 >= ccnt;  // the stream's union ends at record j
    const bool seg_end = stream_end || j + 1 == n_rec;
    const uint32_t s_this = cs;
    if (j + 1 < n_rec) {
      uint32_t ns = cs, nii = cii + 1, ncnt = ccnt;
      while (nii >= ncnt) {
        nii = 0;
        ncnt = a.union_count[++ns];
      }
      stage_qk(j + 1, ns);
      cs = ns;
      cii = nii;
      ccnt = ncnt;
    }

    // ---- C(j): PV(j) read back, online-softmax update ----
    mbar_wait(bar_pv, j & 1);
    tc_fence_after();
    int32_t da[NPAD], db[NPAD];  // lanes 32 q + [0, 16): byte rows 16 q + lane
    tmem_ld32<NPAD>(tmem + (tq << 16) + NPAD, da);
    tmem_ld32<NPAD>(tmem + (tq << 16) + 2 * NPAD, db);
    tmem_ld_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // the stage (high nibbles over K, V, params) is consumed
    const float vs0 = vsz.x * (1.0f / 4194304.0f), vz0 = vsz.y;
    const float vs1 = vsz.z * (1.0f / 4194304.0f), vz1 = vsz.w;
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      if (!((hv >> h) & 1u)) continue;
      if (pv_row) {
        // channel 2b + 1 = the high nibbles; channel 2b = bytes - 16 x high (exact in s32)
        const float o1 = combine3(db[4 * h], db[4 * h + 1], db[4 * h + 2]);
        const float o0 = combine3(da[4 * h] - 16 * db[4 * h], da[4 * h + 1] - 16 * db[4 * h + 1],
                                  da[4 * h + 2] - 16 * db[4 * h + 2]);
        acc[0][h] = fmaf(acc[0][h], alpha[h], fmaf(vs0, o0, vz0 * lblk[h]));
        acc[1][h] = fmaf(acc[1][h], alpha[h], fmaf(vs1, o1, vz1 * lblk[h]));
      }
      if (a.literal) {
        l_run[h] = 1.f;
      } else {
        l_run[h] = fmaf(l_run[h], alpha[h], lblk[h]);
        m_run[h] = mnew[h];
      }
    }

    if (seg_end) {  // emit the (acc, m, l) partial of every head of stream s_this
      const uint32_t pitch = 128 + 2;
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        if (h >= (int)G) continue;
        float* pp = reinterpret_cast<float*>(a.part) + (((uint64_t)s_this * G + h) * a.nsc + slot) * pitch;
        const bool any = (seen >> h) & 1u;
        if (pv_row)
          *reinterpret_cast<float2*>(pp + 2 * pb_byte) =
              make_float2(any ? acc[0][h] : 0.f, any ? acc[1][h] : 0.f);
        if (ct == 0) {
          pp[128] = any ? (a.literal ? 0.f : m_run[h]) : -INFINITY;
          pp[129] = any ? (a.literal ? 1.f : l_run[h]) : 0.f;
        }
        m_run[h] = -INFINITY;
        l_run[h] = 0.f;
        acc[0][h] = acc[1][h] = 0.f;
      }
      // the stream's last record is here (its union ends at this CTA)
      if (ct == 0 && stream_end) a.nslots[s_this] = slot + 1;
      seen = 0;
      slot = 0;
    }
  }
  tc_fence_before();
  named_bar(1, nthreads_c);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(4 * NPAD));
  }
  pdl_trigger();
}

template <int GT>
static cudaError_t launch_slow_tc5_t(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  const size_t smem = tc5_smem_bytes<GT>();
  auto kern = slow_attn_tc5_kernel<GT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_chained(kern, dim3(grid_ctas), dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
}

static cudaError_t launch_slow_tc5(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  if (a.g.G <= 1) return launch_slow_tc5_t<1>(a, grid_ctas, st);
  if (a.g.G <= 2) return launch_slow_tc5_t<2>(a, grid_ctas, st);
  if (a.g.G <= 4) return launch_slow_tc5_t<4>(a, grid_ctas, st);
  return launch_slow_tc5_t<8>(a, grid_ctas, st);
}

bool slow_tc_supported(const Geometry& g) {
  return g.elem == 2 && g.d_k == 128 && g.d_v == 128 && g.B == 128 && g.kb == 8 && g.vb == 4 &&
         g.G <= 8 && g.rec.kp_off == kKBox + kVBox && g.rec.used == kSlowStage;
}

// 2 stages x 3 CTAs/SM (measured: 1.34 ms vs 1.66 ms for 3 stages x 2 CTAs/SM
// at cfg2); TTKV_SLOW_TC_STAGES=3 selects the deeper ring
static int slow_tc_stages() {
  const char* e = std::getenv("TTKV_SLOW_TC_STAGES");
  return (e && e[0] == '3') ? 3 : 2;
}

// TTKV_SLOW_TC5=0: the mma.sync kernel instead of the tcgen05 one (measurement)
static bool slow_tc5_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TTKV_SLOW_TC5");
    return e && e[0] == '1';
  }();
  return on;
}

uint32_t slow_tc_ctas_per_sm(const Geometry& g) {
  if (slow_tc5_enabled()) return g.G <= 4 ? 3u : 2u;
  return slow_tc_stages() == 3 ? 2u : 3u;
}

template <int GT, int ST>
static size_t slow_tc_smem() {
  return 1024 + (size_t)ST * kSlowStage + slow_tc_tail_bytes<GT>() + 2 * ST * 8;
}

template <int GT, int ST>
static cudaError_t launch_slow_tc_t(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  const size_t smem = slow_tc_smem<GT, ST>();
  auto kern = slow_attn_tc_kernel<GT, ST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_chained(kern, dim3(grid_ctas), dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
}

template <int ST>
static cudaError_t launch_slow_tc_s(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  if (a.g.G <= 1) return launch_slow_tc_t<1, ST>(a, grid_ctas, st);
  if (a.g.G <= 2) return launch_slow_tc_t<2, ST>(a, grid_ctas, st);
  if (a.g.G <= 4) return launch_slow_tc_t<4, ST>(a, grid_ctas, st);
  return launch_slow_tc_t<8, ST>(a, grid_ctas, st);
}

cudaError_t launch_slow_tc(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  if (grid_ctas == 0) return cudaSuccess;
  if (slow_tc5_enabled()) return launch_slow_tc5(a, grid_ctas, st);
  static const int stages = slow_tc_stages();
  return stages == 2 ? launch_slow_tc_s<2>(a, grid_ctas, st)
                     : launch_slow_tc_s<3>(a, grid_ctas, st);
}

template <int GT>
static cudaError_t launch_slow_tc_spec_t(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  // 2 stages | qsf + phl | sc | usc, mst, pst, bst | srec | full, empty
  const size_t smem = 1024 + 2 * (size_t)kSlowStage + 2 * 256 * 16 + (size_t)GT * kScPitch * 4 +
                      4 * 8 * 4 + 16 + 2 * 2 * 8;
  auto kern = slow_attn_tc_spec_kernel<GT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_chained(kern, dim3(grid_ctas), dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
}

bool slow_tc_spec_supported(const Geometry& g) { return slow_tc_supported(g) && g.G <= 4; }

cudaError_t launch_slow_tc_spec(const SlowTcArgs& a, uint32_t grid_ctas, cudaStream_t st) {
  if (grid_ctas == 0 || a.spec_n == 0) return cudaSuccess;
  if (a.g.G <= 1) return launch_slow_tc_spec_t<1>(a, grid_ctas, st);
  if (a.g.G <= 2) return launch_slow_tc_spec_t<2>(a, grid_ctas, st);
  return launch_slow_tc_spec_t<4>(a, grid_ctas, st);
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
static cudaError_t launch_fast_tc_t(const FastTcArgs& a, cudaStream_t st, int chained) {
  const size_t smem = fast_tc_smem(a.g);
  auto kern = fast_attn_tc_kernel<ND, GT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max smem
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nfc, a.g.S);
  if (chained == 1) return launch_chained(kern, grid, dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
  if (chained == 2)
    return launch_chained_background(kern, grid, dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
  return launch_background(kern, grid, dim3(32 + kSlowConsumerWarps * 32), smem, st, a);
}

template <int ND>
static cudaError_t launch_fast_tc_g(const FastTcArgs& a, cudaStream_t st, int chained) {
  if (a.g.G <= 1) return launch_fast_tc_t<ND, 1>(a, st, chained);
  if (a.g.G <= 2) return launch_fast_tc_t<ND, 2>(a, st, chained);
  if (a.g.G <= 4) return launch_fast_tc_t<ND, 4>(a, st, chained);
  return launch_fast_tc_t<ND, 8>(a, st, chained);
}

cudaError_t launch_fast_tc(const FastTcArgs& a, cudaStream_t st, int chained) {
  return a.g.d_k == 128 ? launch_fast_tc_g<2>(a, st, chained) : launch_fast_tc_g<1>(a, st, chained);
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
