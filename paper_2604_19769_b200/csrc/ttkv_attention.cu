// ttkv_attention.cu -- block-wise streaming decode attention on B200.
//
// Replaces the three accumulation loops of Engine::decode_step
// (engine.cpp:36-40 fast tier, 61-83 fetched blocks, 85-86 finalize) and the
// AttentionAccumulator they drive (attention.hpp:29-61).  Every partition
// produces an online-softmax partial (m, l, acc) in log2 units and
// combine_partials merges them by LSE rescaling -- the exact merge the
// reference proves partition-invariant.
//
//  fast_attn_partial  split-K over the fp16/fp32 HBM ring.  Each lane owns 4
//                     channels (8-byte / 16-byte coalesced loads), the G query
//                     heads of a KV head share every K/V load (GQA), dot
//                     products reduce with warp shuffles.  HBM-bound:
//                     F * (d_k + d_v) * elem bytes per stream.
//  slow_stream_attn   one producer warp streams the selected records of a
//                     stream from pinned host DRAM (zero-copy over PCIe) into
//                     a ring of shared-memory stages with cp.async.bulk +
//                     mbarrier complete_tx (or 16-byte LDG when copy_mode=2);
//                     four consumer warps dequantize in registers
//                     (x = code * scale + zp, quantizer.cpp:109-110) fused into
//                     QK and PV for all G heads, so transfer of block i+1..i+NS
//                     overlaps compute of block i.  Each record crosses PCIe
//                     once per step, shared by every head that selected it.
//                     PCIe-bound: union_blocks * 26,624 B per step.
//  combine_partials   per (stream, head) LSE merge + normalisation
//                     (attention.hpp:54-61).
#include <math.h>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"

namespace ttkv_dev {

// ---------------------------------------------------------------------------
// fast tier
// ---------------------------------------------------------------------------
template <typename T, int GT>
__global__ void __launch_bounds__(kFastWarps * 32) fast_attn_kernel(FastArgs a) {
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, f = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t c0 = lane * 4;
  const uint32_t t0 = f * a.FC;
  const uint32_t t1 = min(t0 + a.FC, a.F);
  const bool vec_k = (g.d_k & 3) == 0, vec_v = (g.d_v & 3) == 0;

  float qr[GT][4];
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      qr[h][j] = (h < (int)g.G && c0 + j < g.d_k)
                     ? a.q[((uint64_t)s * g.G + h) * g.d_k + c0 + j] * a.scale_log2
                     : 0.0f;
  float m[GT], l[GT], acc[GT][4];
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.0f;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[h][j] = 0.0f;
  }

  const T* rk = static_cast<const T*>(a.ring_k) + (uint64_t)s * g.C * g.d_k;
  const T* rv = static_cast<const T*>(a.ring_v) + (uint64_t)s * g.C * g.d_v;
  for (uint32_t t = t0 + warp; t < t1; t += kFastWarps) {
    const uint64_t slot = (a.front + t) % g.C;
    float kf[4], vf[4];
    if (vec_k && c0 < g.d_k) {
      load4(rk + slot * g.d_k + c0, kf);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) kf[j] = c0 + j < g.d_k ? to_f(rk[slot * g.d_k + c0 + j]) : 0.0f;
    }
    if (vec_v && c0 < g.d_v) {
      load4(rv + slot * g.d_v + c0, vf);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) vf[j] = c0 + j < g.d_v ? to_f(rv[slot * g.d_v + c0 + j]) : 0.0f;
    }
#pragma unroll
    for (int h = 0; h < GT; ++h) {
      if (h >= (int)g.G) break;
      float d = qr[h][0] * kf[0] + qr[h][1] * kf[1] + qr[h][2] * kf[2] + qr[h][3] * kf[3];
      d = warp_sum(d);
      if (d > m[h]) {
        const float alpha = exp2f(m[h] - d);
        l[h] *= alpha;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[h][j] *= alpha;
        m[h] = d;
      }
      const float p = exp2f(d - m[h]);
      l[h] += p;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[h][j] += p * vf[j];
    }
  }

  // merge the warps' partials
  __shared__ float sm_m[kFastWarps][kMaxG], sm_l[kFastWarps][kMaxG];
  __shared__ float sm_acc[kFastWarps][kMaxG][kMaxD];
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    if (h >= (int)g.G) break;
    if (lane == 0) { sm_m[warp][h] = m[h]; sm_l[warp][h] = l[h]; }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c0 + j < g.d_v) sm_acc[warp][h][c0 + j] = acc[h][j];
  }
  __syncthreads();
  const uint32_t pitch = g.d_v + 2;
  for (uint32_t i = threadIdx.x; i < g.G * g.d_v; i += blockDim.x) {
    const uint32_t h = i / g.d_v, c = i % g.d_v;
    float M = -INFINITY;
    for (int w = 0; w < kFastWarps; ++w) M = fmaxf(M, sm_m[w][h]);
    float L = 0.0f, A = 0.0f;
    if (M != -INFINITY) {
      for (int w = 0; w < kFastWarps; ++w) {
        const float sc = exp2f(sm_m[w][h] - M);
        L += sm_l[w][h] * sc;
        A += sm_acc[w][h][c] * sc;
      }
    }
    float* p = a.part + (((uint64_t)s * g.G + h) * a.nfc + f) * pitch;
    p[c] = A;
    if (c == 0) { p[g.d_v] = M; p[g.d_v + 1] = L; }
  }
}

template <typename T>
static cudaError_t launch_fast_t(const FastArgs& a, cudaStream_t st) {
  dim3 grid(a.nfc, a.g.S);
  if (a.g.G <= 1) fast_attn_kernel<T, 1><<<grid, kFastWarps * 32, 0, st>>>(a);
  else if (a.g.G <= 2) fast_attn_kernel<T, 2><<<grid, kFastWarps * 32, 0, st>>>(a);
  else if (a.g.G <= 4) fast_attn_kernel<T, 4><<<grid, kFastWarps * 32, 0, st>>>(a);
  else fast_attn_kernel<T, 8><<<grid, kFastWarps * 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fast(const FastArgs& a, cudaStream_t st) {
  return a.g.elem == 2 ? launch_fast_t<__half>(a, st) : launch_fast_t<float>(a, st);
}

// ---------------------------------------------------------------------------
// slow tier: streamed, dequant fused
// ---------------------------------------------------------------------------

// Dequantize the 4 channels [c0, c0+4) of row t of a packed tensor.
// KB: compile-time bit width (8, 4) or 0 = runtime `bits` (2..8 or 16).
template <int KB, typename T>
__device__ __forceinline__ void dequant4(const uint8_t* payload, uint32_t t, uint32_t c0,
                                         uint32_t dim, uint32_t bits, const float (&sc)[4],
                                         const float (&zp)[4], float (&o)[4]) {
  if constexpr (KB == 8) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(payload + t * dim + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = fmaf((float)((w >> (8 * j)) & 0xffu), sc[j], zp[j]);
  } else if constexpr (KB == 4) {
    const uint32_t w = *reinterpret_cast<const uint16_t*>(payload + ((t * dim + c0) >> 1));
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = fmaf((float)((w >> (4 * j)) & 0xfu), sc[j], zp[j]);
  } else {
    if (bits == 16) {
      const T* e = reinterpret_cast<const T*>(payload) + (uint64_t)t * dim;
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = c0 + j < dim ? to_f(e[c0 + j]) : 0.0f;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = c0 + j < dim ? fmaf((float)extract_code(payload, t * dim + c0 + j, bits), sc[j], zp[j])
                            : 0.0f;
    }
  }
}

template <typename T, int KB, int VB, int GT, int COPY>
__global__ void __launch_bounds__(32 + kSlowConsumerWarps * 32) slow_attn_kernel(SlowArgs a) {
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y, chunk = blockIdx.x;
  const uint32_t cnt = a.union_count[s];
  const uint32_t i0 = chunk * a.CH;
  if (i0 >= cnt) return;  // uniform across the CTA
  const uint32_t nb = min(i0 + a.CH, cnt) - i0;
  const uint32_t NS = a.stages;
  const uint32_t stride = g.rec.stride;

  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stages = smem;                                             // [NS][stride]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stage_region);  // [NS]
  uint64_t* empty = full + NS;                                        // [NS]
  float* sc = reinterpret_cast<float*>(empty + NS);                   // [2][GT][B]
  float* mst = sc + 2 * GT * g.B;                                     // [GT]
  float* lst = mst + GT;                                              // [GT]
  float* ast = lst + GT;                                              // [GT]

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < NS; ++i) {
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

  const uint32_t* uids = a.union_ids + (uint64_t)s * g.n_cap + i0;
  const uint32_t* umask = a.union_mask + (uint64_t)s * g.n_cap + i0;
  const uint8_t* arena_s = a.arena + (uint64_t)s * g.n_cap * stride;

  if (warp == 0) {
    // ---------------- producer ----------------
    for (uint32_t i = 0; i < nb; ++i) {
      const uint32_t st = i % NS;
      if (i >= NS) mbar_wait(&empty[st], ((i / NS) - 1) & 1);
      const uint32_t blk = uids[i];
      const uint8_t* src = arena_s + (uint64_t)blk * stride;
      const uint32_t pay = g.rec.kp_off, pbytes = g.rec.used - g.rec.kp_off;
      const uint8_t* psrc = a.params + ((uint64_t)s * g.n_cap + blk) * pbytes;
      uint8_t* dst = stages + st * stride;
      if constexpr (COPY == 1) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], g.rec.used);
          for (uint32_t off = 0; off < pay; off += 16384u)
            bulk_g2s(dst + off, src + off, min(16384u, pay - off), &full[st]);
          if (pbytes) bulk_g2s(dst + pay, psrc, pbytes, &full[st]);
        }
      } else {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const uint32_t n16 = pay >> 4;
        uint32_t j = lane;
        for (; j + 7 * 32 < n16; j += 8 * 32) {
          uint4 r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) r[u] = s4[j + u * 32];
#pragma unroll
          for (int u = 0; u < 8; ++u) d4[j + u * 32] = r[u];
        }
        for (; j < n16; j += 32) d4[j] = s4[j];
        const uint4* p4 = reinterpret_cast<const uint4*>(psrc);
        uint4* dp4 = reinterpret_cast<uint4*>(dst + pay);
        for (uint32_t jj = lane; jj < (pbytes >> 4); jj += 32) dp4[jj] = p4[jj];
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const uint32_t cw = warp - 1;
  const uint32_t c0 = lane * 4;
  const int nthreads_c = kSlowConsumerWarps * 32;
  float qr[GT][4];
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      qr[h][j] = (h < (int)g.G && c0 + j < g.d_k)
                     ? a.q[((uint64_t)s * g.G + h) * g.d_k + c0 + j] * a.scale_log2
                     : 0.0f;
  float acc[GT][4];
#pragma unroll
  for (int h = 0; h < GT; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[h][j] = 0.0f;
  uint32_t seen = 0;  // heads that absorbed at least one block in this chunk

  for (uint32_t i = 0; i < nb; ++i) {
    const uint32_t st = i % NS;
    mbar_wait(&full[st], (i / NS) & 1);
    const uint8_t* rec = stages + st * stride;
    const uint32_t hm = umask[i];
    seen |= hm;
    float* scb = sc + (i & 1) * GT * g.B;

    // ---- QK: dequantized keys, all heads share each row ----
    {
      float ks[4], kz[4];
      const float* kp = reinterpret_cast<const float*>(rec + g.rec.kp_off);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = g.kb != 16 && c0 + j < g.d_k;
        ks[j] = ok ? kp[2 * (c0 + j)] : 0.0f;
        kz[j] = ok ? kp[2 * (c0 + j) + 1] : 0.0f;
      }
      for (uint32_t t = cw; t < g.B; t += kSlowConsumerWarps) {
        float kf[4];
        if (c0 < g.d_k) dequant4<KB, T>(rec, t, c0, g.d_k, g.kb, ks, kz, kf);
        else kf[0] = kf[1] = kf[2] = kf[3] = 0.0f;
#pragma unroll
        for (int h = 0; h < GT; ++h) {
          if (h >= (int)g.G) break;
          if (!((hm >> h) & 1u)) continue;
          float d = qr[h][0] * kf[0] + qr[h][1] * kf[1] + qr[h][2] * kf[2] + qr[h][3] * kf[3];
          d = warp_sum(d);
          if (lane == 0) scb[h * g.B + t] = d;
        }
      }
    }
    named_bar(1, nthreads_c);

    // ---- block softmax statistics (one warp per head) ----
    for (uint32_t h = cw; h < g.G; h += kSlowConsumerWarps) {
      if (!((hm >> h) & 1u)) {
        if (lane == 0) ast[h] = 1.0f;
        continue;
      }
      float* row = scb + h * g.B;
      float bm = -INFINITY;
      for (uint32_t t = lane; t < g.B; t += 32) bm = fmaxf(bm, row[t]);
      bm = warp_max(bm);
      const float m_old = mst[h];
      const float m_new = a.literal ? bm : fmaxf(m_old, bm);
      float sum = 0.0f;
      for (uint32_t t = lane; t < g.B; t += 32) {
        const float p = exp2f(row[t] - m_new);
        row[t] = p;
        sum += p;
      }
      sum = warp_sum(sum);
      __syncwarp();
      if (a.literal) {
        // literal additive merge (engine.cpp:67-72): each block is its own
        // normalized partition, summed without rescaling
        const float inv = 1.0f / sum;
        for (uint32_t t = lane; t < g.B; t += 32) row[t] *= inv;
        if (lane == 0) ast[h] = 1.0f;
        continue;
      }
      if (lane == 0) {
        const float alpha = exp2f(m_old - m_new);  // 0 when m_old = -inf
        lst[h] = lst[h] * alpha + sum;
        mst[h] = m_new;
        ast[h] = alpha;
      }
    }
    named_bar(1, nthreads_c);

    // ---- PV: dequantized values ----
    {
#pragma unroll
      for (int h = 0; h < GT; ++h) {
        if (h >= (int)g.G) break;
        if (!((hm >> h) & 1u)) continue;
        const float alpha = ast[h];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[h][j] *= alpha;
      }
      float vs[4], vz[4];
      const float* vp = reinterpret_cast<const float*>(rec + g.rec.vp_off);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = g.vb != 16 && c0 + j < g.d_v;
        vs[j] = ok ? vp[2 * (c0 + j)] : 0.0f;
        vz[j] = ok ? vp[2 * (c0 + j) + 1] : 0.0f;
      }
      const uint8_t* vpay = rec + g.rec.v_off;
      for (uint32_t t = cw; t < g.B; t += kSlowConsumerWarps) {
        float vf[4];
        if (c0 < g.d_v) dequant4<VB, T>(vpay, t, c0, g.d_v, g.vb, vs, vz, vf);
        else vf[0] = vf[1] = vf[2] = vf[3] = 0.0f;
#pragma unroll
        for (int h = 0; h < GT; ++h) {
          if (h >= (int)g.G) break;
          if (!((hm >> h) & 1u)) continue;
          const float p = scb[h * g.B + t];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[h][j] = fmaf(p, vf[j], acc[h][j]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ---- merge the consumer warps' accumulators, emit the chunk partial ----
  named_bar(1, nthreads_c);
  float* red = reinterpret_cast<float*>(stages);  // reuse stage memory
#pragma unroll
  for (int h = 0; h < GT; ++h) {
    if (h >= (int)g.G) break;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c0 + j < g.d_v) red[(cw * GT + h) * g.d_v + c0 + j] = acc[h][j];
  }
  named_bar(1, nthreads_c);
  const uint32_t pitch = g.d_v + 2;
  const uint32_t ct = threadIdx.x - 32;
  for (uint32_t i = ct; i < g.G * g.d_v; i += nthreads_c) {
    const uint32_t h = i / g.d_v, c = i % g.d_v;
    float A = 0.0f;
    for (int w = 0; w < kSlowConsumerWarps; ++w) A += red[(w * GT + h) * g.d_v + c];
    float* p = a.part + (((uint64_t)s * g.G + h) * a.nsc + chunk) * pitch;
    const bool any = (seen >> h) & 1u;
    p[c] = any ? A : 0.0f;
    if (c == 0) {
      p[g.d_v] = any ? (a.literal ? 0.0f : mst[h]) : -INFINITY;
      p[g.d_v + 1] = any ? (a.literal ? 1.0f : lst[h]) : 0.0f;
    }
  }
}

static size_t slow_fixed_smem(const Geometry& g, uint32_t GT) {
  return (size_t)2 * GT * g.B * 4 + 3 * GT * 4 + 64;
}

uint32_t slow_stages_for(const Geometry& g) {
  const size_t budget = 110 * 1024;  // two CTAs per SM
  const size_t fixed = slow_fixed_smem(g, kMaxG);
  size_t ns = budget > fixed ? (budget - fixed) / (g.rec.stride + 16) : 0;
  if (ns > 4) ns = 4;
  if (ns < 1) {  // large records: one CTA per SM
    const size_t big = 220 * 1024;
    ns = big > fixed ? (big - fixed) / (g.rec.stride + 16) : 0;
    if (ns > 2) ns = 2;
  }
  return (uint32_t)ns;
}

template <typename T, int KB, int VB, int GT, int COPY>
static cudaError_t launch_slow_t(const SlowArgs& a, uint32_t grid_chunks, cudaStream_t st) {
  const Geometry& g = a.g;
  SlowArgs b = a;
  const size_t red = (size_t)kSlowConsumerWarps * GT * g.d_v * 4;
  b.stage_region = (uint32_t)((size_t)a.stages * g.rec.stride > red ? (size_t)a.stages * g.rec.stride : red);
  b.stage_region = (b.stage_region + 15u) & ~15u;
  const size_t smem = (size_t)b.stage_region + 16 * a.stages + slow_fixed_smem(g, GT);
  auto kern = slow_attn_kernel<T, KB, VB, GT, COPY>;
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

// ---------------------------------------------------------------------------
// combine
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) combine_kernel(CombineArgs a) {
  const Geometry& g = a.g;
  const uint32_t idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (idx >= g.S * g.G) return;
  const uint32_t s = idx / g.G;
  const uint32_t pitch = g.d_v + 2;
  const uint32_t nsc_used = a.union_count ? (a.union_count[s] + a.CH - 1) / a.CH : 0u;
  const float* fp = a.fpart + (uint64_t)idx * a.nfc * pitch;
  const float* sp = a.spart ? a.spart + (uint64_t)idx * a.nsc * pitch : nullptr;

  // literal additive merge: slow partials are already normalized sums
  const uint32_t nlse = a.literal ? 0u : nsc_used;
  float M = -INFINITY;
  for (uint32_t i = lane; i < a.nfc; i += 32)
    if (fp[i * pitch + g.d_v + 1] > 0.0f) M = fmaxf(M, fp[i * pitch + g.d_v]);
  for (uint32_t i = lane; i < nlse; i += 32)
    if (sp[i * pitch + g.d_v + 1] > 0.0f) M = fmaxf(M, sp[i * pitch + g.d_v]);
  M = warp_max(M);

  float L = 0.0f;
  for (uint32_t i = lane; i < a.nfc; i += 32) {
    const float l = fp[i * pitch + g.d_v + 1];
    if (l > 0.0f) L += l * exp2f(fp[i * pitch + g.d_v] - M);
  }
  for (uint32_t i = lane; i < nlse; i += 32) {
    const float l = sp[i * pitch + g.d_v + 1];
    if (l > 0.0f) L += l * exp2f(sp[i * pitch + g.d_v] - M);
  }
  L = warp_sum(L);
  const float inv = 1.0f / L;

  for (uint32_t c = lane; c < g.d_v; c += 32) {
    float A = 0.0f;
    for (uint32_t i = 0; i < a.nfc; ++i) {
      const float l = fp[i * pitch + g.d_v + 1];
      if (l > 0.0f) A += fp[i * pitch + c] * exp2f(fp[i * pitch + g.d_v] - M);
    }
    for (uint32_t i = 0; i < nlse; ++i) {
      const float l = sp[i * pitch + g.d_v + 1];
      if (l > 0.0f) A += sp[i * pitch + c] * exp2f(sp[i * pitch + g.d_v] - M);
    }
    float o = A * inv;
    if (a.literal)
      for (uint32_t i = 0; i < nsc_used; ++i)
        if (sp[i * pitch + g.d_v + 1] > 0.0f) o += sp[i * pitch + c];
    a.out[(uint64_t)idx * g.d_v + c] = o;
  }
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  const uint32_t warps = a.g.S * a.g.G;
  combine_kernel<<<(warps + 7) / 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ttkv_dev
