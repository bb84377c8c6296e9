// ttkv_quantize.cu -- evict_quantize: bit-exact K/V block quantization on B200.
//
// Replaces TierStore::evict_and_compress (tier_store.cpp:71-98) +
// quantize_block / quantize_tensor / pack_codes (quantizer.cpp:126-155, 51-88,
// 22-32).  One CTA per (block, stream); one thread per channel walks the
// block's rows sequentially in fp64 exactly as the reference does:
//   lo/hi with std::min/std::max tie semantics (quantizer.cpp:66-72),
//   scale = float((double(hi) - lo) / levels)            (77-78),
//   code  = clamp(round((double(x) - lo) / scale), 0, L) (80-84),
//   centroid = float(sum_r double(key) / n)              (141-148),
// with __dadd_rn/__dsub_rn/__ddiv_rn so nothing is FMA-contracted.  Codes are
// packed LSB-first in smem, then the finished record is written to the arena
// (pinned host DRAM through the mapping = zero-copy PCIe stores, or HBM) with
// 16-byte coalesced stores.  Centroids go to HBM.
//
// Roofline: per block it reads B*(d_k+d_v)*elem bytes from HBM (64 KB at
// K/V fp16 128x128) and writes one record (26,624 B) to the arena; the fp64
// divide per element is the ALU cost (~40 DFMA-equivalents).
#include <algorithm>
#include <cstdlib>

#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"

namespace ttkv_dev {

template <typename T, typename Tin>
__global__ void evict_quantize_kernel(EvictArgs a) {
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y;
  const uint64_t blk = a.first_block + blockIdx.x;
  const uint64_t pos0 = blk * g.B;
  const uint32_t dkv = g.d_k + g.d_v;

  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* rec = smem;                             // [stride]
  uint8_t* codes = smem + g.rec.stride;            // [B][d_k + d_v]

  const T* ring_k = static_cast<const T*>(a.ring_k) + (uint64_t)s * g.C * g.d_k;
  const T* ring_v = static_cast<const T*>(a.ring_v) + (uint64_t)s * g.C * g.d_v;
  const Tin* in_k = static_cast<const Tin*>(a.in_k) + (uint64_t)s * a.in_tokens * g.d_k;
  const Tin* in_v = static_cast<const Tin*>(a.in_v) + (uint64_t)s * a.in_tokens * g.d_v;

  // zero the record (padding bytes are deterministic)
  for (uint32_t i = threadIdx.x * 16; i < g.rec.stride; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(rec + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();

  const uint32_t c = threadIdx.x;
  if (c < dkv) {
    const bool is_k = c < g.d_k;
    const uint32_t ch = is_k ? c : c - g.d_k;
    const uint32_t dim = is_k ? g.d_k : g.d_v;
    const uint32_t bits = is_k ? g.kb : g.vb;
    const T* ring = is_k ? ring_k : ring_v;
    const Tin* in = is_k ? in_k : in_v;
    // A block never straddles the ring wrap (C and every eviction start are
    // multiples of B), so its ring rows are slot0 .. slot0 + B - 1; rows at
    // positions >= split_pos come from the staging input instead.
    const T* ring_col = ring + (pos0 % g.C) * dim + ch;
    const uint32_t n_ring = a.split_pos > pos0
                                ? (uint32_t)(a.split_pos - pos0 < (uint64_t)g.B ? a.split_pos - pos0 : (uint64_t)g.B)
                                : 0u;
    const Tin* in_col = in + (pos0 + n_ring - a.split_pos) * dim + ch;  // row n_ring
    auto load = [&](uint32_t r) -> float {
      if (r < n_ring) return to_f(ring_col[(size_t)r * dim]);
      return through<T, Tin>(in_col[(size_t)(r - n_ring) * dim]);
    };

    // rows are read kU at a time so kU loads are in flight per thread (the
    // per-row dependence is only through lo/hi/sum, in row order as the
    // reference walks them)
    constexpr uint32_t kU = 8;
    float lo = __int_as_float(0x7f800000);   // +inf
    float hi = __int_as_float(0xff800000);   // -inf
    double sum = 0.0;
    for (uint32_t r0 = 0; r0 < g.B; r0 += kU) {
      float x[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) x[u] = r0 + u < g.B ? load(r0 + u) : 0.0f;
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        if (r0 + u >= g.B) break;
        lo = (x[u] < lo) ? x[u] : lo;   // std::min(lo, x)
        hi = (hi < x[u]) ? x[u] : hi;   // std::max(hi, x)
        if (is_k) sum = __dadd_rn(sum, (double)x[u]);
      }
    }
    if (is_k)
      a.cent[((uint64_t)s * g.n_cap + blk) * g.d_k + ch] =
          __double2float_rn(__ddiv_rn(sum, (double)g.B));

    if (bits == 16) {
      // lossless passthrough: the ring element itself (quantizer.cpp:55-59)
      T* dst = reinterpret_cast<T*>(rec + (is_k ? 0u : g.rec.v_off));
      for (uint32_t r = 0; r < g.B; ++r) dst[r * dim + ch] = from_f<T>(load(r));
    } else {
      float scale, zp = lo;
      uint8_t* cc = codes + ch + (is_k ? 0u : g.d_k);
      if (hi == lo) {
        scale = 1.0f;
        for (uint32_t r = 0; r < g.B; ++r) cc[r * dkv] = 0;
      } else {
        const double levels = (double)((1u << bits) - 1u);
        scale = __double2float_rn(__ddiv_rn(__dsub_rn((double)hi, (double)lo), levels));
        const double dlo = (double)lo, dscale = (double)scale;
        // code = round(a / scale) with a = x - lo.  The product with the
        // rounded reciprocal is within a few ulp of the correctly rounded
        // quotient, so the two round to the same integer unless the quotient
        // sits within 2^-36 of a half-integer; those rare elements take the
        // exact __ddiv_rn the reference uses (quantizer.cpp:80-84).
        const double rcp = __drcp_rn(dscale);
        for (uint32_t r0 = 0; r0 < g.B; r0 += kU) {
          float x[kU];
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u) x[u] = r0 + u < g.B ? load(r0 + u) : 0.0f;
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u) {
            if (r0 + u >= g.B) break;
            const double a = __dsub_rn((double)x[u], dlo);
            const double t = __dmul_rn(a, rcp);
            const double fr = t - floor(t);
            double q = fabs(fr - 0.5) > 0x1p-36 ? round(t) : round(__ddiv_rn(a, dscale));
            q = q < 0.0 ? 0.0 : (levels < q ? levels : q);
            cc[(r0 + u) * dkv] = (uint8_t)(uint32_t)q;
          }
        }
      }
      float* par = reinterpret_cast<float*>(rec + (is_k ? g.rec.kp_off : g.rec.vp_off)) + 2 * ch;
      par[0] = scale;
      par[1] = zp;
    }
  }
  __syncthreads();

  // LSB-first packing over the flat row-major index (quantizer.cpp:22-32)
  for (int t = 0; t < 2; ++t) {
    const uint32_t bits = t == 0 ? g.kb : g.vb;
    if (bits == 16) continue;
    const uint32_t dim = t == 0 ? g.d_k : g.d_v;
    const uint32_t coff = t == 0 ? 0u : g.d_k;
    const uint32_t nbytes = t == 0 ? g.rec.k_bytes : g.rec.v_bytes;
    uint8_t* dst = rec + (t == 0 ? 0u : g.rec.v_off);
    for (uint32_t j = threadIdx.x; j < nbytes; j += blockDim.x) {
      uint32_t byte = 0;
      if (bits == 8) {
        byte = codes[(j / dim) * dkv + coff + j % dim];
      } else if (bits == 4) {
        const uint32_t i0 = 2 * j, i1 = 2 * j + 1;
        byte = codes[(i0 / dim) * dkv + coff + i0 % dim];
        if (i1 < g.B * dim) byte |= (uint32_t)codes[(i1 / dim) * dkv + coff + i1 % dim] << 4;
      } else {
        const uint32_t b0 = 8 * j, total = g.B * dim;
        for (uint32_t i = b0 / bits; i < total && i * bits < b0 + 8; ++i) {
          const uint32_t v = codes[(i / dim) * dkv + coff + i % dim];
          const int sh = (int)(i * bits) - (int)b0;
          byte |= sh >= 0 ? (v << sh) : (v >> (-sh));
        }
        byte &= 0xffu;
      }
      dst[j] = (uint8_t)byte;
    }
  }
  __syncthreads();

  // record -> arena (pinned DRAM via PCIe posted writes, or HBM)
  uint8_t* out = a.arena + ((uint64_t)s * g.n_cap + blk) * g.rec.stride;
  for (uint32_t i = threadIdx.x * 16; i < g.rec.stride; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(out + i) = *reinterpret_cast<const uint4*>(rec + i);
  // params -> HBM mirror (staged by slow_stream_attn from HBM, not PCIe)
  const uint32_t pbytes = g.rec.used - g.rec.kp_off;
  if (a.params && pbytes) {
    uint8_t* pm = a.params + ((uint64_t)s * g.n_cap + blk) * pbytes;
    for (uint32_t i = threadIdx.x * 16; i < pbytes; i += blockDim.x * 16)
      *reinterpret_cast<uint4*>(pm + i) = *reinterpret_cast<const uint4*>(rec + g.rec.kp_off + i);
  }
}

// ---------------------------------------------------------------------------
// Staged variant: one CTA per (block, stream, tensor).  The block's rows are
// first copied into shared memory with 16-byte cp.async (every load in
// flight at once), then each thread walks its channel's column from shared
// memory with the same sequential fp64 recipe as above.  The key CTA owns the
// record bytes [0, v_off) and [kp_off, vp_off), the value CTA [v_off, kp_off)
// and [vp_off, stride), so the two halves of a record are written by
// different CTAs without overlap; padding is written as zeros.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ uint32_t al16(uint32_t x) { return (x + 15u) & ~15u; }

template <typename T, typename Tin>
__global__ void __launch_bounds__(128) evict_staged_kernel(EvictArgs a) {
  const Geometry& g = a.g;
  const uint32_t s = blockIdx.y;
  const bool is_k = blockIdx.z == 0;
  const uint64_t blk = a.first_block + blockIdx.x;
  const uint64_t pos0 = blk * g.B;
  const uint32_t B = g.B;
  const uint32_t dim = is_k ? g.d_k : g.d_v, bits = is_k ? g.kb : g.vb;
  const uint32_t n_ring =
      a.split_pos > pos0 ? (uint32_t)(a.split_pos - pos0 < B ? a.split_pos - pos0 : B) : 0u;
  const RecordLayout& L = g.rec;
  const uint32_t lo0 = is_k ? 0u : L.v_off, hi0 = is_k ? L.v_off : L.kp_off;
  const uint32_t lo1 = is_k ? L.kp_off : L.vp_off, hi1 = is_k ? L.vp_off : L.stride;

  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t ring_bytes = n_ring * dim * (uint32_t)sizeof(T);
  const uint32_t in_bytes = (B - n_ring) * dim * (uint32_t)sizeof(Tin);
  uint8_t* tile_r = smem;
  uint8_t* tile_i = smem + al16(ring_bytes);
  const uint32_t tile_max = B * dim * (uint32_t)(sizeof(T) > sizeof(Tin) ? sizeof(T) : sizeof(Tin));
  uint8_t* codes = smem + al16(tile_max) + 16;
  uint8_t* img0 = codes + al16(B * dim);  // record bytes [lo0, hi0)
  uint8_t* img1 = img0 + (hi0 - lo0);     // record bytes [lo1, hi1)

  // ---- stage the rows (ring part contiguous: a block never straddles the wrap)
  {
    const T* ring = static_cast<const T*>(is_k ? a.ring_k : a.ring_v) +
                    ((uint64_t)s * g.C + pos0 % g.C) * dim;
    const Tin* in = static_cast<const Tin*>(is_k ? a.in_k : a.in_v) +
                    ((uint64_t)s * a.in_tokens + (pos0 + n_ring - a.split_pos)) * dim;
    for (uint32_t o = threadIdx.x * 16; o < ring_bytes; o += blockDim.x * 16)
      cp_async16(tile_r + o, reinterpret_cast<const uint8_t*>(ring) + o);
    for (uint32_t o = threadIdx.x * 16; o < in_bytes; o += blockDim.x * 16)
      cp_async16(tile_i + o, reinterpret_cast<const uint8_t*>(in) + o);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (uint32_t o = threadIdx.x * 16; o < (hi0 - lo0) + (hi1 - lo1); o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(img0 + o) = make_uint4(0, 0, 0, 0);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  const uint32_t c = threadIdx.x;
  if (c < dim) {
    const T* tr = reinterpret_cast<const T*>(tile_r) + c;
    const Tin* ti = reinterpret_cast<const Tin*>(tile_i) + c;
    auto val = [&](uint32_t r) -> float {
      return r < n_ring ? to_f(tr[r * dim]) : through<T, Tin>(ti[(r - n_ring) * dim]);
    };
    float lo = __int_as_float(0x7f800000);  // +inf
    float hi = __int_as_float(0xff800000);  // -inf
    double sum = 0.0;
    for (uint32_t r = 0; r < B; ++r) {
      const float x = val(r);
      lo = (x < lo) ? x : lo;  // std::min(lo, x)
      hi = (hi < x) ? x : hi;  // std::max(hi, x)
      if (is_k) sum = __dadd_rn(sum, (double)x);
    }
    if (is_k)
      a.cent[((uint64_t)s * g.n_cap + blk) * g.d_k + c] =
          __double2float_rn(__ddiv_rn(sum, (double)B));
    if (bits == 16) {  // lossless passthrough of the ring element (quantizer.cpp:55-59)
      T* dst = reinterpret_cast<T*>(img0);
      for (uint32_t r = 0; r < B; ++r) dst[r * dim + c] = from_f<T>(val(r));
    } else {
      float scale, zp = lo;
      if (hi == lo) {
        scale = 1.0f;
        for (uint32_t r = 0; r < B; ++r) codes[r * dim + c] = 0;
      } else {
        const double levels = (double)((1u << bits) - 1u);
        scale = __double2float_rn(__ddiv_rn(__dsub_rn((double)hi, (double)lo), levels));
        const double dlo = (double)lo, dscale = (double)scale;
        const double rcp = __drcp_rn(dscale);  // see evict_quantize_kernel
        for (uint32_t r = 0; r < B; ++r) {
          const double av = __dsub_rn((double)val(r), dlo);
          const double t = __dmul_rn(av, rcp);
          const double fr = t - floor(t);
          double q = fabs(fr - 0.5) > 0x1p-36 ? round(t) : round(__ddiv_rn(av, dscale));
          q = q < 0.0 ? 0.0 : (levels < q ? levels : q);
          codes[r * dim + c] = (uint8_t)(uint32_t)q;
        }
      }
      float* par = reinterpret_cast<float*>(img1) + 2 * c;  // params lead region 1
      par[0] = scale;
      par[1] = zp;
    }
  }
  __syncthreads();

  // ---- LSB-first packing over the flat row-major index (quantizer.cpp:22-32)
  if (bits != 16) {
    const uint32_t nbytes = is_k ? L.k_bytes : L.v_bytes;
    for (uint32_t j = threadIdx.x; j < nbytes; j += blockDim.x) {
      uint32_t byte;
      if (bits == 8) {
        byte = codes[j];
      } else if (bits == 4) {
        byte = codes[2 * j] | (2 * j + 1 < B * dim ? (uint32_t)codes[2 * j + 1] << 4 : 0u);
      } else {
        byte = 0;
        const uint32_t b0 = 8 * j, total = B * dim;
        for (uint32_t i = b0 / bits; i < total && i * bits < b0 + 8; ++i) {
          const uint32_t v = codes[i];
          const int sh = (int)(i * bits) - (int)b0;
          byte |= sh >= 0 ? (v << sh) : (v >> (-sh));
        }
        byte &= 0xffu;
      }
      img0[j] = (uint8_t)byte;
    }
  }
  __syncthreads();

  // ---- record halves -> arena (pinned DRAM via PCIe posted writes, or HBM);
  // params -> HBM mirror
  uint8_t* out = a.arena + ((uint64_t)s * g.n_cap + blk) * L.stride;
  for (uint32_t o = threadIdx.x * 16; o < hi0 - lo0; o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(out + lo0 + o) = *reinterpret_cast<const uint4*>(img0 + o);
  for (uint32_t o = threadIdx.x * 16; o < hi1 - lo1; o += blockDim.x * 16)
    *reinterpret_cast<uint4*>(out + lo1 + o) = *reinterpret_cast<const uint4*>(img1 + o);
  const uint32_t pbytes = L.used - L.kp_off;
  if (a.params && pbytes) {
    const uint32_t pe = (hi1 < L.used ? hi1 : L.used);
    uint8_t* pm = a.params + ((uint64_t)s * g.n_cap + blk) * pbytes + (lo1 - L.kp_off);
    for (uint32_t o = threadIdx.x * 16; o < pe - lo1; o += blockDim.x * 16)
      *reinterpret_cast<uint4*>(pm + o) = *reinterpret_cast<const uint4*>(img1 + o);
  }
}

template <typename T, typename Tin>
static size_t evict_staged_smem(const Geometry& g) {
  const size_t dmax = g.d_k > g.d_v ? g.d_k : g.d_v;
  const size_t tile = (size_t)g.B * dmax * (sizeof(T) > sizeof(Tin) ? sizeof(T) : sizeof(Tin));
  const RecordLayout& L = g.rec;
  const size_t img = std::max<size_t>(L.v_off + (L.vp_off - L.kp_off),
                                      (L.kp_off - L.v_off) + (L.stride - L.vp_off));
  return ((tile + 15) & ~size_t(15)) + 16 + (((size_t)g.B * dmax + 15) & ~size_t(15)) + img;
}

template <typename T, typename Tin>
static bool evict_staged_ok(const Geometry& g) {
  // 16-byte rows for cp.async, one thread per channel, smem within 2 CTAs/SM
  const bool rows16 = (g.d_k * sizeof(T)) % 16 == 0 && (g.d_v * sizeof(T)) % 16 == 0 &&
                      (g.d_k * sizeof(Tin)) % 16 == 0 && (g.d_v * sizeof(Tin)) % 16 == 0;
  return rows16 && g.d_k <= 128 && g.d_v <= 128 && evict_staged_smem<T, Tin>(g) <= 110 * 1024;
}

size_t evict_smem_bytes(const Geometry& g) {
  return (size_t)g.rec.stride + (size_t)g.B * (g.d_k + g.d_v);
}

template <typename T, typename Tin>
static cudaError_t launch_evict_t(const EvictArgs& a, uint32_t n_blocks, cudaStream_t st) {
  static const bool staged_off = [] {
    const char* e = std::getenv("TTKV_EVICT_STAGED");
    return e && e[0] == '0';
  }();
  if (!staged_off && evict_staged_ok<T, Tin>(a.g) && a.in_tokens < (1ull << 31)) {
    const size_t smem = evict_staged_smem<T, Tin>(a.g);
    auto kern = evict_staged_kernel<T, Tin>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3(n_blocks, a.g.S, 2), 128, smem, st>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = evict_smem_bytes(a.g);
  auto kern = evict_quantize_kernel<T, Tin>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t threads = ((a.g.d_k + a.g.d_v + 31) / 32) * 32;
  dim3 grid(n_blocks, a.g.S);
  kern<<<grid, threads < 64 ? 64 : threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_evict(const EvictArgs& a, uint32_t n_blocks, int in_dtype, cudaStream_t st) {
  if (n_blocks == 0) return cudaSuccess;
  if (a.g.elem == 2) {
    if (in_dtype == kInF16) return launch_evict_t<__half, __half>(a, n_blocks, st);
    return launch_evict_t<__half, float>(a, n_blocks, st);
  }
  if (in_dtype == kInF16) return launch_evict_t<float, __half>(a, n_blocks, st);
  return launch_evict_t<float, float>(a, n_blocks, st);
}

}  // namespace ttkv_dev
