// ttkv_freefn.cu -- the reference's stateless numeric free functions on the GPU
// (the cold-path API surface of the drop-in; the hot path fuses these):
//   dequantize_block  quantizer.cpp:90-113, 157-170  (bit-exact fp64 affine)
//   score_block       relevance.cpp:19-27            (bit-exact fp64, one exact fma per term)
//   select_top_k      relevance.cpp:29-43            (bitonic sort, total order: one CTA
//                                                     in shared memory up to 8192 scores,
//                                                     a global-memory network above)
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/ttkv_gpu.h"
#include "ttkv_kernels.cuh"
#include "ttkv_launch.h"

namespace ttkv_dev {

__global__ void dequant_kernel(const uint8_t* packed, const float* params, uint64_t rows,
                               uint32_t dim, uint32_t bits, float* out) {
  const uint64_t n = rows * dim;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (bits == 16) {
      out[i] = reinterpret_cast<const float*>(packed)[i];
      continue;
    }
    const uint64_t bit = i * bits;
    const uint32_t lo = packed[bit >> 3];
    const uint32_t hi = (((bit & 7) + bits) > 8) ? packed[(bit >> 3) + 1] : 0u;
    const uint32_t code = ((lo | (hi << 8)) >> (bit & 7)) & ((1u << bits) - 1u);
    const uint32_t c = (uint32_t)(i % dim);
    const double x = __dadd_rn(__dmul_rn((double)code, (double)params[2 * c]),
                               (double)params[2 * c + 1]);
    out[i] = __double2float_rn(x);
  }
}

__global__ void score_free_kernel(const float* q, const float* cent, uint64_t n, uint32_t d,
                                  double* out) {
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n;
       b += (uint64_t)gridDim.x * blockDim.x) {
    // exact products of float-valued doubles: one fma == mul + add (see score_kernel)
    double acc = 0.0;
    for (uint32_t i = 0; i < d; ++i) acc = __fma_rn((double)q[i], (double)cent[b * d + i], acc);
    out[b] = acc;
  }
}

__device__ __forceinline__ uint64_t order_key_free(double d) {
  if (d == 0.0) d = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void topk_free_kernel(const double* scores, const uint64_t* ids, uint32_t n,
                                 uint32_t N2, uint32_t k, uint64_t* out) {
  extern __shared__ __align__(16) uint64_t sm[];
  uint64_t* key = sm;
  uint64_t* id = sm + N2;
  for (uint32_t i = threadIdx.x; i < N2; i += blockDim.x) {
    key[i] = i < n ? order_key_free(scores[i]) : 0ull;
    id[i] = i < n ? ids[i] : 0ull;
  }
  __syncthreads();
  for (uint32_t size = 2; size <= N2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < N2 / 2; i += blockDim.x) {
        const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t kl = key[lo], kh = key[hi], il = id[lo], ih = id[hi];
        const bool less = (kl < kh) || (kl == kh && il < ih);
        if (less == desc) {
          key[lo] = kh; key[hi] = kl;
          id[lo] = ih; id[hi] = il;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) out[i] = id[i];
}

// Global-memory bitonic network for select_top_k above the shared-memory
// kernel's 8192 scores: one launch per (size, stride) stage, one thread per
// compare-exchange pair, the same order as topk_free_kernel.
__global__ void topk_keys_kernel(const double* scores, uint64_t* key, uint32_t n, uint32_t N2) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N2; i += gridDim.x * blockDim.x)
    key[i] = i < n ? order_key_free(scores[i]) : 0ull;
}

__global__ void bitonic_stage_kernel(uint64_t* key, uint64_t* id, uint32_t N2, uint32_t size,
                                     uint32_t stride) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N2 / 2;
       i += gridDim.x * blockDim.x) {
    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
    const bool desc = (lo & size) == 0;
    const uint64_t kl = key[lo], kh = key[hi], il = id[lo], ih = id[hi];
    const bool less = (kl < kh) || (kl == kh && il < ih);
    if (less == desc) {
      key[lo] = kh; key[hi] = kl;
      id[lo] = ih; id[hi] = il;
    }
  }
}

// Thread-local, grow-only device scratch for the stateless entry points:
// token-at-a-time callers (10^4 quantize_block / dequantize_block calls in the
// reference's acceptance gate) were dominated by a cudaMalloc + cudaFree pair
// per buffer per call, each free an implicit device synchronization.  Slots
// are reused across calls (every entry point is synchronous) and live for the
// thread.
void* scratch(int slot, size_t bytes, cudaError_t* err) {
  struct Pool {
    void* p[8] = {};
    size_t cap[8] = {};
  };
  constexpr int kMaxDev = 64;
  thread_local Pool pools[kMaxDev];  // one pool per device: a thread that
                                     // alternates devices keeps (and reuses) both
  int dev = 0;
  *err = cudaGetDevice(&dev);
  if (*err != cudaSuccess) return nullptr;
  if (dev < 0 || dev >= kMaxDev) {
    *err = cudaErrorInvalidDevice;
    return nullptr;
  }
  Pool& pool = pools[dev];
  bytes = bytes ? bytes : 16;
  if (pool.cap[slot] < bytes) {
    const size_t want = std::max(bytes, 2 * pool.cap[slot]);
    if (pool.p[slot]) cudaFree(pool.p[slot]);
    pool.p[slot] = nullptr;
    pool.cap[slot] = 0;
    *err = cudaMalloc(&pool.p[slot], want);
    if (*err != cudaSuccess) return nullptr;
    pool.cap[slot] = want;
  }
  return pool.p[slot];
}

}  // namespace ttkv_dev

namespace {


// A slot of the thread-local scratch pool (ttkv_dev::scratch).
struct DevBuf {
  int slot;
  void* p = nullptr;
  explicit DevBuf(int s) : slot(s) {}
  cudaError_t alloc(size_t n) {
    cudaError_t e = cudaSuccess;
    p = ttkv_dev::scratch(slot, n, &e);
    return e;
  }
};

int fail(cudaError_t e) {
  ttkv_dev::set_last_error(cudaGetErrorString(e));
  return TTKV_ECUDA;
}
}  // namespace

#define FCU(x)                          \
  do {                                  \
    cudaError_t e__ = (x);              \
    if (e__ != cudaSuccess) return fail(e__); \
  } while (0)

extern "C" {


int ttkv_gpu_dequantize_block(int device, const uint8_t* packed_k, const uint8_t* packed_v,
                              const float* key_params, const float* value_params, uint64_t rows,
                              uint32_t d_k, uint32_t d_v, uint32_t kb, uint32_t vb, float* keys,
                              float* values) {
  auto valid_bits = [](uint32_t b) { return (b >= 2 && b <= 8) || b == 16; };
  if (!valid_bits(kb) || !valid_bits(vb)) return TTKV_EINTEGRITY;
  FCU(cudaSetDevice(device));
  auto bytes = [](uint64_t cnt, uint32_t bits) -> size_t {
    return bits == 16 ? cnt * 4 : (cnt * bits + 7) / 8;
  };
  for (int t = 0; t < 2; ++t) {
    const uint8_t* pk = t ? packed_v : packed_k;
    const float* pp = t ? value_params : key_params;
    const uint32_t dim = t ? d_v : d_k, bits = t ? vb : kb;
    float* out = t ? values : keys;
    if (!out || rows * dim == 0) continue;
    DevBuf dp(0), dpar(1), dout(2);
    const size_t nb = bytes(rows * dim, bits);
    FCU(dp.alloc(nb + 8));
    FCU(cudaMemset(dp.p, 0, nb + 8));
    FCU(cudaMemcpy(dp.p, pk, nb, cudaMemcpyHostToDevice));
    FCU(dpar.alloc(8 * dim));
    if (bits != 16) FCU(cudaMemcpy(dpar.p, pp, 8 * dim, cudaMemcpyHostToDevice));
    FCU(dout.alloc(rows * dim * 4));
    const unsigned grid = (unsigned)std::min<uint64_t>((rows * dim + 255) / 256, 148 * 8);
    ttkv_dev::dequant_kernel<<<grid, 256>>>((const uint8_t*)dp.p, (const float*)dpar.p, rows,
                                             dim, bits, (float*)dout.p);
    FCU(cudaGetLastError());
    FCU(cudaMemcpy(out, dout.p, rows * dim * 4, cudaMemcpyDeviceToHost));
  }
  return TTKV_OK;
}

int ttkv_gpu_score_blocks(int device, const float* query, const float* centroids, uint64_t n,
                          uint32_t d, double* scores) {
  if (n == 0) return TTKV_OK;
  if (!query || !centroids || !scores) return TTKV_EINVAL;
  FCU(cudaSetDevice(device));
  DevBuf dq(0), dc(1), ds(2);
  FCU(dq.alloc(d * 4));
  FCU(dc.alloc(n * d * 4));
  FCU(ds.alloc(n * 8));
  FCU(cudaMemcpy(dq.p, query, d * 4, cudaMemcpyHostToDevice));
  FCU(cudaMemcpy(dc.p, centroids, n * d * 4, cudaMemcpyHostToDevice));
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 127) / 128, 148 * 8);
  ttkv_dev::score_free_kernel<<<grid, 128>>>((const float*)dq.p, (const float*)dc.p, n, d,
                                              (double*)ds.p);
  FCU(cudaGetLastError());
  FCU(cudaMemcpy(scores, ds.p, n * 8, cudaMemcpyDeviceToHost));
  return TTKV_OK;
}

int ttkv_gpu_select_top_k(int device, const double* scores, const uint64_t* ids, uint64_t n,
                          uint64_t k, uint64_t* out) {
  if (k > n) k = n;
  if (n == 0 || k == 0) return TTKV_OK;
  if (n > (1ull << 31)) {
    ttkv_dev::set_last_error("select_top_k: more than 2^31 blocks");
    return TTKV_ECONFIG;
  }
  FCU(cudaSetDevice(device));
  uint64_t N2 = 2;
  while (N2 < n) N2 <<= 1;
  DevBuf ds(0), di(1), dout(2);
  FCU(ds.alloc(n * 8));
  FCU(di.alloc(N2 * 8));
  FCU(dout.alloc(k * 8));
  FCU(cudaMemcpy(ds.p, scores, n * 8, cudaMemcpyHostToDevice));
  FCU(cudaMemcpy(di.p, ids, n * 8, cudaMemcpyHostToDevice));
  if (N2 > 8192) {
    DevBuf dk(3);
    FCU(dk.alloc(N2 * 8));
    FCU(cudaMemset((uint64_t*)di.p + n, 0, (N2 - n) * 8));
    const unsigned grid = (unsigned)std::min<uint64_t>((N2 / 2 + 255) / 256, 148 * 16);
    ttkv_dev::topk_keys_kernel<<<grid, 256>>>((const double*)ds.p, (uint64_t*)dk.p, (uint32_t)n,
                                               (uint32_t)N2);
    for (uint64_t size = 2; size <= N2; size <<= 1)
      for (uint64_t stride = size >> 1; stride > 0; stride >>= 1)
        ttkv_dev::bitonic_stage_kernel<<<grid, 256>>>((uint64_t*)dk.p, (uint64_t*)di.p,
                                                       (uint32_t)N2, (uint32_t)size,
                                                       (uint32_t)stride);
    FCU(cudaGetLastError());
    FCU(cudaMemcpy(out, di.p, k * 8, cudaMemcpyDeviceToHost));
    return TTKV_OK;
  }
  const size_t smem = (size_t)N2 * 16;
  FCU(cudaFuncSetAttribute(ttkv_dev::topk_free_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem));
  ttkv_dev::topk_free_kernel<<<1, 1024, smem>>>((const double*)ds.p, (const uint64_t*)di.p,
                                                 (uint32_t)n, N2, (uint32_t)k, (uint64_t*)dout.p);
  FCU(cudaGetLastError());
  FCU(cudaMemcpy(out, dout.p, k * 8, cudaMemcpyDeviceToHost));
  return TTKV_OK;
}

}  // extern "C"
