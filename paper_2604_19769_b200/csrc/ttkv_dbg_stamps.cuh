// Measurement-only build (make stamps: -DTTKV_STAMPS, a separate library
// under build/stamps/): %globaltimer stamps of the layer-sequential chain,
// read back by tools/chain_stamps.py.  Nothing here is compiled into the
// product library.
//   * kernel phases: CTA (0, 0) thread 0 writes stamp k of the kernel's
//     launch number (counted by that thread at stamp 0);
//   * kernel ends: the last CTA to finish writes the end stamp.
// Without relocatable device code each .cu file has its own copy of these
// variables, so each file exports its own reader.
#pragma once
#ifdef TTKV_STAMPS
#include <cstdint>

namespace ttkv_dbg {
constexpr unsigned kSlots = 4096;
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
}  // namespace ttkv_dbg

// one table per kernel family: stamps[slot][16], launch counter, end counter
#define TTKV_DBG_TABLE(name)                                              \
  __device__ unsigned long long name##_st[ttkv_dbg::kSlots][16];          \
  __device__ unsigned name##_launch;                                      \
  __device__ unsigned name##_cur;                                         \
  __device__ unsigned name##_done;                                        \
  __device__ unsigned name##_ends;

// stamp k (k = 0 starts a new launch) from CTA (0, 0), thread 0
#define TTKV_DBG_STAMP(name, k)                                                       \
  do {                                                                                \
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {                      \
      if ((k) == 0) name##_cur = atomicAdd(&name##_launch, 1u);                       \
      name##_st[name##_cur % ttkv_dbg::kSlots][(k)] = ttkv_dbg::now_ns();             \
    }                                                                                 \
  } while (0)

// end of the launch: the last CTA to arrive writes stamp 15 (every thread of
// every CTA must call it)
#define TTKV_DBG_END(name)                                                            \
  do {                                                                                \
    __syncthreads();                                                                  \
    if (threadIdx.x == 0) {                                                           \
      __threadfence();                                                                \
      const unsigned n_ = atomicAdd(&name##_done, 1u);                                \
      if (n_ == gridDim.x * gridDim.y * gridDim.z - 1) {                              \
        name##_done = 0;                                                              \
        const unsigned e_ = atomicAdd(&name##_ends, 1u);                              \
        name##_st[e_ % ttkv_dbg::kSlots][15] = ttkv_dbg::now_ns();                    \
      }                                                                               \
    }                                                                                 \
  } while (0)

// per-CTA stamps of the latest launch (blockIdx.x < 1024), thread `tid`
#define TTKV_DBG_CTA_TABLE(name) __device__ unsigned long long name##_cta[1024][8];
#define TTKV_DBG_CTA(name, k, tid)                                                    \
  do {                                                                                \
    if (threadIdx.x == (tid) && blockIdx.x < 1024 && blockIdx.y == 0)                 \
      name##_cta[blockIdx.x][(k)] = ttkv_dbg::now_ns();                               \
  } while (0)
#define TTKV_DBG_CTA_READER(name)                                                     \
  extern "C" int ttkv_dbg_read_##name##_cta(unsigned long long* out) {                \
    return cudaMemcpyFromSymbol(out, name##_cta, sizeof(name##_cta)) != cudaSuccess;  \
  }

#define TTKV_DBG_READER(name)                                                         \
  extern "C" int ttkv_dbg_read_##name(unsigned long long* out, unsigned n_slots,      \
                                      unsigned* launches) {                           \
    if (n_slots > ttkv_dbg::kSlots) n_slots = ttkv_dbg::kSlots;                       \
    if (cudaMemcpyFromSymbol(out, name##_st, (size_t)n_slots * 16 * 8) != cudaSuccess) \
      return 1;                                                                       \
    return cudaMemcpyFromSymbol(launches, name##_launch, 4) != cudaSuccess;           \
  }
#else
#define TTKV_DBG_STAMP(name, k)
#define TTKV_DBG_END(name)
#define TTKV_DBG_CTA(name, k, tid)
#endif
