// ttkv_kernels.cuh -- sm_100a kernels of the TTKV decode hot path.
//
// Data layout in device-visible memory (one handle, S lockstep streams):
//   ring_k  [S][C][d_k] T      fast tier, slot = position mod C, C = L_fast + B
//   ring_v  [S][C][d_v] T      (T = half for bytes_full_precision 2, float for 4)
//   cent    [S][n_cap][d_k] f32  key centroids, resident in HBM
//   arena   [S][n_cap][stride] u8 slow-tier records (pinned host DRAM, mapped):
//           [K payload][V payload][K {scale,zp} f32 x d_k][V {scale,zp} x d_v]
//           payloads are the reference's LSB-first packed codes
//           (quantizer.cpp:22-32), so a record is serialize_block's payload
//           verbatim.  K8/V4, d=128, B=128: 16384+8192+1024+1024 = 26,624 B.
//   params  [S][n_cap][used - kp_off] u8  HBM mirror of each record's params
//   scores  [S][Gs][n_cap] f64 (bit-exact; the fetched_blocks order is
//           materialized from them on demand),
//   union_ids / union_mask [S][n_cap] u32, union_count [S]
//   partials [S][G][chunks][d_v + 2] f32  (acc[d_v], m (log2 units), l)
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace ttkv_dev {

constexpr int kMaxG = 8;
constexpr int kMaxD = 128;
constexpr int kSlowConsumerWarps = 4;
constexpr int kFastWarps = 4;

struct RecordLayout {
  uint32_t k_bytes, v_bytes;  // payload bytes as stored
  uint32_t v_off, kp_off, vp_off;
  uint32_t used;    // bytes of the record (16-aligned)
  uint32_t stride;  // record pitch (128-aligned)
  // The streamed part is the payload [0, kp_off); the params [kp_off, used)
  // are mirrored in HBM (resident like the centroids) and staged from there.
};

struct Geometry {
  uint32_t S, G, Gs, d_k, d_v, B, kb, vb, elem;
  uint64_t C;      // ring capacity (tokens)
  uint64_t n_cap;  // slow-block capacity per stream
  RecordLayout rec;
};

// ---------------------------------------------------------------------------
// element helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }

// Round an input value through the ring type (a token enters the fast tier
// before it can be evicted, so the slow tier sees the ring-rounded value).
template <typename T, typename Tin>
__device__ __forceinline__ float through(Tin x) { return to_f(from_f<T>(to_f(x))); }
template <> __device__ __forceinline__ float through<__half, __half>(__half x) { return __half2float(x); }

// 4 consecutive elements starting at a 4-element-aligned index.
__device__ __forceinline__ void load4(const __half* p, float (&o)[4]) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const __half2 a = *reinterpret_cast<const __half2*>(&u.x);
  const __half2 b = *reinterpret_cast<const __half2*>(&u.y);
  const float2 fa = __half22float2(a), fb = __half22float2(b);
  o[0] = fa.x; o[1] = fa.y; o[2] = fb.x; o[3] = fb.y;
}
__device__ __forceinline__ void load4(const float* p, float (&o)[4]) {
  const float4 u = *reinterpret_cast<const float4*>(p);
  o[0] = u.x; o[1] = u.y; o[2] = u.z; o[3] = u.w;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// warp-wide fp32 max in one instruction (CREDUX.MAX.F32, sm_100a; NaN-ignoring
// like fmaxf)
// Programmatic dependent launch: a kernel started by launch_chained() may run
// while its predecessor on the stream drains, so it calls pdl_wait() before
// touching anything the predecessor writes (griddepcontrol.wait returns once
// that grid has completed and its memory is visible; a no-op for a normal
// launch).  pdl_trigger() lets the successor's CTAs be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float warp_max_redux(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy PTX (sm_90+; used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// Non-blocking probe + a backing-off wait for the producer warp, so its spin
// does not steal issue slots from the consumer warps on the same SMSP.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) __nanosleep(128);
}
// global (incl. host-mapped sysmem) -> shared bulk copy, completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---------------------------------------------------------------------------
// code extraction from an LSB-first packed stream (quantizer.cpp:34-47)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t extract_code(const uint8_t* p, uint32_t idx, uint32_t bits) {
  const uint32_t bit = idx * bits;
  const uint32_t lo = p[bit >> 3];
  const uint32_t hi = p[(bit >> 3) + 1];
  return ((lo | (hi << 8)) >> (bit & 7)) & ((1u << bits) - 1u);
}

}  // namespace ttkv_dev
