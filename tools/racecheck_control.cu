// Control case for compute-sanitizer racecheck: a textbook mbarrier
// producer/consumer hand-off (producer warp: st.shared, __syncwarp,
// mbarrier.arrive [release]; consumer warp: mbarrier.try_wait [acquire], ld.shared).
// This ordering is correct under the PTX memory model; if racecheck reports a
// hazard here it does not model mbarrier synchronisation, which is the same
// pattern the engine's producer/consumer pipelines use.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__global__ void handoff(int* out) {
  __shared__ int buf[32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  __syncthreads();
  if (threadIdx.x < 32) {
    buf[threadIdx.x] = threadIdx.x * 3;
    __syncwarp();
    if (threadIdx.x == 0)
      asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(&bar))
                   : "memory");
  } else {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
    out[threadIdx.x - 32] = buf[threadIdx.x - 32];
  }
}
// Control case 2: the bulk-copy pipeline of the attention kernels, reduced
// to one stage reused R times.  Producer (one thread): mbarrier.arrive.expect_tx
// + cp.async.bulk global -> shared completing on `full`; consumers: try_wait
// on `full`, ld.shared, then arrive on `empty`; the producer waits on `empty`
// before refilling the stage (the WAR side).  Correct under the PTX memory
// model (complete_tx makes the async-proxy writes visible to the waiters).
__global__ void bulk_handoff(const int* src, int* out, int R) {
  __shared__ __align__(128) int stage[256];
  __shared__ __align__(8) uint64_t full, empty;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    if (threadIdx.x == 0) {
      if (r > 0) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(su32(&empty)), "r"((r - 1) & 1) : "memory");
      }
      asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], 1024; }" ::"r"(su32(&full))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(
                       su32(stage)), "l"(src + 256 * r), "r"(su32(&full))
                   : "memory");
    } else if (threadIdx.x >= 32) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&full)), "r"(r & 1) : "memory");
      const int t = threadIdx.x - 32;
      int acc = 0;
      for (int j = t; j < 256; j += 32) acc += stage[j];
      out[r * 32 + t] = acc;
      __syncwarp();
      if (t == 0)
        asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(&empty)) : "memory");
    }
  }
}

int main() {
  int* d; cudaMalloc(&d, 32 * sizeof(int));
  handoff<<<1, 64>>>(d);
  int h[32]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int ok = 1; for (int i = 0; i < 32; ++i) ok &= h[i] == 3 * i;
  printf("handoff %s\n", ok ? "ok" : "WRONG");
  const int R = 8;
  int* hs = new int[256 * R];
  for (int i = 0; i < 256 * R; ++i) hs[i] = i % 977;
  int *ds, *dout;
  cudaMalloc(&ds, 256 * R * sizeof(int));
  cudaMalloc(&dout, 32 * R * sizeof(int));
  cudaMemcpy(ds, hs, 256 * R * sizeof(int), cudaMemcpyHostToDevice);
  bulk_handoff<<<1, 64>>>(ds, dout, R);
  int ho[32 * R];
  cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
  int ok2 = 1;
  for (int r = 0; r < R; ++r)
    for (int t = 0; t < 32; ++t) {
      int e = 0;
      for (int j = t; j < 256; j += 32) e += hs[256 * r + j];
      ok2 &= ho[r * 32 + t] == e;
    }
  printf("bulk handoff %s\n", ok2 ? "ok" : "WRONG");
  return ok && ok2 ? 0 : 1;
}
