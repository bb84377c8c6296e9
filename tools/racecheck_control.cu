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
int main() {
  int* d; cudaMalloc(&d, 32 * sizeof(int));
  handoff<<<1, 64>>>(d);
  int h[32]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int ok = 1; for (int i = 0; i < 32; ++i) ok &= h[i] == 3 * i;
  printf("handoff %s\n", ok ? "ok" : "WRONG");
  return ok ? 0 : 1;
}
