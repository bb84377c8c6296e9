// mma.sync throughput probe on sm_100a: f16 m16n8k16 (f32 acc) vs u8.s8
// m16n8k32 (s32 acc), 8 independent accumulator chains per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void probe(uint32_t* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 13;
  float f[8][4] = {};
  int32_t n[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (KIND == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(f[c][0]), "+f"(f[c][1]), "+f"(f[c][2]), "+f"(f[c][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+r"(n[c][0]), "+r"(n[c][1]), "+r"(n[c][2]), "+r"(n[c][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
  }
  uint32_t acc = 0;
  for (int c = 0; c < 8; ++c)
    for (int e = 0; e < 4; ++e) acc += (uint32_t)n[c][e] + __float_as_uint(f[c][e]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 16 * 1024 * 4);
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind) {
    for (int warps : {4, 8, 16}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) probe<0><<<148, warps * 32>>>(out, iters);
        else probe<1><<<148, warps * 32>>>(out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double mmas = 148.0 * warps * iters * 8;
      const double flop = mmas * (kind == 0 ? 16 * 8 * 16 : 16 * 8 * 32) * 2;
      printf("%s warps/SM=%2d: %.3f ms, %.2f warp-mma/clk/SM @1.9GHz, %.1f T(FL)OP/s\n",
             kind == 0 ? "HMMA m16n8k16 f16->f32" : "IMMA m16n8k32 u8s8->s32", warps, ms,
             mmas / 148 / (ms * 1e-3 * 1.9e9), flop / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
