// Does mma.sync f16 -> f32 keep fp16 subnormal inputs exactly, and does
// feeding u8 codes as subnormals (n * 2^-24) instead of normal integers (n)
// change the accumulated result?  Random codes against random fp16 B values
// (magnitudes spread over 2^-16 .. 2^0); prints the max |error| relative to
// the exact sum for both encodings.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <random>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

// one m16n8k16: A row-major [16][16] halves, B col-major [8][16], D [16][8]
__global__ void mma1(const uint16_t* A, const uint16_t* B, float* D) {
  const int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
  auto a2 = [&](int r, int c) { return (uint32_t)A[r * 16 + c] | ((uint32_t)A[r * 16 + c + 1] << 16); };
  auto b2 = [&](int n, int k) { return (uint32_t)B[n * 16 + k] | ((uint32_t)B[n * 16 + k + 1] << 16); };
  const uint32_t a0 = a2(g, 2 * q), a1 = a2(g + 8, 2 * q), a2_ = a2(g, 2 * q + 8), a3 = a2(g + 8, 2 * q + 8);
  const uint32_t b0 = b2(g, 2 * q), b1 = b2(g, 2 * q + 8);
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2_), "r"(a3), "r"(b0), "r"(b1));
  D[g * 8 + 2 * q] = d[0];
  D[g * 8 + 2 * q + 1] = d[1];
  D[(g + 8) * 8 + 2 * q] = d[2];
  D[(g + 8) * 8 + 2 * q + 1] = d[3];
}

int main() {
  uint16_t *A, *B;
  float* D;
  cudaMallocManaged(&A, 512);
  cudaMallocManaged(&B, 256);
  cudaMallocManaged(&D, 512);
  std::mt19937 rng(1);
  double worst[2] = {0, 0};
  int nonzero_diff = 0;
  for (int trial = 0; trial < 2000; ++trial) {
    uint8_t code[256];
    double bv[128];
    for (int i = 0; i < 256; ++i) code[i] = rng() & 255;
    for (int i = 0; i < 128; ++i) {
      const float f = std::ldexp((float)(rng() % 2048) / 2048.f + 0.5f, -(int)(rng() % 17)) *
                      ((rng() & 1) ? 1.f : -1.f);
      const __half h = __float2half_rn(f);
      memcpy(&B[i], &h, 2);
      bv[i] = (double)__half2float(h);
    }
    float res[2][128];
    for (int enc = 0; enc < 2; ++enc) {
      for (int i = 0; i < 256; ++i) {
        if (enc == 0) {
          const __half h = __float2half_rn((float)code[i]);
          memcpy(&A[i], &h, 2);
        } else {
          A[i] = code[i];  // subnormal n * 2^-24
        }
      }
      mma1<<<1, 32>>>(A, B, D);
      cudaDeviceSynchronize();
      for (int r = 0; r < 16; ++r)
        for (int n = 0; n < 8; ++n) {
          double exact = 0, mag = 0;
          for (int k = 0; k < 16; ++k) {
            exact += code[r * 16 + k] * bv[n * 16 + k];
            mag += std::fabs(code[r * 16 + k] * bv[n * 16 + k]);
          }
          const double got = enc == 0 ? D[r * 8 + n] : std::ldexp((double)D[r * 8 + n], 24);
          res[enc][r * 8 + n] = (float)got;
          worst[enc] = std::fmax(worst[enc], std::fabs(got - exact) / mag);
        }
    }
    for (int i = 0; i < 128; ++i) nonzero_diff += res[0][i] != res[1][i];
  }
  printf("max |err| / sum|terms|: normal-integer codes %.3e, subnormal codes %.3e; "
         "%d of %d results differ between encodings\n",
         worst[0], worst[1], nonzero_diff, 2000 * 128);
  return 0;
}
