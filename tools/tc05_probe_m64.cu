// tcgen05 kind::i8 probe (not product code): M = 64 with the A operand an
// MN-major [K = 128 tokens][M = 64 bytes] u8 tile in the 64B-swizzle layout
// the V nibbles arrive in (TMA SWIZZLE_64B).  Dumps all 128 TMEM lanes of the
// accumulator to find where the 64 rows land, and checks the values.
//   make -C tools (build/tc05_probe_m64)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t sw64(uint32_t row, uint32_t byte) {  // TMA SWIZZLE_64B, 64 B rows
  const uint32_t off = row * 64 + byte;
  return off ^ (((off >> 7) & 3u) << 4);
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* out, uint32_t layout, uint32_t sbo) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint8_t* sA = base;          // 8 KB
  uint8_t* sB = base + 8192;   // 2 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (uint32_t i = t; i < 128 * 64; i += 128) sA[sw64(i / 64, i % 64)] = A[i];
  for (uint32_t i = t; i < 128 * 16; i += 128) sB[i] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  // zero the accumulator region first (all 128 lanes x 16 cols) so unused lanes read 0
  {
    uint32_t z[16] = {0};
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            tm + ((32 * warp) << 16)),
        "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]),
        "r"(z[8]), "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    // D[m][n] = sum_k A[k][m] * B[k][n]; M = 64, N = 16, A MN-major, B MN-major (u8 x u8)
    const uint32_t id = (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) | ((16u >> 3) << 17) |
                        ((64u >> 4) << 24);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t da = desc(su32(sA) + 2048 * kk, 8192, sbo, layout);
      const uint64_t db = desc(su32(sB) + 512 * kk, 128, 256, 0);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
          "l"(da), "l"(db), "r"(id), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tm + ((32 * warp) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < 16; ++n) out[t * 16 + n] = (int32_t)r[n];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

int main() {
  std::vector<uint8_t> A(128 * 64), B(128 * 16);
  srand(3);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : B) x = rand() & 255;
  uint8_t *dA, *dB;
  int32_t* dO;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  // want[m][n]
  std::vector<int32_t> want(64 * 16);
  for (int m = 0; m < 64; ++m)
    for (int n = 0; n < 16; ++n) {
      int32_t e = 0;
      for (int k = 0; k < 128; ++k) e += (int32_t)A[k * 64 + m] * (int32_t)B[k * 16 + n];
      want[m * 16 + n] = e;
    }
  for (uint32_t layout : {4u, 6u, 2u}) {
    for (uint32_t sbo : {512u, 1024u, 256u}) {
      cudaMemset(dO, 0, 128 * 16 * 4);
      probe<<<1, 128, 16384>>>(dA, dB, dO, layout, sbo);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        std::printf("layout %u sbo %u: %s\n", layout, sbo, cudaGetErrorString(e));
        return 1;
      }
      std::vector<int32_t> got(128 * 16);
      cudaMemcpy(got.data(), dO, got.size() * 4, cudaMemcpyDeviceToHost);
      // for each want row m, find lanes whose 16 columns match
      int found = 0;
      std::printf("layout %u sbo %u: rows->lanes:", layout, sbo);
      for (int m = 0; m < 64; ++m) {
        int lane = -1;
        for (int l = 0; l < 128; ++l) {
          bool ok = true;
          for (int n = 0; n < 16; ++n) ok &= got[l * 16 + n] == want[m * 16 + n];
          if (ok) { lane = l; break; }
        }
        if (lane >= 0) ++found;
        if (m < 8 || (m >= 16 && m < 18) || m >= 62) std::printf(" %d:%d", m, lane);
      }
      std::printf("  (found %d of 64)\n", found);
    }
  }
  return 0;
}
