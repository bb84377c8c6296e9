// tcgen05 kind::i8 probe (not product code): can the record's u8 K codes,
// TMA-loaded with SWIZZLE_128B exactly as the HBM slow kernel loads them,
// feed tcgen05.mma directly (A K-major, no conversion) against s8 digit
// planes (B K-major, written by threads in the SW128 pattern), and can
// expanded V codes (A MN-major SW128) do the same for PV?  Results (s32 in
// TMEM, read back with tcgen05.ld) are checked against the CPU.
//   make -C tools (build/tc05_probe)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// SW128: 16-byte chunk index XOR (row % 8) within 1024-byte atoms of 8 x 128 B rows
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte) {
  return row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}
__device__ __forceinline__ uint64_t smem_desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100); layout SWIZZLE_NONE = 0
  return d;
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// kind::i8 instruction descriptor: D s32, A u8 (0) / B s8 (1), majors, N, M
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N, uint32_t a_fmt,
                                                uint32_t b_fmt, uint32_t a_mn, uint32_t b_mn) {
  return (2u << 4) | (a_fmt << 7) | (b_fmt << 10) | (a_mn << 15) | (b_mn << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}

struct Args {
  CUtensorMap tk;
  const int8_t* bq;   // [16][128] s8 QK B rows (n, k)
  const uint8_t* vt;  // [128 tok][128 ch] u8 expanded V
  const int8_t* bp;   // [16][128] s8 PV B rows (n, token)
  int32_t* out_qk;    // [128 tok][16]
  int32_t* out_pv;    // [128 ch][16]
  const uint8_t* bm;  // [128 tok][16] u8 PV B, MN-major (n contiguous per token)
  int32_t* out_pm;    // [128 ch][16]
};

__global__ void __launch_bounds__(128) probe(const __grid_constant__ Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  uint8_t* sK = base;              // 16 KB K codes (TMA, SW128)
  uint8_t* sBq = base + 16384;     // 2 KB
  uint8_t* sV = base + 18432;      // 16 KB V expanded, MN-major SW128 [tok][ch]
  uint8_t* sBp = base + 34816;     // 2 KB
  uint8_t* sBm = base + 36864;     // 2 KB, [tok][16] MN-major, no swizzle
  __shared__ __align__(8) uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B tiles and expanded V written by threads in the SW128 layouts
  for (uint32_t i = t; i < 16 * 128; i += 128) {
    const uint32_t n = i / 128, k = i % 128;
    sBq[sw128(n, k)] = (uint8_t)a.bq[i];
    sBp[sw128(n, k)] = (uint8_t)a.bp[i];
  }
  for (uint32_t i = t; i < 128 * 128; i += 128) {
    const uint32_t tok = i / 128, ch = i % 128;
    sV[sw128(tok, ch)] = a.vt[i];
  }
  for (uint32_t i = t; i < 128 * 16; i += 128) sBm[i] = a.bm[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(su32(&bar_tma))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(sK)),
        "l"(reinterpret_cast<uint64_t>(&a.tk)), "r"(0), "r"(0), "r"(0), "r"(su32(&bar_tma))
        : "memory");
    mbar_wait(&bar_tma, 0);
    // QK: D[tok][n] (cols 0..15) = sum_k K[tok][k] * Bq[n][k]; 4 MMAs of K = 32
    const uint32_t iq = idesc_i8(128, 16, 0, 1, 0, 0);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t da = smem_desc(su32(sK) + 32 * kk, 16, 1024);
      const uint64_t db = smem_desc(su32(sBq) + 32 * kk, 16, 1024);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
          "l"(da), "l"(db), "r"(iq), "r"(kk));
    }
    // PV: D[ch][n] (cols 16..31) = sum_tok V[tok][ch] * Bp[n][tok]; A MN-major
    const uint32_t ip = idesc_i8(128, 16, 0, 1, 1, 0);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t da = smem_desc(su32(sV) + 4096 * kk, 16384, 1024);
      const uint64_t db = smem_desc(su32(sBp) + 32 * kk, 16, 1024);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + 16),
          "l"(da), "l"(db), "r"(ip), "r"(kk));
    }
    // PV with u8 B MN-major (no swizzle): D cols 32..47
    const uint32_t im = idesc_i8(128, 16, 0, 0, 1, 1);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t da = smem_desc(su32(sV) + 4096 * kk, 16384, 1024);
      const uint64_t db = smem_desc_none(su32(sBm) + 512 * kk, 128, 256);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + 32),
          "l"(da), "l"(db), "r"(im), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&bar_mma))
                 : "memory");
  }
  mbar_wait(&bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[32];
  const uint32_t ta = tm + ((32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(ta + 16));
  uint32_t rm[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(rm[0]), "=r"(rm[1]), "=r"(rm[2]), "=r"(rm[3]), "=r"(rm[4]), "=r"(rm[5]), "=r"(rm[6]),
        "=r"(rm[7]), "=r"(rm[8]), "=r"(rm[9]), "=r"(rm[10]), "=r"(rm[11]), "=r"(rm[12]), "=r"(rm[13]),
        "=r"(rm[14]), "=r"(rm[15])
      : "r"(ta + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const uint32_t row = 32 * warp + lane;
  for (int n = 0; n < 16; ++n) a.out_pm[row * 16 + n] = (int32_t)rm[n];
  for (int n = 0; n < 16; ++n) {
    a.out_qk[row * 16 + n] = (int32_t)r[n];
    a.out_pv[row * 16 + n] = (int32_t)r[16 + n];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
  std::vector<uint8_t> K(128 * 128), V(128 * 128);
  std::vector<int8_t> Bq(16 * 128), Bp(16 * 128);
  srand(7);
  for (auto& x : K) x = rand() & 255;
  for (auto& x : V) x = rand() & 15;
  for (auto& x : Bq) x = (int8_t)((rand() & 255) - 128);
  for (auto& x : Bp) x = (int8_t)((rand() & 255) - 128);
  uint8_t *dK, *dV;
  int8_t *dBq, *dBp;
  int32_t *dq, *dp;
  CK(cudaMalloc(&dK, K.size()));
  CK(cudaMalloc(&dV, V.size()));
  CK(cudaMalloc(&dBq, Bq.size()));
  CK(cudaMalloc(&dBp, Bp.size()));
  CK(cudaMalloc(&dq, 128 * 16 * 4));
  CK(cudaMalloc(&dp, 128 * 16 * 4));
  CK(cudaMemcpy(dK, K.data(), K.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dV, V.data(), V.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBq, Bq.data(), Bq.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBp, Bp.data(), Bp.size(), cudaMemcpyHostToDevice));
  Args a{};
  {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    cuuint64_t dims[3] = {128, 128, 1}, strides[2] = {128, 128 * 128};
    cuuint32_t box[3] = {128, 128, 1}, es[3] = {1, 1, 1};
    CUresult r = ((EncodeFn)fn)(&a.tk, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dK, dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      std::printf("encode failed %d\n", (int)r);
      return 1;
    }
  }
  a.bq = dBq;
  a.vt = dV;
  a.bp = dBp;
  a.out_qk = dq;
  a.out_pv = dp;
  std::vector<uint8_t> Bm(128 * 16);
  for (auto& x : Bm) x = rand() & 255;
  uint8_t* dBm;
  int32_t* dpm;
  CK(cudaMalloc(&dBm, Bm.size()));
  CK(cudaMalloc(&dpm, 128 * 16 * 4));
  CK(cudaMemcpy(dBm, Bm.data(), Bm.size(), cudaMemcpyHostToDevice));
  a.bm = dBm;
  a.out_pm = dpm;
  const int smem = 1024 + 38912;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(a);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> oq(128 * 16), op(128 * 16);
  CK(cudaMemcpy(oq.data(), dq, oq.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(op.data(), dp, op.size() * 4, cudaMemcpyDeviceToHost));
  int bad_q = 0, bad_p = 0;
  for (int tok = 0; tok < 128; ++tok)
    for (int n = 0; n < 16; ++n) {
      int32_t e = 0;
      for (int k = 0; k < 128; ++k) e += (int32_t)K[tok * 128 + k] * Bq[n * 128 + k];
      if (e != oq[tok * 16 + n] && bad_q++ < 4)
        std::printf("qk tok %d n %d got %d want %d\n", tok, n, oq[tok * 16 + n], e);
    }
  for (int ch = 0; ch < 128; ++ch)
    for (int n = 0; n < 16; ++n) {
      int32_t e = 0;
      for (int tk = 0; tk < 128; ++tk) e += (int32_t)V[tk * 128 + ch] * Bp[n * 128 + tk];
      if (e != op[ch * 16 + n] && bad_p++ < 4)
        std::printf("pv ch %d n %d got %d want %d\n", ch, n, op[ch * 16 + n], e);
    }
  std::vector<int32_t> om(128 * 16);
  CK(cudaMemcpy(om.data(), dpm, om.size() * 4, cudaMemcpyDeviceToHost));
  int bad_m = 0;
  for (int ch = 0; ch < 128; ++ch)
    for (int n = 0; n < 16; ++n) {
      int32_t e = 0;
      for (int tk = 0; tk < 128; ++tk) e += (int32_t)V[tk * 128 + ch] * (int32_t)Bm[tk * 16 + n];
      if (e != om[ch * 16 + n] && bad_m++ < 4)
        std::printf("pv-mn ch %d n %d got %d want %d\n", ch, n, om[ch * 16 + n], e);
    }
  std::printf("{\"probe\": \"tcgen05 kind::i8\", \"qk_mismatches\": %d, \"pv_mismatches\": %d, "
              "\"pv_mn_b_mismatches\": %d}\n", bad_q, bad_p, bad_m);
  return bad_q || bad_p || bad_m;
}
