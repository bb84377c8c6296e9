// Phase timing of select_fused_kernel (%globaltimer stamps per CTA), not a
// product path: compiles ttkv_select.cu with TTKV_PHASE_STAMP defined.
//   ../build/fused_probe [S] [n] [Gs]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
__device__ unsigned long long g_stamp[8192][8];
#define TTKV_PHASE_STAMP(k)                                                               \
  do {                                                                                    \
    if (threadIdx.x == 0) {                                                               \
      unsigned long long t_;                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      g_stamp[blockIdx.y * gridDim.x + blockIdx.x][k] = t_;                               \
    }                                                                                     \
  } while (0)
#include "../paper_2604_19769_b200/csrc/ttkv_select.cu"
bool ttkv_dev::pdl_enabled() { return false; }
int ttkv_dev::launch_priority(bool) { return 0; }
using namespace ttkv_dev;
int main(int argc, char** argv) {
  const uint32_t S = argc > 1 ? atoi(argv[1]) : 8, n = argc > 2 ? atoi(argv[2]) : 992;
  const uint32_t Gs = argc > 3 ? atoi(argv[3]) : 4, d = 128;
  Geometry g{};
  g.S = S; g.G = Gs; g.Gs = Gs; g.d_k = d; g.d_v = d; g.B = 128; g.n_cap = n;
  std::vector<float> hc((size_t)S * n * d), hq((size_t)S * Gs * d);
  srand(1);
  for (auto& x : hc) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : hq) x = (float)rand() / RAND_MAX - 0.5f;
  FusedSelectArgs a{};
  a.g = g; a.n = n; a.k = (uint32_t)(0.45 * n);
  float *q, *c; double* sc; uint32_t *ui, *um, *uc;
  cudaMalloc(&q, hq.size() * 4); cudaMalloc(&c, hc.size() * 4);
  cudaMalloc(&sc, (size_t)S * Gs * n * 8);
  cudaMalloc(&ui, (size_t)S * n * 4); cudaMalloc(&um, (size_t)S * n * 4); cudaMalloc(&uc, S * 4);
  cudaMemcpy(q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(c, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
  a.q = q; a.cent = c; a.scores = sc; a.union_ids = ui; a.union_mask = um; a.union_count = uc;
  if (!select_fused_supported(g, n, 148)) { printf("unsupported\n"); return 1; }
  const FusedLayout L = fused_layout(g, n);
  printf("S=%u n=%u Gs=%u CL=%u nb=%u smem=%zu\n", S, n, Gs, L.CL, L.nb, L.bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0);
    cudaError_t e = launch_select_fused(a, 0);  // probe: default stream
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> st(8192 * 8);
    cudaMemcpyFromSymbol(st.data(), g_stamp, st.size() * 8);
    const uint32_t nct = L.CL * S;
    unsigned long long t0 = ~0ull;
    for (uint32_t i = 0; i < nct; ++i) t0 = std::min(t0, st[i * 8 + 0]);
    double mx[8] = {0};
    for (uint32_t i = 0; i < nct; ++i)
      for (int k = 0; k < 8; ++k) {
        if ((k == 4 || k == 5) && (i % L.CL) >= Gs) continue;
        if (k == 7 && (i % L.CL) != 0) continue;
        mx[k] = std::max(mx[k], (double)(st[i * 8 + k] - t0) / 1e3);
      }
    printf("event %.2f us | max over CTAs (us from first start): start %.2f loaded %.2f scored %.2f "
           "sync1 %.2f gathered %.2f radix %.2f sync2 %.2f union %.2f\n", ms * 1e3, mx[0], mx[1],
           mx[2], mx[3], mx[4], mx[5], mx[6], mx[7]);
  }
  return 0;
}
