// host_issue_probe.cu -- where the host time of one synchronous decode step
// goes (the e2e gap of small steps, cfg1 with the slow tier in HBM).
//
//   build/host_issue_probe [streams] [heads] [ctx] [slow_tier 0|1]
//
// Prints (median over 600 calls -- means where named -- microseconds):
//   * the synchronous host-buffer step (ttkv_gpu_decode_step) with pinned and
//     pageable caller buffers,
//   * the device-buffer step split into its enqueue (the call returns without
//     synchronizing) and the wait after it,
//   * the host cost of the CUDA runtime calls a step issues, each alone:
//     cudaLaunchKernelEx (PDL attribute), cudaFuncSetAttribute,
//     cudaMemcpyAsync (16 KB pinned), cudaEventRecord, cudaStreamWaitEvent,
//     cudaPointerGetAttributes, cudaSetDevice, and the empty-stream sync.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <random>
#include <vector>

#include "../include/ttkv_gpu.h"

__global__ void empty_kernel(int) {}

static double g_mean = 0;  // mean of the last median_us run
static double median_us(int n, const std::function<void()>& f) {
  std::vector<double> t(n);
  double sum = 0;
  for (int i = 0; i < n; ++i) {
    const auto a = std::chrono::steady_clock::now();
    f();
    t[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
    sum += t[i];
  }
  g_mean = sum / n;
  std::sort(t.begin(), t.end());
  return t[n / 2];
}

static int fail(ttkv_gpu* h, const char* what) {
  std::fprintf(stderr, "%s: %s\n", what, h ? ttkv_gpu_last_error(h) : ttkv_last_error());
  return 1;
}

int main(int argc, char** argv) {
  const uint32_t S = argc > 1 ? std::atoi(argv[1]) : 32;
  const uint32_t G = argc > 2 ? std::atoi(argv[2]) : 1;
  const uint64_t ctx = argc > 3 ? std::atoll(argv[3]) : 32768;
  const uint32_t tier = argc > 4 ? std::atoi(argv[4]) : 1;
  const uint32_t d = 128;
  const int N = 600;

  ttkv_tier_config cfg;
  ttkv_default_config(&cfg);
  cfg.d_k = cfg.d_v = d;
  cfg.block_size = 128;
  cfg.hbm_budget_bytes = 4096ull * 2 * d * 2;  // L_fast = 4096
  ttkv_selection_policy pol = {0, 0, 0.45};
  ttkv_gpu_options opt = {};
  opt.n_streams = S;
  opt.heads_per_stream = G;
  opt.reserve_tokens = ctx + 4 * N + 256;
  opt.slow_tier = tier ? TTKV_SLOW_DEVICE : TTKV_SLOW_PINNED_HOST;
  ttkv_gpu* h = nullptr;
  if (ttkv_gpu_create(&cfg, &pol, &opt, &h)) return fail(nullptr, "create");
  if (ttkv_gpu_prefill_synthetic(h, ctx, 1)) return fail(h, "prefill");

  const size_t qn = (size_t)S * G * d, kn = (size_t)S * d, on = (size_t)S * G * d;
  std::vector<float> q(qn), k(kn), v(kn);
  std::vector<double> out(on);
  std::mt19937 gen(0);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (auto& x : q) x = nd(gen);
  for (auto& x : k) x = nd(gen);
  for (auto& x : v) x = nd(gen);
  float *pq, *pk, *pv;
  double* pout;
  cudaHostAlloc(&pq, qn * 4, 0);
  cudaHostAlloc(&pk, kn * 4, 0);
  cudaHostAlloc(&pv, kn * 4, 0);
  cudaHostAlloc(&pout, on * 8, 0);
  std::copy(q.begin(), q.end(), pq);
  std::copy(k.begin(), k.end(), pk);
  std::copy(v.begin(), v.end(), pv);
  float *dq, *dk, *dv;
  double* dout;
  cudaMalloc(&dq, qn * 4);
  cudaMalloc(&dk, kn * 4);
  cudaMalloc(&dv, kn * 4);
  cudaMalloc(&dout, on * 8);
  cudaMemcpy(dq, pq, qn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, pk, kn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, pv, kn * 4, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (ttkv_gpu_set_stream(h, st)) return fail(h, "set_stream");

  ttkv_step_report rep{};
  int rc = 0;
  auto step_pinned = [&] {
    rc |= ttkv_gpu_decode_step(h, pq, pk, pv, TTKV_DTYPE_F32, pout, &rep);
  };
  auto step_pageable = [&] {
    rc |= ttkv_gpu_decode_step(h, q.data(), k.data(), v.data(), TTKV_DTYPE_F32, out.data(), &rep);
  };
  // four page-locked buffer sets used in turn (as bench.py's e2e leg does)
  constexpr int kPool = 4;
  float *rq[kPool], *rk[kPool], *rv[kPool];
  for (int j = 0; j < kPool; ++j) {
    cudaHostAlloc(&rq[j], qn * 4, 0);
    cudaHostAlloc(&rk[j], kn * 4, 0);
    cudaHostAlloc(&rv[j], kn * 4, 0);
    std::copy(q.begin(), q.end(), rq[j]);
    std::copy(k.begin(), k.end(), rk[j]);
    std::copy(v.begin(), v.end(), rv[j]);
  }
  int turn = 0;
  auto step_rotating = [&] {
    const int j = turn++ % kPool;
    rc |= ttkv_gpu_decode_step(h, rq[j], rk[j], rv[j], TTKV_DTYPE_F32, pout, &rep);
  };
  for (int i = 0; i < 5; ++i) step_pinned();
  const double t_pinned = median_us(N, step_pinned);
  const double m_pinned = g_mean;
  const double t_pageable = median_us(N, step_pageable);
  const double m_pageable = g_mean;
  const double t_rot = median_us(N, step_rotating);
  const double m_rot = g_mean;
  // device buffers: enqueue, then wait
  std::vector<double> enq(N), wait(N);
  for (int i = 0; i < N; ++i) {
    const auto a = std::chrono::steady_clock::now();
    rc |= ttkv_gpu_decode_step_device(h, dq, dk, dv, TTKV_DTYPE_F32, dout, nullptr);
    const auto b = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    const auto c = std::chrono::steady_clock::now();
    enq[i] = std::chrono::duration<double, std::micro>(b - a).count();
    wait[i] = std::chrono::duration<double, std::micro>(c - b).count();
  }
  if (rc) return fail(h, "decode");
  std::sort(enq.begin(), enq.end());
  std::sort(wait.begin(), wait.end());

  // the runtime calls, each alone
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(1);
  lc.blockDim = dim3(32);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const double t_launch = median_us(N, [&] { cudaLaunchKernelEx(&lc, empty_kernel, 0); });
  cudaStreamSynchronize(st);
  const double t_launch_plain = median_us(N, [&] { empty_kernel<<<1, 32, 0, st>>>(0); });
  cudaStreamSynchronize(st);
  const double t_attr = median_us(N, [&] {
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  });
  const double t_h2d = median_us(N, [&] { cudaMemcpyAsync(dk, pk, kn * 4, cudaMemcpyHostToDevice, st); });
  cudaStreamSynchronize(st);
  const double t_d2h = median_us(N, [&] { cudaMemcpyAsync(pk, dk, kn * 4, cudaMemcpyDeviceToHost, st); });
  cudaStreamSynchronize(st);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  const double t_rec = median_us(N, [&] { cudaEventRecord(ev, st); });
  const double t_wait = median_us(N, [&] { cudaStreamWaitEvent(st, ev, 0); });
  cudaPointerAttributes pa;
  const double t_ptr = median_us(N, [&] { cudaPointerGetAttributes(&pa, q.data()); cudaGetLastError(); });
  const double t_ptr_pinned = median_us(N, [&] { cudaPointerGetAttributes(&pa, pq); });
  const double t_setdev = median_us(N, [&] { cudaSetDevice(0); });
  const double t_sync = median_us(N, [&] { cudaStreamSynchronize(st); });
  // a round trip: one kernel + sync
  const double t_rt = median_us(N, [&] {
    empty_kernel<<<1, 32, 0, st>>>(0);
    cudaStreamSynchronize(st);
  });
  const double t_rt_copy = median_us(N, [&] {
    cudaMemcpyAsync(dk, pk, kn * 4, cudaMemcpyHostToDevice, st);
    empty_kernel<<<1, 32, 0, st>>>(0);
    cudaMemcpyAsync(pout, dout, on * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  });
  std::printf(
      "{\"probe\": \"host_issue\", \"streams\": %u, \"heads\": %u, \"ctx\": %llu, \"tier\": %u,\n"
      " \"step_host_pinned_us\": %.2f, \"step_host_pageable_us\": %.2f,\n"
      " \"mean_incl_recaptures_pinned_us\": %.2f, \"mean_pageable_us\": %.2f,\n"
      " \"step_host_4_buffer_sets_us\": %.2f, \"mean_4_buffer_sets_us\": %.2f,\n"
      " \"step_device_enqueue_us\": %.2f, \"step_device_wait_us\": %.2f,\n"
      " \"launch_ex_pdl_us\": %.2f, \"launch_plain_us\": %.2f, \"func_set_attr_us\": %.2f,\n"
      " \"memcpy_h2d_16k_us\": %.2f, \"memcpy_d2h_16k_us\": %.2f, \"event_record_us\": %.2f,\n"
      " \"stream_wait_event_us\": %.2f, \"pointer_attr_pageable_us\": %.2f,\n"
      " \"pointer_attr_pinned_us\": %.2f, \"set_device_us\": %.2f, \"empty_sync_us\": %.2f,\n"
      " \"kernel_roundtrip_us\": %.2f, \"copy_kernel_copy_roundtrip_us\": %.2f}\n",
      S, G, (unsigned long long)ctx, tier, t_pinned, t_pageable, m_pinned, m_pageable, t_rot,
      m_rot, enq[N / 2], wait[N / 2], t_launch,
      t_launch_plain, t_attr, t_h2d, t_d2h, t_rec, t_wait, t_ptr, t_ptr_pinned, t_setdev, t_sync,
      t_rt, t_rt_copy);
  ttkv_gpu_destroy(h);
  return 0;
}
