// fp64 roofline denominator: DFMA throughput microbenchmark (MEASURED_PEAKS.json
// carries HBM and bf16 only).  Eight independent FMA chains per thread, enough
// resident warps to cover the DFMA latency on every SM.
#include <cuda_runtime.h>

#include "../../include/dgb.h"
#include "context.hpp"

namespace {
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}
// FP64 tensor-core path (DMMA, mma.sync m8n8k4): 256 FMA per warp instruction, eight
// independent accumulator pairs per thread.  On B200 it shares the FP64 pipe with DFMA
// (profiles/fp64_dfma_dmma_mixed_r02.txt) and peaks ~8 % higher.
__global__ void k_dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i][0] = i;
    c[i][1] = -i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

extern "C" int dgb_fp64_peak_dmma(dgb_ctx* h, double* tflops) {
  if (!h || !tflops) return DGB_E_ARG;
  DevGuard guard_(h);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->c.device);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return DGB_E_CUDA;
  const int blocks = sms * 2, threads = 256, iters = 20000;
  cudaStream_t s = h->c.dc.stream;
  k_dmma_peak<<<blocks, threads, 0, s>>>(d, 200);
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(h->c.ev0, s);
    k_dmma_peak<<<blocks, threads, 0, s>>>(d, iters);
    cudaEventRecord(h->c.ev1, s);
    cudaEventSynchronize(h->c.ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->c.ev0, h->c.ev1);
    // one m8n8k4 = 8 * 8 * 4 FMA per warp
    const double tf = 2.0 * 256.0 * 8 * (double)iters * (threads / 32) * blocks / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaFree(d);
  *tflops = best;
  return cudaGetLastError() == cudaSuccess ? DGB_OK : DGB_E_CUDA;
}

extern "C" int dgb_fp64_peak(dgb_ctx* h, double* tflops) {
  if (!h || !tflops) return DGB_E_ARG;
  DevGuard guard_(h);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->c.device);
  double* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return DGB_E_CUDA;
  const int blocks = sms * 8, threads = 256, iters = 20000;
  cudaStream_t s = h->c.dc.stream;
  k_dfma_peak<<<blocks, threads, 0, s>>>(d, 200, 1.0000001, 1e-7);
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(h->c.ev0, s);
    k_dfma_peak<<<blocks, threads, 0, s>>>(d, iters, 1.0000001, 1e-7);
    cudaEventRecord(h->c.ev1, s);
    cudaEventSynchronize(h->c.ev1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->c.ev0, h->c.ev1);
    const double tf = 2.0 * 8 * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaFree(d);
  *tflops = best;
  return cudaGetLastError() == cudaSuccess ? DGB_OK : DGB_E_CUDA;
}
