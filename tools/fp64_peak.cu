// fp64 throughput microbenchmark: DFMA (CUDA cores) and DMMA (mma.sync m8n8k4 f64).
// Used once to record the fp64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// DFMA and DMMA interleaved in the same warps: if the combined rate exceeds either
// alone, the two run on separate pipes (the DMMA-for-contractions design question).
template <int ILPF, int ILPM>
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double r[ILPF];
#pragma unroll
  for (int i = 0; i < ILPF; ++i) r[i] = threadIdx.x * 1e-9 + i;
  double ma = threadIdx.x * 1e-3, mb = 0.5;
  double c[ILPM][2];
#pragma unroll
  for (int i = 0; i < ILPM; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILPM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(ma), "d"(mb));
#pragma unroll
    for (int i = 0; i < ILPF; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILPF; ++i) s += r[i];
#pragma unroll
  for (int i = 0; i < ILPM; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// dependent-chain latency of one DMMA / one DFMA (one warp)
__global__ void lat_kernel(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 0.5, c0 = 1.0, c1 = 2.0, r = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  for (int it = 0; it < iters; ++it) r = fma(r, 1.0000001, 1e-7);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  if (c0 + c1 + r == 12345.678) out[0] = c0;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm : {2, 4, 8}) {
      int iters = 20000; const int ILP = 8; int threads = 256;
      dfma_kernel<ILP><<<sms * bpsm, threads>>>(d, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dfma_kernel<ILP><<<sms * bpsm, threads>>>(d, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * ILP * (double)iters * threads * sms * bpsm;
      printf("DFMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
    }
    for (int bpsm : {1, 2, 4, 8}) {
      int iters = 20000; const int ILP = 4; int threads = 128;
      dmma_kernel<ILP><<<sms * bpsm, threads>>>(d, 100);
      cudaEventRecord(e0);
      dmma_kernel<ILP><<<sms * bpsm, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * ILP * (double)iters * (threads / 32) * sms * bpsm;
      printf("DMMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
    }
  }
  for (int bpsm : {2, 4}) {
    const int iters = 20000, threads = 256;
    mixed_kernel<8, 4><<<sms * bpsm, threads>>>(d, 100, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    mixed_kernel<8, 4><<<sms * bpsm, threads>>>(d, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (threads / 32.0) * sms * bpsm;
    const double ff = 2.0 * 8 * (double)iters * threads * sms * bpsm, fm = 2.0 * 256 * 4 * (double)iters * warps;
    printf("MIXED blocks/SM=%d: DFMA %.2f + DMMA %.2f = %.2f TFLOP/s (%.3f ms)\n", bpsm, ff / ms / 1e9,
           fm / ms / 1e9, (ff + fm) / ms / 1e9, ms);
  }
  {
    long long* cyc; cudaMalloc(&cyc, 16);
    lat_kernel<<<1, 32>>>(d, 1000, cyc);
    long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("latency: DMMA %.1f cycles, DFMA %.1f cycles (dependent chain)\n", h[0] / 1000.0, h[1] / 1000.0);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
