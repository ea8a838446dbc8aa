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
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
