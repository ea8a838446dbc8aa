// North-star item (1) experiment: FP64 DMMA (mma.sync.m8n8k4.f64) vs DFMA for the 1D
// sum-factorisation contractions of the Q3 momentum kernel, in isolation.
//
// The contraction: Y[line][q] = sum_l T[q][l] X[line][l] for many lines of N = 4 nodal
// values (evaluation at the Q = 5 points of the k+2 rule, T = B; or an N x N line operator
// of pass A, T = [S; M] stacked to 8 rows).  Lines live in shared memory (the kernel's
// staging), results go back to shared memory, as inside k_momentum_axis; odd line
// strides (N + 1, 9) keep both variants' shared accesses bank-conflict-free.
//
//   DFMA: one line per thread, T in constant memory (the production kernel's form).
//   DMMA: 8 lines per m8n8k4 (A = lines 8 x 4, B = T^T 4 x 8, rows q >= Q zero), T in
//         registers (one element per lane), lines loaded as A fragments from shared memory.
//
// Reports useful TFLOP/s (2 * Q * N per line) for Q = 5 (B, 5 of 8 output columns used) and
// Q = 8 (a stacked pair of 4-row operators, all 8 used).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4;
__constant__ double cT[8][N];

template <int Q, int LINES_PER_WARP>
__global__ void dfma_lines(const double* __restrict__ gx, double* __restrict__ out, int reps) {
  __shared__ double sx[8][LINES_PER_WARP * (N + 1)];
  __shared__ double sy[8][LINES_PER_WARP * 9];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < LINES_PER_WARP * N; i += 32) sx[w][(i / N) * (N + 1) + i % N] = gx[(blockIdx.x * 8 + w) * LINES_PER_WARP * N + i];
  __syncwarp();
  double keep = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (int line = lane; line < LINES_PER_WARP; line += 32) {
      double x[N];
#pragma unroll
      for (int l = 0; l < N; ++l) x[l] = sx[w][line * (N + 1) + l];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(cT[q][l], x[l], s);
        sy[w][line * 9 + q] = s;
      }
    }
    __syncwarp();
    keep += sy[w][lane];
    __syncwarp();
  }
  if (keep == 12345.678) out[0] = keep;
}

template <int Q, int LINES_PER_WARP>
__global__ void dmma_lines(const double* __restrict__ gx, double* __restrict__ out, int reps) {
  __shared__ double sx[8][LINES_PER_WARP * (N + 1)];
  __shared__ double sy[8][LINES_PER_WARP * 9];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < LINES_PER_WARP * N; i += 32) sx[w][(i / N) * (N + 1) + i % N] = gx[(blockIdx.x * 8 + w) * LINES_PER_WARP * N + i];
  __syncwarp();
  // B fragment (4 x 8, col-major): B[k][n] = T[n][k], lane holds k = lane % 4, n = lane / 4
  const int g = lane >> 2, t = lane & 3;
  const double b = g < Q ? cT[g][t] : 0.0;
  double keep = 0.0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int l0 = 0; l0 < LINES_PER_WARP; l0 += 8) {
      // A fragment (8 x 4, row-major): lane holds A[g][t] = X[line l0 + g][t]
      const double a = sx[w][(l0 + g) * (N + 1) + t];
      double c0 = 0.0, c1 = 0.0;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      // C fragment: lane holds C[g][2t], C[g][2t+1] = Y[line l0+g][q = 2t, 2t+1]
      if (2 * t < Q) sy[w][(l0 + g) * 9 + 2 * t] = c0;
      if (2 * t + 1 < Q) sy[w][(l0 + g) * 9 + 2 * t + 1] = c1;
    }
    __syncwarp();
    keep += sy[w][lane];
    __syncwarp();
  }
  if (keep == 12345.678) out[0] = keep;
}

template <int Q>
void run(int sms) {
  constexpr int LPW = 48;
  const int blocks = sms * 8, reps = 2000;
  double *gx, *out;
  cudaMalloc(&gx, (size_t)blocks * 8 * LPW * N * sizeof(double));
  cudaMemset(gx, 0, (size_t)blocks * 8 * LPW * N * sizeof(double));
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flop = 2.0 * Q * N * (double)LPW * reps * blocks * 8;
  for (int v = 0; v < 2; ++v) {
    for (int warm = 0; warm < 2; ++warm) {
      cudaEventRecord(e0);
      if (v == 0)
        dfma_lines<Q, LPW><<<blocks, 256>>>(gx, out, reps);
      else
        dmma_lines<Q, LPW><<<blocks, 256>>>(gx, out, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("Q=%d %s: %.2f useful TFLOP/s (%.3f ms)\n", Q, v ? "DMMA m8n8k4" : "DFMA       ", flop / ms / 1e9, ms);
  }
  cudaFree(gx);
  cudaFree(out);
}

int main() {
  double T[8][N];
  for (int q = 0; q < 8; ++q)
    for (int l = 0; l < N; ++l) T[q][l] = 0.1 * (q + 1) - 0.07 * l;
  cudaMemcpyToSymbol(cT, T, sizeof(T));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<5>(sms);
  run<8>(sms);
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
