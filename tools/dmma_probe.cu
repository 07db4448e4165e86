// Dev probe: is the FP64 tensor-core path (mma.sync .f64, "DMMA") a pipe
// separate from the DFMA pipe on B200, and at what rate?  Standalone binary:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe tools/dmma_probe.cu
// Prints FMA/s for: DFMA alone, DMMA m8n8k4 alone, m16n8k4/k8/k16 alone, and
// mixed warps (every warp interleaves DMMA and DFMA chains).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double* d, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double* d, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double* d, const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// MODE 0: DFMA only (8 chains).  1: m8n8k4 only (8 independent accumulators).
// 2: m16n8k4.  3: m16n8k8.  4: m16n8k16.  5: mixed m8n8k4 (4 acc) + 8 DFMA
// chains per iteration.  6: mixed with 16 DFMA chains per 4 DMMA.
template <int MODE>
__global__ void __launch_bounds__(256) k_probe(double* out, int iters, double seed) {
  const double m = 0.999999999, c = 1e-9;
  double a[8], acc[8][4];
  for (int k = 0; k < 8; ++k) {
    a[k] = seed + threadIdx.x + k;
    for (int j = 0; j < 4; ++j) acc[k][j] = 0.0;
  }
  double av[8], bv[4];
  for (int k = 0; k < 8; ++k) av[k] = 1e-3 * (threadIdx.x + k);
  for (int k = 0; k < 4; ++k) bv[k] = 1e-3 * (k + 1);
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0 || MODE >= 5) {
#pragma unroll
      for (int r = 0; r < (MODE == 6 ? 2 : 1); ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    if (MODE == 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma884(acc[k][0], acc[k][1], av[k], bv[k & 3]);
    }
    if (MODE >= 5) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma884(acc[k][0], acc[k][1], av[k], bv[k & 3]);
    }
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma1684(acc[k], av[k], av[(k + 1) & 7], bv[k & 3]);
    }
    if (MODE == 3) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma1688(acc[k], av + (k & 4), bv + (k & 2));
    }
    if (MODE == 4) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma16816(acc[k], av, bv);
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k] + acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
static double run(double* out, int blocks, int iters, double fma_per_thread_iter) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_probe<MODE><<<blocks, 256>>>(out, 10, 1.0);
  cudaEventRecord(e0);
  k_probe<MODE><<<blocks, 256>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("mode %d: %s\n", MODE, cudaGetErrorString(e));
  const double fmas = (double)blocks * 256 * iters * fma_per_thread_iter;
  return fmas / (ms * 1e-3) * 2 / 1e12;  // TFLOP/s (FMA = 2)
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8;
  const int it = 20000;
  // per thread per iteration FMAs: DFMA 8; m8n8k4 = 256 FMA per warp = 8 per thread
  printf("DFMA only          %.2f TFLOP/s\n", run<0>(out, blocks, it, 8));
  printf("m8n8k4 only        %.2f TFLOP/s\n", run<1>(out, blocks, it, 8 * 8));
  printf("m16n8k4 only       %.2f TFLOP/s\n", run<2>(out, blocks, it, 8 * 16));
  printf("m16n8k8 only       %.2f TFLOP/s\n", run<3>(out, blocks, it, 8 * 32));
  printf("m16n8k16 only      %.2f TFLOP/s\n", run<4>(out, blocks, it, 8 * 64));
  const double t5 = run<5>(out, blocks, it, 8 + 4 * 8);
  printf("mixed 8 DFMA + 4 m8n8k4  %.2f TFLOP/s total (DFMA share %.0f%%)\n", t5, 100.0 * 8 / 40);
  const double t6 = run<6>(out, blocks, it, 16 + 4 * 8);
  printf("mixed 16 DFMA + 4 m8n8k4 %.2f TFLOP/s total (DFMA share %.0f%%)\n", t6, 100.0 * 16 / 48);
  return 0;
}
