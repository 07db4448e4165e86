// Roofline denominators measured on the box (MEASURED_PEAKS.json has no
// FP64 entry): a DFMA-throughput kernel (8 independent FMA chains per
// thread, full occupancy) and a read-only HBM stream.
#include "launch.cuh"

namespace hvb {

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// read-only HBM stream with 256-bit non-allocating loads (the GEMV's load)
__global__ void __launch_bounds__(256) k_read_stream4(const double* __restrict__ p, long long n4, double* out) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    double a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p + 4 * i));
    acc += (a + b) + (c + d);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __launch_bounds__(256) k_read_stream(const double2* __restrict__ p, long long n2, double* out) {
  double acc = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2 * stride),
            v3 = __ldcs(p + i + 3 * stride);
    acc += (v0.x + v0.y) + (v1.x + v1.y) + (v2.x + v2.y) + (v3.x + v3.y);
  }
  for (; i < n2; i += stride) {
    double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

}  // namespace hvb

extern "C" int hvb_bench_dfma(double* out, int blocks, int iters, void* stream) {
  hvb::k_dfma_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters, 1.0);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int hvb_bench_read(const double* p, long long n, double* out, int blocks, void* stream) {
  if (n % 4 == 0)
    hvb::k_read_stream4<<<blocks, 256, 0, (cudaStream_t)stream>>>(p, n / 4, out);
  else
    hvb::k_read_stream<<<blocks, 256, 0, (cudaStream_t)stream>>>((const double2*)p, n / 2, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
