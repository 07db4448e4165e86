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

// dependent-chain latency (cycles per op) of a few FP64 operations
__global__ void k_latency(double* out, int n, double seed) {
  double x = seed, y = 1.0000001, z = 1e-9;
  long long t0, t1;
  double res[5];
  // 0: DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, z);
  t1 = clock64();
  res[0] = (double)(t1 - t0) / n;
  double s = x;
  // 1: DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + z;
  t1 = clock64();
  res[1] = (double)(t1 - t0) / n;
  s += x;
  // 2: MUFU.RSQ64H chain
  x = 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r + 1.5;
  }
  t1 = clock64();
  res[2] = (double)(t1 - t0) / n;
  s += x;
  // 3: full rsqrt (seed + cubic step) chain
  x = 2.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt_full(x) + 1.5;
  t1 = clock64();
  res[3] = (double)(t1 - t0) / n;
  s += x;
  // 4: LDS -> DADD -> STS round trip on shared memory
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = 1.0;
  __syncwarp();
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    volatile double* v = sm;
    v[i & 7] = v[(i + 7) & 7] + z;
  }
  t1 = clock64();
  res[4] = (double)(t1 - t0) / n;
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) out[k] = res[k];
  if (s == 12345.0) out[7] = s;
}

// Node-loop throughput probe: the SL node of the regular sweep with operands
// in registers (no shared memory, no window).  VAR 0: full node (MUFU seed
// + cubic step); 1: without the rsqrt (FP64 arithmetic only); 2: quadratic
// step.  Each thread evaluates `iters` x 12 nodes for 2 targets.
template <int VAR>
__global__ void __launch_bounds__(256) k_node_probe(double* out, int iters) {
  const double t = 1e-3 * threadIdx.x;
  double x0 = 0.3 + t, y0 = 0.2, z0 = 0.1 - t, x1 = 0.31, y1 = 0.21 + t, z1 = 0.12;
  double a0 = 0, a1 = 0, a2 = 0, b0 = 0, b1 = 0, b2 = 0;
  for (int i = 0; i < iters; ++i) {
    const double s = 1e-7 * i;
#pragma unroll
    for (int q = 0; q < 12; ++q) {
      const double px = 0.01 * q + s, py = 0.02 * q, pz = -0.01 * q;
      const double w0 = 0.1 + 0.001 * q, w1 = 0.2, w2 = 0.3 - 0.001 * q;
      const double dx0 = x0 - px, dy0 = y0 - py, dz0 = z0 - pz;
      const double dx1 = x1 - px, dy1 = y1 - py, dz1 = z1 - pz;
      const double r20 = fma(dz0, dz0, fma(dy0, dy0, dx0 * dx0));
      const double r21 = fma(dz1, dz1, fma(dy1, dy1, dx1 * dx1));
      double k0, k1;
      if (VAR == 0) {
        k0 = rsqrt_full(r20);
        k1 = rsqrt_full(r21);
      } else if (VAR == 1) {
        k0 = r20;
        k1 = r21;
      } else if (VAR == 3) {
        k0 = rsqrt2_newton(r20);
        k1 = rsqrt2_newton(r21);
      } else {
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r20));
        k0 = fma(y * 0.5, fma(-r20 * y, y, 1.0), y);
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r21));
        k1 = fma(y * 0.5, fma(-r21 * y, y, 1.0), y);
      }
      a0 = fma(k0, w0, a0); a1 = fma(k0, w1, a1); a2 = fma(k0, w2, a2);
      b0 = fma(k1, w0, b0); b1 = fma(k1, w1, b1); b2 = fma(k1, w2, b2);
    }
  }
  const double r = a0 + a1 + a2 + b0 + b1 + b2;
  if (r == 12345.678) out[0] = r;
}

}  // namespace hvb

namespace hvb {
__global__ void k_rsqrt_probe(const double* r2, int n, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[3 * i] = rsqrt2_newton(r2[i]);
  out[3 * i + 1] = rsqrt_full(r2[i]);
  out[3 * i + 2] = rinv3(r2[i]);
}
}  // namespace hvb

// accuracy probe of the rsqrt refinements: out (n, 3) = 2/sqrt, 1/sqrt, r^-3
extern "C" int hvb_bench_rsqrt(const double* r2, int n, double* out, void* stream) {
  hvb::k_rsqrt_probe<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(r2, n, out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int hvb_bench_nodes(double* out, int var, int blocks, int threads, int iters, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (var == 0) hvb::k_node_probe<0><<<blocks, threads, 0, st>>>(out, iters);
  else if (var == 1) hvb::k_node_probe<1><<<blocks, threads, 0, st>>>(out, iters);
  else if (var == 3) hvb::k_node_probe<3><<<blocks, threads, 0, st>>>(out, iters);
  else hvb::k_node_probe<2><<<blocks, threads, 0, st>>>(out, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int hvb_bench_latency(double* out, int n, void* stream) {
  hvb::k_latency<<<1, 32, 0, (cudaStream_t)stream>>>(out, n, 1.0);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

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
