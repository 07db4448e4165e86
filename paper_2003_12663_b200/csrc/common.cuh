// Shared device helpers for the hvb sm_100a kernels.
//
// Rounding contract: every *discrete*
// decision of the reference (pair classification, flat closest point,
// subdivision, grading trigger) is evaluated with the reference's exact
// operation sequence -- unfused products/sums through __dmul_rn/__dadd_rn
// (never contracted into FMAs by nvcc) and FMA chains where NumPy's ddot
// uses them.  Kernel *values* are free to use FMAs and the MUFU rsqrt seed
// plus a cubic Newton step; they differ from NumPy by O(1 ulp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HVB_DEV __device__ __forceinline__

namespace hvb {

constexpr double kInv4Pi = 0.079577471545947667884441881686257181;  // 1/(4 pi)

struct d3 {
  double x, y, z;
};

HVB_DEV d3 mk3(double x, double y, double z) { return d3{x, y, z}; }

// a - b with IEEE subtraction (component-wise, never fused)
HVB_DEV d3 sub_rn(d3 a, d3 b) {
  return mk3(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z));
}

// NumPy axis norm: sqrt((x*x + y*y) + z*z), unfused (src/assembly.py:156)
HVB_DEV double sumsq_unfused(d3 d) {
  return __dadd_rn(__dadd_rn(__dmul_rn(d.x, d.x), __dmul_rn(d.y, d.y)), __dmul_rn(d.z, d.z));
}

// NumPy 1-d length-3 dot through OpenBLAS ddot: fma(a2,b2, fma(a1,b1, a0*b0))
HVB_DEV double dot3_blas(d3 a, d3 b) {
  return __fma_rn(a.z, b.z, __fma_rn(a.y, b.y, __dmul_rn(a.x, b.x)));
}

// reciprocal square root: MUFU.RSQ64H seed + one cubic Householder step
// (relative error ~1e-17, i.e. O(ulp) against NumPy's 1/sqrt).
HVB_DEV double rsqrt_full(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  double h = r2 * y;
  double e = __fma_rn(-h, y, 1.0);          // e = 1 - r2 y^2
  double t = __fma_rn(e, 0.375, 0.5);       // 1/2 + 3/8 e
  double u = y * e;
  return __fma_rn(u, t, y);
}

// MUFU.RSQ64H seed + one Newton step (4 FP64 ops, relative error ~1e-12):
// used for the single-layer kernel, whose regular entries are sums of
// positive terms (entry error <= node error, 100x inside the 1e-10 parity).
HVB_DEV double rsqrt_newton(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double h = r2 * y;
  const double e = __fma_rn(-h, y, 1.0);
  return __fma_rn(y * 0.5, e, y);
}

// r2^(-3/2) from the MUFU.RSQ64H seed y0 in 5 FP64 ops: with a = y0^2 and
// e = r2 a - 1 (|e| ~ 2^-21), r^-3 = y0 a (1+e)^(-3/2) ~ y0 a (1 - 3/2 e);
// truncation 15/8 e^2 ~ 4e-13 relative (the second-order term would cost a
// sixth op for 1e-19).
HVB_DEV double rinv3_fast(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double a = y * y;
  const double e = __fma_rn(r2, a, -1.0);
  return (y * a) * __fma_rn(e, -1.5, 1.0);
}

// 2/sqrt(r2): MUFU.RSQ64H seed + one Newton step with the 1/2 folded out,
// y (3 - r2 y^2) -- 3 FP64 ops.  Callers scale their sums by 1/2 (or 1/8
// for r^-3) at the end, which is exact.
HVB_DEV double rsqrt2_newton(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double h = r2 * y;
  return y * __fma_rn(-h, y, 3.0);
}

// Classification "regular iff ||x - cc|| > eta R" exactly as the reference
// decides it (sqrt of the unfused sum, strict compare against fl(eta*R)).
// thr = fl(eta*R) and the squared bracket [lo, hi] are precomputed per
// triangle.  The bracket test uses the 3-op FMA sum of squares (within 4 ulp
// of the unfused sum, far inside the 1e-13 margins, so it decides as the
// unfused sum would); only pairs inside the bracket pay for the unfused sum
// and the IEEE sqrt.
HVB_DEV bool is_regular(d3 x, d3 cc, double thr, double thr2_lo, double thr2_hi) {
  const d3 d = sub_rn(x, cc);
  const double s = fma(d.z, d.z, fma(d.y, d.y, d.x * d.x));
  if (s > thr2_hi) return true;
  if (s < thr2_lo) return false;
  return __dsqrt_rn(sumsq_unfused(d)) > thr;
}

// Flat closest point (u*, v*) -- reference closest_point_flat,
// src/quadrature.py:236-277, same region order and rounding.
HVB_DEV void closest_point_flat(d3 x, d3 a, d3 b, d3 c, double& uo, double& vo) {
  d3 ab = sub_rn(b, a), ac = sub_rn(c, a);
  d3 ap = sub_rn(x, a);
  double d1 = dot3_blas(ab, ap), d2 = dot3_blas(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) { uo = 0.0; vo = 0.0; return; }
  d3 bp = sub_rn(x, b);
  double d3_ = dot3_blas(ab, bp), d4 = dot3_blas(ac, bp);
  if (d3_ >= 0.0 && d4 <= d3_) { uo = 1.0; vo = 0.0; return; }
  d3 cp = sub_rn(x, c);
  double d5 = dot3_blas(ab, cp), d6 = dot3_blas(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) { uo = 0.0; vo = 1.0; return; }
  double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3_, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) {
    uo = __ddiv_rn(d1, __dsub_rn(d1, d3_)); vo = 0.0; return;
  }
  double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    uo = 0.0; vo = __ddiv_rn(d2, __dsub_rn(d2, d6)); return;
  }
  double va = __dsub_rn(__dmul_rn(d3_, d6), __dmul_rn(d5, d4));
  double e43 = __dsub_rn(d4, d3_), e56 = __dsub_rn(d5, d6);
  if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
    double t = __ddiv_rn(e43, __dadd_rn(e43, e56));
    uo = __dsub_rn(1.0, t); vo = t; return;
  }
  double inv = __ddiv_rn(1.0, __dadd_rn(__dadd_rn(va, vb), vc));
  uo = __dmul_rn(vb, inv);
  vo = __dmul_rn(vc, inv);
}

// Quadratic 6-node map: shape values / gradients at (u, v)
// (reference src/mesh.py:124-158).  Values only (no rounding contract).
HVB_DEV void shape6(double u, double v, double* N, double* Nu, double* Nv) {
  double w = 1.0 - u - v;
  N[0] = w * (2.0 * w - 1.0);
  N[1] = u * (2.0 * u - 1.0);
  N[2] = v * (2.0 * v - 1.0);
  N[3] = 4.0 * w * u;
  N[4] = 4.0 * u * v;
  N[5] = 4.0 * v * w;
  Nu[0] = 1.0 - 4.0 * w; Nu[1] = 4.0 * u - 1.0; Nu[2] = 0.0;
  Nu[3] = 4.0 * (w - u); Nu[4] = 4.0 * v;       Nu[5] = -4.0 * v;
  Nv[0] = 1.0 - 4.0 * w; Nv[1] = 0.0;           Nv[2] = 4.0 * v - 1.0;
  Nv[3] = -4.0 * u;      Nv[4] = 4.0 * u;       Nv[5] = 4.0 * (w - v);
}

// Point and area element of the curved triangle (nodes: 18 doubles,
// node-major x,y,z) at (u, v).
HVB_DEV void curved_point(const double* __restrict__ X, double u, double v, d3& p, double& jac) {
  double N[6], Nu[6], Nv[6];
  shape6(u, v, N, Nu, Nv);
  double px = 0, py = 0, pz = 0, ux = 0, uy = 0, uz = 0, vx = 0, vy = 0, vz = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double xk = X[3 * k], yk = X[3 * k + 1], zk = X[3 * k + 2];
    px = fma(N[k], xk, px); py = fma(N[k], yk, py); pz = fma(N[k], zk, pz);
    ux = fma(Nu[k], xk, ux); uy = fma(Nu[k], yk, uy); uz = fma(Nu[k], zk, uz);
    vx = fma(Nv[k], xk, vx); vy = fma(Nv[k], yk, vy); vz = fma(Nv[k], zk, vz);
  }
  double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
  jac = sqrt(cx * cx + cy * cy + cz * cz);
  p = mk3(px, py, pz);
}

template <typename T>
HVB_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace hvb
