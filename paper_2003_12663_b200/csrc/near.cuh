// Near-singular pair machinery shared by the assembly / field near pass
// (near.cu) and the tracer's per-target near scan (trace.cu).
// Reference: row_pass2 src/assembly.py:245-292, near_singular_rule
// src/quadrature.py:409-450, subdivide_at 296-332.
#pragma once
#include "launch.cuh"

namespace hvb {

struct Piece {
  double ou, ov, e1u, e1v, e2u, e2v, wscale;
};

HVB_DEV int near_plan(const d3 X, const double* Xn, double R, int depth_cfg, double trigger, Piece* pc,
                      int& depth) {
  const d3 A = mk3(Xn[0], Xn[1], Xn[2]);
  const d3 B = mk3(Xn[3], Xn[4], Xn[5]);
  const d3 C = mk3(Xn[6], Xn[7], Xn[8]);
  double us, vs;
  closest_point_flat(X, A, B, C, us, vs);
  const d3 ba = sub_rn(B, A), ca = sub_rn(C, A);
  const d3 nearest = mk3(__dadd_rn(__dadd_rn(A.x, __dmul_rn(us, ba.x)), __dmul_rn(vs, ca.x)),
                         __dadd_rn(__dadd_rn(A.y, __dmul_rn(us, ba.y)), __dmul_rn(vs, ca.y)),
                         __dadd_rn(__dadd_rn(A.z, __dmul_rn(us, ba.z)), __dmul_rn(vs, ca.z)));
  const d3 dd = sub_rn(X, nearest);
  const double dist = __dsqrt_rn(dot3_blas(dd, dd));
  depth = (dist < __dmul_rn(trigger, R)) ? depth_cfg : 0;

  // subdivision at (u*, v*)
  const double bary[3] = {__dsub_rn(__dsub_rn(1.0, us), vs), us, vs};
  const double ref[3][2] = {{0.0, 0.0}, {1.0, 0.0}, {0.0, 1.0}};
  double sub[3][3][2];
  int nsub = 0;
  const double one_m = 1.0 - 1e-9;
  int corner = -1;
  for (int k = 0; k < 3; ++k)
    if (corner < 0 && bary[k] > one_m) corner = k;
  if (corner >= 0) {
    // whole reference triangle, rolled so the anchor is first
    for (int j = 0; j < 3; ++j) {
      sub[0][j][0] = ref[(corner + j) % 3][0];
      sub[0][j][1] = ref[(corner + j) % 3][1];
    }
    nsub = 1;
  } else {
    int zero = -1;
    for (int k = 0; k < 3; ++k)
      if (zero < 0 && bary[k] < 1e-9) zero = k;
    // fan edges: interior -> (0,1),(1,2),(2,0); on edge opposite k -> two
    int fan[3][2];
    if (zero == 0) { fan[0][0] = 2; fan[0][1] = 0; fan[1][0] = 0; fan[1][1] = 1; nsub = 2; }
    else if (zero == 1) { fan[0][0] = 0; fan[0][1] = 1; fan[1][0] = 1; fan[1][1] = 2; nsub = 2; }
    else if (zero == 2) { fan[0][0] = 1; fan[0][1] = 2; fan[1][0] = 2; fan[1][1] = 0; nsub = 2; }
    else {
      fan[0][0] = 0; fan[0][1] = 1; fan[1][0] = 1; fan[1][1] = 2; fan[2][0] = 2; fan[2][1] = 0;
      nsub = 3;
    }
    for (int s = 0; s < nsub; ++s) {
      sub[s][0][0] = us; sub[s][0][1] = vs;
      sub[s][1][0] = ref[fan[s][0]][0]; sub[s][1][1] = ref[fan[s][0]][1];
      sub[s][2][0] = ref[fan[s][1]][0]; sub[s][2][1] = ref[fan[s][1]][1];
    }
  }
  int np = 0;
  for (int s = 0; s < nsub; ++s) {
    double c[3][2] = {{sub[s][0][0], sub[s][0][1]}, {sub[s][1][0], sub[s][1][1]}, {sub[s][2][0], sub[s][2][1]}};
    double pcs[2][3][2];
    int npc;
    if (depth == 0) {
      for (int j = 0; j < 3; ++j) { pcs[0][j][0] = c[j][0]; pcs[0][j][1] = c[j][1]; }
      npc = 1;
    } else {
      double mu = 0.5 * (c[1][0] + c[2][0]), mv = 0.5 * (c[1][1] + c[2][1]);
      pcs[0][0][0] = c[0][0]; pcs[0][0][1] = c[0][1];
      pcs[0][1][0] = c[1][0]; pcs[0][1][1] = c[1][1];
      pcs[0][2][0] = mu;      pcs[0][2][1] = mv;
      pcs[1][0][0] = c[0][0]; pcs[1][0][1] = c[0][1];
      pcs[1][1][0] = mu;      pcs[1][1][1] = mv;
      pcs[1][2][0] = c[2][0]; pcs[1][2][1] = c[2][1];
      npc = 2;
    }
    for (int k = 0; k < npc; ++k) {
      Piece& P = pc[np++];
      P.ou = pcs[k][0][0];
      P.ov = pcs[k][0][1];
      P.e1u = pcs[k][1][0] - P.ou;
      P.e1v = pcs[k][1][1] - P.ov;
      P.e2u = pcs[k][2][0] - P.ou;
      P.e2v = pcs[k][2][1] - P.ov;
      double det = fabs(P.e1u * P.e2v - P.e1v * P.e2u);
      P.wscale = (2.0 * det) * 0.5;
    }
  }
  return np;
}

// Warp-cooperative composite-rule sum of one (point, panel) pair: lanes
// split the 128..3072 nodes; acc[9] (E: corner c, component d at 3c+d) or
// acc[0..2] (SL / ADL / potential) are this lane's partial sums (the caller
// reduces them with warp_sum).
HVB_DEV void near_pair_acc(const d3 X, const d3 N, int kind, const double* __restrict__ Xn, double R,
                           const double* __restrict__ duffy, int n_duffy, const double* __restrict__ graded,
                           int n_graded, int bisect_depth, double bisect_trigger, double* acc) {
  const int lane = threadIdx.x & 31;
  Piece pc[6];
  int depth;
  const int npc = near_plan(X, Xn, R, bisect_depth, bisect_trigger, pc, depth);
  const double* base = depth == 0 ? duffy : graded;
  const int nb = depth == 0 ? n_duffy : n_graded;
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = 0.0;
  for (int p = 0; p < npc; ++p) {
    const Piece Q = pc[p];
    for (int m = lane; m < nb; m += 32) {
      const double bu = base[4 * m], bv = base[4 * m + 1], bw = base[4 * m + 2];
      const double u = Q.ou + bu * Q.e1u + bv * Q.e2u;
      const double v = Q.ov + bu * Q.e1v + bv * Q.e2v;
      const double wq = bw * Q.wscale;
      d3 y;
      double jac;
      curved_point(Xn, u, v, y, jac);
      const double dx = X.x - y.x, dy = X.y - y.y, dz = X.z - y.z;
      const double r = sqrt(dx * dx + dy * dy + dz * dz);
      const double wj = wq * jac * kInv4Pi;
      const double h0 = 1.0 - u - v, h1 = u, h2 = v;
      if (kind == 2) {
        const double s = wj / (r * r * r);
        const double ex = dx * s, ey = dy * s, ez = dz * s;
        acc[0] = fma(h0, ex, acc[0]); acc[1] = fma(h0, ey, acc[1]); acc[2] = fma(h0, ez, acc[2]);
        acc[3] = fma(h1, ex, acc[3]); acc[4] = fma(h1, ey, acc[4]); acc[5] = fma(h1, ez, acc[5]);
        acc[6] = fma(h2, ex, acc[6]); acc[7] = fma(h2, ey, acc[7]); acc[8] = fma(h2, ez, acc[8]);
      } else {
        double k = (kind == 1) ? (dx * N.x + dy * N.y + dz * N.z) / (r * r * r) : 1.0 / r;
        k *= wj;
        acc[0] = fma(k, h0, acc[0]);
        acc[1] = fma(k, h1, acc[1]);
        acc[2] = fma(k, h2, acc[2]);
      }
    }
  }
}

}  // namespace hvb
