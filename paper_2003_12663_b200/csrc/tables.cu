// Assembly support kernels: regular-rule sample table (K1), panel-stream
// packing, the singular Duffy pass (K4) and the floating columns (K6).  The
// regular sweep itself is csrc/assemble.cu.
//
// Reference: TriangleTables src/assembly.py:73-118, row_pass1 singular batch
// 202-235, _row_equation 408-468.
#include "launch.cuh"

namespace hvb {

// K1: regular-rule sample table.  out[t][q] = (y_tq, jw_tq*hat_c(q)/(4 pi))
// (reference TriangleTables.__init__, src/assembly.py:78-103).
__global__ void k_build_table(const double* __restrict__ nodes6, int nt, int nq,
                              const double* __restrict__ rule,  // nq x 4: u, v, w, pad
                              double* __restrict__ out) {
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nt * nq) return;
  int t = gid / nq, q = gid % nq;
  double u = rule[4 * q], v = rule[4 * q + 1], w = rule[4 * q + 2];
  d3 p;
  double jac;
  curved_point(nodes6 + 18 * (size_t)t, u, v, p, jac);
  double jw = w * jac * kInv4Pi;
  double* o = out + 6 * (size_t)gid;
  o[0] = p.x; o[1] = p.y; o[2] = p.z;
  o[3] = jw * (1.0 - u - v);
  o[4] = jw * u;
  o[5] = jw * v;
}

// Per-panel device arrays from the circumcircles (one warp per aligned
// group of 32 panels, the tail padded with the last panel):
//   ccr    (nt, 4) = cc, R                          (surface distance, streams)
//   cls    (nt, 6) = cc, thr = fl(eta R), thr^2 (1 -+ 1e-13)  (field kernels)
//   groups (ng, 8) = C, rho_cls, rho_sd, 0, 0, 0    (device.py panel_groups)
// with numpy's rounding order (no contraction), so the arrays equal the host
// statement device.py:panel_groups bit for bit (tests/test_gpu_edge.py).
__global__ void k_panel_data(const double* __restrict__ cc, const double* __restrict__ radii, int nt, double eta,
                             double* __restrict__ ccr, double* __restrict__ cls, double* __restrict__ groups) {
  const int lane = threadIdx.x & 31;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= (nt + 31) / 32) return;
  const int i = g * 32 + lane;
  const int t = min(i, nt - 1);
  const double cx = cc[3 * (size_t)t], cy = cc[3 * (size_t)t + 1], cz = cc[3 * (size_t)t + 2];
  const double R = radii[t];
  const double thr = __dmul_rn(eta, R);
  if (i < nt) {
    double* o = ccr + 4 * (size_t)i;
    o[0] = cx; o[1] = cy; o[2] = cz; o[3] = R;
    const double t2 = __dmul_rn(thr, thr);
    double* c = cls + 6 * (size_t)i;
    c[0] = cx; c[1] = cy; c[2] = cz; c[3] = thr;
    c[4] = __dmul_rn(t2, 1.0 - 1e-13);
    c[5] = __dmul_rn(t2, 1.0 + 1e-13);
  }
  double lo[3] = {cx, cy, cz}, hi[3] = {cx, cy, cz};
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  const double Cx = __dmul_rn(0.5, __dadd_rn(lo[0], hi[0]));
  const double Cy = __dmul_rn(0.5, __dadd_rn(lo[1], hi[1]));
  const double Cz = __dmul_rn(0.5, __dadd_rn(lo[2], hi[2]));
  const double dx = __dsub_rn(cx, Cx), dy = __dsub_rn(cy, Cy), dz = __dsub_rn(cz, Cz);
  const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  double rc = __dadd_rn(d, thr), rs = __dadd_rn(d, R);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    rc = fmax(rc, __shfl_xor_sync(0xffffffffu, rc, o));
    rs = fmax(rs, __shfl_xor_sync(0xffffffffu, rs, o));
  }
  if (lane == 0) {
    double* o = groups + 8 * (size_t)g;
    o[0] = Cx; o[1] = Cy; o[2] = Cz;
    o[3] = __dmul_rn(rc, 1.0 + 1e-12);
    o[4] = __dmul_rn(rs, 1.0 + 1e-12);
    o[5] = o[6] = o[7] = 0.0;
  }
}

// Pack one stream record per (tile, panel) entry (record formats: see
// csrc/assemble.cu).  mode 0 = SL stream: per node q of panel t, with
// w = jw/(4 pi) (the table's three weights summed), s = 1/w^2 and
// y' = y - cc (IEEE):  Y = -2 s y', P = s |y'|^2, Q = s, stored per node
// pair as [Y0x Y0y | Y0z P0 | Q0 Q1 | Y1x Y1y | Y1z P1]; an odd nq is padded
// with a node (Y = 0, P = 1, Q = 0) whose hat values are zero.  mode 1 = ADL
// stream: the table's (y, w hat_0, w hat_1, w hat_2) per node.
__global__ void k_build_stream(const double* __restrict__ table, int nq,
                               const double* __restrict__ ccr,  // (nt,4): cc, R
                               double eta, const int* __restrict__ ent_tri,
                               const int* __restrict__ ent_meta,  // (ne,5): mfirst, slot0, slot1, slot2, flags
                               int64_t ne, int mode, int rec, int window, int wstride, double* __restrict__ out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int t = ent_tri[e];  // -1: dummy record padding a stage (dump slot, never emits)
  double* o = out + e * rec;
  if (t < 0) {
    for (int k = 0; k < rec - 2; ++k) o[k] = 0.0;
    if (mode == 0)
      for (int q = 0; q < ((nq + 1) & ~1); ++q) o[10 * (q >> 1) + ((q & 1) ? 9 : 3)] = 1.0;  // P = 1: finite
  } else {
    const double* s = table + (size_t)t * 6 * nq;
    const double* c = ccr + 4 * (size_t)t;
    if (mode == 0) {
      const int nqp = (nq + 1) & ~1;
      for (int q = 0; q < nqp; ++q) {
        double Y[3] = {0.0, 0.0, 0.0}, P = 1.0, Q = 0.0;
        if (q < nq) {
          const double* y = s + 6 * q;
          const d3 yc = sub_rn(mk3(y[0], y[1], y[2]), mk3(c[0], c[1], c[2]));
          const double w = (y[3] + y[4]) + y[5];
          const double sc = 1.0 / (w * w);
          Y[0] = -2.0 * sc * yc.x;
          Y[1] = -2.0 * sc * yc.y;
          Y[2] = -2.0 * sc * yc.z;
          P = sc * sumsq_unfused(yc);
          Q = sc;
        }
        double* op = o + 10 * (q >> 1);
        if ((q & 1) == 0) {
          op[0] = Y[0]; op[1] = Y[1]; op[2] = Y[2]; op[3] = P; op[4] = Q;
        } else {
          op[5] = Q; op[6] = Y[0]; op[7] = Y[1]; op[8] = Y[2]; op[9] = P;
        }
      }
    } else {
      for (int k = 0; k < 6 * nq; ++k) o[k] = s[k];
    }
    const double thr = __dmul_rn(eta, c[3]);
    const double t2 = thr * thr;
    double* tail = o + rec - 8;
    tail[0] = c[0];
    tail[1] = c[1];
    tail[2] = c[2];
    tail[3] = thr;
    tail[4] = t2 * (1.0 - 1e-13);
    tail[5] = t2 * (1.0 + 1e-13);
  }
  int* m = reinterpret_cast<int*>(o + rec - 2);
  const int* em = ent_meta + 5 * e;
  m[0] = t < 0 ? 0 : t;
  m[1] = em[0];
  short* l = reinterpret_cast<short*>(m + 2);
  // byte offset of each corner's window column (local column mod window,
  // csrc/assemble.cu WSTRIDE doubles per column); the dump column (index
  // window) for dummy records
  for (int c = 0; c < 3; ++c) l[c] = (short)((em[1 + c] >= 0 ? em[1 + c] % window : window) * wstride * 8);
  l[3] = (short)em[4];
}

// K4: singular (corner) pairs.  One warp per row; the row's star panels are
// processed in triangle order (reference row_pass1 singular batch,
// src/assembly.py:202-235) and added to the row after the regular sweep.
// Duffy rule tables per corner: rule[c][m] = (u, v, w, pad).


__global__ void k_assemble_singular(SingularArgs a) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // rows_per_warp > 1 (charge-reduce mode): the rows of one 32-row tile add
  // into the tile's shared partial row, sequentially (deterministic order)
  for (int w = wg * a.rows_per_warp; w < min(a.n_rows, (wg + 1) * a.rows_per_warp); ++w) {
    const double* rd = a.rowdata + 6 * (size_t)w;
    const d3 X = mk3(rd[0], rd[1], rd[2]);
    const double nx = rd[3], ny = rd[4], nz = rd[5];
    const bool adl = a.row_kind[w] == 1;
    const int own = a.row_col[w];
    const double sc = a.row_scale[w];
    double* Arow = a.A + a.row_out[w];
    if (own < 0) continue;
    for (int s = a.vc_ptr[own]; s < a.vc_ptr[own + 1]; ++s) {
      const int t = a.vc_tri[s], c = a.vc_corner[s];
      const double* Xn = a.nodes6 + 18 * (size_t)t;
      const double* R = a.rule + (size_t)c * a.nm * 4;
      double s0 = 0, s1 = 0, s2 = 0;
      for (int m = lane; m < a.nm; m += 32) {
        double u = R[4 * m], v = R[4 * m + 1], wq = R[4 * m + 2];
        d3 p;
        double jac;
        curved_point(Xn, u, v, p, jac);
        double dx = X.x - p.x, dy = X.y - p.y, dz = X.z - p.z;
        double r = sqrt(dx * dx + dy * dy + dz * dz);
        double k = adl ? (dx * nx + dy * ny + dz * nz) / (r * r * r) : 1.0 / r;
        k *= wq * jac * kInv4Pi;
        s0 = fma(k, 1.0 - u - v, s0);
        s1 = fma(k, u, s1);
        s2 = fma(k, v, s2);
      }
      s0 = warp_sum(s0);
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        const int* tc = a.tri_cols + 3 * (size_t)t;
        Arow[a.col_dev[tc[0]]] += sc * s0;
        Arow[a.col_dev[tc[1]]] += sc * s1;
        Arow[a.col_dev[tc[2]]] += sc * s2;
      }
      __syncwarp();
    }
    if (lane == 0) Arow[a.col_dev[own]] += a.row_diag[w];
    __syncwarp();
  }
}

// K7 (charge / neutrality rows, reference charge_row src/assembly.py:540-569
// and _row_equation 441-468): out[c] (+)= sum over the partial rows p (in
// order) of part[p][c] -- the column sums of the charge-reduce sweep.
__global__ void k_charge_reduce(const double* part, int n_parts, int64_t part_ld, int n, double* out,
                                int accumulate) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double s = 0.0;
  for (int p = 0; p < n_parts; ++p) s += part[(size_t)p * part_ld + c];
  out[c] = accumulate ? out[c] + s : s;
}

// Columns n .. N-1 (floating potentials) of collocation rows: -1 in the
// row's own floating column, 0 elsewhere (reference src/assembly.py:425-426).
__global__ void k_fill_float_cols(double* A, const int64_t* row_out, const int* row_float, int n_rows,
                                  int n, int n_fl) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= (int64_t)n_rows * n_fl) return;
  int r = (int)(g / n_fl), k = (int)(g % n_fl);
  A[row_out[r] + n + k] = (row_float[r] == k) ? -1.0 : 0.0;
}

}  // namespace hvb

// ---------------------------------------------------------------------------
// launchers (called by hvb_api.cu)
// ---------------------------------------------------------------------------
namespace hvb {

cudaError_t launch_build_table(const double* nodes6, int nt, int nq, const double* rule, double* out,
                               cudaStream_t st) {
  int n = nt * nq;
  k_build_table<<<(n + 255) / 256, 256, 0, st>>>(nodes6, nt, nq, rule, out);
  return cudaGetLastError();
}

cudaError_t launch_panel_data(const double* cc, const double* radii, int nt, double eta, double* ccr, double* cls,
                              double* groups, cudaStream_t st) {
  if (nt == 0) return cudaSuccess;
  const int warps = (nt + 31) / 32;
  k_panel_data<<<(warps + 3) / 4, 128, 0, st>>>(cc, radii, nt, eta, ccr, cls, groups);
  return cudaGetLastError();
}

cudaError_t launch_build_stream(const double* table, int nq, const double* ccr, double eta,
                                const int* ent_tri, const int* ent_meta, int64_t ne, int mode, int window,
                                double* out, cudaStream_t st) {
  if (ne == 0) return cudaSuccess;
  const int rec = sweep_record_doubles(nq, mode);
  if (rec < 0) return cudaErrorInvalidValue;
  k_build_stream<<<(unsigned)((ne + 127) / 128), 128, 0, st>>>(table, nq, ccr, eta, ent_tri, ent_meta, ne, mode, rec,
                                                              window, sweep_window_stride(), out);
  return cudaGetLastError();
}

cudaError_t launch_charge_reduce(const double* part, int n_parts, int64_t part_ld, int n, double* out, int accumulate,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_charge_reduce<<<(n + 255) / 256, 256, 0, st>>>(part, n_parts, part_ld, n, out, accumulate);
  return cudaGetLastError();
}

cudaError_t launch_singular(const SingularArgs& a, cudaStream_t st) {
  if (a.n_rows == 0) return cudaSuccess;
  int threads = 128;
  const int items = (a.n_rows + a.rows_per_warp - 1) / a.rows_per_warp;
  int blocks = (items * 32 + threads - 1) / threads;
  k_assemble_singular<<<blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fill_float_cols(double* A, const int64_t* row_out, const int* row_float, int n_rows,
                                   int n, int n_fl, cudaStream_t st) {
  int64_t tot = (int64_t)n_rows * n_fl;
  if (tot == 0) return cudaSuccess;
  k_fill_float_cols<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, row_out, row_float, n_rows, n, n_fl);
  return cudaGetLastError();
}

}  // namespace hvb
