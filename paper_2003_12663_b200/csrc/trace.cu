// K12-K14: device-resident field-line tracer.
//
// Reference: trace_fieldline src/postprocess.py:244-357 (Dormand-Prince
// 5(4) on the unit tangent, step control, surface-hit arming / snapping,
// termination order), _surface_distance 198-218 (12 circumcircle
// candidates, flat closest point -> curved map), streamer_integral 365-374.
//
// Every line is a small state machine held in HBM (LineState).  The host
// drives rounds; in each round every live line consumes the result of its
// outstanding request and runs until it needs the next one:
//
//   k_trace_ctrl (mode E)  -- consume E at the line's last request point
//   k_surface_distance     -- for lines that asked for d_surf(x)
//   k_trace_ctrl (mode SD) -- consume d_surf, continue to the next E request
//   field eval (field.cu)  -- ONE batched N-body launch over all requests
//
// so the device sees (#live lines)-point N-body launches, one per round,
// and the host only reads four counters per round.  Requests are compacted
// with atomics (slot order is irrelevant: each target's field is computed
// independently of its slot, with a panel split fixed per mesh).
//
// Arithmetic follows the reference statement by statement (unfused
// products/sums where Python evaluates scalar/vector expressions, ddot FMA
// chains for np.linalg.norm of a 3-vector, OpenBLAS dgemv_n order for the
// b5 @ K / b4 @ K products).  The accepted point reuses the stage-6 field
// (x5 is within 1 ulp of the stage-6 point) instead of evaluating E(x5) a
// second time: 6 field evaluations per accepted step instead of the
// reference's 7.
#include "near.cuh"

namespace hvb {

namespace tr {

// Dormand-Prince tableau (reference src/postprocess.py:229-241), as Python
// evaluates the rational literals (correctly rounded quotients).
__constant__ double kA[7][6] = {
    {0, 0, 0, 0, 0, 0},
    {1.0 / 5, 0, 0, 0, 0, 0},
    {3.0 / 40, 9.0 / 40, 0, 0, 0, 0},
    {44.0 / 45, -56.0 / 15, 32.0 / 9, 0, 0, 0},
    {19372.0 / 6561, -25360.0 / 2187, 64448.0 / 6561, -212.0 / 729, 0, 0},
    {9017.0 / 3168, -355.0 / 33, 46732.0 / 5247, 49.0 / 176, -5103.0 / 18656, 0},
    {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84},
};
__constant__ double kB4[7] = {5179.0 / 57600, 0.0, 7571.0 / 16695, 393.0 / 640, -92097.0 / 339200, 187.0 / 2100,
                              1.0 / 40};
__constant__ double kB5[7] = {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84, 0.0};

// (b @ K)[d] for the (7,) coefficients and the 7 stage tangents, in the order
// numpy's vector @ (7,3) matrix takes through OpenBLAS dgemv_n (m = 3, n = 7):
// a 4-column block fma(b0,k0, b1 k1) + fma(b2,k2, b3 k3), then the remaining
// columns one FMA each (bitwise on random inputs in the reference container;
// the same kernel order as map_reference_blas below)
HVB_DEV double dgemv7(const double* b, const double (*k)[3], int d) {
  double t = __dadd_rn(__fma_rn(b[0], k[0][d], __dmul_rn(b[1], k[1][d])),
                       __fma_rn(b[2], k[2][d], __dmul_rn(b[3], k[3][d])));
  t = __fma_rn(b[4], k[4][d], t);
  t = __fma_rn(b[5], k[5][d], t);
  return __fma_rn(b[6], k[6][d], t);
}

HVB_DEV double norm3(const double* v) { return __dsqrt_rn(dot3_blas(mk3(v[0], v[1], v[2]), mk3(v[0], v[1], v[2]))); }

HVB_DEV void request_e(const TraceArgs& a, LineState& L, int line, const double* p, int phase) {
  L.phase = phase;
  L.req[0] = p[0];
  L.req[1] = p[1];
  L.req[2] = p[2];
  const unsigned long long slot = atomicAdd(&a.counters[0], 1ull);
  atomicAdd(&a.counters[3], 1ull);  // field evaluations, never reset
  L.slot = (int)slot;
  a.e_pts[3 * slot] = p[0];
  a.e_pts[3 * slot + 1] = p[1];
  a.e_pts[3 * slot + 2] = p[2];
  a.e_line[slot] = line;
}

HVB_DEV void request_sd(const TraceArgs& a, LineState& L, int line) {
  L.phase = kPhaseSD;
  const unsigned long long slot = atomicAdd(&a.counters[1], 1ull);
  L.slot = (int)slot;
  a.sd_pts[3 * slot] = L.x[0];
  a.sd_pts[3 * slot + 1] = L.x[1];
  a.sd_pts[3 * slot + 2] = L.x[2];
  a.sd_line[slot] = line;
}

HVB_DEV void finish(const TraceArgs& a, LineState& L, int term, int status) {
  L.term = term;
  L.status = status;
  L.phase = kPhaseDone;
}

HVB_DEV void append(const TraceArgs& a, LineState& L, int line, const double* x, double mag, double s) {
  const int k = L.npts;
  double* P = a.out_pts + ((size_t)line * a.cap + k) * 5;
  P[0] = x[0];
  P[1] = x[1];
  P[2] = x[2];
  P[3] = mag;
  P[4] = s;
  L.npts = k + 1;
  atomicMax(&a.counters[2], (unsigned long long)(k + 1));
}

// tangent of E: returns false if |E| <= floor or == 0 (reference tangent())
HVB_DEV bool tangent(const TraceArgs& a, const LineState& L, const double* e, double* t, double& mag) {
  mag = norm3(e);
  if (mag <= a.e_floor || mag == 0.0) return false;
  for (int d = 0; d < 3; ++d) t[d] = __ddiv_rn(__dmul_rn(L.sign, e[d]), mag);
  return true;
}

// h = clip(h * clip(factor, 0.2, 2), h_min, h_max) with the stored err/tol
HVB_DEV void step_size(const TraceArgs& a, LineState& L) {
  double factor = L.err > 0.0 ? __dmul_rn(0.9, pow(__ddiv_rn(L.tol, L.err), 0.2)) : 2.0;
  factor = fmin(fmax(factor, 0.2), 2.0);
  double h = __dmul_rn(L.h, factor);
  L.h = fmin(fmax(h, a.h_min), a.h_max);
}

HVB_DEV void stage_point(const LineState& L, int stage, double* xi) {
  double acc[3] = {0.0, 0.0, 0.0};
  for (int j = 0; j < stage; ++j)
    for (int d = 0; d < 3; ++d) acc[d] = __dadd_rn(acc[d], __dmul_rn(kA[stage][j], L.k[j][d]));
  for (int d = 0; d < 3; ++d) xi[d] = __dadd_rn(L.x[d], __dmul_rn(L.h, acc[d]));
}

// loop body after the surface distance of x is known (reference lines
// 283-318 up to the first stage request)
HVB_DEV void loop_body(const TraceArgs& a, LineState& L, int line) {
  const double hit_tol = __dmul_rn(a.tol_frac, L.local_r);
  if (L.d_surf > __dmul_rn(2.0, hit_tol)) L.armed = 1;
  if (L.armed && L.d_surf < hit_tol) {
    double xe[3];
    for (int d = 0; d < 3; ++d) xe[d] = __dadd_rn(L.x[d], __dmul_rn(L.k[0][d], L.d_surf));
    double* P = a.out_pts + ((size_t)line * a.cap + (L.npts - 1)) * 5;
    P[0] = xe[0];
    P[1] = xe[1];
    P[2] = xe[2];
    P[4] = __dadd_rn(P[4], L.d_surf);
    L.term = kSurfaceHit;
    request_e(a, L, line, xe, kPhaseSnap);
    return;
  }
  if (L.s >= a.l_max) {
    finish(a, L, kMaxLength, kStatusDone);
    return;
  }
  for (int d = 0; d < 3; ++d) {
    if (fabs(__dsub_rn(L.x[d], a.center[d])) > a.half[d]) {
      finish(a, L, kLeftDomain, kStatusDone);
      return;
    }
  }
  if (a.max_steps > 0 && L.steps >= a.max_steps) {  // extension: bounded step budget
    finish(a, L, kMaxSteps, kStatusDone);
    return;
  }
  L.steps += 1;
  const double h_cap = L.d_surf > __dmul_rn(4.0, a.h_max) ? a.h_max : fmax(a.h_min, __dmul_rn(0.45, L.d_surf));
  L.h = fmin(fmin(L.h, h_cap), __dadd_rn(__dsub_rn(a.l_max, L.s), a.h_min));
  double xi[3];
  stage_point(L, 1, xi);
  L.stage = 1;
  request_e(a, L, line, xi, kPhaseStage);
}

}  // namespace tr

// mode 0: init (request E at the start point); 1: consume E; 2: consume SD
__global__ void k_trace_ctrl(TraceArgs a, int mode) {
  using namespace tr;
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= a.n_lines) return;
  LineState L = a.state[line];
  if (mode == 0) {
    L.x[0] = a.starts[3 * (size_t)line];
    L.x[1] = a.starts[3 * (size_t)line + 1];
    L.x[2] = a.starts[3 * (size_t)line + 2];
    L.sign = a.orient[line] >= 0 ? 1.0 : -1.0;
    L.npts = 0;
    L.armed = 0;
    L.term = kMaxLength;
    L.status = kStatusRunning;
    L.s = 0.0;
    L.h = a.h_max;
    L.steps = 0;
    request_e(a, L, line, L.x, kPhaseStart);
    a.state[line] = L;
    return;
  }
  if (L.phase == kPhaseDone) return;
  if (mode == 2) {
    if (L.phase != kPhaseSD) return;
    L.d_surf = a.sd_out[2 * L.slot];
    L.local_r = a.sd_out[2 * L.slot + 1];
    loop_body(a, L, line);
    a.state[line] = L;
    return;
  }
  if (L.phase == kPhaseSD) return;
  // consume E at the outstanding request
  double e[3] = {a.e_out[3 * (size_t)L.slot], a.e_out[3 * (size_t)L.slot + 1], a.e_out[3 * (size_t)L.slot + 2]};
  const bool coincident = a.e_flag[L.slot] != 0;
  double t[3], mag;
  switch (L.phase) {
    case kPhaseStart: {
      if (coincident) {
        finish(a, L, kMaxLength, kStatusCoincident);
        break;
      }
      if (!tangent(a, L, e, t, mag)) {
        L.d_surf = mag;  // reported in the TraceError message
        finish(a, L, kWeakField, kStatusWeakStart);
        break;
      }
      append(a, L, line, L.x, mag, 0.0);
      for (int d = 0; d < 3; ++d) L.k[0][d] = t[d];
      request_sd(a, L, line);
      break;
    }
    case kPhaseStage: {
      if (coincident) {
        finish(a, L, L.term, kStatusCoincident);
        break;
      }
      if (!tangent(a, L, e, t, mag)) {
        finish(a, L, kWeakField, kStatusDone);
        break;
      }
      const int j = L.stage;
      for (int d = 0; d < 3; ++d) L.k[j][d] = t[d];
      if (j < 6) {
        double xi[3];
        L.stage = j + 1;
        stage_point(L, j + 1, xi);
        request_e(a, L, line, xi, kPhaseStage);
        break;
      }
      // x5 = x + h (b5 @ K), x4 = x + h (b4 @ K) in the reference's order
      // (numpy vector @ matrix = OpenBLAS dgemv_n over m = 3, n = 7, measured
      // bitwise in the reference container: dgemv7).  x5 is within 1 ulp of
      // the stage-6 point (same coefficients, Python's sum order), so E(x5)
      // -- which the reference evaluates again after accepting
      // (src/postprocess.py:323) -- is taken from the stage-6 result.
      double x5[3], x4[3], df[3];
      for (int d = 0; d < 3; ++d) {
        x5[d] = __dadd_rn(L.x[d], __dmul_rn(L.h, dgemv7(kB5, L.k, d)));
        x4[d] = __dadd_rn(L.x[d], __dmul_rn(L.h, dgemv7(kB4, L.k, d)));
        df[d] = __dsub_rn(x5[d], x4[d]);
      }
      const double err = norm3(df);
      const double tol = __dmul_rn(__dmul_rn(a.rel_tol, fmax(1.0, __ddiv_rn(norm3(x5), a.diag))), a.diag);
      L.err = err;
      L.tol = tol;
      if (err <= tol || L.h <= __dmul_rn(a.h_min, 1.0000001)) {
        // accept: the tangent at x5 is k7 (non-weak, checked above)
        for (int d = 0; d < 3; ++d) L.x[d] = x5[d];
        L.s = __dadd_rn(L.s, L.h);
        append(a, L, line, L.x, mag, L.s);
        for (int d = 0; d < 3; ++d) L.k[0][d] = L.k[6][d];
        step_size(a, L);
        request_sd(a, L, line);
        break;
      }
      step_size(a, L);
      loop_body(a, L, line);  // x unchanged: the cached surface distance holds
      break;
    }
    case kPhaseSnap: {
      if (!coincident) a.out_pts[((size_t)line * a.cap + (L.npts - 1)) * 5 + 3] = norm3(e);
      finish(a, L, kSurfaceHit, kStatusDone);
      break;
    }
    default:
      break;
  }
  a.state[line] = L;
}

// ---------------------------------------------------------------------------
// K12: surface distance.  One CTA per query point: every thread keeps the 12
// smallest circumcircle lower bounds ||x-cc|| - R of its strided panel
// subset (ties by panel index), the CTA merges them, and 12 threads run the
// flat closest point -> curved map -> distance; first minimum wins.
// ---------------------------------------------------------------------------
// map_reference (src/mesh.py:161-165): n @ nodes for one (u, v) -- NumPy
// routes the (1,6)@(6,3) product to OpenBLAS dgemv_n, whose m=3 path sums
// fma(n0,x0, n1*x1) + fma(n2,x2, n3*x3), then fma n4, n5 (measured in the
// reference container: bitwise on 2e4 random cases).  Shape functions as
// shape_functions (src/mesh.py:124-137).
HVB_DEV d3 map_reference_blas(const double* __restrict__ X, double u, double v) {
  const double l0 = __dsub_rn(__dsub_rn(1.0, u), v);
  double n[6];
  n[0] = __dmul_rn(l0, __dsub_rn(__dmul_rn(2.0, l0), 1.0));
  n[1] = __dmul_rn(u, __dsub_rn(__dmul_rn(2.0, u), 1.0));
  n[2] = __dmul_rn(v, __dsub_rn(__dmul_rn(2.0, v), 1.0));
  n[3] = __dmul_rn(__dmul_rn(4.0, l0), u);
  n[4] = __dmul_rn(__dmul_rn(4.0, u), v);
  n[5] = __dmul_rn(__dmul_rn(4.0, v), l0);
  double p[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double t = __dadd_rn(__fma_rn(n[0], X[d], __dmul_rn(n[1], X[3 + d])),
                         __fma_rn(n[2], X[6 + d], __dmul_rn(n[3], X[9 + d])));
    t = __fma_rn(n[4], X[12 + d], t);
    p[d] = __fma_rn(n[5], X[15 + d], t);
  }
  return mk3(p[0], p[1], p[2]);
}

constexpr int SD_THREADS = 256;
constexpr int SD_K = 12;

// m_dev != nullptr: the query count is read on the device (tracer rounds)
// Threads take whole aligned 32-panel groups; a group whose lower bound
// ||x - C|| - rho_sd (device.py panel_groups, with a 1e-12 relative margin)
// is not below the thread's current 12th key cannot insert and is skipped.
// The top-12 set is (key, index) ordered, so it does not depend on the
// visiting order.
__global__ void __launch_bounds__(SD_THREADS) k_surface_distance(const double* __restrict__ pts, int m_host,
                                                                 const unsigned long long* m_dev,
                                                                 const double* __restrict__ ccr,
                                                                 const double* __restrict__ groups, int nt,
                                                                 const double* __restrict__ nodes6,
                                                                 double* __restrict__ out) {
  __shared__ double s_key[SD_THREADS * SD_K];
  __shared__ int s_idx[SD_THREADS * SD_K];
  __shared__ double s_d[SD_K];
  __shared__ int s_t[SD_K];
  const int m = m_dev ? (int)*m_dev : m_host;
  for (int q = blockIdx.x; q < m; q += gridDim.x) {
  __syncthreads();
  const int tid = threadIdx.x;
  const d3 X = mk3(pts[3 * (size_t)q], pts[3 * (size_t)q + 1], pts[3 * (size_t)q + 2]);
  double key[SD_K];
  int idx[SD_K];
#pragma unroll
  for (int k = 0; k < SD_K; ++k) {
    key[k] = INFINITY;
    idx[k] = 0x7fffffff;
  }
  const int ng = (nt + 31) / 32;
  // pass 1: T0 = min over full groups of ||x - C|| + rho_sd bounds the 12th
  // smallest key from above (each such group holds 32 >= 12 panels whose
  // keys are all <= it), so groups with ||x - C|| - rho_sd >= T0 (+ margin)
  // cannot hold a top-12 panel
  double t0 = INFINITY;
  for (int g = tid; g < ng; g += SD_THREADS) {
    if (32 * g + 32 > nt) continue;
    const double* gb = groups + 8 * (size_t)g;
    const double gd = __dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(gb[0], gb[1], gb[2]))));
    t0 = fmin(t0, (gd + gb[4]) * (1.0 + 1e-12));
  }
  s_key[tid] = t0;
  __syncthreads();
  for (int w = SD_THREADS / 2; w > 0; w >>= 1) {
    if (tid < w) s_key[tid] = fmin(s_key[tid], s_key[tid + w]);
    __syncthreads();
  }
  t0 = s_key[0];
  __syncthreads();
  for (int g = tid; g < ng; g += SD_THREADS) {
    const double* gb = groups + 8 * (size_t)g;
    const double gd = __dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(gb[0], gb[1], gb[2]))));
    const double glo = gd - gb[4] - 1e-12 * (gd + gb[4]);
    if (glo >= key[SD_K - 1] || glo > t0) continue;
    const int tend = min(nt, 32 * g + 32);
  for (int t = 32 * g; t < tend; ++t) {
    const double* c = ccr + 4 * (size_t)t;
    const double lower = __dsub_rn(__dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(c[0], c[1], c[2])))), c[3]);
    if (lower < key[SD_K - 1]) {  // t increases: ties keep the earlier panel
      double kv = lower;
      int iv = t;
#pragma unroll
      for (int k = 0; k < SD_K; ++k) {
        const bool sw = kv < key[k];
        const double tk = key[k];
        const int ti = idx[k];
        key[k] = sw ? kv : tk;
        idx[k] = sw ? iv : ti;
        kv = sw ? tk : kv;
        iv = sw ? ti : iv;
      }
    }
  }
  }  // groups
#pragma unroll
  for (int k = 0; k < SD_K; ++k) {
    s_key[tid * SD_K + k] = key[k];
    s_idx[tid * SD_K + k] = idx[k];
  }
  __syncthreads();
  // tree merge of the sorted per-thread lists: (key, index) lexicographic
  for (int width = 1; width < SD_THREADS; width <<= 1) {
    if ((tid % (2 * width)) == 0 && tid + width < SD_THREADS) {
      const int A = tid * SD_K, B = (tid + width) * SD_K;
      double mk[SD_K];
      int mi[SD_K];
      int ia = 0, ib = 0;
#pragma unroll
      for (int k = 0; k < SD_K; ++k) {
        const double ka = s_key[A + ia], kb = s_key[B + ib];
        const int xa = s_idx[A + ia], xb = s_idx[B + ib];
        const bool takeA = (ka < kb) || (ka == kb && xa <= xb);
        mk[k] = takeA ? ka : kb;
        mi[k] = takeA ? xa : xb;
        ia += takeA;
        ib += !takeA;
      }
#pragma unroll
      for (int k = 0; k < SD_K; ++k) {
        s_key[A + k] = mk[k];
        s_idx[A + k] = mi[k];
      }
    }
    __syncthreads();
  }
  if (tid < SD_K) {
    const int t = s_idx[tid];
    double d = INFINITY;
    if (t < nt) {
      const double* Xn = nodes6 + 18 * (size_t)t;
      double u, v;
      closest_point_flat(X, mk3(Xn[0], Xn[1], Xn[2]), mk3(Xn[3], Xn[4], Xn[5]), mk3(Xn[6], Xn[7], Xn[8]), u, v);
      const d3 df = sub_rn(X, map_reference_blas(Xn, u, v));
      d = __dsqrt_rn(dot3_blas(df, df));
    }
    s_d[tid] = d;
    s_t[tid] = t;
  }
  __syncthreads();
  if (tid == 0) {
    double best = INFINITY;
    int bt = s_t[0];
    for (int k = 0; k < SD_K; ++k) {
      if (s_d[k] < best) {
        best = s_d[k];
        bt = s_t[k];
      }
    }
    out[2 * (size_t)q] = best;
    out[2 * (size_t)q + 1] = bt < nt ? ccr[4 * (size_t)bt + 3] : 0.0;
  }
  }  // queries
}

// near-pair vertex coincidence: flag targets within `prox` of a node of a
// near panel (every mesh node belongs to a panel, and a point that close to
// a node classifies that panel as non-regular)
__global__ void k_near_coincide(const int* pairs, long long n_pairs, const double* pts, const double* nodes6,
                                double prox, int* flag) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int i = pairs[2 * p], t = pairs[2 * p + 1];
  const d3 X = mk3(pts[3 * (size_t)i], pts[3 * (size_t)i + 1], pts[3 * (size_t)i + 2]);
  const double* Xn = nodes6 + 18 * (size_t)t;
  for (int k = 0; k < 6; ++k) {
    const double d = __dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(Xn[3 * k], Xn[3 * k + 1], Xn[3 * k + 2]))));
    if (d < prox) flag[i] = 1;
  }
}

// K14: streamer integral per line: trapezoid of alpha(|E|) (np.interp,
// constant beyond the table ends) over the arc lengths; verdict value > K.
__global__ void k_streamer(const double* out_pts, const LineState* state, int n_lines, int cap, const double* e_tab,
                           const double* a_tab, int n_tab, double k_str, double* value, int* verdict) {
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= n_lines) return;
  const int np = state[line].npts;
  const double* P = out_pts + (size_t)line * cap * 5;
  auto alpha = [&](double e) {
    if (e <= e_tab[0]) return a_tab[0];
    if (e >= e_tab[n_tab - 1]) return a_tab[n_tab - 1];
    int lo = 0, hi = n_tab - 1;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (e_tab[mid] <= e) lo = mid; else hi = mid;
    }
    if (e == e_tab[lo]) return a_tab[lo];
    const double slope = __ddiv_rn(__dsub_rn(a_tab[lo + 1], a_tab[lo]), __dsub_rn(e_tab[lo + 1], e_tab[lo]));
    return __dadd_rn(__dmul_rn(slope, __dsub_rn(e, e_tab[lo])), a_tab[lo]);
  };
  double sum = 0.0;
  double a0 = np > 0 ? alpha(P[3]) : 0.0;
  for (int k = 1; k < np; ++k) {
    const double a1 = alpha(P[5 * k + 3]);
    sum = __dadd_rn(sum, __dmul_rn(__dmul_rn(0.5, __dadd_rn(a1, a0)), __dsub_rn(P[5 * k + 4], P[5 * (k - 1) + 4])));
    a0 = a1;
  }
  value[line] = sum;
  verdict[line] = sum > k_str ? 1 : 0;
}

__global__ void k_trace_summary(const LineState* state, int n_lines, int* info, double* dinfo) {
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= n_lines) return;
  const LineState& L = state[line];
  info[4 * line] = L.npts;
  info[4 * line + 1] = L.term;
  info[4 * line + 2] = L.status;
  info[4 * line + 3] = L.phase;
  dinfo[line] = L.d_surf;
}

cudaError_t launch_trace_summary(const LineState* state, int n_lines, int* info, double* dinfo, cudaStream_t st) {
  if (n_lines == 0) return cudaSuccess;
  k_trace_summary<<<(n_lines + 127) / 128, 128, 0, st>>>(state, n_lines, info, dinfo);
  return cudaGetLastError();
}

// Near pass of one tracer round, without a host-side pair list: the field
// kernel flags each (panel chunk, target) holding a non-regular panel; one
// warp per target rescans only the flagged chunks, in chunk then panel
// order, clearing the flags as it goes.  Every non-regular panel gets the
// vertex-coincidence check and its composite-rule field, added to the
// target in panel order -- the same order and arithmetic as the sorted-pair
// path (k_near_pairs + k_near_apply_points), so results are bitwise those
// of eval_efield_batch.
__global__ void k_trace_near(const unsigned long long* m_dev, int split, const double* __restrict__ pts,
                             int* __restrict__ has_near, const double* __restrict__ cls,
                             const double* __restrict__ nodes6, const double* __restrict__ radii,
                             const int* __restrict__ tri_cols, int nt, const double* __restrict__ u,
                             const double* duffy, int n_duffy, const double* graded, int n_graded, int bisect_depth,
                             double bisect_trigger, double prox, double* __restrict__ E, int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int m = (int)*m_dev;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m; i += warps) {
    const d3 X = mk3(pts[3 * (size_t)i], pts[3 * (size_t)i + 1], pts[3 * (size_t)i + 2]);
    double e0 = 0.0, e1 = 0.0, e2 = 0.0;
    bool any = false, coinc = false;
    for (int cb = 0; cb < split; cb += 32) {
      const int cc = cb + lane;
      int* fp = has_near + (size_t)cc * m + i;
      const bool fl = cc < split && *fp;
      if (fl) *fp = 0;
      unsigned cm = __ballot_sync(0xffffffffu, fl);
      while (cm) {
        const int chunk = cb + __ffs(cm) - 1;
        cm &= cm - 1;
        if (!any) {
          any = true;
          e0 = E[3 * (size_t)i];
          e1 = E[3 * (size_t)i + 1];
          e2 = E[3 * (size_t)i + 2];
        }
        const int ngr = (nt + 31) / 32;  // chunk bounds as in field.cu field_tile
        const int tb = min(nt, 32 * (int)((long long)ngr * chunk / split));
        const int te = min(nt, 32 * (int)((long long)ngr * (chunk + 1) / split));
        for (int t0 = tb; t0 < te; t0 += 32) {
          const int t = t0 + lane;
          bool nr = false;
          if (t < te) {
            const double* c = cls + 6 * (size_t)t;
            nr = !is_regular(X, mk3(c[0], c[1], c[2]), c[3], c[4], c[5]);
          }
          unsigned msk = __ballot_sync(0xffffffffu, nr);
          while (msk) {
            const int tn = t0 + __ffs(msk) - 1;
            msk &= msk - 1;
            const double* Xn = nodes6 + 18 * (size_t)tn;
            if (lane < 6) {
              const double d =
                  __dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(Xn[3 * lane], Xn[3 * lane + 1], Xn[3 * lane + 2]))));
              if (d < prox) coinc = true;
            }
            double acc[9];
            near_pair_acc(X, mk3(0.0, 0.0, 0.0), 2, Xn, radii[tn], duffy, n_duffy, graded, n_graded, bisect_depth,
                          bisect_trigger, acc);
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[k] = warp_sum(acc[k]);
            const int* tc = tri_cols + 3 * (size_t)tn;
            const double u0 = u[tc[0]], u1 = u[tc[1]], u2 = u[tc[2]];
            e0 = __dadd_rn(e0, __fma_rn(u2, acc[6], __fma_rn(u1, acc[3], __dmul_rn(u0, acc[0]))));
            e1 = __dadd_rn(e1, __fma_rn(u2, acc[7], __fma_rn(u1, acc[4], __dmul_rn(u0, acc[1]))));
            e2 = __dadd_rn(e2, __fma_rn(u2, acc[8], __fma_rn(u1, acc[5], __dmul_rn(u0, acc[2]))));
          }
        }
      }
    }
    coinc = __any_sync(0xffffffffu, coinc);
    if (lane == 0 && any) {
      E[3 * (size_t)i] = e0;
      E[3 * (size_t)i + 1] = e1;
      E[3 * (size_t)i + 2] = e2;
      if (coinc) flag[i] = 1;
    }
  }
}

__global__ void k_trace_reset_flags(int* flag, int n, unsigned long long* counters) {
  if (blockIdx.x == 0 && threadIdx.x == 0) counters[4] = 0;  // N-body work counter
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) flag[k] = 0;
}

__global__ void k_trace_reset_counters(unsigned long long* counters) {
  if (threadIdx.x < 2) counters[threadIdx.x] = 0;
}

// One tracer round, entirely on the stream (no host synchronisation):
// clear flags -> field of the current request list (count = counters[0])
// -> near pass -> clear counters -> ctrl(consume E) -> surface distances
// (count = counters[1]) -> ctrl(consume SD).  New E requests land in the
// other list (r.ctrl.e_pts / e_line).
cudaError_t launch_trace_round(const TraceRoundArgs& r, cudaStream_t st) {
  const int L = r.ctrl.n_lines;
  if (L == 0) return cudaSuccess;
  cudaError_t e;
  FieldArgs f = r.field;
  int* flag = const_cast<int*>(r.ctrl.e_flag);
  k_trace_reset_flags<<<min((L + 255) / 256, 148 * 4), 256, 0, st>>>(flag, L, r.ctrl.counters);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_field_dyn(f, r.ctrl.counters, 148 * 16, st)) != cudaSuccess) return e;
  k_trace_near<<<148 * 8, 128, 0, st>>>(r.ctrl.counters, f.split, f.pts, f.has_near, f.cls, r.nodes6, r.radii, f.tri_cols,
                                        f.nt, r.u, r.duffy, r.n_duffy, r.graded, r.n_graded, r.bisect_depth,
                                        r.bisect_trigger, r.prox, f.out, flag);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_trace_reset_counters<<<1, 32, 0, st>>>(r.ctrl.counters);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_trace_ctrl(r.ctrl, 1, st)) != cudaSuccess) return e;
  k_surface_distance<<<148 * 8, SD_THREADS, 0, st>>>(r.ctrl.sd_pts, 0, r.ctrl.counters + 1, r.ccr, f.groups, f.nt,
                                                      r.nodes6,
                                                      const_cast<double*>(r.ctrl.sd_out));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return launch_trace_ctrl(r.ctrl, 2, st);
}

cudaError_t launch_trace_ctrl(const TraceArgs& a, int mode, cudaStream_t st) {
  if (a.n_lines == 0) return cudaSuccess;
  k_trace_ctrl<<<(a.n_lines + 127) / 128, 128, 0, st>>>(a, mode);
  return cudaGetLastError();
}

cudaError_t launch_surface_distance(const double* pts, int m, const double* ccr, const double* groups, int nt,
                                    const double* nodes6, double* out, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  k_surface_distance<<<min(m, 148 * 8), SD_THREADS, 0, st>>>(pts, m, nullptr, ccr, groups, nt, nodes6, out);
  return cudaGetLastError();
}

cudaError_t launch_near_coincide(const int* pairs, long long n_pairs, const double* pts, const double* nodes6,
                                 double prox, int* flag, cudaStream_t st) {
  if (n_pairs == 0) return cudaSuccess;
  k_near_coincide<<<(unsigned)((n_pairs + 255) / 256), 256, 0, st>>>(pairs, n_pairs, pts, nodes6, prox, flag);
  return cudaGetLastError();
}

cudaError_t launch_streamer(const double* out_pts, const LineState* state, int n_lines, int cap, const double* e_tab,
                            const double* a_tab, int n_tab, double k_str, double* value, int* verdict,
                            cudaStream_t st) {
  if (n_lines == 0) return cudaSuccess;
  k_streamer<<<(n_lines + 127) / 128, 128, 0, st>>>(out_pts, state, n_lines, cap, e_tab, a_tab, n_tab, k_str, value,
                                                    verdict);
  return cudaGetLastError();
}

}  // namespace hvb
