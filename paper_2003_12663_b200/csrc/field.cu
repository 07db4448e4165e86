// K10/K11: potential and field of the solved density at arbitrary points.
//
// Reference: eval_potential / eval_efield src/postprocess.py:112-133 build a
// full (n,) or (n,3) kernel row and contract it with u; surface field
// 141-170 adds the singular Duffy part and the jump term.  Here the density
// is contracted once per solution into point sources q_tq = sum_c
// u_col(t,c) * jw_tq * hat_c(q) / (4 pi) (k_contract), and each target runs
// an N-body sum over the regular panels (classified exactly like the
// assembly rows), deferring near-singular panels to near.cu and singular
// (own-vertex) panels to k_field_singular.  Targets are split over CTAs, the
// panel range over grid.y; partial sums are reduced in a fixed order.
#include "launch.cuh"

namespace hvb {

// q_tq from the sample table and u (original collocation order)
__global__ void k_contract(const double* __restrict__ table, int nt, int nq, const int* __restrict__ tri_cols,
                           const double* __restrict__ u, double* __restrict__ src) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nt * nq) return;
  int t = g / nq;
  const double* o = table + 6 * (size_t)g;
  const int* tc = tri_cols + 3 * (size_t)t;
  double q = o[3] * u[tc[0]] + o[4] * u[tc[1]] + o[5] * u[tc[2]];
  double* s = src + 4 * (size_t)g;
  s[0] = o[0];
  s[1] = o[1];
  s[2] = o[2];
  s[3] = q;
}



constexpr int FT = 256;   // targets per CTA
constexpr int FCH = 32;   // panels per shared-memory chunk

// Field of one FCH-panel chunk [c0, c0+cn) at the thread's target X: the
// chunk's regular panels summed in panel order into (sx, sy, sz) starting
// from zero, non-regular (near) panels flagged / emitted.  src / cls / cols
// point at the chunk's panel data (shared memory, or global memory in the
// chunk-parallel mode).  POT: 0 = E (the tracer), 1 = potential, 2 = E at
// points; E uses the first-order r^-3 (rinv3_fast, ~4e-13 relative: the
// tracer's step decisions compare err against tol, and a flip needs err/tol
// within ~1e-12 of 1 -- the second-order form, 1 op more, gave the same
// 1,353,839 evaluations on the cfg5 8,192-line trace, 6 % slower).
template <int NQ, int POT>
HVB_DEV void chunk_sum(const FieldArgs& a, d3 X, int own, bool live, int ti, int c0, int cn,
                       const double2* __restrict__ src, const double* __restrict__ cls, const int* __restrict__ cols,
                       double& sx, double& sy, double& sz, bool& any_near) {
  const int lane = threadIdx.x & 31;
  sx = sy = sz = 0.0;
  // whole group far from the target: every panel is regular (exactly;
  // device.py panel_groups) -- skip the per-panel classification
  const double* gb = a.groups + 8 * (size_t)(c0 / FCH);
  const double gd = __dsqrt_rn(sumsq_unfused(sub_rn(X, mk3(gb[0], gb[1], gb[2]))));
  const bool far = gd > gb[3] * (1.0 + 1e-12);
  for (int j = 0; j < cn; ++j) {
    const double* c = cls + 6 * j;
    const bool reg = far || is_regular(X, mk3(c[0], c[1], c[2]), c[3], c[4], c[5]);
    double fx = 0.0, fy = 0.0, fz = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double2 p01 = src[(j * NQ + q) * 2];
      const double2 p2q = src[(j * NQ + q) * 2 + 1];
      const double dx = X.x - p01.x, dy = X.y - p01.y, dz = X.z - p2q.x;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      if (POT == 1) {
        fx = fma(p2q.y, rsqrt_full(r2), fx);
      } else {
        const double s = p2q.y * rinv3_fast(r2);
        fx = fma(s, dx, fx);
        fy = fma(s, dy, fy);
        fz = fma(s, dz, fz);
      }
    }
    if (reg) {
      sx += fx;
      sy += fy;
      sz += fz;
    }
    bool emit = false;
    if (!reg && live) {
      const int* tc = cols + 3 * j;
      emit = !(own >= 0 && (tc[0] == own || tc[1] == own || tc[2] == own));
    }
    if (a.near_list == nullptr) {
      any_near |= emit;
      continue;
    }
    const unsigned msk = __ballot_sync(0xffffffffu, emit);
    if (msk) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(a.near_count, (unsigned long long)__popc(msk));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (emit) {
        long long slot = (long long)b + __popc(msk & ((1u << lane) - 1u));
        if (slot < a.near_cap) {
          a.near_list[2 * slot] = ti;
          a.near_list[2 * slot + 1] = c0 + j;
        }
      }
    }
  }
}

// One (target block bx, panel split by) tile of the N-body sum.  Called by
// every thread of the CTA (it synchronises).  near_list == nullptr: instead
// of emitting (target, panel) near pairs, set has_near[target] = 1.  A
// target's split partial is the sum of its chunk sums in chunk order (the
// same in the chunk-parallel mode below, so results never depend on the
// batch).
template <int NQ, int POT>
HVB_DEV void field_tile(const FieldArgs& a, int bx, int by, double2* s_src, double* s_cls, int* s_cols) {
  const int tid = threadIdx.x;
  const int ti = bx * FT + tid;
  const bool live = ti < a.m;
  const bool warp_live = bx * FT + (tid & ~31) < a.m;
  const int tt = live ? ti : a.m - 1;
  const d3 X = mk3(a.pts[3 * (size_t)tt], a.pts[3 * (size_t)tt + 1], a.pts[3 * (size_t)tt + 2]);
  const int own = a.own_col ? a.own_col[tt] : -1;
  // split boundaries on FCH-panel group boundaries (group bounds, below)
  const int ng = (a.nt + FCH - 1) / FCH;
  const int tb = min(a.nt, FCH * (int)((long long)ng * by / a.split));
  const int te = min(a.nt, FCH * (int)((long long)ng * (by + 1) / a.split));
  double ex = 0.0, ey = 0.0, ez = 0.0;
  bool any_near = false;
  for (int c0 = tb; c0 < te; c0 += FCH) {
    const int cn = min(FCH, te - c0);
    __syncthreads();
    const double2* gs = reinterpret_cast<const double2*>(a.src + (size_t)c0 * NQ * 4);
    for (int k = tid; k < cn * NQ * 2; k += FT) s_src[k] = gs[k];
    for (int k = tid; k < cn * 6; k += FT) s_cls[k] = a.cls[(size_t)c0 * 6 + k];
    for (int k = tid; k < cn * 3; k += FT) s_cols[k] = a.tri_cols[(size_t)c0 * 3 + k];
    __syncthreads();
    // a warp whose 32 targets are all past the count only helps stage the
    // chunk (the tracer's tail rounds have a handful of live targets per CTA)
    if (!warp_live) continue;
    double sx, sy, sz;
    chunk_sum<NQ, POT>(a, X, own, live, ti, c0, cn, s_src, s_cls, s_cols, sx, sy, sz, any_near);
    ex += sx;
    ey += sy;
    ez += sz;
  }
  if (live) {
    double* o = a.part + ((size_t)by * a.m + ti) * 4;
    o[0] = ex;
    o[1] = ey;
    o[2] = ez;
    o[3] = 0.0;
    if (any_near) a.has_near[(size_t)by * a.m + ti] = 1;  // (split, m) chunk flags
  }
}

// Chunk-parallel tile for a block with at most 32 live targets (the
// tracer's tail rounds): warp w takes chunks w, w + 8, ... of the split for
// warp 0's targets, reading the panel data straight from global memory
// (every lane loads the same node: broadcast), and warp 0 adds the chunk
// sums in chunk order -- bitwise field_tile's result, ~8x lower latency.
constexpr int MAXCH = 16;  // chunks per split held in shared memory
template <int NQ>
HVB_DEV void field_tile_small(const FieldArgs& a, int bx, int by, double* s_part, int* s_near) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int ti = bx * FT + lane;
  const bool live = ti < a.m;
  const int tt = live ? ti : a.m - 1;
  const d3 X = mk3(a.pts[3 * (size_t)tt], a.pts[3 * (size_t)tt + 1], a.pts[3 * (size_t)tt + 2]);
  const int own = a.own_col ? a.own_col[tt] : -1;
  const int ng = (a.nt + FCH - 1) / FCH;
  const int tb = min(a.nt, FCH * (int)((long long)ng * by / a.split));
  const int te = min(a.nt, FCH * (int)((long long)ng * (by + 1) / a.split));
  const int nch = (te - tb + FCH - 1) / FCH;
  __syncthreads();  // s_part / s_near of the previous item are consumed
  for (int c = w; c < nch; c += FT / 32) {
    const int c0 = tb + c * FCH;
    const int cn = min(FCH, te - c0);
    double sx, sy, sz;
    bool nf = false;
    chunk_sum<NQ, 0>(a, X, own, live, ti, c0, cn, reinterpret_cast<const double2*>(a.src + (size_t)c0 * NQ * 4),
                     a.cls + (size_t)c0 * 6, a.tri_cols + (size_t)c0 * 3, sx, sy, sz, nf);
    double* o = s_part + (c * 32 + lane) * 3;
    o[0] = sx;
    o[1] = sy;
    o[2] = sz;
    s_near[c * 32 + lane] = nf;
  }
  __syncthreads();
  if (w == 0 && live) {
    double ex = 0.0, ey = 0.0, ez = 0.0;
    bool any_near = false;
    for (int c = 0; c < nch; ++c) {
      const double* o = s_part + (c * 32 + lane) * 3;
      ex += o[0];
      ey += o[1];
      ez += o[2];
      any_near |= s_near[c * 32 + lane] != 0;
    }
    double* o = a.part + ((size_t)by * a.m + ti) * 4;
    o[0] = ex;
    o[1] = ey;
    o[2] = ez;
    o[3] = 0.0;
    if (any_near) a.has_near[(size_t)by * a.m + ti] = 1;
  }
}

// 4 CTAs per SM (64 registers, an 8-byte spill): 1e5 points 249 -> 242 ms
template <int NQ, int POT>
__global__ void __launch_bounds__(FT, 4) k_field(FieldArgs a) {
  __shared__ double2 s_src[FCH * NQ * 2];
  __shared__ double s_cls[FCH * 6];
  __shared__ int s_cols[FCH * 3];
  field_tile<NQ, POT>(a, blockIdx.x, blockIdx.y, s_src, s_cls, s_cols);
}

// Same tiles, target count read on the device (*m_dev) and a grid-stride
// loop over (target block, split) items: launchable without knowing the
// count on the host (the tracer's sync-free rounds).  part is (split, m, 4)
// with the row stride of the CURRENT count.
// Items are handed out through an atomic work counter (m_dev[4], zeroed
// before the launch), so every SM stays busy until the last item whatever
// the count -- the per-target sums do not depend on which CTA runs them.
template <int NQ>
__global__ void __launch_bounds__(FT, 4) k_field_dyn(FieldArgs a, unsigned long long* m_dev) {
  __shared__ double2 s_src[FCH * NQ * 2];
  __shared__ double s_cls[FCH * 6];
  __shared__ int s_cols[FCH * 3];
  __shared__ double s_part[MAXCH * 32 * 3];
  __shared__ int s_near[MAXCH * 32];
  __shared__ long long s_item;
  a.m = (int)m_dev[0];
  const int nb = (a.m + FT - 1) / FT;
  const long long items = (long long)nb * a.split;
  const int ng = (a.nt + FCH - 1) / FCH;
  const bool chunks_fit = (ng + a.split - 1) / a.split + 1 <= MAXCH;
  while (true) {
    if (threadIdx.x == 0) s_item = (long long)atomicAdd(m_dev + 4, 1ull);
    __syncthreads();
    const long long it = s_item;
    __syncthreads();
    if (it >= items) break;
    const int bx = (int)(it % nb), by = (int)(it / nb);
    if (chunks_fit && a.m - bx * FT <= 32)
      field_tile_small<NQ>(a, bx, by, s_part, s_near);
    else
      field_tile<NQ, 0>(a, bx, by, s_src, s_cls, s_cols);
  }
}

// Fixed-order reduction of the panel splits: one warp per target, lane l
// sums splits l, l+32, ... in order, then a fixed butterfly over the lanes --
// the same order in both kernels (the tracer's per-target field is bitwise
// eval_efield_batch's), with the partial loads of a target in flight
// together instead of one dependent load per split.
HVB_DEV void reduce_target(const double* part, int split, int m, int i, int lane, double* out) {
  double s0 = 0, s1 = 0, s2 = 0;
  for (int s = lane; s < split; s += 32) {
    const double* p = part + ((size_t)s * m + i) * 4;
    s0 += p[0];
    s1 += p[1];
    s2 += p[2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    out[3 * (size_t)i] = s0;
    out[3 * (size_t)i + 1] = s1;
    out[3 * (size_t)i + 2] = s2;
  }
}

__global__ void k_field_reduce_dyn(const double* part, int split, const unsigned long long* m_dev, double* out) {
  const int m = (int)*m_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m; i += warps)
    reduce_target(part, split, m, i, lane, out);
}

__global__ void k_field_reduce(const double* part, int split, int m, double* out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i < m) reduce_target(part, split, m, i, threadIdx.x & 31, out);
}

// near-pair contributions (9 per pair, corner x component) contracted with u
// and added to the targets in sorted order (one thread per target segment)
__global__ void k_near_apply_points(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                    const int* tri_cols, const double* u, int potential, double* out) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  for (int p = seg_ptr[s]; p < seg_ptr[s + 1]; ++p) {
    const int i = pairs[2 * p], t = pairs[2 * p + 1];
    const int* tc = tri_cols + 3 * (size_t)t;
    const double* c = contrib + 9 * (size_t)p;
    double* o = out + 3 * (size_t)i;
    const double u0 = u[tc[0]], u1 = u[tc[1]], u2 = u[tc[2]];
    if (potential) {
      o[0] = __dadd_rn(o[0], __fma_rn(u2, c[2], __fma_rn(u1, c[1], __dmul_rn(u0, c[0]))));
    } else {
      // same operation order as the tracer's near pass (trace.cu k_trace_near)
      for (int d = 0; d < 3; ++d)
        o[d] = __dadd_rn(o[d], __fma_rn(u2, c[6 + d], __fma_rn(u1, c[3 + d], __dmul_rn(u0, c[d]))));
    }
  }
}

// Surface field at collocation vertices: singular (own star) panels with the
// corner Duffy rule and the E kernel, contracted with u; then the jump term
// side * u_i/2 * n_i and |E| (reference src/postprocess.py:152-159).
__global__ void k_field_singular(const double* nodes6, const int* tri_cols, const int* vc_ptr, const int* vc_tri,
                                 const int* vc_corner, const double* rule, int nm, const double* pts,
                                 const double* normals, const int* own_col, int m, const double* u, double side,
                                 double* efield, double* emag) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= m) return;
  const int own = own_col[w];
  const d3 X = mk3(pts[3 * (size_t)w], pts[3 * (size_t)w + 1], pts[3 * (size_t)w + 2]);
  double* E = efield + 3 * (size_t)w;
  for (int s = vc_ptr[own]; s < vc_ptr[own + 1]; ++s) {
    const int t = vc_tri[s], c = vc_corner[s];
    const double* Xn = nodes6 + 18 * (size_t)t;
    const double* R = rule + (size_t)c * nm * 4;
    const int* tc = tri_cols + 3 * (size_t)t;
    const double u0 = u[tc[0]], u1 = u[tc[1]], u2 = u[tc[2]];
    double sx = 0, sy = 0, sz = 0;
    for (int q = lane; q < nm; q += 32) {
      double uu = R[4 * q], vv = R[4 * q + 1], wq = R[4 * q + 2];
      d3 p;
      double jac;
      curved_point(Xn, uu, vv, p, jac);
      double dx = X.x - p.x, dy = X.y - p.y, dz = X.z - p.z;
      double r = sqrt(dx * dx + dy * dy + dz * dz);
      double sig = u0 * (1.0 - uu - vv) + u1 * uu + u2 * vv;
      double k = sig * wq * jac * kInv4Pi / (r * r * r);
      sx = fma(k, dx, sx);
      sy = fma(k, dy, sy);
      sz = fma(k, dz, sz);
    }
    sx = warp_sum(sx);
    sy = warp_sum(sy);
    sz = warp_sum(sz);
    if (lane == 0) {
      E[0] += sx;
      E[1] += sy;
      E[2] += sz;
    }
    __syncwarp();
  }
  if (lane == 0 && emag) {
    const double h = side * 0.5 * u[own];
    double ex = E[0] + h * normals[3 * (size_t)own];
    double ey = E[1] + h * normals[3 * (size_t)own + 1];
    double ez = E[2] + h * normals[3 * (size_t)own + 2];
    emag[w] = sqrt(ex * ex + ey * ey + ez * ez);
  }
}

template <int NQ>
static cudaError_t launch_field_nq(const FieldArgs& a, cudaStream_t st) {
  dim3 grid((a.m + FT - 1) / FT, a.split);
  if (a.potential)
    k_field<NQ, 1><<<grid, FT, 0, st>>>(a);
  else
    k_field<NQ, 2><<<grid, FT, 0, st>>>(a);  // E at points (the launch bounds of k_field)
  return cudaGetLastError();
}

cudaError_t launch_field(const FieldArgs& a, cudaStream_t st) {
  if (a.m == 0) return cudaSuccess;
  switch (a.nq) {
    case 3: return launch_field_nq<3>(a, st);
    case 6: return launch_field_nq<6>(a, st);
    case 12: return launch_field_nq<12>(a, st);
    case 16: return launch_field_nq<16>(a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_contract(const double* table, int nt, int nq, const int* tri_cols, const double* u, double* src,
                            cudaStream_t st) {
  int n = nt * nq;
  k_contract<<<(n + 255) / 256, 256, 0, st>>>(table, nt, nq, tri_cols, u, src);
  return cudaGetLastError();
}

cudaError_t launch_field_dyn(const FieldArgs& a, unsigned long long* m_dev, int grid, cudaStream_t st) {
  switch (a.nq) {
    case 3: k_field_dyn<3><<<grid, FT, 0, st>>>(a, m_dev); break;
    case 6: k_field_dyn<6><<<grid, FT, 0, st>>>(a, m_dev); break;
    case 12: k_field_dyn<12><<<grid, FT, 0, st>>>(a, m_dev); break;
    case 16: k_field_dyn<16><<<grid, FT, 0, st>>>(a, m_dev); break;
    default: return cudaErrorInvalidValue;
  }
  if (cudaGetLastError() != cudaSuccess) return cudaErrorLaunchFailure;
  k_field_reduce_dyn<<<1184, 128, 0, st>>>(a.part, a.split, m_dev, a.out);
  return cudaGetLastError();
}

cudaError_t launch_field_reduce(const double* part, int split, int m, double* out, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  k_field_reduce<<<(unsigned)(((long long)m * 32 + 255) / 256), 256, 0, st>>>(part, split, m, out);
  return cudaGetLastError();
}

cudaError_t launch_near_apply_points(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                     const int* tri_cols, const double* u, int potential, double* out,
                                     cudaStream_t st) {
  if (n_seg == 0) return cudaSuccess;
  k_near_apply_points<<<(n_seg + 127) / 128, 128, 0, st>>>(seg_ptr, n_seg, pairs, contrib, tri_cols, u, potential,
                                                           out);
  return cudaGetLastError();
}

cudaError_t launch_field_singular(const double* nodes6, const int* tri_cols, const int* vc_ptr, const int* vc_tri,
                                  const int* vc_corner, const double* rule, int nm, const double* pts,
                                  const double* normals, const int* own_col, int m, const double* u, double side,
                                  double* efield, double* emag, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  k_field_singular<<<(m * 32 + 127) / 128, 128, 0, st>>>(nodes6, tri_cols, vc_ptr, vc_tri, vc_corner, rule, nm, pts,
                                                         normals, own_col, m, u, side, efield, emag);
  return cudaGetLastError();
}

}  // namespace hvb
