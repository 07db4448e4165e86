// Dense collocation assembly: panel tables (K1), the regular sweep (K2+K3,
// fused classification), the singular Duffy pass (K4) and the row-kind
// epilogue pieces (K6).
//
// Reference: row_pass1 src/assembly.py:135-242, TriangleTables 73-118,
// _row_equation 408-468.
//
// Data layout of the regular sweep:
//  * device column order = spatially compact column tiles (<= a few
//    thousand collocation vertices), each swept in a banded order, so a
//    panel's owned corners lie within `band` columns of its first one;
//  * per tile a *panel stream*: one 8*(6*NQ+8)-byte record per panel that
//    touches the tile (nodes with pre-weighted hat factors, circumcircle
//    classification data, owned local columns) -- contiguous, staged into
//    shared memory with cp.async, broadcast to the 32 lanes;
//  * a warp owns 32 rows (one per lane) and a sliding window of WIN owned
//    columns in shared memory; columns are flushed (coalesced 256-byte row
//    segments) as soon as the sweep has passed their last panel, so every
//    matrix element is written exactly once and there are no atomics.
#include "launch.cuh"

namespace hvb {

constexpr int WIN = 96;          // window columns per warp (band <= WIN - 32)
constexpr int WSTRIDE = 33;      // padded row stride of the window (bank spread)
constexpr int RING = 4;          // panel-record pipeline depth per warp

struct RowData {   // per assembled row (one lane)
  double x, y, z;     // collocation point
  double nx, ny, nz;  // normal (ADL rows)
};



__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int REC>
__device__ __forceinline__ void stage_record(double* dst, const double* src, int lane) {
  constexpr int CH = REC / 2;  // 16-byte chunks
#pragma unroll
  for (int c = lane; c < CH; c += 32) cp_async16(dst + 2 * c, src + 2 * c);
}

// MODE: 0 = all SL rows, 1 = all ADL rows, 2 = mixed warp
template <int NQ, int MODE>
__global__ void __launch_bounds__(128) k_assemble_regular(RegularArgs a) {
  constexpr int REC = 6 * NQ + 8;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  double* win = smem + wib * (WIN * WSTRIDE + RING * REC);
  double* ring = win + WIN * WSTRIDE;

  const int rowtile = blockIdx.x * wpb + wib;
  const int tile = blockIdx.y;
  if (rowtile * 32 >= a.n_rows) return;
  const int li0 = rowtile * 32 + lane;
  const bool live = li0 < a.n_rows;
  const int li = a.row_begin + li0;                       // row-list index
  const int lrow = a.row_begin + (live ? li0 : a.n_rows - 1);

  // per-lane row data
  const double* rd = a.rowdata + 6 * (size_t)lrow;
  const d3 X = mk3(rd[0], rd[1], rd[2]);
  const double nx = rd[3], ny = rd[4], nz = rd[5];
  const bool adl = (MODE == 1) || (MODE == 2 && a.row_kind[lrow] == 1);
  const int own_col = a.row_col[lrow];
  const double scale = a.row_scale[lrow];
  const int64_t out_off = live ? a.row_out[lrow] : -1;

  for (int k = lane; k < WIN * WSTRIDE; k += 32) win[k] = 0.0;

  const int64_t e0 = a.tile_ptr[tile], e1 = a.tile_ptr[tile + 1];
  const int col0 = a.tile_col0[tile], width = a.tile_width[tile];
  const double* src = a.stream + e0 * REC;
  const int64_t ne = e1 - e0;

#pragma unroll
  for (int s = 0; s < RING - 1; ++s) {
    if (s < ne) stage_record<REC>(ring + s * REC, src + (int64_t)s * REC, lane);
    cp_async_commit();
  }

  int base = 0;  // first local column held by the window
  auto flush32 = [&](int b) {
    // column b+lane of the 32 rows of this warp: coalesced row segments
    const int c = b + lane;
    double* wcol = win + ((c % WIN) * WSTRIDE);
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      int64_t off = __shfl_sync(0xffffffffu, out_off, j);
      double sc = __shfl_sync(0xffffffffu, scale, j);
      if (off >= 0 && c < width) a.A[off + col0 + c] = wcol[j] * sc;
      wcol[j] = 0.0;
    }
    __syncwarp();
  };

  for (int64_t e = 0; e < ne; ++e) {
    cp_async_wait<RING - 2>();
    __syncwarp();
    const double* rec = ring + (e % RING) * REC;
    {
      int64_t nxt = e + RING - 1;
      if (nxt < ne) stage_record<REC>(ring + (nxt % RING) * REC, src + nxt * REC, lane);
      cp_async_commit();
    }
    const int* meta = reinterpret_cast<const int*>(rec + 6 * NQ + 6);
    const int tri = meta[0];
    const int mfirst = meta[1];
    const short* loc = reinterpret_cast<const short*>(meta + 2);
    const int l0 = loc[0], l1 = loc[1], l2 = loc[2], flags = loc[3];

    while (mfirst >= base + 32) {
      flush32(base);
      base += 32;
    }

    const double* cg = rec + 6 * NQ;
    const bool reg = is_regular(X, mk3(cg[0], cg[1], cg[2]), cg[3], cg[4], cg[5]);

    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double2 p01 = *reinterpret_cast<const double2*>(rec + 6 * q);
      const double2 p2w = *reinterpret_cast<const double2*>(rec + 6 * q + 2);
      const double2 w12 = *reinterpret_cast<const double2*>(rec + 6 * q + 4);
      const double dx = X.x - p01.x, dy = X.y - p01.y, dz = X.z - p2w.x;
      const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
      const double ri = rsqrt_full(r2);
      double k;
      if (MODE == 0) {
        k = ri;
      } else {
        const double dn = fma(dz, nz, fma(dy, ny, dx * nx));
        const double k_adl = dn * (ri * ri * ri);
        k = (MODE == 1) ? k_adl : (adl ? k_adl : ri);
      }
      a0 = fma(k, p2w.y, a0);
      a1 = fma(k, w12.x, a1);
      a2 = fma(k, w12.y, a2);
    }
    if (!reg) {
      a0 = 0.0; a1 = 0.0; a2 = 0.0;
    }
    // deferred near-singular pairs, emitted once per (row, panel): only from
    // the panel's primary tile (flag bit 0)
    bool emit = false;
    if (!reg && live && (flags & 1)) {
      const int* tc = a.tri_cols + 3 * (size_t)tri;
      emit = !(tc[0] == own_col || tc[1] == own_col || tc[2] == own_col);
    }
    const unsigned m = __ballot_sync(0xffffffffu, emit);
    if (m) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(a.near_count, (unsigned long long)__popc(m));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (emit) {
        long long slot = (long long)b + __popc(m & ((1u << lane) - 1u));
        if (slot < a.near_cap) {
          a.near_list[2 * slot] = li;
          a.near_list[2 * slot + 1] = tri;
        }
      }
    }
    if (l0 >= 0) win[(l0 % WIN) * WSTRIDE + lane] += a0;
    if (l1 >= 0) win[(l1 % WIN) * WSTRIDE + lane] += a1;
    if (l2 >= 0) win[(l2 % WIN) * WSTRIDE + lane] += a2;
  }
  cp_async_wait<0>();
  __syncwarp();
  while (base < width) {
    flush32(base);
    base += 32;
  }
}

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

// Pack one stream record per (tile, panel) entry.
__global__ void k_build_stream(const double* __restrict__ table, int nq,
                               const double* __restrict__ ccr,  // (nt,4): cc, R
                               double eta, const int* __restrict__ ent_tri,
                               const int* __restrict__ ent_meta,  // (ne,4): mfirst, l0,l1,l2 | flags<<?
                               int64_t ne, double* __restrict__ out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int rec = 6 * nq + 8;
  int t = ent_tri[e];
  double* o = out + e * rec;
  const double* s = table + (size_t)t * 6 * nq;
  for (int k = 0; k < 6 * nq; ++k) o[k] = s[k];
  const double* c = ccr + 4 * (size_t)t;
  double thr = __dmul_rn(eta, c[3]);
  double t2 = thr * thr;
  o[6 * nq + 0] = c[0];
  o[6 * nq + 1] = c[1];
  o[6 * nq + 2] = c[2];
  o[6 * nq + 3] = thr;
  o[6 * nq + 4] = t2 * (1.0 - 1e-13);
  o[6 * nq + 5] = t2 * (1.0 + 1e-13);
  int* m = reinterpret_cast<int*>(o + 6 * nq + 6);
  const int* em = ent_meta + 5 * e;
  m[0] = t;
  m[1] = em[0];
  short* l = reinterpret_cast<short*>(m + 2);
  l[0] = (short)em[1];
  l[1] = (short)em[2];
  l[2] = (short)em[3];
  l[3] = (short)em[4];
}

// K4: singular (corner) pairs.  One warp per row; the row's star panels are
// processed in triangle order (reference row_pass1 singular batch,
// src/assembly.py:202-235) and added to the row after the regular sweep.
// Duffy rule tables per corner: rule[c][m] = (u, v, w, pad).


__global__ void k_assemble_singular(SingularArgs a) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= a.n_rows) return;
  const double* rd = a.rowdata + 6 * (size_t)w;
  const d3 X = mk3(rd[0], rd[1], rd[2]);
  const double nx = rd[3], ny = rd[4], nz = rd[5];
  const bool adl = a.row_kind[w] == 1;
  const int own = a.row_col[w];
  const double sc = a.row_scale[w];
  double* Arow = a.A + a.row_out[w];
  if (own < 0) return;
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

size_t regular_smem_bytes(int nq, int wpb) {
  return (size_t)wpb * (WIN * WSTRIDE + RING * (6 * nq + 8)) * sizeof(double);
}

template <int NQ>
static cudaError_t launch_regular_nq(const RegularArgs& a, int mode, int wpb, cudaStream_t st) {
  dim3 grid((a.n_rows + 32 * wpb - 1) / (32 * wpb), a.n_tiles);
  size_t smem = regular_smem_bytes(NQ, wpb);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * wpb, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (mode == 0) return go(k_assemble_regular<NQ, 0>);
  if (mode == 1) return go(k_assemble_regular<NQ, 1>);
  return go(k_assemble_regular<NQ, 2>);
}

cudaError_t launch_regular(const RegularArgs& a, int nq, int mode, int wpb, cudaStream_t st) {
  switch (nq) {
    case 3: return launch_regular_nq<3>(a, mode, wpb, st);
    case 6: return launch_regular_nq<6>(a, mode, wpb, st);
    case 12: return launch_regular_nq<12>(a, mode, wpb, st);
    case 16: return launch_regular_nq<16>(a, mode, wpb, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_build_table(const double* nodes6, int nt, int nq, const double* rule, double* out,
                               cudaStream_t st) {
  int n = nt * nq;
  k_build_table<<<(n + 255) / 256, 256, 0, st>>>(nodes6, nt, nq, rule, out);
  return cudaGetLastError();
}

cudaError_t launch_build_stream(const double* table, int nq, const double* ccr, double eta,
                                const int* ent_tri, const int* ent_meta, int64_t ne, double* out,
                                cudaStream_t st) {
  if (ne == 0) return cudaSuccess;
  k_build_stream<<<(unsigned)((ne + 127) / 128), 128, 0, st>>>(table, nq, ccr, eta, ent_tri, ent_meta, ne, out);
  return cudaGetLastError();
}

cudaError_t launch_singular(const SingularArgs& a, cudaStream_t st) {
  if (a.n_rows == 0) return cudaSuccess;
  int threads = 128;
  int blocks = (a.n_rows * 32 + threads - 1) / threads;
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
