// K8/K9: streaming GEMV for the GMRES matvec and the solver's row scans.
//
// Reference: matvec src/assembly.py:376-400 (per-row dot), solver row
// equilibration / diagonal src/solver.py:98-108.
//
// y[i] = left[i] * sum_k A[i,k] * xp[k] with A row-major (lda >= N, 16-byte
// aligned rows) in device column order and xp the (permuted, scaled) Krylov
// vector.  A CTA owns ROWS rows; every thread loads each 16-byte x chunk
// once and reuses it for all ROWS rows, so x costs 1/ROWS of the matrix
// traffic (from L2) and the matrix itself is streamed with evict-first
// loads.  The per-row summation order depends only on N and the thread
// count, never on the row blocking: results are bitwise identical for any
// block partition (reference invariance, tests/test_assembly.py:72-78).
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "launch.cuh"

namespace hvb {

constexpr int GEMV_THREADS = 256;

// 256-bit non-allocating global load of 4 doubles (LDG.E.NA.ENL2.256)
HVB_DEV void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

// outs != nullptr: the fused all-gather -- each row result is stored into
// all n_out replicated vectors (this GPU's and every peer's, mapped over
// NVLink by CUDA IPC) at position out_off + row, instead of into y.
template <int ROWS>
__global__ void __launch_bounds__(GEMV_THREADS) k_gemv_f64(const double* __restrict__ A, int64_t lda, int nrows,
                                                           int ncols, const double* __restrict__ x,
                                                           const double* __restrict__ left,
                                                           double* __restrict__ y, double* const* outs, int n_out,
                                                           int64_t out_off) {
  const int r0 = blockIdx.x * ROWS;
  const int tid = threadIdx.x;
  double acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) acc[r] = 0.0;
  const int n2 = ncols >> 1;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const double2* rowp[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    int rr = min(r0 + r, nrows - 1);
    rowp[r] = reinterpret_cast<const double2*>(A + (int64_t)rr * lda);
  }
#pragma unroll 2
  for (int k = tid; k < n2; k += GEMV_THREADS) {
    const double2 xv = __ldg(x2 + k);
    double2 av[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) av[r] = __ldcs(rowp[r] + k);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) acc[r] = fma(av[r].y, xv.y, fma(av[r].x, xv.x, acc[r]));
  }
  if ((ncols & 1) && tid == 0) {
    const double xv = x[ncols - 1];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      int rr = min(r0 + r, nrows - 1);
      acc[r] = fma(A[(int64_t)rr * lda + ncols - 1], xv, acc[r]);
    }
  }
  __shared__ double red[ROWS][GEMV_THREADS / 32];
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    double v = warp_sum(acc[r]);
    if (lane == 0) red[r][wid] = v;
  }
  __syncthreads();
  if (tid < ROWS && r0 + tid < nrows) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < GEMV_THREADS / 32; ++w) s += red[tid][w];
    const double v = left ? left[r0 + tid] * s : s;
    if (outs) {
      for (int k = 0; k < n_out; ++k) outs[k][out_off + r0 + tid] = v;
    } else {
      y[r0 + tid] = v;
    }
  }
}

// Single-precision storage (reference matvec src/assembly.py:386-392: v is
// cast to float32 and every row is reduced by a float32 dot, data[i] @ vc).
// 256-bit loads (8 floats), 8 rows per CTA.  F32ACC (the reference
// semantics, default): products and every partial sum in float32 (FMA
// chains per thread, then a float32 tree over the CTA), the row result
// widened to double at the end.  !F32ACC (opt-in, hvb_gemv prec 2): float32
// partials over 8 columns accumulated in double.
HVB_DEV void ld256f(const float* p, float* v) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

template <int ROWS, bool F32ACC>
__global__ void __launch_bounds__(GEMV_THREADS) k_gemv_f32_v8(const float* __restrict__ A, int64_t lda, int nrows,
                                                              int ncols, const double* __restrict__ x,
                                                              const double* __restrict__ left,
                                                              double* __restrict__ y) {
  using Acc = typename std::conditional<F32ACC, float, double>::type;
  const int r0 = blockIdx.x * ROWS;
  const int tid = threadIdx.x;
  Acc acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) acc[r] = Acc(0);
  const int n8 = ncols >> 3;
  const float* rowp[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) rowp[r] = A + (int64_t)min(r0 + r, nrows - 1) * lda;
  for (int k = tid; k < n8; k += GEMV_THREADS) {
    float xf[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) xf[j] = (float)x[8 * k + j];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      float a[8];
      ld256f(rowp[r] + 8 * k, a);
      if (F32ACC) {
        float s = (float)acc[r];
#pragma unroll
        for (int j = 0; j < 8; ++j) s = fmaf(a[j], xf[j], s);
        acc[r] = s;
      } else {
        float s = a[0] * xf[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) s = fmaf(a[j], xf[j], s);
        acc[r] += (double)s;
      }
    }
  }
  if (tid == 0) {
    for (int c = 8 * n8; c < ncols; ++c) {
      const float xv = (float)x[c];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        if (F32ACC)
          acc[r] = fmaf(rowp[r][c], xv, (float)acc[r]);
        else
          acc[r] += (double)(rowp[r][c] * xv);
      }
    }
  }
  __shared__ Acc red[ROWS][GEMV_THREADS / 32];
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    Acc v = warp_sum(acc[r]);
    if (lane == 0) red[r][wid] = v;
  }
  __syncthreads();
  if (tid < ROWS && r0 + tid < nrows) {
    Acc s = Acc(0);
#pragma unroll
    for (int w = 0; w < GEMV_THREADS / 32; ++w) s += red[tid][w];
    y[r0 + tid] = left ? left[r0 + tid] * (double)s : (double)s;
  }
}

// xp[k] = z[perm[k]] / right[perm[k]]   (right may be null)
__global__ void k_gather_scale(const double* z, const double* right, const int* perm, int n, double* xp) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int j = perm ? perm[k] : k;
  double v = z[j];
  xp[k] = right ? v / right[j] : v;
}

// per-row max |A[i,:]| and the diagonal A[i, diag_col[i]]
template <typename T>
__global__ void k_rowmax_diag(const T* A, int64_t lda, int nrows, int ncols, const int* diag_col,
                              double* rowmax, double* diag) {
  const int r = blockIdx.x;
  if (r >= nrows) return;
  const T* row = A + (int64_t)r * lda;
  double m = 0.0;
  if (sizeof(T) == 8 && lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 31) == 0) {
    const double* rd = reinterpret_cast<const double*>(row);
    const int n4 = ncols >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) {
      double a, b, c, d;
      ld256(rd + 4 * k, a, b, c, d);
      m = fmax(m, fmax(fmax(fabs(a), fabs(b)), fmax(fabs(c), fabs(d))));
    }
    for (int k = 4 * n4 + threadIdx.x; k < ncols; k += blockDim.x) m = fmax(m, fabs(rd[k]));
  } else {
    for (int k = threadIdx.x; k < ncols; k += blockDim.x) m = fmax(m, fabs((double)row[k]));
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = fmax(mm, red[w]);
    rowmax[r] = mm;
    if (diag) diag[r] = diag_col[r] >= 0 ? (double)row[diag_col[r]] : 0.0;
  }
}

struct PeerSignal {
  unsigned long long* const* flags;  // world pointers: flag row of every rank (null: no signal)
  int world, rank;
  unsigned long long epoch;
  unsigned int* done;                // CTA completion counter (zero between launches)
};

// Release protocol of the fused GEMV + all-gather (csrc/peer.cu): every
// thread that stored row results into peer memory fences at system scope,
// the CTA barrier orders those fences before thread 0's completion count,
// and the LAST CTA publishes the epoch into every rank's flag row with a
// system-scope release store.  A peer that acquires the epoch
// (hvb_peer_wait, ld.acquire.sys) therefore sees every row of this launch.
HVB_DEV void peer_release(const PeerSignal& sig, int tid) {
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(sig.done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      for (int r = 0; r < sig.world; ++r) {
        unsigned long long* f = sig.flags[r] + sig.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(sig.epoch) : "memory");
      }
      *sig.done = 0u;  // stream order: the next launch starts from zero
    }
  }
}

template <int ROWS>
__global__ void k_gemv_f64_v4(const double* __restrict__ A, int64_t lda, int nrows, int ncols,
                              const double* __restrict__ x, const double* __restrict__ left, double* __restrict__ y,
                              double* const* outs, int n_out, int64_t out_off, PeerSignal sig);

// 256-bit loads need 32-byte aligned rows and x: the production FP64 path
// (2 rows per CTA, LDG.256 non-allocating: 7.5 TB/s on a cfg4-width block vs
// 5.7 TB/s for 128-bit loads and 8 rows per CTA, tools/gemv_probe.py)
static bool v4_ok(const void* A, int64_t lda, const double* x) {
  return lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 31) == 0 && (reinterpret_cast<uintptr_t>(x) & 31) == 0;
}

// prec 0: double matrix; 1: float matrix, float32 reduction (reference
// semantics); 2: float matrix, float32 partials accumulated in double
cudaError_t launch_gemv(const void* A, int prec, int64_t lda, int nrows, int ncols, const double* x,
                        const double* left, double* y, cudaStream_t st) {
  if (nrows == 0) return cudaSuccess;
  if (prec != 0) {
    if (lda % 8 != 0 || (reinterpret_cast<uintptr_t>(A) & 31) != 0) return cudaErrorInvalidValue;
    if (prec == 1)
      k_gemv_f32_v8<8, true><<<(nrows + 7) / 8, GEMV_THREADS, 0, st>>>((const float*)A, lda, nrows, ncols, x, left, y);
    else
      k_gemv_f32_v8<8, false><<<(nrows + 7) / 8, GEMV_THREADS, 0, st>>>((const float*)A, lda, nrows, ncols, x, left,
                                                                        y);
  } else if (v4_ok(A, lda, x)) {
    k_gemv_f64_v4<2><<<(nrows + 1) / 2, GEMV_THREADS, 0, st>>>((const double*)A, lda, nrows, ncols, x, left, y,
                                                               nullptr, 0, 0, PeerSignal{});
  } else {
    constexpr int R = 4;
    k_gemv_f64<R><<<(nrows + R - 1) / R, GEMV_THREADS, 0, st>>>((const double*)A, lda, nrows, ncols, x, left, y,
                                                                nullptr, 0, 0);
  }
  return cudaGetLastError();
}

cudaError_t launch_gemv_bcast(const double* A, int64_t lda, int nrows, int ncols, const double* x, const double* left,
                              double* const* outs, int n_out, int64_t out_off, unsigned long long* const* flags,
                              int rank, unsigned long long epoch, unsigned int* done, cudaStream_t st) {
  // the row-sharded store is always 256-byte pitched; every rank owns >= 1 row
  if (!v4_ok(A, lda, x) || nrows < 1) return cudaErrorInvalidValue;
  PeerSignal sig{flags, n_out, rank, epoch, done};
  k_gemv_f64_v4<2><<<(nrows + 1) / 2, GEMV_THREADS, 0, st>>>(A, lda, nrows, ncols, x, left, nullptr, outs, n_out,
                                                             out_off, sig);
  return cudaGetLastError();
}

cudaError_t launch_gather_scale(const double* z, const double* right, const int* perm, int n, double* xp,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_gather_scale<<<(n + 255) / 256, 256, 0, st>>>(z, right, perm, n, xp);
  return cudaGetLastError();
}

cudaError_t launch_rowmax_diag(const void* A, int is_f32, int64_t lda, int nrows, int ncols, const int* diag_col,
                               double* rowmax, double* diag, cudaStream_t st) {
  if (nrows == 0) return cudaSuccess;
  if (is_f32)
    k_rowmax_diag<float><<<nrows, 256, 0, st>>>((const float*)A, lda, nrows, ncols, diag_col, rowmax, diag);
  else
    k_rowmax_diag<double><<<nrows, 256, 0, st>>>((const double*)A, lda, nrows, ncols, diag_col, rowmax, diag);
  return cudaGetLastError();
}

}  // namespace hvb

// ---------------------------------------------------------------------------
// K9: Arnoldi orthogonalisation of one GMRES step in ONE cooperative launch
// (reference _gmres_cycle src/solver.py:177-196): modified Gram-Schmidt of w
// against V[0..j] -- for i = 0..j: h_i = V_i . w; w -= h_i V_i -- plus the
// norms before and after.  Each CTA owns a fixed contiguous slice of the N
// entries; a projection's partial dots are written per CTA, the grid syncs,
// and every CTA sums the partials in CTA order, so h_i (and w) are identical
// on every CTA and bitwise reproducible.  accumulate = 1 adds the
// projections to h (the reference's single re-orthogonalisation pass).
// ---------------------------------------------------------------------------
namespace hvb {
namespace cgk = cooperative_groups;

constexpr int MGS_THREADS = 1024;

HVB_DEV double block_sum(double v, double* s_red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (MGS_THREADS >> 5) ? s_red[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in warp 0
}

__global__ void __launch_bounds__(MGS_THREADS) k_mgs(const double* __restrict__ V, long long ldv, int j,
                                                     double* __restrict__ w, int n, double* __restrict__ h,
                                                     double* __restrict__ norms, double* __restrict__ partial,
                                                     int accumulate) {
  cgk::grid_group grid = cgk::this_grid();
  __shared__ double s_red[MGS_THREADS / 32];
  __shared__ double s_val;
  const int nb = gridDim.x;
  const int chunk = (n + nb - 1) / nb;
  const int a = min(n, blockIdx.x * chunk), b = min(n, a + chunk);
  auto grid_total = [&](double v, int slot) {
    const double t = block_sum(v, s_red);
    if (threadIdx.x == 0) partial[(size_t)slot * nb + blockIdx.x] = t;
    grid.sync();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int k = 0; k < nb; ++k) s += partial[(size_t)slot * nb + k];
      s_val = s;
    }
    __syncthreads();
    return s_val;
  };
  double loc = 0.0;
  for (int k = a + threadIdx.x; k < b; k += MGS_THREADS) loc = fma(w[k], w[k], loc);
  const double nb2 = grid_total(loc, 0);
  for (int i = 0; i <= j; ++i) {
    const double* vi = V + (size_t)i * ldv;
    loc = 0.0;
    for (int k = a + threadIdx.x; k < b; k += MGS_THREADS) loc = fma(vi[k], w[k], loc);
    const double hi = grid_total(loc, 1 + (i & 1));  // alternating slots: no overwrite race
    for (int k = a + threadIdx.x; k < b; k += MGS_THREADS) w[k] = fma(-hi, vi[k], w[k]);
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = accumulate ? h[i] + hi : hi;
  }
  loc = 0.0;
  for (int k = a + threadIdx.x; k < b; k += MGS_THREADS) loc = fma(w[k], w[k], loc);
  const double na2 = grid_total(loc, 3);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    norms[0] = sqrt(nb2);
    norms[1] = sqrt(na2);
  }
}

// Cluster variant (the default when N <= 16 * 1024 * 8): ONE thread-block
// cluster of 16 CTAs x 1024 threads (non-portable size, one CTA per SM).  Each
// thread keeps its PER entries of w in registers for the whole launch and
// reads each V_i entry once (the dot and the update share the load); the
// per-projection reduction goes through distributed shared memory and the
// hardware cluster barrier instead of a global-memory grid sync.  Every CTA
// sums the 16 CTA partials in the same fixed order, so h_i is identical in
// every CTA and the result is bitwise reproducible.
constexpr int MGSC_CTAS = 16;

template <int PER>
__global__ void __launch_bounds__(MGS_THREADS) k_mgs_cluster(const double* __restrict__ V, long long ldv, int j,
                                                             double* __restrict__ w, int n, double* __restrict__ h,
                                                             double* __restrict__ norms, int accumulate) {
  cgk::cluster_group cl = cgk::this_cluster();
  __shared__ double s_red[MGS_THREADS / 32];
  __shared__ double s_part[2];
  __shared__ double s_val;
  const int rank = (int)cl.block_rank();
  const int chunk = (n + MGSC_CTAS - 1) / MGSC_CTAS;
  const int a = min(n, rank * chunk), b = min(n, a + chunk);
  const int lane = threadIdx.x & 31;
  auto total = [&](double v, int slot) {
    const double t = block_sum(v, s_red);
    if (threadIdx.x == 0) s_part[slot] = t;
    cl.sync();  // partials of every CTA visible (also a CTA barrier)
    if (threadIdx.x < 32) {
      double p = lane < MGSC_CTAS ? *cl.map_shared_rank(&s_part[slot], lane) : 0.0;
      // fixed pairwise order over the 16 CTA partials
#pragma unroll
      for (int o = 1; o < MGSC_CTAS; o <<= 1) p += __shfl_down_sync(0xffffffffu, p, o);
      if (threadIdx.x == 0) s_val = p;
    }
    __syncthreads();
    return s_val;
  };
  double wr[PER];
  double loc = 0.0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int k = a + threadIdx.x + e * MGS_THREADS;
    wr[e] = k < b ? w[k] : 0.0;
    loc = fma(wr[e], wr[e], loc);
  }
  const double nb2 = total(loc, 0);
  for (int i = 0; i <= j; ++i) {
    const double* vi = V + (size_t)i * ldv;
    double vr[PER];
    loc = 0.0;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int k = a + threadIdx.x + e * MGS_THREADS;
      vr[e] = k < b ? vi[k] : 0.0;
      loc = fma(vr[e], wr[e], loc);
    }
    const double hi = total(loc, (i + 1) & 1);  // alternating slots: a slot is rewritten two barriers later
#pragma unroll
    for (int e = 0; e < PER; ++e) wr[e] = fma(-hi, vr[e], wr[e]);
    if (rank == 0 && threadIdx.x == 0) h[i] = accumulate ? h[i] + hi : hi;
  }
  loc = 0.0;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int k = a + threadIdx.x + e * MGS_THREADS;
    if (k < b) w[k] = wr[e];
    loc = fma(wr[e], wr[e], loc);
  }
  const double na2 = total(loc, (j + 2) & 1);
  if (rank == 0 && threadIdx.x == 0) {
    norms[0] = sqrt(nb2);
    norms[1] = sqrt(na2);
  }
  cl.sync();  // no CTA leaves while a peer may still read its s_part
}

template <int PER>
static cudaError_t launch_mgs_cluster(const double* V, long long ldv, int j, double* w, int n, double* h,
                                      double* norms, int accumulate, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(k_mgs_cluster<PER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(MGSC_CTAS);
  cfg.blockDim = dim3(MGS_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MGSC_CTAS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mgs_cluster<PER>, V, ldv, j, w, n, h, norms, accumulate);
}

// 1: cluster path usable (HVB_MGS=coop forces the cooperative kernel)
static int mgs_cluster_ok() {
  static int ok = -1;
  if (ok < 0) {
    const char* env = getenv("HVB_MGS");
    ok = 0;
    if (!(env && strcmp(env, "coop") == 0)) {
      int dev = 0, major = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
      if (major >= 9 &&
          cudaFuncSetAttribute(k_mgs_cluster<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(MGSC_CTAS);
        cfg.blockDim = dim3(MGS_THREADS);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = MGSC_CTAS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, k_mgs_cluster<8>, &cfg) == cudaSuccess && clusters >= 1) ok = 1;
      }
      cudaGetLastError();  // clear a failed probe
    }
  }
  return ok;
}

int mgs_grid() {
  static int g = 0;
  if (g == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mgs, MGS_THREADS, 0);
    // the projections are grid-sync bound: 16-48 CTAs of 1024 threads measure
    // the same (34 ms of MGS per cfg4 solve, vs 102 ms with 296 x 256)
    g = per < 1 ? per : (sms < 32 ? sms : 32);
    if (g < 1) g = 1;
  }
  return g;
}

cudaError_t launch_mgs(const double* V, long long ldv, int j, double* w, int n, double* h, double* norms,
                       double* partial, int accumulate, cudaStream_t st) {
  if (mgs_cluster_ok()) {
    if (n <= MGSC_CTAS * MGS_THREADS * 2) return launch_mgs_cluster<2>(V, ldv, j, w, n, h, norms, accumulate, st);
    if (n <= MGSC_CTAS * MGS_THREADS * 4) return launch_mgs_cluster<4>(V, ldv, j, w, n, h, norms, accumulate, st);
    if (n <= MGSC_CTAS * MGS_THREADS * 8) return launch_mgs_cluster<8>(V, ldv, j, w, n, h, norms, accumulate, st);
  }
  const int grid = mgs_grid();
  void* args[] = {(void*)&V, (void*)&ldv, (void*)&j, (void*)&w, (void*)&n, (void*)&h, (void*)&norms,
                  (void*)&partial, (void*)&accumulate};
  return cudaLaunchCooperativeKernel((void*)k_mgs, grid, MGS_THREADS, args, 0, st);
}

}  // namespace hvb

// ---------------------------------------------------------------------------
// 256-bit-load GEMV variant (LDG.E.NA.ENL2.256: 4 doubles per load, no L1
// allocation): same per-row summation structure as k_gemv_f64 over 4-column
// chunks.  Used by hvb_gemv when lda % 4 == 0 (A/B in tools/gemv_probe.py).
// ---------------------------------------------------------------------------
namespace hvb {


template <int ROWS>
__global__ void k_gemv_f64_v4(const double* __restrict__ A, int64_t lda, int nrows, int ncols,
                              const double* __restrict__ x, const double* __restrict__ left, double* __restrict__ y,
                              double* const* outs, int n_out, int64_t out_off, PeerSignal sig) {
  const int r0 = blockIdx.x * ROWS;
  const int tid = threadIdx.x;
  double acc[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) acc[r] = 0.0;
  const int n4 = ncols >> 2;
  const double* rowp[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) rowp[r] = A + (int64_t)min(r0 + r, nrows - 1) * lda;
#pragma unroll 2
  for (int k = tid; k < n4; k += GEMV_THREADS) {
    const double4 xv = *reinterpret_cast<const double4*>(x + 4 * k);
    double a[ROWS][4];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) ld256(rowp[r] + 4 * k, a[r][0], a[r][1], a[r][2], a[r][3]);
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
      acc[r] = fma(a[r][3], xv.w, fma(a[r][2], xv.z, fma(a[r][1], xv.y, fma(a[r][0], xv.x, acc[r]))));
  }
  if (tid == 0) {
    for (int c = 4 * n4; c < ncols; ++c) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) acc[r] = fma(rowp[r][c], x[c], acc[r]);
    }
  }
  __shared__ double red[ROWS][GEMV_THREADS / 32];
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    double v = warp_sum(acc[r]);
    if (lane == 0) red[r][wid] = v;
  }
  __syncthreads();
  if (tid < ROWS && r0 + tid < nrows) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < GEMV_THREADS / 32; ++w) s += red[tid][w];
    const double v = left ? left[r0 + tid] * s : s;
    if (outs) {
      for (int k = 0; k < n_out; ++k) outs[k][out_off + r0 + tid] = v;
    } else {
      y[r0 + tid] = v;
    }
  }
  if (sig.flags) peer_release(sig, tid);
}
}  // namespace hvb

