// K5: deferred near-singular pairs (reference row_pass2 src/assembly.py:245-292,
// near_singular_rule src/quadrature.py:409-450, subdivide_at 296-332).
//
// One warp per (evaluation point, panel) pair.  All lanes evaluate the
// discrete plan redundantly (closest point, subdivision, grading depth --
// with the reference's rounding, common.cuh) and then split the composite
// rule's nodes (128..3072) across lanes; the three (or nine, for the field
// kernel) corner sums are reduced with a fixed butterfly, so the result is
// deterministic.  Pairs arrive sorted by (point, panel); the apply kernels
// add them to their rows / targets sequentially in that order.
#include "near.cuh"

namespace hvb {



__global__ void k_near_pairs(NearArgs a) {
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (w >= a.n_pairs) return;
  const int pi = a.pairs[2 * w], t = a.pairs[2 * w + 1];
  const double* P = a.points + 6 * (size_t)pi;
  const d3 X = mk3(P[0], P[1], P[2]);
  const d3 N = mk3(P[3], P[4], P[5]);
  const int kind = a.kind[pi];
  double acc[9];
  near_pair_acc(X, N, kind, a.nodes6 + 18 * (size_t)t, a.radii[t], a.duffy, a.n_duffy, a.graded, a.n_graded,
                a.bisect_depth, a.bisect_trigger, acc);
  const int nout = kind == 2 ? 9 : 3;
  for (int k = 0; k < nout; ++k) {
    double s = warp_sum(acc[k]);
    if (lane == 0) a.out[9 * w + k] = s;
  }
}

// Add sorted near-pair contributions to assembled rows: one thread per
// row segment, pairs in (row, panel) order.
__global__ void k_near_apply_rows(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                  const int* tri_cols, const int* col_dev, const double* row_scale,
                                  const int64_t* row_out, double* A) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  for (int p = seg_ptr[s]; p < seg_ptr[s + 1]; ++p) {
    const int r = pairs[2 * p], t = pairs[2 * p + 1];
    const double sc = row_scale[r];
    double* Arow = A + row_out[r];
    const int* tc = tri_cols + 3 * (size_t)t;
    for (int c = 0; c < 3; ++c) Arow[col_dev[tc[c]]] += sc * contrib[9 * (size_t)p + c];
  }
}

cudaError_t launch_near_pairs(const NearArgs& a, cudaStream_t st) {
  if (a.n_pairs == 0) return cudaSuccess;
  long long threads = a.n_pairs * 32;
  k_near_pairs<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_near_apply_rows(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                   const int* tri_cols, const int* col_dev, const double* row_scale,
                                   const int64_t* row_out, double* A, cudaStream_t st) {
  if (n_seg == 0) return cudaSuccess;
  k_near_apply_rows<<<(n_seg + 127) / 128, 128, 0, st>>>(seg_ptr, n_seg, pairs, contrib, tri_cols, col_dev,
                                                         row_scale, row_out, A);
  return cudaGetLastError();
}

}  // namespace hvb
