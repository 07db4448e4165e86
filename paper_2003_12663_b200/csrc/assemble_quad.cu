// Regular sweep (K2+K3), "quad" layout: every lane evaluates TWO panel
// records for TWO rows per step (four independent FP64 chains).
//
// A warp owns 32 rows (lane&15 and lane&15 + 16) and sweeps one column tile.
// A step consumes FOUR consecutive panel records of the tile: lanes 0-15
// take records 4p, 4p+1 and lanes 16-31 take records 4p+2, 4p+3.  Compared
// with the dual layout (assemble_dual.cu, one record per lane) the per-step
// control work (ring wait, flush test, slot unpack, near-pair vote, window
// synchronisation) is amortised over twice the node work and each lane has
// four chains in flight, with the same 32-row x WIN-column window.
//
// Window adds go record 4p, 4p+1, 4p+2, 4p+3 in that order, so every matrix
// entry is summed in a fixed order (bitwise reproducible, independent of the
// row blocking).  The host tiling guarantees that each aligned group of four
// records of a tile spans at most WIN - 32 columns from its first record's
// first owned column (device.py column_tiling, group=4).  Records are staged
// with cp.async, two steps deep (prefetch one step ahead).
//
// Classification, near-pair emission and kernel values are exactly those of
// the dual layout (see assemble_dual.cu and common.cuh).
#include "launch.cuh"

namespace hvb {
namespace quad {
constexpr int ROWS = 32;
constexpr int STRIDE = 33;
constexpr int DEPTH = 2;
template <int WIN>
struct Shape {
  static constexpr int SLOTS = WIN + 1;                    // + dump slot
  static constexpr int WREG = (SLOTS * STRIDE + 1) & ~1;   // 16-byte aligned region
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// one (row, record) classification: regular iff ||x - cc|| > fl(eta R)
HVB_DEV bool regular(double sq, const double* cg) {
  bool r = sq > cg[5];
  if (!r && !(sq < cg[4])) r = __dsqrt_rn(sq) > cg[3];
  return r;
}
}  // namespace quad

template <int NQ, int MODE, int WIN>
__global__ void __launch_bounds__(32) k_assemble_quad(RegularArgs a) {
  using namespace quad;
  constexpr int REC = 6 * NQ + 8;
  constexpr int SREC = 4 * REC;
  constexpr int SLOTS = Shape<WIN>::SLOTS;
  constexpr int WREG = Shape<WIN>::WREG;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int rl = lane & 15;
  const int half = lane >> 4;
  double* win = smem;
  double* ring = win + WREG;

  const int rowtile = blockIdx.x;
  const int tile = blockIdx.y;
  const int base_row = rowtile * ROWS;
  if (base_row >= a.n_rows) return;

  const int i0 = base_row + rl, i1 = base_row + rl + 16;
  const bool live0 = i0 < a.n_rows, live1 = i1 < a.n_rows;
  const int lr0 = a.row_begin + (live0 ? i0 : a.n_rows - 1);
  const int lr1 = a.row_begin + (live1 ? i1 : a.n_rows - 1);
  const double* rd0 = a.rowdata + 6 * (size_t)lr0;
  const double* rd1 = a.rowdata + 6 * (size_t)lr1;
  const d3 X0 = mk3(rd0[0], rd0[1], rd0[2]);
  const d3 X1 = mk3(rd1[0], rd1[1], rd1[2]);
  const d3 N0 = mk3(rd0[3], rd0[4], rd0[5]);
  const d3 N1 = mk3(rd1[3], rd1[4], rd1[5]);
  const bool adl0 = (MODE == 1) || (MODE == 2 && a.row_kind[lr0] == 1);
  const bool adl1 = (MODE == 1) || (MODE == 2 && a.row_kind[lr1] == 1);
  const int own0 = a.row_col[lr0], own1 = a.row_col[lr1];
  const int fi = base_row + lane;
  const bool flive = fi < a.n_rows;
  const int flr = a.row_begin + (flive ? fi : a.n_rows - 1);
  const int64_t fout = flive ? a.row_out[flr] : -1;
  const double fscale = a.row_scale[flr] * (MODE == 0 ? 0.5 : 1.0);  // SL sums hold 2/r (exact halving)

  for (int k = lane; k < SLOTS * STRIDE; k += 32) win[k] = 0.0;

  const int64_t e0 = a.tile_ptr[tile], e1 = a.tile_ptr[tile + 1];
  const int col0 = a.tile_col0[tile], width = a.tile_width[tile];
  const double* src = a.stream + e0 * REC;
  const int ne = (int)(e1 - e0);
  const int ns = (ne + 3) >> 2;

  auto stage = [&](int p) {
    double* dst = ring + (p & 1) * SREC;
    const double* s = src + (size_t)(4 * p) * REC;
    const int nrec = min(4, ne - 4 * p);
    const int nch = nrec * (REC / 2);
    for (int c = lane; c < nch; c += 32) cp_async16(dst + 2 * c, s + 2 * c);
  };
  stage(0);
  commit();

  int base = 0;
  auto flush32 = [&](int b) {
    const int c = b + lane;
    double* wcol = win + (c % WIN) * STRIDE;
    const bool in = c < width;
#pragma unroll 8
    for (int j = 0; j < ROWS; ++j) {
      const int64_t off = __shfl_sync(0xffffffffu, fout, j);
      const double sc = __shfl_sync(0xffffffffu, fscale, j);
      if (off >= 0 && in) a.A[off + col0 + c] = wcol[j] * sc;
      wcol[j] = 0.0;
    }
    __syncwarp();
  };

  for (int p = 0; p < ns; ++p) {
    if (p + 1 < ns) stage(p + 1);
    commit();
    wait_group<1>();
    __syncwarp();
    const double* pr = ring + (p & 1) * SREC;
    const int mfirst = reinterpret_cast<const int*>(pr + 6 * NQ + 6)[1];
    while (mfirst >= base + 32) {
      flush32(base);
      base += 32;
    }
    const int r0 = 4 * p + 2 * half;  // this lane's first record index in the tile
    const double* recA = pr + (2 * half) * REC;
    const double* recB = recA + REC;
    const double* cgA = recA + 6 * NQ;
    const double* cgB = recB + 6 * NQ;
    const bool validA = r0 < ne, validB = r0 + 1 < ne;

    // accumulators: [record][row][corner]
    double aA0 = 0.0, aA1 = 0.0, aA2 = 0.0, bA0 = 0.0, bA1 = 0.0, bA2 = 0.0;  // record A, rows 0 / 1
    double aB0 = 0.0, aB1 = 0.0, aB2 = 0.0, bB0 = 0.0, bB1 = 0.0, bB2 = 0.0;  // record B, rows 0 / 1
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double2 pA01 = *reinterpret_cast<const double2*>(recA + 6 * q);
      const double2 pA2w = *reinterpret_cast<const double2*>(recA + 6 * q + 2);
      const double2 wA12 = *reinterpret_cast<const double2*>(recA + 6 * q + 4);
      const double2 pB01 = *reinterpret_cast<const double2*>(recB + 6 * q);
      const double2 pB2w = *reinterpret_cast<const double2*>(recB + 6 * q + 2);
      const double2 wB12 = *reinterpret_cast<const double2*>(recB + 6 * q + 4);
      const double dxA0 = X0.x - pA01.x, dyA0 = X0.y - pA01.y, dzA0 = X0.z - pA2w.x;
      const double dxA1 = X1.x - pA01.x, dyA1 = X1.y - pA01.y, dzA1 = X1.z - pA2w.x;
      const double dxB0 = X0.x - pB01.x, dyB0 = X0.y - pB01.y, dzB0 = X0.z - pB2w.x;
      const double dxB1 = X1.x - pB01.x, dyB1 = X1.y - pB01.y, dzB1 = X1.z - pB2w.x;
      const double rA0 = fma(dzA0, dzA0, fma(dyA0, dyA0, dxA0 * dxA0));
      const double rA1 = fma(dzA1, dzA1, fma(dyA1, dyA1, dxA1 * dxA1));
      const double rB0 = fma(dzB0, dzB0, fma(dyB0, dyB0, dxB0 * dxB0));
      const double rB1 = fma(dzB1, dzB1, fma(dyB1, dyB1, dxB1 * dxB1));
      double kA0, kA1, kB0, kB1;
      if (MODE == 0) {  // 2/r: the flush applies the 1/2
        kA0 = rsqrt2_newton(rA0);
        kA1 = rsqrt2_newton(rA1);
        kB0 = rsqrt2_newton(rB0);
        kB1 = rsqrt2_newton(rB1);
      } else {
        const double iA0 = rsqrt_full(rA0), iA1 = rsqrt_full(rA1);
        const double iB0 = rsqrt_full(rB0), iB1 = rsqrt_full(rB1);
        const double nA0 = fma(dzA0, N0.z, fma(dyA0, N0.y, dxA0 * N0.x));
        const double nA1 = fma(dzA1, N1.z, fma(dyA1, N1.y, dxA1 * N1.x));
        const double nB0 = fma(dzB0, N0.z, fma(dyB0, N0.y, dxB0 * N0.x));
        const double nB1 = fma(dzB1, N1.z, fma(dyB1, N1.y, dxB1 * N1.x));
        const double tA0 = nA0 * (iA0 * iA0 * iA0), tA1 = nA1 * (iA1 * iA1 * iA1);
        const double tB0 = nB0 * (iB0 * iB0 * iB0), tB1 = nB1 * (iB1 * iB1 * iB1);
        kA0 = (MODE == 1) ? tA0 : (adl0 ? tA0 : iA0);
        kA1 = (MODE == 1) ? tA1 : (adl1 ? tA1 : iA1);
        kB0 = (MODE == 1) ? tB0 : (adl0 ? tB0 : iB0);
        kB1 = (MODE == 1) ? tB1 : (adl1 ? tB1 : iB1);
      }
      aA0 = fma(kA0, pA2w.y, aA0);
      aA1 = fma(kA0, wA12.x, aA1);
      aA2 = fma(kA0, wA12.y, aA2);
      bA0 = fma(kA1, pA2w.y, bA0);
      bA1 = fma(kA1, wA12.x, bA1);
      bA2 = fma(kA1, wA12.y, bA2);
      aB0 = fma(kB0, pB2w.y, aB0);
      aB1 = fma(kB0, wB12.x, aB1);
      aB2 = fma(kB0, wB12.y, aB2);
      bB0 = fma(kB1, pB2w.y, bB0);
      bB1 = fma(kB1, wB12.x, bB1);
      bB2 = fma(kB1, wB12.y, bB2);
    }
    const bool regA0 = regular(sumsq_unfused(sub_rn(X0, mk3(cgA[0], cgA[1], cgA[2]))), cgA);
    const bool regA1 = regular(sumsq_unfused(sub_rn(X1, mk3(cgA[0], cgA[1], cgA[2]))), cgA);
    const bool regB0 = regular(sumsq_unfused(sub_rn(X0, mk3(cgB[0], cgB[1], cgB[2]))), cgB);
    const bool regB1 = regular(sumsq_unfused(sub_rn(X1, mk3(cgB[0], cgB[1], cgB[2]))), cgB);
    if (!regA0) aA0 = aA1 = aA2 = 0.0;
    if (!regA1) bA0 = bA1 = bA2 = 0.0;
    if (!regB0) aB0 = aB1 = aB2 = 0.0;
    if (!regB1) bB0 = bB1 = bB2 = 0.0;

    const int* metaA = reinterpret_cast<const int*>(cgA + 6);
    const int* metaB = reinterpret_cast<const int*>(cgB + 6);
    const unsigned slA = static_cast<unsigned>(metaA[2]), sfA = static_cast<unsigned>(metaA[3]);
    const unsigned slB = static_cast<unsigned>(metaB[2]), sfB = static_cast<unsigned>(metaB[3]);
    const int sA0 = validA ? (int)(slA & 0xffffu) : WIN;
    const int sA1 = validA ? (int)(slA >> 16) : WIN;
    const int sA2 = validA ? (int)(sfA & 0xffffu) : WIN;
    const int sB0 = validB ? (int)(slB & 0xffffu) : WIN;
    const int sB1 = validB ? (int)(slB >> 16) : WIN;
    const int sB2 = validB ? (int)(sfB & 0xffffu) : WIN;
    const bool primA = validA && (sfA >> 16) & 1u;
    const bool primB = validB && (sfB >> 16) & 1u;

    // deferred near pairs (rare): emitted from the panel's primary tile only
    const bool nA0 = !regA0 && primA && live0, nA1 = !regA1 && primA && live1;
    const bool nB0 = !regB0 && primB && live0, nB1 = !regB1 && primB && live1;
    if (__any_sync(0xffffffffu, nA0 || nA1 || nB0 || nB1)) {
      const int triA = metaA[0], triB = metaB[0];
      const int* tcA = a.tri_cols + 3 * (size_t)(validA ? triA : 0);
      const int* tcB = a.tri_cols + 3 * (size_t)(validB ? triB : 0);
      const bool eA0 = nA0 && !(tcA[0] == own0 || tcA[1] == own0 || tcA[2] == own0);
      const bool eA1 = nA1 && !(tcA[0] == own1 || tcA[1] == own1 || tcA[2] == own1);
      const bool eB0 = nB0 && !(tcB[0] == own0 || tcB[1] == own0 || tcB[2] == own0);
      const bool eB1 = nB1 && !(tcB[0] == own1 || tcB[1] == own1 || tcB[2] == own1);
      const unsigned mA0 = __ballot_sync(0xffffffffu, eA0), mA1 = __ballot_sync(0xffffffffu, eA1);
      const unsigned mB0 = __ballot_sync(0xffffffffu, eB0), mB1 = __ballot_sync(0xffffffffu, eB1);
      const int total = __popc(mA0) + __popc(mA1) + __popc(mB0) + __popc(mB1);
      unsigned long long b = 0;
      if (lane == 0 && total) b = atomicAdd(a.near_count, (unsigned long long)total);
      b = __shfl_sync(0xffffffffu, b, 0);
      const unsigned lt = (1u << lane) - 1u;
      long long off = (long long)b;
      auto put = [&](bool e, unsigned msk, int row, int tri) {
        if (e) {
          const long long slot = off + __popc(msk & lt);
          if (slot < a.near_cap) {
            a.near_list[2 * slot] = a.row_begin + row;
            a.near_list[2 * slot + 1] = tri;
          }
        }
        off += __popc(msk);
      };
      put(eA0, mA0, i0, triA);
      put(eA1, mA1, i1, triA);
      put(eB0, mB0, i0, triB);
      put(eB1, mB1, i1, triB);
    }

    // window adds in record order 4p, 4p+1 (lanes 0-15), 4p+2, 4p+3 (16-31)
    double* wA0 = win + sA0 * STRIDE + rl;
    double* wA1 = win + sA1 * STRIDE + rl;
    double* wA2 = win + sA2 * STRIDE + rl;
    double* wB0 = win + sB0 * STRIDE + rl;
    double* wB1 = win + sB1 * STRIDE + rl;
    double* wB2 = win + sB2 * STRIDE + rl;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (half == s) {
        wA0[0] += aA0;
        wA0[16] += bA0;
        wA1[0] += aA1;
        wA1[16] += bA1;
        wA2[0] += aA2;
        wA2[16] += bA2;
        wB0[0] += aB0;
        wB0[16] += bB0;
        wB1[0] += aB1;
        wB1[16] += bB1;
        wB2[0] += aB2;
        wB2[16] += bB2;
      }
      __syncwarp();
    }
  }
  wait_group<0>();
  __syncwarp();
  while (base < width) {
    flush32(base);
    base += 32;
  }
}

template <int WIN>
static size_t quad_smem_bytes(int nq) {
  return (size_t)(quad::Shape<WIN>::WREG + quad::DEPTH * 4 * (6 * nq + 8)) * sizeof(double);
}

template <int NQ, int WIN>
static cudaError_t launch_quad_nq(const RegularArgs& a, int mode, cudaStream_t st) {
  dim3 grid((a.n_rows + quad::ROWS - 1) / quad::ROWS, a.n_tiles);
  const size_t smem = quad_smem_bytes<WIN>(NQ);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32, smem, st>>>(a);
    return cudaGetLastError();
  };
  if (mode == 0) return go(k_assemble_quad<NQ, 0, WIN>);
  if (mode == 1) return go(k_assemble_quad<NQ, 1, WIN>);
  return go(k_assemble_quad<NQ, 2, WIN>);
}

// window 64 (group-of-4 band <= 32) or 96 (<= 64)
cudaError_t launch_regular_quad(const RegularArgs& a, int nq, int mode, int window, cudaStream_t st) {
  auto pick = [&](auto win_tag) -> cudaError_t {
    constexpr int W = decltype(win_tag)::value;
    switch (nq) {
      case 3: return launch_quad_nq<3, W>(a, mode, st);
      case 6: return launch_quad_nq<6, W>(a, mode, st);
      case 12: return launch_quad_nq<12, W>(a, mode, st);
      case 16: return launch_quad_nq<16, W>(a, mode, st);
    }
    return cudaErrorInvalidValue;
  };
  if (window == 64) return pick(std::integral_constant<int, 64>{});
  if (window == 96) return pick(std::integral_constant<int, 96>{});
  return cudaErrorInvalidValue;
}

}  // namespace hvb
