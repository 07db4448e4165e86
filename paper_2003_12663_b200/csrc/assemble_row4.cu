// Regular sweep (K2+K3), "row4" layout: lane = row (32 rows per warp), FOUR
// panel records per lane per step (four independent FP64 chains per lane).
// Unlike the quad layout every lane owns its window row exclusively, so the
// window adds need no half-warp serialisation; each node's data feeds one
// row instead of two (twice the shared-memory broadcast loads).  Same
// record stream, tiling guarantee (groups of 4), classification and
// summation order as the quad layout.
#include <cstdlib>

#include "launch.cuh"

namespace hvb {
namespace row4 {
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

// one (row, record) classification: regular iff ||x - cc|| > fl(eta R),
// decided as the reference rounds it.  The bracket test uses the 3-op FMA
// sum of squares: it is within 4 ulp of the unfused sum, far inside the
// bracket's 1e-13 margins, so it decides exactly as the unfused sum would;
// only a pair inside the bracket pays for the unfused sum and the IEEE sqrt.
HVB_DEV bool regular(d3 d, const double* cg) {
  const double sq = fma(d.z, d.z, fma(d.y, d.y, d.x * d.x));
  bool r = sq > cg[5];
  if (!r && !(sq < cg[4])) r = __dsqrt_rn(sumsq_unfused(d)) > cg[3];
  return r;
}
}  // namespace row4

template <int NQ, int MODE, int WIN, int R, int FLUSH, int WPC>
__global__ void __launch_bounds__(32 * WPC) k_assemble_row4(RegularArgs a) {
  using namespace row4;
  constexpr int REC = 6 * NQ + 8;
  constexpr int SREC = R * REC;
  constexpr int SLOTS = Shape<WIN>::SLOTS;
  constexpr int WREG = Shape<WIN>::WREG;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // WPC warps of the CTA take consecutive 32-row tiles of the SAME column
  // tile and share one record ring (staged by all threads, CTA barriers),
  // so the per-warp shared memory is the window plus 1/WPC of the ring
  double* ring = smem;
  double* win = smem + DEPTH * SREC + wib * WREG;

  const int rowtile = blockIdx.x * WPC + wib;
  const int tile = blockIdx.y;
  const int base_row = rowtile * ROWS;
  if (WPC == 1 && base_row >= a.n_rows) return;  // (WPC > 1: warps past the end stay for the barriers)

  const int i0 = base_row + lane;
  const bool live0 = i0 < a.n_rows;
  const int lr0 = a.row_begin + (live0 ? i0 : a.n_rows - 1);
  const double* rd0 = a.rowdata + 6 * (size_t)lr0;
  const d3 X0 = mk3(rd0[0], rd0[1], rd0[2]);
  const d3 N0 = mk3(rd0[3], rd0[4], rd0[5]);
  const bool adl0 = (MODE == 1) || (MODE == 2 && a.row_kind[lr0] == 1);
  const int own0 = a.row_col[lr0];
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
  const int ns = (ne + R - 1) / R;

  auto stage = [&](int p) {
    double* dst = ring + (p & 1) * SREC;
    const double* s = src + (size_t)(R * p) * REC;
    const int nrec = min(R, ne - R * p);
    const int nch = nrec * (REC / 2);
    for (int c = threadIdx.x; c < nch; c += 32 * WPC) cp_async16(dst + 2 * c, s + 2 * c);
  };
  stage(0);
  commit();

  int base = 0;
  // flush FLUSH finished columns: FLUSH = 16 -- lanes 0-15 write rows 0-15
  // and lanes 16-31 rows 16-31 of 16 consecutive columns (128-byte row
  // segments) -- so the window only needs band + 16 columns: a 48-column
  // window holds the band-32 tiling (1.14 redundancy)
  auto flush = [&](int b) {
    const int c = b + (FLUSH == 16 ? (lane & 15) : lane);
    double* wcol = win + (c % WIN) * STRIDE;
    const bool in = c < width;
    if (FLUSH == 16) {
      const int rh = (lane >> 4) * 16;
#pragma unroll 8
      for (int j = 0; j < 16; ++j) {
        const int row = rh + j;
        const int64_t off = __shfl_sync(0xffffffffu, fout, row);
        const double sc = __shfl_sync(0xffffffffu, fscale, row);
        if (off >= 0 && in) a.A[off + col0 + c] = wcol[row] * sc;
        wcol[row] = 0.0;
      }
    } else {
#pragma unroll 8
      for (int j = 0; j < ROWS; ++j) {
        const int64_t off = __shfl_sync(0xffffffffu, fout, j);
        const double sc = __shfl_sync(0xffffffffu, fscale, j);
        if (off >= 0 && in) a.A[off + col0 + c] = wcol[j] * sc;
        wcol[j] = 0.0;
      }
    }
    __syncwarp();
  };

  for (int p = 0; p < ns; ++p) {
    if (WPC > 1) __syncthreads();  // every warp is done with the slot stage(p + 1) overwrites
    if (p + 1 < ns) stage(p + 1);
    commit();
    wait_group<1>();
    if (WPC > 1)
      __syncthreads();
    else
      __syncwarp();
    const double* pr = ring + (p & 1) * SREC;
    const int mfirst = reinterpret_cast<const int*>(pr + 6 * NQ + 6)[1];
    while (mfirst >= base + FLUSH) {
      flush(base);
      base += FLUSH;
    }
    double acc[R][3];
#pragma unroll
    for (int j = 0; j < R; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const double* rec = pr + j * REC;
        const double2 p01 = *reinterpret_cast<const double2*>(rec + 6 * q);
        const double2 p2w = *reinterpret_cast<const double2*>(rec + 6 * q + 2);
        const double2 w12 = *reinterpret_cast<const double2*>(rec + 6 * q + 4);
        const double dx = X0.x - p01.x, dy = X0.y - p01.y, dz = X0.z - p2w.x;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        double k;
        if (MODE == 0) {  // 2/r: the flush applies the 1/2
          k = rsqrt2_newton(r2);
        } else {
          const double ri = rsqrt_full(r2);
          const double dn = fma(dz, N0.z, fma(dy, N0.y, dx * N0.x));
          const double t = dn * (ri * ri * ri);
          k = (MODE == 1) ? t : (adl0 ? t : ri);
        }
        acc[j][0] = fma(k, p2w.y, acc[j][0]);
        acc[j][1] = fma(k, w12.x, acc[j][1]);
        acc[j][2] = fma(k, w12.y, acc[j][2]);
      }
    }
    int slots[R][3];
    bool emit[R];
    int tris[R];
    bool any_emit = false;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double* cg = pr + j * REC + 6 * NQ;
      const bool valid = R * p + j < ne;
      const bool reg = row4::regular(sub_rn(X0, mk3(cg[0], cg[1], cg[2])), cg);
      if (!reg) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
      const int* meta = reinterpret_cast<const int*>(cg + 6);
      const unsigned sl = static_cast<unsigned>(meta[2]), sf = static_cast<unsigned>(meta[3]);
      slots[j][0] = valid ? (int)(sl & 0xffffu) : WIN;
      slots[j][1] = valid ? (int)(sl >> 16) : WIN;
      slots[j][2] = valid ? (int)(sf & 0xffffu) : WIN;
      const bool prim = valid && (sf >> 16) & 1u;
      tris[j] = valid ? meta[0] : 0;
      emit[j] = !reg && prim && live0;
      any_emit |= emit[j];
    }
    // deferred near pairs (rare): emitted from the panel's primary tile only
    if (__any_sync(0xffffffffu, any_emit)) {
      unsigned msk[R];
      int total = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int* tc = a.tri_cols + 3 * (size_t)tris[j];
        emit[j] = emit[j] && !(tc[0] == own0 || tc[1] == own0 || tc[2] == own0);
        msk[j] = __ballot_sync(0xffffffffu, emit[j]);
        total += __popc(msk[j]);
      }
      unsigned long long b = 0;
      if (lane == 0 && total) b = atomicAdd(a.near_count, (unsigned long long)total);
      b = __shfl_sync(0xffffffffu, b, 0);
      const unsigned lt = (1u << lane) - 1u;
      long long off = (long long)b;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (emit[j]) {
          const long long slot = off + __popc(msk[j] & lt);
          if (slot < a.near_cap) {
            a.near_list[2 * slot] = a.row_begin + i0;
            a.near_list[2 * slot + 1] = tris[j];
          }
        }
        off += __popc(msk[j]);
      }
    }
    // window adds in record order (each lane owns its row: no conflicts)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      win[slots[j][0] * STRIDE + lane] += acc[j][0];
      win[slots[j][1] * STRIDE + lane] += acc[j][1];
      win[slots[j][2] * STRIDE + lane] += acc[j][2];
    }
    __syncwarp();
  }
  wait_group<0>();
  __syncwarp();
  while (base < width) {
    flush(base);
    base += FLUSH;
  }
}

template <int WIN>
static size_t row4_smem_bytes(int nq, int r, int wpc) {
  return (size_t)(wpc * row4::Shape<WIN>::WREG + row4::DEPTH * r * (6 * nq + 8)) * sizeof(double);
}

template <int NQ, int WIN, int R, int FLUSH>
static cudaError_t launch_row4_nq(const RegularArgs& a, int mode, cudaStream_t st) {
  // warps per CTA sharing the record ring (HVB_ASM_WPC A/B; 4 by default)
  static const int wpc_env = [] {
    const char* e = getenv("HVB_ASM_WPC");
    return e ? atoi(e) : 4;
  }();
  auto run = [&](auto wpc_tag) -> cudaError_t {
    constexpr int WPC = decltype(wpc_tag)::value;
    dim3 grid((a.n_rows + row4::ROWS * WPC - 1) / (row4::ROWS * WPC), a.n_tiles);
    const size_t smem = row4_smem_bytes<WIN>(NQ, R, WPC);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, 32 * WPC, smem, st>>>(a);
      return cudaGetLastError();
    };
    if (mode == 0) return go(k_assemble_row4<NQ, 0, WIN, R, FLUSH, WPC>);
    if (mode == 1) return go(k_assemble_row4<NQ, 1, WIN, R, FLUSH, WPC>);
    return go(k_assemble_row4<NQ, 2, WIN, R, FLUSH, WPC>);
  };
  if (wpc_env == 1) return run(std::integral_constant<int, 1>{});
  if (wpc_env == 2) return run(std::integral_constant<int, 2>{});
  if (wpc_env == 8) return run(std::integral_constant<int, 8>{});
  return run(std::integral_constant<int, 4>{});
}

// window WIN, R records per lane per step, flush width 16 or 32: the
// stream's band (over groups of R records) must be <= WIN - flush
cudaError_t launch_regular_row4(const RegularArgs& a, int nq, int mode, int window, int r, int flush,
                                cudaStream_t st) {
  auto pick = [&](auto win_tag, auto r_tag, auto f_tag) -> cudaError_t {
    constexpr int W = decltype(win_tag)::value;
    constexpr int RR = decltype(r_tag)::value;
    constexpr int F = decltype(f_tag)::value;
    switch (nq) {
      case 3: return launch_row4_nq<3, W, RR, F>(a, mode, st);
      case 6: return launch_row4_nq<6, W, RR, F>(a, mode, st);
      case 12: return launch_row4_nq<12, W, RR, F>(a, mode, st);
      case 16: return launch_row4_nq<16, W, RR, F>(a, mode, st);
    }
    return cudaErrorInvalidValue;
  };
  using I4 = std::integral_constant<int, 4>;
  using F16 = std::integral_constant<int, 16>;
  using F32 = std::integral_constant<int, 32>;
  if (window == 48 && r == 4 && flush == 16) return pick(std::integral_constant<int, 48>{}, I4{}, F16{});
  if (window == 40 && r == 4 && flush == 16) return pick(std::integral_constant<int, 40>{}, I4{}, F16{});
  if (window == 44 && r == 4 && flush == 16) return pick(std::integral_constant<int, 44>{}, I4{}, F16{});
  if (window == 56 && r == 4 && flush == 16) return pick(std::integral_constant<int, 56>{}, I4{}, F16{});
  if (window == 48 && r == 4 && flush == 32) return pick(std::integral_constant<int, 48>{}, I4{}, F32{});
  if (window == 64 && r == 4 && flush == 32) return pick(std::integral_constant<int, 64>{}, I4{}, F32{});
  if (window == 64 && r == 8 && flush == 32) return pick(std::integral_constant<int, 64>{}, std::integral_constant<int, 8>{}, F32{});
  return cudaErrorInvalidValue;
}

}  // namespace hvb
