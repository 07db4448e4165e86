// Regular sweep (K2+K3 of SURVEY 2.2): reference row_pass1's regular pass
// (src/assembly.py:155-200) for a tile of rows x one column tile.
//
// Work split.  A CTA owns WPC x 32 rows (lane = row) and one column tile;
// its warps share one ring of panel records, staged by the bulk-copy engine
// (cp.async.bulk, one copy of R = 4 consecutive records per stage, completion
// on an mbarrier).  A stage is refilled by the LAST warp that releases it (a
// shared-memory counter), so warps are not lock-stepped by CTA barriers and
// drift up to S stages apart.  Every lane evaluates all R records of a stage
// for its row (R independent FP64 chains), adds the three corner sums into
// its row of a WIN-column shared-memory window of the tile's local columns
// (record order: no atomics, bitwise reproducible) and finished groups of
// FLUSH columns are flushed once: owned columns to A, halo copies and the
// partials of receiving columns to exchange slots, summed after the sweep
// by the last CTA (of the owner and its producers, same rows) to finish
// (csrc/tiling.cpp 5).
//
// Record formats (csrc/tables.cu k_build_stream):
//  * SL (MODE 0): per node pair 10 doubles [Yx0 Yy0 | Yz0 P0 | Q0 Q1 | Yx1 Yy1
//    | Yz1 P1] with, per node q of panel t (cc = circumcentre, w = jw/4pi):
//      s = 1/w^2,  Y = -2 s (y - cc),  P = s |y - cc|^2,  Q = s.
//    With x' = x - cc (computed anyway for the classification) and X = |x'|^2
//      r2' = x'.Y + X Q + P = s |x - y|^2 = (|x - y| / w)^2     (4 DFMA)
//    and rsqrt2(r2') = 2 w / |x - y| (MUFU seed + 3 ops), so a node costs 10
//    FP64 ops instead of 12: the hat functions hat_c(q) are kernel-parameter
//    constants.  Regular pairs have |x'| > 1.2 R >= |y - cc| + 0.2 R, so the
//    expansion loses at most ~120 ulp of r2 (~3e-14 relative).
//  * ADL (MODE 1): per node 6 doubles (y, w hat_0, w hat_1, w hat_2).
// Both end in an 8-double tail: cc, fl(eta R), bracket lo/hi, panel id,
// first local column, window byte offsets of the 3 corners, flags.  Stages
// are built by csrc/tiling.cpp: the corners of one stage are distinct local
// columns (short stages padded with dummy records), so a stage updates the
// window with 12 independent read-modify-writes.
#include <cstdint>

#include "launch.cuh"

// Geometry (compile-time; hvb_sweep_geometry reports it to the host, which
// builds the tiling with band = WIN - FLUSH and stages of R records).
#ifndef HVB_SWEEP_WIN
#define HVB_SWEEP_WIN 64
#endif
#ifndef HVB_SWEEP_FLUSH
#define HVB_SWEEP_FLUSH 16
#endif
#ifndef HVB_SWEEP_WPC
#define HVB_SWEEP_WPC 4
#endif
#ifndef HVB_SWEEP_MINB
#define HVB_SWEEP_MINB 3
#endif

namespace hvb {
namespace sweep {
constexpr int ROWS = 32;
constexpr int STRIDE = 33;
constexpr int WIN = HVB_SWEEP_WIN;                       // window columns
constexpr int SLOTS = WIN + 1;                           // + dump slot
constexpr int WREG = (SLOTS * STRIDE + 1) & ~1;          // doubles per warp window (16-byte aligned)
constexpr int FLUSH = HVB_SWEEP_FLUSH;                   // columns per flush (band <= WIN - FLUSH)
constexpr int R = 4;                                     // records per stage
constexpr int WPC = HVB_SWEEP_WPC;                       // warps per CTA
constexpr int MINB = HVB_SWEEP_MINB;                     // resident CTAs per SM (register budget)
constexpr size_t kSmemBudget = 232448;                   // 227 KB per SM usable by CTAs

template <int NQ, int MODE>
struct Rec {
  static constexpr int NQP = MODE == 0 ? (NQ + 1) & ~1 : NQ;  // SL: node pairs (odd NQ padded)
  static constexpr int DOUBLES = (MODE == 0 ? 5 : 6) * NQP + 8;
  static constexpr int TAIL = DOUBLES - 8;
  // ring stages: as many (<= 4) as fit MINB CTAs per SM
  static constexpr size_t kWin = (size_t)WPC * WREG * 8;
  static constexpr size_t kStage = (size_t)R * DOUBLES * 8 + 16;
  static constexpr int kFit = (int)((kSmemBudget / MINB - 1024 - kWin) / kStage);
  static constexpr int S = kFit > 4 ? 4 : (kFit < 2 ? 2 : kFit);
};

HVB_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

HVB_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

HVB_DEV void mbar_wait(uint64_t* bar, unsigned phase) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 100000;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

// bulk copy global -> shared (the TMA engine's 1-D mode), completing on bar
HVB_DEV void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// hat_c(q) of the regular rule per nq in {3, 6, 12, 16} (index 0..3):
// constant bank operands of the SL node FMAs (uploaded once per device by
// launch_regular; the values depend on nq only)
__constant__ double c_hats[4][16][3];

__host__ __device__ constexpr int hat_index(int nq) { return nq == 3 ? 0 : nq == 6 ? 1 : nq == 12 ? 2 : 3; }
}  // namespace sweep

// RED (charge-reduce mode, MODE 1 only): instead of one row per lane, the
// flush writes the scaled sum over the warp's 32 rows of every column into
// the tile's partial row a.A + tile * a.part_ld (csrc/tables.cu
// k_charge_reduce then sums the partial rows in order).
template <int NQ, int MODE, bool RED = false>
__global__ void __launch_bounds__(32 * sweep::WPC, sweep::MINB) k_sweep(RegularArgs a) {
  using namespace sweep;
  using RC = Rec<NQ, MODE>;
  constexpr int REC = RC::DOUBLES;
  constexpr int S = RC::S;
  extern __shared__ __align__(16) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);         // S mbarriers
  unsigned* released = reinterpret_cast<unsigned*>(smem + S);  // S release counters
  double* ring = smem + 2 * S;                                 // S x R x REC
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double* win = ring + S * R * REC + wib * WREG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      released[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrb = gridDim.x;
  const int rb = blockIdx.x, tile = a.tile_order ? a.tile_order[blockIdx.y] : (int)blockIdx.y;
  const int cta_row0 = rb * (WPC * ROWS);
  const int live_warps = min(WPC, (a.n_rows - cta_row0 + ROWS - 1) / ROWS);
  const int64_t e0 = a.tile_ptr[tile], e1 = a.tile_ptr[tile + 1];
  const int lp0 = a.tile_lptr[tile], width = a.tile_lptr[tile + 1] - lp0;
  const double* src = a.stream + e0 * REC;
  const int ne = (int)(e1 - e0);
  const int ns = (ne + R - 1) / R;

  auto issue = [&](int p) {  // one thread: stage p of this tile into ring slot p % S
    const int nrec = min(R, ne - R * p);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    bulk_load(ring + (p % S) * (R * REC), src + (size_t)(R * p) * REC, (unsigned)(nrec * REC * 8), full + p % S);
  };
  if (threadIdx.x == 0)
    for (int p = 0; p < min(S, ns); ++p) issue(p);
  if (wib >= live_warps) return;  // no live rows: this warp takes no part in the ring

  const int base_row = cta_row0 + wib * ROWS;
  const int i0 = base_row + lane;
  const bool live0 = i0 < a.n_rows;
  const int lr0 = a.row_begin + (live0 ? i0 : a.n_rows - 1);
  const double* rd0 = a.rowdata + 6 * (size_t)lr0;
  const d3 X0 = mk3(rd0[0], rd0[1], rd0[2]);
  const d3 N0 = mk3(rd0[3], rd0[4], rd0[5]);
  const int own0 = a.row_col[lr0];
  const int64_t fout = live0 ? (RED ? 0 : a.row_out[lr0]) : -1;
  const double fscale = live0 ? a.row_scale[lr0] * (MODE == 0 ? 0.5 : 1.0) : 0.0;  // SL sums hold 2w/r
  double* const part = RED ? a.A + (int64_t)((a.row_begin + base_row) / ROWS) * a.part_ld : nullptr;
  double* const halo = a.halo + base_row;  // + slot * n_rows + row

  for (int k = lane; k < SLOTS * STRIDE; k += 32) win[k] = 0.0;
  // each row's output offset and scale in the window's pad doubles (column
  // slot r / 32 + r, element 32: never touched by the sums), read by the
  // flush as shared-memory broadcasts instead of four shuffles per row
  // (branch-free stores + these: 237.5 -> 231.6 ms at cfg4)
  constexpr bool PADS = WIN >= 64 && STRIDE == 33;  // else: shuffles
  __syncwarp();
  if (PADS) {
    win[lane * STRIDE + 32] = __longlong_as_double((long long)fout);
    win[(32 + lane) * STRIDE + 32] = fscale;
  }
  __syncwarp();
  auto row_off = [&](int row) -> int64_t {
    return PADS ? __double_as_longlong(win[row * STRIDE + 32]) : __shfl_sync(0xffffffffu, fout, row);
  };
  auto row_scale = [&](int row) -> double {
    return PADS ? win[(32 + row) * STRIDE + 32] : __shfl_sync(0xffffffffu, fscale, row);
  };

  int base = 0;
  // flush FLUSH finished columns: lane l writes rows (l / FLUSH) * FLUSH ..
  // + FLUSH - 1 of local column b + l % FLUSH -- an owned column to its
  // device column of A (row segments of consecutive device columns), a
  // halo copy or a receiving column's partial raw to its slot.  The window
  // only needs band + FLUSH columns.
  auto flush = [&](int b) {
    const int c = b + (lane & (FLUSH - 1));
    double* wcol = win + (c % WIN) * STRIDE;
    const bool in = c < width;
    const int dst = in ? a.lcol[lp0 + c] : 0;
    double* const hcol = halo + (size_t)(dst < 0 ? ~dst : 0) * a.n_rows;
    const int rh = (lane / FLUSH) * FLUSH;  // FLUSH rows per lane
    if (RED) {
      double sum = 0.0;  // rows rh .. rh+FLUSH-1 in order, then the row groups
#pragma unroll 8
      for (int j = 0; j < FLUSH; ++j) {
        const int row = rh + j;
        const double v = wcol[row];
        const int64_t off = row_off(row);
        sum = fma(v, row_scale(row), sum);
        if (dst < 0 && in && off >= 0) hcol[row] = v;
        wcol[row] = 0.0;
      }
#pragma unroll
      for (int o = FLUSH; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane < FLUSH && in && dst >= 0) part[dst] = sum;
    } else {
      // branch-free: an owned column's entry goes to A[off + dst] scaled, a
      // slot's to hcol[row] raw -- one predicated store per row
      const bool own = dst >= 0;
      double* const colp = own ? a.A + dst : hcol;
#pragma unroll
      for (int j = 0; j < FLUSH; ++j) {
        const int row = rh + j;
        const int64_t off = row_off(row);
        const double sc = row_scale(row);
        const double v = wcol[row];
        wcol[row] = 0.0;
        if (off >= 0 && in) colp[own ? off : row] = own ? v * sc : v;
      }
    }
    __syncwarp();
  };

  char* const winl = reinterpret_cast<char*>(win) + 8 * lane;  // this lane's row of the window
  for (int p = 0; p < ns; ++p) {
    const int s = p % S;
    sweep::mbar_wait(full + s, (unsigned)(p / S) & 1u);
    const double* pr = ring + s * (R * REC);
    const int mfirst = reinterpret_cast<const int*>(pr + RC::TAIL + 6)[1];
    while (mfirst >= base + FLUSH) {
      flush(base);
      base += FLUSH;
    }
    // per record: x' = x - cc (IEEE, also the classification's difference),
    // the classification, the window byte offsets of its corners
    d3 xc[R];
    double sq[R];
    bool reg[R], amb[R], emit[R];
    int tris[R];
    unsigned slw[R], sfw[R];  // packed window byte offsets (+ flags)
    bool any_emit = false;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double* tl = pr + j * REC + RC::TAIL;
      xc[j] = sub_rn(X0, mk3(tl[0], tl[1], tl[2]));
      sq[j] = fma(xc[j].z, xc[j].z, fma(xc[j].y, xc[j].y, xc[j].x * xc[j].x));
      // classification: regular iff ||x - cc|| > fl(eta R), decided as the
      // reference rounds it.  sq is the 3-op FMA sum of squares (within 4 ulp
      // of the unfused sum, far inside the bracket's 1e-13 margins, so the
      // bracket decides as the unfused sum would); pairs inside the bracket
      // are settled below with the unfused sum and the IEEE sqrt
      reg[j] = sq[j] > tl[5];
      amb[j] = !reg[j] && !(sq[j] < tl[4]);
      const int* meta = reinterpret_cast<const int*>(tl + 6);
      slw[j] = static_cast<unsigned>(meta[2]);
      sfw[j] = static_cast<unsigned>(meta[3]);
      tris[j] = meta[0];
    }
    if (__any_sync(0xffffffffu, amb[0] || amb[1] || amb[2] || amb[3])) {  // rare: one uniform branch per stage
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (amb[j]) reg[j] = __dsqrt_rn(sumsq_unfused(xc[j])) > pr[j * REC + RC::TAIL + 3];
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      emit[j] = !reg[j] && ((sfw[j] >> 16) & 1u) && live0;  // from the panel's primary tile only
      any_emit |= emit[j];
    }
    double acc[R][3];
#pragma unroll
    for (int j = 0; j < R; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0.0;
    if (MODE == 0) {
#pragma unroll
      for (int q = 0; q < RC::NQP; q += 2) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const double* nd = pr + j * REC + 5 * q;
          const double2 y01 = *reinterpret_cast<const double2*>(nd);
          const double2 y2p = *reinterpret_cast<const double2*>(nd + 2);
          const double2 qq = *reinterpret_cast<const double2*>(nd + 4);
          const double2 z01 = *reinterpret_cast<const double2*>(nd + 6);
          const double2 z2p = *reinterpret_cast<const double2*>(nd + 8);
          const double r0 = fma(xc[j].x, y01.x, fma(xc[j].y, y01.y, fma(xc[j].z, y2p.x, fma(sq[j], qq.x, y2p.y))));
          const double r1 = fma(xc[j].x, z01.x, fma(xc[j].y, z01.y, fma(xc[j].z, z2p.x, fma(sq[j], qq.y, z2p.y))));
          const double k0 = rsqrt2_newton(r0);
          const double k1 = rsqrt2_newton(r1);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            acc[j][c] = fma(k0, c_hats[hat_index(NQ)][q][c], acc[j][c]);
            acc[j][c] = fma(k1, c_hats[hat_index(NQ)][q + 1][c], acc[j][c]);
          }
        }
      }
    } else {
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
          const double ri = rsqrt_full(r2);
          const double dn = fma(dz, N0.z, fma(dy, N0.y, dx * N0.x));
          const double k = dn * (ri * ri * ri);
          acc[j][0] = fma(k, p2w.y, acc[j][0]);
          acc[j][1] = fma(k, w12.x, acc[j][1]);
          acc[j][2] = fma(k, w12.y, acc[j][2]);
        }
      }
    }
    __syncwarp();
    // this warp is done reading the stage: the last warp to release it
    // refills it with stage p + S (every ring value this warp loaded has
    // been consumed by instructions issued before the release)
    if (lane == 0) {
      unsigned old;
      asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(old)
                   : "r"(sweep::smem_u32(released + s))
                   : "memory");
      if (old == (unsigned)live_warps - 1u) {
        released[s] = 0;
        if (p + S < ns) issue(p + S);
      }
    }
    // deferred near pairs (rare)
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
    // window update of the whole stage at once: the stage's corners are
    // distinct local columns (csrc/tiling.cpp), so the 12 read-modify-writes
    // are independent; only the never-flushed dump column (dummies) may collide
    double wv[R][3];
    int offs[R][3];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      offs[j][0] = (int)(slw[j] & 0xffffu);
      offs[j][1] = (int)(slw[j] >> 16);
      offs[j][2] = (int)(sfw[j] & 0xffffu);
#pragma unroll
      for (int c = 0; c < 3; ++c) wv[j][c] = *reinterpret_cast<const double*>(winl + offs[j][c]);
    }
    if (__all_sync(0xffffffffu, reg[0] && reg[1] && reg[2] && reg[3])) {  // the common case
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c) *reinterpret_cast<double*>(winl + offs[j][c]) = wv[j][c] + acc[j][c];
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          *reinterpret_cast<double*>(winl + offs[j][c]) = reg[j] ? wv[j][c] + acc[j][c] : wv[j][c];
    }
    __syncwarp();
  }
  while (base < width) {
    flush(base);
    base += FLUSH;
  }
  // completion: every lane fences its own slot writes, the live warps meet
  // and warp 0 counts this CTA in for its own tile and for every tile
  // importing its halo copies.  The CTA that completes a tile's count (its
  // partials and all copies of its receiving columns written, same rows)
  // performs that tile's exchange -- nobody waits.
  __shared__ int s_todo[32];
  __shared__ int s_ntodo;
  __threadfence();
  asm volatile("bar.sync 1, %0;" ::"r"(live_warps * 32) : "memory");
  const int cb = a.tile_cptr[tile], nc = a.tile_cptr[tile + 1] - cb;
  for (int i0 = 0; i0 <= nc; i0 += 32) {  // this tile, then its consumers, 32 at a time
    if (wib == 0) {
      const int i = i0 + lane;
      bool done = false;
      int t = 0;
      if (i <= nc) {
        t = i == 0 ? tile : a.cons[cb + i - 1];
        const int need = 1 + a.tile_pptr[t + 1] - a.tile_pptr[t];
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.sched + t * nrb + rb) : "memory");
        done = old == need - 1;
      }
      const unsigned m = __ballot_sync(0xffffffffu, done);
      if (done) s_todo[__popc(m & ((1u << lane) - 1u))] = t;
      __threadfence();
      if (lane == 0) s_ntodo = __popc(m);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(live_warps * 32) : "memory");

    // exchange of tile t: every receiving column = its partial + the halo
    // copies of earlier tiles (producer order), scaled and written once;
    // lane = row, 32 slots loaded per round trip
    const int ntodo = s_ntodo;
    for (int k = 0; k < ntodo; ++k) {
      const int t = s_todo[k];
      const int xb = a.tile_xptr[t], xe = a.tile_xptr[t + 1];
      double acc = 0.0;
      for (int x0 = xb; x0 < xe; x0 += 32) {
        const int nb = min(32, xe - x0);
        const int4 mine = a.xent[x0 + min(lane, nb - 1)];  // lane j holds entry x0 + j
        double h[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int slot = __shfl_sync(0xffffffffu, mine.x, j);
          h[j] = (j < nb && live0) ? __ldcg(halo + (size_t)slot * a.n_rows + lane) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < nb) {  // warp-uniform
            const int dcol = __shfl_sync(0xffffffffu, mine.y, j);
            const int first = __shfl_sync(0xffffffffu, mine.z, j);
            const int last = __shfl_sync(0xffffffffu, mine.w, j);
            acc = first ? h[j] : acc + h[j];
            if (last) {
              if (RED) {
                double v = acc * fscale;
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) part[dcol] = v;
              } else if (live0) {
                a.A[fout + dcol] = acc * fscale;
              }
            }
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(live_warps * 32) : "memory");  // s_todo is rewritten next
  }
}

// scheduling words of one launch: one completion counter per (row block,
// tile)
size_t sweep_sched_ints(int n_rows, int n_tiles) {
  return (size_t)n_tiles * ((n_rows + sweep::ROWS * sweep::WPC - 1) / (sweep::ROWS * sweep::WPC));
}

template <int NQ, int MODE, bool RED = false>
static cudaError_t launch_sweep_nq(const RegularArgs& a, cudaStream_t st) {
  using namespace sweep;
  constexpr int S = Rec<NQ, MODE>::S;
  const size_t smem = (size_t)(2 * S + S * R * Rec<NQ, MODE>::DOUBLES + WPC * WREG) * sizeof(double);
  static bool init = false;
  if (!init) {
    cudaError_t e =
        cudaFuncSetAttribute(k_sweep<NQ, MODE, RED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    init = true;
  }
  const int nrb = (a.n_rows + ROWS * WPC - 1) / (ROWS * WPC);
  cudaError_t e = cudaMemsetAsync(a.sched, 0, sweep_sched_ints(a.n_rows, a.n_tiles) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  k_sweep<NQ, MODE, RED><<<dim3(nrb, a.n_tiles), 32 * WPC, smem, st>>>(a);
  return cudaGetLastError();
}

int sweep_window_stride() { return sweep::STRIDE; }

void sweep_geometry(int* out) {
  out[0] = sweep::WIN;
  out[1] = sweep::FLUSH;
  out[2] = sweep::R;
  out[3] = sweep::STRIDE;
}

int sweep_record_doubles(int nq, int mode) {
  switch (nq) {
    case 3: return mode == 0 ? sweep::Rec<3, 0>::DOUBLES : sweep::Rec<3, 1>::DOUBLES;
    case 6: return mode == 0 ? sweep::Rec<6, 0>::DOUBLES : sweep::Rec<6, 1>::DOUBLES;
    case 12: return mode == 0 ? sweep::Rec<12, 0>::DOUBLES : sweep::Rec<12, 1>::DOUBLES;
    case 16: return mode == 0 ? sweep::Rec<16, 0>::DOUBLES : sweep::Rec<16, 1>::DOUBLES;
  }
  return -1;
}

// mode 0: SL rows (SL record stream), 1: ADL rows (ADL record stream)
cudaError_t launch_regular(const RegularArgs& a, int nq, int mode, cudaStream_t st) {
  if (a.n_rows <= 0 || a.n_tiles <= 0) return cudaSuccess;
  if (mode == 0) {  // the rule's hat values into constant memory, once per (device, nq)
    static bool done[64][4];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int hi = sweep::hat_index(nq);
    if (dev < 64 && !done[dev][hi]) {
      e = cudaMemcpyToSymbol(sweep::c_hats, a.hats, sizeof(a.hats), (size_t)hi * sizeof(a.hats),
                             cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return e;
      done[dev][hi] = true;
    }
  }
  auto go = [&](auto nq_tag) -> cudaError_t {
    constexpr int Q = decltype(nq_tag)::value;
    if (a.part_ld > 0) return launch_sweep_nq<Q, 1, true>(a, st);
    return mode == 0 ? launch_sweep_nq<Q, 0>(a, st) : launch_sweep_nq<Q, 1>(a, st);
  };
  switch (nq) {
    case 3: return go(std::integral_constant<int, 3>{});
    case 6: return go(std::integral_constant<int, 6>{});
    case 12: return go(std::integral_constant<int, 12>{});
    case 16: return go(std::integral_constant<int, 16>{});
  }
  return cudaErrorInvalidValue;
}

}  // namespace hvb
