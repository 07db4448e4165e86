// Argument blocks and launcher prototypes shared by the kernel files and
// the C-ABI layer (hvb_api.cu).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace hvb {

struct RegularArgs {
  const double* stream;     // tile panel streams (csrc/assemble.cu record formats)
  const int64_t* tile_ptr;  // (n_tiles+1) record offsets
  const int* tile_order;    // launch order of the tiles (longest first), nullptr = identity
  const int* tile_lptr;     // (n_tiles+1) local column offsets
  const int* lcol;          // per local column: device column, or ~slot (halo copy / partial)
  const int* tile_xptr;     // (n_tiles+1) exchange entry offsets
  const int4* xent;         // per entry: slot, device column, first, last
  const int* tile_pptr;     // (n_tiles+1) producer offsets
  const int* prods;         // distinct producer tiles of each tile
  const int* tile_cptr;     // (n_tiles+1) consumer offsets
  const int* cons;          // distinct consumer tiles of each tile
  double* halo;             // (n_slots, n_rows) exchange slots of this launch
  int* sched;               // sweep_sched_ints(n_rows, n_tiles): completion counters
  int n_tiles;
  int row_begin;            // first row-list entry of this launch
  int n_rows;               // rows in this launch
  const double* rowdata;    // RowData per row-list entry (6 doubles)
  const int* row_col;       // own collocation column (singular test), -1 none
  const double* row_scale;  // multiplies every entry of the row
  const int64_t* row_out;   // output row offset (in elements) into A
  double* A;                // output matrix (device column order)
  const int* tri_cols;      // (nt,3) original collocation cols of corners
  int* near_list;           // (cap, 2): (row-list index, triangle)
  unsigned long long* near_count;
  long long near_cap;
  double hats[16][3];       // hat_c(q) of the regular rule (SL stream; zero past nq)
  int64_t part_ld;          // > 0: charge-reduce mode (ADL rows only): A holds one partial
                            // row per 32-row tile, sum over the tile's rows of row_scale * entry
};

struct SingularArgs {
  const double* nodes6;
  const int* tri_cols;    // original cols
  const int* col_dev;     // original col -> device col
  const int* vc_ptr;      // star CSR over original collocation cols
  const int* vc_tri;
  const int* vc_corner;
  const double* rule;     // 3 x nm x 4
  int nm;
  const int* rows;        // row-list entries to process
  int n_rows;
  const double* rowdata;
  const int* row_kind;
  const int* row_col;
  const double* row_scale;
  const double* row_diag;  // added to A[row, own col] after scaling
  const int64_t* row_out;
  double* A;
  int rows_per_warp;       // 1; 32 in charge-reduce mode (a tile's rows share one partial row)
};

struct NearArgs {
  const int* pairs;        // (np, 2): point index, triangle
  long long n_pairs;
  const double* points;    // (m, 6): x, y, z, nx, ny, nz
  const int* kind;         // per point: 0 SL, 1 ADL, 2 E (vector), 3 potential
  const double* nodes6;    // (nt, 18)
  const double* radii;     // (nt)
  const double* duffy;     // (n_duffy, 4) Duffy(0, near_duffy_points)
  int n_duffy;
  const double* graded;    // (n_graded, 4) graded(depth, n1d, outer)
  int n_graded;
  int bisect_depth;
  double bisect_trigger;
  double* out;             // (np, 9) corner contributions
};

struct FieldArgs {
  const double* src;      // (nt, nq, 4) contracted sources
  const double* cls;      // (nt, 6): cc, thr, thr2_lo, thr2_hi
  const double* groups;   // (ceil(nt/32), 8): bounds of aligned 32-panel groups (device.py panel_groups)
  const int* tri_cols;    // (nt, 3) original cols (singular test)
  int nt, nq;
  const double* pts;      // (m, 3) targets
  const int* own_col;     // (m) own collocation col or -1 (may be null)
  int m;
  int split;              // panel-range split (grid.y)
  int potential;          // 1: phi, 0: E
  double* part;           // (split, m, 4) partial sums
  int* near_list;         // (cap, 2): (target, triangle); nullptr: set has_near instead
  unsigned long long* near_count;
  long long near_cap;
  int* has_near;          // (split, m) chunk flags (dynamic / tracer path)
  double* out;            // (m, 3) reduced field (dynamic path)
};

cudaError_t launch_regular(const RegularArgs& a, int nq, int mode, cudaStream_t st);
int sweep_record_doubles(int nq, int mode);
int sweep_window_stride();
size_t sweep_sched_ints(int n_rows, int n_tiles);
void sweep_geometry(int* out);
cudaError_t launch_build_table(const double* nodes6, int nt, int nq, const double* rule, double* out,
                               cudaStream_t st);
cudaError_t launch_build_stream(const double* table, int nq, const double* ccr, double eta, const int* ent_tri,
                                const int* ent_meta, int64_t ne, int mode, int window, double* out,
                                cudaStream_t st);
cudaError_t launch_panel_data(const double* cc, const double* radii, int nt, double eta, double* ccr, double* cls,
                              double* groups, cudaStream_t st);
cudaError_t launch_singular(const SingularArgs& a, cudaStream_t st);
cudaError_t launch_charge_reduce(const double* part, int n_parts, int64_t part_ld, int n, double* out, int accumulate,
                                 cudaStream_t st);
cudaError_t launch_fill_float_cols(double* A, const int64_t* row_out, const int* row_float, int n_rows, int n,
                                   int n_fl, cudaStream_t st);
cudaError_t launch_near_pairs(const NearArgs& a, cudaStream_t st);
cudaError_t launch_near_apply_rows(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                   const int* tri_cols, const int* col_dev, const double* row_scale,
                                   const int64_t* row_out, double* A, cudaStream_t st);
cudaError_t launch_gemv(const void* A, int prec, int64_t lda, int nrows, int ncols, const double* x,
                        const double* left, double* y, cudaStream_t st);
cudaError_t launch_gemv_bcast(const double* A, int64_t lda, int nrows, int ncols, const double* x, const double* left,
                              double* const* outs, int n_out, int64_t out_off, unsigned long long* const* flags,
                              int rank, unsigned long long epoch, unsigned int* done, cudaStream_t st);
cudaError_t launch_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch, cudaStream_t st);
cudaError_t launch_gather_scale(const double* z, const double* right, const int* perm, int n, double* xp,
                                cudaStream_t st);
cudaError_t launch_mgs(const double* V, long long ldv, int j, double* w, int n, double* h, double* norms,
                       double* partial, int accumulate, cudaStream_t st);
int mgs_grid();
cudaError_t launch_rowmax_diag(const void* A, int is_f32, int64_t lda, int nrows, int ncols, const int* diag_col,
                               double* rowmax, double* diag, cudaStream_t st);
cudaError_t launch_field(const FieldArgs& a, cudaStream_t st);
cudaError_t launch_field_dyn(const FieldArgs& a, unsigned long long* m_dev, int grid, cudaStream_t st);
cudaError_t launch_contract(const double* table, int nt, int nq, const int* tri_cols, const double* u, double* src,
                            cudaStream_t st);
cudaError_t launch_field_reduce(const double* part, int split, int m, double* out, cudaStream_t st);
cudaError_t launch_near_apply_points(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                                     const int* tri_cols, const double* u, int potential, double* out,
                                     cudaStream_t st);
cudaError_t launch_field_singular(const double* nodes6, const int* tri_cols, const int* vc_ptr, const int* vc_tri,
                                  const int* vc_corner, const double* rule, int nm, const double* pts,
                                  const double* normals, const int* own_col, int m, const double* u, double side,
                                  double* efield, double* emag, cudaStream_t st);

// ---- device tracer (trace.cu) ----
constexpr int kPhaseStart = 0, kPhaseSD = 1, kPhaseStage = 2, kPhaseSnap = 4, kPhaseDone = 5;  // 3: unused
constexpr int kSurfaceHit = 0, kWeakField = 1, kMaxLength = 2, kLeftDomain = 3, kMaxSteps = 4;
constexpr int kStatusRunning = 0, kStatusDone = 1, kStatusWeakStart = 2, kStatusCoincident = 3;

struct LineState {        // 304 bytes, one per line, in HBM
  double x[3];            // current point
  double k[7][3];         // stage tangents (k[0] = FSAL k1)
  double req[3];          // outstanding E request point
  double h, s, err, tol, d_surf, local_r, sign;
  int phase, stage, npts, armed, term, status, slot, steps;  // steps: RK steps taken (max_steps)
};

struct TraceArgs {
  LineState* state;
  int n_lines;
  const double* starts;   // (n_lines, 3)
  const int* orient;      // (n_lines)
  // geometry / parameters (reference trace_fieldline 258-268, TraceParams)
  double center[3], half[3];
  double diag, h_min, h_max, l_max, rel_tol, tol_frac, e_floor;
  long long max_steps;    // 0: unbounded (reference); else end lines with kMaxSteps
  // request lists (compacted by atomics): E requests, SD requests
  double* e_pts;          // (n_lines, 3)
  int* e_line;
  double* sd_pts;         // (n_lines, 3)
  int* sd_line;
  unsigned long long* counters;  // [0] E requests, [1] SD requests, [2] max points per line,
                                 // [3] total E requests (never reset), [4] N-body work
                                 // counter (zeroed each round)
  // results of the previous requests
  const double* e_out;    // (n_req, 3)
  const int* e_flag;      // (n_req) 1 = coincident with a mesh vertex
  const double* sd_out;   // (n_sd, 2) d_surf, local R
  // polylines: (n_lines, cap, 5) x, y, z, |E|, s
  double* out_pts;
  int cap;
};

// one sync-free tracer round (trace.cu): field.pts = current request list,
// field.out = ctrl.e_out, field.has_near = scratch flags; ctrl.e_pts/e_line =
// the next request list
struct TraceRoundArgs {
  TraceArgs ctrl;
  FieldArgs field;
  const double* nodes6;
  const double* radii;
  const double* ccr;
  const double* u;
  const double* duffy;
  int n_duffy;
  const double* graded;
  int n_graded;
  int bisect_depth;
  double bisect_trigger;
  double prox;
};

cudaError_t launch_trace_ctrl(const TraceArgs& a, int mode, cudaStream_t st);
cudaError_t launch_trace_round(const TraceRoundArgs& r, cudaStream_t st);
cudaError_t launch_surface_distance(const double* pts, int m, const double* ccr, const double* groups, int nt,
                                    const double* nodes6, double* out, cudaStream_t st);
cudaError_t launch_near_coincide(const int* pairs, long long n_pairs, const double* pts, const double* nodes6,
                                 double prox, int* flag, cudaStream_t st);
cudaError_t launch_trace_summary(const LineState* state, int n_lines, int* info, double* dinfo, cudaStream_t st);
cudaError_t launch_streamer(const double* out_pts, const LineState* state, int n_lines, int cap, const double* e_tab,
                            const double* a_tab, int n_tab, double k_str, double* value, int* verdict,
                            cudaStream_t st);

}  // namespace hvb
