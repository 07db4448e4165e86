// C-ABI of libhvb.so (declared in include/hvb.h).  Every entry point takes
// raw device pointers owned by the caller (PyTorch tensors on the Python
// side), sizes and a cudaStream_t, launches asynchronously and returns 0 or
// an HVB_E* status; hvb_last_error() gives the message.  No torch types, no
// allocation, no host synchronisation.
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/hvb.h"
#include "launch.cuh"

static thread_local std::string g_err;

static int fail(int code, const char* what, cudaError_t e = cudaSuccess) {
  char buf[512];
  if (e != cudaSuccess)
    snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  else
    snprintf(buf, sizeof buf, "%s", what);
  g_err = buf;
  return code;
}

static int check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(HVB_ECUDA, what, e);
  return HVB_OK;
}

extern "C" {

const char* hvb_last_error(void) { return g_err.c_str(); }

int hvb_version(void) { return HVB_ABI_VERSION; }

int hvb_build_table(const double* nodes6, int nt, int nq, const double* rule, double* table, void* stream) {
  if (nt < 0 || (nq != 3 && nq != 6 && nq != 12 && nq != 16)) return fail(HVB_EARG, "hvb_build_table: bad nt/nq");
  if (nt == 0) return HVB_OK;
  return check(hvb::launch_build_table(nodes6, nt, nq, rule, table, (cudaStream_t)stream), "hvb_build_table");
}

int hvb_panel_data(const double* circumcenters, const double* radii, int nt, double eta, double* ccr, double* cls,
                   double* groups, void* stream) {
  if (nt < 0) return fail(HVB_EARG, "hvb_panel_data: negative panel count");
  return check(hvb::launch_panel_data(circumcenters, radii, nt, eta, ccr, cls, groups, (cudaStream_t)stream),
               "hvb_panel_data");
}

int hvb_build_stream(const double* table, int nq, const double* ccr, double eta, const int* ent_tri,
                     const int* ent_meta, long long n_entries, int mode, int window, double* stream_out,
                     void* stream) {
  if (n_entries < 0) return fail(HVB_EARG, "hvb_build_stream: negative entry count");
  if (mode != 0 && mode != 1) return fail(HVB_EARG, "hvb_build_stream: mode must be 0 (SL) or 1 (ADL)");
  if (window < 1 || window > 32767) return fail(HVB_EARG, "hvb_build_stream: window out of range");
  if (hvb::sweep_record_doubles(nq, mode) < 0) return fail(HVB_EARG, "hvb_build_stream: nq must be 3, 6, 12 or 16");
  return check(hvb::launch_build_stream(table, nq, ccr, eta, ent_tri, ent_meta, n_entries, mode, window,
                                        stream_out, (cudaStream_t)stream),
               "hvb_build_stream");
}

int hvb_stream_record_doubles(int nq, int mode) { return hvb::sweep_record_doubles(nq, mode); }

int hvb_sweep_geometry(int* out) {
  if (!out) return fail(HVB_EARG, "hvb_sweep_geometry: null output");
  hvb::sweep_geometry(out);
  return HVB_OK;
}

long long hvb_sweep_sched_ints(int n_rows, int n_tiles) { return (long long)hvb::sweep_sched_ints(n_rows, n_tiles); }

int hvb_assemble_regular(const double* panel_stream, const long long* tile_ptr, const int* tile_order,
                         const int* tile_lptr,
                         const int* lcol, const int* tile_xptr, const int* xent, const int* tile_pptr,
                         const int* prods, const int* tile_cptr, const int* cons, int n_tiles, int nq,
                         const double* hats, int row_begin, int n_rows, const double* rowdata, const int* row_col,
                         const double* row_scale, const long long* row_out, double* A, long long part_ld,
                         const int* tri_cols, int mode, double* halo, int* sched, int* near_list,
                         unsigned long long* near_count, long long near_cap, void* stream) {
  if (n_rows <= 0 || n_tiles <= 0) return HVB_OK;
  if (part_ld < 0 || (part_ld > 0 && (mode != 1 || row_begin % 32 != 0)))
    return fail(HVB_EARG, "hvb_assemble_regular: charge-reduce mode needs ADL rows starting at a 32-row boundary");
  if (mode != 0 && mode != 1) return fail(HVB_EARG, "hvb_assemble_regular: mode must be 0 (SL) or 1 (ADL)");
  if (hvb::sweep_record_doubles(nq, mode) < 0) return fail(HVB_EARG, "hvb_assemble_regular: nq must be 3, 6, 12 or 16");
  if (mode == 0 && !hats) return fail(HVB_EARG, "hvb_assemble_regular: the SL sweep needs the hat table");
  hvb::RegularArgs a;
  std::memset(&a, 0, sizeof a);
  a.stream = panel_stream;
  a.tile_ptr = (const int64_t*)tile_ptr;
  if (!sched || !tile_lptr || !lcol || !tile_xptr || !tile_pptr || !tile_cptr)
    return fail(HVB_EARG, "hvb_assemble_regular: null schedule");
  a.tile_order = tile_order;
  a.tile_lptr = tile_lptr;
  a.lcol = lcol;
  a.tile_xptr = tile_xptr;
  a.xent = (const int4*)xent;
  a.tile_pptr = tile_pptr;
  a.prods = prods;
  a.tile_cptr = tile_cptr;
  a.cons = cons;
  a.halo = halo;
  a.sched = sched;
  a.n_tiles = n_tiles;
  a.row_begin = row_begin;
  a.n_rows = n_rows;
  a.rowdata = rowdata;
  a.row_col = row_col;
  a.row_scale = row_scale;
  a.row_out = (const int64_t*)row_out;
  a.A = A;
  a.tri_cols = tri_cols;
  a.near_list = near_list;
  a.near_count = near_count;
  a.near_cap = near_cap;
  a.part_ld = part_ld;
  if (hats)
    for (int q = 0; q < nq; ++q)
      for (int c = 0; c < 3; ++c) a.hats[q][c] = hats[3 * q + c];
  return check(hvb::launch_regular(a, nq, mode, (cudaStream_t)stream), "hvb_assemble_regular");
}

int hvb_assemble_singular(const double* nodes6, const int* tri_cols, const int* col_dev, const int* vc_ptr,
                          const int* vc_tri, const int* vc_corner, const double* rule, int n_rule, int n_rows,
                          const double* rowdata, const int* row_kind, const int* row_col, const double* row_scale,
                          const double* row_diag, const long long* row_out, double* A, int rows_per_warp,
                          void* stream) {
  if (rows_per_warp < 1) return fail(HVB_EARG, "hvb_assemble_singular: rows_per_warp must be >= 1");
  hvb::SingularArgs a;
  a.rows_per_warp = rows_per_warp;
  a.nodes6 = nodes6;
  a.tri_cols = tri_cols;
  a.col_dev = col_dev;
  a.vc_ptr = vc_ptr;
  a.vc_tri = vc_tri;
  a.vc_corner = vc_corner;
  a.rule = rule;
  a.nm = n_rule;
  a.rows = nullptr;
  a.n_rows = n_rows;
  a.rowdata = rowdata;
  a.row_kind = row_kind;
  a.row_col = row_col;
  a.row_scale = row_scale;
  a.row_diag = row_diag;
  a.row_out = (const int64_t*)row_out;
  a.A = A;
  return check(hvb::launch_singular(a, (cudaStream_t)stream), "hvb_assemble_singular");
}

int hvb_charge_reduce(const double* part, int n_parts, long long part_ld, int n, double* out, int accumulate,
                      void* stream) {
  if (n_parts < 0 || n < 0 || part_ld < n) return fail(HVB_EARG, "hvb_charge_reduce: bad n_parts / n / part_ld");
  return check(hvb::launch_charge_reduce(part, n_parts, part_ld, n, out, accumulate, (cudaStream_t)stream),
               "hvb_charge_reduce");
}

int hvb_fill_float_cols(double* A, const long long* row_out, const int* row_float, int n_rows, int n, int n_fl,
                        void* stream) {
  return check(hvb::launch_fill_float_cols(A, (const int64_t*)row_out, row_float, n_rows, n, n_fl,
                                           (cudaStream_t)stream),
               "hvb_fill_float_cols");
}

int hvb_near_pairs(const int* pairs, long long n_pairs, const double* points, const int* kind,
                   const double* nodes6, const double* radii, const double* duffy, int n_duffy,
                   const double* graded, int n_graded, int bisect_depth, double bisect_trigger, double* out,
                   void* stream) {
  hvb::NearArgs a;
  a.pairs = pairs;
  a.n_pairs = n_pairs;
  a.points = points;
  a.kind = kind;
  a.nodes6 = nodes6;
  a.radii = radii;
  a.duffy = duffy;
  a.n_duffy = n_duffy;
  a.graded = graded;
  a.n_graded = n_graded;
  a.bisect_depth = bisect_depth;
  a.bisect_trigger = bisect_trigger;
  a.out = out;
  return check(hvb::launch_near_pairs(a, (cudaStream_t)stream), "hvb_near_pairs");
}

int hvb_near_apply_rows(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                        const int* tri_cols, const int* col_dev, const double* row_scale, const long long* row_out,
                        double* A, void* stream) {
  return check(hvb::launch_near_apply_rows(seg_ptr, n_seg, pairs, contrib, tri_cols, col_dev, row_scale,
                                           (const int64_t*)row_out, A, (cudaStream_t)stream),
               "hvb_near_apply_rows");
}

int hvb_gemv(const void* A, int prec, long long lda, int n_rows, int n_cols, const double* x, const double* left,
             double* y, void* stream) {
  if (lda < n_cols || (lda % 4) != 0) return fail(HVB_EARG, "hvb_gemv: lda must be >= n_cols and a multiple of 4");
  if (prec < 0 || prec > 2) return fail(HVB_EARG, "hvb_gemv: prec must be 0 (f64), 1 (f32) or 2 (f32, f64 sums)");
  if (prec != 0 && (lda % 8) != 0) return fail(HVB_EARG, "hvb_gemv: float32 storage needs lda % 8 == 0");
  return check(hvb::launch_gemv(A, prec, lda, n_rows, n_cols, x, left, y, (cudaStream_t)stream), "hvb_gemv");
}

int hvb_gemv_bcast(const double* A, long long lda, int n_rows, int n_cols, const double* x, const double* left,
                   double* const* outs, int n_out, long long out_off, unsigned long long* const* flags, int rank,
                   unsigned long long epoch, unsigned int* done, void* stream) {
  if (n_out < 1 || n_out > 32 || out_off < 0 || rank < 0 || rank >= n_out || n_rows < 1 || !flags || !done)
    return fail(HVB_EARG, "hvb_gemv_bcast: bad n_out/out_off/rank/n_rows or missing flags/counter");
  return check(hvb::launch_gemv_bcast(A, lda, n_rows, n_cols, x, left, outs, n_out, out_off, flags, rank, epoch, done,
                                      (cudaStream_t)stream),
               "hvb_gemv_bcast");
}

int hvb_ipc_alloc(long long bytes, void** ptr) {
  if (bytes <= 0 || !ptr) return fail(HVB_EARG, "hvb_ipc_alloc: bad size");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, (size_t)bytes);
  return check(e, "hvb_ipc_alloc");
}

int hvb_ipc_free(void* ptr) { return check(cudaFree(ptr), "hvb_ipc_free"); }

int hvb_ipc_handle(void* ptr, unsigned char* out) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e == cudaSuccess) memcpy(out, &h, sizeof h);
  return check(e, "hvb_ipc_handle");
}

int hvb_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int hvb_ipc_open(const unsigned char* handle, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return check(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "hvb_ipc_open");
}

int hvb_ipc_close(void* ptr) { return check(cudaIpcCloseMemHandle(ptr), "hvb_ipc_close"); }

int hvb_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch, void* stream) {
  if (world < 1 || world > 32) return fail(HVB_EARG, "hvb_peer_wait: bad world");
  return check(hvb::launch_peer_wait(flags, world, epoch, (cudaStream_t)stream), "hvb_peer_wait");
}

int hvb_gather_scale(const double* z, const double* right, const int* perm, int n, double* xp, void* stream) {
  return check(hvb::launch_gather_scale(z, right, perm, n, xp, (cudaStream_t)stream), "hvb_gather_scale");
}

int hvb_mgs_partial_size(void) { return 4 * hvb::mgs_grid(); }

int hvb_mgs(const double* V, long long ldv, int j, double* w, int n, double* h, double* norms, double* partial,
            int accumulate, void* stream) {
  if (j < 0 || n <= 0 || ldv < n) return fail(HVB_EARG, "hvb_mgs: bad j/n/ldv");
  return check(hvb::launch_mgs(V, ldv, j, w, n, h, norms, partial, accumulate, (cudaStream_t)stream), "hvb_mgs");
}

int hvb_rowmax_diag(const void* A, int is_f32, long long lda, int n_rows, int n_cols, const int* diag_col,
                    double* rowmax, double* diag, void* stream) {
  return check(hvb::launch_rowmax_diag(A, is_f32, lda, n_rows, n_cols, diag_col, rowmax, diag,
                                       (cudaStream_t)stream),
               "hvb_rowmax_diag");
}

int hvb_contract(const double* table, int nt, int nq, const int* tri_cols, const double* u, double* src,
                 void* stream) {
  return check(hvb::launch_contract(table, nt, nq, tri_cols, u, src, (cudaStream_t)stream), "hvb_contract");
}

int hvb_field(const double* src, const double* cls, const double* groups, const int* tri_cols, int nt, int nq,
              const double* pts,
              const int* own_col, int m, int split, int potential, double* part, int* near_list,
              unsigned long long* near_count, long long near_cap, void* stream) {
  if (split < 1) return fail(HVB_EARG, "hvb_field: split must be >= 1");
  hvb::FieldArgs a;
  a.src = src;
  a.cls = cls;
  a.groups = groups;
  a.tri_cols = tri_cols;
  a.nt = nt;
  a.nq = nq;
  a.pts = pts;
  a.own_col = own_col;
  a.m = m;
  a.split = split;
  a.potential = potential;
  a.part = part;
  a.near_list = near_list;
  a.near_count = near_count;
  a.near_cap = near_cap;
  a.has_near = nullptr;
  a.out = nullptr;
  return check(hvb::launch_field(a, (cudaStream_t)stream), "hvb_field");
}

int hvb_field_reduce(const double* part, int split, int m, double* out, void* stream) {
  return check(hvb::launch_field_reduce(part, split, m, out, (cudaStream_t)stream), "hvb_field_reduce");
}

int hvb_near_apply_points(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                          const int* tri_cols, const double* u, int potential, double* out, void* stream) {
  return check(hvb::launch_near_apply_points(seg_ptr, n_seg, pairs, contrib, tri_cols, u, potential, out,
                                             (cudaStream_t)stream),
               "hvb_near_apply_points");
}

int hvb_field_singular(const double* nodes6, const int* tri_cols, const int* vc_ptr, const int* vc_tri,
                       const int* vc_corner, const double* rule, int n_rule, const double* pts,
                       const double* normals, const int* own_col, int m, const double* u, double side,
                       double* efield, double* emag, void* stream) {
  return check(hvb::launch_field_singular(nodes6, tri_cols, vc_ptr, vc_tri, vc_corner, rule, n_rule, pts, normals,
                                          own_col, m, u, side, efield, emag, (cudaStream_t)stream),
               "hvb_field_singular");
}

int hvb_line_state_bytes(void) { return (int)sizeof(hvb::LineState); }

int hvb_trace_ctrl(void* state, int n_lines, const double* starts, const int* orient, const double* geo, int mode,
                   double* e_pts, int* e_line, double* sd_pts, int* sd_line, unsigned long long* counters,
                   const double* e_out, const int* e_flag, const double* sd_out, double* out_pts,
                   int cap, void* stream) {
  if (n_lines < 0 || mode < 0 || mode > 2 || cap < 2) return fail(HVB_EARG, "hvb_trace_ctrl: bad n_lines/mode/cap");
  if (mode == 0 && (!starts || !orient)) return fail(HVB_EARG, "hvb_trace_ctrl: init needs starts and orientations");
  hvb::TraceArgs a;
  a.state = static_cast<hvb::LineState*>(state);
  a.n_lines = n_lines;
  a.starts = starts;
  a.orient = orient;
  for (int d = 0; d < 3; ++d) {
    a.center[d] = geo[d];
    a.half[d] = geo[3 + d];
  }
  a.diag = geo[6];
  a.h_min = geo[7];
  a.h_max = geo[8];
  a.l_max = geo[9];
  a.rel_tol = geo[10];
  a.tol_frac = geo[11];
  a.e_floor = geo[12];
  a.max_steps = (long long)geo[13];
  a.e_pts = e_pts;
  a.e_line = e_line;
  a.sd_pts = sd_pts;
  a.sd_line = sd_line;
  a.counters = counters;
  a.e_out = e_out;
  a.e_flag = e_flag;
  a.sd_out = sd_out;
  a.out_pts = out_pts;
  a.cap = cap;
  return check(hvb::launch_trace_ctrl(a, mode, (cudaStream_t)stream), "hvb_trace_ctrl");
}

int hvb_trace_round(void* state, int n_lines, const double* geo, double* cur_pts, double* nxt_pts, int* nxt_line,
                    double* sd_pts, int* sd_line, double* sd_out, unsigned long long* counters, double* e_out,
                    int* e_flag, int* has_near, double* part, const double* src, const double* cls,
                    const double* groups, const int* tri_cols, int nt, int nq, int split, const double* nodes6, const double* radii,
                    const double* ccr, const double* u, const double* duffy, int n_duffy, const double* graded,
                    int n_graded, int bisect_depth, double bisect_trigger, double prox, double* out_pts, int cap,
                    void* stream) {
  if (n_lines < 0 || cap < 2 || split < 1) return fail(HVB_EARG, "hvb_trace_round: bad n_lines/cap/split");
  hvb::TraceRoundArgs r;
  hvb::TraceArgs& a = r.ctrl;
  a.state = static_cast<hvb::LineState*>(state);
  a.n_lines = n_lines;
  a.starts = nullptr;
  a.orient = nullptr;
  for (int d = 0; d < 3; ++d) {
    a.center[d] = geo[d];
    a.half[d] = geo[3 + d];
  }
  a.diag = geo[6];
  a.h_min = geo[7];
  a.h_max = geo[8];
  a.l_max = geo[9];
  a.rel_tol = geo[10];
  a.tol_frac = geo[11];
  a.e_floor = geo[12];
  a.max_steps = (long long)geo[13];
  a.e_pts = nxt_pts;
  a.e_line = nxt_line;
  a.sd_pts = sd_pts;
  a.sd_line = sd_line;
  a.counters = counters;
  a.e_out = e_out;
  a.e_flag = e_flag;
  a.sd_out = sd_out;
  a.out_pts = out_pts;
  a.cap = cap;
  hvb::FieldArgs& f = r.field;
  f.src = src;
  f.cls = cls;
  f.groups = groups;
  f.tri_cols = tri_cols;
  f.nt = nt;
  f.nq = nq;
  f.pts = cur_pts;
  f.own_col = nullptr;
  f.m = 0;
  f.split = split;
  f.potential = 0;
  f.part = part;
  f.near_list = nullptr;
  f.near_count = nullptr;
  f.near_cap = 0;
  f.has_near = has_near;
  f.out = e_out;
  r.nodes6 = nodes6;
  r.radii = radii;
  r.ccr = ccr;
  r.u = u;
  r.duffy = duffy;
  r.n_duffy = n_duffy;
  r.graded = graded;
  r.n_graded = n_graded;
  r.bisect_depth = bisect_depth;
  r.bisect_trigger = bisect_trigger;
  r.prox = prox;
  return check(hvb::launch_trace_round(r, (cudaStream_t)stream), "hvb_trace_round");
}

int hvb_trace_summary(const void* state, int n_lines, int* info, double* dinfo, void* stream) {
  return check(hvb::launch_trace_summary(static_cast<const hvb::LineState*>(state), n_lines, info, dinfo,
                                         (cudaStream_t)stream),
               "hvb_trace_summary");
}

int hvb_surface_distance(const double* pts, int m, const double* ccr, const double* groups, int nt,
                         const double* nodes6, double* out, void* stream) {
  if (m < 0 || nt < 1) return fail(HVB_EARG, "hvb_surface_distance: bad m/nt");
  return check(hvb::launch_surface_distance(pts, m, ccr, groups, nt, nodes6, out, (cudaStream_t)stream),
               "hvb_surface_distance");
}

int hvb_near_coincide(const int* pairs, long long n_pairs, const double* pts, const double* nodes6, double prox,
                      int* flag, void* stream) {
  return check(hvb::launch_near_coincide(pairs, n_pairs, pts, nodes6, prox, flag, (cudaStream_t)stream),
               "hvb_near_coincide");
}

int hvb_streamer(const double* out_pts, const void* state, int n_lines, int cap, const double* e_tab,
                 const double* a_tab, int n_tab, double k_str, double* value, int* verdict, void* stream) {
  if (n_tab < 1) return fail(HVB_EARG, "hvb_streamer: empty ionization table");
  return check(hvb::launch_streamer(out_pts, static_cast<const hvb::LineState*>(state), n_lines, cap, e_tab, a_tab,
                                    n_tab, k_str, value, verdict, (cudaStream_t)stream),
               "hvb_streamer");
}

}  // extern "C"
