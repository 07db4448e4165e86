/* hvb.h -- C ABI of libhvb.so, the B200 (sm_100a) kernels of the
 * paper_2003_12663_b200 indirect-BEM drop-in.
 *
 * The reference (hvbem 0.1.0, pure Python/NumPy) has no native FFI; its hot
 * path is the Python call chain listed per entry point below (paths are
 * relative to reference pkg/src/hvbem/).  The drop-in keeps that Python API
 * (paper_2003_12663_b200.assembly / solver / postprocess) and routes every
 * heavy loop through these functions.
 *
 * Conventions: all array pointers are DEVICE pointers to caller-owned,
 * contiguous buffers (PyTorch tensors on the Python side); sizes are element
 * counts; `stream` is a cudaStream_t; launches are asynchronous.  Return 0
 * (HVB_OK) or an HVB_E* code; hvb_last_error() returns a thread-local
 * message.  "Original" collocation columns follow the mesh's collocation
 * order; "device" columns are the matrix storage order.
 */
#ifndef HVB_H_
#define HVB_H_

#ifdef __cplusplus
extern "C" {
#endif

#define HVB_ABI_VERSION 1

#define HVB_OK 0
#define HVB_EARG 1    /* invalid argument (maps to ValueError)            */
#define HVB_ECUDA 2   /* CUDA launch/runtime error (maps to RuntimeError)  */

const char* hvb_last_error(void);
int hvb_version(void);

/* K1 -- regular-rule sample table: table[t][q] = (y_tq, jw_tq*hat_c(q)/4pi),
 * 6 doubles per (t,q); rule = nq x (u, v, w, 0).
 * Replaces: TriangleTables.__init__  assembly.py:78-103 */
int hvb_build_table(const double* nodes6, int nt, int nq, const double* rule, double* table, void* stream);

/* Pack the per-column-tile panel streams (one record per panel, in its
 * tile; hvb_stream_record_doubles(nq, mode) doubles each): nodes, then an
 * 8-double tail = cc, thr = fl(eta*R), squared classification bracket,
 * panel id, first local column, window slots of the corners, flags.
 * ent_meta = (mfirst, l0, l1, l2, flags) per entry, l = local column of a
 * corner or -1 (dummy records); the record stores l % window (window = the
 * dump slot for -1).  mode 0 (SL stream): per node pair 10 doubles, per node
 * Y = -2 s (y - cc), P = s |y - cc|^2, Q = s with s = (4 pi / jw)^2;
 * mode 1 (ADL stream): per node (y, jw hat_0..2 / 4 pi).
 * Replaces: the per-row classification setup and the sample tables of
 * row_pass1  assembly.py:155-200 */
int hvb_build_stream(const double* table, int nq, const double* ccr, double eta, const int* ent_tri,
                     const int* ent_meta, long long n_entries, int mode, int window, double* stream_out,
                     void* stream);
int hvb_stream_record_doubles(int nq, int mode);
/* Regular-sweep geometry of this build (HOST pointer out[4]): window
 * columns, flush width, records per stage, window row stride (doubles).
 * The host tiling uses band = window - flush and stages of that size. */
int hvb_sweep_geometry(int* out);

/* Column tiling of the regular sweep (HOST function, host pointers; no
 * GPU needed; csrc/tiling.cpp): recursive coordinate bisection of the n
 * collocation points into tiles of <= max_tile columns swept along their
 * longest axis (the tile's owned columns), one record per panel in the
 * lowest-numbered tile owning one of its corners; a tile's local columns
 * are its owned columns plus its halo (its panels' corners owned by later
 * tiles), numbered along the sweep axis; records sorted by first local
 * column, grouped in stages of `group` records with disjoint corners within
 * `band` columns (short stages padded with dummy records, panel -1).
 * sizes = (n_tiles, n_records, band, real records, local columns,
 * exchange entries, slots, halo copies, producer entries = consumer
 * entries); fetch copies
 * perm (n), tile_col0/width (n_tiles: owned device columns), tile_ptr
 * (n_tiles + 1), ent_tri (n_records), ent_meta (n_records x 5: mfirst, l0,
 * l1, l2, flags; l = local column), tile_lptr (n_tiles + 1), lcol (local
 * columns: device column, or ~slot of a halo copy / receiving column's
 * partial), tile_xptr (n_tiles + 1), xent (entries x 4: slot, device
 * column, first, last -- per receiving column its partial, then its halo
 * copies by producer), tile_pptr (n_tiles + 1) / prods (distinct
 * producer tiles per tile) and tile_cptr (n_tiles + 1) / cons (distinct
 * consumer tiles per tile); free releases the handle.  Returns 0, 1 (bad
 * argument) or 2 (band not bounded).
 * Replaces: nothing in the reference (its rows are independent NumPy
 * sweeps, assembly.py:173-200); this is the schedule of hvb_assemble_regular. */
int hvb_tiling_build(const double* points, int n, const int* tri_cols, int nt, int max_tile, int band, int group,
                     long long* sizes, void** handle);
int hvb_tiling_fetch(void* handle, int* perm, int* tile_col0, int* tile_width, long long* tile_ptr, int* ent_tri,
                     int* ent_meta, int* tile_lptr, int* lcol, int* tile_xptr, int* xent, int* tile_pptr,
                     int* prods, int* tile_cptr, int* cons);
int hvb_tiling_free(void* handle);

/* Per-panel device arrays from the flat circumcircles (cc (nt,3), R (nt)):
 * ccr (nt,4) = cc, R; cls (nt,6) = cc, fl(eta R), fl(eta R)^2 (1 -+ 1e-13);
 * groups (ceil(nt/32), 8) = bounds of aligned 32-panel groups (centre,
 * rho_cls, rho_sd), equal bit for bit to device.py:panel_groups.
 * Replaces: the per-triangle classification inputs of classify_pair
 * quadrature.py:207-221 / assembly.py:155-168 and _surface_distance
 * postprocess.py:198-218 (mesh circumcircles mesh.py:188-200) */
int hvb_panel_data(const double* circumcenters, const double* radii, int nt, double eta, double* ccr, double* cls,
                   double* groups, void* stream);

/* K2+K3 -- regular sweep of n_rows collocation rows against every panel,
 * classification fused (regular iff ||x-cc|| > eta*R with the reference's
 * rounding), SL (mode 0, SL stream) or ADL (mode 1, ADL stream) kernel,
 * each entry written once as row_scale * sum, for row-list entries
 * [row_begin, row_begin+n_rows).  hats (HOST pointer) = nq x 3 hat values
 * hat_c(q) of the regular rule.  Non-regular, non-singular pairs are
 * appended to near_list as (row-list index, triangle).  Schedule arrays
 * from hvb_tiling_fetch (device copies; xent as int4); tile_order (device,
 * n_tiles, or NULL = identity) is the launch order of the tiles -- longest
 * first shortens the launch's last wave.  A column local to
 * several tiles is summed in a fixed order: every tile leaves its raw sums
 * of such a column in a slot of `halo`; whichever CTA (same rows) is the
 * last of the owner and its producers to finish adds the owner's partial
 * and the copies in producer order and writes the entry (completion
 * counters in `sched`; no CTA waits on another).
 * Replaces: row_pass1 regular part  assembly.py:170-200 and
 * _kernel_values 126-132 */
int hvb_assemble_regular(const double* panel_stream, const long long* tile_ptr, const int* tile_order,
                         const int* tile_lptr,
                         const int* lcol, const int* tile_xptr, const int* xent, const int* tile_pptr,
                         const int* prods, const int* tile_cptr, const int* cons, int n_tiles, int nq,
                         const double* hats, int row_begin, int n_rows, const double* rowdata, const int* row_col,
                         const double* row_scale, const long long* row_out, double* A, long long part_ld,
                         const int* tri_cols, int mode, double* halo, int* sched, int* near_list,
                         unsigned long long* near_count, long long near_cap, void* stream);
/* Device scratch of one hvb_assemble_regular call: `sched` holds
 * hvb_sweep_sched_ints(n_rows, n_tiles) ints (zeroed by the call: one
 * completion counter per (row block, tile)); `halo` holds
 * n_slots x n_rows doubles (exchange slots, csrc/tiling.cpp). */
long long hvb_sweep_sched_ints(int n_rows, int n_tiles);

/* K4 (+K6 diagonal) -- singular corner pairs with the split-corner Duffy
 * rule (3 x n_rule x 4 table), then A[row, own] += row_diag.
 * Replaces: row_pass1 singular batch  assembly.py:202-235; dielectric
 * diagonal _row_equation 436-437 */
int hvb_assemble_singular(const double* nodes6, const int* tri_cols, const int* col_dev, const int* vc_ptr,
                          const int* vc_tri, const int* vc_corner, const double* rule, int n_rule, int n_rows,
                          const double* rowdata, const int* row_kind, const int* row_col, const double* row_scale,
                          const double* row_diag, const long long* row_out, double* A, int rows_per_warp,
                          void* stream);

/* K6 -- floating-potential columns n..n+n_fl-1 of collocation rows (-1 in
 * the row's own floating column).  Replaces: _row_equation 425-426 */
int hvb_fill_float_cols(double* A, const long long* row_out, const int* row_float, int n_rows, int n, int n_fl,
                        void* stream);

/* K5 -- deferred near-singular pairs: closest point, subdivision, graded
 * composite rule, kernel (kind 0 SL, 1 ADL, 2 E, 3 potential); writes 9
 * corner contributions per pair.  Replaces: row_pass2  assembly.py:245-292,
 * near_singular_rule  quadrature.py:409-450 */
int hvb_near_pairs(const int* pairs, long long n_pairs, const double* points, const int* kind,
                   const double* nodes6, const double* radii, const double* duffy, int n_duffy,
                   const double* graded, int n_graded, int bisect_depth, double bisect_trigger, double* out,
                   void* stream);

/* add sorted near-pair contributions to matrix rows (deterministic order) */
/* K7 -- charge / neutrality row (charge-reduce mode).  hvb_assemble_regular
 * with part_ld > 0 (ADL rows, row_begin % 32 == 0) writes, per 32-row tile
 * t, part[t][c] = sum over the tile's rows of row_scale * (regular entry c)
 * instead of the rows; hvb_near_apply_rows (segments per tile, row_out[r] =
 * t * part_ld) and hvb_assemble_singular (rows_per_warp = 32) then add the
 * near, singular and diagonal (row_diag) terms into the same partial rows
 * in a fixed order, and hvb_charge_reduce sums them: out[c] (+)= sum_t
 * part[t][c] (accumulate = 1 adds to out: chunk partials in chunk order).
 * Replaces: charge_row  assembly.py:540-569, neutrality rows 441-468 */
int hvb_charge_reduce(const double* part, int n_parts, long long part_ld, int n, double* out, int accumulate,
                      void* stream);

int hvb_near_apply_rows(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                        const int* tri_cols, const int* col_dev, const double* row_scale, const long long* row_out,
                        double* A, void* stream);

/* K8 -- y = left .* (A xp), A row-major (lda % 4 == 0).  prec 0: double
 * storage; 1: float storage with float32 products and sums (the
 * reference's float32 dot, assembly.py:386-392); 2: float storage, float32
 * partials over 8 columns accumulated in double (opt-in).
 * Replaces: matvec  assembly.py:376-400 (inside solver op, solver.py:116-118) */
int hvb_gemv(const void* A, int prec, long long lda, int n_rows, int n_cols, const double* x, const double* left,
             double* y, void* stream);

/* Fused GEMV + all-gather (row-sharded GMRES): as hvb_gemv
 * (f64), but each row result left[i] (A xp)_i is stored into all n_out
 * (= world) replicated vectors outs[k][out_off + i] -- this GPU's and every
 * peer's, mapped by CUDA IPC -- instead of a local y; then the launch's
 * last CTA publishes `epoch` into flags[r][rank] of every rank r with a
 * system-scope release store (after system fences of every storing
 * thread).  outs and flags are DEVICE arrays of n_out pointers; done is a
 * zeroed device counter (reset by the kernel).  Pair with hvb_peer_wait.
 * Replaces: matvec + the NCCL all-gather of the row blocks
 * (parallel.RowGather) */
int hvb_gemv_bcast(const double* A, long long lda, int n_rows, int n_cols, const double* x, const double* left,
                   double* const* outs, int n_out, long long out_off, unsigned long long* const* flags, int rank,
                   unsigned long long epoch, unsigned int* done, void* stream);

/* CUDA IPC plumbing for the peer buffers: a cudaMalloc'd (zeroed) region,
 * its handle (hvb_ipc_handle_bytes() bytes), and a peer's mapping. */
int hvb_ipc_alloc(long long bytes, void** ptr);
int hvb_ipc_free(void* ptr);
int hvb_ipc_handle_bytes(void);
int hvb_ipc_handle(void* ptr, unsigned char* out);
int hvb_ipc_open(const unsigned char* handle, void** ptr);
int hvb_ipc_close(void* ptr);

/* Cross-GPU epoch barrier: spins (system-scope acquire loads) until every
 * slot of this rank's flag row (DEVICE pointer, world slots) reached
 * `epoch` -- the release stores of hvb_gemv_bcast; traps after ~17 s if a
 * peer never signals. */
int hvb_peer_wait(const unsigned long long* flags, int world, unsigned long long epoch, void* stream);

/* xp[k] = z[perm[k]] / right[perm[k]]  (perm/right may be NULL) */
int hvb_gather_scale(const double* z, const double* right, const int* perm, int n, double* xp, void* stream);

/* K9 -- one Arnoldi orthogonalisation in one launch (a 16-CTA cluster with
 * w in registers and DSMEM reductions for n <= 131072, else cooperative): modified
 * Gram-Schmidt of w (n) against rows V[0..j] (row pitch ldv) in order,
 * h[i] = V_i.w (accumulate = 1: h[i] += for the re-orthogonalisation pass),
 * norms = (||w|| before, ||w|| after); partial is scratch of
 * hvb_mgs_partial_size() doubles.  Deterministic (fixed slices, CTA-order
 * sums).  Replaces: the MGS loop of _gmres_cycle  solver.py:177-196 */
int hvb_mgs_partial_size(void);
int hvb_mgs(const double* V, long long ldv, int j, double* w, int n, double* h, double* norms, double* partial,
            int accumulate, void* stream);

/* K9 -- row max |a_ij| and diagonal.  Replaces: solver.py:98-107,
 * SystemMatrix.diagonal assembly.py:348-353 */
int hvb_rowmax_diag(const void* A, int is_f32, long long lda, int n_rows, int n_cols, const int* diag_col,
                    double* rowmax, double* diag, void* stream);

/* K10 -- density contraction: src[t][q] = (y_tq, sum_c u_col(t,c) w_c(t,q)) */
int hvb_contract(const double* table, int nt, int nq, const int* tri_cols, const double* u, double* src,
                 void* stream);

/* K10/K11 -- N-body potential (potential=1) or field at m points over the
 * regular panels; panel range split `split` ways (on 32-panel group
 * boundaries) into part (split, m, 4); near pairs appended as (point,
 * triangle).  groups: (ceil(nt/32), 8) bounds of aligned 32-panel groups
 * (centre, rho_cls, rho_sd): a group farther than rho_cls is regular as a
 * whole, which skips its per-panel classification.
 * Replaces: eval_potential / eval_efield  postprocess.py:112-133 */
int hvb_field(const double* src, const double* cls, const double* groups, const int* tri_cols, int nt, int nq,
              const double* pts,
              const int* own_col, int m, int split, int potential, double* part, int* near_list,
              unsigned long long* near_count, long long near_cap, void* stream);

int hvb_field_reduce(const double* part, int split, int m, double* out, void* stream);

int hvb_near_apply_points(const int* seg_ptr, int n_seg, const int* pairs, const double* contrib,
                          const int* tri_cols, const double* u, int potential, double* out, void* stream);

/* K11 -- singular star of collocation points with the E kernel, jump term
 * side*u_i/2*n_i and |E|.  Replaces: surface_field_magnitudes
 * postprocess.py:141-170 */
int hvb_field_singular(const double* nodes6, const int* tri_cols, const int* vc_ptr, const int* vc_tri,
                       const int* vc_corner, const double* rule, int n_rule, const double* pts,
                       const double* normals, const int* own_col, int m, const double* u, double side,
                       double* efield, double* emag, void* stream);

/* K12-K14 -- device-resident field-line tracer (csrc/trace.cu).
 * state: n_lines opaque records of hvb_line_state_bytes() bytes.
 * geo: HOST pointer to 14 doubles = bbox centre (3), half extent x bbox_factor (3), diag,
 * h_min, h_max, l_max, rel_tol, surface_tol_frac, e_floor, max_steps (0 =
 * unbounded, as the reference; else lines end with termination 4 MaxSteps).
 * mode 0 initialises every line from starts/orient and requests E at the
 * start; mode 1 consumes E results (e_out/e_flag, indexed by the previous
 * request slots); mode 2 consumes surface distances (sd_out).  New E / SD
 * requests are appended to e_pts/e_line and sd_pts/sd_line through
 * counters[0] / counters[1]; counters[2] = max points per line, counters[3] =
 * total E requests, counters[4] = N-body work counter (6 entries); polylines (n_lines, cap, 5) = x, y, z, |E|, s.
 * Replaces: trace_fieldline  postprocess.py:244-357 (control flow, step
 * control, surface-hit snapping, termination order) */
int hvb_line_state_bytes(void);
int hvb_trace_ctrl(void* state, int n_lines, const double* starts, const int* orient, const double* geo, int mode,
                   double* e_pts, int* e_line, double* sd_pts, int* sd_line, unsigned long long* counters,
                   const double* e_out, const int* e_flag, const double* sd_out, double* out_pts,
                   int cap, void* stream);

/* One tracer round with no host synchronisation: the field of the current
 * request list cur_pts (count = counters[0], on the device; N-body over
 * src/cls with `split` panel chunks into part (split, n_lines, 4); has_near
 * (split, n_lines) int32 chunk flags, zero on entry and left zero; near pass
 * per flagged chunk in panel order with vertex-coincidence flags), then
 * counters[0..1] = 0, the consume-E control step (new requests into
 * nxt_pts/nxt_line), the surface distances of counters[1] queries and the
 * consume-SD control step.  Rounds are enqueued back to back; the host
 * reads counters only every few rounds.  Replaces: the per-stage
 * eval_efield / _surface_distance calls of trace_fieldline
 * postprocess.py:262-330 */
int hvb_trace_round(void* state, int n_lines, const double* geo, double* cur_pts, double* nxt_pts, int* nxt_line,
                    double* sd_pts, int* sd_line, double* sd_out, unsigned long long* counters, double* e_out,
                    int* e_flag, int* has_near, double* part, const double* src, const double* cls,
                    const double* groups, const int* tri_cols, int nt, int nq, int split, const double* nodes6, const double* radii,
                    const double* ccr, const double* u, const double* duffy, int n_duffy, const double* graded,
                    int n_graded, int bisect_depth, double bisect_trigger, double prox, double* out_pts, int cap,
                    void* stream);

/* per line (npts, termination, status, phase) and the start |E| of a
 * weak-start line */
int hvb_trace_summary(const void* state, int n_lines, int* info, double* dinfo, void* stream);

/* K12 -- approximate distance to the curved surface and local circumradius
 * at m points: 12 circumcircle candidates ranked by ||x-cc||-R, flat
 * closest point mapped through the quadratic patch, first minimum wins.
 * out (m, 2).  Replaces: _surface_distance  postprocess.py:198-218 */
int hvb_surface_distance(const double* pts, int m, const double* ccr, const double* groups, int nt,
                         const double* nodes6, double* out, void* stream);

/* flag[i] = 1 for near-pair targets within prox of a node of the pair's
 * panel.  Replaces: _check_point  postprocess.py:104-109 for tracer
 * requests */
int hvb_near_coincide(const int* pairs, long long n_pairs, const double* pts, const double* nodes6, double prox,
                      int* flag, void* stream);

/* K14 -- streamer integral per traced line: trapezoid of alpha(|E|)
 * (linear table interpolation, constant outside) over arc length, verdict
 * value > k_str.  Replaces: streamer_integral  postprocess.py:365-374 */
int hvb_streamer(const double* out_pts, const void* state, int n_lines, int cap, const double* e_tab,
                 const double* a_tab, int n_tab, double k_str, double* value, int* verdict, void* stream);

/* Roofline denominators measured on the box (bench.py): DFMA throughput
 * kernel (blocks x 256 threads x iters x 64 FMAs) and a read-only stream. */
int hvb_bench_dfma(double* out, int blocks, int iters, void* stream);
int hvb_bench_read(const double* p, long long n, double* out, int blocks, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HVB_H_ */
