/* hdk — the thin C-ABI layer between the heterodyn host library (C++) and
 * its sm_100a kernels.  Every entry point takes device pointers, plain sizes
 * and a cudaStream_t (passed as void*), launches asynchronously and returns
 * 0 or a CUDA error number; no exceptions, no torch types.  Device-side
 * solver failures are reported through the int error word in hdk_step
 * (first failing code wins) using the hd_status numbering of heterodyn.h.
 *
 * Each launcher names the reference routine it replaces
 * (paths relative to /root/reference/proj/src).
 */
#ifndef HDK_H
#define HDK_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDK_API __attribute__((visibility("default")))

/* Element-parallel mesh data, structure-of-arrays (mesh.hpp:16-60). */
typedef struct hdk_mesh {
  int nv, ne;
  const int* elem;        /* 4*ne vertex ids, element-major */
  const double* bm;       /* 9*ne: Dm^{-1}(r,c) at bm[(3r+c)*ne + e] */
  const double* mass;     /* nv lumped vertex masses */
  const int* inc_off;     /* nv+1: incident (element, slot) lists per vertex */
  const int* inc;         /* 4*ne entries 4*e + slot, ascending e per vertex */
} hdk_mesh;

/* Per-element weights with the rest volume folded in (material.hpp:40-50). */
typedef struct hdk_material {
  int kind;               /* 0 corotated, 1 neo-hookean */
  int barrier;            /* corotated + log-volume barrier */
  double mu_bar, lambda_bar, k_bar; /* prox means (material.cpp:64-71) */
  const double* w1;       /* NH: (2mu+lambda)V ; corotated: 2mu V */
  const double* w2;       /* corotated: lambda V (unused for NH) */
  const double* mu_e;     /* barrier parameters per element */
  const double* lambda_e;
  const double* beta_vh;  /* beta_e V / h, or NULL when beta0 == 0 */
  const double* vol;      /* rest volumes */
  /* Segmented batch (lockstep C5 engine): seg_ne elements per sample; the
   * prox means of sample s are seg_means[3 s .. 3 s + 2] (mu, lambda, k),
   * and hdk_differential reads sample s's tau at tau[s * tau_stride].
   * seg_means == NULL: the scalars above, one tau. */
  const double* seg_means;
  int seg_ne, tau_stride;
} hdk_material;

/* Explicit inverse factor A^{-1} = S'^T S' in postordered elimination order.
 * Row r of S' is dense over columns [r - len_r + 1, r] (its etree subtree),
 * so no column indices are stored.  Columns are cut into tiles of tile_w;
 * a segment is one row's part inside one tile.  The values are stored
 * tile-major as one stream of chunks: a chunk is a 16-byte aligned contiguous
 * block of at most HDK_CHUNK_VALS values holding whole segments of one tile,
 * with its segment descriptors contiguous too.  Each pass hands every
 * persistent CTA an equal contiguous range of chunks, streamed into shared
 * memory with bulk asynchronous copies (factor.cpp:106-109). */
#define HDK_CHUNK_VALS 3072
#define HDK_CHUNK_SEGS 64 /* caps the per-stage segment (and pass-2 z-row) staging */

typedef struct hdk_seg {   /* 16 bytes */
  int row;                 /* S' row */
  int pslot;               /* slot of this segment's partial row dot */
  int clo_len;             /* first column within the tile | (len << 16) */
  int coff;                /* offset of the first value within the chunk */
} hdk_seg;

typedef struct hdk_chunk {  /* 24 bytes */
  long long off;            /* stream offset (doubles, even) */
  int len;                  /* values incl. padding (even) */
  int seg0, nseg;           /* descriptors [seg0, seg0 + nseg) */
  int tile;
} hdk_chunk;

typedef struct hdk_factor {
  int n;                  /* free vertices */
  int tile_w, n_tiles, n_chunks;
  int max_ctas;           /* part2 holds (n_tiles + max_ctas) tile partials */
  int l2_hint;            /* 1: stream the values with an L2 evict_first policy */
  const int* run_flag;    /* optional: the passes do nothing while *run_flag == 0 (an unrolled
                             iteration past convergence) */
  int grid_cap;           /* 0: one resident wave per pass; else at most this many CTAs per pass
                             (lets concurrent samples of a batch share the SMs) */
  const double* sval;     /* tile-major value stream */
  const hdk_seg* seg;
  const hdk_chunk* chunk;
  const int* tile_chunk;  /* n_tiles+1: first chunk of each tile */
  const int* row_pslot;   /* n+1: partial-dot slots of row r */
  int n_pslot;            /* row_pslot[n] */
  int n_ztask;
  const int2* ztask;      /* z-fold warp tasks: {row, -1} one long row, {first row, k} k <= 4 short rows */
  const int* p2v;         /* n: elimination position -> vertex */
  const int* v2p;         /* nv: vertex -> position or -1 (fixed) */
  double* part1;          /* 3*row_pslot[n] scratch */
  double* part2;          /* 3*tile_w*(n_tiles+max_ctas) scratch */
  double* z;              /* 3*n scratch */
  /* Cost-balanced CTA ranges (chunk cost = values + alpha * segments), built
   * on the host for the grids hdk_solve_grids reports; NULL = equal chunk
   * counts per CTA. */
  int grid1, grid2;
  const int* first1;      /* grid1+1: first chunk of pass-1 CTA b */
  const int* first2;      /* grid2+1: first chunk of pass-2 CTA b */
  const int* tile_cta2;   /* 2*n_tiles: first and last pass-2 CTA touching tile t */
  const int2* vfold;      /* nv: (first tile-partial slot of the vertex's column, slot count; 0 if fixed) */
  /* fp32 copy of the value stream for preconditioner-only solves (the
   * adjoint CG: an approximate SPD preconditioner leaves CG's answer and
   * its residuals exact).  chunk32: the chunks with offsets into sval32
   * (each chunk padded to a multiple of 4 values for 16-byte bulk copies);
   * use32 != 0 makes hdk_apply_inverse3_* stream sval32. */
  const float* sval32;
  const hdk_chunk* chunk32;
  int use32;
} hdk_factor;
/* sval32[chunk32[c].off + i] = (float) sval[chunk[c].off + i], padding 0. */
HDK_API int hdk_factor_to_fp32(const hdk_factor* f, float* sval32, const hdk_chunk* chunk32, void* stream);

/* Scalar CSR in elimination order (a_free / a_free_fixed, factor.hpp:98-99). */
typedef struct hdk_csr {
  int rows;
  const int* off;
  const int* col;
  const double* val;
} hdk_csr;

/* Device build of the factor values (inverse.cu): S' = D^{-1/2} L^{-1}
 * column by column along the elimination tree, written straight into the
 * tile-major stream (zero-initialised, stream_len values).  Bitwise the host
 * build's values; fails with cudaErrorInvalidValue if the tree is too deep
 * for a path to fit in shared memory. */
typedef struct hdk_inverse_build {
  int n, max_depth, tile_w;
  const int* parent;       /* n, postordered elimination tree, -1 at roots */
  const int* depth;        /* n, distance to the root */
  const long long* lp;     /* n+1, L by columns */
  const int* ldist;        /* depth(v) - depth(row) of each entry of L(:, v) */
  const double* lx;        /* L values */
  const double* dis;       /* D^{-1/2} */
  const int* row_first;    /* n, first column of row r of S' */
  const int* row_pslot;    /* n+1, (row, tile) segment slots */
  const long long* seg_off;  /* per slot: stream index of the segment's first value */
  const int* seg_clo;      /* per slot: its first column */
} hdk_inverse_build;
HDK_API int hdk_inverse_values(const hdk_inverse_build* b, double* stream, void* stream_handle);

/* Solve x = A^{-1} rhs on 3 axes: rhs in elimination order [n][3]; the result
 * is scattered into out_full[3*v+a] for free vertices (fixed entries are not
 * touched).  Replaces GlobalSystem::solve_free (factor.cpp:196-208). */
HDK_API int hdk_apply_inverse3(const hdk_factor* f, const double* rhs_perm, double* out_full, void* stream);
/* Grid sizes (CTAs) of the two streaming passes hdk_apply_inverse3 launches
 * for this factor (persistent: one resident wave, capped by grid_cap). */
HDK_API int hdk_solve_grids(const hdk_factor* f, int* grid1, int* grid2);
/* Same, result kept in elimination order (out_perm [n][3]). */
/* Solve passes without the final fold: the tile partials stay in f->part2
 * for hdk_aa_dots_fused. */
HDK_API int hdk_apply_inverse3_partial(const hdk_factor* f, const double* rhs_perm, void* stream);
/* R independent right-hand sides (R = 1, 2, 4) through one stream of the
 * factor: rhs_perm holds R vectors [n][3] back to back; part1, z and part2
 * must be sized for R columns (column c's tile partials at
 * part2 + c * hdk_factor_part2_stride(f)).  Leaves the tile partials for the
 * callers' folds, like hdk_apply_inverse3_partial. */
HDK_API int hdk_apply_inverse3_multi(const hdk_factor* f, const double* rhs_perm, int columns, void* stream);
HDK_API size_t hdk_factor_part2_stride(const hdk_factor* f);
/* Profiling only: hdk_apply_inverse3_partial with passes dropped (bit 0 row
 * dots, bit 1 z-fold, bit 2 column pass). */
HDK_API int hdk_apply_inverse3_ablate(const hdk_factor* f, const double* rhs_perm, unsigned skip, void* stream);
HDK_API int hdk_apply_inverse3_perm(const hdk_factor* f, const double* rhs_perm, double* out_perm, void* stream);

/* Per-element local step (local_solve + the element part of pd_rhs,
 * forward.cpp:70-117).  Writes the weighted element force V G^T target
 * (12 doubles per element) and, when cache != NULL, the projection cache
 * (24 doubles per element: sigma*, sigma_F, U, V; corotated adds 3 more for
 * the volume target).  Errors: PROX_DIVERGED (6) into *err. */
/* A/B switch of the local step's Newton direction: 1 = always the 3x3
 * eigen-solve, 0 = Sherman-Morrison when the eigenvalue floor is inactive. */
HDK_API int hdk_set_newton_eigen(int on);
HDK_API int hdk_local_step(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                           double* cache, int* err, void* stream);

/* V_e * model energy density at q (backward.cpp:23-73, element part); *bad
 * receives NON_POSITIVE_JACOBIAN (5) or PROX_DIVERGED (6). */
HDK_API int hdk_element_energy(const hdk_mesh* m, const hdk_material* mat, const double* q, double* energy, int* bad,
                               void* stream);
/* Both energies of the trust-region test (q*^{-1} and q*) in one launch. */
HDK_API int hdk_element_energy2(const hdk_mesh* m, const hdk_material* mat, const double* q1, double* energy1,
                                const double* q2, double* energy2, int* bad, void* stream);
/* Compact prox differential per element from the projection cache and the
 * device scalar *tau (tr_blend + nh/polar/volume/barrier differentials,
 * localstep.cpp:276-423): 30 doubles SoA.  Errors: SINGULAR_FILTERED_HESSIAN. */
HDK_API int hdk_differential(const hdk_mesh* m, const hdk_material* mat, const double* cache, const double* tau,
                             double* dcomp, int* err, void* stream);
/* Element forces of B x (matrix-free assemble_db_dq + apply, backward.cpp:117-163). */
HDK_API int hdk_bapply(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force, void* stream);
/* hdk_bapply with each corner force stored at its slot of the elimination-
 * order incidence list (corner_pos[4 e + k] = index into hdk_vtx::pinc, -1
 * for fixed vertices); read back by hdk_gather_sorted.  corner_pos NULL: the
 * plain layout.  Does nothing while *run_flag == 0. */
HDK_API int hdk_bapply_sorted(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                              const int* corner_pos, const int* run_flag, void* stream);
/* B x for a segmented batch's per-sample CG: samples whose CG has ended
 * (cond0[sample * cond_stride] == 0) are skipped. */
HDK_API int hdk_bapply_sorted_seg(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                                  const int* corner_pos, const int* cond0, int cond_stride, int seg_ne, void* stream);
/* hdk_bapply that does nothing while *run_flag == 0 (unrolled backbone). */
HDK_API int hdk_bapply_flag(const hdk_mesh* m, const double* dcomp, const double* x, double* elem_force,
                            const int* run_flag, void* stream);
/* Per-element dL/dw (accumulated into dl_dw), dL/dE (accumulated into dl_de)
 * and the damping element force of mu (backward.cpp:311, 361-391). */
HDK_API int hdk_route_elements(const hdk_mesh* m, const hdk_material* mat, const double* cache, const double* q_star,
                               const double* mu, double unit_mu, double unit_lambda, double* dl_dw, double* dl_de,
                               double* ef_damp, void* stream);
/* Element forces of the stiffness-damping term beta_e V_e / h G^T F(q)
 * (damping_rhs, forward.cpp:119-138). */
HDK_API int hdk_damping_elements(const hdk_mesh* m, const double* beta_vh, const double* q, double* elem_force,
                                 void* stream);

/* ---- loop control block (device-resident) ------------------------------- */
#define HDK_AA_MAX 8
#define HDK_RED_BLOCKS 296 /* 2 x 148 SMs: fixed reduction grid (deterministic) */
#define HDK_RED_Q 24       /* partial slots per block */

typedef struct hdk_ctl {
  int k, k_max, iterations, converged;
  int err, done, bad, cond;
  int window, count, head, has_last, mixed, nonfinite;  /* nonfinite: set by the backbone mix */
  double eps_rel, eps_abs, guard, tol;
  double gamma[HDK_AA_MAX];
  double gram[HDK_AA_MAX * HDK_AA_MAX];
  double red[HDK_RED_Q];
  double tau, rho, model, eps_tr;
} hdk_ctl;
/* Forward sweeps whose forces feed the sorted rhs gathers: corner k of
 * element e writes its force at slot corner_vpos[4 e + k] of the
 * vertex-ordered incidence list (3 doubles per slot); no projection cache.
 * _seg: elements of samples whose loop has ended (ctl[sample].cond == 0)
 * are skipped (corner_vpos may be NULL there: element order). */
HDK_API int hdk_local_step_seg(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                               int* err, const hdk_ctl* ctl, const int* corner_vpos, void* stream);
HDK_API int hdk_local_step_sorted(const hdk_mesh* m, const hdk_material* mat, const double* q, double* elem_force,
                                  int* err, const int* corner_vpos, void* stream);

/* Vector kernels (vec.cu).  Vectors are full xyz-interleaved (3 nv) unless
 * named *_perm ([n][3] in elimination order). */
typedef struct hdk_vtx {
  int nv, n;
  const int* v2p;         /* nv */
  const int* p2v;         /* n */
  const double* mass;     /* nv */
  const int* inc_off;
  const int* inc;
  const int* pinc_off;    /* n+1: incidence offsets in elimination order (optional) */
  const int* pinc;        /* incidence lists concatenated in elimination order */
} hdk_vtx;

/* q~ = q + h v + h^2 (f_ext + hook) / m; q_cur = q~ with fixed rows pinned to q
 * (free_fall_target + pin, forward.cpp:59-68,165-169,210-211). */
HDK_API int hdk_free_fall(const hdk_vtx* x, const double* q, const double* v, const double* f_ext, double h,
                          int hook_vertex, const double* hook /* ax ay az k d */, double* q_tilde, double* q_cur,
                          void* stream);
/* out[v] = cm * m_v * base[v] + add[v] + sum of element forces at v (add may be NULL). */
HDK_API int hdk_gather(const hdk_vtx* x, const double* ef, double cm, const double* base, const double* add,
                       double* out, void* stream);
/* Forward rhs b = M/h^2 q~ + damp + sum ef (pd_rhs, forward.cpp:96-117);
 * rhs_perm = b - A_fd q_d at free rows; gate partials of |b - b_prev|, |b|;
 * b_prev <- b. */
HDK_API int hdk_gather_rhs(const hdk_vtx* x, const double* ef, double inv_h2, const double* q_tilde, const double* damp,
                           const double* fixcoup, double* b_prev, double* rhs_perm, double* partial, void* stream);
/* The same from forces stored by incidence slot (hdk_local_step_sorted). */
HDK_API int hdk_gather_rhs_sorted(const hdk_vtx* x, const double* efs, double inv_h2, const double* q_tilde,
                                  const double* damp, const double* fixcoup, double* b_prev, double* rhs_perm,
                                  double* partial, void* stream);
/* rhs_perm[p] = base[p2v[p]] (+ element forces when ef != NULL). */
HDK_API int hdk_gather_perm(const hdk_vtx* x, const double* base, const double* ef, double* rhs_perm, void* stream);
/* rhs_perm[p] = base_perm[p] (0 if base_perm is NULL) + element forces,
 * through the elimination-order incidence (x->pinc_off / x->pinc). */
HDK_API int hdk_gather_pp(const hdk_vtx* x, const double* base_perm, const double* ef, double* rhs_perm,
                          const int* run_flag, void* stream);
/* Same sums from forces already in incidence order (hdk_bapply_sorted):
 * contiguous reads, no index indirection; bitwise the same result. */
HDK_API int hdk_gather_sorted(const hdk_vtx* x, const double* base_perm, const double* ef_sorted, double* rhs_perm,
                              const int* run_flag, void* stream);
/* fixcoup[p] = sum_k A_fd(p, k) q[fixed_k] (solve_free's coupling, factor.cpp:201-205). */
HDK_API int hdk_fixed_coupling(const hdk_csr* a_fd, const int* fixed, const double* q, double* fixcoup, void* stream);
/* Type-II Anderson mixing (forward.cpp:17-51) in three launches: history
 * update + dot partials, coefficient solve (1 block), mix.  mode 0: forward
 * (pins fixed rows, gate partials, rotates q_prev <- q_cur <- q_next);
 * mode 1: adjoint backbone (convergence test |t-x| <= tol |t|, backward.cpp:188-199). */
HDK_API int hdk_aa_dots(const hdk_vtx* x, hdk_ctl* ctl, const double* qhat, const double* qcur, double* last_q,
                        double* last_g, double* dq, double* dg, double* partial, void* stream);
HDK_API int hdk_aa_solve(hdk_ctl* ctl, const double* partial, int mode, void* stream);
/* Fused iteration tail after hdk_apply_inverse3_partial: folds the solve's
 * pass-2 tile partials into qhat (free rows, full vertex order; fixed rows are
 * read as they are), then hdk_aa_dots, then — in the block that finishes last —
 * hdk_aa_solve; mode 1 also sets the WHILE condition (cond_handle != 0).
 * ticket: one zero-initialised device counter per concurrent stream. */
HDK_API int hdk_aa_dots_fused(const hdk_vtx* x, const hdk_factor* f, hdk_ctl* ctl, double* qhat, const double* qcur,
                              double* last_q, double* last_g, double* dq, double* dg, double* partial,
                              unsigned int* ticket, int mode, unsigned long long cond_handle, void* stream);
/* Profiling: in-graph timeline of the backbone kernels (launch.cuh TraceId).
 * hdk_trace_install_{local,vec,solve} point each translation unit at a
 * buffer (NULL: off); hdk_trace_epoch advances its record slot. */
HDK_API int hdk_trace_install_local(unsigned long long* buf);
HDK_API int hdk_trace_install_vec(unsigned long long* buf);
HDK_API int hdk_trace_install_solve(unsigned long long* buf);
HDK_API int hdk_trace_epoch(unsigned long long* buf, void* stream);
/* Adjoint backbone in elimination order ([n][3]), one iteration =
 *   solve -> hdk_bb_dots -> { hdk_bb_solve || B t, gather } -> hdk_bb_mix.
 * hdk_bb_dots: t folded from the solve's tile partials by column (also
 * written by vertex to t_full), Anderson history update and dot partials;
 * block 0 snapshots ctl into snap.  hdk_bb_solve (1 block): coefficient
 * solve from snap (convergence test first), publishes the new state and the
 * WHILE condition to ctl, the mixing inputs to `result`
 * (hdk_bb_result_bytes()).  The x-space ring `dq` of hdk_bb_dots holds
 * s_j = dq_j + dg_j (sum_hist), `dg` holds dg_j.  hdk_bb_mix: x <- t -
 * sum gamma s_j and, by linearity, R(x) <- R(t) - sum gamma R(s_j) with
 * R = gather o B (rt_perm = R(t) from the branch; rsum_hist = R(s_j));
 * rhs_perm = seed_perm + R(x). */
HDK_API int hdk_bb_dots(const hdk_factor* f, hdk_ctl* ctl, hdk_ctl* snap, double* t_perm, double* t_full,
                        const double* x_perm, double* last_q, double* last_g, double* dq, double* dg, double* partial,
                        int mode, void* stream);
HDK_API int hdk_bb_solve(hdk_ctl* ctl, const hdk_ctl* snap, const double* partial, void* result,
                         unsigned long long cond_handle, void* stream);
HDK_API size_t hdk_bb_result_bytes(void);
/* *any = OR over count (<= 32) control blocks of "still iterating"; sets the
 * WHILE condition when cond_handle != 0 (multi-column contact adjoint). */
HDK_API int hdk_any_cond(hdk_ctl* ctls, int count, int* any, unsigned long long cond_handle, void* stream);
/* *any = 1 while exactly *expected (> 0) of the count columns are still iterating
 * (the contact-adjoint column refill loop); sets the WHILE condition. */
HDK_API int hdk_cols_cond(hdk_ctl* ctls, int count, const int* expected, int* any, unsigned long long cond_handle,
                          void* stream);
HDK_API int hdk_bb_mix(const hdk_factor* f, hdk_ctl* ctl, const hdk_ctl* snap, const void* result,
                       const double* t_perm, double* x_perm, double* x_full, const double* sum_hist,
                       const double* rt_perm, double* rx_perm, double* last_rx, double* last_rg, double* rsum_hist,
                       const double* seed_perm, double* rhs_perm, void* stream);
HDK_API int hdk_aa_mix(const hdk_vtx* x, hdk_ctl* ctl, const double* qhat, double* qcur, double* qprev,
                       const double* qpin, const double* dq, const double* dg, double* partial, int mode, void* stream);
/* Dual gate (forward.cpp:140-146) and loop condition for the graph while node. */
HDK_API int hdk_gate(hdk_ctl* ctl, const double* partial_b, const double* partial_q, unsigned long long cond_handle,
                     void* stream);

/* A_ff dq dot partials for the trust-region model (backward.cpp:77-79). */
HDK_API int hdk_tr_model(const hdk_vtx* x, const hdk_csr* a_ff, const double* q_star, const double* q_prev,
                         double* dq_perm, double* partial, void* stream);
/* Energy partials and rho / tau selection (backward.cpp:75-108). */
HDK_API int hdk_tr_select(const hdk_vtx* x, int ne, const double* e_prev, const double* e_star, const double* q_prev,
                          const double* q_star, const double* q_tilde, double inv_h2, const double* model_partial,
                          double* partial, hdk_ctl* ctl, void* stream);
/* Vertex part of route_gradients (backward.cpp:296-356) and the chain update
 * (drivers.cpp:84-95). */
HDK_API int hdk_route_vertices(const hdk_vtx* x, const double* mu, const double* ef_damp, const double* b_mu,
                               const double* q_bar, const double* v_bar, const double* coup_fixed, double h,
                               double alpha, int hook_vertex, double hook_k, double hook_d, double* dl_dq_t,
                               double* dl_dv_t, double* dl_df_acc, void* stream);
/* coup[v] = sum_p A_fd(p, k(v)) mu[p2v[p]] for fixed vertices (A_fd^T mu). */
HDK_API int hdk_fixed_coupling_t(const hdk_csr* a_df, const int* fixed, const int* p2v, const double* mu, double* coup,
                                 void* stream);
/* Resets the loop-control block (first kernel of every step graph). */
HDK_API int hdk_ctl_init(hdk_ctl* ctl, int window, double guard, int k_max, double eps_rel, double eps_abs, double tol,
                         double eps_tr, int iterations0, void* stream);
/* Resets the loop counter and Anderson history only (tau/rho/err kept). */
HDK_API int hdk_aa_reset(hdk_ctl* ctl, int window, double guard, int k_max, double tol, void* stream);
/* State commit after a successful step: v = (q* - q)/h, q = q* (skipped when
 * ctl->err != 0 so a failed step leaves the state intact, heterodyn.h:87-90). */
HDK_API int hdk_commit(int n, const hdk_ctl* ctl, const double* q_star, double h, double* q, double* v, void* stream);

/* ---- batched system-ID reductions (batch.cu) ---------------------------
 * out = 1/2 |q - ref|^2 (n doubles, one deterministic block). */
HDK_API int hdk_half_sqdist(int n, const double* q, const double* ref, double* out, void* stream);
/* out[0] = sum_s loss[s], out[1 + i] = sum_s vec[s][i] in sample order; vec is
 * a device array of `samples` device pointers to n doubles. */
HDK_API int hdk_batch_sum(int samples, int n, const double* const* vec, const double* loss, double* out,
                          void* stream);
/* y = a x + b z elementwise over n doubles (z may be NULL). */
HDK_API int hdk_axpby(int n, double a, const double* x, double b, const double* z, double* y, void* stream);
/* v* = (q* - q_t)/h (forward.cpp:253). */
HDK_API int hdk_velocity(int n, const double* q_star, const double* q_t, double h, double* v_star, void* stream);

/* ---- contact (contact.cu) ------------------------------------------------ */
/* One step's contact set on the device, in the reference's stacked row order:
 * nc normal rows, then two tangent rows per frictional contact
 * (contact.hpp:59-88).  Every array is sized for the capacities; the live
 * counts are device-resident (cnt), written by hdk_contact_setup, so the
 * whole contact step runs inside the forward CUDA graph without a host round
 * trip.  cnt: HDK_CNT_* below. */
#define HDK_CNT_NC 0
#define HDK_CNT_NF 1
#define HDK_CNT_K 2
#define HDK_CNT_NU 3
#define HDK_CNT_OVERFLOW 4   /* capacities exceeded: the step is voided (ctl->err = HDK_ERR_CAPACITY) */
#define HDK_CNT_SPIKE 5      /* next unique slot of the inverse-column loop */
#define HDK_CNT_SPIKE_COND 6 /* inverse-column loop still running */
#define HDK_CNT_NEED_C 7     /* counts that overflowed: contacts, rows, unique vertices */
#define HDK_CNT_NEED_K 8
#define HDK_CNT_NEED_U 9
#define HDK_CNT_INTS 16
#define HDK_ERR_CAPACITY 100 /* internal: grow the contact capacities and re-run the step */

typedef struct hdk_contacts {
  int cap_c, cap_k, cap_u;  /* capacities: contacts, rows, unique vertices */
  int n;                    /* free vertices (leading dimension of U) */
  int* cnt;                 /* HDK_CNT_INTS device counters */
  int* vertex;              /* cap_c: contact vertex (vertex-major, obstacle-minor scan order) */
  int* obstacle;            /* cap_c: obstacle id */
  double* normal;           /* 3 cap_c */
  double* t1;               /* 3 cap_c */
  double* t2;               /* 3 cap_c */
  double* gap;              /* cap_c: gap offsets n.x - sd */
  double* mu;               /* cap_c: friction coefficients */
  double* r_n;              /* cap_c: h^2 W_nn */
  double* r_f;              /* cap_c: h^2 mean tangent W */
  int* fric;                /* cap_c: contact index of the f-th frictional contact */
  int* fpre;                /* cap_c+1: frictional contacts before contact i */
  int* row_unique;          /* cap_k: unique-vertex slot of each row */
  int* urow_off;            /* cap_u+1 */
  int* urow;                /* cap_k: rows of each unique vertex, ascending */
  int* unique_pos;          /* cap_u: elimination position of each unique vertex */
  int* nfirst;              /* cap_u+1: first contact of each unique vertex */
  double* U;                /* n x cap_u scalar inverse columns A_s^{-1} e_{p(u)} (column-major) */
  double* W;                /* k x k Delassus matrix (leading dimension k) within cap_k^2 */
  double* lambda;           /* cap_k multipliers */
  double* omega;            /* cap_k NCP weights (weights_star after the step) */
  double* e_diag;           /* cap_k */
  double* g;                /* 3 cap_u: per unique vertex sum of omega lambda d over its rows */
  double* y;                /* cap_k: reduced adjoint multipliers (backward) */
} hdk_contacts;

/* Device bytes of a contact block with these capacities, and the carving of
 * one such block (base: that many bytes, 256-aligned) into *c. */
HDK_API size_t hdk_contact_block_bytes(int cap_c, int cap_k, int cap_u, int n);
HDK_API void hdk_contact_block_layout(void* base, int cap_c, int cap_k, int cap_u, int n, hdk_contacts* c);

/* Per-iteration contact trace (parity observability, B200 extension): the
 * decision values of project_multipliers (contact.cpp:218-235) —
 * clamp[it * cap_c + i] = normal multiplier i before the clamp of iteration
 * it (clamped iff < 0), cone[it * cap_c + f] = (|lambda_t| - mu lambda_n) /
 * (mu lambda_n) of frictional contact f before the projection (projected iff
 * > 0; -1 when mu lambda_n = 0, where the pair is zeroed either way).
 * Iterations >= cap are not recorded. */
typedef struct hdk_contact_trace {
  double* clamp;
  double* cone;
  int cap;
} hdk_contact_trace;

/* Detection at q (free vertices x obstacles, vertex-major / obstacle-minor,
 * signed distance <= margin: detect_contacts contact.cpp:117-144), the
 * order-preserving compaction, the contact geometry (normal, gap offset,
 * tangent basis, contact.cpp:39-66), the frictional list, the unique-vertex
 * rows, zero multipliers and the counts, in one single-CTA kernel.
 * obstacles: HDK_OBSTACLE_DOUBLES each {kind(0 half-space, 1 sphere), nx, ny,
 * nz, offset|radius, cx, cy, cz, friction, -, -, -}.  Sets the inverse-column
 * loop's WHILE condition (nu > 0) when cond_handle != 0.  On overflow the
 * counts read 0, HDK_CNT_NEED_* hold the sizes and ctl->err =
 * HDK_ERR_CAPACITY. */
#define HDK_OBSTACLE_DOUBLES 12
HDK_API int hdk_contact_setup(int nv, const int* v2p, const double* q, int n_obstacles, const double* obstacles,
                              double margin, const hdk_contacts* c, hdk_ctl* ctl, unsigned long long cond_handle,
                              void* stream);
/* Inverse-column loop body (factor.cpp:237-289): unit spikes of the next
 * three unique vertices into the three axes of rhs_perm; after the solve,
 * their columns into U and the loop advanced (WHILE condition). */
HDK_API int hdk_contact_spikes(const hdk_contacts* c, double* rhs_perm, void* stream);
HDK_API int hdk_contact_unspike(const hdk_contacts* c, const double* x_perm, unsigned long long cond_handle,
                                void* stream);
/* W(r, s) = (d_r . d_s) U[p(u_s), u_r] and r_n = h^2 W_nn, r_f = h^2 (W_t1t1 + W_t2t2)/2
 * (Delassus, factor.cpp:237-289; forward.cpp:178-193). */
HDK_API int hdk_contact_delassus(const hdk_contacts* c, double h, void* stream);
/* NCP weights at (q, q_t, lambda) into omega / e_diag (contact_weights,
 * contact.cpp:160-196); the post-loop weights_star. */
HDK_API int hdk_contact_weights(const hdk_contacts* c, const double* q, const double* q_t, void* stream);
/* One multiplier update of the PD loop (forward.cpp:226-235): NCP weights at
 * q_cur, J q_mid = J q0 + W (omega o lambda), the lifted system
 * M = Omega W Omega + E + lift I and offset vector (contact_iteration /
 * offset_vector, contact.cpp:198-256), its LDL^T solve (dense.cuh), the
 * projection (contact.cpp:218-235) and the per-unique-vertex coefficients g
 * of the corrected iterate.  One CTA.  Errors: SINGULAR_CONTACT_SYSTEM (9).
 * trace may be NULL. */
HDK_API int hdk_contact_ncp(const hdk_contacts* c, const double* q_cur, const double* q_t, const double* q0,
                            double* M_scratch, hdk_ctl* ctl, const hdk_contact_trace* trace, void* stream);
/* Scratch doubles hdk_contact_ncp / hdk_contact_reduced need in global memory
 * for these capacities (0 when the system fits in shared memory). */
HDK_API size_t hdk_contact_scratch_doubles(int cap_k);
/* Test hook: out[i] = hypot(x[i], y[i]) as the contact kernels compute it
 * (glibc-exact, dense.cuh); device arrays. */
HDK_API int hdk_test_hypot(const double* x, const double* y, double* out, int n, void* stream);
/* Largest row capacity whose system factors in shared memory. */
HDK_API int hdk_contact_smem_rows(void);
/* out = q0 + A^{-1} J^T (omega o lambda) on free vertices through U
 * (contact_corrected, forward.cpp:196-206). */
HDK_API int hdk_contact_correct(const hdk_contacts* c, const int* p2v, const double* q0, double* out, void* stream);
/* Reduced adjoint multiplier system (backward.cpp:240-262): w_tan(d, c) =
 * d_d . X_c[v_d], symmetrised; M = Omega sym Omega + E + lift I; rhs =
 * omega o (J z0); LDL^T solve into c->y.  Errors: ADJOINT_DIVERGED (10). */
HDK_API int hdk_contact_reduced(const hdk_contacts* c, const double* X, size_t ldx, const double* z0,
                                double* M_scratch, int* err, void* stream);
/* mu = z0 - sum_c (omega_c y_c) X_c (backward.cpp:266-268). */
HDK_API int hdk_contact_combine(const hdk_contacts* c, int n3, const double* z0, const double* X, size_t ldx,
                                double* mu, void* stream);
/* Right-hand side e_v d_row and warm start a_row (backward.cpp:229-238) of one column. */
HDK_API int hdk_contact_column_init(const hdk_contacts* c, int row, int nv, const int* v2p, double* rhs, double* x0,
                                    void* stream);
/* Friction rows push back into dL/dq_t (backward.cpp:342-356). */
HDK_API int hdk_contact_friction_pushback(const hdk_contacts* c, double* dl_dq, void* stream);

/* Contact-adjoint columns (engine_columns.cpp): the per-column backbone
 * buffers of HDK_BB_COLUMNS columns, so each backbone stage is one launch
 * for all columns (blockIdx.y / blockIdx.x = column). */
#define HDK_BB_COLUMNS 8
typedef struct hdk_bb_column {
  hdk_factor f;  /* the column's view of the multi-column factor (part2 offset) */
  hdk_ctl* ctl;
  hdk_ctl* snap;
  void* res;
  double *t, *tv, *xp, *x, *lastq, *lastg, *dq, *dg, *part, *rt, *rx, *lrx, *lrg, *rsq, *ef, *rhs;
  const double* seedp;
} hdk_bb_column;
typedef struct hdk_bb_columns {
  hdk_bb_column col[HDK_BB_COLUMNS];
} hdk_bb_columns;
HDK_API int hdk_bb_columns_dots(const hdk_bb_columns* c, int mode, void* stream);
HDK_API int hdk_bb_columns_solve(const hdk_bb_columns* c, void* stream);
HDK_API int hdk_bb_columns_bapply(const hdk_mesh* m, const double* dcomp, const hdk_bb_columns* c, void* stream);
HDK_API int hdk_bb_columns_gather(const hdk_vtx* x, const hdk_bb_columns* c, void* stream);
HDK_API int hdk_bb_columns_mix(const hdk_bb_columns* c, void* stream);

/* ---- device refactorization (refactor.cu, refactor.hpp) -------------------
 * A's values for a fixed pattern (factor.cpp assemble, same order), the
 * multifrontal LDL^T over the supernodal elimination tree (one CTA per front,
 * one launch per tree level, panels of HDK_MF_PANEL pivot columns) and
 * D^{-1/2}; L lands in the host factor's column layout (lp), ready for
 * hdk_inverse_values.  Replaces SparseFactor::factorize (factor.cpp:11-104)
 * and assemble_global_scalar (factor.cpp:121-136) on a refactorization. */
#define HDK_MF_PANEL 8
typedef struct hdk_mf {
  int n, nsuper, nlevels;
  const int* sfirst;      /* nsuper + 1 */
  const int* fm;          /* front order per supernode */
  const long long* foff;  /* front offset in pool (m x m column-major) */
  const int* level_off;   /* nlevels + 1 */
  const int* level_node;
  const int* child_off;
  const int* child;
  const int* emap_off;
  const int* emap;        /* update rows -> parent front positions */
  const int* aent_off;
  const int* aent_src;    /* a_ff value index */
  const int* aent_dst;    /* front offset */
  const long long* lp;    /* L by columns */
  double* pool;
  const int* h_level_off; /* host copy of level_off (launch grids) */
  const int* h_level_maxm; /* host: largest front per level (CTA width) */
} hdk_mf;
/* W_e = (2 mu_e + lambda_e + beta_e / h) V_e */
HDK_API int hdk_asm_weights(int ne, const double* mu, const double* lambda, const double* beta, const double* vol,
                            double h, double* w, void* stream);
/* out[k] = [diag[k] >= 0] inertia m + sum over corner pairs pair[off[k]..off[k+1]) ((4e+i) << 2 | j) of W_e g_i.g_j */
HDK_API int hdk_asm_values(int count, const int* off, const int* pair, const int* diag, const double* mass,
                           double inertia, const double* w, const double* g, double* out, void* stream);
HDK_API int hdk_gather_values(int count, const int* from, const double* src, double* dst, void* stream);
/* L (lx, host layout), D and D^{-1/2}; a non-positive pivot sets *err = 8 (NotPositiveDefinite). */
HDK_API int hdk_mf_factor(const hdk_mf* p, const double* aval, double* lx, double* d, double* dis, int* err,
                          void* stream);

/* ---- adjoint backbone by preconditioned CG (pcg.cu) ----------------------
 * (A - B) x = s with the preconditioner A^{-1}: z = A^{-1} r is the
 * reference's t - x, so the loop stops on the reference's test
 * ||z|| <= tol ||x + z|| and returns x + z.  Vectors in elimination order
 * [n][3]; state on the device; err = -1: p.q <= 0 (not positive definite
 * along p, the caller falls back to the Anderson backbone), 10: cap. */
typedef struct hdk_pcg {
  double rz, pq, alpha, beta, tol;
  int iter, k_max, done, err, cond;
} hdk_pcg;
HDK_API int hdk_pcg_init(hdk_pcg* st, double tol, int k_max, void* stream);
HDK_API int hdk_pcg_r0(int n3, const double* s, const double* ax, const double* rx, double* r, void* stream);
HDK_API int hdk_pcg_spmv(const hdk_csr* a, const double* p, double* y, const hdk_pcg* st, void* stream);
HDK_API int hdk_pcg_rz(int n3, const double* r, const double* z, const double* x, double* partial,
                       unsigned int* ticket, hdk_pcg* st, void* stream);
HDK_API int hdk_pcg_cond(const hdk_pcg* st, unsigned long long cond_handle, void* stream);
/* p = z + beta p (and by vertex); sets the WHILE condition (last kernel of the body). */
HDK_API int hdk_pcg_p(int n, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                      unsigned long long cond_handle, void* stream);
/* q = A p - gather(B p) from the sorted element forces, p.q, alpha (one launch). */
HDK_API int hdk_pcg_apply(const hdk_vtx* x, const hdk_csr* a, const double* ef_sorted, const double* p, double* q,
                          double* partial, unsigned int* ticket, hdk_pcg* st, void* stream);
HDK_API int hdk_pcg_q(int n3, const double* ap, const double* rp, const double* p, double* q, double* partial,
                      unsigned int* ticket, hdk_pcg* st, void* stream);
HDK_API int hdk_pcg_xr(int n3, double* x, double* r, const double* p, const double* q, const hdk_pcg* st,
                       void* stream);
HDK_API int hdk_pcg_final(int n, const double* x, const double* z, double* x_full, const int* p2v, void* stream);
/* Segmented batch: one CG per sample (sample s owns rows [s ns, (s+1) ns)),
 * count states, per-sample partials at HDK_SEG_PSTRIDE and tickets; *any is
 * the OR of the samples' conditions (solve run flag, WHILE condition). */
HDK_API int hdk_spcg_init(hdk_pcg* st, int count, double tol, int k_max, int* any, void* stream);
HDK_API int hdk_spcg_spmv(const hdk_csr* a, int ns, const double* p, double* y, const hdk_pcg* st, void* stream);
HDK_API int hdk_spcg_apply(const hdk_vtx* x, const hdk_csr* a, int ns, int count, const double* ef_sorted,
                           const double* p, double* q, double* partial, unsigned int* tickets, hdk_pcg* st,
                           void* stream);
HDK_API int hdk_spcg_xr(int n3s, int n3, double* x, double* r, const double* p, const double* q, const hdk_pcg* st,
                        void* stream);
HDK_API int hdk_spcg_rz(int n3s, int count, const double* r, const double* z, const double* x, double* partial,
                        unsigned int* tickets, hdk_pcg* st, void* stream);
HDK_API int hdk_spcg_p(int n3s, int n3, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                       int count, int* any, unsigned long long cond_handle, void* stream);
/* Contact-adjoint columns: one CG per column, all columns per launch (column
 * c's vectors at base + c 3n, by vertex at + c 3nv, sorted element forces at
 * + c ef_stride); z = A^{-1} r folded from hdk_apply_inverse3_multi's tile
 * partials. */
HDK_API int hdk_cpcg_spmv(const hdk_csr* a, int columns, const double* p, double* y, const hdk_pcg* st,
                          void* stream);
/* Block CG over a batch of m <= 8 contact-adjoint columns (pcg.cu): one
 * block Krylov space for the batch's right-hand sides (O'Leary's block PCG:
 * alpha = (P^T Q)^{-1} (Z^T R), beta = (Z^T R)_old^{-1} (Z^T R)), the
 * columns' vectors as for hdk_cpcg_*.  err = -1: a Gram matrix lost
 * definiteness (the caller solves the batch column by column). */
typedef struct hdk_defl hdk_defl; /* below */
typedef struct hdk_bcg {
  double rz[64], rz_old[64], g[64], alpha[64], beta[64];
  double tol;
  int m, iter, k_max, err, cond, done;
} hdk_bcg;
HDK_API size_t hdk_bcg_partial_doubles(int n);
HDK_API int hdk_bcg_init(hdk_bcg* st, const int* m, double tol, int k_max, int* any, hdk_pcg* cst, int cst_count,
                         void* stream);
HDK_API int hdk_bcg_gram_pq(int n3, const double* p, const double* q, double* partial, unsigned int* ticket,
                            hdk_bcg* st, void* stream);
HDK_API int hdk_bcg_xr(int n3, double* x, double* r, const double* p, const double* q, const hdk_bcg* st,
                       void* stream);
HDK_API int hdk_bcg_zfold(const hdk_factor* f, const double* r, double* z, const double* x, double* partial,
                          unsigned int* ticket, hdk_bcg* st, void* stream);
HDK_API int hdk_bcg_p(int n, int nv, const double* z, double* p, double* pv, const int* p2v, hdk_bcg* st, int* any,
                      const hdk_defl* d, const double* w, unsigned long long cond_handle, void* stream);

/* Deflated CG for the single backbone (pcg.cu, Saad et al.'s deflated PCG):
 * k <= HDK_DEFL_MAX approximate slow eigenvectors W of A^{-1}(A - B) (Ritz vectors of an
 * earlier backbone CG, recycled across time steps) are projected out: the
 * first iterate is Galerkin-corrected on span W and every search direction
 * is made (A - B)-orthogonal to W.  Same system, same stopping test; only the
 * iteration count changes.  W and AW = (A - B) W are [MAX][3n] in elimination
 * order; hist records (alpha, beta, r.z) and the z's of a recording solve. */
#define HDK_DEFL_MAX 8
struct hdk_defl {
  double l[HDK_DEFL_MAX * HDK_DEFL_MAX]; /* Cholesky factor of E = W^T (A - B) W, [r * MAX + c] */
  double mu[HDK_DEFL_MAX], c[HDK_DEFL_MAX]; /* per-iteration projection / first-iterate coefficients */
  double cm[HDK_DEFL_MAX * 8];           /* block CG columns: E^{-1} W^T V per column, [i * 8 + c] */
  double einv[HDK_DEFL_MAX * HDK_DEFL_MAX]; /* E^{-1} (the per-iteration projection is a mat-vec) */
  int k, use, active, rec, hcap, cols;   /* cols: deflate the contact columns' block CG too */
};
/* Lockstep batch (segmented engine): the same deflation per sample.  W and
 * AW are [MAX][n3] over the concatenated index space (sample s's vectors in
 * its own range, the block-diagonal operator keeps them apart); per-sample
 * E factors, coefficients and flags in hdk_sdefl; the global flags (k, use,
 * rec, hcap) in the engine's hdk_defl. */
typedef struct hdk_sdefl {
  double l[HDK_DEFL_MAX * HDK_DEFL_MAX];
  double mu[HDK_DEFL_MAX], c[HDK_DEFL_MAX];
  int active, pad;
} hdk_sdefl;
HDK_API int hdk_sdefl_gram(int n3s, int count, const double* w, const double* aw, const hdk_defl* d,
                           hdk_sdefl* ds, double* e, void* stream);
HDK_API int hdk_sdefl_galerkin(int n3s, int count, double* x, double* r, const double* w, const double* aw,
                               const hdk_defl* d, hdk_sdefl* ds, double* partial, unsigned int* tickets, void* stream);
HDK_API int hdk_sdpcg_rz(int n3s, int count, const double* r, const double* z, const double* x, const double* aw,
                         double* partial, unsigned int* tickets, hdk_pcg* st, const hdk_defl* d, hdk_sdefl* ds,
                         double* zhist, double* hist, void* stream);
HDK_API int hdk_sdpcg_p(int n3s, int n3, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                        int count, int* any, const hdk_defl* d, const hdk_sdefl* ds, const double* w,
                        unsigned long long cond_handle, void* stream);
HDK_API int hdk_sritz_combine(int n3s, int n3, const double* zhist, const double* coef, int jmax, int k, double* w,
                              void* stream);

/* Block CG columns deflated by the frame's W: cm = E^{-1} Wsrc^T V for the
 * batch's m columns (Wsrc = W for the first iterate's Galerkin correction,
 * AW for the projection of Z); then X += W cm, R -= AW cm. */
HDK_API size_t hdk_bdefl_partial_doubles(int n);
HDK_API int hdk_bdefl_dots(int n3, const double* v, const double* wsrc, hdk_defl* d, const hdk_bcg* st,
                           double* partial, unsigned int* tickets, void* stream);
HDK_API int hdk_bdefl_correct(int n3, double* x, double* r, const double* w, const double* aw, const hdk_defl* d,
                              const hdk_bcg* st, void* stream);
HDK_API size_t hdk_defl_partial_doubles(int n);
HDK_API int hdk_defl_gram(int n3, const double* w, const double* aw, double* partial, unsigned int* ticket,
                          hdk_defl* d, void* stream);
HDK_API int hdk_defl_galerkin(int n3, double* x, double* r, const double* w, const double* aw, double* partial,
                              unsigned int* ticket, hdk_defl* d, void* stream);
HDK_API int hdk_dpcg_rz(const hdk_factor* f, const double* r, double* z, const double* x, const double* aw,
                        double* partial, unsigned int* ticket, hdk_pcg* st, hdk_defl* d, double* zhist,
                        double* hist, void* stream);
HDK_API int hdk_dpcg_p(int n, const double* z, double* p, double* pv, const int* p2v, const hdk_pcg* st,
                       const hdk_defl* d, const double* w, unsigned long long cond_handle, void* stream);
HDK_API int hdk_ritz_combine(int n3, const double* zhist, const double* coef, int j, int k, double* w, void* stream);
HDK_API int hdk_scatter_cols(int n, int nv, int k, const double* w, double* wv, const int* p2v, const hdk_defl* d,
                             void* stream);

/* Per-column partials of hdk_cpcg_apply / hdk_cpcg_rz: column c's at
 * partial + c pstride, pstride = hdk_cpcg_partial_stride(n) doubles. */
HDK_API size_t hdk_cpcg_partial_stride(int n);
/* Profiling: per-chunk ring timestamps of the multi-column passes (4 int64 per
 * chunk, solve.cu g_chunk_trace); NULL turns the trace off. */
HDK_API int hdk_set_chunk_trace(long long* const* trace, void* stream);
/* Profiling: (alpha, beta) of each column's CG, [column][512][2] doubles. */
HDK_API int hdk_set_cpcg_trace(double* const* trace, void* stream);
HDK_API int hdk_cpcg_apply(const hdk_vtx* x, const hdk_csr* a, int columns, const double* ef_sorted,
                           size_t ef_stride, const double* p, double* q, double* partial, size_t pstride,
                           unsigned int* tickets, hdk_pcg* st, void* stream);
/* q only (no p.q / alpha): the block CG's Gram matrices are formed separately. */
HDK_API int hdk_cpcg_apply_q(const hdk_vtx* x, const hdk_csr* a, int columns, const double* ef_sorted,
                             size_t ef_stride, const double* p, double* q, hdk_pcg* st, void* stream);
HDK_API int hdk_cpcg_rz(const hdk_factor* f, int columns, const double* r, double* z, const double* x,
                        double* partial, size_t pstride, unsigned int* tickets, hdk_pcg* st, void* stream);
HDK_API int hdk_cpcg_p(int n, int nv, int columns, const double* z, double* p, double* pv, const int* p2v,
                       const hdk_pcg* st, int* any, unsigned long long cond_handle, void* stream);
HDK_API int hdk_cpcg_final(int n, int nv, int columns, const double* x, const double* z, double* xv, const int* p2v,
                           void* stream);
HDK_API int hdk_bapply_cols_sorted(const hdk_mesh* m, const double* dcomp, const double* x, size_t x_stride,
                                   double* ef, size_t ef_stride, const int* corner_pos, const int* cond0,
                                   int cond_stride, int columns, void* stream);

/* ---- segmented batch (lockstep C5 engine, engine.cpp segments > 1) --------
 * S samples of one mesh as one concatenated problem: sample s owns vertices
 * [s nv, (s+1) nv), elements [s ne, (s+1) ne) and elimination positions
 * [s n, (s+1) n) (the factor is block diagonal).  Element- and vertex-
 * parallel kernels run on the concatenation unchanged; these launchers are
 * the per-sample reductions and loop control: grid (HDK_SEG_RB, S), sample in
 * blockIdx.y, one hdk_ctl per sample, partials at partial + s HDK_SEG_PSTRIDE
 * (folded over HDK_SEG_RB blocks; the 18-quantity Anderson partials are
 * quantity-major over HDK_RED_BLOCKS and their unused slots must be zero).
 * A sample whose loop has ended (ctl[s].cond == 0) is skipped, so each
 * sample stops at its own iteration count; `any` (device int) is the OR over
 * the samples, which drives the WHILE node and the solve passes' run flag. */
#define HDK_SEG_RB 16
#define HDK_SEG_PSTRIDE (HDK_RED_BLOCKS * HDK_RED_Q)
typedef struct hdk_segs {
  int count;   /* samples */
  int nv, n, ne;  /* per sample: vertices, free vertices, elements */
} hdk_segs;
HDK_API int hdk_seg_ctl_init(hdk_ctl* ctl, const hdk_segs* g, const int* windows, double guard, int k_max,
                             double eps_rel, double eps_abs, double tol, double eps_tr, int* any, void* stream);
HDK_API int hdk_seg_aa_reset(hdk_ctl* ctl, const hdk_segs* g, int window, double guard, int k_max, double tol,
                             int* any, void* stream);
HDK_API int hdk_seg_gather_rhs(const hdk_vtx* x, const hdk_segs* g, const hdk_ctl* ctl, const double* ef,
                               double inv_h2, const double* q_tilde, const double* damp, double* b_prev,
                               double* rhs_perm, double* partial, void* stream);
HDK_API int hdk_seg_gather_rhs_sorted(const hdk_vtx* x, const hdk_segs* g, const hdk_ctl* ctl, const double* efs,
                                      double inv_h2, const double* q_tilde, const double* damp, double* b_prev,
                                      double* rhs_perm, double* partial, void* stream);
HDK_API int hdk_seg_aa_dots_fused(const hdk_vtx* x, const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl,
                                  double* qhat, const double* qcur, double* last_q, double* last_g, double* dq,
                                  double* dg, double* partial18, unsigned int* tickets, void* stream);
HDK_API int hdk_seg_aa_mix(const hdk_vtx* x, const hdk_segs* g, hdk_ctl* ctl, const double* qhat, double* qcur,
                           double* qprev, const double* dq, const double* dg, double* partial, void* stream);
HDK_API int hdk_seg_gate(hdk_ctl* ctl, const hdk_segs* g, const double* partial_b, const double* partial_q, int* any,
                         unsigned int* ticket, unsigned long long cond_handle, void* stream);
HDK_API int hdk_seg_commit(const hdk_segs* g, const hdk_ctl* ctl, const double* q_star, double h, double* q, double* v,
                           void* stream);
HDK_API int hdk_seg_tr_model(const hdk_vtx* x, const hdk_segs* g, const hdk_csr* a_ff, const double* q_star,
                             const double* q_prev, double* dq_perm, double* partial, void* stream);
HDK_API int hdk_seg_tr_select(const hdk_vtx* x, const hdk_segs* g, const double* e_prev, const double* e_star,
                              const double* q_prev, const double* q_star, const double* q_tilde, double inv_h2,
                              const double* model_partial, double* partial, hdk_ctl* ctl, void* stream);
HDK_API int hdk_seg_bb_dots(const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl, hdk_ctl* snap, double* t_perm,
                            double* t_full, const double* x_perm, double* last_q, double* last_g, double* dq,
                            double* dg, double* partial18, void* stream);
HDK_API int hdk_seg_bb_solve(hdk_ctl* ctl, const hdk_segs* g, const hdk_ctl* snap, const double* partial18,
                             void* results, void* stream);
HDK_API int hdk_seg_bb_mix(const hdk_factor* f, const hdk_segs* g, hdk_ctl* ctl, const hdk_ctl* snap,
                           const void* results, const double* t_perm, double* x_perm, double* x_full,
                           const double* sum_hist, const double* rt_perm, double* rx_perm, double* last_rx,
                           double* last_rg, double* rsum_hist, const double* seed_perm, double* rhs_perm,
                           void* stream);
/* any = OR over the samples of "still iterating" (cond, no error, finite);
 * sets the WHILE condition when cond_handle != 0. */
HDK_API int hdk_seg_any(const hdk_ctl* ctl, const hdk_segs* g, int* any, unsigned long long cond_handle, void* stream);
/* out[s] = 1/2 |q_s - ref_s|^2 per sample (3 nv doubles each). */
HDK_API int hdk_seg_half_sqdist(const hdk_segs* g, const double* q, const double* ref, double* out, void* stream);
/* out[0] = sum_s loss[s]; out[1 + i] = sum_s vec[s ne + i], in sample order. */
HDK_API int hdk_seg_sum(const hdk_segs* g, const double* vec, const double* loss, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HDK_H */
