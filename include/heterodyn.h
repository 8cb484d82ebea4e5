/* heterodyn — differentiable projective-dynamics solver, C interface.
 *
 * Drop-in boundary of the B200 build.  The first half of this header is the
 * reference ABI, symbol for symbol (reference: /root/reference/proj/include/
 * heterodyn/heterodyn.h:30-141, implemented by src/capi.cpp:94-322); the
 * second half ("B200 extensions") adds the backward/trajectory surface the
 * reference reaches only through its drivers (drivers.cpp:31-99,
 * backward.hpp:94-97), which the reference ABI does not expose.
 *
 * Semantics kept from the reference: every fallible call returns an
 * hd_status (0 on success) or NULL; the message for the most recent failure
 * on the calling thread is available via hd_last_error() (never NULL);
 * strings returned through char** are malloc'd and released with
 * hd_string_free(); hd_scene is immutable and shareable; hd_sim is
 * single-threaded and borrows its scene; exceptions never cross the boundary.
 *
 * Two libraries export this header: the product
 * (paper_2605_14526_b200/_lib/libheterodyn_b200.so, device-resident solver on
 * sm_100a) and the CPU oracle used by the tests
 * (oracle/_build/libheterodyn_oracle.so).
 */
#ifndef HETERODYN_H
#define HETERODYN_H

#include <stddef.h>

#if defined(_WIN32)
#if defined(HETERODYN_BUILD)
#define HD_API __declspec(dllexport)
#else
#define HD_API __declspec(dllimport)
#endif
#else
#define HD_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* reference heterodyn.h:30-45 */
typedef enum hd_status {
  HD_OK = 0,
  HD_ERR_PARSE = 1,
  HD_ERR_VALIDATION = 2,
  HD_ERR_DEGENERATE_ELEMENT = 3,
  HD_ERR_INVALID_POISSON = 4,
  HD_ERR_NON_POSITIVE_JACOBIAN = 5,
  HD_ERR_PROX_DIVERGED = 6,
  HD_ERR_SINGULAR_FILTERED_HESSIAN = 7,
  HD_ERR_NOT_POSITIVE_DEFINITE = 8,
  HD_ERR_SINGULAR_CONTACT_SYSTEM = 9,
  HD_ERR_ADJOINT_DIVERGED = 10,
  HD_ERR_LINE_SEARCH_FAILED = 11,
  HD_ERR_IO = 12,
  HD_ERR_INVALID_ARGUMENT = 13
} hd_status;

/* reference heterodyn.h:47-54 */
HD_API const char* hd_last_error(void);
HD_API int hd_last_error_code(void);
HD_API void hd_string_free(char* s);

/* ---- scenes (reference heterodyn.h:56-76) ------------------------------ */
typedef struct hd_scene hd_scene;
HD_API hd_scene* hd_scene_load(const char* path);
HD_API hd_scene* hd_scene_parse(const char* json_text);
HD_API hd_scene* hd_scene_builtin(const char* name);
HD_API void hd_scene_free(hd_scene* scene);
HD_API int hd_scene_vertex_count(const hd_scene* scene);
HD_API int hd_scene_element_count(const hd_scene* scene);
HD_API int hd_scene_frame_count(const hd_scene* scene);
HD_API const char* hd_scene_name(const hd_scene* scene);

/* ---- frame-by-frame simulation (reference heterodyn.h:78-107) ---------- */
typedef struct hd_sim hd_sim;
HD_API hd_sim* hd_sim_create(const hd_scene* scene);
HD_API void hd_sim_free(hd_sim* sim);
HD_API hd_status hd_sim_step(hd_sim* sim);
HD_API double hd_sim_time(const hd_sim* sim);
HD_API int hd_sim_dof_count(const hd_sim* sim);
HD_API hd_status hd_sim_positions(const hd_sim* sim, double* out, size_t capacity);
HD_API hd_status hd_sim_velocities(const hd_sim* sim, double* out, size_t capacity);
HD_API int hd_sim_last_iterations(const hd_sim* sim);
HD_API int hd_sim_last_converged(const hd_sim* sim);
HD_API int hd_sim_last_contact_count(const hd_sim* sim);

/* ---- drivers (reference heterodyn.h:109-141) --------------------------- */
HD_API hd_status hd_run_simulate(const hd_scene* scene, const char* out_dir, char** summary_json);
HD_API hd_status hd_run_gradcheck(const hd_scene* scene, const char* vars_csv, const char* out_path,
                                  char** report_json, int* pass);
HD_API hd_status hd_run_identify(const char* problem_json, const char* out_dir, char** result_json,
                                 int* stalled);
HD_API hd_status hd_run_identify_file(const char* problem_path, const char* out_dir, char** result_json,
                                      int* stalled);
HD_API hd_status hd_factor_stats(const hd_scene* scene, char** stats_json);

/* ---- B200 extensions (new; no reference counterpart in the ABI) ---------- */

/* Scene data the system-identification driver needs (drivers.cpp:710-803):
 * element regions (scene.hpp region_of_element / region_count), rest
 * positions (3 doubles per vertex) and lumped vertex masses (one per vertex,
 * TetMesh::vertex_mass).  Capacities are checked. */
HD_API int hd_scene_region_count(const hd_scene* scene);
HD_API hd_status hd_scene_regions(const hd_scene* scene, int* region_of_element, size_t capacity);
HD_API hd_status hd_scene_rest_positions(const hd_scene* scene, double* out, size_t capacity);
HD_API hd_status hd_scene_vertex_masses(const hd_scene* scene, double* out, size_t capacity);
/* Element connectivity (4 vertex indices per element). */
HD_API hd_status hd_scene_elements(const hd_scene* scene, int* out, size_t capacity);
/* Per-element Young's moduli of the scene's material (MaterialField::young). */
HD_API hd_status hd_scene_young_moduli(const hd_scene* scene, double* out, size_t capacity);

/* The external force f_ext the sim steps with (dof doubles; initially the
 * scene's gravity + point forces, scene_external_force scene.cpp:530-540):
 * read it, or replace it for subsequent steps (the gradcheck driver's f_ext
 * perturbations, drivers.cpp:471-483). */
HD_API hd_status hd_sim_external_force(const hd_sim* sim, double* out, size_t capacity);
HD_API hd_status hd_sim_set_external_force(hd_sim* sim, const double* f_ext, size_t count);
/* Frame diagnostics of the simulate driver: the largest |Fischer-Burmeister
 * residual| over the normal contacts of the last step (max_normal_fb_residual,
 * drivers.cpp:147-159) and the current state's deepest obstacle penetration
 * (max_penetration_at, drivers.cpp:101-111). */
HD_API double hd_sim_last_fb_residual(const hd_sim* sim);
/* Contact trace of the last step (B200 extension; parity observability for
 * the contact path): the contacts' (vertex, obstacle) pairs in row order
 * (detect_contacts' vertex-major / obstacle-minor scan, contact.cpp:117-144)
 * and, per forward iteration, the decision values of project_multipliers
 * (contact.cpp:218-235): clamp[it * nc + i] = normal multiplier i before the
 * clamp (clamped at zero iff < 0); cone[it * nf + f] = (|lambda_t| -
 * mu lambda_n) / (mu lambda_n) of frictional contact f before the projection
 * (projected onto the Coulomb cone iff > 0; -1 when mu lambda_n = 0, where the
 * pair is zeroed whatever its value).  counts[3] (may be NULL) receives
 * {nc, nf, iterations}; any buffer may be NULL; capacities (in doubles) are
 * checked (HD_ERR_INVALID_ARGUMENT). */
HD_API hd_status hd_sim_contact_trace(const hd_sim* sim, int* vertex, int* obstacle, size_t row_capacity,
                                      double* clamp, size_t clamp_capacity, double* cone, size_t cone_capacity,
                                      int* counts);
HD_API double hd_sim_penetration(const hd_sim* sim);

/* Records every subsequent frame's adjoint cache (the reference's
 * roll(keep_caches=true), drivers.cpp:31-54).  enable=0 stops recording and
 * discards recorded frames. */
HD_API hd_status hd_sim_record(hd_sim* sim, int enable);
HD_API int hd_sim_recorded_frames(const hd_sim* sim);

/* Replaces the state (3 doubles per vertex each, xyz interleaved) and time;
 * discards recorded frames.  q or v may be NULL to keep that part. */
HD_API hd_status hd_sim_set_state(hd_sim* sim, const double* q, const double* v, double time);

/* Reverse-time adjoint chain over the recorded frames (chain_backward,
 * drivers.cpp:66-99, with backward_step backward.cpp:396-414 per frame).
 * dl_dq_direct: (frames + 1) x dof doubles — the loss's direct partial with
 * respect to the state after frame t (row 0 = initial state) — or NULL, in
 * which case dl_dq_final (dof doubles, may be NULL = zero) seeds the final
 * frame only.  dl_dv_final (dof, may be NULL = zero) seeds the final velocity.
 * Outputs may be NULL: dl_dq0, dl_dv0, dl_df_ext (dof each), dl_de
 * (element_count), dl_dw (element_count, or 2 x element_count for corotated;
 * dl_dw_capacity is checked). */
HD_API hd_status hd_sim_backward(hd_sim* sim, const double* dl_dq_direct, const double* dl_dq_final,
                                 const double* dl_dv_final, double* dl_dq0, double* dl_dv0,
                                 double* dl_df_ext, double* dl_de, double* dl_dw,
                                 size_t dl_dw_capacity);
/* Diagnostics of the most recent hd_sim_backward: per recorded frame tau and
 * trust-region ratio rho (forward frame order), and total adjoint sweeps. */
HD_API hd_status hd_sim_backward_tau(const hd_sim* sim, double* tau, double* rho, size_t capacity);
HD_API int hd_sim_backward_iterations(const hd_sim* sim);

/* One application of the global solve on the current factor:
 * out = solve_free(rhs_full, fixed_q) (factor.cpp:196-208).  fixed_q may be
 * NULL (zero prescribed positions).  All arrays are dof doubles. */
HD_API hd_status hd_sim_solve_free(hd_sim* sim, const double* rhs_full, const double* fixed_q,
                                   double* out);

/* Replaces the per-element Young's moduli (MaterialField::set_young,
 * material.cpp:75-80); the next step refactorizes.  The prox means are frozen
 * at their current values when freeze_means is nonzero (freeze_means,
 * material.cpp:82-86, the gradcheck/identify convention). */
HD_API hd_status hd_sim_set_young(hd_sim* sim, const double* young, size_t count, int freeze_means);
/* B200 extension: recycled-subspace deflation of the adjoint backbone CG
 * (on by default; HETERODYN_DEFLATION=0 at creation turns it off).  The
 * backbone solves reuse Ritz vectors of an earlier solve, so a repeated
 * backward of the same frame agrees with the first to the CG stopping
 * tolerance rather than bitwise; off, every solve is a pure function of its
 * inputs.  Toggling drops the recycled subspace.  (The reference CPU library
 * accepts and ignores it.) */
HD_API hd_status hd_sim_set_deflation(hd_sim* sim, int on);

/* Counters for roofline accounting (factor.hpp:39,119-121; forward.hpp:100;
 * backward.hpp:26): factor nnz, free vertex count, cumulative 3-axis solves,
 * cumulative A-SpMVs, refactorizations. */
HD_API long long hd_sim_factor_nnz(const hd_sim* sim);
HD_API int hd_sim_free_count(const hd_sim* sim);
HD_API long long hd_sim_solve_count(const hd_sim* sim);
/* Passes over the factor that carried those solves: a multi-column solve of
 * several contact-adjoint columns streams the factor once (B200 extension;
 * equals hd_sim_solve_count where every solve is single). */
HD_API long long hd_sim_factor_streams(const hd_sim* sim);
HD_API long long hd_sim_a_spmv_count(const hd_sim* sim);
HD_API long long hd_sim_refactor_count(const hd_sim* sim);

/* Device-resident variant of hd_sim_backward for throughput measurement:
 * seeds the canonical loss L = 1/2 |q_T - rest|^2 + 1/2 |v_T|^2 of the
 * gradient check (drivers.cpp:384-389, 394-396) from the state in device
 * memory and keeps every gradient in device memory (outputs may be NULL).
 * Same adjoint chain as hd_sim_backward. */
HD_API hd_status hd_sim_backward_canonical(hd_sim* sim, double* dl_dq0, double* dl_dv0, double* dl_df_ext,
                                           double* dl_de, double* dl_dw, size_t dl_dw_capacity);

/* The CUDA stream every device operation of this sim is ordered on (as
 * cudaStream_t, NULL for the CPU oracle) and the number of device kernels the
 * sim has launched so far (graph kernel nodes counted per execution). */
HD_API void* hd_sim_stream(const hd_sim* sim);
HD_API long long hd_sim_kernel_launches(const hd_sim* sim);

/* Times `reps` back-to-back applications of the global solve (3 axes) on the
 * sim's stream with CUDA events, inputs resident in HBM; *ms_per_solve
 * receives the mean duration.  Also reports the algorithmic bytes one solve
 * moves (factor values read by both passes plus right-hand sides). */
HD_API hd_status hd_sim_time_solve(hd_sim* sim, int reps, double* ms_per_solve, double* bytes_per_solve);
/* Profiling: times `reps` launches of the adjoint backbone iteration (one
 * body of the backward WHILE loop, run on whatever the buffers hold after a
 * backward step) with CUDA events.  skip_mask drops kernels for ablation:
 * bit 0 B x, bit 1 rhs gather, bit 2 solve passes, bit 3 fused AA dots/solve,
 * bit 4 AA mix.  Results of an ablated body are meaningless; only its time is. */
HD_API hd_status hd_sim_time_backbone(hd_sim* sim, int reps, unsigned skip_mask, double* ms_per_iteration);
/* Profiling: timeline of `reps` (<= 16) consecutive backbone iterations in
 * one graph launch sequence; out receives reps x 14 records (B x, gather, row
 * dots, z-fold, column pass, AA dots, AA mix: {first CTA resident, first CTA
 * past its dependency wait, last CTA end}; then seven point stamps in the
 * third field: AA solve entry / folded / solved, AA dots loop done / partials
 * written, AA bookkeeping done / factorization done) in ns from the earliest
 * stamp. */
HD_API hd_status hd_sim_trace_backbone(hd_sim* sim, int reps, double* out, size_t capacity);
/* Profiling: the same records for the real backbone loop of one forward +
 * backward step from the current state (state restored afterwards): the
 * last min(iterations, 16) iterations, oldest first; *iterations receives
 * how many records were written. */
HD_API hd_status hd_sim_trace_loop(hd_sim* sim, double* out, size_t capacity, int* iterations);

/* ---- batched system-ID (config C5; new) --------------------------------
 * One process's share of a batch of material-parameter samples.  Sample s
 * simulates the scene with per-element Young's moduli young[s * ne .. +ne)
 * (NULL = the scene's own for every sample) from the scene's initial state.
 * One evaluation runs, for every sample, `frames` forward steps and the
 * adjoint chain of L_s = 1/2 |q_T - q_target|^2 (roll + chain_backward,
 * drivers.cpp:31-99, the objective of run_identify, drivers.cpp:848-851)
 * and returns the per-sample losses and the sample-ordered sums
 * sum_s L_s, sum_s dL_s/dE (element_count doubles).  The default target is
 * the scene's initial positions.  threads = host threads driving samples
 * concurrently (the product overlaps them on the device; the oracle runs
 * them in order).  device_out, if not NULL, is a device pointer receiving
 * [sum L, sum dL/dE] (1 + element_count doubles) — the buffer a caller hands
 * to an NCCL all-reduce; it is complete when the call returns. */
typedef struct hd_batch hd_batch;
HD_API hd_batch* hd_batch_create(const hd_scene* scene, int samples, const double* young, size_t young_count,
                                 int threads);
HD_API void hd_batch_free(hd_batch* batch);
HD_API int hd_batch_sample_count(const hd_batch* batch);
HD_API hd_status hd_batch_set_target(hd_batch* batch, const double* q_target, size_t count);
/* New per-sample Young's moduli (samples x element_count values, the layout of
 * hd_batch_create): every sample refactors (MaterialField::set_young +
 * refresh, material.cpp:75-86), in parallel over the batch's host threads —
 * one system-ID parameter update. */
HD_API hd_status hd_batch_set_young(hd_batch* batch, const double* young, size_t count, int freeze_means);
HD_API hd_status hd_batch_evaluate(hd_batch* batch, int frames, double* loss, size_t loss_capacity,
                                   double* dl_de_sum, size_t dl_de_capacity, void* device_out);
/* Device time of the last evaluation in milliseconds (CUDA events spanning
 * every sample's stream; 0 for the oracle) and kernels launched so far. */
HD_API double hd_batch_last_ms(const hd_batch* batch);
HD_API long long hd_batch_kernel_launches(const hd_batch* batch);
/* Global solves (3 axes) run by all samples so far, and the algorithmic bytes
 * of one solve of one sample (16 nnz(S') + 96 n; samples share the pattern). */
HD_API long long hd_batch_solve_count(const hd_batch* batch);
/* ms per solve of the batch's solve path (the lockstep engine's block-diagonal
 * factor: all samples in one launch per pass) and its algorithmic bytes. */
HD_API hd_status hd_batch_time_solve(hd_batch* batch, int reps, double* ms_per_solve, double* bytes_per_solve);
/* 1 when the batch runs as one lockstep segmented engine, 0 for per-sample engines. */
HD_API int hd_batch_lockstep(const hd_batch* batch);
HD_API double hd_batch_solve_bytes(const hd_batch* batch);

#ifdef __cplusplus
}
#endif

#endif /* HETERODYN_H */
