/*
 * pe.h — C ABI of libpe, the B200 (sm_100a) parareal hot path.
 *
 * Drop-in boundary for the reference's online solver (paradiff, arXiv 2411.09244):
 * every entry point replaces one piece of the reference's Python hot path, cited as
 * /root/reference/pkg/src/paradiff/<file>:<line>.  Plain pointers and sizes only; no
 * torch or C++ types cross this boundary.  All functions return 0 on success and a
 * negative PE_ERR_* code on failure; pe_last_error() returns the message of the last
 * failure on the calling thread.  No C++ exception crosses the ABI.
 *
 * Layouts (FP64, little endian):
 *   - operator blocks passed to pe_set_system are HOST, row-major (C order), exactly
 *     the ndarrays of a reference CoarseSystem (msbasis.py:397-418);
 *   - state batches are DEVICE buffers of shape (E, ncols, d1+d2), C order: member-
 *     major, then interval/column, then the stacked [u; w] coefficients of one
 *     SplitState (stepping.py:49-50 `stacked()`).
 *   - `stream` is a cudaStream_t (CUstream) or NULL for the legacy default stream.
 * A context is not thread-safe; callers serialise calls per context.
 */
#ifndef PE_H
#define PE_H

#ifdef __cplusplus
extern "C" {
#endif

#define PE_OK 0
#define PE_ERR_ARG -1      /* bad argument (reference raises ValueError) */
#define PE_ERR_CUDA -2     /* CUDA runtime / launch failure */
#define PE_ERR_SOLVER -3   /* singular factorisation (reference: LinAlgError) */
#define PE_ERR_STATE -4    /* call order violated (e.g. fine before prepare) */
#define PE_ERR_NOMEM -5

/* WR stop reasons, allatonce.py:243-271 */
#define PE_STOP_TOL 0
#define PE_STOP_DIVERGED 1
#define PE_STOP_FLOOR 2
#define PE_STOP_MAX_ITER 3

/* parareal stop rules */
#define PE_RULE_ABSOLUTE 0 /* parareal.py:145-147 check_stop: max_n ||dx_n|| < eps */
#define PE_RULE_RELATIVE 1 /* max_n ||dx_n|| / max_n ||x_n^k|| < eps  */

#define PE_KIND_SEQUENTIAL 0 /* SequentialFine, parareal.py:53-66 */
#define PE_KIND_ALLATONCE 1  /* AllAtOnceFine,  parareal.py:69-84 */

typedef struct pe_ctx pe_ctx;

const char* pe_last_error(void);
const char* pe_version(void);

/* Context for E members of reduced size d1+d2 with at most `max_cols` columns (N
 * coarse intervals) and J fine substeps.  Replaces SplitPropagators.__init__
 * (stepping.py:109-114). */
int pe_create(pe_ctx** ctx, int E, int d1, int d2, int max_cols, int J, int device);
int pe_destroy(pe_ctx* ctx);

/* Upload one member's CoarseSystem blocks (host, row-major) and ConstantLoads
 * (stepping.py:77-91).  M11,A11: d1*d1; M12,A12: d1*d2; M22,A22: d2*d2; f1: d1; f2: d2. */
int pe_set_system(pe_ctx* ctx, int member, const double* M11, const double* A11,
                  const double* M12, const double* A12, const double* M22,
                  const double* A22, const double* f1, const double* f2);

/* Pre-factorise for the sequential fine propagator at substep dt_sub
 * (stepping.py:116-120 _u_factor, :114 M22 Cholesky). */
int pe_prepare_sequential(pe_ctx* ctx, double dt_sub);
/* Pre-factorise the coarse propagator G at step dt (stepping.py:149-159 _g_factor). */
int pe_prepare_coarse(pe_ctx* ctx, double dt);
/* Set up the all-at-once solver (allatonce.py:100-110 ImplicitAllAtOnce.__init__,
 * :184-210 WaveformRelaxation.__init__).  alpha in (0,1). */
int pe_prepare_allatonce(pe_ctx* ctx, double dt_sub, double alpha, double tol, int max_iter);

/* Fine propagator over one coarse interval for `ncols` states per member, lags reset
 * (stepping.py:178-189 fine_interval; parareal.py:62-66 SequentialFine.propagate).
 * X_in, X_out: device (E, ncols, d). */
int pe_fine_sequential(pe_ctx* ctx, const double* X_in, double* X_out, int ncols, void* stream);

/* One fine substep with explicit lags at the prepared dt_sub (stepping.py:122-147
 * split_step): X_prev holds the lagged (u_prev, w_prev).  (E, ncols, d) device. */
int pe_split_step(pe_ctx* ctx, const double* X_in, const double* X_prev, double* X_out,
                  int ncols, void* stream);

/* All-at-once fine propagator (allatonce.py:232-298 WaveformRelaxation.solve) for
 * `ncols` states per member.  Optional device outputs (may be NULL): sweeps and
 * stop reason per (member, column) as int32 (E, ncols); residual history
 * (E, ncols, max_iter) FP64 (unused entries NaN). */
int pe_fine_allatonce(pe_ctx* ctx, const double* X_in, double* X_out, int ncols,
                      int* sweeps, int* reasons, double* resid_hist, void* stream);

/* Waveforms of the last pe_fine_allatonce call (allatonce.py:280-291 trajectory):
 * U_out (E, ncols, J+1, d1), W_out (E, ncols, J+1, d2), row 0 = interval start. */
int pe_wr_waveforms(pe_ctx* ctx, double* U_out, double* W_out, int ncols, void* stream);

/* Coarse propagator G applied to `ncols` states per member
 * (stepping.py:161-176 coarse_step).  Bitwise identical to the G inside
 * pe_coarse_correct. */
int pe_coarse_apply(pe_ctx* ctx, const double* X_in, double* X_out, int ncols, void* stream);

/* Fused coarse sweep + parareal correction + convergence norms for N intervals
 * (parareal.py:198-215 and :140-147; initial sweep :150-157 when F_hat == NULL).
 *   X_old:   (E, N+1, d) iterate k (row 0 = initial state, also used as row 0 of X_new)
 *   F_hat:   (E, N, d)   fine results F(x_n^k), or NULL for the initial sweep
 *   G_cache: (E, N, d)   in: G(x_n^k); out: G(x_n^{k+1})  (parareal.py:179,216)
 *   X_new:   (E, N+1, d) iterate k+1
 *   diff:    (E, 2) device FP64: [max_n ||x_new - x_old||, max_n ||x_new||], n = 1..N
 *   active:  (E) int32 member mask or NULL; inactive members copy X_old to X_new. */
int pe_coarse_correct(pe_ctx* ctx, int N, const double* X_old, const double* F_hat,
                      double* G_cache, double* X_new, double* diff, const int* active,
                      void* stream);

/* One parareal iteration (parareal.py:188-215): the fine sweep on rows 0..N-1 of
 * X_old (E, N+1, d), then the fused coarse sweep / correction / norms into X_new.
 * G_cache as in pe_coarse_correct (initialise it with an initial sweep).  This is the
 * "step" bench.py times. */
int pe_parareal_iterate(pe_ctx* ctx, int kind, int N, const double* X_old, double* X_new,
                        double* G_cache, double* diff, const int* active, int* wr_sweeps,
                        int* wr_reasons, double* wr_resid, void* stream);

/* Device-resident parareal loop (parareal.py:160-236 run_parareal) with one host
 * synchronisation per iteration.  All pointers are device pointers except the
 * `*_h` outputs, which are host arrays.
 *   X0:        (E, d) initial states
 *   history:   ((k_max+1), E, N+1, d) out
 *   diffs_h:   (k_max, E) out, the value the stop rule compared (absolute or relative)
 *   iters_h:   (E) out, iterations per member (includes the stopping sweep)
 *   conv_h:    (E) out, 1 when the member met the rule
 *   wr_sweeps, wr_reasons: (k_max, E, N) int32 device or NULL (all-at-once kind)
 *   wr_resid:  (k_max, E, N, max_iter) FP64 device or NULL
 *   fine_ms_h, coarse_ms_h: (k_max) host, CUDA-event phase times per iteration
 * Returns the number of executed iterations (max over members) in *k_done. */
int pe_parareal_run(pe_ctx* ctx, int kind, int N, const double* X0, int k_max,
                    double epsilon, int rule, double* history, double* diffs_h,
                    int* iters_h, int* conv_h, int* wr_sweeps, int* wr_reasons,
                    double* wr_resid, float* fine_ms_h, float* coarse_ms_h, int* k_done,
                    void* stream);

/* The FP64 DMMA GEMM underneath every contraction, exposed for kernel tests:
 * C[b](i,j) = sum_k A[b](i,k) B[b](k,j), element and batch strides (device pointers). */
int pe_gemm_f64(int M, int N, int K, int batch, const double* A, long long a_i, long long a_k,
                long long a_b, const double* B, long long b_k, long long b_j, long long b_b,
                double* C, long long c_i, long long c_j, long long c_b, void* stream);

/* Launch counter: number of libpe kernels launched since context creation
 * (bench/driver evidence that the native path ran). */
long long pe_launch_count(pe_ctx* ctx);

/* Roofline bookkeeping for bench.py.  With profiling on, every GEMM launch of the
 * fine propagators is bracketed by CUDA events on its stream; pe_last_fine_stats
 * returns, for the most recent fine sweep, the summed GEMM time (ms, 0 when profiling
 * is off), their algorithmic flops and the number of GEMM launches. */
int pe_set_profiling(pe_ctx* ctx, int on);
/* Select the persistent cluster-resident recurrence kernels for the sequential-in-time
 * chains (default on) or one DMMA GEMM launch per step (reference-like structure). */
int pe_set_recurrence(pe_ctx* ctx, int on);
/* Select the modal form of the all-at-once w recursion (default on).  When M22 is SPD
 * and A22 symmetric, pe_prepare_allatonce diagonalises E = I - dt M22^-1 A22 =
 * V diag(lam) V^-1 (M22-orthonormal pencil eigenvectors, accepted only if it reproduces E
 * to 1e-9); each sweep then runs the J-step w chain of WaveformRelaxation._w_sweep
 * (allatonce.py:220-230) as an elementwise scan in z = V^-1 w plus one W = V Z GEMM.
 * When A11 is symmetric and M11 SPD as well, the whole sweep runs in the generalized
 * eigenbases of both pencils (wr_modal.cu): the shifted solves of ImplicitAllAtOnce
 * (allatonce.py:100-133) become one scalar time recurrence per mode.
 * pe_wr_is_modal returns 2 for the full modal sweep, 1 for the modal w recursion only and
 * 0 for the direct path.  Changing the switch invalidates pe_prepare_allatonce. */
int pe_set_modal(pe_ctx* ctx, int on);
int pe_wr_is_modal(pe_ctx* ctx);
int pe_last_fine_stats(pe_ctx* ctx, double* gemm_ms, double* gemm_flops, int* launches);
/* Profiling mode: summed event time (ms) of the last fine sweep's non-DMMA kernels (the
 * modal scans and the stop decision), for the in-situ share breakdown in bench.py. */
int pe_last_fine_other_ms(pe_ctx* ctx, double* other_ms);

/* ---- Fine-scale accuracy path (host buffers in and out) ---------- */

/* Which formulation pe_fine_reference_solve takes for this operator: 0 = one fused dense
 * GEMV (n < 4096), 1 = packed symmetric K^-1 tiles, 2 = block-tridiagonal chain solver
 * (banded operators from 16384 nodes, finechain.cu; PE_FINE_CHAIN=1 / 0 forces / disables
 * it); *block (optional) = the chain solver's block size.  Host CSR index arrays. */
int pe_fine_solver_kind(int n, const int* M_ptr, const int* M_idx, const int* A_ptr,
                        const int* A_idx, int* block);

/* Backward Euler on the fine interior nodes, (M/dt + A) u_{s+1} = M u_s / dt + b with
 * dt = t_end / n_steps (fem.py:292-318 reference_solve).  M, A: host CSR (int32 indptr /
 * indices, FP64 values) of the n x n interior mass and stiffness (FineOperators.M/.A,
 * fem.py:253-270); b: the interior load (FineOperators.load); u0: n values or NULL (zeros).
 * states_h: (n_steps+1, n) when keep_trajectory, else (2, n) = [u0, u_final].
 * step_ms (may be NULL): CUDA-event time of the time-step loop.  M/dt + A must be SPD
 * (PE_ERR_SOLVER otherwise; the reference's splu raises on a singular matrix). */
int pe_fine_reference_solve(int n, const int* M_ptr, const int* M_idx, const double* M_val,
                            const int* A_ptr, const int* A_idx, const double* A_val,
                            const double* b, const double* u0, double t_end, int n_steps,
                            int keep_trajectory, double* states_h, float* step_ms,
                            void* stream);

/* M-norms of ref - [Psi1 Psi2] x_k for K coarse states x_k (K, d) and of ref itself:
 * norms_h[k] = ||ref - reconstruct(x_k)||_M (k < K), norms_h[K] = ||ref||_M
 * (experiment.py:320-325 relative_error, :348-354 error series; msbasis.py:448-450
 * reconstruct; fem.py:272-274 norm).  P: host CSR (n x d) of hstack([Psi1, Psi2]). */
int pe_relative_error_series(int n, int d, const int* P_ptr, const int* P_idx,
                             const double* P_val, const int* M_ptr, const int* M_idx,
                             const double* M_val, const double* ref, int K, const double* X,
                             double* norms_h, void* stream);

/* Galerkin projection (projection part of the offline build):
 * msbasis.py:545-567 project_coarse and :570-572 project_load.  P: host CSR (n x d) of
 * hstack([Psi1, Psi2]), d = d1 + d2; M, A: host CSR (n x n).  Mc_h, Ac_h: host (d, d)
 * row-major = P^T X P with the (1,1) and (2,2) blocks symmetrised ((B + B^T) / 2) and the
 * off-diagonal blocks as computed (B12 = Psi1^T X Psi2).  b (n) / f_h (d) optional: P^T b.
 * asym_h (2) optional: the removed asymmetry max |B - B^T| for M and A. */
int pe_project_coarse(int n, int d1, int d2, const int* P_ptr, const int* P_idx,
                      const double* P_val, const int* M_ptr, const int* M_idx,
                      const double* M_val, const int* A_ptr, const int* A_idx,
                      const double* A_val, const double* b, double* Mc_h, double* Ac_h,
                      double* f_h, double* asym_h, void* stream);

/* Load-only projection f = P^T b (msbasis.py:570-572 project_load), without the operator
 * products.  P: host CSC (n x d) of hstack([Psi1, Psi2]) (column pointers d + 1, row
 * indices, values); b (n) host; f_h (d) host.  One warp per column, fixed order. */
int pe_project_load(int n, int d, const int* P_colptr, const int* P_rowidx, const double* P_val,
                    const double* b, double* f_h, void* stream);

/* ---- reference-API building blocks (api_ops.cu); device pointers unless noted ---- */

/* apply_S (inverse = 0) / apply_S_inverse (inverse = 1) along the time axis
 * (allatonce.py:74-88): x, y (J, ncols) row-major, planar real / imaginary parts (xi, yi
 * may be NULL for a real input / a discarded imaginary output).  Direct DFT. */
int pe_apply_S(int J, long long ncols, double alpha, int inverse, const double* xr,
               const double* xi, double* yr, double* yi, void* stream);

/* build_rhs (allatonce.py:136-158): rhs (J, d1) of the u all-at-once system from f1_rows
 * (J, d1), u_start, u_final_prev (d1), w_start, w_lag (d2), w_rows_prev (J, d2) and the
 * blocks M11 (d1 x d1), M12, A12 (d1 x d2), row-major. */
int pe_build_rhs(int d1, int d2, int J, const double* M11, const double* M12, const double* A12,
                 const double* f1_rows, const double* u_start, const double* w_start,
                 const double* w_lag, const double* w_rows_prev, const double* u_final_prev,
                 double dt, double alpha, double* rhs, void* stream);

/* ImplicitAllAtOnce.solve (allatonce.py:112-133) on the context's all-at-once setup
 * (pe_prepare_allatonce): solves (B kron M11 + I kron A11) u = rhs for nc right-hand
 * sides per member.  R, U: (E, nc, J, d1).  resid (E * nc, optional): the relative
 * residual ||(B kron M11 + I kron A11) u - rhs|| / ||rhs|| of each solve (:125-131). */
int pe_allatonce_usolve(pe_ctx* ctx, const double* R, double* U, int nc, double* resid,
                        void* stream);

/* WRResult.solver_residual (allatonce.py:296; ImplicitAllAtOnce's guard, :125-131) for the
 * intervals of the last all-at-once solve on this context (pe_fine_allatonce[_loads] or a
 * parareal all-at-once iteration): out (device, E x nc) = ||B U M11 + U A11 - rhs|| / ||rhs||
 * with rhs = build_rhs of each interval's final waveforms, solved on the context's
 * factorisation.  PE_ERR_STATE when no solve has run. */
int pe_wr_solver_residual(pe_ctx* ctx, double* out, void* stream);

/* project_initial (stepping.py:216-226), host arrays: u = M11^-1 Psi1^T M u0 and
 * w = M22^-1 Psi2^T M u0.  M: CSR (n x n); P: CSC (n x d) of hstack([Psi1, Psi2]);
 * M11, M22 row-major; u0 (n); u_out (d1), w_out (d2).  LU with partial pivoting. */
int pe_project_initial(int n, int d1, int d2, const int* M_ptr, const int* M_idx,
                       const double* M_val, const int* P_colptr, const int* P_rowidx,
                       const double* P_val, const double* M11, const double* M22,
                       const double* u0, double* u_out, double* w_out, void* stream);

/* SplitPropagators.stability_max_step (stepping.py:191-207) for one member of the context:
 * power iteration on M22^-1 A22 with the reference's Rayleigh quotient and stopping rule
 * (|lam_new - lam| <= tol |lam_new|, at most max_iter iterations).  bound = 2 / lam
 * (INFINITY when d2 = 0 or A22 = 0); iterations (optional) = the count, negative when
 * max_iter was hit (the reference warns and returns the last bound). */
int pe_stability_max_step(pe_ctx* ctx, int member, double tol, int max_iter, double* bound,
                          int* iterations, void* stream);

/* CEM-GMsFEM basis of a uniform nx x nx Q1 grid cut into nb x nb blocks (
 * msbasis.py:296-394 aux_eigen_cem + build_cem_basis for every block), host arrays:
 * kappa (nx * nx cells, row-major), kt_scale (aux weight kt = kappa * kt_scale; nb^2 for
 * the reference's "kappa_h2").  values: per block b the n_eig basis columns on the
 * patch-interior nodes of b (row-major node order, layers rings of blocks, zero
 * Dirichlet rim), column-major, starting at offsets[b] (offsets: nb^2 + 1 entries);
 * eigenvalues (optional): nb^2 x n_eig aux eigenvalues; worst (optional): the largest
 * constraint residual |C phi - e|.  pe_cem_basis_size gives the values length. */
int pe_cem_basis(int nx, int nb, int layers, int n_eig, const double* kappa, double kt_scale,
                 double* values, long long* offsets, double* eigenvalues, double* worst,
                 void* stream);
long long pe_cem_basis_size(int nx, int nb, int layers, int n_eig);

/* ---- time-dependent loads (the reference's `loads.at(t)`, stepping.py:125,164 and
 * allatonce.py:212-218).  F: device (E, nc, J, d) = [f1(t); f2(t)] for every member,
 * interval column and substep s at the time the reference evaluates it (substep end);
 * Fc: device (E, N, d) = [f1; f2](t_n + Dt) per coarse step.  Same results as the
 * constant-load entry points when every row equals (f1, f2).  The all-at-once variant needs
 * the modal sweep (symmetric-definite pencils, d1, d2 > 0): PE_ERR_ARG otherwise. */
int pe_fine_sequential_loads(pe_ctx* ctx, const double* X_in, double* X_out, int nc,
                             const double* F, void* stream);
int pe_split_step_loads(pe_ctx* ctx, const double* X_in, const double* X_prev, double* X_out,
                        int nc, const double* F, void* stream); /* F: (E, nc, 1, d) */
int pe_fine_allatonce_loads(pe_ctx* ctx, const double* X_in, double* X_out, int nc,
                            const double* F, int* sweeps, int* reasons, double* resid_hist,
                            void* stream);
int pe_coarse_correct_loads(pe_ctx* ctx, int N, const double* X_old, const double* F_hat,
                            double* G_cache, double* X_new, double* diff, const int* active,
                            const double* Fc, void* stream);
int pe_coarse_apply_loads(pe_ctx* ctx, const double* X_in, double* X_out, int nc,
                          const double* Fc, void* stream); /* Fc: (E, nc, d), one per state */

/* ---- batched factor / solve (SURVEY kernel K3; batchlu.cu) ---------------------------
 * Ainv[b] = A[b]^-1 for `batch` row-major n x n matrices (device pointers, batch stride
 * n*n; A is not modified): libpe's recursive blocked LU with partial pivoting, every
 * matrix of the batch in the same launches.  info (host, batch ints): 0, or the 1-based
 * index of the first exactly-zero pivot of that matrix (its inverse is then undefined). */
int pe_batched_inverse(int n, int batch, const double* A, double* Ainv, int* info,
                       void* stream);
/* ImplicitAllAtOnce.__init__'s per-mode inverses (allatonce.py:100-110): for every time mode
 * k = 0 .. J-1, inv(d_k M11 + A11) with d_k = (1 - alpha^(1/J) e^(-2 pi i k / J)) / dt, all
 * modes in one batched pass.  M11, A11: device, row-major d1 x d1.  inv_re / inv_im:
 * device (J, d1, d1) planar real / imaginary parts.  Only modes 0 .. J/2 are factored; the
 * rest are their complex conjugates (real M11, A11).  PE_ERR_SOLVER on a zero pivot. */
int pe_shifted_inverses(int d1, int J, double dt, double alpha, const double* M11,
                        const double* A11, double* inv_re, double* inv_im, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PE_H */
