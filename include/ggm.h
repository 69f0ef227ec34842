/*
 * ggm.h — C ABI of libggm.so, the B200 (sm_100a) hot path of the scalable multi-axis
 * Gaussian graphical model of arXiv 2407.19892 ("GmGM", Andrew, Westhead, Cutillo).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; readings Qn/G/T/TOL are listed
 * in DESIGN.md §"Readings of the paper".
 *
 * Conventions (all entry points)
 *  - Pointers are DEVICE pointers unless marked (host).  The caller owns every buffer;
 *    the library never frees caller memory and keeps no device allocation between calls
 *    except per-thread cuBLAS/cuSOLVER handles.
 *  - Work is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *    default stream).  Calls that return host-visible results synchronize `stream`
 *    (stated per call).
 *  - Errors are return codes; nothing throws across the ABI.  On error, output contents
 *    are unspecified but no out-of-bounds write occurs.  ggm_last_error() returns a
 *    thread-local message for the last non-OK status.
 *  - Tensors are row-major with the FIRST axis at the LARGEST stride, so that
 *    ⊕_l Ψ_l = Σ_l I_{d<l} ⊗ Ψ_l ⊗ I_{d>l} matches vec ordering.
 *  - Only a single modality is supported (the Σ_γ of Thm 2, has one term).
 */
#ifndef GGM_H_
#define GGM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GGM_OK = 0,
  GGM_ERR_INVALID_ARGUMENT = 1, /* null pointer, n<2, k<1, k>n, t<1, L<1, bad axis/mode,
                                   row range outside [0,n), workspace too small, tau<0 */
  GGM_ERR_RANK = 2,             /* k_l > attainable rank or E_k <= 1e-12 E_1
                                   (Cor. 3 P:336-344) */
  GGM_ERR_DOMAIN = 3,           /* non-finite input, E<=0 (Thm 4), lambda<=0 in
                                   sparse_precision (PSD factors), grid sum <= 0 */
  GGM_ERR_NO_CONVERGENCE = 4,   /* max_iter reached; info->stationarity = last residual */
  GGM_ERR_CAPACITY = 5,         /* threshold mode: nnz > capacity; *nnz_out = required */
  GGM_ERR_CUDA = 6,             /* CUDA / cuBLAS / cuSOLVER failure (see ggm_last_error) */
  GGM_ERR_UNSUPPORTED = 7       /* e.g. t > GGM_MAX_TOPK */
} ggm_status;

#define GGM_MAX_TOPK 32
#define GGM_MAX_RANKS 1024

const char *ggm_last_error(void);
int ggm_version(void);
/* 1 if the library was built with the sm_100a tcgen05 path and a device of compute
 * capability 10.x is current; 0 otherwise (no compute is attempted). */
int ggm_device_supported(void);

/* ------------------------------------------------------------------------------------
 * (1) Gram spectrum — Algorithm 1 lines 1-4, Theorem 1.
 *
 * Computes the top-k eigenpairs of the effective Gram matrix S_axis = mat_axis(X)
 * mat_axis(X)^T, i.e. the top-k left singular vectors V of D_axis = mat_axis(X)
 * and E = sigma^2.  fp64 internally: the unfolding is
 * formed in fp64, S (or the dual Gram mat^T mat when d_axis > d_\axis, mapped back with
 * V = mat W diag(1/sigma)) by cuBLAS DSYRK, eigendecomposition by cuSOLVER DSYEVD.
 *
 *  X        : float32, prod(shape) entries, row-major, device.
 *  shape    : (host) ndim extents, each >= 1.
 *  axis     : 0 <= axis < ndim.
 *  k        : 1 <= k <= min(d_axis, d_\axis), else GGM_ERR_RANK.
 *  V        : out float32, d_axis x k row-major (k contiguous), orthonormal columns,
 *             column r = eigenvector of E[r]; the sign of each column is fixed so that its
 *             largest-|.| entry is positive.
 *  E        : out float64, k, descending; GGM_ERR_RANK if E[k-1] <= 1e-12 E[0].
 *  trace_S  : (host, optional) out ||X||_F^2 = tr S_axis (for explained variance).
 *  workspace: device scratch of >= ggm_gram_eig_workspace() bytes (256-byte aligned).
 * Synchronizes `stream` (rank check).
 * ---------------------------------------------------------------------------------- */
ggm_status ggm_gram_eig_workspace(int ndim, const int64_t *shape, int axis, int k,
                                  size_t *bytes);
ggm_status ggm_gram_eig(const float *X, int ndim, const int64_t *shape, int axis, int k,
                        float *V, double *E, double *trace_S, void *workspace,
                        size_t workspace_bytes, void *stream);

/* (1b) At-scale Gram spectrum: the top-k eigenpairs of S_axis by
 * randomized subspace iteration in fp64 (Halko–Martinsson–Tropp range finder with power
 * steps and Rayleigh–Ritz), never forming the d x d Gram: M = mat_axis(X) (fp64 copy,
 * d x m), Y = M Ω (Ω: m x r seeded standard normals, r = k + oversample), Q = qr(Y), then
 * repeated { Z = Mᵀ Q; T = Zᵀ Z = Qᵀ S Q; eig(T); Q = qr(M Z) } until the top-k Ritz
 * values change by <= tol relative to the largest (or max_iter).  V = Q W_k, E = Ritz
 * values.  ggm_gram_eig uses it automatically (oversample = max(16, k), tol 1e-13,
 * max_iter 200) when both sides of the unfolding exceed 32768.  Memory: 8·d·m bytes for
 * the fp64 unfolding + O((d + m)·r).  oversample <= 0 selects max(16, k).
 *  iters_out / change_out (host, optional): iterations run and the last relative change
 *  (> tol when max_iter was reached: the subspace did not converge to tol).
 * Synchronizes `stream` once per iteration. */
ggm_status ggm_gram_eig_rsi_workspace(int ndim, const int64_t *shape, int axis, int k,
                                      int oversample, size_t *bytes);
ggm_status ggm_gram_eig_rsi(const float *X, int ndim, const int64_t *shape, int axis, int k,
                            int oversample, int max_iter, double tol, uint64_t seed, float *V,
                            double *E, double *trace_S, int *iters_out, double *change_out,
                            void *workspace, size_t workspace_bytes, void *stream);

/* (1h) Every axis of one tensor (Alg. 1 lines 1-4 for l = 0 .. ndim-1): the same results as
 * ndim ggm_gram_eig calls (V[a]: shape[a] x k[a], E[a]: k[a]), but the per-axis Gram
 * eigensolves run concurrently on library-owned side streams forked from and joined back onto
 * `stream` (cuSOLVER's reduction of a few-hundred-square Gram is latency-bound).  Workspace:
 * the per-axis workspaces, each 256-byte aligned, back to back.  Synchronises `stream`.
 * Errors as ggm_gram_eig (the first failing axis). */
ggm_status ggm_gram_eig_axes_workspace(int ndim, const int64_t *shape, const int *k, size_t *bytes);
ggm_status ggm_gram_eig_axes(const float *X, int ndim, const int64_t *shape, const int *k,
                             float *const *V, double *const *E, double *trace_S, void *workspace,
                             size_t workspace_bytes, void *stream);

/* (1g) Both axes of a matrix X (d0 x d1, row-major fp32) from ONE Gram of the shorter side
 * and one eigensolve (Thm 1 / P:125: the nonzero spectra of X X^T and X^T X coincide, and
 * the longer side's eigenvectors are X^T W diag(1/σ) or X W diag(1/σ)).  Outputs as
 * ggm_gram_eig per axis (V0: d0 x k0, E0; V1: d1 x k1, E1; E0[i] = E1[i]); shorter side
 * <= 32768. */
ggm_status ggm_gram_eig_matrix_workspace(int64_t d0, int64_t d1, int k0, int k1, size_t *bytes);
ggm_status ggm_gram_eig_matrix(const float *X, int64_t d0, int64_t d1, int k0, int k1, float *V0,
                               double *E0, float *V1, double *E1, double *trace_S,
                               void *workspace, size_t workspace_bytes, void *stream);

/* (1c) Multi-modal spectrum of one shared axis l (Alg. 1 line 2): the top-k left
 * singular vectors of D_l = [mat_l(D^γ1) ... mat_l(D^γΓ)] — the eigenpairs of
 * S_l = Σ_γ mat_l(D^γ) mat_l(D^γ)^T.  M modalities; X[g] (host array of DEVICE pointers)
 * is modality g's row-major fp32 tensor with ndim[g] axes, shapes[] concatenates all M
 * shapes (host), axis_pos[g] = position of axis l in modality g or -1 if absent (its X[g]
 * may then be NULL).  The shared axis must have the same length in every modality that has
 * it.  Output as ggm_gram_eig (V: d_l x k fp32, E: k fp64 descending, trace_S = ||D_l||_F^2);
 * dense path up to a 32768^2 Gram of either side, randomized subspace iteration above.
 * Nonparanormal (COCA) on a shared axis ranks each row of the concatenation D_l: build
 * D_l as one d_l x Σm matrix and use ggm_nonparanormal(axis 0) + ggm_gram_eig (or the CSR
 * path with nonparanormal = 1). */
ggm_status ggm_gram_eig_multi_workspace(int M, const int *ndim, const int64_t *shapes,
                                        const int *axis_pos, int k, size_t *bytes);
ggm_status ggm_gram_eig_multi(int M, const float *const *X, const int *ndim,
                              const int64_t *shapes, const int *axis_pos, int k, float *V,
                              double *E, double *trace_S, void *workspace,
                              size_t workspace_bytes, void *stream);

/* (1d) Sparse unfolding (§8(f) rows 1 and 4).  D_l given as CSR: d rows (the
 * axis), m columns, nnz stored entries (row_ptr int64 d+1, col int32, val fp32; DEVICE).
 * Columns ascending within each row.  When min(d, m) <= 32768 the Gram of the shorter
 * side is accumulated exactly over bounded dense chunks (1 GiB) of the matrix by fp64 DSYRK
 * and eigensolved densely (iters_out = 0); otherwise randomized subspace iteration (as
 * (1b)) with cuSPARSE SpMM products.  The whole matrix is never densified.
 * nonparanormal = 1 applies the COCA transform first (row ranks among all m
 * entries incl. the implicit zeros, ties -> smallest rank, Φ^-1(r/(m+1))) in its sparse
 * rank-one form S + z 1^T (S keeps D's pattern): the operator products add the
 * rank-one terms z (1^T X) and 1 (z^T Y) instead of a rank-one SVD update.  Output as
 * ggm_gram_eig; trace_S = ||A||_F^2 of the (transformed) matrix.  Synchronizes `stream`. */
ggm_status ggm_gram_eig_csr_workspace(int64_t d, int64_t m, int64_t nnz, int k, int oversample,
                                      size_t *bytes);
ggm_status ggm_gram_eig_csr(int64_t d, int64_t m, int64_t nnz, const int64_t *row_ptr,
                            const int32_t *col, const float *val, int k, int nonparanormal,
                            int oversample, int max_iter, double tol, uint64_t seed, float *V,
                            double *E, double *trace_S, int *iters_out, double *change_out,
                            void *workspace, size_t workspace_bytes, void *stream);

/* (1e) Dense nonparanormal skeptic / COCA: out (same shape and layout as X) =
 * Φ^-1(r/(m+1)), r = rank of the entry (ties -> smallest rank, reading Q19) among the
 * m = d_rest entries with the same index on `axis`.  Feed `out` to ggm_gram_eig(axis). */
ggm_status ggm_nonparanormal_workspace(int ndim, const int64_t *shape, int axis, size_t *bytes);
ggm_status ggm_nonparanormal(const float *X, int ndim, const int64_t *shape, int axis, float *out,
                             void *workspace, size_t workspace_bytes, void *stream);

/* (1f) Sharded spectrum (§8(f) row 1: "sharded Gram with one all-reduce").  A matrix whose
 * rows (the long axis, e.g. cells) are split over ranks, m <= 32768 columns (e.g. genes):
 *   ggm_gram_accumulate_csr: G (m x m, fp64 column-major, LOWER triangle) = (accumulate ?
 *     G : 0) + A_r^T A_r over this rank's CSR rows (COCA of each row when nonparanormal = 1,
 *     as (1d)); optional *fro_out (host) = ||A_r||_F^2.  The caller all-reduces G.
 *   ggm_eig_gram: top-k eigenpairs of G (G overwritten): V (m x k fp32 row-major, the
 *     short-axis factor), E (k, descending), W (m x k fp64 column-major, same signs as V).
 *   ggm_project_csr: this rank's rows of the long-axis factor V_r = A_r W diag(E^-1/2)
 *     (d x k fp32 row-major; signs follow W, consistent across ranks).
 * With nonparanormal = 1 both factors belong to the row-wise (long-axis) COCA transform. */
ggm_status ggm_gram_accumulate_csr_workspace(int64_t d, int64_t m, int64_t nnz, size_t *bytes);
ggm_status ggm_gram_accumulate_csr(int64_t d, int64_t m, int64_t nnz, const int64_t *row_ptr,
                                   const int32_t *col, const float *val, int nonparanormal,
                                   double *G, int accumulate, double *fro_out, void *workspace,
                                   size_t workspace_bytes, void *stream);
ggm_status ggm_eig_gram_workspace(int64_t dim, int k, size_t *bytes);
ggm_status ggm_eig_gram(int64_t dim, double *G, int k, float *V, double *E, double *W,
                        void *workspace, size_t workspace_bytes, void *stream);
ggm_status ggm_project_csr_workspace(int64_t d, int64_t m, int64_t nnz, int k, size_t *bytes);
ggm_status ggm_project_csr(int64_t d, int64_t m, int64_t nnz, const int64_t *row_ptr,
                           const int32_t *col, const float *val, int nonparanormal, int k,
                           const double *W, const double *E, float *V, void *workspace,
                           size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * (2) Eigenvalue MLE — Theorem 2, Algorithm 1 lines 5-17.
 *
 * Minimises NLL(λ) = ½ Σ_l E_l·λ_l − ½ Σ_{j in k-grid} log s_j, s_j = Σ_l λ_l[j_l]
 * for ONE modality with L axes, over the paper's domain λ_l >= ε (Lemma 6,
 * P:657-690), ε = eps_scale · max(1/E).  The gradient ½(E_l − g_l),
 * g_l[i] = Σ_{j: j_l = i} 1/s_j, is evaluated by a grid-reduction kernel
 * over all prod(k) grid points, never materialising the grid.
 *
 * Reading T: the marginals of every axis sum to the same Σ_j 1/s_j, so an interior
 * stationary point needs equal traces tr E_l.  If the relative trace spread
 * (trace_inconsistency) is <= opts->trace_tol the spectrum is replaced by its projection on
 * G⊥ (the rounding-level gauge component dropped) and the interior MLE is returned
 * (floor_active = 0).  Otherwise the NLL decreases without bound along a gauge direction
 * and the minimum lies on the barrier: the majorise-minimise step is clamped at ε (a
 * separable majoriser minimised on the box), every axis but the smallest-trace one ends with
 * coordinates on the floor, and floor_active = 1 ("pick a smaller k").
 *
 *  L      : number of axes, 1 <= L <= 8.
 *  k      : (host) L ranks; prod(k) < 2^40; max k <= 1024.
 *  E      : float64 sum(k), axis-concatenated Gram eigenvalues, each > 0 and finite
 *           (else GGM_ERR_DOMAIN).
 *  opts   : (host, may be NULL = defaults).
 *  lambda : out float64 sum(k), axis-concatenated, in the gauge opts->gauge (written also
 *           when GGM_ERR_NO_CONVERGENCE is returned: the last iterate).
 *  info   : (host, may be NULL) diagnostics.
 * Scratch of O(Σk) doubles is taken with stream-ordered cudaMallocAsync and released
 * before returning.  Synchronizes `stream`.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  double tol;        /* stop when the stationarity residual <= tol (reading Q4): max over
                        coordinates of |E_li − g_li| (off the floor) or max(0, g_li − E_li) (on
                        it, a KKT multiplier), / max E.  default 1e-7 */
  int max_iter;      /* grid passes (methods 0, 1) or accepted steps (method 2); default 20000 */
  double eps_scale;  /* floor ε = eps_scale * max(1/E). default 1e-10 */
  int method;        /* 0 = majorise-minimise fixed point λ ← λ ⊙ g/E (the NLL decreases
                          monotonically, λ stays > 0) accelerated by SQUAREM extrapolation in
                          log space (3 passes per cycle, residual safeguard); the barrier
                          regime and a non-converging accelerated run use the plain step;
                        1 = the plain majorise-minimise step only;
                        2 = Algorithm 1 as printed: Λ' = Λ − μ·½(E − g) (reading Q1), μ halved
                          while the grid minimum Σ_l min Λ'_l < ε or the NLL does not decrease
                          (readings Q2, Q3), never increased; slow (thousands of steps), the
                          paper's reference method.
                        Other values: GGM_ERR_INVALID_ARGUMENT.  (Projected Newton is the
                        oracle's algorithm, not offered here: DESIGN.md BK4.) */
  int gauge;         /* 0 = min-balanced PSD gauge (default, reading G);
                        1 = Algorithm 1's gauge, (λ − 1/E) ⊥ G (the gauge gradient steps from
                          λ0 = 1/E keep).  In the barrier regime both act only among the axes
                          with no coordinate on the floor. */
  double trace_tol;  /* interior regime when trace_inconsistency <= trace_tol (reading T);
                        default 1e-8 */
} ggm_solve_opts;

typedef struct {
  int iterations;             /* grid passes (methods 0, 1) or accepted steps (method 2) */
  double stationarity;        /* the tol residual at exit (KKT form, against the projected
                                 spectrum in the interior regime) */
  double nll;                 /* NLL of the returned λ with the given E */
  double grid_min;            /* min_j s_j = Σ_l min λ_l */
  double trace_inconsistency; /* max_l |tr E_l − mean| / mean (reading T) */
  int floor_active;           /* 1 if some λ is on the floor ε (barrier regime) */
  int passes;                 /* grid passes evaluated (all methods; method 2 also counts
                                 rejected step sizes) */
  double kernel_ms;           /* device time of the solve kernel(s), CUDA events on `stream` */
} ggm_solve_info;

void ggm_solve_opts_default(ggm_solve_opts *opts);
ggm_status ggm_solve_eigvals(int L, const int *k, const double *E, const ggm_solve_opts *opts,
                             double *lambda, ggm_solve_info *info, void *stream);

/* (2b) Multi-modal eigenvalue MLE (Thm 2 with Σ_γ; shared axes P:170-181):
 * A global axes with ranks k[A] and axis-concatenated E (from ggm_gram_eig_multi of each
 * axis); M <= 8 modalities, modality g = global axes mod_axes[mod_ptr[g] .. mod_ptr[g+1])
 * (host; no repeated axis within a modality, every axis in some modality).  Minimises
 * ½ Σ_l E_l·λ_l − ½ Σ_γ Σ_{j in grid γ} log s^γ_j by the majorise-minimise step
 * λ ← λ ⊙ (Σ_{γ∋l} g^γ_l) / E_l.  Gauge 0 (reading G2): λ_l − (P_G μ)_l with μ_l = min λ_l
 * and P_G the projector onto the shifts that keep every modality's grid sums (one modality:
 * identical to ggm_solve_eigvals' gauge 0).  info as ggm_solve_eigvals (grid_min = the
 * smallest modality grid minimum).  Synchronizes `stream`. */
ggm_status ggm_solve_eigvals_multi(int A, const int *k, const double *E, int M,
                                   const int *mod_ptr, const int *mod_axes,
                                   const ggm_solve_opts *opts, double *lambda,
                                   ggm_solve_info *info, void *stream);

/* Grid marginals alone (the Thm 2 trace term), for parity tests and the bench:
 * g (out, float64 sum(k)) and, if logsum_out != NULL, F = Σ_j log s_j (host).  Synchronizes
 * `stream` only when logsum_out != NULL. */
ggm_status ggm_grid_marginals(int L, const int *k, const double *lambda, double *g,
                              double *logsum_out, void *stream);

/* ------------------------------------------------------------------------------------
 * (3) Fused recomposition + sparsification — Alg. 1 lines 18-20 ("Threshold
 * simultaneously"), P:945, P:949 (never store the n x n matrix), P:1018 (per-vertex top-n).
 *
 * For rows i in [row_begin, row_end) of Ψ = V diag(λ) V^T (Cor. of Thm 2) and
 * ALL n columns j != i, keeps
 *   mode 0: the t_eff = min(t, n−1) entries of largest |ψ_ij|, ties -> smaller j (Q8, Q9)
 *   mode 1: every entry with |ψ_ij| > tau (tau >= 0; e.g. the Thm 5 critical value, Q15)
 * and writes directed per-row CSR, columns ascending within a row (Q10).  The contraction
 * runs on tcgen05 tensor cores with a 3-term fp16 split (hi·hi + hi·lo + lo·hi, one
 * power-of-two scale) accumulated in fp32 TMEM; the n x n matrix is never written.
 *
 *  V        : float32 n x k row-major, finite.
 *  lambda   : float64 k, each > 0 and finite (PSD factors; the solver's gauge 0
 *             guarantees this), else GGM_ERR_DOMAIN.
 *  row_ptr  : out int64 rows+1 (rows = row_end − row_begin), offsets from 0.
 *  col      : out int32 global column ids;  val: out float32 ψ_ij.
 *  capacity : entries available in col/val.  mode 0 needs rows*t_eff.
 *  nnz_out  : (host) out number of entries written (mode 1: required count when
 *             GGM_ERR_CAPACITY is returned — two-call protocol).
 *  workspace: >= ggm_sparse_precision_workspace() bytes, 256-byte aligned.
 * Synchronizes `stream` (status and nnz are host-visible).
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int mode;   /* 0 top-t per row by |ψ| (j != i); 1 |ψ| > tau (j != i) */
  int topk;   /* t, 1 <= t <= GGM_MAX_TOPK; effective t_eff = min(t, n−1) */
  float tau;  /* mode 1 only, >= 0 */
  int col_chunks; /* 0 = automatic; else split each row block's column sweep into this
                     many chunks merged afterwards (balances small row ranges) */
  int symmetric;  /* scheme selection, over the FULL axis (row_begin = 0, row_end = n) with
                     A resident (otherwise always plain):
                     0 = automatic (symmetric for full axes with n >= 16384), 1 = symmetric, 2 = plain.
                     Symmetric scheme (Ψ = Ψ^T): a seed pass over the n/32 columns of
                     largest ||U_j|| (at least 48 256-column tiles while that is <= 1/8 of
                     the axis; hi·hi products) gives each row i a lower bound b_i of
                     its t-th |ψ| (t-th largest 32-column chunk maximum, minus the hi·hi
                     rounding bound 2^-10·1.1·||U_i||·max_j||U_j||); rows are reordered by b_i; each
                     unordered 128x128 block pair is then evaluated once (cyclic window per
                     row block) and entry ψ_ij is kept as a candidate of row i if
                     |ψ| >= b_i and of row j if |ψ| >= the smallest bound of j's 8-column
                     group (a superset of |ψ| >= b_j; bounds in a group are nearly equal);
                     a CUB sort by row and a merge select each row's top t by
                     (|ψ| desc, j asc) — extra candidates below b_j never reach row j's top t.  For k <= 128 the main
                     pass computes hi·hi only, with every threshold lowered by its error
                     bound, and the candidates are re-evaluated exactly (fp64 sums of the
                     fp32 inputs) before the selection.  Mode 1 uses τ as every row's bound
                     (no seed pass; the pool holds 1.25 x capacity).  If the candidate pool
                     fills up, the axis is recomputed with the plain scheme (exact). */
} ggm_sparsify_opts;

ggm_status ggm_sparse_precision_workspace(int64_t n, int k, int64_t row_begin, int64_t row_end,
                                          const ggm_sparsify_opts *opts, int64_t capacity,
                                          size_t *bytes);
ggm_status ggm_sparse_precision(int64_t n, int k, const float *V, const double *lambda,
                                int64_t row_begin, int64_t row_end,
                                const ggm_sparsify_opts *opts, int64_t *row_ptr, int32_t *col,
                                float *val, int64_t capacity, int64_t *nnz_out,
                                void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * (3b) Distributed symmetric scheme (multi-GPU form of symmetric = 1; SURVEY §8(e)/(f),
 * DESIGN.md §5).  One process per GPU; every rank calls with the same (n, k, V, λ, opts).
 *
 * ggm_sparse_precision_sym_shard: runs the replicated phases (row norms, seed pass, the two
 * orderings and splits — deterministic, so every rank derives the same permutation) and
 * this rank's share of the symmetric units (a unit = one of the 8 sub-windows of a 256-row
 * block's column window in the bound-ordered axis).  nranks in {2, 4, 8}: folded
 * part-major — rank r owns sub-windows j and 7 − j of every row block for the j ≡ r (mod
 * nranks) (at nranks = 8: j = r on even, 7 − r on odd row blocks); other nranks:
 * rank-strided units r, r + nranks, ...  (GGM_SYM_ASSIGN=strided forces the latter).
 * Every unit is evaluated by exactly one rank.  Outputs this rank's
 * candidates sorted by target row, as two device arrays: cand_key[e] = target row (bound
 * order index), cand_val[2e..2e+1] = (source row, bound order index; ψ as float bits);
 * counts[r] (host) = number of candidates whose target row rank r owns (contiguous in the
 * sorted arrays, in rank order); perm (device, n int32) = bound order index -> original row
 * id.  Rank r owns bound-order rows [ggm_sym_rows_begin(.., r, ..), ggm_sym_rows_begin(..,
 * r+1, ..)).  Errors: GGM_ERR_CAPACITY if the candidates exceed cand_capacity or the
 * internal pool (callers fall back to the row-sharded plain scheme); GGM_ERR_UNSUPPORTED for
 * mode 1 or k > 128.  Synchronizes `stream`.
 *
 * ggm_sym_merge: after the caller's all-to-all exchange of the buckets, merges the
 * candidates of this rank's rows [row_begin, row_end) (bound order; ncand candidates in any
 * order): row j's top t_eff by (|ψ| desc, original column asc), written at local row
 * j - row_begin: row_id[j - row_begin] = perm[j] (original row id), col/val[(j - row_begin)
 * * t_eff + 0..t_eff-1] in ascending original column order.  Workspace from
 * ggm_sym_merge_workspace(ncand).  Asynchronous. */
int64_t ggm_sym_rows_begin(int64_t n, int k, const ggm_sparsify_opts *opts, int rank,
                           int nranks);
ggm_status ggm_sparse_precision_sym_shard_workspace(int64_t n, int k,
                                                    const ggm_sparsify_opts *opts,
                                                    size_t *bytes);
ggm_status ggm_sparse_precision_sym_shard(int64_t n, int k, const float *V,
                                          const double *lambda, const ggm_sparsify_opts *opts,
                                          int rank, int nranks, uint32_t *cand_key,
                                          uint32_t *cand_val, int64_t cand_capacity,
                                          int64_t *counts, int32_t *perm, void *workspace,
                                          size_t workspace_bytes, void *stream);
/* Sharded seed pass (optional; saves each rank the whole seed pass): ggm_sym_seed_shard
 * writes, into thr_out (DEVICE, n floats), the raw seed values of this rank's equal share of
 * the row blocks (rows in descending-norm order) and +inf for all other rows; the caller
 * combines the ranks' arrays by an element-wise minimum (one all-reduce MIN) and passes the
 * result to ggm_sparse_precision_sym_shard_seeded, which skips the seed pass and is
 * otherwise identical to ggm_sparse_precision_sym_shard.  Same workspace size.  When the
 * seeded call gets the same workspace (and V, λ, n, k, topk, mode, nranks) as this rank's
 * ggm_sym_seed_shard call, it also reuses the scale, row norms and norm order that call left
 * there (host-side stamp per workspace address, consumed once; any other library call on
 * that workspace discards it) — V and λ must not change in between, as thr_all already
 * requires.
 * ggm_sym_seed_shard synchronizes `stream`. */
ggm_status ggm_sym_seed_shard(int64_t n, int k, const float *V, const double *lambda,
                              const ggm_sparsify_opts *opts, int rank, int nranks,
                              float *thr_out, void *workspace, size_t workspace_bytes,
                              void *stream);
ggm_status ggm_sparse_precision_sym_shard_seeded(int64_t n, int k, const float *V,
                                                 const double *lambda,
                                                 const ggm_sparsify_opts *opts, int rank,
                                                 int nranks, const float *thr_all,
                                                 uint32_t *cand_key, uint32_t *cand_val,
                                                 int64_t cand_capacity, int64_t *counts,
                                                 int32_t *perm, void *workspace,
                                                 size_t workspace_bytes, void *stream);
ggm_status ggm_sym_merge_workspace(int64_t ncand, size_t *bytes);
ggm_status ggm_sym_merge(int64_t n, int t, const uint32_t *cand_key, const uint32_t *cand_val,
                         int64_t ncand, const int32_t *perm, int64_t row_begin, int64_t row_end,
                         int64_t *row_id, int32_t *col, float *val, void *workspace,
                         size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * (3c) Whole-graph edge rules (readings in
 * DESIGN.md Q16): keep the n_edges largest undirected edges overall by score |ψ_ij|, or by
 * |ψ_ij| / sqrt(w_i·w_j) with w_i = Σ_{k≠i} |ψ_ik| when downweight = 1 ("down-weighting edges
 * of vertices with high degree"), then add each vertex's min_edges best edges by the
 * same score — ties -> smaller (i, j).  Output: symmetric CSR (each kept edge in
 * rows i and j), columns ascending, values ψ_ij; nnz_out = 2·|edges|.
 * Errors: GGM_ERR_CAPACITY if nnz > capacity (*nnz_out = required), or if the candidate
 * pass needs more than cand_capacity entries (*nnz_out = -required); both retry-able.
 * Synchronizes `stream`. */
typedef struct {
  int64_t n_edges;  /* N >= 1 (the paper keeps ~10 edges per vertex on scRNA-seq) */
  int downweight;   /* 0: score |ψ_ij|; 1: |ψ_ij| / sqrt(w_i w_j) */
  int min_edges;    /* 0..GGM_MAX_TOPK edges per vertex always kept */
} ggm_overall_opts;
ggm_status ggm_sparse_precision_overall_workspace(int64_t n, int k, const ggm_overall_opts *opts,
                                                  int64_t cand_capacity, size_t *bytes);
ggm_status ggm_sparse_precision_overall(int64_t n, int k, const float *V, const double *lambda,
                                        const ggm_overall_opts *opts, int64_t cand_capacity,
                                        int64_t *row_ptr, int32_t *col, float *val,
                                        int64_t capacity, int64_t *nnz_out, void *workspace,
                                        size_t workspace_bytes, void *stream);

/* Candidate path of this thread's last ggm_sparse_precision_overall call: 3 = a global
 * threshold τ from a uniform pair sample + one symmetric pass with per-row bounds
 * min(top-m bound, τ), exact once >= n_edges pairs exceed τ (default from n >= 65,536;
 * otherwise, or when its checks fail, the lists paths): 0 = the per-row top-t1 lists held
 * the top N pairs (no saturated row), 2 = lists + the saturated rows' block, 1 = histogram
 * + full threshold pass; -1 before any call.  *saturated (optional) = rows whose t1-th
 * listed score reached L3 (0 on path 3).  ms (optional, filled when ggm_set_timing(1) was
 * on): device time of the phases (row masses + scaling, top-t1 lists or the path-3 sample +
 * pass, bound L3 + saturation, candidate pass, ranking + CSR). */
int ggm_overall_last_path(int64_t *saturated, float ms[5]);

/* ------------------------------------------------------------------------------------
 * (4) Edge significance (Theorem 5, P:768-; Corollary 10) — host-side scalars.
 * Single modality: z = sqrt(d_rest)·sigma²·psi/2 ~ N(0,1) under the empty-graph null, with
 * d_rest = d_\l (product of the other axes) and sigma² the null variance (1 after whole-data
 * standardisation, 1/L after per-axis standardisation).  p_raw = 2(1 - Phi(|z|)),
 * p_bonferroni = min(1, n_tests·p_raw) (n_tests: all off-diagonal pairs of the tested axes,
 * "after applying the Bonferroni correction").
 * ggm_wald_threshold: the critical magnitude tau = 2·Phi^-1(1 - alpha/(2 n_tests)) /
 * (sqrt(d_rest)·sigma²): |psi| > tau <=> p_bonferroni < alpha (p = 0.05 after
 * Bonferroni), for ggm_sparse_precision mode 1. */
ggm_status ggm_wald_edge(double psi, int64_t d_rest, double sigma2, int64_t n_tests, double *z,
                         double *p_raw, double *p_bonferroni);
ggm_status ggm_wald_threshold(int64_t d_rest, double sigma2, double alpha, int64_t n_tests,
                              double *tau);

/* Per-kernel timing of the last ggm_sparse_precision call on this thread, measured with
 * CUDA events on `stream` when enabled (for bench.py's roofline).  ms[0] = prep (absmax +
 * split, + the seed pass in the symmetric scheme), ms[1] = main fused tcgen05 kernel,
 * ms[2] = merge/CSR assembly. */
void ggm_set_timing(int enabled);
void ggm_last_timing(float ms[3]);
/* Number of libggm kernels launched by the last call on this thread (library kernels such
 * as cuBLAS/cuSOLVER/CUB internals are not counted). */
int ggm_last_launches(void);
/* Statistics of the last ggm_sparse_precision call on this thread: out[0] = scheme (0 plain,
 * 2 symmetric), out[1] = entries evaluated by the main fused kernel (incl. padding),
 * out[2] = candidates emitted (symmetric scheme), out[3] = 1 if the symmetric scheme's
 * candidate pool overflowed and the axis was recomputed with the plain scheme, out[4] = MMA
 * K elements issued per evaluated entry (16 x (3 full slots + packed tail slots)), out[5] =
 * 1 if the CTA-pair (cta_group::2) kernels ran. */
void ggm_last_stats(double out[6]);

#ifdef __cplusplus
}
#endif
#endif /* GGM_H_ */
