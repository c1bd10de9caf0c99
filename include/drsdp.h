/*
 * drsdp.h — C ABI of libdrsdp.so, the B200-native (sm_100a, fp64) hot path of
 * ManiDSDP, the dual Riemannian ADMM for unit-diagonal SDPs of arXiv 2512.04406.
 *
 * Citations "P:n" are line numbers of the paper's LaTeX source.
 *
 * The problem (DSDP), P:19-27:
 *     inf_y  b^T y   s.t.  S = A*(y) - C  is PSD,  diag(S) = 1,
 * with A(X) = (<A_a, X>)_a and A*(y) = sum_a y_a A_a. The library takes A as a
 * monomial-index map: A_a is the symmetric 0/1 indicator of the positions (i, j) whose
 * id is a, so <A_a, X> sums X over those ordered positions (off-diagonal entries count
 * twice) and AA* = Diag(cnt) with cnt_a = number of ordered positions of a.
 * Assumption 2 (AA* invertible) is checked: every id must own a position.
 *
 * Conventions
 *  - fp64 everywhere, row-major, 0-based indices; n = matrix side, m = #constraints,
 *    p = factor width (columns of Y).
 *  - Every call returns a drsdp_status (0 = OK). No exception or abort crosses the ABI.
 *    After an error drsdp_last_error(ctx) holds a one-line message. ERR_CUDA and
 *    ERR_OOM are sticky: the context must be destroyed.
 *  - A context is single-threaded (one host thread at a time); distinct contexts are
 *    independent. All device work of a context runs on its one CUDA stream.
 *  - Ownership: pointers marked HOST are read (or written) during the call only; the
 *    library copies what it keeps. Pointers marked DEVICE are caller-owned device
 *    memory; "BORROWED" ones must stay valid until the documented release point.
 *  - There is no CPU fallback: without a usable CUDA device drsdp_create fails with
 *    DRSDP_ERR_CUDA.
 */
#ifndef DRSDP_H
#define DRSDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct drsdp_ctx drsdp_ctx; /* opaque; owns every device buffer it allocates */

/* Largest factor width p accepted anywhere (evaluations, initial factor, solver rank growth).
 * p <= 64 runs the fused single-pass kernels; 64 < p <= DRSDP_MAX_P runs the product kernel in
 * column chunks of 64 followed by separate row-epilogue kernels (same arithmetic). The solver's rank
 * growth (escape columns) stops at min(DRSDP_MAX_P, n): at d = 100 the cap 1024 of round 1
 * was reached while X still had ~1000 negative eigenvalues, hence 4096. */
#define DRSDP_MAX_P 4096

typedef enum {
  DRSDP_OK = 0,
  DRSDP_ERR_INVALID_ARG = 1,   /* NULL where not allowed, n <= 0, p < 1, id out of range, bad sizes */
  DRSDP_ERR_NOT_SYMMETRIC = 2, /* map(i,j) != map(j,i), duplicate (i,j), or C not symmetric         */
  DRSDP_ERR_SINGULAR_AAT = 3,  /* a constraint id with no position: Assumption 2 violated     */
  DRSDP_ERR_STATE = 4,         /* wrong call order (e.g. solve before set_problem, HVP before COSTGRAD) */
  DRSDP_ERR_CUDA = 5,          /* CUDA / cuSOLVER failure (sticky)                                    */
  DRSDP_ERR_OOM = 6,           /* device allocation failed (sticky)                                   */
  DRSDP_ERR_NOT_CONVERGED = 7, /* solve hit max_outer or time_limit; solution and trace retrievable   */
  DRSDP_ERR_NUMERIC = 8        /* non-finite cost/gradient, or a zero row in a retraction              */
} drsdp_status;

/* ---------------------------------------------------------------------------------------------
 * Lifetime
 * ------------------------------------------------------------------------------------------- */

/* Create a context on CUDA device `device`. cuda_stream is a cudaStream_t to run on (the caller
 * keeps ownership and must keep it alive until destroy; cudaStreamLegacy = (void*)1 selects the
 * legacy default stream), or NULL to let the context create its own non-blocking stream. */
int drsdp_create(drsdp_ctx **out, int device, void *cuda_stream);
void drsdp_destroy(drsdp_ctx *ctx);                 /* NULL-safe; frees all device memory      */
const char *drsdp_last_error(const drsdp_ctx *ctx); /* valid until the next call on ctx        */
int drsdp_sync(drsdp_ctx *ctx);                     /* wait for all work queued on ctx's stream */

/* ---------------------------------------------------------------------------------------------
 * Problem data (DSDP)
 * ------------------------------------------------------------------------------------------- */

/* General index-map problem. HOST pointers, copied.
 *   C       n*n row-major symmetric cost matrix, or NULL meaning C = 0 (the BQP case).
 *   row,col,cons  nnz COO triplets over the upper triangle (row <= col): position (row,col) and
 *           its mirror belong to constraint id cons in [0, m). Each (row,col) at most once.
 *           Positions absent from the list are unconstrained by A (they belong to no A_a).
 *   b       length m.
 * Errors: INVALID_ARG (sizes, ids out of range, row > col), NOT_SYMMETRIC (duplicate position
 * or asymmetric C), SINGULAR_AAT (an id with no position, Assumption 2). */
int drsdp_set_problem(drsdp_ctx *ctx, int64_t n, int64_t m, const double *C, int64_t nnz,
                      const int32_t *row, const int32_t *col, const int32_t *cons,
                      const double *b);

/* Dense second-order BQP relaxation: min x^T Q x + c^T x over x in {-1,1}^d.
 * Basis v(x) = [1, x_1..x_d, x_1x_2, .., x_{d-1}x_d] (graded-lex); one constraint per
 * square-free monomial of degree <= 4 (graded-lex); amap(i,j) = id of the symmetric
 * difference of the two basis monomials; b_{1} = tr Q, b_{x_i} = c_i, b_{x_ix_j} = 2 Q_ij,
 * degree 3-4 -> 0; C = 0. n = 1 + d + d(d-1)/2, m = sum_{k<=4} C(d,k). HOST pointers:
 * Q d*d symmetric, c length d. Requires 1 <= d <= 360 (n < 65536). */
int drsdp_set_bqp(drsdp_ctx *ctx, int32_t d, const double *Q, const double *c);

/* ---------------------------------------------------------------------------------------------
 * Multi-block problems (remark P:434-436: Algorithm 2 on multi-block SDPs;
 * the sparse BQP relaxation DSDP-sparse). S = diag(S_1, .., S_t), every block
 * S_k = Y_k Y_k^T in S^+_{nb}, diag S_k = 1; one y per constraint, SHARED by all blocks whose
 * positions it owns; C = 0. The factor Y stacks the blocks' rows: n = t * nb rows (block k owns
 * rows k*nb .. (k+1)*nb - 1); only the diagonal blocks exist. Uniform block size nb.
 * Solver differences (readings R37-R39): no tCG preconditioner; the eigen step is one
 * batched decomposition of all blocks (cusolverDnXsyevBatched), eta_d and the escape directions
 * from the union of the blocks' spectra; p <= min(128, nb); ALM mode only.
 * Every call below (solve, alm_eval, y_update, dual_update, get_solution, export_index_map)
 * accepts a block problem with these layouts:
 *   T, M (device): n x ldt "stacked" — row r holds the nb columns of its block (ldt >= nb);
 *   export_index_map: amap n*nb (row r, local column j); seg_pos packs GLOBAL rows (r<<16)|r';
 *   get_solution: X is t column-major nb x nb blocks (t*nb*nb doubles).
 * drsdp_assemble_M and drsdp_x_eigs are dense-only (ERR_INVALID_ARG).
 * ------------------------------------------------------------------------------------------- */

/* General uniform multi-block problem. HOST inputs: amaps t*nb*nb int32 (block k row-major at
 * amaps + k*nb*nb; ids in [0, m), each block symmetric; every constraint owns >= 1 position,
 * Assumption 2), b length m. Requires t*nb < 65536. Errors: INVALID_ARG, NOT_SYMMETRIC,
 * SINGULAR_AAT (empty constraint); on error the previous problem is kept. */
int drsdp_set_blocks(drsdp_ctx *ctx, int32_t t, int32_t nb, int64_t m, const int32_t *amaps, const double *b);

/* Clique-chain sparse BQP relaxation: cliques x_k = {x_{(q-2)k}, .., x_{(q-2)k+q-1}}
 * (0-based, k < t; consecutive cliques share two variables), objective
 * sum_k x_k^T Q_k x_k + c_k^T x_k over {-1,1}^d, d = (q-2)t + 2. One block per clique with basis
 * v(x_k) = [1, x_k, products of two clique variables] (graded-lex, nb = 1 + q + q(q-1)/2); one
 * constraint per square-free monomial of degree <= 4 of some clique, ids in graded-lex order of
 * sorted global index tuples; b_1 = sum_k tr Q_k, b_{x_i} = sum_k c_{k,i}, b_{x_ix_j} =
 * sum_k 2 Q_{k,ij}, degree 3-4 -> 0. HOST inputs: Q t*q*q (block k row-major, symmetric), c t*q.
 * Requires q >= 2, t*nb < 65536. */
int drsdp_set_bqp_chain(drsdp_ctx *ctx, int32_t q, int32_t t, const double *Q, const double *c);

/* Block structure of the current problem: t and nb (t = 0 and nb = n for a dense problem). */
int drsdp_get_block_sizes(drsdp_ctx *ctx, int32_t *t, int32_t *nb);

/* Sizes of the current problem (n, m, and the number of upper-triangle positions owned by
 * some constraint). Any output pointer may be NULL. */
int drsdp_get_sizes(drsdp_ctx *ctx, int64_t *n, int64_t *m, int64_t *n_upper);

/* Bit-exact export of the index map for parity tests. HOST outputs, caller-allocated:
 *   amap     n*n int32, amap[i*n+j] = id of position (i,j), -1 if unconstrained;
 *   seg_ptr  m+1 int64 CSR offsets into seg_pos (constraint-major);
 *   seg_pos  n_upper uint32, upper positions packed (i<<16)|j with i <= j, sorted by
 *            (id, i, j).   Any output may be NULL. */
int drsdp_export_index_map(drsdp_ctx *ctx, int32_t *amap, int64_t *seg_ptr, uint32_t *seg_pos);

/* ---------------------------------------------------------------------------------------------
 * Solver parameters (Alg. 2 inputs P:319 and the constants the paper leaves open; defaults and
 * the reading of each are listed in DESIGN.md)
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  double sigma0, sigma_min, sigma_max; /* penalty: initial value and clipping range (Eq. 5.1)  */
  double gamma, tau1, tau2;            /* Eq. 5.1 constants, gamma > 1, tau2 >= tau1 > 0        */
  double tol;                          /* stop when eta_max <= tol, default 1e-8         */
  double eig_neg_tol;                  /* escape if lambda < -eig_neg_tol (1 + |lambda_max|)     */
  double rank_tol;                     /* rank reduction: keep singular values >= rank_tol_k*max,
                                          rank_tol_k = min(rank_tol, max(1e-8, 0.01 sqrt(eta))) (R32) */
  double eps_scale, eps_floor;         /* inner tolerance eps_k = max(0.1 min(1,eta) eps_scale, eps_floor) on ||XY|| */
  double time_limit_s;                 /* 0 = none                                                */
  int32_t p0;                          /* initial factorization size                      */
  int32_t max_outer, max_rtr, max_tcg; /* iteration caps (max_tcg: truncated-CG cap, default 100,
                                          <= 0: the manifold dimension n(p-1); reading R33)       */
  int32_t escape_max;                  /* at most this many escape eigenvectors per iteration     */
  int32_t mode;                        /* 0 = y-eliminated ALM subproblem (default), 1 = fixed-M  */
  uint64_t seed;                       /* Y^0 draw when no initial factor is given                */
  double rho_reg;                      /* trust-region ratio regularisation: max(1,|f|) eps rho_reg (R12) */
  int32_t stall_rtr;                   /* stagnation: stop RTR when ||grad|| has not halved within
                                          stall_rtr iterations and is within stall_factor x the
                                          inner tolerance (0 = never; reading R30)                       */
  int32_t eig_method;                  /* eigen step (eta_d, escape directions): 0 = auto (block
                                          Lanczos for n >= 16384, dense dsyevd below), 1 = dense dsyevd
                                          every outer iteration, 2 = block Lanczos always. With
                                          Lanczos, convergence (eta_max <= tol) is confirmed by one dense
                                          decomposition before the solve returns OK                    */
  double precond_mu;                   /* truncated-CG preconditioner Prec(R) = P_Y(R W),
                                          W = gbar (Y^T Y + mu gbar I)^{-1}, gbar = tr(Y^T Y)/p
                                          (reading R35); 0 = unpreconditioned; < 0 (default) =
                                          auto: mu = 0.1 for 2048 <= n < 8192, none otherwise              */
  int32_t lanczos_steps;               /* block-Lanczos steps per eigen step (block 16), 0 = 40   */
  int32_t hold_max;                    /* multiplier hold (reading R40): at most this many consecutive
                                          outer iterations may keep X~ (0 = never hold)               */
  double escape_gate;                  /* escape / rank change only when the inner solve ended with
                                          ||grad|| <= escape_gate x its tolerance (reading R36);
                                          0 = always                                               */
  double stall_factor;                 /* the stagnation exit (stall_rtr) applies only within
                                          stall_factor x the inner tolerance (reading R30; default 100) */
  double hold_tau;                     /* multiplier hold (reading R40, the subproblem stopping rule
                                          lambda_min(X^{k+1}) >= -tau_k of Thm 5.3): when
                                          eta_d(X^{k+1}) > hold_tau min(1, eta_p) and X^{k+1} has escape
                                          directions, the X~ update is undone, sigma kept, and the
                                          same subproblem is re-solved from the escaped point; 0 = off */
  double sigma_boost;                  /* penalty boost (reading R41; Alg. 1 step 8 "certain policy",
                                          P:190): when eta_d <= sigma_boost * eta_p the dual side is
                                          ahead of the primal one and sigma_{k+1} = min(gamma sigma_k,
                                          sigma_max) whatever Eq. 5.1 says; 0 = off (Eq. 5.1 alone)  */
} drsdp_params;

int drsdp_default_params(drsdp_params *out);
int drsdp_set_params(drsdp_ctx *ctx, const drsdp_params *prm);

/* Optional starting factor Y^0 (HOST, n*p row-major, rows are normalised by the library).
 * Alg. 2 writes Y^0 = 0, which is not a manifold point; without this call the library
 * draws Gaussian rows from params.seed (reading R1). */
int drsdp_set_initial_factor(drsdp_ctx *ctx, int32_t p, const double *Y0);

/* ---------------------------------------------------------------------------------------------
 * Solve (Algorithm 2, ManiDSDP)
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t status, outer_iters, p_final, p_max;
  int64_t rtr_iters, tcg_iters, n_costgrad, n_hvp;
  double eta_p, eta_d, eta_g;            /* KKT residues (eta_g reading R7)          */
  double dual_obj;                       /* b^T y                                                */
  double primal_obj;                     /* <C, X + Diag z> + 1^T z  (PSDP objective)      */
  double seconds;                        /* wall time of drsdp_solve                             */
} drsdp_info;

/* Runs Algorithm 2 to eta_max <= tol. Returns OK or ERR_NOT_CONVERGED (info filled either way).
 * Synchronous: it orders itself after the work already queued on the context stream, runs on a
 * private stream (the inner truncated CG is a captured CUDA graph), and returns when done.
 * Environment: DRSDP_VERBOSE=1 prints one diagnostic line per outer iteration to stderr. */
int drsdp_solve(drsdp_ctx *ctx, drsdp_info *info);

/* Final tuple: y (m), the factor Y of S = YY^T (n*p_final; pass NULL to skip), p_final,
 * z (n), X = X~ + D - Diag(z) (n*n). HOST outputs, caller-allocated; any may be NULL. */
int drsdp_get_solution(drsdp_ctx *ctx, double *y, double *Y, int32_t *p, double *z, double *X);

/* Per-outer-iteration trace, 13 doubles per row in the order
 * iter, eta_p, eta_d, eta_g, eta_max, primal_obj, dual_obj, sigma, p, inner_iters, cg_iters,
 * escape_delta (negative: a held multiplier, reading R40), time_s.  Copies min(max_rows, available) rows; *n_rows = rows available. */
int drsdp_get_trace(drsdp_ctx *ctx, int32_t max_rows, double *rows, int32_t *n_rows);

/* ---------------------------------------------------------------------------------------------
 * Subproblem evaluation (north-star kernels (b)+(c); bench and parity path)
 *
 * Fixed-M subproblem f(Y) = ||Y Y^T - M||_F^2 on the oblique manifold (Sub-k, with
 * M = A*(y) - C - (X~ + D)/sigma: L_sigma = (sigma/2) f + const). Outputs on the f scale:
 *   cost   f
 *   egrad  E = 4 (Y Y^T Y - M Y)                 (Euclidean gradient)
 *   rgrad  R = E - rowdot(E, Y) o Y = P_Y(E)     (Riemannian gradient, Lemma 4.1 / Eq. 4.6:
 *                                                  grad Psi = (sigma/2) R = 2 X Y)
 *   hvp    H = P_Y(4 [Z Y + (YY^T - M) U]) - rowdot(E, Y) o U,  Z = Y U^T + U Y^T
 *          (Eq. 4.7 with y frozen, times 2/sigma)
 * ------------------------------------------------------------------------------------------- */

/* Register M (DEVICE, BORROWED until the next set_subproblem_matrix or destroy): n x n symmetric,
 * row pitch ldm >= n doubles, 8-byte aligned base. Symmetry is the caller's
 * contract (not re-checked). Computes ||M||_F^2 once (one pass over M). Independent of the
 * problem set by set_problem/set_bqp. */
int drsdp_set_subproblem_matrix(drsdp_ctx *ctx, int64_t n, const double *M_dev, int64_t ldm);

/* Row-block mode for the row-sharded evaluation (one block per GPU): register rows
 * [row0, row1) of the n x n symmetric M (DEVICE, BORROWED as above, (row1 - row0) x ldm, ldm >= n
 * even, 16-byte aligned). drsdp_subproblem_eval then takes the FULL n x p Y (and U), replicated
 * on every block, and writes only the block's rows of egrad / rgrad / hvp ((row1 - row0) x p,
 * pitch p); the cost it returns is the block's additive share -2 sum_{i in block} <(MY)_i, y_i>
 * + ||M_block||_F^2 (+ ||Y^T Y||_F^2 on the block holding row 0), so the sum over the blocks of a
 * partition is f. Needs p <= 64 and the TMA product kernel (else DRSDP_ERR_INVALID_ARG). */
int drsdp_set_subproblem_rows(drsdp_ctx *ctx, int64_t n, int64_t row0, int64_t row1, const double *M_rows_dev,
                              int64_t ldm);

enum { DRSDP_EVAL_COSTGRAD = 1, DRSDP_EVAL_HVP = 2 };

/* DEVICE pointers, caller-owned, asynchronous on the ctx stream (time with CUDA events on that
 * stream; drsdp_sync to wait). Y_dev, U_dev, egrad/rgrad/hvp are n*p row-major (pitch p).
 * Y rows must have unit norm (not re-checked); U must be tangent at Y for the HVP to be the
 * Riemannian Hessian. flags: COSTGRAD computes cost/egrad/rgrad (any output pointer may be NULL);
 * HVP computes hvp and needs U_dev; HVP without COSTGRAD in the same call reuses the Gram matrix
 * and rowdot(E, Y) cached by the last COSTGRAD call at the same Y_dev and p (else ERR_STATE).
 * COSTGRAD | HVP in one call with 5 <= p <= 32 runs ONE pass over M: the product M [Y U] (2p
 * columns, TMA + DMMA) with the cost/gradient epilogue on the Y half and the Hessian-vector
 * epilogue on the U half of each row (same arithmetic as two separate calls; M is streamed once
 * instead of twice). 1 <= p <= DRSDP_MAX_P. */
int drsdp_subproblem_eval(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *Y_dev,
                          const double *U_dev, double *cost_dev, double *egrad_dev,
                          double *rgrad_dev, double *hvp_dev);

/* Same evaluation from HOST buffers (copies in and out inside the call; synchronous).
 * cost, egrad, rgrad, hvp may be NULL. Used for the end-to-end (host<->device) measurement. */
int drsdp_subproblem_eval_host(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *Y,
                               const double *U, double *cost, double *egrad, double *rgrad,
                               double *hvp);

/* ---------------------------------------------------------------------------------------------
 * ADMM-state operator kernels (north-star (a) and (d)); DEVICE pointers, asynchronous.
 * They use the problem set by set_problem / set_bqp.
 * ------------------------------------------------------------------------------------------- */

/* (a) M assembly: M = A*(y) - C - T / sigma (n x ld_out, DEVICE); y (m), T (n x ldt) DEVICE. */
int drsdp_assemble_M(drsdp_ctx *ctx, const double *y_dev, const double *T_dev, int64_t ldt,
                     double sigma, double *M_dev, int64_t ldm);

/* (d) y-update (Lemma 3.1, P:116 / Alg. 2 step 5): y = (AA*)^{-1} A(Y Y^T + C),
 * a deterministic segmented sum over the index map. Y (n x p, pitch p), y_out (m), DEVICE. */
int drsdp_y_update(drsdp_ctx *ctx, int32_t p, const double *Y_dev, double *y_dev);

/* (d) dual update (Alg. 2 steps 6-8): T <- T - sigma (A*(y) - Y Y^T - C) in place,
 * z = rowdot(T Y, Y). Scalars (DEVICE, 4 doubles): [||A*(y) - S - C||_F, b^T y,
 * <C,T> + 1^T z (PSDP objective), ||T||_F^2]. */
int drsdp_dual_update(drsdp_ctx *ctx, int32_t p, const double *Y_dev, const double *y_dev,
                      double sigma, double *T_dev, int64_t ldt, double *z_dev,
                      double *scalars_dev);

/* y-eliminated (ALM) subproblem f^(Y) = ||Y Y^T + C + T/sigma||^2 - sum_a A(YY^T + C)_a^2/cnt_a
 * and its derivatives (gradient 4 (S - M(S)) Y, HVP with the projection term of Eq. 4.7).
 * DEVICE pointers; T (n x ldt). Same flags / outputs as drsdp_subproblem_eval. */
int drsdp_alm_eval(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *T_dev, int64_t ldt,
                   double sigma, const double *Y_dev, const double *U_dev, double *cost_dev,
                   double *egrad_dev, double *rgrad_dev, double *hvp_dev);

/* Extreme eigenpairs of X = T - Diag(z) (Alg. 2 step 9 and eta_d) by block Lanczos
 * with full re-orthogonalisation (block 16, at most `steps` blocks, basis capped at n): the
 * partial eigendecomposition P:342 allows. DEVICE inputs T (n x ldt, symmetric) and z (n) for
 * the current problem's n; V_dev (DEVICE, caller-owned, n*nvec row-major) receives the Ritz
 * vectors of the nvec smallest Ritz values; HOST outputs ritz (nvec ascending Ritz values, NaN past
 * the basis size), resid (their residual norms ||X v - theta v||, may be NULL), lam_max (largest
 * Ritz value, may be NULL) and basis (basis size, may be NULL). Ritz values bound the extreme
 * eigenvalues from inside the spectrum. Synchronous. */
int drsdp_x_eigs(drsdp_ctx *ctx, const double *T_dev, int64_t ldt, const double *z_dev, int32_t steps, int32_t nvec,
                 double *ritz, double *lam_max, double *V_dev, double *resid, int32_t *basis);

/* Device kernel launches issued by this context since creation (for launch accounting). */
int drsdp_launch_count(drsdp_ctx *ctx, int64_t *count);

/* Live per-kernel timing of the fused product kernel (symv.cu): when enabled, CUDA events are
 * recorded on the context stream immediately before and after every launch. enable != 0 starts
 * (and resets) the collection, 0 stops it. */
int drsdp_profile_enable(drsdp_ctx *ctx, int enable);

/* Total device milliseconds and launch count of the product kernel since profile_enable, for
 * kind 0 = all launches, 1 = COSTGRAD epilogue, 2 = HVP epilogue, 3 = other (RAW/ROWDOT),
 * 4 = fused COSTGRAD + HVP (one pass over M, drsdp_subproblem_eval with both flags, 5 <= p <= 32).
 * Synchronizes the context stream. */
int drsdp_profile_read(drsdp_ctx *ctx, int32_t kind, double *ms, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* DRSDP_H */
