// kernels.cuh — launchers of the operator and vector kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace drsdp {

struct GramArgs {
  int n = 0, p = 0;
  const double *Y = nullptr;
  int ldy = 0;
  const double *U = nullptr;  // optional: K = U^T Y + Y^T U
  int ldu = 0;
  double *part = nullptr;  // >= max_blocks * 2 p^2
  unsigned *counter = nullptr;
  double *G = nullptr, *K = nullptr, *gg = nullptr;
  int max_blocks = 296;
  const int *skip = nullptr;  // device flag: kernel is a no-op when set
};
cudaError_t gram_launch(const GramArgs &a, cudaStream_t st);

struct SegArgs {
  int64_t m = 0;
  const int64_t *seg_ptr = nullptr;
  const uint32_t *seg_pos = nullptr;
  const int32_t *cnt = nullptr;
  const uint8_t *is_large = nullptr;
  const int32_t *large_ids = nullptr;  // 33..256 upper positions: one warp each
  int64_t n_large = 0;
  const int32_t *huge_ids = nullptr;   // > 256 upper positions: one block each
  int64_t n_huge = 0;
  const double *cA = nullptr;  // A(C) or nullptr
  const double *Y = nullptr, *U = nullptr;
  int ld = 0, p = 0;
  double *out = nullptr;
  double *part = nullptr;
  unsigned *counter = nullptr;
  double *scal_out = nullptr;  // MODE_Y: sum_a A(S+C)_a^2 / cnt_a
  int nb_small = 0, nb_large = 0;
  const int *skip = nullptr;  // device flag: kernel is a no-op when set
  // dense mode (gram_tile.cu): the position value is D[i][j] (upper triangle, pitch ldd) instead
  // of the p-length dot products; D = Y Y^T (MODE_Y) or Y U^T + U Y^T (MODE_Z)
  const double *D = nullptr;
  int64_t ldd = 0;
  int nbk = 0;  // block problems: D stacked with blocks of nbk rows (blocks.cuh)
};
cudaError_t segsum_launch(const SegArgs &a, bool zmode, cudaStream_t st);
int segsum_blocks(int64_t m, int64_t n_large, int64_t n_huge);

struct AssembleArgs {
  int n = 0;
  const int32_t *amap = nullptr;
  int64_t ldmap = 0;
  const double *y = nullptr, *C = nullptr;
  int64_t ldc = 0;
  const double *T = nullptr;
  int64_t ldt = 0;
  double sigma = 1.0;
  double *M = nullptr;
  int64_t ldm = 0;
  double *part = nullptr;
  unsigned *counter = nullptr;
  double *scal_out = nullptr;
  int blocks = 1184;
};
cudaError_t assemble_launch(const AssembleArgs &a, cudaStream_t st);
// tiled ALM assembly: M(S) plus [sum R^2, <T, S + C>, ||T||^2] in scal_out (3 doubles)
// D (optional): dense S = Y Y^T upper triangle (pitch ldd) read instead of recomputing S tiles
cudaError_t assemble_alm_launch(const AssembleArgs &a, int p, const double *Y, int ldy, cudaStream_t st,
                                const double *D = nullptr, int64_t ldd = 0);
cudaError_t alm_cost_launch(const double *s, double sigma, double *cost, cudaStream_t st);
inline int assemble_alm_blocks(int n) { return ((n + 31) / 32) * ((n + 31) / 32); }

struct DualArgs {
  int n = 0, p = 0;
  const double *Y = nullptr;
  int ldy = 0;
  const int32_t *amap = nullptr;
  int64_t ldmap = 0;
  const double *y = nullptr, *C = nullptr;
  int64_t ldc = 0;
  double sigma = 1.0;
  double *T = nullptr;
  int64_t ldt = 0;
  double *part = nullptr;
  unsigned *counter = nullptr;
  double *scal_out = nullptr;  // [||R||^2, ||T||^2, <C,T>]
};
cudaError_t dual_update_launch(const DualArgs &a, cudaStream_t st);
inline int dual_update_blocks(int n) { return ((n + 31) / 32) * ((n + 31) / 32); }

cudaError_t dot3_launch(int n, int p, int ld, const double *A0, const double *B0, const double *A1,
                        const double *B1, const double *A2, const double *B2, double *part, unsigned *counter,
                        double *out, cudaStream_t st);
cudaError_t retract_launch(int n, int p, int ld, const double *Y, const double *V, double t, double *out,
                           int *flag, cudaStream_t st);
cudaError_t newdir_launch(int n, int p, int ld, const double *Y, const double *r, double beta, double *d,
                          double *part, unsigned *counter, double *dots, cudaStream_t st);
cudaError_t repack_launch(int n, int p_in, int ldi, const double *in, int p_out, int ldo, double *out, int vcol0,
                          int dv, const double *Vcols, int64_t ldv_col, cudaStream_t st);
cudaError_t make_x_launch(int n, const double *T, int64_t ldt, const double *z, double *X, cudaStream_t st);
cudaError_t vdot_launch(int64_t len, const double *a, const double *b, double *part, unsigned *counter,
                        double *out, cudaStream_t st);
cudaError_t init_d_launch(int n, const int32_t *amap, int64_t ldmap, const double *b, const int32_t *cnt,
                          double *T, int64_t ldt, cudaStream_t st);
cudaError_t fro2_rows_launch(int64_t rows, int64_t cols, const double *M, int64_t ld, double *part, unsigned *counter,
                             double *out, cudaStream_t st);
cudaError_t fro2_launch(int n, const double *M, int64_t ld, double *part, unsigned *counter, double *out,
                        cudaStream_t st);
cudaError_t combine_launch(const double *a, double s0, const double *b, double s1, double c, double *out,
                           cudaStream_t st);
cudaError_t rowepi_costgrad_launch(int n, int p, const double *P, int ldp, const double *W, int ldw,
                                   const double *Y, int ldy, double *R, int ldr, double *E, int lde, double *rho_out,
                                   double *part, unsigned *counter, double *scal_out, const double *gg,
                                   const double *extra, double *cost_out, cudaStream_t st);
cudaError_t rowepi_hvp_launch(int n, int p, const double *Q, int ldq, const double *W, int ldw, const double *Y,
                              int ldy, const double *U, int ldu, const double *rho, double *H, int ldh, double *part,
                              unsigned *counter, double *scal_out, const int *skip, cudaStream_t st);

// ---- device-resident truncated CG (Steihaug-Toint; oracle/rtr.py tcg) ----------------------
// The scalar recurrences live in device memory; every kernel of an iteration is a no-op once
// `done` is set, so the host launches batches of iterations and synchronises once per batch.
struct TcgDev {
  double r_r, norm_r0, e_Pe, e_Pd, d_Pd, model, Delta2, alpha, beta, e_Pe_new;
  int done;      // 0 running, 1 finished, 2 non-finite curvature
  int hit;       // stopped on the trust-region boundary
  int iters;     // Hessian-vector products used
  int par;       // which of the ping-pong buffers (0/1) holds eta, H eta, r
  int boundary;  // this iteration steps to the boundary
  int max_iters;
  int prec;      // preconditioned (reading R35): alpha, beta from z_r = <Prec(r), r>
  double z_r;
};
cudaError_t tcg_init_launch(TcgDev *st, double gnorm, double Delta, int max_iters, int prec, cudaStream_t s);
// after H delta: kappa = <delta, H delta> (device scalar) -> alpha or the boundary step tau;
// eta' = eta + alpha delta, (H eta)' = H eta + alpha H delta, r' = r + alpha H delta, then the
// model / residual decisions (last block); use_cond: also set the graph's WHILE condition
cudaError_t tcg_update_launch(int n, int p, int ld, TcgDev *st, double *e0, double *e1, double *h0, double *h1,
                              double *r, const double *d, const double *hd, const double *g, double *part,
                              unsigned *counter, const double *kappa, cudaGraphConditionalHandle cond, int use_cond,
                              cudaStream_t s);
// move the result into buffer 0 (eta, H eta) when it ended in buffer 1
cudaError_t tcg_finalize_launch(int n, int p, int ld, const TcgDev *st, double *e0, const double *e1, double *h0,
                                const double *h1, cudaStream_t s);
// delta = P_Y(-src + beta delta) in place (src = r, or z = Prec(r) when preconditioned)
cudaError_t tcg_newdir_launch(int n, int p, int ld, const TcgDev *st, const double *Y, const double *src, double *d,
                              cudaStream_t s);
// preconditioned tCG (reading R35): z (= r W on entry) <- P_Y(z), z_r = <z, r>; init: delta = -z,
// else beta and the e_Pd / d_Pd recurrences (see kernels.cu)
cudaError_t tcg_prec_launch(int n, int p, int ld, TcgDev *st, const double *Y, double *z, const double *r, double *d,
                            double *part, unsigned *counter, int init, cudaStream_t s);
// A = G / gbar + mu I, B = I (gbar = tr(G)/p): inputs of the Cholesky solve giving W = A^{-1}
cudaError_t tcg_prec_matrix_launch(int p, const double *G, double mu, double *A, double *B, cudaStream_t s);
cudaError_t rowdot_launch(int n, int p, const double *P, int ldp, const double *Y, int ldy, double *z, double *part,
                          unsigned *counter, double *out, cudaStream_t st);
cudaError_t normalize_rows_launch(int n, int r, int ld, double *X, cudaStream_t st);
cudaError_t gather_assemble_launch(int n, const int32_t *amap, int64_t ldmap, const double *w, double *W, int64_t ldw,
                                   const int *skip, cudaStream_t st);
inline int rows_blocks(int64_t n) { return (int)((n + 7) / 8); }

}  // namespace drsdp
