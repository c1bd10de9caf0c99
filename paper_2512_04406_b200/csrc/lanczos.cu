// lanczos.cu — extreme eigenpairs of X = T - Diag(z) by block Lanczos (Alg. 2 step 9 / eta_d,
// PAPER.md P:329, "a partial eigenvalue decomposition ... when the full eigenvalue
// decomposition is too expensive").
//
// Block Lanczos with full re-orthogonalisation ("twice is enough") on the n x (k b) basis Q:
//   W = X Q_j = T Q_j - z o Q_j          (T streamed once per step by the fp64 product kernel)
//   W -= Q_{0..j} (Q_{0..j}^T W)          (two passes; the first pass's coefficients for block j
//                                          and j-1 are the block-tridiagonal A_j and B_j^T)
//   W = Q_{j+1} B_{j+1}                  (Cholesky QR, twice)
// and a Rayleigh-Ritz step on the block-tridiagonal projection H = Q^T X Q (k b x k b, cuSOLVER
// dsyevd on the small matrix). Ritz values are upper bounds of the smallest eigenvalues (and
// lower bounds of the largest); the residual of Ritz pair (theta, Q s) is ||B_{k+1} s_last||.
// The solver (solver.cu) uses the Ritz values for lambda_min / lambda_max and the Ritz vectors
// below the escape threshold as saddle-escape directions, and confirms convergence with a full
// dense decomposition (the certificate eta_d <= tol is never taken from Ritz values alone).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "lanczos.cuh"
#include "symv.cuh"

namespace drsdp {

namespace {

// W (n x b, pitch b) -= z o Qj (pitch ldq)
__global__ void __launch_bounds__(256) diag_sub_kernel(int n, int b, const double *__restrict__ z,
                                                       const double *__restrict__ Qj, int64_t ldq, double *W) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * b) return;
  const int64_t i = e / b, c = e - i * b;
  W[e] -= z[i] * Qj[i * ldq + c];
}

// W (n x b, pitch b) -= P (pitch b)
__global__ void __launch_bounds__(256) sub_kernel(int64_t len, double *W, const double *__restrict__ P) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < len) W[e] -= P[e];
}

// deterministic Gaussian start block (splitmix64 + Box-Muller per element), pitch ldq
__global__ void __launch_bounds__(256) start_kernel(int n, int b, uint64_t seed, double *Q, int64_t ldq) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * b) return;
  const int64_t i = e / b, c = e - i * b;
  auto mix = [](uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  const uint64_t k = seed * 0x9E3779B97F4A7C15ull + (uint64_t)e * 2ull + 1ull;
  const double u1 = ((mix(k) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  const double u2 = ((mix(k + 0x632BE59BD9B4E019ull) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  Q[i * ldq + c] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

}  // namespace

static int lz_check(drsdp_ctx *ctx, cudaError_t e, const char *what) { return cuda_check(ctx, e, what); }

#define LCK(call, what)                     \
  do {                                      \
    int _rc = lz_check(ctx, (call), what);  \
    if (_rc) return _rc;                    \
  } while (0)
#define LKL(call, what)                     \
  do {                                      \
    ctx->launches++;                        \
    int _rc = lz_check(ctx, (call), what);  \
    if (_rc) return _rc;                    \
  } while (0)
#define LRC(call)         \
  do {                    \
    int _rc = (call);     \
    if (_rc) return _rc;  \
  } while (0)

// C (m1 x b, pitch b) = A^T W with A n x m1 (pitch lda), W n x b (pitch b)
static int gemm_tn(drsdp_ctx *ctx, int n, int m1, int b, const double *A, int64_t lda, const double *W, double *C) {
  SymvArgs a;
  a.A = A;
  a.lda = lda;
  a.n = m1;
  a.k = n;
  a.p = b;
  a.V = W;
  a.ldv = b;
  a.out = C;
  a.ldo = b;
  return run_product(ctx, a, EPI_RAW, MODE2_NONE, false, 0);
}
// out (n x b, pitch ldo) = A C with A n x m1 (pitch lda), C m1 x b (pitch b)
static int gemm_nn(drsdp_ctx *ctx, int n, int m1, int b, const double *A, int64_t lda, const double *Cm, double *out,
                   int64_t ldo) {
  SymvArgs a;
  a.A = A;
  a.lda = lda;
  a.n = n;
  a.k = m1;
  a.p = b;
  a.V = Cm;
  a.ldv = b;
  a.out = out;
  a.ldo = (int)ldo;
  return run_product(ctx, a, EPI_RAW, MODE2_NONE, true, 0);
}

// Upper Cholesky factor R of the b x b Gram matrix (row-major), R^T R = G. Returns the number of
// leading pivots above tol * max diag (rank; < b means the block is (numerically) dependent).
static int chol_upper(const std::vector<double> &G, int b, std::vector<double> &R, double rel_tol) {
  R.assign((size_t)b * b, 0.0);
  double dmax = 0.0;
  for (int i = 0; i < b; ++i) dmax = std::max(dmax, G[(size_t)i * b + i]);
  if (!(dmax > 0.0)) return 0;
  for (int i = 0; i < b; ++i) {
    double s = G[(size_t)i * b + i];
    for (int k = 0; k < i; ++k) s -= R[(size_t)k * b + i] * R[(size_t)k * b + i];
    if (!(s > rel_tol * dmax)) return i;
    const double rii = std::sqrt(s);
    R[(size_t)i * b + i] = rii;
    for (int j = i + 1; j < b; ++j) {
      double t = G[(size_t)i * b + j];
      for (int k = 0; k < i; ++k) t -= R[(size_t)k * b + i] * R[(size_t)k * b + j];
      R[(size_t)i * b + j] = t / rii;
    }
  }
  return b;
}

// inverse of an upper-triangular b x b matrix (row-major)
static void inv_upper(const std::vector<double> &R, int b, std::vector<double> &Ri) {
  Ri.assign((size_t)b * b, 0.0);
  for (int j = 0; j < b; ++j) {
    Ri[(size_t)j * b + j] = 1.0 / R[(size_t)j * b + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += R[(size_t)i * b + k] * Ri[(size_t)k * b + j];
      Ri[(size_t)i * b + j] = -s / R[(size_t)i * b + i];
    }
  }
}

int LanczosWork::ensure(int64_t n_, int b_, int kmax_) {
  n = n_;
  b = b_;
  kmax = kmax_;
  ldq = (int64_t)b * (kmax + 1);
  cudaError_t e;
  if ((e = Q.ensure((size_t)n * ldq)) != cudaSuccess) return (int)e;
  if ((e = W.ensure((size_t)n * b)) != cudaSuccess) return (int)e;
  if ((e = P.ensure((size_t)n * b)) != cudaSuccess) return (int)e;
  if ((e = Cc.ensure((size_t)ldq * b)) != cudaSuccess) return (int)e;
  if ((e = Hm.ensure((size_t)ldq * ldq)) != cudaSuccess) return (int)e;
  if ((e = Hw.ensure((size_t)ldq)) != cudaSuccess) return (int)e;
  if ((e = Sx.ensure((size_t)ldq * b)) != cudaSuccess) return (int)e;
  if ((e = info.ensure(1)) != cudaSuccess) return (int)e;
  return 0;
}

void LanczosWork::release() {
  Q.release();
  W.release();
  P.release();
  Cc.release();
  Hm.release();
  Hw.release();
  Sx.release();
  V.release();
  work.release();
  info.release();
}

// Orthonormalise W (n x b, pitch b) against itself by Cholesky QR, twice; the factor R (b x b,
// with W_in = Q R) is returned in Rout, Q written to Qout (pitch ldq). breakdown is set when the
// block is numerically rank-deficient (the Krylov space is exhausted); W is then left unchanged
// by the first pass. Returns a drsdp status.
static int cholqr2(drsdp_ctx *ctx, LanczosWork &L, double *Wd, double *Qout, std::vector<double> &Rout,
                   bool &breakdown) {
  breakdown = false;
  const int n = (int)L.n, b = L.b;
  std::vector<double> G((size_t)b * b), R1, R2, Ri;
  Rout.assign((size_t)b * b, 0.0);
  for (int pass = 0; pass < 2; ++pass) {
    LRC(gemm_tn(ctx, n, b, b, Wd, b, Wd, L.Cc.ptr));
    LCK(cudaMemcpyAsync(G.data(), L.Cc.ptr, sizeof(double) * b * b, cudaMemcpyDeviceToHost, ctx->stream), "read");
    LCK(cudaStreamSynchronize(ctx->stream), "sync");
    for (int i = 0; i < b; ++i)
      for (int j = i + 1; j < b; ++j) G[(size_t)i * b + j] = G[(size_t)j * b + i] = 0.5 * (G[(size_t)i * b + j] + G[(size_t)j * b + i]);
    std::vector<double> &R = pass == 0 ? R1 : R2;
    const int rk = chol_upper(G, b, R, pass == 0 ? 1e-24 : 1e-12);
    if (rk < b) {
      breakdown = true;
      return DRSDP_OK;
    }
    inv_upper(R, b, Ri);
    LCK(cudaMemcpyAsync(L.Sx.ptr, Ri.data(), sizeof(double) * b * b, cudaMemcpyHostToDevice, ctx->stream), "copy");
    double *dst = pass == 0 ? L.P.ptr : Qout;
    const int64_t ldd = pass == 0 ? b : L.ldq;
    LRC(gemm_nn(ctx, n, b, b, Wd, b, L.Sx.ptr, dst, ldd));
    if (pass == 0) {
      LCK(cudaMemcpyAsync(Wd, L.P.ptr, sizeof(double) * n * b, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    }
  }
  // R = R2 R1
  for (int i = 0; i < b; ++i)
    for (int j = i; j < b; ++j) {
      double s = 0.0;
      for (int k = i; k <= j; ++k) s += R2[(size_t)i * b + k] * R1[(size_t)k * b + j];
      Rout[(size_t)i * b + j] = s;
    }
  return DRSDP_OK;
}

int lanczos_extreme(drsdp_ctx *ctx, LanczosWork &L, cusolverDnHandle_t sol, const double *T, int64_t ldt,
                    const double *z, int nvec, uint64_t seed, LanczosResult &res) {
  const int n = (int)L.n, b = L.b;
  const int kmax = L.kmax;
  res = LanczosResult();
  // start block
  LKL((start_kernel<<<(unsigned)(((int64_t)n * b + 255) / 256), 256, 0, ctx->stream>>>(n, b, seed, L.W.ptr, b),
       cudaGetLastError()),
      "lanczos start");
  std::vector<double> R;
  bool brk = false;
  LRC(cholqr2(ctx, L, L.W.ptr, L.Q.ptr, R, brk));
  if (brk) return set_error(ctx, DRSDP_ERR_NUMERIC, "lanczos: degenerate start block");
  // block tridiagonal H (ldq x ldq, row-major), built on the host
  const int64_t ldq = L.ldq;
  std::vector<double> H;
  int k = 0;  // number of blocks in the basis
  std::vector<double> Cfull, Bnext;
  for (int j = 0; j < kmax; ++j) {
    k = j + 1;
    const int m1 = k * b;
    double *Qj = L.Q.ptr + (size_t)j * b;
    // W = T Q_j - z o Q_j
    SymvArgs a;
    a.A = T;
    a.lda = ldt;
    a.n = n;
    a.p = b;
    a.V = Qj;
    a.ldv = (int)ldq;
    a.out = L.W.ptr;
    a.ldo = b;
    LRC(run_product(ctx, a, EPI_RAW, MODE2_NONE, false, 0));
    LKL((diag_sub_kernel<<<(unsigned)(((int64_t)n * b + 255) / 256), 256, 0, ctx->stream>>>(n, b, z, Qj, ldq, L.W.ptr),
         cudaGetLastError()),
        "lanczos diag");
    // two passes of W -= Q (Q^T W); the first pass's block-j coefficients are A_j = Q_j^T X Q_j
    for (int pass = 0; pass < 2; ++pass) {
      LRC(gemm_tn(ctx, n, m1, b, L.Q.ptr, ldq, L.W.ptr, L.Cc.ptr));
      if (pass == 0) {
        Cfull.resize((size_t)m1 * b);
        LCK(cudaMemcpyAsync(Cfull.data(), L.Cc.ptr, sizeof(double) * m1 * b, cudaMemcpyDeviceToHost, ctx->stream),
            "read");
      }
      LRC(gemm_nn(ctx, n, m1, b, L.Q.ptr, ldq, L.Cc.ptr, L.P.ptr, b));
      LKL((sub_kernel<<<(unsigned)(((int64_t)n * b + 255) / 256), 256, 0, ctx->stream>>>((int64_t)n * b, L.W.ptr,
                                                                                         L.P.ptr),
           cudaGetLastError()),
          "lanczos sub");
    }
    LCK(cudaStreamSynchronize(ctx->stream), "sync");
    // H block row j: A_j (symmetrised) from the first pass
    H.resize((size_t)m1 * m1, 0.0);
    {
      // grow H (row-major, m1 x m1) keeping the previous (m1 - b) x (m1 - b) block
      std::vector<double> Hn((size_t)m1 * m1, 0.0);
      const int m0 = m1 - b;
      for (int i = 0; i < m0; ++i)
        for (int c = 0; c < m0; ++c) Hn[(size_t)i * m1 + c] = H[(size_t)i * m0 + c];
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c)
          Hn[(size_t)(m0 + r) * m1 + m0 + c] =
              0.5 * (Cfull[(size_t)(m0 + r) * b + c] + Cfull[(size_t)(m0 + c) * b + r]);
      if (j > 0) {
        // off-diagonal blocks: B_j from the previous QR (Q_j B_j = residual of step j-1):
        // H[j][j-1] = B_j, H[j-1][j] = B_j^T
        for (int r = 0; r < b; ++r)
          for (int c = 0; c < b; ++c) {
            Hn[(size_t)(m0 + r) * m1 + (m0 - b) + c] = Bnext[(size_t)r * b + c];
            Hn[(size_t)(m0 - b + c) * m1 + m0 + r] = Bnext[(size_t)r * b + c];
          }
      }
      H.swap(Hn);
    }
    if (k * b + b > n || j == kmax - 1) break;  // basis would exceed n, or the step budget is spent
    LRC(cholqr2(ctx, L, L.W.ptr, L.Q.ptr + (size_t)(j + 1) * b, R, brk));
    if (brk) break;  // invariant subspace found
    Bnext = R;
  }
  const int m = k * b;
  // Rayleigh-Ritz on H (m x m): cuSOLVER dsyevd on the small projected matrix
  LCK(cudaMemcpyAsync(L.Hm.ptr, H.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, ctx->stream), "copy H");
  int lw = 0;
  if (cusolverDnDsyevd_bufferSize(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, L.Hm.ptr, m, L.Hw.ptr,
                                  &lw) != CUSOLVER_STATUS_SUCCESS)
    return set_error(ctx, DRSDP_ERR_CUDA, "lanczos: dsyevd buffer size");
  LCK(L.work.ensure((size_t)lw + 1), "alloc");
  if (cusolverDnDsyevd(sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, L.Hm.ptr, m, L.Hw.ptr, L.work.ptr, lw,
                       L.info.ptr) != CUSOLVER_STATUS_SUCCESS)
    return set_error(ctx, DRSDP_ERR_CUDA, "lanczos: dsyevd");
  ctx->launches++;
  res.theta.resize(m);
  int info = 0;
  LCK(cudaMemcpyAsync(res.theta.data(), L.Hw.ptr, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream), "read");
  LCK(cudaMemcpyAsync(&info, L.info.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read");
  std::vector<double> S((size_t)m * m);
  LCK(cudaMemcpyAsync(S.data(), L.Hm.ptr, sizeof(double) * m * m, cudaMemcpyDeviceToHost, ctx->stream), "read");
  LCK(cudaStreamSynchronize(ctx->stream), "sync");
  if (info != 0) return set_error(ctx, DRSDP_ERR_NUMERIC, "lanczos: projected eigenproblem failed");
  res.basis = m;
  res.steps = k;
  res.lam_min = res.theta[0];
  res.lam_max = res.theta[m - 1];
  // residual norms of the lowest nvec Ritz pairs: ||W_res s_last||, W_res = X Q_{k-1} residual
  // block (= Q_k B_k when the loop continued); computed from the final residual W (n x b)
  const int nv = std::min(nvec, m);
  res.resid.assign(nv, 0.0);
  if (nv > 0) {
    // Ritz vectors V = Q S[:, 0:nv] (S column-major from cuSOLVER: column c at S[c*m + i]);
    // S_sel (m x nv, row-major) for the product
    std::vector<double> Ssel((size_t)m * nv);
    for (int i = 0; i < m; ++i)
      for (int c = 0; c < nv; ++c) Ssel[(size_t)i * nv + c] = S[(size_t)c * m + i];
    LCK(L.Sx.ensure((size_t)m * nv), "alloc");
    LCK(cudaMemcpyAsync(L.Sx.ptr, Ssel.data(), sizeof(double) * m * nv, cudaMemcpyHostToDevice, ctx->stream), "copy");
    LCK(L.V.ensure((size_t)n * nv), "alloc");
    LRC(gemm_nn(ctx, n, m, nv, L.Q.ptr, ldq, L.Sx.ptr, L.V.ptr, nv));
    // residuals: ||W s_last|| with W the last (orthogonalised) residual block
    std::vector<double> Wtw((size_t)b * b);
    LRC(gemm_tn(ctx, n, b, b, L.W.ptr, b, L.W.ptr, L.Cc.ptr));
    LCK(cudaMemcpyAsync(Wtw.data(), L.Cc.ptr, sizeof(double) * b * b, cudaMemcpyDeviceToHost, ctx->stream), "read");
    LCK(cudaStreamSynchronize(ctx->stream), "sync");
    for (int c = 0; c < nv; ++c) {
      const double *sl = &S[(size_t)c * m + (m - b)];
      double q = 0.0;
      for (int r = 0; r < b; ++r)
        for (int t = 0; t < b; ++t) q += sl[r] * Wtw[(size_t)r * b + t] * sl[t];
      res.resid[c] = std::sqrt(std::max(0.0, q));
    }
  }
  return DRSDP_OK;
}

}  // namespace drsdp

// ---- ABI: extreme eigenpairs of X = T - Diag(z) for the current problem size (parity tests) ---
extern "C" int drsdp_x_eigs(drsdp_ctx *ctx, const double *T_dev, int64_t ldt, const double *z_dev, int32_t steps,
                            int32_t nvec, double *ritz, double *lam_max, double *V_dev, double *resid,
                            int32_t *basis) {
  using namespace drsdp;
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "x_eigs before set_problem");
  if (ctx->prob.nblk > 0) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "x_eigs: dense problems only");
  const int n = (int)ctx->prob.n;
  if (!T_dev || !z_dev || ldt < n || steps < 1 || nvec < 0 || nvec > n || (nvec > 0 && (!ritz || !V_dev)))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "x_eigs: bad arguments");
  cudaSetDevice(ctx->device);
  cusolverDnHandle_t sol = nullptr;
  if (cusolverDnCreate(&sol) != CUSOLVER_STATUS_SUCCESS) return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnCreate");
  cusolverDnSetStream(sol, ctx->stream);
  LanczosWork L;
  const int b = std::min(16, n);
  int rc = DRSDP_OK;
  const int e = L.ensure(n, b, std::max(1, std::min((int)steps, n / b)));
  if (e) rc = cuda_check(ctx, (cudaError_t)e, "alloc lanczos");
  LanczosResult res;
  if (!rc) rc = ensure_workspace(ctx, n, b);
  if (!rc) rc = lanczos_extreme(ctx, L, sol, T_dev, ldt, z_dev, nvec, 12345, res);
  if (!rc) {
    const int nv = std::min(nvec, res.basis);
    for (int c = 0; c < nvec; ++c) {
      if (ritz) ritz[c] = c < nv ? res.theta[c] : NAN;
      if (resid) resid[c] = c < nv ? res.resid[c] : NAN;
    }
    if (lam_max) *lam_max = res.lam_max;
    if (basis) *basis = res.basis;
    if (nv > 0) rc = cuda_check(ctx, cudaMemcpyAsync(V_dev, L.V.ptr, sizeof(double) * n * nv, cudaMemcpyDeviceToDevice,
                                                     ctx->stream), "copy V");
    if (!rc) rc = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "sync");
  }
  L.release();
  cusolverDnDestroy(sol);
  return rc;
}
