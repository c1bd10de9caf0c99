// lanczos.cuh — block Lanczos for extreme eigenpairs of X = T - Diag(z) (lanczos.cu).
#pragma once
#include <cusolverDn.h>
#include <stdint.h>

#include <vector>

#include "ctx.h"

namespace drsdp {

struct LanczosWork {
  int64_t n = 0, ldq = 0;
  int b = 0, kmax = 0;
  DBuf<double> Q;        // n x ldq basis, ldq = b (kmax + 1)
  DBuf<double> W, P;     // n x b residual block / scratch
  DBuf<double> Cc;       // ldq x b projection coefficients
  DBuf<double> Hm, Hw;   // projected matrix (m x m) and its eigenvalues
  DBuf<double> Sx;       // small right factors (b x b, or m x nvec Ritz coefficients)
  DBuf<double> V;        // n x nvec Ritz vectors (row-major, pitch nvec)
  DBuf<double> work;     // cuSOLVER workspace
  DBuf<int> info;
  int ensure(int64_t n, int b, int kmax);  // 0 or a cudaError_t
  void release();
};

struct LanczosResult {
  double lam_min = 0.0, lam_max = 0.0;  // smallest / largest Ritz values
  std::vector<double> theta;            // all Ritz values, ascending
  std::vector<double> resid;            // residual norms of the lowest nvec Ritz pairs
  int basis = 0, steps = 0;
};

// Block Lanczos with full re-orthogonalisation on X = T - Diag(z) (n = L.n, block L.b, at most
// L.kmax steps, basis capped at n). On return L.V holds the Ritz vectors of the nvec smallest Ritz
// values (n x nvec, row-major). Runs on ctx->stream; synchronises a few times per step.
int lanczos_extreme(drsdp_ctx *ctx, LanczosWork &L, cusolverDnHandle_t sol, const double *T, int64_t ldt,
                    const double *z, int nvec, uint64_t seed, LanczosResult &res);

}  // namespace drsdp
