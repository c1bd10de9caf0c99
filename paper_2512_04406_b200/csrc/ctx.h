// ctx.h — the drsdp_ctx object behind the C ABI (host side).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/drsdp.h"

namespace drsdp {

// Process-wide allocation epoch: bumped whenever a DBuf (re)allocates or frees device memory.
// A captured CUDA graph bakes in every device address it touches, so a graph captured at an
// older epoch may reference freed memory and must be re-captured (solver.cu, Graph::epoch).
inline uint64_t &dbuf_epoch() {
  static uint64_t e = 0;
  return e;
}

// device buffer with grow-on-demand (no destructor: ownership is explicit, release() frees)
template <typename T>
struct DBuf {
  T *ptr = nullptr;
  size_t cap = 0;  // elements
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    ++dbuf_epoch();
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&ptr, (n ? n : 1) * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
  }
  // grow and zero-fill on (re)allocation (counters must start at zero)
  cudaError_t ensure_zeroed(size_t n) {
    if (n <= cap) return cudaSuccess;
    cudaError_t e = ensure(n);
    if (e != cudaSuccess) return e;
    return cudaMemset(ptr, 0, cap * sizeof(T));
  }
  void release() {
    if (ptr) ++dbuf_epoch();
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

// scalar slots in ctx->d_scal (device) / ctx->h_scal (pinned host mirror)
enum Slot {
  S_COST = 0,      // cost (subproblem eval)
  S_SCAL = 2,      // 2: symv scalars (s1, ||R||^2) / (<U,H>, -)
  S_GG = 4,        // ||G||^2
  S_EXTRA = 6,     // 2: constant cost terms
  S_MM = 8,        // ||M||^2 of the borrowed fixed M
  S_SEGSQ = 10,    // sum_a A(S+C)_a^2 / cnt_a
  S_M0 = 11,       // ||C + T/sigma||^2
  S_DOTS = 12,     // 4: vector dots
  S_DUAL = 16,     // 3: ||R||^2, ||T||^2, <C,T>
  S_ZSUM = 20,     // 2: sum z
  S_BY = 22,       // 2: b^T y, ||y||^2
  S_YCA = 24,      // 2: yS . cA
  S_ALM = 26,      // 3: ALM assembly sums [sum R^2, <T, S+C>, ||T||^2]
  S_UH = 29,       // <U, H> of a fused cost+grad+HVP evaluation (EPI_BOTH)
  S_FLAG = 30,     // retraction flag (int stored in a double slot)
  S_ZERO = 31,     // constant 0 (row-block cost: ||G||^2 counted once)
  S_TOTAL = 64
};

enum Counter { C_GRAM = 0, C_SEG, C_ASM, C_DUAL, C_VEC, C_SYMV, C_FRO, C_DOT, C_TOTAL };

struct Problem {
  int64_t n = 0, m = 0, ld = 0, n_upper = 0;
  // multi-block problem (blocks.cuh): nblk blocks of nb rows, n = nblk * nb rows of
  // the factor; h_amap / amap / T / M are stacked (row r at r * nb / r * ld, nb columns).
  // nblk = 0: one dense n x n block.
  int64_t nblk = 0, nb = 0;
  bool has_C = false;
  std::vector<int32_t> h_amap;  // n*n (dense; -1 = unconstrained) or n*nb (blocks)
  std::vector<int64_t> h_seg_ptr;
  std::vector<uint32_t> h_seg_pos;
  std::vector<int32_t> h_cnt;
  std::vector<double> h_b;
  DBuf<int32_t> amap;  // n x ld
  DBuf<double> C;      // n x ld (if has_C)
  DBuf<double> cA;     // A(C) (if has_C)
  DBuf<int32_t> cnt;
  DBuf<double> b;
  DBuf<int64_t> seg_ptr;
  DBuf<uint32_t> seg_pos;
  DBuf<uint8_t> is_large;
  DBuf<int32_t> large_ids, huge_ids;
  int64_t n_large = 0, n_huge = 0;
  void release() {
    amap.release();
    C.release();
    cA.release();
    cnt.release();
    b.release();
    seg_ptr.release();
    seg_pos.release();
    is_large.release();
    large_ids.release();
    huge_ids.release();
  }
};

struct SolverState;

}  // namespace drsdp

struct drsdp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t aux_stream = nullptr;  // concurrent branch inside an evaluation (K next to Z)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string err;
  int sticky = 0;
  int64_t launches = 0;
  int num_sms = 148;

  drsdp::Problem prob;
  bool has_problem = false;
  drsdp_params prm{};

  // shared workspaces
  drsdp::DBuf<double> red_part;  // grid_sum partials
  drsdp::DBuf<double> gram_part;
  drsdp::DBuf<double> symv_part;
  drsdp::DBuf<double> big_P, big_W;
  drsdp::DBuf<double> vt_buf;  // V^T staging for the TMA product kernel
  drsdp::DBuf<double> w_dense;  // A*(w) assembled for the TMA gather-product
  // symmetric-half product (symv_symm.cu): unit table for symm_n, partial buffers
  int symm_n = 0, symm_nunits = 0;
  drsdp::DBuf<int4> symm_units;
  drsdp::DBuf<int> symm_ustart;
  drsdp::DBuf<double> symm_F, symm_T;
  const int *skip_flag = nullptr;  // set while device-resident tCG batches are being launched  // generic-p (> 64) product outputs, n x ldv
  drsdp::DBuf<unsigned> tile_cnt;
  drsdp::DBuf<double> tile_scal;
  unsigned *counters = nullptr;  // C_TOTAL
  double *d_scal = nullptr;      // S_TOTAL
  double *h_scal = nullptr;      // pinned mirror
  int *d_flag = nullptr;

  // fixed-M subproblem (borrowed)
  const double *sub_M = nullptr;
  int64_t sub_n = 0, sub_ldm = 0;
  bool sub_rows_mode = false;  // drsdp_set_subproblem_rows: sub_M holds rows [sub_row0, + sub_nloc)
  int64_t sub_row0 = 0, sub_nloc = 0;
  drsdp::DBuf<double> sub_G, sub_K, sub_rho;  // fixed-M eval cache (drsdp_subproblem_eval only)
  drsdp::DBuf<double> g_scratch;              // G recomputed as a by-product of K inside HVPs
  const double *sub_cached_Y = nullptr;
  int sub_cached_p = 0;
  bool sub_cached_valid = false;
  // ALM eval cache (ABI drsdp_alm_eval)
  drsdp::DBuf<double> alm_M, alm_yS, alm_wZ, alm_D, alm_Z;
  drsdp::DBuf<double> alm_G, alm_K, alm_rho;  // ALM eval cache (separate from the fixed-M one)
  const double *alm_cached_Y = nullptr;
  const double *alm_cached_T = nullptr;
  int alm_cached_p = 0;
  double alm_cached_sigma = 0.0;
  bool alm_cached_valid = false;

  // initial factor
  std::vector<double> h_Y0;
  int p0_given = 0;

  // live kernel timing (drsdp_profile_*)
  bool prof_on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  std::vector<int> prof_kind;
  size_t prof_used = 0;

  // host-entry staging buffers
  drsdp::DBuf<double> host_stage;

  // solver
  drsdp::SolverState *solver = nullptr;
  std::vector<double> trace;  // 13 per row
};

namespace drsdp {
// helpers shared by abi.cu and solver.cu
int set_error(drsdp_ctx *ctx, int code, const std::string &msg);
int cuda_check(drsdp_ctx *ctx, cudaError_t e, const char *what);
int ensure_workspace(drsdp_ctx *ctx, int64_t n, int p);
int choose_splits(drsdp_ctx *ctx, int krows, int ntiles);
struct SymvArgs;
int run_product(drsdp_ctx *ctx, SymvArgs &a, int epi, int mode2, bool atr, int prof_kind);
int rowdot_product(drsdp_ctx *ctx, int n, int p, const double *T, int64_t ldt, const double *Y, int ldv, double *z,
                   double *zsum);
// out (n x p, pitch ldo) = A (n x p, pitch lda) B (p x p, pitch p)
int right_product(drsdp_ctx *ctx, int n, int p, const double *A, int lda, const double *B, double *out, int ldo);
int apply_w_product(drsdp_ctx *ctx, int n, int p, const double *Y, int ldv, const double *W, int r, double *out,
                    int ldo);
// fused subproblem evaluations on device pointers (pitch ldv for all n x p arrays)
int eval_fixed(drsdp_ctx *ctx, int flags, int n, int p, const double *M, int64_t ldm, const double *Y, int ldv,
               const double *U, double *cost, double *egrad, double *rgrad, double *hvp, double *G, double *K,
               double *rho, const double *cost_extra_dev, bool have_gram);
// Dbuf / Zbuf (n x ld, optional): dense S / Z for the tensor-core segmented sums (gram_tile.cu)
int alm_costgrad(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, double sigma, const double *Y, int ldv,
                 double *Mout, int64_t ldm, double *yS, double *G, double *rho, double *cost, double *egrad,
                 double *rgrad, double *Dbuf);
int alm_hvp(drsdp_ctx *ctx, int p, const double *M, int64_t ldm, const double *Y, int ldv, const double *U,
            const double *G, double *K, const double *rho, double *wZ, double *hvp, double *Zbuf);
int read_scalars(drsdp_ctx *ctx, int first, int count);
// multi-block problems (blocks.cu): z = rowdot(T Y, Y) per block and the per-block dual update
int blk_rowdot(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, const double *Y, int ldv, double *z, double *zsum);
int blk_dual(drsdp_ctx *ctx, int p, const double *Y, int ldv, const double *y, double sigma, double *T, int64_t ldt);
void free_solver(drsdp_ctx *ctx);
}  // namespace drsdp
