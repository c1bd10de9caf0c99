// abi.cu — extern "C" entry points of libdrsdp.so (see include/drsdp.h), problem setup and the
// device-side subproblem evaluations (fixed-M and y-eliminated ALM).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ctx.h"
#include "kernels.cuh"
#include "gram_tile.cuh"
#include "symv.cuh"
#include "blocks.cuh"

using namespace drsdp;

namespace drsdp {

int set_error(drsdp_ctx *ctx, int code, const std::string &msg) {
  if (ctx) {
    ctx->err = msg;
    if (code == DRSDP_ERR_CUDA || code == DRSDP_ERR_OOM) ctx->sticky = code;
  }
  return code;
}

int cuda_check(drsdp_ctx *ctx, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return DRSDP_OK;
  cudaGetLastError();
  const int code = (e == cudaErrorMemoryAllocation) ? DRSDP_ERR_OOM : DRSDP_ERR_CUDA;
  return set_error(ctx, code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                        \
  do {                                                        \
    int _rc = cuda_check(ctx, (call), what);                  \
    if (_rc) return _rc;                                      \
  } while (0)
#define KL(call, what)                                        \
  do {                                                        \
    ctx->launches++;                                          \
    int _rc = cuda_check(ctx, (call), what);                  \
    if (_rc) return _rc;                                      \
  } while (0)

static int prof_begin(drsdp_ctx *ctx, int kind);
static int prof_end(drsdp_ctx *ctx);

// split-K factor for a product with krows contraction rows and ntiles output tiles (all chunks):
// rows per split are a multiple of 64 (4 rows x 8 warps x unroll 2); cost model = waves x rows.
int choose_splits(drsdp_ctx *ctx, int krows, int ntiles) {
  const int slots = ctx->num_sms * 2;
  int bestS = 1;
  double best = 1e300;
  for (int S = 1; S <= 64; ++S) {
    const int per = (krows + S - 1) / S;
    const int rps = ((per + 63) / 64) * 64;
    if (S > 1 && rps < 64) break;
    if ((int64_t)(S - 1) * rps >= krows) break;  // empty splits
    const int ctas = ntiles * S;
    const int waves = (ctas + slots - 1) / slots;
    const double cost = (double)waves * (rps + 32) + 16.0 * S;
    if (cost < best * 0.999) {
      best = cost;
      bestS = S;
    }
  }
  return bestS;
}

int ensure_workspace(drsdp_ctx *ctx, int64_t n, int p) {
  (void)n;
  (void)p;
  CK(ctx->gram_part.ensure((size_t)296 * 2 * 64 * 64 + 2048), "alloc gram workspace");  // + final-kernel block partials
  return DRSDP_OK;
}

// One launch of the product kernel family (symv.cu): sizes the split-K factor, grows the split
// workspace / tile counters on demand and records the live timing events (kind 1..3) if enabled.
int run_product(drsdp_ctx *ctx, SymvArgs &a, int epi, int mode2, bool atr, int prof_kind) {
  static const bool no_tma = std::getenv("DRSDP_NO_TMA") != nullptr;
  if (a.ncols > 0 && a.ncols != a.n && (no_tma || !symv_tma_supported(a, epi, mode2, atr)))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG,
                     "row-block product needs the TMA kernel (even pitch, 16 B aligned rows, p <= 64)");
  // matrix-light gather-product (f1): A*(w) gathered inside the ring from the TMA-loaded index-map panel;
  // fused HVP epilogue for p <= 64. OFF by default (DRSDP_FUSED_GATHER=1: on, =2: also the raw column
  // chunks of p > 64): the bitwise-repeatability stress test (tests/test_gpu_parity.py
  // test_alm_hvp_bitwise_repeatable) found rare wrong tiles with the 8-gather-warp configuration at
  // p <= 16 (a race not yet located; compute-sanitizer is refused by the pool), which also made the
  // d = 70 / 80 solves nondeterministic and ~2x slower. The dense A*(w) path is bitwise repeatable.
  static const int fused_gather = [] {
    const char *e = std::getenv("DRSDP_FUSED_GATHER");
    return e ? std::atoi(e) : 0;
  }();
  if (!no_tma && fused_gather && mode2 == MODE2_GATHER && a.n >= 2048 && (epi == EPI_HVP || fused_gather >= 2) &&
      symv_gather_supported(a, epi, atr)) {
    const int pt = symv_tma_pt(a.p, epi), bm = symv_tma_rows(), bk = symv_gather_kstep();
    const int ntiles = ((a.n + bm - 1) / bm) * symv_tma_chunks(a.p, epi);
    int S = 1;
    double best = 1e300;
    for (int s = 1; s <= 64; ++s) {
      const int per = ((a.n + s - 1) / s + bk - 1) / bk * bk;
      if (s > 1 && (int64_t)(s - 1) * per >= a.n) break;
      const int waves = (ntiles * s + ctx->num_sms - 1) / ctx->num_sms;
      const double cost = (double)waves * (2 * per + 64) + 24.0 * s;
      if (cost < best * 0.999) {
        best = cost;
        S = s;
      }
    }
    a.rows_per_split = ((a.n + S - 1) / S + bk - 1) / bk * bk;
    if (S > 1) CK(ctx->symv_part.ensure((size_t)ntiles * S * bm * pt), "alloc split workspace");
    CK(ctx->tile_cnt.ensure_zeroed((size_t)ntiles), "alloc tile counters");
    CK(ctx->tile_scal.ensure((size_t)ntiles * 3), "alloc tile scalars");
    const int64_t ldvt = (a.n + 1) / 2 * 2;
    CK(ctx->vt_buf.ensure((size_t)2 * a.p * ldvt), "alloc V^T");
    a.part = ctx->symv_part.ptr;
    a.tile_cnt = ctx->tile_cnt.ptr;
    a.tile_scal = ctx->tile_scal.ptr;
    a.glob_cnt = ctx->counters + C_SYMV;
    int rc = prof_kind ? prof_begin(ctx, prof_kind) : DRSDP_OK;
    if (rc) return rc;
    ctx->launches += 2;  // transposes
    KL(symv_gather_launch(a, epi, S, ctx->vt_buf.ptr, ldvt, ctx->stream), "product kernel (TMA, fused gather)");
    return prof_kind ? prof_end(ctx) : DRSDP_OK;
  }
  // (small n keeps the register-direct gather kernel: one launch instead of assembly + product)
  if (!no_tma && mode2 == MODE2_GATHER && !atr && a.n >= 2048 && (a.lda % 2) == 0 && ((uintptr_t)a.A & 15) == 0 &&
      (a.k == 0 || a.k == a.n)) {
    // gather-product on the TMA path: assemble W = A*(w) densely, then one K-concatenated product
    // [M | W] [V; X] = M U + A*(w) Y, the Q of the HVP epilogue (Eq. 4.7's projection term)
    const int64_t ldw = (a.n + 63) / 64 * 64;
    CK(ctx->w_dense.ensure((size_t)a.n * ldw), "alloc dense A*(w)");
    KL(gather_assemble_launch(a.n, a.amap, a.ldm, a.w, ctx->w_dense.ptr, ldw, a.skip, ctx->stream), "assemble A*(w)");
    SymvArgs b = a;
    b.A2 = ctx->w_dense.ptr;
    b.lda2 = ldw;
    b.V2 = a.X;
    b.ldv2 = a.ldx;
    b.amap = nullptr;
    b.w = nullptr;
    b.X = nullptr;
    if (symv_tma_supported(b, epi, MODE2_PAIR, false)) return run_product(ctx, b, epi, MODE2_PAIR, false, prof_kind);
  }
  static const bool no_symm = std::getenv("DRSDP_NO_SYMM") != nullptr;
  if (!no_tma && !no_symm && a.n >= 4096 && symm_supported(a, epi, mode2, atr)) {
    // upper-triangle product: reads the distinct entries of M only (symv_symm.cu)
    if (ctx->symm_n != a.n) {
      std::vector<int> hu, hs;
      const int nu = symm_units(a.n, hu, hs);
      CK(ctx->symm_units.ensure((size_t)nu), "alloc unit table");
      CK(cudaMemcpy(ctx->symm_units.ptr, hu.data(), sizeof(int) * hu.size(), cudaMemcpyHostToDevice), "copy units");
      CK(ctx->symm_ustart.ensure(hs.size()), "alloc unit starts");
      CK(cudaMemcpy(ctx->symm_ustart.ptr, hs.data(), sizeof(int) * hs.size(), cudaMemcpyHostToDevice), "copy starts");
      ctx->symm_n = a.n;
      ctx->symm_nunits = nu;
    }
    const int nb = (a.n + 127) / 128;
    CK(ctx->symm_F.ensure(symm_fpart_elems(ctx->symm_nunits, 16)), "alloc forward partials");
    CK(ctx->symm_T.ensure(symm_tpart_elems(a.n, 16)), "alloc transposed partials");
    CK(ctx->tile_scal.ensure((size_t)nb * 2 * 4), "alloc tile scalars");
    const int64_t ldvt = (a.n + 1) / 2 * 2;
    CK(ctx->vt_buf.ensure((size_t)a.p * ldvt), "alloc V^T");
    a.tile_scal = ctx->tile_scal.ptr;
    a.glob_cnt = ctx->counters + C_SYMV;
    int rc = prof_kind ? prof_begin(ctx, prof_kind) : DRSDP_OK;
    if (rc) return rc;
    ctx->launches += 2;  // transpose + partial kernel (+ the reduce below)
    KL(symm_launch(a, epi, ctx->vt_buf.ptr, ldvt, ctx->symm_units.ptr, ctx->symm_nunits, ctx->symm_ustart.ptr,
                   ctx->symm_F.ptr, ctx->symm_T.ptr, ctx->stream),
       "product kernel (upper triangle)");
    return prof_kind ? prof_end(ctx) : DRSDP_OK;
  }
  if (!no_tma && symv_tma_supported(a, epi, mode2, atr)) {
    const int pt = symv_tma_pt(a.p, epi), bm = symv_tma_rows(), bk = symv_tma_kstep();
    const bool pair = mode2 == MODE2_PAIR;
    const int kn = a.ncols > 0 ? a.ncols : a.n;
    const int ktot = pair ? 2 * ((kn + bk - 1) / bk * bk) : kn;
    const int ntiles = ((a.n + bm - 1) / bm) * symv_tma_chunks(a.p, epi);
    // split-K: one CTA per SM (the ring uses most of shared memory); waves x k-rows cost model
    int S = 1;
    double best = 1e300;
    for (int s = 1; s <= 64; ++s) {
      const int per = ((ktot + s - 1) / s + bk - 1) / bk * bk;
      if (s > 1 && (int64_t)(s - 1) * per >= ktot) break;
      const int slots = ctx->num_sms * symv_tma_ctas_per_sm(pt, epi);
      const int waves = (ntiles * s + slots - 1) / slots;
      const double cost = (double)waves * (per + 64) + 24.0 * s;
      if (cost < best * 0.999) {
        best = cost;
        S = s;
      }
    }
    a.rows_per_split = ((ktot + S - 1) / S + bk - 1) / bk * bk;
    if (S > 1) CK(ctx->symv_part.ensure((size_t)ntiles * S * bm * pt), "alloc split workspace");
    CK(ctx->tile_cnt.ensure_zeroed((size_t)ntiles), "alloc tile counters");
    CK(ctx->tile_scal.ensure((size_t)ntiles * 3), "alloc tile scalars");
    const int64_t ldvt = (kn + 1) / 2 * 2;
    CK(ctx->vt_buf.ensure((size_t)(pair || epi == EPI_BOTH ? 2 : 1) * a.p * ldvt), "alloc V^T");
    if (!pair) a.A2 = nullptr;
    a.part = ctx->symv_part.ptr;
    a.tile_cnt = ctx->tile_cnt.ptr;
    a.tile_scal = ctx->tile_scal.ptr;
    a.glob_cnt = ctx->counters + C_SYMV;
    int rc = prof_kind ? prof_begin(ctx, prof_kind) : DRSDP_OK;
    if (rc) return rc;
    ctx->launches += epi == EPI_BOTH ? 2 : 1;  // transposes
    KL(symv_tma_launch(a, epi, S, ctx->vt_buf.ptr, ldvt, ctx->stream), "product kernel (TMA)");
    return prof_kind ? prof_end(ctx) : DRSDP_OK;
  }
  const int pt = symv_pt(a.p);
  const int bn = symv_bn(pt, mode2);
  const int kext = a.k > 0 ? a.k : a.n;
  const int ntiles = ((a.n + bn - 1) / bn) * symv_chunks(a.p, epi);
  const int S = choose_splits(ctx, kext, ntiles);
  const int per = (kext + S - 1) / S;
  a.rows_per_split = ((per + 63) / 64) * 64;
  if (S > 1) CK(ctx->symv_part.ensure((size_t)ntiles * S * bn * pt), "alloc split workspace");
  CK(ctx->tile_cnt.ensure_zeroed((size_t)ntiles), "alloc tile counters");
  CK(ctx->tile_scal.ensure((size_t)ntiles * 2), "alloc tile scalars");
  a.part = ctx->symv_part.ptr;
  a.tile_cnt = ctx->tile_cnt.ptr;
  a.tile_scal = ctx->tile_scal.ptr;
  a.glob_cnt = ctx->counters + C_SYMV;
  int rc = prof_kind ? prof_begin(ctx, prof_kind) : DRSDP_OK;
  if (rc) return rc;
  KL(symv_launch(a, epi, mode2, atr, S, ctx->stream), "product kernel");
  return prof_kind ? prof_end(ctx) : DRSDP_OK;
}

static int ensure_red(drsdp_ctx *ctx, int64_t blocks, int k) {
  CK(ctx->red_part.ensure((size_t)blocks * k + 64), "alloc reduction workspace");
  return DRSDP_OK;
}

int read_scalars(drsdp_ctx *ctx, int first, int count) {
  CK(cudaMemcpyAsync(ctx->h_scal + first, ctx->d_scal + first, sizeof(double) * count, cudaMemcpyDeviceToHost,
                     ctx->stream),
     "read scalars");
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  return DRSDP_OK;
}

static int gram(drsdp_ctx *ctx, int n, int p, const double *Y, int ldv, const double *U, double *G, double *K,
                double *gg) {
  GramArgs g;
  g.n = n;
  g.p = p;
  g.Y = Y;
  g.ldy = ldv;
  g.U = U;
  g.ldu = ldv;
  g.part = ctx->gram_part.ptr;
  g.counter = ctx->counters + C_GRAM;
  g.G = G;
  g.K = K;
  g.gg = gg;
  g.max_blocks = 296;
  g.skip = ctx->skip_flag;
  KL(gram_launch(g, ctx->stream), "gram kernel");
  return DRSDP_OK;
}

static SymvArgs base_symv(drsdp_ctx *ctx, int n, int p, const double *A, int64_t lda) {
  SymvArgs a;
  a.A = A;
  a.lda = lda;
  a.n = n;
  a.p = p;
  a.skip = ctx->skip_flag;
  return a;
}

static int prof_begin(drsdp_ctx *ctx, int kind) {
  if (!ctx->prof_on) return DRSDP_OK;
  if (ctx->prof_used == ctx->prof_events.size()) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a), "event create");
    CK(cudaEventCreate(&b), "event create");
    ctx->prof_events.push_back({a, b});
    ctx->prof_kind.push_back(0);
  }
  ctx->prof_kind[ctx->prof_used] = kind;
  CK(cudaEventRecord(ctx->prof_events[ctx->prof_used].first, ctx->stream), "event record");
  return DRSDP_OK;
}

static int prof_end(drsdp_ctx *ctx) {
  if (!ctx->prof_on) return DRSDP_OK;
  CK(cudaEventRecord(ctx->prof_events[ctx->prof_used].second, ctx->stream), "event record");
  ctx->prof_used++;
  return DRSDP_OK;
}

static int run_symv(drsdp_ctx *ctx, SymvArgs &a, int epi, bool gather) {
  return run_product(ctx, a, epi, gather ? MODE2_GATHER : MODE2_NONE, false,
                     epi == EPI_COSTGRAD ? 1 : epi == EPI_HVP ? 2 : epi == EPI_BOTH ? 4 : 3);
}

// ---- generic-p building blocks (p > 64: column-chunked RAW products + row epilogues) ----------
// G = Y^T Y (p x p, pitch p) and ||G||^2 -> gg; with U also K = U^T Y + Y^T U
static int gram_generic(drsdp_ctx *ctx, int n, int p, const double *Y, int ldv, const double *U, double *G,
                        double *K, double *gg) {
  if (G) {
    SymvArgs a = base_symv(ctx, p, p, Y, ldv);
    a.k = n;
    a.V = Y;
    a.ldv = ldv;
    a.out = G;
    a.ldo = p;
    int rc = run_product(ctx, a, EPI_RAW, MODE2_NONE, false, 0);
    if (rc) return rc;
    if (gg) KL(fro2_launch(p, G, p, ctx->red_part.ptr, ctx->counters + C_FRO, gg, ctx->stream), "fro2 G");
  }
  if (U && K) {
    SymvArgs a = base_symv(ctx, p, p, U, ldv);
    a.k = n;
    a.V = Y;
    a.ldv = ldv;
    a.A2 = Y;
    a.lda2 = ldv;
    a.V2 = U;
    a.ldv2 = ldv;
    a.out = K;
    a.ldo = p;
    return run_product(ctx, a, EPI_RAW, MODE2_PAIR, false, 0);
  }
  return DRSDP_OK;
}

// W = A1 B1 (+ A2 B2): n x p rows times p x p (pitch p)
static int small_right(drsdp_ctx *ctx, int n, int p, const double *A1, int lda, const double *B1, const double *A2,
                       const double *B2, double *W, int ldw) {
  SymvArgs a = base_symv(ctx, n, p, A1, lda);
  a.k = p;
  a.V = B1;
  a.ldv = p;
  if (A2) {
    a.A2 = A2;
    a.lda2 = lda;
    a.V2 = B2;
    a.ldv2 = p;
  }
  a.out = W;
  a.ldo = ldw;
  return run_product(ctx, a, EPI_RAW, A2 ? MODE2_PAIR : MODE2_NONE, true, 0);
}

int right_product(drsdp_ctx *ctx, int n, int p, const double *A, int lda, const double *B, double *out, int ldo) {
  return small_right(ctx, n, p, A, lda, B, nullptr, nullptr, out, ldo);
}

static int ensure_big(drsdp_ctx *ctx, int n, int ldv) {
  CK(ctx->big_P.ensure((size_t)n * ldv), "alloc product buffer");
  CK(ctx->big_W.ensure((size_t)n * ldv), "alloc product buffer");
  return DRSDP_OK;
}

// generic cost+grad at Y given G (gg already in S_GG): P = M Y, W = Y G, row epilogue
static int costgrad_generic(drsdp_ctx *ctx, int n, int p, const double *M, int64_t ldm, const double *Y, int ldv,
                            const double *G, double *cost, double *egrad, double *rgrad, double *rho,
                            const double *cost_extra_dev) {
  int rc = ensure_big(ctx, n, ldv);
  if (rc) return rc;
  SymvArgs a = base_symv(ctx, n, p, M, ldm);
  a.V = Y;
  a.ldv = ldv;
  a.out = ctx->big_P.ptr;
  a.ldo = ldv;
  rc = run_product(ctx, a, EPI_RAW, MODE2_NONE, false, 1);
  if (rc) return rc;
  rc = small_right(ctx, n, p, Y, ldv, G, nullptr, nullptr, ctx->big_W.ptr, ldv);
  if (rc) return rc;
  KL(rowepi_costgrad_launch(n, p, ctx->big_P.ptr, ldv, ctx->big_W.ptr, ldv, Y, ldv, rgrad, ldv, egrad, ldv, rho,
                            ctx->red_part.ptr, ctx->counters + C_VEC, ctx->d_scal + S_SCAL, ctx->d_scal + S_GG,
                            cost_extra_dev, cost, ctx->stream),
     "row epilogue (cost+grad)");
  return DRSDP_OK;
}

// generic HVP at Y along U given G, K: Q = M U (+ gather), W = U G + Y K, row epilogue
static int hvp_generic(drsdp_ctx *ctx, int n, int p, const double *M, int64_t ldm, const double *Y, int ldv,
                       const double *U, const double *G, const double *K, const double *rho, const int32_t *amap,
                       int64_t ldmap, const double *w, double *hvp) {
  int rc = ensure_big(ctx, n, ldv);
  if (rc) return rc;
  SymvArgs a = base_symv(ctx, n, p, M, ldm);
  a.V = U;
  a.ldv = ldv;
  if (amap) {
    a.amap = amap;
    a.ldm = ldmap;
    a.w = w;
    a.X = Y;
    a.ldx = ldv;
  }
  a.out = ctx->big_P.ptr;
  a.ldo = ldv;
  rc = run_product(ctx, a, EPI_RAW, amap ? MODE2_GATHER : MODE2_NONE, false, 2);
  if (rc) return rc;
  rc = small_right(ctx, n, p, U, ldv, G, Y, K, ctx->big_W.ptr, ldv);
  if (rc) return rc;
  KL(rowepi_hvp_launch(n, p, ctx->big_P.ptr, ldv, ctx->big_W.ptr, ldv, Y, ldv, U, ldv, rho, hvp, ldv,
                       ctx->red_part.ptr, ctx->counters + C_VEC, ctx->d_scal + S_SCAL, ctx->skip_flag, ctx->stream),
     "row epilogue (hvp)");
  return DRSDP_OK;
}

// z = rowdot(T Y, Y), sum z -> zsum (any p)
int rowdot_product(drsdp_ctx *ctx, int n, int p, const double *T, int64_t ldt, const double *Y, int ldv, double *z,
                   double *zsum) {
  if (ctx->prob.nblk > 0) return blk_rowdot(ctx, p, T, ldt, Y, ldv, z, zsum);
  if (p <= 64) {
    SymvArgs a = base_symv(ctx, n, p, T, ldt);
    a.V = Y;
    a.ldv = ldv;
    a.Y = Y;
    a.ldy = ldv;
    a.zout = z;
    a.scal_out = zsum;
    return run_product(ctx, a, EPI_ROWDOT, MODE2_NONE, false, 3);
  }
  int rc = ensure_big(ctx, n, ldv);
  if (rc) return rc;
  SymvArgs a = base_symv(ctx, n, p, T, ldt);
  a.V = Y;
  a.ldv = ldv;
  a.out = ctx->big_P.ptr;
  a.ldo = ldv;
  rc = run_product(ctx, a, EPI_RAW, MODE2_NONE, false, 3);
  if (rc) return rc;
  KL(rowdot_launch(n, p, ctx->big_P.ptr, ldv, Y, ldv, z, ctx->red_part.ptr, ctx->counters + C_VEC, zsum, ctx->stream),
     "rowdot");
  return DRSDP_OK;
}

// out = normalize_rows(Y W), W p x r (pitch r); columns [r, ldo) of out zeroed
int apply_w_product(drsdp_ctx *ctx, int n, int p, const double *Y, int ldv, const double *W, int r, double *out,
                    int ldo) {
  SymvArgs a = base_symv(ctx, n, r, Y, ldv);
  a.k = p;
  a.V = W;
  a.ldv = r;
  a.out = out;
  a.ldo = ldo;
  int rc = run_product(ctx, a, EPI_RAW, MODE2_NONE, true, 0);
  if (rc) return rc;
  KL(normalize_rows_launch(n, r, ldo, out, ctx->stream), "normalize rows");
  return DRSDP_OK;
}

// Fixed-M evaluation: cost/egrad/rgrad (COSTGRAD) and hvp (HVP), device pointers.
int eval_fixed(drsdp_ctx *ctx, int flags, int n, int p, const double *M, int64_t ldm, const double *Y, int ldv,
               const double *U, double *cost, double *egrad, double *rgrad, double *hvp, double *G, double *K,
               double *rho, const double *cost_extra_dev, bool have_gram) {
  int rc = ensure_workspace(ctx, n, p);
  if (rc) return rc;
  if (p > 64 && ctx->sub_rows_mode && M == ctx->sub_M)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "row-block evaluation supports p <= 64");
  if (p > 64) {
    if (flags & DRSDP_EVAL_COSTGRAD) {
      rc = gram_generic(ctx, n, p, Y, ldv, nullptr, G, nullptr, ctx->d_scal + S_GG);
      if (rc) return rc;
      rc = costgrad_generic(ctx, n, p, M, ldm, Y, ldv, G, cost ? cost : ctx->d_scal + S_COST, egrad, rgrad, rho,
                            cost_extra_dev);
      if (rc) return rc;
    }
    if (flags & DRSDP_EVAL_HVP) {
      rc = gram_generic(ctx, n, p, Y, ldv, U, G, K, nullptr);
      if (rc) return rc;
      rc = hvp_generic(ctx, n, p, M, ldm, Y, ldv, U, G, K, rho, nullptr, 0, nullptr, hvp);
      if (rc) return rc;
    }
    return DRSDP_OK;
  }
  // row-block mode (drsdp_set_subproblem_rows): M holds rows [r0, r0 + nloc) of the n x n matrix;
  // G, K come from the full (replicated) Y, U; the epilogue works on the block's rows
  const bool rows = ctx->sub_rows_mode && M == ctx->sub_M;
  const int r0 = rows ? (int)ctx->sub_row0 : 0;
  const int nloc = rows ? (int)ctx->sub_nloc : n;
  static const bool no_both = std::getenv("DRSDP_NO_BOTH") != nullptr;
  if (flags == (DRSDP_EVAL_COSTGRAD | DRSDP_EVAL_HVP) && !no_both && p >= 5 && p <= 32) {
    // cost + gradient and the HVP along U at the same Y in ONE pass over M: the product M [Y U]
    // (2p columns) with both row epilogues (EPI_BOTH); falls through when the TMA path is unavailable
    SymvArgs a = base_symv(ctx, nloc, p, M, ldm);
    if (rows) a.ncols = n;
    a.V = Y;
    a.ldv = ldv;
    a.Y = Y + (size_t)r0 * ldv;
    a.ldy = ldv;
    a.U = U + (size_t)r0 * ldv;
    a.ldu = ldv;
    a.V2 = U;  // all rows of U: the second half of the contraction operand [Y U]
    a.ldv2 = ldv;
    if (symv_tma_supported(a, EPI_BOTH, MODE2_NONE, false)) {
      rc = gram(ctx, n, p, Y, ldv, U, G, K, ctx->d_scal + S_GG);
      if (rc) return rc;
      a.G = G;
      a.K = K;
      a.out = rgrad;
      a.ldo = ldv;
      a.egrad = egrad;
      a.lde = ldv;
      a.rho_out = rho;
      a.out2 = hvp;
      a.ldo2 = ldv;
      a.scal_out = ctx->d_scal + S_SCAL;
      a.scal_out2 = ctx->d_scal + S_UH;
      a.gg = (rows && r0 > 0) ? ctx->d_scal + S_ZERO : ctx->d_scal + S_GG;
      a.cost_extra = cost_extra_dev;
      a.cost_out = cost ? cost : ctx->d_scal + S_COST;
      return run_symv(ctx, a, EPI_BOTH, false);
    }
  }
  if (flags & DRSDP_EVAL_COSTGRAD) {
    rc = gram(ctx, n, p, Y, ldv, nullptr, G, nullptr, ctx->d_scal + S_GG);
    if (rc) return rc;
    SymvArgs a = base_symv(ctx, nloc, p, M, ldm);
    if (rows) a.ncols = n;
    a.V = Y;
    a.ldv = ldv;
    a.Y = Y + (size_t)r0 * ldv;
    a.ldy = ldv;
    a.G = G;
    a.out = rgrad;
    a.ldo = ldv;
    a.egrad = egrad;
    a.lde = ldv;
    a.rho_out = rho;
    a.scal_out = ctx->d_scal + S_SCAL;
    // row blocks: the cost is additive over blocks with ||G||^2 counted by the block holding row 0
    a.gg = (rows && r0 > 0) ? ctx->d_scal + S_ZERO : ctx->d_scal + S_GG;
    a.cost_extra = cost_extra_dev;
    a.cost_out = cost ? cost : ctx->d_scal + S_COST;
    rc = run_symv(ctx, a, EPI_COSTGRAD, false);
    if (rc) return rc;
  }
  if (flags & DRSDP_EVAL_HVP) {
    rc = gram(ctx, n, p, Y, ldv, U, G, K, ctx->d_scal + S_GG);
    if (rc) return rc;
    SymvArgs a = base_symv(ctx, nloc, p, M, ldm);
    if (rows) a.ncols = n;
    a.V = U;
    a.ldv = ldv;
    a.Y = Y + (size_t)r0 * ldv;
    a.ldy = ldv;
    a.U = U + (size_t)r0 * ldv;
    a.ldu = ldv;
    a.G = G;
    a.K = K;
    a.rho = rho;
    a.out = hvp;
    a.ldo = ldv;
    a.scal_out = ctx->d_scal + S_SCAL;
    rc = run_symv(ctx, a, EPI_HVP, false);
    if (rc) return rc;
  }
  (void)have_gram;
  return DRSDP_OK;
}

static SegArgs seg_args(drsdp_ctx *ctx, int p, const double *Y, const double *U, int ldv, double *out) {
  Problem &P = ctx->prob;
  SegArgs s;
  s.m = P.m;
  s.seg_ptr = P.seg_ptr.ptr;
  s.seg_pos = P.seg_pos.ptr;
  s.cnt = P.cnt.ptr;
  s.is_large = P.is_large.ptr;
  s.large_ids = P.large_ids.ptr;
  s.n_large = P.n_large;
  s.huge_ids = P.huge_ids.ptr;
  s.n_huge = P.n_huge;
  s.cA = P.has_C ? P.cA.ptr : nullptr;
  s.Y = Y;
  s.U = U;
  s.ld = ldv;
  s.p = p;
  s.out = out;
  s.part = ctx->red_part.ptr;
  s.counter = ctx->counters + C_SEG;
  s.scal_out = ctx->d_scal + S_SEGSQ;
  s.skip = ctx->skip_flag;
  return s;
}

// ----------------------------------------------------------------------------------------------
// multi-block problems (blocks.cu): the same evaluations over the diagonal blocks
// ----------------------------------------------------------------------------------------------
static int blk_tiles(drsdp_ctx *ctx, SymvArgs &a) {
  const Problem &P = ctx->prob;
  CK(ctx->tile_scal.ensure((size_t)blk_product_tiles((int)P.nblk, (int)P.nb) * 2), "alloc tile scalars");
  a.tile_scal = ctx->tile_scal.ptr;
  a.glob_cnt = ctx->counters + C_SYMV;
  return DRSDP_OK;
}

int blk_rowdot(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, const double *Y, int ldv, double *z, double *zsum) {
  const Problem &P = ctx->prob;
  if (p > kBlkMaxP) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "block problems support p <= 128");
  SymvArgs a = base_symv(ctx, (int)P.n, p, T, ldt);
  a.V = Y;
  a.ldv = ldv;
  a.Y = Y;
  a.ldy = ldv;
  a.zout = z;
  a.scal_out = zsum;
  int rc = blk_tiles(ctx, a);
  if (rc) return rc;
  KL(blk_product_launch(a, EPI_ROWDOT, false, (int)P.nblk, (int)P.nb, ctx->stream), "block product (z)");
  return DRSDP_OK;
}

// T <- T - sigma (A*(y) - S) on every block (Alg. 2 step 6); scal_out = S_DUAL slots
int blk_dual(drsdp_ctx *ctx, int p, const double *Y, int ldv, const double *y, double sigma, double *T, int64_t ldt) {
  const Problem &P = ctx->prob;
  CK(ctx->red_part.ensure((size_t)blk_elem_blocks((int)P.nblk, (int)P.nb) * 3 + 64), "alloc reduction workspace");
  BlkElemArgs e;
  e.t = (int)P.nblk;
  e.nb = (int)P.nb;
  e.p = p;
  e.Y = Y;
  e.ldy = ldv;
  e.amap = P.amap.ptr;
  e.ldm = P.ld;
  e.y = y;
  e.T = T;
  e.ldt = ldt;
  e.sigma = sigma;
  e.part = ctx->red_part.ptr;
  e.counter = ctx->counters + C_DUAL;
  e.scal_out = ctx->d_scal + S_DUAL;
  KL(blk_elem_launch(e, BLK_DUAL, ctx->stream), "block dual update");
  return DRSDP_OK;
}

static int alm_costgrad_blocks(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, double sigma, const double *Y,
                               int ldv, double *Mout, int64_t ldm, double *yS, double *G, double *rho, double *cost,
                               double *egrad, double *rgrad, double *Dbuf);
static int alm_hvp_blocks(drsdp_ctx *ctx, int p, const double *M, int64_t ldm, const double *Y, int ldv,
                          const double *U, const double *G, double *K, const double *rho, double *wZ, double *hvp,
                          double *Zbuf);

// y-eliminated subproblem at Y: y(S), M(S) (materialised into Mout), cost/gradients.
static bool use_dense(const double *Y, const double *U, int ldv) {
  static const bool off = std::getenv("DRSDP_NO_DENSE") != nullptr;
  return !off && gram_tile_supported(Y, U, ldv);
}

int alm_costgrad(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, double sigma, const double *Y, int ldv,
                 double *Mout, int64_t ldm, double *yS, double *G, double *rho, double *cost, double *egrad,
                 double *rgrad, double *Dbuf) {
  Problem &P = ctx->prob;
  if (P.nblk > 0)
    return alm_costgrad_blocks(ctx, p, T, ldt, sigma, Y, ldv, Mout, ldm, yS, G, rho, cost, egrad, rgrad, Dbuf);
  const int n = (int)P.n;
  int rc = ensure_workspace(ctx, n, p);
  if (rc) return rc;
  rc = ensure_red(ctx, std::max<int64_t>({(int64_t)segsum_blocks(P.m, P.n_large, P.n_huge), (int64_t)assemble_alm_blocks(n), 1184}), 4);
  if (rc) return rc;
  rc = p > 64 ? gram_generic(ctx, n, p, Y, ldv, nullptr, G, nullptr, ctx->d_scal + S_GG)
             : gram(ctx, n, p, Y, ldv, nullptr, G, nullptr, ctx->d_scal + S_GG);
  if (rc) return rc;
  SegArgs s = seg_args(ctx, p, Y, nullptr, ldv, yS);
  const bool dense = Dbuf && use_dense(Y, Y, ldv);
  if (dense) {
    // S = Y Y^T as dense upper tiles (tensor path), then the segmented sum gathers from it
    KL(gram_tile_launch(n, p, Y, Y, nullptr, nullptr, ldv, Dbuf, P.ld, ctx->skip_flag, ctx->stream), "gram tiles");
    s.D = Dbuf;
    s.ldd = P.ld;
  }
  KL(segsum_launch(s, false, ctx->stream), "segsum kernel");
  AssembleArgs as;
  as.n = n;
  as.amap = P.amap.ptr;
  as.ldmap = P.ld;
  as.y = yS;
  as.C = P.has_C ? P.C.ptr : nullptr;
  as.ldc = P.ld;
  as.T = T;
  as.ldt = ldt;
  as.sigma = sigma;
  as.M = Mout;
  as.ldm = ldm;
  as.part = ctx->red_part.ptr;
  as.counter = ctx->counters + C_ASM;
  as.scal_out = ctx->d_scal + S_ALM;
  KL(assemble_alm_launch(as, p, Y, ldv, ctx->stream, dense ? Dbuf : nullptr, P.ld), "assemble (ALM) kernel");
  // accurate cost f^ = sum R^2 + (2/sigma) <T, S + C> + ||T||^2/sigma^2 (reading R29)
  KL(alm_cost_launch(ctx->d_scal + S_ALM, sigma, cost ? cost : ctx->d_scal + S_COST, ctx->stream), "alm cost");
  if (p > 64) return costgrad_generic(ctx, n, p, Mout, ldm, Y, ldv, G, nullptr, egrad, rgrad, rho, nullptr);
  SymvArgs a = base_symv(ctx, n, p, Mout, ldm);
  a.V = Y;
  a.ldv = ldv;
  a.Y = Y;
  a.ldy = ldv;
  a.G = G;
  a.out = rgrad;
  a.ldo = ldv;
  a.egrad = egrad;
  a.lde = ldv;
  a.rho_out = rho;
  a.scal_out = ctx->d_scal + S_SCAL;
  a.gg = ctx->d_scal + S_GG;
  a.cost_extra = nullptr;
  a.cost_out = nullptr;  // the cost comes from the assembly pass (accurate form)
  return run_symv(ctx, a, EPI_COSTGRAD, false);
}

int alm_hvp(drsdp_ctx *ctx, int p, const double *M, int64_t ldm, const double *Y, int ldv, const double *U,
            const double *G, double *K, const double *rho, double *wZ, double *hvp, double *Zbuf) {
  Problem &P = ctx->prob;
  if (P.nblk > 0) return alm_hvp_blocks(ctx, p, M, ldm, Y, ldv, U, G, K, rho, wZ, hvp, Zbuf);
  const int n = (int)P.n;
  // K = U^T Y + Y^T U runs on the auxiliary stream, concurrently with Z and its segmented sum
  // (fork / join with events; inside a graph capture this becomes two parallel branches)
  cudaStream_t main_stream = ctx->stream;
  const bool fork = ctx->aux_stream != nullptr;
  if (fork) {
    CK(cudaEventRecord(ctx->ev_fork, main_stream), "event record");
    CK(cudaStreamWaitEvent(ctx->aux_stream, ctx->ev_fork, 0), "stream wait");
    ctx->stream = ctx->aux_stream;
  }
  int rc = ctx->g_scratch.cap >= (size_t)p * p ? DRSDP_OK
                                                : cuda_check(ctx, ctx->g_scratch.ensure((size_t)p * p), "alloc G");
  if (rc) return rc;
  rc = p > 64 ? gram_generic(ctx, n, p, Y, ldv, U, nullptr, K, nullptr)
              : gram(ctx, n, p, Y, ldv, U, ctx->g_scratch.ptr, K, nullptr);
  if (fork) {
    ctx->stream = main_stream;
    if (rc) return rc;
    CK(cudaEventRecord(ctx->ev_join, ctx->aux_stream), "event record");
  }
  if (rc) return rc;
  SegArgs s = seg_args(ctx, p, Y, U, ldv, wZ);
  if (Zbuf && use_dense(Y, U, ldv)) {
    // Z = Y U^T + U Y^T = [Y U][U Y]^T as dense upper tiles
    KL(gram_tile_launch(n, p, Y, U, U, Y, ldv, Zbuf, P.ld, ctx->skip_flag, ctx->stream), "gram tiles (Z)");
    s.D = Zbuf;
    s.ldd = P.ld;
  }
  KL(segsum_launch(s, true, ctx->stream), "segsum kernel (Z)");
  if (fork) CK(cudaStreamWaitEvent(main_stream, ctx->ev_join, 0), "stream wait");
  if (p > 64) return hvp_generic(ctx, n, p, M, ldm, Y, ldv, U, G, K, rho, P.amap.ptr, P.ld, wZ, hvp);
  SymvArgs a = base_symv(ctx, n, p, M, ldm);
  a.V = U;
  a.ldv = ldv;
  a.amap = P.amap.ptr;
  a.ldm = P.ld;
  a.w = wZ;
  a.X = Y;
  a.ldx = ldv;
  a.Y = Y;
  a.ldy = ldv;
  a.U = U;
  a.ldu = ldv;
  a.G = G;
  a.K = K;
  a.rho = rho;
  a.out = hvp;
  a.ldo = ldv;
  a.scal_out = ctx->d_scal + S_SCAL;
  return run_symv(ctx, a, EPI_HVP, true);
}


// Block ALM cost + gradients (oracle/sparse_bqp.py BlockALMProblem.costgrad): G_k, y(S) by the
// segmented sum over all blocks' positions (global rows), M(S) and the accurate cost sums fused
// with the S tiles, then the block product with the COSTGRAD row epilogue.
static int alm_costgrad_blocks(drsdp_ctx *ctx, int p, const double *T, int64_t ldt, double sigma, const double *Y,
                               int ldv, double *Mout, int64_t ldm, double *yS, double *G, double *rho, double *cost,
                               double *egrad, double *rgrad, double *Dbuf) {
  Problem &P = ctx->prob;
  const int t = (int)P.nblk, nb = (int)P.nb;
  if (p > kBlkMaxP) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "block problems support p <= 128");
  int rc = ensure_red(ctx, std::max<int64_t>(segsum_blocks(P.m, P.n_large, P.n_huge), blk_elem_blocks(t, nb)), 4);
  if (rc) return rc;
  KL(blk_gram_launch(t, nb, p, Y, ldv, nullptr, 0, G, nullptr, ctx->skip_flag, ctx->stream), "block gram");
  SegArgs s = seg_args(ctx, p, Y, nullptr, ldv, yS);
  if (Dbuf) {
    // S_k = Y_k Y_k^T as dense stacked tiles: the segmented sum gathers one entry per position and
    // the assembly reads them back (instead of p-length dot products per position)
    KL(blk_tile_launch(t, nb, p, Y, nullptr, ldv, Dbuf, P.ld, ctx->skip_flag, ctx->stream), "block tiles (S)");
    s.D = Dbuf;
    s.ldd = P.ld;
    s.nbk = nb;
  }
  KL(segsum_launch(s, false, ctx->stream), "segsum kernel");
  BlkElemArgs e;
  e.D = Dbuf;
  e.ldd = P.ld;
  e.t = t;
  e.nb = nb;
  e.p = p;
  e.Y = Y;
  e.ldy = ldv;
  e.amap = P.amap.ptr;
  e.ldm = P.ld;
  e.y = yS;
  e.T = const_cast<double *>(T);  // read only in BLK_ASM
  e.ldt = ldt;
  e.sigma = sigma;
  e.M = Mout;
  e.ldmo = ldm;
  e.part = ctx->red_part.ptr;
  e.counter = ctx->counters + C_ASM;
  e.scal_out = ctx->d_scal + S_ALM;
  KL(blk_elem_launch(e, BLK_ASM, ctx->stream), "block assembly");
  KL(alm_cost_launch(ctx->d_scal + S_ALM, sigma, cost ? cost : ctx->d_scal + S_COST, ctx->stream), "alm cost");
  SymvArgs a = base_symv(ctx, (int)P.n, p, Mout, ldm);
  a.V = Y;
  a.ldv = ldv;
  a.Y = Y;
  a.ldy = ldv;
  a.G = G;
  a.out = rgrad;
  a.ldo = ldv;
  a.egrad = egrad;
  a.lde = ldv;
  a.rho_out = rho;
  a.scal_out = ctx->d_scal + S_SCAL;
  rc = blk_tiles(ctx, a);
  if (rc) return rc;
  KL(blk_product_launch(a, EPI_COSTGRAD, false, t, nb, ctx->stream), "block product (cost+grad)");
  return DRSDP_OK;
}

// Block ALM HVP (BlockALMProblem.hess): K_k, w = A(Z)/cnt (Z_k = Y_k U_k^T + U_k Y_k^T, segmented
// sum from Y, U rows), then one block product Q = M U + A*(w) Y (gather) with the HVP epilogue:
// three launches per Hessian-vector product.
static int alm_hvp_blocks(drsdp_ctx *ctx, int p, const double *M, int64_t ldm, const double *Y, int ldv,
                          const double *U, const double *G, double *K, const double *rho, double *wZ, double *hvp,
                          double *Zbuf) {
  Problem &P = ctx->prob;
  const int t = (int)P.nblk, nb = (int)P.nb;
  if (p > kBlkMaxP) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "block problems support p <= 128");
  KL(blk_gram_launch(t, nb, p, Y, ldv, U, ldv, nullptr, K, ctx->skip_flag, ctx->stream), "block gram (K)");
  SegArgs s = seg_args(ctx, p, Y, U, ldv, wZ);
  if (Zbuf) {
    KL(blk_tile_launch(t, nb, p, Y, U, ldv, Zbuf, P.ld, ctx->skip_flag, ctx->stream), "block tiles (Z)");
    s.D = Zbuf;
    s.ldd = P.ld;
    s.nbk = nb;
  }
  KL(segsum_launch(s, true, ctx->stream), "segsum kernel (Z)");
  SymvArgs a = base_symv(ctx, (int)P.n, p, M, ldm);
  a.V = U;
  a.ldv = ldv;
  a.amap = P.amap.ptr;
  a.ldm = P.ld;
  a.w = wZ;
  a.X = Y;
  a.ldx = ldv;
  a.Y = Y;
  a.ldy = ldv;
  a.U = U;
  a.ldu = ldv;
  a.G = G;
  a.K = K;
  a.rho = rho;
  a.out = hvp;
  a.ldo = ldv;
  a.scal_out = ctx->d_scal + S_SCAL;
  int rc = blk_tiles(ctx, a);
  if (rc) return rc;
  KL(blk_product_launch(a, EPI_HVP, true, t, nb, ctx->stream), "block product (HVP)");
  return DRSDP_OK;
}

// ----------------------------------------------------------------------------------------------
// Problem construction
// ----------------------------------------------------------------------------------------------
// Validates the staged problem P (host arrays filled by set_problem / set_bqp), builds its CSR
// segments and device copies, and only then replaces ctx->prob (releasing the previous problem's
// device buffers). On any error ctx->prob is left untouched and P's partial allocations freed.
static int finalize_staged(drsdp_ctx *ctx, Problem &P, const double *C_host);
static int finalize_problem(drsdp_ctx *ctx, Problem &P, const double *C_host) {
  const int rc = finalize_staged(ctx, P, C_host);
  if (rc) {
    P.release();
    return rc;
  }
  ctx->has_problem = false;
  ctx->prob.release();
  ctx->prob = P;  // DBufs move by copy (no destructor); P is not used again
  ctx->has_problem = true;
  ctx->alm_cached_valid = false;
  ctx->h_Y0.clear();  // an initial factor belongs to the problem it was given for
  ctx->p0_given = 0;
  free_solver(ctx);
  ctx->trace.clear();
  return DRSDP_OK;
}

static int finalize_staged(drsdp_ctx *ctx, Problem &P, const double *C_host) {
  const int64_t n = P.n, m = P.m;
  // counts, CSR over upper positions (constraint-major, row-major within a constraint)
  std::vector<int64_t> cnt_upper(m, 0);
  std::vector<int64_t> cnt_ord(m, 0);
  // dense: one n x n block; blocks: row r of block r / nb holds columns [0, nb) of that block
  const bool blk = P.nblk > 0;
  const int64_t cols = blk ? P.nb : n;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t base = blk ? r / cols * cols : 0;
    for (int64_t j = r - base; j < cols; ++j) {
      const int32_t id = P.h_amap[r * cols + j];
      if (id < 0) continue;
      cnt_upper[id]++;
      cnt_ord[id] += (r - base == j) ? 1 : 2;
    }
  }
  for (int64_t a = 0; a < m; ++a)
    if (cnt_ord[a] == 0)
      return set_error(ctx, DRSDP_ERR_SINGULAR_AAT,
                       "constraint " + std::to_string(a) + " has no position (Assumption 2, P:33)");
  P.h_cnt.assign(m, 0);
  for (int64_t a = 0; a < m; ++a) {
    if (cnt_ord[a] > INT32_MAX) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "constraint too large");
    P.h_cnt[a] = (int32_t)cnt_ord[a];
  }
  P.h_seg_ptr.assign(m + 1, 0);
  for (int64_t a = 0; a < m; ++a) P.h_seg_ptr[a + 1] = P.h_seg_ptr[a] + cnt_upper[a];
  P.n_upper = P.h_seg_ptr[m];
  P.h_seg_pos.assign(P.n_upper, 0);
  {
    std::vector<int64_t> fill(P.h_seg_ptr.begin(), P.h_seg_ptr.end() - 1);
    for (int64_t r = 0; r < n; ++r) {
      const int64_t base = blk ? r / cols * cols : 0;
      for (int64_t j = r - base; j < cols; ++j) {
        const int32_t id = P.h_amap[r * cols + j];
        if (id < 0) continue;
        P.h_seg_pos[fill[id]++] = ((uint32_t)r << 16) | (uint32_t)(base + j);  // global rows
      }
    }
  }
  // segment tiers for segsum: <= 32 upper positions one thread, 33..256 one warp, > 256 one block
  std::vector<uint8_t> is_large(m, 0);
  std::vector<int32_t> large_ids, huge_ids;
  for (int64_t a = 0; a < m; ++a)
    if (cnt_upper[a] > 32) {
      is_large[a] = 1;
      (cnt_upper[a] > 256 ? huge_ids : large_ids).push_back((int32_t)a);
    }
  P.n_large = (int64_t)large_ids.size();
  P.n_huge = (int64_t)huge_ids.size();
  // device copies
  P.ld = ((cols + 63) / 64) * 64;
  std::vector<int32_t> amap_pad((size_t)n * P.ld, -1);
  for (int64_t i = 0; i < n; ++i) std::memcpy(&amap_pad[i * P.ld], &P.h_amap[i * cols], sizeof(int32_t) * cols);
  CK(P.amap.ensure(amap_pad.size()), "alloc amap");
  CK(cudaMemcpy(P.amap.ptr, amap_pad.data(), sizeof(int32_t) * amap_pad.size(), cudaMemcpyHostToDevice), "copy amap");
  CK(P.cnt.ensure(m), "alloc cnt");
  CK(cudaMemcpy(P.cnt.ptr, P.h_cnt.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice), "copy cnt");
  CK(P.b.ensure(m), "alloc b");
  CK(cudaMemcpy(P.b.ptr, P.h_b.data(), sizeof(double) * m, cudaMemcpyHostToDevice), "copy b");
  CK(P.seg_ptr.ensure(m + 1), "alloc seg_ptr");
  CK(cudaMemcpy(P.seg_ptr.ptr, P.h_seg_ptr.data(), sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice), "copy seg_ptr");
  CK(P.seg_pos.ensure(std::max<int64_t>(P.n_upper, 1)), "alloc seg_pos");
  CK(cudaMemcpy(P.seg_pos.ptr, P.h_seg_pos.data(), sizeof(uint32_t) * P.n_upper, cudaMemcpyHostToDevice),
     "copy seg_pos");
  CK(P.is_large.ensure(m), "alloc is_large");
  CK(cudaMemcpy(P.is_large.ptr, is_large.data(), m, cudaMemcpyHostToDevice), "copy is_large");
  CK(P.large_ids.ensure(std::max<int64_t>(P.n_large, 1)), "alloc large_ids");
  if (P.n_large)
    CK(cudaMemcpy(P.large_ids.ptr, large_ids.data(), sizeof(int32_t) * P.n_large, cudaMemcpyHostToDevice),
       "copy large_ids");
  CK(P.huge_ids.ensure(std::max<int64_t>(P.n_huge, 1)), "alloc huge_ids");
  if (P.n_huge)
    CK(cudaMemcpy(P.huge_ids.ptr, huge_ids.data(), sizeof(int32_t) * P.n_huge, cudaMemcpyHostToDevice),
       "copy huge_ids");
  P.has_C = C_host != nullptr;
  if (P.has_C) {
    std::vector<double> cpad((size_t)n * P.ld, 0.0);
    std::vector<double> cA(m, 0.0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        cpad[i * P.ld + j] = C_host[i * n + j];
        const int32_t id = P.h_amap[i * n + j];
        if (id >= 0) cA[id] += C_host[i * n + j];
      }
    CK(P.C.ensure(cpad.size()), "alloc C");
    CK(cudaMemcpy(P.C.ptr, cpad.data(), sizeof(double) * cpad.size(), cudaMemcpyHostToDevice), "copy C");
    CK(P.cA.ensure(m), "alloc cA");
    CK(cudaMemcpy(P.cA.ptr, cA.data(), sizeof(double) * m, cudaMemcpyHostToDevice), "copy cA");
  }
  return DRSDP_OK;
}

// graded-lex rank of square-free monomials of degree <= 4 over d variables
struct MonoRank {
  int d;
  std::vector<int64_t> off;              // offset of degree k
  std::vector<std::vector<int64_t>> cum;  // cum[k][x] = sum_{v < x} C(d - v - 1, k - 1)
  static int64_t binom(int64_t a, int64_t b) {
    if (b < 0 || a < b) return 0;
    int64_t r = 1;
    for (int64_t i = 1; i <= b; ++i) r = r * (a - b + i) / i;
    return r;
  }
  explicit MonoRank(int d_) : d(d_) {
    off.assign(6, 0);
    for (int k = 0; k < 5; ++k) off[k + 1] = off[k] + binom(d, k);
    cum.assign(5, std::vector<int64_t>(d + 1, 0));
    for (int k = 1; k <= 4; ++k)
      for (int x = 0; x < d; ++x) cum[k][x + 1] = cum[k][x] + binom(d - x - 1, k - 1);
  }
  // a: sorted indices, k = size
  int64_t id(const int *a, int k) const {
    int64_t r = 0;
    int prev = -1;
    for (int i = 0; i < k; ++i) {
      const int kk = k - i;
      r += cum[kk][a[i]] - cum[kk][prev + 1];
      prev = a[i];
    }
    return off[k] + r;
  }
};

}  // namespace drsdp

// ==============================================================================================
// extern "C"
// ==============================================================================================
extern "C" {

int drsdp_create(drsdp_ctx **out, int device, void *cuda_stream) {
  if (!out) return DRSDP_ERR_INVALID_ARG;
  *out = nullptr;
  drsdp_ctx *ctx = new (std::nothrow) drsdp_ctx();
  if (!ctx) return DRSDP_ERR_OOM;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    delete ctx;
    return DRSDP_ERR_CUDA;
  }
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return DRSDP_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return DRSDP_ERR_CUDA;
    }
    ctx->own_stream = true;
  }
  bool ok = cudaMalloc(&ctx->counters, sizeof(unsigned) * C_TOTAL) == cudaSuccess &&
            cudaMemset(ctx->counters, 0, sizeof(unsigned) * C_TOTAL) == cudaSuccess &&
            cudaMalloc(&ctx->d_scal, sizeof(double) * S_TOTAL) == cudaSuccess &&
            cudaMemset(ctx->d_scal, 0, sizeof(double) * S_TOTAL) == cudaSuccess &&
            cudaMallocHost(&ctx->h_scal, sizeof(double) * S_TOTAL) == cudaSuccess &&
            cudaMalloc(&ctx->d_flag, sizeof(int)) == cudaSuccess &&
            ctx->sub_G.ensure(2 * 64 * 64) == cudaSuccess && ctx->sub_K.ensure(64 * 64) == cudaSuccess &&
            ctx->red_part.ensure(1 << 16) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    drsdp_destroy(ctx);
    return DRSDP_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    drsdp_destroy(ctx);
    return DRSDP_ERR_CUDA;
  }
  drsdp_default_params(&ctx->prm);
  *out = ctx;
  return DRSDP_OK;
}

void drsdp_destroy(drsdp_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  free_solver(ctx);
  ctx->prob.release();
  ctx->red_part.release();
  ctx->gram_part.release();
  ctx->symv_part.release();
  ctx->big_P.release();
  ctx->big_W.release();
  ctx->vt_buf.release();
  ctx->w_dense.release();
  ctx->symm_units.release();
  ctx->symm_ustart.release();
  ctx->symm_F.release();
  ctx->symm_T.release();
  ctx->tile_cnt.release();
  ctx->tile_scal.release();
  ctx->sub_G.release();
  ctx->sub_K.release();
  ctx->sub_rho.release();
  ctx->g_scratch.release();
  ctx->alm_G.release();
  ctx->alm_K.release();
  ctx->alm_rho.release();
  ctx->alm_M.release();
  ctx->alm_yS.release();
  ctx->alm_wZ.release();
  ctx->alm_D.release();
  ctx->alm_Z.release();
  ctx->host_stage.release();
  for (auto &e : ctx->prof_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (ctx->counters) cudaFree(ctx->counters);
  if (ctx->d_scal) cudaFree(ctx->d_scal);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->d_flag) cudaFree(ctx->d_flag);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->aux_stream) {
    cudaStreamSynchronize(ctx->aux_stream);
    cudaStreamDestroy(ctx->aux_stream);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

const char *drsdp_last_error(const drsdp_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int drsdp_sync(drsdp_ctx *ctx) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "stream sync");
}

int drsdp_launch_count(drsdp_ctx *ctx, int64_t *count) {
  if (!ctx || !count) return DRSDP_ERR_INVALID_ARG;
  *count = ctx->launches;
  return DRSDP_OK;
}

int drsdp_profile_enable(drsdp_ctx *ctx, int enable) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  ctx->prof_on = enable != 0;
  ctx->prof_used = 0;
  return DRSDP_OK;
}

int drsdp_profile_read(drsdp_ctx *ctx, int32_t kind, double *ms, int64_t *launches) {
  if (!ctx || kind < 0 || kind > 4) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  double tot = 0.0;
  int64_t cnt = 0;
  for (size_t k = 0; k < ctx->prof_used; ++k) {
    if (kind != 0 && ctx->prof_kind[k] != kind) continue;
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ctx->prof_events[k].first, ctx->prof_events[k].second), "event elapsed");
    tot += t;
    ++cnt;
  }
  if (ms) *ms = tot;
  if (launches) *launches = cnt;
  return DRSDP_OK;
}

int drsdp_set_problem(drsdp_ctx *ctx, int64_t n, int64_t m, const double *C, int64_t nnz, const int32_t *row,
                      const int32_t *col, const int32_t *cons, const double *b) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (n <= 0 || n >= 65536 || m <= 0 || nnz < 0 || !b || (nnz > 0 && (!row || !col || !cons)))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_problem: bad sizes or NULL arrays");
  cudaSetDevice(ctx->device);
  Problem P;  // staged: ctx->prob is replaced only after validation succeeds
  P.n = n;
  P.m = m;
  P.h_amap.assign((size_t)n * n, -1);
  for (int64_t k = 0; k < nnz; ++k) {
    const int32_t i = row[k], j = col[k], a = cons[k];
    if (i < 0 || j < 0 || i >= n || j >= n || i > j || a < 0 || a >= m)
      return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_problem: triplet " + std::to_string(k) + " out of range");
    if (P.h_amap[(size_t)i * n + j] != -1)
      return set_error(ctx, DRSDP_ERR_NOT_SYMMETRIC, "set_problem: duplicate position " + std::to_string(k));
    P.h_amap[(size_t)i * n + j] = a;
    P.h_amap[(size_t)j * n + i] = a;
  }
  if (C) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i + 1; j < n; ++j)
        if (C[i * n + j] != C[j * n + i]) return set_error(ctx, DRSDP_ERR_NOT_SYMMETRIC, "set_problem: C not symmetric");
  }
  P.h_b.assign(b, b + m);
  return finalize_problem(ctx, P, C);
}

int drsdp_set_bqp(drsdp_ctx *ctx, int32_t d, const double *Q, const double *c) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (d < 1 || d > 360 || !Q || !c) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_bqp: need 1 <= d <= 360");
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j)
      if (Q[i * d + j] != Q[j * d + i]) return set_error(ctx, DRSDP_ERR_NOT_SYMMETRIC, "set_bqp: Q not symmetric");
  cudaSetDevice(ctx->device);
  MonoRank mr(d);
  Problem P;  // staged (see finalize_problem)
  const int64_t n = 1 + d + (int64_t)d * (d - 1) / 2;
  P.n = n;
  P.m = mr.off[5];
  // basis monomials, graded-lex: [], [i], [i,j]
  std::vector<int> bs(n * 2, -1);
  std::vector<int> bk(n, 0);
  int64_t t = 1;
  for (int i = 0; i < d; ++i, ++t) {
    bs[2 * t] = i;
    bk[t] = 1;
  }
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j, ++t) {
      bs[2 * t] = i;
      bs[2 * t + 1] = j;
      bk[t] = 2;
    }
  P.h_amap.assign((size_t)n * n, -1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i; j < n; ++j) {
      // symmetric difference of two sorted sets of size <= 2
      int a[4], k = 0;
      int ia = 0, ja = 0;
      const int *A = &bs[2 * i], *B = &bs[2 * j];
      const int ka = bk[i], kb = bk[j];
      while (ia < ka || ja < kb) {
        if (ja >= kb || (ia < ka && A[ia] < B[ja])) a[k++] = A[ia++];
        else if (ia >= ka || B[ja] < A[ia]) a[k++] = B[ja++];
        else {
          ++ia;
          ++ja;
        }
      }
      const int32_t id = (int32_t)mr.id(a, k);
      P.h_amap[(size_t)i * n + j] = id;
      P.h_amap[(size_t)j * n + i] = id;
    }
  P.h_b.assign(P.m, 0.0);
  double tr = 0.0;
  for (int i = 0; i < d; ++i) tr += Q[i * d + i];
  P.h_b[0] = tr;
  for (int i = 0; i < d; ++i) {
    int a[1] = {i};
    P.h_b[mr.id(a, 1)] = c[i];
  }
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j) {
      int a[2] = {i, j};
      P.h_b[mr.id(a, 2)] = 2.0 * Q[i * d + j];
    }
  return finalize_problem(ctx, P, nullptr);
}

int drsdp_set_blocks(drsdp_ctx *ctx, int32_t nblk, int32_t nb, int64_t m, const int32_t *amaps, const double *b) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (nblk < 1 || nb < 1 || (int64_t)nblk * nb >= 65536 || m <= 0 || !amaps || !b)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_blocks: need nblk, nb >= 1, nblk * nb < 65536, m >= 1");
  const int64_t N = (int64_t)nblk * nb;
  for (int64_t k = 0; k < nblk; ++k)
    for (int64_t i = 0; i < nb; ++i)
      for (int64_t j = 0; j < nb; ++j) {
        const int32_t a = amaps[(k * nb + i) * nb + j];
        if (a < 0 || a >= m) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_blocks: id out of range");
        if (a != amaps[(k * nb + j) * nb + i])
          return set_error(ctx, DRSDP_ERR_NOT_SYMMETRIC, "set_blocks: block map not symmetric");
      }
  cudaSetDevice(ctx->device);
  Problem P;  // staged
  P.n = N;
  P.m = m;
  P.nblk = nblk;
  P.nb = nb;
  P.h_amap.assign(amaps, amaps + N * nb);
  P.h_b.assign(b, b + m);
  return finalize_problem(ctx, P, nullptr);
}

int drsdp_set_bqp_chain(drsdp_ctx *ctx, int32_t q, int32_t t, const double *Q, const double *c) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  const int64_t nb = 1 + q + (int64_t)q * (q - 1) / 2;
  if (q < 2 || t < 1 || !Q || !c || nb * t >= 65536 || (int64_t)(q - 2) * t + 2 > 32767)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_bqp_chain: need q >= 2, t >= 1, t (1 + q + q(q-1)/2) < 65536");
  for (int64_t k = 0; k < t; ++k)
    for (int i = 0; i < q; ++i)
      for (int j = i + 1; j < q; ++j)
        if (Q[(k * q + i) * q + j] != Q[(k * q + j) * q + i])
          return set_error(ctx, DRSDP_ERR_NOT_SYMMETRIC, "set_bqp_chain: Q_k not symmetric");
  // monomial keys: degree in bits 60.., sorted global indices in 15-bit fields (graded-lex order of
  // the keys = graded-lex order of sorted index tuples, reading R18)
  auto key = [](const int *a, int k) {
    uint64_t v = (uint64_t)k << 60;
    for (int i = 0; i < k; ++i) v |= (uint64_t)a[i] << (45 - 15 * i);
    return v;
  };
  std::vector<uint64_t> keys;
  std::vector<int> cl(q);
  for (int k = 0; k < t; ++k) {
    for (int i = 0; i < q; ++i) cl[i] = (q - 2) * k + i;  // clique x_k, 0-based
    int a[4];
    keys.push_back(key(a, 0));
    for (int i0 = 0; i0 < q; ++i0) {
      a[0] = cl[i0];
      keys.push_back(key(a, 1));
      for (int i1 = i0 + 1; i1 < q; ++i1) {
        a[1] = cl[i1];
        keys.push_back(key(a, 2));
        for (int i2 = i1 + 1; i2 < q; ++i2) {
          a[2] = cl[i2];
          keys.push_back(key(a, 3));
          for (int i3 = i2 + 1; i3 < q; ++i3) {
            a[3] = cl[i3];
            keys.push_back(key(a, 4));
          }
        }
      }
    }
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  auto id_of = [&](const int *a, int k) {
    return (int32_t)(std::lower_bound(keys.begin(), keys.end(), key(a, k)) - keys.begin());
  };
  cudaSetDevice(ctx->device);
  Problem P;  // staged
  P.nblk = t;
  P.nb = nb;
  P.n = nb * t;
  P.m = (int64_t)keys.size();
  P.h_amap.assign((size_t)P.n * nb, 0);
  P.h_b.assign(P.m, 0.0);
  std::vector<int> bs(nb * 2, -1), bk(nb, 0);
  for (int k = 0; k < t; ++k) {
    // block basis v(x_k), graded-lex (P:466 per clique): [], [i], [i, j] over the clique's variables
    int64_t u = 1;
    for (int i = 0; i < q; ++i, ++u) {
      bs[2 * u] = (q - 2) * k + i;
      bk[u] = 1;
    }
    for (int i = 0; i < q; ++i)
      for (int j = i + 1; j < q; ++j, ++u) {
        bs[2 * u] = (q - 2) * k + i;
        bs[2 * u + 1] = (q - 2) * k + j;
        bk[u] = 2;
      }
    for (int64_t i = 0; i < nb; ++i)
      for (int64_t j = i; j < nb; ++j) {
        int a[4], kk = 0, ia = 0, ja = 0;
        const int *A = &bs[2 * i], *B = &bs[2 * j];
        const int ka = bk[i], kb = bk[j];
        while (ia < ka || ja < kb) {  // symmetric difference of two sorted sets
          if (ja >= kb || (ia < ka && A[ia] < B[ja])) a[kk++] = A[ia++];
          else if (ia >= ka || B[ja] < A[ia]) a[kk++] = B[ja++];
          else {
            ++ia;
            ++ja;
          }
        }
        const int32_t id = id_of(a, kk);
        P.h_amap[((size_t)k * nb + i) * nb + j] = id;
        P.h_amap[((size_t)k * nb + j) * nb + i] = id;
      }
    // b: coefficients of x_k^T Q_k x_k + c_k^T x_k mod (x^2 - 1), summed over cliques
    const double *Qk = Q + (size_t)k * q * q;
    for (int i = 0; i < q; ++i) P.h_b[0] += Qk[i * q + i];
    for (int i = 0; i < q; ++i) {
      int a[1] = {(q - 2) * k + i};
      P.h_b[id_of(a, 1)] += c[(size_t)k * q + i];
    }
    for (int i = 0; i < q; ++i)
      for (int j = i + 1; j < q; ++j) {
        int a[2] = {(q - 2) * k + i, (q - 2) * k + j};
        P.h_b[id_of(a, 2)] += 2.0 * Qk[i * q + j];
      }
  }
  return finalize_problem(ctx, P, nullptr);
}

int drsdp_get_block_sizes(drsdp_ctx *ctx, int32_t *nblk, int32_t *nb) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "no problem set");
  if (nblk) *nblk = (int32_t)ctx->prob.nblk;
  if (nb) *nb = (int32_t)(ctx->prob.nblk ? ctx->prob.nb : ctx->prob.n);
  return DRSDP_OK;
}

int drsdp_get_sizes(drsdp_ctx *ctx, int64_t *n, int64_t *m, int64_t *n_upper) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "no problem set");
  if (n) *n = ctx->prob.n;
  if (m) *m = ctx->prob.m;
  if (n_upper) *n_upper = ctx->prob.n_upper;
  return DRSDP_OK;
}

int drsdp_export_index_map(drsdp_ctx *ctx, int32_t *amap, int64_t *seg_ptr, uint32_t *seg_pos) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "no problem set");
  Problem &P = ctx->prob;
  if (amap) std::memcpy(amap, P.h_amap.data(), sizeof(int32_t) * P.h_amap.size());
  if (seg_ptr) std::memcpy(seg_ptr, P.h_seg_ptr.data(), sizeof(int64_t) * P.h_seg_ptr.size());
  if (seg_pos) std::memcpy(seg_pos, P.h_seg_pos.data(), sizeof(uint32_t) * P.h_seg_pos.size());
  return DRSDP_OK;
}

int drsdp_default_params(drsdp_params *o) {
  if (!o) return DRSDP_ERR_INVALID_ARG;
  std::memset(o, 0, sizeof(*o));
  o->sigma0 = 1.0;
  o->sigma_min = 1e-3;
  o->sigma_max = 1e7;
  o->gamma = 2.0;
  o->tau1 = 0.1;
  o->tau2 = 1.0;
  o->tol = 1e-8;
  o->eig_neg_tol = 1e-9;
  o->rank_tol = 1e-4;
  o->eps_scale = 1e-2;
  o->eps_floor = 1e-12;
  o->time_limit_s = 0.0;
  o->p0 = 2;
  o->max_outer = 300;
  o->max_rtr = 500;
  o->max_tcg = 100;
  o->escape_max = 8;
  o->mode = 0;
  o->seed = 0;
  o->rho_reg = 1e3;
  o->stall_rtr = 10;
  o->precond_mu = -1.0;  // auto (reading R35)
  o->stall_factor = 100.0;
  o->escape_gate = 0.0;
  o->hold_max = 0;
  o->hold_tau = 0.0;
  o->sigma_boost = 0.0;
  return DRSDP_OK;
}

int drsdp_set_params(drsdp_ctx *ctx, const drsdp_params *prm) {
  if (!ctx || !prm) return DRSDP_ERR_INVALID_ARG;
  const drsdp_params &q = *prm;
  if (!(q.sigma0 > 0 && q.sigma_min > 0 && q.sigma_max > q.sigma_min && q.gamma > 1 && q.tau1 > 0 &&
        q.tau2 >= q.tau1 && q.tol > 0 && q.p0 >= 1 && q.p0 <= DRSDP_MAX_P && q.max_outer >= 1 && q.max_rtr >= 1 &&
        q.escape_max >= 0 && (q.mode == 0 || q.mode == 1) && q.rank_tol > 0 && q.eig_neg_tol >= 0 &&
        q.rho_reg >= 0 && q.stall_rtr >= 0 && q.stall_factor > 0 && q.eig_method >= 0 && q.eig_method <= 2 &&
        q.escape_gate >= 0 && q.hold_max >= 0 && q.hold_tau >= 0 && q.sigma_boost >= 0))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_params: parameter out of range");
  ctx->prm = q;
  return DRSDP_OK;
}

int drsdp_set_initial_factor(drsdp_ctx *ctx, int32_t p, const double *Y0) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "set_initial_factor before set_problem");
  if (p < 1 || p > DRSDP_MAX_P || !Y0)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_initial_factor: need 1 <= p <= DRSDP_MAX_P");
  const int64_t n = ctx->prob.n;
  ctx->h_Y0.assign(Y0, Y0 + (size_t)n * p);
  for (int64_t i = 0; i < n; ++i) {
    double s = 0;
    for (int c = 0; c < p; ++c) s += ctx->h_Y0[i * p + c] * ctx->h_Y0[i * p + c];
    if (!(s > 0)) return set_error(ctx, DRSDP_ERR_NUMERIC, "set_initial_factor: zero row");
    const double inv = 1.0 / std::sqrt(s);
    for (int c = 0; c < p; ++c) ctx->h_Y0[i * p + c] *= inv;
  }
  ctx->p0_given = p;
  return DRSDP_OK;
}

int drsdp_set_subproblem_matrix(drsdp_ctx *ctx, int64_t n, const double *M_dev, int64_t ldm) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (n <= 0 || n > (1 << 30) || !M_dev || ldm < n || ((uintptr_t)M_dev & 7))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "set_subproblem_matrix: need n > 0, ldm >= n, 8B-aligned M");
  cudaSetDevice(ctx->device);
  ctx->sub_M = M_dev;
  ctx->sub_n = n;
  ctx->sub_ldm = ldm;
  ctx->sub_rows_mode = false;
  ctx->sub_row0 = 0;
  ctx->sub_nloc = n;
  ctx->sub_cached_valid = false;
  CK(ctx->sub_rho.ensure(n), "alloc rho");
  int rc = ensure_red(ctx, 1184, 2);
  if (rc) return rc;
  KL(fro2_launch((int)n, M_dev, ldm, ctx->red_part.ptr, ctx->counters + C_FRO, ctx->d_scal + S_MM, ctx->stream),
     "fro2");
  // cost extra = [||M||^2, 0]
  KL(combine_launch(ctx->d_scal + S_MM, 1.0, nullptr, 0.0, 0.0, ctx->d_scal + S_EXTRA, ctx->stream), "combine");
  KL(combine_launch(nullptr, 0.0, nullptr, 0.0, 0.0, ctx->d_scal + S_EXTRA + 1, ctx->stream), "combine");
  return DRSDP_OK;
}

int drsdp_set_subproblem_rows(drsdp_ctx *ctx, int64_t n, int64_t row0, int64_t row1, const double *M_rows_dev,
                              int64_t ldm) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (n <= 0 || n > (1 << 30) || row0 < 0 || row1 <= row0 || row1 > n || !M_rows_dev || ldm < n || (ldm & 1) ||
      ((uintptr_t)M_rows_dev & 15))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG,
                     "set_subproblem_rows: need 0 <= row0 < row1 <= n, ldm >= n even, 16 B aligned rows");
  cudaSetDevice(ctx->device);
  const int64_t nloc = row1 - row0;
  ctx->sub_M = M_rows_dev;
  ctx->sub_n = n;
  ctx->sub_ldm = ldm;
  ctx->sub_rows_mode = true;
  ctx->sub_row0 = row0;
  ctx->sub_nloc = nloc;
  ctx->sub_cached_valid = false;
  CK(ctx->sub_rho.ensure(n), "alloc rho");
  int rc = ensure_red(ctx, 1184, 2);
  if (rc) return rc;
  // ||M_rows||_F^2 over the block (nloc rows of n columns): the block's share of the cost constant
  KL(fro2_rows_launch(nloc, n, M_rows_dev, ldm, ctx->red_part.ptr, ctx->counters + C_FRO, ctx->d_scal + S_MM,
                      ctx->stream),
     "fro2");
  KL(combine_launch(ctx->d_scal + S_MM, 1.0, nullptr, 0.0, 0.0, ctx->d_scal + S_EXTRA, ctx->stream), "combine");
  KL(combine_launch(nullptr, 0.0, nullptr, 0.0, 0.0, ctx->d_scal + S_EXTRA + 1, ctx->stream), "combine");
  KL(combine_launch(nullptr, 0.0, nullptr, 0.0, 0.0, ctx->d_scal + S_ZERO, ctx->stream), "combine");
  return DRSDP_OK;
}

int drsdp_subproblem_eval(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *Y_dev, const double *U_dev,
                          double *cost_dev, double *egrad_dev, double *rgrad_dev, double *hvp_dev) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->sub_M) return set_error(ctx, DRSDP_ERR_STATE, "subproblem_eval before set_subproblem_matrix");
  if (p < 1 || p > DRSDP_MAX_P || !Y_dev || (flags & ~3) || !flags)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "subproblem_eval: need 1 <= p <= DRSDP_MAX_P, flags in {1,2,3}");
  if ((flags & DRSDP_EVAL_HVP) && (!U_dev || !hvp_dev))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "subproblem_eval: HVP needs U and hvp");
  if ((flags & DRSDP_EVAL_HVP) && !(flags & DRSDP_EVAL_COSTGRAD) &&
      !(ctx->sub_cached_valid && ctx->sub_cached_Y == Y_dev && ctx->sub_cached_p == p))
    return set_error(ctx, DRSDP_ERR_STATE, "HVP needs a prior COSTGRAD at the same Y");
  const int n = (int)ctx->sub_n;
  CK(ctx->sub_G.ensure((size_t)2 * p * p), "alloc G");
  CK(ctx->sub_K.ensure((size_t)p * p), "alloc K");
  int rc = eval_fixed(ctx, flags, n, p, ctx->sub_M, ctx->sub_ldm, Y_dev, p, U_dev, cost_dev, egrad_dev, rgrad_dev,
                      hvp_dev, ctx->sub_G.ptr, ctx->sub_K.ptr, ctx->sub_rho.ptr, ctx->d_scal + S_EXTRA, false);
  if (rc) return rc;
  if (flags & DRSDP_EVAL_COSTGRAD) {
    ctx->sub_cached_valid = true;
    ctx->sub_cached_Y = Y_dev;
    ctx->sub_cached_p = p;
  }
  return DRSDP_OK;
}

int drsdp_subproblem_eval_host(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *Y, const double *U,
                               double *cost, double *egrad, double *rgrad, double *hvp) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->sub_M) return set_error(ctx, DRSDP_ERR_STATE, "subproblem_eval_host before set_subproblem_matrix");
  if (p < 1 || p > DRSDP_MAX_P || !Y || (flags & ~3) || !flags || ((flags & DRSDP_EVAL_HVP) && !U))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "subproblem_eval_host: bad arguments");
  cudaSetDevice(ctx->device);
  const size_t np = (size_t)ctx->sub_n * p;
  DBuf<double> &buf = ctx->host_stage;
  CK(buf.ensure(5 * np + 8), "alloc host-eval buffers");
  double *dY = buf.ptr, *dU = dY + np, *dE = dU + np, *dR = dE + np, *dH = dR + np, *dC = dH + np;
  CK(cudaMemcpyAsync(dY, Y, np * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D Y");
  if (flags & DRSDP_EVAL_HVP) CK(cudaMemcpyAsync(dU, U, np * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D U");
  int rc = drsdp_subproblem_eval(ctx, flags | DRSDP_EVAL_COSTGRAD, p, dY, dU, dC, egrad ? dE : nullptr, dR,
                                 (flags & DRSDP_EVAL_HVP) ? dH : nullptr);
  if (rc) return rc;
  if (cost) CK(cudaMemcpyAsync(cost, dC, 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H cost");
  if (egrad) CK(cudaMemcpyAsync(egrad, dE, np * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H egrad");
  if (rgrad) CK(cudaMemcpyAsync(rgrad, dR, np * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H rgrad");
  if (hvp && (flags & DRSDP_EVAL_HVP)) CK(cudaMemcpyAsync(hvp, dH, np * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H hvp");
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  ctx->sub_cached_valid = false;  // device scratch Y is not the caller's pointer
  return DRSDP_OK;
}

int drsdp_assemble_M(drsdp_ctx *ctx, const double *y_dev, const double *T_dev, int64_t ldt, double sigma,
                     double *M_dev, int64_t ldm) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "assemble_M before set_problem");
  Problem &P = ctx->prob;
  if (P.nblk > 0) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "assemble_M: dense problems only (fixed-M reading)");
  if (!y_dev || !T_dev || !M_dev || ldt < P.n || ldm < P.n || !(sigma > 0))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "assemble_M: bad arguments");
  int rc = ensure_red(ctx, 1184, 2);
  if (rc) return rc;
  AssembleArgs as;
  as.n = (int)P.n;
  as.amap = P.amap.ptr;
  as.ldmap = P.ld;
  as.y = y_dev;
  as.C = P.has_C ? P.C.ptr : nullptr;
  as.ldc = P.ld;
  as.T = T_dev;
  as.ldt = ldt;
  as.sigma = sigma;
  as.M = M_dev;
  as.ldm = ldm;
  as.part = ctx->red_part.ptr;
  as.counter = ctx->counters + C_ASM;
  as.scal_out = ctx->d_scal + S_M0;
  KL(assemble_launch(as, ctx->stream), "assemble kernel");
  return DRSDP_OK;
}

int drsdp_y_update(drsdp_ctx *ctx, int32_t p, const double *Y_dev, double *y_dev) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "y_update before set_problem");
  if (p < 1 || !Y_dev || !y_dev) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "y_update: bad arguments");
  Problem &P = ctx->prob;
  int rc = ensure_red(ctx, segsum_blocks(P.m, P.n_large, P.n_huge), 2);
  if (rc) return rc;
  SegArgs s = seg_args(ctx, p, Y_dev, nullptr, p, y_dev);
  KL(segsum_launch(s, false, ctx->stream), "segsum kernel");
  return DRSDP_OK;
}

int drsdp_dual_update(drsdp_ctx *ctx, int32_t p, const double *Y_dev, const double *y_dev, double sigma,
                      double *T_dev, int64_t ldt, double *z_dev, double *scalars_dev) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "dual_update before set_problem");
  Problem &P = ctx->prob;
  if (p < 1 || p > DRSDP_MAX_P || !Y_dev || !y_dev || !T_dev || ldt < (P.nblk ? P.nb : P.n) || !z_dev ||
      !scalars_dev)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "dual_update: bad arguments");
  const int n = (int)P.n;
  int rc = ensure_red(ctx, std::max(dual_update_blocks(n), P.nblk ? blk_elem_blocks((int)P.nblk, (int)P.nb) : 0), 3);
  if (rc) return rc;
  rc = ensure_workspace(ctx, n, p);
  if (rc) return rc;
  if (P.nblk > 0) {
    rc = blk_dual(ctx, p, Y_dev, p, y_dev, sigma, T_dev, ldt);
    if (rc) return rc;
  } else {
  DualArgs da;
  da.n = n;
  da.p = p;
  da.Y = Y_dev;
  da.ldy = p;
  da.amap = P.amap.ptr;
  da.ldmap = P.ld;
  da.y = y_dev;
  da.C = P.has_C ? P.C.ptr : nullptr;
  da.ldc = P.ld;
  da.sigma = sigma;
  da.T = T_dev;
  da.ldt = ldt;
  da.part = ctx->red_part.ptr;
  da.counter = ctx->counters + C_DUAL;
  da.scal_out = ctx->d_scal + S_DUAL;
  KL(dual_update_launch(da, ctx->stream), "dual update kernel");
  }
  rc = rowdot_product(ctx, n, p, T_dev, ldt, Y_dev, p, z_dev, ctx->d_scal + S_ZSUM);
  if (rc) return rc;
  KL(vdot_launch(P.m, y_dev, P.b.ptr, ctx->red_part.ptr, ctx->counters + C_DOT, ctx->d_scal + S_BY, ctx->stream),
     "vdot");
  // scalars: [||R||, b^T y, <C,T> + sum z, ||T||^2]
  KL(combine_launch(nullptr, 0, nullptr, 0, 0, scalars_dev, ctx->stream), "combine");
  CK(cudaMemcpyAsync(ctx->h_scal + S_DUAL, ctx->d_scal + S_DUAL, 8 * 10, cudaMemcpyDeviceToHost, ctx->stream),
     "read");
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  double h[4] = {std::sqrt(ctx->h_scal[S_DUAL]), ctx->h_scal[S_BY], ctx->h_scal[S_DUAL + 2] + ctx->h_scal[S_ZSUM],
                 ctx->h_scal[S_DUAL + 1]};
  CK(cudaMemcpyAsync(scalars_dev, h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream), "write scalars");
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  return DRSDP_OK;
}

int drsdp_alm_eval(drsdp_ctx *ctx, int32_t flags, int32_t p, const double *T_dev, int64_t ldt, double sigma,
                   const double *Y_dev, const double *U_dev, double *cost_dev, double *egrad_dev, double *rgrad_dev,
                   double *hvp_dev) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "alm_eval before set_problem");
  Problem &P = ctx->prob;
  if (p < 1 || p > DRSDP_MAX_P || !Y_dev || !T_dev || ldt < (P.nblk ? P.nb : P.n) || !(sigma > 0) || (flags & ~3) ||
      !flags)
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "alm_eval: bad arguments");
  if ((flags & DRSDP_EVAL_HVP) && (!U_dev || !hvp_dev))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "alm_eval: HVP needs U and hvp");
  const int n = (int)P.n;
  const size_t gmul = P.nblk > 0 ? (size_t)P.nblk : 1;  // one G, K per block
  if (P.nblk > 0 && (p > kBlkMaxP || ldt < P.nb))
    return set_error(ctx, DRSDP_ERR_INVALID_ARG, "alm_eval: block problems need p <= 128 and ldt >= nb");
  CK(ctx->alm_M.ensure((size_t)n * P.ld), "alloc M");
  CK(ctx->alm_yS.ensure(P.m), "alloc yS");
  CK(ctx->alm_wZ.ensure(P.m), "alloc wZ");
  CK(ctx->alm_rho.ensure(n), "alloc rho");
  CK(ctx->alm_G.ensure((size_t)2 * p * p * gmul), "alloc G");
  CK(ctx->alm_K.ensure((size_t)p * p * gmul), "alloc K");
  int rc;
  if (flags & DRSDP_EVAL_COSTGRAD) {
    CK(ctx->alm_D.ensure((size_t)n * P.ld), "alloc dense S");
    rc = alm_costgrad(ctx, p, T_dev, ldt, sigma, Y_dev, p, ctx->alm_M.ptr, P.ld, ctx->alm_yS.ptr, ctx->alm_G.ptr,
                      ctx->alm_rho.ptr, cost_dev, egrad_dev, rgrad_dev, ctx->alm_D.ptr);
    if (rc) return rc;
    ctx->alm_cached_valid = true;
    ctx->alm_cached_Y = Y_dev;
    ctx->alm_cached_T = T_dev;
    ctx->alm_cached_p = p;
    ctx->alm_cached_sigma = sigma;
  } else if (!(ctx->alm_cached_valid && ctx->alm_cached_Y == Y_dev && ctx->alm_cached_T == T_dev &&
               ctx->alm_cached_p == p && ctx->alm_cached_sigma == sigma)) {
    return set_error(ctx, DRSDP_ERR_STATE, "HVP needs a prior COSTGRAD at the same Y, T, sigma");
  }
  if (flags & DRSDP_EVAL_HVP) {
    CK(ctx->alm_Z.ensure((size_t)n * P.ld), "alloc dense Z");
    rc = alm_hvp(ctx, p, ctx->alm_M.ptr, P.ld, Y_dev, p, U_dev, ctx->alm_G.ptr, ctx->alm_K.ptr, ctx->alm_rho.ptr,
                 ctx->alm_wZ.ptr, hvp_dev, ctx->alm_Z.ptr);
    if (rc) return rc;
  }
  return DRSDP_OK;
}

}  // extern "C"
