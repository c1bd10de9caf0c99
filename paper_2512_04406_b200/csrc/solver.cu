// solver.cu — Algorithm 2 (ManiDSDP) driven from the host: the ADMM/ALM outer
// loop, the Riemannian trust-region inner solver with truncated CG, saddle escape
// (Thm 4.5), rank adaptation (reading R15) and the sigma rule (Eq. 5.1).
// All vector and matrix work runs in the device kernels on the context stream; the host reads
// back a handful of scalars per tCG iteration. The eigen-decomposition of X (step 9, P:329,
// and eta_d) uses cuSOLVER dsyevd (library call).
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "ctx.h"
#include "kernels.cuh"
#include "lanczos.cuh"
#include "blocks.cuh"
#include "symv.cuh"
#include "nvtx_ranges.h"

namespace drsdp {

#define CK(call, what)                       \
  do {                                       \
    int _rc = cuda_check(ctx, (call), what); \
    if (_rc) return _rc;                     \
  } while (0)
#define KL(call, what)                       \
  do {                                       \
    ctx->launches++;                         \
    int _rc = cuda_check(ctx, (call), what); \
    if (_rc) return _rc;                     \
  } while (0)
#define RC(call)          \
  do {                    \
    int _rc = (call);     \
    if (_rc) return _rc;  \
  } while (0)

struct Point {
  double *Y = nullptr, *R = nullptr, *M = nullptr, *G = nullptr, *rho = nullptr, *yS = nullptr;
  double *D = nullptr;  // dense S = Y Y^T (upper tiles) for the tensor-core segmented sums
  double f = 0.0, gn = 0.0;
};

struct SolverState {
  int64_t n = 0, m = 0, ld = 0;
  int ldp = 0;  // pitch of the n x p vectors: a multiple of 64 >= p, grown with the rank (grow_pitch)
  DBuf<double> Ybuf[2], Rbuf[2], Mbuf[2], Gbuf[2], rhobuf[2], ySbuf[2], Dbuf[2], Zbuf;
  DBuf<double> eta, eta2, Heta, Heta2, r, r2, delta, Hdelta, Uw, tmp, K, wZ;
  DBuf<double> T, X, W, ystar, z, Vst, Wsmall, Geig, Gw;
  DBuf<double> Tsave;  // X~^k + D kept while a multiplier hold is possible (reading R40)
  DBuf<double> Apre, Wpre, pwork;  // tCG preconditioner (reading R35): A = G/gbar + mu I, W = A^{-1}
  LanczosWork lz;                  // block Lanczos eigen step (lanczos.cu)
  DBuf<int> devinfo;
  DBuf<double> work, gwork;
  DBuf<TcgDev> tcg;              // device-resident tCG scalars
  TcgDev *h_tcg = nullptr;       // pinned mirror
  // tCG loop captured as a CUDA graph with a conditional WHILE node, one per current-point
  // buffer (the accepted point alternates between Ybuf[0] and Ybuf[1]) at the current p
  struct Graph {
    const double *Y = nullptr;
    int p = -1, ldp = -1;
    uint64_t epoch = 0;  // dbuf_epoch() at capture: any (re)allocation since then invalidates
    bool warm = false, failed = false;  // failed: graph capture unsupported, use batched launches
    cudaGraphExec_t exec = nullptr;
  } graphs[2];
  cudaStream_t priv = nullptr;   // private capture-capable stream used for the whole solve
  cusolverDnHandle_t sol = nullptr;
  // multi-block problems: batched eigen step (cusolverDnXsyevBatched) workspaces
  cusolverDnParams_t sparams = nullptr;
  size_t bwork_dev = 0;
  std::vector<char> bwork_host;
  DBuf<int> binfo;
  Point cur, prop;
  int p = 0;
  bool have_solution = false;
  double dual_obj = 0, primal_obj = 0;
};

void free_solver(drsdp_ctx *ctx) {
  SolverState *s = ctx->solver;
  if (!s) return;
  for (int k = 0; k < 2; ++k) {
    s->Ybuf[k].release();
    s->Rbuf[k].release();
    s->Mbuf[k].release();
    s->Gbuf[k].release();
    s->rhobuf[k].release();
    s->ySbuf[k].release();
    s->Dbuf[k].release();
  }
  s->Zbuf.release();
  DBuf<double> *bs[] = {&s->eta, &s->eta2, &s->Heta, &s->Heta2, &s->r, &s->r2, &s->delta, &s->Hdelta, &s->Uw,
                        &s->tmp, &s->K, &s->wZ, &s->T, &s->X, &s->W, &s->ystar, &s->z, &s->Vst, &s->Wsmall,
                        &s->work, &s->Geig, &s->Gw, &s->gwork, &s->Apre, &s->Wpre, &s->pwork, &s->Tsave};
  for (auto *b : bs) b->release();
  s->devinfo.release();
  s->lz.release();
  s->tcg.release();
  if (s->h_tcg) cudaFreeHost(s->h_tcg);
  for (auto &g : s->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (s->priv) cudaStreamDestroy(s->priv);
  s->binfo.release();
  if (s->sparams) cusolverDnDestroyParams(s->sparams);
  if (s->sol) cusolverDnDestroy(s->sol);
  delete s;
  ctx->solver = nullptr;
}

static double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

struct Run {
  drsdp_ctx *ctx;
  SolverState *s;
  const drsdp_params &prm;
  int n;
  double sigma = 1.0;
  int64_t costgrad = 0, hvp = 0, rtr_total = 0, tcg_total = 0, lz_steps = 0;

  int costgrad_at(Point &P, int p) {
    NvtxRange nv("drsdp:costgrad");
    ++costgrad;
    RC(alm_or_fixed_costgrad(P, p));
    RC(read_scalars(ctx, S_COST, 4));
    P.f = ctx->h_scal[S_COST];
    P.gn = std::sqrt(std::max(0.0, ctx->h_scal[S_SCAL + 1]));
    if (!std::isfinite(P.f) || !std::isfinite(P.gn)) return set_error(ctx, DRSDP_ERR_NUMERIC, "non-finite cost");
    return DRSDP_OK;
  }
  // fixed-M reading: M = A*(y^k) - C - T/sigma assembled once per outer iteration into s->X
  bool fixed_mode() const { return prm.mode == 1; }
  int alm_or_fixed_costgrad(Point &P, int p) {
    if (!fixed_mode())
      return alm_costgrad(ctx, p, s->T.ptr, s->ld, sigma, P.Y, s->ldp, P.M, s->ld, P.yS, P.G, P.rho,
                          ctx->d_scal + S_COST, nullptr, P.R, P.D);
    // fixed M lives in s->Mbuf[0] (never swapped in this mode); yS = y(S) for the outer update
    RC(eval_fixed(ctx, DRSDP_EVAL_COSTGRAD, n, p, s->Mbuf[0].ptr, s->ld, P.Y, s->ldp, nullptr, ctx->d_scal + S_COST,
                  nullptr, P.R, nullptr, P.G, nullptr, P.rho, ctx->d_scal + S_EXTRA, false));
    return DRSDP_OK;
  }
  int hvp_at(Point &P, int p, const double *U, double *H) {
    if (!fixed_mode()) return alm_hvp(ctx, p, P.M, s->ld, P.Y, s->ldp, U, P.G, s->K.ptr, P.rho, s->wZ.ptr, H, s->Zbuf.ptr);
    return eval_fixed(ctx, DRSDP_EVAL_HVP, n, p, s->Mbuf[0].ptr, s->ld, P.Y, s->ldp, U, nullptr, nullptr, nullptr, H,
                      ctx->g_scratch.ptr, s->K.ptr, P.rho, nullptr, true);
  }
  int dots(double *out3, const double *A0, const double *B0, const double *A1, const double *B1, const double *A2,
           const double *B2, int p) {
    KL(dot3_launch(n, p, s->ldp, A0, B0, A1, B1, A2, B2, ctx->red_part.ptr, ctx->counters + C_VEC,
                   ctx->d_scal + S_DOTS, ctx->stream),
       "dot3");
    RC(read_scalars(ctx, S_DOTS, 3));
    for (int k = 0; k < 3; ++k) out3[k] = ctx->h_scal[S_DOTS + k];
    return DRSDP_OK;
  }
  void swap_pts() { std::swap(s->cur, s->prop); }

  // Steihaug-Toint truncated CG (oracle/rtr.py tcg), device-resident: the scalar recurrences run
  // in tcg_update (kernels.cu). The loop body (HVP, update + stopping rules, new direction)
  // is captured once per (current point, p) into a CUDA graph whose conditional WHILE node
  // repeats it until the device flag `done` is set, so a whole tCG runs from one graph launch
  // with no host round trip. The result is left in s->eta / s->Heta and the scalars in
  // s->tcg (read back with the trust-region step's synchronisation).
  int tcg_body(int p, cudaGraphConditionalHandle cond, int use_cond) {
    Point &C = s->cur;
    TcgDev *st = s->tcg.ptr;
    RC(hvp_at(C, p, s->delta.ptr, s->Hdelta.ptr));
    KL(tcg_update_launch(n, p, s->ldp, st, s->eta.ptr, s->eta2.ptr, s->Heta.ptr, s->Heta2.ptr, s->r.ptr,
                         s->delta.ptr, s->Hdelta.ptr, C.R, ctx->red_part.ptr, ctx->counters + C_VEC,
                         ctx->d_scal + S_SCAL, cond, use_cond, ctx->stream),
       "tcg update");
    if (precond()) {
      // z = P_Y(r W) (s->r2 holds z), beta from <z, r> (reading R35)
      RC(right_product(ctx, n, p, s->r.ptr, s->ldp, s->Wpre.ptr, s->r2.ptr, s->ldp));
      KL(tcg_prec_launch(n, p, s->ldp, st, C.Y, s->r2.ptr, s->r.ptr, s->delta.ptr, ctx->red_part.ptr,
                         ctx->counters + C_VEC, 0, ctx->stream),
         "tcg prec");
    }
    KL(tcg_newdir_launch(n, p, s->ldp, st, C.Y, precond() ? s->r2.ptr : s->r.ptr, s->delta.ptr, ctx->stream),
       "tcg newdir");
    return DRSDP_OK;
  }

  // Returns DRSDP_OK with g.exec set, or DRSDP_OK with g.exec == nullptr when the graph could not
  // be built (the caller then keeps the batched launches); kernel-launch errors inside the body
  // are real errors and are returned.
  int capture_graph(SolverState::Graph &g, int p) {
    cudaGraph_t graph = nullptr, body_out = nullptr;
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    auto give_up = [&](cudaGraph_t gr) {
      if (gr) cudaGraphDestroy(gr);
      cudaGetLastError();
      g.failed = true;
      return DRSDP_OK;
    };
    if (cudaGraphCreate(&graph, 0) != cudaSuccess) return give_up(nullptr);
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) != cudaSuccess) return give_up(graph);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, graph, nullptr, 0, &cp) != cudaSuccess) return give_up(graph);
    if (cudaStreamBeginCaptureToGraph(ctx->stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed) != cudaSuccess)
      return give_up(graph);
    ctx->skip_flag = &s->tcg.ptr->done;
    int rc = tcg_body(p, h, 1);
    ctx->skip_flag = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->stream, &body_out);
    if (rc) {
      cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return give_up(graph);
    const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
      g.exec = nullptr;
      return give_up(nullptr);
    }
    return DRSDP_OK;
  }

  // reading R35: precond_mu < 0 selects mu = 0.1 for 2048 <= n < 8192 (measured: d = 80 2.5x faster,
  // d = 40 slower, d = 150 (n = 11326) not converged after 3360 s with it against 1451 s without)
  // block problems: off (reading R37; the Gram of one block is not the operator of the others)
  double mu() const {
    if (ctx->prob.nblk > 0) return 0.0;
    return prm.precond_mu >= 0.0 ? prm.precond_mu : (n >= 2048 && n < 8192 ? 0.1 : 0.0);
  }
  bool precond() const { return mu() > 0.0; }
  // W = gbar (G + mu gbar I)^{-1} at the current point: A = G/gbar + mu I (kernel), Cholesky
  // A = L L^T and W = A^{-1} by potrs on the identity (cuSOLVER, p x p); info checked with the
  // trust-region step's read-back
  int prec_matrix(int p) {
    KL(tcg_prec_matrix_launch(p, s->cur.G, mu(), s->Apre.ptr, s->Wpre.ptr, ctx->stream), "prec matrix");
    const int lw = (int)s->pwork.cap - 1;
    if (cusolverDnDpotrf(s->sol, CUBLAS_FILL_MODE_LOWER, p, s->Apre.ptr, p, s->pwork.ptr, lw, s->devinfo.ptr) !=
        CUSOLVER_STATUS_SUCCESS)
      return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDpotrf");
    if (cusolverDnDpotrs(s->sol, CUBLAS_FILL_MODE_LOWER, p, p, s->Apre.ptr, p, s->Wpre.ptr, p, s->devinfo.ptr) !=
        CUSOLVER_STATUS_SUCCESS)
      return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDpotrs");
    ctx->launches += 2;
    return DRSDP_OK;
  }

  int tcg(int p, double Delta, int max_tcg) {
    NvtxRange nv("drsdp:tcg");
    Point &C = s->cur;
    const size_t bytes = (size_t)n * s->ldp * 8;
    CK(cudaMemsetAsync(s->eta.ptr, 0, bytes, ctx->stream), "memset");
    CK(cudaMemsetAsync(s->Heta.ptr, 0, bytes, ctx->stream), "memset");
    CK(cudaMemcpyAsync(s->r.ptr, C.R, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
    CK(cudaMemsetAsync(s->delta.ptr, 0, bytes, ctx->stream), "memset");
    TcgDev *st = s->tcg.ptr;
    KL(tcg_init_launch(st, C.gn, Delta, max_tcg, precond() ? 1 : 0, ctx->stream), "tcg init");
    if (precond()) {
      // z_0 = Prec(g), delta_0 = -z_0, z_r = d_Pd = <z_0, g>
      RC(prec_matrix(p));
      RC(right_product(ctx, n, p, s->r.ptr, s->ldp, s->Wpre.ptr, s->r2.ptr, s->ldp));
      KL(tcg_prec_launch(n, p, s->ldp, st, C.Y, s->r2.ptr, s->r.ptr, s->delta.ptr, ctx->red_part.ptr,
                         ctx->counters + C_VEC, 1, ctx->stream),
         "tcg prec");
    } else {
      KL(newdir_launch(n, p, s->ldp, C.Y, s->r.ptr, 0.0, s->delta.ptr, ctx->red_part.ptr, ctx->counters + C_VEC,
                       ctx->d_scal + S_DOTS, ctx->stream),
         "newdir");
    }
    const bool graphs_ok = !ctx->prof_on && std::getenv("DRSDP_NO_GRAPH") == nullptr;
    SolverState::Graph &g = s->graphs[C.Y == s->Ybuf[0].ptr ? 0 : 1];
    if (g.Y != C.Y || g.p != p || g.ldp != s->ldp || (g.exec && g.epoch != dbuf_epoch())) {
      // a new point buffer / rank / pitch, or device memory the graph references was reallocated
      // since capture (workspaces grow with p): drop the graph and warm up again
      g.Y = C.Y;
      g.p = p;
      g.ldp = s->ldp;
      g.warm = false;
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
    if (graphs_ok && g.warm && !g.exec && !g.failed) {
      RC(capture_graph(g, p));
      g.epoch = dbuf_epoch();
    }
    if (graphs_ok && g.exec) {
      CK(cudaGraphLaunch(g.exec, ctx->stream), "graph launch");
      ctx->launches += 1;
    } else {
      // batches of iterations with one synchronisation per batch (first call at this point / p
      // warms the workspaces so that the next call can be captured)
      int batch = 4;
      for (;;) {
        ctx->skip_flag = &st->done;
        for (int b = 0; b < batch; ++b) {
          int rc = tcg_body(p, cudaGraphConditionalHandle{}, 0);
          if (rc) {
            ctx->skip_flag = nullptr;
            return rc;
          }
        }
        ctx->skip_flag = nullptr;
        CK(cudaMemcpyAsync(s->h_tcg, st, sizeof(TcgDev), cudaMemcpyDeviceToHost, ctx->stream), "read tcg state");
        CK(cudaStreamSynchronize(ctx->stream), "sync");
        if (s->h_tcg->done) break;
        batch = std::min(2 * batch, 16);
      }
      g.warm = true;
    }
    KL(tcg_finalize_launch(n, p, s->ldp, st, s->eta.ptr, s->eta2.ptr, s->Heta.ptr, s->Heta2.ptr, ctx->stream),
       "tcg finalize");
    return DRSDP_OK;
  }

  int retract_into(const double *Y, const double *V, double t, double *out, int p, bool &bad) {
    CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream), "memset");
    KL(retract_launch(n, p, s->ldp, Y, V, t, out, ctx->d_flag, ctx->stream), "retract");
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read flag");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
    bad = flag != 0;
    return DRSDP_OK;
  }

  // Riemannian trust region (oracle/rtr.py rtr); s->cur holds Y on entry, the result on exit.
  bool debug = std::getenv("DRSDP_DEBUG_RTR") != nullptr;
  // diagnostics of the last inner solve (DRSDP_VERBOSE)
  int last_exit = 0;  // 0 gradient tolerance, 1 stagnation, 2 max_rtr, 3 tiny radius
  double last_warm_t = -1.0, last_gn0 = 0.0;
  int rtr(int p, double grad_tol, bool warm, int &iters_out, int &tcg_out) {
    NvtxRange nv("drsdp:rtr");
    RC(costgrad_at(s->cur, p));
    last_warm_t = -1.0;
    if (warm) {
      double t = 1.0;
      last_warm_t = 0.0;
      for (int h = 0; h < 25; ++h) {
        bool bad = false;
        RC(retract_into(s->cur.Y, s->Uw.ptr, t, s->prop.Y, p, bad));
        if (!bad) {
          RC(costgrad_at(s->prop, p));
          if (s->prop.f < s->cur.f) {
            swap_pts();
            last_warm_t = t;
            break;
          }
        }
        t *= 0.5;
      }
    }
    last_gn0 = s->cur.gn;
    last_exit = 2;
    const double delta_bar = std::sqrt((double)n);
    double Delta = delta_bar / 8.0;
    const int max_tcg = prm.max_tcg > 0 ? prm.max_tcg : std::max(1, n * (p - 1));
    iters_out = 0;
    tcg_out = 0;
    // stagnation exit (reading R30): stop when the gradient norm has not halved within the last
    // stall_rtr trust-region iterations and is within stall_factor (100) x the tolerance
    double best_gn = s->cur.gn;
    int since_best = 0;
    for (int it = 0; it < prm.max_rtr; ++it) {
      if (s->cur.gn <= grad_tol) {
        last_exit = 0;
        break;
      }
      if (s->cur.gn <= 0.5 * best_gn) {
        best_gn = s->cur.gn;
        since_best = 0;
      } else if (prm.stall_rtr > 0 && ++since_best > prm.stall_rtr && s->cur.gn <= prm.stall_factor * grad_tol) {
        // stagnation exit only near the tolerance (reading R30): far from it the inner solve
        // keeps going (an inexact subproblem solution steers the ALM multiplier update wrongly)
        last_exit = 1;
        break;
      }
      ++iters_out;
      RC(tcg(p, Delta, max_tcg));
      // one synchronisation per trust-region iteration: model dots, retraction flag and the
      // cost / gradient norm at the trial point are read back together
      KL(dot3_launch(n, p, s->ldp, s->cur.R, s->eta.ptr, s->eta.ptr, s->Heta.ptr, nullptr, nullptr, ctx->red_part.ptr,
                     ctx->counters + C_VEC, ctx->d_scal + S_DOTS, ctx->stream),
         "dot3");
      CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream), "memset");
      KL(retract_launch(n, p, s->ldp, s->cur.Y, s->eta.ptr, 1.0, s->prop.Y, ctx->d_flag, ctx->stream), "retract");
      ++costgrad;
      RC(alm_or_fixed_costgrad(s->prop, p));
      int flag = 0;
      CK(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read flag");
      CK(cudaMemcpyAsync(s->h_tcg, s->tcg.ptr, sizeof(TcgDev), cudaMemcpyDeviceToHost, ctx->stream), "read tcg");
      int pinfo = 0;
      if (precond())
        CK(cudaMemcpyAsync(&pinfo, s->devinfo.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read info");
      RC(read_scalars(ctx, 0, S_DOTS + 3));
      if (pinfo != 0) return set_error(ctx, DRSDP_ERR_NUMERIC, "preconditioner Cholesky failed");
      if (s->h_tcg->done == 2) return set_error(ctx, DRSDP_ERR_NUMERIC, "non-finite curvature");
      const int nin = s->h_tcg->iters;
      const bool hit = s->h_tcg->hit != 0;
      tcg_out += nin;
      hvp += nin;
      ctx->launches += (int64_t)nin * 5;
      const double d3[2] = {ctx->h_scal[S_DOTS], ctx->h_scal[S_DOTS + 1]};
      if (flag) {
        Delta /= 4.0;
        continue;
      }
      s->prop.f = ctx->h_scal[S_COST];
      s->prop.gn = std::sqrt(std::max(0.0, ctx->h_scal[S_SCAL + 1]));
      if (!std::isfinite(s->prop.f) || !std::isfinite(s->prop.gn))
        return set_error(ctx, DRSDP_ERR_NUMERIC, "non-finite cost");
      double rhonum = s->cur.f - s->prop.f;
      double rhoden = -d3[0] - 0.5 * d3[1];
      const double reg = std::max(1.0, std::fabs(s->cur.f)) * 2.220446049250313e-16 * prm.rho_reg;
      rhonum += reg;
      rhoden += reg;
      const double rho = rhonum / rhoden;
      if (debug)
        std::fprintf(stderr, "  rtr %4d f=%.17e gn=%.3e Delta=%.3e tcg=%d hit=%d num=%.3e den=%.3e rho=%.4f fp=%.17e gnp=%.3e\n",
                     it, s->cur.f, s->cur.gn, Delta, nin, (int)hit, rhonum - reg, rhoden - reg, rho, s->prop.f,
                     s->prop.gn);
      if (rho < 0.25)
        Delta /= 4.0;
      else if (rho > 0.75 && hit)
        Delta = std::min(2.0 * Delta, delta_bar);
      if (rhoden >= 0 && rho > 0.1) swap_pts();
      if (Delta < 1e-300) {
        last_exit = 3;
        break;
      }
    }
    if (iters_out == 0 && s->cur.gn <= grad_tol) last_exit = 0;
    return DRSDP_OK;
  }
};

static void assign_points(SolverState *s) {
  for (int k = 0; k < 2; ++k) {
    Point &pt = k == 0 ? s->cur : s->prop;
    pt.Y = s->Ybuf[k].ptr;
    pt.R = s->Rbuf[k].ptr;
    pt.M = s->Mbuf[k].ptr;
    pt.G = s->Gbuf[k].ptr;
    pt.rho = s->rhobuf[k].ptr;
    pt.yS = s->ySbuf[k].ptr;
    pt.D = s->Dbuf[k].ptr;
  }
}

// (Re)allocate every n x ldp vector and p x p buffer for pitch ldp_new (a multiple of 64).
// With keep_cur, the current factor s->cur.Y (first p columns) survives, moved to Ybuf[0].
static int set_pitch(drsdp_ctx *ctx, int ldp_new, bool keep_cur, int p) {
  SolverState *s = ctx->solver;
  const int64_t n = s->n;
  const size_t nv = (size_t)n * ldp_new;
  DBuf<double> keep;
  if (keep_cur) {
    CK(keep.ensure(nv), "alloc");
    KL(repack_launch((int)n, p, s->ldp, s->cur.Y, p, ldp_new, keep.ptr, 0, 0, nullptr, 0, ctx->stream), "repack");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
  }
  DBuf<double> *vs[] = {&s->Ybuf[0], &s->Ybuf[1], &s->Rbuf[0], &s->Rbuf[1], &s->eta, &s->eta2, &s->Heta,
                        &s->Heta2,    &s->r,       &s->r2,      &s->delta,   &s->Hdelta, &s->Uw,  &s->tmp};
  for (auto *b : vs) b->release();
  for (auto *b : vs)
    if (!(keep_cur && b == &s->Ybuf[0])) CK(b->ensure(nv), "alloc factor-sized vectors");
  if (keep_cur) std::swap(s->Ybuf[0], keep);
  const size_t pp = (size_t)ldp_new * ldp_new;
  const size_t gmul = ctx->prob.nblk > 0 ? (size_t)ctx->prob.nblk : 1;  // block problems: one G, K per block
  for (int k = 0; k < 2; ++k) CK(s->Gbuf[k].ensure(pp * gmul), "alloc G");
  CK(s->K.ensure(pp * gmul), "alloc K");
  CK(s->Wsmall.ensure(pp), "alloc W");
  CK(s->Geig.ensure(pp), "alloc");
  CK(s->Gw.ensure(ldp_new), "alloc");
  CK(ctx->g_scratch.ensure(2 * pp * gmul), "alloc G");
  int lw = 0;
  if (cusolverDnDsyevd_bufferSize(s->sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ldp_new, s->Geig.ptr,
                                  ldp_new, s->Gw.ptr, &lw) != CUSOLVER_STATUS_SUCCESS)
    return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDsyevd_bufferSize (Gram)");
  CK(s->gwork.ensure((size_t)lw + 1), "alloc");
  CK(s->Apre.ensure(pp), "alloc");
  CK(s->Wpre.ensure(pp), "alloc");
  if (cusolverDnDpotrf_bufferSize(s->sol, CUBLAS_FILL_MODE_LOWER, ldp_new, s->Apre.ptr, ldp_new, &lw) !=
      CUSOLVER_STATUS_SUCCESS)
    return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDpotrf_bufferSize");
  CK(s->pwork.ensure((size_t)lw + 1), "alloc");
  s->ldp = ldp_new;
  assign_points(s);
  for (auto &g : s->graphs) g.p = -1;  // buffers moved: recapture
  return DRSDP_OK;
}

static int alloc_solver(drsdp_ctx *ctx, int p0) {
  if (!ctx->solver) ctx->solver = new SolverState();
  SolverState *s = ctx->solver;
  Problem &P = ctx->prob;
  s->n = P.n;
  s->m = P.m;
  s->ld = P.ld;
  if (!s->sol) {
    if (cusolverDnCreate(&s->sol) != CUSOLVER_STATUS_SUCCESS) return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnCreate");
  }
  cusolverDnSetStream(s->sol, ctx->stream);
  for (int k = 0; k < 2; ++k) {
    CK(s->Mbuf[k].ensure((size_t)P.n * P.ld), "alloc M");
    CK(s->rhobuf[k].ensure(P.n), "alloc");
    CK(s->ySbuf[k].ensure(P.m), "alloc");
    if (std::getenv("DRSDP_NO_DENSE") == nullptr) CK(s->Dbuf[k].ensure((size_t)P.n * P.ld), "alloc dense S");
  }
  if (std::getenv("DRSDP_NO_DENSE") == nullptr) CK(s->Zbuf.ensure((size_t)P.n * P.ld), "alloc dense Z");
  s->ldp = 0;
  RC(set_pitch(ctx, std::max(64, ((p0 + 63) / 64) * 64), false, 0));
  CK(s->wZ.ensure(P.m), "alloc");
  CK(s->T.ensure((size_t)P.n * P.ld), "alloc T");
  CK(s->X.ensure(P.nblk ? (size_t)P.n * P.nb : (size_t)P.n * P.n), "alloc X");
  CK(s->W.ensure(P.n), "alloc W");
  CK(s->ystar.ensure(P.m), "alloc");
  CK(s->z.ensure(P.n), "alloc");
  CK(s->devinfo.ensure(1), "alloc");
  CK(s->tcg.ensure(1), "alloc");
  if (!s->h_tcg) CK(cudaMallocHost(&s->h_tcg, sizeof(TcgDev)), "alloc pinned");
  CK(s->Vst.ensure((size_t)P.n * std::max(1, ctx->prm.escape_max)), "alloc escape vectors");
  CK(ctx->red_part.ensure((size_t)std::max<int64_t>({(int64_t)segsum_blocks(P.m, P.n_large, P.n_huge),
                                                     (int64_t)dual_update_blocks((int)P.n), rows_blocks(P.n), 1184,
                                                     P.nblk ? (int64_t)blk_elem_blocks((int)P.nblk, (int)P.nb) : 0}) *
                              4 + 64),
     "alloc red");
  if (P.nblk > 0) {
    // batched eigen step over the blocks (X_k = T_k - Diag z_k, column-major, contiguous)
    if (!s->sparams && cusolverDnCreateParams(&s->sparams) != CUSOLVER_STATUS_SUCCESS)
      return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnCreateParams");
    size_t dbytes = 0, hbytes = 0;
    if (cusolverDnXsyevBatched_bufferSize(s->sol, s->sparams, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, P.nb,
                                          CUDA_R_64F, s->X.ptr, P.nb, CUDA_R_64F, s->W.ptr, CUDA_R_64F, &dbytes, &hbytes,
                                          P.nblk) != CUSOLVER_STATUS_SUCCESS)
      return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnXsyevBatched_bufferSize");
    CK(s->work.ensure(dbytes / sizeof(double) + 2), "alloc batched eig workspace");
    s->bwork_dev = dbytes;
    s->bwork_host.resize(hbytes + 1);
    CK(s->binfo.ensure((size_t)P.nblk), "alloc info");
    return DRSDP_OK;
  }
  int lwork = 0;
  if (cusolverDnDsyevd_bufferSize(s->sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)P.n, s->X.ptr,
                                  (int)P.n, s->W.ptr, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDsyevd_bufferSize");
  CK(s->work.ensure((size_t)lwork + 1), "alloc eig workspace");
  return DRSDP_OK;
}

// gaussian rows, normalised (splitmix64 + Box-Muller), used when no initial factor was given
static void draw_initial(uint64_t seed, int64_t n, int p, std::vector<double> &Y) {
  Y.assign((size_t)n * p, 0.0);
  uint64_t st = seed * 0x9E3779B97F4A7C15ull + 0x1234567ull;
  auto next = [&]() {
    uint64_t z = (st += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  for (size_t k = 0; k < Y.size(); ++k) {
    const double u1 = ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    Y[k] = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  for (int64_t i = 0; i < n; ++i) {
    double s = 0;
    for (int c = 0; c < p; ++c) s += Y[i * p + c] * Y[i * p + c];
    s = 1.0 / std::sqrt(s);
    for (int c = 0; c < p; ++c) Y[i * p + c] *= s;
  }
}

}  // namespace drsdp

using namespace drsdp;

static int solve_impl(drsdp_ctx *ctx, drsdp_info *info);

// drsdp_solve is synchronous: it runs on a private non-blocking stream (CUDA graph capture is not
// allowed on the legacy default stream), ordered after the context stream's prior work.
extern "C" int drsdp_solve(drsdp_ctx *ctx, drsdp_info *info) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  if (!ctx->has_problem) return set_error(ctx, DRSDP_ERR_STATE, "solve before set_problem");
  cudaSetDevice(ctx->device);
  if (!ctx->solver) ctx->solver = new SolverState();
  SolverState *s = ctx->solver;
  if (!s->priv && cudaStreamCreateWithFlags(&s->priv, cudaStreamNonBlocking) != cudaSuccess)
    return set_error(ctx, DRSDP_ERR_CUDA, "stream create");
  int rc = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "sync");
  if (rc) return rc;
  cudaStream_t user = ctx->stream;
  ctx->stream = s->priv;
  rc = solve_impl(ctx, info);
  cudaError_t e = cudaStreamSynchronize(s->priv);
  ctx->stream = user;
  if (s->sol) cusolverDnSetStream(s->sol, user);
  if (rc == DRSDP_OK || rc == DRSDP_ERR_NOT_CONVERGED) {
    int rc2 = cuda_check(ctx, e, "sync");
    if (rc2) return rc2;
  }
  return rc;
}

static int solve_impl(drsdp_ctx *ctx, drsdp_info *info) {
  const double t0 = now_s();
  const bool verbose = std::getenv("DRSDP_VERBOSE") != nullptr;
  const drsdp_params &prm = ctx->prm;
  if (ctx->p0_given && ctx->h_Y0.size() != (size_t)ctx->prob.n * ctx->p0_given)
    return set_error(ctx, DRSDP_ERR_STATE, "initial factor does not match the problem size");
  int p = ctx->p0_given ? ctx->p0_given : prm.p0;
  const bool blocks = ctx->prob.nblk > 0;
  const int nblk = (int)ctx->prob.nblk, nbk = (int)ctx->prob.nb;
  // rank cap: p <= n (S has rank <= n); block problems: p <= min(128, n_b) (blocks.cuh)
  const int pcap = blocks ? std::min(kBlkMaxP, nbk) : std::min<int>(DRSDP_MAX_P, (int)ctx->prob.n);
  if (blocks && prm.mode == 1) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "block problems: ALM mode only");
  if (blocks && p > pcap) return set_error(ctx, DRSDP_ERR_INVALID_ARG, "block problems: p0 <= min(128, n_b)");
  RC(alloc_solver(ctx, p));
  SolverState *s = ctx->solver;
  Problem &P = ctx->prob;
  const int n = (int)P.n;
  RC(ensure_workspace(ctx, n, 64));
  Run run{ctx, s, prm, n};
  run.sigma = prm.sigma0;
  // Y^0
  std::vector<double> Y0;
  if (ctx->p0_given)
    Y0 = ctx->h_Y0;
  else
    draw_initial(prm.seed, n, p, Y0);
  {
    std::vector<double> pad((size_t)n * s->ldp, 0.0);
    for (int i = 0; i < n; ++i) std::memcpy(&pad[(size_t)i * s->ldp], &Y0[(size_t)i * p], sizeof(double) * p);
    CK(cudaMemcpyAsync(s->cur.Y, pad.data(), pad.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy Y0");
    CK(cudaStreamSynchronize(ctx->stream), "sync");
  }
  // T^0 = D = A*(b/cnt) (X~^0 = 0), y^0 = 0
  if (blocks)
    KL(blk_initd_launch(nblk, nbk, P.amap.ptr, P.ld, P.b.ptr, P.cnt.ptr, s->T.ptr, P.ld, ctx->stream), "init D");
  else
    KL(init_d_launch(n, P.amap.ptr, P.ld, P.b.ptr, P.cnt.ptr, s->T.ptr, P.ld, ctx->stream), "init D");
  CK(cudaMemsetAsync(s->ystar.ptr, 0, sizeof(double) * P.m, ctx->stream), "memset y");
  double b_norm = 0.0;
  for (double v : P.h_b) b_norm += v * v;
  b_norm = std::sqrt(b_norm);
  double C_norm = 0.0;
  if (P.has_C) {
    // ||C||_F from the device copy via fro2
    KL(fro2_launch(n, P.C.ptr, P.ld, ctx->red_part.ptr, ctx->counters + C_FRO, ctx->d_scal + S_MM, ctx->stream),
       "fro2");
    RC(read_scalars(ctx, S_MM, 1));
    C_norm = std::sqrt(ctx->h_scal[S_MM]);
  }
  ctx->trace.clear();
  bool warm = false;
  double eta_prev = 1.0;
  int p_max = p;
  int status = DRSDP_ERR_NOT_CONVERGED;
  double eta_p = 0, eta_d = 0, eta_g = 0, dobj = 0, pobj = 0;
  int outer = 0;
  int holds = 0;  // consecutive multiplier holds (reading R40)
  std::vector<double> lam(n);
  for (int k = 0; k < prm.max_outer; ++k) {
    outer = k + 1;
    NvtxPhase phase;  // NVTX: inner solve / multiplier update / eigen step / rank update
    phase.set("drsdp:outer/inner_solve");
    if (prm.mode == 1) {
      // fixed-M: M = A*(y^k) - C - T/sigma and ||M||^2 as the cost constant
      AssembleArgs as;
      as.n = n;
      as.amap = P.amap.ptr;
      as.ldmap = P.ld;
      as.y = s->ystar.ptr;
      as.C = P.has_C ? P.C.ptr : nullptr;
      as.ldc = P.ld;
      as.T = s->T.ptr;
      as.ldt = P.ld;
      as.sigma = run.sigma;
      as.M = s->Mbuf[0].ptr;
      as.ldm = P.ld;
      as.part = ctx->red_part.ptr;
      as.counter = ctx->counters + C_ASM;
      as.scal_out = ctx->d_scal + S_M0;
      KL(assemble_launch(as, ctx->stream), "assemble");
      KL(fro2_launch(n, s->Mbuf[0].ptr, P.ld, ctx->red_part.ptr, ctx->counters + C_FRO, ctx->d_scal + S_EXTRA,
                     ctx->stream),
         "fro2");
      KL(combine_launch(nullptr, 0, nullptr, 0, 0, ctx->d_scal + S_EXTRA + 1, ctx->stream), "combine");
    }
    const double eps_k = std::max(0.1 * std::min(1.0, eta_prev) * prm.eps_scale, prm.eps_floor);
    const double grad_tol = 4.0 * eps_k / run.sigma;
    int rtr_it = 0, tcg_it = 0;
    RC(run.rtr(p, grad_tol, warm, rtr_it, tcg_it));
    run.rtr_total += rtr_it;
    run.tcg_total += tcg_it;
    const double grad_paper = 0.5 * run.sigma * s->cur.gn;
    phase.set("drsdp:outer/multiplier_update");
    // y^{k+1} = y(S^{k+1})
    if (prm.mode == 1) {
      SegArgs sg;
      sg.m = P.m;
      sg.seg_ptr = P.seg_ptr.ptr;
      sg.seg_pos = P.seg_pos.ptr;
      sg.cnt = P.cnt.ptr;
      sg.is_large = P.is_large.ptr;
      sg.large_ids = P.large_ids.ptr;
      sg.n_large = P.n_large;
      sg.huge_ids = P.huge_ids.ptr;
      sg.n_huge = P.n_huge;
      sg.cA = P.has_C ? P.cA.ptr : nullptr;
      sg.Y = s->cur.Y;
      sg.ld = s->ldp;
      sg.p = p;
      sg.out = s->ystar.ptr;
      sg.part = ctx->red_part.ptr;
      sg.counter = ctx->counters + C_SEG;
      sg.scal_out = ctx->d_scal + S_SEGSQ;
      KL(segsum_launch(sg, false, ctx->stream), "segsum");
    } else {
      CK(cudaMemcpyAsync(s->ystar.ptr, s->cur.yS, sizeof(double) * P.m, cudaMemcpyDeviceToDevice, ctx->stream),
         "copy y");
    }
    // multiplier hold (reading R40): keep X~^k + D so that the update below can be undone when
    // X^{k+1} shows that subproblem k is not yet solved to lambda_min >= -tau_k (Thm 5.3)
    const bool can_hold = prm.hold_max > 0 && prm.hold_tau > 0.0 && holds < prm.hold_max;
    if (can_hold) {
      CK(s->Tsave.ensure((size_t)n * P.ld), "alloc T copy");
      CK(cudaMemcpyAsync(s->Tsave.ptr, s->T.ptr, sizeof(double) * (size_t)n * P.ld, cudaMemcpyDeviceToDevice,
                         ctx->stream),
         "save T");
    }
    // T <- T - sigma (A*(y) - S - C)
    DualArgs da;
    da.n = n;
    da.p = p;
    da.Y = s->cur.Y;
    da.ldy = s->ldp;
    da.amap = P.amap.ptr;
    da.ldmap = P.ld;
    da.y = s->ystar.ptr;
    da.C = P.has_C ? P.C.ptr : nullptr;
    da.ldc = P.ld;
    da.sigma = run.sigma;
    da.T = s->T.ptr;
    da.ldt = P.ld;
    da.part = ctx->red_part.ptr;
    da.counter = ctx->counters + C_DUAL;
    da.scal_out = ctx->d_scal + S_DUAL;
    if (blocks)
      RC(blk_dual(ctx, p, s->cur.Y, s->ldp, s->ystar.ptr, run.sigma, s->T.ptr, P.ld));
    else
      KL(dual_update_launch(da, ctx->stream), "dual update");
    // z = rowdot(T Y, Y)
    RC(rowdot_product(ctx, n, p, s->T.ptr, P.ld, s->cur.Y, s->ldp, s->z.ptr, ctx->d_scal + S_ZSUM));
    KL(vdot_launch(P.m, s->ystar.ptr, P.b.ptr, ctx->red_part.ptr, ctx->counters + C_DOT, ctx->d_scal + S_BY,
                   ctx->stream),
       "vdot");
    phase.set("drsdp:outer/eigen_step");
    // X = T - Diag(z) and its extreme eigenpairs: block Lanczos on
    // T V - z o V (partial decomposition) or the dense dsyevd; eta_max <= tol reported by
    // Lanczos is confirmed by one dense decomposition (the certificate never rests on Ritz values)
    RC(read_scalars(ctx, S_DUAL, 8));
    const double R_norm = std::sqrt(std::max(0.0, ctx->h_scal[S_DUAL]));
    const double CT = ctx->h_scal[S_DUAL + 2];
    const double zsum = ctx->h_scal[S_ZSUM];
    dobj = ctx->h_scal[S_BY];
    pobj = CT + zsum;
    eta_p = R_norm / (1.0 + C_norm);
    eta_g = std::fabs(dobj - pobj) / (1.0 + std::fabs(dobj) + std::fabs(pobj));
    // auto: dense below n = 16384 (measured at d = 80: Lanczos escape directions cost 162 outer
    // iterations / 65 s against 29 / 21 s with dsyevd; reading R17)
    const bool lanczos = !blocks && (prm.eig_method == 2 || (prm.eig_method == 0 && n >= 16384));
    const int nvec = std::max(1, std::min(prm.escape_max, n));
    int nlam = 0;                   // smallest eigen/Ritz values available in lam[0..nlam)
    double lam_top = 0.0;           // largest eigen/Ritz value
    const double *vec_cols = nullptr;  // escape candidates, column-major (column c at vec_cols + c n)
    bool dense_done = false;
    auto dense_eig = [&]() -> int {
      KL(make_x_launch(n, s->T.ptr, P.ld, s->z.ptr, s->X.ptr, ctx->stream), "make X");
      int lwork = (int)s->work.cap - 1;
      if (cusolverDnDsyevd(s->sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, s->X.ptr, n, s->W.ptr,
                           s->work.ptr, lwork, s->devinfo.ptr) != CUSOLVER_STATUS_SUCCESS)
        return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDsyevd");
      ctx->launches++;
      CK(cudaMemcpyAsync(lam.data(), s->W.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "read eig");
      int eig_info = 0;
      CK(cudaMemcpyAsync(&eig_info, s->devinfo.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read info");
      CK(cudaStreamSynchronize(ctx->stream), "sync");
      if (eig_info != 0)
        return set_error(ctx, DRSDP_ERR_NUMERIC,
                         "eigen-decomposition of X failed (dsyevd info " + std::to_string(eig_info) + ")");
      nlam = n;
      lam_top = lam[n - 1];
      vec_cols = s->X.ptr;
      dense_done = true;
      return DRSDP_OK;
    };
    // block problems: the spectrum of the block-diagonal X is the union of the blocks' spectra
    // (reading R38); all blocks in one batched decomposition, merged on the host in ascending
    // order (ties: lower block, then lower index first), escape vectors embedded in their rows
    std::vector<double> blk_w;  // per-block ascending eigenvalues (block k at k * n_b)
    auto block_eig = [&]() -> int {
      KL(blk_makex_launch(nblk, nbk, s->T.ptr, P.ld, s->z.ptr, s->X.ptr, ctx->stream), "make X (blocks)");
      if (cusolverDnXsyevBatched(s->sol, s->sparams, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nbk, CUDA_R_64F,
                                 s->X.ptr, nbk, CUDA_R_64F, s->W.ptr, CUDA_R_64F, s->work.ptr, s->bwork_dev,
                                 s->bwork_host.data(), s->bwork_host.size() - 1, s->binfo.ptr,
                                 nblk) != CUSOLVER_STATUS_SUCCESS)
        return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnXsyevBatched");
      ctx->launches++;
      std::vector<double> &wb = blk_w;
      wb.resize((size_t)n);
      std::vector<int> infos(nblk);
      CK(cudaMemcpyAsync(wb.data(), s->W.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "read eig");
      CK(cudaMemcpyAsync(infos.data(), s->binfo.ptr, sizeof(int) * nblk, cudaMemcpyDeviceToHost, ctx->stream),
         "read info");
      CK(cudaStreamSynchronize(ctx->stream), "sync");
      for (int k2 = 0; k2 < nblk; ++k2)
        if (infos[k2] != 0)
          return set_error(ctx, DRSDP_ERR_NUMERIC, "batched eigen-decomposition failed (block " + std::to_string(k2) + ")");
      for (int i = 0; i < n; ++i) lam[i] = wb[i];
      std::sort(lam.begin(), lam.end());
      nlam = n;
      lam_top = lam[n - 1];
      vec_cols = nullptr;
      dense_done = true;
      return DRSDP_OK;
    };
    if (blocks) {
      RC(block_eig());
    } else if (lanczos) {
      const int b = std::min(16, n);
      const int kmax = std::max(1, std::min(prm.lanczos_steps > 0 ? prm.lanczos_steps : 40, n / b));
      if (s->lz.n != n || s->lz.b != b || s->lz.kmax != kmax) {
        const int e = s->lz.ensure(n, b, kmax);
        if (e) RC(cuda_check(ctx, (cudaError_t)e, "alloc lanczos"));
      }
      LanczosResult lr;
      RC(lanczos_extreme(ctx, s->lz, s->sol, s->T.ptr, P.ld, s->z.ptr, nvec, prm.seed * 7919ull + (uint64_t)k, lr));
      nlam = std::min((int)lr.theta.size(), n);
      for (int i = 0; i < nlam; ++i) lam[i] = lr.theta[i];
      lam_top = lr.lam_max;
      run.lz_steps += lr.steps;
      // Ritz vectors of the nvec smallest Ritz values, transposed to column-major
      KL(symv_transpose(n, std::min(nvec, lr.basis), s->lz.V.ptr, std::min(nvec, lr.basis), s->Vst.ptr, n, nullptr,
                        ctx->stream),
         "transpose Ritz vectors");
      vec_cols = s->Vst.ptr;
      const double ed = std::max(0.0, -lam[0]) / (1.0 + std::fabs(lam_top));
      if (std::max(eta_p, std::max(ed, eta_g)) <= prm.tol) RC(dense_eig());  // confirm
    } else {
      RC(dense_eig());
    }
    eta_d = std::max(0.0, -lam[0]) / (1.0 + std::fabs(lam_top));
    const double eta_max = std::max(eta_p, std::max(eta_d, eta_g));
    double row[13] = {(double)(k + 1), eta_p, eta_d, eta_g, eta_max, pobj, dobj, run.sigma, (double)p,
                      (double)rtr_it, (double)tcg_it, 0.0, 0.0};
    if (verbose) {
      int nneg = 0;
      const double th = -prm.eig_neg_tol * (1.0 + std::fabs(lam_top));
      while (nneg < nlam && lam[nneg] < th) ++nneg;
      std::fprintf(stderr,
                   "[drsdp] k=%d p=%d sigma=%.3e eta_p=%.3e eta_d=%.3e eta_g=%.3e dobj=%.12f rtr=%d tcg=%d exit=%s "
                   "gn0=%.2e gn=%.2e tol=%.2e warm_t=%.2g neg=%d%s lmin=%.3e lmax=%.3e t=%.2fs\n",
                   k + 1, p, run.sigma, eta_p, eta_d, eta_g, dobj, rtr_it, tcg_it,
                   run.last_exit == 0 ? "tol" : run.last_exit == 1 ? "stall" : run.last_exit == 2 ? "maxit" : "radius",
                   run.last_gn0, s->cur.gn, grad_tol, run.last_warm_t, nneg, dense_done ? "" : "(ritz)", lam[0],
                   lam_top, now_s() - t0);
    }
    if (eta_max <= prm.tol) {
      status = DRSDP_OK;
      row[12] = now_s() - t0;
      ctx->trace.insert(ctx->trace.end(), row, row + 13);
      break;
    }
    phase.set("drsdp:outer/rank_update");
    // escape directions: eigenvectors (Ritz vectors) with lambda < -eig_neg_tol (1 + |lambda_max|)
    const double thresh = -prm.eig_neg_tol * (1.0 + std::fabs(lam_top));
    int dv = 0;
    std::vector<int> blk_neg;  // block problems: negative eigenvalues per block (reading R39)
    if (blocks) {
      blk_neg.assign(nblk, 0);
      for (int k2 = 0; k2 < nblk; ++k2) {
        while (blk_neg[k2] < nbk && blk_w[(size_t)k2 * nbk + blk_neg[k2]] < thresh) ++blk_neg[k2];
        dv = std::max(dv, std::min(prm.escape_max, blk_neg[k2]));
      }
    } else {
      while (dv < prm.escape_max && dv < nlam && dv < (dense_done ? n : nvec) && lam[dv] < thresh) ++dv;
    }
    if (dv > 0 && p + dv > pcap) dv = std::max(0, pcap - p);
    // escape gate (reading R36): the certificate X^{k+1} is the subproblem's (Prop 4.3) only at a
    // stationary point; while the inner solve ends far above its tolerance, keep the rank (no escape,
    // no reduction)
    const bool gated = prm.escape_gate > 0.0 && s->cur.gn > prm.escape_gate * grad_tol;
    if (gated) dv = 0;
    // multiplier hold (reading R40): subproblem k's certificate X^{k+1} = grad Phi_k(S^{k+1}) - Diag(z)
    // still has escape directions with eta_d above hold_tau min(1, eta_p): undo the X~ update, keep
    // sigma, escape, and re-solve subproblem k (at most hold_max times in a row)
    const bool hold = can_hold && dv > 0 && eta_d > prm.hold_tau * std::min(1.0, eta_p);
    // rank reduction (readings R15, R32, R34): only in an iteration that does not escape, compress
    // Y to its numerical rank at the tolerance rank_tol_k = min(rank_tol, max(1e-8, 0.01 sqrt(eta_max))).
    // Eigenpairs of the p x p Gram matrix G = Y^T Y (cuSOLVER dsyevd; G is symmetric so
    // row/column-major agree).
    if (dv == 0 && !gated) {
      if (blocks)
        KL(blk_gsum_launch(nblk, p, s->cur.G, s->Geig.ptr, ctx->stream), "sum block Gram");  // Y^T Y = sum_k G_k
      else
        CK(cudaMemcpyAsync(s->Geig.ptr, s->cur.G, sizeof(double) * p * p, cudaMemcpyDeviceToDevice, ctx->stream),
           "copy G");
      const int lw = (int)s->gwork.cap - 1;
      if (cusolverDnDsyevd(s->sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, s->Geig.ptr, p, s->Gw.ptr,
                           s->gwork.ptr, lw, s->devinfo.ptr) != CUSOLVER_STATUS_SUCCESS)
        return set_error(ctx, DRSDP_ERR_CUDA, "cusolverDnDsyevd (Gram)");
      ctx->launches++;
      const double rtol = std::min(prm.rank_tol, std::max(1e-8, 0.01 * std::sqrt(eta_max)));
      std::vector<double> w(p), V((size_t)p * p);
      CK(cudaMemcpyAsync(w.data(), s->Gw.ptr, sizeof(double) * p, cudaMemcpyDeviceToHost, ctx->stream), "read");
      CK(cudaMemcpyAsync(V.data(), s->Geig.ptr, sizeof(double) * p * p, cudaMemcpyDeviceToHost, ctx->stream), "read");
      int g_info = 0;
      CK(cudaMemcpyAsync(&g_info, s->devinfo.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "read info");
      CK(cudaStreamSynchronize(ctx->stream), "sync");
      if (g_info != 0)
        return set_error(ctx, DRSDP_ERR_NUMERIC, "eigen-decomposition of Y^T Y failed (dsyevd info " + std::to_string(g_info) + ")");
      int r = 0;
      for (int i = 0; i < p; ++i)
        if (w[i] > rtol * rtol * w[p - 1]) ++r;
      r = std::max(1, r);
      if (r < p) {
        // W_r = eigenvectors of the r largest eigenvalues (ascending order: the last r columns);
        // column k of the column-major result is V[k p + i]
        std::vector<double> Wr((size_t)p * r);
        for (int i = 0; i < p; ++i)
          for (int c = 0; c < r; ++c) Wr[(size_t)i * r + c] = V[(size_t)(p - r + c) * p + i];
        CK(cudaMemcpyAsync(s->Wsmall.ptr, Wr.data(), Wr.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy W");
        RC(apply_w_product(ctx, n, p, s->cur.Y, s->ldp, s->Wsmall.ptr, r, s->tmp.ptr, s->ldp));
        CK(cudaMemcpyAsync(s->cur.Y, s->tmp.ptr, (size_t)n * s->ldp * 8, cudaMemcpyDeviceToDevice, ctx->stream),
           "copy");
        CK(cudaStreamSynchronize(ctx->stream), "sync");
        p = r;
      }
    }
    if (dv > 0) {
      if (p + dv > s->ldp) RC(set_pitch(ctx, ((p + dv + 63) / 64) * 64, true, p));
      // canonical signs (largest-|.| entry positive), then Y <- [Y, 0], U <- [0, V]
      std::vector<double> Vh((size_t)n * dv, 0.0);
      if (blocks) {
        // reading R39: column c holds the c-th most negative eigenvector of every block that has one
        // (its rows only); the first dv eigenvectors of each block are contiguous in the column-major
        // X_k, so one strided copy brings them all
        std::vector<double> Vb((size_t)nblk * dv * nbk);
        CK(cudaMemcpy2DAsync(Vb.data(), sizeof(double) * dv * nbk, s->X.ptr, sizeof(double) * nbk * nbk,
                             sizeof(double) * dv * nbk, nblk, cudaMemcpyDeviceToHost, ctx->stream),
           "read V");
        CK(cudaStreamSynchronize(ctx->stream), "sync");
        for (int k2 = 0; k2 < nblk; ++k2)
          for (int c = 0; c < std::min(dv, blk_neg[k2]); ++c) {
            const double *v = &Vb[((size_t)k2 * dv + c) * nbk];
            int km = 0;
            for (int i = 1; i < nbk; ++i)
              if (std::fabs(v[i]) > std::fabs(v[km])) km = i;
            const double sg = v[km] < 0 ? -1.0 : 1.0;  // canonical sign per block (reading R25)
            for (int i = 0; i < nbk; ++i) Vh[(size_t)c * n + (size_t)k2 * nbk + i] = sg * v[i];
          }
      } else {
        CK(cudaMemcpyAsync(Vh.data(), vec_cols, sizeof(double) * n * dv, cudaMemcpyDeviceToHost, ctx->stream),
           "read V");
      }
      CK(cudaStreamSynchronize(ctx->stream), "sync");
      for (int c = 0; c < (blocks ? 0 : dv); ++c) {
        int km = 0;
        for (int i = 1; i < n; ++i)
          if (std::fabs(Vh[(size_t)c * n + i]) > std::fabs(Vh[(size_t)c * n + km])) km = i;
        if (Vh[(size_t)c * n + km] < 0)
          for (int i = 0; i < n; ++i) Vh[(size_t)c * n + i] = -Vh[(size_t)c * n + i];
      }
      CK(cudaMemcpyAsync(s->Vst.ptr, Vh.data(), Vh.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy V");
      KL(repack_launch(n, p, s->ldp, s->cur.Y, p + dv, s->ldp, s->tmp.ptr, 0, 0, nullptr, 0, ctx->stream), "repack");
      CK(cudaMemcpyAsync(s->cur.Y, s->tmp.ptr, (size_t)n * s->ldp * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy");
      KL(repack_launch(n, 0, s->ldp, nullptr, p + dv, s->ldp, s->Uw.ptr, p, dv, s->Vst.ptr, n, ctx->stream),
         "repack");
      p += dv;
      warm = true;
    } else {
      warm = false;
    }
    p_max = std::max(p_max, p);
    if (hold && !(prm.time_limit_s > 0 && now_s() - t0 > prm.time_limit_s)) {
      CK(cudaMemcpyAsync(s->T.ptr, s->Tsave.ptr, sizeof(double) * (size_t)n * P.ld, cudaMemcpyDeviceToDevice,
                         ctx->stream),
         "restore T");
      ++holds;
      row[11] = -dv;  // trace: a negative escape_delta marks a held multiplier
      row[12] = now_s() - t0;
      ctx->trace.insert(ctx->trace.end(), row, row + 13);
      if (verbose) std::fprintf(stderr, "[drsdp] k=%d hold %d (multiplier kept, %d escape columns)\n", k + 1, holds, dv);
      continue;
    }
    holds = 0;
    // sigma update, Eq. 5.1
    const double ratio = R_norm / (1.0 + b_norm);
    double sig = run.sigma;
    if (ratio < prm.tau1 * grad_paper)
      sig = std::max(run.sigma / prm.gamma, prm.sigma_min);
    else if (ratio > prm.tau2 * grad_paper)
      sig = std::min(prm.gamma * run.sigma, prm.sigma_max);
    // reading R41: the dual residue is far ahead of the primal one -> raise the penalty
    if (prm.sigma_boost > 0.0 && eta_d <= prm.sigma_boost * eta_p) sig = std::min(prm.gamma * run.sigma, prm.sigma_max);
    row[11] = dv;
    row[12] = now_s() - t0;
    ctx->trace.insert(ctx->trace.end(), row, row + 13);
    run.sigma = sig;
    eta_prev = eta_max;
    if (prm.time_limit_s > 0 && now_s() - t0 > prm.time_limit_s) break;
  }
  s->p = p;
  s->have_solution = true;
  s->dual_obj = dobj;
  s->primal_obj = pobj;
  if (info) {
    info->status = status;
    info->outer_iters = outer;
    info->p_final = p;
    info->p_max = p_max;
    info->rtr_iters = run.rtr_total;
    info->tcg_iters = run.tcg_total;
    info->n_costgrad = run.costgrad;
    info->n_hvp = run.hvp;
    info->eta_p = eta_p;
    info->eta_d = eta_d;
    info->eta_g = eta_g;
    info->dual_obj = dobj;
    info->primal_obj = pobj;
    info->seconds = now_s() - t0;
  }
  return status;
}

extern "C" int drsdp_get_solution(drsdp_ctx *ctx, double *y, double *Y, int32_t *p, double *z, double *X) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  if (ctx->sticky) return ctx->sticky;
  SolverState *s = ctx->solver;
  if (!s || !s->have_solution) return set_error(ctx, DRSDP_ERR_STATE, "no solution (call drsdp_solve first)");
  const int64_t n = s->n;
  if (p) *p = s->p;
  if (y) CK(cudaMemcpyAsync(y, s->ystar.ptr, sizeof(double) * s->m, cudaMemcpyDeviceToHost, ctx->stream), "read y");
  if (Y)
    CK(cudaMemcpy2DAsync(Y, sizeof(double) * s->p, s->cur.Y, sizeof(double) * s->ldp, sizeof(double) * s->p, n,
                         cudaMemcpyDeviceToHost, ctx->stream),
       "read Y");
  if (z) CK(cudaMemcpyAsync(z, s->z.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "read z");
  if (X) {
    const Problem &P = ctx->prob;
    if (P.nblk > 0) {
      KL(blk_makex_launch((int)P.nblk, (int)P.nb, s->T.ptr, s->ld, s->z.ptr, s->X.ptr, ctx->stream), "make X");
      CK(cudaMemcpyAsync(X, s->X.ptr, sizeof(double) * n * P.nb, cudaMemcpyDeviceToHost, ctx->stream), "read X");
    } else {
      KL(make_x_launch((int)n, s->T.ptr, s->ld, s->z.ptr, s->X.ptr, ctx->stream), "make X");
      CK(cudaMemcpyAsync(X, s->X.ptr, sizeof(double) * n * n, cudaMemcpyDeviceToHost, ctx->stream), "read X");
    }
  }
  CK(cudaStreamSynchronize(ctx->stream), "sync");
  return DRSDP_OK;
}

extern "C" int drsdp_get_trace(drsdp_ctx *ctx, int32_t max_rows, double *rows, int32_t *n_rows) {
  if (!ctx) return DRSDP_ERR_INVALID_ARG;
  const int avail = (int)(ctx->trace.size() / 13);
  if (n_rows) *n_rows = avail;
  if (rows && max_rows > 0) std::memcpy(rows, ctx->trace.data(), sizeof(double) * 13 * std::min(avail, (int)max_rows));
  return DRSDP_OK;
}
