// tile_epilogue.cuh — the row epilogue shared by the product kernels (symv_tma.cu, symv_symm.cu):
// on a finished 128-row tile of P = M V (shared memory, [rows][PT]) it computes, warp per row:
//   EPI_RAW       out = P (column chunk c0)
//   EPI_ROWDOT    z_j = <P_j, y_j>                                   (Alg. 2 step 7)
//   EPI_COSTGRAD  E = 4 (y G - P), rho = <E, y>, R = E - rho y      (Eq. 4.6, Lemma 4.1)
//   EPI_HVP       H = P_y(4 (u G + y K - P)) - rho u                (Eq. 4.7)
// then the tile scalars, summed over tiles in tile order by the last tile (atomic ticket).
#pragma once
#include "common.cuh"
#include "symv.cuh"

namespace drsdp {

// GS_GLOBAL: read G (and K) from global memory (L1/L2) instead of staging them in shared memory
// (wide p, where 2 p^2 doubles exceed the shared-memory budget)
template <int PT, int EPI, int BMR, int NTH, bool GS_GLOBAL = false>
DRSDP_DEV void tile_epilogue(const SymvArgs &a, const double *ptile, double *gs_smem, double *scratch,
                             unsigned *s_ticket, int tile, int j0, int c0, int n, int p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NWARPS = NTH / 32;
  constexpr int CPL = (PT + 31) / 32;
  if constexpr (!GS_GLOBAL && (EPI == EPI_COSTGRAD || EPI == EPI_HVP || EPI == EPI_BOTH)) {
    for (int t = threadIdx.x; t < p * p; t += NTH) gs_smem[t] = a.G[t];
    if constexpr (EPI == EPI_HVP || EPI == EPI_BOTH)
      for (int t = threadIdx.x; t < p * p; t += NTH) gs_smem[p * p + t] = a.K[t];
  }
  const double *gs = GS_GLOBAL ? a.G : gs_smem;
  __syncthreads();
  double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0;
  if constexpr (EPI == EPI_BOTH) {
    // P = M Y in columns [0, p), Q = M U in columns [p, 2p) of the tile row; p <= PT / 2
    constexpr int CP = (PT / 2 + 31) / 32;
    const double *ks = gs + p * p;
    for (int jj = warp; jj < BMR; jj += NWARPS) {
      const int j = j0 + jj;
      if (j >= n) break;
      double pv[CP], qv[CP], yv[CP], uv[CP];
#pragma unroll
      for (int h = 0; h < CP; ++h) {
        const int c = lane + 32 * h;
        pv[h] = (c < p) ? ptile[jj * PT + c] : 0.0;
        qv[h] = (c < p) ? ptile[jj * PT + p + c] : 0.0;
        yv[h] = (c < p) ? a.Y[(size_t)j * a.ldy + c] : 0.0;
        uv[h] = (c < p) ? a.U[(size_t)j * a.ldu + c] : 0.0;
      }
      double yg[CP], acc2[CP];
#pragma unroll
      for (int h = 0; h < CP; ++h) yg[h] = acc2[h] = 0.0;
      for (int k = 0; k < p; ++k) {
        const double yk = __shfl_sync(0xffffffffu, yv[k >> 5], k & 31);
        const double uk = __shfl_sync(0xffffffffu, uv[k >> 5], k & 31);
#pragma unroll
        for (int h = 0; h < CP; ++h) {
          const int c = lane + 32 * h;
          if (c < p) {
            yg[h] = fma(yk, gs[k * p + c], yg[h]);
            acc2[h] = fma(yk, ks[k * p + c], fma(uk, gs[k * p + c], acc2[h]));
          }
        }
      }
      // COSTGRAD part (same arithmetic as EPI_COSTGRAD)
      double e[CP], py = 0.0, ey = 0.0;
#pragma unroll
      for (int h = 0; h < CP; ++h) {
        e[h] = 4.0 * (yg[h] - pv[h]);
        py += pv[h] * yv[h];
        ey += e[h] * yv[h];
      }
      py = warp_sum(py);
      const double rho = warp_sum(ey);
      double rr = 0.0;
#pragma unroll
      for (int h = 0; h < CP; ++h) {
        const int c = lane + 32 * h;
        const double rv = e[h] - rho * yv[h];
        rr += rv * rv;
        if (c < p) {
          if (a.out) a.out[(size_t)j * a.ldo + c] = rv;
          if (a.egrad) a.egrad[(size_t)j * a.lde + c] = e[h];
        }
      }
      rr = warp_sum(rr);
      // HVP part (same arithmetic as EPI_HVP) with this row's rho
      double eh[CP], ehy = 0.0;
#pragma unroll
      for (int h = 0; h < CP; ++h) {
        eh[h] = 4.0 * (acc2[h] - qv[h]);
        ehy += eh[h] * yv[h];
      }
      ehy = warp_sum(ehy);
      double uh = 0.0;
#pragma unroll
      for (int h = 0; h < CP; ++h) {
        const int c = lane + 32 * h;
        const double hv = eh[h] - ehy * yv[h] - rho * uv[h];
        uh += uv[h] * hv;
        if (c < p) a.out2[(size_t)j * a.ldo2 + c] = hv;
      }
      uh = warp_sum(uh);
      if (lane == 0) {
        if (a.rho_out) a.rho_out[j] = rho;
        sc0 += py;
        sc1 += rr;
        sc2 += uh;
      }
    }
  }
  for (int jj = warp; jj < (EPI == EPI_BOTH ? 0 : BMR); jj += NWARPS) {
    const int j = j0 + jj;
    if (j >= n) break;
    double pv[CPL], yv[CPL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      const int c = lane + 32 * h;
      pv[h] = (c < p) ? ptile[jj * PT + c] : 0.0;
      yv[h] = 0.0;
      if constexpr (EPI != EPI_RAW) yv[h] = (c < p) ? a.Y[(size_t)j * a.ldy + c] : 0.0;
    }
    if constexpr (EPI == EPI_RAW) {
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        const int c = lane + 32 * h;
        if (c < p) a.out[(size_t)j * a.ldo + c0 + c] = pv[h];
      }
    } else if constexpr (EPI == EPI_ROWDOT) {
      double d = 0.0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) d += pv[h] * yv[h];
      d = warp_sum(d);
      if (lane == 0) a.zout[j] = d;
      sc0 += (lane == 0) ? d : 0.0;
    } else if constexpr (EPI == EPI_COSTGRAD) {
      double yg[CPL];
#pragma unroll
      for (int h = 0; h < CPL; ++h) yg[h] = 0.0;
      for (int k = 0; k < p; ++k) {
        const double yk = __shfl_sync(0xffffffffu, yv[k >> 5], k & 31);
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          const int c = lane + 32 * h;
          if (c < p) yg[h] = fma(yk, gs[k * p + c], yg[h]);
        }
      }
      double e[CPL], py = 0.0, ey = 0.0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        e[h] = 4.0 * (yg[h] - pv[h]);
        py += pv[h] * yv[h];
        ey += e[h] * yv[h];
      }
      py = warp_sum(py);
      const double rho = warp_sum(ey);
      double rr = 0.0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        const int c = lane + 32 * h;
        const double rv = e[h] - rho * yv[h];
        rr += rv * rv;
        if (c < p) {
          if (a.out) a.out[(size_t)j * a.ldo + c] = rv;
          if (a.egrad) a.egrad[(size_t)j * a.lde + c] = e[h];
        }
      }
      rr = warp_sum(rr);
      if (lane == 0) {
        if (a.rho_out) a.rho_out[j] = rho;
        sc0 += py;
        sc1 += rr;
      }
    } else if constexpr (EPI == EPI_HVP) {
      double uv[CPL];
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        const int c = lane + 32 * h;
        uv[h] = (c < p) ? a.U[(size_t)j * a.ldu + c] : 0.0;
      }
      double acc2[CPL];
#pragma unroll
      for (int h = 0; h < CPL; ++h) acc2[h] = 0.0;
      const double *ks = GS_GLOBAL ? a.K : gs + p * p;
      for (int k = 0; k < p; ++k) {
        const double yk = __shfl_sync(0xffffffffu, yv[k >> 5], k & 31);
        const double uk = __shfl_sync(0xffffffffu, uv[k >> 5], k & 31);
#pragma unroll
        for (int h = 0; h < CPL; ++h) {
          const int c = lane + 32 * h;
          if (c < p) acc2[h] = fma(yk, ks[k * p + c], fma(uk, gs[k * p + c], acc2[h]));
        }
      }
      double eh[CPL], ehy = 0.0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        eh[h] = 4.0 * (acc2[h] - pv[h]);
        ehy += eh[h] * yv[h];
      }
      ehy = warp_sum(ehy);
      const double rho = a.rho[j];
      double uh = 0.0;
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        const int c = lane + 32 * h;
        const double hv = eh[h] - ehy * yv[h] - rho * uv[h];
        uh += uv[h] * hv;
        if (c < p) a.out[(size_t)j * a.ldo + c] = hv;
      }
      uh = warp_sum(uh);
      if (lane == 0) sc0 += uh;
    }
  }
  if constexpr (EPI == EPI_RAW) return;
  // tile scalars (2 per tile; 3 for EPI_BOTH)
  constexpr int NS = EPI == EPI_BOTH ? 3 : 2;
  double v[NS];
  v[0] = sc0;
  v[1] = sc1;
  if constexpr (NS == 3) v[2] = sc2;
  __syncthreads();
  block_sum<NS>(v, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) a.tile_scal[NS * tile + k] = v[k];
    __threadfence();
    *s_ticket = atomicAdd(a.glob_cnt, 1u);
  }
  __syncthreads();
  if (*s_ticket != gridDim.x - 1) return;
  __threadfence();
  // tile scalars: thread t sums tiles t, t + blockDim, ... then a fixed-order block reduction
  double tv[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) tv[k] = 0.0;
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NS; ++k) tv[k] += __ldcg(a.tile_scal + NS * t + k);
  }
  block_sum<NS>(tv, scratch);
  if (threadIdx.x == 0) {
    const double t0 = tv[0], t1 = tv[1];
    if (a.scal_out) {
      a.scal_out[0] = t0;
      a.scal_out[1] = t1;
    }
    if constexpr (EPI == EPI_BOTH) {
      if (a.scal_out2) a.scal_out2[0] = tv[NS - 1];
    }
    if constexpr (EPI == EPI_COSTGRAD || EPI == EPI_BOTH) {
      if (a.cost_out) a.cost_out[0] = a.gg[0] - 2.0 * t0 + a.cost_extra[0] + a.cost_extra[1];
    }
    *a.glob_cnt = 0u;
  }
}

}  // namespace drsdp
