// symv.cu — the tall-skinny symmetric product P = A V (n x n times n x p, p <= 64), fp64 on the
// DMMA tensor path (mma.sync m8n8k4 f64), deterministic split-K, fused row epilogues.
//
// North-star kernel (b)/(c) (BASELINE.json): M.Y fused with the Gram-based Euclidean gradient
// 4 (Y Y^T Y - M Y), the cost expansion, the Riemannian gradient (Lemma 4.1, Eq. 4.6, PAPER.md
// P:223-231) and the Hessian-vector product (Eq. 4.7), plus the ALM gather-product
// A*(w) Y of Eq. 4.7's projection term (fused into the same accumulators).
//
// Mapping. A is symmetric, so P[j, :] = sum_i A[i, j] V[i, :]: a CTA owns BN = 8*JB output rows j
// (a column block of A) and a contiguous range of K-rows i (split s of S). Each warp streams
// row groups of 4 (one m8n8k4 k-step) straight from HBM into DMMA A-fragments
// (a = A[i0 + (lane&3)][j0 + 8*jb + (lane>>2)]) and V rows into B-fragments; there is no shared
// memory in the main loop. Warps reduce through shared memory in fixed order, split partials go
// to a workspace and the last CTA of a column block (atomic ticket) sums them in split order and
// runs the epilogue; the last column block sums tile scalars in tile order. Bit-deterministic.
#include "common.cuh"
#include "symv.cuh"

namespace drsdp {

template <int PT, int JB, int UNR, int MODE2, int EPI, bool ATR>
__global__ void __launch_bounds__(256, 2) symv_kernel(SymvArgs a) {
  constexpr int NW = 8, BN = 8 * JB, CB = PT / 8;
  constexpr int TILE = BN * PT;
  constexpr bool GATHER = MODE2 == MODE2_GATHER, PAIR = MODE2 == MODE2_PAIR;
  if (a.skip && *(volatile const int *)a.skip) return;  // device-resident tCG finished (solver.cu)
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane & 3, q = lane >> 2;
  const int split = blockIdx.y, S = gridDim.y;
  // column chunk z covers output columns [PT z, PT z + PT) (EPI_RAW only when gridDim.z > 1)
  const int c0 = PT * blockIdx.z;
  const int tile = blockIdx.x + gridDim.x * blockIdx.z;  // workspace / ticket slot
  const int n = a.n, p = EPI == EPI_RAW ? min(PT, a.p - c0) : a.p;
  const int kext = a.k > 0 ? a.k : n;
  const int j0 = blockIdx.x * BN;
  const int kbeg = split * a.rows_per_split;
  const int kend = min(kext, kbeg + a.rows_per_split);

  double acc[JB][CB][2];
#pragma unroll
  for (int jb = 0; jb < JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) acc[jb][cb][0] = acc[jb][cb][1] = 0.0;

  bool colok[JB];
#pragma unroll
  for (int jb = 0; jb < JB; ++jb) colok[jb] = (j0 + 8 * jb + q) < n;
  bool vok[CB];
#pragma unroll
  for (int cb = 0; cb < CB; ++cb) vok[cb] = (8 * cb + q) < p;

  // A element (i, j): A[i lda + j], or A[j lda + i] when ATR (the product is then A^T-free: out = A V)
  const double *__restrict__ Ab = ATR ? a.A + (size_t)(j0 + q) * a.lda : a.A + j0 + q;
  const double *__restrict__ Vb = a.V + c0 + q;
  const int32_t *__restrict__ Mb = GATHER ? a.amap + j0 + q : nullptr;
  const double *__restrict__ Xb = GATHER ? a.X + c0 + q : nullptr;
  const double *__restrict__ A2b =
      PAIR ? (ATR ? a.A2 + (size_t)(j0 + q) * a.lda2 : a.A2 + j0 + q) : nullptr;
  const double *__restrict__ V2b = PAIR ? a.V2 + c0 + q : nullptr;

  for (int i0 = kbeg + 4 * warp; i0 < kend; i0 += 4 * NW * UNR) {
    constexpr bool TWO = MODE2 != MODE2_NONE;
    double af[UNR][JB], bf[UNR][CB];
    double gf[TWO ? UNR : 1][TWO ? JB : 1], xf[TWO ? UNR : 1][TWO ? CB : 1];
    int32_t mf[GATHER ? UNR : 1][GATHER ? JB : 1];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int i = i0 + u * 4 * NW + r;
      const bool ok = i < kend;
      const double *vrow = Vb + (size_t)i * a.ldv;
#pragma unroll
      for (int jb = 0; jb < JB; ++jb) {
        const double *ap = ATR ? Ab + (size_t)(8 * jb) * a.lda + i : Ab + (size_t)i * a.lda + 8 * jb;
        af[u][jb] = (ok && colok[jb]) ? __ldg(ap) : 0.0;
      }
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) bf[u][cb] = (ok && vok[cb]) ? __ldg(vrow + 8 * cb) : 0.0;
      if constexpr (PAIR) {
        const double *v2row = V2b + (size_t)i * a.ldv2;
#pragma unroll
        for (int jb = 0; jb < JB; ++jb) {
          const double *ap = ATR ? A2b + (size_t)(8 * jb) * a.lda2 + i : A2b + (size_t)i * a.lda2 + 8 * jb;
          gf[u][jb] = (ok && colok[jb]) ? __ldg(ap) : 0.0;
        }
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) xf[u][cb] = (ok && vok[cb]) ? __ldg(v2row + 8 * cb) : 0.0;
      }
      if constexpr (GATHER) {
        const int32_t *mrow = Mb + (size_t)i * a.ldm;
        const double *xrow = Xb + (size_t)i * a.ldx;
#pragma unroll
        for (int jb = 0; jb < JB; ++jb) mf[u][jb] = (ok && colok[jb]) ? __ldg(mrow + 8 * jb) : -1;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) xf[u][cb] = (ok && vok[cb]) ? __ldg(xrow + 8 * cb) : 0.0;
      }
    }
    if constexpr (GATHER) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int jb = 0; jb < JB; ++jb) gf[u][jb] = mf[u][jb] >= 0 ? __ldg(a.w + mf[u][jb]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int jb = 0; jb < JB; ++jb)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          dmma_884(acc[jb][cb][0], acc[jb][cb][1], af[u][jb], bf[u][cb]);
          if constexpr (TWO) dmma_884(acc[jb][cb][0], acc[jb][cb][1], gf[u][jb], xf[u][cb]);
        }
  }

  // ---- cross-warp reduction (fixed warp order) ----
  double *red = smem;  // [NW][BN][PT]
#pragma unroll
  for (int jb = 0; jb < JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      const int row = 8 * jb + q, col = 8 * cb + 2 * r;
      red[(warp * BN + row) * PT + col] = acc[jb][cb][0];
      red[(warp * BN + row) * PT + col + 1] = acc[jb][cb][1];
    }
  __syncthreads();
  constexpr int RED = (NW * TILE > 2 * PT * PT) ? NW * TILE : 2 * PT * PT;  // red / G,K region
  double *ptile = smem + RED;  // [BN][PT] final tile
  constexpr int EPT = TILE / 256;    // elements per thread (TILE is a multiple of 256)
  double part[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int idx = threadIdx.x + 256 * e;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w * TILE + idx];
    part[e] = s;
  }
  __shared__ unsigned s_ticket;
  if (S > 1) {
    double *wp = a.part + ((size_t)tile * S + split) * TILE;
#pragma unroll
    for (int e = 0; e < EPT; ++e) wp[threadIdx.x + 256 * e] = part[e];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.tile_cnt + tile, 1u);
    __syncthreads();
    if (s_ticket != (unsigned)(S - 1)) return;
    __threadfence();
    const double *rp = a.part + (size_t)tile * S * TILE;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int idx = threadIdx.x + 256 * e;
      double s = 0.0;
      s = ordered_sum(rp + idx, S, (size_t)TILE);
      ptile[idx] = s;
    }
    if (threadIdx.x == 0) a.tile_cnt[tile] = 0u;
  } else {
#pragma unroll
    for (int e = 0; e < EPT; ++e) ptile[threadIdx.x + 256 * e] = part[e];
  }
  __syncthreads();

  // ---- row epilogue on the finished tile (warp per row, lanes over columns) ----
  constexpr int CPL = (PT + 31) / 32;  // columns per lane
  double *gs = smem;                   // reuse: G (p x p) then K (p x p)
  if constexpr (EPI == EPI_COSTGRAD || EPI == EPI_HVP) {
    for (int t = threadIdx.x; t < p * p; t += 256) gs[t] = a.G[t];
    if constexpr (EPI == EPI_HVP)
      for (int t = threadIdx.x; t < p * p; t += 256) gs[p * p + t] = a.K[t];
  }
  __syncthreads();
  double sc0 = 0.0, sc1 = 0.0;
  for (int jj = warp; jj < BN; jj += NW) {
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
      const double *ks = gs + p * p;
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
  // ---- tile scalars, then the last tile reduces them in tile order ----
  double v[2] = {sc0, sc1};
  __syncthreads();
  double *scratch = smem + RED + TILE;
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) {
    a.tile_scal[2 * tile] = v[0];
    a.tile_scal[2 * tile + 1] = v[1];
    __threadfence();
    s_ticket = atomicAdd(a.glob_cnt, 1u);
  }
  __syncthreads();
  if (s_ticket != gridDim.x - 1) return;
  __threadfence();
  // tile scalars: thread t sums tiles t, t + blockDim, ... then a fixed-order block reduction
  double tv[2] = {0.0, 0.0};
  for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x) {
    tv[0] += __ldcg(a.tile_scal + 2 * t);
    tv[1] += __ldcg(a.tile_scal + 2 * t + 1);
  }
  block_sum<2>(tv, scratch);
  if (threadIdx.x == 0) {
    const double t0 = tv[0], t1 = tv[1];
    if (a.scal_out) {
      a.scal_out[0] = t0;
      a.scal_out[1] = t1;
    }
    if constexpr (EPI == EPI_COSTGRAD) {
      // f = ||G||^2 - 2 <M Y, Y> + extra (extra = ||M||^2 for the fixed-M subproblem, the ALM
      // constant terms otherwise; see kernels.cu and DESIGN.md "cost by expansion")
      if (a.cost_out) a.cost_out[0] = a.gg[0] - 2.0 * t0 + a.cost_extra[0] + a.cost_extra[1];
    }
    *a.glob_cnt = 0u;
  }
}

// ----------------------------------------------------------------------------------------------
template <int PT, int JB, int UNR, int MODE2, int EPI, bool ATR>
static cudaError_t launch_t(const SymvArgs &a, int S, cudaStream_t st) {
  constexpr int NW = 8, BN = 8 * JB;
  constexpr int TILE = BN * PT;
  constexpr int RED = (NW * TILE > 2 * PT * PT) ? NW * TILE : 2 * PT * PT;
  const size_t smem = (size_t)(RED + TILE + 64) * 8;
  auto k = symv_kernel<PT, JB, UNR, MODE2, EPI, ATR>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nz = EPI == EPI_RAW ? (a.p + PT - 1) / PT : 1;
  dim3 grid((a.n + BN - 1) / BN, S, nz);
  k<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

int symv_bn(int pt, int mode2) {
  const bool two = mode2 != MODE2_NONE;
  if (pt <= 8) return 64;
  if (pt <= 16) return two ? 32 : 64;
  if (pt <= 32) return two ? 16 : 32;
  return two ? 8 : 16;
}

int symv_pt(int p) { return p <= 8 ? 8 : p <= 16 ? 16 : p <= 32 ? 32 : 64; }

int symv_chunks(int p, int epi) { return epi == EPI_RAW ? (p + symv_pt(p) - 1) / symv_pt(p) : 1; }

template <int PT, int JB, int MODE2, bool ATR>
static cudaError_t dispatch_epi(const SymvArgs &a, int epi, int S, cudaStream_t st) {
  if constexpr (ATR || MODE2 == MODE2_PAIR) {
    if (epi != EPI_RAW) return cudaErrorInvalidValue;
    return launch_t<PT, JB, 2, MODE2, EPI_RAW, ATR>(a, S, st);
  } else if constexpr (MODE2 == MODE2_GATHER) {
    if (epi == EPI_RAW) return launch_t<PT, JB, 2, MODE2, EPI_RAW, false>(a, S, st);
    if (epi == EPI_HVP) return launch_t<PT, JB, 2, MODE2, EPI_HVP, false>(a, S, st);
    return cudaErrorInvalidValue;
  } else {
    switch (epi) {
      case EPI_RAW: return launch_t<PT, JB, 2, MODE2, EPI_RAW, false>(a, S, st);
      case EPI_COSTGRAD: return launch_t<PT, JB, 2, MODE2, EPI_COSTGRAD, false>(a, S, st);
      case EPI_HVP: return launch_t<PT, JB, 2, MODE2, EPI_HVP, false>(a, S, st);
      default: return launch_t<PT, JB, 2, MODE2, EPI_ROWDOT, false>(a, S, st);
    }
  }
}

template <int MODE2, bool ATR>
static cudaError_t dispatch_pt(const SymvArgs &a, int epi, int S, cudaStream_t st) {
  const int pt = symv_pt(a.p);
  if (epi != EPI_RAW && a.p > 64) return cudaErrorInvalidValue;  // fused epilogues need whole rows
  constexpr bool two = MODE2 != MODE2_NONE;
  if (pt == 8) return dispatch_epi<8, 8, MODE2, ATR>(a, epi, S, st);
  if (pt == 16) return dispatch_epi<16, two ? 4 : 8, MODE2, ATR>(a, epi, S, st);
  if (pt == 32) return dispatch_epi<32, two ? 2 : 4, MODE2, ATR>(a, epi, S, st);
  return dispatch_epi<64, two ? 1 : 2, MODE2, ATR>(a, epi, S, st);
}

cudaError_t symv_launch(const SymvArgs &a, int epi, int mode2, bool atr, int S, cudaStream_t st) {
  if (atr) {
    if (mode2 == MODE2_PAIR) return dispatch_pt<MODE2_PAIR, true>(a, epi, S, st);
    if (mode2 == MODE2_NONE) return dispatch_pt<MODE2_NONE, true>(a, epi, S, st);
    return cudaErrorInvalidValue;
  }
  if (mode2 == MODE2_PAIR) return dispatch_pt<MODE2_PAIR, false>(a, epi, S, st);
  if (mode2 == MODE2_GATHER) return dispatch_pt<MODE2_GATHER, false>(a, epi, S, st);
  return dispatch_pt<MODE2_NONE, false>(a, epi, S, st);
}

}  // namespace drsdp
