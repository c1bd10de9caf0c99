// blocks.cu — multi-block (clique-chain) relaxation kernels, SURVEY §8(f) row f2.
// PAPER.md:434-436 (Algorithm 2 on multi-block SDPs) and P:555-602 (DSDP-sparse): every block
// S_k = Y_k Y_k^T is an n_b x n_b moment matrix (n_b = 211 at q = 20), the y of a monomial is
// shared by the blocks it appears in. The blocks are small (t = 120 blocks of 211 rows: 43 MB of
// M, L2-resident), so the kernels are latency/L2-bound batched operations: one CTA per block or
// per 16-32-row strip of a block, operands staged in shared memory, FP64 FMA (a 211-wide
// contraction per output; DMMA fragments would not pay at these sizes). Reductions are fixed-order
// (bit-reproducible). See blocks.cuh for the stacked layout.
#include <algorithm>

#include "blocks.cuh"
#include "common.cuh"
#include "tile_epilogue.cuh"

namespace drsdp {

// ------------------------------------------------------------------------------------------------
// per-block Gram (P:239 per block): G_k = Y_k^T Y_k, K_k = U_k^T Y_k + Y_k^T U_k
// ------------------------------------------------------------------------------------------------
constexpr int BG_MAXO = 16;  // outputs per thread; a CTA covers 256 * 16 entries of G_k (grid.y chunks)
// rows of Y_k (and U_k) staged per step: as many as fit 64 KB (one step for p <= 16 at n_b = 211),
// so that few dependent load rounds are paid per block
inline int bg_rows(int nb, int p, bool u) { return std::max(16, std::min(nb, 8192 / (p * (u ? 2 : 1)))); }

__global__ void __launch_bounds__(256) blk_gram_kernel(int nb, int p, const double *__restrict__ Y, int ldy,
                                                       const double *__restrict__ U, int ldu, double *__restrict__ G,
                                                       double *__restrict__ K, const int *skip, int BG_ROWS) {
  if (skip && *(volatile const int *)skip) return;
  extern __shared__ double sm[];
  double *ys = sm;
  double *us = sm + BG_ROWS * p;
  const int k = blockIdx.x;
  const int64_t r0 = (int64_t)k * nb;
  const int pp = p * p;
  const int o0 = blockIdx.y * 256 * BG_MAXO;
  constexpr int MAXO = BG_MAXO;
  double g[MAXO], kk[MAXO];
#pragma unroll
  for (int q = 0; q < MAXO; ++q) g[q] = kk[q] = 0.0;
  for (int i0 = 0; i0 < nb; i0 += BG_ROWS) {
    const int rows = min(BG_ROWS, nb - i0);
    __syncthreads();
    for (int t = threadIdx.x; t < rows * p; t += blockDim.x) {
      const int i = t / p, c = t - i * p;
      ys[t] = Y[(r0 + i0 + i) * ldy + c];
      if (U) us[t] = U[(r0 + i0 + i) * ldu + c];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < MAXO; ++q) {
      const int o = o0 + threadIdx.x + 256 * q;
      if (o < pp) {
        const int a = o / p, b = o - a * p;
        double s = g[q], s2 = kk[q];
        for (int i = 0; i < rows; ++i) {
          const double ya = ys[i * p + a], yb = ys[i * p + b];
          s = fma(ya, yb, s);
          if (U) s2 = fma(us[i * p + a], yb, fma(ya, us[i * p + b], s2));
        }
        g[q] = s;
        kk[q] = s2;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < MAXO; ++q) {
    const int o = o0 + threadIdx.x + 256 * q;
    if (o < pp) {
      if (G) G[(size_t)k * pp + o] = g[q];
      if (K && U) K[(size_t)k * pp + o] = kk[q];
    }
  }
}

cudaError_t blk_gram_launch(int t, int nb, int p, const double *Y, int ldy, const double *U, int ldu, double *G,
                            double *K, const int *skip, cudaStream_t st) {
  if (p > kBlkMaxP) return cudaErrorInvalidValue;
  const int rows = bg_rows(nb, p, U != nullptr);
  const size_t smem = sizeof(double) * rows * p * (U ? 2 : 1);
  static bool attr = false;  // bg_rows keeps the staging <= 64 KB: opt in once
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(blk_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid(t, (p * p + 256 * BG_MAXO - 1) / (256 * BG_MAXO));
  blk_gram_kernel<<<grid, 256, smem, st>>>(nb, p, Y, ldy, U, ldu, G, K, skip, rows);
  return cudaGetLastError();
}

__global__ void blk_gsum_kernel(int t, int p, const double *__restrict__ G, double *__restrict__ out) {
  const int pp = p * p;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < pp; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < t; ++k) s += G[(size_t)k * pp + o];
    out[o] = s;
  }
}

cudaError_t blk_gsum_launch(int t, int p, const double *G, double *out, cudaStream_t st) {
  blk_gsum_kernel<<<(p * p + 255) / 256, 256, 0, st>>>(t, p, G, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// elementwise block work with S tiles: ALM assembly (M(S) = A*(y(S)) - T/sigma and the accurate
// cost sums, reading R29) and the dual update (Alg. 2 step 6: T <- T - sigma (A*(y) - S))
// 32 x 64 tile of one block per CTA; thread (tx, ty) owns column tx and rows ty + 4q (q < 8).
// ------------------------------------------------------------------------------------------------
constexpr int BE_R = 32, BE_C = 64, BE_PC = 32;

template <int MODE>
__global__ void __launch_bounds__(256) blk_elem_kernel(BlkElemArgs a) {
  __shared__ double yr[BE_R][BE_PC + 1];
  __shared__ double yc[BE_C][BE_PC + 1];
  __shared__ double scratch[64];
  const int k = blockIdx.z;
  const int i0 = blockIdx.y * BE_R, j0 = blockIdx.x * BE_C;
  const int64_t b0 = (int64_t)k * a.nb;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  double s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  if (a.D) {  // S tiles already written by blk_tile (the segmented sum's input)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = i0 + ty + 4 * q, j = j0 + tx;
      if (i < a.nb && j < a.nb) s[q] = a.D[(b0 + i) * a.ldd + j];
    }
  }
  for (int c0 = 0; c0 < (a.D ? 0 : a.p); c0 += BE_PC) {
    const int pc = min(BE_PC, a.p - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < BE_R * BE_PC; t += 256) {
      const int i = t / BE_PC, c = t - i * BE_PC;
      yr[i][c] = (i0 + i < a.nb && c < pc) ? a.Y[(b0 + i0 + i) * a.ldy + c0 + c] : 0.0;
    }
    for (int t = threadIdx.x; t < BE_C * BE_PC; t += 256) {
      const int j = t / BE_PC, c = t - j * BE_PC;
      yc[j][c] = (j0 + j < a.nb && c < pc) ? a.Y[(b0 + j0 + j) * a.ldy + c0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < pc; ++c) {
      const double v = yc[tx][c];
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] = fma(yr[ty + 4 * q][c], v, s[q]);
    }
  }
  double v3[3] = {0.0, 0.0, 0.0};
  const int j = j0 + tx;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + ty + 4 * q;
    if (i < a.nb && j < a.nb) {
      const int64_t r = b0 + i;
      const double yv = __ldg(a.y + a.amap[r * a.ldm + j]);
      const double tv = a.T[r * a.ldt + j];
      if (MODE == BLK_ASM) {
        a.M[r * a.ldmo + j] = yv - tv / a.sigma;
        const double rr = s[q] - yv;
        v3[0] = fma(rr, rr, v3[0]);
        v3[1] = fma(tv, s[q], v3[1]);
        v3[2] = fma(tv, tv, v3[2]);
      } else {
        const double rr = yv - s[q];
        const double tn = tv - a.sigma * rr;
        a.T[r * a.ldt + j] = tn;
        v3[0] = fma(rr, rr, v3[0]);
        v3[1] = fma(tn, tn, v3[1]);
      }
    }
  }
  grid_sum<3>(v3, a.part, a.counter, a.scal_out, scratch);
}

// dense block tiles for the segmented sums (the block analogue of gram_tile.cu): D_k = Y_k Y_k^T
// (full block: the assembly reads it back) or Z_k = Y_k U_k^T + U_k Y_k^T (upper tiles only: the
// segmented sum reads upper positions), stacked rows, pitch ldd
constexpr int BT_PC = 16;  // p chunk of the tile kernel (4 staged operands: 26 KB of static shared memory)

template <bool ZM>
__global__ void __launch_bounds__(256) blk_tile_kernel(int nb, int p, const double *__restrict__ Y,
                                                       const double *__restrict__ U, int ldy, double *__restrict__ D,
                                                       int64_t ldd, const int *skip) {
  if (skip && *(volatile const int *)skip) return;
  const int i0 = blockIdx.y * BE_R, j0 = blockIdx.x * BE_C;
  if (ZM && j0 + BE_C <= i0) return;  // tile entirely below the diagonal
  __shared__ double yr[BE_R][BT_PC + 1];
  __shared__ double yc[BE_C][BT_PC + 1];
  __shared__ double ur[ZM ? BE_R : 1][BT_PC + 1];
  __shared__ double uc[ZM ? BE_C : 1][BT_PC + 1];
  const int64_t b0 = (int64_t)blockIdx.z * nb;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  double s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  for (int c0 = 0; c0 < p; c0 += BT_PC) {
    const int pc = min(BT_PC, p - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < BE_R * BT_PC; t += 256) {
      const int i = t / BT_PC, c = t - i * BT_PC;
      const bool ok = i0 + i < nb && c < pc;
      yr[i][c] = ok ? Y[(b0 + i0 + i) * ldy + c0 + c] : 0.0;
      if (ZM) ur[i][c] = ok ? U[(b0 + i0 + i) * ldy + c0 + c] : 0.0;
    }
    for (int t = threadIdx.x; t < BE_C * BT_PC; t += 256) {
      const int j = t / BT_PC, c = t - j * BT_PC;
      const bool ok = j0 + j < nb && c < pc;
      yc[j][c] = ok ? Y[(b0 + j0 + j) * ldy + c0 + c] : 0.0;
      if (ZM) uc[j][c] = ok ? U[(b0 + j0 + j) * ldy + c0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < pc; ++c) {
      const double v = yc[tx][c];
      const double w = ZM ? uc[tx][c] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s[q] = fma(yr[ty + 4 * q][c], ZM ? w : v, s[q]);
        if (ZM) s[q] = fma(ur[ty + 4 * q][c], v, s[q]);
      }
    }
  }
  const int j = j0 + tx;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + ty + 4 * q;
    if (i < nb && j < nb) D[(b0 + i) * ldd + j] = s[q];
  }
}

cudaError_t blk_tile_launch(int t, int nb, int p, const double *Y, const double *U, int ldy, double *D, int64_t ldd,
                            const int *skip, cudaStream_t st) {
  dim3 grid((nb + BE_C - 1) / BE_C, (nb + BE_R - 1) / BE_R, t);
  if (U)
    blk_tile_kernel<true><<<grid, 256, 0, st>>>(nb, p, Y, U, ldy, D, ldd, skip);
  else
    blk_tile_kernel<false><<<grid, 256, 0, st>>>(nb, p, Y, nullptr, ldy, D, ldd, skip);
  return cudaGetLastError();
}

int blk_elem_blocks(int t, int nb) { return t * ((nb + BE_R - 1) / BE_R) * ((nb + BE_C - 1) / BE_C); }

cudaError_t blk_elem_launch(const BlkElemArgs &a, int mode, cudaStream_t st) {
  dim3 grid((a.nb + BE_C - 1) / BE_C, (a.nb + BE_R - 1) / BE_R, a.t);
  if (mode == BLK_ASM)
    blk_elem_kernel<BLK_ASM><<<grid, 256, 0, st>>>(a);
  else
    blk_elem_kernel<BLK_DUAL><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

__global__ void blk_initd_kernel(int64_t total, int nb, const int32_t *__restrict__ amap, int64_t ldm,
                                 const double *__restrict__ b, const int32_t *__restrict__ cnt, double *__restrict__ T,
                                 int64_t ldt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / nb;
    const int j = (int)(e - r * nb);
    const int32_t id = amap[r * ldm + j];
    T[r * ldt + j] = b[id] / (double)cnt[id];
  }
}

cudaError_t blk_initd_launch(int t, int nb, const int32_t *amap, int64_t ldm, const double *b, const int32_t *cnt,
                             double *T, int64_t ldt, cudaStream_t st) {
  const int64_t total = (int64_t)t * nb * nb;
  blk_initd_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(total, nb, amap, ldm, b,
                                                                                          cnt, T, ldt);
  return cudaGetLastError();
}

__global__ void blk_makex_kernel(int64_t total, int nb, const double *__restrict__ T, int64_t ldt,
                                 const double *__restrict__ z, double *__restrict__ X) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / nb;  // global row = k nb + i
    const int j = (int)(e - r * nb);
    const int i = (int)(r % nb);
    // column-major block k: element (i, j) at X[k nb^2 + j nb + i]; X symmetric, so the row-major
    // element index e = (k nb + i) nb + j addresses element (j, i) = (i, j)
    X[e] = T[r * ldt + j] - (i == j ? z[r] : 0.0);
  }
}

cudaError_t blk_makex_launch(int t, int nb, const double *T, int64_t ldt, const double *z, double *X, cudaStream_t st) {
  const int64_t total = (int64_t)t * nb * nb;
  blk_makex_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(total, nb, T, ldt, z, X);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// block-diagonal product + row epilogue
// ------------------------------------------------------------------------------------------------
// One CTA per 32-row strip of a block; 8 warps = 4 row groups of 8 rows x 2 column halves. The
// strip of A (and, for the HVP, the gathered strip W = w[amap]) and the block's rows of V (and X)
// are staged per 32-wide k-chunk in padded shared memory; every warp runs fp64 DMMA (m8n8k4) on its
// 8 x PT/2 output slice (2 shared-memory fragment loads per 8 x 8 x 4 step instead of 4 loads per
// scalar FMA pair), then the shared row epilogue runs on the finished strip.
constexpr int BP_J = 32, BP_LDA = BP_J + 4;
// rows per strip: 32 (4 row groups x 2 column halves), 16 at PT = 128 (2 row groups x 4 column
// quarters) so that two CTAs fit an SM
template <int PT>
constexpr int bp_rows() { return PT >= 128 ? 16 : 32; }

template <int PT, int EPI, bool GATHER>
__global__ void __launch_bounds__(256) blk_product_kernel(SymvArgs a, int nb, int nstrip) {
  if (a.skip && *(volatile const int *)a.skip) return;
  extern __shared__ double sm[];
  constexpr int BP_R = bp_rows<PT>();
  constexpr int RG = BP_R / 8, CG = 8 / RG;  // warps across rows / columns
  constexpr bool GSG = PT > 64;  // wide p: G_k, K_k read from global memory in the epilogue
  constexpr bool NEEDG = (EPI == EPI_COSTGRAD || EPI == EPI_HVP) && !GSG;
  constexpr int LDV = PT + 4;
  constexpr int NCB = PT / (8 * CG);  // 8-column DMMA blocks per warp (each warp owns PT / CG columns)
  const int p = a.p;
  double *gs = sm;                                        // 2 p^2 (G, K)
  double *ptile = gs + (NEEDG ? 2 * p * p : 0);           // BP_R x PT
  double *As = ptile + BP_R * PT;                         // BP_R x BP_LDA
  double *Vs = As + BP_R * BP_LDA;                        // BP_J x LDV
  double *Ws = Vs + BP_J * LDV;                           // BP_R x BP_LDA (gather)
  double *Xs = Ws + (GATHER ? BP_R * BP_LDA : 0);         // BP_J x LDV (gather)
  __shared__ double scratch[64];
  __shared__ unsigned s_ticket;
  const int tile = blockIdx.x;
  const int k = tile / nstrip, st = tile - k * nstrip;
  const int64_t b0 = (int64_t)k * nb;
  const int li0 = st * BP_R;
  const int rows = min(BP_R, nb - li0);
  const int64_t r0 = b0 + li0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane >> 2, r = lane & 3;
  const int rg = warp % RG, ch = warp / RG;
  const int arow = rg * 8 + q, vcol = ch * (PT / CG) + q;
  double acc[NCB][2];
#pragma unroll
  for (int cb = 0; cb < NCB; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
  for (int j0 = 0; j0 < nb; j0 += BP_J) {
    const int jn = min(BP_J, nb - j0);
    __syncthreads();
    for (int e = threadIdx.x; e < BP_R * BP_J; e += 256) {
      const int i = e / BP_J, jj = e - i * BP_J;
      const bool ok = i < rows && jj < jn;
      As[i * BP_LDA + jj] = ok ? a.A[(r0 + i) * a.lda + j0 + jj] : 0.0;
      if constexpr (GATHER) Ws[i * BP_LDA + jj] = ok ? __ldg(a.w + a.amap[(r0 + i) * a.ldm + j0 + jj]) : 0.0;
    }
    for (int e = threadIdx.x; e < BP_J * PT; e += 256) {
      const int jj = e / PT, c = e - jj * PT;
      const bool ok = jj < jn && c < p;
      Vs[jj * LDV + c] = ok ? a.V[(b0 + j0 + jj) * a.ldv + c] : 0.0;
      if constexpr (GATHER) Xs[jj * LDV + c] = ok ? a.X[(b0 + j0 + jj) * a.ldx + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BP_J; kk += 4) {
      const double af = As[arow * BP_LDA + kk + r];
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) dmma_884(acc[cb][0], acc[cb][1], af, Vs[(kk + r) * LDV + vcol + 8 * cb]);
      if constexpr (GATHER) {
        const double wf = Ws[arow * BP_LDA + kk + r];
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) dmma_884(acc[cb][0], acc[cb][1], wf, Xs[(kk + r) * LDV + vcol + 8 * cb]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int cb = 0; cb < NCB; ++cb) {
    const int col = ch * (PT / CG) + 8 * cb + 2 * r;
    ptile[arow * PT + col] = acc[cb][0];
    ptile[arow * PT + col + 1] = acc[cb][1];
  }
  SymvArgs al = a;
  if constexpr (EPI == EPI_COSTGRAD || EPI == EPI_HVP) {
    al.G = a.G + (size_t)k * p * p;
    if (a.K) al.K = a.K + (size_t)k * p * p;
  }
  __syncthreads();
  tile_epilogue<PT, EPI, BP_R, 256, GSG>(al, ptile, gs, scratch, &s_ticket, tile, (int)r0, 0, (int)(b0 + nb), p);
}

int blk_product_tiles(int t, int nb) { return t * ((nb + 15) / 16); }  // upper bound over the strip heights

template <int PT, int EPI, bool GATHER>
static cudaError_t launch_bp(const SymvArgs &a, int t, int nb, cudaStream_t st) {
  constexpr bool NEEDG = (EPI == EPI_COSTGRAD || EPI == EPI_HVP) && PT <= 64;
  constexpr int BP_R = bp_rows<PT>();
  const int nstrip = (nb + BP_R - 1) / BP_R;
  const size_t smem = sizeof(double) * ((NEEDG ? 2 * a.p * a.p : 0) + BP_R * PT + BP_R * BP_LDA + BP_J * (PT + 4) +
                                        (GATHER ? BP_R * BP_LDA + BP_J * (PT + 4) : 0));
  auto kern = blk_product_kernel<PT, EPI, GATHER>;
  static size_t attr_smem = 0;  // per instantiation: opt in once for the largest size seen
  if (smem > 48 * 1024 && smem > attr_smem) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem = smem;
  }
  kern<<<t * nstrip, 256, smem, st>>>(a, nb, nstrip);
  return cudaGetLastError();
}

template <int PT>
static cudaError_t launch_bp_pt(const SymvArgs &a, int epi, bool gather, int t, int nb, cudaStream_t st) {
  switch (epi) {
    case EPI_COSTGRAD:
      return launch_bp<PT, EPI_COSTGRAD, false>(a, t, nb, st);
    case EPI_HVP:
      return gather ? launch_bp<PT, EPI_HVP, true>(a, t, nb, st) : launch_bp<PT, EPI_HVP, false>(a, t, nb, st);
    case EPI_ROWDOT:
      return launch_bp<PT, EPI_ROWDOT, false>(a, t, nb, st);
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t blk_product_launch(const SymvArgs &a, int epi, bool gather, int t, int nb, cudaStream_t st) {
  if (a.p <= 16) return launch_bp_pt<16>(a, epi, gather, t, nb, st);
  if (a.p <= 32) return launch_bp_pt<32>(a, epi, gather, t, nb, st);
  if (a.p <= 64) return launch_bp_pt<64>(a, epi, gather, t, nb, st);
  if (a.p <= 128) return launch_bp_pt<128>(a, epi, gather, t, nb, st);
  return cudaErrorInvalidValue;
}

}  // namespace drsdp
