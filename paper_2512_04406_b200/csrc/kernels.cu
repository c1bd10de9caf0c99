// kernels.cu — the ADMM operator kernels and the manifold vector kernels (sm_100a, fp64).
//
//  gram        G = Y^T Y, K = U^T Y + Y^T U, ||G||^2            (Eq. 4.7 terms)
//  segsum      y(S) = (AA*)^{-1} A(Y Y^T + C) and A(Z)/cnt,  Z = Y U^T + U Y^T
//              deterministic CSR segmented sum over the index map (north star (d))
//  assemble    M = A*(y) - C - T/sigma, with ||C + T/sigma||^2 (north star (a))
//  dual_update T <- T - sigma (A*(y) - Y Y^T - C), ||R||, ||T||^2, <C,T>  (Alg. 2 step 6)
//  vector ops  row-normalisation retraction, the tCG new direction (tangent projection,
//              Lemma 4.1), fused inner products, escape padding (Thm 4.5)
//  row epilogues for p > 64 (cost/gradient, HVP, z), A*(w) assembly for the TMA gather-product
//  device tCG  Steihaug-Toint recurrences in device memory (tcg_init / tcg_update / tcg_newdir)
// All reductions are fixed-order (block partials + last-block sum): results are bit-identical
// from run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace drsdp {

// ----------------------------------------------------------------------------------------------
// Gram: G = Y^T Y (p x p), optional K = U^T Y + Y^T U; gg = ||G||_F^2
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gram_kernel(int n, int p, const double *__restrict__ Y, int ldy,
                                                   const double *__restrict__ U, int ldu, int rows_per_block,
                                                   double *part, unsigned *counter, double *G, double *K,
                                                   double *gg, const int *skip, int split_final) {
  if (skip && *(volatile const int *)skip) return;
  extern __shared__ double sh[];
  const int pp = p * p;
  const int nval = U ? 2 * pp : pp;
  double *ys = sh;                  // [32][p]
  double *us = sh + 32 * p;         // [32][p]
  double acc[32];                   // up to 32 entries per thread (nval <= 8192)
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  const int r0 = blockIdx.x * rows_per_block, r1 = min(n, r0 + rows_per_block);
  for (int c0 = r0; c0 < r1; c0 += 32) {
    const int cn = min(32, r1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < cn * p; t += blockDim.x) {
      const int i = t / p, c = t - i * p;
      ys[t] = Y[(size_t)(c0 + i) * ldy + c];
      if (U) us[t] = U[(size_t)(c0 + i) * ldu + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int e = threadIdx.x + k * 256;
      if (e < nval) {
        const bool isK = e >= pp;
        const int ee = isK ? e - pp : e;
        const int a = ee / p, b = ee - a * p;
        double s = acc[k];
        if (!isK) {
          for (int i = 0; i < cn; ++i) s = fma(ys[i * p + a], ys[i * p + b], s);
        } else {
          for (int i = 0; i < cn; ++i) s = fma(us[i * p + a], ys[i * p + b], fma(ys[i * p + a], us[i * p + b], s));
        }
        acc[k] = s;
      }
    }
  }
  double *mine = part + (size_t)blockIdx.x * nval;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int e = threadIdx.x + k * 256;
    if (e < nval) mine[e] = acc[k];
  }
  if (split_final) return;  // gram_final_kernel sums the partials
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  double g2 = 0.0;
  for (int e = threadIdx.x; e < nval; e += blockDim.x) {
    double s = 0.0;
    s = ordered_sum(part + e, (int)gridDim.x, (size_t)nval);
    if (e < pp) {
      G[e] = s;
      g2 += s * s;
    } else {
      K[e - pp] = s;
    }
  }
  __shared__ double scratch[64];
  double v[1] = {g2};
  block_sum<1>(v, scratch);
  if (threadIdx.x == 0) {
    if (gg) gg[0] = v[0];
    *counter = 0u;
  }
}

// second phase: one warp per entry e; lane l sums the block partials l, l + 32, ... in order and
// the warp combines the 32 lane sums with a fixed butterfly (deterministic). G / K written,
// ||G||^2 by a deterministic grid reduction. (A single last block summing nb partials per entry
// serially cost ~40 us at nb = 296: one dependent L2 round trip per partial.)
__global__ void __launch_bounds__(256) gram_final_kernel(int nval, int pp, int nb, const double *__restrict__ part,
                                                         double *G, double *K, double *gg, double *red,
                                                         unsigned *counter, const int *skip) {
  if (skip && *(volatile const int *)skip) return;
  __shared__ double scratch[8];
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  double v[1] = {0.0};
  if (e < nval) {
    double s = 0.0;
    int b = lane;
    for (; b + 96 < nb; b += 128) {
      const double t0 = __ldcg(part + (size_t)b * nval + e), t1 = __ldcg(part + (size_t)(b + 32) * nval + e);
      const double t2 = __ldcg(part + (size_t)(b + 64) * nval + e), t3 = __ldcg(part + (size_t)(b + 96) * nval + e);
      s += t0;
      s += t1;
      s += t2;
      s += t3;
    }
    for (; b < nb; b += 32) s += __ldcg(part + (size_t)b * nval + e);
    s = warp_sum(s);
    if (lane == 0) {
      if (e < pp) {
        G[e] = s;
        v[0] = s * s;
      } else {
        K[e - pp] = s;
      }
    }
  }
  grid_sum<1>(v, red, counter, gg, scratch);
}
cudaError_t gram_launch(const GramArgs &a, cudaStream_t st) {
  const int nval = a.U ? 2 * a.p * a.p : a.p * a.p;
  if (nval > 32 * 256) return cudaErrorInvalidValue;
  int nb = (a.n + 31) / 32;  // >= 32 rows per block: small n still spreads over many SMs
  if (nb > a.max_blocks) nb = a.max_blocks;
  if (nb < 1) nb = 1;
  int rpb = (a.n + nb - 1) / nb;
  nb = (a.n + rpb - 1) / rpb;
  const size_t smem = (size_t)2 * 32 * a.p * 8;
  // the partials are summed by a second kernel, one warp per entry (gram_final_kernel), unless
  // there are only a few blocks
  const int split_final = nb > 8 ? 1 : 0;
  gram_kernel<<<nb, 256, smem, st>>>(a.n, a.p, a.Y, a.ldy, a.U, a.ldu, rpb, a.part, a.counter, a.G, a.K, a.gg,
                                     a.skip, split_final);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !split_final) return e;
  double *red = a.part + (size_t)nb * nval;
  gram_final_kernel<<<(nval + 7) / 8, 256, 0, st>>>(nval, a.p * a.p, nb, a.part, a.G, a.K, a.gg, red, a.counter,
                                                    a.skip);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// Segmented sums over the index map. Upper positions (i <= j) of each constraint are stored
// CSR (constraint-major, (i, j) sorted), packed (i << 16) | j. Ordered-position sums count an
// off-diagonal upper position twice.
//   MODE_Y: out[a] = (sum_pos w_ij <y_i, y_j> + cA[a]) / cnt[a],  scalar sum_a (..)^2 / cnt[a]
//   MODE_Z: out[a] = (sum_pos w_ij (<y_i, u_j> + <u_i, y_j>)) / cnt[a]
// Small segments: one thread each (blocks [0, nb_small)); large segments: one warp each.
// ----------------------------------------------------------------------------------------------
template <bool ZMODE>
DRSDP_DEV double seg_pos_value(uint32_t pk, const double *__restrict__ Y, const double *__restrict__ U, int ld,
                               int p, const double *__restrict__ D, int64_t ldd, int nbk) {
  const int i = pk >> 16, j = pk & 0xffff;
  if (D) {
    // block problems: D is stacked (row i holds the columns of its own block of nbk rows)
    const double v = __ldg(D + (size_t)i * ldd + (nbk ? j - i / nbk * nbk : j));
    return (i == j) ? v : 2.0 * v;
  }
  const double *yi = Y + (size_t)i * ld, *yj = Y + (size_t)j * ld;
  double s = 0.0;
  if (!ZMODE) {
    for (int c = 0; c < p; ++c) s = fma(__ldg(yi + c), __ldg(yj + c), s);
  } else {
    const double *ui = U + (size_t)i * ld, *uj = U + (size_t)j * ld;
    for (int c = 0; c < p; ++c) s = fma(__ldg(yi + c), __ldg(uj + c), fma(__ldg(ui + c), __ldg(yj + c), s));
  }
  return (i == j) ? s : 2.0 * s;
}

template <bool ZMODE>
__global__ void __launch_bounds__(256) segsum_kernel(SegArgs a) {
  if (a.skip && *(volatile const int *)a.skip) return;
  __shared__ double scratch[64];
  double sq = 0.0;
  if ((int)blockIdx.x < a.nb_small) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < a.m && !a.is_large[s]) {
      const int64_t b0 = a.seg_ptr[s], b1 = a.seg_ptr[s + 1];
      double acc = 0.0;
      // up to 8 positions per step with all their loads in flight (a serial walk paid two dependent
      // L2/HBM round trips per position); the sum keeps the position order, so results are unchanged
      for (int64_t k = b0; k < b1; k += 8) {
        const int cn = (int)min((int64_t)8, b1 - k);
        uint32_t pk[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pk[u] = u < cn ? __ldg(a.seg_pos + k + u) : 0u;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = u < cn ? seg_pos_value<ZMODE>(pk[u], a.Y, a.U, a.ld, a.p, a.D, a.ldd, a.nbk) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < cn) acc += v[u];
      }
      if (!ZMODE && a.cA) acc += a.cA[s];
      a.out[s] = acc / (double)a.cnt[s];
      if (!ZMODE) sq = acc * acc / (double)a.cnt[s];
    }
  } else if ((int)blockIdx.x < a.nb_small + a.nb_large) {
    const int lane = threadIdx.x & 31;
    const int64_t li = (int64_t)(blockIdx.x - a.nb_small) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (li < a.n_large) {
      const int s = a.large_ids[li];
      const int64_t b0 = a.seg_ptr[s], b1 = a.seg_ptr[s + 1];
      double acc = 0.0;
      for (int64_t k = b0 + lane; k < b1; k += 32) acc += seg_pos_value<ZMODE>(__ldg(a.seg_pos + k), a.Y, a.U, a.ld, a.p, a.D, a.ldd, a.nbk);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (!ZMODE && a.cA) acc += a.cA[s];
        a.out[s] = acc / (double)a.cnt[s];
        if (!ZMODE) sq = acc * acc / (double)a.cnt[s];
      }
    }
  } else {
    // one block per huge segment (e.g. the constant monomial: the n diagonal positions)
    const int s = a.huge_ids[blockIdx.x - a.nb_small - a.nb_large];
    const int64_t b0 = a.seg_ptr[s], b1 = a.seg_ptr[s + 1];
    double acc[1] = {0.0};
    // 8 strided positions per thread and step with their loads in flight (multi-block problems put
    // ~10^2 diagonal positions on every thread); per-thread order unchanged
    const int64_t bs = blockDim.x;
    for (int64_t k0 = b0 + threadIdx.x; k0 < b1; k0 += 8 * bs) {
      uint32_t pk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) pk[u] = k0 + u * bs < b1 ? __ldg(a.seg_pos + k0 + u * bs) : 0u;
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = k0 + u * bs < b1 ? seg_pos_value<ZMODE>(pk[u], a.Y, a.U, a.ld, a.p, a.D, a.ldd, a.nbk) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u * bs < b1) acc[0] += v[u];
    }
    block_sum<1>(acc, scratch);
    if (threadIdx.x == 0) {
      double t = acc[0];
      if (!ZMODE && a.cA) t += a.cA[s];
      a.out[s] = t / (double)a.cnt[s];
      if (!ZMODE) sq = t * t / (double)a.cnt[s];
    }
  }
  if (ZMODE) return;
  double v[1] = {sq};
  grid_sum<1>(v, a.part, a.counter, a.scal_out, scratch);
}

cudaError_t segsum_launch(const SegArgs &a0, bool zmode, cudaStream_t st) {
  SegArgs a = a0;
  a.nb_small = (int)((a.m + 255) / 256);
  a.nb_large = (int)((a.n_large + 7) / 8);
  const int nb = a.nb_small + a.nb_large + (int)a.n_huge;
  if (zmode)
    segsum_kernel<true><<<nb, 256, 0, st>>>(a);
  else
    segsum_kernel<false><<<nb, 256, 0, st>>>(a);
  return cudaGetLastError();
}

int segsum_blocks(int64_t m, int64_t n_large, int64_t n_huge) {
  return (int)((m + 255) / 256 + (n_large + 7) / 8 + n_huge);
}

// ----------------------------------------------------------------------------------------------
// Assembly M = A*(y) - C - T/sigma (north star (a)); padding columns [n, ldm) are zeroed.
// scal_out[0] = ||C + T/sigma||_F^2 = ||M_0||^2 (the y-independent cost constant).
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) assemble_kernel(int n, const int32_t *__restrict__ amap, int64_t ldmap,
                                                       const double *__restrict__ y, const double *__restrict__ C,
                                                       int64_t ldc, const double *__restrict__ T, int64_t ldt,
                                                       double inv_sigma, double *__restrict__ M, int64_t ldm,
                                                       double *part, unsigned *counter, double *scal_out) {
  __shared__ double scratch[64];
  double s2 = 0.0;
  const int64_t total = (int64_t)n * ldm;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ldm, j = e - i * ldm;
    double v = 0.0;
    if (j < n) {
      const int32_t id = __ldg(amap + i * ldmap + j);
      const double m0 = (C ? __ldg(C + i * ldc + j) : 0.0) + __ldg(T + i * ldt + j) * inv_sigma;
      v = (id >= 0 ? __ldg(y + id) : 0.0) - m0;
      s2 = fma(m0, m0, s2);
    }
    M[e] = v;
  }
  double vv[1] = {s2};
  grid_sum<1>(vv, part, counter, scal_out, scratch);
}

cudaError_t assemble_launch(const AssembleArgs &a, cudaStream_t st) {
  assemble_kernel<<<a.blocks, 256, 0, st>>>(a.n, a.amap, a.ldmap, a.y, a.C, a.ldc, a.T, a.ldt, 1.0 / a.sigma,
                                            a.M, a.ldm, a.part, a.counter, a.scal_out);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// ALM assembly with the accurate cost (y-eliminated subproblem, reading R29):
//   S_ij = <y_i, y_j>,  M_ij = y(S)[amap_ij] - C_ij - T_ij/sigma   (written, symmetric, mirrored)
//   R_ij = S_ij + C_ij - y(S)[amap_ij]  ((I - P_A)(S + C) entry)
//   scal_out = [sum R^2, sum T (S + C), sum T^2]  so that
//   f^ = sum R^2 + (2/sigma) <T, S + C> + ||T||^2 / sigma^2.
// Upper 32x32 tiles only (T, C, amap, M symmetric); an off-diagonal tile is mirrored through
// shared memory and counted twice in the sums.
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) assemble_alm_kernel(int n, int p, const double *__restrict__ Y, int ldy,
                                                           const int32_t *__restrict__ amap, int64_t ldmap,
                                                           const double *__restrict__ y, const double *__restrict__ C,
                                                           int64_t ldc, const double *__restrict__ T, int64_t ldt,
                                                           double inv_sigma, double *__restrict__ M, int64_t ldm,
                                                           double *part, unsigned *counter, double *scal_out,
                                                           const double *__restrict__ D, int64_t ldd) {
  __shared__ double yi_s[32][33], yj_s[32][33];
  __shared__ double mt[32][33];
  __shared__ double scratch[3 * 8];
  const int I = blockIdx.y, J = blockIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  if (I <= J) {
    const int i0 = I * 32, j0 = J * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (D) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = i0 + ty + 8 * k, j = j0 + tx;
        s[k] = (i < n && j < n) ? D[(size_t)i * ldd + j] : 0.0;
      }
    }
    for (int c0 = 0; !D && c0 < p; c0 += 32) {
      const int cn = min(32, p - c0);
      __syncthreads();
      for (int t = threadIdx.x; t < 32 * 32; t += 256) {
        const int rr = t >> 5, cc = t & 31;
        yi_s[rr][cc] = (i0 + rr < n && cc < cn) ? Y[(size_t)(i0 + rr) * ldy + c0 + cc] : 0.0;
        yj_s[rr][cc] = (j0 + rr < n && cc < cn) ? Y[(size_t)(j0 + rr) * ldy + c0 + cc] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ii = ty + 8 * k;
        double acc = s[k];
        for (int c = 0; c < cn; ++c) acc = fma(yi_s[ii][c], yj_s[tx][c], acc);
        s[k] = acc;
      }
    }
    const double w = (I == J) ? 1.0 : 2.0;
    const int j = j0 + tx;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ii = ty + 8 * k, i = i0 + ii;
      double mval = 0.0;
      if (i < n && j < n) {
        const int32_t id = amap[(int64_t)i * ldmap + j];
        const double ya = id >= 0 ? y[id] : 0.0;
        const double cij = C ? C[(int64_t)i * ldc + j] : 0.0;
        const double tij = T[(int64_t)i * ldt + j];
        mval = ya - cij - tij * inv_sigma;
        M[(int64_t)i * ldm + j] = mval;
        const double sc = s[k] + cij;
        const double R = sc - ya;
        v[0] = fma(w * R, R, v[0]);
        v[1] = fma(w * tij, sc, v[1]);
        v[2] = fma(w * tij, tij, v[2]);
      }
      mt[ii][tx] = mval;
    }
    if (I != J) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int jj = ty + 8 * k;  // row of the mirrored tile = column jj of the tile
        const int jr = j0 + jj, ic = i0 + tx;
        if (jr < n && ic < n) M[(int64_t)jr * ldm + ic] = mt[tx][jj];
      }
    }
  }
  grid_sum<3>(v, part, counter, scal_out, scratch);
}

cudaError_t assemble_alm_launch(const AssembleArgs &a, int p, const double *Y, int ldy, cudaStream_t st,
                                const double *D, int64_t ldd) {
  dim3 grid((a.n + 31) / 32, (a.n + 31) / 32);
  assemble_alm_kernel<<<grid, 256, 0, st>>>(a.n, p, Y, ldy, a.amap, a.ldmap, a.y, a.C, a.ldc, a.T, a.ldt,
                                            1.0 / a.sigma, a.M, a.ldm, a.part, a.counter, a.scal_out, D, ldd);
  if (a.ldm > a.n) {
    cudaError_t e = cudaMemset2DAsync(a.M + a.n, a.ldm * sizeof(double), 0, (a.ldm - a.n) * sizeof(double), a.n, st);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// cost = s[0] + (2/sigma) s[1] + s[2] / sigma^2
__global__ void alm_cost_kernel(const double *s, double inv_sigma, double *cost) {
  if (threadIdx.x == 0) cost[0] = s[0] + 2.0 * inv_sigma * s[1] + s[2] * inv_sigma * inv_sigma;
}

cudaError_t alm_cost_launch(const double *s, double sigma, double *cost, cudaStream_t st) {
  alm_cost_kernel<<<1, 32, 0, st>>>(s, 1.0 / sigma, cost);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// Dual update (Alg. 2 step 6): R_ij = y[amap_ij] - <y_i, y_j> - C_ij ; T_ij -= sigma R_ij.
// 32x32 tiles, rows of Y for the tile staged in shared memory (p in chunks of 32).
// scal_out = [||R||_F^2, ||T_new||_F^2, <C, T_new>]
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) dual_update_kernel(int n, int p, const double *__restrict__ Y, int ldy,
                                                          const int32_t *__restrict__ amap, int64_t ldmap,
                                                          const double *__restrict__ y, const double *__restrict__ C,
                                                          int64_t ldc, double sigma, double *__restrict__ T,
                                                          int64_t ldt, double *part, unsigned *counter,
                                                          double *scal_out) {
  __shared__ double yi_s[32][33], yj_s[32][33];
  __shared__ double scratch[3 * 8];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 x 32
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int cn = min(32, p - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < 32 * 32; t += 256) {
      const int rr = t >> 5, cc = t & 31;
      yi_s[rr][cc] = (i0 + rr < n && cc < cn) ? Y[(size_t)(i0 + rr) * ldy + c0 + cc] : 0.0;
      yj_s[rr][cc] = (j0 + rr < n && cc < cn) ? Y[(size_t)(j0 + rr) * ldy + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ii = ty + 8 * k;
      double acc = s[k];
      for (int c = 0; c < cn; ++c) acc = fma(yi_s[ii][c], yj_s[tx][c], acc);
      s[k] = acc;
    }
  }
  double r2 = 0.0, t2 = 0.0, ct = 0.0;
  const int j = j0 + tx;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = i0 + ty + 8 * k;
    if (i < n && j < n) {
      const int32_t id = amap[(int64_t)i * ldmap + j];
      const double cij = C ? C[(int64_t)i * ldc + j] : 0.0;
      const double R = (id >= 0 ? y[id] : 0.0) - s[k] - cij;
      const double tn = T[(int64_t)i * ldt + j] - sigma * R;
      T[(int64_t)i * ldt + j] = tn;
      r2 = fma(R, R, r2);
      t2 = fma(tn, tn, t2);
      ct = fma(cij, tn, ct);
    }
  }
  double v[3] = {r2, t2, ct};
  grid_sum<3>(v, part, counter, scal_out, scratch);
}

cudaError_t dual_update_launch(const DualArgs &a, cudaStream_t st) {
  dim3 grid((a.n + 31) / 32, (a.n + 31) / 32);
  dual_update_kernel<<<grid, 256, 0, st>>>(a.n, a.p, a.Y, a.ldy, a.amap, a.ldmap, a.y, a.C, a.ldc, a.sigma, a.T,
                                           a.ldt, a.part, a.counter, a.scal_out);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// Vector kernels on n x p row-major arrays (pitch ld). Warp per row, lanes over columns.
// ----------------------------------------------------------------------------------------------
#define ROW_LOOP_BEGIN                                                       \
  const int lane = threadIdx.x & 31;                                       \
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); \
  if (row < n) {
#define ROW_LOOP_END }

// dots[k] = <A_k, B_k> for up to 3 pairs
__global__ void __launch_bounds__(256) dot3_kernel(int n, int p, int ld, const double *A0, const double *B0,
                                                   const double *A1, const double *B1, const double *A2,
                                                   const double *B2, double *part, unsigned *counter,
                                                   double *out) {
  __shared__ double scratch[3 * 8];
  double v[3] = {0.0, 0.0, 0.0};
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  for (int c = lane; c < p; c += 32) {
    if (A0) v[0] = fma(A0[o + c], B0[o + c], v[0]);
    if (A1) v[1] = fma(A1[o + c], B1[o + c], v[1]);
    if (A2) v[2] = fma(A2[o + c], B2[o + c], v[2]);
  }
  ROW_LOOP_END
  grid_sum<3>(v, part, counter, out, scratch);
}

// out_row = (Y_row + t V_row) / ||Y_row + t V_row||; flag[0] = 1 if a norm <= 1e-14
__global__ void __launch_bounds__(256) retract_kernel(int n, int p, int ld, const double *Y, const double *V,
                                                      double t, double *out, int *flag) {
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  double s = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double x = fma(t, V[o + c], Y[o + c]);
    s = fma(x, x, s);
  }
  s = warp_sum(s);
  const double nrm = sqrt(s);
  if (nrm <= 1e-14) {
    if (lane == 0) atomicExch(flag, 1);
  } else {
    const double inv = 1.0 / nrm;
    for (int c = lane; c < p; c += 32) out[o + c] = fma(t, V[o + c], Y[o + c]) * inv;
  }
  ROW_LOOP_END
}

// tCG new direction: d = P_Y(-r + beta d) in place; dots = [<d,d>]
__global__ void __launch_bounds__(256) newdir_kernel(int n, int p, int ld, const double *Y, const double *r,
                                                     double beta, double *d, double *part, unsigned *counter,
                                                     double *dots) {
  __shared__ double scratch[8];
  double v[1] = {0.0};
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  double s = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double x = fma(beta, d[o + c], -r[o + c]);
    s = fma(x, Y[o + c], s);
  }
  s = warp_sum(s);
  for (int c = lane; c < p; c += 32) {
    const double x = fma(beta, d[o + c], -r[o + c]) - s * Y[o + c];
    d[o + c] = x;
    v[0] = fma(x, x, v[0]);
  }
  ROW_LOOP_END
  grid_sum<1>(v, part, counter, dots, scratch);
}

// out[:, 0:p_out] from in (pitch ldi) : out = [in[:, 0:p_in] * scale_in  | 0 ]  then optional
// escape columns V (n x dv, column k at Vcols + k*ldv_col, i.e. column-major as cuSOLVER returns)
// placed at columns [vcol0, vcol0 + dv).
__global__ void __launch_bounds__(256) repack_kernel(int n, int p_in, int ldi, const double *in, int p_out,
                                                     int ldo, double *out, int vcol0, int dv, const double *Vcols,
                                                     int64_t ldv_col) {
  ROW_LOOP_BEGIN
  for (int c = lane; c < ldo; c += 32) {
    double x = 0.0;
    if (in && c < p_in) x = in[(size_t)row * ldi + c];
    if (Vcols && c >= vcol0 && c < vcol0 + dv) x = Vcols[(size_t)(c - vcol0) * ldv_col + row];
    if (c >= p_out) x = 0.0;
    out[(size_t)row * ldo + c] = x;
  }
  ROW_LOOP_END
}

// X (n x n, compact) = T - Diag(z)
__global__ void __launch_bounds__(256) make_x_kernel(int n, const double *T, int64_t ldt, const double *z,
                                                     double *X) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e - i * n;
    double v = T[i * ldt + j];
    if (i == j) v -= z[i];
    X[e] = v;
  }
}

// out[k] = sum_e a[e] * b[e] over length len vectors (k = 0), plus sum a^2 (k = 1)
__global__ void __launch_bounds__(256) vdot_kernel(int64_t len, const double *a, const double *b, double *part,
                                                   unsigned *counter, double *out) {
  __shared__ double scratch[16];
  double v[2] = {0.0, 0.0};
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[e];
    v[0] = fma(x, b ? b[e] : 0.0, v[0]);
    v[1] = fma(x, x, v[1]);
  }
  grid_sum<2>(v, part, counter, out, scratch);
}

// D = A*(b / cnt) written into T (n x ldt); padding zeroed.
__global__ void __launch_bounds__(256) init_d_kernel(int n, const int32_t *amap, int64_t ldmap, const double *b,
                                                     const int32_t *cnt, double *T, int64_t ldt) {
  const int64_t total = (int64_t)n * ldt;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / ldt, j = e - i * ldt;
    double v = 0.0;
    if (j < n) {
      const int32_t id = amap[i * ldmap + j];
      if (id >= 0) v = b[id] / (double)cnt[id];
    }
    T[e] = v;
  }
}

// ||M||_F^2 over a rows x cols matrix with pitch ld
__global__ void __launch_bounds__(256) fro2_kernel(int64_t rows, int cols, const double *M, int64_t ld, double *part,
                                                   unsigned *counter, double *out) {
  __shared__ double scratch[8];
  double v[1] = {0.0};
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    const double x = __ldcs(M + i * ld + j);
    v[0] = fma(x, x, v[0]);
  }
  grid_sum<1>(v, part, counter, out, scratch);
}

// scalars: out[0] = a[0] * s0 + b[0] * s1 + c  (tiny host-free combine)
__global__ void combine_kernel(const double *a, double s0, const double *b, double s1, double c, double *out) {
  if (threadIdx.x == 0) out[0] = (a ? a[0] * s0 : 0.0) + (b ? b[0] * s1 : 0.0) + c;
}

// ----------------------------------------------------------------------------------------------
// Generic-p row epilogues (p > 64, where the product kernels run column-chunked in RAW mode).
// COSTGRAD (Eq. 4.6, Lemma 4.1): P = M Y, W = Y G:  E = 4 (W - P), rho_i = <E_i, y_i>,
//   R = E - rho o Y;  scal_out = [sum_i <P_i, y_i>, ||R||^2];  cost = gg - 2 s1 + extra[0] + extra[1]
// HVP (Eq. 4.7): Q = M U (+ A*(w) Y), W = U G + Y K:  EH = 4 (W - Q),
//   H = EH - rowdot(EH, Y) o Y - rho o U;  scal_out = [<U, H>, 0]
// ----------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rowepi_costgrad_kernel(int n, int p, const double *__restrict__ P, int ldp,
                                                              const double *__restrict__ W, int ldw,
                                                              const double *__restrict__ Y, int ldy, double *R,
                                                              int ldr, double *E, int lde, double *rho_out,
                                                              double *part, unsigned *counter, double *scal_out,
                                                              const double *gg, const double *extra,
                                                              double *cost_out) {
  __shared__ double scratch[2 * 8];
  double v[2] = {0.0, 0.0};
  ROW_LOOP_BEGIN
  const double *pr = P + (size_t)row * ldp, *wr = W + (size_t)row * ldw, *yr = Y + (size_t)row * ldy;
  double py = 0.0, ey = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double e = 4.0 * (wr[c] - pr[c]);
    py = fma(pr[c], yr[c], py);
    ey = fma(e, yr[c], ey);
  }
  py = warp_sum(py);
  const double rho = warp_sum(ey);
  double rr = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double e = 4.0 * (wr[c] - pr[c]);
    const double r = e - rho * yr[c];
    rr = fma(r, r, rr);
    if (R) R[(size_t)row * ldr + c] = r;
    if (E) E[(size_t)row * lde + c] = e;
  }
  rr = warp_sum(rr);
  if (lane == 0) {
    if (rho_out) rho_out[row] = rho;
    v[0] = py;
    v[1] = rr;
  }
  ROW_LOOP_END
  if (grid_sum<2>(v, part, counter, scal_out, scratch) && threadIdx.x == 0 && cost_out)
    cost_out[0] = gg[0] - 2.0 * v[0] + extra[0] + extra[1];
}

__global__ void __launch_bounds__(256) rowepi_hvp_kernel(int n, int p, const double *__restrict__ Q, int ldq,
                                                         const double *__restrict__ W, int ldw,
                                                         const double *__restrict__ Y, int ldy,
                                                         const double *__restrict__ U, int ldu,
                                                         const double *__restrict__ rho, double *H, int ldh,
                                                         double *part, unsigned *counter, double *scal_out,
                                                         const int *skip) {
  if (skip && *(volatile const int *)skip) return;
  __shared__ double scratch[2 * 8];
  double v[2] = {0.0, 0.0};
  ROW_LOOP_BEGIN
  const double *qr = Q + (size_t)row * ldq, *wr = W + (size_t)row * ldw;
  const double *yr = Y + (size_t)row * ldy, *ur = U + (size_t)row * ldu;
  double ehy = 0.0;
  for (int c = lane; c < p; c += 32) ehy = fma(4.0 * (wr[c] - qr[c]), yr[c], ehy);
  ehy = warp_sum(ehy);
  const double rh = rho[row];
  double uh = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double h = 4.0 * (wr[c] - qr[c]) - ehy * yr[c] - rh * ur[c];
    H[(size_t)row * ldh + c] = h;
    uh = fma(ur[c], h, uh);
  }
  uh = warp_sum(uh);
  if (lane == 0) v[0] = uh;
  ROW_LOOP_END
  grid_sum<2>(v, part, counter, scal_out, scratch);
}

// z_i = <P_i, y_i> (P = T Y), out[0] = sum_i z_i   (Alg. 2 step 7, generic p)
__global__ void __launch_bounds__(256) rowdot_kernel(int n, int p, const double *__restrict__ P, int ldp,
                                                     const double *__restrict__ Y, int ldy, double *z, double *part,
                                                     unsigned *counter, double *out) {
  __shared__ double scratch[2 * 8];
  double v[2] = {0.0, 0.0};
  ROW_LOOP_BEGIN
  double d = 0.0;
  for (int c = lane; c < p; c += 32) d = fma(P[(size_t)row * ldp + c], Y[(size_t)row * ldy + c], d);
  d = warp_sum(d);
  if (lane == 0) {
    z[row] = d;
    v[0] = d;
  }
  ROW_LOOP_END
  grid_sum<2>(v, part, counter, out, scratch);
}

// rows of X (n x r, pitch ld) scaled to unit norm in place; columns [r, ld) zeroed
__global__ void __launch_bounds__(256) normalize_rows_kernel(int n, int r, int ld, double *X) {
  ROW_LOOP_BEGIN
  double *xr = X + (size_t)row * ld;
  double s = 0.0;
  for (int c = lane; c < r; c += 32) s = fma(xr[c], xr[c], s);
  s = warp_sum(s);
  const double inv = 1.0 / sqrt(s);
  for (int c = lane; c < ld; c += 32) xr[c] = c < r ? xr[c] * inv : 0.0;
  ROW_LOOP_END
}

// ----------------------------------------------------------------------------------------------
// Device-resident truncated CG (Steihaug-Toint, the recurrences of oracle/rtr.py tcg).
// ----------------------------------------------------------------------------------------------
__global__ void tcg_init_kernel(TcgDev *st, double gnorm, double Delta, int max_iters, int prec) {
  if (threadIdx.x) return;
  st->prec = prec;
  st->z_r = gnorm * gnorm;  // prec: replaced by <Prec(r), r> (tcg_prec_kernel, init)
  st->r_r = gnorm * gnorm;
  st->norm_r0 = gnorm;
  st->e_Pe = 0.0;
  st->e_Pd = 0.0;
  st->d_Pd = gnorm * gnorm;
  st->model = 0.0;
  st->Delta2 = Delta * Delta;
  st->alpha = 0.0;
  st->beta = 0.0;
  st->e_Pe_new = 0.0;
  st->done = 0;
  st->hit = 0;
  st->iters = 0;
  st->par = 0;
  st->boundary = 0;
  st->max_iters = max_iters;
}

// One tCG iteration after H delta is known (oracle/rtr.py tcg, lines "d_Hd = ..." to the new
// direction): every block derives the same step (alpha, or the boundary step tau) from kappa =
// <delta, H delta> and the device scalars, updates its rows (ping-pong buffers), and the last
// block applies the acceptance / stopping rules. With use_cond it also drives the conditional
// WHILE node of the captured graph (keep looping while the tCG runs).
__global__ void __launch_bounds__(256) tcg_update_kernel(int n, int p, int ld, TcgDev *st, double *e0, double *e1,
                                                         double *h0, double *h1, double *r,
                                                         const double *__restrict__ d, const double *__restrict__ hd,
                                                         const double *__restrict__ g, double *part,
                                                         unsigned *counter, const double *kappa,
                                                         cudaGraphConditionalHandle cond, int use_cond) {
  if (*(volatile const int *)&st->done) return;
  __shared__ double scratch[3 * 8];
  const double dHd = *(volatile const double *)kappa;
  if (!isfinite(dHd)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->done = 2;
      if (use_cond) cudaGraphSetConditional(cond, 0u);
    }
    return;
  }
  const double r_r = st->r_r, z_r = st->z_r, e_Pe = st->e_Pe, e_Pd = st->e_Pd, d_Pd = st->d_Pd;
  const double Delta2 = st->Delta2;
  const int prec = st->prec;
  const double alpha = dHd != 0.0 ? (prec ? z_r : r_r) / dHd : INFINITY;
  const double e_Pe_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd;
  const int bnd = (dHd <= 0.0 || e_Pe_new >= Delta2) ? 1 : 0;
  const double a = bnd ? (-e_Pd + sqrt(e_Pd * e_Pd + d_Pd * (Delta2 - e_Pe))) / d_Pd : alpha;
  const int par = st->par;
  // eta and H eta ping-pong (a rejected step keeps the previous ones); r is updated in place
  // (it is only needed while the tCG continues)
  const double *e = par ? e1 : e0, *h = par ? h1 : h0;
  double *eo = par ? e0 : e1, *ho = par ? h0 : h1;
  double v[3] = {0.0, 0.0, 0.0};
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  for (int c = lane; c < p; c += 32) {
    const size_t k = o + c;
    const double hdv = hd[k];
    const double ev = fma(a, d[k], e[k]);
    const double hv = fma(a, hdv, h[k]);
    eo[k] = ev;
    ho[k] = hv;
    v[0] = fma(ev, g[k], v[0]);
    v[1] = fma(ev, hv, v[1]);
    if (!bnd) {
      const double rv = fma(a, hdv, r[k]);
      r[k] = rv;
      v[2] = fma(rv, rv, v[2]);
    }
  }
  ROW_LOOP_END
  if (!grid_sum<3>(v, part, counter, nullptr, scratch) || threadIdx.x != 0) return;
  st->iters += 1;
  st->alpha = a;
  st->boundary = bnd;
  if (bnd) {
    st->par = 1 - par;
    st->hit = 1;
    st->done = 1;
  } else {
    const double new_model = v[0] + 0.5 * v[1];
    if (new_model >= st->model) {  // no model decrease: keep the previous eta (oracle/rtr.py)
      st->done = 1;
    } else {
      st->par = 1 - par;
      st->model = new_model;
      st->e_Pe = e_Pe_new;
      st->r_r = v[2];
      if (sqrt(v[2]) <= st->norm_r0 * fmin(st->norm_r0, 0.1)) {  // theta = 1, kappa = 0.1
        st->done = 1;
      } else if (prec) {
        // beta, e_Pd, d_Pd need <Prec(r), r>: tcg_prec_kernel after the preconditioner product
        if (st->iters >= st->max_iters) st->done = 1;
      } else {
        const double beta = v[2] / r_r;
        st->e_Pd = beta * (e_Pd + a * d_Pd);
        st->d_Pd = v[2] + beta * beta * d_Pd;
        st->beta = beta;
        if (st->iters >= st->max_iters) st->done = 1;
      }
    }
  }
  if (use_cond) cudaGraphSetConditional(cond, st->done ? 0u : 1u);
}

// delta = P_Y(-src + beta delta), src = r (or Prec(r) when preconditioned)
__global__ void __launch_bounds__(256) tcg_newdir_kernel(int n, int p, int ld, const TcgDev *st,
                                                         const double *__restrict__ Y, const double *r, double *d) {
  if (*(volatile const int *)&st->done) return;
  const double beta = st->beta;
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  double s = 0.0;
  for (int c = lane; c < p; c += 32) s = fma(fma(beta, d[o + c], -r[o + c]), Y[o + c], s);
  s = warp_sum(s);
  for (int c = lane; c < p; c += 32) d[o + c] = fma(beta, d[o + c], -r[o + c]) - s * Y[o + c];
  ROW_LOOP_END
}

// Preconditioned tCG (reading R35; oracle/rtr.py tcg with prec): z holds r W on entry (W the
// Gram preconditioner, tcg_prec_matrix_kernel); z <- P_Y(z) in place and <z, r> by a fixed-order
// grid reduction. init: delta = -z and z_r = d_Pd = <z, r>. Otherwise the last block forms
// beta = <z, r> / z_r_old and the recurrences e_Pd = beta (e_Pd + alpha d_Pd),
// d_Pd = <z, r> + beta^2 d_Pd (the trust region is measured in the Prec^{-1} norm).
__global__ void __launch_bounds__(256) tcg_prec_kernel(int n, int p, int ld, TcgDev *st, const double *__restrict__ Y,
                                                       double *z, const double *__restrict__ r, double *d,
                                                       double *part, unsigned *counter, int init) {
  if (*(volatile const int *)&st->done) return;
  __shared__ double scratch[8];
  double v[1] = {0.0};
  ROW_LOOP_BEGIN
  const size_t o = (size_t)row * ld;
  double s = 0.0;
  for (int c = lane; c < p; c += 32) s = fma(z[o + c], Y[o + c], s);
  s = warp_sum(s);
  double zr = 0.0;
  for (int c = lane; c < p; c += 32) {
    const double zv = z[o + c] - s * Y[o + c];
    z[o + c] = zv;
    zr = fma(zv, r[o + c], zr);
    if (init) d[o + c] = -zv;
  }
  zr = warp_sum(zr);
  if (lane == 0) v[0] = zr;
  ROW_LOOP_END
  if (!grid_sum<1>(v, part, counter, nullptr, scratch) || threadIdx.x != 0) return;
  const double zr = v[0];
  if (init) {
    st->z_r = zr;
    st->d_Pd = zr;
    return;
  }
  const double beta = zr / st->z_r;
  st->e_Pd = beta * (st->e_Pd + st->alpha * st->d_Pd);
  st->d_Pd = zr + beta * beta * st->d_Pd;
  st->z_r = zr;
  st->beta = beta;
}

// A = G / gbar + mu I and B = I (p x p, pitch p), gbar = tr(G) / p: the Cholesky solve A W = I
// (cuSOLVER potrf / potrs on p x p) then gives the preconditioner matrix W = gbar (G + mu gbar I)^-1.
__global__ void __launch_bounds__(256) tcg_prec_matrix_kernel(int p, const double *__restrict__ G, double mu,
                                                              double *A, double *B) {
  __shared__ double scratch[8];
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < p; i += blockDim.x) v[0] += G[(size_t)i * p + i];
  block_sum<1>(v, scratch);
  __shared__ double s_inv;
  if (threadIdx.x == 0) s_inv = v[0] > 0.0 ? (double)p / v[0] : 1.0;
  __syncthreads();
  const double inv = s_inv;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, j = e - i * p;
    A[e] = G[e] * inv + (i == j ? mu : 0.0);
    B[e] = i == j ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(256) tcg_finalize_kernel(int n, int p, int ld, const TcgDev *st, double *e0,
                                                           const double *e1, double *h0, const double *h1) {
  if (st->par == 0) return;
  const size_t total = (size_t)n * ld;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
    e0[k] = e1[k];
    h0[k] = h1[k];
  }
}

// W = A*(w) as a dense matrix: W_ij = w[amap_ij] (0 where unconstrained); padding columns zeroed.
// Feeds the gather-product A*(w) Y of Eq. 4.7's projection term to the TMA product kernel.
__global__ void __launch_bounds__(256) gather_assemble_kernel(int n, const int32_t *__restrict__ amap, int64_t ldmap,
                                                              const double *__restrict__ w, double *__restrict__ W,
                                                              int64_t ldw, const int *skip) {
  if (skip && *(volatile const int *)skip) return;
  // row = blockIdx.y, four consecutive columns per thread (ldw, ldmap are multiples of 4): one
  // int4 load of ids, four gathers of w (L2-resident), two double2 stores
  const int64_t i = blockIdx.y;
  const int j = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (j >= ldw) return;
  int4 id = make_int4(-1, -1, -1, -1);
  if (j < n) id = __ldg(reinterpret_cast<const int4 *>(amap + i * ldmap + j));
  const int ids[4] = {id.x, id.y, id.z, id.w};
  double v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = (j + k < n && ids[k] >= 0) ? __ldg(w + ids[k]) : 0.0;
  double2 *out = reinterpret_cast<double2 *>(W + i * ldw + j);
  out[0] = make_double2(v[0], v[1]);
  out[1] = make_double2(v[2], v[3]);
}

// ---------------------------------------------------------------------------------------------
static inline int rows_grid(int64_t n) { return (int)((n + 7) / 8); }

cudaError_t dot3_launch(int n, int p, int ld, const double *A0, const double *B0, const double *A1,
                        const double *B1, const double *A2, const double *B2, double *part, unsigned *counter,
                        double *out, cudaStream_t st) {
  dot3_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, ld, A0, B0, A1, B1, A2, B2, part, counter, out);
  return cudaGetLastError();
}
cudaError_t retract_launch(int n, int p, int ld, const double *Y, const double *V, double t, double *out,
                           int *flag, cudaStream_t st) {
  retract_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, ld, Y, V, t, out, flag);
  return cudaGetLastError();
}
cudaError_t newdir_launch(int n, int p, int ld, const double *Y, const double *r, double beta, double *d,
                          double *part, unsigned *counter, double *dots, cudaStream_t st) {
  newdir_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, ld, Y, r, beta, d, part, counter, dots);
  return cudaGetLastError();
}
cudaError_t repack_launch(int n, int p_in, int ldi, const double *in, int p_out, int ldo, double *out, int vcol0,
                          int dv, const double *Vcols, int64_t ldv_col, cudaStream_t st) {
  repack_kernel<<<rows_grid(n), 256, 0, st>>>(n, p_in, ldi, in, p_out, ldo, out, vcol0, dv, Vcols, ldv_col);
  return cudaGetLastError();
}
cudaError_t make_x_launch(int n, const double *T, int64_t ldt, const double *z, double *X, cudaStream_t st) {
  make_x_kernel<<<1184, 256, 0, st>>>(n, T, ldt, z, X);
  return cudaGetLastError();
}
cudaError_t vdot_launch(int64_t len, const double *a, const double *b, double *part, unsigned *counter,
                        double *out, cudaStream_t st) {
  int nb = (int)((len + 255) / 256);
  if (nb > 592) nb = 592;
  if (nb < 1) nb = 1;
  vdot_kernel<<<nb, 256, 0, st>>>(len, a, b, part, counter, out);
  return cudaGetLastError();
}
cudaError_t init_d_launch(int n, const int32_t *amap, int64_t ldmap, const double *b, const int32_t *cnt,
                          double *T, int64_t ldt, cudaStream_t st) {
  init_d_kernel<<<1184, 256, 0, st>>>(n, amap, ldmap, b, cnt, T, ldt);
  return cudaGetLastError();
}
cudaError_t fro2_launch(int n, const double *M, int64_t ld, double *part, unsigned *counter, double *out,
                        cudaStream_t st) {
  fro2_kernel<<<1184, 256, 0, st>>>(n, n, M, ld, part, counter, out);
  return cudaGetLastError();
}
cudaError_t fro2_rows_launch(int64_t rows, int64_t cols, const double *M, int64_t ld, double *part, unsigned *counter,
                             double *out, cudaStream_t st) {
  fro2_kernel<<<1184, 256, 0, st>>>(rows, (int)cols, M, ld, part, counter, out);
  return cudaGetLastError();
}
cudaError_t combine_launch(const double *a, double s0, const double *b, double s1, double c, double *out,
                           cudaStream_t st) {
  combine_kernel<<<1, 32, 0, st>>>(a, s0, b, s1, c, out);
  return cudaGetLastError();
}

cudaError_t rowepi_costgrad_launch(int n, int p, const double *P, int ldp, const double *W, int ldw,
                                   const double *Y, int ldy, double *R, int ldr, double *E, int lde, double *rho_out,
                                   double *part, unsigned *counter, double *scal_out, const double *gg,
                                   const double *extra, double *cost_out, cudaStream_t st) {
  rowepi_costgrad_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, P, ldp, W, ldw, Y, ldy, R, ldr, E, lde, rho_out, part,
                                                       counter, scal_out, gg, extra, cost_out);
  return cudaGetLastError();
}
cudaError_t rowepi_hvp_launch(int n, int p, const double *Q, int ldq, const double *W, int ldw, const double *Y,
                              int ldy, const double *U, int ldu, const double *rho, double *H, int ldh, double *part,
                              unsigned *counter, double *scal_out, const int *skip, cudaStream_t st) {
  rowepi_hvp_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, Q, ldq, W, ldw, Y, ldy, U, ldu, rho, H, ldh, part, counter,
                                                  scal_out, skip);
  return cudaGetLastError();
}
cudaError_t rowdot_launch(int n, int p, const double *P, int ldp, const double *Y, int ldy, double *z, double *part,
                          unsigned *counter, double *out, cudaStream_t st) {
  rowdot_kernel<<<rows_grid(n), 256, 0, st>>>(n, p, P, ldp, Y, ldy, z, part, counter, out);
  return cudaGetLastError();
}
cudaError_t normalize_rows_launch(int n, int r, int ld, double *X, cudaStream_t st) {
  normalize_rows_kernel<<<rows_grid(n), 256, 0, st>>>(n, r, ld, X);
  return cudaGetLastError();
}

cudaError_t tcg_init_launch(TcgDev *st, double gnorm, double Delta, int max_iters, int prec, cudaStream_t s) {
  tcg_init_kernel<<<1, 32, 0, s>>>(st, gnorm, Delta, max_iters, prec);
  return cudaGetLastError();
}
cudaError_t tcg_update_launch(int n, int p, int ld, TcgDev *st, double *e0, double *e1, double *h0, double *h1,
                              double *r, const double *d, const double *hd, const double *g, double *part,
                              unsigned *counter, const double *kappa, cudaGraphConditionalHandle cond, int use_cond,
                              cudaStream_t s) {
  tcg_update_kernel<<<rows_grid(n), 256, 0, s>>>(n, p, ld, st, e0, e1, h0, h1, r, d, hd, g, part, counter, kappa,
                                                 cond, use_cond);
  return cudaGetLastError();
}
cudaError_t tcg_newdir_launch(int n, int p, int ld, const TcgDev *st, const double *Y, const double *src, double *d,
                              cudaStream_t s) {
  tcg_newdir_kernel<<<rows_grid(n), 256, 0, s>>>(n, p, ld, st, Y, src, d);
  return cudaGetLastError();
}
cudaError_t tcg_prec_launch(int n, int p, int ld, TcgDev *st, const double *Y, double *z, const double *r, double *d,
                            double *part, unsigned *counter, int init, cudaStream_t s) {
  tcg_prec_kernel<<<rows_grid(n), 256, 0, s>>>(n, p, ld, st, Y, z, r, d, part, counter, init);
  return cudaGetLastError();
}
cudaError_t tcg_prec_matrix_launch(int p, const double *G, double mu, double *A, double *B, cudaStream_t s) {
  tcg_prec_matrix_kernel<<<1, 256, 0, s>>>(p, G, mu, A, B);
  return cudaGetLastError();
}

cudaError_t tcg_finalize_launch(int n, int p, int ld, const TcgDev *st, double *e0, const double *e1, double *h0,
                                const double *h1, cudaStream_t s) {
  (void)p;
  int nb = (int)(((size_t)n * ld + 255) / 256);
  if (nb > 1184) nb = 1184;
  tcg_finalize_kernel<<<nb, 256, 0, s>>>(n, p, ld, st, e0, e1, h0, h1);
  return cudaGetLastError();
}

cudaError_t gather_assemble_launch(int n, const int32_t *amap, int64_t ldmap, const double *w, double *W, int64_t ldw,
                                   const int *skip, cudaStream_t st) {
  if ((ldw & 3) || (ldmap & 3) || n > 65535) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((ldw / 4 + 255) / 256), (unsigned)n);
  gather_assemble_kernel<<<grid, 256, 0, st>>>(n, amap, ldmap, w, W, ldw, skip);
  return cudaGetLastError();
}

}  // namespace drsdp
