// blocks.cuh — kernels of the multi-block (clique-chain) relaxation, SURVEY §8(f) row f2
// (PAPER.md:434-436 remark, P:555-602 DSDP-sparse). Layout: t blocks of n_b rows; the factor Y
// stacks the blocks' rows (N = t n_b rows, pitch ldy); every block matrix (amap, T, M) is stored
// "stacked": row r of block k = r / n_b lives at row r of an N x ld array whose first n_b columns
// are the block's columns. Only diagonal blocks exist (cross-block products never appear).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "symv.cuh"

namespace drsdp {

constexpr int kBlkMaxP = 128;  // factor width supported by the block kernels (p <= min(128, n_b))

// G_k = Y_k^T Y_k and (U != nullptr) K_k = U_k^T Y_k + Y_k^T U_k, p x p each (pitch p), k < t
cudaError_t blk_gram_launch(int t, int nb, int p, const double *Y, int ldy, const double *U, int ldu, double *G,
                            double *K, const int *skip, cudaStream_t st);
// out (p x p) = sum_k G_k (rank-reduction Gram, reading R15)
cudaError_t blk_gsum_launch(int t, int p, const double *G, double *out, cudaStream_t st);

enum BlkElem { BLK_ASM = 0, BLK_DUAL = 1 };
struct BlkElemArgs {
  int t = 0, nb = 0, p = 0;
  const double *Y = nullptr;
  int ldy = 0;
  const int32_t *amap = nullptr;
  int64_t ldm = 0;
  const double *y = nullptr;  // y(S) (ASM) or y^{k+1} (DUAL)
  double *T = nullptr;        // read (ASM) / updated (DUAL)
  int64_t ldt = 0;
  double sigma = 1.0;
  double *M = nullptr;  // ASM output M = A*(y) - T/sigma
  int64_t ldmo = 0;
  const double *D = nullptr;  // ASM: S tiles from blk_tile (stacked, pitch ldd) instead of recomputing
  int64_t ldd = 0;
  double *part = nullptr;
  unsigned *counter = nullptr;
  // ASM: [sum (S - A*(y))^2, <T, S>, ||T||^2] (the accurate ALM cost, reading R29)
  // DUAL: [||A*(y) - S||^2, ||T_new||^2, 0]
  double *scal_out = nullptr;
};
// S_k tiles recomputed from Y (32 x 64 tiles, p in chunks of 32) fused with the elementwise work
cudaError_t blk_elem_launch(const BlkElemArgs &a, int mode, cudaStream_t st);
int blk_elem_blocks(int t, int nb);

// D_k = Y_k Y_k^T (U == nullptr, full blocks) or Y_k U_k^T + U_k Y_k^T (upper tiles), stacked
cudaError_t blk_tile_launch(int t, int nb, int p, const double *Y, const double *U, int ldy, double *D, int64_t ldd,
                            const int *skip, cudaStream_t st);

// T = A*(b / cnt) on every block (T^0 = D, X~^0 = 0)
cudaError_t blk_initd_launch(int t, int nb, const int32_t *amap, int64_t ldm, const double *b, const int32_t *cnt,
                             double *T, int64_t ldt, cudaStream_t st);
// X (t column-major n_b x n_b matrices, contiguous) = T_k - Diag(z_k)
cudaError_t blk_makex_launch(int t, int nb, const double *T, int64_t ldt, const double *z, double *X, cudaStream_t st);

// Block-diagonal product with the shared row epilogue (tile_epilogue.cuh): per row r of block k,
// P_r = sum_j A[r, j] V[k n_b + j]  (+ sum_j w[amap[r, j]] X[k n_b + j] with gather), then EPI_*
// with G = a.G + k p^2, K = a.K + k p^2. One CTA per 16-row strip; a.tile_scal (2 per tile) and
// a.glob_cnt as in the dense kernels. p <= kBlkMaxP.
cudaError_t blk_product_launch(const SymvArgs &a, int epi, bool gather, int t, int nb, cudaStream_t st);
int blk_product_tiles(int t, int nb);

}  // namespace drsdp
