// gram_tile.cuh — dense upper-triangle Gram tiles (gram_tile.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace drsdp {

// D[i][j] (i <= j, 128 x 128 tiles; tiles below the diagonal are not written) =
//   sum_k A1[i][k] B1[j][k]  (+ sum_k A2[i][k] B2[j][k] when A2 != nullptr),
// A*, B* n x p row-major with even pitch ld and 16 B aligned bases (TMA), D pitch ldd.
bool gram_tile_supported(const double *A, const double *B, int ld);
cudaError_t gram_tile_launch(int n, int p, const double *A1, const double *B1, const double *A2, const double *B2,
                             int ld, double *D, int64_t ldd, const int *skip, cudaStream_t st);

}  // namespace drsdp
