// tma.cuh — TMA / mbarrier helpers shared by the TMA-fed DMMA kernels (symv_tma.cu, symv_symm.cu,
// gram_tile.cu): 2D fp64 tensor maps with 16-column SWIZZLE_128B boxes, mbarrier ring primitives,
// and the swizzled shared-memory fragment load.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace drsdp {

// ---- device side --------------------------------------------------------------------------------
DRSDP_DEV uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
DRSDP_DEV void bar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
DRSDP_DEV void bar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
DRSDP_DEV void bar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
DRSDP_DEV void bar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
// 2D tile load [c_outer, c_inner] of map into dst, completing on mbarrier b
DRSDP_DEV void tma2d(void *dst, const CUtensorMap *m, int ci, int co, uint64_t *b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(m), "r"(ci), "r"(co), "r"(su32(b))
      : "memory");
}
// element (row, col) of a [rows][16] fp64 box written by TMA with SWIZZLE_128B (1024 B aligned):
// the 16-byte chunk index (col / 2) is XORed with row % 8. Explicit ld.shared on a 32-bit shared
// address (a generic pointer compiles to LD.E).
DRSDP_DEV double ldsw(uint32_t box, int row, int col) {
  const uint32_t a = box + row * 128 + ((((col >> 1) ^ (row & 7))) << 4) + ((col & 1) << 3);
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

// ---- host side ----------------------------------------------------------------------------------
typedef CUresult (*TmaEncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link dependency)
inline TmaEncodeFn tma_encoder() {
  static TmaEncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<TmaEncodeFn>(f);
    else
      cudaGetLastError();
  }
  return fn;
}

// 2D fp64 tensor map: rows x cols (cols contiguous, row pitch ld doubles), box [box_rows][16],
// SWIZZLE_128B, zero fill out of range (ragged n, p)
inline bool tma_map_f64(CUtensorMap *m, const double *base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  TmaEncodeFn fn = tma_encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace drsdp
