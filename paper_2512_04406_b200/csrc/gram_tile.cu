// gram_tile.cu — dense upper-triangle Gram tiles D = A1 B1^T (+ A2 B2^T) on the fp64 DMMA path,
// operands streamed by TMA. Used to evaluate the segmented sums of the y-eliminated subproblem
// through a dense intermediate instead of one gathered p-length dot product per position:
//   y(S) = A(Y Y^T + C) / cnt       -> D = Y Y^T                  (Lemma 3.1)
//   A(Z), Z = Y U^T + U Y^T         -> D = [Y U] [U Y]^T          (Prop 4.2's projection term)
// then segsum_dense (kernels.cu) sums D over the positions of each constraint. The dense route
// costs 2 n^2 p tensor flops + one n^2/2 write, against ~16 n^2 p bytes of L2 gathers for the
// per-position dot products; it is the only practical route at d = 100 / 150 with p in the hundreds.
//
// CTA = one 128 x 128 tile (I <= J); 8 consumer warps as 2 x 4 warp tiles of 64 x 32
// (8 x 4 DMMA m8n8k4 per k-step), one producer warp feeding a 3-stage ring of
// [128 x 32] boxes of both operands (SWIZZLE_128B; both operands k-contiguous, conflict free).
#include <cuda.h>

#include "common.cuh"
#include "tma.cuh"
#include "gram_tile.cuh"

namespace drsdp {

namespace {
constexpr int TB = 128, BK = 32, NCW = 8, STAGES = 3;
constexpr int NT = (NCW + 1) * 32;
constexpr int WR = 2, WC = 4, WM = TB / WR, WN = TB / WC, JB = WM / 8, CB = WN / 8;
constexpr int OP_ELEMS = TB * BK;                // one operand per stage
constexpr int STAGE_ELEMS = 2 * OP_ELEMS;
constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * 8;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_ELEMS * 8 + 1024;

}  // namespace

// upper tile t (row-major over I <= J) -> (I, J)
DRSDP_DEV void upper_tile(int t, int nb, int &I, int &J) {
  I = 0;
  while (t >= nb - I) {
    t -= nb - I;
    ++I;
  }
  J = I + t;
}

// One CTA per upper tile (I <= J; D is symmetric and its consumers read i <= j). The contraction
// runs over 16-column TMA boxes of the concatenated K = [A1 | A2] (p columns each, the last box of
// each operand zero-filled past p): a stage holds two consecutive boxes, so at p <= 16 the pair
// product [Y U][U Y]^T is a single stage of 32 useful columns.
__global__ void __launch_bounds__(NT, 1)
    gram_tile_kernel(const __grid_constant__ CUtensorMap mA1, const __grid_constant__ CUtensorMap mB1,
                     const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mB2, int n, int p,
                     int pair, double *__restrict__ D, int64_t ldd, const int *skip) {
  int I, J;
  upper_tile(blockIdx.x, (n + TB - 1) / TB, I, J);
  if (skip && *(volatile const int *)skip) return;
  extern __shared__ unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nbx1 = (p + 15) / 16;              // 16-column boxes per operand
  const int nbx = pair ? 2 * nbx1 : nbx1;
  const int nk = (nbx + 1) / 2;                 // stages of two boxes
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % STAGES;
        if (kt >= STAGES) bar_wait(&empty[st], ((kt / STAGES) - 1) & 1);
        double *sa = smem + st * STAGE_ELEMS, *sb = sa + OP_ELEMS;
        bar_expect(&full[st], STAGE_BYTES);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int bx = 2 * kt + h;  // box index in the concatenated K (past the end: zero-filled)
          const bool second = bx >= nbx1 && bx < nbx;
          // bx >= nbx: a box entirely past column p of A1 (TMA zero-fills out-of-range elements)
          const int c0 = bx >= nbx ? nbx1 * 16 : (second ? bx - nbx1 : bx) * 16;
          const CUtensorMap *ma = second ? &mA2 : &mA1, *mb = second ? &mB2 : &mB1;
          tma2d(sa + h * TB * 16, ma, c0, I * TB, &full[st]);
          tma2d(sb + h * TB * 16, mb, c0, J * TB, &full[st]);
        }
      }
    }
    return;
  }
  const int q = lane >> 2, r = lane & 3;
  const int wr = warp % WR, wc = warp / WR;
  double acc[JB][CB][2];
#pragma unroll
  for (int jb = 0; jb < JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) acc[jb][cb][0] = acc[jb][cb][1] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % STAGES;
    bar_wait(&full[st], (kt / STAGES) & 1);
    const uint32_t sa = su32(smem) + st * STAGE_BYTES, sb = sa + OP_ELEMS * 8;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int box = ks >> 2, col = ((ks & 3) << 2) + r;
      const uint32_t ba = sa + box * TB * 128, bb = sb + box * TB * 128;
      double af[JB], bf[CB];
#pragma unroll
      for (int jb = 0; jb < JB; ++jb) af[jb] = ldsw(ba, wr * WM + 8 * jb + q, col);
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) bf[cb] = ldsw(bb, wc * WN + 8 * cb + q, col);
#pragma unroll
      for (int jb = 0; jb < JB; ++jb)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) dmma_884(acc[jb][cb][0], acc[jb][cb][1], af[jb], bf[cb]);
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[st]);
  }
#pragma unroll
  for (int jb = 0; jb < JB; ++jb) {
    const int i = I * TB + wr * WM + 8 * jb + q;
    if (i >= n) continue;
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      const int j = J * TB + wc * WN + 8 * cb + 2 * r;
      if (j + 1 < n) {
        *reinterpret_cast<double2 *>(D + (size_t)i * ldd + j) = make_double2(acc[jb][cb][0], acc[jb][cb][1]);
      } else if (j < n) {
        D[(size_t)i * ldd + j] = acc[jb][cb][0];
      }
    }
  }
}

static bool map_rows(CUtensorMap *m, const double *base, int64_t rows, int64_t cols, int64_t ld) {
  return tma_map_f64(m, base, rows, cols, ld, TB);
}

bool gram_tile_supported(const double *A, const double *B, int ld) {
  return !(ld & 1) && !((uintptr_t)A & 15) && !((uintptr_t)B & 15) && tma_encoder() != nullptr;
}

cudaError_t gram_tile_launch(int n, int p, const double *A1, const double *B1, const double *A2, const double *B2,
                             int ld, double *D, int64_t ldd, const int *skip, cudaStream_t st) {
  CUtensorMap m[4];
  if (!map_rows(&m[0], A1, n, p, ld) || !map_rows(&m[1], B1, n, p, ld)) return cudaErrorInvalidValue;
  const bool pair = A2 != nullptr;
  if (pair) {
    if (!map_rows(&m[2], A2, n, p, ld) || !map_rows(&m[3], B2, n, p, ld)) return cudaErrorInvalidValue;
  } else {
    m[2] = m[0];
    m[3] = m[1];
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gram_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nb = (n + TB - 1) / TB;
  gram_tile_kernel<<<nb * (nb + 1) / 2, NT, SMEM_BYTES, st>>>(m[0], m[1], m[2], m[3], n, p, pair ? 1 : 0, D, ldd,
                                                              skip);
  return cudaGetLastError();
}

}  // namespace drsdp
