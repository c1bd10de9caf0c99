// symv_gather.cu — matrix-light ALM Hessian-vector product (Eq. 4.7 with the
// projection term of Prop 4.2): the tile
//     Q = M U + A*(w) Y,     A*(w)_jk = w[amap_jk],  w = A(Y U^T + U Y^T) / cnt,
// is accumulated in ONE pass in which A*(w) is never materialised: the index-map panel
// amap[j0:j0+128, k0:k0+32] (int32) is TMA-loaded next to the M panel and a group of gather warps
// turns it into the fp64 operand tile w[amap] directly in the shared-memory ring, in the swizzled
// layout the DMMA consumers read. Per HVP the product then streams 8 n^2 (M) + 4 n^2 (amap) bytes
// instead of 8 n^2 + a dense A*(w) written (8 n^2) and read back (8 n^2) plus the amap read of its
// assembly (4 n^2).
//
// Pipeline (one CTA = 128 output rows x a k-range, 13 or 17 warps):
//   warp 8      producer: per 32-column k-tile two ring stages — an M stage (TMA: M panel + U^T
//               chunk) and a gather stage (TMA: amap panel into the stage's staging area + Y^T chunk);
//   warps 9-..  gather (4; 8 at PT <= 16): wait for the staging panel (raw barrier), write w[amap] into the stage's
//               operand area (SWIZZLE_128B layout), arrive on the stage's full barrier;
//   warps 0-7   consumers: the DMMA loop of symv_tma.cu, unchanged — both stage kinds look alike.
// The gathers of stage k overlap the DMMAs of the stages before it. Split-K, the ticketed fixed-order
// reduction and the row epilogue (tile_epilogue.cuh) are those of the full-matrix kernel.
#include <cuda.h>

#include "common.cuh"
#include "tma.cuh"
#include "symv.cuh"
#include "tile_epilogue.cuh"

namespace drsdp {

namespace {

constexpr int BM = 128, BK = 32, NCW = 8;  // rows per CTA, k per stage, consumer warps
constexpr int STAGES = 3;

template <int PT>
struct GCfg {
  // gather warps: 4 (32 panel rows each); 8 at PT <= 16, where a stage's DMMA work (~1000 clocks at
  // PT = 16) is shorter than the L2 round trips of a 4096-entry gather issued 8 loads per lane at a time
  // (the 8-warp configuration raced: rare wrong tiles in the bitwise-repeatability test; 4 warps everywhere
  // until the race is located — the kernel is off by default, see run_product in abi.cu)
  static constexpr int NGW = 4;
  static constexpr int NTHREADS = (NCW + 1 + NGW) * 32;
  static constexpr int RG = BM / NGW;  // panel rows per gather warp
  static constexpr int WC = PT >= 32 ? 2 : 1;
  static constexpr int WR = NCW / WC;
  static constexpr int WM = BM / WR, WN = PT / WC;
  static constexpr int JB = WM / 8, CB = WN / 8;
  static constexpr int A_ELEMS = BM * BK, V_ELEMS = PT * BK;
  static constexpr int MAP_ELEMS = BM * BK / 2;  // int32 panel, counted in doubles
  static constexpr int STAGE_ELEMS = A_ELEMS + V_ELEMS + MAP_ELEMS;
  static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * 8;
  static constexpr uint32_t A_BYTES = A_ELEMS * 8, V_BYTES = V_ELEMS * 8, MAP_BYTES = MAP_ELEMS * 8;
  static constexpr int TILE = BM * PT;
  static constexpr int RING = STAGES * STAGE_ELEMS;
  static constexpr int EPI_ELEMS = TILE + 2 * PT * PT + 64;
  static constexpr int SMEM_ELEMS = RING > EPI_ELEMS ? RING : EPI_ELEMS;
  static constexpr size_t SMEM_BYTES = (size_t)SMEM_ELEMS * 8 + 1024;
};

}  // namespace

template <int PT, int EPI>
__global__ void __launch_bounds__(GCfg<PT>::NTHREADS, 1)
    symv_gather_kernel(const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmU,
                       const __grid_constant__ CUtensorMap tmMap, const __grid_constant__ CUtensorMap tmY, SymvArgs a) {
  using C = GCfg<PT>;
  constexpr int NTHREADS = C::NTHREADS, NGW = C::NGW;
  if (a.skip && *(volatile const int *)a.skip) return;
  extern __shared__ unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES], raw_bar[STAGES];
  __shared__ unsigned s_ticket;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.y, S = gridDim.y;
  const int c0 = PT * blockIdx.z;
  const int tile = blockIdx.x + gridDim.x * blockIdx.z;
  const int n = a.n, p = EPI == EPI_RAW ? min(PT, a.p - c0) : a.p;
  const int j0 = blockIdx.x * BM;
  const int kbeg = split * a.rows_per_split;  // a multiple of BK
  const int kend = min(n, kbeg + a.rows_per_split);
  const int nk = 2 * ((kend - kbeg + BK - 1) / BK);  // stage 2t: M panel of k-tile t, stage 2t + 1: its amap panel

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full_bar[s], 1 + NGW);
      bar_init(&empty_bar[s], NCW);
      bar_init(&raw_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double acc[C::JB][C::CB][2];
#pragma unroll
  for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < C::CB; ++cb) acc[jb][cb][0] = acc[jb][cb][1] = 0.0;

  if (warp == NCW) {
    // ---- producer ----
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % STAGES;
        if (kt >= STAGES) bar_wait(&empty_bar[st], ((kt / STAGES) - 1) & 1);
        double *sa = smem + st * C::STAGE_ELEMS;
        double *sv = sa + C::A_ELEMS;
        const int k0 = kbeg + (kt >> 1) * BK;
        if ((kt & 1) == 0) {
          bar_expect(&full_bar[st], C::A_BYTES + C::V_BYTES);
          tma2d(sa, &tmM, k0, j0, &full_bar[st]);
          tma2d(sa + BM * 16, &tmM, k0 + 16, j0, &full_bar[st]);
          tma2d(sv, &tmU, k0, c0, &full_bar[st]);
          tma2d(sv + PT * 16, &tmU, k0 + 16, c0, &full_bar[st]);
          bar_arrive(&raw_bar[st]);  // nothing to gather: the gather warps pass straight through
        } else {
          bar_expect(&full_bar[st], C::V_BYTES);
          tma2d(sv, &tmY, k0, c0, &full_bar[st]);
          tma2d(sv + PT * 16, &tmY, k0 + 16, c0, &full_bar[st]);
          bar_expect(&raw_bar[st], C::MAP_BYTES);
          tma2d(sv + C::V_ELEMS, &tmMap, k0, j0, &raw_bar[st]);
        }
      }
    }
  } else if (warp > NCW) {
    // ---- gather warps: rows [RG g, RG g + RG) of the panel, one row per step, lane = column ----
    const int g = warp - NCW - 1;
    const double *__restrict__ w = a.w;
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % STAGES;
      bar_wait(&raw_bar[st], (kt / STAGES) & 1);
      if (kt & 1) {
        const uint32_t sa = su32(smem) + st * C::STAGE_BYTES;
        const int *smap = reinterpret_cast<const int *>(smem + st * C::STAGE_ELEMS + C::A_ELEMS + C::V_ELEMS);
        const int k0 = kbeg + (kt >> 1) * BK;
        const bool colok = k0 + lane < n;
        const uint32_t boxoff = sa + (lane >> 4) * BM * 128 + ((lane & 1) << 3);
        const int chunk = (lane & 15) >> 1;
#pragma unroll 1
        for (int r8 = 0; r8 < C::RG; r8 += 8) {
          int id[8];
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) id[u] = smap[(g * C::RG + r8 + u) * BK + lane];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            v[u] = (colok && id[u] >= 0 && j0 + g * C::RG + r8 + u < n) ? __ldg(w + id[u]) : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int row = g * C::RG + r8 + u;
            const uint32_t addr = boxoff + row * 128 + ((chunk ^ (row & 7)) << 4);
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v[u]) : "memory");
          }
        }
        // generic-proxy writes: visible to the consumers (barrier release below) and ordered before the
        // TMA (async-proxy) refill of this stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __threadfence_block();
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&full_bar[st]);
    }
  } else {
    // ---- consumers (as symv_tma.cu) ----
    const int q = lane >> 2, r = lane & 3;
    const int wr = warp % C::WR, wc = warp / C::WR;
    const int arow = wr * C::WM + q;
    const int vrow = wc * C::WN + q;
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % STAGES;
      bar_wait(&full_bar[st], (kt / STAGES) & 1);
      const uint32_t sa = su32(smem) + st * C::STAGE_BYTES;
      const uint32_t sv = sa + C::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int box = ks >> 2, col = ((ks & 3) << 2) + r;
        const uint32_t ba = sa + box * BM * 128, bv = sv + box * PT * 128;
        double af[C::JB], bf[C::CB];
#pragma unroll
        for (int jb = 0; jb < C::JB; ++jb) af[jb] = ldsw(ba, arow + 8 * jb, col);
#pragma unroll
        for (int cb = 0; cb < C::CB; ++cb) bf[cb] = ldsw(bv, vrow + 8 * cb, col);
#pragma unroll
        for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
          for (int cb = 0; cb < C::CB; ++cb) dmma_884(acc[jb][cb][0], acc[jb][cb][1], af[jb], bf[cb]);
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty_bar[st]);
    }
  }
  __syncthreads();  // ring drained: reuse it for the tile

  double *ptile = smem;
  double *gs = smem + C::TILE;
  double *scratch = gs + 2 * PT * PT;
  if (warp < NCW) {
    const int q = lane >> 2, r = lane & 3;
    const int wr = warp % C::WR, wc = warp / C::WR;
#pragma unroll
    for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
      for (int cb = 0; cb < C::CB; ++cb) {
        const int row = wr * C::WM + 8 * jb + q, col = wc * C::WN + 8 * cb + 2 * r;
        ptile[row * PT + col] = acc[jb][cb][0];
        ptile[row * PT + col + 1] = acc[jb][cb][1];
      }
  }
  __syncthreads();
  if (S > 1) {
    double *wp = a.part + ((size_t)tile * S + split) * C::TILE;
    for (int e = threadIdx.x; e < C::TILE; e += NTHREADS) wp[e] = ptile[e];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_ticket = atomicAdd(a.tile_cnt + tile, 1u);
    __syncthreads();
    if (s_ticket != (unsigned)(S - 1)) return;
    __threadfence();
    const double *rp = a.part + (size_t)tile * S * C::TILE;
    for (int e = threadIdx.x; e < C::TILE; e += NTHREADS) ptile[e] = ordered_sum(rp + e, S, (size_t)C::TILE);
    if (threadIdx.x == 0) a.tile_cnt[tile] = 0u;
    __syncthreads();
  }
  tile_epilogue<PT, EPI, BM, NTHREADS>(a, ptile, gs, scratch, &s_ticket, tile, j0, c0, n, p);
}

// 2D int32 tensor map of the index map: n x n (row pitch ld ints), box [128][32] = 128 B rows, no swizzle
static bool make_map_i32(CUtensorMap *m, const int32_t *base, int64_t n, int64_t ld) {
  TmaEncodeFn fn = tma_encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the fused gather-product: symmetric n x n M and index map, HVP epilogue (p <= 64) or raw column chunks
bool symv_gather_supported(const SymvArgs &a, int epi, bool atr) {
  if (atr || a.k > 0 || a.ncols > 0 || !a.amap || !a.w || !a.X) return false;
  if (epi != EPI_HVP && epi != EPI_RAW) return false;
  if (epi == EPI_HVP && a.p > 64) return false;
  if ((a.lda & 1) || ((uintptr_t)a.A & 15) || (a.ldm & 3) || ((uintptr_t)a.amap & 15)) return false;
  return tma_encoder() != nullptr;
}
int symv_gather_kstep() { return BK; }

template <int PT, int EPI>
static cudaError_t gather_launch_t(const SymvArgs &a, const CUtensorMap *m, int S, cudaStream_t st) {
  using C = GCfg<PT>;
  auto k = symv_gather_kernel<PT, EPI>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nz = EPI == EPI_RAW ? (a.p + PT - 1) / PT : 1;
  dim3 grid((a.n + BM - 1) / BM, S, nz);
  k<<<grid, C::NTHREADS, C::SMEM_BYTES, st>>>(m[0], m[1], m[2], m[3], a);
  return cudaGetLastError();
}

// Vt: workspace of 2 p ldvt doubles (U^T then Y^T), ldvt = round_up(n, 2); a.V = U, a.X = Y
cudaError_t symv_gather_launch(const SymvArgs &a, int epi, int S, double *Vt, int64_t ldvt, cudaStream_t st) {
  const int pt = symv_tma_pt(a.p, epi);
  cudaError_t e = symv_transpose(a.n, a.p, a.V, a.ldv, Vt, ldvt, a.skip, st);
  if (e != cudaSuccess) return e;
  double *Vt2 = Vt + (size_t)a.p * ldvt;
  e = symv_transpose(a.n, a.p, a.X, a.ldx, Vt2, ldvt, a.skip, st);
  if (e != cudaSuccess) return e;
  CUtensorMap m[4];
  if (!tma_map_f64(&m[0], a.A, a.n, a.n, a.lda, BM) || !tma_map_f64(&m[1], Vt, a.p, a.n, ldvt, pt) ||
      !make_map_i32(&m[2], a.amap, a.n, a.ldm) || !tma_map_f64(&m[3], Vt2, a.p, a.n, ldvt, pt))
    return cudaErrorInvalidValue;
  const bool raw = epi == EPI_RAW;
  switch (pt) {
    case 8: return raw ? gather_launch_t<8, EPI_RAW>(a, m, S, st) : gather_launch_t<8, EPI_HVP>(a, m, S, st);
    case 16: return raw ? gather_launch_t<16, EPI_RAW>(a, m, S, st) : gather_launch_t<16, EPI_HVP>(a, m, S, st);
    case 32: return raw ? gather_launch_t<32, EPI_RAW>(a, m, S, st) : gather_launch_t<32, EPI_HVP>(a, m, S, st);
    default: return raw ? gather_launch_t<64, EPI_RAW>(a, m, S, st) : gather_launch_t<64, EPI_HVP>(a, m, S, st);
  }
}

}  // namespace drsdp
