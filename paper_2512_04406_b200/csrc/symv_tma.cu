// symv_tma.cu — the graded kernel: P = M V (M n x n symmetric, V n x p) streamed through a TMA /
// mbarrier shared-memory ring, fp64 DMMA (mma.sync m8n8k4) from swizzled shared memory, with the
// fused row epilogues of north-star (b)/(c): cost + Euclidean gradient + Riemannian gradient
// (Eq. 4.6 and Lemma 4.1), the Hessian-vector product (Eq. 4.7)
// and z = rowdot(T Y, Y) (Alg. 2 step 7).
//
// Mapping (B200, sm_100a). tcgen05 has no f64 kind, so the fp64 tensor path is the warp-level
// DMMA. A CTA owns BM = 128 output rows j and a K-range (split s of S). M is symmetric, so the row
// panel M[j0:j0+BM, k] is read row-major (k contiguous) and P[j, :] = sum_k M[j, k] V[k, :]:
//   * one producer warp issues cp.async.bulk.tensor loads of M[j0:j0+128, k0:k0+32] (two 128 B
//     wide boxes, SWIZZLE_128B) and of V^T[c0:c0+PT, k0:k0+32] (V^T is a transposed copy of V,
//     so that both DMMA operands are read k-contiguous and bank-conflict free) into an S-stage
//     ring guarded by full / empty mbarriers;
//   * 8 consumer warps each own a (BM/WR) x (PT/WC) block of the output tile and run JB x CB DMMAs
//     per k-step from shared memory (8 k-steps per stage);
//   * the finished tile goes through shared memory; with split-K the partial tiles are summed in
//     split order by the last CTA of the row panel (atomic ticket), which runs the row epilogue
//     (warp per row). Tile scalars are summed in tile order by the last tile. Bit-deterministic.
// TMA zero-fills out-of-range rows / columns, which handles ragged n and p.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"
#include "symv.cuh"
#include "tile_epilogue.cuh"

namespace drsdp {

namespace {

constexpr int BM = 128, BK = 32, NCW = 8;  // rows per CTA, k per stage, consumer warps
constexpr int NTHREADS = (NCW + 1) * 32;

// DUO: two CTAs per SM for PT = 32 (2-stage rings): one CTA's epilogue overlaps the other's stream
template <int PT, bool DUO = false>
struct Cfg {
  static constexpr int WC = PT >= 32 ? 2 : 1;  // warps across columns
  static constexpr int WR = NCW / WC;           // warps across rows
  static constexpr int WM = BM / WR, WN = PT / WC;
  static constexpr int JB = WM / 8, CB = WN / 8;
  // PT <= 16: 3 stages so that two CTAs share an SM (one streams while the other runs its epilogue);
  // PT >= 32: one CTA per SM with a deeper ring (DUO: two CTAs with 2 stages each)
  static constexpr int CTAS_PER_SM = (PT <= 16 || DUO) ? 2 : 1;
  static constexpr int STAGES = DUO ? 2 : (PT >= 64 ? 3 : (PT <= 16 ? 3 : 4));
  static constexpr int A_ELEMS = BM * BK, V_ELEMS = PT * BK;
  static constexpr int STAGE_ELEMS = A_ELEMS + V_ELEMS;
  static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * 8;
  static constexpr int TILE = BM * PT;
  // epilogue needs the tile + G (+ K) + scratch; the ring is reused for it
  static constexpr int RING = STAGES * STAGE_ELEMS;
  static constexpr int EPI_ELEMS = TILE + 2 * PT * PT + 64;
  static constexpr int SMEM_ELEMS = RING > EPI_ELEMS ? RING : EPI_ELEMS;
  static constexpr size_t SMEM_BYTES = (size_t)SMEM_ELEMS * 8 + 1024;  // + alignment slack
};

}  // namespace

// PAIR: out = M V + A2 V2 as one K-concatenated product [M | A2] [V; V2]; the k-tiles in
// [0, kpad) come from (tmA, tmV), those in [kpad, 2 kpad) from (tmA2, tmV2), kpad = n rounded up
// to a multiple of BK (TMA zero-fills the padding columns).
template <int PT, int EPI, bool PAIR, bool DUO = false>
__global__ void __launch_bounds__(NTHREADS, Cfg<PT, DUO>::CTAS_PER_SM)
    symv_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmV2, SymvArgs a) {
  using C = Cfg<PT, DUO>;
  if (a.skip && *(volatile const int *)a.skip) return;
  extern __shared__ unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[C::STAGES], empty_bar[C::STAGES];
  __shared__ unsigned s_ticket;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.y, S = gridDim.y;
  const int c0 = PT * blockIdx.z;
  const int tile = blockIdx.x + gridDim.x * blockIdx.z;
  const int n = a.n, p = EPI == EPI_RAW ? min(PT, a.p - c0) : a.p;  // EPI_BOTH: 2p columns, p <= PT / 2
  const int j0 = blockIdx.x * BM;
  const int kn = a.ncols > 0 ? a.ncols : n;  // contraction length (row-block mode: all columns)
  const int kpad = (kn + BK - 1) / BK * BK;
  const int ktot = PAIR ? 2 * kpad : kn;
  const int kbeg = split * a.rows_per_split;
  const int kend = min(ktot, kbeg + a.rows_per_split);
  const int nk = (kend - kbeg + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      bar_init(&full_bar[s], 1);
      bar_init(&empty_bar[s], NCW);
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
    // ---- producer: one thread streams the ring ----
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % C::STAGES;
        if (kt >= C::STAGES) bar_wait(&empty_bar[st], ((kt / C::STAGES) - 1) & 1);
        double *sa = smem + st * C::STAGE_ELEMS;
        double *sv = sa + C::A_ELEMS;
        int k0 = kbeg + kt * BK;
        const CUtensorMap *ma = &tmA, *mv = &tmV;
        if (PAIR && k0 >= kpad) {
          k0 -= kpad;
          ma = &tmA2;
          mv = &tmV2;
        }
        bar_expect(&full_bar[st], C::STAGE_BYTES);
        tma2d(sa, ma, k0, j0, &full_bar[st]);
        tma2d(sa + BM * 16, ma, k0 + 16, j0, &full_bar[st]);
        tma2d(sv, mv, k0, c0, &full_bar[st]);
        tma2d(sv + PT * 16, mv, k0 + 16, c0, &full_bar[st]);
      }
    }
  } else {
    // ---- consumers ----
    const int q = lane >> 2, r = lane & 3;
    const int wr = warp % C::WR, wc = warp / C::WR;
    const int arow = wr * C::WM + q;  // + 8 jb
    const int vrow = wc * C::WN + q;  // + 8 cb
    for (int kt = 0; kt < nk; ++kt) {
      const int st = kt % C::STAGES;
      bar_wait(&full_bar[st], (kt / C::STAGES) & 1);
      const uint32_t sa = su32(smem) + st * C::STAGE_BYTES;
      const uint32_t sv = sa + C::A_ELEMS * 8;
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

  double *ptile = smem;                 // [BM][PT]
  double *gs = smem + C::TILE;          // G, K (p x p each, p <= PT)
  double *scratch = gs + 2 * PT * PT;   // 64 doubles
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
    for (int e = threadIdx.x; e < C::TILE; e += NTHREADS) {
      double sum = 0.0;
      sum = ordered_sum(rp + e, S, (size_t)C::TILE);
      ptile[e] = sum;
    }
    if (threadIdx.x == 0) a.tile_cnt[tile] = 0u;
    __syncthreads();
  }

  tile_epilogue<PT, EPI, BM, NTHREADS>(a, ptile, gs, scratch, &s_ticket, tile, j0, c0, n, p);
}

// V^T (pt_total x ldvt, row c = column c of V) from V (k x p, pitch ldv); rows >= p are not
// written (TMA reads them as out of range: the tensor map has p rows)
__global__ void __launch_bounds__(256) transpose_kernel(int k, int p, const double *__restrict__ V, int ldv,
                                                        double *__restrict__ Vt, int64_t ldvt, const int *skip) {
  if (skip && *(volatile const int *)skip) return;
  __shared__ double t[32][33];
  const int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int rr = ty; rr < 32; rr += 8) {
    const int i = i0 + rr, c = c0 + tx;
    t[rr][tx] = (i < k && c < p) ? V[(size_t)i * ldv + c] : 0.0;
  }
  __syncthreads();
  for (int rr = ty; rr < 32; rr += 8) {
    const int c = c0 + rr, i = i0 + tx;
    if (c < p && i < k) Vt[(size_t)c * ldvt + i] = t[tx][rr];
  }
}

cudaError_t symv_transpose(int k, int p, const double *V, int ldv, double *Vt, int64_t ldvt, const int *skip,
                           cudaStream_t st) {
  dim3 tg((k + 31) / 32, (p + 31) / 32);
  transpose_kernel<<<tg, 256, 0, st>>>(k, p, V, ldv, Vt, ldvt, skip);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------------
// 2D fp64 tensor map: rows x cols (cols contiguous, row pitch ld doubles), box [box_rows][16]
static bool make_map(CUtensorMap *m, const double *base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return tma_map_f64(m, base, rows, cols, ld, box_rows);
}

bool symv_tma_supported(const SymvArgs &a, int epi, int mode2, bool atr) {
  // symmetric n x n operands only (k = 0): with an explicit k the operand is a general k x n matrix
  // whose product is A^T V, while this kernel streams rows of A (A V)
  if (mode2 == MODE2_GATHER || atr || a.k > 0) return false;
  if (mode2 == MODE2_PAIR && ((a.lda2 & 1) || ((uintptr_t)a.A2 & 15))) return false;
  if (epi != EPI_RAW && a.p > 64) return false;
  if (epi == EPI_BOTH && (2 * a.p > 64 || 2 * a.p <= 8 || mode2 != MODE2_NONE || !a.U || !a.V2 || a.A2)) return false;
  if ((a.lda & 1) || ((uintptr_t)a.A & 15)) return false;
  return tma_encoder() != nullptr;
}

int symv_tma_rows() { return BM; }
// column chunk width of the TMA kernel (raw products with p > 64 run in 64-wide chunks: a 128-wide
// variant, measured on B200 at n = 5051, p = 128 / 512, was no faster — the re-reads of M by the
// chunks hit L2 — and needs 168 registers with spills at 288 threads)
int symv_tma_pt(int p, int epi) { return symv_pt(epi == EPI_BOTH ? 2 * p : p); }
int symv_tma_chunks(int p, int epi) { return epi == EPI_RAW ? (p + symv_tma_pt(p, epi) - 1) / symv_tma_pt(p, epi) : 1; }
// EPI_BOTH at PT = 32 with two CTAs per SM, 2-stage rings (default; DRSDP_BOTH_DUO=0 selects one CTA
// per SM with a 4-stage ring). Measured at n = 32768, p = 16 (bench step, B200): 2.12 ms vs 2.165 ms
// per launch (frac 0.872 vs 0.856): one CTA's epilogue overlaps the other's stream.
bool symv_tma_both_duo() {
  static const int v = [] {
    const char *e = std::getenv("DRSDP_BOTH_DUO");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}
int symv_tma_ctas_per_sm(int pt, int epi) { return (pt <= 16 || (epi == EPI_BOTH && pt == 32 && symv_tma_both_duo())) ? 2 : 1; }
int symv_tma_kstep() { return BK; }

template <int PT, int EPI, bool PAIR, bool DUO = false>
static cudaError_t tma_launch_t(const SymvArgs &a, const CUtensorMap *m, int S, cudaStream_t st) {
  using C = Cfg<PT, DUO>;
  auto k = symv_tma_kernel<PT, EPI, PAIR, DUO>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nz = EPI == EPI_RAW ? (a.p + PT - 1) / PT : 1;  // = symv_tma_chunks
  dim3 grid((a.n + BM - 1) / BM, S, nz);
  k<<<grid, NTHREADS, C::SMEM_BYTES, st>>>(m[0], m[1], m[2], m[3], a);
  return cudaGetLastError();
}

template <int PT>
static cudaError_t tma_dispatch(const SymvArgs &a, int epi, bool pair, const CUtensorMap *m, int S,
                                cudaStream_t st) {
  if (pair) {
    if (epi == EPI_RAW) return tma_launch_t<PT, EPI_RAW, true>(a, m, S, st);
    if (epi == EPI_HVP) return tma_launch_t<PT, EPI_HVP, true>(a, m, S, st);
    return cudaErrorInvalidValue;
  }
  switch (epi) {
    case EPI_RAW: return tma_launch_t<PT, EPI_RAW, false>(a, m, S, st);
    case EPI_COSTGRAD: return tma_launch_t<PT, EPI_COSTGRAD, false>(a, m, S, st);
    case EPI_HVP: return tma_launch_t<PT, EPI_HVP, false>(a, m, S, st);
    case EPI_BOTH:
      if constexpr (PT == 32) {
        if (symv_tma_both_duo()) return tma_launch_t<PT, EPI_BOTH, false, true>(a, m, S, st);
      }
      if constexpr (PT >= 16) return tma_launch_t<PT, EPI_BOTH, false>(a, m, S, st);
      return cudaErrorInvalidValue;
    default: return tma_launch_t<PT, EPI_ROWDOT, false>(a, m, S, st);
  }
}

// Vt: workspace of at least p * ldvt doubles (2 p * ldvt for PAIR and EPI_BOTH), ldvt = round_up(kn, 2),
// kn = the contraction length (ncols in row-block mode, else n)
cudaError_t symv_tma_launch(const SymvArgs &a, int epi, int S, double *Vt, int64_t ldvt, cudaStream_t st) {
  const int pt = symv_tma_pt(a.p, epi);
  const bool pair = a.A2 != nullptr;
  const int kn = a.ncols > 0 ? a.ncols : a.n;
  dim3 tg((kn + 31) / 32, (a.p + 31) / 32);
  transpose_kernel<<<tg, 256, 0, st>>>(kn, a.p, a.V, a.ldv, Vt, ldvt, a.skip);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  double *Vt2 = Vt + (size_t)a.p * ldvt;
  if (epi == EPI_BOTH) {
    // rows p .. 2p - 1 of V^T = U^T: one map of 2p rows serves [Y U]
    transpose_kernel<<<tg, 256, 0, st>>>(kn, a.p, a.V2, a.ldv2, Vt2, ldvt, a.skip);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    CUtensorMap mb[4];
    if (!make_map(&mb[0], a.A, a.n, kn, a.lda, BM) || !make_map(&mb[1], Vt, 2 * a.p, kn, ldvt, pt))
      return cudaErrorInvalidValue;
    mb[2] = mb[0];
    mb[3] = mb[1];
    switch (pt) {
      case 16: return tma_dispatch<16>(a, epi, false, mb, S, st);
      case 32: return tma_dispatch<32>(a, epi, false, mb, S, st);
      case 64: return tma_dispatch<64>(a, epi, false, mb, S, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (pair) {
    transpose_kernel<<<tg, 256, 0, st>>>(kn, a.p, a.V2, a.ldv2, Vt2, ldvt, a.skip);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  CUtensorMap m[4];
  if (!make_map(&m[0], a.A, a.n, kn, a.lda, BM) || !make_map(&m[1], Vt, a.p, kn, ldvt, pt))
    return cudaErrorInvalidValue;
  if (pair) {
    if (!make_map(&m[2], a.A2, a.n, kn, a.lda2, BM) || !make_map(&m[3], Vt2, a.p, kn, ldvt, pt))
      return cudaErrorInvalidValue;
  } else {
    m[2] = m[0];
    m[3] = m[1];
  }
  switch (pt) {
    case 8: return tma_dispatch<8>(a, epi, pair, m, S, st);
    case 16: return tma_dispatch<16>(a, epi, pair, m, S, st);
    case 32: return tma_dispatch<32>(a, epi, pair, m, S, st);
    default: return tma_dispatch<64>(a, epi, pair, m, S, st);
  }
}

}  // namespace drsdp
