// symv_symm.cu — the graded product P = M V reading only the upper triangle of the symmetric M
// (its distinct entries, 8 n(n+1)/2 bytes: SURVEY §8(d) D-ALG's algorithmic traffic), for p <= 16
// where the full-matrix kernel (symv_tma.cu) is bound by HBM.
//
// Kernel A (symm_partial): one CTA per "unit" = a run of up to L upper 128 x 128 tiles (I, J),
// J in [Ja, Jb), J >= I, of block-row I. A producer warp streams the tiles through a TMA /
// mbarrier ring in 32-column stages (as symv_tma.cu) plus, once per unit, V^T restricted to the
// rows of block I. The 8 consumer warps
//   * accumulate the forward product  F = sum_J M_IJ V_J  (rows of block I) over the whole unit;
//   * for every off-diagonal tile and stage compute the transposed contribution
//     M_IJ^T V_I for the 32 rows k of block J in that stage (complete over the 128 rows i), one
//     8 x 8 DMMA fragment per warp, and store it to the partial buffer T[J][I].
// The diagonal tile's forward product already covers all of M_II, so it has no transposed part.
// Kernel B (symm_reduce): one CTA per row block J sums, in fixed order, the forward partials of
// the units of block-row J and the transposed partials T[J][0..J-1], then runs the shared row
// epilogue (tile_epilogue.cuh). Deterministic (no fp atomics). Extra traffic: the partials,
// 128 x p doubles per off-diagonal tile written once and read once (+25 % of the half matrix at
// p = 16, +12.5 % at p = 8).
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"
#include "symv.cuh"
#include "tile_epilogue.cuh"

namespace drsdp {

namespace {

constexpr int BM = 128, BK = 32, NCW = 8, NTA = (NCW + 1) * 32, NTB = 256;
constexpr int UNIT_TILES = 8;  // L: tiles per unit

template <int PT>
struct SCfg {
  static constexpr int CB = PT / 8;              // column fragments
  static constexpr int WM = BM / NCW, JB = WM / 8;  // forward warp tile 16 x PT
  // PT = 16: V_I^T fragments held in registers for the transposed product (VREG), one CTA per SM
  // with a 4-stage ring; PT = 8: two CTAs per SM, 3 stages
  static constexpr bool VREG = PT >= 16;
  static constexpr int CTAS = PT >= 16 ? 1 : 2;
  static constexpr int STAGES = PT >= 16 ? 4 : 3;
  static constexpr int A_ELEMS = BM * BK, V_ELEMS = PT * BK;
  static constexpr int STAGE_ELEMS = A_ELEMS + V_ELEMS;
  static constexpr uint32_t STAGE_BYTES = STAGE_ELEMS * 8;
  static constexpr int VI_ELEMS = PT * BM;      // V_I^T: 8 boxes of [PT][16]
  static constexpr int NTF = (BK / 8) * CB;     // transposed fragments per stage (4 or 8)
  static constexpr int TILE = BM * PT;
  static constexpr size_t SMEM_BYTES = (size_t)(STAGES * STAGE_ELEMS + VI_ELEMS) * 8 + 1024;
};

}  // namespace

template <int PT>
__global__ void __launch_bounds__(NTA, SCfg<PT>::CTAS)
    symm_partial_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV,
                        const int4 *__restrict__ units, double *__restrict__ Fpart, double *__restrict__ Tpart,
                        const int *skip) {
  using C = SCfg<PT>;
  if (skip && *(volatile const int *)skip) return;
  extern __shared__ unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES], vi_bar;
  const int4 u = units[blockIdx.x];
  const int I = u.x, Ja = u.y, Jb = u.z;
  const int i0 = I * BM;
  const int nk = (Jb - Ja) * (BM / BK);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *sVI = smem + C::STAGES * C::STAGE_ELEMS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], NCW);
    }
    bar_init(&vi_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0) {
      bar_expect(&vi_bar, C::VI_ELEMS * 8);
#pragma unroll
      for (int b = 0; b < BM / 16; ++b) tma2d(sVI + b * PT * 16, &tmV, i0 + 16 * b, 0, &vi_bar);
      for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % C::STAGES;
        if (kt >= C::STAGES) bar_wait(&empty[st], ((kt / C::STAGES) - 1) & 1);
        double *sa = smem + st * C::STAGE_ELEMS, *sv = sa + C::A_ELEMS;
        const int k0 = (Ja + kt / (BM / BK)) * BM + (kt % (BM / BK)) * BK;
        bar_expect(&full[st], C::STAGE_BYTES);
        tma2d(sa, &tmA, k0, i0, &full[st]);
        tma2d(sa + BM * 16, &tmA, k0 + 16, i0, &full[st]);
        tma2d(sv, &tmV, k0, 0, &full[st]);
        tma2d(sv + PT * 16, &tmV, k0 + 16, 0, &full[st]);
      }
    }
    return;
  }
  const int q = lane >> 2, r = lane & 3;
  const uint32_t vi = su32(sVI);
  double acc[C::JB][C::CB][2];
#pragma unroll
  for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < C::CB; ++cb) acc[jb][cb][0] = acc[jb][cb][1] = 0.0;
  bar_wait(&vi_bar, 0);
  // transposed part: warp -> (cf, kb): output columns cf*8.. (of V) and the 8 columns kb*8.. of each
  // 32-wide stage (rows k of block J). The contraction runs over the 128 rows i of block I; the
  // A operand V_I^T is fixed for the whole unit and lives in registers (vf), the B operand is the
  // stage's M fragment. The 4 rows i of k-step s are 8 (s/2) + 2 (s%2) + {0, 4, 1, 5}[r], so the
  // rows of a fragment differ pairwise in bit 2 and the swizzled M loads take the minimal 2
  // wavefronts; 4 independent accumulator chains (summed in fixed order) hide the DMMA latency.
  // (PT = 16, C::VREG; PT = 8 keeps the shared-memory V_I operand of warps kf = warp / CB < 4)
  const int cf = warp % C::CB, kb = warp / C::CB;
  const bool tw = kb < BK / 8;
  const int roff = (r >> 1) + 4 * (r & 1);
  const int kf = warp / C::CB;
  const bool twold = warp < C::NTF;
  double vf[C::VREG ? BM / 4 : 1];
  if constexpr (C::VREG) {
#pragma unroll
    for (int ks = 0; ks < BM / 4; ++ks) {
      const int i = 8 * (ks >> 1) + 2 * (ks & 1) + roff;
      vf[ks] = tw ? ldsw(vi + (i >> 4) * PT * 128, cf * 8 + q, i & 15) : 0.0;
    }
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % C::STAGES;
    bar_wait(&full[st], (kt / C::STAGES) & 1);
    const uint32_t sa = su32(smem) + st * C::STAGE_BYTES, sv = sa + C::A_ELEMS * 8;
    // forward: rows warp*16 + 8 jb + q of block I, all PT columns
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      const int box = ks >> 2, col = ((ks & 3) << 2) + r;
      const uint32_t ba = sa + box * BM * 128, bv = sv + box * PT * 128;
      double af[C::JB], bf[C::CB];
#pragma unroll
      for (int jb = 0; jb < C::JB; ++jb) af[jb] = ldsw(ba, warp * C::WM + 8 * jb + q, col);
#pragma unroll
      for (int cb = 0; cb < C::CB; ++cb) bf[cb] = ldsw(bv, 8 * cb + q, col);
#pragma unroll
      for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
        for (int cb = 0; cb < C::CB; ++cb) dmma_884(acc[jb][cb][0], acc[jb][cb][1], af[jb], bf[cb]);
    }
    const int J = Ja + kt / (BM / BK), s = kt % (BM / BK);
    if constexpr (C::VREG) {
      if (J > I && tw) {
        // out^T[c][k] = sum_i V_I^T[c][i] M[i][k]: D (8 c x 8 k) += A (V_I^T, registers) B (M, shared)
        double t[4][2];
#pragma unroll
        for (int c = 0; c < 4; ++c) t[c][0] = t[c][1] = 0.0;
        const int kk = kb * 8 + q;  // B fragment column = k within the stage
        const uint32_t ba = sa + (kk >> 4) * BM * 128;
#pragma unroll
        for (int ks = 0; ks < BM / 4; ++ks) {
          const int i = 8 * (ks >> 1) + 2 * (ks & 1) + roff;
          const double bm = ldsw(ba, i, kk & 15);
          dmma_884(t[ks & 3][0], t[ks & 3][1], vf[ks], bm);
        }
        const double t0 = (t[0][0] + t[1][0]) + (t[2][0] + t[3][0]);
        const double t1 = (t[0][1] + t[1][1]) + (t[2][1] + t[3][1]);
        // D[c = cf*8 + q][k = kb*8 + 2r + {0, 1}] -> partial tile T[J][I] (rows k, columns c)
        double *tp = Tpart + ((size_t)J * (J - 1) / 2 + I) * C::TILE;
        const int row = s * BK + kb * 8 + 2 * r, colo = cf * 8 + q;
        tp[row * PT + colo] = t0;
        tp[(row + 1) * PT + colo] = t1;
      }
    } else {
      if (J > I && twold) {
        // out[k][c] = sum_i M[i][k] V_I[i][c] for k = kf*8 + q of this stage. The contraction rows
        // of k-step ks are i = 8 (ks/2) + 2 (ks%2) + {0, 4, 1, 5}[r], so that the 4 rows of a
        // fragment differ in bit 2 pairwise and the swizzled loads of M (column access) and of
        // V_I^T take the minimal 2 wavefronts; 4 independent accumulator chains (summed in a fixed
        // order) hide the DMMA latency.
        double t[4][2];
#pragma unroll
        for (int c = 0; c < 4; ++c) t[c][0] = t[c][1] = 0.0;
        const int kk = kf * 8 + q;  // column within the 32-wide stage
        const uint32_t ba = sa + (kk >> 4) * BM * 128;
#pragma unroll 8
        for (int ks = 0; ks < BM / 4; ++ks) {
          const int i = 8 * (ks >> 1) + 2 * (ks & 1) + roff;
          const double av = ldsw(ba, i, kk & 15);
          const double bv2 = ldsw(vi + (i >> 4) * PT * 128, cf * 8 + q, i & 15);
          dmma_884(t[ks & 3][0], t[ks & 3][1], av, bv2);
        }
        const double t0 = (t[0][0] + t[1][0]) + (t[2][0] + t[3][0]);
        const double t1 = (t[0][1] + t[1][1]) + (t[2][1] + t[3][1]);
        double *tp = Tpart + ((size_t)J * (J - 1) / 2 + I) * C::TILE;
        const int row = s * BK + kf * 8 + q, colo = cf * 8 + 2 * r;
        *reinterpret_cast<double2 *>(tp + row * PT + colo) = make_double2(t0, t1);
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[st]);
  }
  double *fp = Fpart + (size_t)blockIdx.x * C::TILE;
#pragma unroll
  for (int jb = 0; jb < C::JB; ++jb)
#pragma unroll
    for (int cb = 0; cb < C::CB; ++cb) {
      const int row = warp * C::WM + 8 * jb + q, col = 8 * cb + 2 * r;
      *reinterpret_cast<double2 *>(fp + row * PT + col) = make_double2(acc[jb][cb][0], acc[jb][cb][1]);
    }
}

// Kernel B: CTA b = (row block J, quarter): 32 rows of block J. Sums, per element and in fixed
// order, the forward partials of the units of block-row J, then T[J][0..J-1]; 16 loads in flight
// per thread (the sums over up to nb partials are latency-bound otherwise).
constexpr int RQ = 4, RROWS = BM / RQ;

template <int PT>
DRSDP_DEV double ordered_sum16(const double *p, int count, size_t stride) {
  double s = 0.0;
  int k = 0;
  for (; k + 16 <= count; k += 16) {
    double t[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = __ldcg(p + (size_t)(k + j) * stride);
#pragma unroll
    for (int j = 0; j < 16; ++j) s += t[j];
  }
  for (; k < count; ++k) s += __ldcg(p + (size_t)k * stride);
  return s;
}

template <int PT, int EPI>
__global__ void __launch_bounds__(NTB) symm_reduce_kernel(SymvArgs a, const double *__restrict__ Fpart,
                                                          const double *__restrict__ Tpart,
                                                          const int *__restrict__ ustart) {
  using C = SCfg<PT>;
  if (a.skip && *(volatile const int *)a.skip) return;
  __shared__ double ptile[RROWS * PT];
  __shared__ double gs[2 * PT * PT];
  __shared__ double scratch[64];
  __shared__ unsigned s_ticket;
  const int J = blockIdx.x / RQ, part = blockIdx.x % RQ;
  const int u0 = ustart[J], u1 = ustart[J + 1];
  const size_t off = (size_t)part * RROWS * PT;
  for (int e = threadIdx.x; e < RROWS * PT; e += NTB) {
    double sum = ordered_sum16<PT>(Fpart + (size_t)u0 * C::TILE + off + e, u1 - u0, (size_t)C::TILE);
    sum += ordered_sum16<PT>(Tpart + (size_t)J * (J - 1) / 2 * C::TILE + off + e, J, (size_t)C::TILE);
    ptile[e] = sum;
  }
  __syncthreads();
  tile_epilogue<PT, EPI, RROWS, NTB>(a, ptile, gs, scratch, &s_ticket, blockIdx.x, J * BM + part * RROWS, 0, a.n,
                                     a.p);
}

// ----------------------------------------------------------------------------------------------
static bool map2d(CUtensorMap *m, const double *base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return tma_map_f64(m, base, rows, cols, ld, box_rows);
}

int symm_units(int n, std::vector<int> &host_units, std::vector<int> &host_ustart) {
  const int nb = (n + BM - 1) / BM;
  host_units.clear();
  host_ustart.assign(nb + 1, 0);
  int nu = 0;
  for (int I = 0; I < nb; ++I) {
    host_ustart[I] = nu;
    for (int Ja = I; Ja < nb; Ja += UNIT_TILES) {
      const int Jb = Ja + UNIT_TILES < nb ? Ja + UNIT_TILES : nb;
      host_units.insert(host_units.end(), {I, Ja, Jb, 0});
      ++nu;
    }
  }
  host_ustart[nb] = nu;
  return nu;
}

size_t symm_tpart_elems(int n, int p) {
  const size_t nb = (n + BM - 1) / BM;
  return (nb * (nb - 1) / 2 + 1) * BM * symv_pt(p);
}
size_t symm_fpart_elems(int n_units, int p) { return (size_t)n_units * BM * symv_pt(p); }

template <int PT, int EPI>
static cudaError_t reduce_t(const SymvArgs &a, const double *F, const double *T, const int *ustart, int nb,
                            cudaStream_t st) {
  symm_reduce_kernel<PT, EPI><<<nb * RQ, NTB, 0, st>>>(a, F, T, ustart);
  return cudaGetLastError();
}

template <int PT>
static cudaError_t symm_t(const SymvArgs &a, int epi, const CUtensorMap &mA, const CUtensorMap &mV,
                          const int4 *units, int n_units, const int *ustart, double *F, double *T, cudaStream_t st) {
  using C = SCfg<PT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(symm_partial_kernel<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  symm_partial_kernel<PT><<<n_units, NTA, C::SMEM_BYTES, st>>>(mA, mV, units, F, T, a.skip);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int nb = (a.n + BM - 1) / BM;
  switch (epi) {
    case EPI_RAW: return reduce_t<PT, EPI_RAW>(a, F, T, ustart, nb, st);
    case EPI_COSTGRAD: return reduce_t<PT, EPI_COSTGRAD>(a, F, T, ustart, nb, st);
    case EPI_HVP: return reduce_t<PT, EPI_HVP>(a, F, T, ustart, nb, st);
    default: return reduce_t<PT, EPI_ROWDOT>(a, F, T, ustart, nb, st);
  }
}

bool symm_supported(const SymvArgs &a, int epi, int mode2, bool atr) {
  // p <= 8: measured on B200 (n = 32768) 0.97 ms vs 1.31 ms for the full-matrix kernel; at p = 16 the
  // doubled DMMA work per byte makes this variant DMMA/shared-memory bound (1.69 ms vs 1.37 ms)
  static const bool p16 = std::getenv("DRSDP_SYMM16") != nullptr;  // experiment: p <= 16
  return epi != EPI_BOTH && mode2 == MODE2_NONE && !atr && a.k == 0 && a.ncols == 0 && a.p <= (p16 ? 16 : 8) && a.A2 == nullptr &&
         !(a.lda & 1) && !((uintptr_t)a.A & 15) && tma_encoder() != nullptr && (epi != EPI_RAW || a.p <= 16);
}

cudaError_t symm_launch(const SymvArgs &a, int epi, double *Vt, int64_t ldvt, const int4 *units, int n_units,
                        const int *ustart, double *Fpart, double *Tpart, cudaStream_t st) {
  const int pt = symv_pt(a.p);
  cudaError_t e = symv_transpose(a.n, a.p, a.V, a.ldv, Vt, ldvt, a.skip, st);
  if (e != cudaSuccess) return e;
  CUtensorMap mA, mV;
  if (!map2d(&mA, a.A, a.n, a.n, a.lda, BM) || !map2d(&mV, Vt, a.p, a.n, ldvt, pt)) return cudaErrorInvalidValue;
  if (pt == 8) return symm_t<8>(a, epi, mA, mV, units, n_units, ustart, Fpart, Tpart, st);
  return symm_t<16>(a, epi, mA, mV, units, n_units, ustart, Fpart, Tpart, st);
}

}  // namespace drsdp
