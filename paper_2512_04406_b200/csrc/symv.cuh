// symv.cuh — interface of the fused tall-skinny symmetric product kernels (symv.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace drsdp {

// EPI_BOTH: one product M [Y U] (V = Y, V2 = U: V^T rows 0..p-1 = Y^T, p..2p-1 = U^T) with the
// COSTGRAD epilogue on columns [0, p) and the HVP epilogue on columns [p, 2p) of the same row (TMA
// kernel, 8 < 2p <= 64)
enum Epi { EPI_RAW = 0, EPI_COSTGRAD = 1, EPI_HVP = 2, EPI_ROWDOT = 3, EPI_BOTH = 4 };
// second product accumulated into the same tile: none, the ALM gather-product sum_i w[amap_ij] X_i,
// or a plain second pair A2^T V2 (A2 V2 when ATR)
enum Mode2 { MODE2_NONE = 0, MODE2_GATHER = 1, MODE2_PAIR = 2 };

struct SymvArgs {
  // out (n x p) = A^T V with A k x n (element (i, j) at A[i lda + j]; A symmetric n x n for the
  // subproblem product M Y), or, with ATR, out = A V with A n x k (element (j, i) at A[j lda + i]).
  // V is k x p (pitch ldv). k = 0 means k = n.
  const double *A = nullptr;
  int64_t lda = 0;
  int n = 0, p = 0, k = 0;
  // row-block mode of the TMA kernel (row-sharded evaluation): A holds n rows of a
  // symmetric ncols x ncols matrix (output rows), contracted against all ncols rows of V; the
  // epilogue operands (Y, U, rho, outputs) are then the block's own n rows. 0 = square (ncols = n).
  int ncols = 0;
  const int *skip = nullptr;  // device flag: when non-zero at launch time the kernel does nothing
  // MODE2_PAIR: second operand pair, same access pattern as (A, V)
  const double *A2 = nullptr;
  int64_t lda2 = 0;
  const double *V2 = nullptr;
  int ldv2 = 0;
  const double *V = nullptr;
  int ldv = 0;
  // optional gather-product: acc += sum_i w[amap[i, j]] X[i, :]  (ALM HVP projection term)
  const int32_t *amap = nullptr;
  int64_t ldm = 0;
  const double *w = nullptr;
  const double *X = nullptr;
  int ldx = 0;
  // split-K
  int rows_per_split = 0;
  double *part = nullptr;      // [ntiles][S][BN*PT]
  unsigned *tile_cnt = nullptr;  // [ntiles], zero on entry, left zero
  // epilogue inputs
  const double *Y = nullptr;  // rows y_j (n x p, pitch ldy)
  int ldy = 0;
  const double *U = nullptr;  // rows u_j (HVP)
  int ldu = 0;
  const double *G = nullptr;    // p x p Y^T Y
  const double *K = nullptr;    // p x p U^T Y + Y^T U (HVP)
  const double *rho = nullptr;  // n, rowdot(E, Y) at the same Y (HVP)
  // outputs
  double *out = nullptr;  // RAW: P; COSTGRAD: R; HVP: H
  int ldo = 0;
  double *egrad = nullptr;  // COSTGRAD, optional
  int lde = 0;
  double *rho_out = nullptr;  // COSTGRAD, optional
  double *zout = nullptr;     // ROWDOT
  double *out2 = nullptr;     // BOTH: H (pitch ldo2); scal_out2[0] = <U, H>
  int ldo2 = 0;
  double *scal_out2 = nullptr;
  // scalars
  double *tile_scal = nullptr;  // [ntiles][2]
  unsigned *glob_cnt = nullptr;
  double *scal_out = nullptr;  // [2]: COSTGRAD (s1, ||R||^2), HVP (<U,H>, 0), ROWDOT (sum z, 0)
  const double *gg = nullptr;          // ||G||_F^2 (COSTGRAD)
  const double *cost_extra = nullptr;  // [2] constant cost terms (COSTGRAD)
  double *cost_out = nullptr;
};

int symv_pt(int p);                // padded chunk width used by the kernels (8, 16, 32, 64)
int symv_bn(int pt, int mode2);     // output rows per CTA
int symv_chunks(int p, int epi);    // column chunks (grid z) of one launch: RAW splits p > 64
// EPI_RAW: any p (column chunks of 64 on grid z); fused epilogues: p <= 64.  The split-K
// workspace needs ceil(n/BN) * chunks * S * BN * PT doubles and as many zeroed tile counters.
cudaError_t symv_launch(const SymvArgs &a, int epi, int mode2, bool atr, int S, cudaStream_t st);

// TMA / mbarrier pipelined variant (symv_tma.cu) for the symmetric product M V (MODE2_NONE, no
// ATR, even lda, 16 B aligned M): CTA = 128 rows, split-K in multiples of 32 rows. Transposes V
// into Vt (ceil(p/PT)*PT... rows p, pitch ldvt = even >= n) first.
bool symv_tma_supported(const SymvArgs &a, int epi, int mode2, bool atr);
int symv_tma_rows();
int symv_tma_pt(int p, int epi);      // column chunk width of the TMA kernel (8 ... 64, 128 for raw p > 64)
int symv_tma_chunks(int p, int epi);
int symv_tma_ctas_per_sm(int pt, int epi);
bool symv_tma_both_duo();
int symv_tma_kstep();
cudaError_t symv_tma_launch(const SymvArgs &a, int epi, int S, double *Vt, int64_t ldvt, cudaStream_t st);
// Vt (p x ldvt) = V^T for a k x p row-major V (pitch ldv)
cudaError_t symv_transpose(int k, int p, const double *V, int ldv, double *Vt, int64_t ldvt, const int *skip,
                           cudaStream_t st);

// Matrix-light ALM gather-product (symv_gather.cu): out = M V + A*(w) X with A*(w) gathered
// from w through the TMA-loaded index-map panel inside the ring (never materialised); a.V = U, a.X = Y,
// a.amap / a.ldm / a.w as for MODE2_GATHER. EPI_HVP (p <= 64) or EPI_RAW (column chunks on grid z).
// Vt: 2 p ldvt doubles, ldvt = round_up(n, 2). Split-K in multiples of symv_gather_kstep() columns.
bool symv_gather_supported(const SymvArgs &a, int epi, bool atr);
int symv_gather_kstep();
cudaError_t symv_gather_launch(const SymvArgs &a, int epi, int S, double *Vt, int64_t ldvt, cudaStream_t st);

// Upper-triangle ("symmetric half") variant (symv_symm.cu) for p <= 16: a partial-product kernel
// over runs of 128 x 128 upper tiles and a reduce + row-epilogue kernel (one CTA per 128 rows).
// symm_units fills the unit table (int4 {I, Ja, Jb, 0} per unit) and the per-block-row start
// offsets (nb + 1), returning the unit count.
bool symm_supported(const SymvArgs &a, int epi, int mode2, bool atr);
int symm_units(int n, std::vector<int> &host_units, std::vector<int> &host_ustart);
size_t symm_tpart_elems(int n, int p);
size_t symm_fpart_elems(int n_units, int p);
cudaError_t symm_launch(const SymvArgs &a, int epi, double *Vt, int64_t ldvt, const int4 *units, int n_units,
                        const int *ustart, double *Fpart, double *Tpart, cudaStream_t st);

}  // namespace drsdp
