// common.cuh — shared device helpers for libdrsdp (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DRSDP_DEV __device__ __forceinline__

namespace drsdp {

constexpr int kWarp = 32;

DRSDP_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction of K values per thread; result valid in thread 0.
// scratch: at least K * (blockDim.x / 32) doubles of shared memory.
template <int K>
DRSDP_DEV void block_sum(double (&v)[K], double *scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[k * nw + warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += scratch[k * nw + w];
      v[k] = s;
    }
  }
  __syncthreads();
}

// Deterministic grid reduction: every block calls with its thread-local K values.
// Block partials go to partials[block*K + k]; the last block to arrive (atomic ticket)
// sums them in block order and writes out[k] (out may be nullptr) and returns true in
// all of its threads (so it may run a finalizer). The counter is reset for reuse.
// Returns false in non-last blocks.
template <int K>
DRSDP_DEV bool grid_sum(double (&v)[K], double *partials, unsigned *counter, double *out,
                        double *scratch) {
  block_sum<K>(v, scratch);
  const int nb = gridDim.x * gridDim.y * gridDim.z;
  const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  __shared__ unsigned s_ticket;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) partials[(size_t)bid * K + k] = v[k];
    __threadfence();
    s_ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  if (s_ticket != (unsigned)(nb - 1)) return false;
  __threadfence();
  // last block: thread t sums blocks t, t + nt, ... in order, then fixed-order block sum
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] += __ldcg(partials + (size_t)b * K + k);
  }
  block_sum<K>(acc, scratch);
  if (threadIdx.x == 0) {
    if (out) {
#pragma unroll
      for (int k = 0; k < K; ++k) out[k] = acc[k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = acc[k];
    *counter = 0u;
  }
  __syncthreads();
  return true;
}

// sum_{k < count} p[k * stride] in index order, with the loads issued 8 at a time (independent
// __ldcg loads in flight instead of one L2 round trip per term). Same order as a plain loop.
DRSDP_DEV double ordered_sum(const double *p, int count, size_t stride) {
  double s = 0.0;
  int k = 0;
  for (; k + 8 <= count; k += 8) {
    double t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = __ldcg(p + (size_t)(k + j) * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += t[j];
  }
  for (; k < count; ++k) s += __ldcg(p + (size_t)k * stride);
  return s;
}

DRSDP_DEV void dmma_884(double &c0, double &c1, double a, double b) {
  // D(8x8) += A(8x4, row) * B(4x8, col); fragments:
  //   a = A[lane>>2][lane&3], b = B[lane&3][lane>>2], {c0,c1} = C[lane>>2][2*(lane&3) + {0,1}]
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace drsdp
