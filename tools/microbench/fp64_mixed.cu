// Does DFMA co-issue with DMMA on B200? Times DMMA-only, DFMA-only and an interleaved kernel
// (same per-thread DMMA and DFMA counts) and prints the achieved fp64 TFLOP/s of each.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <bool DO_MMA, bool DO_FMA>
__global__ void mixed(double *out, int iters, double a, double b) {
  double x = threadIdx.x * 1e-3, y = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  double f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (DO_MMA)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(x), "d"(y));
      if (DO_FMA) {
        // 8 DFMA per thread per DMMA slot = 256 FMA per warp = one m8n8k4's FMA count
#pragma unroll
        for (int k = 0; k < 8; ++k) f[(i * 8 + k) & 15] = fma(f[(i * 8 + k) & 15], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

template <bool M, bool F>
int run(const char *name, double *out, int sms) {
  const int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  mixed<M, F><<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    mixed<M, F><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  const double warps = (double)blocks * threads / 32;
  const double fl = warps * iters * 8 * 512.0 * ((M ? 1 : 0) + (F ? 1 : 0));  // 256 FMA = 512 flop per slot
  printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f}\n", name, best, fl / best / 1e9);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *out; CK(cudaMalloc(&out, 64));
  run<true, false>("dmma_only", out, sms);
  run<false, true>("dfma_only", out, sms);
  run<true, true>("dmma+dfma interleaved", out, sms);
  return 0;
}
