// Micro-benchmark: cost of DADD runs interleaved in the DMMA warps' own
// instruction streams (8 warps, 2 per SMSP): loop { 16 m16n8k4 DMMAs; R
// independent DADDs }.  Prints the extra cycles per warp-DADD per SMSP as a
// function of the run length R (and of how many warps carry DADDs).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int R>
__global__ void __launch_bounds__(256, 1) inl(double *out, int iters, int every, int dwarps) {
  const int warp = threadIdx.x >> 5;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double acc[R > 0 ? R : 1];
#pragma unroll
  for (int i = 0; i < (R > 0 ? R : 1); ++i) acc[i] = threadIdx.x + i;
  const double d = 1e-30;
  const bool dw = warp < dwarps;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    if (dw && (it % every) == 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(acc[i]) : "d"(d));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
#pragma unroll
  for (int i = 0; i < (R > 0 ? R : 1); ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R>
float run(double *out, int iters, int every, int dwarps, float base) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  inl<R><<<148, 256>>>(out, iters, every, dwarps);
  cudaEventRecord(e0);
  inl<R><<<148, 256>>>(out, iters, every, dwarps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dadds_per_smsp = (double)R * (iters / every) * dwarps / 4.0;  // warp-DADDs per SMSP
  const double lost = (ms - base) * 1e-3 * 1.965e9;
  printf("R=%2d every=%2d dwarps=%d  %8.3f ms  slowdown %6.2f%%  warp-DADD per SMSP per 32 DMMA %6.2f  cycles per warp-DADD %6.2f\n",
         R, every, dwarps, ms, base > 0 ? 100.0 * (ms / base - 1) : 0.0,
         (double)R * dwarps / 4.0 / every / 2.0, base > 0 ? lost / dadds_per_smsp : 0.0);
  return ms;
}

int main() {
  double *out;
  CK(cudaMalloc(&out, 148 * 256 * 8));
  const int iters = 4096;
  float base = run<0>(out, iters, 1, 8, 0);
  run<1>(out, iters, 1, 8, base);
  run<2>(out, iters, 1, 8, base);
  run<4>(out, iters, 1, 8, base);
  run<8>(out, iters, 1, 8, base);
  run<8>(out, iters, 2, 8, base);
  run<16>(out, iters, 2, 8, base);
  run<16>(out, iters, 4, 8, base);
  run<32>(out, iters, 4, 8, base);
  run<32>(out, iters, 8, 8, base);
  run<64>(out, iters, 8, 8, base);
  run<64>(out, iters, 16, 8, base);
  run<8>(out, iters, 1, 4, base);
  run<32>(out, iters, 4, 4, base);
  return 0;
}
