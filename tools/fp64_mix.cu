// Micro-benchmark: cost of DADDs issued by separate warps while other warps keep
// the FP64 pipe busy with DMMAs (the summing warpgroup of stc_fused.cu).
// 8 "MMA" warps (2 per SMSP) run m16n8k4 DMMAs on 16 register accumulators;
// 4 "adder" warps (1 per SMSP) loop { R independent DADDs; spin D cycles } until
// the MMA warps finish.  Prints the DMMA rate and the adders' DADD rate for a
// sweep of run lengths R and spacings D.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int R>
__global__ void __launch_bounds__(384, 1) mix(double *out, unsigned long long *dadds, int iters, int spin, int adders) {
  __shared__ volatile int stop;
  __shared__ int done;
  if (threadIdx.x == 0) { stop = 0; done = 0; }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp < 8) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
    double c[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0 && atomicAdd(&done, 1) == 7) stop = 1;
  } else if (warp - 8 < adders) {
    double acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = threadIdx.x + i;
    const double d = 1e-30;
    unsigned long long n = 0;
    while (!stop) {
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = __dadd_rn(acc[i], d);
      n += R;
      if (spin) {
        const long long t0 = clock64();
        while (clock64() - t0 < spin) {}
      }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) atomicAdd(dadds, n);
  }
}

template <int R>
int run(double *out, unsigned long long *dd, int iters, int spin, int adders, float base_ms) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  mix<R><<<148, 384>>>(out, dd, iters, spin, adders);
  CK(cudaMemset(dd, 0, 8));
  CK(cudaEventRecord(e0));
  mix<R><<<148, 384>>>(out, dd, iters, spin, adders);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  unsigned long long h;
  CK(cudaMemcpy(&h, dd, 8, cudaMemcpyDeviceToHost));
  const double flops = 148.0 * 256 * iters * 16 * 2 * 16 * 8 * 4 / 32;  // per-thread share of m16n8k4
  const double cyc = ms * 1e-3 * 1.965e9;
  const double dmma_per_smsp = 148.0 * 8 * iters * 16 * 2 / 148 / 4;  // DMMA.8x8x4 per SMSP
  const double dadd_per_smsp = (double)h / 148 / 4;                    // warp-DADDs per SMSP
  printf("R=%2d spin=%5d adders=%d  %8.3f ms  DMMA %6.2f TF/s  slowdown %5.1f%%  warp-DADD/SMSP %9.0f  per 2048 cyc %6.1f  cyc lost per DADD %6.2f\n",
         R, spin, adders, ms, flops / ms / 1e9, base_ms > 0 ? 100.0 * (ms / base_ms - 1) : 0.0, dadd_per_smsp,
         dadd_per_smsp / cyc * 2048, base_ms > 0 ? (ms - base_ms) * 1e-3 * 1.965e9 / dadd_per_smsp : 0.0);
  (void)dmma_per_smsp;
  return 0;
}

int main() {
  double *out;
  unsigned long long *dd;
  CK(cudaMalloc(&out, 148 * 384 * 8));
  CK(cudaMalloc(&dd, 8));
  const int iters = 4000;
  // baseline: MMA warps alone
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  mix<1><<<148, 384>>>(out, dd, iters, 0, 0);
  CK(cudaEventRecord(e0));
  mix<1><<<148, 384>>>(out, dd, iters, 0, 0);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float base;
  CK(cudaEventElapsedTime(&base, e0, e1));
  run<1>(out, dd, iters, 0, 0, base);
  const int spins[] = {200, 800, 3200};
  for (int sp : spins) {
    run<1>(out, dd, iters, sp / 8, 4, base);
    run<2>(out, dd, iters, sp / 4, 4, base);
    run<8>(out, dd, iters, sp, 4, base);
    run<16>(out, dd, iters, sp * 2, 4, base);
    run<32>(out, dd, iters, sp * 4, 4, base);
  }
  run<8>(out, dd, iters, 0, 4, base);
  run<32>(out, dd, iters, 0, 4, base);
  return 0;
}
