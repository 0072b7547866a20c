// Does cp.reduce.async.bulk.tensor add.f64 work on this GPU?  C (64 x 64 fp64) += S (32 x 16 box from smem).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(const __grid_constant__ CUtensorMap m) {
  __shared__ __align__(1024) double s[32 * 16];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s[i] = 0.5 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&m),
                 "r"(16), "r"(8), "r"(sa)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  double *d;
  cudaMalloc(&d, 64 * 64 * 8);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = 1.0;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  void *fnp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  CUtensorMap m;
  cuuint64_t dims[2] = {64, 64}, str[1] = {64 * 8};
  cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(m);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  // expect rows 8..39, cols 16..31 += 0.5 + (row-8)*16 + (col-16)
  int bad = 0;
  for (int r0 = 0; r0 < 64; ++r0)
    for (int c = 0; c < 64; ++c) {
      double want = 1.0;
      if (r0 >= 8 && r0 < 40 && c >= 16 && c < 32) want += 0.5 + (r0 - 8) * 16 + (c - 16);
      if (h[r0 * 64 + c] != want) ++bad;
    }
  printf("mismatches %d (C[8][16] = %g, want 1.5)\n", bad, h[8 * 64 + 16]);
  return 0;
}
