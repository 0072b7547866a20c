// TMA box-load throughput micro-benchmark: one CTA per SM, one elected thread
// streams 16 KB boxes (2048 doubles) of a row-major [R][C] fp64 matrix into a
// ring of NSLOT smem slots (mbarrier per slot, 8 consumer warps release), for
// box shapes of 16, 32, 64, 128 and 256 doubles per row.  Prints GB/s per
// shape; the question is whether short rows limit a single SM's TMA unit.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NSLOT, int RANK>
__global__ void __launch_bounds__(288, 1) tma_stream(const __grid_constant__ CUtensorMap map, int box_cols, int box_rows,
                                                     int n_rows_total, int iters, double *sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double *slots = (double *)sm;
  uint64_t *full = (uint64_t *)(sm + NSLOT * 16384);
  uint64_t *empty = full + NSLOT;
  const int t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sa(empty + i)));
    }
  }
  __syncthreads();
  const int warp = t >> 5;
  const int nbox_rows = n_rows_total / box_rows;
  if (warp == 8) {
    if (t == 256) {
      for (int j = 0; j < iters; ++j) {
        const int s = j % NSLOT;
        const uint32_t ph = ((j / NSLOT) & 1) ^ 1;
        asm volatile("{ .reg .pred P; W1: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W1; }" ::"r"(
                         sa(empty + s)),
                     "r"(ph));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384));
        const int br = (blockIdx.x * 131 + j * 7) % nbox_rows;
        if (RANK == 2) {
          const int x = 0, y = br * box_rows;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  sa(slots + s * 2048)),
              "l"((uint64_t)&map), "r"(x), "r"(y), "r"(sa(full + s))
              : "memory");
        } else {
          // 3D: (16 contiguous, 8 rows of stride 4096, 16 planes of stride 262144); br picks (row block, plane block)
          const uint32_t h = (uint32_t)(blockIdx.x * 2654435761u + j * 40503u);
          const int y = (int)(h % 8) * 8, z = (int)((h >> 3) % (n_rows_total / 16)) * 16, x = (int)((h >> 11) % 256) * 16;
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  sa(slots + s * 2048)),
              "l"((uint64_t)&map), "r"(x), "r"(y), "r"(z), "r"(sa(full + s))
              : "memory");
        }
      }
    }
  } else {
    double acc = 0;
    for (int j = 0; j < iters; ++j) {
      const int s = j % NSLOT;
      const uint32_t ph = (j / NSLOT) & 1;
      asm volatile("{ .reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W2; }" ::"r"(
                       sa(full + s)),
                   "r"(ph));
      acc += slots[s * 2048 + t * 8];
      __syncwarp();
      if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)));
    }
    if (acc == 12345.0) sink[0] = acc;
  }
}

// 3D boxes (16 contiguous, 8 rows of stride 4096, 16 planes of stride 262144) at random
// positions in a tensor of `planes` 2 MB planes (256: 512 MB, DRAM; 16: 32 MB, L2-resident).
template <int NS>
void run3d(PFN_cuTensorMapEncodeTiled_v12000 enc, double *d, int sms, double *sink, int planes) {
  CUtensorMap m;
  cuuint64_t dims[3] = {4096, 64, (cuuint64_t)planes};
  cuuint64_t str[2] = {4096 * 8, 262144 * 8};
  cuuint32_t box[3] = {16, 8, 16};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode 3d failed\n");
  const size_t smem = NS * 16384 + 2 * NS * 8;
  CK(cudaFuncSetAttribute(tma_stream<NS, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int grid : {1, sms}) {
    const int iters = 2000;
    tma_stream<NS, 3><<<grid, 288, smem>>>(m, 16, 128, planes, 50, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    tma_stream<NS, 3><<<grid, 288, smem>>>(m, 16, 128, planes, iters, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)grid * iters * 16384;
    const double bpc = bytes / grid / (ms * 1e-3 * 1.9e9);
    printf("3D box planes %3d  slots %d  grid %3d: %8.1f GB/s total, %6.2f B/clk/SM, latency ~%6.0f clk\n", planes, NS, grid,
           bytes / ms / 1e6, bpc, NS * 16384.0 / bpc);
  }
}

int main() {
  const long R = 1 << 16, C = 1024;  // 512 MB
  double *d;
  CK(cudaMalloc(&d, R * C * 8));
  CK(cudaMemset(d, 0x3f, R * C * 8));  // non-zero data
  double *sink;
  CK(cudaMalloc(&sink, 8));
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  constexpr int NSLOT = 8;
  const size_t smem = NSLOT * 16384 + 2 * NSLOT * 8;
  CK(cudaFuncSetAttribute(tma_stream<NSLOT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(tma_stream<NSLOT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int cols : {16, 32, 64, 128, 256}) {
    for (long row_stride : {C, 4096L}) {
      const long rows_total = R * C / row_stride;
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows_total};
      cuuint64_t str[1] = {(cuuint64_t)row_stride * 8};
      cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)(2048 / cols)};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed cols=%d\n", cols);
        continue;
      }
      const int iters = 2000;
      for (int grid : {1, sms}) {
        tma_stream<NSLOT, 2><<<grid, 288, smem>>>(m, cols, 2048 / cols, (int)rows_total, 50, sink);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        tma_stream<NSLOT, 2><<<grid, 288, smem>>>(m, cols, 2048 / cols, (int)rows_total, iters, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)grid * iters * 16384;
        printf("row %4d B  stride %5ld  grid %3d: %8.1f GB/s total, %6.2f B/clk/SM (at 1.9 GHz)\n", cols * 8, row_stride,
               grid, bytes / ms / 1e6, bytes / grid / (ms * 1e-3 * 1.9e9));
      }
    }
  }
  run3d<1>(enc, d, sms, sink, 256);
  run3d<2>(enc, d, sms, sink, 256);
  run3d<4>(enc, d, sms, sink, 256);
  run3d<8>(enc, d, sms, sink, 256);
  run3d<1>(enc, d, sms, sink, 16);
  run3d<2>(enc, d, sms, sink, 16);
  run3d<4>(enc, d, sms, sink, 16);
  run3d<8>(enc, d, sms, sink, 16);
  return 0;
}
