// Dev probe (not product): L2 -> SM TMA delivery per stage of 16 KB, whole GPU, data L2-resident,
// for the box shapes the step GEMM uses: kind 0 = one K-major box {64, 128 rows}; kind 1 = two
// MN-major boxes {64, 64 rows} (the dW operands today); kind 2 = the same 16 KB as one 3-D box
// {64, 64 rows, 2 atoms} (both MN atoms in one instruction, identical shared-memory layout).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_01635_b200/csrc \
//      -o build/tma_box tools/probes/tma_box.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace rtpb::ptx;

constexpr int STAGE = 16384;

__device__ __forceinline__ void tma3(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) box_loop(const __grid_constant__ CUtensorMap m2a, const __grid_constant__ CUtensorMap m2b,
                                                  const __grid_constant__ CUtensorMap m3, int iters, int kind, int rows,
                                                  int cols) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nbx = cols / 128, nby = rows / 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], STAGE);
      const int b = (int(blockIdx.x) * 7919 + i) % (nbx * nby);
      const int bx = b % nbx, by = b / nbx;
      uint8_t* d = smem + s * STAGE;
      if (kind == 0) {
        tma_load_2d(d, &m2a, &full[s], (bx % (cols / 64)) * 64, (by / 2) * 128);
      } else if (kind == 1) {
        tma_load_2d(d, &m2b, &full[s], bx * 128, by * 64);
        tma_load_2d(d + 8192, &m2b, &full[s], bx * 128 + 64, by * 64);
      } else {
        tma3(d, &m3, &full[s], 0, by * 64, bx * 2);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main() {
  const int rows = 8192, cols = 4096;  // 64 MB bf16, L2-resident
  void* g;
  cudaMalloc(&g, size_t(rows) * cols * 2);
  cudaMemset(g, 0, size_t(rows) * cols * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m2a, m2b, m3;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t es[3] = {1, 1, 1};
  cuuint32_t boxa[2] = {64, 128}, boxb[2] = {64, 64};
  CUresult r1 = enc(&m2a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&m2b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d3[3] = {64, cuuint64_t(rows), cuuint64_t(cols / 64)};
  cuuint64_t s3[2] = {cuuint64_t(cols) * 2, 128};
  cuuint32_t box3[3] = {64, 64, 2};
  CUresult r3 = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, d3, s3, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d %d %d\n", int(r1), int(r2), int(r3));
  constexpr int STAGES = 6;
  auto k = box_loop<STAGES>;
  const int smem = STAGES * STAGE + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"K-major 1 box {64,128}", "MN-major 2 boxes {64,64}", "MN-major 1 box {64,64,2}"};
  for (int rep = 0; rep < 2; ++rep)
    for (int kind = 0; kind < 3; ++kind) {
      if (kind == 2 && r3 != CUDA_SUCCESS) continue;
      const int iters = 4000;
      k<<<148, 64, smem>>>(m2a, m2b, m3, 200, kind, rows, cols);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, 64, smem>>>(m2a, m2b, m3, iters, kind, rows, cols);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-28s %s %.3f ms  SM-delivered %6.2f TB/s\n", names[kind], cudaGetErrorString(e), ms,
             148.0 * iters * STAGE / (ms * 1e-3) / 1e12);
    }
  return 0;
}
