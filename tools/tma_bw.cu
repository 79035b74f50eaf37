// Dev probe (not product): L2 -> SM TMA load throughput, whole GPU, data
// L2-resident. Modes: 0 = every CTA streams distinct boxes; 1 = the CTAs of a
// cluster stream the same boxes (unicast); 2 = the cluster's boxes are
// multicast (each CTA issues 1/CS of them to every CTA of the cluster).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_01635_b200/csrc \
//      -o build/tma_bw tools/tma_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace rtpb::ptx;

constexpr int BOX_BYTES = 64 * 2 * 128;  // 64 bf16 x 128 rows = 16 KB

__device__ __forceinline__ void tma_load_mc(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) tma_loop(const __grid_constant__ CUtensorMap map, int iters, int mode,
                                                  int nbx, int nby) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  uint32_t cs;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mode == 2 ? cs : 1);
    }
    fence_mbar_init();
  }
  cluster_sync();
  const int cid = blockIdx.x / cs;
  const int src = mode == 0 ? int(blockIdx.x) : cid;
  const int nb = nbx * nby;
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], BOX_BYTES);
      const int b = (src * 7919 + i) % nb;
      const int bx = b % nbx, by = b / nbx;
      if (mode == 2) {
        if (int(i % cs) == int(rank)) tma_load_mc(smem + s * BOX_BYTES, &map, &full[s], bx * 64, by * 128, uint16_t((1u << cs) - 1));
      } else {
        tma_load_2d(smem + s * BOX_BYTES, &map, &full[s], bx * 64, by * 128);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&full[s], ph);
      if (mode == 2) {
        for (uint32_t c = 0; c < cs; ++c) mbar_arrive_cluster(&empty[s], c);
      } else {
        mbar_arrive(&empty[s]);
      }
    }
  }
  cluster_sync();
}

template <int STAGES>
int run(const CUtensorMap& m, int rows, int cols, int all);

int main() {
  const int rows = 8192, cols = 4096;  // 64 MB bf16, L2-resident
  void* g;
  cudaMalloc(&g, size_t(rows) * cols * 2);
  cudaMemset(g, 0, size_t(rows) * cols * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<4>(m, rows, cols, 0);
  run<8>(m, rows, cols, 0);
  run<12>(m, rows, cols, 0);
  run<8>(m, rows, cols, 1);
  return 0;
}

template <int STAGES>
int run(const CUtensorMap& m, int rows, int cols, int all) {
  auto k = tma_loop<STAGES>;
  const int smem = STAGES * BOX_BYTES + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int iters = 4000;
  const char* names[] = {"distinct", "same-unicast", "multicast"};
  for (int mode = 0; mode < 3; ++mode)
    for (int cs : {0, 1, 2}) {
      const bool half = cs == 0;
      if (half) cs = 1;
      if (mode > 0 && cs == 1) continue;
      if (!all && mode > 0) continue;
      const int grid = half ? 74 : (148 / cs) * cs;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(64);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchKernelEx(&cfg, k, m, 200, mode, cols / 64, rows / 128);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k, m, iters, mode, cols / 64, rows / 128);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double delivered = double(grid) * iters * BOX_BYTES;
      const double l2 = mode == 0 ? delivered : delivered / cs;
      printf("stages=%2d %-13s cs=%d grid=%3d %s %.3f ms  SM-delivered %6.2f TB/s  unique-from-L2 %6.2f TB/s\n", STAGES, names[mode], cs,
             grid, cudaGetErrorString(e), ms, delivered / (ms * 1e-3) / 1e12, l2 / (ms * 1e-3) / 1e12);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
