// Dev probe (not product): raw tcgen05.mma issue rate with operands resident
// in shared memory (no TMA), per shape / major-ness / cta_group, whole GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_01635_b200/csrc \
//      -o build/mma_rate tools/mma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels/ptx.cuh"

using namespace rtpb::ptx;

template <int N, bool PAIR, bool AMN, bool BMN>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr int M = PAIR ? 256 : 128;
  constexpr uint32_t IDESC = idesc_make(M, N, 1, AMN, BMN);
  constexpr int A_BYTES = 128 * 128, B_BYTES = (PAIR ? N / 2 : N) * 128;
  unsigned long long t0 = clock64();
  if (warp == 0 && threadIdx.x == 0 && rank == 0) {
    const uint32_t a_base = smem_u32(smem), b_base = a_base + A_BYTES;
    for (int it = 0; it < iters; ++it) {
      const int st = it & 1;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t a_off = AMN ? kk * 16 * 128 : kk * 32, b_off = BMN ? kk * 16 * 128 : kk * 32;
        const uint64_t ad = sdesc_sw128(a_base + a_off, AMN ? 64 * 128 : 16, 1024);
        const uint64_t bd = sdesc_sw128(b_base + b_off, BMN ? 64 * 128 : 16, 1024);
        if constexpr (PAIR)
          umma_f16_pair(tmem + st * N, ad, bd, IDESC, 1);
        else
          umma_f16(tmem + st * N, ad, bd, IDESC, 1);
      }
    }
    if constexpr (PAIR) umma_commit_pair(&bar); else umma_commit(&bar);
  }
  (void)B_BYTES;
  if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    if (blockIdx.x == 0) *cyc = clock64() - t0;
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

template <int N, bool PAIR, bool AMN, bool BMN>
void run(const char* name, unsigned long long* cyc) {
  auto k = mma_loop<N, PAIR, AMN, BMN>;
  const int smem = 128 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k, 100, cyc);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double M = PAIR ? 256 : 128;
  const double ctas = PAIR ? 74 : 148;
  const double flop = 2.0 * M * N * 16 * 4 * double(iters) * ctas;
  printf("%-28s %s  %.3f ms  %7.1f TFLOP/s  %6.1f clk/MMA (block 0)  flop/clk/SM %.0f\n", name,
         cudaGetErrorString(e), ms, flop / (ms * 1e-3) / 1e12, double(c) / (4.0 * iters),
         (2.0 * M * N * 16 / (PAIR ? 2 : 1)) / (double(c) / (4.0 * iters)));
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  run<256, false, false, false>("single 128x256 K,K", cyc);
  run<128, false, false, false>("single 128x128 K,K", cyc);
  run<256, false, true, true>("single 128x256 MN,MN", cyc);
  run<256, false, false, true>("single 128x256 K,MN", cyc);
  run<256, true, false, false>("pair 256x256 K,K", cyc);
  run<256, true, true, true>("pair 256x256 MN,MN", cyc);
  run<256, true, false, true>("pair 256x256 K,MN", cyc);
  run<128, true, false, false>("pair 256x128 K,K", cyc);
  return 0;
}
