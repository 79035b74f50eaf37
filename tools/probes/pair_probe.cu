// Dev probe (not product): shared-address encoding inside a 2-CTA cluster and
// which mbarrier a cta_group::2 TMA completion lands on.
// nvcc -gencode arch=compute_100a,code=sm_100a -o build/pair_probe tools/pair_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>

__global__ void __cluster_dims__(2, 1, 1) probe(const __grid_constant__ CUtensorMap map, int variant) {
  __shared__ __align__(1024) unsigned char buf[8192];
  __shared__ __align__(8) unsigned long long bar;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const unsigned a = unsigned(__cvta_generic_to_shared(&bar));
  unsigned m0, m1;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(m0) : "r"(a));
  asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(m1) : "r"(a));
  if (threadIdx.x == 0) {
    printf("rank %u: local 0x%x mapa0 0x%x mapa1 0x%x buf 0x%x\n", rank, a, m0, m1,
           unsigned(__cvta_generic_to_shared(buf)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (threadIdx.x == 0) {
    // leader expects both CTAs' bytes; each CTA loads 4 KB
    if (rank == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(8192));
    unsigned target = variant == 0 ? (a & 0xFEFFFFFFu) : (variant == 1 ? m0 : a);
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            unsigned(__cvta_generic_to_shared(buf + rank * 4096))),
        "l"(&map), "r"(target), "r"(0), "r"(int(rank) * 32)
        : "memory");
    if (rank == 0) {
      unsigned ok = 0;
      for (long i = 0; i < (1l << 24) && !ok; ++i)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(ok)
                     : "r"(a));
      printf("variant %d: leader barrier %s\n", variant, ok ? "COMPLETED" : "timed out");
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
}

int main() {
  void* g;
  cudaMalloc(&g, 64 * 64 * 2);
  cudaMemset(g, 0, 64 * 64 * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {64, 64};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 32};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int v = 0; v < 3; ++v) {
    probe<<<2, 32>>>(m, v);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d -> %s\n", v, cudaGetErrorString(e));
    if (e != cudaSuccess) break;
  }
  return 0;
}
