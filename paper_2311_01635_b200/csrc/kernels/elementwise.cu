// HBM-bound helper kernels of the RTP path: Flyweight shard init, bias-grad
// column sums, 3xTF32 operand split, standalone GELU. Grid-stride loops with
// grids sized in multiples of the SM count.
#include <cuda_bf16.h>

#include "launch.hpp"

namespace rtpb {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
  // rng.hpp:16-22 in counter form: the k-th next_u64() of SplitMix64(seed).
  uint64_t z = seed + (k + 1) * kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int grid_for(size_t work, int threads, int max_waves = 8) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  size_t blocks = (work + threads - 1) / threads;
  const size_t cap = size_t(sms) * max_waves;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  return int(blocks);
}

template <typename T>
__global__ void flyweight_kernel(T* __restrict__ dst, uint64_t seed, uint64_t base, uint64_t I, uint64_t O,
                                 uint64_t per, uint64_t j, double lo, double hi) {
  const uint64_t wn = I * per, total = wn + per;
  const double span = __dsub_rn(hi, lo);
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t k;
    if (e < wn) {
      const uint64_t i = e / per, c = e - i * per;
      k = base + i * O + j * per + c;  // W[i, j*per + c], row-major draw order
    } else {
      k = base + I * O + j * per + (e - wn);  // bias follows the weight
    }
    // tensor.cpp:99-103 / rng.hpp:25-27 without FMA contraction.
    const double unit = __dmul_rn(__ull2double_rn(splitmix_at(seed, k) >> 11), 0x1.0p-53);
    const double v = __dadd_rn(lo, __dmul_rn(span, unit));
    if constexpr (sizeof(T) == 4)
      dst[e] = __double2float_rn(v);
    else
      dst[e] = __double2bfloat16(v);
  }
}

// Bias gradient db_j += colsum(dY[:, blk_j]) (layers_linear.cpp:63) in one
// launch. grid = (column groups of 64) x (row splits); block = 32 row lanes x
// 8 column groups of 8 (16-byte loads, 4 rows in flight per thread). Each
// block writes its partial sums; the last block to finish a column group
// (ticket) adds the splits in split order, so the result is deterministic.
// The tickets live in the caller's workspace and are left at zero.
template <bool F32>
__global__ void colsum_kernel(const void* __restrict__ dy, size_t ldy, int M, int per, int rows_per_split,
                              float* __restrict__ partial, unsigned* __restrict__ tickets,
                              const float* __restrict__ g_in, float* __restrict__ g_out) {
  __shared__ float red[32][65];
  __shared__ bool is_last;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: predecessor's dY complete
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;
  const int c0 = blockIdx.x * 64 + cg * 8;
  const int r_begin = blockIdx.y * rows_per_split;
  const int r_end = min(M, r_begin + rows_per_split);
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto add_row = [&](int r) {
    if constexpr (F32) {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(dy) + size_t(r) * ldy + c0);
      const float4 a = __ldg(p), b = __ldg(p + 1);
      s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w; s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
    } else {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(dy) + size_t(r) * ldy + c0));
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s[2 * q] += __uint_as_float(w[q] << 16);
        s[2 * q + 1] += __uint_as_float(w[q] & 0xFFFF0000u);
      }
    }
  };
  if (c0 < per) {
    int r = r_begin + rl;
#pragma unroll 4
    for (; r < r_end; r += 32) add_row(r);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) red[rl][cg * 8 + q] = s[q];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = blockIdx.x * 64 + threadIdx.x;
    float acc = 0.f;
    for (int l = 0; l < 32; ++l) acc += red[l][threadIdx.x];  // fixed order
    if (c < per) partial[size_t(blockIdx.y) * per + c] = acc;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(&tickets[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (is_last && threadIdx.x < 64) {
    __threadfence();
    const int c = blockIdx.x * 64 + threadIdx.x;
    if (c < per) {
      float acc = 0.f;
      for (int sp = 0; sp < int(gridDim.y); ++sp) acc += __ldcg(&partial[size_t(sp) * per + c]);
      g_out[c] = (g_in ? g_in[c] : 0.f) + acc;  // g_in == nullptr: gradient known zero
    }
    if (threadIdx.x == 0) tickets[blockIdx.x] = 0u;  // leave the workspace reusable
  }
}

int colsum_splits(size_t M, size_t per) {
  const int col_blocks = int((per + 63) / 64);
  int splits = (4 * 148 + col_blocks - 1) / col_blocks;  // ~4 CTAs per SM
  const int max_splits = int((M + 127) / 128);          // >= 128 rows per split
  if (splits > max_splits) splits = max_splits;
  return splits < 1 ? 1 : splits;
}

__global__ void tf32_split_kernel(const float* __restrict__ src, size_t rows, size_t cols, size_t ld,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const size_t total = rows * cols;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t r = e / cols, c = e - r * cols;
    const float x = src[r * ld + c];
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);  // exactly representable in tf32
    hi[e] = h;
    lo[e] = x - h;  // exact in fp32
  }
}

// Split + transpose through a 32x32 smem tile: out[c][r] (ld_out = rows).
__global__ void tf32_split_t_kernel(const float* __restrict__ src, size_t rows, size_t cols, size_t ld,
                                    float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ float tile[32][33];
  const size_t r0 = size_t(blockIdx.y) * 32, c0 = size_t(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? src[r * ld + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      const float x = tile[threadIdx.x][i];
      const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
      const size_t ld_out = (rows + 7) & ~size_t(7);  // 16-byte TMA rows
      hi[c * ld_out + r] = h;
      lo[c * ld_out + r] = x - h;
    }
  }
}

template <typename T>
__device__ __forceinline__ float ld_f(const T* p, size_t i) {
  if constexpr (sizeof(T) == 4) return p[i];
  else return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, size_t i, float v) {
  if constexpr (sizeof(T) == 4) p[i] = v;
  else p[i] = __float2bfloat16_rn(v);
}

template <typename T>
__global__ void gelu_kernel(const T* __restrict__ x, T* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float v = ld_f(x, i);
    st_f(y, i, v * 0.5f * (1.0f + erff(v * 0.70710678118654752f)));
  }
}

template <typename T>
__global__ void gelu_bwd_kernel(const T* __restrict__ x, const T* __restrict__ up, T* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float v = ld_f(x, i);
    const float phi = 0.5f * (1.0f + erff(v * 0.70710678118654752f));
    const float pdf = 0.39894228040143267794f * __expf(-0.5f * v * v);
    st_f(out, i, ld_f(up, i) * (phi + v * pdf));
  }
}

__global__ void cast_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// Any-to-any dtype conversion (device Tensor casts): each element read as
// fp64 then rounded once to the destination (RN; bf16 from fp64 directly, no
// double rounding through fp32). code = src_dtype * 3 + dst_dtype.
__device__ __forceinline__ double ld_any(const void* p, int dt, size_t i) {
  if (dt == RTPB_F64) return static_cast<const double*>(p)[i];
  if (dt == RTPB_F32) return double(static_cast<const float*>(p)[i]);
  return double(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
}
__device__ __forceinline__ void st_any(void* p, int dt, size_t i, double v) {
  if (dt == RTPB_F64)
    static_cast<double*>(p)[i] = v;
  else if (dt == RTPB_F32)
    static_cast<float*>(p)[i] = __double2float_rn(v);
  else
    static_cast<__nv_bfloat16*>(p)[i] = __double2bfloat16(v);
}
__global__ void convert_kernel(const void* __restrict__ src, int sdt, void* __restrict__ dst, int ddt, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    st_any(dst, ddt, i, ld_any(src, sdt, i));
}
__global__ void add_kernel(const void* __restrict__ a, const void* __restrict__ b, void* __restrict__ out, int dt,
                           size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    st_any(out, dt, i, ld_any(a, dt, i) + ld_any(b, dt, i));
}
__global__ void fill_kernel(void* __restrict__ dst, int dt, size_t n, double v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    st_any(dst, dt, i, v);
}

int post_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  count_launch();
  return RTPB_OK;
}

}  // namespace

int flyweight_init(void* dst, bool f32, uint64_t seed, uint64_t base, size_t I, size_t O, size_t n, size_t j,
                   double lo, double hi, cudaStream_t s) {
  if (n == 0 || O % n) return set_error(RTPB_ERR_CONFIG, "flyweight_init: out_dim not divisible by n");
  if (j >= n) return set_error(RTPB_ERR_CONFIG, "flyweight_init: shard index out of range");
  const size_t per = O / n, total = I * per + per;
  const int grid = grid_for(total, 256);
  if (f32)
    flyweight_kernel<float><<<grid, 256, 0, s>>>(static_cast<float*>(dst), seed, base, I, O, per, j, lo, hi);
  else
    flyweight_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), seed, base, I, O, per,
                                                         j, lo, hi);
  return post_launch("flyweight_kernel");
}

// Workspace: [tickets: one per column group, 256 B aligned][partials].
size_t colsum_workspace_bytes(size_t M, size_t per) {
  const size_t tick = ((per + 63) / 64 * sizeof(unsigned) + 255) & ~size_t(255);
  return tick + size_t(colsum_splits(M, per)) * per * sizeof(float);
}

int colsum_bias_grad(bool f32, const void* dy, size_t ldy, size_t M, size_t per, const float* g_in, float* g_out,
                     void* ws, cudaStream_t s) {
  if (per % 8) return set_error(RTPB_ERR_CONFIG, "bias grad: per must be a multiple of 8");
  const int splits = colsum_splits(M, per);
  const int rows_per_split = int((M + splits - 1) / splits);
  const unsigned col_blocks = unsigned((per + 63) / 64);
  dim3 grid(col_blocks, unsigned(splits));
  unsigned* tickets = static_cast<unsigned*>(ws);
  float* partial = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                            ((col_blocks * sizeof(unsigned) + 255) & ~size_t(255)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int Mi = int(M), peri = int(per);
  cudaError_t e = f32 ? cudaLaunchKernelEx(&cfg, colsum_kernel<true>, dy, ldy, Mi, peri, rows_per_split, partial,
                                           tickets, g_in, g_out)
                      : cudaLaunchKernelEx(&cfg, colsum_kernel<false>, dy, ldy, Mi, peri, rows_per_split, partial,
                                           tickets, g_in, g_out);
  if (e != cudaSuccess) return set_cuda_error(e, "colsum_kernel launch");
  return post_launch("colsum_kernel");
}

int tf32_split(const float* src, size_t rows, size_t cols, size_t ld, float* hi, float* lo, cudaStream_t s) {
  tf32_split_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(src, rows, cols, ld, hi, lo);
  return post_launch("tf32_split_kernel");
}

int tf32_split_t(const float* src, size_t rows, size_t cols, size_t ld, float* hi, float* lo, cudaStream_t s) {
  dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32));
  tf32_split_t_kernel<<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, ld, hi, lo);
  return post_launch("tf32_split_t_kernel");
}

int gelu_fwd(bool f32, const void* x, void* y, size_t n, cudaStream_t s) {
  const int g = grid_for(n, 256);
  if (f32)
    gelu_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(y), n);
  else
    gelu_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                  static_cast<__nv_bfloat16*>(y), n);
  return post_launch("gelu_kernel");
}

int gelu_bwd(bool f32, const void* x, const void* up, void* out, size_t n, cudaStream_t s) {
  const int g = grid_for(n, 256);
  if (f32)
    gelu_bwd_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x), static_cast<const float*>(up),
                                              static_cast<float*>(out), n);
  else
    gelu_bwd_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                      static_cast<const __nv_bfloat16*>(up),
                                                      static_cast<__nv_bfloat16*>(out), n);
  return post_launch("gelu_bwd_kernel");
}

int convert(const void* src, int src_dtype, void* dst, int dst_dtype, size_t n, cudaStream_t s) {
  if (n == 0) return RTPB_OK;
  convert_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, src_dtype, dst, dst_dtype, n);
  return post_launch("convert_kernel");
}

int add(const void* a, const void* b, void* out, int dtype, size_t n, cudaStream_t s) {
  if (n == 0) return RTPB_OK;
  add_kernel<<<grid_for(n, 256), 256, 0, s>>>(a, b, out, dtype, n);
  return post_launch("add_kernel");
}

int fill(void* dst, int dtype, size_t n, double v, cudaStream_t s) {
  if (n == 0) return RTPB_OK;
  fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(dst, dtype, n, v);
  return post_launch("fill_kernel");
}

int cast_f32_to_bf16(const float* src, void* dst, size_t n, cudaStream_t s) {
  cast_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, static_cast<__nv_bfloat16*>(dst), n);
  return post_launch("cast_kernel");
}

// Module anchor for preload_device_kernels (launch.hpp): any kernel of this
// translation unit's module.
const void* kernel_anchor_elementwise() { return reinterpret_cast<const void*>(&tf32_split_kernel); }

}  // namespace rtpb
