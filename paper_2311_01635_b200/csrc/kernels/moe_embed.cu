// Routing and gather / scatter kernels of RtpMoe (layers_moe.cpp:18-198) and
// RtpEmbedding (layers_linear.cpp:74-136). The expert MLPs themselves run on
// the step GEMMs; these kernels are HBM / latency-bound glue: grid-stride
// loops, one warp per token row, grids capped at a multiple of the SM count.
//
// Gate arithmetic is fp64 in the reference's order (kern::matmul: c = 0,
// c += a[i,t] * b[t,j] for t ascending, no FMA; softmax_rows max-subtracted),
// so the top-1 routing matches the reference whenever the activations do.
#include <cuda_bf16.h>

#include "launch.hpp"

namespace rtpb {

namespace {

constexpr int kWarps = 8;

template <typename T>
__device__ __forceinline__ float ldf(const T* p, size_t i) {
  if constexpr (sizeof(T) == 4)
    return p[i];
  else
    return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void stf(T* p, size_t i, float v) {
  if constexpr (sizeof(T) == 4)
    p[i] = v;
  else
    p[i] = __float2bfloat16_rn(v);
}

unsigned grid_warps(size_t items) {
  size_t blocks = (items + kWarps - 1) / kWarps;
  if (blocks > 148 * 32) blocks = 148 * 32;
  return unsigned(blocks ? blocks : 1);
}

#define WARP_LOOP(count)                                                                   \
  const int lane = threadIdx.x & 31;                                                       \
  for (size_t w = blockIdx.x * size_t(kWarps) + threadIdx.x / 32; w < (count);             \
       w += size_t(gridDim.x) * kWarps)

// logits = x . gate (fp64, reference order), probs = softmax_rows, sel = argmax
// (ties to the lower index). Lane e < n owns expert e.
template <typename T>
__global__ void moe_gate_kernel(const T* __restrict__ x, size_t rows, int H, const double* __restrict__ gate, int n,
                                double* __restrict__ probs, int* __restrict__ sel) {
  WARP_LOOP(rows) {
    double l = 0.0;
    if (lane < n)
      for (int t = 0; t < H; ++t)
        l = __dadd_rn(l, __dmul_rn(double(ldf(x, w * H + t)), gate[size_t(t) * n + lane]));
    double m = lane < n ? l : -INFINITY;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    const double e = lane < n ? exp(__dsub_rn(l, m)) : 0.0;
    // sum in index order (softmax_rows sums j ascending)
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = __dadd_rn(s, __shfl_sync(0xffffffffu, e, j));
    const double p = __ddiv_rn(e, s);
    if (lane < n) probs[w * n + lane] = p;
    // argmax_row: first maximum
    double best = __shfl_sync(0xffffffffu, p, 0);
    int bi = 0;
    for (int j = 1; j < n; ++j) {
      const double pj = __shfl_sync(0xffffffffu, p, j);
      if (pj > best) {
        best = pj;
        bi = j;
      }
    }
    if (lane == 0) sel[w] = bi;
  }
}

// dst[i, :] = src[idx[i], :]   (gather_rows, layers_moe.cpp:8-14)
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ src, size_t lds, const int* __restrict__ idx, size_t cnt,
                                   int cols, T* __restrict__ dst) {
  WARP_LOOP(cnt) {
    const T* s = src + size_t(idx[w]) * lds;
    T* d = dst + w * cols;
    for (int c = lane; c < cols; c += 32) d[c] = s[c];
  }
}

// y[t, :] = p[t, sel[t]] * eout[pos[t], :]  (layers_moe.cpp:90-94, applied once
// all experts have passed: each token is routed to exactly one)
template <typename T>
__global__ void moe_combine_kernel(const T* __restrict__ eout, const int* __restrict__ pos,
                                   const int* __restrict__ sel, const double* __restrict__ probs, int n, size_t rows,
                                   int H, T* __restrict__ y, size_t ldy) {
  WARP_LOOP(rows) {
    const double p = probs[w * n + sel[w]];
    const T* e = eout + size_t(pos[w]) * H;
    for (int c = lane; c < H; c += 32) stf(y, w * ldy + c, float(p * double(ldf(e, c))));
  }
}

// Per routed row i of expert j (token t = rows[i]): de_i = p_tj dy_t;
// dp = dy_t . e_i; dlogits[t, k] = dp p_tj (delta_jk - p_tk)  (:146-160)
template <typename T>
__global__ void moe_route_bwd_kernel(const T* __restrict__ dy, size_t ldy, const T* __restrict__ eout,
                                     const int* __restrict__ rows_j, size_t cnt, int j, const double* __restrict__ probs,
                                     int n, int H, T* __restrict__ de, double* __restrict__ dlogits) {
  WARP_LOOP(cnt) {
    const size_t t = size_t(rows_j[w]);
    const double pj = probs[t * n + j];
    double dp = 0.0;
    for (int c = lane; c < H; c += 32) {
      const float d = ldf(dy, t * ldy + c);
      stf(de, w * H + c, float(pj * double(d)));
      dp += double(d) * double(ldf(eout, w * H + c));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dp += __shfl_xor_sync(0xffffffffu, dp, o);
    if (lane < n) dlogits[t * n + lane] = dp * pj * ((lane == j ? 1.0 : 0.0) - probs[t * n + lane]);
  }
}

// dx[t, :] = dxs[pos[t], :] + dlogits[t, :] . gate^T   (:178-186)
template <typename T>
__global__ void moe_dx_kernel(const T* __restrict__ dxs, const int* __restrict__ pos,
                              const double* __restrict__ dlogits, const double* __restrict__ gate, int n, size_t rows,
                              int H, T* __restrict__ dx, size_t ldx) {
  WARP_LOOP(rows) {
    const T* s = dxs + size_t(pos[w]) * H;
    for (int c = lane; c < H; c += 32) {
      double acc = double(ldf(s, c));
      for (int k = 0; k < n; ++k) acc += dlogits[w * n + k] * gate[size_t(c) * n + k];
      stf(dx, w * ldx + c, float(acc));
    }
  }
}

// gate_grad (H x n) (+)= X^T dlogits: thread per (c, k), tokens in order (deterministic).
template <typename T>
__global__ void moe_gate_grad_kernel(const T* __restrict__ x, size_t ldx, const double* __restrict__ dlogits, int n,
                                     size_t rows, int H, double* __restrict__ gg, int accumulate) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < size_t(H) * n;
       e += size_t(gridDim.x) * blockDim.x) {
    const int c = int(e / n), k = int(e - size_t(c) * n);
    double acc = accumulate ? gg[e] : 0.0;
    for (size_t t = 0; t < rows; ++t) acc += double(ldf(x, t * ldx + c)) * dlogits[t * n + k];
    gg[e] = acc;
  }
}

// y[i, col0 : col0 + per] = block[ids[i], :]   (layers_linear.cpp:96-103)
template <typename T>
__global__ void embed_gather_kernel(const T* __restrict__ block, int per, const int64_t* __restrict__ ids, size_t cnt,
                                    T* __restrict__ y, size_t ldy, int col0) {
  WARP_LOOP(cnt) {
    const T* s = block + size_t(ids[w]) * per;
    T* d = y + w * ldy + col0;
    for (int c = lane; c < per; c += 32) d[c] = s[c];
  }
}

// grad[v, :] += dy[i, col0 : col0 + per] for the tokens i of id v in
// ascending order (the reference's axpy order, :123-131); CSR over unique ids.
template <typename T>
__global__ void embed_scatter_kernel(const T* __restrict__ dy, size_t ldy, int col0, const int64_t* __restrict__ uniq,
                                     const int* __restrict__ offs, const int* __restrict__ toks, size_t nuniq, int per,
                                     float* __restrict__ grad) {
  WARP_LOOP(nuniq) {
    float* g = grad + size_t(uniq[w]) * per;
    const int a = offs[w], b = offs[w + 1];
    for (int c = lane; c < per; c += 32) {
      float acc = g[c];
      for (int i = a; i < b; ++i) acc += ldf(dy, size_t(toks[i]) * ldy + col0 + c);
      g[c] = acc;
    }
  }
}

int post(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  count_launch();
  return RTPB_OK;
}

}  // namespace

#define DISPATCH(f32, KERNEL, ...)                                                                     \
  ((f32) ? (KERNEL<float><<<__VA_ARGS__>>>) : (KERNEL<__nv_bfloat16><<<__VA_ARGS__>>>))

int moe_gate(bool f32, const void* x, size_t rows, size_t H, const double* gate, size_t n, double* probs, int* sel,
             cudaStream_t s) {
  if (n == 0 || n > 32) return set_error(RTPB_ERR_CONFIG, "moe gate: 1..32 experts");
  if (!rows) return RTPB_OK;
  if (f32)
    moe_gate_kernel<float><<<grid_warps(rows), kWarps * 32, 0, s>>>(static_cast<const float*>(x), rows, int(H), gate,
                                                                    int(n), probs, sel);
  else
    moe_gate_kernel<__nv_bfloat16><<<grid_warps(rows), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), rows, int(H), gate, int(n), probs, sel);
  return post("moe_gate_kernel");
}

int gather_rows(bool f32, const void* src, size_t lds, const int* idx, size_t cnt, size_t cols, void* dst,
                cudaStream_t s) {
  if (!cnt) return RTPB_OK;
  if (f32)
    gather_rows_kernel<float><<<grid_warps(cnt), kWarps * 32, 0, s>>>(static_cast<const float*>(src), lds, idx, cnt,
                                                                      int(cols), static_cast<float*>(dst));
  else
    gather_rows_kernel<__nv_bfloat16><<<grid_warps(cnt), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(src), lds, idx, cnt, int(cols), static_cast<__nv_bfloat16*>(dst));
  return post("gather_rows_kernel");
}

int moe_combine(bool f32, const void* eout, const int* pos, const int* sel, const double* probs, size_t n, size_t rows,
                size_t H, void* y, size_t ldy, cudaStream_t s) {
  if (!rows) return RTPB_OK;
  if (f32)
    moe_combine_kernel<float><<<grid_warps(rows), kWarps * 32, 0, s>>>(
        static_cast<const float*>(eout), pos, sel, probs, int(n), rows, int(H), static_cast<float*>(y), ldy);
  else
    moe_combine_kernel<__nv_bfloat16><<<grid_warps(rows), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(eout), pos, sel, probs, int(n), rows, int(H),
        static_cast<__nv_bfloat16*>(y), ldy);
  return post("moe_combine_kernel");
}

int moe_route_bwd(bool f32, const void* dy, size_t ldy, const void* eout, const int* rows_j, size_t cnt, size_t j,
                  const double* probs, size_t n, size_t H, void* de, double* dlogits, cudaStream_t s) {
  if (!cnt) return RTPB_OK;
  if (f32)
    moe_route_bwd_kernel<float><<<grid_warps(cnt), kWarps * 32, 0, s>>>(
        static_cast<const float*>(dy), ldy, static_cast<const float*>(eout), rows_j, cnt, int(j), probs, int(n),
        int(H), static_cast<float*>(de), dlogits);
  else
    moe_route_bwd_kernel<__nv_bfloat16><<<grid_warps(cnt), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(dy), ldy, static_cast<const __nv_bfloat16*>(eout), rows_j, cnt, int(j),
        probs, int(n), int(H), static_cast<__nv_bfloat16*>(de), dlogits);
  return post("moe_route_bwd_kernel");
}

int moe_dx(bool f32, const void* dxs, const int* pos, const double* dlogits, const double* gate, size_t n, size_t rows,
           size_t H, void* dx, size_t ldx, cudaStream_t s) {
  if (!rows) return RTPB_OK;
  if (f32)
    moe_dx_kernel<float><<<grid_warps(rows), kWarps * 32, 0, s>>>(static_cast<const float*>(dxs), pos, dlogits, gate,
                                                                  int(n), rows, int(H), static_cast<float*>(dx), ldx);
  else
    moe_dx_kernel<__nv_bfloat16><<<grid_warps(rows), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(dxs), pos, dlogits, gate, int(n), rows, int(H),
        static_cast<__nv_bfloat16*>(dx), ldx);
  return post("moe_dx_kernel");
}

int moe_gate_grad(bool f32, const void* x, size_t ldx, const double* dlogits, size_t n, size_t rows, size_t H,
                  double* gg, bool accumulate, cudaStream_t s) {
  const size_t work = H * n;
  const unsigned blocks = unsigned(std::min<size_t>((work + 255) / 256, 148 * 8));
  if (f32)
    moe_gate_grad_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(x), ldx, dlogits, int(n), rows,
                                                       int(H), gg, accumulate);
  else
    moe_gate_grad_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), ldx, dlogits,
                                                               int(n), rows, int(H), gg, accumulate);
  return post("moe_gate_grad_kernel");
}

int embed_gather(bool f32, const void* block, size_t per, const int64_t* ids, size_t cnt, void* y, size_t ldy,
                 size_t col0, cudaStream_t s) {
  if (!cnt) return RTPB_OK;
  if (f32)
    embed_gather_kernel<float><<<grid_warps(cnt), kWarps * 32, 0, s>>>(static_cast<const float*>(block), int(per), ids,
                                                                       cnt, static_cast<float*>(y), ldy, int(col0));
  else
    embed_gather_kernel<__nv_bfloat16><<<grid_warps(cnt), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(block), int(per), ids, cnt, static_cast<__nv_bfloat16*>(y), ldy, int(col0));
  return post("embed_gather_kernel");
}

int embed_scatter(bool f32, const void* dy, size_t ldy, size_t col0, const int64_t* uniq, const int* offs,
                  const int* toks, size_t nuniq, size_t per, float* grad, cudaStream_t s) {
  if (!nuniq) return RTPB_OK;
  if (f32)
    embed_scatter_kernel<float><<<grid_warps(nuniq), kWarps * 32, 0, s>>>(
        static_cast<const float*>(dy), ldy, int(col0), uniq, offs, toks, nuniq, int(per), grad);
  else
    embed_scatter_kernel<__nv_bfloat16><<<grid_warps(nuniq), kWarps * 32, 0, s>>>(
        static_cast<const __nv_bfloat16*>(dy), ldy, int(col0), uniq, offs, toks, nuniq, int(per), grad);
  return post("embed_scatter_kernel");
}

const void* kernel_anchor_moe_embed() {
  return reinterpret_cast<const void*>(&gather_rows_kernel<__nv_bfloat16>);
}

}  // namespace rtpb
