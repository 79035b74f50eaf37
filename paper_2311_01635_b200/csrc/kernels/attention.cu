// Attention core of RtpAttention (layers_attention.cpp:84-101 forward,
// :134-166 backward) for one head group: per (sequence b, head h) of the
// group, S = Q_bh K_bh^T / sqrt(hd), P = softmax_rows(S), O = P V_bh, and its
// backward. Q, K, V, O are rows x gw (gw = g * hd) with row = b * seq + t and
// head h in columns [h * hd, (h + 1) * hd): the reference's read_head /
// write_head packing.
//
// Flash-style: the forward keeps one running (max, sum) per query row
// (online softmax over key tiles) and saves lse = max + log(sum) per (row,
// head) instead of the seq x seq probabilities the reference tapes; the
// backward recomputes P from Q, K and lse. Deterministic (no atomics): dQ is
// reduced per query row, dK / dV per key row.
//
// Execution: one warp per query (forward, dQ) or key (dK / dV) row, 8 warps
// per CTA sharing 32-row tiles of the other side staged in shared memory;
// lanes own key/query positions for the dot products and head dimensions for
// the weighted sums. fp32 arithmetic, bf16 or fp32 storage. hd <= 256.
#include <cuda_bf16.h>

#include "launch.hpp"

namespace rtpb {

namespace {

constexpr int kWarps = 8;
constexpr int kTile = 32;
constexpr int kMaxHd = 256;

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

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stages rows [r0, r0 + kTile) of head columns [c0, c0 + hd) of src (ld = gw)
// into dst[kTile][hd] (rows past `limit` zero).
template <typename T>
__device__ __forceinline__ void stage_tile(float* dst, const T* src, size_t base_row, int r0, int limit, int hd,
                                           int gw, int c0) {
  for (int i = threadIdx.x; i < kTile * hd; i += blockDim.x) {
    const int r = i / hd, d = i - r * hd;
    dst[i] = (r0 + r < limit) ? ldf(src, (base_row + r0 + r) * size_t(gw) + c0 + d) : 0.f;
  }
}

// grid: (ceil(seq / kWarps), g, batch); warp w handles query t = blockIdx.x * kWarps + w.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) attn_fwd_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                               const T* __restrict__ v, T* __restrict__ o,
                                                               float* __restrict__ lse, int seq, int g, int hd,
                                                               float scale) {
  extern __shared__ float sm[];
  float* ks = sm;                       // kTile x hd
  float* vs = ks + kTile * hd;          // kTile x hd
  float* qs = vs + kTile * hd;          // kWarps x hd
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z, gw = g * hd, c0 = h * hd;
  const int t = blockIdx.x * kWarps + warp;
  const bool active = t < seq;
  const size_t base = size_t(b) * seq;
  float* qw = qs + warp * hd;
  for (int d = lane; d < hd; d += 32) qw[d] = active ? ldf(q, (base + t) * gw + c0 + d) * scale : 0.f;
  float m = -INFINITY, l = 0.f;
  float acc[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) acc[i] = 0.f;
  for (int j0 = 0; j0 < seq; j0 += kTile) {
    __syncthreads();  // previous tile consumed
    stage_tile(ks, k, base, j0, seq, hd, gw, c0);
    stage_tile(vs, v, base, j0, seq, hd, gw, c0);
    __syncthreads();
    // lane = key j0 + lane: s = (q * scale) . k
    float s = -INFINITY;
    if (j0 + lane < seq) {
      s = 0.f;
      const float* kr = ks + lane * hd;
      for (int d = 0; d < hd; ++d) s = fmaf(qw[d], kr[d], s);
    }
    const float mt = warp_max(s);
    const float mn = fmaxf(m, mt);
    const float corr = m == -INFINITY ? 0.f : __expf(m - mn);
    const float p = (j0 + lane < seq) ? __expf(s - mn) : 0.f;
    l = l * corr + warp_sum(p);
#pragma unroll
    for (int i = 0; i < kMaxHd / 32; ++i) acc[i] *= corr;
    const int nk = min(kTile, seq - j0);
    for (int jj = 0; jj < nk; ++jj) {
      const float pj = __shfl_sync(0xffffffffu, p, jj);
      const float* vr = vs + jj * hd;
#pragma unroll
      for (int i = 0; i < kMaxHd / 32; ++i) {
        const int d = lane + 32 * i;
        if (d < hd) acc[i] = fmaf(pj, vr[d], acc[i]);
      }
    }
    m = mn;
  }
  if (!active) return;
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) stf(o, (base + t) * gw + c0 + d, acc[i] * inv);
  }
  if (lane == 0) lse[(base + t) * g + h] = m + __logf(l);
}

// Dt[row, h] = rowsum(dO_t * O_t) over the head's columns (= rowsum(dP * P)).
template <typename T>
__global__ void attn_bwd_delta_kernel(const T* __restrict__ o, const T* __restrict__ dout, float* __restrict__ delta,
                                      size_t rows, int g, int hd) {
  const int gw = g * hd;
  const size_t warps = size_t(gridDim.x) * kWarps;
  for (size_t w = blockIdx.x * size_t(kWarps) + threadIdx.x / 32; w < rows * g; w += warps) {
    const size_t row = w / g;
    const int h = int(w - row * g), lane = threadIdx.x & 31;
    float s = 0.f;
    for (int d = lane; d < hd; d += 32) s += ldf(o, row * gw + h * hd + d) * ldf(dout, row * gw + h * hd + d);
    s = warp_sum(s);
    if (lane == 0) delta[w] = s;
  }
}

// dQ: warp per query row t; key tiles staged. dS = P * (dP - D) * scale,
// dQ = dS K (dq_scale = scale applied once at the end).
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) attn_bwd_dq_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                                  const T* __restrict__ v, const T* __restrict__ dout,
                                                                  const float* __restrict__ lse,
                                                                  const float* __restrict__ delta, T* __restrict__ dq,
                                                                  int seq, int g, int hd, float scale) {
  extern __shared__ float sm[];
  float* ks = sm;
  float* vs = ks + kTile * hd;
  float* qs = vs + kTile * hd;   // kWarps x hd (q * scale)
  float* dos = qs + kWarps * hd; // kWarps x hd
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z, gw = g * hd, c0 = h * hd;
  const int t = blockIdx.x * kWarps + warp;
  const bool active = t < seq;
  const size_t base = size_t(b) * seq;
  float* qw = qs + warp * hd;
  float* dw = dos + warp * hd;
  for (int d = lane; d < hd; d += 32) {
    qw[d] = active ? ldf(q, (base + t) * gw + c0 + d) * scale : 0.f;
    dw[d] = active ? ldf(dout, (base + t) * gw + c0 + d) : 0.f;
  }
  const float L = active ? lse[(base + t) * g + h] : 0.f;
  const float D = active ? delta[(base + t) * g + h] : 0.f;
  float acc[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) acc[i] = 0.f;
  for (int j0 = 0; j0 < seq; j0 += kTile) {
    __syncthreads();
    stage_tile(ks, k, base, j0, seq, hd, gw, c0);
    stage_tile(vs, v, base, j0, seq, hd, gw, c0);
    __syncthreads();
    float ds = 0.f;
    if (j0 + lane < seq && active) {
      const float* kr = ks + lane * hd;
      const float* vr = vs + lane * hd;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < hd; ++d) {
        s = fmaf(qw[d], kr[d], s);
        dp = fmaf(dw[d], vr[d], dp);
      }
      const float p = __expf(s - L);
      ds = p * (dp - D);
    }
    const int nk = min(kTile, seq - j0);
    for (int jj = 0; jj < nk; ++jj) {
      const float dsj = __shfl_sync(0xffffffffu, ds, jj);
      const float* kr = ks + jj * hd;
#pragma unroll
      for (int i = 0; i < kMaxHd / 32; ++i) {
        const int d = lane + 32 * i;
        if (d < hd) acc[i] = fmaf(dsj, kr[d], acc[i]);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) stf(dq, (base + t) * gw + c0 + d, acc[i] * scale);
  }
}

// dK, dV: warp per key row j; query tiles staged. dV = P^T dO, dK = dS^T Q * scale.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) attn_bwd_dkdv_kernel(
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, const T* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ delta, T* __restrict__ dk, T* __restrict__ dv, int seq,
    int g, int hd, float scale) {
  extern __shared__ float sm[];
  float* qs = sm;                    // kTile x hd (q * scale)
  float* dos = qs + kTile * hd;      // kTile x hd
  float* ls = dos + kTile * hd;      // kTile lse
  float* dl = ls + kTile;            // kTile delta
  float* kw_all = dl + kTile;        // kWarps x hd
  float* vw_all = kw_all + kWarps * hd;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int h = blockIdx.y, b = blockIdx.z, gw = g * hd, c0 = h * hd;
  const int j = blockIdx.x * kWarps + warp;
  const bool active = j < seq;
  const size_t base = size_t(b) * seq;
  float* kw = kw_all + warp * hd;
  float* vw = vw_all + warp * hd;
  for (int d = lane; d < hd; d += 32) {
    kw[d] = active ? ldf(k, (base + j) * gw + c0 + d) : 0.f;
    vw[d] = active ? ldf(v, (base + j) * gw + c0 + d) : 0.f;
  }
  float ak[kMaxHd / 32], av[kMaxHd / 32];
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) ak[i] = av[i] = 0.f;
  for (int t0 = 0; t0 < seq; t0 += kTile) {
    __syncthreads();
    for (int i = threadIdx.x; i < kTile * hd; i += blockDim.x) {
      const int r = i / hd, d = i - r * hd;
      const bool ok = t0 + r < seq;
      qs[i] = ok ? ldf(q, (base + t0 + r) * gw + c0 + d) * scale : 0.f;
      dos[i] = ok ? ldf(dout, (base + t0 + r) * gw + c0 + d) : 0.f;
    }
    for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
      const bool ok = t0 + i < seq;
      ls[i] = ok ? lse[(base + t0 + i) * g + h] : 0.f;
      dl[i] = ok ? delta[(base + t0 + i) * g + h] : 0.f;
    }
    __syncthreads();
    // lane = query t0 + lane
    float p = 0.f, ds = 0.f;
    if (t0 + lane < seq && active) {
      const float* qr = qs + lane * hd;
      const float* dr = dos + lane * hd;
      float s = 0.f, dp = 0.f;
      for (int d = 0; d < hd; ++d) {
        s = fmaf(qr[d], kw[d], s);
        dp = fmaf(dr[d], vw[d], dp);
      }
      p = __expf(s - ls[lane]);
      ds = p * (dp - dl[lane]);
    }
    const int nq = min(kTile, seq - t0);
    for (int tt = 0; tt < nq; ++tt) {
      const float pt = __shfl_sync(0xffffffffu, p, tt);
      const float dst = __shfl_sync(0xffffffffu, ds, tt);
      const float* qr = qs + tt * hd;  // already * scale: dK = dS^T (Q scale)
      const float* dr = dos + tt * hd;
#pragma unroll
      for (int i = 0; i < kMaxHd / 32; ++i) {
        const int d = lane + 32 * i;
        if (d < hd) {
          av[i] = fmaf(pt, dr[d], av[i]);
          ak[i] = fmaf(dst, qr[d], ak[i]);
        }
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int i = 0; i < kMaxHd / 32; ++i) {
    const int d = lane + 32 * i;
    if (d < hd) {
      stf(dk, (base + j) * gw + c0 + d, ak[i]);
      stf(dv, (base + j) * gw + c0 + d, av[i]);
    }
  }
}

// Opt a kernel into more than 48 KB of dynamic shared memory (hd > 96).
template <typename K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

int post(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  count_launch();
  return RTPB_OK;
}

int check(size_t rows, size_t seq, size_t g, size_t hd) {
  if (!rows || !seq || !g || !hd) return set_error(RTPB_ERR_DIMENSION, "attention core: dimensions must be positive");
  if (rows % seq) return set_error(RTPB_ERR_DIMENSION, "attention core: rows must be whole sequences");
  if (hd > size_t(kMaxHd)) return set_error(RTPB_ERR_CONFIG, "attention core: head_dim above 256");
  if (rows / seq > 65535 || g > 65535) return set_error(RTPB_ERR_DIMENSION, "attention core: grid too large");
  return RTPB_OK;
}

}  // namespace

int attention_core_fwd(bool f32, const void* q, const void* k, const void* v, void* o, float* lse, size_t rows,
                       size_t seq, size_t g, size_t hd, float scale, cudaStream_t s) {
  int rc = check(rows, seq, g, hd);
  if (rc) return rc;
  dim3 grid(unsigned((seq + kWarps - 1) / kWarps), unsigned(g), unsigned(rows / seq));
  const size_t smem = (2 * kTile + kWarps) * hd * sizeof(float);
  allow_smem(attn_fwd_kernel<float>, smem);
  allow_smem(attn_fwd_kernel<__nv_bfloat16>, smem);
  if (f32)
    attn_fwd_kernel<float><<<grid, kWarps * 32, smem, s>>>(static_cast<const float*>(q), static_cast<const float*>(k),
                                                           static_cast<const float*>(v), static_cast<float*>(o), lse,
                                                           int(seq), int(g), int(hd), scale);
  else
    attn_fwd_kernel<__nv_bfloat16><<<grid, kWarps * 32, smem, s>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
        static_cast<const __nv_bfloat16*>(v), static_cast<__nv_bfloat16*>(o), lse, int(seq), int(g), int(hd), scale);
  return post("attn_fwd_kernel");
}

int attention_core_bwd(bool f32, const void* q, const void* k, const void* v, const void* o, const float* lse,
                       const void* dout, void* dq, void* dk, void* dv, float* delta, size_t rows, size_t seq,
                       size_t g, size_t hd, float scale, cudaStream_t s) {
  int rc = check(rows, seq, g, hd);
  if (rc) return rc;
  const unsigned dgrid = unsigned(std::min<size_t>((rows * g + kWarps - 1) / kWarps, 148 * 16));
  dim3 grid(unsigned((seq + kWarps - 1) / kWarps), unsigned(g), unsigned(rows / seq));
  const size_t smem_q = (2 * kTile + 2 * kWarps) * hd * sizeof(float);
  const size_t smem_k = ((2 * kTile + 2 * kWarps) * hd + 2 * kTile) * sizeof(float);
  allow_smem(attn_bwd_dq_kernel<float>, smem_q);
  allow_smem(attn_bwd_dq_kernel<__nv_bfloat16>, smem_q);
  allow_smem(attn_bwd_dkdv_kernel<float>, smem_k);
  allow_smem(attn_bwd_dkdv_kernel<__nv_bfloat16>, smem_k);
  if (f32) {
    using T = float;
    attn_bwd_delta_kernel<T><<<dgrid, kWarps * 32, 0, s>>>(static_cast<const T*>(o), static_cast<const T*>(dout),
                                                           delta, rows, int(g), int(hd));
    if ((rc = post("attn_bwd_delta_kernel"))) return rc;
    attn_bwd_dq_kernel<T><<<grid, kWarps * 32, smem_q, s>>>(
        static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<const T*>(dout), lse,
        delta, static_cast<T*>(dq), int(seq), int(g), int(hd), scale);
    if ((rc = post("attn_bwd_dq_kernel"))) return rc;
    attn_bwd_dkdv_kernel<T><<<grid, kWarps * 32, smem_k, s>>>(
        static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<const T*>(dout), lse,
        delta, static_cast<T*>(dk), static_cast<T*>(dv), int(seq), int(g), int(hd), scale);
  } else {
    using T = __nv_bfloat16;
    attn_bwd_delta_kernel<T><<<dgrid, kWarps * 32, 0, s>>>(static_cast<const T*>(o), static_cast<const T*>(dout),
                                                           delta, rows, int(g), int(hd));
    if ((rc = post("attn_bwd_delta_kernel"))) return rc;
    attn_bwd_dq_kernel<T><<<grid, kWarps * 32, smem_q, s>>>(
        static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<const T*>(dout), lse,
        delta, static_cast<T*>(dq), int(seq), int(g), int(hd), scale);
    if ((rc = post("attn_bwd_dq_kernel"))) return rc;
    attn_bwd_dkdv_kernel<T><<<grid, kWarps * 32, smem_k, s>>>(
        static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<const T*>(dout), lse,
        delta, static_cast<T*>(dk), static_cast<T*>(dv), int(seq), int(g), int(hd), scale);
  }
  return post("attn_bwd_dkdv_kernel");
}

const void* kernel_anchor_attention() {
  return reinterpret_cast<const void*>(&attn_bwd_delta_kernel<__nv_bfloat16>);
}

}  // namespace rtpb
