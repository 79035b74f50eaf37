/* oracle/rtp_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * Plain-C fp64 restatement of the reference RTP linear/MLP path; see
 * rtp_oracle.h. Compiled with -ffp-contract=off so every product/sum rounds
 * exactly as the reference's kernels do (reference CMakeLists.txt:8-14).
 * OpenMP only splits independent output rows; the per-element summation order
 * is the reference's, so results are bit-identical at any thread count.
 */
#include "rtp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN_GAMMA 0x9E3779B97F4A7C15ULL

/* rng.hpp:16-22: state += gamma; z = state; two xor-shift-multiply rounds. */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t orc_splitmix_at(uint64_t seed, uint64_t k) { return mix64(seed + (k + 1) * GOLDEN_GAMMA); }

/* rng.hpp:25-27: lo + (hi - lo) * ((u >> 11) * 2^-53), two separate roundings. */
double orc_uniform_at(uint64_t seed, uint64_t k, double lo, double hi) {
  const double unit = (double)(orc_splitmix_at(seed, k) >> 11) * 0x1.0p-53;
  const double span = hi - lo;
  const double scaled = span * unit;
  return lo + scaled;
}

void orc_uniform(uint64_t seed, uint64_t skip, uint64_t count, double lo, double hi, double* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = orc_uniform_at(seed, skip + i, lo, hi);
}

void orc_linear_shard(uint64_t seed, uint64_t base, size_t I, size_t O, size_t n, size_t j,
                      double* out) {
  const size_t per = O / n;
  for (size_t i = 0; i < I; ++i)
    for (size_t c = 0; c < per; ++c)
      out[i * per + c] = orc_uniform_at(seed, base + i * O + j * per + c, -0.1, 0.1);
  for (size_t c = 0; c < per; ++c)
    out[I * per + c] = orc_uniform_at(seed, base + I * O + j * per + c, -0.1, 0.1);
}

/* kernels_scalar.cpp:6-17: c = 0, then c[i,j] += a[i,t]*b[t,j], t ascending. */
void orc_matmul(const double* a, size_t lda, const double* b, size_t ldb, double* c, size_t ldc,
                size_t m, size_t k, size_t n) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; ++i) {
    double* crow = c + i * ldc;
    for (size_t j = 0; j < n; ++j) crow[j] = 0.0;
    for (size_t t = 0; t < k; ++t) {
      const double av = a[i * lda + t];
      const double* brow = b + t * ldb;
      for (size_t j = 0; j < n; ++j) crow[j] += av * brow[j];
    }
  }
}

/* kernels_scalar.cpp:31-42: c[i,j] += a[t,i]*b[t,j], t outermost ascending. */
void orc_matmul_tn_acc(const double* a, size_t lda, const double* b, size_t ldb, double* c,
                       size_t ldc, size_t m, size_t k, size_t n) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; ++i) {
    double* crow = c + i * ldc;
    for (size_t t = 0; t < k; ++t) {
      const double av = a[t * lda + i];
      const double* brow = b + t * ldb;
      for (size_t j = 0; j < n; ++j) crow[j] += av * brow[j];
    }
  }
}

/* kernels_scalar.cpp:44-56: acc = c[i,j]; acc += a[i,t]*b[j,t]; t ascending. */
void orc_matmul_nt_acc(const double* a, size_t lda, const double* b, size_t ldb, double* c,
                       size_t ldc, size_t m, size_t k, size_t n) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < m; ++i) {
    const double* arow = a + i * lda;
    double* crow = c + i * ldc;
    for (size_t j = 0; j < n; ++j) {
      const double* brow = b + j * ldb;
      double acc = crow[j];
      for (size_t t = 0; t < k; ++t) acc += arow[t] * brow[t];
      crow[j] = acc;
    }
  }
}

static const double kInvSqrt2 = 0.7071067811865475244;
static const double kInvSqrt2Pi = 0.3989422804014326779;

/* tensor.cpp:328-337 */
void orc_gelu(const double* x, double* y, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    const double phi = 0.5 * (1.0 + erf(x[i] * kInvSqrt2));
    y[i] = x[i] * phi;
  }
}

/* tensor.cpp:339-351 */
void orc_gelu_backward(const double* x, const double* up, double* out, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    const double phi = 0.5 * (1.0 + erf(x[i] * kInvSqrt2));
    const double pdf = kInvSqrt2Pi * exp(-0.5 * x[i] * x[i]);
    out[i] = up[i] * (phi + x[i] * pdf);
  }
}

/* One worker's resident state (ring.hpp:23-28). Rotation permutes whole
 * slots' buffers; values are never mutated by it (ring.cpp:247-293). */
typedef struct {
  double* weight;
  double* grad;
  size_t logical_id;
} slot_t;

/* rotate_clockwise, PayloadKind::Weight (ring.cpp:265-278): rank r's weight
 * and id move to r+1; grad buffers stay put. */
static void rotate_cw_weight(slot_t* s, size_t n) {
  double* w_last = s[n - 1].weight;
  size_t id_last = s[n - 1].logical_id;
  for (size_t r = n - 1; r > 0; --r) {
    s[r].weight = s[r - 1].weight;
    s[r].logical_id = s[r - 1].logical_id;
  }
  s[0].weight = w_last;
  s[0].logical_id = id_last;
}

/* rotate_counterclockwise, PayloadKind::WeightAndGrad (ring.cpp:280-293):
 * rank r's weight, grad and id move to r-1. */
static void rotate_ccw_weight_grad(slot_t* s, size_t n) {
  slot_t first = s[0];
  for (size_t r = 0; r + 1 < n; ++r) s[r] = s[r + 1];
  s[n - 1] = first;
}

int orc_rtp_linear(size_t n, size_t rows, size_t I, size_t O, const double* w, const double* b,
                   const double* x, const double* dy, double* y, double* dx, double* grads,
                   int64_t* trace) {
  if (n == 0 || O % n != 0 || rows % n != 0) return 2; /* partition.cpp:58-69, model.cpp:166 */
  const size_t per = O / n, L = I * per + per, M = rows / n;
  double* store = (double*)calloc(2 * n * L, sizeof(double));
  slot_t* slots = (slot_t*)malloc(n * sizeof(slot_t));
  /* init_slots (layers_common.cpp:100-118): shard r -> worker r, zero grads. */
  for (size_t r = 0; r < n; ++r) {
    slots[r].weight = store + r * L;
    slots[r].grad = store + (n + r) * L;
    slots[r].logical_id = r;
    for (size_t i = 0; i < I; ++i)
      for (size_t c = 0; c < per; ++c) slots[r].weight[i * per + c] = w[i * O + r * per + c];
    for (size_t c = 0; c < per; ++c) slots[r].weight[I * per + c] = b[r * per + c];
  }
  /* forward (layers_linear.cpp:26-41) */
  for (size_t s = 0; s < n; ++s) {
    for (size_t r = 0; r < n; ++r) {
      const size_t j = slots[r].logical_id;
      if (trace) trace[s * n + r] = (int64_t)j;
      const double* wj = slots[r].weight;
      const double* bj = wj + I * per;
      double* block = y + r * M * O + j * per;
      orc_matmul(x + r * M * I, I, wj, per, block, O, M, I, per);
      for (size_t i = 0; i < M; ++i)
        for (size_t c = 0; c < per; ++c) block[i * O + c] = block[i * O + c] + bj[c];
    }
    if (s + 1 < n) rotate_cw_weight(slots, n);
  }
  /* backward (layers_linear.cpp:46-72) */
  memset(dx, 0, rows * I * sizeof(double));
  for (size_t s = 0; s < n; ++s) {
    for (size_t r = 0; r < n; ++r) {
      const size_t j = slots[r].logical_id;
      if (trace) trace[n * n + s * n + r] = (int64_t)j;
      const double* dyj = dy + r * M * O + j * per;
      const double* xr = x + r * M * I;
      double* gw = slots[r].grad;
      double* gb = gw + I * per;
      orc_matmul_tn_acc(xr, I, dyj, O, gw, per, I, M, per);
      for (size_t i = 0; i < M; ++i)
        for (size_t c = 0; c < per; ++c) gb[c] = gb[c] + dyj[i * O + c];
      orc_matmul_nt_acc(dyj, O, slots[r].weight, per, dx + r * M * I, I, M, per, I);
    }
    if (s + 1 < n) rotate_ccw_weight_grad(slots, n);
  }
  for (size_t r = 0; r < n; ++r) memcpy(grads + r * L, slots[r].grad, L * sizeof(double));
  free(slots);
  free(store);
  return 0;
}

int orc_rtp_mlp(size_t n, size_t rows, size_t h, size_t f, const double* w1, const double* b1,
                const double* w2, const double* b2, const double* x, const double* dy, double* y,
                double* dx, double* grads1, double* grads2) {
  if (n == 0 || f % n != 0 || h % n != 0 || rows % n != 0) return 2;
  double* pre = (double*)malloc(rows * f * sizeof(double));
  double* hh = (double*)malloc(rows * f * sizeof(double));
  double* dh = (double*)malloc(rows * f * sizeof(double));
  double* dpre = (double*)malloc(rows * f * sizeof(double));
  /* model.cpp order: ffn1 fwd, gelu, ffn2 fwd+bwd, gelu', ffn1 bwd.
   * orc_rtp_linear fuses a layer's fwd and bwd, so ffn1's forward is first
   * run alone (identical arithmetic) to obtain pre, and ffn1's fwd+bwd call
   * later recomputes the same bits while consuming the true dpre. */
  {
    /* pre = ffn1.forward(x): same loop as orc_rtp_linear's forward. */
    const size_t per = f / n, M = rows / n;
    for (size_t r = 0; r < n; ++r)
      for (size_t s = 0; s < n; ++s) {
        const size_t j = (r + n - s) % n; /* check_forward_position law */
        double* block = pre + r * M * f + j * per;
        orc_matmul(x + r * M * h, h, w1 + j * per, f, block, f, M, h, per);
        for (size_t i = 0; i < M; ++i)
          for (size_t c = 0; c < per; ++c) block[i * f + c] = block[i * f + c] + b1[j * per + c];
      }
  }
  orc_gelu(pre, hh, rows * f);
  int rc = orc_rtp_linear(n, rows, f, h, w2, b2, hh, dy, y, dh, grads2, NULL);
  if (rc == 0) {
    orc_gelu_backward(pre, dh, dpre, rows * f);
    double* pre2 = (double*)malloc(rows * f * sizeof(double));
    rc = orc_rtp_linear(n, rows, h, f, w1, b1, x, dpre, pre2, dx, grads1, NULL);
    free(pre2);
  }
  free(pre);
  free(hh);
  free(dh);
  free(dpre);
  return rc;
}

/* kernels_scalar.cpp:19-29 (matmul_acc): c[i,j] += a[i,t]*b[t,j], t ascending. */
static void orc_matmul_acc(const double* a, size_t lda, const double* b, size_t ldb, double* c,
                           size_t ldc, size_t m, size_t k, size_t n) {
  for (size_t i = 0; i < m; ++i) {
    double* crow = c + i * ldc;
    for (size_t t = 0; t < k; ++t) {
      const double av = a[i * lda + t];
      const double* brow = b + t * ldb;
      for (size_t j = 0; j < n; ++j) crow[j] += av * brow[j];
    }
  }
}

/* tensor.cpp:305-320: max-subtracted exp, row sum, divide. */
static void orc_softmax_rows(const double* in, double* out, size_t m, size_t n) {
  for (size_t i = 0; i < m; ++i) {
    const double* row = in + i * n;
    double* orow = out + i * n;
    double mx = row[0];
    for (size_t j = 1; j < n; ++j) mx = row[j] > mx ? row[j] : mx;
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j) {
      orow[j] = exp(row[j] - mx);
      sum += orow[j];
    }
    for (size_t j = 0; j < n; ++j) orow[j] /= sum;
  }
}

/* One (sequence b, head h) tile: rows b*seq .. +seq, columns h*hd .. +hd of
 * a rows x width matrix (layers_attention.cpp:12-24). */
static void read_head(const double* src, size_t width, size_t b, size_t h, size_t seq, size_t hd,
                      double* dst) {
  for (size_t t = 0; t < seq; ++t) memcpy(dst + t * hd, src + (b * seq + t) * width + h * hd, hd * sizeof(double));
}
static void write_head(double* dst, size_t width, size_t b, size_t h, size_t seq, size_t hd,
                       const double* src) {
  for (size_t t = 0; t < seq; ++t) memcpy(dst + (b * seq + t) * width + h * hd, src + t * hd, hd * sizeof(double));
}

int orc_rtp_attention(size_t n, size_t rows, size_t H, size_t heads, size_t seq, const double* wq,
                      const double* wk, const double* wv, const double* wo, const double* x,
                      const double* dy, double* y, double* dx, double* grads) {
  /* layout_attention (partition.cpp:71-84), attention_shard_groups
   * (layers_common.cpp:54-74): shard j = [Wq[:, blk j] | Wk[:, blk j] |
   * Wv[:, blk j] | Wo[blk j, :]], each H x gw / gw x H row-major. */
  if (n == 0 || heads == 0 || H % heads != 0 || heads % n != 0 || rows % n != 0) return 2;
  const size_t hd = H / heads, g = heads / n, gw = g * hd, M = rows / n;
  if (M % seq != 0) return 3;
  const size_t batch = M / seq, L = 4 * H * gw;
  const double inv_sqrt_hd = 1.0 / sqrt((double)hd);
  double* store = (double*)calloc(2 * n * L, sizeof(double));
  slot_t* slots = (slot_t*)malloc(n * sizeof(slot_t));
  for (size_t r = 0; r < n; ++r) {
    slots[r].weight = store + r * L;
    slots[r].grad = store + (n + r) * L;
    slots[r].logical_id = r;
    double* w = slots[r].weight;
    for (size_t i = 0; i < H; ++i)
      for (size_t c = 0; c < gw; ++c) {
        w[i * gw + c] = wq[i * H + r * gw + c];
        w[H * gw + i * gw + c] = wk[i * H + r * gw + c];
        w[2 * H * gw + i * gw + c] = wv[i * H + r * gw + c];
      }
    for (size_t i = 0; i < gw; ++i)
      for (size_t c = 0; c < H; ++c) w[3 * H * gw + i * H + c] = wo[(r * gw + i) * H + c];
  }
  /* the tape (layers.hpp:26-55): per (rank, shard) the forward's q, k, v, probs, attn_out */
  const size_t qs = M * gw, ps = batch * g * seq * seq;
  double* tape = (double*)calloc(n * n * (4 * qs + ps), sizeof(double));
#define TAPE(r, j) (tape + ((r) * n + (j)) * (4 * qs + ps))
  double *qbh = (double*)malloc(seq * hd * sizeof(double)), *kbh = (double*)malloc(seq * hd * sizeof(double)),
         *vbh = (double*)malloc(seq * hd * sizeof(double)), *dobh = (double*)malloc(seq * hd * sizeof(double)),
         *obh = (double*)malloc(seq * hd * sizeof(double)), *sc = (double*)malloc(seq * seq * sizeof(double)),
         *dprobs = (double*)malloc(seq * seq * sizeof(double)), *ds = (double*)malloc(seq * seq * sizeof(double)),
         *t1 = (double*)malloc(seq * hd * sizeof(double)), *t2 = (double*)malloc(seq * hd * sizeof(double)),
         *t3 = (double*)malloc(seq * hd * sizeof(double));
  double* da = (double*)malloc(qs * sizeof(double));
  double *dq = (double*)malloc(qs * sizeof(double)), *dk = (double*)malloc(qs * sizeof(double)),
         *dv = (double*)malloc(qs * sizeof(double));
  memset(y, 0, rows * H * sizeof(double));
  /* forward (layers_attention.cpp:55-112) */
  for (size_t s = 0; s < n; ++s) {
    for (size_t r = 0; r < n; ++r) {
      const size_t j = slots[r].logical_id;
      const double* w = slots[r].weight;
      const double* xr = x + r * M * H;
      double* T = TAPE(r, j);
      double *q = T, *k = T + qs, *v = T + 2 * qs, *probs = T + 3 * qs, *ao = T + 3 * qs + ps;
      orc_matmul(xr, H, w, gw, q, gw, M, H, gw);
      orc_matmul(xr, H, w + H * gw, gw, k, gw, M, H, gw);
      orc_matmul(xr, H, w + 2 * H * gw, gw, v, gw, M, H, gw);
      for (size_t b = 0; b < batch; ++b)
        for (size_t h = 0; h < g; ++h) {
          read_head(q, gw, b, h, seq, hd, qbh);
          read_head(k, gw, b, h, seq, hd, kbh);
          read_head(v, gw, b, h, seq, hd, vbh);
          memset(sc, 0, seq * seq * sizeof(double));
          orc_matmul_nt_acc(qbh, hd, kbh, hd, sc, seq, seq, hd, seq);
          for (size_t e = 0; e < seq * seq; ++e) sc[e] = sc[e] * inv_sqrt_hd;
          double* pbh = probs + (b * g + h) * seq * seq;
          orc_softmax_rows(sc, pbh, seq, seq);
          orc_matmul(pbh, seq, vbh, hd, obh, hd, seq, seq, hd);
          write_head(ao, gw, b, h, seq, hd, obh);
        }
      orc_matmul_acc(ao, gw, w + 3 * H * gw, H, y + r * M * H, H, M, gw, H);
    }
    if (s + 1 < n) rotate_cw_weight(slots, n);
  }
  /* backward (layers_attention.cpp:114-198) */
  memset(dx, 0, rows * H * sizeof(double));
  for (size_t s = 0; s < n; ++s) {
    for (size_t r = 0; r < n; ++r) {
      const size_t j = slots[r].logical_id;
      const double* w = slots[r].weight;
      double* gr = slots[r].grad;
      const double* T = TAPE(r, j);
      const double *q = T, *k = T + qs, *v = T + 2 * qs, *probs = T + 3 * qs, *ao = T + 3 * qs + ps;
      const double* dyr = dy + r * M * H;
      const double* xr = x + r * M * H;
      orc_matmul_tn_acc(ao, gw, dyr, H, gr + 3 * H * gw, H, gw, M, H);
      memset(da, 0, qs * sizeof(double));
      orc_matmul_nt_acc(dyr, H, w + 3 * H * gw, H, da, gw, M, H, gw);
      for (size_t b = 0; b < batch; ++b)
        for (size_t h = 0; h < g; ++h) {
          read_head(da, gw, b, h, seq, hd, dobh);
          read_head(q, gw, b, h, seq, hd, qbh);
          read_head(k, gw, b, h, seq, hd, kbh);
          read_head(v, gw, b, h, seq, hd, vbh);
          const double* pbh = probs + (b * g + h) * seq * seq;
          memset(dprobs, 0, seq * seq * sizeof(double));
          orc_matmul_nt_acc(dobh, hd, vbh, hd, dprobs, seq, seq, hd, seq);
          memset(t3, 0, seq * hd * sizeof(double)); /* dvbh */
          orc_matmul_tn_acc(pbh, seq, dobh, hd, t3, hd, seq, seq, hd);
          for (size_t i = 0; i < seq; ++i) { /* softmax_backward_rows (:27-36) */
            double dot = 0.0;
            for (size_t jj = 0; jj < seq; ++jj) dot += dprobs[i * seq + jj] * pbh[i * seq + jj];
            for (size_t jj = 0; jj < seq; ++jj) ds[i * seq + jj] = pbh[i * seq + jj] * (dprobs[i * seq + jj] - dot);
          }
          for (size_t e = 0; e < seq * seq; ++e) ds[e] = ds[e] * inv_sqrt_hd;
          orc_matmul(ds, seq, kbh, hd, t1, hd, seq, seq, hd); /* dqbh */
          memset(t2, 0, seq * hd * sizeof(double));            /* dkbh */
          orc_matmul_tn_acc(ds, seq, qbh, hd, t2, hd, seq, seq, hd);
          write_head(dq, gw, b, h, seq, hd, t1);
          write_head(dk, gw, b, h, seq, hd, t2);
          write_head(dv, gw, b, h, seq, hd, t3);
        }
      orc_matmul_tn_acc(xr, H, dq, gw, gr, gw, H, M, gw);
      orc_matmul_tn_acc(xr, H, dk, gw, gr + H * gw, gw, H, M, gw);
      orc_matmul_tn_acc(xr, H, dv, gw, gr + 2 * H * gw, gw, H, M, gw);
      orc_matmul_nt_acc(dq, gw, w, gw, dx + r * M * H, H, M, gw, H);
      orc_matmul_nt_acc(dk, gw, w + H * gw, gw, dx + r * M * H, H, M, gw, H);
      orc_matmul_nt_acc(dv, gw, w + 2 * H * gw, gw, dx + r * M * H, H, M, gw, H);
    }
    if (s + 1 < n) rotate_ccw_weight_grad(slots, n);
  }
#undef TAPE
  for (size_t r = 0; r < n; ++r) memcpy(grads + r * L, slots[r].grad, L * sizeof(double));
  free(qbh); free(kbh); free(vbh); free(dobh); free(obh); free(sc); free(dprobs); free(ds);
  free(t1); free(t2); free(t3); free(da); free(dq); free(dk); free(dv);
  free(tape);
  free(slots);
  free(store);
  return 0;
}

void orc_sampled_dots(const double* a, size_t lda, size_t sa, const double* b, size_t ldb,
                      size_t sb, size_t k, const int64_t* ri, const int64_t* ci, size_t nq,
                      double* out) {
#pragma omp parallel for schedule(static)
  for (size_t q = 0; q < nq; ++q) {
    const double* ap = a + (size_t)ri[q] * lda;
    const double* bp = b + (size_t)ci[q] * ldb;
    double acc = 0.0;
    for (size_t t = 0; t < k; ++t) acc += ap[t * sa] * bp[t * sb];
    out[q] = acc;
  }
}

uint64_t orc_rtp_memory(uint64_t W, uint64_t G, uint64_t N, int outofplace) {
  const uint64_t mx = W > G ? W : G;
  if (N <= 1) return W + G; /* analysis.cpp:37 */
  return (W + G + (outofplace ? mx : 0)) / N;
}
