/* oracle/rtp_oracle.h — TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * Plain-C fp64 restatement of the reference's RTP linear/MLP path
 * (/root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never does. Every function
 * cites the reference file:line it restates. Parity of this restatement is
 * PINNED against the reference itself: tests/golden/*.npz are produced by
 * tests/golden/make_golden.py from oracle/_ref/librtpref.so (the reference
 * sources compiled by path) and tests/test_oracle.py requires bit-equality.
 */
#ifndef RTP_ORACLE_H
#define RTP_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64 (rng.hpp:10-32) in counter form: the k-th (0-based) next_u64()
 * of a stream seeded with `seed`. */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t k);
/* next_uniform(lo, hi) of draw k (rng.hpp:25-27, tensor.cpp:99-103). */
double orc_uniform_at(uint64_t seed, uint64_t k, double lo, double hi);
void orc_uniform(uint64_t seed, uint64_t skip, uint64_t count, double lo, double hi, double* out);

/* Flyweight closed form of shard j of a linear I->O whose weight (I x O,
 * row-major) is drawn starting at stream index `base` and whose bias (O)
 * follows it: [W[:, j*per:(j+1)*per] row-major | b[j*per:(j+1)*per]]
 * (serial.cpp:329-353 draw order; layers_common.cpp:33-45 + partition.cpp:15-56
 * shard layout). out has I*per + per doubles. */
void orc_linear_shard(uint64_t seed, uint64_t base, size_t I, size_t O, size_t n, size_t j,
                      double* out);

/* Reference kernel arithmetic order (kernels_scalar.cpp:6-56), no FMA. */
void orc_matmul(const double* a, size_t lda, const double* b, size_t ldb, double* c, size_t ldc,
                size_t m, size_t k, size_t n);
void orc_matmul_tn_acc(const double* a, size_t lda, const double* b, size_t ldb, double* c,
                       size_t ldc, size_t m, size_t k, size_t n);
void orc_matmul_nt_acc(const double* a, size_t lda, const double* b, size_t ldb, double* c,
                       size_t ldc, size_t m, size_t k, size_t n);

/* Exact-erf GELU and its derivative (tensor.cpp:323-351). */
void orc_gelu(const double* x, double* y, size_t count);
void orc_gelu_backward(const double* x, const double* up, double* out, size_t count);

/* RtpLinear Train forward + backward over n simulated workers
 * (layers_linear.cpp:18-72; rotation ring.cpp:265-293), batch-major rows
 * (model.cpp:165-178). w: I x O, b: O, x: rows x I, dy: rows x O.
 * Outputs: y (rows x O), dx (rows x I), grads (n * (I*per+per), the grad_acc
 * resident at each rank after backward, accumulated from zero).
 * trace (optional, 2*n*n int64): logical id held by rank r at forward step s
 * (trace[s*n+r]) then at backward step s (trace[n*n + s*n + r]).
 * Returns 0, or 2 (ConfigError: O % n or rows % n != 0). */
int orc_rtp_linear(size_t n, size_t rows, size_t I, size_t O, const double* w, const double* b,
                   const double* x, const double* dy, double* y, double* dx, double* grads,
                   int64_t* trace);

/* The FFN block as RtpModel composes it (model.cpp:77-83, 99-105):
 * pre = ffn1(x); y = ffn2(gelu(pre)); dh = ffn2'(dy); dpre = gelu'(pre, dh);
 * dx = ffn1'(dpre). grads1/grads2: n * shard_len of each layer. */
int orc_rtp_mlp(size_t n, size_t rows, size_t h, size_t f, const double* w1, const double* b1,
                const double* w2, const double* b2, const double* x, const double* dy, double* y,
                double* dx, double* grads1, double* grads2);

/* Sampled fp64 dot products for large configs (SURVEY §8c "spot-check"):
 * out[q] = sum_t a[ri[q]*lda + t*sa] * b[t*sb + ci[q]*ldb] over t < k, t ascending.
 * Covers Y = X.W (sa=1, sb=ldw, ldb=1), dX = dY.W^T and dW = X^T.dY via strides. */
/* RtpAttention fwd (Train) + bwd (layers_attention.cpp:43-198), heads split
 * across n workers (HeadPartition), batch-major row shards of `rows` (each a
 * multiple of seq); grads = n shards of [gq | gk | gv | go] (4 H gw each). */
int orc_rtp_attention(size_t n, size_t rows, size_t H, size_t heads, size_t seq, const double* wq,
                      const double* wk, const double* wv, const double* wo, const double* x,
                      const double* dy, double* y, double* dx, double* grads);

void orc_sampled_dots(const double* a, size_t lda, size_t sa, const double* b, size_t ldb,
                      size_t sb, size_t k, const int64_t* ri, const int64_t* ci, size_t nq,
                      double* out);

/* RTP memory model (analysis.cpp:45-46 rows / N): in-place (W+G)/N,
 * out-of-place (W+G+max(W,G))/N, bytes per worker. */
uint64_t orc_rtp_memory(uint64_t W, uint64_t G, uint64_t N, int outofplace);

#ifdef __cplusplus
}
#endif
#endif
