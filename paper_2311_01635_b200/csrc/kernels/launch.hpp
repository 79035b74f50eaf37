// Internal launcher interface shared by the kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../../include/rtpb.h"

namespace rtpb {

// Thread-local error slot behind rtpb_last_error(); returns `code`.
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
// Counts kernel launches issued by this library (bench.py's gpu_launches).
void count_launch(uint64_t n = 1);

struct StepFwd {
  const void* x; const void* x_lo; size_t ldx;
  const void* w; const void* w_lo;  // I x per block of the shard
  const void* bias;                 // per values (dtype)
  void* y; size_t ldy; size_t col0; // pre / Y output (EF_STORE_PRE)
  void* act; size_t ld_act;         // gelu(pre) output (EF_GELU)
  size_t M, I, per;
  int flags;
  int force_bn;
};

struct StepDgrad {
  const void* dy; const void* dy_lo; size_t ldy;  // dy points at the column block
  const void* w; const void* w_lo;
  const void* dy2; const void* w2;  // optional second (column block, shard): bf16, same per
  float* acc; size_t ld_acc;
  void* dx; size_t ldx;
  const void* pre; size_t ldpre;
  size_t M, I, per;
  int flags;
  int force_bn;
};

struct StepWgrad {
  const void* x; const void* x_lo; size_t ldx;
  const void* dy; const void* dy_lo; size_t ldy;  // dy points at the column block
  const float* g_in; float* g_out;                // I x per block of the grad shard
  unsigned* split_flags;                          // zeroed per-tile counters (split-K order)
  const float* gbias_in; float* gbias_out;        // bias gradient, when the GEMM fuses it
  float* bias_part; unsigned* bias_tick;          // its partial sums / zeroed arrival counters
  float* wpart;                                   // split-K fp32 partials (nullable: ordered split-K)
  size_t M, I, per;
  int force_bn;
};
// K splits the dW launch uses on the whole machine (1: none) and the fp32
// partial floats its workspace needs for them (splits x I rounded to 256 x per).
int wgrad_splits(bool f32, size_t M, size_t I, size_t per, int force_bn);
size_t wgrad_partial_floats(bool f32, size_t M, size_t I, size_t per);
// True when gemm_wgrad runs a CTA-pair config, whose extra warp also sums dY
// columns into the bias gradient (gbias_*); otherwise colsum_bias_grad does.
bool wgrad_fuses_bias(bool f32, size_t M, size_t I, size_t per, unsigned* split_flags, int force_bn);

int gemm_fwd(bool f32, const StepFwd& p, cudaStream_t s);
// Pass launches (bf16): every rotation step of one layer pass in one
// persistent launch (GemmArgs::pass_steps). p.w = buffer 0's shard block,
// w1 = buffer 1's; *done_target: the per-step count-in total on pa.done.
struct PassArgs {
  int steps;
  unsigned buf_mask;         // bit s: step s reads buffer 1
  const int* cols;           // [steps] column block offsets (elements)
  const unsigned* ready;     // [steps] arrival flags (nullable)
  unsigned* done;            // [steps] zeroed count-in counters (nullable)
  unsigned* reset_ctr;       // zeroed CTA counter: the launch re-zeroes ready / done (nullable)
  int pair = 0;              // DGRAD: units over step pairs (GemmArgs::pass_pair)
};
unsigned pass_done_target(bool dgrad, size_t M, size_t N, bool gelu, int force, int groups);
int gemm_fwd_pass(const StepFwd& p, const void* w1, size_t y_cols, const PassArgs& pa, cudaStream_t s,
                  unsigned* done_target);
int gemm_dgrad_pass(const StepDgrad& p, const void* w1, size_t dy_cols, const PassArgs& pa, cudaStream_t s,
                    unsigned* done_target);
// p.dy = the whole dY (dy_cols wide), p.g_out = the travelling gradient
// shard [W | b]; db (nullable): dY's column sums (dy_cols floats), added to
// the bias part at each step; g_zero: the shard is known zero at step 0.
int gemm_wgrad_pass(const StepWgrad& p, size_t dy_cols, bool g_zero, const float* db, const PassArgs& pa,
                    cudaStream_t s, unsigned* done_target);
unsigned wgrad_pass_done_target(size_t M, size_t I, size_t per, int force);
// Fused N = 1 MLP forward (ffn1 + GELU and ffn2 in one scheduled launch).
struct FusedFwdPlan {
  std::vector<int> sched;  // [slots + 1 offsets][unit codes], uploaded by the caller
  int slots = 0;           // CTA pairs the schedule is built for
  int dep_rows = 0;        // row-block counters (zeroed device memory, self-resetting)
  unsigned dep_target = 0;
  int k_splits2 = 1;       // ffn2 K splits (> 1: fp32 partials in acc2, ordered)
  int tiles2 = 0;          // ffn2 tiles (split counters)
  double est_us = 0;       // cost-model makespan
};
// Device workspace of the fused forward: zero-filled once, then self-resetting.
struct FusedFwdWs {
  const int* sched;
  unsigned* dep_count;     // [dep_rows]
  unsigned* done_ctas;     // [1]
  unsigned* split_flags2;  // [tiles2]
  float* acc2;             // M x h fp32 (k_splits2 > 1)
};
bool plan_fused_fwd(size_t M, size_t h, size_t f, FusedFwdPlan& plan);
int gemm_fwd_fused(const StepFwd& p0, const StepFwd& p1, const FusedFwdPlan& plan, const FusedFwdWs& ws,
                   cudaStream_t s);

// Fused N = 1 MLP backward: D (dX chain) and W (dW pair) launches.
struct FusedBwdPlan {
  std::vector<int> sched_d, sched_w;  // [slots + 1 offsets][unit codes] each
  int slots_d = 0, slots_w = 0;       // CTA pairs of D and W (together <= SMs / 2)
  int w_splits = 1;                   // dW K splits (ordered, deterministic)
  int dep_rows = 0;
  unsigned dep_target = 0;
  double est_us = 0;
};
struct FusedBwdWs {
  const int* sched_d;
  const int* sched_w;
  unsigned* dep_count;  // [dep_rows], zeroed once, self-resetting
  unsigned* done_ctas;  // [1]
};
struct FusedBwdArgs {
  const void* dy; size_t ldy;   // M x h upstream gradient
  const void* act;              // M x f gelu(pre): ffn2's input
  const void* x; size_t ldx;    // M x h block input: ffn1's input
  void* pre;                    // M x f: pre in, dpre out (in place)
  void* dx; size_t lddx;        // M x h output
  const void* w1; const void* w2;  // shards [W | b] (bf16)
  float* g1; float* g2;         // gradient shards (fp32)
  bool g1_zero, g2_zero;        // known-zero gradients: store instead of accumulate
  float* bias_part1; unsigned* bias_tick1;  // per-layer workspace parts (zeroed counters)
  float* bias_part2; unsigned* bias_tick2;
  unsigned* split_flags1; unsigned* split_flags2;
  float* wpart1; float* wpart2;  // split-K partial buffers of the layers (nullable)
  size_t M, h, f;
  bool exact_gelu;  // RTPB_EPI_EXACT_GELU in ffn2's dX epilogue
};
bool plan_fused_bwd(size_t M, size_t h, size_t f, FusedBwdPlan& plan);
int gemm_bwd_fused(const FusedBwdArgs& a, const FusedBwdPlan& plan, const FusedBwdWs& ws, cudaStream_t compute,
                   cudaStream_t aux);
int fused_bwd_step(FusedBwdArgs a, void* ws1, size_t ws1_bytes, void* ws2, size_t ws2_bytes,
                   const FusedBwdPlan& plan, const FusedBwdWs& ws, cudaStream_t compute, cudaStream_t aux);

// The fused forward as a step (capi_steps.cu): bf16, shards [W | b];
// store_pre: also write pre (Train). Timed as one fwd launch when profiling.
int fused_fwd_step(const void* x, size_t ldx, const void* w1_shard, void* pre, void* act, const void* w2_shard,
                   void* y, size_t ldy, size_t M, size_t h, size_t f, bool store_pre, const FusedFwdPlan& plan,
                   const FusedFwdWs& ws, cudaStream_t s, bool exact_gelu = false);

// Caps the SMs the calling thread's following GEMM launches occupy (0 = all);
// sm_budget() returns the effective count.
// Load every device kernel of the library on the current device now. Under
// CUDA's lazy module loading (the default), the first launch of a kernel
// loads it, and a load may wait for the device's running work — which
// deadlocks once a running grid spins on an arrival flag that work queued
// behind the load would raise (pass launches, flag waits). Called once per
// device by every Worker.
void preload_device_kernels();

void set_sm_budget(int sms);
// Programmatic (PDL) launch overlap between consecutive step GEMMs (default on).
void set_pdl_enabled(bool on);
int sm_budget();
// The calling thread's following GEMM launches load no operand before
// *flag >= 1 (nullptr: no wait). See GemmArgs::ready_flag.
void set_launch_wait_flag(const unsigned* flag);
// The next dW launch of this thread: its epilogue (not its mainloop) waits
// for the travelling gradient's arrival flag (GemmArgs::g_flag).
void set_launch_g_flag(const unsigned* flag);
// The calling thread's next step-GEMM launch clears [flags, +count) (and the
// CTA counter ctr) when all its CTAs are done; nullptr = none.
void set_launch_flag_reset(unsigned* flags, int count, unsigned* ctr);
// Debug: route per-CTA timeline stamps of the following GEMM launches into buf.
void set_trace(void* buf, size_t bytes);
int gemm_dgrad(bool f32, const StepDgrad& p, cudaStream_t s);
int gemm_wgrad(bool f32, const StepWgrad& p, cudaStream_t s);

// elementwise.cu
int flyweight_init(void* dst, bool f32, uint64_t seed, uint64_t base, size_t I, size_t O, size_t n, size_t j,
                   double lo, double hi, cudaStream_t s);
size_t colsum_workspace_bytes(size_t M, size_t per);
int colsum_bias_grad(bool f32, const void* dy, size_t ldy, size_t M, size_t per, const float* g_in,
                     float* g_out, void* ws, cudaStream_t s);
int tf32_split(const float* src, size_t rows, size_t cols, size_t ld, float* hi, float* lo, cudaStream_t s);
// Split and transpose: hi/lo are cols x rows, row stride round_up(rows, 8).
int tf32_split_t(const float* src, size_t rows, size_t cols, size_t ld, float* hi, float* lo, cudaStream_t s);
int gelu_fwd(bool f32, const void* x, void* y, size_t count, cudaStream_t s);
int gelu_bwd(bool f32, const void* x, const void* up, void* out, size_t count, cudaStream_t s);
int cast_f32_to_bf16(const float* src, void* dst, size_t count, cudaStream_t s);
// attention.cu: the attention core of one head group (rows = batch * seq,
// q/k/v/o rows x g*hd; lse / delta rows x g fp32).
int attention_core_fwd(bool f32, const void* q, const void* k, const void* v, void* o, float* lse, size_t rows,
                       size_t seq, size_t g, size_t hd, float scale, cudaStream_t s);
int attention_core_bwd(bool f32, const void* q, const void* k, const void* v, const void* o, const float* lse,
                       const void* dout, void* dq, void* dk, void* dv, float* delta, size_t rows, size_t seq,
                       size_t g, size_t hd, float scale, cudaStream_t s);
// moe_embed.cu: RtpMoe routing / combine and RtpEmbedding gather / scatter.
int moe_gate(bool f32, const void* x, size_t rows, size_t H, const double* gate, size_t n, double* probs, int* sel,
             cudaStream_t s);
int gather_rows(bool f32, const void* src, size_t lds, const int* idx, size_t cnt, size_t cols, void* dst,
                cudaStream_t s);
int moe_combine(bool f32, const void* eout, const int* pos, const int* sel, const double* probs, size_t n, size_t rows,
                size_t H, void* y, size_t ldy, cudaStream_t s);
int moe_route_bwd(bool f32, const void* dy, size_t ldy, const void* eout, const int* rows_j, size_t cnt, size_t j,
                  const double* probs, size_t n, size_t H, void* de, double* dlogits, cudaStream_t s);
int moe_dx(bool f32, const void* dxs, const int* pos, const double* dlogits, const double* gate, size_t n, size_t rows,
           size_t H, void* dx, size_t ldx, cudaStream_t s);
int moe_gate_grad(bool f32, const void* x, size_t ldx, const double* dlogits, size_t n, size_t rows, size_t H,
                  double* gg, bool accumulate, cudaStream_t s);
int embed_gather(bool f32, const void* block, size_t per, const int64_t* ids, size_t cnt, void* y, size_t ldy,
                 size_t col0, cudaStream_t s);
int embed_scatter(bool f32, const void* dy, size_t ldy, size_t col0, const int64_t* uniq, const int* offs,
                  const int* toks, size_t nuniq, size_t per, float* grad, cudaStream_t s);
// dtype codes RTPB_BF16 / RTPB_F32 / RTPB_F64
int convert(const void* src, int src_dtype, void* dst, int dst_dtype, size_t count, cudaStream_t s);
int fill(void* dst, int dtype, size_t count, double v, cudaStream_t s);
// out = a + b elementwise (residual connections, model.cpp:72,85,108,111)
int add(const void* a, const void* b, void* out, int dtype, size_t count, cudaStream_t s);

}  // namespace rtpb
