/* rtpb.h — C ABI of the B200-native RTP (Rotated Tensor Parallelism) hot path.
 *
 * Plain pointers and sizes only; no torch types. Two layers:
 *
 *  (1) Step kernels: the device replacement for the reference's op plug-in
 *      point, the rtp::kern::Kernels table (proj/include/rtp/kernels.hpp:17-47,
 *      dispatched through kern::active(), proj/src/kernels.cpp:23-27). One call
 *      = one rotation step of one RtpLinear on one worker, asynchronous on the
 *      given cudaStream_t. No allocation, no host sync.
 *
 *  (2) Group / layer handles: the reference's host API
 *      (WorkerGroup proj/include/rtp/ring.hpp:65-125, RtpLinear
 *      proj/include/rtp/layers.hpp:129-147, the ffn1->gelu->ffn2 block of
 *      proj/src/model.cpp:77-83,99-105) over device shards. The C++ classes in
 *      include/rtpb/rtp.hpp implement it; these functions expose them to
 *      FFI callers (ctypes in paper_2311_01635_b200/_lib.py).
 *
 * Errors: every function returns RTPB_OK (0) or one of the codes below, which
 * mirror the reference's exception taxonomy (proj/include/rtp/errors.hpp:8-33);
 * rtpb_last_error() returns the thread-local message.
 *
 * Device dtypes: RTPB_BF16 (bf16 operands, fp32 accumulation) or RTPB_F32
 * (fp32 operands, 3xTF32 tensor-core products). Gradient shards are fp32.
 * Alignment: operand base pointers 16-byte aligned, row strides multiples of
 * 16 bytes (in_dim, out_dim/N multiples of 8) — RTPB_ERR_CONFIG otherwise.
 */
#ifndef RTPB_H
#define RTPB_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTPB_OK 0
#define RTPB_ERR_GENERIC 1
#define RTPB_ERR_CONFIG 2    /* rtp::ConfigError    */
#define RTPB_ERR_DIMENSION 3 /* rtp::DimensionError */
#define RTPB_ERR_PROTOCOL 4  /* rtp::ProtocolError  */
#define RTPB_ERR_STATE 5     /* rtp::StateError     */
#define RTPB_ERR_INDEX 6     /* rtp::IndexError     */
#define RTPB_ERR_CUDA 7
#define RTPB_ERR_NCCL 8

#define RTPB_BF16 0
#define RTPB_F32 1
#define RTPB_F64 2 /* host-API tensors and rtpb_convert only; the step kernels take BF16 / F32 */

/* Step-kernel epilogue flags (rtpb_fwd_step / rtpb_dgrad_step). */
#define RTPB_EPI_GELU 1      /* fwd: also write gelu(pre) to `act` (model.cpp:80)       */
#define RTPB_EPI_FIRST 2     /* dgrad: first step, overwrite the fp32 accumulator        */
#define RTPB_EPI_LAST 4      /* dgrad: last step, emit dX in the activation dtype        */
#define RTPB_EPI_GELU_BWD 8  /* dgrad last step: dX *= gelu'(pre) (model.cpp:101-104)   */
#define RTPB_EPI_STORE_PRE 16 /* fwd: write X.W_j + b_j to `y` (default for plain linear) */
#define RTPB_EPI_NO_BIAS 32   /* fwd / wgrad_ex: the shard block has no bias part (projections) */
#define RTPB_EPI_EXACT_GELU 64 /* bf16: exact-erf GELU / GELU' in the epilogue (default: tanh.approx form) */
#define RTPB_PASS_PAIR 128    /* rtpb_dgrad_pass: each unit covers a step pair (2g, 2g+1), one accumulation over
                                 K = 2 per (paired dX); counters and the done target per pair */

const char* rtpb_last_error(void);
/* Load every kernel of the library on the current device now (groups do it
 * for their devices). Under CUDA's lazy loading a kernel is loaded at its
 * first launch, and a load may wait for running work: a caller that queues
 * waits on a kernel's progress (stream memory operations on pass-launch
 * counters) before that kernel's first launch must preload. */
void rtpb_preload_kernels(void);
const char* rtpb_version(void);
/* Number of device kernels this library has launched (all threads). */
uint64_t rtpb_launch_count(void);

/* ------------------------------------------------------------------ */
/* (1) Step kernels                                                    */
/* ------------------------------------------------------------------ */

/* Flyweight shard initialisation (replaces Tensor::uniform + split +
 * shard_view: serial.cpp:329-353, tensor.cpp:99-103, layers_common.cpp:33-45,
 * partition.cpp:49-56). Writes shard j of a linear I->O whose weight draws
 * start at SplitMix64 stream index `stream_base`:
 *   dst[i*per + c]   = U(stream_base + i*O + j*per + c)
 *   dst[I*per + c]   = U(stream_base + I*O + j*per + c)          (bias)
 * with U(k) = lo + (hi-lo)*((splitmix64(seed, k) >> 11) * 2^-53) evaluated in
 * fp64 without contraction, then rounded to nearest into `dtype`. */
int rtpb_flyweight_init(void* dst, int dtype, uint64_t seed, uint64_t stream_base, size_t I, size_t O,
                        size_t n, size_t j, double lo, double hi, void* stream);

/* Forward step (layers_linear.cpp:29-37): for the shard w_shard = [W_j | b_j]
 *   pre = X . W_j + b_j   (M x per)
 *   y[:, col0 : col0+per]   = pre          if flags & RTPB_EPI_STORE_PRE
 *   act[:, col0 : col0+per] = gelu(pre)    if flags & RTPB_EPI_GELU
 * X: M x I (row stride ldx). Workspace: rtpb_step_workspace_bytes(0, ...). */
int rtpb_fwd_step(int dtype, const void* x, size_t ldx, const void* w_shard, void* y, size_t ldy, size_t col0,
                  void* act, size_t ld_act, size_t M, size_t I, size_t per, int flags, void* workspace,
                  size_t workspace_bytes, void* stream);

/* dX step (layers_linear.cpp:65, kern::matmul_nt_acc):
 *   acc (+)= dY[:, col0:col0+per] . W_j^T     (fp32 accumulator, M x I, ld_acc)
 * RTPB_EPI_FIRST: acc is overwritten instead of read. RTPB_EPI_LAST: the sum
 * is written to dx (dtype, ldx) instead of acc, multiplied by gelu'(pre) when
 * RTPB_EPI_GELU_BWD. FIRST|LAST (N = 1) never touches acc. */
int rtpb_dgrad_step(int dtype, const void* dy, size_t ldy, size_t col0, const void* w_shard, float* acc,
                    size_t ld_acc, void* dx, size_t ldx, const void* pre, size_t ldpre, size_t M, size_t I,
                    size_t per, int flags, void* workspace, size_t workspace_bytes, void* stream);

/* Two dX steps in one pass (layers_linear.cpp:65 for two consecutive steps;
 * bf16; two weight shards resident, out-of-place mode):
 * acc (+)= dY[:, col0:+per] . W_a^T + dY[:, col1:+per] . W_b^T, one
 * fp32 accumulation over K = 2 per; flags as rtpb_dgrad_step. Halves the
 * cross-step accumulator passes (RTPB_DX_PAIR in the layers). */
int rtpb_dgrad_step2(int dtype, const void* dy, size_t ldy, size_t col0, const void* w_a, size_t col1,
                     const void* w_b, float* acc, size_t ld_acc, void* dx, size_t ldx, const void* pre,
                     size_t ldpre, size_t M, size_t I, size_t per, int flags, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Pass launches (bf16, one worker per GPU, out-of-place mode): every rotation
 * step of one layer pass (layers_linear.cpp:29-43 forward, :57-67 dX) in ONE
 * persistent launch instead of one launch per step. Step s (0 <= s < steps)
 * computes on the weight shard in buffer (buf_mask >> s) & 1 (buf0 = the
 * resident shard at pass start, buf1 = the spare; they alternate) and on the
 * activation column block col0[s] (= j_s * per):
 *   fwd  : y / act[:, col0[s] : +per] = (gelu)(X . W_{j_s} + b_{j_s})   (flags as rtpb_fwd_step)
 *   dgrad: dX = sum_s dY[:, col0[s] : +per] . W_{j_s}^T, accumulated in the
 *          fp32 `acc` in step order (bit-identical to `steps` rtpb_dgrad_step
 *          calls), times gelu'(pre) with RTPB_EPI_GELU_BWD.
 * `ready` (nullable): step s >= 1 reads its shard only once ready[s] >= 1
 * (written by the comm stream when the shard landed). `done` (steps zeroed
 * counters): once step s's operands have been read, done[s] reaches
 * *done_target (written by the call; with RTPB_PASS_PAIR done[g] counts the
 * pair (2g, 2g + 1)); a nonzero *done_target on entry is the target the
 * caller announced (rtpb_pass_done_target): the call fails without
 * launching if the launch would count to another — the comm stream waits for that value
 * (cuStreamWaitValue32) before it lands step s + 2's shard in step s's
 * buffer. The launch re-zeroes `done` (and, with reset_flags, the `ready`
 * range) when it completes; reset_ctr is a zeroed counter. y_cols / dy_cols:
 * width of the Y / dY activations (N * per). Requires per % 32 == 0 and
 * steps <= 16. */
/* The count-in total a pass launch of this geometry reaches on done[s]
 * (which = 0 fwd, 1 dgrad, 2 wgrad; steps and flags as the launch's), for
 * comm-stream waits enqueued before the launch. */
unsigned rtpb_pass_done_target(int which, size_t M, size_t I, size_t per, size_t steps, int flags);
int rtpb_fwd_pass(const void* x, size_t ldx, const void* buf0, const void* buf1, void* y, size_t ldy, void* act,
                  size_t ld_act, size_t y_cols, const size_t* col0, unsigned buf_mask, size_t steps, size_t M,
                  size_t I, size_t per, int flags, const unsigned* ready, unsigned* done, unsigned* done_target,
                  unsigned* reset_ctr, void* stream);
int rtpb_dgrad_pass(const void* dy, size_t ldy, size_t dy_cols, const void* buf0, const void* buf1,
                    const size_t* col0, unsigned buf_mask, size_t steps, float* acc, size_t ld_acc, void* dx,
                    size_t ldx, const void* pre, size_t ldpre, size_t M, size_t I, size_t per, int flags,
                    const unsigned* ready, unsigned* done, unsigned* done_target, unsigned* reset_ctr,
                    void* stream);

/* dW of every step of a pass into the travelling gradient shard g = [W | b]
 * (fp32) in ONE persistent launch:
 *   step s: g[0 : I*per] += X^T . dY[:, col0[s] : +per]   (RTPB_EPI_FIRST in
 *           flags: g known zero at step 0, stored instead of accumulated)
 *           g[I*per : +per] += db[col0[s] : +per]          (db nullable: dY's
 *           column sums, rtpb_colsum)
 * The mainloops run ahead; each step's accumulation waits for ready[s] >= 1
 * (s >= 1: the comm stream's flag that G(s) landed) and counts in on done[s]
 * once its updates of g have landed (*done_target per step, also from
 * rtpb_pass_done_target(2, ...)): the comm stream then sends g on. Workspace:
 * rtpb_step_workspace_bytes(2, BF16, M, I, per), zeroed once. bf16 only. */
int rtpb_wgrad_pass(const void* x, size_t ldx, const void* dy, size_t ldy, size_t dy_cols, float* g,
                    const size_t* col0, size_t steps, size_t M, size_t I, size_t per, int flags, const float* db,
                    const unsigned* ready, unsigned* done, unsigned* done_target, unsigned* reset_ctr,
                    void* workspace, size_t workspace_bytes, void* stream);
/* out[c] = sum over the M rows of dy[:, c] (bf16 in, fp32 out; fixed order,
 * deterministic). Workspace: rtpb_colsum_workspace_bytes(M, cols), zeroed once. */
size_t rtpb_colsum_workspace_bytes(size_t M, size_t cols);
int rtpb_colsum(const void* dy, size_t ldy, size_t M, size_t cols, float* out, void* workspace, size_t workspace_bytes,
                void* stream);

/* dW step with the travelling-gradient accumulation fused into the epilogue
 * (layers_linear.cpp:61-63, kern::matmul_tn_acc + bias column sums):
 *   g_out[0 : I*per]      = g_in[0 : I*per] + X^T . dY[:, col0:col0+per]
 *   g_out[I*per : +per]   = g_in[I*per : +per] + colsum(dY[:, col0:col0+per])
 * g_in may equal g_out (in-place accumulation), or be NULL when the gradient
 * is known to be zero (the reference's zero_grads): then g_out = X^T . dY
 * (+ colsum) is written without reading anything. */
int rtpb_wgrad_step(int dtype, const void* x, size_t ldx, const void* dy, size_t ldy, size_t col0,
                    const float* g_in, float* g_out, size_t M, size_t I, size_t per, void* workspace,
                    size_t workspace_bytes, void* stream);

/* rtpb_wgrad_step with epilogue flags: RTPB_EPI_NO_BIAS computes only
 * g_out[0 : I*per] (= g_in + X^T . dY block), for bias-free projection blocks
 * (RtpAttention: layers_attention.cpp:136-137, :164-166). */
int rtpb_wgrad_step_ex(int dtype, const void* x, size_t ldx, const void* dy, size_t ldy, size_t col0,
                       const float* g_in, float* g_out, size_t M, size_t I, size_t per, int epi_flags,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes for a step kernel: which = 0 fwd, 1 dgrad, 2 wgrad.
 * A workspace must be zero-filled before its first use; the kernels leave
 * their completion tickets at zero, so it can then be reused indefinitely
 * (by one stream at a time). */
size_t rtpb_step_workspace_bytes(int which, int dtype, size_t M, size_t I, size_t per);

/* Exact-erf GELU and derivative (tensor.cpp:323-351), elementwise. */
int rtpb_gelu(int dtype, const void* x, void* y, size_t count, void* stream);
/* Elementwise dtype conversion dst[i] = (dst_dtype) src[i], one rounding (RN)
 * from the value read; fill sets every element to v. The device half of
 * rtpb::Tensor's conversions (the reference's Tensor is fp64, tensor.hpp). */
int rtpb_convert(const void* src, int src_dtype, void* dst, int dst_dtype, size_t count, void* stream);
int rtpb_fill(void* dst, int dtype, size_t count, double v, void* stream);
/* out = a + b elementwise (the model's residual connections, model.cpp:72,85). */
int rtpb_add(int dtype, const void* a, const void* b, void* out, size_t count, void* stream);
int rtpb_gelu_backward(int dtype, const void* x, const void* upstream, void* out, size_t count, void* stream);

/* Per-launch timing of the step GEMMs: when enabled, a CUDA event pair is
 * recorded on the launching stream around every step GEMM. profile_read
 * returns the record count; with cap > 0 it fills (each array nullable) kind
 * (0 fwd, 1 dgrad, 2 wgrad), algorithmic flops, duration in ms, start in ms
 * after the first record's start, and the SMs the launch was sized for, then
 * clears the records. */
void rtpb_profile_enable(int on);
size_t rtpb_profile_read(int* kinds, double* flops, float* ms, float* start_ms, int* sms, size_t cap);

/* The calling thread's following step-kernel launches occupy at most `sms`
 * SMs (persistent grid, tile and split-K choice sized for them); 0 = all.
 * Lets a caller run two step GEMMs side by side on two streams. */
void rtpb_set_sm_budget(int sms);

/* Debug: cost-model makespan (us) of the fused N = 1 MLP schedule for rows M,
 * hidden h, ffn f: which 0 = forward, 1 = backward (-1 if no plan). */
double rtpb_debug_fused_plan(size_t M, size_t h, size_t f, int which);

/* Test hook: force the GEMM tile width (0 = heuristic; 64/128/256). */
void rtpb_debug_force_bn(int bn);
/* Debug hook: the following step-GEMM launches write per-CTA %globaltimer
 * stamps (80 u64 per CTA, layout in gemm_sm100.cuh GemmArgs::trace) into
 * consecutive blocks of this device buffer until it is full; NULL disables. */
void rtpb_debug_trace(void* device_buf, size_t bytes);

/* Measurement hook: while on, every ring shift of every group keeps its
 * schedule, events and bookkeeping but moves no bytes — the compute-only
 * baseline from which bench.py derives the exposed rotation time. Results
 * are wrong while it is on. */
void rtpb_debug_skip_comm(int on);

/* Ring schedule of an RtpLinear pass, pure host logic shared by every
 * transport: the logical shard id `rank` holds at (phase, step) — forward
 * (phase 0) (rank - step) mod n, backward (phase 1) (rank + 1 + step) mod n
 * (layers_common.cpp:135-151) — and the peers of the rotation that follows
 * that step (clockwise forward, counter-clockwise backward; ring.cpp:265-293).
 * send_to / recv_from are -1 after the last step. */
int rtpb_ring_plan(size_t n, size_t rank, int phase, size_t step, int64_t* logical_id, int64_t* send_to,
                   int64_t* recv_from);

/* ------------------------------------------------------------------ */
/* (2) Group / layer handles                                           */
/* ------------------------------------------------------------------ */

typedef struct rtpb_group_s* rtpb_group;
typedef struct rtpb_linear_s* rtpb_linear;
typedef struct rtpb_mlp_s* rtpb_mlp;
typedef struct rtpb_attention_s* rtpb_attention;
typedef struct rtpb_embedding_s* rtpb_embedding;
typedef struct rtpb_moe_s* rtpb_moe;
typedef struct rtpb_model_s* rtpb_model;

#define RTPB_TRANSPORT_LOCKSTEP 0   /* one host thread drives all local workers        */
#define RTPB_TRANSPORT_CONCURRENT 1 /* one host thread per local worker                */
#define RTPB_TRANSPORT_NCCL 2       /* one process per GPU, ncclSend/ncclRecv on NVLink */
#define RTPB_TRANSPORT_IPC 3        /* one process per GPU, copy-engine pushes via CUDA IPC */

#define RTPB_MODE_TRAIN 0
#define RTPB_MODE_EVAL 1
#define RTPB_ROT_INPLACE 0
#define RTPB_ROT_OUTOFPLACE 1

/* Memory ledger categories (ledger.hpp:10). */
#define RTPB_MEM_PARAM 0
#define RTPB_MEM_GRAD 1
#define RTPB_MEM_ACTIVATION 2
#define RTPB_MEM_COMMBUFFER 3
#define RTPB_MEM_OTHER 4

/* WorkerGroup(n, kind) with all n workers in this process; devices[r] is the
 * CUDA device of worker r (several workers may share one device: the ring
 * exchange is then a device-local copy, mirroring the Lockstep transport). */
int rtpb_group_create(size_t n, int transport, const int* devices, rtpb_group* out);
/* Distributed group: this process is worker `rank` of `n` on `device`; the
 * ring exchange is ncclSend/ncclRecv. nccl_id: 128 bytes from
 * rtpb_nccl_unique_id() on rank 0, broadcast by the caller. */
int rtpb_nccl_unique_id(void* out128);
int rtpb_group_create_nccl(size_t n, size_t rank, int device, const void* nccl_id, rtpb_group* out);
/* Distributed group on the IPC transport: the ring shift is a copy-engine
 * push into the neighbour's buffer through a CUDA IPC mapping (NVLink P2P,
 * or a device-local copy when workers share a GPU), ordered by stream memory
 * operations — no SMs used. Processes on one node; id: 128 bytes from
 * rtpb_ipc_unique_id() on rank 0, broadcast by the caller. Not capturable in
 * a CUDA graph (the flags carry per-shift sequence numbers). */
int rtpb_ipc_unique_id(void* out128);
int rtpb_group_create_ipc(size_t n, size_t rank, int device, const void* id, rtpb_group* out);
/* Measurement group: worker `rank` of an n-worker ring with no peers present;
 * every ring shift is skipped (schedule, events, bookkeeping unchanged), so one
 * GPU runs one rank's N-way step at its real shapes. Results are not the
 * model's (shards do not move). */
int rtpb_group_create_solo(size_t n, size_t rank, int device, rtpb_group* out);
int rtpb_group_destroy(rtpb_group g);
size_t rtpb_group_size(rtpb_group g);
/* Local worker ranks hosted by this process (count returned, ranks written). */
size_t rtpb_group_local_ranks(rtpb_group g, size_t* ranks);
/* Compute / comm stream of a local worker (cudaStream_t as void*), its device. */
void* rtpb_group_stream(rtpb_group g, size_t rank, int comm);
int rtpb_group_device(rtpb_group g, size_t rank);
int rtpb_group_synchronize(rtpb_group g);

/* Debug hook: copy `count` entries of a local worker's arrival-flag pool
 * (from index `first`) to host memory through a private stream (does not
 * wait for the worker's streams), and report which of its streams (bit 0
 * compute, 1 comm, 2 aux) still have work pending. The private stream is
 * made on the first call, on the device current then (call it once before
 * the work to watch starts); host_dst should be pinned memory. */
int rtpb_debug_read_flags(rtpb_group g, size_t rank, size_t first, size_t count, unsigned* host_dst,
                          int* busy_streams);
/* Debug hook: device address of entry `index` of a local worker's flag pool. */
uint64_t rtpb_debug_flag_address(rtpb_group g, size_t rank, size_t index);
/* Traffic log (ring.hpp:41-46): kind 0 rotation_cw, 1 rotation_ccw, 2 allgather. */
size_t rtpb_group_traffic(rtpb_group g, int64_t* kinds, int64_t* w_elems, int64_t* g_elems, size_t cap);
void rtpb_group_clear_traffic(rtpb_group g);
/* WorkerGroup::corrupt_next_exchange (ring.cpp:223-238): what 1 = Tag, 2 = ShardId. */
int rtpb_group_corrupt_next_exchange(rtpb_group g, size_t rank, int what);
/* Per-worker ledger (ledger.hpp:23-41): current/peak bytes per category, peak total. */
int rtpb_group_ledger(rtpb_group g, size_t rank, size_t* current5, size_t* peak5, size_t* peak_total);
int rtpb_group_reset_ledger_peaks(rtpb_group g);
/* Ring primitive on raw device slots (test / micro-bench entry, ring.cpp:265-333):
 * weight[r], grad[r]: device buffers of `w_bytes` / `g_bytes` for local rank r.
 * op: 0 cw(W), 1 ccw(W+G), 2 cw(W+G), 3 ccw(W); spare != NULL -> out-of-place W
 * (received into spare[r], then copied back into weight[r] unless op has
 * RTPB_ROTATE_KEEP_SPARE, in which case the caller swaps the two roles). */
#define RTPB_ROTATE_KEEP_SPARE 8
int rtpb_group_rotate(rtpb_group g, int op, void** weight, void** grad, void** spare, size_t w_bytes,
                      size_t g_bytes);
/* ring_allgather (ring.cpp:335-376) of `bytes` per rank into out (n*bytes). */
int rtpb_group_allgather(rtpb_group g, void** in, void** out, size_t bytes);

/* RtpLinear(group, label, weight, bias, n) (layers_linear.cpp:6-16): w (I x O)
 * and b (O) are fp64 host arrays as in the reference; pass w = b = NULL for
 * Flyweight initialisation from (seed, stream_base) instead — each worker's
 * shard is generated on its device, the full weight never exists. */
int rtpb_linear_create(rtpb_group g, const char* label, size_t in_dim, size_t out_dim, int dtype,
                       const double* w, const double* b, uint64_t seed, uint64_t stream_base, rtpb_linear* out);
int rtpb_linear_destroy(rtpb_linear l);
int rtpb_linear_set_rotation_mode(rtpb_linear l, int mode);
int rtpb_linear_allocate_comm_spares(rtpb_linear l);
int rtpb_linear_release_comm_spares(rtpb_linear l);
int rtpb_linear_zero_grads(rtpb_linear l);
size_t rtpb_linear_shard_len(rtpb_linear l);
/* forward(x, mode) / backward(dy) (layers_linear.cpp:18-72). x[k], y[k], dy[k],
 * dx[k]: device activations of the k-th local rank, `rows` rows each,
 * contiguous (ld = in_dim / out_dim). x must stay valid until backward. */
int rtpb_linear_forward(rtpb_linear l, const void* const* x, size_t rows, void* const* y, int mode);
int rtpb_linear_backward(rtpb_linear l, const void* const* dy, size_t rows, void* const* dx);
/* Slot state of local rank r: logical_id, rotation_offset, device pointers. */
int rtpb_linear_slot(rtpb_linear l, size_t rank, int64_t* logical_id, int64_t* rotation_offset, void** weight,
                     void** grad);
/* Per-(phase, step, rank) logical ids seen by the last forward/backward:
 * ids[phase*n*n + step*n + rank] (phase 0 fwd, 1 bwd), -1 where not local. */
int rtpb_linear_trace(rtpb_linear l, int64_t* ids);
/* Synchronous copy of the shard resident at local rank r into dst (device
 * memory): which 0 = weight [W_j | b_j] (layer dtype), 1 = grad_acc (fp32). */
int rtpb_linear_read_shard(rtpb_linear l, size_t rank, int which, void* dst);
/* Numerics options of a layer (and of both layers of an MLP):
 *  RTPB_OPT_EXACT_GELU (default 0): bf16 epilogues evaluate the exact-erf
 *    GELU / GELU' (tensor.cpp:323-351) instead of the tanh.approx form.
 *  RTPB_OPT_PAIRED_DX (default 1, or RTPB_DX_PAIR): out-of-place bf16
 *    backward runs two steps' dX as one GEMM over the two resident shards;
 *    0 restores the reference's per-step summation (out-of-place ==
 *    in-place bitwise, layers_test.cpp:343-365). */
#define RTPB_OPT_EXACT_GELU 1
#define RTPB_OPT_PAIRED_DX 2
int rtpb_linear_set_option(rtpb_linear l, int option, int value);

/* The FFN block (model.cpp:77-83, 99-105): ffn1 (h->f) -> gelu -> ffn2 (f->h),
 * GELU fused into ffn1's forward epilogue and ffn2's last dX epilogue.
 * Flyweight init when w1..b2 are NULL: ffn1 draws from stream_base, ffn2 from
 * stream_base + h*f + f (SerialModel order, serial.cpp:349-350). */
int rtpb_mlp_create(rtpb_group g, const char* label, size_t h, size_t f, int dtype, const double* w1,
                    const double* b1, const double* w2, const double* b2, uint64_t seed, uint64_t stream_base,
                    rtpb_mlp* out);
int rtpb_mlp_destroy(rtpb_mlp m);
int rtpb_mlp_set_rotation_mode(rtpb_mlp m, int mode);
int rtpb_mlp_begin_step(rtpb_mlp m); /* RtpModel::begin_step (model.cpp:54-57) */
int rtpb_mlp_zero_grads(rtpb_mlp m);
int rtpb_mlp_forward(rtpb_mlp m, const void* const* x, size_t rows, void* const* y, int mode);
int rtpb_mlp_backward(rtpb_mlp m, const void* const* dy, size_t rows, void* const* dx);
/* Stack order (RtpModel's block sequence, model.cpp:77-83 / 99-105): `next`
 * follows `m` in forward. Linked blocks post the neighbour's first weight
 * shift under their own last step (out-of-place mode). next = NULL unlinks. */
int rtpb_mlp_chain(rtpb_mlp m, rtpb_mlp next);
int rtpb_mlp_set_option(rtpb_mlp m, int option, int value); /* RTPB_OPT_*, both layers */
/* layer 0 = ffn1, 1 = ffn2 */
rtpb_linear rtpb_mlp_layer(rtpb_mlp m, int layer);

/* RtpAttention(group, label, wq, wk, wv, wo, heads, seq, n)
 * (layers.hpp:170-191, layers_attention.cpp:43-198): head-partitioned
 * attention, projections without bias. wq..wo: hidden x hidden fp64 host
 * arrays. Activations are (batch * seq) x hidden per local rank. */
int rtpb_attention_create(rtpb_group g, const char* label, size_t hidden, size_t heads, size_t seq, int dtype,
                          const double* wq, const double* wk, const double* wv, const double* wo,
                          rtpb_attention* out);
int rtpb_attention_destroy(rtpb_attention a);
int rtpb_attention_set_rotation_mode(rtpb_attention a, int mode);
int rtpb_attention_allocate_comm_spares(rtpb_attention a);
int rtpb_attention_release_comm_spares(rtpb_attention a);
int rtpb_attention_zero_grads(rtpb_attention a);
size_t rtpb_attention_shard_len(rtpb_attention a);
int rtpb_attention_forward(rtpb_attention a, const void* const* x, size_t rows, void* const* y, int mode);
int rtpb_attention_backward(rtpb_attention a, const void* const* dy, size_t rows, void* const* dx);
int rtpb_attention_slot(rtpb_attention a, size_t rank, int64_t* logical_id, int64_t* rotation_offset);
int rtpb_attention_trace(rtpb_attention a, int64_t* ids);
/* Shard resident at local rank r in the reference's flat layout
 * [Wq_j | Wk_j | Wv_j | Wo_j] as fp64 into host memory dst (shard_len values):
 * which 0 = weight, 1 = gradient. */
int rtpb_attention_read_shard(rtpb_attention a, size_t rank, int which, double* dst);

/* RtpEmbedding(group, label, table, n) (layers.hpp:150-168,
 * layers_linear.cpp:74-136): table vocab x emb fp64 host, sharded on the
 * embedding dimension. forward: ids[k] = `counts[k]` int64 host token ids of
 * local rank k, y[k] device counts[k] x emb. backward: dy[k] device, no input
 * gradient. */
int rtpb_embedding_create(rtpb_group g, const char* label, size_t vocab, size_t emb, int dtype, const double* table,
                          rtpb_embedding* out);
int rtpb_embedding_destroy(rtpb_embedding e);
int rtpb_embedding_set_rotation_mode(rtpb_embedding e, int mode);
int rtpb_embedding_allocate_comm_spares(rtpb_embedding e);
int rtpb_embedding_release_comm_spares(rtpb_embedding e);
int rtpb_embedding_zero_grads(rtpb_embedding e);
size_t rtpb_embedding_shard_len(rtpb_embedding e);
int rtpb_embedding_forward(rtpb_embedding e, const int64_t* const* ids, const size_t* counts, void* const* y,
                           int mode);
int rtpb_embedding_backward(rtpb_embedding e, const void* const* dy, size_t rows);
int rtpb_embedding_slot(rtpb_embedding e, size_t rank, int64_t* logical_id, int64_t* rotation_offset);
/* shard resident at local rank r (vocab x emb/n) as fp64 host values: which 0 weight, 1 gradient */
int rtpb_embedding_read_shard(rtpb_embedding e, size_t rank, int which, double* dst);

/* RtpMoe(group, label, gate, experts, n) (layers.hpp:193-229,
 * layers_moe.cpp:18-198): gate hidden x n fp64 host; experts[e] packed
 * [w1 (hidden x ffn) | b1 | w2 (ffn x hidden) | b2] fp64 host, one per worker. */
int rtpb_moe_create(rtpb_group g, const char* label, size_t hidden, size_t ffn, int dtype, const double* gate,
                    const double* const* experts, rtpb_moe* out);
int rtpb_moe_destroy(rtpb_moe m);
int rtpb_moe_set_rotation_mode(rtpb_moe m, int mode);
int rtpb_moe_allocate_comm_spares(rtpb_moe m);
int rtpb_moe_release_comm_spares(rtpb_moe m);
int rtpb_moe_zero_grads(rtpb_moe m);
size_t rtpb_moe_shard_len(rtpb_moe m);
int rtpb_moe_forward(rtpb_moe m, const void* const* x, size_t rows, void* const* y, int mode);
int rtpb_moe_backward(rtpb_moe m, const void* const* dy, size_t rows, void* const* dx);
int rtpb_moe_slot(rtpb_moe m, size_t rank, int64_t* logical_id, int64_t* rotation_offset);
/* expert shard resident at local rank r (fp64 host, packed as created): which 0 weight, 1 gradient */
int rtpb_moe_read_shard(rtpb_moe m, size_t rank, int which, double* dst);
/* the per-worker gate gradient (hidden x n, fp64 host) */
int rtpb_moe_gate_grad(rtpb_moe m, size_t rank, double* dst);

/* RtpModel (model.cpp:7-121) with SerialModel(dims, seed)'s parameters
 * (serial.cpp:325-353): embedding -> layers x (attention + FFN or MoE with
 * residual connections) -> head. moe != 0: one expert per worker. */
int rtpb_model_create(rtpb_group g, size_t heads, size_t hidden, size_t layers, size_t seq, size_t vocab, size_t ffn,
                      int moe, uint64_t seed, int rotation_mode, int dtype, rtpb_model* out);
int rtpb_model_destroy(rtpb_model m);
int rtpb_model_begin_step(rtpb_model m);
int rtpb_model_zero_grads(rtpb_model m);
/* ids[k]: counts[k] host token ids of local rank k; logits[k]: device
 * counts[k] x vocab in the layer dtype. */
int rtpb_model_forward(rtpb_model m, const int64_t* const* ids, const size_t* counts, void* const* logits, int mode);
int rtpb_model_backward(rtpb_model m, const void* const* dlogits, size_t rows);
/* layers in all_layers() order: embedding, per block attention, ffn1, ffn2
 * (or moe), head */
size_t rtpb_model_layer_count(rtpb_model m);
size_t rtpb_model_layer_shard_len(rtpb_model m, size_t layer);
int rtpb_model_read_layer_shard(rtpb_model m, size_t layer, size_t rank, int which, double* dst);
int rtpb_model_gate_grad(rtpb_model m, size_t block, size_t rank, double* dst);

#ifdef __cplusplus
}
#endif
#endif /* RTPB_H */
