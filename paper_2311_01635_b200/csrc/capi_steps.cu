// C ABI, layer (1): per-rotation-step kernels (include/rtpb.h). Each entry
// validates its geometry, carves the caller's workspace and enqueues the
// tcgen05 GEMM (+ helpers) on the given stream. No allocation, no sync.
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "kernels/launch.hpp"

namespace rtpb {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
int g_force_bn = 0;

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

struct Carve {
  char* p;
  size_t left;
  bool ok = true;
  float* take(size_t floats) {
    const size_t b = align256(floats * sizeof(float));
    if (b > left) {
      ok = false;
      return nullptr;
    }
    float* r = reinterpret_cast<float*>(p);
    p += b;
    left -= b;
    return r;
  }
};

int check_geom(size_t M, size_t I, size_t per) {
  if (M == 0 || I == 0 || per == 0) return set_error(RTPB_ERR_DIMENSION, "step: dimensions must be positive");
  if (I % 8 || per % 8)
    return set_error(RTPB_ERR_CONFIG,
                     "step: in_dim and out_dim/N must be multiples of 8 for 16-byte TMA rows; choose "
                     "dimensions that are a multiple of 8 times the worker count");
  if (M > (1u << 30) || I > (1u << 30) || per > (1u << 30))
    return set_error(RTPB_ERR_DIMENSION, "step: dimension too large");
  return RTPB_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Zero-initialised, self-resetting part of a step workspace.
// (16 per tile: one per epilogue warp slot of a CTA pair, for the split-K
// partials' per-region counters; the ordered split-K uses the first.)
size_t split_flag_bytes(size_t I, size_t per) {  // per-tile counters, tiles 256 x (256 or 128)
  return ((I + 255) / 256) * ((per + 127) / 128) * 16 * sizeof(unsigned);
}
// Fused dW bias sums (CTA-pair dW): arrival counter per 64-column group, and
// one partial row per (256-row tile block, K split <= 8).
size_t bias_tick_bytes(size_t per) { return ((per + 63) / 64) * sizeof(unsigned); }
size_t bias_part_bytes(size_t I, size_t per) { return ((I + 255) / 256) * 8 * per * sizeof(float); }
size_t persistent_ws_bytes(size_t M, size_t I, size_t per) {
  return align256(colsum_workspace_bytes(M, per)) + align256(split_flag_bytes(I, per)) +
         align256(bias_tick_bytes(per)) + align256(bias_part_bytes(I, per)) +
         align256(wgrad_partial_floats(false, M, I, per) * sizeof(float));
}

// Optional per-launch timing of the step GEMMs: a CUDA event pair recorded on
// the launching stream around each GEMM (bench.py's roofline numerator).
struct ProfRec {
  int kind;
  double flops;
  cudaEvent_t a, b;
  int sms;  // SM budget of the launch
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Runs `launch` between two recorded events when profiling is on.
template <class F>
int timed(int kind, double flops, cudaStream_t s, F&& launch) {
  if (!g_prof_on) return launch();
  cudaEvent_t a, b;
  {
    std::lock_guard lk(g_prof_mu);
    a = prof_event();
    b = prof_event();
  }
  // Inside stream capture the records must be external event-record nodes so
  // every replay of the graph re-times the launch.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const unsigned fl = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  cudaEventRecordWithFlags(a, s, fl);
  const int rc = launch();
  cudaEventRecordWithFlags(b, s, fl);
  std::lock_guard lk(g_prof_mu);
  g_prof.push_back({kind, flops, a, b, sm_budget()});
  return rc;
}
}  // namespace

int set_error(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  g_last_error = buf;
  return RTPB_ERR_CUDA;
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int fused_fwd_step(const void* x, size_t ldx, const void* w1_shard, void* pre, void* act, const void* w2_shard,
                   void* y, size_t ldy, size_t M, size_t h, size_t f, bool store_pre, const FusedFwdPlan& plan,
                   const FusedFwdWs& ws, cudaStream_t s, bool exact_gelu) {
  int rc;
  if ((rc = check_geom(M, h, f))) return rc;
  const auto* w1 = static_cast<const uint16_t*>(w1_shard);  // bf16 elements
  const auto* w2 = static_cast<const uint16_t*>(w2_shard);
  StepFwd p0{};
  p0.x = x; p0.ldx = ldx; p0.w = w1; p0.bias = w1 + h * f;
  p0.y = pre; p0.ldy = f; p0.act = act; p0.ld_act = f;
  p0.M = M; p0.I = h; p0.per = f;
  p0.flags = RTPB_EPI_GELU | (store_pre ? RTPB_EPI_STORE_PRE : 0) | (exact_gelu ? RTPB_EPI_EXACT_GELU : 0);
  StepFwd p1{};
  p1.x = act; p1.ldx = f; p1.w = w2; p1.bias = w2 + f * h;
  p1.y = y; p1.ldy = ldy; p1.M = M; p1.I = f; p1.per = h; p1.flags = RTPB_EPI_STORE_PRE;
  return timed(0, 4.0 * M * h * f, s, [&] { return gemm_fwd_fused(p0, p1, plan, ws, s); });
}

int fused_bwd_step(FusedBwdArgs a, void* ws1, size_t ws1_bytes, void* ws2, size_t ws2_bytes,
                   const FusedBwdPlan& plan, const FusedBwdWs& ws, cudaStream_t compute, cudaStream_t aux) {
  int rc;
  if ((rc = check_geom(a.M, a.h, a.f))) return rc;
  // each layer's persistent workspace part, carved as rtpb_wgrad_step does
  auto carve = [&](void* w, size_t bytes, size_t I, size_t per, float** part, unsigned** tick, unsigned** flags,
                   float** wpart) {
    Carve c{static_cast<char*>(w), w ? bytes : 0};
    c.take(colsum_workspace_bytes(a.M, per) / sizeof(float));
    *flags = reinterpret_cast<unsigned*>(c.take(split_flag_bytes(I, per) / sizeof(float)));
    *tick = reinterpret_cast<unsigned*>(c.take(bias_tick_bytes(per) / sizeof(float)));
    *part = c.take(bias_part_bytes(I, per) / sizeof(float));
    const size_t wpf = wgrad_partial_floats(false, a.M, I, per);
    // the layer's partial buffer holds its own (whole-machine) split count
    // (no partial buffer: the dW launch falls back to the ordered split-K chain)
    if (wpf && plan.w_splits > 1 && size_t(plan.w_splits) * ((I + 255) / 256 * 256) * per > wpf) return false;
    *wpart = wpf ? c.take(wpf) : nullptr;
    return c.ok;
  };
  if (!carve(ws1, ws1_bytes, a.h, a.f, &a.bias_part1, &a.bias_tick1, &a.split_flags1, &a.wpart1) ||
      !carve(ws2, ws2_bytes, a.f, a.h, &a.bias_part2, &a.bias_tick2, &a.split_flags2, &a.wpart2))
    return set_error(RTPB_ERR_DIMENSION, "fused backward: layer workspace too small");
  // profiled as the two launches: D (both dX GEMMs) and W (both dW GEMMs)
  const double fl = 2.0 * double(a.M) * double(a.h) * double(a.f) * 2.0;
  if (!g_prof_on) return gemm_bwd_fused(a, plan, ws, compute, aux);
  cudaEvent_t e[4];
  {
    std::lock_guard lk(g_prof_mu);
    for (auto& x : e) x = prof_event();
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(compute, &cap);
  const unsigned flg = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  cudaEventRecordWithFlags(e[0], compute, flg);
  cudaEventRecordWithFlags(e[2], aux, flg);
  rc = gemm_bwd_fused(a, plan, ws, compute, aux);
  cudaEventRecordWithFlags(e[1], compute, flg);
  cudaEventRecordWithFlags(e[3], aux, flg);
  std::lock_guard lk(g_prof_mu);
  g_prof.push_back({1, fl, e[0], e[1], 2 * plan.slots_d});
  g_prof.push_back({2, fl, e[2], e[3], 2 * plan.slots_w});
  return rc;
}

}  // namespace rtpb

using namespace rtpb;

extern "C" {

const char* rtpb_last_error(void) { return g_last_error.c_str(); }
const char* rtpb_version(void) { return "rtpb 0.1 (sm_100a tcgen05)"; }
uint64_t rtpb_launch_count(void) { return g_launches.load(); }
void rtpb_debug_force_bn(int bn) { g_force_bn = bn; }
void rtpb_set_sm_budget(int sms) { set_sm_budget(sms); }

double rtpb_debug_fused_plan(size_t M, size_t h, size_t f, int which) {
  if (which == 0) {
    FusedFwdPlan p;
    return plan_fused_fwd(M, h, f, p) ? p.est_us : -1.0;
  }
  FusedBwdPlan p;
  return plan_fused_bwd(M, h, f, p) ? p.est_us : -1.0;
}
void rtpb_debug_trace(void* device_buf, size_t bytes) { set_trace(device_buf, bytes); }

// Workspace layout, identical for every step kind of a layer so one buffer
// serves all three: [bias-grad tickets + partials][dW split-K tile counters]
// (both left at zero by the kernels) [fp32 mode: tf32 hi/lo operand splits].
size_t rtpb_step_workspace_bytes(int which, int dtype, size_t M, size_t I, size_t per) {
  const bool f32 = dtype == RTPB_F32;
  size_t b = persistent_ws_bytes(M, I, per);
  if (f32) {
    if (which == 0) b += 2 * align256(M * I * 4) + 2 * align256(I * per * 4);
    if (which == 1) b += 2 * align256(M * per * 4) + 2 * align256(I * per * 4);
    const size_t Mp = (M + 7) & ~size_t(7);  // transposed operands: 16-byte rows
    if (which == 2) b += 2 * align256(Mp * I * 4) + 2 * align256(Mp * per * 4);
  }
  return b;
}

int rtpb_flyweight_init(void* dst, int dtype, uint64_t seed, uint64_t stream_base, size_t I, size_t O, size_t n,
                        size_t j, double lo, double hi, void* stream) {
  if (!dst) return set_error(RTPB_ERR_DIMENSION, "flyweight_init: null destination");
  return flyweight_init(dst, dtype == RTPB_F32, seed, stream_base, I, O, n, j, lo, hi, as_stream(stream));
}

int rtpb_fwd_step(int dtype, const void* x, size_t ldx, const void* w_shard, void* y, size_t ldy, size_t col0,
                  void* act, size_t ld_act, size_t M, size_t I, size_t per, int flags, void* workspace,
                  size_t workspace_bytes, void* stream) {
  int rc = check_geom(M, I, per);
  if (rc) return rc;
  if ((flags & RTPB_EPI_STORE_PRE) && !y) return set_error(RTPB_ERR_DIMENSION, "fwd_step: null y");
  if ((flags & RTPB_EPI_GELU) && !act) return set_error(RTPB_ERR_DIMENSION, "fwd_step: null act");
  if (!(flags & (RTPB_EPI_STORE_PRE | RTPB_EPI_GELU))) flags |= RTPB_EPI_STORE_PRE;
  const bool f32 = dtype == RTPB_F32;
  const size_t esz = f32 ? 4 : 2;
  cudaStream_t s = as_stream(stream);
  StepFwd p{};
  p.x = x; p.ldx = ldx; p.w = w_shard;
  p.bias = (flags & RTPB_EPI_NO_BIAS) ? nullptr : static_cast<const char*>(w_shard) + I * per * esz;
  flags &= ~RTPB_EPI_NO_BIAS;
  p.y = y; p.ldy = ldy; p.col0 = col0; p.act = act; p.ld_act = ld_act;
  p.M = M; p.I = I; p.per = per; p.flags = flags; p.force_bn = g_force_bn;
  if (f32) {
    Carve c{static_cast<char*>(workspace), workspace ? workspace_bytes : 0};
    c.take(persistent_ws_bytes(M, I, per) / sizeof(float));  // keep the zeroed counters intact
    float *xh = c.take(M * I), *xl = c.take(M * I), *wh = c.take(I * per), *wl = c.take(I * per);
    if (!c.ok) return set_error(RTPB_ERR_DIMENSION, "fwd_step: workspace too small");
    if ((rc = tf32_split(static_cast<const float*>(x), M, I, ldx, xh, xl, s))) return rc;
    if ((rc = tf32_split_t(static_cast<const float*>(w_shard), I, per, per, wh, wl, s))) return rc;
    p.x = xh; p.x_lo = xl; p.ldx = I; p.w = wh; p.w_lo = wl;
  }
  return timed(0, 2.0 * M * I * per, s, [&] { return gemm_fwd(f32, p, s); });
}

int rtpb_dgrad_step(int dtype, const void* dy, size_t ldy, size_t col0, const void* w_shard, float* acc,
                    size_t ld_acc, void* dx, size_t ldx, const void* pre, size_t ldpre, size_t M, size_t I,
                    size_t per, int flags, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_geom(M, I, per);
  if (rc) return rc;
  const bool first = flags & RTPB_EPI_FIRST, last = flags & RTPB_EPI_LAST;
  if (!(first && last) && !acc) return set_error(RTPB_ERR_DIMENSION, "dgrad_step: null fp32 accumulator");
  if (last && !dx) return set_error(RTPB_ERR_DIMENSION, "dgrad_step: null dx");
  if ((flags & RTPB_EPI_GELU_BWD) && !pre) return set_error(RTPB_ERR_DIMENSION, "dgrad_step: null pre");
  const bool f32 = dtype == RTPB_F32;
  const size_t esz = f32 ? 4 : 2;
  cudaStream_t s = as_stream(stream);
  StepDgrad p{};
  p.dy = static_cast<const char*>(dy) + col0 * esz; p.ldy = ldy;
  p.w = w_shard; p.acc = acc; p.ld_acc = ld_acc; p.dx = dx; p.ldx = ldx; p.pre = pre; p.ldpre = ldpre;
  p.M = M; p.I = I; p.per = per; p.flags = flags; p.force_bn = g_force_bn;
  if (f32) {
    Carve c{static_cast<char*>(workspace), workspace ? workspace_bytes : 0};
    c.take(persistent_ws_bytes(M, I, per) / sizeof(float));  // keep the zeroed counters intact
    float *dh = c.take(M * per), *dl = c.take(M * per), *wh = c.take(I * per), *wl = c.take(I * per);
    if (!c.ok) return set_error(RTPB_ERR_DIMENSION, "dgrad_step: workspace too small");
    if ((rc = tf32_split(static_cast<const float*>(p.dy), M, per, ldy, dh, dl, s))) return rc;
    if ((rc = tf32_split(static_cast<const float*>(w_shard), I, per, per, wh, wl, s))) return rc;
    p.dy = dh; p.dy_lo = dl; p.ldy = per; p.w = wh; p.w_lo = wl;
  }
  return timed(1, 2.0 * M * I * per, s, [&] { return gemm_dgrad(f32, p, s); });
}

namespace {
int check_pass(size_t M, size_t I, size_t per, const size_t* col0, size_t steps, size_t cols, int* icol) {
  int rc = check_geom(M, I, per);
  if (rc) return rc;
  if (steps < 2 || steps > 16) return set_error(RTPB_ERR_CONFIG, "pass launch: 2..16 steps");
  if (per % 32) return set_error(RTPB_ERR_CONFIG, "pass launch: out_dim / N must be a multiple of 32");
  if (!col0) return set_error(RTPB_ERR_DIMENSION, "pass launch: null column offsets");
  for (size_t s = 0; s < steps; ++s) {
    if (col0[s] + per > cols) return set_error(RTPB_ERR_DIMENSION, "pass launch: column block out of range");
    icol[s] = int(col0[s]);
  }
  return RTPB_OK;
}
}  // namespace

void rtpb_preload_kernels(void) { preload_device_kernels(); }

unsigned rtpb_pass_done_target(int which, size_t M, size_t I, size_t per, size_t steps, int flags) {
  if (which == 2) return wgrad_pass_done_target(M, I, per, g_force_bn);
  const int groups = int((which == 1 && (flags & RTPB_PASS_PAIR)) ? (steps + 1) / 2 : steps);
  return which == 1 ? pass_done_target(true, M, I, flags & RTPB_EPI_GELU_BWD, g_force_bn, groups)
                    : pass_done_target(false, M, per, false, g_force_bn, groups);
}

int rtpb_fwd_pass(const void* x, size_t ldx, const void* buf0, const void* buf1, void* y, size_t ldy, void* act,
                  size_t ld_act, size_t y_cols, const size_t* col0, unsigned buf_mask, size_t steps, size_t M,
                  size_t I, size_t per, int flags, const unsigned* ready, unsigned* done, unsigned* done_target,
                  unsigned* reset_ctr, void* stream) {
  int icol[16];
  int rc = check_pass(M, I, per, col0, steps, y_cols, icol);
  if (rc) return rc;
  if (!buf0 || !buf1 || !done_target) return set_error(RTPB_ERR_DIMENSION, "fwd_pass: null shard buffer / target");
  if ((flags & RTPB_EPI_STORE_PRE) && !y) return set_error(RTPB_ERR_DIMENSION, "fwd_pass: null y");
  if ((flags & RTPB_EPI_GELU) && !act) return set_error(RTPB_ERR_DIMENSION, "fwd_pass: null act");
  if (!(flags & (RTPB_EPI_STORE_PRE | RTPB_EPI_GELU))) flags |= RTPB_EPI_STORE_PRE;
  cudaStream_t s = as_stream(stream);
  StepFwd p{};
  p.x = x; p.ldx = ldx; p.w = buf0;
  p.bias = (flags & RTPB_EPI_NO_BIAS) ? nullptr : static_cast<const char*>(buf0) + I * per * 2;
  flags &= ~RTPB_EPI_NO_BIAS;
  p.y = y; p.ldy = ldy; p.act = act; p.ld_act = ld_act;
  p.M = M; p.I = I; p.per = per; p.flags = flags; p.force_bn = g_force_bn;
  const PassArgs pa{int(steps), buf_mask, icol, ready, done, reset_ctr};
  return timed(0, 2.0 * M * I * per * steps, s, [&] { return gemm_fwd_pass(p, buf1, y_cols, pa, s, done_target); });
}

int rtpb_dgrad_pass(const void* dy, size_t ldy, size_t dy_cols, const void* buf0, const void* buf1,
                    const size_t* col0, unsigned buf_mask, size_t steps, float* acc, size_t ld_acc, void* dx,
                    size_t ldx, const void* pre, size_t ldpre, size_t M, size_t I, size_t per, int flags,
                    const unsigned* ready, unsigned* done, unsigned* done_target, unsigned* reset_ctr,
                    void* stream) {
  int icol[16];
  int rc = check_pass(M, I, per, col0, steps, dy_cols, icol);
  if (rc) return rc;
  if (!buf0 || !buf1 || !done_target) return set_error(RTPB_ERR_DIMENSION, "dgrad_pass: null shard buffer / target");
  if (!acc || !dx) return set_error(RTPB_ERR_DIMENSION, "dgrad_pass: null accumulator / dx");
  if ((flags & RTPB_EPI_GELU_BWD) && !pre) return set_error(RTPB_ERR_DIMENSION, "dgrad_pass: null pre");
  cudaStream_t s = as_stream(stream);
  StepDgrad p{};
  p.dy = dy; p.ldy = ldy; p.w = buf0; p.acc = acc; p.ld_acc = ld_acc; p.dx = dx; p.ldx = ldx;
  p.pre = pre; p.ldpre = ldpre;
  const int pair = (flags & RTPB_PASS_PAIR) ? 1 : 0;
  flags &= ~RTPB_PASS_PAIR;
  p.M = M; p.I = I; p.per = per; p.flags = flags; p.force_bn = g_force_bn;
  const PassArgs pa{int(steps), buf_mask, icol, ready, done, reset_ctr, pair};
  return timed(1, 2.0 * M * I * per * steps, s,
               [&] { return gemm_dgrad_pass(p, buf1, dy_cols, pa, s, done_target); });
}

size_t rtpb_colsum_workspace_bytes(size_t M, size_t cols) { return colsum_workspace_bytes(M, cols); }

int rtpb_colsum(const void* dy, size_t ldy, size_t M, size_t cols, float* out, void* workspace, size_t workspace_bytes,
                void* stream) {
  if (!dy || !out) return set_error(RTPB_ERR_DIMENSION, "colsum: null buffer");
  if (!workspace || workspace_bytes < colsum_workspace_bytes(M, cols))
    return set_error(RTPB_ERR_DIMENSION, "colsum: workspace too small");
  return colsum_bias_grad(false, dy, ldy, M, cols, nullptr, out, workspace, as_stream(stream));
}

int rtpb_wgrad_pass(const void* x, size_t ldx, const void* dy, size_t ldy, size_t dy_cols, float* g,
                    const size_t* col0, size_t steps, size_t M, size_t I, size_t per, int flags, const float* db,
                    const unsigned* ready, unsigned* done, unsigned* done_target, unsigned* reset_ctr,
                    void* workspace, size_t workspace_bytes, void* stream) {
  int icol[16];
  int rc = check_pass(M, I, per, col0, steps, dy_cols, icol);
  if (rc) return rc;
  if (!g || !done_target) return set_error(RTPB_ERR_DIMENSION, "wgrad_pass: null gradient shard / target");
  if (reinterpret_cast<uintptr_t>(g) & 15) return set_error(RTPB_ERR_CONFIG, "wgrad_pass: gradient shard not 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  Carve c{static_cast<char*>(workspace), workspace ? workspace_bytes : 0};
  c.take(colsum_workspace_bytes(M, per) / sizeof(float));
  unsigned* sflags = reinterpret_cast<unsigned*>(c.take(split_flag_bytes(I, per) / sizeof(float)));
  if (!c.ok) return set_error(RTPB_ERR_DIMENSION, "wgrad_pass: workspace too small");
  StepWgrad p{};
  p.x = x; p.ldx = ldx; p.dy = dy; p.ldy = ldy; p.g_in = g; p.g_out = g;
  p.M = M; p.I = I; p.per = per; p.force_bn = g_force_bn; p.split_flags = sflags;
  const PassArgs pa{int(steps), 0u, icol, ready, done, reset_ctr};
  return timed(2, 2.0 * M * I * per * steps, s, [&] {
    return gemm_wgrad_pass(p, dy_cols, (flags & RTPB_EPI_FIRST) != 0, db, pa, s, done_target);
  });
}

int rtpb_dgrad_step2(int dtype, const void* dy, size_t ldy, size_t col0, const void* w_a, size_t col1,
                     const void* w_b, float* acc, size_t ld_acc, void* dx, size_t ldx, const void* pre,
                     size_t ldpre, size_t M, size_t I, size_t per, int flags, void* workspace,
                     size_t workspace_bytes, void* stream) {
  int rc = check_geom(M, I, per);
  if (rc) return rc;
  if (dtype != RTPB_BF16) return set_error(RTPB_ERR_CONFIG, "dgrad_step2: bf16 only");
  if (!w_a || !w_b) return set_error(RTPB_ERR_DIMENSION, "dgrad_step2: null weight shard");
  const bool first = flags & RTPB_EPI_FIRST, last = flags & RTPB_EPI_LAST;
  if (!(first && last) && !acc) return set_error(RTPB_ERR_DIMENSION, "dgrad_step2: null fp32 accumulator");
  if (last && !dx) return set_error(RTPB_ERR_DIMENSION, "dgrad_step2: null dx");
  if ((flags & RTPB_EPI_GELU_BWD) && !pre) return set_error(RTPB_ERR_DIMENSION, "dgrad_step2: null pre");
  cudaStream_t s = as_stream(stream);
  StepDgrad p{};
  p.dy = static_cast<const char*>(dy) + col0 * 2; p.ldy = ldy;
  p.w = w_a;
  p.dy2 = static_cast<const char*>(dy) + col1 * 2;
  p.w2 = w_b;
  p.acc = acc; p.ld_acc = ld_acc; p.dx = dx; p.ldx = ldx; p.pre = pre; p.ldpre = ldpre;
  p.M = M; p.I = I; p.per = per; p.flags = flags; p.force_bn = g_force_bn;
  (void)workspace;
  (void)workspace_bytes;
  return timed(1, 4.0 * M * I * per, s, [&] { return gemm_dgrad(false, p, s); });
}

int rtpb_wgrad_step(int dtype, const void* x, size_t ldx, const void* dy, size_t ldy, size_t col0,
                    const float* g_in, float* g_out, size_t M, size_t I, size_t per, void* workspace,
                    size_t workspace_bytes, void* stream) {
  return rtpb_wgrad_step_ex(dtype, x, ldx, dy, ldy, col0, g_in, g_out, M, I, per, 0, workspace, workspace_bytes,
                            stream);
}

int rtpb_wgrad_step_ex(int dtype, const void* x, size_t ldx, const void* dy, size_t ldy, size_t col0,
                       const float* g_in, float* g_out, size_t M, size_t I, size_t per, int epi_flags,
                       void* workspace, size_t workspace_bytes, void* stream) {
  const bool no_bias = epi_flags & RTPB_EPI_NO_BIAS;
  int rc = check_geom(M, I, per);
  if (rc) return rc;
  if (!g_out) return set_error(RTPB_ERR_DIMENSION, "wgrad_step: null gradient shard");
  const bool f32 = dtype == RTPB_F32;
  const size_t esz = f32 ? 4 : 2;
  cudaStream_t s = as_stream(stream);
  Carve c{static_cast<char*>(workspace), workspace ? workspace_bytes : 0};
  float* part = c.take(colsum_workspace_bytes(M, per) / sizeof(float));
  unsigned* flags = reinterpret_cast<unsigned*>(c.take(split_flag_bytes(I, per) / sizeof(float)));
  unsigned* btick = reinterpret_cast<unsigned*>(c.take(bias_tick_bytes(per) / sizeof(float)));
  float* bpart = c.take(bias_part_bytes(I, per) / sizeof(float));
  const size_t wpf = f32 ? 0 : wgrad_partial_floats(false, M, I, per);
  float* wpart = wpf ? c.take(wpf) : nullptr;
  StepWgrad p{};
  p.x = x; p.ldx = ldx; p.dy = static_cast<const char*>(dy) + col0 * esz; p.ldy = ldy;
  p.g_in = g_in; p.g_out = g_out; p.M = M; p.I = I; p.per = per; p.force_bn = g_force_bn;
  p.split_flags = flags;
  p.wpart = wpart;
  if (f32) {
    const size_t Mp = (M + 7) & ~size_t(7);
    float *xh = c.take(Mp * I), *xl = c.take(Mp * I), *dh = c.take(Mp * per), *dl = c.take(Mp * per);
    if (!c.ok) return set_error(RTPB_ERR_DIMENSION, "wgrad_step: workspace too small");
    if ((rc = tf32_split_t(static_cast<const float*>(x), M, I, ldx, xh, xl, s))) return rc;
    if ((rc = tf32_split_t(static_cast<const float*>(p.dy), M, per, ldy, dh, dl, s))) return rc;
    p.x = xh; p.x_lo = xl; p.ldx = Mp; p.dy = dh; p.dy_lo = dl; p.ldy = Mp;
  }
  if (!c.ok) return set_error(RTPB_ERR_DIMENSION, "wgrad_step: workspace too small");
  if ((reinterpret_cast<uintptr_t>(g_out) | reinterpret_cast<uintptr_t>(g_in)) & 15)
    return set_error(RTPB_ERR_CONFIG, "wgrad_step: gradient shards must be 16-byte aligned");
  const float* gb_in = g_in && !no_bias ? g_in + I * per : nullptr;
  float* gb_out = no_bias ? nullptr : g_out + I * per;
  return timed(2, 2.0 * M * I * per, s, [&] {
    if (no_bias) {
      // projection without bias (RtpAttention's Wq/Wk/Wv/Wo blocks): G only
    } else if (wgrad_fuses_bias(f32, M, I, per, flags, g_force_bn)) {
      // CTA-pair dW: the kernel's column-sum warp reduces the staged dY tiles.
      p.gbias_in = gb_in;
      p.gbias_out = gb_out;
      p.bias_part = bpart;
      p.bias_tick = btick;
    } else {
      // Bias part first (reads dY only), then the GEMM with the fused G_in + P epilogue.
      int r = colsum_bias_grad(f32, static_cast<const char*>(dy) + col0 * esz, ldy, M, per, gb_in, gb_out, part, s);
      if (r) return r;
    }
    return gemm_wgrad(f32, p, s);
  });
}

void rtpb_profile_enable(int on) {
  std::lock_guard lk(g_prof_mu);
  g_prof_on = on != 0;
}

size_t rtpb_profile_read(int* kinds, double* flops, float* ms, float* start_ms, int* sms, size_t cap) {
  std::lock_guard lk(g_prof_mu);
  const size_t n = g_prof.size();
  for (size_t i = 0; i < n; ++i) {
    ProfRec& r = g_prof[i];
    if (i < cap) {
      cudaEventSynchronize(r.b);
      float t = 0.f, t0 = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      if (i) cudaEventElapsedTime(&t0, g_prof[0].a, r.a);
      if (kinds) kinds[i] = r.kind;
      if (flops) flops[i] = r.flops;
      if (ms) ms[i] = t;
      if (start_ms) start_ms[i] = t0;
      if (sms) sms[i] = r.sms;
    }
  }
  if (cap) {  // reading consumes the records
    for (auto& r : g_prof) {
      g_prof_pool.push_back(r.a);
      g_prof_pool.push_back(r.b);
    }
    g_prof.clear();
  }
  return n;
}

int rtpb_gelu(int dtype, const void* x, void* y, size_t count, void* stream) {
  return gelu_fwd(dtype == RTPB_F32, x, y, count, as_stream(stream));
}

int rtpb_convert(const void* src, int src_dtype, void* dst, int dst_dtype, size_t count, void* stream) {
  auto ok = [](int d) { return d == RTPB_BF16 || d == RTPB_F32 || d == RTPB_F64; };
  if (!ok(src_dtype) || !ok(dst_dtype)) return set_error(RTPB_ERR_CONFIG, "rtpb_convert: unknown dtype");
  if (count && (!src || !dst)) return set_error(RTPB_ERR_DIMENSION, "rtpb_convert: null buffer");
  return convert(src, src_dtype, dst, dst_dtype, count, as_stream(stream));
}

int rtpb_fill(void* dst, int dtype, size_t count, double v, void* stream) {
  if (dtype != RTPB_BF16 && dtype != RTPB_F32 && dtype != RTPB_F64)
    return set_error(RTPB_ERR_CONFIG, "rtpb_fill: unknown dtype");
  if (count && !dst) return set_error(RTPB_ERR_DIMENSION, "rtpb_fill: null buffer");
  return fill(dst, dtype, count, v, as_stream(stream));
}

int rtpb_add(int dtype, const void* a, const void* b, void* out, size_t count, void* stream) {
  if (dtype != RTPB_BF16 && dtype != RTPB_F32 && dtype != RTPB_F64)
    return set_error(RTPB_ERR_CONFIG, "rtpb_add: unknown dtype");
  if (count && (!a || !b || !out)) return set_error(RTPB_ERR_DIMENSION, "rtpb_add: null buffer");
  return add(a, b, out, dtype, count, as_stream(stream));
}

int rtpb_gelu_backward(int dtype, const void* x, const void* upstream, void* out, size_t count, void* stream) {
  return gelu_bwd(dtype == RTPB_F32, x, upstream, out, count, as_stream(stream));
}

}  // extern "C"
