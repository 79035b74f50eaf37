// RtpLayerBase / RtpLinear / RtpMlp over device shards.
// Reference: proj/src/layers_common.cpp:97-181, layers_linear.cpp:6-72,
// model.cpp:54-57,77-83,99-105.
//
// Per step the host does the reference's bookkeeping (position laws, replay
// tape, logical ids, traffic) and enqueues device work:
//   compute stream : the step GEMMs (rtpb_fwd_step / dgrad / wgrad)
//   comm stream    : the ring shifts
// Overlap (out-of-place mode): the shard for step s+1 is sent/received into
// the spare while step s computes on the resident copy. Backward: the weight
// shift overlaps dX and dW of the step; the gradient shard (carrying its
// accumulation) is shifted right after dW and overlaps the next step's dX;
// the next dW waits only for it. In-place mode: the weight shift follows dX
// (overlapping dW), the gradient shift follows dW (overlapping the next dX);
// forward shifts are exposed, as the paper accepts.
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels/launch.hpp"
#include "worker.hpp"

namespace rtpb {

namespace {
int dtype_code(DType d) { return d == DType::F32 ? RTPB_F32 : RTPB_BF16; }

// SMs for dX when dX and dW of one step run side by side (N = 1): the split
// minimising the slower of the two under a wave-quantised cost model of the
// CTA-pair kernels (256 x 256 tiles, ~0.35 us per 64-deep K block per pair
// when TMA-fed from L2, plus a per-tile epilogue / prologue share; dW splits
// K over idle pairs and pays an ordered reduction per split).
// RTPB_OVERLAP_DX_SMS overrides it (measurement).
int overlap_dx_sms(size_t M, size_t I, size_t per, bool gelu_bwd) {
  if (const char* e = std::getenv("RTPB_OVERLAP_DX_SMS")) return std::atoi(e);
  const int sms = sm_budget();
  auto cdiv = [](double a, double b) { return std::ceil(a / b); };
  const double kd = cdiv(double(per), 64), kw = cdiv(double(M), 64);
  const double tiles_d = cdiv(double(M), 256) * cdiv(double(I), 256);
  const double tiles_w = cdiv(double(I), 256) * cdiv(double(per), 256);
  const double ck = 0.35, ck_d = gelu_bwd ? 0.45 : 0.35;
  double best = 1e30;
  int best_sms = sms / 2;
  for (int d = 16; d <= sms - 16; d += 2) {
    const double pd = d / 2, pw = (sms - d) / 2;
    const double t_d = cdiv(tiles_d, pd) * (kd * ck_d + 0.8) + 2.0;
    const double split = std::max(1.0, std::min(8.0, std::floor(pw / tiles_w)));
    const double t_w = cdiv(tiles_w * split, pw) * (kw / split * ck + 0.8) + 2.5 * split;
    const double t = std::max(t_d, t_w);
    if (t < best) {
      best = t;
      best_sms = d;
    }
  }
  return best_sms;
}
// NCCL's send/recv kernels need SMs, and a persistent step GEMM holds every
// SM it is given (one CTA per SM, ~225 KB of shared memory), so with the NCCL
// transport the layers leave RTPB_NCCL_RESERVED_SMS (default 8) SMs free for
// the rotation to progress under the GEMMs instead of queueing behind them.
// The local transports move bytes with copy engines and reserve nothing.
// Single-worker GEMM scheduling pays off while a step GEMM is a few waves of
// 256 x 256 CTA-pair tiles (wave-quantisation tails, one GEMM not filling the
// machine). For large GEMMs the plain per-step kernels on the whole machine
// were measured faster (config (d), 16384 x 4096 x 16384: 1094 TFLOP/s plain,
// 1071 fused, 1046 with dX || dW): beyond 12 waves the N = 1 fusions and the
// dX || dW split are off.
bool n1_scheduling_pays(size_t rows, size_t a, size_t b) {
  const size_t tiles = ((rows + 255) / 256) * ((std::max(a, b) + 255) / 256);
  return tiles <= size_t(12) * size_t(std::max(1, sm_budget() / 2));
}

// N > 1 (one worker per GPU): SMs for dX when a step's dX and dW run side by
// side (dW on the aux stream). dX accumulates into an fp32 rows x I buffer,
// 8 bytes of HBM traffic per element per step whatever its K (= per), so for
// small per it is HBM-bound while dW stays tensor-bound: sharing
// the SMs overlaps the two. Model: 1.5 PFLOP/s over all SMs, 6 TB/s HBM;
// returns 0 (no split) unless the split step is >= 10 % faster.
// The model takes HBM as reachable from any number of SMs; it is not: the
// dX epilogue streams its fp32 tiles at ~25-50 GB/s per SM, so on a share of
// the SMs dX runs far below 6 TB/s. Measured (`bench.py --solo N`, config
// (b), per-GPU TFLOP/s, both layers split / neither): N = 2 501 / 541, N = 4
// 271 / 329, N = 8 204 / 186; at N = 8 splitting only ffn2 gives 188. The
// gain is ffn1's: its dX (I = 768) is 96 CTA-pair tiles, 1.3 waves, and its
// dW a short split-K chain, so the two fit side by side. So the split is
// kept for a dX of under two waves of pair tiles: N = 2 / 4 / 8 then measure
// 546 / 365 / 203 (vs 546 / 330 / 187 without any split).
bool dx_pair_enabled() {
  const char* e = std::getenv("RTPB_DX_PAIR");
  return !e || std::atoi(e) != 0;
}

int nway_dx_sms(size_t rows, size_t I, size_t per) {
  if (std::getenv("RTPB_NO_OVERLAP")) return 0;
  if (const char* e = std::getenv("RTPB_NWAY_DX_SMS")) return std::atoi(e);
  const size_t tiles_d = ((rows + 255) / 256) * ((I + 255) / 256);
  if (tiles_d >= size_t(sm_budget())) return 0;
  const int all = sm_budget();
  const double flops = 2.0 * double(rows) * double(I) * double(per);
  const double p_sm = 1.5e15 / 148.0, rmw = 8.0 * double(rows) * double(I) / 6e12;
  auto t_dx = [&](int d) { return std::max(flops / (p_sm * d), rmw); };
  auto t_dw = [&](int w) { return flops / (p_sm * w); };
  const double seq = t_dx(all) + t_dw(all);
  double best = seq;
  int best_d = 0;
  for (int d = 16; d <= all - 16; d += 2) {
    const double t = std::max(t_dx(d), t_dw(all - d));
    if (t < best) {
      best = t;
      best_d = d;
    }
  }
  return best < 0.9 * seq ? best_d : 0;
}

// Simulated distributed flags (RTPB_SIM_FLAGS=1, tests / measurement): the
// arrival-flag and pass-launch paths on a Lockstep group whose workers share
// one GPU. Every worker's grids are sized to its share of the SMs and launched
// without programmatic (PDL) overlap, so all workers' spinning grids are
// resident together and the protocol runs as on one GPU per worker.
// RTPB_TRACE_HOST=1: the layers report their pass launches on stderr (debug)
void host_trace(const std::string& label, const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("RTPB_TRACE_HOST");
    return e && std::atoi(e) != 0;
  }();
  if (on) std::fprintf(stderr, "[rtpb] %s: %s\n", label.c_str(), what);
}

// RTPB_SERIAL_PROFILE=1 on a Solo group (no peers, no bytes move): every
// shift's arrival flag is raised before the pass launches instead of after
// them, so a profiler that runs kernels one at a time (ncu) can replay them.
bool serial_profile_env() {
  static const bool on = [] {
    const char* e = std::getenv("RTPB_SERIAL_PROFILE");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

bool sim_flags() {
  static const bool on = [] {
    const char* e = std::getenv("RTPB_SIM_FLAGS");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

class SmReserve {
 public:
  explicit SmReserve(const WorkerGroup& g) {
    if (sim_flags() && g.kind() == TransportKind::Lockstep && g.local_ranks().size() > 1) {
      set_sm_budget(0);
      set_sm_budget(std::max(2, sm_budget() / int(g.local_ranks().size())) & ~1);
      set_pdl_enabled(false);
      active_ = true;
      return;
    }
    if (g.kind() != TransportKind::Nccl || g.size() < 2) return;
    int reserve = 8;
    if (const char* e = std::getenv("RTPB_NCCL_RESERVED_SMS")) reserve = std::max(0, std::atoi(e));
    if (reserve == 0) return;
    set_sm_budget(0);
    const int all = sm_budget();
    set_sm_budget(std::max(2, all - reserve));
    active_ = true;
  }
  ~SmReserve() {
    if (active_) {
      set_sm_budget(0);
      set_pdl_enabled(true);
    }
  }

 private:
  bool active_ = false;
};
}  // namespace

// ------------------------------------------------------------------ base
RtpLayerBase::RtpLayerBase(WorkerGroup& group, std::string label, DType dtype)
    : group_(&group), label_(std::move(label)), dtype_(dtype), paired_dx_(dx_pair_enabled()) {
  // one block of arrival flags per layer (forward W, backward W, backward G
  // for up to 16 steps), reused cyclically across the pool
  static std::atomic<size_t> next_layer{0};
  flag_base_ = (next_layer.fetch_add(1) % (Worker::kFlagPool / Worker::kFlagsPerLayer)) * Worker::kFlagsPerLayer;
}

void RtpLayerBase::init_slots_alloc() {
  const size_t n = group_->size();
  slots_.resize(n);
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    ShardSlot& s = slots_[r];
    s.weight = Tensor({shard_len_}, dtype_, w.device, &w.ledger, MemCategory::Param, false);
    s.grad_acc = Tensor({shard_len_}, DType::F32, w.device, &w.ledger, MemCategory::Grad, true);
    s.logical_id = r;
    s.rotation_offset = 0;
  });
}

void RtpLayerBase::zero_grads() { grads_zero_pending_ = true; }

void RtpLayerBase::set_rotation_mode(RotationMode m) {
  if (m != rotation_mode_) drop_prefetch();
  rotation_mode_ = m;
}

void RtpLayerBase::materialize_grads() {
  if (!grads_zero_pending_) return;
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    cuda_check(cudaMemsetAsync(slots_[r].grad_acc.data(), 0, slots_[r].grad_acc.bytes(), w.compute),
               "zero_grads");
  });
  grads_zero_pending_ = false;
}

bool RtpLayerBase::all_home() const {
  for (size_t r : group_->local_ranks())
    if (slots_[r].logical_id != r) return false;
  return true;
}

void RtpLayerBase::require_home(const char* op) const {
  if (!all_home()) throw StateError(label_ + ": " + op + " requires every slot at its home position");
}

void RtpLayerBase::check_forward_position(size_t rank, size_t step) const {
  int64_t id = 0;
  check_status(rtpb_ring_plan(group_->size(), rank, 0, step, &id, nullptr, nullptr));
  const size_t expected = size_t(id);
  if (slots_[rank].logical_id != expected)
    throw ProtocolError(label_ + ": worker " + std::to_string(rank) + " holds shard " +
                        std::to_string(slots_[rank].logical_id) + " at forward step " + std::to_string(step) +
                        ", expected " + std::to_string(expected));
}

void RtpLayerBase::check_backward_position(size_t rank, size_t step) const {
  int64_t id = 0;
  check_status(rtpb_ring_plan(group_->size(), rank, 1, step, &id, nullptr, nullptr));
  const size_t expected = size_t(id);
  if (slots_[rank].logical_id != expected)
    throw ProtocolError(label_ + ": worker " + std::to_string(rank) + " holds shard " +
                        std::to_string(slots_[rank].logical_id) + " at backward step " + std::to_string(step) +
                        ", expected " + std::to_string(expected));
}

void RtpLayerBase::allocate_comm_spares() {
  drop_prefetch();
  if (group_->size() == 1) return;  // no rotation, no buffer (layers_common.cpp:153-160)
  // One weight-shard-sized spare per worker, as the reference (shard_len
  // elements of the weight dtype): the incoming W lands there while the
  // resident W is still read; gradients move in place (ring.cpp:314,328).
  spares_.resize(group_->size());
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    spares_[r] = Tensor({shard_len_}, dtype_, w.device, &w.ledger, MemCategory::CommBuffer, false);
  });
}

void RtpLayerBase::release_comm_spares() {
  drop_prefetch();
  group_->synchronize();
  spares_.clear();
}

void RtpLayerBase::rotate_forward() {
  if (oop())
    group_->rotate_outofplace(slots_, spares_, Direction::Clockwise, PayloadKind::Weight, label_, shard_len_);
  else
    group_->rotate_clockwise(slots_, PayloadKind::Weight, label_, shard_len_);
}

void RtpLayerBase::rotate_backward() {
  materialize_grads();  // gradients travel: make a pending zero fill real first
  if (oop())
    group_->rotate_outofplace(slots_, spares_, Direction::CounterClockwise, PayloadKind::WeightAndGrad, label_,
                              shard_len_);
  else
    group_->rotate_counterclockwise(slots_, PayloadKind::WeightAndGrad, label_, shard_len_);
}

void RtpLayerBase::rehome_after_eval() {
  if (group_->size() > 1) rotate_forward();
}

// ------------------------------------------------------------------ linear
void RtpLinear::build(size_t in_dim, size_t out_dim, size_t n) {
  if (n != group_->size())
    throw ConfigError("RtpLinear: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  layout_ = layout_linear(in_dim, out_dim, n);  // ConfigError with the reference's "multiple" hint
  in_ = in_dim;
  out_ = out_dim;
  per_ = out_dim / n;
  if (in_ % 8 || per_ % 8)
    throw ConfigError("RtpLinear " + label_ + ": in_dim and out_dim/N must be multiples of 8 on the device path "
                      "(16-byte TMA rows); choose out_dim as a multiple of 8 times the worker count");
  shard_len_ = in_ * per_ + per_;
  init_slots_alloc();
  tapes_.assign(n, {});
  x_cache_.assign(n, {});
  dx_acc_.resize(n);
  workspace_.resize(n);
  trace_.assign(2 * n * n, -1);
}

RtpLinear::RtpLinear(WorkerGroup& group, std::string label, const double* weight, const double* bias,
                     size_t in_dim, size_t out_dim, size_t n, DType dtype)
    : RtpLayerBase(group, std::move(label), dtype) {
  build(in_dim, out_dim, n);
  upload_shards(weight, bias);
}

// linear_shard_groups + flatten_shards + shard_view (layers_common.cpp:33-45):
// shard r = [W[:, r*per:(r+1)*per] row-major | b[r*per:(r+1)*per]].
void RtpLinear::upload_shards(const double* weight, const double* bias) {
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    DeviceGuard dg(w.device);
    std::vector<double> host(shard_len_);
    for (size_t i = 0; i < in_; ++i)
      std::memcpy(&host[i * per_], weight + i * out_ + r * per_, per_ * sizeof(double));
    std::memcpy(&host[in_ * per_], bias + r * per_, per_ * sizeof(double));
    if (dtype_ == DType::F32) {
      std::vector<float> f(shard_len_);
      for (size_t e = 0; e < shard_len_; ++e) f[e] = static_cast<float>(host[e]);
      cuda_check(cudaMemcpy(slots_[r].weight.data(), f.data(), f.size() * 4, cudaMemcpyHostToDevice), "upload");
    } else {
      std::vector<uint16_t> h(shard_len_);
      for (size_t e = 0; e < shard_len_; ++e) h[e] = double_to_bf16_rne(host[e]);
      cuda_check(cudaMemcpy(slots_[r].weight.data(), h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
    }
  });
}

namespace {
DType layer_dtype_of(const Tensor& weight) { return weight.dtype() == DType::BF16 ? DType::BF16 : DType::F32; }
}  // namespace

RtpLinear::RtpLinear(WorkerGroup& group, std::string label, const Tensor& weight, const Tensor& bias, size_t n)
    : RtpLayerBase(group, std::move(label), layer_dtype_of(weight)) {
  if (weight.rank() != 2) throw DimensionError(label_ + ": weight must be rank 2 (in x out), got " + weight.shape_str());
  if (bias.rank() != 1 || bias.dim(0) != weight.cols())
    throw DimensionError(label_ + ": bias of shape " + bias.shape_str() + " does not match weight " +
                         weight.shape_str());
  build(weight.rows(), weight.cols(), n);
  const std::vector<double> w = weight.to_host(), b = bias.to_host();
  upload_shards(w.data(), b.data());
}

// ---- Tensor API (layers.hpp:138-139) over the device-view passes ----
namespace detail {
// x holds either one tensor per rank (n, all local) or one per local rank.
std::vector<const Tensor*> per_local(WorkerGroup& g, std::span<const Tensor> x, const std::string& label,
                                     const char* what) {
  const auto& local = g.local_ranks();
  std::vector<const Tensor*> out(local.size());
  if (x.size() == g.size() && local.size() == g.size()) {
    for (size_t k = 0; k < local.size(); ++k) out[k] = &x[local[k]];
  } else if (x.size() == local.size()) {
    for (size_t k = 0; k < local.size(); ++k) out[k] = &x[k];
  } else {
    throw DimensionError(label + ": " + what + " expects " + std::to_string(local.size()) +
                         " tensors (one per local worker), got " + std::to_string(x.size()));
  }
  return out;
}

// The input for local rank r in the layer dtype on the worker's device:
// `keep` receives a converted copy (or a plain copy when keep_same is set).
const Tensor& as_layer_input(const Tensor& t, DType dt, Worker& w, size_t cols, const std::string& label,
                             Tensor& keep, bool keep_same) {
  if (t.rank() != 2 || t.cols() != cols)
    throw DimensionError(label + ": activation of shape " + t.shape_str() + " does not have " +
                         std::to_string(cols) + " columns");
  if (t.device() != w.device)
    throw DimensionError(label + ": activation on device " + std::to_string(t.device()) + ", worker " +
                         std::to_string(w.rank) + " runs on device " + std::to_string(w.device));
  if (t.dtype() == dt && !keep_same) return t;
  LedgerScope scope(&w.ledger, MemCategory::Activation);
  keep = t.to(dt);
  return keep;
}
}  // namespace detail
using detail::as_layer_input;
using detail::per_local;

std::vector<Tensor> RtpLinear::forward(std::span<const Tensor> x, Mode mode) {
  const auto& local = group_->local_ranks();
  auto xs = per_local(*group_, x, label_, "forward");
  const size_t rows = xs[0]->rank() == 2 ? xs[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), ys(local.size());
  std::vector<DView> xv(local.size()), yv(local.size());
  const bool train = mode == Mode::Train;
  if (train) x_keep_.assign(group_->size(), Tensor());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    Tensor& keep = train ? x_keep_[local[k]] : tmp[k];
    const Tensor& xin = as_layer_input(*xs[k], dtype_, w, in_, label_, keep, train);  // x_cache_ is a copy
    if (xin.rows() != rows) throw DimensionError(label_ + ": workers' activations differ in row count");
    ys[k] = Tensor({rows, out_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    xv[k] = {xin.data(), in_};
    yv[k] = {ys[k].data(), out_};
  }
  forward(xv, rows, yv, mode);
  group_->synchronize();  // the reference returns completed tensors
  return ys;
}

std::vector<Tensor> RtpLinear::backward(std::span<const Tensor> dy) {
  const auto& local = group_->local_ranks();
  auto ds = per_local(*group_, dy, label_, "backward");
  const size_t rows = ds[0]->rank() == 2 ? ds[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), dxs(local.size());
  std::vector<DView> dv(local.size()), xv(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    const Tensor& din = as_layer_input(*ds[k], dtype_, w, out_, label_, tmp[k], false);
    if (din.rows() != rows) throw DimensionError(label_ + ": workers' gradients differ in row count");
    dxs[k] = Tensor({rows, in_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    dv[k] = {din.data(), out_};
    xv[k] = {dxs[k].data(), in_};
  }
  if (!x_keep_.empty() && x_keep_[local[0]].empty() == false && x_keep_[local[0]].rows() != rows)
    throw DimensionError(label_ + ": backward over " + std::to_string(rows) + " rows, forward saw " +
                         std::to_string(x_keep_[local[0]].rows()));
  backward(dv, rows, xv);
  group_->synchronize();
  x_keep_.clear();  // layers_linear.cpp:69
  return dxs;
}

RtpLinear::RtpLinear(WorkerGroup& group, std::string label, size_t in_dim, size_t out_dim, size_t n,
                     uint64_t seed, uint64_t stream_base, DType dtype)
    : RtpLayerBase(group, std::move(label), dtype) {
  build(in_dim, out_dim, n);
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    check_status(rtpb_flyweight_init(slots_[r].weight.data(), dtype_code(dtype_), seed, stream_base, in_, out_, n,
                                     r, -0.1, 0.1, w.compute));
  });
}

void RtpLinear::ensure_scratch(size_t rows) {
  if (rows == scratch_rows_) return;
  group_->synchronize();
  const size_t n = group_->size();
  const int dt = dtype_code(dtype_);
  size_t ws = 0;
  for (int which = 0; which < 3; ++which) ws = std::max(ws, rtpb_step_workspace_bytes(which, dt, rows, in_, per_));
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    dx_acc_[r] = n > 1 ? DeviceBuffer(w.device, rows * in_ * sizeof(float), &w.ledger, MemCategory::Activation, false)
                       : DeviceBuffer();
    workspace_[r] = ws ? DeviceBuffer(w.device, ws, &w.ledger, MemCategory::Other, true) : DeviceBuffer();
  });
  scratch_rows_ = rows;
}

void RtpLinear::forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode) {
  forward_ex(x, rows, y, mode, FwdEpi{});
}

void RtpLinear::backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx) {
  backward_ex(dy, rows, dx, BwdEpi{});
  group_->join_aux();
}

void RtpLinear::forward_ex(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode,
                           const FwdEpi& e) {
  try {
    forward_impl(x, rows, y, mode, e);
  } catch (...) {
    drop_prefetch();  // a prefetched first shift is not trusted after a failed pass
    throw;
  }
}

void RtpLinear::forward_impl(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode,
                             const FwdEpi& e) {
  require_home("forward");
  SmReserve sm_reserve(*group_);
  const auto& local = group_->local_ranks();
  if (x.size() != local.size() || (e.store_pre && y.size() != local.size()))
    throw DimensionError(label_ + ": forward expects one activation per local worker");
  if (!e.act.empty() && e.act.size() != local.size())
    throw DimensionError(label_ + ": forward expects one gelu output per local worker");
  if (rows == 0) throw DimensionError(label_ + ": forward needs at least one row");
  const size_t n = group_->size();
  ensure_scratch(rows);
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  if (mode == Mode::Train) {
    for (size_t k = 0; k < local.size(); ++k) x_cache_[local[k]] = x[k];
    cached_rows_ = rows;
  }
  std::fill(trace_.begin(), trace_.begin() + n * n, -1);
  const int dt = dtype_code(dtype_);
  const bool prefetch = oop();
  std::vector<void*> wp(n, nullptr), sp(n, nullptr);

  if (pass_launch_ok()) {
    // The whole pass as ONE persistent launch per worker (rtpb_fwd_pass): the
    // host does the N steps' bookkeeping up front, each worker's comm stream
    // lands shard s + 1 in the buffer step s - 1 read once the launch has
    // counted step s - 1 out (cuStreamWaitValue32), and the launch's step
    // s + 1 tiles wait for its arrival flag. Same bits as the per-step launches.
    std::vector<std::array<void*, 2>> buf(n);
    std::vector<std::array<size_t, 16>> cols(n);
    for (size_t r : local) buf[r] = {slots_[r].weight.data(), spares_[r].data()};
    unsigned mask = 0;
    for (size_t s = 0; s < n; ++s) {
      group_->each([&](size_t r) {
        check_forward_position(r, s);
        trace_[s * n + r] = int64_t(slots_[r].logical_id);
        if (mode == Mode::Train) tapes_[r].record(slots_[r].logical_id, {});
        cols[r][s] = slots_[r].logical_id * per_;
      });
      if (s & 1) mask |= 1u << s;
      if (s + 1 < n) group_->advance_slots(slots_, Direction::Clockwise, PayloadKind::Weight, label_, shard_len_);
    }
    int flags = e.store_pre ? RTPB_EPI_STORE_PRE : 0;
    if (!e.act.empty()) flags |= RTPB_EPI_GELU | (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0);
    const unsigned target = rtpb_pass_done_target(0, rows, in_, per_, n, flags);
    // Grids first, then the shifts: every stream memory wait is queued after
    // the work it waits for (a wait ahead of it on a hardware queue shared
    // by two streams would block it), and nothing between the launches and
    // the shifts blocks the host (kernels preloaded, no allocation).
    group_->comm_after_compute();  // the spare's last reader (the previous pass) is done
    const bool serial = serial_profile();
    auto post_shifts = [&] {
      host_trace(label_, "forward pass: shifts");
      for (size_t s = 0; s + 1 < n; ++s) {
        if (s == 0 && pre_fwd_) continue;  // posted under the previous layer's last step
        for (size_t r : local) {
          Worker& w = group_->worker(r);
          DeviceGuard dg(w.device);
          if (s >= 1 && !serial) stream_wait_geq_u32(w.comm, w.flag(flag_base_ + kFlagDoneFwd + s - 1), target);
          wp[r] = buf[r][s & 1];
          sp[r] = buf[r][(s + 1) & 1];
        }
        flagged_exchange(Direction::Clockwise, wp, sp, slots_[local[0]].weight.bytes(), kFlagFwd + s + 1);
      }
    };
    if (serial) post_shifts();  // (profiling a Solo group: every flag up front)
    host_trace(label_, "forward pass: launches");
    group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      void* act = e.act.empty() ? nullptr : e.act[k].data;
      const size_t ld_act = e.act.empty() ? 0 : (e.act[k].ld ? e.act[k].ld : out_);
      void* yp = e.store_pre ? y[k].data : nullptr;
      const size_t ldy = e.store_pre && y[k].ld ? y[k].ld : out_;
      unsigned tgt = target;  // checked before the launch
      check_status(rtpb_fwd_pass(x[k].data, x[k].ld ? x[k].ld : in_, buf[r][0], buf[r][1], yp, ldy, act, ld_act, out_,
                                 cols[r].data(), mask, n, rows, in_, per_, flags, w.flag(flag_base_ + kFlagFwd),
                                 w.flag(flag_base_ + kFlagDoneFwd), &tgt, w.flag(flag_base_ + kFlagCtrFwd),
                                 w.compute));
    });
    if (!serial) post_shifts();
    pre_fwd_ = false;
    for (size_t r : local) group_->worker(r).record(Ev::PassEnd, true);
    if (e.before_last_step) {  // the next layer's first shift, queued behind this pass's (fenced above)
      group_->set_comm_fenced(true);
      try {
        e.before_last_step();
      } catch (...) {
        group_->set_comm_fenced(false);
        throw;
      }
      group_->set_comm_fenced(false);
    }
    for (size_t r : local) {
      if ((n - 1) & 1) swap_data(slots_[r].weight, spares_[r]);  // the pass's n - 1 swaps
      group_->worker(r).wait(Ev::PassEnd, false);  // join the pass's shifts (stream capture requires it)
    }
    if (mode == Mode::Eval) rehome_after_eval();
    return;
  }

  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      check_forward_position(r, s);
      trace_[s * n + r] = int64_t(slots_[r].logical_id);
      if (mode == Mode::Train) tapes_[r].record(slots_[r].logical_id, {});
    });
    const bool rotate = s + 1 < n;
    if (rotate && prefetch && !(s == 0 && pre_fwd_)) {
      // Shard for step s+1 streams into the spare while step s computes.
      group_->comm_after_compute();  // spare's last reader (step s-1) is done
      for (size_t r : local) {
        wp[r] = slots_[r].weight.data();
        sp[r] = spares_[r].data();
      }
      flagged_exchange(Direction::Clockwise, wp, sp, slots_[local[0]].weight.bytes(), kFlagFwd + s + 1);
    }
    pre_fwd_ = false;
    if (s + 1 == n && prefetch && use_flags())
      for (size_t r : local) group_->worker(r).record(Ev::PassEnd, true);  // this pass's comm work
    if (s + 1 == n && e.before_last_step) e.before_last_step();
    const bool wait_flag = prefetch && use_flags() && s > 0;
    group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      // this step's shard landed in the previous step's spare
      set_launch_wait_flag(wait_flag ? w.flag(flag_base_ + kFlagFwd + s) : nullptr);
      // the pass's last reader clears the pass's flags when it is done
      if (wait_flag && s + 1 == n)
        set_launch_flag_reset(w.flag(flag_base_ + kFlagFwd), int(kFlagBwdW - kFlagFwd),
                              w.flag(flag_base_ + kFlagCtrFwd));
      const size_t k = k_of[r];
      const size_t j = slots_[r].logical_id;
      int flags = e.store_pre ? RTPB_EPI_STORE_PRE : 0;
      void* act = nullptr;
      size_t ld_act = 0;
      if (!e.act.empty()) {
        flags |= RTPB_EPI_GELU | (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0);
        act = e.act[k].data;
        ld_act = e.act[k].ld ? e.act[k].ld : out_;
      }
      void* yp = e.store_pre ? y[k].data : nullptr;
      const size_t ldy = e.store_pre && y[k].ld ? y[k].ld : out_;
      const int rc = rtpb_fwd_step(dt, x[k].data, x[k].ld ? x[k].ld : in_, slots_[r].weight.data(), yp, ldy,
                                   j * per_, act, ld_act, rows, in_, per_, flags, workspace_[r].data(),
                                   workspace_[r].bytes(), w.compute);
      set_launch_wait_flag(nullptr);
      set_launch_flag_reset(nullptr, 0, nullptr);
      check_status(rc);
    });
    if (!rotate) break;
    if (prefetch) {
      if (!use_flags()) group_->compute_after_comm();
      for (size_t r : local) swap_data(slots_[r].weight, spares_[r]);
      group_->advance_slots(slots_, Direction::Clockwise, PayloadKind::Weight, label_, shard_len_);
    } else {
      rotate_forward();
    }
  }
  // flags: the compute stream never waited for this pass's shifts; join them
  // once at its end (stream capture requires it). A shift the hook prefetched
  // for the next layer stays in flight; that layer's pass joins it.
  if (n > 1 && prefetch && use_flags()) {
    for (size_t r : local) group_->worker(r).wait(Ev::PassEnd, false);
  }
  if (mode == Mode::Eval) rehome_after_eval();
}

// Arrival flags (bf16 mode, one worker per GPU, N <= 16): the shift's comm
// stream moves the shard, then sets the flag with a stream memory operation
// (no SM needed; the pass's last reader grid clears the pass's flags when it
// is done — GemmArgs::flag_reset — after every flag of the pass was set); the consuming step GEMM waits for it on the device
// instead of its stream waiting for comm, so consecutive step GEMMs keep their
// programmatic (PDL) launch overlap. Deadlock freedom: every flag's writer was
// issued before its waiter and waits only on earlier-issued kernels; a waiting
// grid admits no successor (the kernel triggers PDL after the flag), so the
// spinning grids hold at most the SM budgets of the two streams; shifts that
// need SMs (NCCL) run on the SMs reserved for them. fp32 mode keeps event
// ordering: its operand-split pre-passes read the shard before the GEMM.
// Several workers on one device (Lockstep/Concurrent) also keep events: their
// spinning grids would compete for the same SMs.
// Default on (RTPB_FLAGS=0 keeps stream events): the flags carry the pass
// launches (pass_launch_ok), which `bench.py --solo N` (config (b), TFLOP/s
// per GPU) measures at 710 / 585 / 353 for N = 2 / 4 / 8 against 637 / 419 /
// 257 with one event-ordered launch per step; the protocol is checked with
// real shard movement by the simulated ring (tests/test_gpu_pass.py).
bool RtpLinear::use_flags() const {
  // RTPB_FLAGS=0/1 forces; unset: on, except where processes share a GPU
  // (time-sliced: a grid spinning on a flag can hold the GPU while the peer
  // process that would raise it is switched out)
  static const int env = [] {
    const char* e = std::getenv("RTPB_FLAGS");
    return e ? (std::atoi(e) != 0 ? 1 : 0) : -1;
  }();
  const bool on = env >= 0 ? env == 1 : !group_->device_shared();
  const TransportKind k = group_->kind();
  const bool one_per_gpu = k == TransportKind::Nccl || k == TransportKind::Ipc || k == TransportKind::Solo ||
                           (k == TransportKind::Lockstep && sim_flags());
  return on && one_per_gpu && dtype_ == DType::BF16 && group_->size() > 1 && group_->size() <= 16;
}

// Pass launches (rtpb_fwd_pass / rtpb_dgrad_pass) ride on the arrival flags:
// one worker per GPU (or the simulated form, RTPB_SIM_FLAGS), out of place
// (the shard alternates between the resident buffer and the spare), column
// blocks in whole 32-column store boxes, no other process on the GPU.
// RTPB_NO_PASS=1 keeps one launch per step.
bool RtpLinear::serial_profile() const {
  return serial_profile_env() && group_->kind() == TransportKind::Solo;
}

bool RtpLinear::pass_launch_ok() const {
  static const bool off = [] {
    const char* e = std::getenv("RTPB_NO_PASS");
    return e && std::atoi(e) != 0;
  }();
  const size_t n = group_->size();
  return !off && use_flags() && oop() && n >= 2 && n <= 16 && per_ % 32 == 0 &&
         spares_.size() == n && !group_->device_shared();
}

void RtpLinear::flagged_exchange(Direction dir, std::span<void* const> send, std::span<void* const> recv,
                                 size_t bytes, size_t flag, int channel) {
  const auto& local = group_->local_ranks();
  const bool fl = use_flags();
  group_->exchange(dir, send, recv, bytes, channel);
  if (fl)
    for (size_t r : local) {
      Worker& w = group_->worker(r);
      DeviceGuard dg(w.device);
      stream_write_u32(w.comm_of(channel), w.flag(flag_base_ + flag), 1u);
    }
}

// A first shift posted by prefetch_first_shift lives in the spare until its
// pass consumes it. Anything that replaces or re-purposes the spare (release
// / allocate, a rotation-mode switch, a failed pass) drops it, so the next
// pass posts its own step-0 shift instead of computing on a stale spare. With
// arrival flags the prefetched shift also raised its step-1 flag; it is
// lowered once the shift has landed.
void RtpLinear::drop_prefetch() {
  if (!pre_fwd_ && !pre_bwd_) return;
  group_->synchronize();
  if (use_flags())
    for (size_t r : group_->local_ranks()) {
      Worker& w = group_->worker(r);
      DeviceGuard dg(w.device);
      if (pre_fwd_) cuda_check(cudaMemsetAsync(w.flag(flag_base_ + kFlagFwd + 1), 0, 4, w.comm), "drop prefetch");
      if (pre_bwd_) cuda_check(cudaMemsetAsync(w.flag(flag_base_ + kFlagBwdW + 1), 0, 4, w.comm), "drop prefetch");
      cuda_check(cudaStreamSynchronize(w.comm), "drop prefetch");
    }
  pre_fwd_ = pre_bwd_ = false;
}

void RtpLinear::prefetch_first_shift(bool backward) {
  const size_t n = group_->size();
  if (n < 2 || !oop() || (backward ? pre_bwd_ : pre_fwd_)) return;
  const auto& local = group_->local_ranks();
  // forward starts from home; backward from where the train forward left the
  // shards (its tape is recorded)
  if (!backward && !all_home()) return;
  if (backward)
    for (size_t r : local)
      if (tapes_[r].empty()) return;
  std::vector<void*> wp(n, nullptr), sp(n, nullptr);
  group_->comm_after_compute();  // the spare's last reader is done
  for (size_t r : local) {
    wp[r] = slots_[r].weight.data();
    sp[r] = spares_[r].data();
  }
  flagged_exchange(backward ? Direction::CounterClockwise : Direction::Clockwise, wp, sp,
                   slots_[local[0]].weight.bytes(), backward ? kFlagBwdW + 1 : kFlagFwd + 1);
  if (backward)
    for (size_t r : local) group_->worker(r).record(Ev::WDone, true);
  (backward ? pre_bwd_ : pre_fwd_) = true;
}

const void* RtpLinear::begin_forward_n1(const DView& x, size_t rows, Mode mode) {
  require_home("forward");
  if (group_->size() != 1) throw StateError(label_ + ": begin_forward_n1 needs a single-worker group");
  if (rows == 0) throw DimensionError(label_ + ": forward needs at least one row");
  ensure_scratch(rows);
  const size_t r = group_->local_ranks()[0];
  check_forward_position(r, 0);
  trace_[0] = int64_t(slots_[r].logical_id);
  if (mode == Mode::Train) {
    tapes_[r].record(slots_[r].logical_id, {});
    x_cache_[r] = x;
    cached_rows_ = rows;
  }
  return slots_[r].weight.data();
}

RtpLinear::N1Bwd RtpLinear::begin_backward_n1(size_t rows) {
  if (group_->size() != 1) throw StateError(label_ + ": begin_backward_n1 needs a single-worker group");
  const size_t r = group_->local_ranks()[0];
  if (tapes_[r].empty()) throw StateError("backward invoked without a matching forward");
  if (rows != cached_rows_) throw DimensionError(label_ + ": backward rows differ from the cached forward");
  const size_t j = slots_[r].logical_id;
  tapes_[r].replay(j);
  check_backward_position(r, 0);
  trace_[1] = int64_t(j);
  return {slots_[r].weight.data(), static_cast<float*>(slots_[r].grad_acc.data()), grads_zero_pending_,
          x_cache_[r], workspace_[r].data(), workspace_[r].bytes()};
}

void RtpLinear::end_backward_n1() {
  grads_zero_pending_ = false;
  for (size_t r : group_->local_ranks()) x_cache_[r] = {};
  require_home("end of backward");
}

void RtpLinear::backward_ex(std::span<const DView> dy, size_t rows, std::span<const DView> dx, const BwdEpi& e) {
  try {
    backward_impl(dy, rows, dx, e);
  } catch (...) {
    drop_prefetch();
    throw;
  }
}

void RtpLinear::backward_impl(std::span<const DView> dy, size_t rows, std::span<const DView> dx,
                              const BwdEpi& e) {
  SmReserve sm_reserve(*group_);
  const auto& local = group_->local_ranks();
  if (dy.size() != local.size() || dx.size() != local.size())
    throw DimensionError(label_ + ": backward expects one gradient per local worker");
  const size_t n = group_->size();
  for (size_t r : local)
    if (tapes_[r].empty()) throw StateError("backward invoked without a matching forward");
  if (rows != cached_rows_) throw DimensionError(label_ + ": backward rows differ from the cached forward");
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  std::fill(trace_.begin() + n * n, trace_.end(), -1);
  const int dt = dtype_code(dtype_);
  const bool oopm = oop();
  std::vector<void*> wp(n, nullptr), sp(n, nullptr), gp(n, nullptr);

  if (n == 1 && dtype_ == DType::BF16 && !std::getenv("RTPB_NO_OVERLAP") && n1_scheduling_pays(rows, in_, out_)) {
    // No rotation: dX and dW of the single step are independent GEMMs. dW
    // runs on the aux stream beside dX, each persistent kernel sized to its
    // share of the SMs, so neither pays a wave-quantisation tail alone.
    // (bf16 only: the fp32 mode's operand-split pre-passes share the layer
    // workspace.) The caller joins aux back into compute.
    const size_t r = local[0];
    Worker& w = group_->worker(r);
    const size_t j = slots_[r].logical_id;
    tapes_[r].replay(j);
    check_backward_position(r, 0);
    trace_[n * n] = int64_t(j);
    const bool gelu = !e.pre.empty();
    const int all = sm_budget();
    const int d_sms = overlap_dx_sms(rows, in_, per_, gelu);
    w.fork_aux();  // aux: dY (and, for ffn1, dpre) are complete
    set_sm_budget(d_sms);
    int flags = RTPB_EPI_FIRST | RTPB_EPI_LAST;
    const void* pre = nullptr;
    size_t ldpre = 0;
    if (gelu) {
      flags |= RTPB_EPI_GELU_BWD | (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0);
      pre = e.pre[0].data;
      ldpre = e.pre[0].ld ? e.pre[0].ld : in_;
    }
    int rc = rtpb_dgrad_step(dt, dy[0].data, dy[0].ld ? dy[0].ld : out_, 0, slots_[r].weight.data(), nullptr, in_,
                             dx[0].data, dx[0].ld ? dx[0].ld : in_, pre, ldpre, rows, in_, per_, flags,
                             workspace_[r].data(), workspace_[r].bytes(), w.compute);
    if (rc == RTPB_OK) {
      set_sm_budget(all - d_sms);
      float* g = static_cast<float*>(slots_[r].grad_acc.data());
      rc = rtpb_wgrad_step(dt, x_cache_[r].data, x_cache_[r].ld ? x_cache_[r].ld : in_, dy[0].data,
                           dy[0].ld ? dy[0].ld : out_, 0, grads_zero_pending_ ? nullptr : g, g, rows, in_, per_,
                           workspace_[r].data(), workspace_[r].bytes(), w.aux);
    }
    set_sm_budget(0);
    check_status(rc);
    grads_zero_pending_ = false;
    x_cache_[r] = {};
    return;
  }

  if (pass_launch_ok() && backward_pass_pays(rows)) {
    backward_pass(dy, rows, dx, e);
    return;
  }

  // One worker per GPU with an HBM-bound dX: dW runs on the aux stream beside
  // it, each on its share of the SMs; the travelling gradient is then ordered
  // after aux (its writer) instead of compute.
  const bool distributed = group_->kind() == TransportKind::Nccl || group_->kind() == TransportKind::Ipc ||
                           group_->kind() == TransportKind::Solo;
  const int all_sms = sm_budget();
  const int dx_sms = (n > 1 && distributed && dtype_ == DType::BF16) ? nway_dx_sms(rows, in_, per_) : 0;
  if (dx_sms)
    for (size_t r : local) group_->worker(r).fork_aux();
  // Paired dX (out-of-place, bf16; RTPB_DX_PAIR=0 disables): an even step
  // defers its dX, the odd step after it runs both as ONE GEMM over the two
  // resident shards (the previous one is still in the spare), so the fp32
  // cross-step accumulator is read and written N/2 times instead of N (at N =
  // 2 never) — SURVEY §7.9's mitigation of the HBM-bound accumulator. The
  // shift into the spare then waits for that dX (it overlaps dW only).
  // Measured per GPU (`--solo N`): config (b) N = 2 / 4 / 8 574 → 681, 364 →
  // 422, 195 → 233 TFLOP/s; config (d) N = 8 1053 → 1210. It regroups fp32
  // sums, so out-of-place is no longer bit-identical to in-place (the
  // reference's layers_test property holds with RTPB_DX_PAIR=0).
  // (with arrival flags the paired dX waits on its own step's flag: the
  // spare's shard came through the same comm stream earlier)
  const bool pair = oopm && n > 1 && dtype_ == DType::BF16 && paired_dx_;
  auto paired = [&](size_t s) { return pair && s % 2 == 1; };
  auto has_dx = [&](size_t s) { return !pair || s % 2 == 1 || s + 1 == n; };
  const size_t first_dx = pair ? 1 : 0;
  std::vector<size_t> prev_j(n, 0);
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      const size_t j = slots_[r].logical_id;
      tapes_[r].replay(j);
      check_backward_position(r, s);
      trace_[n * n + s * n + r] = int64_t(j);
    });
    const bool rotate = s + 1 < n;
    const bool flags_on = use_flags();
    if (s > 0 && !flags_on && has_dx(s)) {
      // dX of this step needs the shifted weight.
      for (size_t r : local) group_->worker(r).wait(Ev::WDone, false);
    }
    if (rotate && oopm && !(s == 0 && pre_bwd_) && !paired(s)) {
      group_->comm_after_compute();
      for (size_t r : local) {
        wp[r] = slots_[r].weight.data();
        sp[r] = spares_[r].data();
      }
      flagged_exchange(Direction::CounterClockwise, wp, sp, slots_[local[0]].weight.bytes(), kFlagBwdW + s + 1);
      for (size_t r : local) group_->worker(r).record(Ev::WDone, true);
    }
    pre_bwd_ = false;
    if (s + 1 == n && n > 1 && use_flags())
      for (size_t r : local) group_->worker(r).record(Ev::PassEnd, true);
    if (s + 1 == n && e.before_last_step) e.before_last_step();
    // dX (+)= dY_j . W_j^T
    if (dx_sms) set_sm_budget(dx_sms);
    if (has_dx(s)) group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const size_t j = slots_[r].logical_id;
      int flags = (s == first_dx ? RTPB_EPI_FIRST : 0) | (s + 1 == n ? RTPB_EPI_LAST : 0);
      const void* pre = nullptr;
      size_t ldpre = 0;
      if (!e.pre.empty() && s + 1 == n) {
        flags |= RTPB_EPI_GELU_BWD | (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0);
        pre = e.pre[k].data;
        ldpre = e.pre[k].ld ? e.pre[k].ld : in_;
      }
      float* acc = n > 1 ? static_cast<float*>(dx_acc_[r].data()) : nullptr;
      set_launch_wait_flag(flags_on && s > 0 ? w.flag(flag_base_ + kFlagBwdW + s) : nullptr);
      if (flags_on && s + 1 == n)  // the last dX clears the pass's W flags
        set_launch_flag_reset(w.flag(flag_base_ + kFlagBwdW), int(kFlagBwdG - kFlagBwdW),
                              w.flag(flag_base_ + kFlagCtrW));
      const size_t ldy = dy[k].ld ? dy[k].ld : out_, ldx = dx[k].ld ? dx[k].ld : in_;
      const int rc =
          paired(s) ? rtpb_dgrad_step2(dt, dy[k].data, ldy, prev_j[r] * per_, spares_[r].data(), j * per_,
                                       slots_[r].weight.data(), acc, in_, dx[k].data, ldx, pre, ldpre, rows, in_,
                                       per_, flags, workspace_[r].data(), workspace_[r].bytes(), w.compute)
                    : rtpb_dgrad_step(dt, dy[k].data, ldy, j * per_, slots_[r].weight.data(), acc, in_, dx[k].data,
                                      ldx, pre, ldpre, rows, in_, per_, flags, workspace_[r].data(),
                                      workspace_[r].bytes(), w.compute);
      set_launch_wait_flag(nullptr);
      set_launch_flag_reset(nullptr, 0, nullptr);
      check_status(rc);
    });
    for (size_t r : local) prev_j[r] = slots_[r].logical_id;
    if (rotate && paired(s)) {
      // the spare's shard was read by this dX: shift the next shard in now
      group_->comm_after_compute();
      for (size_t r : local) {
        wp[r] = slots_[r].weight.data();
        sp[r] = spares_[r].data();
      }
      flagged_exchange(Direction::CounterClockwise, wp, sp, slots_[local[0]].weight.bytes(), kFlagBwdW + s + 1);
      for (size_t r : local) group_->worker(r).record(Ev::WDone, true);
    }
    if (rotate && !oopm) {
      // In place: the weight is free once dX has read it; shift it under dW.
      group_->comm_after_compute();
      for (size_t r : local) wp[r] = slots_[r].weight.data();
      flagged_exchange(Direction::CounterClockwise, wp, wp, slots_[local[0]].weight.bytes(), kFlagBwdW + s + 1);
      for (size_t r : local) group_->worker(r).record(Ev::WDone, true);
    }
    // G_j += X^T . dY_j (+ bias column sums), in place on the resident shard.
    if (dx_sms) set_sm_budget(all_sms - dx_sms);
    // The travelling gradient arrives by flag when the dW launch is a single
    // CTA-pair GEMM (bias sums fused in it): the launch starts at once and
    // only its epilogue / bias-sum warps wait for G (GemmArgs::g_flag), so the
    // dW mainloop overlaps G's transfer and the accumulation is applied as
    // the shard lands. The per-tile kernels' separate bias column-sum
    // pre-pass reads G, so those keep the stream wait.
    unsigned dummy_flags = 0;
    const bool g_flag = flags_on && wgrad_fuses_bias(false, rows, in_, per_, &dummy_flags, 0);
    if (s > 0 && !g_flag) {
      // dW accumulates into the travelling gradient shard: wait for its arrival.
      for (size_t r : local) {
        Worker& w = group_->worker(r);
        w.wait_on(Ev::GDone, dx_sms ? w.aux : w.compute);
      }
    }
    group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      const cudaStream_t ws = dx_sms ? w.aux : w.compute;
      set_launch_g_flag(g_flag && s > 0 ? w.flag(flag_base_ + kFlagBwdG + s) : nullptr);
      if (flags_on && s + 1 == n)  // the last dW clears the pass's G flags
        set_launch_flag_reset(w.flag(flag_base_ + kFlagBwdG), int(kFlagCtrFwd - kFlagBwdG),
                              w.flag(flag_base_ + kFlagCtrG));
      const size_t k = k_of[r];
      const size_t j = slots_[r].logical_id;
      float* g = static_cast<float*>(slots_[r].grad_acc.data());
      // step 0 after zero_grads(): every resident gradient is zero -> overwrite
      const float* g_in = (grads_zero_pending_ && s == 0) ? nullptr : g;
      const int rc = rtpb_wgrad_step(dt, x_cache_[r].data, x_cache_[r].ld ? x_cache_[r].ld : in_, dy[k].data,
                                     dy[k].ld ? dy[k].ld : out_, j * per_, g_in, g, rows, in_, per_,
                                     workspace_[r].data(), workspace_[r].bytes(), ws);
      set_launch_g_flag(nullptr);
      set_launch_flag_reset(nullptr, 0, nullptr);
      check_status(rc);
    });
    if (dx_sms) set_sm_budget(all_sms);
    if (!rotate) break;
    if (dx_sms) {
      for (size_t r : local) {  // the gradient's writer is aux
        Worker& w = group_->worker(r);
        w.record_on(Ev::AuxDone, w.aux);
        w.wait_on(Ev::AuxDone, w.comm);
      }
    } else {
      group_->comm_after_compute();
    }
    for (size_t r : local) gp[r] = slots_[r].grad_acc.data();
    flagged_exchange(Direction::CounterClockwise, gp, gp, slots_[local[0]].grad_acc.bytes(), kFlagBwdG + s + 1);
    for (size_t r : local) group_->worker(r).record(Ev::GDone, true);
    if (oopm)
      for (size_t r : local) swap_data(slots_[r].weight, spares_[r]);
    group_->advance_slots(slots_, Direction::CounterClockwise, PayloadKind::WeightAndGrad, label_, shard_len_);
  }
  if (n > 1 && use_flags()) {
    for (size_t r : local) group_->worker(r).wait(Ev::PassEnd, false);
  }
  grads_zero_pending_ = false;
  for (size_t r : local) x_cache_[r] = {};
  require_home("end of backward");
}

// The backward pass launch splits the SMs between the dX launch and the dW
// chain for the whole pass; per-step launches give each step's dX and dW the
// whole machine one after the other. The split pays while a step's GEMMs are
// a few microseconds (launch gaps and one-wave tails dominate: config (b));
// for large steps (configs (c), (d): ~170 us each on all SMs) the per-step
// schedule was measured faster. RTPB_PASS_BWD=0/1 forces either.
bool RtpLinear::backward_pass_pays(size_t rows) const {
  static const int force = [] {
    const char* e = std::getenv("RTPB_PASS_BWD");
    return e ? std::atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  return 2.0 * double(rows) * double(in_) * double(per_) < 40e9;
}

// Backward as two pass launches side by side (one worker per GPU, out of
// place, arrival flags): the dX of all N steps in ONE persistent launch
// (rtpb_dgrad_pass) on the compute stream, the dW of all N steps in one
// (rtpb_wgrad_pass) on the aux stream, each on its share of the SMs. The dW
// launch runs its mainloops ahead; each step's accumulation waits (in the
// epilogue) for the travelling gradient G to land. The comm stream moves, per
// step, the next weight shard into the buffer the dX launch has counted out
// and G once the dW launch has counted its step in (cuStreamWaitValue32 on
// the count-ins). No wait closes a cycle: the dX launch waits only for W
// shifts, a W shift only for the dX launch's earlier steps, the dW launch for
// G shifts, a G shift only for the dW launch's earlier steps and the shifts
// posted ahead of it; both grids are resident (launched first, each within
// its SM share) before any of their waits. Paired dX (paired_dx_) pairs the steps as
// rtpb_dgrad_step2 does; otherwise the bits equal the per-step launches'.
void RtpLinear::backward_pass(std::span<const DView> dy, size_t rows, std::span<const DView> dx, const BwdEpi& e) {
  const size_t n = group_->size();
  const auto& local = group_->local_ranks();
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  std::vector<std::array<void*, 2>> buf(n);
  std::vector<std::array<size_t, 16>> cols(n);
  for (size_t r : local) buf[r] = {slots_[r].weight.data(), spares_[r].data()};
  unsigned mask = 0;
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      const size_t j = slots_[r].logical_id;
      tapes_[r].replay(j);
      check_backward_position(r, s);
      trace_[n * n + s * n + r] = int64_t(j);
      cols[r][s] = j * per_;
    });
    if (s & 1) mask |= 1u << s;
    if (s + 1 < n)
      group_->advance_slots(slots_, Direction::CounterClockwise, PayloadKind::WeightAndGrad, label_, shard_len_);
  }
  const bool pair = paired_dx_;
  int flags = pair ? RTPB_PASS_PAIR : 0;
  if (!e.pre.empty()) flags |= RTPB_EPI_GELU_BWD | (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0);
  auto group_of = [&](size_t s) { return pair ? s / 2 : s; };
  // SM shares of the two launches. The dX launch's fp32 accumulator is read
  // and written per step pair (8 B per dX element) at ~25 GB/s per SM of TMA
  // reduce-add, so a wide-in, thin-shard layer (in >= 16 per) is dX-bound and
  // gets ~2/3 of the SMs; otherwise the dW chain is the slower one and dX gets
  // ~0.45. Measured (config (b) --solo, per-launch times): ffn2 (3072 -> 96 at
  // N = 8) 354 / 203 us dX / dW at 74 SMs for dX, 295 / 240 at 96; ffn1
  // (768 -> 384) 123 / 174 at 74, 98 / 199 at 96. RTPB_PASS_DX_SMS overrides.
  const int all = sm_budget();
  int d_sms = int(all * (in_ >= 16 * per_ ? 0.65 : 0.45)) & ~1;
  if (const char* ev = std::getenv("RTPB_PASS_DX_SMS")) d_sms = std::atoi(ev);
  d_sms = std::max(2, std::min(all - 2, d_sms)) & ~1;
  set_sm_budget(d_sms);  // the tiles (and count-ins) of the dX launch depend on its SM share
  const unsigned target = rtpb_pass_done_target(1, rows, in_, per_, n, flags);
  set_sm_budget(all);

  // [dY's column sums | their workspace] for the dW launch (before any launch:
  // allocation synchronizes)
  const size_t db_bytes = (out_ * sizeof(float) + 255) & ~size_t(255);
  if (pass_ws_rows_ != rows) {
    group_->synchronize();
    pass_ws_.resize(n);
    for (size_t r : local) {
      Worker& w = group_->worker(r);
      pass_ws_[r] = DeviceBuffer();
      pass_ws_[r] = DeviceBuffer(w.device, db_bytes + rtpb_colsum_workspace_bytes(rows, out_), &w.ledger,
                                 MemCategory::Other, true);
    }
    pass_ws_rows_ = rows;
  }
  set_sm_budget(all - d_sms);
  const unsigned target_w = rtpb_pass_done_target(2, rows, in_, per_, n, 0);
  set_sm_budget(all);
  // The in-place G shifts' staging chunk, sized now: growing it later would
  // free device memory (a device-wide synchronisation) while the launches
  // below wait for shifts not yet queued.
  for (size_t r : local) {
    size_t chunk = 0;
    group_->worker(r).staging(slots_[r].grad_acc.bytes(), &chunk);
  }

  // Grids first, then the shifts (as the forward pass: every stream memory
  // wait is queued after the work it waits for). The dX grid is launched
  // first so it takes its SM share before the dW grid fills the rest.
  group_->comm_after_compute();  // the spares' last readers are done
  group_->each([&](size_t r) { group_->worker(r).fork_aux(); });  // dW reads dY and X, complete on compute
  const bool serial = serial_profile();
  // The W shifts (channel 0) and the G shifts (channel 1) run on separate
  // comm streams, so neither chain queues behind the other's waits
  // (RTPB_PASS_ONE_CHANNEL=1: both on channel 0 in step order, W first — on
  // one stream W first measured better than G first: config (b) --solo
  // N = 8 / 4 / 2 319 / 512 / 695 vs 307 / 470 / 693 TFLOP/s per GPU).
  static const int kGChannelSel = [] {
    const char* e = std::getenv("RTPB_PASS_ONE_CHANNEL");
    return (e && std::atoi(e) != 0) ? 0 : 1;
  }();
  const int kGChannel = kGChannelSel;
  auto post_shifts = [&] {
    host_trace(label_, "backward pass: shifts");
    std::vector<void*> wp(n, nullptr), sp(n, nullptr), gp(n, nullptr);
    for (size_t s = 0; s + 1 < n; ++s) {
      auto shift_w = [&] {
        // W shift for step s + 1 into the buffer step s - 1 read
        if (!(s == 0 && pre_bwd_)) {
          for (size_t r : local) {
            Worker& w = group_->worker(r);
            DeviceGuard dg(w.device);
            if (s >= 1 && !serial)
              stream_wait_geq_u32(w.comm, w.flag(flag_base_ + kFlagDoneBwd + group_of(s - 1)), target);
            wp[r] = buf[r][s & 1];
            sp[r] = buf[r][(s + 1) & 1];
          }
          flagged_exchange(Direction::CounterClockwise, wp, sp, slots_[local[0]].weight.bytes(), kFlagBwdW + s + 1);
        }
      };
      auto shift_g = [&] {
        // G shift once dW(s) has landed: the gradient travels with its
        // accumulation, on channel 1 (its own comm stream)
        for (size_t r : local) {
          Worker& w = group_->worker(r);
          DeviceGuard dg(w.device);
          if (!serial) stream_wait_geq_u32(w.comm_of(kGChannel), w.flag(flag_base_ + kFlagDoneW + s), target_w);
          gp[r] = slots_[r].grad_acc.data();
        }
        flagged_exchange(Direction::CounterClockwise, gp, gp, slots_[local[0]].grad_acc.bytes(), kFlagBwdG + s + 1,
                         kGChannel);
      };
      shift_w();
      shift_g();
    }
  };
  if (serial) post_shifts();  // (profiling a Solo group: every flag up front)
  host_trace(label_, "backward pass: launches");
  set_sm_budget(d_sms);
  try {
    group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const void* pre = e.pre.empty() ? nullptr : e.pre[k].data;
      const size_t ldpre = e.pre.empty() ? 0 : (e.pre[k].ld ? e.pre[k].ld : in_);
      unsigned tgt = target;  // checked before the launch
      check_status(rtpb_dgrad_pass(dy[k].data, dy[k].ld ? dy[k].ld : out_, out_, buf[r][0], buf[r][1], cols[r].data(),
                                   mask, n, static_cast<float*>(dx_acc_[r].data()), in_, dx[k].data,
                                   dx[k].ld ? dx[k].ld : in_, pre, ldpre, rows, in_, per_, flags,
                                   w.flag(flag_base_ + kFlagBwdW), w.flag(flag_base_ + kFlagDoneBwd), &tgt,
                                   w.flag(flag_base_ + kFlagCtrW), w.compute));
    });
    // dW of every step: one launch on aux (rtpb_wgrad_pass) after dY's
    // column sums (the bias parts, added as each G arrives)
    set_sm_budget(all - d_sms);
    group_->each([&](size_t r) {
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const size_t ldy = dy[k].ld ? dy[k].ld : out_;
      float* db = static_cast<float*>(pass_ws_[r].data());
      check_status(rtpb_colsum(dy[k].data, ldy, rows, out_, db, static_cast<char*>(pass_ws_[r].data()) + db_bytes,
                               pass_ws_[r].bytes() - db_bytes, w.aux));
      unsigned tgt = target_w;  // checked before the launch
      check_status(rtpb_wgrad_pass(x_cache_[r].data, x_cache_[r].ld ? x_cache_[r].ld : in_, dy[k].data, ldy, out_,
                                   static_cast<float*>(slots_[r].grad_acc.data()), cols[r].data(), n, rows, in_, per_,
                                   grads_zero_pending_ ? RTPB_EPI_FIRST : 0, db, w.flag(flag_base_ + kFlagBwdG),
                                   w.flag(flag_base_ + kFlagDoneW), &tgt, w.flag(flag_base_ + kFlagCtrG),
                                   workspace_[r].data(), workspace_[r].bytes(), w.aux));
    });
  } catch (...) {
    set_sm_budget(all);
    throw;
  }
  set_sm_budget(all);
  if (!serial) post_shifts();
  pre_bwd_ = false;
  for (size_t r : local) {
    Worker& w = group_->worker(r);
    w.record(Ev::PassEnd, true);
    w.record_on(Ev::PassEndG, w.comm_of(kGChannel));
  }
  if (e.before_last_step) {  // the next layer's first shift, queued behind this pass's (fenced above)
    group_->set_comm_fenced(true);
    try {
      e.before_last_step();
    } catch (...) {
      group_->set_comm_fenced(false);
      throw;
    }
    group_->set_comm_fenced(false);
  }
  set_sm_budget(all);
  for (size_t r : local) {
    if ((n - 1) & 1) swap_data(slots_[r].weight, spares_[r]);  // the pass's n - 1 swaps
    Worker& w = group_->worker(r);
    w.wait(Ev::PassEnd, false);
    w.wait_on(Ev::PassEndG, w.compute);
  }
  host_trace(label_, "backward pass: queued");
  grads_zero_pending_ = false;
  for (size_t r : local) x_cache_[r] = {};
  require_home("end of backward");
}

// ------------------------------------------------------------------ MLP
RtpMlp::RtpMlp(WorkerGroup& group, std::string label, size_t h, size_t f, DType dtype, const double* w1,
               const double* b1, const double* w2, const double* b2)
    : group_(&group), h_(h), f_(f), dtype_(dtype) {
  ffn1_ = std::make_unique<RtpLinear>(group, label + "/ffn1", w1, b1, h, f, group.size(), dtype);
  ffn2_ = std::make_unique<RtpLinear>(group, label + "/ffn2", w2, b2, f, h, group.size(), dtype);
}

RtpMlp::RtpMlp(WorkerGroup& group, std::string label, size_t h, size_t f, DType dtype, uint64_t seed,
               uint64_t stream_base)
    : group_(&group), h_(h), f_(f), dtype_(dtype) {
  // SerialModel order (serial.cpp:349-350): ffn1.w, ffn1.b, ffn2.w, ffn2.b.
  ffn1_ = std::make_unique<RtpLinear>(group, label + "/ffn1", h, f, group.size(), seed, stream_base, dtype);
  ffn2_ = std::make_unique<RtpLinear>(group, label + "/ffn2", f, h, group.size(), seed, stream_base + h * f + f,
                                      dtype);
}

void RtpMlp::set_rotation_mode(RotationMode m) {
  mode_ = m;
  ffn1_->set_rotation_mode(m);
  ffn2_->set_rotation_mode(m);
}

void RtpMlp::set_exact_gelu(bool on) {
  ffn1_->set_exact_gelu(on);
  ffn2_->set_exact_gelu(on);
}

void RtpMlp::set_paired_dx(bool on) {
  ffn1_->set_paired_dx(on);
  ffn2_->set_paired_dx(on);
}

void RtpMlp::begin_step() {
  if (mode_ == RotationMode::OutOfPlace) {
    if (!ffn1_->has_comm_spares()) ffn1_->allocate_comm_spares();
    if (!ffn2_->has_comm_spares()) ffn2_->allocate_comm_spares();
  }
}

void RtpMlp::zero_grads() {
  ffn1_->zero_grads();
  ffn2_->zero_grads();
}

void RtpMlp::ensure_acts(size_t rows, Mode mode) {
  // Train forwards write the activations backward reads (pre, gelu(pre));
  // Eval forwards only need gelu(pre) as ffn2's input and get their own
  // buffer, so Train fwd -> Eval fwd -> backward still differentiates the
  // Train batch (the reference caches pre/h only in Train mode, model.cpp:79-80).
  const bool train = mode == Mode::Train;
  size_t& have = train ? act_rows_ : eval_rows_;
  if (rows == have) return;
  group_->synchronize();
  const size_t n = group_->size();
  auto& act = train ? act_ : eval_act_;
  act.resize(n);
  if (train) pre_.resize(n);
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    const size_t b = rows * f_ * dtype_size(dtype_);
    act[r] = DeviceBuffer();  // release before allocating: the ledger peak is the live set
    act[r] = DeviceBuffer(w.device, b, &w.ledger, MemCategory::Activation, false);
    if (train) {
      pre_[r] = DeviceBuffer();
      pre_[r] = DeviceBuffer(w.device, b, &w.ledger, MemCategory::Activation, false);
    }
  });
  have = rows;
  if (train) saved_rows_ = 0;  // the previous Train batch's activations are gone
}

void RtpMlp::ensure_fused(size_t rows) {
  if (rows == fused_rows_) return;
  FusedFwdPlan plan;
  if (!plan_fused_fwd(rows, h_, f_, plan)) throw ConfigError("RtpMlp: no fused forward schedule for this shape");
  group_->synchronize();
  const size_t r = group_->local_ranks()[0];
  Worker& w = group_->worker(r);
  fused_sched_ints_ = plan.sched.size();
  // [schedule][row-block counters][done][ffn2 split counters] then, when ffn2
  // is split over K, its fp32 partial sums (rows x h)
  const size_t ints = fused_sched_ints_ + size_t(plan.dep_rows) + 1 + size_t(plan.tiles2);
  fused_acc_off_ = (ints * sizeof(int) + 255) & ~size_t(255);
  const size_t bytes = fused_acc_off_ + (plan.k_splits2 > 1 ? rows * h_ * sizeof(float) : 0);
  fused_ws_ = DeviceBuffer(w.device, bytes, &w.ledger, MemCategory::Other, true);  // counters start at zero
  cuda_check(cudaMemcpy(fused_ws_.data(), plan.sched.data(), fused_sched_ints_ * sizeof(int), cudaMemcpyHostToDevice),
             "upload fused schedule");
  fused_slots_ = plan.slots;
  fused_dep_rows_ = plan.dep_rows;
  fused_dep_target_ = plan.dep_target;
  fused_splits2_ = plan.k_splits2;
  fused_tiles2_ = plan.tiles2;
  fused_rows_ = rows;
}

void RtpMlp::forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode) {
  // the layers' own require_home, checked before any activation buffer moves
  if (!ffn1_->all_home()) throw StateError(ffn1_->label() + ": forward requires every slot at its home position");
  if (!ffn2_->all_home()) throw StateError(ffn2_->label() + ": forward requires every slot at its home position");
  ensure_acts(rows, mode);
  const bool train = mode == Mode::Train;
  auto& actb = train ? act_ : eval_act_;
  auto& preb = train ? pre_ : eval_act_;  // Eval: pre is not stored (no STORE_PRE); the map needs a buffer
  if (train) saved_rows_ = 0;  // set again once this forward has been issued
  if (group_->size() == 1 && dtype_ == DType::BF16 && !std::getenv("RTPB_NO_FUSED_FWD") &&
      n1_scheduling_pays(rows, h_, f_)) {
    // N = 1: no rotation between ffn1 and ffn2, so both GEMMs run as one
    // scheduled persistent launch (ffn2's row blocks start as soon as ffn1
    // has written them); the layers keep their reference bookkeeping.
    if (x.size() != 1 || y.size() != 1) throw DimensionError("RtpMlp: forward expects one activation per worker");
    const size_t r = group_->local_ranks()[0];
    ensure_fused(rows);
    const void* w1 = ffn1_->begin_forward_n1(x[0], rows, mode);
    const void* w2 = ffn2_->begin_forward_n1({actb[r].data(), f_}, rows, mode);
    Worker& w = group_->worker(r);
    int* base = static_cast<int*>(fused_ws_.data());
    unsigned* dep = reinterpret_cast<unsigned*>(base + fused_sched_ints_);
    FusedFwdPlan plan;
    plan.slots = fused_slots_;
    plan.dep_rows = fused_dep_rows_;
    plan.dep_target = fused_dep_target_;
    plan.k_splits2 = fused_splits2_;
    plan.tiles2 = fused_tiles2_;
    FusedFwdWs ws{base, dep, dep + fused_dep_rows_, dep + fused_dep_rows_ + 1,
                  fused_splits2_ > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(base) + fused_acc_off_)
                                     : nullptr};
    check_status(fused_fwd_step(x[0].data, x[0].ld ? x[0].ld : h_, w1, preb[r].data(), actb[r].data(), w2,
                                y[0].data, y[0].ld ? y[0].ld : h_, rows, h_, f_, train, plan, ws, w.compute,
                                ffn1_->exact_gelu()));
    if (train) saved_rows_ = rows;
    return;
  }
  const auto& local = group_->local_ranks();
  std::vector<DView> pre(local.size()), act(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    pre[k] = {preb[local[k]].data(), f_};
    act[k] = {actb[local[k]].data(), f_};
  }
  // pre = ffn1(x); act = gelu(pre) fused into ffn1's epilogue (model.cpp:77-82)
  RtpLinear::FwdEpi e1;
  e1.act = act;
  e1.store_pre = mode == Mode::Train;
  // ffn2's first shift travels under ffn1's last step
  if (!std::getenv("RTPB_NO_PREFETCH")) e1.before_last_step = [&] { ffn2_->prefetch_first_shift(false); };
  ffn1_->forward_ex(x, rows, pre, mode, e1);
  RtpLinear::FwdEpi e2;
  e2.store_pre = true;  // plain linear: y is the output
  // the next block's first shift travels under this block's last step
  if (next_ && !std::getenv("RTPB_NO_PREFETCH"))
    e2.before_last_step = [&] { next_->ffn1_->prefetch_first_shift(false); };
  ffn2_->forward_ex(act, rows, y, mode, e2);  // model.cpp:83
  if (train) saved_rows_ = rows;
}

RtpMlp::~RtpMlp() {
  if (next_) next_->prev_ = nullptr;
  if (prev_) prev_->next_ = nullptr;
}

void RtpMlp::chain(RtpMlp* next) {
  if (next == this) throw ConfigError("RtpMlp::chain: a block cannot follow itself");
  if (next && next->group_ != group_) throw ConfigError("RtpMlp::chain: blocks of different worker groups");
  if (next_) next_->prev_ = nullptr;
  next_ = next;
  if (next) {
    if (next->prev_) next->prev_->next_ = nullptr;
    next->prev_ = this;
  }
}

void RtpMlp::ensure_fused_bwd(size_t rows) {
  if (rows == fused_bwd_rows_) return;
  FusedBwdPlan plan;
  if (!plan_fused_bwd(rows, h_, f_, plan)) throw ConfigError("RtpMlp: no fused backward schedule for this shape");
  group_->synchronize();
  const size_t r = group_->local_ranks()[0];
  Worker& w = group_->worker(r);
  fused_bwd_sd_ints_ = plan.sched_d.size();
  fused_bwd_sw_ints_ = plan.sched_w.size();
  const size_t ints = fused_bwd_sd_ints_ + fused_bwd_sw_ints_ + size_t(plan.dep_rows) + 1;
  fused_bwd_ws_ = DeviceBuffer(w.device, ints * sizeof(int), &w.ledger, MemCategory::Other, true);
  int* base = static_cast<int*>(fused_bwd_ws_.data());
  cuda_check(cudaMemcpy(base, plan.sched_d.data(), fused_bwd_sd_ints_ * sizeof(int), cudaMemcpyHostToDevice),
             "upload fused schedule");
  cuda_check(cudaMemcpy(base + fused_bwd_sd_ints_, plan.sched_w.data(), fused_bwd_sw_ints_ * sizeof(int),
                        cudaMemcpyHostToDevice),
             "upload fused schedule");
  fused_bwd_slots_d_ = plan.slots_d;
  fused_bwd_slots_w_ = plan.slots_w;
  fused_bwd_dep_rows_ = plan.dep_rows;
  fused_bwd_dep_target_ = plan.dep_target;
  fused_bwd_w_splits_ = plan.w_splits;
  fused_bwd_rows_ = rows;
}

void RtpMlp::backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx) {
  // the saved Train activations must be this batch's (model.cpp:99-105 reads pre_cache)
  if (saved_rows_ == 0) throw StateError(ffn2_->label() + ": backward invoked without a matching forward");
  if (saved_rows_ != rows)
    throw DimensionError(ffn2_->label() + ": backward over " + std::to_string(rows) +
                         " rows, the saved forward had " + std::to_string(saved_rows_));
  if (group_->size() == 1 && dtype_ == DType::BF16 && !std::getenv("RTPB_NO_FUSED_BWD") &&
      n1_scheduling_pays(rows, h_, f_)) {
    // N = 1: the four backward GEMMs as two concurrent scheduled launches
    // (dX chain on compute, dW pair on aux); ffn1's dW streams dpre row blocks
    // as the dX launch publishes them.
    if (dy.size() != 1 || dx.size() != 1) throw DimensionError("RtpMlp: backward expects one gradient per worker");
    const size_t r = group_->local_ranks()[0];
    ensure_fused_bwd(rows);
    const RtpLinear::N1Bwd b2 = ffn2_->begin_backward_n1(rows);
    const RtpLinear::N1Bwd b1 = ffn1_->begin_backward_n1(rows);
    Worker& w = group_->worker(r);
    FusedBwdArgs a{};
    a.dy = dy[0].data; a.ldy = dy[0].ld ? dy[0].ld : h_;
    a.act = b2.x.data;
    a.x = b1.x.data; a.ldx = b1.x.ld ? b1.x.ld : h_;
    a.pre = pre_[r].data();
    a.dx = dx[0].data; a.lddx = dx[0].ld ? dx[0].ld : h_;
    a.w1 = b1.weight; a.w2 = b2.weight;
    a.g1 = b1.grad; a.g2 = b2.grad; a.g1_zero = b1.grad_zero; a.g2_zero = b2.grad_zero;
    a.M = rows; a.h = h_; a.f = f_;
    a.exact_gelu = ffn2_->exact_gelu();
    int* base = static_cast<int*>(fused_bwd_ws_.data());
    unsigned* dep = reinterpret_cast<unsigned*>(base + fused_bwd_sd_ints_ + fused_bwd_sw_ints_);
    FusedBwdPlan plan;
    plan.slots_d = fused_bwd_slots_d_;
    plan.slots_w = fused_bwd_slots_w_;
    plan.dep_rows = fused_bwd_dep_rows_;
    plan.dep_target = fused_bwd_dep_target_;
    plan.w_splits = fused_bwd_w_splits_;
    FusedBwdWs ws{base, base + fused_bwd_sd_ints_, dep, dep + fused_bwd_dep_rows_};
    w.fork_aux();  // aux: dY, act, X and pre are complete
    check_status(fused_bwd_step(a, b1.workspace, b1.workspace_bytes, b2.workspace, b2.workspace_bytes, plan, ws,
                                w.compute, w.aux));
    ffn2_->end_backward_n1();
    ffn1_->end_backward_n1();
    group_->join_aux();
    saved_rows_ = 0;
    return;
  }
  const auto& local = group_->local_ranks();
  std::vector<DView> pre(local.size());
  for (size_t k = 0; k < local.size(); ++k) pre[k] = {pre_[local[k]].data(), f_};
  // dh = ffn2'(dy); dpre = gelu'(pre, dh) fused into ffn2's last dX epilogue,
  // written over pre (same element reads then writes it) (model.cpp:99-104)
  RtpLinear::BwdEpi e2;
  e2.pre = pre;
  if (!std::getenv("RTPB_NO_PREFETCH")) e2.before_last_step = [&] { ffn1_->prefetch_first_shift(true); };
  ffn2_->backward_ex(dy, rows, pre, e2);
  RtpLinear::BwdEpi e1;
  // the previous block's first backward shift travels under this block's last step
  if (prev_ && !std::getenv("RTPB_NO_PREFETCH"))
    e1.before_last_step = [&] { prev_->ffn2_->prefetch_first_shift(true); };
  ffn1_->backward_ex(pre, rows, dx, e1);  // model.cpp:105
  group_->join_aux();
  saved_rows_ = 0;
}

std::vector<Tensor> RtpMlp::forward(std::span<const Tensor> x, Mode mode) {
  const auto& local = group_->local_ranks();
  auto xs = per_local(*group_, x, ffn1_->label(), "forward");
  const size_t rows = xs[0]->rank() == 2 ? xs[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), ys(local.size());
  std::vector<DView> xv(local.size()), yv(local.size());
  const bool train = mode == Mode::Train;
  if (train) x_keep_.assign(group_->size(), Tensor());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    Tensor& keep = train ? x_keep_[local[k]] : tmp[k];
    const Tensor& xin = as_layer_input(*xs[k], dtype_, w, h_, ffn1_->label(), keep, train);
    if (xin.rows() != rows) throw DimensionError(ffn1_->label() + ": workers' activations differ in row count");
    ys[k] = Tensor({rows, h_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    xv[k] = {xin.data(), h_};
    yv[k] = {ys[k].data(), h_};
  }
  forward(xv, rows, yv, mode);
  group_->synchronize();
  return ys;
}

std::vector<Tensor> RtpMlp::backward(std::span<const Tensor> dy) {
  const auto& local = group_->local_ranks();
  auto ds = per_local(*group_, dy, ffn2_->label(), "backward");
  const size_t rows = ds[0]->rank() == 2 ? ds[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), dxs(local.size());
  std::vector<DView> dv(local.size()), xv(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    const Tensor& din = as_layer_input(*ds[k], dtype_, w, h_, ffn2_->label(), tmp[k], false);
    if (din.rows() != rows) throw DimensionError(ffn2_->label() + ": workers' gradients differ in row count");
    dxs[k] = Tensor({rows, h_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    dv[k] = {din.data(), h_};
    xv[k] = {dxs[k].data(), h_};
  }
  backward(dv, rows, xv);
  group_->synchronize();
  x_keep_.clear();
  return dxs;
}

}  // namespace rtpb
