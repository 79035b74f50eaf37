// RtpAttention on the device (layers_attention.cpp:43-198): head-partitioned
// multi-head attention whose shards rotate like RtpLinear's. Every product of
// a rotation step is one of the three step kernels (rtpb.h layer 1) or the
// attention core (kernels/attention.cu); the schedule, tape, position laws
// and rotations are RtpLayerBase's.
#include <cmath>
#include <cstring>

#include "kernels/launch.hpp"
#include "worker.hpp"

namespace rtpb {

ShardLayout layout_attention(size_t hidden, size_t heads, size_t n) {
  if (n == 0) throw ConfigError("layout_attention: shard count must be >= 1");
  if (heads == 0 || hidden % heads != 0)
    throw ConfigError("layout_attention: hidden " + std::to_string(hidden) + " not divisible by " +
                      std::to_string(heads) + " heads");
  if (heads % n != 0)
    throw ConfigError("layout_attention: " + std::to_string(heads) + " heads not divisible by " + std::to_string(n) +
                      " shards; choose a head count that is a multiple of the worker count");
  ShardLayout l;
  l.strategy = PartitionStrategy::HeadPartition;
  l.n_shards = n;
  const size_t per = heads / n;
  for (size_t j = 0; j < n; ++j) l.ranges.push_back({j * per, (j + 1) * per});
  return l;
}

namespace {
int dcode(DType d) { return d == DType::F32 ? RTPB_F32 : RTPB_BF16; }
}  // namespace

RtpAttention::RtpAttention(WorkerGroup& group, std::string label, const double* wq, const double* wk,
                           const double* wv, const double* wo, size_t hidden, size_t heads, size_t seq, size_t n,
                           DType dtype)
    : RtpLayerBase(group, std::move(label), dtype), hidden_(hidden), heads_(heads), seq_(seq) {
  if (n != group_->size())
    throw ConfigError("RtpAttention: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  if (dtype != DType::BF16 && dtype != DType::F32) throw ConfigError("RtpAttention: layers compute in BF16 or F32");
  init(wq, wk, wv, wo);
}

RtpAttention::RtpAttention(WorkerGroup& group, std::string label, const Tensor& wq, const Tensor& wk,
                           const Tensor& wv, const Tensor& wo, size_t heads, size_t seq, size_t n)
    : RtpLayerBase(group, std::move(label), wq.dtype() == DType::BF16 ? DType::BF16 : DType::F32),
      hidden_(wq.rank() == 2 ? wq.rows() : 0),
      heads_(heads),
      seq_(seq) {
  for (const Tensor* t : {&wq, &wk, &wv, &wo})
    if (t->rank() != 2 || t->rows() != hidden_ || t->cols() != hidden_)
      throw DimensionError(label_ + ": projection weights must be hidden x hidden, got " + t->shape_str());
  if (n != group_->size())
    throw ConfigError("RtpAttention: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  const auto q = wq.to_host(), k = wk.to_host(), v = wv.to_host(), o = wo.to_host();
  init(q.data(), k.data(), v.data(), o.data());
}

void RtpAttention::init(const double* wq, const double* wk, const double* wv, const double* wo) {
  const size_t n = group_->size();
  layout_ = layout_attention(hidden_, heads_, n);
  if (seq_ == 0) throw ConfigError(label_ + ": sequence length must be positive");
  hd_ = hidden_ / heads_;
  g_ = heads_ / n;
  gw_ = g_ * hd_;
  if (hidden_ % 8 || gw_ % 8)
    throw ConfigError("RtpAttention " + label_ + ": hidden and the head-group width (heads/N * head_dim) must be "
                      "multiples of 8 on the device path (16-byte TMA rows)");
  if (hd_ > 256) throw ConfigError("RtpAttention " + label_ + ": head_dim above 256");
  shard_len_ = 4 * hidden_ * gw_;
  init_slots_alloc();
  tapes_.assign(n, {});
  x_cache_.assign(n, {});
  saved_.resize(n);
  lse_.resize(n);
  scratch_.resize(n);
  acc_.resize(n);
  trace_.assign(2 * n * n, -1);
  // attention_shard_groups + flatten (layers_common.cpp:54-74): shard j =
  // [wq[:, j*gw:+gw] | wk[..] | wv[..] | wo[j*gw:+gw, :]], the last block
  // stored transposed (hidden x gw) on the device.
  const size_t H = hidden_, gw = gw_;
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    DeviceGuard dg(w.device);
    std::vector<double> host(shard_len_);
    const double* cols[3] = {wq, wk, wv};
    for (int b = 0; b < 3; ++b)
      for (size_t i = 0; i < H; ++i)
        for (size_t c = 0; c < gw; ++c) host[b * H * gw + i * gw + c] = cols[b][i * H + r * gw + c];
    for (size_t i = 0; i < H; ++i)
      for (size_t c = 0; c < gw; ++c) host[3 * H * gw + i * gw + c] = wo[(r * gw + c) * H + i];
    if (dtype_ == DType::F32) {
      std::vector<float> f(shard_len_);
      for (size_t e = 0; e < shard_len_; ++e) f[e] = static_cast<float>(host[e]);
      cuda_check(cudaMemcpy(slots_[r].weight.data(), f.data(), f.size() * 4, cudaMemcpyHostToDevice), "upload");
    } else {
      std::vector<uint16_t> hb(shard_len_);
      for (size_t e = 0; e < shard_len_; ++e) hb[e] = double_to_bf16_rne(host[e]);
      cuda_check(cudaMemcpy(slots_[r].weight.data(), hb.data(), hb.size() * 2, cudaMemcpyHostToDevice), "upload");
    }
  });
}

void RtpAttention::ensure_scratch(size_t rows) {
  if (rows == scratch_rows_) return;
  group_->synchronize();
  const size_t n = group_->size(), esz = dtype_size(dtype_);
  const size_t act = rows * gw_ * esz;
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    saved_[r] = DeviceBuffer();
    scratch_[r] = DeviceBuffer();
    saved_[r] = DeviceBuffer(w.device, n * 4 * act, &w.ledger, MemCategory::Activation, false);
    lse_[r] = DeviceBuffer(w.device, n * rows * g_ * sizeof(float), &w.ledger, MemCategory::Activation, false);
    // dA, dq, dk, dv, delta, step workspace (largest of the three step kernels)
    size_t ws = 0;
    for (int which = 0; which < 3; ++which) {
      ws = std::max(ws, rtpb_step_workspace_bytes(which, dcode(dtype_), rows, hidden_, gw_));
    }
    const size_t ws_off = (4 * act + rows * g_ * sizeof(float) + 255) & ~size_t(255);
    scratch_[r] = DeviceBuffer(w.device, ws_off + ws, &w.ledger, MemCategory::Other, true);
    // fp32 Y / dX accumulator: the rotation's steps (and, even at N = 1, dX's
    // three products per step) sum in it
    acc_[r] = DeviceBuffer(w.device, rows * hidden_ * sizeof(float), &w.ledger, MemCategory::Activation, false);
  });
  scratch_rows_ = rows;
}

void RtpAttention::forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode) {
  require_home("forward");
  const auto& local = group_->local_ranks();
  if (x.size() != local.size() || y.size() != local.size())
    throw DimensionError(label_ + ": forward expects one activation per local worker");
  if (rows == 0 || rows % seq_)
    throw DimensionError(label_ + ": rows (" + std::to_string(rows) + ") must be a positive multiple of seq " +
                         std::to_string(seq_));
  const size_t n = group_->size();
  ensure_scratch(rows);
  const bool train = mode == Mode::Train;
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  if (train) {
    for (size_t k = 0; k < local.size(); ++k) x_cache_[local[k]] = x[k];
    cached_rows_ = rows;
  }
  std::fill(trace_.begin(), trace_.begin() + n * n, -1);
  const int dt = dcode(dtype_);
  const bool f32 = dtype_ == DType::F32;
  const size_t esz = dtype_size(dtype_), H = hidden_, gw = gw_;
  const size_t act = rows * gw * esz;
  const float scale = float(1.0 / std::sqrt(double(hd_)));
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      check_forward_position(r, s);
      const size_t j = slots_[r].logical_id;
      trace_[s * n + r] = int64_t(j);
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const char* W = static_cast<const char*>(slots_[r].weight.data());
      char* sv = static_cast<char*>(saved_[r].data()) + s * 4 * act;  // q, k, v, o of this step
      float* lse = static_cast<float*>(lse_[r].data()) + s * rows * g_;
      char* scr = static_cast<char*>(scratch_[r].data());
      const size_t ws_off = (4 * act + rows * g_ * sizeof(float) + 255) & ~size_t(255);
      void* ws = scr + ws_off;
      const size_t ws_bytes = scratch_[r].bytes() - ws_off;
      const size_t ldx = x[k].ld ? x[k].ld : H;
      for (int b = 0; b < 3; ++b)  // Q, K, V = X . W{q,k,v}_j  (layers_attention.cpp:76-78)
        check_status(rtpb_fwd_step(dt, x[k].data, ldx, W + b * H * gw * esz, sv + b * act, gw, 0, nullptr, 0, rows,
                                   H, gw, RTPB_EPI_STORE_PRE | RTPB_EPI_NO_BIAS, ws, ws_bytes, w.compute));
      // per (sequence, head): softmax(Q K^T / sqrt(hd)) V  (:80-95)
      check_status(attention_core_fwd(f32, sv, sv + act, sv + 2 * act, sv + 3 * act, lse, rows, seq_, g_, hd_, scale,
                                      w.compute));
      // Y (+)= A . Wo_j, fp32 across the rotation (:97-98): the dX kernel with
      // W = Wo_j^T (hidden x gw)
      const int fl = (s == 0 ? RTPB_EPI_FIRST : 0) | (s + 1 == n ? RTPB_EPI_LAST : 0);
      float* acc = static_cast<float*>(acc_[r].data());
      check_status(rtpb_dgrad_step(dt, sv + 3 * act, gw, 0, W + 3 * H * gw * esz, acc, H, y[k].data,
                                   y[k].ld ? y[k].ld : H, nullptr, 0, rows, H, gw, fl, ws, ws_bytes, w.compute));
      if (train) tapes_[r].record(j, s);
    });
    if (s + 1 < n) rotate_forward();
  }
  if (!train) rehome_after_eval();
}

void RtpAttention::backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx) {
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
  const int dt = dcode(dtype_);
  const bool f32 = dtype_ == DType::F32;
  const size_t esz = dtype_size(dtype_), H = hidden_, gw = gw_;
  const size_t act = rows * gw * esz;
  const float scale = float(1.0 / std::sqrt(double(hd_)));
  for (size_t s = 0; s < n; ++s) {
    const bool zero = grads_zero_pending_ && s == 0;  // step 0 after zero_grads(): overwrite
    group_->each([&](size_t r) {
      const size_t j = slots_[r].logical_id;
      const size_t fs = tapes_[r].replay(j);  // the forward step whose q, k, v, o, lse this shard made
      check_backward_position(r, s);
      trace_[n * n + s * n + r] = int64_t(j);
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const char* W = static_cast<const char*>(slots_[r].weight.data());
      float* G = static_cast<float*>(slots_[r].grad_acc.data());
      const char* sv = static_cast<const char*>(saved_[r].data()) + fs * 4 * act;
      const float* lse = static_cast<const float*>(lse_[r].data()) + fs * rows * g_;
      char* scr = static_cast<char*>(scratch_[r].data());
      char *dA = scr, *dq = scr + act, *dk = scr + 2 * act, *dv = scr + 3 * act;
      float* delta = reinterpret_cast<float*>(scr + 4 * act);
      const size_t ws_off = (4 * act + rows * g_ * sizeof(float) + 255) & ~size_t(255);
      void* ws = scr + ws_off;
      const size_t ws_bytes = scratch_[r].bytes() - ws_off;
      const size_t ldy = dy[k].ld ? dy[k].ld : H, ldxc = x_cache_[r].ld ? x_cache_[r].ld : H;
      auto gblk = [&](int b) { return G + size_t(b) * H * gw; };
      // dWo_j^T += dY^T . A   (layers_attention.cpp:136-137: dWo_j += A^T dY)
      check_status(rtpb_wgrad_step_ex(dt, dy[k].data, ldy, sv + 3 * act, gw, 0, zero ? nullptr : gblk(3), gblk(3),
                                      rows, H, gw, RTPB_EPI_NO_BIAS, ws, ws_bytes, w.compute));
      // dA = dY . Wo_j^T  (:138-140)
      check_status(rtpb_fwd_step(dt, dy[k].data, ldy, W + 3 * H * gw * esz, dA, gw, 0, nullptr, 0, rows, H, gw,
                                 RTPB_EPI_STORE_PRE | RTPB_EPI_NO_BIAS, ws, ws_bytes, w.compute));
      // the core's backward per (sequence, head)  (:142-166)
      check_status(attention_core_bwd(f32, sv, sv + act, sv + 2 * act, sv + 3 * act, lse, dA, dq, dk, dv, delta,
                                      rows, seq_, g_, hd_, scale, w.compute));
      // dW{q,k,v}_j += X^T . d{Q,K,V}  (:170-172)
      const char* dqkv[3] = {dq, dk, dv};
      for (int b = 0; b < 3; ++b)
        check_status(rtpb_wgrad_step_ex(dt, x_cache_[r].data, ldxc, dqkv[b], gw, 0, zero ? nullptr : gblk(b),
                                        gblk(b), rows, H, gw, RTPB_EPI_NO_BIAS, ws, ws_bytes, w.compute));
      // dX += dQ Wq_j^T + dK Wk_j^T + dV Wv_j^T, fp32 across the rotation (:174-179)
      float* acc = static_cast<float*>(acc_[r].data());
      for (int b = 0; b < 3; ++b) {
        const bool first = s == 0 && b == 0, last = s + 1 == n && b == 2;
        const int fl = (first ? RTPB_EPI_FIRST : 0) | (last ? RTPB_EPI_LAST : 0);
        check_status(rtpb_dgrad_step(dt, dqkv[b], gw, 0, W + b * H * gw * esz, acc, H, dx[k].data,
                                     dx[k].ld ? dx[k].ld : H, nullptr, 0, rows, H, gw, fl, ws, ws_bytes, w.compute));
      }
    });
    if (zero) grads_zero_pending_ = false;  // every block of every resident shard was written
    if (s + 1 < n) rotate_backward();
  }
  for (size_t r : local) x_cache_[r] = {};
  require_home("end of backward");
}

std::vector<Tensor> RtpAttention::forward(std::span<const Tensor> x, Mode mode) {
  const auto& local = group_->local_ranks();
  auto xs = detail::per_local(*group_, x, label_, "forward");
  const size_t rows = xs[0]->rank() == 2 ? xs[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), ys(local.size());
  std::vector<DView> xv(local.size()), yv(local.size());
  const bool train = mode == Mode::Train;
  if (train) x_keep_.assign(group_->size(), Tensor());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    Tensor& keep = train ? x_keep_[local[k]] : tmp[k];
    const Tensor& xin = detail::as_layer_input(*xs[k], dtype_, w, hidden_, label_, keep, train);
    if (xin.rows() != rows) throw DimensionError(label_ + ": workers' activations differ in row count");
    ys[k] = Tensor({rows, hidden_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    xv[k] = {xin.data(), hidden_};
    yv[k] = {ys[k].data(), hidden_};
  }
  forward(xv, rows, yv, mode);
  group_->synchronize();
  return ys;
}

std::vector<Tensor> RtpAttention::backward(std::span<const Tensor> dy) {
  const auto& local = group_->local_ranks();
  auto ds = detail::per_local(*group_, dy, label_, "backward");
  const size_t rows = ds[0]->rank() == 2 ? ds[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size()), dxs(local.size());
  std::vector<DView> dv(local.size()), xv(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    const Tensor& din = detail::as_layer_input(*ds[k], dtype_, w, hidden_, label_, tmp[k], false);
    dxs[k] = Tensor({rows, hidden_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    dv[k] = {din.data(), hidden_};
    xv[k] = {dxs[k].data(), hidden_};
  }
  backward(dv, rows, xv);
  group_->synchronize();
  x_keep_.clear();
  return dxs;
}

std::vector<double> RtpAttention::shard_host(size_t rank, bool grad) {
  if (!group_->is_local(rank)) throw IndexError(label_ + ": shard of a non-local rank");
  if (grad) materialize_grads();
  group_->synchronize();
  const Tensor& t = grad ? slots_[rank].grad_acc : slots_[rank].weight;
  const std::vector<double> dev = t.to_host();  // [Wq | Wk | Wv | Wo^T]
  const size_t H = hidden_, gw = gw_;
  std::vector<double> out(dev.begin(), dev.end());
  for (size_t i = 0; i < H; ++i)
    for (size_t c = 0; c < gw; ++c) out[3 * H * gw + c * H + i] = dev[3 * H * gw + i * gw + c];
  return out;
}

}  // namespace rtpb
