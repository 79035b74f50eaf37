// RtpEmbedding (layers_linear.cpp:74-136) and RtpMoe (layers_moe.cpp:18-198)
// on the device: the same RtpLayerBase schedule (position laws, tapes,
// rotations) as RtpLinear; the expert MLPs run on the step GEMMs, routing and
// gather / scatter on kernels/moe_embed.cu.
#include <algorithm>
#include <cstring>
#include <map>

#include "kernels/launch.hpp"
#include "worker.hpp"

namespace rtpb {

namespace {
int dcode(DType d) { return d == DType::F32 ? RTPB_F32 : RTPB_BF16; }

void upload(void* dst, const void* src, size_t bytes, int device) {
  if (!bytes) return;
  DeviceGuard dg(device);
  cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "upload");
}

// host fp64 -> shard bytes in the layer dtype
void upload_values(void* dst, const std::vector<double>& v, DType dt, int device) {
  if (dt == DType::F32) {
    std::vector<float> f(v.begin(), v.end());
    upload(dst, f.data(), f.size() * 4, device);
  } else {
    std::vector<uint16_t> h(v.size());
    for (size_t i = 0; i < v.size(); ++i) h[i] = double_to_bf16_rne(v[i]);
    upload(dst, h.data(), h.size() * 2, device);
  }
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

ShardLayout layout_moe(size_t n_experts, size_t n) {
  if (n == 0) throw ConfigError("layout_moe: shard count must be >= 1");
  if (n_experts != n)
    throw ConfigError("layout_moe: " + std::to_string(n_experts) + " experts for " + std::to_string(n) +
                      " shards; expert count must equal the worker count (one expert per shard)");
  ShardLayout l;
  l.strategy = PartitionStrategy::ExpertPartition;
  l.n_shards = n;
  for (size_t j = 0; j < n; ++j) l.ranges.push_back({j, j + 1});
  return l;
}

// ================================================================ embedding
RtpEmbedding::RtpEmbedding(WorkerGroup& group, std::string label, const double* table, size_t vocab, size_t emb,
                           size_t n, DType dtype)
    : RtpLayerBase(group, std::move(label), dtype), vocab_(vocab), emb_(emb) {
  if (n != group_->size())
    throw ConfigError("RtpEmbedding: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  if (dtype != DType::BF16 && dtype != DType::F32) throw ConfigError("RtpEmbedding: layers compute in BF16 or F32");
  layout_ = layout_linear(vocab, emb, n);  // columns of the table (layers_linear.cpp:79)
  per_ = emb / n;
  shard_len_ = vocab * per_;
  init_slots_alloc();
  tapes_.assign(n, {});
  ids_dev_.resize(n);
  csr_.resize(n);
  n_ids_.assign(n, 0);
  n_uniq_.assign(n, 0);
  trace_.assign(2 * n * n, -1);
  // embedding_shard_groups (layers_common.cpp:47-52): shard j = table[:, j*per:(j+1)*per]
  group_->each([&](size_t r) {
    std::vector<double> host(shard_len_);
    for (size_t v = 0; v < vocab_; ++v)
      std::memcpy(&host[v * per_], table + v * emb_ + r * per_, per_ * sizeof(double));
    upload_values(slots_[r].weight.data(), host, dtype_, group_->worker(r).device);
  });
}

RtpEmbedding::RtpEmbedding(WorkerGroup& group, std::string label, const Tensor& table, size_t n)
    : RtpEmbedding(group, std::move(label), table.to_host().data(), table.rank() == 2 ? table.rows() : 0,
                   table.rank() == 2 ? table.cols() : 0, n,
                   table.dtype() == DType::BF16 ? DType::BF16 : DType::F32) {}

void RtpEmbedding::forward(std::span<const std::vector<int64_t>> ids, std::span<const DView> y, Mode mode) {
  require_home("forward");
  const auto& local = group_->local_ranks();
  if (ids.size() != local.size() || y.size() != local.size())
    throw DimensionError(label_ + ": forward expects one id list and one output per local worker");
  for (const auto& v : ids)
    for (int64_t id : v)
      if (id < 0 || size_t(id) >= vocab_)
        throw IndexError("embedding id " + std::to_string(id) + " outside vocab of " + std::to_string(vocab_));
  const size_t n = group_->size();
  const bool train = mode == Mode::Train;
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  group_->synchronize();  // the previous pass may still read the id buffers
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    const auto& v = ids[k_of[r]];
    if (ids_dev_[r].bytes() < v.size() * 8)
      ids_dev_[r] = DeviceBuffer(w.device, std::max<size_t>(v.size(), 1) * 8, &w.ledger, MemCategory::Activation,
                                 false);
    upload(ids_dev_[r].data(), v.data(), v.size() * 8, w.device);
    n_ids_[r] = v.size();
    if (train) {
      // CSR of token positions per unique id, tokens ascending: the
      // reference's scatter order (grad[id] += dy_i for i ascending)
      std::map<int64_t, std::vector<int>> by_id;
      for (size_t i = 0; i < v.size(); ++i) by_id[v[i]].push_back(int(i));
      std::vector<int64_t> uniq;
      std::vector<int> offs{0}, toks;
      for (auto& [id, t] : by_id) {
        uniq.push_back(id);
        toks.insert(toks.end(), t.begin(), t.end());
        offs.push_back(int(toks.size()));
      }
      const size_t bytes = align256(uniq.size() * 8) + align256(offs.size() * 4) + toks.size() * 4 + 8;
      if (csr_[r].bytes() < bytes) csr_[r] = DeviceBuffer(w.device, bytes, &w.ledger, MemCategory::Activation, false);
      char* base = static_cast<char*>(csr_[r].data());
      upload(base, uniq.data(), uniq.size() * 8, w.device);
      upload(base + align256(uniq.size() * 8), offs.data(), offs.size() * 4, w.device);
      upload(base + align256(uniq.size() * 8) + align256(offs.size() * 4), toks.data(), toks.size() * 4, w.device);
      n_uniq_[r] = uniq.size();
    }
  });
  std::fill(trace_.begin(), trace_.begin() + n * n, -1);
  const bool f32 = dtype_ == DType::F32;
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      check_forward_position(r, s);
      const size_t j = slots_[r].logical_id;
      trace_[s * n + r] = int64_t(j);
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      check_status(embed_gather(f32, slots_[r].weight.data(), per_, static_cast<const int64_t*>(ids_dev_[r].data()),
                                n_ids_[r], y[k].data, y[k].ld ? y[k].ld : emb_, j * per_, w.compute));
      if (train) tapes_[r].record(j, {});
    });
    if (s + 1 < n) rotate_forward();
  }
  if (!train) rehome_after_eval();
}

void RtpEmbedding::backward(std::span<const DView> dy, size_t rows, const std::function<void()>& after_last_rotation) {
  const auto& local = group_->local_ranks();
  if (dy.size() != local.size()) throw DimensionError(label_ + ": backward expects one gradient per local worker");
  const size_t n = group_->size();
  for (size_t r : local) {
    if (tapes_[r].empty()) throw StateError("backward invoked without a matching forward");
    if (rows != n_ids_[r]) throw DimensionError(label_ + ": backward rows differ from the forward's id count");
  }
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  std::fill(trace_.begin() + n * n, trace_.end(), -1);
  materialize_grads();  // scatter-add touches only the rows of seen ids
  const bool f32 = dtype_ == DType::F32;
  for (size_t s = 0; s < n; ++s) {
    if (s + 1 == n && after_last_rotation) after_last_rotation();
    group_->each([&](size_t r) {
      const size_t j = slots_[r].logical_id;
      tapes_[r].replay(j);
      check_backward_position(r, s);
      trace_[n * n + s * n + r] = int64_t(j);
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      const char* base = static_cast<const char*>(csr_[r].data());
      const size_t nu = n_uniq_[r];
      const auto* uniq = reinterpret_cast<const int64_t*>(base);
      const auto* offs = reinterpret_cast<const int*>(base + align256(nu * 8));
      const auto* toks = reinterpret_cast<const int*>(base + align256(nu * 8) + align256((nu + 1) * 4));
      check_status(embed_scatter(f32, dy[k].data, dy[k].ld ? dy[k].ld : emb_, j * per_, uniq, offs, toks, nu, per_,
                                 static_cast<float*>(slots_[r].grad_acc.data()), w.compute));
    });
    if (s + 1 < n) rotate_backward();
  }
  require_home("end of backward");
}

std::vector<Tensor> RtpEmbedding::forward(std::span<const std::vector<int64_t>> ids, Mode mode) {
  const auto& local = group_->local_ranks();
  std::vector<std::vector<int64_t>> mine;
  if (ids.size() == group_->size() && local.size() == group_->size())
    mine.assign(ids.begin(), ids.end());
  else if (ids.size() == local.size())
    mine.assign(ids.begin(), ids.end());
  else
    throw DimensionError(label_ + ": forward expects one id list per local worker");
  std::vector<Tensor> ys(local.size());
  std::vector<DView> yv(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    ys[k] = Tensor({mine[k].size(), emb_}, dtype_, w.device, &w.ledger, MemCategory::Activation, false);
    yv[k] = {ys[k].data(), emb_};
  }
  forward(mine, yv, mode);
  group_->synchronize();
  return ys;
}

void RtpEmbedding::backward(std::span<const Tensor> dy, const std::function<void()>& after_last_rotation) {
  const auto& local = group_->local_ranks();
  auto ds = detail::per_local(*group_, dy, label_, "backward");
  const size_t rows = ds[0]->rank() == 2 ? ds[0]->rows() : 0;
  std::vector<Tensor> tmp(local.size());
  std::vector<DView> dv(local.size());
  for (size_t k = 0; k < local.size(); ++k) {
    Worker& w = group_->worker(local[k]);
    const Tensor& din = detail::as_layer_input(*ds[k], dtype_, w, emb_, label_, tmp[k], false);
    dv[k] = {din.data(), emb_};
  }
  backward(dv, rows, after_last_rotation);
  group_->synchronize();
}

// ================================================================ MoE
RtpMoe::RtpMoe(WorkerGroup& group, std::string label, const double* gate, const double* const* experts, size_t hidden,
               size_t ffn, size_t n, DType dtype)
    : RtpLayerBase(group, std::move(label), dtype), hidden_(hidden), ffn_(ffn) {
  if (n != group_->size())
    throw ConfigError("RtpMoe: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  if (dtype != DType::BF16 && dtype != DType::F32) throw ConfigError("RtpMoe: layers compute in BF16 or F32");
  init(gate, experts);
}

RtpMoe::RtpMoe(WorkerGroup& group, std::string label, const Tensor& gate, std::span<const ExpertParams> experts,
               size_t n)
    : RtpLayerBase(group, std::move(label),
                   !experts.empty() && experts[0].w1.dtype() == DType::BF16 ? DType::BF16 : DType::F32),
      hidden_(gate.rank() == 2 ? gate.rows() : 0),
      ffn_(!experts.empty() && experts[0].w1.rank() == 2 ? experts[0].w1.cols() : 0) {
  if (experts.size() != n)
    throw ConfigError("moe_shard_groups: " + std::to_string(experts.size()) + " experts for " + std::to_string(n) +
                      " shards");
  if (n != group_->size())
    throw ConfigError("RtpMoe: n = " + std::to_string(n) + " does not match the group of " +
                      std::to_string(group_->size()));
  if (gate.rank() != 2 || gate.cols() != n)
    throw ConfigError("gate weight " + gate.shape_str() + " must have one column per expert (" + std::to_string(n) +
                      ")");
  std::vector<std::vector<double>> packed(n);
  std::vector<const double*> ptrs(n);
  for (size_t e = 0; e < n; ++e) {
    const ExpertParams& x = experts[e];
    if (x.w1.shape() != std::vector<size_t>{hidden_, ffn_} || x.b1.shape() != std::vector<size_t>{ffn_} ||
        x.w2.shape() != std::vector<size_t>{ffn_, hidden_} || x.b2.shape() != std::vector<size_t>{hidden_})
      throw DimensionError(label_ + ": expert " + std::to_string(e) + " shapes do not match hidden / ffn");
    for (const Tensor* t : {&x.w1, &x.b1, &x.w2, &x.b2}) {
      const auto v = t->to_host();
      packed[e].insert(packed[e].end(), v.begin(), v.end());
    }
    ptrs[e] = packed[e].data();
  }
  const auto g = gate.to_host();
  init(g.data(), ptrs.data());
}

void RtpMoe::init(const double* gate, const double* const* experts) {
  const size_t n = group_->size();
  layout_ = layout_moe(n, n);
  if (hidden_ % 8 || ffn_ % 8)
    throw ConfigError("RtpMoe " + label_ + ": hidden and ffn must be multiples of 8 on the device path");
  if (n > 32) throw ConfigError("RtpMoe " + label_ + ": at most 32 experts");
  shard_len_ = 2 * hidden_ * ffn_ + ffn_ + hidden_;
  init_slots_alloc();
  tapes_.assign(n, {});
  x_cache_.assign(n, {});
  gates_.resize(n);
  gate_grads_.resize(n);
  route_.resize(n);
  saved_.resize(n);
  scratch_.resize(n);
  seg_off_.assign(n, std::vector<size_t>(n, 0));
  seg_cnt_.assign(n, std::vector<size_t>(n, 0));
  trace_.assign(2 * n * n, -1);
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    // moe_shard_groups (layers_common.cpp:76-88): shard j = expert j packed
    upload_values(slots_[r].weight.data(), std::vector<double>(experts[r], experts[r] + shard_len_), dtype_,
                  w.device);
    gates_[r] = Tensor({hidden_, n}, DType::F64, w.device, &w.ledger, MemCategory::Param, false);  // replicated
    upload(gates_[r].data(), gate, hidden_ * n * 8, w.device);
    gate_grads_[r] = Tensor({hidden_, n}, DType::F64, w.device, &w.ledger, MemCategory::Grad, true);
  });
}

void RtpMoe::zero_grads() {
  RtpLayerBase::zero_grads();
  gate_zero_pending_ = true;  // the next backward overwrites the gate gradient
}

void RtpMoe::ensure_scratch(size_t rows) {
  if (rows == scratch_rows_) return;
  group_->synchronize();
  const size_t n = group_->size(), esz = dtype_size(dtype_), H = hidden_, F = ffn_;
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    route_[r] = DeviceBuffer();
    saved_[r] = DeviceBuffer();
    scratch_[r] = DeviceBuffer();
    // probs | dlogits (fp64 rows x n) | sel | pos | by-expert rows (int32)
    route_[r] = DeviceBuffer(w.device, 2 * align256(rows * n * 8) + 3 * align256(rows * 4), &w.ledger,
                             MemCategory::Activation, false);
    // gathered X | pre1 | h1 | eout, rows in expert-segment order
    saved_[r] = DeviceBuffer(w.device, align256(rows * H * esz) + 2 * align256(rows * F * esz) + rows * H * esz,
                             &w.ledger, MemCategory::Activation, false);
    size_t ws = 0;
    for (int which = 0; which < 3; ++which) {
      ws = std::max(ws, rtpb_step_workspace_bytes(which, dcode(dtype_), rows, H, F));
      ws = std::max(ws, rtpb_step_workspace_bytes(which, dcode(dtype_), rows, F, H));
    }
    // de | dxs, then the step workspace
    scratch_[r] = DeviceBuffer(w.device, 2 * align256(rows * H * esz) + ws, &w.ledger, MemCategory::Other, true);
  });
  scratch_rows_ = rows;
}

void RtpMoe::forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode) {
  require_home("forward");
  const auto& local = group_->local_ranks();
  if (x.size() != local.size() || y.size() != local.size())
    throw DimensionError(label_ + ": forward expects one activation per local worker");
  if (rows == 0) throw DimensionError(label_ + ": forward needs at least one row");
  const size_t n = group_->size(), esz = dtype_size(dtype_), H = hidden_, F = ffn_;
  ensure_scratch(rows);
  const bool train = mode == Mode::Train, f32 = dtype_ == DType::F32;
  const int dt = dcode(dtype_);
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  if (train) {
    for (size_t k = 0; k < local.size(); ++k) x_cache_[local[k]] = x[k];
    cached_rows_ = rows;
  }
  // routing (layers_moe.cpp:48-61): gate on the device in fp64; the expert
  // segment sizes come back to the host once per pass (GEMM shapes)
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    const size_t k = k_of[r];
    char* rb = static_cast<char*>(route_[r].data());
    double* probs = reinterpret_cast<double*>(rb);
    int* sel = reinterpret_cast<int*>(rb + 2 * align256(rows * n * 8));
    int* pos = sel + align256(rows * 4) / 4;
    int* byexp = pos + align256(rows * 4) / 4;
    check_status(moe_gate(f32, x[k].data, rows, H, static_cast<const double*>(gates_[r].data()), n, probs, sel,
                          w.compute));
    std::vector<int> hs(rows);
    DeviceGuard dg(w.device);
    cuda_check(cudaStreamSynchronize(w.compute), "moe routing");
    cuda_check(cudaMemcpy(hs.data(), sel, rows * 4, cudaMemcpyDeviceToHost), "moe routing");
    std::vector<int> hp(rows), hb;
    auto& off = seg_off_[r];
    auto& cnt = seg_cnt_[r];
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int s_ : hs) ++cnt[size_t(s_)];
    size_t acc = 0;
    for (size_t e = 0; e < n; ++e) {
      off[e] = acc;
      acc += cnt[e];
    }
    hb.assign(rows, 0);
    std::vector<size_t> fill(off.begin(), off.end());
    for (size_t t = 0; t < rows; ++t) {  // tokens ascending within an expert (layers_moe.cpp:73-75)
      const size_t p = fill[size_t(hs[t])]++;
      hb[p] = int(t);
      hp[t] = int(p);
    }
    upload(pos, hp.data(), rows * 4, w.device);
    upload(byexp, hb.data(), rows * 4, w.device);
  });
  std::fill(trace_.begin(), trace_.begin() + n * n, -1);
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      check_forward_position(r, s);
      const size_t j = slots_[r].logical_id;
      trace_[s * n + r] = int64_t(j);
      if (train) tapes_[r].record(j, {});
      const size_t cnt = seg_cnt_[r][j], o = seg_off_[r][j];
      if (!cnt) return;
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      char* rb = static_cast<char*>(route_[r].data());
      const int* byexp = reinterpret_cast<const int*>(rb + 2 * align256(rows * n * 8) + 2 * align256(rows * 4)) + o;
      char* sv = static_cast<char*>(saved_[r].data());
      char* xs = sv + o * H * esz;
      char* pre1 = sv + align256(rows * H * esz) + o * F * esz;
      char* h1 = sv + align256(rows * H * esz) + align256(rows * F * esz) + o * F * esz;
      char* eout = sv + align256(rows * H * esz) + 2 * align256(rows * F * esz) + o * H * esz;
      char* scr = static_cast<char*>(scratch_[r].data());
      void* ws = scr + 2 * align256(rows * H * esz);
      const size_t ws_bytes = scratch_[r].bytes() - 2 * align256(rows * H * esz);
      const char* W = static_cast<const char*>(slots_[r].weight.data());
      check_status(gather_rows(f32, x[k].data, x[k].ld ? x[k].ld : H, byexp, cnt, H, xs, w.compute));
      // expert j: h1 = gelu(xs W1 + b1) (GELU fused), eout = h1 W2 + b2  (:80-88)
      check_status(rtpb_fwd_step(dt, xs, H, W, pre1, F, 0, h1, F, cnt, H, F,
                                 (train ? RTPB_EPI_STORE_PRE : 0) | RTPB_EPI_GELU |
                                     (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0),
                                 ws, ws_bytes, w.compute));
      check_status(rtpb_fwd_step(dt, h1, F, W + (H * F + F) * esz, eout, H, 0, nullptr, 0, cnt, F, H,
                                 RTPB_EPI_STORE_PRE, ws, ws_bytes, w.compute));
    });
    if (s + 1 < n) rotate_forward();
  }
  // y_t = p_t,sel(t) * e_t once every expert has passed (:90-94)
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    const size_t k = k_of[r];
    char* rb = static_cast<char*>(route_[r].data());
    const double* probs = reinterpret_cast<const double*>(rb);
    const int* sel = reinterpret_cast<const int*>(rb + 2 * align256(rows * n * 8));
    const int* pos = sel + align256(rows * 4) / 4;
    const char* eout = static_cast<const char*>(saved_[r].data()) + align256(rows * H * esz) +
                       2 * align256(rows * F * esz);
    check_status(moe_combine(f32, eout, pos, sel, probs, n, rows, H, y[k].data, y[k].ld ? y[k].ld : H, w.compute));
  });
  if (!train) rehome_after_eval();
}

void RtpMoe::backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx) {
  const auto& local = group_->local_ranks();
  if (dy.size() != local.size() || dx.size() != local.size())
    throw DimensionError(label_ + ": backward expects one gradient per local worker");
  const size_t n = group_->size(), esz = dtype_size(dtype_), H = hidden_, F = ffn_;
  for (size_t r : local)
    if (tapes_[r].empty()) throw StateError("backward invoked without a matching forward");
  if (rows != cached_rows_) throw DimensionError(label_ + ": backward rows differ from the cached forward");
  const bool f32 = dtype_ == DType::F32;
  const int dt = dcode(dtype_);
  std::vector<size_t> k_of(n, 0);
  for (size_t k = 0; k < local.size(); ++k) k_of[local[k]] = k;
  std::fill(trace_.begin() + n * n, trace_.end(), -1);
  materialize_grads();  // an expert that saw no token adds nothing: zero fill for real
  for (size_t s = 0; s < n; ++s) {
    group_->each([&](size_t r) {
      const size_t j = slots_[r].logical_id;
      tapes_[r].replay(j);
      check_backward_position(r, s);
      trace_[n * n + s * n + r] = int64_t(j);
      const size_t cnt = seg_cnt_[r][j], o = seg_off_[r][j];
      if (!cnt) return;
      Worker& w = group_->worker(r);
      const size_t k = k_of[r];
      char* rb = static_cast<char*>(route_[r].data());
      const double* probs = reinterpret_cast<const double*>(rb);
      double* dlogits = reinterpret_cast<double*>(rb + align256(rows * n * 8));
      const int* byexp = reinterpret_cast<const int*>(rb + 2 * align256(rows * n * 8) + 2 * align256(rows * 4)) + o;
      char* sv = static_cast<char*>(saved_[r].data());
      char* xs = sv + o * H * esz;
      char* pre1 = sv + align256(rows * H * esz) + o * F * esz;
      char* h1 = sv + align256(rows * H * esz) + align256(rows * F * esz) + o * F * esz;
      char* eout = sv + align256(rows * H * esz) + 2 * align256(rows * F * esz) + o * H * esz;
      char* scr = static_cast<char*>(scratch_[r].data());
      char* de = scr + o * H * esz;
      char* dxs = scr + align256(rows * H * esz) + o * H * esz;
      void* ws = scr + 2 * align256(rows * H * esz);
      const size_t ws_bytes = scratch_[r].bytes() - 2 * align256(rows * H * esz);
      const char* W = static_cast<const char*>(slots_[r].weight.data());
      float* G = static_cast<float*>(slots_[r].grad_acc.data());
      // de = p dy, dlogits from dp = dy . e  (:146-160)
      check_status(moe_route_bwd(f32, dy[k].data, dy[k].ld ? dy[k].ld : H, eout, byexp, cnt, j, probs, n, H, de,
                                 dlogits, w.compute));
      // [gW2 | gb2] += h1^T de (+ colsum)  (:164-167)
      check_status(rtpb_wgrad_step(dt, h1, F, de, H, 0, G + H * F + F, G + H * F + F, cnt, F, H, ws, ws_bytes,
                                   w.compute));
      // dpre1 = (de W2^T) * gelu'(pre1), written over pre1  (:168-171)
      check_status(rtpb_dgrad_step(dt, de, H, 0, W + (H * F + F) * esz, nullptr, F, pre1, F, pre1, F, cnt, F, H,
                                   RTPB_EPI_FIRST | RTPB_EPI_LAST | RTPB_EPI_GELU_BWD |
                                       (exact_gelu_ ? RTPB_EPI_EXACT_GELU : 0),
                                   ws, ws_bytes, w.compute));
      // [gW1 | gb1] += xs^T dpre1 (+ colsum)  (:172-175)
      check_status(rtpb_wgrad_step(dt, xs, H, pre1, F, 0, G, G, cnt, H, F, ws, ws_bytes, w.compute));
      // dxs = dpre1 W1^T  (:176-178)
      check_status(rtpb_dgrad_step(dt, pre1, F, 0, W, nullptr, H, dxs, H, nullptr, 0, cnt, H, F,
                                   RTPB_EPI_FIRST | RTPB_EPI_LAST, ws, ws_bytes, w.compute));
    });
    if (s + 1 < n) rotate_backward();
  }
  // gate path: dX = dxs + dlogits Wg^T; dWg (+)= X^T dlogits  (:183-192)
  group_->each([&](size_t r) {
    Worker& w = group_->worker(r);
    const size_t k = k_of[r];
    char* rb = static_cast<char*>(route_[r].data());
    const double* dlogits = reinterpret_cast<const double*>(rb + align256(rows * n * 8));
    const int* pos = reinterpret_cast<const int*>(rb + 2 * align256(rows * n * 8) + align256(rows * 4));
    const char* dxs = static_cast<const char*>(scratch_[r].data()) + align256(rows * H * esz);
    check_status(moe_dx(f32, dxs, pos, dlogits, static_cast<const double*>(gates_[r].data()), n, rows, H, dx[k].data,
                        dx[k].ld ? dx[k].ld : H, w.compute));
    check_status(moe_gate_grad(f32, x_cache_[r].data, x_cache_[r].ld ? x_cache_[r].ld : H, dlogits, n, rows, H,
                               static_cast<double*>(gate_grads_[r].data()), !gate_zero_pending_, w.compute));
  });
  gate_zero_pending_ = false;
  for (size_t r : local) x_cache_[r] = {};
  require_home("end of backward");
}

std::vector<Tensor> RtpMoe::forward(std::span<const Tensor> x, Mode mode) {
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

std::vector<Tensor> RtpMoe::backward(std::span<const Tensor> dy) {
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

}  // namespace rtpb
