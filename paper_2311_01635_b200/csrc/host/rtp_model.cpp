// RtpModel (model.cpp:7-121): the reference's whole rotated transformer on
// the device — embedding, blocks of attention + FFN (RtpMlp) or MoE with
// residual connections, linear head — composed from the device layers over
// their Tensor API. Parameters from SplitMix64(seed) in SerialModel's draw
// order (serial.cpp:325-353) AS THE REFERENCE IS BUILT: the draws that are
// arguments of one constructor call (SerialAttention(draw, draw, draw, draw),
// SerialLinear(draw, draw)) happen in the compiler's argument evaluation
// order, which C++ leaves unspecified and g++ (the reference's toolchain)
// takes right to left — wo, wv, wk, wq and bias before weight; braced
// ExpertParams{...} lists are left to right.
#include <cstring>

#include "kernels/launch.hpp"
#include "worker.hpp"

namespace rtpb {

std::vector<double> RtpLayerBase::shard_host(size_t rank, bool grad) {
  if (!group_->is_local(rank)) throw IndexError(label_ + ": shard of a non-local rank");
  if (grad) materialize_grads();
  group_->synchronize();
  return (grad ? slots_[rank].grad_acc : slots_[rank].weight).to_host();
}

namespace {
// Tensor::uniform's draws (tensor.cpp:99-103) of one parameter, row-major.
std::vector<double> draw(SplitMix64& rng, size_t count) {
  std::vector<double> v(count);
  for (double& x : v) x = rng.next_uniform(-0.1, 0.1);
  return v;
}

// out[k] = a[k] + b[k] per local rank (model.cpp:72, 85, 108, 111)
std::vector<Tensor> add(WorkerGroup& g, const std::vector<Tensor>& a, const std::vector<Tensor>& b) {
  std::vector<Tensor> out(a.size());
  const auto& local = g.local_ranks();
  for (size_t k = 0; k < a.size(); ++k) {
    Worker& w = g.worker(local[k]);
    if (a[k].shape() != b[k].shape() || a[k].dtype() != b[k].dtype())
      throw DimensionError("residual add: shapes " + a[k].shape_str() + " and " + b[k].shape_str());
    out[k] = Tensor(a[k].shape(), a[k].dtype(), w.device, &w.ledger, MemCategory::Activation, false);
    DeviceGuard dg(w.device);
    check_status(rtpb_add(int(a[k].dtype()), a[k].data(), b[k].data(), out[k].data(), a[k].numel(), w.compute));
  }
  g.synchronize();
  return out;
}
}  // namespace

RtpModel::RtpModel(const ModelDims& dims, uint64_t seed, WorkerGroup& group, RotationMode mode, DType dtype)
    : group_(&group), mode_(mode), dims_(dims), dtype_(dtype) {
  const size_t n = group.size();
  if (dims_.moe && dims_.n_experts != n)
    throw ConfigError("MoE twin built for " + std::to_string(dims_.n_experts) + " experts cannot shard across " +
                      std::to_string(n) + " workers");
  if (dims_.hidden % dims_.heads != 0)
    throw ConfigError("hidden size " + std::to_string(dims_.hidden) + " not divisible by " +
                      std::to_string(dims_.heads) + " heads");
  const size_t h = dims_.hidden, f = dims_.ffn, v = dims_.vocab;
  SplitMix64 rng(seed);
  const auto table = draw(rng, v * h);
  embedding_ = std::make_unique<RtpEmbedding>(group, "embedding", table.data(), v, h, n, dtype);
  blocks_.resize(dims_.layers);
  for (size_t l = 0; l < dims_.layers; ++l) {
    const std::string tag = "block" + std::to_string(l);
    const auto wo = draw(rng, h * h), wv = draw(rng, h * h), wk = draw(rng, h * h), wq = draw(rng, h * h);
    blocks_[l].attn = std::make_unique<RtpAttention>(group, tag + "/attn", wq.data(), wk.data(), wv.data(), wo.data(),
                                                     h, dims_.heads, dims_.seq, n, dtype);
    if (dims_.moe) {
      const auto gate = draw(rng, h * n);
      std::vector<std::vector<double>> ex(n);
      std::vector<const double*> ptr(n);
      for (size_t e = 0; e < n; ++e) {
        for (size_t c : {h * f, f, f * h, h}) {
          const auto p = draw(rng, c);
          ex[e].insert(ex[e].end(), p.begin(), p.end());
        }
        ptr[e] = ex[e].data();
      }
      blocks_[l].moe = std::make_unique<RtpMoe>(group, tag + "/moe", gate.data(), ptr.data(), h, f, n, dtype);
    } else {
      const auto b1 = draw(rng, f), w1 = draw(rng, h * f), b2 = draw(rng, h), w2 = draw(rng, f * h);
      blocks_[l].mlp = std::make_unique<RtpMlp>(group, tag, h, f, dtype, w1.data(), b1.data(), w2.data(), b2.data());
    }
  }
  const auto hb = draw(rng, v), hw = draw(rng, h * v);
  head_ = std::make_unique<RtpLinear>(group, "head", hw.data(), hb.data(), h, v, n, dtype);
  for (RtpLayerBase* l : all_layers()) l->set_rotation_mode(mode);
}

RtpModel::~RtpModel() = default;

std::vector<RtpLayerBase*> RtpModel::all_layers() {
  std::vector<RtpLayerBase*> out{embedding_.get()};
  for (auto& b : blocks_) {
    out.push_back(b.attn.get());
    if (b.moe) {
      out.push_back(b.moe.get());
    } else {
      out.push_back(&b.mlp->ffn1());
      out.push_back(&b.mlp->ffn2());
    }
  }
  out.push_back(head_.get());
  return out;
}

void RtpModel::begin_step() {
  if (mode_ == RotationMode::OutOfPlace)
    for (RtpLayerBase* l : all_layers())
      if (!l->has_comm_spares()) l->allocate_comm_spares();
}

bool RtpModel::comm_spares_active() const {
  bool active = false;
  for (RtpLayerBase* l : const_cast<RtpModel*>(this)->all_layers()) active = active || l->has_comm_spares();
  return active;
}

void RtpModel::zero_grads() {
  for (RtpLayerBase* l : all_layers()) l->zero_grads();  // RtpMoe also zeroes its gate gradient
}

std::vector<Tensor> RtpModel::forward(std::span<const std::vector<int64_t>> ids, Mode mode) {
  std::vector<Tensor> x = embedding_->forward(ids, mode);
  for (auto& b : blocks_) {
    std::vector<Tensor> attn_out = b.attn->forward(x, mode);
    std::vector<Tensor> x1 = add(*group_, x, attn_out);  // model.cpp:72
    std::vector<Tensor> f = b.moe ? b.moe->forward(x1, mode) : b.mlp->forward(x1, mode);
    x = add(*group_, x1, f);  // model.cpp:85
  }
  return head_->forward(x, mode);
}

void RtpModel::backward(std::span<const Tensor> dlogits) {
  std::vector<Tensor> dx = head_->backward(dlogits);
  for (auto it = blocks_.rbegin(); it != blocks_.rend(); ++it) {
    std::vector<Tensor> df = it->moe ? it->moe->backward(dx) : it->mlp->backward(dx);
    std::vector<Tensor> dx1 = add(*group_, dx, df);  // model.cpp:108
    std::vector<Tensor> dattn = it->attn->backward(dx1);
    dx = add(*group_, dx1, dattn);  // model.cpp:111
  }
  std::function<void()> release;
  if (mode_ == RotationMode::OutOfPlace) {
    release = [this] {
      for (RtpLayerBase* l : all_layers()) l->release_comm_spares();
      if (on_comm_release) on_comm_release();
    };
  }
  embedding_->backward(dx, release);
}

}  // namespace rtpb
