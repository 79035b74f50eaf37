// C ABI, layer (2): group / layer handles over the C++ classes of
// include/rtpb/rtp.hpp. Exceptions become status codes + rtpb_last_error().
#include <nccl.h>

#include <atomic>
#include <cstdio>
#include <cstring>

#include "kernels/launch.hpp"
#include "worker.hpp"

using namespace rtpb;

namespace rtpb {
extern std::atomic<int> g_skip_comm;  // rtp_group.cpp
}

// Layers keep their group alive: the WorkerGroup (worker streams, ledgers)
// is destroyed only after its last layer, whatever order FFI callers free in.
struct rtpb_group_s {
  std::unique_ptr<WorkerGroup> g;
  int refs = 1;
};
static void group_release(rtpb_group_s* g) {
  if (g && --g->refs == 0) delete g;
}
struct rtpb_linear_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpLinear> l;
  bool owned = true;
};
struct rtpb_attention_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpAttention> a;
};
struct rtpb_embedding_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpEmbedding> e;
};
struct rtpb_moe_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpMoe> m;
};
struct rtpb_model_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpModel> m;
};
struct rtpb_mlp_s {
  rtpb_group_s* grp;
  std::unique_ptr<RtpMlp> m;
  rtpb_linear_s ffn1, ffn2;  // non-owning views for rtpb_mlp_layer
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return RTPB_OK;
  } catch (const ConfigError& e) {
    return set_error(RTPB_ERR_CONFIG, e.what());
  } catch (const DimensionError& e) {
    return set_error(RTPB_ERR_DIMENSION, e.what());
  } catch (const ProtocolError& e) {
    return set_error(RTPB_ERR_PROTOCOL, e.what());
  } catch (const StateError& e) {
    return set_error(RTPB_ERR_STATE, e.what());
  } catch (const IndexError& e) {
    return set_error(RTPB_ERR_INDEX, e.what());
  } catch (const CudaError& e) {
    return set_error(RTPB_ERR_CUDA, e.what());
  } catch (const NcclError& e) {
    return set_error(RTPB_ERR_NCCL, e.what());
  } catch (const std::exception& e) {
    return set_error(RTPB_ERR_GENERIC, e.what());
  }
}

std::vector<DView> views(const void* const* p, size_t count) {
  std::vector<DView> v(count);
  for (size_t k = 0; k < count; ++k) v[k] = {const_cast<void*>(p[k]), 0};
  return v;
}

DType dt(int d) {
  if (d != RTPB_BF16 && d != RTPB_F32) throw ConfigError("unknown dtype " + std::to_string(d));
  return d == RTPB_F32 ? DType::F32 : DType::BF16;
}

}  // namespace

namespace {
template <class H>
int layer_destroy(H* h) {
  return guard([&] {
    if (h) {
      rtpb_group_s* g = h->grp;
      delete h;
      group_release(g);
    }
  });
}
RotationMode rot(int mode) { return mode == RTPB_ROT_OUTOFPLACE ? RotationMode::OutOfPlace : RotationMode::InPlace; }
void slot_of(RtpLayerBase& l, WorkerGroup& g, size_t rank, int64_t* id, int64_t* off) {
  if (!g.is_local(rank)) throw IndexError("slot of a non-local rank");
  ShardSlot& s = l.slots()[rank];
  if (id) *id = int64_t(s.logical_id);
  if (off) *off = s.rotation_offset;
}
void read_host(RtpLayerBase& l, WorkerGroup& g, size_t rank, int which, double* dst) {
  if (!g.is_local(rank)) throw IndexError("shard of a non-local rank");
  if (which) l.materialize_grads();
  g.synchronize();
  const Tensor& t = which ? l.slots()[rank].grad_acc : l.slots()[rank].weight;
  const std::vector<double> v = t.to_host();
  std::memcpy(dst, v.data(), v.size() * sizeof(double));
}
}  // namespace

extern "C" {

int rtpb_ring_plan(size_t n, size_t rank, int phase, size_t step, int64_t* logical_id, int64_t* send_to,
                   int64_t* recv_from) {
  if (n == 0 || rank >= n) return set_error(RTPB_ERR_CONFIG, "ring_plan: rank out of range");
  if (phase != 0 && phase != 1) return set_error(RTPB_ERR_CONFIG, "ring_plan: phase must be 0 or 1");
  const size_t s = step % n;
  if (logical_id) *logical_id = int64_t(phase == 0 ? (rank + n - s) % n : (rank + 1 + s) % n);
  const bool rotates = step + 1 < n;
  const Direction d = phase == 0 ? Direction::Clockwise : Direction::CounterClockwise;
  if (send_to) *send_to = rotates ? int64_t(ring_dest(rank, n, d)) : -1;
  if (recv_from) *recv_from = rotates ? int64_t(ring_src(rank, n, d)) : -1;
  return RTPB_OK;
}

int rtpb_group_create(size_t n, int transport, const int* devices, rtpb_group* out) {
  return guard([&] {
    if (transport == RTPB_TRANSPORT_NCCL) throw ConfigError("use rtpb_group_create_nccl for NCCL groups");
    std::vector<int> dev;
    if (devices) dev.assign(devices, devices + n);
    auto h = std::make_unique<rtpb_group_s>();
    h->g = std::make_unique<WorkerGroup>(
        n, transport == RTPB_TRANSPORT_CONCURRENT ? TransportKind::Concurrent : TransportKind::Lockstep, dev);
    *out = h.release();
  });
}

int rtpb_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
  });
}

int rtpb_group_create_nccl(size_t n, size_t rank, int device, const void* nccl_id, rtpb_group* out) {
  return guard([&] {
    auto h = std::make_unique<rtpb_group_s>();
    h->g = std::make_unique<WorkerGroup>(n, rank, device, nccl_id);
    *out = h.release();
  });
}

int rtpb_ipc_unique_id(void* out128) {
  return guard([&] {
    unsigned char b[128] = {};
    FILE* f = std::fopen("/dev/urandom", "rb");
    const size_t got = f ? std::fread(b, 1, sizeof b, f) : 0;
    if (f) std::fclose(f);
    if (got != sizeof b) throw ConfigError("rtpb_ipc_unique_id: /dev/urandom unavailable");
    std::memcpy(out128, b, sizeof b);
  });
}

int rtpb_group_create_ipc(size_t n, size_t rank, int device, const void* id, rtpb_group* out) {
  return guard([&] {
    auto h = std::make_unique<rtpb_group_s>();
    h->g = std::make_unique<WorkerGroup>(n, rank, device, id, TransportKind::Ipc);
    *out = h.release();
  });
}

int rtpb_group_create_solo(size_t n, size_t rank, int device, rtpb_group* out) {
  return guard([&] {
    auto h = std::make_unique<rtpb_group_s>();
    h->g = std::make_unique<WorkerGroup>(n, rank, device, nullptr, TransportKind::Solo);
    *out = h.release();
  });
}

int rtpb_group_destroy(rtpb_group g) {
  return guard([&] { group_release(g); });
}

size_t rtpb_group_size(rtpb_group g) { return g ? g->g->size() : 0; }

size_t rtpb_group_local_ranks(rtpb_group g, size_t* ranks) {
  const auto& l = g->g->local_ranks();
  if (ranks)
    for (size_t k = 0; k < l.size(); ++k) ranks[k] = l[k];
  return l.size();
}

void* rtpb_group_stream(rtpb_group g, size_t rank, int comm) {
  try {
    Worker& w = g->g->worker(rank);
    return comm ? w.comm : w.compute;
  } catch (...) {
    return nullptr;
  }
}

int rtpb_group_device(rtpb_group g, size_t rank) {
  try {
    return g->g->worker(rank).device;
  } catch (...) {
    return -1;
  }
}

int rtpb_debug_read_flags(rtpb_group g, size_t rank, size_t first, size_t count, unsigned* host_dst,
                          int* busy_streams) {
  return guard([&] {
    Worker& w = g->g->worker(rank);
    DeviceGuard dg(w.device);
    if (first + count > Worker::kFlagPool) throw DimensionError("debug_read_flags: out of range");
    // one private stream per process, made on the first call (call once
    // before the work to watch starts); host_dst should be pinned memory
    static cudaStream_t s = nullptr;
    if (!s) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "debug stream");
    cuda_check(cudaMemcpyAsync(host_dst, w.flag(first), count * sizeof(unsigned), cudaMemcpyDeviceToHost, s),
               "debug read flags");
    cuda_check(cudaStreamSynchronize(s), "debug read flags");
    if (busy_streams) {
      int b = 0;
      if (cudaStreamQuery(w.compute) == cudaErrorNotReady) b |= 1;
      if (cudaStreamQuery(w.comm) == cudaErrorNotReady) b |= 2;
      if (cudaStreamQuery(w.aux) == cudaErrorNotReady) b |= 4;
      *busy_streams = b;
    }
  });
}

uint64_t rtpb_debug_flag_address(rtpb_group g, size_t rank, size_t index) {
  try {
    return reinterpret_cast<uint64_t>(g->g->worker(rank).flag(index));
  } catch (...) {
    return 0;
  }
}

int rtpb_group_synchronize(rtpb_group g) {
  return guard([&] { g->g->synchronize(); });
}

size_t rtpb_group_traffic(rtpb_group g, int64_t* kinds, int64_t* w_elems, int64_t* g_elems, size_t cap) {
  const auto& t = g->g->traffic();
  for (size_t k = 0; k < t.size() && k < cap; ++k) {
    const std::string kind = t[k].kind;
    if (kinds) kinds[k] = kind == "rotation_cw" ? 0 : kind == "rotation_ccw" ? 1 : 2;
    if (w_elems) w_elems[k] = int64_t(t[k].weight_elems_per_worker);
    if (g_elems) g_elems[k] = int64_t(t[k].grad_elems_per_worker);
  }
  return t.size();
}

void rtpb_group_clear_traffic(rtpb_group g) { g->g->clear_traffic(); }

int rtpb_group_corrupt_next_exchange(rtpb_group g, size_t rank, int what) {
  return guard([&] {
    g->g->corrupt_next_exchange(rank, what == 1   ? WorkerGroup::Corrupt::Tag
                                      : what == 2 ? WorkerGroup::Corrupt::ShardId
                                                  : WorkerGroup::Corrupt::None);
  });
}

int rtpb_group_ledger(rtpb_group g, size_t rank, size_t* current5, size_t* peak5, size_t* peak_total) {
  return guard([&] {
    MemoryLedger& l = g->g->ledger_of(rank);
    for (size_t c = 0; c < kNumMemCategories; ++c) {
      if (current5) current5[c] = l.current(MemCategory(c));
      if (peak5) peak5[c] = l.peak(MemCategory(c));
    }
    if (peak_total) *peak_total = l.peak_total();
  });
}

int rtpb_group_reset_ledger_peaks(rtpb_group g) {
  return guard([&] {
    for (size_t r : g->g->local_ranks()) g->g->ledger_of(r).reset_peaks();
  });
}

int rtpb_group_rotate(rtpb_group g, int op, void** weight, void** grad, void** spare, size_t w_bytes,
                      size_t g_bytes) {
  return guard([&] {
    WorkerGroup& G = *g->g;
    const size_t n = G.size();
    const auto& local = G.local_ranks();
    std::vector<void*> w(n, nullptr), gr(n, nullptr), sp(n, nullptr);
    for (size_t k = 0; k < local.size(); ++k) {
      w[local[k]] = weight[k];
      gr[local[k]] = grad ? grad[k] : nullptr;
      sp[local[k]] = spare ? spare[k] : nullptr;
    }
    const bool keep_spare = op & RTPB_ROTATE_KEEP_SPARE;
    op &= ~RTPB_ROTATE_KEEP_SPARE;
    if (op < 0 || op > 3) throw ConfigError("rotate: op must be 0..3 (optionally | RTPB_ROTATE_KEEP_SPARE)");
    const Direction dir = (op == 0 || op == 2) ? Direction::Clockwise : Direction::CounterClockwise;
    const bool with_grad = op == 1 || op == 2;
    if (n == 1) return;
    G.comm_after_compute();
    G.exchange(dir, w, spare ? sp : w, w_bytes);
    if (with_grad) G.exchange(dir, gr, gr, g_bytes);
    G.compute_after_comm();
    if (spare && !keep_spare) {
      // out-of-place: the received weight is in the spare; copy it home so
      // the caller's pointers keep their roles (raw-buffer test entry).
      for (size_t r : local) {
        Worker& wk = G.worker(r);
        DeviceGuard dg(wk.device);
        cuda_check(cudaMemcpyAsync(w[r], sp[r], w_bytes, cudaMemcpyDeviceToDevice, wk.compute), "spare copy");
      }
    }
  });
}

void rtpb_debug_skip_comm(int on) { g_skip_comm.store(on ? 1 : 0); }

int rtpb_group_allgather(rtpb_group g, void** in, void** out, size_t bytes) {
  return guard([&] {
    WorkerGroup& G = *g->g;
    const size_t n = G.size();
    const auto& local = G.local_ranks();
    std::vector<void*> i(n, nullptr), o(n, nullptr);
    for (size_t k = 0; k < local.size(); ++k) {
      i[local[k]] = in[k];
      o[local[k]] = out[k];
    }
    G.ring_allgather(i, o, bytes, "allgather", 1);
  });
}

int rtpb_linear_create(rtpb_group g, const char* label, size_t in_dim, size_t out_dim, int dtype, const double* w,
                       const double* b, uint64_t seed, uint64_t stream_base, rtpb_linear* out) {
  return guard([&] {
    auto h = std::make_unique<rtpb_linear_s>();
    h->grp = g;
    const size_t n = g->g->size();
    if ((w == nullptr) != (b == nullptr)) throw DimensionError("linear_create: pass both weight and bias, or neither");
    if (w)
      h->l = std::make_unique<RtpLinear>(*g->g, label ? label : "linear", w, b, in_dim, out_dim, n, dt(dtype));
    else
      h->l = std::make_unique<RtpLinear>(*g->g, label ? label : "linear", in_dim, out_dim, n, seed, stream_base,
                                         dt(dtype));
    ++g->refs;
    *out = h.release();
  });
}

int rtpb_linear_destroy(rtpb_linear l) {
  return guard([&] {
    if (l && l->owned) {
      rtpb_group_s* g = l->grp;
      delete l;
      group_release(g);
    }
  });
}

int rtpb_linear_set_rotation_mode(rtpb_linear l, int mode) {
  return guard([&] {
    l->l->set_rotation_mode(mode == RTPB_ROT_OUTOFPLACE ? RotationMode::OutOfPlace : RotationMode::InPlace);
  });
}

int rtpb_linear_allocate_comm_spares(rtpb_linear l) {
  return guard([&] { l->l->allocate_comm_spares(); });
}

int rtpb_linear_release_comm_spares(rtpb_linear l) {
  return guard([&] { l->l->release_comm_spares(); });
}

int rtpb_linear_zero_grads(rtpb_linear l) {
  return guard([&] { l->l->zero_grads(); });
}

size_t rtpb_linear_shard_len(rtpb_linear l) { return l->l->shard_len(); }

int rtpb_linear_forward(rtpb_linear l, const void* const* x, size_t rows, void* const* y, int mode) {
  return guard([&] {
    const size_t k = l->grp->g->local_ranks().size();
    auto xv = views(x, k);
    auto yv = views(y, k);
    l->l->forward(xv, rows, yv, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
  });
}

int rtpb_linear_backward(rtpb_linear l, const void* const* dy, size_t rows, void* const* dx) {
  return guard([&] {
    const size_t k = l->grp->g->local_ranks().size();
    auto dyv = views(dy, k);
    auto dxv = views(dx, k);
    l->l->backward(dyv, rows, dxv);
  });
}

int rtpb_linear_slot(rtpb_linear l, size_t rank, int64_t* logical_id, int64_t* rotation_offset, void** weight,
                     void** grad) {
  return guard([&] {
    if (!l->grp->g->is_local(rank)) throw IndexError("slot of a non-local rank");
    ShardSlot& s = l->l->slots()[rank];
    if (logical_id) *logical_id = int64_t(s.logical_id);
    if (rotation_offset) *rotation_offset = s.rotation_offset;
    if (weight) *weight = s.weight.data();
    if (grad) *grad = s.grad_acc.data();
  });
}

int rtpb_linear_trace(rtpb_linear l, int64_t* ids) {
  return guard([&] {
    const auto& t = l->l->trace();
    std::memcpy(ids, t.data(), t.size() * sizeof(int64_t));
  });
}

int rtpb_linear_read_shard(rtpb_linear l, size_t rank, int which, void* dst) {
  return guard([&] {
    WorkerGroup& G = *l->grp->g;
    Worker& w = G.worker(rank);
    DeviceGuard dg(w.device);
    G.synchronize();
    if (which) {
      l->l->materialize_grads();
      G.synchronize();
    }
    const Tensor& b = which ? l->l->slots()[rank].grad_acc : l->l->slots()[rank].weight;
    cuda_check(cudaMemcpy(dst, b.data(), b.bytes(), cudaMemcpyDeviceToDevice), "read_shard");
  });
}

int rtpb_mlp_create(rtpb_group g, const char* label, size_t h, size_t f, int dtype, const double* w1,
                    const double* b1, const double* w2, const double* b2, uint64_t seed, uint64_t stream_base,
                    rtpb_mlp* out) {
  return guard([&] {
    auto m = std::make_unique<rtpb_mlp_s>();
    m->grp = g;
    const std::string lab = label ? label : "mlp";
    if (w1 || b1 || w2 || b2) {
      if (!(w1 && b1 && w2 && b2)) throw DimensionError("mlp_create: pass all four parameters, or none");
      m->m = std::make_unique<RtpMlp>(*g->g, lab, h, f, dt(dtype), w1, b1, w2, b2);
    } else {
      m->m = std::make_unique<RtpMlp>(*g->g, lab, h, f, dt(dtype), seed, stream_base);
    }
    m->ffn1.grp = g;
    m->ffn2.grp = g;
    m->ffn1.owned = m->ffn2.owned = false;
    ++g->refs;
    *out = m.release();
  });
}

int rtpb_mlp_destroy(rtpb_mlp m) {
  return guard([&] {
    if (!m) return;
    m->ffn1.l.release();
    m->ffn2.l.release();
    rtpb_group_s* g = m->grp;
    delete m;
    group_release(g);
  });
}

int rtpb_mlp_set_rotation_mode(rtpb_mlp m, int mode) {
  return guard([&] {
    m->m->set_rotation_mode(mode == RTPB_ROT_OUTOFPLACE ? RotationMode::OutOfPlace : RotationMode::InPlace);
  });
}

int rtpb_mlp_begin_step(rtpb_mlp m) {
  return guard([&] { m->m->begin_step(); });
}

int rtpb_mlp_zero_grads(rtpb_mlp m) {
  return guard([&] { m->m->zero_grads(); });
}

int rtpb_mlp_forward(rtpb_mlp m, const void* const* x, size_t rows, void* const* y, int mode) {
  return guard([&] {
    const size_t k = m->grp->g->local_ranks().size();
    auto xv = views(x, k);
    auto yv = views(y, k);
    m->m->forward(xv, rows, yv, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
  });
}

int rtpb_mlp_backward(rtpb_mlp m, const void* const* dy, size_t rows, void* const* dx) {
  return guard([&] {
    const size_t k = m->grp->g->local_ranks().size();
    auto dyv = views(dy, k);
    auto dxv = views(dx, k);
    m->m->backward(dyv, rows, dxv);
  });
}

int rtpb_mlp_chain(rtpb_mlp m, rtpb_mlp next) {
  return guard([&] { m->m->chain(next ? next->m.get() : nullptr); });
}

rtpb_linear rtpb_mlp_layer(rtpb_mlp m, int layer) {
  rtpb_linear_s& v = layer == 0 ? m->ffn1 : m->ffn2;
  // Non-owning view: the unique_ptr aliases the MLP's layer and is released
  // (never deleted) in rtpb_mlp_destroy.
  if (!v.l) v.l.reset(layer == 0 ? &m->m->ffn1() : &m->m->ffn2());
  return &v;
}

int rtpb_attention_create(rtpb_group g, const char* label, size_t hidden, size_t heads, size_t seq, int dtype,
                          const double* wq, const double* wk, const double* wv, const double* wo,
                          rtpb_attention* out) {
  return guard([&] {
    if (!wq || !wk || !wv || !wo) throw DimensionError("attention_create: all four projection weights are required");
    auto h = std::make_unique<rtpb_attention_s>();
    h->grp = g;
    h->a = std::make_unique<RtpAttention>(*g->g, label ? label : "attn", wq, wk, wv, wo, hidden, heads, seq,
                                          g->g->size(), dt(dtype));
    ++g->refs;
    *out = h.release();
  });
}

int rtpb_attention_destroy(rtpb_attention a) {
  return guard([&] {
    if (a) {
      rtpb_group_s* g = a->grp;
      delete a;
      group_release(g);
    }
  });
}

int rtpb_attention_set_rotation_mode(rtpb_attention a, int mode) {
  return guard([&] { a->a->set_rotation_mode(mode == RTPB_ROT_OUTOFPLACE ? RotationMode::OutOfPlace : RotationMode::InPlace); });
}
int rtpb_attention_allocate_comm_spares(rtpb_attention a) { return guard([&] { a->a->allocate_comm_spares(); }); }
int rtpb_attention_release_comm_spares(rtpb_attention a) { return guard([&] { a->a->release_comm_spares(); }); }
int rtpb_attention_zero_grads(rtpb_attention a) { return guard([&] { a->a->zero_grads(); }); }
size_t rtpb_attention_shard_len(rtpb_attention a) { return a ? a->a->shard_len() : 0; }

int rtpb_attention_forward(rtpb_attention a, const void* const* x, size_t rows, void* const* y, int mode) {
  return guard([&] {
    const size_t k = a->grp->g->local_ranks().size();
    auto xv = views(x, k);
    auto yv = views(y, k);
    a->a->forward(xv, rows, yv, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
  });
}

int rtpb_attention_backward(rtpb_attention a, const void* const* dy, size_t rows, void* const* dx) {
  return guard([&] {
    const size_t k = a->grp->g->local_ranks().size();
    auto dyv = views(dy, k);
    auto dxv = views(dx, k);
    a->a->backward(dyv, rows, dxv);
  });
}

int rtpb_attention_slot(rtpb_attention a, size_t rank, int64_t* logical_id, int64_t* rotation_offset) {
  return guard([&] {
    if (!a->grp->g->is_local(rank)) throw IndexError("slot of a non-local rank");
    ShardSlot& s = a->a->slots()[rank];
    if (logical_id) *logical_id = int64_t(s.logical_id);
    if (rotation_offset) *rotation_offset = s.rotation_offset;
  });
}

int rtpb_attention_trace(rtpb_attention a, int64_t* ids) {
  return guard([&] {
    const auto& t = a->a->trace();
    std::memcpy(ids, t.data(), t.size() * sizeof(int64_t));
  });
}

int rtpb_attention_read_shard(rtpb_attention a, size_t rank, int which, double* dst) {
  return guard([&] {
    const std::vector<double> v = a->a->shard_host(rank, which != 0);
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

int rtpb_embedding_create(rtpb_group g, const char* label, size_t vocab, size_t emb, int dtype, const double* table,
                          rtpb_embedding* out) {
  return guard([&] {
    if (!table) throw DimensionError("embedding_create: table is required");
    auto h = std::make_unique<rtpb_embedding_s>();
    h->grp = g;
    h->e = std::make_unique<RtpEmbedding>(*g->g, label ? label : "emb", table, vocab, emb, g->g->size(), dt(dtype));
    ++g->refs;
    *out = h.release();
  });
}
int rtpb_embedding_destroy(rtpb_embedding e) { return layer_destroy(e); }
int rtpb_embedding_set_rotation_mode(rtpb_embedding e, int mode) {
  return guard([&] { e->e->set_rotation_mode(rot(mode)); });
}
int rtpb_embedding_allocate_comm_spares(rtpb_embedding e) { return guard([&] { e->e->allocate_comm_spares(); }); }
int rtpb_embedding_release_comm_spares(rtpb_embedding e) { return guard([&] { e->e->release_comm_spares(); }); }
int rtpb_embedding_zero_grads(rtpb_embedding e) { return guard([&] { e->e->zero_grads(); }); }
size_t rtpb_embedding_shard_len(rtpb_embedding e) { return e ? e->e->shard_len() : 0; }
int rtpb_embedding_forward(rtpb_embedding e, const int64_t* const* ids, const size_t* counts, void* const* y,
                           int mode) {
  return guard([&] {
    const size_t k = e->grp->g->local_ranks().size();
    std::vector<std::vector<int64_t>> v(k);
    for (size_t i = 0; i < k; ++i) v[i].assign(ids[i], ids[i] + counts[i]);
    auto yv = views(y, k);
    e->e->forward(v, yv, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
  });
}
int rtpb_embedding_backward(rtpb_embedding e, const void* const* dy, size_t rows) {
  return guard([&] {
    const size_t k = e->grp->g->local_ranks().size();
    auto dyv = views(dy, k);
    e->e->backward(dyv, rows);
  });
}
int rtpb_embedding_slot(rtpb_embedding e, size_t rank, int64_t* logical_id, int64_t* rotation_offset) {
  return guard([&] { slot_of(*e->e, *e->grp->g, rank, logical_id, rotation_offset); });
}
int rtpb_embedding_read_shard(rtpb_embedding e, size_t rank, int which, double* dst) {
  return guard([&] { read_host(*e->e, *e->grp->g, rank, which, dst); });
}

int rtpb_moe_create(rtpb_group g, const char* label, size_t hidden, size_t ffn, int dtype, const double* gate,
                    const double* const* experts, rtpb_moe* out) {
  return guard([&] {
    if (!gate || !experts) throw DimensionError("moe_create: gate and experts are required");
    auto h = std::make_unique<rtpb_moe_s>();
    h->grp = g;
    h->m = std::make_unique<RtpMoe>(*g->g, label ? label : "moe", gate, experts, hidden, ffn, g->g->size(),
                                    dt(dtype));
    ++g->refs;
    *out = h.release();
  });
}
int rtpb_moe_destroy(rtpb_moe m) { return layer_destroy(m); }
int rtpb_moe_set_rotation_mode(rtpb_moe m, int mode) { return guard([&] { m->m->set_rotation_mode(rot(mode)); }); }
int rtpb_moe_allocate_comm_spares(rtpb_moe m) { return guard([&] { m->m->allocate_comm_spares(); }); }
int rtpb_moe_release_comm_spares(rtpb_moe m) { return guard([&] { m->m->release_comm_spares(); }); }
int rtpb_moe_zero_grads(rtpb_moe m) { return guard([&] { m->m->zero_grads(); }); }
size_t rtpb_moe_shard_len(rtpb_moe m) { return m ? m->m->shard_len() : 0; }
int rtpb_moe_forward(rtpb_moe m, const void* const* x, size_t rows, void* const* y, int mode) {
  return guard([&] {
    const size_t k = m->grp->g->local_ranks().size();
    auto xv = views(x, k);
    auto yv = views(y, k);
    m->m->forward(xv, rows, yv, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
  });
}
int rtpb_moe_backward(rtpb_moe m, const void* const* dy, size_t rows, void* const* dx) {
  return guard([&] {
    const size_t k = m->grp->g->local_ranks().size();
    auto dyv = views(dy, k);
    auto dxv = views(dx, k);
    m->m->backward(dyv, rows, dxv);
  });
}
int rtpb_moe_slot(rtpb_moe m, size_t rank, int64_t* logical_id, int64_t* rotation_offset) {
  return guard([&] { slot_of(*m->m, *m->grp->g, rank, logical_id, rotation_offset); });
}
int rtpb_moe_read_shard(rtpb_moe m, size_t rank, int which, double* dst) {
  return guard([&] { read_host(*m->m, *m->grp->g, rank, which, dst); });
}
int rtpb_moe_gate_grad(rtpb_moe m, size_t rank, double* dst) {
  return guard([&] {
    if (!m->grp->g->is_local(rank)) throw IndexError("gate gradient of a non-local rank");
    m->grp->g->synchronize();
    const std::vector<double> v = m->m->gate_grad(rank).to_host();
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

int rtpb_linear_set_option(rtpb_linear l, int option, int value) {
  return guard([&] {
    if (option == RTPB_OPT_EXACT_GELU)
      l->l->set_exact_gelu(value != 0);
    else if (option == RTPB_OPT_PAIRED_DX)
      l->l->set_paired_dx(value != 0);
    else
      throw ConfigError("unknown option " + std::to_string(option));
  });
}

int rtpb_mlp_set_option(rtpb_mlp m, int option, int value) {
  return guard([&] {
    if (option == RTPB_OPT_EXACT_GELU)
      m->m->set_exact_gelu(value != 0);
    else if (option == RTPB_OPT_PAIRED_DX)
      m->m->set_paired_dx(value != 0);
    else
      throw ConfigError("unknown option " + std::to_string(option));
  });
}

int rtpb_model_create(rtpb_group g, size_t heads, size_t hidden, size_t layers, size_t seq, size_t vocab, size_t ffn,
                      int moe, uint64_t seed, int rotation_mode, int dtype, rtpb_model* out) {
  return guard([&] {
    ModelDims d;
    d.heads = heads;
    d.hidden = hidden;
    d.layers = layers;
    d.seq = seq;
    d.vocab = vocab;
    d.ffn = ffn;
    d.moe = moe != 0;
    d.n_experts = moe ? g->g->size() : 1;
    auto h = std::make_unique<rtpb_model_s>();
    h->grp = g;
    h->m = std::make_unique<RtpModel>(d, seed, *g->g, rot(rotation_mode), dt(dtype));
    ++g->refs;
    *out = h.release();
  });
}
int rtpb_model_destroy(rtpb_model m) { return layer_destroy(m); }
int rtpb_model_begin_step(rtpb_model m) { return guard([&] { m->m->begin_step(); }); }
int rtpb_model_zero_grads(rtpb_model m) { return guard([&] { m->m->zero_grads(); }); }
int rtpb_model_forward(rtpb_model m, const int64_t* const* ids, const size_t* counts, void* const* logits, int mode) {
  return guard([&] {
    WorkerGroup& G = *m->grp->g;
    const size_t k = G.local_ranks().size();
    std::vector<std::vector<int64_t>> v(k);
    for (size_t i = 0; i < k; ++i) v[i].assign(ids[i], ids[i] + counts[i]);
    auto out = m->m->forward(v, mode == RTPB_MODE_EVAL ? Mode::Eval : Mode::Train);
    for (size_t i = 0; i < k; ++i) {
      DeviceGuard dg(out[i].device());
      cuda_check(cudaMemcpy(logits[i], out[i].data(), out[i].bytes(), cudaMemcpyDeviceToDevice), "model logits");
    }
  });
}
int rtpb_model_backward(rtpb_model m, const void* const* dlogits, size_t rows) {
  return guard([&] {
    WorkerGroup& G = *m->grp->g;
    const auto& local = G.local_ranks();
    const size_t V = m->m->dims().vocab;
    const DType d = m->m->head().dtype();
    std::vector<Tensor> t(local.size());
    for (size_t i = 0; i < local.size(); ++i) {
      Worker& w = G.worker(local[i]);
      t[i] = Tensor({rows, V}, d, w.device, &w.ledger, MemCategory::Activation, false);
      DeviceGuard dg(w.device);
      cuda_check(cudaMemcpy(t[i].data(), dlogits[i], t[i].bytes(), cudaMemcpyDeviceToDevice), "model dlogits");
    }
    m->m->backward(t);
  });
}
size_t rtpb_model_layer_count(rtpb_model m) { return m ? m->m->all_layers().size() : 0; }
size_t rtpb_model_layer_shard_len(rtpb_model m, size_t layer) {
  if (!m) return 0;
  auto all = m->m->all_layers();
  return layer < all.size() ? all[layer]->shard_len() : 0;
}
int rtpb_model_read_layer_shard(rtpb_model m, size_t layer, size_t rank, int which, double* dst) {
  return guard([&] {
    auto all = m->m->all_layers();
    if (layer >= all.size()) throw IndexError("layer index out of range");
    const std::vector<double> v = all[layer]->shard_host(rank, which != 0);
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}
int rtpb_model_gate_grad(rtpb_model m, size_t block, size_t rank, double* dst) {
  return guard([&] {
    auto& blocks = m->m->rtp_blocks();
    if (block >= blocks.size() || !blocks[block].moe) throw IndexError("not an MoE block");
    if (!m->grp->g->is_local(rank)) throw IndexError("gate gradient of a non-local rank");
    m->grp->g->synchronize();
    const std::vector<double> v = blocks[block].moe->gate_grad(rank).to_host();
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
  });
}

}  // extern "C"
