// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference C++ sources, which
// oracle/Makefile compiles by path from /root/reference/proj/src into
// oracle/_ref/librtpref.so. Nothing here re-implements the algorithm: every
// function drives the reference's own public classes
// (rtp::RtpLinear, rtp::SerialLinear, rtp::WorkerGroup, rtp::gelu, ...)
// exactly as its own callers do (model.cpp:77-83 / 99-105 for the MLP,
// layers_test.cpp:86-113 for a single linear). Only tests/, the golden
// fixture generator and bench.py's reference arm load this library.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <sstream>

#include "rtp/analysis.hpp"
#include "rtp/commands.hpp"
#include "rtp/config.hpp"
#include "rtp/layers.hpp"
#include "rtp/ledger.hpp"
#include "rtp/model.hpp"
#include "rtp/partition.hpp"
#include "rtp/ring.hpp"
#include "rtp/serial.hpp"
#include "rtp/tensor.hpp"

using namespace rtp;

namespace {
thread_local std::string g_err;

Tensor from_ptr(std::vector<size_t> shape, const double* p) {
  size_t n = 1;
  for (size_t d : shape) n *= d;
  return Tensor(std::move(shape), std::vector<double>(p, p + n));
}

void to_ptr(const Tensor& t, double* p) { std::memcpy(p, t.data(), t.numel() * sizeof(double)); }

TransportKind kind_of(int transport) {
  return transport ? TransportKind::Concurrent : TransportKind::Lockstep;
}

std::vector<Tensor> shard(const Tensor& t, size_t n) { return shard_rows(t, t.rows(), n); }

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD(...)                                               \
  try {                                                              \
    __VA_ARGS__;                                                     \
    return 0;                                                        \
  } catch (const ConfigError& e) { return fail(e, 2); }              \
  catch (const DimensionError& e) { return fail(e, 3); }             \
  catch (const ProtocolError& e) { return fail(e, 4); }              \
  catch (const StateError& e) { return fail(e, 5); }                 \
  catch (const std::exception& e) { return fail(e, 1); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// SplitMix64(seed) -> `count` draws of Tensor::uniform(lo, hi) (tensor.cpp:99-103).
int ref_uniform(uint64_t seed, uint64_t skip, uint64_t count, double lo, double hi, double* out) {
  REF_GUARD({
    SplitMix64 rng(seed);
    for (uint64_t i = 0; i < skip; ++i) rng.next_u64();
    Tensor t = Tensor::uniform({count}, rng, lo, hi);
    to_ptr(t, out);
  })
}

// Shard r of flatten_shards(linear_shard_groups(w, b, n)) (layers_common.cpp:33-45,
// partition.cpp:49-56): the exact bytes RtpLayerBase::init_slots gives worker r.
int ref_linear_shard(size_t in, size_t out, size_t n, size_t r, const double* w, const double* b,
                     double* shard_out) {
  REF_GUARD({
    Tensor W = from_ptr({in, out}, w), B = from_ptr({out}, b);
    FlatParameter fp = flatten_shards(linear_shard_groups(W, B, n));
    to_ptr(shard_view(fp, r), shard_out);
  })
}

// The SerialModel draw order restricted to the FFN block (serial.cpp:329-353):
// ffn1.w (h x f), ffn1.b (f), ffn2.w (f x h), ffn2.b (h) for `blocks` blocks,
// each drawn from one SplitMix64(seed) stream with U[-0.1, 0.1].
int ref_mlp_params(uint64_t seed, size_t h, size_t f, size_t blocks, double* out) {
  REF_GUARD({
    SplitMix64 rng(seed);
    double* p = out;
    for (size_t l = 0; l < blocks; ++l) {
      for (auto shape : {std::vector<size_t>{h, f}, std::vector<size_t>{f},
                         std::vector<size_t>{f, h}, std::vector<size_t>{h}}) {
        Tensor t = Tensor::uniform(shape, rng, -0.1, 0.1);
        to_ptr(t, p);
        p += t.numel();
      }
    }
  })
}

// SerialLinear fwd (Train) + bwd from zeroed grads (serial.cpp:59-77).
int ref_serial_linear(size_t rows, size_t in, size_t out, const double* w, const double* b,
                      const double* x, const double* dy, double* y, double* dx, double* gw,
                      double* gb) {
  REF_GUARD({
    SerialLinear lin(from_ptr({in, out}, w), from_ptr({out}, b));
    lin.zero_grads();
    Tensor Y = lin.forward(from_ptr({rows, in}, x), Mode::Train);
    Tensor DX = lin.backward(from_ptr({rows, out}, dy));
    to_ptr(Y, y);
    to_ptr(DX, dx);
    to_ptr(lin.gw, gw);
    to_ptr(lin.gb, gb);
  })
}

// RtpLinear fwd (Train) + bwd on a WorkerGroup of n (layers_linear.cpp:18-72),
// batch-major row shards (model.cpp:165-178). Outputs gathered y/dx, every
// rank's grad_acc shard (n * shard_len), the per-rank logical id after
// forward (fwd_ids[n]) and after backward (bwd_ids[n]), and the traffic log as
// (kind: 0 cw, 1 ccw, 2 allgather; w_elems; g_elems) triples.
int ref_rtp_linear(size_t n, int transport, int outofplace, size_t rows, size_t in, size_t out,
                   const double* w, const double* b, const double* x, const double* dy,
                   double* y, double* dx, double* grads, int64_t* fwd_ids, int64_t* bwd_ids,
                   int64_t* traffic, size_t* n_traffic) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    RtpLinear layer(g, "lin", from_ptr({in, out}, w), from_ptr({out}, b), n);
    layer.set_rotation_mode(outofplace ? RotationMode::OutOfPlace : RotationMode::InPlace);
    if (outofplace) layer.allocate_comm_spares();
    layer.zero_grads();
    auto ys = layer.forward(shard(from_ptr({rows, in}, x), n), Mode::Train);
    for (size_t r = 0; r < n; ++r) fwd_ids[r] = int64_t(layer.slots()[r].logical_id);
    auto dxs = layer.backward(shard(from_ptr({rows, out}, dy), n));
    for (size_t r = 0; r < n; ++r) bwd_ids[r] = int64_t(layer.slots()[r].logical_id);
    to_ptr(concat(ys, 0), y);
    to_ptr(concat(dxs, 0), dx);
    const size_t L = layer.shard_len();
    for (size_t r = 0; r < n; ++r) to_ptr(layer.slots()[r].grad_acc, grads + r * L);
    size_t k = 0;
    for (const auto& rec : g.traffic()) {
      const std::string kind = rec.kind;
      traffic[3 * k + 0] = kind == "rotation_cw" ? 0 : kind == "rotation_ccw" ? 1 : 2;
      traffic[3 * k + 1] = int64_t(rec.weight_elems_per_worker);
      traffic[3 * k + 2] = int64_t(rec.grad_elems_per_worker);
      ++k;
    }
    *n_traffic = k;
  })
}

// RtpAttention fwd (Train) + bwd (layers_attention.cpp:43-198) on a
// WorkerGroup of n, batch-major row shards; grads: n * shard_len.
int ref_rtp_attention(size_t n, int transport, size_t rows, size_t hidden, size_t heads, size_t seq,
                      const double* wq, const double* wk, const double* wv, const double* wo,
                      const double* x, const double* dy, double* y, double* dx, double* grads) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    RtpAttention attn(g, "attn", from_ptr({hidden, hidden}, wq), from_ptr({hidden, hidden}, wk),
                      from_ptr({hidden, hidden}, wv), from_ptr({hidden, hidden}, wo), heads, seq, n);
    attn.zero_grads();
    auto ys = attn.forward(shard(from_ptr({rows, hidden}, x), n), Mode::Train);
    auto dxs = attn.backward(shard(from_ptr({rows, hidden}, dy), n));
    to_ptr(concat(ys, 0), y);
    to_ptr(concat(dxs, 0), dx);
    const size_t L = attn.shard_len();
    for (size_t r = 0; r < n; ++r) to_ptr(attn.slots()[r].grad_acc, grads + r * L);
  })
}

// The FFN block exactly as RtpModel composes it (model.cpp:77-83 forward,
// 99-105 backward): pre = ffn1(x); h = gelu(pre); y = ffn2(h);
// dh = ffn2.backward(dy); dpre = gelu_backward(pre, dh); dx = ffn1.backward(dpre).
// Residual adds (model.cpp:72,85,108) are outside the MLP unit and omitted.
// grads1 / grads2: n * shard_len of ffn1 / ffn2.
int ref_rtp_mlp(size_t n, int transport, int outofplace, size_t rows, size_t h, size_t f,
                const double* w1, const double* b1, const double* w2, const double* b2,
                const double* x, const double* dy, double* y, double* dx, double* grads1,
                double* grads2) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    RtpLinear ffn1(g, "ffn1", from_ptr({h, f}, w1), from_ptr({f}, b1), n);
    RtpLinear ffn2(g, "ffn2", from_ptr({f, h}, w2), from_ptr({h}, b2), n);
    for (RtpLinear* l : {&ffn1, &ffn2}) {
      l->set_rotation_mode(outofplace ? RotationMode::OutOfPlace : RotationMode::InPlace);
      if (outofplace) l->allocate_comm_spares();
      l->zero_grads();
    }
    auto pre = ffn1.forward(shard(from_ptr({rows, h}, x), n), Mode::Train);
    std::vector<Tensor> hs(n), pre_cache(n);
    g.each([&](size_t r) {
      hs[r] = gelu(pre[r]);
      pre_cache[r] = std::move(pre[r]);
    });
    auto ys = ffn2.forward(hs, Mode::Train);
    auto dh = ffn2.backward(shard(from_ptr({rows, h}, dy), n));
    std::vector<Tensor> dpre(n);
    g.each([&](size_t r) { dpre[r] = gelu_backward(pre_cache[r], dh[r]); });
    auto dxs = ffn1.backward(dpre);
    to_ptr(concat(ys, 0), y);
    to_ptr(concat(dxs, 0), dx);
    const size_t L1 = ffn1.shard_len(), L2 = ffn2.shard_len();
    for (size_t r = 0; r < n; ++r) {
      to_ptr(ffn1.slots()[r].grad_acc, grads1 + r * L1);
      to_ptr(ffn2.slots()[r].grad_acc, grads2 + r * L2);
    }
  })
}

// Wall-clock seconds of `iters` MLP fwd+bwd steps through the reference
// (same composition as ref_rtp_mlp), for bench.py's reference arm. Inputs are
// drawn once from the fixture stream; only the layer calls are timed.
int ref_time_mlp(size_t n, int transport, size_t rows, size_t h, size_t f, uint64_t seed,
                 int iters, double* seconds) {
  REF_GUARD({
    SplitMix64 prng(seed);
    Tensor w1 = Tensor::uniform({h, f}, prng, -0.1, 0.1), b1 = Tensor::uniform({f}, prng, -0.1, 0.1);
    Tensor w2 = Tensor::uniform({f, h}, prng, -0.1, 0.1), b2 = Tensor::uniform({h}, prng, -0.1, 0.1);
    SplitMix64 xrng(seed ^ 0xA5A5A5A5A5A5A5A5ULL);
    Tensor x = Tensor::uniform({rows, h}, xrng, -1, 1), dy = Tensor::uniform({rows, h}, xrng, -1, 1);
    WorkerGroup g(n, kind_of(transport));
    RtpLinear ffn1(g, "ffn1", w1, b1, n), ffn2(g, "ffn2", w2, b2, n);
    auto xs = shard(x, n), dys = shard(dy, n);
    double total = 0;
    for (int it = 0; it < iters; ++it) {
      ffn1.zero_grads();
      ffn2.zero_grads();
      auto t0 = std::chrono::steady_clock::now();
      auto pre = ffn1.forward(xs, Mode::Train);
      std::vector<Tensor> hs(n), pc(n);
      g.each([&](size_t r) {
        hs[r] = gelu(pre[r]);
        pc[r] = std::move(pre[r]);
      });
      auto ys = ffn2.forward(hs, Mode::Train);
      auto dh = ffn2.backward(dys);
      std::vector<Tensor> dpre(n);
      g.each([&](size_t r) { dpre[r] = gelu_backward(pc[r], dh[r]); });
      auto dxs = ffn1.backward(dpre);
      total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    *seconds = total;
  })
}

// Peak ledger bytes per category for one MLP step (two RtpLinear), per-rank
// ledgers bound as ledger_instrumented_run does (analysis.cpp:286-318).
// peaks[5] = max over ranks of {Param, Grad, Activation, CommBuffer, Other}.
int ref_mlp_ledger(size_t n, int outofplace, size_t rows, size_t h, size_t f, uint64_t seed,
                   size_t* peaks, size_t* flat_param_bytes) {
  REF_GUARD({
    SplitMix64 prng(seed);
    Tensor w1 = Tensor::uniform({h, f}, prng, -0.1, 0.1), b1 = Tensor::uniform({f}, prng, -0.1, 0.1);
    Tensor w2 = Tensor::uniform({f, h}, prng, -0.1, 0.1), b2 = Tensor::uniform({h}, prng, -0.1, 0.1);
    SplitMix64 xrng(seed ^ 0xA5A5A5A5A5A5A5A5ULL);
    Tensor x = Tensor::uniform({rows, h}, xrng, -1, 1), dy = Tensor::uniform({rows, h}, xrng, -1, 1);
    std::vector<MemoryLedger> ledgers(n);
    std::vector<MemoryLedger*> lp(n);
    for (size_t r = 0; r < n; ++r) lp[r] = &ledgers[r];
    WorkerGroup g(n, TransportKind::Lockstep);
    g.bind_ledgers(lp);
    RtpLinear ffn1(g, "ffn1", w1, b1, n), ffn2(g, "ffn2", w2, b2, n);
    for (RtpLinear* l : {&ffn1, &ffn2}) {
      l->set_rotation_mode(outofplace ? RotationMode::OutOfPlace : RotationMode::InPlace);
      if (outofplace) l->allocate_comm_spares();
    }
    std::vector<Tensor> xs(n), dys(n);
    {
      auto xr = shard(x, n), dr = shard(dy, n);
      g.each([&](size_t r) {
        CategoryScope s(MemCategory::Other);
        xs[r] = xr[r];
        dys[r] = dr[r];
      });
    }
    auto pre = ffn1.forward(xs, Mode::Train);
    std::vector<Tensor> hs(n), pc(n);
    g.each([&](size_t r) {
      hs[r] = gelu(pre[r]);
      pc[r] = std::move(pre[r]);
    });
    auto ys = ffn2.forward(hs, Mode::Train);
    auto dh = ffn2.backward(dys);
    std::vector<Tensor> dpre(n);
    g.each([&](size_t r) { dpre[r] = gelu_backward(pc[r], dh[r]); });
    auto dxs = ffn1.backward(dpre);
    for (size_t c = 0; c < kNumMemCategories; ++c) {
      size_t mx = 0;
      for (size_t r = 0; r < n; ++r) mx = std::max(mx, ledgers[r].peak(static_cast<MemCategory>(c)));
      peaks[c] = mx;
    }
    *flat_param_bytes = ffn1.flat_param_bytes() + ffn2.flat_param_bytes();
  })
}

// Ring primitive on id-encoded slots (ring_test.cpp:16-28): slot r's weight
// holds r*100+i, grad holds r. ops[k] = 0 cw(W), 1 ccw(W+G), 2 cw(W+G), 3 ccw(W).
// Returns per-rank logical_id, rotation_offset and weight[0] after all ops.
int ref_ring_ops(size_t n, int transport, const int* ops, size_t n_ops, size_t len,
                 int64_t* ids, int64_t* offsets, double* w0, double* g0) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    std::vector<ShardSlot> slots(n);
    for (size_t r = 0; r < n; ++r) {
      slots[r].weight = Tensor({len});
      for (size_t i = 0; i < len; ++i) slots[r].weight.at(i) = double(r * 100 + i);
      slots[r].grad_acc = Tensor({len});
      slots[r].grad_acc.fill(double(r));
      slots[r].logical_id = r;
    }
    for (size_t k = 0; k < n_ops; ++k) {
      switch (ops[k]) {
        case 0: g.rotate_clockwise(slots, PayloadKind::Weight); break;
        case 1: g.rotate_counterclockwise(slots, PayloadKind::WeightAndGrad); break;
        case 2: g.rotate_clockwise(slots, PayloadKind::WeightAndGrad); break;
        default: g.rotate_counterclockwise(slots, PayloadKind::Weight); break;
      }
    }
    for (size_t r = 0; r < n; ++r) {
      ids[r] = int64_t(slots[r].logical_id);
      offsets[r] = slots[r].rotation_offset;
      w0[r] = slots[r].weight.at(0);
      g0[r] = slots[r].grad_acc.at(0);
    }
  })
}

// table1_memory (analysis.cpp:32-49): {activation, param+grad, duplication}.
int ref_table1(int strategy, uint64_t W, uint64_t G, uint64_t A, uint64_t Ap, uint64_t N,
               uint64_t* out3) {
  REF_GUARD({
    MemoryBreakdown m = table1_memory(static_cast<Strategy>(strategy), W, G, A, Ap, N);
    out3[0] = m.activation_mem;
    out3[1] = m.param_mem;
    out3[2] = m.duplication;
  })
}

// RtpMoe (layers_moe.cpp:18-198): gate (hidden x n), n experts of
// [w1 (hidden x f) | b1 (f) | w2 (f x hidden) | b2 (hidden)] packed per expert
// in `experts` (n * (2*hidden*f + f + hidden)); one Train forward + backward
// from zeroed gradients. grads: n * shard_len; gate_grads: n * hidden * n
// (per worker, before any data-parallel combine).
int ref_rtp_moe(size_t n, int transport, size_t rows, size_t hidden, size_t f, const double* gate,
                const double* experts, const double* x, const double* dy, double* y, double* dx,
                double* grads, double* gate_grads) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    std::vector<ExpertParams> ex(n);
    const size_t per = 2 * hidden * f + f + hidden;
    for (size_t e = 0; e < n; ++e) {
      const double* p = experts + e * per;
      ex[e].w1 = from_ptr({hidden, f}, p);
      ex[e].b1 = from_ptr({f}, p + hidden * f);
      ex[e].w2 = from_ptr({f, hidden}, p + hidden * f + f);
      ex[e].b2 = from_ptr({hidden}, p + hidden * f + f + f * hidden);
    }
    RtpMoe moe(g, "moe", from_ptr({hidden, n}, gate), ex, n);
    moe.zero_grads();
    auto ys = moe.forward(shard(from_ptr({rows, hidden}, x), n), Mode::Train);
    auto dxs = moe.backward(shard(from_ptr({rows, hidden}, dy), n));
    to_ptr(concat(ys, 0), y);
    to_ptr(concat(dxs, 0), dx);
    const size_t L = moe.shard_len();
    for (size_t r = 0; r < n; ++r) {
      to_ptr(moe.slots()[r].grad_acc, grads + r * L);
      to_ptr(moe.gate_grad(r), gate_grads + r * hidden * n);
    }
  })
}

// RtpEmbedding (layers_linear.cpp:74-136): table vocab x emb, ids[r] the
// rows_per_worker token ids of worker r; Train forward + backward.
// y: (n * rows_per_worker) x emb, grads: n * shard_len (vocab x emb/n each).
int ref_rtp_embedding(size_t n, int transport, size_t vocab, size_t emb, size_t rows_per_worker,
                      const double* table, const int64_t* ids, const double* dy, double* y, double* grads) {
  REF_GUARD({
    WorkerGroup g(n, kind_of(transport));
    RtpEmbedding layer(g, "emb", from_ptr({vocab, emb}, table), n);
    layer.zero_grads();
    std::vector<std::vector<int64_t>> id(n);
    for (size_t r = 0; r < n; ++r) id[r].assign(ids + r * rows_per_worker, ids + (r + 1) * rows_per_worker);
    auto ys = layer.forward(id, Mode::Train);
    layer.backward(shard(from_ptr({n * rows_per_worker, emb}, dy), n));
    to_ptr(concat(ys, 0), y);
    const size_t L = layer.shard_len();
    for (size_t r = 0; r < n; ++r) to_ptr(layer.slots()[r].grad_acc, grads + r * L);
  })
}

// The reference's own report commands (commands.cpp:87-181): which 0 =
// cmd_memtable (analytic, no literals), 1 = cmd_ledger, 2 = cmd_sweep over
// per-worker batches {1, 2}; default ExperimentConfig with n_workers, strategy
// and batch_size set. The CSV text is copied into out (NUL-terminated).
int ref_cmd_csv(int which, size_t n, const char* strategy, size_t batch, char* out, size_t cap) {
  REF_GUARD({
    ExperimentConfig cfg;
    cfg.n_workers = n;
    cfg.strategy = strategy;
    cfg.batch_size = batch;
    std::ostringstream csv, summary;
    if (which == 0) {
      cmd_memtable(cfg, std::nullopt, csv);
    } else if (which == 1) {
      cmd_ledger(cfg, csv, summary);
    } else {
      const size_t b[2] = {1, 2};
      cmd_sweep(cfg, b, csv);
    }
    const std::string t = csv.str();
    if (t.size() + 1 > cap) throw DimensionError("ref_cmd_csv: output buffer too small");
    std::memcpy(out, t.c_str(), t.size() + 1);
  })
}

// The whole RtpModel (model.cpp:7-121): SerialModel(dims, seed) parameters
// (serial.cpp:325-353), make_batch_fixture ids / MSE target, Train forward,
// dlogits = mse_grad, backward — verify.cpp:54-79's equivalence run. Outputs:
// ids (batch*seq), logits and dlogits ((batch*seq) x vocab, rank-major),
// grads: every layer of all_layers() in order, n * shard_len each
// (layer_lens[l] = shard_len), gate_grads: per MoE block n * hidden * n.
// Query sizes with grads == nullptr: *n_layers and layer_lens are filled.
int ref_rtp_model(size_t n, int transport, int oop, size_t heads, size_t hidden, size_t layers, size_t seq,
                  size_t vocab, size_t ffn, int moe, uint64_t seed, size_t batch, int64_t* ids, double* logits,
                  double* dlogits, double* grads, double* gate_grads, size_t* n_layers, size_t* layer_lens) {
  REF_GUARD({
    ModelDims d;
    d.heads = heads;
    d.hidden = hidden;
    d.layers = layers;
    d.seq = seq;
    d.vocab = vocab;
    d.ffn = ffn;
    d.moe = moe != 0;
    d.n_experts = moe ? n : 1;
    SerialModel serial(d, seed);
    WorkerGroup g(n, kind_of(transport));
    RtpModel model(serial, g, oop ? RotationMode::OutOfPlace : RotationMode::InPlace);
    auto all = model.all_layers();
    *n_layers = all.size();
    for (size_t l = 0; l < all.size(); ++l) layer_lens[l] = all[l]->shard_len();
    if (!grads) return 0;
    BatchFixture fx = make_batch_fixture(d, batch, seed);
    std::memcpy(ids, fx.ids.data(), fx.ids.size() * sizeof(int64_t));
    auto ids_sh = shard_ids(fx, n);
    auto target_sh = shard_rows(fx.target, batch, n);
    model.zero_grads();
    model.begin_step();
    auto out = model.forward(ids_sh, Mode::Train);
    std::vector<Tensor> dl(n);
    for (size_t r = 0; r < n; ++r) dl[r] = mse_grad(out[r], target_sh[r], fx.target.numel());
    model.backward(dl);
    to_ptr(concat(out, 0), logits);
    to_ptr(concat(dl, 0), dlogits);
    double* gp = grads;
    for (RtpLayerBase* l : all)
      for (size_t r = 0; r < n; ++r) {
        to_ptr(l->slots()[r].grad_acc, gp);
        gp += l->shard_len();
      }
    if (moe) {
      double* q = gate_grads;
      for (auto& b : model.rtp_blocks())
        for (size_t r = 0; r < n; ++r) {
          to_ptr(b.moe->gate_grad(r), q);
          q += hidden * n;
        }
    }
  })
}

}  // extern "C"
