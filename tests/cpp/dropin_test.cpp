// Drop-in check of the C++ host API (include/rtpb/rtp.hpp) against the
// reference's own unit tests, compiled as a reference caller would be: the
// reference's layers_test.cpp:27-123,343-385 and ring_test.cpp:39-200 cases,
// ported onto rtpb:: by changing the namespace and the element checks.
//
// Differences from the reference tests, all forced by the device path:
//  * dimensions: `in` and `out / n` are multiples of 8 (16-byte TMA rows,
//    DESIGN §1), so the tiny 2x4 / 3x6 / 5x8 layers become 16 x 32 / 16 x 48 /
//    16 x 64 with the same structure;
//  * numerics: the reference is fp64 and checks max_rel_diff < 1e-10; a layer
//    built from fp64 Tensors here computes in fp32 mode (3xTF32) and is
//    checked normwise against an fp64 host computation at the north_star's
//    1e-5 (bf16 layers: 2e-2);
//  * Tensor elements live on the device: the tests read them with at() /
//    to_host() and build them with Tensor::from_host.
// Build: make cpptest (build/dropin_test); run from tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "rtpb/rtp.hpp"

using namespace rtpb;

// ---- a doctest-shaped harness ----
namespace {
int g_checks = 0, g_failures = 0;
std::vector<std::pair<const char*, void (*)()>>& registry() {
  static std::vector<std::pair<const char*, void (*)()>> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
}  // namespace
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                   \
  static void CAT(tc_, __LINE__)();                        \
  static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(c)                                                               \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(c)) {                                                                \
      ++g_failures;                                                            \
      std::fprintf(stderr, "  %s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                                               \
  do {                                                                                         \
    ++g_checks;                                                                                \
    bool thrown_ = false;                                                                      \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const T&) {                                                                       \
      thrown_ = true;                                                                          \
    } catch (const std::exception& e_) {                                                       \
      std::fprintf(stderr, "  %s:%d: wrong exception: %s\n", __FILE__, __LINE__, e_.what());  \
    }                                                                                          \
    if (!thrown_) {                                                                            \
      ++g_failures;                                                                            \
      std::fprintf(stderr, "  %s:%d: CHECK_THROWS_AS(%s, %s) failed\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                                          \
  } while (0)

namespace {

// ---- host fp64 helpers (the SerialLinear oracle, serial.cpp:59-77) ----
using HostM = std::vector<double>;

HostM matmul(const HostM& a, const HostM& b, size_t m, size_t k, size_t n) {
  HostM c(m * n, 0.0);
  for (size_t i = 0; i < m; ++i)
    for (size_t t = 0; t < k; ++t)
      for (size_t j = 0; j < n; ++j) c[i * n + j] += a[i * k + t] * b[t * n + j];
  return c;
}

HostM transpose(const HostM& a, size_t m, size_t n) {
  HostM t(m * n);
  for (size_t i = 0; i < m; ++i)
    for (size_t j = 0; j < n; ++j) t[j * m + i] = a[i * n + j];
  return t;
}

struct Serial {
  HostM y, dx, gw, gb;
};

Serial serial_linear(const HostM& w, const HostM& b, const HostM& x, const HostM& dy, size_t rows, size_t in,
                     size_t out) {
  Serial s;
  s.y = matmul(x, w, rows, in, out);
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < out; ++j) s.y[i * out + j] += b[j];
  if (!dy.empty()) {
    s.gw = matmul(transpose(x, rows, in), dy, in, rows, out);
    s.gb.assign(out, 0.0);
    for (size_t i = 0; i < rows; ++i)
      for (size_t j = 0; j < out; ++j) s.gb[j] += dy[i * out + j];
    s.dx = matmul(dy, transpose(w, in, out), rows, out, in);
  }
  return s;
}

double nerr(const std::vector<double>& got, const std::vector<double>& ref) {
  double num = 0, den = 1e-300;
  for (size_t i = 0; i < ref.size(); ++i) {
    num = std::max(num, std::fabs(got[i] - ref[i]));
    den = std::max(den, std::fabs(ref[i]));
  }
  return got.size() == ref.size() ? num / den : 1e300;
}

HostM rows_of(const HostM& a, size_t r0, size_t r1, size_t cols) {
  return HostM(a.begin() + r0 * cols, a.begin() + r1 * cols);
}

std::vector<Tensor> shard_batch(const HostM& x, size_t rows, size_t cols, size_t n, DType dt = DType::F64) {
  std::vector<Tensor> out;
  const size_t m = rows / n;
  for (size_t r = 0; r < n; ++r) out.push_back(Tensor::from_host({m, cols}, rows_of(x, r * m, (r + 1) * m, cols), dt));
  return out;
}

HostM gather(const std::vector<Tensor>& parts) {
  HostM all;
  for (const Tensor& t : parts) {
    HostM h = t.to_host();
    all.insert(all.end(), h.begin(), h.end());
  }
  return all;
}

HostM uniform(SplitMix64& rng, size_t count, double lo, double hi) {
  HostM v(count);
  for (double& e : v) e = rng.next_uniform(lo, hi);
  return v;
}

bool bitwise_equal(const HostM& a, const HostM& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// layer shard r of (w, b): [W[:, r*per:(r+1)*per] row-major | b[r*per:...]]
HostM shard_of(const HostM& w, const HostM& b, size_t in, size_t out, size_t n, size_t r) {
  const size_t per = out / n;
  HostM s;
  for (size_t i = 0; i < in; ++i)
    for (size_t c = 0; c < per; ++c) s.push_back(w[i * out + r * per + c]);
  for (size_t c = 0; c < per; ++c) s.push_back(b[r * per + c]);
  return s;
}

}  // namespace

// ================================================================ layers_test.cpp
TEST_CASE("rtp linear with one worker reproduces the serial layer") {  // layers_test.cpp:27-40
  SplitMix64 rng(1);
  const size_t in = 16, out = 32, rows = 8;
  Tensor w = Tensor::uniform({in, out}, rng, -0.1, 0.1);
  Tensor b = Tensor::uniform({out}, rng, -0.1, 0.1);
  Tensor x = Tensor::uniform({rows, in}, rng, -1, 1);
  Serial s = serial_linear(w.to_host(), b.to_host(), x.to_host(), {}, rows, in, out);

  WorkerGroup g(1, TransportKind::Lockstep);
  RtpLinear layer(g, "lin", w, b, 1);
  CHECK(layer.dtype() == DType::F32);  // an fp64 weight selects the fp32 (3xTF32) mode
  auto y = layer.forward(std::vector<Tensor>{x}, Mode::Eval);
  CHECK(y.size() == 1);
  CHECK(y[0].rows() == rows && y[0].cols() == out);
  CHECK(nerr(y[0].to_host(), s.y) < 1e-5);
}

TEST_CASE("rtp linear forward equals the serial oracle on the gathered batch") {  // :43-58
  SplitMix64 rng(2);
  const size_t in = 16, out = 32, n = 2, rows = 16;
  Tensor w = Tensor::uniform({in, out}, rng, -0.1, 0.1);
  Tensor b = Tensor::uniform({out}, rng, -0.1, 0.1);
  HostM x = uniform(rng, rows * in, -1, 1);
  Serial s = serial_linear(w.to_host(), b.to_host(), x, {}, rows, in, out);

  WorkerGroup g(n, TransportKind::Lockstep);
  RtpLinear layer(g, "lin", w, b, n);
  auto y = layer.forward(shard_batch(x, rows, in, n), Mode::Eval);
  CHECK(nerr(gather(y), s.y) < 1e-5);
  // Eval re-homes every slot (layers_common.cpp:179-181)
  CHECK(layer.all_home());
}

TEST_CASE("per-step column blocks match the independently computed products") {  // :60-84
  SplitMix64 rng(3);
  const size_t in = 16, out = 48, n = 2, rows = 16;
  HostM w = uniform(rng, in * out, -0.1, 0.1), b = uniform(rng, out, -0.1, 0.1), x = uniform(rng, rows * in, -1, 1);
  WorkerGroup g(n, TransportKind::Lockstep);
  RtpLinear layer(g, "lin", Tensor::from_host({in, out}, w), Tensor::from_host({out}, b), n);
  auto y = layer.forward(shard_batch(x, rows, in, n), Mode::Eval);
  const size_t per = out / n, m = rows / n;
  for (size_t r = 0; r < n; ++r) {
    HostM yr = y[r].to_host();
    for (size_t j = 0; j < n; ++j) {
      HostM blk, ref;
      for (size_t i = 0; i < m; ++i)
        for (size_t c = 0; c < per; ++c) {
          double acc = b[j * per + c];
          for (size_t t = 0; t < in; ++t) acc += x[(r * m + i) * in + t] * w[t * out + j * per + c];
          ref.push_back(acc);
          blk.push_back(yr[i * out + j * per + c]);
        }
      CHECK(nerr(blk, ref) < 1e-5);
    }
  }
}

TEST_CASE("rtp linear backward matches serial gradients and re-homes its shards") {  // :86-113
  SplitMix64 rng(4);
  const size_t in = 16, out = 64, rows = 32;
  HostM w = uniform(rng, in * out, -0.1, 0.1), b = uniform(rng, out, -0.1, 0.1);
  HostM x = uniform(rng, rows * in, -1, 1), dy = uniform(rng, rows * out, -1, 1);
  Serial s = serial_linear(w, b, x, dy, rows, in, out);
  for (size_t n : {2u, 4u}) {
    WorkerGroup g(n, TransportKind::Lockstep);
    RtpLinear layer(g, "lin", Tensor::from_host({in, out}, w), Tensor::from_host({out}, b), n);
    layer.zero_grads();
    auto y = layer.forward(shard_batch(x, rows, in, n), Mode::Train);
    CHECK(!layer.all_home());  // Train forward ends displaced: rank r holds shard r+1
    auto dx = layer.backward(shard_batch(dy, rows, out, n));
    CHECK(nerr(gather(dx), s.dx) < 1e-5);
    for (size_t r = 0; r < n; ++r) {
      CHECK(layer.slots()[r].logical_id == r);
      CHECK(nerr(layer.slots()[r].grad_acc.to_host(), shard_of(s.gw, s.gb, in, out, n, r)) < 1e-5);
    }
    CHECK(layer.layout().n_shards == n);
    CHECK(layer.layout().ranges.size() == n);
    CHECK(layer.layout().ranges[n - 1].end == out);
    CHECK(layer.layout().ranges[1].extent() == out / n);
    (void)y;
  }
}

TEST_CASE("backward without forward raises a state error") {  // :115-123
  SplitMix64 rng(5);
  Tensor w = Tensor::uniform({16, 32}, rng, -0.1, 0.1);
  Tensor b = Tensor::uniform({32}, rng, -0.1, 0.1);
  WorkerGroup g(2, TransportKind::Lockstep);
  RtpLinear layer(g, "lin", w, b, 2);
  Tensor dy({8, 32});
  CHECK_THROWS_AS(layer.backward(std::vector<Tensor>{dy, dy}), StateError);
}

TEST_CASE("layout_linear rejects a shard count that does not divide the output") {  // partition.cpp:58-69
  CHECK_THROWS_AS(layout_linear(16, 30, 4), ConfigError);
  WorkerGroup g(4, TransportKind::Lockstep);
  SplitMix64 rng(6);
  Tensor w = Tensor::uniform({16, 30}, rng, -0.1, 0.1), b = Tensor::uniform({30}, rng, -0.1, 0.1);
  CHECK_THROWS_AS(RtpLinear(g, "bad", w, b, 4), ConfigError);
  Tensor b_bad = Tensor::uniform({31}, rng, -0.1, 0.1);
  CHECK_THROWS_AS(RtpLinear(g, "bad", w, b_bad, 4), DimensionError);
}

TEST_CASE("out-of-place rotation produces bitwise the in-place results") {  // :343-365
  // The reference runs a model; here the same property on RtpLinear and the
  // MLP block, fp32 mode (bf16 out-of-place pairs dX steps unless
  // RTPB_DX_PAIR=0, which is checked below).
  SplitMix64 rng(7);
  const size_t in = 32, f = 64, rows = 32;
  HostM w1 = uniform(rng, in * f, -0.1, 0.1), b1 = uniform(rng, f, -0.1, 0.1);
  HostM w2 = uniform(rng, f * in, -0.1, 0.1), b2 = uniform(rng, in, -0.1, 0.1);
  HostM x = uniform(rng, rows * in, -1, 1), dy = uniform(rng, rows * in, -1, 1);
  for (DType dt : {DType::F32, DType::BF16}) {
    if (dt == DType::BF16) setenv("RTPB_DX_PAIR", "0", 1);
    auto run = [&](RotationMode mode) {
      WorkerGroup g(2, TransportKind::Lockstep);
      RtpMlp mlp(g, "mlp", in, f, dt, w1.data(), b1.data(), w2.data(), b2.data());
      mlp.set_rotation_mode(mode);
      mlp.begin_step();
      mlp.zero_grads();
      auto y = mlp.forward(shard_batch(x, rows, in, 2), Mode::Train);
      auto dx = mlp.backward(shard_batch(dy, rows, in, 2));
      return std::tuple{gather(y), gather(dx), mlp.ffn1().slots()[0].grad_acc.to_host(),
                        mlp.ffn2().slots()[1].grad_acc.to_host()};
    };
    auto [y_in, dx_in, g1_in, g2_in] = run(RotationMode::InPlace);
    auto [y_of, dx_of, g1_of, g2_of] = run(RotationMode::OutOfPlace);
    CHECK(bitwise_equal(y_in, y_of));
    CHECK(bitwise_equal(dx_in, dx_of));
    CHECK(bitwise_equal(g1_in, g1_of));
    CHECK(bitwise_equal(g2_in, g2_of));
    unsetenv("RTPB_DX_PAIR");
  }
}

TEST_CASE("lockstep and concurrent transports produce bitwise identical results") {  // :367-385
  SplitMix64 rng(11);
  const size_t in = 32, out = 64, rows = 32, n = 4;
  HostM w = uniform(rng, in * out, -0.1, 0.1), b = uniform(rng, out, -0.1, 0.1);
  HostM x = uniform(rng, rows * in, -1, 1), dy = uniform(rng, rows * out, -1, 1);
  auto run = [&](TransportKind kind) {
    WorkerGroup g(n, kind);
    RtpLinear layer(g, "lin", Tensor::from_host({in, out}, w, DType::BF16), Tensor::from_host({out}, b, DType::BF16),
                    n);
    layer.set_rotation_mode(RotationMode::OutOfPlace);
    layer.allocate_comm_spares();
    auto y = layer.forward(shard_batch(x, rows, in, n, DType::BF16), Mode::Train);
    auto dx = layer.backward(shard_batch(dy, rows, out, n, DType::BF16));
    std::vector<HostM> grads;
    for (size_t r = 0; r < n; ++r) grads.push_back(layer.slots()[r].grad_acc.to_host());
    return std::tuple{gather(y), gather(dx), grads};
  };
  auto [ya, dxa, ga] = run(TransportKind::Lockstep);
  auto [yb, dxb, gb] = run(TransportKind::Concurrent);
  CHECK(bitwise_equal(ya, yb));
  CHECK(bitwise_equal(dxa, dxb));
  for (size_t r = 0; r < n; ++r) CHECK(bitwise_equal(ga[r], gb[r]));
}

TEST_CASE("corrupting a rotation message trips the replay assertion") {  // :387-401
  SplitMix64 rng(13);
  Tensor w = Tensor::uniform({16, 32}, rng, -0.1, 0.1), b = Tensor::uniform({32}, rng, -0.1, 0.1);
  WorkerGroup g(2, TransportKind::Lockstep);
  RtpLinear layer(g, "lin", w, b, 2);
  HostM x = uniform(rng, 16 * 16, -1, 1), dy = uniform(rng, 16 * 32, -1, 1);
  layer.forward(shard_batch(x, 16, 16, 2), Mode::Train);
  g.corrupt_next_exchange(0, WorkerGroup::Corrupt::ShardId);
  CHECK_THROWS_AS(layer.backward(shard_batch(dy, 16, 32, 2)), ProtocolError);
}

// ================================================================ ring_test.cpp
namespace {
// Slots whose payload value identifies the logical shard (ring_test.cpp:16-28).
std::vector<ShardSlot> make_slots(size_t n, size_t len = 2) {
  std::vector<ShardSlot> slots(n);
  for (size_t r = 0; r < n; ++r) {
    HostM w(len), gr(len, double(r));
    for (size_t i = 0; i < len; ++i) w[i] = double(r * 100 + i);
    slots[r].weight = Tensor::from_host({len}, w);
    slots[r].grad_acc = Tensor::from_host({len}, gr);
    slots[r].logical_id = r;
  }
  return slots;
}

size_t payload_id(const ShardSlot& s) { return size_t(s.weight.at(0)) / 100; }

double group_checksum(const std::vector<ShardSlot>& slots) {
  double sum = 0;
  for (const auto& s : slots) {
    HostM w = s.weight.to_host();
    for (size_t i = 0; i < w.size(); ++i) sum += w[i] * double(i + 1);
  }
  return sum;
}
}  // namespace

TEST_CASE("clockwise rotation across 4 workers") {  // ring_test.cpp:39-48
  WorkerGroup g(4, TransportKind::Lockstep);
  auto slots = make_slots(4);
  g.rotate_clockwise(slots);
  g.synchronize();
  for (size_t r = 0; r < 4; ++r) {
    CHECK(payload_id(slots[r]) == (r + 3) % 4);
    CHECK(slots[r].logical_id == (r + 3) % 4);
    CHECK(slots[r].rotation_offset == 1);
  }
}

TEST_CASE("single worker rotation is a no-op") {  // :50-57
  WorkerGroup g(1, TransportKind::Lockstep);
  auto slots = make_slots(1);
  g.rotate_clockwise(slots);
  g.rotate_counterclockwise(slots);
  CHECK(payload_id(slots[0]) == 0);
  CHECK(g.traffic().empty());
}

TEST_CASE("n-1 clockwise rotations leave each worker holding its successor's shard") {  // :59-64
  WorkerGroup g(4, TransportKind::Lockstep);
  auto slots = make_slots(4);
  for (int s = 0; s < 3; ++s) g.rotate_clockwise(slots);
  for (size_t r = 0; r < 4; ++r) CHECK(slots[r].logical_id == (r + 1) % 4);
}

TEST_CASE("clockwise then counter-clockwise is the identity placement") {  // :66-77
  WorkerGroup g(4, TransportKind::Lockstep);
  auto slots = make_slots(4);
  g.rotate_clockwise(slots, PayloadKind::WeightAndGrad);
  g.rotate_counterclockwise(slots, PayloadKind::WeightAndGrad);
  g.synchronize();
  for (size_t r = 0; r < 4; ++r) {
    CHECK(slots[r].logical_id == r);
    CHECK(payload_id(slots[r]) == r);
    CHECK(slots[r].grad_acc.at(0) == double(r));
    CHECK(slots[r].rotation_offset == 0);
  }
}

TEST_CASE("with two workers both directions coincide with a swap") {  // :79-88
  WorkerGroup g(2, TransportKind::Lockstep);
  auto slots = make_slots(2);
  g.rotate_clockwise(slots);
  g.synchronize();
  CHECK(payload_id(slots[0]) == 1);
  CHECK(payload_id(slots[1]) == 0);
  g.rotate_counterclockwise(slots, PayloadKind::Weight);
  g.synchronize();
  CHECK(payload_id(slots[0]) == 0);
  CHECK(payload_id(slots[1]) == 1);
}

TEST_CASE("backward rotation carries weight and gradient together") {  // :90-98
  WorkerGroup g(3, TransportKind::Lockstep);
  auto slots = make_slots(3);
  g.rotate_counterclockwise(slots);  // default WeightAndGrad
  g.synchronize();
  for (size_t r = 0; r < 3; ++r) {
    CHECK(slots[r].logical_id == (r + 1) % 3);
    CHECK(slots[r].grad_acc.at(0) == double((r + 1) % 3));
  }
}

TEST_CASE("position, permutation and volume laws under random sequences") {  // :100-132
  SplitMix64 rng(77);
  for (size_t n : {1u, 2u, 3u, 4u, 8u}) {
    WorkerGroup g(n, TransportKind::Lockstep);
    const size_t len = 6;
    auto slots = make_slots(n, len);
    const double checksum = group_checksum(slots);
    long net = 0;
    size_t steps = 0;
    for (int iter = 0; iter < 200; ++iter) {
      if (rng.next_index(2) == 0) {
        g.rotate_clockwise(slots, PayloadKind::WeightAndGrad);
        ++net;
      } else {
        g.rotate_counterclockwise(slots, PayloadKind::WeightAndGrad);
        --net;
      }
      ++steps;
      if (iter % 37 == 0) {
        for (size_t r = 0; r < n; ++r) {
          const size_t expected = (r + n - (net % long(n) + n) % n) % n;
          CHECK(slots[r].logical_id == expected);
          if (n > 1) CHECK(slots[r].rotation_offset == net);
        }
        CHECK(group_checksum(slots) == checksum);  // contents permuted, never mutated
      }
    }
    size_t elems = 0;
    for (const auto& rec : g.traffic()) elems += rec.weight_elems_per_worker;
    CHECK(elems == (n == 1 ? 0 : steps * len));
  }
}

TEST_CASE("a full pass moves the same volume as a ring allgather") {  // :134-168
  const size_t n = 4, shard_len = 8;
  WorkerGroup g(n, TransportKind::Lockstep);
  auto slots = make_slots(n, shard_len);
  for (size_t s = 0; s + 1 < n; ++s) g.rotate_clockwise(slots, PayloadKind::Weight, "pass");
  size_t rotation_elems = 0;
  for (const auto& rec : g.traffic())
    if (rec.label == "pass") rotation_elems += rec.weight_elems_per_worker;
  CHECK(rotation_elems == (n - 1) * shard_len);

  std::vector<Tensor> shards;
  for (size_t r = 0; r < n; ++r) {
    Tensor t({shard_len});
    t.fill(double(r));
    shards.push_back(std::move(t));
  }
  g.clear_traffic();
  auto gathered = g.ring_allgather(shards, "ag");
  size_t ag_elems = 0;
  for (const auto& rec : g.traffic()) ag_elems += rec.weight_elems_per_worker;
  CHECK(ag_elems == (n - 1) * shard_len);
  CHECK(ag_elems == rotation_elems);
  for (size_t r = 0; r < n; ++r) {
    CHECK(gathered[r].numel() == n * shard_len);
    HostM h = gathered[r].to_host();
    for (size_t j = 0; j < n; ++j)
      for (size_t i = 0; i < shard_len; ++i) CHECK(h[j * shard_len + i] == double(j));
  }
  WorkerGroup g1(1, TransportKind::Lockstep);
  auto one = g1.ring_allgather(std::vector<Tensor>{shards[0]});
  CHECK(one[0].numel() == shard_len);
}

TEST_CASE("out-of-place rotation matches in-place placement and uses the spare") {  // :170-200
  const size_t n = 4, len = 4;
  WorkerGroup a(n, TransportKind::Lockstep), b(n, TransportKind::Lockstep);
  auto in_place = make_slots(n, len);
  auto out_place = make_slots(n, len);

  MemoryLedger ledgers[4];
  std::vector<MemoryLedger*> lp{&ledgers[0], &ledgers[1], &ledgers[2], &ledgers[3]};
  b.bind_ledgers(lp);

  std::vector<Tensor> spares(n);
  b.each([&](size_t r) {
    CategoryScope comm(MemCategory::CommBuffer);
    spares[r] = Tensor({len});
  });
  for (size_t r = 0; r < n; ++r) CHECK(ledgers[r].current(MemCategory::CommBuffer) == len * sizeof(double));

  a.rotate_clockwise(in_place);
  b.rotate_outofplace(out_place, spares, Direction::Clockwise);
  a.synchronize();
  b.synchronize();
  for (size_t r = 0; r < n; ++r) {
    CHECK(out_place[r].logical_id == in_place[r].logical_id);
    CHECK(bitwise_equal(out_place[r].weight.to_host(), in_place[r].weight.to_host()));
  }
  Tensor wrong({len + 1});
  std::vector<Tensor> bad(n, wrong);
  CHECK_THROWS_AS(b.rotate_outofplace(out_place, bad, Direction::Clockwise), DimensionError);
}

TEST_CASE("bound ledgers see the layers' device bytes") {  // analysis.cpp:286-318 binding
  SplitMix64 rng(21);
  const size_t in = 16, out = 64, n = 2;
  MemoryLedger ledgers[2];
  WorkerGroup g(n, TransportKind::Lockstep);
  g.bind_ledgers({&ledgers[0], &ledgers[1]});
  RtpLinear layer(g, "lin", Tensor::uniform({in, out}, rng, -0.1, 0.1, DType::BF16),
                  Tensor::uniform({out}, rng, -0.1, 0.1, DType::BF16), n);
  const size_t L = in * (out / n) + out / n;
  for (size_t r = 0; r < n; ++r) {
    CHECK(ledgers[r].current(MemCategory::Param) == L * 2);  // W/N, bf16
    CHECK(ledgers[r].current(MemCategory::Grad) == L * 4);   // G/N, fp32
  }
  layer.set_rotation_mode(RotationMode::OutOfPlace);
  layer.allocate_comm_spares();
  for (size_t r = 0; r < n; ++r) CHECK(ledgers[r].current(MemCategory::CommBuffer) == L * 2);
  layer.release_comm_spares();
  for (size_t r = 0; r < n; ++r) CHECK(ledgers[r].current(MemCategory::CommBuffer) == 0);
}

int main() {
  int failed_cases = 0;
  for (auto& [name, fn] : registry()) {
    const int before = g_failures;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_failures;
      std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
    }
    const bool ok = g_failures == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", name);
  }
  std::printf("%zu test cases, %d checks, %d failures\n", registry().size(), g_checks, g_failures);
  return g_failures ? 1 : 0;
}
