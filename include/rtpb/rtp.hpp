// rtpb/rtp.hpp — C++ host API of the B200-native RTP hot path.
//
// Mirrors the reference's layer API (proj/include/rtp/{errors,ledger,ring,
// layers}.hpp) with device-resident shards: same class names, argument
// meaning and exception types, so callers written against rtp::RtpLinear /
// rtp::WorkerGroup switch by changing the namespace and passing device
// activations. Compute goes through the step kernels of include/rtpb.h;
// rotation through the group's Transport (device copies in-process, or
// ncclSend/ncclRecv with one process per GPU).
#pragma once
#include <array>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../rtpb.h"

namespace rtpb {

// ---- errors (errors.hpp:8-33) ----
struct DimensionError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IndexError : std::out_of_range {
  using std::out_of_range::out_of_range;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Throws the exception class matching an rtpb.h status code.
void throw_status(int code, const std::string& msg);
void check_status(int code);

enum class Mode { Train, Eval };
enum class RotationMode { InPlace, OutOfPlace };
enum class Direction { Clockwise, CounterClockwise };
// Solo: one rank of an n-rank ring with no peers (shifts skipped; measurement only).
enum class TransportKind { Lockstep, Concurrent, Nccl, Ipc, Solo };
enum class PayloadKind { Weight, WeightAndGrad };
// Layers compute in BF16 or F32 (3xTF32); F64 is the reference's Tensor
// element type (tensor.hpp), accepted at the Tensor API boundary.
enum class DType { BF16 = RTPB_BF16, F32 = RTPB_F32, F64 = RTPB_F64 };
inline size_t dtype_size(DType d) { return d == DType::F64 ? 8 : d == DType::F32 ? 4 : 2; }

// ---- rng (rng.hpp:10-32): the fixtures' generator, host side ----
class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t seed) : state_(seed) {}
  uint64_t next_u64() {
    state_ += 0x9E3779B97F4A7C15ULL;
    uint64_t z = state_;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_uniform(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
  uint64_t next_index(uint64_t n) { return next_u64() % n; }

 private:
  uint64_t state_;
};

// ---- ledger (ledger.hpp:10-41), per worker, device bytes ----
enum class MemCategory : uint8_t { Param, Grad, Activation, CommBuffer, Other };
inline constexpr size_t kNumMemCategories = 5;

const char* mem_category_name(MemCategory c);

class MemoryLedger {
 public:
  void on_alloc(MemCategory c, size_t bytes);
  void on_release(MemCategory c, size_t bytes);
  size_t current(MemCategory c) const { return current_[size_t(c)]; }
  size_t peak(MemCategory c) const { return peak_[size_t(c)]; }
  size_t current_total() const { return current_total_; }
  size_t peak_total() const { return peak_total_; }
  void reset();        // all counters to zero (ledger.cpp)
  void reset_peaks();  // peaks down to the current bytes
  // Every charge / release is also applied to `m` (WorkerGroup::bind_ledgers);
  // the bytes already held are charged to it at binding. nullptr unbinds.
  void mirror_to(MemoryLedger* m);

 private:
  std::array<size_t, kNumMemCategories> current_{};
  std::array<size_t, kNumMemCategories> peak_{};
  size_t current_total_ = 0;
  size_t peak_total_ = 0;
  MemoryLedger* mirror_ = nullptr;
};

// RAII binding of the calling thread's Tensor allocations to a ledger +
// category (ledger.hpp LedgerScope / CategoryScope); scopes nest.
class LedgerScope {
 public:
  LedgerScope(MemoryLedger* ledger, MemCategory category);
  ~LedgerScope();
  LedgerScope(const LedgerScope&) = delete;
  LedgerScope& operator=(const LedgerScope&) = delete;
  static MemoryLedger* current_ledger();
  static MemCategory current_category();

 private:
  MemoryLedger* prev_ledger_;
  MemCategory prev_category_;
};

class CategoryScope {
 public:
  explicit CategoryScope(MemCategory category) : inner_(LedgerScope::current_ledger(), category) {}

 private:
  LedgerScope inner_;
};

// Owning device allocation charged to a worker ledger under one category
// (the device analogue of Tensor::register_bytes, tensor.cpp:86-97).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(int device, size_t bytes, MemoryLedger* ledger, MemCategory cat, bool zero = true);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept;
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;

  void* data() const { return ptr_; }
  size_t bytes() const { return bytes_; }
  int device() const { return device_; }
  bool empty() const { return ptr_ == nullptr; }
  void reset();
  // Exchange storage between equal-sized buffers without touching either
  // charge (swap_data, tensor.hpp:65-72): rotation moves contents, not residency.
  friend void swap_data(DeviceBuffer& a, DeviceBuffer& b);

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
  int device_ = 0;
  MemoryLedger* ledger_ = nullptr;
  MemCategory cat_ = MemCategory::Other;
};

// ---- tensor (tensor.hpp): dense row-major DEVICE tensor ----
// Owns one device allocation, charged to a ledger under one category: the
// calling thread's LedgerScope at construction (as Tensor::register_bytes,
// tensor.cpp:86-97), or an explicit ledger. Copies are deep (device-to-
// device) and charge the copying thread's scope; moves keep the charge;
// swap_data exchanges storage between equal-sized tensors without touching
// either charge — how rotation moves shard contents (tensor.hpp:65-72).
// Host access (at, to_host, from_host) synchronises and is for setup and tests.
class Tensor {
 public:
  Tensor() = default;
  // Zero-filled, on the current device.
  explicit Tensor(std::vector<size_t> shape, DType dtype = DType::F64);
  // On `device`, charged to `ledger` (may be null) under `cat`.
  Tensor(std::vector<size_t> shape, DType dtype, int device, MemoryLedger* ledger, MemCategory cat,
         bool zero = true);
  Tensor(const Tensor& other);
  Tensor& operator=(const Tensor& other);
  Tensor(Tensor&&) noexcept = default;
  Tensor& operator=(Tensor&&) noexcept = default;

  static Tensor zeros(std::vector<size_t> shape, DType dtype = DType::F64) { return Tensor(std::move(shape), dtype); }
  // Host values (fp64, row-major) rounded once to dtype, uploaded to `device` (-1: current).
  static Tensor from_host(std::vector<size_t> shape, std::span<const double> values, DType dtype = DType::F64,
                          int device = -1);
  // Tensor::uniform (tensor.cpp:99-103): draws on the host, then uploads.
  static Tensor uniform(std::vector<size_t> shape, SplitMix64& rng, double lo, double hi,
                        DType dtype = DType::F64, int device = -1);

  const std::vector<size_t>& shape() const { return shape_; }
  size_t rank() const { return shape_.size(); }
  size_t dim(size_t i) const { return shape_[i]; }
  size_t numel() const;
  size_t rows() const;  // rank-2 only
  size_t cols() const;
  DType dtype() const { return dtype_; }
  size_t bytes() const { return buf_.bytes(); }
  int device() const { return buf_.device(); }
  bool empty() const { return buf_.empty(); }
  void* data() const { return buf_.data(); }
  std::string shape_str() const;

  // Element i widened to fp64 (synchronous device read).
  double at(size_t i) const;
  double at(size_t i, size_t j) const { return at(i * shape_[1] + j); }
  std::vector<double> to_host() const;
  void fill(double v);                // device fill (synchronous)
  Tensor to(DType dtype) const;       // converted copy (one RN rounding per element)
  Tensor reshaped(std::vector<size_t> shape) const&;
  Tensor reshaped(std::vector<size_t> shape) &&;
  void reset() { buf_.reset(); shape_.clear(); }

  friend void swap_data(Tensor& a, Tensor& b);

 private:
  std::vector<size_t> shape_;
  DType dtype_ = DType::F64;
  DeviceBuffer buf_;
};

// ---- partition (partition.hpp:44-60) ----
enum class PartitionStrategy { OutputPartition, HeadPartition, ExpertPartition };
struct ShardRange {
  size_t begin = 0;
  size_t end = 0;
  size_t extent() const { return end - begin; }
};
struct ShardLayout {
  PartitionStrategy strategy = PartitionStrategy::OutputPartition;
  size_t n_shards = 1;
  std::vector<ShardRange> ranges;
};
// Columns of the weight (output features) plus the matching bias slice;
// ConfigError unless out_dim % n == 0 (partition.cpp:58-69).
ShardLayout layout_linear(size_t in_dim, size_t out_dim, size_t n);

// ---- ring (ring.hpp:23-46) ----
struct ShardSlot {
  Tensor weight;    // [W_j : I x per | b_j : per] in the layer dtype
  Tensor grad_acc;  // same element layout, fp32
  size_t logical_id = 0;
  long rotation_offset = 0;
};

struct CommRecord {
  std::string label;
  const char* kind;  // "rotation_cw" | "rotation_ccw" | "allgather"
  size_t weight_elems_per_worker;
  size_t grad_elems_per_worker;
};

struct Worker;
class Transport;

class WorkerGroup {
 public:
  // All n workers in this process; devices[r] hosts worker r (empty: all on
  // the current device). kind: Lockstep (one host thread) or Concurrent
  // (a host thread per worker).
  WorkerGroup(size_t n, TransportKind kind, std::vector<int> devices = {});
  // One process per GPU: this process is worker `rank` of `n`. kind Nccl:
  // ncclSend/ncclRecv (unique id from ncclGetUniqueId); kind Ipc: copy-engine
  // pushes through CUDA IPC mappings (unique id from rtpb_ipc_unique_id).
  WorkerGroup(size_t n, size_t rank, int device, const void* unique_id, TransportKind kind = TransportKind::Nccl);
  ~WorkerGroup();
  WorkerGroup(const WorkerGroup&) = delete;
  WorkerGroup& operator=(const WorkerGroup&) = delete;

  size_t size() const { return n_; }
  TransportKind kind() const { return kind_; }
  // A peer process shares a local worker's GPU (IPC transport on one device).
  bool device_shared() const;
  const std::vector<size_t>& local_ranks() const { return local_; }
  bool is_local(size_t rank) const;
  Worker& worker(size_t rank);

  // Runs fn(rank) for every LOCAL rank (all ranks in-process; the own rank
  // under NCCL), in rank order or one host thread per worker; exceptions are
  // re-thrown in rank order (ring.cpp:134-174).
  void each(const std::function<void(size_t)>& fn);

  // Ring steps on slots (ring.cpp:265-333). Device transfers are enqueued on
  // each worker's comm stream behind its compute stream and the compute
  // stream then waits for them: stream-ordered, no host sync.
  // shard_elems: elements per shard, for the traffic log (ring.hpp:41-46).
  void rotate_clockwise(std::span<ShardSlot> slots, PayloadKind kind = PayloadKind::Weight,
                        std::string_view label = {}, size_t shard_elems = 0);
  void rotate_counterclockwise(std::span<ShardSlot> slots, PayloadKind kind = PayloadKind::WeightAndGrad,
                               std::string_view label = {}, size_t shard_elems = 0);
  void rotate_outofplace(std::span<ShardSlot> slots, std::span<Tensor> spares, Direction dir,
                         PayloadKind kind = PayloadKind::Weight, std::string_view label = {},
                         size_t shard_elems = 0);
  // ring_allgather (ring.cpp:335-376): out[r] holds all n chunks in canonical order.
  void ring_allgather(std::span<void* const> in, std::span<void* const> out, size_t bytes,
                      std::string_view label = {}, size_t elem_size = 1);
  // Reference signature: every local worker ends with the n shards
  // concatenated in canonical order.
  std::vector<Tensor> ring_allgather(std::span<const Tensor> shards, std::string_view label = {});

  // Lower-level pieces used by the layers' overlap scheduler.
  // Raw ring shift of per-local-rank buffers: recv[dest(r)] <- send[r];
  // send == recv means in place (chunked through a staging buffer).
  // channel: 0 weights (and per-step gradients), 1 a backward pass launch's travelling gradient
  void exchange(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
                int channel = 0);
  // Advances slot bookkeeping for one hop (ids, offsets, tag, fault hook,
  // traffic record) exactly as the reference's install_payload does.
  void advance_slots(std::span<ShardSlot> slots, Direction dir, PayloadKind kind, std::string_view label,
                     size_t shard_elems);

  // compute stream <-> comm stream fencing per local worker.
  void comm_after_compute();
  // While set, comm_after_compute() is a no-op: a pass launch that already
  // fenced its comm streams (before its grids) runs the next layer's
  // prefetch hook after queueing those grids, whose first shift must not
  // wait for them.
  void set_comm_fenced(bool on) { comm_fenced_ = on; }
  void compute_after_comm();
  void synchronize();
  // Orders each local worker's compute stream after its aux stream.
  void join_aux();

  const std::vector<CommRecord>& traffic() const { return traffic_; }
  void clear_traffic() { traffic_.clear(); }
  uint64_t next_tag() const { return tag_; }
  enum class Corrupt { None, Tag, ShardId };
  void corrupt_next_exchange(size_t rank, Corrupt what);

  // Per-worker device ledger (every allocation the library makes for the
  // worker is charged to it).
  MemoryLedger& ledger_of(size_t rank);
  // ring.hpp:69-71: caller-owned per-rank ledgers. Each local worker's ledger
  // is mirrored into ledgers[rank] (bytes already held are charged at
  // binding), and each() runs its thunks under LedgerScope(ledgers[rank],
  // Activation), so Tensors the thunks create are charged there too.
  void bind_ledgers(std::vector<MemoryLedger*> ledgers);
  MemoryLedger* bound_ledger(size_t rank) const;

 private:
  std::vector<MemoryLedger*> bound_;
  friend class Transport;
  size_t n_;
  TransportKind kind_;
  std::vector<size_t> local_;
  std::vector<std::unique_ptr<Worker>> workers_;  // indexed by rank; null when remote
  std::unique_ptr<Transport> transport_;
  bool comm_fenced_ = false;
  std::vector<CommRecord> traffic_;
  uint64_t tag_ = 0;
  size_t corrupt_rank_ = 0;
  Corrupt corrupt_ = Corrupt::None;
};

// ---- layers (layers.hpp:22-147) ----
template <typename Saved>
class ReplayTape {
 public:
  void record(size_t logical_id, Saved saved) { entries_.push_back(Entry{logical_id, std::move(saved)}); }
  Saved replay(size_t resident_id) {
    if (entries_.empty()) throw StateError("backward invoked without a matching forward");
    Entry& e = entries_.back();
    if (e.logical_id != resident_id)
      throw ProtocolError("shard identity mismatch on replay: resident shard " + std::to_string(resident_id) +
                          ", tape recorded " + std::to_string(e.logical_id));
    Saved s = std::move(e.saved);
    entries_.pop_back();
    return s;
  }
  size_t size() const { return entries_.size(); }
  bool empty() const { return entries_.empty(); }
  void clear() { entries_.clear(); }

 private:
  struct Entry {
    size_t logical_id;
    Saved saved;
  };
  std::vector<Entry> entries_;
};

struct Empty {};

// Device activation view for one local rank: rows x cols, row stride ld.
struct DView {
  void* data = nullptr;
  size_t ld = 0;
};

class RtpLayerBase {
 public:
  RtpLayerBase(WorkerGroup& group, std::string label, DType dtype);
  virtual ~RtpLayerBase() = default;

  const std::string& label() const { return label_; }
  size_t n() const { return group_->size(); }
  std::span<ShardSlot> slots() { return slots_; }
  size_t shard_len() const { return shard_len_; }
  size_t flat_param_bytes() const { return shard_len_ * n() * dtype_size(dtype_); }
  size_t flat_grad_bytes() const { return shard_len_ * n() * sizeof(float); }
  DType dtype() const { return dtype_; }

  // zero_grads (layers_common.cpp:120-122) is lazy: the next backward's first
  // dW step overwrites the resident gradient instead of accumulating into it
  // (no memset). materialize_grads() performs the zero fill for readers that
  // look at grad_acc before that backward.
  virtual void zero_grads();
  void materialize_grads();
  bool all_home() const;
  void allocate_comm_spares();
  void release_comm_spares();
  bool has_comm_spares() const { return !spares_.empty(); }
  void set_rotation_mode(RotationMode m);
  // Numerics options (rtpb.h RTPB_OPT_*): exact-erf GELU in bf16 epilogues
  // (default: tanh.approx form); paired dX steps out of place (default on,
  // or RTPB_DX_PAIR; off restores out-of-place == in-place bitwise).
  void set_exact_gelu(bool on) { exact_gelu_ = on; }
  bool exact_gelu() const { return exact_gelu_; }
  void set_paired_dx(bool on) { paired_dx_ = on; }
  bool paired_dx() const { return paired_dx_; }
  RotationMode rotation_mode() const { return rotation_mode_; }
  // Logical id seen by (phase 0 fwd / 1 bwd, step, rank) in the last pass.
  const std::vector<int64_t>& trace() const { return trace_; }
  // The weight (grad = false) or gradient shard resident at a local rank as
  // host fp64 values in the reference's flat shard layout (synchronous).
  virtual std::vector<double> shard_host(size_t rank, bool grad);

 protected:
  void init_slots_alloc();
  void require_home(const char* op) const;
  void check_forward_position(size_t rank, size_t step) const;
  void check_backward_position(size_t rank, size_t step) const;
  void rotate_forward();
  void rotate_backward();
  void rehome_after_eval();
  // Forgets a prefetched first shift (RtpLinear); called whenever the spare
  // it landed in is replaced or the pass that would consume it fails.
  virtual void drop_prefetch() {}
  bool oop() const { return rotation_mode_ == RotationMode::OutOfPlace && !spares_.empty(); }

  WorkerGroup* group_;
  std::string label_;
  DType dtype_;
  std::vector<ShardSlot> slots_;  // indexed by rank (remote entries stay empty)
  std::vector<Tensor> spares_;
  size_t shard_len_ = 0;
  size_t flag_base_ = 0;  // this layer's block of the workers' shard-arrival flags
  RotationMode rotation_mode_ = RotationMode::InPlace;
  bool exact_gelu_ = false;
  bool paired_dx_ = true;  // initialised from RTPB_DX_PAIR
  std::vector<int64_t> trace_;
  bool grads_zero_pending_ = false;
};

// Linear layer sharded on output features (layers_linear.cpp:6-72).
class RtpLinear : public RtpLayerBase {
 public:
  // Host fp64 weight (in x out, row-major) and bias (out), as the reference.
  RtpLinear(WorkerGroup& group, std::string label, const double* weight, const double* bias, size_t in_dim,
            size_t out_dim, size_t n, DType dtype = DType::BF16);
  // Flyweight: shard r generated on worker r's device from SplitMix64(seed)
  // starting at stream index stream_base; the full weight never exists.
  RtpLinear(WorkerGroup& group, std::string label, size_t in_dim, size_t out_dim, size_t n, uint64_t seed,
            uint64_t stream_base, DType dtype = DType::BF16);
  // The reference's constructor (layers.hpp:133-134): weight (in x out) and
  // bias (out) as Tensors of any dtype; the layer computes in BF16 for a BF16
  // weight, else in F32 (3xTF32) — an F64 weight (the reference's type)
  // selects the fp32 mode, the tolerance-1e-5 path.
  RtpLinear(WorkerGroup& group, std::string label, const Tensor& weight, const Tensor& bias, size_t n);

  size_t in_dim() const { return in_; }
  size_t out_dim() const { return out_; }
  size_t per() const { return per_; }
  const ShardLayout& layout() const { return layout_; }

  // Reference signatures (layers.hpp:138-139). x: one (rows x in) Tensor per
  // local worker (all n in-process; the own rank under NCCL / IPC), on the
  // worker's device, any dtype (converted to the layer dtype). Returns
  // (rows x out) per local worker in the layer dtype, charged to the worker's
  // ledger as Activation. Train keeps a copy of X for backward (x_cache_).
  std::vector<Tensor> forward(std::span<const Tensor> x, Mode mode);
  std::vector<Tensor> backward(std::span<const Tensor> dy);

  // x[k] / y[k]: activations of local rank k (rows x in / rows x out).
  void forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode);
  void backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx);

  // Fused variants used by RtpMlp (GELU in the epilogues).
  struct FwdEpi {
    std::span<const DView> act;  // gelu(pre) outputs (nullable span)
    bool store_pre = true;
    std::function<void()> before_last_step;  // called once the layer's last shift is posted
  };
  struct BwdEpi {
    std::span<const DView> pre;  // multiply the final dX by gelu'(pre)
    std::function<void()> before_last_step;
  };
  // Cross-layer pipelining: post this layer's first weight
  // shift of the coming forward (backward = false) or backward pass now, into
  // the out-of-place spare, so it travels under the previous layer's last
  // step; the pass then skips posting it. No-op unless out of place and N > 1.
  void prefetch_first_shift(bool backward);
  void forward_ex(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode, const FwdEpi& e);
  void backward_ex(std::span<const DView> dy, size_t rows, std::span<const DView> dx, const BwdEpi& e);
  // N = 1 (no rotation): the bookkeeping of forward_ex (position law, replay
  // tape, X kept for backward, trace) without a launch; returns the resident
  // shard [W_0 | b_0] for a caller that issues the GEMM itself (RtpMlp's
  // fused forward).
  const void* begin_forward_n1(const DView& x, size_t rows, Mode mode);
  // N = 1 backward for a caller that issues the GEMMs itself (RtpMlp's fused
  // backward): replay / position checks and trace, then what the step needs.
  struct N1Bwd {
    const void* weight;  // resident shard [W | b]
    float* grad;         // resident gradient shard (fp32)
    bool grad_zero;      // zero_grads() pending: overwrite instead of accumulate
    DView x;             // X cached by forward
    void* workspace;
    size_t workspace_bytes;
  };
  N1Bwd begin_backward_n1(size_t rows);
  void end_backward_n1();

 private:
  void build(size_t in_dim, size_t out_dim, size_t n);
  void upload_shards(const double* weight, const double* bias);
  void ensure_scratch(size_t rows);
  void drop_prefetch() override;
  void forward_impl(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode, const FwdEpi& e);
  void backward_impl(std::span<const DView> dy, size_t rows, std::span<const DView> dx, const BwdEpi& e);
  void backward_pass(std::span<const DView> dy, size_t rows, std::span<const DView> dx, const BwdEpi& e);
  // Shard-arrival flags (rtp_layers.cpp): forward W, backward W, backward G
  // blocks of the layer's flag range, indexed by the step the shard is for.
  static constexpr size_t kFlagFwd = 0, kFlagBwdW = 16, kFlagBwdG = 32;
  // CTA counters of the grids that clear each block (the pass's last reader)
  static constexpr size_t kFlagCtrFwd = 48, kFlagCtrW = 49, kFlagCtrG = 50;
  // Pass launches: per-step count-in counters of the forward / dX launch
  static constexpr size_t kFlagDoneFwd = 64, kFlagDoneBwd = 80, kFlagDoneW = 96;
  bool use_flags() const;
  bool pass_launch_ok() const;
  bool serial_profile() const;  // RTPB_SERIAL_PROFILE on a Solo group
  bool backward_pass_pays(size_t rows) const;
  void flagged_exchange(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
                        size_t flag, int channel = 0);

  size_t in_ = 0, out_ = 0, per_ = 0;
  ShardLayout layout_;
  std::vector<Tensor> x_keep_;  // Tensor API: X (layer dtype) held from Train forward to backward
  std::vector<ReplayTape<Empty>> tapes_;
  std::vector<DView> x_cache_;          // per rank: caller-owned X kept for backward
  std::vector<DeviceBuffer> dx_acc_;    // per rank: fp32 cross-step dX accumulator
  std::vector<DeviceBuffer> workspace_; // per rank: step-kernel workspace
  std::vector<DeviceBuffer> pass_ws_;   // per rank, pass launches: [dY column sums (out) | colsum workspace]
  size_t pass_ws_rows_ = 0;
  size_t scratch_rows_ = 0;
  size_t cached_rows_ = 0;
  bool pre_fwd_ = false, pre_bwd_ = false;  // first shift already posted
};

// Q/K/V projections split by head group; the output projection owns the
// matching row block (partition.cpp:71-84): ConfigError unless hidden % heads
// == 0 and heads % n == 0.
ShardLayout layout_attention(size_t hidden, size_t heads, size_t n);

// Multi-head attention sharded by head group (layers.hpp:170-191,
// layers_attention.cpp:43-198): shard j holds head group j's Q/K/V column
// blocks and the matching row block of the output projection, no bias.
// Forward step s (shard j): Q,K,V = X Wq_j, X Wk_j, X Wv_j (step GEMMs), the
// attention core per (sequence, head) (kernels/attention.cu), Y += A Wo_j
// through the dX kernel's fp32 cross-step accumulator. Backward: dWo_j,
// dA, the core's backward, dWq/k/v_j (dW kernel, fused into the travelling
// gradient) and dX += dQ Wq_j^T + dK Wk_j^T + dV Wv_j^T (fp32 accumulator).
// Device shard layout: [Wq_j | Wk_j | Wv_j | Wo_j^T], each hidden x gw
// row-major (gw = heads/n * head_dim): the reference's flat shard with the
// Wo block stored transposed, so every product maps onto the three step
// kernels; shard_host() returns the reference layout.
class RtpAttention : public RtpLayerBase {
 public:
  // Host fp64 weights (hidden x hidden each, as the reference).
  RtpAttention(WorkerGroup& group, std::string label, const double* wq, const double* wk, const double* wv,
               const double* wo, size_t hidden, size_t heads, size_t seq, size_t n, DType dtype = DType::BF16);
  // The reference's constructor (layers.hpp:175-176); dtype as RtpLinear's.
  RtpAttention(WorkerGroup& group, std::string label, const Tensor& wq, const Tensor& wk, const Tensor& wv,
               const Tensor& wo, size_t heads, size_t seq, size_t n);

  size_t hidden() const { return hidden_; }
  size_t heads() const { return heads_; }
  size_t seq() const { return seq_; }
  size_t head_dim() const { return hd_; }
  size_t group_heads() const { return g_; }
  size_t group_width() const { return gw_; }
  const ShardLayout& layout() const { return layout_; }

  // x[k]: (batch * seq) x hidden per local worker; y, dx the same shape.
  void forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode);
  void backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx);
  std::vector<Tensor> forward(std::span<const Tensor> x, Mode mode);
  std::vector<Tensor> backward(std::span<const Tensor> dy);

  // The resident weight (grad = false) or gradient shard of a local rank in
  // the reference's flat layout [Wq_j | Wk_j | Wv_j | Wo_j (gw x hidden)].
  std::vector<double> shard_host(size_t rank, bool grad) override;

 private:
  void init(const double* wq, const double* wk, const double* wv, const double* wo);
  void ensure_scratch(size_t rows);
  size_t hidden_, heads_, seq_, hd_, g_, gw_;
  ShardLayout layout_;
  std::vector<ReplayTape<size_t>> tapes_;  // saved: the forward step whose buffers backward reads
  std::vector<DView> x_cache_;
  std::vector<Tensor> x_keep_;
  size_t scratch_rows_ = 0, cached_rows_ = 0;
  // per rank: per forward step s: q, k, v, o (rows x gw, dtype) and lse
  // (rows x g fp32); backward scratch dA, dq, dk, dv, delta; fp32 Y / dX
  // cross-step accumulators (rows x hidden)
  std::vector<DeviceBuffer> saved_, lse_, scratch_, acc_;
};

// Embedding sharded on the embedding dimension (layers.hpp:150-168,
// layers_linear.cpp:74-136): shard j = table[:, j*per:(j+1)*per] (vocab x
// per), the same rotation schedule as RtpLinear; forward gathers rows into
// the output's column block, backward scatter-adds dY's block into the
// travelling gradient in token order (no input gradient). Ids are host
// vectors as in the reference (IndexError outside the vocabulary).
class RtpEmbedding : public RtpLayerBase {
 public:
  RtpEmbedding(WorkerGroup& group, std::string label, const double* table, size_t vocab, size_t emb, size_t n,
               DType dtype = DType::BF16);
  RtpEmbedding(WorkerGroup& group, std::string label, const Tensor& table, size_t n);  // layers.hpp:153

  size_t vocab() const { return vocab_; }
  size_t emb_dim() const { return emb_; }
  const ShardLayout& layout() const { return layout_; }

  // ids[k]: the token ids of local rank k; y[k]: ids[k].size() x emb.
  void forward(std::span<const std::vector<int64_t>> ids, std::span<const DView> y, Mode mode);
  void backward(std::span<const DView> dy, size_t rows, const std::function<void()>& after_last_rotation = {});
  std::vector<Tensor> forward(std::span<const std::vector<int64_t>> ids, Mode mode);
  void backward(std::span<const Tensor> dy, const std::function<void()>& after_last_rotation = {});

 private:
  size_t vocab_, emb_, per_;
  ShardLayout layout_;
  std::vector<ReplayTape<Empty>> tapes_;
  // per rank: device ids (int64) and, for backward, the CSR of token
  // positions per unique id (uniq int64, offsets int32, tokens int32)
  std::vector<DeviceBuffer> ids_dev_, csr_;
  std::vector<size_t> n_ids_, n_uniq_;
};

// One expert per shard; ConfigError unless n_experts == n (partition.cpp:86-96).
ShardLayout layout_moe(size_t n_experts, size_t n);

// One two-layer GELU expert per shard (layers.hpp:113-116).
struct ExpertParams {
  Tensor w1, b1, w2, b2;
};

// Mixture of experts (layers.hpp:193-229, layers_moe.cpp:18-198): top-1
// gating with a replicated gate (hidden x n, fp64 on every worker so routing
// follows the reference's fp64 arithmetic), one expert per shard; tokens meet
// every expert as experts rotate past the sharded batch (no all-to-all).
// Shard j = [w1 (hidden x f) | b1 | w2 (f x hidden) | b2]: two linear shards
// back to back, so the expert MLP runs on the step GEMMs (GELU fused).
class RtpMoe : public RtpLayerBase {
 public:
  // gate: hidden x n fp64; experts[e]: packed [w1 | b1 | w2 | b2] fp64.
  RtpMoe(WorkerGroup& group, std::string label, const double* gate, const double* const* experts, size_t hidden,
         size_t ffn, size_t n, DType dtype = DType::BF16);
  RtpMoe(WorkerGroup& group, std::string label, const Tensor& gate, std::span<const ExpertParams> experts,
         size_t n);  // layers.hpp:197-198

  size_t hidden() const { return hidden_; }
  size_t ffn_dim() const { return ffn_; }
  size_t n_experts() const { return n(); }
  size_t gate_bytes() const { return hidden_ * n() * sizeof(double); }
  const ShardLayout& layout() const { return layout_; }

  void forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode);
  void backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx);
  std::vector<Tensor> forward(std::span<const Tensor> x, Mode mode);
  std::vector<Tensor> backward(std::span<const Tensor> dy);

  // Per-worker gate gradient over the local batch shard (data-parallel
  // semantics: the caller combines replicas), and the replicated gate (fp64).
  const Tensor& gate_grad(size_t rank) const { return gate_grads_[rank]; }
  const Tensor& gate_weight(size_t rank) const { return gates_[rank]; }
  Tensor& gate_weight_mut(size_t rank) { return gates_[rank]; }
  void zero_grads() override;

 private:
  void init(const double* gate, const double* const* experts);
  void ensure_scratch(size_t rows);
  size_t hidden_, ffn_;
  ShardLayout layout_;
  std::vector<Tensor> gates_, gate_grads_;
  std::vector<ReplayTape<Empty>> tapes_;
  std::vector<DView> x_cache_;
  std::vector<Tensor> x_keep_;
  size_t scratch_rows_ = 0, cached_rows_ = 0;
  bool gate_zero_pending_ = false;
  // per rank: routing (probs fp64 rows x n, sel / pos / rows-by-expert int32,
  // dlogits fp64), per-expert saved pre1 / h1 / eout segments, scratch
  std::vector<DeviceBuffer> route_, saved_, scratch_;
  std::vector<std::vector<size_t>> seg_off_, seg_cnt_;  // per rank: expert segment offsets / counts
};

// ffn1 (h -> f) -> gelu -> ffn2 (f -> h), composed as model.cpp:77-83,99-105.
class RtpMlp {
 public:
  RtpMlp(WorkerGroup& group, std::string label, size_t h, size_t f, DType dtype, const double* w1,
         const double* b1, const double* w2, const double* b2);
  RtpMlp(WorkerGroup& group, std::string label, size_t h, size_t f, DType dtype, uint64_t seed,
         uint64_t stream_base);

  void set_rotation_mode(RotationMode m);
  void set_exact_gelu(bool on);  // both layers and the fused N = 1 launches
  void set_paired_dx(bool on);   // both layers
  void begin_step();  // RtpModel::begin_step (model.cpp:54-57)
  void zero_grads();
  void forward(std::span<const DView> x, size_t rows, std::span<const DView> y, Mode mode);
  void backward(std::span<const DView> dy, size_t rows, std::span<const DView> dx);
  // Tensor API (the shapes of model.cpp:77-105's block): one (rows x h)
  // Tensor per local worker in, one out.
  std::vector<Tensor> forward(std::span<const Tensor> x, Mode mode);
  std::vector<Tensor> backward(std::span<const Tensor> dy);
  RtpLinear& ffn1() { return *ffn1_; }
  RtpLinear& ffn2() { return *ffn2_; }
  // Stack order (RtpModel's block sequence, model.cpp:77-83 / 99-105): `next`
  // runs after this block in forward and before it in backward. Linked
  // blocks post the neighbour's first weight shift under their own last step
  // (SURVEY §8f.1): this block's forward prefetches next's ffn1 forward
  // shift; next's backward prefetches this block's ffn2 backward shift.
  // nullptr unlinks. Out-of-place mode only (the shift lands in the spare).
  void chain(RtpMlp* next);
  ~RtpMlp();  // unlinks its neighbours
  RtpMlp(const RtpMlp&) = delete;
  RtpMlp& operator=(const RtpMlp&) = delete;

 private:
  RtpMlp* next_ = nullptr;
  RtpMlp* prev_ = nullptr;
  void ensure_acts(size_t rows, Mode mode);
  WorkerGroup* group_;
  size_t h_, f_;
  DType dtype_;
  RotationMode mode_ = RotationMode::InPlace;
  std::unique_ptr<RtpLinear> ffn1_, ffn2_;
  std::vector<DeviceBuffer> pre_, act_;  // per rank, rows x f (Activation): the Train batch
  std::vector<DeviceBuffer> eval_act_;   // per rank, rows x f: Eval forwards only
  std::vector<Tensor> x_keep_;           // Tensor API: X held from Train forward to backward
  size_t act_rows_ = 0, eval_rows_ = 0;
  size_t saved_rows_ = 0;  // rows of the Train forward backward will read (0: none)
  // N = 1 fused forward: unit schedule + row-block counters (Other), per rows.
  void ensure_fused(size_t rows);
  DeviceBuffer fused_ws_;
  size_t fused_rows_ = 0;
  int fused_slots_ = 0, fused_dep_rows_ = 0, fused_splits2_ = 1, fused_tiles2_ = 0;
  unsigned fused_dep_target_ = 0;
  size_t fused_sched_ints_ = 0, fused_acc_off_ = 0;
  // N = 1 fused backward: D / W schedules + shared row-block counters.
  void ensure_fused_bwd(size_t rows);
  DeviceBuffer fused_bwd_ws_;
  size_t fused_bwd_rows_ = 0, fused_bwd_sd_ints_ = 0, fused_bwd_sw_ints_ = 0;
  int fused_bwd_slots_d_ = 0, fused_bwd_slots_w_ = 0, fused_bwd_dep_rows_ = 0, fused_bwd_w_splits_ = 1;
  unsigned fused_bwd_dep_target_ = 0;
};

// ---- model (model.hpp:15-61, model.cpp:7-121) ----
struct ModelDims {  // serial.hpp:74-83
  size_t heads = 4;
  size_t hidden = 32;
  size_t layers = 2;
  size_t seq = 16;
  size_t vocab = 64;
  size_t ffn = 128;
  bool moe = false;
  size_t n_experts = 1;  // MoE variant: equals the worker count
};

// Embedding -> layers x (attention + FFN-or-MoE, residual connections) ->
// linear head, every layer rotated (model.cpp:64-121). Parameters are drawn
// from SplitMix64(seed) in SerialModel's order (serial.cpp:325-353), so the
// model equals the reference's RtpModel(SerialModel(dims, seed), ...). The
// FFN of a dense block is an RtpMlp (GELU fused into the step epilogues).
class RtpModel {
 public:
  RtpModel(const ModelDims& dims, uint64_t seed, WorkerGroup& group, RotationMode mode, DType dtype = DType::BF16);
  ~RtpModel();

  // ids[k]: local rank k's tokens (local_batch * seq); returns its logits
  // ((local_batch * seq) x vocab, layer dtype).
  std::vector<Tensor> forward(std::span<const std::vector<int64_t>> ids, Mode mode);
  // Gradients land in the travelling accumulators (and MoE gate gradients).
  void backward(std::span<const Tensor> dlogits);
  void zero_grads();
  // Out of place: one shard-sized spare per layer per worker for the step,
  // all released right after the step's final rotation (model.cpp:113-120).
  void begin_step();
  std::function<void()> on_comm_release;
  bool comm_spares_active() const;

  WorkerGroup& group() { return *group_; }
  RotationMode rotation_mode() const { return mode_; }
  const ModelDims& dims() const { return dims_; }
  // embedding, per block: attention, ffn1, ffn2 (or moe), head (model.cpp:34-52)
  std::vector<RtpLayerBase*> all_layers();
  RtpEmbedding& embedding() { return *embedding_; }
  RtpLinear& head() { return *head_; }
  struct Block {
    std::unique_ptr<RtpAttention> attn;
    std::unique_ptr<RtpMlp> mlp;
    std::unique_ptr<RtpMoe> moe;
  };
  std::vector<Block>& rtp_blocks() { return blocks_; }

 private:
  WorkerGroup* group_;
  RotationMode mode_;
  ModelDims dims_;
  DType dtype_;
  std::unique_ptr<RtpEmbedding> embedding_;
  std::vector<Block> blocks_;
  std::unique_ptr<RtpLinear> head_;
};

// Host fp64 -> device dtype, round-to-nearest-even from the double (no
// double rounding through fp32).
uint16_t double_to_bf16_rne(double v);

}  // namespace rtpb
