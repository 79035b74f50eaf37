// WorkerGroup, transports (in-process device copies; NCCL over NVLink),
// device buffers and per-worker ledgers.
// Reference: proj/src/ring.cpp (rotation, transports), ledger.cpp, tensor.cpp:86-157.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <chrono>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "kernels/launch.hpp"
#include "worker.hpp"

namespace rtpb {

// ------------------------------------------------------------------ errors
void throw_status(int code, const std::string& msg) {
  switch (code) {
    case RTPB_ERR_CONFIG: throw ConfigError(msg);
    case RTPB_ERR_DIMENSION: throw DimensionError(msg);
    case RTPB_ERR_PROTOCOL: throw ProtocolError(msg);
    case RTPB_ERR_STATE: throw StateError(msg);
    case RTPB_ERR_INDEX: throw IndexError(msg);
    case RTPB_ERR_CUDA: throw CudaError(msg);
    case RTPB_ERR_NCCL: throw NcclError(msg);
    default: throw std::runtime_error(msg);
  }
}

void check_status(int code) {
  if (code != RTPB_OK) throw_status(code, rtpb_last_error());
}

void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess)
    throw CudaError(std::string(where) + ": " + cudaGetErrorString(e) + " (" + cudaGetErrorName(e) + ")");
}

static void nccl_check(ncclResult_t r, const char* where) {
  if (r != ncclSuccess) throw NcclError(std::string(where) + ": " + ncclGetErrorString(r));
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev_);
  if (prev_ != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() {
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != prev_) cudaSetDevice(prev_);
}

// ------------------------------------------------------------------ ledger
void MemoryLedger::on_alloc(MemCategory c, size_t bytes) {
  const size_t i = size_t(c);
  current_[i] += bytes;
  peak_[i] = std::max(peak_[i], current_[i]);
  current_total_ += bytes;
  peak_total_ = std::max(peak_total_, current_total_);
  if (mirror_) mirror_->on_alloc(c, bytes);
}
void MemoryLedger::on_release(MemCategory c, size_t bytes) {
  current_[size_t(c)] -= bytes;
  current_total_ -= bytes;
  if (mirror_) mirror_->on_release(c, bytes);
}
void MemoryLedger::reset() {
  current_.fill(0);
  peak_.fill(0);
  current_total_ = 0;
  peak_total_ = 0;
}
void MemoryLedger::reset_peaks() {
  peak_ = current_;
  peak_total_ = current_total_;
}
void MemoryLedger::mirror_to(MemoryLedger* m) {
  if (mirror_)
    for (size_t c = 0; c < kNumMemCategories; ++c) mirror_->on_release(MemCategory(c), current_[c]);
  mirror_ = m;
  if (mirror_)
    for (size_t c = 0; c < kNumMemCategories; ++c)
      if (current_[c]) mirror_->on_alloc(MemCategory(c), current_[c]);
}

// ------------------------------------------------------------------ buffers
DeviceBuffer::DeviceBuffer(int device, size_t bytes, MemoryLedger* ledger, MemCategory cat, bool zero)
    : bytes_(bytes), device_(device), ledger_(ledger), cat_(cat) {
  if (bytes == 0) return;
  DeviceGuard g(device);
  // Whole 2 MiB pages: the driver packs smaller cudaMalloc allocations into a
  // shared page block, and a CUDA IPC mapping covers the block, so two packed
  // buffers could not both be mapped by a peer (the IPC transport exports
  // receive buffers). The ledger keeps the requested size.
  const size_t page = size_t(2) << 20;
  cuda_check(cudaMalloc(&ptr_, (bytes + page - 1) / page * page), "cudaMalloc");
  if (zero) {
    // The worker streams are non-blocking: they do not order behind the legacy
    // stream, so the fill completes here, before any stream can touch the
    // buffer (split-K / bias-tick counters must read 0 on first use).
    cuda_check(cudaMemsetAsync(ptr_, 0, bytes, cudaStreamLegacy), "cudaMemsetAsync");
    cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "zero fill");
  }
  if (ledger_) ledger_->on_alloc(cat_, bytes_);
}
DeviceBuffer::~DeviceBuffer() { reset(); }
void DeviceBuffer::reset() {
  if (ptr_) {
    DeviceGuard g(device_);
    cudaFree(ptr_);
    if (ledger_) ledger_->on_release(cat_, bytes_);
  }
  ptr_ = nullptr;
  bytes_ = 0;
  ledger_ = nullptr;
}
DeviceBuffer::DeviceBuffer(DeviceBuffer&& o) noexcept
    : ptr_(o.ptr_), bytes_(o.bytes_), device_(o.device_), ledger_(o.ledger_), cat_(o.cat_) {
  o.ptr_ = nullptr;
  o.bytes_ = 0;
  o.ledger_ = nullptr;
}
DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
  if (this != &o) {
    reset();
    ptr_ = o.ptr_;
    bytes_ = o.bytes_;
    device_ = o.device_;
    ledger_ = o.ledger_;
    cat_ = o.cat_;
    o.ptr_ = nullptr;
    o.bytes_ = 0;
    o.ledger_ = nullptr;
  }
  return *this;
}
void swap_data(DeviceBuffer& a, DeviceBuffer& b) {
  if (a.bytes_ != b.bytes_ || a.device_ != b.device_)
    throw DimensionError("swap_data: buffers differ in size or device");
  std::swap(a.ptr_, b.ptr_);
}

uint16_t double_to_bf16_rne(double v) {
  // Round to odd into fp32 (sticky bit), then RNE to bf16: a correct single
  // rounding of the double for every normal/subnormal fp32-range value.
  float f = static_cast<float>(v);
  if (static_cast<double>(f) != v && std::isfinite(f)) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    // towards zero if RN went away from zero
    if (std::fabs(static_cast<double>(f)) > std::fabs(v)) u -= 1;
    u |= 1u;
    std::memcpy(&f, &u, 4);
  }
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
  const uint32_t rounding = 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>((u + rounding) >> 16);
}

// ------------------------------------------------------------------ worker
Worker::Worker(size_t r, int dev) : rank(r), device(dev) {
  DeviceGuard g(dev);
  cuda_check(cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&comm, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&comm_g, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking), "stream");
  flags = DeviceBuffer(dev, kFlagPool * sizeof(unsigned), nullptr, MemCategory::Other, true);
  for (auto& e : ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (auto& c : ch_ev)
    for (auto& e : c) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  preload_device_kernels();  // no lazy kernel load may wait behind a spinning grid (launch.hpp)
}
Worker::~Worker() {
  DeviceGuard g(device);
  cudaStreamSynchronize(compute);
  cudaStreamSynchronize(comm);
  cudaStreamSynchronize(comm_g);
  cudaStreamSynchronize(aux);
  stage.reset();
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto& c : ch_ev)
    for (auto& e : c) cudaEventDestroy(e);
  cudaStreamDestroy(aux);
  cudaStreamDestroy(compute);
  cudaStreamDestroy(comm);
  cudaStreamDestroy(comm_g);
}

void stream_write_u32(cudaStream_t s, unsigned* addr, unsigned v) {
  static PFN_cuStreamWriteValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(f);
  }();
  if (!fn) throw CudaError("cuStreamWriteValue32 unavailable");
  const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                        CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed: " + std::to_string(int(r)));
}

void stream_wait_geq_u32(cudaStream_t s, const unsigned* addr, unsigned v) {
  static PFN_cuStreamWaitValue32_v11070 fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(f);
  }();
  if (!fn) throw CudaError("cuStreamWaitValue32 unavailable");
  const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(const_cast<unsigned*>(addr)), v,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed: " + std::to_string(int(r)));
}

size_t inplace_chunk_bytes(size_t shard_bytes) {
  const size_t floor_b = size_t(1) << 20, frac = shard_bytes / 32;
  size_t c = std::max(floor_b, frac);
  c = (c + 255) & ~size_t(255);
  return std::min(c, shard_bytes);
}

void* Worker::staging(size_t bytes, size_t* chunk) {
  const size_t want = inplace_chunk_bytes(bytes);
  if (stage.bytes() < want) {
    cuda_check(cudaStreamSynchronize(comm), "stage sync");  // both channels use the chunk
    cuda_check(cudaStreamSynchronize(comm_g), "stage sync");
    stage.reset();  // release before growing: one staging chunk is ever resident
    stage = DeviceBuffer(device, want, &ledger, MemCategory::CommBuffer, false);
  }
  *chunk = std::min(stage.bytes(), bytes);
  return stage.data();
}

// ------------------------------------------------------------------ local transport
namespace {

class ThreadPool {
 public:
  explicit ThreadPool(size_t n) : tasks_(n), errors_(n) {
    for (size_t i = 0; i < n; ++i) threads_.emplace_back([this, i] { run(i); });
  }
  ~ThreadPool() {
    {
      std::lock_guard lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  // Runs fn(i) on thread i for i < n; re-throws the first failure in index order.
  void dispatch(const std::function<void(size_t)>& fn) {
    {
      std::lock_guard lk(m_);
      for (size_t i = 0; i < tasks_.size(); ++i) {
        tasks_[i] = fn;
        errors_[i] = nullptr;
      }
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    {
      std::unique_lock lk(m_);
      cv_done_.wait(lk, [&] { return done_ == tasks_.size(); });
    }
    for (auto& e : errors_)
      if (e) std::rethrow_exception(e);
  }

 private:
  void run(size_t i) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(size_t)> task;
      {
        std::unique_lock lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ > seen; });
        if (stop_) return;
        seen = gen_;
        task = tasks_[i];
      }
      try {
        task(i);
      } catch (...) {
        errors_[i] = std::current_exception();
      }
      {
        std::lock_guard lk(m_);
        if (++done_ == tasks_.size()) cv_done_.notify_all();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::vector<std::function<void(size_t)>> tasks_;
  std::vector<std::exception_ptr> errors_;
  std::mutex m_;
  std::condition_variable cv_, cv_done_;
  uint64_t gen_ = 0;
  size_t done_ = 0;
  bool stop_ = false;
};

// All n workers in this process (devices may repeat). A shift is a set of
// device-to-device copies, each issued on the RECEIVER's comm stream after
// the sender's comm stream signalled readiness (rendezvous by events).
class LocalTransport final : public Transport {
 public:
  LocalTransport(WorkerGroup& g, bool concurrent) : g_(g) {
    if (concurrent && g.size() > 1) pool_ = std::make_unique<ThreadPool>(g.size());
    // Enable peer access between distinct devices where the platform allows.
    for (size_t a = 0; a < g.size(); ++a)
      for (size_t b = 0; b < g.size(); ++b) {
        const int da = g.worker(a).device, db = g.worker(b).device;
        if (da == db) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, da, db);
        if (can) {
          DeviceGuard dg(da);
          cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
      }
  }

  void each(const std::function<void(size_t)>& fn) override {
    if (pool_) {
      pool_->dispatch([&](size_t r) {
        DeviceGuard dg(g_.worker(r).device);
        fn(r);
      });
    } else {
      for (size_t r = 0; r < g_.size(); ++r) {
        DeviceGuard dg(g_.worker(r).device);
        fn(r);
      }
    }
  }

  void shift(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
             int ch) override {
    const size_t n = g_.size();
    if (n == 1 || bytes == 0) return;
    auto rec = [&](Worker& w, ChEv e, cudaStream_t st) {
      cuda_check(cudaEventRecord(w.ch_event(ch, e), st), "record");
    };
    auto wait = [&](cudaStream_t st, const Worker& w, ChEv e) {
      cuda_check(cudaStreamWaitEvent(st, w.ch_event(ch, e), 0), "wait");
    };
    bool inplace = false;
    for (size_t r = 0; r < n; ++r) inplace = inplace || send[r] == recv[r];
    if (!inplace) {
      for (size_t r = 0; r < n; ++r) {
        Worker& w = g_.worker(r);
        DeviceGuard dg(w.device);
        rec(w, ChEv::Ready, w.comm_of(ch));
      }
      for (size_t r = 0; r < n; ++r) {
        Worker& dst = g_.worker(ring_dest(r, n, dir));
        Worker& src = g_.worker(r);
        DeviceGuard dg(dst.device);
        wait(dst.comm_of(ch), src, ChEv::Ready);
        copy(recv[dst.rank], dst.device, send[r], src.device, bytes, dst.comm_of(ch));
      }
      finish(dir, ch);
      return;
    }
    // In place: chunked ring shift through each sender's staging chunk.
    std::vector<void*> stage(n);
    size_t chunk = bytes;
    for (size_t r = 0; r < n; ++r) {
      size_t c = 0;
      stage[r] = g_.worker(r).staging(bytes, &c);
      chunk = std::min(chunk, c);
    }
    for (size_t off = 0; off < bytes; off += chunk) {
      const size_t c = std::min(chunk, bytes - off);
      for (size_t r = 0; r < n; ++r) {
        Worker& w = g_.worker(r);
        DeviceGuard dg(w.device);
        if (off) wait(w.comm_of(ch), w, ChEv::Consumed);  // previous chunk left my staging buffer
        copy(stage[r], w.device, static_cast<char*>(send[r]) + off, w.device, c, w.comm_of(ch));
        rec(w, ChEv::Staged, w.comm_of(ch));
      }
      for (size_t r = 0; r < n; ++r) {
        Worker& src = g_.worker(r);
        Worker& dst = g_.worker(ring_dest(r, n, dir));
        DeviceGuard dg(dst.device);
        wait(dst.comm_of(ch), src, ChEv::Staged);
        copy(static_cast<char*>(recv[dst.rank]) + off, dst.device, stage[r], src.device, c, dst.comm_of(ch));
        rec(src, ChEv::Consumed, dst.comm_of(ch));
      }
    }
    for (size_t r = 0; r < n; ++r) {
      Worker& w = g_.worker(r);
      DeviceGuard dg(w.device);
      wait(w.comm_of(ch), w, ChEv::Consumed);
    }
    finish(dir, ch);
  }

 private:
  static void copy(void* dst, int ddev, const void* src, int sdev, size_t bytes, cudaStream_t s) {
    if (ddev == sdev)
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync");
    else
      cuda_check(cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, s), "cudaMemcpyPeerAsync");
  }
  // Each rank's comm stream must also be ordered after the copy that read
  // its send buffer (issued on its destination's comm stream).
  void finish(Direction dir, int ch) {
    const size_t n = g_.size();
    for (size_t r = 0; r < n; ++r) {
      Worker& w = g_.worker(r);
      DeviceGuard dg(w.device);
      cuda_check(cudaEventRecord(w.ch_event(ch, ChEv::Comm), w.comm_of(ch)), "record");
    }
    for (size_t r = 0; r < n; ++r) {
      Worker& w = g_.worker(r);
      Worker& reader = g_.worker(ring_dest(r, n, dir));
      DeviceGuard dg(w.device);
      cuda_check(cudaStreamWaitEvent(w.comm_of(ch), reader.ch_event(ch, ChEv::Comm), 0), "wait reader");
    }
  }

  WorkerGroup& g_;
  std::unique_ptr<ThreadPool> pool_;
};

// One process per GPU; the ring shift is ncclSend/ncclRecv on the comm stream.
class NcclTransport final : public Transport {
 public:
  NcclTransport(WorkerGroup& g, size_t rank, const void* id) : g_(g), rank_(rank) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    DeviceGuard dg(g.worker(rank).device);
    nccl_check(ncclCommInitRank(&comm_, int(g.size()), uid, int(rank)), "ncclCommInitRank");
    // channel 1 (a backward pass launch's travelling gradient) gets its own
    // communicator — two streams must not issue on one — made here, not on
    // first use: a collective that may synchronise the device must not run
    // between a pass launch and the shifts it waits for
    nccl_check(ncclCommSplit(comm_, 0, int(rank), &comm2_, nullptr), "ncclCommSplit");
  }
  ~NcclTransport() override {
    if (comm2_) ncclCommDestroy(comm2_);
    if (comm_) ncclCommDestroy(comm_);  // an aborted communicator is already gone
  }
  bool polled() const override { return true; }
  void check_async() override {
    ncclResult_t st = ncclSuccess;
    if (!comm_ || aborted_) return;
    nccl_check(ncclCommGetAsyncError(comm_, &st), "ncclCommGetAsyncError");
    if ((st == ncclSuccess || st == ncclInProgress) && comm2_)
      nccl_check(ncclCommGetAsyncError(comm2_, &st), "ncclCommGetAsyncError");
    if (st != ncclSuccess && st != ncclInProgress) {
      abort();
      throw NcclError(std::string("ring shift failed asynchronously: ") + ncclGetErrorString(st));
    }
  }
  void abort() override {
    if (comm_ && !aborted_) {
      if (comm2_) ncclCommAbort(comm2_);
      ncclCommAbort(comm_);
      comm_ = comm2_ = nullptr;
      aborted_ = true;
    }
  }
  void each(const std::function<void(size_t)>& fn) override {
    DeviceGuard dg(g_.worker(rank_).device);
    fn(rank_);
  }
  void shift(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
             int ch) override {
    const size_t n = g_.size();
    if (n == 1 || bytes == 0) return;
    if (aborted_) throw NcclError("ring shift on an aborted communicator");
    Worker& w = g_.worker(rank_);
    DeviceGuard dg(w.device);
    ncclComm_t comm = ch ? comm2_ : comm_;
    cudaStream_t st = w.comm_of(ch);
    const int dst = int(ring_dest(rank_, n, dir)), src = int(ring_src(rank_, n, dir));
    if (send[rank_] != recv[rank_]) {
      nccl_check(ncclGroupStart(), "ncclGroupStart");
      nccl_check(ncclSend(send[rank_], bytes, ncclUint8, dst, comm, st), "ncclSend");
      nccl_check(ncclRecv(recv[rank_], bytes, ncclUint8, src, comm, st), "ncclRecv");
      nccl_check(ncclGroupEnd(), "ncclGroupEnd");
      return;
    }
    size_t chunk = 0;
    void* stage = w.staging(bytes, &chunk);
    char* buf = static_cast<char*>(send[rank_]);
    for (size_t off = 0; off < bytes; off += chunk) {
      const size_t c = std::min(chunk, bytes - off);
      nccl_check(ncclGroupStart(), "ncclGroupStart");
      nccl_check(ncclSend(buf + off, c, ncclUint8, dst, comm, st), "ncclSend");
      nccl_check(ncclRecv(stage, c, ncclUint8, src, comm, st), "ncclRecv");
      nccl_check(ncclGroupEnd(), "ncclGroupEnd");
      cuda_check(cudaMemcpyAsync(buf + off, stage, c, cudaMemcpyDeviceToDevice, st), "stage copy");
    }
  }

 private:
  WorkerGroup& g_;
  size_t rank_;
  ncclComm_t comm_ = nullptr;
  ncclComm_t comm2_ = nullptr;  // channel 1, split from comm_ at construction
  bool aborted_ = false;
};

}  // namespace

namespace {
// One rank of an n-rank ring with no peers present: every shift is skipped
// (the schedule, events and bookkeeping run as under NCCL). Measurement only:
// the per-GPU compute of an N-way step at its real shapes on one GPU.
class SoloTransport final : public Transport {
 public:
  SoloTransport(WorkerGroup& g, size_t rank) : g_(g), rank_(rank) {}
  void each(const std::function<void(size_t)>& fn) override {
    DeviceGuard dg(g_.worker(rank_).device);
    fn(rank_);
  }
  void shift(Direction, std::span<void* const>, std::span<void* const>, size_t, int) override {}

 private:
  WorkerGroup& g_;
  size_t rank_;
};
}  // namespace

std::unique_ptr<Transport> make_solo_transport(WorkerGroup& g, size_t rank) {
  return std::make_unique<SoloTransport>(g, rank);
}

std::unique_ptr<Transport> make_local_transport(WorkerGroup& g, bool concurrent) {
  return std::make_unique<LocalTransport>(g, concurrent);
}
std::unique_ptr<Transport> make_nccl_transport(WorkerGroup& g, size_t rank, const void* id) {
  return std::make_unique<NcclTransport>(g, rank, id);
}

// ------------------------------------------------------------------ group
WorkerGroup::WorkerGroup(size_t n, TransportKind kind, std::vector<int> devices) : n_(n), kind_(kind) {
  if (n == 0) throw ConfigError("worker group needs at least one worker");
  if (kind == TransportKind::Nccl) throw ConfigError("NCCL groups are created with (n, rank, device, id)");
  if (!devices.empty() && devices.size() != n)
    throw ConfigError("device list size " + std::to_string(devices.size()) + " does not match " +
                      std::to_string(n) + " workers");
  int cur = 0;
  cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
  workers_.resize(n);
  for (size_t r = 0; r < n; ++r) {
    workers_[r] = std::make_unique<Worker>(r, devices.empty() ? cur : devices[r]);
    local_.push_back(r);
  }
  transport_ = make_local_transport(*this, kind == TransportKind::Concurrent);
}

WorkerGroup::WorkerGroup(size_t n, size_t rank, int device, const void* unique_id, TransportKind kind)
    : n_(n), kind_(kind) {
  if (kind != TransportKind::Nccl && kind != TransportKind::Ipc && kind != TransportKind::Solo)
    throw ConfigError("one-process-per-worker groups use the NCCL, IPC or Solo transport");
  if (n == 0) throw ConfigError("worker group needs at least one worker");
  if (rank >= n) throw ConfigError("rank " + std::to_string(rank) + " out of range for " + std::to_string(n));
  workers_.resize(n);
  workers_[rank] = std::make_unique<Worker>(rank, device);
  local_.push_back(rank);
  transport_ = kind == TransportKind::Ipc    ? make_ipc_transport(*this, rank, unique_id)
               : kind == TransportKind::Solo ? make_solo_transport(*this, rank)
                                             : make_nccl_transport(*this, rank, unique_id);
}

WorkerGroup::~WorkerGroup() {
  try {
    synchronize();
  } catch (...) {
  }
  transport_.reset();
}

bool WorkerGroup::is_local(size_t rank) const { return rank < n_ && workers_[rank] != nullptr; }

Worker& WorkerGroup::worker(size_t rank) {
  if (!is_local(rank)) throw IndexError("worker " + std::to_string(rank) + " is not hosted by this process");
  return *workers_[rank];
}

MemoryLedger& WorkerGroup::ledger_of(size_t rank) { return worker(rank).ledger; }

void WorkerGroup::each(const std::function<void(size_t)>& fn) {
  if (bound_.empty()) {
    transport_->each(fn);
    return;
  }
  // bind_ledgers: thunks allocate under the rank's ledger (ring.cpp each())
  transport_->each([&](size_t r) {
    LedgerScope scope(bound_[r], MemCategory::Activation);
    fn(r);
  });
}

void WorkerGroup::bind_ledgers(std::vector<MemoryLedger*> ledgers) {
  if (!ledgers.empty() && ledgers.size() != n_)
    throw ConfigError("bind_ledgers: got " + std::to_string(ledgers.size()) + " ledgers for " + std::to_string(n_) +
                      " workers");
  for (size_t r : local_) worker(r).ledger.mirror_to(ledgers.empty() ? nullptr : ledgers[r]);
  bound_ = std::move(ledgers);
}

MemoryLedger* WorkerGroup::bound_ledger(size_t rank) const { return bound_.empty() ? nullptr : bound_.at(rank); }

std::atomic<int> g_skip_comm{0};

void WorkerGroup::exchange(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
                           int channel) {
  if (send.size() != n_ || recv.size() != n_) throw ConfigError("exchange: buffer arrays must have n entries");
  // rtpb_debug_skip_comm: the schedule, events and bookkeeping stay; only the
  // bytes do not move (compute-only baseline for the exposed-comm measurement).
  if (g_skip_comm.load(std::memory_order_relaxed)) return;
  transport_->shift(dir, send, recv, bytes, channel);
}

bool WorkerGroup::device_shared() const { return transport_ && transport_->device_shared(); }

void WorkerGroup::comm_after_compute() {
  if (comm_fenced_) return;
  for (size_t r : local_) {
    Worker& w = *workers_[r];
    DeviceGuard dg(w.device);
    w.record(Ev::Compute, false);
    w.wait(Ev::Compute, true);
    // channel 1 too: its stream joins a stream capture through this edge
    cuda_check(cudaStreamWaitEvent(w.comm_g, w.ev[int(Ev::Compute)], 0), "wait");
  }
}

void WorkerGroup::compute_after_comm() {
  for (size_t r : local_) {
    Worker& w = *workers_[r];
    DeviceGuard dg(w.device);
    w.record(Ev::Comm, true);
    w.wait(Ev::Comm, false);
  }
}

void WorkerGroup::join_aux() {
  for (size_t r : local_) {
    Worker& w = *workers_[r];
    DeviceGuard dg(w.device);
    w.join_aux();
  }
}

// With a transport whose peers can fail (NCCL), the wait is polled: an
// asynchronous communicator error aborts the communicator and raises
// NcclError, and a wait longer than RTPB_COMM_TIMEOUT_S (default 120 s)
// aborts it and raises ProtocolError — the reference's rendezvous timeout
// (ring.cpp:78-81) for a ring whose neighbour never posts its shift.
void WorkerGroup::synchronize() {
  if (!transport_ || !transport_->polled()) {
    for (size_t r : local_) {
      Worker& w = *workers_[r];
      DeviceGuard dg(w.device);
      cuda_check(cudaStreamSynchronize(w.aux), "sync aux");
      cuda_check(cudaStreamSynchronize(w.compute), "sync compute");
      cuda_check(cudaStreamSynchronize(w.comm), "sync comm");
      cuda_check(cudaStreamSynchronize(w.comm_g), "sync comm (channel 1)");
    }
    return;
  }
  static const double limit_s = [] {
    const char* e = std::getenv("RTPB_COMM_TIMEOUT_S");
    return e ? std::max(0.1, std::atof(e)) : 120.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (size_t r : local_) {
    Worker& w = *workers_[r];
    DeviceGuard dg(w.device);
    for (cudaStream_t s : {w.aux, w.compute, w.comm, w.comm_g}) {
      for (;;) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) cuda_check(q, "sync (polled)");
        transport_->check_async();
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit_s) {
          transport_->abort();
          throw ProtocolError("ring shift timed out after " + std::to_string(limit_s) +
                              " s: a neighbour never posted its shift (RTPB_COMM_TIMEOUT_S)");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      }
    }
  }
}

void WorkerGroup::corrupt_next_exchange(size_t rank, Corrupt what) {
  corrupt_rank_ = rank;
  corrupt_ = what;
}

// Bookkeeping of one hop, as run_exchange + install_payload (ring.cpp:228-261):
// step tag, fault hook, logical id / offset permutation, traffic record.
void WorkerGroup::advance_slots(std::span<ShardSlot> slots, Direction dir, PayloadKind kind,
                                std::string_view label, size_t shard_elems) {
  if (slots.size() != n_)
    throw ConfigError("rotate: got " + std::to_string(slots.size()) + " slots for " + std::to_string(n_) +
                      " workers");
  // traffic volume per worker: the resident shard's element count unless the
  // caller states it (ring.cpp record())
  if (!shard_elems) shard_elems = slots[local_[0]].weight.numel();
  const uint64_t tag = tag_++;
  const long hop = dir == Direction::Clockwise ? +1 : -1;
  const Corrupt what = corrupt_;
  corrupt_ = Corrupt::None;
  const size_t victim = ring_dest(corrupt_rank_, n_, dir);  // receiver of the corrupted message
  if (what == Corrupt::Tag && is_local(victim))
    throw ProtocolError("step tag mismatch at worker " + std::to_string(victim) + ": got " +
                        std::to_string(tag ^ 1) + ", expected " + std::to_string(tag));
  if (kind_ == TransportKind::Nccl || kind_ == TransportKind::Ipc || kind_ == TransportKind::Solo) {
    // SPMD: every rank holds the same offset, so the incoming id is the
    // sender's, i.e. ours shifted by one position against the direction.
    for (size_t r : local_) {
      ShardSlot& s = slots[r];
      s.logical_id = dir == Direction::Clockwise ? (s.logical_id + n_ - 1) % n_ : (s.logical_id + 1) % n_;
      s.rotation_offset += hop;
      if (what == Corrupt::ShardId && r == victim) s.logical_id += 1;
    }
  } else {
    std::vector<size_t> ids(n_);
    std::vector<long> offs(n_);
    for (size_t r = 0; r < n_; ++r) {
      const size_t d = ring_dest(r, n_, dir);
      ids[d] = slots[r].logical_id + ((what == Corrupt::ShardId && r == corrupt_rank_) ? 1 : 0);
      offs[d] = slots[r].rotation_offset + hop;
    }
    for (size_t r = 0; r < n_; ++r) {
      slots[r].logical_id = ids[r];
      slots[r].rotation_offset = offs[r];
    }
  }
  traffic_.push_back({std::string(label), dir == Direction::Clockwise ? "rotation_cw" : "rotation_ccw",
                      shard_elems, kind == PayloadKind::WeightAndGrad ? shard_elems : 0});
}

namespace {
std::vector<void*> ptrs_of(std::span<ShardSlot> slots, bool grad) {
  std::vector<void*> v(slots.size(), nullptr);
  for (size_t r = 0; r < slots.size(); ++r) v[r] = grad ? slots[r].grad_acc.data() : slots[r].weight.data();
  return v;
}
}  // namespace

void WorkerGroup::rotate_clockwise(std::span<ShardSlot> slots, PayloadKind kind, std::string_view label,
                                   size_t shard_elems) {
  if (slots.size() != n_)
    throw ConfigError("rotate: got " + std::to_string(slots.size()) + " slots for " + std::to_string(n_) +
                      " workers");
  if (n_ == 1) return;
  comm_after_compute();
  const size_t r0 = local_[0];
  auto w = ptrs_of(slots, false);
  exchange(Direction::Clockwise, w, w, slots[r0].weight.bytes());
  if (kind == PayloadKind::WeightAndGrad) {
    auto g = ptrs_of(slots, true);
    exchange(Direction::Clockwise, g, g, slots[r0].grad_acc.bytes());
  }
  compute_after_comm();
  advance_slots(slots, Direction::Clockwise, kind, label, shard_elems);
}

void WorkerGroup::rotate_counterclockwise(std::span<ShardSlot> slots, PayloadKind kind, std::string_view label,
                                          size_t shard_elems) {
  if (slots.size() != n_)
    throw ConfigError("rotate: got " + std::to_string(slots.size()) + " slots for " + std::to_string(n_) +
                      " workers");
  if (n_ == 1) return;
  comm_after_compute();
  const size_t r0 = local_[0];
  auto w = ptrs_of(slots, false);
  exchange(Direction::CounterClockwise, w, w, slots[r0].weight.bytes());
  if (kind == PayloadKind::WeightAndGrad) {
    auto g = ptrs_of(slots, true);
    exchange(Direction::CounterClockwise, g, g, slots[r0].grad_acc.bytes());
  }
  compute_after_comm();
  advance_slots(slots, Direction::CounterClockwise, kind, label, shard_elems);
}

void WorkerGroup::rotate_outofplace(std::span<ShardSlot> slots, std::span<Tensor> spares, Direction dir,
                                    PayloadKind kind, std::string_view label, size_t shard_elems) {
  if (slots.size() != n_ || spares.size() != n_)
    throw ConfigError("rotate_outofplace: slot/spare counts do not match worker count");
  for (size_t r : local_)
    if (spares[r].bytes() != slots[r].weight.bytes())
      throw DimensionError("rotate_outofplace: spare buffer of " + std::to_string(spares[r].bytes()) +
                           " bytes does not match shard of " + std::to_string(slots[r].weight.bytes()) + " bytes");
  if (n_ == 1) return;
  comm_after_compute();
  const size_t r0 = local_[0];
  auto w = ptrs_of(slots, false);
  std::vector<void*> sp(n_, nullptr);
  for (size_t r : local_) sp[r] = spares[r].data();
  exchange(dir, w, sp, slots[r0].weight.bytes());
  if (kind == PayloadKind::WeightAndGrad) {  // gradients move in place (ring.cpp:314,328)
    auto g = ptrs_of(slots, true);
    exchange(dir, g, g, slots[r0].grad_acc.bytes());
  }
  compute_after_comm();
  // Receive landed in the spare: swap roles (charges unchanged).
  for (size_t r : local_) swap_data(slots[r].weight, spares[r]);
  advance_slots(slots, dir, kind, label, shard_elems);
}

void WorkerGroup::ring_allgather(std::span<void* const> in, std::span<void* const> out, size_t bytes,
                                 std::string_view label, size_t elem_size) {
  if (in.size() != n_ || out.size() != n_) throw ConfigError("ring_allgather: got wrong number of buffers");
  // Own chunk into place, then N-1 clockwise forwarding steps; each step
  // forwards the chunk received in the previous one (ring.cpp:335-376).
  for (size_t r : local_) {
    Worker& w = worker(r);
    DeviceGuard dg(w.device);
    cuda_check(cudaMemcpyAsync(static_cast<char*>(out[r]) + r * bytes, in[r], bytes, cudaMemcpyDeviceToDevice,
                               w.compute),
               "allgather own");
  }
  if (n_ == 1) return;
  comm_after_compute();
  for (size_t s = 0; s + 1 < n_; ++s) {
    std::vector<void*> snd(n_, nullptr), rcv(n_, nullptr);
    for (size_t r : local_) {
      const size_t fwd_id = (r + n_ - s) % n_;      // chunk being forwarded
      const size_t src_id = (r + n_ - s - 1) % n_;  // chunk arriving
      snd[r] = static_cast<char*>(out[r]) + fwd_id * bytes;
      rcv[r] = static_cast<char*>(out[r]) + src_id * bytes;
    }
    exchange(Direction::Clockwise, snd, rcv, bytes);
    traffic_.push_back({std::string(label), "allgather", bytes / elem_size, 0});
  }
  compute_after_comm();
}

std::vector<Tensor> WorkerGroup::ring_allgather(std::span<const Tensor> shards, std::string_view label) {
  if (shards.size() != n_) throw ConfigError("ring_allgather: got wrong number of shards");
  const Tensor& t0 = shards[local_[0]];
  std::vector<Tensor> out(n_);
  std::vector<void*> in(n_, nullptr), op(n_, nullptr);
  for (size_t r : local_) {
    if (shards[r].bytes() != t0.bytes() || shards[r].dtype() != t0.dtype())
      throw DimensionError("ring_allgather: shards differ in size or dtype");
    Worker& w = worker(r);
    MemoryLedger* l = bound_.empty() ? LedgerScope::current_ledger() : bound_[r];
    out[r] = Tensor({n_ * t0.numel()}, t0.dtype(), w.device, l, MemCategory::Activation, false);
    in[r] = shards[r].data();
    op[r] = out[r].data();
  }
  ring_allgather(in, op, t0.bytes(), label, dtype_size(t0.dtype()));
  synchronize();
  return out;
}

}  // namespace rtpb
