// Internal: per-worker device state and the Transport interface.
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <span>

#include "rtpb/rtp.hpp"

namespace rtpb {

// RAII cudaSetDevice scope.
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev);
  ~DeviceGuard();

 private:
  int prev_ = 0;
};

void cuda_check(cudaError_t e, const char* where);

// Stream-ordering markers of one worker. Compute: last enqueued compute
// work; WDone / GDone: completion of the latest weight / gradient exchange.
// Fork / Join: compute <-> aux stream hand-offs (N = 1 dX || dW overlap).
enum class Ev : int {
  Compute = 0, WDone = 1, GDone = 2, Comm = 3, Ready = 4, Consumed = 5, Staged = 6, Fork = 7, Join = 8, AuxDone = 9,
  PassEnd = 10, PassEndG = 11, kCount = 12
};

// Ring-shift channels: 0 carries the weight shards (and, outside the pass
// launches, the gradients), 1 the travelling gradient of a backward pass
// launch, so the dW chain and the dX launch's weight shifts do not queue
// behind each other on one stream. Each channel has its own comm stream and
// transport events (and, under NCCL, its own communicator).
constexpr int kChannels = 2;
enum class ChEv : int { Ready = 0, Comm = 1, Staged = 2, Consumed = 3, kCount = 4 };

struct Worker {
  Worker(size_t rank, int device);
  ~Worker();
  size_t rank;
  int device;
  cudaStream_t compute = nullptr;
  cudaStream_t comm = nullptr;    // channel 0
  cudaStream_t comm_g = nullptr;  // channel 1
  cudaEvent_t ch_ev[kChannels][int(ChEv::kCount)] = {};
  cudaStream_t comm_of(int channel) const { return channel ? comm_g : comm; }
  cudaEvent_t ch_event(int channel, ChEv e) const { return ch_ev[channel][int(e)]; }
  // Second compute stream: with no rotation to wait for (N = 1), dW runs here
  // beside dX, each GEMM on its share of the SMs (RtpLinear::backward_ex).
  cudaStream_t aux = nullptr;
  bool aux_pending = false;  // aux has work compute has not joined yet
  cudaEvent_t ev[int(Ev::kCount)] = {};
  MemoryLedger ledger;
  DeviceBuffer stage;  // in-place rotation staging chunk (CommBuffer)
  // Shard-arrival flags written by the comm stream (stream memory ops) and
  // waited on inside the step GEMMs; kFlagsPerLayer per layer.
  static constexpr size_t kFlagPool = 16384, kFlagsPerLayer = 128;
  DeviceBuffer flags;
  unsigned* flag(size_t i) { return static_cast<unsigned*>(flags.data()) + i; }

  void record(Ev e, bool on_comm) { cuda_check(cudaEventRecord(ev[int(e)], on_comm ? comm : compute), "record"); }
  void wait(Ev e, bool on_comm) {
    cuda_check(cudaStreamWaitEvent(on_comm ? comm : compute, ev[int(e)], 0), "wait");
  }
  // aux waits for everything enqueued on compute so far.
  void fork_aux() {
    cuda_check(cudaEventRecord(ev[int(Ev::Fork)], compute), "record fork");
    cuda_check(cudaStreamWaitEvent(aux, ev[int(Ev::Fork)], 0), "wait fork");
    aux_pending = true;
  }
  // compute waits for everything enqueued on aux so far.
  void join_aux() {
    if (!aux_pending) return;
    cuda_check(cudaEventRecord(ev[int(Ev::Join)], aux), "record join");
    cuda_check(cudaStreamWaitEvent(compute, ev[int(Ev::Join)], 0), "wait join");
    aux_pending = false;
  }
  // Generic record / wait on any of this worker's streams.
  void record_on(Ev e, cudaStream_t s) { cuda_check(cudaEventRecord(ev[int(e)], s), "record"); }
  void wait_on(Ev e, cudaStream_t s) { cuda_check(cudaStreamWaitEvent(s, ev[int(e)], 0), "wait"); }
  // Staging for an in-place shift of `bytes`: one chunk, charged as CommBuffer.
  void* staging(size_t bytes, size_t* chunk);
};

// Stream memory operation: *addr = v once the stream's prior work is done
// (cuStreamWriteValue32 with its default memory barrier).
void stream_write_u32(cudaStream_t s, unsigned* addr, unsigned v);
// Stream memory operation: the stream waits until *addr >= v
// (cuStreamWaitValue32, GEQ) — written by a kernel still running on another
// stream (a pass launch's count-ins).
void stream_wait_geq_u32(cudaStream_t s, const unsigned* addr, unsigned v);

// In-place rotation staging chunk: a small fraction of the shard so the
// in-place mode stays within its (W+G)/N memory model.
size_t inplace_chunk_bytes(size_t shard_bytes);

class Transport {
 public:
  virtual ~Transport() = default;
  virtual void each(const std::function<void(size_t)>& fn) = 0;
  // recv[dest(r)] <- send[r] for every rank r; arrays indexed by rank (only
  // local entries are read). Enqueued on the comm streams; send == recv at a
  // rank means in place. On return the comm streams are ordered after the
  // transfer (both the rank's receive and its send).
  virtual void shift(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
                     int channel) = 0;
  // Host-side wait watchdog (WorkerGroup::synchronize): true when waits on
  // this transport's streams must be polled (a peer can fail or vanish).
  virtual bool polled() const { return false; }
  // Called while polling: throws (after aborting the transport) on an
  // asynchronous transport error.
  virtual void check_async() {}
  // The wait exceeded its deadline: abort the transport (unblocks the
  // streams) before the caller throws.
  virtual void abort() {}
  // Another worker's process shares this worker's GPU (time-sliced between
  // processes): a grid that spins on arrival flags for a whole pass can hold
  // the GPU while the peer it waits for is switched out, so pass launches
  // are off for such groups (RtpLinear::pass_launch_ok).
  virtual bool device_shared() const { return false; }
};

std::unique_ptr<Transport> make_local_transport(WorkerGroup& g, bool concurrent);
std::unique_ptr<Transport> make_nccl_transport(WorkerGroup& g, size_t rank, const void* nccl_id);
std::unique_ptr<Transport> make_ipc_transport(WorkerGroup& g, size_t rank, const void* unique_id);
std::unique_ptr<Transport> make_solo_transport(WorkerGroup& g, size_t rank);

inline size_t ring_dest(size_t r, size_t n, Direction d) {
  return d == Direction::Clockwise ? (r + 1) % n : (r + n - 1) % n;
}
inline size_t ring_src(size_t r, size_t n, Direction d) {
  return d == Direction::Clockwise ? (r + n - 1) % n : (r + 1) % n;
}

// Tensor-API helpers shared by the layers (rtp_layers.cpp).
namespace detail {
// x holds one tensor per rank (n, all local) or one per local rank: the
// tensors of the local ranks, in local order.
std::vector<const Tensor*> per_local(WorkerGroup& g, std::span<const Tensor> x, const std::string& label,
                                     const char* what);
// t as a layer input on worker w: checked (rank 2, `cols` columns, w's
// device); converted to dt into `keep` when its dtype differs, or copied
// there when keep_same (the layer holds it past the call).
const Tensor& as_layer_input(const Tensor& t, DType dt, Worker& w, size_t cols, const std::string& label,
                             Tensor& keep, bool keep_same);
}  // namespace detail

}  // namespace rtpb
