// IPC transport: one process per worker, the ring shift is a copy-engine push
// (cudaMemcpyAsync into the neighbour's buffer through a CUDA IPC mapping —
// NVLink P2P between GPUs, a device-local copy when two workers share a GPU)
// ordered by stream memory operations on flags in the peers' device memory.
// No SMs are used, so a shift overlaps the persistent step GEMMs completely.
//
// Per shift q (every rank issues the same sequence of shifts, as the SPMD
// schedule guarantees), on the rank's comm stream, which is already ordered
// after its compute stream (comm_after_compute):
//   a) write ready[dir] = q into the SOURCE's flags   (my receive buffer is free)
//   b) wait  my ready[dir] >= q                        (the destination's is)
//   c) copy  send -> destination's receive buffer      (copy engine)
//   d) write done[dir] = q into the DESTINATION's flags (its data has landed)
//   e) wait  my done[dir] >= q                         (mine has)
// Every rank writes (a) before it waits (b), so the chain cannot deadlock.
// In place (send == recv), each chunk goes through the destination's staging
// chunk the same way and is then copied locally into place.
//
// Receive pointers are exchanged on the host per shift through a POSIX
// shared-memory mailbox (node-local rendezvous keyed by the group's unique
// id): the receiver publishes (IPC handle of the allocation, offset); the
// sender maps it (handles cached per peer). The flags buffers are exchanged
// once at group creation. Counterpart of the reference's Transport::exchange
// (ring.cpp:38-48, 113-131) for processes instead of threads.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>

#include "worker.hpp"

namespace rtpb {

namespace {

PFN_cuStreamWriteValue32_v11070 p_write = nullptr;
PFN_cuStreamWaitValue32_v11070 p_wait = nullptr;
PFN_cuMemGetAddressRange_v3020 p_range = nullptr;
PFN_cuPointerGetAttribute_v4000 p_attr = nullptr;
std::once_flag g_drv_once;

void load_driver() {
  std::call_once(g_drv_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      p_attr = reinterpret_cast<PFN_cuPointerGetAttribute_v4000>(fn);
  });
  if (!p_write || !p_wait || !p_range || !p_attr)
    throw CudaError("IPC transport: stream memory operations unavailable");
}

void cu_check(CUresult r, const char* where) {
  if (r != CUDA_SUCCESS) throw CudaError(std::string(where) + ": CUDA driver error " + std::to_string(int(r)));
}

constexpr int kMaxRanks = 64;
constexpr int kSlots = 64;  // mailbox depth (shifts a host may run ahead of its neighbour)

struct Mail {
  std::atomic<uint64_t> seq;  // q + 1 once published
  cudaIpcMemHandle_t handle;
  uint64_t buffer_id;  // CU_POINTER_ATTRIBUTE_BUFFER_ID: unique per allocation in the exporter
  uint64_t offset;
};
struct Shm {
  std::atomic<uint32_t> joined, left;
  std::atomic<uint32_t> flags_ready[kMaxRanks];
  char bus_id[kMaxRanks][32];  // PCI bus id of each rank's device (written before flags_ready)
  cudaIpcMemHandle_t flags_handle[kMaxRanks];
  std::atomic<uint64_t> consumed[kMaxRanks];  // highest q+1 whose mailbox entry the reader took
  Mail mail[kMaxRanks][kSlots];
};

template <class Pred>
void spin_until(Pred p, const char* what) {
  const auto t0 = std::chrono::steady_clock::now();
  while (!p()) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
      throw ProtocolError(std::string("IPC transport: timed out waiting for ") + what +
                          " (a peer process stopped or issued a different shift sequence)");
    std::this_thread::yield();
  }
}

class IpcTransport final : public Transport {
 public:
  IpcTransport(WorkerGroup& g, size_t rank, const void* id) : g_(g), rank_(rank), n_(g.size()) {
    if (n_ > size_t(kMaxRanks)) throw ConfigError("IPC transport: at most 64 workers");
    load_driver();
    const unsigned char* b = static_cast<const unsigned char*>(id);
    char name[64];
    std::snprintf(name, sizeof name, "/rtpb_ipc_%02x%02x%02x%02x%02x%02x%02x%02x", b[0], b[1], b[2], b[3], b[4], b[5],
                  b[6], b[7]);
    name_ = name;
    const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) throw ConfigError(std::string("IPC transport: shm_open failed for ") + name);
    if (ftruncate(fd, sizeof(Shm)) != 0) {
      close(fd);
      throw ConfigError("IPC transport: ftruncate failed");
    }
    void* m = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) throw ConfigError("IPC transport: mmap failed");
    shm_ = static_cast<Shm*>(m);
    Worker& w = g_.worker(rank_);
    DeviceGuard dg(w.device);
    // flags: ready[2], done[2] (uint32, zeroed), exported to every peer
    flags_ = DeviceBuffer(w.device, 256, nullptr, MemCategory::Other, true);
    cuda_check(cudaIpcGetMemHandle(&shm_->flags_handle[rank_], flags_.data()), "cudaIpcGetMemHandle(flags)");
    cuda_check(cudaDeviceGetPCIBusId(shm_->bus_id[rank_], 32, w.device), "cudaDeviceGetPCIBusId");
    shm_->flags_ready[rank_].store(1, std::memory_order_release);
    shm_->joined.fetch_add(1);
    peer_flags_.assign(n_, nullptr);
    for (size_t r = 0; r < n_; ++r) {
      if (r == rank_) {
        peer_flags_[r] = static_cast<uint32_t*>(flags_.data());
        continue;
      }
      spin_until([&] { return shm_->flags_ready[r].load(std::memory_order_acquire) != 0; }, "peer flags");
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, shm_->flags_handle[r], cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle(flags)");
      peer_flags_[r] = static_cast<uint32_t*>(p);
      opened_.push_back(p);
      if (std::strncmp(shm_->bus_id[r], shm_->bus_id[rank_], 32) == 0) shared_ = true;
    }
  }

  bool device_shared() const override { return shared_; }

  ~IpcTransport() override {
    try {
      Worker& w = g_.worker(rank_);
      DeviceGuard dg(w.device);
      cudaStreamSynchronize(w.comm);
      for (void* p : opened_) cudaIpcCloseMemHandle(p);
    } catch (...) {
    }
    if (shm_) {
      if (shm_->left.fetch_add(1) + 1 == uint32_t(n_)) shm_unlink(name_.c_str());
      munmap(shm_, sizeof(Shm));
    }
  }

  void each(const std::function<void(size_t)>& fn) override {
    DeviceGuard dg(g_.worker(rank_).device);
    fn(rank_);
  }

  // A peer that dies after publishing its buffer leaves this rank's comm
  // stream in cuStreamWaitValue32 with no deadline: the group's host wait is
  // polled instead (WorkerGroup::synchronize, RTPB_COMM_TIMEOUT_S — the
  // reference's rendezvous timeout, ring.cpp:78-81), and on timeout abort()
  // releases the device waits by raising this rank's own flags past any
  // sequence number, then refuses further shifts.
  bool polled() const override { return true; }
  void abort() override {
    if (aborted_) return;
    aborted_ = true;
    Worker& w = g_.worker(rank_);
    DeviceGuard dg(w.device);
    cudaStream_t st = nullptr;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess) {
      cudaMemsetAsync(flags_.data(), 0xFF, 8 * sizeof(uint32_t), st);  // both channels' ready / done := UINT32_MAX
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }

  void shift(Direction dir, std::span<void* const> send, std::span<void* const> recv, size_t bytes,
             int ch) override {
    if (n_ == 1 || bytes == 0) return;
    if (aborted_) throw ProtocolError("IPC transport: aborted after a ring shift timed out");
    Worker& w = g_.worker(rank_);
    DeviceGuard dg(w.device);
    const size_t dst = ring_dest(rank_, n_, dir), src = ring_src(rank_, n_, dir);
    // flag words per channel: [ready cw, ready ccw, done cw, done ccw]
    const int d = (dir == Direction::Clockwise ? 0 : 1) + 4 * ch;
    uint32_t* mine = static_cast<uint32_t*>(flags_.data());
    cudaStream_t st = w.comm_of(ch);
    auto write = [&](uint32_t* addr, uint32_t v) {
      cu_check(p_write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v,
                       CU_STREAM_WRITE_VALUE_DEFAULT),
               "cuStreamWriteValue32");
    };
    auto wait = [&](uint32_t* addr, uint32_t v) {
      cu_check(p_wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v,
                      CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue32");
    };
    if (send[rank_] != recv[rank_]) {
      const uint32_t q = ++seq_[d];
      void* peer_recv = publish_and_fetch(recv[rank_], dst, src);
      write(peer_flags_[src] + 0 + d, q);  // a) my receive buffer is free
      wait(mine + 0 + d, q);               // b) the destination's is
      cuda_check(cudaMemcpyAsync(peer_recv, send[rank_], bytes, cudaMemcpyDeviceToDevice, st), "IPC push");
      write(peer_flags_[dst] + 2 + d, q);  // d) the destination's data landed
      wait(mine + 2 + d, q);               // e) mine has
      return;
    }
    // In place: chunked through the destination's staging chunk.
    size_t chunk = 0;
    void* stage = w.staging(bytes, &chunk);
    void* peer_stage = publish_and_fetch(stage, dst, src);
    char* buf = static_cast<char*>(send[rank_]);
    for (size_t off = 0; off < bytes; off += chunk) {
      const size_t c = std::min(chunk, bytes - off);
      const uint32_t q = ++seq_[d];
      write(peer_flags_[src] + 0 + d, q);  // my staging chunk is free
      wait(mine + 0 + d, q);
      cuda_check(cudaMemcpyAsync(peer_stage, buf + off, c, cudaMemcpyDeviceToDevice, st), "IPC push chunk");
      write(peer_flags_[dst] + 2 + d, q);
      wait(mine + 2 + d, q);               // the source's chunk is in my staging
      cuda_check(cudaMemcpyAsync(buf + off, stage, c, cudaMemcpyDeviceToDevice, st), "IPC stage copy");
    }
  }

 private:
  // Publish my receive buffer for this shift; return the destination's.
  void* publish_and_fetch(void* my_recv, size_t dst, size_t src) {
    const uint64_t q = ++host_seq_;
    const int slot = int(q % kSlots);
    // every rank must have taken its entries of the shift this slot held
    // kSlots shifts ago (its reader depended on that shift's direction)
    spin_until(
        [&] {
          for (size_t r = 0; r < n_; ++r)
            if (shm_->consumed[r].load(std::memory_order_acquire) + kSlots < q) return false;
          return true;
        },
        "mailbox slot");
    (void)src;
    CUdeviceptr base = 0;
    size_t size = 0;
    cu_check(p_range(&base, &size, reinterpret_cast<CUdeviceptr>(my_recv)), "cuMemGetAddressRange");
    Mail& m = shm_->mail[rank_][slot];
    cuda_check(cudaIpcGetMemHandle(&m.handle, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
    unsigned long long my_bid = 0;
    cu_check(p_attr(&my_bid, CU_POINTER_ATTRIBUTE_BUFFER_ID, base), "cuPointerGetAttribute(BUFFER_ID)");
    m.buffer_id = my_bid;
    m.offset = reinterpret_cast<uint64_t>(my_recv) - uint64_t(base);
    m.seq.store(q, std::memory_order_release);
    // the destination's entry for the same shift
    Mail& theirs = shm_->mail[dst][slot];
    spin_until([&] { return theirs.seq.load(std::memory_order_acquire) == q; }, "peer receive buffer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, &theirs.handle, sizeof h);
    const uint64_t off = theirs.offset, bid = theirs.buffer_id;
    shm_->consumed[rank_].store(q, std::memory_order_release);  // I (dst's source) took dst's entry q
    // One mapping per peer allocation, keyed by its buffer id: a freed and
    // re-made allocation at the same address (same handle bytes) gets a new
    // id, so a stale mapping is never reused. Stale mappings stay open until
    // the transport closes (their memory is not reused meanwhile).
    auto it = mapped_.find({dst, bid});
    void* p = nullptr;
    if (it != mapped_.end()) {
      p = it->second;
    } else {
      cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      opened_.push_back(p);
      mapped_[{dst, bid}] = p;
    }
    return static_cast<char*>(p) + off;
  }

  WorkerGroup& g_;
  size_t rank_, n_;
  std::string name_;
  Shm* shm_ = nullptr;
  DeviceBuffer flags_;
  std::vector<uint32_t*> peer_flags_;
  std::vector<void*> opened_;
  std::map<std::pair<size_t, uint64_t>, void*> mapped_;  // (peer rank, buffer id) -> mapping
  uint32_t seq_[8] = {};  // per flag word (direction + 4 * channel)
  uint64_t host_seq_ = 0;
  bool aborted_ = false;
  bool shared_ = false;  // a peer process runs on the same GPU
};

}  // namespace

std::unique_ptr<Transport> make_ipc_transport(WorkerGroup& g, size_t rank, const void* id) {
  return std::make_unique<IpcTransport>(g, rank, id);
}

}  // namespace rtpb
