// Device Tensor, ledger scopes and layout_linear: the value types of the
// reference's host API (tensor.hpp, ledger.hpp, partition.hpp) with device
// storage. Element conversions run on the device (rtpb_convert / rtpb_fill).
#include <cuda_runtime.h>

#include <cstring>

#include "worker.hpp"

namespace rtpb {

const char* mem_category_name(MemCategory c) {
  switch (c) {
    case MemCategory::Param: return "Param";
    case MemCategory::Grad: return "Grad";
    case MemCategory::Activation: return "Activation";
    case MemCategory::CommBuffer: return "CommBuffer";
    case MemCategory::Other: return "Other";
  }
  return "?";
}

namespace {
thread_local MemoryLedger* t_ledger = nullptr;
thread_local MemCategory t_category = MemCategory::Other;

int current_device() {
  int d = 0;
  cuda_check(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}

size_t count_of(const std::vector<size_t>& shape) {
  size_t n = 1;
  for (size_t d : shape) n *= d;
  return shape.empty() ? 0 : n;
}
}  // namespace

LedgerScope::LedgerScope(MemoryLedger* ledger, MemCategory category)
    : prev_ledger_(t_ledger), prev_category_(t_category) {
  t_ledger = ledger;
  t_category = category;
}
LedgerScope::~LedgerScope() {
  t_ledger = prev_ledger_;
  t_category = prev_category_;
}
MemoryLedger* LedgerScope::current_ledger() { return t_ledger; }
MemCategory LedgerScope::current_category() { return t_category; }

// ------------------------------------------------------------------ Tensor
Tensor::Tensor(std::vector<size_t> shape, DType dtype)
    : Tensor(std::move(shape), dtype, current_device(), t_ledger, t_category, true) {}

Tensor::Tensor(std::vector<size_t> shape, DType dtype, int device, MemoryLedger* ledger, MemCategory cat, bool zero)
    : shape_(std::move(shape)), dtype_(dtype) {
  const size_t n = count_of(shape_);
  if (n) buf_ = DeviceBuffer(device, n * dtype_size(dtype_), ledger, cat, zero);
}

Tensor::Tensor(const Tensor& o) : shape_(o.shape_), dtype_(o.dtype_) {
  if (o.empty()) return;
  buf_ = DeviceBuffer(o.device(), o.bytes(), t_ledger, t_category, false);
  DeviceGuard g(o.device());
  cuda_check(cudaMemcpy(buf_.data(), o.data(), o.bytes(), cudaMemcpyDeviceToDevice), "Tensor copy");
}

Tensor& Tensor::operator=(const Tensor& o) {
  if (this != &o) {
    Tensor t(o);
    *this = std::move(t);
  }
  return *this;
}

Tensor Tensor::from_host(std::vector<size_t> shape, std::span<const double> values, DType dtype, int device) {
  const size_t n = count_of(shape);
  if (values.size() != n)
    throw DimensionError("Tensor::from_host: " + std::to_string(values.size()) + " values for shape of " +
                         std::to_string(n) + " elements");
  if (device < 0) device = current_device();
  Tensor t(std::move(shape), dtype, device, t_ledger, t_category, false);
  if (!n) return t;
  DeviceGuard g(device);
  if (dtype == DType::F64) {
    cuda_check(cudaMemcpy(t.data(), values.data(), n * 8, cudaMemcpyHostToDevice), "Tensor upload");
    return t;
  }
  // stage as fp64, round once on the device (RN, no double rounding)
  void* tmp = nullptr;
  cuda_check(cudaMalloc(&tmp, n * 8), "cudaMalloc");
  cuda_check(cudaMemcpy(tmp, values.data(), n * 8, cudaMemcpyHostToDevice), "Tensor upload");
  const int rc = rtpb_convert(tmp, RTPB_F64, t.data(), int(dtype), n, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(tmp);
  check_status(rc);
  cuda_check(e, "Tensor upload convert");
  return t;
}

Tensor Tensor::uniform(std::vector<size_t> shape, SplitMix64& rng, double lo, double hi, DType dtype, int device) {
  std::vector<double> v(count_of(shape));
  for (double& x : v) x = rng.next_uniform(lo, hi);
  return from_host(std::move(shape), v, dtype, device);
}

size_t Tensor::numel() const { return count_of(shape_); }

size_t Tensor::rows() const {
  if (shape_.size() != 2) throw DimensionError("rows() on a tensor of shape " + shape_str());
  return shape_[0];
}

size_t Tensor::cols() const {
  if (shape_.size() != 2) throw DimensionError("cols() on a tensor of shape " + shape_str());
  return shape_[1];
}

std::string Tensor::shape_str() const {
  std::string s = "[";
  for (size_t i = 0; i < shape_.size(); ++i) s += (i ? ", " : "") + std::to_string(shape_[i]);
  return s + "]";
}

std::vector<double> Tensor::to_host() const {
  const size_t n = numel();
  std::vector<double> out(n);
  if (!n) return out;
  DeviceGuard g(device());
  cuda_check(cudaDeviceSynchronize(), "Tensor read (pending work)");
  if (dtype_ == DType::F64) {
    cuda_check(cudaMemcpy(out.data(), data(), n * 8, cudaMemcpyDeviceToHost), "Tensor read");
    return out;
  }
  void* tmp = nullptr;
  cuda_check(cudaMalloc(&tmp, n * 8), "cudaMalloc");
  const int rc = rtpb_convert(data(), int(dtype_), tmp, RTPB_F64, n, nullptr);
  cudaError_t e = cudaMemcpy(out.data(), tmp, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  check_status(rc);
  cuda_check(e, "Tensor read");
  return out;
}

double Tensor::at(size_t i) const {
  if (i >= numel()) throw IndexError("Tensor::at: index " + std::to_string(i) + " out of range " + shape_str());
  DeviceGuard g(device());
  cuda_check(cudaDeviceSynchronize(), "Tensor read (pending work)");
  const size_t es = dtype_size(dtype_);
  unsigned char raw[8] = {};
  cuda_check(cudaMemcpy(raw, static_cast<const char*>(data()) + i * es, es, cudaMemcpyDeviceToHost), "Tensor::at");
  if (dtype_ == DType::F64) {
    double v;
    std::memcpy(&v, raw, 8);
    return v;
  }
  if (dtype_ == DType::F32) {
    float v;
    std::memcpy(&v, raw, 4);
    return v;
  }
  uint32_t u = uint32_t(raw[0] | (raw[1] << 8)) << 16;
  float v;
  std::memcpy(&v, &u, 4);
  return v;
}

void Tensor::fill(double v) {
  if (empty()) return;
  DeviceGuard g(device());
  check_status(rtpb_fill(data(), int(dtype_), numel(), v, nullptr));
  cuda_check(cudaDeviceSynchronize(), "Tensor::fill");
}

Tensor Tensor::to(DType dtype) const {
  if (dtype == dtype_) return *this;
  Tensor t(shape_, dtype, device(), t_ledger, t_category, false);
  if (empty()) return t;
  DeviceGuard g(device());
  cuda_check(cudaDeviceSynchronize(), "Tensor::to (pending work)");
  check_status(rtpb_convert(data(), int(dtype_), t.data(), int(dtype), numel(), nullptr));
  cuda_check(cudaDeviceSynchronize(), "Tensor::to");
  return t;
}

Tensor Tensor::reshaped(std::vector<size_t> shape) const& {
  Tensor t(*this);
  return std::move(t).reshaped(std::move(shape));
}

Tensor Tensor::reshaped(std::vector<size_t> shape) && {
  if (count_of(shape) != numel())
    throw DimensionError("reshaped: " + shape_str() + " has " + std::to_string(numel()) + " elements");
  shape_ = std::move(shape);
  return std::move(*this);
}

void swap_data(Tensor& a, Tensor& b) {
  if (a.bytes() != b.bytes() || a.device() != b.device())
    throw DimensionError("swap_data: tensors differ in size or device");
  swap_data(a.buf_, b.buf_);
}

// ------------------------------------------------------------------ partition
ShardLayout layout_linear(size_t in_dim, size_t out_dim, size_t n) {
  if (n == 0) throw ConfigError("layout_linear: shard count must be >= 1");
  if (in_dim == 0 || out_dim == 0) throw ConfigError("layout_linear: dimensions must be positive");
  if (out_dim % n != 0)
    throw ConfigError("layout_linear: out_dim " + std::to_string(out_dim) + " not divisible by " +
                      std::to_string(n) + " shards; choose out_dim as a multiple of the worker count");
  ShardLayout l;
  l.strategy = PartitionStrategy::OutputPartition;
  l.n_shards = n;
  const size_t per = out_dim / n;
  for (size_t j = 0; j < n; ++j) l.ranges.push_back({j * per, (j + 1) * per});
  return l;
}

}  // namespace rtpb
