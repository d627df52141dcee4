// Host-value Tensor / slice / merge (reshard/tensor.hpp): the reference's tensor-core
// interface (proj/include/reshard/tensor/tensor.hpp:16-47) over the GPU tile-copy path.
#include "reshard/tensor.hpp"

#include <cuda_runtime.h>

#include <memory>
#include <mutex>

#include "reshard/executor.hpp"
#include "reshard/trace.hpp"

namespace reshard {

// tensor.cpp:9-17: zero extents and a payload of the wrong size are InvalidTensor
Tensor::Tensor(Dtype dtype, Shape shape, std::vector<uint8_t> payload)
    : dtype_(dtype), shape_(std::move(shape)), payload_(std::move(payload)) {
  for (uint64_t e : shape_)
    if (e == 0) raise(Errc::InvalidTensor, "zero extent");
  const uint64_t want = shape_elements(shape_) * dtype_width(dtype_);
  if (payload_.size() != want)
    raise(Errc::InvalidTensor, "payload " + std::to_string(payload_.size()) + " bytes, expected " + std::to_string(want));
}

Tensor Tensor::zeros(Dtype dtype, Shape shape) {
  const uint64_t bytes = shape_elements(shape) * dtype_width(dtype);
  return Tensor(dtype, std::move(shape), std::vector<uint8_t>(bytes, 0));
}

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffers of one call, freed on every exit path.
struct DeviceBuffers {
  int dev;
  std::vector<void*> p;
  explicit DeviceBuffers(int d) : dev(d) {}
  void* alloc(size_t bytes) {
    void* x = nullptr;
    ck(cudaMalloc(&x, std::max<size_t>(bytes, 1)), "cudaMalloc");
    p.push_back(x);
    return x;
  }
  ~DeviceBuffers() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    for (void* x : p) cudaFree(x);
    cudaSetDevice(cur);
  }
};

std::mutex g_mu;  // the default context and every host-value call on it
int g_device = 0;
std::unique_ptr<Context> g_ctx;

Context& default_context() {
  if (!g_ctx) g_ctx = std::make_unique<Context>(1, std::vector<int>{0}, std::vector<int>{g_device});
  return *g_ctx;
}

}  // namespace

void set_default_device(int cuda_device) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (g_ctx) raise(Errc::InvalidArgument, "set_default_device after the first slice / merge");
  g_device = cuda_device;
}

void host_slice(Context& ctx, int gpu, const HostTensorView& t, const Range& r, void* out) {
  TraceRange trace_("host_slice");
  for (auto e : t.shape)
    if (e == 0) raise(Errc::InvalidTensor, "zero extent");
  const uint64_t w = dtype_width(t.dtype);
  r.check_against(t.shape);  // every reference error before any device work
  const uint64_t in_bytes = shape_elements(t.shape) * w, out_bytes = r.elements() * w;
  const int dev = ctx.cuda_device(gpu);
  ck(cudaSetDevice(dev), "cudaSetDevice");
  DeviceBuffers b(dev);
  void* din = b.alloc(in_bytes);
  void* dout = b.alloc(out_bytes);
  ck(cudaMemcpy(din, t.data, in_bytes, cudaMemcpyHostToDevice), "H2D");
  device_slice(ctx, gpu, DeviceTensorView{t.dtype, t.shape, din}, r, dout);
  ck(cudaMemcpy(out, dout, out_bytes, cudaMemcpyDeviceToHost), "D2H");
}

void host_merge(Context& ctx, int gpu, const std::vector<std::pair<Range, HostTensorView>>& parts, const Shape& target,
                void* out) {
  TraceRange trace_("host_merge");
  std::vector<MergePartSpec> spec;
  spec.reserve(parts.size());
  for (const auto& [r, p] : parts) spec.push_back({&r, p.dtype, &p.shape});
  validate_merge(spec, target);  // every reference error before any device work
  const uint64_t w = dtype_width(parts.front().second.dtype);
  const int dev = ctx.cuda_device(gpu);
  ck(cudaSetDevice(dev), "cudaSetDevice");
  DeviceBuffers b(dev);
  std::vector<std::pair<Range, DeviceTensorView>> dparts;
  dparts.reserve(parts.size());
  for (const auto& [r, p] : parts) {
    const uint64_t bytes = shape_elements(p.shape) * w;
    void* d = b.alloc(bytes);
    ck(cudaMemcpy(d, p.data, bytes, cudaMemcpyHostToDevice), "H2D");
    dparts.push_back({r, DeviceTensorView{p.dtype, p.shape, d}});
  }
  const uint64_t out_bytes = shape_elements(target) * w;
  void* dout = b.alloc(out_bytes);
  device_merge(ctx, gpu, dparts, target, dout);
  ck(cudaMemcpy(out, dout, out_bytes, cudaMemcpyDeviceToHost), "D2H");
}

Tensor slice(const Tensor& t, const Range& r) {
  r.check_against(t.shape());  // the reference's errors first, GPU or not
  std::vector<uint8_t> out(r.elements() * t.width());
  std::lock_guard<std::mutex> lock(g_mu);
  host_slice(default_context(), 0, HostTensorView{t.dtype(), t.shape(), t.payload().data()}, r, out.data());
  return Tensor(t.dtype(), r.extents(), std::move(out));
}

Tensor merge(const std::vector<std::pair<Range, Tensor>>& parts, const Shape& target_shape) {
  std::vector<MergePartSpec> spec;
  spec.reserve(parts.size());
  for (const auto& [r, p] : parts) spec.push_back({&r, p.dtype(), &p.shape()});
  validate_merge(spec, target_shape);
  std::vector<std::pair<Range, HostTensorView>> views;
  views.reserve(parts.size());
  for (const auto& [r, p] : parts) views.push_back({r, HostTensorView{p.dtype(), p.shape(), p.payload().data()}});
  const Dtype dt = parts.front().second.dtype();
  std::vector<uint8_t> out(shape_elements(target_shape) * dtype_width(dt));
  std::lock_guard<std::mutex> lock(g_mu);
  host_merge(default_context(), 0, views, target_shape, out.data());
  return Tensor(dt, target_shape, std::move(out));
}

}  // namespace reshard
