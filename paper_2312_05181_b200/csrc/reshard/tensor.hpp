// reshard/tensor.hpp — the reference's host value type and its two data operations, as a
// drop-in: the same class and free functions as proj/include/reshard/tensor/tensor.hpp:16-47
// (Tensor(Dtype, Shape, payload), Tensor::zeros, slice, merge), the same validation order and
// error codes (tensor.cpp:9-17, 61-114), values immutable after construction.  The bytes move
// on the GPU: slice / merge validate on the host exactly as the reference does, then stage the
// payload(s) to the device, run the tile-copy kernel (device_slice / device_merge) and read the
// result back.  They run on a process-wide context (cuda:0 unless set_default_device chose
// another device); without a GPU they fail with Errc::DeviceUnavailable after validation —
// there is no CPU path.  Calls are serialised on that context, so concurrent callers stay
// correct (the reference's functions are pure and lock-free).
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "reshard/core.hpp"

namespace reshard {

class Tensor {
 public:
  Tensor(Dtype dtype, Shape shape, std::vector<uint8_t> payload);
  static Tensor zeros(Dtype dtype, Shape shape);

  Dtype dtype() const { return dtype_; }
  const Shape& shape() const { return shape_; }
  size_t rank() const { return shape_.size(); }
  uint64_t elements() const { return shape_elements(shape_); }
  size_t width() const { return dtype_width(dtype_); }
  const std::vector<uint8_t>& payload() const { return payload_; }
  std::span<const uint8_t> bytes() const { return payload_; }
  bool operator==(const Tensor& other) const = default;

 private:
  Dtype dtype_;
  Shape shape_;
  std::vector<uint8_t> payload_;
};

// The element at output index v equals the input element at v + r.lo (tensor.hpp:40-42).
Tensor slice(const Tensor& t, const Range& r);
// Reassemble `target_shape` from parts that tile it exactly (tensor.hpp:44-47); TilingGap /
// TilingOverlap / DtypeMismatch / ShapeMismatch in the reference's order.
Tensor merge(const std::vector<std::pair<Range, Tensor>>& parts, const Shape& target_shape);

// The CUDA device the host-value operations run on (default 0).  Takes effect before the
// first slice / merge of the process.
void set_default_device(int cuda_device);

// Host-buffer forms used by the C ABI (rs_slice_host / rs_merge_host): the same validation,
// then staging through the given context's GPU.  `out` receives r.elements() * width bytes.
struct HostTensorView {
  Dtype dtype;
  Shape shape;
  const void* data;
};
class Context;
void host_slice(Context& ctx, int gpu, const HostTensorView& t, const Range& r, void* out);
void host_merge(Context& ctx, int gpu, const std::vector<std::pair<Range, HostTensorView>>& parts,
                const Shape& target_shape, void* out);

}  // namespace reshard
