// reshard/ptc.hpp — the parallelizable tensor collection PTC = (T, sigma, phi, alpha)
// (Eq. 1) and its builders, per the SPEC parallel-config module
// (SPEC.md:111-199).  No reference code exists for this layer; semantics pinned in DESIGN.md.
#pragma once

#include <compare>
#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "reshard/core.hpp"

namespace reshard {

// DeviceId: worker index, local device index; ordered worker-major.
struct DeviceId {
  uint32_t worker = 0;
  uint32_t local = 0;
  auto operator<=>(const DeviceId&) const = default;
  std::string to_string() const { return std::to_string(worker) + ":" + std::to_string(local); }
};

constexpr int kLayerPre = -1;   // embeddings: first pipeline stage
constexpr int kLayerPost = -2;  // final layernorm: last pipeline stage

// One base tensor of the catalog T.  tp_dim < 0: replicated under TP (sigma = identity).
struct TensorSpec {
  std::string path;
  Dtype dtype = Dtype::F32;
  Shape shape;
  int tp_dim = -1;
  int layer = 0;
};

enum class StateKind : int {
  Fp32Adam = 0,   // fp32 param + exp_avg + exp_avg_sq                     (12 B/param)
  MixedAdam = 1,  // bf16 param + fp32 master + exp_avg + exp_avg_sq       (14 B/param)
  Fp32Param = 2,  // fp32 param only
};

struct Catalog {
  std::vector<TensorSpec> tensors;
  void add(TensorSpec t);
  // Megatron GPT naming: per state, word/position embeddings, L layers x 12
  // tensors, final layernorm; param-major with the optimizer states of a param adjacent.
  static Catalog gpt(uint64_t hidden, uint64_t layers, uint64_t seq, uint64_t vocab, StateKind kind);
  uint64_t total_bytes() const;
};

struct JobConfig {
  int tp = 1, pp = 1, dp = 1;
};

// PTC.  Partitions: (stage s, tp rank j) -> s*T + j for TP-sliced cells; the replicated
// tensors of stage s -> P*T + s.  alpha holds device ordinals into `devices`.
struct PTC {
  Catalog catalog;
  std::vector<DeviceId> devices;  // (dp, pp, tp) = devices[dp*P*T + pp*T + tp]
  JobConfig job;
  std::vector<int> stage;                       // per tensor
  std::vector<SplitGrid> sigma;                 // per tensor
  std::vector<std::vector<Range>> cells;        // sigma cells per tensor (cached)
  std::vector<std::vector<uint32_t>> phi;       // [tensor][cell] -> partition
  std::vector<std::vector<uint32_t>> alpha;     // [partition] -> device ordinals

  int ordinal(const DeviceId& d) const;         // -1 when d is not in this PTC
  bool hosts(uint32_t t, uint32_t cell, uint32_t dev_ordinal) const;
};

PTC build_strategy(const Catalog& catalog, const std::vector<DeviceId>& devices, const JobConfig& job);

// (tensor, cell index) hosted by `dev`, in (tensor, cell) order.  UnknownDevice.
std::vector<std::pair<uint32_t, uint32_t>> hosted_subtensors(const PTC& ptc, const DeviceId& dev);

// Violations as "<Kind>: <detail>" lines; empty iff the PTC is well formed.
std::vector<std::string> validate(const PTC& ptc);

}  // namespace reshard
