// PTC builders.  Pinned choices:
//  * layers 0..L-1 split into P contiguous stages, balanced within one layer, remainder to
//    the earliest stages; kLayerPre -> stage 0, kLayerPost -> stage P-1;
//  * TP-replicated tensors (LN, row-parallel biases, position embeddings) keep sigma =
//    identity and are allocated to every tp rank of their stage;
//  * device (dp, pp, tp) = devices[dp*P*T + pp*T + tp].
#include <algorithm>
#include <set>

#include "reshard/ptc.hpp"

namespace reshard {

void Catalog::add(TensorSpec t) {
  dtype_width(t.dtype);
  if (t.shape.size() > size_t(kMaxRank)) raise(Errc::RankMismatch, t.path + ": rank above 8");
  for (auto e : t.shape)
    if (e == 0) raise(Errc::InvalidTensor, t.path + ": zero extent");
  tensors.push_back(std::move(t));
}

uint64_t Catalog::total_bytes() const {
  uint64_t n = 0;
  for (auto& t : tensors) n += shape_elements(t.shape) * dtype_width(t.dtype);
  return n;
}

Catalog Catalog::gpt(uint64_t h, uint64_t L, uint64_t S, uint64_t V, StateKind kind) {
  struct Param {
    std::string name;
    Shape shape;
    int tp_dim, layer;
  };
  std::vector<Param> params = {{"embedding.word_embeddings.weight", {V, h}, 0, kLayerPre},
                               {"embedding.position_embeddings.weight", {S, h}, -1, kLayerPre}};
  static const struct {
    const char* name;
    int rows, cols;  // multiples of h; cols == 0 -> rank-1
    int tp_dim;
  } kLayer[] = {{"input_layernorm.weight", 1, 0, -1},
                {"input_layernorm.bias", 1, 0, -1},
                {"self_attention.query_key_value.weight", 3, 1, 0},
                {"self_attention.query_key_value.bias", 3, 0, 0},
                {"self_attention.dense.weight", 1, 1, 1},
                {"self_attention.dense.bias", 1, 0, -1},
                {"post_attention_layernorm.weight", 1, 0, -1},
                {"post_attention_layernorm.bias", 1, 0, -1},
                {"mlp.dense_h_to_4h.weight", 4, 1, 0},
                {"mlp.dense_h_to_4h.bias", 4, 0, 0},
                {"mlp.dense_4h_to_h.weight", 1, 4, 1},
                {"mlp.dense_4h_to_h.bias", 1, 0, -1}};
  for (uint64_t l = 0; l < L; ++l)
    for (auto& p : kLayer) {
      Shape s = p.cols ? Shape{p.rows * h, p.cols * h} : Shape{p.rows * h};
      params.push_back({"layers." + std::to_string(l) + "." + p.name, s, p.tp_dim, int(l)});
    }
  params.push_back({"final_layernorm.weight", {h}, -1, kLayerPost});
  params.push_back({"final_layernorm.bias", {h}, -1, kLayerPost});

  std::vector<std::pair<const char*, Dtype>> states;
  switch (kind) {
    case StateKind::Fp32Adam: states = {{"param", Dtype::F32}, {"exp_avg", Dtype::F32}, {"exp_avg_sq", Dtype::F32}}; break;
    case StateKind::MixedAdam:
      states = {{"param", Dtype::BF16}, {"master", Dtype::F32}, {"exp_avg", Dtype::F32}, {"exp_avg_sq", Dtype::F32}};
      break;
    case StateKind::Fp32Param: states = {{"param", Dtype::F32}}; break;
  }
  Catalog c;
  for (auto& p : params)
    for (auto& [sname, dt] : states) c.add({std::string(sname) + "/" + p.name, dt, p.shape, p.tp_dim, p.layer});
  return c;
}

int PTC::ordinal(const DeviceId& d) const {
  auto it = std::find(devices.begin(), devices.end(), d);
  return it == devices.end() ? -1 : int(it - devices.begin());
}

bool PTC::hosts(uint32_t t, uint32_t cell, uint32_t dev) const {
  const auto& a = alpha[phi[t][cell]];
  return std::find(a.begin(), a.end(), dev) != a.end();
}

PTC build_strategy(const Catalog& catalog, const std::vector<DeviceId>& devices, const JobConfig& job) {
  const int T = job.tp, P = job.pp, D = job.dp;
  if (T < 1 || P < 1 || D < 1) raise(Errc::InvalidJobConfig, "tp/pp/dp degrees must be positive");
  if (devices.size() != size_t(T) * size_t(P) * size_t(D))
    raise(Errc::DeviceCountMismatch, std::to_string(devices.size()) + " devices for T*P*D = " + std::to_string(T * P * D));
  PTC p;
  p.catalog = catalog;
  p.devices = devices;
  p.job = job;

  // stage of every tensor
  int L = 0;
  for (auto& t : catalog.tensors) L = std::max(L, t.layer + 1);
  if (P > 1 && L < P)
    raise(Errc::IndivisibleLayerCount, std::to_string(L) + " layers cannot fill " + std::to_string(P) + " stages");
  std::vector<int> layer_stage(size_t(std::max(L, 0)));
  for (int l = 0, s = 0, left = 0; l < L; ++l) {
    if (left == 0) left = L / P + (s < L % P ? 1 : 0), ++s;
    layer_stage[size_t(l)] = s - 1;
    --left;
  }
  for (auto& t : catalog.tensors)
    p.stage.push_back(t.layer == kLayerPre ? 0 : t.layer == kLayerPost ? P - 1 : layer_stage[size_t(t.layer)]);

  // alpha
  auto dev = [&](int d, int s, int j) { return uint32_t(size_t(d) * P * T + size_t(s) * T + size_t(j)); };
  p.alpha.resize(size_t(P) * T + P);
  for (int s = 0; s < P; ++s)
    for (int j = 0; j < T; ++j)
      for (int d = 0; d < D; ++d) p.alpha[size_t(s) * T + j].push_back(dev(d, s, j));
  for (int s = 0; s < P; ++s)
    for (int d = 0; d < D; ++d)
      for (int j = 0; j < T; ++j) p.alpha[size_t(P) * T + s].push_back(dev(d, s, j));

  // sigma, cells, phi
  for (size_t t = 0; t < catalog.tensors.size(); ++t) {
    const TensorSpec& e = catalog.tensors[t];
    SplitGrid g = e.tp_dim >= 0 ? SplitGrid::even_split(e.shape, size_t(e.tp_dim), uint64_t(T))
                                : SplitGrid::identity(e.shape.size());
    p.cells.push_back(g.cells(e.shape));
    std::vector<uint32_t> ph(p.cells.back().size());
    for (size_t i = 0; i < ph.size(); ++i)
      ph[i] = e.tp_dim >= 0 ? uint32_t(p.stage[t] * T + int(i)) : uint32_t(P * T + p.stage[t]);
    p.sigma.push_back(std::move(g));
    p.phi.push_back(std::move(ph));
  }
  return p;
}

std::vector<std::pair<uint32_t, uint32_t>> hosted_subtensors(const PTC& p, const DeviceId& d) {
  int o = p.ordinal(d);
  if (o < 0) raise(Errc::UnknownDevice, d.to_string());
  std::vector<std::pair<uint32_t, uint32_t>> out;
  for (uint32_t t = 0; t < p.phi.size(); ++t)
    for (uint32_t c = 0; c < p.phi[t].size(); ++c)
      if (p.hosts(t, c, uint32_t(o))) out.emplace_back(t, c);
  return out;
}

std::vector<std::string> validate(const PTC& p) {
  std::vector<std::string> v;
  std::set<uint32_t> used;
  for (size_t t = 0; t < p.catalog.tensors.size(); ++t) {
    const auto& e = p.catalog.tensors[t];
    if (t >= p.sigma.size() || t >= p.phi.size()) {
      v.push_back("MissingSigma: " + e.path);
      continue;
    }
    try {
      p.sigma[t].check_against(e.shape);
    } catch (const Error&) {
      v.push_back("InvalidSplitPoint: " + e.path);
      continue;
    }
    if (p.phi[t].size() != p.sigma[t].cell_count()) v.push_back("UnmappedSubtensor: " + e.path);
    for (uint32_t part : p.phi[t]) {
      if (part >= p.alpha.size()) v.push_back("UnmappedSubtensor: " + e.path);
      else used.insert(part);
    }
  }
  for (uint32_t part : used) {
    if (p.alpha[part].empty()) v.push_back("UnhostedPartition: " + std::to_string(part));
    for (uint32_t d : p.alpha[part])
      if (d >= p.devices.size()) v.push_back("UnknownDevice: ordinal " + std::to_string(d));
  }
  return v;
}

}  // namespace reshard
