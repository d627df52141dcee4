// Reconfiguration plan generation — Algorithm 1.
//
//   SPLIT  for r in R, v hosted on r:        split(v, sigma, sigma')  -> refined fragments
//   MOVE   for r' in R', cell c hosted on r': for w in W(c) not resident on r':
//                                             move(w, choose_source(holders(w)), r')
//   MERGE  merge(W(c)) when |W(c)| > 1       (single full-cell merge elided)
//
// Each tensor's common refinement G = grid_refine(sigma(t), sigma'(t)) is computed once;
// every G cell knows its source and destination cell index by per-dim binary search, so
// the planner is O(#fragments) rather than the O(cells^2) containment scans of a literal
// reading.  Op order (hence choose_source's egress accounting) follows Alg. 1 exactly.
#include <algorithm>
#include <numeric>
#include <sstream>

#include "reshard/planner.hpp"
#include "reshard/trace.hpp"

namespace reshard {

namespace {

// Lexicographic cell index (last dim fastest) of the cell of `g` holding box `b`.
uint32_t cell_index(const SplitGrid& g, const Range& b) {
  uint64_t idx = 0;
  for (size_t d = 0; d < g.rank(); ++d)
    idx = idx * (g.points()[d].size() + 1) + g.interval_of(d, b.dim(int(d)).lo);
  return uint32_t(idx);
}

struct TensorGeometry {
  std::vector<Range> frags;             // G cells, lexicographic
  std::vector<uint32_t> src_cell;       // per G cell: sigma cell index
  std::vector<std::vector<uint32_t>> by_src;  // sigma cell -> G cells (lex order)
  std::vector<std::vector<uint32_t>> by_dst;  // sigma' cell -> G cells (lex order)
};

std::shared_ptr<const ReconfigPlan> plan_impl(std::shared_ptr<const PTC> from, std::shared_ptr<const PTC> to,
                                              const std::vector<DeviceId>& failed) {
  const PTC& a = *from;
  const PTC& b = *to;
  if (a.catalog.tensors.size() != b.catalog.tensors.size())
    raise(Errc::CatalogMismatch, "catalog sizes differ");
  for (size_t t = 0; t < a.catalog.tensors.size(); ++t) {
    const auto &x = a.catalog.tensors[t], &y = b.catalog.tensors[t];
    if (x.path != y.path || x.dtype != y.dtype || x.shape != y.shape) raise(Errc::CatalogMismatch, x.path);
  }
  auto plan = std::make_shared<ReconfigPlan>();
  plan->from = from, plan->to = to, plan->failed = failed;

  const size_t nt = a.catalog.tensors.size();
  std::vector<TensorGeometry> geo(nt);
  for (size_t t = 0; t < nt; ++t) {
    const Shape& shape = a.catalog.tensors[t].shape;
    plan->refine.push_back(grid_refine(a.sigma[t], b.sigma[t]));
    TensorGeometry& g = geo[t];
    g.frags = plan->refine.back().cells(shape);
    g.by_src.resize(a.cells[t].size());
    g.by_dst.resize(b.cells[t].size());
    for (uint32_t k = 0; k < g.frags.size(); ++k) {
      uint32_t s = cell_index(a.sigma[t], g.frags[k]), d = cell_index(b.sigma[t], g.frags[k]);
      g.src_cell.push_back(s);
      g.by_src[s].push_back(k);
      g.by_dst[d].push_back(k);
    }
  }

  std::vector<char> dead(a.devices.size(), 0);
  for (auto& f : failed) {
    int o = a.ordinal(f);
    if (o >= 0) dead[size_t(o)] = 1;
  }
  std::vector<int> b_to_a(b.devices.size());
  for (size_t i = 0; i < b.devices.size(); ++i) b_to_a[i] = a.ordinal(b.devices[i]);

  std::vector<PlanOp> splits, moves, merges;
  for (uint32_t r = 0; r < a.devices.size(); ++r) {
    if (dead[r]) continue;
    for (uint32_t t = 0; t < nt; ++t)
      for (uint32_t v = 0; v < a.cells[t].size(); ++v) {
        if (!a.hosts(t, v, r) || geo[t].by_src[v].size() < 2) continue;
        PlanOp op{PlanOp::Kind::Split, t, a.devices[r], a.devices[r], a.cells[t][v], {}, 0};
        for (uint32_t k : geo[t].by_src[v]) op.parts.push_back(geo[t].frags[k]);
        splits.push_back(std::move(op));
      }
  }

  std::vector<uint64_t> egress(a.devices.size(), 0);
  std::vector<uint32_t> cand;
  for (uint32_t r2 = 0; r2 < b.devices.size(); ++r2) {
    const DeviceId& dst = b.devices[r2];
    const int here = b_to_a[r2];
    for (uint32_t t = 0; t < nt; ++t) {
      const uint64_t width = dtype_width(a.catalog.tensors[t].dtype);
      for (uint32_t c = 0; c < b.cells[t].size(); ++c) {
        if (!b.hosts(t, c, r2)) continue;
        PlanDstCell cell{r2, t, c, uint32_t(plan->fragments.size()), 0, false};
        for (uint32_t k : geo[t].by_dst[c]) {
          const Range& w = geo[t].frags[k];
          const uint32_t v = geo[t].src_cell[k];
          if (here >= 0 && !dead[size_t(here)] && a.hosts(t, v, uint32_t(here))) {
            plan->fragments.push_back({w, v, uint32_t(here), true});
            continue;
          }
          cand.clear();
          for (uint32_t o : a.alpha[a.phi[t][v]])
            if (!dead[o]) cand.push_back(o);
          if (cand.empty())
            raise(failed.empty() ? Errc::UnsatisfiableFragment : Errc::CheckpointRequired,
                  a.catalog.tensors[t].path + " " + w.to_string() + " survives on no device");
          // choose_source: same-worker candidates first, then least egress, then smallest id
          bool any_same = std::any_of(cand.begin(), cand.end(), [&](uint32_t o) { return a.devices[o].worker == dst.worker; });
          uint32_t best = UINT32_MAX;
          for (uint32_t o : cand) {
            if (any_same && a.devices[o].worker != dst.worker) continue;
            if (best == UINT32_MAX || egress[o] < egress[best] || (egress[o] == egress[best] && a.devices[o] < a.devices[best]))
              best = o;
          }
          const uint64_t bytes = w.elements() * width;
          egress[best] += bytes;
          moves.push_back(PlanOp{PlanOp::Kind::Move, t, a.devices[best], dst, w, {}, bytes});
          plan->fragments.push_back({w, v, best, false});
        }
        cell.count = uint32_t(plan->fragments.size()) - cell.first;
        if (cell.count == 1) {
          const PlanFragment& f = plan->fragments[cell.first];
          cell.kept = f.resident && f.box == a.cells[t][f.src_cell] && f.box == b.cells[t][c];
        } else {
          PlanOp op{PlanOp::Kind::Merge, t, dst, dst, b.cells[t][c], {}, 0};
          for (uint32_t k : geo[t].by_dst[c]) op.parts.push_back(geo[t].frags[k]);
          merges.push_back(std::move(op));
        }
        plan->dst_cells.push_back(cell);
      }
    }
  }
  plan->ops.reserve(splits.size() + moves.size() + merges.size());
  for (auto* v : {&splits, &moves, &merges})
    for (auto& op : *v) plan->ops.push_back(std::move(op));
  plan->split_end = splits.size();
  plan->move_end = splits.size() + moves.size();
  return plan;
}

}  // namespace

std::shared_ptr<const ReconfigPlan> generate_plan(std::shared_ptr<const PTC> from, std::shared_ptr<const PTC> to) {
  TraceRange trace_("reshard::generate_plan");
  return plan_impl(std::move(from), std::move(to), {});
}

std::shared_ptr<const ReconfigPlan> recover(std::shared_ptr<const PTC> from, const std::vector<DeviceId>& failed,
                                            std::shared_ptr<const PTC> to) {
  for (auto& f : failed)
    if (from->ordinal(f) < 0) raise(Errc::UnknownDevice, "failed device " + f.to_string() + " not in the layout");
  // the target layout must leave the failed devices out (a Move into a dead device is a bug)
  for (auto& f : failed)
    if (to->ordinal(f) >= 0)
      raise(Errc::InvalidArgument, "failed device " + f.to_string() + " is part of the target layout");
  return plan_impl(std::move(from), std::move(to), failed);
}

DeviceId choose_source(const std::vector<DeviceId>& cand, const DeviceId& dst, const std::map<DeviceId, uint64_t>& egress) {
  if (cand.empty()) raise(Errc::NoSource, "no candidate for " + dst.to_string());
  if (std::find(cand.begin(), cand.end(), dst) != cand.end()) return dst;
  bool any_same = std::any_of(cand.begin(), cand.end(), [&](const DeviceId& d) { return d.worker == dst.worker; });
  auto eg = [&](const DeviceId& d) {
    auto it = egress.find(d);
    return it == egress.end() ? uint64_t(0) : it->second;
  };
  const DeviceId* best = nullptr;
  for (auto& c : cand) {
    if (any_same && c.worker != dst.worker) continue;
    if (!best || eg(c) < eg(*best) || (eg(c) == eg(*best) && c < *best)) best = &c;
  }
  return *best;
}

PlanCost plan_cost(const ReconfigPlan& p) {
  PlanCost c;
  c.devices = p.from->devices;
  c.devices.insert(c.devices.end(), p.to->devices.begin(), p.to->devices.end());
  std::sort(c.devices.begin(), c.devices.end());
  c.devices.erase(std::unique(c.devices.begin(), c.devices.end()), c.devices.end());
  c.ingress.assign(c.devices.size(), 0);
  c.egress.assign(c.devices.size(), 0);
  auto at = [&](const DeviceId& d) { return size_t(std::lower_bound(c.devices.begin(), c.devices.end(), d) - c.devices.begin()); };
  for (size_t i = p.split_end; i < p.move_end; ++i) {
    const PlanOp& op = p.ops[i];
    c.ingress[at(op.dst)] += op.bytes;
    c.egress[at(op.dev)] += op.bytes;
    c.total += op.bytes;
  }
  return c;
}

PlanCost plan_cost_central(const ReconfigPlan& p, const DeviceId& central) {
  PlanCost c = plan_cost(p);  // device set (sorted union)
  if (!std::binary_search(c.devices.begin(), c.devices.end(), central)) {
    c.devices.insert(std::lower_bound(c.devices.begin(), c.devices.end(), central), central);
  }
  c.ingress.assign(c.devices.size(), 0);
  c.egress.assign(c.devices.size(), 0);
  c.total = 0;
  auto at = [&](const DeviceId& d) { return size_t(std::lower_bound(c.devices.begin(), c.devices.end(), d) - c.devices.begin()); };
  auto leg = [&](const DeviceId& from, const DeviceId& to, uint64_t b) {
    if (from == to) return;
    c.egress[at(from)] += b;
    c.ingress[at(to)] += b;
    c.total += b;
  };
  for (size_t i = p.split_end; i < p.move_end; ++i) {
    const PlanOp& op = p.ops[i];
    leg(op.dev, central, op.bytes);
    leg(central, op.dst, op.bytes);
  }
  return c;
}

PlanStats plan_stats(const ReconfigPlan& p) {
  PlanStats s;
  s.n_split = p.n_split(), s.n_move = p.n_move(), s.n_merge = p.n_merge();
  for (size_t i = p.split_end; i < p.move_end; ++i) s.moved_bytes += p.ops[i].bytes;
  for (auto& c : p.dst_cells) {
    const uint64_t w = dtype_width(p.to->catalog.tensors[c.tensor].dtype);
    s.dst_bytes += p.to->cells[c.tensor][c.cell].elements() * w;
    for (uint32_t k = c.first; k < c.first + c.count; ++k) {
      const PlanFragment& f = p.fragments[k];
      if (!f.resident) continue;
      (c.kept ? s.kept_bytes : s.relayout_bytes) += f.box.elements() * w;
    }
  }
  return s;
}

std::string plan_text(const ReconfigPlan& p) {
  std::string out;
  auto join = [&](const std::vector<Range>& v) {
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) out.push_back(';');
      out += v[i].to_string();
    }
  };
  for (const PlanOp& op : p.ops) {
    const std::string& path = p.from->catalog.tensors[op.tensor].path;
    switch (op.kind) {
      case PlanOp::Kind::Split:
        out += "SPLIT dev=" + op.dev.to_string() + " t=" + path + " r=" + op.range.to_string() + " -> ";
        join(op.parts);
        break;
      case PlanOp::Kind::Move:
        out += "MOVE t=" + path + " r=" + op.range.to_string() + " " + op.dev.to_string() + " -> " +
               op.dst.to_string() + " bytes=" + std::to_string(op.bytes);
        break;
      case PlanOp::Kind::Merge:
        out += "MERGE dev=" + op.dev.to_string() + " t=" + path + " ";
        join(op.parts);
        out += " -> " + op.range.to_string();
        break;
    }
    out.push_back('\n');
  }
  return out;
}

}  // namespace reshard
