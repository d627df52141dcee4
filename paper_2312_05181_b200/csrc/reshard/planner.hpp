// reshard/planner.hpp — reconfiguration plan generation, Algorithm 1 as
// specified by the SPEC planner module.  Besides the Split/Move/Merge op
// list (text format SPEC.md:268), the plan records for every destination cell the refined
// fragments and where each is read from; the executor lowers that to device copy tiles.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "reshard/ptc.hpp"

namespace reshard {

struct PlanOp {
  enum class Kind : uint8_t { Split, Move, Merge };
  Kind kind;
  uint32_t tensor;
  DeviceId dev;              // Split/Merge: acting device; Move: source
  DeviceId dst;              // Move: destination
  Range range;               // Split: source cell; Move: fragment; Merge: merged cell
  std::vector<Range> parts;  // Split: fragments; Merge: parts
  uint64_t bytes = 0;        // Move: elements(range) * width
};

// One refined fragment of a destination cell and the source cell it is read from.
struct PlanFragment {
  Range box;             // absolute base-tensor coordinates
  uint32_t src_cell;     // sigma cell index in `from`
  uint32_t src_device;   // ordinal in from->devices (== destination for resident fragments)
  bool resident;         // read on the destination itself (no Move)
};

// One cell hosted by a destination device in `to`.
struct PlanDstCell {
  uint32_t dst_device;   // ordinal in to->devices
  uint32_t tensor;
  uint32_t cell;         // sigma' cell index
  uint32_t first, count; // fragments [first, first+count) in ReconfigPlan::fragments
  bool kept;             // one resident fragment equal to both cells: no byte moves
};

struct ReconfigPlan {
  std::shared_ptr<const PTC> from, to;
  std::vector<DeviceId> failed;
  std::vector<SplitGrid> refine;       // grid_refine(sigma(t), sigma'(t)) per tensor
  std::vector<PlanOp> ops;             // [0, split_end) splits, [split_end, move_end) moves, rest merges
  size_t split_end = 0, move_end = 0;
  std::vector<PlanDstCell> dst_cells;  // Alg. 1 destination order
  std::vector<PlanFragment> fragments;

  size_t n_split() const { return split_end; }
  size_t n_move() const { return move_end - split_end; }
  size_t n_merge() const { return ops.size() - move_end; }
};

struct PlanStats {
  uint64_t n_split = 0, n_move = 0, n_merge = 0;
  uint64_t moved_bytes = 0;     // sum of Move bytes (cross-device)
  uint64_t relayout_bytes = 0;  // resident fragments copied into a re-shaped cell
  uint64_t kept_bytes = 0;      // resident cells reused as is
  uint64_t dst_bytes = 0;       // all destination cells
};

std::shared_ptr<const ReconfigPlan> generate_plan(std::shared_ptr<const PTC> from, std::shared_ptr<const PTC> to);
// recover: plan with `failed` excluded from every candidate set;
// CheckpointRequired when some needed fragment survives nowhere.
std::shared_ptr<const ReconfigPlan> recover(std::shared_ptr<const PTC> from, const std::vector<DeviceId>& failed,
                                            std::shared_ptr<const PTC> to);

// choose_source: dst if resident; else same-worker candidates if any;
// least accumulated egress; ties by smallest device id.
DeviceId choose_source(const std::vector<DeviceId>& candidates, const DeviceId& dst,
                       const std::map<DeviceId, uint64_t>& egress);

struct PlanCost {
  std::vector<DeviceId> devices;  // union of both PTCs, sorted
  std::vector<uint64_t> ingress, egress;
  uint64_t total = 0;
};
PlanCost plan_cost(const ReconfigPlan& plan);
// Traffic attribution of apply_plan's central mode (the paper's baseline,
// PAPER.md:523-527): every moved fragment is fetched by `central` and re-uploaded from it,
// so it is charged src -> central and central -> dst (legs that start and end on `central`
// cost nothing).  Same final state as the distributed mode.
PlanCost plan_cost_central(const ReconfigPlan& plan, const DeviceId& central);
PlanStats plan_stats(const ReconfigPlan& plan);
std::string plan_text(const ReconfigPlan& plan);

}  // namespace reshard
