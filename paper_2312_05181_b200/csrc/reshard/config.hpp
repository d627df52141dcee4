// reshard/config.hpp — parallelization-configuration documents (
// PAPER.md:408 "processes these configurations as JSON objects"): the interchange format
// with model parallelizers (Megatron, Alpa).  Top level: a list ordered by rank; each rank
// object mirrors the model tree (path split at '/' and '.'); each leaf is
//   {"base": <tensor path>, "shape": [full extents], "range": [[lo, hi], ...] | null, "dtype": "f32"|...}
#pragma once

#include <string>
#include <vector>

#include "reshard/ptc.hpp"

namespace reshard {

// Rebuilds the PTC whose alpha∘phi hosts, on device r (devices[r], default (0, r)), exactly
// the sub-tensors rank r declares.  sigma(t) is the grid spanned by the declared ranges.
// Errors: MalformedConfig (syntax, missing fields, unknown dtype), InconsistentBaseShape
// (ranks disagree on a base tensor's shape or dtype), CoverageGap (the declared ranges of a
// tensor do not tile it as a grid: overlap, gap or non-grid rectangles).
PTC parse_parallel_config(const std::string& json, const std::vector<DeviceId>& devices = {});

// The document of a PTC (inverse of parse_parallel_config up to partition numbering).
std::string serialize_parallel_config(const PTC& ptc);

}  // namespace reshard
