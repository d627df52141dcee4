// Host-visible launchers for the sm_100a kernels in kernels.cu.  Plain C++ declarations so
// the host C++ (compiled by g++) never includes CUDA device code.
#pragma once

#include <cstdint>

#include "reshard/executor.hpp"

namespace reshard::cuda {

// Geometry of one cell of a base tensor for the synthetic payload (K6) and its check (K7).
struct CellGeom {
  uint64_t bytes;          // cell bytes
  uint64_t run_bytes;      // innermost extent * width
  uint64_t lo[kMaxRank];   // cell origin in the base tensor
  uint64_t ext[kMaxRank];  // cell extents
  uint64_t stride[kMaxRank];  // base tensor row-major strides in BYTES
  uint32_t rank, width;
};

// K1/K2: persistent tile copy.  `grid` CTAs of `block` threads walk the tile list.
void launch_copy_tiles(const CopyTile* d_tiles, uint64_t n_tiles, int grid, int block, void* stream);
// K6: write the splitmix64 payload of `g` at dst.
void launch_fill(void* dst, uint64_t seed, const CellGeom& g, void* stream);
// K7: count bytes of `data` that differ from the payload of `g` into *d_count (atomic add).
void launch_verify(const void* data, uint64_t seed, const CellGeom& g, unsigned long long* d_count, void* stream);

// Fill a CellGeom from a base shape and a cell box.
CellGeom make_geom(const Shape& base, size_t width, const Range& cell);

}  // namespace reshard::cuda
