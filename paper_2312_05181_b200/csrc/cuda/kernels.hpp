// Host-visible launchers for the sm_100a kernels in kernels.cu.  Plain C++ declarations so
// the host C++ (compiled by g++) never includes CUDA device code.
#pragma once

#include <cstdint>
#include <vector>

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

// K1/K2 (LDG/STG, 16-byte vectors) or K3 (TMA bulk pipeline): persistent tile copy over a
// tile list.  aligned16: every tile is 16-byte aligned (else the generic-width kernel runs).
// claim: a zeroed 2 x u64 counter for dynamic tile claims (used when cfg.ldg_dyn; the aligned
// kernel only), else the static grid-stride order.
void launch_copy(const CopyTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, bool aligned16,
                 void* stream, unsigned long long* claim = nullptr);
// K2 fan-out (LDG/STG): every tile 16-byte aligned, n_dst <= kMaxFan destinations, natural
// order; the source is read once for all destinations (peer destinations store over NVLink).
void launch_copy_fan(const FanTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, void* stream,
                     unsigned long long* claim = nullptr);
// K3 with fan-out: every tile 16-byte aligned and <= cfg.stage_bytes.  The array must be in
// interleave_for_grid order for bulk_grid(n_tiles, sms, cfg) CTAs.
// bulk_dyn (cfg.kernel == BulkDyn) claims tiles from `claim` (2 x u64, zero before the first
// launch; the kernel leaves it zero again), required for that kernel only.
void launch_bulk(const FanTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, void* stream,
                 unsigned long long* claim = nullptr);
inline int bulk_grid(uint64_t n_tiles, int sms, const CopyConfig& cfg) {
  const uint64_t g = uint64_t(sms) * uint64_t(cfg.ctas_per_sm > 0 ? cfg.ctas_per_sm : 1);
  return int(n_tiles < g ? n_tiles : g);
}
// Reorder tiles so that CTA c of a `grid`-CTA launch finds original tiles c, c+grid, ... as
// one contiguous run (the bulk kernel fetches its descriptors in contiguous batches).
template <class T>
std::vector<T> interleave_for_grid(const T* tiles, size_t n, size_t grid) {
  std::vector<T> out;
  out.reserve(n);
  for (size_t c = 0; c < grid; ++c)
    for (size_t i = c; i < n; i += grid) out.push_back(tiles[i]);
  return out;
}
// Expand pieces (device array, `first` = tile prefix) into tiles: tiles [t0, t1) of the
// concatenated schedule go to out[0 .. t1-t0), in natural order (grid == 0) or in
// interleave_for_grid order for a `grid`-CTA bulk launch.  FanTile for the bulk kernel;
// CopyTile (n_dst == 1 pieces) for the LDG/STG kernels.
void launch_expand_fan(const DevPiece* d_pieces, uint32_t n_pieces, uint64_t t0, uint64_t t1, FanTile* out,
                       unsigned grid, int sms, void* stream);
void launch_expand_copy(const DevPiece* d_pieces, uint32_t n_pieces, uint64_t n_tiles, CopyTile* out, int sms,
                        void* stream);
// K6 / K7 over a batch of cells (device array of tasks): write the splitmix64 payload, or
// count the bytes that differ from it into *d_count (atomic add).  One launch per 65535 cells.
struct PayloadTask {
  void* data;
  uint64_t seed;
  CellGeom g;
};
void launch_payload(const PayloadTask* d_tasks, uint64_t n_tasks, uint64_t max_bytes, bool verify,
                    unsigned long long* d_count, void* stream);

// Fill a CellGeom from a base shape and a cell box.
CellGeom make_geom(const Shape& base, size_t width, const Range& cell);

}  // namespace reshard::cuda
