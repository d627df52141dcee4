// reshard/executor.hpp — the B200 State Transformer: executes a ReconfigPlan as device copy
// tiles.  Replaces the SPEC executor's apply_plan, whose data
// plane is the reference's slice()/merge() row walker (proj/src/tensor/tensor.cpp:35-114).
//
// Layout in HBM: every GPU of the world owns two arenas.
//   src arena: the cells of `from` hosted by the logical devices mapped to the GPU, in
//              (device, tensor, cell) order, each 256-byte aligned;
//   dst arena: the cells of `to` that are NOT kept (a kept cell is a resident cell whose
//              range does not change; it stays where it is in the src arena).
// Every refined fragment becomes one strided 2-D copy (rows x row_bytes, two pitches)
// from its source cell into its final offset of the destination cell, i.e. split, move
// and merge are fused into a single write; no staging, no merge pass.  The host lowers
// each copy to a few pieces (DevPiece); prepare() uploads them and the GPU expands them into
// shared-memory-stage-sized tiles, executed by one persistent kernel per source GPU (push:
// a cross-GPU tile stores straight into the peer's dst arena over NVLink).
#pragma once

#include <cstdint>
#include <memory>
#include <unordered_map>
#include <vector>

#include "reshard/planner.hpp"

namespace reshard {

namespace cuda {
struct PayloadTask;
}

// Must match the device struct in cuda/kernels.cuh.
struct CopyTile {
  uint64_t src, dst;              // absolute device addresses (dst may be a peer mapping)
  uint64_t src_pitch, dst_pitch;  // bytes between consecutive rows
  uint32_t rows, row_bytes;
};
static_assert(sizeof(CopyTile) == 40, "CopyTile layout");

// Bulk (TMA) kernel tile: one source box, up to kMaxFan destinations with the same row
// structure (DP replicas of one fragment are read once, stored n_dst times).
constexpr int kMaxFan = 4;
struct FanTile {
  uint64_t src, src_pitch;
  uint32_t rows, row_bytes, n_dst, pad;
  uint64_t dst[kMaxFan];
  uint64_t dst_pitch[kMaxFan];
};
static_assert(sizeof(FanTile) == 96, "FanTile layout");

#if defined(__CUDACC__)
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD inline
#endif

// A piece of one strided box copy, i.e. the tiles one lower_box step produces, kept as one
// record until the bases are known and expanded into tiles on the GPU (the device-resident
// copy schedule): row mode (per > 0) — tile t covers rows [t per, min(rows, (t+1) per)) of
// row_bytes each; split mode (per == 0) — each row is cut into `tile`-byte tiles, row-major.
struct DevPiece {
  uint64_t src, src_pitch;
  uint64_t dst[kMaxFan], dst_pitch[kMaxFan];
  uint64_t first;       // index of the piece's first tile in the expanded array
  uint64_t row_bytes;   // split mode: a whole contiguous run (may exceed 4 GiB)
  uint32_t rows, per, tile, n_dst;
};
static_assert(sizeof(DevPiece) == 112, "DevPiece layout");

RS_HD uint64_t piece_tile_count(uint32_t rows, uint64_t row_bytes, uint32_t per, uint32_t tile) {
  return per ? (uint64_t(rows) + per - 1) / per : uint64_t(rows) * ((row_bytes + tile - 1) / tile);
}
// Tile t of a piece: first row r0, byte offset c within the row, rows and bytes per row.
RS_HD void piece_tile(uint32_t rows, uint64_t row_bytes, uint32_t per, uint32_t tile, uint64_t t, uint64_t& r0,
                      uint64_t& c, uint32_t& n_rows, uint32_t& n_bytes) {
  if (per) {
    r0 = t * per, c = 0;
    n_rows = uint32_t(rows - r0 < per ? rows - r0 : per), n_bytes = uint32_t(row_bytes);
  } else {
    const uint64_t cpr = (row_bytes + tile - 1) / tile;
    r0 = t / cpr, c = (t % cpr) * tile;
    n_rows = 1, n_bytes = uint32_t(row_bytes - c < tile ? row_bytes - c : tile);
  }
}

// Which copy kernel moves the 16-byte-aligned tiles (misaligned ones always take the
// generic-width LDG/STG kernel).  Defaults can be overridden by RESHARD_COPY_KERNEL
// (ldg | ldg8 | bulk), RESHARD_CTAS_PER_SM, RESHARD_BULK_STAGES, RESHARD_BULK_STAGE_KIB.
// Defaults from the round-1 B200 sweep (profiles/r02_sweep.json): TMA bulk, 1 CTA/SM,
// 8 stages x 24 KiB reached 6.59 TB/s on GPT-3 1.3B vs 6.17 TB/s for LDG/STG at 3 CTAs/SM.
enum class CopyKernel : int { Ldg = 0, Ldg8 = 1, Bulk = 2, BulkStrided = 3, BulkWarp = 4, BulkDyn = 5 };
inline bool is_bulk(CopyKernel k) {
  return k == CopyKernel::Bulk || k == CopyKernel::BulkStrided || k == CopyKernel::BulkWarp || k == CopyKernel::BulkDyn;
}
struct CopyConfig {
  CopyKernel kernel = CopyKernel::BulkStrided;  // r08 same-box A/B: 3-4% faster than Bulk
  int ctas_per_sm = 1;
  int stages = 6;               // bulk: shared-memory ring depth
  unsigned cell_align = 256;    // arena placement of cells (bytes, power of two >= 256; RESHARD_CELL_ALIGN)
  // bulk: bytes per stage (tiles are cut to fit one stage).  r2_43 A/B on all four copy
  // workloads: 6 x 32 KiB beats the earlier 7 x 29 KiB everywhere (GPT-2 small 0.470 vs 0.489 ms,
  // 1.3B 5.40 vs 5.46, 6.7B 42.2 vs 44.3, recovery 13.6 vs 13.8): power-of-two stages hold whole
  // 4 / 8 / 16 KiB rows, so a tile fills its stage (29 KiB left 17 % of a stage empty on 8 KiB rows)
  unsigned stage_bytes = 32768;
  int host_chunks = 64;         // pipeline depth of the host-buffer path (run_host); r13 sweep
  int dyn_claim = 2;            // bulk_dyn: tiles per claim (RESHARD_DYN_CLAIM); r2_18 at 29 KiB tiles: 1 loses 15 %, 8 best;
                                // r2_45 at 32 KiB: 2 best (1.3B 5.33 / 5.34 / 5.38 ms for 2 / 4 / 8, 6.7B 41.6 / 41.7 / 41.9)
  int dyn_min_tiles = 200000;   // bulk_strided launches of at least this many tiles run as bulk_dyn (0: never; RESHARD_DYN_MIN_TILES)
  bool ldg_dyn = false;         // K1/K2 aligned + fan-out kernels: dynamic tile claims (RESHARD_LDG_DYN)
  int dyn_tail = -1;            // bulk_dyn: tiles per CTA claimed dynamically at the end (-1: all; RESHARD_DYN_TAIL)
  bool tensor = false;          // bulk_strided: strided 2-D pieces as TMA tensor boxes (K3T, RESHARD_TMA_TENSOR=1)
  int l2_hint = 0;              // bulk_strided: L2 evict_first on loads (1), stores (2), both (3); r25 A/B: 0 is best (loads evict_first -2.3 %)
  static CopyConfig from_env();
};

struct CellBinding {
  int32_t gpu = -1;    // world GPU index
  int32_t arena = 0;   // 0: src arena, 1: dst arena
  uint64_t offset = 0; // byte offset inside the arena
  uint64_t bytes = 0;
};

// run_host flags (the C ABI's RS_HOST_* bits)
enum : unsigned { kHostSkipUnread = 1u };

struct Timing {
  float ms = 0;        // device time of the copy kernel(s), CUDA events on the launch stream
  uint64_t tiles = 0;
  uint64_t bytes = 0;       // algorithmic bytes written (each destination byte once)
  uint64_t launches = 0;
  uint64_t read_bytes = 0;  // algorithmic bytes read (a fan-out tile reads its source once)
  float main_ms = 0;        // device time of the dominant kernel alone, when timed separately (K5: gather pass)
};

// The GPUs this process drives.  World GPU w is local iff local_of(w) >= 0.
class Context {
 public:
  Context(int world_gpus, std::vector<int> world_ids, std::vector<int> cuda_devices);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  int world() const { return world_; }
  int local_of(int world_gpu) const;
  int cuda_device(int world_gpu) const;       // DeviceUnavailable when not local
  void* stream(int world_gpu) const;          // cudaStream_t
  const std::vector<int>& local_world_ids() const { return world_ids_; }
  int sm_count(int world_gpu) const;

 private:
  int world_;
  std::vector<int> world_ids_, cuda_devs_;
  std::vector<void*> streams_;
  std::vector<int> sms_;
};

class Executor {
 public:
  // src_gpu[i]: world GPU of from->devices[i]; dst_gpu[j]: world GPU of to->devices[j].
  // [t_begin, t_end): only the tensors of this catalog window get storage and work — a plan
  // too large for the world's HBM is executed as several windows (waves) over the same arenas.
  // central_gpu >= 0 selects apply_plan's central mode (the paper's §6.3
  // baseline): every moved fragment is first fetched into a staging region at the end of
  // that GPU's dst arena, then re-uploaded from there to its destination cell (two
  // dependent phases); resident fragments stay local.  Same final state as distributed mode.
  Executor(Context& ctx, std::shared_ptr<const ReconfigPlan> plan, std::vector<int> src_gpu, std::vector<int> dst_gpu,
           uint64_t tile_bytes = 256 << 10, CopyConfig cfg = CopyConfig::from_env(), uint32_t t_begin = 0,
           uint32_t t_end = UINT32_MAX, int central_gpu = -1);
  const CopyConfig& copy_config() const { return cfg_; }
  int central_gpu() const { return central_; }        // -1: distributed mode
  uint64_t staging_bytes() const { return staging_bytes_; }  // central mode: part of dst_arena_bytes(central)
  ~Executor();

  uint64_t src_arena_bytes(int gpu) const { return src_size_[size_t(gpu)]; }
  uint64_t dst_arena_bytes(int gpu) const { return dst_size_[size_t(gpu)]; }
  // Arena base addresses as seen by THIS process (own GPUs: local pointers; peers: P2P/IPC
  // mappings).  Every GPU that a local tile reads from or writes to must be bound.
  void bind(int gpu, void* src_base, void* dst_base);
  void prepare();  // lower fragments to tiles for the local GPUs and upload them

  void run();                       // launch on every local GPU (async), all from one common start mark
  std::vector<Timing> wait();       // per local GPU, after completion
  // The last wait()'s world time: from the common start (recorded on the first local GPU,
  // waited on by every other) to the end of the last local GPU's kernels, peer pushes included.
  float world_ms() const { return world_ms_; }
  // End to end through host buffers over every local GPU (multi-GPU single-process worlds,
  // and one GPU): H2D of each src arena, each GPU's kernels once its own src landed, world
  // barrier, D2H of each dst arena, all GPUs concurrently; returns the ms from the common start
  // to the last D2H.
  float run_host_world(const std::vector<const void*>& host_src, const std::vector<void*>& host_dst);
  // End-to-end on host buffers (single-GPU world): H2D of the whole src arena from
  // `host_src`, the copy kernel, D2H of the whole dst arena into `host_dst`; CUDA events
  // bracket all three.  Pinned host memory gives full PCIe bandwidth.
  // flags & kHostSkipUnread: upload only the source ranges the tiles read (the pipelined path);
  // state no tile reads (kept cells) stays in the host buffer and is not copied to the device.
  Timing run_host(int gpu, const void* host_src, void* host_dst, unsigned flags = 0);
  // Bytes run_host(gpu, ..., flags) copies host -> device.
  uint64_t host_upload_bytes(int gpu, unsigned flags);
  // The same end-to-end step for multi-process worlds, in phases the caller separates with
  // cross-rank barriers: 0 = start mark + H2D of this GPU's src arena, 1 = the kernels,
  // 2 = D2H of this GPU's dst arena + stop mark.  Each phase is async on the GPU's stream
  // and synchronized before returning; host_elapsed() is the event time from mark to mark.
  void host_phase(int gpu, int phase, void* host_buf);
  float host_elapsed(int gpu);

  // Synthetic payload (K6) into the src cells of local GPUs; K7 verification of every
  // destination cell on local GPUs (kept cells included).  Returns mismatching bytes.
  void fill_sources();
  uint64_t verify_destinations();
  // ExecutionReport verification digests: per base tensor of the window,
  // FNV-1a-64 of the tensor reassembled from one replica of each cell of side 0 (source
  // layout) or 1 (destination layout), read back from the local GPUs (off the clock).
  // End-to-end preservation <=> digests(0) == digests(1).
  struct Digest {
    uint32_t tensor;
    uint32_t ok;   // 0: some cell is not held by a local GPU (no digest)
    uint64_t fnv;
  };
  std::vector<Digest> digests(int side, int replica = 0);  // replica: which DP copy of each cell (< 0: from the end)

  void* arena_base(int gpu, int arena) const { return arena == 0 ? src_base_[size_t(gpu)] : dst_base_[size_t(gpu)]; }
  Context& context() const { return ctx_; }
  const std::vector<CellBinding>& src_bindings() const { return src_bind_; }  // per (from dev, t, cell) in order
  const std::vector<CellBinding>& dst_bindings() const { return dst_bind_; }  // per plan->dst_cells entry
  const ReconfigPlan& plan() const { return *plan_; }
  uint64_t tiles_for(int gpu) const;
  uint64_t copy_bytes_for(int gpu) const;  // bytes written by the tiles GPU `gpu` executes
  uint64_t read_bytes_for(int gpu) const;  // bytes they read (fan-out reads once)
  // bytes GPU `gpu`'s tiles write into each world GPU's memory (index = destination GPU):
  // the egress row of the all-to-all (entry `gpu` itself: local HBM writes)
  std::vector<uint64_t> bytes_to(int gpu) const;

 private:
  struct Logical {  // a piece (DevPiece geometry) before arena bases are known; n_dst > 1: fan-out
    int32_t src_gpu;
    uint32_t n_dst;
    uint32_t src_arena;  // 0: src arena of src_gpu, 1: its dst arena (central mode's staging)
    uint64_t src_off, src_pitch;
    uint64_t row_bytes;       // the contiguous run (split mode: may exceed one tile)
    uint32_t rows, per, tile;  // per == 0: split mode, `tile` bytes per tile
    uint64_t n_tiles;
    int32_t dst_gpu[kMaxFan];
    uint64_t dst_off[kMaxFan], dst_pitch[kMaxFan];
  };
  struct Local;
  void launch_local(Local& l, void* stream);
  using SrcLookup = std::vector<std::unordered_map<uint64_t, size_t>>;  // (tensor<<32|cell) -> src_bind_ index
  void build_distributed(const SrcLookup& src_lookup);
  void build_central(const SrcLookup& src_lookup);
  void lower_tiles(Local& l, const std::vector<Logical>& lt, bool host_chunks);
  void plan_host_chunks(Local& l);
  bool plan_world_chunks();
  float run_host_world_pipelined(const std::vector<const void*>& host_src, const std::vector<void*>& host_dst);
  uint64_t payload_pass(const std::vector<std::vector<cuda::PayloadTask>>& per_local, bool verify);

  Context& ctx_;
  std::shared_ptr<const ReconfigPlan> plan_;
  std::vector<int> src_gpu_, dst_gpu_;
  CopyConfig cfg_;
  uint64_t tile_bytes_;
  uint32_t t_begin_, t_end_;
  std::vector<uint64_t> src_size_, dst_size_;
  std::vector<CellBinding> src_bind_, dst_bind_;
  std::vector<std::vector<Logical>> logical_;   // per executing (source) world GPU
  int central_ = -1;
  std::vector<Logical> logical_b_;              // central mode: staging -> destinations (on central_)
  uint64_t staging_bytes_ = 0;
  std::vector<void*> src_base_, dst_base_;
  std::vector<std::unique_ptr<Local>> local_;   // per local GPU: device tiles, events
  void* w_start_ = nullptr;  // cudaEvent_t on local_[0]'s device: world marks
  void* w_stop_ = nullptr;
  float world_ms_ = 0;
  bool world_chunks_ready_ = false, world_pipelined_ = false;
};

// DP replication as a single push (SURVEY §8(b) rs_broadcast): `bytes` at `src` on world GPU
// `gpu` copied to every pointer in `dsts` (local memory or peer mappings) by one kernel on
// that GPU — fan-out tiles read the source once per group of kMaxFan destinations and store
// it to each (TMA bulk when everything is 16-byte aligned, LDG/STG otherwise).  No NCCL
// ring on the data path; this is what the executor's fan-out tiles do inside a reshard.
Timing broadcast(Context& ctx, int gpu, const void* src, const std::vector<void*>& dsts, uint64_t bytes);

// Device-side slice / merge on one GPU (reference slice tensor.cpp:61-78, merge :80-114):
// same validation and error precedence, bytes moved by the tile kernel.
struct DeviceTensorView {
  Dtype dtype;
  Shape shape;
  const void* data;
};
void device_slice(Context& ctx, int gpu, const DeviceTensorView& t, const Range& r, void* out);
// The reference merge's checks alone, in its order (tensor.cpp:81-98), for callers that
// validate before staging data (host_merge).
struct MergePartSpec {
  const Range* range;
  Dtype dtype;
  const Shape* shape;
};
void validate_merge(const std::vector<MergePartSpec>& parts, const Shape& target);
void device_merge(Context& ctx, int gpu, const std::vector<std::pair<Range, DeviceTensorView>>& parts,
                  const Shape& target, void* out);

}  // namespace reshard
