// Executor: lowers a ReconfigPlan to copy tiles and runs them (see reshard/executor.hpp).
#include "reshard/executor.hpp"

#include <cstdio>
#include <cuda.h>  // CUtensorMap and its encoder's signature (resolved through the runtime: no -lcuda)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>
#include <cstring>
#include <map>
#include <unordered_map>

#include "cuda/kernels.hpp"
#include "reshard/trace.hpp"

namespace reshard {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr uint64_t kCellAlign = 256;
uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Emit the copy of box `ext` from (src cell shape ss, origin sl) to (dst cell shape ds,
// origin dl), collapsing dimensions that are full on both sides into one contiguous run
// and cutting the rest into tiles of about `tile` bytes.
// One strided box copy (extents `ext`, source origin/shape sl/ss, destination origin/shape
// dl/ds, element width w) as pieces: dims full on both sides collapse into one contiguous
// run; for every index of the dims outside (row dim, run) one piece of `rows` rows, cut into
// tiles of ~`tile` bytes — several rows per tile (row mode, in-tile byte offsets < 2^31 for
// the kernels) or, when a run is longer than a tile, `tile`-byte slices of each row (split
// mode).  emit(src_off, dst_off, src_pitch, dst_pitch, rows, run, per, split_tile).
template <class Emit>
void lower_box_pieces(const Shape& ext, const Shape& sl, const Shape& ss, const Shape& dl, const Shape& ds, uint64_t w,
                      uint64_t tile, Emit&& emit) {
  const int r = int(ext.size());
  std::vector<uint64_t> sst(size_t(r), w), dst(size_t(r), w);
  for (int d = r - 1; d > 0; --d) sst[size_t(d - 1)] = sst[size_t(d)] * ss[size_t(d)], dst[size_t(d - 1)] = dst[size_t(d)] * ds[size_t(d)];
  uint64_t soff = 0, doff = 0;
  for (int d = 0; d < r; ++d) soff += sl[size_t(d)] * sst[size_t(d)], doff += dl[size_t(d)] * dst[size_t(d)];
  if (r == 0) {
    emit(soff, doff, uint64_t(0), uint64_t(0), uint64_t(1), w, uint32_t(1), uint32_t(0));
    return;
  }
  // innermost run: dims k..r-1, where every dim > k is full on both sides
  int k = r - 1;
  uint64_t run = ext[size_t(k)] * w;
  while (k > 0 && ext[size_t(k)] == ss[size_t(k)] && ext[size_t(k)] == ds[size_t(k)]) {
    --k;
    run *= ext[size_t(k)];
  }
  // rows = dim k-1 (if any); dims 0..k-2 enumerated here
  const uint64_t rows = k > 0 ? ext[size_t(k - 1)] : 1;
  const uint64_t sp = k > 0 ? sst[size_t(k - 1)] : run, dp = k > 0 ? dst[size_t(k - 1)] : run;
  const int outer = std::max(k - 1, 0);
  const bool split = run >= tile;
  // rows per tile: ~tile bytes, and in-tile byte offsets must fit 31 bits (kernel math)
  const uint64_t span = std::max<uint64_t>(std::max(sp, dp), 1);
  const uint32_t per = split ? 0u : uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(tile / run, ((1ull << 31) - run) / span + 1)));
  std::vector<uint64_t> idx(size_t(outer), 0);
  for (;;) {
    uint64_t so = soff, dof = doff;
    for (int d = 0; d < outer; ++d) so += idx[size_t(d)] * sst[size_t(d)], dof += idx[size_t(d)] * dst[size_t(d)];
    emit(so, dof, sp, dp, rows, run, per, split ? uint32_t(tile) : uint32_t(0));
    int d = outer - 1;
    for (; d >= 0; --d) {
      if (++idx[size_t(d)] < ext[size_t(d)]) break;
      idx[size_t(d)] = 0;
    }
    if (d < 0) return;
  }
}

// The same copy as tiles: emit(src_off, dst_off, src_pitch, dst_pitch, rows, bytes) — the
// host expansion of lower_box_pieces, with the device expansion's tile math.
template <class Emit>
void lower_box(const Shape& ext, const Shape& sl, const Shape& ss, const Shape& dl, const Shape& ds, uint64_t w,
               uint64_t tile, Emit&& emit) {
  lower_box_pieces(ext, sl, ss, dl, ds, w, tile,
                   [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run, uint32_t per,
                       uint32_t tl) {
                     const uint64_t n = piece_tile_count(uint32_t(rows), run, per, tl);
                     for (uint64_t t = 0; t < n; ++t) {
                       uint64_t r0, c;
                       uint32_t nr, nb;
                       piece_tile(uint32_t(rows), run, per, tl, t, r0, c, nr, nb);
                       emit(so + r0 * sp + c, dof + r0 * dp + c, per ? sp : uint64_t(0), per ? dp : uint64_t(0),
                            uint64_t(nr), uint64_t(nb));
                     }
                   });
}

bool aligned16(const CopyTile& t) {
  return ((t.src | t.dst | t.row_bytes | (t.rows > 1 ? (t.src_pitch | t.dst_pitch) : 0)) & 15) == 0;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  if (!fn) raise(Errc::CudaError, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// K3T box geometry of a strided row-mode piece: the row of R bytes is e 8-byte words x nch
// chunks (e <= 256 words: the TMA box limit), a box is e x bc x br; one tensor tile per box.
struct TensorBox {
  uint32_t e, nch, bc, br;
};
TensorBox tensor_box(uint64_t row_bytes, uint32_t rows, uint64_t stage_bytes) {
  TensorBox b{};
  const uint64_t words = row_bytes / 8;
  b.e = uint32_t(words);
  if (words > 256) {
    b.e = 256;
    while (words % b.e) b.e -= 2;
  }
  b.nch = uint32_t(words / b.e);
  const uint64_t eb = uint64_t(b.e) * 8;
  b.bc = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>({b.nch, 256, stage_bytes / eb})));
  b.br = b.bc < b.nch ? 1u : uint32_t(std::max<uint64_t>(1, std::min<uint64_t>({256, rows, stage_bytes / (eb * b.nch)})));
  return b;
}
void encode_map(CUtensorMap* m, uint64_t base, const TensorBox& b, uint32_t rows, uint64_t pitch) {
  const cuuint64_t dims[3] = {b.e, b.nch, rows};
  const cuuint64_t strides[2] = {uint64_t(b.e) * 8, pitch};
  const cuuint32_t box[3] = {b.e, b.bc, b.br}, es[3] = {1, 1, 1};
  const CUresult r = encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, reinterpret_cast<void*>(base), dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(Errc::CudaError, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}


}  // namespace

CopyConfig CopyConfig::from_env() {
  CopyConfig c;
  if (const char* k = std::getenv("RESHARD_COPY_KERNEL")) {
    std::string s(k);
    if (s == "ldg") c.kernel = CopyKernel::Ldg;
    else if (s == "ldg8") c.kernel = CopyKernel::Ldg8;
    else if (s == "bulk") c.kernel = CopyKernel::Bulk;
    else if (s == "bulk_strided") c.kernel = CopyKernel::BulkStrided;
    else if (s == "bulk_warp") c.kernel = CopyKernel::BulkWarp;
    else if (s == "bulk_dyn") c.kernel = CopyKernel::BulkDyn;
    else if (!s.empty())
      raise(Errc::InvalidArgument, "RESHARD_COPY_KERNEL must be ldg, ldg8, bulk, bulk_strided, bulk_warp or bulk_dyn");
  }
  c.ctas_per_sm = std::max(1, env_int("RESHARD_CTAS_PER_SM", is_bulk(c.kernel) ? 1 : 3));
  c.stages = env_int("RESHARD_BULK_STAGES", c.stages);
  c.l2_hint = env_int("RESHARD_BULK_HINT", c.l2_hint) & 3;
  c.stage_bytes = unsigned(std::max(1, env_int("RESHARD_BULK_STAGE_KIB", int(c.stage_bytes >> 10)))) << 10;
  c.host_chunks = std::max(1, env_int("RESHARD_HOST_CHUNKS", c.host_chunks));
  c.tensor = env_int("RESHARD_TMA_TENSOR", c.tensor ? 1 : 0) != 0;
  c.dyn_tail = env_int("RESHARD_DYN_TAIL", c.dyn_tail);
  c.dyn_claim = env_int("RESHARD_DYN_CLAIM", c.dyn_claim);
  c.dyn_min_tiles = env_int("RESHARD_DYN_MIN_TILES", c.dyn_min_tiles);
  c.ldg_dyn = env_int("RESHARD_LDG_DYN", c.ldg_dyn ? 1 : 0) != 0;
  c.cell_align = unsigned(std::max(256, env_int("RESHARD_CELL_ALIGN", int(c.cell_align))));
  if (c.cell_align & (c.cell_align - 1)) raise(Errc::InvalidArgument, "RESHARD_CELL_ALIGN must be a power of two");
  return c;
}

// ---- Context ---------------------------------------------------------------------------
Context::Context(int world, std::vector<int> world_ids, std::vector<int> cuda_devices)
    : world_(world), world_ids_(std::move(world_ids)), cuda_devs_(std::move(cuda_devices)) {
  if (world_ids_.size() != cuda_devs_.size()) raise(Errc::InvalidArgument, "world ids / cuda devices length");
  if (world_ < 1) raise(Errc::InvalidArgument, "world must have at least one GPU");
  // A context with no local GPU is a planning-only view of the world: layouts and tiles can
  // be computed (and compared across ranks) but nothing runs.
  int n = 0;
  if (!cuda_devs_.empty() && (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)) {
    cudaGetLastError();
    raise(Errc::DeviceUnavailable, "no CUDA device visible");
  }
  for (size_t i = 0; i < cuda_devs_.size(); ++i) {
    if (cuda_devs_[i] < 0 || cuda_devs_[i] >= n) raise(Errc::DeviceUnavailable, "cuda device " + std::to_string(cuda_devs_[i]));
    if (world_ids_[i] < 0 || world_ids_[i] >= world_) raise(Errc::InvalidArgument, "world id out of range");
    DeviceGuard g(cuda_devs_[i]);
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    streams_.push_back(s);
    int sm = 0;
    ck(cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, cuda_devs_[i]), "sm count");
    sms_.push_back(sm);
    // Pre-size the stream-ordered pool the copy schedules come from: the pool keeps what it
    // maps (release threshold: never) and is primed once per device here, at context creation,
    // so a reconfiguration's prepare() sub-allocates descriptors without mapping new memory.
    if (std::find(cuda_devs_.begin(), cuda_devs_.begin() + long(i), cuda_devs_[i]) == cuda_devs_.begin() + long(i)) {
      cudaMemPool_t pool;
      ck(cudaDeviceGetDefaultMemPool(&pool, cuda_devs_[i]), "default mem pool");
      uint64_t keep = UINT64_MAX;
      ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool release threshold");
      const uint64_t prime = uint64_t(std::max(0, env_int("RESHARD_DESC_POOL_MIB", 256))) << 20;
      if (prime) {
        void* p = nullptr;
        ck(cudaMallocAsync(&p, prime, s), "prime descriptor pool");
        ck(cudaFreeAsync(p, s), "prime descriptor pool");
        ck(cudaStreamSynchronize(s), "prime descriptor pool");
      }
    }
    // direct peer access between the local GPUs (single-process multi-GPU runs)
    for (size_t j = 0; j < cuda_devs_.size(); ++j) {
      if (j == i) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, cuda_devs_[i], cuda_devs_[j]);
      if (ok) {
        cudaError_t e = cudaDeviceEnablePeerAccess(cuda_devs_[j], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ck(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
}
Context::~Context() {
  for (size_t i = 0; i < streams_.size(); ++i) {
    cudaSetDevice(cuda_devs_[i]);
    cudaStreamDestroy(static_cast<cudaStream_t>(streams_[i]));
  }
}
int Context::local_of(int w) const {
  auto it = std::find(world_ids_.begin(), world_ids_.end(), w);
  return it == world_ids_.end() ? -1 : int(it - world_ids_.begin());
}
int Context::cuda_device(int w) const {
  int l = local_of(w);
  if (l < 0) raise(Errc::DeviceUnavailable, "world GPU " + std::to_string(w) + " is not driven by this process");
  return cuda_devs_[size_t(l)];
}
void* Context::stream(int w) const {
  int l = local_of(w);
  if (l < 0) raise(Errc::DeviceUnavailable, "world GPU " + std::to_string(w) + " is not local");
  return streams_[size_t(l)];
}
int Context::sm_count(int w) const {
  int l = local_of(w);
  return l < 0 ? 148 : sms_[size_t(l)];
}

// ---- Executor --------------------------------------------------------------------------
// A slice of the destination-ordered tile list for the pipelined host path: it reads src
// arena bytes below src_end and writes nothing below dst_min.
struct HostChunk {
  uint64_t t0, t1, src_end, dst_min;
  std::vector<std::pair<uint64_t, uint64_t>> uploads;  // src arena [off, off+len) first needed by this chunk
};

// Src arena byte ranges first read by each chunk (chunks in order): the union of the
// chunk's tile spans minus everything earlier chunks already uploaded.  Uploading exactly
// these keeps the H2D stream in the order the kernels consume it, so D2H of early chunks
// overlaps the rest of the upload whatever the src/dst arena orders are.
void plan_uploads(std::vector<HostChunk>& chunks, const std::vector<std::vector<std::pair<uint64_t, uint64_t>>>& spans) {
  std::map<uint64_t, uint64_t> done;  // start -> end, disjoint
  auto covered_minus = [&](uint64_t a, uint64_t b, std::vector<std::pair<uint64_t, uint64_t>>& out) {
    auto it = done.upper_bound(a);
    if (it != done.begin()) --it;
    uint64_t cur = a;
    for (; it != done.end() && it->first < b; ++it) {
      if (it->second <= cur) continue;
      if (it->first > cur) out.emplace_back(cur, it->first - cur);
      cur = std::max(cur, it->second);
      if (cur >= b) break;
    }
    if (cur < b) out.emplace_back(cur, b - cur);
  };
  for (size_t k = 0; k < chunks.size(); ++k) {
    auto v = spans[k];
    std::sort(v.begin(), v.end());
    std::vector<std::pair<uint64_t, uint64_t>> merged;  // [a, b)
    for (auto& [a, b] : v) {
      if (!merged.empty() && a <= merged.back().second) merged.back().second = std::max(merged.back().second, b);
      else merged.emplace_back(a, b);
    }
    for (auto& [a, b] : merged) covered_minus(a, b, chunks[k].uploads);
    for (auto& [a, b] : merged) {  // insert [a, b) into done, coalescing
      uint64_t lo = a, hi = b;
      auto it = done.lower_bound(a);
      if (it != done.begin() && std::prev(it)->second >= a) --it;
      while (it != done.end() && it->first <= hi) {
        lo = std::min(lo, it->first), hi = std::max(hi, it->second);
        it = done.erase(it);
      }
      done[lo] = hi;
    }
  }
}

struct Executor::Local {
  int world = -1, dev = -1;
  FanTile* d_fan = nullptr;     // bulk kernel tiles (sorted by first destination, interleaved for the grid)
  FanTile* d_fan_chunks = nullptr;  // the same tiles, interleaved per host chunk (pipelined host path)
  CopyTile* d_tiles = nullptr;  // [LDG aligned tiles, sorted by dst | misaligned tiles]
  FanTile* d_fanl = nullptr;    // K2 fan-out tiles (LDG once, STG to every destination; peers included)
  void* d_maps = nullptr;       // K3T: CUtensorMaps of the strided pieces (src + one per destination)
  uint64_t n_tensor = 0;        // K3T tiles, appended to d_fan after the expanded 1-D tiles
  uint64_t n_fan = 0, n_aligned = 0, n_misc = 0, n_fanl = 0, bytes = 0, read_bytes = 0;
  cudaEvent_t e_h2d = nullptr, e_kern = nullptr, e_d2h = nullptr;  // run_host_world phase marks
  cudaEvent_t start = nullptr, stop = nullptr;
  unsigned long long* d_count = nullptr;
  unsigned long long* d_claim = nullptr;  // bulk_dyn's tile-claim counter (2 x u64, kept zero between launches)
  unsigned long long* d_claim2 = nullptr; // the LDG/STG kernels' (they may run beside K3 on the side stream)
  std::vector<HostChunk> chunks;
  std::vector<DevPiece> chunk_pieces;  // the one tile list the host pipeline cuts into chunks (lazy)
  bool chunks_ready = true;           // chunks planned (or not applicable)
  bool chunk_fan = false;             // chunk_pieces feed the bulk kernel (else the aligned LDG kernel)
  // world host pipeline (run_host_world): the piece lists per kernel (0 K3 bulk, 1 aligned LDG,
  // 2 misaligned, 3 K2 fan-out), their chunks, and per round the end of this GPU's dst-arena
  // prefix that no later chunk of any GPU writes
  std::vector<DevPiece> lists[4];
  struct WorldChunk {
    uint64_t t0[4] = {0, 0, 0, 0}, t1[4] = {0, 0, 0, 0};
    std::vector<std::pair<uint64_t, uint64_t>> uploads;  // src arena ranges first read by this chunk
  };
  std::vector<WorldChunk> wchunks;
  std::vector<uint64_t> wsafe;
  std::vector<cudaEvent_t> wev;  // per chunk: H2D landed, kernels done (2K events)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaStream_t s_aux = nullptr;                       // LDG/STG tiles beside the bulk kernel
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> ev;
  std::unique_ptr<Local> phase_b;  // central mode, on the central GPU: staging -> destination tiles
  uint64_t launches() const { return (n_fan ? 1 : 0) + (n_aligned ? 1 : 0) + (n_misc ? 1 : 0) + (n_fanl ? 1 : 0); }
  uint64_t tiles() const { return n_fan + n_aligned + n_misc + n_fanl; }
  ~Local() {
    if (dev < 0) return;
    cudaSetDevice(dev);
    if (d_fan) cudaFree(d_fan);
    if (d_fan_chunks) cudaFree(d_fan_chunks);
    if (d_tiles) cudaFree(d_tiles);
    if (d_fanl) cudaFree(d_fanl);
    if (d_maps) cudaFree(d_maps);
    for (auto e : {e_h2d, e_kern, e_d2h})
      if (e) cudaEventDestroy(e);
    if (d_count) cudaFree(d_count);
    if (d_claim) cudaFree(d_claim);
    if (d_claim2) cudaFree(d_claim2);
    if (start) cudaEventDestroy(start);
    if (stop) cudaEventDestroy(stop);
    for (auto e : ev) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    if (s_aux) cudaStreamDestroy(s_aux);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
  }
};

// The bulk kernel (one 32-thread CTA per SM, TMA-driven) and the LDG/STG kernels (tiles
// with a peer destination, or not 16-byte aligned) run concurrently on two streams: they
// co-reside on every SM (32 + 3 x 512 threads, the LDG kernels use no shared memory), so a
// GPU's local relayout (HBM) overlaps its NVLink pushes instead of preceding them.
void Executor::launch_local(Local& l, void* stream) {
  const int sms = ctx_.sm_count(l.world);
  auto s = static_cast<cudaStream_t>(stream);
  const bool both = l.n_fan && (l.n_aligned || l.n_misc || l.n_fanl);
  cudaStream_t side = s;
  if (both) {
    if (!l.s_aux) {
      ck(cudaStreamCreateWithFlags(&l.s_aux, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&l.fork, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&l.join, cudaEventDisableTiming), "event");
    }
    ck(cudaEventRecord(l.fork, s), "fork");
    ck(cudaStreamWaitEvent(l.s_aux, l.fork, 0), "fork wait");
    side = l.s_aux;
  }
  cuda::launch_bulk(l.d_fan, l.n_fan, cfg_, sms, s, l.d_claim);
  cuda::launch_copy(l.d_tiles, l.n_aligned, cfg_, sms, true, side, l.d_claim2);
  cuda::launch_copy(l.d_tiles + l.n_aligned, l.n_misc, cfg_, sms, false, side);
  cuda::launch_copy_fan(l.d_fanl, l.n_fanl, cfg_, sms, side, l.d_claim2);
  if (both) {
    ck(cudaEventRecord(l.join, side), "join");
    ck(cudaStreamWaitEvent(s, l.join, 0), "join wait");
  }
}

Executor::Executor(Context& ctx, std::shared_ptr<const ReconfigPlan> plan, std::vector<int> src_gpu,
                   std::vector<int> dst_gpu, uint64_t tile_bytes, CopyConfig cfg, uint32_t t_begin, uint32_t t_end,
                   int central_gpu)
    : ctx_(ctx), plan_(std::move(plan)), src_gpu_(std::move(src_gpu)), dst_gpu_(std::move(dst_gpu)), cfg_(cfg),
      tile_bytes_(std::max<uint64_t>(4096, std::min<uint64_t>(tile_bytes, is_bulk(cfg.kernel) ? cfg.stage_bytes
                                                                                                        : UINT64_MAX) /
                                               16 * 16)),
      t_begin_(t_begin), t_end_(t_end), central_(central_gpu) {
  auto in = [&](uint32_t t) { return t >= t_begin_ && t < t_end_; };
  const PTC& a = *plan_->from;
  const PTC& b = *plan_->to;
  const int G = ctx_.world();
  if (src_gpu_.size() != a.devices.size() || dst_gpu_.size() != b.devices.size())
    raise(Errc::InvalidArgument, "device -> GPU maps must cover both layouts");
  for (int g : src_gpu_)
    if (g < 0 || g >= G) raise(Errc::InvalidArgument, "src GPU out of range");
  for (int g : dst_gpu_)
    if (g < 0 || g >= G) raise(Errc::InvalidArgument, "dst GPU out of range");
  if (central_ >= G) raise(Errc::InvalidArgument, "central GPU out of range");
  // (a planning-only context, with no local GPU, may still compute central layouts)
  if (central_ >= 0 && !ctx_.local_world_ids().empty() && int(ctx_.local_world_ids().size()) != G)
    raise(Errc::InvalidArgument, "central mode needs every GPU of the world in this process");
  src_size_.assign(size_t(G), 0);
  dst_size_.assign(size_t(G), 0);
  src_base_.assign(size_t(G), nullptr);
  dst_base_.assign(size_t(G), nullptr);

  using clk = std::chrono::steady_clock;
  const bool trace = std::getenv("RESHARD_HOST_TRACE") && std::string(std::getenv("RESHARD_HOST_TRACE")) == "1";
  auto t_mark = clk::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    std::fprintf(stderr, "lower-trace %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(clk::now() - t_mark).count());
    t_mark = clk::now();
  };
  // src arena layout (a failed device of a recovery plan holds nothing: no storage, no fill)
  std::vector<char> dead(a.devices.size(), 0);
  for (const DeviceId& f : plan_->failed)
    if (int o = a.ordinal(f); o >= 0) dead[size_t(o)] = 1;
  SrcLookup src_lookup(a.devices.size());
  for (uint32_t i = 0; i < a.devices.size(); ++i)
    for (auto [t, c] : hosted_subtensors(a, a.devices[i])) {
      if (!in(t) || dead[i]) {  // outside this executor's tensor window / failed: no storage, no work
        src_lookup[i][(uint64_t(t) << 32) | c] = src_bind_.size();
        src_bind_.push_back(CellBinding{-1, 0, 0, 0});
        continue;
      }
      const int g = src_gpu_[i];
      CellBinding bnd{g, 0, src_size_[size_t(g)], a.cells[t][c].elements() * dtype_width(a.catalog.tensors[t].dtype)};
      src_size_[size_t(g)] = align_up(bnd.offset + bnd.bytes, cfg_.cell_align);
      src_lookup[i][(uint64_t(t) << 32) | c] = src_bind_.size();
      src_bind_.push_back(bnd);
    }
  // dst arena layout (kept cells alias their src cell when the logical device stays on its GPU)
  for (const PlanDstCell& dc : plan_->dst_cells) {
    if (!in(dc.tensor)) {
      dst_bind_.push_back(CellBinding{-1, 1, 0, 0});
      continue;
    }
    const int g = dst_gpu_[dc.dst_device];
    const uint64_t bytes = b.cells[dc.tensor][dc.cell].elements() * dtype_width(b.catalog.tensors[dc.tensor].dtype);
    if (dc.kept) {
      const PlanFragment& f = plan_->fragments[dc.first];
      const CellBinding& sb = src_bind_[src_lookup[f.src_device].at((uint64_t(dc.tensor) << 32) | f.src_cell)];
      if (sb.gpu == g) {
        dst_bind_.push_back(sb);
        continue;
      }
    }
    CellBinding bnd{g, 1, dst_size_[size_t(g)], bytes};
    dst_size_[size_t(g)] = align_up(bnd.offset + bnd.bytes, cfg_.cell_align);
    dst_bind_.push_back(bnd);
  }
  lap("arenas");
  logical_.assign(size_t(G), {});
  if (central_ >= 0) build_central(src_lookup);
  else build_distributed(src_lookup);
  lap("pieces");
  for (int w : ctx_.local_world_ids()) {
    auto l = std::make_unique<Local>();
    l->world = w;
    l->dev = ctx_.cuda_device(w);
    DeviceGuard g(l->dev);
    ck(cudaEventCreate(&l->start), "cudaEventCreate");
    ck(cudaEventCreate(&l->stop), "cudaEventCreate");
    // from the context's primed stream-ordered pool (a plain cudaMalloc may map a new page)
    ck(cudaMallocAsync(reinterpret_cast<void**>(&l->d_count), sizeof(unsigned long long),
                       static_cast<cudaStream_t>(ctx_.stream(w))), "cudaMallocAsync");
    for (cudaEvent_t* e : {&l->e_h2d, &l->e_kern, &l->e_d2h}) ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    auto claim_counter = [&](Local& x) {
      auto st = static_cast<cudaStream_t>(ctx_.stream(w));
      for (unsigned long long** p : {&x.d_claim, &x.d_claim2}) {
        ck(cudaMallocAsync(reinterpret_cast<void**>(p), 2 * sizeof(unsigned long long), st), "cudaMallocAsync");
        ck(cudaMemsetAsync(*p, 0, 2 * sizeof(unsigned long long), st), "memset claim");
      }
    };
    claim_counter(*l);
    if (w == central_) {
      l->phase_b = std::make_unique<Local>();
      l->phase_b->world = w, l->phase_b->dev = l->dev;
      claim_counter(*l->phase_b);
    }
    local_.push_back(std::move(l));
  }
  if (!local_.empty()) {  // world marks on the first local GPU: one common start, the last GPU's end
    DeviceGuard g(local_[0]->dev);
    ck(cudaEventCreate(reinterpret_cast<cudaEvent_t*>(&w_start_)), "cudaEventCreate");
    ck(cudaEventCreate(reinterpret_cast<cudaEvent_t*>(&w_stop_)), "cudaEventCreate");
  }
  lap("device setup");
}

// apply_plan central mode: each Move's fragment is fetched into the
// central GPU's staging region (dense box, one slot per Move as plan_cost_central counts
// it), then written from there into its destination cell.  Resident fragments are copied
// locally as in distributed mode.
void Executor::build_central(const SrcLookup& src_lookup) {
  const PTC& a = *plan_->from;
  const PTC& b = *plan_->to;
  const uint64_t stage_base = dst_size_[size_t(central_)];
  uint64_t stage = 0;
  for (size_t j = 0; j < plan_->dst_cells.size(); ++j) {
    const PlanDstCell& dc = plan_->dst_cells[j];
    const CellBinding& db = dst_bind_[j];
    if (db.arena == 0 || db.gpu < 0) continue;  // kept in place / outside the tensor window
    const Range& dbox = b.cells[dc.tensor][dc.cell];
    const uint64_t w = dtype_width(a.catalog.tensors[dc.tensor].dtype);
    for (uint32_t k = dc.first; k < dc.first + dc.count; ++k) {
      const PlanFragment& f = plan_->fragments[k];
      const CellBinding& sb = src_bind_[src_lookup[f.src_device].at((uint64_t(dc.tensor) << 32) | f.src_cell)];
      const Range& sbox = a.cells[dc.tensor][f.src_cell];
      const Range rs = f.box.rebase_into(sbox), rd = f.box.rebase_into(dbox);
      Shape sl, dl, ext = f.box.extents();
      for (int d = 0; d < rs.rank(); ++d) sl.push_back(rs.dim(d).lo), dl.push_back(rd.dim(d).lo);
      const Shape zero(ext.size(), 0);
      auto piece = [](int32_t sg, uint32_t sa, uint64_t so, uint64_t sp, int32_t dg, uint64_t dof, uint64_t dp,
                      uint64_t rows, uint64_t run, uint32_t per, uint32_t tl) {
        Logical x{};
        x.src_gpu = sg, x.src_arena = sa, x.n_dst = 1, x.src_off = so, x.src_pitch = sp;
        x.rows = uint32_t(rows), x.row_bytes = run, x.per = per, x.tile = tl;
        x.n_tiles = piece_tile_count(x.rows, run, per, tl);
        x.dst_gpu[0] = dg, x.dst_off[0] = dof, x.dst_pitch[0] = dp;
        return x;
      };
      if (f.resident) {
        lower_box_pieces(ext, sl, sbox.extents(), dl, dbox.extents(), w, tile_bytes_,
                         [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run, uint32_t per,
                             uint32_t tl) {
                           logical_[size_t(sb.gpu)].push_back(
                               piece(sb.gpu, 0, sb.offset + so, sp, db.gpu, db.offset + dof, dp, rows, run, per, tl));
                         });
        continue;
      }
      const uint64_t slot = stage_base + stage;
      stage = align_up(stage + f.box.elements() * w, kCellAlign);
      lower_box_pieces(ext, sl, sbox.extents(), zero, ext, w, tile_bytes_,  // fetch: source cell -> staging slot
                       [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run, uint32_t per,
                           uint32_t tl) {
                         logical_[size_t(sb.gpu)].push_back(
                             piece(sb.gpu, 0, sb.offset + so, sp, central_, slot + dof, dp, rows, run, per, tl));
                       });
      lower_box_pieces(ext, zero, ext, dl, dbox.extents(), w, tile_bytes_,  // re-upload: staging slot -> destination
                       [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run, uint32_t per,
                           uint32_t tl) {
                         logical_b_.push_back(piece(central_, 1, slot + so, sp, db.gpu, db.offset + dof, dp, rows, run, per, tl));
                       });
    }
  }
  staging_bytes_ = stage;
  dst_size_[size_t(central_)] = stage_base + stage;
}

// fragments -> logical tiles, grouped by the executing (source) GPU.  Fragments that read
// the same source box for several destination cells (DP replicas) are grouped; with the
// bulk kernel their tiles are fused into fan-out tiles (source read once).
void Executor::build_distributed(const SrcLookup& src_lookup) {
  const PTC& a = *plan_->from;
  const PTC& b = *plan_->to;
  const char* fan_env = std::getenv("RESHARD_FANOUT");
  const bool fan = !(fan_env && std::string(fan_env) == "0");  // K3 (TMA) or K2 (LDG) fan-out tiles
  struct Member {
    int32_t dst_gpu;
    uint64_t dst_base;
    Shape dl, dshape;
  };
  struct Group {
    size_t src_bind;
    uint32_t tensor, src_cell;
    Range box;
    std::vector<Member> members;
  };
  std::vector<Group> groups;
  std::map<std::pair<size_t, Range>, size_t> group_of;
  for (size_t j = 0; j < plan_->dst_cells.size(); ++j) {
    const PlanDstCell& dc = plan_->dst_cells[j];
    const CellBinding& db = dst_bind_[j];
    if (db.arena == 0 || db.gpu < 0) continue;  // kept in place / outside the tensor window
    const Range& dbox = b.cells[dc.tensor][dc.cell];
    for (uint32_t k = dc.first; k < dc.first + dc.count; ++k) {
      const PlanFragment& f = plan_->fragments[k];
      const size_t si = src_lookup[f.src_device].at((uint64_t(dc.tensor) << 32) | f.src_cell);
      const Range rd = f.box.rebase_into(dbox);
      Shape dl;
      for (int d = 0; d < rd.rank(); ++d) dl.push_back(rd.dim(d).lo);
      auto key = std::make_pair(si, f.box);
      auto it = group_of.find(key);
      if (it == group_of.end() || !fan) {
        group_of[key] = groups.size();
        groups.push_back(Group{si, dc.tensor, f.src_cell, f.box, {}});
        it = group_of.find(key);
      }
      groups[fan ? it->second : groups.size() - 1].members.push_back(Member{db.gpu, db.offset, dl, dbox.extents()});
    }
  }
  // one fragment group -> logical tiles of its executing GPU (fan-out tiles when every
  // member lowers to the same source tiles)
  auto lower_group = [&](const Group& grp, std::vector<std::vector<Logical>>& outs) {
    const CellBinding& sb = src_bind_[grp.src_bind];
    const Range& sbox = a.cells[grp.tensor][grp.src_cell];
    const Range rs = grp.box.rebase_into(sbox);
    Shape sl;
    for (int d = 0; d < rs.rank(); ++d) sl.push_back(rs.dim(d).lo);
    const uint64_t w = dtype_width(a.catalog.tensors[grp.tensor].dtype);
    auto& out = outs[size_t(sb.gpu)];
    auto lower_member = [&](const Member& mem, std::vector<Logical>& dst) {
      lower_box_pieces(grp.box.extents(), sl, sbox.extents(), mem.dl, mem.dshape, w, tile_bytes_,
                       [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run, uint32_t per,
                           uint32_t tl) {
                         Logical& x = dst.emplace_back();
                         x.src_gpu = sb.gpu, x.src_arena = 0, x.n_dst = 1, x.src_off = sb.offset + so, x.src_pitch = sp;
                         x.rows = uint32_t(rows), x.row_bytes = run, x.per = per, x.tile = tl;
                         x.n_tiles = piece_tile_count(x.rows, run, per, tl);
                         x.dst_gpu[0] = mem.dst_gpu, x.dst_off[0] = mem.dst_base + dof, x.dst_pitch[0] = dp;
                       });
    };
    if (grp.members.size() == 1) {  // the common case: pieces straight into the executing GPU's list
      lower_member(grp.members[0], out);
      return;
    }
    std::vector<std::vector<Logical>> per(grp.members.size());
    for (size_t m = 0; m < grp.members.size(); ++m) lower_member(grp.members[m], per[m]);
    // fan-out needs the same source tiles for every member: same pieces with the same cut
    bool same = per.size() > 1;
    for (size_t m = 1; same && m < per.size(); ++m) {
      same = per[m].size() == per[0].size();
      for (size_t t = 0; same && t < per[0].size(); ++t)
        same = per[m][t].src_off == per[0][t].src_off && per[m][t].rows == per[0][t].rows &&
               per[m][t].row_bytes == per[0][t].row_bytes && per[m][t].per == per[0][t].per &&
               per[m][t].tile == per[0][t].tile &&
               (per[0][t].rows == 1 || per[m][t].src_pitch == per[0][t].src_pitch);
    }
    if (!same) {
      for (auto& v : per) out.insert(out.end(), v.begin(), v.end());
      return;
    }
    for (size_t m0 = 0; m0 < per.size(); m0 += kMaxFan)
      for (size_t t = 0; t < per[0].size(); ++t) {
        Logical x = per[m0][t];
        x.n_dst = 0;
        for (size_t m = m0; m < per.size() && m < m0 + kMaxFan; ++m, ++x.n_dst) {
          x.dst_gpu[x.n_dst] = per[m][t].dst_gpu[0];
          x.dst_off[x.n_dst] = per[m][t].dst_off[0];
          x.dst_pitch[x.n_dst] = per[m][t].dst_pitch[0];
        }
        out.push_back(x);
      }
  };
  for (const Group& grp : groups) lower_group(grp, logical_);
}

Executor::~Executor() {
  if (!local_.empty()) {
    cudaSetDevice(local_[0]->dev);
    if (w_start_) cudaEventDestroy(static_cast<cudaEvent_t>(w_start_));
    if (w_stop_) cudaEventDestroy(static_cast<cudaEvent_t>(w_stop_));
  }
}

void Executor::bind(int gpu, void* src, void* dst) {
  if (gpu < 0 || gpu >= ctx_.world()) raise(Errc::InvalidArgument, "bind: GPU out of range");
  // null is allowed for an arena this process never touches (e.g. a peer's src arena)
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % kCellAlign)
    raise(Errc::InvalidArgument, "bind: arenas must be 256-byte aligned");
  src_base_[size_t(gpu)] = src;
  dst_base_[size_t(gpu)] = dst;
}

void Executor::prepare() {
  TraceRange trace_("Executor::prepare");
  for (auto& l : local_) {
    lower_tiles(*l, logical_[size_t(l->world)], central_ < 0);
    if (l->phase_b) lower_tiles(*l->phase_b, logical_b_, false);
  }
}

// Pieces -> the device-resident copy schedule of one local GPU (bases known after bind()):
// the host binds the arena bases into the few pieces, classifies them (bulk fan tiles /
// 16-byte aligned LDG tiles / misaligned LDG tiles), orders them by destination and uploads
// them; the expansion kernels write the tile arrays in device memory.
void Executor::lower_tiles(Local& local, const std::vector<Logical>& lt, bool host_chunks) {
  const bool bulk = is_bulk(cfg_.kernel);
  const bool interleave = cfg_.kernel == CopyKernel::Bulk;  // bulk_strided walks the natural order
  using clk = std::chrono::steady_clock;
  const bool trace = std::getenv("RESHARD_HOST_TRACE") && std::string(std::getenv("RESHARD_HOST_TRACE")) == "1";
  auto t_mark = clk::now();
  auto ms_since = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
  const char* bp = std::getenv("RESHARD_BULK_PEER");
  const bool bulk_peer = bp && std::string(bp) == "1";
  Local* l = &local;
  std::vector<DevPiece> fanp, alignedp, miscp, fanlp;
  uint64_t bytes = 0, read_bytes = 0;
  for (const Logical& x : lt) {
    char* s = static_cast<char*>(x.src_arena ? dst_base_[size_t(x.src_gpu)] : src_base_[size_t(x.src_gpu)]);
    if (!s) raise(Errc::InvalidArgument, "prepare: GPU " + std::to_string(x.src_gpu) + " not bound");
    DevPiece q{};
    q.src = uint64_t(reinterpret_cast<uintptr_t>(s + x.src_off)), q.src_pitch = x.src_pitch;
    q.row_bytes = x.row_bytes, q.rows = x.rows, q.per = x.per, q.tile = x.tile, q.n_dst = x.n_dst;
    // every tile is 16-byte aligned iff the base, the pitch (several rows), the run and the
    // split stride are
    const uint64_t common = x.row_bytes | (x.per ? 0 : x.tile);
    uint64_t bits = q.src | common | (x.rows > 1 ? x.src_pitch : 0);
    bool remote = false;
    for (uint32_t d = 0; d < x.n_dst; ++d) {
      char* dp = static_cast<char*>(dst_base_[size_t(x.dst_gpu[d])]);
      if (!dp) raise(Errc::InvalidArgument, "prepare: GPU " + std::to_string(x.dst_gpu[d]) + " not bound");
      q.dst[d] = uint64_t(reinterpret_cast<uintptr_t>(dp + x.dst_off[d]));
      q.dst_pitch[d] = x.dst_pitch[d];
      bits |= q.dst[d] | (x.rows > 1 ? x.dst_pitch[d] : 0);
      remote |= x.dst_gpu[d] != l->world;
    }
    const uint64_t pb = uint64_t(x.rows) * x.row_bytes;  // the piece's bytes per destination
    const uint64_t max_tile = x.per ? uint64_t(x.per) * x.row_bytes : x.tile;
    bytes += pb * x.n_dst;
    // Cross-GPU tiles use plain st.global through the peer mapping (K2) unless
    // RESHARD_BULK_PEER=1 lets the TMA engine store to peer addresses too: that variant
    // has not been validated on a multi-GPU box yet (one GPU in this environment).
    if (bulk && (!remote || bulk_peer) && (bits & 15) == 0 && max_tile <= cfg_.stage_bytes) {
      fanp.push_back(q);
      read_bytes += pb;
      continue;
    }
    // several destinations, one of them (at least) a peer: K2 fan-out reads the source once
    // and stores every replica (local HBM and NVLink) from registers
    if (x.n_dst > 1 && (bits & 15) == 0) {
      fanlp.push_back(q);
      read_bytes += pb;
      continue;
    }
    for (uint32_t d = 0; d < x.n_dst; ++d) {  // one single-destination piece per destination
      DevPiece one = q;
      one.n_dst = 1, one.dst[0] = q.dst[d], one.dst_pitch[0] = q.dst_pitch[d];
      for (int e = 1; e < kMaxFan; ++e) one.dst[e] = 0, one.dst_pitch[e] = 0;
      const uint64_t b1 = q.src | common | (x.rows > 1 ? (x.src_pitch | q.dst_pitch[d]) : 0) | q.dst[d];
      ((b1 & 15) == 0 ? alignedp : miscp).push_back(one);
      read_bytes += pb;
    }
  }
  // Order: by destination GPU in the all-to-all's shift order — this GPU's own arena first, then
  // GPU world+1, world+2, ... (mod G) — and by destination address within a GPU (sequential
  // writes; monotone destinations per host chunk).  The persistent kernels sweep their list
  // front to back with every CTA, so at any moment a GPU pushes into one peer; with the shift
  // every peer is the target of a different source at the same time and no GPU's NVLink ingress
  // is oversubscribed while others idle (a plain address order would send every source to the
  // lowest-address peer first).  A fan-out piece is keyed by its nearest remote member.
  const int G = ctx_.world();
  std::vector<std::pair<uint64_t, int>> dbases;
  for (int j = 0; j < G; ++j)
    if (dst_base_[size_t(j)]) dbases.emplace_back(uint64_t(reinterpret_cast<uintptr_t>(dst_base_[size_t(j)])), j);
  std::sort(dbases.begin(), dbases.end());
  auto gpu_of = [&](uint64_t a) {
    auto it = std::upper_bound(dbases.begin(), dbases.end(), std::make_pair(a, INT32_MAX));
    return it == dbases.begin() ? -1 : std::prev(it)->second;
  };
  auto by_dst = [&](std::vector<DevPiece>& v) {
    std::vector<std::pair<uint64_t, size_t>> key(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      int best = G;
      for (uint32_t d = 0; d < v[i].n_dst; ++d) {
        const int j = gpu_of(v[i].dst[d]);
        if (j >= 0 && j != l->world) best = std::min(best, (j - l->world + G) % G);
      }
      key[i] = {uint64_t(best == G ? 0 : best), i};
    }
    std::stable_sort(key.begin(), key.end(), [&](const auto& x, const auto& y) {
      return x.first != y.first ? x.first < y.first : v[x.second].dst[0] < v[y.second].dst[0];
    });
    std::vector<DevPiece> out;
    out.reserve(v.size());
    for (auto& k : key) out.push_back(v[k.second]);
    v.swap(out);
  };
  by_dst(fanp), by_dst(alignedp);
  auto number = [](std::vector<DevPiece>& v) {
    uint64_t n = 0;
    for (DevPiece& q : v) q.first = n, n += piece_tile_count(q.rows, q.row_bytes, q.per, q.tile);
    return n;
  };
  by_dst(fanlp);
  // K3T (RESHARD_TMA_TENSOR=1, bulk_strided): strided row-mode pieces become TMA tensor tiles,
  // one box per tile, maps encoded here (bases are known) and uploaded with the tiles
  std::vector<FanTile> tensor_tiles;
  std::vector<CUtensorMap> maps;
  if (cfg_.tensor && (cfg_.kernel == CopyKernel::BulkStrided || cfg_.kernel == CopyKernel::BulkDyn)) {
    std::vector<DevPiece> keep;
    for (const DevPiece& q : fanp) {
      if (!(q.per > 1 && q.rows > 1 && q.src_pitch != q.row_bytes)) {
        keep.push_back(q);
        continue;
      }
      const TensorBox tb = tensor_box(q.row_bytes, q.rows, cfg_.stage_bytes);
      const size_t m0 = maps.size();
      maps.resize(m0 + 1 + q.n_dst);
      encode_map(&maps[m0], q.src, tb, q.rows, q.src_pitch);
      for (uint32_t d = 0; d < q.n_dst; ++d) encode_map(&maps[m0 + 1 + d], q.dst[d], tb, q.rows, q.dst_pitch[d]);
      for (uint32_t r = 0; r < q.rows; r += tb.br)
        for (uint32_t c = 0; c < tb.nch; c += tb.bc) {
          FanTile f{};
          f.src = m0;  // map index until the device address is known
          f.src_pitch = (uint64_t(r) << 32) | c;
          f.rows = 1, f.row_bytes = tb.e * 8 * tb.bc * tb.br, f.n_dst = q.n_dst, f.pad = 1;
          for (uint32_t d = 0; d < q.n_dst; ++d) f.dst[d] = m0 + 1 + d;
          tensor_tiles.push_back(f);
        }
    }
    fanp.swap(keep);
  }
  const uint64_t nf = number(fanp), na = number(alignedp), nm = number(miscp), nl = number(fanlp);
  const uint64_t ntt = tensor_tiles.size();
  if (trace) std::fprintf(stderr, "prepare-trace pieces %.1f ms (%zu pieces -> %llu tiles)\n", ms_since(t_mark), lt.size(),
                          (unsigned long long)(nf + na + nm + nl)), t_mark = clk::now();
  l->chunks.clear();
  l->chunk_pieces.clear();
  const bool one_list = nm == 0 && nl == 0 && ntt == 0 && ((nf == 0) != (na == 0));
  // the host-buffer pipeline's chunks are planned on first use (run_host), not here: they are
  // a per-tile host walk that the device-resident path never needs
  l->chunks_ready = !(host_chunks && ctx_.world() == 1 && one_list);
  if (!l->chunks_ready) l->chunk_pieces = nf ? fanp : alignedp, l->chunk_fan = nf != 0;
  DeviceGuard g(l->dev);
  auto st = static_cast<cudaStream_t>(ctx_.stream(l->world));
  const int sms = ctx_.sm_count(l->world);
  if (l->d_fan) cudaFree(l->d_fan), l->d_fan = nullptr;
  if (l->d_fan_chunks) cudaFree(l->d_fan_chunks), l->d_fan_chunks = nullptr;
  if (l->d_tiles) cudaFree(l->d_tiles), l->d_tiles = nullptr;
  if (l->d_fanl) cudaFree(l->d_fanl), l->d_fanl = nullptr;
  if (l->d_maps) cudaFree(l->d_maps), l->d_maps = nullptr;
  // stream-ordered pool allocations (a plain cudaMalloc after the arenas took 62 ms, r47b)
  auto upload = [&](const std::vector<DevPiece>& v) -> DevPiece* {
    if (v.empty()) return nullptr;
    DevPiece* d = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&d), v.size() * sizeof(DevPiece), st), "cudaMallocAsync pieces");
    ck(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(DevPiece), cudaMemcpyHostToDevice, st), "upload pieces");
    return d;
  };
  DevPiece* dfan = upload(fanp);
  DevPiece* dal = upload(alignedp);
  DevPiece* dmi = upload(miscp);
  DevPiece* dfl = upload(fanlp);
  if (trace) std::fprintf(stderr, "prepare-trace upload %.2f ms\n", ms_since(t_mark)), t_mark = clk::now();
  if (nf + ntt) {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&l->d_fan), (nf + ntt) * sizeof(FanTile), st), "cudaMallocAsync tiles");
    cuda::launch_expand_fan(dfan, uint32_t(fanp.size()), 0, nf, l->d_fan,
                            interleave ? unsigned(cuda::bulk_grid(nf, sms, cfg_)) : 0u, sms, st);
  }
  if (ntt) {  // maps first (their device addresses go into the tiles), then the tiles after the 1-D ones
    ck(cudaMalloc(&l->d_maps, maps.size() * sizeof(CUtensorMap)), "cudaMalloc tensor maps");
    ck(cudaMemcpyAsync(l->d_maps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, st), "maps h2d");
    const uint64_t mb = uint64_t(reinterpret_cast<uintptr_t>(l->d_maps));
    for (FanTile& f : tensor_tiles) {
      f.src = mb + f.src * sizeof(CUtensorMap);
      for (uint32_t d = 0; d < f.n_dst; ++d) f.dst[d] = mb + f.dst[d] * sizeof(CUtensorMap);
    }
    ck(cudaMemcpyAsync(l->d_fan + nf, tensor_tiles.data(), ntt * sizeof(FanTile), cudaMemcpyHostToDevice, st), "tiles h2d");
    ck(cudaStreamSynchronize(st), "tensor tiles");  // the host vector dies with this frame
  }
  if (na + nm) {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&l->d_tiles), (na + nm) * sizeof(CopyTile), st), "cudaMallocAsync tiles");
    cuda::launch_expand_copy(dal, uint32_t(alignedp.size()), na, l->d_tiles, sms, st);
    cuda::launch_expand_copy(dmi, uint32_t(miscp.size()), nm, l->d_tiles + na, sms, st);
  }
  if (nl) {
    ck(cudaMallocAsync(reinterpret_cast<void**>(&l->d_fanl), nl * sizeof(FanTile), st), "cudaMallocAsync tiles");
    cuda::launch_expand_fan(dfl, uint32_t(fanlp.size()), 0, nl, l->d_fanl, 0u, sms, st);
  }
  for (DevPiece* d : {dfan, dal, dmi, dfl})
    if (d) ck(cudaFreeAsync(d, st), "cudaFreeAsync pieces");
  if (trace) std::fprintf(stderr, "prepare-trace alloc+expand launch %.2f ms\n", ms_since(t_mark)), t_mark = clk::now();
  ck(cudaStreamSynchronize(st), "expand schedule");
  if (trace) std::fprintf(stderr, "prepare-trace expand sync %.2f ms\n", ms_since(t_mark));
  l->n_fan = nf + ntt;
  l->n_tensor = ntt;
  l->n_aligned = na;
  l->n_misc = nm;
  l->n_fanl = nl;
  l->bytes = bytes;
  l->read_bytes = read_bytes;
  l->lists[0] = std::move(fanp), l->lists[1] = std::move(alignedp), l->lists[2] = std::move(miscp), l->lists[3] = std::move(fanlp);
  world_chunks_ready_ = false;
}

void Executor::run() {
  TraceRange trace_("Executor::run");
  Local* central = nullptr;
  if (local_.empty()) return;
  auto ws = static_cast<cudaEvent_t>(w_start_), we = static_cast<cudaEvent_t>(w_stop_);
  auto origin = static_cast<cudaStream_t>(ctx_.stream(local_[0]->world));
  {
    DeviceGuard g(local_[0]->dev);
    ck(cudaEventRecord(ws, origin), "cudaEventRecord");
  }
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    auto s = static_cast<cudaStream_t>(ctx_.stream(l->world));
    if (l != local_[0]) ck(cudaStreamWaitEvent(s, ws, 0), "common start");  // every GPU starts at the same mark
    ck(cudaEventRecord(l->start, s), "cudaEventRecord");
    launch_local(*l, s);
    ck(cudaEventRecord(l->stop, s), "cudaEventRecord");
    if (l->phase_b) central = l.get();
  }
  if (central) {  // central mode, phase 2: once every GPU's fetch into the staging region landed
    DeviceGuard g(central->dev);
    auto s = static_cast<cudaStream_t>(ctx_.stream(central->world));
    for (auto& l : local_)
      if (l.get() != central) ck(cudaStreamWaitEvent(s, l->stop, 0), "cudaStreamWaitEvent");
    launch_local(*central->phase_b, s);
    ck(cudaEventRecord(central->stop, s), "cudaEventRecord");
  }
  DeviceGuard g(local_[0]->dev);  // the world is done when the last GPU's kernels (and pushes) are
  for (auto& l : local_)
    if (l != local_[0]) ck(cudaStreamWaitEvent(origin, l->stop, 0), "join");
  ck(cudaEventRecord(we, origin), "cudaEventRecord");
}

std::vector<Timing> Executor::wait() {
  TraceRange trace_("Executor::wait");
  std::vector<Timing> out;
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    ck(cudaEventSynchronize(l->stop), "cudaEventSynchronize");
    Timing t;
    ck(cudaEventElapsedTime(&t.ms, l->start, l->stop), "cudaEventElapsedTime");
    t.tiles = l->tiles();
    t.bytes = l->bytes;
    t.read_bytes = l->read_bytes;
    t.launches = l->launches();
    if (const Local* p = l->phase_b.get()) {
      t.tiles += p->tiles();
      t.bytes += p->bytes, t.read_bytes += p->read_bytes, t.launches += p->launches();
    }
    out.push_back(t);
  }
  if (!local_.empty()) {
    DeviceGuard g(local_[0]->dev);
    ck(cudaEventSynchronize(static_cast<cudaEvent_t>(w_stop_)), "cudaEventSynchronize");
    ck(cudaEventElapsedTime(&world_ms_, static_cast<cudaEvent_t>(w_start_), static_cast<cudaEvent_t>(w_stop_)),
       "cudaEventElapsedTime");
  }
  return out;
}

// End to end over every local GPU from one common start: H2D of each GPU's src arena (all GPUs
// at once), each GPU's kernels as soon as ITS source landed (push: a GPU's tiles read only its
// own src arena), a world barrier (every peer's pushes into a GPU's dst arena are done), D2H
// of each dst arena; the origin stream joins the last D2H.  Host buffers are indexed by world
// GPU (null: not local).
// The world host pipeline's chunks (lazy, first run_host_world): every local GPU's tile lists
// cut into K chunks of equal tile counts (lists are in destination order); per chunk the source
// ranges it first reads (uploaded in chunk order) and, per destination GPU, the lowest offset it
// writes.  After round k (chunk k done on every GPU) a GPU's dst arena is final below the lowest
// offset any later chunk of any GPU writes: that prefix goes down while later rounds run.
bool Executor::plan_world_chunks() {
  world_chunks_ready_ = true;
  world_pipelined_ = false;
  if (central_ >= 0 || cfg_.kernel == CopyKernel::Bulk) return false;  // interleaved tiles: no sub-ranges
  for (auto& l : local_)
    if (l->n_tensor) return false;
  const size_t K = size_t(std::max(1, cfg_.host_chunks / 4));  // rounds
  const int G = ctx_.world();
  // absolute dst address -> (world GPU, arena offset)
  std::vector<std::pair<uint64_t, int>> bases;
  for (int j = 0; j < G; ++j)
    if (dst_base_[size_t(j)] && dst_size_[size_t(j)]) bases.emplace_back(uint64_t(reinterpret_cast<uintptr_t>(dst_base_[size_t(j)])), j);
  std::sort(bases.begin(), bases.end());
  auto locate = [&](uint64_t a, int& j, uint64_t& off) {
    auto it = std::upper_bound(bases.begin(), bases.end(), std::make_pair(a, INT32_MAX));
    if (it == bases.begin()) return false;
    --it;
    j = it->second, off = a - it->first;
    return off < dst_size_[size_t(j)];
  };
  // min_dst[g][j][k]: lowest offset of GPU j's dst arena written by chunk k of local GPU g
  std::vector<std::vector<std::vector<uint64_t>>> min_dst(local_.size(), std::vector<std::vector<uint64_t>>(size_t(G), std::vector<uint64_t>(K, UINT64_MAX)));
  for (size_t li = 0; li < local_.size(); ++li) {
    Local& l = *local_[li];
    l.wchunks.assign(K, {});
    const uint64_t sb = uint64_t(reinterpret_cast<uintptr_t>(src_base_[size_t(l.world)]));
    const uint64_t n[4] = {l.n_fan, l.n_aligned, l.n_misc, l.n_fanl};
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> spans(K);
    for (int i = 0; i < 4; ++i) {
      for (size_t k = 0; k < K; ++k) l.wchunks[k].t0[i] = n[i] * k / K, l.wchunks[k].t1[i] = n[i] * (k + 1) / K;
      uint64_t t = 0;
      size_t k = 0;
      for (const DevPiece& q : l.lists[i]) {
        const uint64_t nt = piece_tile_count(q.rows, q.row_bytes, q.per, q.tile);
        for (uint64_t u = 0; u < nt; ++u, ++t) {
          while (k + 1 < K && t >= l.wchunks[k].t1[i]) ++k;
          uint64_t r0, cc;
          uint32_t nr, nb;
          piece_tile(q.rows, q.row_bytes, q.per, q.tile, u, r0, cc, nr, nb);
          const uint64_t s0 = q.src + r0 * q.src_pitch + cc - sb, s1 = s0 + (nr ? (nr - 1) * q.src_pitch : 0) + nb;
          auto& sv = spans[k];
          if (!sv.empty() && s0 >= sv.back().first && s0 <= sv.back().second) sv.back().second = std::max(sv.back().second, s1);
          else sv.emplace_back(s0, s1);
          for (uint32_t d = 0; d < q.n_dst; ++d) {
            int j;
            uint64_t off;
            if (!locate(q.dst[d] + r0 * q.dst_pitch[d] + cc, j, off)) return false;  // not a dst arena: no pipeline
            uint64_t& m = min_dst[li][size_t(j)][k];
            m = std::min(m, off);
          }
        }
      }
    }
    std::vector<HostChunk> hc(K);
    plan_uploads(hc, spans);
    for (size_t k = 0; k < K; ++k) l.wchunks[k].uploads = std::move(hc[k].uploads);
    while (l.wev.size() < 2 * K) {
      DeviceGuard g(l.dev);
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      l.wev.push_back(e);
    }
  }
  // every destination GPU must be local (the D2H side): single-process worlds only
  for (auto& l : local_) {
    const size_t j = size_t(l->world);
    l->wsafe.assign(K, dst_size_[j]);
    uint64_t m = dst_size_[j];
    for (size_t k = K; k-- > 0;) {
      l->wsafe[k] = m;  // final below m once rounds 0..k are done
      for (size_t li = 0; li < local_.size(); ++li) m = std::min(m, min_dst[li][j][k]);
    }
  }
  world_pipelined_ = true;
  return true;
}

float Executor::run_host_world(const std::vector<const void*>& host_src, const std::vector<void*>& host_dst) {
  TraceRange trace_("Executor::run_host_world");
  // RESHARD_WORLD_PIPELINE=0: the three-phase form below (A/B); default: pipelined rounds
  // whenever every GPU of the world is local and the tile lists can be cut into sub-ranges
  const char* pv = std::getenv("RESHARD_WORLD_PIPELINE");
  if (!(pv && std::string(pv) == "0") && local_.size() == size_t(ctx_.world())) {
    if (!world_chunks_ready_) plan_world_chunks();
    if (world_pipelined_) return run_host_world_pipelined(host_src, host_dst);
  }
  if (local_.empty()) raise(Errc::DeviceUnavailable, "run_host_world: no local GPU");
  if (central_ >= 0) raise(Errc::InvalidArgument, "run_host_world: distributed mode only");
  if (host_src.size() != size_t(ctx_.world()) || host_dst.size() != size_t(ctx_.world()))
    raise(Errc::InvalidArgument, "run_host_world: one host buffer pair per world GPU");
  auto ws = static_cast<cudaEvent_t>(w_start_), we = static_cast<cudaEvent_t>(w_stop_);
  auto origin = static_cast<cudaStream_t>(ctx_.stream(local_[0]->world));
  auto stream_of = [&](const Local& l) { return static_cast<cudaStream_t>(ctx_.stream(l.world)); };
  {
    DeviceGuard g(local_[0]->dev);
    ck(cudaEventRecord(ws, origin), "cudaEventRecord");
  }
  auto barrier = [&](cudaEvent_t Local::*mark) {  // every local stream waits for every other's mark
    for (auto& l : local_) {
      DeviceGuard g(l->dev);
      for (auto& o : local_)
        if (o != l) ck(cudaStreamWaitEvent(stream_of(*l), (*o).*mark, 0), "world barrier");
    }
  };
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    auto s = stream_of(*l);
    const size_t w = size_t(l->world);
    if (l != local_[0]) ck(cudaStreamWaitEvent(s, ws, 0), "common start");
    if (src_size_[w]) {
      if (!host_src[w]) raise(Errc::InvalidArgument, "run_host_world: null host source for a local GPU");
      ck(cudaMemcpyAsync(src_base_[w], host_src[w], src_size_[w], cudaMemcpyHostToDevice, s), "h2d src arena");
    }
    ck(cudaEventRecord(l->e_h2d, s), "cudaEventRecord");
  }
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    launch_local(*l, stream_of(*l));
    ck(cudaEventRecord(l->e_kern, stream_of(*l)), "cudaEventRecord");
  }
  barrier(&Local::e_kern);  // peers' pushes into this GPU's dst arena have landed
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    const size_t w = size_t(l->world);
    if (dst_size_[w]) {
      if (!host_dst[w]) raise(Errc::InvalidArgument, "run_host_world: null host destination for a local GPU");
      ck(cudaMemcpyAsync(host_dst[w], dst_base_[w], dst_size_[w], cudaMemcpyDeviceToHost, stream_of(*l)), "d2h dst arena");
    }
    ck(cudaEventRecord(l->e_d2h, stream_of(*l)), "cudaEventRecord");
  }
  DeviceGuard g(local_[0]->dev);
  for (auto& l : local_)
    if (l != local_[0]) ck(cudaStreamWaitEvent(origin, l->e_d2h, 0), "join");
  ck(cudaEventRecord(we, origin), "cudaEventRecord");
  ck(cudaEventSynchronize(we), "cudaEventSynchronize");
  for (auto& l : local_) {
    DeviceGuard gl(l->dev);
    ck(cudaEventSynchronize(l->e_d2h), "cudaEventSynchronize");
  }
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, ws, we), "cudaEventElapsedTime");
  return ms;
}

// Rounds k = 0..K-1 over every local GPU g: the H2D of the source ranges chunk k of g first
// reads (g's upload stream), chunk k of g's tile lists once they landed (g's stream), then on
// every GPU j's download stream — after chunk k is done on EVERY GPU (cross-device event waits)
// — the D2H of j's dst-arena bytes that no later chunk writes.  H2D, kernels and D2H of
// different rounds overlap on every link; peers' pushes are ordered by the events.
float Executor::run_host_world_pipelined(const std::vector<const void*>& host_src, const std::vector<void*>& host_dst) {
  if (host_src.size() != size_t(ctx_.world()) || host_dst.size() != size_t(ctx_.world()))
    raise(Errc::InvalidArgument, "run_host_world: one host buffer pair per world GPU");
  const size_t K = local_[0]->wchunks.size();
  auto ws = static_cast<cudaEvent_t>(w_start_), we = static_cast<cudaEvent_t>(w_stop_);
  auto origin = static_cast<cudaStream_t>(ctx_.stream(local_[0]->world));
  auto stream_of = [&](const Local& l) { return static_cast<cudaStream_t>(ctx_.stream(l.world)); };
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    if (!l->s_h2d) {
      ck(cudaStreamCreateWithFlags(&l->s_h2d, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&l->s_d2h, cudaStreamNonBlocking), "stream");
    }
    const size_t w = size_t(l->world);
    if (src_size_[w] && !host_src[w]) raise(Errc::InvalidArgument, "run_host_world: null host source for a local GPU");
    if (dst_size_[w] && !host_dst[w]) raise(Errc::InvalidArgument, "run_host_world: null host destination for a local GPU");
  }
  {
    DeviceGuard g(local_[0]->dev);
    ck(cudaEventRecord(ws, origin), "cudaEventRecord");
  }
  for (auto& l : local_) {
    DeviceGuard g(l->dev);
    for (cudaStream_t s : {stream_of(*l), l->s_h2d, l->s_d2h})
      if (s != origin) ck(cudaStreamWaitEvent(s, ws, 0), "common start");
  }
  std::vector<uint64_t> down(local_.size(), 0);
  for (size_t k = 0; k < K; ++k) {
    for (auto& l : local_) {
      DeviceGuard g(l->dev);
      const size_t w = size_t(l->world);
      char* dsrc = static_cast<char*>(src_base_[w]);
      const char* hsrc = static_cast<const char*>(host_src[w]);
      for (auto [off, len] : l->wchunks[k].uploads)
        ck(cudaMemcpyAsync(dsrc + off, hsrc + off, len, cudaMemcpyHostToDevice, l->s_h2d), "h2d piece");
      ck(cudaEventRecord(l->wev[k], l->s_h2d), "event");
      cudaStream_t s = stream_of(*l);
      ck(cudaStreamWaitEvent(s, l->wev[k], 0), "wait h2d");
      const int sms = ctx_.sm_count(l->world);
      const auto& c = l->wchunks[k];
      cuda::launch_bulk(l->d_fan + c.t0[0], c.t1[0] - c.t0[0], cfg_, sms, s, l->d_claim);
      cuda::launch_copy(l->d_tiles + c.t0[1], c.t1[1] - c.t0[1], cfg_, sms, true, s, l->d_claim2);
      cuda::launch_copy(l->d_tiles + l->n_aligned + c.t0[2], c.t1[2] - c.t0[2], cfg_, sms, false, s);
      cuda::launch_copy_fan(l->d_fanl + c.t0[3], c.t1[3] - c.t0[3], cfg_, sms, s, l->d_claim2);
      ck(cudaEventRecord(l->wev[K + k], s), "event");
    }
    for (size_t lj = 0; lj < local_.size(); ++lj) {
      Local& j = *local_[lj];
      DeviceGuard g(j.dev);
      const size_t w = size_t(j.world);
      const uint64_t safe = j.wsafe[k];
      if (safe <= down[lj]) continue;
      for (auto& l : local_) ck(cudaStreamWaitEvent(j.s_d2h, l->wev[K + k], 0), "wait round");
      ck(cudaMemcpyAsync(static_cast<char*>(host_dst[w]) + down[lj], static_cast<char*>(dst_base_[w]) + down[lj], safe - down[lj],
                         cudaMemcpyDeviceToHost, j.s_d2h),
         "d2h piece");
      down[lj] = safe;
    }
  }
  for (size_t lj = 0; lj < local_.size(); ++lj) {  // the tail, and the source bytes no tile reads
    Local& j = *local_[lj];
    DeviceGuard g(j.dev);
    const size_t w = size_t(j.world);
    if (dst_size_[w] > down[lj]) {
      for (auto& l : local_) ck(cudaStreamWaitEvent(j.s_d2h, l->wev[2 * K - 1], 0), "wait last round");
      ck(cudaMemcpyAsync(static_cast<char*>(host_dst[w]) + down[lj], static_cast<char*>(dst_base_[w]) + down[lj],
                         dst_size_[w] - down[lj], cudaMemcpyDeviceToHost, j.s_d2h),
         "d2h tail");
    }
    std::vector<std::pair<uint64_t, uint64_t>> all;
    for (auto& c : j.wchunks)
      for (auto [off, len] : c.uploads) all.emplace_back(off, off + len);
    std::sort(all.begin(), all.end());
    uint64_t cur = 0;
    char* dsrc = static_cast<char*>(src_base_[w]);
    const char* hsrc = static_cast<const char*>(host_src[w]);
    for (auto [a, b] : all) {
      if (a > cur) ck(cudaMemcpyAsync(dsrc + cur, hsrc + cur, a - cur, cudaMemcpyHostToDevice, j.s_h2d), "h2d rest");
      cur = std::max(cur, b);
    }
    if (cur < src_size_[w]) ck(cudaMemcpyAsync(dsrc + cur, hsrc + cur, src_size_[w] - cur, cudaMemcpyHostToDevice, j.s_h2d), "h2d rest");
  }
  DeviceGuard g(local_[0]->dev);
  for (auto& l : local_) {
    for (cudaStream_t s : {l->s_h2d, l->s_d2h, stream_of(*l)}) {
      if (s == origin) continue;
      DeviceGuard gl(l->dev);
      ck(cudaEventRecord(l->e_d2h, s), "event");
      DeviceGuard g0(local_[0]->dev);
      ck(cudaStreamWaitEvent(origin, l->e_d2h, 0), "join");
    }
  }
  ck(cudaEventRecord(we, origin), "cudaEventRecord");
  ck(cudaEventSynchronize(we), "cudaEventSynchronize");
  float ms = 0;
  ck(cudaEventElapsedTime(&ms, ws, we), "cudaEventElapsedTime");
  return ms;
}

void Executor::host_phase(int gpu, int phase, void* host_buf) {
  TraceRange trace_("Executor::host_phase");
  Local* l = nullptr;
  for (auto& x : local_)
    if (x->world == gpu) l = x.get();
  if (!l) raise(Errc::DeviceUnavailable, "host_phase: GPU " + std::to_string(gpu) + " is not local");
  DeviceGuard g(l->dev);
  auto s = static_cast<cudaStream_t>(ctx_.stream(gpu));
  switch (phase) {
    case 0:
      ck(cudaEventRecord(l->start, s), "cudaEventRecord");
      if (src_size_[size_t(gpu)])
        ck(cudaMemcpyAsync(src_base_[size_t(gpu)], host_buf, src_size_[size_t(gpu)], cudaMemcpyHostToDevice, s), "h2d");
      break;
    case 1:
      launch_local(*l, s);
      if (l->phase_b) launch_local(*l->phase_b, s);  // central mode (single-process worlds only)
      break;
    case 2:
      if (dst_size_[size_t(gpu)])
        ck(cudaMemcpyAsync(host_buf, dst_base_[size_t(gpu)], dst_size_[size_t(gpu)], cudaMemcpyDeviceToHost, s), "d2h");
      ck(cudaEventRecord(l->stop, s), "cudaEventRecord");
      break;
    default: raise(Errc::InvalidArgument, "host_phase: phase must be 0, 1 or 2");
  }
  ck(cudaStreamSynchronize(s), "host_phase sync");
}

float Executor::host_elapsed(int gpu) {
  for (auto& x : local_)
    if (x->world == gpu) {
      DeviceGuard g(x->dev);
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, x->start, x->stop), "cudaEventElapsedTime");
      return ms;
    }
  raise(Errc::DeviceUnavailable, "host_elapsed: GPU " + std::to_string(gpu) + " is not local");
}

// Host-buffer pipeline (run_host): chunks of ~bytes / host_chunks in tile order, each with the
// source spans its tiles read and the lowest destination it writes (tile math on the host).
void Executor::plan_host_chunks(Local& local) {
  Local* l = &local;
  l->chunks_ready = true;
  const std::vector<DevPiece>& pv = l->chunk_pieces;
  if (pv.empty()) return;
  const uint64_t sb = uint64_t(reinterpret_cast<uintptr_t>(src_base_[0]));
  const uint64_t db = uint64_t(reinterpret_cast<uintptr_t>(dst_base_[0]));
  // chunks of bytes / host_chunks; RESHARD_HOST_MIN_CHUNK_MIB sets a floor on the chunk size
  // (A/B knob: pinned copies of a few tens of MB lose ~7 % of the bidirectional PCIe rate,
  // profiles/r2_54, but a 44 MiB floor on GPT-2 small's 1.5 GB was within the run-to-run PCIe
  // noise on a same-box A/B, r2_57: 38.3 vs 38.3 ms mean; default: no floor)
  const uint64_t min_chunk = uint64_t(std::max(0, env_int("RESHARD_HOST_MIN_CHUNK_MIB", 0))) << 20;
  const uint64_t target = std::max<uint64_t>({l->bytes / uint64_t(cfg_.host_chunks), min_chunk, 1});
  const uint64_t n = l->chunk_fan ? l->n_fan : l->n_aligned;
  HostChunk c{0, 0, 0, UINT64_MAX, {}};
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> spans(1);
  uint64_t acc = 0, i = 0;
  for (const DevPiece& q : pv) {
    const uint64_t nt = piece_tile_count(q.rows, q.row_bytes, q.per, q.tile);
    for (uint64_t t = 0; t < nt; ++t, ++i) {
      uint64_t r0, cc;
      uint32_t nr, nb;
      piece_tile(q.rows, q.row_bytes, q.per, q.tile, t, r0, cc, nr, nb);
      const uint64_t s0 = q.src + r0 * q.src_pitch + cc - sb, s1 = s0 + (nr ? (nr - 1) * q.src_pitch : 0) + nb;
      auto& sv = spans.back();  // consecutive tiles usually continue the previous source run
      if (!sv.empty() && s0 >= sv.back().first && s0 <= sv.back().second) sv.back().second = std::max(sv.back().second, s1);
      else sv.emplace_back(s0, s1);
      c.src_end = std::max(c.src_end, s1);
      for (uint32_t d = 0; d < q.n_dst; ++d) c.dst_min = std::min(c.dst_min, q.dst[d] + r0 * q.dst_pitch[d] + cc - db);
      acc += uint64_t(nr) * nb * q.n_dst;
      if (acc >= target || i + 1 == n) {
        c.t1 = i + 1;
        l->chunks.push_back(c);
        c = HostChunk{i + 1, 0, 0, UINT64_MAX, {}};
        if (i + 1 < n) spans.emplace_back();
        acc = 0;
      }
    }
  }
  plan_uploads(l->chunks, spans);
  if (l->chunk_fan && cfg_.kernel == CopyKernel::Bulk) {  // each chunk its own launch, interleaved for its grid
    DeviceGuard g(l->dev);
    auto st = static_cast<cudaStream_t>(ctx_.stream(l->world));
    const int sms = ctx_.sm_count(l->world);
    DevPiece* d = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&d), pv.size() * sizeof(DevPiece), st), "cudaMallocAsync pieces");
    ck(cudaMemcpyAsync(d, pv.data(), pv.size() * sizeof(DevPiece), cudaMemcpyHostToDevice, st), "upload pieces");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&l->d_fan_chunks), l->n_fan * sizeof(FanTile), st), "cudaMallocAsync tiles");
    for (const HostChunk& k : l->chunks)
      cuda::launch_expand_fan(d, uint32_t(pv.size()), k.t0, k.t1, l->d_fan_chunks + k.t0,
                              unsigned(cuda::bulk_grid(k.t1 - k.t0, sms, cfg_)), sms, st);
    ck(cudaFreeAsync(d, st), "cudaFreeAsync pieces");
    ck(cudaStreamSynchronize(st), "expand chunks");
  }  // other kernels walk the natural order: the chunks are slices of the tile array
}

uint64_t Executor::host_upload_bytes(int gpu, unsigned flags) {
  Local* l = nullptr;
  for (auto& x : local_)
    if (x->world == gpu) l = x.get();
  if (!l) raise(Errc::DeviceUnavailable, "host_upload_bytes: GPU " + std::to_string(gpu) + " is not local");
  if (ctx_.world() != 1) raise(Errc::InvalidArgument, "host_upload_bytes: single-GPU worlds only");
  if (!l->chunks_ready) plan_host_chunks(*l);
  if (l->chunks.empty() || !(flags & kHostSkipUnread)) return src_size_[size_t(gpu)];
  uint64_t n = 0;
  for (const HostChunk& c : l->chunks)
    for (auto [off, len] : c.uploads) n += len;
  return n;
}

Timing Executor::run_host(int gpu, const void* host_src, void* host_dst, unsigned flags) {
  TraceRange trace_("Executor::run_host");
  Local* l = nullptr;
  for (auto& x : local_)
    if (x->world == gpu) l = x.get();
  if (!l) raise(Errc::DeviceUnavailable, "run_host: GPU " + std::to_string(gpu) + " is not local");
  if (ctx_.world() != 1) raise(Errc::InvalidArgument, "run_host: single-GPU worlds only");
  if (flags & ~kHostSkipUnread) raise(Errc::InvalidArgument, "run_host: unknown flags");
  if (!l->chunks_ready) plan_host_chunks(*l);
  DeviceGuard g(l->dev);
  auto s = static_cast<cudaStream_t>(ctx_.stream(gpu));
  char* dsrc = static_cast<char*>(src_base_[size_t(gpu)]);
  char* ddst = static_cast<char*>(dst_base_[size_t(gpu)]);
  const char* hsrc = static_cast<const char*>(host_src);
  char* hdst = static_cast<char*>(host_dst);
  const uint64_t ssize = src_size_[size_t(gpu)], dsize = dst_size_[size_t(gpu)];
  Timing t;
  t.tiles = l->tiles(), t.bytes = l->bytes, t.read_bytes = l->read_bytes;
  if (l->chunks.empty()) {  // sequential: H2D, kernels, D2H
    ck(cudaEventRecord(l->start, s), "cudaEventRecord");
    ck(cudaMemcpyAsync(dsrc, hsrc, ssize, cudaMemcpyHostToDevice, s), "h2d src arena");
    launch_local(*l, s);
    if (l->phase_b) launch_local(*l->phase_b, s);  // central mode: staging -> destinations
    // the staging region (central mode) sits at the end of the dst arena and is not state
    ck(cudaMemcpyAsync(hdst, ddst, dsize - (l->phase_b ? staging_bytes_ : 0), cudaMemcpyDeviceToHost, s),
       "d2h dst arena");
    t.launches = l->launches() + (l->phase_b ? l->phase_b->launches() : 0);
  } else {
    // Pipelined over destination-ordered chunks: H2D of src pieces (copy engine 1), the
    // chunk's kernel once the src bytes it reads have landed, D2H of the dst bytes that no
    // later chunk writes (below the minimum destination of all later chunks; copy engine 2).
    const size_t K = l->chunks.size();
    if (!l->s_h2d) {
      ck(cudaStreamCreateWithFlags(&l->s_h2d, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&l->s_d2h, cudaStreamNonBlocking), "stream");
    }
    // RESHARD_HOST_TRACE=1 (diagnostic): timing-enabled events and a per-chunk timeline
    // (H2D landed / kernel done / D2H done, ms from the start) on stderr
    const bool trace = std::getenv("RESHARD_HOST_TRACE") && std::string(std::getenv("RESHARD_HOST_TRACE")) == "1";
    if (trace)
      for (auto e : l->ev) cudaEventDestroy(e);
    if (trace) l->ev.clear();
    while (l->ev.size() < 2 * K + 1) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, trace ? cudaEventDefault : cudaEventDisableTiming), "event");
      l->ev.push_back(e);
    }
    std::vector<cudaEvent_t> ed;  // trace: D2H done per chunk
    if (trace)
      for (size_t k = 0; k < K; ++k) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "event");
        ed.push_back(e);
      }
    cudaEvent_t* eh = l->ev.data();
    cudaEvent_t* ec = l->ev.data() + K;
    cudaEvent_t done = l->ev[2 * K];
    std::vector<uint64_t> safe(K);
    uint64_t m = dsize;
    for (size_t k = K; k-- > 0;) {
      safe[k] = m;
      m = std::min(m, l->chunks[k].dst_min);
    }
    ck(cudaEventRecord(l->start, s), "cudaEventRecord");
    ck(cudaStreamWaitEvent(l->s_h2d, l->start, 0), "wait");
    ck(cudaStreamWaitEvent(l->s_d2h, l->start, 0), "wait");
    uint64_t down = 0;
    std::vector<std::pair<uint64_t, uint64_t>> all;
    for (size_t k = 0; k < K; ++k) {
      for (auto [off, len] : l->chunks[k].uploads) {
        ck(cudaMemcpyAsync(dsrc + off, hsrc + off, len, cudaMemcpyHostToDevice, l->s_h2d), "h2d piece");
        all.emplace_back(off, off + len);
      }
      ck(cudaEventRecord(eh[k], l->s_h2d), "event");
    }
    // state no tile reads (kept cells nobody copies) still goes to the device, last — unless
    // the caller keeps it on the host (kHostSkipUnread)
    if (!(flags & kHostSkipUnread)) {
      std::sort(all.begin(), all.end());
      uint64_t cur = 0;
      for (auto [a, b] : all) {
        if (a > cur) ck(cudaMemcpyAsync(dsrc + cur, hsrc + cur, a - cur, cudaMemcpyHostToDevice, l->s_h2d), "h2d rest");
        cur = std::max(cur, b);
      }
      if (cur < ssize) ck(cudaMemcpyAsync(dsrc + cur, hsrc + cur, ssize - cur, cudaMemcpyHostToDevice, l->s_h2d), "h2d rest");
    }
    const int sms = ctx_.sm_count(gpu);
    for (size_t k = 0; k < K; ++k) {
      ck(cudaStreamWaitEvent(s, eh[k], 0), "wait");
      const uint64_t n = l->chunks[k].t1 - l->chunks[k].t0;
      if (l->n_fan)
        cuda::launch_bulk((l->d_fan_chunks ? l->d_fan_chunks : l->d_fan) + l->chunks[k].t0, n, cfg_, sms, s, l->d_claim);
      else cuda::launch_copy(l->d_tiles + l->chunks[k].t0, n, cfg_, sms, true, s, l->d_claim2);
      ck(cudaEventRecord(ec[k], s), "event");
    }
    for (size_t k = 0; k < K; ++k) {
      ck(cudaStreamWaitEvent(l->s_d2h, ec[k], 0), "wait");
      if (safe[k] > down) ck(cudaMemcpyAsync(hdst + down, ddst + down, safe[k] - down, cudaMemcpyDeviceToHost, l->s_d2h), "d2h piece");
      down = std::max(down, safe[k]);
      if (trace) ck(cudaEventRecord(ed[k], l->s_d2h), "event");
    }
    ck(cudaEventRecord(done, l->s_d2h), "event");
    ck(cudaStreamWaitEvent(s, done, 0), "wait");
    ck(cudaEventRecord(done, l->s_h2d), "event");  // the H2D tail must land too
    ck(cudaStreamWaitEvent(s, done, 0), "wait");
    t.launches = K;
    if (trace) {
      ck(cudaEventSynchronize(done), "sync");
      uint64_t up = 0, dn = 0, pieces = 0;
      for (size_t k = 0; k < K; ++k) {
        float a = 0, b = 0, c = 0;
        ck(cudaEventElapsedTime(&a, l->start, eh[k]), "elapsed");
        ck(cudaEventElapsedTime(&b, l->start, ec[k]), "elapsed");
        ck(cudaEventElapsedTime(&c, l->start, ed[k]), "elapsed");
        uint64_t ub = 0;
        for (auto [off, len] : l->chunks[k].uploads) ub += len, ++pieces;
        up += ub;
        std::fprintf(stderr, "host-trace chunk %zu: up %.2f MB (%zu pieces) h2d@%.3f kern@%.3f d2h@%.3f safe %.2f MB\n", k,
                     ub / 1e6, l->chunks[k].uploads.size(), a, b, c, safe[k] / 1e6);
      }
      dn = down;
      std::fprintf(stderr, "host-trace total: %zu chunks, %llu pieces, %.2f GB up in chunks (of %.2f), %.2f GB down\n", K,
                   (unsigned long long)pieces, up / 1e9, ssize / 1e9, dn / 1e9);
      for (auto e : ed) cudaEventDestroy(e);
    }
  }
  ck(cudaEventRecord(l->stop, s), "cudaEventRecord");
  ck(cudaEventSynchronize(l->stop), "cudaEventSynchronize");
  ck(cudaEventElapsedTime(&t.ms, l->start, l->stop), "cudaEventElapsedTime");
  return t;
}

uint64_t Executor::tiles_for(int gpu) const {
  uint64_t n = 0;
  for (auto& x : logical_[size_t(gpu)]) n += x.n_tiles;
  if (gpu == central_)
    for (auto& x : logical_b_) n += x.n_tiles;
  return n;
}
uint64_t Executor::copy_bytes_for(int gpu) const {
  uint64_t n = 0;
  for (auto& x : logical_[size_t(gpu)]) n += uint64_t(x.rows) * x.row_bytes * x.n_dst;
  if (gpu == central_)
    for (auto& x : logical_b_) n += uint64_t(x.rows) * x.row_bytes * x.n_dst;
  return n;
}
std::vector<uint64_t> Executor::bytes_to(int gpu) const {
  std::vector<uint64_t> out(size_t(ctx_.world()), 0);
  auto add = [&](const std::vector<Logical>& v) {
    for (auto& x : v)
      for (uint32_t d = 0; d < x.n_dst; ++d) out[size_t(x.dst_gpu[d])] += uint64_t(x.rows) * x.row_bytes;
  };
  add(logical_[size_t(gpu)]);
  if (gpu == central_) add(logical_b_);
  return out;
}
// A fan-out piece is read once when it is 16-byte aligned (K3 TMA or K2 LDG fan-out tiles, as
// lower_tiles routes it; arenas are 256-byte aligned, so the offsets decide), else once per
// destination (the generic-width kernel).
uint64_t Executor::read_bytes_for(int gpu) const {
  uint64_t n = 0;
  auto add = [&](const Logical& x) {
    uint64_t bits = x.src_off | x.row_bytes | (x.per ? 0 : x.tile) | (x.rows > 1 ? x.src_pitch : 0);
    for (uint32_t d = 0; d < x.n_dst; ++d) bits |= x.dst_off[d] | (x.rows > 1 ? x.dst_pitch[d] : 0);
    n += uint64_t(x.rows) * x.row_bytes * ((bits & 15) == 0 ? 1 : x.n_dst);
  };
  for (auto& x : logical_[size_t(gpu)]) add(x);
  if (gpu == central_)
    for (auto& x : logical_b_) add(x);
  return n;
}

// Upload a batch of payload tasks per local GPU and run K6 (fill) or K7 (verify) in one
// launch each; returns the mismatch count (verify).
uint64_t Executor::payload_pass(const std::vector<std::vector<cuda::PayloadTask>>& per_local, bool verify) {
  TraceRange trace_("Executor::payload_pass");
  uint64_t bad = 0;
  for (size_t li = 0; li < local_.size(); ++li) {
    Local& l = *local_[li];
    const auto& tasks = per_local[li];
    DeviceGuard g(l.dev);
    auto s = static_cast<cudaStream_t>(ctx_.stream(l.world));
    if (tasks.empty()) continue;
    uint64_t max_bytes = 0;
    for (auto& t : tasks) max_bytes = std::max(max_bytes, t.g.bytes);
    cuda::PayloadTask* d = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&d), tasks.size() * sizeof(cuda::PayloadTask), s), "cudaMallocAsync");
    ck(cudaMemcpyAsync(d, tasks.data(), tasks.size() * sizeof(cuda::PayloadTask), cudaMemcpyHostToDevice, s), "tasks h2d");
    if (verify) ck(cudaMemsetAsync(l.d_count, 0, sizeof(unsigned long long), s), "memset");
    cuda::launch_payload(d, tasks.size(), max_bytes, verify, l.d_count, s);
    ck(cudaFreeAsync(d, s), "cudaFreeAsync");
    unsigned long long h = 0;
    if (verify) ck(cudaMemcpyAsync(&h, l.d_count, sizeof(h), cudaMemcpyDeviceToHost, s), "count d2h");
    ck(cudaStreamSynchronize(s), "payload sync");
    bad += h;
  }
  return bad;
}

void Executor::fill_sources() {
  const PTC& a = *plan_->from;
  std::vector<std::vector<cuda::PayloadTask>> per(local_.size());
  size_t k = 0;
  for (uint32_t i = 0; i < a.devices.size(); ++i)
    for (auto [t, c] : hosted_subtensors(a, a.devices[i])) {
      const CellBinding& b = src_bind_[k++];
      const int li = ctx_.local_of(b.gpu);
      if (li < 0) continue;
      const TensorSpec& e = a.catalog.tensors[t];
      per[size_t(li)].push_back({static_cast<char*>(src_base_[size_t(b.gpu)]) + b.offset, payload_seed(e.path),
                                 cuda::make_geom(e.shape, dtype_width(e.dtype), a.cells[t][c])});
    }
  payload_pass(per, false);
}

uint64_t Executor::verify_destinations() {
  const PTC& b = *plan_->to;
  std::vector<std::vector<cuda::PayloadTask>> per(local_.size());
  for (size_t j = 0; j < plan_->dst_cells.size(); ++j) {
    const CellBinding& bd = dst_bind_[j];
    const int li = ctx_.local_of(bd.gpu);
    if (li < 0) continue;
    const PlanDstCell& dc = plan_->dst_cells[j];
    const TensorSpec& e = b.catalog.tensors[dc.tensor];
    char* base = static_cast<char*>(bd.arena == 0 ? src_base_[size_t(bd.gpu)] : dst_base_[size_t(bd.gpu)]);
    per[size_t(li)].push_back({base + bd.offset, payload_seed(e.path),
                               cuda::make_geom(e.shape, dtype_width(e.dtype), b.cells[dc.tensor][dc.cell])});
  }
  return payload_pass(per, true);
}

// ---- ExecutionReport verification digests ---------------------------------------
// Per base tensor of this executor's window: FNV-1a-64 (proj/include/reshard/util/hash.hpp:13-42)
// of the base tensor reassembled from one replica of each cell of the chosen side (0: the
// source layout's cells, 1: the destination layout's).  Each cell comes back with one strided
// D2H straight into its place in the reassembled tensor (cudaMemcpy2D per outer index);
// tensors are hashed by a pool of host threads.  FNV-1a is byte-sequential, so this stays off
// the clock.  A tensor some cell of which is not held by a local GPU gets no digest (ok = 0).
std::vector<Executor::Digest> Executor::digests(int side, int replica) {
  TraceRange trace_("Executor::digests");
  const PTC& p = side == 0 ? *plan_->from : *plan_->to;
  const size_t nt = p.catalog.tensors.size();
  // one binding per (tensor, cell): the `replica`-th local replica in layout order (the last
  // one when the cell has fewer; replica < 0 counts from the end)
  std::vector<std::vector<std::vector<const CellBinding*>>> reps(nt);
  for (size_t t = 0; t < nt; ++t) reps[t].resize(p.cells[t].size());
  auto offer = [&](uint32_t t, uint32_t c, const CellBinding& b) {
    if (b.gpu >= 0 && ctx_.local_of(b.gpu) >= 0) reps[t][c].push_back(&b);
  };
  if (side == 0) {
    size_t k = 0;
    for (uint32_t i = 0; i < p.devices.size(); ++i)
      for (auto [t, c] : hosted_subtensors(p, p.devices[i])) offer(t, c, src_bind_[k++]);
  } else {
    for (size_t j = 0; j < plan_->dst_cells.size(); ++j) offer(plan_->dst_cells[j].tensor, plan_->dst_cells[j].cell, dst_bind_[j]);
  }
  std::vector<std::vector<const CellBinding*>> pick(nt);
  for (size_t t = 0; t < nt; ++t)
    for (auto& v : reps[t]) {
      const long n = long(v.size());
      const long r = replica >= 0 ? std::min<long>(replica, n - 1) : std::max<long>(0, n + replica);
      pick[t].push_back(n ? v[size_t(r)] : nullptr);
    }
  std::vector<Digest> out;
  for (uint32_t t = t_begin_; t < std::min<uint32_t>(t_end_, uint32_t(nt)); ++t) out.push_back(Digest{t, 0, 0});
  std::atomic<size_t> next{0};
  std::vector<std::exception_ptr> err;
  std::mutex em;
  auto work = [&] {
    try {
      std::vector<uint8_t> buf;
      for (size_t i; (i = next.fetch_add(1)) < out.size();) {
        const uint32_t t = out[i].tensor;
        const TensorSpec& e = p.catalog.tensors[t];
        const uint64_t w = dtype_width(e.dtype);
        const Shape& shape = e.shape;
        bool all = true;
        for (auto* b : pick[t]) all &= b != nullptr;
        if (!all) continue;
        buf.assign(shape_elements(shape) * w, 0);
        for (size_t c = 0; c < p.cells[t].size(); ++c) {
          const CellBinding& b = *pick[t][c];
          DeviceGuard g(ctx_.cuda_device(b.gpu));
          const char* dev = static_cast<const char*>(b.arena == 0 ? src_base_[size_t(b.gpu)] : dst_base_[size_t(b.gpu)]) + b.offset;
          const Range& box = p.cells[t][c];
          Shape lo, ext = box.extents();
          for (int d = 0; d < box.rank(); ++d) lo.push_back(box.dim(d).lo);
          lower_box(ext, Shape(ext.size(), 0), ext, lo, shape, w, uint64_t(1) << 30,
                    [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run) {
                      ck(cudaMemcpy2D(buf.data() + dof, rows > 1 ? dp : run, dev + so, rows > 1 ? sp : run, run, rows,
                                      cudaMemcpyDeviceToHost),
                         "digest d2h");
                    });
        }
        out[i].fnv = fnv1a64(buf.data(), buf.size());
        out[i].ok = 1;
      }
    } catch (...) {
      std::lock_guard<std::mutex> g(em);
      err.push_back(std::current_exception());
    }
  };
  const size_t workers = std::max<size_t>(1, std::min<size_t>({out.size(), 16, std::max(1u, std::thread::hardware_concurrency())}));
  std::vector<std::thread> th;
  for (size_t k = 1; k < workers; ++k) th.emplace_back(work);
  work();
  for (auto& x : th) x.join();
  if (!err.empty()) std::rethrow_exception(err.front());
  return out;
}

// ---- broadcast (fan-out push) ----------------------------------------------------------------
Timing broadcast(Context& ctx, int gpu, const void* src, const std::vector<void*>& dsts, uint64_t bytes) {
  TraceRange trace_("broadcast");
  if (!src) raise(Errc::InvalidArgument, "broadcast: null source");
  if (dsts.empty()) raise(Errc::InvalidArgument, "broadcast: no destinations");
  for (void* d : dsts)
    if (!d) raise(Errc::InvalidArgument, "broadcast: null destination");
  const CopyConfig cfg = CopyConfig::from_env();
  DeviceGuard g(ctx.cuda_device(gpu));
  auto s = static_cast<cudaStream_t>(ctx.stream(gpu));
  const int sms = ctx.sm_count(gpu);
  uint64_t bits = reinterpret_cast<uintptr_t>(src) | bytes;
  for (void* d : dsts) bits |= reinterpret_cast<uintptr_t>(d);
  const bool bulk = is_bulk(cfg.kernel) && (bits & 15) == 0;
  const uint32_t tile = bulk ? cfg.stage_bytes / 16 * 16 : 256u << 10;
  Timing t;
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  if (bytes == 0) {
    t.ms = 0;
  } else if (bulk) {
    std::vector<DevPiece> pieces;
    for (size_t i = 0; i < dsts.size(); i += kMaxFan) {
      DevPiece q{};
      q.src = reinterpret_cast<uintptr_t>(src), q.row_bytes = bytes, q.rows = 1, q.per = 0, q.tile = tile;
      for (size_t d = i; d < dsts.size() && d < i + kMaxFan; ++d) q.dst[q.n_dst++] = reinterpret_cast<uintptr_t>(dsts[d]);
      q.first = uint64_t(pieces.size()) * piece_tile_count(1, bytes, 0, tile);
      pieces.push_back(q);
    }
    const uint64_t n = uint64_t(pieces.size()) * piece_tile_count(1, bytes, 0, tile);
    DevPiece* dp = nullptr;
    FanTile* dt = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dp), pieces.size() * sizeof(DevPiece), s), "cudaMallocAsync");
    ck(cudaMemcpyAsync(dp, pieces.data(), pieces.size() * sizeof(DevPiece), cudaMemcpyHostToDevice, s), "pieces h2d");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dt), n * sizeof(FanTile), s), "cudaMallocAsync");
    const bool interleave = cfg.kernel == CopyKernel::Bulk;
    cuda::launch_expand_fan(dp, uint32_t(pieces.size()), 0, n, dt, interleave ? unsigned(cuda::bulk_grid(n, sms, cfg)) : 0u,
                            sms, s);
    unsigned long long* claim = nullptr;  // bulk_dyn's counter
    ck(cudaMallocAsync(reinterpret_cast<void**>(&claim), 2 * sizeof(unsigned long long), s), "cudaMallocAsync");
    ck(cudaMemsetAsync(claim, 0, 2 * sizeof(unsigned long long), s), "memset claim");
    ck(cudaEventRecord(e0, s), "event");
    cuda::launch_bulk(dt, n, cfg, sms, s, claim);
    ck(cudaEventRecord(e1, s), "event");
    ck(cudaFreeAsync(claim, s), "cudaFreeAsync");
    ck(cudaFreeAsync(dp, s), "cudaFreeAsync");
    ck(cudaFreeAsync(dt, s), "cudaFreeAsync");
    t.tiles = n, t.launches = 1, t.read_bytes = bytes * pieces.size();
  } else {
    std::vector<CopyTile> tiles;
    for (void* d : dsts)
      for (uint64_t c = 0; c < bytes; c += tile)
        tiles.push_back(CopyTile{uint64_t(reinterpret_cast<uintptr_t>(src)) + c, uint64_t(reinterpret_cast<uintptr_t>(d)) + c,
                                 0, 0, 1, uint32_t(std::min<uint64_t>(tile, bytes - c))});
    CopyTile* dt = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dt), tiles.size() * sizeof(CopyTile), s), "cudaMallocAsync");
    ck(cudaMemcpyAsync(dt, tiles.data(), tiles.size() * sizeof(CopyTile), cudaMemcpyHostToDevice, s), "tiles h2d");
    ck(cudaEventRecord(e0, s), "event");
    cuda::launch_copy(dt, tiles.size(), cfg, sms, false, s);
    ck(cudaEventRecord(e1, s), "event");
    ck(cudaFreeAsync(dt, s), "cudaFreeAsync");
    t.tiles = tiles.size(), t.launches = 1, t.read_bytes = bytes * dsts.size();
  }
  if (bytes) {
    ck(cudaEventSynchronize(e1), "sync");
    ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ck(cudaStreamSynchronize(s), "broadcast sync");
  t.bytes = bytes * dsts.size();
  return t;
}

// ---- device slice / merge ----------------------------------------------------------------
namespace {
void run_tiles_once(Context& ctx, int gpu, const std::vector<CopyTile>& tiles) {
  if (tiles.empty()) return;
  DeviceGuard g(ctx.cuda_device(gpu));
  auto s = static_cast<cudaStream_t>(ctx.stream(gpu));
  CopyTile* d = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d), tiles.size() * sizeof(CopyTile), s), "cudaMallocAsync");
  ck(cudaMemcpyAsync(d, tiles.data(), tiles.size() * sizeof(CopyTile), cudaMemcpyHostToDevice, s), "tiles h2d");
  cuda::launch_copy(d, tiles.size(), CopyConfig{}, ctx.sm_count(gpu), false, s);
  ck(cudaFreeAsync(d, s), "cudaFreeAsync");
  ck(cudaStreamSynchronize(s), "slice/merge sync");
}
void append_box(std::vector<CopyTile>& tiles, const char* src, char* dst, const Shape& ext, const Shape& sl, const Shape& ss,
                const Shape& dl, const Shape& ds, uint64_t w) {
  lower_box(ext, sl, ss, dl, ds, w, 256 << 10, [&](uint64_t so, uint64_t dof, uint64_t sp, uint64_t dp, uint64_t rows, uint64_t run) {
    tiles.push_back(CopyTile{uint64_t(reinterpret_cast<uintptr_t>(src + so)), uint64_t(reinterpret_cast<uintptr_t>(dst + dof)), sp, dp,
                             uint32_t(rows), uint32_t(run)});
  });
}
}  // namespace

void device_slice(Context& ctx, int gpu, const DeviceTensorView& t, const Range& r, void* out) {
  for (auto e : t.shape)
    if (e == 0) raise(Errc::InvalidTensor, "zero extent");
  const uint64_t w = dtype_width(t.dtype);
  r.check_against(t.shape);
  Shape lo;
  for (int d = 0; d < r.rank(); ++d) lo.push_back(r.dim(d).lo);
  std::vector<CopyTile> tiles;
  append_box(tiles, static_cast<const char*>(t.data), static_cast<char*>(out), r.extents(), lo, t.shape,
             Shape(lo.size(), 0), r.extents(), w);
  run_tiles_once(ctx, gpu, tiles);
}

void validate_merge(const std::vector<MergePartSpec>& parts, const Shape& target) {
  // validation order of the reference merge (tensor.cpp:81-98)
  if (parts.empty()) raise(Errc::TilingGap, "no parts");
  const Dtype dt = parts.front().dtype;
  uint64_t covered = 0;
  for (const MergePartSpec& p : parts) {
    p.range->check_against(target);
    if (p.dtype != dt) raise(Errc::DtypeMismatch, "parts disagree on dtype");
    if (*p.shape != p.range->extents()) raise(Errc::ShapeMismatch, "part shape does not match its range " + p.range->to_string());
    covered += p.range->elements();
  }
  for (size_t i = 0; i < parts.size(); ++i)
    for (size_t j = i + 1; j < parts.size(); ++j)
      if (parts[i].range->overlaps(*parts[j].range))
        raise(Errc::TilingOverlap, parts[i].range->to_string() + " overlaps " + parts[j].range->to_string());
  if (covered != shape_elements(target))
    raise(Errc::TilingGap, "parts cover " + std::to_string(covered) + " of " + std::to_string(shape_elements(target)) + " elements");
  for (auto e : target)
    if (e == 0) raise(Errc::InvalidTensor, "zero extent");
}

void device_merge(Context& ctx, int gpu, const std::vector<std::pair<Range, DeviceTensorView>>& parts, const Shape& target,
                  void* out) {
  std::vector<MergePartSpec> spec;
  spec.reserve(parts.size());
  for (const auto& [r, p] : parts) spec.push_back({&r, p.dtype, &p.shape});
  validate_merge(spec, target);
  const Dtype dt = parts.front().second.dtype;
  const uint64_t w = dtype_width(dt);
  std::vector<CopyTile> tiles;
  for (const auto& [r, p] : parts) {
    Shape lo;
    for (int d = 0; d < r.rank(); ++d) lo.push_back(r.dim(d).lo);
    append_box(tiles, static_cast<const char*>(p.data), static_cast<char*>(out), r.extents(), Shape(lo.size(), 0), r.extents(),
               lo, target, w);
  }
  run_tiles_once(ctx, gpu, tiles);
}

}  // namespace reshard
