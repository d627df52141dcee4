// sm_100a kernels of the reshard data plane.
//
//  K1/K2 copy_tiles  — persistent strided sub-tensor copy.  Replaces the reference row walker
//                      (proj/src/tensor/tensor.cpp:35-57) and the memcpy loops of slice()
//                      (:73-76) and merge() (:108-111).  One CTA per tile at a time; a tile is
//                      rows x row_bytes with independent src/dst pitches, moved with the
//                      widest common alignment (16 B vectors for every GPT-catalog tile).
//                      Loads are non-coherent streaming loads (L1 no-allocate, 256 B L2
//                      prefetch); a tile whose dst is a peer mapping stores over NVLink (K2).
//  K2 fan-out       — copy_fan_v16_kernel: a DP-replicated fragment read once, stored to every
//                      destination (local and peer) — the multi-GPU fan-out default.
//  K6 fill_cell      — counter-based splitmix64 payload (proj/include/reshard/util/hash.hpp:46-51)
//                      for any sub-box of a base tensor, bit-identical to the CPU stream.
//  K7 verify_cell    — regenerates K6's bytes and counts mismatches (off the clock).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "cuda/kernels.hpp"

namespace reshard::cuda {

namespace {

struct DevTile {
  unsigned long long src, dst, src_pitch, dst_pitch;
  unsigned rows, row_bytes;
};
static_assert(sizeof(DevTile) == sizeof(CopyTile), "tile layout");

template <typename V>
__device__ __forceinline__ V ld_nc(const V* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ uint4 ld_nc<uint4>(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
template <typename V>
__device__ __forceinline__ void st_na(V* p, const V& v) {
  *p = v;
}
template <>
__device__ __forceinline__ void st_na<uint4>(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Copy one tile with vectors of type V.  Thread i of the CTA handles vectors i, i+B, ...
// of the flattened rows x (row_bytes/W) index space.  Byte offsets inside the tile are
// 32-bit (the host keeps (rows-1)*pitch + row_bytes < 2^31) and advance incrementally:
// +step per B vectors, +wrap when the column wraps into the next row, so there is no
// per-vector division or 64-bit multiply.  U vectors are loaded before any is stored.
template <typename V, int U>
__device__ __forceinline__ void copy_tile(const DevTile& t) {
  constexpr unsigned W = sizeof(V);
  const unsigned vpr = t.row_bytes / W;
  const unsigned n = t.rows * vpr;
  const unsigned B = blockDim.x;
  const unsigned drow = B / vpr, dcol = B % vpr;
  const unsigned sp = unsigned(t.src_pitch), dp = unsigned(t.dst_pitch);
  const unsigned s_step = drow * sp + dcol * W, s_wrap = sp - vpr * W;
  const unsigned d_step = drow * dp + dcol * W, d_wrap = dp - vpr * W;
  unsigned col = threadIdx.x % vpr;
  unsigned so = (threadIdx.x / vpr) * sp + col * W, doff = (threadIdx.x / vpr) * dp + col * W;
  const char* s = reinterpret_cast<const char*>(t.src);
  char* d = reinterpret_cast<char*>(t.dst);
  for (unsigned i = threadIdx.x; i < n; i += U * B) {
    V v[U];
    const unsigned col0 = col;  // the store pass replays the column walk from here
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * B < n) v[u] = ld_nc(reinterpret_cast<const V*>(s + so));
      col += dcol, so += s_step;
      if (col >= vpr) col -= vpr, so += s_wrap;
    }
    unsigned c = col0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * B < n) st_na(reinterpret_cast<V*>(d + doff), v[u]);
      c += dcol, doff += d_step;
      if (c >= vpr) c -= vpr, doff += d_wrap;
    }
  }
}

// Tile schedule of the persistent LDG/STG kernels: the static grid-stride order (claim null),
// or dynamic claims of 2 tiles from a global counter — thread 0 issues the next claim while
// the CTA copies the current tiles, so the atomic's latency hides behind them; the last CTA
// out resets the counter for the next launch on the stream (the drift argument of
// copy_bulk_dyn_kernel, for the peer-push kernels).
template <bool DYN, class F>
__device__ __forceinline__ void for_each_tile(unsigned long long n, unsigned long long* claim, F&& f) {
  if (!DYN) {
    for (unsigned long long k = blockIdx.x; k < n; k += gridDim.x) f(k);
    return;
  }
  constexpr unsigned long long B = 2;
  __shared__ unsigned long long s_base[2];
  if (threadIdx.x == 0) s_base[0] = atomicAdd(claim, B);
  __syncthreads();
  int buf = 0;
  for (;;) {
    const unsigned long long base = s_base[buf];
    if (base >= n) break;
    unsigned long long nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(claim, B);
    for (unsigned long long k = base; k < base + B && k < n; ++k) f(k);
    if (threadIdx.x == 0) s_base[buf ^ 1] = nxt;
    __syncthreads();
    buf ^= 1;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(claim + 1, 1ull) == gridDim.x - 1) {
      claim[0] = 0, claim[1] = 0;
      __threadfence();
    }
  }
}

// K1 fast path: every tile 16-byte aligned (the host routes the others to copy_any_kernel).
// Only the uint4 path is instantiated, so register use stays low enough for MINB CTAs/SM.
template <int U, int MINB, bool DYN>
__global__ void __launch_bounds__(512, MINB) copy_v16_kernel(const DevTile* __restrict__ tiles, unsigned long long n,
                                                            unsigned long long* claim) {
  for_each_tile<DYN>(n, claim, [&](unsigned long long k) {
    const DevTile t = tiles[k];
    copy_tile<uint4, U>(t);
  });
}

// K1 general path: widest common alignment per tile.
__global__ void __launch_bounds__(256) copy_any_kernel(const DevTile* __restrict__ tiles, unsigned long long n) {
  for (unsigned long long k = blockIdx.x; k < n; k += gridDim.x) {
    const DevTile t = tiles[k];
    if (t.rows == 0 || t.row_bytes == 0) continue;
    const unsigned long long a = t.src | t.dst | t.row_bytes | (t.rows > 1 ? (t.src_pitch | t.dst_pitch) : 0ull);
    if ((a & 15) == 0) copy_tile<uint4, 4>(t);
    else if ((a & 7) == 0) copy_tile<uint2, 4>(t);
    else if ((a & 3) == 0) copy_tile<unsigned, 4>(t);
    else if ((a & 1) == 0) copy_tile<unsigned short, 4>(t);
    else copy_tile<unsigned char, 4>(t);
  }
}

// K2 fan-out: one source box read ONCE (16-byte LDG) and stored to each of its n_dst
// destinations (STG; local HBM or peer memory over NVLink).  The multi-GPU default for DP
// replicas whose destinations include a peer: every source byte crosses HBM once however many
// replicas it feeds.  Same incremental 32-bit offset walk as copy_tile, one walk per
// destination on the store side (each destination has its own pitch).
struct DevFanTileL {
  unsigned long long src, src_pitch;
  unsigned rows, row_bytes, n_dst, pad;
  unsigned long long dst[kMaxFan];
  unsigned long long dst_pitch[kMaxFan];
};
static_assert(sizeof(DevFanTileL) == sizeof(FanTile), "fan tile layout");

template <int U>
__device__ __forceinline__ void copy_fan_tile(const DevFanTileL& t) {
  constexpr unsigned W = 16;
  const unsigned vpr = t.row_bytes / W;
  const unsigned n = t.rows * vpr;
  const unsigned B = blockDim.x;
  const unsigned drow = B / vpr, dcol = B % vpr;
  const unsigned sp = unsigned(t.src_pitch);
  const unsigned s_step = drow * sp + dcol * W, s_wrap = sp - vpr * W;
  const unsigned nd = t.n_dst;
  unsigned col = threadIdx.x % vpr;
  unsigned so = (threadIdx.x / vpr) * sp + col * W;
  unsigned doff[kMaxFan];
#pragma unroll
  for (int d = 0; d < kMaxFan; ++d) doff[d] = (threadIdx.x / vpr) * unsigned(t.dst_pitch[d]) + col * W;
  const char* s = reinterpret_cast<const char*>(t.src);
  for (unsigned i = threadIdx.x; i < n; i += U * B) {
    uint4 v[U];
    const unsigned col0 = col;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * B < n) v[u] = ld_nc(reinterpret_cast<const uint4*>(s + so));
      col += dcol, so += s_step;
      if (col >= vpr) col -= vpr, so += s_wrap;
    }
#pragma unroll
    for (int d = 0; d < kMaxFan; ++d) {
      if (d >= int(nd)) break;
      char* dd = reinterpret_cast<char*>(t.dst[d]);
      const unsigned dp = unsigned(t.dst_pitch[d]);
      const unsigned d_step = drow * dp + dcol * W, d_wrap = dp - vpr * W;
      unsigned c = col0, o = doff[d];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u * B < n) st_na(reinterpret_cast<uint4*>(dd + o), v[u]);
        c += dcol, o += d_step;
        if (c >= vpr) c -= vpr, o += d_wrap;
      }
      doff[d] = o;
    }
  }
}

template <bool DYN>
__global__ void __launch_bounds__(512, 2) copy_fan_v16_kernel(const DevFanTileL* __restrict__ tiles, unsigned long long n,
                                                             unsigned long long* claim) {
  for_each_tile<DYN>(n, claim, [&](unsigned long long k) {
    const DevFanTileL t = tiles[k];
    copy_fan_tile<4>(t);
  });
}

// ---- K3: TMA bulk-copy pipeline ------------------------------------------------------------
// One elected thread per CTA streams its tiles through a ring of shared-memory stages:
//   cp.async.bulk (global -> smem, completion on a per-stage mbarrier)   one op per row
//   cp.async.bulk (smem -> global, bulk_group)                           one op per row
// Loads run `stages-2` chunks ahead of stores; a stage is refilled only once the bulk store
// that read it has finished reading (cp.async.bulk.wait_group.read).  Tiles are sized by
// the host to fit one stage and are 16-byte aligned (bulk-copy requirement).  SM threads
// do no data movement at all: the TMA engine moves every byte (SASS: UBLKCP).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst_smem, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_smem),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, unsigned src_smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
               : "memory");
}
// The same copies with an L2 cache policy (bulk_*_hint): HINT bit 0 = loads evict_first,
// bit 1 = stores evict_first (the state streams through once; RESHARD_BULK_HINT A/B).
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(unsigned dst_smem, const void* src, unsigned bytes, unsigned bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst_smem),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, unsigned src_smem, unsigned bytes, unsigned long long pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst), "r"(src_smem),
               "r"(bytes), "l"(pol)
               : "memory");
}
// K3T: TMA tensor copies of one 3-D box (dims {e x 8-byte words, chunks, rows}) between a
// tensor map's region and a shared-memory stage — ONE instruction per box instead of one bulk
// copy per row (strided 2-D TP fragments).  The map pointer is a global-memory CUtensorMap.
__device__ __forceinline__ void tma_load_3d(unsigned dst_smem, unsigned long long map, unsigned c1, unsigned c2,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst_smem),
      "l"(map), "r"(0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(unsigned long long map, unsigned c1, unsigned c2, unsigned src_smem) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(map), "r"(0),
               "r"(c1), "r"(c2), "r"(src_smem)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int kBulkMaxStages = 16;

// FanTile: one source box read ONCE into shared memory and stored to up to kMaxFan
// destinations (DP replicas of the same fragment: the same source bytes feed several new
// cells, e.g. GPT-3 6.7B (4,2,1)->(2,2,2) where every TP4 fragment goes to both dp
// replicas).  Saves one HBM read per extra replica (and one NVLink read when remote).
struct DevFanTile {
  unsigned long long src, src_pitch;
  unsigned rows, row_bytes, n_dst, pad;
  unsigned long long dst[kMaxFan];
  unsigned long long dst_pitch[kMaxFan];
};
static_assert(sizeof(DevFanTile) == sizeof(FanTile), "fan tile layout");

// Descriptors are themselves streamed by the TMA engine: each CTA owns a contiguous run of
// tiles and pulls them 32 at a time (3 KiB bulk copies) into a 2-slot shared-memory ring,
// so the issuing thread never waits on a global load of a descriptor (profiles/r05: 65% of
// stall samples were descriptor loads when each tile was read from global on demand).
constexpr int kDescBatch = 32;
constexpr size_t kDescRingBytes = 2 * kDescBatch * sizeof(DevFanTile);

__global__ void __launch_bounds__(32, 1) copy_bulk_kernel(const DevFanTile* __restrict__ tiles, unsigned long long n,
                                                          int stages, unsigned stage_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[kBulkMaxStages];
  __shared__ __align__(8) unsigned long long dbars[2];
  if (threadIdx.x != 0) return;
  DevFanTile* desc = reinterpret_cast<DevFanTile*>(smem + size_t(stages) * stage_bytes);
  for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), 1);
  mbar_init(smem_u32(&dbars[0]), 1);
  mbar_init(smem_u32(&dbars[1]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  // my tiles: a contiguous run [t0, t0 + mine); CTAs below n % grid take one extra.  The
  // host stores CTA c's run as the original tiles c, c + grid, c + 2 grid, ... (see
  // interleave_for_grid), so descriptors are contiguous per CTA while the CTAs still sweep
  // memory together as one window (r06: a plain blocked split lost 10% of bandwidth).
  const unsigned long long q = n / gridDim.x, rem = n % gridDim.x, c = blockIdx.x;
  const unsigned long long t0 = c * q + (c < rem ? c : rem), mine = q + (c < rem ? 1 : 0);
  const unsigned long long batches = (mine + kDescBatch - 1) / kDescBatch;
  auto fetch_batch = [&](unsigned long long b) {
    const unsigned cnt = unsigned(min((unsigned long long)kDescBatch, mine - b * kDescBatch));
    const unsigned bar = smem_u32(&dbars[b & 1]);
    mbar_expect_tx(bar, cnt * unsigned(sizeof(DevFanTile)));
    bulk_g2s(smem_u32(desc + (b & 1) * kDescBatch), tiles + t0 + b * kDescBatch, cnt * unsigned(sizeof(DevFanTile)), bar);
  };
  if (batches > 0) fetch_batch(0);
  if (batches > 1) fetch_batch(1);
  unsigned long long waited = ~0ull;  // last descriptor batch known to have landed
  auto D = [&](unsigned long long i) -> const DevFanTile& {
    const unsigned long long b = i / kDescBatch;
    if (waited == ~0ull || b > waited) {
      mbar_wait(smem_u32(&dbars[b & 1]), unsigned((b >> 1) & 1));
      waited = b;
    }
    return desc[(b & 1) * kDescBatch + (i % kDescBatch)];
  };

  const int ahead = stages > 2 ? stages - 2 : 1;
  int s_load = 0;                // stage of the next load
  int s_store = 0;               // stage of the next store
  unsigned phase = 0;            // parity of the store side's next wait
  auto issue_load = [&](unsigned long long i) {
    const DevFanTile& t = D(i);
    const unsigned rows = t.rows, rb = t.row_bytes;
    const char* src = reinterpret_cast<const char*>(t.src);
    const unsigned long long sp = t.src_pitch;
    const unsigned bar = smem_u32(&bars[s_load]);
    const unsigned base = smem_u32(smem + size_t(s_load) * stage_bytes);
    mbar_expect_tx(bar, rows * rb);
    for (unsigned r = 0; r < rows; ++r) bulk_g2s(base + r * rb, src + r * sp, rb, bar);
    if (++s_load == stages) s_load = 0;
  };
  for (unsigned long long i = 0; i < mine && i < (unsigned long long)ahead; ++i) issue_load(i);
  for (unsigned long long i = 0; i < mine; ++i) {
    const unsigned long long j = i + ahead;
    if (j < mine) {
      // stage of chunk j was last read by the store of chunk j - stages (<= i - 2): allow
      // the most recent store group (chunk i - 1) to still be reading.
      bulk_wait_read<1>();
      issue_load(j);
    }
    const DevFanTile& t = D(i);
    const unsigned rows = t.rows, rb = t.row_bytes, nd = t.n_dst;
    mbar_wait(smem_u32(&bars[s_store]), phase);
    const unsigned base = smem_u32(smem + size_t(s_store) * stage_bytes);
    for (unsigned d = 0; d < nd; ++d) {
      char* dst = reinterpret_cast<char*>(t.dst[d]);
      const unsigned long long dp = t.dst_pitch[d];
      for (unsigned r = 0; r < rows; ++r) bulk_s2g(dst + r * dp, base + r * rb, rb);
    }
    bulk_commit();
    if (++s_store == stages) s_store = 0, phase ^= 1u;
    // last chunk of a descriptor batch: its slot is free (all loads up to i + ahead and all
    // stores up to i are issued); refill it with the batch after next
    if (i % kDescBatch == kDescBatch - 1 && i / kDescBatch + 2 < batches) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      fetch_batch(i / kDescBatch + 2);
    }
  }
  bulk_wait_all();
}

// Variant for A/B measurement (RESHARD_COPY_KERNEL=bulk_strided): the round-1 first bulk
// kernel's schedule — CTA c takes tiles c, c+grid, ... straight from the natural array — with
// each descriptor loaded by six independent 16-byte loads when its chunk is issued and
// parked in shared memory for the store phase.
__device__ __forceinline__ void load_desc(const DevFanTile* p, DevFanTile& out) {
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&out);
  uint4 v[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = __ldg(s + k);
#pragma unroll
  for (int k = 0; k < 6; ++k) d[k] = v[k];
}

template <int HINT>
__global__ void __launch_bounds__(32, 1) copy_bulk_strided_kernel(const DevFanTile* __restrict__ tiles,
                                                                  unsigned long long n, int stages, unsigned stage_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[kBulkMaxStages];
  __shared__ DevFanTile sdesc[kBulkMaxStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const unsigned long long pol = HINT ? policy_evict_first() : 0ull;
  const unsigned long long first = blockIdx.x, step = gridDim.x;
  const unsigned long long mine = first < n ? (n - first + step - 1) / step : 0;
  const int ahead = stages > 2 ? stages - 2 : 1;
  int s_load = 0, s_store = 0;
  unsigned phase = 0;
  // one-deep register prefetch: the six loads of chunk i+1's descriptor are in flight
  // while chunk i is issued and stored
  DevFanTile nxt;
  if (mine) load_desc(tiles + first, nxt);
  auto issue_load = [&](unsigned long long i) {
    const DevFanTile t = nxt;
    sdesc[s_load] = t;
    if (i + 1 < mine) load_desc(tiles + first + (i + 1) * step, nxt);
    const unsigned bar = smem_u32(&bars[s_load]);
    const unsigned base = smem_u32(smem + size_t(s_load) * stage_bytes);
    mbar_expect_tx(bar, t.rows * t.row_bytes);
    if (t.pad) {  // K3T tensor tile: src = map, src_pitch = (row << 32 | chunk), row_bytes = box bytes
      tma_load_3d(base, t.src, unsigned(t.src_pitch), unsigned(t.src_pitch >> 32), bar);
    } else {
      for (unsigned r = 0; r < t.rows; ++r) {
        const char* src = reinterpret_cast<const char*>(t.src) + r * t.src_pitch;
        if (HINT & 1) bulk_g2s_hint(base + r * t.row_bytes, src, t.row_bytes, bar, pol);
        else bulk_g2s(base + r * t.row_bytes, src, t.row_bytes, bar);
      }
    }
    if (++s_load == stages) s_load = 0;
  };
  for (unsigned long long i = 0; i < mine && i < (unsigned long long)ahead; ++i) issue_load(i);
  for (unsigned long long i = 0; i < mine; ++i) {
    if (i + ahead < mine) {
      bulk_wait_read<1>();
      issue_load(i + ahead);
    }
    const DevFanTile& t = sdesc[s_store];
    mbar_wait(smem_u32(&bars[s_store]), phase);
    const unsigned base = smem_u32(smem + size_t(s_store) * stage_bytes);
    if (t.pad) {
      for (unsigned d = 0; d < t.n_dst; ++d) tma_store_3d(t.dst[d], unsigned(t.src_pitch), unsigned(t.src_pitch >> 32), base);
    } else {
      for (unsigned d = 0; d < t.n_dst; ++d)
        for (unsigned r = 0; r < t.rows; ++r) {
          char* dst = reinterpret_cast<char*>(t.dst[d]) + r * t.dst_pitch[d];
          if (HINT & 2) bulk_s2g_hint(dst, base + r * t.row_bytes, t.row_bytes, pol);
          else bulk_s2g(dst, base + r * t.row_bytes, t.row_bytes);
        }
    }
    bulk_commit();
    if (++s_store == stages) s_store = 0, phase ^= 1u;
  }
  bulk_wait_all();
}

// Variant RESHARD_COPY_KERNEL=bulk_dyn: the bulk_strided pipeline with DYNAMIC tile
// assignment.  A static c, c+grid, ... split leaves the CTAs finishing up to 6 % of the kernel
// apart on short launches (r2_09 ncu: sm__cycles_active min/max 0.94 on GPT-2 small); here each
// CTA claims the next kClaim tiles of the natural order from a global counter (one atomic per
// claim, issued one claim ahead so its latency hides behind the previous claim's tiles), so the
// CTAs still sweep memory together as one window and finish together.  The last CTA out resets
// the counter for the next launch on the stream.
__global__ void __launch_bounds__(32, 1) copy_bulk_dyn_kernel(const DevFanTile* __restrict__ tiles, unsigned long long n,
                                                              int stages, unsigned stage_bytes, unsigned long long* claim,
                                                              unsigned long long n_static, unsigned long long kClaim) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[kBulkMaxStages];
  __shared__ DevFanTile sdesc[kBulkMaxStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // tiles [0, n_static) in the static c, c + grid, ... order; the rest claimed dynamically
  unsigned long long s_next = blockIdx.x;
  unsigned long long cur = n_static + atomicAdd(claim, kClaim);  // consumed after the static share
  unsigned long long nxt_claim = n, end = cur < n ? min(cur + kClaim, n) : cur;
  bool second = false;  // nxt_claim issued
  auto next_index = [&](unsigned long long& idx) -> bool {
    if (s_next < n_static) {
      idx = s_next;
      s_next += gridDim.x;
      return true;
    }
    if (!second) nxt_claim = n_static + atomicAdd(claim, kClaim), second = true;
    if (cur >= end) {
      if (nxt_claim >= n) return false;
      cur = nxt_claim, end = min(cur + kClaim, n);
      nxt_claim = n_static + atomicAdd(claim, kClaim);  // consumed a whole claim later: its latency is hidden
    }
    idx = cur++;
    return true;
  };
  const int ahead = stages > 2 ? stages - 2 : 1;
  int s_load = 0, s_store = 0;
  unsigned phase = 0;
  DevFanTile nxt;
  unsigned long long ni = 0, issued = 0, stored = 0;
  bool have = next_index(ni);
  if (have) load_desc(tiles + ni, nxt);
  auto issue_load = [&]() {
    const DevFanTile t = nxt;
    sdesc[s_load] = t;
    have = next_index(ni);
    if (have) load_desc(tiles + ni, nxt);
    const unsigned bar = smem_u32(&bars[s_load]);
    const unsigned base = smem_u32(smem + size_t(s_load) * stage_bytes);
    mbar_expect_tx(bar, t.rows * t.row_bytes);
    if (t.pad) {
      tma_load_3d(base, t.src, unsigned(t.src_pitch), unsigned(t.src_pitch >> 32), bar);
    } else {
      for (unsigned r = 0; r < t.rows; ++r)
        bulk_g2s(base + r * t.row_bytes, reinterpret_cast<const char*>(t.src) + r * t.src_pitch, t.row_bytes, bar);
    }
    if (++s_load == stages) s_load = 0;
    ++issued;
  };
  while (have && issued < (unsigned long long)ahead) issue_load();
  while (stored < issued) {
    if (have) {
      bulk_wait_read<1>();  // the stage about to be refilled was last read by the store two back
      issue_load();
    }
    const DevFanTile& t = sdesc[s_store];
    mbar_wait(smem_u32(&bars[s_store]), phase);
    const unsigned base = smem_u32(smem + size_t(s_store) * stage_bytes);
    if (t.pad) {
      for (unsigned d = 0; d < t.n_dst; ++d) tma_store_3d(t.dst[d], unsigned(t.src_pitch), unsigned(t.src_pitch >> 32), base);
    } else {
      for (unsigned d = 0; d < t.n_dst; ++d)
        for (unsigned r = 0; r < t.rows; ++r)
          bulk_s2g(reinterpret_cast<char*>(t.dst[d]) + r * t.dst_pitch[d], base + r * t.row_bytes, t.row_bytes);
    }
    bulk_commit();
    if (++s_store == stages) s_store = 0, phase ^= 1u;
    ++stored;
  }
  bulk_wait_all();
  __threadfence();  // this CTA's claims precede its exit count
  if (atomicAdd(claim + 1, 1ull) == gridDim.x - 1) {
    claim[0] = 0, claim[1] = 0;
    __threadfence();
  }
}

// Variant RESHARD_COPY_KERNEL=bulk_warp: the same schedule, but the 32 lanes share the
// issue work — lane l issues the bulk copies of rows l, l+32, ... of a tile (strided 2-D
// fragments such as row-parallel TP slices have tens of rows per stage).  Lane 0 owns the
// mbarriers; every lane commits and drains its own bulk groups before a stage is reused.
__global__ void __launch_bounds__(32, 1) copy_bulk_warp_kernel(const DevFanTile* __restrict__ tiles, unsigned long long n,
                                                               int stages, unsigned stage_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bars[kBulkMaxStages];
  __shared__ DevFanTile sdesc[kBulkMaxStages];
  const unsigned lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const unsigned long long first = blockIdx.x, step = gridDim.x;
  const unsigned long long mine = first < n ? (n - first + step - 1) / step : 0;
  const int ahead = stages > 2 ? stages - 2 : 1;
  int s_load = 0, s_store = 0;
  unsigned phase = 0;
  DevFanTile nxt;
  if (mine) load_desc(tiles + first, nxt);
  auto issue_load = [&](unsigned long long i) {
    const DevFanTile t = nxt;
    if (i + 1 < mine) load_desc(tiles + first + (i + 1) * step, nxt);
    const unsigned bar = smem_u32(&bars[s_load]);
    const unsigned base = smem_u32(smem + size_t(s_load) * stage_bytes);
    if (lane == 0) {
      sdesc[s_load] = t;
      mbar_expect_tx(bar, t.rows * t.row_bytes);
    }
    __syncwarp();
    for (unsigned r = lane; r < t.rows; r += 32)
      bulk_g2s(base + r * t.row_bytes, reinterpret_cast<const char*>(t.src) + r * t.src_pitch, t.row_bytes, bar);
    if (++s_load == stages) s_load = 0;
  };
  for (unsigned long long i = 0; i < mine && i < (unsigned long long)ahead; ++i) issue_load(i);
  for (unsigned long long i = 0; i < mine; ++i) {
    if (i + ahead < mine) {
      bulk_wait_read<1>();  // this lane's older store groups have read their stage
      __syncwarp();         // ... and so have every other lane's
      issue_load(i + ahead);
    }
    mbar_wait(smem_u32(&bars[s_store]), phase);
    const DevFanTile& t = sdesc[s_store];
    const unsigned base = smem_u32(smem + size_t(s_store) * stage_bytes);
    for (unsigned d = 0; d < t.n_dst; ++d)
      for (unsigned r = lane; r < t.rows; r += 32)
        bulk_s2g(reinterpret_cast<char*>(t.dst[d]) + r * t.dst_pitch[d], base + r * t.row_bytes, t.row_bytes);
    bulk_commit();
    if (++s_store == stages) s_store = 0, phase ^= 1u;
  }
  bulk_wait_all();
}

// ---- synthetic payload ------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long word_at(unsigned long long seed, unsigned long long k) {
  return mix64(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ unsigned char byte_at(unsigned long long seed, unsigned long long b) {
  return (unsigned char)(word_at(seed, b >> 3) >> (8 * (b & 7)));
}
// Base-tensor byte offset of cell byte o.
__device__ __forceinline__ unsigned long long base_byte(const CellGeom& g, unsigned long long o) {
  if (g.rank == 0) return o;
  unsigned long long row = o / g.run_bytes, col = o - row * g.run_bytes;
  unsigned long long off = g.lo[g.rank - 1] * g.stride[g.rank - 1] + col;
  for (int d = int(g.rank) - 2; d >= 0; --d) {
    unsigned long long e = g.ext[d], i = row % e;
    row /= e;
    off += (g.lo[d] + i) * g.stride[d];
  }
  return off;
}
// 16 payload bytes starting at base byte b, as two little-endian words.
__device__ __forceinline__ void stream16(unsigned long long seed, unsigned long long b, unsigned long long& lo,
                                         unsigned long long& hi) {
  const unsigned long long k = b >> 3;
  const unsigned sh = unsigned(b & 7) * 8;
  unsigned long long w0 = word_at(seed, k), w1 = word_at(seed, k + 1);
  if (sh == 0) {
    lo = w0, hi = w1;
  } else {
    unsigned long long w2 = word_at(seed, k + 2);
    lo = (w0 >> sh) | (w1 << (64 - sh));
    hi = (w1 >> sh) | (w2 << (64 - sh));
  }
}
__device__ __forceinline__ int nonzero_bytes(unsigned long long x) {
  const unsigned long long m = 0x7F7F7F7F7F7F7F7Full;
  unsigned long long t = (x & m) + m;
  t = ~(t | x | m);  // high bit set in every zero byte
  return 8 - __popcll(t);
}

// One launch for a whole batch of cells: blockIdx.y (+ y_base) picks the cell, blockIdx.x
// strides over its 16-byte chunks.
template <bool kVerify>
__global__ void __launch_bounds__(256) payload_kernel(const PayloadTask* __restrict__ tasks, unsigned y_base,
                                                      unsigned long long* count) {
  const PayloadTask& task = tasks[y_base + blockIdx.y];
  unsigned char* data = static_cast<unsigned char*>(task.data);
  const unsigned long long seed = task.seed;
  const CellGeom& g = task.g;
  unsigned long long bad = 0;
  const unsigned long long chunks = (g.bytes + 15) / 16;
  const bool aligned = (reinterpret_cast<unsigned long long>(data) & 15) == 0;
  for (unsigned long long q = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; q < chunks;
       q += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long o = q * 16;
    const unsigned long long in_row = g.rank == 0 ? o : o % g.run_bytes;
    if (aligned && o + 16 <= g.bytes && in_row + 16 <= (g.rank == 0 ? g.bytes : g.run_bytes)) {
      unsigned long long lo, hi;
      stream16(seed, base_byte(g, o), lo, hi);
      ulonglong2* p = reinterpret_cast<ulonglong2*>(data + o);
      if (kVerify) {
        ulonglong2 v = *p;
        bad += nonzero_bytes(v.x ^ lo) + nonzero_bytes(v.y ^ hi);
      } else {
        *p = make_ulonglong2(lo, hi);
      }
    } else {
      for (unsigned long long b = o; b < o + 16 && b < g.bytes; ++b) {
        unsigned char want = byte_at(seed, base_byte(g, b));
        if (kVerify) bad += data[b] != want;
        else data[b] = want;
      }
    }
  }
  if (kVerify) {
    for (int off = 16; off > 0; off >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, off);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
  }
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void launch_copy(const CopyTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, bool aligned16,
                 void* stream, unsigned long long* claim) {
  if (n_tiles == 0) return;
  if (!cfg.ldg_dyn) claim = nullptr;
  auto s = static_cast<cudaStream_t>(stream);
  auto tiles = reinterpret_cast<const DevTile*>(d_tiles);
  auto grid = [&](int per_sm) { return int(std::min<uint64_t>(n_tiles, uint64_t(sms) * uint64_t(per_sm))); };
  if (!aligned16) {
    copy_any_kernel<<<grid(8), 256, 0, s>>>(tiles, n_tiles);
  } else if (cfg.kernel == CopyKernel::Ldg8) {
    copy_v16_kernel<8, 2, false><<<grid(cfg.ctas_per_sm), 512, 0, s>>>(tiles, n_tiles, nullptr);
  } else if (claim) {
    copy_v16_kernel<4, 2, true><<<grid(std::min(cfg.ctas_per_sm, 2)), 512, 0, s>>>(tiles, n_tiles, claim);
  } else if (cfg.ctas_per_sm >= 3) {
    copy_v16_kernel<4, 3, false><<<grid(cfg.ctas_per_sm), 512, 0, s>>>(tiles, n_tiles, nullptr);
  } else {
    copy_v16_kernel<4, 2, false><<<grid(cfg.ctas_per_sm), 512, 0, s>>>(tiles, n_tiles, nullptr);
  }
  check(cudaGetLastError(), "copy launch");
}

void launch_copy_fan(const FanTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, void* stream,
                     unsigned long long* claim) {
  if (n_tiles == 0) return;
  if (!cfg.ldg_dyn) claim = nullptr;
  const int grid = int(std::min<uint64_t>(n_tiles, uint64_t(sms) * uint64_t(std::min(cfg.ctas_per_sm < 2 ? 2 : cfg.ctas_per_sm, 2))));
  if (claim)
    copy_fan_v16_kernel<true><<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const DevFanTileL*>(d_tiles), n_tiles, claim);
  else
    copy_fan_v16_kernel<false><<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const DevFanTileL*>(d_tiles), n_tiles, nullptr);
  check(cudaGetLastError(), "fan copy launch");
}

void launch_bulk(const FanTile* d_tiles, uint64_t n_tiles, const CopyConfig& cfg, int sms, void* stream,
                 unsigned long long* claim) {
  if (n_tiles == 0) return;
  // bulk_strided on a long launch switches to dynamic claims (r2_16-r2_18 same-box A/Bs: 2-3 %
  // faster from ~6e5 tiles up, 2.5 % slower on GPT-2 small's 5e4), when a claim counter is given
  const bool dyn = cfg.kernel == CopyKernel::BulkDyn ||
                   (cfg.kernel == CopyKernel::BulkStrided && cfg.l2_hint == 0 && claim && cfg.dyn_min_tiles > 0 &&
                    n_tiles >= uint64_t(cfg.dyn_min_tiles));
  if (dyn) {
    if (!claim) raise(Errc::InvalidArgument, "bulk_dyn needs a zeroed claim counter");
    const size_t smem = size_t(cfg.stages) * cfg.stage_bytes;
    if (cfg.stages < 3 || cfg.stages > kBulkMaxStages || smem > 227 * 1024)
      raise(Errc::InvalidArgument, "bulk stages x stage bytes exceed shared memory");
    check(cudaFuncSetAttribute(copy_bulk_dyn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
          "bulk smem attribute");
    // the static prefix: all but `dyn_tail` tiles per CTA (RESHARD_DYN_TAIL; < 0: everything dynamic)
    const uint64_t grid = uint64_t(bulk_grid(n_tiles, sms, cfg));
    const uint64_t tail = cfg.dyn_tail < 0 ? n_tiles : uint64_t(cfg.dyn_tail) * grid;
    const uint64_t n_static = n_tiles > tail ? (n_tiles - tail) / grid * grid : 0;
    copy_bulk_dyn_kernel<<<unsigned(grid), 32, smem, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const DevFanTile*>(d_tiles), n_tiles, cfg.stages, cfg.stage_bytes, claim, n_static,
        (unsigned long long)std::max(1, cfg.dyn_claim));
    check(cudaGetLastError(), "bulk copy launch");
    return;
  }
  if (cfg.stages < 3 || cfg.stages > kBulkMaxStages) raise(Errc::InvalidArgument, "bulk copy needs 3..16 stages");
  const bool strided = cfg.kernel == CopyKernel::BulkStrided || cfg.kernel == CopyKernel::BulkWarp;
  const size_t smem = size_t(cfg.stages) * cfg.stage_bytes + (strided ? 0 : kDescRingBytes);
  if (smem > 227 * 1024) raise(Errc::InvalidArgument, "bulk stages x stage bytes exceed shared memory");
  auto strided_kern = cfg.l2_hint == 1   ? copy_bulk_strided_kernel<1>
                      : cfg.l2_hint == 2 ? copy_bulk_strided_kernel<2>
                      : cfg.l2_hint == 3 ? copy_bulk_strided_kernel<3>
                                         : copy_bulk_strided_kernel<0>;
  auto kern = cfg.kernel == CopyKernel::BulkWarp ? copy_bulk_warp_kernel
              : strided                          ? strided_kern
                                                 : copy_bulk_kernel;
  check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "bulk smem attribute");
  const int grid = bulk_grid(n_tiles, sms, cfg);
  kern<<<grid, 32, smem, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const DevFanTile*>(d_tiles), n_tiles,
                                                             cfg.stages, cfg.stage_bytes);
  check(cudaGetLastError(), "bulk copy launch");
}

// ---- schedule expansion: pieces -> tiles, on the device ---------------------------------------
// One thread per output tile: binary search of its piece by `first`, then the same tile math
// the host lowering uses (piece_tile, reshard/executor.hpp).  The host uploads only the
// pieces (one per fragment and outer index: thousands), not the tiles (~10^5-10^6).
__device__ __forceinline__ uint32_t piece_of(const DevPiece* __restrict__ p, uint32_t n, uint64_t t) {
  uint32_t lo = 0, hi = n;  // last piece with first <= t
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (__ldg(&p[mid].first) <= t) lo = mid;
    else hi = mid;
  }
  return lo;
}
// position of tile i of n in interleave_for_grid(., n, grid) order
__device__ __forceinline__ uint64_t interleaved(uint64_t i, uint64_t n, uint64_t grid) {
  const uint64_t q = n / grid, r = n % grid, c = i % grid;
  return c * q + (c < r ? c : r) + i / grid;
}

__global__ void __launch_bounds__(256) expand_fan_kernel(const DevPiece* __restrict__ p, uint32_t np, uint64_t t0,
                                                         uint64_t t1, FanTile* __restrict__ out, unsigned grid) {
  const uint64_t n = t1 - t0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = t0 + i;
    const DevPiece& q = p[piece_of(p, np, t)];
    uint64_t r0, c;
    uint32_t rows, bytes;
    piece_tile(q.rows, q.row_bytes, q.per, q.tile, t - q.first, r0, c, rows, bytes);
    FanTile f;
    f.src = q.src + r0 * q.src_pitch + c, f.src_pitch = q.src_pitch;
    f.rows = rows, f.row_bytes = bytes, f.n_dst = q.n_dst, f.pad = 0;
#pragma unroll
    for (int d = 0; d < kMaxFan; ++d) {
      f.dst[d] = d < int(q.n_dst) ? q.dst[d] + r0 * q.dst_pitch[d] + c : 0ull;
      f.dst_pitch[d] = d < int(q.n_dst) ? q.dst_pitch[d] : 0ull;
    }
    out[grid ? interleaved(i, n, grid) : i] = f;
  }
}

__global__ void __launch_bounds__(256) expand_copy_kernel(const DevPiece* __restrict__ p, uint32_t np, uint64_t n,
                                                          CopyTile* __restrict__ out) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const DevPiece& q = p[piece_of(p, np, t)];
    uint64_t r0, c;
    uint32_t rows, bytes;
    piece_tile(q.rows, q.row_bytes, q.per, q.tile, t - q.first, r0, c, rows, bytes);
    out[t] = CopyTile{q.src + r0 * q.src_pitch + c, q.dst[0] + r0 * q.dst_pitch[0] + c, q.src_pitch, q.dst_pitch[0],
                      rows, bytes};
  }
}

void launch_expand_fan(const DevPiece* d_pieces, uint32_t n_pieces, uint64_t t0, uint64_t t1, FanTile* out,
                       unsigned grid, int sms, void* stream) {
  if (t1 <= t0 || n_pieces == 0) return;
  const uint64_t blocks = std::min<uint64_t>((t1 - t0 + 255) / 256, uint64_t(sms) * 8);
  expand_fan_kernel<<<unsigned(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_pieces, n_pieces, t0, t1, out,
                                                                                      grid);
  check(cudaGetLastError(), "expand launch");
}
void launch_expand_copy(const DevPiece* d_pieces, uint32_t n_pieces, uint64_t n_tiles, CopyTile* out, int sms,
                        void* stream) {
  if (n_tiles == 0 || n_pieces == 0) return;
  const uint64_t blocks = std::min<uint64_t>((n_tiles + 255) / 256, uint64_t(sms) * 8);
  expand_copy_kernel<<<unsigned(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_pieces, n_pieces, n_tiles, out);
  check(cudaGetLastError(), "expand launch");
}

void launch_payload(const PayloadTask* d_tasks, uint64_t n_tasks, uint64_t max_bytes, bool verify,
                    unsigned long long* d_count, void* stream) {
  if (n_tasks == 0) return;
  const unsigned long long chunks = (max_bytes + 15) / 16;
  const unsigned gx = unsigned(std::max<unsigned long long>(1, std::min<unsigned long long>((chunks + 255) / 256, 512)));
  auto s = static_cast<cudaStream_t>(stream);
  for (uint64_t y = 0; y < n_tasks; y += 65535) {
    dim3 grid(gx, unsigned(std::min<uint64_t>(65535, n_tasks - y)));
    if (verify) payload_kernel<true><<<grid, 256, 0, s>>>(d_tasks, unsigned(y), d_count);
    else payload_kernel<false><<<grid, 256, 0, s>>>(d_tasks, unsigned(y), nullptr);
    check(cudaGetLastError(), "payload launch");
  }
}

CellGeom make_geom(const Shape& base, size_t width, const Range& cell) {
  CellGeom g{};
  g.rank = uint32_t(base.size());
  g.width = uint32_t(width);
  uint64_t stride = width;
  for (size_t d = base.size(); d-- > 0;) {
    g.stride[d] = stride;
    stride *= base[d];
    g.lo[d] = cell.dim(int(d)).lo;
    g.ext[d] = cell.dim(int(d)).extent();
  }
  g.bytes = cell.elements() * width;
  g.run_bytes = base.empty() ? width : g.ext[base.size() - 1] * width;
  return g;
}

}  // namespace reshard::cuda
