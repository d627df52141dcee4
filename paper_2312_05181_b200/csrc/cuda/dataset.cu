// K5 dataset_repartition (sm_100a): for one new DP rank, over its remaining samples k —
//   pos[k]  = closed-form global position,
//   ent[k]  = samples[perm[pos[k]]]                (24-byte gather through the permutation),
//   boff[k] = exclusive prefix sum of lengths       (the sample's offset in the read buffer),
//   queue[class] += k                               (stable compaction by locator class,
//                                                    local > peer > remote).
// Default (split2): a register-light gather pass at full occupancy writes pos / entries,
// parks each length in boff and each class in a byte, and reduces one aggregate per
// 1024-sample tile; a few-CTA tile scan (decoupled look-back over 1024-tile blocks) turns
// the aggregates into prefixes; a finalize pass turns the parked lengths into offsets in
// place and fills the class queues.  The single-pass decoupled look-back kernel
// (repartition_kernel) stays selectable (RESHARD_K5=lookback).
// Replaces the CPU loops of oracle.cpp orc_dataset_gather (SPEC restatement).
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "reshard/dataset.hpp"
#include "reshard/trace.hpp"

namespace reshard {

namespace {

constexpr int kThreads = 256, kItems = 8, kTile = kThreads * kItems, kWarps = kThreads / 32;

struct Agg {
  unsigned long long len, c0, c1, c2;
};
__device__ __forceinline__ Agg operator+(const Agg& a, const Agg& b) { return {a.len + b.len, a.c0 + b.c0, a.c1 + b.c1, a.c2 + b.c2}; }

struct Params {
  const unsigned long long* perm;
  const unsigned long long* samples;
  const unsigned char* file_class;
  unsigned long long n, B, at_step, b, rank, count, in_full, full;
};
struct Outs {
  unsigned long long *pos, *ent, *boff;
  unsigned *q0, *q1, *q2;
  unsigned long long* qcount;
};
struct Scratch {
  unsigned* counter;
  unsigned* flags;  // 0 empty, 1 aggregate, 2 inclusive prefix
  Agg* agg;
  Agg* inc;
  unsigned ntiles;
};

__device__ __forceinline__ Agg shfl_up(const Agg& v, int d) {
  return {__shfl_up_sync(0xffffffffu, v.len, d), __shfl_up_sync(0xffffffffu, v.c0, d),
          __shfl_up_sync(0xffffffffu, v.c1, d), __shfl_up_sync(0xffffffffu, v.c2, d)};
}
__device__ __forceinline__ Agg ldcg(const Agg* p) {
  return {__ldcg(&p->len), __ldcg(&p->c0), __ldcg(&p->c1), __ldcg(&p->c2)};
}
__device__ __forceinline__ void stcg(Agg* p, const Agg& v) {
  __stcg(&p->len, v.len), __stcg(&p->c0, v.c0), __stcg(&p->c1, v.c1), __stcg(&p->c2, v.c2);
}

template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) repartition_kernel(Params p, Outs o, Scratch s) {
  __shared__ unsigned tile_sh;
  __shared__ Agg warp_tot[kWarps];
  __shared__ Agg tile_prefix;
  if (threadIdx.x == 0) tile_sh = atomicAdd(s.counter, 1u);
  __syncthreads();
  const unsigned tile = tile_sh;
  const unsigned long long k0 = (unsigned long long)tile * kTile + (unsigned long long)threadIdx.x * kItems;

  // position of k0, then advanced incrementally
  unsigned long long batch = 0, r = 0;
  if (k0 < p.in_full) batch = p.at_step + k0 / p.b, r = k0 % p.b;
  unsigned long long len[kItems];
  unsigned char cls[kItems];
  Agg mine{0, 0, 0, 0};
  // Three dependent gathers per sample (perm -> entry -> file class).  Issue each level for
  // all kItems samples before consuming any, so kItems independent random loads are in
  // flight per thread at every level (memory-level parallelism, not latency chains).
  unsigned long long pos[kItems], idx[kItems], f[kItems], off[kItems];
  const unsigned nv = p.count > k0 ? unsigned(min(p.count - k0, (unsigned long long)kItems)) : 0u;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long k = k0 + j;
    if (k < p.in_full) {
      pos[j] = batch * p.B + p.rank * p.b + r;
      if (++r == p.b) r = 0, ++batch;
    } else {
      pos[j] = p.full * p.B + p.rank * p.b + (k - p.in_full);
    }
    idx[j] = j < nv ? __ldg(p.perm + pos[j]) : 0ull;
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long* e = p.samples + 3 * idx[j];
    if (j < nv) f[j] = __ldg(e), off[j] = __ldg(e + 1), len[j] = __ldg(e + 2);
    else f[j] = 0, off[j] = 0, len[j] = 0;
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    cls[j] = j < nv ? __ldg(p.file_class + f[j]) : (unsigned char)3;
    if (j < nv) {
      const unsigned long long k = k0 + j;
      o.pos[k] = pos[j];
      o.ent[3 * k] = f[j], o.ent[3 * k + 1] = off[j], o.ent[3 * k + 2] = len[j];
      mine.len += len[j];
      mine.c0 += cls[j] == 0, mine.c1 += cls[j] == 1, mine.c2 += cls[j] == 2;
    }
  }
  // block exclusive scan of the per-thread aggregates
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Agg inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Agg up = shfl_up(inc, d);
    if (lane >= d) inc = inc + up;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  Agg warp_base{0, 0, 0, 0}, total{0, 0, 0, 0};
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) warp_base = warp_base + warp_tot[w];
    total = total + warp_tot[w];
  }
  const Agg excl_in_tile = warp_base + (Agg{inc.len - mine.len, inc.c0 - mine.c0, inc.c1 - mine.c1, inc.c2 - mine.c2});

  // decoupled look-back, warp-parallel (warp 0): lane l inspects predecessor tile-1-l-32*w;
  // the window stops at the nearest predecessor that already published an inclusive prefix.
  if (warp == 0) {
    Agg prefix{0, 0, 0, 0};
    if (tile == 0) {
      if (lane == 0) {
        stcg(&s.inc[0], total);
        __threadfence();
        ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[0]).store(2u, ::cuda::memory_order_release);
      }
    } else {
      if (lane == 0) {
        stcg(&s.agg[tile], total);
        __threadfence();
        ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[tile]).store(1u, ::cuda::memory_order_release);
      }
      for (long long base = (long long)tile - 1;; base -= 32) {
        const long long j = base - lane;
        unsigned f = 2u;  // before tile 0: an inclusive prefix of zero
        Agg v{0, 0, 0, 0};
        if (j >= 0) {
          ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device> fl(s.flags[j]);
          while ((f = fl.load(::cuda::memory_order_acquire)) == 0u) {
          }
          v = f == 2u ? ldcg(&s.inc[j]) : ldcg(&s.agg[j]);
        }
        const unsigned inc_mask = __ballot_sync(0xffffffffu, f == 2u);
        const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;  // nearest inclusive predecessor
        if (lane > stop) v = Agg{0, 0, 0, 0};
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
          v.len += __shfl_xor_sync(0xffffffffu, v.len, d);
          v.c0 += __shfl_xor_sync(0xffffffffu, v.c0, d);
          v.c1 += __shfl_xor_sync(0xffffffffu, v.c1, d);
          v.c2 += __shfl_xor_sync(0xffffffffu, v.c2, d);
        }
        prefix = prefix + v;
        if (inc_mask) break;
      }
      if (lane == 0) {
        stcg(&s.inc[tile], prefix + total);
        __threadfence();
        ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[tile]).store(2u, ::cuda::memory_order_release);
      }
    }
    if (lane == 0) {
      tile_prefix = prefix;
      if (tile == s.ntiles - 1) {
        const Agg all = prefix + total;
        o.qcount[0] = all.c0, o.qcount[1] = all.c1, o.qcount[2] = all.c2;
      }
    }
  }
  __syncthreads();
  Agg run = tile_prefix + excl_in_tile;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long k = k0 + j;
    if (k >= p.count) break;
    o.boff[k] = run.len;
    run.len += len[j];
    if (cls[j] == 0) o.q0[run.c0++] = unsigned(k);
    else if (cls[j] == 1) o.q1[run.c1++] = unsigned(k);
    else o.q2[run.c2++] = unsigned(k);
  }
}

// ---- shared helpers ---------------------------------------------------------------------

// Warp 0: publish this tile's aggregate, walk back over predecessors (warp-parallel), publish
// the inclusive prefix.  Returns the exclusive prefix of the tile (every lane).
__device__ __forceinline__ Agg decoupled_lookback(unsigned tile, const Agg& total, const Scratch& s, int lane) {
  Agg prefix{0, 0, 0, 0};
  if (tile == 0) {
    if (lane == 0) {
      stcg(&s.inc[0], total);
      __threadfence();
      ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[0]).store(2u, ::cuda::memory_order_release);
    }
    return prefix;
  }
  if (lane == 0) {
    stcg(&s.agg[tile], total);
    __threadfence();
    ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[tile]).store(1u, ::cuda::memory_order_release);
  }
  for (long long base = (long long)tile - 1;; base -= 32) {
    const long long j = base - lane;
    unsigned f = 2u;
    Agg v{0, 0, 0, 0};
    if (j >= 0) {
      ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device> fl(s.flags[j]);
      while ((f = fl.load(::cuda::memory_order_acquire)) == 0u) {
      }
      v = f == 2u ? ldcg(&s.inc[j]) : ldcg(&s.agg[j]);
    }
    const unsigned inc_mask = __ballot_sync(0xffffffffu, f == 2u);
    const int stop = inc_mask ? __ffs(inc_mask) - 1 : 31;
    if (lane > stop) v = Agg{0, 0, 0, 0};
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      v.len += __shfl_xor_sync(0xffffffffu, v.len, d);
      v.c0 += __shfl_xor_sync(0xffffffffu, v.c0, d);
      v.c1 += __shfl_xor_sync(0xffffffffu, v.c1, d);
      v.c2 += __shfl_xor_sync(0xffffffffu, v.c2, d);
    }
    prefix = prefix + v;
    if (inc_mask) break;
  }
  if (lane == 0) {
    stcg(&s.inc[tile], prefix + total);
    __threadfence();
    ::cuda::atomic_ref<unsigned, ::cuda::thread_scope_device>(s.flags[tile]).store(2u, ::cuda::memory_order_release);
  }
  return prefix;
}

// count < 2^32 (checked by the host), so k and the in-batch arithmetic are 32-bit
__device__ __forceinline__ unsigned long long sample_pos(const Params& p, unsigned k) {
  if (k < p.in_full) {
    const unsigned b = unsigned(p.b), q = k / b;
    return (p.at_step + q) * p.B + p.rank * p.b + (k - q * b);
  }
  return p.full * p.B + p.rank * p.b + (k - p.in_full);
}

// One index entry {file, offset, length}: the reference's packed 24-byte record (LD 0:
// three 8-byte loads, one record in 8 straddles a 128-byte line), or the padded 32-byte
// device layout of dataset_index_pad (LD 1..3: one 16-byte and one 8-byte load, or one 32-byte load, from a single
// 32-byte sector).
//
// LD (the padded layout's load flavour, RESHARD_K5_LOAD): 1 "ldg" (default) — 16 + 8-byte
// non-coherent loads through L1; 2 "v4na" — ONE 32-byte load (ld.global.nc.L1::no_allocate.v4.u64,
// sm_100) that does not allocate in L1; 3 "cg" — 16 + 8-byte loads cached in L2 only.  r2_03 ncu
// (profiles/r2_03/k5_sectors.json): L1 sectors per sample drop from 2.88 to 1.88 with v4na, yet
// L2 sectors (4.2) and DRAM bytes (134 per sample = 8 of perm + one 128-byte line per random
// record) do not move with the L1 request size nor with cudaLimitMaxL2FetchGranularity: a
// random record costs a whole DRAM line — the hardware floor K5 is measured against.
template <int LD>
__device__ __forceinline__ void load_entry(const unsigned long long* samples, unsigned long long idx,
                                           unsigned long long& f, unsigned long long& off, unsigned long long& len) {
  if (LD == 1) {
    const unsigned long long* e = samples + 4 * idx;
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(e));
    f = a.x, off = a.y, len = __ldg(e + 2);
  } else if (LD == 2) {
    const unsigned long long* e = samples + 4 * idx;
    unsigned long long pad;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(f), "=l"(off), "=l"(len), "=l"(pad)
                 : "l"(e));
  } else if (LD == 3) {
    const unsigned long long* e = samples + 4 * idx;
    const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2*>(e));
    f = a.x, off = a.y, len = __ldcg(e + 2);
  } else {
    const unsigned long long* e = samples + 3 * idx;
    f = __ldg(e), off = __ldg(e + 1), len = __ldg(e + 2);
  }
}

// dataset_index_pad: packed 24-byte records -> padded 32-byte records (pad word zero); one
// streaming pass, coalesced 8-byte loads and 16-byte stores.
__global__ void __launch_bounds__(kThreads) index_pad_kernel(const unsigned long long* __restrict__ src,
                                                             unsigned long long* __restrict__ dst, unsigned long long n) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * kThreads) {
    const unsigned long long f = __ldg(src + 3 * i), off = __ldg(src + 3 * i + 1), len = __ldg(src + 3 * i + 2);
    reinterpret_cast<ulonglong2*>(dst + 4 * i)[0] = make_ulonglong2(f, off);
    reinterpret_cast<ulonglong2*>(dst + 4 * i)[1] = make_ulonglong2(len, 0ull);
  }
}

// ---- random-gather floors (diagnostic) --------------------------------------------------------
// gather_probe_kernel: K5's two HBM-random levels alone — the rank's perm positions, one
// 24-byte entry gather per position, nothing written but one word per thread — at the
// configuration the standalone probe found fastest (4 items per thread, 256 threads;
// scripts/probe_gather.cu, profiles/r12).  gather_write_probe_kernel (below, the default of
// repartition_gather_probe): the same gathers plus every output byte K5 must write.  bench.py
// reports K5 against the latter next to the streaming-HBM roofline.
constexpr int kProbeItems = 4;
template <int LD>
__global__ void __launch_bounds__(kThreads) gather_probe_kernel(Params p, unsigned long long* sink) {
  const unsigned long long k0 =
      ((unsigned long long)blockIdx.x * kThreads + threadIdx.x) * (unsigned long long)kProbeItems;
  unsigned long long batch = 0, r = 0;
  if (k0 < p.in_full) batch = p.at_step + k0 / p.b, r = k0 % p.b;
  unsigned long long idx[kProbeItems], acc = 0;
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    const unsigned long long k = k0 + j;
    unsigned long long pos;
    if (k < p.in_full) {
      pos = batch * p.B + p.rank * p.b + r;
      if (++r == p.b) r = 0, ++batch;
    } else {
      pos = p.full * p.B + p.rank * p.b + (k - p.in_full);
    }
    idx[j] = k < p.count ? __ldg(p.perm + pos) : 0ull;
  }
  unsigned long long f[kProbeItems], off[kProbeItems], len[kProbeItems];
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    load_entry<LD>(p.samples, idx[j], f[j], off[j], len[j]);
  }
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) acc ^= f[j] + off[j] + len[j];
  if (acc == 0x9e3779b97f4a7c15ull) *sink = acc;  // keeps the loads; practically never stores
}

// The same gathers plus K5's 44 output bytes per sample (pos, entry, a length word, a u32
// queue word), warp-striped so every store is coalesced, and no scan: the floor of any
// kernel that must both gather the entries and write the partition (RESHARD_PROBE=write).
template <int LD>
__global__ void __launch_bounds__(kThreads) gather_write_probe_kernel(Params p, Outs o) {
  unsigned long long idx[kProbeItems], pos[kProbeItems];
  const unsigned long long base = (unsigned long long)blockIdx.x * (kThreads * kProbeItems) + threadIdx.x;
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    const unsigned long long k = base + j * kThreads;
    pos[j] = k < p.count ? sample_pos(p, unsigned(k)) : 0ull;
    idx[j] = k < p.count ? __ldg(p.perm + pos[j]) : 0ull;
  }
  unsigned long long f[kProbeItems], off[kProbeItems], len[kProbeItems];
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    load_entry<LD>(p.samples, idx[j], f[j], off[j], len[j]);
  }
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) {
    const unsigned long long k = base + j * kThreads;
    if (k >= p.count) break;
    o.pos[k] = pos[j];
    o.ent[3 * k] = f[j], o.ent[3 * k + 1] = off[j], o.ent[3 * k + 2] = len[j];
    o.boff[k] = len[j];
    o.q0[k] = unsigned(f[j]);
  }
}

// ---- K5 split2: register-light gather at full occupancy / scan / finalize ------------------
// r16 probes: the entry gathers plus every output store of K5 (44 B / sample, coalesced) run
// in 3.50 ms per step when nothing waits (gather_write_probe_kernel), against 6.36 ms for the
// single-pass kernel, whose 80-register threads (3 CTAs / SM) hold 8 entries each and then
// stall behind the look-back.  split2 keeps the probe's shape for the heavy pass: 4 items per
// thread, 32 registers, 8 CTAs / SM (8192 gathers in flight per SM), warp-contiguous items so
// every store is coalesced, and a register-only tile reduction instead of a scan.  Lengths are
// parked in boff and classes in a byte array (9 B / sample written and re-read); one CTA scans
// the tile aggregates; the finalize pass turns the parked lengths into offsets in place and
// fills the class queues with ballots.
constexpr int kGItems = 4, kGTile = kThreads * kGItems, kGWarpItems = 32 * kGItems;
constexpr int kClsBits = 21;  // per-class counts packed into one u64 (a tile has <= 1024 items)
constexpr unsigned long long kClsMask = (1ull << kClsBits) - 1;

// The gather pass of tile `bid` of one rank (the single-rank kernel passes blockIdx.x; the
// multi-rank kernel the block's index within its rank's tiles).
template <int LD>
__device__ __forceinline__ void gather2_tile(const Params& p, const Outs& o, const Scratch& sc, unsigned char* cls_out,
                                             unsigned bid) {
  __shared__ unsigned long long warp_len[kWarps], warp_cnt[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long k0 = (unsigned long long)bid * kGTile + warp * kGWarpItems + lane;
  unsigned long long idx[kGItems];
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    const unsigned long long k = k0 + 32 * j;
    idx[j] = k < p.count ? __ldg(p.perm + sample_pos(p, unsigned(k))) : 0ull;
  }
  unsigned long long f[kGItems], off[kGItems], len[kGItems];
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    f[j] = 0, off[j] = 0, len[j] = 0;
    if (k0 + 32 * j < p.count) load_entry<LD>(p.samples, idx[j], f[j], off[j], len[j]);
  }
  unsigned long long lsum = 0, cnt = 0;
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    const unsigned long long k = k0 + 32 * j;
    if (k < p.count) {
      const unsigned char c = min(__ldg(p.file_class + f[j]), (unsigned char)2);  // 0 local, 1 peer, 2 remote
      o.pos[k] = sample_pos(p, unsigned(k));
      o.ent[3 * k] = f[j], o.ent[3 * k + 1] = off[j], o.ent[3 * k + 2] = len[j];
      o.boff[k] = len[j];  // parked; finalize turns it into the offset
      cls_out[k] = c;
      lsum += len[j];
      cnt += 1ull << (kClsBits * c);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lsum += __shfl_xor_sync(0xffffffffu, lsum, d);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
  }
  if (lane == 0) warp_len[warp] = lsum, warp_cnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long L = 0, C = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) L += warp_len[q], C += warp_cnt[q];
    sc.agg[bid] = Agg{L, C & kClsMask, (C >> kClsBits) & kClsMask, C >> (2 * kClsBits)};
  }
  if (bid == 0) {  // the tile scan's ticket counter and look-back flags, consumed after this launch
    if (threadIdx.x == 0) *sc.counter = 0u;
    for (unsigned i = threadIdx.x; i < (sc.ntiles + 1023) / 1024; i += kThreads) sc.flags[i] = 0u;
  }
}

template <int MINB, int LD>
__global__ void __launch_bounds__(kThreads, MINB) repart_gather2_kernel(Params p, Outs o, Scratch sc,
                                                                         unsigned char* cls_out) {
  gather2_tile<LD>(p, o, sc, cls_out, blockIdx.x);
}

// One rank of a multi-rank launch (several new DP ranks on one GPU, one launch per pass):
// its parameters and where its blocks start in the gather / finalize grid and the scan grid.
struct RankK5 {
  Params p;
  Outs o;
  Scratch s;
  unsigned char* cls;
  Agg* blk;
  unsigned tile0, sblock0, fin0;  // first block in the gather grid, the scan grid, the finalize grid
};
// The ranks of one launch, passed BY VALUE (kernel parameters live in the constant bank: the
// per-block rank lookup and field loads are uniform constant-cache reads, no global round trip
// before a block's first data load).  Batches with more ranks launch in chunks.
constexpr int kMaxRanksPerLaunch = 16;
struct RankTable {
  RankK5 r[kMaxRanksPerLaunch];
  int n;
};
static_assert(sizeof(RankTable) <= 4000, "kernel parameter space");
// The grids of a multi-rank batch: gather pass, tile scan, finalize.
enum class K5Grid { Gather, Scan, Fin };
template <K5Grid G>
__device__ __forceinline__ unsigned first_block(const RankK5& k) {
  return G == K5Grid::Gather ? k.tile0 : G == K5Grid::Scan ? k.sblock0 : k.fin0;
}
// The rank a block belongs to: the last rank whose first block is at or below it (ranks in
// launch order, empty ranks left out); every thread computes it from uniform loads.
template <K5Grid G>
__device__ __forceinline__ int rank_of_block(const RankTable& t, unsigned b) {
  int r = 0;
#pragma unroll 1
  for (int i = 1; i < t.n; ++i)
    if (first_block<G>(t.r[i]) <= b) r = i;
  return r;
}

template <int MINB, int LD>
__global__ void __launch_bounds__(kThreads, MINB) repart_gather2_multi_kernel(const __grid_constant__ RankTable t) {
  const RankK5& k = t.r[rank_of_block<K5Grid::Gather>(t, blockIdx.x)];
  gather2_tile<LD>(k.p, k.o, k.s, k.cls, blockIdx.x - k.tile0);
}

// Exclusive scan of the tile aggregates: one 1024-thread CTA per 1024 tiles (coalesced loads,
// block scan in registers and shared memory), chained by a decoupled look-back over the few
// block aggregates (the flags were cleared by the gather pass).  Writes prefix[t] (s.inc)
// and the queue totals.
__device__ __forceinline__ void tile_scan_block(const Scratch& sc, Agg* blk_agg, Agg* blk_inc, const Outs& o,
                                                unsigned nblocks) {
  __shared__ Agg warp_tot[32];
  __shared__ Agg blk_prefix;
  __shared__ unsigned ticket;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // block order from an atomic ticket, not blockIdx: a block only ever waits on blocks that
  // already run, whatever order the hardware schedules them in
  if (threadIdx.x == 0) ticket = atomicAdd(sc.counter, 1u);
  __syncthreads();
  const unsigned b = ticket;
  const unsigned t = b * 1024u + threadIdx.x;
  const Agg mine = t < sc.ntiles ? sc.agg[t] : Agg{0, 0, 0, 0};
  Agg inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Agg up = shfl_up(inc, d);
    if (lane >= d) inc = inc + up;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  Agg base{0, 0, 0, 0}, total{0, 0, 0, 0};
  for (int q = 0; q < 32; ++q) {
    if (q < warp) base = base + warp_tot[q];
    total = total + warp_tot[q];
  }
  if (warp == 0) {
    const Scratch bs{nullptr, sc.flags, blk_agg, blk_inc, nblocks};
    const Agg prefix = decoupled_lookback(b, total, bs, lane);
    if (lane == 0) {
      blk_prefix = prefix;
      if (b == nblocks - 1) {
        const Agg all = prefix + total;
        o.qcount[0] = all.c0, o.qcount[1] = all.c1, o.qcount[2] = all.c2;
      }
    }
  }
  __syncthreads();
  if (t < sc.ntiles)
    sc.inc[t] = blk_prefix + base + Agg{inc.len - mine.len, inc.c0 - mine.c0, inc.c1 - mine.c1, inc.c2 - mine.c2};
}

__global__ void __launch_bounds__(1024) repart_tile_scan_kernel(Scratch sc, Agg* blk_agg, Agg* blk_inc, Outs o) {
  tile_scan_block(sc, blk_agg, blk_inc, o, gridDim.x);
}

// Every rank's tile scan in one launch: a block serves the rank its index falls in and takes a
// ticket among that rank's blocks, so it only ever waits on blocks of its rank that already run.
__global__ void __launch_bounds__(1024) repart_tile_scan_multi_kernel(const __grid_constant__ RankTable t) {
  const RankK5& k = t.r[rank_of_block<K5Grid::Scan>(t, blockIdx.x)];
  const unsigned nb = (k.s.ntiles + 1023) / 1024;
  tile_scan_block(k.s, k.blk, k.blk + nb, k.o, nb);
}

// Finalize: thread t of tile T owns the 4 consecutive samples T*1024 + 4t .. 4t+3 (16-byte
// vector loads / stores of the parked lengths, one 4-byte load of the classes), so the scan
// is a sequential sum in registers plus ONE warp scan of (length total, packed class counts)
// per thread instead of one per item (r21 ncu: the warp-striped version was issue-bound,
// 61 % SM throughput, 107 us per launch).
constexpr int kCntBits = 10;  // per-class counts of one warp (<= 128) packed into a u32
// One thread's inputs of a finalize tile: its 4 parked lengths, their class bytes, the tile's
// exclusive prefix.
struct FinIn {
  unsigned long long len[kGItems];
  unsigned cls4;  // 4 class bytes, item j in byte j
  Agg pre;
};
__device__ __forceinline__ bool fin_full(const Params& p, const Outs& o, unsigned long long k0) {
  return k0 + kGItems <= p.count && (reinterpret_cast<uintptr_t>(o.boff) & 15) == 0;
}
__device__ __forceinline__ void fin_load(const Params& p, const Outs& o, const Agg* prefix, const unsigned char* cls_in,
                                         unsigned bid, FinIn& in) {
  const unsigned long long k0 = (unsigned long long)bid * kGTile + (unsigned long long)threadIdx.x * kGItems;
  in.pre = prefix[bid];  // issued with the data loads, not after the barrier
  if (fin_full(p, o, k0)) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(o.boff + k0);
    const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(o.boff + k0 + 2);
    in.len[0] = a.x, in.len[1] = a.y, in.len[2] = b.x, in.len[3] = b.y;
    in.cls4 = *reinterpret_cast<const unsigned*>(cls_in + k0);
  } else {
    in.cls4 = 0x03030303u;
#pragma unroll
    for (int j = 0; j < kGItems; ++j) {
      in.len[j] = k0 + j < p.count ? o.boff[k0 + j] : 0ull;
      if (k0 + j < p.count) in.cls4 = (in.cls4 & ~(0xffu << (8 * j))) | (unsigned(cls_in[k0 + j]) << (8 * j));
    }
  }
}
// The scan of one tile and its stores; warp_tot: kWarps Aggs of shared memory (one barrier)
__device__ __forceinline__ void fin_store(const Params& p, const Outs& o, unsigned bid, const FinIn& in, Agg* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long k0 = (unsigned long long)bid * kGTile + (unsigned long long)threadIdx.x * kGItems;
  unsigned long long tl = 0;
  unsigned tc = 0;
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    const unsigned c = (in.cls4 >> (8 * j)) & 0xffu;
    tl += in.len[j];
    if (c < 3) tc += 1u << (kCntBits * c);
  }
  unsigned long long il = tl;
  unsigned ic = tc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long ul = __shfl_up_sync(0xffffffffu, il, d);
    const unsigned uc = __shfl_up_sync(0xffffffffu, ic, d);
    if (lane >= d) il += ul, ic += uc;
  }
  constexpr unsigned m = (1u << kCntBits) - 1u;
  if (lane == 31) warp_tot[warp] = Agg{il, ic & m, (ic >> kCntBits) & m, ic >> (2 * kCntBits)};
  __syncthreads();
  Agg run = in.pre;
#pragma unroll
  for (int q = 0; q < kWarps; ++q)
    if (q < warp) run = run + warp_tot[q];
  const unsigned ex = ic - tc;  // exclusive class counts within the warp
  unsigned long long off = run.len + il - tl;
  unsigned long long qi[3] = {run.c0 + (ex & m), run.c1 + ((ex >> kCntBits) & m), run.c2 + (ex >> (2 * kCntBits))};
  unsigned long long out[kGItems];
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    out[j] = off;
    off += in.len[j];
    const unsigned c = (in.cls4 >> (8 * j)) & 0xffu;
    if (c == 0) o.q0[qi[0]++] = unsigned(k0 + j);
    else if (c == 1) o.q1[qi[1]++] = unsigned(k0 + j);
    else if (c == 2) o.q2[qi[2]++] = unsigned(k0 + j);
  }
  if (fin_full(p, o, k0)) {
    *reinterpret_cast<ulonglong2*>(o.boff + k0) = make_ulonglong2(out[0], out[1]);
    *reinterpret_cast<ulonglong2*>(o.boff + k0 + 2) = make_ulonglong2(out[2], out[3]);
  } else {
#pragma unroll
    for (int j = 0; j < kGItems; ++j)
      if (k0 + j < p.count) o.boff[k0 + j] = out[j];
  }
}
__device__ __forceinline__ void finalize2_tile(const Params& p, const Outs& o, const Agg* prefix, const unsigned char* cls_in,
                                               unsigned bid) {
  __shared__ Agg warp_tot[kWarps];
  FinIn in;
  fin_load(p, o, prefix, cls_in, bid, in);
  fin_store(p, o, bid, in, warp_tot);
}

__global__ void __launch_bounds__(kThreads) repart_finalize2_kernel(Params p, Outs o, const Agg* prefix,
                                                                     const unsigned char* cls_in) {
  finalize2_tile(p, o, prefix, cls_in, blockIdx.x);
}

// Fused finalize: a block owns kFinTiles consecutive tiles of one rank and software-pipelines
// them — the next tile's lengths, classes and prefix are loaded while the current one is scanned
// and stored — so the loads of a short CTA's single tile are no longer its whole lifetime (r2_37
// ncu of one tile per block: 50 % of DRAM peak, 48 % of warp samples on the load scoreboard).
// warp_tot is double-buffered: one barrier per tile.
constexpr unsigned kFinTiles = 8;  // default tiles per block (RESHARD_K5_FIN_TILES; r2_40 sweep: 1 3.59, 2 3.50, 4 3.47, 8 3.45, 16 3.45 ms per step)
template <int FMINB>
__global__ void __launch_bounds__(kThreads, FMINB) repart_finalize2_multi_kernel(const __grid_constant__ RankTable t,
                                                                                 unsigned fin_tiles) {
  __shared__ Agg warp_tot[2][kWarps];
  const RankK5& k = t.r[rank_of_block<K5Grid::Fin>(t, blockIdx.x)];
  const unsigned first = (blockIdx.x - k.fin0) * fin_tiles;
  const unsigned last = min(first + fin_tiles, k.s.ntiles);
  FinIn cur, nxt;
  fin_load(k.p, k.o, k.s.inc, k.cls, first, cur);
  for (unsigned b = first; b < last; ++b) {
    if (b + 1 < last) fin_load(k.p, k.o, k.s.inc, k.cls, b + 1, nxt);
    fin_store(k.p, k.o, b, cur, warp_tot[(b - first) & 1]);
    cur = nxt;
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}
uint64_t align256(uint64_t x) { return (x + 255) / 256 * 256; }

// K5 variant (RESHARD_K5): "split2" (default: gather pass at 5 resident CTAs / SM, tile
// scan, finalize), "split2_6" / "split2_8" (gather pass at 6 / 8 CTAs / SM), "lookback" /
// "lookback4" (the single-pass decoupled look-back kernel at 3 / 4 CTAs / SM).  r16 same-box
// A/B (profiles/r16): split2 4.25 ms, split2_6 4.31, split2_8 4.88, lookback 6.34 per step
// (packed index).  Finalize at 6 / 8 CTAs per SM or 8 items per thread: within +-1 % or 5 %
// slower (r18b), not kept.
struct K5Mode {
  bool lookback = false;
  int minb = 5;  // resident CTAs per SM the chosen gather kernel is compiled for
};
// RESHARD_K5_LOAD: the padded record's load flavour (load_entry): ldg | v4na | cg.
int k5_load() {
  const char* v = std::getenv("RESHARD_K5_LOAD");
  const std::string s = v ? v : "";
  if (s.empty() || s == "ldg") return 1;  // r2_03 A/B: ldg 3.17, v4na 3.24, cg 4.66 ms per step
  if (s == "v4na") return 2;
  if (s == "cg") return 3;
  raise(Errc::InvalidArgument, "RESHARD_K5_LOAD must be ldg, v4na or cg");
}

K5Mode k5_mode() {
  K5Mode m;
  const char* v = std::getenv("RESHARD_K5");
  const std::string s = v ? v : "";
  if (s == "lookback") m.lookback = true, m.minb = 3;
  else if (s == "lookback4") m.lookback = true, m.minb = 4;
  else if (s == "split2_6") m.minb = 6;
  else if (s == "split2_8") m.minb = 8;
  else if (!s.empty() && s != "split2") raise(Errc::InvalidArgument, "RESHARD_K5: unknown variant " + s);
  return m;
}

// The dataset kernels are random 8- and 24-byte gathers: with the default L2 fetch
// granularity every miss pulls a full 128-byte line from HBM (measured 154 DRAM bytes per
// 24-byte entry, profiles/r03_repartition_ncu.json).  Lower the granularity for the
// duration of the launch (RESHARD_L2_FETCH bytes, default 32), restore it afterwards.
struct L2FetchScope {
  size_t old = 0;
  bool set = false;
  L2FetchScope() {
    const char* v = std::getenv("RESHARD_L2_FETCH");
    const size_t want = v && *v ? size_t(std::atoi(v)) : 0;  // r05: 32/64/128 made no difference; off by default
    if (want == 0 || cudaDeviceGetLimit(&old, cudaLimitMaxL2FetchGranularity) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    set = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, want) == cudaSuccess;
    if (!set) cudaGetLastError();
  }
  ~L2FetchScope() {
    if (set) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, old);
  }
};

// ---- K8: bit-exact parallel Fisher-Yates (deterministic reservations) -----------------------
// The sequential shuffle (host shuffle_epoch) performs swap(A[i], A[H[i]]) for i = N-1 .. 1
// with H[i] = splitmix64 draw (N-1-i) mod (i+1).  The draws are counter-based, so every
// H[i] is computed where it is needed.  Iteration i may run once no earlier (higher-index)
// pending iteration touches location i or H[i]: each round, every active iteration reserves
// both its locations with atomicMax of (round << 32 | i); an iteration holding both
// reservations swaps, the others carry over to the next round.  The result is identical to
// the sequential loop (Shun et al., SODA'15, "deterministic reservations").
__device__ __forceinline__ unsigned long long mix64d(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Windowed rounds: a round's active set is the iterations carried over from the last round
// plus the next fresh (highest unprocessed) iterations, up to `window` in all.  Every pending
// iteration of higher priority than an active one is itself active, so the result is still
// the sequential loop's; but the low iterations, which almost always lose their reservations
// while the high ones are pending, no longer reserve and fail round after round (work ~1.1 N
// at window N/160 instead of ~3.5 N with every pending iteration active).  Fresh iterations
// compute their draw inline (no N-entry list), and the round state lives on the device.
// N = 10^8: 33 ms (all pending active, r04-r30) -> 14 ms (window, r67) -> 12.5 (packed
// reservations, r70) -> 8.5 ms (6-round graphs, state checked one batch behind, N/160; r71).
struct ShufState {
  unsigned carried;          // iterations carried into this round (in the carried list)
  unsigned pad;
  unsigned long long lo;     // highest unprocessed fresh iteration (fresh: lo, lo-1, .., 1)
};

__device__ __forceinline__ unsigned long long shuf_entry(const unsigned long long* __restrict__ carried, unsigned c,
                                                         unsigned long long lo, unsigned long long n,
                                                         unsigned long long s0, unsigned long long t) {
  if (t < c) return carried[t];
  const unsigned long long i = lo - (t - c);
  const unsigned long long draw = mix64d(s0 + (n - i) * 0x9e3779b97f4a7c15ull);  // draw number n-1-i
  return (i << 32) | (draw % (i + 1));
}

__device__ __forceinline__ unsigned long long shuf_active(const ShufState& st, unsigned long long window) {
  const unsigned long long take = window > st.carried ? window - st.carried : 0;
  return st.carried + (take < st.lo ? take : st.lo);
}

// Reservations live in the high word of the permutation entry itself, A[x] = reserver << 32
// | value (values and iterations are < 2^32), so a reservation and the value it guards share
// one DRAM sector; key = i (>= 1, 0 = free).  A winner stores its swapped values with the high
// word cleared, which releases both its locations; a loser still holding a location is pending
// and re-reserves it next round, so no stale key can block, and the finished array is the u64
// permutation with no extra pass.  (A separate N-entry array of round << 32 | i keys, r67-r68,
// moved two random sectors per location instead of one: 14.3 vs 12.5 ms, profiles/r70.)
__global__ void shuffle_win_reserve_kernel(const unsigned long long* __restrict__ carried, ShufState* state,
                                           unsigned long long* perm, unsigned round, unsigned long long window,
                                           unsigned long long n, unsigned long long s0) {
  const ShufState st = state[round % 3];
  if (blockIdx.x == 0 && threadIdx.x == 0) state[(round + 1) % 3].carried = 0;  // commit appends into it
  const unsigned long long m = shuf_active(st, window);
  auto* hi = reinterpret_cast<unsigned*>(perm) + 1;  // the high word of A[x] is hi[2x]
  for (unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; t < m;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long e = shuf_entry(carried, st.carried, st.lo, n, s0, t), i = e >> 32, h = e & 0xffffffffull;
    atomicMax(hi + 2 * i, unsigned(i));
    if (h != i) atomicMax(hi + 2 * h, unsigned(i));
  }
}

__global__ void shuffle_win_commit_kernel(const unsigned long long* __restrict__ carried, ShufState* state,
                                          unsigned long long* perm, unsigned long long* next, unsigned round,
                                          unsigned long long window, unsigned long long n, unsigned long long s0,
                                          unsigned* rounds_done) {
  const ShufState st = state[round % 3];
  const unsigned long long m = shuf_active(st, window);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[(round + 1) % 3].lo = st.lo - (m - st.carried);
    if (m) atomicAdd(rounds_done, 1u);
  }
  unsigned* next_count = &state[(round + 1) % 3].carried;
  const unsigned lane = threadIdx.x & 31;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) & ~31ull; base < m;
       base += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long t = base + lane;
    bool pending = false;
    unsigned long long e = 0;
    if (t < m) {
      e = shuf_entry(carried, st.carried, st.lo, n, s0, t);
      const unsigned long long i = e >> 32, h = e & 0xffffffffull;
      const unsigned long long a = __ldcg(perm + i), b = h != i ? __ldcg(perm + h) : a;
      if ((a >> 32) == i && (b >> 32) == i) {
        perm[i] = b & 0xffffffffull;
        if (h != i) perm[h] = a & 0xffffffffull;
      } else {
        pending = true;
      }
    }
    // warp-aggregated append of the iterations that wait for the next round (any order)
    const unsigned mask = __ballot_sync(0xffffffffu, pending);
    unsigned slot = 0;
    if (lane == 0 && mask) slot = atomicAdd(next_count, unsigned(__popc(mask)));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (pending) next[slot + __popc(mask & ((1u << lane) - 1u))] = e;
  }
}

__global__ void shuffle_win_init_kernel(unsigned long long* perm, ShufState* state, unsigned* rounds_done,
                                        unsigned long long n) {
  for (unsigned long long x = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; x < n;
       x += (unsigned long long)gridDim.x * blockDim.x)
    perm[x] = x;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[1].carried = 0, state[1].lo = n - 1;  // round 1 reads slot 1
    *rounds_done = 0;
  }
}

// active iterations per round: N/160 (at least 64 Ki; RESHARD_K8_WINDOW overrides), capped at
// the carried-list capacity the scratch provides
uint64_t shuffle_window_cap(uint64_t n) {
  return std::min<uint64_t>(std::max<uint64_t>(n / 20, 1ull << 16), std::max<uint64_t>(n, 1));
}
uint64_t shuffle_window(uint64_t n) {
  uint64_t w = std::max<uint64_t>(n / 160, 1ull << 16);
  if (const char* v = std::getenv("RESHARD_K8_WINDOW"))
    if (const uint64_t e = std::strtoull(v, nullptr, 10)) w = e;
  return std::min(w, shuffle_window_cap(n));
}
}  // namespace

// round state [3] + rounds counter, two carried lists (window cap each)
uint64_t shuffle_scratch_bytes(uint64_t n) { return 256 + 2 * align256(shuffle_window_cap(n) * 8); }

Timing shuffle_epoch_device(Context& ctx, int gpu, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm, void* scratch) {
  TraceRange trace_("shuffle_epoch_device");
  if (n >= (1ull << 32)) raise(Errc::InvalidArgument, "GPU shuffle supports N < 2^32");
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  L2FetchScope l2fetch;
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  char* sc = static_cast<char*>(scratch);
  const uint64_t cap = align256(shuffle_window_cap(n) * 8);
  unsigned long long* lists[2] = {reinterpret_cast<unsigned long long*>(sc + 256),
                                  reinterpret_cast<unsigned long long*>(sc + 256 + cap)};
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  Timing t;
  void* pinned = nullptr;
  ck(cudaMallocHost(&pinned, 256), "pinned");
  const int grid_full = ctx.sm_count(gpu) * 8;  // 8 resident 256-thread CTAs per SM
  auto* p64 = reinterpret_cast<unsigned long long*>(perm);
  auto* state = reinterpret_cast<ShufState*>(sc);  // slots [3]; rounds counter at sc + 64
  auto* rounds_done = reinterpret_cast<unsigned*>(sc + 64);
  const uint64_t window = shuffle_window(n);
  const int grid = int(std::min<unsigned long long>(grid_full, (window + 255) / 256));
  const unsigned long long s0 = seed ^ epoch;
  // One batch = 6 rounds (the state slots cycle mod 3, the carried lists mod 2), captured
  // once as a graph and replayed; the host checks a batch's final state while the next batch
  // runs, so the GPU does not drain between batches (the last batch is empty rounds).
  cudaGraphExec_t exec = nullptr;
  if (n > 1) {
    cudaStream_t cs;
    ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "capture stream");
    ck(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture");
    for (unsigned round = 1; round <= 6; ++round) {
      const unsigned cur = round & 1;
      shuffle_win_reserve_kernel<<<grid, 256, 0, cs>>>(lists[cur], state, p64, round, window, n, s0);
      shuffle_win_commit_kernel<<<grid, 256, 0, cs>>>(lists[cur], state, p64, lists[cur ^ 1], round, window, n, s0,
                                                      rounds_done);
    }
    cudaGraph_t graph;
    ck(cudaStreamEndCapture(cs, &graph), "capture end");
    ck(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
  }
  ck(cudaEventRecord(e0, st), "event");
  if (n > 1) {
    shuffle_win_init_kernel<<<grid_full, 256, 0, st>>>(p64, state, rounds_done, n);
    ck(cudaGetLastError(), "shuffle init");
    t.launches = 1;
    auto* snap = static_cast<ShufState*>(pinned);  // [2] batch snapshots
    cudaEvent_t done_ev[2];
    ck(cudaEventCreateWithFlags(&done_ev[0], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&done_ev[1], cudaEventDisableTiming), "event");
    for (unsigned b = 0;; ++b) {
      ck(cudaGraphLaunch(exec, st), "graph launch");
      t.launches += 12;
      ck(cudaMemcpyAsync(snap + (b & 1), state + 1, sizeof(ShufState), cudaMemcpyDeviceToHost, st), "state d2h");
      ck(cudaEventRecord(done_ev[b & 1], st), "event");
      if (b == 0) continue;
      ck(cudaEventSynchronize(done_ev[(b - 1) & 1]), "shuffle sync");
      const ShufState s = snap[(b - 1) & 1];
      if (s.carried == 0 && s.lo == 0) break;
    }
    ck(cudaMemcpyAsync(static_cast<char*>(pinned) + 64, rounds_done, sizeof(unsigned), cudaMemcpyDeviceToHost, st),
       "rounds d2h");
    ck(cudaStreamSynchronize(st), "shuffle sync");
    t.tiles = *reinterpret_cast<unsigned*>(static_cast<char*>(pinned) + 64);
    cudaEventDestroy(done_ev[0]);
    cudaEventDestroy(done_ev[1]);
    cudaGraphExecDestroy(exec);
  } else if (n == 1) {
    const unsigned long long zero = 0;
    ck(cudaMemcpyAsync(perm, &zero, 8, cudaMemcpyHostToDevice, st), "perm");
  }
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeHost(pinned);
  t.bytes = n * 8;
  return t;
}

// entry_bytes 0 / 24: the packed reference records; 32: the padded device layout
bool entry_padded(const DatasetIndexView& idx) {
  if (idx.entry_bytes != 0 && idx.entry_bytes != 24 && idx.entry_bytes != 32)
    raise(Errc::InvalidArgument, "entry_bytes must be 24 (packed) or 32 (padded), got " + std::to_string(idx.entry_bytes));
  if (idx.entry_bytes == 32 && (reinterpret_cast<uintptr_t>(idx.samples) & 15))
    raise(Errc::InvalidArgument, "padded index must be 16-byte aligned");
  return idx.entry_bytes == 32;
}

Timing dataset_index_pad(Context& ctx, int gpu, const uint64_t* packed, uint64_t* padded, uint64_t n) {
  TraceRange trace_("dataset_index_pad");
  if ((reinterpret_cast<uintptr_t>(padded) & 15) || (reinterpret_cast<uintptr_t>(packed) & 7))
    raise(Errc::InvalidArgument, "dataset_index_pad: misaligned buffers");
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventRecord(e0, st), "event");
  const uint64_t grid = std::min<uint64_t>((n + kThreads - 1) / kThreads, uint64_t(ctx.sm_count(gpu)) * 8);
  if (grid) index_pad_kernel<<<unsigned(grid), kThreads, 0, st>>>(reinterpret_cast<const unsigned long long*>(packed),
                                                                 reinterpret_cast<unsigned long long*>(padded), n);
  ck(cudaGetLastError(), "index pad launch");
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t.launches = grid ? 1 : 0, t.bytes = 32 * n, t.read_bytes = 24 * n;
  return t;
}

Timing dataset_index_upload(Context& ctx, int gpu, const uint64_t* host_perm, const uint64_t* host_samples,
                            uint64_t n, uint64_t* perm, uint64_t* samples, uint64_t* padded) {
  TraceRange trace_("dataset_index_upload");
  if (padded && (reinterpret_cast<uintptr_t>(padded) & 15))
    raise(Errc::InvalidArgument, "dataset_index_upload: padded index must be 16-byte aligned");
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventRecord(e0, st), "event");
  ck(cudaMemcpyAsync(perm, host_perm, 8 * n, cudaMemcpyHostToDevice, st), "H2D perm");
  ck(cudaMemcpyAsync(samples, host_samples, 24 * n, cudaMemcpyHostToDevice, st), "H2D samples");
  const uint64_t grid = std::min<uint64_t>((n + kThreads - 1) / kThreads, uint64_t(ctx.sm_count(gpu)) * 8);
  if (padded && grid)
    index_pad_kernel<<<unsigned(grid), kThreads, 0, st>>>(reinterpret_cast<const unsigned long long*>(samples),
                                                          reinterpret_cast<unsigned long long*>(padded), n);
  ck(cudaGetLastError(), "index pad launch");
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t.launches = padded && grid ? 1 : 0, t.bytes = 32 * n;
  return t;
}

uint64_t repartition_scratch_bytes(uint64_t count) {
  const uint64_t tiles = (count + kGTile - 1) / kGTile;  // the smaller tile of the variants
  // counter + flags + tile aggregates + tile prefixes; split2: + class bytes + the tile
  // scan's block aggregates / inclusive prefixes
  return 256 + align256(tiles * 4) + 2 * align256(tiles * sizeof(Agg)) + align256(count) +
         2 * align256((tiles + 1023) / 1024 * sizeof(Agg));
}

// One rank's split2 launch state: kernel parameters and its scratch carved into the tile
// counters / aggregates / class bytes / scan blocks (repartition_scratch_bytes).
struct K5Job {
  Params p;
  Outs o;
  Scratch s;
  unsigned char* cls = nullptr;
  Agg* blk = nullptr;
  uint64_t count = 0, tiles = 0, sblocks = 0;
};

K5Job k5_job(const DatasetIndexView& idx, uint64_t B, uint64_t at_step, uint64_t new_dp, uint64_t rank,
             const PartitionOut& out, void* scratch, uint64_t tile) {
  K5Job j;
  j.count = repartition_count(idx.n, B, at_step, new_dp, rank);
  if (j.count >= (1ull << 32)) raise(Errc::InvalidArgument, "partition above 2^32 samples (u32 queues)");
  j.tiles = (j.count + tile - 1) / tile;
  j.sblocks = (j.tiles + 1023) / 1024;
  char* sc = static_cast<char*>(scratch);
  const uint64_t tl = j.tiles;
  j.s = Scratch{reinterpret_cast<unsigned*>(sc), reinterpret_cast<unsigned*>(sc + 256),
                reinterpret_cast<Agg*>(sc + 256 + align256(tl * 4)),
                reinterpret_cast<Agg*>(sc + 256 + align256(tl * 4) + align256(tl * sizeof(Agg))), unsigned(tl)};
  const uint64_t b = B / new_dp, full = idx.n / B;
  using ull = unsigned long long;
  j.p = Params{reinterpret_cast<const ull*>(idx.perm), reinterpret_cast<const ull*>(idx.samples), idx.file_class, idx.n, B,
               at_step, b, rank, j.count, full > at_step ? (full - at_step) * b : 0, full};
  j.o = Outs{reinterpret_cast<ull*>(out.pos), reinterpret_cast<ull*>(out.ent), reinterpret_cast<ull*>(out.boff),
             out.queue[0], out.queue[1], out.queue[2], reinterpret_cast<ull*>(out.qcount)};
  j.cls = reinterpret_cast<unsigned char*>(sc + 256 + align256(tl * 4) + 2 * align256(tl * sizeof(Agg)));
  j.blk = reinterpret_cast<Agg*>(j.cls + align256(j.count));
  return j;
}

// split2's gather pass (the dominant kernel) for one rank
void k5_gather(const K5Job& j, const K5Mode& mode, bool pad, cudaStream_t st) {
  K5Job k = j;  // the kernels take their arguments by value
  const unsigned g = unsigned(k.tiles);
  const int ld = pad ? k5_load() : 0;
  if (mode.minb == 8) {
    if (ld == 0) repart_gather2_kernel<8, 0><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else repart_gather2_kernel<8, 1><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
  } else if (mode.minb == 6) {
    if (ld == 0) repart_gather2_kernel<6, 0><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else if (ld == 1) repart_gather2_kernel<6, 1><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else if (ld == 2) repart_gather2_kernel<6, 2><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else repart_gather2_kernel<6, 3><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
  } else {
    if (ld == 0) repart_gather2_kernel<5, 0><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else if (ld == 1) repart_gather2_kernel<5, 1><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else if (ld == 2) repart_gather2_kernel<5, 2><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
    else repart_gather2_kernel<5, 3><<<g, kThreads, 0, st>>>(k.p, k.o, k.s, k.cls);
  }
}

// split2's tile scan + finalize for one rank (after its gather pass on the same or another stream)
void k5_finish(const K5Job& j, cudaStream_t st) {
  K5Job k = j;
  repart_tile_scan_kernel<<<unsigned(k.sblocks), 1024, 0, st>>>(k.s, k.blk, k.blk + k.sblocks, k.o);
  repart_finalize2_kernel<<<unsigned(k.tiles), kThreads, 0, st>>>(k.p, k.o, k.s.inc, k.cls);
}

Timing repartition_device(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                          uint64_t new_dp, uint64_t rank, const PartitionOut& out, void* scratch) {
  TraceRange trace_("repartition_device");
  const bool pad = entry_padded(idx);
  const K5Mode mode = k5_mode();
  const K5Job j = k5_job(idx, B, at_step, new_dp, rank, out, scratch, mode.lookback ? kTile : kGTile);
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  L2FetchScope l2fetch;
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  cudaEvent_t e0, e1, em;  // em: end of the gather pass (the dominant kernel)
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventCreate(&em), "event");
  if (mode.lookback && pad) raise(Errc::InvalidArgument, "RESHARD_K5=lookback reads the packed index only");
  if (mode.lookback) ck(cudaMemsetAsync(scratch, 0, 256 + align256(j.tiles * 4), st), "clear scratch");
  ck(cudaEventRecord(e0, st), "event");
  if (j.tiles && !mode.lookback) {
    k5_gather(j, mode, pad, st);
    ck(cudaEventRecord(em, st), "event");
    k5_finish(j, st);
    ck(cudaGetLastError(), "repartition launch");
  } else if (j.tiles) {
    K5Job k = j;
    if (mode.minb == 4) repartition_kernel<4><<<unsigned(k.tiles), kThreads, 0, st>>>(k.p, k.o, k.s);
    else repartition_kernel<3><<<unsigned(k.tiles), kThreads, 0, st>>>(k.p, k.o, k.s);
    ck(cudaGetLastError(), "repartition launch");
  } else {
    ck(cudaMemsetAsync(out.qcount, 0, 3 * sizeof(uint64_t), st), "qcount");
  }
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  if (j.tiles && !mode.lookback) ck(cudaEventElapsedTime(&t.main_ms, e0, em), "elapsed");
  else t.main_ms = t.ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(em);
  t.tiles = j.tiles;
  t.bytes = j.count * (8 + 24 + 8 + 24 + 8 + 4);  // algorithmic: perm+entry in, pos+entry+boff+queue out
  t.launches = j.tiles ? (mode.lookback ? 1 : 3) : 0;
  return t;
}

// Every rank of the batch in ONE launch per pass (gather, tile scan, finalize): no launch tail
// between ranks and one full-GPU finalize over all of them.  The rank table goes to the device
// on the stream (stream-ordered pool memory, freed on the stream after the last pass).
Timing repartition_fused(cudaStream_t st, const std::vector<K5Job>& kj, const RepartJob* jobs, const K5Mode& mode,
                         bool pad, std::vector<Timing>* per_job) {
  (void)mode;
  // the non-empty ranks in launch chunks of <= kMaxRanksPerLaunch; block offsets per chunk
  const char* fv = std::getenv("RESHARD_K5_FIN_TILES");
  const unsigned fin_tiles = fv && *fv ? unsigned(std::max(1, std::atoi(fv))) : kFinTiles;
  const char* mv = std::getenv("RESHARD_K5_FIN_MINB");  // A/B: resident finalize blocks per SM the compiler targets
  const int fin_minb = mv && *mv ? std::atoi(mv) : 0;
  std::vector<RankTable> chunks;
  std::vector<unsigned> chunk_tiles, chunk_sblocks, chunk_fin;
  for (size_t i = 0; i < kj.size(); ++i) {
    if (!kj[i].tiles) continue;
    if (chunks.empty() || chunks.back().n == kMaxRanksPerLaunch) {
      chunks.emplace_back();
      chunks.back().n = 0;
      chunk_tiles.push_back(0), chunk_sblocks.push_back(0), chunk_fin.push_back(0);
    }
    RankTable& t = chunks.back();
    unsigned& tl = chunk_tiles.back();
    unsigned& sb = chunk_sblocks.back();
    unsigned& fb = chunk_fin.back();
    if (uint64_t(tl) + kj[i].tiles >= (1ull << 31)) raise(Errc::InvalidArgument, "batch above 2^31 tiles per launch");
    t.r[t.n++] = RankK5{kj[i].p, kj[i].o, kj[i].s, kj[i].cls, kj[i].blk, tl, sb, fb};
    tl += unsigned(kj[i].tiles), sb += unsigned(kj[i].sblocks);
    fb += unsigned((kj[i].tiles + fin_tiles - 1) / fin_tiles);
  }
  cudaEvent_t e0, eg, em, e1;  // batch start, gather start / end, batch end
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&eg), "event");
  ck(cudaEventCreate(&em), "event");
  ck(cudaEventCreate(&e1), "event");
  struct Free {
    cudaEvent_t a, b, c, d;
    ~Free() { cudaEventDestroy(a), cudaEventDestroy(b), cudaEventDestroy(c), cudaEventDestroy(d); }
  } free_{e0, eg, em, e1};
  ck(cudaEventRecord(e0, st), "event");
  for (size_t i = 0; i < kj.size(); ++i)
    if (!kj[i].tiles) ck(cudaMemsetAsync(jobs[i].out.qcount, 0, 3 * sizeof(uint64_t), st), "qcount");
  ck(cudaEventRecord(eg, st), "event");
  const int ld = pad ? k5_load() : 0;
  for (size_t c = 0; c < chunks.size(); ++c) {
    if (ld == 1) repart_gather2_multi_kernel<5, 1><<<chunk_tiles[c], kThreads, 0, st>>>(chunks[c]);
    else if (ld == 0) repart_gather2_multi_kernel<5, 0><<<chunk_tiles[c], kThreads, 0, st>>>(chunks[c]);
    else raise(Errc::InvalidArgument, "fused K5: the default gather variant only (split2, ldg)");
  }
  ck(cudaEventRecord(em, st), "event");
  for (size_t c = 0; c < chunks.size(); ++c) {
    repart_tile_scan_multi_kernel<<<chunk_sblocks[c], 1024, 0, st>>>(chunks[c]);
    if (fin_minb >= 6) repart_finalize2_multi_kernel<6><<<chunk_fin[c], kThreads, 0, st>>>(chunks[c], fin_tiles);
    else if (fin_minb == 5) repart_finalize2_multi_kernel<5><<<chunk_fin[c], kThreads, 0, st>>>(chunks[c], fin_tiles);
    else repart_finalize2_multi_kernel<1><<<chunk_fin[c], kThreads, 0, st>>>(chunks[c], fin_tiles);
  }
  ck(cudaGetLastError(), "repartition launch");
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  ck(cudaEventElapsedTime(&t.main_ms, eg, em), "elapsed");
  for (size_t i = 0; i < kj.size(); ++i) {
    Timing r;  // one launch per pass for the whole batch: per-rank times are not separable (0)
    r.tiles = kj[i].tiles, r.bytes = kj[i].count * (8 + 24 + 8 + 24 + 8 + 4);
    t.tiles += r.tiles, t.bytes += r.bytes;
    if (per_job) (*per_job)[i] = r;
  }
  t.launches = 3 * chunks.size();
  return t;
}

// Streams and events of one batch, released on every exit path (a failed launch raises).
struct BatchResources {
  cudaStream_t sg = nullptr, sf = nullptr;
  std::vector<cudaEvent_t> ev;
  ~BatchResources() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (sg) cudaStreamDestroy(sg);
    if (sf) cudaStreamDestroy(sf);
  }
};

Timing repartition_batch_device(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, const RepartJob* jobs,
                                size_t n, std::vector<Timing>* per_job) {
  TraceRange trace_("repartition_batch_device");
  const K5Mode mode = k5_mode();
  if (per_job) per_job->assign(n, Timing{});
  if (mode.lookback) {  // the single-pass variant: one rank after another
    Timing t;
    for (size_t i = 0; i < n; ++i) {
      DatasetIndexView v = idx;
      v.file_class = jobs[i].file_class;
      Timing r = repartition_device(ctx, gpu, v, B, jobs[i].at_step, jobs[i].new_dp, jobs[i].rank, jobs[i].out, jobs[i].scratch);
      if (per_job) (*per_job)[i] = r;
      t.ms += r.ms, t.main_ms += r.main_ms, t.tiles += r.tiles, t.bytes += r.bytes, t.launches += r.launches;
    }
    return t;
  }
  const bool pad = entry_padded(idx);
  std::vector<K5Job> kj;
  kj.reserve(n);
  for (size_t i = 0; i < n; ++i) {
    DatasetIndexView v = idx;
    v.file_class = jobs[i].file_class;
    kj.push_back(k5_job(v, B, jobs[i].at_step, jobs[i].new_dp, jobs[i].rank, jobs[i].out, jobs[i].scratch, kGTile));
  }
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  L2FetchScope l2fetch;
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  // fused: the default gather variant (5 CTAs / SM, __ldg records); other RESHARD_K5 /
  // RESHARD_K5_LOAD variants (A/B knobs) take the two-stream schedule
  const char* fv = std::getenv("RESHARD_K5_FUSE");
  const int ld = pad ? k5_load() : 0;
  if (!(fv && std::string(fv) == "0") && mode.minb == 5 && ld <= 1)
    return repartition_fused(st, kj, jobs, mode, pad, per_job);
  // sg: the gather passes, back to back, at the highest stream priority; sf: the ranks' tile
  // scans + finalizes at the lowest, so their blocks fill the gather passes' tails instead of
  // taking SMs from them (RESHARD_K5_PRIO=0: both at the default priority, A/B)
  int least = 0, greatest = 0;
  const char* pv = std::getenv("RESHARD_K5_PRIO");
  if (!(pv && std::string(pv) == "0")) ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  BatchResources res;
  ck(cudaStreamCreateWithPriority(&res.sg, cudaStreamNonBlocking, greatest), "stream");
  ck(cudaStreamCreateWithPriority(&res.sf, cudaStreamNonBlocking, least), "stream");
  cudaStream_t sg = res.sg, sf = res.sf;
  res.ev.assign(2 * n + 4, nullptr);
  std::vector<cudaEvent_t>& ev = res.ev;
  for (auto& e : ev) ck(cudaEventCreate(&e), "event");
  cudaEvent_t e0 = ev[2 * n], e1 = ev[2 * n + 1], ef = ev[2 * n + 2], eg = ev[2 * n + 3];
  ck(cudaEventRecord(e0, st), "event");
  ck(cudaStreamWaitEvent(sg, e0, 0), "wait");
  ck(cudaStreamWaitEvent(sf, e0, 0), "wait");
  for (size_t i = 0; i < n; ++i) {
    ck(cudaEventRecord(ev[2 * i], sg), "event");
    if (kj[i].tiles) {
      k5_gather(kj[i], mode, pad, sg);
      ck(cudaEventRecord(ev[2 * i + 1], sg), "event");
      ck(cudaStreamWaitEvent(sf, ev[2 * i + 1], 0), "wait gather");
      k5_finish(kj[i], sf);
    } else {
      ck(cudaMemsetAsync(jobs[i].out.qcount, 0, 3 * sizeof(uint64_t), sg), "qcount");
      ck(cudaEventRecord(ev[2 * i + 1], sg), "event");
    }
    ck(cudaGetLastError(), "repartition launch");
  }
  ck(cudaEventRecord(ef, sf), "event");
  ck(cudaEventRecord(eg, sg), "event");
  ck(cudaStreamWaitEvent(st, ef, 0), "join");
  ck(cudaStreamWaitEvent(st, eg, 0), "join");
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  for (size_t i = 0; i < n; ++i) {
    Timing r;
    ck(cudaEventElapsedTime(&r.main_ms, ev[2 * i], ev[2 * i + 1]), "elapsed");
    r.ms = r.main_ms;  // the scan + finalize overlap the next gather pass: not attributable
    r.tiles = kj[i].tiles, r.launches = kj[i].tiles ? 3 : 0;
    r.bytes = kj[i].count * (8 + 24 + 8 + 24 + 8 + 4);
    t.main_ms += r.main_ms, t.tiles += r.tiles, t.bytes += r.bytes, t.launches += r.launches;
    if (per_job) (*per_job)[i] = r;
  }
  return t;
}

Timing repartition_to_host(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                           uint64_t new_dp, uint64_t rank, const PartitionOut& out, void* scratch,
                           const PartitionHost& host) {
  TraceRange trace_("repartition_to_host");
  const uint64_t count = repartition_count(idx.n, B, at_step, new_dp, rank);
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  cudaEvent_t e0, e1;
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventRecord(e0, st), "event");
  Timing t = repartition_device(ctx, gpu, idx, B, at_step, new_dp, rank, out, scratch);
  // the queue lengths decide how much of each queue comes back: read them first
  ck(cudaMemcpyAsync(host.qcount, out.qcount, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "D2H qcount");
  ck(cudaMemcpyAsync(host.pos, out.pos, 8 * count, cudaMemcpyDeviceToHost, st), "D2H pos");
  ck(cudaMemcpyAsync(host.ent, out.ent, 24 * count, cudaMemcpyDeviceToHost, st), "D2H ent");
  ck(cudaMemcpyAsync(host.boff, out.boff, 8 * count, cudaMemcpyDeviceToHost, st), "D2H boff");
  ck(cudaStreamSynchronize(st), "sync");
  uint64_t qbytes = 0;
  for (int c = 0; c < 3; ++c) {
    if (host.qcount[c] > count) raise(Errc::CudaError, "repartition_to_host: queue length above the count");
    if (host.qcount[c])
      ck(cudaMemcpyAsync(host.queue[c], out.queue[c], 4 * host.qcount[c], cudaMemcpyDeviceToHost, st), "D2H queue");
    qbytes += 4 * host.qcount[c];
  }
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t.bytes = 24 + 40 * count + qbytes;  // D2H bytes
  return t;
}

Timing repartition_gather_probe(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                                uint64_t new_dp, uint64_t rank, int reps) {
  const uint64_t count = repartition_count(idx.n, B, at_step, new_dp, rank);
  const bool pad = entry_padded(idx);
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  const uint64_t b = B / new_dp, full = idx.n / B;
  using ull = unsigned long long;
  Params p{reinterpret_cast<const ull*>(idx.perm), reinterpret_cast<const ull*>(idx.samples), idx.file_class, idx.n, B,
           at_step, b, rank, count, full > at_step ? (full - at_step) * b : 0, full};
  const uint64_t per = uint64_t(kThreads) * kProbeItems, blocks = (count + per - 1) / per;
  ull* sink = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&sink), sizeof(ull), st), "cudaMallocAsync");
  // default: the gather + write floor (scratch outputs of 44 B / sample); RESHARD_PROBE=read:
  // the gathers alone
  const bool wr = !(std::getenv("RESHARD_PROBE") && std::string(std::getenv("RESHARD_PROBE")) == "read");
  void* wbuf = nullptr;
  Outs wo{};
  if (wr && count) {
    ck(cudaMallocAsync(&wbuf, count * 44 + 256, st), "cudaMallocAsync");
    char* w = static_cast<char*>(wbuf);
    wo.pos = reinterpret_cast<ull*>(w), wo.ent = reinterpret_cast<ull*>(w + 8 * count);
    wo.boff = reinterpret_cast<ull*>(w + 32 * count), wo.q0 = reinterpret_cast<unsigned*>(w + 40 * count);
  }
  L2FetchScope l2fetch;
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  Timing t;
  t.ms = 1e30f;
  for (int i = 0; i < std::max(1, reps) + 1; ++i) {  // first launch warms up
    ck(cudaEventRecord(e0, st), "event");
    const int ld = pad ? k5_load() : 0;
    auto launch = [&](auto wk, auto gk) {
      if (blocks && wr) wk<<<unsigned(blocks), kThreads, 0, st>>>(p, wo);
      else if (blocks) gk<<<unsigned(blocks), kThreads, 0, st>>>(p, sink);
    };
    if (ld == 0) launch(gather_write_probe_kernel<0>, gather_probe_kernel<0>);
    else if (ld == 1) launch(gather_write_probe_kernel<1>, gather_probe_kernel<1>);
    else if (ld == 2) launch(gather_write_probe_kernel<2>, gather_probe_kernel<2>);
    else launch(gather_write_probe_kernel<3>, gather_probe_kernel<3>);
    ck(cudaGetLastError(), "probe launch");
    ck(cudaEventRecord(e1, st), "event");
    ck(cudaEventSynchronize(e1), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    if (i > 0) t.ms = std::min(t.ms, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ck(cudaFreeAsync(sink, st), "cudaFreeAsync");
  if (wbuf) ck(cudaFreeAsync(wbuf, st), "cudaFreeAsync");
  t.tiles = blocks, t.launches = blocks ? 1 : 0, t.bytes = count * (8 + 24);
  return t;
}

}  // namespace reshard
