// K5 dataset_repartition (sm_100a): for one new DP rank, in ONE pass over its remaining
// samples —
//   pos[k]  = closed-form global position,
//   ent[k]  = samples[perm[pos[k]]]                (24-byte gather through the permutation),
//   boff[k] = exclusive prefix sum of lengths       (the sample's offset in the read buffer),
//   queue[class] += k                               (stable compaction by locator class,
//                                                    local > peer > remote).
// The scan is a single-pass decoupled look-back: each CTA takes the next tile from an
// atomic counter (so it only ever waits on tiles already owned by running CTAs), scans its
// 2048 items with warp shuffles, publishes its aggregate, looks back over predecessors'
// aggregates / inclusive prefixes, and publishes its inclusive prefix.
// Replaces the CPU loops of oracle.cpp orc_dataset_gather (SPEC restatement).
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "reshard/dataset.hpp"

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

// ---- K5 persistent variant: tiles software-pipelined across the look-back ---------------------
// r13 profile of the single-pass kernel: 41 % of warp samples wait at the barrier behind the
// look-back while no gather of that CTA is in flight.  Here each CTA keeps pulling tiles in
// order and runs two tiles ahead: while tile T is scanned (look-back, offsets, queues), the
// entry gathers of T+1 and the permutation reads of T+2 are already in flight.  Tiles are
// 1024 samples (4 per thread) so three tiles' worth of loads fit the register budget.
constexpr int kPItems = 4, kPTile = kThreads * kPItems;

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

// Position (in the epoch order) of the rank's k-th remaining sample and the cursor after it.
struct PosCursor {
  unsigned long long batch, r;
};
__device__ __forceinline__ PosCursor pos_cursor(const Params& p, unsigned long long k) {
  return k < p.in_full ? PosCursor{p.at_step + k / p.b, k % p.b} : PosCursor{0, 0};
}
__device__ __forceinline__ unsigned long long next_pos(const Params& p, PosCursor& c, unsigned long long k) {
  if (k < p.in_full) {
    const unsigned long long pos = c.batch * p.B + p.rank * p.b + c.r;
    if (++c.r == p.b) c.r = 0, ++c.batch;
    return pos;
  }
  return p.full * p.B + p.rank * p.b + (k - p.in_full);
}

__device__ __forceinline__ void load_perm(const Params& p, unsigned tile, unsigned long long (&idx)[kPItems]) {
  const unsigned long long k0 = (unsigned long long)tile * kPTile + (unsigned long long)threadIdx.x * kPItems;
  PosCursor c = pos_cursor(p, k0);
#pragma unroll
  for (int j = 0; j < kPItems; ++j) {
    const unsigned long long k = k0 + j;
    const unsigned long long pos = next_pos(p, c, k);
    idx[j] = k < p.count ? __ldg(p.perm + pos) : 0ull;
  }
}
struct Entries {
  unsigned long long f[kPItems], off[kPItems], len[kPItems];
};
__device__ __forceinline__ void load_entries(const Params& p, const unsigned long long (&idx)[kPItems], Entries& e) {
#pragma unroll
  for (int j = 0; j < kPItems; ++j) {
    const unsigned long long* q = p.samples + 3 * idx[j];
    e.f[j] = __ldg(q), e.off[j] = __ldg(q + 1), e.len[j] = __ldg(q + 2);
  }
}

template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB) repartition_persistent_kernel(Params p, Outs o, Scratch s) {
  __shared__ unsigned next_sh;
  __shared__ Agg warp_tot[kWarps];
  __shared__ Agg tile_prefix;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) next_sh = atomicAdd(s.counter, 1u);
  __syncthreads();
  unsigned cur = next_sh;
  __syncthreads();
  if (threadIdx.x == 0) next_sh = atomicAdd(s.counter, 1u);
  __syncthreads();
  unsigned nxt = next_sh;
  __syncthreads();  // everyone has read nxt before thread 0 overwrites next_sh in the loop
  unsigned long long idx[kPItems];
  Entries ec, en;
  if (cur < s.ntiles) {
    load_perm(p, cur, idx);
    load_entries(p, idx, ec);
  }
  if (nxt < s.ntiles) load_perm(p, nxt, idx);
  while (cur < s.ntiles) {
    // (1) gathers of the next tile, (2) permutation reads of the one after, both in flight
    // while the current tile is scanned
    if (nxt < s.ntiles) load_entries(p, idx, en);
    if (threadIdx.x == 0) next_sh = atomicAdd(s.counter, 1u);
    // (3) the current tile: class lookups, pos / entry stores, block scan, look-back
    const unsigned long long k0 = (unsigned long long)cur * kPTile + (unsigned long long)threadIdx.x * kPItems;
    unsigned char cls[kPItems];
    Agg mine{0, 0, 0, 0};
    PosCursor c = pos_cursor(p, k0);
#pragma unroll
    for (int j = 0; j < kPItems; ++j) {
      const unsigned long long k = k0 + j;
      const unsigned long long pos = next_pos(p, c, k);
      cls[j] = 3;
      if (k < p.count) {
        cls[j] = __ldg(p.file_class + ec.f[j]);
        o.pos[k] = pos;
        o.ent[3 * k] = ec.f[j], o.ent[3 * k + 1] = ec.off[j], o.ent[3 * k + 2] = ec.len[j];
        mine.len += ec.len[j];
        mine.c0 += cls[j] == 0, mine.c1 += cls[j] == 1, mine.c2 += cls[j] == 2;
      }
    }
    Agg inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Agg up = shfl_up(inc, d);
      if (lane >= d) inc = inc + up;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();  // barrier 1: warp totals and next_sh visible
    const unsigned after = next_sh;
    Agg warp_base{0, 0, 0, 0}, total{0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      if (w < warp) warp_base = warp_base + warp_tot[w];
      total = total + warp_tot[w];
    }
    if (after < s.ntiles) load_perm(p, after, idx);
    if (warp == 0) {
      const Agg prefix = decoupled_lookback(cur, total, s, lane);
      if (lane == 0) {
        tile_prefix = prefix;
        if (cur == s.ntiles - 1) {
          const Agg all = prefix + total;
          o.qcount[0] = all.c0, o.qcount[1] = all.c1, o.qcount[2] = all.c2;
        }
      }
    }
    __syncthreads();  // barrier 2: tile prefix visible
    Agg run = tile_prefix + warp_base +
              Agg{inc.len - mine.len, inc.c0 - mine.c0, inc.c1 - mine.c1, inc.c2 - mine.c2};
#pragma unroll
    for (int j = 0; j < kPItems; ++j) {
      const unsigned long long k = k0 + j;
      if (k >= p.count) break;
      o.boff[k] = run.len;
      run.len += ec.len[j];
      if (cls[j] == 0) o.q0[run.c0++] = unsigned(k);
      else if (cls[j] == 1) o.q1[run.c1++] = unsigned(k);
      else o.q2[run.c2++] = unsigned(k);
    }
    cur = nxt, nxt = after, ec = en;
  }
}

// ---- random-gather ceiling (diagnostic) -----------------------------------------------------
// K5's two HBM-random levels alone — the rank's perm positions, one 24-byte entry gather per
// position, nothing written but one word per thread — at the configuration the standalone
// probe found fastest (4 items per thread, 256 threads; scripts/probe_gather.cu, profiles/r12).
// Its time is the floor for any kernel that must gather these entries: bench.py reports K5
// against it next to the streaming-HBM roofline.
constexpr int kProbeItems = 4;
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
    const unsigned long long* e = p.samples + 3 * idx[j];
    f[j] = __ldg(e), off[j] = __ldg(e + 1), len[j] = __ldg(e + 2);
  }
#pragma unroll
  for (int j = 0; j < kProbeItems; ++j) acc ^= f[j] + off[j] + len[j];
  if (acc == 0x9e3779b97f4a7c15ull) *sink = acc;  // keeps the loads; practically never stores
}

// ---- K5 split variant: gather / scan / finalize -------------------------------------------
// r05 profile: 27% of the single-pass kernel's stall samples sit behind the block barrier
// that waits for the decoupled look-back.  The split variant never waits: (a) a pure
// gather kernel writes pos / entry, parks each sample's length in boff and its class in a
// byte array, and reduces one aggregate per tile; (b) one CTA scans the tile aggregates;
// (c) a streaming kernel turns lengths into offsets and fills the locator queues.  Extra
// traffic: 9 bytes per sample written and read back (~5% of the gather's DRAM bytes).
__device__ __forceinline__ Agg block_exclusive(const Agg& mine, Agg* warp_tot, Agg& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Agg inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Agg up = shfl_up(inc, d);
    if (lane >= d) inc = inc + up;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  Agg base{0, 0, 0, 0};
  total = Agg{0, 0, 0, 0};
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) base = base + warp_tot[w];
    total = total + warp_tot[w];
  }
  return base + Agg{inc.len - mine.len, inc.c0 - mine.c0, inc.c1 - mine.c1, inc.c2 - mine.c2};
}

__global__ void __launch_bounds__(kThreads) repart_gather_kernel(Params p, Outs o, Agg* agg, unsigned char* cls_out) {
  __shared__ Agg warp_tot[kWarps];
  const unsigned long long k0 = (unsigned long long)blockIdx.x * kTile + (unsigned long long)threadIdx.x * kItems;
  unsigned long long batch = 0, r = 0;
  if (k0 < p.in_full) batch = p.at_step + k0 / p.b, r = k0 % p.b;
  unsigned long long pos[kItems], idx[kItems], f[kItems], off[kItems], len[kItems];
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
  Agg mine{0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (j >= nv) continue;
    const unsigned long long k = k0 + j;
    const unsigned char c = __ldg(p.file_class + f[j]);
    o.pos[k] = pos[j];
    o.ent[3 * k] = f[j], o.ent[3 * k + 1] = off[j], o.ent[3 * k + 2] = len[j];
    o.boff[k] = len[j];  // parked; finalize turns it into the offset
    cls_out[k] = c;
    mine.len += len[j];
    mine.c0 += c == 0, mine.c1 += c == 1, mine.c2 += c == 2;
  }
  Agg total;
  block_exclusive(mine, warp_tot, total);
  if (threadIdx.x == 0) agg[blockIdx.x] = total;
}

// One CTA: exclusive scan of the tile aggregates, and the queue totals.
__global__ void __launch_bounds__(1024) repart_scan_kernel(const Agg* agg, Agg* prefix, unsigned ntiles, Outs o) {
  __shared__ Agg warp_tot[32];
  const unsigned per = (ntiles + blockDim.x - 1) / blockDim.x;
  const unsigned t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
  Agg mine{0, 0, 0, 0};
  for (unsigned t = t0; t < t1; ++t) mine = mine + agg[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Agg inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Agg up = shfl_up(inc, d);
    if (lane >= d) inc = inc + up;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  Agg base{0, 0, 0, 0}, total{0, 0, 0, 0};
  for (int w = 0; w < int(blockDim.x >> 5); ++w) {
    if (w < warp) base = base + warp_tot[w];
    total = total + warp_tot[w];
  }
  Agg run = base + Agg{inc.len - mine.len, inc.c0 - mine.c0, inc.c1 - mine.c1, inc.c2 - mine.c2};
  for (unsigned t = t0; t < t1; ++t) {
    prefix[t] = run;
    run = run + agg[t];
  }
  if (threadIdx.x == 0) o.qcount[0] = total.c0, o.qcount[1] = total.c1, o.qcount[2] = total.c2;
}

__global__ void __launch_bounds__(kThreads) repart_finalize_kernel(Params p, Outs o, const Agg* prefix,
                                                                   const unsigned char* cls_in) {
  __shared__ Agg warp_tot[kWarps];
  const unsigned long long k0 = (unsigned long long)blockIdx.x * kTile + (unsigned long long)threadIdx.x * kItems;
  unsigned long long len[kItems];
  unsigned char cls[kItems];
  Agg mine{0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long k = k0 + j;
    len[j] = k < p.count ? o.boff[k] : 0ull;
    cls[j] = k < p.count ? cls_in[k] : (unsigned char)3;
    mine.len += len[j];
    mine.c0 += cls[j] == 0, mine.c1 += cls[j] == 1, mine.c2 += cls[j] == 2;
  }
  Agg total;
  const Agg excl = block_exclusive(mine, warp_tot, total);
  Agg run = prefix[blockIdx.x] + excl;
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

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}
uint64_t align256(uint64_t x) { return (x + 255) / 256 * 256; }

bool k5_split() {
  const char* v = std::getenv("RESHARD_K5");
  // r11: split 6.59 ms vs single-pass 6.38 ms per step; r13 (single-pass with pos stored
  // early, 80 regs and no spills): 6.57 vs 6.78 — that change was reverted
  return v && std::string(v) == "split";
}
// resident CTAs per SM the single-pass kernel is compiled for (RESHARD_K5=lookback4: 4)
int k5_min_blocks() {
  const char* v = std::getenv("RESHARD_K5");
  return v && std::string(v) == "lookback4" ? 4 : 3;
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
// H[i] is computed up front.  Iteration i may run once no earlier (higher-index) pending
// iteration touches location i or H[i]: each round, every pending iteration reserves both
// its locations with atomicMax of (round << 32 | i); an iteration holding both
// reservations swaps, the others carry over to the next round.  The result is identical
// to the sequential loop (Shun et al., SODA'15, "deterministic reservations"); rounds are
// O(log N) (about 70 for N = 10^8).
__device__ __forceinline__ unsigned long long mix64d(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void shuffle_init_kernel(unsigned long long* perm, unsigned long long* resv, unsigned long long* list,
                                    unsigned long long n, unsigned long long s0) {
  for (unsigned long long x = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; x < n;
       x += (unsigned long long)gridDim.x * blockDim.x) {
    perm[x] = x;
    resv[x] = 0;
    if (x >= 1) {
      const unsigned long long draw = mix64d(s0 + (n - x) * 0x9e3779b97f4a7c15ull);  // draw number n-1-x
      list[x - 1] = (x << 32) | (draw % (x + 1));
    }
  }
}

__global__ void shuffle_reserve_kernel(const unsigned long long* __restrict__ list, const unsigned* __restrict__ count,
                                       unsigned long long* resv, unsigned long long round) {
  const unsigned n = *count;
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const unsigned long long e = list[k], i = e >> 32, h = e & 0xffffffffull;
    const unsigned long long key = (round << 32) | i;
    atomicMax(resv + i, key);
    if (h != i) atomicMax(resv + h, key);
  }
}

__global__ void shuffle_commit_kernel(const unsigned long long* __restrict__ list, const unsigned* __restrict__ count,
                                      const unsigned long long* __restrict__ resv, unsigned long long* perm,
                                      unsigned long long* next, unsigned* next_count, unsigned long long round) {
  const unsigned n = *count;
  const unsigned lane = threadIdx.x & 31;
  // grid-stride with whole-warp trip counts so the ballot below is warp-uniform
  for (unsigned base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; base < n; base += gridDim.x * blockDim.x) {
    const unsigned k = base + lane;
    bool pending = false;
    unsigned long long e = 0;
    if (k < n) {
      e = list[k];
      const unsigned long long i = e >> 32, h = e & 0xffffffffull, key = (round << 32) | i;
      if (__ldcg(resv + i) == key && __ldcg(resv + h) == key) {
        if (h != i) {
          const unsigned long long a = perm[i];
          perm[i] = perm[h];
          perm[h] = a;
        }
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

}  // namespace

uint64_t shuffle_scratch_bytes(uint64_t n) { return 256 + 3 * align256(n * 8); }

Timing shuffle_epoch_device(Context& ctx, int gpu, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm, void* scratch) {
  if (n >= (1ull << 32)) raise(Errc::InvalidArgument, "GPU shuffle supports N < 2^32");
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  L2FetchScope l2fetch;
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  char* sc = static_cast<char*>(scratch);
  auto* counts = reinterpret_cast<unsigned*>(sc);  // [2] list sizes (ping-pong)
  auto* resv = reinterpret_cast<unsigned long long*>(sc + 256);
  unsigned long long* lists[2] = {reinterpret_cast<unsigned long long*>(sc + 256 + align256(n * 8)),
                                  reinterpret_cast<unsigned long long*>(sc + 256 + 2 * align256(n * 8))};
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  ck(cudaEventRecord(e0, st), "event");
  Timing t;
  unsigned* pinned = nullptr;
  ck(cudaMallocHost(&pinned, sizeof(unsigned)), "pinned");
  const unsigned init = n ? unsigned(n - 1) : 0u;
  ck(cudaMemcpyAsync(counts, &init, sizeof(unsigned), cudaMemcpyHostToDevice, st), "count");
  const int grid_full = 148 * 8;
  shuffle_init_kernel<<<grid_full, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(perm), resv, lists[0], n,
                                                 seed ^ epoch);
  ck(cudaGetLastError(), "shuffle init");
  t.launches = 1;
  unsigned pending = init;
  for (unsigned long long round = 1, cur = 0; pending > 0; ++round, cur ^= 1) {
    const int grid = int(std::min<unsigned long long>(grid_full, (pending + 255) / 256));
    ck(cudaMemsetAsync(counts + (cur ^ 1), 0, sizeof(unsigned), st), "reset count");
    shuffle_reserve_kernel<<<grid, 256, 0, st>>>(lists[cur], counts + cur, resv, round);
    shuffle_commit_kernel<<<grid, 256, 0, st>>>(lists[cur], counts + cur, resv, reinterpret_cast<unsigned long long*>(perm),
                                                lists[cur ^ 1], counts + (cur ^ 1), round);
    ck(cudaGetLastError(), "shuffle round");
    t.launches += 2;
    ck(cudaMemcpyAsync(pinned, counts + (cur ^ 1), sizeof(unsigned), cudaMemcpyDeviceToHost, st), "count d2h");
    ck(cudaStreamSynchronize(st), "shuffle sync");
    pending = *pinned;
    t.tiles = round;  // rounds
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

// RESHARD_K5=persistent: 2 CTAs per SM (no spills); persistent3: 3 CTAs per SM (spills)
int k5_persistent() {
  const char* v = std::getenv("RESHARD_K5");
  if (!v) return 0;
  const std::string s(v);
  return s == "persistent" ? 2 : s == "persistent3" ? 3 : 0;
}

uint64_t repartition_scratch_bytes(uint64_t count) {
  const uint64_t tiles = (count + kPTile - 1) / kPTile;  // the smallest tile of the variants
  // look-back: counter + flags + aggregates + inclusive prefixes; split: + class bytes
  return 256 + align256(tiles * 4) + 2 * align256(tiles * sizeof(Agg)) + align256(count);
}

Timing repartition_device(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                          uint64_t new_dp, uint64_t rank, const PartitionOut& out, void* scratch) {
  const uint64_t count = repartition_count(idx.n, B, at_step, new_dp, rank);
  if (count >= (1ull << 32)) raise(Errc::InvalidArgument, "partition above 2^32 samples (u32 queues)");
  const int persistent = k5_persistent();  // resident CTAs per SM, 0: not persistent
  const uint64_t tile = persistent ? kPTile : kTile;
  const uint64_t tiles = (count + tile - 1) / tile;
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  L2FetchScope l2fetch;
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  char* sc = static_cast<char*>(scratch);
  Scratch s{reinterpret_cast<unsigned*>(sc), reinterpret_cast<unsigned*>(sc + 256),
            reinterpret_cast<Agg*>(sc + 256 + align256(tiles * 4)),
            reinterpret_cast<Agg*>(sc + 256 + align256(tiles * 4) + align256(tiles * sizeof(Agg))), unsigned(tiles)};
  const uint64_t b = B / new_dp, full = idx.n / B;
  using ull = unsigned long long;
  Params p{reinterpret_cast<const ull*>(idx.perm), reinterpret_cast<const ull*>(idx.samples), idx.file_class, idx.n, B,
           at_step, b, rank, count, full > at_step ? (full - at_step) * b : 0, full};
  Outs o{reinterpret_cast<ull*>(out.pos), reinterpret_cast<ull*>(out.ent), reinterpret_cast<ull*>(out.boff),
         out.queue[0], out.queue[1], out.queue[2], reinterpret_cast<ull*>(out.qcount)};
  const bool split = k5_split();
  if (!split) ck(cudaMemsetAsync(scratch, 0, 256 + align256(tiles * 4), st), "clear scratch");
  ck(cudaEventRecord(e0, st), "event");
  if (tiles && split) {
    auto* cls = reinterpret_cast<unsigned char*>(sc + 256 + align256(tiles * 4) + 2 * align256(tiles * sizeof(Agg)));
    repart_gather_kernel<<<unsigned(tiles), kThreads, 0, st>>>(p, o, s.agg, cls);
    repart_scan_kernel<<<1, 1024, 0, st>>>(s.agg, s.inc, unsigned(tiles), o);
    repart_finalize_kernel<<<unsigned(tiles), kThreads, 0, st>>>(p, o, s.inc, cls);
    ck(cudaGetLastError(), "repartition launch");
  } else if (tiles && persistent) {
    const uint64_t grid = std::min<uint64_t>(tiles, uint64_t(ctx.sm_count(gpu)) * uint64_t(persistent));
    if (persistent == 3) repartition_persistent_kernel<3><<<unsigned(grid), kThreads, 0, st>>>(p, o, s);
    else repartition_persistent_kernel<2><<<unsigned(grid), kThreads, 0, st>>>(p, o, s);
    ck(cudaGetLastError(), "repartition launch");
  } else if (tiles) {
    if (k5_min_blocks() == 4) repartition_kernel<4><<<unsigned(tiles), kThreads, 0, st>>>(p, o, s);
    else repartition_kernel<3><<<unsigned(tiles), kThreads, 0, st>>>(p, o, s);
    ck(cudaGetLastError(), "repartition launch");
  } else {
    ck(cudaMemsetAsync(out.qcount, 0, 3 * sizeof(uint64_t), st), "qcount");
  }
  ck(cudaEventRecord(e1, st), "event");
  ck(cudaEventSynchronize(e1), "sync");
  Timing t;
  ck(cudaEventElapsedTime(&t.ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  t.tiles = tiles;
  t.bytes = count * (8 + 24 + 8 + 24 + 8 + 4);  // algorithmic: perm+entry in, pos+entry+boff+queue out
  t.launches = tiles ? (split ? 3 : 1) : 0;
  return t;
}

Timing repartition_gather_probe(Context& ctx, int gpu, const DatasetIndexView& idx, uint64_t B, uint64_t at_step,
                                uint64_t new_dp, uint64_t rank, int reps) {
  const uint64_t count = repartition_count(idx.n, B, at_step, new_dp, rank);
  ck(cudaSetDevice(ctx.cuda_device(gpu)), "cudaSetDevice");
  auto st = static_cast<cudaStream_t>(ctx.stream(gpu));
  const uint64_t b = B / new_dp, full = idx.n / B;
  using ull = unsigned long long;
  Params p{reinterpret_cast<const ull*>(idx.perm), reinterpret_cast<const ull*>(idx.samples), idx.file_class, idx.n, B,
           at_step, b, rank, count, full > at_step ? (full - at_step) * b : 0, full};
  const uint64_t per = uint64_t(kThreads) * kProbeItems, blocks = (count + per - 1) / per;
  ull* sink = nullptr;
  ck(cudaMallocAsync(reinterpret_cast<void**>(&sink), sizeof(ull), st), "cudaMallocAsync");
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  Timing t;
  t.ms = 1e30f;
  for (int i = 0; i < std::max(1, reps) + 1; ++i) {  // first launch warms up
    ck(cudaEventRecord(e0, st), "event");
    if (blocks) gather_probe_kernel<<<unsigned(blocks), kThreads, 0, st>>>(p, sink);
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
  t.tiles = blocks, t.launches = blocks ? 1 : 0, t.bytes = count * (8 + 24);
  return t;
}

}  // namespace reshard
