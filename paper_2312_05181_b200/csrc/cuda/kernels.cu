// sm_100a kernels of the reshard data plane.
//
//  K1/K2 copy_tiles  — persistent strided sub-tensor copy.  Replaces the reference row walker
//                      (proj/src/tensor/tensor.cpp:35-57) and the memcpy loops of slice()
//                      (:73-76) and merge() (:108-111).  One CTA per tile at a time; a tile is
//                      rows x row_bytes with independent src/dst pitches, moved with the
//                      widest common alignment (16 B vectors for every GPT-catalog tile).
//                      Loads are non-coherent streaming loads (L1 no-allocate, 256 B L2
//                      prefetch); a tile whose dst is a peer mapping stores over NVLink (K2).
//  K6 fill_cell      — counter-based splitmix64 payload (proj/include/reshard/util/hash.hpp:46-51)
//                      for any sub-box of a base tensor, bit-identical to the CPU stream.
//  K7 verify_cell    — regenerates K6's bytes and counts mismatches (off the clock).
#include <cuda_runtime.h>

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
// of the flattened rows x (row_bytes/W) index space; (row, col) advance incrementally, so
// there is no per-vector division.  U vectors are loaded before any is stored.
template <typename V, int U>
__device__ __forceinline__ void copy_tile(const DevTile& t) {
  constexpr unsigned W = sizeof(V);
  const unsigned vpr = t.row_bytes / W;
  const unsigned long long n = (unsigned long long)t.rows * vpr;
  const unsigned B = blockDim.x;
  const unsigned drow = B / vpr, dcol = B % vpr;
  unsigned row = threadIdx.x / vpr, col = threadIdx.x % vpr;
  const char* __restrict__ s = reinterpret_cast<const char*>(t.src);
  char* __restrict__ d = reinterpret_cast<char*>(t.dst);
  for (unsigned long long i = threadIdx.x; i < n; i += (unsigned long long)U * B) {
    V v[U];
    unsigned rr[U], cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rr[u] = row, cc[u] = col;
      if (i + (unsigned long long)u * B < n)
        v[u] = ld_nc(reinterpret_cast<const V*>(s + (unsigned long long)row * t.src_pitch + (unsigned long long)col * W));
      col += dcol, row += drow;
      if (col >= vpr) col -= vpr, ++row;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + (unsigned long long)u * B < n)
        st_na(reinterpret_cast<V*>(d + (unsigned long long)rr[u] * t.dst_pitch + (unsigned long long)cc[u] * W), v[u]);
  }
}

__global__ void __launch_bounds__(512) copy_tiles_kernel(const DevTile* __restrict__ tiles, unsigned long long n) {
  for (unsigned long long k = blockIdx.x; k < n; k += gridDim.x) {
    const DevTile t = tiles[k];
    if (t.rows == 0 || t.row_bytes == 0) continue;
    const unsigned long long a = t.src | t.dst | t.row_bytes | (t.rows > 1 ? (t.src_pitch | t.dst_pitch) : 0ull);
    if ((a & 15) == 0) copy_tile<uint4, 4>(t);
    else if ((a & 7) == 0) copy_tile<uint2, 8>(t);
    else if ((a & 3) == 0) copy_tile<unsigned, 8>(t);
    else if ((a & 1) == 0) copy_tile<unsigned short, 8>(t);
    else copy_tile<unsigned char, 8>(t);
  }
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

template <bool kVerify>
__global__ void __launch_bounds__(256) payload_kernel(unsigned char* data, unsigned long long seed, CellGeom g,
                                                      unsigned long long* count) {
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

int payload_grid(const CellGeom& g) {
  unsigned long long chunks = (g.bytes + 15) / 16;
  unsigned long long blocks = (chunks + 255) / 256;
  return int(blocks < 148 * 16 ? (blocks ? blocks : 1) : 148 * 16);
}

}  // namespace

void launch_copy_tiles(const CopyTile* d_tiles, uint64_t n_tiles, int grid, int block, void* stream) {
  if (n_tiles == 0) return;
  copy_tiles_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const DevTile*>(d_tiles),
                                                                             n_tiles);
  check(cudaGetLastError(), "copy_tiles launch");
}

void launch_fill(void* dst, uint64_t seed, const CellGeom& g, void* stream) {
  if (g.bytes == 0) return;
  payload_kernel<false><<<payload_grid(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<unsigned char*>(dst), seed, g, nullptr);
  check(cudaGetLastError(), "fill launch");
}

void launch_verify(const void* data, uint64_t seed, const CellGeom& g, unsigned long long* d_count, void* stream) {
  if (g.bytes == 0) return;
  payload_kernel<true><<<payload_grid(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<unsigned char*>(const_cast<void*>(data)), seed, g, d_count);
  check(cudaGetLastError(), "verify launch");
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
