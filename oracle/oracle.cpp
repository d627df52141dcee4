// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// CPU restatement of the reference's reshard path:
//   * tensor-core  (slice / merge / SplitGrid / grid_refine / Range text) restated from
//     /root/reference/proj/src/tensor/{tensor,split_grid,range,dtype}.cpp and
//     proj/include/reshard/util/hash.hpp — or, when compiled with -DORACLE_REFERENCE_CORE,
//     routed to the reference's own compiled tensor-core (oracle/_ref/, see oracle/Makefile),
//     so that every byte of the CPU baseline moves through the reference's slice()/merge().
//   * the SPEC-only modules above it (no reference code exists for them):
//     parallel-config, planner / Algorithm 1 (SPEC.md:201-273,
//     PAPER.md:338-372), executor apply_plan / recover and the dataset
//     index shuffle / repartition / locate.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library.  The product (paper_2312_05181_b200/) never links it.
//
// C ABI: every entry point returns 0 on success or 1 + Errc (numbering of
// proj/include/reshard/error.hpp:8-48); orc_last_error() holds the message.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#ifdef ORACLE_REFERENCE_CORE
#include "reshard/error.hpp"
#include "reshard/tensor/split_grid.hpp"
#include "reshard/tensor/tensor.hpp"
#include "reshard/util/hash.hpp"
#endif

namespace orc {

// ---------------------------------------------------------------------------------------
// Errors — numeric codes follow enum class Errc, proj/include/reshard/error.hpp:8-48.
// ---------------------------------------------------------------------------------------
enum Code : int {
  RangeOutOfBounds = 0, RankMismatch, ShapeMismatch, TilingGap, TilingOverlap, DtypeMismatch,
  InvalidSplitPoint, InvalidTensor, IndivisibleLayerCount, IndivisibleSliceDim,
  DeviceCountMismatch, InvalidJobConfig, MalformedConfig, InconsistentBaseShape, CoverageGap,
  UnknownDevice, CatalogMismatch, UnsatisfiableFragment, NoSource, NotFound, IndivisibleBatch,
  StepBeyondEpoch, IndexOutOfRange, InvalidReplicaCount, MalformedFrame, UnknownVerb, BadRange,
  ConnectionFailed, CheckpointRequired, LayoutMismatch, IoError, ScriptError,
  Internal  // oracle-only (allocation failure etc.)
};

static const char* const kCodeNames[] = {
    "RangeOutOfBounds", "RankMismatch", "ShapeMismatch", "TilingGap", "TilingOverlap",
    "DtypeMismatch", "InvalidSplitPoint", "InvalidTensor", "IndivisibleLayerCount",
    "IndivisibleSliceDim", "DeviceCountMismatch", "InvalidJobConfig", "MalformedConfig",
    "InconsistentBaseShape", "CoverageGap", "UnknownDevice", "CatalogMismatch",
    "UnsatisfiableFragment", "NoSource", "NotFound", "IndivisibleBatch", "StepBeyondEpoch",
    "IndexOutOfRange", "InvalidReplicaCount", "MalformedFrame", "UnknownVerb", "BadRange",
    "ConnectionFailed", "CheckpointRequired", "LayoutMismatch", "IoError", "ScriptError",
    "Internal"};

struct Fault {
  int code;
  std::string msg;
};

[[noreturn]] static void fail(int code, const std::string& msg) {
  throw Fault{code, std::string(kCodeNames[code]) + ": " + msg};
}

using Shape = std::vector<uint64_t>;
struct Iv {
  uint64_t lo = 0, hi = 0;
  bool operator==(const Iv&) const = default;
  auto operator<=>(const Iv&) const = default;
};
using Box = std::vector<Iv>;  // restated reshard::Range (range.hpp:27-66)

static uint64_t count_of(const Shape& s) {
  uint64_t n = 1;
  for (auto e : s) n *= e;
  return n;
}
static Shape extents_of(const Box& b) {
  Shape s(b.size());
  for (size_t i = 0; i < b.size(); ++i) s[i] = b[i].hi - b[i].lo;
  return s;
}
static Box full_box(const Shape& s) {
  Box b(s.size());
  for (size_t i = 0; i < s.size(); ++i) b[i] = {0, s[i]};
  return b;
}
// Range::contains / overlaps (range.cpp:56-68)
static bool box_contains(const Box& outer, const Box& in) {
  if (in.size() != outer.size()) return false;
  for (size_t i = 0; i < in.size(); ++i)
    if (in[i].lo < outer[i].lo || in[i].hi > outer[i].hi) return false;
  return true;
}
[[maybe_unused]] static bool box_overlaps(const Box& a, const Box& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (b[i].hi <= a[i].lo || a[i].hi <= b[i].lo) return false;
  return true;
}
// Range::rebase_into (range.cpp:70-78): coordinates of `in` relative to `outer`.
static Box box_rebase(const Box& in, const Box& outer) {
  if (!box_contains(outer, in)) fail(RangeOutOfBounds, "cannot rebase box");
  Box r(in.size());
  for (size_t i = 0; i < in.size(); ++i) r[i] = {in[i].lo - outer[i].lo, in[i].hi - outer[i].lo};
  return r;
}
// Range::to_string (range.cpp:92-101)
static std::string box_text(const Box& b) {
  std::string s = "[";
  for (size_t i = 0; i < b.size(); ++i) {
    if (i) s += ',';
    s += std::to_string(b[i].lo) + ':' + std::to_string(b[i].hi);
  }
  return s + "]";
}

// dtype widths, dtype.hpp:19-27 ; codes > 3 rejected as in dtype_from_code (dtype.cpp:25-28)
static size_t width_of(int dtype) {
  switch (dtype) {
    case 0: return 4;
    case 1: return 2;
    case 2: return 8;
    case 3: return 1;
  }
  fail(InvalidTensor, "unknown dtype code " + std::to_string(dtype));
}

// ---------------------------------------------------------------------------------------
// Tensor core.  Restated (default) or the reference's compiled code (ORACLE_REFERENCE_CORE).
// ---------------------------------------------------------------------------------------
namespace core {

#ifndef ORACLE_REFERENCE_CORE
// Restatement of reshard::Tensor (tensor.hpp:16-38, tensor.cpp:9-17).
struct Tensor {
  int dtype = 0;
  Shape shape;
  std::vector<uint8_t> bytes;
};
static Tensor make(int dtype, Shape shape, std::vector<uint8_t> bytes) {
  for (auto e : shape)
    if (e == 0) fail(InvalidTensor, "zero extent");
  uint64_t want = count_of(shape) * width_of(dtype);
  if (bytes.size() != want)
    fail(InvalidTensor, "payload " + std::to_string(bytes.size()) + " bytes, expected " +
                            std::to_string(want));
  return Tensor{dtype, std::move(shape), std::move(bytes)};
}
[[maybe_unused]] static int dtype_of(const Tensor& t) { return t.dtype; }
[[maybe_unused]] static const Shape& shape_of(const Tensor& t) { return t.shape; }
static const std::vector<uint8_t>& bytes_of(const Tensor& t) { return t.bytes; }

// Range::check_against (range.cpp:36-47)
static void check_box(const Box& b, const Shape& s) {
  if (b.size() != s.size())
    fail(RankMismatch, "range rank " + std::to_string(b.size()) + " vs tensor rank " +
                           std::to_string(s.size()));
  for (size_t i = 0; i < b.size(); ++i)
    if (b[i].lo >= b[i].hi || b[i].hi > s[i]) fail(RangeOutOfBounds, "interval invalid in dim " + std::to_string(i));
}

// Row walker: the reference walks an odometer over all but the innermost dimension and
// copies one contiguous innermost run per step (tensor.cpp:35-57).  Restated as an explicit
// recursion over the leading dims; `visit(elem_offset_in_full)` per run, in row-major order.
template <class Visit>
static void walk_runs(const Box& at, const Shape& full, Visit&& visit) {
  const size_t r = full.size();
  if (r == 0) {
    visit(uint64_t{0});
    return;
  }
  std::vector<uint64_t> stride(r, 1);
  for (size_t d = r - 1; d > 0; --d) stride[d - 1] = stride[d] * full[d];
  std::vector<uint64_t> idx(r, 0);
  for (size_t d = 0; d < r; ++d) idx[d] = at[d].lo;
  while (true) {
    uint64_t off = 0;
    for (size_t d = 0; d < r; ++d) off += idx[d] * stride[d];
    visit(off);
    // advance leading dims (innermost is one whole run)
    size_t d = r - 1;
    for (;;) {
      if (d == 0) return;
      --d;
      if (++idx[d] < at[d].hi) break;
      idx[d] = at[d].lo;
      if (d == 0) return;
    }
  }
}

// slice (tensor.cpp:61-78)
static Tensor slice(const Tensor& t, const Box& b) {
  check_box(b, t.shape);
  const size_t w = width_of(t.dtype);
  Shape ext = extents_of(b);
  const uint64_t run = (ext.empty() ? 1 : ext.back()) * w;
  std::vector<uint8_t> out(count_of(ext) * w);
  uint64_t pos = 0;
  walk_runs(b, t.shape, [&](uint64_t elem) {
    std::memcpy(out.data() + pos, t.bytes.data() + elem * w, run);
    pos += run;
  });
  return make(t.dtype, std::move(ext), std::move(out));
}

// merge (tensor.cpp:80-114), with the same validation order.
static Tensor merge(std::vector<std::pair<Box, Tensor>>&& parts, const Shape& target) {
  if (parts.empty()) fail(TilingGap, "no parts");
  const int dt = parts.front().second.dtype;
  uint64_t covered = 0;
  for (const auto& [b, p] : parts) {
    check_box(b, target);
    if (p.dtype != dt) fail(DtypeMismatch, "parts disagree on dtype");
    if (p.shape != extents_of(b)) fail(ShapeMismatch, "part shape does not match its range " + box_text(b));
    covered += count_of(extents_of(b));
  }
  for (size_t i = 0; i < parts.size(); ++i)
    for (size_t j = i + 1; j < parts.size(); ++j)
      if (box_overlaps(parts[i].first, parts[j].first))
        fail(TilingOverlap, box_text(parts[i].first) + " overlaps " + box_text(parts[j].first));
  if (covered != count_of(target)) fail(TilingGap, "parts do not cover the target");
  const size_t w = width_of(dt);
  std::vector<uint8_t> out(count_of(target) * w);
  for (const auto& [b, p] : parts) {
    Shape ext = extents_of(b);
    const uint64_t run = (ext.empty() ? 1 : ext.back()) * w;
    uint64_t pos = 0;
    walk_runs(b, target, [&](uint64_t elem) {
      std::memcpy(out.data() + elem * w, p.bytes.data() + pos, run);
      pos += run;
    });
  }
  return make(dt, target, std::move(out));
}

// SplitGrid::check_against (split_grid.cpp:20-33)
static void grid_check(const std::vector<std::vector<uint64_t>>& g, const Shape& s) {
  if (g.size() != s.size())
    fail(RankMismatch, "grid rank " + std::to_string(g.size()) + " vs tensor rank " + std::to_string(s.size()));
  for (size_t d = 0; d < g.size(); ++d) {
    uint64_t prev = 0;
    for (auto p : g[d]) {
      if (p == 0 || p >= s[d] || p <= prev) fail(InvalidSplitPoint, "split point " + std::to_string(p) + " invalid");
      prev = p;
    }
  }
}
// SplitGrid::cells (split_grid.cpp:62-86): lexicographic, last dim fastest.
static std::vector<Box> grid_cells(const std::vector<std::vector<uint64_t>>& g, const Shape& s) {
  grid_check(g, s);
  std::vector<std::vector<Iv>> per(g.size());
  for (size_t d = 0; d < g.size(); ++d) {
    uint64_t lo = 0;
    for (auto p : g[d]) per[d].push_back({lo, p}), lo = p;
    per[d].push_back({lo, s[d]});
  }
  uint64_t n = 1;
  for (auto& v : per) n *= v.size();
  std::vector<Box> out;
  out.reserve(n);
  for (uint64_t k = 0; k < n; ++k) {
    Box b(g.size());
    uint64_t rest = k;
    for (size_t d = g.size(); d-- > 0;) {
      b[d] = per[d][rest % per[d].size()];
      rest /= per[d].size();
    }
    out.push_back(std::move(b));
  }
  return out;
}
// grid_refine (split_grid.cpp:119-130)
static std::vector<std::vector<uint64_t>> grid_refine(const std::vector<std::vector<uint64_t>>& a,
                                                      const std::vector<std::vector<uint64_t>>& b) {
  if (a.size() != b.size()) fail(ShapeMismatch, "grids of different rank");
  std::vector<std::vector<uint64_t>> r(a.size());
  for (size_t d = 0; d < a.size(); ++d) {
    std::set<uint64_t> u(a[d].begin(), a[d].end());
    u.insert(b[d].begin(), b[d].end());
    r[d].assign(u.begin(), u.end());
  }
  return r;
}
// SplitGrid::even_split (split_grid.cpp:9-18)
static std::vector<std::vector<uint64_t>> even_split(const Shape& s, size_t dim, uint64_t ways) {
  if (dim >= s.size()) fail(RankMismatch, "split dim out of rank");
  if (ways == 0 || s[dim] % ways != 0) fail(IndivisibleSliceDim, "extent not divisible");
  std::vector<std::vector<uint64_t>> g(s.size());
  for (uint64_t k = 1; k < ways; ++k) g[dim].push_back(k * (s[dim] / ways));
  return g;
}
static std::vector<Iv> intervals_of(const std::vector<uint64_t>& pts, uint64_t extent) {
  std::vector<Iv> v;
  uint64_t lo = 0;
  for (auto p : pts) v.push_back({lo, p}), lo = p;
  v.push_back({lo, extent});
  return v;
}
// SplitGrid::cell (split_grid.cpp:88-101)
static Box grid_cell(const std::vector<std::vector<uint64_t>>& g, const Shape& s, uint64_t index) {
  grid_check(g, s);
  Box b(g.size());
  uint64_t rest = index;
  for (size_t d = g.size(); d-- > 0;) {
    auto iv = intervals_of(g[d], s[d]);
    b[d] = iv[rest % iv.size()];
    rest /= iv.size();
  }
  if (rest != 0) fail(IndexOutOfRange, "cell index out of range");
  return b;
}
// SplitGrid::cell_index_of (split_grid.cpp:103-117)
static uint64_t grid_cell_index_of(const std::vector<std::vector<uint64_t>>& g, const Shape& s, const Box& r) {
  grid_check(g, s);
  check_box(r, s);
  uint64_t idx = 0;
  for (size_t d = 0; d < g.size(); ++d) {
    auto iv = intervals_of(g[d], s[d]);
    size_t i = 0;
    while (i < iv.size() && iv[i].hi <= r[d].lo) ++i;
    if (i == iv.size() || r[d].lo < iv[i].lo || r[d].hi > iv[i].hi) fail(InvalidSplitPoint, "range crosses a grid boundary");
    idx = idx * iv.size() + i;
  }
  return idx;
}
// Range::offset_by (range.cpp:80-90)
static Box offset_by(const Box& in, const Box& outer) {
  if (in.size() != outer.size()) fail(RankMismatch, "offset_by rank mismatch");
  Box r(in.size());
  for (size_t i = 0; i < in.size(); ++i) {
    if (in[i].hi + outer[i].lo > outer[i].hi) fail(RangeOutOfBounds, "range exceeds outer");
    r[i] = {in[i].lo + outer[i].lo, in[i].hi + outer[i].lo};
  }
  return r;
}
// RangeSpec::resolve (range.cpp:153-164); unconstrained dims are lo = hi = UINT64_MAX
static Box spec_resolve(const Box& spec, const Shape& s) {
  if (spec.size() != s.size()) fail(RankMismatch, "range spec rank mismatch");
  Box r(spec.size());
  for (size_t i = 0; i < spec.size(); ++i)
    r[i] = (spec[i].lo == UINT64_MAX && spec[i].hi == UINT64_MAX) ? Iv{0, s[i]} : spec[i];
  check_box(r, s);
  return r;
}

#else  // ---- reference tensor-core (compiled from /root/reference by oracle/Makefile) ----

using Tensor = reshard::Tensor;
template <class F>
static auto guarded(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const reshard::Error& e) {
    throw Fault{static_cast<int>(e.code()), e.what()};
  }
}
static reshard::Range to_ref(const Box& b) {
  std::vector<reshard::Interval> v;
  for (auto& i : b) v.push_back({i.lo, i.hi});
  return reshard::Range(std::move(v));
}
static Box from_ref(const reshard::Range& r) {
  Box b;
  for (auto& i : r.dims()) b.push_back({i.lo, i.hi});
  return b;
}
static Tensor make(int dtype, Shape shape, std::vector<uint8_t> bytes) {
  return guarded([&] {
    return reshard::Tensor(reshard::dtype_from_code(static_cast<uint8_t>(dtype)), std::move(shape), std::move(bytes));
  });
}
[[maybe_unused]] static int dtype_of(const Tensor& t) { return static_cast<int>(t.dtype()); }
[[maybe_unused]] static const Shape& shape_of(const Tensor& t) { return t.shape(); }
static const std::vector<uint8_t>& bytes_of(const Tensor& t) { return t.payload(); }
static Tensor slice(const Tensor& t, const Box& b) {
  return guarded([&] { return reshard::slice(t, to_ref(b)); });
}
static Tensor merge(std::vector<std::pair<Box, Tensor>>&& parts, const Shape& target) {
  return guarded([&] {
    std::vector<std::pair<reshard::Range, reshard::Tensor>> p;
    p.reserve(parts.size());
    for (auto& [b, t] : parts) p.emplace_back(to_ref(b), std::move(t));
    return reshard::merge(p, target);
  });
}
static std::vector<Box> grid_cells(const std::vector<std::vector<uint64_t>>& g, const Shape& s) {
  return guarded([&] {
    std::vector<Box> out;
    for (auto& r : reshard::SplitGrid(g).cells(s)) out.push_back(from_ref(r));
    return out;
  });
}
static std::vector<std::vector<uint64_t>> grid_refine(const std::vector<std::vector<uint64_t>>& a,
                                                      const std::vector<std::vector<uint64_t>>& b) {
  return guarded([&] { return reshard::grid_refine(reshard::SplitGrid(a), reshard::SplitGrid(b)).points(); });
}
static std::vector<std::vector<uint64_t>> even_split(const Shape& s, size_t dim, uint64_t ways) {
  return guarded([&] { return reshard::SplitGrid::even_split(s, dim, ways).points(); });
}
static Box grid_cell(const std::vector<std::vector<uint64_t>>& g, const Shape& s, uint64_t index) {
  return guarded([&] { return from_ref(reshard::SplitGrid(g).cell(s, index)); });
}
static uint64_t grid_cell_index_of(const std::vector<std::vector<uint64_t>>& g, const Shape& s, const Box& r) {
  return guarded([&] { return reshard::SplitGrid(g).cell_index_of(s, to_ref(r)); });
}
static Box offset_by(const Box& in, const Box& outer) {
  return guarded([&] { return from_ref(to_ref(in).offset_by(to_ref(outer))); });
}
static Box spec_resolve(const Box& spec, const Shape& s) {
  return guarded([&] {
    std::vector<std::optional<reshard::Interval>> v;
    for (auto& i : spec)
      v.push_back(i.lo == UINT64_MAX && i.hi == UINT64_MAX ? std::optional<reshard::Interval>{}
                                                           : std::optional<reshard::Interval>{reshard::Interval{i.lo, i.hi}});
    return from_ref(reshard::RangeSpec(v).resolve(s));
  });
}
static void grid_check(const std::vector<std::vector<uint64_t>>& g, const Shape& s) {
  guarded([&] {
    reshard::SplitGrid(g).check_against(s);
    return 0;
  });
}
#endif
}  // namespace core

// ---------------------------------------------------------------------------------------
// Range text parsing: restated Range::parse / RangeSpec::parse (range.cpp:103-193).
// ---------------------------------------------------------------------------------------
static uint64_t parse_num(const std::string& s) {
  if (s.empty()) fail(MalformedFrame, "bad integer ''");
  uint64_t v = 0;
  for (char c : s) {
    if (c < '0' || c > '9') fail(MalformedFrame, "bad integer '" + s + "'");
    uint64_t nv = v * 10 + uint64_t(c - '0');
    if (nv / 10 != v) fail(MalformedFrame, "bad integer '" + s + "'");  // overflow (from_chars errc)
    v = nv;
  }
  return v;
}
static std::vector<std::string> bracket_items(const std::string& t) {
  if (t.size() < 2 || t.front() != '[' || t.back() != ']') fail(MalformedFrame, "range must be bracketed");
  std::string in = t.substr(1, t.size() - 2);
  std::vector<std::string> items;
  if (in.empty()) return items;
  size_t start = 0;
  for (;;) {
    size_t c = in.find(',', start);
    if (c == std::string::npos) {
      items.push_back(in.substr(start));
      break;
    }
    items.push_back(in.substr(start, c - start));
    start = c + 1;
  }
  return items;
}
// spec=true: RangeSpec::parse (":" leaves a dim unconstrained, reported as lo=hi=UINT64_MAX)
[[maybe_unused]] static Box parse_box(const std::string& t, bool spec) {
  Box b;
  for (auto& item : bracket_items(t)) {
    if (spec && item == ":") {
      b.push_back({UINT64_MAX, UINT64_MAX});
      continue;
    }
    size_t c = item.find(':');
    if (c == std::string::npos) fail(MalformedFrame, "interval needs ':'");
    b.push_back({parse_num(item.substr(0, c)), parse_num(item.substr(c + 1))});
  }
  return b;
}

// ---------------------------------------------------------------------------------------
// Hashing / RNG: restated hash.hpp:13-63.
// ---------------------------------------------------------------------------------------
static constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
struct Rng {  // SplitMix64 (hash.hpp:53-63)
  uint64_t s;
  uint64_t next() { return mix64(s += kGolden); }
  uint64_t below(uint64_t n) { return n == 0 ? 0 : next() % n; }
};
// Synthetic payload: byte b of a base tensor is byte (b % 8) of draw b/8 of the
// splitmix64 stream seeded `seed`; draw k = mix64(seed + (k+1)*golden).  Counter-based, so
// any byte range can be produced independently.
static void stream_bytes(uint64_t seed, uint64_t off, uint64_t n, uint8_t* out) {
  uint64_t k = off / 8;
  size_t sh = off % 8;
  uint64_t i = 0;
  while (i < n) {
    uint64_t w = mix64(seed + (k + 1) * kGolden);
    for (size_t b = sh; b < 8 && i < n; ++b) out[i++] = uint8_t(w >> (8 * b));
    sh = 0;
    ++k;
  }
}
static uint64_t path_seed(const std::string& path) {
  return fnv1a(reinterpret_cast<const uint8_t*>(path.data()), path.size()) ^ 0x7E9B1E0Cull;
}

// ---------------------------------------------------------------------------------------
// parallel-config: catalog, PTC (T, sigma, phi, alpha), builders.
// ---------------------------------------------------------------------------------------
static constexpr int kLayerPre = -1;   // embeddings: first stage
static constexpr int kLayerPost = -2;  // final layernorm: last stage

struct Entry {
  std::string path;
  int dtype;
  Shape shape;
  int tp_dim;  // -1: replicated under TP (sigma = identity)
  int layer;
};
struct Catalog {
  std::vector<Entry> e;
};

struct Dev {
  uint32_t w = 0, l = 0;  // (worker, local index)
  auto operator<=>(const Dev&) const = default;
  std::string text() const { return std::to_string(w) + ":" + std::to_string(l); }
};

struct Ptc {
  Catalog cat;
  std::vector<Dev> devices;  // enumeration order (worker-major, local index)
  int T = 1, P = 1, D = 1;
  std::vector<std::vector<std::vector<uint64_t>>> sigma;  // per tensor: split points per dim
  std::vector<std::vector<Box>> cells;                    // sigma cells (cached)
  std::vector<std::vector<int>> phi;                      // phi[t][cell] -> partition
  std::vector<std::vector<Dev>> alpha;                    // alpha[partition] -> devices
  std::vector<int> stage;                                 // stage per tensor
};

// GPT catalog in Megatron naming.  kind 0: fp32 param+Adam (12 B/param);
// kind 1: 2-byte param + fp32 master + Adam (14 B/param; bf16 carried as F16);
// kind 2: fp32 params only.
static Catalog gpt_catalog(uint64_t h, uint64_t L, uint64_t S, uint64_t V, int kind) {
  struct P {
    std::string name;
    Shape shape;
    int tp;
    int layer;
  };
  std::vector<P> ps;
  ps.push_back({"embedding.word_embeddings.weight", {V, h}, 0, kLayerPre});
  ps.push_back({"embedding.position_embeddings.weight", {S, h}, -1, kLayerPre});
  for (uint64_t i = 0; i < L; ++i) {
    std::string p = "layers." + std::to_string(i) + ".";
    int l = int(i);
    ps.push_back({p + "input_layernorm.weight", {h}, -1, l});
    ps.push_back({p + "input_layernorm.bias", {h}, -1, l});
    ps.push_back({p + "self_attention.query_key_value.weight", {3 * h, h}, 0, l});
    ps.push_back({p + "self_attention.query_key_value.bias", {3 * h}, 0, l});
    ps.push_back({p + "self_attention.dense.weight", {h, h}, 1, l});
    ps.push_back({p + "self_attention.dense.bias", {h}, -1, l});
    ps.push_back({p + "post_attention_layernorm.weight", {h}, -1, l});
    ps.push_back({p + "post_attention_layernorm.bias", {h}, -1, l});
    ps.push_back({p + "mlp.dense_h_to_4h.weight", {4 * h, h}, 0, l});
    ps.push_back({p + "mlp.dense_h_to_4h.bias", {4 * h}, 0, l});
    ps.push_back({p + "mlp.dense_4h_to_h.weight", {h, 4 * h}, 1, l});
    ps.push_back({p + "mlp.dense_4h_to_h.bias", {h}, -1, l});
  }
  ps.push_back({"final_layernorm.weight", {h}, -1, kLayerPost});
  ps.push_back({"final_layernorm.bias", {h}, -1, kLayerPost});
  std::vector<std::pair<std::string, int>> states;
  if (kind == 0) states = {{"param", 0}, {"exp_avg", 0}, {"exp_avg_sq", 0}};
  else if (kind == 1) states = {{"param", 1}, {"master", 0}, {"exp_avg", 0}, {"exp_avg_sq", 0}};
  else states = {{"param", 0}};
  Catalog c;
  for (auto& p : ps)
    for (auto& [sn, dt] : states) c.e.push_back({sn + "/" + p.name, dt, p.shape, p.tp, p.layer});
  return c;
}

// Stage of each tensor: layers 0..L-1 in P contiguous groups balanced within one layer,
// remainder to the earliest stages; embeddings first, final LN last.
static std::vector<int> stages_of(const Catalog& c, int P) {
  int L = 0;
  for (auto& e : c.e) L = std::max(L, e.layer + 1);
  if (P > 1 && L < P) fail(IndivisibleLayerCount, std::to_string(L) + " layers into " + std::to_string(P) + " stages");
  std::vector<int> layer_stage(std::max(L, 0));
  int base = L / P, rem = L % P, l = 0;
  for (int s = 0; s < P; ++s)
    for (int k = 0; k < base + (s < rem ? 1 : 0); ++k) layer_stage[l++] = s;
  std::vector<int> st;
  for (auto& e : c.e) st.push_back(e.layer == kLayerPre ? 0 : e.layer == kLayerPost ? P - 1 : layer_stage[e.layer]);
  return st;
}

// build_strategy: device (dp, pp, tp) = devices[dp*P*T + pp*T + tp].
static Ptc build_strategy(const Catalog& c, const std::vector<Dev>& devs, int T, int P, int D) {
  if (T < 1 || P < 1 || D < 1) fail(InvalidJobConfig, "degrees must be positive");
  if (devs.size() != size_t(T) * P * D) fail(DeviceCountMismatch, "T*P*D != device count");
  Ptc p;
  p.cat = c;
  p.devices = devs;
  p.T = T, p.P = P, p.D = D;
  p.stage = stages_of(c, P);
  // partitions: (stage s, tp j) -> s*T+j ; replicated-under-TP tensors of stage s -> P*T+s
  p.alpha.assign(size_t(P) * T + P, {});
  for (int s = 0; s < P; ++s)
    for (int j = 0; j < T; ++j)
      for (int d = 0; d < D; ++d) {
        Dev dv = devs[size_t(d) * P * T + size_t(s) * T + j];
        p.alpha[size_t(s) * T + j].push_back(dv);
      }
  for (int s = 0; s < P; ++s)
    for (int d = 0; d < D; ++d)
      for (int j = 0; j < T; ++j) p.alpha[size_t(P) * T + s].push_back(devs[size_t(d) * P * T + size_t(s) * T + j]);
  for (size_t t = 0; t < c.e.size(); ++t) {
    const Entry& e = c.e[t];
    std::vector<std::vector<uint64_t>> g(e.shape.size());
    if (e.tp_dim >= 0) g = core::even_split(e.shape, size_t(e.tp_dim), uint64_t(T));
    p.sigma.push_back(g);
    p.cells.push_back(core::grid_cells(g, e.shape));
    std::vector<int> ph;
    for (size_t i = 0; i < p.cells.back().size(); ++i)
      ph.push_back(e.tp_dim >= 0 ? p.stage[t] * T + int(i) : P * T + p.stage[t]);
    p.phi.push_back(ph);
  }
  return p;
}

static bool hosts(const Ptc& p, size_t t, size_t cell, const Dev& d) {
  for (auto& x : p.alpha[p.phi[t][cell]])
    if (x == d) return true;
  return false;
}

// hosted_subtensors
static std::vector<std::pair<size_t, size_t>> hosted(const Ptc& p, const Dev& d) {
  if (std::find(p.devices.begin(), p.devices.end(), d) == p.devices.end()) fail(UnknownDevice, d.text());
  std::vector<std::pair<size_t, size_t>> out;
  for (size_t t = 0; t < p.cat.e.size(); ++t)
    for (size_t i = 0; i < p.cells[t].size(); ++i)
      if (hosts(p, t, i, d)) out.push_back({t, i});
  return out;
}

// validate: violations are data.
static std::vector<std::string> validate(const Ptc& p) {
  std::vector<std::string> v;
  for (size_t t = 0; t < p.cat.e.size(); ++t) {
    if (t >= p.sigma.size()) {
      v.push_back("MissingSigma: " + p.cat.e[t].path);
      continue;
    }
    try {
      core::grid_check(p.sigma[t], p.cat.e[t].shape);
    } catch (const Fault&) {
      v.push_back("InvalidSplitPoint: " + p.cat.e[t].path);
      continue;
    }
    for (size_t i = 0; i < p.phi[t].size(); ++i) {
      int part = p.phi[t][i];
      if (part < 0 || size_t(part) >= p.alpha.size()) v.push_back("UnmappedSubtensor: " + p.cat.e[t].path);
    }
  }
  std::set<int> used;
  for (auto& ph : p.phi) used.insert(ph.begin(), ph.end());
  for (int part : used) {
    if (part < 0 || size_t(part) >= p.alpha.size()) continue;
    if (p.alpha[part].empty()) v.push_back("UnhostedPartition: " + std::to_string(part));
    for (auto& d : p.alpha[part])
      if (std::find(p.devices.begin(), p.devices.end(), d) == p.devices.end())
        v.push_back("UnknownDevice: " + d.text());
  }
  return v;
}

// ---------------------------------------------------------------------------------------
// planner (Algorithm 1)
// ---------------------------------------------------------------------------------------
struct Op {
  enum Kind { Split, Move, Merge } kind;
  size_t t;
  Dev dev;            // Split / Merge actor ; Move: src
  Dev dst;            // Move only
  Box box;            // Split: source cell ; Move: fragment ; Merge: merged cell
  std::vector<Box> parts;  // Split targets / Merge parts
  uint64_t bytes = 0;
};
struct Plan {
  std::shared_ptr<const Ptc> a, b;
  std::vector<std::vector<std::vector<uint64_t>>> refine;  // per tensor
  std::vector<Op> ops;                                     // splits, then moves, then merges
  size_t n_split = 0, n_move = 0, n_merge = 0;
  std::set<Dev> failed;
};

static size_t cell_containing(const std::vector<Box>& cells, const Box& w) {
  for (size_t i = 0; i < cells.size(); ++i)
    if (box_contains(cells[i], w)) return i;
  return SIZE_MAX;
}

// choose_source: resident -> dst; else same-worker candidates if any;
// least accumulated egress; ties by smallest device id.
static Dev choose_source(const std::vector<Dev>& cand, const Dev& dst, const std::map<Dev, uint64_t>& egress) {
  if (cand.empty()) fail(NoSource, "no candidate for " + dst.text());
  for (auto& c : cand)
    if (c == dst) return dst;
  std::vector<Dev> pool;
  for (auto& c : cand)
    if (c.w == dst.w) pool.push_back(c);
  if (pool.empty()) pool = cand;
  Dev best = pool.front();
  uint64_t be = UINT64_MAX;
  for (auto& c : pool) {
    auto it = egress.find(c);
    uint64_t e = it == egress.end() ? 0 : it->second;
    if (e < be || (e == be && c < best)) best = c, be = e;
  }
  return best;
}

static Plan generate_plan(std::shared_ptr<const Ptc> a, std::shared_ptr<const Ptc> b, const std::set<Dev>& failed) {
  if (a->cat.e.size() != b->cat.e.size()) fail(CatalogMismatch, "catalog sizes differ");
  for (size_t t = 0; t < a->cat.e.size(); ++t) {
    auto &x = a->cat.e[t], &y = b->cat.e[t];
    if (x.path != y.path || x.dtype != y.dtype || x.shape != y.shape) fail(CatalogMismatch, x.path);
  }
  Plan plan;
  plan.a = a, plan.b = b, plan.failed = failed;
  std::vector<std::vector<Box>> gcells;
  for (size_t t = 0; t < a->cat.e.size(); ++t) {
    plan.refine.push_back(core::grid_refine(a->sigma[t], b->sigma[t]));
    gcells.push_back(core::grid_cells(plan.refine.back(), a->cat.e[t].shape));
  }
  auto frags_in = [&](size_t t, const Box& cell) {
    std::vector<Box> f;
    for (auto& g : gcells[t])
      if (box_contains(cell, g)) f.push_back(g);
    return f;
  };
  // SPLIT phase: per source device, per hosted cell (Alg. 1 lines 2-5)
  std::vector<Op> splits, moves, merges;
  for (auto& r : a->devices) {
    if (failed.count(r)) continue;
    for (auto [t, i] : hosted(*a, r)) {
      auto f = frags_in(t, a->cells[t][i]);
      if (f.size() > 1) splits.push_back(Op{Op::Split, t, r, r, a->cells[t][i], f, 0});
    }
  }
  // RE-PARTITION + MERGE: per destination device, per hosted cell (Alg. 1 lines 6-14)
  std::map<Dev, uint64_t> egress;
  for (auto& r2 : b->devices) {
    for (auto [t, i] : hosted(*b, r2)) {
      const Box& c = b->cells[t][i];
      auto W = frags_in(t, c);
      const uint64_t w8 = width_of(a->cat.e[t].dtype);
      for (auto& w : W) {
        size_t v = cell_containing(a->cells[t], w);
        std::vector<Dev> cand;
        for (auto& d : a->alpha[a->phi[t][v]])
          if (!failed.count(d)) cand.push_back(d);
        if (std::find(cand.begin(), cand.end(), r2) != cand.end()) continue;  // resident: no Move
        if (cand.empty())
          fail(failed.empty() ? UnsatisfiableFragment : CheckpointRequired,
               a->cat.e[t].path + " " + box_text(w) + " has no surviving holder");
        Dev src = choose_source(cand, r2, egress);
        uint64_t bytes = count_of(extents_of(w)) * w8;
        egress[src] += bytes;
        moves.push_back(Op{Op::Move, t, src, r2, w, {}, bytes});
      }
      if (W.size() > 1) merges.push_back(Op{Op::Merge, t, r2, r2, c, W, 0});  // single full-cell merge elided
    }
  }
  plan.n_split = splits.size(), plan.n_move = moves.size(), plan.n_merge = merges.size();
  for (auto* v : {&splits, &moves, &merges})
    for (auto& o : *v) plan.ops.push_back(std::move(o));
  return plan;
}

// Plan serialization.
static std::string plan_text(const Plan& p) {
  std::ostringstream o;
  auto join = [](const std::vector<Box>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? ";" : "") + box_text(v[i]);
    return s;
  };
  for (auto& op : p.ops) {
    const std::string& path = p.a->cat.e[op.t].path;
    if (op.kind == Op::Split)
      o << "SPLIT dev=" << op.dev.text() << " t=" << path << " r=" << box_text(op.box) << " -> " << join(op.parts) << "\n";
    else if (op.kind == Op::Move)
      o << "MOVE t=" << path << " r=" << box_text(op.box) << " " << op.dev.text() << " -> " << op.dst.text()
        << " bytes=" << op.bytes << "\n";
    else
      o << "MERGE dev=" << op.dev.text() << " t=" << path << " " << join(op.parts) << " -> " << box_text(op.box) << "\n";
  }
  return o.str();
}

// ---------------------------------------------------------------------------------------
// executor: per-device stores, pull-based apply with one task per
// destination; every byte moves through core::slice / core::merge.
// ---------------------------------------------------------------------------------------
using TensorP = std::shared_ptr<const core::Tensor>;
struct CellKey {
  size_t t;
  Box box;
  auto operator<=>(const CellKey&) const = default;
};
struct State {
  std::map<Dev, std::map<CellKey, TensorP>> store;
};

// Bytes of box `b` of base tensor t (row-major), generated from the counter stream.
static std::vector<uint8_t> gen_box(const Entry& e, const Box& b) {
  const size_t w = width_of(e.dtype);
  const uint64_t seed = path_seed(e.path);
  Shape ext = extents_of(b);
  const uint64_t run = (ext.empty() ? 1 : ext.back()) * w;
  std::vector<uint8_t> out(count_of(ext) * w);
  uint64_t pos = 0;
  std::vector<uint64_t> stride(e.shape.size(), 1);
  for (size_t d = e.shape.size(); d-- > 1;) stride[d - 1] = stride[d] * e.shape[d];
  std::vector<uint64_t> idx(b.size());
  for (size_t d = 0; d < b.size(); ++d) idx[d] = b[d].lo;
  if (b.empty()) {
    stream_bytes(seed, 0, w, out.data());
    return out;
  }
  for (;;) {
    uint64_t off = 0;
    for (size_t d = 0; d < b.size(); ++d) off += idx[d] * stride[d];
    stream_bytes(seed, off * w, run, out.data() + pos);
    pos += run;
    size_t d = b.size() - 1;
    for (;;) {
      if (d == 0) return out;
      --d;
      if (++idx[d] < b[d].hi) break;
      idx[d] = b[d].lo;
      if (d == 0) return out;
    }
  }
}

static bool in_range(size_t t, size_t t0, size_t t1) { return t >= t0 && t < t1; }

// One thread per device (input generation is not timed).  Devices in `skip` (the failed
// devices of a recovery) hold nothing: their stores stay empty.
static State fill_state(const Ptc& p, size_t t0, size_t t1, const std::set<Dev>& skip = {}) {
  State s;
  for (auto& d : p.devices) s.store[d];
  std::vector<std::thread> th;
  std::vector<Fault> errs(p.devices.size(), Fault{-1, ""});
  for (size_t k = 0; k < p.devices.size(); ++k)
    th.emplace_back([&, k] {
      try {
        const Dev& d = p.devices[k];
        auto& st = s.store.at(d);
        if (skip.count(d)) return;
        for (auto [t, i] : hosted(p, d)) {
          if (!in_range(t, t0, t1)) continue;
          const Entry& e = p.cat.e[t];
          st[CellKey{t, p.cells[t][i]}] =
              std::make_shared<const core::Tensor>(core::make(e.dtype, extents_of(p.cells[t][i]), gen_box(e, p.cells[t][i])));
        }
      } catch (const Fault& f) {
        errs[k] = f;
      }
    });
  for (auto& x : th) x.join();
  for (auto& f : errs)
    if (f.code >= 0) throw f;
  return s;
}

struct ApplyReport {
  double seconds = 0;
  uint64_t moved = 0, local = 0;
};

// apply_plan, distributed mode.
// per_device: SPEC.md:504 literally — one task per destination device, i.e. thread k runs the
// cells of destination devices k, k + nt, ... in order (nt = min(n_threads, devices)); else any
// thread takes the next (destination, tensor, cell) from a shared queue.
static State apply_plan(const Plan& plan, const State& src, size_t t0, size_t t1, int n_threads, ApplyReport* rep,
                        bool per_device = false) {
  const Ptc& a = *plan.a;
  const Ptc& b = *plan.b;
  // (dst, tensor, fragment) -> source, from the plan's Moves
  std::map<std::tuple<Dev, size_t, Box>, Dev> move_src;
  for (auto& op : plan.ops)
    if (op.kind == Op::Move) move_src[{op.dst, op.t, op.box}] = op.dev;
  std::vector<std::vector<Box>> gcells;
  for (size_t t = 0; t < a.cat.e.size(); ++t) gcells.push_back(core::grid_cells(plan.refine[t], a.cat.e[t].shape));

  State out;
  for (auto& d : b.devices) out.store[d];  // one store per destination
  // SPEC.md:504 runs one transformer task per destination device; the cells of one
  // destination are independent, so the work list is (destination, tensor, cell) and any
  // number of host threads drain it (the CPU arm uses every core it has).
  struct Task {
    const Dev* dst;
    size_t t, i, dev;
  };
  std::vector<Task> tasks;
  for (size_t k = 0; k < b.devices.size(); ++k)
    for (auto [t, i] : hosted(b, b.devices[k]))
      if (in_range(t, t0, t1)) tasks.push_back({&b.devices[k], t, i, k});
  const int nt = std::max(1, std::min<int>(n_threads, int(per_device ? b.devices.size() : tasks.size())));
  std::map<Dev, std::mutex> store_mu;
  for (auto& d : b.devices) store_mu[d];
  std::atomic<size_t> next{0};
  std::atomic<uint64_t> moved{0}, local{0};
  std::vector<Fault> errs;
  std::mutex em;
  // barrier 1: every source store is complete before any fetch.
  auto t_start = std::chrono::steady_clock::now();
  auto worker = [&](int me) {
    try {
      for (size_t pos = 0;;) {
        size_t k;
        if (per_device) {  // this thread's devices, in task order
          while (pos < tasks.size() && int(tasks[pos].dev % size_t(nt)) != me) ++pos;
          k = pos++;
        } else {
          k = next.fetch_add(1);
        }
        if (k >= tasks.size()) return;
        const Dev& r2 = *tasks[k].dst;
        const size_t t = tasks[k].t, i = tasks[k].i;
        const Box& c = b.cells[t][i];
        std::vector<std::pair<Box, core::Tensor>> parts;
        TensorP whole, made;
        for (auto& w : gcells[t]) {
          if (!box_contains(c, w)) continue;
          size_t v = cell_containing(a.cells[t], w);
          const Box& vb = a.cells[t][v];
          Dev holder;
          bool resident = hosts(a, t, v, r2) && !plan.failed.count(r2);
          if (resident) holder = r2;
          else holder = move_src.at({r2, t, w});
          const TensorP& stored = src.store.at(holder).at(CellKey{t, vb});
          if (resident && w == vb && w == c) {  // cell kept as is, no byte moves
            whole = stored;
            continue;
          }
          // fetch(peer, path, range) == query == slice of the stored cell
          core::Tensor frag = core::slice(*stored, box_rebase(w, vb));
          (resident ? local : moved) += core::bytes_of(frag).size();
          parts.emplace_back(box_rebase(w, c), std::move(frag));
        }
        if (whole) {
          made = whole;
        } else if (parts.size() == 1 && parts[0].first == full_box(extents_of(c))) {
          made = std::make_shared<const core::Tensor>(std::move(parts[0].second));  // merge elided
        } else {
          made = std::make_shared<const core::Tensor>(core::merge(std::move(parts), extents_of(c)));
        }
        std::lock_guard<std::mutex> g(store_mu.at(r2));
        out.store.at(r2)[CellKey{t, c}] = std::move(made);
      }
    } catch (const Fault& f) {
      std::lock_guard<std::mutex> g(em);
      errs.push_back(f);
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < nt; ++i) pool.emplace_back(worker, i);
  for (auto& th : pool) th.join();  // barrier 2: all fetches and merges done
  auto t_end = std::chrono::steady_clock::now();
  if (!errs.empty()) throw errs.front();
  if (rep) {
    rep->seconds = std::chrono::duration<double>(t_end - t_start).count();
    rep->moved = moved, rep->local = local;
  }
  return out;
}

// End-to-end preservation digest: reassemble base tensor t from one replica
// of each sigma cell held in `s`, FNV-1a-64 of the bytes.
static uint64_t state_digest(const Ptc& p, const State& s, size_t t) {
  std::vector<std::pair<Box, core::Tensor>> parts;
  for (size_t i = 0; i < p.cells[t].size(); ++i) {
    bool found = false;
    for (auto& d : p.alpha[p.phi[t][i]]) {
      auto it = s.store.find(d);
      if (it == s.store.end()) continue;
      auto jt = it->second.find(CellKey{t, p.cells[t][i]});
      if (jt == it->second.end()) continue;
      parts.emplace_back(p.cells[t][i], *jt->second);
      found = true;
      break;
    }
    if (!found) fail(NotFound, "cell of " + p.cat.e[t].path + " held nowhere");
  }
  core::Tensor full = core::merge(std::move(parts), p.cat.e[t].shape);
  auto& by = core::bytes_of(full);
  return fnv1a(by.data(), by.size());
}

// ---------------------------------------------------------------------------------------
// dataset index
// ---------------------------------------------------------------------------------------
// shuffle_epoch: Fisher-Yates (descending i, j = next_below(i+1)) on splitmix64 seeded
// (seed XOR epoch).  The loop direction is a builder choice (parity unpinned).
static void shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm) {
  for (uint64_t i = 0; i < n; ++i) perm[i] = i;
  Rng r{seed ^ epoch};
  for (uint64_t i = n; i-- > 1;) {
    uint64_t j = r.below(i + 1);
    std::swap(perm[i], perm[j]);
  }
}

// repartition: batches >= at_step; rank d owns [i*B + d*B/D', i*B + (d+1)*B/D') of each
// batch i, clipped at N for a trailing partial batch.
static void repart_check(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp) {
  if (B == 0 || dp == 0) fail(InvalidJobConfig, "B and new_dp must be positive");
  if (B % dp) fail(IndivisibleBatch, "B not divisible by new_dp");
  uint64_t nb = (n + B - 1) / B;
  if (at_step > nb) fail(StepBeyondEpoch, "at_step beyond the epoch");
}
static uint64_t repart_count(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t d) {
  uint64_t b = B / dp, nb = (n + B - 1) / B, c = 0;
  for (uint64_t i = at_step; i < nb; ++i) {
    uint64_t lo = i * B + d * b, hi = std::min(lo + b, n);
    if (hi > lo) c += hi - lo;
  }
  return c;
}

struct Sample {
  uint64_t file, off, len;
};

}  // namespace orc

// =======================================================================================
// C ABI
// =======================================================================================
using namespace orc;

static thread_local std::string g_err;

template <class F>
static int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Fault& e) {
    g_err = e.msg;
    return 1 + e.code;
  } catch (const std::exception& e) {
    g_err = std::string("Internal: ") + e.what();
    return 1 + Internal;
  }
}

static constexpr int kMaxRank = 8;
static Box box_from(int rank, const uint64_t* lo, const uint64_t* hi) {
  Box b(rank);
  for (int i = 0; i < rank; ++i) b[i] = {lo[i], hi[i]};
  return b;
}
static Shape shape_from(int rank, const uint64_t* s) { return Shape(s, s + rank); }
static std::vector<std::vector<uint64_t>> grid_from(int rank, const int* npts, const uint64_t* pts) {
  std::vector<std::vector<uint64_t>> g(rank);
  size_t k = 0;
  for (int d = 0; d < rank; ++d)
    for (int i = 0; i < npts[d]; ++i) g[d].push_back(pts[k++]);
  return g;
}

struct OrcPlan {
  Plan p;
};

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_errc_name(int c) { return (c >= 0 && c <= Internal) ? kCodeNames[c] : "UnknownError"; }
int orc_uses_reference_core(void) {
#ifdef ORACLE_REFERENCE_CORE
  return 1;
#else
  return 0;
#endif
}

// ---- tensor core -----------------------------------------------------------------------
int orc_slice(int dtype, int rank, const uint64_t* shape, const uint8_t* payload, int rrank, const uint64_t* lo,
              const uint64_t* hi, uint8_t* out) {
  return guard([&] {
    Shape s = shape_from(rank, shape);
    uint64_t n = count_of(s) * width_of(dtype);
    core::Tensor t = core::make(dtype, s, std::vector<uint8_t>(payload, payload + n));
    core::Tensor r = core::slice(t, box_from(rrank, lo, hi));
    std::memcpy(out, core::bytes_of(r).data(), core::bytes_of(r).size());
  });
}

// parts i: dtype[i], rank[i], shapes[i*8..], payload[i], range rank rr[i], lo/hi[i*8..]
int orc_merge(int n, const int* dtypes, const int* ranks, const uint64_t* shapes, const uint8_t* const* payloads,
              const int* rranks, const uint64_t* los, const uint64_t* his, int trank, const uint64_t* tshape,
              uint8_t* out) {
  return guard([&] {
    std::vector<std::pair<Box, core::Tensor>> parts;
    for (int i = 0; i < n; ++i) {
      Shape s = shape_from(ranks[i], shapes + size_t(i) * kMaxRank);
      uint64_t nb = count_of(s) * width_of(dtypes[i]);
      parts.emplace_back(box_from(rranks[i], los + size_t(i) * kMaxRank, his + size_t(i) * kMaxRank),
                         core::make(dtypes[i], s, std::vector<uint8_t>(payloads[i], payloads[i] + nb)));
    }
    core::Tensor r = core::merge(std::move(parts), shape_from(trank, tshape));
    std::memcpy(out, core::bytes_of(r).data(), core::bytes_of(r).size());
  });
}

int orc_grid_cells(int rank, const uint64_t* shape, const int* npts, const uint64_t* pts, int cap, uint64_t* lo_out,
                   uint64_t* hi_out, int* n_out) {
  return guard([&] {
    auto cells = core::grid_cells(grid_from(rank, npts, pts), shape_from(rank, shape));
    *n_out = int(cells.size());
    for (int i = 0; i < int(cells.size()) && i < cap; ++i)
      for (int d = 0; d < rank; ++d) lo_out[size_t(i) * kMaxRank + d] = cells[i][d].lo, hi_out[size_t(i) * kMaxRank + d] = cells[i][d].hi;
  });
}

int orc_grid_refine(int rank_a, const int* na, const uint64_t* pa, int rank_b, const int* nb, const uint64_t* pb,
                    int* n_out, uint64_t* pts_out) {
  return guard([&] {
    auto g = core::grid_refine(grid_from(rank_a, na, pa), grid_from(rank_b, nb, pb));
    size_t k = 0;
    for (size_t d = 0; d < g.size(); ++d) {
      n_out[d] = int(g[d].size());
      for (auto p : g[d]) pts_out[k++] = p;
    }
  });
}

int orc_grid_cell(int rank, const uint64_t* shape, const int* npts, const uint64_t* pts, uint64_t index, uint64_t* lo,
                  uint64_t* hi) {
  return guard([&] {
    Box b = core::grid_cell(grid_from(rank, npts, pts), shape_from(rank, shape), index);
    for (size_t d = 0; d < b.size(); ++d) lo[d] = b[d].lo, hi[d] = b[d].hi;
  });
}
int orc_grid_cell_index_of(int rank, const uint64_t* shape, const int* npts, const uint64_t* pts, int rrank,
                           const uint64_t* lo, const uint64_t* hi, uint64_t* index) {
  return guard([&] {
    *index = core::grid_cell_index_of(grid_from(rank, npts, pts), shape_from(rank, shape), box_from(rrank, lo, hi));
  });
}
int orc_offset_by(int rank, const uint64_t* lo, const uint64_t* hi, int orank, const uint64_t* olo, const uint64_t* ohi,
                  uint64_t* out_lo, uint64_t* out_hi) {
  return guard([&] {
    Box b = core::offset_by(box_from(rank, lo, hi), box_from(orank, olo, ohi));
    for (size_t d = 0; d < b.size(); ++d) out_lo[d] = b[d].lo, out_hi[d] = b[d].hi;
  });
}
// spec dims with lo = hi = UINT64_MAX are unconstrained
int orc_spec_resolve(int rank, const uint64_t* lo, const uint64_t* hi, int srank, const uint64_t* shape, uint64_t* out_lo,
                     uint64_t* out_hi) {
  return guard([&] {
    Box b = core::spec_resolve(box_from(rank, lo, hi), shape_from(srank, shape));
    for (size_t d = 0; d < b.size(); ++d) out_lo[d] = b[d].lo, out_hi[d] = b[d].hi;
  });
}

int orc_even_split(int rank, const uint64_t* shape, int dim, uint64_t ways, int* n_out, uint64_t* pts_out) {
  return guard([&] {
    auto g = core::even_split(shape_from(rank, shape), size_t(dim), ways);
    size_t k = 0;
    for (size_t d = 0; d < g.size(); ++d) {
      n_out[d] = int(g[d].size());
      for (auto p : g[d]) pts_out[k++] = p;
    }
  });
}

// spec=1 parses a RangeSpec; unconstrained dims come back as lo=hi=UINT64_MAX
int orc_range_parse(const char* text, int spec, int* rank, uint64_t* lo, uint64_t* hi) {
  return guard([&] {
#ifdef ORACLE_REFERENCE_CORE
    // the reference's own Range::parse / RangeSpec::parse (range.cpp:135-193)
    Box b = core::guarded([&] {
      Box r;
      if (spec) {
        const reshard::RangeSpec rs = reshard::RangeSpec::parse(text);
        for (auto& d : rs.dims())
          r.push_back(d ? Iv{d->lo, d->hi} : Iv{UINT64_MAX, UINT64_MAX});
      } else {
        r = core::from_ref(reshard::Range::parse(text));
      }
      return r;
    });
#else
    Box b = parse_box(text, spec != 0);
#endif
    if (b.size() > kMaxRank) fail(MalformedFrame, "rank too large");
    *rank = int(b.size());
    for (size_t i = 0; i < b.size(); ++i) lo[i] = b[i].lo, hi[i] = b[i].hi;
  });
}

// ---- hash / rng ------------------------------------------------------------------------
#ifdef ORACLE_REFERENCE_CORE
// the reference's header-only hash.hpp
uint64_t orc_fnv1a64(const uint8_t* p, uint64_t n) { return reshard::fnv1a64(std::span<const uint8_t>(p, n)); }
uint64_t orc_splitmix64_next(uint64_t* state) { return reshard::splitmix64_next(*state); }
uint64_t orc_next_below(uint64_t* state, uint64_t n) {
  // SplitMix64 keeps its state private; replay from the seed through the public API
  reshard::SplitMix64 r(*state);
  uint64_t v = r.next_below(n);
  if (n != 0) reshard::splitmix64_next(*state);
  return v;
}
#else
uint64_t orc_fnv1a64(const uint8_t* p, uint64_t n) { return fnv1a(p, n); }
uint64_t orc_splitmix64_next(uint64_t* state) { return mix64(*state += kGolden); }
uint64_t orc_next_below(uint64_t* state, uint64_t n) {
  Rng r{*state};
  uint64_t v = r.below(n);
  *state = r.s;
  return v;
}
#endif
void orc_stream_bytes(uint64_t seed, uint64_t off, uint64_t n, uint8_t* out) { stream_bytes(seed, off, n, out); }
uint64_t orc_path_seed(const char* path) { return path_seed(path); }

// ---- catalog ---------------------------------------------------------------------------
void* orc_catalog_new(void) { return new Catalog; }
void orc_catalog_free(void* c) { delete static_cast<Catalog*>(c); }
int orc_catalog_add(void* c, const char* path, int dtype, int rank, const uint64_t* shape, int tp_dim, int layer) {
  return guard([&] {
    width_of(dtype);
    static_cast<Catalog*>(c)->e.push_back({path, dtype, shape_from(rank, shape), tp_dim, layer});
  });
}
void* orc_catalog_gpt(uint64_t h, uint64_t L, uint64_t S, uint64_t V, int kind) {
  return new Catalog(gpt_catalog(h, L, S, V, kind));
}
int orc_catalog_size(const void* c) { return int(static_cast<const Catalog*>(c)->e.size()); }
int orc_catalog_get(const void* c, int i, char* name, int cap, int* dtype, int* rank, uint64_t* shape, int* tp_dim,
                    int* layer) {
  return guard([&] {
    const Entry& e = static_cast<const Catalog*>(c)->e.at(size_t(i));
    std::snprintf(name, size_t(cap), "%s", e.path.c_str());
    *dtype = e.dtype, *rank = int(e.shape.size()), *tp_dim = e.tp_dim, *layer = e.layer;
    for (size_t d = 0; d < e.shape.size(); ++d) shape[d] = e.shape[d];
  });
}

// ---- PTC -------------------------------------------------------------------------------
int orc_build_strategy(const void* cat, int n_dev, const uint32_t* workers, const uint32_t* locals, int T, int P,
                       int D, void** out) {
  return guard([&] {
    std::vector<Dev> devs;
    for (int i = 0; i < n_dev; ++i) devs.push_back({workers[i], locals[i]});
    *out = new std::shared_ptr<const Ptc>(std::make_shared<const Ptc>(build_strategy(*static_cast<const Catalog*>(cat), devs, T, P, D)));
  });
}
void orc_ptc_free(void* p) { delete static_cast<std::shared_ptr<const Ptc>*>(p); }

// test hook: replace alpha of one partition (to construct invalid PTCs for validate())
int orc_ptc_set_alpha(void* p, int part, int n, const uint32_t* workers, const uint32_t* locals) {
  return guard([&] {
    auto& sp = *static_cast<std::shared_ptr<const Ptc>*>(p);
    auto q = std::make_shared<Ptc>(*sp);
    q->alpha.at(size_t(part)).clear();
    for (int i = 0; i < n; ++i) q->alpha[size_t(part)].push_back({workers[i], locals[i]});
    sp = q;
  });
}
int orc_ptc_set_sigma(void* p, int t, int rank, const int* npts, const uint64_t* pts) {
  return guard([&] {
    auto& sp = *static_cast<std::shared_ptr<const Ptc>*>(p);
    auto q = std::make_shared<Ptc>(*sp);
    q->sigma.at(size_t(t)) = grid_from(rank, npts, pts);
    sp = q;
  });
}

int orc_validate(const void* p, char* buf, int cap, int* n_violations) {
  return guard([&] {
    auto v = validate(**static_cast<const std::shared_ptr<const Ptc>*>(p));
    std::string s;
    for (auto& x : v) s += x + "\n";
    std::snprintf(buf, size_t(cap), "%s", s.c_str());
    *n_violations = int(v.size());
  });
}

// hosted_subtensors: tensor index + cell box per entry; returns count in *n (may exceed cap)
int orc_hosted(const void* p, uint32_t worker, uint32_t local, int cap, int* t_out, uint64_t* lo, uint64_t* hi,
               int* n) {
  return guard([&] {
    const Ptc& ptc = **static_cast<const std::shared_ptr<const Ptc>*>(p);
    auto h = hosted(ptc, Dev{worker, local});
    *n = int(h.size());
    for (int i = 0; i < int(h.size()) && i < cap; ++i) {
      t_out[i] = int(h[i].first);
      const Box& b = ptc.cells[h[i].first][h[i].second];
      for (size_t d = 0; d < b.size(); ++d) lo[size_t(i) * kMaxRank + d] = b[d].lo, hi[size_t(i) * kMaxRank + d] = b[d].hi;
    }
  });
}

// ---- planner ---------------------------------------------------------------------------
int orc_generate_plan(const void* a, const void* b, int n_failed, const uint32_t* fw, const uint32_t* fl, void** out) {
  return guard([&] {
    std::set<Dev> failed;
    for (int i = 0; i < n_failed; ++i) failed.insert({fw[i], fl[i]});
    auto* pl = new OrcPlan{generate_plan(*static_cast<const std::shared_ptr<const Ptc>*>(a),
                                         *static_cast<const std::shared_ptr<const Ptc>*>(b), failed)};
    *out = pl;
  });
}
void orc_plan_free(void* p) { delete static_cast<OrcPlan*>(p); }

// stats[0..6] = n_split, n_move, n_merge, moved bytes, resident-relayout bytes, kept bytes, total dst bytes
int orc_plan_stats(const void* pp, uint64_t* stats) {
  return guard([&] {
    const Plan& p = static_cast<const OrcPlan*>(pp)->p;
    uint64_t moved = 0, relayout = 0, kept = 0, total = 0;
    for (auto& op : p.ops)
      if (op.kind == Op::Move) moved += op.bytes;
    const Ptc &a = *p.a, &b = *p.b;
    for (auto& r2 : b.devices)
      for (auto [t, i] : hosted(b, r2)) {
        const Box& c = b.cells[t][i];
        uint64_t w = width_of(b.cat.e[t].dtype);
        total += count_of(extents_of(c)) * w;
        auto g = core::grid_cells(p.refine[t], b.cat.e[t].shape);
        for (auto& f : g) {
          if (!box_contains(c, f)) continue;
          size_t v = cell_containing(a.cells[t], f);
          if (hosts(a, t, v, r2) && !p.failed.count(r2)) {
            if (f == a.cells[t][v] && f == c) kept += count_of(extents_of(f)) * w;
            else relayout += count_of(extents_of(f)) * w;
          }
        }
      }
    stats[0] = p.n_split, stats[1] = p.n_move, stats[2] = p.n_merge, stats[3] = moved, stats[4] = relayout;
    stats[5] = kept, stats[6] = total;
  });
}

// plan_cost: per device of a ∪ b (sorted), ingress/egress.
int orc_plan_cost(const void* pp, int cap, uint32_t* w, uint32_t* l, uint64_t* ingress, uint64_t* egress, int* n) {
  return guard([&] {
    const Plan& p = static_cast<const OrcPlan*>(pp)->p;
    std::map<Dev, std::pair<uint64_t, uint64_t>> m;
    for (auto& d : p.a->devices) m[d];
    for (auto& d : p.b->devices) m[d];
    for (auto& op : p.ops)
      if (op.kind == Op::Move) m[op.dst].first += op.bytes, m[op.dev].second += op.bytes;
    *n = int(m.size());
    int i = 0;
    for (auto& [d, io] : m) {
      if (i >= cap) break;
      w[i] = d.w, l[i] = d.l, ingress[i] = io.first, egress[i] = io.second, ++i;
    }
  });
}

// returns bytes needed (including NUL); writes min(cap) bytes
int64_t orc_plan_text(const void* pp, char* buf, int64_t cap) {
  std::string s = plan_text(static_cast<const OrcPlan*>(pp)->p);
  if (buf && cap > 0) std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int64_t(s.size()) + 1;
}

// ---- executor --------------------------------------------------------------------------
// Source stores of `ptc` filled with the synthetic payload, tensors [t0, t1) only.
int orc_state_fill(const void* ptc, int64_t t0, int64_t t1, int n_skip, const uint32_t* skip_worker,
                   const uint32_t* skip_local, void** out) {
  return guard([&] {
    std::set<Dev> skip;
    for (int i = 0; i < n_skip; ++i) skip.insert(Dev{skip_worker[i], skip_local[i]});
    *out = new State(fill_state(**static_cast<const std::shared_ptr<const Ptc>*>(ptc), size_t(t0), size_t(t1), skip));
  });
}
void orc_state_free(void* s) { delete static_cast<State*>(s); }

int orc_apply(const void* plan, const void* src, int64_t t0, int64_t t1, int n_threads, int per_device, double* seconds,
              uint64_t* moved, uint64_t* local, void** out) {
  return guard([&] {
    ApplyReport rep;
    *out = new State(apply_plan(static_cast<const OrcPlan*>(plan)->p, *static_cast<const State*>(src), size_t(t0),
                                size_t(t1), n_threads, &rep, per_device != 0));
    if (seconds) *seconds = rep.seconds;
    if (moved) *moved = rep.moved;
    if (local) *local = rep.local;
  });
}

// Copy out one stored cell; *nbytes = its size.  buf may be null to query the size.
int orc_state_cell(const void* s, uint32_t worker, uint32_t local, int t, int rank, const uint64_t* lo,
                   const uint64_t* hi, uint8_t* buf, uint64_t cap, uint64_t* nbytes) {
  return guard([&] {
    const State& st = *static_cast<const State*>(s);
    auto it = st.store.find(Dev{worker, local});
    if (it == st.store.end()) fail(UnknownDevice, "no store");
    auto jt = it->second.find(CellKey{size_t(t), box_from(rank, lo, hi)});
    if (jt == it->second.end()) fail(NotFound, "cell not stored");
    auto& by = core::bytes_of(*jt->second);
    *nbytes = by.size();
    if (buf) std::memcpy(buf, by.data(), std::min<uint64_t>(cap, by.size()));
  });
}

int orc_state_digest(const void* ptc, const void* s, int t, uint64_t* digest) {
  return guard([&] {
    *digest = state_digest(**static_cast<const std::shared_ptr<const Ptc>*>(ptc), *static_cast<const State*>(s), size_t(t));
  });
}

// Full base tensor bytes (small tensors only) and its digest.
int orc_base_bytes(const void* cat, int t, uint8_t* out) {
  return guard([&] {
    const Entry& e = static_cast<const Catalog*>(cat)->e.at(size_t(t));
    auto v = gen_box(e, full_box(e.shape));
    std::memcpy(out, v.data(), v.size());
  });
}
int orc_base_digest(const void* cat, int t, uint64_t* digest) {
  return guard([&] {
    const Entry& e = static_cast<const Catalog*>(cat)->e.at(size_t(t));
    auto v = gen_box(e, full_box(e.shape));
    *digest = fnv1a(v.data(), v.size());
  });
}
int orc_box_bytes(const void* cat, int t, int rank, const uint64_t* lo, const uint64_t* hi, uint8_t* out) {
  return guard([&] {
    const Entry& e = static_cast<const Catalog*>(cat)->e.at(size_t(t));
    auto v = gen_box(e, box_from(rank, lo, hi));
    std::memcpy(out, v.data(), v.size());
  });
}

// ---- dataset ---------------------------------------------------------------------------
void orc_shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm) { shuffle_epoch(n, seed, epoch, perm); }

int orc_repartition_counts(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t* counts) {
  return guard([&] {
    repart_check(n, B, at_step, dp);
    for (uint64_t d = 0; d < dp; ++d) counts[d] = repart_count(n, B, at_step, dp, d);
  });
}

int orc_repartition_positions(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t d, uint64_t* pos) {
  return guard([&] {
    repart_check(n, B, at_step, dp);
    if (d >= dp) fail(IndexOutOfRange, "rank out of range");
    uint64_t b = B / dp, nb = (n + B - 1) / B, k = 0;
    for (uint64_t i = at_step; i < nb; ++i)
      for (uint64_t p = i * B + d * b; p < std::min(i * B + d * b + b, n); ++p) pos[k++] = p;
  });
}

// locate_sample for the k-th local sample of rank d, class from the
// caller's per-file table (0 local, 1 peer, 2 remote — priority order of SPEC.md:357).
int orc_locate_sample(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t d, uint64_t k,
                      const uint64_t* perm, const uint64_t* samples, const uint8_t* file_class, uint64_t* out4) {
  return guard([&] {
    repart_check(n, B, at_step, dp);
    uint64_t cnt = repart_count(n, B, at_step, dp, d);
    if (k >= cnt) fail(IndexOutOfRange, "k beyond the local partition");
    uint64_t b = B / dp, nb = (n + B - 1) / B, seen = 0;
    for (uint64_t i = at_step; i < nb; ++i) {
      uint64_t lo = i * B + d * b, hi = std::min(lo + b, n);
      if (hi <= lo) continue;
      if (k < seen + (hi - lo)) {
        uint64_t pos = lo + (k - seen);
        const uint64_t* s = samples + 3 * perm[pos];
        out4[0] = s[0], out4[1] = s[1], out4[2] = s[2], out4[3] = file_class[s[0]];
        return;
      }
      seen += hi - lo;
    }
  });
}

// The repartition gather for rank d — the CPU reference of the K5 kernel.  Outputs, for
// the rank's k-th remaining sample: pos[k], ent[3k..3k+2] = samples[perm[pos]], boff[k] =
// exclusive prefix sum of lengths, and qidx = k's stably partitioned by locator class
// (local, then peer, then remote) with qcount[3].  n_threads > 1 splits positions in
// contiguous chunks (two-pass scan).  Returns seconds spent in *seconds.
int orc_dataset_gather(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t d, const uint64_t* perm,
                       const uint64_t* samples, const uint8_t* file_class, uint64_t* pos, uint64_t* ent,
                       uint64_t* boff, uint32_t* qidx, uint64_t* qcount, int n_threads, double* seconds) {
  return guard([&] {
    repart_check(n, B, at_step, dp);
    if (d >= dp) fail(IndexOutOfRange, "rank out of range");
    const uint64_t cnt = repart_count(n, B, at_step, dp, d);
    const uint64_t b = B / dp;
    auto t0 = std::chrono::steady_clock::now();
    int nt = std::max(1, n_threads);
    std::vector<uint64_t> chunk_len(nt, 0), chunk_cls(size_t(nt) * 3, 0);
    auto range_of = [&](int i) { return std::pair<uint64_t, uint64_t>(cnt * i / nt, cnt * (i + 1) / nt); };
    // pass 1: positions, gather, per-chunk sums
    auto pass1 = [&](int i) {
      auto [k0, k1] = range_of(i);
      uint64_t s = 0, c[3] = {0, 0, 0};
      for (uint64_t k = k0; k < k1; ++k) {
        uint64_t batch = at_step + k / b, p = batch * B + d * b + k % b;
        pos[k] = p;
        const uint64_t* e = samples + 3 * perm[p];
        ent[3 * k] = e[0], ent[3 * k + 1] = e[1], ent[3 * k + 2] = e[2];
        s += e[2];
        ++c[file_class[e[0]]];
      }
      chunk_len[i] = s;
      for (int q = 0; q < 3; ++q) chunk_cls[size_t(i) * 3 + q] = c[q];
    };
    // trailing partial batch: positions beyond N are skipped by construction of cnt only
    // when N % B == 0 or the slice is full; handle the general case serially.
    bool regular = (n % B) == 0;
    if (!regular) nt = 1, chunk_len.assign(1, 0), chunk_cls.assign(3, 0);
    if (regular) {
      std::vector<std::thread> th;
      for (int i = 0; i < nt; ++i) th.emplace_back(pass1, i);
      for (auto& x : th) x.join();
    } else {
      uint64_t k = 0, s = 0, c[3] = {0, 0, 0};
      uint64_t nb = (n + B - 1) / B;
      for (uint64_t i = at_step; i < nb; ++i)
        for (uint64_t p = i * B + d * b; p < std::min(i * B + d * b + b, n); ++p, ++k) {
          pos[k] = p;
          const uint64_t* e = samples + 3 * perm[p];
          ent[3 * k] = e[0], ent[3 * k + 1] = e[1], ent[3 * k + 2] = e[2];
          s += e[2];
          ++c[file_class[e[0]]];
        }
      chunk_len[0] = s;
      for (int q = 0; q < 3; ++q) chunk_cls[q] = c[q];
    }
    // exclusive scans over chunks
    std::vector<uint64_t> len_base(nt, 0), cls_base(size_t(nt) * 3, 0);
    uint64_t tot[3] = {0, 0, 0};
    for (int q = 0; q < 3; ++q)
      for (int i = 0; i < nt; ++i) cls_base[size_t(i) * 3 + q] = tot[q], tot[q] += chunk_cls[size_t(i) * 3 + q];
    for (int i = 1; i < nt; ++i) len_base[i] = len_base[i - 1] + chunk_len[i - 1];
    const uint64_t qstart[3] = {0, tot[0], tot[0] + tot[1]};
    auto pass2 = [&](int i) {
      auto [k0, k1] = nt == 1 ? std::pair<uint64_t, uint64_t>(0, cnt) : range_of(i);
      uint64_t s = len_base[i];
      uint64_t c[3] = {cls_base[size_t(i) * 3], cls_base[size_t(i) * 3 + 1], cls_base[size_t(i) * 3 + 2]};
      for (uint64_t k = k0; k < k1; ++k) {
        boff[k] = s;
        s += ent[3 * k + 2];
        int q = file_class[ent[3 * k]];
        qidx[qstart[q] + c[q]++] = uint32_t(k);
      }
    };
    {
      std::vector<std::thread> th;
      for (int i = 0; i < nt; ++i) th.emplace_back(pass2, i);
      for (auto& x : th) x.join();
    }
    for (int q = 0; q < 3; ++q) qcount[q] = tot[q];
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

}  // extern "C"
