// reshard/core.hpp — error codes, dtypes, box algebra and split grids for the B200 reshard
// path.  Same API names and error numbering as the reference tensor-core:
//   Errc / Error / raise      proj/include/reshard/error.hpp:8-64
//   Dtype / dtype_width        proj/include/reshard/tensor/dtype.hpp:12-31  (+ BF16 = 4)
//   Interval / Range           proj/include/reshard/tensor/range.hpp:17-66
//   SplitGrid / grid_refine    proj/include/reshard/tensor/split_grid.hpp:13-55
//   fnv1a64 / splitmix64       proj/include/reshard/util/hash.hpp:13-63
// Implementation is independent: fixed-capacity boxes (no heap per range) because the
// planner walks ~10^4 fragments per reshard and lowers them to device copy descriptors.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <span>
#include <string_view>
#include <vector>

namespace reshard {

enum class Errc : int {
  RangeOutOfBounds = 0, RankMismatch, ShapeMismatch, TilingGap, TilingOverlap, DtypeMismatch,
  InvalidSplitPoint, InvalidTensor,
  IndivisibleLayerCount, IndivisibleSliceDim, DeviceCountMismatch, InvalidJobConfig,
  MalformedConfig, InconsistentBaseShape, CoverageGap, UnknownDevice,
  CatalogMismatch, UnsatisfiableFragment, NoSource,
  NotFound, IndivisibleBatch, StepBeyondEpoch, IndexOutOfRange, InvalidReplicaCount,
  MalformedFrame, UnknownVerb, BadRange, ConnectionFailed,
  CheckpointRequired, LayoutMismatch, IoError,
  ScriptError,
  // appended after ScriptError (the reference numbering above is stable):
  CudaError,         // a CUDA runtime / driver call failed
  DeviceUnavailable, // no usable GPU, or the extension was built without one
  InvalidArgument,   // C-ABI misuse (null handle, bad size)
};
constexpr int kErrcCount = static_cast<int>(Errc::InvalidArgument) + 1;

const char* errc_name(Errc c);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what)
      : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

[[noreturn]] void raise(Errc code, const std::string& what);

// ---- dtypes --------------------------------------------------------------------------
enum class Dtype : uint8_t { F32 = 0, F16 = 1, I64 = 2, U8 = 3, BF16 = 4 };
size_t dtype_width(Dtype d);          // InvalidTensor for unknown codes
Dtype dtype_from_code(int code);      // InvalidTensor for unknown codes
Dtype dtype_from_name(std::string_view name);  // "f32"/"F32", ... "bf16"; MalformedConfig otherwise
const char* dtype_name(Dtype d);

// ---- boxes ---------------------------------------------------------------------------
constexpr int kMaxRank = 8;
using Shape = std::vector<uint64_t>;
uint64_t shape_elements(const Shape& s);

struct Interval {
  uint64_t lo = 0, hi = 0;
  uint64_t extent() const { return hi - lo; }
  bool operator==(const Interval&) const = default;
};

// Axis-aligned half-open box, rank <= kMaxRank, stored inline.
class Range {
 public:
  Range() = default;
  explicit Range(const std::vector<Interval>& dims);
  static Range full(const Shape& s);

  int rank() const { return rank_; }
  const Interval& dim(int i) const { return d_[i]; }
  Interval& dim(int i) { return d_[i]; }
  std::vector<Interval> dims() const { return {d_.begin(), d_.begin() + rank_}; }
  Shape extents() const;
  uint64_t elements() const;

  void check_against(const Shape& s) const;  // RankMismatch / RangeOutOfBounds
  bool valid_for(const Shape& s) const;
  bool contains(const Range& o) const;
  bool overlaps(const Range& o) const;
  Range rebase_into(const Range& outer) const;  // RangeOutOfBounds unless outer.contains(*this)
  Range offset_by(const Range& outer) const;    // inverse of rebase_into; RankMismatch / RangeOutOfBounds
  std::string to_string() const;
  static Range parse(std::string_view text);  // MalformedFrame

  bool operator==(const Range& o) const;
  bool operator<(const Range& o) const;

 private:
  int rank_ = 0;
  std::array<Interval, kMaxRank> d_{};
};

// A possibly partial selection `[:,2:4]` (range.hpp:70-91): unconstrained dims are nullopt.
class RangeSpec {
 public:
  RangeSpec() = default;
  explicit RangeSpec(std::vector<std::optional<Interval>> dims) : dims_(std::move(dims)) {}
  static RangeSpec from_range(const Range& r);
  size_t rank() const { return dims_.size(); }
  const std::vector<std::optional<Interval>>& dims() const { return dims_; }
  Range resolve(const Shape& s) const;  // RankMismatch / RangeOutOfBounds
  std::string to_string() const;
  static RangeSpec parse(std::string_view text);  // MalformedFrame
  bool operator==(const RangeSpec&) const = default;

 private:
  std::vector<std::optional<Interval>> dims_;
};

// Sorted interior split points per dimension; cells in lexicographic order, last dim fastest.
class SplitGrid {
 public:
  SplitGrid() = default;
  explicit SplitGrid(std::vector<std::vector<uint64_t>> pts) : pts_(std::move(pts)) {}
  static SplitGrid identity(size_t rank) { return SplitGrid(std::vector<std::vector<uint64_t>>(rank)); }
  static SplitGrid even_split(const Shape& s, size_t dim, uint64_t ways);

  size_t rank() const { return pts_.size(); }
  const std::vector<std::vector<uint64_t>>& points() const { return pts_; }
  void check_against(const Shape& s) const;  // RankMismatch / InvalidSplitPoint
  bool valid_for(const Shape& s) const;
  uint64_t cell_count() const;
  std::vector<Range> cells(const Shape& s) const;
  Range cell(const Shape& s, uint64_t index) const;               // IndexOutOfRange
  uint64_t cell_index_of(const Shape& s, const Range& r) const;   // InvalidSplitPoint when r crosses a boundary
  // per-dim index of the grid interval holding coordinate x (binary search)
  size_t interval_of(size_t dim, uint64_t x) const;
  bool operator==(const SplitGrid&) const = default;

 private:
  std::vector<std::vector<uint64_t>> pts_;
};

SplitGrid grid_refine(const SplitGrid& a, const SplitGrid& b);  // ShapeMismatch on rank

// ---- hashing / rng (hash.hpp) ----------------------------------------------------------
constexpr uint64_t kSplitmixGamma = 0x9e3779b97f4a7c15ull;
inline uint64_t splitmix64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t splitmix64_next(uint64_t& s) { return splitmix64_mix(s += kSplitmixGamma); }
class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t seed) : s_(seed) {}
  uint64_t next() { return splitmix64_next(s_); }
  uint64_t next_below(uint64_t n) { return n == 0 ? 0 : next() % n; }
  uint64_t state() const { return s_; }

 private:
  uint64_t s_;
};
uint64_t fnv1a64(const void* data, size_t n);
inline uint64_t fnv1a64(std::span<const uint8_t> bytes) { return fnv1a64(bytes.data(), bytes.size()); }  // hash.hpp:42
class Fnv1a64 {  // incremental digest (hash.hpp:13-40)
 public:
  static constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  static constexpr uint64_t kPrime = 0x100000001b3ull;
  Fnv1a64& update(const void* data, size_t n);
  Fnv1a64& update(std::span<const uint8_t> bytes) { return update(bytes.data(), bytes.size()); }
  Fnv1a64& update(std::string_view s) { return update(s.data(), s.size()); }
  Fnv1a64& update_u64(uint64_t v);  // 8 little-endian bytes
  uint64_t digest() const { return h_; }

 private:
  uint64_t h_ = 0xcbf29ce484222325ull;
};
// Synthetic payload seed of a base tensor: fnv1a64(path) ^ 0x7E9B1E0C.
uint64_t payload_seed(std::string_view path);

}  // namespace reshard
