// Host implementation of reshard/core.hpp.  Semantics (including error precedence) follow
// the reference tensor-core: range.cpp:36-193, split_grid.cpp:9-130, dtype.cpp:7-28,
// error.cpp:5-41; checked against it by tests/test_host_core.py through the C-ABI.
#include "reshard/core.hpp"

#include <algorithm>
#include <charconv>

namespace reshard {

static constexpr const char* kNames[kErrcCount] = {
    "RangeOutOfBounds", "RankMismatch", "ShapeMismatch", "TilingGap", "TilingOverlap",
    "DtypeMismatch", "InvalidSplitPoint", "InvalidTensor", "IndivisibleLayerCount",
    "IndivisibleSliceDim", "DeviceCountMismatch", "InvalidJobConfig", "MalformedConfig",
    "InconsistentBaseShape", "CoverageGap", "UnknownDevice", "CatalogMismatch",
    "UnsatisfiableFragment", "NoSource", "NotFound", "IndivisibleBatch", "StepBeyondEpoch",
    "IndexOutOfRange", "InvalidReplicaCount", "MalformedFrame", "UnknownVerb", "BadRange",
    "ConnectionFailed", "CheckpointRequired", "LayoutMismatch", "IoError", "ScriptError",
    "CudaError", "DeviceUnavailable", "InvalidArgument"};

const char* errc_name(Errc c) {
  int i = static_cast<int>(c);
  return (i >= 0 && i < kErrcCount) ? kNames[i] : "UnknownError";
}

void raise(Errc code, const std::string& what) { throw Error(code, what); }

size_t dtype_width(Dtype d) {
  static constexpr size_t w[] = {4, 2, 8, 1, 2};
  auto i = static_cast<unsigned>(d);
  if (i > 4) raise(Errc::InvalidTensor, "unknown dtype code " + std::to_string(i));
  return w[i];
}
Dtype dtype_from_code(int code) {
  if (code < 0 || code > 4) raise(Errc::InvalidTensor, "unknown dtype code " + std::to_string(code));
  return static_cast<Dtype>(code);
}
const char* dtype_name(Dtype d) {
  static constexpr const char* n[] = {"f32", "f16", "i64", "u8", "bf16"};
  auto i = static_cast<unsigned>(d);
  return i <= 4 ? n[i] : "?";
}

uint64_t shape_elements(const Shape& s) {
  uint64_t n = 1;
  for (uint64_t e : s) n *= e;
  return n;
}

// ---- Range -----------------------------------------------------------------------------
Range::Range(const std::vector<Interval>& dims) {
  if (dims.size() > size_t(kMaxRank)) raise(Errc::RankMismatch, "rank above " + std::to_string(kMaxRank));
  rank_ = int(dims.size());
  std::copy(dims.begin(), dims.end(), d_.begin());
}
Range Range::full(const Shape& s) {
  std::vector<Interval> v;
  for (uint64_t e : s) v.push_back({0, e});
  return Range(v);
}
Shape Range::extents() const {
  Shape s(static_cast<size_t>(rank_));
  for (int i = 0; i < rank_; ++i) s[size_t(i)] = d_[i].extent();
  return s;
}
uint64_t Range::elements() const {
  uint64_t n = 1;
  for (int i = 0; i < rank_; ++i) n *= d_[i].extent();
  return n;
}
void Range::check_against(const Shape& s) const {
  if (size_t(rank_) != s.size())
    raise(Errc::RankMismatch, "range rank " + std::to_string(rank_) + " vs tensor rank " + std::to_string(s.size()));
  for (int i = 0; i < rank_; ++i) {
    const Interval& v = d_[i];
    if (!(v.lo < v.hi && v.hi <= s[size_t(i)]))
      raise(Errc::RangeOutOfBounds, "interval [" + std::to_string(v.lo) + ":" + std::to_string(v.hi) +
                                        ") invalid for extent " + std::to_string(s[size_t(i)]) + " in dim " +
                                        std::to_string(i));
  }
}
bool Range::contains(const Range& o) const {
  if (o.rank_ != rank_) return false;
  for (int i = 0; i < rank_; ++i)
    if (o.d_[i].lo < d_[i].lo || o.d_[i].hi > d_[i].hi) return false;
  return true;
}
bool Range::overlaps(const Range& o) const {
  if (o.rank_ != rank_) return false;
  for (int i = 0; i < rank_; ++i)
    if (!(o.d_[i].lo < d_[i].hi && d_[i].lo < o.d_[i].hi)) return false;
  return true;
}
Range Range::rebase_into(const Range& outer) const {
  if (!outer.contains(*this)) raise(Errc::RangeOutOfBounds, "cannot rebase " + to_string() + " into " + outer.to_string());
  Range r = *this;
  for (int i = 0; i < rank_; ++i) r.d_[i].lo -= outer.d_[i].lo, r.d_[i].hi -= outer.d_[i].lo;
  return r;
}
std::string Range::to_string() const {
  std::string s(1, '[');
  for (int i = 0; i < rank_; ++i) {
    if (i) s.push_back(',');
    s += std::to_string(d_[i].lo);
    s.push_back(':');
    s += std::to_string(d_[i].hi);
  }
  s.push_back(']');
  return s;
}
bool Range::operator==(const Range& o) const {
  if (o.rank_ != rank_) return false;
  for (int i = 0; i < rank_; ++i)
    if (!(o.d_[i] == d_[i])) return false;
  return true;
}
bool Range::operator<(const Range& o) const {
  if (rank_ != o.rank_) return rank_ < o.rank_;
  for (int i = 0; i < rank_; ++i) {
    if (d_[i].lo != o.d_[i].lo) return d_[i].lo < o.d_[i].lo;
    if (d_[i].hi != o.d_[i].hi) return d_[i].hi < o.d_[i].hi;
  }
  return false;
}

static uint64_t parse_u64(std::string_view t) {
  uint64_t v = 0;
  auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
  if (ec != std::errc() || p != t.data() + t.size()) raise(Errc::MalformedFrame, "bad integer '" + std::string(t) + "'");
  return v;
}
Range Range::parse(std::string_view text) {
  if (text.size() < 2 || text.front() != '[' || text.back() != ']')
    raise(Errc::MalformedFrame, "range must be bracketed: '" + std::string(text) + "'");
  std::string_view body = text.substr(1, text.size() - 2);
  std::vector<Interval> dims;
  while (!body.empty() || !dims.empty()) {
    size_t comma = body.find(',');
    std::string_view item = body.substr(0, comma);
    size_t colon = item.find(':');
    if (colon == std::string_view::npos) raise(Errc::MalformedFrame, "interval needs ':' in '" + std::string(item) + "'");
    dims.push_back({parse_u64(item.substr(0, colon)), parse_u64(item.substr(colon + 1))});
    if (comma == std::string_view::npos) break;
    body = body.substr(comma + 1);
  }
  return Range(dims);
}

// ---- SplitGrid -------------------------------------------------------------------------
SplitGrid SplitGrid::even_split(const Shape& s, size_t dim, uint64_t ways) {
  if (dim >= s.size()) raise(Errc::RankMismatch, "split dim " + std::to_string(dim) + " out of rank");
  if (ways == 0 || s[dim] % ways) raise(Errc::IndivisibleSliceDim, "extent " + std::to_string(s[dim]) + " not divisible by " + std::to_string(ways));
  std::vector<std::vector<uint64_t>> p(s.size());
  const uint64_t step = s[dim] / ways;
  for (uint64_t k = 1; k < ways; ++k) p[dim].push_back(step * k);
  return SplitGrid(std::move(p));
}
void SplitGrid::check_against(const Shape& s) const {
  if (pts_.size() != s.size())
    raise(Errc::RankMismatch, "grid rank " + std::to_string(pts_.size()) + " vs tensor rank " + std::to_string(s.size()));
  for (size_t d = 0; d < pts_.size(); ++d)
    for (size_t i = 0; i < pts_[d].size(); ++i) {
      uint64_t p = pts_[d][i], prev = i ? pts_[d][i - 1] : 0;
      if (p == 0 || p >= s[d] || p <= prev)
        raise(Errc::InvalidSplitPoint, "split point " + std::to_string(p) + " invalid for extent " + std::to_string(s[d]) + " in dim " + std::to_string(d));
    }
}
uint64_t SplitGrid::cell_count() const {
  uint64_t n = 1;
  for (auto& p : pts_) n *= p.size() + 1;
  return n;
}
std::vector<Range> SplitGrid::cells(const Shape& s) const {
  check_against(s);
  const size_t r = pts_.size();
  const uint64_t n = cell_count();
  std::vector<Range> out;
  out.reserve(n);
  std::vector<Interval> dims(r);
  for (uint64_t k = 0; k < n; ++k) {
    uint64_t rest = k;
    for (size_t d = r; d-- > 0;) {
      const size_t m = pts_[d].size() + 1, i = rest % m;
      rest /= m;
      dims[d] = {i ? pts_[d][i - 1] : 0, i < pts_[d].size() ? pts_[d][i] : s[d]};
    }
    out.emplace_back(dims);
  }
  return out;
}
size_t SplitGrid::interval_of(size_t dim, uint64_t x) const {
  const auto& p = pts_[dim];
  return size_t(std::upper_bound(p.begin(), p.end(), x) - p.begin());
}
SplitGrid grid_refine(const SplitGrid& a, const SplitGrid& b) {
  if (a.rank() != b.rank()) raise(Errc::ShapeMismatch, "grids of different rank");
  std::vector<std::vector<uint64_t>> p(a.rank());
  for (size_t d = 0; d < a.rank(); ++d) {
    std::merge(a.points()[d].begin(), a.points()[d].end(), b.points()[d].begin(), b.points()[d].end(),
               std::back_inserter(p[d]));
    std::sort(p[d].begin(), p[d].end());  // inputs need not be sorted
    p[d].erase(std::unique(p[d].begin(), p[d].end()), p[d].end());
  }
  return SplitGrid(std::move(p));
}

uint64_t fnv1a64(const void* data, size_t n) {
  const auto* p = static_cast<const uint8_t*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}
uint64_t payload_seed(std::string_view path) { return fnv1a64(path.data(), path.size()) ^ 0x7E9B1E0Cull; }

}  // namespace reshard
