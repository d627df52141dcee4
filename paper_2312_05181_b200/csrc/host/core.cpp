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
Dtype dtype_from_name(std::string_view name) {
  static constexpr std::pair<const char*, Dtype> names[] = {
      {"f32", Dtype::F32}, {"F32", Dtype::F32}, {"f16", Dtype::F16}, {"F16", Dtype::F16},   {"i64", Dtype::I64},
      {"I64", Dtype::I64}, {"u8", Dtype::U8},   {"U8", Dtype::U8},   {"bf16", Dtype::BF16}, {"BF16", Dtype::BF16}};
  for (auto& [n, d] : names)
    if (name == n) return d;
  raise(Errc::MalformedConfig, "unknown dtype '" + std::string(name) + "'");
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
// Calls f(item) for every comma-separated item between the brackets; "[]" has none.
template <class F>
static void for_each_bracket_item(std::string_view text, F&& f) {
  if (text.size() < 2 || text.front() != '[' || text.back() != ']')
    raise(Errc::MalformedFrame, "range must be bracketed: '" + std::string(text) + "'");
  std::string_view body = text.substr(1, text.size() - 2);
  if (body.empty()) return;
  for (;;) {
    size_t comma = body.find(',');
    f(body.substr(0, comma));
    if (comma == std::string_view::npos) return;
    body = body.substr(comma + 1);
  }
}
static Interval parse_interval(std::string_view item) {
  size_t colon = item.find(':');
  if (colon == std::string_view::npos) raise(Errc::MalformedFrame, "interval needs ':' in '" + std::string(item) + "'");
  return {parse_u64(item.substr(0, colon)), parse_u64(item.substr(colon + 1))};
}
Range Range::parse(std::string_view text) {
  std::vector<Interval> dims;
  for_each_bracket_item(text, [&](std::string_view item) { dims.push_back(parse_interval(item)); });
  return Range(dims);
}
bool Range::valid_for(const Shape& s) const {
  if (size_t(rank_) != s.size()) return false;
  for (int i = 0; i < rank_; ++i)
    if (!(d_[i].lo < d_[i].hi && d_[i].hi <= s[size_t(i)])) return false;
  return true;
}
Range Range::offset_by(const Range& outer) const {
  if (rank_ != outer.rank_) raise(Errc::RankMismatch, "offset_by rank mismatch");
  Range r = *this;
  for (int i = 0; i < rank_; ++i) {
    if (d_[i].hi + outer.d_[i].lo > outer.d_[i].hi)
      raise(Errc::RangeOutOfBounds, "range " + to_string() + " exceeds " + outer.to_string());
    r.d_[i].lo += outer.d_[i].lo;
    r.d_[i].hi += outer.d_[i].lo;
  }
  return r;
}

// ---- RangeSpec -------------------------------------------------------------------------
RangeSpec RangeSpec::from_range(const Range& r) {
  std::vector<std::optional<Interval>> dims;
  for (int i = 0; i < r.rank(); ++i) dims.emplace_back(r.dim(i));
  return RangeSpec(std::move(dims));
}
Range RangeSpec::resolve(const Shape& s) const {
  if (dims_.size() != s.size())
    raise(Errc::RankMismatch, "range spec rank " + std::to_string(dims_.size()) + " vs tensor rank " + std::to_string(s.size()));
  std::vector<Interval> dims;
  for (size_t i = 0; i < dims_.size(); ++i) dims.push_back(dims_[i] ? *dims_[i] : Interval{0, s[i]});
  Range r(dims);
  r.check_against(s);
  return r;
}
std::string RangeSpec::to_string() const {
  std::string s(1, '[');
  for (size_t i = 0; i < dims_.size(); ++i) {
    if (i) s.push_back(',');
    if (dims_[i])
      s += std::to_string(dims_[i]->lo) + ":" + std::to_string(dims_[i]->hi);
    else
      s.push_back(':');
  }
  s.push_back(']');
  return s;
}
RangeSpec RangeSpec::parse(std::string_view text) {
  std::vector<std::optional<Interval>> dims;
  for_each_bracket_item(text, [&](std::string_view item) {
    if (item == ":")
      dims.emplace_back(std::nullopt);
    else
      dims.emplace_back(parse_interval(item));
  });
  return RangeSpec(std::move(dims));
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
bool SplitGrid::valid_for(const Shape& s) const {
  try {
    check_against(s);
    return true;
  } catch (const Error&) {
    return false;
  }
}
Range SplitGrid::cell(const Shape& s, uint64_t index) const {
  check_against(s);
  std::vector<Interval> dims(pts_.size());
  uint64_t rest = index;
  for (size_t d = pts_.size(); d-- > 0;) {
    const uint64_t m = pts_[d].size() + 1, i = rest % m;
    rest /= m;
    dims[d] = {i ? pts_[d][i - 1] : 0, i < pts_[d].size() ? pts_[d][i] : s[d]};
  }
  if (rest != 0) raise(Errc::IndexOutOfRange, "cell index " + std::to_string(index) + " out of range");
  return Range(dims);
}
uint64_t SplitGrid::cell_index_of(const Shape& s, const Range& r) const {
  check_against(s);
  r.check_against(s);
  uint64_t index = 0;
  for (size_t d = 0; d < pts_.size(); ++d) {
    const Interval& v = r.dim(int(d));
    const size_t i = interval_of(d, v.lo);
    const uint64_t hi = i < pts_[d].size() ? pts_[d][i] : s[d];
    if (v.hi > hi) raise(Errc::InvalidSplitPoint, "range " + r.to_string() + " crosses a grid boundary");
    index = index * (pts_[d].size() + 1) + i;
  }
  return index;
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

Fnv1a64& Fnv1a64::update(const void* data, size_t n) {
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < n; ++i) h_ = (h_ ^ p[i]) * 0x100000001b3ull;
  return *this;
}
Fnv1a64& Fnv1a64::update_u64(uint64_t v) {
  uint8_t le[8];
  for (int i = 0; i < 8; ++i) le[i] = uint8_t(v >> (8 * i));
  return update(le, 8);
}
uint64_t fnv1a64(const void* data, size_t n) { return Fnv1a64().update(data, n).digest(); }
uint64_t payload_seed(std::string_view path) { return fnv1a64(path.data(), path.size()) ^ 0x7E9B1E0Cull; }

}  // namespace reshard
