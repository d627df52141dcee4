// Parallelization-configuration documents (see reshard/config.hpp).  Includes a small
// strict JSON reader/writer (no third-party JSON library is available).
#include "reshard/config.hpp"

#include <algorithm>
#include <map>
#include <set>

namespace reshard {

namespace {

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  std::string s;  // string value, or the literal text of a number
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (auto& [key, v] : obj)
      if (key == k) return &v;
    return nullptr;
  }
};

class Reader {
 public:
  explicit Reader(const std::string& t) : p_(t.data()), e_(t.data() + t.size()) {}
  Json document() {
    Json v = value();
    ws();
    if (p_ != e_) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const std::string& what) { raise(Errc::MalformedConfig, "JSON: " + what); }
  void ws() {
    while (p_ != e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ != e_ && *p_ == c) return ++p_, true;
    return false;
  }
  void expect(char c) {
    if (!eat(c)) bad(std::string("expected '") + c + "'");
  }
  Json value() {
    ws();
    if (p_ == e_) bad("unexpected end");
    Json v;
    switch (*p_) {
      case '{':
        ++p_;
        v.kind = Json::Obj;
        if (eat('}')) return v;
        do {
          ws();
          std::string k = string();
          expect(':');
          v.obj.emplace_back(std::move(k), value());
        } while (eat(','));
        expect('}');
        return v;
      case '[':
        ++p_;
        v.kind = Json::Arr;
        if (eat(']')) return v;
        do v.arr.push_back(value());
        while (eat(','));
        expect(']');
        return v;
      case '"':
        v.kind = Json::Str;
        v.s = string();
        return v;
      case 't': word("true"), v.kind = Json::Bool, v.b = true; return v;
      case 'f': word("false"), v.kind = Json::Bool; return v;
      case 'n': word("null"); return v;
      default: {
        const char* q = p_;
        if (p_ != e_ && (*p_ == '-' || *p_ == '+')) ++p_;
        while (p_ != e_ && ((*p_ >= '0' && *p_ <= '9') || *p_ == '.' || *p_ == 'e' || *p_ == 'E' || *p_ == '-' || *p_ == '+')) ++p_;
        if (q == p_) bad("unexpected character");
        v.kind = Json::Num;
        v.s.assign(q, p_);
        return v;
      }
    }
  }
  void word(const char* w) {
    for (const char* c = w; *c; ++c, ++p_)
      if (p_ == e_ || *p_ != *c) bad("bad literal");
  }
  std::string string() {
    if (p_ == e_ || *p_ != '"') bad("expected string");
    ++p_;
    std::string out;
    while (p_ != e_ && *p_ != '"') {
      char c = *p_++;
      if (c == '\\') {
        if (p_ == e_) bad("bad escape");
        char x = *p_++;
        switch (x) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (e_ - p_ < 4) bad("bad \\u escape");
            unsigned cp = std::stoul(std::string(p_, p_ + 4), nullptr, 16);
            p_ += 4;
            if (cp < 0x80) out += char(cp);
            else if (cp < 0x800) out += char(0xC0 | (cp >> 6)), out += char(0x80 | (cp & 0x3F));
            else out += char(0xE0 | (cp >> 12)), out += char(0x80 | ((cp >> 6) & 0x3F)), out += char(0x80 | (cp & 0x3F));
            break;
          }
          default: out += x;
        }
      } else {
        out += c;
      }
    }
    if (p_ == e_) bad("unterminated string");
    ++p_;
    return out;
  }
  const char* p_;
  const char* e_;
};

uint64_t as_u64(const Json& j, const char* what) {
  if (j.kind != Json::Num || j.s.empty() || j.s.find_first_not_of("0123456789") != std::string::npos)
    raise(Errc::MalformedConfig, std::string(what) + " must be a non-negative integer");
  uint64_t v = 0;
  for (char c : j.s) {
    const uint64_t nv = v * 10 + uint64_t(c - '0');
    if (nv / 10 != v) raise(Errc::MalformedConfig, std::string(what) + " overflows 64 bits");
    v = nv;
  }
  return v;
}

Dtype dtype_named(const std::string& n) {
  static const std::map<std::string, Dtype> m = {{"f32", Dtype::F32}, {"F32", Dtype::F32}, {"f16", Dtype::F16},
                                                 {"F16", Dtype::F16}, {"i64", Dtype::I64}, {"I64", Dtype::I64},
                                                 {"u8", Dtype::U8},   {"U8", Dtype::U8},   {"bf16", Dtype::BF16},
                                                 {"BF16", Dtype::BF16}};
  auto it = m.find(n);
  if (it == m.end()) raise(Errc::MalformedConfig, "unknown dtype '" + n + "'");  // dtype.cpp:17-23
  return it->second;
}

struct Leaf {
  std::string base;
  Dtype dtype;
  Shape shape;
  Range range;
};

void collect(const Json& node, std::vector<Leaf>& out) {
  if (node.kind != Json::Obj) raise(Errc::MalformedConfig, "model tree nodes must be objects");
  if (const Json* base = node.get("base")) {
    const Json *shape = node.get("shape"), *range = node.get("range"), *dtype = node.get("dtype");
    if (base->kind != Json::Str || !shape || shape->kind != Json::Arr || !dtype || dtype->kind != Json::Str)
      raise(Errc::MalformedConfig, "leaf needs base, shape and dtype");
    Leaf l{base->s, dtype_named(dtype->s), {}, {}};
    for (auto& e : shape->arr) l.shape.push_back(as_u64(e, "extent"));
    if (l.shape.size() > size_t(kMaxRank)) raise(Errc::MalformedConfig, l.base + ": rank above 8");
    for (auto e : l.shape)
      if (e == 0) raise(Errc::MalformedConfig, l.base + ": zero extent");
    if (!range || range->kind == Json::Null) {
      l.range = Range::full(l.shape);
    } else {
      if (range->kind != Json::Arr || range->arr.size() != l.shape.size())
        raise(Errc::MalformedConfig, l.base + ": range rank differs from shape");
      std::vector<Interval> iv;
      for (auto& d : range->arr) {
        if (d.kind != Json::Arr || d.arr.size() != 2) raise(Errc::MalformedConfig, l.base + ": range entries are [lo, hi]");
        iv.push_back({as_u64(d.arr[0], "lo"), as_u64(d.arr[1], "hi")});
      }
      l.range = Range(iv);
      try {
        l.range.check_against(l.shape);
      } catch (const Error& e) {
        raise(Errc::MalformedConfig, l.base + ": " + e.what());
      }
    }
    out.push_back(std::move(l));
    return;
  }
  for (auto& [k, v] : node.obj) collect(v, out);
}

void esc(std::string& out, const std::string& s) {
  out += '"';
  for (char c : s) {
    if (c == '"' || c == '\\') out += '\\', out += c;
    else if (c == '\n') out += "\\n";
    else out += c;
  }
  out += '"';
}

// Insertion-ordered tree of path segments for serialization.
struct Node {
  std::vector<std::pair<std::string, Node>> kids;
  std::string leaf;  // JSON text of a leaf
  Node& child(const std::string& k) {
    for (auto& [key, n] : kids)
      if (key == k) return n;
    kids.emplace_back(k, Node{});
    return kids.back().second;
  }
  void emit(std::string& out) const {
    if (!leaf.empty()) {
      out += leaf;
      return;
    }
    out += '{';
    for (size_t i = 0; i < kids.size(); ++i) {
      if (i) out += ", ";
      esc(out, kids[i].first);
      out += ": ";
      kids[i].second.emit(out);
    }
    out += '}';
  }
};

// Tree position of a tensor: the parameter path split at '.', then the optimizer state
// ("<state>/<param>") as the innermost key, so the model tree keeps the catalog's
// param-major order and parsing it back reproduces the tensor order.
std::vector<std::string> segments(const std::string& path) {
  std::vector<std::string> seg;
  const size_t slash = path.find('/');
  const std::string state = slash == std::string::npos ? "" : path.substr(0, slash);
  const std::string rest = slash == std::string::npos ? path : path.substr(slash + 1);
  std::string cur;
  for (char c : rest) {
    if (c == '.' || c == '/') {
      seg.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  seg.push_back(cur);
  if (!state.empty()) seg.push_back(state);
  return seg;
}

}  // namespace

PTC parse_parallel_config(const std::string& json, const std::vector<DeviceId>& devices) {
  const Json root = Reader(json).document();
  if (root.kind != Json::Arr) raise(Errc::MalformedConfig, "top level must be a list of ranks");
  const size_t ranks = root.arr.size();
  if (!devices.empty() && devices.size() != ranks)
    raise(Errc::DeviceCountMismatch, std::to_string(ranks) + " ranks for " + std::to_string(devices.size()) + " devices");
  PTC p;
  for (size_t r = 0; r < ranks; ++r) p.devices.push_back(devices.empty() ? DeviceId{0, uint32_t(r)} : devices[r]);
  if (std::set<DeviceId>(p.devices.begin(), p.devices.end()).size() != p.devices.size())
    raise(Errc::MalformedConfig, "duplicate devices");
  p.job = JobConfig{1, 1, 1};
  std::map<std::string, uint32_t> index;
  std::vector<std::map<Range, std::vector<uint32_t>>> holders;  // per tensor: range -> ranks
  for (size_t r = 0; r < ranks; ++r) {
    std::vector<Leaf> leaves;
    collect(root.arr[r], leaves);
    for (auto& l : leaves) {
      auto it = index.find(l.base);
      if (it == index.end()) {
        it = index.emplace(l.base, uint32_t(p.catalog.tensors.size())).first;
        p.catalog.add(TensorSpec{l.base, l.dtype, l.shape, -1, 0});
        holders.emplace_back();
      }
      const TensorSpec& t = p.catalog.tensors[it->second];
      if (t.shape != l.shape || t.dtype != l.dtype)
        raise(Errc::InconsistentBaseShape, l.base + ": ranks disagree on shape or dtype");
      auto& hs = holders[it->second][l.range];
      if (std::find(hs.begin(), hs.end(), uint32_t(r)) == hs.end()) hs.push_back(uint32_t(r));
    }
  }
  for (uint32_t t = 0; t < p.catalog.tensors.size(); ++t) {
    const Shape& shape = p.catalog.tensors[t].shape;
    std::vector<std::vector<uint64_t>> pts(shape.size());
    for (auto& [rg, _] : holders[t])
      for (int d = 0; d < rg.rank(); ++d) {
        for (uint64_t x : {rg.dim(d).lo, rg.dim(d).hi})
          if (x > 0 && x < shape[size_t(d)]) pts[size_t(d)].push_back(x);
      }
    for (auto& v : pts) std::sort(v.begin(), v.end()), v.erase(std::unique(v.begin(), v.end()), v.end());
    SplitGrid g(std::move(pts));
    std::vector<Range> cells = g.cells(shape);
    std::vector<uint32_t> phi(cells.size(), UINT32_MAX);
    for (auto& [rg, hs] : holders[t]) {
      auto it = std::find(cells.begin(), cells.end(), rg);
      if (it == cells.end())
        raise(Errc::CoverageGap, p.catalog.tensors[t].path + ": " + rg.to_string() + " is not a cell of the grid its ranges span");
      const size_t c = size_t(it - cells.begin());
      phi[c] = uint32_t(p.alpha.size());
      p.alpha.push_back(hs);
    }
    for (auto x : phi)
      if (x == UINT32_MAX) raise(Errc::CoverageGap, p.catalog.tensors[t].path + ": declared ranges leave a gap");
    p.sigma.push_back(std::move(g));
    p.cells.push_back(std::move(cells));
    p.phi.push_back(std::move(phi));
    p.stage.push_back(0);
  }
  return p;
}

std::string serialize_parallel_config(const PTC& p) {
  std::string out = "[";
  for (uint32_t r = 0; r < p.devices.size(); ++r) {
    Node root;
    for (auto [t, c] : hosted_subtensors(p, p.devices[r])) {
      const TensorSpec& e = p.catalog.tensors[t];
      const Range& rg = p.cells[t][c];
      std::string leaf = "{\"base\": ";
      esc(leaf, e.path);
      leaf += ", \"shape\": [";
      for (size_t d = 0; d < e.shape.size(); ++d) leaf += (d ? ", " : "") + std::to_string(e.shape[d]);
      leaf += "], \"range\": ";
      if (rg == Range::full(e.shape)) {
        leaf += "null";
      } else {
        leaf += '[';
        for (int d = 0; d < rg.rank(); ++d)
          leaf += std::string(d ? ", " : "") + "[" + std::to_string(rg.dim(d).lo) + ", " + std::to_string(rg.dim(d).hi) + "]";
        leaf += ']';
      }
      leaf += ", \"dtype\": \"" + std::string(dtype_name(e.dtype)) + "\"}";
      Node* n = &root;
      for (auto& s : segments(e.path)) n = &n->child(s);
      if (!n->kids.empty() || !n->leaf.empty()) raise(Errc::MalformedConfig, e.path + ": path collides with another tensor");
      n->leaf = leaf;
    }
    if (r) out += ",\n ";
    root.emit(out);
  }
  out += "]\n";
  return out;
}

}  // namespace reshard
