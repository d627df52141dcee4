// examples/tensor_values.cpp — a translation unit written against the reference's own headers
// (the include paths of proj/include/reshard/...: error.hpp, tensor/{dtype,range,split_grid,
// tensor,ptx_io}.hpp, util/hash.hpp) compiled unchanged against this library: Tensor, slice,
// merge, SplitGrid, grid_refine, Range, PTX1, FNV-1a, splitmix64.  The validation errors and
// the host-only calls need no GPU; slice / merge move their bytes on the GPU.
//
//   g++ -std=c++20 -I paper_2312_05181_b200/csrc examples/tensor_values.cpp \
//       -L paper_2312_05181_b200 -lreshard_b200 -Wl,-rpath,$PWD/paper_2312_05181_b200 -o tensor_values
#include <cstdio>
#include <cstring>

#include "reshard/error.hpp"
#include "reshard/tensor/dtype.hpp"
#include "reshard/tensor/ptx_io.hpp"
#include "reshard/tensor/range.hpp"
#include "reshard/tensor/split_grid.hpp"
#include "reshard/tensor/tensor.hpp"
#include "reshard/util/hash.hpp"

using namespace reshard;

static Tensor iota_f32(Shape shape) {
  std::vector<uint8_t> p(shape_elements(shape) * 4);
  for (uint64_t i = 0; i < shape_elements(shape); ++i) {
    const float v = float(i);
    std::memcpy(p.data() + 4 * i, &v, 4);
  }
  return Tensor(Dtype::F32, std::move(shape), std::move(p));
}

template <class F>
static void expect_error(const char* what, Errc want, F&& f) {
  try {
    f();
    std::printf("%s: no error\n", what);
  } catch (const Error& e) {
    std::printf("%s: %s\n", what, errc_name(e.code()));
    if (e.code() != want) std::exit(3);
  }
}

int main() {
  try {
    // validation, in the reference's order, before any device work
    expect_error("zero extent", Errc::InvalidTensor, [] { Tensor(Dtype::F32, {0}, {}); });
    expect_error("payload size", Errc::InvalidTensor, [] { Tensor(Dtype::F32, {2}, std::vector<uint8_t>(4)); });
    const Tensor t = iota_f32({4, 6});
    expect_error("slice out of bounds", Errc::RangeOutOfBounds, [&] { slice(t, Range::parse("[0:5,0:6]")); });
    expect_error("merge gap", Errc::TilingGap,
                 [&] { merge({{Range::parse("[0:3]"), iota_f32({3})}}, Shape{6}); });
    expect_error("merge overlap", Errc::TilingOverlap, [&] {
      merge({{Range::parse("[0:4]"), iota_f32({4})}, {Range::parse("[2:6]"), iota_f32({4})}}, Shape{6});
    });
    // SURVEY §4 KATs: grid_refine({3}, {2,4}) on [6]; the first splitmix64 output from state 0
    const SplitGrid g = grid_refine(SplitGrid({{3}}), SplitGrid({{2, 4}}));
    std::printf("refine:");
    for (const Range& c : g.cells(Shape{6})) std::printf("%s", c.to_string().c_str());
    std::printf(" splitmix64(0) %016llx dtype %s\n", (unsigned long long)SplitMix64(0).next(),
                dtype_name(dtype_from_code(uint8_t(0))));
    // the per-base-tensor digest the SPEC verifies against (hash.hpp:42)
    std::printf("digest %016llx\n", (unsigned long long)fnv1a64(t.bytes()));
    // PTX1 container: header 6 + 8 x rank bytes, then the payload
    const std::vector<uint8_t> enc = ptx_encode(t);
    std::printf("ptx round trip: %s (%zu bytes, encoded_size %zu)\n", ptx_decode(enc) == t ? "equal" : "DIFFERENT",
                enc.size(), ptx_encoded_size(t));
    // data: SPEC.md:60-62 and the quadrant round trip
    const Tensor s = slice(t, Range::parse("[0:4,2:4]"));
    std::printf("slice [0:4,2:4]:");
    for (uint64_t i = 0; i < s.elements(); ++i) {
      float v;
      std::memcpy(&v, s.payload().data() + 4 * i, 4);
      std::printf(" %g", v);
    }
    std::printf("\n");
    std::vector<std::pair<Range, Tensor>> quads;
    for (const char* q : {"[0:2,0:3]", "[0:2,3:6]", "[2:4,0:3]", "[2:4,3:6]"}) {
      const Range r = Range::parse(q);
      quads.emplace_back(r, slice(t, r));
    }
    std::printf("quadrant round trip: %s\n", merge(quads, t.shape()) == t ? "equal" : "DIFFERENT");
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1 + int(e.code());
  }
}
