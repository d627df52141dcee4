// reshard/checkpoint.hpp — the PTX1 tensor container (declared by the reference,
// proj/include/reshard/tensor/ptx_io.hpp:10-20, format SPEC.md:104; the reference ships no
// implementation) and the per-device checkpoint of an executor's cells
// (checkpoint_roundtrip): `<dir>/<rank>/<tensor path>.ptx`.
//
// PTX1: magic "PTX1" (50 54 58 31), u8 dtype code, u8 rank, rank x u64-LE extents, raw
// payload; no padding, no checksum.  BF16 payloads are written with the F16 code (2-byte
// opaque elements) so reference readers (dtype_from_code rejects codes > 3) accept them.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "reshard/executor.hpp"
#include "reshard/tensor.hpp"

namespace reshard {

size_t ptx_header_size(size_t rank);
size_t ptx_encoded_size(Dtype d, const Shape& s);
// Header bytes for a tensor of dtype/shape (payload follows).
std::vector<uint8_t> ptx_encode_header(Dtype d, const Shape& s);
struct PtxHeader {
  Dtype dtype;
  Shape shape;
  size_t header_bytes;
  uint64_t payload_bytes;
};
// Parses and validates a PTX1 buffer of `n` bytes (header + payload): InvalidTensor on a
// bad magic, truncated header, unknown dtype code, zero extent or payload size mismatch.
PtxHeader ptx_decode_header(const uint8_t* bytes, size_t n);

// The reference's value-level PTX1 functions, same signatures as ptx_io.hpp:13-20.
std::vector<uint8_t> ptx_encode(const Tensor& t);
Tensor ptx_decode(std::span<const uint8_t> bytes);  // InvalidTensor
void ptx_write_file(const std::string& path, const Tensor& t);
Tensor ptx_read_file(const std::string& path);      // InvalidTensor on a bad file
size_t ptx_encoded_size(const Tensor& t);

struct IoStats {
  uint64_t files = 0, bytes = 0;
  double seconds = 0;
};
// Save the cells of one layout from the executor's arenas: side 0 = `from` (src arena),
// side 1 = `to` (dst bindings, kept cells read from the src arena).  Only cells on GPUs
// this process drives.
IoStats checkpoint_save(Executor& ex, int side, const std::string& dir);
// Load the `from` layout's cells from `dir` into the src arena.  LayoutMismatch when the
// directory's rank set or a file's shape/width does not match the layout.
IoStats checkpoint_load(Executor& ex, const std::string& dir);

}  // namespace reshard
