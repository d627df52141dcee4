// PTX1 codec and per-device checkpoints of executor cells (see reshard/checkpoint.hpp).
// Device <-> file traffic is staged through two pinned buffers so the D2H (H2D) of one
// chunk overlaps the write (read) of the previous one.
#include "reshard/checkpoint.hpp"
#include "reshard/trace.hpp"

#include <cuda_runtime.h>

#include <chrono>
#include <exception>
#include <thread>
#include <map>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <set>
#include <tuple>

namespace reshard {

namespace fs = std::filesystem;

namespace {

constexpr uint8_t kMagic[4] = {0x50, 0x54, 0x58, 0x31};  // "PTX1"
constexpr size_t kChunk = 64ull << 20;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// PTX1 has codes 0..3 only.  BF16 payloads are written with the F16 code (same
// width; payloads are opaque bytes) so reference readers accept the files; the
// real dtype is the layout's, which checkpoint_load takes from the catalog, not the file.
uint8_t wire_code(Dtype d) { return d == Dtype::BF16 ? uint8_t(Dtype::F16) : uint8_t(d); }

struct File {
  std::FILE* f = nullptr;
  File(const fs::path& p, const char* mode) : f(std::fopen(p.c_str(), mode)) {
    if (!f) raise(Errc::IoError, "cannot open " + p.string());
  }
  // explicit close for writers: a buffered write that fails at close (ENOSPC) is an error
  void close(const fs::path& p) {
    std::FILE* g = f;
    f = nullptr;
    if (std::fclose(g) != 0) raise(Errc::IoError, "close " + p.string());
  }
  ~File() {
    if (f) std::fclose(f);
  }
};

// <dir>/<rank>/<tensor path>[.c<cell>].ptx.  The cell suffix appears only when
// the rank hosts several cells of the tensor, so the common one-cell layout keeps the plain
// name.  Tensor paths are relative and may not climb out of the rank directory.
fs::path cell_file(const std::string& dir, uint32_t rank, const std::string& tensor, uint32_t cell, bool several) {
  const fs::path rel(tensor);
  if (tensor.empty() || rel.is_absolute() || rel.has_root_name())
    raise(Errc::InvalidArgument, "checkpoint: tensor path '" + tensor + "' is not relative");
  for (const auto& part : rel)
    if (part == "..") raise(Errc::InvalidArgument, "checkpoint: tensor path '" + tensor + "' contains '..'");
  return fs::path(dir) / std::to_string(rank) / (tensor + (several ? ".c" + std::to_string(cell) : std::string()) + ".ptx");
}

// per (device, tensor): how many cells the device hosts
std::map<std::pair<uint32_t, uint32_t>, uint32_t> cells_per_device(const std::vector<std::tuple<uint32_t, uint32_t, uint32_t>>& v) {
  std::map<std::pair<uint32_t, uint32_t>, uint32_t> n;
  for (auto [d, t, c] : v) ++n[{d, t}];
  return n;
}

// Two pinned staging buffers and a stream on the current device.
struct Staging {
  void* buf[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  Staging() {
    ck(cudaHostAlloc(&buf[0], kChunk, cudaHostAllocDefault), "pinned staging");
    ck(cudaHostAlloc(&buf[1], kChunk, cudaHostAllocDefault), "pinned staging");
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming), "event");
  }
  ~Staging() {
    cudaStreamSynchronize(s);
    for (int i = 0; i < 2; ++i) cudaFreeHost(buf[i]), cudaEventDestroy(ev[i]);
    cudaStreamDestroy(s);
  }
};

void write_cell(Staging& st, const fs::path& p, Dtype dt, const Shape& shape, const char* dev, uint64_t bytes) {
  fs::create_directories(p.parent_path());
  File f(p, "wb");
  auto hdr = ptx_encode_header(dt, shape);
  if (std::fwrite(hdr.data(), 1, hdr.size(), f.f) != hdr.size()) raise(Errc::IoError, "write " + p.string());
  const uint64_t n = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](uint64_t i) {
    const uint64_t off = i * kChunk, len = std::min<uint64_t>(kChunk, bytes - off);
    ck(cudaMemcpyAsync(st.buf[i & 1], dev + off, len, cudaMemcpyDeviceToHost, st.s), "d2h");
    ck(cudaEventRecord(st.ev[i & 1], st.s), "event");
  };
  if (n) issue(0);
  for (uint64_t i = 0; i < n; ++i) {
    if (i + 1 < n) issue(i + 1);  // next chunk's D2H overlaps this chunk's write
    ck(cudaEventSynchronize(st.ev[i & 1]), "sync");
    const uint64_t len = std::min<uint64_t>(kChunk, bytes - i * kChunk);
    if (std::fwrite(st.buf[i & 1], 1, len, f.f) != len) raise(Errc::IoError, "write " + p.string());
  }
  f.close(p);
}

void read_cell(Staging& st, const fs::path& p, Dtype dt, const Shape& shape, char* dev, uint64_t bytes) {
  std::error_code ec;
  const auto fsize = fs::file_size(p, ec);
  if (ec) raise(Errc::LayoutMismatch, "missing checkpoint file " + p.string());
  File f(p, "rb");
  std::vector<uint8_t> head(std::min<uintmax_t>(fsize, ptx_header_size(kMaxRank)));
  if (std::fread(head.data(), 1, head.size(), f.f) != head.size()) raise(Errc::IoError, "read " + p.string());
  // validate the header against the file size without reading the payload twice
  if (head.size() < 6 || std::memcmp(head.data(), kMagic, 4) != 0) raise(Errc::InvalidTensor, "bad PTX1 magic in " + p.string());
  const size_t hb = ptx_header_size(head[5]);
  if (head.size() < hb) raise(Errc::InvalidTensor, "truncated PTX1 header in " + p.string());
  head.resize(hb);
  // same checks as ptx_decode_header, with the payload size taken from the file size
  const PtxHeader h = [&] {
    Shape s(head[5]);
    for (size_t d = 0; d < s.size(); ++d) std::memcpy(&s[d], head.data() + 6 + 8 * d, 8);
    if (head[4] > 3) raise(Errc::InvalidTensor, "unknown dtype code in " + p.string());
    for (auto e : s)
      if (e == 0) raise(Errc::InvalidTensor, "zero extent in " + p.string());
    PtxHeader r{static_cast<Dtype>(head[4]), s, hb, shape_elements(s) * dtype_width(static_cast<Dtype>(head[4]))};
    if (hb + r.payload_bytes != fsize) raise(Errc::InvalidTensor, "payload size mismatch in " + p.string());
    return r;
  }();
  if (h.shape != shape || dtype_width(h.dtype) != dtype_width(dt))
    raise(Errc::LayoutMismatch, p.string() + " does not hold this layout's cell");
  if (std::fseek(f.f, long(hb), SEEK_SET) != 0) raise(Errc::IoError, "seek " + p.string());
  const uint64_t n = (bytes + kChunk - 1) / kChunk;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t off = i * kChunk, len = std::min<uint64_t>(kChunk, bytes - off);
    if (i >= 2) ck(cudaEventSynchronize(st.ev[i & 1]), "sync");  // buffer free again
    if (std::fread(st.buf[i & 1], 1, len, f.f) != len) raise(Errc::IoError, "read " + p.string());
    ck(cudaMemcpyAsync(dev + off, st.buf[i & 1], len, cudaMemcpyHostToDevice, st.s), "h2d");
    ck(cudaEventRecord(st.ev[i & 1], st.s), "event");
  }
  ck(cudaStreamSynchronize(st.s), "sync");
}

}  // namespace

size_t ptx_header_size(size_t rank) { return 4 + 1 + 1 + 8 * rank; }
size_t ptx_encoded_size(Dtype d, const Shape& s) { return ptx_header_size(s.size()) + shape_elements(s) * dtype_width(d); }

std::vector<uint8_t> ptx_encode_header(Dtype d, const Shape& s) {
  if (s.size() > 255) raise(Errc::InvalidTensor, "rank above 255");
  std::vector<uint8_t> h(ptx_header_size(s.size()));
  std::memcpy(h.data(), kMagic, 4);
  h[4] = wire_code(d);
  h[5] = uint8_t(s.size());
  for (size_t i = 0; i < s.size(); ++i)
    for (int b = 0; b < 8; ++b) h[6 + 8 * i + size_t(b)] = uint8_t(s[i] >> (8 * b));  // little-endian
  return h;
}

PtxHeader ptx_decode_header(const uint8_t* p, size_t n) {
  if (n < 6 || std::memcmp(p, kMagic, 4) != 0) raise(Errc::InvalidTensor, "bad PTX1 magic");
  if (p[4] > 3) raise(Errc::InvalidTensor, "unknown dtype code " + std::to_string(p[4]));
  const size_t rank = p[5], hb = ptx_header_size(rank);
  if (n < hb) raise(Errc::InvalidTensor, "truncated PTX1 header");
  Shape s(rank);
  for (size_t i = 0; i < rank; ++i) {
    uint64_t v = 0;
    for (int b = 7; b >= 0; --b) v = (v << 8) | p[6 + 8 * i + size_t(b)];
    if (v == 0) raise(Errc::InvalidTensor, "zero extent");
    s[i] = v;
  }
  const Dtype d = static_cast<Dtype>(p[4]);
  const uint64_t payload = shape_elements(s) * dtype_width(d);
  if (n - hb != payload)
    raise(Errc::InvalidTensor, "payload " + std::to_string(n - hb) + " bytes, expected " + std::to_string(payload));
  return PtxHeader{d, s, hb, payload};
}

std::vector<uint8_t> ptx_encode(const Tensor& t) {
  std::vector<uint8_t> out = ptx_encode_header(t.dtype(), t.shape());
  out.insert(out.end(), t.payload().begin(), t.payload().end());
  return out;
}

Tensor ptx_decode(std::span<const uint8_t> bytes) {
  const PtxHeader h = ptx_decode_header(bytes.data(), bytes.size());
  return Tensor(h.dtype, h.shape,
                std::vector<uint8_t>(bytes.begin() + std::ptrdiff_t(h.header_bytes), bytes.end()));
}

size_t ptx_encoded_size(const Tensor& t) { return ptx_encoded_size(t.dtype(), t.shape()); }

void ptx_write_file(const std::string& path, const Tensor& t) {
  const std::vector<uint8_t> b = ptx_encode(t);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) raise(Errc::InvalidArgument, "cannot open " + path + " for writing");
  const size_t w = std::fwrite(b.data(), 1, b.size(), f);
  const bool ok = std::fclose(f) == 0 && w == b.size();
  if (!ok) raise(Errc::InvalidArgument, "short write to " + path);
}

Tensor ptx_read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) raise(Errc::InvalidTensor, "cannot open " + path);
  std::vector<uint8_t> b;
  uint8_t buf[1 << 16];
  for (size_t n; (n = std::fread(buf, 1, sizeof buf, f)) > 0;) b.insert(b.end(), buf, buf + n);
  std::fclose(f);
  return ptx_decode(b);
}

// Cells move through W host threads (RESHARD_IO_THREADS, default min(8, cores)): each worker
// takes the next cell, with its own pinned double buffer and stream per GPU, so file I/O of
// one cell overlaps the D2H / H2D of others (r61: one thread reached 3.3 GB/s save and 6.2
// GB/s load to tmpfs).
struct CellJob {
  int gpu;
  fs::path path;
  Dtype dtype;
  Shape shape;
  char* dev;
  uint64_t bytes;
};
template <class Fn>
void run_cell_jobs(Context& ctx, const std::vector<CellJob>& jobs, Fn&& fn) {
  const char* v = std::getenv("RESHARD_IO_THREADS");
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  uint64_t total = 0;
  for (const CellJob& j : jobs) total += j.bytes;
  // one worker per ~1 GiB (each pins 2 staging buffers): small checkpoints stay single-threaded
  const size_t by_size = size_t(std::max<uint64_t>(1, total >> 30));
  const size_t workers = std::max<size_t>(
      1, std::min<size_t>({jobs.size(), by_size, v && *v ? size_t(std::atoi(v)) : std::min<size_t>(8, hw)}));
  std::atomic<size_t> next{0};
  std::vector<std::exception_ptr> err(workers);
  auto work = [&](size_t w) {
    try {
      std::map<int, std::unique_ptr<Staging>> st;  // per GPU
      for (size_t i; (i = next.fetch_add(1)) < jobs.size();) {
        const CellJob& j = jobs[i];
        auto& s = st[j.gpu];
        if (!s) {
          ck(cudaSetDevice(ctx.cuda_device(j.gpu)), "cudaSetDevice");
          s = std::make_unique<Staging>();
        }
        ck(cudaSetDevice(ctx.cuda_device(j.gpu)), "cudaSetDevice");
        fn(*s, j);
      }
    } catch (...) {
      err[w] = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  for (size_t w = 1; w < workers; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

IoStats checkpoint_save(Executor& ex, int side, const std::string& dir) {
  TraceRange trace_("checkpoint_save");
  const auto t0 = std::chrono::steady_clock::now();
  const ReconfigPlan& plan = ex.plan();
  Context& ctx = ex.context();
  IoStats io;
  std::vector<CellJob> jobs;
  std::set<fs::path> dirs;
  // (device, tensor, cell) and binding of every cell on this side, in layout order
  std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> cells;
  std::vector<const CellBinding*> binds;
  const PTC& ptc = side == 0 ? *plan.from : *plan.to;
  if (side == 0) {
    size_t k = 0;
    for (uint32_t i = 0; i < ptc.devices.size(); ++i)
      for (auto [t, c] : hosted_subtensors(ptc, ptc.devices[i])) cells.emplace_back(i, t, c), binds.push_back(&ex.src_bindings()[k++]);
  } else {
    for (size_t j = 0; j < plan.dst_cells.size(); ++j) {
      const PlanDstCell& dc = plan.dst_cells[j];
      cells.emplace_back(dc.dst_device, dc.tensor, dc.cell), binds.push_back(&ex.dst_bindings()[j]);
    }
  }
  const auto per = cells_per_device(cells);
  for (size_t k = 0; k < cells.size(); ++k) {
    const auto [dev, t, c] = cells[k];
    const CellBinding& b = *binds[k];
    const TensorSpec& e = ptc.catalog.tensors[t];
    const fs::path p = cell_file(dir, dev, e.path, c, per.at({dev, t}) > 1);  // validates every path
    if (b.gpu < 0 || ctx.local_of(b.gpu) < 0) continue;
    char* base = static_cast<char*>(ex.arena_base(b.gpu, b.arena));
    if (!base) raise(Errc::InvalidArgument, "checkpoint_save: arena not bound");
    dirs.insert(p.parent_path());
    jobs.push_back(CellJob{b.gpu, p, e.dtype, ptc.cells[t][c].extents(), base + b.offset, b.bytes});
    io.files += 1, io.bytes += b.bytes;
  }
  for (const fs::path& d : dirs) fs::create_directories(d);  // before the workers: no creation races
  run_cell_jobs(ctx, jobs, [](Staging& st, const CellJob& j) { write_cell(st, j.path, j.dtype, j.shape, j.dev, j.bytes); });
  io.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return io;
}

IoStats checkpoint_load(Executor& ex, const std::string& dir) {
  TraceRange trace_("checkpoint_load");
  const auto t0 = std::chrono::steady_clock::now();
  const PTC& a = *ex.plan().from;
  Context& ctx = ex.context();
  // the directory must hold exactly this layout's ranks
  std::set<std::string> ranks;
  std::error_code ec;
  for (auto& entry : fs::directory_iterator(dir, ec))
    if (entry.is_directory()) ranks.insert(entry.path().filename().string());
  if (ec) raise(Errc::IoError, "cannot list " + dir);
  std::set<std::string> want;
  for (size_t i = 0; i < a.devices.size(); ++i) want.insert(std::to_string(i));
  if (ranks != want)
    raise(Errc::LayoutMismatch, "checkpoint has " + std::to_string(ranks.size()) + " ranks, layout has " +
                                    std::to_string(want.size()));
  IoStats io;
  std::vector<CellJob> jobs;
  std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> cells;
  for (uint32_t i = 0; i < a.devices.size(); ++i)
    for (auto [t, c] : hosted_subtensors(a, a.devices[i])) cells.emplace_back(i, t, c);
  const auto per = cells_per_device(cells);
  for (size_t k = 0; k < cells.size(); ++k) {
    const auto [i, t, c] = cells[k];
    const CellBinding& b = ex.src_bindings()[k];
    const TensorSpec& e = a.catalog.tensors[t];
    fs::path p = cell_file(dir, i, e.path, c, per.at({i, t}) > 1);
    if (b.gpu < 0 || ctx.local_of(b.gpu) < 0) continue;
    char* base = static_cast<char*>(ex.arena_base(b.gpu, 0));
    if (!base) raise(Errc::InvalidArgument, "checkpoint_load: arena not bound");
    jobs.push_back(CellJob{b.gpu, std::move(p), e.dtype, a.cells[t][c].extents(), base + b.offset, b.bytes});
    io.files += 1, io.bytes += b.bytes;
  }
  run_cell_jobs(ctx, jobs, [](Staging& st, const CellJob& j) { read_cell(st, j.path, j.dtype, j.shape, j.dev, j.bytes); });
  io.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return io;
}

}  // namespace reshard
