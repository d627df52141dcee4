// extern "C" boundary (include/reshard_b200.h).  Every entry point catches reshard::Error
// and maps it to 1 + Errc; no exception crosses the boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/reshard_b200.h"
#include "reshard/checkpoint.hpp"
#include "reshard/config.hpp"
#include "reshard/dataset.hpp"
#include "reshard/executor.hpp"
#include "reshard/tensor.hpp"

using namespace reshard;

struct rs_context {
  std::unique_ptr<Context> ctx;
};
struct rs_catalog {
  Catalog c;
};
struct rs_ptc {
  std::shared_ptr<const PTC> p;
};
struct rs_plan {
  std::shared_ptr<const ReconfigPlan> p;
};
struct rs_executor {
  std::unique_ptr<Executor> e;
};

namespace {

thread_local std::string g_last;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::bad_alloc&) {
    g_last = "InvalidArgument: host allocation failed";
    return 1 + static_cast<int>(Errc::InvalidArgument);
  } catch (const std::exception& e) {
    g_last = std::string("InvalidArgument: ") + e.what();
    return 1 + static_cast<int>(Errc::InvalidArgument);
  }
}

void need(const void* p, const char* what) {
  if (!p) raise(Errc::InvalidArgument, std::string("null ") + what);
}
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

Range to_range(const rs_range& r) {
  if (r.rank < 0 || r.rank > RS_MAX_RANK) raise(Errc::RankMismatch, "rank out of [0, 8]");
  std::vector<Interval> v;
  for (int i = 0; i < r.rank; ++i) v.push_back({r.lo[i], r.hi[i]});
  return Range(v);
}
rs_range from_range(const Range& r) {
  rs_range o{};
  o.rank = r.rank();
  for (int i = 0; i < r.rank(); ++i) o.lo[i] = r.dim(i).lo, o.hi[i] = r.dim(i).hi;
  return o;
}
Shape to_shape(int rank, const uint64_t* s) {
  if (rank < 0 || rank > RS_MAX_RANK) raise(Errc::RankMismatch, "rank out of [0, 8]");
  if (rank) need(s, "shape");
  return Shape(s, s + rank);
}
SplitGrid to_grid(int rank, const int32_t* npts, const uint64_t* pts) {
  if (rank < 0 || rank > RS_MAX_RANK) raise(Errc::RankMismatch, "rank out of [0, 8]");
  std::vector<std::vector<uint64_t>> g(static_cast<size_t>(rank));
  if (rank) need(npts, "split point counts");
  size_t k = 0;
  for (int d = 0; d < rank; ++d) {
    if (npts[d] < 0) raise(Errc::InvalidArgument, "negative split point count");
    if (npts[d]) need(pts, "split points");
    for (int i = 0; i < npts[d]; ++i) g[size_t(d)].push_back(pts[k++]);
  }
  return SplitGrid(std::move(g));
}
void from_grid(const SplitGrid& g, int32_t* npts, uint64_t* pts) {
  if (g.rank()) need(npts, "split point count output");
  size_t total = 0;
  for (size_t d = 0; d < g.rank(); ++d) total += g.points()[d].size();
  if (total) need(pts, "split point output");
  size_t k = 0;
  for (size_t d = 0; d < g.rank(); ++d) {
    npts[d] = int32_t(g.points()[d].size());
    for (auto p : g.points()[d]) pts[k++] = p;
  }
}
DeviceId to_dev(const rs_device& d) { return DeviceId{d.worker, d.local}; }
DeviceTensorView to_view(const rs_tensor& t) {
  return DeviceTensorView{dtype_from_code(t.dtype), to_shape(t.rank, t.shape), t.data};
}
Context& ctx_of(rs_context* c) {
  need(c, "context");
  return *c->ctx;
}

}  // namespace

extern "C" {

const char* rs_last_error(void) { return g_last.c_str(); }
const char* rs_errc_name(int c) { return errc_name(static_cast<Errc>(c)); }
int rs_errc_count(void) { return kErrcCount; }
uint64_t rs_fnv1a64(const void* data, uint64_t n) { return fnv1a64(data, n); }
uint64_t rs_payload_seed(const char* path) { return payload_seed(path ? path : ""); }
const char* rs_build_info(void) {
  return "reshard_b200 sm_100a (K3 TMA bulk copy with fan-out, K3T TMA tensor-map boxes, K1/K2 LDG/STG copy with "
         "read-once fan-out to peers, K5 repartition, K8 shuffle, K6/K7 payload); CUDA " RESHARD_CUDA_VERSION;
}

// ---- box algebra ------------------------------------------------------------------------
int rs_range_parse(const char* text, rs_range* out) {
  return guard([&] {
    need(text, "text"), need(out, "out");
    *out = from_range(Range::parse(text));
  });
}
int rs_range_format(const rs_range* r, char* buf, uint64_t cap) {
  return guard([&] {
    need(r, "range"), need(buf, "buf");
    std::string s = to_range(*r).to_string();
    if (s.size() + 1 > cap) raise(Errc::InvalidArgument, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}
int rs_grid_cells(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts, int cap, rs_range* cells,
                  int* n) {
  return guard([&] {
    need(n, "n");
    if (cap > 0) need(cells, "cells");
    auto v = to_grid(rank, npts, pts).cells(to_shape(rank, shape));
    *n = int(v.size());
    for (int i = 0; i < int(v.size()) && i < cap; ++i) cells[i] = from_range(v[size_t(i)]);
  });
}
int rs_grid_refine(int ra, const int32_t* na, const uint64_t* pa, int rb, const int32_t* nb, const uint64_t* pb,
                   int32_t* nout, uint64_t* pout) {
  return guard([&] { from_grid(grid_refine(to_grid(ra, na, pa), to_grid(rb, nb, pb)), nout, pout); });
}
int rs_even_split(int rank, const uint64_t* shape, int dim, uint64_t ways, int32_t* nout, uint64_t* pout) {
  return guard([&] {
    if (dim < 0) raise(Errc::RankMismatch, "negative split dim");
    from_grid(SplitGrid::even_split(to_shape(rank, shape), size_t(dim), ways), nout, pout);
  });
}
int rs_grid_cell(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts, uint64_t index,
                 rs_range* out) {
  return guard([&] {
    need(out, "out");
    *out = from_range(to_grid(rank, npts, pts).cell(to_shape(rank, shape), index));
  });
}
int rs_grid_cell_index_of(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts,
                          const rs_range* r, uint64_t* index) {
  return guard([&] {
    need(r, "range"), need(index, "index");
    *index = to_grid(rank, npts, pts).cell_index_of(to_shape(rank, shape), to_range(*r));
  });
}
int rs_range_offset_by(const rs_range* r, const rs_range* outer, rs_range* out) {
  return guard([&] {
    need(r, "range"), need(outer, "outer"), need(out, "out");
    *out = from_range(to_range(*r).offset_by(to_range(*outer)));
  });
}
int rs_range_valid_for(const rs_range* r, int rank, const uint64_t* shape, int32_t* ok) {
  return guard([&] {
    need(r, "range"), need(ok, "ok");
    *ok = to_range(*r).valid_for(to_shape(rank, shape)) ? 1 : 0;
  });
}
int rs_rangespec_resolve(const char* spec, int rank, const uint64_t* shape, rs_range* out) {
  return guard([&] {
    need(spec, "spec"), need(out, "out");
    *out = from_range(RangeSpec::parse(spec).resolve(to_shape(rank, shape)));
  });
}
int rs_dtype_from_name(const char* name, int32_t* code) {
  return guard([&] {
    need(name, "name"), need(code, "code");
    *code = int32_t(dtype_from_name(name));
  });
}

// ---- device runtime ------------------------------------------------------------------------
int rs_device_count(int* n) {
  return guard([&] {
    need(n, "n");
    *n = 0;
    if (cudaGetDeviceCount(n) != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
  });
}
int rs_init(int world, int n_local, const int32_t* world_ids, const int32_t* cuda_devices, rs_context** out) {
  return guard([&] {
    need(out, "out");
    if (n_local > 0) need(world_ids, "world_ids"), need(cuda_devices, "cuda_devices");
    auto c = std::make_unique<rs_context>();
    c->ctx = std::make_unique<Context>(world, std::vector<int>(world_ids, world_ids + n_local),
                                       std::vector<int>(cuda_devices, cuda_devices + n_local));
    *out = c.release();
  });
}
void rs_destroy(rs_context* c) { delete c; }

int rs_malloc(rs_context* c, int gpu, uint64_t bytes, void** out) {
  return guard([&] {
    need(out, "out");
    cuda_ok(cudaSetDevice(ctx_of(c).cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaMalloc(out, bytes ? bytes : 256), "cudaMalloc");
  });
}
int rs_free(rs_context* c, int gpu, void* p) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx_of(c).cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaFree(p), "cudaFree");
  });
}
int rs_host_alloc(uint64_t bytes, void** out) {
  return guard([&] { cuda_ok(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable), "cudaHostAlloc"); });
}
int rs_host_free(void* p) {
  return guard([&] { cuda_ok(cudaFreeHost(p), "cudaFreeHost"); });
}
static int copy_impl(rs_context* c, int gpu, void* dst, const void* src, uint64_t n, cudaMemcpyKind kind) {
  return guard([&] {
    Context& x = ctx_of(c);
    cuda_ok(cudaSetDevice(x.cuda_device(gpu)), "cudaSetDevice");
    auto s = static_cast<cudaStream_t>(x.stream(gpu));
    cuda_ok(cudaMemcpyAsync(dst, src, n, kind, s), "cudaMemcpyAsync");
    cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}
int rs_memcpy_htod(rs_context* c, int gpu, void* dst, const void* src, uint64_t n) {
  return copy_impl(c, gpu, dst, src, n, cudaMemcpyHostToDevice);
}
int rs_memcpy_dtoh(rs_context* c, int gpu, void* dst, const void* src, uint64_t n) {
  return copy_impl(c, gpu, dst, src, n, cudaMemcpyDeviceToHost);
}
int rs_memset(rs_context* c, int gpu, void* dst, int value, uint64_t n) {
  return guard([&] {
    Context& x = ctx_of(c);
    cuda_ok(cudaSetDevice(x.cuda_device(gpu)), "cudaSetDevice");
    auto s = static_cast<cudaStream_t>(x.stream(gpu));
    cuda_ok(cudaMemsetAsync(dst, value, n, s), "cudaMemsetAsync");
    cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}
int rs_sync(rs_context* c, int gpu) {
  return guard([&] {
    Context& x = ctx_of(c);
    cuda_ok(cudaSetDevice(x.cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(x.stream(gpu))), "cudaStreamSynchronize");
  });
}
int rs_ipc_get_handle(rs_context* c, int gpu, void* ptr, void* h64) {
  return guard([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    cuda_ok(cudaSetDevice(ctx_of(c).cuda_device(gpu)), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    cuda_ok(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
    std::memcpy(h64, &h, 64);
  });
}
int rs_ipc_open_handle(rs_context* c, int gpu, const void* h64, void** out) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx_of(c).cuda_device(gpu)), "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h64, 64);
    cuda_ok(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}
int rs_ipc_close_handle(rs_context* c, int gpu, void* ptr) {
  return guard([&] {
    cuda_ok(cudaSetDevice(ctx_of(c).cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
  });
}

// ---- cross-process stream events and stream timers (one process per GPU) -----------------------
struct rs_event {
  cudaEvent_t e = nullptr;
  int dev = -1;
  bool timing = false;
  ~rs_event() {
    if (e) {
      cudaSetDevice(dev);
      cudaEventDestroy(e);
    }
  }
};
int rs_ipc_event_create(rs_context* c, int gpu, void* h64, rs_event** out) {
  return guard([&] {
    need(h64, "handle"), need(out, "out");
    static_assert(sizeof(cudaIpcEventHandle_t) == 64, "ipc event handle size");
    auto ev = std::make_unique<rs_event>();
    ev->dev = ctx_of(c).cuda_device(gpu);
    cuda_ok(cudaSetDevice(ev->dev), "cudaSetDevice");
    cuda_ok(cudaEventCreateWithFlags(&ev->e, cudaEventInterprocess | cudaEventDisableTiming), "cudaEventCreate");
    cudaIpcEventHandle_t h;
    cuda_ok(cudaIpcGetEventHandle(&h, ev->e), "cudaIpcGetEventHandle");
    std::memcpy(h64, &h, 64);
    *out = ev.release();
  });
}
int rs_ipc_event_open(rs_context* c, int gpu, const void* h64, rs_event** out) {
  return guard([&] {
    need(h64, "handle"), need(out, "out");
    auto ev = std::make_unique<rs_event>();
    ev->dev = ctx_of(c).cuda_device(gpu);
    cuda_ok(cudaSetDevice(ev->dev), "cudaSetDevice");
    cudaIpcEventHandle_t h;
    std::memcpy(&h, h64, 64);
    cuda_ok(cudaIpcOpenEventHandle(&ev->e, h), "cudaIpcOpenEventHandle");
    *out = ev.release();
  });
}
int rs_timing_event_create(rs_context* c, int gpu, rs_event** out) {
  return guard([&] {
    need(out, "out");
    auto ev = std::make_unique<rs_event>();
    ev->dev = ctx_of(c).cuda_device(gpu), ev->timing = true;
    cuda_ok(cudaSetDevice(ev->dev), "cudaSetDevice");
    cuda_ok(cudaEventCreate(&ev->e), "cudaEventCreate");
    *out = ev.release();
  });
}
int rs_event_record(rs_context* c, int gpu, rs_event* ev) {
  return guard([&] {
    need(ev, "event");
    Context& x = ctx_of(c);
    cuda_ok(cudaSetDevice(x.cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaEventRecord(ev->e, static_cast<cudaStream_t>(x.stream(gpu))), "cudaEventRecord");
  });
}
int rs_event_wait(rs_context* c, int gpu, rs_event* ev) {
  return guard([&] {
    need(ev, "event");
    Context& x = ctx_of(c);
    cuda_ok(cudaSetDevice(x.cuda_device(gpu)), "cudaSetDevice");
    cuda_ok(cudaStreamWaitEvent(static_cast<cudaStream_t>(x.stream(gpu)), ev->e, 0), "cudaStreamWaitEvent");
  });
}
int rs_event_elapsed(rs_event* a, rs_event* b, float* ms) {
  return guard([&] {
    need(a, "event"), need(b, "event"), need(ms, "ms");
    if (!a->timing || !b->timing) raise(reshard::Errc::InvalidArgument, "elapsed time needs two timing events");
    cuda_ok(cudaSetDevice(b->dev), "cudaSetDevice");
    cuda_ok(cudaEventSynchronize(b->e), "cudaEventSynchronize");
    cuda_ok(cudaEventElapsedTime(ms, a->e, b->e), "cudaEventElapsedTime");
  });
}
void rs_event_destroy(rs_event* ev) { delete ev; }

// ---- tensor core on device ----------------------------------------------------------------
int rs_slice(rs_context* c, int gpu, const rs_tensor* t, const rs_range* r, void* out) {
  return guard([&] {
    need(t, "tensor"), need(r, "range");
    device_slice(ctx_of(c), gpu, to_view(*t), to_range(*r), out);
  });
}
int rs_merge(rs_context* c, int gpu, int n, const rs_range* ranges, const rs_tensor* parts, int rank,
             const uint64_t* target, void* out) {
  return guard([&] {
    std::vector<std::pair<Range, DeviceTensorView>> v;
    for (int i = 0; i < n; ++i) v.emplace_back(to_range(ranges[i]), to_view(parts[i]));
    device_merge(ctx_of(c), gpu, v, to_shape(rank, target), out);
  });
}

int rs_broadcast(rs_context* c, int gpu, const void* src, int n_dst, void* const* dsts, uint64_t bytes, rs_timing* timing) {
  return guard([&] {
    if (n_dst < 0 || (n_dst > 0 && !dsts)) raise(Errc::InvalidArgument, "broadcast: bad destination list");
    std::vector<void*> d(dsts, dsts + n_dst);
    Timing t = broadcast(ctx_of(c), gpu, src, d, bytes);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_slice_host(rs_context* c, int gpu, const rs_tensor* t, const rs_range* r, void* out) {
  return guard([&] {
    need(t, "tensor"), need(r, "range");
    const DeviceTensorView v = to_view(*t);
    host_slice(ctx_of(c), gpu, HostTensorView{v.dtype, v.shape, v.data}, to_range(*r), out);
  });
}
int rs_merge_host(rs_context* c, int gpu, int n, const rs_range* ranges, const rs_tensor* parts, int rank,
                  const uint64_t* target, void* out) {
  return guard([&] {
    std::vector<std::pair<Range, HostTensorView>> v;
    for (int i = 0; i < n; ++i) {
      const DeviceTensorView d = to_view(parts[i]);
      v.emplace_back(to_range(ranges[i]), HostTensorView{d.dtype, d.shape, d.data});
    }
    host_merge(ctx_of(c), gpu, v, to_shape(rank, target), out);
  });
}

// ---- collection description ----------------------------------------------------------------
int rs_catalog_create(rs_catalog** out) {
  return guard([&] { *out = new rs_catalog(); });
}
int rs_catalog_gpt(uint64_t h, uint64_t L, uint64_t S, uint64_t V, int kind, rs_catalog** out) {
  return guard([&] {
    if (kind < 0 || kind > 2) raise(Errc::MalformedConfig, "unknown state kind");
    if (h == 0 || S == 0 || V == 0) raise(Errc::InvalidTensor, "zero model dimension");
    *out = new rs_catalog{Catalog::gpt(h, L, S, V, static_cast<StateKind>(kind))};
  });
}
int rs_catalog_add(rs_catalog* c, const char* path, int dtype, int rank, const uint64_t* shape, int tp_dim, int layer) {
  return guard([&] {
    need(c, "catalog"), need(path, "path");
    if (!*path) raise(Errc::MalformedConfig, "empty tensor path");
    c->c.add(TensorSpec{path, dtype_from_code(dtype), to_shape(rank, shape), tp_dim, layer});
  });
}
int rs_catalog_size(const rs_catalog* c) { return c ? int(c->c.tensors.size()) : 0; }
int rs_catalog_get(const rs_catalog* c, int i, char* path, int cap, int32_t* dtype, int32_t* rank, uint64_t* shape,
                   int32_t* tp_dim, int32_t* layer) {
  return guard([&] {
    need(c, "catalog");
    if (i < 0 || size_t(i) >= c->c.tensors.size()) raise(Errc::IndexOutOfRange, "catalog index");
    const TensorSpec& t = c->c.tensors[size_t(i)];
    if (path && cap > 0) std::snprintf(path, size_t(cap), "%s", t.path.c_str());
    *dtype = int32_t(t.dtype), *rank = int32_t(t.shape.size()), *tp_dim = t.tp_dim, *layer = t.layer;
    for (size_t d = 0; d < t.shape.size(); ++d) shape[d] = t.shape[d];
  });
}
uint64_t rs_catalog_bytes(const rs_catalog* c) { return c ? c->c.total_bytes() : 0; }
void rs_catalog_destroy(rs_catalog* c) { delete c; }

int rs_build_strategy(const rs_catalog* c, int n, const rs_device* devs, int tp, int pp, int dp, rs_ptc** out) {
  return guard([&] {
    need(c, "catalog"), need(out, "out");
    std::vector<DeviceId> d;
    for (int i = 0; i < n; ++i) d.push_back(to_dev(devs[i]));
    *out = new rs_ptc{std::make_shared<const PTC>(build_strategy(c->c, d, JobConfig{tp, pp, dp}))};
  });
}
void rs_ptc_destroy(rs_ptc* p) { delete p; }
int rs_ptc_set_alpha(rs_ptc* p, int part, int n, const rs_device* devs) {
  return guard([&] {
    need(p, "ptc");
    auto q = std::make_shared<PTC>(*p->p);
    if (part < 0 || size_t(part) >= q->alpha.size()) raise(Errc::IndexOutOfRange, "partition");
    q->alpha[size_t(part)].clear();
    for (int i = 0; i < n; ++i) {
      int o = q->ordinal(to_dev(devs[i]));
      q->alpha[size_t(part)].push_back(o < 0 ? uint32_t(q->devices.size() + size_t(i)) : uint32_t(o));
    }
    p->p = q;
  });
}
int rs_ptc_set_sigma(rs_ptc* p, int t, int rank, const int32_t* npts, const uint64_t* pts) {
  return guard([&] {
    need(p, "ptc");
    auto q = std::make_shared<PTC>(*p->p);
    if (t < 0 || size_t(t) >= q->sigma.size()) raise(Errc::IndexOutOfRange, "tensor");
    q->sigma[size_t(t)] = to_grid(rank, npts, pts);
    p->p = q;
  });
}
int rs_validate(const rs_ptc* p, char* buf, uint64_t cap, int* n) {
  return guard([&] {
    need(p, "ptc");
    auto v = validate(*p->p);
    std::string s;
    for (auto& x : v) s += x + "\n";
    if (buf && cap) std::snprintf(buf, size_t(cap), "%s", s.c_str());
    *n = int(v.size());
  });
}
int rs_hosted_subtensors(const rs_ptc* p, rs_device dev, int cap, int32_t* tensor, rs_range* cells, int* n) {
  return guard([&] {
    need(p, "ptc");
    auto h = hosted_subtensors(*p->p, to_dev(dev));
    *n = int(h.size());
    for (int i = 0; i < int(h.size()) && i < cap; ++i) {
      tensor[i] = int32_t(h[size_t(i)].first);
      cells[i] = from_range(p->p->cells[h[size_t(i)].first][h[size_t(i)].second]);
    }
  });
}
int rs_ptc_devices(const rs_ptc* p, int cap, rs_device* out, int* n) {
  return guard([&] {
    need(p, "ptc");
    *n = int(p->p->devices.size());
    for (int i = 0; i < *n && i < cap; ++i) out[i] = rs_device{p->p->devices[size_t(i)].worker, p->p->devices[size_t(i)].local};
  });
}

int rs_ptc_cell(const rs_ptc* p, int t, int c, rs_range* out) {
  return guard([&] {
    need(p, "ptc"), need(out, "out");
    const auto& cells = p->p->cells;
    if (t < 0 || size_t(t) >= cells.size() || c < 0 || size_t(c) >= cells[size_t(t)].size())
      raise(Errc::IndexOutOfRange, "tensor/cell index");
    *out = from_range(cells[size_t(t)][size_t(c)]);
  });
}
int rs_ptc_cell_count(const rs_ptc* p, int t, int* n) {
  return guard([&] {
    need(p, "ptc"), need(n, "out");
    if (t < 0 || size_t(t) >= p->p->cells.size()) raise(Errc::IndexOutOfRange, "tensor index");
    *n = int(p->p->cells[size_t(t)].size());
  });
}

// ---- planner ------------------------------------------------------------------------------
int rs_generate_plan(const rs_ptc* a, const rs_ptc* b, rs_plan** out) {
  return guard([&] {
    need(a, "from"), need(b, "to"), need(out, "out");
    *out = new rs_plan{generate_plan(a->p, b->p)};
  });
}
int rs_recover(const rs_ptc* a, int nf, const rs_device* failed, const rs_ptc* b, rs_plan** out) {
  return guard([&] {
    need(a, "from"), need(b, "to"), need(out, "out");
    std::vector<DeviceId> f;
    for (int i = 0; i < nf; ++i) f.push_back(to_dev(failed[i]));
    *out = new rs_plan{recover(a->p, f, b->p)};
  });
}
void rs_plan_destroy(rs_plan* p) { delete p; }
int rs_plan_get_stats(const rs_plan* p, rs_plan_stats* out) {
  return guard([&] {
    need(p, "plan"), need(out, "out");
    PlanStats s = plan_stats(*p->p);
    *out = rs_plan_stats{s.n_split, s.n_move, s.n_merge, s.moved_bytes, s.relayout_bytes, s.kept_bytes, s.dst_bytes};
  });
}
int rs_plan_cost(const rs_plan* p, int cap, rs_device* devs, uint64_t* in, uint64_t* eg, int* n) {
  return guard([&] {
    need(p, "plan");
    PlanCost c = plan_cost(*p->p);
    *n = int(c.devices.size());
    for (int i = 0; i < *n && i < cap; ++i)
      devs[i] = rs_device{c.devices[size_t(i)].worker, c.devices[size_t(i)].local}, in[i] = c.ingress[size_t(i)],
      eg[i] = c.egress[size_t(i)];
  });
}
int rs_parse_parallel_config(const char* json, int n, const rs_device* devs, rs_ptc** out) {
  return guard([&] {
    need(json, "json"), need(out, "out");
    std::vector<DeviceId> d;
    if (devs)
      for (int i = 0; i < n; ++i) d.push_back(to_dev(devs[i]));
    *out = new rs_ptc{std::make_shared<const PTC>(parse_parallel_config(json, d))};
  });
}
int64_t rs_serialize_parallel_config(const rs_ptc* p, char* buf, int64_t cap) {
  if (!p) return -1;
  try {
    std::string s = serialize_parallel_config(*p->p);
    if (buf && cap > 0) std::snprintf(buf, size_t(cap), "%s", s.c_str());
    return int64_t(s.size()) + 1;
  } catch (const Error& e) {
    g_last = e.what();
    return -1;
  }
}
int rs_plan_cost_central(const rs_plan* p, rs_device central, int cap, rs_device* devs, uint64_t* in, uint64_t* eg,
                         int* n) {
  return guard([&] {
    need(p, "plan");
    PlanCost c = plan_cost_central(*p->p, to_dev(central));
    *n = int(c.devices.size());
    for (int i = 0; i < *n && i < cap; ++i)
      devs[i] = rs_device{c.devices[size_t(i)].worker, c.devices[size_t(i)].local}, in[i] = c.ingress[size_t(i)],
      eg[i] = c.egress[size_t(i)];
  });
}
int64_t rs_plan_text(const rs_plan* p, char* buf, int64_t cap) {
  if (!p) return -1;
  std::string s = plan_text(*p->p);
  if (buf && cap > 0) std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int64_t(s.size()) + 1;
}
int rs_choose_source(int n, const rs_device* cand, const uint64_t* egress, rs_device dst, rs_device* out) {
  return guard([&] {
    std::vector<DeviceId> c;
    std::map<DeviceId, uint64_t> eg;
    for (int i = 0; i < n; ++i) c.push_back(to_dev(cand[i])), eg[to_dev(cand[i])] = egress ? egress[i] : 0;
    DeviceId d = choose_source(c, to_dev(dst), eg);
    *out = rs_device{d.worker, d.local};
  });
}

// ---- executor ---------------------------------------------------------------------------------
int rs_executor_create(rs_context* c, const rs_plan* p, const int32_t* src_gpu, const int32_t* dst_gpu,
                       uint64_t tile_bytes, rs_executor** out) {
  return guard([&] {
    need(p, "plan"), need(out, "out");
    std::vector<int> s(src_gpu, src_gpu + p->p->from->devices.size());
    std::vector<int> d(dst_gpu, dst_gpu + p->p->to->devices.size());
    *out = new rs_executor{std::make_unique<Executor>(ctx_of(c), p->p, s, d, tile_bytes ? tile_bytes : (256u << 10))};
  });
}
int rs_executor_create_window(rs_context* c, const rs_plan* p, const int32_t* src_gpu, const int32_t* dst_gpu,
                              uint64_t tile_bytes, uint32_t t_begin, uint32_t t_end, rs_executor** out) {
  return guard([&] {
    need(p, "plan"), need(out, "out");
    std::vector<int> s(src_gpu, src_gpu + p->p->from->devices.size());
    std::vector<int> d(dst_gpu, dst_gpu + p->p->to->devices.size());
    *out = new rs_executor{std::make_unique<Executor>(ctx_of(c), p->p, s, d, tile_bytes ? tile_bytes : (256u << 10),
                                                      CopyConfig::from_env(), t_begin, t_end)};
  });
}
int rs_executor_create_central(rs_context* c, const rs_plan* p, const int32_t* src_gpu, const int32_t* dst_gpu,
                               uint64_t tile_bytes, int central_gpu, rs_executor** out) {
  return guard([&] {
    need(p, "plan"), need(out, "out");
    if (central_gpu < 0) raise(Errc::InvalidArgument, "central GPU must be >= 0");
    std::vector<int> s(src_gpu, src_gpu + p->p->from->devices.size());
    std::vector<int> d(dst_gpu, dst_gpu + p->p->to->devices.size());
    *out = new rs_executor{std::make_unique<Executor>(ctx_of(c), p->p, s, d, tile_bytes ? tile_bytes : (256u << 10),
                                                      CopyConfig::from_env(), 0, UINT32_MAX, central_gpu)};
  });
}
int rs_executor_staging_bytes(const rs_executor* e, uint64_t* bytes) {
  return guard([&] {
    need(e, "executor"), need(bytes, "bytes");
    *bytes = e->e->staging_bytes();
  });
}
void rs_executor_destroy(rs_executor* e) { delete e; }
int rs_executor_arena_bytes(const rs_executor* e, int gpu, uint64_t* s, uint64_t* d) {
  return guard([&] {
    need(e, "executor");
    *s = e->e->src_arena_bytes(gpu), *d = e->e->dst_arena_bytes(gpu);
  });
}
int rs_executor_bind(rs_executor* e, int gpu, void* s, void* d) {
  return guard([&] {
    need(e, "executor");
    e->e->bind(gpu, s, d);
  });
}
int rs_executor_prepare(rs_executor* e) {
  return guard([&] {
    need(e, "executor");
    e->e->prepare();
  });
}
int rs_executor_run(rs_executor* e) {
  return guard([&] {
    need(e, "executor");
    e->e->run();
  });
}
int rs_executor_wait(rs_executor* e, int cap, rs_timing* out, int* n) {
  return guard([&] {
    need(e, "executor");
    auto t = e->e->wait();
    *n = int(t.size());
    for (int i = 0; i < *n && i < cap; ++i)
      out[i] = rs_timing{t[size_t(i)].ms, t[size_t(i)].tiles, t[size_t(i)].bytes, t[size_t(i)].launches, t[size_t(i)].read_bytes, t[size_t(i)].main_ms};
  });
}
int rs_executor_run_host(rs_executor* e, int gpu, const void* host_src, void* host_dst, rs_timing* out) {
  return guard([&] {
    need(e, "executor"), need(out, "out");
    Timing t = e->e->run_host(gpu, host_src, host_dst);
    *out = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_executor_run_host_flags(rs_executor* e, int gpu, const void* host_src, void* host_dst, unsigned flags,
                               rs_timing* out) {
  return guard([&] {
    need(e, "executor"), need(out, "out");
    Timing t = e->e->run_host(gpu, host_src, host_dst, flags);
    *out = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_executor_host_upload_bytes(rs_executor* e, int gpu, unsigned flags, uint64_t* bytes) {
  return guard([&] {
    need(e, "executor"), need(bytes, "bytes");
    *bytes = e->e->host_upload_bytes(gpu, flags);
  });
}
int rs_executor_host_phase(rs_executor* e, int gpu, int phase, void* host_buf) {
  return guard([&] {
    need(e, "executor");
    e->e->host_phase(gpu, phase, host_buf);
  });
}
int rs_executor_host_elapsed(rs_executor* e, int gpu, float* ms) {
  return guard([&] {
    need(e, "executor"), need(ms, "ms");
    *ms = e->e->host_elapsed(gpu);
  });
}
int rs_executor_world_ms(const rs_executor* e, float* ms) {
  return guard([&] {
    need(e, "executor"), need(ms, "ms");
    *ms = e->e->world_ms();
  });
}
int rs_executor_run_host_world(rs_executor* e, int n, const void* const* host_src, void* const* host_dst, float* ms) {
  return guard([&] {
    need(e, "executor"), need(host_src, "host_src"), need(host_dst, "host_dst"), need(ms, "ms");
    if (n != e->e->context().world()) raise(reshard::Errc::InvalidArgument, "one host buffer pair per world GPU");
    *ms = e->e->run_host_world(std::vector<const void*>(host_src, host_src + n), std::vector<void*>(host_dst, host_dst + n));
  });
}
int rs_executor_digests(rs_executor* e, int side, int replica, int cap, int32_t* tensor, uint64_t* fnv, int32_t* ok,
                        int* n) {
  return guard([&] {
    need(e, "executor"), need(n, "n");
    if (side != 0 && side != 1) raise(reshard::Errc::InvalidArgument, "side must be 0 (source) or 1 (destination)");
    const auto d = e->e->digests(side, replica);
    *n = int(d.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      if (tensor) tensor[i] = int32_t(d[size_t(i)].tensor);
      if (fnv) fnv[i] = d[size_t(i)].fnv;
      if (ok) ok[i] = int32_t(d[size_t(i)].ok);
    }
  });
}
int rs_executor_fill_sources(rs_executor* e) {
  return guard([&] {
    need(e, "executor");
    e->e->fill_sources();
  });
}
int rs_executor_verify(rs_executor* e, uint64_t* bad) {
  return guard([&] {
    need(e, "executor"), need(bad, "out");
    *bad = e->e->verify_destinations();
  });
}
int rs_executor_src_cells(const rs_executor* e, int cap, rs_cell_binding* out, int* n) {
  return guard([&] {
    need(e, "executor");
    const auto& v = e->e->src_bindings();
    *n = int(v.size());
    for (int i = 0; i < *n && i < cap; ++i) out[i] = rs_cell_binding{v[size_t(i)].gpu, v[size_t(i)].arena, v[size_t(i)].offset, v[size_t(i)].bytes};
  });
}
int rs_executor_dst_cells(const rs_executor* e, int cap, rs_cell_binding* out, int32_t* dev, int32_t* tensor, int32_t* cell,
                          int* n) {
  return guard([&] {
    need(e, "executor");
    const auto& v = e->e->dst_bindings();
    const auto& dc = e->e->plan().dst_cells;
    *n = int(v.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      out[i] = rs_cell_binding{v[size_t(i)].gpu, v[size_t(i)].arena, v[size_t(i)].offset, v[size_t(i)].bytes};
      if (dev) dev[i] = int32_t(dc[size_t(i)].dst_device);
      if (tensor) tensor[i] = int32_t(dc[size_t(i)].tensor);
      if (cell) cell[i] = int32_t(dc[size_t(i)].cell);
    }
  });
}
int rs_executor_read_bytes(const rs_executor* e, int gpu, uint64_t* bytes) {
  return guard([&] {
    need(e, "executor"), need(bytes, "bytes");
    *bytes = e->e->read_bytes_for(gpu);
  });
}
int rs_executor_bytes_to(const rs_executor* e, int gpu, int n, uint64_t* bytes) {
  return guard([&] {
    need(e, "executor"), need(bytes, "bytes");
    const std::vector<uint64_t> v = e->e->bytes_to(gpu);
    if (n < int(v.size())) raise(Errc::InvalidArgument, "bytes_to: array shorter than the world");
    std::copy(v.begin(), v.end(), bytes);
  });
}
int rs_executor_tiles(const rs_executor* e, int gpu, uint64_t* tiles, uint64_t* bytes) {
  return guard([&] {
    need(e, "executor");
    *tiles = e->e->tiles_for(gpu), *bytes = e->e->copy_bytes_for(gpu);
  });
}

// ---- PTX1 / checkpoint -----------------------------------------------------------------------
int rs_ptx_encoded_size(int dtype, int rank, const uint64_t* shape, uint64_t* bytes) {
  return guard([&] {
    need(bytes, "bytes");
    *bytes = ptx_encoded_size(dtype_from_code(dtype), to_shape(rank, shape));
  });
}
int rs_ptx_encode_header(int dtype, int rank, const uint64_t* shape, uint8_t* out, uint64_t cap, uint64_t* written) {
  return guard([&] {
    need(out, "out"), need(written, "written");
    auto h = ptx_encode_header(dtype_from_code(dtype), to_shape(rank, shape));
    if (h.size() > cap) raise(Errc::InvalidArgument, "buffer too small");
    std::memcpy(out, h.data(), h.size());
    *written = h.size();
  });
}
int rs_ptx_decode_header(const uint8_t* bytes, uint64_t n, int32_t* dtype, int32_t* rank, uint64_t* shape,
                         uint64_t* header_bytes) {
  return guard([&] {
    need(bytes, "bytes");
    PtxHeader h = ptx_decode_header(bytes, n);
    if (h.shape.size() > RS_MAX_RANK) raise(Errc::InvalidTensor, "rank above 8");
    *dtype = int32_t(h.dtype), *rank = int32_t(h.shape.size()), *header_bytes = h.header_bytes;
    for (size_t d = 0; d < h.shape.size(); ++d) shape[d] = h.shape[d];
  });
}
int rs_checkpoint_save(rs_executor* e, int side, const char* dir, uint64_t* files, uint64_t* bytes, double* seconds) {
  return guard([&] {
    need(e, "executor"), need(dir, "dir");
    IoStats s = checkpoint_save(*e->e, side, dir);
    if (files) *files = s.files;
    if (bytes) *bytes = s.bytes;
    if (seconds) *seconds = s.seconds;
  });
}
int rs_checkpoint_load(rs_executor* e, const char* dir, uint64_t* files, uint64_t* bytes, double* seconds) {
  return guard([&] {
    need(e, "executor"), need(dir, "dir");
    IoStats s = checkpoint_load(*e->e, dir);
    if (files) *files = s.files;
    if (bytes) *bytes = s.bytes;
    if (seconds) *seconds = s.seconds;
  });
}

// ---- dataset ---------------------------------------------------------------------------------
int rs_shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm) {
  return guard([&] {
    if (n) need(perm, "perm");
    shuffle_epoch(n, seed, epoch, perm);
  });
}
int rs_repartition_count(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t rank, uint64_t* count) {
  return guard([&] {
    need(count, "count");
    *count = repartition_count(n, B, at_step, dp, rank);
  });
}
int rs_repartition_position(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t rank, uint64_t k,
                            uint64_t* pos) {
  return guard([&] {
    need(pos, "pos");
    *pos = repartition_position(n, B, at_step, dp, rank, k);
  });
}
int rs_locate_sample(uint64_t n, uint64_t B, uint64_t at_step, uint64_t dp, uint64_t rank, uint64_t k, const uint64_t* perm,
                     const uint64_t* samples, const uint8_t* file_class, uint64_t* out4) {
  return guard([&] {
    need(perm, "perm"), need(samples, "samples"), need(file_class, "file_class"), need(out4, "out");
    const uint64_t pos = repartition_position(n, B, at_step, dp, rank, k);
    const uint64_t* e = samples + 3 * perm[pos];
    out4[0] = e[0], out4[1] = e[1], out4[2] = e[2], out4[3] = file_class[e[0]];
  });
}
int rs_shuffle_scratch_bytes(uint64_t n, uint64_t* bytes) {
  return guard([&] {
    need(bytes, "bytes");
    *bytes = shuffle_scratch_bytes(n);
  });
}
int rs_shuffle_epoch_device(rs_context* c, int gpu, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm,
                            void* scratch, rs_timing* timing) {
  return guard([&] {
    need(perm, "perm"), need(scratch, "scratch");
    Timing t = shuffle_epoch_device(ctx_of(c), gpu, n, seed, epoch, perm, scratch);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_dataset_index_pad(rs_context* c, int gpu, const uint64_t* packed, uint64_t* padded, uint64_t n,
                         rs_timing* timing) {
  return guard([&] {
    need(packed, "packed"), need(padded, "padded");
    Timing t = dataset_index_pad(ctx_of(c), gpu, packed, padded, n);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_dataset_index_upload(rs_context* c, int gpu, const uint64_t* host_perm, const uint64_t* host_samples,
                            uint64_t n, uint64_t* perm, uint64_t* samples, uint64_t* padded, rs_timing* timing) {
  return guard([&] {
    need(host_perm, "host_perm"), need(host_samples, "host_samples"), need(perm, "perm"), need(samples, "samples");
    Timing t = dataset_index_upload(ctx_of(c), gpu, host_perm, host_samples, n, perm, samples, padded);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_repartition_to_host(rs_context* c, int gpu, const rs_dataset_index* idx, uint64_t B, uint64_t at_step,
                           uint64_t dp, uint64_t rank, const rs_partition_out* out, void* scratch,
                           const rs_partition_host* host, rs_timing* timing) {
  return guard([&] {
    need(idx, "index"), need(out, "out"), need(scratch, "scratch"), need(host, "host");
    need(host->pos, "host pos"), need(host->ent, "host ent"), need(host->boff, "host boff"), need(host->qcount, "host qcount");
    for (int q = 0; q < 3; ++q) need(host->queue[q], "host queue");
    DatasetIndexView v{idx->perm, idx->samples, idx->file_class, idx->n, idx->entry_bytes};
    PartitionOut o{out->pos, out->ent, out->boff, {out->queue[0], out->queue[1], out->queue[2]}, out->qcount};
    PartitionHost h{host->pos, host->ent, host->boff, {host->queue[0], host->queue[1], host->queue[2]}, host->qcount};
    Timing t = repartition_to_host(ctx_of(c), gpu, v, B, at_step, dp, rank, o, scratch, h);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_repartition_scratch_bytes(uint64_t count, uint64_t* bytes) {
  return guard([&] {
    need(bytes, "bytes");
    *bytes = repartition_scratch_bytes(count);
  });
}
int rs_repartition(rs_context* c, int gpu, const rs_dataset_index* idx, uint64_t B, uint64_t at_step, uint64_t dp,
                   uint64_t rank, const rs_partition_out* out, void* scratch, rs_timing* timing) {
  return guard([&] {
    need(idx, "index"), need(out, "out"), need(scratch, "scratch");
    DatasetIndexView v{idx->perm, idx->samples, idx->file_class, idx->n, idx->entry_bytes};
    PartitionOut o{out->pos, out->ent, out->boff, {out->queue[0], out->queue[1], out->queue[2]}, out->qcount};
    Timing t = repartition_device(ctx_of(c), gpu, v, B, at_step, dp, rank, o, scratch);
    if (timing) *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}
int rs_repartition_batch(rs_context* c, int gpu, const rs_dataset_index* idx, uint64_t B, const rs_repartition_job* jobs,
                         int n, rs_timing* per_job, rs_timing* total) {
  return guard([&] {
    need(idx, "index"), need(total, "total");
    if (n < 0) raise(Errc::InvalidArgument, "negative job count");
    if (n > 0) need(jobs, "jobs");
    DatasetIndexView v{idx->perm, idx->samples, idx->file_class, idx->n, idx->entry_bytes};
    std::vector<RepartJob> js;
    js.reserve(size_t(n));
    for (int i = 0; i < n; ++i) {
      const rs_repartition_job& j = jobs[i];
      need(j.scratch, "scratch"), need(j.file_class, "file_class");
      js.push_back(RepartJob{j.at_step, j.new_dp, j.rank, j.file_class,
                             PartitionOut{j.out.pos, j.out.ent, j.out.boff, {j.out.queue[0], j.out.queue[1], j.out.queue[2]},
                                          j.out.qcount},
                             j.scratch});
    }
    std::vector<Timing> pj;
    Timing t = repartition_batch_device(ctx_of(c), gpu, v, B, js.data(), js.size(), per_job ? &pj : nullptr);
    *total = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
    if (per_job)
      for (int i = 0; i < n; ++i) {
        const Timing& r = pj[size_t(i)];
        per_job[i] = rs_timing{r.ms, r.tiles, r.bytes, r.launches, r.read_bytes, r.main_ms};
      }
  });
}
int rs_repartition_gather_probe(rs_context* c, int gpu, const rs_dataset_index* idx, uint64_t B, uint64_t at_step,
                                uint64_t dp, uint64_t rank, int reps, rs_timing* timing) {
  return guard([&] {
    need(idx, "index"), need(timing, "timing");
    DatasetIndexView v{idx->perm, idx->samples, idx->file_class, idx->n, idx->entry_bytes};
    Timing t = repartition_gather_probe(ctx_of(c), gpu, v, B, at_step, dp, rank, reps);
    *timing = rs_timing{t.ms, t.tiles, t.bytes, t.launches, t.read_bytes, t.main_ms};
  });
}

}  // extern "C"
