// reshard/trace.hpp — NVTX ranges around the host phases (plan, lower/upload, execute,
// host-buffer path, dataset kernels, checkpoint I/O), so an nsys / ncu --nvtx capture shows
// which phase a kernel or copy belongs to (SURVEY §5 tracing; the reference records only
// elapsed phase markers).  NVTX 3 is header-only: without a tool attached a
// range is a no-op call.  Builds without the CUDA include path get an empty stub.
#pragma once

#if __has_include(<nvtx3/nvToolsExt.h>)
#include <nvtx3/nvToolsExt.h>
namespace reshard {
struct TraceRange {
  explicit TraceRange(const char* name) { nvtxRangePushA(name); }
  ~TraceRange() { nvtxRangePop(); }
  TraceRange(const TraceRange&) = delete;
  TraceRange& operator=(const TraceRange&) = delete;
};
}  // namespace reshard
#else
namespace reshard {
struct TraceRange {
  explicit TraceRange(const char*) {}
};
}  // namespace reshard
#endif
