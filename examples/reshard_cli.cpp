// examples/reshard_cli.cpp — the whole reconfiguration from C++ (no Python), the way a host
// program of the reference would drive it: build the two PTCs, plan (Alg. 1), lay out and
// bind the arenas, prepare the device-resident schedule, fill the synthetic state, execute,
// verify every destination byte, and print the timings.
//
//   g++ -std=c++20 -I paper_2312_05181_b200/csrc -I /usr/local/cuda/include examples/reshard_cli.cpp
//       -L paper_2312_05181_b200 -lreshard_b200 -L /usr/local/cuda/lib64 -lcudart
//       -Wl,-rpath,$PWD/paper_2312_05181_b200 -o reshard_cli
//   ./reshard_cli [h L S V  T P D  T' P' D']      (default: GPT-3 1.3B (2,1,1) -> (2,1,2))
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "reshard/executor.hpp"

using namespace reshard;
using clk = std::chrono::steady_clock;

static double ms_since(clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); }

int main(int argc, char** argv) {
  uint64_t h = 2048, L = 24, S = 2048, V = 50304;
  int T = 2, P = 1, D = 1, T2 = 2, P2 = 1, D2 = 2;
  if (argc == 11) {
    h = std::strtoull(argv[1], nullptr, 10), L = std::strtoull(argv[2], nullptr, 10);
    S = std::strtoull(argv[3], nullptr, 10), V = std::strtoull(argv[4], nullptr, 10);
    T = std::atoi(argv[5]), P = std::atoi(argv[6]), D = std::atoi(argv[7]);
    T2 = std::atoi(argv[8]), P2 = std::atoi(argv[9]), D2 = std::atoi(argv[10]);
  }
  try {
    const Catalog cat = Catalog::gpt(h, L, S, V, StateKind::MixedAdam);
    auto devices = [](int n) {
      std::vector<DeviceId> d;
      for (int i = 0; i < n; ++i) d.push_back({0, uint32_t(i)});
      return d;
    };
    auto from = std::make_shared<const PTC>(build_strategy(cat, devices(T * P * D), JobConfig{T, P, D}));
    auto to = std::make_shared<const PTC>(build_strategy(cat, devices(T2 * P2 * D2), JobConfig{T2, P2, D2}));
    auto t0 = clk::now();
    auto plan = generate_plan(from, to);
    const double plan_ms = ms_since(t0);

    Context ctx(1, {0}, {0});  // every logical device on cuda:0
    t0 = clk::now();
    Executor ex(ctx, plan, std::vector<int>(from->devices.size(), 0), std::vector<int>(to->devices.size(), 0));
    const double lower_ms = ms_since(t0);
    void *src = nullptr, *dst = nullptr;
    if (cudaMalloc(&src, std::max<uint64_t>(ex.src_arena_bytes(0), 256)) != cudaSuccess ||
        cudaMalloc(&dst, std::max<uint64_t>(ex.dst_arena_bytes(0), 256)) != cudaSuccess) {
      std::fprintf(stderr, "cudaMalloc failed\n");
      return 2;
    }
    ex.bind(0, src, dst);
    t0 = clk::now();
    ex.prepare();
    const double prepare_ms = ms_since(t0);
    ex.fill_sources();
    ex.run();
    ex.wait();  // warm-up
    ex.run();
    const Timing t = ex.wait()[0];
    const uint64_t bad = ex.verify_destinations();
    std::printf("plan %.2f ms, lower %.2f ms, prepare %.2f ms, reshard %.3f ms, %llu tiles, %.2f GB written, "
                "%.1f GB/s r+w, mismatched bytes %llu\n",
                plan_ms, lower_ms, prepare_ms, t.ms, (unsigned long long)t.tiles, t.bytes / 1e9,
                (t.bytes + t.read_bytes) / (t.ms * 1e-3) / 1e9, (unsigned long long)bad);
    cudaFree(src);
    cudaFree(dst);
    return bad == 0 ? 0 : 3;
  } catch (const Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1 + int(e.code());
  }
}
