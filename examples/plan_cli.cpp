// examples/plan_cli.cpp — using the C++ drop-in API directly (no Python), the way a
// reference maintainer would: build two PTCs, generate the Alg. 1 plan, print it in the
// SPEC.md:268 text format and the plan_cost table.
//
//   g++ -std=c++20 -I paper_2312_05181_b200/csrc examples/plan_cli.cpp \
//       -L paper_2312_05181_b200 -lreshard_b200 -Wl,-rpath,$PWD/paper_2312_05181_b200 -o plan_cli
//   ./plan_cli fig6            # the Fig. 6 scenario (TP2 on 2 devices -> TP3 x PP2 on 6)
//   ./plan_cli gpt T P D T' P' D' [h L S V]
#include <cstdio>
#include <cstdlib>
#include <string>

#include "reshard/planner.hpp"

using namespace reshard;

static std::vector<DeviceId> devices(int n) {
  std::vector<DeviceId> d;
  for (int i = 0; i < n; ++i) d.push_back({0, uint32_t(i)});
  return d;
}

int main(int argc, char** argv) {
  try {
    std::string mode = argc > 1 ? argv[1] : "fig6";
    Catalog cat;
    JobConfig a{2, 1, 1}, b{3, 2, 1};
    if (mode == "fig6") {
      cat.add({"t1", Dtype::F32, {6}, 0, 0});
      cat.add({"t2", Dtype::F32, {6}, 0, 1});
    } else if (mode == "gpt" && argc >= 8) {
      a = {std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4])};
      b = {std::atoi(argv[5]), std::atoi(argv[6]), std::atoi(argv[7])};
      uint64_t h = argc > 8 ? std::strtoull(argv[8], nullptr, 10) : 64, L = argc > 9 ? std::strtoull(argv[9], nullptr, 10) : 4;
      uint64_t S = argc > 10 ? std::strtoull(argv[10], nullptr, 10) : 16, V = argc > 11 ? std::strtoull(argv[11], nullptr, 10) : 128;
      cat = Catalog::gpt(h, L, S, V, StateKind::MixedAdam);
    } else {
      std::fprintf(stderr, "usage: plan_cli fig6 | gpt T P D T2 P2 D2 [h L S V]\n");
      return 2;
    }
    auto from = std::make_shared<const PTC>(build_strategy(cat, devices(a.tp * a.pp * a.dp), a));
    auto to = std::make_shared<const PTC>(build_strategy(cat, devices(b.tp * b.pp * b.dp), b));
    auto plan = generate_plan(from, to);
    std::fputs(plan_text(*plan).c_str(), stdout);
    PlanCost c = plan_cost(*plan);
    for (size_t i = 0; i < c.devices.size(); ++i)
      std::printf("# %s ingress=%llu egress=%llu\n", c.devices[i].to_string().c_str(),
                  (unsigned long long)c.ingress[i], (unsigned long long)c.egress[i]);
    std::printf("# total=%llu\n", (unsigned long long)c.total);
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1 + static_cast<int>(e.code());
  }
}
