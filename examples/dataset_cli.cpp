// examples/dataset_cli.cpp — the dataset side of a reconfiguration from C++ (no Python): the
// epoch permutation on the GPU (bit-identical to the host shuffle_epoch),
// the index laid out once, then every new DP rank of a DP change repartitioned in one batch
// and checked against the host's closed-form positions and the index.
//
//   g++ -std=c++20 -I paper_2312_05181_b200/csrc -I /usr/local/cuda/include examples/dataset_cli.cpp
//       -L paper_2312_05181_b200 -lreshard_b200 -L /usr/local/cuda/lib64 -lcudart
//       -Wl,-rpath,$PWD/paper_2312_05181_b200 -o dataset_cli
//   ./dataset_cli [N B at_step new_dp files]      (default: 10^7 samples, B 1280, step 2500, DP 4)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "reshard/dataset.hpp"

using namespace reshard;

#define CUDA(x)                                                      \
  do {                                                               \
    if (cudaError_t e_ = (x); e_ != cudaSuccess) {                   \
      std::fprintf(stderr, "CudaError: %s\n", cudaGetErrorString(e_)); \
      return 1 + int(Errc::CudaError);                               \
    }                                                                \
  } while (0)

int main(int argc, char** argv) {
  uint64_t n = 10'000'000, B = 1280, at = 2500, dp = 4, files = 100;
  if (argc == 6) {
    n = std::strtoull(argv[1], nullptr, 10), B = std::strtoull(argv[2], nullptr, 10);
    at = std::strtoull(argv[3], nullptr, 10), dp = std::strtoull(argv[4], nullptr, 10);
    files = std::strtoull(argv[5], nullptr, 10);
  }
  try {
    repartition_check(n, B, at, dp);  // IndivisibleBatch / StepBeyondEpoch before any device work
    Context ctx(1, {0}, {0});
    // the index as the reference stores it: per sample {file, offset, length}
    std::vector<uint64_t> samples(3 * n);
    const uint64_t per_file = (n + files - 1) / files;
    for (uint64_t k = 0; k < n; ++k)
      samples[3 * k] = k / per_file, samples[3 * k + 1] = (k % per_file) * 8206, samples[3 * k + 2] = 8206;
    uint64_t *d_perm, *d_packed, *d_padded;
    CUDA(cudaMalloc(&d_perm, 8 * n));
    CUDA(cudaMalloc(&d_packed, 24 * n));
    CUDA(cudaMalloc(&d_padded, 32 * n));
    CUDA(cudaMemcpy(d_packed, samples.data(), 24 * n, cudaMemcpyHostToDevice));
    dataset_index_pad(ctx, 0, d_packed, d_padded, n);  // once per index load

    // K8: the epoch order on the GPU, compared with the host loop
    std::vector<uint64_t> perm(n), got(n);
    shuffle_epoch(n, 0x5EED, 0, perm.data());
    void* shuf_scratch;
    CUDA(cudaMalloc(&shuf_scratch, shuffle_scratch_bytes(n)));
    const Timing ts = shuffle_epoch_device(ctx, 0, n, 0x5EED, 0, d_perm, shuf_scratch);
    CUDA(cudaMemcpy(got.data(), d_perm, 8 * n, cudaMemcpyDeviceToHost));
    const bool shuffle_ok = got == perm;

    // every new rank of the DP change: its outputs, scratch and locator classes; one batch
    std::vector<RepartJob> jobs;
    std::vector<uint64_t> counts;
    std::vector<void*> owned{d_perm, d_packed, d_padded, shuf_scratch};
    for (uint64_t d = 0; d < dp; ++d) {
      const uint64_t c = repartition_count(n, B, at, dp, d);
      std::vector<uint8_t> cls(files);
      for (uint64_t f = 0; f < files; ++f) cls[f] = uint8_t(f % (dp + 1) == d ? 0 : f % (dp + 1) == dp ? 2 : 1);
      PartitionOut o{};
      void *fc, *scratch;
      const uint64_t m = c ? c : 1;
      CUDA(cudaMalloc(reinterpret_cast<void**>(&o.pos), 8 * m));
      CUDA(cudaMalloc(reinterpret_cast<void**>(&o.ent), 24 * m));
      CUDA(cudaMalloc(reinterpret_cast<void**>(&o.boff), 8 * m));
      for (auto& q : o.queue) CUDA(cudaMalloc(reinterpret_cast<void**>(&q), 4 * m));
      CUDA(cudaMalloc(reinterpret_cast<void**>(&o.qcount), 24));
      CUDA(cudaMalloc(&fc, files));
      CUDA(cudaMalloc(&scratch, repartition_scratch_bytes(c)));
      CUDA(cudaMemcpy(fc, cls.data(), files, cudaMemcpyHostToDevice));
      for (void* p : {(void*)o.pos, (void*)o.ent, (void*)o.boff, (void*)o.queue[0], (void*)o.queue[1], (void*)o.queue[2],
                      (void*)o.qcount, fc, scratch})
        owned.push_back(p);
      jobs.push_back(RepartJob{at, dp, d, static_cast<const uint8_t*>(fc), o, scratch});
      counts.push_back(c);
    }
    const DatasetIndexView idx{d_perm, d_padded, nullptr, n, 32};
    repartition_batch_device(ctx, 0, idx, B, jobs.data(), jobs.size(), nullptr);  // warm-up
    const Timing t = repartition_batch_device(ctx, 0, idx, B, jobs.data(), jobs.size(), nullptr);

    // every rank: positions = the closed form, entries = the index at perm[pos], offsets = the
    // prefix sum of lengths (a sample of 4096 per rank)
    uint64_t checked = 0, bad = 0;
    for (size_t j = 0; j < jobs.size(); ++j) {
      const uint64_t c = counts[j];
      std::vector<uint64_t> pos(c), ent(3 * c), boff(c);
      CUDA(cudaMemcpy(pos.data(), jobs[j].out.pos, 8 * c, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(ent.data(), jobs[j].out.ent, 24 * c, cudaMemcpyDeviceToHost));
      CUDA(cudaMemcpy(boff.data(), jobs[j].out.boff, 8 * c, cudaMemcpyDeviceToHost));
      uint64_t run = 0;
      for (uint64_t k = 0; k < c; ++k) {
        if (boff[k] != run) ++bad;
        run += ent[3 * k + 2];
      }
      for (uint64_t k = 0; k < c; k += (c / 4096) + 1, ++checked) {
        const uint64_t p = repartition_position(n, B, at, dp, jobs[j].rank, k), s = perm[p];
        if (pos[k] != p || ent[3 * k] != samples[3 * s] || ent[3 * k + 1] != samples[3 * s + 1] ||
            ent[3 * k + 2] != samples[3 * s + 2])
          ++bad;
      }
    }
    std::printf("shuffle of %llu: %.3f ms on the GPU, %s the host loop\n", (unsigned long long)n, ts.ms,
                shuffle_ok ? "identical to" : "DIFFERENT FROM");
    std::printf("repartition of %zu ranks (%llu samples) in %.3f ms (gather pass %.3f ms, %llu launches)\n", jobs.size(),
                (unsigned long long)(n > at * B ? n - at * B : 0), t.ms, t.main_ms, (unsigned long long)t.launches);
    std::printf("checked %llu sampled positions / entries and every offset: mismatches %llu\n",
                (unsigned long long)checked, (unsigned long long)bad);
    for (void* p : owned) cudaFree(p);
    return shuffle_ok && bad == 0 ? 0 : 100;
  } catch (const Error& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1 + int(e.code());
  }
}
