// PCIe probe for the host-buffer e2e path: can SM-issued (zero-copy) stores or loads over
// mapped pinned memory move more bytes while the copy engine runs the other direction than
// two copy-engine streams do?  Scenarios (2 GiB each way):
//   ce_h2d, ce_d2h            one direction alone, copy engine
//   ce_both                   both directions at once, two copy-engine streams (run_host today)
//   sm_d2h, sm_h2d            one direction alone, SM kernel through the mapped host pointer
//   ce_h2d+sm_d2h, sm_h2d+ce_d2h   mixed
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_pcie probe_pcie.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                               \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__global__ void copy16(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main(int argc, char** argv) {
  const size_t bytes = size_t(2) << 30, n16 = bytes / 16;
  const int blocks = argc > 1 ? atoi(argv[1]) : 148 * 4;
  void *h_in, *h_out, *d_a, *d_b;
  CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped));
  CK(cudaMalloc(&d_a, bytes));
  CK(cudaMalloc(&d_b, bytes));
  void *m_in, *m_out;
  CK(cudaHostGetDevicePointer(&m_in, h_in, 0));
  CK(cudaHostGetDevicePointer(&m_out, h_out, 0));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  auto h2d_ce = [&](cudaStream_t s) { CK(cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s)); };
  auto d2h_ce = [&](cudaStream_t s) { CK(cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s)); };
  auto h2d_sm = [&](cudaStream_t s) { copy16<<<blocks, 256, 0, s>>>((const uint4*)m_in, (uint4*)d_a, n16); };
  auto d2h_sm = [&](cudaStream_t s) { copy16<<<blocks, 256, 0, s>>>((const uint4*)d_b, (uint4*)m_out, n16); };
  struct Sc {
    const char* name;
    int a, b;  // 0 none, 1 ce_h2d, 2 ce_d2h, 3 sm_h2d, 4 sm_d2h
  } sc[] = {{"ce_h2d", 1, 0}, {"ce_d2h", 2, 0}, {"ce_both", 1, 2}, {"sm_h2d", 3, 0},
            {"sm_d2h", 4, 0}, {"ce_h2d+sm_d2h", 1, 4}, {"sm_h2d+ce_d2h", 3, 2}, {"sm_both", 3, 4}};
  auto run = [&](int op, cudaStream_t s) {
    if (op == 1) h2d_ce(s);
    if (op == 2) d2h_ce(s);
    if (op == 3) h2d_sm(s);
    if (op == 4) d2h_sm(s);
  };
  // two copy streams per direction (halves of the buffers), 4 streams at once for "both"
  {
    cudaStream_t q[4];
    for (auto& x : q) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    const size_t h = bytes / 2;
    for (int mode = 0; mode < 3; ++mode) {  // 0: H2D x2, 1: D2H x2, 2: both x2
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, q[0]));
        for (int i = 1; i < 4; ++i) CK(cudaStreamWaitEvent(q[i], e0, 0));
        if (mode != 1)
          for (int i = 0; i < 2; ++i)
            CK(cudaMemcpyAsync((char*)d_a + i * h, (char*)h_in + i * h, h, cudaMemcpyHostToDevice, q[i]));
        if (mode != 0)
          for (int i = 0; i < 2; ++i)
            CK(cudaMemcpyAsync((char*)h_out + i * h, (char*)d_b + i * h, h, cudaMemcpyDeviceToHost, q[2 + i]));
        for (int i = 1; i < 4; ++i) {
          CK(cudaEventRecord(e2, q[i]));
          CK(cudaStreamWaitEvent(q[0], e2, 0));
        }
        CK(cudaEventRecord(e1, q[0]));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r && ms < best) best = ms;
      }
      const char* name = mode == 0 ? "ce_h2d_x2" : mode == 1 ? "ce_d2h_x2" : "ce_both_x2";
      const double dirs = mode == 2 ? 2.0 : 1.0;
      printf("{\"scenario\": \"%s\", \"ms\": %.3f, \"gbs_each\": %.1f, \"gbs_total\": %.1f}\n", name, best,
             bytes / (best * 1e-3) / 1e9, dirs * bytes / (best * 1e-3) / 1e9);
    }
  }
  for (auto& c : sc) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0, s1));
      CK(cudaStreamWaitEvent(s2, e0, 0));
      run(c.a, s1);
      run(c.b, s2);
      CK(cudaEventRecord(e1, s1));
      CK(cudaEventRecord(e2, s2));
      CK(cudaStreamWaitEvent(s1, e2, 0));
      CK(cudaEventRecord(e1, s1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r && ms < best) best = ms;
    }
    const double dirs = c.b ? 2.0 : 1.0;
    printf("{\"scenario\": \"%s\", \"blocks\": %d, \"ms\": %.3f, \"gbs_each\": %.1f, \"gbs_total\": %.1f}\n", c.name,
           blocks, best, bytes / (best * 1e-3) / 1e9, dirs * bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
