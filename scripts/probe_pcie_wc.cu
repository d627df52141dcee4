// PCIe probe: does a write-combined pinned SOURCE buffer (cudaHostAllocWriteCombined: the host
// only writes it, the GPU only reads it — the e2e path's host_src) change the copy-engine H2D
// rate, alone and with a concurrent D2H into a normal pinned buffer?  2 GiB each way, best of 5.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_pcie_wc probe_pcie_wc.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                    \
  do {                                                           \
    cudaError_t e = (x);                                         \
    if (e != cudaSuccess) {                                      \
      printf("%s: %s\n", #x, cudaGetErrorString(e));             \
      exit(1);                                                   \
    }                                                            \
  } while (0)

static float run(cudaStream_t s1, cudaStream_t s2, void* d_a, const void* h_in, void* h_out, const void* d_b,
                 size_t bytes, bool up, bool down) {
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEvent_t a0, a1, b0, b1;
    CK(cudaEventCreate(&a0));
    CK(cudaEventCreate(&a1));
    CK(cudaEventCreate(&b0));
    CK(cudaEventCreate(&b1));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a0, s1));
    CK(cudaEventRecord(b0, s2));
    if (up) CK(cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1));
    if (down) CK(cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2));
    CK(cudaEventRecord(a1, s1));
    CK(cudaEventRecord(b1, s2));
    CK(cudaDeviceSynchronize());
    float ta = 0, tb = 0;
    CK(cudaEventElapsedTime(&ta, a0, a1));
    CK(cudaEventElapsedTime(&tb, b0, b1));
    const float t = (up ? ta : 0) > (down ? tb : 0) ? ta : tb;
    if (t < best) best = t;
    cudaEventDestroy(a0), cudaEventDestroy(a1), cudaEventDestroy(b0), cudaEventDestroy(b1);
  }
  return best;
}

int main() {
  const size_t bytes = size_t(2) << 30;
  void *h_in, *h_wc, *h_out, *d_a, *d_b;
  CK(cudaHostAlloc(&h_in, bytes, cudaHostAllocPortable));
  CK(cudaHostAlloc(&h_wc, bytes, cudaHostAllocPortable | cudaHostAllocWriteCombined));
  CK(cudaHostAlloc(&h_out, bytes, cudaHostAllocPortable));
  CK(cudaMalloc(&d_a, bytes));
  CK(cudaMalloc(&d_b, bytes));
  CK(cudaMemset(d_b, 1, bytes));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  const double gb = bytes / 1e9;
  for (int rep = 0; rep < 2; ++rep) {
    for (int wc = 0; wc < 2; ++wc) {
      const void* src = wc ? h_wc : h_in;
      const float up = run(s1, s2, d_a, src, h_out, d_b, bytes, true, false);
      const float both = run(s1, s2, d_a, src, h_out, d_b, bytes, true, true);
      printf("{\"src\": \"%s\", \"h2d_gbs\": %.1f, \"bidir_gbs_each\": %.1f}\n", wc ? "write-combined" : "default",
             gb / (up * 1e-3), gb / (both * 1e-3));
    }
  }
  const float down = run(s1, s2, d_a, h_in, h_out, d_b, bytes, false, true);
  printf("{\"d2h_gbs\": %.1f}\n", gb / (down * 1e-3));
  return 0;
}
