// Random-access cost probe (diagnostic for K5's traffic): 10^8 records through a random
// permutation, as gathers (K5's pattern: out[i] = rec[perm[i]]) and as scatters (out[perm[i]]
// = rec[i]) of 8-, 24- and 32-byte records; sequential copy for reference.  Best of 5, events.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_scatter probe_scatter.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                    \
  do {                                                           \
    cudaError_t e = (x);                                         \
    if (e != cudaSuccess) {                                      \
      printf("%s: %s\n", #x, cudaGetErrorString(e));             \
      exit(1);                                                   \
    }                                                            \
  } while (0)

typedef unsigned long long u64;
__global__ void gather8(const u64* __restrict__ perm, const u64* __restrict__ in, u64* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) out[i] = __ldg(in + perm[i]);
}
__global__ void scatter8(const u64* __restrict__ perm, const u64* __restrict__ in, u64* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) out[perm[i]] = in[i];
}
__global__ void gather32(const u64* __restrict__ perm, const ulonglong4* __restrict__ in, ulonglong4* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const ulonglong2* s = reinterpret_cast<const ulonglong2*>(in + perm[i]);
    const ulonglong2 a = __ldg(s), b = __ldg(s + 1);
    out[i] = make_ulonglong4(a.x, a.y, b.x, b.y);
  }
}
__global__ void scatter32(const u64* __restrict__ perm, const ulonglong4* __restrict__ in, ulonglong4* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const ulonglong2* s = reinterpret_cast<const ulonglong2*>(in + i);
    ulonglong2* d = reinterpret_cast<ulonglong2*>(out + perm[i]);
    d[0] = s[0], d[1] = s[1];
  }
}
__global__ void scatter24(const u64* __restrict__ perm, const u64* __restrict__ in, u64* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 p = perm[i];
    out[3 * p] = in[3 * i], out[3 * p + 1] = in[3 * i + 1], out[3 * p + 2] = in[3 * i + 2];
  }
}
__global__ void copy32(const ulonglong4* __restrict__ in, ulonglong4* __restrict__ out, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const ulonglong2* s = reinterpret_cast<const ulonglong2*>(in + i);
    ulonglong2* d = reinterpret_cast<ulonglong2*>(out + i);
    d[0] = s[0], d[1] = s[1];
  }
}

int main() {
  const u64 n = 100000000ull;
  std::vector<u64> h(n);
  for (u64 i = 0; i < n; ++i) h[i] = i;
  u64 x = 0x9e3779b97f4a7c15ull;
  for (u64 i = n - 1; i > 0; --i) {  // Fisher-Yates with splitmix64
    x += 0x9e3779b97f4a7c15ull;
    u64 z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    const u64 j = z % (i + 1);
    const u64 t = h[i];
    h[i] = h[j], h[j] = t;
  }
  u64 *perm, *a, *b;
  CK(cudaMalloc(&perm, 8 * n));
  CK(cudaMalloc(&a, 32 * n));
  CK(cudaMalloc(&b, 32 * n));
  CK(cudaMemcpy(perm, h.data(), 8 * n, cudaMemcpyHostToDevice));
  CK(cudaMemset(a, 1, 32 * n));
  CK(cudaMemset(b, 0, 32 * n));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int grid = 148 * 8, block = 256;
  auto timeit = [&](const char* name, auto launch, double useful_bytes) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r && ms < best) best = ms;
    }
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"useful_gbs\": %.1f}\n", name, best, useful_bytes / (best * 1e-3) / 1e9);
  };
  timeit("copy32 (sequential)", [&] { copy32<<<grid, block>>>((const ulonglong4*)a, (ulonglong4*)b, n); }, 64.0 * n);
  timeit("gather8", [&] { gather8<<<grid, block>>>(perm, a, b, n); }, 24.0 * n);
  timeit("scatter8", [&] { scatter8<<<grid, block>>>(perm, a, b, n); }, 24.0 * n);
  timeit("gather32", [&] { gather32<<<grid, block>>>(perm, (const ulonglong4*)a, (ulonglong4*)b, n); }, 72.0 * n);
  timeit("scatter32", [&] { scatter32<<<grid, block>>>(perm, (const ulonglong4*)a, (ulonglong4*)b, n); }, 72.0 * n);
  timeit("scatter24", [&] { scatter24<<<grid, block>>>(perm, a, b, n); }, 56.0 * n);
  CK(cudaGetLastError());
  return 0;
}
