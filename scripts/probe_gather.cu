// Random-gather probe for the K5 access pattern: read a permutation
// sequentially, gather one 24-byte index entry per position, reduce.  Measures how many
// random entry gathers per second this B200 sustains, as a function of items in flight per
// thread, CTA size and entry stride (24 B packed vs 32 B padded), to bound K5 from above.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o probe_gather probe_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int K, int STRIDE_WORDS>
__global__ void gather(const unsigned long long* __restrict__ perm, const unsigned long long* __restrict__ ent,
                       unsigned long long n, unsigned long long* __restrict__ out) {
  const unsigned long long base = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * K;
  unsigned long long idx[K], a[K], b[K], c[K];
#pragma unroll
  for (int j = 0; j < K; ++j) idx[j] = base + j < n ? __ldg(perm + base + j) : 0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const unsigned long long* e = ent + STRIDE_WORDS * idx[j];
    a[j] = __ldg(e), b[j] = __ldg(e + 1), c[j] = __ldg(e + 2);
  }
  unsigned long long s = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) s += a[j] ^ b[j] ^ c[j];
  if (base < n) out[base / K] = s;
}

__global__ void init_perm(unsigned long long* p, unsigned long long n, unsigned long long mod, unsigned long long seed) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    unsigned long long z = (i + seed) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    p[i] = (z ^ (z >> 31)) % mod;  // random (not a permutation; same access statistics)
  }
}

template <int K, int S>
void run(const unsigned long long* perm, const unsigned long long* ent, unsigned long long n, unsigned long long* out,
         int threads, const char* tag) {
  const unsigned long long per = (unsigned long long)threads * K;
  const unsigned grid = unsigned((n + per - 1) / per);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  gather<K, S><<<grid, threads>>>(perm, ent, n, out);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    gather<K, S><<<grid, threads>>>(perm, ent, n, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, gather<K, S>) == cudaSuccess) regs = fa.numRegs;
  printf("{\"tag\": \"%s\", \"K\": %d, \"stride_b\": %d, \"threads\": %d, \"regs\": %d, \"n\": %llu, \"ms\": %.4f, "
         "\"gathers_per_s_G\": %.2f, \"alg_GBs\": %.1f}\n",
         tag, K, S * 8, threads, regs, n, best, n / (best * 1e-3) / 1e9, n * (8.0 + 24.0 + 8.0 / K) / (best * 1e-3) / 1e9);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

int main(int argc, char** argv) {
  const unsigned long long N = 100000000ull;  // index entries (config 5)
  const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 36000000ull;  // gathers per launch
  unsigned long long *perm, *ent, *out;
  CK(cudaMalloc(&perm, n * 8));
  CK(cudaMalloc(&ent, N * 32));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMemset(ent, 1, N * 32));
  init_perm<<<1184, 256>>>(perm, n, N, 777);  // indices in [0, N)
  CK(cudaDeviceSynchronize());
  run<4, 3>(perm, ent, n, out, 256, "packed24");
  run<8, 3>(perm, ent, n, out, 256, "packed24");
  run<16, 3>(perm, ent, n, out, 256, "packed24");
  run<8, 3>(perm, ent, n, out, 512, "packed24");
  run<16, 3>(perm, ent, n, out, 128, "packed24");
  run<32, 3>(perm, ent, n, out, 128, "packed24");
  run<8, 4>(perm, ent, n, out, 256, "padded32");
  run<16, 4>(perm, ent, n, out, 256, "padded32");
  run<16, 4>(perm, ent, n, out, 128, "padded32");
  return 0;
}
