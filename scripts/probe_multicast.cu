// Probe: can this box's B200 use NVLink SHARP (NVLS) multicast memory, and at what rate do
// multimem stores land?  A multicast object with a ONE-device team is legal: its stores leave
// the GPU for the NVSwitch, which replicates them to every bound member (here the GPU itself),
// so this is also an NVLink egress+ingress measurement on a one-GPU box.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/probe_multicast scripts/probe_multicast.cu -lcuda
//   ./scripts/probe_multicast [MiB]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(r_, &s_);                                               \
      std::printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s_ ? s_ : "?"); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__global__ void mc_store(unsigned long long mc, size_t n16, unsigned seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    const unsigned v = unsigned(i) * 2654435761u ^ seed;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 16 * i), "r"(v), "r"(v + 1), "r"(v + 2),
                 "r"(v + 3)
                 : "memory");
  }
}
__global__ void uc_store(uint4* p, size_t n16, unsigned seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    const unsigned v = unsigned(i) * 2654435761u ^ seed;
    p[i] = make_uint4(v, v + 1, v + 2, v + 3);
  }
}
__global__ void check(const uint4* p, size_t n16, unsigned seed, unsigned long long* bad) {
  unsigned long long b = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    const unsigned v = unsigned(i) * 2654435761u ^ seed;
    const uint4 x = p[i];
    b += (x.x != v) + (x.y != v + 1) + (x.z != v + 2) + (x.w != v + 3);
  }
  if (b) atomicAdd(bad, b);
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  int mc_ok = 0, fabric_ok = 0, sms = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&fabric_ok, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev));
  CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
  std::printf("{\"multicast_supported\": %d, \"fabric_handles\": %d, \"sms\": %d}\n", mc_ok, fabric_ok, sms);
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  if (!mc_ok) return 0;

  unsigned long long ap_handle_types = 0;
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = mib << 20;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (mp.size + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  // which handle types / team sizes does the driver accept?
  {
    const unsigned long long types[] = {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                        (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC};
    size_t gmin = 0;
    CUresult rg = cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
    std::printf("{\"granularity_recommended\": %zu, \"granularity_minimum\": %zu, \"rg\": %d}\n", gran, gmin, int(rg));
    for (unsigned long long ht : types)
      for (unsigned nd : {1u, 2u})
        for (size_t sz : {size, gmin, gran, size_t(2) << 20}) {
        CUmulticastObjectProp q = mp;
        q.handleTypes = ht, q.numDevices = nd, q.size = sz;
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &q);
        const char* es = nullptr;
        cuGetErrorString(r, &es);
        std::printf("{\"create\": {\"handle_types\": %llu, \"devices\": %u, \"size\": %zu}, \"result\": \"%s\"}\n", ht, nd, sz, es ? es : "?");
        if (r == CUDA_SUCCESS) cuMemRelease(h);
      }
  }
  mp.handleTypes = std::getenv("MC_HT") ? std::strtoull(std::getenv("MC_HT"), nullptr, 10) : 0ull;
  ap_handle_types = mp.handleTypes;
  CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));

  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CUmemAllocationHandleType(ap_handle_types);
  size_t agran = 0;
  CK(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));

  CUdeviceptr uc = 0, mcva = 0;
  CUmemAccessDesc acc{};
  acc.location = ap.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemAddressReserve(&uc, size, std::max(gran, agran), 0, 0));
  CK(cuMemMap(uc, size, 0, mem, 0));
  CK(cuMemSetAccess(uc, size, &acc, 1));
  CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CK(cuMemMap(mcva, size, 0, mc, 0));
  CK(cuMemSetAccess(mcva, size, &acc, 1));
  std::printf("{\"granularity\": %zu, \"alloc_granularity\": %zu, \"bytes\": %zu}\n", gran, agran, size);

  const size_t n16 = size / 16;
  unsigned long long* bad;
  cudaMalloc(&bad, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, int reps) {
    launch(1u);
    cudaDeviceSynchronize();
    cudaMemset(bad, 0, 8);
    check<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(uc), n16, 1u, bad);
    unsigned long long hb = 0;
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch(unsigned(r + 2));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    std::printf("{\"kernel\": \"%s\", \"mismatched_words\": %llu, \"ms_per_pass\": %.4f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
                name, hb, ms / reps, size / (ms / reps) / 1e6, cudaGetErrorString(err));
  };
  for (int blocks : {1, 2, 4}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "multimem.st x%d CTAs/SM", blocks);
    run(nm, [&](unsigned s) { mc_store<<<sms * blocks, 512>>>(mcva, n16, s); }, 10);
  }
  run("st.global (unicast, local HBM)", [&](unsigned s) { uc_store<<<sms * 4, 512>>>(reinterpret_cast<uint4*>(uc), n16, s); },
      10);
  // a plain store to the multicast address (not multimem): defined?
  run("st.global to the multicast VA", [&](unsigned s) { uc_store<<<sms * 4, 512>>>(reinterpret_cast<uint4*>(mcva), n16, s); },
      10);
  CK(cuMemUnmap(mcva, size));
  CK(cuMemUnmap(uc, size));
  CK(cuMulticastUnbind(mc, dev, 0, size));
  CK(cuMemRelease(mem));
  CK(cuMemRelease(mc));
  return 0;
}
