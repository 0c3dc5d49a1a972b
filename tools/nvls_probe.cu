// nvls_probe.cu — feasibility + bandwidth probe of NVLink SHARP multicast
// (NVLS) on this box: one process, N GPUs.  Creates a multicast object over
// the N devices, binds a per-device physical allocation, maps the multicast
// address on device 0 and stores into it with multimem.st (one store stream,
// the switch replicates it to every device); checks that every device's
// buffer holds the data and times the store stream against a plain peer-store
// loop to each device.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

#define CU(x)                                                                     \
  do {                                                                            \
    CUresult r = (x);                                                             \
    if (r != CUDA_SUCCESS) {                                                      \
      const char* s = nullptr;                                                    \
      cuGetErrorString(r, &s);                                                    \
      printf("{\"ok\": false, \"where\": \"%s\", \"err\": \"%s\"}\n", #x, s ? s : "?"); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)
#define CR(x)                                                                     \
  do {                                                                            \
    cudaError_t r = (x);                                                          \
    if (r != cudaSuccess) {                                                       \
      printf("{\"ok\": false, \"where\": \"%s\", \"err\": \"%s\"}\n", #x, cudaGetErrorString(r)); \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

__global__ void mc_store(float4* mc, size_t n4, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i & 1023);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(v), "f"(v), "f"(v), "f"(v)
                 : "memory");
  }
}
__global__ void peer_store(float4* const* dst, int ndst, size_t n4, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i & 1023);
    for (int d = 0; d < ndst; d++) dst[d][i] = make_float4(v, v, v, v);
  }
}
__global__ void check(const float4* p, size_t n4, float base, unsigned int* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i & 1023);
    const float4 x = p[i];
    if (x.x != v || x.y != v || x.z != v || x.w != v) atomicAdd(bad, 1u);
  }
}

int main(int argc, char** argv) {
  const size_t bytes = (argc > 1 ? atoll(argv[1]) : 64ll) << 20;
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  CU(cuInit(0));
  std::vector<CUdevice> devs(ndev);
  int mc_ok = 1;
  for (int d = 0; d < ndev; d++) {
    CU(cuDeviceGet(&devs[d], d));
    int a = 0;
    CU(cuDeviceGetAttribute(&a, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, devs[d]));
    mc_ok &= a;
  }
  if (ndev < 2 || !mc_ok) {
    printf("{\"ok\": false, \"ndev\": %d, \"multicast_supported\": %d}\n", ndev, mc_ok);
    return 0;
  }
  for (int d = 0; d < ndev; d++) {
    CR(cudaSetDevice(d));
    CR(cudaFree(0));
  }
  CUmulticastObjectProp mp = {};
  mp.numDevices = ndev;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = bytes;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (bytes + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < ndev; d++) CU(cuMulticastAddDevice(mc, devs[d]));
  std::vector<CUdeviceptr> uc(ndev);
  std::vector<CUmemGenericAllocationHandle> ph(ndev);
  for (int d = 0; d < ndev; d++) {
    CR(cudaSetDevice(d));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CU(cuMemCreate(&ph[d], size, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, ph[d], 0, size, 0));
    CU(cuMemAddressReserve(&uc[d], size, gran, 0, 0));
    CU(cuMemMap(uc[d], size, 0, ph[d], 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(uc[d], size, &ad, 1));
  }
  CR(cudaSetDevice(0));
  CUdeviceptr mcva;
  CU(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CU(cuMemMap(mcva, size, 0, mc, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(mcva, size, &ad, 1));
  const size_t n4 = size / 16;
  cudaEvent_t e0, e1;
  CR(cudaEventCreate(&e0));
  CR(cudaEventCreate(&e1));
  float ms_mc = 0, ms_peer = 0;
  for (int it = 0; it < 6; it++) {
    CR(cudaEventRecord(e0));
    mc_store<<<2 * 148, 512>>>(reinterpret_cast<float4*>(mcva), n4, 1.0f + it);
    CR(cudaEventRecord(e1));
    CR(cudaEventSynchronize(e1));
    CR(cudaGetLastError());
    if (it >= 2) {
      float m;
      CR(cudaEventElapsedTime(&m, e0, e1));
      ms_mc += m / 4;
    }
  }
  // every device holds the last pattern (base 6)
  unsigned int bad_total = 0;
  for (int d = 0; d < ndev; d++) {
    CR(cudaSetDevice(d));
    unsigned int* bad;
    CR(cudaMalloc(&bad, 4));
    CR(cudaMemset(bad, 0, 4));
    check<<<296, 512>>>(reinterpret_cast<const float4*>(uc[d]), n4, 6.0f, bad);
    unsigned int h = 0;
    CR(cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost));
    bad_total += h;
    CR(cudaFree(bad));
  }
  // the same bytes to every other device by peer stores from device 0 (the
  // unicast addresses of the same allocations, mapped on device 0)
  CR(cudaSetDevice(0));
  for (int d = 1; d < ndev; d++) {
    int can = 0;
    CR(cudaDeviceCanAccessPeer(&can, 0, d));
    if (can) cudaDeviceEnablePeerAccess(d, 0);
    (void)cudaGetLastError();
  }
  std::vector<float4*> dsth;
  for (int d = 1; d < ndev; d++) {
    CUmemAccessDesc a2 = {};
    a2.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a2.location.id = 0;
    a2.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(uc[d], size, &a2, 1));
    dsth.push_back(reinterpret_cast<float4*>(uc[d]));
  }
  float4** dstd;
  CR(cudaMalloc(&dstd, sizeof(float4*) * dsth.size()));
  CR(cudaMemcpy(dstd, dsth.data(), sizeof(float4*) * dsth.size(), cudaMemcpyHostToDevice));
  for (int it = 0; it < 6; it++) {
    CR(cudaEventRecord(e0));
    peer_store<<<2 * 148, 512>>>(dstd, (int)dsth.size(), n4, 1.0f + it);
    CR(cudaEventRecord(e1));
    CR(cudaEventSynchronize(e1));
    CR(cudaGetLastError());
    if (it >= 2) {
      float m;
      CR(cudaEventElapsedTime(&m, e0, e1));
      ms_peer += m / 4;
    }
  }
  printf("{\"ok\": %s, \"ndev\": %d, \"bytes\": %zu, \"bad\": %u, \"multimem_st_ms\": %.4f, "
         "\"multimem_st_GBps_per_dest\": %.1f, \"peer_st_ms\": %.4f, \"peer_st_GBps_per_dest\": %.1f}\n",
         bad_total == 0 ? "true" : "false", ndev, size, bad_total, ms_mc, size / (ms_mc * 1e-3) / 1e9, ms_peer,
         size / (ms_peer * 1e-3) / 1e9);
  return 0;
}
