// Which physical-allocation / granularity variants cuMulticastBindMem accepts
// on this box (2+ GPUs): prints one JSON line per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o nvls_bind_matrix tools/nvls_bind_matrix.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
int main() {
  cuInit(0);
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  for (int d = 0; d < ndev; d++) { cudaSetDevice(d); cudaFree(0); }
  const size_t want = 5ull << 20;
  for (int gflag = 0; gflag < 2; gflag++)
    for (int ht = 0; ht < 2; ht++) {
      CUmulticastObjectProp mp = {};
      mp.numDevices = ndev;
      mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      mp.size = want;
      size_t g = 0, ga = 0;
      cuMulticastGetGranularity(&g, &mp, gflag ? CU_MULTICAST_GRANULARITY_RECOMMENDED : CU_MULTICAST_GRANULARITY_MINIMUM);
      CUmemAllocationProp ap = {};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = 0;
      ap.requestedHandleTypes = ht ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
      cuMemGetAllocationGranularity(&ga, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
      size_t gg = g > ga ? g : ga;
      size_t size = (want + gg - 1) / gg * gg;
      mp.size = size;
      CUmemGenericAllocationHandle mc;
      CUresult r0 = cuMulticastCreate(&mc, &mp), r1 = CUDA_SUCCESS, r2 = CUDA_SUCCESS;
      for (int d = 0; d < ndev && r0 == CUDA_SUCCESS && r1 == CUDA_SUCCESS; d++) {
        CUdevice dv; cuDeviceGet(&dv, d);
        r1 = cuMulticastAddDevice(mc, dv);
      }
      for (int d = 0; d < ndev && r0 == CUDA_SUCCESS && r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS; d++) {
        cudaSetDevice(d);
        ap.location.id = d;
        CUmemGenericAllocationHandle ph;
        r2 = cuMemCreate(&ph, size, &ap, 0);
        if (r2 == CUDA_SUCCESS) r2 = cuMulticastBindMem(mc, 0, ph, 0, size, 0);
      }
      printf("{\"gran\": \"%s\", \"mc_gran\": %zu, \"alloc_gran\": %zu, \"size\": %zu, \"handle\": \"%s\", \"create\": %d, \"add\": %d, \"bind\": %d}\n",
             gflag ? "recommended" : "minimum", g, ga, size, ht ? "fd" : "none", (int)r0, (int)r1, (int)r2);
    }
  return 0;
}
