// Probe: NVLS multicast support on this GPU (cuMulticast* with one device).
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  CUdevice d; cuDeviceGet(&d, 0);
  int mc = -1, fab = -1, vmm = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
  cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
  printf("multicast_supported=%d vmm=%d fabric=%d\n", mc, vmm, fab);
  CUcontext ctx; cuCtxCreate(&ctx, 0, d);
  CUmulticastObjectProp p = {};
  p.numDevices = 1; p.size = 2 << 20; p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CUresult r0 = cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  printf("granularity rc=%d gran=%zu\n", (int)r0, gran);
  CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int v = 0; v < 3; ++v) {
    CUmulticastObjectProp q = p;
    q.handleTypes = hts[v];
    CUmemGenericAllocationHandle mh;
    CUresult r1 = cuMulticastCreate(&mh, &q);
    printf("cuMulticastCreate handleType=%d rc=%d\n", (int)hts[v], (int)r1);
    if (r1 != CUDA_SUCCESS) continue;
    CUresult r2 = cuMulticastAddDevice(mh, d);
    printf("  AddDevice rc=%d\n", (int)r2);
    // physical memory, bind, map, and a multimem access
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = hts[v];
    CUmemGenericAllocationHandle ph;
    CUresult r3 = cuMemCreate(&ph, q.size, &ap, 0);
    CUresult r4 = cuMulticastBindMem(mh, 0, ph, 0, q.size, 0);
    CUdeviceptr mcp = 0;
    CUresult r5 = cuMemAddressReserve(&mcp, q.size, gran, 0, 0);
    CUresult r6 = cuMemMap(mcp, q.size, 0, mh, 0);
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUresult r7 = cuMemSetAccess(mcp, q.size, &ad, 1);
    printf("  memCreate %d bind %d reserve %d map %d access %d\n", (int)r3, (int)r4, (int)r5, (int)r6, (int)r7);
    break;
  }
  return 0;
}
