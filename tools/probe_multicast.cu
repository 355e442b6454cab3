// Probe: NVLS multicast objects on this box (one GPU): attribute, granularity,
// create + add device + bind + map, then multimem.st.global from a kernel and
// read back through the unicast mapping. Prints one line per step.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
__global__ void mc_store(double *mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double v = 1.0 + i;
    asm volatile("multimem.st.global.f64 [%0], %1;" :: "l"(mc + i), "d"(v) : "memory");
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  int fab = 0; cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handles=%d\n", mcs, fab);
  if (!mcs) return 0;
  size_t n = 1 << 20, bytes = n * 8;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.size = bytes; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, gmin = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  printf("granularity recommended=%zu minimum=%zu\n", gran, gmin);
  CUmemGenericAllocationHandle mch = 0;
  bool ok = false;
  const unsigned long long hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, 0};
  for (int nd = 1; nd <= 2 && !ok; nd++)
    for (int h = 0; h < 3 && !ok; h++)
      for (int g = 0; g < 2 && !ok; g++) {
        CUmulticastObjectProp q = {};
        q.numDevices = nd; q.handleTypes = hts[h];
        size_t gg = g ? gran : gmin;
        q.size = (bytes + gg - 1) / gg * gg;
        CUresult r = cuMulticastCreate(&mch, &q);
        const char *es; cuGetErrorString(r, &es);
        printf("create numDevices=%d handle=%llu size=%zu -> %s\n", nd, hts[h], q.size, es);
        if (r == CUDA_SUCCESS) { ok = true; mp = q; gran = gg; if (nd != 1) { printf("(needs %d devices; stop)\n", nd); return 0; } }
      }
  if (!ok) return 1;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0; ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t mg = 0; CK(cuMemGetAllocationGranularity(&mg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t sz = (mp.size + mg - 1) / mg * mg;
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, sz, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, sz, 0));
  CUdeviceptr uc, mc;
  CK(cuMemAddressReserve(&uc, sz, mg, 0, 0)); CK(cuMemMap(uc, sz, 0, ph, 0));
  CK(cuMemAddressReserve(&mc, mp.size, gran, 0, 0)); CK(cuMemMap(mc, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, sz, &ad, 1)); CK(cuMemSetAccess(mc, mp.size, &ad, 1));
  mc_store<<<(n + 255) / 256, 256>>>((double *)mc, (int)n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double h[4]; cudaMemcpy(h, (void *)(uc + 8 * 1000), sizeof(h), cudaMemcpyDeviceToHost);
  printf("readback %g %g %g %g (expect 1001..1004)\n", h[0], h[1], h[2], h[3]);
  return 0;
}
