// Probe: which multicast-object configurations does this driver/system accept?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  cudaSetDevice(0); cudaFree(0);
  typedef CUresult (*Create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  typedef CUresult (*Gran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  typedef CUresult (*Attr)(int*, CUdevice_attribute, CUdevice);
  void *fc, *fg, *fa; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuMulticastCreate", &fc, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastGetGranularity", &fg, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fa, cudaEnableDefault, &q);
  int v = -1; ((Attr)fa)(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0); printf("MULTICAST_SUPPORTED=%d\n", v);
  ((Attr)fa)(&v, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, 0); printf("FABRIC_SUPPORTED=%d\n", v);
  ((Attr)fa)(&v, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, 0); printf("POSIX_FD_SUPPORTED=%d\n", v);
  unsigned long long types[] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int nd = 1; nd <= 2; ++nd)
    for (auto ht : types)
      for (size_t sz : {(size_t)2 << 20, (size_t)512 << 20}) {
        CUmulticastObjectProp p = {}; p.numDevices = nd; p.size = sz; p.handleTypes = ht;
        size_t g1 = 0, g2 = 0;
        CUresult r1 = ((Gran)fg)(&g1, &p, CU_MULTICAST_GRANULARITY_MINIMUM);
        CUresult r2 = ((Gran)fg)(&g2, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        CUmemGenericAllocationHandle h = 0;
        CUresult r = ((Create)fc)(&h, &p);
        printf("nd=%d ht=%llu size=%zuMB gran(min)=%d:%zu gran(rec)=%d:%zu create=%d\n", nd, ht, sz >> 20, r1, g1, r2, g2, r);
      }
  return 0;
}
