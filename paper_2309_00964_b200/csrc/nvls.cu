// nvls.cu -- NVLS multicast buffers for the fused count exchange (include/edkm.h "NVLS").
//
// One multicast object spans the ranks' GPUs; each rank backs it with its own physical
// memory and maps two virtual ranges: the unicast view (its own copy) and the multicast view
// (a multimem reduction issued there is applied by the NVSwitch to every rank's copy).
// Driver entry points are resolved at run time through the runtime (no -lcuda link).
// Cross-process setup: rank 0 creates the object and exports a POSIX file descriptor; the
// caller passes it to the other ranks (SCM_RIGHTS over a local socket -- plumbing in
// paper_2309_00964_b200/dist.py), which import it; every rank adds its device; after a
// barrier every rank binds its memory and maps both views.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "../../include/edkm.h"

namespace {

thread_local char g_nvls_err[256] = "";

#define EDKM_DRV(name) static PFN_##name##_v12000 p_##name = nullptr;
typedef CUresult (*PFN_cuMulticastCreate_v12000)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_cuMulticastAddDevice_v12000)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_cuMulticastBindMem_v12000)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                                                 size_t, unsigned long long);
typedef CUresult (*PFN_cuMulticastUnbind_v12000)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
typedef CUresult (*PFN_cuMulticastGetGranularity_v12000)(size_t*, const CUmulticastObjectProp*,
                                                        CUmulticastGranularity_flags);
typedef CUresult (*PFN_cuMemCreate_v12000)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                                          unsigned long long);
typedef CUresult (*PFN_cuMemRelease_v12000)(CUmemGenericAllocationHandle);
typedef CUresult (*PFN_cuMemAddressReserve_v12000)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_cuMemAddressFree_v12000)(CUdeviceptr, size_t);
typedef CUresult (*PFN_cuMemMap_v12000)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_cuMemUnmap_v12000)(CUdeviceptr, size_t);
typedef CUresult (*PFN_cuMemSetAccess_v12000)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_cuMemExportToShareableHandle_v12000)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                                           unsigned long long);
typedef CUresult (*PFN_cuMemImportFromShareableHandle_v12000)(CUmemGenericAllocationHandle*, void*,
                                                             CUmemAllocationHandleType);
typedef CUresult (*PFN_cuMemGetAllocationGranularity_v12000)(size_t*, const CUmemAllocationProp*,
                                                            CUmemAllocationGranularity_flags);
typedef CUresult (*PFN_cuDeviceGetAttribute_v12000)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*PFN_cuMemGetAddressRange_v12000)(CUdeviceptr*, size_t*, CUdeviceptr);
EDKM_DRV(cuDeviceGetAttribute)
EDKM_DRV(cuMemGetAddressRange)
EDKM_DRV(cuMulticastCreate)
EDKM_DRV(cuMulticastAddDevice)
EDKM_DRV(cuMulticastBindMem)
EDKM_DRV(cuMulticastUnbind)
EDKM_DRV(cuMulticastGetGranularity)
EDKM_DRV(cuMemCreate)
EDKM_DRV(cuMemRelease)
EDKM_DRV(cuMemAddressReserve)
EDKM_DRV(cuMemAddressFree)
EDKM_DRV(cuMemMap)
EDKM_DRV(cuMemUnmap)
EDKM_DRV(cuMemSetAccess)
EDKM_DRV(cuMemExportToShareableHandle)
EDKM_DRV(cuMemImportFromShareableHandle)
EDKM_DRV(cuMemGetAllocationGranularity)

bool resolve() {
  static int state = 0;  // 0 unresolved, 1 ok, -1 failed
  if (state) return state > 0;
  bool ok = true;
#define R(name)                                                                                  \
  {                                                                                              \
    cudaDriverEntryPointQueryResult q;                                                           \
    void* f = nullptr;                                                                           \
    if (cudaGetDriverEntryPoint(#name, &f, cudaEnableDefault, &q) != cudaSuccess || !f) ok = false; \
    p_##name = reinterpret_cast<decltype(p_##name)>(f);                                          \
  }
  R(cuDeviceGetAttribute) R(cuMemGetAddressRange) R(cuMulticastCreate) R(cuMulticastAddDevice) R(cuMulticastBindMem) R(cuMulticastUnbind)
  R(cuMulticastGetGranularity) R(cuMemCreate) R(cuMemRelease) R(cuMemAddressReserve) R(cuMemAddressFree)
  R(cuMemMap) R(cuMemUnmap) R(cuMemSetAccess) R(cuMemExportToShareableHandle) R(cuMemImportFromShareableHandle)
  R(cuMemGetAllocationGranularity)
#undef R
  state = ok ? 1 : -1;
  return ok;
}

edkm_status drv_fail(CUresult r, const char* where) {
  snprintf(g_nvls_err, sizeof(g_nvls_err), "%s: CUresult %d", where, (int)r);
  return EDKM_E_CUDA;
}

}  // namespace

struct edkm_mcbuf {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uva = 0, mva = 0;
  size_t bytes = 0;
  int dev = -1;
  bool bound = false, mem_made = false;
};

extern "C" {

const char* edkm_mc_last_error(void) { return g_nvls_err; }

edkm_status edkm_mc_supported(int* supported) {
  if (!supported) return EDKM_E_ARG;
  *supported = 0;
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return EDKM_E_CUDA;
  if (!resolve()) return EDKM_OK;
  if (p_cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)dev) != CUDA_SUCCESS) return EDKM_E_CUDA;
  *supported = v != 0;
  return EDKM_OK;
}

edkm_status edkm_mc_create(size_t bytes, int nranks, int export_fd, int* fd_out, edkm_mcbuf** out) {
  if (!out || nranks < 1 || bytes == 0 || (export_fd && !fd_out)) return EDKM_E_ARG;
  if (!resolve()) return EDKM_E_UNSUPPORTED;
  CUmulticastObjectProp prop = {};
  prop.numDevices = (unsigned)nranks;
  prop.handleTypes = export_fd ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  size_t g = 0;
  prop.size = bytes;
  CUresult r = p_cuMulticastGetGranularity(&g, &prop, CU_MULTICAST_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuMulticastGetGranularity");
  prop.size = (bytes + g - 1) / g * g;
  edkm_mcbuf* b = new edkm_mcbuf;
  b->bytes = prop.size;
  r = p_cuMulticastCreate(&b->mc, &prop);
  if (r != CUDA_SUCCESS) { delete b; return drv_fail(r, "cuMulticastCreate"); }
  if (export_fd) {
    int fd = -1;
    r = p_cuMemExportToShareableHandle(&fd, b->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) { p_cuMemRelease(b->mc); delete b; return drv_fail(r, "cuMemExportToShareableHandle"); }
    *fd_out = fd;
  }
  *out = b;
  return EDKM_OK;
}

edkm_status edkm_mc_import(int fd, size_t bytes, edkm_mcbuf** out) {
  if (!out || fd < 0 || bytes == 0) return EDKM_E_ARG;
  if (!resolve()) return EDKM_E_UNSUPPORTED;
  edkm_mcbuf* b = new edkm_mcbuf;
  b->bytes = bytes;
  CUresult r = p_cuMemImportFromShareableHandle(&b->mc, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) { delete b; return drv_fail(r, "cuMemImportFromShareableHandle"); }
  *out = b;
  return EDKM_OK;
}

size_t edkm_mc_bytes(const edkm_mcbuf* b) { return b ? b->bytes : 0; }

edkm_status edkm_mc_add_device(edkm_mcbuf* b) {
  if (!b) return EDKM_E_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return EDKM_E_CUDA;
  b->dev = dev;
  CUresult r = p_cuMulticastAddDevice(b->mc, (CUdevice)dev);
  return r == CUDA_SUCCESS ? EDKM_OK : drv_fail(r, "cuMulticastAddDevice");
}

edkm_status edkm_mc_bind(edkm_mcbuf* b, void** local_out, void** mc_out) {
  if (!b || !local_out || !mc_out || b->dev < 0) return EDKM_E_ARG;
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = b->dev;
  size_t g = 0;
  CUresult r = p_cuMemGetAllocationGranularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemGetAllocationGranularity");
  if (b->bytes % g) return drv_fail(CUDA_ERROR_INVALID_VALUE, "multicast size vs allocation granularity");
  r = p_cuMemCreate(&b->mem, b->bytes, &ap, 0);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemCreate");
  b->mem_made = true;
  r = p_cuMulticastBindMem(b->mc, 0, b->mem, 0, b->bytes, 0);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuMulticastBindMem");
  b->bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = b->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = p_cuMemAddressReserve(&b->uva, b->bytes, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = p_cuMemMap(b->uva, b->bytes, 0, b->mem, 0);
  if (r == CUDA_SUCCESS) r = p_cuMemSetAccess(b->uva, b->bytes, &acc, 1);
  if (r != CUDA_SUCCESS) return drv_fail(r, "map unicast view");
  r = p_cuMemAddressReserve(&b->mva, b->bytes, 0, 0, 0);
  if (r == CUDA_SUCCESS) r = p_cuMemMap(b->mva, b->bytes, 0, b->mc, 0);
  if (r == CUDA_SUCCESS) r = p_cuMemSetAccess(b->mva, b->bytes, &acc, 1);
  if (r != CUDA_SUCCESS) return drv_fail(r, "map multicast view");
  *local_out = (void*)b->uva;
  *mc_out = (void*)b->mva;
  return EDKM_OK;
}

// CUDA IPC plumbing of the NVLS protocol's emulation with a real second writer (edkm_nvls.peer_delta):
// another process's device buffer mapped into this one (runtime API; no compute).
edkm_status edkm_ipc_handle(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return EDKM_E_ARG;
  // the handle maps the whole allocation: dev_ptr's offset in it (a caching allocator sub-allocates)
  if (!resolve()) {
    snprintf(g_nvls_err, sizeof(g_nvls_err), "CUDA driver entry points unavailable");
    return EDKM_E_CUDA;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  const CUresult r = p_cuMemGetAddressRange(&base, &size, (CUdeviceptr)dev_ptr);
  if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemGetAddressRange");
  *offset_out = (size_t)((CUdeviceptr)dev_ptr - base);
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) {
    snprintf(g_nvls_err, sizeof(g_nvls_err), "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return EDKM_E_CUDA;
  }
  memcpy(handle_out, &h, sizeof(h));
  return EDKM_OK;
}

edkm_status edkm_ipc_open(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return EDKM_E_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    snprintf(g_nvls_err, sizeof(g_nvls_err), "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return EDKM_E_CUDA;
  }
  return EDKM_OK;
}

edkm_status edkm_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return EDKM_OK;
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? EDKM_OK : EDKM_E_CUDA;
}

edkm_status edkm_mc_destroy(edkm_mcbuf* b) {
  if (!b) return EDKM_OK;
  if (b->mva) { p_cuMemUnmap(b->mva, b->bytes); p_cuMemAddressFree(b->mva, b->bytes); }
  if (b->uva) { p_cuMemUnmap(b->uva, b->bytes); p_cuMemAddressFree(b->uva, b->bytes); }
  if (b->bound) p_cuMulticastUnbind(b->mc, (CUdevice)b->dev, 0, b->bytes);
  if (b->mem_made) p_cuMemRelease(b->mem);
  if (b->mc) p_cuMemRelease(b->mc);
  delete b;
  return EDKM_OK;
}

}  // extern "C"
