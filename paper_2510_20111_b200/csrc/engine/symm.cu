// Symmetric device memory + NVLS multicast (see symm.hpp).
#include "engine/symm.hpp"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <string>

#include "engine/common.cuh"

namespace hzp {
namespace {

// Driver entry points resolved once through the runtime (no -lcuda).
struct Driver {
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemRelease_v10020 release = nullptr;
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemAddressFree_v10020 free_va = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 set_access = nullptr;
  PFN_cuMemExportToShareableHandle_v10020 export_h = nullptr;
  PFN_cuMemImportFromShareableHandle_v10020 import_h = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 granularity = nullptr;
  PFN_cuMulticastCreate_v12010 mc_create = nullptr;
  PFN_cuMulticastAddDevice_v12010 mc_add = nullptr;
  PFN_cuMulticastBindMem_v12010 mc_bind = nullptr;
  PFN_cuMulticastUnbind_v12010 mc_unbind = nullptr;
  PFN_cuMulticastGetGranularity_v12010 mc_granularity = nullptr;
  PFN_cuDeviceGet_v2000 device_get = nullptr;
  PFN_cuDeviceGetAttribute_v2000 attribute = nullptr;
  PFN_cuGetErrorString_v6000 error_string = nullptr;

  template <typename F>
  void resolve(F& f, const char* name, unsigned version) {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    HZP_CUDA(cudaGetDriverEntryPointByVersion(name, &p, version, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError(std::string("driver entry point missing: ") + name);
    f = reinterpret_cast<F>(p);
  }
  Driver() {
    resolve(create, "cuMemCreate", 10020);
    resolve(release, "cuMemRelease", 10020);
    resolve(reserve, "cuMemAddressReserve", 10020);
    resolve(free_va, "cuMemAddressFree", 10020);
    resolve(map, "cuMemMap", 10020);
    resolve(unmap, "cuMemUnmap", 10020);
    resolve(set_access, "cuMemSetAccess", 10020);
    resolve(export_h, "cuMemExportToShareableHandle", 10020);
    resolve(import_h, "cuMemImportFromShareableHandle", 10020);
    resolve(granularity, "cuMemGetAllocationGranularity", 10020);
    resolve(mc_create, "cuMulticastCreate", 12010);
    resolve(mc_add, "cuMulticastAddDevice", 12010);
    resolve(mc_bind, "cuMulticastBindMem", 12010);
    resolve(mc_unbind, "cuMulticastUnbind", 12010);
    resolve(mc_granularity, "cuMulticastGetGranularity", 12010);
    resolve(device_get, "cuDeviceGet", 2000);
    resolve(attribute, "cuDeviceGetAttribute", 2000);
    resolve(error_string, "cuGetErrorString", 6000);
  }
};

Driver& drv() {
  static Driver d;
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  drv().error_string(r, &s);
  throw CudaError(std::string(what) + ": " + (s ? s : "unknown driver error"));
}
#define HZP_CU(call) cu_check((call), #call)

CUmemAllocationProp alloc_prop(int device) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

CUdeviceptr map_rw(CUmemGenericAllocationHandle h, size_t bytes, int device) {
  CUdeviceptr va = 0;
  HZP_CU(drv().reserve(&va, bytes, symm_granularity(device), 0, 0));
  HZP_CU(drv().map(va, bytes, 0, h, 0));
  CUmemAccessDesc a{};
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = device;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  HZP_CU(drv().set_access(va, bytes, &a, 1));
  return va;
}

// A descriptor of another process (a sibling under torchrun) duplicated into
// this one.
int dup_remote_fd(int pid, int fd) {
  const int pfd = static_cast<int>(syscall(SYS_pidfd_open, pid, 0));
  if (pfd < 0) throw CudaError("pidfd_open(" + std::to_string(pid) + "): " + std::strerror(errno));
  const int local = static_cast<int>(syscall(SYS_pidfd_getfd, pfd, fd, 0));
  const int err = errno;
  close(pfd);
  if (local < 0) throw CudaError("pidfd_getfd: " + std::string(std::strerror(err)));
  return local;
}

CUmemGenericAllocationHandle import_fd(int pid, int fd) {
  const int local = dup_remote_fd(pid, fd);
  CUmemGenericAllocationHandle h = 0;
  const CUresult r = drv().import_h(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(local)),
                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  cu_check(r, "cuMemImportFromShareableHandle");
  return h;
}

}  // namespace

bool multicast_supported(int device) {
  CUdevice d = 0;
  HZP_CU(drv().device_get(&d, device));
  int v = 0;
  HZP_CU(drv().attribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  return v != 0;
}

size_t symm_granularity(int device) {
  static size_t g = 0;
  if (g) return g;
  CUmemAllocationProp p = alloc_prop(device);
  size_t a = 0;
  HZP_CU(drv().granularity(&a, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.size = a;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t m = 0;
  if (drv().mc_granularity(&m, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) m = a;
  g = a > m ? a : m;
  return g;
}

SymmBuf symm_alloc(int device, size_t bytes) {
  SymmBuf b;
  const size_t gr = symm_granularity(device);
  b.bytes = (bytes + gr - 1) / gr * gr;
  CUmemAllocationProp p = alloc_prop(device);
  HZP_CU(drv().create(&b.handle, b.bytes, &p, 0));
  b.va = map_rw(b.handle, b.bytes, device);
  int fd = -1;
  HZP_CU(drv().export_h(&fd, b.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  b.fd = fd;
  return b;
}

SymmBuf symm_import(int device, int pid, int fd, size_t bytes) {
  SymmBuf b;
  b.bytes = bytes;
  b.handle = import_fd(pid, fd);
  b.va = map_rw(b.handle, bytes, device);
  return b;
}

void symm_release(SymmBuf& b) {
  if (b.va) {
    drv().unmap(b.va, b.bytes);
    drv().free_va(b.va, b.bytes);
  }
  if (b.handle) drv().release(b.handle);
  if (b.fd >= 0) close(b.fd);
  b = SymmBuf{};
}

McGroup mc_create(int ndevices, size_t bytes) {
  McGroup g;
  CUmulticastObjectProp mp{};
  mp.numDevices = static_cast<unsigned>(ndevices);
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  HZP_CU(drv().mc_create(&g.handle, &mp));
  g.bytes = bytes;
  int fd = -1;
  HZP_CU(drv().export_h(&fd, g.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  g.fd = fd;
  return g;
}

McGroup mc_import(int pid, int fd, size_t bytes) {
  McGroup g;
  g.handle = import_fd(pid, fd);
  g.bytes = bytes;
  return g;
}

void mc_attach(McGroup& g, int device, const SymmBuf& mem, size_t mem_offset) {
  CUdevice d = 0;
  HZP_CU(drv().device_get(&d, device));
  HZP_CU(drv().mc_add(g.handle, d));
  HZP_CU(drv().mc_bind(g.handle, 0, mem.handle, mem_offset, g.bytes, 0));
  g.bound = true;
  g.device = device;
  g.va = map_rw(g.handle, g.bytes, device);
}

void mc_release(McGroup& g) {
  if (g.va) {
    drv().unmap(g.va, g.bytes);
    drv().free_va(g.va, g.bytes);
  }
  if (g.bound) {
    CUdevice d = 0;
    if (drv().device_get(&d, g.device) == CUDA_SUCCESS) drv().mc_unbind(g.handle, d, 0, g.bytes);
  }
  if (g.handle) drv().release(g.handle);
  if (g.fd >= 0) close(g.fd);
  g = McGroup{};
}

}  // namespace hzp
