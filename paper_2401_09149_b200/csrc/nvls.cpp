// NVLS buffers (nvls.h): multicast object + per-rank bound device memory, unicast and multicast
// mappings. The driver functions are resolved with cudaGetDriverEntryPoint, as the memop
// barriers are (isp_block.cpp memops()).
#include "nvls.h"

#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstdint>
#include <cstring>

namespace isp {
namespace {

struct DriverFns {
  CUresult (*mc_granularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mc_create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mc_add_device)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mc_bind_mem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long) = nullptr;
  CUresult (*mc_unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*export_handle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long) =
      nullptr;
  CUresult (*import_handle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*alloc_granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*free_va)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*get_error_string)(CUresult, const char**) = nullptr;
  CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  bool ok = false;
};

template <typename F>
bool resolve(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const DriverFns& fns() {
  static DriverFns d = [] {
    DriverFns r;
    r.ok = resolve("cuMulticastGetGranularity", r.mc_granularity) && resolve("cuMulticastCreate", r.mc_create) &&
           resolve("cuMulticastAddDevice", r.mc_add_device) && resolve("cuMulticastBindMem", r.mc_bind_mem) &&
           resolve("cuMulticastUnbind", r.mc_unbind) && resolve("cuMemExportToShareableHandle", r.export_handle) &&
           resolve("cuMemImportFromShareableHandle", r.import_handle) &&
           resolve("cuMemGetAllocationGranularity", r.alloc_granularity) && resolve("cuMemCreate", r.create) &&
           resolve("cuMemRelease", r.release) && resolve("cuMemAddressReserve", r.reserve) &&
           resolve("cuMemAddressFree", r.free_va) && resolve("cuMemMap", r.map) && resolve("cuMemUnmap", r.unmap) &&
           resolve("cuMemSetAccess", r.set_access) && resolve("cuGetErrorString", r.get_error_string) &&
           resolve("cuDeviceGetAttribute", r.dev_attr);
    return r;
  }();
  return d;
}

bool check(CUresult r, const char* what, std::string* err) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = nullptr;
  if (fns().get_error_string) fns().get_error_string(r, &s);
  if (err) *err = std::string(what) + ": " + (s ? s : "CUDA driver error");
  return false;
}

CUmulticastObjectProp mc_prop(int ndev, size_t bytes) {
  CUmulticastObjectProp p;
  std::memset(&p, 0, sizeof(p));
  p.numDevices = static_cast<unsigned>(ndev);
  p.size = bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

// Size rounded up to the multicast object's recommended granularity.
bool rounded_size(int ndev, size_t bytes, size_t* out, size_t* gran, std::string* err) {
  CUmulticastObjectProp p = mc_prop(ndev, bytes);
  size_t g = 0;
  if (!check(fns().mc_granularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity", err))
    return false;
  *out = (bytes + g - 1) / g * g;
  *gran = g;
  return true;
}

}  // namespace

bool nvls_supported(int device, std::string* why) {
  if (!fns().ok) {
    if (why) *why = "multicast driver entry points unavailable";
    return false;
  }
  int v = 0;
  if (fns().dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, static_cast<CUdevice>(device)) != CUDA_SUCCESS ||
      !v) {
    if (why) *why = "device reports no multicast (NVLS) support";
    return false;
  }
  return true;
}

bool nvls_create(Nvls& n, int device, int ndev, size_t bytes, std::string* err) {
  if (!nvls_supported(device, err)) return false;
  n.device = device;
  if (!rounded_size(ndev, bytes, &n.size, &n.gran, err)) return false;
  CUmulticastObjectProp p = mc_prop(ndev, n.size);
  if (!check(fns().mc_create(&n.mc, &p), "cuMulticastCreate", err)) return false;
  n.have_mc = true;
  int fd = -1;
  if (!check(fns().export_handle(&fd, n.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle", err))
    return false;
  n.export_fd = fd;
  return true;
}

bool nvls_import(Nvls& n, int device, int ndev, size_t bytes, int src_pid, int src_fd, std::string* err) {
  if (!nvls_supported(device, err)) return false;
  n.device = device;
  if (!rounded_size(ndev, bytes, &n.size, &n.gran, err)) return false;
  const long pfd = syscall(SYS_pidfd_open, src_pid, 0);
  const long fd = pfd >= 0 ? syscall(SYS_pidfd_getfd, pfd, src_fd, 0) : -1;
  const int e = errno;
  if (pfd >= 0) close(static_cast<int>(pfd));
  if (fd < 0) {
    if (err) *err = std::string("pidfd_getfd of the multicast handle: ") + std::strerror(e);
    return false;
  }
  const bool ok = check(fns().import_handle(&n.mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                        "cuMemImportFromShareableHandle", err);
  close(static_cast<int>(fd));
  n.have_mc = ok;
  return ok;
}

bool nvls_add_device(Nvls& n, std::string* err) {
  return check(fns().mc_add_device(n.mc, static_cast<CUdevice>(n.device)), "cuMulticastAddDevice", err);
}

bool nvls_bind(Nvls& n, std::string* err) {
  CUmemAllocationProp ap;
  std::memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = n.device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  if (!check(fns().create(&n.phys, n.size, &ap, 0), "cuMemCreate", err)) return false;
  if (!check(fns().mc_bind_mem(n.mc, 0, n.phys, 0, n.size, 0), "cuMulticastBindMem", err)) return false;
  CUmemAccessDesc acc;
  std::memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = n.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!check(fns().reserve(&n.uc, n.size, n.gran, 0, 0), "cuMemAddressReserve", err) ||
      !check(fns().map(n.uc, n.size, 0, n.phys, 0), "cuMemMap (unicast)", err) ||
      !check(fns().set_access(n.uc, n.size, &acc, 1), "cuMemSetAccess (unicast)", err) ||
      !check(fns().reserve(&n.mcva, n.size, n.gran, 0, 0), "cuMemAddressReserve", err) ||
      !check(fns().map(n.mcva, n.size, 0, n.mc, 0), "cuMemMap (multicast)", err) ||
      !check(fns().set_access(n.mcva, n.size, &acc, 1), "cuMemSetAccess (multicast)", err))
    return false;
  n.bound = true;
  if (n.export_fd >= 0) {  // every rank holds its own handle by now
    close(n.export_fd);
    n.export_fd = -1;
  }
  return true;
}

void nvls_release(Nvls& n) {
  if (!fns().ok) return;
  if (n.mcva) {
    fns().unmap(n.mcva, n.size);
    fns().free_va(n.mcva, n.size);
  }
  if (n.uc) {
    fns().unmap(n.uc, n.size);
    fns().free_va(n.uc, n.size);
  }
  if (n.bound) fns().mc_unbind(n.mc, static_cast<CUdevice>(n.device), 0, n.size);
  if (n.phys) fns().release(n.phys);
  if (n.have_mc) fns().release(n.mc);
  if (n.export_fd >= 0) close(n.export_fd);
  n = Nvls{};
}

}  // namespace isp
