// NVLink SHARP (NVLS) buffers: one device allocation per rank bound to a multicast object that
// spans the ranks' GPUs, mapped twice — unicast (this rank's memory, ordinary loads / stores)
// and multicast (multimem.ld_reduce reads the sum over every rank's copy at that offset, reduced
// inside the NVSwitch). Driver entry points are resolved at run time (no -lcuda).
//
// Multi-process setup (seqplan_isp_nvls_*): rank 0 creates the object and exports a POSIX fd;
// every other rank duplicates that fd out of rank 0's process (pidfd_getfd) and imports it; every
// rank adds its device; after all have added (host barrier) every rank binds and maps.
#pragma once

#include <cuda.h>

#include <cstddef>
#include <string>

namespace isp {

struct Nvls {
  CUmemGenericAllocationHandle mc = 0, phys = 0;
  CUdeviceptr uc = 0, mcva = 0;
  size_t size = 0;      // bytes mapped (a multiple of the multicast granularity)
  size_t gran = 0;      // the multicast object's recommended granularity (also the VA alignment)
  int device = -1;
  int export_fd = -1;   // rank 0: the exported handle, kept open until the others hold a copy
  bool have_mc = false, bound = false;
};

// Multicast supported by the device and the driver entry points present.
bool nvls_supported(int device, std::string* why);
// rank 0: object for `ndev` GPUs of at least `bytes`; exports a POSIX fd (n.export_fd).
bool nvls_create(Nvls& n, int device, int ndev, size_t bytes, std::string* err);
// ranks != 0: the object from rank 0's fd `src_fd` in process `src_pid` (pidfd_getfd).
bool nvls_import(Nvls& n, int device, int ndev, size_t bytes, int src_pid, int src_fd, std::string* err);
// every rank, after create / import.
bool nvls_add_device(Nvls& n, std::string* err);
// every rank, after all ranks added their devices: physical memory, bind, both mappings.
bool nvls_bind(Nvls& n, std::string* err);
void nvls_release(Nvls& n);

}  // namespace isp
