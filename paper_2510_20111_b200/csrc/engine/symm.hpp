// Symmetric device memory for the multi-process engine (one process per GPU):
//
//  * every dp rank's arena is ONE cuMem allocation exported as a POSIX file
//    descriptor; peers import it (pidfd_getfd + cuMemImportFromShareableHandle)
//    and map it read/write, so the kernels see peer shards as plain device
//    pointers over NVLink 5 / NVSwitch;
//  * the AG ring of every Z3 group and the bf16 gradient ring of every Z2
//    group are additionally bound to an NVLS multicast object (created by the
//    group's first rank, fd-shared the same way): one multimem.st from the
//    owner lands in every member's AG slot, one multimem.ld_reduce at the
//    owner returns the in-switch sum of every member's gradient slot.
//
// The driver API is reached through cudaGetDriverEntryPointByVersion, so the
// library has no link-time dependency on libcuda (it still loads on a host
// without a driver for the host-only tests).
#pragma once

#include <cuda.h>

#include <cstddef>
#include <cstdint>

namespace hzp {

// Opaque record a rank publishes (over the control plane) so its peers can
// import its arena and the multicast objects it created.
struct ShareRecord {
  int32_t magic = 0;
  int32_t rank = -1;
  int32_t pid = 0;
  int32_t arena_fd = -1;
  int64_t arena_bytes = 0;
  int32_t ag_mc_fd = -1;  // group leaders only
  int32_t wg_mc_fd = -1;
  int64_t ag_mc_bytes = 0;
  int64_t wg_mc_bytes = 0;
};
constexpr int32_t kShareMagic = 0x485a5042;  // "HZPB"

// This process's exportable allocation, or an imported peer mapping.
struct SymmBuf {
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr va = 0;
  size_t bytes = 0;
  int fd = -1;  // exported fd (owner side)
};

// A multicast object bound over one region of every member's arena.
struct McGroup {
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr va = 0;  // multicast address (mapped on this device)
  size_t bytes = 0;
  int fd = -1;  // exported fd (leader only)
  bool bound = false;
  int device = -1;
};

// Allocation granularity that satisfies both cuMem and multicast binding.
size_t symm_granularity(int device);
SymmBuf symm_alloc(int device, size_t bytes);                // exportable, mapped on `device`
SymmBuf symm_import(int device, int pid, int fd, size_t bytes);  // peer arena, mapped RW on `device`
void symm_release(SymmBuf& b);

McGroup mc_create(int ndevices, size_t bytes);         // leader: create + export fd
McGroup mc_import(int pid, int fd, size_t bytes);     // member: import leader's object
// Add this device, bind [mem_offset, +bytes) of `mem` at multicast offset 0
// and map the multicast address on `device` (blocks until every member has
// added its device).
void mc_attach(McGroup& g, int device, const SymmBuf& mem, size_t mem_offset);
void mc_release(McGroup& g);

bool multicast_supported(int device);

}  // namespace hzp
