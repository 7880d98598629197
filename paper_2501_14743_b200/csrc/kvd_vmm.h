// kvd_vmm.h -- internal: exportable cache memory (SURVEY §8 f3 groundwork).
//
// Caches allocated with kvd_mem_alloc are CUDA VMM allocations (cuMemCreate)
// whose physical handle is exported as a POSIX fd (intra-node) or a fabric
// handle (multi-node NVLink through IMEX, the cross-node setting of P:L102,
// P:L457).  The export blob carries one ExportRec per allocation; the
// importer maps the same physical memory into its own VA.  The pull kernel
// does not change: it only ever sees a mapped base address.
#pragma once

#include <cstdint>
#include <string>

namespace kvd {
namespace vmm {

enum Kind : uint32_t {
  kLegacyIpc = 0,   // cudaIpcGetMemHandle (cudaMalloc memory)
  kPosixFd = 1,     // CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
  kFabric = 8,      // CU_MEM_HANDLE_TYPE_FABRIC
};

struct ExportRec {
  uint32_t kind = kLegacyIpc;
  uint32_t fd = 0;                 // kPosixFd: the exporter's fd number
  unsigned char payload[64] = {};  // kLegacyIpc: cudaIpcMemHandle_t; kFabric: CUmemFabricHandle
};

// Allocate `bytes` rounded up to the granularity on `device`; kind 0 = fabric
// when permitted, else POSIX fd.  Returns 0 or a kvd_status, *err set.
int alloc(int device, uint64_t bytes, uint32_t kind, void** ptr, uint64_t* size,
          uint32_t* kind_out, std::string* err);
int free(void* ptr, std::string* err);

// If [base, base+size) is a kvd_mem allocation: fill *rec (exporting its
// shareable handle once) and return 1; 0 if it is not; <0 (a kvd_status) on error.
int lookup_export(uint64_t base, uint64_t* size, ExportRec* rec, std::string* err);

// If addr lies inside a kvd_mem allocation: its base and size, return 1; else 0.
int find(uint64_t addr, uint64_t* base, uint64_t* size);

// Same-process import of a kvd_mem allocation on another device: grant
// `device` read/write access to the range (VMM memory ignores peer access).
int grant_access(uint64_t base, int device, std::string* err);

// Map an exported VMM allocation of `size` bytes (exported by process `pid`)
// on `device`.  Returns 0 or a kvd_status.
int import_map(const ExportRec& rec, int64_t pid, uint64_t size, int device, void** va,
               std::string* err);
void unmap(void* va, uint64_t size);

}  // namespace vmm
}  // namespace kvd
