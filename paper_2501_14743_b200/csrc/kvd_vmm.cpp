// kvd_vmm.cpp -- exportable cache memory through CUDA virtual memory
// management (SURVEY §8 f3 groundwork; interface in kvd_vmm.h).
//
// The paper's decode side reads the prefill cache across nodes over RDMA
// (P:L102).  On NVLink hardware the cross-node equivalent is a VMM
// allocation exported as a FABRIC handle (multi-node NVLink, IMEX): the
// importer maps the remote physical memory into its own address space and the
// same pull kernel reads it.  Inside one node the same allocation exports as
// a POSIX fd, which the importer fetches from the exporter with pidfd_getfd
// (Linux >= 5.6, same user) -- no socket, the blob stays plain bytes.
// Legacy cudaIpc handles (kvd_core.cpp) remain the path for cudaMalloc memory.
#include "kvd_vmm.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>

#include "../../include/kvd.h"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace kvd {
namespace vmm {
namespace {

struct Api {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuGetErrorName) error_name = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Api& api() {
  static const Api a = [] {
    Api x;
    x.ok = entry("cuMemCreate", &x.create) && entry("cuMemRelease", &x.release) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemAddressFree", &x.addr_free) &&
           entry("cuMemMap", &x.map) && entry("cuMemUnmap", &x.unmap) &&
           entry("cuMemSetAccess", &x.set_access) &&
           entry("cuMemExportToShareableHandle", &x.export_handle) &&
           entry("cuMemImportFromShareableHandle", &x.import_handle) &&
           entry("cuMemGetAllocationGranularity", &x.granularity) &&
           entry("cuGetErrorName", &x.error_name);
    return x;
  }();
  return a;
}

std::string cu_msg(const char* what, CUresult r) {
  const char* name = nullptr;
  if (api().error_name) api().error_name(r, &name);
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s (%d)", what, name ? name : "?", (int)r);
  return buf;
}

int cu_status(CUresult r) {
  return r == CUDA_ERROR_OUT_OF_MEMORY ? KVD_ENOMEM
         : (r == CUDA_ERROR_NOT_PERMITTED || r == CUDA_ERROR_NOT_SUPPORTED) ? KVD_EHANDLE
                                                                           : KVD_ECUDA;
}

CUmemAllocationProp prop_for(int device, uint32_t kind) {
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = (CUmemAllocationHandleType)kind;
  return p;
}

CUmemAccessDesc rw(int device) {
  CUmemAccessDesc d;
  memset(&d, 0, sizeof(d));
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.location.id = device;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return d;
}

struct Alloc {
  CUmemGenericAllocationHandle handle = 0;
  uint64_t size = 0;
  int device = -1;
  uint32_t kind = 0;
  bool exported = false;
  ExportRec rec;
};
std::mutex g_mu;
std::map<uint64_t, Alloc> g_allocs;   // VA -> allocation (this process's kvd_mem_alloc)

bool ready(std::string* err) {
  if (api().ok) return true;
  *err = "CUDA virtual memory management entry points unavailable";
  return false;
}

}  // namespace

int alloc(int device, uint64_t bytes, uint32_t kind, void** ptr, uint64_t* size,
          uint32_t* kind_out, std::string* err) {
  if (!ready(err)) return KVD_ECUDA;
  if (cudaFree(nullptr) != cudaSuccess) {   // the primary context must exist
    cudaGetLastError();
    *err = "cannot initialise the device context";
    return KVD_ECUDA;
  }
  const Api& A = api();
  const uint32_t kinds[2] = {kind == 0 ? (uint32_t)kFabric : kind, (uint32_t)kPosixFd};
  const int tries = kind == 0 ? 2 : 1;
  CUresult r = CUDA_SUCCESS;
  for (int t = 0; t < tries; ++t) {
    const uint32_t k = kinds[t];
    CUmemAllocationProp prop = prop_for(device, k);
    size_t gran = 0;
    r = A.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemGetAllocationGranularity", r); continue; }
    const uint64_t sz = (bytes + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h = 0;
    r = A.create(&h, sz, &prop, 0);
    if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemCreate", r); continue; }
    CUdeviceptr va = 0;
    r = A.reserve(&va, sz, gran, 0, 0);
    if (r != CUDA_SUCCESS) { A.release(h); *err = cu_msg("cuMemAddressReserve", r); return cu_status(r); }
    r = A.map(va, sz, 0, h, 0);
    if (r != CUDA_SUCCESS) {
      A.addr_free(va, sz); A.release(h);
      *err = cu_msg("cuMemMap", r);
      return cu_status(r);
    }
    CUmemAccessDesc d = rw(device);
    r = A.set_access(va, sz, &d, 1);
    if (r != CUDA_SUCCESS) {
      A.unmap(va, sz); A.addr_free(va, sz); A.release(h);
      *err = cu_msg("cuMemSetAccess", r);
      return cu_status(r);
    }
    Alloc a;
    a.handle = h;
    a.size = sz;
    a.device = device;
    a.kind = k;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      g_allocs[(uint64_t)va] = a;
    }
    *ptr = (void*)(uintptr_t)va;
    *size = sz;
    *kind_out = k;
    return KVD_OK;
  }
  return cu_status(r);
}

int free(void* ptr, std::string* err) {
  if (!ready(err)) return KVD_ECUDA;
  Alloc a;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_allocs.find((uint64_t)(uintptr_t)ptr);
    if (it == g_allocs.end()) {
      *err = "pointer is not a kvd_mem_alloc allocation";
      return KVD_EINVAL;
    }
    a = it->second;
    g_allocs.erase(it);
  }
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(a.device);
  cudaDeviceSynchronize();   // like cudaFree: no work may still use the range
  const Api& A = api();
  A.unmap((CUdeviceptr)(uintptr_t)ptr, a.size);
  A.addr_free((CUdeviceptr)(uintptr_t)ptr, a.size);
  A.release(a.handle);
  if (a.exported && a.kind == kPosixFd) close((int)a.rec.fd);
  if (prev >= 0) cudaSetDevice(prev);
  return KVD_OK;
}

int lookup_export(uint64_t base, uint64_t* size, ExportRec* rec, std::string* err) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_allocs.find(base);
  if (it == g_allocs.end()) return 0;
  Alloc& a = it->second;
  if (!a.exported) {
    const Api& A = api();
    ExportRec x;
    x.kind = a.kind;
    if (a.kind == kPosixFd) {
      int fd = -1;
      CUresult r = A.export_handle(&fd, a.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
      if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemExportToShareableHandle(fd)", r); return KVD_EHANDLE; }
      x.fd = (uint32_t)fd;
    } else {
      CUmemFabricHandle fh;
      CUresult r = A.export_handle(&fh, a.handle, CU_MEM_HANDLE_TYPE_FABRIC, 0);
      if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemExportToShareableHandle(fabric)", r); return KVD_EHANDLE; }
      static_assert(sizeof(fh) == sizeof(x.payload), "fabric handle size");
      memcpy(x.payload, &fh, sizeof(fh));
    }
    a.rec = x;
    a.exported = true;
  }
  *rec = a.rec;
  *size = a.size;
  return 1;
}

int find(uint64_t addr, uint64_t* base, uint64_t* size) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_allocs.upper_bound(addr);
  if (it == g_allocs.begin()) return 0;
  --it;
  if (addr >= it->first + it->second.size) return 0;
  *base = it->first;
  *size = it->second.size;
  return 1;
}

int grant_access(uint64_t base, int device, std::string* err) {
  uint64_t size = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_allocs.find(base);
    if (it == g_allocs.end()) return KVD_OK;   // not VMM memory: peer access covers it
    size = it->second.size;
  }
  CUmemAccessDesc d = rw(device);
  CUresult r = api().set_access((CUdeviceptr)base, size, &d, 1);
  if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemSetAccess(peer)", r); return KVD_EHANDLE; }
  return KVD_OK;
}

int import_map(const ExportRec& rec, int64_t pid, uint64_t size, int device, void** va_out,
               std::string* err) {
  if (!ready(err)) return KVD_ECUDA;
  const Api& A = api();
  CUmemGenericAllocationHandle h = 0;
  CUresult r;
  if (rec.kind == kPosixFd) {
    const long pidfd = syscall(SYS_pidfd_open, (pid_t)pid, 0);
    if (pidfd < 0) {
      *err = std::string("pidfd_open(exporter pid): ") + strerror(errno) +
             " -- the exporter must be alive and in this PID namespace";
      return KVD_EHANDLE;
    }
    const long fd = syscall(SYS_pidfd_getfd, (int)pidfd, (int)rec.fd, 0);
    const int e = errno;
    close((int)pidfd);
    if (fd < 0) {
      *err = std::string("pidfd_getfd(exported fd): ") + strerror(e) +
             " -- needs the same user and ptrace permission over the exporter";
      return KVD_EHANDLE;
    }
    r = A.import_handle(&h, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close((int)fd);
  } else if (rec.kind == kFabric) {
    r = A.import_handle(&h, (void*)rec.payload, CU_MEM_HANDLE_TYPE_FABRIC);
  } else {
    *err = "not a VMM export record";
    return KVD_EHANDLE;
  }
  if (r != CUDA_SUCCESS) { *err = cu_msg("cuMemImportFromShareableHandle", r); return KVD_EHANDLE; }
  CUmemAllocationProp prop = prop_for(device, rec.kind);
  size_t gran = 0;
  r = A.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS) gran = 2u << 20;
  CUdeviceptr va = 0;
  r = A.reserve(&va, size, gran, 0, 0);
  if (r != CUDA_SUCCESS) { A.release(h); *err = cu_msg("cuMemAddressReserve", r); return cu_status(r); }
  r = A.map(va, size, 0, h, 0);
  A.release(h);   // the mapping keeps the physical memory referenced
  if (r != CUDA_SUCCESS) { A.addr_free(va, size); *err = cu_msg("cuMemMap(import)", r); return KVD_EHANDLE; }
  CUmemAccessDesc d = rw(device);
  r = A.set_access(va, size, &d, 1);
  if (r != CUDA_SUCCESS) {
    A.unmap(va, size); A.addr_free(va, size);
    *err = cu_msg("cuMemSetAccess(import)", r);
    return KVD_EHANDLE;
  }
  *va_out = (void*)(uintptr_t)va;
  return KVD_OK;
}

void unmap(void* va, uint64_t size) {
  if (!api().ok || !va) return;
  api().unmap((CUdeviceptr)(uintptr_t)va, size);
  api().addr_free((CUdeviceptr)(uintptr_t)va, size);
}

}  // namespace vmm
}  // namespace kvd
