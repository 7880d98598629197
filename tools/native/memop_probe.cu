// memop_probe.cu -- can stream memory operations order a resident kernel's
// work with a caller's stream cheaply?  (the "stream-ordered engine" idea in
// DESIGN.md §12).  A persistent one-thread kernel on its own stream P waits
// for go == i in device memory, then releases done = i (device memory).
// Per round the host, on a second stream S:
//   cuStreamWriteValue32(S, go, i)          -- after S's earlier work
//   cuStreamWaitValue32(S, done, i, GEQ)    -- S's later work after the kernel's
//   cuStreamWriteValue32(S, host_ack, i)    -- stands for "later work on S"
// and spins until host_ack == i.  Printed: API cost of the three calls and
// the host-to-host round trip (p10 / p50 / p90 us); also the same round trip
// with the host storing go directly into pinned memory (no stream order).
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/native/memop_probe.cu \
//        -o tools/native/memop_probe && tools/native/memop_probe [iters]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AttrFn)(int*, CUdevice_attribute, CUdevice);

__global__ void responder(volatile unsigned int* go, unsigned int* done, int n) {
  for (unsigned int i = 1; i <= (unsigned int)n; ++i) {
    unsigned int v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(go) : "memory");
    } while (v < i);
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(done), "r"(i) : "memory");
  }
}

template <typename F>
static F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    fprintf(stderr, "no %s\n", name);
    exit(2);
  }
  return reinterpret_cast<F>(p);
}

static void report(const char* what, std::vector<double> v, std::vector<double> api) {
  std::sort(v.begin(), v.end());
  std::sort(api.begin(), api.end());
  auto q = [](const std::vector<double>& x, double f) {
    return x.empty() ? -1.0 : x[(size_t)(f * (x.size() - 1))];
  };
  printf("{\"probe\": \"%s\", \"p10_us\": %.2f, \"p50_us\": %.2f, \"p90_us\": %.2f, "
         "\"api_us_p50\": %.2f}\n", what, q(v, 0.1), q(v, 0.5), q(v, 0.9), q(api, 0.5));
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 3000;
  auto write32 = entry<WriteFn>("cuStreamWriteValue32");
  auto wait32 = entry<WaitFn>("cuStreamWaitValue32");
  auto attr = entry<AttrFn>("cuDeviceGetAttribute");
  int memops = -1;
  attr(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, 0);
  printf("{\"probe\": \"attributes\", \"can_use_stream_mem_ops\": %d}\n", memops);
  cudaFree(0);
  unsigned int *go, *done, *ack, *dack;
  cudaMalloc(&go, 64);
  cudaMalloc(&done, 64);
  cudaMemset(go, 0, 64);
  cudaMemset(done, 0, 64);
  cudaHostAlloc((void**)&ack, 64, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostGetDevicePointer((void**)&dack, ack, 0);
  cudaDeviceSynchronize();
  cudaStream_t P, S;
  cudaStreamCreateWithFlags(&P, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&S, cudaStreamNonBlocking);
  {  // stream-ordered: go by a stream write, later stream work after done
    ack[0] = 0;
    responder<<<1, 1, 0, P>>>(go, done, iters);
    std::vector<double> rt, api;
    volatile unsigned int* A = ack;
    for (unsigned int i = 1; i <= (unsigned int)iters; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      write32((CUstream)S, (CUdeviceptr)go, i, CU_STREAM_WRITE_VALUE_DEFAULT);
      wait32((CUstream)S, (CUdeviceptr)done, i, CU_STREAM_WAIT_VALUE_GEQ);
      write32((CUstream)S, (CUdeviceptr)dack, i, CU_STREAM_WRITE_VALUE_DEFAULT);
      const auto t1 = std::chrono::steady_clock::now();
      while (*A < i) {
      }
      const auto t2 = std::chrono::steady_clock::now();
      if (i > 100) {
        api.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        rt.push_back(std::chrono::duration<double, std::micro>(t2 - t0).count());
      }
    }
    cudaDeviceSynchronize();
    report("stream_ordered_go_wait_ack", rt, api);
  }
  {  // go by a stream write only (the kernel's release observed by the host directly)
    cudaMemset(go, 0, 64);
    cudaMemset(done, 0, 64);
    cudaDeviceSynchronize();
    unsigned int* hdone;
    unsigned int* ddone;
    cudaHostAlloc((void**)&hdone, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostGetDevicePointer((void**)&ddone, hdone, 0);
    hdone[0] = 0;
    responder<<<1, 1, 0, P>>>(go, ddone, iters);
    std::vector<double> rt, api;
    volatile unsigned int* H = hdone;
    for (unsigned int i = 1; i <= (unsigned int)iters; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      write32((CUstream)S, (CUdeviceptr)go, i, CU_STREAM_WRITE_VALUE_DEFAULT);
      const auto t1 = std::chrono::steady_clock::now();
      while (*H < i) {
      }
      const auto t2 = std::chrono::steady_clock::now();
      if (i > 100) {
        api.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        rt.push_back(std::chrono::duration<double, std::micro>(t2 - t0).count());
      }
    }
    cudaDeviceSynchronize();
    report("stream_write_go_host_sees_release", rt, api);
  }
  {  // baseline: the host stores go into pinned memory (no stream order)
    unsigned int *hgo, *dgo, *hdone, *ddone;
    cudaHostAlloc((void**)&hgo, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostAlloc((void**)&hdone, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    cudaHostGetDevicePointer((void**)&dgo, hgo, 0);
    cudaHostGetDevicePointer((void**)&ddone, hdone, 0);
    hgo[0] = 0;
    hdone[0] = 0;
    responder<<<1, 1, 0, P>>>(dgo, ddone, iters);
    std::vector<double> rt, api;
    std::atomic<unsigned int>* G = reinterpret_cast<std::atomic<unsigned int>*>(hgo);
    volatile unsigned int* H = hdone;
    for (unsigned int i = 1; i <= (unsigned int)iters; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      G->store(i, std::memory_order_release);
      while (*H < i) {
      }
      const auto t2 = std::chrono::steady_clock::now();
      if (i > 100) rt.push_back(std::chrono::duration<double, std::micro>(t2 - t0).count());
    }
    cudaDeviceSynchronize();
    report("host_store_go_host_sees_release", rt, api);
  }
  return 0;
}
