// pcie_pingpong.cu -- the host <-> device signalling floor under the resident
// engine's latency: how long a word the host stores into
// pinned memory takes to be seen by a polling kernel, and a word the kernel
// stores back to be seen by the polling host.
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/native/pcie_pingpong.cu \
//        -o tools/native/pcie_pingpong && tools/native/pcie_pingpong [iters]
//
// Prints JSON lines:
//   * read_rtt:   one ld.relaxed.sys of pinned host memory, timed in-kernel
//                 (%globaltimer, dependent loads back to back)
//   * pingpong:   host stores i -> kernel sees it -> kernel stores i back ->
//                 host sees it, host wall per round trip; the kernel's ack is
//                 st.relaxed.sys ("relaxed") or st.release.sys ("release",
//                 what a completion needs), 1 or 4 polling warps
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void read_rtt(const unsigned long long* h, int n, unsigned long long* out) {
  unsigned long long acc = 0;
  const unsigned long long t0 = gtimer();
  for (int i = 0; i < n; ++i) acc += ld_sys(h + (acc & 1));   // each load depends on the last
  const unsigned long long t1 = gtimer();
  out[0] = t1 - t0;
  out[1] = acc;
}

// warps 0..pollers-1 of one CTA poll `h2d`; the first to see round i acks it
__global__ void pong(const unsigned long long* h2d, unsigned long long* d2h, int n, int pollers,
                     int release) {
  __shared__ unsigned long long seen;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) seen = 0;
  __syncthreads();
  if (w >= pollers || lane) return;
  __nanosleep(w * 400);
  for (unsigned long long i = 1; i <= (unsigned long long)n; ++i) {
    for (;;) {
      if (*(volatile unsigned long long*)&seen >= i) break;
      if (ld_sys(h2d) >= i) {
        if (atomicMax(&seen, i) < i) {           // this warp acks round i
          if (release)
            asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(d2h), "l"(i) : "memory");
          else
            asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(d2h), "l"(i) : "memory");
        }
        break;
      }
    }
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 5000;
  unsigned long long *h2d, *d2h, *dh2d, *dd2h, *out;
  cudaHostAlloc((void**)&h2d, 64, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostAlloc((void**)&d2h, 64, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostGetDevicePointer((void**)&dh2d, h2d, 0);
  cudaHostGetDevicePointer((void**)&dd2h, d2h, 0);
  cudaMallocManaged(&out, 16);
  h2d[0] = h2d[1] = 0;
  for (int rep = 0; rep < 3; ++rep) {
    read_rtt<<<1, 1>>>(dh2d, 1000, out);
    cudaDeviceSynchronize();
    printf("{\"probe\": \"read_rtt\", \"us_per_load\": %.3f}\n", out[0] / 1000.0 / 1000.0);
  }
  for (int release = 0; release < 2; ++release)
    for (int pollers : {1, 4}) {
      std::atomic<unsigned long long>* H = reinterpret_cast<std::atomic<unsigned long long>*>(h2d);
      volatile unsigned long long* D = d2h;
      H->store(0);
      *D = 0;
      cudaStream_t s;
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      pong<<<1, 32 * pollers, 0, s>>>(dh2d, dd2h, iters, pollers, release);
      std::vector<double> rt;
      for (unsigned long long i = 1; i <= (unsigned long long)iters; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        H->store(i, std::memory_order_release);
        while (*D < i) {
        }
        const auto t1 = std::chrono::steady_clock::now();
        rt.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        const auto t2 = std::chrono::steady_clock::now();   // idle gap, like a caller between requests
        while (std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t2).count() < 2.0) {
        }
      }
      cudaStreamSynchronize(s);
      std::sort(rt.begin() + 100, rt.end());
      auto q = [&](double f) { return rt[100 + (size_t)(f * (rt.size() - 101))]; };
      printf("{\"probe\": \"pingpong\", \"ack\": \"%s\", \"pollers\": %d, \"p50_us\": %.2f, "
             "\"p10_us\": %.2f, \"p90_us\": %.2f}\n",
             release ? "release" : "relaxed", pollers, q(0.5), q(0.1), q(0.9));
      cudaStreamDestroy(s);
    }
  return 0;
}
