// link_idle_probe.cu -- latency of one remote (NVLink peer) load after the
// link has been idle for X microseconds, vs a local HBM load: does an idle
// NVLink pay a wake-up on the first access of a request?
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/native/link_idle_probe.cu \
//        -o tools/native/link_idle_probe && tools/native/link_idle_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                  \
  do {                                                         \
    cudaError_t _e = (x);                                      \
    if (_e != cudaSuccess) {                                   \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(_e)); \
      exit(1);                                                 \
    }                                                          \
  } while (0)

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// For each idle gap: spin `gap_ns`, then time one uncached 8 B load from a
// fresh line (stride 4 KiB so neither L2 nor the line buffer hits).
__global__ void probe(const unsigned long long* p, unsigned long long gap_ns, int reps,
                      size_t stride, long long* out, unsigned long long* sink) {
  unsigned long long acc = 0;
  long long best = 1ll << 62, sum = 0;
  for (int r = 0; r < reps; ++r) {
    const unsigned long long until = gtime() + gap_ns;
    while (gtime() < until) {}
    const long long t0 = clock64();
    unsigned long long v;
    asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p + (size_t)r * stride) : "memory");
    acc += v;
    const long long t1 = clock64();
    sum += t1 - t0;
    if (t1 - t0 < best) best = t1 - t0;
  }
  out[0] = best;
  out[1] = sum / reps;
  *sink = acc;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("{\"error\": \"needs two GPUs\"}\n"); return 0; }
  const size_t bytes = 64 << 20;
  unsigned long long *remote = nullptr, *local = nullptr, *sink = nullptr;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&remote, bytes));
  CK(cudaMemset(remote, 1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&local, bytes));
  CK(cudaMemset(local, 1, bytes));
  CK(cudaMalloc(&sink, 8));
  long long* out = nullptr;
  CK(cudaMallocManaged(&out, 16));
  int khz = 0;
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
  const double mhz = khz / 1e3;
  for (unsigned long long gap : {0ull, 1000ull, 5000ull, 20000ull, 100000ull, 1000000ull}) {
    const char* names[4] = {"local HBM, 4 KiB stride", "peer HBM over NVLink, 4 KiB stride",
                            "local HBM, new 2 MiB page each", "peer HBM, new 2 MiB page each"};
    for (int side = 0; side < 4; ++side) {
      const size_t stride = side < 2 ? 512 : (2u << 20) / 8;
      // fresh lines each round: offset the start by the round number
      const unsigned long long* base = (side & 1) ? remote : local;
      probe<<<1, 1>>>(base + (gap % 7) * 16, gap, 16, stride, out, sink);
      CK(cudaDeviceSynchronize());
      printf("{\"target\": \"%s\", \"idle_gap_us\": %.0f, \"best_us\": %.3f, \"mean_us\": %.3f}\n",
             names[side], gap / 1e3, out[0] / mhz, out[1] / mhz);
    }
  }
  return 0;
}
