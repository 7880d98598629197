// fence_probe.cu -- cost of the completion-path primitives on B200, measured
// inside one thread with clock64 (SM cycles), to find where the fixed
// per-request time of a pull goes (tools/size_probe.py: a 0-block pull, i.e.
// only the completion kernel, takes ~10 us loopback / ~14 us over NVLink).
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/native/fence_probe.cu \
//        -o tools/native/fence_probe && tools/native/fence_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t _e = (x);                                                  \
    if (_e != cudaSuccess) {                                               \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(_e));             \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

enum Op {
  kNothing, kFenceGpu, kFenceSys, kRelSysHost, kRelSysDev, kAtomSysDev, kAtomSysPeer,
  kAtomGpuDev, kStoreHostFenceSys, kRelGpuDev, kStoresThenFenceGpu, kStoresThenFenceSys,
  kAtomPeerUsed, kAtomPeerThenRelHost, kRelHostThenAtomPeerRelPeer, kAtomPeerRelHostRelPeer,
  kTwoRelSys, kNumOps
};
const char* kName[kNumOps] = {
    "nothing", "fence.gpu (threadfence)", "fence.sys (threadfence_system)",
    "st.release.sys -> pinned host", "st.release.sys -> local HBM",
    "atomicAdd_system -> local HBM", "atomicAdd_system -> peer HBM (NVLink)",
    "atomicAdd (gpu) -> local HBM", "volatile st host + fence.sys", "st.release.gpu -> local HBM",
    "1 MiB CTA stores then fence.gpu", "1 MiB CTA stores then fence.sys",
    "atomicAdd_system -> peer, result used", "peer atomic issued, then st.release.sys host (overlap?)",
    "completion now: rel.sys host; peer atomic; st id; rel.sys peer",
    "completion reordered: peer atomic; rel.sys host; st id; rel.sys peer",
    "two st.release.sys back to back (host, local)"};

__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_rel_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

__global__ void probe(int op, unsigned long long* host, unsigned long long* dev,
                      unsigned long long* peer, uint4* scratch, long long* out, int reps) {
  if (op == kStoresThenFenceGpu || op == kStoresThenFenceSys) {
    // every thread of the CTA stores its share of 1 MiB first
    for (int i = threadIdx.x; i < (1 << 16); i += blockDim.x)
      scratch[i] = make_uint4(i, i, i, i);
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  long long best = 1ll << 62;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    switch (op) {
      case kFenceGpu: __threadfence(); break;
      case kFenceSys: __threadfence_system(); break;
      case kRelSysHost: st_rel_sys(host, r); break;
      case kRelSysDev: st_rel_sys(dev, r); break;
      case kAtomSysDev: atomicAdd_system(dev + 8, 1ull); break;
      case kAtomSysPeer: atomicAdd_system(peer, 1ull); break;
      case kAtomGpuDev: atomicAdd(dev + 16, 1ull); break;
      case kStoreHostFenceSys: *(volatile unsigned long long*)host = r; __threadfence_system(); break;
      case kRelGpuDev: st_rel_gpu(dev + 24, r); break;
      case kStoresThenFenceGpu: __threadfence(); break;
      case kStoresThenFenceSys: __threadfence_system(); break;
      case kAtomPeerUsed: {
        unsigned long long v = atomicAdd_system(peer, 1ull);
        *(volatile unsigned long long*)(dev + 32) = v;
        break;
      }
      case kAtomPeerThenRelHost: {
        unsigned long long v = atomicAdd_system(peer, 1ull);
        st_rel_sys(host, r);
        *(volatile unsigned long long*)(dev + 32) = v;
        break;
      }
      case kRelHostThenAtomPeerRelPeer: {
        st_rel_sys(host, r);
        unsigned long long v = atomicAdd_system(peer, 1ull);
        unsigned long long* e = peer + 8 + 2 * (v % 64);
        *(volatile unsigned long long*)(e + 1) = r;
        st_rel_sys(e, v + 1);
        break;
      }
      case kAtomPeerRelHostRelPeer: {
        unsigned long long v = atomicAdd_system(peer, 1ull);
        st_rel_sys(host, r);
        unsigned long long* e = peer + 8 + 2 * (v % 64);
        *(volatile unsigned long long*)(e + 1) = r;
        st_rel_sys(e, v + 1);
        break;
      }
      case kTwoRelSys: st_rel_sys(host, r); st_rel_sys(dev + 40, r); break;
      default: break;
    }
    const long long t1 = clock64();
    // the first rep is the one a completion path pays (cold), keep both
    if (r == 0) out[1] = t1 - t0;
    if (t1 - t0 < best) best = t1 - t0;
  }
  out[0] = best;
}

__global__ void empty_kernel() {}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  CK(cudaSetDevice(0));
  unsigned long long *host = nullptr, *host_dev = nullptr, *dev = nullptr, *peer = nullptr;
  CK(cudaHostAlloc((void**)&host, 4096, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&host_dev, host, 0));
  CK(cudaMalloc(&dev, 4096));
  CK(cudaMemset(dev, 0, 4096));
  uint4* scratch = nullptr;
  CK(cudaMalloc(&scratch, 1 << 20));
  if (ndev > 1) {
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&peer, 8192));
    CK(cudaMemset(peer, 0, 8192));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
  }
  long long* out = nullptr;
  CK(cudaMallocManaged(&out, 16));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\"sm_clock_mhz\": %.0f}\n", clk_khz / 1e3);
  for (int op = 0; op < kNumOps; ++op) {
    if ((op == kAtomSysPeer || (op >= kAtomPeerUsed && op <= kAtomPeerRelHostRelPeer)) && !peer)
      continue;
    probe<<<1, 256>>>(op, host_dev, dev, peer, scratch, out, 16);
    CK(cudaDeviceSynchronize());
    const long long best = out[0];
    probe<<<1, 256>>>(op, host_dev, dev, peer, scratch, out, 1);   // cold, single
    CK(cudaDeviceSynchronize());
    printf("{\"op\": \"%s\", \"best_cycles\": %lld, \"best_us\": %.3f, \"first_cycles\": %lld, "
           "\"first_us\": %.3f}\n", kName[op], best, best / (clk_khz / 1e3),
           out[1], out[1] / (clk_khz / 1e3));
  }
  // event-timed kernels with the host hidden behind a spin kernel
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int op : {kNothing, kFenceSys, kRelSysHost, kAtomSysPeer}) {
    if (op == kAtomSysPeer && !peer) continue;
    float acc = 1e9;
    for (int r = 0; r < 20; ++r) {
      probe<<<1, 256, 0, s>>>(kStoresThenFenceGpu, host_dev, dev, peer, scratch, out, 200);
      CK(cudaEventRecord(e0, s));
      if (op == kNothing) empty_kernel<<<1, 32, 0, s>>>();
      else probe<<<1, 32, 0, s>>>(op, host_dev, dev, peer, scratch, out, 1);
      CK(cudaEventRecord(e1, s));
      CK(cudaStreamSynchronize(s));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < acc) acc = ms;
    }
    printf("{\"event_timed_kernel\": \"%s\", \"min_us\": %.2f}\n", kName[op], acc * 1e3);
  }
  return 0;
}
