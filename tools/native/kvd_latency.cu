// kvd_latency.cu -- per-request latency of the C ABI without any Python in
// the loop: host wall time from kvd_pull entry to the first kvd_poll_done
// == 1 (reading R16 of DESIGN.md), for C1 (256 tokens) and C2 (8K tokens).
//
//   nvcc -O2 -I include tools/native/kvd_latency.cu -L paper_2501_14743_b200 -lkvd \
//        -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/kvd_latency
//   tools/native/kvd_latency [src_dev] [dst_dev] [iters] [timing 0|1] [engine CTAs]
// timing 1 also reports the in-kernel %globaltimer span (KVD_OPT_TIMING = 2).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kvd.h"

#define CK(x)                                                                 \
  do {                                                                        \
    auto _s = (x);                                                            \
    if ((int)_s != 0) {                                                       \
      fprintf(stderr, "%s failed (%d): %s\n", #x, (int)_s, kvd_last_error()); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

struct Cache {
  std::vector<void*> layers;
  kvd_cache h = nullptr;
};

static Cache make(int dev, const kvd_layout& L) {
  Cache c;
  kvd_geometry g;
  CK(kvd_layout_geometry(&L, &g));
  cudaSetDevice(dev);
  for (uint32_t l = 0; l < L.num_layers; ++l) {
    void* p = nullptr;
    if (cudaMalloc(&p, g.layer_bytes) != cudaSuccess) exit(2);
    cudaMemset(p, (int)(l * 7 + dev), g.layer_bytes);
    c.layers.push_back(p);
  }
  cudaDeviceSynchronize();
  CK(kvd_register_cache(dev, &L, c.layers.data(), &c.h));
  return c;
}

static void run(const char* name, const kvd_layout& L, uint32_t n, int sdev, int ddev, int iters,
                bool timing, int engine) {
  Cache src = make(sdev, L), dst = make(ddev, L);
  std::vector<unsigned char> blob(1 << 16);
  size_t len = blob.size();
  CK(kvd_export_handle(src.h, blob.data(), &len));
  kvd_peer p;
  CK(kvd_open_peer(dst.h, blob.data(), len, &p));
  cudaSetDevice(ddev);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::vector<int32_t> si(n), di(n);
  for (uint32_t i = 0; i < n; ++i) {   // fragmented-ish: every other block
    si[i] = (int32_t)(2 * i % L.num_blocks);
    di[i] = (int32_t)((2 * i + 1) % L.num_blocks);
  }
  std::vector<double> lat, call, span, pre;
  if (timing) CK(kvd_peer_set(p, KVD_OPT_TIMING, 2));   // in-kernel %globaltimer spans
  // KVD_LAT_OPTS="option=value,...": extra kvd_peer_set calls (e.g. "0=16,4=256"
  // for 16 CTAs of 256 threads) to sweep the small-request launch shape
  if (const char* o = getenv("KVD_LAT_OPTS")) {
    int opt = 0;
    long long val = 0;
    for (const char* q = o; sscanf(q, "%d=%lld", &opt, &val) == 2;) {
      CK(kvd_peer_set(p, opt, val));
      q = strchr(q, ',');
      if (!q) break;
      ++q;
    }
  }
  if (engine) CK(kvd_peer_set(p, KVD_OPT_ENGINE, engine));   // resident engine (short requests)
  for (int it = 0; it < iters + 20; ++it) {
    const uint64_t rid = 100 + it;
    auto t0 = std::chrono::steady_clock::now();
    CK(kvd_pull(p, rid, si.data(), di.data(), n, s));
    auto t1 = std::chrono::steady_clock::now();
    int done = 0;
    while (!done) CK(kvd_poll_done(p, rid, &done));
    auto t2 = std::chrono::steady_clock::now();
    if (it >= 20) {
      call.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      lat.push_back(std::chrono::duration<double, std::micro>(t2 - t0).count());
    }
    if (timing) {
      kvd_span sp;
      uint32_t k = 0;
      CK(kvd_peer_spans(p, &sp, 1, &k));
      if (k && it >= 20) {
        span.push_back((sp.end_ns - sp.start_ns) * 1e-3);
        pre.push_back((sp.wait_ns - sp.start_ns) * 1e-3);   // engine: entry seen -> handed over
      }
    }
  }
  std::sort(span.begin(), span.end());
  std::sort(pre.begin(), pre.end());
  std::sort(lat.begin(), lat.end());
  std::sort(call.begin(), call.end());
  auto q = [](const std::vector<double>& v, double f) { return v[(size_t)(f * (v.size() - 1))]; };
  kvd_pull_info info;
  kvd_last_pull_info(p, &info);
  printf("{\"config\": \"%s\", \"src_dev\": %d, \"dst_dev\": %d, \"bytes\": %llu, \"variant\": %u, "
         "\"ctas\": %u, \"call_us_p50\": %.2f, \"latency_us_p50\": %.2f, \"latency_us_p90\": %.2f, "
         "\"latency_us_min\": %.2f, \"kernel_span_us_p50\": %.2f, \"pre_us_p50\": %.2f, \"iters\": %d, \"engine\": %d, "
         "\"launches\": %u, \"threads\": %u, \"opts\": \"%s\"}\n",
         name, sdev, ddev, (unsigned long long)info.bytes, info.variant, info.ctas, q(call, 0.5),
         q(lat, 0.5), q(lat, 0.9), lat.front(), span.empty() ? -1.0 : q(span, 0.5), pre.empty() ? -1.0 : q(pre, 0.5), iters, engine, info.launches, info.threads, getenv("KVD_LAT_OPTS") ? getenv("KVD_LAT_OPTS") : "");
  kvd_close_peer(p);
  kvd_unregister_cache(dst.h);
  kvd_unregister_cache(src.h);
  for (auto* v : {&src.layers, &dst.layers})
    for (void* x : *v) cudaFree(x);
}

int main(int argc, char** argv) {
  const int sdev = argc > 1 ? atoi(argv[1]) : 0;
  const int ddev = argc > 2 ? atoi(argv[2]) : 0;
  const int iters = argc > 3 ? atoi(argv[3]) : 2000;
  const bool timing = argc > 4 && atoi(argv[4]) != 0;
  const int engine = argc > 5 ? atoi(argv[5]) : 0;
  kvd_layout c1{2, 2, 64, 16, 64, KVD_FP16, {0, 0, 0, 0, 0}};
  run("C1", c1, 16, sdev, ddev, iters, timing, engine);
  kvd_layout c2{32, 32, 128, 16, 1024, KVD_FP16, {0, 0, 0, 0, 0}};
  if (!engine && !getenv("KVD_LAT_C1_ONLY"))
    run("C2", c2, 512, sdev, ddev, std::max(20, iters / 50), timing, 0);
  return 0;
}
