// call_cost.cu -- host cost of one kvd_pull call (validate + coalesce + plan +
// stage the run table + launch) by the number of coalesced runs, loopback on
// one GPU.  The run table travels in the kernel parameters up to 2016 runs
// (template buckets), beyond that through a per-slot device buffer.
//
//   nvcc -O2 -I include tools/native/call_cost.cu -L paper_2501_14743_b200 -lkvd \
//        -Xlinker -rpath=$PWD/paper_2501_14743_b200 -o tools/native/call_cost
//   tools/native/call_cost [iters]
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 300;
  // 2 layers x 8 heads x 128 x fp16, 16-token blocks (64 KiB per block and
  // layer), 8192 blocks: up to 4096 runs of one block
  kvd_layout L{2, 8, 128, 16, 8192, KVD_FP16, {0, 0, 0, 0, 0}};
  kvd_geometry g;
  CK(kvd_layout_geometry(&L, &g));
  std::vector<void*> sl(2), dl(2);
  for (int l = 0; l < 2; ++l) {
    cudaMalloc(&sl[l], g.layer_bytes);
    cudaMalloc(&dl[l], g.layer_bytes);
  }
  kvd_cache src, dst;
  CK(kvd_register_cache(0, &L, sl.data(), &src));
  CK(kvd_register_cache(0, &L, dl.data(), &dst));
  std::vector<unsigned char> blob(1 << 16);
  size_t len = blob.size();
  CK(kvd_export_handle(src, blob.data(), &len));
  kvd_peer p;
  CK(kvd_open_peer(dst, blob.data(), len, &p));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  uint64_t rid = 1;
  for (uint32_t runs : {1u, 8u, 9u, 64u, 65u, 130u, 256u, 512u, 513u, 1024u, 2016u, 2017u, 4096u}) {
    // `runs` runs of 2 blocks each (512 blocks when runs <= 256), gaps between them
    const uint32_t per = runs <= 256 ? 512 / runs : 2;
    std::vector<int32_t> si, di;
    for (uint32_t r = 0; r < runs; ++r)
      for (uint32_t b = 0; b < per && si.size() < 8192 / 2; ++b) {
        si.push_back((int32_t)(2 * r * per + b) % 8192);
        di.push_back((int32_t)((2 * r * per + b) % 8192));
      }
    std::vector<double> call;
    kvd_pull_info info{};
    for (int it = 0; it < iters + 10; ++it) {
      const auto t0 = std::chrono::steady_clock::now();
      CK(kvd_pull(p, rid, si.data(), di.data(), (uint32_t)si.size(), s));
      const auto t1 = std::chrono::steady_clock::now();
      CK(kvd_wait_done(p, rid, 10000000));
      ++rid;
      if (it >= 10) call.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    kvd_last_pull_info(p, &info);
    std::sort(call.begin(), call.end());
    printf("{\"runs\": %u, \"blocks\": %zu, \"variant\": %u, \"call_us_p50\": %.2f, "
           "\"call_us_p10\": %.2f, \"launches\": %u}\n",
           info.runs, si.size(), info.variant, call[call.size() / 2], call[call.size() / 10],
           info.launches);
  }
  kvd_close_peer(p);
  return 0;
}
