// kvd_pull.cu -- the sm_100a pull kernels and their
// completion epilogue (row a6).
//
// PAPER.md §4.3: in pull mode the decode worker "reads the blocks
// from the prefill worker" and "performs KV cache reads for all layers in a
// single shot".  Here the reads are one-sided loads from the prefill GPU's
// HBM, mapped into this process with CUDA IPC, over NVLink 5 / NVSwitch; the
// writes are local HBM stores into the decode cache's blocks.  One launch
// covers every layer, both K and V, and every coalesced run; the
// last CTA to finish raises the request's completion word ("The
// completion transaction sends the request ID"), so the host never
// synchronises per block.
//
// Two data movers share the tiling and the epilogue:
//   * LSU  -- every warp copies whole tiles with 16 B (or 32 B) vector
//             loads/stores through registers, 8 loads in flight per lane.
//   * TMA  -- one elected lane per warp ("pipe") runs an S-stage ring of
//             cp.async.bulk copies: peer HBM -> shared memory (mbarrier
//             complete_tx), then shared memory -> local HBM (bulk group).
//             Up to ~200 KiB per SM in flight without registers, so far
//             fewer SMs saturate NVLink and the rest stay free for decode.
//             Single pulls hand tiles out dynamically (per-slot counter);
//             head-sliced peers (§8 f4) have a variant whose stores are
//             warp-wide strided rows (pull_kernel_tma_rows).
// Also here: the resident pull engine (engine_kernel, one thread-block
// cluster draining a descriptor ring in pinned memory, KVD_OPT_ENGINE), the
// link calibration kernel (calib_read_kernel, discarded bulk reads of the
// peer cache: the measured read ceiling) and flag_kernel (completion with no
// bytes).
// All are bit copies through integer registers / shared memory only (no
// float type ever touches the data): NaN payloads, -0, subnormals survive.
// Pull kernels are launched with programmatic stream serialisation
// (griddepcontrol): back-to-back pulls overlap launch with the previous tail.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "kvd_internal.h"

namespace kvd {
namespace {

// Param-resident run tables.  CUDA 12.1+ allows 32764 bytes of kernel
// parameters; PullArgs is ~160 B, so 2016 int4 runs fit.
constexpr int kRunsTiny = 8;      // small requests: keep the launch's parameter block short
constexpr int kRunsSmall = 64;
constexpr int kRunsMid = 512;
constexpr int kRunsLarge = 2016;
constexpr int kMaxStages = 8;
constexpr unsigned int kTilesPerWarp = 4;   // LSU: tiles per warp per chunk

template <int MAXR>
struct PullParams {
  PullArgs a;
  int4 runs[MAXR > 0 ? MAXR : 1];
};

// ---------------------------------------------------------------------------
// vector load/store through integer registers; streaming cache qualifiers
// (each byte is read and written exactly once).
// ---------------------------------------------------------------------------
struct alignas(16) V16 { uint32_t x, y, z, w; };
struct alignas(32) V32 { uint32_t v[8]; };

// Cache qualifiers, A/B-tested with tools/build_ab.sh (profiles/r01_ab_cache_hints.txt):
// streaming ".cs" (evict-first) loads and stores beat ".nc.L1::no_allocate"
// loads + plain stores by ~1 % in loopback and ~0.5 % over NVLink -- every
// byte is touched exactly once, so nothing is worth keeping in L1/L2.
#ifndef KVD_LD_Q
#define KVD_LD_Q "ld.global.cs"
#endif
#ifndef KVD_ST_Q
#define KVD_ST_Q "st.global.cs"
#endif

__device__ __forceinline__ V16 ld_peer(const V16* p) {
  V16 r;
  asm volatile(KVD_LD_Q ".v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_local(V16* p, const V16& v) {
  asm volatile(KVD_ST_Q ".v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ V32 ld_peer(const V32* p) {
  V32 r;
  asm volatile(KVD_LD_Q ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]),
                 "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_local(V32* p, const V32& v) {
  asm volatile(KVD_ST_Q ".v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "r"(v.v[0]), "r"(v.v[1]), "r"(v.v[2]), "r"(v.v[3]),
                  "r"(v.v[4]), "r"(v.v[5]), "r"(v.v[6]), "r"(v.v[7]) : "memory");
}

// A system-scope release costs ~1.5 us on B200 (tools/native/fence_probe.cu:
// ~3000 SM cycles, the same as fence.sc.sys; a gpu-scope fence ~200), so the
// completion path issues as few of them as the ordering needs.
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Programmatic dependent launch: pull kernels are launched with
// programmatic stream serialisation, so a pull queued right behind another
// pull can be scheduled while the first one drains.  Each CTA lets its
// dependents launch once it has finished moving its share (pdl_trigger), and
// every pull waits for the preceding grid to complete and flush before it
// touches any global memory (pdl_wait) -- stream order is unchanged, only the
// launch latency overlaps the tail.  After a non-PDL kernel both are no-ops.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// The first thread of a CTA to execute it triggers the CTA (later executions
// by any thread of the CTA have no further effect).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// KVD_OPT_TIMING: the earliest CTA start of this launch, and the earliest
// return from griddepcontrol.wait (see PullArgs::gt_start)
__device__ __forceinline__ void mark_start(const PullArgs& a, bool waited) {
  if (a.gt_start != nullptr && threadIdx.x == 0) {
    const unsigned long long t = globaltimer();
    atomicMin(a.gt_start, t);
    if (waited) atomicMin(a.gt_start + 1, t);
  }
}
__device__ __forceinline__ void mark_wait(const PullArgs& a) {
  if (a.gt_start != nullptr) atomicMin(a.gt_start + 1, globaltimer());
}

// One warp copies `bytes` (multiple of sizeof(V)) from src to dst.  All U
// loads of a batch are issued before any store so each lane keeps U
// independent NVLink reads in flight (Little's law).
template <typename V, int U>
__device__ __forceinline__ void warp_copy(char* __restrict__ dst, const char* __restrict__ src,
                                          unsigned int bytes, unsigned int lane) {
  const V* s = reinterpret_cast<const V*>(src);
  V* d = reinterpret_cast<V*>(dst);
  const unsigned int nv = bytes / sizeof(V);
  for (unsigned int i = lane; i < nv; i += 32 * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * 32 < nv) v[u] = ld_peer(s + i + u * 32);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * 32 < nv) st_local(d + i + u * 32, v[u]);
  }
}

// Head-slice copy (§8 f4): the unit is `rows` rows of row_bytes; row r sits
// at src + r*src_rs and dst + r*dst_rs.  Same batching as warp_copy.
template <typename V, int U>
__device__ __forceinline__ void warp_copy_rows(char* __restrict__ dst, const char* __restrict__ src,
                                               unsigned int bytes, unsigned int lane,
                                               unsigned int row_bytes, unsigned int src_rs,
                                               unsigned int dst_rs) {
  const unsigned int vpr = row_bytes / sizeof(V);
  const unsigned int nv = bytes / sizeof(V);
  for (unsigned int i = lane; i < nv; i += 32 * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned int idx = i + u * 32;
      if (idx < nv) {
        const unsigned int r = idx / vpr, c = idx - r * vpr;
        v[u] = ld_peer(reinterpret_cast<const V*>(src + (size_t)r * src_rs) + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned int idx = i + u * 32;
      if (idx < nv) {
        const unsigned int r = idx / vpr, c = idx - r * vpr;
        st_local(reinterpret_cast<V*>(dst + (size_t)r * dst_rs) + c, v[u]);
      }
    }
  }
}

__device__ __forceinline__ unsigned long long layer_base(const SideAddr& s, unsigned int l) {
  return s.table ? s.table[l] : s.base + (unsigned long long)l * s.step;
}

// One work item.  `off` is the tile's byte offset inside its run's units
// laid end to end ([0, len * unit_bytes)), used to credit batched requests.
struct Tile {
  const char* src;
  char* dst;
  unsigned int bytes;
  unsigned int run;
  unsigned long long off;
  unsigned int skip;       // bounds audit: counted violation, do not copy
};

// Tile t -> addresses.  Segments are (layer, plane, run); a tile never
// crosses one.  runs[r].w is the inclusive tile prefix over runs within one
// (layer, plane).
__device__ __forceinline__ Tile tile_at(const PullArgs& a, const int4* runs, unsigned int t) {
  unsigned int lp, k;
  if (a.run_major) {
    k = t;
  } else {
    lp = t / a.tiles_per_lp;
    k = t - lp * a.tiles_per_lp;
  }
  int lo = 0, hi = (int)a.nruns - 1;                 // first run with tile_end > k
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((unsigned int)runs[mid].w > k) hi = mid; else lo = mid + 1;
  }
  const int4 run = runs[lo];
  const unsigned int prev = lo ? (unsigned int)runs[lo - 1].w : 0u;
  unsigned int kr = k - prev;
  if (a.run_major) {       // within the run: (layer, plane) major, then tile
    const unsigned int per_lp = ((unsigned int)run.w - prev) / (a.num_layers * a.planes);
    lp = kr / per_lp;
    kr -= lp * per_lp;
  }
  const unsigned int l = (a.planes == 2) ? (lp >> 1) : lp;
  const unsigned int p = (a.planes == 2) ? (lp & 1u) : 0u;
  unsigned long long src_off, dst_off, off, avail, in_run;
  if (a.contiguous) {
    off = (unsigned long long)kr * a.tile_bytes;
    avail = (unsigned long long)(unsigned int)run.z * a.unit_bytes - off;
    src_off = (unsigned long long)run.x * a.src.block_stride + off;
    // head slices (f4): `off` counts remote bytes; locally rows are strided
    dst_off = (unsigned long long)run.y * a.dst.block_stride +
              (a.row_bytes ? off / a.row_bytes * a.dst_row_stride : off);
    in_run = off;
  } else {
    const unsigned int j = kr / a.tiles_per_unit;
    const unsigned int kk = kr - j * a.tiles_per_unit;
    off = (unsigned long long)kk * a.tile_bytes;
    avail = a.unit_bytes - off;
    src_off = (unsigned long long)(run.x + (int)j) * a.src.block_stride + off;
    dst_off = (unsigned long long)(run.y + (int)j) * a.dst.block_stride + off;
    in_run = (unsigned long long)j * a.unit_bytes + off;
  }
  Tile T;
  T.src = reinterpret_cast<const char*>(layer_base(a.src, l) +
                                        (unsigned long long)p * a.src.plane_stride + src_off);
  T.dst = reinterpret_cast<char*>(layer_base(a.dst, l) +
                                  (unsigned long long)p * a.dst.plane_stride + dst_off +
                                  a.dst_unit_offset);
  T.bytes = avail < a.tile_bytes ? (unsigned int)avail : a.tile_bytes;
  T.run = (unsigned int)lo;
  T.off = in_run;
  T.skip = 0;
  return T;
}

// Bounds audit: the bytes a tile touches must lie inside layer l's tensor on
// both sides.  Head-slice tiles span (rows-1) row strides plus one row.
// Scalars only (no Tile address taken), so the hot loop keeps no stack frame.
__device__ __noinline__ bool in_bounds(const PullArgs& a, unsigned long long s,
                                       unsigned long long d, unsigned int bytes, unsigned int t) {
  unsigned int l;
  if (a.run_major) {
    // recover the layer from the tile's source address (run-major order)
    l = 0;
    for (unsigned int k = 0; k < a.num_layers; ++k) {
      const unsigned long long b = layer_base(a.src, k);
      if (s >= b && s < b + a.src_layer_bytes) {
        l = k;
        break;
      }
    }
  } else {
    const unsigned int lp = t / a.tiles_per_lp;
    l = (a.planes == 2) ? (lp >> 1) : lp;
  }
  unsigned long long src_ext = bytes, dst_ext = bytes;
  if (a.row_bytes) {
    const unsigned long long rows = bytes / a.row_bytes;
    src_ext = (rows - 1) * a.src_row_stride + a.row_bytes;
    dst_ext = (rows - 1) * a.dst_row_stride + a.row_bytes;
  }
  const unsigned long long s0 = layer_base(a.src, l), d0 = layer_base(a.dst, l);
  return bytes > 0 && s >= s0 && s + src_ext <= s0 + a.src_layer_bytes && d >= d0 &&
         d + dst_ext <= d0 + a.dst_layer_bytes && (s % 16) == 0 && (d % 16) == 0;
}
__device__ __forceinline__ bool tile_in_bounds(const PullArgs& a, const Tile& T, unsigned int t) {
  return in_bounds(a, (unsigned long long)T.src, (unsigned long long)T.dst, T.bytes, t);
}

// Complete() to the prefill side ("The completion transaction sends
// the request ID to the prefill worker"; it then releases the
// blocks).  The exporter's mailbox is host memory shared with this process;
// this importer owns one single-producer ring of it and the host assigned
// the request its position, so the post is two plain 64-bit stores (each
// single-copy atomic, both tagged with the position), posted over PCIe: no
// atomic round trip over NVLink and no second system-scope fence.  It is
// issued after the slot word's release, i.e. after every byte of the
// request landed -- and so after every read of the prefill's blocks.
__device__ __forceinline__ void mbox_post(const PullArgs& a, unsigned long long pos,
                                          unsigned long long request_id) {
  if (a.mbox == nullptr) return;
  unsigned long long* e = a.mbox + 2 * (pos % kReleaseRing);
  const unsigned long long tag = (unsigned long long)(unsigned int)(pos + 1) << 32;
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(e), "l"(tag | (request_id & 0xffffffffull)) : "memory");
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(e + 1), "l"(tag | (request_id >> 32)) : "memory");
}
// Publish a finished request: release the token into the host-visible slot
// word (one system-scope release orders every byte before it), then post the
// id to the exporter.
__device__ __forceinline__ void publish_token(const PullArgs& a, unsigned long long* flag,
                                              unsigned long long token,
                                              unsigned long long request_id,
                                              unsigned long long pos) {
  st_release_sys(flag, token);
  mbox_post(a, pos, request_id);
}

// --- batched drain (f1): per-request completion inside one launch ----------
// The caller's atomic observed every credit of request q; the acquire fence
// makes their (fenced) stores happen-before this thread's system-scope
// release of the slot word (causality is transitive across the two scopes).
__device__ __forceinline__ void publish(const PullArgs& a, unsigned int q) {
  const uint4 R = a.reqs[q];
  a.bytectr[R.y] = 0ull;                 // slot idle again
  fence_acq_rel_gpu();
  publish_token(a, &a.flags[R.y], a.tokens[q], a.req_ids[q], a.mbox_pos + q);
}

// Credit `bytes` landed bytes to request q; the credit that reaches the
// request's total publishes it.  Callers fence their stores first.
__device__ __forceinline__ void credit(const PullArgs& a, unsigned int q, unsigned long long bytes) {
  const uint4 R = a.reqs[q];
  const unsigned long long total = (unsigned long long)R.z | ((unsigned long long)R.w << 32);
  const unsigned long long old = atomicAdd(&a.bytectr[R.y], bytes);
  if (old + bytes == total) publish(a, q);
}

__device__ __forceinline__ void fence_stores(const PullArgs& a) {
  if (a.remote_stores) __threadfence_system(); else __threadfence();
}

// Per-warp credit accumulator: a warp's tiles of one request are credited
// with ONE atomic when the warp moves on to another request (or finishes),
// after a fence that orders all of the accumulated tiles' stores.  Keeps the
// current request's entry range to skip the request lookup.
struct Credit {
  int q = -1;
  unsigned int first = 0, next = 0;   // entry range [first, next) of request q
  unsigned long long bytes = 0;
};

// LSU: called by every lane of the warp (uniform control flow, warp_sync);
// each lane fences its own stores, the warp syncs, `lane0` does the atomic.
// TMA: called by the pipe's single lane after its bulk stores completed.
__device__ __forceinline__ void credit_flush(const PullArgs& a, Credit& c, bool lane0,
                                             bool warp_sync) {
  if (c.q >= 0 && c.bytes) {
    fence_stores(a);
    if (warp_sync) __syncwarp();
    if (lane0) credit(a, (unsigned int)c.q, c.bytes);
  }
  c.bytes = 0;
}

// A tile may hold blocks of several requests when runs were merged across
// requests (fig:queue): split its bytes at the request boundaries.
__device__ void credit_tile(const PullArgs& a, const Tile& T, Credit& c, bool lane0,
                            bool warp_sync) {
  const unsigned int g0 = a.run_pos[T.run];
  unsigned long long pos = T.off;
  const unsigned long long end = T.off + T.bytes;
  while (pos < end) {
    const unsigned int e = g0 + (unsigned int)(pos / a.unit_bytes);
    if (!(c.q >= 0 && e >= c.first && e < c.next)) {
      int lo = 0, hi = (int)a.nreqs - 1;          // last request whose first entry <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.reqs[mid].x <= e) lo = mid; else hi = mid - 1;
      }
      credit_flush(a, c, lane0, warp_sync);
      c.q = lo;
      c.first = a.reqs[lo].x;
      c.next = (lo + 1 < (int)a.nreqs) ? a.reqs[lo + 1].x : 0xffffffffu;
    }
    unsigned long long q_end = end;
    if (c.next != 0xffffffffu) {
      const unsigned long long nb = (unsigned long long)(c.next - g0) * a.unit_bytes;
      if (nb < q_end) q_end = nb;
    }
    c.bytes += q_end - pos;
    pos = q_end;
  }
}

// Requests with no blocks complete at launch.
__device__ __forceinline__ void publish_empty(const PullArgs& a) {
  if (a.nreqs == 0 || blockIdx.x != 0 || threadIdx.x != 0) return;
  for (unsigned int q = 0; q < a.nreqs; ++q)
    if (a.reqs[q].z == 0 && a.reqs[q].w == 0) publish(a, q);
}

// Completion (row a6): every thread orders its stores (gpu scope for the
// pull's local stores, system scope when push stored into a peer GPU), the
// CTA arrives once; the last CTA acquires (gpu scope: every arrival is on
// this GPU), resets the slot counter and publishes the token with ONE
// system-scope release, so a host acquire load of the word implies every
// byte landed; the prefill-side notification follows (publish_token).
// Batches published their requests one by one; their last CTA only resets
// the launch's counters and releases the descriptor buffer to the host.
__device__ __forceinline__ void complete(const PullArgs& a) {
  if (a.counter == nullptr) return;   // baseline gather/scatter: stream order only
  if (a.remote_stores) __threadfence_system(); else __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(a.counter, 1u);
    if (prev == gridDim.x - 1) {
      *a.counter = 0u;
      fence_acq_rel_gpu();
      if (a.tile_ctr != nullptr) *a.tile_ctr = 0u;   // every claim happened before its CTA arrived
      if (a.nreqs) {                 // batches: requests completed one by one (publish)
        if (a.done_word != nullptr) st_release_sys(a.done_word, a.done_seq);
        return;
      }
      if (a.gt_start != nullptr) {   // first CTA start -> last CTA done, before the release
        const unsigned long long t1 = globaltimer();
        const unsigned long long t0 = *(volatile unsigned long long*)a.gt_start;
        const unsigned long long tw = *(volatile unsigned long long*)(a.gt_start + 1);
        volatile unsigned long long* o = a.gt_out;
        o[0] = t1 - t0;
        o[1] = t0;
        o[2] = tw;
        o[3] = t1;
        a.gt_start[0] = ~0ull;
        a.gt_start[1] = ~0ull;
      }
      publish_token(a, a.flag, a.token, a.request_id, a.mbox_pos);
    }
  }
}

// Stage the run table in shared memory when the launcher reserved room for
// it: the per-tile binary search then costs shared loads (~30 cycles)
// instead of constant-bank / L2 misses, which is what bounds 4-8 KiB
// segments where a pipe must issue a tile every few hundred nanoseconds.
__device__ __forceinline__ const int4* stage_runs(const PullArgs& a, const int4* runs,
                                                  int4* smem_runs) {
  if (!a.smem_runs) return runs;
  for (unsigned int i = threadIdx.x; i < a.nruns; i += blockDim.x) smem_runs[i] = runs[i];
  __syncthreads();
  return smem_runs;
}

// ---------------------------------------------------------------------------
// LSU mover: one warp per tile
// ---------------------------------------------------------------------------
// GENERAL = false is the plain single-request copy (no head-slice rows, no
// batch credits) so the hot path keeps its registers; GENERAL = true adds
// both.  At most 512 threads per CTA: the plain path two CTAs per SM (<= 64
// registers, an 8 B spill outside the copy loop), the general path (batch
// credits, head rows) one (118 registers, no spills: short-request batches
// 761 -> 764.5 GB/s, head slices 741 -> 745).
template <int MAXR, typename V, int U, bool GENERAL>
__global__ void __launch_bounds__(512, GENERAL ? 1 : 2)
pull_kernel(const __grid_constant__ PullParams<MAXR> P) {
  extern __shared__ int4 s_runs[];
  const PullArgs& a = P.a;
  pdl_wait();
  mark_start(a, true);
  const int4* runs = stage_runs(a, (MAXR > 0) ? P.runs : a.runs_dev, s_runs);
  const unsigned int lane = threadIdx.x & 31u;
  const unsigned int warps_per_cta = blockDim.x >> 5;
  const unsigned int warp = threadIdx.x >> 5;
  if (GENERAL) publish_empty(a);
  Credit cr;
  // Chunked order: CTA c owns tiles [c*chunk, (c+1)*chunk), its warps take
  // consecutive tiles.  With the default grid (one chunk per CTA) the GPU
  // sweeps the request front to back in launch order, which keeps DRAM
  // row locality: loopback 2970 -> 3330 GB/s vs a persistent grid-stride.
  const unsigned int chunk = warps_per_cta * (a.tiles_per_warp ? a.tiles_per_warp : kTilesPerWarp);
  for (unsigned int c0 = blockIdx.x * chunk; c0 < a.total_tiles; c0 += gridDim.x * chunk)
  for (unsigned int t = c0 + warp; t < c0 + chunk && t < a.total_tiles; t += warps_per_cta) {
    const Tile T = tile_at(a, runs, t);
    if (a.audit && !tile_in_bounds(a, T, t)) {           // bounds audit: count, skip
      if (lane == 0) atomicAdd(a.audit, 1u);
    } else if (GENERAL && a.row_bytes) {
      warp_copy_rows<V, U>(T.dst, T.src, T.bytes, lane, a.row_bytes, a.src_row_stride,
                           a.dst_row_stride);
    } else {
      warp_copy<V, U>(T.dst, T.src, T.bytes, lane);
    }
    if (GENERAL && a.nreqs) credit_tile(a, T, cr, lane == 0, true);   // batched drain
  }
  if (GENERAL && a.nreqs) credit_flush(a, cr, lane == 0, true);
  pdl_trigger();
  complete(a);
}

// ---------------------------------------------------------------------------
// TMA mover: one elected lane per warp runs an S-stage bulk-copy ring
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load(void* smem, const void* gsrc, unsigned int bytes,
                                         uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
  if (bytes)   // a 0-byte (audited-out) tile completes the phase with the arrive alone
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(smem)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_store(void* gdst, const void* smem, unsigned int bytes) {
  if (bytes)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gdst), "r"(smem_u32(smem)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");   // (possibly empty) group
}

// Bounds audit for the TMA ring: a tile outside its layer tensors is counted
// and skipped (0-byte load/store) so the ring's bookkeeping stays intact.
__device__ __forceinline__ Tile audited(const PullArgs& a, Tile T, unsigned int t) {
  if (a.audit && !tile_in_bounds(a, T, t)) {
    atomicAdd(a.audit, 1u);
    T.skip = 1;
  }
  return T;
}
__device__ __forceinline__ void tma_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_wait_done() {   // all but the newest N groups complete
  asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int MAXR>
__global__ void __launch_bounds__(256)
pull_kernel_tma(const __grid_constant__ PullParams<MAXR> P, unsigned int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[(256 / 32) * kMaxStages];   // <= 8 pipes (launch bound)
  const PullArgs& a = P.a;
  // early_loads: only lane 0 of each pipe touches global memory before the
  // kernel ends (claims, bulk loads, bulk stores), and it waits for the
  // preceding grid right before its first store; everything before that
  // reads the kernel parameters, the layer-base tables (written once at
  // open), this launch's tile counter and the SOURCE blocks.
  const bool early = a.early_loads != 0;
  if (!early) pdl_wait();
  mark_start(a, !early);
  const unsigned int warp = threadIdx.x >> 5;
  const unsigned int pipes_per_cta = blockDim.x >> 5;
  const unsigned int npipes = gridDim.x * pipes_per_cta;
  const unsigned int pipe = blockIdx.x * pipes_per_cta + warp;
  const unsigned int S = stages;
  // the run table (if staged) sits after all pipes' rings
  const int4* runs = stage_runs(
      a, (MAXR > 0) ? P.runs : a.runs_dev,
      reinterpret_cast<int4*>(smem + (size_t)pipes_per_cta * S * a.tile_bytes));
  unsigned char* ring = smem + (size_t)warp * S * a.tile_bytes;
  uint64_t* bar = bars + warp * kMaxStages;

  publish_empty(a);
  if ((threadIdx.x & 31u) == 0) {
    for (unsigned int s = 0; s < S; ++s) mbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

    // Tile i of this pipe: pipes sweep the tile space in groups of K
    // consecutive tiles, group g going to pipe g % npipes.  Single requests
    // use K = 1 (plain grid stride).  Batches use K = 16: a pipe's tiles then
    // mostly belong to one request, so a credit (fence + atomic round trip
    // in the issuing lane) is paid per group, not per tile, while the sweep
    // front still moves through the queue in order.
    const unsigned int K = a.nreqs ? 16u : 1u;
    const unsigned int groups = (a.total_tiles + K - 1) / K;
    const unsigned int my_groups = pipe < groups ? (groups - 1 - pipe) / npipes + 1 : 0u;
    unsigned int count = my_groups * K;
    if (my_groups && pipe + (my_groups - 1) * npipes == groups - 1)
      count -= groups * K - a.total_tiles;   // this pipe owns the partial last group
    auto tile_of = [&](unsigned int i) { return ((i / K) * npipes + pipe) * K + i % K; };
    // With a tile counter (a.tile_ctr) tiles are handed out dynamically
    // instead: a pipe claims kClaim consecutive tiles at a time,
    // so the pipes finish within a few tiles of each other (no static
    // imbalance at the tail) and the front still sweeps the request in order.
    // The first ring needs no atomic: tiles [0, npipes * S) are dealt
    // statically, S consecutive ones per pipe, and the counter hands out the
    // rest.  Each pipe keeps one claim in flight ahead of need (issued when
    // it starts on the previous block), so a claim's round trip to L2 never
    // stalls the ring.
    constexpr unsigned int kNone = 0xffffffffu;
    // batches: credit-friendly groups; single pulls: the host's choice
    const unsigned int kClaim = a.nreqs ? K : (a.claim ? a.claim : 4u);
    const unsigned int dealt = min(npipes * S, a.total_tiles);
    unsigned int handed = 0, cur = min(pipe * S, dealt), cur_end = min(pipe * S + S, dealt);
    unsigned int ahead = 0, ahead_n = 0;
    bool have_ahead = false;
    // guided claiming (single pulls): full claims while plenty remains, single
    // tiles for the last ~2 claims' worth per pipe, so the pipes finish together
    const unsigned int guided_tail = a.nreqs ? 0u : npipes * kClaim * 2u;
    auto claim_n = [&](unsigned int seen) -> unsigned int {
      return (seen >= a.total_tiles || a.total_tiles - seen > guided_tail) ? kClaim : 1u;
    };
    auto next = [&]() -> unsigned int {
      if (a.tile_ctr == nullptr) return handed < count ? tile_of(handed++) : kNone;
      if (cur == cur_end) {
        unsigned int base, n;
        if (have_ahead) {
          base = ahead;
          n = ahead_n;
        } else {
          n = claim_n(cur_end);
          base = dealt + atomicAdd(a.tile_ctr, n);
        }
        ahead_n = claim_n(base + n);
        ahead = dealt + atomicAdd(a.tile_ctr, ahead_n);   // consumed a block from now
        have_ahead = true;
        if (base >= a.total_tiles) return kNone;
        cur = base;
        cur_end = min(base + n, a.total_tiles);
      } else if (!have_ahead && cur + 1 == cur_end) {
        ahead_n = claim_n(cur_end);
        ahead = dealt + atomicAdd(a.tile_ctr, ahead_n);   // ahead of the first dynamic block
        have_ahead = true;
      }
      return cur++;
    };
    Tile tiles[kMaxStages];
    // batched drain: a tile is credited to its request(s) only once its bulk
    // store has COMPLETED; credits lag the stores by kCreditLag groups so the
    // write-completion latency stays hidden behind the ring.
    constexpr unsigned int kCreditLag = 4;
    Tile pend[kCreditLag + 1];
    Credit cr;
    unsigned int issued = 0;                 // tiles loaded into the ring so far
    // Programmatic dependent launch: this pipe lets the next pull on the
    // stream launch as soon as it has claimed its last tile (its ring still
    // drains S tiles), so with early loads the next pull's first ring is in
    // flight over the link while this one drains and completes.  Never
    // before this pipe's own wait returned: at most two pulls (one draining,
    // one ramping) hold SMs at a time.
    bool triggered = false, waited = !early, exhausted = false;
    auto claim = [&]() -> unsigned int {
      const unsigned int t = next();
      if (t == kNone) {
        exhausted = true;
        if (waited && !triggered) {
          pdl_trigger();
          triggered = true;
        }
      }
      return t;
    };
    // the first a.early_loads stages are loaded before the wait (the
    // preceding grid's completion also waits for these reads to land, so
    // the early window is sized to its tail, not to the whole ring)
    auto wait_preceding = [&]() {            // stores below: the preceding grid is done
      pdl_wait();
      mark_wait(a);
      waited = true;
      if (exhausted && !triggered) {
        pdl_trigger();
        triggered = true;
      }
    };
    for (unsigned int k = 0; k < S; ++k) {
      if (!waited && k == a.early_loads) wait_preceding();
      const unsigned int t = claim();
      if (t == kNone) break;
      tiles[k] = audited(a, tile_at(a, runs, t), t);
      tma_load(ring + (size_t)k * a.tile_bytes, tiles[k].src, tiles[k].skip ? 0u : tiles[k].bytes,
               &bar[k]);
      ++issued;
    }
    if (!waited) wait_preceding();
    for (unsigned int i = 0; i < issued; ++i) {
      const unsigned int s = i % S;
      mbar_wait(&bar[s], (i / S) & 1u);
      tma_store(tiles[s].dst, ring + (size_t)s * a.tile_bytes, tiles[s].skip ? 0u : tiles[s].bytes);
      if (a.nreqs) pend[i % (kCreditLag + 1)] = tiles[s];
      if (i >= 1) {
        const unsigned int sp = (i - 1) % S;
        tma_wait_read_1();   // store i-1 has finished reading its stage
        // refill the stage of tile i-1 with the ring's tile number i-1+S
        // (only while no claim has failed: tile j always lives in stage j % S)
        if (issued == i - 1 + S) {
          const unsigned int t = claim();
          if (t != kNone) {
            tiles[sp] = audited(a, tile_at(a, runs, t), t);
            tma_load(ring + (size_t)sp * a.tile_bytes, tiles[sp].src,
                     tiles[sp].skip ? 0u : tiles[sp].bytes, &bar[sp]);
            ++issued;
          }
        }
      }
      if (a.nreqs && i >= kCreditLag) {
        tma_wait_done<kCreditLag>();          // store i - kCreditLag complete
        credit_tile(a, pend[(i - kCreditLag) % (kCreditLag + 1)], cr, true, false);
      }
    }
    tma_wait_all();
    if (a.nreqs) {
      const unsigned int first = issued > kCreditLag ? issued - kCreditLag : 0u;
      for (unsigned int j = first; j < issued; ++j)
        credit_tile(a, pend[j % (kCreditLag + 1)], cr, true, false);
      credit_flush(a, cr, true, false);
    }
  }
  __syncwarp();
  pdl_trigger();
  complete(a);
}

// §8 f4 over NVLink: a head-sliced peer's remote unit (block_size rows of
// row_bytes) is contiguous, its local head slice is strided.  Each warp runs
// an S-stage ring: lane 0 bulk-loads whole units from the peer (TMA, the
// efficient NVLink read), and once a stage's mbarrier completes all 32 lanes
// store its rows to the strided slice with 16 B stores (local HBM writes).
template <int MAXR>
__global__ void __launch_bounds__(256)
pull_kernel_tma_rows(const __grid_constant__ PullParams<MAXR> P, unsigned int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[(256 / 32) * kMaxStages];
  const PullArgs& a = P.a;
  pdl_wait();
  mark_start(a, true);
  const unsigned int lane = threadIdx.x & 31u;
  const unsigned int warp = threadIdx.x >> 5;
  const unsigned int pipes_per_cta = blockDim.x >> 5;
  const unsigned int npipes = gridDim.x * pipes_per_cta;
  const unsigned int pipe = blockIdx.x * pipes_per_cta + warp;
  const unsigned int S = stages;
  const int4* runs = stage_runs(
      a, (MAXR > 0) ? P.runs : a.runs_dev,
      reinterpret_cast<int4*>(smem + (size_t)pipes_per_cta * S * a.tile_bytes));
  unsigned char* ring = smem + (size_t)warp * S * a.tile_bytes;
  uint64_t* bar = bars + warp * kMaxStages;
  publish_empty(a);
  if (lane == 0) {
    for (unsigned int s = 0; s < S; ++s) mbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const unsigned int count =
      pipe < a.total_tiles ? (a.total_tiles - pipe + npipes - 1) / npipes : 0u;
  // every lane derives the same (warp-uniform) tiles; lane 0 counts audit hits
  auto fetch = [&](unsigned int k) {
    const unsigned int t = pipe + k * npipes;
    Tile T = tile_at(a, runs, t);
    if (a.audit && !tile_in_bounds(a, T, t)) {
      if (lane == 0) atomicAdd(a.audit, 1u);
      T.skip = 1;
    }
    return T;
  };
  Tile tiles[kMaxStages];
  for (unsigned int k = 0; k < S && k < count; ++k) {
    tiles[k] = fetch(k);
    if (lane == 0)
      tma_load(ring + (size_t)k * a.tile_bytes, tiles[k].src, tiles[k].skip ? 0u : tiles[k].bytes,
               &bar[k]);
  }
  Credit cr;
  const unsigned int vpr = a.row_bytes / 16u;
  for (unsigned int i = 0; i < count; ++i) {
    const unsigned int s = i % S;
    mbar_wait(&bar[s], (i / S) & 1u);
    const Tile T = tiles[s];
    if (!T.skip) {
      const uint4* st = reinterpret_cast<const uint4*>(ring + (size_t)s * a.tile_bytes);
      const unsigned int nv = T.bytes / 16u;
      for (unsigned int c = lane; c < nv; c += 32) {
        const unsigned int r = c / vpr, col = c - r * vpr;
        const uint4 v = st[c];
        asm volatile(KVD_ST_Q ".v4.u32 [%0], {%1,%2,%3,%4};"
                     :: "l"(T.dst + (size_t)r * a.dst_row_stride + (size_t)col * 16u),
                        "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      }
    }
    if (a.nreqs) credit_tile(a, T, cr, lane == 0, true);
    __syncwarp();                       // every lane has read stage s
    const unsigned int k = i + S;
    if (k < count) {
      tiles[s] = fetch(k);
      if (lane == 0) {
        // generic-proxy reads of the stage before the async-proxy refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load(ring + (size_t)s * a.tile_bytes, tiles[s].src,
                 tiles[s].skip ? 0u : tiles[s].bytes, &bar[s]);
      }
    }
  }
  if (a.nreqs) credit_flush(a, cr, lane == 0, true);
  pdl_trigger();
  complete(a);
}

// ---------------------------------------------------------------------------
// Resident pull engine (KVD_OPT_ENGINE): every CTA walks the descriptor ring
// in order; for each request it takes its share of the tiles (one warp per
// 2 KiB tile, grid-wide round robin), then arrives on the request's slot
// counter -- the last CTA to arrive publishes the request exactly like a
// launched pull (complete()).  Descriptors are read over PCIe from pinned
// host memory: the sequence word with acquire, the rest with relaxed
// system-scope loads, the run table by 64 threads at once.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void ld_relaxed_sys_v2(const unsigned long long* p, unsigned long long& x,
                                                  unsigned long long& y) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}

// The engine is ONE thread-block cluster.  CTA 0 is the leader: it polls the
// pinned ring entry of request k (the header and the first kEnginePollRuns
// runs, 16 B LL chunks, one PCIe round trip per poll), validates it from the
// words' flags and writes the per-request fields and the run table into
// every CTA's shared memory (DSMEM, one remote store per thread in
// parallel).  A cluster barrier hands it over (the other CTAs wait there in
// hardware, they never touch host memory); every CTA copies its tiles, and a
// second cluster barrier replaces the per-request arrival counter: after it
// CTA 0 publishes the request with one system-scope release (cumulative over
// the other CTAs' stores, ordered before it by the barrier's release/acquire).
template <typename V, int U>
__global__ void __launch_bounds__(kEngineThreads, 1)
engine_kernel(const __grid_constant__ EngineParams E) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ int4 runs[kEngineMaxRuns];    // this request's run table (written by CTA 0)
  __shared__ PullArgs A;                   // per-request fields written by CTA 0
  __shared__ unsigned long long ll[kEngineLLWords];
  __shared__ int go;
  constexpr unsigned int kPoll = (kEngineLLHeader + 4 * kEnginePollRuns) / 2;   // 16 B chunks
  constexpr unsigned int kPollers = 1;      // tools/ab_patches/engine_pollers4.patch: 4
  static_assert(kPoll <= 64, "one poll = one warp, two 16 B loads per lane at most");
  const unsigned int rank = cluster.block_rank();
  const unsigned int ncta = cluster.num_blocks();
  const unsigned int lane = threadIdx.x & 31u;
  const unsigned int warps = blockDim.x >> 5;
  const unsigned int gw = rank * warps + (threadIdx.x >> 5);
  const unsigned int nw = ncta * warps;
  // the request-independent fields once; CTA 0 writes the per-request ones.
  // The layer-base tables of both sides live in shared memory too, so a
  // tile's address is not a dependent L2 round trip ahead of its data load.
  __shared__ unsigned long long bases[2][kEngineSmemLayers];
  const unsigned int NL = E.base.num_layers;
  const bool smem_bases = NL <= kEngineSmemLayers && E.base.src.table && E.base.dst.table;
  if (smem_bases)
    for (unsigned int l = threadIdx.x; l < NL; l += blockDim.x) {
      bases[0][l] = E.base.src.table[l];
      bases[1][l] = E.base.dst.table[l];
    }
  if (threadIdx.x == 0) {
    A = E.base;
    if (smem_bases) {
      A.src.table = bases[0];
      A.dst.table = bases[1];
    }
  }
  unsigned long long t_seen = 0;           // CTA 0, timing: entry validated
  for (unsigned long long k = E.first;; ++k) {
    const unsigned int r = (unsigned int)(k % kEngineRing);
    if (rank == 0) {
      const unsigned long long* L = E.ll + (size_t)r * kEngineLLWords;
      const unsigned long long want = (unsigned long long)(unsigned int)(k + 1);
      // kPollers warps poll (staggered by a fraction of the PCIe round trip
      // when there are several).  One poll reads the header and the first
      // kEnginePollRuns runs (two 16 B loads per lane at most, both in
      // flight at once); the first warp that validates it copies its words
      // to shared memory.  ONE poller is fastest: every poll in flight also
      // delays the next poll's detection and the publish's system-scope
      // release (C1 over NVLink, 16 CTAs: 11.9 us host to host with 4
      // pollers, 9.2 with 2, 8.3 with 1; profiles/r02_engine_pollers.jsonl;
      // the same in tools/native/pcie_pingpong.cu: 1.55 vs 3.27 us per
      // host -> device -> host round trip).
      const unsigned int w = threadIdx.x >> 5;
      if (threadIdx.x == 0) go = 0;
      __syncthreads();
      if (w < kPollers) {
        __nanosleep(w * 400);
        const unsigned int c1 = lane + 32;                 // second chunk of this lane
        for (;;) {
          unsigned long long x = 0, y = 0, x1 = 0, y1 = 0;
          if (lane < kPoll) ld_relaxed_sys_v2(L + 2 * lane, x, y);
          if (c1 < kPoll) ld_relaxed_sys_v2(L + 2 * c1, x1, y1);
          // nruns is word 7 = chunk 3's second word
          const unsigned int nr = (unsigned int)__shfl_sync(0xffffffffu, y, 3);
          const unsigned int need = kEngineLLHeader +
              (nr == kEngineStop ? 0u : 4u * min(nr, kEnginePollRuns));
          const bool ok = (lane >= kPoll || ((2 * lane >= need || (x >> 32) == want) &&
                                             (2 * lane + 1 >= need || (y >> 32) == want))) &&
                          (c1 >= kPoll || ((2 * c1 >= need || (x1 >> 32) == want) &&
                                           (2 * c1 + 1 >= need || (y1 >> 32) == want)));
          const bool all = __all_sync(0xffffffffu, ok);
          if (all && lane == 0 && atomicCAS(&go, 0, 1) == 0) go = 2 + (int)w;   // winner
          __syncwarp();
          const int g = *(volatile int*)&go;
          if (g == 2 + (int)w) {
            if (lane < kPoll) {
              ll[2 * lane] = x;
              ll[2 * lane + 1] = y;
            }
            if (c1 < kPoll) {
              ll[2 * c1] = x1;
              ll[2 * c1 + 1] = y1;
            }
          }
          if (g) break;
        }
      }
      __syncthreads();
      t_seen = globaltimer();
      const unsigned int nr = (unsigned int)ll[7];
      const unsigned int nwords = nr == kEngineStop ? 0u : 4u * nr;
      if (nwords > 4 * kEnginePollRuns) {      // beyond the polled runs: wait for each word
        for (unsigned int q = 4 * kEnginePollRuns + threadIdx.x; q < nwords; q += blockDim.x) {
          unsigned long long v;
          do {
            v = ld_relaxed_sys(L + kEngineLLHeader + q);
          } while ((v >> 32) != want);
          ll[kEngineLLHeader + q] = v;
        }
        __syncthreads();
      }
      // the descriptor into every CTA's shared memory (distributed shared
      // memory), one remote store per thread: thread c < ncta writes CTA c's
      // per-request fields, the rest of the threads the run words
      if (threadIdx.x < ncta) {
        PullArgs* Ac = cluster.map_shared_rank(&A, threadIdx.x);
        Ac->nruns = nr;                        // kEngineStop: exit
        if (nr != kEngineStop) {
          const unsigned int slot = (unsigned int)ll[6];
          Ac->token = (ll[0] & 0xffffffffull) | (ll[1] << 32);
          Ac->request_id = (ll[2] & 0xffffffffull) | (ll[3] << 32);
          Ac->mbox_pos = (ll[4] & 0xffffffffull) | (ll[5] << 32);
          Ac->tiles_per_lp = (unsigned int)ll[8];
          Ac->total_tiles = (unsigned int)ll[9];
          Ac->flag = E.base.flag + slot;
          Ac->gt_out = (ll[10] & 1u) ? E.base.gt_out + 4 * (size_t)slot : nullptr;
        }
      }
      for (unsigned int i = threadIdx.x; i < ncta * nwords; i += blockDim.x) {
        const unsigned int c = i / nwords, q = i - c * nwords;
        reinterpret_cast<int*>(cluster.map_shared_rank(runs, c))[q] =
            (int)(unsigned int)ll[kEngineLLHeader + q];
      }
    }
    cluster.sync();                          // the descriptor is valid in every CTA
    if (A.nruns == kEngineStop) return;
    const unsigned long long t_handed = globaltimer();   // timing: descriptor in every CTA
    for (unsigned int t = gw; t < A.total_tiles; t += nw) {
      const Tile T = tile_at(A, runs, t);
      if (A.audit && !tile_in_bounds(A, T, t)) {          // bounds audit: count, skip
        if (lane == 0) atomicAdd(A.audit, 1u);
        continue;
      }
      warp_copy<V, U>(T.dst, T.src, T.bytes, lane);
    }
    // every CTA's tiles landed: the barrier's cluster-scope release/acquire
    // puts the other CTAs' stores before CTA 0's system-scope release in
    // causality order (no per-thread gpu-scope fence needed)
    cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
      if (A.gt_out != nullptr) {             // timed: CTA 0 saw the entry -> all tiles landed
        const unsigned long long t1 = globaltimer();
        volatile unsigned long long* o = A.gt_out;
        o[0] = t1 - t_seen;
        o[1] = t_seen;
        o[2] = t_handed;                     // the span's "wait": descriptor handed over
        o[3] = t1;
      }
      publish_token(A, A.flag, A.token, A.request_id, A.mbox_pos);
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(E.done + r), "l"(k + 1)
                   : "memory");
    }
    // A and runs are rewritten for the next request only after the next
    // iteration's poll: every CTA has passed the barrier above by then
  }
}

// ---------------------------------------------------------------------------
// Link calibration (kvd_peer_calibrate, SURVEY.md §8 d "fraction of the
// measured achievable link ceiling"): pure ingress.  One elected lane per
// CTA runs an S-stage ring of kCalibChunk bulk loads from the peer-mapped
// source layers into shared memory and discards them -- no stores, no block
// table, no completion -- so the rate is what this GPU's SMs can pull from
// the mapping at all.  The launch reads the region `passes` times: chunk i
// is chunk j = i % total_chunks of the region, byte (j % layer_chunks) *
// kCalibChunk of layer j / layer_chunks; CTA c takes chunks c, c + G, ...
// (one long launch, so its ramp and tail are a negligible part of it).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32)
calib_read_kernel(const unsigned long long* __restrict__ bases, unsigned long long layer_chunks,
                  unsigned long long total_chunks, unsigned int passes, unsigned int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar[kMaxStages];
  if (threadIdx.x != 0) return;
  for (unsigned int s = 0; s < stages; ++s) mbar_init(&bar[s]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto src = [&](unsigned long long i) {
    const unsigned long long j = i % total_chunks;
    return reinterpret_cast<const char*>(bases[j / layer_chunks] + (j % layer_chunks) * kCalibChunk);
  };
  const unsigned long long end = total_chunks * passes;
  unsigned long long next = blockIdx.x;
  unsigned int issued = 0;
  for (unsigned int s = 0; s < stages && next < end; ++s, next += gridDim.x, ++issued)
    tma_load(smem + (size_t)s * kCalibChunk, src(next), kCalibChunk, &bar[s]);
  for (unsigned int i = 0; i < issued; ++i) {
    const unsigned int s = i % stages;
    mbar_wait(&bar[s], (i / stages) & 1u);
    // the stage was written by the async proxy and never read: refill at once
    if (next < end) {
      tma_load(smem + (size_t)s * kCalibChunk, src(next), kCalibChunk, &bar[s]);
      next += gridDim.x;
      ++issued;
    }
  }
}

__global__ void flag_kernel(unsigned long long* flag, unsigned long long token,
                            unsigned long long* mbox, unsigned long long mbox_pos,
                            unsigned long long request_id) {
  // no data: earlier stream work is ordered by the stream itself
  PullArgs a{};
  a.mbox = mbox;
  publish_token(a, flag, token, request_id, mbox_pos);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int MAXR>
void fill(PullParams<MAXR>& P, const PullArgs& args, const int4* runs_host) {
  P.a = args;
  if (MAXR > 0)
    for (unsigned int r = 0; r < args.nruns; ++r) P.runs[r] = runs_host[r];
}

// Stage run tables of more than 64 runs (a binary search of >= 7 steps) when
// they fit next to whatever else the kernel keeps in shared memory.
constexpr unsigned int kStageMinRuns = 64;
constexpr size_t kStageMaxBytes = 32 * 1024;

// Launch with programmatic stream serialisation (see pdl_wait/pdl_trigger).
template <typename Kernel, typename... Args>
cudaError_t launch_pdl(Kernel kernel, unsigned int ctas, unsigned int threads, size_t smem,
                       cudaStream_t stream, const Args&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int MAXR, typename V, int U>
cudaError_t launch_t(const PullArgs& args, const int4* runs_host, unsigned int ctas,
                     unsigned int threads, cudaStream_t stream) {
  PullParams<MAXR> P;
  fill(P, args, runs_host);
  const size_t table = (size_t)args.nruns * sizeof(int4);
  const bool stage = args.nruns > kStageMinRuns && table <= kStageMaxBytes;
  P.a.smem_runs = stage ? 1u : 0u;
  if (args.nreqs || args.row_bytes)
    return launch_pdl(pull_kernel<MAXR, V, U, true>, ctas, threads, stage ? table : 0, stream, P);
  return launch_pdl(pull_kernel<MAXR, V, U, false>, ctas, threads, stage ? table : 0, stream, P);
}

template <int MAXR, bool ROWS>
cudaError_t launch_tma_t(const PullArgs& args, const int4* runs_host, unsigned int ctas,
                         unsigned int threads, unsigned int stages, cudaStream_t stream) {
  auto kernel = ROWS ? pull_kernel_tma_rows<MAXR> : pull_kernel_tma<MAXR>;
  PullParams<MAXR> P;
  fill(P, args, runs_host);
  const size_t ring = (size_t)(threads / 32) * stages * args.tile_bytes;
  const size_t table = (size_t)args.nruns * sizeof(int4);
  const bool stage = args.nruns > kStageMinRuns && table <= kStageMaxBytes &&
                     ring + table <= 225 * 1024;
  P.a.smem_runs = stage ? 1u : 0u;
  const size_t smem = ring + (stage ? table : 0);
  // The opt-in limit is per function and device (the static mbarrier array
  // counts against the 48 KiB default too): raise it once per device to the
  // maximum and remember that.
  static std::atomic<unsigned long long> raised{0};   // bit d: device d done
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(raised.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         225 * 1024);
    if (e != cudaSuccess) return e;
    raised.fetch_or(bit);
  }
  return launch_pdl(kernel, ctas, threads, smem, stream, P, stages);
}

template <typename V, int U>
cudaError_t launch_v(const PullArgs& args, const int4* runs_host, unsigned int ctas,
                     unsigned int threads, cudaStream_t stream) {
  if (args.nruns <= (unsigned)kRunsTiny)
    return launch_t<kRunsTiny, V, U>(args, runs_host, ctas, threads, stream);
  if (args.nruns <= (unsigned)kRunsSmall)
    return launch_t<kRunsSmall, V, U>(args, runs_host, ctas, threads, stream);
  if (args.nruns <= (unsigned)kRunsMid)
    return launch_t<kRunsMid, V, U>(args, runs_host, ctas, threads, stream);
  if (args.nruns <= (unsigned)kRunsLarge)
    return launch_t<kRunsLarge, V, U>(args, runs_host, ctas, threads, stream);
  return launch_t<0, V, U>(args, runs_host, ctas, threads, stream);
}

template <bool ROWS>
cudaError_t launch_tma_r(const PullArgs& args, const int4* runs_host, unsigned int ctas,
                         unsigned int threads, unsigned int stages, cudaStream_t stream) {
  if (args.nruns <= (unsigned)kRunsTiny)
    return launch_tma_t<kRunsTiny, ROWS>(args, runs_host, ctas, threads, stages, stream);
  if (args.nruns <= (unsigned)kRunsSmall)
    return launch_tma_t<kRunsSmall, ROWS>(args, runs_host, ctas, threads, stages, stream);
  if (args.nruns <= (unsigned)kRunsMid)
    return launch_tma_t<kRunsMid, ROWS>(args, runs_host, ctas, threads, stages, stream);
  if (args.nruns <= (unsigned)kRunsLarge)
    return launch_tma_t<kRunsLarge, ROWS>(args, runs_host, ctas, threads, stages, stream);
  return launch_tma_t<0, ROWS>(args, runs_host, ctas, threads, stages, stream);
}

cudaError_t launch_tma(const PullArgs& args, const int4* runs_host, unsigned int ctas,
                       unsigned int threads, unsigned int stages, cudaStream_t stream) {
  // head-sliced peers (row_bytes > 0): bulk loads, warp-wide strided stores
  return args.row_bytes ? launch_tma_r<true>(args, runs_host, ctas, threads, stages, stream)
                        : launch_tma_r<false>(args, runs_host, ctas, threads, stages, stream);
}

template <int MAXR, typename V, int U>
int occ(unsigned int threads) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, pull_kernel<MAXR, V, U, true>,
                                                    (int)threads, 0) != cudaSuccess)
    return 1;
  return n > 0 ? n : 1;
}

}  // namespace

unsigned int max_param_runs() { return (unsigned int)kRunsLarge; }
unsigned int max_stages() { return (unsigned int)kMaxStages; }
unsigned int lsu_tiles_per_warp() { return kTilesPerWarp; }

cudaError_t launch_pull(const PullArgs& args, const int4* runs_host, int variant,
                        unsigned int ctas, unsigned int threads, unsigned int stages,
                        cudaStream_t stream) {
  if (variant == kTma) return launch_tma(args, runs_host, ctas, threads, stages, stream);
  if (variant == kLsu32) return launch_v<V32, 4>(args, runs_host, ctas, threads, stream);
  return launch_v<V16, 8>(args, runs_host, ctas, threads, stream);
}

cudaError_t launch_engine(const EngineParams& params, int variant, unsigned int ctas,
                          cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kEngineThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;   // the whole grid is one cluster
  attr[0].val.clusterDim.x = ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto kernel = variant == kLsu32 ? engine_kernel<V32, 4> : engine_kernel<V16, 8>;
  if (ctas > 8) {   // 16: a non-portable cluster size (B200 allows it on request)
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchKernelEx(&cfg, kernel, params);
}

cudaError_t launch_flag_only(unsigned long long* flag, unsigned long long token,
                             unsigned long long* mbox, unsigned long long mbox_pos,
                             unsigned long long request_id, cudaStream_t stream) {
  flag_kernel<<<1, 1, 0, stream>>>(flag, token, mbox, mbox_pos, request_id);
  return cudaGetLastError();
}

cudaError_t launch_calib_read(const unsigned long long* bases, unsigned long long layer_chunks,
                              unsigned long long total_chunks, unsigned int passes,
                              unsigned int ctas, unsigned int stages, cudaStream_t stream) {
  const size_t smem = (size_t)stages * kCalibChunk;
  cudaError_t e = cudaFuncSetAttribute(calib_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  calib_read_kernel<<<ctas, 32, smem, stream>>>(bases, layer_chunks, total_chunks, passes, stages);
  return cudaGetLastError();
}

int pull_ctas_per_sm(int variant, unsigned int threads, unsigned int nruns) {
  if (variant == kTma) return 1;   // shared-memory ring sized for one CTA per SM
  const bool big = nruns > (unsigned)kRunsLarge;
  if (variant == kLsu32) return big ? occ<0, V32, 4>(threads) : occ<kRunsSmall, V32, 4>(threads);
  return big ? occ<0, V16, 8>(threads) : occ<kRunsSmall, V16, 8>(threads);
}

}  // namespace kvd
