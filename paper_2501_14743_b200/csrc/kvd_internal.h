// kvd_internal.h -- interface between the host core (kvd_core.cpp) and the
// sm_100a kernels (kvd_pull.cu).  Not part of the public ABI (include/kvd.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kvd {

// Release mailbox (Complete() -> prefill, "sends the request ID to the
// prefill worker"): pinned HOST memory owned by the EXPORTER (a memfd the
// importers map and register with cudaHostRegister), so the prefill host
// reads completions with plain loads -- no CUDA call, no NVLink atomic.
// u64 words: a header of kMailboxHeaderWords (magic, rings, entries, then
// per ring an owner word and a next-position word), then kMailboxRings
// single-producer rings of kReleaseRing entries.  An importer claims one
// ring at open (CPU compare-and-swap on its owner word) and assigns each
// request a position p in issue order; the completing CTA writes entry
// p % kReleaseRing as two 64-bit words {tag | id_lo32, tag | id_hi32} with
// tag = low32(p + 1) << 32 (each word is single-copy atomic, so the reader
// accepts an entry once both words carry the expected tag; no fence and no
// read-modify-write over the link).
constexpr unsigned int kReleaseRing = 4096;
constexpr unsigned int kMailboxRings = 64;
constexpr size_t kMailboxHeaderWords = 8 + 2 * (size_t)kMailboxRings;
constexpr size_t kMailboxWords = kMailboxHeaderWords + 2 * (size_t)kReleaseRing * kMailboxRings;
constexpr unsigned long long kMailboxMagic = 0x584f42444b56444bull;   // "KDVKDBOX"

// Where layer l of one side starts: table ? table[l] : base + l * step.
// The peer's source side uses a device table of IPC-mapped prefill layer
// bases; the baseline staging buffer uses the affine form.
struct SideAddr {
  const unsigned long long* table;  // device array [num_layers] or nullptr
  unsigned long long base;
  unsigned long long step;
  long long plane_stride;           // bytes between the K and V sub-tensors of a block
  long long block_stride;           // bytes between consecutive blocks
};

// Everything one pull launch needs except the run table.
//
// Work decomposition: the request is a set of
// segments (layer l, plane p, run r).  Each segment is cut into "tiles" of at
// most tile_bytes that never cross a segment; one WARP copies one tile.
// runs[r] = {src_start, dst_start, len, tile_end} where tile_end is the
// inclusive prefix sum of tiles over runs 0..r within one (layer, plane).
struct PullArgs {
  SideAddr src, dst;
  unsigned long long unit_bytes;    // bytes of one (block, plane) unit: span, or 2*span when K,V adjacent on both sides
  unsigned int num_layers;
  unsigned int planes;              // 2, or 1 when the unit folds K and V
  unsigned int tile_bytes;          // multiple of 512
  unsigned int contiguous;          // 1: a run is one byte-contiguous segment on both sides
  unsigned int tiles_per_unit;      // ceil(unit_bytes / tile_bytes) (non-contiguous runs)
  unsigned int nruns;
  unsigned int tiles_per_lp;        // tiles of one (layer, plane) = runs[nruns-1].w
  unsigned int total_tiles;         // num_layers * planes * tiles_per_lp
  unsigned int* counter;            // per-slot arrive counter (device, zero at launch)
  unsigned long long* flag;         // per-slot completion word (pinned, host-mapped)
  unsigned long long token;         // value stored to *flag when every byte has landed
  unsigned long long request_id;    // posted to the exporter's release mailbox (if any)
  unsigned long long* mbox;         // this importer's ring of the exporter's mailbox, mapped
                                    // here (device pointer to host memory; nullptr: none)
  unsigned long long mbox_pos;      // ring position of this request (batches: of request 0)
  const int4* runs_dev;             // run table in device memory when nruns > params capacity
  unsigned int remote_stores;       // 1: stores target a peer GPU (push) -> system-scope fences
  unsigned int tiles_per_warp;      // LSU chunk = warps * this (host sets it; grid follows)
  unsigned int smem_runs;           // 1: the kernel copies the run table into shared memory
                                    //    (set by launch_pull when it fits)
  // Bounds audit (KVD_OPT_AUDIT; compute-sanitizer is closed on this pool):
  // when non-null every tile checks that its source and destination bytes
  // lie inside their layer tensors, counts violations here and skips them.
  unsigned int* audit;
  unsigned long long src_layer_bytes, dst_layer_bytes;
  // Device-side timeline (KVD_OPT_TIMING, single pulls), %globaltimer ns:
  // every CTA atomicMin's its start into gt_start[0]; the pipes that read
  // early atomicMin the moment their griddepcontrol.wait returned into
  // gt_start[1] (the others: their start); the last CTA writes {end - start,
  // start, wait, end} to gt_out[0..3] (pinned, host-mapped) before it
  // releases the slot word and resets gt_start to ~0.  nullptr: off.
  unsigned long long* gt_start;
  unsigned long long* gt_out;
  // TMA single pulls: per-slot tile counter (device, zero at launch) from
  // which pipes claim tiles dynamically; reset by the last CTA.  nullptr:
  // static grid-stride order.
  unsigned int* tile_ctr;
  unsigned int claim;               // tiles per dynamic claim (single pulls; 0: 4)
  // TMA single pulls over NVLink: lane 0 of each pipe claims and issues its
  // first early_loads ring stages of bulk loads from the SOURCE before
  // griddepcontrol.wait (0: none), so the ramp of a pull overlaps the drain
  // and completion tail of the pull before it on the stream.  Only the
  // source (the prefill's finished cache) is read early; every store into
  // the decode cache waits.
  unsigned int early_loads;
  // Batches: the launch's own arrival/tile counters live with its
  // descriptor buffer; the last CTA resets them and then releases done_seq
  // into *done_word (pinned, host-mapped), after which the host may reuse
  // the buffer and its counters.
  unsigned long long* done_word;
  unsigned long long done_seq;

  // TP-resharding (§8 f4): row_bytes > 0 makes every unit block_size rows
  // of row_bytes, src_row_stride / dst_row_stride apart, and shifts the
  // destination by dst_unit_offset (the head slice).  One tile = one unit.
  unsigned int row_bytes;
  unsigned int src_row_stride;
  unsigned int dst_row_stride;
  unsigned long long dst_unit_offset;

  // Batched drain: nreqs > 0 means several requests share
  // this launch and each is completed on its own.  The concatenated block
  // table is coalesced as one queue (runs may span requests, fig:queue);
  // every tile credits its bytes to the request(s) that own its blocks and
  // the credit that completes a request publishes that request's token.
  unsigned int nreqs;
  // run-major tile order (batches): runs[r].w is the inclusive prefix of
  // tiles_r * num_layers * planes over runs, so a run's tiles (all layers and
  // both planes) are consecutive and requests finish in queue order.
  unsigned int run_major;
  const unsigned int* run_pos;      // [nruns] position of each run's first entry in the batch
  const uint4* reqs;                // [nreqs] {first entry, slot, total bytes lo, hi}
  const unsigned long long* tokens; // [nreqs]
  const unsigned long long* req_ids;  // [nreqs] ids posted to the release mailbox
  unsigned long long* bytectr;      // per-slot byte counters (device, zero when idle)
  unsigned long long* flags;        // per-slot completion words (pinned, host-mapped)
};

// Resident pull engine (KVD_OPT_ENGINE): a persistent kernel of a few CTAs
// that drains a ring of request descriptors the host writes into pinned,
// mapped memory -- the paper's transaction queue posted
// straight to the device, so a short request costs neither a launch call nor
// the launch latency.
//
// Ring entries use a low-latency ("LL") encoding: every 32-bit field is
// stored as one 64-bit word {flag = low32(position + 1), value}, each word
// single-copy atomic, so the engine validates an entry from the words it
// read -- header and the first kEnginePollRuns runs in ONE PCIe round trip
// of 16 B loads -- without a separate sequence word and a second read.
// Word layout: [0,1] token, [2,3] request id, [4,5] mailbox position (lo,
// hi), [6] slot, [7] nruns (kEngineStop: stop marker), [8] tiles per
// (layer, plane), [9] total tiles, [10] flags (bit 0: timed), [11] pad,
// then 4 words {src_start, dst_start, len, tile prefix} per run.
constexpr unsigned int kEngineRing = 128;          // descriptors
constexpr unsigned int kEngineMaxRuns = 64;        // larger tables take the launch path
constexpr unsigned int kEngineTile = 2048;         // bytes per warp work item
constexpr unsigned int kEngineThreads = 512;
constexpr unsigned int kEngineMaxCtas = 16;        // one thread-block cluster (> 8: non-portable)
constexpr unsigned int kEngineSmemLayers = 128;    // layer-base tables kept in shared memory
constexpr unsigned int kEngineLLHeader = 12;
constexpr unsigned int kEngineLLWords = kEngineLLHeader + 4 * kEngineMaxRuns;
// one poll reads the header and this many runs (two 16 B loads per lane):
// fragmented short requests rarely have more, and more words would cost a
// second PCIe round trip (C1 with 16 runs: entry seen -> handed over 1.7 us)
constexpr unsigned int kEnginePollRuns = 16;
constexpr unsigned int kEngineStop = 0xffffffffu;  // nruns of a stop marker
struct EngineParams {
  PullArgs base;                    // request-independent fields (tiling, sides, slots)
  const unsigned long long* ll;     // device pointer to the pinned ring [kEngineRing][LLWords]
  unsigned long long first;         // ring position this launch starts at
  unsigned long long* done;         // pinned [kEngineRing]: done[k % ring] = k + 1 once
                                    // request k completed (its descriptor may be reused)
};

enum Variant : int { kLsu16 = 1, kLsu32 = 2, kTma = 4 };

// Largest run table that travels inside the kernel parameters.
unsigned int max_param_runs();
// Deepest TMA ring (stages per pipe).
unsigned int max_stages();
// LSU mover: tiles each warp copies per CTA chunk (grid = tiles / (warps * this)).
unsigned int lsu_tiles_per_warp();

// Launch one pull kernel.  runs_host must hold args.nruns entries when
// args.nruns <= max_param_runs(); otherwise args.runs_dev is used.
// variant kTma: threads/32 pipes per CTA, each an S-stage ring of tile_bytes
// buffers in dynamic shared memory (stages in [2, max_stages()]).
cudaError_t launch_pull(const PullArgs& args, const int4* runs_host, int variant,
                        unsigned int ctas, unsigned int threads, unsigned int stages,
                        cudaStream_t stream);

// Completion with no bytes (n = 0, or after copy-engine copies); also posts
// request_id at ring position mbox_pos of the exporter's release mailbox when
// mbox is non-null.
cudaError_t launch_flag_only(unsigned long long* flag, unsigned long long token,
                             unsigned long long* mbox, unsigned long long mbox_pos,
                             unsigned long long request_id, cudaStream_t stream);

// Launch the resident engine: ONE cluster of `ctas` (<= kEngineMaxCtas) CTAs
// of kEngineThreads on `stream`; it runs until it reads a stop marker.
// variant kLsu32 (32 B lanes) or kLsu16.
cudaError_t launch_engine(const EngineParams& params, int variant, unsigned int ctas,
                          cudaStream_t stream);

// Link calibration (kvd_peer_calibrate): `ctas` CTAs each run an
// `stages`-deep ring of kCalibChunk bulk loads over total_chunks chunks of
// the layers at bases[] (device array; layer_chunks chunks per layer),
// `passes` times in one launch, and discard them.  stages in
// [1, kCalibMaxStages].
constexpr unsigned int kCalibChunk = 32768;
constexpr unsigned int kCalibMaxStages = 7;   // 224 KiB of shared memory
cudaError_t launch_calib_read(const unsigned long long* bases, unsigned long long layer_chunks,
                              unsigned long long total_chunks, unsigned int passes,
                              unsigned int ctas, unsigned int stages, cudaStream_t stream);

// Resident CTAs per SM of the pull kernel for the given threads per CTA.
int pull_ctas_per_sm(int variant, unsigned int threads, unsigned int nruns);

}  // namespace kvd
