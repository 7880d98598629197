/*
 * kvd.h -- C ABI of the B200-native paged-KV pull (KVDirect, arXiv 2501.14743).
 *
 * The library moves a finished prefill request's paged KV cache into a
 * decode worker's paged KV cache by PULLING it: one kernel, launched on the
 * decode GPU, loads the source blocks straight out of the prefill GPU's HBM
 * over NVLink 5 / NVSwitch (CUDA IPC mapping) and stores them into the
 * decode cache's blocks, for every layer and both K and V, then raises a
 * per-request completion flag the host polls (§4.3 pull mode,
 * P:L404 "pull-mode performs KV cache reads for all layers in a single
 * shot"; §4.1 Connect/Transfer/Complete).
 *
 * Citations: P:Lnnn = line nnn of the paper's source.
 *
 * Conventions for every entry point
 *   - Return a kvd_status; 0 is success, negative is an error.  No entry
 *     point aborts or throws across the ABI.  kvd_last_error() returns a
 *     thread-local detail string for the most recent failure on the thread.
 *   - Pointers named *_dev are device pointers (CUDA global memory); all
 *     other pointers are host pointers.  `stream` is a cudaStream_t passed
 *     as void* (NULL = legacy default stream) of the device that owns the
 *     decode-side cache.
 *   - Host arrays (block ids, blobs) are borrowed for the duration of the
 *     call only; the library copies what it keeps.
 *   - Every entry point saves and restores the calling thread's current
 *     CUDA device.
 *   - Entry points marked [host-only] make no CUDA call and work on a
 *     machine without a GPU.
 *   - Threading (SURVEY §8 b): calls that issue transfers or change a peer
 *     (kvd_pull, kvd_pull_batch, kvd_push, kvd_peer_set, ...) are serialised
 *     per peer by an internal mutex; different peers are independent.
 *     kvd_poll_done, kvd_poll_many and kvd_wait_done take NO lock and make
 *     no CUDA call: a decode thread polling completions never waits behind
 *     another thread's validation, planning or kernel launch (P:L380-382:
 *     completions never block reads).  If several threads poll the same
 *     request concurrently exactly one of them reports it done.
 *     kvd_poll_released (exporter side) makes no CUDA call.
 */
#ifndef KVD_H
#define KVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVD_ABI_VERSION 3

#if defined(__GNUC__)
#define KVD_API __attribute__((visibility("default")))
#else
#define KVD_API
#endif

typedef enum {
  KVD_OK = 0,
  KVD_EINVAL = -1,   /* bad argument: null pointer, duplicate destination id, unknown request */
  KVD_ERANGE = -2,   /* a block id outside [0, num_blocks) of its side */
  KVD_ELAYOUT = -3,  /* unsupported / incompatible / misaligned layout */
  KVD_EHANDLE = -4,  /* IPC export or import failed, malformed blob */
  KVD_ECUDA = -5,    /* a CUDA runtime call failed (detail in kvd_last_error) */
  KVD_ENOMEM = -6,   /* host or device allocation failed */
  KVD_EBUSY = -7,    /* request id already in flight on this peer, or no free completion slot */
  KVD_ESTATE = -8    /* object used in the wrong state (e.g. closed) */
} kvd_status;

/* Element type of the cache.  Only its size matters: the pull is a bit copy. */
typedef enum { KVD_FP16 = 0, KVD_BF16 = 1, KVD_FP8 = 2, KVD_FP32 = 3 } kvd_dtype;

/*
 * Tensor-centric metadata of one side's paged KV cache (Fig. 5).
 * vLLM keeps one tensor per layer; all layers share this layout.  The
 * logical tensor is cache[B][KV][L][H][D]: B = num_blocks,
 * KV = 2 (K and V), L = block_size tokens, H = num_kv_heads (per shard),
 * D = head_dim.  `stride` holds ELEMENT strides in that Dims order; all
 * zeros selects Fig. 5's layout, stride = (L*H*D, B*L*H*D, H*D, D, 1),
 * i.e. vLLM's flash layout (2, num_blocks, block_size, heads, head_dim).
 * Requirements (else KVD_ELAYOUT): strides > 0; the (L, H, D) sub-tensor of
 * a block is self-contiguous (reading R4); the element offsets of
 * distinct (B, KV) pairs do not overlap; span and byte strides are
 * multiples of 16 bytes.
 */
typedef struct {
  uint32_t num_layers;
  uint32_t num_kv_heads;
  uint32_t head_dim;
  uint32_t block_size;
  uint32_t num_blocks;
  uint32_t dtype;        /* kvd_dtype */
  int64_t stride[5];     /* element strides, Dims order (B, KV, L, H, D) */
} kvd_layout;

/* Byte geometry derived from a kvd_layout. */
typedef struct {
  uint64_t span_bytes;          /* one (block, K|V) sub-tensor: "shape x stride" */
  int64_t block_stride_bytes;   /* e * stride[B] */
  int64_t plane_stride_bytes;   /* e * stride[KV] */
  uint64_t layer_bytes;         /* bytes one layer tensor spans from its base */
  uint32_t elem_bytes;
  uint32_t kv_adjacent;         /* 1 if plane_stride == span: K,V of a block are one 2*span unit */
} kvd_geometry;

/* A coalesced run: blocks src_start+j -> dst_start+j for j < len. */
typedef struct {
  int32_t src_start;
  int32_t dst_start;
  uint32_t len;
} kvd_run;

/* What the most recent kvd_pull on a peer did (for benchmarks and tests). */
typedef struct {
  uint64_t request_id;
  uint64_t bytes;        /* algorithmic bytes moved: n * layers * 2 * span */
  uint32_t blocks;       /* n */
  uint32_t runs;         /* coalesced runs m (<= n) */
  uint64_t segments;     /* contiguous byte segments: layers * planes * (runs or blocks) */
  uint64_t tiles;        /* warp work items */
  uint32_t ctas;         /* grid size */
  uint32_t threads;      /* threads per CTA */
  uint32_t variant;      /* kvd_variant actually launched */
  uint32_t launches;     /* kernels (or copies) issued by the call */
} kvd_pull_info;

typedef enum {
  KVD_VARIANT_AUTO = 0,  /* default: the library's choice -- the TMA ring over NVLink, LSU32
                            for loopback, requests <= 2 MiB and batches of short requests
                             */
  KVD_VARIANT_LSU = 1,   /* SM loads 16 B/lane from the peer, stores locally */
  KVD_VARIANT_LSU32 = 2, /* 32 B/lane (sm_100 256-bit ld/st); needs 32 B alignment */
  KVD_VARIANT_CE = 3,    /* copy engine: one cudaMemcpyAsync per segment (comparator only) */
  KVD_VARIANT_TMA = 4    /* one lane per warp runs an S-stage cp.async.bulk ring peer HBM ->
                            shared memory -> local HBM; saturates NVLink with few SMs */
} kvd_variant;

typedef enum {
  KVD_OPT_MAX_CTAS = 0,     /* cap on the pull grid (default: SMs * resident CTAs/SM) */
  KVD_OPT_TILE_BYTES = 1,   /* bytes per warp work item, multiple of 512 (default: auto policy;
                               16384 for an explicit variant) */
  KVD_OPT_COALESCE = 2,     /* 1 (default) merge bi-contiguous runs; 0 one run per block (E10 ablation) */
  KVD_OPT_VARIANT = 3,      /* kvd_variant */
  KVD_OPT_THREADS = 4,      /* threads per CTA: multiple of 32; LSU 32..512 (default 512);
                               TMA: threads/32 pipes per CTA, 32..256 (default 96 for an
                               explicit TMA variant; the auto policy picks its own) */
  KVD_OPT_STAGES = 5,       /* TMA ring depth per pipe, 2..8 (default 4; auto: 6 or 3); with an
                               explicit TMA variant pipes * stages * tile_bytes must fit in
                               225 KiB of shared memory (KVD_EINVAL otherwise); under AUTO the
                               library fits THREADS / STAGES / TILE_BYTES to the ring (at most
                               8 pipes, then fewer stages and pipes) or takes the LSU mover */
  KVD_OPT_AUDIT = 6,        /* 1: every tile checks that it stays inside its layer tensors on
                               both sides (every mover, the resident engine included);
                               violations are counted (kvd_peer_audit) and not copied.  A
                               test/debug mode; 0 (default) off */
  KVD_OPT_TIMING = 7,       /* 1: record CUDA events right around every pull kernel on the
                               caller's stream (kvd_peer_kernel_time sums them) and have single
                               pulls measure first-CTA-start -> last-CTA-done with %globaltimer
                               (kvd_peer_device_time).  2: the %globaltimer spans only (no events
                               between launches, so back-to-back pulls still overlap launch and
                               tail).  0 (default) off */
  KVD_OPT_STREAMS = 8,      /* 0 or 1 (default): every transfer runs on the caller's stream, in
                               stream order.  k in [2, 8]: a transfer still waits for the work
                               already on the caller's stream, but runs on the next of k library
                               streams, so consecutive transfers overlap (their launch, ramp and
                               completion tails hide behind each other); the caller's stream does
                               NOT wait for it -- observe completion with kvd_poll_done /
                               kvd_wait_done (the paper's decode worker polls) or order a
                               stream after it with kvd_stream_wait.  Changing it synchronises the
                               library streams */
  KVD_OPT_EARLY_LOADS = 9,  /* k in [0, 8], default 2: a pull with the TMA mover reads the first
                               k stages of every pipe's ring from the SOURCE before the
                               preceding kernel on the stream has finished (programmatic
                               dependent launch), so consecutive pulls overlap ramp and tail;
                               its stores into the decode cache still wait for that kernel.
                               The caller guarantees that the source blocks are not written by
                               work queued earlier on the same stream (in the paper's flow they
                               are the prefill worker's finished cache, written by another
                               process).  0: every access waits (strict stream order) */
  KVD_OPT_ENGINE = 10       /* c in [0, 16], default 0 (off): the resident pull engine for short
                               requests -- one thread-block cluster of c CTAs (a persistent
                               kernel; c > 8 is a non-portable cluster size B200 allows)
                               drains a ring of request descriptors the host writes into
                               pinned memory (the paper's transaction queue, P:L373-378,
                               posted straight to the device), so a kvd_pull of <= 2 MiB in
                               <= 64 runs (AUTO variant, not head-sliced) makes no CUDA call
                               and pays no launch latency (C1 over NVLink: 8.2 us host to
                               host with 16 CTAs vs 13.4 launched).  The
                               engine is launched on the first such request and exits after
                               2 ms without one (a watchdog thread), so it holds c SMs only
                               while short requests flow.  Such requests are NOT ordered with
                               the caller's stream (like KVD_OPT_STREAMS): the destination
                               blocks must be free when kvd_pull is called, and completion is
                               observed with kvd_poll_done / kvd_wait_done.  While the engine
                               runs, a device-wide synchronise (cudaDeviceSynchronize) waits up
                               to the idle timeout; synchronise streams instead (library calls
                               that must synchronise the device stop the engine first).  0
                               stops it */
} kvd_option;

typedef struct kvd_cache_s* kvd_cache;
typedef struct kvd_peer_s* kvd_peer;

/* ---------------------------------------------------------------------------
 * Host-only helpers (row a1 / a3 of the design; usable without a GPU)
 * ------------------------------------------------------------------------- */

/* [host-only] Validate a layout and derive its byte geometry.
 * Errors: KVD_EINVAL (null), KVD_ELAYOUT (see kvd_layout requirements). */
KVD_API kvd_status kvd_layout_geometry(const kvd_layout* layout, kvd_geometry* out);

/* [host-only] Validate a block table and coalesce it into maximal runs
 * (merge consecutive entries only when both the remote and the
 * local blocks continue the previous ones).  src_ids/dst_ids: n entries;
 * ids must lie in [0, src_num_blocks) / [0, dst_num_blocks) (else
 * KVD_ERANGE) and dst ids must be distinct (else KVD_EINVAL).  coalesce=0
 * emits one run per entry.  Writes at most `cap` runs to `runs` and the run
 * count to *m; KVD_ENOMEM if cap is too small (then *m is the count needed). */
KVD_API kvd_status kvd_plan(const int32_t* src_ids, const int32_t* dst_ids, uint32_t n,
                    uint32_t src_num_blocks, uint32_t dst_num_blocks, int coalesce,
                    kvd_run* runs, uint32_t cap, uint32_t* m);

/* [host-only] Decode an export blob's header without opening it.
 * Any out pointer may be NULL.  KVD_EHANDLE on a malformed blob. */
KVD_API kvd_status kvd_blob_info(const void* blob, size_t blob_len, kvd_layout* layout,
                         int32_t* device, int64_t* pid, uint32_t* num_allocations);

/* ---------------------------------------------------------------------------
 * Row a1: register a cache (both sides, once)
 * ------------------------------------------------------------------------- */

/* Register the paged cache whose layer l starts at device address
 * layer_base_dev[l] (num_layers entries) on CUDA device `device`.
 * The caller keeps ownership of the memory and must keep it alive until
 * kvd_unregister_cache and, for an exporter, until every importer has
 * closed its peer (CUDA IPC rule).  Bases must be 16 B aligned and each
 * layer's extent must lie inside one allocation (checked when a GPU is
 * present).  Errors: KVD_EINVAL, KVD_ELAYOUT, KVD_ECUDA, KVD_ENOMEM. */
KVD_API kvd_status kvd_register_cache(int device, const kvd_layout* layout,
                              void* const* layer_base_dev, kvd_cache* out);

KVD_API kvd_status kvd_unregister_cache(kvd_cache cache);

/* ---------------------------------------------------------------------------
 * §8 f3 groundwork: exportable cache memory (CUDA virtual memory management)
 *
 * The paper pulls across nodes.  With NVLink hardware the
 * cross-node handle is a FABRIC handle of a VMM allocation (multi-node
 * NVLink; needs an IMEX channel); inside one node the same allocation
 * exports as a POSIX fd.  Caches placed in kvd_mem_alloc memory export such
 * handles from kvd_export_handle automatically; the pull kernel is unchanged.
 * ------------------------------------------------------------------------- */
typedef enum {
  KVD_MEM_AUTO = 0,      /* FABRIC when the driver permits it, else POSIX_FD */
  KVD_MEM_POSIX_FD = 1,  /* intra-node: the importer fetches the exporter's fd
                            with pidfd_getfd (Linux >= 5.6, same user, the
                            exporter alive and in the importer's PID namespace) */
  KVD_MEM_FABRIC = 8     /* multi-node NVLink: 64 B handle, importable on any
                            node of the NVLink domain (IMEX) */
} kvd_mem_kind;

/* Allocate `bytes` (rounded up to the recommended granularity, 2 MiB on
 * B200) of device memory on `device`, mapped read/write for that device.
 * *size (may be NULL) = bytes reserved; *kind_out (may be NULL) = the kind
 * obtained.  The caller owns the memory: free it with kvd_mem_free after
 * every cache over it is unregistered and every importer has closed its
 * peer.  Errors: KVD_EINVAL (null, zero size, unknown kind), KVD_ENOMEM,
 * KVD_EHANDLE (kind not permitted here, e.g. FABRIC without IMEX),
 * KVD_ECUDA. */
KVD_API kvd_status kvd_mem_alloc(int device, uint64_t bytes, int kind, void** ptr,
                                 uint64_t* size, int* kind_out);

/* Free kvd_mem_alloc memory (synchronises its device first, like cudaFree).
 * KVD_EINVAL if ptr is not the start of a kvd_mem_alloc allocation. */
KVD_API kvd_status kvd_mem_free(void* ptr);

/* ---------------------------------------------------------------------------
 * Row a2: one-time tensor-centric exchange (Connect())
 * ------------------------------------------------------------------------- */

/* Serialise the cache's metadata -- layout (Address/Dims/Shape/Stride,
 * P:L294) plus one CUDA IPC handle per distinct allocation and each layer's
 * (allocation, offset) -- into the caller's buffer.  *blob_len: in =
 * capacity, out = bytes written (or needed, with KVD_ENOMEM).  The blob is
 * plain bytes; ship it to the decode process any way (torch.distributed,
 * TCPStore, socket).  An allocation from kvd_mem_alloc is exported as its
 * POSIX fd or fabric handle instead of a CUDA IPC handle (blob v3 records
 * the kind per allocation).  Errors: KVD_EINVAL, KVD_ENOMEM, KVD_EHANDLE
 * (memory neither cudaMalloc nor kvd_mem_alloc, e.g. torch expandable
 * segments). */
KVD_API kvd_status kvd_export_handle(kvd_cache cache, void* blob, size_t* blob_len);

/* Import a peer cache's blob and bind it to a local cache.  For the pull
 * path (the product) the decode process imports the prefill cache's blob and
 * `local_dst` is its decode cache; for the push variant (kvd_push) the
 * prefill process imports the decode cache's blob and `local_dst` is its
 * prefill cache.  Checks compatibility (same layers, heads, head_dim,
 * block_size, element size; B/KV strides and num_blocks may differ)
 * -> KVD_ELAYOUT; maps each allocation with cudaIpcOpenMemHandle on the
 * local device (or, for a blob exported by this same process, uses the raw
 * pointers and enables peer access) -> KVD_EHANDLE / KVD_ECUDA.
 * Allocates the completion-slot ring (pinned mapped host flags). */
KVD_API kvd_status kvd_open_peer(kvd_cache local_dst, const void* blob, size_t blob_len,
                         kvd_peer* out);

/* TP-resharding import (not in the paper, which keeps prefill
 * and decode TP degrees equal): bind a prefill SHARD cache with H_r KV heads
 * to heads [head_offset, head_offset + H_r) of the local decode cache (H_l
 * heads, H_r + head_offset <= H_l).  kvd_pull / kvd_pull_batch on the
 * returned peer then copy, for every requested block, layer, K/V and token,
 * the shard's H_r heads into that head slice (a strided copy: block_size
 * rows of H_r*head_dim elements, destination rows H_l*head_dim apart).
 * Example: prefill TP=8 -> decode TP=4, decode shard j opens prefill shards
 * 2j (offset 0) and 2j+1 (offset H_r) and pulls the same block table from
 * both.  Both caches must use the default (L, H, D) inner order (else
 * KVD_ELAYOUT); layers, head_dim, block_size and element size must match;
 * H_r * head_dim * elem and head_offset * head_dim * elem must be multiples
 * of 16 B.  LSU mover only; kvd_push is not available on such a peer. */
KVD_API kvd_status kvd_open_peer_heads(kvd_cache local_dst, const void* blob, size_t blob_len,
                                       uint32_t head_offset, kvd_peer* out);

/* Close a peer: synchronises the local device (transfers still in flight
 * finish first), unmaps the imported allocations and frees the completion
 * slots.  Request ids not yet polled are forgotten. */
KVD_API kvd_status kvd_close_peer(kvd_peer peer);

/* Tune a peer (see kvd_option).  KVD_EINVAL on an unknown option/value. */
KVD_API kvd_status kvd_peer_set(kvd_peer peer, int option, int64_t value);

/* ---------------------------------------------------------------------------
 * Rows a3-a6: the per-request pull (Transfer() x n + Complete())
 * ------------------------------------------------------------------------- */

/* Pull request `request_id`: for every i < n, every layer and K and V,
 * copy remote block src_ids[i] of the prefill cache into local block
 * dst_ids[i] of the decode cache, bit for bit.  Validates (KVD_ERANGE,
 * KVD_EINVAL) and coalesces on the host, then issues exactly ONE kernel
 * launch on `stream` ("post ... without block") and returns without
 * waiting.  Stream order: the pull's stores into the decode cache follow
 * all earlier work on `stream`; over NVLink it may start READING the source
 * blocks before that work has finished (KVD_OPT_EARLY_LOADS, default on).  On any error nothing is launched and no byte changes.
 * request_id must not be in flight on this peer (KVD_EBUSY).  n = 0 is
 * valid: a flag-only launch; the request completes with no bytes moved. */
KVD_API kvd_status kvd_pull(kvd_peer peer, uint64_t request_id, const int32_t* src_ids,
                    const int32_t* dst_ids, uint32_t n, void* stream);

/* Non-blocking completion check (Complete()): *done = 1
 * once every byte of the request has landed in decode HBM and is visible
 * to later work on the decode GPU and to the host; the request is then
 * retired (its id may be reused; a later poll of it returns KVD_EINVAL).
 * *done = 0 while in flight.  Lock-free and makes no CUDA call: a lookup in
 * the peer's request -> slot table, an acquire load of the pinned slot word
 * and a compare-and-swap to retire.  Errors: KVD_EINVAL for an unknown
 * request id (or one a concurrent poll just retired). */
KVD_API kvd_status kvd_poll_done(kvd_peer peer, uint64_t request_id, int* done);

/* Batched drain (§4.2 "Tensor communication",
 * P:L373-378, fig:queue): pull `num_requests` requests with ONE launch.
 * Request q is entries [offsets[q], offsets[q+1]) of src_ids/dst_ids
 * (offsets has num_requests+1 entries, offsets[0] = 0, non-decreasing).
 * The concatenated table is validated as one queue (destination ids
 * distinct across the whole batch, else KVD_EINVAL) and coalesced as one:
 * runs may merge across requests ("Read 0->5 from R1 and Read 1->6 from R2
 * can be merged").  Each request keeps its own completion slot and
 * completes as soon as ITS bytes have landed (poll each id with
 * kvd_poll_done); requests with no entries complete at launch.  Ids must be
 * distinct and not in flight (KVD_EINVAL / KVD_EBUSY).  Issues one small
 * host-to-device copy of the descriptor table and one kernel on `stream`.
 * Not available with KVD_VARIANT_CE (KVD_EINVAL). */
KVD_API kvd_status kvd_pull_batch(kvd_peer peer, uint32_t num_requests,
                                  const uint64_t* request_ids, const uint32_t* offsets,
                                  const int32_t* src_ids, const int32_t* dst_ids, void* stream);

/* Push variant (§4.3 push mode, P:L402,
 * fig:push_pull): launched on the PREFILL GPU, copies local blocks
 * src_ids[i] of the peer's local cache into REMOTE blocks dst_ids[i] of the
 * imported (decode) cache with NVLink stores, all layers and K/V in one
 * launch.  Same validation, coalescing, errors and completion slots as
 * kvd_pull (the completion word lives in the pusher's host memory; the
 * caller tells the decode side).  The paper pushes layer by layer while
 * prefill computes; this variant pushes the finished request in one shot
 * so the two transfer directions are compared on equal terms. */
KVD_API kvd_status kvd_push(kvd_peer peer, uint64_t request_id, const int32_t* src_ids,
                            const int32_t* dst_ids, uint32_t n, void* stream);

/* Prefill side of Complete() ("When the prefill worker receives the
 * Complete() message, it notifies the inference engine to release the KV
 * cache block"; P:L375 the request ID is written into the prefill's memory
 * one-sidedly).  Every pull from an exported cache, on completion, posts its
 * request_id into a mailbox in the EXPORTER's host memory: a memfd created
 * at the first kvd_export_handle, which each importer maps (pidfd_getfd;
 * same node), registers with CUDA and owns one ring of (64 importers per
 * exporter at a time).  The completing CTA writes the id at the ring
 * position its host assigned in issue order -- two plain 64-bit stores over
 * PCIe, no atomic over NVLink.  Called on the exporter's cache, this copies
 * up to `cap` newly completed request ids into `request_ids` and sets *n;
 * the caller may then reuse those source blocks.  Each id is returned once;
 * per importer in issue order (a request whose pull completes before an
 * earlier-issued one of the same importer is reported after it).  Each
 * ring holds 4096 notifications: poll at least that often, else KVD_EBUSY
 * reports lost notifications.  Plain loads, no CUDA call; *n = 0 before the
 * first export. */
KVD_API kvd_status kvd_poll_released(kvd_cache exporter, uint64_t* request_ids, uint32_t cap,
                                     uint32_t* n);

/* Spin on kvd_poll_done until done or `timeout_us` elapses (KVD_EBUSY). */
KVD_API kvd_status kvd_wait_done(kvd_peer peer, uint64_t request_id, int64_t timeout_us);

/* kvd_poll_done over n in-flight requests in one call (a decode loop admitting
 * many requests): done[i] = 1 and the request retired when it completed, else
 * 0; *ndone = how many completed.  All or nothing on bad input: if any id is
 * not in flight or appears twice, KVD_EINVAL is returned before any request
 * is retired (*ndone = 0, done[] unspecified).  Lock-free, no CUDA call. */
KVD_API kvd_status kvd_poll_many(kvd_peer peer, const uint64_t* request_ids, uint32_t n,
                                 uint8_t* done, uint32_t* ndone);

/* Bounds-audit violations counted on this peer since KVD_OPT_AUDIT was set
 * (synchronises the local device first).  KVD_ESTATE if auditing is off. */
KVD_API kvd_status kvd_peer_audit(kvd_peer peer, uint64_t* violations);

/* Kernel-only device time of the launches recorded since the previous call
 * (KVD_OPT_TIMING = 1; at most 65536 launches are recorded between calls):
 * waits for them, returns the summed milliseconds and the number of
 * launches, and forgets them.  KVD_ESTATE if timing is off. */
KVD_API kvd_status kvd_peer_kernel_time(kvd_peer peer, double* total_ms, uint64_t* launches);

/* In-kernel duration (KVD_OPT_TIMING, single pulls, SURVEY §8 d's
 * %globaltimer cross-check): the summed nanosecond-timer spans from the
 * first CTA's start to the last CTA's completion, over the requests retired
 * by kvd_poll_done / kvd_wait_done since the previous call, in ms, and their
 * count; then resets.  Unlike the events it excludes launch latency. */
KVD_API kvd_status kvd_peer_device_time(kvd_peer peer, double* total_ms, uint64_t* launches);

/* KVD_OPT_STREAMS >= 2: make `stream` (of the peer's local device) wait for
 * every transfer issued on this peer so far.  A no-op otherwise (transfers
 * are then already in the caller's stream order).  Errors: KVD_EINVAL,
 * KVD_ECUDA. */
KVD_API kvd_status kvd_stream_wait(kvd_peer peer, void* stream);

/* %globaltimer timeline of one retired single pull (KVD_OPT_TIMING), in the
 * decode GPU's nanosecond timer: the earliest CTA start, the earliest return
 * from the wait for the preceding kernel on the stream (after early source
 * reads, KVD_OPT_EARLY_LOADS; else = start), and the last CTA's completion
 * right before the slot word's release. */
typedef struct {
  uint64_t request_id;
  uint64_t start_ns;
  uint64_t wait_ns;
  uint64_t end_ns;
} kvd_span;

/* Diagnostics: the timelines of the timed single pulls retired (by any
 * poller) since the previous call, oldest first, at most `cap` (and at most
 * the 4096 most recent); *n = how many were written. */
KVD_API kvd_status kvd_peer_spans(kvd_peer peer, kvd_span* out, uint32_t cap, uint32_t* n);

/* Link calibration (SURVEY.md §8 d: GB/s "as a fraction of the measured
 * achievable link ceiling (calibration kernel)"): reads `bytes` of the
 * peer's SOURCE cache memory -- layer after layer from each layer's base,
 * contiguous 32 KiB chunks, no block table -- with bulk (TMA) loads into
 * shared memory that are discarded (no stores), `reps` passes in one launch
 * (after one untimed pass), and returns bytes * reps / device time (CUDA
 * events) in GB/s (1e9 B/s).
 * That is the most this GPU's SMs can read through the mapping (over NVLink
 * for a peer on another GPU), the ceiling a pull can approach.  `ctas` CTAs
 * of one `stages`-deep ring each (0: one per SM; stages 0: 6).  Synchronous
 * (runs on an internal stream, waits for it); takes the peer lock; a
 * measurement tool, not part of the transfer path.
 * Errors: KVD_EINVAL (null gbs, reps 0, stages > 7 -- 7 x 32 KiB fill the
 * shared memory -- or bytes < 32 KiB),
 * KVD_ERANGE (bytes more than the source layers hold), KVD_ECUDA. */
KVD_API kvd_status kvd_peer_calibrate(kvd_peer peer, uint64_t bytes, uint32_t ctas,
                                      uint32_t stages, uint32_t reps, double* gbs);

/* Describe the most recent kvd_pull on this peer. */
KVD_API kvd_status kvd_last_pull_info(kvd_peer peer, kvd_pull_info* out);

/* ---------------------------------------------------------------------------
 * Message-passing baseline helpers (fig:diff(a): gather kernel ->
 * send -> receive -> scatter kernel).  Used only by the NCCL comparator.
 * Staging layout: [layer][kv][i][span] -- n blocks of every (layer, K|V)
 * packed back to back; staging_dev holds layers * 2 * n * span bytes.
 * ------------------------------------------------------------------------- */

/* Gather cache blocks ids[0..n) into staging_dev (one launch on stream). */
KVD_API kvd_status kvd_gather(kvd_cache cache, const int32_t* ids, uint32_t n, void* staging_dev,
                      void* stream);

/* Scatter staging_dev into cache blocks ids[0..n) (one launch on stream). */
KVD_API kvd_status kvd_scatter(kvd_cache cache, const int32_t* ids, uint32_t n,
                       const void* staging_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------- */

KVD_API const char* kvd_strerror(kvd_status status);
KVD_API const char* kvd_last_error(void);
KVD_API int kvd_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KVD_H */
