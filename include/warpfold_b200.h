/*
 * warpfold_b200.h — C ABI of the B200-native warp-primitive path.
 *
 * This is the drop-in boundary for the data-parallel path that the warpfold
 * CPU reference (arXiv 2112.10034, "COX" hierarchical collapsing) emulates.
 * In the reference that path is
 *
 *     launch(hybrid_transform(kernel, cfg), cfg, memory, args)
 *         runtime/launch.py:90          (block scheduling over a fork pool)
 *         passes/pipeline.py:103-179    (collapse warps/blocks into loop nests)
 *         passes/warp_lower.py:17-88    (lane-array emulation of shfl / vote)
 *         interp/mpmd.py:237-255        (per-block interpreter, the CPU hot loop)
 *
 * Here every one of those layers is replaced by a hand-written sm_100a kernel
 * reached through the plain-C entry points below.  Conventions:
 *
 *   - Pointers are device pointers unless the name says `host_`.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - The library never allocates or frees caller buffers.  Scratch state
 *     (tile descriptors, block partials, tickets) lives in a caller-provided
 *     workspace of wf_workspace_bytes() bytes that must be zero-filled once
 *     (wf_workspace_init) and may then be reused by any number of calls of
 *     the same op on the same stream.  Kernels leave it ready for reuse.
 *   - Every call is stream-ordered and asynchronous; results are valid once
 *     the stream is synchronised (the Python `launch` does that, preserving
 *     the reference's join semantics, runtime/launch.py:1-8).
 *   - Return value: 0 = OK, > 0 = cudaError_t, < 0 = WF_ERR_* below.
 *     wf_last_error() returns a thread-local message for the last failure.
 *     The Python wrapper maps WF_ERR_CONFIG -> ConfigError, WF_ERR_ARG ->
 *     LaunchError, WF_ERR_UNSUPPORTED -> UnsupportedFeatureError and CUDA
 *     errors -> ExecutionError (reference errors.py:22-47).
 *
 * Integer arithmetic wraps modulo 2^32 exactly like the reference's i32
 * (numerics.py:20-22); f32 is IEEE single precision with a fixed,
 * run-to-run reproducible association order.
 */
#ifndef WARPFOLD_B200_H
#define WARPFOLD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WF_ABI_VERSION 1

/* error codes (negative); positive values are cudaError_t */
#define WF_OK 0
#define WF_ERR_CONFIG (-1)      /* bad block/grid/width (config.py:26-41)      */
#define WF_ERR_ARG (-2)         /* bad pointer/size/alignment (launch.py:28-46) */
#define WF_ERR_COMM (-3)        /* reserved for the cross-GPU exchange          */
#define WF_ERR_UNSUPPORTED (-4) /* op/variant not provided (errors.py:18-19)    */
#define WF_ERR_WORKSPACE (-5)   /* workspace missing or too small               */
#define WF_ERR_EXEC (-6)        /* device-side fault flagged by a kernel        */

/* op ids for wf_workspace_bytes */
#define WF_OP_REDUCE_SUM_I32 1
#define WF_OP_REDUCE_SUM_F32 2
#define WF_OP_SCAN_INCLUSIVE_I32 3
#define WF_OP_COMPACT_GT0_I32 4
#define WF_OP_HISTOGRAM256_U8 5
#define WF_OP_WARP_COLLECTIVE 6

/* warp collective kinds for wf_warp_collective (Appendix B of SURVEY.md) */
#define WF_COLL_SHFL_DOWN 0 /* passes/warp_lower.py:36-45 shuffle_down      */
#define WF_COLL_SHFL_UP 1   /* extension: CUDA __shfl_up_sync              */
#define WF_COLL_SHFL_XOR 2  /* extension: CUDA __shfl_xor_sync             */
#define WF_COLL_SHFL_IDX 3  /* extension: CUDA __shfl_sync                 */
#define WF_COLL_VOTE_ALL 4  /* passes/warp_lower.py:17-33 reduce_vote all  */
#define WF_COLL_VOTE_ANY 5  /* passes/warp_lower.py:17-33 reduce_vote any  */
#define WF_COLL_BALLOT 6    /* extension: CUDA __ballot_sync               */
#define WF_COLL_REDUCE_ADD 7 /* extension: CUDA __reduce_add_sync (REDUX)  */

/* synthetic input generators for wf_fill_synthetic:
 * h = splitmix64(seed ^ (index_base + i)) */
#define WF_GEN_I32_FULL 0   /* (int32)(h >> 32)                             */
#define WF_GEN_I32_SMALL 1  /* (int32)((h >> 32) % 21) - 10  (corpus.py:320)*/
#define WF_GEN_F32_UNIT 2   /* (float)(h >> 40) * 2^-24 - 0.5 (exact)      */
#define WF_GEN_U8_UNIFORM 3 /* h & 0xff                                     */
#define WF_GEN_U8_CONST 4   /* param & 0xff                                 */
#define WF_GEN_U8_GEOM 5    /* min(clz64(h), 255): geometric, skewed        */
#define WF_GEN_I32_SELECT 6 /* > 0 with probability param/1000              */

typedef void *wf_stream_t;

/* ---- housekeeping ------------------------------------------------------ */
const char *wf_version(void);
int wf_abi_version(void);
const char *wf_last_error(void);
int wf_device_sm_count(int device);
size_t wf_workspace_bytes(int op, uint64_t n, int block);
int wf_workspace_init(void *ws, size_t ws_bytes, wf_stream_t stream);
void wf_shutdown(void);

/* ---- K1/K2: shuffle reductions ----------------------------------------
 * Replaces the reference's per-warp-partials shfl_down reduction executed by
 * launch() (runtime/launch.py:90 -> interp/mpmd.py:237) plus its host fold.
 * out[0] = sum(in[0..n)); i32 wraps mod 2^32.  grid = 0 picks the persistent
 * grid (SM count x resident blocks); block in {128, 256, 512, 1024}.
 * f32: fixed order (per-thread chains, butterfly warp tree, block tree,
 * fixed-order fold of block partials) => bitwise reproducible for a given
 * (n, block, grid, device). */
int wf_reduce_sum_i32(const int32_t *in, uint64_t n, int32_t *out, int block,
                      int grid, void *ws, size_t ws_bytes, wf_stream_t stream);
int wf_reduce_sum_f32(const float *in, uint64_t n, float *out, int block,
                      int grid, void *ws, size_t ws_bytes, wf_stream_t stream);

/* Launch flags of the *_ex entry points.
 * WF_FLAG_INPUT_STABLE: the caller promises that the kernel issued just
 *   before this call on `stream` does not write `in` (e.g. the previous call
 *   of a loop over the same input, or anything after a stream / event
 *   synchronisation).  The reduction is then a programmatic dependent launch:
 *   it streams `in` while that kernel drains and touches `ws` / `out` only
 *   after it has completed.  Same result bits as without the flag. */
#define WF_FLAG_INPUT_STABLE 1u
int wf_reduce_sum_f32_ex(const float *in, uint64_t n, float *out, int block,
                         int grid, void *ws, size_t ws_bytes, unsigned flags,
                         wf_stream_t stream);

/* Fixed-order folds of `count` device values (cross-GPU partial combine,
 * SURVEY.md §8e).  out[0] = vals[0] + vals[1] + ... + vals[count-1] in that
 * association order for f32; wrapping for i32. */
int wf_fold_f32(const float *vals, uint32_t count, float *out,
                wf_stream_t stream);
int wf_fold_i32(const int32_t *vals, uint32_t count, int32_t *out,
                wf_stream_t stream);
int wf_fold_u64(const uint64_t *vals, uint32_t count, uint64_t *out,
                wf_stream_t stream);

/* ---- multi-GPU: fused reduce + exchange over peer memory --------------
 * Replaces, for the sharded C2 reduction, the all-gather of per-rank partials
 * plus wf_fold_f32 (the reference's only parallelism is the
 * block-range split of runtime/launch.py:137-147) with ONE kernel per rank:
 * its last block stores the rank partial straight into every rank's mailbox
 * (CUDA IPC mappings over NVLink / NVSwitch), waits for all ranks' partials in
 * its own mailbox and folds them with wf_fold_f32's association, so out[0] is
 * bit-identical on every rank and to the NCCL path.
 *   mailbox:   wf_mailbox_bytes(world) bytes of device memory per rank
 *              (wf_mailbox_alloc: cudaMalloc + zero), exported with
 *              wf_ipc_handle (64-byte cudaIpcMemHandle) and mapped by the other
 *              ranks with wf_ipc_open.
 *   d_peers:   device array of `world` mailbox pointers (rank order).
 *   epoch:     1, 2, 3, ... — the same sequence on every rank, one per call.
 * A rank whose peers do not arrive within ~4 s writes NaN to out[0]. */
size_t wf_mailbox_bytes(int world);
int wf_mailbox_alloc(int world, void **d_mailbox);
int wf_mailbox_free(void *d_mailbox);
int wf_ipc_handle(void *d_ptr, void *handle64);
int wf_ipc_open(const void *handle64, void **d_ptr);
int wf_ipc_close(void *d_ptr);
int wf_reduce_sum_f32_mg(const float *in, uint64_t n, float *out, int block,
                         int grid, void *ws, size_t ws_bytes,
                         void *const *d_peers, const void *d_mailbox, int rank,
                         int world, uint32_t epoch, wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE, as wf_reduce_sum_f32_ex) */
int wf_reduce_sum_f32_mg_ex(const float *in, uint64_t n, float *out, int block,
                            int grid, void *ws, size_t ws_bytes,
                            void *const *d_peers, const void *d_mailbox,
                            int rank, int world, uint32_t epoch,
                            unsigned flags, wf_stream_t stream);

/* Small collectives over the same kind of peer-memory mailboxes, one
 * single-block kernel per rank (replace NCCL all-gather / all-reduce + fold
 * for the exchange steps of C3-C5).  A peer mailbox holds `cap` payload words
 * per source rank (wf_peer_mailbox_alloc; free with wf_mailbox_free).
 *   mode WF_PEER_ALLGATHER: d_out[r * count + i] = vals_r[i]          (u64)
 *   mode WF_PEER_EXSCAN:    d_out = {sum_{r<rank} vals_r[0], sum_r vals_r[0]} (u64)
 *   mode WF_PEER_ALLREDUCE: d_out[i] = sum_r vals_r[i]               (u64)
 *   mode WF_PEER_EXSCAN_U32: as EXSCAN on u32 values mod 2^32, d_out = 2 x u32
 * Results are identical on every rank (rank-order combine).  *d_err is set to
 * 1 when a peer did not arrive within ~4 s (results then undefined). */
#define WF_PEER_ALLGATHER 0
#define WF_PEER_EXSCAN 1
#define WF_PEER_ALLREDUCE 2
#define WF_PEER_EXSCAN_U32 3
size_t wf_peer_mailbox_bytes(int world, uint32_t cap);
/* The same exchange fused into the last block of the producing kernel (one
 * kernel per rank and step instead of kernel + exchange kernel), on a
 * wf_peer_mailbox_alloc mailbox and the same epoch sequence as
 * wf_peer_exchange:
 *   wf_reduce_sum_i32_exscan_mg: K1 over the rank's shard, then
 *     d_out2 = {sum of the shards of ranks < rank, sum of all shards}
 *     (int32, wrapping) — the carry-in and total of the sharded C3 scan.
 *   wf_histogram256_u8_mg: K5 over the rank's shard, then d_bins = the
 *     element-wise sum of every rank's 256 bins (cap >= 256).
 *   wf_compact_gt0_i32_mg: K4 over the rank's shard (output stays local),
 *     d_counts3 = {this rank's count, its global offset, the global total}
 *     (u64); the exchange runs in the compaction kernel's last finisher warp
 *     on the default (TMEM) path, as a second kernel otherwise.
 * Every rank must issue the same sequence of exchange calls. */
int wf_reduce_sum_i32_exscan_mg(const int32_t *in, uint64_t n, int32_t *d_out2,
                                int block, int grid, void *ws, size_t ws_bytes,
                                void *const *d_peers, const void *d_mailbox,
                                uint32_t cap, int rank, int world, uint32_t epoch,
                                uint32_t *d_err, wf_stream_t stream);
int wf_compact_gt0_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                          uint64_t *d_counts3, void *ws, size_t ws_bytes,
                          void *const *d_peers, const void *d_mailbox,
                          uint32_t cap, int rank, int world, uint32_t epoch,
                          uint32_t *d_err, wf_stream_t stream);
/* Single-pass sharded scan of a BLOCK-CYCLIC distributed array: global
 * super-tile g (round_elems elements, a multiple of 8192) lives on rank
 * g % world as its local super-tile g / world; this rank's `in` holds its
 * super-tiles back to back (n elements, the last may be short) and `out`
 * receives the GLOBAL inclusive scan at those positions.  Each round's
 * super-tile totals are all-gathered over the peer mailbox inside the scan
 * kernel (cap >= rounds words per rank), so every element is read once and
 * written once (8 B/elem; the contiguous-shard reduce-then-scan needs 12).
 * `rounds` must be the same on every rank (>= ceil(n / round_elems)); in /
 * out 16-byte aligned.  max_grid > 0 caps the grid (ranks sharing one GPU
 * must all be resident at once).  flags: WF_FLAG_INPUT_STABLE. */
int wf_scan_inclusive_i32_cyclic_mg(const int32_t *in, int32_t *out, uint64_t n,
                                    void *ws, size_t ws_bytes, void *const *d_peers,
                                    const void *d_mailbox, uint32_t cap, int rank,
                                    int world, uint32_t epoch, uint32_t *d_err,
                                    uint64_t round_elems, uint32_t rounds,
                                    int max_grid, unsigned flags,
                                    wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE, as wf_reduce_sum_f32_ex) */
int wf_reduce_sum_i32_exscan_mg_ex(const int32_t *in, uint64_t n, int32_t *d_out2,
                                   int block, int grid, void *ws, size_t ws_bytes,
                                   void *const *d_peers, const void *d_mailbox,
                                   uint32_t cap, int rank, int world,
                                   uint32_t epoch, uint32_t *d_err,
                                   unsigned flags, wf_stream_t stream);
int wf_compact_gt0_i32_mg_ex(const int32_t *in, uint64_t n, int32_t *out,
                             uint64_t *d_counts3, void *ws, size_t ws_bytes,
                             void *const *d_peers, const void *d_mailbox,
                             uint32_t cap, int rank, int world, uint32_t epoch,
                             uint32_t *d_err, unsigned flags, wf_stream_t stream);
int wf_histogram256_u8_mg(const uint8_t *in, uint64_t n, uint64_t *d_bins,
                          void *ws, size_t ws_bytes, void *const *d_peers,
                          const void *d_mailbox, uint32_t cap, int rank,
                          int world, uint32_t epoch, uint32_t *d_err,
                          wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE, as wf_reduce_sum_f32_ex) */
int wf_histogram256_u8_mg_ex(const uint8_t *in, uint64_t n, uint64_t *d_bins,
                             void *ws, size_t ws_bytes, void *const *d_peers,
                             const void *d_mailbox, uint32_t cap, int rank,
                             int world, uint32_t epoch, uint32_t *d_err,
                             unsigned flags, wf_stream_t stream);
int wf_peer_mailbox_alloc(int world, uint32_t cap, void **d_mailbox);
int wf_peer_exchange(int mode, const void *d_vals, uint32_t count, uint32_t cap,
                     void *d_out, void *const *d_peers, const void *d_mailbox,
                     int rank, int world, uint32_t epoch, uint32_t *d_err,
                     wf_stream_t stream);

/* ---- single-process multi-GPU (wf_mg_init + wf_mg_<op>) --
 * One host thread drives `ngpus` ranks on the listed devices (ranks may share
 * a device).  Each call enqueues one rank's kernel per device on the
 * context's per-rank stream, each kernel carrying its exchange over peer
 * memory (NVLink / NVSwitch peer access, enabled by wf_mg_init); arrays are
 * indexed by rank, pointers are device pointers on that rank's device, shards
 * are the caller's contiguous split (runtime/launch.py:137-147 `_split`
 * across devices).  Results are valid after wf_mg_synchronize, which returns
 * WF_ERR_COMM if a rank's peers never arrived.
 *   reduce_sum_f32: d_out[r][0] = the fp32 sum of all shards, bit-identical
 *                   on every rank (fixed rank-order fold)
 *   scan_inclusive_i32: d_out[r] = the global inclusive scan over rank r's shard
 *   compact_gt0_i32: d_out[r] = rank r's selected elements, d_counts3[r] =
 *                   {count, global offset, global total}
 *   histogram256_u8: d_bins[r] = the global 256 bins on every rank
 * Reference anchor: runtime/launch.py:95-147 (block-range split + join). */
typedef struct wf_mg wf_mg_t;
int wf_mg_init(int ngpus, const int *devs, wf_mg_t **ctx);
int wf_mg_size(const wf_mg_t *ctx);
int wf_mg_stream(wf_mg_t *ctx, int rank, wf_stream_t *stream);
int wf_mg_reduce_sum_f32(wf_mg_t *ctx, const float *const *d_in,
                         const uint64_t *n, float *const *d_out);
int wf_mg_scan_inclusive_i32(wf_mg_t *ctx, const int32_t *const *d_in,
                             int32_t *const *d_out, const uint64_t *n);
int wf_mg_compact_gt0_i32(wf_mg_t *ctx, const int32_t *const *d_in,
                          const uint64_t *n, int32_t *const *d_out,
                          uint64_t *const *d_counts3);
int wf_mg_histogram256_u8(wf_mg_t *ctx, const uint8_t *const *d_in,
                          const uint64_t *n, uint64_t *const *d_bins);
int wf_mg_synchronize(wf_mg_t *ctx);
void wf_mg_destroy(wf_mg_t *ctx);

/* ---- K3: shfl_scan inclusive prefix sum --------------------------------
 * out[i] = carry + in[0] + ... + in[i] (wrapping), single pass with
 * decoupled look-back.  d_carry_in: device int32 (NULL = 0), used by the
 * cross-GPU reduce-then-scan.  in/out may alias exactly (in-place). */
int wf_scan_inclusive_i32(const int32_t *in, int32_t *out, uint64_t n,
                          const int32_t *d_carry_in, void *ws, size_t ws_bytes,
                          wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE: the first tiles' loads overlap
 * the previous kernel's drain; d_carry_in is read after it has completed, so
 * it may be that kernel's output) */
int wf_scan_inclusive_i32_ex(const int32_t *in, int32_t *out, uint64_t n,
                             const int32_t *d_carry_in, void *ws, size_t ws_bytes,
                             unsigned flags, wf_stream_t stream);

/* ---- K4: warp-aggregated stream compaction -----------------------------
 * out[0..m) = in[i] for in[i] > 0 in index order; *d_count = m (uint64).
 * n < 2^32 per call.  out must hold n elements. */
int wf_compact_gt0_i32(const int32_t *in, uint64_t n, int32_t *out,
                       uint64_t *d_count, void *ws, size_t ws_bytes,
                       wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE, as wf_scan_inclusive_i32_ex) */
int wf_compact_gt0_i32_ex(const int32_t *in, uint64_t n, int32_t *out,
                          uint64_t *d_count, void *ws, size_t ws_bytes,
                          unsigned flags, wf_stream_t stream);

/* ---- K5: smem-privatised 256-bin histogram -----------------------------
 * bins[b] = #{i : in[i] == b} as uint64 (overwrites bins). */
int wf_histogram256_u8(const uint8_t *in, uint64_t n, uint64_t *bins, int grid,
                       void *ws, size_t ws_bytes, wf_stream_t stream);
/* ... with launch flags (WF_FLAG_INPUT_STABLE, as wf_reduce_sum_f32_ex: the
 * counting overlaps the previous kernel's drain) */
int wf_histogram256_u8_ex(const uint8_t *in, uint64_t n, uint64_t *bins, int grid,
                          void *ws, size_t ws_bytes, unsigned flags,
                          wf_stream_t stream);

/* ---- P: warp collectives with reference semantics ----------------------
 * Runs n_threads logical threads as blocks of `block` threads (the last warp
 * of a block is partial when block % 32 != 0; n_threads % block == 0).
 * Lanes are grouped into segments of `width` lanes (1,2,4,8,16,32: the
 * reference's warp_size, config.py:17-23).  Thread i, if its lane is in
 * `mask`, computes the collective over its segment's participating lanes
 * (mask & present lanes) and writes out[i]; other threads leave out[i].
 * `a` is the value/predicate operand, `b` the per-lane offset/lane-mask/
 * source-lane operand (NULL = use `operand` for every lane).
 * Semantics (reference passes/warp_lower.py:17-45, interp/oracle.py:147-161):
 *   SHFL_DOWN  src = l + off, own value unless 0 <= src < width and src
 *              participates (reference clamp, any int offset)
 *   SHFL_UP    src = l - off, same clamp
 *   SHFL_XOR   src = l ^ off, same clamp
 *   SHFL_IDX   src = off mod width (CUDA rule), own value if src absent
 *   VOTE_ALL/VOTE_ANY  0/1 over participating lanes
 *   BALLOT     bit j set iff participating lane j of the segment has a != 0
 *   REDUCE_ADD wrapping sum over participating lanes */
int wf_warp_collective(int kind, const int32_t *a, const int32_t *b,
                       int32_t operand, int32_t *out, uint64_t n_threads,
                       int block, int width, uint32_t mask,
                       wf_stream_t stream);

/* ---- the reference's own DSL formulations (registry: dsl/patterns.py) ---
 * Reached from launch(hybrid_transform(kernel)) when the kernel is, up to
 * renaming, one the reference itself runs for this path; each writes exactly
 * what that DSL kernel writes.  Replaces runtime/launch.py:90 +
 * interp/mpmd.py:237-255 for these kernels.
 *
 * wf_warp_partials_sum_{i32,f32}: tests/golden/C1_{I32,F32}.spk = the
 *   SURVEY 8c per-warp-partials kernel.  out[b*(block/32) + w] = shfl_down
 *   tree (16,8,4,2,1) of each lane's grid-stride sum (i = tid, tid+S, ...
 *   while i < n, S = grid*block), fp32 in exactly that order.  Needs
 *   block % 32 == 0 and grid*block + n <= 2^31-1 (no i32 index wrap).
 * wf_warp_prefix32_i32: tests/golden/C3_WARP_PREFIX.spk (lane-reversed
 *   shfl_down suffix tree).  out[32s+k] = a[32s] + ... + a[32s+k], wrapping,
 *   for n = grid*block elements (n % 32 == 0). */
int wf_warp_partials_sum_i32(const int32_t *a, int32_t n, int32_t *out,
                             int grid, int block, wf_stream_t stream);
int wf_warp_partials_sum_f32(const float *a, int32_t n, float *out,
                             int grid, int block, wf_stream_t stream);
int wf_warp_prefix32_i32(const int32_t *a, int32_t *out, uint64_t n,
                         wf_stream_t stream);

/* ---- synthetic inputs (identical to oracle/synthetic.py) --------------- */
int wf_fill_synthetic(int gen, void *out, uint64_t n, uint64_t seed,
                      uint64_t index_base, uint32_t param, wf_stream_t stream);

/* ---- host-buffer entry points (end-to-end path) ------------------------
 * Same result contract as the device entry points, but `host_in` is host
 * memory (pinned for full PCIe speed).  The input is streamed through a
 * caller-provided device staging buffer in double-buffered chunks, each
 * chunk's copy overlapping the previous chunk's kernel; the scalar result is
 * copied back into *host_out.  Synchronous (returns after the result is in
 * host memory).  staging_bytes >= 2 MiB.  Concurrent calls on one device
 * are serialised (they share the device's copy streams); calls on different
 * devices run concurrently. */
int wf_reduce_sum_f32_host(const float *host_in, uint64_t n, float *host_out,
                           void *staging, size_t staging_bytes, void *ws,
                           size_t ws_bytes, wf_stream_t stream);
int wf_reduce_sum_i32_host(const int32_t *host_in, uint64_t n,
                           int32_t *host_out, void *staging,
                           size_t staging_bytes, void *ws, size_t ws_bytes,
                           wf_stream_t stream);
int wf_histogram256_u8_host(const uint8_t *host_in, uint64_t n,
                            uint64_t *host_bins, void *staging,
                            size_t staging_bytes, void *ws, size_t ws_bytes,
                            wf_stream_t stream);
/* Scan and compaction from host memory into host memory: a three-slot ring
 * in the staging buffer overlaps chunk c's H2D, chunk c-1's kernel and chunk
 * c-2's D2H (PCIe is full duplex).  The scan continues each chunk from the
 * previous chunk's last output (one carry chain, identical to one device
 * scan); `host_carry_in` may be NULL (carry 0).  The compaction writes the
 * selected elements of every chunk behind those of the previous ones
 * (== a[a > 0]) and their number into *host_count.  `ws` is sized for one
 * chunk (wf_workspace_bytes(op, staging_bytes / 4, 0) always suffices).
 * staging: 256-byte aligned, >= 3 MiB (scan) / 6 MiB (compaction).
 * Replaces the reference's copy-in / launch / copy-out of host buffers
 * (runtime/launch.py:105-134, runtime/memory.py:62-81). */
int wf_scan_inclusive_i32_host(const int32_t *host_in, int32_t *host_out,
                               uint64_t n, const int32_t *host_carry_in,
                               void *staging, size_t staging_bytes, void *ws,
                               size_t ws_bytes, wf_stream_t stream);
int wf_compact_gt0_i32_host(const int32_t *host_in, uint64_t n,
                            int32_t *host_out, uint64_t *host_count,
                            void *staging, size_t staging_bytes, void *ws,
                            size_t ws_bytes, wf_stream_t stream);

/* ---- DSL kernels compiled natively (replaces hybrid_transform + run_mpmd)
 * passes/pipeline.py:103-179 / interp/mpmd.py:237-255: the Python front end
 * (paper_2112_10034_b200/dsl) emits CUDA C with the reference's scalar and
 * collective semantics; these entry points compile it with NVRTC for sm_100a
 * (--fmad=false: one rounding per f32 op), load the cubin and
 * launch it.  `options` = extra space-separated NVRTC options (may be NULL);
 * the compile log (or error) is copied into `log`. */
int wf_jit_compile(const char *src, const char *kernel_name, const char *options,
                   void **module, char *log, size_t log_bytes);
int wf_jit_launch(void *module, uint32_t grid, uint32_t block, uint32_t smem_bytes,
                  void **args, wf_stream_t stream);
int wf_jit_unload(void *module);

#ifdef __cplusplus
}
#endif

#endif /* WARPFOLD_B200_H */
