// wf_abi.cu — the extern "C" boundary declared in include/warpfold_b200.h.
//
// Argument validation mirrors the reference's launch-time checks
// (runtime/launch.py:28-46 bind_args, config.py:26-41 validate) so the
// Python wrapper can raise the same exception classes; nothing here falls
// back to the CPU.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "wf_device.cuh"
#include "wf_internal.h"
#include "../../include/warpfold_b200.h"

namespace wf {

static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int set_error(int code, const char *msg) { return fail(code, "%s", msg); }

static int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return WF_OK;
  cudaGetLastError();  // clear the sticky-free error state
  return fail(int(e), "%s: %s", what, cudaGetErrorString(e));
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int sm_count(int device) {
  static int cache[64] = {};
  if (device < 0 || device >= 64) return 148;
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    cache[device] = v;
  }
  return cache[device];
}

static bool valid_reduce_block(int b) { return b == 128 || b == 256 || b == 512 || b == 1024; }

static size_t ws_need(int op, uint64_t n) {
  switch (op) {
    case WF_OP_REDUCE_SUM_I32:
    case WF_OP_REDUCE_SUM_F32:
      return kWsHeader + size_t(kMaxReduceGrid) * 8;
    case WF_OP_SCAN_INCLUSIVE_I32:
    case WF_OP_COMPACT_GT0_I32: {
      const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
      return kTileWsHeader + size_t(tiles < 1 ? 1 : tiles) * 8 * kDescStride;
    }
    case WF_OP_HISTOGRAM256_U8:
      return kWsHeader + 256 * 8;
    case WF_OP_WARP_COLLECTIVE:
      return 0;
    default:
      return 0;
  }
}

static int check_ws(int op, uint64_t n, void *ws, size_t ws_bytes) {
  const size_t need = ws_need(op, n);
  if (need == 0) return WF_OK;
  if (ws == nullptr) return fail(WF_ERR_WORKSPACE, "workspace is NULL (need %zu bytes)", need);
  if (ws_bytes < need)
    return fail(WF_ERR_WORKSPACE, "workspace of %zu bytes is too small (need %zu)", ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 255u)
    return fail(WF_ERR_WORKSPACE, "workspace must be 256-byte aligned");
  return WF_OK;
}

// ---- streams for the host-buffer (e2e) entry points ---------------------
struct CopyStreams {
  cudaStream_t copy[2] = {nullptr, nullptr};
  cudaEvent_t copied[2] = {nullptr, nullptr};
  cudaEvent_t consumed[2] = {nullptr, nullptr};
  // slot ring of the scan / compaction host paths (H2D in, kernel, D2H out,
  // all overlapped): landed / computed / drained per slot (kHostRing slots)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t landed[8] = {}, computed[8] = {}, drained[8] = {};
  uint64_t *pinned = nullptr;  // per-slot compaction counts read by the host
};
static std::mutex g_streams_mu;
static CopyStreams g_streams[64];
// Host-buffer calls on one device share its copy streams and events, so they
// are serialised per device (each call is synchronous and PCIe-bound anyway);
// calls on different devices run concurrently.
static std::mutex g_host_mu[64];
static std::unique_lock<std::mutex> host_call_lock() {
  const int dev = current_device();
  return std::unique_lock<std::mutex>(g_host_mu[dev >= 0 && dev < 64 ? dev : 0]);
}

static int get_copy_streams(CopyStreams *&cs) {
  const int dev = current_device();
  if (dev < 0 || dev >= 64) return fail(WF_ERR_CONFIG, "device %d out of range", dev);
  std::lock_guard<std::mutex> lk(g_streams_mu);
  CopyStreams &c = g_streams[dev];
  if (c.copy[0] == nullptr) {
    for (int k = 0; k < 2; ++k) {
      cudaError_t e = cudaStreamCreateWithFlags(&c.copy[k], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.copied[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.consumed[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_status(e, "creating copy streams");
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.d2h, cudaStreamNonBlocking);
    for (int k = 0; k < 8 && e == cudaSuccess; ++k) {
      e = cudaEventCreateWithFlags(&c.landed[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.computed[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.drained[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaHostAlloc(&c.pinned, 64, cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_status(e, "creating copy streams");
  }
  cs = &c;
  return WF_OK;
}

// Streams `n` elements of `elem` bytes from host memory through two staging
// halves.  `consume(dev_ptr, count, chunk_index)` enqueues the chunk's kernel
// on `stream`.  Copy of chunk c+1 overlaps the kernel of chunk c.
template <class F>
static int stream_chunks(const void *host_in, uint64_t n, size_t elem, void *staging,
                         size_t staging_bytes, cudaStream_t stream, F consume) {
  CopyStreams *cs = nullptr;
  int rc = get_copy_streams(cs);
  if (rc) return rc;
  const size_t half = (staging_bytes / 2) & ~size_t(255);
  const uint64_t per_chunk = half / elem;
  const uint64_t nchunks = (n + per_chunk - 1) / per_chunk;
  for (uint64_t c = 0; c < nchunks; ++c) {
    const int k = int(c & 1);
    const uint64_t first = c * per_chunk;
    const uint64_t cnt = (n - first) < per_chunk ? (n - first) : per_chunk;
    char *dst = static_cast<char *>(staging) + size_t(k) * half;
    cudaError_t e = cudaSuccess;
    if (c >= 2) e = cudaStreamWaitEvent(cs->copy[k], cs->consumed[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dst, static_cast<const char *>(host_in) + first * elem, cnt * elem,
                          cudaMemcpyHostToDevice, cs->copy[k]);
    if (e == cudaSuccess) e = cudaEventRecord(cs->copied[k], cs->copy[k]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, cs->copied[k], 0);
    if (e != cudaSuccess) return cuda_status(e, "staging copy");
    e = consume(dst, cnt, c);
    if (e == cudaSuccess) e = cudaEventRecord(cs->consumed[k], stream);
    if (e != cudaSuccess) return cuda_status(e, "chunk kernel");
  }
  return WF_OK;
}

}  // namespace wf

using namespace wf;

extern "C" {

const char *wf_version(void) { return "warpfold_b200 0.1.0 (sm_100a)"; }
int wf_abi_version(void) { return WF_ABI_VERSION; }
const char *wf_last_error(void) { return g_last_error.c_str(); }

int wf_device_sm_count(int device) { return sm_count(device); }

size_t wf_workspace_bytes(int op, uint64_t n, int block) {
  (void)block;
  return ws_need(op, n);
}

int wf_workspace_init(void *ws, size_t ws_bytes, wf_stream_t stream) {
  if (ws == nullptr || ws_bytes == 0) return WF_OK;
  return cuda_status(cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream)),
                     "workspace init");
}

void wf_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  for (auto &c : g_streams) {
    for (int k = 0; k < 2; ++k) {
      if (c.copy[k]) cudaStreamDestroy(c.copy[k]);
      if (c.copied[k]) cudaEventDestroy(c.copied[k]);
      if (c.consumed[k]) cudaEventDestroy(c.consumed[k]);
      c.copy[k] = nullptr;
      c.copied[k] = c.consumed[k] = nullptr;
    }
    if (c.h2d) cudaStreamDestroy(c.h2d);
    if (c.d2h) cudaStreamDestroy(c.d2h);
    for (int k = 0; k < 3; ++k) {
      if (c.landed[k]) cudaEventDestroy(c.landed[k]);
      if (c.computed[k]) cudaEventDestroy(c.computed[k]);
      if (c.drained[k]) cudaEventDestroy(c.drained[k]);
      c.landed[k] = c.computed[k] = c.drained[k] = nullptr;
    }
    if (c.pinned) cudaFreeHost(c.pinned);
    c.h2d = c.d2h = nullptr;
    c.pinned = nullptr;
  }
}

static int reduce_common(int op, const void *in, uint64_t n, void *out, int block, int grid,
                         void *ws, size_t ws_bytes) {
  if (!valid_reduce_block(block))
    return fail(WF_ERR_CONFIG, "block size must be one of 128/256/512/1024, got %d", block);
  if (grid < 0 || grid > int(kMaxReduceGrid))
    return fail(WF_ERR_CONFIG, "grid size must be in [0, %u], got %d", kMaxReduceGrid, grid);
  if (out == nullptr) return fail(WF_ERR_ARG, "output pointer is NULL");
  if (n > 0 && in == nullptr) return fail(WF_ERR_ARG, "input pointer is NULL");
  if (reinterpret_cast<uintptr_t>(in) & 3u) return fail(WF_ERR_ARG, "input must be 4-byte aligned");
  return check_ws(op, n, ws, ws_bytes);
}

int wf_reduce_sum_i32(const int32_t *in, uint64_t n, int32_t *out, int block, int grid,
                      void *ws, size_t ws_bytes, wf_stream_t stream) {
  int rc = reduce_common(WF_OP_REDUCE_SUM_I32, in, n, out, block, grid, ws, ws_bytes);
  if (rc) return rc;
  if (grid == 0) grid = auto_reduce_grid(kRedI32, block, n);
  return cuda_status(launch_reduce_i32(in, n, out, block, grid, ws, static_cast<cudaStream_t>(stream)),
                     "reduce_sum_i32");
}

int wf_reduce_sum_f32(const float *in, uint64_t n, float *out, int block, int grid, void *ws,
                      size_t ws_bytes, wf_stream_t stream) {
  return wf_reduce_sum_f32_ex(in, n, out, block, grid, ws, ws_bytes, 0u, stream);
}

int wf_reduce_sum_f32_ex(const float *in, uint64_t n, float *out, int block, int grid, void *ws,
                         size_t ws_bytes, unsigned flags, wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  int rc = reduce_common(WF_OP_REDUCE_SUM_F32, in, n, out, block, grid, ws, ws_bytes);
  if (rc) return rc;
  if (grid == 0) grid = auto_reduce_grid(kRedF32, block, n);
  return cuda_status(launch_reduce_f32(in, n, out, block, grid, ws, static_cast<cudaStream_t>(stream),
                                       (flags & WF_FLAG_INPUT_STABLE) != 0),
                     "reduce_sum_f32");
}

size_t wf_mailbox_bytes(int world) {
  return world < 1 ? 0 : (size_t(2) * size_t(world) * 8 + 255) & ~size_t(255);
}

// Every kernel that may spin on its peers, loaded on the current device at
// mailbox set-up (before any exchange can be in flight): with lazy module
// loading, the first launch of a not-yet-loaded kernel can wait for the
// device to go idle — which a peer kernel already spinning on the same
// device never lets happen (ranks sharing a device, the wf_mg ABI).
static int preload_exchange_kernels() {
  cudaError_t e = preload_peer_kernels();
  if (e == cudaSuccess) e = preload_hist_mg_kernels();
  if (e == cudaSuccess) e = preload_reduce_mg_kernels();
  if (e == cudaSuccess) e = preload_tmem_mg_kernels();
  return cuda_status(e, "loading the exchange kernels");
}

int wf_mailbox_alloc(int world, void **d_mailbox) {
  if (d_mailbox == nullptr || world < 1 || world > 32)
    return fail(WF_ERR_ARG, "mailbox: world must be in [1, 32]");
  if (int rc = preload_exchange_kernels()) return rc;
  const size_t b = wf_mailbox_bytes(world);
  int rc = cuda_status(cudaMalloc(d_mailbox, b), "mailbox alloc");
  if (rc) return rc;
  return cuda_status(cudaMemset(*d_mailbox, 0, b), "mailbox zero");
}

int wf_mailbox_free(void *d_mailbox) { return cuda_status(cudaFree(d_mailbox), "mailbox free"); }

int wf_ipc_handle(void *d_ptr, void *handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  if (d_ptr == nullptr || handle64 == nullptr) return fail(WF_ERR_ARG, "NULL pointer");
  cudaIpcMemHandle_t h;
  int rc = cuda_status(cudaIpcGetMemHandle(&h, d_ptr), "cudaIpcGetMemHandle");
  if (rc) return rc;
  memcpy(handle64, &h, sizeof h);
  return WF_OK;
}

int wf_ipc_open(const void *handle64, void **d_ptr) {
  if (d_ptr == nullptr || handle64 == nullptr) return fail(WF_ERR_ARG, "NULL pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  return cuda_status(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess),
                     "cudaIpcOpenMemHandle");
}

int wf_ipc_close(void *d_ptr) { return cuda_status(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle"); }

int wf_reduce_sum_f32_mg(const float *in, uint64_t n, float *out, int block, int grid, void *ws,
                         size_t ws_bytes, void *const *d_peers, const void *d_mailbox, int rank,
                         int world, uint32_t epoch, wf_stream_t stream) {
  return wf_reduce_sum_f32_mg_ex(in, n, out, block, grid, ws, ws_bytes, d_peers, d_mailbox, rank,
                                 world, epoch, 0u, stream);
}

int wf_reduce_sum_f32_mg_ex(const float *in, uint64_t n, float *out, int block, int grid,
                            void *ws, size_t ws_bytes, void *const *d_peers,
                            const void *d_mailbox, int rank, int world, uint32_t epoch,
                            unsigned flags, wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  int rc = reduce_common(WF_OP_REDUCE_SUM_F32, in, n, out, block, grid, ws, ws_bytes);
  if (rc) return rc;
  if (d_peers == nullptr || d_mailbox == nullptr) return fail(WF_ERR_ARG, "NULL mailbox pointer");
  if (world < 1 || world > 32 || rank < 0 || rank >= world)
    return fail(WF_ERR_ARG, "rank %d / world %d out of range (world <= 32)", rank, world);
  if (epoch == 0) return fail(WF_ERR_ARG, "epoch must start at 1");
  if (grid == 0) grid = auto_reduce_grid(kRedF32Mg, block, n);
  return cuda_status(launch_reduce_f32_mg(in, n, out, block, grid, ws, d_peers, d_mailbox, rank,
                                          world, epoch, (flags & WF_FLAG_INPUT_STABLE) != 0,
                                          static_cast<cudaStream_t>(stream)),
                     "reduce_sum_f32_mg");
}

size_t wf_peer_mailbox_bytes(int world, uint32_t cap) {
  return world < 1 ? 0 : peer_mailbox_bytes(world, cap);
}

int wf_peer_mailbox_alloc(int world, uint32_t cap, void **d_mailbox) {
  if (d_mailbox == nullptr || world < 1 || world > 256 || cap < 1 || cap > (1u << 20))
    return fail(WF_ERR_ARG, "peer mailbox: world in [1, 256], cap in [1, 2^20]");
  if (int rc = preload_exchange_kernels()) return rc;
  const size_t b = peer_mailbox_bytes(world, cap);
  int rc = cuda_status(cudaMalloc(d_mailbox, b), "peer mailbox alloc");
  if (rc) return rc;
  return cuda_status(cudaMemset(*d_mailbox, 0, b), "peer mailbox zero");
}

static int check_peer(void *const *d_peers, const void *d_mailbox, uint32_t cap, uint32_t need,
                      int rank, int world, uint32_t epoch, uint32_t *d_err) {
  if (d_peers == nullptr || d_mailbox == nullptr || d_err == nullptr)
    return fail(WF_ERR_ARG, "NULL pointer");
  if (world < 1 || world > 256 || rank < 0 || rank >= world)
    return fail(WF_ERR_ARG, "rank %d / world %d out of range", rank, world);
  if (cap < need) return fail(WF_ERR_ARG, "peer mailbox cap %u < %u payload words", cap, need);
  if (epoch == 0) return fail(WF_ERR_ARG, "epoch must start at 1");
  return WF_OK;
}

int wf_reduce_sum_i32_exscan_mg(const int32_t *in, uint64_t n, int32_t *d_out2, int block,
                                int grid, void *ws, size_t ws_bytes, void *const *d_peers,
                                const void *d_mailbox, uint32_t cap, int rank, int world,
                                uint32_t epoch, uint32_t *d_err, wf_stream_t stream) {
  return wf_reduce_sum_i32_exscan_mg_ex(in, n, d_out2, block, grid, ws, ws_bytes, d_peers,
                                        d_mailbox, cap, rank, world, epoch, d_err, 0u, stream);
}

int wf_reduce_sum_i32_exscan_mg_ex(const int32_t *in, uint64_t n, int32_t *d_out2, int block,
                                   int grid, void *ws, size_t ws_bytes, void *const *d_peers,
                                   const void *d_mailbox, uint32_t cap, int rank, int world,
                                   uint32_t epoch, uint32_t *d_err, unsigned flags,
                                   wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  int rc = reduce_common(WF_OP_REDUCE_SUM_I32, in, n, d_out2, block, grid, ws, ws_bytes);
  if (rc) return rc;
  rc = check_peer(d_peers, d_mailbox, cap, 1, rank, world, epoch, d_err);
  if (rc) return rc;
  if (grid == 0) grid = auto_reduce_grid(kRedI32Px, block, n);
  return cuda_status(launch_reduce_i32_exscan_mg(in, n, d_out2, block, grid, ws, d_peers,
                                                 d_mailbox, cap, rank, world, epoch, d_err,
                                                 static_cast<cudaStream_t>(stream),
                                                 (flags & WF_FLAG_INPUT_STABLE) != 0),
                     "reduce_sum_i32_exscan_mg");
}

int wf_scan_inclusive_i32_cyclic_mg(const int32_t *in, int32_t *out, uint64_t n, void *ws,
                                    size_t ws_bytes, void *const *d_peers,
                                    const void *d_mailbox, uint32_t cap, int rank, int world,
                                    uint32_t epoch, uint32_t *d_err, uint64_t round_elems,
                                    uint32_t rounds, int max_grid, unsigned flags,
                                    wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (n > 0 && (in == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u)
    return fail(WF_ERR_ARG, "the block-cyclic scan takes 16-byte aligned buffers");
  if (round_elems == 0 || round_elems % kTmemTile != 0 || round_elems > (uint64_t(1) << 31))
    return fail(WF_ERR_ARG, "round_elems must be a positive multiple of %u (<= 2^31), got %llu",
                unsigned(kTmemTile), (unsigned long long)round_elems);
  if (uint64_t(rounds) * round_elems < n)
    return fail(WF_ERR_ARG, "%u rounds of %llu elements cannot hold n=%llu", rounds,
                (unsigned long long)round_elems, (unsigned long long)n);
  if (world > 32) return fail(WF_ERR_ARG, "world %d > 32", world);
  if (max_grid < 0) return fail(WF_ERR_CONFIG, "max_grid must be >= 0, got %d", max_grid);
  int rc = check_ws(WF_OP_SCAN_INCLUSIVE_I32, n, ws, ws_bytes);
  if (rc) return rc;
  rc = check_peer(d_peers, d_mailbox, cap, rounds, rank, world, epoch, d_err);
  if (rc) return rc;
  return cuda_status(
      launch_scan_tmem_i32_cyclic(in, out, n, ws, d_peers, d_mailbox, cap, rank, world, epoch,
                                  d_err, uint32_t(round_elems / kTmemTile), rounds, max_grid,
                                  static_cast<cudaStream_t>(stream),
                                  (flags & WF_FLAG_INPUT_STABLE) != 0),
      "scan_inclusive_i32_cyclic_mg");
}

int wf_compact_gt0_i32_mg(const int32_t *in, uint64_t n, int32_t *out, uint64_t *d_counts3,
                          void *ws, size_t ws_bytes, void *const *d_peers, const void *d_mailbox,
                          uint32_t cap, int rank, int world, uint32_t epoch, uint32_t *d_err,
                          wf_stream_t stream) {
  return wf_compact_gt0_i32_mg_ex(in, n, out, d_counts3, ws, ws_bytes, d_peers, d_mailbox, cap,
                                  rank, world, epoch, d_err, 0u, stream);
}

int wf_compact_gt0_i32_mg_ex(const int32_t *in, uint64_t n, int32_t *out, uint64_t *d_counts3,
                             void *ws, size_t ws_bytes, void *const *d_peers,
                             const void *d_mailbox, uint32_t cap, int rank, int world,
                             uint32_t epoch, uint32_t *d_err, unsigned flags,
                             wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (d_counts3 == nullptr) return fail(WF_ERR_ARG, "counts pointer is NULL");
  if (n > 0 && (in == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 3u)
    return fail(WF_ERR_ARG, "buffers must be 4-byte aligned");
  if (n > 0xffffffffull)
    return fail(WF_ERR_ARG, "compaction takes n < 2^32 per call, got %llu", (unsigned long long)n);
  int rc = check_ws(WF_OP_COMPACT_GT0_I32, n, ws, ws_bytes);
  if (rc) return rc;
  rc = check_peer(d_peers, d_mailbox, cap, 1, rank, world, epoch, d_err);
  if (rc) return rc;
  return cuda_status(launch_compact_gt0_i32_mg(in, n, out, d_counts3, ws, d_peers, d_mailbox, cap,
                                               rank, world, epoch, d_err,
                                               static_cast<cudaStream_t>(stream),
                                               (flags & WF_FLAG_INPUT_STABLE) != 0),
                     "compact_gt0_i32_mg");
}

int wf_histogram256_u8_mg(const uint8_t *in, uint64_t n, uint64_t *d_bins, void *ws,
                          size_t ws_bytes, void *const *d_peers, const void *d_mailbox,
                          uint32_t cap, int rank, int world, uint32_t epoch, uint32_t *d_err,
                          wf_stream_t stream) {
  return wf_histogram256_u8_mg_ex(in, n, d_bins, ws, ws_bytes, d_peers, d_mailbox, cap, rank,
                                  world, epoch, d_err, 0u, stream);
}

int wf_histogram256_u8_mg_ex(const uint8_t *in, uint64_t n, uint64_t *d_bins, void *ws,
                             size_t ws_bytes, void *const *d_peers, const void *d_mailbox,
                             uint32_t cap, int rank, int world, uint32_t epoch, uint32_t *d_err,
                             unsigned flags, wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (d_bins == nullptr) return fail(WF_ERR_ARG, "bins pointer is NULL");
  if (n && in == nullptr) return fail(WF_ERR_ARG, "input pointer is NULL");
  int rc = check_ws(WF_OP_HISTOGRAM256_U8, n, ws, ws_bytes);
  if (rc) return rc;
  rc = check_peer(d_peers, d_mailbox, cap, 256, rank, world, epoch, d_err);
  if (rc) return rc;
  return cuda_status(launch_hist256_mg(in, n, d_bins, auto_hist_grid(n), ws, d_peers, d_mailbox,
                                       cap, rank, world, epoch, d_err,
                                       static_cast<cudaStream_t>(stream),
                                       (flags & WF_FLAG_INPUT_STABLE) != 0),
                     "histogram256_u8_mg");
}

int wf_peer_exchange(int mode, const void *d_vals, uint32_t count, uint32_t cap, void *d_out,
                     void *const *d_peers, const void *d_mailbox, int rank, int world,
                     uint32_t epoch, uint32_t *d_err, wf_stream_t stream) {
  if (mode < WF_PEER_ALLGATHER || mode > WF_PEER_EXSCAN_U32)
    return fail(WF_ERR_ARG, "unknown peer exchange mode %d", mode);
  if (d_vals == nullptr || d_out == nullptr || d_peers == nullptr || d_mailbox == nullptr ||
      d_err == nullptr)
    return fail(WF_ERR_ARG, "NULL pointer");
  if (world < 1 || world > 256 || rank < 0 || rank >= world)
    return fail(WF_ERR_ARG, "rank %d / world %d out of range", rank, world);
  if (count < 1 || count > cap) return fail(WF_ERR_ARG, "count %u must be in [1, cap=%u]", count, cap);
  if ((mode == WF_PEER_EXSCAN || mode == WF_PEER_EXSCAN_U32) && count != 1)
    return fail(WF_ERR_ARG, "exclusive scan exchanges one value per rank");
  if (epoch == 0) return fail(WF_ERR_ARG, "epoch must start at 1");
  return cuda_status(launch_peer_exchange(mode, d_vals, count, cap, d_out, d_peers, d_mailbox,
                                          rank, world, epoch, d_err,
                                          static_cast<cudaStream_t>(stream)),
                     "peer_exchange");
}

int wf_fold_f32(const float *vals, uint32_t count, float *out, wf_stream_t stream) {
  if (out == nullptr || (count && vals == nullptr)) return fail(WF_ERR_ARG, "NULL pointer");
  return cuda_status(launch_fold_f32(vals, count, out, static_cast<cudaStream_t>(stream)), "fold_f32");
}

int wf_fold_i32(const int32_t *vals, uint32_t count, int32_t *out, wf_stream_t stream) {
  if (out == nullptr || (count && vals == nullptr)) return fail(WF_ERR_ARG, "NULL pointer");
  return cuda_status(launch_fold_i32(vals, count, out, static_cast<cudaStream_t>(stream)), "fold_i32");
}

int wf_fold_u64(const uint64_t *vals, uint32_t count, uint64_t *out, wf_stream_t stream) {
  if (out == nullptr || (count && vals == nullptr)) return fail(WF_ERR_ARG, "NULL pointer");
  return cuda_status(launch_fold_u64(vals, count, out, static_cast<cudaStream_t>(stream)), "fold_u64");
}

int wf_scan_inclusive_i32(const int32_t *in, int32_t *out, uint64_t n, const int32_t *d_carry_in,
                          void *ws, size_t ws_bytes, wf_stream_t stream) {
  return wf_scan_inclusive_i32_ex(in, out, n, d_carry_in, ws, ws_bytes, 0u, stream);
}

int wf_scan_inclusive_i32_ex(const int32_t *in, int32_t *out, uint64_t n,
                             const int32_t *d_carry_in, void *ws, size_t ws_bytes, unsigned flags,
                             wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (n > 0 && (in == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 3u)
    return fail(WF_ERR_ARG, "buffers must be 4-byte aligned");
  if (n > (uint64_t(0xffffffffu) * kScanTile))
    return fail(WF_ERR_ARG, "n=%llu exceeds the tile-id range", (unsigned long long)n);
  int rc = check_ws(WF_OP_SCAN_INCLUSIVE_I32, n, ws, ws_bytes);
  if (rc) return rc;
  return cuda_status(launch_scan_i32(in, out, n, d_carry_in, ws, static_cast<cudaStream_t>(stream),
                                     (flags & WF_FLAG_INPUT_STABLE) != 0),
                     "scan_inclusive_i32");
}

int wf_compact_gt0_i32(const int32_t *in, uint64_t n, int32_t *out, uint64_t *d_count, void *ws,
                       size_t ws_bytes, wf_stream_t stream) {
  return wf_compact_gt0_i32_ex(in, n, out, d_count, ws, ws_bytes, 0u, stream);
}

int wf_compact_gt0_i32_ex(const int32_t *in, uint64_t n, int32_t *out, uint64_t *d_count,
                          void *ws, size_t ws_bytes, unsigned flags, wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (d_count == nullptr) return fail(WF_ERR_ARG, "count pointer is NULL");
  if (n > 0 && (in == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 3u)
    return fail(WF_ERR_ARG, "buffers must be 4-byte aligned");
  if (n > 0xffffffffull)
    return fail(WF_ERR_ARG, "compaction takes n < 2^32 per call, got %llu", (unsigned long long)n);
  int rc = check_ws(WF_OP_COMPACT_GT0_I32, n, ws, ws_bytes);
  if (rc) return rc;
  return cuda_status(
      launch_compact_gt0_i32(in, n, out, d_count, ws, static_cast<cudaStream_t>(stream),
                             (flags & WF_FLAG_INPUT_STABLE) != 0),
      "compact_gt0_i32");
}

int wf_histogram256_u8(const uint8_t *in, uint64_t n, uint64_t *bins, int grid, void *ws,
                       size_t ws_bytes, wf_stream_t stream) {
  return wf_histogram256_u8_ex(in, n, bins, grid, ws, ws_bytes, 0u, stream);
}

int wf_histogram256_u8_ex(const uint8_t *in, uint64_t n, uint64_t *bins, int grid, void *ws,
                          size_t ws_bytes, unsigned flags, wf_stream_t stream) {
  if (flags & ~unsigned(WF_FLAG_INPUT_STABLE)) return fail(WF_ERR_ARG, "unknown flags 0x%x", flags);
  if (bins == nullptr) return fail(WF_ERR_ARG, "bins pointer is NULL");
  if (n > 0 && in == nullptr) return fail(WF_ERR_ARG, "input pointer is NULL");
  if (grid < 0) return fail(WF_ERR_CONFIG, "grid size must be >= 0, got %d", grid);
  int rc = check_ws(WF_OP_HISTOGRAM256_U8, n, ws, ws_bytes);
  if (rc) return rc;
  if (grid == 0) grid = auto_hist_grid(n);
  if (grid < min_hist_grid(n)) grid = min_hist_grid(n);  // u32 lane counters stay < 2^32
  return cuda_status(
      launch_hist256(in, n, bins, false, grid, ws, static_cast<cudaStream_t>(stream),
                     (flags & WF_FLAG_INPUT_STABLE) != 0),
      "histogram256_u8");
}

int wf_warp_collective(int kind, const int32_t *a, const int32_t *b, int32_t operand, int32_t *out,
                       uint64_t n_threads, int block, int width, uint32_t mask,
                       wf_stream_t stream) {
  if (kind < WF_COLL_SHFL_DOWN || kind > WF_COLL_REDUCE_ADD)
    return fail(WF_ERR_UNSUPPORTED, "unknown warp collective kind %d", kind);
  if (block < 1 || block > 1024) return fail(WF_ERR_CONFIG, "block size must be in [1, 1024], got %d", block);
  if (width < 1 || width > 32 || (width & (width - 1)))
    return fail(WF_ERR_CONFIG, "warp width must be a power of two in [1, 32], got %d", width);
  if (n_threads % uint64_t(block))
    return fail(WF_ERR_CONFIG, "n_threads (%llu) must be a multiple of the block size (%d)",
                (unsigned long long)n_threads, block);
  if (n_threads / uint64_t(block) > 0x7fffffffull) return fail(WF_ERR_CONFIG, "grid too large");
  if (n_threads && (a == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  return cuda_status(launch_warp_collective(kind, a, b, operand, out, n_threads, block, width, mask,
                                            static_cast<cudaStream_t>(stream)),
                     "warp_collective");
}

// ---- the reference's DSL formulations (dsl/patterns.py registry) ---------
static int check_partials(const void *a, int32_t n, const void *out, int grid, int block) {
  if (block < 32 || block > 1024 || block % 32)
    return fail(WF_ERR_CONFIG, "block size must be a multiple of 32 in [32, 1024], got %d", block);
  if (grid < 0) return fail(WF_ERR_CONFIG, "grid size must be >= 0, got %d", grid);
  if (int64_t(grid) * block + (n > 0 ? n : 0) > 0x7fffffffll)
    return fail(WF_ERR_ARG, "grid-stride index would overflow i32 (grid %d x block %d, n %d)",
                grid, block, n);
  if (grid && (out == nullptr || (n > 0 && a == nullptr)))
    return fail(WF_ERR_ARG, "NULL buffer pointer");
  return WF_OK;
}

int wf_warp_partials_sum_i32(const int32_t *a, int32_t n, int32_t *out, int grid, int block,
                             wf_stream_t stream) {
  if (int rc = check_partials(a, n, out, grid, block)) return rc;
  return cuda_status(launch_warp_partials(false, a, n, out, grid, block,
                                          static_cast<cudaStream_t>(stream)),
                     "warp_partials_sum_i32");
}

int wf_warp_partials_sum_f32(const float *a, int32_t n, float *out, int grid, int block,
                             wf_stream_t stream) {
  if (int rc = check_partials(a, n, out, grid, block)) return rc;
  return cuda_status(launch_warp_partials(true, a, n, out, grid, block,
                                          static_cast<cudaStream_t>(stream)),
                     "warp_partials_sum_f32");
}

int wf_warp_prefix32_i32(const int32_t *a, int32_t *out, uint64_t n, wf_stream_t stream) {
  if (n % 32) return fail(WF_ERR_CONFIG, "n (%llu) must be a multiple of 32", (unsigned long long)n);
  if (n && (a == nullptr || out == nullptr)) return fail(WF_ERR_ARG, "NULL buffer pointer");
  return cuda_status(launch_warp_prefix32(a, out, n, static_cast<cudaStream_t>(stream)),
                     "warp_prefix32_i32");
}

int wf_fill_synthetic(int gen, void *out, uint64_t n, uint64_t seed, uint64_t index_base,
                      uint32_t param, wf_stream_t stream) {
  if (gen < WF_GEN_I32_FULL || gen > WF_GEN_I32_SELECT)
    return fail(WF_ERR_UNSUPPORTED, "unknown generator %d", gen);
  if (n && out == nullptr) return fail(WF_ERR_ARG, "output pointer is NULL");
  return cuda_status(
      launch_fill_synthetic(gen, out, n, seed, index_base, param, static_cast<cudaStream_t>(stream)),
      "fill_synthetic");
}

}  // extern "C"

// ---- host-buffer entry points --------------------------------------------
namespace wf {
template <class T, class Launch, class Fold>
static int reduce_host(int op, const T *host_in, uint64_t n, T *host_out, void *staging,
                       size_t staging_bytes, void *ws, size_t ws_bytes, wf_stream_t stream,
                       Launch launch_one, Fold fold) {
  if (host_out == nullptr) return fail(WF_ERR_ARG, "host output pointer is NULL");
  if (n && host_in == nullptr) return fail(WF_ERR_ARG, "host input pointer is NULL");
  if (staging == nullptr || staging_bytes < (size_t(2) << 20))
    return fail(WF_ERR_ARG, "staging buffer must be at least 2 MiB");
  // chunk partials live in the tail of the staging buffer
  const size_t slots = 4096;
  const size_t body = (staging_bytes - slots * sizeof(T)) & ~size_t(511);
  T *partials = reinterpret_cast<T *>(static_cast<char *>(staging) + body);
  const uint64_t per_chunk = (body / 2 & ~size_t(255)) / sizeof(T);
  if ((n + per_chunk - 1) / per_chunk > slots)
    return fail(WF_ERR_ARG, "staging buffer too small for n=%llu", (unsigned long long)n);
  int rc = check_ws(op, n, ws, ws_bytes);
  if (rc) return rc;
  auto lk = host_call_lock();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t nchunks = 0;
  rc = stream_chunks(host_in, n, sizeof(T), staging, body, s,
                     [&](void *dev, uint64_t cnt, uint64_t c) {
                       nchunks = c + 1;
                       return launch_one(static_cast<const T *>(dev), cnt, partials + c, s);
                     });
  if (rc) return rc;
  cudaError_t e = fold(partials, uint32_t(nchunks), partials + slots - 1, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(host_out, partials + slots - 1, sizeof(T), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e, "host reduction");
}
}  // namespace wf

extern "C" {

int wf_reduce_sum_f32_host(const float *host_in, uint64_t n, float *host_out, void *staging,
                           size_t staging_bytes, void *ws, size_t ws_bytes, wf_stream_t stream) {
  return reduce_host<float>(
      WF_OP_REDUCE_SUM_F32, host_in, n, host_out, staging, staging_bytes, ws, ws_bytes, stream,
      [&](const float *d, uint64_t cnt, float *o, cudaStream_t s) {
        return launch_reduce_f32(d, cnt, o, 512, auto_reduce_grid(kRedF32, 512, cnt), ws, s);
      },
      [](const float *v, uint32_t c, float *o, cudaStream_t s) { return launch_fold_f32(v, c, o, s); });
}

int wf_reduce_sum_i32_host(const int32_t *host_in, uint64_t n, int32_t *host_out, void *staging,
                           size_t staging_bytes, void *ws, size_t ws_bytes, wf_stream_t stream) {
  return reduce_host<int32_t>(
      WF_OP_REDUCE_SUM_I32, host_in, n, host_out, staging, staging_bytes, ws, ws_bytes, stream,
      [&](const int32_t *d, uint64_t cnt, int32_t *o, cudaStream_t s) {
        return launch_reduce_i32(d, cnt, o, 256, auto_reduce_grid(kRedI32, 256, cnt), ws, s);
      },
      [](const int32_t *v, uint32_t c, int32_t *o, cudaStream_t s) { return launch_fold_i32(v, c, o, s); });
}

int wf_histogram256_u8_host(const uint8_t *host_in, uint64_t n, uint64_t *host_bins, void *staging,
                            size_t staging_bytes, void *ws, size_t ws_bytes, wf_stream_t stream) {
  if (host_bins == nullptr) return fail(WF_ERR_ARG, "host bins pointer is NULL");
  if (n && host_in == nullptr) return fail(WF_ERR_ARG, "host input pointer is NULL");
  if (staging == nullptr || staging_bytes < (size_t(2) << 20))
    return fail(WF_ERR_ARG, "staging buffer must be at least 2 MiB");
  int rc = check_ws(WF_OP_HISTOGRAM256_U8, n, ws, ws_bytes);
  if (rc) return rc;
  auto lk = host_call_lock();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t body = (staging_bytes - 4096) & ~size_t(511);
  uint64_t *dbins = reinterpret_cast<uint64_t *>(static_cast<char *>(staging) + body);
  cudaError_t e = cudaMemsetAsync(dbins, 0, 256 * sizeof(uint64_t), s);
  if (e != cudaSuccess) return cuda_status(e, "bins init");
  rc = stream_chunks(host_in, n, 1, staging, body, s, [&](void *dev, uint64_t cnt, uint64_t) {
    return launch_hist256(static_cast<const uint8_t *>(dev), cnt, dbins, true, auto_hist_grid(cnt),
                          ws, s);
  });
  if (rc) return rc;
  e = cudaMemcpyAsync(host_bins, dbins, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e, "host histogram");
}

}  // extern "C"

// ---- host-buffer scan and compaction: three-slot H2D / kernel / D2H ring ---
// Reference analog: the reference's memory is host memory and its launch
// copies every buffer in and out (runtime/launch.py:105-134,
// runtime/memory.py:62-81).  Here chunk c's H2D (h2d stream), chunk c-1's
// kernel (caller's stream) and chunk c-2's D2H (d2h stream) run at once; PCIe
// is full duplex, so the D2H of the result hides under the H2D of the input.
namespace wf {
namespace {
// 8 slots of at most 16 MiB: the pipeline fill (first H2D) and drain (last
// D2H) that no copy in the other direction hides are one small chunk each
// (3 slots of 85 MiB measured 0.905 of the concurrent-copy ceiling for the
// 2^28 scan: 8 % of the time was fill + drain)
#ifndef WF_RING_CHUNK_MB
#define WF_RING_CHUNK_MB 16
#endif
#ifndef WF_RING_SKIP_KERNEL
#define WF_RING_SKIP_KERNEL 0  // tools-only A/B: the ring's copies without the scan kernel
#endif
constexpr int kRing = 8;
constexpr size_t kRingChunkMax = size_t(WF_RING_CHUNK_MB) << 20;

int host_ring_checks(const void *host_in, const void *host_out, uint64_t n, void *staging,
                     size_t staging_bytes, size_t min_bytes) {
  if (n && (host_in == nullptr || host_out == nullptr))
    return fail(WF_ERR_ARG, "host buffer pointer is NULL");
  if (staging == nullptr || staging_bytes < min_bytes)
    return fail(WF_ERR_ARG, "staging buffer must be at least %zu bytes", min_bytes);
  if (reinterpret_cast<uintptr_t>(staging) & 255u)
    return fail(WF_ERR_ARG, "staging buffer must be 256-byte aligned");
  return WF_OK;
}
}  // namespace
}  // namespace wf

extern "C" {

int wf_scan_inclusive_i32_host(const int32_t *host_in, int32_t *host_out, uint64_t n,
                               const int32_t *host_carry_in, void *staging, size_t staging_bytes,
                               void *ws, size_t ws_bytes, wf_stream_t stream) {
  int rc = host_ring_checks(host_in, host_out, n, staging, staging_bytes, size_t(3) << 20);
  if (rc) return rc;
  // [0, 256): carry-in slot; then kRing in-place chunk buffers
  size_t buf = ((staging_bytes - 256) / kRing) & ~size_t(255);
  if (buf > kRingChunkMax) buf = kRingChunkMax;
  const uint64_t per_chunk = buf / 4;
  rc = check_ws(WF_OP_SCAN_INCLUSIVE_I32, per_chunk, ws, ws_bytes);
  if (rc) return rc;
  auto lk = host_call_lock();
  CopyStreams *cs = nullptr;
  if ((rc = get_copy_streams(cs))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char *base = static_cast<char *>(staging);
  int32_t *d_carry = reinterpret_cast<int32_t *>(base);
  cudaError_t e = cudaSuccess;
  if (host_carry_in != nullptr)
    e = cudaMemcpyAsync(d_carry, host_carry_in, 4, cudaMemcpyHostToDevice, s);
  const int32_t *carry = host_carry_in != nullptr ? d_carry : nullptr;
  const uint64_t nchunks = (n + per_chunk - 1) / per_chunk;
  for (uint64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    const int k = int(c % kRing);
    const uint64_t first = c * per_chunk;
    const uint64_t cnt = (n - first) < per_chunk ? (n - first) : per_chunk;
    int32_t *dbuf = reinterpret_cast<int32_t *>(base + 256 + size_t(k) * buf);
    if (c >= kRing) {  // slot k: chunk c-kRing drained, and chunk c-kRing+1 read its carry from it
      e = cudaStreamWaitEvent(cs->h2d, cs->drained[k], 0);
      if (e == cudaSuccess)
        e = cudaStreamWaitEvent(cs->h2d, cs->computed[(c - kRing + 1) % kRing], 0);
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dbuf, host_in + first, cnt * 4, cudaMemcpyHostToDevice, cs->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(cs->landed[k], cs->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, cs->landed[k], 0);
    if (e == cudaSuccess && !WF_RING_SKIP_KERNEL) e = launch_scan_i32(dbuf, dbuf, cnt, carry, ws, s);
    if (e == cudaSuccess) e = cudaEventRecord(cs->computed[k], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs->d2h, cs->computed[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(host_out + first, dbuf, cnt * 4, cudaMemcpyDeviceToHost, cs->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(cs->drained[k], cs->d2h);
    carry = dbuf + (cnt - 1);  // the next chunk continues from this chunk's last output
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs->d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e, "host scan");
}

int wf_compact_gt0_i32_host(const int32_t *host_in, uint64_t n, int32_t *host_out,
                            uint64_t *host_count, void *staging, size_t staging_bytes, void *ws,
                            size_t ws_bytes, wf_stream_t stream) {
  if (host_count == nullptr) return fail(WF_ERR_ARG, "host count pointer is NULL");
  int rc = host_ring_checks(host_in, host_out, n, staging, staging_bytes, size_t(6) << 20);
  if (rc) return rc;
  // [0, 256): per-slot device counts; then kRing input and kRing output buffers
  size_t buf = ((staging_bytes - 256) / (2 * kRing)) & ~size_t(255);
  if (buf > kRingChunkMax) buf = kRingChunkMax;
  const uint64_t per_chunk = buf / 4;
  rc = check_ws(WF_OP_COMPACT_GT0_I32, per_chunk, ws, ws_bytes);
  if (rc) return rc;
  auto lk = host_call_lock();
  CopyStreams *cs = nullptr;
  if ((rc = get_copy_streams(cs))) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char *base = static_cast<char *>(staging);
  uint64_t *d_counts = reinterpret_cast<uint64_t *>(base);
  auto in_buf = [&](int k) { return reinterpret_cast<int32_t *>(base + 256 + size_t(k) * buf); };
  auto out_buf = [&](int k) {
    return reinterpret_cast<int32_t *>(base + 256 + size_t(kRing + k) * buf);
  };
  cudaError_t e = cudaSuccess;
  uint64_t offset = 0;
  // chunk c-1's output is drained once its count is on the host
  auto drain = [&](uint64_t c) -> cudaError_t {
    const int k = int(c % kRing);
    cudaError_t r = cudaEventSynchronize(cs->computed[k]);
    if (r != cudaSuccess) return r;
    const uint64_t m = cs->pinned[k];
    if (m) r = cudaMemcpyAsync(host_out + offset, out_buf(k), m * 4, cudaMemcpyDeviceToHost,
                               cs->d2h);
    if (r == cudaSuccess) r = cudaEventRecord(cs->drained[k], cs->d2h);
    offset += m;
    return r;
  };
  const uint64_t nchunks = (n + per_chunk - 1) / per_chunk;
  for (uint64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    const int k = int(c % kRing);
    const uint64_t first = c * per_chunk;
    const uint64_t cnt = (n - first) < per_chunk ? (n - first) : per_chunk;
    if (c >= kRing) e = cudaStreamWaitEvent(cs->h2d, cs->computed[k], 0);  // in-slot read
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(in_buf(k), host_in + first, cnt * 4, cudaMemcpyHostToDevice, cs->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(cs->landed[k], cs->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, cs->landed[k], 0);
    if (e == cudaSuccess && c >= kRing) e = cudaStreamWaitEvent(s, cs->drained[k], 0);  // out-slot
    if (e == cudaSuccess) e = launch_compact_gt0_i32(in_buf(k), cnt, out_buf(k), d_counts + k, ws, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(cs->pinned + k, d_counts + k, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaEventRecord(cs->computed[k], s);
    if (e == cudaSuccess && c >= 1) e = drain(c - 1);
  }
  if (e == cudaSuccess && nchunks >= 1) e = drain(nchunks - 1);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs->d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) *host_count = offset;
  return cuda_status(e, "host compaction");
}

}  // extern "C"
