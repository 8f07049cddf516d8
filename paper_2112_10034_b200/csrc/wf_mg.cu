// wf_mg.cu — single-process multi-GPU C ABI (wf_mg_init +
// wf_mg_<op>): one host thread drives every device of a context, each rank's
// kernel carrying its exchange over peer memory (the fused *_mg kernels of
// wf_reduce.cu / wf_scan_tmem.cu / wf_hist.cu), no NCCL and no host round
// trip inside a call.
//
// Reference anchor: the reference's only parallelism is the block-range split
// of one launch over CPU workers with join semantics (runtime/launch.py:
// 95-147, _split :137-147); a context applies that split across devices, the
// caller passing each rank's contiguous shard.
//
// Ranks may share a device (tests on a one-GPU box): their kernels then run
// concurrently on one GPU from different streams, which the fused kernels
// allow because only one block (or warp) of each spins on its peers.
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "wf_device.cuh"
#include "wf_internal.h"
#include "../../include/warpfold_b200.h"

namespace wf {
namespace {

constexpr uint32_t kMgCap = 256;  // peer-mailbox payload words (histogram bins)
constexpr int kMgOps = 6;         // workspace slots per rank, by WF_OP_* id

struct Rank {
  int dev = 0;
  cudaStream_t stream = nullptr;
  void *box_k2 = nullptr;    // wf_mailbox_alloc layout (fused K2)
  void *box_px = nullptr;    // wf_peer_mailbox_alloc layout (C3-C5 exchanges)
  void **peers_k2 = nullptr; // device array of every rank's box_k2, on this rank's device
  void **peers_px = nullptr;
  uint32_t *err = nullptr;   // sticky peer-timeout flag
  int32_t *carry = nullptr;  // scan pass 1: {carry-in, global total}
  void *ws[kMgOps + 1] = {};
  size_t ws_bytes[kMgOps + 1] = {};
};

struct DeviceGuard {  // restores the caller's current device
  int saved = 0;
  DeviceGuard() { cudaGetDevice(&saved); }
  ~DeviceGuard() { cudaSetDevice(saved); }
};

int cerr(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return WF_OK;
  cudaGetLastError();
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(int(e), m.c_str());
}

}  // namespace
}  // namespace wf

struct wf_mg {
  std::vector<wf::Rank> ranks;
  uint32_t epoch_k2 = 0, epoch_px = 0;
  std::mutex mu;  // one call at a time per context (the epoch sequences)
};

using wf::cerr;

extern "C" {

void wf_mg_destroy(wf_mg_t *ctx);

int wf_mg_init(int ngpus, const int *devs, wf_mg_t **out) {
  if (out == nullptr || devs == nullptr || ngpus < 1 || ngpus > 32)
    return wf::set_error(WF_ERR_ARG, "wf_mg_init: 1 <= ngpus <= 32 devices and an output pointer");
  *out = nullptr;
  wf::DeviceGuard guard;
  int count = 0;
  if (int rc = cerr(cudaGetDeviceCount(&count), "cudaGetDeviceCount")) return rc;
  for (int r = 0; r < ngpus; ++r)
    if (devs[r] < 0 || devs[r] >= count)
      return wf::set_error(WF_ERR_CONFIG, "wf_mg_init: device index out of range");
  auto *ctx = new wf_mg;
  ctx->ranks.resize(size_t(ngpus));
  int rc = WF_OK;
  // peer access between every pair of distinct devices (NVLink / NVSwitch)
  for (int i = 0; i < ngpus && rc == WF_OK; ++i) {
    for (int j = 0; j < ngpus && rc == WF_OK; ++j) {
      if (devs[i] == devs[j]) continue;
      int ok = 0;
      rc = cerr(cudaDeviceCanAccessPeer(&ok, devs[i], devs[j]), "cudaDeviceCanAccessPeer");
      if (rc == WF_OK && !ok) rc = wf::set_error(WF_ERR_COMM, "wf_mg_init: no peer access between two of the devices");
      if (rc == WF_OK) rc = cerr(cudaSetDevice(devs[i]), "cudaSetDevice");
      if (rc == WF_OK) {
        cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          e = cudaSuccess;
        }
        rc = cerr(e, "cudaDeviceEnablePeerAccess");
      }
    }
  }
  std::vector<void *> k2(static_cast<size_t>(ngpus)), px(static_cast<size_t>(ngpus));
  for (int r = 0; r < ngpus && rc == WF_OK; ++r) {
    wf::Rank &k = ctx->ranks[size_t(r)];
    k.dev = devs[r];
    rc = cerr(cudaSetDevice(k.dev), "cudaSetDevice");
    if (rc == WF_OK) rc = cerr(cudaStreamCreateWithFlags(&k.stream, cudaStreamNonBlocking), "stream");
    if (rc == WF_OK) rc = wf_mailbox_alloc(ngpus, &k.box_k2);
    if (rc == WF_OK) rc = wf_peer_mailbox_alloc(ngpus, wf::kMgCap, &k.box_px);
    if (rc == WF_OK) rc = cerr(cudaMalloc(&k.peers_k2, sizeof(void *) * size_t(ngpus)), "alloc");
    if (rc == WF_OK) rc = cerr(cudaMalloc(&k.peers_px, sizeof(void *) * size_t(ngpus)), "alloc");
    if (rc == WF_OK) rc = cerr(cudaMalloc(&k.err, 256), "alloc");
    if (rc == WF_OK) rc = cerr(cudaMemset(k.err, 0, 256), "memset");
    k.carry = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(k.err) + 128);
    k2[size_t(r)] = k.box_k2;
    px[size_t(r)] = k.box_px;
  }
  for (int r = 0; r < ngpus && rc == WF_OK; ++r) {
    wf::Rank &k = ctx->ranks[size_t(r)];
    rc = cerr(cudaSetDevice(k.dev), "cudaSetDevice");
    if (rc == WF_OK) rc = cerr(cudaMemcpy(k.peers_k2, k2.data(), sizeof(void *) * k2.size(),
                                          cudaMemcpyHostToDevice), "peer table");
    if (rc == WF_OK) rc = cerr(cudaMemcpy(k.peers_px, px.data(), sizeof(void *) * px.size(),
                                          cudaMemcpyHostToDevice), "peer table");
  }
  if (rc != WF_OK) {
    wf_mg_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return WF_OK;
}

int wf_mg_size(const wf_mg_t *ctx) { return ctx ? int(ctx->ranks.size()) : 0; }

void wf_mg_destroy(wf_mg_t *ctx) {
  if (ctx == nullptr) return;
  wf::DeviceGuard guard;
  for (wf::Rank &k : ctx->ranks) {
    if (cudaSetDevice(k.dev) != cudaSuccess) continue;
    if (k.stream) cudaStreamSynchronize(k.stream);
    for (void *w : k.ws) cudaFree(w);
    cudaFree(k.box_k2);
    cudaFree(k.box_px);
    cudaFree(k.peers_k2);
    cudaFree(k.peers_px);
    cudaFree(k.err);
    if (k.stream) cudaStreamDestroy(k.stream);
  }
  cudaGetLastError();
  delete ctx;
}

}  // extern "C"

namespace wf {
namespace {

// the rank's workspace for `op`, grown (and zeroed once) as needed
int rank_ws(Rank &k, int op, uint64_t n, void **ws, size_t *bytes) {
  const size_t need = wf_workspace_bytes(op, n, 256);
  if (need > k.ws_bytes[op]) {
    if (int rc = cerr(cudaStreamSynchronize(k.stream), "stream sync")) return rc;
    cudaFree(k.ws[op]);
    k.ws[op] = nullptr;
    k.ws_bytes[op] = 0;
    if (int rc = cerr(cudaMalloc(&k.ws[op], need), "workspace alloc")) return rc;
    if (int rc = cerr(cudaMemsetAsync(k.ws[op], 0, need, k.stream), "workspace zero")) return rc;
    k.ws_bytes[op] = need;
  }
  *ws = k.ws[op];
  *bytes = k.ws_bytes[op];
  return WF_OK;
}

// Workspaces of every rank for `ops` are sized BEFORE any rank's kernel is
// launched: cudaMalloc / cudaFree may synchronise the device, and a kernel
// already spinning on its peers would then wait for launches that the host
// thread can no longer issue (measured: the 4 s peer timeout).
int prepare_ws(wf_mg_t *ctx, const uint64_t *n, std::initializer_list<int> ops) {
  DeviceGuard guard;
  for (size_t r = 0; r < ctx->ranks.size(); ++r) {
    Rank &k = ctx->ranks[r];
    if (int rc = cerr(cudaSetDevice(k.dev), "cudaSetDevice")) return rc;
    for (int op : ops) {
      void *ws;
      size_t wb;
      if (int rc = rank_ws(k, op, n[r], &ws, &wb)) return rc;
    }
  }
  return WF_OK;
}

template <class F>
int each_rank(wf_mg_t *ctx, F f) {
  if (ctx == nullptr) return set_error(WF_ERR_ARG, "NULL wf_mg context");
  DeviceGuard guard;
  const int world = int(ctx->ranks.size());
  for (int r = 0; r < world; ++r) {
    Rank &k = ctx->ranks[size_t(r)];
    if (int rc = cerr(cudaSetDevice(k.dev), "cudaSetDevice")) return rc;
    if (int rc = f(r, world, k)) return rc;
  }
  return WF_OK;
}

}  // namespace
}  // namespace wf

extern "C" {

int wf_mg_reduce_sum_f32(wf_mg_t *ctx, const float *const *d_in, const uint64_t *n,
                         float *const *d_out) {
  if (ctx == nullptr || d_in == nullptr || n == nullptr || d_out == nullptr)
    return wf::set_error(WF_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (int rc = wf::prepare_ws(ctx, n, {WF_OP_REDUCE_SUM_F32})) return rc;
  const uint32_t epoch = ++ctx->epoch_k2;
  return wf::each_rank(ctx, [&](int r, int world, wf::Rank &k) {
    void *ws;
    size_t wb;
    if (int rc = wf::rank_ws(k, WF_OP_REDUCE_SUM_F32, n[r], &ws, &wb)) return rc;
    return wf_reduce_sum_f32_mg(d_in[r], n[r], d_out[r], 512, 0, ws, wb, k.peers_k2, k.box_k2, r,
                                world, epoch, k.stream);
  });
}

int wf_mg_scan_inclusive_i32(wf_mg_t *ctx, const int32_t *const *d_in, int32_t *const *d_out,
                             const uint64_t *n) {
  if (ctx == nullptr || d_in == nullptr || n == nullptr || d_out == nullptr)
    return wf::set_error(WF_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (int e = wf::prepare_ws(ctx, n, {WF_OP_REDUCE_SUM_I32, WF_OP_SCAN_INCLUSIVE_I32})) return e;
  const uint32_t epoch = ++ctx->epoch_px;
  // pass 1 + carry exchange (one fused kernel per rank), then every rank's scan
  int rc = wf::each_rank(ctx, [&](int r, int world, wf::Rank &k) {
    void *ws;
    size_t wb;
    if (int e = wf::rank_ws(k, WF_OP_REDUCE_SUM_I32, n[r], &ws, &wb)) return e;
    return wf_reduce_sum_i32_exscan_mg(d_in[r], n[r], k.carry, 256, 0, ws, wb, k.peers_px,
                                       k.box_px, wf::kMgCap, r, world, epoch, k.err, k.stream);
  });
  if (rc) return rc;
  return wf::each_rank(ctx, [&](int r, int, wf::Rank &k) {
    void *ws;
    size_t wb;
    if (int e = wf::rank_ws(k, WF_OP_SCAN_INCLUSIVE_I32, n[r], &ws, &wb)) return e;
    return wf_scan_inclusive_i32(d_in[r], d_out[r], n[r], k.carry, ws, wb, k.stream);
  });
}

int wf_mg_compact_gt0_i32(wf_mg_t *ctx, const int32_t *const *d_in, const uint64_t *n,
                          int32_t *const *d_out, uint64_t *const *d_counts3) {
  if (ctx == nullptr || d_in == nullptr || n == nullptr || d_out == nullptr || d_counts3 == nullptr)
    return wf::set_error(WF_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (int rc = wf::prepare_ws(ctx, n, {WF_OP_COMPACT_GT0_I32})) return rc;
  const uint32_t epoch = ++ctx->epoch_px;
  return wf::each_rank(ctx, [&](int r, int world, wf::Rank &k) {
    void *ws;
    size_t wb;
    if (int rc = wf::rank_ws(k, WF_OP_COMPACT_GT0_I32, n[r], &ws, &wb)) return rc;
    return wf_compact_gt0_i32_mg(d_in[r], n[r], d_out[r], d_counts3[r], ws, wb, k.peers_px,
                                 k.box_px, wf::kMgCap, r, world, epoch, k.err, k.stream);
  });
}

int wf_mg_histogram256_u8(wf_mg_t *ctx, const uint8_t *const *d_in, const uint64_t *n,
                          uint64_t *const *d_bins) {
  if (ctx == nullptr || d_in == nullptr || n == nullptr || d_bins == nullptr)
    return wf::set_error(WF_ERR_ARG, "NULL argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (int rc = wf::prepare_ws(ctx, n, {WF_OP_HISTOGRAM256_U8})) return rc;
  const uint32_t epoch = ++ctx->epoch_px;
  return wf::each_rank(ctx, [&](int r, int world, wf::Rank &k) {
    void *ws;
    size_t wb;
    if (int rc = wf::rank_ws(k, WF_OP_HISTOGRAM256_U8, n[r], &ws, &wb)) return rc;
    return wf_histogram256_u8_mg(d_in[r], n[r], d_bins[r], ws, wb, k.peers_px, k.box_px,
                                 wf::kMgCap, r, world, epoch, k.err, k.stream);
  });
}

int wf_mg_synchronize(wf_mg_t *ctx) {
  if (ctx == nullptr) return wf::set_error(WF_ERR_ARG, "NULL wf_mg context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  bool timed_out = false;
  int rc = wf::each_rank(ctx, [&](int, int, wf::Rank &k) {
    if (int e = cerr(cudaStreamSynchronize(k.stream), "rank stream")) return e;
    uint32_t flag = 0;
    if (int e = cerr(cudaMemcpy(&flag, k.err, 4, cudaMemcpyDeviceToHost), "error flag")) return e;
    timed_out |= flag != 0;
    return int(WF_OK);
  });
  if (rc) return rc;
  return timed_out ? wf::set_error(WF_ERR_COMM, "a rank's peers did not arrive within ~4 s") : WF_OK;
}

int wf_mg_stream(wf_mg_t *ctx, int rank, wf_stream_t *stream) {
  if (ctx == nullptr || stream == nullptr || rank < 0 || rank >= int(ctx->ranks.size()))
    return wf::set_error(WF_ERR_ARG, "bad context / rank");
  *stream = ctx->ranks[size_t(rank)].stream;
  return WF_OK;
}

}  // extern "C"
