// wf_internal.h — host-side launchers shared between the kernel translation
// units and the C ABI (wf_abi.cu).  Not part of the public interface.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace wf {

// Workspace layout: a 256-byte header followed by op-specific arrays.
constexpr size_t kWsHeader = 256;
// Scan / compaction workspaces have a larger header: bytes [256, 8192) are
// reserved for the two-pass variant build's per-chunk arrival counters (16 B
// apart; tools/variants/wf_scan2p.cu) — no product kernel writes them, so a
// workspace stays valid for either build.
constexpr size_t kTileWsHeader = 8192;
constexpr size_t kChunkCnt2P = 1024;  // [256, 1024): two-pass tickets
constexpr uint32_t kMaxChunks2P = uint32_t((kTileWsHeader - kChunkCnt2P) / 16);
constexpr uint32_t kMaxChunkTiles2P = 1024;
#ifndef WF_2P_MIN_N
#define WF_2P_MIN_N (1ull << 22)
#endif
constexpr uint64_t kTwoPassMinN = WF_2P_MIN_N;
constexpr uint32_t kMaxReduceGrid = 8192;   // partial slots for reductions
constexpr int kScanBlock = 256;             // threads per scan/compact tile
constexpr int kScanVec = 4;                 // int4 loads per thread per tile
constexpr uint64_t kScanTile = uint64_t(kScanBlock) * kScanVec * 4;  // 4096
constexpr uint64_t kTmemTile = 8192;  // elements per TMEM-kernel tile (wf_scan_tmem.cu TM_TILE)
#ifndef WF_HIST_BLOCK
#define WF_HIST_BLOCK 1024
#endif
constexpr int kHistBlock = WF_HIST_BLOCK;
#ifndef WF_HIST_PRMT
#define WF_HIST_PRMT 0  // 1: 256 B bin stride, one PRMT per address (slower, wf_hist.cu)
#endif
#ifndef WF_HIST_LOP3
#define WF_HIST_LOP3 1  // 32 KiB layout, address by one 3-input LOP3 (wf_hist.cu; 0: + IADD, 646 vs 635 us)
#endif
#ifndef WF_HIST_BINW
#define WF_HIST_BINW 32  // words per bin row in the non-PRMT layout (32 or 64)
#endif
constexpr size_t kHistSmem = 256 * (WF_HIST_PRMT ? 64 : WF_HIST_BINW) * sizeof(uint32_t);

int sm_count(int device);
int set_error(int code, const char *msg);  // wf_last_error() text + return code
// load the exchange-carrying kernels on the current device (see wf_peer.cu)
cudaError_t preload_peer_kernels();
cudaError_t preload_hist_mg_kernels();
cudaError_t preload_reduce_mg_kernels();
cudaError_t preload_tmem_mg_kernels();
int current_device();

// Per-device one-time configuration: function attributes such as the
// dynamic-smem opt-in are per device, so every launcher that needs one runs
// ensure(f) before each launch; f runs once per device (idempotent, so two
// threads racing on a first call is harmless).
struct DeviceMask {
  std::atomic<uint64_t> bits{0};
  template <class F>
  void ensure(F &&f) {
    const int dev = current_device();
    if (dev < 0 || dev >= 64) {
      f();
      return;
    }
    const uint64_t b = uint64_t(1) << dev;
    if (bits.load(std::memory_order_acquire) & b) return;
    f();
    bits.fetch_or(b, std::memory_order_acq_rel);
  }
};

// reductions (wf_reduce.cu)
cudaError_t launch_reduce_i32(const int32_t *in, uint64_t n, int32_t *out,
                              int block, int grid, void *ws,
                              cudaStream_t s);
// early: programmatic dependent launch on the caller's WF_FLAG_INPUT_STABLE
// promise (wf_reduce.cu)
cudaError_t launch_reduce_f32(const float *in, uint64_t n, float *out,
                              int block, int grid, void *ws, cudaStream_t s,
                              bool early = false);
// grid for the reduce kernel of `kind` (its own occupancy x SMs, capped by n)
enum { kRedI32 = 0, kRedF32 = 1, kRedF32Mg = 2, kRedI32Px = 3 };
int auto_reduce_grid(int kind, int block, uint64_t n);
cudaError_t launch_reduce_f32_mg(const float *in, uint64_t n, float *out, int block, int grid,
                                 void *ws, void *const *peers, const void *mine, int rank,
                                 int world, uint32_t epoch, bool early, cudaStream_t s);
cudaError_t launch_reduce_i32_exscan_mg(const int32_t *in, uint64_t n, int32_t *out2, int block,
                                        int grid, void *ws, void *const *peers, const void *mine,
                                        uint32_t cap, int rank, int world, uint32_t epoch,
                                        uint32_t *err, cudaStream_t s, bool early = false);
cudaError_t launch_hist256_mg(const uint8_t *in, uint64_t n, uint64_t *bins, int grid, void *ws,
                              void *const *peers, const void *mine, uint32_t cap, int rank,
                              int world, uint32_t epoch, uint32_t *err, cudaStream_t s,
                              bool early = false);
size_t peer_mailbox_bytes(int world, uint32_t count);
cudaError_t launch_peer_exchange(int mode, const void *vals, uint32_t count, uint32_t cap,
                                 void *out, void *const *peers, const void *mine, int rank,
                                 int world, uint32_t epoch, uint32_t *err, cudaStream_t s);
cudaError_t launch_fold_f32(const float *v, uint32_t count, float *out,
                            cudaStream_t s);
cudaError_t launch_fold_i32(const int32_t *v, uint32_t count, int32_t *out,
                            cudaStream_t s);
cudaError_t launch_fold_u64(const uint64_t *v, uint32_t count, uint64_t *out,
                            cudaStream_t s);

// scan / compaction (wf_scan.cu)
// early: programmatic dependent launch on the caller's WF_FLAG_INPUT_STABLE
// promise (the round-1 variant kernels ignore it)
cudaError_t launch_scan_i32(const int32_t *in, int32_t *out, uint64_t n,
                            const int32_t *carry, void *ws, cudaStream_t s,
                            bool early = false);
cudaError_t launch_compact_gt0_i32(const int32_t *in, uint64_t n,
                                   int32_t *out, uint64_t *count, void *ws,
                                   cudaStream_t s, bool early = false);

// TMEM-parked single-pass scan / compaction (wf_scan_tmem.cu), any 4-byte
// aligned buffers — the product kernels
cudaError_t launch_scan_tmem_i32(const int32_t *in, int32_t *out, uint64_t n,
                                 const int32_t *carry, void *ws, cudaStream_t s,
                                 bool early = false);
cudaError_t launch_compact_tmem_i32(const int32_t *in, uint64_t n, int32_t *out,
                                    uint64_t *count, void *ws, cudaStream_t s,
                                    bool early = false);
struct PeerArgs;  // wf_peer.cuh
cudaError_t launch_compact_tmem_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                                       uint64_t *counts3, void *ws, const PeerArgs &pa,
                                       cudaStream_t s, bool early = false);
cudaError_t launch_scan_tmem_i32_cyclic(const int32_t *in, int32_t *out, uint64_t n, void *ws,
                                        void *const *peers, const void *mine, uint32_t cap,
                                        int rank, int world, uint32_t epoch, uint32_t *err,
                                        uint32_t round_tiles, uint32_t rounds, int max_grid,
                                        cudaStream_t s, bool early);
cudaError_t launch_compact_gt0_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                                      uint64_t *counts3, void *ws, void *const *peers,
                                      const void *mine, uint32_t cap, int rank, int world,
                                      uint32_t epoch, uint32_t *err, cudaStream_t s,
                                      bool early = false);

// Variant builds only (tools/variants/, -DWF_SCAN_IMPL != 0): the round-1
// register-tile / smem-stage kernels and the L2-streamed two-pass kernels.
#ifndef WF_SCAN_IMPL
#define WF_SCAN_IMPL 0  // 0: TMEM (product) 1: smem-stage persistent 2: register tile 3: two-pass
#endif
#if WF_SCAN_IMPL != 0
cudaError_t launch_scan_legacy_i32(int impl, const int32_t *in, int32_t *out, uint64_t n,
                                   const int32_t *carry, void *ws, cudaStream_t s);
cudaError_t launch_compact_legacy_i32(int impl, const int32_t *in, uint64_t n, int32_t *out,
                                      uint64_t *count, void *ws, cudaStream_t s);
bool two_pass_usable(uint64_t n);
cudaError_t launch_scan2p_i32(const int32_t *in, int32_t *out, uint64_t n,
                              const int32_t *carry, void *ws, cudaStream_t s);
cudaError_t launch_compact2p_i32(const int32_t *in, uint64_t n, int32_t *out,
                                 uint64_t *count, void *ws, cudaStream_t s);
#endif

// histogram (wf_hist.cu)
cudaError_t launch_hist256(const uint8_t *in, uint64_t n, uint64_t *bins,
                           bool accumulate, int grid, void *ws,
                           cudaStream_t s, bool early = false);
int auto_hist_grid(uint64_t n);
int min_hist_grid(uint64_t n);  // counter-overflow floor for a caller's grid

// warp collectives (wf_warp.cu)
// wf_patterns.cu: the reference's own DSL formulations, natively (dsl/patterns.py)
cudaError_t launch_warp_partials(bool f32, const void *a, int64_t n, void *out, int grid,
                                 int block, cudaStream_t s);
cudaError_t launch_warp_prefix32(const int32_t *a, int32_t *out, uint64_t n, cudaStream_t s);
cudaError_t launch_warp_collective(int kind, const int32_t *a,
                                   const int32_t *b, int32_t operand,
                                   int32_t *out, uint64_t n_threads, int block,
                                   int width, uint32_t mask, cudaStream_t s);

// synthetic inputs (wf_gen.cu)
cudaError_t launch_fill_synthetic(int gen, void *out, uint64_t n,
                                  uint64_t seed, uint64_t base, uint32_t param,
                                  cudaStream_t s);

}  // namespace wf
