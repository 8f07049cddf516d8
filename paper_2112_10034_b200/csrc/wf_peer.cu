// wf_peer.cu — the stand-alone form of the peer-memory exchange (NVLink 5 /
// NVSwitch) of the sharded paths: ONE single-block kernel
// per rank instead of an NCCL all-gather / all-reduce plus a fold kernel.
// The default paths run the same exchange inside the producing kernel
// (K1 -> scan carries, K4 -> compaction offsets, K5 -> bins); this kernel
// serves any other value and the non-default compaction kernels.
//
// The protocol (mailbox layout, banks, fences) lives in wf_peer.cuh, shared
// with the kernels that run the same exchange in their last block
// (wf_reduce.cu: reduce + scan-carry exchange, wf_hist.cu: bins + all-reduce).
//
// Reference anchor: the reference's only parallelism is the block-range split
// over CPU workers joined by the launcher (runtime/launch.py:95-147).
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"

namespace wf {
namespace {

constexpr int PB = 256;

__global__ void __launch_bounds__(PB)
    peer_exchange_kernel(int mode, const void *__restrict__ vals, uint32_t count, void *out,
                         PeerArgs pa) {
  peer_exchange_block(mode, mode == kPeerExscanU32 ? nullptr : static_cast<const uint64_t *>(vals),
                      mode == kPeerExscanU32 ? static_cast<const uint32_t *>(vals) : nullptr,
                      count, out, pa);
}

}  // namespace

size_t peer_mailbox_bytes(int world, uint32_t count) {
  return (size_t(2) * size_t(world) * (size_t(count) + 1) * 8 + 255) & ~size_t(255);
}

cudaError_t launch_peer_exchange(int mode, const void *vals, uint32_t count, uint32_t cap,
                                 void *out, void *const *peers, const void *mine, int rank,
                                 int world, uint32_t epoch, uint32_t *err, cudaStream_t s) {
  PeerArgs pa{reinterpret_cast<uint64_t *const *>(peers), static_cast<const uint64_t *>(mine),
              cap, rank, world, epoch, err};
  peer_exchange_kernel<<<1, PB, 0, s>>>(mode, vals, count, out, pa);
  return cudaGetLastError();
}

// Loads the exchange kernel's module on the current device now: with lazy
// module loading a first launch can wait for the device to go idle, which a
// peer already spinning on this exchange never lets happen (wf_mg / ranks
// sharing a device).
cudaError_t preload_peer_kernels() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, peer_exchange_kernel);
}

}  // namespace wf
