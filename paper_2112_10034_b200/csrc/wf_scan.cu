// wf_scan.cu — K3 scan_inclusive_i32 and K4 compact_gt0_i32 dispatch.
//
// The product kernels are the TMEM-parked, warp-specialised single-pass
// decoupled-look-back kernels of wf_scan_tmem.cu; they take any 4-byte
// aligned in/out, so there is one code path and no run-time switch.  The
// round-1 alternatives (register-tile and smem-stage kernels, the L2-streamed
// two-pass kernels) live in tools/variants/ and are compiled in only by
// variant builds (-DWF_SCAN_IMPL=1|2|3, tools/build_variants.py) for A/B runs.
//
// K3 reference analog: the CUDA SDK shfl_scan that the reference can only
// express as a lane-reversed shfl_down suffix scan (corpus.py:347-364,
// SURVEY.md §8a C3); its cross-block carries would need several launches
// through a host description (runtime/hostdesc.py:109-129).  Here the carries
// flow between tiles inside one launch through the look-back descriptors.
//
// K4 reference analog: none expressible (no ballot / atomics in the DSL,
// dsl/lexer.py:18-25); CUDA-semantics extension with the warp-aggregated
// ballot + popc idiom, made order-preserving by the tile look-back.
//
// Roofline: HBM. K3 moves 8 B/elem (read + write); K4 4 B/elem read plus
// 4 B per selected element written.
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"

namespace wf {

cudaError_t launch_scan_i32(const int32_t *in, int32_t *out, uint64_t n,
                            const int32_t *carry, void *ws, cudaStream_t s, bool early) {
  if (n == 0) return cudaSuccess;
#if WF_SCAN_IMPL == 3
  if ((((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) &&
      two_pass_usable(n))
    return launch_scan2p_i32(in, out, n, carry, ws, s);
#elif WF_SCAN_IMPL != 0
  return launch_scan_legacy_i32(WF_SCAN_IMPL, in, out, n, carry, ws, s);
#endif
  return launch_scan_tmem_i32(in, out, n, carry, ws, s, early);
}

cudaError_t launch_compact_gt0_i32(const int32_t *in, uint64_t n, int32_t *out,
                                   uint64_t *count, void *ws, cudaStream_t s, bool early) {
  if (n == 0) return cudaMemsetAsync(count, 0, sizeof(uint64_t), s);
#if WF_SCAN_IMPL == 3
  if ((reinterpret_cast<uintptr_t>(in) & 15u) == 0 && two_pass_usable(n))
    return launch_compact2p_i32(in, n, out, count, ws, s);
#elif WF_SCAN_IMPL != 0
  return launch_compact_legacy_i32(WF_SCAN_IMPL, in, n, out, count, ws, s);
#endif
  return launch_compact_tmem_i32(in, n, out, count, ws, s, early);
}

// Sharded compaction + offset exchange, fused into the TMEM kernel's last
// finisher warp.  counts3 = {count, offset, total}.  An empty shard (no tile
// to carry the exchange) runs the stand-alone exchange kernel.
cudaError_t launch_compact_gt0_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                                      uint64_t *counts3, void *ws, void *const *peers,
                                      const void *mine, uint32_t cap, int rank, int world,
                                      uint32_t epoch, uint32_t *err, cudaStream_t s, bool early) {
  PeerArgs pa{reinterpret_cast<uint64_t *const *>(peers), static_cast<const uint64_t *>(mine),
              cap, rank, world, epoch, err};
#if WF_SCAN_IMPL == 0
  if (n > 0) return launch_compact_tmem_i32_mg(in, n, out, counts3, ws, pa, s, early);
#endif
  cudaError_t e = launch_compact_gt0_i32(in, n, out, counts3, ws, s);
  if (e != cudaSuccess) return e;
  return launch_peer_exchange(kPeerExscan, counts3, 1, cap, counts3 + 1, peers, mine, rank, world,
                              epoch, err, s);
}

}  // namespace wf
