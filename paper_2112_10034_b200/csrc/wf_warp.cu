// wf_warp.cu — P: warp collectives with the reference's semantics, run as
// native SHFL / VOTE / REDUX instead of lane-buffer loops.
//
// Reference: passes/warp_lower.py:36-45 (shuffle_down: own value when the
// source lane is out of range), passes/warp_lower.py:17-33 (reduce_vote ->
// i32 0/1), interp/oracle.py:147-161 (_resolve_collective over the lanes of
// one warp).  The reference lowers every collective to
//   buf[lane] = v ; RAW warp barrier ; read ; WAR warp barrier
// executed as two W-iteration lane loops (passes/warp_lower.py:52-88); here
// it is one SHFL.IDX / VOTE.ANY / REDUX instruction.
//
// Raw __shfl_down_sync only honours the low 5 bits of the offset, so offsets
// < 0 or >= 33 would differ from the reference clamp; the source lane is
// therefore computed explicitly and the exchange is a single SHFL.IDX
// (SURVEY.md Appendix B.1).
//
// Extensions (no reference pin; CUDA semantics):
// non-full masks, partial warps (block % 32 != 0), sub-warp widths, shfl_up /
// shfl_xor / shfl_idx, ballot and REDUX add.  A source lane that does not
// participate (outside the mask or beyond the partial warp) yields the
// reader's own value.
#include "wf_device.cuh"
#include "wf_internal.h"
#include "../../include/warpfold_b200.h"

namespace wf {
namespace {

__global__ void warp_collective_kernel(int kind, const int32_t *__restrict__ a,
                                       const int32_t *__restrict__ b,
                                       int32_t operand, int32_t *__restrict__ out,
                                       uint32_t width, uint32_t mask) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp_first = threadIdx.x & ~31u;
  const uint32_t present_n = min(32u, blockDim.x - warp_first);
  const uint32_t present = present_n == 32 ? kFull : ((1u << present_n) - 1u);
  const uint32_t part = mask & present;
  if (!((part >> lane) & 1u)) return;  // not a caller of the collective

  const uint32_t seg = lane & ~(width - 1u);
  const uint32_t segbits = width == 32 ? kFull : ((1u << width) - 1u) << seg;
  const uint32_t seg_part = part & segbits;
  const int32_t l = int32_t(lane - seg);
  const int32_t v = a[i];
  const int32_t o = b ? b[i] : operand;

  // source lane (absolute) for the shuffles; own lane when out of range
  auto pick = [&](int64_t src_in_seg) -> uint32_t {
    if (src_in_seg < 0 || src_in_seg >= int64_t(width)) return lane;
    const uint32_t s = seg + uint32_t(src_in_seg);
    return ((seg_part >> s) & 1u) ? s : lane;
  };

  int32_t r;
  switch (kind) {
    case WF_COLL_SHFL_DOWN:
      r = __shfl_sync(part, v, pick(int64_t(l) + o));
      break;
    case WF_COLL_SHFL_UP:
      r = __shfl_sync(part, v, pick(int64_t(l) - o));
      break;
    case WF_COLL_SHFL_XOR:
      r = __shfl_sync(part, v, pick(int64_t(uint32_t(l) ^ uint32_t(o))));
      break;
    case WF_COLL_SHFL_IDX: {
      int64_t s = int64_t(o) % int64_t(width);
      if (s < 0) s += width;
      r = __shfl_sync(part, v, pick(s));
      break;
    }
    case WF_COLL_VOTE_ALL: {
      const uint32_t bal = __ballot_sync(part, v != 0) & seg_part;
      r = bal == seg_part ? 1 : 0;
      break;
    }
    case WF_COLL_VOTE_ANY: {
      const uint32_t bal = __ballot_sync(part, v != 0) & seg_part;
      r = bal != 0 ? 1 : 0;
      break;
    }
    case WF_COLL_BALLOT: {
      const uint32_t bal = __ballot_sync(part, v != 0) & seg_part;
      r = int32_t(bal >> seg);
      break;
    }
    case WF_COLL_REDUCE_ADD: {
      if (width == 32) {
        r = int32_t(__reduce_add_sync(part, uint32_t(v)));  // REDUX.SUM
      } else {
        uint32_t acc = 0;
        for (uint32_t j = 0; j < width; ++j) {
          const uint32_t s = seg + j;
          const bool ok = (seg_part >> s) & 1u;
          const uint32_t t = __shfl_sync(part, uint32_t(v), ok ? s : lane);
          acc += ok ? t : 0u;
        }
        r = int32_t(acc);
      }
      break;
    }
    default:
      r = v;
  }
  out[i] = r;
}

}  // namespace

cudaError_t launch_warp_collective(int kind, const int32_t *a, const int32_t *b,
                                   int32_t operand, int32_t *out,
                                   uint64_t n_threads, int block, int width,
                                   uint32_t mask, cudaStream_t s) {
  if (n_threads == 0) return cudaSuccess;
  const uint64_t grid = n_threads / uint64_t(block);
  warp_collective_kernel<<<dim3(uint32_t(grid)), block, 0, s>>>(kind, a, b, operand, out,
                                                                 uint32_t(width), mask);
  return cudaGetLastError();
}

}  // namespace wf
