// wf_device.cuh — device helpers shared by the sm_100a kernels.
//
// Everything here maps 1:1 onto a SASS instruction class that the reference
// emulates in Python: SHFL (passes/warp_lower.py:36-45), VOTE
// (passes/warp_lower.py:17-33), REDUX.SUM, and the lane/warp indices the
// collapsing pass materialises as __tx / __wid loop variables
// (passes/wrap.py:136-147).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wf {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// 128-bit streaming load: read-only path, no L1 allocation (pure stream, no
// reuse), 256-byte L2 prefetch so each warp-load pulls whole DRAM bursts.
__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

// 128-bit streaming store (evict-first: output is not re-read by the kernel).
__device__ __forceinline__ void stg_stream(uint4 *p, const uint4 &v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];"
               : "=l"(v)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v)
               : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  return *reinterpret_cast<const volatile uint32_t *>(p);
}

// ---- splitmix64 index hash: the synthetic-input contract --
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---- decoupled look-back tile descriptors ------------------------------
// One 64-bit word per tile: [epoch:30][status:2][value:32].  The epoch is
// bumped by the last CTA of every launch, so stale descriptors of earlier
// launches read as "not yet published" and the descriptor array never needs
// clearing between launches.
enum : uint32_t { kStInvalid = 0, kStAggregate = 1, kStPrefix = 2 };
constexpr uint32_t kEpochMask = (1u << 30) - 1;

__device__ __forceinline__ uint64_t pack_desc(uint32_t epoch, uint32_t st,
                                              uint32_t value) {
  return (uint64_t(epoch & kEpochMask) << 34) | (uint64_t(st) << 32) |
         uint64_t(value);
}

// Workspace header of the look-back kernels (first 256 bytes of the ws).
struct TileHeader {
  uint32_t ticket;  // dynamic tile-id counter, reset by the last CTA
  uint32_t epoch;   // launch epoch, bumped by the last CTA
};

// Thread 0 of every CTA: read the epoch, then take a ticket.  The CTA that
// draws the last ticket knows every CTA has already read the epoch, so it can
// reset the counter and bump the epoch for the next stream-ordered launch.
__device__ __forceinline__ void take_ticket(TileHeader *hdr, uint32_t ntiles,
                                            uint32_t &tile, uint32_t &epoch) {
  epoch = ld_volatile_u32(&hdr->epoch) & kEpochMask;
  __threadfence();
  tile = atomicAdd(&hdr->ticket, 1u);
  if (tile == ntiles - 1) {
    atomicExch(&hdr->ticket, 0u);
    atomicExch(&hdr->epoch, (epoch + 1) & kEpochMask);
  }
}

// Warp-parallel decoupled look-back (called by all 32 lanes of one warp).
// Returns the exclusive prefix (wrapping uint32 sum) of all tiles < `tile`.
// Each lane inspects one predecessor; the window slides back 32 tiles at a
// time until a tile with an inclusive prefix is found.
__device__ __forceinline__ uint32_t lookback_exclusive(const uint64_t *desc,
                                                       uint32_t tile,
                                                       uint32_t epoch) {
  const uint32_t lane = lane_id();
  uint32_t excl = 0;
  int64_t pred_base = int64_t(tile) - 1;
  while (true) {
    const int64_t p = pred_base - int64_t(lane);
    uint32_t st, val;
    while (true) {
      if (p >= 0) {
        const uint64_t d = ld_relaxed_gpu(desc + p);
        const bool live = uint32_t(d >> 34) == epoch;
        st = live ? uint32_t(d >> 32) & 3u : kStInvalid;
        val = uint32_t(d);
      } else {
        st = kStPrefix;  // virtual tile before tile 0 contributes nothing
        val = 0;
      }
      if (__all_sync(kFull, st != kStInvalid)) break;
      __nanosleep(32);
    }
    const uint32_t prefix_lanes = __ballot_sync(kFull, st == kStPrefix);
    if (prefix_lanes) {
      const uint32_t first = __ffs(prefix_lanes) - 1;  // nearest prefix tile
      excl += __reduce_add_sync(kFull, lane <= first ? val : 0u);
      return excl;
    }
    excl += __reduce_add_sync(kFull, val);
    pred_base -= 32;
  }
}

}  // namespace wf
