// wf_peer.cuh — the block-wide peer-memory exchange shared by the
// stand-alone exchange kernel (wf_peer.cu) and the kernels that fuse it into
// their last block (K1 reduce -> scan carries, K5 histogram -> bin sums).
//
// Mailbox (per rank, mapped by every peer through CUDA IPC):
//   [bank = epoch & 1][source rank][cap payload words + 1 flag word]  (u64)
// A rank stores its payload into slot [bank][rank] of every mailbox
// (st.relaxed.sys over NVLink), a release fence, then the flag = epoch; it
// then waits until every flag of its own bank carries the epoch (acquire) and
// combines the payloads in rank order (deterministic, identical on every
// rank).  Two banks suffice: a rank can be at most one call ahead of any peer
// (it cannot finish call e without every peer's call-e payload, and a peer
// posts call e only after its call e-1 kernel has finished reading).
#pragma once

#include <cstdint>

namespace wf {

struct PeerArgs {
  uint64_t *const *peers;  // [world] mailbox of each rank (device array)
  const uint64_t *mine;    // this rank's mailbox
  uint32_t cap;            // payload words per slot
  int rank, world;
  uint32_t epoch;          // 1, 2, 3, ... (same sequence on every rank)
  uint32_t *err;           // set to 1 if a peer never arrives (~4 s)
};

// modes (include/warpfold_b200.h WF_PEER_*)
constexpr int kPeerAllgather = 0, kPeerExscan = 1, kPeerAllreduce = 2, kPeerExscanU32 = 3;

__device__ __forceinline__ void peer_st_relaxed_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t peer_ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t peer_ld_relaxed_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Every thread of the block must call this (it contains barriers).  `vals`
// (u64) or `vals32` (u32, zero-extended; mode 3) may point to global or
// shared memory.  Results (mode semantics as wf_peer_exchange):
//   0: out[r * count + i] = vals_r[i]
//   1: out[0] = sum_{r < rank} vals_r[0], out[1] = sum_r vals_r[0]   (u64)
//   2: out[i] = sum_r vals_r[i]                                       (u64)
//   3: as 1 on u32 values mod 2^32, written as two u32
// Returns false (and sets *err) if a peer did not arrive.
static __device__ __noinline__ bool peer_exchange_block(int mode, const uint64_t *vals,
                                                 const uint32_t *vals32, uint32_t count,
                                                 void *out_, const PeerArgs pa) {
  __shared__ uint32_t s_fail;
  const uint32_t nt = blockDim.x, tid = threadIdx.x;
  const uint32_t world = uint32_t(pa.world);
  const uint32_t stride = pa.cap + 1;
  const uint64_t bank_off = uint64_t(pa.epoch & 1u) * world * stride;
  const uint64_t my_slot = bank_off + uint64_t(pa.rank) * stride;
  // 1. payload into slot [bank][rank] of every rank's mailbox
  for (uint32_t k = tid; k < world * count; k += nt) {
    const uint32_t p = k / count, i = k % count;
    peer_st_relaxed_sys(pa.peers[p] + my_slot + i, vals32 ? uint64_t(vals32[i]) : vals[i]);
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  // 2. flags after a system-scope release fence (cumulative over the block's
  //    payload stores, which the barrier ordered before it)
  for (uint32_t p = tid; p < world; p += nt) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    peer_st_relaxed_sys(pa.peers[p] + my_slot + pa.cap, uint64_t(pa.epoch));
  }
  // 3. wait for every source's flag in this rank's own mailbox
  for (uint32_t p = tid; p < world; p += nt) {
    const uint64_t *flag = pa.mine + bank_off + uint64_t(p) * stride + pa.cap;
    uint32_t spins = 0;
    while (peer_ld_acquire_sys(flag) != uint64_t(pa.epoch)) {
      if (++spins > (1u << 25)) {  // ~4 s: a peer never arrived
        atomicExch(&s_fail, 1u);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) *pa.err = 1u;
    return false;
  }
  // 4. combine in rank order
  const uint64_t *src = pa.mine + bank_off;
  uint64_t *out = static_cast<uint64_t *>(out_);
  if (mode == kPeerAllgather) {
    for (uint32_t k = tid; k < world * count; k += nt)
      out[k] = peer_ld_relaxed_sys(src + uint64_t(k / count) * stride + k % count);
  } else if (mode == kPeerExscan || mode == kPeerExscanU32) {
    if (tid == 0) {
      uint64_t excl = 0, total = 0;
      for (uint32_t r = 0; r < world; ++r) {
        const uint64_t v = peer_ld_relaxed_sys(src + uint64_t(r) * stride);
        if (int(r) < pa.rank) excl += v;
        total += v;
      }
      if (mode == kPeerExscan) {
        out[0] = excl;
        out[1] = total;
      } else {
        uint32_t *o32 = static_cast<uint32_t *>(out_);
        o32[0] = uint32_t(excl);
        o32[1] = uint32_t(total);
      }
    }
  } else {
    for (uint32_t i = tid; i < count; i += nt) {
      uint64_t s = 0;
      for (uint32_t r = 0; r < world; ++r) s += peer_ld_relaxed_sys(src + uint64_t(r) * stride + i);
      out[i] = s;
    }
  }
  return true;
}

// One warp's form of mode 1 (exclusive scan + total of one u64 per rank),
// for kernels where only one warp holds the value when it becomes known (the
// compaction's last finisher warp).  Lane p handles peer p (p, p+32, ...):
// payload store, release fence, flag store — per-thread program order, so no
// barrier cumulativity is needed.  out2 = {sum_{r<rank} v_r, sum_r v_r}.
static __device__ __noinline__ bool peer_exscan_warp(uint64_t v, uint64_t *out2,
                                                     const PeerArgs pa) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t world = uint32_t(pa.world);
  const uint32_t stride = pa.cap + 1;
  const uint64_t bank_off = uint64_t(pa.epoch & 1u) * world * stride;
  const uint64_t my_slot = bank_off + uint64_t(pa.rank) * stride;
  for (uint32_t p = lane; p < world; p += 32) {
    peer_st_relaxed_sys(pa.peers[p] + my_slot, v);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    peer_st_relaxed_sys(pa.peers[p] + my_slot + pa.cap, uint64_t(pa.epoch));
  }
  bool fail = false;
  uint64_t excl = 0, total = 0;
  for (uint32_t p = lane; p < world; p += 32) {
    const uint64_t *slot = pa.mine + bank_off + uint64_t(p) * stride;
    uint32_t spins = 0;
    while (peer_ld_acquire_sys(slot + pa.cap) != uint64_t(pa.epoch)) {
      if (++spins > (1u << 25)) {  // ~4 s: a peer never arrived
        fail = true;
        break;
      }
      __nanosleep(128);
    }
    const uint64_t x = fail ? 0 : peer_ld_relaxed_sys(slot);
    if (int(p) < pa.rank) excl += x;
    total += x;
  }
  if (__any_sync(0xffffffffu, fail)) {
    if (lane == 0) *pa.err = 1u;
    return false;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    excl += __shfl_xor_sync(0xffffffffu, excl, o);
    total += __shfl_xor_sync(0xffffffffu, total, o);
  }
  if (lane == 0) {
    out2[0] = excl;
    out2[1] = total;
  }
  return true;
}

}  // namespace wf
