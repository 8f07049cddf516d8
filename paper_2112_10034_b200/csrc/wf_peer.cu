// wf_peer.cu — small collectives over peer memory (NVLink 5 / NVSwitch) for
// the exchange steps of the sharded paths: the shard totals
// that become scan carries (C3), the compaction counts that become global
// offsets (C4) and the 256 histogram bins (C5).  Each is ONE single-block
// kernel per rank instead of an NCCL all-gather / all-reduce plus a fold
// kernel.
//
// Mailbox (per rank, mapped by every peer through CUDA IPC):
//   [bank = epoch & 1][source rank][count payload words + 1 flag word]  (u64)
// A rank stores its payload into slot [bank][rank] of every mailbox
// (st.relaxed.sys over NVLink), a release fence, then the flag = epoch; it
// then waits until every flag of its own bank carries the epoch (acquire) and
// combines the payloads in rank order (deterministic, identical on every
// rank).  Two banks suffice: a rank can be at most one call ahead of any peer
// (it cannot finish call e without every peer's call-e payload).
//
// Reference anchor: the reference's only parallelism is the block-range split
// over CPU workers joined by the launcher (runtime/launch.py:95-147).
#include "wf_device.cuh"
#include "wf_internal.h"

namespace wf {
namespace {

__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int PB = 256;

// u64 payloads (mode 3: one u32, zero-extended in the slot):
// mode 0: out[r * count + i] = vals_r[i]                       (all-gather)
// mode 1: out[0] = sum_{r < rank} vals_r[0], out[1] = sum_r vals_r[0]
//         (exclusive scan + total: compaction offsets)
// mode 2: out[i] = sum_r vals_r[i]                               (all-reduce)
// mode 3: as mode 1 on u32 values, wrapping mod 2^32, written as two u32
//         (scan carries)
// `cap` is the mailbox's payload capacity per slot (slot stride = cap + 1).
__global__ void __launch_bounds__(PB)
    peer_exchange_kernel(int mode, const void *__restrict__ vals_, uint32_t count, uint32_t cap,
                         void *__restrict__ out_, uint64_t *const *peers,
                         const uint64_t *mine, int rank, int world, uint32_t epoch,
                         uint32_t *__restrict__ err) {
  const uint64_t *vals = static_cast<const uint64_t *>(vals_);
  const uint32_t *vals32 = static_cast<const uint32_t *>(vals_);
  uint64_t *out = static_cast<uint64_t *>(out_);
  const uint32_t stride = cap + 1;
  const uint32_t bank = epoch & 1u;
  const uint64_t bank_off = uint64_t(bank) * uint32_t(world) * stride;
  // 1. payload into slot [bank][rank] of every rank's mailbox
  for (uint32_t k = threadIdx.x; k < uint32_t(world) * count; k += PB) {
    const uint32_t p = k / count, i = k % count;
    st_relaxed_sys_u64(peers[p] + bank_off + uint64_t(rank) * stride + i,
                       mode == 3 ? uint64_t(vals32[i]) : vals[i]);
  }
  __syncthreads();
  // 2. flags after a system-scope release fence (cumulative over the block's
  //    payload stores, which the barrier ordered before it)
  if (threadIdx.x < uint32_t(world)) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_relaxed_sys_u64(peers[threadIdx.x] + bank_off + uint64_t(rank) * stride + cap,
                       uint64_t(epoch));
  }
  // 3. wait for every source's flag in this rank's own mailbox
  __shared__ uint32_t s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  __syncthreads();
  if (threadIdx.x < uint32_t(world)) {
    const uint64_t *flag = mine + bank_off + uint64_t(threadIdx.x) * stride + cap;
    uint32_t spins = 0;
    while (ld_acquire_sys_u64(flag) != uint64_t(epoch)) {
      if (++spins > (1u << 25)) {  // ~4 s: a peer never arrived
        atomicExch(&s_fail, 1u);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  if (s_fail) {
    if (threadIdx.x == 0) *err = 1u;
    return;
  }
  // 4. combine in rank order
  const uint64_t *src = mine + bank_off;
  if (mode == 0) {
    for (uint32_t k = threadIdx.x; k < uint32_t(world) * count; k += PB)
      out[k] = ld_relaxed_sys_u64(src + uint64_t(k / count) * stride + k % count);
  } else if (mode == 1 || mode == 3) {
    if (threadIdx.x == 0) {
      uint64_t excl = 0, total = 0;
      for (int r = 0; r < world; ++r) {
        const uint64_t v = ld_relaxed_sys_u64(src + uint64_t(r) * stride);
        if (r < rank) excl += v;
        total += v;
      }
      if (mode == 1) {
        out[0] = excl;
        out[1] = total;
      } else {
        uint32_t *o32 = static_cast<uint32_t *>(out_);
        o32[0] = uint32_t(excl);
        o32[1] = uint32_t(total);
      }
    }
  } else {
    for (uint32_t i = threadIdx.x; i < count; i += PB) {
      uint64_t s = 0;
      for (int r = 0; r < world; ++r) s += ld_relaxed_sys_u64(src + uint64_t(r) * stride + i);
      out[i] = s;
    }
  }
}

}  // namespace

size_t peer_mailbox_bytes(int world, uint32_t count) {
  return (size_t(2) * size_t(world) * (size_t(count) + 1) * 8 + 255) & ~size_t(255);
}

cudaError_t launch_peer_exchange(int mode, const void *vals, uint32_t count, uint32_t cap,
                                 void *out, void *const *peers, const void *mine, int rank,
                                 int world, uint32_t epoch, uint32_t *err, cudaStream_t s) {
  peer_exchange_kernel<<<1, PB, 0, s>>>(mode, vals, count, cap, out,
                                        reinterpret_cast<uint64_t *const *>(peers),
                                        static_cast<const uint64_t *>(mine), rank, world, epoch,
                                        err);
  return cudaGetLastError();
}

}  // namespace wf
