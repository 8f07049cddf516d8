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

// 128-bit load marking the line evict_last in L2 (cache-policy form): for
// data the next kernel re-reads (the sharded scan's pass 1).
__device__ __forceinline__ uint4 ldg_keep(const uint4 *p) {
  uint4 r;
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

// 128-bit load marking the line evict_first in L2: read once, never again.
__device__ __forceinline__ uint4 ldg_evict_first(const uint4 *p) {
  uint4 r;
  asm volatile(
      "{\n\t.reg .b64 pol;\n\t"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], pol;\n\t}"
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

// Release/acquire ticket: orders this thread's earlier global writes (and
// reductions) before the increment, and makes every earlier increment's
// writes visible to the thread that draws the last ticket.  Cheaper than a
// full __threadfence() (MEMBAR.SC) on the critical path of the last block.
__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Relaxed ticket draw: no fence, so it does not wait for this thread's
// outstanding stores to be acknowledged (a release draw right after a tile's
// output stores costs microseconds under full HBM load).
__device__ __forceinline__ uint32_t atom_add_relaxed_gpu(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// 64-bit relaxed draw on a TileHeader read as one word {epoch:32 | ticket:32}
// (little-endian: ticket in the low half): returns the launch's epoch with
// the ticket in ONE L2 round trip (wf_scan_tmem.cu).
__device__ __forceinline__ uint64_t atom_add_relaxed_gpu_u64(uint64_t *p, uint64_t v) {
  uint64_t old;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ void red_add_relaxed_gpu(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  return *reinterpret_cast<const volatile uint32_t *>(p);
}

// ---- splitmix64 index hash: the synthetic-input contract --
// CTA-scope release store / acquire load on shared memory: publish a flag
// after plain shared stores it guards (PTX memory model, not store order).
__device__ __forceinline__ void st_release_cta_smem(uint32_t *p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(p))),
               "r"(v)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta_smem(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p)))
               : "memory");
  return v;
}

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
#ifndef WF_DSTRIDE
#define WF_DSTRIDE 16  // descriptor stride in 8-byte words (16 = one per 128-byte line)
#endif
constexpr int kDescStride = WF_DSTRIDE;
constexpr uint32_t kEpochMask = (1u << 30) - 1;

__device__ __forceinline__ uint64_t pack_desc(uint32_t epoch, uint32_t st,
                                              uint32_t value) {
  return (uint64_t(epoch & kEpochMask) << 34) | (uint64_t(st) << 32) |
         uint64_t(value);
}

// Workspace header of the look-back kernels (first 256 bytes of the ws).
struct alignas(8) TileHeader {
  uint32_t ticket;  // dynamic tile-id counter, reset by the last CTA
  uint32_t epoch;   // launch epoch, bumped by the last CTA
};
static_assert(sizeof(TileHeader) == 8, "TileHeader is one 64-bit word {epoch, ticket}");

// (Round-1 variant kernels, tools/variants/; the product TMEM kernel draws
// ticket and epoch in one 64-bit atomic instead.)
// Thread 0 of every CTA: read the epoch, then take a ticket.  The CTA that
// draws the last ticket knows every CTA has already read the epoch, so it can
// reset the counter and bump the epoch for the next stream-ordered launch.
__device__ __forceinline__ void take_ticket(TileHeader *hdr, uint32_t ntiles,
                                            uint32_t &tile, uint32_t &epoch) {
  epoch = ld_volatile_u32(&hdr->epoch) & kEpochMask;
  tile = atom_add_acq_rel_gpu(&hdr->ticket, 1u);  // release orders the epoch read first
  if (tile == ntiles - 1) {
    atomicExch(&hdr->ticket, 0u);
    atomicExch(&hdr->epoch, (epoch + 1) & kEpochMask);
  }
}

// Wide look-back: lane l inspects the K predecessors tile-1-K*l-k (k = 0..K-1),
// so one round trip to L2 covers 32*K tiles and the prefix frontier advances
// up to 32*K tiles per round trip instead of 32.  Descriptors already seen
// valid are kept (an aggregate never changes), only not-yet-published ones
// are re-polled, and the window resolves as soon as every tile nearer than
// the nearest inclusive prefix is valid — so polling traffic stays small.
template <int K>
__device__ __forceinline__ uint32_t lookback_exclusive_wide(const uint64_t *desc,
                                                            uint32_t tile, uint32_t epoch,
                                                            uint32_t *polls = nullptr) {
  const uint32_t lane = lane_id();
  uint32_t excl = 0;
  int64_t hi = int64_t(tile) - 1;
  while (true) {
    uint32_t st[K], val[K];
#pragma unroll
    for (int k = 0; k < K; ++k) st[k] = kStInvalid;
    uint32_t backoff = 16;
    while (true) {
      if (polls) ++*polls;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (st[k] == kStInvalid) {
          const int64_t p = hi - int64_t(lane) * K - k;
          if (p >= 0) {
            const uint64_t d = ld_relaxed_gpu(desc + p * kDescStride);
            st[k] = uint32_t(d >> 34) == epoch ? uint32_t(d >> 32) & 3u : kStInvalid;
            val[k] = uint32_t(d);
          } else {
            st[k] = kStPrefix;
            val[k] = 0;
          }
        }
      }
      int kp = K, ki = K;  // nearest prefix / nearest invalid in this lane's run
#pragma unroll
      for (int k = K - 1; k >= 0; --k) {
        if (st[k] == kStPrefix) kp = k;
        if (st[k] == kStInvalid) ki = k;
      }
      const uint32_t lp = __ballot_sync(kFull, kp < K);
      const uint32_t li = __ballot_sync(kFull, ki < K);
      const uint32_t pos_p = lp ? (__ffs(lp) - 1) * K + __shfl_sync(kFull, kp, __ffs(lp) - 1) : ~0u;
      const uint32_t pos_i = li ? (__ffs(li) - 1) * K + __shfl_sync(kFull, ki, __ffs(li) - 1) : ~0u;
      if (lp && pos_p < pos_i) {  // resolved: everything nearer than the prefix is valid
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (lane * K + k <= pos_p) c += val[k];
        excl += __reduce_add_sync(kFull, c);
        return excl;
      }
      if (!li) break;  // all aggregates, no prefix: slide the window
#ifndef WF_BACKOFF_MAX
#define WF_BACKOFF_MAX 256
#endif
      if (WF_BACKOFF_MAX > 0) __nanosleep(backoff);
      backoff = backoff < WF_BACKOFF_MAX ? backoff * 2 : WF_BACKOFF_MAX;
    }
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) run += val[k];
    excl += __reduce_add_sync(kFull, run);
    hi -= 32 * K;
  }
}

}  // namespace wf

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a async proxy) ------------
namespace wf {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// make barrier initialisation visible to the async proxy (TMA unit)
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 1-D bulk copy global -> shared, completion reported on `bar` (UBLKCP)
#ifndef WF_TMA_EVICT_FIRST
#define WF_TMA_EVICT_FIRST 0  // 1: streamed tiles marked evict-first in L2
#endif
__device__ __forceinline__ void tma_load_1d(void *dst_smem, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
#if WF_TMA_EVICT_FIRST
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
#endif
}

// 1-D bulk copy shared -> global, tracked by bulk groups
__device__ __forceinline__ void tma_store_1d(void *dst, const void *src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// wait until every committed bulk store has finished READING shared memory
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// wait until every committed bulk store has fully completed
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// generic-proxy smem writes -> visible to the async proxy (before a TMA store)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace wf
