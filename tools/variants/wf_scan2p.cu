// wf_scan2p.cu — K3 scan / K4 compaction, L2-streamed two-pass variant.
//
// Why a second design next to the single-pass decoupled look-back of
// wf_scan.cu: per-tile traces (profiles/r01_scan_compact_experiments.md)
// showed the single-pass kernels are limited by how long each 32 KiB smem
// stage is parked waiting for its prefix (~3 us after the LAST predecessor
// landed), which caps the reads in flight at ~3 TB/s (Little's law).  Here no
// tile ever waits for a predecessor while holding HBM bandwidth hostage:
//
//   P1 (tile t): stream the tile from HBM (loads tagged L2::evict_last so it
//     stays in the 126 MB L2) and publish one value per tile (sum for the
//     scan, number of x > 0 for compaction);
//   the LAST P1 tile of chunk c (per-chunk arrival counter) scans the chunk's
//     tile values, resolves the chunk base by a decoupled look-back over CHUNK
//     descriptors (one per C tiles, so the chain never serialises), writes
//     absolute tile offsets and marks the chunk ready;
//   P2 (tile t): re-read the tile from L2, scan / compact it locally while
//     the offset is fetched, write it out.
//
// Scheduling: two tickets (P1 tile ids, P2 tile ids) and a per-CTA choice:
// run a claimed P2 tile as soon as its chunk is ready, otherwise claim P1
// work (bounded lead so the live set fits L2).  Thread 0 prefetches the next
// claims while the current tile's loads are in flight.  Every wait is for
// work already claimed by a running CTA that never blocks on later work, so
// the scheme cannot deadlock at any residency.
// DRAM traffic stays algorithmic (8 B/elem scan, 4 + 4p B/elem compaction)
// as long as the live set fits L2 (ncu: dram__bytes_read = 1.09 GB for 2^28
// with 8-16 MiB chunks).
//
// Measured outcome (2^28 int32, B200): NOT faster than the single-pass
// kernels — best 432 us scan / 411 us compaction vs 378 / 337.  P2 can only
// run once every P1 tile of its chunk has landed, so P1 must lead by at least
// the bytes in flight (~BW x item latency ~ 20-33 MB at 6.5 TB/s), and the
// L2 must hold lead + chunk + dirty output (~2x that): more than the ~50-60 MB
// that survived in practice, so either P2 waits (small lead) or P2 misses L2
// and DRAM reads double (large lead).  Kept as an opt-in, parity-tested
// variant (WF_SCAN_2P=1) for that evidence.
//
// Reference analog: the reference can only express the scan warp-level
// (corpus.py:347-364) and needs several launches for block carries
// (runtime/hostdesc.py:109-129); compaction is not expressible
// (dsl/lexer.py:18-25).  Semantics (uint32 wrap scan, ordered a[a>0]) are the
// oracle's (oracle/numpy_oracle.py).
#include "wf_device.cuh"
#include "wf_internal.h"

#include <cstdlib>

#ifndef WF_2P_BLOCK
#define WF_2P_BLOCK 256
#endif
#ifndef WF_2P_VEC
#define WF_2P_VEC 8  // 128-item chunks per warp per tile (tile = BLOCK * VEC * 4 items)
#endif
#ifndef WF_2P_CHUNK
#define WF_2P_CHUNK 128  // tiles per chunk (finisher granularity)
#endif
#ifndef WF_2P_LEAD
#define WF_2P_LEAD 768  // max P1 tiles claimed ahead of the P2 ticket
#endif
#ifndef WF_2P_MINB
#define WF_2P_MINB 4  // __launch_bounds__ min CTAs per SM
#endif
#ifndef WF_2P_P1POL
#define WF_2P_P1POL 1  // 1: P1 loads L2::evict_last
#endif
#ifndef WF_2P_P2POL
#define WF_2P_P2POL 1  // 1: P2 loads L2::evict_first
#endif
#ifndef WF_2P_CLAIM_GAP
#define WF_2P_CLAIM_GAP 128  // claim P2 work once our P1 claims are this far past it
#endif
#ifndef WF_2P_STATS
#define WF_2P_STATS 0
#endif

namespace wf {
#if WF_2P_STATS
// [0] P2 wait ns  [1] chunk look-back ns  [2] finisher ns  [3] P2 items that
// waited  [4] P1 items  [5] P2 items  [6] CTA lifetime ns  [7] lead-bounded claims
__device__ unsigned long long g_2p_stats[8];
__device__ __forceinline__ unsigned long long gt2() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WF_2P_ADD(i, v) atomicAdd(&g_2p_stats[i], (unsigned long long)(v))
#else
#define WF_2P_ADD(i, v)
#endif
namespace {

constexpr int B2 = WF_2P_BLOCK;
constexpr int NW2 = B2 / 32;
constexpr int V2 = WF_2P_VEC;
constexpr uint32_t TILE2 = uint32_t(B2) * V2 * 4;
constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kExit = 0xfffffffeu;
constexpr uint32_t kP2Bit = 0x80000000u;

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int POL>
__device__ __forceinline__ uint4 ldg_pol(const uint4 *p, uint64_t pol) {
  uint4 r;
  if (POL) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p), "l"(pol));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  }
  return r;
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool is_prefix(uint64_t d, uint32_t epoch) {
  return uint32_t(d >> 34) == epoch && ((uint32_t(d >> 32) & 3u) == kStPrefix);
}

// Workspace of the two-pass kernels (header rule in wf_internal.h):
//   header bytes 256 / 384 / 512: P1 ticket, P2 ticket, exit counter
//   header [kChunkCnt2P, 8192): per-chunk arrival counters, 16 B apart
//   body: tile_val[T], tile_off[T], then one 128 B line per chunk descriptor
struct Layout2P {
  uint32_t *p1, *p2, *exits;
  uint32_t *chunk_cnt;
  uint32_t *tile_val;
  uint32_t *tile_off;
  uint64_t *chunk_desc;
};

__device__ __forceinline__ Layout2P layout2p(void *ws, uint32_t T) {
  Layout2P L;
  char *base = static_cast<char *>(ws);
  L.p1 = reinterpret_cast<uint32_t *>(base + 256);
  L.p2 = reinterpret_cast<uint32_t *>(base + 384);
  L.exits = reinterpret_cast<uint32_t *>(base + 512);
  L.chunk_cnt = reinterpret_cast<uint32_t *>(base + kChunkCnt2P);
  char *r = base + kTileWsHeader;
  L.tile_val = reinterpret_cast<uint32_t *>(r);
  L.tile_off = L.tile_val + T;
  const size_t off = (size_t(T) * 8 + 127) & ~size_t(127);
  L.chunk_desc = reinterpret_cast<uint64_t *>(r + off);
  return L;
}

struct Shared2P {
  uint32_t item;    // tile id | kP2Bit, or kExit
  uint32_t offset;  // P2: tile offset
  uint32_t last;    // P1: this CTA finishes the chunk
  uint32_t base;
  uint32_t epoch;
  uint32_t wtot[NW2];
};

// Thread-0 scheduler state (meaningful in thread 0 only).
struct Sched {
  uint32_t next1 = kNone;  // prefetched P1 tile
  uint32_t pend = kNone;   // claimed P2 tile not yet run
  uint32_t last1 = 0;      // highest P1 tile claimed by this CTA
  uint32_t hint2 = 0;      // lower bound of the global P2 ticket
  bool p1_done = false, p2_done = false;
};

template <int POLI>
__device__ __forceinline__ void load_tile2(const int32_t *__restrict__ in, uint64_t n,
                                           uint64_t base, bool full, uint64_t pol,
                                           uint32_t (&x)[V2][4]) {
  if (full) {
#pragma unroll
    for (int j = 0; j < V2; ++j) {
      const uint4 q = ldg_pol<POLI>(reinterpret_cast<const uint4 *>(in + base + j * 128), pol);
      x[j][0] = q.x; x[j][1] = q.y; x[j][2] = q.z; x[j][3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < V2; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t idx = base + j * 128 + k;
        x[j][k] = idx < n ? uint32_t(in[idx]) : 0u;
      }
  }
}

// Pick the next item (thread 0).  Preference: a pending P2 tile whose chunk is
// ready, the prefetched P1 tile, then waiting for a pending (or freshly
// claimed) P2 tile — but only once every P1 tile of its chunk has been
// claimed; otherwise claim P1 work first.  So a CTA blocks only on chunks
// whose P1 tiles are all held by CTAs that are running them.
__device__ __forceinline__ uint32_t pick(Sched &S, const Layout2P &L, uint32_t T, uint32_t C,
                                         uint32_t epoch) {
  if (S.pend != kNone &&
      is_prefix(ld_acquire_u64(L.chunk_desc + uint64_t(S.pend / C) * kDescStride), epoch)) {
    const uint32_t t = S.pend;
    S.pend = kNone;
    return t | kP2Bit;
  }
  if (S.next1 != kNone) {
    const uint32_t t = S.next1;
    S.next1 = kNone;
    return t;
  }
  if (S.pend == kNone && !S.p2_done) {
    const uint32_t t = atom_add_relaxed_gpu(L.p2, 1u);
    if (t < T) {
      S.pend = t;
      S.hint2 = t + 1;
    } else {
      S.p2_done = true;
    }
  }
  if (S.pend != kNone) {
    const uint32_t chunk_end = min((S.pend / C + 1) * C, T);
    if (S.p1_done || ld_relaxed_u32(L.p1) >= chunk_end) {
      const uint32_t t = S.pend;
      S.pend = kNone;
      return t | kP2Bit;
    }
  }
  if (!S.p1_done) {
    const uint32_t t = atom_add_relaxed_gpu(L.p1, 1u);
    if (t < T) {
      S.last1 = t;
      return t;
    }
    S.p1_done = true;
  }
  if (S.pend != kNone) {  // every P1 tile is claimed now
    const uint32_t t = S.pend;
    S.pend = kNone;
    return t | kP2Bit;
  }
  return kExit;
}

// Prefetch claims for the next pick (thread 0, while this item's loads fly).
__device__ __forceinline__ void prefetch(Sched &S, const Layout2P &L, uint32_t T, uint32_t lead) {
  if (S.pend == kNone && !S.p2_done && (S.p1_done || S.last1 >= S.hint2 + WF_2P_CLAIM_GAP)) {
    const uint32_t t = atom_add_relaxed_gpu(L.p2, 1u);
    if (t < T) {
      S.pend = t;
      S.hint2 = t + 1;
    } else {
      S.p2_done = true;
    }
  }
  if (S.next1 == kNone && !S.p1_done) {
    if (S.last1 < S.hint2 + lead) {
      const uint32_t t = atom_add_relaxed_gpu(L.p1, 1u);
      if (t < T) {
        S.next1 = t;
        S.last1 = t;
      } else {
        S.p1_done = true;
      }
    } else {
      WF_2P_ADD(7, 1);
    }
  }
}

template <bool COMPACT>
__global__ void __launch_bounds__(B2, WF_2P_MINB)
    two_pass_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out, uint64_t n,
                    uint32_t T, uint32_t C, uint32_t K, uint32_t lead,
                    const int32_t *__restrict__ carry_in, uint64_t *__restrict__ count,
                    void *ws) {
  __shared__ Shared2P sh;
#if WF_2P_STATS
  const unsigned long long life0 = gt2();
#endif
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  const Layout2P L = layout2p(ws, T);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pol_p1 = policy_evict_last();
  const uint64_t pol_p2 = policy_evict_first();
  Sched S;

  if (threadIdx.x == 0) {
    sh.epoch = ld_volatile_u32(&hdr->epoch) & kEpochMask;
    // the first claim is a release: it orders the epoch read before it, so the
    // last exiting CTA's epoch bump cannot overtake any CTA's epoch read
    const uint32_t t = atom_add_acq_rel_gpu(L.p1, 1u);
    if (t < T) {
      S.next1 = t;
      S.last1 = t;
    } else {
      S.p1_done = true;
    }
    sh.item = pick(S, L, T, C, sh.epoch);
  }
  __syncthreads();
  const uint32_t epoch = sh.epoch;

  while (true) {
    const uint32_t item = sh.item;
    if (item == kExit) break;
    const bool p2 = (item & kP2Bit) != 0;
    const uint32_t tile = item & ~kP2Bit;
    const uint32_t c = tile / C;
    const uint64_t base = uint64_t(tile) * TILE2 + uint64_t(warp) * (V2 * 128) + lane * 4;
    const bool full = uint64_t(tile + 1) * TILE2 <= n;
    uint32_t x[V2][4];
    if (p2)
      load_tile2<WF_2P_P2POL>(in, n, base, full, pol_p2, x);
    else
      load_tile2<WF_2P_P1POL>(in, n, base, full, pol_p1, x);
    if (threadIdx.x == 0) prefetch(S, L, T, lead);

    if (!p2) {
      // ---------------- P1: tile value, chunk arrival ----------------
      uint32_t t = 0;
#pragma unroll
      for (int j = 0; j < V2; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) t += COMPACT ? uint32_t(int32_t(x[j][k]) > 0) : x[j][k];
      t = __reduce_add_sync(kFull, t);
      if (lane == 0) sh.wtot[warp] = t;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t agg = 0;
#pragma unroll
        for (int w = 0; w < NW2; ++w) agg += sh.wtot[w];
        L.tile_val[tile] = agg;
        WF_2P_ADD(4, 1);
        const uint32_t nt = min(C, T - c * C);
        const uint32_t old = atom_add_acq_rel_gpu(L.chunk_cnt + 4 * c, 1u);
        sh.last = old == nt - 1;
      }
      __syncthreads();
      if (sh.last) {
        // ------------- chunk finisher: tile offsets of chunk c ----------
        // (the acq_rel arrival made every P1 tile_val of chunk c visible to
        // thread 0; the barrier extends that to the CTA)
#if WF_2P_STATS
        const unsigned long long f0 = gt2();
#endif
        const uint32_t t0 = c * C;
        const uint32_t nt = min(C, T - t0);
        constexpr int PER = (kMaxChunkTiles2P + B2 - 1) / B2;
        uint32_t v[PER], run = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const uint32_t i = threadIdx.x * PER + k;
          v[k] = i < nt ? ld_relaxed_u32(L.tile_val + t0 + i) : 0u;
          run += v[k];
        }
        uint32_t incl = run;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, incl, d);
          if (lane >= uint32_t(d)) incl += y;
        }
        __syncthreads();  // sh.wtot of the arrival step is consumed
        if (lane == 31) sh.wtot[warp] = incl;
        __syncthreads();
        uint32_t wex = 0, ctot = 0;
#pragma unroll
        for (int w = 0; w < NW2; ++w) {
          const uint32_t y = sh.wtot[w];
          wex += uint32_t(w) < warp ? y : 0u;
          ctot += y;
        }
        // chunk base: decoupled look-back over the chunk descriptors (warp 0)
        if (warp == 0) {
          uint32_t excl;
          if (c == 0) {
            excl = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
          } else {
            if (lane == 0)
              st_relaxed_gpu(L.chunk_desc + uint64_t(c) * kDescStride,
                             pack_desc(epoch, kStAggregate, ctot));
#if WF_2P_STATS
            const unsigned long long l0 = gt2();
#endif
            excl = lookback_exclusive_wide<1>(L.chunk_desc, c, epoch);
#if WF_2P_STATS
            if (lane == 0) WF_2P_ADD(1, gt2() - l0);
#endif
          }
          if (lane == 0) sh.base = excl;
        }
        __syncthreads();
        uint32_t o = sh.base + wex + incl - run;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const uint32_t i = threadIdx.x * PER + k;
          if (i < nt) L.tile_off[t0 + i] = o;
          o += v[k];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          L.chunk_cnt[4 * c] = 0u;  // last arrival of this launch: ready for the next
          __threadfence();
          // PREFIX = chunk ready: its tile offsets are written (release)
          st_release_u64(L.chunk_desc + uint64_t(c) * kDescStride,
                         pack_desc(epoch, kStPrefix, sh.base + ctot));
          if (COMPACT && c == K - 1) *count = uint64_t(sh.base + ctot);
#if WF_2P_STATS
          WF_2P_ADD(2, gt2() - f0);
#endif
        }
      }
    } else {
      // ---------------- P2: local scan / compaction, then write --------
      if (threadIdx.x == 0) {
        const uint64_t *d = L.chunk_desc + uint64_t(c) * kDescStride;
#if WF_2P_STATS
        const unsigned long long w0 = gt2();
        const bool ready = is_prefix(ld_acquire_u64(d), epoch);
#endif
        uint32_t backoff = 32;
        while (!is_prefix(ld_acquire_u64(d), epoch)) {
          __nanosleep(backoff);
          backoff = backoff < 512 ? backoff * 2 : 512;
        }
        sh.offset = ld_relaxed_u32(L.tile_off + tile);
#if WF_2P_STATS
        WF_2P_ADD(0, gt2() - w0);
        WF_2P_ADD(5, 1);
        if (!ready) WF_2P_ADD(3, 1);
#endif
      }
      if (!COMPACT) {
        uint32_t carry = 0;
#pragma unroll
        for (int j = 0; j < V2; ++j) {
          x[j][1] += x[j][0];
          x[j][2] += x[j][1];
          x[j][3] += x[j][2];
          const uint32_t tt = x[j][3];
          uint32_t v = tt;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, v, d);
            if (lane >= uint32_t(d)) v += y;
          }
          const uint32_t add = carry + v - tt;
          carry += __shfl_sync(kFull, v, 31);
#pragma unroll
          for (int k = 0; k < 4; ++k) x[j][k] += add;
        }
        if (lane == 0) sh.wtot[warp] = carry;
        __syncthreads();
        uint32_t add = sh.offset;
#pragma unroll
        for (int w = 0; w < NW2; ++w) add += uint32_t(w) < warp ? sh.wtot[w] : 0u;
        if (full) {
#pragma unroll
          for (int j = 0; j < V2; ++j) {
            uint4 q;
            q.x = x[j][0] + add; q.y = x[j][1] + add; q.z = x[j][2] + add; q.w = x[j][3] + add;
            stg_stream(reinterpret_cast<uint4 *>(out + base + j * 128), q);
          }
        } else {
#pragma unroll
          for (int j = 0; j < V2; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t idx = base + j * 128 + k;
              if (idx < n) out[idx] = int32_t(x[j][k] + add);
            }
        }
      } else {
        const uint32_t lt = lanemask_lt();
        uint32_t pos[V2];
        uint32_t carry = 0;
#pragma unroll
        for (int j = 0; j < V2; ++j) {
          uint32_t excl = 0, tot = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool f = int32_t(x[j][k]) > 0;  // ragged padding is 0: never selected
            const uint32_t b = __ballot_sync(kFull, f);
            excl += __popc(b & lt);
            tot += __popc(b);
          }
          pos[j] = carry + excl;
          carry += tot;
        }
        if (lane == 0) sh.wtot[warp] = carry;
        __syncthreads();
        uint32_t p0 = sh.offset;
#pragma unroll
        for (int w = 0; w < NW2; ++w) p0 += uint32_t(w) < warp ? sh.wtot[w] : 0u;
#pragma unroll
        for (int j = 0; j < V2; ++j) {
          uint32_t p = p0 + pos[j];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (int32_t(x[j][k]) > 0) out[p++] = int32_t(x[j][k]);
        }
      }
    }
    __syncthreads();  // everyone is done with sh.* of this item
    if (threadIdx.x == 0) sh.item = pick(S, L, T, C, epoch);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // every claim of this CTA is behind it; the last CTA to leave resets the
    // tickets and bumps the epoch for the next stream-ordered launch
    if (atom_add_acq_rel_gpu(L.exits, 1u) == gridDim.x - 1) {
      atomicExch(L.p1, 0u);
      atomicExch(L.p2, 0u);
      atomicExch(L.exits, 0u);
      atomicExch(&hdr->epoch, (epoch + 1) & kEpochMask);
    }
#if WF_2P_STATS
    WF_2P_ADD(6, gt2() - life0);
#endif
  }
}

struct Plan2P {
  uint32_t T, C, K, lead;
};

uint32_t env_u32(const char *name, uint32_t dflt) {
  const char *e = getenv(name);
  return e ? uint32_t(strtoul(e, nullptr, 0)) : dflt;
}

Plan2P plan2p(uint64_t n) {
  Plan2P p;
  p.T = uint32_t((n + TILE2 - 1) / TILE2);
  uint32_t C = env_u32("WF_2P_CHUNK_TILES", WF_2P_CHUNK);
  if (C < 1) C = 1;
  const uint32_t cmin = (p.T + kMaxChunks2P - 1) / kMaxChunks2P;
  if (C < cmin) C = cmin;
  p.C = C;
  p.K = (p.T + C - 1) / C;
  p.lead = env_u32("WF_2P_LEAD", WF_2P_LEAD);
  return p;
}

template <bool COMPACT>
int grid2p(uint32_t T) {
  static int per_sm[2] = {0, 0};
  int &b = per_sm[COMPACT];
  if (b == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, two_pass_kernel<COMPACT>, B2, 0);
    if (b < 1) b = 1;
  }
  const uint32_t g = uint32_t(b) * uint32_t(sm_count(current_device()));
  return int(T < g ? T : g);
}

}  // namespace

#if WF_2P_STATS
extern "C" int wf_debug_2p_stats(unsigned long long *host8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host8, g_2p_stats, sizeof(unsigned long long) * 8);
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {};
    e = cudaMemcpyToSymbol(g_2p_stats, z, sizeof z);
  }
  return int(e);
}
#endif

// Opt-in (measured slower than the single-pass kernels on B200, see the file
// header and profiles/r01_scan_compact_experiments.md).  Env knobs, read per
// call so tests can flip them: WF_SCAN_2P=1 enables the two-pass kernels,
// WF_2P_MIN_N moves the size threshold, WF_2P_CHUNK_TILES and WF_2P_LEAD set
// the chunk size and the P1 lead in tiles.
bool two_pass_usable(uint64_t n) {
  const char *e = getenv("WF_SCAN_2P");
  if (e == nullptr || e[0] != '1') return false;
  const char *m = getenv("WF_2P_MIN_N");
  const uint64_t min_n = m ? strtoull(m, nullptr, 0) : kTwoPassMinN;
  if (n == 0 || n < min_n) return false;
  const Plan2P p = plan2p(n);
  // the layout must fit the scan workspace (ws_need of the op for this n)
  const size_t need = ((size_t(p.T) * 8 + 127) & ~size_t(127)) + size_t(p.K) * 128;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  return p.C <= kMaxChunkTiles2P && p.K <= kMaxChunks2P && need <= tiles * 8 * kDescStride;
}

cudaError_t launch_scan2p_i32(const int32_t *in, int32_t *out, uint64_t n, const int32_t *carry,
                              void *ws, cudaStream_t s) {
  const Plan2P p = plan2p(n);
  two_pass_kernel<false><<<grid2p<false>(p.T), B2, 0, s>>>(in, out, n, p.T, p.C, p.K, p.lead,
                                                            carry, nullptr, ws);
  return cudaGetLastError();
}

cudaError_t launch_compact2p_i32(const int32_t *in, uint64_t n, int32_t *out, uint64_t *count,
                                 void *ws, cudaStream_t s) {
  const Plan2P p = plan2p(n);
  two_pass_kernel<true><<<grid2p<true>(p.T), B2, 0, s>>>(in, out, n, p.T, p.C, p.K, p.lead,
                                                          nullptr, count, ws);
  return cudaGetLastError();
}

}  // namespace wf
