// wf_scan_legacy.cu — NOT part of the product library.  The pre-TMEM K3/K4
// kernels of round 1, kept as variant builds for A/B evidence
// (profiles/r01_scan_compact_experiments.md): the register-tile single-pass
// kernel and the smem-stage persistent kernel with a TMA ring.  Built only by
// tools/build_variants.py with -DWF_SCAN_IMPL=1|2 (see csrc/wf_scan.cu).
//
// Register-tile kernels: one 16 KiB tile per CTA in registers.  Persistent
// kernel: grid = SMs x resident CTAs, each CTA draws tile ids from an atomic
// ticket, pulls the 32 KiB tile into shared memory with ONE 1-D bulk copy
// (cp.async.bulk, completion on an mbarrier), reduces it (REDUX.SUM), looks
// back (warp 0) and scans / ballot-compacts it.  Both were measured slower
// than the TMEM-parked kernel (390 / 347 us vs 320 / 262 us at 2^28).
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"

#include <cstdlib>

#ifndef WF_LBK
#define WF_LBK 1  // scan: look-back predecessors per lane (window = 32 * WF_LBK)
#endif
#ifndef WF_LBK_COMPACT
#define WF_LBK_COMPACT 2  // compaction look-back width (measured best, tools/sweep3.sh)
#endif
#ifndef WF_PVEC
#define WF_PVEC 8  // persistent tile = 256 threads x 4 x WF_PVEC items
#endif
#ifndef WF_MINB
#define WF_MINB 8  // __launch_bounds__ min blocks per SM of the tile kernels
#endif
#ifndef WF_TRACE
#define WF_TRACE 0
#endif
#ifndef WF_PSTAGES
#define WF_PSTAGES 1  // >1 prefetches tiles whose aggregates then publish late
#endif

namespace wf {
#if WF_TRACE
__device__ unsigned long long *g_wf_trace = nullptr;  // [tile][4] globaltimer stamps
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WF_STAMP(tile, k) \
  if (threadIdx.x == 0 && g_wf_trace) g_wf_trace[uint64_t(tile) * 4 + (k)] = gtimer()
#else
#define WF_STAMP(tile, k)
#endif
namespace {

constexpr int BLOCK = kScanBlock;
constexpr int VEC = kScanVec;
constexpr int NW = BLOCK / 32;
constexpr int CHUNK = 128;               // items per warp-load
constexpr int WSEG = CHUNK * VEC;        // items per warp per tile
constexpr uint32_t TILE = uint32_t(kScanTile);

__device__ __forceinline__ void load_tile(const int32_t *__restrict__ in,
                                          uint64_t n, uint64_t base, bool vec,
                                          uint32_t (&x)[VEC][4]) {
  if (vec) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const uint4 q = ldg_stream(reinterpret_cast<const uint4 *>(in + base + j * CHUNK));
      x[j][0] = q.x; x[j][1] = q.y; x[j][2] = q.z; x[j][3] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t idx = base + j * CHUNK + k;
        x[j][k] = idx < n ? uint32_t(in[idx]) : 0u;
      }
  }
}

// Tile-level look-back shared by scan and compaction.  Called by all threads
// after the tile aggregate is known; returns the tile's exclusive prefix.
__device__ __forceinline__ uint32_t tile_prefix(uint64_t *__restrict__ desc,
                                                uint32_t tile, uint32_t epoch,
                                                uint32_t aggregate,
                                                uint32_t carry_in) {
  __shared__ uint32_t s_prefix;
  if (threadIdx.x < 32) {
    uint32_t excl;
    if (tile == 0) {
      excl = carry_in;
      if (threadIdx.x == 0) st_relaxed_gpu(desc, pack_desc(epoch, kStPrefix, excl + aggregate));
    } else {
      if (threadIdx.x == 0) st_relaxed_gpu(desc + uint64_t(tile) * kDescStride, pack_desc(epoch, kStAggregate, aggregate));
      excl = lookback_exclusive_wide<WF_LBK>(desc, tile, epoch);
      if (threadIdx.x == 0) st_relaxed_gpu(desc + uint64_t(tile) * kDescStride, pack_desc(epoch, kStPrefix, excl + aggregate));
    }
    if (threadIdx.x == 0) s_prefix = excl;
  }
  __syncthreads();
  return s_prefix;
}

__global__ void __launch_bounds__(BLOCK, WF_MINB)
    scan_i32_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out,
                    uint64_t n, uint32_t ntiles, bool aligned,
                    const int32_t *__restrict__ carry_in,
                    uint64_t *__restrict__ desc, TileHeader *__restrict__ hdr) {
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ uint32_t s_wtot[NW];
  if (threadIdx.x == 0) {
    uint32_t t, e;
    take_ticket(hdr, ntiles, t, e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const uint32_t tile = s_tile, epoch = s_epoch;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = uint64_t(tile) * TILE + uint64_t(warp) * WSEG + lane * 4;
  const bool vec = aligned && uint64_t(tile + 1) * TILE <= n;
  WF_STAMP(tile, 0);

  uint32_t x[VEC][4];
  load_tile(in, n, base, vec, x);

  // per 128-item chunk: thread-serial scan of 4 items, SHFL.UP warp scan of
  // the thread totals (the SDK shfl_scan step), running warp carry.
  uint32_t carry = 0;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    x[j][1] += x[j][0];
    x[j][2] += x[j][1];
    x[j][3] += x[j][2];
    const uint32_t t = x[j][3];
    uint32_t s = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, s, d);
      if (lane >= uint32_t(d)) s += y;
    }
    const uint32_t add = carry + s - t;
    carry += __shfl_sync(kFull, s, 31);
#pragma unroll
    for (int k = 0; k < 4; ++k) x[j][k] += add;
  }
  if (lane == 0) s_wtot[warp] = carry;
  __syncthreads();
  uint32_t wexcl = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t v = s_wtot[w];
    wexcl += uint32_t(w) < warp ? v : 0u;
    agg += v;
  }
  const uint32_t cin = (tile == 0 && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
  WF_STAMP(tile, 1);
  const uint32_t add = tile_prefix(desc, tile, epoch, agg, cin) + wexcl;
  WF_STAMP(tile, 2);

  if (vec) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      uint4 q;
      q.x = x[j][0] + add; q.y = x[j][1] + add; q.z = x[j][2] + add; q.w = x[j][3] + add;
      stg_stream(reinterpret_cast<uint4 *>(out + base + j * CHUNK), q);
    }
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t idx = base + j * CHUNK + k;
        if (idx < n) out[idx] = int32_t(x[j][k] + add);
      }
  }
  WF_STAMP(tile, 3);
}

__global__ void __launch_bounds__(BLOCK, WF_MINB)
    compact_gt0_kernel(const int32_t *__restrict__ in, uint64_t n,
                       uint32_t ntiles, bool aligned,
                       int32_t *__restrict__ out, uint64_t *__restrict__ count,
                       uint64_t *__restrict__ desc,
                       TileHeader *__restrict__ hdr) {
  __shared__ uint32_t s_tile, s_epoch;
  __shared__ uint32_t s_wtot[NW];
  __shared__ int32_t s_stage[TILE];  // tile-local compacted output
  if (threadIdx.x == 0) {
    uint32_t t, e;
    take_ticket(hdr, ntiles, t, e);
    s_tile = t;
    s_epoch = e;
  }
  __syncthreads();
  const uint32_t tile = s_tile, epoch = s_epoch;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = uint64_t(tile) * TILE + uint64_t(warp) * WSEG + lane * 4;
  const bool vec = aligned && uint64_t(tile + 1) * TILE <= n;

  uint32_t x[VEC][4];
  load_tile(in, n, base, vec, x);

  // warp-aggregated selection: one ballot per item slot, popc of the lanes
  // below gives this lane's position inside the chunk (memory order).
  const uint32_t lt = lanemask_lt();
  uint32_t pos[VEC];
  uint32_t carry = 0;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    uint32_t excl = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t idx = base + j * CHUNK + k;
      const bool f = int32_t(x[j][k]) > 0 && (vec || idx < n);
      const uint32_t b = __ballot_sync(kFull, f);
      excl += __popc(b & lt);
      tot += __popc(b);
      if (!f) x[j][k] = 0u;  // 0 marks "not selected" (selected values are > 0)
    }
    pos[j] = carry + excl;
    carry += tot;
  }
  if (lane == 0) s_wtot[warp] = carry;
  __syncthreads();
  uint32_t wexcl = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t v = s_wtot[w];
    wexcl += uint32_t(w) < warp ? v : 0u;
    agg += v;
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    uint32_t p = wexcl + pos[j];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (x[j][k] != 0u) s_stage[p++] = int32_t(x[j][k]);
    }
  }
  const uint32_t prefix = tile_prefix(desc, tile, epoch, agg, 0u);  // syncs
  int32_t *dst = out + prefix;
  for (uint32_t i = threadIdx.x; i < agg; i += BLOCK) dst[i] = s_stage[i];
  if (tile == ntiles - 1 && threadIdx.x == 0) *count = uint64_t(prefix) + agg;
}


// ---------------------------------------------------------------------------
// Persistent, TMA-pipelined variant (16-byte aligned buffers).
//
// grid = SMs x resident CTAs.  Each CTA draws tile ids from the ticket
// counter and keeps a ring of PSTAGES shared-memory stages: the 1-D bulk copy
// (cp.async.bulk -> UBLKCP) of tile t+1 is in flight while tile t is scanned
// and looks back, so HBM latency overlaps the look-back latency.  Scan results
// are written back into the stage and leave through a bulk store
// (cp.async.bulk.global.shared); compaction writes its (unaligned) output with
// coalesced stores from the stage.
//
// Ticket protocol: every CTA draws until it receives an id >= ntiles (exactly
// one over-draw per CTA), so the CTA whose draw returns ntiles + grid - 1 is
// the last drawer: it resets the counter and bumps the epoch.  Every CTA read
// the epoch before its first draw, hence before the bump.
#ifndef WF_PBLOCK
#define WF_PBLOCK 256
#endif
constexpr int PBLOCK = WF_PBLOCK;
constexpr int PNW = PBLOCK / 32;
constexpr int PVEC = WF_PVEC;                     // 128-item chunks per warp
constexpr uint32_t PTILE = uint32_t(PBLOCK) * PVEC * 4;   // 8192 items, 32 KiB
constexpr int PSTAGES = WF_PSTAGES;
constexpr uint32_t kNoTile = 0xffffffffu;

struct PersistShared {
  uint64_t full[PSTAGES];
  uint32_t tile[PSTAGES];
  uint32_t epoch;
  uint32_t prefix;
  uint32_t wtot[PNW];
};

// The first draw of a CTA is a release (it orders the CTA's epoch read before
// the draw); later draws are relaxed — nothing the tile protocol needs is
// ordered by them (descriptor values travel inside the descriptor word), and
// a release there would wait for the previous tile's output stores to be
// acknowledged (measured: scan 404 -> 390 us, compaction 369 -> 348 us at
// 2^28).  The last drawer acquires through the counter's release sequence
// before it resets the counter and bumps the epoch.
template <bool FIRST>
__device__ __forceinline__ uint32_t draw_ticket(TileHeader *hdr, uint32_t ntiles,
                                                uint32_t epoch, bool &drained) {
  const uint32_t t = FIRST ? atom_add_acq_rel_gpu(&hdr->ticket, 1u)
                           : atom_add_relaxed_gpu(&hdr->ticket, 1u);
  if (t >= ntiles) {
    drained = true;
    if (t == ntiles + gridDim.x - 1) {  // last of all draws
      fence_acq_rel_gpu();
      atomicExch(&hdr->ticket, 0u);
      atomicExch(&hdr->epoch, (epoch + 1) & kEpochMask);
    }
    return kNoTile;
  }
  return t;
}

template <bool COMPACT>
__global__ void __launch_bounds__(PBLOCK)
    tile_persistent_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out,
                           uint64_t n, uint32_t ntiles,
                           const int32_t *__restrict__ carry_in,
                           uint64_t *__restrict__ count, uint64_t *__restrict__ desc,
                           TileHeader *__restrict__ hdr) {
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  __shared__ PersistShared sh;
  int32_t *stage0 = reinterpret_cast<int32_t *>(dyn_smem);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();

  bool drained = false;  // meaningful in thread 0 only
  if (threadIdx.x == 0) {
    for (int s = 0; s < PSTAGES; ++s) mbar_init(&sh.full[s], 1);
    fence_barrier_init();
    sh.epoch = ld_volatile_u32(&hdr->epoch) & kEpochMask;  // ordered by the release draw
    for (int s = 0; s < PSTAGES; ++s) {
      const uint32_t t = drained ? kNoTile : draw_ticket<true>(hdr, ntiles, sh.epoch, drained);
      if (t != kNoTile) WF_STAMP(t, 0);
      sh.tile[s] = t;
      if (t != kNoTile && uint64_t(t + 1) * PTILE <= n) {
        mbar_arrive_expect_tx(&sh.full[s], PTILE * 4);
        tma_load_1d(stage0 + s * PTILE, in + uint64_t(t) * PTILE, PTILE * 4, &sh.full[s]);
      }
    }
  }
  __syncthreads();
  const uint32_t epoch = sh.epoch;
  uint32_t phase = 0;  // bit s = parity of stage s

  for (uint32_t it = 0;; ++it) {
    const int s = int(it % PSTAGES);
    const uint32_t tile = sh.tile[s];
    if (tile == kNoTile) break;
    int32_t *buf = stage0 + s * PTILE;
    const uint64_t base = uint64_t(tile) * PTILE;
    const bool full = base + PTILE <= n;
    if (full) {
      mbar_wait(&sh.full[s], (phase >> s) & 1u);
      phase ^= 1u << s;
      WF_STAMP(tile, 1);
    } else {  // ragged last tile: guarded cooperative loads, zero padding
      for (uint32_t i = threadIdx.x; i < PTILE; i += PBLOCK)
        buf[i] = base + i < n ? in[base + i] : 0;
      __syncthreads();
    }
    // warp w owns PVEC consecutive 128-item chunks of the stage
    const uint32_t off0 = warp * (PVEC * 128) + lane * 4;

    // pass A: warp totals (sum, or number of selected items)
    uint32_t t = 0;
#pragma unroll 4
    for (int j = 0; j < PVEC; ++j) {
      const uint4 q = *reinterpret_cast<const uint4 *>(buf + off0 + j * 128);
      if (COMPACT)
        t += (int32_t(q.x) > 0) + (int32_t(q.y) > 0) + (int32_t(q.z) > 0) + (int32_t(q.w) > 0);
      else
        t += q.x + q.y + q.z + q.w;
    }
    t = __reduce_add_sync(kFull, t);
    if (lane == 0) sh.wtot[warp] = t;
    __syncthreads();
    uint32_t wexcl = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < PNW; ++w) {
      const uint32_t v = sh.wtot[w];
      wexcl += uint32_t(w) < warp ? v : 0u;
      agg += v;
    }
    // decoupled look-back (warp 0)
    if (warp == 0) {
      uint32_t excl;
      if (tile == 0) {
        excl = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
        if (lane == 0) st_relaxed_gpu(desc, pack_desc(epoch, kStPrefix, excl + agg));
      } else {
        if (lane == 0)
          st_relaxed_gpu(desc + uint64_t(tile) * kDescStride, pack_desc(epoch, kStAggregate, agg));
        excl = lookback_exclusive_wide<COMPACT ? WF_LBK_COMPACT : WF_LBK>(desc, tile, epoch);
        if (lane == 0)
          st_relaxed_gpu(desc + uint64_t(tile) * kDescStride, pack_desc(epoch, kStPrefix, excl + agg));
      }
      if (lane == 0) sh.prefix = excl;
    }
    __syncthreads();
    const uint32_t prefix = sh.prefix;
    WF_STAMP(tile, 2);

    // pass B: chunk-serial scan with the running warp carry
    uint32_t carry = prefix + wexcl;
    if (!COMPACT) {
#pragma unroll 4
      for (int j = 0; j < PVEC; ++j) {
        uint4 q = *reinterpret_cast<const uint4 *>(buf + off0 + j * 128);
        q.y += q.x;
        q.z += q.y;
        q.w += q.z;
        uint32_t v = q.w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, v, d);
          if (lane >= uint32_t(d)) v += y;
        }
        const uint32_t add = carry + v - q.w;
        carry += __shfl_sync(kFull, v, 31);
        q.x += add; q.y += add; q.z += add; q.w += add;
        *reinterpret_cast<uint4 *>(buf + off0 + j * 128) = q;
      }
      if (full) {
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
          tma_store_1d(out + base, buf, PTILE * 4);
          bulk_commit();
        }
      } else {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < PTILE && base + i < n; i += PBLOCK) out[base + i] = buf[i];
      }
    } else {
      // ballot + popc positions; each chunk's selected items land contiguously
#pragma unroll 2
      for (int j = 0; j < PVEC; ++j) {
        const uint4 q = *reinterpret_cast<const uint4 *>(buf + off0 + j * 128);
        const uint32_t v[4] = {q.x, q.y, q.z, q.w};
        uint32_t b[4], excl = 0, tot = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          b[k] = __ballot_sync(kFull, int32_t(v[k]) > 0);
          excl += __popc(b[k] & lt);
          tot += __popc(b[k]);
        }
        uint32_t p = carry + excl;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (int32_t(v[k]) > 0) out[p++] = int32_t(v[k]);
        carry += tot;
      }
      if (tile == ntiles - 1 && threadIdx.x == 0) *count = uint64_t(prefix) + agg;
    }
    WF_STAMP(tile, 3);
    __syncthreads();  // stage s fully consumed by the threads
    if (threadIdx.x == 0) {  // refill stage s with the next tile
      const uint32_t tn = drained ? kNoTile : draw_ticket<false>(hdr, ntiles, epoch, drained);
      if (tn != kNoTile) WF_STAMP(tn, 0);
      sh.tile[s] = tn;
      if (!COMPACT && tn != kNoTile) bulk_wait_read_all();  // bulk store has left stage s
      if (tn != kNoTile && uint64_t(tn + 1) * PTILE <= n) {
        mbar_arrive_expect_tx(&sh.full[s], PTILE * 4);
        tma_load_1d(buf, in + uint64_t(tn) * PTILE, PTILE * 4, &sh.full[s]);
      }
    }
    __syncthreads();
  }
  if (!COMPACT && threadIdx.x == 0) bulk_wait_all();
}

constexpr size_t kPersistSmem = size_t(PSTAGES) * PTILE * 4;

template <bool COMPACT>
int persistent_grid(uint32_t ntiles) {
  static int per_sm[2] = {0, 0};
  static DeviceMask configured[2];
  int &b = per_sm[COMPACT];
  configured[COMPACT].ensure([] {
    cudaFuncSetAttribute(tile_persistent_kernel<COMPACT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPersistSmem));
  });
  if (b == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tile_persistent_kernel<COMPACT>, PBLOCK,
                                                  kPersistSmem);
    if (b < 1) b = 1;
  }
  const uint32_t full = uint32_t(b) * uint32_t(sm_count(current_device()));
  return int(ntiles < full ? ntiles : full);
}

}  // namespace
cudaError_t launch_scan_legacy_i32(int impl, const int32_t *in, int32_t *out, uint64_t n,
                                   const int32_t *carry, void *ws, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  if (impl == 1 && aligned) {
    const uint64_t pt = (n + PTILE - 1) / PTILE;
    const int grid = persistent_grid<false>(uint32_t(pt));
    tile_persistent_kernel<false><<<grid, PBLOCK, kPersistSmem, s>>>(
        in, out, n, uint32_t(pt), carry, nullptr, desc, hdr);
    return cudaGetLastError();
  }
  scan_i32_kernel<<<uint32_t(ntiles), BLOCK, 0, s>>>(in, out, n, uint32_t(ntiles), aligned,
                                                      carry, desc, hdr);
  return cudaGetLastError();
}

cudaError_t launch_compact_legacy_i32(int impl, const int32_t *in, uint64_t n, int32_t *out,
                                      uint64_t *count, void *ws, cudaStream_t s) {
  if (n == 0) return cudaMemsetAsync(count, 0, sizeof(uint64_t), s);
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
  if (impl == 1 && aligned) {
    const uint64_t pt = (n + PTILE - 1) / PTILE;
    const int grid = persistent_grid<true>(uint32_t(pt));
    tile_persistent_kernel<true><<<grid, PBLOCK, kPersistSmem, s>>>(
        in, out, n, uint32_t(pt), nullptr, count, desc, hdr);
    return cudaGetLastError();
  }
  compact_gt0_kernel<<<uint32_t(ntiles), BLOCK, 0, s>>>(in, n, uint32_t(ntiles), aligned, out,
                                                         count, desc, hdr);
  return cudaGetLastError();
}

}  // namespace wf
