// wf_scan.cu — K3 scan_inclusive_i32 and K4 compact_gt0_i32.
//
// Both are single-pass tile kernels with decoupled look-back:
//   tile = 256 threads x 16 items = 4096 int32 (16 KiB).  Warp w of the tile
//   owns 4 consecutive 128-item chunks; in chunk j lane l holds items
//   4l..4l+3 (one 16-byte load), so a warp-load is 512 contiguous bytes and a
//   lane's items stay in memory order.
//
// K3 reference analog: the CUDA SDK shfl_scan (warp scan with __shfl_up_sync,
// warp sums in smem, block carry) that the reference can only express as a
// lane-reversed shfl_down suffix scan (corpus.py:347-364);
// its cross-block carries would need several launches through a host
// description (runtime/hostdesc.py:109-129).  Here the carries flow between
// tiles in the same launch through the look-back descriptors.
//
// K4 reference analog: none expressible (no ballot / atomics in the DSL,
// dsl/lexer.py:18-25); CUDA-semantics extension with the warp-aggregated
// ballot + popc idiom, made order-preserving by the tile look-back.
//
// Roofline: HBM. K3 moves 8 B/elem (read + write); K4 4 B/elem read plus
// 4 B per selected element written.
#include "wf_device.cuh"
#include "wf_internal.h"

namespace wf {
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
      if (threadIdx.x == 0) st_relaxed_gpu(desc + tile, pack_desc(epoch, kStAggregate, aggregate));
      excl = lookback_exclusive(desc, tile, epoch);
      if (threadIdx.x == 0) st_relaxed_gpu(desc + tile, pack_desc(epoch, kStPrefix, excl + aggregate));
    }
    if (threadIdx.x == 0) s_prefix = excl;
  }
  __syncthreads();
  return s_prefix;
}

__global__ void __launch_bounds__(BLOCK)
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
  const uint32_t add = tile_prefix(desc, tile, epoch, agg, cin) + wexcl;

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
}

__global__ void __launch_bounds__(BLOCK)
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

}  // namespace

cudaError_t launch_scan_i32(const int32_t *in, int32_t *out, uint64_t n,
                            const int32_t *carry, void *ws, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kWsHeader);
  const bool aligned = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  scan_i32_kernel<<<uint32_t(ntiles), BLOCK, 0, s>>>(in, out, n, uint32_t(ntiles), aligned,
                                                      carry, desc, hdr);
  return cudaGetLastError();
}

cudaError_t launch_compact_gt0_i32(const int32_t *in, uint64_t n, int32_t *out,
                                   uint64_t *count, void *ws, cudaStream_t s) {
  if (n == 0) return cudaMemsetAsync(count, 0, sizeof(uint64_t), s);
  const uint64_t ntiles = (n + TILE - 1) / TILE;
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kWsHeader);
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
  compact_gt0_kernel<<<uint32_t(ntiles), BLOCK, 0, s>>>(in, n, uint32_t(ntiles), aligned, out,
                                                         count, desc, hdr);
  return cudaGetLastError();
}

}  // namespace wf
