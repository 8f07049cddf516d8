// wf_patterns.cu — native kernels for the reference's OWN DSL formulations
// of the hot path, reached when dsl/patterns.py recognises a kernel
// structurally (the "DSL AST -> native symbol" registry of SURVEY §8b).
//
// The reference can express C1/C2 only as the per-warp-partials kernel of
// SURVEY §8c (tests/golden/C1_I32.spk / C1_F32.spk) and C3 only as the
// in-warp prefix on lane-reversed data (C3_WARP_PREFIX.spk).  Run through
// launch(hybrid_transform(...)) (runtime/launch.py:90, passes/pipeline.py:
// 103-179) those kernels would otherwise go through the generic DSL codegen
// (bounds-checked scalar code with a fault record).  The kernels below write
// EXACTLY what the DSL kernel writes — same outputs, same fp32 association —
// at streaming speed:
//
//   warp_partials_kernel<T>  out[b * (B/32) + w] = the shfl_down tree
//                            (off 16, 8, 4, 2, 1) of each lane's grid-stride
//                            sum, each lane summing a[i] for i = gt, gt + S,
//                            ... in increasing i, one add per element (the
//                            reference order; fp32 bit-exact)
//   warp_prefix32_kernel     out[32 s + k] = a[32 s] + ... + a[32 s + k]
//                            (wrapping i32) — what the reversed shfl_down
//                            suffix tree of C3_WARP_PREFIX.spk computes for
//                            every aligned 32-element warp segment
//
// Preconditions (checked by the Python matcher, which otherwise keeps the
// generic path so faults and wrap-around behave as the DSL would): warp
// size 32, block % 32 == 0, index arithmetic that cannot overflow i32, and
// buffers long enough for every access.
#include "wf_device.cuh"
#include "wf_internal.h"

namespace wf {
namespace {

#ifndef WF_PARTIALS_UNROLL
#define WF_PARTIALS_UNROLL 16
#endif
constexpr int kPartialsUnroll = WF_PARTIALS_UNROLL;  // loads in flight per thread ahead of the in-order adds

__device__ __forceinline__ uint32_t ldg_na_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

template <bool F32>
__global__ void __launch_bounds__(1024) warp_partials_kernel(const uint32_t *__restrict__ a,
                                                             int64_t n,
                                                             uint32_t *__restrict__ out) {
  const int64_t stride = int64_t(blockDim.x) * gridDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  float fs = 0.0f;
  uint32_t is = 0u;
  auto add = [&](uint32_t v) {
    if (F32)
      fs = __fadd_rn(fs, __uint_as_float(v));  // one rounding per element, in i order
    else
      is += v;  // i32 wrap (numerics.py:20-22)
  };
  // software-pipelined: the U loads of batch k+1 are in flight while batch
  // k is added; the adds keep the reference's order exactly
  constexpr int U = kPartialsUnroll;
  uint32_t cur[U];
  bool have = i + (U - 1) * stride < n;
  if (have) {
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = ldg_na_u32(a + i + u * stride);
  }
  while (have) {
    const int64_t j = i + U * stride;
    const bool have_next = j + (U - 1) * stride < n;
    uint32_t nxt[U];
    if (have_next) {
#pragma unroll
      for (int u = 0; u < U; ++u) nxt[u] = ldg_na_u32(a + j + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) add(cur[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    i = j;
    have = have_next;
  }
  for (; i < n; i += stride) add(ldg_na_u32(a + i));
  // sum = sum + shfl_down(sum, off), off = 16, 8, 4, 2, 1; out-of-range
  // sources return the lane's own value (passes/warp_lower.py:36-45), which
  // is also what __shfl_down_sync does
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    if (F32)
      fs = __fadd_rn(fs, __shfl_down_sync(kFull, fs, off));
    else
      is += __shfl_down_sync(kFull, is, off);
  }
  if ((threadIdx.x & 31u) == 0)
    out[uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)] =
        F32 ? __float_as_uint(fs) : is;
}

// grid * block >= n: every DSL thread sums at most ONE element, so the warp
// partial of global warp w is the shfl_down tree over elements 32w .. 32w+31
// (lane value 0 + a[i], 0 past n).  Here 8 lanes hold one 32-element segment
// as 16-byte vectors (lane j: elements 4j .. 4j+3) and replay the same tree:
//   off 16: lanes j < 4 add lane j+4 component-wise   (e + 16)
//   off  8: lanes j < 2 add lane j+2                  (e + 8)
//   off  4: lane 0 adds lane 1                        (e + 4)
//   off  2: (c0 + c2), (c1 + c3);  off 1: their sum
// — the same fp32 additions in the same association, so the bits are the
// DSL kernel's; persistent grid instead of the DSL's grid * block threads.
template <bool F32>
__global__ void __launch_bounds__(256) warp_partials_1pt_kernel(const uint32_t *__restrict__ a,
                                                                int64_t n, uint32_t nseg,
                                                                uint32_t *__restrict__ out) {
  const uint32_t j = threadIdx.x & 7u;  // lane within the segment
  const uint64_t T = uint64_t(blockDim.x) * gridDim.x / 8;  // segments per grid step
  for (uint64_t seg = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 8; seg < nseg;
       seg += T) {
    const int64_t e0 = int64_t(seg) * 32 + 4 * j;
    uint4 q;
    if (e0 + 3 < n) {
      q = ldg_stream(reinterpret_cast<const uint4 *>(a + e0));
    } else {
      q.x = e0 < n ? a[e0] : 0u;
      q.y = e0 + 1 < n ? a[e0 + 1] : 0u;
      q.z = e0 + 2 < n ? a[e0 + 2] : 0u;
      q.w = 0u;
    }
    if (F32) {
      float v[4] = {__fadd_rn(0.0f, __uint_as_float(q.x)), __fadd_rn(0.0f, __uint_as_float(q.y)),
                    __fadd_rn(0.0f, __uint_as_float(q.z)), __fadd_rn(0.0f, __uint_as_float(q.w))};
#pragma unroll
      for (int d = 4; d >= 1; d >>= 1) {  // element offsets 16, 8, 4
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float o = __shfl_down_sync(kFull, v[c], d, 8);
          if (j < uint32_t(d)) v[c] = __fadd_rn(v[c], o);
        }
      }
      if (j == 0) out[seg] = __float_as_uint(__fadd_rn(__fadd_rn(v[0], v[2]), __fadd_rn(v[1], v[3])));
    } else {
      uint32_t t = q.x + q.y + q.z + q.w;  // i32 wrap: any order is the same value
#pragma unroll
      for (int d = 4; d >= 1; d >>= 1) t += __shfl_down_sync(kFull, t, d, 8);
      if (j == 0) out[seg] = t;
    }
  }
}

// 8 lanes per 32-element segment, 4 elements per lane (one 16-byte load),
// kPrefixVec vectors per thread per iteration (all loads issued first),
// grid-stride over the n/4 vectors; width-8 SHFL.UP scan of the lane totals.
#ifndef WF_PREFIX_VEC
#define WF_PREFIX_VEC 4
#endif
#ifndef WF_PREFIX_CTAS
#define WF_PREFIX_CTAS 32  // CTAs per SM the grid is sized for (8 / 16 / 32: 361 / 345-349 / 339 us at 2^28; tools/patterns_probe.py)
#endif
constexpr int kPrefixVec = WF_PREFIX_VEC;
#ifndef WF_PREFIX_MINB
#define WF_PREFIX_MINB 1  // resident CTAs the register budget must allow
#endif
__global__ void __launch_bounds__(256, WF_PREFIX_MINB) warp_prefix32_vec_kernel(const uint4 *__restrict__ a,
                                                                uint4 *__restrict__ out,
                                                                uint64_t nvec) {
  const uint32_t sl = threadIdx.x & 7u;  // lane within the segment
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t T = uint64_t(blockDim.x) * gridDim.x;
  // warp-uniform trip count (the shuffles need all 32 lanes); nvec % 8 == 0,
  // so a segment is either entirely in range or entirely out
  for (uint64_t v0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v0 - lane < nvec;
       v0 += kPrefixVec * T) {
    uint4 x[kPrefixVec];
#pragma unroll
    for (int k = 0; k < kPrefixVec; ++k) {
      const uint64_t v = v0 + k * T;
      x[k] = v < nvec ? ldg_stream(a + v) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < kPrefixVec; ++k) {
      x[k].y += x[k].x;
      x[k].z += x[k].y;
      x[k].w += x[k].z;
    }
    uint32_t run[kPrefixVec];
#pragma unroll
    for (int k = 0; k < kPrefixVec; ++k) run[k] = x[k].w;
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
#pragma unroll
      for (int k = 0; k < kPrefixVec; ++k) {
        const uint32_t y = __shfl_up_sync(kFull, run[k], d, 8);
        if (sl >= uint32_t(d)) run[k] += y;
      }
    }
#pragma unroll
    for (int k = 0; k < kPrefixVec; ++k) {
      const uint32_t excl = run[k] - x[k].w;
      x[k].x += excl;
      x[k].y += excl;
      x[k].z += excl;
      x[k].w += excl;
      const uint64_t v = v0 + k * T;
      if (v < nvec) stg_stream(out + v, x[k]);
    }
  }
}

// any alignment: one element per lane, 32-lane SHFL.UP scan
__global__ void __launch_bounds__(256) warp_prefix32_scalar_kernel(const uint32_t *__restrict__ a,
                                                                   uint32_t *__restrict__ out,
                                                                   uint64_t n) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i - lane < n;
       i += uint64_t(blockDim.x) * gridDim.x) {
    uint32_t v = a[i];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, v, d);
      if (lane >= uint32_t(d)) v += y;
    }
    out[i] = v;
  }
}

}  // namespace

cudaError_t launch_warp_partials(bool f32, const void *a, int64_t n, void *out, int grid,
                                 int block, cudaStream_t s) {
  if (grid == 0) return cudaSuccess;
  const auto *in = static_cast<const uint32_t *>(a);
  auto *o = static_cast<uint32_t *>(out);
  const int64_t threads = int64_t(grid) * block;
  if (threads >= n && (reinterpret_cast<uintptr_t>(a) & 15u) == 0) {  // one element per DSL thread
    const uint32_t nseg = uint32_t(threads / 32);  // every warp of the DSL grid writes its partial
    const uint64_t want = (uint64_t(nseg) * 8 + 255) / 256;
    const uint64_t cap = uint64_t(sm_count(current_device())) * 8;
    const unsigned g = unsigned(want < cap ? want : cap);
    if (f32)
      warp_partials_1pt_kernel<true><<<g, 256, 0, s>>>(in, n, nseg, o);
    else
      warp_partials_1pt_kernel<false><<<g, 256, 0, s>>>(in, n, nseg, o);
    return cudaGetLastError();
  }
  if (f32)
    warp_partials_kernel<true><<<grid, block, 0, s>>>(in, n, o);
  else
    warp_partials_kernel<false><<<grid, block, 0, s>>>(in, n, o);
  return cudaGetLastError();
}

// n % 32 == 0 (grid * block with block % 32 == 0)
cudaError_t launch_warp_prefix32(const int32_t *a, int32_t *out, uint64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int sms = sm_count(current_device());
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) {
    const uint64_t nvec = n / 4;
    const uint64_t want = (nvec + 256 * kPrefixVec - 1) / (256 * kPrefixVec);
    const uint64_t cap = uint64_t(sms) * WF_PREFIX_CTAS;
    const uint64_t grid = want < cap ? want : cap;
    warp_prefix32_vec_kernel<<<unsigned(grid), 256, 0, s>>>(reinterpret_cast<const uint4 *>(a),
                                                            reinterpret_cast<uint4 *>(out), nvec);
  } else {
    const uint64_t want = (n + 255) / 256;
    const uint64_t grid = want < uint64_t(sms) * 8 ? want : uint64_t(sms) * 8;
    warp_prefix32_scalar_kernel<<<unsigned(grid), 256, 0, s>>>(
        reinterpret_cast<const uint32_t *>(a), reinterpret_cast<uint32_t *>(out), n);
  }
  return cudaGetLastError();
}

}  // namespace wf
