// wf_reduce.cu — K1 reduce_sum_i32 and K2 reduce_sum_f32.
//
// Reference analog: the per-warp-partials shuffle reduction of SURVEY.md §8c
// (grid-stride per-thread sum -> five shfl_down rounds -> out[warp]) that the
// reference executes through launch() (runtime/launch.py:90) and the
// collapsed lane loops of passes/warp_lower.py:64-73, followed by a host
// wrap-fold.  Here the whole thing is ONE persistent-grid launch:
//
//   1. every thread streams 16-byte vectors (UNROLL loads in flight) into
//      4*UNROLL independent accumulator chains;
//   2. the chains fold in a fixed pairwise order, then the warp folds with
//      REDUX.SUM (i32) or a SHFL.BFLY butterfly (f32; REDUX has no f32 add);
//   3. warp sums fold through shared memory inside the block;
//   4. i32: one RED.ADD per block into a workspace accumulator; the block
//      that draws the last acq_rel ticket publishes it and resets both.
//      f32: block partials go to the workspace and the last block folds
//      them in block-index order (no fp atomics -> reproducible bits).
//
// The element->thread assignment depends only on (n, block, grid), so the f32
// result is bitwise reproducible run to run.  Roofline: HBM read, 4 B/elem.
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"

// Programmatic dependent launch (PDL).  Every reduce kernel signals
// `griddepcontrol.launch_dependents` as it starts, so a dependent launch may
// get its CTAs going on SMs this grid no longer needs.  Only EARLY launches
// (the caller's WF_FLAG_INPUT_STABLE promise: the kernel issued just before
// on the stream does not write `in`) are dependent launches: they stream
// their input while the previous grid drains (its last CTAs, its partial
// fold, the kernel boundary: ~6 us per launch, tools/red_trace.py) and wait
// for it (`griddepcontrol.wait`: completed and flushed) before touching the
// workspace or the output.  Without the flag the launch is stream-ordered as
// usual.

#ifndef WF_RED_OUTER_UNROLL1
// 1: the streaming loop is not unrolled beyond UNROLL by the compiler.  Its
// own 4x unroll (16 loads per trip, issued a few at a time) was 5 % slower at
// 256-thread CTAs and 10 % slower in the fused-exchange kernel at 1024
// (tools/k2_pdl_probe.py, profiles/r01_reduce_experiments.md "Round 2"); with
// 1, 256-thread CTAs are the fastest K2 configuration for both kernels
#define WF_RED_OUTER_UNROLL1 1
#endif
#ifndef WF_RED_TRACE
#define WF_RED_TRACE 0  // tools-only: per-block globaltimer stamps (tools/red_trace.py)
#endif

namespace wf {
#if WF_RED_TRACE
// per block: [0] start, [1] streaming done (block sum formed), [2] SM id;
// [4 * grid]: the last block's fold done.  Launch number g_red_seq (bumped by
// the last block) stamps record g_red_seq of stride 4 * 16384 + 8 words.
__device__ unsigned long long *g_red_trace = nullptr;
__device__ unsigned int g_red_seq = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RED_STAMP(k, v) \
  if (g_red_trace) g_red_trace[uint64_t(*(volatile unsigned *)&g_red_seq) * (4 * 16384 + 8) + (k)] = (v)
#else
#define RED_STAMP(k, v)
#endif
namespace {

struct SumI32 {
  using elem_t = int32_t;
  using acc_t = uint32_t;
  static constexpr bool kOrderFree = true;
  __device__ static uint32_t bits(acc_t v) { return v; }
  __device__ static acc_t zero() { return 0u; }
  __device__ static acc_t add(acc_t a, acc_t b) { return a + b; }
  __device__ static acc_t from_bits(uint32_t b) { return b; }
  __device__ static acc_t load(const elem_t *p) { return uint32_t(*p); }
  __device__ static acc_t warp_sum(acc_t v) {
    return __reduce_add_sync(kFull, v);  // REDUX.SUM
  }
  __device__ static elem_t to_elem(acc_t v) { return int32_t(v); }
};

struct SumF32 {
  using elem_t = float;
  using acc_t = float;
  static constexpr bool kOrderFree = false;  // fp: fixed-order fold for determinism
  __device__ static uint32_t bits(acc_t v) { return __float_as_uint(v); }
  __device__ static acc_t zero() { return 0.0f; }
  __device__ static acc_t add(acc_t a, acc_t b) { return __fadd_rn(a, b); }
  __device__ static acc_t from_bits(uint32_t b) { return __uint_as_float(b); }
  __device__ static acc_t load(const elem_t *p) { return *p; }
  __device__ static acc_t warp_sum(acc_t v) {
    // butterfly: every lane ends with identical bits (fp add commutes)
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v = __fadd_rn(v, __shfl_xor_sync(kFull, v, m));
    return v;
  }
  __device__ static elem_t to_elem(acc_t v) { return v; }
};

template <class Op, int BLOCK>
__device__ __forceinline__ typename Op::acc_t block_sum(typename Op::acc_t v) {
  using acc_t = typename Op::acc_t;
  constexpr int NW = BLOCK / 32;
  __shared__ acc_t warp_sums[NW];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = Op::warp_sum(v);
  if (lane == 0) warp_sums[warp] = v;
  __syncthreads();
  acc_t r = Op::zero();
  if (warp == 0) {
    r = Op::warp_sum(lane < NW ? warp_sums[lane] : Op::zero());
  }
  __syncthreads();  // warp_sums reusable by a second call
  return r;         // valid in warp 0
}

// Multi-GPU fused exchange (wf_reduce_sum_f32_mg): the last block of every
// rank writes its rank partial, tagged with the call's epoch, into slot
// [epoch & 1][rank] of EVERY rank's mailbox over peer memory (NVLink, CUDA IPC
// mappings), then waits for all ranks' slots in its own mailbox and folds them
// with the association of fold_kernel (so the result is bit-identical to the
// NCCL all-gather + wf_fold_f32 path, and identical on every rank).  Two banks
// by epoch parity: a rank can be at most one call ahead of a peer (it needs
// the peer's slot of the current call to finish it), so it never overwrites a
// slot the peer has not read yet.
struct MgArgs {
  unsigned long long *const *peers;  // [world] mailbox of each rank (device array)
  const unsigned long long *mine;    // this rank's mailbox
  int rank, world;
  uint32_t epoch;
};

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

#ifndef WF_PX_KEEP_MB
#define WF_PX_KEEP_MB 32  // pass 1 of the sharded scan: its last 32 MB read are marked evict_last, the rest evict_first
#endif
#ifndef WF_PX_REV
#define WF_PX_REV 1  // pass 1 of the sharded scan streams its shard backwards
#endif

// PX (i32 only): the last block also runs the peer exchange of wf_peer.cuh on
// the rank total (exclusive scan over ranks, mod 2^32), so out = {carry of
// this rank's shard, global total} — the sharded scan's pass 1 and its carry
// exchange in ONE kernel (wf_reduce_sum_i32_exscan_mg).
template <class Op, int BLOCK, int UNROLL, bool MG = false, bool PX = false, bool EARLY = false>
__global__ void __launch_bounds__(BLOCK)
    reduce_kernel(const typename Op::elem_t *__restrict__ in, uint64_t n,
                  typename Op::elem_t *__restrict__ out,
                  typename Op::acc_t *__restrict__ partials,
                  uint32_t *__restrict__ ticket, MgArgs mg = MgArgs{},
                  PeerArgs pa = PeerArgs{}) {
  using acc_t = typename Op::acc_t;
  using elem_t = typename Op::elem_t;
  const uint64_t gtid = uint64_t(blockIdx.x) * BLOCK + threadIdx.x;
  const uint64_t nthreads = uint64_t(gridDim.x) * BLOCK;
#if WF_RED_TRACE
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    RED_STAMP(blockIdx.x * 4ull, gtimer());
    RED_STAMP(blockIdx.x * 4ull + 2, smid);
  }
#endif
  // a dependent (EARLY) launch behind this one may start its streaming now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // head (scalar until 16 B alignment) | body (16 B vectors) | tail (scalar)
  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  uint64_t head = ((16u - (addr & 15u)) & 15u) / sizeof(elem_t);
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  const uint64_t tail0 = head + nvec * 4;
  const uint4 *vin = reinterpret_cast<const uint4 *>(in + head);

  acc_t acc[UNROLL][4];
#pragma unroll
  for (int u = 0; u < UNROLL; ++u)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[u][k] = Op::zero();

  // PX (pass 1 of the sharded scan) streams the shard from its END to its
  // start, so the lines read last — the shard's head, which the scan that
  // follows reads first — are the ones still in L2 when it starts (the i32
  // wrapping sum is order-free)
  auto vec_at = [&](uint64_t v) { return (PX && WF_PX_REV) ? vin + (nvec - 1 - v) : vin + v; };
  const uint64_t keep_vec = (uint64_t(WF_PX_KEEP_MB) << 20) / 16;
  uint64_t i = gtid;
  auto trip = [&](uint64_t i0) {  // UNROLL vectors per thread
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t v = i0 + u * nthreads;
      if (PX && WF_PX_KEEP_MB > 0)  // read last = the scan's first reads: keep; the rest: evict first
        q[u] = v + keep_vec >= nvec ? ldg_keep(vec_at(v)) : ldg_evict_first(vec_at(v));
      else
        q[u] = ldg_stream(vec_at(v));
    }
    // keep the trip's UNROLL loads ahead of their adds (the compiler may not
    // consume a load before the last one of the trip is issued)
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      asm volatile("" : "+r"(q[u].x), "+r"(q[u].y), "+r"(q[u].z), "+r"(q[u].w));
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      acc[u][0] = Op::add(acc[u][0], Op::from_bits(q[u].x));
      acc[u][1] = Op::add(acc[u][1], Op::from_bits(q[u].y));
      acc[u][2] = Op::add(acc[u][2], Op::from_bits(q[u].z));
      acc[u][3] = Op::add(acc[u][3], Op::from_bits(q[u].w));
    }
  };
  if constexpr (PX || !WF_RED_OUTER_UNROLL1) {
    // (the sharded scan's pass 1 keeps the compiler's unroll: with its
    // reversed, hinted loads it is 14 % faster that way, 23.3 vs 27.1 us
    // per 2^25 shard, tools/c3_shard_probe.py)
    for (; i + uint64_t(UNROLL - 1) * nthreads < nvec; i += UNROLL * nthreads) trip(i);
  } else {
#pragma unroll 1
    for (; i + uint64_t(UNROLL - 1) * nthreads < nvec; i += UNROLL * nthreads) trip(i);
  }
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {  // remainder: < UNROLL vectors left
    if (i < nvec) {
      const uint4 q = ldg_stream(vec_at(i));
      acc[u][0] = Op::add(acc[u][0], Op::from_bits(q.x));
      acc[u][1] = Op::add(acc[u][1], Op::from_bits(q.y));
      acc[u][2] = Op::add(acc[u][2], Op::from_bits(q.z));
      acc[u][3] = Op::add(acc[u][3], Op::from_bits(q.w));
      i += nthreads;
    }
  }
  if (gtid < head) acc[0][0] = Op::add(acc[0][0], Op::load(in + gtid));
  if (tail0 + gtid < n) acc[0][1] = Op::add(acc[0][1], Op::load(in + tail0 + gtid));

  // fixed pairwise fold of the 4*UNROLL chains
#pragma unroll
  for (int u = 0; u < UNROLL; ++u) {
    acc[u][0] = Op::add(Op::add(acc[u][0], acc[u][1]), Op::add(acc[u][2], acc[u][3]));
  }
#pragma unroll
  for (int s = 1; s < UNROLL; s <<= 1)
#pragma unroll
    for (int u = 0; u + s < UNROLL; u += 2 * s) acc[u][0] = Op::add(acc[u][0], acc[u + s][0]);

  const acc_t bsum = block_sum<Op, BLOCK>(acc[0][0]);
#if WF_RED_TRACE
  if (threadIdx.x == 0) RED_STAMP(blockIdx.x * 4ull + 1, gtimer());
#endif
  if constexpr (EARLY) {
    // the streaming above overlapped the previous grid's tail; the workspace
    // and the output are touched only once that grid has completed and flushed
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }

  if constexpr (PX) {
    __shared__ bool s_last;
    __shared__ uint32_t s_total;
    if (threadIdx.x == 0) {
      auto *word = reinterpret_cast<unsigned long long *>(ticket);
      const unsigned long long mine = (1ull << 48) | Op::bits(bsum);
      const unsigned long long old = atomicAdd(word, mine);
      s_last = (old >> 48) == gridDim.x - 1;
      if (s_last) {
        s_total = uint32_t(old + mine);
        *word = 0ull;
      }
    }
    __syncthreads();
    if (s_last) peer_exchange_block(kPeerExscanU32, nullptr, &s_total, 1, out, pa);
    return;
  }
  if (Op::kOrderFree) {
    // integer Σ is order-independent: ONE 64-bit atomic per block carries both
    // the block sum (low 48 bits: 32 bits of sum + up to 2^16 wraps) and an
    // arrival count (high 16 bits).  The block that sees count == grid-1 holds
    // the full sum in the returned value — no fence, no second atomic, no
    // separate ticket on the critical path of this latency-bound kernel.
    if (threadIdx.x == 0) {
      auto *word = reinterpret_cast<unsigned long long *>(ticket);
      const unsigned long long mine = (1ull << 48) | Op::bits(bsum);
      const unsigned long long old = atomicAdd(word, mine);
      if ((old >> 48) == gridDim.x - 1) {
        out[0] = Op::to_elem(Op::from_bits(uint32_t(old + mine)));
        *word = 0ull;  // next stream-ordered launch starts from zero
      }
    }
    return;
  }
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bsum;
    am_last = atom_add_acq_rel_gpu(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  // fixed-order fold of the block partials (thread t: t, t+BLOCK, ...)
  acc_t f = Op::zero();
  for (uint32_t j = threadIdx.x; j < gridDim.x; j += BLOCK) {
    f = Op::add(f, __ldcg(partials + j));
  }
  f = block_sum<Op, BLOCK>(f);
  if constexpr (MG) {
    __shared__ acc_t s_part;
    if (threadIdx.x == 0) {
      s_part = f;
      *ticket = 0u;
    }
    __syncthreads();
    const uint32_t bank = mg.epoch & 1u;
    const unsigned long long tag = (unsigned long long)mg.epoch << 32;
    if (int(threadIdx.x) < mg.world)  // one peer store per thread, all in flight at once
      st_relaxed_sys(mg.peers[threadIdx.x] + bank * mg.world + mg.rank, tag | Op::bits(s_part));
    acc_t v = Op::zero();
    if (int(threadIdx.x) < mg.world) {
      const unsigned long long *slot = mg.mine + bank * mg.world + threadIdx.x;
      unsigned long long w = ld_relaxed_sys(slot);
      uint32_t spins = 0;
      while (uint32_t(w >> 32) != mg.epoch) {
        if (++spins > (1u << 25)) {  // ~4 s: a peer never arrived
          w = tag | 0x7fc00000u;     // NaN marks the failure to the host
          break;
        }
        __nanosleep(128);
        w = ld_relaxed_sys(slot);
      }
      v = Op::add(Op::zero(), Op::from_bits(uint32_t(w)));
    }
    v = block_sum<Op, BLOCK>(v);  // fold_kernel's association for world <= 32
    if (threadIdx.x == 0) out[0] = Op::to_elem(v);
    return;
  }
  if (threadIdx.x == 0) {
    out[0] = Op::to_elem(f);
    *ticket = 0u;
#if WF_RED_TRACE
    RED_STAMP(gridDim.x * 4ull, gtimer());
    g_red_seq += 1;
#endif
  }
}

// Single-block fold with a fixed association (thread-strided chains, then the
// block tree), so a cross-GPU combine over ranks is deterministic and every
// rank computes identical bits.
template <class Op>
__global__ void __launch_bounds__(256)
    fold_kernel(const typename Op::elem_t *__restrict__ v, uint32_t count,
                typename Op::elem_t *__restrict__ out) {
  using acc_t = typename Op::acc_t;
  acc_t f = Op::zero();
  for (uint32_t j = threadIdx.x; j < count; j += 256) f = Op::add(f, Op::load(v + j));
  f = block_sum<Op, 256>(f);
  if (threadIdx.x == 0) out[0] = Op::to_elem(f);
}

__global__ void __launch_bounds__(256)
    fold_u64_kernel(const uint64_t *__restrict__ v, uint32_t count,
                    uint64_t *__restrict__ out) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long f = 0;
  for (uint32_t j = threadIdx.x; j < count; j += 256) f += v[j];
  atomicAdd(&s, f);
  __syncthreads();
  if (threadIdx.x == 0) out[0] = s;
}

#ifndef WF_RED_UNROLL
#define WF_RED_UNROLL 4  // 16-byte loads in flight per thread
#endif
constexpr int kUnroll = WF_RED_UNROLL;

// EARLY: a programmatic dependent launch (see the top of this file)
template <class Kernel, class... Args>
cudaError_t launch_pdl(Kernel k, int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <class Op, int BLOCK>
cudaError_t launch_block(const typename Op::elem_t *in, uint64_t n,
                         typename Op::elem_t *out, int grid, void *ws, bool early,
                         cudaStream_t s) {
  auto *ticket = reinterpret_cast<uint32_t *>(ws);
  auto *partials = reinterpret_cast<typename Op::acc_t *>(
      static_cast<char *>(ws) + kWsHeader);
  if (early)
    return launch_pdl(reduce_kernel<Op, BLOCK, kUnroll, false, false, true>, grid, BLOCK, s, in,
                      n, out, partials, ticket, MgArgs{}, PeerArgs{});
  reduce_kernel<Op, BLOCK, kUnroll>
      <<<grid, BLOCK, 0, s>>>(in, n, out, partials, ticket);
  return cudaGetLastError();
}

template <class Op>
cudaError_t launch_reduce(const typename Op::elem_t *in, uint64_t n,
                          typename Op::elem_t *out, int block, int grid,
                          void *ws, bool early, cudaStream_t s) {
  switch (block) {
    case 128: return launch_block<Op, 128>(in, n, out, grid, ws, early, s);
    case 256: return launch_block<Op, 256>(in, n, out, grid, ws, early, s);
    case 512: return launch_block<Op, 512>(in, n, out, grid, ws, early, s);
    case 1024: return launch_block<Op, 1024>(in, n, out, grid, ws, early, s);
    default: return cudaErrorInvalidValue;
  }
}

// Resident blocks per SM of the instantiation a launch actually uses (plain,
// dependent and fused forms differ in registers: sizing the sharded scan's
// pass-1 kernel from the plain K1's occupancy gave it two waves, 27 vs 23 us
// per 2^25 shard); the smaller of the stream-ordered and dependent forms.
template <class Op, int BLOCK, bool MG, bool PX>
int occupancy_blocks() {
  int b0 = 0, b1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b0, reduce_kernel<Op, BLOCK, kUnroll, MG, PX, false>, BLOCK, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b1, reduce_kernel<Op, BLOCK, kUnroll, MG, PX, true>, BLOCK, 0);
  const int b = b0 < b1 ? b0 : b1;
  return b > 0 ? b : 1;
}

template <class Op, bool MG, bool PX>
int resident_blocks(int block) {
  switch (block) {
    case 128: return occupancy_blocks<Op, 128, MG, PX>();
    case 256: return occupancy_blocks<Op, 256, MG, PX>();
    case 512: return occupancy_blocks<Op, 512, MG, PX>();
    default: return occupancy_blocks<Op, 1024, MG, PX>();
  }
}

template <int BLOCK>
cudaError_t launch_mg_block(const float *in, uint64_t n, float *out, int grid, void *ws,
                            const MgArgs &mg, bool early, cudaStream_t s) {
  auto *ticket = reinterpret_cast<uint32_t *>(ws);
  auto *partials = reinterpret_cast<float *>(static_cast<char *>(ws) + kWsHeader);
  if (early)
    return launch_pdl(reduce_kernel<SumF32, BLOCK, kUnroll, true, false, true>, grid, BLOCK, s,
                      in, n, out, partials, ticket, mg, PeerArgs{});
  reduce_kernel<SumF32, BLOCK, kUnroll, true><<<grid, BLOCK, 0, s>>>(in, n, out, partials,
                                                                     ticket, mg);
  return cudaGetLastError();
}

template <int BLOCK>
cudaError_t launch_px_block(const int32_t *in, uint64_t n, int32_t *out2, int grid, void *ws,
                            const PeerArgs &pa, bool early, cudaStream_t s) {
  auto *ticket = reinterpret_cast<uint32_t *>(ws);
  auto *partials = reinterpret_cast<uint32_t *>(static_cast<char *>(ws) + kWsHeader);
  if (early)
    return launch_pdl(reduce_kernel<SumI32, BLOCK, kUnroll, false, true, true>, grid, BLOCK, s,
                      in, n, out2, partials, ticket, MgArgs{}, pa);
  reduce_kernel<SumI32, BLOCK, kUnroll, false, true>
      <<<grid, BLOCK, 0, s>>>(in, n, out2, partials, ticket, MgArgs{}, pa);
  return cudaGetLastError();
}

}  // namespace

#if WF_RED_TRACE
extern "C" int wf_debug_set_trace_red(void *buf) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  unsigned int z = 0;
  cudaError_t e = cudaMemcpyToSymbol(g_red_trace, &p, sizeof(p));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_red_seq, &z, sizeof(z));
  return int(e);
}
#endif

cudaError_t launch_reduce_i32_exscan_mg(const int32_t *in, uint64_t n, int32_t *out2, int block,
                                        int grid, void *ws, void *const *peers, const void *mine,
                                        uint32_t cap, int rank, int world, uint32_t epoch,
                                        uint32_t *err, cudaStream_t s, bool early) {
  PeerArgs pa{reinterpret_cast<uint64_t *const *>(peers), static_cast<const uint64_t *>(mine),
              cap, rank, world, epoch, err};
  switch (block) {
    case 128: return launch_px_block<128>(in, n, out2, grid, ws, pa, early, s);
    case 256: return launch_px_block<256>(in, n, out2, grid, ws, pa, early, s);
    case 512: return launch_px_block<512>(in, n, out2, grid, ws, pa, early, s);
    case 1024: return launch_px_block<1024>(in, n, out2, grid, ws, pa, early, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce_f32_mg(const float *in, uint64_t n, float *out, int block, int grid,
                                 void *ws, void *const *peers, const void *mine, int rank,
                                 int world, uint32_t epoch, bool early, cudaStream_t s) {
  MgArgs mg;
  mg.peers = reinterpret_cast<unsigned long long *const *>(peers);
  mg.mine = static_cast<const unsigned long long *>(mine);
  mg.rank = rank;
  mg.world = world;
  mg.epoch = epoch;
  switch (block) {
    case 128: return launch_mg_block<128>(in, n, out, grid, ws, mg, early, s);
    case 256: return launch_mg_block<256>(in, n, out, grid, ws, mg, early, s);
    case 512: return launch_mg_block<512>(in, n, out, grid, ws, mg, early, s);
    case 1024: return launch_mg_block<1024>(in, n, out, grid, ws, mg, early, s);
    default: return cudaErrorInvalidValue;
  }
}

int auto_reduce_grid(int kind, int block, uint64_t n) {
  static int cache[4][11] = {};
  const int lg = block == 128 ? 7 : block == 256 ? 8 : block == 512 ? 9 : 10;
  int &per_sm = cache[kind & 3][lg];
  if (per_sm == 0) {
    switch (kind) {
      case kRedI32: per_sm = resident_blocks<SumI32, false, false>(block); break;
      case kRedF32:
      case kRedF32Mg: {
        // one grid for the plain and the fused-exchange K2: the fp32
        // association depends on the grid, and the fused result must be
        // bit-identical to the NCCL path's (plain K2 per rank + fold)
        const int a = resident_blocks<SumF32, false, false>(block);
        const int b = resident_blocks<SumF32, true, false>(block);
        per_sm = a < b ? a : b;
        break;
      }
      default: per_sm = resident_blocks<SumI32, false, true>(block); break;  // kRedI32Px
    }
  }
  uint64_t full = uint64_t(per_sm) * uint64_t(sm_count(current_device()));
  if (full > kMaxReduceGrid) full = kMaxReduceGrid;
  // enough blocks that each thread issues at least one UNROLL batch
  const uint64_t per_block = uint64_t(block) * kUnroll * 4;
  uint64_t need = (n + per_block - 1) / per_block;
  if (need < 1) need = 1;
  return int(need < full ? need : full);
}

cudaError_t launch_reduce_i32(const int32_t *in, uint64_t n, int32_t *out,
                              int block, int grid, void *ws, cudaStream_t s) {
  return launch_reduce<SumI32>(in, n, out, block, grid, ws, false, s);
}

cudaError_t launch_reduce_f32(const float *in, uint64_t n, float *out,
                              int block, int grid, void *ws, cudaStream_t s, bool early) {
  return launch_reduce<SumF32>(in, n, out, block, grid, ws, early, s);
}

cudaError_t launch_fold_f32(const float *v, uint32_t count, float *out,
                            cudaStream_t s) {
  fold_kernel<SumF32><<<1, 256, 0, s>>>(v, count, out);
  return cudaGetLastError();
}

cudaError_t launch_fold_i32(const int32_t *v, uint32_t count, int32_t *out,
                            cudaStream_t s) {
  fold_kernel<SumI32><<<1, 256, 0, s>>>(v, count, out);
  return cudaGetLastError();
}

cudaError_t launch_fold_u64(const uint64_t *v, uint32_t count, uint64_t *out,
                            cudaStream_t s) {
  fold_u64_kernel<<<1, 256, 0, s>>>(v, count, out);
  return cudaGetLastError();
}

cudaError_t preload_reduce_mg_kernels() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
  auto get = [&](const void *f) {
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, f);
  };
  get(reinterpret_cast<const void *>(reduce_kernel<SumI32, 128, kUnroll, false, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumI32, 256, kUnroll, false, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumI32, 512, kUnroll, false, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumI32, 1024, kUnroll, false, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumF32, 128, kUnroll, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumF32, 256, kUnroll, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumF32, 512, kUnroll, true>));
  get(reinterpret_cast<const void *>(reduce_kernel<SumF32, 1024, kUnroll, true>));
  return e;
}

}  // namespace wf
