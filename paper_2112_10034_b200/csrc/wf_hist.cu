// wf_hist.cu — K5 histogram256_u8: shared-memory-privatised 256-bin byte
// histogram.
//
// Reference analog: none expressible (no u8 type, no atomics in the DSL,
// dsl/parser.py:83-88, dsl/lexer.py:18-25); under hierarchical collapsing a
// block's smem histogram becomes plain increments inside the block loop
// (one CPU thread runs the whole block).  On B200 the block's 1024 threads
// share ONE lane-banked sub-histogram in shared memory:
//
//     counter(bin b, lane l) at word b*32 + l        (256 x 32 x u32 = 32 KiB)
//
// Every lane of a warp updates its own bank, so one ATOMS.ADD warp
// instruction is bank-conflict-free whatever the data (uniform, all-equal,
// skewed); lanes of different warps that hit the same (bin, lane) word are
// serialised by the shared-memory atomic unit.  Input streams in as 16-byte
// vectors over a persistent grid.  At the end each block folds its 32 lane
// columns per bin (rotated reads, conflict-free) and adds them into 256
// uint64 accumulators in the workspace; the last block (atomic ticket) moves
// them to `bins` and re-zeroes the accumulators.
//
// Roofline: HBM, 1 B/elem read.
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"

namespace wf {
namespace {

constexpr int BLOCK = kHistBlock;
#ifndef WF_HIST_UNROLL
#define WF_HIST_UNROLL 3  // 16-byte loads in flight per thread (2: 674 us, 3: 652 us, 4: 653 us at 2^32)
#endif
constexpr int UNROLL = WF_HIST_UNROLL;

#if WF_HIST_PRMT
// Bin stride 256 B ([bin][64 words], lanes use the first 32): the byte
// offset of (bin, lane) is (bin << 8) | (lane << 2), which ONE byte permute
// assembles from the data word and lane*4 — PRMT + ATOMS per input byte
// instead of SHF + LOP3 + IADD + ATOMS (the 32 KiB layout).  Measured
// slower (686 vs 644 us at 2^32): the loop is bound by shared-atomic
// wavefronts, not issue, and the 256 B stride costs ~9 % extra wavefronts
// (146 M vs 134 M; the same 32 KiB code at WF_HIST_BINW=64 is as slow).
// Kept as the documented negative result (profiles/r01_hist_experiments.md).
constexpr uint32_t kBinWords = 64;
__device__ __forceinline__ void count_word(uint32_t *sh, uint32_t lane4, uint32_t w) {
  char *base = reinterpret_cast<char *>(sh);
  atomicAdd(reinterpret_cast<uint32_t *>(base + __byte_perm(w, lane4, 0x5504)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + __byte_perm(w, lane4, 0x5514)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + __byte_perm(w, lane4, 0x5524)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + __byte_perm(w, lane4, 0x5534)), 1u);
}
__device__ __forceinline__ void count_byte(uint32_t *sh, uint32_t lane4, uint32_t b) {
  atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(sh) + ((b << 8) | lane4)), 1u);
}
#elif WF_HIST_LOP3
// (default) 32 KiB layout, byte offset (bin << 7) | (lane << 2) formed by ONE
// 3-input LOP3 ((shifted word & 0x7f80) | lane*4: disjoint bits) after one
// shift, the smem base in the ATOMS's uniform-register operand: SHF + LOP3 +
// ATOMS per byte instead of SHF + LOP3 + IADD + ATOMS (the #else form).  The
// loop is bound by shared-atomic wavefronts, but under the board power cap
// fewer issued instructions per byte are measurably faster (2^32 bytes:
// uniform 645.6 -> 634.7 us, all-equal 692-751 -> 642-676 us, geometric
// 648-654 -> 628-647 us; alternating runs, tools/hist_probe.py)
constexpr uint32_t kBinWords = 32;
__device__ __forceinline__ void count_word(uint32_t *sh, uint32_t lane4, uint32_t w) {
  char *base = reinterpret_cast<char *>(sh);
  atomicAdd(reinterpret_cast<uint32_t *>(base + (((w << 7) & 0x7f80u) | lane4)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + (((w >> 1) & 0x7f80u) | lane4)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + (((w >> 9) & 0x7f80u) | lane4)), 1u);
  atomicAdd(reinterpret_cast<uint32_t *>(base + (((w >> 17) & 0x7f80u) | lane4)), 1u);
}
__device__ __forceinline__ void count_byte(uint32_t *sh, uint32_t lane4, uint32_t b) {
  atomicAdd(reinterpret_cast<uint32_t *>(reinterpret_cast<char *>(sh) + ((b << 7) | lane4)), 1u);
}
#else
constexpr uint32_t kBinWords = WF_HIST_BINW;
constexpr uint32_t kBinShift = WF_HIST_BINW == 64 ? 6 : 5;
__device__ __forceinline__ void count_word(uint32_t *col, uint32_t w) {
  atomicAdd(col + ((w & 0xffu) << kBinShift), 1u);
  atomicAdd(col + (((w >> 8) & 0xffu) << kBinShift), 1u);
  atomicAdd(col + (((w >> 16) & 0xffu) << kBinShift), 1u);
  atomicAdd(col + ((w >> 24) << kBinShift), 1u);
}
#endif

// PX: the last block runs the peer all-reduce of wf_peer.cuh on the rank's
// 256 bins, so `bins` receives the sum over all ranks — the sharded
// histogram and its bin exchange in ONE kernel (wf_histogram256_u8_mg).
//
// EARLY (the caller's WF_FLAG_INPUT_STABLE promise; a programmatic dependent
// launch, as K2 in wf_reduce.cu): the counting overlaps the previous grid's
// drain, and `griddepcontrol.wait` precedes the first workspace access.
template <bool PX, bool EARLY = false>
__global__ void __launch_bounds__(BLOCK, 2048 / BLOCK)
    hist256_kernel(const uint8_t *__restrict__ in, uint64_t n,
                   unsigned long long *__restrict__ bins, bool accumulate,
                   unsigned long long *__restrict__ accum,
                   uint32_t *__restrict__ ticket, PeerArgs pa) {
  // a dependent (EARLY) launch behind this one may start counting now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint32_t sh[];  // [256][kBinWords], lane l counts in word l
  for (uint32_t i = threadIdx.x; i < 256 * kBinWords; i += BLOCK) sh[i] = 0u;
  __syncthreads();

#if WF_HIST_PRMT || WF_HIST_LOP3
  const uint32_t lane4 = (threadIdx.x & 31) << 2;
#define WF_CNT4(w) count_word(sh, lane4, (w))
#define WF_CNT1(b) count_byte(sh, lane4, (b))
#else
  uint32_t *col = sh + (threadIdx.x & 31);
#define WF_CNT4(w) count_word(col, (w))
#define WF_CNT1(b) atomicAdd(col + (uint32_t(b) << kBinShift), 1u)
#endif
  const uint64_t gtid = uint64_t(blockIdx.x) * BLOCK + threadIdx.x;
  const uint64_t nthreads = uint64_t(gridDim.x) * BLOCK;

  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  uint64_t head = (16u - (addr & 15u)) & 15u;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 16;
  const uint64_t tail0 = head + nvec * 16;
  const uint4 *vin = reinterpret_cast<const uint4 *>(in + head);

  uint64_t i = gtid;
  for (; i + uint64_t(UNROLL - 1) * nthreads < nvec; i += UNROLL * nthreads) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(vin + i + u * nthreads);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      WF_CNT4(q[u].x);
      WF_CNT4(q[u].y);
      WF_CNT4(q[u].z);
      WF_CNT4(q[u].w);
    }
  }
  for (; i < nvec; i += nthreads) {
    const uint4 q = ldg_stream(vin + i);
    WF_CNT4(q.x);
    WF_CNT4(q.y);
    WF_CNT4(q.z);
    WF_CNT4(q.w);
  }
  if (gtid < head) WF_CNT1(in[gtid]);
  if (tail0 + gtid < n) WF_CNT1(in[tail0 + gtid]);
#undef WF_CNT4
#undef WF_CNT1
  __syncthreads();
  // EARLY: the counting overlapped the previous grid's drain; the workspace
  // (accumulators, ticket) and the bins only once it has completed
  if constexpr (EARLY) asm volatile("griddepcontrol.wait;" ::: "memory");

  // fold the 32 lane columns of each bin; rotation keeps the reads of a warp
  // on 32 distinct banks.  The fold is 64-bit: one block may count >= 2^32
  // copies of a byte (each lane column stays < 2^32 by the grid floor of
  // min_hist_grid, SURVEY.md §8d "a single bin can reach 2^32").
  if (threadIdx.x < 256) {
    const uint32_t b = threadIdx.x;
    unsigned long long s = 0;
#pragma unroll 8
    for (uint32_t l = 0; l < 32; ++l) s += sh[b * kBinWords + ((l + b) & 31u)];
    if (s) atomicAdd(accum + b, s);
  }
  __shared__ bool am_last;
  __syncthreads();
  if (threadIdx.x == 0) am_last = atom_add_acq_rel_gpu(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  if constexpr (PX) {
    __shared__ uint64_t s_bins[256];
    if (threadIdx.x < 256) s_bins[threadIdx.x] = atomicExch(accum + threadIdx.x, 0ull);
    if (threadIdx.x == 0) *ticket = 0u;
    __syncthreads();
    peer_exchange_block(kPeerAllreduce, s_bins, nullptr, 256, bins, pa);
    return;
  }
  if (threadIdx.x < 256) {
    const unsigned long long v = atomicExch(accum + threadIdx.x, 0ull);
    bins[threadIdx.x] = accumulate ? bins[threadIdx.x] + v : v;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

}  // namespace

// Grid floor that keeps every u32 (bin, lane) counter below 2^32: a lane
// column of a block counts the bytes of 32 threads, at most
// 32 * (ceil(nvec / threads) * 16 + 2) <= n / (32 * grid) + 576 for any data,
// so grid >= n / 2^36 bounds it by 2^31 + 576.
int min_hist_grid(uint64_t n) {
  const uint64_t g = (n + (uint64_t(1) << 36) - 1) >> 36;
  return int(g < 1 ? 1 : g);
}

int auto_hist_grid(uint64_t n) {
  static int per_sm = 0;
  if (per_sm == 0) {  // (32 KiB of dynamic smem needs no opt-in for the query)
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, hist256_kernel<false>, BLOCK, kHistSmem);
    per_sm = b > 0 ? b : 1;
  }
  const uint64_t full = uint64_t(per_sm) * uint64_t(sm_count(current_device()));
  const uint64_t per_block = uint64_t(BLOCK) * 16 * UNROLL * 4;
  uint64_t need = (n + per_block - 1) / per_block;
  if (need < 1) need = 1;
  const uint64_t g = need < full ? need : full;
  const uint64_t floor_g = uint64_t(min_hist_grid(n));
  return int(g > floor_g ? g : floor_g);
}

static void configure_hist(bool px) {
  static DeviceMask configured[2];
  configured[px].ensure([px] {
    if (px) {
      cudaFuncSetAttribute(hist256_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(kHistSmem));
      cudaFuncSetAttribute(hist256_kernel<true, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHistSmem));
    } else {
      cudaFuncSetAttribute(hist256_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(kHistSmem));
      cudaFuncSetAttribute(hist256_kernel<false, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHistSmem));
    }
  });
}

template <class Kernel, class... Args>
cudaError_t launch_hist_kernel(Kernel k, bool early, int grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(BLOCK);
  cfg.dynamicSmemBytes = kHistSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = early ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

cudaError_t launch_hist256(const uint8_t *in, uint64_t n, uint64_t *bins,
                           bool accumulate, int grid, void *ws,
                           cudaStream_t s, bool early) {
  auto *ticket = reinterpret_cast<uint32_t *>(ws);
  auto *accum = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + kWsHeader);
  configure_hist(false);
  auto *b = reinterpret_cast<unsigned long long *>(bins);
  return early ? launch_hist_kernel(hist256_kernel<false, true>, true, grid, s, in, n, b,
                                    accumulate, accum, ticket, PeerArgs{})
               : launch_hist_kernel(hist256_kernel<false>, false, grid, s, in, n, b, accumulate,
                                    accum, ticket, PeerArgs{});
}

cudaError_t launch_hist256_mg(const uint8_t *in, uint64_t n, uint64_t *bins, int grid, void *ws,
                              void *const *peers, const void *mine, uint32_t cap, int rank,
                              int world, uint32_t epoch, uint32_t *err, cudaStream_t s,
                              bool early) {
  auto *ticket = reinterpret_cast<uint32_t *>(ws);
  auto *accum = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + kWsHeader);
  configure_hist(true);
  PeerArgs pa{reinterpret_cast<uint64_t *const *>(peers), static_cast<const uint64_t *>(mine),
              cap, rank, world, epoch, err};
  auto *b = reinterpret_cast<unsigned long long *>(bins);
  return early ? launch_hist_kernel(hist256_kernel<true, true>, true, grid, s, in, n, b, false,
                                    accum, ticket, pa)
               : launch_hist_kernel(hist256_kernel<true>, false, grid, s, in, n, b, false, accum,
                                    ticket, pa);
}

cudaError_t preload_hist_mg_kernels() {
  configure_hist(true);
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, hist256_kernel<true>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, hist256_kernel<true, true>);
  return e;
}

}  // namespace wf
