// wf_scan_tmem.cu — K3 scan / K4 compaction: warp-specialised single-pass
// decoupled look-back with tiles PARKED IN TENSOR MEMORY while their prefix
// resolves.
//
// Why: the smem-stage kernel of wf_scan.cu holds each 32 KiB stage from its
// TMA load until the tile's prefix is known (~3 us after the latest
// predecessor landed), so only a fraction of the stages is ever loading and
// reads in flight cap at ~3 TB/s (profiles/r01_scan_compact_experiments.md).
// A first TMEM version that parked one tile per CTA but aggregated the next
// tile only after finishing the previous one measured slower (490 / 474 us):
// every aggregate then waited behind a prefix (convoy).  Here every role has
// its own warps and its own mbarrier pipeline, so a landed tile is reduced
// and published at once whatever the state of older tiles:
//
//   producer warp    claims tile ids (ticket, drawn one stage ahead) and
//                    TMA-loads them into a ring of S smem stages
//                    (cp.async.bulk + mbarrier complete_tx); ragged last tile
//                    by guarded copy
//   aggregator warps 0-3: LDS the landed stage once (the x[j][k] layout of the
//                    SDK shfl_scan), tcgen05.st it into one of P TMEM slots
//                    (64 columns = 32 KiB), release the stage, REDUX the tile
//                    value and publish its look-back descriptor at once
//   look-back warps  run the decoupled look-back over the tile descriptors
//                    (round-robin over tiles, so several resolve at once) and
//                    post each prefix into a 2P-entry ring
//   finisher warps   4-11, one per tile eighth: tcgen05.ld the tile back, free
//                    the slot, scan (SHFL.UP, 8 chunk chains interleaved) /
//                    ballot-compact (VOTE + POPC) it locally, then wait for
//                    the prefix and store (STG.128 for the scan)
//
// Hand-offs are mbarriers (full / empty per stage; parked / freed per slot;
// pref per ring entry), each with a phase per use, so no role ever waits on a
// CTA-wide barrier.
//
// Per SM (default: one CTA, S=6 stages, P=8 slots = all 512 TMEM columns,
// 6 look-back warps): 6 stages loading + 8 parked tiles = 448 KiB of tiles on
// chip, against 224 KiB for the smem-only kernel.
//
// Deadlock freedom: a CTA's tiles are claimed, aggregated, looked back and
// finished in claim order; the smallest unfinished tile in the grid has all
// predecessors finished, its CTA's older slots are free, so it progresses.
//
// Reference analog: as wf_scan.cu (corpus.py:347-364 warp-level scan; the
// block/grid carries the reference needs several launches for,
// runtime/hostdesc.py:109-129; compaction not expressible, dsl/lexer.py:18-25).
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"


#ifndef WF_TM_STAGES
#define WF_TM_STAGES 6  // smem stages per CTA (32 KiB each)
#endif
#ifndef WF_TM_SLOTS
#define WF_TM_SLOTS 8  // TMEM slots per CTA (64 columns each; power of two)
#endif
#ifndef WF_TM_NLB
#define WF_TM_NLB 3  // look-back warps per CTA (with 2 aggregator groups; tools/nag_sweep3.sh)
#endif
#ifndef WF_TM_NFG
#define WF_TM_NFG 1  // finisher groups (8 warps each), taking tiles round-robin
#endif
#ifndef WF_TM_MINB
#define WF_TM_MINB 1  // CTAs per SM the register budget must allow
#endif
#ifndef WF_LBK_TM
#define WF_LBK_TM 1  // scan look-back predecessors per lane (window = 32 * K tiles)
#endif
#ifndef WF_LBK_COMPACT_TM
#define WF_LBK_COMPACT_TM 1  // compaction look-back width (1: 277.7 vs 2: 281.6 us, tools/lbk_sweep.sh)
#endif

#ifndef WF_CMP_STCS
#define WF_CMP_STCS 0  // 1: compaction stores with the streaming (.cs) hint
#endif

#ifndef WF_TM_TRACE
#define WF_TM_TRACE 0
#endif

namespace wf {
#if WF_TM_TRACE
// per tile: [0] claimed+TMA issued  [1] aggregator start (landed, slot free)
// [2] parked  [3] prefix known  [4] finisher done (warp W_FIN)
__device__ unsigned long long *g_tm_trace = nullptr;
__device__ __forceinline__ void tm_stamp(uint32_t tile, int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (g_tm_trace) g_tm_trace[uint64_t(tile) * 5 + k] = t;
}
#define TM_STAMP(tile, k) tm_stamp(tile, k)
#else
#define TM_STAMP(tile, k)
#endif
namespace {

constexpr int S = WF_TM_STAGES;
constexpr int P = WF_TM_SLOTS;
constexpr int NLB = WF_TM_NLB;
constexpr int W_FIN = 4;                  // aggregators: warps 0-3, finishers 4-11
constexpr int NFG = WF_TM_NFG;
constexpr int NFIN = 8 * NFG;             // per group: one finisher warp per tile eighth
constexpr int W_LB = W_FIN + NFIN;        // look-back warps W_LB .. W_LB+NLB-1
constexpr int W_PROD = W_LB + NLB;        // producer warp
#ifndef WF_TM_NAG
#define WF_TM_NAG 2  // aggregator groups (4 warps each), taking stage items round-robin
#endif
constexpr int NAG = WF_TM_NAG;
constexpr int W_AGG2 = ((W_PROD + 1 + 3) / 4) * 4;  // 2nd group: warp % 4 = TMEM lane quarter
constexpr int TM_THREADS = (NAG == 2 ? W_AGG2 + 4 : W_PROD + 1) * 32;
constexpr uint32_t kExitOnly = 0xfffffffdu;  // second stop item (NAG = 2): just leave
#ifndef WF_TM_TMUL
#define WF_TM_TMUL 1  // tile = 32 KiB x TMUL
#endif
constexpr int TMUL = WF_TM_TMUL;
constexpr int QVEC = 16 * TMUL;           // 128-item chunks per warp-quarter of a tile
constexpr uint32_t TM_TILE = 4u * QVEC * 128;  // 8192 x TMUL items
constexpr uint32_t SLOT_COLS = 64u * TMUL;     // TMEM columns per parked tile
constexpr uint32_t TM_COLS = uint32_t(P) * SLOT_COLS;
constexpr uint32_t kNoTileTm = 0xffffffffu;
constexpr uint32_t kNoItem = 0xffffffffu;  // item_seq before the first publish
static_assert((P & (P - 1)) == 0 && TM_COLS <= 512, "TMEM slots: power of two, <= 512 cols");
static_assert(NLB >= 1 && NLB <= P, "look-back warps must not outnumber TMEM slots");
static_assert(NFG <= NLB, "every finisher group must see one of the NLB stop items");
static_assert(!(NAG == 2 && NFG > 1), "two aggregator groups with two finisher groups hang "
              "(tools/sweep_final.sh): not a supported combination");
// With two aggregator groups taking stage items round-robin, an odd stage
// count would hand one stage to both groups alternately: a group could then
// wait on that stage's mbarrier for a phase two ahead of the current one,
// which a parity wait reports as already complete (S = 5 hung,
// tools/sweep_final2.sh).  Even S keeps every stage (and, P being a power of
// two, every slot) with one group, so waiters are never more than one phase
// ahead.
static_assert(NAG == 1 || (S % 2 == 0 && P % 2 == 0),
              "two aggregator groups need an even number of stages and slots");

// ---- TMEM helpers (tcgen05, cta_group::1) --------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 consecutive columns of this thread's TMEM lane <- / -> 32 registers
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// named barrier over the 128 aggregator threads (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void agg_sync(uint32_t grp) {
  asm volatile("bar.sync %0, 128;" ::"r"(1u + grp) : "memory");
}

__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct TmShared {
  uint64_t full[S];    // producer -> aggregators: stage landed
  uint64_t empty[S];   // aggregators -> producer: stage read (4 arrivals)
  uint64_t parked[P];  // aggregators -> look-back + finishers: slot holds a tile
  uint64_t freed[P];   // finishers -> aggregators: slot read back (NFIN arrivals)
  uint64_t pref[2 * P];  // look-back -> finishers: prefix of item i known (ring by i % 2P)
  uint32_t stage_tile[S];
  uint32_t slot_tile[P];
  uint32_t slot_agg[P];
  uint32_t item_prefix[2 * P];  // prefix of item i at i % 2P (outlives the slot's reuse)
  // look-back copy of the slot metadata, by item (i % 2P): the look-back warp
  // of item i reads it after the slot may already hold item i + P; entry i is
  // only rewritten for item i + 2P, which cannot be parked before the
  // finishers have item i's prefix, i.e. after this warp read its entry
  uint32_t item_tile[2 * P];
  uint32_t item_agg[2 * P];
  uint32_t item_seq[2 * P];
  uint32_t slot_wtot[P][4][2];  // per tile quarter and half
  uint32_t tmem_base;
  uint32_t epoch;
};

// PX (compaction only): the finisher warp of the last tile also runs the
// offset exchange of wf_peer.cuh (peer_exscan_warp): count = {this rank's
// count, its global offset, the global total} — the sharded compaction and
// its exchange in ONE kernel (wf_compact_gt0_i32_mg).
template <bool COMPACT, bool PX = false>
__global__ void __launch_bounds__(TM_THREADS, WF_TM_MINB)
    tile_tmem_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out, uint64_t n,
                     uint32_t ntiles, const int32_t *__restrict__ carry_in,
                     uint64_t *__restrict__ count, uint64_t *__restrict__ desc,
                     TileHeader *__restrict__ hdr, uint32_t head, bool vec_out,
                     PeerArgs pa) {
  // `head` (0-3): the buffers were rounded down to 16 B, so virtual elements
  // [0, head) precede the caller's data; they read as 0 (neutral for the sum,
  // never selected) and are never stored.  Only tile 0 is affected.
  // `vec_out` false (scan output at a different 16-byte offset than the
  // input): every tile is stored with scalar stores.
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  __shared__ TmShared sh;
  int32_t *stages = reinterpret_cast<int32_t *>(dyn_smem);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (warp == 0) tmem_alloc(&sh.tmem_base, TM_COLS);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], 4);
    }
    for (int p = 0; p < P; ++p) {
      mbar_init(&sh.parked[p], 1);
      mbar_init(&sh.freed[p], 8);
    }
    for (int p = 0; p < 2 * P; ++p) mbar_init(&sh.pref[p], 1);
    fence_barrier_init();
  }
  // item ring: no entry holds a valid item index before its first publish
  // (shared memory keeps whatever an earlier CTA left there)
  if (threadIdx.x < 2 * P) sh.item_seq[threadIdx.x] = kNoItem;
  if (warp == W_PROD && lane == 0)
    sh.epoch = ld_volatile_u32(&hdr->epoch) & kEpochMask;  // before this CTA's first (release) draw
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t epoch = sh.epoch;

  if (warp == W_PROD) {
    // ------------------------------ producer ------------------------------
    // Tickets are drawn one stage ahead: the atomic's round trip overlaps the
    // wait for the next free stage instead of serialising with it.
    auto draw = [&](bool first) -> uint32_t {
      uint32_t t = first ? atom_add_acq_rel_gpu(&hdr->ticket, 1u) : atom_add_relaxed_gpu(&hdr->ticket, 1u);
      if (t >= ntiles) {
        if (t == ntiles + gridDim.x - 1) {  // last of all draws: reset for the next launch
          fence_acq_rel_gpu();
          atomicExch(&hdr->ticket, 0u);
          atomicExch(&hdr->epoch, (epoch + 1) & kEpochMask);
        }
        t = kNoTileTm;
      }
      return t;
    };
    uint32_t ahead = lane == 0 ? draw(true) : 0u;
    for (uint32_t i = 0;; ++i) {
      const int s = int(i % S);
      const uint32_t k = i / S;
      if (k > 0) mbar_wait(&sh.empty[s], (k - 1) & 1u);
      uint32_t t = ahead;
      if (lane == 0 && t != kNoTileTm) ahead = draw(false);
      t = __shfl_sync(kFull, t, 0);
      int32_t *stage = stages + s * TM_TILE;
      const uint64_t tbase = uint64_t(t) * TM_TILE;
      if (t != kNoTileTm && tbase + TM_TILE <= n) {  // (tile 0's masked head: aggregator)
        if (lane == 0) {
          sh.stage_tile[s] = t;
          TM_STAMP(t, 0);
          mbar_arrive_expect_tx(&sh.full[s], TM_TILE * 4);
          tma_load_1d(stage, in + tbase, TM_TILE * 4, &sh.full[s]);
        }
      } else {
        if (t != kNoTileTm)  // ragged last tile: guarded copy, zero padding
          for (uint32_t e = lane; e < TM_TILE; e += 32)
            stage[e] = (tbase + e < n && tbase + e >= head) ? in[tbase + e] : 0;
        __syncwarp();
        if (lane == 0) {
          sh.stage_tile[s] = t;
          mbar_arrive1(&sh.full[s]);
        }
      }
      if (t == kNoTileTm) {
        if (NAG == 2) {  // the other aggregator group's stop item
          const int s2 = int((i + 1) % S);
          const uint32_t k2 = (i + 1) / S;
          if (k2 > 0) mbar_wait(&sh.empty[s2], (k2 - 1) & 1u);
          if (lane == 0) {
            sh.stage_tile[s2] = kExitOnly;
            mbar_arrive1(&sh.full[s2]);
          }
        }
        break;
      }
    }
  } else if (warp < W_FIN || (NAG == 2 && warp >= W_AGG2)) {
    // ----------------------------- aggregators ----------------------------
    const uint32_t q = warp & 3u;  // tile quarter and TMEM lane quarter
    const uint32_t grp = (NAG == 2 && warp >= W_AGG2) ? 1u : 0u;
    const bool leader = warp == (grp ? uint32_t(W_AGG2) : 0u) && lane == 0;
    const uint32_t tcol = sh.tmem_base + ((32u * q) << 16);
    for (uint32_t i = grp;; i += NAG) {
      const int s = int(i % S), p = int(i % P);
      const uint32_t kp = i / P;
      mbar_wait(&sh.full[s], (i / S) & 1u);
      const uint32_t t = sh.stage_tile[s];
      if (t == kExitOnly) break;
      if (kp > 0) mbar_wait(&sh.freed[p], (kp - 1) & 1u);
      tc_fence_after();
      if (leader && t != kNoTileTm) TM_STAMP(t, 1);
      if (t == kNoTileTm) {
        // one stop item per look-back warp (items i .. i+NLB-1); the finishers
        // stop at the first.  Slot p is free (waited above); the next NLB-1
        // slots held items that the finishers have completed or will complete.
        for (uint32_t e = 0; e < uint32_t(NLB); ++e) {
          const uint32_t ie = i + e;
          const int pe = int(ie % P);
          if (e > 0 && ie / P > 0) mbar_wait(&sh.freed[pe], (ie / P - 1) & 1u);
          if (leader) {
            sh.slot_tile[pe] = kNoTileTm;
            sh.item_tile[ie % (2 * P)] = kNoTileTm;
            st_release_cta_smem(&sh.item_seq[ie % (2 * P)], ie);
            mbar_arrive1(&sh.parked[pe]);
          }
        }
        break;
      }
      const int32_t *stage = stages + s * TM_TILE + q * (QVEC * 128) + lane * 4;
      uint32_t hsum[2] = {0u, 0u};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int m = 0; m < TMUL; ++m) {
          uint32_t v[32], sum = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 x = *reinterpret_cast<const uint4 *>(stage + (8 * (TMUL * h + m) + j) * 128);
            if (head && t == 0 && q == 0 && h == 0 && m == 0 && j == 0 && lane == 0) {
              // the 0-3 virtual elements before the caller's data (the TMA
              // loaded the whole 16-byte-aligned tile)
              if (head > 0) x.x = 0;
              if (head > 1) x.y = 0;
              if (head > 2) x.z = 0;
            }
            v[4 * j] = x.x; v[4 * j + 1] = x.y; v[4 * j + 2] = x.z; v[4 * j + 3] = x.w;
            if (COMPACT)
              sum += (int32_t(x.x) > 0) + (int32_t(x.y) > 0) + (int32_t(x.z) > 0) + (int32_t(x.w) > 0);
            else
              sum += x.x + x.y + x.z + x.w;
          }
          tmem_st32(tcol + uint32_t(p) * SLOT_COLS + 32u * (TMUL * h + m), v);
          hsum[h] += sum;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&sh.empty[s]);  // this warp is done with the stage
      hsum[0] = __reduce_add_sync(kFull, hsum[0]);
      hsum[1] = __reduce_add_sync(kFull, hsum[1]);
      if (lane == 0) {
        sh.slot_wtot[p][q][0] = hsum[0];
        sh.slot_wtot[p][q][1] = hsum[1];
      }
      tmem_wait_st();
      tc_fence_before();
      agg_sync(grp);
      if (leader) {
        uint32_t a = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) a += sh.slot_wtot[p][w][0] + sh.slot_wtot[p][w][1];
        sh.slot_tile[p] = t;
        sh.slot_agg[p] = a;
        sh.item_tile[i % (2 * P)] = t;
        sh.item_agg[i % (2 * P)] = a;
        st_release_cta_smem(&sh.item_seq[i % (2 * P)], i);  // after tile / agg
        // publish the aggregate right here, not in the look-back warp: a
        // look-back warp busy with an older tile must never delay it
        if (t == 0) {
          const uint32_t c0 = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
          st_relaxed_gpu(desc, pack_desc(epoch, kStPrefix, c0 + a));
        } else {
          st_relaxed_gpu(desc + uint64_t(t) * kDescStride, pack_desc(epoch, kStAggregate, a));
        }
        TM_STAMP(t, 2);
        mbar_arrive1(&sh.parked[p]);
      }
    }
  } else if (warp < W_LB) {
    // ------------------------------ finishers -----------------------------
    // warp f handles tile eighth (q, h): TMEM lane quarter q = warp % 4 (the
    // only lanes it may read), columns 32*TMUL*h .. +32*TMUL of the slot
    const uint32_t q = warp & 3u, h = ((warp - W_FIN) >> 2) & 1u;
    const uint32_t grp = (warp - W_FIN) >> 3;
    const uint32_t tcol = sh.tmem_base + ((32u * q) << 16);
    const uint32_t lt = lanemask_lt();
    for (uint32_t i = grp;; i += NFG) {
      const int p = int(i % P);
      const uint32_t kp = i / P;
      mbar_wait(&sh.parked[p], kp & 1u);
      const uint32_t t = sh.slot_tile[p];
      if (t == kNoTileTm) break;
      tc_fence_after();
      // everything that does not need the prefix happens before waiting for
      // it: read the slot (metadata + TMEM), free it at once — the tile now
      // waits in this warp's registers, not in TMEM — and do the local scan /
      // ballot positions
      uint32_t wexcl = h ? sh.slot_wtot[p][q][0] : 0u;
#pragma unroll
      for (uint32_t w = 0; w < 4; ++w) wexcl += w < q ? sh.slot_wtot[p][w][0] + sh.slot_wtot[p][w][1] : 0u;
      const uint32_t agg = sh.slot_agg[p];
      uint32_t v[TMUL][32];
#pragma unroll
      for (int m = 0; m < TMUL; ++m) tmem_ld32(tcol + uint32_t(p) * SLOT_COLS + 32u * (TMUL * h + m), v[m]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&sh.freed[p]);
      const bool full = vec_out && uint64_t(t + 1) * TM_TILE <= n && (t > 0 || head == 0);
      const uint64_t base0 = uint64_t(t) * TM_TILE + q * (QVEC * 128) + (8 * TMUL * h) * 128 + lane * 4;
      uint32_t loc[TMUL][8];  // scan: chunk add (local); compaction: chunk write position (local)
      uint32_t run = 0;
#pragma unroll
      for (int m = 0; m < TMUL; ++m) {
        if (!COMPACT) {
          // the 8 chunk scans are independent until the carry: interleave them
          uint32_t sc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t *x = v[m] + 4 * j;
            x[1] += x[0];
            x[2] += x[1];
            x[3] += x[2];
            sc[j] = x[3];
          }
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t y = __shfl_up_sync(kFull, sc[j], d);
              if (lane >= uint32_t(d)) sc[j] += y;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            loc[m][j] = run + sc[j] - v[m][4 * j + 3];
            run += __shfl_sync(kFull, sc[j], 31);
          }
        } else {
          // ballot + popc positions (per-lane stores after the prefix; staging
          // in smem for 16-byte stores measured slower: 330 vs 290 us)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t *x = v[m] + 4 * j;
            uint32_t excl = 0, tot = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t b = __ballot_sync(kFull, int32_t(x[k]) > 0);
              excl += __popc(b & lt);
              tot += __popc(b);
            }
            loc[m][j] = run + excl;
            run += tot;
          }
        }
      }
      const int r = int(i % (2 * P));
      mbar_wait(&sh.pref[r], (i / (2 * P)) & 1u);
      const uint32_t prefix = sh.item_prefix[r];
      const uint32_t off = prefix + wexcl;
#pragma unroll
      for (int m = 0; m < TMUL; ++m) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t *x = v[m] + 4 * j;
          const uint64_t e = base0 + (8 * m + j) * 128;
          if (!COMPACT) {
            const uint32_t add = off + loc[m][j];
            if (full) {
              uint4 o;
              o.x = x[0] + add; o.y = x[1] + add; o.z = x[2] + add; o.w = x[3] + add;
              stg_stream(reinterpret_cast<uint4 *>(out + e), o);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (e + k < n && e + k >= head) out[e + k] = int32_t(x[k] + add);
            }
          } else {
            uint32_t pos = off + loc[m][j];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (int32_t(x[k]) > 0) {
#if WF_CMP_STCS
                __stcs(out + pos++, int32_t(x[k]));
#else
                out[pos++] = int32_t(x[k]);
#endif
              }
          }
        }
      }
      if constexpr (PX) {
        if (COMPACT && t == ntiles - 1 && q == 0 && h == 0) {
          const uint64_t total = uint64_t(prefix) + agg;
          if (lane == 0) *count = total;
          peer_exscan_warp(total, count + 1, pa);
        }
      } else {
        if (COMPACT && t == ntiles - 1 && q == 0 && h == 0 && lane == 0) *count = uint64_t(prefix) + agg;
      }
      if (q == 0 && h == 0 && lane == 0) TM_STAMP(t, 4);
    }
  } else if (warp < W_PROD) {
    // ----------------------------- look-back ------------------------------
    const uint32_t me = warp - W_LB;
    for (uint32_t i = me;; i += NLB) {
      const int p = int(i % P);
      const uint32_t kp = i / P;
      mbar_wait(&sh.parked[p], kp & 1u);
      // Look-back warps take items round-robin (NLB need not divide P), so the
      // previous use of this slot belonged to another warp; a parity wait
      // issued while that phase is still open passes early.  The item ring
      // entry carries the item index, written before the arrive: wait for it.
      // The acquire load pairs with the aggregator's release store, so the
      // tile / aggregate read below are the ones published with index i.
      const int ri = int(i % (2 * P));
      if (ld_acquire_cta_smem(&sh.item_seq[ri]) != i) {
        while (ld_acquire_cta_smem(&sh.item_seq[ri]) != i) __nanosleep(32);
      }
      const uint32_t t = sh.item_tile[ri];
      if (t == kNoTileTm) break;
      const uint32_t agg = sh.item_agg[ri];
      uint32_t excl;
      if (t == 0) {  // its prefix descriptor was published by the aggregator
        excl = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
      } else {
        excl = lookback_exclusive_wide<COMPACT ? WF_LBK_COMPACT_TM : WF_LBK_TM>(desc, t, epoch);
        if (lane == 0)
          st_relaxed_gpu(desc + uint64_t(t) * kDescStride, pack_desc(epoch, kStPrefix, excl + agg));
      }
      if (lane == 0) {
        const int r = int(i % (2 * P));
        sh.item_prefix[r] = excl;
        TM_STAMP(t, 3);
        mbar_arrive1(&sh.pref[r]);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(sh.tmem_base, TM_COLS);
  }
}

template <bool COMPACT>
constexpr size_t tm_smem() {
  return size_t(S) * TM_TILE * 4;
}

// Sets the dynamic-smem opt-in of the instantiation on the current device
// (per device, before every launch) and returns the persistent grid.
template <bool COMPACT, bool PX = false>
int tmem_grid(uint32_t ntiles) {
  static int per_sm[2] = {0, 0};
  static DeviceMask configured;
  configured.ensure([] {
    cudaFuncSetAttribute(tile_tmem_kernel<COMPACT, PX>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(tm_smem<COMPACT>()));
  });
  int &b = per_sm[COMPACT];
  if (b == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tile_tmem_kernel<COMPACT, PX>, TM_THREADS,
                                                  tm_smem<COMPACT>());
    if (b > int(512 / TM_COLS)) b = int(512 / TM_COLS);  // TMEM: 512 columns per SM
    if (b < 1) b = 1;
  }
  const uint32_t g = uint32_t(b) * uint32_t(sm_count(current_device()));
  return int(ntiles < g ? ntiles : g);
}

}  // namespace

#if WF_TM_TRACE
extern "C" int wf_debug_set_trace_tm(void *buf) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  return int(cudaMemcpyToSymbol(g_tm_trace, &p, sizeof(p)));
}
#endif

// `in` / `out` need only 4-byte alignment: the input is rounded down to 16 B
// and its 0-3 leading elements masked; a scan output at another 16-byte
// offset is written with scalar stores.
cudaError_t launch_scan_tmem_i32(const int32_t *in, int32_t *out, uint64_t n,
                                 const int32_t *carry, void *ws, cudaStream_t s) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  tile_tmem_kernel<false><<<tmem_grid<false>(nt), TM_THREADS, tm_smem<false>(), s>>>(
      in - head, out - head, nv, nt, carry, nullptr, desc, hdr, head,
      ((reinterpret_cast<uintptr_t>(in) ^ reinterpret_cast<uintptr_t>(out)) & 15u) == 0,
      PeerArgs{});
  return cudaGetLastError();
}

cudaError_t launch_compact_tmem_i32(const int32_t *in, uint64_t n, int32_t *out, uint64_t *count,
                                    void *ws, cudaStream_t s) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  tile_tmem_kernel<true><<<tmem_grid<true>(nt), TM_THREADS, tm_smem<true>(), s>>>(
      in - head, out, nv, nt, nullptr, count, desc, hdr, head, false, PeerArgs{});
  return cudaGetLastError();
}

// n >= 1.  counts3 = {count, global offset, global total}.
cudaError_t launch_compact_tmem_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                                       uint64_t *counts3, void *ws, const PeerArgs &pa,
                                       cudaStream_t s) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  tile_tmem_kernel<true, true><<<tmem_grid<true, true>(nt), TM_THREADS, tm_smem<true>(), s>>>(
      in - head, out, nv, nt, nullptr, counts3, desc, hdr, head, false, pa);
  return cudaGetLastError();
}

}  // namespace wf
