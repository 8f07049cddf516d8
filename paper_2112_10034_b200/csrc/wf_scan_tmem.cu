// wf_scan_tmem.cu — K3 scan / K4 compaction: warp-specialised single-pass
// scan with tiles PARKED IN TENSOR MEMORY while their prefix resolves.
//
// Why: a kernel that holds each 32 KiB smem stage from its TMA load until the
// tile's prefix is known keeps only a fraction of the stages loading, so reads
// cap at ~3 TB/s (profiles/r01_scan_compact_experiments.md).  Here every role
// has its own warps and its own mbarrier pipeline, so a landed tile is
// reduced and published at once whatever the state of older tiles:
//
//   producer warp    claims tile ids (one ticket per tile, the next ticket
//                    examined only when needed) and TMA-loads them into a
//                    ring of S smem stages (cp.async.bulk + mbarrier
//                    complete_tx); ragged last tile by guarded copy
//   aggregator warps two groups of 4 taking stage items alternately: LDS the
//                    landed stage once (the x[j][k] layout of the SDK
//                    shfl_scan), tcgen05.st it into one of P TMEM slots
//                    (64 columns = 32 KiB), release the stage, REDUX the tile
//                    value and publish its aggregate at once
//   sweeper warp     (CTA 0 only) reads the published aggregates in tile
//                    order, 256 per L2 round trip, and publishes every tile's
//                    exclusive prefix: no per-tile look-back
//                    (WF_TM_SWEEP=0 builds a decoupled look-back instead)
//   waiter warp      watches the prefixes of the CTA's parked tiles (one lane
//                    per item, all polled in the same round trip) and posts
//                    them to the finishers
//   finisher warps   4-11, one per tile eighth: tcgen05.ld the tile back, free
//                    the slot, scan (SHFL.UP, 8 chunk chains interleaved) /
//                    compact (packed per-chunk counts, one pair of warp
//                    scans) it locally, then wait for the prefix and store
//                    (STG.128 for the scan)
//
// Hand-offs are mbarriers (full / empty per stage; parked / freed per slot;
// pref per ring entry), each with a phase per use, so no role ever waits on a
// CTA-wide barrier.
//
// Per SM (default: one CTA, S=4 stages, P=8 slots = all 512 TMEM columns):
// 4 stages loading + 8 parked tiles = 384 KiB of tiles on chip.  Per-role
// cycle accounting (-DWF_TM_PROF=1, tools/prof_tmem.py) and per-tile traces
// (-DWF_TM_TRACE=1, tools/trace_tmem.py, tools/trace_sweep.py) drove the
// current split: profiles/r02_scan_compact.md.
//
// Deadlock freedom: a CTA's tiles are claimed, aggregated, resolved and
// finished in claim order; the smallest unfinished tile in the grid has all
// predecessors finished (their aggregates are published, so the sweeper
// reaches it), its CTA's older slots are free, so it progresses.
//
// Reference analog: corpus.py:347-364 (warp-level scan); the block/grid
// carries the reference needs several launches for, runtime/hostdesc.py:
// 109-129; compaction is not expressible (dsl/lexer.py:18-25).
#include "wf_device.cuh"
#include "wf_internal.h"
#include "wf_peer.cuh"


#ifndef WF_TM_STAGES
#define WF_TM_STAGES 4  // smem stages per CTA (32 KiB each; 4 vs 6: 248 vs 250 us compaction, tools/tm_sweep.sh)
#endif
#ifndef WF_TM_SLOTS
#define WF_TM_SLOTS 8  // TMEM slots per CTA (64 columns each; power of two)
#endif
#ifndef WF_TM_SWEEP
#define WF_TM_SWEEP 1  // 1: one grid-wide prefix sweeper + one waiter warp per CTA; 0: per-tile look-back
#endif
#ifndef WF_TM_NLB
#if WF_TM_SWEEP
#define WF_TM_NLB 1  // the waiter warp
#else
#define WF_TM_NLB 3  // look-back warps per CTA (with 2 aggregator groups; tools/nag_sweep3.sh)
#endif
#endif
#ifndef WF_SWEEP_K
#define WF_SWEEP_K 8  // the sweeper reads 32 * K aggregates per round trip (4 / 8 / 16 / 32: 274 / 248 / 271 / 363 us)
#endif
#ifndef WF_TM_BATCH
#define WF_TM_BATCH 1  // consecutive tiles claimed per ticket draw (2 / 4 measured slower)
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

#ifndef WF_TM_PREFETCH
#define WF_TM_PREFETCH 1  // L2 prefetch of the first S tiles per CTA before griddepcontrol.wait
#endif

#ifndef WF_CMP_PK
#define WF_CMP_PK 1  // compaction: aggregators hand the packed per-chunk counts to the finishers
#endif

#ifndef WF_CMP_CHUNK_SKIP
#define WF_CMP_CHUNK_SKIP 1  // compaction: skip the stores of chunks with nothing selected (uniform branch)
#endif

#ifndef WF_CMP_STCS
#define WF_CMP_STCS 0  // 1: compaction stores with the streaming (.cs) hint
#endif

#ifndef WF_TM_TRACE
#define WF_TM_TRACE 0
#endif

namespace wf {
#ifndef WF_TM_PROF
#define WF_TM_PROF 0
#endif
#if WF_TM_PROF
// per CTA, 16 counters: [0..4] finisher (warp W_FIN lane 0) cycles waiting parked, TMEM read +
// free, local work, waiting prefix, stores; [5] finisher items; [6..8] aggregator leader
// (group 0) waiting full, waiting freed, work; [9] its items; [10,11] producer waiting
// empty, issuing; [12] producer items
__device__ unsigned long long *g_tm_prof = nullptr;
#define PROF_T(v) unsigned long long v = clock64()
#define PROF_ADD(k, a, b) (acc[k] += (b) - (a))
#else
#define PROF_T(v)
#define PROF_ADD(k, a, b)
#endif
#if WF_TM_TRACE
// per tile: [0] claimed+TMA issued  [1] aggregator start (landed, slot free)
// [2] parked  [3] prefix known  [4] finisher done (warp W_FIN)
// [5] look-back warp picked the item up  [6] look-back polls  [7] SM id
constexpr int kTmTraceWords = 8;
__device__ unsigned long long *g_tm_trace = nullptr;
__device__ __forceinline__ void tm_stamp(uint32_t tile, int k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (g_tm_trace) g_tm_trace[uint64_t(tile) * kTmTraceWords + k] = t;
}
__device__ __forceinline__ void tm_put(uint32_t tile, int k, unsigned long long v) {
  if (g_tm_trace) g_tm_trace[uint64_t(tile) * kTmTraceWords + k] = v;
}
#define TM_STAMP(tile, k) tm_stamp(tile, k)
#define TM_PUT(tile, k, v) tm_put(tile, k, v)
// sweeper iterations: [2 j] = globaltimer at the start of iteration j, [2 j + 1] = f | ready << 32
__device__ unsigned long long *g_sweep_trace = nullptr;
__device__ uint32_t g_sweep_cap = 0;
#else
#define TM_STAMP(tile, k)
#define TM_PUT(tile, k, v)
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
constexpr int W_SWEEP = W_PROD + 1;       // prefix sweeper (CTA 0 only; WF_TM_SWEEP)
#ifndef WF_TM_NAG
#define WF_TM_NAG 2  // aggregator groups (4 warps each), taking stage items round-robin
#endif
constexpr int NAG = WF_TM_NAG;
constexpr int W_AGG2 = ((W_PROD + 1 + 3) / 4) * 4;  // 2nd group: warp % 4 = TMEM lane quarter
constexpr int W_TOTAL = W_SWEEP + 1;  // CX round totaler (CTA 0): the idle warp before W_AGG2
constexpr int TM_THREADS = (NAG == 2 ? W_AGG2 + 4 : (WF_TM_SWEEP ? W_SWEEP + 1 : W_PROD + 1)) * 32;
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
constexpr uint32_t kBatch = WF_TM_BATCH;
constexpr uint32_t kNoItem = 0xffffffffu;  // item_seq before the first publish
static_assert((P & (P - 1)) == 0 && TM_COLS <= 512, "TMEM slots: power of two, <= 512 cols");
static_assert(TM_TILE == kTmemTile, "wf_internal.h kTmemTile: the block-cyclic scan's tile unit");
static_assert(NLB >= 1 && NLB <= P, "look-back warps must not outnumber TMEM slots");
static_assert(!WF_TM_SWEEP || (NLB == 1 && (NAG == 1 || W_SWEEP < W_AGG2)),
              "the sweeper warp sits in the gap before the second aggregator group");
// stop items: one per look-back warp and one per finisher group
constexpr int NSTOP = NLB > NFG ? NLB : NFG;
static_assert(NSTOP <= P, "stop items must fit the TMEM slots");
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
// issue only: the registers are valid after tmem_wait_ld()
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
}
// completes the loads issued by tmem_ld32; the registers are operands so no
// use of them can be scheduled before the wait
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                 "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                 "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                 "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
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
  uint32_t item_posted[2 * P];  // waiter: item whose prefix was posted at this ring entry
  uint32_t slot_wtot[P][4][2];  // per tile quarter and half
#if WF_CMP_PK
  // compaction: each lane's selected count per 128-element chunk (0-4), 4
  // chunks per byte-packed word, written by the aggregators with the slot so
  // the finisher does not recount: [slot][quarter][half * TMUL + m][word][lane]
  // (0-4 % selectivity 172 -> 162 us, 1 % 200 -> 181 us, 50 % unchanged at
  // 2^28; also moving the pair of warp scans into the aggregators made them
  // the slower stage: 50 % 241 -> 250 us, tools/c4_sel_probe.py)
  uint32_t slot_pk[P][4][2 * TMUL][2][32];
#endif
  uint32_t cx_wtot[2][2][4];  // CX aggregators: [group][item parity][warp] quarter sums
  uint32_t tmem_base;
  uint32_t epoch;
};

// sweeper layout: aggregates desc[0, ntiles), exclusive prefixes from
// desc[pref_offset) on, both one u64 per tile (the workspace holds 128 B per
// 4096 elements, far more)
__device__ __forceinline__ uint32_t pref_offset(uint32_t ntiles) { return (ntiles + 15u) & ~15u; }

// CX sweeper (one warp, CTA 0; tile_tmem_kernel's CX note).  Mailbox word of
// (bank, source rank, round): bank * world * cap + src * cap + round, holding
// {(0x80000000 | epoch) << 32 | value} — one 64-bit store carries tag and
// value together.  This rank's round-r prefixes need only the totals of the
// LOWER ranks' round r (and every rank's earlier rounds), not its own: the
// round is swept as its aggregates arrive, exactly like the plain sweeper, and
// its total is published when the round ends.
static __device__ __forceinline__ uint32_t cx_poll(const PeerArgs &pa, uint64_t bank,
                                                   uint32_t src, uint32_t round, uint32_t tag,
                                                   bool &failed) {
  if (failed) return 0u;  // one missing peer costs one timeout, not one per round
  const uint64_t *slot = pa.mine + bank + src * pa.cap + round;
  uint64_t w = peer_ld_relaxed_sys(slot);
  uint32_t spins = 0;
  while (uint32_t(w >> 32) != tag) {
    if (++spins > (1u << 25)) {  // ~4 s: a peer never arrived
      failed = true;
      return 0u;
    }
    __nanosleep(64);
    w = peer_ld_relaxed_sys(slot);
  }
  return uint32_t(w);
}

// Round totaler: sum the round's aggregates as they arrive, publish.
static __device__ __noinline__ void cx_totals(const uint64_t *desc, uint32_t ntiles,
                                              uint32_t epoch, const PeerArgs pa,
                                              uint32_t round_tiles, uint32_t rounds) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t tag_agg = uint32_t(pack_desc(epoch, kStAggregate, 0u) >> 32);
  const uint32_t world = uint32_t(pa.world), rank = uint32_t(pa.rank);
  const uint64_t bank = uint64_t(pa.epoch & 1u) * world * pa.cap;
  const uint32_t tag = 0x80000000u | pa.epoch;  // cx_sweep
  constexpr int K = WF_SWEEP_K;
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint32_t t0 = r * round_tiles < ntiles ? r * round_tiles : ntiles;
    const uint32_t t1 = t0 + round_tiles < ntiles ? t0 + round_tiles : ntiles;
    uint32_t part = 0, backoff = 32;
    for (uint32_t f = t0; f < t1;) {
      uint64_t d[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t idx = f + lane + 32u * k;
        d[k] = idx < t1 ? ld_relaxed_gpu(desc + idx) : 0ull;
      }
      uint32_t ready = 0;
      bool gap = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t bal = __ballot_sync(kFull, uint32_t(d[k] >> 32) == tag_agg);
        if (!gap) {
          const uint32_t take = bal == kFull ? 32u : uint32_t(__ffs(~bal)) - 1u;
          if (lane < take) part += uint32_t(d[k]);
          ready += take;
          gap = take < 32u;
        }
      }
      if (ready == 0) {
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
        continue;
      }
      backoff = 32;
      f += ready;
    }
    // the 64-bit word is self-contained (tag and value) and nothing else is
    // read through it: a relaxed system-scope store, no release fence
    const uint64_t word = (uint64_t(tag) << 32) | __reduce_add_sync(kFull, part);
    for (uint32_t q = lane; q < world; q += 32)
      peer_st_relaxed_sys(pa.peers[q] + bank + rank * pa.cap + r, word);
  }
}

static __device__ __noinline__ void cx_sweep(const uint64_t *desc_c, uint32_t ntiles,
                                             uint32_t epoch, const PeerArgs pa,
                                             uint32_t round_tiles, uint32_t rounds) {
  uint64_t *desc = const_cast<uint64_t *>(desc_c);
  uint64_t *pref = desc + pref_offset(ntiles);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t tag_agg = uint32_t(pack_desc(epoch, kStAggregate, 0u) >> 32);
  const uint32_t world = uint32_t(pa.world), rank = uint32_t(pa.rank);
  const uint64_t bank = uint64_t(pa.epoch & 1u) * world * pa.cap;
  const uint32_t tag = 0x80000000u | pa.epoch;
  constexpr int K = WF_SWEEP_K;
  uint32_t before = 0;  // every rank's totals of the rounds done (wrapping i32 sum)
  bool failed = false;
  for (uint32_t r = 0; r < rounds; ++r) {
    const uint32_t t0 = r * round_tiles < ntiles ? r * round_tiles : ntiles;
    const uint32_t t1 = t0 + round_tiles < ntiles ? t0 + round_tiles : ntiles;
    // the lower ranks' totals of this round (lane q polls rank q)
    uint32_t lower = 0;
    for (uint32_t q = lane; q < rank; q += 32) lower += cx_poll(pa, bank, q, r, tag, failed);
    lower = __reduce_add_sync(kFull, lower);
    failed = __any_sync(kFull, failed);
    // sweep this rank's tiles of the round as their aggregates arrive
    const uint32_t start = before + lower;
    uint32_t run = start, backoff = 32;
    for (uint32_t f = t0; f < t1;) {
      uint64_t d[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t idx = f + lane + 32u * k;
        d[k] = idx < t1 ? ld_relaxed_gpu(desc + idx) : 0ull;
      }
      uint32_t v[K], ready = 0;
      bool ok[K], gap = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ok[k] = uint32_t(d[k] >> 32) == tag_agg;
        v[k] = uint32_t(d[k]);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t b = __ballot_sync(kFull, ok[k]);
        if (!gap) {
          if (b == kFull) {
            ready += 32;
          } else {
            ready += uint32_t(__ffs(~b)) - 1u;
            gap = true;
          }
        }
      }
      if (ready == 0) {
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
        continue;
      }
      backoff = 32;
      uint32_t sc[K];
#pragma unroll
      for (int k = 0; k < K; ++k) sc[k] = 32u * k + lane < ready ? v[k] : 0u;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t y = __shfl_up_sync(kFull, sc[k], dd);
          if (lane >= uint32_t(dd)) sc[k] += y;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t j = 32u * k + lane;
        if (j < ready) st_relaxed_gpu(pref + f + j, pack_desc(epoch, kStPrefix, run + sc[k] - v[k]));
        run += __shfl_sync(kFull, sc[k], 31);
      }
      f += ready;
    }
    // the next round starts after every other rank's total of this one (this
    // rank's own is `run - start`; the totaler publishes it for the others)
    uint32_t others = 0;
    for (uint32_t q = lane; q < world; q += 32)
      if (q != rank) others += cx_poll(pa, bank, q, r, tag, failed);
    others = __reduce_add_sync(kFull, others);
    failed = __any_sync(kFull, failed);
    before = run + others - lower;
  }
  if (failed && lane == 0) *pa.err = 1u;
}

// PX (compaction only): the finisher warp of the last tile also runs the
// offset exchange of wf_peer.cuh (peer_exscan_warp): count = {this rank's
// count, its global offset, the global total} — the sharded compaction and
// its exchange in ONE kernel (wf_compact_gt0_i32_mg).
//
// CX (scan only): the cross-rank single-pass scan of a BLOCK-CYCLIC sharded
// array.  Global super-tile g (round_tiles tiles) lives on rank g % world as
// its local super-tile g / world, so this rank's local super-tile s is global
// super-tile s * world + rank.  The sweeper sums the aggregates of each local
// super-tile, all-gathers the round's totals over peer memory (one u64
// {epoch, value} word per rank and round, wf_peer.cuh mailbox, bank by epoch
// parity), and publishes every tile's prefix = (all ranks' totals of earlier
// rounds) + (lower ranks' totals of this round) + its local prefix.  Every
// element is read once and written once (8 B/elem, against the 12 B of
// reduce-then-scan), and no rank waits for another rank's whole shard — only
// for its same-round super-tile.  Deadlock freedom needs every claimed tile's
// aggregate published without a free TMEM slot: CX aggregators sum a landed
// stage and publish before they wait for the slot (a round's last tile can
// otherwise be stuck in a stage whose CTA's slots all hold tiles of the same
// round).  `rounds` is the same on every rank (ranks with fewer local
// super-tiles contribute 0).
template <bool COMPACT, bool PX = false, bool CX = false>
__global__ void __launch_bounds__(TM_THREADS, WF_TM_MINB)
    tile_tmem_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out, uint64_t n,
                     uint32_t ntiles, const int32_t *__restrict__ carry_in,
                     uint64_t *__restrict__ count, uint64_t *__restrict__ desc,
                     TileHeader *__restrict__ hdr, uint32_t head, bool vec_out,
                     PeerArgs pa, uint32_t round_tiles, uint32_t rounds) {
  static_assert(!CX || (!COMPACT && !PX && WF_TM_SWEEP && NAG == 2 && W_TOTAL < W_AGG2),
                "CX: the sweeper scan only, with a spare warp for the round totals");
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
  if (threadIdx.x < 2 * P) {
    sh.item_seq[threadIdx.x] = kNoItem;
    sh.item_posted[threadIdx.x] = kNoItem;
  }
  // a programmatic dependent launch behind this one may start its loads now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // Early L2 prefetch of the first tiles: between them, the CTAs warm L2 with
  // tiles [0, S * grid) — exactly the tiles the first claims will take —
  // before anything touches the workspace.  For a programmatic dependent
  // launch (the caller's WF_FLAG_INPUT_STABLE promise: the previous kernel on
  // the stream does not write `in`) these reads overlap the previous grid's
  // drain.  Only a hint: claims stay dynamic (ticket order), so no tile is
  // ever owned by a CTA that is not running, and a grid that is only partly
  // resident (other kernels on the GPU) still makes progress.
  if (WF_TM_PREFETCH && warp == W_PROD && lane == 0)
    for (uint32_t i = 0; i < uint32_t(S); ++i) {
      const uint64_t t = uint64_t(blockIdx.x) + uint64_t(i) * gridDim.x;
      if ((t + 1) * TM_TILE > n) break;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(in + t * TM_TILE),
                   "r"(TM_TILE * 4u)
                   : "memory");
    }
  // Nothing below touches the workspace, the carry or the outputs before the
  // previous grid on the stream has completed and flushed (returns at once
  // for an ordinary stream-ordered launch).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // The CTA's first ticket draw returns the launch epoch with it: the header
  // is one 64-bit word {epoch | ticket}, so one L2 round trip instead of an
  // epoch read ordered before the draw (a draw can only see this launch's
  // epoch: the reset for the next launch needs every CTA's last draw, and
  // this one precedes that CTA's last)
  uint64_t *const hdr64 = reinterpret_cast<uint64_t *>(hdr);
  uint32_t first = 0;
  if (warp == W_PROD && lane == 0) {
    const uint64_t w = atom_add_relaxed_gpu_u64(hdr64, kBatch);
    first = uint32_t(w);
    sh.epoch = uint32_t(w >> 32) & kEpochMask;
  }
  __syncthreads();
  const uint32_t epoch = sh.epoch;

  if (warp == W_PROD) {
    // ------------------------------ producer ------------------------------
    // Tiles are claimed in batches of B consecutive tiles per ticket (one
    // atomicAdd(ticket, B)), and the next batch's ticket is drawn when the
    // current batch starts and examined only when it is needed: the atomic's
    // L2 round trip (~1 us under full HBM load) never sits between a stage
    // becoming free and its TMA load.  (One tile per draw, examined at once,
    // capped the CTA at one tile per round trip: ~140 tiles/us grid-wide.)
    const uint32_t nbatches = (ntiles + kBatch - 1) / kBatch;
    auto failing = [&](uint32_t base) {  // each CTA examines exactly one failing draw
      if (base == (nbatches + gridDim.x - 1) * kBatch) {  // last of all draws: reset for the next launch
        fence_acq_rel_gpu();
        atomicExch(reinterpret_cast<unsigned long long *>(hdr64),
                   (unsigned long long)((epoch + 1) & kEpochMask) << 32);
      }
    };
    uint32_t cur = first;
    uint32_t nxt = 0, j = 0;
#if WF_TM_PROF
    unsigned long long acc[3] = {0, 0, 0};
#endif
    for (uint32_t i = 0;; ++i) {
      const int s = int(i % S);
      const uint32_t k = i / S;
      PROF_T(p0);
      if (k > 0) mbar_wait(&sh.empty[s], (k - 1) & 1u);
      PROF_T(p1);
      uint32_t t = kNoTileTm;
      if (lane == 0) {
        if (j == 0) {
          if (cur >= ntiles) {
            failing(cur);
          } else {
            nxt = uint32_t(atom_add_relaxed_gpu_u64(hdr64, kBatch));  // examined at the end of this batch
            t = cur;
          }
        } else {
          t = cur + j < ntiles ? cur + j : kNoTileTm;
          if (t == kNoTileTm) failing(nxt);  // ragged last batch: the draw behind it failed
        }
        if (t != kNoTileTm && ++j == kBatch) {
          cur = nxt;
          j = 0;
        }
      }
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
#if WF_TM_PROF
      PROF_T(p2);
      PROF_ADD(0, p0, p1);
      PROF_ADD(1, p1, p2);
      acc[2] += 1;
      if (t == kNoTileTm && lane == 0 && g_tm_prof)
        for (int q = 0; q < 3; ++q) g_tm_prof[blockIdx.x * 16 + 10 + q] = acc[q];
#endif
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
#if WF_TM_PROF
    unsigned long long acc[4] = {0, 0, 0, 0};
#endif
    for (uint32_t i = grp;; i += NAG) {
      const int s = int(i % S), p = int(i % P);
      const uint32_t kp = i / P;
      PROF_T(g0);
      mbar_wait(&sh.full[s], (i / S) & 1u);
      PROF_T(g1);
      const uint32_t t = sh.stage_tile[s];
      if (t == kExitOnly) break;
      if constexpr (CX) {
        if (t != kNoTileTm) {
          // publish the tile's aggregate straight from the stage, before the
          // TMEM slot wait (see CX above); the same sums as the parking pass
          const int32_t *st = stages + s * TM_TILE + q * (QVEC * 128) + lane * 4;
          uint32_t qs = 0;
#pragma unroll 4
          for (int j = 0; j < 16 * TMUL; ++j) {
            uint4 x = *reinterpret_cast<const uint4 *>(st + j * 128);
            if (head && t == 0 && q == 0 && j == 0 && lane == 0) {
              if (head > 0) x.x = 0;
              if (head > 1) x.y = 0;
              if (head > 2) x.z = 0;
            }
            qs += x.x + x.y + x.z + x.w;
          }
          qs = __reduce_add_sync(kFull, qs);
          const uint32_t b = (i / NAG) & 1u;
          if (lane == 0) sh.cx_wtot[grp][b][q] = qs;
          agg_sync(grp);
          if (leader) {
            const uint32_t a = sh.cx_wtot[grp][b][0] + sh.cx_wtot[grp][b][1] +
                               sh.cx_wtot[grp][b][2] + sh.cx_wtot[grp][b][3];
            st_relaxed_gpu(desc + t, pack_desc(epoch, kStAggregate, a));
          }
        }
      }
      if (kp > 0) mbar_wait(&sh.freed[p], (kp - 1) & 1u);
      PROF_T(g2);
      tc_fence_after();
      if (leader && t != kNoTileTm) TM_STAMP(t, 1);
      if (t == kNoTileTm) {
        // one stop item per look-back warp (items i .. i+NLB-1); the finishers
        // stop at the first.  Slot p is free (waited above); the next NLB-1
        // slots held items that the finishers have completed or will complete.
        for (uint32_t e = 0; e < uint32_t(NSTOP); ++e) {
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
          uint32_t v[32], sum = 0, pk[2] = {0u, 0u};
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
            if (COMPACT) {
              const uint32_t c = (int32_t(x.x) > 0) + (int32_t(x.y) > 0) + (int32_t(x.z) > 0) +
                                 (int32_t(x.w) > 0);
              sum += c;
              pk[j >> 2] |= c << (8 * (j & 3));
            } else {
              sum += x.x + x.y + x.z + x.w;
            }
          }
          tmem_st32(tcol + uint32_t(p) * SLOT_COLS + 32u * (TMUL * h + m), v);
#if WF_CMP_PK
          if (COMPACT) {
            sh.slot_pk[p][q][TMUL * h + m][0][lane] = pk[0];
            sh.slot_pk[p][q][TMUL * h + m][1][lane] = pk[1];
          }
#endif
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
#if WF_TM_SWEEP
        if constexpr (!CX)  // (CX: published before the slot wait)
          st_relaxed_gpu(desc + t, pack_desc(epoch, kStAggregate, a));  // dense: the sweeper reads 32 K per trip
#else
        if (t == 0) {
          const uint32_t c0 = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
          st_relaxed_gpu(desc, pack_desc(epoch, kStPrefix, c0 + a));
        } else {
          st_relaxed_gpu(desc + uint64_t(t) * kDescStride, pack_desc(epoch, kStAggregate, a));
        }
#endif
        TM_STAMP(t, 2);
        mbar_arrive1(&sh.parked[p]);
      }
#if WF_TM_PROF
      PROF_T(g3);
      PROF_ADD(0, g0, g1);
      PROF_ADD(1, g1, g2);
      PROF_ADD(2, g2, g3);
      acc[3] += 1;
#endif
    }
#if WF_TM_PROF
    if (warp == 0 && lane == 0 && g_tm_prof)
      for (int k = 0; k < 4; ++k) g_tm_prof[blockIdx.x * 16 + 6 + k] = acc[k];
#endif
  } else if (warp < W_LB) {
    // ------------------------------ finishers -----------------------------
    // warp f handles tile eighth (q, h): TMEM lane quarter q = warp % 4 (the
    // only lanes it may read), columns 32*TMUL*h .. +32*TMUL of the slot
    const uint32_t q = warp & 3u, h = ((warp - W_FIN) >> 2) & 1u;
    const uint32_t grp = (warp - W_FIN) >> 3;
    const uint32_t tcol = sh.tmem_base + ((32u * q) << 16);
#if WF_TM_PROF
    unsigned long long acc[6] = {0, 0, 0, 0, 0, 0};
#endif
    for (uint32_t i = grp;; i += NFG) {
      const int p = int(i % P);
      const uint32_t kp = i / P;
      PROF_T(f0);
      mbar_wait(&sh.parked[p], kp & 1u);
      PROF_T(f1);
      const uint32_t t = sh.slot_tile[p];
      if (t == kNoTileTm) break;
#if WF_TM_TRACE && WF_TM_SWEEP
      if (q == 0 && h == 0 && lane == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        TM_STAMP(t, 5);
        TM_PUT(t, 7, smid);
      }
#endif
      tc_fence_after();
      // everything that does not need the prefix happens before waiting for
      // it: read the slot (metadata + TMEM), free it at once — the tile now
      // waits in this warp's registers, not in TMEM — and do the local scan /
      // ballot positions
      uint32_t v[TMUL][32];
#pragma unroll
      for (int m = 0; m < TMUL; ++m) tmem_ld32(tcol + uint32_t(p) * SLOT_COLS + 32u * (TMUL * h + m), v[m]);
      // the slot's shared metadata is read while the TMEM load is in flight
      uint32_t wexcl = h ? sh.slot_wtot[p][q][0] : 0u;
#pragma unroll
      for (uint32_t w = 0; w < 4; ++w) wexcl += w < q ? sh.slot_wtot[p][w][0] + sh.slot_wtot[p][w][1] : 0u;
      const uint32_t agg = sh.slot_agg[p];
#if WF_CMP_PK
      uint32_t pkm[TMUL][2];
      if (COMPACT) {  // read before the slot is freed (the next item rewrites it)
#pragma unroll
        for (int m = 0; m < TMUL; ++m) {
          pkm[m][0] = sh.slot_pk[p][q][TMUL * h + m][0][lane];
          pkm[m][1] = sh.slot_pk[p][q][TMUL * h + m][1][lane];
        }
      }
#endif
#pragma unroll
      for (int m = 0; m < TMUL; ++m) tmem_wait_ld(v[m]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&sh.freed[p]);
      PROF_T(f2);
      const bool full = vec_out && uint64_t(t + 1) * TM_TILE <= n && (t > 0 || head == 0);
      const uint64_t base0 = uint64_t(t) * TM_TILE + q * (QVEC * 128) + (8 * TMUL * h) * 128 + lane * 4;
      uint32_t loc[TMUL][8];  // scan: chunk add (local); compaction: chunk write position (local)
      uint32_t nzc[TMUL];  // compaction: bit j = chunk j of the eighth has a selected element
#pragma unroll
      for (int m = 0; m < TMUL; ++m) nzc[m] = 0u;
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
          // positions: each lane's selected count per chunk (0-4) packed
          // into byte fields, chunks 0-3 in one word and 4-7 in another, so
          // ONE pair of warp scans yields every chunk's lane offset (a field
          // sums to at most 128: no carry between fields).  32 ballots +
          // 64 POPC per tile eighth took ~1150 cycles of the finisher's
          // ~2000 per tile (WF_TM_PROF), the finisher being the pipeline's
          // slowest stage.
#if WF_CMP_PK
          const uint32_t pk[2] = {pkm[m][0], pkm[m][1]};  // counted by the aggregator
#else
          uint32_t pk[2] = {0u, 0u};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t *x = v[m] + 4 * j;
            const uint32_t c = (int32_t(x[0]) > 0) + (int32_t(x[1]) > 0) + (int32_t(x[2]) > 0) +
                               (int32_t(x[3]) > 0);
            pk[j >> 2] |= c << (8 * (j & 3));
          }
#endif
          uint32_t inc[2] = {pk[0], pk[1]};
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              const uint32_t y = __shfl_up_sync(kFull, inc[w], d);
              if (lane >= uint32_t(d)) inc[w] += y;
            }
          }
          const uint32_t tot[2] = {__shfl_sync(kFull, inc[0], 31), __shfl_sync(kFull, inc[1], 31)};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t sh8 = 8 * (j & 3);
            loc[m][j] = run + (((inc[j >> 2] - pk[j >> 2]) >> sh8) & 0xffu);
            const uint32_t cj = (tot[j >> 2] >> sh8) & 0xffu;
            run += cj;
            nzc[m] |= uint32_t(cj != 0u) << j;  // warp-uniform
            if (!WF_CMP_CHUNK_SKIP && cj != 0u) nzc[m] = 0xffu;  // A/B: the whole eighth
          }
        }
      }
      const int r = int(i % (2 * P));
#if WF_TM_SWEEP
      if (q == 0 && h == 0 && lane == 0) TM_STAMP(t, 6);
#endif
      PROF_T(f3);
      mbar_wait(&sh.pref[r], (i / (2 * P)) & 1u);
      PROF_T(f4);
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
          } else if ((nzc[m] >> j) & 1u) {
            // warp-uniform: nothing selected in this eighth / chunk, nothing to store
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
#if !WF_TM_SWEEP  // (sweeper builds: the sweeper publishes the count, below)
      if constexpr (PX) {
        if (COMPACT && t == ntiles - 1 && q == 0 && h == 0) {
          const uint64_t total = uint64_t(prefix) + agg;
          if (lane == 0) *count = total;
          peer_exscan_warp(total, count + 1, pa);
        }
      } else {
        if (COMPACT && t == ntiles - 1 && q == 0 && h == 0 && lane == 0) *count = uint64_t(prefix) + agg;
      }
#endif
      if (q == 0 && h == 0 && lane == 0) TM_STAMP(t, 4);
#if WF_TM_PROF
      PROF_T(f5);
      PROF_ADD(0, f0, f1);
      PROF_ADD(1, f1, f2);
      PROF_ADD(2, f2, f3);
      PROF_ADD(3, f3, f4);
      PROF_ADD(4, f4, f5);
      acc[5] += 1;
#endif
    }
#if WF_TM_PROF
    if (warp == W_FIN && lane == 0 && g_tm_prof)
      for (int k = 0; k < 6; ++k) g_tm_prof[blockIdx.x * 16 + k] = acc[k];
#endif
#if WF_TM_SWEEP
  } else if (warp == W_LB) {
    // ------------------------------- waiter -------------------------------
    // The prefixes come from the grid's sweeper (below); this warp only
    // watches them.  Lane j follows this CTA's item base + j (j < 2P, the
    // item ring): once the item is parked it polls pref[tile] and posts the
    // prefix to the finishers.  All of the CTA's parked items are polled in
    // the same L2 round trip, so a late prefix never delays the next ones.
    const uint64_t *pref = desc + pref_offset(ntiles);
    const uint32_t tag_pref = uint32_t(pack_desc(epoch, kStPrefix, 0u) >> 32);
    uint32_t base = 0;
    while (true) {
      const uint32_t item = base + lane;
      const int r = int(item % (2 * P));
      bool posted = false, stop = false, polled = false;
      if (lane < 2 * P && ld_acquire_cta_smem(&sh.item_seq[r]) == item) {
        const uint32_t t = sh.item_tile[r];
        if (t == kNoTileTm) {
          stop = true;
        } else if (sh.item_posted[r] == item) {
          posted = true;
        } else {
          polled = true;
          const uint64_t d = ld_relaxed_gpu(pref + t);
          if (uint32_t(d >> 32) == tag_pref) {  // epoch AND status: zeroed memory is epoch 0
            sh.item_prefix[r] = uint32_t(d);
            sh.item_posted[r] = item;
            TM_STAMP(t, 3);
            mbar_arrive1(&sh.pref[r]);  // release: the finishers read item_prefix
            posted = true;
          }
        }
      }
      const uint32_t done = __ballot_sync(kFull, posted);
      const uint32_t stops = __ballot_sync(kFull, stop);
      const uint32_t adv = uint32_t(__ffs(~done)) - 1u;  // items posted in a row from base
      if ((stops >> adv) & 1u) break;                      // the next item is the stop item
      base += adv;
      if (!__any_sync(kFull, polled)) __nanosleep(64);  // nothing parked: do not hammer smem
      __syncwarp();
    }
  } else if (CX && warp == W_TOTAL) {
    // ---------------------------- round totaler ---------------------------
    // (CX, CTA 0) this rank's total of every round, published to all ranks as
    // soon as the round's aggregates are in — independent of any other rank,
    // so the ranks' rounds never chain
    if (blockIdx.x == 0) cx_totals(desc, ntiles, epoch, pa, round_tiles, rounds);
  } else if (warp == W_SWEEP) {
    // ------------------------------- sweeper ------------------------------
    // One warp of CTA 0 turns the aggregates into exclusive prefixes in tile
    // order: it reads 32 K aggregates per L2 round trip, takes the run that is
    // published from the frontier on, scans it and publishes the prefixes.
    // Every tile thus waits one sweep + one poll for its prefix, instead of a
    // per-tile look-back that must walk back to an older resolved prefix and
    // occupies a look-back warp for its whole duration (per-tile traces:
    // ~5 us waiting for a free look-back warp + ~2.8 us of look-back).
    if (CX && blockIdx.x == 0) {
      cx_sweep(desc, ntiles, epoch, pa, round_tiles, rounds);
    } else if (blockIdx.x == 0) {
      uint64_t *pref = desc + pref_offset(ntiles);
      const uint32_t tag_agg = uint32_t(pack_desc(epoch, kStAggregate, 0u) >> 32);
      uint32_t run = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
      uint32_t f = 0, backoff = 32;
      constexpr int K = WF_SWEEP_K;
#if WF_TM_TRACE
      uint32_t it = 0;
#endif
      while (f < ntiles) {
#if WF_TM_TRACE
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
        // all K loads are issued before any result is examined: a compare
        // scheduled right behind its load would serialise the K round trips
        // (measured: 5-6 us per iteration instead of one round trip)
        uint64_t d[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t idx = f + lane + 32u * k;
          d[k] = idx < ntiles ? ld_relaxed_gpu(desc + idx) : 0ull;
        }
        uint32_t v[K];
        bool ok[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          ok[k] = uint32_t(d[k] >> 32) == tag_agg;  // zeroed memory (epoch 0, status 0) never matches
          v[k] = uint32_t(d[k]);
        }
        uint32_t ready = 0;
        bool gap = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t b = __ballot_sync(kFull, ok[k]);
          if (!gap) {
            if (b == kFull) {
              ready += 32;
            } else {
              ready += uint32_t(__ffs(~b)) - 1u;
              gap = true;
            }
          }
        }
#if WF_TM_TRACE
        if (lane == 0 && g_sweep_trace && it < g_sweep_cap) {
          g_sweep_trace[2 * it] = t0;
          g_sweep_trace[2 * it + 1] = f | (uint64_t(ready) << 32);
        }
        ++it;
#endif
        if (ready == 0) {
          __nanosleep(backoff);
          backoff = backoff < 256 ? backoff * 2 : 256;
          continue;
        }
        backoff = 32;
        uint32_t sc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) sc[k] = 32u * k + lane < ready ? v[k] : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const uint32_t y = __shfl_up_sync(kFull, sc[k], d);
            if (lane >= uint32_t(d)) sc[k] += y;
          }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const uint32_t j = 32u * k + lane;
          if (j < ready) st_relaxed_gpu(pref + f + j, pack_desc(epoch, kStPrefix, run + sc[k] - v[k]));
          run += __shfl_sync(kFull, sc[k], 31);
        }
        f += ready;
      }
      // compaction: once the last tile is swept, `run` is the selected count
      // (< 2^32: n < 2^32 per call).  Publish it — and run the sharded
      // offset exchange — here, while the finishers still store the last
      // parked tiles: the exchange's fence + flag round trip hides in that
      // drain instead of following it (2^25 shard: the finishers' drain is
      // ~5 us, tools/trace_tmem.py)
      if constexpr (COMPACT) {
        if constexpr (PX) {
          if (lane == 0) *count = run;
          peer_exscan_warp(uint64_t(run), count + 1, pa);
        } else if (lane == 0) {
          *count = run;
        }
      }
    }
  }
#else
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
      if (lane == 0) TM_STAMP(t, 5);
      uint32_t excl;
      if (t == 0) {  // its prefix descriptor was published by the aggregator
        excl = (!COMPACT && carry_in != nullptr) ? uint32_t(*carry_in) : 0u;
      } else {
#if WF_TM_TRACE
        uint32_t polls = 0;
        excl = lookback_exclusive_wide<COMPACT ? WF_LBK_COMPACT_TM : WF_LBK_TM>(desc, t, epoch,
                                                                               &polls);
        if (lane == 0) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          TM_PUT(t, 6, polls);
          TM_PUT(t, 7, smid);
        }
#else
        excl = lookback_exclusive_wide<COMPACT ? WF_LBK_COMPACT_TM : WF_LBK_TM>(desc, t, epoch);
#endif
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
#endif
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
template <bool COMPACT, bool PX = false, bool CX = false>
int tmem_grid(uint32_t ntiles) {
  static int per_sm[2] = {0, 0};
  static DeviceMask configured;
  configured.ensure([] {
    cudaFuncSetAttribute(tile_tmem_kernel<COMPACT, PX, CX>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(tm_smem<COMPACT>()));
  });
  int &b = per_sm[COMPACT];
  if (b == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tile_tmem_kernel<COMPACT, PX, CX>,
                                                  TM_THREADS, tm_smem<COMPACT>());
    if (b > int(512 / TM_COLS)) b = int(512 / TM_COLS);  // TMEM: 512 columns per SM
    if (b < 1) b = 1;
  }
  const uint32_t g = uint32_t(b) * uint32_t(sm_count(current_device()));
  const uint32_t want = (ntiles + kBatch - 1) / kBatch;  // a CTA's first draw is a whole batch
  return int(want < g ? want : g);
}

}  // namespace

#if WF_TM_TRACE
extern "C" int wf_debug_set_trace_tm(void *buf) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  return int(cudaMemcpyToSymbol(g_tm_trace, &p, sizeof(p)));
}
#endif
#if WF_TM_PROF
extern "C" int wf_debug_set_prof_tm(void *buf) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  return int(cudaMemcpyToSymbol(g_tm_prof, &p, sizeof(p)));
}
#endif
#if WF_TM_TRACE
extern "C" int wf_debug_set_trace_sweep(void *buf, uint32_t cap) {
  unsigned long long *p = static_cast<unsigned long long *>(buf);
  cudaError_t e = cudaMemcpyToSymbol(g_sweep_trace, &p, sizeof(p));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_sweep_cap, &cap, sizeof(cap));
  return int(e);
}
#endif

// `in` / `out` need only 4-byte alignment: the input is rounded down to 16 B
// and its 0-3 leading elements masked; a scan output at another 16-byte
// offset is written with scalar stores.
// `early`: a programmatic dependent launch (the caller's WF_FLAG_INPUT_STABLE
// promise); the kernel's static first loads then overlap the previous grid.
template <bool COMPACT, bool PX, bool CX = false>
cudaError_t launch_tmem(uint32_t nt, bool early, cudaStream_t s, const int32_t *in, int32_t *out,
                        uint64_t nv, const int32_t *carry, uint64_t *count, uint64_t *desc,
                        TileHeader *hdr, uint32_t head, bool vec_out, const PeerArgs &pa,
                        uint32_t round_tiles = 0, uint32_t rounds = 0, int max_grid = 0) {
  cudaLaunchConfig_t cfg = {};
  int grid = tmem_grid<COMPACT, PX, CX>(nt);
  if (max_grid > 0 && grid > max_grid) grid = max_grid;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TM_THREADS);
  cfg.dynamicSmemBytes = tm_smem<COMPACT>();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = early ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, tile_tmem_kernel<COMPACT, PX, CX>, in, out, nv, nt, carry,
                            count, desc, hdr, head, vec_out, pa, round_tiles, rounds);
}

cudaError_t launch_scan_tmem_i32(const int32_t *in, int32_t *out, uint64_t n,
                                 const int32_t *carry, void *ws, cudaStream_t s, bool early) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  return launch_tmem<false, false>(
      nt, early, s, in - head, out - head, nv, carry, nullptr, desc, hdr, head,
      ((reinterpret_cast<uintptr_t>(in) ^ reinterpret_cast<uintptr_t>(out)) & 15u) == 0,
      PeerArgs{});
}

cudaError_t launch_compact_tmem_i32(const int32_t *in, uint64_t n, int32_t *out, uint64_t *count,
                                    void *ws, cudaStream_t s, bool early) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  return launch_tmem<true, false>(nt, early, s, in - head, out, nv, nullptr, count, desc, hdr,
                                  head, false, PeerArgs{});
}

// n >= 1.  counts3 = {count, global offset, global total}.
cudaError_t launch_compact_tmem_i32_mg(const int32_t *in, uint64_t n, int32_t *out,
                                       uint64_t *counts3, void *ws, const PeerArgs &pa,
                                       cudaStream_t s, bool early) {
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t head = uint32_t((reinterpret_cast<uintptr_t>(in) & 15u) / 4u);
  const uint64_t nv = n + head;
  const uint32_t nt = uint32_t((nv + TM_TILE - 1) / TM_TILE);
  return launch_tmem<true, true>(nt, early, s, in - head, out, nv, nullptr, counts3, desc, hdr,
                                 head, false, pa);
}

// Cross-rank single-pass scan of a block-cyclic sharded array (CX above):
// `in` / `out` 16-byte aligned, this rank's local super-tiles of
// round_tiles * 8192 elements back to back (the last may be short), the same
// `rounds` on every rank.  `max_grid` > 0 caps the grid (ranks sharing one
// GPU in tests: their grids must be co-resident, as the rounds wait on each
// other mid-kernel).
cudaError_t launch_scan_tmem_i32_cyclic(const int32_t *in, int32_t *out, uint64_t n, void *ws,
                                        void *const *peers, const void *mine, uint32_t cap,
                                        int rank, int world, uint32_t epoch, uint32_t *err,
                                        uint32_t round_tiles, uint32_t rounds, int max_grid,
                                        cudaStream_t s, bool early) {
  const PeerArgs pa{reinterpret_cast<uint64_t *const *>(peers), static_cast<const uint64_t *>(mine),
                    cap, rank, world, epoch, err};
  auto *hdr = reinterpret_cast<TileHeader *>(ws);
  auto *desc = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kTileWsHeader);
  const uint32_t nt = uint32_t((n + TM_TILE - 1) / TM_TILE);
  return launch_tmem<false, false, true>(nt, early, s, in, out, n, nullptr, nullptr, desc, hdr,
                                         0u, true, pa, round_tiles, rounds, max_grid);
}

cudaError_t preload_tmem_mg_kernels() {
  tmem_grid<true, true>(1);  // dynamic-smem opt-in on this device
  tmem_grid<false, false, true>(1);
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, tile_tmem_kernel<true, true>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, tile_tmem_kernel<false, false, true>);
  return e;
}

}  // namespace wf
