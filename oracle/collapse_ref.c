/*
 * collapse_ref.c — C restatement of the programs the warpfold reference
 * executes for the warp-primitive path.  TEST INFRASTRUCTURE ONLY (the parity
 * checker and the CPU baseline of bench.py; never linked into the product).
 *
 * The reference (arXiv 2112.10034 "COX", pure-Python re-implementation)
 * compiles a CUDA-style kernel into a sequential program per block by
 * hierarchical collapsing (passes/pipeline.py:103-179):
 *   - every warp collective becomes a lane-buffer store, a RAW warp barrier,
 *     the read, and a WAR warp barrier (passes/warp_lower.py:52-88);
 *   - barrier-delimited parallel regions are wrapped in a `for __tx < W`
 *     lane loop, nested in a `for __wid < blockDim/W` warp loop
 *     (passes/wrap.py:85-170);
 *   - locals that live across regions become [W] / [B] arrays
 *     (passes/replicate.py:47-170);
 * and the runtime runs contiguous block ranges on a worker pool with join
 * semantics (runtime/launch.py:90-147, `_split` at :137-147).
 * This file writes those collapsed loop nests out by hand, in C, for the
 * five BASELINE kernels, with pthreads standing in for the fork pool.  i32
 * arithmetic is done in uint32_t (the reference's wrap mod 2^32,
 * numerics.py:20-22); f32 is IEEE single with no contraction (build with
 * -ffp-contract=off).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define W 32

/* ---- block-range worker pool (runtime/launch.py:95-128, _split :137-147) */
typedef void (*block_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct {
  block_fn fn;
  void *ctx;
  int64_t lo, hi;
} job_t;

static void *run_job(void *p) {
  job_t *j = (job_t *)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}

static void parallel_blocks(int64_t grid, int workers, block_fn fn, void *ctx) {
  if (workers > grid) workers = (int)grid;
  if (workers <= 1) {
    if (grid > 0) fn(ctx, 0, grid);
    return;
  }
  pthread_t th[256];
  job_t jobs[256];
  if (workers > 256) workers = 256;
  int64_t base = grid / workers, extra = grid % workers, lo = 0;
  for (int i = 0; i < workers; ++i) {
    int64_t hi = lo + base + (i < extra ? 1 : 0);
    jobs[i].fn = fn;
    jobs[i].ctx = ctx;
    jobs[i].lo = lo;
    jobs[i].hi = hi;
    lo = hi;
    pthread_create(&th[i], NULL, run_job, &jobs[i]);
  }
  for (int i = 0; i < workers; ++i) pthread_join(th[i], NULL);
}

/* ---- C1 / C2: per-warp-partials shfl_down reduction ----
 *   sum = 0; for (i = tid; i < n; i += blockDim*gridDim) sum += a[i];
 *   for (off = 16; off > 0; off /= 2) sum += shfl_down(sum, off);
 *   if (tx % 32 == 0) out[bid * (blockDim/32) + tx/32] = sum;            */
typedef struct {
  const void *a;
  int64_t n;
  int grid, block;
  void *out;
} reduce_ctx;

static void reduce_i32_blocks(void *p, int64_t lo, int64_t hi) {
  reduce_ctx *c = (reduce_ctx *)p;
  const int32_t *a = (const int32_t *)c->a;
  int32_t *out = (int32_t *)c->out;
  const int64_t stride = (int64_t)c->block * c->grid;
  for (int64_t b = lo; b < hi; ++b) {
    for (int wid = 0; wid < c->block / W; ++wid) {
      uint32_t sum[W], buf[W];
      for (int tx = 0; tx < W; ++tx) { /* region 1: lane loop */
        uint32_t s = 0;
        for (int64_t i = (int64_t)wid * W + tx + b * c->block; i < c->n; i += stride)
          s += (uint32_t)a[i];
        sum[tx] = s;
      }
      for (int off = 16; off > 0; off /= 2) {
        for (int tx = 0; tx < W; ++tx) buf[tx] = sum[tx]; /* lane store; RAW */
        for (int tx = 0; tx < W; ++tx)                    /* read; WAR      */
          sum[tx] += (tx + off < W) ? buf[tx + off] : buf[tx];
      }
      for (int tx = 0; tx < W; ++tx)
        if (tx % 32 == 0) out[b * (c->block / 32) + (wid * W + tx) / 32] = (int32_t)sum[tx];
    }
  }
}

static void reduce_f32_blocks(void *p, int64_t lo, int64_t hi) {
  reduce_ctx *c = (reduce_ctx *)p;
  const float *a = (const float *)c->a;
  float *out = (float *)c->out;
  const int64_t stride = (int64_t)c->block * c->grid;
  for (int64_t b = lo; b < hi; ++b) {
    for (int wid = 0; wid < c->block / W; ++wid) {
      float sum[W], buf[W];
      for (int tx = 0; tx < W; ++tx) {
        float s = 0.0f;
        for (int64_t i = (int64_t)wid * W + tx + b * c->block; i < c->n; i += stride) s = s + a[i];
        sum[tx] = s;
      }
      for (int off = 16; off > 0; off /= 2) {
        for (int tx = 0; tx < W; ++tx) buf[tx] = sum[tx];
        for (int tx = 0; tx < W; ++tx) sum[tx] = sum[tx] + ((tx + off < W) ? buf[tx + off] : buf[tx]);
      }
      for (int tx = 0; tx < W; ++tx)
        if (tx % 32 == 0) out[b * (c->block / 32) + (wid * W + tx) / 32] = sum[tx];
    }
  }
}

int wfo_reduce_partials_i32(const int32_t *a, int64_t n, int grid, int block, int32_t *partials,
                            int workers) {
  if (block % W) return -1;
  reduce_ctx c = {a, n, grid, block, partials};
  parallel_blocks(grid, workers, reduce_i32_blocks, &c);
  return 0;
}

int wfo_reduce_partials_f32(const float *a, int64_t n, int grid, int block, float *partials,
                            int workers) {
  if (block % W) return -1;
  reduce_ctx c = {a, n, grid, block, partials};
  parallel_blocks(grid, workers, reduce_f32_blocks, &c);
  return 0;
}

/* host fold of the partials, in warp order (the host code of the C1 pin) */
int32_t wfo_fold_i32(const int32_t *p, int64_t m) {
  uint32_t s = 0;
  for (int64_t i = 0; i < m; ++i) s += (uint32_t)p[i];
  return (int32_t)s;
}

float wfo_fold_f32(const float *p, int64_t m) {
  float s = 0.0f;
  for (int64_t i = 0; i < m; ++i) s = s + p[i];
  return s;
}

/* ---- C3: SDK shfl_scan, collapsed ----------------------------------------
 * kernel 1 (one element per thread): warp inclusive scan with shfl_up
 * (lane buffer + RAW/WAR), warp totals to smem, __syncthreads, warp 0 scans
 * the totals, __syncthreads, add the warp carry; block total -> sums[bid].
 * kernel 2: scan of the block sums.  kernel 3: uniform add of the carries. */
typedef struct {
  const int32_t *a;
  int64_t n;
  int block;
  int32_t *out;
  uint32_t *sums;
} scan_ctx;

static void scan_blocks(void *p, int64_t lo, int64_t hi) {
  scan_ctx *c = (scan_ctx *)p;
  const int nw = c->block / W;
  uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * c->block); /* replicated local [B] */
  uint32_t wsum[32];                                              /* shared [32]        */
  for (int64_t b = lo; b < hi; ++b) {
    const int64_t g0 = b * c->block;
    for (int wid = 0; wid < nw; ++wid) {
      uint32_t *x = v + wid * W, buf[W];
      for (int tx = 0; tx < W; ++tx) {
        const int64_t g = g0 + wid * W + tx;
        x[tx] = g < c->n ? (uint32_t)c->a[g] : 0u;
      }
      for (int d = 1; d < W; d <<= 1) {
        for (int tx = 0; tx < W; ++tx) buf[tx] = x[tx];
        for (int tx = 0; tx < W; ++tx) x[tx] += (tx >= d) ? buf[tx - d] : 0u;
      }
      wsum[wid] = x[W - 1];
    }
    /* __syncthreads(); warp 0 scans the warp totals (lanes >= nw read 0) */
    {
      uint32_t y[W], buf[W];
      for (int tx = 0; tx < W; ++tx) y[tx] = tx < nw ? wsum[tx] : 0u;
      for (int d = 1; d < W; d <<= 1) {
        for (int tx = 0; tx < W; ++tx) buf[tx] = y[tx];
        for (int tx = 0; tx < W; ++tx) y[tx] += (tx >= d) ? buf[tx - d] : 0u;
      }
      for (int tx = 0; tx < nw; ++tx) wsum[tx] = y[tx];
    }
    /* __syncthreads(); add the exclusive warp carry and store */
    for (int wid = 0; wid < nw; ++wid)
      for (int tx = 0; tx < W; ++tx) {
        const int64_t g = g0 + wid * W + tx;
        const uint32_t r = v[wid * W + tx] + (wid > 0 ? wsum[wid - 1] : 0u);
        if (g < c->n) c->out[g] = (int32_t)r;
      }
    c->sums[b] = wsum[nw - 1];
  }
  free(v);
}

typedef struct {
  int64_t n;
  int block;
  int32_t *out;
  const uint32_t *carry;
} add_ctx;

static void uniform_add_blocks(void *p, int64_t lo, int64_t hi) {
  add_ctx *c = (add_ctx *)p;
  for (int64_t b = lo; b < hi; ++b) {
    if (b == 0) continue;
    const uint32_t k = c->carry[b - 1];
    for (int tx = 0; tx < c->block; ++tx) {
      const int64_t g = b * c->block + tx;
      if (g < c->n) c->out[g] = (int32_t)((uint32_t)c->out[g] + k);
    }
  }
}

int wfo_scan_i32(const int32_t *a, int64_t n, int block, int32_t *out, int workers) {
  if (block % W || block / W > 32) return -1;
  const int64_t grid = (n + block - 1) / block;
  uint32_t *sums = (uint32_t *)malloc(sizeof(uint32_t) * (grid ? grid : 1));
  scan_ctx c = {a, n, block, out, sums};
  parallel_blocks(grid, workers, scan_blocks, &c);
  for (int64_t b = 1; b < grid; ++b) sums[b] += sums[b - 1]; /* kernel 2 */
  add_ctx d = {n, block, out, sums};
  parallel_blocks(grid, workers, uniform_add_blocks, &d);
  free(sums);
  return 0;
}

/* ---- C4: warp-aggregated compaction with ordered output, collapsed -------
 * kernel 1: per warp, ballot (lane loop builds the mask) + popc -> block
 * count.  host: exclusive scan of block counts.  kernel 2: per lane,
 * position = block offset + warp offset + popc(ballot & lanemask_lt).      */
typedef struct {
  const int32_t *a;
  int64_t n;
  int block;
  int32_t *out;
  uint64_t *counts;
} compact_ctx;

static uint32_t warp_ballot(const int32_t *a, int64_t n, int64_t g0) {
  uint32_t m = 0;
  for (int tx = 0; tx < W; ++tx) {
    const int64_t g = g0 + tx;
    if (g < n && a[g] > 0) m |= 1u << tx;
  }
  return m;
}

static void compact_count_blocks(void *p, int64_t lo, int64_t hi) {
  compact_ctx *c = (compact_ctx *)p;
  for (int64_t b = lo; b < hi; ++b) {
    uint64_t cnt = 0;
    for (int wid = 0; wid < c->block / W; ++wid)
      cnt += (uint64_t)__builtin_popcount(warp_ballot(c->a, c->n, b * c->block + wid * W));
    c->counts[b] = cnt;
  }
}

static void compact_write_blocks(void *p, int64_t lo, int64_t hi) {
  compact_ctx *c = (compact_ctx *)p;
  for (int64_t b = lo; b < hi; ++b) {
    uint64_t off = c->counts[b];
    for (int wid = 0; wid < c->block / W; ++wid) {
      const int64_t g0 = b * c->block + wid * W;
      const uint32_t m = warp_ballot(c->a, c->n, g0);
      for (int tx = 0; tx < W; ++tx)
        if (m >> tx & 1u) c->out[off + __builtin_popcount(m & ((1u << tx) - 1u))] = c->a[g0 + tx];
      off += (uint64_t)__builtin_popcount(m);
    }
  }
}

int64_t wfo_compact_gt0_i32(const int32_t *a, int64_t n, int block, int32_t *out, int workers) {
  if (block % W) return -1;
  const int64_t grid = (n + block - 1) / block;
  uint64_t *counts = (uint64_t *)malloc(sizeof(uint64_t) * (grid ? grid : 1));
  compact_ctx c = {a, n, block, out, counts};
  parallel_blocks(grid, workers, compact_count_blocks, &c);
  uint64_t run = 0;
  for (int64_t b = 0; b < grid; ++b) {
    const uint64_t k = counts[b];
    counts[b] = run;
    run += k;
  }
  parallel_blocks(grid, workers, compact_write_blocks, &c);
  free(counts);
  return (int64_t)run;
}

/* ---- C5: smem-privatised 256-bin histogram, collapsed --------------------
 * shared u32 bins[256] = 0; __syncthreads(); grid-stride: atomicAdd(&bins[
 * a[i]], 1) — one CPU thread runs the whole block, so the shared atomic is a
 * plain increment; __syncthreads(); atomicAdd(&global[b], bins[b]).        */
typedef struct {
  const uint8_t *a;
  int64_t n;
  int grid, block;
  uint64_t *partial; /* [workers][256], the global atomics per worker */
  int64_t blocks_per_worker_hint;
} hist_ctx;

static pthread_mutex_t g_hist_mu = PTHREAD_MUTEX_INITIALIZER;

static void hist_blocks(void *p, int64_t lo, int64_t hi) {
  hist_ctx *c = (hist_ctx *)p;
  uint64_t local[256];
  memset(local, 0, sizeof local);
  const int64_t stride = (int64_t)c->grid * c->block;
  uint32_t bins[256];
  for (int64_t b = lo; b < hi; ++b) {
    memset(bins, 0, sizeof bins);
    for (int tx = 0; tx < c->block; ++tx)
      for (int64_t i = b * c->block + tx; i < c->n; i += stride) bins[c->a[i]] += 1u;
    for (int k = 0; k < 256; ++k) local[k] += bins[k];
  }
  pthread_mutex_lock(&g_hist_mu);
  for (int k = 0; k < 256; ++k) c->partial[k] += local[k];
  pthread_mutex_unlock(&g_hist_mu);
}

int wfo_hist256_u8(const uint8_t *a, int64_t n, int grid, int block, uint64_t *bins, int workers) {
  memset(bins, 0, 256 * sizeof(uint64_t));
  hist_ctx c = {a, n, grid, block, bins, 0};
  parallel_blocks(grid, workers, hist_blocks, &c);
  return 0;
}
