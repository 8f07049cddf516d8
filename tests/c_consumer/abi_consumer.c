/* A plain C99 consumer of the drop-in boundary (include/warpfold_b200.h):
 * what a reference-side binding links against, with no Python or torch in
 * the process.  Built and run by tests/test_host.py ("cpu": header compiles
 * as C, library links, argument errors map to codes) and
 * tests/test_gpu_integration.py ("gpu": the host-buffer entry points of
 * C2-C5 end to end, checked against serial C loops).
 *
 * usage: abi_consumer cpu|gpu                        exit 0 = all checks passed */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "warpfold_b200.h"

/* the CUDA runtime calls the caller makes for its own buffers */
typedef int cudaError_t;
extern cudaError_t cudaMalloc(void **p, size_t bytes);
extern cudaError_t cudaMemset(void *p, int v, size_t bytes);
extern cudaError_t cudaFree(void *p);

static int failures = 0;
#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);            \
      fprintf(stderr, "\n");                   \
      ++failures;                              \
    }                                          \
  } while (0)

static int cpu_checks(void) {
  float out = 0.0f;
  int rc;
  CHECK(wf_abi_version() > 0, "abi version %d", wf_abi_version());
  CHECK(strlen(wf_version()) > 0, "empty version");
  CHECK(wf_workspace_bytes(WF_OP_SCAN_INCLUSIVE_I32, 1u << 20, 0) > 0, "scan workspace size");
  CHECK(wf_workspace_bytes(WF_OP_HISTOGRAM256_U8, 1u << 20, 0) > 0, "hist workspace size");
  /* NULL input with n > 0: an argument error before any device work */
  rc = wf_reduce_sum_f32(NULL, 5, &out, 256, 0, NULL, 0, NULL);
  CHECK(rc == WF_ERR_ARG, "NULL input -> %d (%s)", rc, wf_last_error());
  CHECK(strlen(wf_last_error()) > 0, "no error message");
  rc = wf_scan_inclusive_i32_ex(NULL, NULL, 0, NULL, NULL, 0, 0x80u, NULL);
  CHECK(rc == WF_ERR_ARG, "unknown flag -> %d (%s)", rc, wf_last_error());
  return failures;
}

static int gpu_checks(void) {
  const uint64_t n = 3000007;
  const size_t staging_bytes = 8u << 20;
  /* one zero-filled workspace PER OP (the header's contract: a workspace is
   * reused by calls of the same op; another op's leftovers are not zero) */
  void *staging = NULL, *wss[WF_OP_HISTOGRAM256_U8 + 1] = {NULL};
  size_t wsb[WF_OP_HISTOGRAM256_U8 + 1] = {0};
  int op;
  if (cudaMalloc(&staging, staging_bytes)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  for (op = WF_OP_REDUCE_SUM_I32; op <= WF_OP_HISTOGRAM256_U8; ++op) {
    wsb[op] = wf_workspace_bytes(op, n, 0);
    if (cudaMalloc(&wss[op], wsb[op]) || cudaMemset(wss[op], 0, wsb[op])) {
      fprintf(stderr, "cudaMalloc failed\n");
      return 1;
    }
  }
#define WS(op) wss[op], wsb[op]
  float *f = malloc(n * sizeof(float));
  int32_t *a = malloc(n * sizeof(int32_t)), *y = malloc(n * sizeof(int32_t));
  uint8_t *u = malloc(n);
  uint64_t i;
  double want_f = 0.0;
  for (i = 0; i < n; ++i) {
    f[i] = (float)((int)(i % 7) - 3); /* partial sums stay exact in fp32 */
    want_f += f[i];
    a[i] = (int32_t)((i * 2654435761u) ^ (i >> 3)) - (int32_t)(1u << 30);
    u[i] = (uint8_t)(i * 131u + (i >> 9));
  }

  float got_f = 0.0f;
  int rc = wf_reduce_sum_f32_host(f, n, &got_f, staging, staging_bytes, WS(WF_OP_REDUCE_SUM_F32), NULL);
  CHECK(rc == 0 && (double)got_f == want_f, "reduce_f32 rc %d got %f want %f (%s)", rc, got_f, want_f,
        wf_last_error());

  int32_t got_i = 0;
  uint32_t want_i = 0;
  for (i = 0; i < n; ++i) want_i += (uint32_t)a[i];
  rc = wf_reduce_sum_i32_host(a, n, &got_i, staging, staging_bytes, WS(WF_OP_REDUCE_SUM_I32), NULL);
  CHECK(rc == 0 && (uint32_t)got_i == want_i, "reduce_i32 rc %d (%s)", rc, wf_last_error());

  int32_t carry = 17;
  rc = wf_scan_inclusive_i32_host(a, y, n, &carry, staging, staging_bytes, WS(WF_OP_SCAN_INCLUSIVE_I32),
                                  NULL);
  {
    uint32_t run = (uint32_t)carry;
    uint64_t bad = 0;
    for (i = 0; i < n; ++i) {
      run += (uint32_t)a[i];
      bad += (uint32_t)y[i] != run;
    }
    CHECK(rc == 0 && bad == 0, "scan rc %d, %llu mismatches (%s)", rc, (unsigned long long)bad,
          wf_last_error());
  }

  uint64_t count = 0;
  rc = wf_compact_gt0_i32_host(a, n, y, &count, staging, staging_bytes, WS(WF_OP_COMPACT_GT0_I32), NULL);
  {
    uint64_t k = 0, bad = 0;
    for (i = 0; i < n; ++i) {
      if (a[i] > 0) {
        bad += k < count && y[k] != a[i];
        ++k;
      }
    }
    CHECK(rc == 0 && count == k && bad == 0, "compact rc %d count %llu want %llu (%s)", rc,
          (unsigned long long)count, (unsigned long long)k, wf_last_error());
  }

  uint64_t bins[256], want_b[256];
  memset(want_b, 0, sizeof want_b);
  for (i = 0; i < n; ++i) ++want_b[u[i]];
  rc = wf_histogram256_u8_host(u, n, bins, staging, staging_bytes, WS(WF_OP_HISTOGRAM256_U8), NULL);
  CHECK(rc == 0 && memcmp(bins, want_b, sizeof bins) == 0, "histogram rc %d (%s)", rc, wf_last_error());

  free(f), free(a), free(y), free(u);
  cudaFree(staging);
  for (op = WF_OP_REDUCE_SUM_I32; op <= WF_OP_HISTOGRAM256_U8; ++op) cudaFree(wss[op]);
  return failures;
}

int main(int argc, char **argv) {
  if (argc != 2 || (strcmp(argv[1], "cpu") && strcmp(argv[1], "gpu"))) {
    fprintf(stderr, "usage: %s cpu|gpu\n", argv[0]);
    return 2;
  }
  int bad = strcmp(argv[1], "cpu") == 0 ? cpu_checks() : gpu_checks();
  if (bad == 0) printf("OK %s\n", argv[1]);
  return bad ? 1 : 0;
}
