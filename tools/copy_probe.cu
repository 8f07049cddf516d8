// Read + write HBM ceiling on this B200: a plain 16-byte-vector copy kernel
// (grid-stride, UNROLL loads in flight, streaming stores) over 1 GiB in /
// 1 GiB out, i.e. exactly the traffic of K3 at 2^28 (8 B per element), plus a
// read-only pass for comparison.  Tools only — the ceiling the TMEM scan and
// the 100 % compaction are judged against.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/copy_probe tools/copy_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int UNROLL>
__global__ void __launch_bounds__(256) copy_kernel(const uint4 *__restrict__ in,
                                                   uint4 *__restrict__ out, uint64_t nvec) {
  const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * T < nvec; i += UNROLL * T) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(q[u].x), "=r"(q[u].y), "=r"(q[u].z), "=r"(q[u].w)
                   : "l"(in + i + u * T));
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + i + u * T),
                   "r"(q[u].x), "r"(q[u].y), "r"(q[u].z), "r"(q[u].w)
                   : "memory");
  }
  for (; i < nvec; i += T) out[i] = in[i];
}

__global__ void __launch_bounds__(256) read_kernel(const uint4 *__restrict__ in, uint64_t nvec,
                                                   uint32_t *sink) {
  const uint64_t T = uint64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += T) {
    uint4 q;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "l"(in + i));
    acc ^= q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;  // us
}

int main() {
  const uint64_t bytes = uint64_t(1) << 30, nvec = bytes / 16;
  uint4 *in, *out;
  uint32_t *sink;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(in, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {4, 8}) {
    const int grid = sms * per_sm;
    float t2 = time_it([&] { copy_kernel<2><<<grid, 256>>>(in, out, nvec); }, 20);
    float t4 = time_it([&] { copy_kernel<4><<<grid, 256>>>(in, out, nvec); }, 20);
    float t8 = time_it([&] { copy_kernel<8><<<grid, 256>>>(in, out, nvec); }, 20);
    float tr = time_it([&] { read_kernel<<<grid, 256>>>(in, nvec, sink); }, 20);
    printf("{\"ctas_per_sm\": %d, \"copy_u2_us\": %.1f, \"copy_u4_us\": %.1f, \"copy_u8_us\": %.1f, "
           "\"copy_best_tbs\": %.3f, \"read_us\": %.1f, \"read_tbs\": %.3f}\n",
           per_sm, t2, t4, t8, 2.0 * bytes / (1e6 * (t2 < t4 ? (t2 < t8 ? t2 : t8) : (t4 < t8 ? t4 : t8))),
           tr, bytes / (1e6 * tr));
  }
  return 0;
}
