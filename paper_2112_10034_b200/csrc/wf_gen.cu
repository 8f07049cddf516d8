// wf_gen.cu — on-device synthetic inputs.
//
// Element i of every generator is a pure function of splitmix64(seed ^
// (base + i)), so the GPU writes multi-GiB inputs straight into HBM and the
// CPU oracle (oracle/synthetic.py) regenerates any slice of the same input
// bit-exactly — no multi-GiB host->device copies for parity checks.
#include "wf_device.cuh"
#include "wf_internal.h"
#include "../../include/warpfold_b200.h"

namespace wf {
namespace {

__device__ __forceinline__ uint32_t gen_word(int gen, uint64_t h, uint32_t param) {
  switch (gen) {
    case WF_GEN_I32_FULL: return uint32_t(h >> 32);
    case WF_GEN_I32_SMALL: return uint32_t(int32_t((h >> 32) % 21u) - 10);
    case WF_GEN_F32_UNIT:
      return __float_as_uint(float(uint32_t(h >> 40)) * 5.9604644775390625e-08f - 0.5f);
    case WF_GEN_I32_SELECT: {
      const uint32_t mag = uint32_t(h >> 33);          // 31-bit magnitude
      const uint32_t draw = uint32_t(h & 0xffffu) * 1000u >> 16;  // 0..999
      return draw < param ? (mag | 1u) : uint32_t(-int32_t(mag));
    }
    default: return 0u;
  }
}

__device__ __forceinline__ uint8_t gen_byte(int gen, uint64_t h, uint32_t param) {
  switch (gen) {
    case WF_GEN_U8_UNIFORM: return uint8_t(h & 0xffu);
    case WF_GEN_U8_CONST: return uint8_t(param & 0xffu);
    case WF_GEN_U8_GEOM: return uint8_t(min(__clzll(static_cast<long long>(h)), 255));
    default: return 0;
  }
}

__global__ void fill_words(int gen, uint32_t *__restrict__ out, uint64_t n,
                           uint64_t seed, uint64_t base, uint32_t param) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    out[i] = gen_word(gen, splitmix64(seed ^ (base + i)), param);
  }
}

__global__ void fill_bytes(int gen, uint8_t *__restrict__ out, uint64_t n,
                           uint64_t seed, uint64_t base, uint32_t param) {
  // 4 bytes per thread-iteration, one 32-bit store when aligned
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t nq = n / 4;
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 3u) == 0;
  for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint64_t i = q * 4;
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w |= uint32_t(gen_byte(gen, splitmix64(seed ^ (base + i + k)), param)) << (8 * k);
    if (aligned) {
      reinterpret_cast<uint32_t *>(out)[q] = w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) out[i + k] = uint8_t(w >> (8 * k));
    }
  }
  const uint64_t t = nq * 4 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = gen_byte(gen, splitmix64(seed ^ (base + t)), param);
}

}  // namespace

cudaError_t launch_fill_synthetic(int gen, void *out, uint64_t n, uint64_t seed,
                                  uint64_t base, uint32_t param, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int block = 256;
  const int grid = sm_count(current_device()) * 8;
  if (gen == WF_GEN_U8_UNIFORM || gen == WF_GEN_U8_CONST || gen == WF_GEN_U8_GEOM) {
    fill_bytes<<<grid, block, 0, s>>>(gen, static_cast<uint8_t *>(out), n, seed, base, param);
  } else {
    fill_words<<<grid, block, 0, s>>>(gen, static_cast<uint32_t *>(out), n, seed, base, param);
  }
  return cudaGetLastError();
}

}  // namespace wf
