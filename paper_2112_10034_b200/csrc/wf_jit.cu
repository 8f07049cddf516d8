// wf_jit.cu — native compilation of warpfold DSL kernels for sm_100a.
//
// Reference analog: hybrid_transform (passes/pipeline.py:103-179) turns a DSL
// kernel into collapsed loop nests that run_mpmd (interp/mpmd.py:237-255)
// interprets on CPU workers.  On B200 the kernel runs as real SIMT code: the
// Python front end (paper_2112_10034_b200/dsl) emits CUDA C with the
// reference's scalar semantics, and this file compiles it with NVRTC straight
// to an sm_100a cubin, loads it with the runtime library API
// (cudaLibraryLoadData / cudaLibraryGetKernel) and launches it.  libnvrtc is
// opened lazily with dlopen, so the library itself has no NVRTC dependency.
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/warpfold_b200.h"

namespace wf {
namespace {

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram *nvrtcProgram_t;

struct Nvrtc {
  void *h = nullptr;
  nvrtcResult_t (*create)(nvrtcProgram_t *, const char *, const char *, int, const char *const *,
                          const char *const *) = nullptr;
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char *const *) = nullptr;
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t *) = nullptr;
  nvrtcResult_t (*log)(nvrtcProgram_t, char *) = nullptr;
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t *) = nullptr;
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char *) = nullptr;
  nvrtcResult_t (*destroy)(nvrtcProgram_t *) = nullptr;
  const char *(*errstr)(nvrtcResult_t) = nullptr;
};

std::mutex g_nvrtc_mu;
Nvrtc g_nvrtc;

bool load_nvrtc(std::string &err) {
  std::lock_guard<std::mutex> lk(g_nvrtc_mu);
  if (g_nvrtc.h) return true;
  const char *env = getenv("WF_NVRTC");
  const char *names[] = {env, "libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void *h = nullptr;
  for (const char *nm : names) {
    if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  }
  if (!h) {
    err = "cannot dlopen libnvrtc (set WF_NVRTC)";
    return false;
  }
  Nvrtc n;
  n.h = h;
#define WF_SYM(field, name)                                           \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));      \
  if (!n.field) {                                                     \
    err = std::string("libnvrtc lacks ") + name;                      \
    return false;                                                     \
  }
  WF_SYM(create, "nvrtcCreateProgram");
  WF_SYM(compile, "nvrtcCompileProgram");
  WF_SYM(log_size, "nvrtcGetProgramLogSize");
  WF_SYM(log, "nvrtcGetProgramLog");
  WF_SYM(cubin_size, "nvrtcGetCUBINSize");
  WF_SYM(cubin, "nvrtcGetCUBIN");
  WF_SYM(destroy, "nvrtcDestroyProgram");
  WF_SYM(errstr, "nvrtcGetErrorString");
#undef WF_SYM
  g_nvrtc = n;
  return true;
}

struct JitModule {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  int smem_configured_device = -1;
  unsigned smem_configured = 0;
};

void copy_log(char *dst, size_t cap, const std::string &s) {
  if (!dst || cap == 0) return;
  const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  memcpy(dst, s.data(), n);
  dst[n] = 0;
}

std::vector<std::string> split_opts(const char *options) {
  std::vector<std::string> out;
  if (!options) return out;
  std::string cur;
  for (const char *p = options;; ++p) {
    if (*p == ' ' || *p == 0) {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
      if (*p == 0) break;
    } else {
      cur.push_back(*p);
    }
  }
  return out;
}

}  // namespace
}  // namespace wf

using namespace wf;

extern "C" {

int wf_jit_compile(const char *src, const char *kernel_name, const char *options, void **module,
                   char *log, size_t log_bytes) {
  if (!src || !kernel_name || !module) {
    copy_log(log, log_bytes, "NULL argument");
    return WF_ERR_ARG;
  }
  *module = nullptr;
  std::string err;
  if (!load_nvrtc(err)) {
    copy_log(log, log_bytes, err);
    return WF_ERR_UNSUPPORTED;
  }
  nvrtcProgram_t prog = nullptr;
  if (g_nvrtc.create(&prog, src, "wf_dsl_kernel.cu", 0, nullptr, nullptr) != 0) {
    copy_log(log, log_bytes, "nvrtcCreateProgram failed");
    return WF_ERR_EXEC;
  }
  std::vector<std::string> opts = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17",
                                   "-default-device", "-lineinfo"};
  for (auto &o : split_opts(options)) opts.push_back(o);
  std::vector<const char *> argv;
  for (auto &o : opts) argv.push_back(o.c_str());
  const nvrtcResult_t rc = g_nvrtc.compile(prog, int(argv.size()), argv.data());
  size_t ls = 0;
  g_nvrtc.log_size(prog, &ls);
  std::string lg(ls, '\0');
  if (ls) g_nvrtc.log(prog, &lg[0]);
  if (rc != 0) {
    copy_log(log, log_bytes, std::string(g_nvrtc.errstr(rc)) + "\n" + lg);
    g_nvrtc.destroy(&prog);
    return WF_ERR_EXEC;
  }
  size_t cs = 0;
  g_nvrtc.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  g_nvrtc.cubin(prog, cubin.data());
  g_nvrtc.destroy(&prog);

  auto *m = new JitModule();
  cudaError_t e = cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0, nullptr,
                                      nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&m->kernel, m->lib, kernel_name);
  if (e != cudaSuccess) {
    cudaGetLastError();
    copy_log(log, log_bytes, std::string("loading cubin: ") + cudaGetErrorString(e));
    if (m->lib) cudaLibraryUnload(m->lib);
    delete m;
    return int(e);
  }
  copy_log(log, log_bytes, lg);
  *module = m;
  return WF_OK;
}

int wf_jit_launch(void *module, uint32_t grid, uint32_t block, uint32_t smem_bytes, void **args,
                  wf_stream_t stream) {
  auto *m = static_cast<JitModule *>(module);
  if (!m || !m->kernel) return WF_ERR_ARG;
  if (grid == 0) return WF_OK;
  if (block == 0 || block > 1024) return WF_ERR_CONFIG;
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem_bytes > 48 * 1024 &&
      (m->smem_configured_device != dev || m->smem_configured < smem_bytes)) {
    cudaError_t e = cudaKernelSetAttributeForDevice(
        m->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes), dev);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return int(e);
    }
    m->smem_configured_device = dev;
    m->smem_configured = smem_bytes;
  }
  cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void *>(m->kernel), dim3(grid),
                                   dim3(block), args, smem_bytes,
                                   static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) cudaGetLastError();
  return int(e);
}

int wf_jit_unload(void *module) {
  auto *m = static_cast<JitModule *>(module);
  if (!m) return WF_OK;
  if (m->lib) cudaLibraryUnload(m->lib);
  delete m;
  return WF_OK;
}

}  // extern "C"
