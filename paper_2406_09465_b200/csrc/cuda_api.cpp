#include "cuda_api.h"

#include <dlfcn.h>

#include <mutex>

namespace korch {

#define KORCH_XSTR(x) KORCH_STR(x)
#define KORCH_STR(x) #x

CudaApi& cuda() {
  static CudaApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libcuda.so.1: ") + dlerror();
      return;
    }
    // names go through cuda.h's versioning macros (e.g. cuMemAlloc -> cuMemAlloc_v2)
#define KORCH_LOAD(name)                                                          \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, KORCH_XSTR(name)));    \
  if (!api.name) { api.err = std::string("missing symbol ") + KORCH_XSTR(name); return; }
    KORCH_CU_FUNCS(KORCH_LOAD)
#undef KORCH_LOAD
    CUresult r = api.cuInit(0);
    if (r != CUDA_SUCCESS) {
      api.err = "cuInit failed (" + std::to_string((int)r) + ")";
      return;
    }
    api.ok = true;
  });
  return api;
}

NvrtcApi& nvrtc() {
  static NvrtcApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("cannot load libnvrtc.so.12: ") + dlerror();
      return;
    }
#define KORCH_LOADN(name)                                                        \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, #name));              \
  if (!api.name) { api.err = std::string("missing symbol ") + #name; return; }
    KORCH_LOADN(nvrtcCreateProgram)
    KORCH_LOADN(nvrtcCompileProgram)
    KORCH_LOADN(nvrtcDestroyProgram)
    KORCH_LOADN(nvrtcGetProgramLogSize)
    KORCH_LOADN(nvrtcGetProgramLog)
    KORCH_LOADN(nvrtcGetCUBINSize)
    KORCH_LOADN(nvrtcGetCUBIN)
    KORCH_LOADN(nvrtcGetErrorString)
    KORCH_LOADN(nvrtcVersion)
#undef KORCH_LOADN
    api.ok = true;
  });
  return api;
}

std::string cu_err(CUresult r) {
  const char* s = nullptr;
  if (cuda().cuGetErrorString) cuda().cuGetErrorString(r, &s);
  return std::string("CUDA error ") + std::to_string((int)r) + (s ? std::string(": ") + s : "");
}

}  // namespace korch
