// CUDA driver API + NVRTC, loaded with dlopen so that libkorch.so loads (and can
// enumerate / generate / compile) on machines without a GPU driver.
#pragma once
#include <cuda.h>
#include <nvrtc.h>

#include <string>

namespace korch {

#define KORCH_CU_FUNCS(X)                                                                          \
  X(cuInit) X(cuDeviceGet) X(cuDeviceGetAttribute) X(cuDeviceGetName) X(cuDevicePrimaryCtxRetain)   \
  X(cuDevicePrimaryCtxRelease) X(cuCtxSetCurrent) X(cuCtxGetCurrent) X(cuCtxSynchronize)           \
  X(cuModuleLoadData) X(cuModuleUnload) X(cuModuleGetFunction) X(cuFuncSetAttribute)               \
  X(cuLaunchKernel) X(cuLaunchKernelEx) X(cuMemAlloc) X(cuMemFree) X(cuMemsetD8Async)              \
  X(cuMemsetD16Async) X(cuMemsetD32Async) X(cuStreamCreate) X(cuStreamDestroy)                     \
  X(cuStreamSynchronize) X(cuEventCreate) X(cuEventDestroy) X(cuEventRecord)                       \
  X(cuEventSynchronize) X(cuEventElapsedTime) X(cuStreamBeginCapture) X(cuStreamEndCapture)        \
  X(cuGraphInstantiateWithFlags) X(cuGraphLaunch) X(cuGraphExecDestroy) X(cuGraphDestroy)          \
  X(cuGetErrorString) X(cuTensorMapEncodeTiled) X(cuMemcpyHtoD) X(cuMemcpyDtoH)                 \
  X(cuMemcpyHtoDAsync) X(cuMemcpyDtoHAsync) X(cuPointerGetAttribute) X(cuEventRecordWithFlags) X(cuStreamWaitEvent)

struct CudaApi {
#define KORCH_DECL(name) decltype(&::name) name = nullptr;
  KORCH_CU_FUNCS(KORCH_DECL)
#undef KORCH_DECL
  bool ok = false;
  std::string err;
};

struct NvrtcApi {
  decltype(&::nvrtcCreateProgram) nvrtcCreateProgram = nullptr;
  decltype(&::nvrtcCompileProgram) nvrtcCompileProgram = nullptr;
  decltype(&::nvrtcDestroyProgram) nvrtcDestroyProgram = nullptr;
  decltype(&::nvrtcGetProgramLogSize) nvrtcGetProgramLogSize = nullptr;
  decltype(&::nvrtcGetProgramLog) nvrtcGetProgramLog = nullptr;
  decltype(&::nvrtcGetCUBINSize) nvrtcGetCUBINSize = nullptr;
  decltype(&::nvrtcGetCUBIN) nvrtcGetCUBIN = nullptr;
  decltype(&::nvrtcGetErrorString) nvrtcGetErrorString = nullptr;
  decltype(&::nvrtcVersion) nvrtcVersion = nullptr;
  bool ok = false;
  std::string err;
};

CudaApi& cuda();    // loads on first use; check .ok
NvrtcApi& nvrtc();  // loads on first use; check .ok
std::string cu_err(CUresult r);

}  // namespace korch
