// Host-side helpers shared by the C-ABI entry points: status codes, the
// thread-local last-error string, TMA descriptor encoding (driver entry point
// fetched through the runtime, so the library does not link libcuda), and
// per-device properties.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <cstdarg>
#include <mutex>
#include <utility>

#include "../../include/aqb.h"

namespace aqb {

int set_error(int code, const char* fmt, ...);
const char* last_error();

#define AQB_CHECK_ARG(cond, ...)                         \
  do {                                                   \
    if (!(cond)) return ::aqb::set_error(AQB_EINVAL, __VA_ARGS__); \
  } while (0)

#define AQB_CUDA_TRY(expr)                                                                         \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess)                                                                         \
      return ::aqb::set_error(AQB_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                              __LINE__);                                                           \
  } while (0)

#define AQB_LAUNCH_CHECK()                                                                      \
  do {                                                                                          \
    cudaError_t _e = cudaGetLastError();                                                        \
    if (_e != cudaSuccess)                                                                      \
      return ::aqb::set_error(AQB_ECUDA, "launch failed: %s (%s:%d)", cudaGetErrorString(_e), __FILE__, \
                              __LINE__);                                                        \
  } while (0)

int sm_count();

// Launch with programmatic stream serialization (PDL) unless AQB_PDL=0: the kernel
// must call pdl_wait() before reading anything the previous kernel wrote.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel *and device*: the
// attribute is per-device state, so a process driving several GPUs must set it on each.
// Lock-free and reentrant (a race just repeats the idempotent call).
struct FuncAttrOnce {
  std::atomic<uint64_t> devices{0};  // bit d: set on device d
};

template <typename K>
cudaError_t set_smem_once(FuncAttrOnce& once, K kern, int smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (once.devices.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) once.devices.fetch_or(bit, std::memory_order_release);
  return e;
}

// Encode a bf16 tensor map with 128B swizzle.  dims/strides innermost first;
// strides in bytes for dims 1..rank-1.  Returns 0 or a negative status.
int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);
int make_tmap(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);

}  // namespace aqb
