// Host helpers: error reporting, TMA descriptor encoding, device properties.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "host.cuh"

namespace aqb {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

const char* last_error() { return g_err; }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

static std::atomic<int> g_pdl{-1};

bool pdl_enabled() {
  int on = g_pdl.load(std::memory_order_relaxed);
  if (on < 0) {
    const char* e = getenv("AQB_PDL");
    int want = (e && e[0] == '0') ? 0 : 1;
    g_pdl.compare_exchange_strong(on, want);
    on = g_pdl.load(std::memory_order_relaxed);
  }
  return on == 1;
}

int set_pdl(int on) {
  const int prev = pdl_enabled() ? 1 : 0;
  g_pdl.store(on ? 1 : 0, std::memory_order_relaxed);
  return prev;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  return make_tmap(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, rank, dims, strides_bytes, box, swz);
}

int make_tmap(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return set_error(AQB_ECUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (reinterpret_cast<uintptr_t>(base) % 16) return set_error(AQB_EINVAL, "TMA base pointer not 16B aligned");
  cuuint64_t gdim[5], gstride[4];
  cuuint32_t bdim[5], estride[5];
  for (int i = 0; i < rank; ++i) {
    gdim[i] = dims[i];
    bdim[i] = box[i];
    estride[i] = 1;
    if (i > 0) {
      if (strides_bytes[i - 1] % 16) return set_error(AQB_EINVAL, "TMA stride not a multiple of 16 bytes");
      gstride[i - 1] = strides_bytes[i - 1];
    }
  }
  CUresult r = fn(map, dtype, rank, const_cast<void*>(base), gdim, gstride, bdim,
                  estride, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(AQB_ECUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", int(r));
  return AQB_OK;
}

}  // namespace aqb

extern "C" {

int aqb_abi_version(void) { return AQB_ABI_VERSION; }

#ifndef AQB_HEADER_HASH
#define AQB_HEADER_HASH "unknown"
#endif
const char* aqb_build_id(void) { return AQB_HEADER_HASH; }

const char* aqb_last_error(void) { return aqb::last_error(); }

int aqb_sm_count(void) { return aqb::sm_count(); }
int aqb_set_pdl(int on) { return aqb::set_pdl(on); }

}  // extern "C"
