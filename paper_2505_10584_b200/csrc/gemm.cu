// tcgen05 / TMEM / TMA persistent GEMM with fused DiT epilogues (sm_100a).
//
//   acc[m, n] = sum_k A[m, k] * W[n, k]        A: activations, W: nn.Linear weight
//
// Implements the projection rows of the paper's Table 2 with
// GeLU and Gate fused into the epilogue, plus the
// flow-matching Euler update for the final layer.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A[128 x 64] + W[BN x 64] per k-block into a
//               STAGES-deep ring (128B swizzle), mbarrier full/empty.
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128,
//               N=BN, K=16) into one of two TMEM accumulators (2 x BN columns),
//               tcgen05.commit frees smem stages / signals the epilogue.
//   warp 2      TMEM allocator.
//   warps 4-7   epilogue: tcgen05.ld 32 columns at a time (thread = row),
//               bias / GeLU / gate*residual / Euler, vectorised global stores;
//               overlaps the MMA of the next tile (double-buffered TMEM).
#include <cmath>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int kThreads = 256;

struct Params {
  int M, N, K;
  int num_m, num_n, num_tiles, group_m;
  void* out;
  int64_t ldo;
  const float* bias;
  const float* gate;
  const float* alpha;
  __nv_bfloat16* aux;
  int64_t ld_aux;
  const int32_t* run_flag;
  int32_t run_if;
};

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mb, int& nb) {
  const int per_group = p.group_m * p.num_n;
  const int g = t / per_group;
  const int first_m = g * p.group_m;
  const int gsz = min(p.num_m - first_m, p.group_m);
  const int r = t - g * per_group;
  mb = first_m + r % gsz;
  nb = r / gsz;
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
  return STAGES * (BM + BN) * BK * 2 + 1024 /*align slack*/ + 256 /*barriers*/;
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const Params& p, int row, int col0, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (p.bias != nullptr) {
    const float4* b4 = reinterpret_cast<const float4*>(p.bias + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (col0 + 4 * i < p.N) {
        float4 b = __ldg(b4 + i);
        v[4 * i] += b.x, v[4 * i + 1] += b.y, v[4 * i + 2] += b.z, v[4 * i + 3] += b.w;
      }
    }
  }
  if (row >= p.M) return;
  if constexpr (EPI == AQB_EPI_BF16 || EPI == AQB_EPI_GELU_BF16) {
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out) + static_cast<int64_t>(row) * p.ldo + col0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (col0 + 8 * i < p.N) {
        float t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = (EPI == AQB_EPI_GELU_BF16) ? gelu_tanh(v[8 * i + j]) : v[8 * i + j];
        uint4 pk = make_uint4(pack_bf16(t[0], t[1]), pack_bf16(t[2], t[3]), pack_bf16(t[4], t[5]),
                              pack_bf16(t[6], t[7]));
        *reinterpret_cast<uint4*>(out + 8 * i) = pk;
      }
    }
  } else if constexpr (EPI == AQB_EPI_F32) {
    float* out = reinterpret_cast<float*>(p.out) + static_cast<int64_t>(row) * p.ldo + col0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (col0 + 4 * i < p.N)
        *reinterpret_cast<float4*>(out + 4 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else if constexpr (EPI == AQB_EPI_GATE_RES) {
    float* out = reinterpret_cast<float*>(p.out) + static_cast<int64_t>(row) * p.ldo + col0;
    const float4* g4 = reinterpret_cast<const float4*>(p.gate + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (col0 + 4 * i < p.N) {
        float4 x = *reinterpret_cast<float4*>(out + 4 * i);
        float4 g = p.gate ? __ldg(g4 + i) : make_float4(1.f, 1.f, 1.f, 1.f);
        x.x += g.x * v[4 * i];
        x.y += g.y * v[4 * i + 1];
        x.z += g.z * v[4 * i + 2];
        x.w += g.w * v[4 * i + 3];
        *reinterpret_cast<float4*>(out + 4 * i) = x;
      }
    }
  } else if constexpr (EPI == AQB_EPI_EULER) {
    const float a = __ldg(p.alpha);
    float* out = reinterpret_cast<float*>(p.out) + static_cast<int64_t>(row) * p.ldo + col0;
    __nv_bfloat16* aux = p.aux + static_cast<int64_t>(row) * p.ld_aux + col0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (col0 + 8 * i < p.N) {
        float4 x0 = *reinterpret_cast<float4*>(out + 8 * i);
        float4 x1 = *reinterpret_cast<float4*>(out + 8 * i + 4);
        x0.x += a * v[8 * i + 0], x0.y += a * v[8 * i + 1], x0.z += a * v[8 * i + 2], x0.w += a * v[8 * i + 3];
        x1.x += a * v[8 * i + 4], x1.y += a * v[8 * i + 5], x1.z += a * v[8 * i + 6], x1.w += a * v[8 * i + 7];
        *reinterpret_cast<float4*>(out + 8 * i) = x0;
        *reinterpret_cast<float4*>(out + 8 * i + 4) = x1;
        if (p.aux)
          *reinterpret_cast<uint4*>(aux + 8 * i) = make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w),
                                                              pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
      }
    }
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b, Params p) {
  if (!gate_open(p.run_flag, p.run_if)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(base);
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(base + STAGES * BM * BK * 2);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * (BM + BN) * BK * 2);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  constexpr uint32_t kTmemCols = 2 * BN;
  const uint32_t warp = warp_idx(), lane = lane_idx();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = (p.K + BK - 1) / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, (BM + BN) * BK * 2);
          tma_load_2d(sa + stage * BM * BK, &tma_a, full + stage, kb * BK, mb * BM);
          tma_load_2d(sb + stage * BN * BK, &tma_b, full + stage, kb * BK, nb * BN);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdesc = idesc_bf16(BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + stage * BM * BK);
          const uint32_t b0 = smem_u32(sb + stage * BN * BK);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major SW128: +32 B per 16-element K step inside the 128 B swizzle row.
            umma_bf16_ss(d, smem_desc(a0 + 32 * k, 0, 1024), smem_desc(b0 + 32 * k, 0, 1024), kIdesc,
                         (kb | k) != 0);
          }
          umma_commit(empty + stage);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        umma_commit(tfull + acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int row = mb * BM + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        const int col0 = nb * BN + c;
        if (col0 >= p.N) break;  // warp-uniform
        uint32_t r[32];
        tmem_ld32(tmem + acc * BN + c + ((q * 32) << 16), r);
        tmem_wait_ld();
        epilogue_chunk<EPI>(p, row, col0, r);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

template <int BN, int STAGES, int EPI>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, cudaStream_t stream) {
  constexpr int smem = smem_bytes<BN, STAGES>();
  static bool configured = false;  // per instantiation; attribute is per-function
  if (!configured) {
    AQB_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<BN, STAGES, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  const int grid = p.num_tiles < sm_count() ? p.num_tiles : sm_count();
  gemm_kernel<BN, STAGES, EPI><<<grid, kThreads, smem, stream>>>(ta, tb, p);
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

template <int BN, int STAGES>
int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p, cudaStream_t s) {
  switch (epi) {
    case AQB_EPI_BF16: return launch<BN, STAGES, AQB_EPI_BF16>(ta, tb, p, s);
    case AQB_EPI_GELU_BF16: return launch<BN, STAGES, AQB_EPI_GELU_BF16>(ta, tb, p, s);
    case AQB_EPI_GATE_RES: return launch<BN, STAGES, AQB_EPI_GATE_RES>(ta, tb, p, s);
    case AQB_EPI_F32: return launch<BN, STAGES, AQB_EPI_F32>(ta, tb, p, s);
    case AQB_EPI_EULER: return launch<BN, STAGES, AQB_EPI_EULER>(ta, tb, p, s);
  }
  return set_error(AQB_EINVAL, "unknown epilogue %d", epi);
}

// Pick the N tile: 256 (lower smem-operand traffic per MMA) unless it leaves
// the last wave badly under-filled relative to 128.
static int pick_bn(int64_t m, int64_t n) {
  if (n <= 128) return 128;
  const int sms = sm_count();
  auto eff = [&](int bn) {
    const double tiles = double((m + BM - 1) / BM) * double((n + bn - 1) / bn);
    const double waves = tiles / sms;
    const double used = tiles * bn;  // useful-ish work units
    return used / (std::ceil(waves) * sms * bn) * (bn == 256 ? 1.0 : 0.9);  // 128-wide tiles pay smem bw
  };
  return eff(256) >= eff(128) ? 256 : 128;
}

}  // namespace gemm
}  // namespace aqb

extern "C" int aqb_gemm_bf16(const void* a, int64_t lda, const void* w, int64_t ldw, void* out, int64_t ldo,
                             int64_t m, int64_t n, int64_t k, const float* bias, const float* gate, int32_t epilogue,
                             const float* alpha, void* aux, int64_t ld_aux, const int32_t* run_flag, int32_t run_if,
                             void* stream) {
  using namespace aqb;
  using namespace aqb::gemm;
  AQB_CHECK_ARG(a && w && out, "gemm: null pointer");
  AQB_CHECK_ARG(m >= 1 && n >= 1 && k >= 1, "gemm: bad shape m=%lld n=%lld k=%lld", (long long)m, (long long)n,
                (long long)k);
  AQB_CHECK_ARG(k % 8 == 0 && n % 16 == 0, "gemm: need k %% 8 == 0 and n %% 16 == 0 (k=%lld n=%lld)",
                (long long)k, (long long)n);
  AQB_CHECK_ARG(lda % 8 == 0 && ldw % 8 == 0 && lda >= k && ldw >= k, "gemm: bad lda/ldw");
  AQB_CHECK_ARG(epilogue >= 0 && epilogue <= AQB_EPI_EULER, "gemm: bad epilogue");
  AQB_CHECK_ARG(epilogue != AQB_EPI_EULER || alpha != nullptr, "gemm: EULER needs alpha");
  AQB_CHECK_ARG(ldo >= n && ldo % 8 == 0, "gemm: bad ldo");
  AQB_CHECK_ARG(m < (1ll << 31) && n < (1ll << 31), "gemm: shape too large");

  const int bn = pick_bn(m, n);
  CUtensorMap ta, tb;
  {
    uint64_t dims[2] = {uint64_t(k), uint64_t(m)};
    uint64_t strides[1] = {uint64_t(lda) * 2};
    uint32_t box[2] = {BK, BM};
    int rc = make_tmap_bf16(&ta, a, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    uint64_t dims[2] = {uint64_t(k), uint64_t(n)};
    uint64_t strides[1] = {uint64_t(ldw) * 2};
    uint32_t box[2] = {BK, uint32_t(bn)};
    int rc = make_tmap_bf16(&tb, w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  Params p{};
  p.M = int(m), p.N = int(n), p.K = int(k);
  p.num_m = int((m + BM - 1) / BM);
  p.num_n = int((n + bn - 1) / bn);
  p.num_tiles = p.num_m * p.num_n;
  p.group_m = 16;
  p.out = out, p.ldo = ldo, p.bias = bias, p.gate = gate, p.alpha = alpha;
  p.aux = reinterpret_cast<__nv_bfloat16*>(aux), p.ld_aux = ld_aux;
  p.run_flag = run_flag, p.run_if = run_if;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (bn == 256) return dispatch_epi<256, 4>(epilogue, ta, tb, p, s);
  return dispatch_epi<128, 6>(epilogue, ta, tb, p, s);
}
