// fp32 validation mode (north_star: per-step latent rel-L2 <= 1e-4 against the
// CPU reference).  The product path computes bf16 x bf16 -> fp32 on tcgen05;
// this mode keeps every activation in fp32 so the only difference from the
// fp32 oracle is summation order.  Weights are the same bf16-valued tensors the
// oracle uses (exact in fp32).  These are plain SIMT kernels — correctness
// instruments for small geometries, not a second fast path.
#include <cmath>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {
namespace f32 {

constexpr int TM = 64, TN = 64, TK = 16;

__device__ __forceinline__ float gelu_precise(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}

// out[m, n] (f32) = epi(sum_k A[m, k] * W[n, k] + bias[n]); A f32, W bf16 (nn.Linear layout).
__global__ void __launch_bounds__(256) gemm_kernel(const float* __restrict__ A, int64_t lda,
                                                   const __nv_bfloat16* __restrict__ W, int64_t ldw,
                                                   float* __restrict__ out, int64_t ldo, int M, int N, int K,
                                                   const float* __restrict__ bias, const float* __restrict__ gate,
                                                   int epi, const float* __restrict__ alpha, float* __restrict__ aux,
                                                   int64_t ld_aux, const int32_t* flag, int32_t run_if) {
  if (!gate_open(flag, run_if)) return;
  __shared__ float As[TK][TM + 4];
  __shared__ float Ws[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + 256 * i;  // 1024 elements of each 64 x 16 tile
      const int r = e / TK, c = e % TK;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[static_cast<int64_t>(gm) * lda + gk] : 0.f;
      Ws[c][r] = (gn < N && gk < K) ? __bfloat162float(W[static_cast<int64_t>(gn) * ldw + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i], b[i] = Ws[kk][tx * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const float al = (epi == AQB_EPI_EULER) ? *alpha : 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] + (bias ? bias[n] : 0.f);
      float* o = out + static_cast<int64_t>(m) * ldo + n;
      switch (epi) {
        case AQB_EPI_GELU_BF16: *o = gelu_precise(v); break;
        case AQB_EPI_GATE_RES: {
          const float x = *o + (gate ? gate[n] : 1.f) * v;
          *o = x;
          if (aux) aux[static_cast<int64_t>(m) * ld_aux + n] = x;
          break;
        }
        case AQB_EPI_EULER: {
          const float x = *o + al * v;
          *o = x;
          if (aux) aux[static_cast<int64_t>(m) * ld_aux + n] = x;
          break;
        }
        default: *o = v;
      }
    }
  }
}

// Non-causal attention in fp32: CTA = 16 queries of one head, 8 warps x 2 queries;
// 32-key K/V tiles in smem, lane = key for the scores, lane = output column for PV.
template <int D>
__global__ void __launch_bounds__(256) attention_kernel(const float* __restrict__ q, int64_t ldq, int64_t qhs,
                                                        const float* __restrict__ k, int64_t ldk, int64_t khs,
                                                        const float* __restrict__ v, int64_t ldv, int64_t vhs,
                                                        float* __restrict__ o, int64_t ldo, int64_t ohs, int Sq,
                                                        int Skv, float scale, const int32_t* flag, int32_t run_if) {
  if (!gate_open(flag, run_if)) return;
  constexpr int QW = 2, QB = 8 * QW;  // queries per warp / per CTA
  __shared__ float Qs[QB][D];
  __shared__ float Ks[32][D + 1];
  __shared__ float Vs[32][D];
  const int head = blockIdx.y, q0 = blockIdx.x * QB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < QB * D; e += 256) {
    const int r = e / D, c = e % D;
    Qs[r][c] = (q0 + r < Sq) ? q[static_cast<int64_t>(q0 + r) * ldq + head * qhs + c] : 0.f;
  }
  constexpr int NJ = D / 32;
  float m_run[QW], l_run[QW], acc[QW][NJ];
#pragma unroll
  for (int i = 0; i < QW; ++i) {
    m_run[i] = -INFINITY, l_run[i] = 0.f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = 0.f;
  }
  for (int k0 = 0; k0 < Skv; k0 += 32) {
    __syncthreads();
    for (int e = tid; e < 32 * D; e += 256) {
      const int r = e / D, c = e % D;
      const bool ok = k0 + r < Skv;
      Ks[r][c] = ok ? k[static_cast<int64_t>(k0 + r) * ldk + head * khs + c] : 0.f;
      Vs[r][c] = ok ? v[static_cast<int64_t>(k0 + r) * ldv + head * vhs + c] : 0.f;
    }
    __syncthreads();
    const bool valid = k0 + lane < Skv;
#pragma unroll
    for (int i = 0; i < QW; ++i) {
      const int qi = warp * QW + i;
      float s = 0.f;
#pragma unroll 8
      for (int d = 0; d < D; ++d) s = fmaf(Qs[qi][d], Ks[lane][d], s);
      s = valid ? s * scale : -INFINITY;
      float mx = s;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_run[i], mx);
      const float corr = expf(m_run[i] - m_new);
      const float p = valid ? expf(s - m_new) : 0.f;
      float ps = p;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      l_run[i] = l_run[i] * corr + ps;
      m_run[i] = m_new;
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j] *= corr;
      for (int kk = 0; kk < 32; ++kk) {
        const float pk = __shfl_sync(0xffffffffu, p, kk);
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j] = fmaf(pk, Vs[kk][lane + 32 * j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < QW; ++i) {
    const int row = q0 + warp * QW + i;
    if (row >= Sq) continue;
    const float inv = 1.f / l_run[i];
#pragma unroll
    for (int j = 0; j < NJ; ++j) o[static_cast<int64_t>(row) * ldo + head * ohs + lane + 32 * j] = acc[i][j] * inv;
  }
}

}  // namespace f32
}  // namespace aqb

extern "C" int aqb_gemm_f32(const float* a, int64_t lda, const void* w, int64_t ldw, float* out, int64_t ldo,
                            int64_t m, int64_t n, int64_t k, const float* bias, const float* gate, int32_t epilogue,
                            const float* alpha, float* aux, int64_t ld_aux, const int32_t* run_flag, int32_t run_if,
                            void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(a && w && out, "gemm_f32: null pointer");
  AQB_CHECK_ARG(m >= 1 && n >= 1 && k >= 1 && m < (1ll << 31) && n < (1ll << 31), "gemm_f32: bad shape");
  AQB_CHECK_ARG(lda >= k && ldw >= k && ldo >= n, "gemm_f32: bad strides");
  AQB_CHECK_ARG(epilogue >= 0 && epilogue <= AQB_EPI_EULER, "gemm_f32: bad epilogue");
  AQB_CHECK_ARG(epilogue != AQB_EPI_EULER || alpha, "gemm_f32: EULER needs alpha");
  dim3 grid(unsigned((n + f32::TN - 1) / f32::TN), unsigned((m + f32::TM - 1) / f32::TM));
  f32::gemm_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      a, lda, reinterpret_cast<const __nv_bfloat16*>(w), ldw, out, ldo, int(m), int(n), int(k), bias, gate, epilogue,
      alpha, aux, ld_aux, run_flag, run_if);
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_attention_f32(const float* q, int64_t ldq, int64_t q_head_stride, const float* k, int64_t ldk,
                                 int64_t k_head_stride, const float* v, int64_t ldv, int64_t v_head_stride, float* o,
                                 int64_t ldo, int64_t o_head_stride, int64_t seq_q, int64_t seq_kv, int32_t heads,
                                 int32_t head_dim, float softmax_scale, const int32_t* run_flag, int32_t run_if,
                                 void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(q && k && v && o, "attention_f32: null pointer");
  AQB_CHECK_ARG(seq_q >= 1 && seq_kv >= 1 && heads >= 1 && seq_q < (1ll << 31) && seq_kv < (1ll << 31),
                "attention_f32: bad shape");
  dim3 grid(unsigned((seq_q + 15) / 16), unsigned(heads));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define F32_ATTN(D)                                                                                                 \
  f32::attention_kernel<D><<<grid, 256, 0, s>>>(q, ldq, q_head_stride, k, ldk, k_head_stride, v, ldv, v_head_stride, \
                                                o, ldo, o_head_stride, int(seq_q), int(seq_kv), softmax_scale,        \
                                                run_flag, run_if)
  switch (head_dim) {
    case 32: F32_ATTN(32); break;
    case 64: F32_ATTN(64); break;
    case 128: F32_ATTN(128); break;
    default: return set_error(AQB_EUNSUPPORTED, "attention_f32: head_dim %d unsupported", head_dim);
  }
#undef F32_ATTN
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}
