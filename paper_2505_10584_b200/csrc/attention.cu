// tcgen05 / TMEM / TMA flash-attention forward (sm_100a), non-causal.
//
// The paper's hottest op: "Flash Attention" of Table 2 — full
// 3D attention over video (+ text) tokens.  RoPE/QK-norm
// are applied by the producer of Q/K (aqb_qk_norm_rope) so this kernel reads
// Q/K/V straight from the QKV-projection layout with TMA (no transposes).
//
// One CTA = one head x 256 queries (two 128-row Q tiles ping-ponged so the
// tensor core always has the other tile's work while one tile's softmax runs).
//   warp 0      TMA producer: Q0, Q1 once; K_j, V_j through an NS-deep ring.
//   warp 1      MMA issuer (one thread):  S_t = Q_t K_j^T  (SS, M=128 N=128)
//               O_t += P_t V_j  (P from smem K-major, V MN-major, N=D).
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: thread = query
//               row (TMEM lane), 224 registers each (setmaxnreg).  Online
//               softmax in the exp2 domain: scale folded into one packed
//               FFMA2 per pair, 3/8 of the exponentials evaluated by a
//               degree-3 polynomial on the FMA pipe (the rest on MUFU) so
//               neither pipe caps the tensor core; lazy rescaling (only when
//               the running max grows by > 8, so O in TMEM is rarely
//               touched); P written with st.shared.v4 in the 128B-swizzled
//               K-major layout the MMA reads; final 1/l normalisation and
//               bf16 store from the same warps.
// TMEM: S0 | S1 | O0 | O1  (128 + 128 + D + D columns).
#include <cmath>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {
namespace attn {

constexpr int BQ = 128;   // rows per Q tile (MMA M)
constexpr int BKV = 128;  // keys per KV tile (MMA N of QK^T, K of PV)
constexpr int kThreads = 384;    // 3 warpgroups: control | softmax tile 0 | softmax tile 1
constexpr uint32_t kCtrlRegs = 56;     // setmaxnreg budgets: 56 + 2 * 224 <= 512 per SMSP
constexpr uint32_t kSoftmaxRegs = 224;
constexpr uint32_t kPolyMask = 0x52;   // pairs (i & 7) in {1,4,6}: exp2 by polynomial (3/8 off the MUFU)

template <int D>
struct Cfg {
  static constexpr int NS = D == 128 ? 3 : 4;                // K/V ring depth
  static constexpr int kQBytes = BQ * D * 2;                 // one Q tile
  static constexpr int kKVBytes = BKV * D * 2;               // one K or V tile
  static constexpr int kPBytes = BQ * BKV * 2;               // one P tile
  static constexpr int kOffQ = 0;
  static constexpr int kOffKV = 2 * kQBytes;
  static constexpr int kOffP = kOffKV + NS * kKVBytes;
  static constexpr int kOffBar = kOffP + 2 * kPBytes;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr int kBoxes = D / 64;                      // 64-column TMA boxes per row
};

struct Params {
  int seq_q, seq_kv, heads, head_dim;
  float scale_log2;
  __nv_bfloat16* o;
  int64_t ldo, o_head_stride;
  const int32_t* run_flag;
  int32_t run_if;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, Params p) {
  using C = Cfg<D>;
  if (!gate_open(p.run_flag, p.run_if)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base + C::kOffQ;
  uint8_t* sKV = base + C::kOffKV;
  uint8_t* sP = base + C::kOffP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::kOffBar);
  uint64_t* q_full = bars;              // 1
  uint64_t* kv_full = bars + 1;         // NS
  uint64_t* kv_empty = kv_full + C::NS; // NS
  uint64_t* s_full = kv_empty + C::NS;  // 2
  uint64_t* p_full = s_full + 2;        // 2
  uint64_t* o_ready = p_full + 2;       // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_ready + 2);

  const uint32_t warp = warp_idx(), lane = lane_idx();
  const int head = blockIdx.y;
  const int q0 = blockIdx.x * (2 * BQ);
  const int nkv = (p.seq_kv + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    mbar_init(q_full, 1);
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(kv_full + s, 1);
      mbar_init(kv_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_full + t, 1);
      mbar_init(p_full + t, 128);
      mbar_init(o_ready + t, 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    setmaxnreg_dec<kCtrlRegs>();
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * C::kQBytes);
      for (int t = 0; t < 2; ++t)
        for (int c = 0; c < C::kBoxes; ++c)
          tma_load_3d(sQ + t * C::kQBytes + c * (BQ * 128), &tq, q_full, c * 64, head, q0 + t * BQ, kEvictFirst);
      for (int i = 0; i < 2 * nkv; ++i) {
        const int s = i % C::NS;
        const uint32_t ph = (i / C::NS) & 1;
        mbar_wait(kv_empty + s, ph ^ 1);
        mbar_arrive_expect_tx(kv_full + s, C::kKVBytes);
        const CUtensorMap* m = (i & 1) ? &tv : &tk;
        const int row = (i >> 1) * BKV;
        for (int c = 0; c < C::kBoxes; ++c)
          tma_load_3d(sKV + s * C::kKVBytes + c * (BKV * 128), m, kv_full + s, c * 64, head, row, kEvictLast);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    setmaxnreg_dec<kCtrlRegs>();
    if (lane == 0) {
      constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV, 0, 0);  // Q, K both K-major
      constexpr uint32_t kIdescO = idesc_bf16(BQ, D, 0, 1);    // P K-major, V MN-major
      const uint32_t q_addr = smem_u32(sQ), kv_addr = smem_u32(sKV), p_addr = smem_u32(sP);
      auto issue_qk = [&](int t, int stage) {
        const uint32_t a0 = q_addr + t * C::kQBytes, b0 = kv_addr + stage * C::kKVBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (BQ * 128) + (kk & 3) * 32;
          umma_bf16_ss(tmem + t * 128, smem_desc(a0 + off, 0, 1024), smem_desc(b0 + off, 0, 1024), kIdescS, kk > 0);
        }
      };
      auto issue_pv = [&](int t, int stage, bool acc) {
        const uint32_t a0 = p_addr + t * C::kPBytes, b0 = kv_addr + stage * C::kKVBytes;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * (BQ * 128) + (kk & 3) * 32;
          const uint32_t boff = kk * 16 * 128;  // 16 keys x 128 B rows
          umma_bf16_ss(tmem + 256 + t * D, smem_desc(a0 + aoff, 0, 1024), smem_desc(b0 + boff, BKV * 128, 1024),
                       kIdescO, (acc || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= nkv; ++j) {
        const int ik = 2 * j, iv = 2 * (j - 1) + 1;  // ring indices of K_j and V_{j-1}
        if (j < nkv) {
          mbar_wait(kv_full + ik % C::NS, (ik / C::NS) & 1);
          tc_fence_after();
        }
        if (j > 0) {
          mbar_wait(kv_full + iv % C::NS, (iv / C::NS) & 1);
          mbar_wait(p_full + 0, (j - 1) & 1);
          tc_fence_after();
          issue_pv(0, iv % C::NS, j > 1);
          umma_commit(o_ready + 0);
        }
        if (j < nkv) {
          issue_qk(0, ik % C::NS);
          umma_commit(s_full + 0);
        }
        if (j > 0) {
          mbar_wait(p_full + 1, (j - 1) & 1);
          tc_fence_after();
          issue_pv(1, iv % C::NS, j > 1);
          umma_commit(o_ready + 1);
          umma_commit(kv_empty + iv % C::NS);
        }
        if (j < nkv) {
          issue_qk(1, ik % C::NS);
          umma_commit(s_full + 1);
          umma_commit(kv_empty + ik % C::NS);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    setmaxnreg_inc<kSoftmaxRegs>();
    const int t = (warp - 4) / 4;             // Q tile of this warpgroup
    const uint32_t quad = warp & 3;           // TMEM lane quadrant
    const int r = quad * 32 + lane;           // row within the tile
    const uint32_t lane_base = (quad * 32) << 16;
    const uint32_t s_tmem = tmem + lane_base + t * 128;
    const uint32_t o_tmem = tmem + lane_base + 256 + t * D;
    const uint32_t prow = smem_u32(sP + t * C::kPBytes + r * 128);
    const uint32_t sw = r & 7;
    const float c = p.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    const uint64_t kM = f2pack(12582912.f, 12582912.f);  // 1.5 * 2^23: round-to-nearest
    const uint64_t kC0 = f2pack(0.99992806f, 0.99992806f), kC1 = f2pack(0.69326103f, 0.69326103f);
    const uint64_t kC2 = f2pack(0.24261117f, 0.24261117f), kC3 = f2pack(0.05517162f, 0.05517162f);
    float m_run = -INFINITY, l_run = 0.f;     // m_run in raw score units

    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full + t, j & 1);
      tc_fence_after();
      uint32_t sr[BKV];
      tmem_ld64(s_tmem, sr);
      tmem_ld64(s_tmem + 64, sr + 64);
      tmem_wait_ld();
      const int kv_valid = p.seq_kv - j * BKV;
      if (kv_valid < BKV) {
#pragma unroll
        for (int i = 0; i < BKV; ++i)
          if (i >= kv_valid) sr[i] = 0xff800000u;  // -inf
      }
      float mx = __uint_as_float(sr[0]);
#pragma unroll
      for (int i = 1; i + 1 < BKV; i += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])));
      mx = fmaxf(mx, __uint_as_float(sr[BKV - 1]));
      // PV_{j-1} must be done before O is rescaled or P_t overwritten.
      if (j > 0) {
        mbar_wait(o_ready + t, (j - 1) & 1);
        tc_fence_after();
      }
      // lazy rescale: only when the running max grows by more than 2^8 in exp2 units
      const bool need = (mx - m_run) * c > 8.f;
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? mx : m_run;
        const float alpha = need ? ex2((m_run - m_new) * c) : 1.f;
        if (j > 0) {
#pragma unroll 1
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t u[32];
            tmem_ld32(o_tmem + cc * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
            tmem_st32(o_tmem + cc * 32, u);
          }
          tmem_wait_st();
        }
        l_run *= alpha;
        m_run = m_new;
      }
      const float nm = -m_run * c;
      const uint64_t nm2 = f2pack(nm, nm);
      uint64_t acc2 = f2pack(0.f, 0.f);
#pragma unroll
      for (int kc = 0; kc < BKV / 8; ++kc) {  // 16-byte chunks of the P row
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int pi = kc * 4 + q;
          const uint64_t x2 = ffma2(f2pack(__uint_as_float(sr[2 * pi]), __uint_as_float(sr[2 * pi + 1])), c2, nm2);
          float x0, x1, p0, p1;
          f2unpack(x2, x0, x1);
          if ((kPolyMask >> (pi & 7)) & 1) {
            // exp2 on the FMA pipe: 2^x = 2^round(x) * poly(x - round(x)), |rel err| < 8e-5
            const uint64_t xc = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
            const uint64_t tt = fadd2(xc, kM);
            const uint64_t fr = fsub2(xc, fsub2(tt, kM));
            uint64_t pp = ffma2(fr, kC3, kC2);
            pp = ffma2(pp, fr, kC1);
            pp = ffma2(pp, fr, kC0);
            float q0, q1, t0, t1;
            f2unpack(pp, q0, q1);
            f2unpack(tt, t0, t1);
            p0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
            p1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          acc2 = fadd2(acc2, f2pack(p0, p1));
          pk[q] = pack_bf16(p0, p1);
        }
        const int box = kc >> 3, cch = kc & 7;
        st_shared_v4(prow + box * (BQ * 128) + ((cch ^ sw) << 4), pk[0], pk[1], pk[2], pk[3]);
      }
      float a0, a1;
      f2unpack(acc2, a0, a1);
      l_run += a0 + a1;
      fence_proxy_async_smem();  // generic-proxy P stores -> visible to the tensor core
      tc_fence_before();
      mbar_arrive(p_full + t);
    }
    // epilogue: O / l -> bf16
    mbar_wait(o_ready + t, (nkv - 1) & 1);
    tc_fence_after();
    const int row = q0 + t * BQ + r;
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    __nv_bfloat16* orow = p.o + static_cast<int64_t>(head) * p.o_head_stride + static_cast<int64_t>(row) * p.ldo;
#pragma unroll 1
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t u[32];
      tmem_ld32(o_tmem + cc * 32, u);
      tmem_wait_ld();
      if (row < p.seq_q && cc * 32 < p.head_dim) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint4 pk = make_uint4(pack_bf16(__uint_as_float(u[8 * g]) * inv, __uint_as_float(u[8 * g + 1]) * inv),
                                      pack_bf16(__uint_as_float(u[8 * g + 2]) * inv, __uint_as_float(u[8 * g + 3]) * inv),
                                      pack_bf16(__uint_as_float(u[8 * g + 4]) * inv, __uint_as_float(u[8 * g + 5]) * inv),
                                      pack_bf16(__uint_as_float(u[8 * g + 6]) * inv, __uint_as_float(u[8 * g + 7]) * inv));
          *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * g) = pk;
        }
      }
    }
  } else {
    setmaxnreg_dec<kCtrlRegs>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
int launch(const void* q, int64_t ldq, int64_t qhs, const void* k, int64_t ldk, int64_t khs, const void* v,
           int64_t ldv, int64_t vhs, const Params& p, cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  const uint32_t box[3] = {64, 1, 128};
  {
    const uint64_t dims[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(p.seq_q)};
    const uint64_t str[2] = {uint64_t(qhs) * 2, uint64_t(ldq) * 2};
    int rc = make_tmap_bf16(&tq, q, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    const uint64_t dims[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(p.seq_kv)};
    const uint64_t str[2] = {uint64_t(khs) * 2, uint64_t(ldk) * 2};
    int rc = make_tmap_bf16(&tk, k, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    const uint64_t dims[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(p.seq_kv)};
    const uint64_t str[2] = {uint64_t(vhs) * 2, uint64_t(ldv) * 2};
    int rc = make_tmap_bf16(&tv, v, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  constexpr int smem = Cfg<D>::kSmem;
  static bool configured = false;
  if (!configured) {
    AQB_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  dim3 grid((p.seq_q + 2 * BQ - 1) / (2 * BQ), p.heads);
  attn_fwd_kernel<D><<<grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

}  // namespace attn
}  // namespace aqb

extern "C" int aqb_attention_fwd(const void* q, int64_t ldq, int64_t q_head_stride, const void* k, int64_t ldk,
                                 int64_t k_head_stride, const void* v, int64_t ldv, int64_t v_head_stride, void* o,
                                 int64_t ldo, int64_t o_head_stride, int64_t seq_q, int64_t seq_kv, int32_t heads,
                                 int32_t head_dim, float softmax_scale, const int32_t* run_flag, int32_t run_if,
                                 void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(q && k && v && o, "attention: null pointer");
  AQB_CHECK_ARG(head_dim == 32 || head_dim == 64 || head_dim == 128, "attention: head_dim %d unsupported", head_dim);
  AQB_CHECK_ARG(seq_q >= 1 && seq_kv >= 1 && heads >= 1, "attention: bad shape");
  AQB_CHECK_ARG(seq_q < (1ll << 31) && seq_kv < (1ll << 31), "attention: sequence too long");
  AQB_CHECK_ARG(ldq % 8 == 0 && ldk % 8 == 0 && ldv % 8 == 0 && ldo % 8 == 0, "attention: rows must be 16B aligned");
  AQB_CHECK_ARG(q_head_stride % 8 == 0 && k_head_stride % 8 == 0 && v_head_stride % 8 == 0 && o_head_stride % 8 == 0,
                "attention: head strides must be 16B aligned");
  attn::Params p{};
  p.seq_q = int(seq_q), p.seq_kv = int(seq_kv), p.heads = heads, p.head_dim = head_dim;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.o = reinterpret_cast<__nv_bfloat16*>(o), p.ldo = ldo, p.o_head_stride = o_head_stride;
  p.run_flag = run_flag, p.run_if = run_if;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (head_dim == 128) return attn::launch<128>(q, ldq, q_head_stride, k, ldk, k_head_stride, v, ldv, v_head_stride, p, s);
  return attn::launch<64>(q, ldq, q_head_stride, k, ldk, k_head_stride, v, ldv, v_head_stride, p, s);
}
