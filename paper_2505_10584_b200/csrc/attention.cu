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
//               O_t += P_t V_j  (P from TMEM — the TS form — V MN-major, N=D).
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: thread = query
//               row (TMEM lane), 224 registers each (setmaxnreg).  Online
//               softmax in the exp2 domain: scale folded into one packed
//               FFMA2 per pair, 3/8 of the exponentials evaluated by a
//               degree-3 polynomial on the FMA pipe (the rest on MUFU) so
//               neither pipe caps the tensor core; lazy rescaling (only when
//               the running max grows by > 8, so O in TMEM is rarely
//               touched); P written back to TMEM as packed bf16 pairs over
//               the consumed half of S_t (tcgen05.st), so the PV MMA reads A
//               from TMEM and only V from shared memory (smem operand traffic
//               per KV block drops from 160 KB to 96 KB per Q tile); final
//               1/l normalisation and TMA-staged bf16 store from the same warps.
// TMEM: S0 | S1 | O0 | O1  (128 + 128 + D + D columns).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <mutex>
#include <tuple>
#include <vector>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {
namespace attn {

constexpr int BQ = 128;   // rows per Q tile (MMA M)
constexpr int BKV = 128;  // keys per KV tile (MMA N of QK^T, K of PV)
constexpr int kThreads = 384;    // 3 warpgroups: control | softmax tile 0 | softmax tile 1
constexpr uint32_t kCtrlRegs = 56;     // setmaxnreg budgets: 56 + 2 * 224 <= 512 per SMSP
constexpr uint32_t kSoftmaxRegs = 224;
constexpr uint32_t kPolyMaskDefault = 0x52;  // pairs (i & 7) in {1,4,6}: exp2 by polynomial (3/8 off the MUFU)
constexpr uint32_t kPCol = 64;               // P_t (bf16 pairs) lives in columns 64..127 of S_t

template <int D>
struct Cfg {
  static constexpr int NS = D == 128 ? 5 : 6;                // K/V ring depth
  static constexpr int kQBytes = BQ * D * 2;                 // one Q tile
  static constexpr int kKVBytes = BKV * D * 2;               // one K or V tile
  static constexpr int kOffQ = 0;
  static constexpr int kOffKV = 2 * kQBytes;
  static constexpr int kOffBar = kOffKV + NS * kKVBytes;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr int kBoxes = D / 64;                      // 64-column TMA boxes per row
};

constexpr int kMaxPeers = 8;

// Where output row `row` of head `head` lands.  Local: o + head*ohs + row*ldo.
// Ulysses scatter (nranks > 0): video row `row` belongs to rank row / rpr and
// goes straight into that rank's O buffer (peer memory over NVLink) at row
// row % rpr; text rows (row >= text_row0) are replicated into every rank's
// buffer after its rpr video rows.  peer_o[r] already points at this rank's
// head-column slice of rank r's buffer.
struct OutMap {
  __nv_bfloat16* o;
  int64_t ldo, o_head_stride;
  __nv_bfloat16* peer_o[kMaxPeers];
  int nranks;
  int64_t rows_per_rank, text_row0;
};

// TMA store maps of the output (3-D: d, head, row; box 64 x 1 x 128).  Local:
// `local` over o[seq_q].  Scatter: vid[r] over rank r's rows_per_rank video
// rows, txt[r] over its text rows (so a tile straddling a rank boundary is
// clipped by each map, never spilling into the neighbour's rows).
struct OutMaps {
  CUtensorMap local;
  CUtensorMap vid[kMaxPeers];
  CUtensorMap txt[kMaxPeers];
};

struct Params {
  int seq_q, seq_kv, heads, head_dim;
  float scale_log2;
  OutMap out;
  // Work plan (1-D grid; tile = head * q_pairs + 256-query block): CTAs [0, n_whole)
  // run tiles 0..n_whole-1 over all KV blocks; every later tile is split over KV
  // into `splits` CTAs of kv_blocks_per_split blocks (the wave-quantisation tail,
  // or every tile when heads x Q blocks leave SMs idle).  Split partials go to
  // opart/lse in compact order ((tile - n_whole) * splits + split) * 256 + row.
  int q_pairs, n_whole;
  // split tiles: split 0 covers KV blocks [0, kv_first), split k >= 1 the kv_blocks_per_split
  // blocks after kv_first + (k - 1) * kv_blocks_per_split (uneven: a long first part and short
  // tails fill the SMs the long parts leave idle).  split_major: tail CTAs are launched split 0
  // of every tail tile first (else tile-major).
  int splits, kv_blocks_per_split, kv_first, split_major;
  // Short KV (2 * KV blocks <= ring depth, e.g. cross-attention to 256 text tokens):
  // a whole CTA runs `pairs_per_cta` consecutive 256-query blocks of one head with
  // K/V loaded once and resident, so the per-CTA fixed cost (prologue, K/V load,
  // pipeline fill) is paid once per pairs_per_cta blocks.  CTA c: head c / cpb,
  // blocks [(c % cpb) * pairs_per_cta, +pairs_per_cta), cpb = ceil(q_pairs / ppc).
  // 1 = one block per CTA (the tile plan above).
  int pairs_per_cta;
  float* opart;                     // [tail tiles][splits][256][part_d] f32 (O / l of the split)
  float* lse;                       // [tail tiles][splits][256] f32, log2-sum-exp2 of the split
  int part_d;                       // row stride of opart (the kernel's D)
  const int32_t* run_flag;
  int32_t run_if;
};

// Calls fn(ptr) for every destination of (head, row): one, or all ranks for
// replicated text rows under the Ulysses scatter.
template <typename F>
__device__ __forceinline__ void for_each_out(const OutMap& m, int head, int64_t row, F&& fn) {
  const int64_t hoff = static_cast<int64_t>(head) * m.o_head_stride;
  if (m.nranks == 0) {
    fn(m.o + hoff + row * m.ldo);
  } else if (row < m.text_row0) {
    const int r = int(row / m.rows_per_rank);
    fn(m.peer_o[r] + hoff + (row - r * m.rows_per_rank) * m.ldo);
  } else {
    const int64_t lr = m.rows_per_rank + (row - m.text_row0);
    for (int r = 0; r < m.nranks; ++r) fn(m.peer_o[r] + hoff + lr * m.ldo);
  }
}

template <int D, uint32_t kPolyMask = kPolyMaskDefault>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const __grid_constant__ OutMaps om, Params p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base + C::kOffQ;
  uint8_t* sKV = base + C::kOffKV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::kOffBar);
  uint64_t* q_full = bars;              // 2 (per Q tile)
  uint64_t* q_empty = bars + 2;         // 2 (last QK^T of a block done: Q buffer free)
  uint64_t* kv_full = bars + 4;         // NS
  uint64_t* kv_empty = kv_full + C::NS; // NS
  uint64_t* s_full = kv_empty + C::NS;  // 2
  uint64_t* p_full = s_full + 2;        // 2
  uint64_t* o_ready = p_full + 2;       // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_ready + 2);

  const uint32_t warp = warp_idx(), lane = lane_idx();
  const int cta = blockIdx.x;
  const bool whole = cta < p.n_whole;
  const int ppc = p.pairs_per_cta;
  const int cpb = (p.q_pairs + ppc - 1) / ppc;  // CTAs per head (multi-block mode)
  const int tail_tiles = p.q_pairs * p.heads - p.n_whole;
  const int ti = cta - p.n_whole;  // index among the split CTAs
  const int tile = whole ? (ppc > 1 ? (cta / cpb) * p.q_pairs + (cta % cpb) * ppc : cta)
                         : p.n_whole + (p.split_major ? ti % tail_tiles : ti / p.splits);
  const int split = whole ? 0 : (p.split_major ? ti / tail_tiles : ti % p.splits);
  const int head = tile / p.q_pairs;
  const int pair0 = tile % p.q_pairs;                        // first 256-query block
  const int npair = ppc > 1 ? min(ppc, p.q_pairs - pair0) : 1;
  const int nkv_all = (p.seq_kv + BKV - 1) / BKV;
  const int j0 = whole || split == 0 ? 0 : p.kv_first + (split - 1) * p.kv_blocks_per_split;  // first KV block
  const int nkv = whole ? nkv_all : min(nkv_all - j0, split == 0 ? p.kv_first : p.kv_blocks_per_split);
  const int nblk = npair * nkv;                              // flattened (block, KV block) steps

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    for (int t = 0; t < 2; ++t) {
      mbar_init(q_full + t, 1);
      mbar_init(q_empty + t, 1);
    }
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
  pdl_wait();  // the prologue above overlapped the previous kernel (PDL); inputs only after this
  pdl_trigger();
  const bool run = gate_open(p.run_flag, p.run_if);

  if (!run) {
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    setmaxnreg_dec<kCtrlRegs>();
    // warp-wide loop, one elected lane per TMA op (keeps operands in uniform registers)
    auto load_q = [&](int t, int kk) {
      if (elect_one()) mbar_arrive_expect_tx(q_full + t, C::kQBytes);
      for (int c = 0; c < C::kBoxes; ++c)
        if (elect_one())
          tma_load_3d(sQ + t * C::kQBytes + c * (BQ * 128), &tq, q_full + t, c * 64, head,
                      (pair0 + kk) * (2 * BQ) + t * BQ, kEvictFirst);
    };
    load_q(0, 0);
    load_q(1, 0);
    for (int i = 0; i < 2 * nkv; ++i) {
      const int s = i % C::NS;
      const uint32_t ph = (i / C::NS) & 1;
      mbar_wait(kv_empty + s, ph ^ 1);
      if (elect_one()) mbar_arrive_expect_tx(kv_full + s, C::kKVBytes);
      const CUtensorMap* m = (i & 1) ? &tv : &tk;
      const int row = (j0 + (i >> 1)) * BKV;
      for (int c = 0; c < C::kBoxes; ++c)
        if (elect_one())
          tma_load_3d(sKV + s * C::kKVBytes + c * (BKV * 128), m, kv_full + s, c * 64, head, row, kEvictLast);
    }
    // later blocks (K/V stay resident): tile t's next Q as soon as its last QK^T has read Q_t
    for (int kk = 1; kk < npair; ++kk)
      for (int t = 0; t < 2; ++t) {
        mbar_wait(q_empty + t, (kk - 1) & 1);
        load_q(t, kk);
      }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop (all values warp-uniform) and one elected lane
    // issues each tcgen05 op: issuing from a `lane == 0` branch made the compiler
    // wrap every MMA in a uniform-register waterfall loop (R2UR/ELECT/BRA.U.ANY), and
    // at one 128x128x16 MMA per ~68 cycles that issue cost throttled the tensor pipe.
    setmaxnreg_dec<kCtrlRegs>();
    {
      constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV, 0, 0);  // Q, K both K-major
      constexpr uint32_t kIdescO = idesc_bf16(BQ, D, 0, 1);    // P K-major, V MN-major
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t q_addr = __shfl_sync(0xffffffffu, smem_u32(sQ), 0);
      const uint32_t kv_addr = __shfl_sync(0xffffffffu, smem_u32(sKV), 0);
      auto issue_qk = [&](int t, int stage) {
        const uint32_t a0 = q_addr + t * C::kQBytes, b0 = kv_addr + stage * C::kKVBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (BQ * 128) + (kk & 3) * 32;
          const uint64_t da = smem_desc(a0 + off, 0, 1024), db = smem_desc(b0 + off, 0, 1024);
          if (elect_one()) umma_bf16_ss(tm + t * 128, da, db, kIdescS, kk > 0);
        }
      };
      auto issue_pv = [&](int t, int stage, bool acc) {
        // A = P_t straight from TMEM (columns 64..127 of S_t, bf16 pairs), B = V (MN-major smem)
        const uint32_t a0 = tm + t * 128 + kPCol, b0 = kv_addr + stage * C::kKVBytes;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint64_t db = smem_desc(b0 + kk * 16 * 128, BKV * 128, 1024);  // 16 keys x 128 B rows
          if (elect_one()) umma_bf16_ts(tm + 256 + t * D, a0 + kk * 8, db, kIdescO, (acc || kk > 0) ? 1u : 0u);
        }
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) umma_commit(bar);
      };
      // Flattened over (256-query block kk, KV block j): step J = kk * nkv + j issues
      // PV of step J-1 and QK^T of step J for both tiles.  At a block boundary both
      // PVs go first (tile 1's epilogue must not wait behind tile 0's Q reload).
      for (int J = 0; J <= nblk; ++J) {
        const int j = J % nkv, kk = J / nkv, jp = (J + nkv - 1) % nkv;
        const int ik = 2 * j, iv = 2 * jp + 1;  // ring indices of K_j and V_{jp} (resident when npair > 1)
        const bool qk = J < nblk, pv = J > 0, first = qk && j == 0;
        if (qk) {
          mbar_wait(kv_full + ik % C::NS, (ik / C::NS) & 1);
          tc_fence_after();
        }
        auto do_pv = [&](int t) {
          mbar_wait(p_full + t, (J - 1) & 1);
          tc_fence_after();
          issue_pv(t, iv % C::NS, jp > 0);
          commit(o_ready + t);
        };
        auto do_qk = [&](int t) {
          if (first) {
            mbar_wait(q_full + t, kk & 1);
            tc_fence_after();
          }
          issue_qk(t, ik % C::NS);
          commit(s_full + t);
          if (j == nkv - 1 && kk + 1 < npair) commit(q_empty + t);  // Q_t read: the next block's Q may land
        };
        if (pv) {
          mbar_wait(kv_full + iv % C::NS, (iv / C::NS) & 1);
          tc_fence_after();
          do_pv(0);
          if (first) {
            do_pv(1);
            commit(kv_empty + iv % C::NS);
          }
        }
        if (qk) do_qk(0);
        if (pv && !first) {
          do_pv(1);
          commit(kv_empty + iv % C::NS);
        }
        if (qk) {
          do_qk(1);
          commit(kv_empty + ik % C::NS);
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
    const uint32_t sw = r & 7;
    const float c = p.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    const uint64_t kM = f2pack(12582912.f, 12582912.f);  // 1.5 * 2^23: round-to-nearest
    const uint64_t kC0 = f2pack(0.99992806f, 0.99992806f), kC1 = f2pack(0.69326103f, 0.69326103f);
    const uint64_t kC2 = f2pack(0.24261117f, 0.24261117f), kC3 = f2pack(0.05517162f, 0.05517162f);
    for (int kk = 0; kk < npair; ++kk) {
      const int q0 = (pair0 + kk) * (2 * BQ);
      float m_run = -INFINITY, l_run = 0.f;     // m_run in raw score units

      for (int j = 0; j < nkv; ++j) {
        const int J = kk * nkv + j;
        mbar_wait(s_full + t, J & 1);
        tc_fence_after();
        uint32_t sr[BKV];
        tmem_ld64(s_tmem, sr);
        tmem_ld64(s_tmem + 64, sr + 64);
        tmem_wait_ld();
        const int kv_valid = p.seq_kv - (j0 + j) * BKV;
        if (kv_valid < BKV) {
#pragma unroll
          for (int i = 0; i < BKV; ++i)
            if (i >= kv_valid) sr[i] = 0xff800000u;  // -inf
        }
        // row max as 8 independent FMNMX3 chains + a 3-level tree (a single 64-long
        // dependent chain was the softmax's critical path)
        float mm[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mm[k] = fmaxf(__uint_as_float(sr[k]), __uint_as_float(sr[k + 8]));
#pragma unroll
        for (int i = 16; i < BKV; i += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mm[k] = fmaxf(mm[k], fmaxf(__uint_as_float(sr[i + k]), __uint_as_float(sr[i + 8 + k])));
        const float mx = fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])),
                               fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7])));
        // PV_{j-1} must be done before O is rescaled or P_t overwritten.
        if (j > 0) {
          mbar_wait(o_ready + t, (J - 1) & 1);
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
        uint64_t acc2[4];  // 4 independent packed row-sum chains
#pragma unroll
        for (int q = 0; q < 4; ++q) acc2[q] = f2pack(0.f, 0.f);
        uint32_t pp[16];  // 16 packed bf16 pairs = 16 TMEM columns, stored as they fill
#pragma unroll
        for (int kc = 0; kc < BKV / 8; ++kc) {
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
              uint64_t pq = ffma2(fr, kC3, kC2);
              pq = ffma2(pq, fr, kC1);
              pq = ffma2(pq, fr, kC0);
              float q0, q1, t0, t1;
              f2unpack(pq, q0, q1);
              f2unpack(tt, t0, t1);
              p0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
              p1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            acc2[q] = fadd2(acc2[q], f2pack(p0, p1));
            pp[(kc & 3) * 4 + q] = pack_bf16(p0, p1);
          }
          if ((kc & 3) == 3) tmem_st16(s_tmem + kPCol + (kc >> 2) * 16, pp);
        }
        float a0, a1;
        f2unpack(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])), a0, a1);
        l_run += a0 + a1;
        tmem_wait_st();  // P in TMEM before the MMA warp may read it
        tc_fence_before();
        mbar_arrive(p_full + t);
      }
      // epilogue: O / l -> bf16 (or the split's f32 partial + log2-sum-exp2)
      mbar_wait(o_ready + t, (kk * nkv + nkv - 1) & 1);
      tc_fence_after();
      const int row = q0 + t * BQ + r;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
      const bool live = row < p.seq_q;
      if (!whole) {
        const int64_t prow = (static_cast<int64_t>(tile - p.n_whole) * p.splits + split) * (2 * BQ) + t * BQ + r;
        if (live) p.lse[prow] = m_run * c + __log2f(l_run);
        float* orow = p.opart + prow * D;
#pragma unroll 1
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t u[32];
          tmem_ld32(o_tmem + cc * 32, u);
          tmem_wait_ld();
          if (live) {
#pragma unroll
            for (int g = 0; g < 8; ++g)
              *reinterpret_cast<float4*>(orow + cc * 32 + 4 * g) =
                  make_float4(__uint_as_float(u[4 * g]) * inv, __uint_as_float(u[4 * g + 1]) * inv,
                              __uint_as_float(u[4 * g + 2]) * inv, __uint_as_float(u[4 * g + 3]) * inv);
          }
        }
      } else {
        // O/l -> bf16 into this tile's Q buffer (idle once its last QK^T is done; same
        // 128B-swizzled [64-col box][128 rows][128 B] layout), then TMA stores: coalesced,
        // and under the Ulysses scatter straight into the owning ranks' buffers.
        uint8_t* stile = sQ + t * C::kQBytes;
        const uint32_t srow = smem_u32(stile) + r * 128;
        const OutMap& m = p.out;
        const int tr0 = q0 + t * BQ;  // first row of this tile
        // TMA coordinates must be >= 0: a tile that starts in one rank's rows and ends in
        // the next (or in the text rows) is written with direct stores instead.
        const int64_t last = min(int64_t(tr0 + BQ - 1), int64_t(p.seq_q - 1));
        // Several blocks per CTA: direct stores, so the Q buffer is not needed for staging and
        // the next block's Q loads while this one's softmax / PV / epilogue run.
        const bool use_tma = npair == 1 && tr0 < p.seq_q &&  // a tile wholly past the end stores nothing
                             (m.nranks == 0 || tr0 >= m.text_row0 ||
                              (last < m.text_row0 && tr0 / m.rows_per_rank == last / m.rows_per_rank));
#pragma unroll 1
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t u[32];
          tmem_ld32(o_tmem + cc * 32, u);
          tmem_wait_ld();
          uint4 pk[4];
#pragma unroll
          for (int g = 0; g < 4; ++g)
            pk[g] = make_uint4(pack_bf16(__uint_as_float(u[8 * g]) * inv, __uint_as_float(u[8 * g + 1]) * inv),
                               pack_bf16(__uint_as_float(u[8 * g + 2]) * inv, __uint_as_float(u[8 * g + 3]) * inv),
                               pack_bf16(__uint_as_float(u[8 * g + 4]) * inv, __uint_as_float(u[8 * g + 5]) * inv),
                               pack_bf16(__uint_as_float(u[8 * g + 6]) * inv, __uint_as_float(u[8 * g + 7]) * inv));
          if (use_tma) {
            const uint32_t bx = srow + (cc >> 1) * (BQ * 128);
#pragma unroll
            for (int g = 0; g < 4; ++g)
              st_shared_v4(bx + ((((cc & 1) * 4 + g) ^ sw) << 4), pk[g].x, pk[g].y, pk[g].z, pk[g].w);
          } else if (live && cc * 32 < p.head_dim) {
            for_each_out(m, head, row, [&](__nv_bfloat16* orow) {
#pragma unroll
              for (int g = 0; g < 4; ++g) *reinterpret_cast<uint4*>(orow + cc * 32 + 8 * g) = pk[g];
            });
          }
        }
        if (use_tma) {
          fence_proxy_async_smem();
          named_bar_sync(1 + t, 128);
          if (quad == 0 && lane == 0) {
            for (int c = 0; c < C::kBoxes; ++c) {
              const uint8_t* src = stile + c * (BQ * 128);
              if (m.nranks == 0)
                tma_store_3d(&om.local, src, c * 64, head, tr0);
              else if (tr0 >= m.text_row0)
                for (int rr = 0; rr < m.nranks; ++rr)
                  tma_store_3d(&om.txt[rr], src, c * 64, head, int(tr0 - m.text_row0));
              else
                tma_store_3d(&om.vid[tr0 / m.rows_per_rank], src, c * 64, head, int(tr0 % m.rows_per_rank));
            }
            bulk_commit();
            bulk_wait<0>();  // complete (not just read out of smem) before the CTA exits
          }
        }
      }
    }  // block kk
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

// ----------------------------------------------------------------------------
// Short-KV attention (seq_kv <= 256, head_dim 128): the Single-DiT cross-attention to
// the 256 text tokens.  The general kernel walks KV in 128-key blocks
// with an online softmax, so each Q tile's QK^T -> softmax -> PV chain is serial per
// block and only 2 blocks long — the tensor pipe idled at 33%.  Here a Q tile's whole
// score row fits TMEM: S_t = Q_t K^T is one 128 x 256 fp32 tile (two N=128 MMAs), the
// softmax is exact (max over all 256 keys, no rescale), P_t is packed as bf16 pairs over
// the first 128 columns of S_t, and O_t = P_t V accumulates in the last 128 columns
// (K = 256 from TMEM, the TS form).  A CTA owns consecutive 128-query tiles of one head
// with K and V resident (128 KB), two TMEM slots of 256 columns ping-pong between two
// softmax warpgroups; the epilogue frees its slot as soon as O is in registers.
//   warp 0: TMA (K, V once; Q tiles through 2 buffers)   warp 1: MMA issuer
//   warps 4-7 / 8-11: softmax + epilogue of even / odd tiles (thread = query row)
struct ShortCfg {
  static constexpr int D = 128;
  static constexpr int kQBytes = BQ * D * 2;          // 32 KB per Q tile
  static constexpr int kKVBlock = BKV * D * 2;        // 32 KB per 128 keys
  static constexpr int kOffK = 0;                     // [2 key blocks][2 d-chunks][128][128 B]
  static constexpr int kOffV = 2 * kKVBlock;
  static constexpr int kOffQ = 4 * kKVBlock;          // [2 buffers][2 d-chunks][128][128 B]
  static constexpr int kStage = 32 * 128;             // per softmax warp: 32 rows x 64 bf16 (128B swizzle)
  static constexpr int kOffO = kOffQ + 2 * kQBytes;   // [8 warps][kStage]
  static constexpr int kOffBar = kOffO + 8 * kStage;
  static constexpr int kSmem = kOffBar + 256 + 1024;
};

struct ShortParams {
  int seq_q, seq_kv, heads;
  int q_tiles, tiles_per_cta, ctas_per_head;
  float scale_log2;
  __nv_bfloat16* o;
  int64_t ldo, o_head_stride;
  const int32_t* run_flag;
  int32_t run_if;
  // profiling hook (aqb_attention_trace): per CTA 64 clock64 stamps of the pipeline events of
  // its first 8 tiles (MMA QK / PV issue, softmax s_full / p_full / o_ready / slot release)
  unsigned long long* trace;
};

__device__ __forceinline__ void short_stamp(const ShortParams& p, int slot) {
  if (p.trace != nullptr && slot < 64) p.trace[int64_t(blockIdx.x) * 64 + slot] = clock64();
}

// exp2((s - m)·c) of 32 scores (16 pairs), row-sum into acc2, packed bf16 pairs into pp[16]
template <uint32_t kPolyMask>
__device__ __forceinline__ void exp_pack32(const uint32_t* sr, uint64_t c2, uint64_t nm2, uint64_t (&acc2)[4],
                                           uint32_t (&pp)[16]) {
  const uint64_t kM = f2pack(12582912.f, 12582912.f);
  const uint64_t kC0 = f2pack(0.99992806f, 0.99992806f), kC1 = f2pack(0.69326103f, 0.69326103f);
  const uint64_t kC2 = f2pack(0.24261117f, 0.24261117f), kC3 = f2pack(0.05517162f, 0.05517162f);
#pragma unroll
  for (int pi = 0; pi < 16; ++pi) {
    const uint64_t x2 = ffma2(f2pack(__uint_as_float(sr[2 * pi]), __uint_as_float(sr[2 * pi + 1])), c2, nm2);
    float x0, x1, p0, p1;
    f2unpack(x2, x0, x1);
    if ((kPolyMask >> (pi & 7)) & 1) {
      const uint64_t xc = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
      const uint64_t tt = fadd2(xc, kM);
      const uint64_t fr = fsub2(xc, fsub2(tt, kM));
      uint64_t pq = ffma2(fr, kC3, kC2);
      pq = ffma2(pq, fr, kC1);
      pq = ffma2(pq, fr, kC0);
      float q0, q1, t0, t1;
      f2unpack(pq, q0, q1);
      f2unpack(tt, t0, t1);
      p0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
      p1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
    } else {
      p0 = ex2(x0);
      p1 = ex2(x1);
    }
    acc2[pi & 3] = fadd2(acc2[pi & 3], f2pack(p0, p1));
    pp[pi] = pack_bf16(p0, p1);
  }
}

template <uint32_t kPolyMask = kPolyMaskDefault>
__global__ void __launch_bounds__(kThreads, 1)
    attn_short_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
                      ShortParams p) {
  using C = ShortCfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = base + C::kOffK;
  uint8_t* sV = base + C::kOffV;
  uint8_t* sQ = base + C::kOffQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + C::kOffBar);
  uint64_t* k_full = bars;          // 1
  uint64_t* v_full = bars + 1;      // 1
  uint64_t* q_full = bars + 2;      // 2 (Q buffers)
  uint64_t* q_empty = bars + 4;     // 2
  uint64_t* s_full = bars + 6;      // 2 (TMEM slots)
  uint64_t* p_full = bars + 8;      // 2
  uint64_t* o_ready = bars + 10;    // 2
  uint64_t* slot_free = bars + 12;  // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const uint32_t warp = warp_idx(), lane = lane_idx();
  const int head = blockIdx.x / p.ctas_per_head;
  const int tile0 = (blockIdx.x % p.ctas_per_head) * p.tiles_per_cta;
  const int ntile = min(p.tiles_per_cta, p.q_tiles - tile0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    tma_prefetch_desc(&to);
    mbar_init(k_full, 1);
    mbar_init(v_full, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(q_full + b, 1);
      mbar_init(q_empty + b, 1);
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 128);
      mbar_init(o_ready + b, 1);
      mbar_init(slot_free + b, 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();
  const bool run = gate_open(p.run_flag, p.run_if) && ntile > 0;

  if (!run) {
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer
    setmaxnreg_dec<kCtrlRegs>();
    if (elect_one()) mbar_arrive_expect_tx(k_full, 2 * C::kKVBlock);
    for (int kb = 0; kb < 2; ++kb)
      for (int c = 0; c < 2; ++c)
        if (elect_one())
          tma_load_3d(sK + kb * C::kKVBlock + c * (BKV * 128), &tk, k_full, c * 64, head, kb * BKV, kEvictLast);
    auto load_q = [&](int i) {
      const int b = i & 1;
      if (elect_one()) mbar_arrive_expect_tx(q_full + b, C::kQBytes);
      for (int c = 0; c < 2; ++c)
        if (elect_one())
          tma_load_3d(sQ + b * C::kQBytes + c * (BQ * 128), &tq, q_full + b, c * 64, head, (tile0 + i) * BQ,
                      kEvictFirst);
    };
    load_q(0);
    if (elect_one()) mbar_arrive_expect_tx(v_full, 2 * C::kKVBlock);
    for (int kb = 0; kb < 2; ++kb)
      for (int c = 0; c < 2; ++c)
        if (elect_one())
          tma_load_3d(sV + kb * C::kKVBlock + c * (BKV * 128), &tv, v_full, c * 64, head, kb * BKV, kEvictLast);
    if (ntile > 1) load_q(1);
    for (int i = 2; i < ntile; ++i) {
      mbar_wait(q_empty + (i & 1), ((i >> 1) - 1) & 1);  // QK^T of tile i-2 has read its buffer
      load_q(i);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (warp-wide, elected lane)
    setmaxnreg_dec<kCtrlRegs>();
    constexpr uint32_t kIdescS = idesc_bf16(BQ, BKV, 0, 0);  // Q, K both K-major
    constexpr uint32_t kIdescO = idesc_bf16(BQ, D, 0, 1);    // P (TMEM) K-major, V MN-major
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t q_addr = __shfl_sync(0xffffffffu, smem_u32(sQ), 0);
    const uint32_t k_addr = __shfl_sync(0xffffffffu, smem_u32(sK), 0);
    const uint32_t v_addr = __shfl_sync(0xffffffffu, smem_u32(sV), 0);
    // keys past seq_kv (short text, e.g. 77 tokens): no QK^T for an all-padding 128-key block,
    // no PV steps past the last 16 keys that hold a valid one (their P is masked to 0)
    const int nkb = p.seq_kv > BKV ? 2 : 1;
    const int nkk = (p.seq_kv + 15) / 16;
    auto qk = [&](int i) {
      const int b = i & 1, sl = i & 1;
      if (i >= 2) {  // slot reused: the epilogue of tile i-2 has read O out of it
        mbar_wait(slot_free + sl, ((i >> 1) - 1) & 1);
        tc_fence_after();
      }
      mbar_wait(q_full + b, (i >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && i < 8) short_stamp(p, i);
      const uint32_t a0 = q_addr + b * C::kQBytes;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        if (kb >= nkb) break;
        const uint32_t b0 = k_addr + kb * C::kKVBlock;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (BQ * 128) + (kk & 3) * 32;
          const uint64_t da = smem_desc(a0 + off, 0, 1024), db = smem_desc(b0 + off, 0, 1024);
          if (elect_one()) umma_bf16_ss(tm + sl * 256 + kb * 128, da, db, kIdescS, kk > 0);
        }
      }
      if (elect_one()) umma_commit(s_full + sl);
      if (elect_one()) umma_commit(q_empty + b);
    };
    auto pv = [&](int i) {
      const int sl = i & 1;
      mbar_wait(p_full + sl, (i >> 1) & 1);
      tc_fence_after();
      if (lane == 0 && i < 8) short_stamp(p, 8 + i);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {  // 16 keys per MMA (8 packed TMEM columns of P)
        if (kk >= nkk) break;
        const uint64_t db = smem_desc(v_addr + (kk >> 3) * C::kKVBlock + (kk & 7) * 16 * 128, BKV * 128, 1024);
        if (elect_one()) umma_bf16_ts(tm + sl * 256 + 128, tm + sl * 256 + kk * 8, db, kIdescO, kk > 0);
      }
      if (elect_one()) umma_commit(o_ready + sl);
    };
    if (lane == 0) short_stamp(p, 48);
    mbar_wait(k_full, 0);
    tc_fence_after();
    if (lane == 0) short_stamp(p, 49);
    qk(0);
    if (ntile > 1) qk(1);
    mbar_wait(v_full, 0);
    tc_fence_after();
    for (int i = 0; i < ntile; ++i) {
      pv(i);
      if (i + 2 < ntile) qk(i + 2);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    setmaxnreg_inc<kSoftmaxRegs>();
    const int wg = (warp - 4) / 4;  // tiles i with i % 2 == wg
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32) << 16;
    const uint32_t s_tmem = tmem + lane_base + wg * 256;
    const float c = p.scale_log2;
    const uint64_t c2 = f2pack(c, c);
    const int nh = min(4, (p.seq_kv + 63) / 64);  // 64-key chunks holding a valid key (the PV reads no more)
    for (int i = wg; i < ntile; i += 2) {
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait(s_full + wg, ph);
      tc_fence_after();
      const bool stamp = (warp & 3) == 0 && lane == 0 && i < 8;
      if (stamp) short_stamp(p, 16 + i);
      uint32_t sr[64];
      // pass 1: row max over the valid keys, 64 columns at a time
      float mx = -INFINITY;
#pragma unroll 1
      for (int h = 0; h < nh; ++h) {
        tmem_ld64(s_tmem + h * 64, sr);
        tmem_wait_ld();
        const int valid = p.seq_kv - h * 64;
        if (valid < 64) {  // partial chunk (short text): keys past seq_kv do not count
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= valid) sr[j] = 0xff800000u;
        }
        // 8 independent 3-input max chains (FMNMX3), then a tree
        float mm[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mm[k] = fmaxf(__uint_as_float(sr[k]), __uint_as_float(sr[k + 8]));
#pragma unroll
        for (int j = 16; j < 64; j += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mm[k] = fmaxf(mm[k], fmaxf(__uint_as_float(sr[j + k]), __uint_as_float(sr[j + 8 + k])));
        mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])),
                             fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7]))));
      }
      // pass 2: p = exp2((s - max)·c), packed bf16 pairs: keys [64h, 64h+64) -> P columns
      // [32h, 32h+32) of the slot, i.e. over scores this thread has already read
      const uint64_t nm2 = f2pack(-mx * c, -mx * c);
      uint64_t acc2[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc2[q] = f2pack(0.f, 0.f);
#pragma unroll 1
      for (int h = 0; h < nh; ++h) {
        tmem_ld64(s_tmem + h * 64, sr);
        tmem_wait_ld();
        const int valid = p.seq_kv - h * 64;
        if (valid < 64) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= valid) sr[j] = 0xff800000u;  // -inf -> p = 0
        }
#pragma unroll
        for (int q32 = 0; q32 < 2; ++q32) {
          uint32_t pp[16];
          exp_pack32<kPolyMask>(sr + 32 * q32, c2, nm2, acc2, pp);
          tmem_st16(s_tmem + h * 32 + q32 * 16, pp);
        }
      }
      float a0, a1;
      f2unpack(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])), a0, a1);
      const float l = a0 + a1;
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + wg);
      if (stamp) short_stamp(p, 24 + i);
      // epilogue: O (columns [128, 256) of the slot) -> bf16 rows; the slot is free once read
      mbar_wait(o_ready + wg, ph);
      tc_fence_after();
      if (stamp) short_stamp(p, 32 + i);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      uint32_t u[D];  // all of O in registers first: the slot is released before the stores
      tmem_ld64(s_tmem + 128, u);
      tmem_ld64(s_tmem + 192, u + 64);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(slot_free + wg);
      if (stamp) short_stamp(p, 40 + i);
      // bf16 rows -> this warp's 128B-swizzled staging buffer (32 rows x 64 columns), one TMA
      // store per half: coalesced, and the warp does not wait for the write to land
      const uint32_t sbuf = smem_u32(base + C::kOffO + (warp - 4) * C::kStage) + lane * 128;
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        if (lane == 0) bulk_wait_read<0>();  // the previous store has read the buffer
        __syncwarp();
#pragma unroll
        for (int g8 = 0; g8 < 8; ++g8) {
          const uint32_t* w = u + hf * 64 + 8 * g8;
          st_shared_v4(sbuf + ((g8 ^ (lane & 7)) << 4),
                       pack_bf16(__uint_as_float(w[0]) * inv, __uint_as_float(w[1]) * inv),
                       pack_bf16(__uint_as_float(w[2]) * inv, __uint_as_float(w[3]) * inv),
                       pack_bf16(__uint_as_float(w[4]) * inv, __uint_as_float(w[5]) * inv),
                       pack_bf16(__uint_as_float(w[6]) * inv, __uint_as_float(w[7]) * inv));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&to, base + C::kOffO + (warp - 4) * C::kStage, hf * 64, head,
                       (tile0 + i) * BQ + int(quad) * 32);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait<0>();  // stores complete before the CTA exits
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

// Split-KV combine: one warp per row of a split tile; lane owns 4 of the D columns.
//   O = sum_s 2^(lse_s - M) O_s / sum_s 2^(lse_s - M),  M = max_s lse_s
__global__ void __launch_bounds__(256) attn_combine_kernel(Params p) {
  pdl_wait();
  pdl_trigger();
  if (!gate_open(p.run_flag, p.run_if)) return;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t tail = static_cast<int64_t>(p.q_pairs) * p.heads - p.n_whole;
  if (w >= tail * (2 * BQ)) return;
  const int64_t tl = w / (2 * BQ);
  const int r = int(w % (2 * BQ));
  const int tile = p.n_whole + int(tl);
  const int head = tile / p.q_pairs;
  const int64_t row = int64_t(tile % p.q_pairs) * (2 * BQ) + r;
  if (row >= p.seq_q) return;
  const int64_t base = tl * p.splits * (2 * BQ) + r;  // split s at base + s * 256
  float mx = -INFINITY;
  for (int s = 0; s < p.splits; ++s) mx = fmaxf(mx, p.lse[base + s * (2 * BQ)]);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float den = 0.f;
  const int D = p.head_dim, PD = p.part_d;
  for (int s = 0; s < p.splits; ++s) {
    const int64_t pr = base + s * (2 * BQ);
    const float wt = exp2f(p.lse[pr] - mx);
    den += wt;
    if (lane * 4 < D) {
      const float4 v = *reinterpret_cast<const float4*>(p.opart + pr * PD + lane * 4);
      acc.x += wt * v.x, acc.y += wt * v.y, acc.z += wt * v.z, acc.w += wt * v.w;
    }
  }
  if (lane * 4 >= D) return;
  const float inv = 1.f / den;
  const uint2 pk = make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
  for_each_out(p.out, head, row, [&](__nv_bfloat16* orow) { *reinterpret_cast<uint2*>(orow + lane * 4) = pk; });
}

// Work plan for one launch (see Params): which tiles run whole and how the rest split
// over KV.  Candidates — no split; the last `tail` tiles (every tile, or the tails left by
// 0..3 whole waves) split s ways, uniformly or with a longer first part (the short parts fill
// the SMs the long ones leave idle), launched tile- or split-major — are list-scheduled onto
// one CTA slot per SM in launch order (the order the hardware hands out CTAs), each CTA costing
// its KV blocks + 2 (Q load, epilogue); the combine pass costs its partial traffic in KV-block
// units (~2.3 us per 256-query KV block on one SM).  Lowest makespan wins, a split plan only
// if it saves > 5%.
struct Plan {
  int n_whole, splits, first, per, split_major;
};

static int split_blocks(const Plan& pl, int nkv, int k) {
  const int j0 = k == 0 ? 0 : pl.first + (k - 1) * pl.per;
  return std::max(0, std::min(nkv - j0, k == 0 ? pl.first : pl.per));
}

static double simulate(int64_t tiles, const Plan& pl, int nkv, int slots) {
  std::priority_queue<double, std::vector<double>, std::greater<double>> fin;
  for (int i = 0; i < slots; ++i) fin.push(0.0);
  auto put = [&](double len) {
    const double t = fin.top();
    fin.pop();
    fin.push(t + len);
  };
  const int64_t n_whole = pl.n_whole;
  if (n_whole > 4 * slots) {  // long uniform prefix: whole waves, then the remainder
    const double base = double((n_whole - 2 * slots) / slots) * (nkv + 2.0);
    std::priority_queue<double, std::vector<double>, std::greater<double>> f2;
    for (int i = 0; i < slots; ++i) f2.push(base);
    fin.swap(f2);
    for (int64_t i = 0; i < (n_whole - 2 * slots) % slots + 2 * slots; ++i) put(nkv + 2.0);
  } else {
    for (int64_t i = 0; i < n_whole; ++i) put(nkv + 2.0);
  }
  const int64_t tail = tiles - n_whole;
  if (pl.split_major) {
    for (int k = 0; k < pl.splits; ++k)
      for (int64_t t = 0; t < tail; ++t) put(split_blocks(pl, nkv, k) + 2.0);
  } else {
    for (int64_t t = 0; t < tail; ++t)
      for (int k = 0; k < pl.splits; ++k) put(split_blocks(pl, nkv, k) + 3.0);
  }
  double mx = 0.0;
  while (!fin.empty()) mx = std::max(mx, fin.top()), fin.pop();
  return mx;
}

static Plan choose_plan_uncached(int64_t seq_q, int64_t seq_kv, int heads, int head_dim) {
  const int nkv = int((seq_kv + BKV - 1) / BKV);
  const int64_t tiles = ((seq_q + 2 * BQ - 1) / (2 * BQ)) * heads;
  const int slots = sm_count();
  Plan best{int(tiles), 1, nkv, nkv, 0};
  const double t1 = simulate(tiles, best, nkv, slots);
  double bt = t1;
  auto consider = [&](int64_t tail, int s, int first) {
    if (s < 2 || tail <= 0 || tail > tiles || tail * s > 64 * int64_t(slots) || first < 1 || first >= nkv) return;
    const int per = (nkv - first + s - 2) / (s - 1);
    if (per < 1) return;
    const int s_eff = 1 + (nkv - first + per - 1) / per;  // no empty split
    for (int major = 0; major < 2; ++major) {
      const Plan pl{int(tiles - tail), s_eff, first, per, major};
      double t = simulate(tiles, pl, nkv, slots);
      t += double(s_eff) * tail * (2 * BQ) * (head_dim * 4 + 4) * 2.0 / 5e12 / 2.3e-6 + 1.0;  // combine pass
      if (t < bt - 1e-9 && t < t1 * 0.95) bt = t, best = pl;
    }
  };
  const int64_t rem = tiles % slots;
  for (int s = 2; s <= 16 && s <= nkv; ++s) {
    const int uniform = (nkv + s - 1) / s;
    // first part from the uniform share up to all but s-1 blocks, in <= 16 steps
    const int span = nkv - (s - 1) - uniform;
    const int step = std::max(1, span / 16);
    for (int first = uniform; first <= nkv - (s - 1); first += step) {
      consider(tiles, s, first);
      for (int k = 0; k < 4; ++k) consider(rem + int64_t(k) * slots, s, first);
    }
  }
  return best;
}

Plan choose_plan(int64_t seq_q, int64_t seq_kv, int heads, int head_dim) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int, int>, Plan> cache;
  const auto key = std::make_tuple(seq_q, seq_kv, heads, head_dim);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const Plan pl = choose_plan_uncached(seq_q, seq_kv, heads, head_dim);
  if (cache.size() < 4096) cache.emplace(key, pl);
  return pl;
}

// Blocks per CTA for a short-KV launch with no split (see Params::pairs_per_cta): g
// consecutive 256-query blocks of one head per CTA, K/V loaded once.  Cost in the
// simulate() units: a block costs its KV blocks + 1 (Q load / epilogue bubble), a CTA
// one more (prologue, K/V load); waves of CTAs over one slot per SM.  AQB_ATTN_PAIRS
// forces g (1 = one block per CTA).
static int choose_pairs_per_cta(int q_pairs, int heads, int nkv, int ring) {
  if (2 * nkv > ring) return 1;  // K/V must stay resident in the ring
  if (const char* e = getenv("AQB_ATTN_PAIRS")) return std::min(std::max(1, atoi(e)), q_pairs);
  const int slots = sm_count();
  int best = 1;
  double bt = 1e30;
  for (int g = 1; g <= 16 && g <= q_pairs; ++g) {
    const int64_t ctas = int64_t(heads) * ((q_pairs + g - 1) / g);
    const double t = double((ctas + slots - 1) / slots) * (g * (nkv + 1.0) + 1.0);
    if (t < bt - 1e-9) bt = t, best = g;
  }
  return best;
}

static int64_t split_ws_bytes(int64_t tail_tiles, int splits, int head_dim) {
  if (splits <= 1 || tail_tiles <= 0) return 0;
  const int64_t rows = tail_tiles * splits * (2 * BQ);
  const int64_t d = head_dim <= 64 ? 64 : 128;
  return ((rows + 63) / 64 * 64 + rows * d) * 4;
}

// Output TMA maps for p.out (see OutMaps).
static int make_out_maps(const Params& p, OutMaps& om) {
  memset(&om, 0, sizeof(om));
  const OutMap& m = p.out;
  const uint64_t str[2] = {uint64_t(m.o_head_stride) * 2, uint64_t(m.ldo) * 2};
  const uint32_t box[3] = {64, 1, 128};
  if (m.nranks == 0) {
    const uint64_t dims[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(p.seq_q)};
    return make_tmap_bf16(&om.local, m.o, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const int64_t text_rows = p.seq_q - m.text_row0;
  for (int r = 0; r < m.nranks; ++r) {
    const uint64_t dv[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(m.rows_per_rank)};
    int rc = make_tmap_bf16(&om.vid[r], m.peer_o[r], 3, dv, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    if (text_rows > 0) {
      const uint64_t dt[3] = {uint64_t(p.head_dim), uint64_t(p.heads), uint64_t(text_rows)};
      rc = make_tmap_bf16(&om.txt[r], m.peer_o[r] + m.rows_per_rank * m.ldo, 3, dt, str, box,
                          CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
    }
  }
  return AQB_OK;
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
  // AQB_ATTN_POLY (tuning): which of every 8 exp2 pairs run on the FMA pipe instead of MUFU
  static int poly = -1;
  if (poly < 0) {
    const char* e = getenv("AQB_ATTN_POLY");
    poly = (e && !strcmp(e, "0")) ? 0 : (e && !strcmp(e, "2")) ? 2 : (e && !strcmp(e, "4")) ? 4 : 3;
  }
  auto kern = poly == 0 ? attn_fwd_kernel<D, 0x00> : poly == 2 ? attn_fwd_kernel<D, 0x22>
                       : poly == 4 ? attn_fwd_kernel<D, 0x55> : attn_fwd_kernel<D, kPolyMaskDefault>;
  static FuncAttrOnce attr[4];  // one per exp2-split variant; per device inside
  AQB_CUDA_TRY(set_smem_once(attr[poly == 0 ? 0 : poly == 2 ? 1 : poly == 4 ? 2 : 3], kern, smem));
  OutMaps om;
  if (p.n_whole > 0) {
    int rc = make_out_maps(p, om);
    if (rc) return rc;
  } else {
    memset(&om, 0, sizeof(om));
  }
  const int64_t tiles = static_cast<int64_t>(p.q_pairs) * p.heads;
  const int64_t ctas = p.pairs_per_cta > 1
                           ? int64_t(p.heads) * ((p.q_pairs + p.pairs_per_cta - 1) / p.pairs_per_cta)
                           : p.n_whole + (tiles - p.n_whole) * p.splits;
  AQB_CUDA_TRY(launch_pdl(kern, dim3(unsigned(ctas)), dim3(kThreads), smem, stream, tq, tk, tv, om, p));
  AQB_LAUNCH_CHECK();
  if (p.n_whole < tiles) {
    const int64_t warps = (tiles - p.n_whole) * (2 * BQ);
    AQB_CUDA_TRY(launch_pdl(attn_combine_kernel, dim3(unsigned((warps * 32 + 255) / 256)), dim3(256), 0, stream, p));
    AQB_LAUNCH_CHECK();
  }
  return AQB_OK;
}

// aqb_attention_trace: device buffer the short-KV kernel stamps its pipeline events into
static std::atomic<unsigned long long*> g_short_trace{nullptr};

// Tiles per CTA of a short-KV launch: one wave of CTAs over the SMs when possible (each CTA
// pays the K/V load once), otherwise the fewest waves.
static void short_plan(int q_tiles, int heads, int& tpc, int& cpb) {
  const int slots = sm_count();
  tpc = q_tiles;
  for (int t = 1; t <= q_tiles; ++t) {
    const int64_t ctas = int64_t(heads) * ((q_tiles + t - 1) / t);
    if (ctas <= slots) {
      tpc = t;
      break;
    }
  }
  cpb = (q_tiles + tpc - 1) / tpc;
}

static int launch_short(const void* q, int64_t ldq, int64_t qhs, const void* k, int64_t ldk, int64_t khs,
                        const void* v, int64_t ldv, int64_t vhs, int64_t seq_q, int64_t seq_kv, int heads,
                        float scale, const OutMap& om, const int32_t* run_flag, int32_t run_if, cudaStream_t stream) {
  constexpr int D = 128;
  CUtensorMap tq, tk, tv;
  const uint32_t box[3] = {64, 1, 128};
  {
    const uint64_t dims[3] = {D, uint64_t(heads), uint64_t(seq_q)};
    const uint64_t str[2] = {uint64_t(qhs) * 2, uint64_t(ldq) * 2};
    int rc = make_tmap_bf16(&tq, q, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    const uint64_t dims[3] = {D, uint64_t(heads), uint64_t(seq_kv)};
    const uint64_t str[2] = {uint64_t(khs) * 2, uint64_t(ldk) * 2};
    int rc = make_tmap_bf16(&tk, k, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  {
    const uint64_t dims[3] = {D, uint64_t(heads), uint64_t(seq_kv)};
    const uint64_t str[2] = {uint64_t(vhs) * 2, uint64_t(ldv) * 2};
    int rc = make_tmap_bf16(&tv, v, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  CUtensorMap to;
  {
    const uint64_t dims[3] = {D, uint64_t(heads), uint64_t(seq_q)};
    const uint64_t str[2] = {uint64_t(om.o_head_stride) * 2, uint64_t(om.ldo) * 2};
    const uint32_t obox[3] = {64, 1, 32};
    int rc = make_tmap_bf16(&to, om.o, 3, dims, str, obox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  ShortParams p{};
  p.seq_q = int(seq_q), p.seq_kv = int(seq_kv), p.heads = heads;
  p.q_tiles = int((seq_q + BQ - 1) / BQ);
  short_plan(p.q_tiles, heads, p.tiles_per_cta, p.ctas_per_head);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.o = om.o, p.ldo = om.ldo, p.o_head_stride = om.o_head_stride;
  p.run_flag = run_flag, p.run_if = run_if;
  p.trace = g_short_trace.load();
  static int poly = -1;  // AQB_ATTN_POLY: exp2 pairs (of 8) on the FMA pipe, as for the general kernel
  if (poly < 0) {
    const char* e = getenv("AQB_ATTN_POLY");
    poly = (e && !strcmp(e, "0")) ? 0 : (e && !strcmp(e, "2")) ? 2 : (e && !strcmp(e, "4")) ? 4 : 3;
  }
  auto kern = poly == 0 ? attn_short_kernel<0x00> : poly == 2 ? attn_short_kernel<0x22>
                       : poly == 4 ? attn_short_kernel<0x55> : attn_short_kernel<kPolyMaskDefault>;
  static FuncAttrOnce attr[4];
  AQB_CUDA_TRY(set_smem_once(attr[poly == 0 ? 0 : poly == 2 ? 1 : poly == 4 ? 2 : 3], kern, ShortCfg::kSmem));
  const int64_t ctas = int64_t(heads) * p.ctas_per_head;
  AQB_CUDA_TRY(launch_pdl(kern, dim3(unsigned(ctas)), dim3(kThreads), ShortCfg::kSmem, stream, tq, tk, tv, to, p));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

// AQB_ATTN_SHORT=0 routes short KV through the general kernel (benchmarking)
static bool short_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("AQB_ATTN_SHORT");
    on = (e && !strcmp(e, "0")) ? 0 : 1;
  }
  return on == 1;
}

}  // namespace attn
}  // namespace aqb

namespace aqb {
namespace attn {

static int run(const void* q, int64_t ldq, int64_t qhs, const void* k, int64_t ldk, int64_t khs, const void* v,
               int64_t ldv, int64_t vhs, int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim,
               float softmax_scale, int32_t kv_splits, void* workspace, int64_t workspace_bytes, const OutMap& om,
               const int32_t* run_flag, int32_t run_if, cudaStream_t s) {
  AQB_CHECK_ARG(q && k && v, "attention: null pointer");
  AQB_CHECK_ARG(head_dim == 32 || head_dim == 64 || head_dim == 128, "attention: head_dim %d unsupported", head_dim);
  AQB_CHECK_ARG(seq_q >= 1 && seq_kv >= 1 && heads >= 1, "attention: bad shape");
  AQB_CHECK_ARG(seq_q < (1ll << 31) && seq_kv < (1ll << 31), "attention: sequence too long");
  AQB_CHECK_ARG(ldq % 8 == 0 && ldk % 8 == 0 && ldv % 8 == 0 && om.ldo % 8 == 0, "attention: rows must be 16B aligned");
  AQB_CHECK_ARG(qhs % 8 == 0 && khs % 8 == 0 && vhs % 8 == 0 && om.o_head_stride % 8 == 0,
                "attention: head strides must be 16B aligned");
  if (head_dim == 128 && seq_kv <= 2 * BKV && om.nranks == 0 && kv_splits == 0 && short_enabled())
    return launch_short(q, ldq, qhs, k, ldk, khs, v, ldv, vhs, seq_q, seq_kv, heads, softmax_scale, om, run_flag,
                        run_if, s);
  const int nkv = int((seq_kv + BKV - 1) / BKV);
  const int64_t tiles = ((seq_q + 2 * BQ - 1) / (2 * BQ)) * heads;
  AQB_CHECK_ARG(tiles * std::min(kv_splits > 0 ? kv_splits : 16, nkv) < (1ll << 31), "attention: grid too large");
  Plan plan;
  if (kv_splits > 0) {  // forced: every tile split the same way (1 = one pass)
    const int s = std::min(int(kv_splits), nkv);
    const int per = (nkv + s - 1) / s;
    plan = Plan{0, (nkv + per - 1) / per, per, per, 0};
    if (plan.splits == 1) plan = Plan{int(tiles), 1, nkv, nkv, 0};
  } else {
    plan = choose_plan(seq_q, seq_kv, heads, head_dim);
  }
  const int64_t need = split_ws_bytes(tiles - plan.n_whole, plan.splits, head_dim);
  if (need > 0 && (workspace == nullptr || workspace_bytes < need)) {
    AQB_CHECK_ARG(kv_splits <= 1, "attention: workspace of %lld B needed for %d splits", (long long)need, plan.splits);
    plan = Plan{int(tiles), 1, nkv, nkv, 0};  // automatic choice without (enough) workspace: one pass
  }
  Params p{};
  p.seq_q = int(seq_q), p.seq_kv = int(seq_kv), p.heads = heads, p.head_dim = head_dim;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.out = om;
  p.q_pairs = int((seq_q + 2 * BQ - 1) / (2 * BQ));
  p.n_whole = plan.n_whole;
  p.splits = plan.splits;
  p.kv_blocks_per_split = plan.per;
  p.kv_first = plan.first;
  p.split_major = plan.split_major;
  p.part_d = head_dim <= 64 ? 64 : 128;
  const int ring = head_dim == 128 ? Cfg<128>::NS : Cfg<64>::NS;
  p.pairs_per_cta = plan.n_whole == tiles ? choose_pairs_per_cta(p.q_pairs, heads, nkv, ring) : 1;
  if (plan.n_whole < tiles) {
    float* ws = reinterpret_cast<float*>(workspace);
    p.lse = ws;
    const int64_t rows = (tiles - plan.n_whole) * plan.splits * (2 * BQ);
    p.opart = ws + (rows + 63) / 64 * 64;
  }
  p.run_flag = run_flag, p.run_if = run_if;
  if (head_dim == 128) return launch<128>(q, ldq, qhs, k, ldk, khs, v, ldv, vhs, p, s);
  return launch<64>(q, ldq, qhs, k, ldk, khs, v, ldv, vhs, p, s);
}

}  // namespace attn
}  // namespace aqb

extern "C" int64_t aqb_attention_workspace_bytes(int64_t seq_q, int32_t heads, int32_t head_dim, int32_t kv_splits) {
  // any plan with <= kv_splits splits (the all-tiles-split plan is the largest)
  return aqb::attn::split_ws_bytes((seq_q + 255) / 256 * heads, kv_splits, head_dim);
}

extern "C" int64_t aqb_attention_auto_workspace_bytes(int64_t seq_q, int64_t seq_kv, int32_t heads,
                                                      int32_t head_dim) {
  const aqb::attn::Plan pl = aqb::attn::choose_plan(seq_q, seq_kv, heads, head_dim);
  return aqb::attn::split_ws_bytes((seq_q + 255) / 256 * heads - pl.n_whole, pl.splits, head_dim);
}

extern "C" int aqb_attention_splits(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim) {
  return aqb::attn::choose_plan(seq_q, seq_kv, heads, head_dim).splits;
}

extern "C" int aqb_attention_pairs_per_cta(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim) {
  using namespace aqb::attn;
  const Plan pl = choose_plan(seq_q, seq_kv, heads, head_dim);
  const int q_pairs = int((seq_q + 2 * BQ - 1) / (2 * BQ));
  if (pl.n_whole != int64_t(q_pairs) * heads) return 1;
  const int nkv = int((seq_kv + BKV - 1) / BKV);
  return choose_pairs_per_cta(q_pairs, heads, nkv, head_dim == 128 ? Cfg<128>::NS : Cfg<64>::NS);
}

extern "C" int aqb_attention_trace(void* buffer) {
  aqb::attn::g_short_trace.store(reinterpret_cast<unsigned long long*>(buffer));
  return AQB_OK;
}

extern "C" int aqb_attention_plan(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim, int32_t* out) {
  if (out == nullptr) return AQB_EINVAL;
  const aqb::attn::Plan pl = aqb::attn::choose_plan(seq_q, seq_kv, heads, head_dim);
  out[0] = pl.n_whole, out[1] = pl.splits, out[2] = pl.first, out[3] = pl.per, out[4] = pl.split_major;
  return AQB_OK;
}

extern "C" int aqb_attention_whole_tiles(int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim) {
  return aqb::attn::choose_plan(seq_q, seq_kv, heads, head_dim).n_whole;
}

extern "C" int aqb_attention_fwd(const void* q, int64_t ldq, int64_t q_head_stride, const void* k, int64_t ldk,
                                 int64_t k_head_stride, const void* v, int64_t ldv, int64_t v_head_stride, void* o,
                                 int64_t ldo, int64_t o_head_stride, int64_t seq_q, int64_t seq_kv, int32_t heads,
                                 int32_t head_dim, float softmax_scale, int32_t kv_splits, void* workspace,
                                 int64_t workspace_bytes, const int32_t* run_flag, int32_t run_if, void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(o, "attention: null output");
  attn::OutMap om{};
  om.o = reinterpret_cast<__nv_bfloat16*>(o), om.ldo = ldo, om.o_head_stride = o_head_stride;
  return attn::run(q, ldq, q_head_stride, k, ldk, k_head_stride, v, ldv, v_head_stride, seq_q, seq_kv, heads,
                   head_dim, softmax_scale, kv_splits, workspace, workspace_bytes, om, run_flag, run_if,
                   reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int aqb_attention_fwd_scatter(const void* q, int64_t ldq, int64_t q_head_stride, const void* k,
                                         int64_t ldk, int64_t k_head_stride, const void* v, int64_t ldv,
                                         int64_t v_head_stride, void* const* peer_o, int32_t nranks, int64_t ldo,
                                         int64_t o_head_stride, int64_t rows_per_rank, int64_t text_row0,
                                         int64_t seq_q, int64_t seq_kv, int32_t heads, int32_t head_dim,
                                         float softmax_scale, int32_t kv_splits, void* workspace,
                                         int64_t workspace_bytes, const int32_t* run_flag, int32_t run_if,
                                         void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(peer_o && nranks >= 1 && nranks <= attn::kMaxPeers, "attention_scatter: 1..%d ranks", attn::kMaxPeers);
  AQB_CHECK_ARG(rows_per_rank >= 1 && text_row0 == rows_per_rank * nranks && text_row0 <= seq_q,
                "attention_scatter: text_row0 must equal rows_per_rank * nranks");
  attn::OutMap om{};
  om.ldo = ldo, om.o_head_stride = o_head_stride, om.nranks = nranks;
  om.rows_per_rank = rows_per_rank, om.text_row0 = text_row0;
  for (int r = 0; r < nranks; ++r) {
    AQB_CHECK_ARG(peer_o[r] && reinterpret_cast<uintptr_t>(peer_o[r]) % 16 == 0, "attention_scatter: peer_o[%d]", r);
    om.peer_o[r] = reinterpret_cast<__nv_bfloat16*>(peer_o[r]);
  }
  return attn::run(q, ldq, q_head_stride, k, ldk, k_head_stride, v, ldv, v_head_stride, seq_q, seq_kv, heads,
                   head_dim, softmax_scale, kv_splits, workspace, workspace_bytes, om, run_flag, run_if,
                   reinterpret_cast<cudaStream_t>(stream));
}
