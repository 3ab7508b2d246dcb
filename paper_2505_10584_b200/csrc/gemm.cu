// tcgen05 / TMEM / TMA persistent GEMM with fused DiT epilogues (sm_100a).
//
//   acc[m, n] = sum_k A[m, k] * W[n, k]        A: activations, W: nn.Linear weight
//
// Implements the projection rows of the paper's Table 2 with
// GeLU and Gate fused into the epilogue, plus the
// flow-matching Euler update for the final layer.
//
// Two kernels share one epilogue:
//  * gemm_kernel   1 CTA per 128 x BN tile (cta_group::1, UMMA M=128).
//  * gemm2_kernel  a CTA pair (cluster of 2) per 256 x BN tile: each CTA loads
//                  its 128 rows of A and BN/2 rows of W, the leader issues
//                  cta_group::2 MMAs (M=256) that read both CTAs' smem and write
//                  both CTAs' TMEM — half the W bytes per SM (L2->SM operand
//                  bandwidth is what limits 1-CTA tiles).
// Roles (both): warp 0 TMA producer (STAGES-deep 128B-swizzled ring, mbarrier
// full/empty), warp 1 MMA issuer (single thread, TMEM double-buffered 2 x BN
// columns so the epilogue of tile i overlaps the MMAs of tile i+1), warp 2 TMEM
// allocator, warp 3 idle, warps 4-7 epilogue.
//
// Epilogue: per 128-byte-wide column chunk (32 fp32 / 64 bf16 columns), each
// thread (= one TMEM lane = one row) pulls its accumulators with tcgen05.ld,
// the residual chunk (gate*residual) arrives by TMA into a 128B-swizzled smem
// buffer (requested several chunks ahead, across tile boundaries), the thread combines bias / GeLU / gate / residual in registers,
// writes the result back to the swizzled buffer (conflict-free 16 B accesses),
// and one thread TMA-stores the chunk.  All global traffic is TMA (coalesced);
// the two smem buffers alternate so a chunk's store overlaps the next chunk.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int kThreads = 256;
// Internal epilogue (not in the C-ABI): AQB_EPI_GATE_RES without the bf16 copy.  The
// epilogue stages gate * (acc + bias) and a TMA reduce-add performs residual += it at
// L2, so the SM never reads the residual: no residual buffers (full pipeline depth)
// and a third of the epilogue's shared-memory traffic.
constexpr int kEpiGateAdd = 100;
// Internal epilogue of aqb_gemm_gate_add_scatter (TP-SP row-parallel projection +
// reduce-scatter): the same staged gate * (acc + bias), reduce-added into the residual
// of the rank that owns each row (peer memory) — a TMA reduce-add per 128-row CTA
// block that lies in one rank's rows, per-thread red.global.add.v4 for a block that
// straddles two ranks.
constexpr int kEpiGateAddScatter = 101;
// Internal: the QK-norm epilogue without RoPE (cross-attention q, text rows): no shared
// RoPE tiles, so the pair kernel keeps its full pipeline depth.
constexpr int kEpiQkNoRope = 102;
__host__ __device__ constexpr bool is_qk(int epi) { return epi == AQB_EPI_QKNORM_ROPE || epi == kEpiQkNoRope; }
constexpr int kEpiBuf = 128 * 128;  // one epilogue chunk: 128 rows x 128 B
constexpr int kAuxBuf = 128 * 64;   // bf16 copy of a gate*residual chunk: 128 rows x 64 B (64B swizzle)

struct Params {
  int M, N, K;
  int num_m, num_n, num_tiles, group_m;
  // Work units: tiles [0, n_full) are whole BN-wide tiles; each later tile runs as two
  // BN/2-wide units (pair kernel, BN = 256), so a short last wave takes half as long.
  int n_full, num_units;
  void* out;
  int64_t ldo;
  const float* bias;
  const float* gate;
  const float* alpha;
  __nv_bfloat16* aux;
  int64_t ld_aux;
  const int32_t* run_flag;
  int32_t run_if;
  // QK-norm + RoPE epilogue (AQB_EPI_QKNORM_ROPE): columns are [parts][heads][128]
  const float* norm_w0;   // q weight [128]
  const float* norm_w1;   // k weight [128]
  const float* rope_cos;  // [rope_rows, 64]
  const float* rope_sin;
  int64_t rope_row0, rope_rows;
  int part_width;         // heads * 128
  int norm_parts;         // parts < norm_parts are RMS-normed (+ RoPE)
  int hpg, g_base, groups;  // heads per output group (Ulysses), group offset, group count
  int peer_groups;          // 1: group g is TMA-stored through PeerMaps::m[g] (another rank's buffer)
  float eps;
  // gate-add scatter (kEpiGateAddScatter): rank r's residual, rows_per_rank rows of stride ldo
  float* red_dst[8];
  int64_t red_rpr;
  // profiling hook (aqb_gemm_trace): per CTA 128 clock64 stamps (see gstamp); null: off
  unsigned long long* trace;
};

// Trace slots per CTA: 0 entry, 1 entry globaltimer, 2 setup done, 3 after the PDL wait,
// 8 + i: MMA warp passes the full barrier of its i-th k-block (i < 96; pair kernel: leader),
// 104 + 2j / 105 + 2j: epilogue warp 4 sees tile j's accumulator / finishes it (j < 8),
// 120: epilogue stores drained, 121: exit globaltimer.
// Compiled in only with -DAQB_GEMM_TRACE (AQB_BUILD_DEFINES=-DAQB_GEMM_TRACE at build time): the
// per-k-block check cost 0.3-1% on the small shards when always present.
__device__ __forceinline__ void gstamp(const Params& p, int slot, bool global_timer = false) {
#ifdef AQB_GEMM_TRACE
  if (p.trace != nullptr) {
    unsigned long long t;
    if (global_timer)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    else
      t = clock64();
    p.trace[int64_t(blockIdx.x) * 128 + slot] = t;
  }
#else
  (void)p, (void)slot, (void)global_timer;
#endif
}

// Per-destination-rank output maps of the Ulysses scatter (QK-norm epilogue):
// map g addresses this rank's row block inside rank g's attention-input buffer.
constexpr int kMaxPeers = 8;
struct PeerMaps {
  CUtensorMap m[kMaxPeers];
  CUtensorMap bh;  // W with a BN/4-row box: the half-width tail units of the pair kernel
  CUtensorMap rcos, rsin;  // QK-norm + RoPE epilogue: [rope_rows, 64] f32 tables, 32 x 128-row boxes
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

// Unit u -> (M block, first column, width): whole tiles first, then half-width tail units.
template <int BN>
__device__ __forceinline__ void unit_coords(const Params& p, int u, int& mb, int& col0, int& width) {
  int nb;
  if (u < p.n_full) {
    tile_coords(p, u, mb, nb);
    col0 = nb * BN, width = BN;
  } else {
    const int v = u - p.n_full;
    tile_coords(p, p.n_full + (v >> 1), mb, nb);
    col0 = nb * BN + (v & 1) * (BN / 2), width = BN / 2;
  }
}

__device__ __forceinline__ float4 ld_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_f4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// Euler epilogue of the (tiny, N = patch_dim) final layer: direct stores.
__device__ __forceinline__ void euler_chunk(const Params& p, int row, int col0, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (p.bias != nullptr) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (col0 + i < p.N) v[i] += __ldg(p.bias + col0 + i);
  }
  if (row >= p.M) return;
  const float a = __ldg(p.alpha);
  float* out = reinterpret_cast<float*>(p.out) + static_cast<int64_t>(row) * p.ldo + col0;
  __nv_bfloat16* aux = p.aux + static_cast<int64_t>(row) * p.ld_aux + col0;
  float4 xs[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) xs[i] = (col0 + 4 * i < p.N) ? ld_f4(out + 4 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (col0 + 8 * i < p.N) {
      float4 x0 = xs[2 * i], x1 = xs[2 * i + 1];
      x0.x += a * v[8 * i + 0], x0.y += a * v[8 * i + 1], x0.z += a * v[8 * i + 2], x0.w += a * v[8 * i + 3];
      x1.x += a * v[8 * i + 4], x1.y += a * v[8 * i + 5], x1.z += a * v[8 * i + 6], x1.w += a * v[8 * i + 7];
      st_f4(out + 8 * i, x0);
      st_f4(out + 8 * i + 4, x1);
      if (p.aux)
        *reinterpret_cast<uint4*>(aux + 8 * i) = make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w),
                                                            pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
    }
  }
}

// Per-CTA epilogue state (warps 4-7 only).
struct EpiState {
  uint8_t* buf;      // epi_bufs x kEpiBuf, 1024-aligned (gate*residual: + 2 x kAuxBuf bf16 copies)
  uint64_t* bar;     // one mbarrier per buffer (residual TMA loads)
  uint32_t chunk;    // chunks processed by this CTA (buffer / phase bookkeeping; aux buffers)
  // gate*residual residual stream: chunk index space idx = tile_iter * (BN / 32) + c, where
  // tile_iter counts this CTA's tiles (first_tile, first_tile + tile_stride, ...)
  int first_tile, tile_stride, tile_m, row_off;
  uint32_t tiles_done;   // tile_iter of the tile being drained
  uint32_t issued;       // residual chunks requested so far (idx < issued)
  uint32_t phase_bits;   // per-buffer mbarrier parity (loads happen only for valid chunks)
  // QK-norm + RoPE (pair kernel): the tile's 128 rows of the cos / sin tables, TMA-loaded
  // into shared memory (cos lo|hi, sin lo|hi: 4 x [128 rows][128 B], 128B-swizzled) while
  // the accumulator fills, instead of per-row global loads in the epilogue
  uint8_t* rope;         // nullptr: global loads
  uint64_t* rbar;
  uint32_t rphase;
};

constexpr int kSmemMax = 232448;
constexpr int kFixedRes = 2 * kAuxBuf + 1024 + 256;  // aux copies + alignment + barriers

template <int BN, bool PAIR>
constexpr int stage_bytes() { return (BM + (PAIR ? BN / 2 : BN)) * BK * 2; }

// gate*residual streams the f32 residual through NB buffers, requested NB-2 chunks
// ahead (across tile boundaries); every buffer left after the pipeline stages is used,
// up to 8.  Measured: 5 buffers / 4 stages was no faster than 3 / 5 on the K = H
// projections and 10% slower on K = 4H, so res_stages keeps the stages.  The
// store-only epilogues need two.
template <int BN, int STAGES, bool PAIR, int EPI>
constexpr int epi_bufs() {
  if (EPI != AQB_EPI_GATE_RES) return 2;
  const int n = (kSmemMax - kFixedRes - STAGES * stage_bytes<BN, PAIR>()) / kEpiBuf;
  return n > 8 ? 8 : n;
}

// pipeline stages of the gate*residual variant: the most that leave >= 3 residual buffers
template <int BN, int STAGES, bool PAIR>
constexpr int res_stages() {
  for (int s = STAGES; s > 3; --s)
    if ((kSmemMax - kFixedRes - s * stage_bytes<BN, PAIR>()) / kEpiBuf >= 3) return s;
  return 3;
}

template <int EPI>
constexpr int aux_bytes() { return EPI == AQB_EPI_GATE_RES ? 2 * kAuxBuf : 0; }

// shared-memory RoPE tables of the QK-norm epilogue (pair kernel only)
template <int EPI, bool PAIR>
constexpr int rope_bytes() { return (EPI == AQB_EPI_QKNORM_ROPE && PAIR) ? 4 * kEpiBuf : 0; }

// pipeline stages of the QK-norm variant: the most that leave room for the RoPE tiles
template <int BN, int STAGES, bool PAIR>
constexpr int qk_stages() {
  for (int s = STAGES; s > 2; --s)
    if (s * stage_bytes<BN, PAIR>() + 2 * kEpiBuf + rope_bytes<AQB_EPI_QKNORM_ROPE, PAIR>() + 1024 + 256 <=
        kSmemMax)
      return s;
  return 2;
}

template <int EPI>
constexpr int epi_cols() {
  return (EPI == AQB_EPI_F32 || EPI == AQB_EPI_GATE_RES || EPI == kEpiGateAdd || EPI == kEpiGateAddScatter) ? 32 : 64;
}

// Request residual chunk `idx` (leader thread; no-op past the last tile / column N).
template <int BN, int NB>
__device__ __forceinline__ void res_request(const Params& p, const CUtensorMap* tmo, EpiState& es, uint32_t idx) {
  constexpr int CPT = BN / 32;
  const int u = es.first_tile + int(idx / CPT) * es.tile_stride;
  if (u >= p.num_units) return;
  int mb, col0, width;
  unit_coords<BN>(p, u, mb, col0, width);
  const int c = int(idx % CPT) * 32;
  const int col = col0 + c;
  if (c >= width || col >= p.N) return;
  const uint32_t b = idx % NB;
  bulk_wait_read<1>();  // buffer b was last TMA-stored from two chunks ago
  mbar_arrive_expect_tx(es.bar + b, kEpiBuf);
  tma_load_2d(es.buf + b * kEpiBuf, tmo, es.bar + b, col, mb * es.tile_m + es.row_off, kEvictFirst);
}

// Residual prefetch before the first tile's accumulator wait, so the stream's
// start-up latency hides behind the first tile's MMAs.
template <int EPI, int BN, int NB>
__device__ __forceinline__ void epilogue_prologue(const Params& p, const CUtensorMap* tmo, const PeerMaps* pm,
                                                  EpiState& es, int row0, bool leader_thread) {
  if constexpr (is_qk(EPI)) {
    // the previous tile's epilogue ended with a named barrier: the rope buffer is free
    if (es.rope != nullptr && leader_thread && p.rope_row0 + row0 < p.rope_rows) {
      mbar_arrive_expect_tx(es.rbar, 4 * kEpiBuf);
      const int y = int(p.rope_row0 + row0);
      tma_load_2d(es.rope + 0 * kEpiBuf, &pm->rcos, es.rbar, 0, y, kEvictNormal);
      tma_load_2d(es.rope + 1 * kEpiBuf, &pm->rcos, es.rbar, 32, y, kEvictNormal);
      tma_load_2d(es.rope + 2 * kEpiBuf, &pm->rsin, es.rbar, 0, y, kEvictNormal);
      tma_load_2d(es.rope + 3 * kEpiBuf, &pm->rsin, es.rbar, 32, y, kEvictNormal);
    }
  }
  if constexpr (EPI == AQB_EPI_GATE_RES) {
    if (es.issued == 0) {
      if (leader_thread)
        for (uint32_t i = 0; i < NB - 2; ++i) res_request<BN, NB>(p, tmo, es, i);
      es.issued = NB - 2;
    }
  }
}

// One accumulator tile (this CTA's 128 rows x BN columns starting at col_base).
template <int EPI, int BN, int NB>
__device__ __forceinline__ void epilogue_tile(const Params& p, const CUtensorMap* tmo, const PeerMaps* pm, EpiState& es,
                                              uint32_t tacc, int row0, int col_base, int width, uint32_t q,
                                              uint32_t lane) {
  const int r = q * 32 + lane;           // row within the CTA tile (= TMEM lane)
  const uint32_t lane_off = (q * 32) << 16;
  const bool leader_thread = (q == 0 && lane == 0);
  if constexpr (EPI == AQB_EPI_EULER) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      if (c >= width || col_base + c >= p.N) break;
      uint32_t u[32];
      tmem_ld32(tacc + c + lane_off, u);
      tmem_wait_ld();
      euler_chunk(p, row0 + r, col_base + c, u);
    }
    return;
  } else if constexpr (is_qk(EPI)) {
    // One 128-column head at a time: RMS-norm (+ RoPE) in registers, then two
    // 64-column chunks through the swizzled smem buffers and a 5-D TMA store
    // that lands in the [group][row][part][head][128] layout (natural or packed).
    const bool rope_tile = p.rope_row0 + row0 < p.rope_rows;  // CTA-uniform
    const bool rope_smem = es.rope != nullptr && rope_tile;
    if (rope_smem) {
      mbar_wait(es.rbar, es.rphase);
      es.rphase ^= 1;
    }
    const uint32_t rope_row = smem_u32(es.rope) + r * 128, rsw = r & 7;
#pragma unroll 1
    for (int hc = 0; hc < BN; hc += 128) {
      const int colh = col_base + hc;
      if (hc >= width || colh >= p.N) break;
      // bias requested before the accumulator load (its latency overlaps it; -0 is the
      // additive identity, so the sum has the same bits as adding after)
      float v[128];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float4 bb = p.bias != nullptr ? __ldg(reinterpret_cast<const float4*>(p.bias + colh) + i)
                                            : make_float4(-0.f, -0.f, -0.f, -0.f);
        v[4 * i] = bb.x, v[4 * i + 1] = bb.y, v[4 * i + 2] = bb.z, v[4 * i + 3] = bb.w;
      }
      {
        uint32_t u[32];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          tmem_ld32(tacc + hc + 32 * h + lane_off, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[32 * h + i] += __uint_as_float(u[i]);
        }
      }
      const int part = colh / p.part_width;
      const int head = (colh - part * p.part_width) >> 7;
      const int grp = head / p.hpg - p.g_base;
      if (grp < 0 || grp >= p.groups) continue;  // head not stored on this rank (TMA stores need coords >= 0)
      if (part < p.norm_parts) {
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < 128; ++i) ss += v[i] * v[i];
        const float rstd = rsqrtf(ss * (1.f / 128.f) + p.eps);
        const float4* w4 = reinterpret_cast<const float4*>(part == 0 ? p.norm_w0 : p.norm_w1);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float4 w = __ldg(w4 + i);
          v[4 * i] *= rstd * w.x, v[4 * i + 1] *= rstd * w.y, v[4 * i + 2] *= rstd * w.z, v[4 * i + 3] *= rstd * w.w;
        }
        const int64_t grow = p.rope_row0 + row0 + r;
        if (grow < p.rope_rows) {
          const float4* c4 = reinterpret_cast<const float4*>(p.rope_cos + grow * 64);
          const float4* s4 = reinterpret_cast<const float4*>(p.rope_sin + grow * 64);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float4 cc, sn;
            if (rope_smem) {  // float4 i of the row: box i/8, 16-byte chunk i%8 (128B swizzle)
              const uint32_t off = rope_row + (i >> 3) * kEpiBuf + ((((i & 7) ^ rsw)) << 4);
              const uint4 a = lds128(off), b = lds128(off + 2 * kEpiBuf);
              cc = make_float4(__uint_as_float(a.x), __uint_as_float(a.y), __uint_as_float(a.z), __uint_as_float(a.w));
              sn = make_float4(__uint_as_float(b.x), __uint_as_float(b.y), __uint_as_float(b.z), __uint_as_float(b.w));
            } else {
              cc = __ldg(c4 + i), sn = __ldg(s4 + i);
            }
            const float cs[4] = {cc.x, cc.y, cc.z, cc.w}, sv[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int e = 8 * i + 2 * j;
              const float a = v[e], b = v[e + 1];
              v[e] = a * cs[j] - b * sv[j];
              v[e + 1] = a * sv[j] + b * cs[j];
            }
          }
        }
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t b = es.chunk & 1;
        uint8_t* buf = es.buf + b * kEpiBuf;
        if (leader_thread) bulk_wait_read<1>();
        named_bar_sync(1, 128);
        const uint32_t rowaddr = smem_u32(buf) + r * 128;
        const uint32_t sw = r & 7;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float* t = v + 64 * half + 8 * i;
          st_shared_v4(rowaddr + ((i ^ sw) << 4), pack_bf16(t[0], t[1]), pack_bf16(t[2], t[3]), pack_bf16(t[4], t[5]),
                       pack_bf16(t[6], t[7]));
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (leader_thread) {
          if (p.peer_groups)
            tma_store_5d(&pm->m[grp], buf, 64 * half, head % p.hpg, part, row0, 0);
          else
            tma_store_5d(tmo, buf, 64 * half, head % p.hpg, part, row0, grp);
          bulk_commit();
        }
        ++es.chunk;
      }
    }
    if (es.rope != nullptr) named_bar_sync(1, 128);  // every row's RoPE read: the next tile may reload
  } else {
    constexpr int CW = epi_cols<EPI>();  // columns per 128-byte chunk
#pragma unroll 1
    for (int c = 0; c < BN; c += CW) {
      const int col0 = col_base + c;
      uint32_t b;
      if constexpr (EPI == AQB_EPI_GATE_RES) {
        // chunk idx's residual was requested NB-2 chunks ago; request idx + NB - 2
        const uint32_t idx = es.tiles_done * (BN / 32) + c / 32;
        if (leader_thread && idx + NB - 2 >= es.issued) res_request<BN, NB>(p, tmo, es, idx + NB - 2);
        es.issued = idx + NB - 1;
        if (c >= width || col0 >= p.N) continue;  // uniform over the 128 epilogue threads
        b = idx % NB;
      } else {
        if (c >= width || col0 >= p.N) break;  // uniform over the 128 epilogue threads
        b = es.chunk % NB;
      }
      uint8_t* buf = es.buf + b * kEpiBuf;
      if constexpr (EPI == AQB_EPI_GATE_RES) {
      } else {
        // buffer b was last read by the TMA store issued NB chunks ago
        if (leader_thread) bulk_wait_read<NB - 1>();
        named_bar_sync(1, 128);
      }
      // bias and gate are requested before the accumulator load so their L2 latency
      // overlaps it (acc + bias == bias + acc: the same bits as adding after)
      float v[CW];
#pragma unroll
      for (int i = 0; i < CW / 4; ++i) {
        const float4 bb = (p.bias != nullptr && col0 + 4 * i < p.N)
                              ? __ldg(reinterpret_cast<const float4*>(p.bias + col0) + i)
                              : make_float4(-0.f, -0.f, -0.f, -0.f);  // -0: the additive identity
        v[4 * i] = bb.x, v[4 * i + 1] = bb.y, v[4 * i + 2] = bb.z, v[4 * i + 3] = bb.w;
      }
      constexpr bool kGate = EPI == AQB_EPI_GATE_RES || EPI == kEpiGateAdd || EPI == kEpiGateAddScatter;
      float4 gr[kGate ? 8 : 1];
      if constexpr (kGate) {
        const float4* g4 = reinterpret_cast<const float4*>(p.gate + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          gr[i] = (p.gate && col0 + 4 * i < p.N) ? __ldg(g4 + i) : make_float4(1.f, 1.f, 1.f, 1.f);
      }
      {
        uint32_t u[32];
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) {
          tmem_ld32(tacc + c + 32 * h + lane_off, u);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[32 * h + i] += __uint_as_float(u[i]);
        }
      }
      const uint32_t rowaddr = smem_u32(buf) + r * 128;
      const uint32_t sw = r & 7;
      uint8_t* abuf = es.buf + NB * kEpiBuf + (es.chunk & 1) * kAuxBuf;
      if constexpr (EPI == AQB_EPI_GATE_RES) {
        if (p.aux != nullptr) {  // the aux buffer was last stored two chunks ago
          if (leader_thread) bulk_wait_read<1>();
          named_bar_sync(1, 128);
        }
        mbar_wait(es.bar + b, (es.phase_bits >> b) & 1);
        es.phase_bits ^= 1u << b;
        const uint32_t arow = smem_u32(abuf) + r * 64, asw = (r >> 1) & 3;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          float nx[8];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t a = rowaddr + (((i + h) ^ sw) << 4);
            const uint4 xr = lds128(a);
            const float4 g = gr[i + h];
            nx[4 * h + 0] = __uint_as_float(xr.x) + g.x * v[4 * (i + h)];
            nx[4 * h + 1] = __uint_as_float(xr.y) + g.y * v[4 * (i + h) + 1];
            nx[4 * h + 2] = __uint_as_float(xr.z) + g.z * v[4 * (i + h) + 2];
            nx[4 * h + 3] = __uint_as_float(xr.w) + g.w * v[4 * (i + h) + 3];
            st_shared_v4(a, __float_as_uint(nx[4 * h]), __float_as_uint(nx[4 * h + 1]),
                         __float_as_uint(nx[4 * h + 2]), __float_as_uint(nx[4 * h + 3]));
          }
          if (p.aux != nullptr)  // bf16(new residual): the next projection's A operand
            st_shared_v4(arow + (((i >> 1) ^ asw) << 4), pack_bf16(nx[0], nx[1]), pack_bf16(nx[2], nx[3]),
                         pack_bf16(nx[4], nx[5]), pack_bf16(nx[6], nx[7]));
        }
      } else if constexpr (EPI == AQB_EPI_F32) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          st_shared_v4(rowaddr + ((i ^ sw) << 4), __float_as_uint(v[4 * i]), __float_as_uint(v[4 * i + 1]),
                       __float_as_uint(v[4 * i + 2]), __float_as_uint(v[4 * i + 3]));
      } else if constexpr (EPI == kEpiGateAddScatter) {
        const int64_t first = int64_t(row0), last = min(int64_t(row0) + BM, int64_t(p.M)) - 1;
        if (first / p.red_rpr == last / p.red_rpr) {  // CTA block inside one rank: stage for TMA
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 g = gr[i];
            st_shared_v4(rowaddr + ((i ^ sw) << 4), __float_as_uint(g.x * v[4 * i]),
                         __float_as_uint(g.y * v[4 * i + 1]), __float_as_uint(g.z * v[4 * i + 2]),
                         __float_as_uint(g.w * v[4 * i + 3]));
          }
        } else {  // straddles a rank boundary: each thread reduces its own row
          const int64_t row = int64_t(row0) + r;
          if (row < p.M) {
            const int64_t rk = row / p.red_rpr;
            float* dst = p.red_dst[rk] + (row - rk * p.red_rpr) * p.ldo + col0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (col0 + 4 * i < p.N) {
                const float4 g = gr[i];
                red_add_v4_sys(dst + 4 * i, g.x * v[4 * i], g.y * v[4 * i + 1], g.z * v[4 * i + 2],
                               g.w * v[4 * i + 3]);
              }
            }
          }
          ++es.chunk;
          continue;  // uniform: no staged tile, no TMA op for this chunk
        }
      } else if constexpr (EPI == kEpiGateAdd) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 g = gr[i];
          st_shared_v4(rowaddr + ((i ^ sw) << 4), __float_as_uint(g.x * v[4 * i]), __float_as_uint(g.y * v[4 * i + 1]),
                       __float_as_uint(g.z * v[4 * i + 2]), __float_as_uint(g.w * v[4 * i + 3]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float t[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) t[j] = (EPI == AQB_EPI_GELU_BF16) ? gelu_tanh(v[8 * i + j]) : v[8 * i + j];
          st_shared_v4(rowaddr + ((i ^ sw) << 4), pack_bf16(t[0], t[1]), pack_bf16(t[2], t[3]), pack_bf16(t[4], t[5]),
                       pack_bf16(t[6], t[7]));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (leader_thread) {
        if constexpr (EPI == kEpiGateAdd)
          tma_reduce_add_2d(tmo, buf, col0, row0);  // residual += staged tile (clipped like a store)
        else if constexpr (EPI == kEpiGateAddScatter)
          tma_reduce_add_2d(&pm->m[row0 / p.red_rpr], buf, col0, int(row0 % p.red_rpr));  // owner's rows
        else
          tma_store_2d(tmo, buf, col0, row0);  // clips rows >= M and columns >= N
        if constexpr (EPI == AQB_EPI_GATE_RES) {
          if (p.aux != nullptr) tma_store_2d(&pm->m[0], abuf, col0, row0);
        }
        bulk_commit();
      }
      ++es.chunk;
    }
    if constexpr (EPI == AQB_EPI_GATE_RES) ++es.tiles_done;
  }
}

template <int BN, int STAGES, bool PAIR, int EPI>
constexpr int smem_bytes() {
  return STAGES * (BM + (PAIR ? BN / 2 : BN)) * BK * 2 + epi_bufs<BN, STAGES, PAIR, EPI>() * kEpiBuf + aux_bytes<EPI>() +
         rope_bytes<EPI, PAIR>() +
         1024 /*align*/ + 256 /*bars*/;
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ CUtensorMap tma_o, const __grid_constant__ PeerMaps pm, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(base);
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(base + STAGES * BM * BK * 2);
  uint8_t* ebuf = base + STAGES * (BM + BN) * BK * 2;
  constexpr int NB = epi_bufs<BN, STAGES, false, EPI>();
  static_assert(EPI != AQB_EPI_GATE_RES || NB >= 3, "gate*residual needs >= 3 residual buffers (NB - 2 prefetch)");
  uint64_t* full = reinterpret_cast<uint64_t*>(ebuf + NB * kEpiBuf + aux_bytes<EPI>());
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + NB + 1);  // ebar[NB]: rope barrier slot (unused here)

  constexpr uint32_t kTmemCols = 2 * BN;
  const uint32_t warp = warp_idx(), lane = lane_idx();

  if (warp == 0 && lane == 0) {
    gstamp(p, 0);
    gstamp(p, 1, true);
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    tma_prefetch_desc(&tma_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    for (int b = 0; b < NB; ++b) mbar_init(ebar + b, 1);
    mbar_init(ebar + NB, 1);  // rope tables (QK-norm epilogue)
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nk = (p.K + BK - 1) / BK;
  if (threadIdx.x == 0) gstamp(p, 2);
  // the prologue above overlaps the previous kernel's tail (PDL); inputs only after this
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) gstamp(p, 3);
  const bool run = gate_open(p.run_flag, p.run_if);

  if (!run) {
  } else if (warp == 0) {
    // producer and MMA issuer run warp-wide with one elected lane per TMA / tcgen05 op,
    // so descriptors stay in uniform registers (no per-op waterfall loop)
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < p.num_units; t += gridDim.x) {  // 1-CTA: every unit is a whole tile
      int mb, nb;
      tile_coords(p, t, mb, nb);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(empty + stage, phase ^ 1);
        if (elect_one()) mbar_arrive_expect_tx(full + stage, (BM + BN) * BK * 2);
        if (elect_one()) tma_load_2d(sa + stage * BM * BK, &tma_a, full + stage, kb * BK, mb * BM);
        if (elect_one()) tma_load_2d(sb + stage * BN * BK, &tma_b, full + stage, kb * BK, nb * BN);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t kIdesc = idesc_bf16(BM, BN, 0, 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int kseen = 0;
    for (int t = blockIdx.x; t < p.num_units; t += gridDim.x) {
      mbar_wait(tempty + acc, acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tm + acc * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(full + stage, phase);
        tc_fence_after();
        if (lane == 0 && kseen < 96) gstamp(p, 8 + kseen);
        ++kseen;
        const uint32_t a0 = smem_u32(sa + stage * BM * BK);
        const uint32_t b0 = smem_u32(sb + stage * BN * BK);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // K-major SW128: +32 B per 16-element K step inside the 128 B swizzle row.
          const uint64_t da = smem_desc(a0 + 32 * k, 0, 1024), db = smem_desc(b0 + 32 * k, 0, 1024);
          if (elect_one()) umma_bf16_ss(d, da, db, kIdesc, (kb | k) != 0);
        }
        if (elect_one()) umma_commit(empty + stage);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
      if (elect_one()) umma_commit(tfull + acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    EpiState es{ebuf, ebar, 0, int(blockIdx.x), int(gridDim.x), BM, 0, 0, 0, 0, nullptr, nullptr, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    int j = 0;
    for (int t = blockIdx.x; t < p.num_units; t += gridDim.x, ++j) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      epilogue_prologue<EPI, BN, NB>(p, &tma_o, &pm, es, mb * BM, q == 0 && lane == 0);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      if (q == 0 && lane == 0 && j < 8) gstamp(p, 104 + 2 * j);
      epilogue_tile<EPI, BN, NB>(p, &tma_o, &pm, es, tmem + acc * BN, mb * BM, nb * BN, BN, q, lane);
      if (q == 0 && lane == 0 && j < 8) gstamp(p, 105 + 2 * j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (q == 0 && lane == 0) {
      bulk_wait<0>();
      gstamp(p, 120);
      gstamp(p, 121, true);
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
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 const __grid_constant__ CUtensorMap tma_o, const __grid_constant__ PeerMaps pm, Params p) {
  constexpr int BNH = BN / 2;  // W rows per CTA
  constexpr int kABytes = BM * BK * 2, kBBytes = BNH * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = base;
  uint8_t* sb = base + STAGES * kABytes;
  uint8_t* ebuf = base + STAGES * (kABytes + kBBytes);
  constexpr int NB = epi_bufs<BN, STAGES, true, EPI>();
  static_assert(EPI != AQB_EPI_GATE_RES || NB >= 3, "gate*residual needs >= 3 residual buffers (NB - 2 prefetch)");
  uint8_t* rope_buf = ebuf + NB * kEpiBuf + aux_bytes<EPI>();  // rope_bytes<EPI, true>() (QK-norm only)
  uint64_t* full = reinterpret_cast<uint64_t*>(rope_buf + rope_bytes<EPI, true>());
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;
  uint64_t* rbar = ebar + NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);

  constexpr uint32_t kTmemCols = 2 * BN;
  const uint32_t warp = warp_idx(), lane = lane_idx();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    gstamp(p, 0);
    gstamp(p, 1, true);
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    tma_prefetch_desc(&tma_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 2);   // leader's expect_tx arrive + the peer's remote arrive
      mbar_init(empty + s, 1);  // multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);   // multicast MMA commit
      mbar_init(tempty + a, 8);  // 4 epilogue warps x 2 CTAs (used on the leader)
    }
    for (int b = 0; b < NB; ++b) mbar_init(ebar + b, 1);
    mbar_init(ebar + NB, 1);  // rope tables (QK-norm epilogue)
    fence_barrier_init();
    gstamp(p, 4);
  }
  // one cluster barrier publishes both the initialised mbarriers (before any remote arrive or
  // pair TMA signals them) and the pair TMEM allocation (written to this CTA's own smem);
  // a second barrier between the two cost 700-1,200 cycles of prologue per launch
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, kTmemCols);
    if (lane == 0) gstamp(p, 6);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x == 0) gstamp(p, 7);
  const uint32_t tmem = *tmem_slot;
  const int nk = (p.K + BK - 1) / BK;
  if (threadIdx.x == 0) gstamp(p, 2);
  pdl_wait();  // prologue overlapped the previous kernel (PDL); inputs only after this
  pdl_trigger();
  if (threadIdx.x == 0) gstamp(p, 3);
  const bool run = gate_open(p.run_flag, p.run_if);

  if (!run) {
  } else if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int u = cluster; u < p.num_units; u += nclusters) {
      int mb, col0, width;
      unit_coords<BN>(p, u, mb, col0, width);
      const bool half = width != BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(empty + stage, phase ^ 1);
        if (elect_one())
          tma_load_2d_pair(sa + stage * kABytes, &tma_a, full + stage, kb * BK, mb * (2 * BM) + rank * BM);
        if (elect_one()) {
          if (half)
            tma_load_2d_pair(sb + stage * kBBytes, &pm.bh, full + stage, kb * BK, col0 + rank * (BNH / 2));
          else
            tma_load_2d_pair(sb + stage * kBBytes, &tma_b, full + stage, kb * BK, col0 + rank * BNH);
        }
        if (elect_one()) {
          if (leader)
            mbar_arrive_expect_tx(full + stage, 2 * (kABytes + (half ? kBBytes / 2 : kBBytes)));
          else
            mbar_arrive_cluster(full + stage, 0);
        }
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t kIdesc = idesc_bf16(2 * BM, BN, 0, 0);
      constexpr uint32_t kIdescHalf = idesc_bf16(2 * BM, BN / 2, 0, 0);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int kseen = 0;
      for (int u = cluster; u < p.num_units; u += nclusters) {
        const uint32_t idesc = u < p.n_full ? kIdesc : kIdescHalf;
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tm + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          if (lane == 0 && kseen < 96) gstamp(p, 8 + kseen);
          ++kseen;
          const uint32_t a0 = smem_u32(sa + stage * kABytes);
          const uint32_t b0 = smem_u32(sb + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = smem_desc(a0 + 32 * k, 0, 1024), db = smem_desc(b0 + 32 * k, 0, 1024);
            if (elect_one()) umma_bf16_pair(d, da, db, idesc, (kb | k) != 0);
          }
          if (elect_one()) umma_commit_pair(empty + stage);
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
        if (elect_one()) umma_commit_pair(tfull + acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;
    EpiState es{ebuf, ebar, 0, cluster, nclusters, 2 * BM, int(rank) * BM, 0, 0, 0,
                rope_bytes<EPI, true>() ? rope_buf : nullptr, rbar, 0};
    int acc = 0;
    uint32_t acc_phase = 0;
    int j = 0;
    for (int u = cluster; u < p.num_units; u += nclusters, ++j) {
      int mb, col0, width;
      unit_coords<BN>(p, u, mb, col0, width);
      epilogue_prologue<EPI, BN, NB>(p, &tma_o, &pm, es, mb * (2 * BM) + int(rank) * BM, q == 0 && lane == 0);
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      if (q == 0 && lane == 0 && j < 8) gstamp(p, 104 + 2 * j);
      epilogue_tile<EPI, BN, NB>(p, &tma_o, &pm, es, tmem + acc * BN, mb * (2 * BM) + rank * BM, col0, width, q,
                                 lane);
      if (q == 0 && lane == 0 && j < 8) gstamp(p, 105 + 2 * j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(tempty + acc);
        else
          mbar_arrive_cluster(tempty + acc, 0);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (q == 0 && lane == 0) {
      bulk_wait<0>();
      gstamp(p, 120);
      gstamp(p, 121, true);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, kTmemCols);
  }
}

template <int BN, int STAGES, int EPI, bool PAIR>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const PeerMaps& pm, const Params& p,
           cudaStream_t stream) {
  constexpr int smem = smem_bytes<BN, STAGES, PAIR, EPI>();
  static_assert(smem <= 232448, "shared memory budget");
  // select at compile time: only the variant that runs is instantiated (a pair variant's
  // stage count need not leave room for the single-CTA kernel's buffers)
  auto kern = [] {
    if constexpr (PAIR) return gemm2_kernel<BN, STAGES, EPI>;
    else return gemm_kernel<BN, STAGES, EPI>;
  }();
  static FuncAttrOnce attr;  // per instantiation; the attribute is per function and per device
  AQB_CUDA_TRY(set_smem_once(attr, kern, smem));
  int grid;
  if (PAIR) {
    const int pairs = sm_count() / 2;
    grid = 2 * (p.num_units < pairs ? p.num_units : pairs);
  } else {
    grid = p.num_units < sm_count() ? p.num_units : sm_count();
  }
  AQB_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kThreads), smem, stream, ta, tb, to, pm, p));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

template <int BN, int STAGES, bool PAIR>
int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const PeerMaps& pm,
                 const Params& p, cudaStream_t s) {
  // gate*residual trades pipeline stages for residual buffers (see epi_bufs / res_stages)
  constexpr int kResStages = res_stages<BN, STAGES, PAIR>();
  switch (epi) {
    case AQB_EPI_BF16: return launch<BN, STAGES, AQB_EPI_BF16, PAIR>(ta, tb, to, pm, p, s);
    case AQB_EPI_GELU_BF16: return launch<BN, STAGES, AQB_EPI_GELU_BF16, PAIR>(ta, tb, to, pm, p, s);
    case AQB_EPI_GATE_RES:
      // the residual-reading epilogue needs >= 3 residual buffers (it requests NB-2 chunks
      // ahead); variants whose shared memory cannot hold them are never instantiated
      if constexpr (epi_bufs<BN, kResStages, PAIR, AQB_EPI_GATE_RES>() >= 3)
        return launch<BN, kResStages, AQB_EPI_GATE_RES, PAIR>(ta, tb, to, pm, p, s);
      else
        return set_error(AQB_EINVAL, "gate*residual epilogue does not fit variant BN=%d pair=%d", BN, int(PAIR));
    case AQB_EPI_F32: return launch<BN, STAGES, AQB_EPI_F32, PAIR>(ta, tb, to, pm, p, s);
    case kEpiGateAdd: return launch<BN, STAGES, kEpiGateAdd, PAIR>(ta, tb, to, pm, p, s);
    case kEpiGateAddScatter: return launch<BN, STAGES, kEpiGateAddScatter, PAIR>(ta, tb, to, pm, p, s);
    case AQB_EPI_EULER: return launch<BN, STAGES, AQB_EPI_EULER, PAIR>(ta, tb, to, pm, p, s);
    case AQB_EPI_QKNORM_ROPE: return launch<BN, qk_stages<BN, STAGES, PAIR>(), AQB_EPI_QKNORM_ROPE, PAIR>(ta, tb, to, pm, p, s);
    case kEpiQkNoRope: return launch<BN, STAGES, kEpiQkNoRope, PAIR>(ta, tb, to, pm, p, s);
  }
  return set_error(AQB_EINVAL, "unknown epilogue %d", epi);
}

// Variant choice.  Cost model: waves of tiles x per-tile time, where the
// per-tile time is max(MMA, L2->SM operand bytes); 2-CTA tiles halve the W
// bytes each SM loads.  AQB_GEMM_VARIANT=1cta256|1cta128|2cta256|2cta128
// forces one (benchmarking).
enum Variant { V1_256 = 0, V1_128, V2_256, V2_128 };

// aqb_gemm_trace: device buffer [grid][128] of pipeline stamps for the next launches (null: off)
static std::atomic<unsigned long long*> g_gemm_trace{nullptr};

// AQB_GEMM_GATE_ADD=0: gate*residual always through the residual-reading epilogue (benchmarking)
static bool gate_add_enabled() {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("AQB_GEMM_GATE_ADD");
    enabled = (e && !strcmp(e, "0")) ? 0 : 1;
  }
  return enabled == 1;
}

// Tiles of a pair-kernel launch (BN = 256) that run as two half-width units: the
// partial last wave when it fills at most half the CTA pairs (it then takes half a
// tile's time instead of a whole one).  Needs at least one whole wave: a launch of
// only half-width units streams 1.5x the operand bytes per FLOP from L2 and measured
// no faster (975x2048x8192: -8%).  AQB_GEMM_HALF_TAIL=0 disables (benchmarking).
// Measured (B200, L2 flushed): 7800x2048x2048 1162 -> 1302 TFLOP/s, x8192 1428 -> 1588,
// 7800x8192x2048 GeLU 1588 -> 1692, 7800x6144x2048 1534 -> 1585, 975x6144x2048 685 -> 825.
static int half_tail_tiles(int tiles, bool pair, int bn) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("AQB_GEMM_HALF_TAIL");
    enabled = (e && !strcmp(e, "0")) ? 0 : 1;
  }
  if (!enabled || !pair || bn != 256) return 0;
  const int pairs = sm_count() / 2;
  const int r = tiles % pairs;
  return (tiles > pairs && r > 0 && 2 * r <= pairs) ? r : 0;
}

static int pick_variant(int64_t m, int64_t n, int64_t k, bool f32_out = false) {
  static int forced = -2;
  if (forced == -2) {
    forced = -1;
    if (const char* e = getenv("AQB_GEMM_VARIANT")) {
      if (!strcmp(e, "1cta256")) forced = V1_256;
      if (!strcmp(e, "1cta128")) forced = V1_128;
      if (!strcmp(e, "2cta256")) forced = V2_256;
      if (!strcmp(e, "2cta128")) forced = V2_128;
    }
  }
  if (forced >= 0) return forced;
  const double sms = sm_count();
  struct C { int v, tm, tn, ctas; } cs[4] = {{V2_256, 256, 256, 2}, {V1_256, 128, 256, 1}, {V2_128, 256, 128, 2},
                                             {V1_128, 128, 128, 1}};
  double best = 1e30;
  int bv = V2_256;
  for (auto& c : cs) {
    const double tiles = double((m + c.tm - 1) / c.tm) * double((n + c.tn - 1) / c.tn);
    double waves = std::ceil(tiles / (sms / c.ctas));
    if (half_tail_tiles(int(tiles), c.ctas == 2, c.tn) > 0) waves -= 0.5;
    const double rows = c.tm / c.ctas;                        // A rows per SM
    const double bytes = (rows + double(c.tn) / c.ctas) * 2;  // per SM per k
    const double mma = rows * c.tn / 4096.0 * 0.5;            // cycles per SM per k
    const double l2 = bytes / 64.0;                           // ~64 B/cycle/SM sustainable from L2
    const double t = waves * std::max(mma, l2) * double(k);
    if (t < best * 0.97) best = t, bv = c.v;
  }
  // f32-output epilogues (gate*residual, reduce-scatter) on a shard small enough that the
  // 256x256 pair tiles fill at most one wave (or two with a short K): little overlaps the
  // exposed f32 epilogue, and 256x128 pair tiles (twice the CTAs, half the epilogue each)
  // measured faster: 1950x2048x2048 515 -> 592 TFLOP/s, 975x2048x8192 561 -> 821; two
  // waves, K = 2048: 3900x2048x2048 44.0 -> 39.9 us, with the bf16 residual copy 50.0 ->
  // 48.0; but K = 8192 keeps the pair tiles (3900x2048x8192 99.2 vs 113.5 us;
  // `scripts/kernel_bench.py --only gemm-variants`).
  // K = 8192 with most pairs busy keeps the pair tiles (1950x2048x8192: 52.8 vs 55.3 us in a
  // CUDA graph, `scripts/gemm_bench.py`), a quarter-filled wave does not (975 rows: 29.6 vs 47.7).
  if (f32_out && bv == V2_256) {
    const double tiles = double((m + 255) / 256) * double((n + 255) / 256);
    const bool long_k_busy = k >= 8192 && tiles > sms / 4;
    if ((tiles <= sms / 2 && !long_k_busy) || (tiles <= sms && k <= 4096)) bv = V2_128;
  }
  return bv;
}

}  // namespace gemm
}  // namespace aqb

namespace aqb {
namespace gemm {

// Shared host path: A/W tensor maps, variant choice, tile bookkeeping, launch.
static int run(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m, int64_t n, int64_t k, int epilogue,
               Params& p, const CUtensorMap& to, int variant, cudaStream_t s, const PeerMaps* pm_in = nullptr) {
  PeerMaps pm;
  if (pm_in)
    pm = *pm_in;
  else
    memset(&pm, 0, sizeof(pm));
  const bool pair = variant == V2_256 || variant == V2_128;
  const int bn = (variant == V1_256 || variant == V2_256) ? 256 : 128;
  const int tile_m = pair ? 2 * BM : BM;
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
    uint32_t box[2] = {BK, uint32_t(pair ? bn / 2 : bn)};
    int rc = make_tmap_bf16(&tb, w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  p.M = int(m), p.N = int(n), p.K = int(k);
  p.num_m = int((m + tile_m - 1) / tile_m);
  p.num_n = int((n + bn - 1) / bn);
  p.num_tiles = p.num_m * p.num_n;
  {
    // Raster: tiles walk M first inside groups of group_m M blocks.  With small groups a wave
    // covers every column tile of a few row blocks (each A row block is consumed while
    // L2-resident, all of W streams per wave); with groups of 16 it covers a few column tiles
    // of 16 row blocks (a W column slab stays resident instead).  Measured in a CUDA graph
    // (`profiles/r02_gemm_group_m.jsonl`, interleaved repeats): groups of 2 when W fits well in
    // L2 (<= 40 MB: every config-2 weight; QKV 7800x6144x2048 135.8 -> 132.4 us, FFN2
    // 7800x2048x8192 190.2 -> 184.1, out-projection 3900x2048x2048 39.1 -> 35.5), else 4 for
    // narrow outputs and 16 for wide ones (MM-DiT QKV / FFN1 with 57-75 MB of W: 16 is 5-10%
    // faster than 2-4).  AQB_GEMM_GROUP_M forces (benchmarking).
    static int gm = -1;
    if (gm < 0) {
      const char* e = getenv("AQB_GEMM_GROUP_M");
      gm = e ? std::max(1, atoi(e)) : 0;
    }
    const bool w_fits = n * k * 2 <= (int64_t(40) << 20);
    p.group_m = gm > 0 ? gm : w_fits ? 2 : (p.num_n <= 16 ? 4 : 16);
  }
  p.n_full = p.num_tiles;
  const int tail = half_tail_tiles(p.num_tiles, pair, bn);
  if (tail > 0) {  // the last `tail` tiles run as two half-width units each
    uint64_t dims[2] = {uint64_t(k), uint64_t(n)};
    uint64_t strides[1] = {uint64_t(ldw) * 2};
    uint32_t box[2] = {BK, uint32_t(bn / 4)};
    int rc = make_tmap_bf16(&pm.bh, w, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    p.n_full = p.num_tiles - tail;
  }
  p.num_units = p.n_full + 2 * (p.num_tiles - p.n_full);
  p.trace = g_gemm_trace.load();
  switch (variant) {
    case V1_256: return dispatch_epi<256, 4, false>(epilogue, ta, tb, to, pm, p, s);
    case V1_128: return dispatch_epi<128, 6, false>(epilogue, ta, tb, to, pm, p, s);
    case V2_256: return dispatch_epi<256, 6, true>(epilogue, ta, tb, to, pm, p, s);
    default: return dispatch_epi<128, 8, true>(epilogue, ta, tb, to, pm, p, s);
  }
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

  const int variant = pick_variant(m, n, k, epilogue == AQB_EPI_GATE_RES || epilogue == AQB_EPI_F32);
  CUtensorMap to;
  if (epilogue == AQB_EPI_EULER) {
    memset(&to, 0, sizeof(to));  // direct stores; map unused
  } else {
    const bool f32 = epilogue == AQB_EPI_F32 || epilogue == AQB_EPI_GATE_RES;
    const int esz = f32 ? 4 : 2;
    uint64_t dims[2] = {uint64_t(n), uint64_t(m)};
    uint64_t strides[1] = {uint64_t(ldo) * esz};
    uint32_t box[2] = {uint32_t(128 / esz), uint32_t(BM)};
    int rc = make_tmap(&to, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, 2, dims,
                       strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  Params p{};
  p.out = out, p.ldo = ldo, p.bias = bias, p.gate = gate, p.alpha = alpha;
  p.aux = reinterpret_cast<__nv_bfloat16*>(aux), p.ld_aux = ld_aux;
  p.run_flag = run_flag, p.run_if = run_if;
  if (epilogue == AQB_EPI_GATE_RES && aux != nullptr) {
    // bf16 copy of the new residual, TMA-stored beside it (64B-swizzled 32-column chunks)
    AQB_CHECK_ARG(ld_aux >= n && ld_aux % 8 == 0, "gemm: bad ld_aux");
    PeerMaps xm;
    memset(&xm, 0, sizeof(xm));
    const uint64_t dims[2] = {uint64_t(n), uint64_t(m)};
    const uint64_t strides[1] = {uint64_t(ld_aux) * 2};
    const uint32_t box[2] = {32, uint32_t(BM)};
    int rc = make_tmap(&xm.m[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, aux, 2, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
    return run(a, lda, w, ldw, m, n, k, epilogue, p, to, variant, reinterpret_cast<cudaStream_t>(stream), &xm);
  }
  if (epilogue == AQB_EPI_GATE_RES && gate_add_enabled()) epilogue = kEpiGateAdd;
  return run(a, lda, w, ldw, m, n, k, epilogue, p, to, variant, reinterpret_cast<cudaStream_t>(stream));
}

namespace aqb {
namespace gemm {

static int qknorm_rope(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m, int64_t n, int64_t k,
                       const float* bias, int32_t part_width, int32_t norm_parts, const float* q_w, const float* k_w,
                       float eps, const float* rope_cos, const float* rope_sin, int64_t rope_row0, int64_t rope_rows,
                       void* out, int64_t out_row_stride, int32_t groups, int64_t group_stride, int32_t hpg,
                       int32_t g_base, void* const* peer_out, const int32_t* run_flag, int32_t run_if,
                       cudaStream_t stream) {
  AQB_CHECK_ARG(a && w && (out || peer_out), "gemm_qknorm_rope: null pointer");
  AQB_CHECK_ARG(m >= 1 && k >= 1 && k % 8 == 0 && lda % 8 == 0 && ldw % 8 == 0, "gemm_qknorm_rope: bad shape");
  AQB_CHECK_ARG(part_width >= 128 && part_width % 128 == 0 && n % part_width == 0 && n / part_width <= 3,
                "gemm_qknorm_rope: columns must be [parts<=3][heads][128]");
  AQB_CHECK_ARG(norm_parts >= 0 && norm_parts <= 2 && norm_parts <= n / part_width, "gemm_qknorm_rope: norm_parts");
  AQB_CHECK_ARG(norm_parts < 1 || q_w, "gemm_qknorm_rope: q_w missing");
  AQB_CHECK_ARG(norm_parts < 2 || k_w, "gemm_qknorm_rope: k_w missing");
  AQB_CHECK_ARG(rope_rows <= 0 || (rope_cos && rope_sin), "gemm_qknorm_rope: rope tables missing");
  AQB_CHECK_ARG(hpg >= 1 && groups >= 1 && out_row_stride % 8 == 0 && group_stride % 8 == 0,
                "gemm_qknorm_rope: bad output layout");
  const int parts = int(n / part_width);
  // (d:128, head-in-group:hpg, part, row:m, group) ; strides in bytes
  const uint64_t strides[4] = {256, uint64_t(hpg) * 256, uint64_t(out_row_stride) * 2, uint64_t(group_stride) * 2};
  const uint32_t box[5] = {64, 1, 1, uint32_t(BM), 1};
  CUtensorMap to;
  PeerMaps pm;
  memset(&pm, 0, sizeof(pm));
  if (peer_out == nullptr) {
    const uint64_t dims[5] = {128, uint64_t(hpg), uint64_t(parts), uint64_t(m), uint64_t(groups)};
    int rc = make_tmap(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  } else {
    AQB_CHECK_ARG(groups <= kMaxPeers && g_base == 0, "gemm_qknorm_rope_scatter: 1..%d ranks", kMaxPeers);
    const uint64_t dims[5] = {128, uint64_t(hpg), uint64_t(parts), uint64_t(m), 1};
    for (int g = 0; g < groups; ++g) {
      AQB_CHECK_ARG(peer_out[g] != nullptr, "gemm_qknorm_rope_scatter: peer_out[%d] is null", g);
      int rc = make_tmap(&pm.m[g], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, peer_out[g], 5, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
    }
    to = pm.m[0];
  }
  Params p{};
  p.out = out, p.ldo = out_row_stride, p.bias = bias;
  p.run_flag = run_flag, p.run_if = run_if;
  p.norm_w0 = q_w, p.norm_w1 = k_w, p.rope_cos = rope_cos, p.rope_sin = rope_sin;
  p.rope_row0 = rope_row0, p.rope_rows = rope_rows, p.part_width = part_width, p.norm_parts = norm_parts;
  p.hpg = hpg, p.g_base = g_base, p.groups = groups, p.eps = eps;
  p.peer_groups = peer_out != nullptr;
  if (rope_rows > 0) {  // cos / sin tables for the pair kernel's TMA-staged RoPE
    AQB_CHECK_ARG(reinterpret_cast<uintptr_t>(rope_cos) % 16 == 0 && reinterpret_cast<uintptr_t>(rope_sin) % 16 == 0,
                  "gemm_qknorm_rope: rope tables must be 16B aligned");
    const uint64_t dims[2] = {64, uint64_t(rope_rows)};
    const uint64_t strides[1] = {256};
    const uint32_t box[2] = {32, uint32_t(BM)};
    int rc = make_tmap(&pm.rcos, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rope_cos, 2, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_tmap(&pm.rsin, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rope_sin, 2, dims, strides, box,
                   CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  // QK-norm without RoPE (cross-attention q) on a shard whose 256x256 pair tiles fill at most one
  // wave: 128x128 single-CTA tiles overlap each tile's epilogue with the next tile's MMAs and
  // measured fastest (1950x2048x2048: 17.6 vs 19.9 us, 975 rows: 11.0 vs 12.1; CUDA graph,
  // `scripts/gemm_bench.py`)
  int variant = pick_variant(m, n, k);
  if (rope_rows == 0 && !getenv("AQB_GEMM_VARIANT") &&
      double((m + 255) / 256) * double((n + 255) / 256) <= sm_count() / 2)
    variant = V1_128;
  return run(a, lda, w, ldw, m, n, k, rope_rows > 0 ? AQB_EPI_QKNORM_ROPE : kEpiQkNoRope, p, to, variant, stream,
             &pm);
}

}  // namespace gemm
}  // namespace aqb

extern "C" int aqb_gemm_qknorm_rope(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m, int64_t n,
                                    int64_t k, const float* bias, int32_t part_width, int32_t norm_parts,
                                    const float* q_w, const float* k_w, float eps, const float* rope_cos,
                                    const float* rope_sin, int64_t rope_row0, int64_t rope_rows, void* out,
                                    int64_t out_row_stride, int32_t groups, int64_t group_stride, int32_t hpg,
                                    int32_t g_base, const int32_t* run_flag, int32_t run_if, void* stream) {
  return aqb::gemm::qknorm_rope(a, lda, w, ldw, m, n, k, bias, part_width, norm_parts, q_w, k_w, eps, rope_cos,
                                rope_sin, rope_row0, rope_rows, out, out_row_stride, groups, group_stride, hpg, g_base,
                                nullptr, run_flag, run_if, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int aqb_gemm_qknorm_rope_scatter(const void* a, int64_t lda, const void* w, int64_t ldw, int64_t m,
                                            int64_t n, int64_t k, const float* bias, int32_t part_width,
                                            int32_t norm_parts, const float* q_w, const float* k_w, float eps,
                                            const float* rope_cos, const float* rope_sin, int64_t rope_row0,
                                            int64_t rope_rows, void* const* peer_out, int32_t nranks,
                                            int64_t out_row_stride, int32_t hpg, const int32_t* run_flag,
                                            int32_t run_if, void* stream) {
  AQB_CHECK_ARG(peer_out != nullptr && nranks >= 1, "gemm_qknorm_rope_scatter: peer_out");
  return aqb::gemm::qknorm_rope(a, lda, w, ldw, m, n, k, bias, part_width, norm_parts, q_w, k_w, eps, rope_cos,
                                rope_sin, rope_row0, rope_rows, nullptr, out_row_stride, nranks, 0, hpg, 0, peer_out,
                                run_flag, run_if, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int aqb_gemm_gate_add_scatter(const void* a, int64_t lda, const void* w, int64_t ldw, float* const* peer_out,
                                         int32_t nranks, int64_t ldo, int64_t rows_per_rank, int64_t m, int64_t n,
                                         int64_t k, const float* bias, const float* gate, const int32_t* run_flag,
                                         int32_t run_if, void* stream) {
  using namespace aqb;
  using namespace aqb::gemm;
  AQB_CHECK_ARG(a && w && peer_out, "gemm_gate_add_scatter: null pointer");
  AQB_CHECK_ARG(nranks >= 1 && nranks <= kMaxPeers, "gemm_gate_add_scatter: 1..%d ranks", kMaxPeers);
  AQB_CHECK_ARG(m >= 1 && n >= 1 && k >= 1 && k % 8 == 0 && n % 16 == 0, "gemm_gate_add_scatter: bad shape");
  AQB_CHECK_ARG(lda % 8 == 0 && ldw % 8 == 0 && lda >= k && ldw >= k, "gemm_gate_add_scatter: bad lda/ldw");
  AQB_CHECK_ARG(ldo >= n && ldo % 4 == 0, "gemm_gate_add_scatter: bad ldo");
  AQB_CHECK_ARG(rows_per_rank >= 1 && rows_per_rank * nranks == m, "gemm_gate_add_scatter: m != nranks * rows_per_rank");
  Params p{};
  p.out = peer_out[0], p.ldo = ldo, p.bias = bias, p.gate = gate;
  p.run_flag = run_flag, p.run_if = run_if;
  p.red_rpr = rows_per_rank;
  PeerMaps pm;
  memset(&pm, 0, sizeof(pm));
  for (int r = 0; r < nranks; ++r) {
    AQB_CHECK_ARG(peer_out[r] && reinterpret_cast<uintptr_t>(peer_out[r]) % 16 == 0,
                  "gemm_gate_add_scatter: peer_out[%d] null/misaligned", r);
    p.red_dst[r] = peer_out[r];
    const uint64_t dims[2] = {uint64_t(n), uint64_t(rows_per_rank)};
    const uint64_t strides[1] = {uint64_t(ldo) * 4};
    const uint32_t box[2] = {32, uint32_t(BM)};
    int rc = make_tmap(&pm.m[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, peer_out[r], 2, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  return run(a, lda, w, ldw, m, n, k, kEpiGateAddScatter, p, pm.m[0], pick_variant(m, n, k, true),
             reinterpret_cast<cudaStream_t>(stream), &pm);
}

extern "C" int aqb_gemm_trace(void* buffer) {
#ifdef AQB_GEMM_TRACE
  aqb::gemm::g_gemm_trace.store(reinterpret_cast<unsigned long long*>(buffer));
  return AQB_OK;
#else
  if (buffer == nullptr) return AQB_OK;
  return aqb::set_error(AQB_EINVAL, "aqb_gemm_trace: library built without -DAQB_GEMM_TRACE");
#endif
}
