// HBM-bound kernels of the DiT block (sm_100a): AdaLN norm+modulate (with the
// diffusion-cache rel-L1 probe fused in), QK-RMSNorm + 3D RoPE (+ Ulysses
// pack), AdaLN/timestep GEMV, cache-offset and device-side cache decision,
// latent (un)patchify and the Ulysses head->sequence repack.
//
// Design rules (blackwell guide G2/G7/G13): thread->contiguous element,
// 16-byte vector loads/stores, warp-shuffle reductions, one warp per row
// so the whole row lives in registers (single HBM read), fp32 statistics.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "host.cuh"
#include "ptx.cuh"

namespace aqb {

AQB_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

AQB_DEV float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------ norm+modulate
// One warp per row; NV float4 per lane (hidden = 128 * NV).
AQB_DEV void store4(__nv_bfloat16* p, float4 o) {
  *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(o.x, o.y), pack_bf16(o.z, o.w));
}
AQB_DEV void store4(float* p, float4 o) { *reinterpret_cast<float4*>(p) = o; }
AQB_DEV float2 load2(const __nv_bfloat16* p) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p)); }
AQB_DEV float2 load2(const float* p) { return *reinterpret_cast<const float2*>(p); }
AQB_DEV void store2(__nv_bfloat16* p, float2 v) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v.x, v.y);
}
AQB_DEV void store2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

// Output rows go to up to 8 destinations (same row index and stride in each): one
// for the plain kernel; every rank's gathered buffer for the TP-SP all-gather
// (aqb_norm_modulate_gather: the rows this rank normalised are stored straight into
// each peer's copy over NVLink, so no separate all-gather runs).
constexpr int kMaxOuts = 8;
template <typename OutT>
struct Outs {
  OutT* p[kMaxOuts];
  int n;
};

// y = LN(x) * (1 + scale) + shift as t = x*rstd - mean*rstd, y = t*scale + (t + shift):
// 3 FP ops per element (the SASS of the plain form spent a third of its issue slots on
// the per-row 1 + scale)
AQB_DEV float4 modulate4(float4 x, float rstd, float nmr, float4 sc, float4 sh) {
  float4 o;
  float t;
  t = fmaf(x.x, rstd, nmr), o.x = fmaf(t, sc.x, t + sh.x);
  t = fmaf(x.y, rstd, nmr), o.y = fmaf(t, sc.y, t + sh.y);
  t = fmaf(x.z, rstd, nmr), o.z = fmaf(t, sc.z, t + sh.z);
  t = fmaf(x.w, rstd, nmr), o.w = fmaf(t, sc.w, t + sh.w);
  return o;
}

// one destination: the pointer stays in the parameter space (a dynamic index into
// Outs::p put it in local memory: an LDL per store)
template <typename OutT>
AQB_DEV void store_outs(const Outs<OutT>& ys, int64_t off, float4 o) {
  if (ys.n == 1) {
    store4(ys.p[0] + off, o);
    return;
  }
#pragma unroll 1
  for (int d = 0; d < ys.n; ++d) store4(ys.p[d] + off, o);
}

// OutT = bf16 (product path) or float (fp32 validation mode).
template <int NV, typename OutT>
__global__ void __launch_bounds__(256) norm_mod_kernel(const float* __restrict__ x, int64_t ldx,
                                                       const float* __restrict__ shift,
                                                       const float* __restrict__ scale, const Outs<OutT> ys,
                                                       int64_t ldy, int64_t rows, float eps, int kind,
                                                       float* __restrict__ prev, float* __restrict__ partials,
                                                       const int32_t* flag, int32_t run_if) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  constexpr int H = NV * 128;
  const float4* xr = reinterpret_cast<const float4*>(x + row * ldx);
  float4 v[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = ld_stream(xr + lane + 32 * j);
  float mean = 0.f;
  if (kind == 0) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    mean = warp_sum(s) * (1.f / H);
  }
  float rstd = 1.f;
  if (kind != 2) {
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const float a = v[j].x - mean, b = v[j].y - mean, c = v[j].z - mean, d = v[j].w - mean;
      ss += (a * a + b * b) + (c * c + d * d);
    }
    rstd = rsqrtf(warp_sum(ss) * (1.f / H) + eps);
  }
  const float4* sh4 = reinterpret_cast<const float4*>(shift);
  const float4* sc4 = reinterpret_cast<const float4*>(scale);
  const float nmr = -mean * rstd;
  const int64_t yoff = row * ldy;
  float4* pr = prev ? reinterpret_cast<float4*>(prev + row * H) : nullptr;
  float dsum = 0.f, psum = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c4 = lane + 32 * j;
    const float4 sc = scale ? __ldg(sc4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 sh = shift ? __ldg(sh4 + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 o = modulate4(v[j], rstd, nmr, sc, sh);
    store_outs(ys, yoff + 4 * c4, o);
    if (pr) {
      const float4 p = pr[c4];
      dsum += (fabsf(o.x - p.x) + fabsf(o.y - p.y)) + (fabsf(o.z - p.z) + fabsf(o.w - p.w));
      psum += (fabsf(p.x) + fabsf(p.y)) + (fabsf(p.z) + fabsf(p.w));
      pr[c4] = o;
    }
  }
  if (pr) {
    dsum = warp_sum(dsum);
    psum = warp_sum(psum);
    if (lane == 0) {
      partials[row] = dsum;
      partials[rows + row] = psum;
    }
  }
}

// CTA per row for wide rows (hidden >= 1024): hidden/16 threads, 4 float4 each,
// so a few thousand rows (one Ulysses shard) still fill the SMs with enough
// loads in flight; block reductions through shared memory.
template <int NW>
AQB_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red[] reuse across calls
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}

template <int NW, int VPT, typename OutT>
__global__ void __launch_bounds__(NW * 32) norm_mod_row_kernel(const float* __restrict__ x, int64_t ldx,
                                                               const float* __restrict__ shift,
                                                               const float* __restrict__ scale, const Outs<OutT> ys,
                                                               int64_t ldy, int64_t rows, float eps, int kind,
                                                               float* __restrict__ prev, float* __restrict__ partials,
                                                               const int32_t* flag, int32_t run_if) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  __shared__ float red[NW];
  constexpr int T = NW * 32, H = T * 4 * VPT;
  const int tid = threadIdx.x;
  // persistent over rows (grid-stride) with the next row's loads issued before this row's
  // reductions, so each CTA keeps two rows in flight
  float4 v[VPT], vn[VPT];
  // this thread's columns are the same for every row: scale/shift stay in registers
  float4 sc[VPT], sh[VPT];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    sc[j] = scale ? __ldg(reinterpret_cast<const float4*>(scale) + tid + T * j) : make_float4(0.f, 0.f, 0.f, 0.f);
    sh[j] = shift ? __ldg(reinterpret_cast<const float4*>(shift) + tid + T * j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  int64_t row = blockIdx.x;
  if (row < rows) {
    const float4* xr = reinterpret_cast<const float4*>(x + row * ldx);
#pragma unroll
    for (int j = 0; j < VPT; ++j) v[j] = ld_stream(xr + tid + T * j);
  }
  for (; row < rows; row += gridDim.x) {
  if (row + gridDim.x < rows) {
    const float4* xn = reinterpret_cast<const float4*>(x + (row + gridDim.x) * ldx);
#pragma unroll
    for (int j = 0; j < VPT; ++j) vn[j] = ld_stream(xn + tid + T * j);
  }
  float mean = 0.f;
  float rstd = 1.f;
  if (kind == 0) {
    // mean and variance in ONE block round: per-thread (mean, M2) over its 16 values,
    // merged pairwise (Chan et al., equal counts) through the warp and then the NW warps
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) m += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    m *= 1.f / (4 * VPT);
    float m2 = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const float a = v[j].x - m, b = v[j].y - m, c = v[j].z - m, d = v[j].w - m;
      m2 += (a * a + b * b) + (c * c + d * d);
    }
    float n = 4.f * VPT;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, m, o), m2o = __shfl_xor_sync(0xffffffffu, m2, o);
      const float d = mo - m;
      m2 = m2 + m2o + d * d * (0.5f * n);
      m = 0.5f * (m + mo);
      n *= 2.f;
    }
    __shared__ float2 wstat[NW];
    if ((tid & 31) == 0) wstat[tid >> 5] = make_float2(m, m2);
    __syncthreads();
    constexpr float kW = 128.f * VPT;  // values per warp
    float bm = wstat[0].x, bm2 = wstat[0].y, bn = kW;
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const float d = wstat[w].x - bm, nn = bn + kW;
      bm += d * (kW / nn);
      bm2 += wstat[w].y + d * d * (bn * kW / nn);
      bn = nn;
    }
    mean = bm;
    rstd = rsqrtf(bm2 * (1.f / H) + eps);
  } else if (kind == 1) {
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const float a = v[j].x - mean, b = v[j].y - mean, c = v[j].z - mean, d = v[j].w - mean;
      ss += (a * a + b * b) + (c * c + d * d);
    }
    rstd = rsqrtf(block_sum<NW>(ss, red) * (1.f / H) + eps);
  }
  const float nmr = -mean * rstd;
  const int64_t yoff = row * ldy;
  float4* pr = prev ? reinterpret_cast<float4*>(prev + row * H) : nullptr;
  float dsum = 0.f, psum = 0.f;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c4 = tid + T * j;
    const float4 o = modulate4(v[j], rstd, nmr, sc[j], sh[j]);
    store_outs(ys, yoff + 4 * c4, o);
    if (pr) {
      const float4 p = pr[c4];
      dsum += (fabsf(o.x - p.x) + fabsf(o.y - p.y)) + (fabsf(o.z - p.z) + fabsf(o.w - p.w));
      psum += (fabsf(p.x) + fabsf(p.y)) + (fabsf(p.z) + fabsf(p.w));
      pr[c4] = o;
    }
  }
  if (pr) {
    dsum = block_sum<NW>(dsum, red);
    psum = block_sum<NW>(psum, red);
    if (tid == 0) {
      partials[row] = dsum;
      partials[rows + row] = psum;
    }
  }
  __syncthreads();  // wstat / red reused by the next row
#pragma unroll
  for (int j = 0; j < VPT; ++j) v[j] = vn[j];
  }
}

// ------------------------------------------------------- QK-norm + 3D RoPE
// One warp per (row, head); lane handles pairs lane, lane+32, ... (D/2 pairs).
template <int D, typename T>
__global__ void __launch_bounds__(256) qk_norm_rope_kernel(
    const T* __restrict__ src, int64_t ld_src, int64_t rows, int heads, int head_begin, int head_count,
    const float* __restrict__ qw, const float* __restrict__ kw, float eps, const float* __restrict__ rcos,
    const float* __restrict__ rsin, int64_t rope_row0, int64_t rope_rows, T* dst, int64_t g_stride,
    int64_t r_stride, int64_t w_stride, int hpg, int parts, int norm_parts, const int32_t* flag, int32_t run_if) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  constexpr int NP = (D / 2 + 31) / 32;  // pairs per lane
  const int lane = threadIdx.x & 31;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (item >= rows * head_count) return;
  const int64_t r = item / head_count;
  const int j = static_cast<int>(item - r * head_count);
  const int h = head_begin + j;
  const T* s = src + r * ld_src;
  T* d = dst + static_cast<int64_t>(j / hpg) * g_stride + r * r_stride + static_cast<int64_t>(j % hpg) * D;
  const int64_t grow = rope_row0 + r;
  const bool rope = grow < rope_rows;
#pragma unroll 1
  for (int which = 0; which < parts; ++which) {
    const T* sp = s + static_cast<int64_t>(which) * heads * D + static_cast<int64_t>(h) * D;
    float2 e[NP];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const int p = lane + 32 * i;
      e[i] = (p < D / 2) ? load2(sp + 2 * p) : make_float2(0.f, 0.f);
      ss += e[i].x * e[i].x + e[i].y * e[i].y;
    }
    if (which < norm_parts) {
      const float rstd = rsqrtf(warp_sum(ss) * (1.f / D) + eps);
      const float* w = which == 0 ? qw : kw;
#pragma unroll
      for (int i = 0; i < NP; ++i) {
        const int p = lane + 32 * i;
        if (p < D / 2) {
          const float2 wv = __ldg(reinterpret_cast<const float2*>(w) + p);
          float a = e[i].x * rstd * wv.x, b = e[i].y * rstd * wv.y;
          if (rope) {
            const float c = __ldg(rcos + grow * (D / 2) + p), sn = __ldg(rsin + grow * (D / 2) + p);
            const float a2 = a * c - b * sn;
            b = a * sn + b * c;
            a = a2;
          }
          e[i] = make_float2(a, b);
        }
      }
    }
    T* dp = d + static_cast<int64_t>(which) * w_stride;
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const int p = lane + 32 * i;
      if (p < D / 2) store2(dp + 2 * p, e[i]);
    }
  }
}

// ---------------------------------------------------------------- GEMV
// y[n] = W[n,:] . in(x) + b[n] + add[n];  x staged in smem (SiLU or timestep features).
__global__ void __launch_bounds__(256) gemv_kernel(const __nv_bfloat16* __restrict__ W, const float* __restrict__ x,
                                                   const float* __restrict__ t, const float* __restrict__ b,
                                                   const float* __restrict__ add, float* __restrict__ y, int64_t n,
                                                   int k, int in_silu) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  extern __shared__ float xs[];
  const float tv = t ? __ldg(t) : 0.f;
  const int half = k / 2;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    float v;
    if (x) {
      v = x[i];
    } else {
      const int fi = i < half ? i : i - half;
      const float f = expf(-9.210340371976184f * fi / half);  // ln(10000)
      const float a = 1000.f * tv * f;
      v = i < half ? cosf(a) : sinf(a);
    }
    if (in_silu) v = v / (1.f + __expf(-v));
    xs[i] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nvec = k / 8;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); row < n;
       row += static_cast<int64_t>(gridDim.x) * 8) {
    const uint4* wr = reinterpret_cast<const uint4*>(W + row * k);
    float acc = 0.f;
    for (int v = lane; v < nvec; v += 32) {
      const uint4 w8 = __ldg(wr + v);
      const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&w8);
      const float* xv = xs + 8 * v;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(w2[q]);
        acc += f.x * xv[2 * q] + f.y * xv[2 * q + 1];
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc + (b ? b[row] : 0.f) + (add ? add[row] : 0.f);
  }
}

__global__ void add_bcast_kernel(float* out, const float* a, int64_t period, const float* b, int64_t n) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = a[i % period] + b[i];
}

// ------------------------------------------------------- TP-SP replicated rows
// The text rows of an MM-DiT under TP-SP are replicated on every rank, so their
// row-parallel projections need an all-reduce.  Deterministically: every rank writes
// gate * partial into slot `rank` of every rank's slot buffer (peer stores), then after
// the barrier each rank adds its P slots in rank order (identical bits everywhere).
struct SlotDsts {
  float* p[8];
  int n;
};

__global__ void gate_bcast_kernel(const float* __restrict__ src, int64_t lds, const float* __restrict__ gate,
                                  SlotDsts dst, int64_t ldd, int64_t rows, int cols4, const int32_t* flag,
                                  int32_t run_if) {
  pdl_wait();
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  const int64_t total = rows * cols4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols4;
    const int c = int(i % cols4);
    float4 v = *reinterpret_cast<const float4*>(src + r * lds + 4 * c);
    if (gate) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(gate) + c);
      v.x *= g.x, v.y *= g.y, v.z *= g.z, v.w *= g.w;
    }
#pragma unroll 1
    for (int d = 0; d < dst.n; ++d) *reinterpret_cast<float4*>(dst.p[d] + r * ldd + 4 * c) = v;
  }
}

__global__ void sum_slots_kernel(float* __restrict__ x, int64_t ldx, const float* __restrict__ slots, int nslots,
                                 int64_t slot_stride, int64_t lds, int64_t rows, int cols4, const int32_t* flag,
                                 int32_t run_if) {
  pdl_wait();
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  const int64_t total = rows * cols4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols4;
    const int c = int(i % cols4);
    float4 a = *reinterpret_cast<const float4*>(x + r * ldx + 4 * c);
    for (int k = 0; k < nslots; ++k) {  // rank order
      const float4 b = *reinterpret_cast<const float4*>(slots + k * slot_stride + r * lds + 4 * c);
      a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    }
    *reinterpret_cast<float4*>(x + r * ldx + 4 * c) = a;
  }
}

// ------------------------------------------------------- diffusion cache
__global__ void __launch_bounds__(1024) rel_l1_reduce_kernel(const float* partials, int64_t rows, float* sums) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  __shared__ float sd[32], sp[32];
  float d = 0.f, p = 0.f;
  for (int64_t i = threadIdx.x; i < rows; i += 1024) {
    d += partials[i];
    p += partials[rows + i];
  }
  d = warp_sum(d);
  p = warp_sum(p);
  if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = d, sp[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x < 32) {
    d = warp_sum(sd[threadIdx.x]);
    p = warp_sum(sp[threadIdx.x]);
    if (threadIdx.x == 0) sums[0] = d, sums[1] = p;
  }
}

__global__ void cache_decide_kernel(const float* sums, int32_t* state, float thr, int warmup, int total,
                                    int force_last, int32_t* flags_out, float* rel_out) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  const int s = state[0] + 1;
  float* accp = reinterpret_cast<float*>(state + 2);
  float acc = *accp;
  const float rel = sums[1] > 0.f ? sums[0] / sums[1] : 0.f;
  int full;
  if (s <= (warmup > 1 ? warmup : 1) || (force_last && s == total)) {
    full = 1;
    acc = 0.f;
  } else {
    acc += rel;
    if (acc >= thr) {
      full = 1;
      acc = 0.f;
    } else {
      full = 0;
    }
  }
  state[0] = s;
  state[1] = full;
  *accp = acc;
  if (flags_out && s - 1 < total) flags_out[s - 1] = full;
  if (rel_out && s - 1 < total) rel_out[s - 1] = rel;
}

__global__ void cache_offset_kernel(float* x, int64_t ldx, float* off, int64_t rows, int hidden, int mode,
                                    const int32_t* flag, int32_t run_if) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  const int64_t n4 = rows * (hidden / 4);
  const int h4 = hidden / 4;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h4, c = i - r * h4;
    float4* xp = reinterpret_cast<float4*>(x + r * ldx) + c;
    float4* op = reinterpret_cast<float4*>(off + r * hidden) + c;
    if (mode == 0) {
      *op = *xp;
    } else if (mode == 1) {
      const float4 a = *xp, b = *op;
      *op = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
    } else {
      const float4 a = *xp, b = *op;
      *xp = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
  }
}

__global__ void step_scalars_kernel(const float* ts, const float* dts, int32_t* idx, float* cur, int mode) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  const int i = *idx;
  cur[0] = ts[i];
  cur[1] = dts[i];
  if (mode == 1) *idx = i + 1;
}

// ----------------------------------------------------------- latent layout
// lat is [C, Tl, H*ph, W*pw]; the T*pt frames starting at frame t0 are (un)patchified
// (a temporal window of a longer latent: MultiDiffusion clips).
__global__ void patchify_kernel(const float* lat, float* tok, __nv_bfloat16* tokb, int C, int T, int H, int W, int pt,
                                int ph, int pw, int Tl, int t0) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  const int F = pt * ph * pw * C;
  const int64_t n = static_cast<int64_t>(T) * H * W * F;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = i / F;
    int f = static_cast<int>(i - s * F);
    const int c = f % C;
    f /= C;
    const int iw = f % pw;
    f /= pw;
    const int ih = f % ph;
    const int it = f / ph;
    const int w = static_cast<int>(s % W), h = static_cast<int>((s / W) % H), t = static_cast<int>(s / (W * H));
    const float v = lat[((static_cast<int64_t>(c) * Tl + t0 + t * pt + it) * H * ph + h * ph + ih) * W * pw + w * pw + iw];
    tok[i] = v;
    if (tokb) tokb[i] = __float2bfloat16(v);
  }
}

__global__ void unpatchify_kernel(const float* tok, float* lat, int C, int T, int H, int W, int pt, int ph, int pw,
                                  int Tl, int t0) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  const int F = pt * ph * pw * C;
  const int64_t n = static_cast<int64_t>(T) * H * W * F;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = i / F;
    int f = static_cast<int>(i - s * F);
    const int c = f % C;
    f /= C;
    const int iw = f % pw;
    f /= pw;
    const int ih = f % ph;
    const int it = f / ph;
    const int w = static_cast<int>(s % W), h = static_cast<int>((s / W) % H), t = static_cast<int>(s / (W * H));
    lat[((static_cast<int64_t>(c) * Tl + t0 + t * pt + it) * H * ph + h * ph + ih) * W * pw + w * pw + iw] = tok[i];
  }
}

// src [P, rows, width] -> dst [rows, P*width] (16-byte units)
__global__ void heads_to_seq_kernel(const uint4* src, int64_t rows, int P, int w16, uint4* dst, int64_t ld16,
                                    const int32_t* flag, int32_t run_if) {
  pdl_wait();  // PDL: predecessor's writes visible from here
  pdl_trigger();
  if (!gate_open(flag, run_if)) return;
  const int64_t n = rows * P * w16;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / (P * w16);
    const int rem = static_cast<int>(i - r * P * w16);
    const int p = rem / w16, c = rem - p * w16;
    dst[r * ld16 + rem] = src[(static_cast<int64_t>(p) * rows + r) * w16 + c];
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 32;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace aqb

using namespace aqb;

template <typename OutT>
static int norm_modulate(const float* x, int64_t ldx, const float* shift, const float* scale, void* const* y,
                         int32_t ny, int64_t ldy, int64_t rows, int32_t hidden, float eps, int32_t norm_kind,
                         float* probe_prev, float* probe_partials, const int32_t* run_flag, int32_t run_if,
                         void* stream) {
  AQB_CHECK_ARG(x && y && ny >= 1 && ny <= kMaxOuts, "norm_modulate: null pointer or 1..%d outputs", kMaxOuts);
  Outs<OutT> yb{};
  yb.n = ny;
  for (int d = 0; d < ny; ++d) {
    AQB_CHECK_ARG(y[d] && reinterpret_cast<uintptr_t>(y[d]) % 16 == 0, "norm_modulate: output %d null/misaligned", d);
    yb.p[d] = reinterpret_cast<OutT*>(y[d]);
  }
  AQB_CHECK_ARG(hidden % 128 == 0 && hidden >= 128 && hidden <= 4096, "norm_modulate: hidden %d unsupported", hidden);
  AQB_CHECK_ARG(ldx % 4 == 0 && ldy % 4 == 0 && ldx >= hidden && ldy >= hidden, "norm_modulate: bad strides");
  AQB_CHECK_ARG(!probe_prev || probe_partials, "norm_modulate: probe needs partials");
  AQB_CHECK_ARG(norm_kind >= 0 && norm_kind <= 2, "norm_modulate: bad kind");
  if (rows <= 0) return AQB_OK;
  const int grid = static_cast<int>((rows + 7) / 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // CTA per row for wide rows: NW warps x VPT float4 per thread.  Measured (B200, L2
  // flushed): hidden 2048 VPT 4 (4 warps) 3.34 TB/s vs 2.60 / 2.92 for VPT 2 / 8;
  // hidden 3072 VPT 8 (3 warps) 4.69 TB/s vs 4.12 for VPT 4.  AQB_NORM_VPT = 2|4|8 forces.
  static int vpt_env = -1;
  if (vpt_env < 0) {
    const char* e = getenv("AQB_NORM_VPT");
    vpt_env = e ? atoi(e) : 0;
    if (vpt_env != 2 && vpt_env != 4 && vpt_env != 8) vpt_env = 0;
  }
  const int vpt = vpt_env ? vpt_env : (hidden >= 3072 && hidden % 1024 == 0 ? 8 : 4);
  if (hidden >= 1024 && hidden % (128 * vpt) == 0 && hidden / (128 * vpt) >= 2 && hidden / (128 * vpt) <= 16) {
    const int nw = hidden / (128 * vpt);
    // persistent CTAs per SM (AQB_NORM_CTAS_PER_SM overrides).  Measured: hidden 2048
    // (VPT 4) 8 per SM 3.74 TB/s vs 3.34 with a CTA per row; hidden 3072 (VPT 8) 4 per SM.
    static int cps_env = -1;
    if (cps_env < 0) {
      const char* e = getenv("AQB_NORM_CTAS_PER_SM");
      cps_env = e ? atoi(e) : 0;
      if (cps_env < 0) cps_env = 0;
    }
    // r02, measured with PDL off in a CUDA graph (`scripts/norm_bench.py`): 16 warps per SM beat
    // 32 at hidden 2048 (975 rows 6.0 -> 4.8 us, 1,950 rows 7.6 -> 6.8, 7,800 rows equal) while
    // hidden 1024 (2-warp CTAs) keeps 8 CTAs per SM (11.3 vs 14.3 us at 8,056 rows)
    const int cps = cps_env ? cps_env : (vpt == 8 ? 4 : std::max(4, 16 / nw));
    const int64_t row_grid = int64_t(sm_count()) * cps;
#define NMR_LAUNCH(NW, VPT)                                                                                      \
  AQB_CUDA_TRY(launch_pdl(norm_mod_row_kernel<NW, VPT, OutT>, dim3(unsigned(std::min<int64_t>(rows, row_grid))),    \
                          dim3(NW * 32), 0, s, x, ldx,                                                           \
                          shift, scale, yb, ldy, rows, eps, norm_kind, probe_prev, probe_partials, run_flag,     \
                          run_if));                                                                              \
  AQB_LAUNCH_CHECK();                                                                                            \
  return AQB_OK;
#define NMR_CASE(NW, VPT) \
  case NW:                \
    NMR_LAUNCH(NW, VPT)
    if (vpt == 4) {
      switch (nw) { NMR_CASE(2, 4) NMR_CASE(3, 4) NMR_CASE(4, 4) NMR_CASE(5, 4) NMR_CASE(6, 4) NMR_CASE(7, 4) NMR_CASE(8, 4) default: break; }
    } else if (vpt == 2) {
      switch (nw) { NMR_CASE(4, 2) NMR_CASE(6, 2) NMR_CASE(8, 2) NMR_CASE(12, 2) NMR_CASE(16, 2) default: break; }
    } else {
      switch (nw) { NMR_CASE(2, 8) NMR_CASE(3, 8) NMR_CASE(4, 8) default: break; }
    }
#undef NMR_CASE
#undef NMR_LAUNCH
  }
#define NM_CASE(NV)                                                                                          \
  case NV:                                                                                                   \
    AQB_CUDA_TRY(launch_pdl(norm_mod_kernel<NV, OutT>, dim3(grid), dim3(256), 0, s, x, ldx, shift, scale, yb, ldy, rows, eps, norm_kind,      \
                                                   probe_prev, probe_partials, run_flag, run_if));            \
    break;
  switch (hidden / 128) {
    NM_CASE(1) NM_CASE(2) NM_CASE(3) NM_CASE(4) NM_CASE(6) NM_CASE(8) NM_CASE(12) NM_CASE(16) NM_CASE(20)
    NM_CASE(24) NM_CASE(32)
    default:
      return set_error(AQB_EUNSUPPORTED, "norm_modulate: hidden %d not instantiated", hidden);
  }
#undef NM_CASE
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_norm_modulate(const float* x, int64_t ldx, const float* shift, const float* scale, void* y,
                                 int64_t ldy, int64_t rows, int32_t hidden, float eps, int32_t norm_kind,
                                 float* probe_prev, float* probe_partials, const int32_t* run_flag, int32_t run_if,
                                 void* stream) {
  void* ys[1] = {y};
  return norm_modulate<__nv_bfloat16>(x, ldx, shift, scale, ys, 1, ldy, rows, hidden, eps, norm_kind, probe_prev,
                                      probe_partials, run_flag, run_if, stream);
}

extern "C" int aqb_norm_modulate_gather(const float* x, int64_t ldx, const float* shift, const float* scale,
                                        void* const* y, int32_t ny, int64_t ldy, int64_t rows, int32_t hidden,
                                        float eps, int32_t norm_kind, float* probe_prev, float* probe_partials,
                                        const int32_t* run_flag, int32_t run_if, void* stream) {
  return norm_modulate<__nv_bfloat16>(x, ldx, shift, scale, y, ny, ldy, rows, hidden, eps, norm_kind, probe_prev,
                                      probe_partials, run_flag, run_if, stream);
}

extern "C" int aqb_norm_modulate_f32(const float* x, int64_t ldx, const float* shift, const float* scale, float* y,
                                     int64_t ldy, int64_t rows, int32_t hidden, float eps, int32_t norm_kind,
                                     float* probe_prev, float* probe_partials, const int32_t* run_flag,
                                     int32_t run_if, void* stream) {
  void* ys[1] = {y};
  return norm_modulate<float>(x, ldx, shift, scale, ys, 1, ldy, rows, hidden, eps, norm_kind, probe_prev,
                              probe_partials, run_flag, run_if, stream);
}

template <typename T>
static int qk_norm_rope(const void* src, int64_t ld_src, int64_t rows, int32_t heads, int32_t head_begin,
                        int32_t head_count, int32_t head_dim, const float* q_w, const float* k_w, float eps,
                        const float* rope_cos, const float* rope_sin, int64_t rope_row0, int64_t rope_rows, void* dst,
                        int64_t dst_group_stride, int64_t dst_row_stride, int64_t dst_which_stride, int32_t hpg,
                        int32_t parts, int32_t norm_parts, const int32_t* run_flag, int32_t run_if, void* stream) {
  AQB_CHECK_ARG(src && dst, "qk_norm_rope: null pointer");
  AQB_CHECK_ARG(parts >= 1 && parts <= 3 && norm_parts >= 0 && norm_parts <= parts && norm_parts <= 2,
                "qk_norm_rope: bad parts");
  AQB_CHECK_ARG(norm_parts < 1 || q_w, "qk_norm_rope: q_w missing");
  AQB_CHECK_ARG(norm_parts < 2 || k_w, "qk_norm_rope: k_w missing");
  AQB_CHECK_ARG(head_begin >= 0 && head_count >= 1 && head_begin + head_count <= heads, "qk_norm_rope: bad heads");
  AQB_CHECK_ARG(hpg >= 1 && head_count % hpg == 0, "qk_norm_rope: bad heads-per-group");
  AQB_CHECK_ARG(rope_rows <= 0 || (rope_cos && rope_sin), "qk_norm_rope: rope tables missing");
  AQB_CHECK_ARG(ld_src >= int64_t(parts) * heads * head_dim, "qk_norm_rope: bad ld_src");
  if (rows <= 0) return AQB_OK;
  const int64_t items = rows * head_count;
  const int grid = static_cast<int>((items + 7) / 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto sp = reinterpret_cast<const T*>(src);
  auto dp = reinterpret_cast<T*>(dst);
#define QK_CASE(D)                                                                                                \
  case D:                                                                                                         \
    AQB_CUDA_TRY(launch_pdl(qk_norm_rope_kernel<D, T>, dim3(grid), dim3(256), 0, s, sp, ld_src, rows, heads, head_begin, head_count, q_w, k_w,     \
                                                   eps, rope_cos, rope_sin, rope_row0, rope_rows, dp,             \
                                                   dst_group_stride, dst_row_stride, dst_which_stride, hpg, parts, \
                                                   norm_parts, run_flag, run_if));                                 \
    break;
  switch (head_dim) {
    QK_CASE(32) QK_CASE(64) QK_CASE(128) QK_CASE(256)
    default:
      return set_error(AQB_EUNSUPPORTED, "qk_norm_rope: head_dim %d unsupported", head_dim);
  }
#undef QK_CASE
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_qk_norm_rope(const void* src, int64_t ld_src, int64_t rows, int32_t heads, int32_t head_begin,
                                int32_t head_count, int32_t head_dim, const float* q_w, const float* k_w, float eps,
                                const float* rope_cos, const float* rope_sin, int64_t rope_row0, int64_t rope_rows,
                                void* dst, int64_t dst_group_stride, int64_t dst_row_stride, int64_t dst_which_stride,
                                int32_t hpg, int32_t parts, int32_t norm_parts, const int32_t* run_flag,
                                int32_t run_if, void* stream) {
  return qk_norm_rope<__nv_bfloat16>(src, ld_src, rows, heads, head_begin, head_count, head_dim, q_w, k_w, eps,
                                     rope_cos, rope_sin, rope_row0, rope_rows, dst, dst_group_stride, dst_row_stride,
                                     dst_which_stride, hpg, parts, norm_parts, run_flag, run_if, stream);
}

extern "C" int aqb_qk_norm_rope_f32(const float* src, int64_t ld_src, int64_t rows, int32_t heads, int32_t head_begin,
                                    int32_t head_count, int32_t head_dim, const float* q_w, const float* k_w,
                                    float eps, const float* rope_cos, const float* rope_sin, int64_t rope_row0,
                                    int64_t rope_rows, float* dst, int64_t dst_group_stride, int64_t dst_row_stride,
                                    int64_t dst_which_stride, int32_t hpg, int32_t parts, int32_t norm_parts,
                                    const int32_t* run_flag, int32_t run_if, void* stream) {
  return qk_norm_rope<float>(src, ld_src, rows, heads, head_begin, head_count, head_dim, q_w, k_w, eps, rope_cos,
                             rope_sin, rope_row0, rope_rows, dst, dst_group_stride, dst_row_stride, dst_which_stride,
                             hpg, parts, norm_parts, run_flag, run_if, stream);
}

extern "C" int aqb_gemv(const void* w, const float* x, const float* t, const float* b, const float* add, float* y,
                        int64_t n, int64_t k, int32_t in_silu, void* stream) {
  AQB_CHECK_ARG(w && y, "gemv: null pointer");
  AQB_CHECK_ARG(x || t, "gemv: need x or t");
  AQB_CHECK_ARG(k % 8 == 0 && k >= 8 && k <= 16384, "gemv: k=%lld unsupported", (long long)k);
  if (n <= 0) return AQB_OK;
  int64_t g = (n + 7) / 8;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  if (g > cap) g = cap;
  AQB_CUDA_TRY(launch_pdl(gemv_kernel, dim3(static_cast<int>(g)), dim3(256), k * sizeof(float), reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const __nv_bfloat16*>(w), x, t, b, add, y, n, static_cast<int>(k), in_silu));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_add_bcast(float* out, const float* a, int64_t period, const float* b, int64_t n, void* stream) {
  AQB_CHECK_ARG(out && a && b && period >= 1, "add_bcast: bad args");
  if (n <= 0) return AQB_OK;
  AQB_CUDA_TRY(launch_pdl(add_bcast_kernel, dim3(grid_for(n, 256)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), out, a, period, b, n));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_gate_bcast(const float* src, int64_t lds, const float* gate, float* const* dst, int32_t ndst,
                              int64_t ldd, int64_t rows, int64_t cols, const int32_t* run_flag, int32_t run_if,
                              void* stream) {
  AQB_CHECK_ARG(src && dst && ndst >= 1 && ndst <= 8 && cols % 4 == 0 && lds % 4 == 0 && ldd % 4 == 0,
                "gate_bcast: bad args");
  SlotDsts d{};
  d.n = ndst;
  for (int i = 0; i < ndst; ++i) {
    AQB_CHECK_ARG(dst[i] && reinterpret_cast<uintptr_t>(dst[i]) % 16 == 0, "gate_bcast: dst[%d]", i);
    d.p[i] = dst[i];
  }
  if (rows <= 0) return AQB_OK;
  AQB_CUDA_TRY(launch_pdl(gate_bcast_kernel, dim3(grid_for(rows * cols / 4, 256)), dim3(256), 0,
                          reinterpret_cast<cudaStream_t>(stream), src, lds, gate, d, ldd, rows, int(cols / 4),
                          run_flag, run_if));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_sum_slots(float* x, int64_t ldx, const float* slots, int32_t nslots, int64_t slot_stride,
                             int64_t lds, int64_t rows, int64_t cols, const int32_t* run_flag, int32_t run_if,
                             void* stream) {
  AQB_CHECK_ARG(x && slots && nslots >= 1 && cols % 4 == 0 && ldx % 4 == 0 && lds % 4 == 0 && slot_stride % 4 == 0,
                "sum_slots: bad args");
  if (rows <= 0) return AQB_OK;
  AQB_CUDA_TRY(launch_pdl(sum_slots_kernel, dim3(grid_for(rows * cols / 4, 256)), dim3(256), 0,
                          reinterpret_cast<cudaStream_t>(stream), x, ldx, slots, nslots, slot_stride, lds, rows,
                          int(cols / 4), run_flag, run_if));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_rel_l1_reduce(const float* partials, int64_t rows, float* sums, void* stream) {
  AQB_CHECK_ARG(partials && sums && rows >= 1, "rel_l1_reduce: bad args");
  AQB_CUDA_TRY(launch_pdl(rel_l1_reduce_kernel, dim3(1), dim3(1024), 0, reinterpret_cast<cudaStream_t>(stream), partials, rows, sums));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_cache_decide(const float* sums, int32_t* state, float threshold, int32_t warmup,
                                int32_t total_steps, int32_t force_last, int32_t* flags_out, float* rel_out,
                                void* stream) {
  AQB_CHECK_ARG(sums && state && total_steps >= 1, "cache_decide: bad args");
  AQB_CUDA_TRY(launch_pdl(cache_decide_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), sums, state, threshold, warmup, total_steps,
                                                                            force_last, flags_out, rel_out));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_cache_offset(float* x, int64_t ldx, float* off, int64_t rows, int32_t hidden, int32_t mode,
                                const int32_t* run_flag, int32_t run_if, void* stream) {
  AQB_CHECK_ARG(x && off && hidden % 4 == 0 && ldx % 4 == 0 && mode >= 0 && mode <= 2, "cache_offset: bad args");
  if (rows <= 0) return AQB_OK;
  AQB_CUDA_TRY(launch_pdl(cache_offset_kernel, dim3(grid_for(rows * hidden / 4, 256)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), x, ldx, off, rows, hidden, mode, run_flag, run_if));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_step_scalars(const float* ts, const float* dts, int32_t* idx, float* cur, int32_t mode,
                                void* stream) {
  AQB_CHECK_ARG(ts && dts && idx && cur, "step_scalars: null pointer");
  AQB_CUDA_TRY(launch_pdl(step_scalars_kernel, dim3(1), dim3(1), 0, reinterpret_cast<cudaStream_t>(stream), ts, dts, idx, cur, mode));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_patchify(const float* lat, float* tok, void* tok_bf16, int32_t C, int32_t T, int32_t H, int32_t W,
                            int32_t pt, int32_t ph, int32_t pw, int32_t lat_frames, int32_t frame_offset,
                            void* stream) {
  AQB_CHECK_ARG(lat && tok && C > 0 && T > 0 && H > 0 && W > 0 && pt > 0 && ph > 0 && pw > 0, "patchify: bad args");
  AQB_CHECK_ARG(frame_offset >= 0 && frame_offset + T * pt <= lat_frames, "patchify: frame window out of range");
  const int64_t n = static_cast<int64_t>(C) * T * H * W * pt * ph * pw;
  AQB_CUDA_TRY(launch_pdl(patchify_kernel, dim3(grid_for(n, 256)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), lat, tok, reinterpret_cast<__nv_bfloat16*>(tok_bf16), C, T, H, W, pt, ph, pw, lat_frames, frame_offset));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_unpatchify(const float* tok, float* lat, int32_t C, int32_t T, int32_t H, int32_t W, int32_t pt,
                              int32_t ph, int32_t pw, int32_t lat_frames, int32_t frame_offset, void* stream) {
  AQB_CHECK_ARG(lat && tok && C > 0 && T > 0 && H > 0 && W > 0 && pt > 0 && ph > 0 && pw > 0, "unpatchify: bad args");
  AQB_CHECK_ARG(frame_offset >= 0 && frame_offset + T * pt <= lat_frames, "unpatchify: frame window out of range");
  const int64_t n = static_cast<int64_t>(C) * T * H * W * pt * ph * pw;
  AQB_CUDA_TRY(launch_pdl(unpatchify_kernel, dim3(grid_for(n, 256)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), tok, lat, C, T, H, W, pt,
                                                                                           ph, pw, lat_frames,
                                                                                           frame_offset));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_heads_to_seq(const void* src, int64_t rows, int32_t P, int32_t width, void* dst, int64_t ld_dst,
                                const int32_t* run_flag, int32_t run_if, void* stream) {
  AQB_CHECK_ARG(src && dst && P >= 1 && width % 8 == 0 && ld_dst % 8 == 0 && ld_dst >= int64_t(P) * width,
                "heads_to_seq: bad args");
  if (rows <= 0) return AQB_OK;
  const int w16 = width / 8;
  AQB_CUDA_TRY(launch_pdl(heads_to_seq_kernel, dim3(grid_for(rows * P * w16, 256)), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), reinterpret_cast<const uint4*>(src), rows, P, w16, reinterpret_cast<uint4*>(dst), ld_dst / 8, run_flag, run_if));
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}
