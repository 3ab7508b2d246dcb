// VAE tile blend and temporal MultiDiffusion averaging (sm_100a) — the HBM-bound
// steps either side of the denoise loop.
//
// aqb_tile_blend: the linear combination of overlapping decoded tiles
// ("blend the corresponding block features through a linear combination",
// PAPER.md:79; "linearly summing the overlapping parts") with the
// reference plan's separable ramps (pkg/src/ditplan/inference.py:104-176):
//   out[c, p] = sum_k prof_k(p) * tile_k[c, p - start_k] / sum_k prof_k(p).
// One thread per latent position: the covering tiles (a contiguous index range
// per axis, starts sorted) and their weights are found once and reused for all
// channels; accumulation in fp64 in plan order (deterministic).
//
// aqb_window_average: Eq. 3 of PAPER.md:415 over the clips of a WindowPlan
// (inference.py:229-279): out[c, i, :] = (sum_{k in S(i)} clip_k[c, i - s_k, :]) / |S(i)|,
// sum in clip order.  A CTA row is one (c, i) frame plane, so the clip choice is
// uniform per CTA and the HW plane streams with 16-byte accesses.
#include "host.cuh"

namespace aqb {
namespace tiles {

struct Axis {
  const int32_t* starts;
  int n, size, overlap;
};

__device__ __forceinline__ double ramp(int j, int size, int overlap) {
  const int e = overlap < size ? overlap : size;
  double r = 1.0;
  if (j < e) r = (j + 1.0) / (e + 1.0);
  if (j >= size - e) r = fmin(r, (size - j) / (e + 1.0));
  return r;
}

__device__ __forceinline__ void cover(const Axis& a, int x, int& lo, int& hi) {
  lo = a.n, hi = -1;
  for (int k = 0; k < a.n; ++k) {
    const int s = a.starts[k];
    if (s <= x && x < s + a.size) {
      lo = min(lo, k);
      hi = k;
    }
  }
}

__global__ void __launch_bounds__(256) blend_kernel(const int64_t* __restrict__ ptrs, Axis at, Axis ah, Axis aw,
                                                    int T, int H, int W, int C, float* __restrict__ out) {
  const int64_t plane = static_cast<int64_t>(T) * H * W;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= plane) return;
  const int w = int(p % W), h = int((p / W) % H), t = int(p / (static_cast<int64_t>(H) * W));
  int t0, t1, h0, h1, w0, w1;
  cover(at, t, t0, t1);
  cover(ah, h, h0, h1);
  cover(aw, w, w0, w1);
  double total = 0.0;
  for (int it = t0; it <= t1; ++it)
    for (int ih = h0; ih <= h1; ++ih)
      for (int iw = w0; iw <= w1; ++iw)
        total += ramp(t - at.starts[it], at.size, at.overlap) * ramp(h - ah.starts[ih], ah.size, ah.overlap) *
                 ramp(w - aw.starts[iw], aw.size, aw.overlap);
  const int64_t tplane = static_cast<int64_t>(at.size) * ah.size * aw.size;
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
    for (int it = t0; it <= t1; ++it)
      for (int ih = h0; ih <= h1; ++ih)
        for (int iw = w0; iw <= w1; ++iw) {
          const int lt = t - at.starts[it], lh = h - ah.starts[ih], lw = w - aw.starts[iw];
          const double wt = ramp(lt, at.size, at.overlap) * ramp(lh, ah.size, ah.overlap) *
                            ramp(lw, aw.size, aw.overlap);
          const float* tile = reinterpret_cast<const float*>(ptrs[(static_cast<int64_t>(it) * ah.n + ih) * aw.n + iw]);
          acc += wt * tile[c * tplane + (static_cast<int64_t>(lt) * ah.size + lh) * aw.size + lw];
        }
    out[c * plane + p] = static_cast<float>(acc / total);
  }
}

__global__ void __launch_bounds__(256) window_kernel(const int64_t* __restrict__ ptrs,
                                                     const int32_t* __restrict__ starts, int nclips, int n,
                                                     int n_prime, int64_t HW, float* __restrict__ out) {
  const int row = blockIdx.y;  // c * n_prime + i
  const int c = row / n_prime, i = row % n_prime;
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool vec = (HW % 4) == 0;
  const int64_t width = vec ? HW / 4 : HW;
  if (x >= width) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int cnt = 0;
  for (int k = 0; k < nclips; ++k) {
    const int s = starts[k];
    if (i < s || i >= s + n) continue;
    const float* clip = reinterpret_cast<const float*>(ptrs[k]) + (static_cast<int64_t>(c) * n + (i - s)) * HW;
    if (vec) {
      const float4 v = reinterpret_cast<const float4*>(clip)[x];
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    } else {
      acc.x += clip[x];
    }
    ++cnt;
  }
  const float inv = static_cast<float>(cnt);
  float* o = out + static_cast<int64_t>(row) * HW;
  if (vec)
    reinterpret_cast<float4*>(o)[x] = make_float4(acc.x / inv, acc.y / inv, acc.z / inv, acc.w / inv);
  else
    o[x] = acc.x / inv;
}

}  // namespace tiles
}  // namespace aqb

extern "C" int aqb_tile_blend(const int64_t* tile_ptrs, const int32_t* axis_starts, int32_t nt, int32_t nh,
                              int32_t nw, int32_t tile_t, int32_t tile_h, int32_t tile_w, int32_t ov_t, int32_t ov_h,
                              int32_t ov_w, int32_t T, int32_t H, int32_t W, int32_t C, float* out, void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(tile_ptrs && axis_starts && out, "tile_blend: null pointer");
  AQB_CHECK_ARG(nt >= 1 && nh >= 1 && nw >= 1 && C >= 1 && T >= 1 && H >= 1 && W >= 1, "tile_blend: bad shape");
  AQB_CHECK_ARG(tile_t >= 1 && tile_h >= 1 && tile_w >= 1 && tile_t <= T && tile_h <= H && tile_w <= W,
                "tile_blend: tile size must be in [1, latent]");
  AQB_CHECK_ARG(ov_t >= 0 && ov_h >= 0 && ov_w >= 0 && ov_t < tile_t && ov_h < tile_h && ov_w < tile_w,
                "tile_blend: need tile size > overlap >= 0");
  tiles::Axis at{axis_starts, nt, tile_t, ov_t}, ah{axis_starts + nt, nh, tile_h, ov_h},
      aw{axis_starts + nt + nh, nw, tile_w, ov_w};
  const int64_t plane = static_cast<int64_t>(T) * H * W;
  tiles::blend_kernel<<<unsigned((plane + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      tile_ptrs, at, ah, aw, T, H, W, C, out);
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}

extern "C" int aqb_window_average(const int64_t* clip_ptrs, const int32_t* clip_starts, int32_t nclips, int32_t n,
                                  int32_t n_prime, int32_t C, int64_t hw, float* out, void* stream) {
  using namespace aqb;
  AQB_CHECK_ARG(clip_ptrs && clip_starts && out, "window_average: null pointer");
  AQB_CHECK_ARG(nclips >= 1 && n >= 1 && n <= n_prime && C >= 1 && hw >= 1, "window_average: bad shape");
  AQB_CHECK_ARG(int64_t(C) * n_prime < 65536, "window_average: C * n' must be < 65536");
  const int64_t width = hw % 4 == 0 ? hw / 4 : hw;
  dim3 grid(unsigned((width + 255) / 256), unsigned(C * n_prime));
  tiles::window_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(clip_ptrs, clip_starts, nclips, n,
                                                                                 n_prime, hw, out);
  AQB_LAUNCH_CHECK();
  return AQB_OK;
}
