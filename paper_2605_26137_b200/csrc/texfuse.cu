// texfuse.cu — device-resident consumers of the G-buffer:
// the texture-fusion steps of proj/src/texfuse/fuse.cpp and mips.cpp.
//
//   edgeMask          (fuse.cpp:66-101)   k_edge_mask        one thread per view pixel
//   buildMips         (mips.cpp:96-112)   k_halve_x/_y, k_blur_x, k_unsharp (separable passes)
//   backprojectView   (fuse.cpp:103-186)  k_valid_bounds -> k_backproject (one thread per texel)
//   incidenceMap      (fuse.cpp:188-221)  k_incidence        one thread per texel
//   blendViews        (fuse.cpp:223-280)  k_blend            one thread per texel over the views
//   footprintFromJacobian (fuse.cpp:39-64) footprint()       per texel inside k_backproject
//
// Arithmetic follows the reference expression by expression (TUs built with
// --fmad=false): projections, jacobians, gates, bilinear/trilinear weights and
// the Lanczos/unsharp sums are IEEE + - * / sqrt and floor/ceil/llround, so they
// are bit-identical; std::hypot is glibc's own algorithm (below), so the
// footprint's singular values are too. The remaining transcendental calls
// (log2 of the footprint, log/exp of the blend) are CUDA's, within 1 ulp of
// glibc's; they perturb doubles at the 1e-16 level before the final f32 cast.
// Host-side constants that the reference computes with libm (the Lanczos taps,
// log(prior), log(epsilon)) are computed on the host with the same calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "bake.cuh"

namespace mfb {
namespace {

// glibc's __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, glibc >= 2.35, the
// non-FMA kernel this image's libm runs: 0 mismatches in 2e7 random pairs):
// Borges' correction of sqrt(ax^2 + ay^2) with range scaling.
__device__ double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
__device__ double glibc_hypot(double x, double y) {
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return x + y;
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return hypot_kernel(ax, ay);
}

__device__ __forceinline__ d3 ldf3(const float* p) {
  return mk3(static_cast<double>(p[0]), static_cast<double>(p[1]), static_cast<double>(p[2]));
}

// OrthoCamera::project (render/camera.h:33-37) and imagePixel (fuse.cpp:15-18)
__device__ __forceinline__ d3 cam_project(const TfCamera& c, d3 p) {
  return mk3(dot(p, mk3(c.right[0], c.right[1], c.right[2])), dot(p, mk3(c.up[0], c.up[1], c.up[2])),
             dot(p, mk3(-c.dir[0], -c.dir[1], -c.dir[2])));
}
__device__ __forceinline__ void image_pixel(const TfCamera& c, d3 uv, double& px, double& py) {
  const double s = c.res / (2.0 * c.he);
  px = (uv.x + c.he) * s - 0.5;
  py = (c.he - uv.y) * s - 0.5;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// ---------------------------------------------------------------- edgeMask
__global__ void k_edge_mask(int w, int h, const float* __restrict__ pos, const int32_t* __restrict__ face,
                            double limit2, uint8_t* __restrict__ mask) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(w) * h) return;
  const int x = static_cast<int>(i % w), y = static_cast<int>(i / w);
  const bool fg = face[i] >= 0;
  const d3 p = ldf3(pos + 3 * i);
  bool masked = false;
  for (int dy = -1; dy <= 1 && !masked; ++dy)
    for (int dx = -1; dx <= 1 && !masked; ++dx) {
      if (dx == 0 && dy == 0) continue;
      const int nx = x + dx, ny = y + dy;
      if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
      const int64_t n = static_cast<int64_t>(ny) * w + nx;
      const bool nfg = face[n] >= 0;
      if (fg != nfg) {
        masked = true;  // either side of the silhouette ring
      } else if (fg) {
        masked = sqnorm(p - ldf3(pos + 3 * n)) > limit2;
      }
    }
  mask[i] = masked ? 1 : 0;
}

// ---------------------------------------------------------------- buildMips
struct Taps8 {
  double k[8];
};
// halveX (mips.cpp:36-51): out ow x h x c
__global__ void k_halve_x(int w, int h, int c, const float* __restrict__ in, float* __restrict__ out, Taps8 kt) {
  const int ow = max(1, (w + 1) / 2);
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(ow) * h * c) return;
  const int ch = static_cast<int>(i % c);
  const int64_t px = i / c;
  const int x = static_cast<int>(px % ow), y = static_cast<int>(px / ow);
  double acc = 0.0;
  for (int d = -3; d <= 4; ++d) {
    const int sx = min(max(2 * x + d, 0), w - 1);
    acc += kt.k[d + 3] * static_cast<double>(in[(static_cast<int64_t>(y) * w + sx) * c + ch]);
  }
  out[i] = static_cast<float>(acc);
}
// halveY (mips.cpp:53-68): out w x oh x c
__global__ void k_halve_y(int w, int h, int c, const float* __restrict__ in, float* __restrict__ out, Taps8 kt) {
  const int oh = max(1, (h + 1) / 2);
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(w) * oh * c) return;
  const int ch = static_cast<int>(i % c);
  const int64_t px = i / c;
  const int x = static_cast<int>(px % w), y = static_cast<int>(px / w);
  double acc = 0.0;
  for (int d = -3; d <= 4; ++d) {
    const int sy = min(max(2 * y + d, 0), h - 1);
    acc += kt.k[d + 3] * static_cast<double>(in[(static_cast<int64_t>(sy) * w + x) * c + ch]);
  }
  out[i] = static_cast<float>(acc);
}
// unsharp (mips.cpp:71-92): the x blur, then the y blur fused with the update
__global__ void k_blur_x(int w, int h, int c, const float* __restrict__ in, float* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(w) * h * c) return;
  const int ch = static_cast<int>(i % c);
  const int64_t px = i / c;
  const int x = static_cast<int>(px % w), y = static_cast<int>(px / w);
  const double wt[3] = {0.25, 0.5, 0.25};
  double acc = 0.0;
  for (int d = -1; d <= 1; ++d)
    acc += wt[d + 1] * static_cast<double>(in[(static_cast<int64_t>(y) * w + min(max(x + d, 0), w - 1)) * c + ch]);
  out[i] = static_cast<float>(acc);
}
__global__ void k_unsharp(int w, int h, int c, const float* __restrict__ in, const float* __restrict__ blur_x,
                          float strength, float* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(w) * h * c) return;
  const int ch = static_cast<int>(i % c);
  const int64_t px = i / c;
  const int x = static_cast<int>(px % w), y = static_cast<int>(px / w);
  const double wt[3] = {0.25, 0.5, 0.25};
  double blur = 0.0;
  for (int d = -1; d <= 1; ++d)
    blur += wt[d + 1] * static_cast<double>(blur_x[(static_cast<int64_t>(min(max(y + d, 0), h - 1)) * w + x) * c + ch]);
  const double v = in[i];
  out[i] = static_cast<float>(v + strength * (v - blur));
}

// ---------------------------------------------------------------- backprojectView
// bounds of the valid texels' positions (fuse.cpp:122-130) as ordered f32 keys
__device__ __forceinline__ unsigned f2o(float f) {
  const unsigned b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float o2f(unsigned o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__global__ void k_valid_bounds(int64_t n, const float* __restrict__ pos, const uint8_t* __restrict__ valid,
                               unsigned* __restrict__ b6) {
  unsigned lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!valid[t]) continue;
    for (int k = 0; k < 3; ++k) {
      const unsigned o = f2o(pos[3 * t + k]);
      lo[k] = min(lo[k], o);
      hi[k] = max(hi[k], o);
    }
  }
  for (int k = 0; k < 3; ++k)
    for (int off = 16; off > 0; off >>= 1) {
      lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], off));
      hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], off));
    }
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < 3; ++k) {
      if (lo[k] != 0xffffffffu) atomicMin(&b6[k], lo[k]);
      if (hi[k] != 0u) atomicMax(&b6[3 + k], hi[k]);
    }
}

struct MipChain {
  const float* base = nullptr;
  int n = 0, c = 0;
  int w[kTfMaxMips], h[kTfMaxMips];
  int64_t off[kTfMaxMips];
};

// Image::bilinear (core/image.h:28-42) at level l
__device__ double bilinear(const MipChain& mc, int l, double x, double y, int ch) {
  const int w = mc.w[l], h = mc.h[l];
  const float* im = mc.base + mc.off[l];
  const double cx = clampd(x, 0.0, static_cast<double>(w - 1));
  const double cy = clampd(y, 0.0, static_cast<double>(h - 1));
  const int x0 = static_cast<int>(floor(cx));
  const int y0 = static_cast<int>(floor(cy));
  const int x1 = min(x0 + 1, w - 1);
  const int y1 = min(y0 + 1, h - 1);
  const double fx = cx - x0, fy = cy - y0;
  const double v00 = im[(static_cast<int64_t>(y0) * w + x0) * mc.c + ch];
  const double v10 = im[(static_cast<int64_t>(y0) * w + x1) * mc.c + ch];
  const double v01 = im[(static_cast<int64_t>(y1) * w + x0) * mc.c + ch];
  const double v11 = im[(static_cast<int64_t>(y1) * w + x1) * mc.c + ch];
  return (v00 * (1 - fx) + v10 * fx) * (1 - fy) + (v01 * (1 - fx) + v11 * fx) * fy;
}

// sampleTrilinear (fuse.cpp:22-35)
__device__ double trilinear(const MipChain& mc, double px, double py, double mip, int ch) {
  const int last = mc.n - 1;
  const double m = clampd(mip, 0.0, static_cast<double>(last));
  const int l0 = static_cast<int>(floor(m));
  const int l1 = min(l0 + 1, last);
  const double f = m - l0;
  const double s0 = ldexp(1.0, -l0);
  const double v0 = bilinear(mc, l0, (px + 0.5) * s0 - 0.5, (py + 0.5) * s0 - 0.5, ch);
  if (f == 0.0) return v0;
  const double s1 = ldexp(1.0, -l1);
  return (1.0 - f) * v0 + f * bilinear(mc, l1, (px + 0.5) * s1 - 0.5, (py + 0.5) * s1 - 0.5, ch);
}

// trilinear for all channels (up to kTfFastChannels) at once: the same
// per-channel expressions as trilinear / bilinear, shared weights and offsets
constexpr int kTfFastChannels = 4;
__device__ void bilinear_all(const MipChain& mc, int l, double x, double y, double* out) {
  const int w = mc.w[l], h = mc.h[l];
  const float* im = mc.base + mc.off[l];
  const double cx = clampd(x, 0.0, static_cast<double>(w - 1));
  const double cy = clampd(y, 0.0, static_cast<double>(h - 1));
  const int x0 = static_cast<int>(floor(cx));
  const int y0 = static_cast<int>(floor(cy));
  const int x1 = min(x0 + 1, w - 1);
  const int y1 = min(y0 + 1, h - 1);
  const double fx = cx - x0, fy = cy - y0;
  const double gx = 1 - fx, gy = 1 - fy;
  const float* p00 = im + (static_cast<int64_t>(y0) * w + x0) * mc.c;
  const float* p10 = im + (static_cast<int64_t>(y0) * w + x1) * mc.c;
  const float* p01 = im + (static_cast<int64_t>(y1) * w + x0) * mc.c;
  const float* p11 = im + (static_cast<int64_t>(y1) * w + x1) * mc.c;
#pragma unroll
  for (int ch = 0; ch < kTfFastChannels; ++ch) {
    if (ch >= mc.c) break;
    const double v00 = p00[ch], v10 = p10[ch], v01 = p01[ch], v11 = p11[ch];
    out[ch] = (v00 * gx + v10 * fx) * gy + (v01 * gx + v11 * fx) * fy;
  }
}
__device__ void trilinear_all(const MipChain& mc, double px, double py, double mip, double* out) {
  const int last = mc.n - 1;
  const double m = clampd(mip, 0.0, static_cast<double>(last));
  const int l0 = static_cast<int>(floor(m));
  const int l1 = min(l0 + 1, last);
  const double f = m - l0;
  const double s0 = ldexp(1.0, -l0);
  bilinear_all(mc, l0, (px + 0.5) * s0 - 0.5, (py + 0.5) * s0 - 0.5, out);
  if (f == 0.0) return;
  double v1[kTfFastChannels];
  const double s1 = ldexp(1.0, -l1);
  bilinear_all(mc, l1, (px + 0.5) * s1 - 0.5, (py + 0.5) * s1 - 0.5, v1);
#pragma unroll
  for (int ch = 0; ch < kTfFastChannels; ++ch)
    if (ch < mc.c) out[ch] = (1.0 - f) * out[ch] + f * v1[ch];
}

struct Footprint {
  double ax = 1.0, ay = 0.0;  // major axis (unit)
  double major = 1.0;
  double mip = 0.0;
  int taps = 1;
};

// footprintFromJacobian (fuse.cpp:39-64); J = [colX colY]
__device__ Footprint footprint(double jx0, double jx1, double jy0, double jy1) {
  Footprint fp;
  // m = J J^T (Eigen's 2x2 lazy product: m(i,j) = J(i,0) J(j,0) + J(i,1) J(j,1))
  const double m00 = jx0 * jx0 + jy0 * jy0;
  const double m01 = jx0 * jx1 + jy0 * jy1;
  const double m11 = jx1 * jx1 + jy1 * jy1;
  const double mean = 0.5 * (m00 + m11);
  const double disc = glibc_hypot(0.5 * (m00 - m11), m01);
  const double sp = mean + disc, sm = mean - disc;
  const double s1 = sqrt(0.0 < sp ? sp : 0.0);  // std::max(0.0, .) keeps its first argument on ties / NaN
  const double s2 = sqrt(0.0 < sm ? sm : 0.0);
  constexpr double kTiny = 1e-12;
  if (!(s1 > kTiny)) return fp;
  double axx = m01, axy = mean + disc - m00;
  const double alx = mean + disc - m11, aly = m01;
  if (alx * alx + aly * aly > axx * axx + axy * axy) {
    axx = alx;
    axy = aly;
  }
  const double z = axx * axx + axy * axy;
  if (z > 0.0) {  // normalized(): v / sqrt(squaredNorm)
    const double r = sqrt(z);
    fp.ax = axx / r;
    fp.ay = axy / r;
  }
  fp.major = s1;
  const double s2c = s2 < kTiny ? kTiny : s2;  // std::max(s2, kTiny)
  const double ratio = s1 / s2c;
  fp.taps = static_cast<int>(clampd(ceil(ratio), 1.0, 8.0));
  const double capped = 8.0 < ratio ? 8.0 : ratio;  // std::min(ratio, 8.0)
  const double mip = log2(s2c) - 0.5 + 0.5 * log2(capped);
  fp.mip = 0.0 < mip ? mip : 0.0;  // std::max(0.0, .)
  return fp;
}

// 8 CTAs of 128 threads per SM (64 registers; 96 unbounded at 5 CTAs): 10
// views 4.64 -> 4.06 ms per mf_fuse_views_dev (6 CTAs: 4.39, 10: 4.19)
__global__ void __launch_bounds__(128, 8) k_backproject(int n, const float* __restrict__ pos,
                                                     const uint8_t* __restrict__ valid,
                                                     const unsigned* __restrict__ b6, TfCamera cam, MipChain mc,
                                                     const uint8_t* __restrict__ mask, float* __restrict__ color,
                                                     uint8_t* __restrict__ sampled) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<int64_t>(n) * n) return;
  const int x = static_cast<int>(t % n), y = static_cast<int>(t / n);
  for (int ch = 0; ch < mc.c; ++ch) color[t * mc.c + ch] = 0.0f;
  sampled[t] = 0;
  if (!valid[t]) return;
  // neighbour gate (fuse.cpp:131-134)
  const d3 lo = mk3(o2f(b6[0]), o2f(b6[1]), o2f(b6[2])), hi = mk3(o2f(b6[3]), o2f(b6[4]), o2f(b6[5]));
  double gate2 = 0.05 * norm(hi - lo);
  gate2 *= gate2;
  const d3 p = ldf3(pos + 3 * t);
  double px, py;
  image_pixel(cam, cam_project(cam, p), px, py);
  const int cx = static_cast<int>(llround(px));
  const int cy = static_cast<int>(llround(py));
  if (cx < 0 || cy < 0 || cx >= cam.res || cy >= cam.res) return;
  if (mask[static_cast<int64_t>(cy) * cam.res + cx]) return;
  // finite differences (fuse.cpp:136-151)
  auto diff = [&](int64_t fwd, int64_t bwd, bool has_fwd, bool has_bwd, double& c0, double& c1) {
    if (has_fwd && valid[fwd]) {
      const d3 q = ldf3(pos + 3 * fwd);
      if (sqnorm(q - p) <= gate2) {
        double qx, qy;
        image_pixel(cam, cam_project(cam, q), qx, qy);
        c0 = qx - px;
        c1 = qy - py;
        return true;
      }
    }
    if (has_bwd && valid[bwd]) {
      const d3 q = ldf3(pos + 3 * bwd);
      if (sqnorm(p - q) <= gate2) {
        double qx, qy;
        image_pixel(cam, cam_project(cam, q), qx, qy);
        c0 = px - qx;
        c1 = py - qy;
        return true;
      }
    }
    return false;
  };
  Footprint fp;
  double jx0, jx1, jy0, jy1;
  if (diff(t + 1, t - 1, x + 1 < n, x > 0, jx0, jx1) && diff(t + n, t - n, y + 1 < n, y > 0, jy0, jy1))
    fp = footprint(jx0, jx1, jy0, jy1);
  if (mc.c <= kTfFastChannels) {
    // taps outer, channels inner: each tap's level pick, bilinear weights and
    // addresses once for all channels (adjacent floats of one texel); every
    // channel still accumulates its taps in order (bit-identical)
    double acc[kTfFastChannels];
#pragma unroll
    for (int ch = 0; ch < kTfFastChannels; ++ch) acc[ch] = 0.0;
    for (int i = 0; i < fp.taps; ++i) {
      const double s = (i + 0.5) / fp.taps - 0.5;
      const double k = fp.major * s;
      double v[kTfFastChannels];
      trilinear_all(mc, px + fp.ax * k, py + fp.ay * k, fp.mip, v);
#pragma unroll
      for (int ch = 0; ch < kTfFastChannels; ++ch) acc[ch] += v[ch];
    }
#pragma unroll
    for (int ch = 0; ch < kTfFastChannels; ++ch)
      if (ch < mc.c) color[t * mc.c + ch] = static_cast<float>(acc[ch] / fp.taps);
  } else {
    for (int ch = 0; ch < mc.c; ++ch) {
      double acc = 0.0;
      for (int i = 0; i < fp.taps; ++i) {
        const double s = (i + 0.5) / fp.taps - 0.5;
        const double k = fp.major * s;
        acc += trilinear(mc, px + fp.ax * k, py + fp.ay * k, fp.mip, ch);
      }
      color[t * mc.c + ch] = static_cast<float>(acc / fp.taps);
    }
  }
  sampled[t] = 1;
}

// ---------------------------------------------------------------- incidenceMap
__global__ void k_incidence(int n, const float* __restrict__ pos, const float* __restrict__ nrm,
                            const uint8_t* __restrict__ valid, TfCamera cam, const float* __restrict__ depth,
                            double tolerance, float* __restrict__ out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= static_cast<int64_t>(n) * n) return;
  float r = 0.0f;
  if (valid[t]) {
    const double cosine = dot(ldf3(nrm + 3 * t), mk3(-cam.dir[0], -cam.dir[1], -cam.dir[2]));
    if (cosine > 0.0) {
      const d3 uvd = cam_project(cam, ldf3(pos + 3 * t));
      double px, py;
      image_pixel(cam, uvd, px, py);
      const int cx = static_cast<int>(llround(px));
      const int cy = static_cast<int>(llround(py));
      if (cx >= 0 && cy >= 0 && cx < cam.res && cy < cam.res) {
        const double view_depth = depth[static_cast<int64_t>(cy) * cam.res + cx];
        if (fabs(uvd.z - view_depth) <= tolerance) r = static_cast<float>(cosine);
      }
    }
  }
  out[t] = r;
}

// ---------------------------------------------------------------- blendViews
// Per texel: the contributor terms l_k = log(prior_k) + alpha log(I_k) are
// recomputed in each of the three passes (peak, denominator, colours) instead
// of being stored, so any view count fits; the values are the same bits.
constexpr int kParamViews = 64;
constexpr int kBlendCache = 16;  // views whose blend terms stay in registers
struct BlendParams {
  double lp[kParamViews];
  uint8_t pos[kParamViews];
};
__global__ void k_blend(int k, int64_t n, int c, const float* __restrict__ colors, const uint8_t* __restrict__ sampled,
                        const float* __restrict__ inc, const BlendParams bp, const double* __restrict__ logp_big,
                        const uint8_t* __restrict__ pos_big, double alpha, double log_eps, float* __restrict__ out,
                        uint8_t* __restrict__ filled) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  for (int ch = 0; ch < c; ++ch) out[t * c + ch] = 0.0f;
  filled[t] = 0;
  auto term = [&](int i, double& l) {
    const bool ppos = i < kParamViews ? bp.pos[i] != 0 : pos_big[i] != 0;
    if (!sampled[i * n + t] || !ppos) return false;
    const double iv = inc[i * n + t];
    if (iv <= 0.0) return false;
    l = (i < kParamViews ? bp.lp[i] : logp_big[i]) + alpha * log(iv);
    return true;
  };
  if (k <= kBlendCache) {
    // up to kBlendCache views: the contributor terms and weights computed once
    // and kept in registers (the same values as the recomputing path below)
    double lt[kBlendCache], wt[kBlendCache];
    int who[kBlendCache];
    int m = 0;
    double peak = -INFINITY;
#pragma unroll
    for (int i = 0; i < kBlendCache; ++i) {
      if (i >= k) break;
      double l;
      if (!term(i, l)) continue;
      lt[m] = l;
      who[m] = i;
      peak = peak < l ? l : peak;  // std::max(peak, l)
      ++m;
    }
    if (m == 0) return;
    double sum = 0.0;
    for (int j = 0; j < m; ++j) sum += exp(lt[j] - peak);
    const double log_denom = peak + log(sum);
    if (!(log_denom > log_eps)) return;
    const double shrink = 1.0 / (1.0 + exp(log_eps - log_denom));
    for (int j = 0; j < m; ++j) wt[j] = exp(lt[j] - log_denom);
    for (int ch = 0; ch < c; ++ch) {
      double acc = 0.0;
      for (int j = 0; j < m; ++j) acc += wt[j] * static_cast<double>(colors[(who[j] * n + t) * c + ch]);
      out[t * c + ch] = static_cast<float>(acc * shrink);
    }
    filled[t] = 1;
    return;
  }
  int m = 0;
  double peak = -INFINITY;
  for (int i = 0; i < k; ++i) {
    double l;
    if (!term(i, l)) continue;
    peak = peak < l ? l : peak;  // std::max(peak, l)
    ++m;
  }
  if (m == 0) return;
  double sum = 0.0;
  for (int i = 0; i < k; ++i) {
    double l;
    if (term(i, l)) sum += exp(l - peak);
  }
  const double log_denom = peak + log(sum);
  if (!(log_denom > log_eps)) return;
  const double shrink = 1.0 / (1.0 + exp(log_eps - log_denom));
  for (int ch = 0; ch < c; ++ch) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) {
      double l;
      if (term(i, l)) acc += exp(l - log_denom) * static_cast<double>(colors[(i * n + t) * c + ch]);
    }
    out[t * c + ch] = static_cast<float>(acc * shrink);
  }
  filled[t] = 1;
}

constexpr int kThreads = 256;
int blocks(int64_t n) { return static_cast<int>(std::max<int64_t>(1, (n + kThreads - 1) / kThreads)); }

// reductionKernel (mips.cpp:21-33), with the reference's libm calls on the host
Taps8 lanczos_taps() {
  auto sinc = [](double x) {
    if (x == 0.0) return 1.0;
    const double px = M_PI * x;
    return std::sin(px) / px;
  };
  Taps8 k{};
  double sum = 0.0;
  for (int d = -3; d <= 4; ++d) {
    const double t = (d - 0.5) / 2.0;
    k.k[d + 3] = sinc(t) * sinc(t / 2.0);
    sum += k.k[d + 3];
  }
  for (double& w : k.k) w /= sum;
  return k;
}

}  // namespace

TfCamera tf_camera(const double* cam7, int res) {
  TfCamera c;
  for (int k = 0; k < 3; ++k) {
    c.dir[k] = cam7[k];
    c.up[k] = cam7[3 + k];
  }
  // right() = direction.cross(up) (render/camera.h:18)
  c.right[0] = c.dir[1] * c.up[2] - c.dir[2] * c.up[1];
  c.right[1] = c.dir[2] * c.up[0] - c.dir[0] * c.up[2];
  c.right[2] = c.dir[0] * c.up[1] - c.dir[1] * c.up[0];
  c.he = cam7[6];
  c.res = res;
  return c;
}

int tf_mip_layout(int w, int h, int c, int levels, int* lw, int* lh, int64_t* off) {
  int n = 0;
  int64_t o = 0;
  while (n < levels && n < kTfMaxMips) {
    if (n > 0 && lw[n - 1] == 1 && lh[n - 1] == 1) break;
    lw[n] = n == 0 ? w : std::max(1, (lw[n - 1] + 1) / 2);
    lh[n] = n == 0 ? h : std::max(1, (lh[n - 1] + 1) / 2);
    off[n] = o;
    o += static_cast<int64_t>(lw[n]) * lh[n] * c;
    ++n;
  }
  off[n] = o;
  return n;
}

void tf_edge_mask(Ctx& ctx, cudaStream_t s, int w, int h, const float* pos, const int32_t* face, double limit2,
                  uint8_t* mask) {
  const int64_t n = static_cast<int64_t>(w) * h;
  k_edge_mask<<<blocks(n), kThreads, 0, s>>>(w, h, pos, face, limit2, mask);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

int tf_build_mips(Ctx& ctx, cudaStream_t s, int w, int h, int c, const float* base, int levels, float sharpen,
                  float* chain, const std::string& tag) {
  int lw[kTfMaxMips + 1], lh[kTfMaxMips + 1];
  int64_t off[kTfMaxMips + 1];
  const int n = tf_mip_layout(w, h, c, levels, lw, lh, off);
  if (chain != base)
    MFB_CUDA_TRY(cudaMemcpyAsync(chain, base, sizeof(float) * off[1], cudaMemcpyDeviceToDevice, s));
  const Taps8 kt = lanczos_taps();
  for (int l = 1; l < n; ++l) {
    const int pw = lw[l - 1], ph = lh[l - 1], ow = lw[l], oh = lh[l];
    float* hx = ctx.buf<float>(tag + ".hx", static_cast<size_t>(ow) * ph * c);
    float* out = chain + off[l];
    k_halve_x<<<blocks(static_cast<int64_t>(ow) * ph * c), kThreads, 0, s>>>(pw, ph, c, chain + off[l - 1], hx, kt);
    if (sharpen == 0.0f) {
      k_halve_y<<<blocks(static_cast<int64_t>(ow) * oh * c), kThreads, 0, s>>>(ow, ph, c, hx, out, kt);
      ctx.count_launch(2);
    } else {
      float* hy = ctx.buf<float>(tag + ".hy", static_cast<size_t>(ow) * oh * c);
      float* bx = ctx.buf<float>(tag + ".bx", static_cast<size_t>(ow) * oh * c);
      k_halve_y<<<blocks(static_cast<int64_t>(ow) * oh * c), kThreads, 0, s>>>(ow, ph, c, hx, hy, kt);
      k_blur_x<<<blocks(static_cast<int64_t>(ow) * oh * c), kThreads, 0, s>>>(ow, oh, c, hy, bx);
      k_unsharp<<<blocks(static_cast<int64_t>(ow) * oh * c), kThreads, 0, s>>>(ow, oh, c, hy, bx, sharpen, out);
      ctx.count_launch(4);
    }
    MFB_CUDA_TRY(cudaGetLastError());
  }
  return n;
}

void tf_valid_bounds(Ctx& ctx, cudaStream_t s, int64_t n, const float* pos, const uint8_t* valid, unsigned* b6) {
  static const unsigned init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
  MFB_CUDA_TRY(cudaMemcpyAsync(b6, init, sizeof(init), cudaMemcpyHostToDevice, s));
  const int g = std::min<int64_t>(blocks(n), 4 * kNumSMs);
  k_valid_bounds<<<g, kThreads, 0, s>>>(n, pos, valid, b6);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void tf_backproject(Ctx& ctx, cudaStream_t s, int gres, const float* pos, const uint8_t* valid, const unsigned* b6,
                    const TfCamera& cam, int channels, int n_mips, const float* chain, const uint8_t* mask,
                    float* color, uint8_t* sampled) {
  MipChain mc;
  int lw[kTfMaxMips + 1], lh[kTfMaxMips + 1];
  int64_t off[kTfMaxMips + 1];
  mc.n = tf_mip_layout(cam.res, cam.res, channels, n_mips, lw, lh, off);
  if (mc.n != n_mips) throw ApiError(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: mip chain length does not match the view");
  mc.base = chain;
  mc.c = channels;
  for (int l = 0; l < mc.n; ++l) {
    mc.w[l] = lw[l];
    mc.h[l] = lh[l];
    mc.off[l] = off[l];
  }
  const int64_t n = static_cast<int64_t>(gres) * gres;
  k_backproject<<<static_cast<int>((n + 127) / 128), 128, 0, s>>>(gres, pos, valid, b6, cam, mc, mask, color, sampled);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void tf_incidence(Ctx& ctx, cudaStream_t s, int gres, const float* pos, const float* nrm, const uint8_t* valid,
                  const TfCamera& cam, const float* depth, double tolerance, float* out) {
  const int64_t n = static_cast<int64_t>(gres) * gres;
  k_incidence<<<blocks(n), kThreads, 0, s>>>(gres, pos, nrm, valid, cam, depth, tolerance, out);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void tf_blend(Ctx& ctx, cudaStream_t s, int k, int64_t n, int c, const float* colors, const uint8_t* sampled,
              const float* inc, const double* priors_host, double alpha, double epsilon, float* out,
              uint8_t* filled) {
  // log(prior) and log(epsilon) with the reference's own libm (fuse.cpp:246, :255)
  // log(prior) per view as a kernel parameter (no host -> device copy on the
  // stream) for up to kParamViews views; more views go through device scratch
  BlendParams bp{};
  const int kp = std::min(k, kParamViews);
  for (int i = 0; i < kp; ++i) {
    bp.pos[i] = priors_host[i] > 0.0 ? 1 : 0;
    bp.lp[i] = bp.pos[i] ? std::log(priors_host[i]) : 0.0;
  }
  double* dlp = nullptr;
  uint8_t* dpos = nullptr;
  if (k > kParamViews) {
    std::vector<double> lp(k);
    std::vector<uint8_t> pos(k);
    for (int i = 0; i < k; ++i) {
      pos[i] = priors_host[i] > 0.0 ? 1 : 0;
      lp[i] = pos[i] ? std::log(priors_host[i]) : 0.0;
    }
    dlp = ctx.buf<double>("tf.logp", k);
    dpos = ctx.buf<uint8_t>("tf.ppos", k);
    MFB_CUDA_TRY(cudaMemcpyAsync(dlp, lp.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
    MFB_CUDA_TRY(cudaMemcpyAsync(dpos, pos.data(), k, cudaMemcpyHostToDevice, s));
  }
  k_blend<<<blocks(n), kThreads, 0, s>>>(k, n, c, colors, sampled, inc, bp, dlp, dpos, alpha, std::log(epsilon),
                                         out, filled);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

}  // namespace mfb
