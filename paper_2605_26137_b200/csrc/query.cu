// query.cu — bounded closest-point traversal (Bvh::closestPointWithin,
// spatial/bvh.cpp:151-176) fused with the tangent-space transfer epilogue of
// transferNormals (bake/gbuffer.cpp:215-250), plus the bulk closest-point and
// raycastFirst (bvh.cpp:100-140) kernels.
//
// Exactness: the triangle test is the reference's f64 closestPointTriangle
// (tri_geom.h:37-95) evaluated in the same order without FMA, and the winner
// is argmin over (distSq, face) exactly as `improves` (bvh.cpp:17-23). The
// traversal order is depth-first nearest-child-first instead of the
// reference's heap, which is result-neutral because node pruning is
// conservative: fp32 child boxes rounded outward, fp32 lower bounds computed
// with round-down intrinsics, compared against an upper bound of the current
// best inflated by the scene-scale f64 error slack.
#include <algorithm>
#include <cmath>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "bake.cuh"

namespace mfb {
namespace {

__device__ __forceinline__ double from_ordered_dev(unsigned long long b) {
  b = (b & 0x8000000000000000ull) ? (b & ~0x8000000000000000ull) : ~b;
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ unsigned long long ordered_bits_dev(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// Upper bound (as float) on the squared distance any face that can still win
// may have, given the incumbent `best` and slack E: (sqrt(best) + E)^2.
__device__ __forceinline__ float prune_bound(double best, double E) {
  if (isnan(best) || best < 0.0) return -INFINITY;  // nothing can improve on NaN or -inf
  if (isinf(best)) return INFINITY;
  const double r = sqrt(best) + E;
  return __double2float_ru(r * r * (1.0 + 0x1p-30));
}

// One 64-byte node record in two 256-bit read-only loads (LDG.E.256 on
// sm_100).
__device__ __forceinline__ void ld_node(const BNode* __restrict__ nd, float4& a, float4& b, float4& c, int4& d) {
  const float* p = reinterpret_cast<const float*>(nd);
  float dx, dy, dz, dw;
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(c.x), "=f"(c.y), "=f"(c.z), "=f"(c.w), "=f"(dx), "=f"(dy), "=f"(dz), "=f"(dw)
               : "l"(p + 8));
  d = make_int4(__float_as_int(dx), __float_as_int(dy), __float_as_int(dz), __float_as_int(dw));
}

// Lower bound of the squared distance from [qlo, qhi] (per axis) to a box.
__device__ __forceinline__ float box_lb(float mnx, float mny, float mnz, float mxx, float mxy,
                                        float mxz, float3 qlo, float3 qhi) {
  const float dx = fmaxf(fmaxf(__fsub_rd(mnx, qhi.x), __fsub_rd(qlo.x, mxx)), 0.0f);
  const float dy = fmaxf(fmaxf(__fsub_rd(mny, qhi.y), __fsub_rd(qlo.y, mxy)), 0.0f);
  const float dz = fmaxf(fmaxf(__fsub_rd(mnz, qhi.z), __fsub_rd(qlo.z, mxz)), 0.0f);
  // fused multiply-adds rounded down: one rounding each, still a lower bound
  // (2 instructions fewer per box than separate products and sums)
  return __fmaf_rd(dz, dz, __fmaf_rd(dy, dy, __fmul_rd(dx, dx)));
}

// Both children's box lower bounds from one node (BNode's interleaved
// (left, right) coordinate pairs) with packed f32x2 arithmetic: per axis two
// FADD2.RM against the broadcast query coordinate, one FMNMX3 per child, then
// FMUL2.RM + 2 FFMA2.RM - 15 instructions instead of box_lb's 24, the same
// round-down operations in the same order (bit-identical bounds).
typedef unsigned long long u64x;
__device__ __forceinline__ u64x pk2(float lo, float hi) {
  u64x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(u64x v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64x sub_rd2(u64x a, u64x b) {
  u64x r;
  asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64x mul_rd2(u64x a, u64x b) {
  u64x r;
  asm("mul.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64x fma_rd2(u64x a, u64x b, u64x c) {
  u64x r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ void box_lb2(const float4& a, const float4& b, const float4& c, float3 q, float& lbL,
                                        float& lbR) {
  const u64x qx = pk2(q.x, q.x), qy = pk2(q.y, q.y), qz = pk2(q.z, q.z);
  float l0, l1, h0, h1;
  upk2(sub_rd2(pk2(a.x, a.y), qx), l0, l1);  // min - q
  upk2(sub_rd2(qx, pk2(b.z, b.w)), h0, h1);  // q - max
  const float dxL = fmaxf(fmaxf(l0, h0), 0.0f), dxR = fmaxf(fmaxf(l1, h1), 0.0f);
  upk2(sub_rd2(pk2(a.z, a.w), qy), l0, l1);
  upk2(sub_rd2(qy, pk2(c.x, c.y)), h0, h1);
  const float dyL = fmaxf(fmaxf(l0, h0), 0.0f), dyR = fmaxf(fmaxf(l1, h1), 0.0f);
  upk2(sub_rd2(pk2(b.x, b.y), qz), l0, l1);
  upk2(sub_rd2(qz, pk2(c.z, c.w)), h0, h1);
  const float dzL = fmaxf(fmaxf(l0, h0), 0.0f), dzR = fmaxf(fmaxf(l1, h1), 0.0f);
  const u64x dx = pk2(dxL, dxR), dy = pk2(dyL, dyR), dz = pk2(dzL, dzR);
  upk2(fma_rd2(dz, dz, fma_rd2(dy, dy, mul_rd2(dx, dx))), lbL, lbR);
}

// spatial/tri_geom.h:37-95 — same branch order, same expression order.
__device__ __forceinline__ d3 closest_point_triangle(d3 p, d3 a, d3 b, d3 c, d3& bary) {
  const d3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    bary = mk3(1.0, 0.0, 0.0);
    return a;
  }
  const d3 bp = p - b;
  const double d3_ = dot(ab, bp), d4 = dot(ac, bp);
  if (d3_ >= 0.0 && d4 <= d3_) {
    bary = mk3(0.0, 1.0, 0.0);
    return b;
  }
  const double vc = d1 * d4 - d3_ * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) {
    const double w = d1 / (d1 - d3_);
    bary = mk3(1.0 - w, w, 0.0);
    return a + w * ab;
  }
  const d3 cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) {
    bary = mk3(0.0, 0.0, 1.0);
    return c;
  }
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double w = d2 / (d2 - d6);
    bary = mk3(1.0 - w, 0.0, w);
    return a + w * ac;
  }
  const double va = d3_ * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3_) >= 0.0 && (d5 - d6) >= 0.0) {
    const double w = (d4 - d3_) / ((d4 - d3_) + (d5 - d6));
    bary = mk3(0.0, 1.0 - w, w);
    return b + w * (c - b);
  }
  const double denom = 1.0 / ((va + vb) + vc);
  const double wb = vb * denom, wc = vc * denom;
  bary = mk3((1.0 - wb) - wc, wb, wc);
  return (a + ab * wb) + ac * wc;
}

// Branch-free form of closestPointTriangle for the SIMT pair rounds: every
// lane evaluates all Voronoi-region predicates in the reference's order and
// then the one formula of its region, with a single shared f64 division
// (num / den selected per region: edge weight, or 1 / (va + vb + vc) for the
// interior). Each region's outputs are computed with exactly the expressions
// of tri_geom.h:37-95 (selects, never "+ 0"), so results are bit-identical to
// closest_point_triangle; only the control flow differs.
__device__ __forceinline__ d3 closest_point_triangle_sel(d3 p, d3 a, d3 b, d3 c, d3& bary) {
  const d3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  const d3 bp = p - b;
  const double d3_ = dot(ab, bp), d4 = dot(ac, bp);
  const d3 cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  const double vc = d1 * d4 - d3_ * d2;
  const double vb = d5 * d2 - d1 * d6;
  const double va = d3_ * d6 - d5 * d4;
  const double e43 = d4 - d3_, e56 = d5 - d6;
  // region: 0 A, 1 B, 2 AB, 3 C, 4 AC, 5 BC, 6 interior (reference test order)
  int r;
  if (d1 <= 0.0 && d2 <= 0.0) r = 0;
  else if (d3_ >= 0.0 && d4 <= d3_) r = 1;
  else if (vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) r = 2;
  else if (d6 >= 0.0 && d5 <= d6) r = 3;
  else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) r = 4;
  else if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) r = 5;
  else r = 6;
  const double num = r == 2 ? d1 : (r == 4 ? d2 : (r == 5 ? e43 : 1.0));
  const double den = r == 2 ? (d1 - d3_) : (r == 4 ? (d2 - d6) : (r == 5 ? (e43 + e56) : ((va + vb) + vc)));
  const double w = (r == 0 || r == 1 || r == 3) ? 0.0 : num / den;
  const double wb = vb * w, wc = vc * w;  // interior weights (only used when r == 6)
  // edge / interior first step: base + dir * s
  const d3 cb = c - b;
  const d3 base = r == 5 ? b : a;
  const d3 dir = r == 4 ? ac : (r == 5 ? cb : ab);
  const double sc = r == 6 ? wb : w;
  d3 pt;
  if (r == 6) {
    pt = (base + dir * sc) + ac * wc;  // (a + ab*wb) + ac*wc
  } else {
    // a + w*ab, a + w*ac, b + w*(c-b): scalar*vector, same rounding as dir*w
    pt = base + sc * dir;
  }
  pt = r == 0 ? a : (r == 1 ? b : (r == 3 ? c : pt));
  const double om = 1.0 - w;
  bary = r == 0 ? mk3(1.0, 0.0, 0.0)
       : r == 1 ? mk3(0.0, 1.0, 0.0)
       : r == 3 ? mk3(0.0, 0.0, 1.0)
       : r == 2 ? mk3(om, w, 0.0)
       : r == 4 ? mk3(om, 0.0, w)
       : r == 5 ? mk3(0.0, om, w)
                : mk3((1.0 - wb) - wc, wb, wc);
  return pt;
}

struct Best {
  double d;
  int face;
  d3 bary;
  d3 point;
};

__device__ __forceinline__ void load_tri(const BTri* __restrict__ t, d3& a, d3& b, d3& c, int& face) {
  const double2* p = reinterpret_cast<const double2*>(t);
  const double2 r0 = __ldg(p + 0), r1 = __ldg(p + 1), r2 = __ldg(p + 2), r3 = __ldg(p + 3);
  const double2 r4 = __ldg(p + 4);
  a = mk3(r0.x, r0.y, r1.x);
  b = mk3(r1.y, r2.x, r2.y);
  c = mk3(r3.x, r3.y, r4.x);
  face = __double_as_longlong(r4.y) & 0xffffffff;
}

// Depth-first, nearest-child-first bounded closest point. `best` must be
// initialised by the caller (d = maxDist^2 or +inf, face = -1).
template <bool kPoint>
__device__ __forceinline__ void traverse_closest(const BNode* __restrict__ nodes,
                                                 const BTri* __restrict__ tris, int32_t root, d3 q,
                                                 float3 qlo, float3 qhi, double E, Best& best) {
  float bnd = prune_bound(best.d, E);
  int32_t st_ref[kStackMax];
  float st_lb[kStackMax];
  int sp = 0;
  int32_t ref = root;
  for (;;) {
    if (ref >= 0) {
      const float4* np = reinterpret_cast<const float4*>(nodes + ref);
      const float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
      const int4 d = __ldg(reinterpret_cast<const int4*>(np + 3));
      const float lbL = box_lb(a.x, a.z, b.x, b.z, c.x, c.z, qlo, qhi);
      const float lbR = box_lb(a.y, a.w, b.y, b.w, c.y, c.w, qlo, qhi);
      const bool hL = lbL <= bnd, hR = lbR <= bnd;
      if (hL && hR) {
        const bool lf = lbL <= lbR;
        st_ref[sp] = lf ? d.y : d.x;
        st_lb[sp] = lf ? lbR : lbL;
        ++sp;
        ref = lf ? d.x : d.y;
        continue;
      }
      if (hL) {
        ref = d.x;
        continue;
      }
      if (hR) {
        ref = d.y;
        continue;
      }
    } else {
      int first, count;
      leaf_decode(ref, first, count);
      for (int i = 0; i < count; ++i) {
        d3 A, B, C;
        int face;
        load_tri(tris + first + i, A, B, C, face);
        d3 bary;
        const d3 pt = closest_point_triangle(q, A, B, C, bary);
        const double ds = sqnorm(pt - q);
        if (ds < best.d || (ds == best.d && face < best.face)) {
          best.d = ds;
          best.face = face;
          best.bary = bary;
          if (kPoint) best.point = pt;
          bnd = prune_bound(ds, E);
        }
      }
    }
    bool found = false;
    while (sp > 0) {
      --sp;
      if (st_lb[sp] <= bnd) {
        ref = st_ref[sp];
        found = true;
        break;
      }
    }
    if (!found) break;
  }
}


// ---------------------------------------------------------------- per-thread while-while transfer
// One query per thread over the compacted, spatially coherent query list.
// Aila-Laine "while-while" structure: each lane descends internal nodes until
// it holds a leaf (or finishes); the leaf loop then runs with every lane that
// holds one, so the expensive exact f64 test executes at high SIMT width.
// Depth-first nearest-child-first with conservative fp32 pruning (see
// traverse_closest) - result-neutral vs the reference's best-first heap.
// The triangle test's form per bake (template kSel of k_transfer_t): the
// branch-free one for leaves of <= 3 triangles (config B transfer 0.994 vs
// 1.005 ms), the branchy one for the larger leaves of a wide search
// (config E, leaves up to 11: 49.2 vs 54.6 ms). Measured and removed (numbers
// in DESIGN.md): L1 prefetch hints, per-triangle fp32 box pre-test, quad-seeded
// two-pass lists, carrying the incumbent's barycentrics through the walk.

// Pop of the per-thread stack that skips entries whose lower bound no longer
// passes `bnd` four at a time: one aligned 16-byte local load covers the top
// (up to) four lower bounds, so a run of pruned entries costs one dependent
// L1 round trip per four entries instead of one per entry. Returns the
// topmost surviving entry's ref (sp = its slot) or kDoneRef (sp = 0).
// Query records are read once: loaded evict-first (__ldcs) so they do not
// displace node / triangle lines from L1 (1.008 -> 1.005 ms transfer at B).
constexpr int32_t kDoneRef = static_cast<int32_t>(0x80000000);
__device__ __forceinline__ int32_t pop_within(const int32_t* st_ref, const float* st_lb, int& sp, float bnd) {
  while (sp > 0) {
    const int base = (sp - 1) & ~3;
    const float4 v = *reinterpret_cast<const float4*>(st_lb + base);
    unsigned m = (v.x <= bnd ? 1u : 0u) | (v.y <= bnd ? 2u : 0u) | (v.z <= bnd ? 4u : 0u) | (v.w <= bnd ? 8u : 0u);
    m &= (1u << (sp - base)) - 1u;
    if (m) {
      const int top = base + 31 - __clz(m);
      sp = top;
      return st_ref[top];
    }
    sp = base;
  }
  return kDoneRef;
}

// Triangle pre-test of the wide searches (Lbvh::tplane, built for leaf caps
// >= kPlaneLeafMin): a lower bound of the distance from q to the triangle from
// its containment slab and edge half-spaces in fp32; the exact f64 test is
// skipped when that bound, less the slack 2^-16 M (M = the scene/query
// magnitude behind E = M 2^-32; it covers the fp32 evaluation and the rounded
// vectors' departure from unit length and orthogonality, a few 2^-23 M),
// already exceeds the pruning bound. Result-neutral like node pruning: a
// skipped face is farther than any face that can still win.
__device__ __forceinline__ bool tri_plane_skip(const TPlane* tp, float3 q, float bnd, float E) {
  // (80-byte records: 16-byte aligned, five 128-bit loads)
  const float4 a = __ldg(&tp->m0), b = __ldg(&tp->m1), c = __ldg(&tp->m2), nn = __ldg(&tp->n);
  const float hi = __ldg(&tp->hi.x);
  const float m0x = a.x, m0y = a.y, m0z = a.z, o0 = a.w, m1x = b.x, m1y = b.y, m1z = b.z, o1 = b.w;
  const float m2x = c.x, m2y = c.y, m2z = c.z, o2 = c.w, nx = nn.x, ny = nn.y, nz = nn.z, lo = nn.w;
  const float s0 = fmaf(m0z, q.z, fmaf(m0y, q.y, m0x * q.x)) - o0;
  const float s1 = fmaf(m1z, q.z, fmaf(m1y, q.y, m1x * q.x)) - o1;
  const float s2 = fmaf(m2z, q.z, fmaf(m2y, q.y, m2x * q.x)) - o2;
  const float nq = fmaf(nz, q.z, fmaf(ny, q.y, nx * q.x));
  const float delta = E * 65536.0f;
  const float hh = fmaxf(__fsub_rd(fmaxf(lo - nq, nq - hi), delta), 0.0f);
  const float ss = fmaxf(__fsub_rd(fmaxf(s0, fmaxf(s1, s2)), delta), 0.0f);
  return __fmaf_rd(ss, ss, __fmul_rd(hh, hh)) > bnd;
}

// Leaf pre-test (Lbvh::lplane): the leaf's oriented box, same slack as
// tri_plane_skip; skips every triangle of a leaf that cannot hold a winner.
#pragma nv_diag_suppress 550  // the second load's padding lane is not used
__device__ __forceinline__ bool leaf_skip(const LPlane* lp, float3 q, float bnd, float E) {
  const float* p = reinterpret_cast<const float*>(lp);
  float nx, ny, nz, lo, hi, ux, uy, uz, umin, umax, vx, vy, vz, vmin, vmax, pad;
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(nx), "=f"(ny), "=f"(nz), "=f"(lo), "=f"(hi), "=f"(ux), "=f"(uy), "=f"(uz)
      : "l"(p));
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(umin), "=f"(umax), "=f"(vx), "=f"(vy), "=f"(vz), "=f"(vmin), "=f"(vmax), "=f"(pad)
      : "l"(p + 8));
  (void)pad;
  const float nq = fmaf(nz, q.z, fmaf(ny, q.y, nx * q.x));
  const float uq = fmaf(uz, q.z, fmaf(uy, q.y, ux * q.x));
  const float vq = fmaf(vz, q.z, fmaf(vy, q.y, vx * q.x));
  const float delta = E * 65536.0f;
  const float a = fmaxf(__fsub_rd(fmaxf(lo - nq, nq - hi), delta), 0.0f);
  const float b = fmaxf(__fsub_rd(fmaxf(umin - uq, uq - umax), delta), 0.0f);
  const float c = fmaxf(__fsub_rd(fmaxf(vmin - vq, vq - vmax), delta), 0.0f);
  return __fmaf_rd(c, c, __fmaf_rd(b, b, __fmul_rd(a, a))) > bnd;
}
#pragma nv_diag_default 550

// Row-band completion (BandSync, bake.cuh). Band b is complete once all its
// queries are done; its rows are final once b-1, b, b+1 (those that exist)
// are complete. The caller has fenced its stores.
// (rare path: full fences are fine here)
__device__ __forceinline__ void band_complete(const BandSync& bs, int band) {
  for (int k = max(0, band - 1); k <= min(bs.nb - 1, band + 1); ++k) {
    const int need = 1 + (k > 0) + (k < bs.nb - 1);
    __threadfence();
    if (atomicAdd(&bs.nbr[k], 1) + 1 == need) {
      __threadfence_system();
      atomicExch(&bs.ready[k], 1);
    }
  }
}
// Per-batch publication: a release add (MEMBAR.GPU + atomic). __threadfence
// here would be MEMBAR.SC + CCTL.IVALL - an L1 invalidation per batch that
// costs the walk its cached nodes (measured +40 us per transfer). The other
// lanes' stores are ordered before the leader's release by __syncwarp.
__device__ __forceinline__ int atom_add_release_gpu(int* p, int v) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void band_arrive(const BandSync& bs, int band, int n) {
  const int old = atom_add_release_gpu(&bs.done[band], n);
  if (old + n == __ldcg(bs.tot + band)) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire the other publishers' releases
    band_complete(bs, band);
  }
}
__global__ void k_band_init(BandSync bs) {
  for (int b = threadIdx.x; b < bs.nb; b += blockDim.x)
    if (bs.tot[b] == 0) band_complete(bs, b);
}

// Occupancy over registers: the walk is bound by dependent L1/L2 latency
// (node record -> box test -> child record), so resident warps matter more
// than the spills a 64-register cap costs. Measured at config B (transfer
// ms): no cap (92 regs, 5 blocks/SM) 1.34, 6 blocks 1.24, 7 blocks 1.19,
// 8 blocks (64 regs) 1.15, 9 blocks 1.23, 10 blocks 1.50.
#ifndef MFB_XFER_T_MINB
#define MFB_XFER_T_MINB 8
#endif
// The wide-leaf instantiations (kSel false: f64 triangle tests dominate)
// run best at 7 (config E per bake: 6 / 7 / 8 / 9 CTAs 46.4 / 43.0 / 44.3 /
// 46.7 ms).
#if MFB_XFER_T_MINB > 0
#define MFB_XFER_T_BOUNDS __launch_bounds__(128, kSel ? MFB_XFER_T_MINB : 7)
#else
#define MFB_XFER_T_BOUNDS __launch_bounds__(128)
#endif
// kBands: the row-band publication of the host path's overlapped download
// (compiled only into that instantiation: it costs the walk registers)
template <bool kDebug, bool kProf, bool kBands = false, bool kSel = true>
__global__ void MFB_XFER_T_BOUNDS k_transfer_t(
    const BNode* __restrict__ nodes, const BTri* __restrict__ tris, int32_t root,
    const unsigned long long* __restrict__ scene_acc, const float4* __restrict__ qpos,
    const float* __restrict__ qtbn, const int* __restrict__ qcount, const double* __restrict__ hiN,
    const int32_t* __restrict__ hiF, double max_dist, uint8_t* __restrict__ rgb,
    int32_t* __restrict__ dbg_face, double* __restrict__ dbg_ts, unsigned long long* __restrict__ counters,
    unsigned long long* __restrict__ prof_out, const double* __restrict__ hiPos = nullptr,
    const int* __restrict__ dep_head = nullptr,
    const int* __restrict__ dep_next = nullptr, BandSync bands = BandSync{}, int fmt = MF_ATLAS_RGB8,
    const TPlane* __restrict__ tplane = nullptr, const LPlane* __restrict__ lplane = nullptr,
    const LPlane* __restrict__ nplane = nullptr) {
  const int nq = qcount[0];
  const int lane = threadIdx.x & 31;
  if (kProf && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&prof_out[4], t);
  }
  unsigned long long pv[5] = {0, 0, 0, 0, 0};  // internal visits, leaf visits, leaf triangles, queries, exact tests
  const double scene_max = from_ordered_dev(scene_acc[6]);
  const double init = isinf(max_dist) ? max_dist : max_dist * max_dist;  // bvh.cpp:153-154
  unsigned hits = 0;
  // Dynamic 32-query batches (single pass): lane 0 of each warp takes the
  // next batch from the list's cursor (qcount[3], zeroed by the producer), so
  // warps that drew cheap batches keep working instead of idling in the tail.
  // Measured at config B: transfer 1.055 -> 1.003 ms; config E 69.7 -> 62.1 ms.
  int* cursor = const_cast<int*>(qcount) + 3;
  auto next_batch = [&]() {
    int b = 0;
    if (lane == 0) b = atomicAdd(cursor, 1);
    return __shfl_sync(0xffffffffu, b, 0) * 32 + lane;
  };
  for (int li = next_batch(); li - lane < nq; li = next_batch()) {
    const bool live = li < nq;
    const int i = li;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) p = __ldcs(qpos + i);
    // a dead record (texel id stored as ~texel by k_interp: the texel's face
    // is unreliable) is not walked; its epilogue stores the (128, 128, 255)
    // of gbuffer.cpp:218-227 into the texel and the gutter texels linked to it
    const bool dead = live && __float_as_int(p.w) < 0;
    const float3 qf = make_float3(p.x, p.y, p.z);
    const d3 q = mk3(p.x, p.y, p.z);
    // pruning slack, rounded up to fp32 (conservative; one register)
    const float E = __double2float_ru(fmax(scene_max, fmax(fabs(q.x), fmax(fabs(q.y), fabs(q.z)))) * 0x1p-32);
    Best best;
    best.d = init;
    best.face = -1;
    best.bary = mk3(0.0, 0.0, 0.0);
    float bnd = live && !dead ? prune_bound(best.d, E) : -INFINITY;
    int32_t st_ref[kStackMax];
    alignas(16) float st_lb[kStackMax];
    int sp = 0;
    // ref: node (>= 0), leaf (< 0 and != kDone), or kDone
    constexpr int32_t kDone = static_cast<int32_t>(0x80000000);
    int32_t ref = live && !dead ? root : kDone;
    while (ref != kDone) {
      // ---- descend until this lane holds a leaf
      while (ref >= 0) {
        if (kProf) ++pv[0];
        float4 a, b, c;
        int4 d;
        ld_node(nodes + ref, a, b, c, d);
        // wide searches: the node's own oriented box (loaded beside the node)
        if (!kSel && nplane && leaf_skip(nplane + ref, qf, bnd, E)) {
          ref = pop_within(st_ref, st_lb, sp, bnd);
          continue;
        }
        float lbL, lbR;
        box_lb2(a, b, c, qf, lbL, lbR);
        const bool hL = lbL <= bnd, hR = lbR <= bnd;
        if (hL && hR) {
          const bool lf = lbL <= lbR;
          st_ref[sp] = lf ? d.y : d.x;
          st_lb[sp] = lf ? lbR : lbL;
          ++sp;
          ref = lf ? d.x : d.y;
        } else if (hL || hR) {
          ref = hL ? d.x : d.y;
        } else {
          ref = pop_within(st_ref, st_lb, sp, bnd);
        }
      }
      if (ref == kDone) break;
      // ---- leaf: exact f64 tests (branch-free, reference arithmetic)
      int first, count;
      leaf_decode(ref, first, count);
      if (kProf) {
        ++pv[1];
        pv[2] += count;
      }
      // (iterate [first, end): two live loop values instead of three, so the
      // loop state stays in registers under the 64-register cap)
      const int end = (!kSel && lplane && leaf_skip(lplane + first, qf, bnd, E)) ? first : first + count;
      for (int k = first; k < end; ++k) {
        if (!kSel && tplane && tri_plane_skip(tplane + k, qf, bnd, E)) continue;
        if (kProf) ++pv[4];
        d3 A, B, C;
        int face;
        load_tri(tris + k, A, B, C, face);
        d3 bary;
        const d3 ql = q;
        const d3 pt = kSel ? closest_point_triangle_sel(ql, A, B, C, bary) : closest_point_triangle(ql, A, B, C, bary);
        const double ds = sqnorm(pt - ql);
        if (ds < best.d || (ds == best.d && face < best.face)) {
          best.d = ds;
          best.face = face;
          bnd = prune_bound(ds, E);
        }
      }
      ref = pop_within(st_ref, st_lb, sp, bnd);
    }
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    const unsigned dead_mask = __ballot_sync(0xffffffffu, dead);
    if (counters && dead_mask && lane == __ffs(dead_mask) - 1)
      atomicAdd(&counters[3], static_cast<unsigned long long>(__popc(dead_mask)));
    if (!live) continue;
    if (kProf) ++pv[3];
    const int texel = dead ? ~__float_as_int(p.w) : __float_as_int(p.w);
    const d3 qe = q;
    uint32_t px = px_neutral(fmt);
    double ts3[3] = {0.0, 0.0, 0.0};
    if (best.face >= 0) {
      ++hits;
      const float* tb = qtbn + 9ll * i;
      const int v0 = hiF[3 * best.face], v1 = hiF[3 * best.face + 1], v2 = hiF[3 * best.face + 2];
      // the winner's barycentrics, recomputed (lean walk state): same inputs
      // (BTri holds copies of these positions), same function, same bits
      closest_point_triangle(qe, ld3(hiPos + 3 * v0), ld3(hiPos + 3 * v1), ld3(hiPos + 3 * v2), best.bary);
      const d3 n = (best.bary.x * ld3(hiN + 3 * v0) + best.bary.y * ld3(hiN + 3 * v1)) +
                   best.bary.z * ld3(hiN + 3 * v2);
      const d3 T = mk3(__ldcs(tb), __ldcs(tb + 1), __ldcs(tb + 2));
      const d3 B = mk3(__ldcs(tb + 3), __ldcs(tb + 4), __ldcs(tb + 5));
      const d3 N = mk3(__ldcs(tb + 6), __ldcs(tb + 7), __ldcs(tb + 8));
      d3 ts = mk3(dot(n, T), dot(n, B), dot(n, N));
      const double len = norm(ts);
      if (!(len < 1e-12)) {
        ts = ts / len;
        px = px_encode(fmt, ts.x, ts.y, ts.z);  // encodeChannel (gbuffer.cpp:85-88) per channel
        ts3[0] = ts.x;
        ts3[1] = ts.y;
        ts3[2] = ts.z;
      }
    }
    px_store(rgb, texel, fmt, px);
    if (dep_head) {  // dilation: the gutter texels whose source is this texel
      for (int t = __ldcs(dep_head + i); t >= 0; t = dep_next[t]) px_store(rgb, t, fmt, px);
    }
    if (kBands && bands.done) {  // this batch's texels (and their gutter texels) are written
      const int band = texel / bands.res / bands.rows;
      // (a batch can hold several raster tiles' segments: group by band)
      const unsigned grp = __match_any_sync(live_mask, band);
      __syncwarp(live_mask);
      if (lane == __ffs(grp) - 1) band_arrive(bands, band, __popc(grp));
    }
    if (kDebug) {
      if (dbg_face) dbg_face[texel] = dead ? -2 : (best.face >= 0 ? best.face : -3);
      if (dbg_ts) {
        dbg_ts[3ll * texel] = ts3[0];
        dbg_ts[3ll * texel + 1] = ts3[1];
        dbg_ts[3ll * texel + 2] = ts3[2];
      }
    }
  }
  if (kProf) {
    for (int k = 0; k < 5; ++k) {
      unsigned long long v = pv[k];
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) atomicAdd(&prof_out[k < 4 ? k : 7], v);
    }
    if (lane == 0) {  // warp exit times (tail spread): [5] first, [6] last, [4] kernel start
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMin(&prof_out[5], t);
      atomicMax(&prof_out[6], t);
    }
  }
  if (counters) {
    for (int off = 16; off > 0; off >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, off);
    if (lane == 0 && hits) atomicAdd(&counters[1], static_cast<unsigned long long>(hits));
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&counters[0], static_cast<unsigned long long>(nq));
  }
}

__global__ void __launch_bounds__(128) k_closest(const BNode* __restrict__ nodes,
                                                 const BTri* __restrict__ tris, int32_t root,
                                                 const unsigned long long* __restrict__ scene_acc,
                                                 const double* __restrict__ q, int64_t n,
                                                 double max_dist, int32_t* __restrict__ face,
                                                 double* __restrict__ dist_sq,
                                                 double* __restrict__ point,
                                                 double* __restrict__ bary) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d3 p = ld3(q + 3 * i);
  const float3 lo = make_float3(__double2float_rd(p.x), __double2float_rd(p.y), __double2float_rd(p.z));
  const float3 hi = make_float3(__double2float_ru(p.x), __double2float_ru(p.y), __double2float_ru(p.z));
  const double M = fmax(from_ordered_dev(scene_acc[6]), fmax(fabs(p.x), fmax(fabs(p.y), fabs(p.z))));
  Best best;
  best.d = isinf(max_dist) ? max_dist : max_dist * max_dist;
  best.face = -1;
  best.bary = mk3(0.0, 0.0, 0.0);
  best.point = mk3(0.0, 0.0, 0.0);
  if (!isnan(p.x) && !isnan(p.y) && !isnan(p.z))
    traverse_closest<true>(nodes, tris, root, p, lo, hi, M * 0x1p-32, best);
  if (best.face < 0) best.d = INFINITY;  // bvh.cpp:174
  face[i] = best.face;
  dist_sq[i] = best.d;
  if (point) st3(point + 3 * i, best.point);
  if (bary) st3(bary + 3 * i, best.bary);
}

// ---------------------------------------------------------------- ray cast
// core/aabb.h:45-56 slab test on an fp32 box, evaluated in f64 and widened by
// a relative slack so that no box containing an accepted hit is culled.
__device__ __forceinline__ bool slab(float mnx, float mny, float mnz, float mxx, float mxy, float mxz,
                                     d3 o, d3 inv, double tmin, double tmax, double slack,
                                     double& tnear) {
  const double mn[3] = {mnx, mny, mnz}, mx[3] = {mxx, mxy, mxz};
  const double oo[3] = {o.x, o.y, o.z}, iv[3] = {inv.x, inv.y, inv.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double t0 = (mn[a] - oo[a]) * iv[a];
    double t1 = (mx[a] - oo[a]) * iv[a];
    if (iv[a] < 0.0) {
      const double s = t0;
      t0 = t1;
      t1 = s;
    }
    t0 = t0 - (fabs(t0) + 1.0) * slack;
    t1 = t1 + (fabs(t1) + 1.0) * slack;
    tmin = t0 > tmin ? t0 : tmin;
    tmax = t1 < tmax ? t1 : tmax;
    if (tmax < tmin) return false;
  }
  tnear = tmin;
  return true;
}

// spatial/tri_geom.h:14-33 Moller-Trumbore in the reference's order.
__device__ __forceinline__ bool ray_triangle(d3 o, d3 d, d3 a, d3 b, d3 c, double& t, double& u,
                                             double& v) {
  const d3 e1 = b - a, e2 = c - a;
  const d3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  if (fabs(det) < 1e-9) return false;
  const double inv = 1.0 / det;
  const d3 sv = o - a;
  u = dot(sv, pv) * inv;
  if (u < 0.0 || u > 1.0) return false;
  const d3 qv = cross(sv, e1);
  v = dot(d, qv) * inv;
  if (v < 0.0 || u + v > 1.0) return false;
  t = dot(e2, qv) * inv;
  return true;
}

__global__ void __launch_bounds__(128) k_raycast(const BNode* __restrict__ nodes,
                                                 const BTri* __restrict__ tris, int32_t root,
                                                 const double* __restrict__ org,
                                                 const double* __restrict__ dir, int64_t n,
                                                 double tmin, double tmax, int32_t* __restrict__ face_out,
                                                 double* __restrict__ t_out, double* __restrict__ u_out,
                                                 double* __restrict__ v_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const d3 o = ld3(org + 3 * i), d = ld3(dir + 3 * i);
  const d3 inv = mk3(1.0 / d.x, 1.0 / d.y, 1.0 / d.z);
  const double slack = 0x1p-24;
  int bf = -1;
  double bt = INFINITY, bu = 0.0, bv = 0.0;
  int32_t st[kStackMax];
  int sp = 0;
  int32_t ref = root;
  for (;;) {
    const double limit = tmax < bt ? tmax : bt;
    if (ref >= 0) {
      const float4* np = reinterpret_cast<const float4*>(nodes + ref);
      const float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
      const int4 dd = __ldg(reinterpret_cast<const int4*>(np + 3));
      double tl = 0.0, tr = 0.0;
      const bool hl = slab(a.x, a.z, b.x, b.z, c.x, c.z, o, inv, tmin, limit, slack, tl);
      const bool hr = slab(a.y, a.w, b.y, b.w, c.y, c.w, o, inv, tmin, limit, slack, tr);
      if (hl && hr) {
        const bool lf = tl <= tr;
        st[sp++] = lf ? dd.y : dd.x;
        ref = lf ? dd.x : dd.y;
        continue;
      }
      if (hl) {
        ref = dd.x;
        continue;
      }
      if (hr) {
        ref = dd.y;
        continue;
      }
    } else {
      int first, count;
      leaf_decode(ref, first, count);
      for (int k = 0; k < count; ++k) {
        d3 A, B, C;
        int f;
        load_tri(tris + first + k, A, B, C, f);
        double t, u, v;
        if (ray_triangle(o, d, A, B, C, t, u, v) && t >= tmin && t <= tmax &&
            (t < bt || (t == bt && f < bf))) {
          bf = f;
          bt = t;
          bu = u;
          bv = v;
        }
      }
    }
    if (sp == 0) break;
    ref = st[--sp];
  }
  face_out[i] = bf;
  t_out[i] = bt;
  u_out[i] = bu;
  v_out[i] = bv;
}

// ---------------------------------------------------------------- brute force
// One CTA per query strides over all faces and reduces the lexicographic
// minimum (distSq, face) / (t, face) - the reference's O(F) oracles.
__global__ void __launch_bounds__(256) k_closest_brute(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                                       int nf, const double* __restrict__ q, int64_t n,
                                                       int32_t* __restrict__ face_out, double* __restrict__ dist_out,
                                                       double* __restrict__ point_out, double* __restrict__ bary_out) {
  const int64_t qi = blockIdx.x;
  if (qi >= n) return;
  const d3 p = ld3(q + 3 * qi);
  double bd = INFINITY;
  int bf = -1;
  d3 bp = mk3(0.0, 0.0, 0.0), bb = mk3(0.0, 0.0, 0.0);
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    d3 bary;
    const d3 pt = closest_point_triangle(p, ld3(pos + 3 * faces[3 * f]), ld3(pos + 3 * faces[3 * f + 1]),
                                         ld3(pos + 3 * faces[3 * f + 2]), bary);
    const double ds = sqnorm(pt - p);
    if (ds < bd || (ds == bd && f < bf)) {  // improves(), bvh.cpp:21-23 (bf = -1 never wins a tie)
      bd = ds;
      bf = f;
      bp = pt;
      bb = bary;
    }
  }
  __shared__ double sd[256];
  __shared__ int sf[256];
  sd[threadIdx.x] = bd;
  sf[threadIdx.x] = bf < 0 ? 0x7fffffff : bf;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double od = sd[threadIdx.x + w];
      const int of = sf[threadIdx.x + w];
      if (od < sd[threadIdx.x] || (od == sd[threadIdx.x] && of < sf[threadIdx.x])) {
        sd[threadIdx.x] = od;
        sf[threadIdx.x] = of;
      }
    }
    __syncthreads();
  }
  const int wf = sf[0];
  if (threadIdx.x == 0 && (wf == 0x7fffffff)) {
    face_out[qi] = -1;
    dist_out[qi] = INFINITY;
    if (point_out) st3(point_out + 3 * qi, mk3(0.0, 0.0, 0.0));
    if (bary_out) st3(bary_out + 3 * qi, mk3(0.0, 0.0, 0.0));
  }
  if (wf != 0x7fffffff && bf == wf) {
    face_out[qi] = bf;
    dist_out[qi] = bd;
    if (point_out) st3(point_out + 3 * qi, bp);
    if (bary_out) st3(bary_out + 3 * qi, bb);
  }
}

__global__ void __launch_bounds__(256) k_raycast_brute(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                                       int nf, const double* __restrict__ org,
                                                       const double* __restrict__ dir, int64_t n, double tmin,
                                                       double tmax, int32_t* __restrict__ face_out,
                                                       double* __restrict__ t_out, double* __restrict__ u_out,
                                                       double* __restrict__ v_out) {
  const int64_t qi = blockIdx.x;
  if (qi >= n) return;
  const d3 o = ld3(org + 3 * qi), d = ld3(dir + 3 * qi);
  double bt = INFINITY, bu = 0.0, bv = 0.0;
  int bf = -1;
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    double t, u, v;
    if (ray_triangle(o, d, ld3(pos + 3 * faces[3 * f]), ld3(pos + 3 * faces[3 * f + 1]),
                     ld3(pos + 3 * faces[3 * f + 2]), t, u, v) &&
        t >= tmin && t <= tmax && (t < bt || (t == bt && f < bf))) {  // testFace, bvh.cpp:25-34
      bt = t;
      bu = u;
      bv = v;
      bf = f;
    }
  }
  __shared__ double st[256];
  __shared__ int sf[256];
  st[threadIdx.x] = bt;
  sf[threadIdx.x] = bf < 0 ? 0x7fffffff : bf;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double ot = st[threadIdx.x + w];
      const int of = sf[threadIdx.x + w];
      if (ot < st[threadIdx.x] || (ot == st[threadIdx.x] && of < sf[threadIdx.x])) {
        st[threadIdx.x] = ot;
        sf[threadIdx.x] = of;
      }
    }
    __syncthreads();
  }
  const int wf = sf[0];
  if (threadIdx.x == 0 && wf == 0x7fffffff) {
    face_out[qi] = -1;
    t_out[qi] = INFINITY;
    u_out[qi] = 0.0;
    v_out[qi] = 0.0;
  }
  if (wf != 0x7fffffff && bf == wf) {
    face_out[qi] = bf;
    t_out[qi] = bt;
    u_out[qi] = bu;
    v_out[qi] = bv;
  }
}



// True when some leaf (range) box of the tree has a fp32 lower-bound distance
// to the query box [qlo, qhi] of at most `bnd` (depth-first, stops at the
// first such leaf).
__device__ __forceinline__ bool any_leaf_within(const BNode* __restrict__ nodes, int32_t root, float3 qlo,
                                                float3 qhi, float bnd) {
  if (root < 0) return true;
  int32_t st[kStackMax];
  int sp = 0;
  int32_t ref = root;
  for (;;) {
    const float4* np = reinterpret_cast<const float4*>(nodes + ref);
    const float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
    const int4 d = __ldg(reinterpret_cast<const int4*>(np + 3));
    const bool hL = box_lb(a.x, a.z, b.x, b.z, c.x, c.z, qlo, qhi) <= bnd;
    const bool hR = box_lb(a.y, a.w, b.y, b.w, c.y, c.w, qlo, qhi) <= bnd;
    if ((hL && d.x < 0) || (hR && d.y < 0)) return true;
    if (hL && hR) {
      st[sp++] = d.y;
      ref = d.x;
    } else if (hL || hR) {
      ref = hL ? d.x : d.y;
    } else {
      if (sp == 0) return false;
      ref = st[--sp];
    }
  }
}
// ---------------------------------------------------------------- surface band
// markSurfaceBand's voxel sweep (signfield/sign_grid.cpp:56-66): per voxel,
// Bvh::closestPointWithin(voxelCenter, truncation); distance = sqrt(distSq)
// stored as f32 and SurfaceBand (1) where it is below bandWorld, else the
// voxel keeps (Unknown, f32(truncation)). voxelCenter (sign_grid.h:30-32) is
// origin + voxelSize * (x + 0.5, ...), component by component, no FMA.
// Threads are mapped to 4x4x2 voxel bricks (one brick per warp) so a warp's
// queries are spatial neighbours; storage stays x-fastest.
__global__ void __launch_bounds__(128) k_surface_band(const BNode* __restrict__ nodes, const BTri* __restrict__ tris,
                                                      int32_t root, const unsigned long long* __restrict__ scene_acc,
                                                      int res, double ox, double oy, double oz, double h,
                                                      double truncation, double band_world,
                                                      uint8_t* __restrict__ labels, float* __restrict__ dist) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int bx = (res + 3) >> 2, by = (res + 3) >> 2, bz = (res + 1) >> 1;
  const int64_t brick = t >> 5;
  const int lane = static_cast<int>(t & 31);
  if (brick >= static_cast<int64_t>(bx) * by * bz) return;
  const int kx = static_cast<int>(brick % bx);
  const int ky = static_cast<int>((brick / bx) % by);
  const int kz = static_cast<int>(brick / (static_cast<int64_t>(bx) * by));
  const int x = kx * 4 + (lane & 3), y = ky * 4 + ((lane >> 2) & 3), z = kz * 2 + (lane >> 4);
  // Brick cull (warp-uniform): if no leaf box of the tree lies within the
  // truncation of the box spanning the brick's voxel centres, no voxel of
  // the brick can find a surface point (a leaf box's distance bounds its
  // triangles' from below), so every voxel keeps (Unknown, truncation).
  const double M0 = from_ordered_dev(scene_acc[6]);
  {
    const int x1 = min(kx * 4 + 3, res - 1), y1 = min(ky * 4 + 3, res - 1), z1 = min(kz * 2 + 1, res - 1);
    const double cx0 = ox + h * (kx * 4 + 0.5), cy0 = oy + h * (ky * 4 + 0.5), cz0 = oz + h * (kz * 2 + 0.5);
    const double cx1 = ox + h * (x1 + 0.5), cy1 = oy + h * (y1 + 0.5), cz1 = oz + h * (z1 + 0.5);
    const float3 blo = make_float3(__double2float_rd(cx0), __double2float_rd(cy0), __double2float_rd(cz0));
    const float3 bhi = make_float3(__double2float_ru(cx1), __double2float_ru(cy1), __double2float_ru(cz1));
    const double Mb = fmax(M0, fmax(fmax(fabs(cx0), fabs(cx1)), fmax(fmax(fabs(cy0), fabs(cy1)),
                                                                     fmax(fabs(cz0), fabs(cz1)))));
    const double t2 = isinf(truncation) ? truncation : truncation * truncation;
    if (!any_leaf_within(nodes, root, blo, bhi, prune_bound(t2, Mb * 0x1p-32))) {
      if (x < res && y < res && z < res) {
        const int64_t i = x + static_cast<int64_t>(res) * (y + static_cast<int64_t>(res) * z);
        labels[i] = 0;
        dist[i] = static_cast<float>(truncation);
      }
      return;
    }
  }
  if (x >= res || y >= res || z >= res) return;
  const d3 p = mk3(ox + h * (x + 0.5), oy + h * (y + 0.5), oz + h * (z + 0.5));
  const float3 lo = make_float3(__double2float_rd(p.x), __double2float_rd(p.y), __double2float_rd(p.z));
  const float3 hi = make_float3(__double2float_ru(p.x), __double2float_ru(p.y), __double2float_ru(p.z));
  const double M = fmax(M0, fmax(fabs(p.x), fmax(fabs(p.y), fabs(p.z))));
  Best best;
  best.d = isinf(truncation) ? truncation : truncation * truncation;  // bvh.cpp:153-154
  best.face = -1;
  best.bary = mk3(0.0, 0.0, 0.0);
  traverse_closest<false>(nodes, tris, root, p, lo, hi, M * 0x1p-32, best);
  const int64_t i = x + static_cast<int64_t>(res) * (y + static_cast<int64_t>(res) * z);  // sign_grid.h:27-29
  uint8_t lab = 0;
  float dv = static_cast<float>(truncation);
  if (best.face >= 0) {
    const double d = sqrt(best.d);  // SurfacePoint::distance (bvh.h:24)
    dv = static_cast<float>(d);
    if (d < band_world) lab = 1;
  }
  labels[i] = lab;
  dist[i] = dv;
}

// Exact vertex bounds of a mesh (core/mesh.cpp:12-16): acc[0..2] min, acc[3..5] max (ordered bits).
__global__ void k_vertex_bounds(const double* __restrict__ pos, int nv, unsigned long long* acc) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double c = pos[3 * v + k];
      mn[k] = c < mn[k] ? c : mn[k];
      mx[k] = mx[k] < c ? c : mx[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    for (int off = 16; off > 0; off >>= 1) {
      mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
      mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&acc[k], ordered_bits_dev(mn[k]));
      atomicMax(&acc[3 + k], ordered_bits_dev(mx[k]));
    }
  }
}

// ---------------------------------------------------------------- ortho views
// renderView (render/raster.cpp:12-102) as one pixel ray per thread through
// the LBVH. Per pixel the reference keeps, over faces in index order, the
// first face whose depth f32(-t) is strictly larger than the stored one: the
// winner is argmax f32(-t), ties to the lowest face, among faces whose
// Moller-Trumbore test (same expressions as rayTriangle, tri_geom.h:14-33)
// passes and whose padded pixel box (raster.cpp:53-61) holds the pixel. The
// ray is the full line (no t range). The walk prunes a box only when its
// slab entry exceeds -prev_f32(best depth): such faces cannot reach the
// stored depth, so the result is the reference's for any tree.
// castVisibility (visibility/visibility.cpp:13-59) adds one hit per won pixel
// to the winner's counter over all views.
struct ViewCam {
  double dir[3], up[3], right[3];
  double he, step;  // halfExtent, 2 * halfExtent / resolution
};

__global__ void __launch_bounds__(128) k_render_views(
    const BNode* __restrict__ nodes, const BTri* __restrict__ tris, int32_t root, const ViewCam* __restrict__ cams,
    int nviews, int res, int cull, unsigned long long* __restrict__ hits, int32_t* __restrict__ face_img,
    float* __restrict__ depth_img, float* __restrict__ pos_img, float* __restrict__ nrm_img,
    const int32_t* __restrict__ faces, const double* __restrict__ vnormals) {
  const int tiles_x = (res + 7) >> 3, tiles_y = (res + 3) >> 2;
  const int64_t per_view = static_cast<int64_t>(tiles_x) * tiles_y * 32;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int view = static_cast<int>(t / per_view);
  if (view >= nviews) return;
  const int64_t r = t - view * per_view;
  const int tile = static_cast<int>(r >> 5), lane = static_cast<int>(r & 31);
  const int px = (tile % tiles_x) * 8 + (lane & 7), py = (tile / tiles_x) * 4 + (lane >> 3);
  if (px >= res || py >= res) return;
  const ViewCam& c = cams[view];
  const d3 dir = mk3(c.dir[0], c.dir[1], c.dir[2]);
  const d3 up = mk3(c.up[0], c.up[1], c.up[2]);
  const d3 right = mk3(c.right[0], c.right[1], c.right[2]);
  // camera.h:22-33: pixelU/V, origin = colU[px] + rowV[py] (raster.cpp:31-35, :70)
  const double pu = -c.he + (px + 0.5) * c.step;
  const double pv = c.he - (py + 0.5) * c.step;
  const d3 o = pu * right + pv * up;
  const d3 inv = mk3(1.0 / dir.x, 1.0 / dir.y, 1.0 / dir.z);
  const double slack = 0x1p-24;
  int bf = -1;
  float bd = -INFINITY;
  double bt = 0.0, bu = 0.0, bv = 0.0;
  double limit = INFINITY;
  int32_t st[kStackMax];
  int sp = 0;
  int32_t ref = root;
  for (;;) {
    if (ref >= 0) {
      const float4* np = reinterpret_cast<const float4*>(nodes + ref);
      const float4 a = __ldg(np), b = __ldg(np + 1), cc = __ldg(np + 2);
      const int4 dd = __ldg(reinterpret_cast<const int4*>(np + 3));
      double tl = 0.0, tr = 0.0;
      const bool hl = slab(a.x, a.z, b.x, b.z, cc.x, cc.z, o, inv, -INFINITY, limit, slack, tl);
      const bool hr = slab(a.y, a.w, b.y, b.w, cc.y, cc.w, o, inv, -INFINITY, limit, slack, tr);
      if (hl && hr) {
        const bool lf = tl <= tr;
        st[sp++] = lf ? dd.y : dd.x;
        ref = lf ? dd.x : dd.y;
        continue;
      }
      if (hl || hr) {
        ref = hl ? dd.x : dd.y;
        continue;
      }
    } else {
      int first, count;
      leaf_decode(ref, first, count);
      for (int k = 0; k < count; ++k) {
        d3 A, B, C;
        int f;
        load_tri(tris + first + k, A, B, C, f);
        // RasterOptions::backfaceCull (raster.cpp:44): faces whose geometric
        // normal points along the view direction are skipped
        if (cull && dot(cross(B - A, C - A), dir) > 0.0) continue;
        double tt, u, v;
        if (!ray_triangle(o, dir, A, B, C, tt, u, v)) continue;
        const float depth = __double2float_rn(-tt);
        if (!(bf < 0 || depth > bd || (depth == bd && f < bf))) continue;
        // candidate pixel box of the face (raster.cpp:46-61)
        const double u0 = dot(A, right), u1 = dot(B, right), u2 = dot(C, right);
        const double v0 = dot(A, up), v1 = dot(B, up), v2 = dot(C, up);
        const double umin = fmin(u0, fmin(u1, u2)), umax = fmax(u0, fmax(u1, u2));
        const double vmin = fmin(v0, fmin(v1, v2)), vmax = fmax(v0, fmax(v1, v2));
        const int pxLo = max(0, static_cast<int>(floor((umin + c.he) / c.step - 0.5)) - 1);
        const int pxHi = min(res - 1, static_cast<int>(ceil((umax + c.he) / c.step - 0.5)) + 1);
        const int pyLo = max(0, static_cast<int>(floor((c.he - vmax) / c.step - 0.5)) - 1);
        const int pyHi = min(res - 1, static_cast<int>(ceil((c.he - vmin) / c.step - 0.5)) + 1);
        if (px < pxLo || px > pxHi || py < pyLo || py > pyHi) continue;
        bf = f;
        bd = depth;
        bt = tt;
        bu = u;
        bv = v;
        limit = -static_cast<double>(nextafterf(bd, -INFINITY));
      }
    }
    if (sp == 0) break;
    ref = st[--sp];
  }
  if (hits && bf >= 0) atomicAdd(&hits[bf], 1ull);
  if (!face_img) return;
  const int64_t pi = static_cast<int64_t>(view) * res * res + static_cast<int64_t>(py) * res + px;
  face_img[pi] = bf;
  if (depth_img) depth_img[pi] = bf >= 0 ? bd : INFINITY;
  if (pos_img) {
    const d3 hit = o + bt * dir;  // raster.cpp:88
    pos_img[3 * pi] = bf >= 0 ? __double2float_rn(hit.x) : 0.f;
    pos_img[3 * pi + 1] = bf >= 0 ? __double2float_rn(hit.y) : 0.f;
    pos_img[3 * pi + 2] = bf >= 0 ? __double2float_rn(hit.z) : 0.f;
  }
  if (nrm_img) {
    float nf[3] = {0.f, 0.f, 0.f};
    if (bf >= 0 && vnormals) {  // raster.cpp:89-92
      const d3 n0 = ld3(vnormals + 3 * faces[3 * bf]), n1 = ld3(vnormals + 3 * faces[3 * bf + 1]),
               n2 = ld3(vnormals + 3 * faces[3 * bf + 2]);
      d3 n = ((1.0 - bu - bv) * n0 + bu * n1) + bv * n2;
      const double len = norm(n);
      if (len > 0) n = n / len;
      nf[0] = __double2float_rn(n.x);
      nf[1] = __double2float_rn(n.y);
      nf[2] = __double2float_rn(n.z);
    }
    nrm_img[3 * pi] = nf[0];
    nrm_img[3 * pi + 1] = nf[1];
    nrm_img[3 * pi + 2] = nf[2];
  }
}

// castVisibility's centring (visibility.cpp:20-30): out = p - center, and the
// largest |out| (ordered bits, max) into acc.
__global__ void k_center_mesh(const double* __restrict__ pos, int nv, double cx, double cy, double cz,
                              double* __restrict__ out, unsigned long long* acc) {
  double m = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const d3 p = mk3(pos[3 * v] - cx, pos[3 * v + 1] - cy, pos[3 * v + 2] - cz);
    st3(out + 3 * v, p);
    const double n = norm(p);
    m = m < n ? n : m;
  }
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(acc, ordered_bits_dev(m));
}

// ---------------------------------------------------------------- view z-buffer rasteriser
// renderView's own face loop (render/raster.cpp:39-98), one thread per
// (view, face): the face's padded pixel box, the per-face Moller-Trumbore
// factors, and per pixel the reference's expressions; the z-test becomes a
// 64-bit atomicMax on key = ordered(f32 depth) << 32 | (0xffffffff - face),
// i.e. the largest depth wins and equal depths go to the lowest face - the
// order-independent form of "replace iff depth > stored" over faces in index
// order. Key 0 = background.
__device__ __forceinline__ unsigned ordered_f32(float f) {
  const unsigned b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(128) k_zbuf_faces(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                                    int nf, const ViewCam* __restrict__ cams, int res, int cull,
                                                    unsigned long long* __restrict__ zbuf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  const int view = blockIdx.y;
  if (f >= nf) return;
  const ViewCam& c = cams[view];
  const d3 dir = mk3(c.dir[0], c.dir[1], c.dir[2]);
  const d3 up = mk3(c.up[0], c.up[1], c.up[2]);
  const d3 right = mk3(c.right[0], c.right[1], c.right[2]);
  const d3 a = ld3(pos + 3 * faces[3 * f]), b = ld3(pos + 3 * faces[3 * f + 1]), cc = ld3(pos + 3 * faces[3 * f + 2]);
  if (cull && dot(cross(b - a, cc - a), dir) > 0.0) return;
  const double u0 = dot(a, right), u1 = dot(b, right), u2 = dot(cc, right);
  const double v0 = dot(a, up), v1 = dot(b, up), v2 = dot(cc, up);
  const double umin = fmin(u0, fmin(u1, u2)), umax = fmax(u0, fmax(u1, u2));
  const double vmin = fmin(v0, fmin(v1, v2)), vmax = fmax(v0, fmax(v1, v2));
  const int pxLo = max(0, static_cast<int>(floor((umin + c.he) / c.step - 0.5)) - 1);
  const int pxHi = min(res - 1, static_cast<int>(ceil((umax + c.he) / c.step - 0.5)) + 1);
  const int pyLo = max(0, static_cast<int>(floor((c.he - vmax) / c.step - 0.5)) - 1);
  const int pyHi = min(res - 1, static_cast<int>(ceil((c.he - vmin) / c.step - 0.5)) + 1);
  if (pxLo > pxHi || pyLo > pyHi) return;
  const d3 e1 = b - a, e2 = cc - a;
  const d3 pvec = cross(dir, e2);
  const double det = dot(e1, pvec);
  if (fabs(det) < 1e-9) return;
  const double inv = 1.0 / det;
  unsigned long long* zb = zbuf + static_cast<int64_t>(view) * res * res;
  const unsigned fkey = 0xffffffffu - static_cast<unsigned>(f);
  for (int py = pyLo; py <= pyHi; ++py) {
    const d3 rowV = (c.he - (py + 0.5) * c.step) * up;
    for (int px = pxLo; px <= pxHi; ++px) {
      const d3 origin = (-c.he + (px + 0.5) * c.step) * right + rowV;
      const d3 sv = origin - a;
      const double bu = dot(sv, pvec) * inv;
      if (bu < 0.0 || bu > 1.0) continue;
      const d3 qv = cross(sv, e1);
      const double bv = dot(dir, qv) * inv;
      if (bv < 0.0 || bu + bv > 1.0) continue;
      const double t = dot(e2, qv) * inv;
      // + 0.0f maps -0 to +0: the reference's `depth > stored` treats the two
      // as equal (ties go to the lower face), so they must share one key
      const unsigned long long key =
          (static_cast<unsigned long long>(ordered_f32(__fadd_rn(__double2float_rn(-t), 0.0f))) << 32) | fkey;
      unsigned long long* z = zb + static_cast<int64_t>(py) * res + px;
      if (key > *z) atomicMax(z, key);
    }
  }
}

// castVisibility's tally (visibility.cpp:41-45): one hit per won pixel.
__global__ void k_zbuf_hits(const unsigned long long* __restrict__ zbuf, int64_t n,
                            unsigned long long* __restrict__ hits) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = zbuf[i];
    if (k) atomicAdd(&hits[0xffffffffu - static_cast<unsigned>(k & 0xffffffffu)], 1ull);
  }
}
}  // namespace

// Resident 128-thread blocks per SM of `kern` (>= 1); callers cache it in a
// function-local static (thread-safe initialisation).
template <class K>
int occupancy(K kern) {
  int v = 0;
  MFB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 128, 0));
  return v < 1 ? 1 : v;
}

static const unsigned long long* scene_acc_of(Ctx&, const Lbvh& bvh) { return bvh.scene_acc; }

void band_init(Ctx& ctx, cudaStream_t s, const BandSync& bs) {
  k_band_init<<<1, 64, 0, s>>>(bs);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void transfer_normals(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const TransferArgs& a) {
  // Per-thread while-while walk (k_transfer_t) on a persistent grid of the
  // resident CTAs; warps take 32-query batches from the list's cursor.
  // Variants measured on config B and removed: the
  // warp-coherent walk (2.49 ms), persistent lanes with refill (1.54-1.86 ms),
  // the 4-wide collapsed BVH (slower on B and E).
  const bool dbg = a.dbg_face || a.dbg_ts;
  static const bool prof = std::getenv("MFB_PROF") != nullptr;
  unsigned long long* pbuf = nullptr;
  if (prof) {
    pbuf = ctx.buf<unsigned long long>("xfer.prof", 8);
    ctx.fill(pbuf, 0, 8 * sizeof(unsigned long long), s);
    ctx.fill(pbuf + 4, 0xff, 2 * sizeof(unsigned long long), s);
  }
  const bool sel = bvh.leaf_max <= 3;
  static const int bps_sel = occupancy(k_transfer_t<false, false, false, true>);
  static const int bps_wide = occupancy(k_transfer_t<false, false, false, false>);
  const int g2 = std::max(1, std::min(kNumSMs * (sel ? bps_sel : bps_wide), div_up(a.q.capacity, 128)));
#define MFB_XFER_T(D, P, BANDS)                                                                               \
  do {                                                                                                        \
    if (sel)                                                                                                  \
      k_transfer_t<D, P, BANDS, true><<<g2, 128, 0, s>>>(                                                     \
          bvh.nodes, bvh.tris, bvh.root_ref, bvh.scene_acc, a.q.qpos, a.q.qtbn, a.q.count, a.hi_normals,      \
          a.hi_faces, a.max_dist, a.rgb, D ? a.dbg_face : nullptr, D ? a.dbg_ts : nullptr, a.counters, pbuf,  \
          a.hi_positions, a.dep_head, a.dep_next, a.bands, a.fmt, bvh.tplane, bvh.lplane, bvh.nplane);                    \
    else                                                                                                      \
      k_transfer_t<D, P, BANDS, false><<<g2, 128, 0, s>>>(                                                    \
          bvh.nodes, bvh.tris, bvh.root_ref, bvh.scene_acc, a.q.qpos, a.q.qtbn, a.q.count, a.hi_normals,      \
          a.hi_faces, a.max_dist, a.rgb, D ? a.dbg_face : nullptr, D ? a.dbg_ts : nullptr, a.counters, pbuf,  \
          a.hi_positions, a.dep_head, a.dep_next, a.bands, a.fmt, bvh.tplane, bvh.lplane, bvh.nplane);                    \
  } while (0)
  // the row-band publication is compiled only into the host path's
  // instantiation (it costs the walk registers)
  if (a.bands.done) {
    MFB_XFER_T(false, false, true);
  } else if (prof) {
    if (dbg) MFB_XFER_T(true, true, false); else MFB_XFER_T(false, true, false);
  } else {
    if (dbg) MFB_XFER_T(true, false, false); else MFB_XFER_T(false, false, false);
  }
#undef MFB_XFER_T
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
  if (prof) {
    unsigned long long h[8];
    MFB_CUDA_TRY(cudaMemcpyAsync(h, pbuf, sizeof(h), cudaMemcpyDeviceToHost, s));
    MFB_CUDA_TRY(cudaStreamSynchronize(s));
    const double nqd = h[3] ? static_cast<double>(h[3]) : 1.0;
    std::fprintf(stderr,
                 "[mfb prof] per query: internal %.2f leaves %.2f triangles %.2f exact tests %.2f (queries %llu); "
                 "warp exits %.1f..%.1f us after the first start\n",
                 h[0] / nqd, h[1] / nqd, h[2] / nqd, h[7] / nqd, h[3], (h[5] - h[4]) * 1e-3, (h[6] - h[4]) * 1e-3);
  }
}

namespace {
// sampleSdf's per-point tail (signfield/watertight.cpp:29-38): magnitude
// sqrt(distSq) of the unbounded closest point (SurfacePoint::distance,
// bvh.h:24), sign from sampleSignedField (sign_grid.cpp:239-264, the same f64
// operations: lattice coordinates, clamped cell, trilinear weights summed
// z-y-x in order).
__global__ void k_sdf_finish(int64_t n, const double* __restrict__ pts, const double* __restrict__ dist_sq,
                             int res, double ox, double oy, double oz, double h, const float* __restrict__ field,
                             double* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double q[3] = {(pts[3 * i] - ox) / h - 0.5, (pts[3 * i + 1] - oy) / h - 0.5, (pts[3 * i + 2] - oz) / h - 0.5};
  int i0[3];
  double f[3];
  for (int k = 0; k < 3; ++k) {
    const double hi = static_cast<double>(res - 1);
    const double c = q[k] < 0.0 ? 0.0 : (hi < q[k] ? hi : q[k]);  // std::clamp(v, 0, res - 1)
    int a = min(static_cast<int>(floor(c)), res - 2);
    a = max(a, 0);
    const double fr = c - a;
    i0[k] = a;
    f[k] = fr < 0.0 ? 0.0 : (1.0 < fr ? 1.0 : fr);
  }
  double result = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double w = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
        const int64_t idx = static_cast<int64_t>(i0[0] + dx) +
                            static_cast<int64_t>(res) * ((i0[1] + dy) + static_cast<int64_t>(res) * (i0[2] + dz));
        result += w * field[idx];
      }
  const double sign = result < 0 ? -1.0 : 1.0;
  out[i] = sign * sqrt(dist_sq[i]);
}
}  // namespace

void sample_sdf(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* pts, int64_t n, int res,
                const double origin[3], double voxel, const float* field, double* out) {
  if (n <= 0) return;
  int32_t* face = ctx.buf<int32_t>("sdf.face", n);
  double* ds = ctx.buf<double>("sdf.ds", n);
  closest_within(ctx, s, bvh, pts, n, INFINITY, face, ds, nullptr, nullptr);
  k_sdf_finish<<<div_up(n, 256), 256, 0, s>>>(n, pts, ds, res, origin[0], origin[1], origin[2], voxel, field, out);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void closest_within(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* q, int64_t n,
                    double max_dist, int32_t* face, double* dist_sq, double* point, double* bary) {
  if (n <= 0) return;
  k_closest<<<div_up(n, 128), 128, 0, s>>>(bvh.nodes, bvh.tris, bvh.root_ref, scene_acc_of(ctx, bvh),
                                           q, n, max_dist, face, dist_sq, point, bary);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void closest_brute(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* q, int64_t n, int32_t* face,
                   double* dist_sq, double* point, double* bary) {
  if (n <= 0) return;
  k_closest_brute<<<static_cast<unsigned>(n), 256, 0, s>>>(m.pos, m.faces, m.nf, q, n, face, dist_sq, point, bary);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void raycast_brute(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* o, const double* d, int64_t n,
                   double tmin, double tmax, int32_t* face, double* t, double* u, double* v) {
  if (n <= 0) return;
  k_raycast_brute<<<static_cast<unsigned>(n), 256, 0, s>>>(m.pos, m.faces, m.nf, o, d, n, tmin, tmax, face, t, u, v);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}


void vertex_bounds(Ctx& ctx, cudaStream_t s, const DevMesh& m, double* out6) {
  auto* acc = ctx.buf<unsigned long long>("vb.acc", 6);
  ctx.fill(acc, 0xff, 3 * sizeof(unsigned long long), s);
  ctx.fill(acc + 3, 0x00, 3 * sizeof(unsigned long long), s);
  if (m.nv > 0) {
    k_vertex_bounds<<<std::min(div_up(m.nv, 256), kNumSMs * 4), 256, 0, s>>>(m.pos, m.nv, acc);
    ctx.count_launch();
    MFB_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long h[6];
  MFB_CUDA_TRY(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
  MFB_CUDA_TRY(cudaStreamSynchronize(s));
  for (int k = 0; k < 6; ++k) {
    unsigned long long b = h[k];
    b = (b & 0x8000000000000000ull) ? (b & ~0x8000000000000000ull) : ~b;
    std::memcpy(&out6[k], &b, 8);
  }
  if (m.nv == 0) {
    for (int k = 0; k < 3; ++k) {
      out6[k] = INFINITY;
      out6[3 + k] = -INFINITY;
    }
  }
}

void surface_band(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, int res, const double origin[3], double h,
                  double truncation, double band_world, uint8_t* labels, float* dist) {
  const int64_t bricks = static_cast<int64_t>((res + 3) / 4) * ((res + 3) / 4) * ((res + 1) / 2);
  const int64_t threads = bricks * 32;
  k_surface_band<<<static_cast<unsigned>(div_up(threads, 128)), 128, 0, s>>>(
      bvh.nodes, bvh.tris, bvh.root_ref, bvh.scene_acc, res, origin[0], origin[1], origin[2], h, truncation,
      band_world, labels, dist);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}


// fibonacciCameras (render/camera.cpp:38-55) + right() (camera.h:19), host f64.
static std::vector<ViewCam> view_cams(const double* cams7, int nviews, int res) {
  std::vector<ViewCam> v(nviews);
  for (int i = 0; i < nviews; ++i) {
    const double* c = cams7 + 7 * i;
    const d3 dir = mk3(c[0], c[1], c[2]), up = mk3(c[3], c[4], c[5]);
    const d3 right = cross(dir, up);
    for (int k = 0; k < 3; ++k) {
      v[i].dir[k] = (&dir.x)[k];
      v[i].up[k] = (&up.x)[k];
      v[i].right[k] = (&right.x)[k];
    }
    v[i].he = c[6];
    v[i].step = 2.0 * c[6] / res;
  }
  return v;
}

void fibonacci_cameras(int count, double half_extent, double* cams7) {
  const double golden = M_PI * (3.0 - std::sqrt(5.0));
  for (int i = 0; i < count; ++i) {
    const double z = 1.0 - 2.0 * (i + 0.5) / count;
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double a = golden * i;
    const d3 viewpoint = mk3(r * std::cos(a), r * std::sin(a), z);
    const d3 dir = mk3(-viewpoint.x, -viewpoint.y, -viewpoint.z);
    const d3 refv = std::abs(z) < 0.9 ? mk3(0, 0, 1) : mk3(0, 1, 0);
    d3 up = cross(dir, refv);
    const double z2 = dot(up, up);
    if (z2 > 0.0) up = up / std::sqrt(z2);  // Eigen normalized() (shim order)
    double* c = cams7 + 7 * i;
    c[0] = dir.x, c[1] = dir.y, c[2] = dir.z;
    c[3] = up.x, c[4] = up.y, c[5] = up.z;
    c[6] = half_extent;
  }
}

void render_views(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* cams7, int nviews, int res, int cull,
                  unsigned long long* hits, int32_t* face_img, float* depth_img, float* pos_img, float* nrm_img,
                  const int32_t* faces, const double* vnormals) {
  if (nviews <= 0 || res <= 0) return;
  const std::vector<ViewCam> hv = view_cams(cams7, nviews, res);
  auto* dc = ctx.buf<ViewCam>("view.cams", nviews);
  MFB_CUDA_TRY(cudaMemcpyAsync(dc, hv.data(), sizeof(ViewCam) * nviews, cudaMemcpyHostToDevice, s));
  const int64_t per_view = static_cast<int64_t>((res + 7) / 8) * ((res + 3) / 4) * 32;
  // views in launch-sized groups (grid.x stays well inside 2^31 blocks)
  const int group = static_cast<int>(std::max<int64_t>(1, (int64_t{1} << 30) / per_view));
  for (int v0 = 0; v0 < nviews; v0 += group) {
    const int nv = std::min(group, nviews - v0);
    const int64_t threads = per_view * nv;
    const int64_t img_off = static_cast<int64_t>(v0) * res * res;
    k_render_views<<<static_cast<unsigned>(div_up(threads, 128)), 128, 0, s>>>(
        bvh.nodes, bvh.tris, bvh.root_ref, dc + v0, nv, res, cull, hits, face_img ? face_img + img_off : nullptr,
        depth_img ? depth_img + img_off : nullptr, pos_img ? pos_img + 3 * img_off : nullptr,
        nrm_img ? nrm_img + 3 * img_off : nullptr, faces, vnormals);
    ctx.count_launch();
  }
  MFB_CUDA_TRY(cudaGetLastError());
}


void raster_visibility(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* cams7, int nviews, int res,
                       unsigned long long* hits) {
  if (nviews <= 0 || res <= 0 || m.nf <= 0) return;
  const std::vector<ViewCam> hv = view_cams(cams7, nviews, res);
  auto* dc = ctx.buf<ViewCam>("view.cams", nviews);
  MFB_CUDA_TRY(cudaMemcpyAsync(dc, hv.data(), sizeof(ViewCam) * nviews, cudaMemcpyHostToDevice, s));
  const int64_t px = static_cast<int64_t>(res) * res;
  // views per pass: z-buffers of <= 256 MiB
  const int group = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(65535, (int64_t{256} << 20) / (8 * px))));
  auto* zb = ctx.buf<unsigned long long>("view.zbuf", static_cast<size_t>(std::min(group, nviews)) * px);
  for (int v0 = 0; v0 < nviews; v0 += group) {
    const int nv = std::min(group, nviews - v0);
    ctx.fill(zb, 0, sizeof(unsigned long long) * nv * px, s);
    k_zbuf_faces<<<dim3(div_up(m.nf, 128), nv), 128, 0, s>>>(m.pos, m.faces, m.nf, dc + v0, res, 0, zb);
    k_zbuf_hits<<<kNumSMs * 8, 256, 0, s>>>(zb, nv * px, hits);
    ctx.count_launch(2);
  }
  MFB_CUDA_TRY(cudaGetLastError());
}

double center_mesh(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double center[3], double* out) {
  auto* acc = ctx.buf<unsigned long long>("ctr.acc", 1);
  ctx.fill(acc, 0, sizeof(unsigned long long), s);
  if (m.nv > 0) {
    k_center_mesh<<<std::min(div_up(m.nv, 256), kNumSMs * 4), 256, 0, s>>>(m.pos, m.nv, center[0], center[1],
                                                                            center[2], out, acc);
    ctx.count_launch();
    MFB_CUDA_TRY(cudaGetLastError());
  }
  unsigned long long h = 0;
  MFB_CUDA_TRY(cudaMemcpyAsync(&h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
  MFB_CUDA_TRY(cudaStreamSynchronize(s));
  h = (h & 0x8000000000000000ull) ? (h & ~0x8000000000000000ull) : ~h;
  double r;
  std::memcpy(&r, &h, 8);
  return m.nv > 0 ? r : 0.0;
}

void raycast_first(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* o, const double* d,
                   int64_t n, double tmin, double tmax, int32_t* face, double* t, double* u,
                   double* v) {
  if (n <= 0) return;
  k_raycast<<<div_up(n, 128), 128, 0, s>>>(bvh.nodes, bvh.tris, bvh.root_ref, o, d, n, tmin, tmax,
                                           face, t, u, v);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

}  // namespace mfb
