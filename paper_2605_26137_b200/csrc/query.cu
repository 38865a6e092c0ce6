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
#include "bake.cuh"

namespace mfb {
namespace {

__device__ __forceinline__ double from_ordered_dev(unsigned long long b) {
  b = (b & 0x8000000000000000ull) ? (b & ~0x8000000000000000ull) : ~b;
  return __longlong_as_double(static_cast<long long>(b));
}

// Upper bound (as float) on the squared distance any face that can still win
// may have, given the incumbent `best` and slack E: (sqrt(best) + E)^2.
__device__ __forceinline__ float prune_bound(double best, double E) {
  if (isnan(best) || best < 0.0) return -INFINITY;  // nothing can improve on NaN or -inf
  if (isinf(best)) return INFINITY;
  const double r = sqrt(best) + E;
  return __double2float_ru(r * r * (1.0 + 0x1p-30));
}

// Lower bound of the squared distance from [qlo, qhi] (per axis) to a box.
__device__ __forceinline__ float box_lb(float mnx, float mny, float mnz, float mxx, float mxy,
                                        float mxz, float3 qlo, float3 qhi) {
  const float dx = fmaxf(fmaxf(__fsub_rd(mnx, qhi.x), __fsub_rd(qlo.x, mxx)), 0.0f);
  const float dy = fmaxf(fmaxf(__fsub_rd(mny, qhi.y), __fsub_rd(qlo.y, mxy)), 0.0f);
  const float dz = fmaxf(fmaxf(__fsub_rd(mnz, qhi.z), __fsub_rd(qlo.z, mxz)), 0.0f);
  return __fadd_rd(__fadd_rd(__fmul_rd(dx, dx), __fmul_rd(dy, dy)), __fmul_rd(dz, dz));
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
      const float lbL = box_lb(a.x, a.y, a.z, a.w, b.x, b.y, qlo, qhi);
      const float lbR = box_lb(b.z, b.w, c.x, c.y, c.z, c.w, qlo, qhi);
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

__device__ __forceinline__ uint8_t encode_channel(double v) {
  const long long q = llround((v + 1.0) * 0.5 * 255.0);
  return static_cast<uint8_t>(q < 0 ? 0 : (q > 255 ? 255 : q));
}

// One 16x16 texel tile per 256-thread block; warp = 8x4 sub-tile.
__global__ void __launch_bounds__(256) k_transfer(
    const BNode* __restrict__ nodes, const BTri* __restrict__ tris, int32_t root,
    const unsigned long long* __restrict__ scene_acc, int res, int g_row0,
    const float* __restrict__ gpos, const float* __restrict__ gnrm, const float* __restrict__ gtan,
    const float* __restrict__ gbit, const uint8_t* __restrict__ gvalid,
    const uint8_t* __restrict__ grel, int row_begin, int row_end,
    const double* __restrict__ hiN, const int32_t* __restrict__ hiF, double max_dist,
    uint8_t* __restrict__ rgb, int32_t* __restrict__ dbg_face, double* __restrict__ dbg_ts,
    unsigned long long* __restrict__ counters) {
  const int tiles_x = (res + 15) >> 4;
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int x = tx * 16 + (warp & 1) * 8 + (lane & 7);
  const int y = row_begin + ty * 16 + (warp >> 1) * 4 + (lane >> 3);
  const bool in = x < res && y < row_end;
  const int64_t gi = (static_cast<int64_t>(y - g_row0)) * res + x;       // G-buffer slab index
  const int64_t oi = (static_cast<int64_t>(y - row_begin)) * res + x;    // output slab index
  bool valid = false, query = false, hit = false;
  int32_t face_out = -1;
  double ts3[3] = {0.0, 0.0, 0.0};
  uint8_t px[3] = {128, 128, 128};
  if (in) {
    valid = gvalid[gi] != 0;
    if (valid) {
      px[2] = 255;  // neutral (128,128,255) unless a hit is encoded below
      if (!grel[gi]) {
        face_out = -2;
      } else {
        query = true;
        const float qx = gpos[3 * gi], qy = gpos[3 * gi + 1], qz = gpos[3 * gi + 2];
        const d3 q = mk3(qx, qy, qz);
        const float3 qf = make_float3(qx, qy, qz);
        const double M = fmax(from_ordered_dev(scene_acc[6]),
                              fmax(fabs(q.x), fmax(fabs(q.y), fabs(q.z))));
        Best best;
        best.d = isinf(max_dist) ? max_dist : max_dist * max_dist;  // bvh.cpp:153-154
        best.face = -1;
        traverse_closest<false>(nodes, tris, root, q, qf, qf, M * 0x1p-32, best);
        if (best.face < 0) {
          face_out = -3;
        } else {
          hit = true;
          face_out = best.face;
          const int v0 = hiF[3 * best.face], v1 = hiF[3 * best.face + 1], v2 = hiF[3 * best.face + 2];
          const d3 n = (best.bary.x * ld3(hiN + 3 * v0) + best.bary.y * ld3(hiN + 3 * v1)) +
                       best.bary.z * ld3(hiN + 3 * v2);
          const d3 T = mk3(gtan[3 * gi], gtan[3 * gi + 1], gtan[3 * gi + 2]);
          const d3 B = mk3(gbit[3 * gi], gbit[3 * gi + 1], gbit[3 * gi + 2]);
          const d3 N = mk3(gnrm[3 * gi], gnrm[3 * gi + 1], gnrm[3 * gi + 2]);
          d3 ts = mk3(dot(n, T), dot(n, B), dot(n, N));
          const double len = norm(ts);
          if (!(len < 1e-12)) {
            ts = ts / len;
            px[0] = encode_channel(ts.x);
            px[1] = encode_channel(ts.y);
            px[2] = encode_channel(ts.z);
            ts3[0] = ts.x;
            ts3[1] = ts.y;
            ts3[2] = ts.z;
          }
        }
      }
    }
    uint8_t* o = rgb + 3 * oi;
    o[0] = px[0];
    o[1] = px[1];
    o[2] = px[2];
    if (dbg_face) dbg_face[oi] = face_out;
    if (dbg_ts) {
      dbg_ts[3 * oi] = ts3[0];
      dbg_ts[3 * oi + 1] = ts3[1];
      dbg_ts[3 * oi + 2] = ts3[2];
    }
  }
  if (counters) {
    const unsigned bv = __ballot_sync(0xffffffffu, valid);
    const unsigned bq = __ballot_sync(0xffffffffu, query);
    const unsigned bh = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) {
      if (bv) atomicAdd(&counters[0], static_cast<unsigned long long>(__popc(bv)));
      if (bq) atomicAdd(&counters[1], static_cast<unsigned long long>(__popc(bq)));
      if (bh) atomicAdd(&counters[2], static_cast<unsigned long long>(__popc(bh)));
    }
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
      const bool hl = slab(a.x, a.y, a.z, a.w, b.x, b.y, o, inv, tmin, limit, slack, tl);
      const bool hr = slab(b.z, b.w, c.x, c.y, c.z, c.w, o, inv, tmin, limit, slack, tr);
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

}  // namespace

static const unsigned long long* scene_acc_of(Ctx&, const Lbvh& bvh) { return bvh.scene_acc; }

void transfer_normals(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const TransferArgs& a) {
  const int res = a.g->res;
  const int rows = a.row_end - a.row_begin;
  if (rows <= 0) return;
  const int tiles = ((res + 15) / 16) * ((rows + 15) / 16);
  k_transfer<<<tiles, 256, 0, s>>>(bvh.nodes, bvh.tris, bvh.root_ref, scene_acc_of(ctx, bvh), res,
                                   a.g->row0, a.g->pos, a.g->nrm, a.g->tan, a.g->bit, a.g->valid,
                                   a.g->rel, a.row_begin, a.row_end, a.hi_normals, a.hi_faces,
                                   a.max_dist, a.rgb, a.dbg_face, a.dbg_ts, a.counters);
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
