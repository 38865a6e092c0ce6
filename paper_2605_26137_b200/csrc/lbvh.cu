// lbvh.cu — GPU LBVH over the dense mesh (replaces Bvh::Bvh/build,
// spatial/bvh.cpp:48-98).
//
// Pipeline (one stream; the repack / segment tree on a helper stream):
//   1. bounds      : centroid bounds + max |coordinate| (ordered-int atomics)
//   2. morton      : 30-bit Morton key of each face centroid
//   3. sort        : hand-written stable 3-pass onesweep radix sort of
//                    (key, face) pairs (sort.cu), histograms built in step 2
//   4. emit        : Karras 2012 hierarchy emission; subtrees covering
//                    <= kLeafMax primitives become leaf ranges (the
//                    reference's leaf size, bvh.cpp:13)
//   5. repack      : gather each primitive's f64 vertices into Morton order
//                    (BTri) plus its outward-rounded fp32 box (TBox)
//   6. refit       : propagate the fp32 boxes up the tree; each parent stores
//                    both child boxes (64-B nodes).
// Query results do not depend on the tree shape: the reference
// answer is argmin over faces of (distSq, face), which any conservative tree
// reproduces exactly.
#include <cuda/atomic>

#include <cstdlib>

#include "bake.cuh"

namespace mfb {
namespace {

__device__ __forceinline__ unsigned long long ordered_bits(double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double from_ordered(unsigned long long b) {
  b = (b & 0x8000000000000000ull) ? (b & ~0x8000000000000000ull) : ~b;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}

// acc[0..2] = min vertex, acc[3..5] = max vertex (the Morton quantisation
// domain: it contains every centroid, and one streaming pass over the
// positions is cheaper than gathering every face's corners), acc[6] = max
// |vertex coord|
// vflags (optional): validateMesh's non-finite-coordinate check
// (mesh.cpp:37-48) on the way, bit 0 (the host path defers the mesh's
// validation pass into the LBVH build)
__global__ void k_bounds(const double* __restrict__ pos, int nv, unsigned long long* acc, int* vflags) {
  pdl_wait();
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  double amax = 0.0;
  bool bad = false;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double c = pos[3 * v + k];
      bad |= !isfinite(c);
      mn[k] = fmin(mn[k], c);
      mx[k] = fmax(mx[k], c);
      amax = fmax(amax, fabs(c));
    }
  }
  if (vflags && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(vflags, 1);
  // warp reduce, then block reduce in shared memory, one atomic per block
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
      mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
    }
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  }
  __shared__ double red[7][32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      red[k][w] = mn[k];
      red[3 + k][w] = mx[k];
    }
    red[6][w] = amax;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int k = threadIdx.x;
    double v = red[k][0];
    for (int i = 1; i < nw; ++i) v = k < 3 ? fmin(v, red[k][i]) : fmax(v, red[k][i]);
    if (k < 3) atomicMin(&acc[k], ordered_bits(v));
    else atomicMax(&acc[k], ordered_bits(v));
  }
}

// min slots (0..2) to all-ones, max / |max| slots (3..7) to zero; the sort's
// 3 x 1024 digit histograms and 3 tile counters to zero
__global__ void k_acc_init(unsigned long long* acc, int* hist) {
  if (threadIdx.x < 8) acc[threadIdx.x] = threadIdx.x < 3 ? ~0ull : 0ull;
  for (int i = threadIdx.x; i < 3 * 1024 + 4; i += blockDim.x) hist[i] = 0;
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// 30-bit Morton keys (10 bits per axis over the centroid bounds), fused with
// the sort's three 10-bit digit histograms (block histograms in shared
// memory, one global atomic per non-empty bin) and the zeroing of its
// look-back status words. Duplicate keys are fine - Karras' emission breaks
// ties with the primitive index.
constexpr int kMortonThreads = 512, kMortonPer = 8;
__global__ void __launch_bounds__(kMortonThreads) k_morton(const double* __restrict__ pos,
                                                           const int32_t* __restrict__ faces, int nf,
                                                           const unsigned long long* __restrict__ acc,
                                                           uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                           int* __restrict__ hist, uint32_t* __restrict__ status,
                                                           int64_t status_words, int nv, int* vflags) {
  pdl_wait();
  __shared__ int h[3 * 1024];
  for (int i = threadIdx.x; i < 3 * 1024; i += blockDim.x) h[i] = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < status_words;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    status[i] = 0u;
  __syncthreads();
  constexpr double cells = 1023.0;
  double lo[3], inv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = from_ordered(acc[k]);
    const double ext = from_ordered(acc[3 + k]) - lo[k];
    inv[k] = ext > 0.0 ? cells / ext : 0.0;
  }
  const int f0 = blockIdx.x * (kMortonThreads * kMortonPer);
#pragma unroll
  for (int j = 0; j < kMortonPer; ++j) {
    const int f = f0 + j * kMortonThreads + threadIdx.x;
    if (f >= nf) break;
    int a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
    if (vflags && (static_cast<unsigned>(a) >= static_cast<unsigned>(nv) ||
                   static_cast<unsigned>(b) >= static_cast<unsigned>(nv) ||
                   static_cast<unsigned>(c) >= static_cast<unsigned>(nv))) {
      // validateMesh's face-index check (bit 1); the index is zeroed in the
      // device copy so every later kernel stays in bounds (the bake's result
      // is discarded: the host reports InvalidGeometry)
      int32_t* fw = const_cast<int32_t*>(faces);
      if (static_cast<unsigned>(a) >= static_cast<unsigned>(nv)) fw[3 * f] = a = 0;
      if (static_cast<unsigned>(b) >= static_cast<unsigned>(nv)) fw[3 * f + 1] = b = 0;
      if (static_cast<unsigned>(c) >= static_cast<unsigned>(nv)) fw[3 * f + 2] = c = 0;
      atomicOr(vflags, 2);
    }
    uint32_t q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double ck = ((pos[3 * a + k] + pos[3 * b + k]) + pos[3 * c + k]) / 3.0;
      double t = (ck - lo[k]) * inv[k];
      t = fmin(fmax(t, 0.0), cells);
      q[k] = static_cast<uint32_t>(t);
    }
    const uint32_t key = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
    keys[f] = key;
    vals[f] = static_cast<uint32_t>(f);
    atomicAdd(&h[key & 1023u], 1);
    atomicAdd(&h[1024 + ((key >> 10) & 1023u)], 1);
    atomicAdd(&h[2048 + (key >> 20)], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * 1024; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Karras delta over augmented keys (key, index): -1 outside [0, n).
__device__ __forceinline__ int kdelta(const uint32_t* __restrict__ k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  const uint32_t a = __ldg(k + i), b = __ldg(k + j);
  if (a == b) return 32 + __clz(static_cast<uint32_t>(i ^ j));
  return __clz(a ^ b);
}

// parent links: (parent << 1) | side; prim_parent for primitives, node_parent for internals.
// Also appends every reachable node with a leaf-range child to `starts`
// (count in starts_n): the refit climbs start there, so it never reads the
// nodes buried inside leaf ranges.
// (reach_list: `starts` instead lists every reachable node - the root and
// every node covering more than leaf_max primitives - for k_node_boxes)
__global__ void k_emit(const uint32_t* __restrict__ keys, int n, int leaf_max, BNode* __restrict__ nodes,
                       int32_t* __restrict__ prim_parent, int32_t* __restrict__ node_parent,
                       int32_t* __restrict__ starts, int* __restrict__ starts_n, int reach_list = 0) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n - 1;
  bool start = false;
  if (active) {
    const int d = (kdelta(keys, n, i, i + 1) - kdelta(keys, n, i, i - 1)) > 0 ? 1 : -1;
    const int dmin = kdelta(keys, n, i, i - d);
    int lmax = 2;
    while (kdelta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
      if (kdelta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    const int j = i + l * d;
    const int dnode = kdelta(keys, n, i, j);
    int s = 0, t = l;
    do {
      t = (t + 1) >> 1;
      if (kdelta(keys, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    const int gamma = i + s * d + min(d, 0);
    const int first = min(i, j), last = max(i, j);
    const int cl = gamma - first + 1, cr = last - gamma;
    int4 dd;
    dd.x = cl <= leaf_max ? leaf_ref(first, cl) : gamma;
    dd.y = cr <= leaf_max ? leaf_ref(gamma + 1, cr) : gamma + 1;
    dd.z = first;
    dd.w = last - first + 1;
    nodes[i].d = dd;
    if (first == gamma) prim_parent[gamma] = (i << 1) | 0;
    else node_parent[gamma] = (i << 1) | 0;
    if (last == gamma + 1) prim_parent[gamma + 1] = (i << 1) | 1;
    else node_parent[gamma + 1] = (i << 1) | 1;
    start = (i == 0 || dd.w > leaf_max) && (reach_list || dd.x < 0 || dd.y < 0);
  }
  // warp-aggregated append
  const unsigned m = __ballot_sync(0xffffffffu, start);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(starts_n, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (start) starts[base + __popc(m & ((1u << lane) - 1u))] = i;
}

// Arrival counter of a refit node: release (our child box store is made
// visible at L2 before the count moves; MEMBAR.GPU) but no acquire fence -
// the second arriver reads its sibling's box with ld.cg from L2, the point of
// coherence, after (control-dependent on) the atomic's result, so the L1-wide
// CCTL.IVALL an acq_rel atomic adds on every level is avoided (the
// threadFenceReduction pattern). Returns the previous count.
__device__ __forceinline__ int arrive(int* f) {
  int old;
  asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(f) : "memory");
  return old;
}

struct FBox {
  float mn[3], mx[3];
};

__device__ __forceinline__ void store_child_box(BNode* nd, int side, const FBox& b) {
  float* f = reinterpret_cast<float*>(nd);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    f[bnode_coord(side, k)] = b.mn[k];
    f[bnode_coord(side, 3 + k)] = b.mx[k];
  }
}
__device__ __forceinline__ FBox load_child_box_cg(const BNode* nd, int side) {
  const float* f = reinterpret_cast<const float*>(nd);
  FBox b;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    b.mn[k] = __ldcg(f + bnode_coord(side, k));
    b.mx[k] = __ldcg(f + bnode_coord(side, 3 + k));
  }
  return b;
}

// Gathers each primitive's f64 vertices into leaf order and its outward-
// rounded fp32 box (fully parallel; random reads, coalesced writes).
// The containment planes of one triangle (TPlane): directions in f64,
// rounded to fp32, and the vertex bounds evaluated in f64 with those fp32
// directions, rounded outward. Degenerate triangles get zero vectors (their
// lower bound is 0: never skipped).
__device__ __forceinline__ double dot_f(const float4& m, const double* v) {
  return (static_cast<double>(m.x) * v[0] + static_cast<double>(m.y) * v[1]) + static_cast<double>(m.z) * v[2];
}
__device__ void tri_planes(const double* v, TPlane& tp) {
  const double e1[3] = {v[3] - v[0], v[4] - v[1], v[5] - v[2]};
  const double e2[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
  double nn[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  const double len = sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!(len > 0.0) || !isfinite(len)) {
    tp.m0 = tp.m1 = tp.m2 = tp.n = tp.hi = zero;
    return;
  }
  float4 n4 = make_float4(static_cast<float>(nn[0] / len), static_cast<float>(nn[1] / len),
                          static_cast<float>(nn[2] / len), 0.f);
  const double nf[3] = {n4.x, n4.y, n4.z};
  double lo = INFINITY, hi = -INFINITY;
  for (int c = 0; c < 3; ++c) {
    const double t = dot_f(n4, v + 3 * c);
    lo = fmin(lo, t);
    hi = fmax(hi, t);
  }
  n4.w = __double2float_rd(lo);
  tp.n = n4;
  tp.hi = make_float4(__double2float_ru(hi), 0.f, 0.f, 0.f);
  float4* ms[3] = {&tp.m0, &tp.m1, &tp.m2};
  for (int e = 0; e < 3; ++e) {
    const double* a = v + 3 * e;
    const double* b = v + 3 * ((e + 1) % 3);
    const double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    // in-plane direction perpendicular to the edge: d x n (f64, from the fp32 n)
    double m[3] = {d[1] * nf[2] - d[2] * nf[1], d[2] * nf[0] - d[0] * nf[2], d[0] * nf[1] - d[1] * nf[0]};
    const double ml = sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
    if (!(ml > 0.0) || !isfinite(ml)) {
      *ms[e] = zero;
      continue;
    }
    float4 m4 = make_float4(static_cast<float>(m[0] / ml), static_cast<float>(m[1] / ml),
                            static_cast<float>(m[2] / ml), 0.f);
    const double* opp = v + 3 * ((e + 2) % 3);
    if (dot_f(m4, opp) > dot_f(m4, a)) {  // outward: away from the opposite vertex
      m4.x = -m4.x;
      m4.y = -m4.y;
      m4.z = -m4.z;
    }
    double o = -INFINITY;
    for (int c = 0; c < 3; ++c) o = fmax(o, dot_f(m4, v + 3 * c));
    m4.w = __double2float_ru(o);
    *ms[e] = m4;
  }
}

// Area vector (b - a) x (c - a) of one leaf-order triangle, and its first edge.
__device__ __forceinline__ void tri_area(const double* v, double c[3], double e[3]) {
  e[0] = v[3] - v[0];
  e[1] = v[4] - v[1];
  e[2] = v[5] - v[2];
  const double b[3] = {v[6] - v[0], v[7] - v[1], v[8] - v[2]};
  c[0] = e[1] * b[2] - e[2] * b[1];
  c[1] = e[2] * b[0] - e[0] * b[2];
  c[2] = e[0] * b[1] - e[1] * b[0];
}
// The LPlane frame from a patch's summed area vector s, its summed area
// magnitudes sa and one edge e0: false (zero record) for a folded or
// degenerate patch.
__device__ bool plane_frame(const double s[3], double sa, const double e0[3], LPlane& lp) {
  lp = LPlane{};
  const double sl = sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
  if (!(sl > 1e-3 * sa) || !isfinite(sl)) return false;
  const double n[3] = {s[0] / sl, s[1] / sl, s[2] / sl};
  const double en = e0[0] * n[0] + e0[1] * n[1] + e0[2] * n[2];
  double u[3] = {e0[0] - en * n[0], e0[1] - en * n[1], e0[2] - en * n[2]};
  const double ul = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  if (!(ul > 0.0) || !isfinite(ul)) return false;
  for (int k = 0; k < 3; ++k) u[k] /= ul;
  const double v[3] = {n[1] * u[2] - n[2] * u[1], n[2] * u[0] - n[0] * u[2], n[0] * u[1] - n[1] * u[0]};
  for (int k = 0; k < 3; ++k) {
    lp.n[k] = static_cast<float>(n[k]);
    lp.u[k] = static_cast<float>(u[k]);
    lp.v[k] = static_cast<float>(v[k]);
  }
  return true;
}
// Extends r[d] = [min, max] of the three rounded directions' projections by
// one triangle's vertices (f64 products of the fp32 directions).
__device__ __forceinline__ void plane_ranges(const LPlane& lp, const double* x, double r[3][2]) {
  const float* dir[3] = {lp.n, lp.u, lp.v};
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d) {
      const double p = (static_cast<double>(dir[d][0]) * x[3 * c] + static_cast<double>(dir[d][1]) * x[3 * c + 1]) +
                       static_cast<double>(dir[d][2]) * x[3 * c + 2];
      r[d][0] = fmin(r[d][0], p);
      r[d][1] = fmax(r[d][1], p);
    }
}
__device__ __forceinline__ void plane_store_ranges(LPlane& lp, const double r[3][2]) {
  lp.lo = __double2float_rd(r[0][0]);
  lp.hi = __double2float_ru(r[0][1]);
  lp.umin = __double2float_rd(r[1][0]);
  lp.umax = __double2float_ru(r[1][1]);
  lp.vmin = __double2float_rd(r[2][0]);
  lp.vmax = __double2float_ru(r[2][1]);
}

// LPlane of the leaf [first, first + count) of leaf-order triangles.
__device__ void leaf_plane(const BTri* __restrict__ tris, int first, int count, LPlane& lp) {
  double s[3] = {0.0, 0.0, 0.0}, sa = 0.0, e0[3] = {0.0, 0.0, 0.0};
  for (int t = 0; t < count; ++t) {
    double c[3], e[3];
    tri_area(tris[first + t].v, c, e);
    s[0] += c[0];
    s[1] += c[1];
    s[2] += c[2];
    sa += sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    if (t == 0) {
      e0[0] = e[0];
      e0[1] = e[1];
      e0[2] = e[2];
    }
  }
  if (!plane_frame(s, sa, e0, lp)) return;
  double r[3][2] = {{INFINITY, -INFINITY}, {INFINITY, -INFINITY}, {INFINITY, -INFINITY}};
  for (int t = 0; t < count; ++t) plane_ranges(lp, tris[first + t].v, r);
  plane_store_ranges(lp, r);
}

// One warp per reachable internal node (the segment-tree build lists them
// all): its own oriented box when its range holds <= kNodePlaneMax
// triangles. Lanes stride over the range; the frame comes from lane 0's
// reduced sums (every lane then uses the same rounded directions), the
// ranges reduce exactly (min / max).
__device__ void node_plane(const BNode* __restrict__ nodes, const BTri* __restrict__ tris, int i, int lane,
                           LPlane* __restrict__ nplane) {
  const int4 d = nodes[i].d;
  LPlane lp{};
  if (d.w <= kNodePlaneMax) {
    double s[3] = {0.0, 0.0, 0.0}, sa = 0.0;
    for (int t = lane; t < d.w; t += 32) {
      double c[3], e[3];
      tri_area(tris[d.z + t].v, c, e);
      s[0] += c[0];
      s[1] += c[1];
      s[2] += c[2];
      sa += sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    }
    for (int off = 16; off > 0; off >>= 1) {
      s[0] += __shfl_xor_sync(0xffffffffu, s[0], off);
      s[1] += __shfl_xor_sync(0xffffffffu, s[1], off);
      s[2] += __shfl_xor_sync(0xffffffffu, s[2], off);
      sa += __shfl_xor_sync(0xffffffffu, sa, off);
    }
    for (int k = 0; k < 3; ++k) s[k] = __shfl_sync(0xffffffffu, s[k], 0);
    sa = __shfl_sync(0xffffffffu, sa, 0);
    double c[3], e0[3];
    tri_area(tris[d.z].v, c, e0);
    if (plane_frame(s, sa, e0, lp)) {
      double r[3][2] = {{INFINITY, -INFINITY}, {INFINITY, -INFINITY}, {INFINITY, -INFINITY}};
      for (int t = lane; t < d.w; t += 32) plane_ranges(lp, tris[d.z + t].v, r);
      for (int off = 16; off > 0; off >>= 1)
        for (int k = 0; k < 3; ++k) {
          r[k][0] = fmin(r[k][0], __shfl_xor_sync(0xffffffffu, r[k][0], off));
          r[k][1] = fmax(r[k][1], __shfl_xor_sync(0xffffffffu, r[k][1], off));
        }
      plane_store_ranges(lp, r);
    }
  }
  if (lane == 0) nplane[i] = lp;
}
__global__ void k_node_planes(const BNode* __restrict__ nodes, const BTri* __restrict__ tris,
                              const int32_t* __restrict__ list, const int* __restrict__ list_n,
                              LPlane* __restrict__ nplane) {
  const int lane = threadIdx.x & 31, nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const int cnt = *list_n;
  for (int w = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5); w < cnt; w += nw)  // warp-uniform
    node_plane(nodes, tris, list[w], lane, nplane);
}

// One thread per listed node (every reachable node with a leaf child is in
// the list); each leaf has one parent, so each record is written once.
__global__ void k_leaf_planes(const BNode* __restrict__ nodes, const BTri* __restrict__ tris,
                              const int32_t* __restrict__ list, const int* __restrict__ list_n, int n,
                              LPlane* __restrict__ lplane) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (n == 1) {
    if (j == 0) leaf_plane(tris, 0, 1, lplane[0]);
    return;
  }
  if (j >= *list_n) return;
  const int4 d = nodes[list[j]].d;
  const int refs[2] = {d.x, d.y};
  for (int c = 0; c < 2; ++c) {
    if (refs[c] >= 0) continue;
    int first, count;
    leaf_decode(refs[c], first, count);
    LPlane lp;
    leaf_plane(tris, first, count, lp);
    lplane[first] = lp;
  }
}

// (kPlanes: the wide-leaf instantiation; the plane arithmetic costs the
// gather its occupancy, 72 vs 32 registers, so the leaf-<=3 trees
// of configs A-D run the plain one)
template <bool kPlanes>
__global__ void k_repack(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                         const uint32_t* __restrict__ order, int n, BTri* __restrict__ tris,
                         TBox* __restrict__ tbox, TPlane* __restrict__ tplane) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int f = static_cast<int>(order[p]);
  const int vi[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
  BTri t;
  FBox box;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    box.mn[k] = INFINITY;
    box.mx[k] = -INFINITY;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double x = pos[3 * vi[c] + k];
      t.v[3 * c + k] = x;
      box.mn[k] = fminf(box.mn[k], __double2float_rd(x));
      box.mx[k] = fmaxf(box.mx[k], __double2float_ru(x));
    }
  }
  t.face = f;
  t.pad = 0;
  const double2* src = reinterpret_cast<const double2*>(&t);
  double2* dst = reinterpret_cast<double2*>(&tris[p]);
#pragma unroll
  for (int q = 0; q < 5; ++q) dst[q] = src[q];
  tbox[p].a = make_float4(box.mn[0], box.mn[1], box.mn[2], box.mx[0]);
  tbox[p].b = make_float4(box.mx[1], box.mx[2], 0.f, 0.f);
  if (kPlanes) {
    TPlane tp;
    tri_planes(t.v, tp);
    tplane[p] = tp;
  }
}

// ---- node boxes from a segment tree over the leaf-order triangle boxes -----
// Every Karras node covers a contiguous range of leaf-order triangles, so its
// children's boxes are range unions: a power-of-two segment tree over the
// TBox array (leaves at N + i, internal node j = union of 2j and 2j+1, built
// 10 levels per 1024-thread CTA in shared memory) answers each child box
// with O(log range) independent loads - no bottom-up climb with one atomic
// and one dependent L2 round trip per level. The unions are exact (fminf /
// fmaxf), so the boxes are the ones the climb would produce.
__device__ __forceinline__ FBox fbox_empty() {
  FBox b;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    b.mn[k] = INFINITY;
    b.mx[k] = -INFINITY;
  }
  return b;
}
__device__ __forceinline__ void fbox_union(FBox& a, const FBox& b) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    a.mn[k] = fminf(a.mn[k], b.mn[k]);
    a.mx[k] = fmaxf(a.mx[k], b.mx[k]);
  }
}
#pragma nv_diag_suppress 550  // the load's two padding lanes are not used
__device__ __forceinline__ FBox fbox_load(const TBox* p) {  // one 256-bit read-only load
  FBox r;
  float p0, p1;
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r.mn[0]), "=f"(r.mn[1]), "=f"(r.mn[2]), "=f"(r.mx[0]), "=f"(r.mx[1]), "=f"(r.mx[2]), "=f"(p0), "=f"(p1)
      : "l"(p));
  return r;
}
#pragma nv_diag_default 550
__device__ __forceinline__ void fbox_store(TBox* p, const FBox& r) {
  p->a = make_float4(r.mn[0], r.mn[1], r.mn[2], r.mx[0]);
  p->b = make_float4(r.mx[1], r.mx[2], 0.f, 0.f);
}
// Thread t holds node base + t of a level [L, 2L) (empty box past `cnt`);
// the CTA's nodes are consecutive and 1024-aligned (or the whole level when
// L < 1024). Writes their ancestors up to 10 levels, or to the root (index 1):
// five levels inside each warp with shuffles, five more across the CTA's
// warps in warp 0 - one barrier.
__device__ __forceinline__ FBox fbox_shfl_down(const FBox& b, int d) {
  FBox r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.mn[k] = __shfl_down_sync(0xffffffffu, b.mn[k], d);
    r.mx[k] = __shfl_down_sync(0xffffffffu, b.mx[k], d);
  }
  return r;
}
__device__ __forceinline__ void seg_reduce_block(FBox box, unsigned base, int cnt, TBox* seg, FBox* sm) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int lv = 1; lv <= 5; ++lv) {
    if ((base >> lv) == 0) return;  // past the root (uniform across the CTA)
    fbox_union(box, fbox_shfl_down(box, 1 << (lv - 1)));  // (lanes past 31 get their own box)
    if ((lane & ((1 << lv) - 1)) == 0 && t < cnt) fbox_store(seg + ((base + t) >> lv), box);
  }
  if ((base >> 6) == 0) return;
  if (lane == 0) sm[w] = box;
  __syncthreads();
  if (w != 0) return;
  const int nw = (cnt + 31) >> 5;
  box = lane < nw ? sm[lane] : fbox_empty();
  for (int lv = 6; lv <= 10; ++lv) {
    if ((base >> lv) == 0) return;
    fbox_union(box, fbox_shfl_down(box, 1 << (lv - 6)));
    if ((lane & ((1 << (lv - 5)) - 1)) == 0 && lane < nw) fbox_store(seg + ((base + 32u * lane) >> lv), box);
  }
}

// The first 10 levels above the leaf-order boxes written by k_repack (a
// separate pass: the 256-thread gather runs at full occupancy, and this
// streaming reduction reads the 32-byte boxes once).
__global__ void __launch_bounds__(1024) k_seg_leaves(const TBox* __restrict__ tbox, int n, int N,
                                                     TBox* __restrict__ seg) {
  pdl_wait();
  __shared__ FBox sm[32];
  const int p = blockIdx.x * 1024 + threadIdx.x;
  const FBox box = p < n ? fbox_load(tbox + p) : fbox_empty();
  seg_reduce_block(box, static_cast<unsigned>(N + blockIdx.x * 1024), min(1024, N), seg, sm);
}

// The next 10 levels: nodes [L, 2L) -> their ancestors.
__global__ void __launch_bounds__(1024) k_seg_up(TBox* __restrict__ seg, int L) {
  pdl_wait();
  __shared__ FBox sm[32];
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const FBox box = i < L ? fbox_load(seg + L + i) : fbox_empty();
  seg_reduce_block(box, static_cast<unsigned>(L + blockIdx.x * 1024), min(1024, L), seg, sm);
}

#ifndef MFB_NODEBOX_LEVELS
#define MFB_NODEBOX_LEVELS 2
#endif
// One thread per reachable node, from emit's compacted list (full warps of
// range queries instead of one active lane in three).
// (72 registers, 3 CTAs of 256 per SM; capped at 64 / 48 registers: 1.437 / 1.474 vs 1.425 ms per bake)
__global__ void k_node_boxes(const TBox* __restrict__ seg, const TBox* __restrict__ tbox, int N, int n, int leaf_max,
                             BNode* __restrict__ nodes, float* __restrict__ root_box,
                             const int32_t* __restrict__ reach, const int* __restrict__ reach_n) {
  pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *reach_n) return;
  const int i = reach[j];
  const int4 d = nodes[i].d;
  int gamma;
  if (d.x >= 0) {
    gamma = d.x;
  } else {
    int f, c;
    leaf_decode(d.x, f, c);
    gamma = f + c - 1;
  }
  // both children's ranges walked together: the up-to-four loads of a level
  // are issued before any of them is used (one L2 round trip per level)
  FBox L = fbox_empty(), R = fbox_empty();
  const unsigned uN = static_cast<unsigned>(N);
  unsigned l1 = static_cast<unsigned>(d.z) + uN, h1 = static_cast<unsigned>(gamma) + uN + 1;
  unsigned l2 = h1, h2 = static_cast<unsigned>(d.z + d.w) + uN;
  auto ld = [&](unsigned j) { return j >= uN ? fbox_load(tbox + (j - uN)) : fbox_load(seg + j); };
  // MFB_NODEBOX_LEVELS levels per iteration: their (up to 4 per level) loads
  // depend only on index arithmetic, so all are in flight before the first union
  constexpr int kLv = MFB_NODEBOX_LEVELS;
  while (l1 < h1 || l2 < h2) {
    bool take[kLv][4];
    unsigned at[kLv][4];
#pragma unroll
    for (int v = 0; v < kLv; ++v) {
      take[v][0] = l1 < h1 && (l1 & 1);
      take[v][1] = l1 < h1 && (h1 & 1);
      take[v][2] = l2 < h2 && (l2 & 1);
      take[v][3] = l2 < h2 && (h2 & 1);
      at[v][0] = l1;
      at[v][1] = h1 - 1;
      at[v][2] = l2;
      at[v][3] = h2 - 1;
      l1 = (l1 + take[v][0]) >> 1;
      h1 = (h1 - take[v][1]) >> 1;
      l2 = (l2 + take[v][2]) >> 1;
      h2 = (h2 - take[v][3]) >> 1;
    }
    FBox x[kLv][4];
#pragma unroll
    for (int v = 0; v < kLv; ++v)
#pragma unroll
      for (int k = 0; k < 4; ++k) x[v][k] = take[v][k] ? ld(at[v][k]) : fbox_empty();
#pragma unroll
    for (int v = 0; v < kLv; ++v) {
      fbox_union(L, x[v][0]);
      fbox_union(L, x[v][1]);
      fbox_union(R, x[v][2]);
      fbox_union(R, x[v][3]);
    }
  }
  store_child_box(&nodes[i], 0, L);
  store_child_box(&nodes[i], 1, R);
  if (i == 0) {
    FBox u = L;
    fbox_union(u, R);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      root_box[k] = u.mn[k];
      root_box[3 + k] = u.mx[k];
    }
  }
}

// Bottom-up refit: each primitive's thread climbs while it is the second
// child to arrive (acquire/release counter per node), storing the child box
// into its parent's slot.
__global__ void k_refit(const TBox* __restrict__ tbox, int n, BNode* nodes, const int32_t* __restrict__ prim_parent,
                        const int32_t* __restrict__ node_parent, int* __restrict__ flags,
                        float* __restrict__ root_box) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float4 ba = tbox[p].a, bb = tbox[p].b;
  FBox box;
  box.mn[0] = ba.x;
  box.mn[1] = ba.y;
  box.mn[2] = ba.z;
  box.mx[0] = ba.w;
  box.mx[1] = bb.x;
  box.mx[2] = bb.y;
  if (n == 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      root_box[k] = box.mn[k];
      root_box[3 + k] = box.mx[k];
    }
    return;
  }
  int link = prim_parent[p];
  for (;;) {
    const int par = link >> 1, side = link & 1;
    store_child_box(&nodes[par], side, box);
    if (arrive(&flags[par]) == 0) return;  // sibling carries on
    const FBox other = load_child_box_cg(&nodes[par], side ^ 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      box.mn[k] = fminf(box.mn[k], other.mn[k]);
      box.mx[k] = fmaxf(box.mx[k], other.mx[k]);
    }
    if (par == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        root_box[k] = box.mn[k];
        root_box[3 + k] = box.mx[k];
      }
      return;
    }
    link = node_parent[par];
  }
}

// Refit from the leaf ranges. Internal nodes whose range holds <= leaf_max
// primitives are never visited (their parent references them as a leaf
// range), so the climb starts at the reachable nodes that have leaf-range
// children: such a node unions its leaf ranges' triangle boxes into its child
// slots and counts them as arrivals; a node is complete after two arrivals,
// and the thread that completes it carries its box up to the parent's slot
// (acquire/release counter per node).
__global__ void k_refit_ranges(const TBox* __restrict__ tbox, const BNode* __restrict__ nodes_in,
                               const int32_t* __restrict__ starts, const int* __restrict__ starts_n,
                               BNode* nodes, const int32_t* __restrict__ node_parent,
                               int* __restrict__ flags, float* __restrict__ root_box) {
  const int si = blockIdx.x * blockDim.x + threadIdx.x;
  if (si >= *starts_n) return;
  const int i = starts[si];
  const int4 d = nodes_in[i].d;
  const int refs[2] = {d.x, d.y};
  FBox box;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    box.mn[k] = INFINITY;
    box.mx[k] = -INFINITY;
  }
  int leaves = 0;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    if (refs[side] >= 0) continue;
    int first, count;
    leaf_decode(refs[side], first, count);
    FBox lb;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lb.mn[k] = INFINITY;
      lb.mx[k] = -INFINITY;
    }
    for (int t = 0; t < count; ++t) {
      const float4 a = tbox[first + t].a, b = tbox[first + t].b;
      lb.mn[0] = fminf(lb.mn[0], a.x);
      lb.mn[1] = fminf(lb.mn[1], a.y);
      lb.mn[2] = fminf(lb.mn[2], a.z);
      lb.mx[0] = fmaxf(lb.mx[0], a.w);
      lb.mx[1] = fmaxf(lb.mx[1], b.x);
      lb.mx[2] = fmaxf(lb.mx[2], b.y);
    }
    store_child_box(&nodes[i], side, lb);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      box.mn[k] = fminf(box.mn[k], lb.mn[k]);
      box.mx[k] = fmaxf(box.mx[k], lb.mx[k]);
    }
    ++leaves;
  }
  if (leaves == 0) return;  // both children internal: climbers arrive from below
  int node = i;
  if (leaves == 1) {
    if (arrive(&flags[node]) == 0) return;  // internal sibling still climbing
    const int internal_side = refs[0] >= 0 ? 0 : 1;
    const FBox other = load_child_box_cg(&nodes[node], internal_side);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      box.mn[k] = fminf(box.mn[k], other.mn[k]);
      box.mx[k] = fmaxf(box.mx[k], other.mx[k]);
    }
  }
  // `node` is complete with `box`: climb. The parent's own link is loaded
  // before the arrival atomic, so the next level does not start with a
  // dependent load.
  int link = node != 0 ? __ldg(node_parent + node) : 0;
  for (;;) {
    if (node == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        root_box[k] = box.mn[k];
        root_box[3 + k] = box.mx[k];
      }
      return;
    }
    const int par = link >> 1, side = link & 1;
    store_child_box(&nodes[par], side, box);
    link = par != 0 ? __ldg(node_parent + par) : 0;
    if (arrive(&flags[par]) == 0) return;
    const FBox other = load_child_box_cg(&nodes[par], side ^ 1);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      box.mn[k] = fminf(box.mn[k], other.mn[k]);
      box.mx[k] = fmaxf(box.mx[k], other.mx[k]);
    }
    node = par;
  }
}

}  // namespace

// Leaf-range cap of a build: the caller's hint or kLeafMaxDefault (the
// reference uses 4, bvh.cpp:13; results are tree-independent) unless
// MFB_LEAF_MAX (1..15) overrides it.
int lbvh_leaf_max(int leaf_hint) {
  static const int leaf_env = [] {
    const char* e = std::getenv("MFB_LEAF_MAX");
    const int v = e ? std::atoi(e) : 0;
    return v >= 1 && v <= kLeafCountMax ? v : 0;
  }();
  return leaf_env ? leaf_env : (leaf_hint >= 1 && leaf_hint <= kLeafCountMax ? leaf_hint : kLeafMaxDefault);
}

// segment-tree node boxes (MFB_SEGTREE=0: the bottom-up refit climb)
static bool lbvh_segtree() {
  static const bool on = [] {
    const char* e = std::getenv("MFB_SEGTREE");
    return !(e && e[0] == '0');
  }();
  return on;
}

void lbvh_layout(Ctx& ctx, const DevMesh& m, Lbvh& out, const std::string& tag, int leaf_hint) {
  out.leaf_max = lbvh_leaf_max(leaf_hint);
  const int n = m.nf;
  // leaf refs hold first < 2^27 (bake.cuh), which also bounds the traversal
  // stacks: a root-to-leaf path's Karras deltas strictly increase over the 30
  // Morton bits and the 27 index bits, so depth <= 58 < kStackMax
  if (n >= kMaxFaces)
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: the device LBVH supports fewer than 2^27 faces");
  out.n_tris = n;
  out.n_nodes = n > 1 ? n - 1 : 0;
  out.nodes = ctx.buf<BNode>(tag + ".nodes", out.n_nodes > 0 ? out.n_nodes : 1);
  out.tris = ctx.buf<BTri>(tag + ".tris", n);
  out.tbox = ctx.buf<TBox>(tag + ".tbox", n);
  static const int plane_env = [] {  // MFB_TPLANE=0 / 1: never / always build the triangle planes
    const char* e = std::getenv("MFB_TPLANE");
    return e ? std::atoi(e) : -1;
  }();
  const bool planes = plane_env < 0 ? out.leaf_max >= kPlaneLeafMin : plane_env != 0;
  out.tplane = planes ? ctx.buf<TPlane>(tag + ".tplane", n) : nullptr;
  out.lplane = planes ? ctx.buf<LPlane>(tag + ".lplane", n) : nullptr;
  // node boxes need every reachable node listed (the segment-tree build's list)
  out.nplane = planes && n > 1 && lbvh_segtree() ? ctx.buf<LPlane>(tag + ".nplane", n - 1) : nullptr;
  out.root_box_dev = ctx.buf<float>(tag + ".rootbox", 8);
  out.root_ref = n > 1 ? 0 : leaf_ref(0, 1);
  out.scene_acc = ctx.buf<unsigned long long>(tag + ".acc", 8);
}

void lbvh_build(Ctx& ctx, cudaStream_t s, const DevMesh& m, Lbvh& out, const std::string& tag, int leaf_hint,
                int* vflags) {
  const int n = m.nf;
  lbvh_layout(ctx, m, out, tag, leaf_hint);
  auto* acc = ctx.buf<unsigned long long>(tag + ".acc", 8);
  auto* keys = ctx.buf<uint32_t>(tag + ".keys", n);
  auto* keys2 = ctx.buf<uint32_t>(tag + ".keys2", n);
  auto* vals = ctx.buf<uint32_t>(tag + ".vals", n);
  auto* vals2 = ctx.buf<uint32_t>(tag + ".vals2", n);
  auto* prim_parent = ctx.buf<int32_t>(tag + ".pparent", n);
  auto* node_parent = ctx.buf<int32_t>(tag + ".nparent", n);
  auto* flags = ctx.buf<int>(tag + ".flags", n);
  auto* starts = ctx.buf<int32_t>(tag + ".starts", n);
  auto* starts_n = ctx.buf<int>(tag + ".starts_n", 1);

  // sort scratch: 3 x 1024 digit histograms + 3 tile counters, look-back status
  auto* hist = ctx.buf<int>(tag + ".hist", 3 * 1024 + 4);
  const int64_t status_words = sort_status_words(n);
  auto* status = ctx.buf<uint32_t>(tag + ".sortst", status_words);
  k_acc_init<<<1, 1024, 0, s>>>(acc, hist);
  ctx.count_launch();
  // segment-tree node boxes (MFB_SEGTREE=0: the bottom-up refit climb)
  const bool use_seg = lbvh_segtree() && n > 1;
  if (out.n_nodes > 0 && !use_seg) ctx.fill(flags, 0, sizeof(int) * out.n_nodes, s);

  const int T = 256;
  const int grid_b = std::min(div_up(std::max(n, m.nv), T), kNumSMs * 8);
  // the chain up to the sort runs with programmatic dependent launch
  launch_pdl(k_bounds, grid_b, T, 0, s, m.pos, m.nv, acc, vflags);
  launch_pdl(k_morton, std::max(1, div_up(n, kMortonThreads * kMortonPer)), kMortonThreads, 0, s, m.pos, m.faces, n,
             acc, keys, vals, hist, status, status_words, m.nv, vflags);
  ctx.count_launch(2);
  // stable 3-pass radix sort (sort.cu): sorted pairs in keys2 / vals2
  SortArgs sa;
  sa.keys = keys;
  sa.vals = vals;
  sa.keys_alt = keys2;
  sa.vals_alt = vals2;
  sa.n = n;
  sa.hist = hist;
  sa.status = status;
  sa.counters = hist + 3 * 1024;
  radix_sort_morton30(ctx, s, sa);

  const int leaf_max = out.leaf_max = lbvh_leaf_max(leaf_hint);
  // repack (gathers) and emit (key searches) both need only the sorted
  // keys / ids: repack runs on the context's helper stream alongside emit
  cudaStream_t rs = ctx.side2 ? ctx.side2 : s;
  auto repack = [&](cudaStream_t st) {
    if (out.tplane)
      k_repack<true><<<div_up(n, T), T, 0, st>>>(m.pos, m.faces, vals2, n, out.tris, out.tbox, out.tplane);
    else
      k_repack<false><<<div_up(n, T), T, 0, st>>>(m.pos, m.faces, vals2, n, out.tris, out.tbox, nullptr);
  };
  if (rs != s) {
    MFB_CUDA_TRY(cudaEventRecord(ctx.lfork, s));
    MFB_CUDA_TRY(cudaStreamWaitEvent(rs, ctx.lfork, 0));
  }
  // segment tree over the leaf-order boxes (node boxes without a refit climb)
  int N = 1;
  while (N < n) N <<= 1;
  TBox* seg = nullptr;
  if (use_seg) {
    seg = ctx.buf<TBox>(tag + ".seg", N);
    // (the repack fused with the first seg levels in 1024-thread CTAs measured
    // slower: the 256-thread gather runs at full occupancy)
    int launches = 2;
    repack(rs);
    launch_pdl(k_seg_leaves, div_up(N, 1024), 1024, 0, rs, out.tbox, n, N, seg);
    for (int L = N >> 10; L > 1; L >>= 10, ++launches) launch_pdl(k_seg_up, div_up(L, 1024), 1024, 0, rs, seg, L);
    ctx.count_launch(launches - 1);
  } else {
    repack(rs);
  }
  if (rs != s) MFB_CUDA_TRY(cudaEventRecord(ctx.ljoin, rs));
  if (n > 1) {
    ctx.fill(starts_n, 0, sizeof(int), s);
    k_emit<<<div_up(n - 1, T), T, 0, s>>>(keys2, n, leaf_max, out.nodes, prim_parent, node_parent, starts,
                                          starts_n, use_seg ? 1 : 0);
    ctx.count_launch();
  }
  if (rs != s) MFB_CUDA_TRY(cudaStreamWaitEvent(s, ctx.ljoin, 0));
  if (seg) {
    // (grid for every internal node; threads past the device count exit)
    k_node_boxes<<<div_up(n - 1, T), T, 0, s>>>(seg, out.tbox, N, n, leaf_max, out.nodes, out.root_box_dev,
                                                    starts, starts_n);
  } else if (n > 1) {
    // starts <= leaf ranges <= n; threads past the device count exit at once
    k_refit_ranges<<<div_up(n, T), T, 0, s>>>(out.tbox, out.nodes, starts, starts_n, out.nodes,
                                                       node_parent, flags, out.root_box_dev);
  } else {
    k_refit<<<1, 32, 0, s>>>(out.tbox, n, out.nodes, prim_parent, node_parent, flags, out.root_box_dev);
  }
  ctx.count_launch(2);
  if (out.lplane) {  // after the boxes: the list and the child refs are final
    k_leaf_planes<<<div_up(std::max(n - 1, 1), T), T, 0, s>>>(out.nodes, out.tris, starts, starts_n, n, out.lplane);
    ctx.count_launch();
  }
  if (out.nplane) {
    k_node_planes<<<kNumSMs * 8, T, 0, s>>>(out.nodes, out.tris, starts, starts_n, out.nplane);
    ctx.count_launch();
  }
  MFB_CUDA_TRY(cudaGetLastError());
  out.root_ref = n > 1 ? 0 : leaf_ref(0, 1);
  out.scene_acc = acc;
}

}  // namespace mfb
