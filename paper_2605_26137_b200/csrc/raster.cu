// raster.cu — rasterizeGBuffer (bake/gbuffer.cpp:92-191) and the per-mesh
// pre-passes it depends on, all on the device:
//   vertex_normals  computeVertexNormals (core/mesh.cpp:24-35): per-vertex
//                   CSR of incident corners, summed in face order
//                   (deterministic, no float atomics);
//   wedge frames    computeWedgeTangents (bake/tangent.cpp:22-82): corner
//                   contributions summed per (vertex, uv) wedge in face order
//                   over the vertex's sorted incident-corner list;
//   reliable faces  reliableFaces (gbuffer.cpp:31-83): lock-free union-find
//                   whose roots are island minima, ratios grouped per island,
//                   median = element size/2 by an exact per-island radix select;
//   face setup      canonical edge functions + texel bbox per face;
//   binning         counting sort of faces into 16x16 texel tiles
//                   (conservative: every tile the face's texel bbox touches);
//   raster          one tile per 256-thread CTA, one texel per thread: exact
//                   reference coverage predicate (tie rule ownsBoundary,
//                   gbuffer.cpp:21-27,146-154), AtlasOverlap detection,
//                   f64 attribute interpolation, coalesced G-buffer stores.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "bake.cuh"

namespace mfb {
namespace {

constexpr int kTile = 16;

struct alignas(16) RasterFace {
  double px[3], py[3];
  double doubled;
  double ox[3], oy[3], dx[3], dy[3], sg[3];
  int x0, y0, x1, y1;  // clamped texel bbox; x0 > x1 when the face is skipped
  int rel, pad[3];     // reliableFaces flag (gbuffer.cpp:74-81), carried for the split raster
};
static_assert(sizeof(RasterFace) % 16 == 0, "RasterFace must stay 16-B aligned");

struct alignas(16) AttrFace {
  double P[9];  // corner positions
  double N[9];  // corner frame normals
  double T[9];  // corner frame tangents
  int reliable;
  int pad;
};

// ------------------------------------------------------------ vertex normals
// Each pre-pass is a __device__ body over one item index, called by its own
// kernel (the dense mesh, mf_wedge_tangents, ...) and by the cooperative
// lowpoly kernel (k_lowpoly_prep), which runs them as grid-synchronised
// phases. No __restrict__ / read-only loads on buffers the cooperative kernel
// produces itself: the non-coherent path could return stale lines.
__device__ __forceinline__ void d_corner_count(const int32_t* faces, int c, int* cnt) {
  atomicAdd(&cnt[faces[c]], 1);
}
__device__ __forceinline__ void d_corner_fill(const int32_t* faces, int c, const int* start, int* cursor, int* list) {
  const int v = faces[c];
  list[start[v] + atomicAdd(&cursor[v], 1)] = c;
}
__device__ __forceinline__ void d_face_area_vec(const double* pos, const int32_t* faces, int f, double* av) {
  const d3 p0 = ld3(pos + 3 * faces[3 * f]), p1 = ld3(pos + 3 * faces[3 * f + 1]),
           p2 = ld3(pos + 3 * faces[3 * f + 2]);
  st3(av + 3 * f, 0.5 * cross(p1 - p0, p2 - p0));  // faceAreaVector, mesh.h:28-31
}
// Sorts vertex v's incident-corner list into face order (valence is small).
__device__ __forceinline__ void d_csr_sort(int v, const int* start, int* list) {
  const int b = start[v], e = start[v + 1];
  for (int i = b + 1; i < e; ++i) {
    const int key = list[i];
    int j = i - 1;
    while (j >= b && list[j] > key) {
      list[j + 1] = list[j];
      --j;
    }
    list[j + 1] = key;
  }
}
// computeVertexNormals (mesh.cpp:24-35): area vectors summed in face order.
__device__ __forceinline__ void d_vertex_sum(int v, const int* start, const int* list, const double* av,
                                             double* out, int renorm) {
  const int b = start[v], e = start[v + 1];
  d3 n = mk3(0.0, 0.0, 0.0);
  for (int i = b; i < e; ++i) n = n + ld3(av + 3 * (list[i] / 3));
  const double len = norm(n);
  if (len > 0) n = n / len;
  if (renorm) {
    const double l2 = norm(n);
    if (l2 > 1e-20) n = n / l2;
  }
  st3(out + 3 * v, n);
}
__device__ __forceinline__ void d_renorm(int v, const double* in, double* out) {
  d3 n = ld3(in + 3 * v);
  const double len = norm(n);
  if (len > 1e-20) n = n / len;
  st3(out + 3 * v, n);
}
__global__ void k_corner_count(const int32_t* __restrict__ faces, int nc, int* __restrict__ cnt) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) d_corner_count(faces, c, cnt);
}
__global__ void k_corner_fill(const int32_t* __restrict__ faces, int nc, const int* __restrict__ start,
                              int* __restrict__ cursor, int* __restrict__ list) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nc) d_corner_fill(faces, c, start, cursor, list);
}
__global__ void k_face_area_vec(const double* __restrict__ pos, const int32_t* __restrict__ faces, int nf,
                                double* __restrict__ av) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_face_area_vec(pos, faces, f, av);
}
__global__ void k_csr_sort(int nv, const int* __restrict__ start, int* __restrict__ list) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) d_csr_sort(v, start, list);
}
__global__ void k_vertex_sum(int nv, const int* __restrict__ start, const int* __restrict__ list,
                             const double* __restrict__ av, double* __restrict__ out, int renorm) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) d_vertex_sum(v, start, list, av, out, renorm);
}
// Dense-mesh vertex normals without a CSR build: each face stores its area
// vector and drops its three corner ids into fixed per-vertex slots
// (kVnSlots; a vertex of higher valence spills the rest into an overflow
// list); the summation orders a vertex's corners in registers and adds the
// area vectors in face order, exactly as computeVertexNormals' face loop
// (mesh.cpp:24-35).
constexpr int kVnSlots = 16;
__global__ void k_vn_slots(const double* __restrict__ pos, const int32_t* __restrict__ faces, int nf, int nv,
                           double* __restrict__ av, int* __restrict__ cnt, int* __restrict__ slots,
                           int* __restrict__ ovf, int ovf_cap) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  // (indices clamped: on the host path this kernel runs beside the LBVH's
  // Morton kernel, which validates and zeroes bad indices; the bake is then
  // discarded with InvalidGeometry)
  int t[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t[k] = faces[3 * f + k];
    if (static_cast<unsigned>(t[k]) >= static_cast<unsigned>(nv)) t[k] = 0;
  }
  const d3 p0 = ld3(pos + 3 * t[0]), p1 = ld3(pos + 3 * t[1]), p2 = ld3(pos + 3 * t[2]);
  st3(av + 3 * f, 0.5 * cross(p1 - p0, p2 - p0));  // faceAreaVector, mesh.h:28-31
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int c = 3 * f + k, v = t[k];
    const int s = atomicAdd(&cnt[v], 1);
    if (s < kVnSlots) {
      slots[static_cast<int64_t>(v) * kVnSlots + s] = c;
    } else {
      const int o = atomicAdd(ovf, 1);
      if (o < ovf_cap) {
        ovf[1 + 2 * o] = v;
        ovf[2 + 2 * o] = c;
      }
    }
  }
}
__global__ void k_vn_sum(int nv, const int* __restrict__ cnt, const int* __restrict__ slots,
                         const int* __restrict__ ovf, const double* __restrict__ av, double* __restrict__ out,
                         int renorm) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int k = cnt[v];
  const int* sl = slots + static_cast<int64_t>(v) * kVnSlots;
  d3 n = mk3(0.0, 0.0, 0.0);
  if (k <= kVnSlots) {
    int c[kVnSlots];
#pragma unroll
    for (int i = 0; i < kVnSlots; ++i) c[i] = i < k ? sl[i] : 0x7fffffff;
#pragma unroll
    for (int i = 1; i < kVnSlots; ++i) {  // insertion sort, fully unrolled (register resident)
#pragma unroll
      for (int j = i; j > 0; --j) {
        const int lo = min(c[j - 1], c[j]), hi = max(c[j - 1], c[j]);
        c[j - 1] = lo;
        c[j] = hi;
      }
    }
#pragma unroll
    for (int i = 0; i < kVnSlots; ++i)
      if (i < k) n = n + ld3(av + 3 * (c[i] / 3));
  } else {
    // valence above kVnSlots (rare): the slots plus this vertex's overflow
    // entries, taken in increasing corner order by repeated minimum search
    const int no = ovf[0];
    int last = -1;
    for (int it = 0; it < k; ++it) {
      int nxt = 0x7fffffff;
      for (int i = 0; i < kVnSlots; ++i) {
        const int c = sl[i];
        if (c > last && c < nxt) nxt = c;
      }
      for (int o = 0; o < no; ++o)
        if (ovf[1 + 2 * o] == v) {
          const int c = ovf[2 + 2 * o];
          if (c > last && c < nxt) nxt = c;
        }
      n = n + ld3(av + 3 * (nxt / 3));
      last = nxt;
    }
  }
  const double len = norm(n);
  if (len > 0) n = n / len;
  if (renorm) {
    const double l2 = norm(n);
    if (l2 > 1e-20) n = n / l2;
  }
  st3(out + 3 * v, n);
}
__global__ void k_renorm(int nv, const double* __restrict__ in, double* __restrict__ out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) d_renorm(v, in, out);
}

// ------------------------------------------------------------ wedge frames
__device__ __forceinline__ void d_wedge_contrib(const double* pos, const int32_t* faces, const double* uvs,
                                                const int32_t* fuv, int f, double* contrib, uint8_t* present) {
  const int t[3] = {faces[3 * f], faces[3 * f + 1], faces[3 * f + 2]};
  const int u[3] = {fuv[3 * f], fuv[3 * f + 1], fuv[3 * f + 2]};
  const d3 p0 = ld3(pos + 3 * t[0]), p1 = ld3(pos + 3 * t[1]), p2 = ld3(pos + 3 * t[2]);
  const double d1x = uvs[2 * u[1]] - uvs[2 * u[0]], d1y = uvs[2 * u[1] + 1] - uvs[2 * u[0] + 1];
  const double d2x = uvs[2 * u[2]] - uvs[2 * u[0]], d2y = uvs[2 * u[2] + 1] - uvs[2 * u[0] + 1];
  const double det = d1x * d2y - d2x * d1y;
  const bool face_ok = !(fabs(det) < 1e-20);
  d3 ft = mk3(0.0, 0.0, 0.0);
  if (face_ok) ft = ((p1 - p0) * d2y - (p2 - p0) * d1y) / det;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int c = 3 * f + k;
    bool ok = face_ok;
    d3 w = mk3(0.0, 0.0, 0.0);
    if (ok) {
      const d3 self = ld3(pos + 3 * t[k]);
      const d3 ea = ld3(pos + 3 * t[(k + 1) % 3]) - self;
      const d3 eb = ld3(pos + 3 * t[(k + 2) % 3]) - self;
      const double la = norm(ea), lb = norm(eb);
      if (la < 1e-20 || lb < 1e-20) {
        ok = false;
      } else {
        double cs = dot(ea, eb) / (la * lb);
        cs = cs < -1.0 ? -1.0 : (cs > 1.0 ? 1.0 : cs);
        w = acos(cs) * ft;
      }
    }
    present[c] = ok ? 1 : 0;
    st3(contrib + 3 * c, w);
  }
}
// Per vertex: each wedge (vertex, uv index) sums its corners' contributions
// in face order (the vertex's corner list is sorted by corner id) - exactly
// the unordered_map accumulation of tangent.cpp:40-63 - and every corner
// receives its wedge's sum.
__device__ __forceinline__ void d_wedge_acc(int v, const int* start, const int* list, const int32_t* fuv,
                                            const double* contrib, const uint8_t* present, double* acc) {
  const int b = start[v], e = start[v + 1];
  for (int i = b; i < e; ++i) {
    const int ui = fuv[list[i]];
    bool seen = false;
    for (int j = b; j < i && !seen; ++j) seen = fuv[list[j]] == ui;
    if (seen) continue;
    d3 sum = mk3(0.0, 0.0, 0.0);
    for (int j = i; j < e; ++j) {
      const int cj = list[j];
      if (fuv[cj] == ui && present[cj]) sum = sum + ld3(contrib + 3 * cj);
    }
    for (int j = i; j < e; ++j) {
      const int cj = list[j];
      if (fuv[cj] == ui) st3(acc + 3 * cj, sum);
    }
  }
}
// frames[c] = {T, B, N}; also fills the raster attribute block when attrs != null.
__device__ __forceinline__ void d_wedge_frames(const int32_t* faces, int c, const double* unitN, const double* acc,
                                               double* frames, AttrFace* attrs, const double* pos) {
  const int v = faces[c];
  d3 N = ld3(unitN + 3 * v);
  if (norm(N) < 1e-20) N = mk3(0.0, 0.0, 1.0);
  d3 t = ld3(acc + 3 * c);
  t = t - N * dot(N, t);
  const double len = norm(t);
  const d3 T = len > 1e-12 ? t / len : any_perpendicular(N);
  if (frames) {
    st3(frames + 9 * c, T);
    st3(frames + 9 * c + 3, cross(N, T));
    st3(frames + 9 * c + 6, N);
  }
  if (attrs) {
    const int f = c / 3, k = c % 3;
    st3(attrs[f].P + 3 * k, ld3(pos + 3 * v));
    st3(attrs[f].N + 3 * k, N);
    st3(attrs[f].T + 3 * k, T);
  }
}
__global__ void k_wedge_contrib(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                                const double* __restrict__ uvs, const int32_t* __restrict__ fuv, int nf,
                                double* __restrict__ contrib, uint8_t* __restrict__ present) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_wedge_contrib(pos, faces, uvs, fuv, f, contrib, present);
}
__global__ void k_wedge_acc(int nv, const int* __restrict__ start, const int* __restrict__ list,
                            const int32_t* __restrict__ fuv, const double* __restrict__ contrib,
                            const uint8_t* __restrict__ present, double* __restrict__ acc) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nv) d_wedge_acc(v, start, list, fuv, contrib, present, acc);
}
__global__ void k_wedge_frames(const int32_t* __restrict__ faces, int nf, const double* __restrict__ unitN,
                               const double* __restrict__ acc, double* __restrict__ frames,
                               AttrFace* __restrict__ attrs, const double* __restrict__ pos) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < 3 * nf) d_wedge_frames(faces, c, unitN, acc, frames, attrs, pos);
}

// ------------------------------------------------------------ reliable faces
// find with path halving: parent[x] <- parent[parent[x]] (a benign race:
// any ancestor is a valid parent, and roots never change except by the CAS).
__device__ __forceinline__ int uf_find(int* parent, int x) {
  int p = __ldcg(&parent[x]);
  while (p != x) {
    const int gp = __ldcg(&parent[p]);
    if (gp != p) atomicCAS(&parent[x], p, gp);
    x = p;
    p = gp;
  }
  return x;
}
// Hook the larger root under the smaller one, so every root is its island's
// minimum UV index — exactly the reference's parent[max] = min (gbuffer.cpp:41-45).
__device__ __forceinline__ void d_uf_unite(const int32_t* fuv, int f, int* parent) {
  for (int e = 1; e <= 2; ++e) {
    int a = fuv[3 * f], b = fuv[3 * f + e];
    for (;;) {
      a = uf_find(parent, a);
      b = uf_find(parent, b);
      if (a == b) break;
      const int hi = a > b ? a : b, lo = a > b ? b : a;
      if (atomicCAS(&parent[hi], hi, lo) == hi) break;
      a = hi;
      b = lo;
    }
  }
}
__device__ __forceinline__ void d_face_ratio(const double* pos, const int32_t* faces, const double* uvs,
                                             const int32_t* fuv, int f, const int* parent, double* uv_area,
                                             double* ratio, int* island, int* count) {
  const int u0 = fuv[3 * f], u1 = fuv[3 * f + 1], u2 = fuv[3 * f + 2];
  const double a = 0.5 * fabs(cross2(uvs[2 * u1] - uvs[2 * u0], uvs[2 * u1 + 1] - uvs[2 * u0 + 1],
                                     uvs[2 * u2] - uvs[2 * u0], uvs[2 * u2 + 1] - uvs[2 * u0 + 1]));
  const d3 p0 = ld3(pos + 3 * faces[3 * f]), p1 = ld3(pos + 3 * faces[3 * f + 1]),
           p2 = ld3(pos + 3 * faces[3 * f + 2]);
  const double surf = norm(0.5 * cross(p1 - p0, p2 - p0));  // faceArea, mesh.h:33
  const int isl = uf_find(const_cast<int*>(parent), u0);  // = parent[u0] once flattened
  double r = -1.0;
  if (surf > 1e-20) {
    r = a / surf;
    atomicAdd(&count[isl], 1);
  }
  uv_area[f] = a;
  ratio[f] = r;
  island[f] = isl;
}
// Groups the sampled ratios by island (order within an island is irrelevant
// to its median).
__device__ __forceinline__ void d_island_fill(int f, const double* ratio, const int* island, const int* start,
                                              int* cursor, unsigned long long* items) {
  if (ratio[f] < 0.0) return;
  const int isl = island[f];
  // ratio >= 0, so its IEEE bit pattern orders like its value
  items[start[isl] + atomicAdd(&cursor[isl], 1)] = static_cast<unsigned long long>(__double_as_longlong(ratio[f]));
}
// Island median = element size/2 of the island's sorted ratios (the
// std::nth_element of gbuffer.cpp:69-71), by an exact 8-pass radix select
// over the 64-bit patterns; one CTA per island (any blockDim >= 32).
struct SelectSmem {
  int hist[256];
  unsigned long long prefix;
  int k;
};
__device__ void d_island_select(int isl, const int* count, const int* start, const unsigned long long* items,
                                double* median, SelectSmem& sm) {
  const int n = count[isl];
  if (n == 0) {
    if (threadIdx.x == 0) median[isl] = 0.0;
    return;
  }
  const unsigned long long* it = items + start[isl];
  if (threadIdx.x == 0) {
    sm.prefix = 0;
    sm.k = n / 2;
  }
  for (int pass = 7; pass >= 0; --pass) {
    const int shift = pass * 8;
    const unsigned long long hi_mask = pass == 7 ? 0ull : (~0ull << (shift + 8));
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sm.hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = sm.prefix;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long v = it[i];
      if ((v & hi_mask) == prefix) atomicAdd(&sm.hist[(v >> shift) & 0xff], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // warp 0: bucket holding rank k. Lane l owns buckets 8l..8l+7; an
      // inclusive scan of the lane sums finds the lane, then its 8 buckets.
      const int lane = threadIdx.x;
      int c[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = sm.hist[8 * lane + j];
        sum += c[j];
      }
      int incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      const int k = sm.k;
      const unsigned owner = __ballot_sync(0xffffffffu, incl > k);  // k < n: some lane holds it
      const int ol = __ffs(owner) - 1;
      if (lane == ol) {
        int kk = k - (incl - sum), b = 8 * lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (kk < c[j]) break;
          kk -= c[j];
          ++b;
        }
        sm.k = kk;
        sm.prefix = prefix | (static_cast<unsigned long long>(b) << shift);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) median[isl] = __longlong_as_double(static_cast<long long>(sm.prefix));
  __syncthreads();  // sm is reused by the caller's next island
}
__global__ void k_iota(int n, int* __restrict__ a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
__global__ void k_uf_unite(const int32_t* __restrict__ fuv, int nf, int* parent) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_uf_unite(fuv, f, parent);
}
__global__ void k_uf_flatten(int n, int* parent) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) parent[i] = uf_find(parent, i);
}
__global__ void k_face_ratio(const double* __restrict__ pos, const int32_t* __restrict__ faces,
                             const double* __restrict__ uvs, const int32_t* __restrict__ fuv, int nf,
                             const int* __restrict__ parent, double* __restrict__ uv_area,
                             double* __restrict__ ratio, int* __restrict__ island, int* __restrict__ count) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_face_ratio(pos, faces, uvs, fuv, f, parent, uv_area, ratio, island, count);
}
__global__ void k_island_fill(int nf, const double* __restrict__ ratio, const int* __restrict__ island,
                              const int* __restrict__ start, int* __restrict__ cursor,
                              unsigned long long* __restrict__ items) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_island_fill(f, ratio, island, start, cursor, items);
}
__global__ void __launch_bounds__(256) k_island_select(int nu, const int* __restrict__ count,
                                                       const int* __restrict__ start,
                                                       const unsigned long long* __restrict__ items,
                                                       double* __restrict__ median) {
  __shared__ SelectSmem sm;
  if (blockIdx.x < nu) d_island_select(blockIdx.x, count, start, items, median, sm);
}

// ------------------------------------------------------------ face setup
// reliable (gbuffer.cpp:74-81) into the face's raster record and attributes;
// runs after the face setup, which leaves rel = 0
__device__ __forceinline__ void d_face_rel(int f, const double* uv_area, const double* ratio, const int* island,
                                           const double* median, RasterFace* rf, AttrFace* attrs) {
  int rel = 0;
  if (!(uv_area[f] < 1e-8) && !(ratio[f] < 0.0)) {
    const double m = median[island[f]];
    if (!(ratio[f] > 100.0 * m || 100.0 * ratio[f] < m)) rel = 1;
  }
  attrs[f].reliable = rel;
  attrs[f].pad = 0;
  if (rf) rf[f].rel = rel;
}
__global__ void k_face_rel(int nf, const double* __restrict__ uv_area, const double* __restrict__ ratio,
                           const int* __restrict__ island, const double* __restrict__ median,
                           RasterFace* __restrict__ rf, AttrFace* __restrict__ attrs) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_face_rel(f, uv_area, ratio, island, median, rf, attrs);
}

// UV-space raster setup of a face (gbuffer.cpp:114-144): everything the
// binning and the coverage test need, from the UVs alone
__device__ __forceinline__ void d_face_setup(const double* uvs, const int32_t* fuv, int f, int res, RasterFace* rf) {
  RasterFace s;
  s.rel = 0;
  s.pad[0] = s.pad[1] = s.pad[2] = 0;
  const double R = static_cast<double>(res);
  const int u[3] = {fuv[3 * f], fuv[3 * f + 1], fuv[3 * f + 2]};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    s.px[k] = uvs[2 * u[k]] * R;
    s.py[k] = uvs[2 * u[k] + 1] * R;
  }
  s.doubled = cross2(s.px[1] - s.px[0], s.py[1] - s.py[0], s.px[2] - s.px[0], s.py[2] - s.py[0]);
  bool skip = s.doubled == 0.0;
  const double orient = s.doubled > 0.0 ? 1.0 : -1.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int i0 = u[k], i1 = u[(k + 1) % 3];
    const int lo = i0 < i1 ? i0 : i1, hi = i0 < i1 ? i1 : i0;
    if (lo == hi) {
      skip = true;
      s.ox[k] = s.oy[k] = s.dx[k] = s.dy[k] = s.sg[k] = 0.0;
      continue;
    }
    s.ox[k] = uvs[2 * lo] * R;
    s.oy[k] = uvs[2 * lo + 1] * R;
    s.dx[k] = uvs[2 * hi] * R - s.ox[k];
    s.dy[k] = uvs[2 * hi + 1] * R - s.oy[k];
    s.sg[k] = (i0 == lo ? 1.0 : -1.0) * orient;
  }
  // Eigen cwiseMin/Max: b < a ? b : a / a < b ? b : a (shim, include/Eigen/Core)
  double lx = s.px[0], ly = s.py[0], hx = s.px[0], hy = s.py[0];
#pragma unroll
  for (int k = 1; k < 3; ++k) {
    lx = s.px[k] < lx ? s.px[k] : lx;
    ly = s.py[k] < ly ? s.py[k] : ly;
    hx = hx < s.px[k] ? s.px[k] : hx;
    hy = hy < s.py[k] ? s.py[k] : hy;
  }
  s.x0 = max(0, static_cast<int>(floor(lx - 0.5)));
  s.y0 = max(0, static_cast<int>(floor(ly - 0.5)));
  s.x1 = min(res - 1, static_cast<int>(ceil(hx - 0.5)));
  s.y1 = min(res - 1, static_cast<int>(ceil(hy - 0.5)));
  if (skip) {
    s.x0 = 1;
    s.x1 = 0;
  }
  rf[f] = s;
}
__global__ void k_face_setup(const double* __restrict__ uvs, const int32_t* __restrict__ fuv, int nf, int res,
                             RasterFace* __restrict__ rf) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_face_setup(uvs, fuv, f, res, rf);
}

// ------------------------------------------------------------ binning
__device__ __forceinline__ bool face_tiles(const RasterFace& s, int row_begin, int row_end, int& tx0,
                                           int& tx1, int& ty0, int& ty1) {
  const int y0 = max(s.y0, row_begin), y1 = min(s.y1, row_end - 1);
  if (s.x0 > s.x1 || y0 > y1) return false;
  tx0 = s.x0 / kTile;
  tx1 = s.x1 / kTile;
  ty0 = (y0 - row_begin) / kTile;
  ty1 = (y1 - row_begin) / kTile;
  return true;
}
__device__ __forceinline__ void d_bin_count(const RasterFace* rf, int f, int row_begin, int row_end, int tiles_x,
                                            int* tile_cnt) {
  int tx0, tx1, ty0, ty1;
  if (!face_tiles(rf[f], row_begin, row_end, tx0, tx1, ty0, ty1)) return;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&tile_cnt[ty * tiles_x + tx], 1);
}
__device__ __forceinline__ void d_bin_fill(const RasterFace* rf, int f, int row_begin, int row_end, int tiles_x,
                                           const int* tile_start, int* cursor, int* bins, int capacity,
                                           int* overflow) {
  int tx0, tx1, ty0, ty1;
  if (!face_tiles(rf[f], row_begin, row_end, tx0, tx1, ty0, ty1)) return;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const int t = ty * tiles_x + tx;
      const int p = tile_start[t] + atomicAdd(&cursor[t], 1);
      if (p < capacity) bins[p] = f;
      else *overflow = 1;
    }
}
__global__ void k_bin_count(const RasterFace* __restrict__ rf, int nf, int row_begin, int row_end,
                            int tiles_x, int* __restrict__ tile_cnt) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < nf) d_bin_count(rf, f, row_begin, row_end, tiles_x, tile_cnt);
}
__global__ void k_bin_fill(const RasterFace* __restrict__ rf, int nf, int row_begin, int row_end,
                           int tiles_x, const int* __restrict__ tile_start, int* __restrict__ cursor,
                           int* __restrict__ bins, int capacity, int* __restrict__ overflow, int ntiles,
                           int* __restrict__ zero4 = nullptr) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f == 0) overflow[1] = tile_start[ntiles];  // the bins' exact total (flags[2])
  if (zero4 && f < 4) zero4[f] = 0;              // query-list counters of the raster that follows
  if (f < nf) d_bin_fill(rf, f, row_begin, row_end, tiles_x, tile_start, cursor, bins, capacity, overflow);
}

// ------------------------------------------------------------ cooperative lowpoly prep
// Everything per corner c of the lowpoly once the incident-corner lists are
// filled (unordered): the corner's vertex list sorted into face order in
// registers (up to 16 corners; longer lists are walked in order by repeated
// minimum selection), the unit vertex
// normal (computeVertexNormals + the tangent.cpp:26-31 re-normalisation, or
// the mesh's own normal), the corner's wedge sum (tangent.cpp:40-63: the
// same-uv corners of the vertex in face order) and its frame
// (tangent.cpp:65-80) into the raster attributes - the work of k_csr_sort,
// k_vertex_sum, k_wedge_acc and k_wedge_frames with one thread per corner
// and independent loads instead of per-vertex dependent chains (each of a
// vertex's corners repeats the vertex's sums: same operands, same order,
// same bits).
__device__ __forceinline__ void d_corner_pass(int c, const int32_t* faces, const int* start, const int* list,
                                              const double* av, const double* nrm, const int32_t* fuv,
                                              const double* contrib, const uint8_t* present, const double* pos,
                                              double* unitN, AttrFace* attrs) {
  constexpr int K = 16;
  const int v = faces[c];
  const int b = start[v], e = start[v + 1], k = e - b;
  const int ui = fuv[c];
  d3 N, sum = mk3(0.0, 0.0, 0.0);
  bool first = false;
  if (k <= K) {
    int cs[K];
#pragma unroll
    for (int i = 0; i < K; ++i) cs[i] = i < k ? list[b + i] : 0x7fffffff;
#pragma unroll
    for (int i = 1; i < K; ++i) {
#pragma unroll
      for (int j = i; j > 0; --j) {
        const int lo = min(cs[j - 1], cs[j]), hi = max(cs[j - 1], cs[j]);
        cs[j - 1] = lo;
        cs[j] = hi;
      }
    }
    first = cs[0] == c;
    d3 n = mk3(0.0, 0.0, 0.0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i < k) {
        const int cj = cs[i];
        if (!nrm) n = n + ld3(av + 3 * (cj / 3));
        if (fuv[cj] == ui && present[cj]) sum = sum + ld3(contrib + 3 * cj);
      }
    }
    N = n;
  } else {  // rare high valence: visit the unsorted list in face order by selection, O(k^2)
    d3 n = mk3(0.0, 0.0, 0.0);
    int prev = -1;
    for (int step = 0; step < k; ++step) {
      int cj = 0x7fffffff;
      for (int i = b; i < e; ++i) {
        const int x = list[i];
        if (x > prev && x < cj) cj = x;
      }
      if (step == 0) first = cj == c;
      if (!nrm) n = n + ld3(av + 3 * (cj / 3));
      if (fuv[cj] == ui && present[cj]) sum = sum + ld3(contrib + 3 * cj);
      prev = cj;
    }
    N = n;
  }
  if (nrm) {
    N = ld3(nrm + 3 * v);
    const double len = norm(N);
    if (len > 1e-20) N = N / len;
  } else {
    const double len = norm(N);
    if (len > 0) N = N / len;
    const double l2 = norm(N);
    if (l2 > 1e-20) N = N / l2;
  }
  if (first) st3(unitN + 3 * v, N);
  if (norm(N) < 1e-20) N = mk3(0.0, 0.0, 1.0);
  const d3 t = sum - N * dot(N, sum);
  const double len = norm(t);
  const d3 T = len > 1e-12 ? t / len : any_perpendicular(N);
  const int f = c / 3, q = c % 3;
  st3(attrs[f].P + 3 * q, ld3(pos + 3 * v));
  st3(attrs[f].N + 3 * q, N);
  st3(attrs[f].T + 3 * q, T);
}

// Block-wide exclusive scan of in[0, n) into out[0, n) by one CTA (the
// callers' last element is a zero pad, so out[n - 1] is the total, as the
// DeviceScan::ExclusiveSum it replaces).
__device__ void block_exclusive_scan(const int* in, int* out, int n) {
  // tiles of 8 x blockDim elements: coalesced independent loads into shared
  // memory, each thread scans 8 consecutive elements, one block scan of the
  // thread sums, coalesced stores; a running carry links the tiles
  constexpr int kPer = 8, kMaxT = 512;
  __shared__ int tile[kPer * kMaxT];
  __shared__ int wsum[32];
  __shared__ int carry_s;
  const int T = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  int carry = 0;
  for (int base = 0; base < n; base += kPer * T) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = base + k * T + t;
      tile[k * T + t] = i < n ? in[i] : 0;
    }
    __syncthreads();
    int v[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      v[k] = tile[kPer * t + k];
      sum += v[k];
    }
    int incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      const int nw = T >> 5;
      int x = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      if (lane < nw) wsum[lane] = x;  // inclusive warp totals
      if (lane == nw - 1) carry_s = x;
    }
    __syncthreads();
    int run = carry + (w ? wsum[w - 1] : 0) + incl - sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      tile[kPer * t + k] = run;
      run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = base + k * T + t;
      if (i < n) out[i] = tile[k * T + t];
    }
    carry += carry_s;
    __syncthreads();  // tile / wsum / carry_s reused
  }
}

struct PrepArgs {
  // lowpoly
  const double* pos;
  const int32_t* faces;
  const double* nrm;  // mesh normals (re-normalised) or null: computed from the corner CSR
  const double* uvs;
  const int32_t* fuv;
  int nv, nf, nu, res;
  // corner CSR + normals + wedges
  int* ccnt;  // 2 (nv + 1): counts, cursors
  int* cstart;
  int* clist;
  double* av;
  double* unitN;
  double* contrib;
  uint8_t* present;
  double* wacc;
  // reliability
  int* parent;
  double* uv_area;
  double* ratio;
  int* island;
  int* icnt;  // 2 (nu + 1)
  int* istart;
  unsigned long long* items;
  double* median;
  int* roots;   // islands with sampled faces
  int* nroots;
  // face records
  AttrFace* attrs;
};

// The lowpoly pre-pass the interpolation needs - vertex normals
// (mesh.cpp:24-35), computeWedgeTangents (tangent.cpp:22-82) and
// reliableFaces (gbuffer.cpp:31-83) - as one cooperative kernel: seven
// phases separated by grid-wide barriers, each phase the same per-item bodies
// the separate kernels run. It replaces ~20 dependent launches (each a few
// us of work on a 20k-face mesh) on two streams, and runs beside the UV
// setup, binning and coverage kernel: only k_interp waits for it (r02 CUPTI
// timeline: the separate kernels took 0.17 ms before the coverage kernel
// could start).
#ifndef MFB_PREP_PROF
#define MFB_PREP_PROF 0  // variant builds: block 0 prints its per-phase times
#endif
__global__ void __launch_bounds__(512) k_lowpoly_prep(PrepArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
#if MFB_PREP_PROF
  unsigned long long ts[8];
  int nts = 0;
  auto stamp = [&] { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[nts])); ++nts; };
  stamp();
#define PREP_SYNC() \
  do {              \
    grid.sync();    \
    stamp();        \
  } while (0)
#else
#define PREP_SYNC() grid.sync()
#endif
  __shared__ SelectSmem sel;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int nc = 3 * a.nf;
  const bool own_n = a.nrm == nullptr;
  // P0: resets, UV setup, wedge contributions, area vectors, parent = iota
  for (int i = gt; i < 2 * (a.nv + 1); i += gs) a.ccnt[i] = 0;
  for (int i = gt; i < 2 * (a.nu + 1); i += gs) a.icnt[i] = 0;
  for (int i = gt; i < a.nu; i += gs) a.parent[i] = i;
  if (gt == 0) *a.nroots = 0;
  for (int f = gt; f < a.nf; f += gs) {
    d_wedge_contrib(a.pos, a.faces, a.uvs, a.fuv, f, a.contrib, a.present);
    if (own_n) d_face_area_vec(a.pos, a.faces, f, a.av);
  }
  PREP_SYNC();
  // P1: corner counts, union-find
  for (int c = gt; c < nc; c += gs) d_corner_count(a.faces, c, a.ccnt);
  for (int f = gt; f < a.nf; f += gs) d_uf_unite(a.fuv, f, a.parent);
  PREP_SYNC();
  // P2: corner scan (one CTA); per-face ratios and island counts (the
  // roots are final: find without flattening)
  if (blockIdx.x == 0) block_exclusive_scan(a.ccnt, a.cstart, a.nv + 1);
  for (int f = gt; f < a.nf; f += gs)
    d_face_ratio(a.pos, a.faces, a.uvs, a.fuv, f, a.parent, a.uv_area, a.ratio, a.island, a.icnt);
  PREP_SYNC();
  // P3: corner lists, island scan
  for (int c = gt; c < nc; c += gs) d_corner_fill(a.faces, c, a.cstart, a.ccnt + a.nv + 1, a.clist);
  if (blockIdx.x == (gridDim.x > 1 ? 1 : 0)) block_exclusive_scan(a.icnt, a.istart, a.nu + 1);
  PREP_SYNC();
  // P4: per vertex normals, wedges and corner frames; island ratio lists
  for (int c = gt; c < nc; c += gs)
    d_corner_pass(c, a.faces, a.cstart, a.clist, a.av, a.nrm, a.fuv, a.contrib, a.present, a.pos, a.unitN,
                  a.attrs);
  for (int f = gt; f < a.nf; f += gs) d_island_fill(f, a.ratio, a.island, a.istart, a.icnt + a.nu + 1, a.items);
  // the islands with sampled faces (a handful of roots among nu UV indices)
  for (int isl = gt; isl < a.nu; isl += gs) {
    const bool has = a.icnt[isl] > 0;
    if (!has) a.median[isl] = 0.0;
    const unsigned m = __ballot_sync(__activemask(), has);
    if (!m) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(a.nroots, __popc(m));
    base = __shfl_sync(__activemask(), base, leader);
    if (has) a.roots[base + __popc(m & ((1u << lane) - 1u))] = isl;
  }
  PREP_SYNC();
  // P5: island medians (one CTA per island with samples)
  const int nroots = __ldcg(a.nroots);
  for (int r = blockIdx.x; r < nroots; r += gridDim.x)
    d_island_select(__ldcg(&a.roots[r]), a.icnt, a.istart, a.items, a.median, sel);
  PREP_SYNC();
  // P6: reliable flags
  for (int f = gt; f < a.nf; f += gs) d_face_rel(f, a.uv_area, a.ratio, a.island, a.median, nullptr, a.attrs);
#if MFB_PREP_PROF
  stamp();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("[prep] %d CTAs  phases us: %.1f %.1f %.1f %.1f %.1f %.1f %.1f  total %.1f\n", gridDim.x,
           (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
           (ts[5] - ts[4]) * 1e-3, (ts[6] - ts[5]) * 1e-3, (ts[7] - ts[6]) * 1e-3, (ts[7] - ts[0]) * 1e-3);
#endif
#undef PREP_SYNC
}


// ------------------------------------------------------------ raster
__device__ __forceinline__ bool owns_boundary(double dx, double dy) {
  if (dy != 0.0) return dy > 0.0;
  return dx < 0.0;
}

constexpr int kChunk = 32;

// Texel of thread t in a 16x16 tile: 8 warps of 8x4 texels (so a warp's
// compacted queries are spatial neighbours).
__device__ __forceinline__ void tile_texel(int t, int& lx, int& ly) {
  const int w = t >> 5, l = t & 31;
  lx = (w & 1) * 8 + (l & 7);
  ly = (w >> 1) * 4 + (l >> 3);
}

// Block-wide compaction of this thread's query flag: returns the query slot
// (or -1). One atomicAdd per block on the global counter.
__device__ __forceinline__ int compact_slot(bool is_q, int* counter, int capacity, int* overflow,
                                            bool extra = false, unsigned long long* extra_count = nullptr,
                                            int* band_add = nullptr) {
  __shared__ int warp_base[8];
  __shared__ int warp_extra[8];
  __shared__ int block_base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, is_q);
  const unsigned me = __ballot_sync(0xffffffffu, extra);
  if (lane == 0) {
    warp_base[w] = __popc(m);
    warp_extra[w] = __popc(me);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0, ex = 0;
    for (int k = 0; k < (blockDim.x >> 5); ++k) {
      const int c = warp_base[k];
      warp_base[k] = acc;
      acc += c;
      ex += warp_extra[k];
    }
    block_base = acc ? atomicAdd(counter, acc) : 0;
    if (acc && block_base + acc > capacity) *overflow = 1;
    if (band_add && acc) {  // slots actually granted to this block
      const int got = min(acc, capacity - block_base);
      if (got > 0) atomicAdd(band_add, got);
    }
    if (extra_count && ex) atomicAdd(extra_count, static_cast<unsigned long long>(ex));
  }
  __syncthreads();
  if (!is_q) return -1;
  const int slot = block_base + warp_base[w] + __popc(m & ((1u << lane) - 1u));
  return slot < capacity ? slot : -1;
}

// Writes one query record into the list.
__device__ __forceinline__ void store_query(const QueryList& q, int slot, int64_t gi, const float* P,
                                            const float* Nf, const float* Tf, const float* Bf) {
  if (slot < 0) return;
  const int idx = slot;
  q.qpos[idx] = make_float4(P[0], P[1], P[2], __int_as_float(static_cast<int>(gi)));
  float* t = q.qtbn + 9ll * idx;
  t[0] = Tf[0];
  t[1] = Tf[1];
  t[2] = Tf[2];
  t[3] = Bf[0];
  t[4] = Bf[1];
  t[5] = Bf[2];
  t[6] = Nf[0];
  t[7] = Nf[1];
  t[8] = Nf[2];
}

// Fused-mode stores of one texel: valid mask, raw map for non-query texels,
// the query record otherwise (pass A for even (x, y), else pass B), and the
// debug planes.
__device__ __forceinline__ void emit_fused(int64_t gi, int x, int y, bool in, uint8_t valid, uint8_t rel,
                                           const float* P, const float* Nf, const float* Tf, const float* Bf,
                                           uint8_t* gvalid, const RasterFused& fo, int* overflow) {
  const bool is_q = in && valid && rel;
  // one block-level compaction; the valid-texel count rides along
  const int slot = compact_slot(is_q, fo.q.count, fo.q.capacity, overflow, in && valid != 0, fo.valid_count);
  if (!in) return;
  if (gvalid) gvalid[gi] = valid;
  if (!is_q) {
    px_store(fo.rgb, gi, fo.fmt, valid ? px_neutral(fo.fmt) : px_background(fo.fmt));  // gbuffer.cpp:212-227
    if (fo.dbg_face) fo.dbg_face[gi] = valid ? -2 : -1;
    if (fo.dbg_ts) {
      fo.dbg_ts[3 * gi] = 0.0;
      fo.dbg_ts[3 * gi + 1] = 0.0;
      fo.dbg_ts[3 * gi + 2] = 0.0;
    }
    return;
  }
  store_query(fo.q, slot, gi, P, Nf, Tf, Bf);
}

// gbuffer.cpp:162-186 for texel centre (cx, cy) inside face `sfc`: f64
// barycentrics, position, renormalised normal, Gram-Schmidt tangent,
// bitangent = N x T, stored as f32 (the G-buffer's types).
__device__ __forceinline__ void interp_texel(const RasterFace& sfc, const AttrFace& a, double cx, double cy,
                                             float* P, float* Nf, float* Tf, float* Bf) {
  const double px0 = sfc.px[0], py0 = sfc.py[0], px1 = sfc.px[1], py1 = sfc.py[1], px2 = sfc.px[2],
               py2 = sfc.py[2];
  const double w0 = cross2(px2 - px1, py2 - py1, cx - px1, cy - py1) / sfc.doubled;
  const double w1 = cross2(px0 - px2, py0 - py2, cx - px2, cy - py2) / sfc.doubled;
  const double w2 = cross2(px1 - px0, py1 - py0, cx - px0, cy - py0) / sfc.doubled;
  const d3 pos = (w0 * ld3(a.P) + w1 * ld3(a.P + 3)) + w2 * ld3(a.P + 6);
  d3 n = (w0 * ld3(a.N) + w1 * ld3(a.N + 3)) + w2 * ld3(a.N + 6);
  const double nl = norm(n);
  n = nl > 1e-12 ? n / nl : ld3(a.N);
  d3 tg = (w0 * ld3(a.T) + w1 * ld3(a.T + 3)) + w2 * ld3(a.T + 6);
  tg = tg - n * dot(n, tg);
  const double tl = norm(tg);
  tg = tl > 1e-12 ? tg / tl : any_perpendicular(n);
  const d3 bt = cross(n, tg);
  P[0] = __double2float_rn(pos.x);
  P[1] = __double2float_rn(pos.y);
  P[2] = __double2float_rn(pos.z);
  Nf[0] = __double2float_rn(n.x);
  Nf[1] = __double2float_rn(n.y);
  Nf[2] = __double2float_rn(n.z);
  Tf[0] = __double2float_rn(tg.x);
  Tf[1] = __double2float_rn(tg.y);
  Tf[2] = __double2float_rn(tg.z);
  Bf[0] = __double2float_rn(bt.x);
  Bf[1] = __double2float_rn(bt.y);
  Bf[2] = __double2float_rn(bt.z);
}

// Split raster, second kernel: one thread per compacted query (texel, face)
// written by k_raster<2>; interpolates exactly as the fused path and writes
// the same query record. No barriers, full SIMT width for the f64 chain.
// (__launch_bounds__(256, 5 | 6): 48 / 40 registers, 1.425 / 1.439 vs 1.425 ms per bake at B)
__global__ void __launch_bounds__(256) k_interp(const RasterFace* __restrict__ rf,
                                                const AttrFace* __restrict__ attrs,
                                                const int2* __restrict__ pend, const int* __restrict__ count,
                                                int res, int g_row0, QueryList q) {
  const int n = *count;
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int2 nxt = i < n ? pend[i] : make_int2(0, 0);
  for (; i < n; i += stride) {
    const int2 tf = nxt;
    if (i + stride < n) nxt = pend[i + stride];
    const int yr = tf.x / res, x = tf.x - yr * res;
    const double cx = x + 0.5, cy = (yr + g_row0) + 0.5;
    if (!attrs[tf.y].reliable) {  // gbuffer.cpp:218-227: not a query; texel id stored as ~gi
      q.qpos[i] = make_float4(0.f, 0.f, 0.f, __int_as_float(~tf.x));
      continue;
    }
    float P[3], Nf[3], Tf[3], Bf[3];
    interp_texel(rf[tf.y], attrs[tf.y], cx, cy, P, Nf, Tf, Bf);
    store_query(q, i, tf.x, P, Nf, Tf, Bf);
  }
}

#ifndef MFB_RASTER_MINB
#define MFB_RASTER_MINB 6  // 40 registers: 6 CTAs per SM (measured 1.676 -> 1.652 ms per bake at config B; 5: 1.660)
#endif
#if MFB_RASTER_MINB > 0
#define MFB_RASTER_BOUNDS __launch_bounds__(256, MFB_RASTER_MINB)
#else
#define MFB_RASTER_BOUNDS __launch_bounds__(256)
#endif
// kMode 0: full G-buffer planes (mf_raster_gbuffer); 1: fused bake, query
// records interpolated in-kernel; 2: fused bake, split: coverage and
// compaction here, (texel, face) pairs to fo.pend, k_interp interpolates.
template <int kMode>
__global__ void MFB_RASTER_BOUNDS k_raster(const RasterFace* __restrict__ rf,
                                                const AttrFace* __restrict__ attrs,
                                                const int* __restrict__ tile_start,
                                                const int* __restrict__ bins, int capacity, int res,
                                                int row_begin, int row_end, int g_row0,
                                                float* __restrict__ gpos, float* __restrict__ gnrm,
                                                float* __restrict__ gtan, float* __restrict__ gbit,
                                                uint8_t* __restrict__ gvalid, uint8_t* __restrict__ grel,
                                                int* __restrict__ flags,
                                                unsigned long long* __restrict__ row_counts, RasterFused fo) {
  __shared__ RasterFace sf[kChunk];
  __shared__ int sfid[kChunk];
  const int tiles_x = (res + kTile - 1) / kTile;
  const int t = blockIdx.x;
  const int tx = t % tiles_x, ty = t / tiles_x;
  int lx, ly;
  tile_texel(threadIdx.x, lx, ly);
  const int x = tx * kTile + lx;
  const int y = row_begin + ty * kTile + ly;
  const bool in = x < res && y < row_end;
  const double cx = x + 0.5, cy = y + 0.5;
  const int b = tile_start[t], e = min(tile_start[t + 1], capacity);
  int cover = -1, hits = 0;
  for (int base = b; base < e; base += kChunk) {
    const int n = min(kChunk, e - base);
    __syncthreads();
    {
      const int words = n * static_cast<int>(sizeof(RasterFace) / 16);
      for (int w = threadIdx.x; w < words; w += blockDim.x) {
        const int i = w / static_cast<int>(sizeof(RasterFace) / 16);
        const int o = w % static_cast<int>(sizeof(RasterFace) / 16);
        const int f = bins[base + i];
        reinterpret_cast<float4*>(&sf[i])[o] = __ldg(reinterpret_cast<const float4*>(&rf[f]) + o);
        if (o == 0) sfid[i] = f;
      }
    }
    __syncthreads();
    if (in) {
      for (int i = 0; i < n; ++i) {
        const RasterFace& sfc = sf[i];
        if (x < sfc.x0 || x > sfc.x1 || y < sfc.y0 || y > sfc.y1) continue;
        bool inside = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double ev = sfc.sg[k] * cross2(sfc.dx[k], sfc.dy[k], cx - sfc.ox[k], cy - sfc.oy[k]);
          if (ev < 0.0 || (ev == 0.0 && !owns_boundary(sfc.sg[k] * sfc.dx[k], sfc.sg[k] * sfc.dy[k]))) {
            inside = false;
            break;
          }
        }
        if (!inside) continue;
        ++hits;
        if (cover < 0 || sfid[i] < cover) cover = sfid[i];
      }
    }
  }
  if (hits > 1) atomicExch(&flags[0], 1);
  const int64_t gi = static_cast<int64_t>(y - g_row0) * res + x;
  float P[3] = {0.f, 0.f, 0.f}, Nf[3] = {0.f, 0.f, 0.f}, Tf[3] = {0.f, 0.f, 0.f}, Bf[3] = {0.f, 0.f, 0.f};
  uint8_t valid = 0, rel = 0;
  if (kMode != 2 && in && cover >= 0) {
    interp_texel(rf[cover], attrs[cover], cx, cy, P, Nf, Tf, Bf);
    valid = 1;
    rel = static_cast<uint8_t>(attrs[cover].reliable);
  }
  if (kMode == 2 && in && cover >= 0) {
    // late reliability: every valid texel is compacted as a query; k_interp
    // (which runs after the reliability pass) turns the texels of unreliable
    // faces into dead records the transfer encodes as (128, 128, 255)
    valid = 1;
    rel = 1;
  }
  if (row_counts) {
    // warp = 8 columns x 4 rows: lanes 8r..8r+7 share row r
    const unsigned m = __ballot_sync(0xffffffffu, in && valid);
    const int lane = threadIdx.x & 31;
    if (lane < 4) {
      const unsigned rowbits = (m >> (8 * lane)) & 0xffu;
      const int yr = row_begin + ty * kTile + (threadIdx.x >> 6) * 4 + lane;
      if (rowbits && yr < row_end) atomicAdd(&row_counts[yr - row_begin], static_cast<unsigned long long>(__popc(rowbits)));
    }
  }
  if (kMode == 1) {
    emit_fused(gi, x, y, in, valid, rel, P, Nf, Tf, Bf, gvalid, fo, &flags[3]);
    return;
  }
  if (kMode == 2) {
    const bool is_q = in && valid && rel;
    if (fo.tile_state) {  // coverage class of this 16x16 tile (the dilation's tile skip)
      const int nin = __syncthreads_count(in), nval = __syncthreads_count(in && valid);
      if (threadIdx.x == 0) fo.tile_state[t] = nval == 0 ? 0 : (nval == nin ? 2 : 1);
    }
    int* band_add = fo.band_tot ? fo.band_tot + (row_begin + ty * kTile - g_row0) / fo.band_rows : nullptr;
    const int slot = compact_slot(is_q, fo.q.count, fo.q.capacity, &flags[3], in && valid != 0, fo.valid_count,
                                  band_add);
    if (!in) return;
    if (gvalid) gvalid[gi] = fo.qslot && is_q ? 3 : valid;
    if (is_q) {
      if (slot >= 0) {
        fo.pend[slot] = make_int2(static_cast<int>(gi), cover);
        if (fo.qslot) {
          fo.qslot[gi] = slot;
          fo.dep_head[slot] = -1;
        }
      }
      return;
    }
    px_store(fo.rgb, gi, fo.fmt, valid ? px_neutral(fo.fmt) : px_background(fo.fmt));  // gbuffer.cpp:212-227
    if (fo.dbg_face) fo.dbg_face[gi] = valid ? -2 : -1;
    if (fo.dbg_ts) {
      fo.dbg_ts[3 * gi] = 0.0;
      fo.dbg_ts[3 * gi + 1] = 0.0;
      fo.dbg_ts[3 * gi + 2] = 0.0;
    }
    return;
  }
  if (!in) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    gpos[3 * gi + k] = P[k];
    gnrm[3 * gi + k] = Nf[k];
    gtan[3 * gi + k] = Tf[k];
    gbit[3 * gi + k] = Bf[k];
  }
  gvalid[gi] = valid;
  grel[gi] = rel;
}

// Query list from a full G-buffer slab (mf_transfer_normals), same tiling.
__global__ void __launch_bounds__(256) k_gbuffer_queries(int res, int rows, const float* __restrict__ gpos,
                                                         const float* __restrict__ gnrm,
                                                         const float* __restrict__ gtan,
                                                         const float* __restrict__ gbit,
                                                         const uint8_t* __restrict__ gvalid,
                                                         const uint8_t* __restrict__ grel, RasterFused fo,
                                                         int* overflow) {
  const int tiles_x = (res + kTile - 1) / kTile;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  int lx, ly;
  tile_texel(threadIdx.x, lx, ly);
  const int x = tx * kTile + lx, y = ty * kTile + ly;
  const bool in = x < res && y < rows;
  const int64_t gi = static_cast<int64_t>(y) * res + x;
  uint8_t valid = 0, rel = 0;
  float P[3] = {0, 0, 0}, N[3] = {0, 0, 0}, T[3] = {0, 0, 0}, B[3] = {0, 0, 0};
  if (in) {
    valid = gvalid[gi];
    rel = grel[gi];
    for (int k = 0; k < 3; ++k) {
      P[k] = gpos[3 * gi + k];
      N[k] = gnrm[3 * gi + k];
      T[k] = gtan[3 * gi + k];
      B[k] = gbit[3 * gi + k];
    }
  }
  emit_fused(gi, x, y, in, valid, rel, P, N, T, B, nullptr, fo, overflow);
}



}  // namespace

// ---------------------------------------------------------------- host side
namespace {
// Incident-corner CSR of a mesh: start[v]..start[v+1] lists the corners 3f+k
// of vertex v in face order.
void corner_csr(Ctx& ctx, cudaStream_t s, const DevMesh& m, const std::string& tag, int** start_out,
                int** list_out) {
  const int T = 256;
  const int nc = 3 * m.nf;
  int* cnt = ctx.buf<int>(tag + ".csr.cc", 2 * (m.nv + 1));  // counts, then fill cursors: one fill
  int* cursor = cnt + m.nv + 1;
  int* start = ctx.buf<int>(tag + ".csr.start", m.nv + 1);
  int* list = ctx.buf<int>(tag + ".csr.list", nc);
  ctx.fill(cnt, 0, sizeof(int) * 2 * (m.nv + 1), s);
  k_corner_count<<<div_up(nc, T), T, 0, s>>>(m.faces, nc, cnt);
  scan_exclusive(ctx, s, cnt, start, m.nv + 1, tag + ".csr");
  k_corner_fill<<<div_up(nc, T), T, 0, s>>>(m.faces, nc, start, cursor, list);
  k_csr_sort<<<div_up(m.nv, T), T, 0, s>>>(m.nv, start, list);
  ctx.count_launch(3);
  *start_out = start;
  *list_out = list;
}

void normals_from_csr(Ctx& ctx, cudaStream_t s, const DevMesh& m, const int* start, const int* list,
                      double* out, bool renorm, const std::string& tag) {
  const int T = 256;
  double* av = ctx.buf<double>(tag + ".vn.av", 3 * static_cast<size_t>(m.nf));
  k_face_area_vec<<<div_up(m.nf, T), T, 0, s>>>(m.pos, m.faces, m.nf, av);
  k_vertex_sum<<<div_up(m.nv, T), T, 0, s>>>(m.nv, start, list, av, out, renorm ? 1 : 0);
  ctx.count_launch(2);
}
}  // namespace

void vertex_normals(Ctx& ctx, cudaStream_t s, const DevMesh& m, double* out, bool renorm,
                    const std::string& tag) {
  const int T = 256;
  if (m.has_normals()) {
    if (renorm) {
      k_renorm<<<div_up(m.nv, T), T, 0, s>>>(m.nv, m.nrm, out);
      ctx.count_launch();
    } else {
      MFB_CUDA_TRY(cudaMemcpyAsync(out, m.nrm, sizeof(double) * 3 * m.nv, cudaMemcpyDeviceToDevice, s));
    }
    return;
  }
  // per-vertex corner slots + in-register ordering inside the summation kernel
  int* cnt = ctx.buf<int>(tag + ".vn.cnt", static_cast<size_t>(m.nv) + 1);  // [nv]: overflow count
  int* slots = ctx.buf<int>(tag + ".vn.slots", static_cast<size_t>(m.nv) * kVnSlots);
  const int ovf_cap = 3 * m.nf;
  int* ovf = ctx.buf<int>(tag + ".vn.ovf", 1 + 2 * static_cast<size_t>(ovf_cap));
  double* av = ctx.buf<double>(tag + ".vn.av", 3 * static_cast<size_t>(m.nf));
  ctx.fill(cnt, 0, sizeof(int) * (m.nv + 1), s);
  ctx.fill(ovf, 0, sizeof(int), s);
  k_vn_slots<<<div_up(m.nf, T), T, 0, s>>>(m.pos, m.faces, m.nf, m.nv, av, cnt, slots, ovf, ovf_cap);
  k_vn_sum<<<div_up(m.nv, T), T, 0, s>>>(m.nv, cnt, slots, ovf, av, out, renorm ? 1 : 0);
  ctx.count_launch(2);
  MFB_CUDA_TRY(cudaGetLastError());
}

namespace {
// computeWedgeTangents (tangent.cpp:22-82); shared by prepare_lowpoly and wedge_frames.
void wedge_pipeline(Ctx& ctx, cudaStream_t s, const DevMesh& lo, double* frames, AttrFace* attrs) {
  const int T = 256;
  const int nf = lo.nf, nc = 3 * nf;
  int *start, *list;
  corner_csr(ctx, s, lo, "lo", &start, &list);
  double* unitN = ctx.buf<double>("lo.unitN", 3 * static_cast<size_t>(lo.nv));
  if (lo.has_normals()) {
    k_renorm<<<div_up(lo.nv, T), T, 0, s>>>(lo.nv, lo.nrm, unitN);
    ctx.count_launch();
  } else {
    normals_from_csr(ctx, s, lo, start, list, unitN, true, "lo");
  }
  double* contrib = ctx.buf<double>("lo.wt.contrib", 3 * static_cast<size_t>(nc));
  uint8_t* present = ctx.buf<uint8_t>("lo.wt.present", nc);
  double* acc = ctx.buf<double>("lo.wt.acc", 3 * static_cast<size_t>(nc));
  k_wedge_contrib<<<div_up(nf, T), T, 0, s>>>(lo.pos, lo.faces, lo.uvs, lo.fuv, nf, contrib, present);
  k_wedge_acc<<<div_up(lo.nv, T), T, 0, s>>>(lo.nv, start, list, lo.fuv, contrib, present, acc);
  k_wedge_frames<<<div_up(nc, T), T, 0, s>>>(lo.faces, nf, unitN, acc, frames, attrs, lo.pos);
  ctx.count_launch(3);
  MFB_CUDA_TRY(cudaGetLastError());
}
}  // namespace

void wedge_frames(Ctx& ctx, cudaStream_t s, const DevMesh& lo, double* frames_out) {
  wedge_pipeline(ctx, s, lo, frames_out, nullptr);
}

#ifndef MFB_PREP_CTAS
#define MFB_PREP_CTAS 64  // the cooperative prep holds its SMs through every barrier (measured 16: 1.350, 32: 1.273, 64: 1.252, 148: 1.257 ms per bake)
#endif
namespace {
int bin_capacity_for(const Ctx& ctx, int nf, int ntiles) {
  // a bound that holds for ordinary atlases; the bake driver re-runs with
  // the exact total (flags[1] set, total in flags[2]) otherwise
  const int64_t cap64 = std::max<int64_t>(ctx.bin_capacity, 8ll * nf + 4ll * ntiles + 1024);
  return static_cast<int>(std::min<int64_t>(cap64, 0x7fffffff));
}

// One cooperative launch of k_lowpoly_prep: wedge frames and reliable
// flags into the faces' raster attributes.
void prepare_lowpoly_coop(Ctx& ctx, cudaStream_t s, const DevMesh& lo, AttrFace* attrs) {
  const int nf = lo.nf, nu = lo.nu, nv = lo.nv, nc = 3 * nf;
  PrepArgs a{};
  a.pos = lo.pos;
  a.faces = lo.faces;
  a.uvs = lo.uvs;
  a.fuv = lo.fuv;
  a.nv = nv;
  a.nf = nf;
  a.nu = nu;
  a.nrm = lo.has_normals() ? lo.nrm : nullptr;
  a.ccnt = ctx.buf<int>("lo.csr.cc", 2 * (nv + 1));
  a.cstart = ctx.buf<int>("lo.csr.start", nv + 1);
  a.clist = ctx.buf<int>("lo.csr.list", nc);
  a.av = ctx.buf<double>("lo.vn.av", 3 * static_cast<size_t>(nf));
  a.unitN = ctx.buf<double>("lo.unitN", 3 * static_cast<size_t>(nv));
  a.contrib = ctx.buf<double>("lo.wt.contrib", 3 * static_cast<size_t>(nc));
  a.present = ctx.buf<uint8_t>("lo.wt.present", nc);
  a.parent = ctx.buf<int>("lo.rel.parent", nu);
  a.uv_area = ctx.buf<double>("lo.rel.uvarea", nf);
  a.ratio = ctx.buf<double>("lo.rel.ratio", nf);
  a.island = ctx.buf<int>("lo.rel.island", nf);
  a.icnt = ctx.buf<int>("lo.rel.cc", 2 * (nu + 1));
  a.istart = ctx.buf<int>("lo.rel.start", nu + 1);
  a.items = ctx.buf<unsigned long long>("lo.rel.items", nf);
  a.median = ctx.buf<double>("lo.rel.median", nu);
  a.roots = ctx.buf<int>("lo.rel.roots", nu + 1);
  a.nroots = a.roots + nu;
  a.attrs = attrs;
  // grid: every CTA co-resident (cooperative launch); the kernel holds its
  // SMs through every barrier, so it stays small beside the LBVH
  static int max_blocks = [] {
    int per_sm = 0;
    MFB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lowpoly_prep, 512, 0));
    return std::max(1, per_sm) * kNumSMs;
  }();
  const int want = div_up(std::max(nc, nu), 512);
  const int grid = std::max(1, std::min(std::min(MFB_PREP_CTAS, max_blocks), want));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MFB_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_lowpoly_prep, a));
  ctx.count_launch();
}

// UV setup fused with the tile counts (the face's record is in registers)
__global__ void k_face_setup_count(const double* __restrict__ uvs, const int32_t* __restrict__ fuv, int nf, int res,
                                   RasterFace* __restrict__ rf, int row_begin, int row_end, int tiles_x,
                                   int* __restrict__ tile_cnt) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  d_face_setup(uvs, fuv, f, res, rf);
  d_bin_count(rf, f, row_begin, row_end, tiles_x, tile_cnt);
}

// Tile binning of the faces over slab rows [b.row0, b.row0 + b.rows) on `s`:
// setup + counts, scan, fill (which also stores the exact total in flags[2]
// and resets the query-list counters).
void bin_faces(Ctx& ctx, cudaStream_t s, const DevMesh& lo, int res, RasterFace* rf, const PrepBinning& b,
               RasterPlan& plan) {
  const int T = 256, nf = lo.nf;
  const int row_begin = b.row0, row_end = b.row0 + b.rows;
  const int tiles_x = (res + kTile - 1) / kTile;
  const int ntiles = tiles_x * ((b.rows + kTile - 1) / kTile);
  int* cnt = ctx.buf<int>("ras.cc", 2 * (ntiles + 1));  // counts, then fill cursors: one fill
  int* cursor = cnt + ntiles + 1;
  int* tstart = ctx.buf<int>("ras.start", ntiles + 1);
  const int capacity = bin_capacity_for(ctx, nf, ntiles);
  int* bins = ctx.buf<int>("ras.bins", capacity);
  ctx.fill(cnt, 0, sizeof(int) * 2 * (ntiles + 1), s);
  k_face_setup_count<<<div_up(nf, T), T, 0, s>>>(lo.uvs, lo.fuv, nf, res, rf, row_begin, row_end, tiles_x, cnt);
  scan_exclusive(ctx, s, cnt, tstart, ntiles + 1, std::string("ras"));
  k_bin_fill<<<div_up(nf, T), T, 0, s>>>(rf, nf, row_begin, row_end, tiles_x, tstart, cursor, bins, capacity,
                                         b.flags + 1, ntiles, b.zero4);
  ctx.count_launch(2);
  if (b.row_counts) ctx.fill(b.row_counts, 0, sizeof(int64_t) * b.rows, s);
  MFB_CUDA_TRY(cudaGetLastError());
  plan.binned = true;
  plan.tile_start = tstart;
  plan.bins = bins;
  plan.capacity = capacity;
}
}  // namespace

void prepare_lowpoly(Ctx& ctx, cudaStream_t s, const DevMesh& lo, int res, RasterPlan& plan,
                     const PrepBinning* bin) {
  auto* rf = ctx.buf<RasterFace>("lo.rf", lo.nf);
  auto* attrs = ctx.buf<AttrFace>("lo.attrs", lo.nf);
  cudaStream_t ws = ctx.aux ? ctx.aux : s;
  if (MFB_COOP_PREP && ws != s) {
    // frames + reliability: one cooperative kernel on aux, beside the
    // setup and binning on s
    MFB_CUDA_TRY(cudaEventRecord(ctx.fork2, s));
    MFB_CUDA_TRY(cudaStreamWaitEvent(ws, ctx.fork2, 0));
    prepare_lowpoly_coop(ctx, ws, lo, attrs);
    MFB_CUDA_TRY(cudaEventRecord(ctx.join2, ws));
    if (bin) {
      bin_faces(ctx, s, lo, res, rf, *bin, plan);
    } else {
      k_face_setup<<<div_up(lo.nf, 256), 256, 0, s>>>(lo.uvs, lo.fuv, lo.nf, res, rf);
      ctx.count_launch();
    }
    plan.faces = rf;
    plan.attrs = attrs;
    plan.nf = lo.nf;
    plan.res = res;
    plan.pending[0] = ctx.join2;
    plan.pending[1] = nullptr;
    return;
  }
  const int T = 256;
  const int nf = lo.nf, nu = lo.nu;
  // Three branches: the UV-only raster setup on `s` (the binning follows it
  // there in raster_gbuffer), the wedge frames (computeWedgeTangents) on aux
  // and the reliability pass (reliableFaces) on aux2, which ends by setting
  // the faces' rel flags after the setup; raster_gbuffer joins both side
  // branches just before the texel kernel. They write disjoint fields.
  cudaStream_t us = ctx.aux2 ? ctx.aux2 : s;
  if (ws != s || us != s) MFB_CUDA_TRY(cudaEventRecord(ctx.fork2, s));
  if (ws != s) MFB_CUDA_TRY(cudaStreamWaitEvent(ws, ctx.fork2, 0));
  if (us != s) MFB_CUDA_TRY(cudaStreamWaitEvent(us, ctx.fork2, 0));
  wedge_pipeline(ctx, ws, lo, nullptr, attrs);
  if (ws != s) MFB_CUDA_TRY(cudaEventRecord(ctx.join2, ws));

  k_face_setup<<<div_up(nf, T), T, 0, s>>>(lo.uvs, lo.fuv, nf, res, rf);
  if (us != s) MFB_CUDA_TRY(cudaEventRecord(ctx.setup_done, s));

  // reliableFaces (gbuffer.cpp:31-83)
  int* parent = ctx.buf<int>("lo.rel.parent", nu);
  double* uv_area = ctx.buf<double>("lo.rel.uvarea", nf);
  double* ratio = ctx.buf<double>("lo.rel.ratio", nf);
  int* island = ctx.buf<int>("lo.rel.island", nf);
  int* count = ctx.buf<int>("lo.rel.cc", 2 * (nu + 1));  // counts, then fill cursors: one fill
  int* cursor = count + nu + 1;
  int* start = ctx.buf<int>("lo.rel.start", nu + 1);
  auto* items = ctx.buf<unsigned long long>("lo.rel.items", nf);
  double* median = ctx.buf<double>("lo.rel.median", nu);
  ctx.fill(count, 0, sizeof(int) * 2 * (nu + 1), us);
  k_iota<<<div_up(nu, T), T, 0, us>>>(nu, parent);
  k_uf_unite<<<div_up(nf, T), T, 0, us>>>(lo.fuv, nf, parent);
  k_uf_flatten<<<div_up(nu, T), T, 0, us>>>(nu, parent);
  k_face_ratio<<<div_up(nf, T), T, 0, us>>>(lo.pos, lo.faces, lo.uvs, lo.fuv, nf, parent, uv_area, ratio, island,
                                            count);
  scan_exclusive(ctx, us, count, start, nu + 1, std::string("lo.rel"));
  k_island_fill<<<div_up(nf, T), T, 0, us>>>(nf, ratio, island, start, cursor, items);
  k_island_select<<<nu, 256, 0, us>>>(nu, count, start, items, median);
  if (us != s) MFB_CUDA_TRY(cudaStreamWaitEvent(us, ctx.setup_done, 0));
  k_face_rel<<<div_up(nf, T), T, 0, us>>>(nf, uv_area, ratio, island, median, rf, attrs);
  ctx.count_launch(9);
  MFB_CUDA_TRY(cudaGetLastError());
  if (us != s) MFB_CUDA_TRY(cudaEventRecord(ctx.join4, us));
  plan.faces = rf;
  plan.attrs = attrs;
  plan.nf = nf;
  plan.res = res;
  plan.pending[0] = ws != s ? ctx.join2 : nullptr;
  plan.pending[1] = us != s ? ctx.join4 : nullptr;
}

void raster_gbuffer(Ctx& ctx, cudaStream_t s, const DevMesh& lo, const RasterPlan& plan, GBufDev& g,
                    int* flags_dev, int64_t* row_counts_dev, const RasterFused* fused) {
  (void)lo;
  const int T = 256;
  const int res = plan.res;
  const int row_begin = g.row0, row_end = g.row0 + g.rows;
  const int tiles_x = (res + kTile - 1) / kTile;
  const int tiles_y = (g.rows + kTile - 1) / kTile;
  const int ntiles = tiles_x * tiles_y;
  auto* rf = static_cast<const RasterFace*>(plan.faces);
  auto* attrs = static_cast<const AttrFace*>(plan.attrs);
  const int* start = plan.tile_start;
  const int* bins = plan.bins;
  int capacity = plan.capacity;
  if (!plan.binned) {  // (the cooperative prep bins, resets the counters and the row counts itself)
    int* cnt = ctx.buf<int>("ras.cc", 2 * (ntiles + 1));  // counts, then fill cursors: one fill
    int* cursor = cnt + ntiles + 1;
    int* tstart = ctx.buf<int>("ras.start", ntiles + 1);
    capacity = bin_capacity_for(ctx, plan.nf, ntiles);
    int* tbins = ctx.buf<int>("ras.bins", capacity);
    ctx.fill(cnt, 0, sizeof(int) * 2 * (ntiles + 1), s);
    k_bin_count<<<div_up(plan.nf, T), T, 0, s>>>(rf, plan.nf, row_begin, row_end, tiles_x, cnt);
    scan_exclusive(ctx, s, cnt, tstart, ntiles + 1, std::string("ras"));
    k_bin_fill<<<div_up(plan.nf, T), T, 0, s>>>(rf, plan.nf, row_begin, row_end, tiles_x, tstart, cursor, tbins,
                                                capacity, flags_dev + 1, ntiles);
    ctx.count_launch(3);
    if (row_counts_dev) ctx.fill(row_counts_dev, 0, sizeof(int64_t) * g.rows, s);
    start = tstart;
    bins = tbins;
  }
  // the wedge frames and reliability branches of prepare_lowpoly: joined
  // before the texel kernel, or (split raster) before the interpolation
  auto join_prep = [&] {
    for (cudaEvent_t e : plan.pending)
      if (e) MFB_CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
  };
  auto* rc = reinterpret_cast<unsigned long long*>(row_counts_dev);
  // Split raster (default): coverage + compaction, then a barrier-free
  // interpolation kernel over the compacted queries. MFB_RASTER_SPLIT=0
  // selects the single fused kernel (A/B).
  const bool split = raster_links_supported();
  if (fused && split) {
    if (!plan.binned) ctx.fill(fused->q.count, 0, 4 * sizeof(int), s);  // [3]: transfer batch cursor
    RasterFused f2 = *fused;
    f2.pend = ctx.buf<int2>("ras.pend", g.texels());
    k_raster<2><<<ntiles, 256, 0, s>>>(rf, attrs, start, bins, capacity, res, row_begin, row_end, g.row0, g.pos,
                                       g.nrm, g.tan, g.bit, g.valid, g.rel, flags_dev, rc, f2);
    if (fused->cover_done) MFB_CUDA_TRY(cudaEventRecord(fused->cover_done, s));
    join_prep();
    k_interp<<<kNumSMs * 8, 256, 0, s>>>(rf, attrs, f2.pend, fused->q.count, res, g.row0, fused->q);
    ctx.count_launch();
  } else if (fused) {
    if (!plan.binned) ctx.fill(fused->q.count, 0, 4 * sizeof(int), s);  // [3]: transfer batch cursor
    join_prep();
    k_raster<1><<<ntiles, 256, 0, s>>>(rf, attrs, start, bins, capacity, res, row_begin, row_end, g.row0, g.pos,
                                       g.nrm, g.tan, g.bit, g.valid, g.rel, flags_dev, rc, *fused);
  } else {
    join_prep();
    k_raster<0><<<ntiles, 256, 0, s>>>(rf, attrs, start, bins, capacity, res, row_begin, row_end, g.row0,
                                       g.pos, g.nrm, g.tan, g.bit, g.valid, g.rel, flags_dev, rc, RasterFused{});
  }
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

bool raster_links_supported() {
  static const bool split = [] {
    const char* e = std::getenv("MFB_RASTER_SPLIT");
    return !(e && e[0] == '0');
  }();
  return split;
}

void gbuffer_queries(Ctx& ctx, cudaStream_t s, const GBufDev& g, const RasterFused& out) {
  const int tiles = ((g.res + kTile - 1) / kTile) * ((g.rows + kTile - 1) / kTile);
  int* overflow = ctx.buf<int>("gq.overflow", 1);
  ctx.fill(out.q.count, 0, 4 * sizeof(int), s);  // [3]: transfer batch cursor
  k_gbuffer_queries<<<tiles, 256, 0, s>>>(g.res, g.rows, g.pos, g.nrm, g.tan, g.bit, g.valid, g.rel, out,
                                          overflow);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

}  // namespace mfb
