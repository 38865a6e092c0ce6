// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the
// product). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load the library built from it.
//
// A thin extern "C" shell around the reference's OWN translation units
// (compiled in place from /root/reference/proj by oracle/Makefile against the
// Eigen-subset shim in include/eigen_shim). Nothing here re-implements the
// algorithm; it converts flat arrays to meshforge::TriangleMesh / GBuffer /
// ImageU8, calls the reference entry points, and copies results back:
//   rasterizeGBuffer / transferNormals / dilateSeams  (src/bake/gbuffer.cpp:92-322)
//   Bvh::closestPointWithin / raycastFirst / brute     (src/spatial/bvh.cpp:100-189)
//   computeWedgeTangents / computeVertexNormals        (src/bake/tangent.cpp:22-82,
//                                                       src/core/mesh.cpp:24-35)
//   fixtures::icosphere / uvSphere / starBlob / random* (tests/support/fixtures.cpp)
//   bakedMeanErrorDeg                                  (src/metrics/metrics.cpp:213-290)
//   texfuse: footprintFromJacobian / edgeMask / backprojectView / incidenceMap /
//   blendViews (src/texfuse/fuse.cpp:39-280), buildMips (src/texfuse/mips.cpp:96-112)
// plus the Appendix-D instrumented replica of the per-texel transfer body
// (gbuffer.cpp:218-248) that reports hit faces, pre-quantisation ts, and the
// N_node / N_tri counters of the reference best-first loop (bvh.cpp:151-176).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <queue>
#include <string>
#include <vector>

#include "meshforge/bake/gbuffer.h"
#include "meshforge/bake/tangent.h"
#include "meshforge/core/error.h"
#include "meshforge/core/mesh.h"
#include "meshforge/core/parallel.h"
#include "meshforge/metrics/metrics.h"
#include "meshforge/render/camera.h"
#include "meshforge/render/raster.h"
#include "meshforge/signfield/sign_grid.h"
#include "meshforge/signfield/watertight.h"
#include "meshforge/visibility/visibility.h"
#include "meshforge/spatial/bvh.h"
#include "meshforge/spatial/tri_geom.h"
#include "meshforge/texfuse/fuse.h"
#include "meshforge/texfuse/mips.h"
#include "mfbake.h"
#include "support/fixtures.h"

using namespace meshforge;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

TriangleMesh toMesh(const mf_mesh_view* v) {
  TriangleMesh m;
  if (!v) return m;
  m.positions.resize(v->n_vertices);
  for (int i = 0; i < v->n_vertices; ++i)
    m.positions[i] = {v->positions[3 * i], v->positions[3 * i + 1], v->positions[3 * i + 2]};
  m.faces.resize(v->n_faces);
  for (int f = 0; f < v->n_faces; ++f)
    m.faces[f] = {v->faces[3 * f], v->faces[3 * f + 1], v->faces[3 * f + 2]};
  if (v->normals && v->n_vertices > 0) {
    m.normals.resize(v->n_vertices);
    for (int i = 0; i < v->n_vertices; ++i)
      m.normals[i] = {v->normals[3 * i], v->normals[3 * i + 1], v->normals[3 * i + 2]};
  }
  if (v->uvs && v->n_uvs > 0) {
    m.uvs.resize(v->n_uvs);
    for (int i = 0; i < v->n_uvs; ++i) m.uvs[i] = {v->uvs[2 * i], v->uvs[2 * i + 1]};
  }
  if (v->face_uvs) {
    m.faceUvs.resize(v->n_faces);
    for (int f = 0; f < v->n_faces; ++f)
      m.faceUvs[f] = {v->face_uvs[3 * f], v->face_uvs[3 * f + 1], v->face_uvs[3 * f + 2]};
  }
  return m;
}

GBuffer toGBuffer(int res, const float* pos, const float* nrm, const float* tan, const float* bit,
                  const uint8_t* valid, const uint8_t* rel) {
  GBuffer g;
  if (res < 1 || !valid) return g;
  g.resolution = res;
  const size_t n = static_cast<size_t>(res) * res;
  auto fill = [&](std::vector<Eigen::Vector3f>& dst, const float* src) {
    dst.resize(n);
    if (src) std::memcpy(dst.data(), src, n * sizeof(Eigen::Vector3f));
    else std::fill(dst.begin(), dst.end(), Eigen::Vector3f::Zero());
  };
  fill(g.position, pos);
  fill(g.normal, nrm);
  fill(g.tangent, tan);
  fill(g.bitangent, bit);
  g.valid.assign(valid, valid + n);
  if (rel) g.reliable.assign(rel, rel + n);
  else g.reliable.assign(n, 0);
  return g;
}

void storeGBuffer(const GBuffer& g, float* pos, float* nrm, float* tan, float* bit,
                  uint8_t* valid, uint8_t* rel) {
  const size_t n = g.valid.size();
  if (pos) std::memcpy(pos, g.position.data(), n * 12);
  if (nrm) std::memcpy(nrm, g.normal.data(), n * 12);
  if (tan) std::memcpy(tan, g.tangent.data(), n * 12);
  if (bit) std::memcpy(bit, g.bitangent.data(), n * 12);
  if (valid) std::memcpy(valid, g.valid.data(), n);
  if (rel) std::memcpy(rel, g.reliable.data(), n);
}

double secondsSince(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Instrumented copy of the best-first loop (bvh.cpp:151-176) using only the
// public accessors (bvh.h:56-59): same result, plus pop/test counters.
SurfacePoint countedClosestWithin(const Bvh& bvh, const Eigen::Vector3d& q, double maxDist,
                                  int64_t& pops, int64_t& tris) {
  SurfacePoint best;
  best.distanceSquared = std::isinf(maxDist) ? maxDist : maxDist * maxDist;
  const auto& nodes = bvh.nodes();
  const auto& order = bvh.faceOrder();
  const auto& mesh = bvh.mesh();
  using Entry = std::pair<double, int>;
  std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
  heap.emplace(nodes[0].box.squaredDistance(q), 0);
  while (!heap.empty()) {
    auto [d, idx] = heap.top();
    heap.pop();
    if (d > best.distanceSquared) break;
    ++pops;
    const auto& node = nodes[idx];
    if (node.leaf()) {
      for (int i = 0; i < node.count; ++i) {
        const int f = order[node.first + i];
        const auto& tri = mesh.faces[f];
        Eigen::Vector3d bary;
        Eigen::Vector3d p = closestPointTriangle<double>(q, mesh.positions[tri[0]],
                                                         mesh.positions[tri[1]],
                                                         mesh.positions[tri[2]], &bary);
        const double ds = (p - q).squaredNorm();
        ++tris;
        if (ds < best.distanceSquared || (ds == best.distanceSquared && f < best.face))
          best = {f, ds, p, bary};
      }
      continue;
    }
    heap.emplace(nodes[node.left].box.squaredDistance(q), node.left);
    heap.emplace(nodes[node.right].box.squaredDistance(q), node.right);
  }
  if (!best.valid()) best.distanceSquared = std::numeric_limits<double>::infinity();
  return best;
}

thread_local TriangleMesh g_fixture;

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_hardware_threads(void) { return hardwareThreads(); }

int ref_raster_gbuffer(const mf_mesh_view* lo, int res, float* pos, float* nrm, float* tan,
                       float* bit, uint8_t* valid, uint8_t* rel) {
  return guarded([&] {
    const GBuffer g = rasterizeGBuffer(toMesh(lo), res);
    storeGBuffer(g, pos, nrm, tan, bit, valid, rel);
  });
}

int ref_transfer_normals(int res, const float* pos, const float* nrm, const float* tan,
                         const float* bit, const uint8_t* valid, const uint8_t* rel,
                         const mf_mesh_view* hi, double diag, double frac, uint8_t* rgb) {
  return guarded([&] {
    const GBuffer g = toGBuffer(res, pos, nrm, tan, bit, valid, rel);
    const ImageU8 map = transferNormals(g, toMesh(hi), diag, frac);
    std::memcpy(rgb, map.data.data(), map.data.size());
  });
}

int ref_dilate_seams(int w, int h, int c, const uint8_t* map_in, int gres, const uint8_t* valid,
                     int radius, uint8_t* out) {
  return guarded([&] {
    ImageU8 map(w, h, c);
    std::memcpy(map.data.data(), map_in, map.data.size());
    GBuffer g;
    g.resolution = gres;
    g.valid.assign(valid, valid + static_cast<size_t>(gres) * gres);
    const ImageU8 res = dilateSeams(map, g, radius);
    std::memcpy(out, res.data.data(), res.data.size());
  });
}

// Full bake as the tests compose it (test_bake.cpp:205-206), timed per stage
// with steady_clock. times[5] = {raster, bvh standalone, transfer (incl. its
// own normals + BVH), dilate, total raster+transfer+dilate}. When dbg_face /
// dbg_ts are given, the Appendix-D replica also runs (untimed) and counters[4]
// = {N_v, N_q, mean nodes popped per query, mean triangles tested per query}.
int ref_bake(const mf_mesh_view* lo, const mf_mesh_view* hi, int res, double diag, double frac,
             int radius, uint8_t* rgb_out, uint8_t* rgb_raw_out, int32_t* dbg_face,
             double* dbg_ts, double* times, double* counters, int time_bvh) {
  return guarded([&] {
    const TriangleMesh low = toMesh(lo);
    const TriangleMesh high = toMesh(hi);
    auto t0 = std::chrono::steady_clock::now();
    const GBuffer g = rasterizeGBuffer(low, res);
    const double tRaster = secondsSince(t0);
    double tBvh = 0.0;
    if (time_bvh) {
      t0 = std::chrono::steady_clock::now();
      const Bvh standalone(high);
      tBvh = secondsSince(t0);
    }
    t0 = std::chrono::steady_clock::now();
    const ImageU8 raw = transferNormals(g, high, diag, frac);
    const double tTransfer = secondsSince(t0);
    t0 = std::chrono::steady_clock::now();
    const ImageU8 out = dilateSeams(raw, g, radius);
    const double tDilate = secondsSince(t0);
    if (times) {
      times[0] = tRaster;
      times[1] = tBvh;
      times[2] = tTransfer;
      times[3] = tDilate;
      times[4] = tRaster + tTransfer + tDilate;
    }
    if (rgb_out) std::memcpy(rgb_out, out.data.data(), out.data.size());
    if (rgb_raw_out) std::memcpy(rgb_raw_out, raw.data.data(), raw.data.size());
    if (!dbg_face && !dbg_ts && !counters) return;

    // Appendix-D replica of gbuffer.cpp:218-248 around the reference's Bvh.
    std::vector<Eigen::Vector3d> hiN = high.hasNormals() ? high.normals : computeVertexNormals(high);
    for (auto& n : hiN) {
      const double len = n.norm();
      if (len > 1e-20) n /= len;
    }
    const Bvh bvh(high);
    const double maxDist = frac * diag;
    const int64_t texels = static_cast<int64_t>(res) * res;
    std::vector<int64_t> pops(texels, 0), tris(texels, 0);
    parallelFor(
        0, texels,
        [&](int64_t t) {
          int32_t face = -1;
          double ts3[3] = {0, 0, 0};
          if (g.valid[t]) {
            if (!g.reliable[t]) {
              face = -2;
            } else {
              const SurfacePoint hit =
                  countedClosestWithin(bvh, g.position[t].cast<double>(), maxDist, pops[t], tris[t]);
              if (!hit.valid()) {
                face = -3;
              } else {
                face = hit.face;
                const auto& tri = high.faces[hit.face];
                Eigen::Vector3d n = hit.barycentric.x() * hiN[tri[0]] +
                                    hit.barycentric.y() * hiN[tri[1]] +
                                    hit.barycentric.z() * hiN[tri[2]];
                Eigen::Vector3d ts(n.dot(g.tangent[t].cast<double>()),
                                   n.dot(g.bitangent[t].cast<double>()),
                                   n.dot(g.normal[t].cast<double>()));
                const double len = ts.norm();
                if (len >= 1e-12) {
                  ts /= len;
                  ts3[0] = ts[0];
                  ts3[1] = ts[1];
                  ts3[2] = ts[2];
                }
              }
            }
          }
          if (dbg_face) dbg_face[t] = face;
          if (dbg_ts)
            for (int c = 0; c < 3; ++c) dbg_ts[3 * t + c] = ts3[c];
        },
        4096);
    if (counters) {
      int64_t nv = 0, nq = 0, sp = 0, st = 0;
      for (int64_t t = 0; t < texels; ++t) {
        nv += g.valid[t];
        nq += (g.valid[t] && g.reliable[t]);
        sp += pops[t];
        st += tris[t];
      }
      counters[0] = static_cast<double>(nv);
      counters[1] = static_cast<double>(nq);
      counters[2] = nq ? static_cast<double>(sp) / nq : 0.0;
      counters[3] = nq ? static_cast<double>(st) / nq : 0.0;
    }
  });
}

// Traversal counters of the reference's best-first loop on every `stride`-th
// texel only (configs whose full bake is too slow to instrument, e.g. E):
// counters = [valid, queries (full), sampled queries, mean pops, mean tests].
int ref_sampled_counters(const mf_mesh_view* lo, const mf_mesh_view* hi, int res, double diag, double frac,
                         int stride, double* counters) {
  return guarded([&] {
    const TriangleMesh low = toMesh(lo);
    const TriangleMesh high = toMesh(hi);
    const GBuffer g = rasterizeGBuffer(low, res);
    const Bvh bvh(high);
    const double maxDist = frac * diag;
    const int64_t texels = static_cast<int64_t>(res) * res;
    std::vector<int64_t> idx;
    int64_t nv = 0, nq = 0;
    for (int64_t t = 0; t < texels; ++t) {
      nv += g.valid[t];
      if (g.valid[t] && g.reliable[t]) {
        if (nq % stride == 0) idx.push_back(t);
        ++nq;
      }
    }
    std::vector<int64_t> pops(idx.size(), 0), tris(idx.size(), 0);
    parallelFor(
        0, static_cast<int64_t>(idx.size()),
        [&](int64_t k) { countedClosestWithin(bvh, g.position[idx[k]].cast<double>(), maxDist, pops[k], tris[k]); },
        256);
    int64_t sp = 0, st = 0;
    for (size_t k = 0; k < idx.size(); ++k) {
      sp += pops[k];
      st += tris[k];
    }
    const double ns = idx.empty() ? 1.0 : static_cast<double>(idx.size());
    counters[0] = static_cast<double>(nv);
    counters[1] = static_cast<double>(nq);
    counters[2] = static_cast<double>(idx.size());
    counters[3] = sp / ns;
    counters[4] = st / ns;
  });
}

// markSurfaceBand (src/signfield/sign_grid.cpp:23-69), as the reference runs it.
int ref_surface_band(const mf_mesh_view* mesh, int res, double band_voxels, int dilate, const double* domain,
                     uint8_t* labels, float* dist, double* grid_out) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    const Bvh bvh(m);
    GridParams p;
    p.resolution = res;
    p.bandVoxels = band_voxels;
    p.dilateRadius = dilate;
    if (domain) p.domain = Aabb3d{{domain[0], domain[1], domain[2]}, {domain[3], domain[4], domain[5]}};
    const SignGrid g = markSurfaceBand(m, bvh, p);
    for (size_t i = 0; i < g.cells(); ++i) {
      labels[i] = static_cast<uint8_t>(g.labels[i]);
      dist[i] = g.distance[i];
    }
    if (grid_out) {
      for (int k = 0; k < 3; ++k) grid_out[k] = g.origin[k];
      grid_out[3] = g.voxelSize;
      grid_out[4] = g.truncation;
    }
  });
}

// fibonacciCameras (src/render/camera.cpp:38-55) -> direction, up, halfExtent.
void ref_fibonacci_cameras(int count, int res, double half_extent, double* cams7) {
  const auto cams = fibonacciCameras(count, res, half_extent);
  for (int i = 0; i < count; ++i) {
    for (int k = 0; k < 3; ++k) {
      cams7[7 * i + k] = cams[i].direction[k];
      cams7[7 * i + 3 + k] = cams[i].up[k];
    }
    cams7[7 * i + 6] = cams[i].halfExtent;
  }
}

// renderView (src/render/raster.cpp:12-102) per camera.
int ref_render_views(const mf_mesh_view* mesh, const double* cams7, int n_views, int res, const double* vn,
                     int cull, int32_t* face, float* depth, float* pos, float* nrm) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    std::vector<Eigen::Vector3d> normals(m.positions.size(), Eigen::Vector3d::Zero());
    if (vn)
      for (size_t i = 0; i < normals.size(); ++i) normals[i] = {vn[3 * i], vn[3 * i + 1], vn[3 * i + 2]};
    const size_t n = static_cast<size_t>(res) * res;
    for (int v = 0; v < n_views; ++v) {
      OrthoCamera cam;
      cam.direction = {cams7[7 * v], cams7[7 * v + 1], cams7[7 * v + 2]};
      cam.up = {cams7[7 * v + 3], cams7[7 * v + 4], cams7[7 * v + 5]};
      cam.halfExtent = cams7[7 * v + 6];
      cam.resolution = res;
      RasterOptions opt;
      opt.backfaceCull = cull != 0;
      const RenderedView r = renderView(m, normals, cam, opt);
      std::memcpy(face + v * n, r.face.data.data(), n * sizeof(int32_t));
      std::memcpy(depth + v * n, r.depth.data.data(), n * sizeof(float));
      if (pos) std::memcpy(pos + 3 * v * n, r.position.data.data(), 3 * n * sizeof(float));
      if (nrm) std::memcpy(nrm + 3 * v * n, r.normal.data.data(), 3 * n * sizeof(float));
    }
  });
}

// castVisibility (src/visibility/visibility.cpp:13-59).
int ref_cast_visibility(const mf_mesh_view* mesh, int viewpoints, int res, int64_t* hits) {
  return guarded([&] {
    const VisibilityMask mask = castVisibility(toMesh(mesh), viewpoints, res);
    std::memcpy(hits, mask.hits.data(), mask.hits.size() * sizeof(int64_t));
  });
}

int ref_bvh_build_time(const mf_mesh_view* mesh, double* seconds, int* nodes) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    auto t0 = std::chrono::steady_clock::now();
    const Bvh bvh(m);
    if (seconds) *seconds = secondsSince(t0);
    if (nodes) *nodes = static_cast<int>(bvh.nodes().size());
  });
}

int ref_closest_within(const mf_mesh_view* mesh, const double* q, int64_t n, double maxDist,
                       int brute, int32_t* face, double* distSq, double* point, double* bary) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    const Bvh bvh(m);
    parallelFor(0, n, [&](int64_t i) {
      const Eigen::Vector3d p(q[3 * i], q[3 * i + 1], q[3 * i + 2]);
      const SurfacePoint sp = brute ? closestPointBrute(m, p) : bvh.closestPointWithin(p, maxDist);
      face[i] = sp.face;
      distSq[i] = sp.distanceSquared;
      for (int c = 0; c < 3; ++c) {
        if (point) point[3 * i + c] = sp.point[c];
        if (bary) bary[3 * i + c] = sp.barycentric[c];
      }
    });
  });
}

int ref_raycast_first(const mf_mesh_view* mesh, const double* o, const double* d, int64_t n,
                      double tmin, double tmax, int brute, int32_t* face, double* t, double* u,
                      double* v) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    const Bvh bvh(m);
    parallelFor(0, n, [&](int64_t i) {
      const Eigen::Vector3d oo(o[3 * i], o[3 * i + 1], o[3 * i + 2]);
      const Eigen::Vector3d dd(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
      const RayHit h = brute ? raycastFirstBrute(m, oo, dd, tmin, tmax)
                             : bvh.raycastFirst(oo, dd, tmin, tmax);
      face[i] = h.face;
      t[i] = h.t;
      u[i] = h.u;
      v[i] = h.v;
    });
  });
}

int ref_bvh_export(const mf_mesh_view* mesh, int* n_nodes, double* boxes, int32_t* links,
                   int32_t* face_order) {
  return guarded([&] {
    const TriangleMesh m = toMesh(mesh);
    const Bvh bvh(m);
    const auto& nodes = bvh.nodes();
    if (n_nodes) *n_nodes = static_cast<int>(nodes.size());
    if (boxes)
      for (size_t i = 0; i < nodes.size(); ++i)
        for (int c = 0; c < 3; ++c) {
          boxes[6 * i + c] = nodes[i].box.min[c];
          boxes[6 * i + 3 + c] = nodes[i].box.max[c];
        }
    if (links)
      for (size_t i = 0; i < nodes.size(); ++i) {
        links[4 * i] = nodes[i].left;
        links[4 * i + 1] = nodes[i].right;
        links[4 * i + 2] = nodes[i].first;
        links[4 * i + 3] = nodes[i].count;
      }
    if (face_order)
      std::memcpy(face_order, bvh.faceOrder().data(), bvh.faceOrder().size() * 4);
  });
}

int ref_wedge_tangents(const mf_mesh_view* mesh, double* frames) {
  return guarded([&] {
    const auto fr = computeWedgeTangents(toMesh(mesh));
    for (size_t f = 0; f < fr.size(); ++f)
      for (int k = 0; k < 3; ++k) {
        double* o = frames + (f * 3 + k) * 9;
        for (int c = 0; c < 3; ++c) {
          o[c] = fr[f][k].tangent[c];
          o[3 + c] = fr[f][k].bitangent[c];
          o[6 + c] = fr[f][k].normal[c];
        }
      }
  });
}

int ref_vertex_normals(const mf_mesh_view* mesh, double* normals) {
  return guarded([&] {
    const auto n = computeVertexNormals(toMesh(mesh));
    std::memcpy(normals, n.data(), n.size() * sizeof(Eigen::Vector3d));
  });
}

int ref_baked_mean_error(const mf_mesh_view* lo, const uint8_t* rgb, int w, int h,
                         const mf_mesh_view* hi, int samples, uint64_t seed, double* meanDeg,
                         int* used, int* excluded) {
  return guarded([&] {
    ImageU8 map(w, h, 3);
    std::memcpy(map.data.data(), rgb, map.data.size());
    const BakedError e = bakedMeanErrorDeg(toMesh(lo), map, toMesh(hi), samples, seed);
    *meanDeg = e.meanDeg;
    *used = e.used;
    *excluded = e.excluded;
  });
}

// ---- fixtures (tests/support/fixtures.cpp) -----------------------------------
// kind: 0 icosphere(a), 1 uvSphere(a, b), 2 starBlob(seed=c, a, b), 3 box(n=a),
//       4 planeGrid(a, b), 5 torus(a, b). radius r where applicable.
int ref_fixture_make(int kind, int a, int b, uint64_t c, double r, int* nv, int* nf) {
  return guarded([&] {
    switch (kind) {
      case 0: g_fixture = fixtures::icosphere(a, r); break;
      case 1: g_fixture = fixtures::uvSphere(a, b, r); break;
      case 2: g_fixture = fixtures::starBlob(c, a, b, r); break;
      case 3: g_fixture = fixtures::box({r, r, r}, a); break;
      case 4: g_fixture = fixtures::planeGrid(a, b); break;
      case 5: g_fixture = fixtures::torus(a, b); break;
      default: throw Error(ErrorCode::InvalidConfig, "unknown fixture kind");
    }
    *nv = g_fixture.vertexCount();
    *nf = g_fixture.faceCount();
  });
}

void ref_fixture_get(double* positions, int32_t* faces) {
  std::memcpy(positions, g_fixture.positions.data(), g_fixture.positions.size() * 24);
  std::memcpy(faces, g_fixture.faces.data(), g_fixture.faces.size() * 12);
}

void ref_random_points(int n, const double* box6, uint64_t seed, double* out) {
  Aabb3d box;
  box.min = {box6[0], box6[1], box6[2]};
  box.max = {box6[3], box6[4], box6[5]};
  const auto p = fixtures::randomPointsInBox(n, box, seed);
  std::memcpy(out, p.data(), p.size() * 24);
}

void ref_random_units(int n, uint64_t seed, double* out) {
  const auto p = fixtures::randomUnitVectors(n, seed);
  std::memcpy(out, p.data(), p.size() * 24);
}

double ref_star_blob_radius(uint64_t seed, const double* dir, double base) {
  return fixtures::starBlobRadius(seed, Eigen::Vector3d(dir[0], dir[1], dir[2]), base);
}

}  // extern "C"

// ---------------------------------------------------------------- texfuse
// The reference declares inpaintAtlas (texfuse/fuse.h:110) and calls it from
// fuseViews (fuse.cpp:321) but never defines it; this stub
// only lets fuse.cpp link. Nothing here calls fuseViews.
namespace meshforge {
TextureAtlas inpaintAtlas(const TextureAtlas&, const GBuffer&, double, const InpaintOptions&) {
  throw Error(ErrorCode::InvalidConfig, "inpaintAtlas is not defined by the reference");
}
}  // namespace meshforge

namespace {
OrthoCamera toCamera(const double* cam7, int res) {
  OrthoCamera cam;
  cam.direction = {cam7[0], cam7[1], cam7[2]};
  cam.up = {cam7[3], cam7[4], cam7[5]};
  cam.halfExtent = cam7[6];
  cam.resolution = res;
  return cam;
}
ImageF toImage(int w, int h, int c, const float* p) {
  ImageF im(w, h, c);
  std::memcpy(im.data.data(), p, sizeof(float) * static_cast<size_t>(w) * h * c);
  return im;
}
std::vector<ImageF> toChain(int w, int h, int c, int levels, const float* p) {
  std::vector<ImageF> chain;
  for (int l = 0; l < levels; ++l) {
    chain.push_back(toImage(w, h, c, p));
    p += static_cast<size_t>(w) * h * c;
    w = std::max(1, (w + 1) / 2);
    h = std::max(1, (h + 1) / 2);
  }
  return chain;
}
}  // namespace

extern "C" {

// footprintFromJacobian (fuse.cpp:39-64): jac4 column-major; out7 = major axis
// xy, major length, minor length, mip, taps.
void ref_footprint(const double* jac4, double* out7) {
  Eigen::Matrix2d j;
  j(0, 0) = jac4[0];
  j(1, 0) = jac4[1];
  j(0, 1) = jac4[2];
  j(1, 1) = jac4[3];
  const TexelFootprint fp = footprintFromJacobian(j);
  out7[0] = fp.majorAxis.x();
  out7[1] = fp.majorAxis.y();
  out7[2] = fp.majorLength;
  out7[3] = fp.minorLength;
  out7[4] = fp.mip;
  out7[5] = fp.taps;
  out7[6] = 0.0;
}

// edgeMask (fuse.cpp:66-101) of a rendered view (position f32x3, face i32).
int ref_edge_mask(int w, int h, const float* pos, const int32_t* face, double diag, double threshold,
                  uint8_t* mask) {
  return guarded([&] {
    RenderedView v;
    v.position = toImage(w, h, 3, pos);
    v.face = Image<std::int32_t>(w, h, 1);
    std::memcpy(v.face.data.data(), face, sizeof(int32_t) * static_cast<size_t>(w) * h);
    const auto m = edgeMask(v, diag, threshold);
    std::memcpy(mask, m.data(), m.size());
  });
}

// buildMips (mips.cpp:96-112): the chain concatenated level after level into
// out; *n_levels = its length.
int ref_build_mips(int w, int h, int c, const float* base, int levels, float sharpen, float* out, int* n_levels) {
  return guarded([&] {
    const auto chain = buildMips(toImage(w, h, c, base), levels, sharpen);
    for (const ImageF& im : chain) {
      std::memcpy(out, im.data.data(), im.data.size() * sizeof(float));
      out += im.data.size();
    }
    *n_levels = static_cast<int>(chain.size());
  });
}

// backprojectView (fuse.cpp:103-186) over a G-buffer (position + valid).
int ref_backproject_view(int gres, const float* pos, const uint8_t* valid, const double* cam7, int view_res,
                         int channels, int n_mips, const float* mips, const uint8_t* mask, float* color,
                         uint8_t* sampled) {
  return guarded([&] {
    const GBuffer g = toGBuffer(gres, pos, nullptr, nullptr, nullptr, valid, nullptr);
    const auto chain = toChain(view_res, view_res, channels, n_mips, mips);
    std::vector<std::uint8_t> m(mask, mask + static_cast<size_t>(view_res) * view_res);
    const PartialAtlas pa = backprojectView(g, toCamera(cam7, view_res), chain, m);
    std::memcpy(color, pa.color.data.data(), pa.color.data.size() * sizeof(float));
    std::memcpy(sampled, pa.sampled.data(), pa.sampled.size());
  });
}

// incidenceMap (fuse.cpp:188-221).
int ref_incidence_map(int gres, const float* pos, const float* nrm, const uint8_t* valid, const double* cam7,
                      int view_res, const float* depth, double diag, double tol, float* out) {
  return guarded([&] {
    const GBuffer g = toGBuffer(gres, pos, nrm, nullptr, nullptr, valid, nullptr);
    const ImageF r = incidenceMap(g, toCamera(cam7, view_res), toImage(view_res, view_res, 1, depth), diag, tol);
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
  });
}

// blendViews (fuse.cpp:223-280): k partial atlases (w x h x c colours + sampled
// flags), k incidence maps, k priors.
int ref_blend_views(int k, int w, int h, int c, const float* colors, const uint8_t* sampled, const float* inc,
                    const double* priors, double alpha, double eps, float* out, uint8_t* filled) {
  return guarded([&] {
    const size_t n = static_cast<size_t>(w) * h;
    std::vector<PartialAtlas> parts(k);
    std::vector<ImageF> incs;
    for (int i = 0; i < k; ++i) {
      parts[i].color = toImage(w, h, c, colors + i * n * c);
      parts[i].sampled.assign(sampled + i * n, sampled + (i + 1) * n);
      incs.push_back(toImage(w, h, 1, inc + i * n));
    }
    BlendOptions opt;
    opt.alpha = alpha;
    opt.epsilon = eps;
    const TextureAtlas a = blendViews(parts, incs, std::vector<double>(priors, priors + k), opt);
    std::memcpy(out, a.color.data.data(), a.color.data.size() * sizeof(float));
    std::memcpy(filled, a.filled.data(), a.filled.size());
  });
}

// sampleSdf (src/signfield/watertight.cpp:29-38) over a WatertightResult
// holding `mesh`, the grid geometry and `field` (res^3).
int ref_sample_sdf(const mf_mesh_view* mesh, int res, const double* origin, double voxel, const float* field,
                   const double* pts, int64_t n, double* out) {
  return guarded([&] {
    WatertightResult wt;
    wt.mesh = toMesh(mesh);
    wt.grid.res = res;
    wt.grid.voxelSize = voxel;
    wt.grid.origin = {origin[0], origin[1], origin[2]};
    wt.field.assign(field, field + static_cast<size_t>(res) * res * res);
    const Bvh bvh(wt.mesh);
    std::vector<Eigen::Vector3d> p(n);
    for (int64_t i = 0; i < n; ++i) p[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    const auto v = sampleSdf(wt, bvh, p);
    std::memcpy(out, v.data(), sizeof(double) * n);
  });
}

void ref_standard_cameras(double half_extent, double* cams7) {
  const auto cams = standardCameras(64, half_extent);
  for (size_t i = 0; i < cams.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      cams7[7 * i + k] = cams[i].direction[k];
      cams7[7 * i + 3 + k] = cams[i].up[k];
    }
    cams7[7 * i + 6] = cams[i].halfExtent;
  }
}

}  // extern "C"
