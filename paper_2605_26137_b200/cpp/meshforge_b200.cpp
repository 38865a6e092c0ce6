// meshforge_b200.cpp — the reference's C++ bake/spatial API (include/meshforge)
// implemented over the C ABI of libmfbake.so (include/mfbake.h).
//
// Every compute call crosses the ABI to the B200 kernels; the few host-side
// helpers here (bounds, validateMesh, anyPerpendicular) are the reference's
// own scalar utilities, not a fallback for any device path. Errors map back
// to meshforge::Error with the reference's codes; runtime failures become
// Error(IoError, "cuda: ...").
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "meshforge/bake/gbuffer.h"
#include "meshforge/bake/tangent.h"
#include "meshforge/core/error.h"
#include "meshforge/core/mesh.h"
#include "meshforge/render/camera.h"
#include "meshforge/render/raster.h"
#include "meshforge/signfield/sign_grid.h"
#include "meshforge/visibility/visibility.h"
#include "meshforge/spatial/bvh.h"
#include "mfbake.h"

namespace meshforge {
namespace {

[[noreturn]] void throwStatus(int rc) {
  std::string msg = mf_last_error();
  if (rc > 0 && rc <= 13) {
    const ErrorCode code = static_cast<ErrorCode>(rc - 1);
    const std::string prefix = std::string(errorCodeName(code)) + ": ";
    if (msg.compare(0, prefix.size(), prefix) == 0) msg = msg.substr(prefix.size());
    throw Error(code, msg);
  }
  throw Error(ErrorCode::IoError, "cuda: " + msg);
}
void check(int rc) {
  if (rc != MF_OK) throwStatus(rc);
}

// One context per host thread (a context is single-threaded), on the device
// named by MFB_DEVICE (default 0).
mf_ctx* context() {
  struct Holder {
    mf_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) mf_ctx_destroy(ctx);
    }
  };
  thread_local Holder h;
  if (!h.ctx) {
    const char* dev = std::getenv("MFB_DEVICE");
    check(mf_ctx_create(dev ? std::atoi(dev) : 0, nullptr, &h.ctx));
  }
  return h.ctx;
}

mf_mesh_view viewOf(const TriangleMesh& m) {
  mf_mesh_view v{};
  v.positions = m.positions.empty() ? nullptr : m.positions.data()->data();
  v.n_vertices = m.vertexCount();
  v.faces = m.faces.empty() ? nullptr : m.faces.data()->data();
  v.n_faces = m.faceCount();
  v.normals = m.hasNormals() ? m.normals.data()->data() : nullptr;
  if (m.hasUvs()) {
    v.uvs = m.uvs.data()->data();
    v.n_uvs = static_cast<int32_t>(m.uvs.size());
    v.face_uvs = m.faceUvs.data()->data();
  }
  return v;
}

float* f3(std::vector<Eigen::Vector3f>& v) { return v.empty() ? nullptr : v.data()->data(); }
const float* f3(const std::vector<Eigen::Vector3f>& v) { return v.empty() ? nullptr : v.data()->data(); }

}  // namespace

// ------------------------------------------------------------------ core
Aabb3d bounds(const TriangleMesh& m) {
  Aabb3d box;
  for (const auto& p : m.positions) box.extend(p);
  return box;
}

void validateMesh(const TriangleMesh& m) {
  if (m.faces.empty()) throw Error(ErrorCode::EmptyMesh, "mesh has no faces");
  for (const auto& p : m.positions)
    if (!p.allFinite()) throw Error(ErrorCode::InvalidGeometry, "non-finite vertex coordinate");
  const int nv = m.vertexCount();
  for (const auto& f : m.faces)
    for (int k = 0; k < 3; ++k)
      if (f[k] < 0 || f[k] >= nv) throw Error(ErrorCode::InvalidGeometry, "face index out of range");
}

std::vector<Eigen::Vector3d> computeVertexNormals(const TriangleMesh& m) {
  std::vector<Eigen::Vector3d> out(m.positions.size(), Eigen::Vector3d::Zero());
  if (m.positions.empty()) return out;
  const mf_mesh_view v = viewOf(m);
  check(mf_vertex_normals(context(), &v, out.data()->data()));
  return out;
}

// ------------------------------------------------------------------ tangents
Eigen::Vector3d anyPerpendicular(const Eigen::Vector3d& n) {
  int smallest = 0;
  for (int k = 1; k < 3; ++k)
    if (std::abs(n[k]) < std::abs(n[smallest])) smallest = k;
  const Eigen::Vector3d p = Eigen::Vector3d::Unit(smallest).cross(n);
  const double len = p.norm();
  return len > 1e-20 ? Eigen::Vector3d(p / len) : Eigen::Vector3d::UnitX();
}

std::vector<std::array<TangentFrame, 3>> computeWedgeTangents(const TriangleMesh& mesh) {
  if (!mesh.hasUvs()) throw Error(ErrorCode::InvalidGeometry, "tangent frames require a UV-mapped mesh");
  std::vector<double> raw(static_cast<size_t>(mesh.faceCount()) * 27);
  const mf_mesh_view v = viewOf(mesh);
  check(mf_wedge_tangents(context(), &v, raw.data()));
  std::vector<std::array<TangentFrame, 3>> frames(mesh.faceCount());
  for (size_t f = 0; f < frames.size(); ++f)
    for (int k = 0; k < 3; ++k) {
      const double* o = raw.data() + (f * 3 + k) * 9;
      frames[f][k].tangent = Eigen::Vector3d(o[0], o[1], o[2]);
      frames[f][k].bitangent = Eigen::Vector3d(o[3], o[4], o[5]);
      frames[f][k].normal = Eigen::Vector3d(o[6], o[7], o[8]);
    }
  return frames;
}

// ------------------------------------------------------------------ bake
GBuffer rasterizeGBuffer(const TriangleMesh& lowpoly, int resolution) {
  const mf_mesh_view v = viewOf(lowpoly);
  GBuffer g;
  const size_t n = resolution > 0 ? static_cast<size_t>(resolution) * resolution : 0;
  g.position.assign(n, Eigen::Vector3f::Zero());
  g.normal.assign(n, Eigen::Vector3f::Zero());
  g.tangent.assign(n, Eigen::Vector3f::Zero());
  g.bitangent.assign(n, Eigen::Vector3f::Zero());
  g.valid.assign(n, 0);
  g.reliable.assign(n, 0);
  check(mf_raster_gbuffer(context(), &v, resolution, f3(g.position), f3(g.normal), f3(g.tangent),
                          f3(g.bitangent), g.valid.data(), g.reliable.data()));
  g.resolution = resolution;
  return g;
}

ImageU8 transferNormals(const GBuffer& gbuffer, const TriangleMesh& highpoly, double bboxDiagonal,
                        double maxDistanceFraction) {
  const int res = gbuffer.empty() ? 0 : gbuffer.resolution;
  ImageU8 map(res, res, 3, 128);
  const mf_mesh_view v = viewOf(highpoly);
  check(mf_transfer_normals(context(), res, f3(gbuffer.position), f3(gbuffer.normal), f3(gbuffer.tangent),
                            f3(gbuffer.bitangent), gbuffer.empty() ? nullptr : gbuffer.valid.data(),
                            gbuffer.reliable.empty() ? nullptr : gbuffer.reliable.data(), &v, bboxDiagonal,
                            maxDistanceFraction, map.data.empty() ? nullptr : map.data.data()));
  return map;
}

ImageU8 dilateSeams(const ImageU8& map, const GBuffer& gbuffer, int radius) {
  ImageU8 out = map;
  check(mf_dilate_seams(context(), map.width, map.height, map.channels, map.data.empty() ? nullptr : map.data.data(),
                        gbuffer.resolution, gbuffer.valid.empty() ? nullptr : gbuffer.valid.data(), radius,
                        out.data.empty() ? nullptr : out.data.data()));
  return out;
}

ImageU8 bakeNormalMap(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                      double bboxDiagonal, double maxDistanceFraction, int radius) {
  ImageU8 map(resolution > 0 ? resolution : 0, resolution > 0 ? resolution : 0, 3);
  const mf_mesh_view lv = viewOf(lowpoly), hv = viewOf(highpoly);
  check(mf_bake_normal_map(context(), &lv, &hv, resolution, bboxDiagonal, maxDistanceFraction, radius,
                           map.data.empty() ? nullptr : map.data.data(), nullptr, nullptr, nullptr));
  return map;
}

ImageU8 bakeNormalMapRGBA8(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                           double bboxDiagonal, double maxDistanceFraction, int radius) {
  ImageU8 map(resolution > 0 ? resolution : 0, resolution > 0 ? resolution : 0, 4);
  const mf_mesh_view lv = viewOf(lowpoly), hv = viewOf(highpoly);
  check(mf_bake_normal_map_ex(context(), &lv, &hv, resolution, bboxDiagonal, maxDistanceFraction, radius,
                              MF_ATLAS_RGBA8, map.data.empty() ? nullptr : map.data.data(), nullptr));
  return map;
}

Image<std::uint16_t> bakeNormalMapRG16(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                                       double bboxDiagonal, double maxDistanceFraction, int radius) {
  Image<std::uint16_t> map(resolution > 0 ? resolution : 0, resolution > 0 ? resolution : 0, 2);
  const mf_mesh_view lv = viewOf(lowpoly), hv = viewOf(highpoly);
  check(mf_bake_normal_map_ex(context(), &lv, &hv, resolution, bboxDiagonal, maxDistanceFraction, radius,
                              MF_ATLAS_RG16, map.data.empty() ? nullptr : map.data.data(), nullptr));
  return map;
}

// ------------------------------------------------------------------ Bvh
struct Bvh::Handle {
  mf_mesh* mesh = nullptr;
  mf_bvh* bvh = nullptr;
  Aabb3d box;
  bool exported = false;
  std::mutex mu;
  ~Handle() {
    if (bvh) mf_bvh_destroy(bvh);
    if (mesh) mf_mesh_destroy(mesh);
  }
};

Bvh::Bvh(const TriangleMesh& mesh) : mesh_(&mesh), h_(std::make_shared<Handle>()) {
  validateMesh(mesh);  // Bvh::Bvh validates first (bvh.cpp:49)
  const mf_mesh_view v = viewOf(mesh);
  check(mf_mesh_upload(context(), &v, &h_->mesh));
  check(mf_bvh_build(context(), h_->mesh, &h_->bvh));
}

SurfacePoint Bvh::closestPointWithin(const Eigen::Vector3d& query, double maxDistance) const {
  return closestPointsWithin({query}, maxDistance)[0];
}

SurfacePoint Bvh::closestPoint(const Eigen::Vector3d& query) const {
  return closestPointWithin(query, std::numeric_limits<double>::infinity());
}

std::vector<SurfacePoint> Bvh::closestPointsWithin(const std::vector<Eigen::Vector3d>& q,
                                                   double maxDistance) const {
  const int64_t n = static_cast<int64_t>(q.size());
  std::vector<int32_t> face(n);
  std::vector<double> ds(n);
  std::vector<Eigen::Vector3d> pt(n), bary(n);
  if (n)
    check(mf_bvh_closest_within(h_->bvh, q.data()->data(), n, maxDistance, face.data(), ds.data(),
                                pt.data()->data(), bary.data()->data()));
  std::vector<SurfacePoint> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = SurfacePoint{face[i], ds[i], pt[i], bary[i]};
  return out;
}

RayHit Bvh::raycastFirst(const Eigen::Vector3d& origin, const Eigen::Vector3d& dir, double tMin,
                         double tMax) const {
  return raycastFirstBatch(std::vector<Eigen::Vector3d>{origin}, std::vector<Eigen::Vector3d>{dir}, tMin, tMax)[0];
}

std::vector<RayHit> Bvh::raycastFirstBatch(const std::vector<Eigen::Vector3d>& o,
                                           const std::vector<Eigen::Vector3d>& d, double tMin, double tMax) const {
  const int64_t n = static_cast<int64_t>(std::min(o.size(), d.size()));
  std::vector<int32_t> face(n);
  std::vector<double> t(n), u(n), v(n);
  if (n)
    check(mf_bvh_raycast_first(h_->bvh, o.data()->data(), d.data()->data(), n, tMin, tMax, face.data(), t.data(),
                               u.data(), v.data()));
  std::vector<RayHit> out(n);
  for (int64_t i = 0; i < n; ++i) out[i] = RayHit{face[i], t[i], u[i], v[i]};
  return out;
}

void Bvh::exportTree() const {
  std::lock_guard<std::mutex> lock(h_->mu);
  if (h_->exported) return;
  int32_t nn = 0, leaves = 0, depth = 0;
  check(mf_bvh_info(h_->bvh, &nn, &leaves, &depth));
  std::vector<double> boxes(static_cast<size_t>(nn) * 6);
  std::vector<int32_t> links(static_cast<size_t>(nn) * 4);
  faceOrder_.resize(mesh_->faceCount());
  check(mf_bvh_export(h_->bvh, boxes.data(), links.data(), faceOrder_.data()));
  nodes_.resize(nn);
  for (int32_t i = 0; i < nn; ++i) {
    Node& nd = nodes_[i];
    nd.box.min = Eigen::Vector3d(boxes[6 * i], boxes[6 * i + 1], boxes[6 * i + 2]);
    nd.box.max = Eigen::Vector3d(boxes[6 * i + 3], boxes[6 * i + 4], boxes[6 * i + 5]);
    nd.left = links[4 * i];
    nd.right = links[4 * i + 1];
    nd.first = links[4 * i + 2];
    nd.count = links[4 * i + 3];
  }
  h_->box = nn ? nodes_[0].box : Aabb3d{};
  h_->exported = true;
}

const Aabb3d& Bvh::bounds() const {
  exportTree();
  return h_->box;
}
const std::vector<Bvh::Node>& Bvh::nodes() const {
  exportTree();
  return nodes_;
}
const std::vector<std::int32_t>& Bvh::faceOrder() const {
  exportTree();
  return faceOrder_;
}

RayHit raycastFirstBrute(const TriangleMesh& mesh, const Eigen::Vector3d& origin, const Eigen::Vector3d& dir,
                         double tMin, double tMax) {
  const mf_mesh_view v = viewOf(mesh);
  RayHit h;
  check(mf_raycast_first_brute(context(), &v, origin.data(), dir.data(), 1, tMin, tMax, &h.face, &h.t, &h.u, &h.v));
  return h;
}

SurfacePoint closestPointBrute(const TriangleMesh& mesh, const Eigen::Vector3d& query) {
  const mf_mesh_view v = viewOf(mesh);
  SurfacePoint sp;
  check(mf_closest_point_brute(context(), &v, query.data(), 1, &sp.face, &sp.distanceSquared, sp.point.data(),
                               sp.barycentric.data()));
  return sp;
}

// ------------------------------------------------------------------ sign grid
SignGrid markSurfaceBand(const TriangleMesh& mesh, const Bvh& bvh, const GridParams& params) {
  (void)mesh;  // the device derives bounds(mesh) from the tree's own copy of it
  SignGrid g;
  const int res = params.resolution;
  double dom[6];
  if (params.domain) {
    for (int k = 0; k < 3; ++k) {
      dom[k] = params.domain->min[k];
      dom[3 + k] = params.domain->max[k];
    }
  }
  std::vector<std::uint8_t> labels;
  double grid[5];
  // (invalid resolutions get 1-element buffers so the ABI reports the
  // reference's InvalidConfig rather than a null-argument error)
  const std::size_t cells = res >= 8 ? static_cast<std::size_t>(res) * res * res : 1;
  labels.resize(cells);
  g.distance.resize(cells);
  check(mf_surface_band(bvh.handle()->bvh, res, params.bandVoxels, params.dilateRadius,
                        params.domain ? dom : nullptr, labels.data(), g.distance.data(), grid));
  g.res = res;
  g.origin = Eigen::Vector3d(grid[0], grid[1], grid[2]);
  g.voxelSize = grid[3];
  g.truncation = grid[4];
  g.labels.resize(labels.size());
  for (std::size_t i = 0; i < labels.size(); ++i) g.labels[i] = static_cast<VoxelLabel>(labels[i]);
  return g;
}

// ------------------------------------------------------------------ cameras, views, visibility
std::vector<OrthoCamera> standardCameras(int resolution, double halfExtent) {  // render/camera.cpp:7-31
  const double s2 = std::sqrt(0.5);
  const double cosA[8] = {1, s2, 0, -s2, -1, -s2, 0, s2};
  const double sinA[8] = {0, s2, 1, s2, 0, -s2, -1, -s2};
  std::vector<OrthoCamera> cams(10);
  for (int k = 0; k < 8; ++k) {
    cams[k].direction = Eigen::Vector3d(-cosA[k], -sinA[k], 0.0);
    cams[k].up = Eigen::Vector3d(0, 0, 1);
  }
  cams[8].direction = Eigen::Vector3d(0, 0, -1);
  cams[8].up = Eigen::Vector3d(0, 1, 0);
  cams[9].direction = Eigen::Vector3d(0, 0, 1);
  cams[9].up = Eigen::Vector3d(0, 1, 0);
  for (auto& cam : cams) {
    cam.halfExtent = halfExtent;
    cam.resolution = resolution;
  }
  return cams;
}

std::vector<OrthoCamera> fibonacciCameras(int count, int resolution, double halfExtent) {
  std::vector<double> raw(7 * static_cast<size_t>(std::max(count, 0)));
  check(mf_fibonacci_cameras(count, halfExtent, raw.data()));
  std::vector<OrthoCamera> cams(std::max(count, 0));
  for (int i = 0; i < count; ++i) {
    const double* c = raw.data() + 7 * i;
    cams[i].direction = Eigen::Vector3d(c[0], c[1], c[2]);
    cams[i].up = Eigen::Vector3d(c[3], c[4], c[5]);
    cams[i].halfExtent = c[6];
    cams[i].resolution = resolution;
  }
  return cams;
}

namespace {
// One mf_render_views call for cameras sharing a resolution.
std::vector<RenderedView> renderSameRes(const TriangleMesh& mesh, const std::vector<Eigen::Vector3d>& vn,
                                        const std::vector<OrthoCamera>& cams, const RasterOptions& options) {
  std::vector<RenderedView> out;
  if (cams.empty()) return out;
  const int res = cams[0].resolution;
  const size_t px = static_cast<size_t>(res) * res;
  std::vector<double> raw(7 * cams.size());
  for (size_t i = 0; i < cams.size(); ++i) {
    for (int k = 0; k < 3; ++k) {
      raw[7 * i + k] = cams[i].direction[k];
      raw[7 * i + 3 + k] = cams[i].up[k];
    }
    raw[7 * i + 6] = cams[i].halfExtent;
  }
  std::vector<std::int32_t> face(px * cams.size());
  std::vector<float> depth(px * cams.size()), pos(3 * px * cams.size()), nrm(3 * px * cams.size());
  const mf_mesh_view v = viewOf(mesh);
  check(mf_render_views(context(), &v, raw.data(), static_cast<int>(cams.size()), res,
                        vn.empty() ? nullptr : vn.data()->data(), options.backfaceCull ? 1 : 0, face.data(),
                        depth.data(), pos.data(), nrm.data()));
  out.resize(cams.size());
  for (size_t i = 0; i < cams.size(); ++i) {
    RenderedView& r = out[i];
    r.face = Image<std::int32_t>(res, res, 1);
    r.depth = ImageF(res, res, 1);
    r.position = ImageF(res, res, 3);
    r.normal = ImageF(res, res, 3);
    std::memcpy(r.face.data.data(), face.data() + i * px, px * sizeof(std::int32_t));
    std::memcpy(r.depth.data.data(), depth.data() + i * px, px * sizeof(float));
    std::memcpy(r.position.data.data(), pos.data() + 3 * i * px, 3 * px * sizeof(float));
    std::memcpy(r.normal.data.data(), nrm.data() + 3 * i * px, 3 * px * sizeof(float));
  }
  return out;
}
}  // namespace

RenderedView renderView(const TriangleMesh& mesh, const std::vector<Eigen::Vector3d>& vertexNormals,
                        const OrthoCamera& camera, const RasterOptions& options) {
  return renderSameRes(mesh, vertexNormals, {camera}, options)[0];
}

ViewSet renderGeometry(const TriangleMesh& mesh, const std::vector<OrthoCamera>& cameras,
                       const RasterOptions& options) {  // render/raster.cpp:104-115
  ViewSet set;
  set.cameras = cameras;
  set.views.resize(cameras.size());
  const std::vector<Eigen::Vector3d> normals = mesh.hasNormals() ? mesh.normals : computeVertexNormals(mesh);
  for (size_t i = 0; i < cameras.size();) {  // batch consecutive cameras of one resolution
    size_t j = i + 1;
    while (j < cameras.size() && cameras[j].resolution == cameras[i].resolution) ++j;
    std::vector<OrthoCamera> batch(cameras.begin() + i, cameras.begin() + j);
    std::vector<RenderedView> views = renderSameRes(mesh, normals, batch, options);
    for (size_t k = i; k < j; ++k) set.views[k] = std::move(views[k - i]);
    i = j;
  }
  return set;
}

VisibilityMask castVisibility(const TriangleMesh& mesh, int viewpoints, int resolution) {
  VisibilityMask mask;
  mask.hits.assign(mesh.faceCount(), 0);
  std::vector<std::uint8_t> state(mesh.faceCount() > 0 ? mesh.faceCount() : 1);
  const mf_mesh_view v = viewOf(mesh);
  std::int64_t dummy = 0;
  check(mf_cast_visibility(context(), &v, viewpoints, resolution, mesh.faceCount() > 0 ? mask.hits.data() : &dummy,
                           state.data()));
  mask.state.resize(mesh.faceCount());
  for (int f = 0; f < mesh.faceCount(); ++f) mask.state[f] = static_cast<FaceVisibility>(state[f]);
  return mask;
}

// ------------------------------------------------------------------ mesh topology + cull stage (host)
std::vector<std::array<int, 3>> faceAdjacency(const TriangleMesh& m) {
  // every (edge, face, corner) incidence, ordered by edge then face then
  // corner; consecutive incidences of an edge pair up two by two
  struct Inc {
    std::uint64_t key;
    int face, corner;
  };
  std::vector<Inc> inc;
  inc.reserve(3 * m.faces.size());
  for (int f = 0; f < m.faceCount(); ++f)
    for (int k = 0; k < 3; ++k) inc.push_back({edgeKey(m.faces[f][k], m.faces[f][(k + 1) % 3]), f, k});
  std::stable_sort(inc.begin(), inc.end(), [](const Inc& a, const Inc& b) { return a.key < b.key; });
  std::vector<std::array<int, 3>> adj(m.faces.size(), {-1, -1, -1});
  for (size_t i = 0; i + 1 < inc.size();) {
    if (inc[i].key == inc[i + 1].key) {
      adj[inc[i].face][inc[i].corner] = inc[i + 1].face;
      adj[inc[i + 1].face][inc[i + 1].corner] = inc[i].face;
      i += 2;
    } else {
      ++i;
    }
  }
  return adj;
}

TriangleMesh extractFaces(const TriangleMesh& m, const std::vector<std::uint8_t>& keep) {
  TriangleMesh out;
  std::vector<int> vmap(m.positions.size(), -1);
  const bool uv = m.hasUvs();
  std::vector<int> tmap(uv ? m.uvs.size() : 0, -1);
  for (int f = 0; f < m.faceCount(); ++f) {
    if (!keep[f]) continue;
    Eigen::Vector3i tri, tuv;
    for (int k = 0; k < 3; ++k) {
      int& slot = vmap[m.faces[f][k]];
      if (slot < 0) {
        slot = static_cast<int>(out.positions.size());
        out.positions.push_back(m.positions[m.faces[f][k]]);
        if (m.hasNormals()) out.normals.push_back(m.normals[m.faces[f][k]]);
      }
      tri[k] = slot;
      if (uv) {
        int& ts = tmap[m.faceUvs[f][k]];
        if (ts < 0) {
          ts = static_cast<int>(out.uvs.size());
          out.uvs.push_back(m.uvs[m.faceUvs[f][k]]);
        }
        tuv[k] = ts;
      }
    }
    out.faces.push_back(tri);
    if (uv) out.faceUvs.push_back(tuv);
  }
  return out;
}

VisibilityMask promoteExterior(const TriangleMesh& mesh, const VisibilityMask& mask, double cosThreshold) {
  if (static_cast<int>(mask.state.size()) != mesh.faceCount() || mask.hits.size() != mask.state.size())
    throw Error(ErrorCode::ShapeMismatch, "visibility mask does not match the mesh");
  const int nf = mesh.faceCount();
  std::vector<Eigen::Vector3d> n(nf);
  for (int f = 0; f < nf; ++f) n[f] = faceNormal(mesh, f);
  const auto adj = faceAdjacency(mesh);
  VisibilityMask out = mask;
  // the result is the closure under accepting edges, so any visiting order
  // gives it; a work stack of reached faces
  std::vector<int> work;
  for (int f = 0; f < nf; ++f)
    if (out.state[f] == FaceVisibility::Visible) work.push_back(f);
  while (!work.empty()) {
    const int f = work.back();
    work.pop_back();
    for (int g : adj[f]) {
      if (g < 0 || out.state[g] != FaceVisibility::Hidden) continue;
      if (n[g].dot(n[f]) >= cosThreshold) {
        out.state[g] = FaceVisibility::PromotedExterior;
        work.push_back(g);
      }
    }
  }
  return out;
}

TriangleMesh removeHidden(const TriangleMesh& mesh, const VisibilityMask& mask) {
  if (static_cast<int>(mask.state.size()) != mesh.faceCount())
    throw Error(ErrorCode::ShapeMismatch, "visibility mask does not match the mesh");
  std::vector<std::uint8_t> keep(mesh.faceCount());
  int kept = 0;
  for (int f = 0; f < mesh.faceCount(); ++f) kept += (keep[f] = mask.keep(f) ? 1 : 0);
  if (kept == 0) throw Error(ErrorCode::AllHidden, "every face is occluded from all viewpoints");
  if (kept == mesh.faceCount()) return mesh;
  return extractFaces(mesh, keep);
}

TriangleMesh cullHiddenFaces(const TriangleMesh& mesh, int viewpoints, int resolution, double cosThreshold) {
  return removeHidden(mesh, promoteExterior(mesh, castVisibility(mesh, viewpoints, resolution), cosThreshold));
}

}  // namespace meshforge
