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
#include "meshforge/signfield/watertight.h"
#include "meshforge/visibility/visibility.h"
#include "meshforge/spatial/bvh.h"
#include "meshforge/texfuse/fuse.h"
#include "meshforge/texfuse/mips.h"
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
// A tree owns its context (stream + query scratch) instead of borrowing the
// building thread's: the reference queries one const Bvh from many threads
// (metrics.cpp: toBvh.closestPoint inside parallelChunks) and a Bvh may outlive
// the thread that built it. `mu` serialises every query on the shared scratch.
struct Bvh::Handle {
  mf_ctx* ctx = nullptr;
  mf_mesh* mesh = nullptr;
  mf_bvh* bvh = nullptr;
  Aabb3d box;
  bool exported = false;
  mutable std::mutex mu;
  ~Handle() {
    if (bvh) mf_bvh_destroy(bvh);
    if (mesh) mf_mesh_destroy(mesh);
    if (ctx) mf_ctx_destroy(ctx);
  }
};

static std::unique_lock<std::mutex> lockTree(const Bvh& bvh) { return std::unique_lock<std::mutex>(bvh.handle()->mu); }

Bvh::Bvh(const TriangleMesh& mesh) : mesh_(&mesh), h_(std::make_shared<Handle>()) {
  validateMesh(mesh);  // Bvh::Bvh validates first (bvh.cpp:49)
  const mf_mesh_view v = viewOf(mesh);
  const char* dev = std::getenv("MFB_DEVICE");
  check(mf_ctx_create(dev ? std::atoi(dev) : 0, nullptr, &h_->ctx));
  check(mf_mesh_upload(h_->ctx, &v, &h_->mesh));
  check(mf_bvh_build(h_->ctx, h_->mesh, &h_->bvh));
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
  if (n) {
    const auto lock = lockTree(*this);
    check(mf_bvh_closest_within(h_->bvh, q.data()->data(), n, maxDistance, face.data(), ds.data(),
                                pt.data()->data(), bary.data()->data()));
  }
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
  if (n) {
    const auto lock = lockTree(*this);
    check(mf_bvh_raycast_first(h_->bvh, o.data()->data(), d.data()->data(), n, tMin, tMax, face.data(), t.data(),
                               u.data(), v.data()));
  }
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
  const auto lock = lockTree(bvh);
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

double sampleSignedField(const SignGrid& grid, const std::vector<float>& field, const Eigen::Vector3d& p) {
  const Eigen::Vector3d q = (p - grid.origin) / grid.voxelSize - Eigen::Vector3d::Constant(0.5);
  double result = 0;
  int i0[3];
  double f[3];
  for (int k = 0; k < 3; ++k) {
    const double c = std::clamp(q[k], 0.0, static_cast<double>(grid.res - 1));
    i0[k] = std::max(std::min(static_cast<int>(std::floor(c)), grid.res - 2), 0);
    f[k] = std::clamp(c - i0[k], 0.0, 1.0);
  }
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double w = (dx ? f[0] : 1 - f[0]) * (dy ? f[1] : 1 - f[1]) * (dz ? f[2] : 1 - f[2]);
        result += w * field[grid.index(i0[0] + dx, i0[1] + dy, i0[2] + dz)];
      }
  return result;
}

std::vector<double> sampleSdf(const WatertightResult& wt, const Bvh& watertightBvh,
                              const std::vector<Eigen::Vector3d>& points) {
  std::vector<double> values(points.size());
  if (points.empty()) return values;
  if (wt.field.size() != wt.grid.cells())
    throw Error(ErrorCode::ShapeMismatch, "signed field does not match the grid");
  const double origin[3] = {wt.grid.origin.x(), wt.grid.origin.y(), wt.grid.origin.z()};
  const auto lock = lockTree(watertightBvh);
  check(mf_sample_sdf(watertightBvh.handle()->bvh, wt.grid.res, origin, wt.grid.voxelSize, wt.field.data(),
                      points.data()->data(), static_cast<int64_t>(points.size()), values.data()));
  return values;
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

// ------------------------------------------------------------------ texfuse
// fuse.h / mips.h over the texfuse entry points of include/mfbake.h. Argument
// checks are the reference's, in its order (fuse.cpp:66-326, mips.cpp:96-102);
// the images go to the device in one call each.
namespace meshforge {
namespace {

void camera7(const OrthoCamera& c, double* out) {
  for (int k = 0; k < 3; ++k) {
    out[k] = c.direction[k];
    out[3 + k] = c.up[k];
  }
  out[6] = c.halfExtent;
}

void checkEdgeMask(const RenderedView& view, double bboxDiagonal, double threshold) {
  const int w = view.position.width, h = view.position.height;
  if (w < 1 || h < 1 || view.face.width != w || view.face.height != h)
    throw Error(ErrorCode::InvalidConfig, "edge mask needs a rendered view");
  if (!(bboxDiagonal > 0.0) || !(threshold > 0.0))
    throw Error(ErrorCode::InvalidConfig, "edge mask scale must be positive");
}
void checkMips(const ImageF& base, int levels, float sharpen) {
  if (base.width < 1 || base.height < 1 || base.channels < 1)
    throw Error(ErrorCode::InvalidConfig, "mip base image is empty");
  if (levels < 1) throw Error(ErrorCode::InvalidConfig, "mip chain needs >= 1 level");
  if (!(sharpen >= 0.0f)) throw Error(ErrorCode::InvalidConfig, "sharpen strength must be >= 0");
}
void checkBackproject(const GBuffer& geom, int res, int w0, int h0, std::size_t maskSize) {
  if (geom.empty()) throw Error(ErrorCode::InvalidConfig, "geometry image is empty");
  if (w0 < 1) throw Error(ErrorCode::InvalidConfig, "view mip chain is empty");
  if (w0 != res || h0 != res) throw Error(ErrorCode::ShapeMismatch, "view image does not match the camera");
  if (maskSize != static_cast<std::size_t>(res) * res)
    throw Error(ErrorCode::ShapeMismatch, "edge mask does not match the view");
}
void checkIncidence(const GBuffer& geom, const OrthoCamera& camera, const ImageF& depth, double diag, double tol) {
  if (geom.empty()) throw Error(ErrorCode::InvalidConfig, "geometry image is empty");
  if (!(diag > 0.0) || !(tol > 0.0)) throw Error(ErrorCode::InvalidConfig, "incidence scale must be positive");
  const int res = camera.resolution;
  if (depth.width != res || depth.height != res || depth.channels != 1)
    throw Error(ErrorCode::ShapeMismatch, "depth buffer does not match the camera");
}
// buildMips' halving layout (the device chain format)
bool standardChain(const std::vector<ImageF>& mips) {
  for (std::size_t l = 1; l < mips.size(); ++l)
    if (mips[l].width != std::max(1, (mips[l - 1].width + 1) / 2) ||
        mips[l].height != std::max(1, (mips[l - 1].height + 1) / 2) || mips[l].channels != mips[0].channels ||
        (mips[l - 1].width == 1 && mips[l - 1].height == 1))
      return false;
  return true;
}

}  // namespace

TexelFootprint footprintFromJacobian(const Eigen::Matrix2d& jacobian) {
  TexelFootprint fp;
  fp.jacobian = jacobian;
  const Eigen::Matrix2d m = jacobian * jacobian.transpose();
  const double mean = 0.5 * (m(0, 0) + m(1, 1));
  const double disc = std::hypot(0.5 * (m(0, 0) - m(1, 1)), m(0, 1));
  const double s1 = std::sqrt(std::max(0.0, mean + disc));
  const double s2 = std::sqrt(std::max(0.0, mean - disc));
  constexpr double kTiny = 1e-12;
  if (!(s1 > kTiny)) return fp;
  Eigen::Vector2d axis(m(0, 1), mean + disc - m(0, 0));
  const Eigen::Vector2d alt(mean + disc - m(1, 1), m(0, 1));
  if (alt.squaredNorm() > axis.squaredNorm()) axis = alt;
  fp.majorAxis = axis.squaredNorm() > 0.0 ? axis.normalized() : Eigen::Vector2d::UnitX();
  fp.majorLength = s1;
  fp.minorLength = s2;
  const double ratio = s1 / std::max(s2, kTiny);
  fp.taps = static_cast<int>(std::clamp(std::ceil(ratio), 1.0, 8.0));
  fp.mip = std::max(0.0, std::log2(std::max(s2, kTiny)) - 0.5 + 0.5 * std::log2(std::min(ratio, 8.0)));
  return fp;
}

std::vector<std::uint8_t> edgeMask(const RenderedView& view, double bboxDiagonal, double threshold) {
  checkEdgeMask(view, bboxDiagonal, threshold);
  const int w = view.position.width, h = view.position.height;
  std::vector<std::uint8_t> mask(static_cast<std::size_t>(w) * h, 0);
  check(mf_edge_mask(context(), w, h, view.position.data.data(), view.face.data.data(), bboxDiagonal, threshold,
                     mask.data()));
  return mask;
}

std::vector<ImageF> buildMips(const ImageF& base, int levels, float sharpenStrength) {
  checkMips(base, levels, sharpenStrength);
  int n = 0;
  const int64_t total = mf_mip_chain_floats(base.width, base.height, base.channels, levels, &n);
  std::vector<float> flat(static_cast<std::size_t>(total));
  check(mf_build_mips(context(), base.width, base.height, base.channels, base.data.data(), levels, sharpenStrength,
                      flat.data(), &n));
  std::vector<ImageF> chain;
  int w = base.width, h = base.height;
  std::size_t o = 0;
  for (int l = 0; l < n; ++l) {
    ImageF im(w, h, base.channels);
    std::copy(flat.begin() + o, flat.begin() + o + im.data.size(), im.data.begin());
    o += im.data.size();
    chain.push_back(std::move(im));
    w = std::max(1, (w + 1) / 2);
    h = std::max(1, (h + 1) / 2);
  }
  return chain;
}

PartialAtlas backprojectView(const GBuffer& geom, const OrthoCamera& camera, const std::vector<ImageF>& viewMips,
                             const std::vector<std::uint8_t>& mask) {
  if (geom.empty()) throw Error(ErrorCode::InvalidConfig, "geometry image is empty");
  if (viewMips.empty() || viewMips[0].width < 1) throw Error(ErrorCode::InvalidConfig, "view mip chain is empty");
  checkBackproject(geom, camera.resolution, viewMips[0].width, viewMips[0].height, mask.size());
  if (!standardChain(viewMips))
    throw Error(ErrorCode::InvalidConfig, "mip chain levels must follow buildMips' halving");
  std::vector<float> flat;
  for (const ImageF& im : viewMips) flat.insert(flat.end(), im.data.begin(), im.data.end());
  const int n = geom.resolution, ch = viewMips[0].channels;
  PartialAtlas out;
  out.color = ImageF(n, n, ch, 0.0f);
  out.sampled.assign(static_cast<std::size_t>(n) * n, 0);
  double cam[7];
  camera7(camera, cam);
  check(mf_backproject_view(context(), n, f3(geom.position), geom.valid.data(), cam, camera.resolution, ch,
                            static_cast<int>(viewMips.size()), flat.data(), mask.data(), out.color.data.data(),
                            out.sampled.data()));
  return out;
}

ImageF incidenceMap(const GBuffer& geom, const OrthoCamera& camera, const ImageF& depthBuffer, double bboxDiagonal,
                    double depthTolerance) {
  checkIncidence(geom, camera, depthBuffer, bboxDiagonal, depthTolerance);
  const int n = geom.resolution;
  ImageF out(n, n, 1, 0.0f);
  double cam[7];
  camera7(camera, cam);
  check(mf_incidence_map(context(), n, f3(geom.position), f3(geom.normal), geom.valid.data(), cam, camera.resolution,
                         depthBuffer.data.data(), bboxDiagonal, depthTolerance, out.data.data()));
  return out;
}

TextureAtlas blendViews(const std::vector<PartialAtlas>& partials, const std::vector<ImageF>& incidence,
                        const std::vector<double>& priors, const BlendOptions& options) {
  const std::size_t k = partials.size();
  if (k == 0) throw Error(ErrorCode::InvalidConfig, "no views to blend");
  if (incidence.size() != k || priors.size() != k)
    throw Error(ErrorCode::InvalidConfig, "views, incidence maps and priors must pair up");
  if (!(options.epsilon > 0.0) || !(options.alpha >= 0.0))
    throw Error(ErrorCode::InvalidConfig, "blend needs epsilon > 0 and alpha >= 0");
  for (double p : priors)
    if (!(p >= 0.0)) throw Error(ErrorCode::InvalidConfig, "priors must be >= 0");
  const int w = partials[0].color.width, h = partials[0].color.height, ch = partials[0].color.channels;
  const std::size_t n = static_cast<std::size_t>(w) * h;
  std::vector<float> colors, inc;
  std::vector<std::uint8_t> sampled;
  colors.reserve(k * n * ch);
  inc.reserve(k * n);
  sampled.reserve(k * n);
  for (std::size_t i = 0; i < k; ++i) {
    const PartialAtlas& p = partials[i];
    if (p.color.width != w || p.color.height != h || p.color.channels != ch || p.sampled.size() != n)
      throw Error(ErrorCode::ShapeMismatch, "partial atlases disagree on resolution");
    if (incidence[i].width != w || incidence[i].height != h || incidence[i].channels != 1)
      throw Error(ErrorCode::ShapeMismatch, "incidence maps disagree on resolution");
    colors.insert(colors.end(), p.color.data.begin(), p.color.data.end());
    sampled.insert(sampled.end(), p.sampled.begin(), p.sampled.end());
    inc.insert(inc.end(), incidence[i].data.begin(), incidence[i].data.end());
  }
  TextureAtlas atlas;
  atlas.color = ImageF(w, h, ch, 0.0f);
  atlas.filled.assign(n, 0);
  check(mf_blend_views(context(), static_cast<int>(k), w, h, ch, colors.data(), sampled.data(), inc.data(),
                       priors.data(), options.alpha, options.epsilon, atlas.color.data.data(), atlas.filled.data()));
  return atlas;
}

std::vector<double> standardViewPriors() { return {1.0, 0.1, 0.01, 0.001, 1.0, 0.001, 0.01, 0.1, 0.3, 0.3}; }

TextureAtlas inpaintAtlas(const TextureAtlas&, const GBuffer&, double, const InpaintOptions&) {
  throw Error(ErrorCode::InvalidConfig, "inpaintAtlas is declared but never defined by the reference (fuse.h:110)");
}

TextureAtlas fuseViews(const GBuffer& geom, const std::vector<OrthoCamera>& cameras,
                       const std::vector<RenderedView>& views, const std::vector<ImageF>& colors,
                       const std::vector<double>& priors, double bboxDiagonal, const FuseOptions& options) {
  const std::size_t k = cameras.size();
  if (k == 0 || views.size() != k || colors.size() != k || priors.size() != k)
    throw Error(ErrorCode::InvalidConfig, "cameras, views, colors and priors must pair up");
  // the reference's per-view checks, in its order (fuse.cpp:305-312)
  for (std::size_t i = 0; i < k; ++i) {
    checkEdgeMask(views[i], bboxDiagonal, options.edgeThreshold);
    checkMips(colors[i], options.mipLevels, options.sharpenStrength);
    const std::size_t maskSize = static_cast<std::size_t>(views[i].position.width) * views[i].position.height;
    checkBackproject(geom, cameras[i].resolution, colors[i].width, colors[i].height, maskSize);
    checkIncidence(geom, cameras[i], views[i].depth, bboxDiagonal, options.depthTolerance);
  }
  if (!(options.blend.epsilon > 0.0) || !(options.blend.alpha >= 0.0))
    throw Error(ErrorCode::InvalidConfig, "blend needs epsilon > 0 and alpha >= 0");
  for (double p : priors)
    if (!(p >= 0.0)) throw Error(ErrorCode::InvalidConfig, "priors must be >= 0");
  const int vres = cameras[0].resolution, ch = colors[0].channels;
  for (std::size_t i = 1; i < k; ++i)
    if (cameras[i].resolution != vres || colors[i].channels != ch)
      throw Error(ErrorCode::InvalidConfig, "fused views must share one resolution and channel count");
  const std::size_t vn = static_cast<std::size_t>(vres) * vres;
  std::vector<double> cams(7 * k);
  std::vector<float> vpos, vdepth, cols;
  std::vector<std::int32_t> vface;
  vpos.reserve(3 * vn * k);
  vdepth.reserve(vn * k);
  vface.reserve(vn * k);
  cols.reserve(vn * k * ch);
  for (std::size_t i = 0; i < k; ++i) {
    camera7(cameras[i], cams.data() + 7 * i);
    vpos.insert(vpos.end(), views[i].position.data.begin(), views[i].position.data.end());
    vdepth.insert(vdepth.end(), views[i].depth.data.begin(), views[i].depth.data.end());
    vface.insert(vface.end(), views[i].face.data.begin(), views[i].face.data.end());
    cols.insert(cols.end(), colors[i].data.begin(), colors[i].data.end());
  }
  mf_fuse_options o;
  mf_fuse_options_default(&o);
  o.edge_threshold = options.edgeThreshold;
  o.depth_tolerance = options.depthTolerance;
  o.mip_levels = options.mipLevels;
  o.sharpen_strength = options.sharpenStrength;
  o.alpha = options.blend.alpha;
  o.epsilon = options.blend.epsilon;
  const int n = geom.resolution;
  TextureAtlas atlas;
  atlas.color = ImageF(n, n, ch, 0.0f);
  atlas.filled.assign(static_cast<std::size_t>(n) * n, 0);
  check(mf_fuse_views(context(), n, f3(geom.position), f3(geom.normal), geom.valid.data(), static_cast<int>(k),
                      cams.data(), vres, vpos.data(), vface.data(), vdepth.data(), ch, cols.data(), priors.data(),
                      bboxDiagonal, &o, atlas.color.data.data(), atlas.filled.data()));
  if (options.runInpaint) {
    for (std::size_t t = 0; t < atlas.filled.size(); ++t)
      if (geom.valid[t] && !atlas.filled[t]) return inpaintAtlas(atlas, geom, bboxDiagonal, options.inpaint);
  }
  return atlas;
}

}  // namespace meshforge
