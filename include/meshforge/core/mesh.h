// TriangleMesh and the mesh helpers the bake path uses, source-compatible with
// proj/include/meshforge/core/mesh.h:15-40 (arrays of Eigen vectors whose
// data() the C ABI takes directly: Vector3d = 3 x f64, Vector3i = 3 x i32,
// Vector2d = 2 x f64). UVs are a separate pool indexed per corner by faceUvs.
#pragma once

#include <Eigen/Core>
#include <Eigen/Geometry>
#include <array>
#include <cstdint>
#include <utility>
#include <vector>

#include "meshforge/core/aabb.h"

namespace meshforge {

struct TriangleMesh {
  std::vector<Eigen::Vector3d> positions;
  std::vector<Eigen::Vector3i> faces;
  std::vector<Eigen::Vector3d> normals;   // empty, or one per position
  std::vector<Eigen::Vector2d> uvs;       // corner UV pool
  std::vector<Eigen::Vector3i> faceUvs;   // empty, or one per face

  int vertexCount() const { return static_cast<int>(positions.size()); }
  int faceCount() const { return static_cast<int>(faces.size()); }
  bool hasNormals() const { return !positions.empty() && normals.size() == positions.size(); }
  bool hasUvs() const { return !uvs.empty() && faceUvs.size() == faces.size(); }
};

// 0.5 * (p1 - p0) x (p2 - p0)
inline Eigen::Vector3d faceAreaVector(const TriangleMesh& m, int f) {
  const Eigen::Vector3d& p0 = m.positions[m.faces[f][0]];
  return 0.5 * (m.positions[m.faces[f][1]] - p0).cross(m.positions[m.faces[f][2]] - p0);
}
inline double faceArea(const TriangleMesh& m, int f) { return faceAreaVector(m, f).norm(); }
inline Eigen::Vector3d faceNormal(const TriangleMesh& m, int f) {
  const Eigen::Vector3d a = faceAreaVector(m, f);
  const double len = a.norm();
  return len > 0 ? Eigen::Vector3d(a / len) : Eigen::Vector3d::Zero();
}

// Bounding box of the positions.
Aabb3d bounds(const TriangleMesh& m);
// Sum of face areas in face order (core/mesh.cpp:18-22).
double surfaceArea(const TriangleMesh& m);
// Uniform scale + translation putting the mesh inside the sphere of the given
// radius centred at the origin; returns the scale (core/mesh.cpp:50-59).
double normalizeToSphere(TriangleMesh& m, double radius = 0.5);
// One shared transform mapping the pair's union bounding box into the unit
// cube (core/mesh.cpp:61-70).
void normalizePairToUnitCube(TriangleMesh& a, TriangleMesh& b);
// Area-weighted vertex normals summed in face order, normalised (zero stays
// zero) - computed on the B200 (mf_vertex_normals).
std::vector<Eigen::Vector3d> computeVertexNormals(const TriangleMesh& m);
// EmptyMesh when there are no faces; InvalidGeometry on a non-finite
// coordinate or an out-of-range face index.
void validateMesh(const TriangleMesh& m);

// Per-face edge-adjacent neighbour faces (-1 where none). Incidences of one
// edge pair up in face (then corner) order, first with second, third with
// fourth, as core/mesh.cpp:114-133 does.
std::vector<std::array<int, 3>> faceAdjacency(const TriangleMesh& m);
// Keeps the flagged faces in order and the vertices (and uv corners) they
// reference, renumbered in first-use order (core/mesh.cpp:154-186).
TriangleMesh extractFaces(const TriangleMesh& m, const std::vector<std::uint8_t>& keep);

// Order-independent 64-bit key of an undirected edge.
inline std::uint64_t edgeKey(int a, int b) {
  const auto lo = static_cast<std::uint32_t>(a < b ? a : b), hi = static_cast<std::uint32_t>(a < b ? b : a);
  return (static_cast<std::uint64_t>(lo) << 32) | hi;
}

}  // namespace meshforge
