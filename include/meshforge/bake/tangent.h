// Wedge tangent frames, source-compatible with
// proj/include/meshforge/bake/tangent.h:13-29; computed on the B200
// (mf_wedge_tangents). bitangent = normal x tangent.
#pragma once

#include <Eigen/Core>
#include <array>
#include <vector>

#include "meshforge/core/mesh.h"

namespace meshforge {

struct TangentFrame {
  Eigen::Vector3d tangent = Eigen::Vector3d::UnitX();
  Eigen::Vector3d bitangent = Eigen::Vector3d::UnitY();
  Eigen::Vector3d normal = Eigen::Vector3d::UnitZ();
};

// Per face, per corner {T, B, N}; throws InvalidGeometry without UVs.
std::vector<std::array<TangentFrame, 3>> computeWedgeTangents(const TriangleMesh& mesh);

// Unit vector perpendicular to n: axis of the smallest |n_k| (first minimum)
// crossed with n, normalised; UnitX when that vanishes (tangent.cpp:11-20).
Eigen::Vector3d anyPerpendicular(const Eigen::Vector3d& n);

}  // namespace meshforge
