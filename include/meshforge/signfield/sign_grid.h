// meshforge sign-grid surface band backed by the B200 LBVH (include/mfbake.h
// mf_surface_band). Source-compatible subset of
// proj/include/meshforge/signfield/sign_grid.h:11-50: the SignGrid /
// GridParams / VoxelLabel types and markSurfaceBand, the sign-field
// builder's bulk closest-point sweep (one bounded query per voxel centre,
// SURVEY §8f row 1). The grid-label passes that follow it in the reference
// (dilateBand, floodFillExterior, resolveUndetermined, ...) are integer
// flood fills outside the normal-bake hot path and are not provided here.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "meshforge/core/aabb.h"
#include "meshforge/core/mesh.h"
#include "meshforge/spatial/bvh.h"

namespace meshforge {

enum class VoxelLabel : std::uint8_t { Unknown, SurfaceBand, DilatedBand, Exterior, Interior };

// Cubic voxel grid of per-voxel labels and unsigned distances. Voxel (x,y,z)
// is centered at origin + (x+0.5, y+0.5, z+0.5) * voxelSize; storage is
// x-fastest (sign_grid.h:14-38).
struct SignGrid {
  int res = 0;
  double voxelSize = 0;
  Eigen::Vector3d origin = Eigen::Vector3d::Zero();
  double truncation = 0;
  std::vector<VoxelLabel> labels;
  std::vector<float> distance;
  std::int64_t failOpenCount = 0;

  std::size_t cells() const { return static_cast<std::size_t>(res) * res * res; }
  std::size_t index(int x, int y, int z) const {
    return static_cast<std::size_t>(x) + static_cast<std::size_t>(res) * (y + static_cast<std::size_t>(res) * z);
  }
  Eigen::Vector3d voxelCenter(int x, int y, int z) const {
    return origin + voxelSize * Eigen::Vector3d(x + 0.5, y + 0.5, z + 0.5);
  }
  std::int64_t countLabel(VoxelLabel label) const {
    std::int64_t n = 0;
    for (VoxelLabel l : labels) n += (l == label);
    return n;
  }
};

struct GridParams {
  int resolution = 128;
  double bandVoxels = 1.0;
  int dilateRadius = 2;
  std::optional<Aabb3d> domain;
};

// sign_grid.cpp:23-69 on the device. `bvh` must be built over `mesh` (as at
// every reference call site); the grid's bounds come from that mesh.
SignGrid markSurfaceBand(const TriangleMesh& mesh, const Bvh& bvh, const GridParams& params);

// Trilinear interpolation of the signed field at a world point, clamped to
// the voxel-center lattice (sign_grid.cpp:239-264; host, one point; sampleSdf
// evaluates it per point on the device).
double sampleSignedField(const SignGrid& grid, const std::vector<float>& field, const Eigen::Vector3d& p);

}  // namespace meshforge
