// The bake entry points, source-compatible with
// proj/include/meshforge/bake/gbuffer.h:17-55, implemented on the B200
// through include/mfbake.h. Layouts are the reference's: G-buffer texel
// (x, y) covers uv [x, x+1]/res x [y, y+1]/res with v running down the rows,
// attributes sampled at texel centres; the normal map is ImageU8(res, res, 3).
#pragma once

#include <Eigen/Core>
#include <cstdint>
#include <vector>

#include "meshforge/core/image.h"
#include "meshforge/core/mesh.h"

namespace meshforge {

struct GBuffer {
  int resolution = 0;
  std::vector<Eigen::Vector3f> position;
  std::vector<Eigen::Vector3f> normal;
  std::vector<Eigen::Vector3f> tangent;
  std::vector<Eigen::Vector3f> bitangent;
  std::vector<std::uint8_t> valid;
  std::vector<std::uint8_t> reliable;

  std::size_t index(int x, int y) const { return static_cast<std::size_t>(y) * resolution + x; }
  bool empty() const { return valid.empty(); }
};

// Centre-sampled UV rasterisation with the reference's canonical-edge tie
// rule; AtlasOverlap when two triangles claim a texel.
GBuffer rasterizeGBuffer(const TriangleMesh& lowpoly, int resolution);

// Bounded closest-point normal transfer into tangent space, RGB8 encoded.
ImageU8 transferNormals(const GBuffer& gbuffer, const TriangleMesh& highpoly, double bboxDiagonal,
                        double maxDistanceFraction = 0.01);

// 8-neighbour chamfer seam dilation over `radius` passes.
ImageU8 dilateSeams(const ImageU8& map, const GBuffer& gbuffer, int radius = 4);

// The three calls fused on the device (G-buffer never leaves HBM):
// dilateSeams(transferNormals(rasterizeGBuffer(lowpoly, res), highpoly, diag, frac), g, radius).
ImageU8 bakeNormalMap(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                      double bboxDiagonal, double maxDistanceFraction = 0.01, int radius = 4);

// B200 extensions (no reference equivalent; north_star item 4): the same
// fused bake written as RGBA8 (the RGB8 bytes plus alpha 255, 4 bytes per
// texel) or as RG16 (tangent-space x, y as unorm16 round((v + 1) / 2 * 65535);
// z = sqrt(1 - x^2 - y^2) on decode; background and neutral texels (0, 0)).
ImageU8 bakeNormalMapRGBA8(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                           double bboxDiagonal, double maxDistanceFraction = 0.01, int radius = 4);
Image<std::uint16_t> bakeNormalMapRG16(const TriangleMesh& lowpoly, const TriangleMesh& highpoly, int resolution,
                                       double bboxDiagonal, double maxDistanceFraction = 0.01, int radius = 4);

}  // namespace meshforge
