// meshforge multi-view visibility backed by the B200 LBVH (include/mfbake.h
// mf_cast_visibility): source-compatible subset of
// proj/include/meshforge/visibility/visibility.h:10-35 — FaceVisibility,
// VisibilityMask and castVisibility (one pixel ray per thread over all views,
// per-face won-pixel counts identical to the reference). The edge-flood
// passes that follow it (promoteExterior, removeHidden) are host graph
// algorithms outside the bake hot path and are not provided here.
#pragma once

#include <cstdint>
#include <vector>

#include "meshforge/core/mesh.h"

namespace meshforge {

enum class FaceVisibility : std::uint8_t { Hidden = 0, Visible = 1, PromotedExterior = 2 };

struct VisibilityMask {
  std::vector<FaceVisibility> state;
  std::vector<std::int64_t> hits;

  bool keep(int face) const { return state[face] != FaceVisibility::Hidden; }
  std::int64_t countState(FaceVisibility s) const {
    std::int64_t n = 0;
    for (auto v : state)
      if (v == s) ++n;
    return n;
  }
};

VisibilityMask castVisibility(const TriangleMesh& mesh, int viewpoints = 512, int resolution = 1024);

}  // namespace meshforge
