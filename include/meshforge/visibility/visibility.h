// meshforge multi-view visibility backed by the B200 LBVH (include/mfbake.h
// mf_cast_visibility): source-compatible subset of
// proj/include/meshforge/visibility/visibility.h:10-35 — FaceVisibility,
// VisibilityMask and castVisibility (one pixel ray per thread over all views,
// per-face won-pixel counts identical to the reference), plus the host-side
// edge flood and compaction that complete the cull stage.
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

// Closure of Visible faces over edges whose unit face normals agree with the
// reached face's (dot >= cosThreshold): newly reached faces become
// PromotedExterior (visibility.cpp:60-93). ShapeMismatch on a foreign mask.
VisibilityMask promoteExterior(const TriangleMesh& mesh, const VisibilityMask& mask, double cosThreshold = 0.5);

// Keeps the Visible and PromotedExterior faces (extractFaces order); AllHidden
// when none survive; the mesh is returned untouched when all do (:95-113).
TriangleMesh removeHidden(const TriangleMesh& mesh, const VisibilityMask& mask);

// castVisibility -> promoteExterior -> removeHidden (:115-120).
TriangleMesh cullHiddenFaces(const TriangleMesh& mesh, int viewpoints = 512, int resolution = 1024,
                             double cosThreshold = 0.5);

}  // namespace meshforge
