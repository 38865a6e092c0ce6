// meshforge OBJ I/O (source-compatible with proj/include/meshforge/io/obj_io.h).
// readObj parses in parallel over line chunks (std::from_chars, correctly
// rounded like the reference's istream extraction) with the reference's
// semantics (io/obj_io.cpp:46-136): v / vt / vn / f, 1-based or negative
// indices, fan triangulation, uv sets kept only when every corner has one,
// per-vertex normals only when every corner names one consistent normal.
#pragma once

#include <string>

#include "meshforge/core/mesh.h"

namespace meshforge {

TriangleMesh readObj(const std::string& path);
// Doubles printed with max_digits10 (%.17g) so a write/read round trip is exact.
void writeObj(const std::string& path, const TriangleMesh& mesh);

}  // namespace meshforge
