// Host-format tests of the B200 library's C++ API that need no GPU: OBJ
// (io/obj_io.cpp:46-165) and PNG (io/png_io.cpp) restating
// proj/tests/test_io.cpp:25-116 without its device-computed normals, plus
// reader edge cases. Run on the CPU by tests/test_io_cpu.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>

#include "meshforge/core/error.h"
#include "meshforge/io/obj_io.h"
#include "meshforge/io/png_io.h"
#include "meshforge/io/raster_io.h"

using namespace meshforge;

namespace {
std::string tmp(const std::string& name) { return "/tmp/mfb_io_" + name; }
void put(const std::string& path, const std::string& text) { std::ofstream(path) << text; }
}  // namespace

TEST_CASE("obj round trip is exact (positions, uvs, normals, faces)") {  // test_io.cpp:25-50
  TriangleMesh m;
  for (int i = 0; i < 40; ++i) m.positions.emplace_back(0.1 * i + 1e-17 * i, 1.0 / (i + 3), -0.3 * i * i);
  for (int i = 0; i < 40; ++i) m.normals.emplace_back(0.0, 1.0 / (i + 1), 0.7);
  m.uvs = {{0.0, 0.0}, {1.0, 0.0}, {0.25, 0.75}};
  for (int f = 0; f + 2 < 40; ++f) {
    m.faces.emplace_back(f, f + 1, f + 2);
    m.faceUvs.emplace_back(f % 3, (f + 1) % 3, (f + 2) % 3);
  }
  writeObj(tmp("rt.obj"), m);
  const TriangleMesh r = readObj(tmp("rt.obj"));
  REQUIRE(r.positions.size() == m.positions.size());
  REQUIRE(r.normals.size() == m.normals.size());
  REQUIRE(r.uvs.size() == m.uvs.size());
  REQUIRE(r.faces.size() == m.faces.size());
  for (size_t v = 0; v < m.positions.size(); ++v) {
    CHECK(r.positions[v] == m.positions[v]);
    CHECK(r.normals[v] == m.normals[v]);
  }
  for (size_t f = 0; f < m.faces.size(); ++f) {
    CHECK(r.faces[f] == m.faces[f]);
    CHECK(r.faceUvs[f] == m.faceUvs[f]);
  }
  std::remove(tmp("rt.obj").c_str());
}

TEST_CASE("polygons fan-triangulate and negative indices count back") {  // test_io.cpp:52-66
  put(tmp("quad.obj"), "# c\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf -4 -3 -2 -1\n\nv 2 2 2\nf 1 5 2\n");
  const TriangleMesh m = readObj(tmp("quad.obj"));
  REQUIRE(m.faceCount() == 3);
  CHECK(m.faces[0] == Eigen::Vector3i(0, 1, 2));
  CHECK(m.faces[1] == Eigen::Vector3i(0, 2, 3));
  CHECK(m.faces[2] == Eigen::Vector3i(0, 4, 1));
  CHECK(!m.hasUvs());
  CHECK(!m.hasNormals());
  std::remove(tmp("quad.obj").c_str());
}

TEST_CASE("partial uv sets and inconsistent normals are dropped") {  // test_io.cpp:68-79
  put(tmp("p.obj"), "v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nvt 0 0\nvt 1 0\nvt 0 1\nvn 0 0 1\nvn 0 1 0\n"
                    "f 1/1/1 2/2/1 3/3/1\nf 2//2 4//2 3//2\n");
  const TriangleMesh m = readObj(tmp("p.obj"));
  CHECK(m.faceCount() == 2);
  CHECK(m.uvs.empty());
  CHECK(m.faceUvs.empty());
  CHECK(m.normals.empty());  // vertex 1 names normal 1 then normal 2
  std::remove(tmp("p.obj").c_str());
}

TEST_CASE("reader errors keep the reference's codes and first-error order") {  // test_io.cpp:81-90
  CHECK_THROWS_AS(readObj(tmp("missing_422.obj")), Error);
  put(tmp("bad.obj"), "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\nf 1 2\n");
  try {
    readObj(tmp("bad.obj"));
    CHECK(false);
  } catch (const Error& e) {
    CHECK(e.code() == ErrorCode::InvalidGeometry);
    CHECK(std::string(e.what()).find("vertex index out of range") != std::string::npos);
  }
  put(tmp("few.obj"), "v 0 0 0\nv 1 0 0\nf 1 2\n");
  CHECK_THROWS_AS(readObj(tmp("few.obj")), Error);
  put(tmp("empty.obj"), "# nothing\n");
  try {
    readObj(tmp("empty.obj"));
    CHECK(false);
  } catch (const Error& e) {
    CHECK(e.code() == ErrorCode::EmptyMesh);
  }
  for (const char* n : {"bad.obj", "few.obj", "empty.obj"}) std::remove(tmp(n).c_str());
}

TEST_CASE("png round trip gray and rgb, odd sizes, many bands") {  // test_io.cpp:92-116
  for (int channels : {1, 3})
    for (int w : {1, 37, 2048})
      for (int h : {1, 23, 301}) {
        ImageU8 img(w, h, channels);
        uint32_t x = 12345u + w * 7u + h;
        for (auto& v : img.data) {
          x = x * 1664525u + 1013904223u;
          v = static_cast<uint8_t>((x >> 24) & (w == 2048 ? 0x0f : 0xff));
        }
        const auto bytes = encodePng(img);
        const ImageU8 r = decodePng(bytes.data(), bytes.size());
        REQUIRE(r.width == w);
        REQUIRE(r.height == h);
        REQUIRE(r.channels == channels);
        CHECK(r.data == img.data);
      }
  ImageU8 bad(4, 4, 2);
  CHECK_THROWS_AS(encodePng(bad), Error);
  const uint8_t junk[16] = {1, 2, 3};
  CHECK_THROWS_AS(decodePng(junk, sizeof(junk)), Error);
}
