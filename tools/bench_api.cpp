// bench_api — end-to-end timing of the reference-facing C++ API
// (include/meshforge/bake/gbuffer.h) through libmeshforge_b200, the way a
// drop-in caller uses it: TriangleMesh std::vectors (pageable host memory)
// in, ImageU8 out, synchronous calls, wall-clock time (steady_clock).
//
//   bench_api <mesh_dir> <res> <diag> <frac> <radius> <warmup> <steps>
//
// <mesh_dir> holds the raw arrays written by bench.py: lo_pos.f64, lo_faces.i32,
// lo_uvs.f64, lo_fuv.i32, hi_pos.f64, hi_faces.i32. Prints one JSON object:
// the fused bakeNormalMap and the reference's three-call composition
// dilateSeams(transferNormals(rasterizeGBuffer(lo, res), hi, diag, frac), g, r)
// (test_bake.cpp:205-206), per-call times in ms.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "meshforge/bake/gbuffer.h"

using namespace meshforge;

template <typename T>
static std::vector<T> load(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) {
    std::fprintf(stderr, "cannot open %s\n", path.c_str());
    std::exit(2);
  }
  const std::streamsize n = f.tellg();
  f.seekg(0);
  std::vector<T> v(static_cast<size_t>(n) / sizeof(T));
  f.read(reinterpret_cast<char*>(v.data()), n);
  return v;
}

template <typename V, typename S>
static std::vector<V> pack(const std::vector<S>& flat, int k) {
  std::vector<V> out(flat.size() / k);
  for (size_t i = 0; i < out.size(); ++i)
    for (int j = 0; j < k; ++j) out[i][j] = flat[i * k + j];
  return out;
}

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s mesh_dir res diag frac radius warmup steps\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const int res = std::atoi(argv[2]);
  const double diag = std::atof(argv[3]), frac = std::atof(argv[4]);
  const int radius = std::atoi(argv[5]), warmup = std::atoi(argv[6]), steps = std::atoi(argv[7]);
  TriangleMesh lo, hi;
  lo.positions = pack<Eigen::Vector3d>(load<double>(dir + "/lo_pos.f64"), 3);
  lo.faces = pack<Eigen::Vector3i>(load<int32_t>(dir + "/lo_faces.i32"), 3);
  lo.uvs = pack<Eigen::Vector2d>(load<double>(dir + "/lo_uvs.f64"), 2);
  lo.faceUvs = pack<Eigen::Vector3i>(load<int32_t>(dir + "/lo_fuv.i32"), 3);
  hi.positions = pack<Eigen::Vector3d>(load<double>(dir + "/hi_pos.f64"), 3);
  hi.faces = pack<Eigen::Vector3i>(load<int32_t>(dir + "/hi_faces.i32"), 3);

  using clk = std::chrono::steady_clock;
  auto time_calls = [&](auto&& fn, std::vector<double>& ms) {
    for (int i = 0; i < warmup; ++i) fn();
    for (int i = 0; i < steps; ++i) {
      const auto t0 = clk::now();
      fn();
      ms.push_back(std::chrono::duration<double, std::milli>(clk::now() - t0).count());
    }
  };
  size_t check = 0;
  std::vector<double> fused, three;
  time_calls([&] {
    const ImageU8 m = bakeNormalMap(lo, hi, res, diag, frac, radius);
    check += m.data[m.data.size() / 2];
  }, fused);
  ImageU8 last3;
  time_calls([&] {
    const GBuffer g = rasterizeGBuffer(lo, res);
    last3 = dilateSeams(transferNormals(g, hi, diag, frac), g, radius);
  }, three);
  const ImageU8 m = bakeNormalMap(lo, hi, res, diag, frac, radius);
  const bool same = m.data == last3.data;
  auto stats = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    double s = 0;
    for (double x : v) s += x;
    return std::make_pair(s / v.size(), v[v.size() / 2]);
  };
  const auto a = stats(fused), b = stats(three);
  std::printf("{\"fused_ms_mean\": %.4f, \"fused_ms_median\": %.4f, \"three_call_ms_mean\": %.4f, "
              "\"three_call_ms_median\": %.4f, \"steps\": %d, \"warmup\": %d, \"same_atlas\": %s, \"check\": %zu}\n",
              a.first, a.second, b.first, b.second, steps, warmup, same ? "true" : "false", check);
  return same ? 0 : 1;
}
