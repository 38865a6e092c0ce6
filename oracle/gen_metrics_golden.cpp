// Test infrastructure (not shipped): prints the reference's own metrics
// (oracle/_ref/libmfref.so, proj/src/metrics/metrics.cpp) on reference
// fixtures as hex floats; tests/cpp/test_bake_b200.cpp pins the B200 C++ API
// to them. Build/run: make -C oracle metrics-golden
#include <cstdio>

#include "meshforge/metrics/metrics.h"
#include "support/fixtures.h"

using namespace meshforge;

int main() {
  const TriangleMesh a = fixtures::icosphere(3), b = fixtures::icosphere(4);
  std::printf("chamfer(ico3, ico4, 20000, 7)   = %a\n", chamferDistance(a, b, 20000, 7));
  std::printf("hausdorff(ico3, ico4, 20000, 7) = %a\n", hausdorffDistance(a, b, 20000, 7));
  std::printf("geoMeanErrorDeg(ico2, ico4, 5000, 7) = %a\n", geoMeanErrorDeg(fixtures::icosphere(2), b, 5000, 7));
  return 0;
}
