// common.cuh — shared device/host plumbing for libmfbake (sm_100a).
//
// Numeric policy: every translation unit is
// compiled with --fmad=false so fp64 expressions evaluate exactly as the
// reference's scalar code does under -ffp-contract=off (no DFMA contraction);
// fp32 pruning math uses explicit directed-rounding intrinsics.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "mfbake.h"

namespace mfb {

// ---------------------------------------------------------------- errors
struct Status {
  int code = MF_OK;
  std::string msg;
  bool ok() const { return code == MF_OK; }
};

void set_last_error(const std::string& msg);

#define MFB_CUDA_TRY(expr)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      throw ::mfb::CudaFailure(e_, #expr, __FILE__, __LINE__);                          \
    }                                                                                   \
  } while (0)

struct CudaFailure {
  cudaError_t err;
  const char* expr;
  const char* file;
  int line;
  CudaFailure(cudaError_t e, const char* x, const char* f, int l) : err(e), expr(x), file(f), line(l) {}
};

// A reference-code error (maps to 1 + ErrorCode across the ABI).
// Thrown by Ctx::buf / cub_temp when a buffer must grow while a stream
// capture is open (the old buffer cannot be freed without a sync): the
// capturing code discards the capture and runs the sequence eagerly.
struct CaptureRealloc {};

struct ApiError {
  int code;
  std::string msg;
  ApiError(int c, std::string m) : code(c), msg(std::move(m)) {}
};

// ---------------------------------------------------------------- device math
// Small fp64 3-vector with the reference's (Eigen-shim) operation order.
struct d3 {
  double x, y, z;
};
__host__ __device__ __forceinline__ d3 mk3(double x, double y, double z) { return d3{x, y, z}; }
__host__ __device__ __forceinline__ d3 operator+(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ __forceinline__ d3 operator-(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ __forceinline__ d3 operator*(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }
__host__ __device__ __forceinline__ d3 operator*(d3 a, double s) { return d3{a.x * s, a.y * s, a.z * s}; }
__host__ __device__ __forceinline__ d3 operator/(d3 a, double s) { return d3{a.x / s, a.y / s, a.z / s}; }
__host__ __device__ __forceinline__ double dot(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__host__ __device__ __forceinline__ double sqnorm(d3 a) { return dot(a, a); }
__host__ __device__ __forceinline__ double norm(d3 a) { return sqrt(sqnorm(a)); }
__host__ __device__ __forceinline__ d3 cross(d3 a, d3 b) {
  return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ __forceinline__ double cross2(double ax, double ay, double bx, double by) {
  return ax * by - ay * bx;
}
__device__ __forceinline__ d3 ld3(const double* p) { return d3{p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double* p, d3 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
}

// anyPerpendicular (bake/tangent.cpp:11-20)
__host__ __device__ __forceinline__ d3 any_perpendicular(d3 n) {
  const double an[3] = {fabs(n.x), fabs(n.y), fabs(n.z)};
  int s = 0;
  if (an[1] < an[s]) s = 1;
  if (an[2] < an[s]) s = 2;
  d3 axis = mk3(s == 0 ? 1.0 : 0.0, s == 1 ? 1.0 : 0.0, s == 2 ? 1.0 : 0.0);
  d3 p = cross(axis, n);
  double len = norm(p);
  return len > 1e-20 ? p / len : mk3(1.0, 0.0, 0.0);
}

// ---------------------------------------------------------------- launch geometry
constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace mfb
