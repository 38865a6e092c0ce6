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

// ---------------------------------------------------------------- atlas pixel formats
// (north_star item 4; MF_ATLAS_* in mfbake.h). RGB8 is the reference's
// ImageU8(res, res, 3) (gbuffer.cpp:212) with encodeChannel (gbuffer.cpp:85-88);
// RGBA8 is the same bytes plus alpha 255 as one aligned 32-bit store; RG16 is
// the tangent-space x, y as unorm16 (z = sqrt(1 - x^2 - y^2) on decode), one
// 32-bit store: the background and the neutral texel both encode (0, 0).
__host__ __device__ __forceinline__ int atlas_bpp(int fmt) { return fmt == MF_ATLAS_RGB8 ? 3 : 4; }
__device__ __forceinline__ uint32_t enc8(double v) {
  const long long q = llround((v + 1.0) * 0.5 * 255.0);
  return static_cast<uint32_t>(q < 0 ? 0 : (q > 255 ? 255 : q));
}
__device__ __forceinline__ uint32_t enc16(double v) {
  const long long q = llround((v + 1.0) * 0.5 * 65535.0);
  return static_cast<uint32_t>(q < 0 ? 0 : (q > 65535 ? 65535 : q));
}
// packed pixel: RGB8/RGBA8 little-endian r | g << 8 | b << 16 | a << 24, RG16 x | y << 16
__device__ __forceinline__ uint32_t px_rgb(int fmt, uint32_t r, uint32_t g, uint32_t b) {
  return r | (g << 8) | (b << 16) | (fmt == MF_ATLAS_RGBA8 ? 0xff000000u : 0u);
}
__device__ __forceinline__ uint32_t px_encode(int fmt, double x, double y, double z) {
  if (fmt == MF_ATLAS_RG16) return enc16(x) | (enc16(y) << 16);
  return px_rgb(fmt, enc8(x), enc8(y), enc8(z));
}
constexpr uint32_t kRG16Zero = 32768u | (32768u << 16);  // enc16(0), enc16(0)
// tangent-space (0, 0, 1): (128, 128, 255) (gbuffer.cpp:212-227)
__device__ __forceinline__ uint32_t px_neutral(int fmt) {
  return fmt == MF_ATLAS_RG16 ? kRG16Zero : px_rgb(fmt, 128, 128, 255);
}
// invalid texel: ImageU8(res, res, 3, 128) (gbuffer.cpp:212)
__device__ __forceinline__ uint32_t px_background(int fmt) {
  return fmt == MF_ATLAS_RG16 ? kRG16Zero : px_rgb(fmt, 128, 128, 128);
}
__device__ __forceinline__ void px_store(uint8_t* base, int64_t t, int fmt, uint32_t v) {
  if (fmt == MF_ATLAS_RGB8) {
    uint8_t* o = base + 3 * t;
    o[0] = static_cast<uint8_t>(v);
    o[1] = static_cast<uint8_t>(v >> 8);
    o[2] = static_cast<uint8_t>(v >> 16);
  } else {
    reinterpret_cast<uint32_t*>(base)[t] = v;
  }
}

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with launch_pdl may start (its CTAs become resident and
// run their prologue) while its same-stream predecessor is finishing; it must
// call pdl_wait() before touching anything the predecessor writes or reads.
// Predecessors call pdl_trigger() once every CTA has started, so the
// dependent's launch overlaps their tail. Inside a captured graph the
// dependency becomes a programmatic edge. Without the launch attribute both
// instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// Where the chain's kernels trigger: the sort passes before their write-out
// (the next pass's CTAs become resident meanwhile), the others implicitly at
// exit. Measured on config B: triggering right after each kernel's own wait
// 1.390-1.394 ms per bake (r01 timing), late 1.404-1.411, no PDL 1.409-1.414;
// with the bracketed per-step events of r02 the late form won.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef MFB_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  MFB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// ---------------------------------------------------------------- launch geometry
constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace mfb
