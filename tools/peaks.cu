// Microbenchmarks for the two peaks SURVEY §8(d) says MEASURED_PEAKS.json
// lacks: L2 read bandwidth (the roofline denominator of the closest-point
// traversal, whose node/triangle records live in L2) and FP64 FMA throughput.
// Built as build/libmfpeaks.so (Makefile target `peaks`); bench.py calls it
// live on the box before the timed region. Not part of the product path.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace {

// Every CTA streams the whole buffer with 16-B loads that bypass L1
// (ld.global.cg), `reps` times; the buffer is sized to stay L2-resident.
__global__ void __launch_bounds__(512) k_l2_read(const uint4* __restrict__ buf, size_t n16, int reps,
                                                 unsigned* __restrict__ sink) {
  unsigned acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    // rotate the starting CTA per rep so every SM touches every slice
    const size_t base = (static_cast<size_t>(blockIdx.x + r * 37u) % gridDim.x) * blockDim.x + threadIdx.x;
    for (size_t i = base; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(buf + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;  // never true for the zeroed buffer; keeps the loads
}

// 8 independent DFMA chains per thread.
__global__ void __launch_bounds__(256) k_fp64(int iters, double seed, double* __restrict__ sink) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + k + threadIdx.x;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.0) sink[0] = s;
}

int sms(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

template <class F>
float time_best(F launch, int trials) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  float best = 1e30f;
  for (int t = 0; t < trials; ++t) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

}  // namespace

extern "C" {

// Sustained L2 read bandwidth over an L2-resident buffer of `bytes`, GB/s
// (10^9 B/s), best of 5.
int mfp_l2_read_gbs(int device, size_t bytes, int reps, double* gbs) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  uint4* buf = nullptr;
  unsigned* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return -2;
  cudaMalloc(&sink, sizeof(unsigned));
  cudaMemset(buf, 0, bytes);
  const size_t n16 = bytes / 16;
  const int grid = sms(device) * 4;
  const float ms = time_best([&] { k_l2_read<<<grid, 512>>>(buf, n16, reps, sink); }, 5);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(buf);
  cudaFree(sink);
  if (e != cudaSuccess) return -3;
  *gbs = static_cast<double>(n16) * 16.0 * reps / (ms * 1e-3) / 1e9;
  return 0;
}

// Dense FP64 FMA throughput, TFLOP/s (2 flops per FMA), best of 5.
int mfp_fp64_tflops(int device, double* tflops) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  double* sink = nullptr;
  cudaMalloc(&sink, sizeof(double));
  const int grid = sms(device) * 8, block = 256, iters = 4096;
  const float ms = time_best([&] { k_fp64<<<grid, block>>>(iters, 1.0, sink); }, 5);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(sink);
  if (e != cudaSuccess) return -3;
  const double flops = 2.0 * 8.0 * iters * static_cast<double>(grid) * block;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return 0;
}

}  // extern "C"
