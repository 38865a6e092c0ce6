// Zero-copy read bandwidth: SM loads from pinned (mapped) host memory, with
// and without a store of the data into a device buffer, vs cudaMemcpyAsync
// H2D of the same bytes.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/zc_bw.cu -o build/zc_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const int4* __restrict__ src, size_t n, int4* __restrict__ dst, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int4 v = __ldcs(src + i);
    if (dst) dst[i] = v;
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const size_t bytes = 12u << 20;
  const size_t n = bytes / 16;
  int4 *h, *d;
  unsigned* sink;
  cudaMallocHost(&h, bytes);
  for (size_t i = 0; i < n; ++i) h[i] = make_int4((int)i, 1, 2, 3);
  cudaMalloc(&d, bytes);
  cudaMalloc(&sink, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, s);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("memcpy H2D 12 MiB: %.1f us (%.1f GB/s)\n", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    for (int per : {2, 4, 8, 16}) {
      for (int store = 0; store < 2; ++store) {
        cudaEventRecord(a, s);
        k_read<<<sms * per, 256, 0, s>>>(h, n, store ? d : nullptr, sink);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("zero-copy read %2d CTAs/SM store=%d: %.1f us (%.1f GB/s)\n", per, store, ms * 1e3,
               bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
