// Standalone check of the LBVH radix sort (sort.cu) against std::stable_sort:
//   nvcc ... tools/sort_check.cu -Lpaper_2605_26137_b200 -lmfbake -o build/sort_check && build/sort_check
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "../paper_2605_26137_b200/csrc/bake.cuh"

using namespace mfb;

static int run(int n, unsigned seed, int key_bits) {
  std::mt19937 rng(seed);
  std::vector<uint32_t> k(n), v(n);
  for (int i = 0; i < n; ++i) {
    k[i] = rng() & ((1u << key_bits) - 1u);
    v[i] = i;
  }
  std::vector<int> hist(3 * 1024 + 4, 0);
  for (uint32_t x : k) {
    ++hist[x & 1023];
    ++hist[1024 + ((x >> 10) & 1023)];
    ++hist[2048 + (x >> 20)];
  }
  Ctx ctx;
  const int64_t sw = sort_status_words(n);
  uint32_t *dk, *dv, *dk2, *dv2, *st;
  int* dh;
  cudaMalloc(&dk, 4 * n);
  cudaMalloc(&dv, 4 * n);
  cudaMalloc(&dk2, 4 * n);
  cudaMalloc(&dv2, 4 * n);
  cudaMalloc(&st, 4 * sw);
  cudaMalloc(&dh, 4 * hist.size());
  cudaMemcpy(dk, k.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dh, hist.data(), 4 * hist.size(), cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 4 * sw);
  SortArgs a;
  a.keys = dk;
  a.vals = dv;
  a.keys_alt = dk2;
  a.vals_alt = dv2;
  a.n = n;
  a.hist = dh;
  a.status = st;
  a.counters = dh + 3 * 1024;
  try {
    radix_sort_morton30(ctx, 0, a);
  } catch (const CudaFailure& e) {
    std::printf("cuda failure %s\n", cudaGetErrorString(e.err));
    return 1;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("n=%d: %s\n", n, cudaGetErrorString(e));
    return 1;
  }
  std::vector<uint32_t> ok(n), ov(n);
  cudaMemcpy(ok.data(), dk2, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(ov.data(), dv2, 4 * n, cudaMemcpyDeviceToHost);
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return k[a] < k[b]; });
  int bad = 0, first = -1;
  for (int i = 0; i < n; ++i)
    if (ov[i] != static_cast<uint32_t>(idx[i]) || ok[i] != k[idx[i]]) {
      if (first < 0) first = i;
      ++bad;
    }
  std::printf("n=%8d bits=%2d: %s (%d mismatches, first %d)\n", n, key_bits, bad ? "FAIL" : "ok", bad, first);
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(dk2);
  cudaFree(dv2);
  cudaFree(st);
  cudaFree(dh);
  return bad != 0;
}

int main() {
  int fails = 0;
  for (int n : {1, 2, 100, 2047, 2048, 2049, 8191, 8192, 8193, 20000, 100000, 200000, 262144, 262145, 1003520})
    for (int bits : {30, 12}) fails += run(n, 7u + n, bits);
  std::printf("%s\n", fails ? "FAILED" : "all ok");
  {  // timing: 1,003,520 random 30-bit keys, 20 sorts
    const int n = 1003520;
    std::mt19937 rng(1);
    std::vector<uint32_t> k(n), v(n);
    std::vector<int> hist(3 * 1024 + 4, 0);
    for (int i = 0; i < n; ++i) {
      k[i] = rng() & ((1u << 30) - 1u);
      v[i] = i;
      ++hist[k[i] & 1023];
      ++hist[1024 + ((k[i] >> 10) & 1023)];
      ++hist[2048 + (k[i] >> 20)];
    }
    Ctx ctx;
    const int64_t sw = sort_status_words(n);
    uint32_t *dk, *dv, *dk2, *dv2, *st;
    int* dh;
    cudaMalloc(&dk, 4 * n);
    cudaMalloc(&dv, 4 * n);
    cudaMalloc(&dk2, 4 * n);
    cudaMalloc(&dv2, 4 * n);
    cudaMalloc(&st, 4 * sw);
    cudaMalloc(&dh, 4 * hist.size());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int it = 0; it < 20; ++it) {
      cudaMemcpy(dk, k.data(), 4 * n, cudaMemcpyHostToDevice);
      cudaMemcpy(dv, v.data(), 4 * n, cudaMemcpyHostToDevice);
      cudaMemcpy(dh, hist.data(), 4 * hist.size(), cudaMemcpyHostToDevice);
      cudaMemset(st, 0, 4 * sw);
      SortArgs sa;
      sa.keys = dk;
      sa.vals = dv;
      sa.keys_alt = dk2;
      sa.vals_alt = dv2;
      sa.n = n;
      sa.hist = dh;
      sa.status = st;
      sa.counters = dh + 3 * 1024;
      cudaEventRecord(a, 0);
      radix_sort_morton30(ctx, 0, sa);
      cudaEventRecord(b, 0);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    std::printf("sort of %d keys: best %.1f us (3 passes)\n", n, best * 1e3f);
  }
  return fails != 0;
}
