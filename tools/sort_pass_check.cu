// One onesweep pass of sort.cu vs a host stable counting sort (debug).
#define MFB_SORT_DEBUG 1
#include "../paper_2605_26137_b200/csrc/sort.cu"
#include <cstdio>
#include <random>
#include <vector>
using namespace mfb;
int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 8193;
  std::mt19937 rng(3);
  std::vector<uint32_t> k(n), v(n);
  for (int i = 0; i < n; ++i) { k[i] = rng() & ((1u << 30) - 1); v[i] = i; }
  std::vector<int> hist(1024, 0);
  for (uint32_t x : k) ++hist[x & 1023];
  const int tiles = (n + kTile - 1) / kTile;
  uint32_t *dk, *dv, *dk2, *dv2, *st; int *dh, *cnt;
  cudaMalloc(&dk, 4 * n); cudaMalloc(&dv, 4 * n); cudaMalloc(&dk2, 4 * n); cudaMalloc(&dv2, 4 * n);
  cudaMalloc(&st, 4 * tiles * kBins); cudaMalloc(&dh, 4096); cudaMalloc(&cnt, 4);
  cudaMemcpy(dk, k.data(), 4 * n, cudaMemcpyHostToDevice); cudaMemcpy(dv, v.data(), 4 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dh, hist.data(), 4096, cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 4 * tiles * kBins); cudaMemset(cnt, 0, 4);
  cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(SortSmem));
  k_onesweep<<<tiles, kSortThreads, sizeof(SortSmem)>>>(dk, dv, dk2, dv2, n, 0, dh, st, cnt);
  printf("launch %s sync %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<uint32_t> ok(n), ov(n), stat(tiles * kBins);
  cudaMemcpy(ok.data(), dk2, 4 * n, cudaMemcpyDeviceToHost); cudaMemcpy(ov.data(), dv2, 4 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(stat.data(), st, 4 * tiles * kBins, cudaMemcpyDeviceToHost);
  std::vector<int> start(1024, 0);
  for (int d = 1; d < 1024; ++d) start[d] = start[d - 1] + hist[d - 1];
  std::vector<uint32_t> ek(n), ev(n);
  for (int i = 0; i < n; ++i) { int d = k[i] & 1023; ek[start[d]] = k[i]; ev[start[d]] = v[i]; ++start[d]; }
  int bad = 0;
  for (int i = 0; i < n; ++i) if (ek[i] != ok[i] || ev[i] != ov[i]) { if (bad < 8) printf("pos %d: got (%u,%u) want (%u,%u)\n", i, ok[i] & 1023, ov[i], ek[i] & 1023, ev[i]); ++bad; }
  printf("n=%d tiles=%d mismatches %d\n", n, tiles, bad);
  int hd[64];
  cudaMemcpyFromSymbol(hd, g_sort_dbg, sizeof(hd));
  for (int b = 0; b < tiles && b < 8; ++b) printf("cta %d: tile %d excl0 %d first_status %08x iters %d\n", b, hd[4*b], hd[4*b+1], hd[4*b+2], hd[4*b+3]);
  for (int t = 0; t < tiles && t < 3; ++t) printf("tile %d status d0..3: %08x %08x %08x %08x\n", t, stat[t*kBins], stat[t*kBins+1], stat[t*kBins+2], stat[t*kBins+3]);
}
