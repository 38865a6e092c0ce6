// sort.cu — the LBVH's key sort and the library's prefix sums, hand-written
// for sm_100a (no CUB on the bake path).
//
// radix_sort_morton30: stable LSD sort of (30-bit Morton key, face id) pairs in
//   three 10-bit passes. The three 1024-bin digit histograms are built by the
//   Morton kernel itself (morton_hist_args); each pass is ONE kernel in the
//   onesweep style: a CTA takes the next 8192-key tile (dynamic tile order, so
//   look-back only ever waits on running CTAs), ranks its keys per warp with
//   __match_any_sync (stable: element order within the warp, warps in tile
//   order), publishes its per-digit tile counts, sums the earlier tiles'
//   published counts (8 independent loads in flight per digit) back to the
//   first inclusive prefix for its exclusive digit prefix, publishes its own
//   inclusive prefix, shuffles the tile
//   into digit order in shared memory and writes it out in per-digit runs.
//   Config B (1,003,520 keys): 123 tiles, one wave at 2 CTAs/SM.
// scan_exclusive: single-pass decoupled look-back exclusive sum of int32.
//
// Stability makes the result identical to any stable sort by key (the former
// CUB onesweep included): equal keys keep face order.
#include <cuda_runtime.h>

#include <algorithm>

#include "bake.cuh"

namespace mfb {
namespace {

constexpr int kWin = 8;  // look-back status loads in flight per digit
constexpr int kDigitBits = 10;
constexpr int kBins = 1 << kDigitBits;
constexpr int kSortThreads = 512;
constexpr int kSortWarps = kSortThreads / 32;
// Keys per thread: 16 (8192-key tiles) for large sorts; 4 (2048-key tiles)
// up to kSmallSortKeys, where a pass is one short wave of few tiles and the
// per-CTA latency is the pass time. Measured per bake (ms): config B (1M keys)
// 16 / 8 / 4: 1.424 / 1.434 / 1.439; config D (500k) 0.481 / 0.485 / 0.480;
// config A (200k) 0.237 / 0.234 / 0.218.
constexpr int kPerLaneLarge = 16;
constexpr int kPerLaneSmall = 4;
constexpr int kSmallSortKeys = 1 << 18;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kCountMask = (1u << 30) - 1u;

// Look-back status words: relaxed GPU-scope loads / stores as volatile asm.
// (A plain or __ldcg load in a spin loop has no side effect, so the compiler
// may assume the loop exits after one iteration.)
__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int kPerLane>
struct SortSmem {
  static constexpr int kTile = kSortThreads * kPerLane;
  uint16_t warp_hist[kSortWarps][kBins];  // per-warp digit counts -> per-warp exclusive prefix
  int tile_start[kBins];                  // exclusive scan of the tile's digit counts
  int out_off[kBins];                     // global destination of the digit's first tile element
  uint32_t keys[kTile];
  uint32_t vals[kTile];
  int tile_id;
  int scan_carry[kSortWarps];
};

// exclusive scan of v over the block's 512 threads (2 values per thread: lo, hi)
__device__ __forceinline__ void block_scan_pairs(int& lo, int& hi, int* carry) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s = lo + hi;
  int incl = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) carry[w] = incl;
  __syncthreads();
  if (w == 0) {
    int c = lane < kSortWarps ? carry[lane] : 0;
    int ci = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ci, off);
      if (lane >= off) ci += y;
    }
    if (lane < kSortWarps) carry[lane] = ci - c;
  }
  __syncthreads();
  const int excl = carry[w] + incl - s;
  hi = excl + lo;
  lo = excl;
  __syncthreads();
}

template <int kPerLane>
__global__ void __launch_bounds__(kSortThreads, kPerLane <= 8 ? 3 : 2)
    k_onesweep(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
               uint32_t* __restrict__ vout, int n, int shift, const int* __restrict__ ghist,
               uint32_t* __restrict__ status, int* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kTile = kSortThreads * kPerLane;  // keys per tile
  constexpr int kWarpKeys = 32 * kPerLane;        // keys per warp
  SortSmem<kPerLane>& sm = *reinterpret_cast<SortSmem<kPerLane>*>(smem_raw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  pdl_wait();
  if (threadIdx.x == 0) sm.tile_id = atomicAdd(tile_counter, 1);
  for (int i = threadIdx.x; i < kSortWarps * kBins / 2; i += kSortThreads)
    reinterpret_cast<uint32_t*>(sm.warp_hist)[i] = 0u;
  __syncthreads();
  const int tile = sm.tile_id;
  const int base = tile * kTile + w * kWarpKeys;
  // load: warp-striped (element base + j*32 + lane), i.e. j-major = element order
  uint32_t key[kPerLane], val[kPerLane];
  uint16_t rank[kPerLane];
#pragma unroll
  for (int j = 0; j < kPerLane; ++j) {
    const int e = base + j * 32 + lane;
    key[j] = e < n ? __ldcs(kin + e) : 0xffffffffu;
    val[j] = e < n ? __ldcs(vin + e) : 0u;
  }
  // stable per-warp ranks
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kPerLane; ++j) {
    const bool live = key[j] != 0xffffffffu;
    const int d = live ? static_cast<int>((key[j] >> shift) & (kBins - 1)) : kBins;
    // warp multi-split: lanes with the same 10-bit digit by 10 ballots
    // (instead of __match_any_sync: 75.7 -> 65.5 us per 1M-key sort)
    unsigned peers = __ballot_sync(0xffffffffu, live);
#pragma unroll
    for (int b = 0; b < kDigitBits; ++b) {
      const bool bit = (d >> b) & 1;
      const unsigned m = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? m : ~m;
    }
    if (!live) peers = 1u << lane;
    const int leader = __ffs(peers) - 1;
    int old = 0;
    if (live && lane == leader) {
      old = sm.warp_hist[w][d];
      sm.warp_hist[w][d] = static_cast<uint16_t>(old + __popc(peers));
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[j] = static_cast<uint16_t>(old + __popc(peers & lt));
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp prefix (in place), tile total; thread owns digits 2t, 2t+1
  int tot[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int d = 2 * threadIdx.x + k;
    int acc = 0;
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const int c = sm.warp_hist[ww][d];
      sm.warp_hist[ww][d] = static_cast<uint16_t>(acc);
      acc += c;
    }
    tot[k] = acc;
    // publish the tile's aggregate
    const uint32_t v = kFlagAgg | static_cast<uint32_t>(acc);
    st_status(status + static_cast<int64_t>(tile) * kBins + d, v);
  }
  // tile-local digit starts (exclusive scan over the 1024 digits)
  int s0 = tot[0], s1 = tot[1];
  block_scan_pairs(s0, s1, sm.scan_carry);
  sm.tile_start[2 * threadIdx.x] = s0;
  sm.tile_start[2 * threadIdx.x + 1] = s1;
  // decoupled look-back for the tile's exclusive prefix per digit, plus the
  // global digit base (exclusive scan of this pass's histogram)
  int gb0 = ghist[2 * threadIdx.x], gb1 = ghist[2 * threadIdx.x + 1];
  block_scan_pairs(gb0, gb1, sm.scan_carry);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int d = 2 * threadIdx.x + k;
    // look back over the earlier tiles 8 at a time (independent loads): sum
    // their published counts down to the first inclusive prefix; every tile
    // publishes its aggregate right after ranking, so no tile waits on a
    // serial chain of inclusive prefixes
    int excl = 0;
    for (int t1 = tile - 1; t1 >= 0; t1 -= kWin) {
      uint32_t v[kWin];
#pragma unroll
      for (int u = 0; u < kWin; ++u)
        v[u] = t1 - u >= 0 ? ld_status(status + static_cast<int64_t>(t1 - u) * kBins + d) : kFlagInc;
      bool done = false;
#pragma unroll
      for (int u = 0; u < kWin; ++u) {
        if (done) break;
        if (t1 - u < 0) {
          done = true;
          break;
        }
        while ((v[u] & (kFlagAgg | kFlagInc)) == 0u) v[u] = ld_status(status + static_cast<int64_t>(t1 - u) * kBins + d);
        excl += static_cast<int>(v[u] & kCountMask);
        done = (v[u] & kFlagInc) != 0u;
      }
      if (done) break;
    }
    st_status(status + static_cast<int64_t>(tile) * kBins + d, kFlagInc | static_cast<uint32_t>(excl + tot[k]));
    sm.out_off[d] = (k == 0 ? gb0 : gb1) + excl - sm.tile_start[d];
  }
  __syncthreads();
  // shuffle into digit order in shared memory
#pragma unroll
  for (int j = 0; j < kPerLane; ++j) {
    if (key[j] == 0xffffffffu) continue;
    const int d = static_cast<int>((key[j] >> shift) & (kBins - 1));
    const int s = sm.tile_start[d] + sm.warp_hist[w][d] + rank[j];
    sm.keys[s] = key[j];
    sm.vals[s] = val[j];
  }
  __syncthreads();
  // write out: consecutive threads take consecutive tile slots (per-digit runs)
  pdl_trigger();  // before the write-out: the next pass's CTAs become resident
  const int count = min(kTile, n - tile * kTile);
  for (int i = threadIdx.x; i < count; i += kSortThreads) {
    const uint32_t k = sm.keys[i];
    const int d = static_cast<int>((k >> shift) & (kBins - 1));
    const int dst = sm.out_off[d] + i;
    kout[dst] = k;
    vout[dst] = sm.vals[i];
  }
}

// ---------------------------------------------------------------- exclusive scan
constexpr int kScanThreads = 512;
constexpr int kScanPer = 8;
constexpr int kScanTile = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) k_scan_exclusive(const int* __restrict__ in, int* __restrict__ out,
                                                                 int n, uint32_t* __restrict__ status,
                                                                 int* __restrict__ tile_counter) {
  __shared__ int carry[kScanThreads / 32];
  __shared__ int tile_s, prefix_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = tile_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = static_cast<int64_t>(tile) * kScanTile + threadIdx.x * kScanPer;
  int v[kScanPer], s = 0;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    v[j] = b + j < n ? in[b + j] : 0;
    s += v[j];
  }
  int incl = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) carry[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int c = lane < kScanThreads / 32 ? carry[lane] : 0;
    int ci = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ci, off);
      if (lane >= off) ci += y;
    }
    if (lane < kScanThreads / 32) carry[lane] = ci - c;
    if (lane == kScanThreads / 32 - 1) {  // tile total: publish, look back
      const int total = ci;
      if (tile == 0) {
        st_status(status, kFlagInc | static_cast<uint32_t>(total));
        prefix_s = 0;
      } else {
        st_status(status + tile, kFlagAgg | static_cast<uint32_t>(total));
        int excl = 0;
        for (int t = tile - 1; t >= 0; --t) {
          uint32_t x;
          do {
            x = ld_status(status + t);
          } while ((x & (kFlagAgg | kFlagInc)) == 0u);
          excl += static_cast<int>(x & kCountMask);
          if (x & kFlagInc) break;
        }
        st_status(status + tile, kFlagInc | static_cast<uint32_t>(excl + total));
        prefix_s = excl;
      }
    }
  }
  __syncthreads();
  int run = prefix_s + carry[w] + incl - s;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    if (b + j < n) out[b + j] = run;
    run += v[j];
  }
}

__global__ void k_zero_u32(uint32_t* __restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = 0u;
}

}  // namespace

static int sort_tile_keys(int n) { return kSortThreads * (n <= kSmallSortKeys ? kPerLaneSmall : kPerLaneLarge); }

int64_t sort_status_words(int n) {
  return static_cast<int64_t>(3) * div_up(std::max(n, 1), sort_tile_keys(n)) * kBins + 8;
}

template <int kPerLane>
static void onesweep_passes(cudaStream_t s, const SortArgs& a) {
  const int n = a.n;
  static const size_t smem = sizeof(SortSmem<kPerLane>);
  static bool attr = [] {
    MFB_CUDA_TRY(cudaFuncSetAttribute(k_onesweep<kPerLane>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return true;
  }();
  (void)attr;
  const int tiles = div_up(n, kSortThreads * kPerLane);
  uint32_t* kin = a.keys;
  uint32_t* vin = a.vals;
  uint32_t* kout = a.keys_alt;
  uint32_t* vout = a.vals_alt;
  for (int pass = 0; pass < 3; ++pass) {
    uint32_t* status = a.status + static_cast<int64_t>(pass) * tiles * kBins;
    launch_pdl(k_onesweep<kPerLane>, tiles, kSortThreads, smem, s, kin, vin, kout, vout, n, pass * kDigitBits,
               a.hist + pass * kBins, status, a.counters + pass);
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
}

void radix_sort_morton30(Ctx& ctx, cudaStream_t s, const SortArgs& a) {
  if (a.n <= 0) return;
  if (a.n <= kSmallSortKeys)
    onesweep_passes<kPerLaneSmall>(s, a);
  else
    onesweep_passes<kPerLaneLarge>(s, a);
  ctx.count_launch(3);
  MFB_CUDA_TRY(cudaGetLastError());
  // three passes: the sorted pairs end in keys_alt / vals_alt
}

void scan_exclusive(Ctx& ctx, cudaStream_t s, const int* in, int* out, int n, const std::string& tag) {
  if (n <= 0) return;
  const int tiles = div_up(n, kScanTile);
  auto* status = ctx.buf<uint32_t>(tag + ".scanst", tiles + 1);  // [0, tiles): tile status, [tiles]: counter
  k_zero_u32<<<1, 256, 0, s>>>(status, tiles + 1);
  k_scan_exclusive<<<tiles, kScanThreads, 0, s>>>(in, out, n, status, reinterpret_cast<int*>(status + tiles));
  ctx.count_launch(2);
  MFB_CUDA_TRY(cudaGetLastError());
}

}  // namespace mfb
