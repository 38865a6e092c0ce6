// dilate.cu — dilateSeams (bake/gbuffer.cpp:254-322) on the device.
//
// The reference runs `radius` double-buffered 8-neighbour chamfer passes over
// the whole atlas, each texel keeping (source, dist2) with dist2 ==
// |texel - source|^2 exactly, and finally copies the input map at the source.
// Bit-exact restatement:
//   * state is the source offset (dx, dy) relative to the texel; dist2 is
//     recomputed exactly from it (int32 suffices while |offset| <= radius);
//   * neighbours are scanned in the reference's (dy, dx) raster order and a
//     candidate wins only if strictly nearer, so ties keep the current source,
//     then the first neighbour in scan order (gbuffer.cpp:288-303).
// k_dilate_fused runs all passes for one 64x16 tile inside shared memory over
// a (64+2r) x (16+2r) halo region (one launch, ~1.7x halo read of the 1-byte
// mask at r = 4); k_dilate_pass is the multi-launch global fallback for radii
// whose halo does not fit in shared memory.
#include <atomic>
#include "bake.cuh"

namespace mfb {
namespace {

constexpr int kTW = 64, kTH = 16;
constexpr int16_t kNone = -32768;  // "no source" marker in the x offset

__device__ __forceinline__ int sq(int v) { return v * v; }

// One chamfer step (gbuffer.cpp:284-305) for the texel at region coords
// (cx, cy) of a rw x rh region whose origin is (x0, y0) in the image. ox/oy
// hold source offsets; ox == kNone means no source. Neighbours outside the
// image are skipped exactly as in the reference; cells outside the region are
// never read (the caller only updates cells at least one step inside).
// Distances are exact in int32: |offset| <= radius <= 64 keeps them below
// 2^14 (the reference's int64 values are the same integers). kBorder = false
// for tiles whose region lies inside the image (no neighbour bounds checks).
template <bool kBorder>
__device__ __forceinline__ void chamfer_step(const int16_t* __restrict__ ox, const int16_t* __restrict__ oy,
                                             int rw, int cx, int cy, int gx, int gy, int width, int height,
                                             int16_t& nox, int16_t& noy) {
  const int self = cy * rw + cx;
  const int16_t sx = ox[self], sy = oy[self];
  nox = sx;
  noy = sy;
  if (sx == 0 && sy == 0) return;  // valid texel: dist2 == 0, skipped
  int best = sx == kNone ? 0x7fffffff : sq(sx) + sq(sy);
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      if (kBorder) {
        const int nx = gx + dx, ny = gy + dy;
        if (nx < 0 || nx >= width || ny < 0 || ny >= height) continue;
      }
      const int n = self + dy * rw + dx;
      const int16_t nsx = ox[n];
      if (nsx == kNone) continue;
      const int cxo = dx + nsx, cyo = dy + oy[n];
      const int d = sq(cxo) + sq(cyo);
      if (d < best) {
        best = d;
        nox = static_cast<int16_t>(cxo);
        noy = static_cast<int16_t>(cyo);
      }
    }
  }
}

// The chamfer state of one 64x16 output tile over its (64+2r) x (16+2r) halo
// region in shared memory (sm: 4 planes of rw*rh int16). Returns false for
// tiles whose output texels are all valid, or whose region holds no valid
// texel (nothing to propagate); otherwise runs the r passes and leaves the
// final source offsets in *ox / *oy. Pass k (1-based) updates only cells at
// least k steps inside the region: exactly the cells the output depends on,
// so the region shrinks by one ring per pass.
__device__ __forceinline__ bool chamfer_tile(int width, int height, const uint8_t* __restrict__ valid,
                                             int in_row0, int in_rows, int radius, int out_row0, int out_rows,
                                             int16_t* sm, const int16_t** ox, const int16_t** oy) {
  const int rw = kTW + 2 * radius, rh = kTH + 2 * radius, cells = rw * rh;
  int16_t* ox0 = sm;
  int16_t* oy0 = sm + cells;
  int16_t* ox1 = sm + 2 * cells;
  int16_t* oy1 = sm + 3 * cells;
  const int tiles_x = (width + kTW - 1) / kTW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x0 = tx * kTW - radius;            // region origin (absolute)
  const int y0 = out_row0 + ty * kTH - radius;
  const int in_end = in_row0 + in_rows;
  const int out_end = out_row0 + out_rows;
  int any_valid = 0, any_hole = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // (row per warp, lanes along the row: no integer division per cell)
  for (int ly = warp; ly < rh; ly += nwarps)
    for (int lx = lane; lx < rw; lx += 32) {
      const int c = ly * rw + lx;
      const int gx = x0 + lx, gy = y0 + ly;
      int16_t v = kNone;
      const bool inimg = gx >= 0 && gx < width && gy >= in_row0 && gy < in_end && gy < height;
      if (inimg && valid[static_cast<int64_t>(gy - in_row0) * width + gx]) v = 0;
      ox0[c] = v;
      oy0[c] = 0;
      any_valid |= v == 0;
      const bool out_cell = lx >= radius && lx < radius + kTW && ly >= radius && ly < radius + kTH &&
                            gx < width && gy < out_end;
      any_hole |= out_cell && v != 0;
    }
  const bool work = __syncthreads_or(any_valid) && __syncthreads_or(any_hole);
  if (!work) return false;
  // the region (and so every neighbour read) lies inside the image
  const bool interior = x0 >= 0 && x0 + rw <= width && y0 >= 0 && y0 + rh <= height;
  for (int pass = 1; pass <= radius; ++pass) {
    for (int cy = pass + warp; cy < rh - pass; cy += nwarps)
      for (int cx = pass + lane; cx < rw - pass; cx += 32) {
        const int i = cy * rw + cx;
        int16_t a, b;
        if (interior) chamfer_step<false>(ox0, oy0, rw, cx, cy, x0 + cx, y0 + cy, width, height, a, b);
        else chamfer_step<true>(ox0, oy0, rw, cx, cy, x0 + cx, y0 + cy, width, height, a, b);
        ox1[i] = a;
        oy1[i] = b;
      }
    __syncthreads();
    int16_t* t = ox0;
    ox0 = ox1;
    ox1 = t;
    t = oy0;
    oy0 = oy1;
    oy1 = t;
    // (pass k + 1 reads only cells in [k, rw - k) x [k, rh - k), all
    // written by pass k, so the stale outer ring is never read)
  }
  *ox = ox0;
  *oy = oy0;
  return true;
}

// One 64x16 output tile per 256-thread CTA: the chamfer state in shared
// memory (chamfer_tile), then every output texel copies the input map at its
// source; copy-only tiles move 16-byte words.
__global__ void __launch_bounds__(256) k_dilate_fused(int width, int height, int channels,
                                                      const uint8_t* __restrict__ map_in,
                                                      const uint8_t* __restrict__ valid, int in_row0,
                                                      int in_rows, int radius, OutSet outs,
                                                      int out_row0, int out_rows) {
  extern __shared__ int16_t sm[];
  const int rw = kTW + 2 * radius;
  const int tiles_x = (width + kTW - 1) / kTW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int out_end = out_row0 + out_rows;
  const int16_t *ox0 = nullptr, *oy0 = nullptr;
  const bool work = chamfer_tile(width, height, valid, in_row0, in_rows, radius, out_row0, out_rows, sm, &ox0, &oy0);
  // copy-only tile, full width, 16-byte aligned rows: 16-byte moves
  const int gx0 = tx * kTW, gy0 = out_row0 + ty * kTH;
  if (!work && gx0 + kTW <= width && gy0 + kTH <= out_end) {
    const int64_t row_bytes = static_cast<int64_t>(width) * channels;
    const uint8_t* src0 = map_in + (static_cast<int64_t>(gy0 - in_row0) * width + gx0) * channels;
    const int64_t dst_off = (static_cast<int64_t>(gy0 - outs.row0) * width + gx0) * channels;
    const int vec_per_row = kTW * channels / 16;
    bool aligned = kTW * channels % 16 == 0 && row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src0) & 15) == 0;
    for (int k = 0; k < outs.n; ++k) aligned = aligned && (reinterpret_cast<uintptr_t>(outs.p[k] + dst_off) & 15) == 0;
    if (aligned) {
      for (int c = threadIdx.x; c < vec_per_row * kTH; c += blockDim.x) {
        const int r = c / vec_per_row, k = c % vec_per_row;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src0 + r * row_bytes) + k);
        for (int o = 0; o < outs.n; ++o) reinterpret_cast<uint4*>(outs.p[o] + dst_off + r * row_bytes)[k] = v;
      }
      return;
    }
  }
  // output: tile interior (4 texels per thread, row-contiguous)
  for (int c = threadIdx.x; c < kTW * kTH; c += blockDim.x) {
    const int lx = c % kTW, ly = c / kTW;
    const int gx = tx * kTW + lx, gy = out_row0 + ty * kTH + ly;
    if (gx >= width || gy >= out_end) continue;
    int srcx = gx, srcy = gy;
    if (work) {
      const int rc = (ly + radius) * rw + (lx + radius);
      const int16_t sx = ox0[rc], sy = oy0[rc];
      if (sx != kNone && !(sx == 0 && sy == 0)) {
        srcx = gx + sx;
        srcy = gy + sy;
      }
    }
    const uint8_t* src = map_in + (static_cast<int64_t>(srcy - in_row0) * width + srcx) * channels;
    const int64_t doff = (static_cast<int64_t>(gy - outs.row0) * width + gx) * channels;
    for (int o = 0; o < outs.n; ++o)
      for (int ch = 0; ch < channels; ++ch) outs.p[o][doff + ch] = src[ch];
  }
}


// ---- sparse chamfer (radius <= 32) -----------------------------------------
// Only invalid in-image cells within Chebyshev distance r of a valid cell can
// ever hold a source after r passes; every other cell keeps its initial state
// (valid: (0,0); far from any valid texel: none). The region's valid mask is
// built as bit rows by warp ballots, dilated by r (funnel shifts across the
// row's words, then an OR over 2r+1 rows), and the candidate cells compacted
// into a list; the passes update only listed cells (the same double-buffered
// chamfer_step, packed as one int32 per cell). At config B, 119k gutter texels
// over 1009 of 4096 tiles: ~20x fewer cell updates than the dense passes.
constexpr int kSparseMaxR = 32;
constexpr int kNoneP = 0x00008000;  // packed (ox = -32768 = none, oy = 0)
constexpr int kWordLoadMaxR = 30;   // 3 + 64 + 2r <= 128: a region row in one warp-wide 4-byte load
__device__ __forceinline__ int pk(int ox, int oy) { return (ox & 0xffff) | (oy << 16); }
__device__ __forceinline__ int pk_x(int v) { return static_cast<int16_t>(v & 0xffff); }
__device__ __forceinline__ int pk_y(int v) { return v >> 16; }

template <bool kBorder>
__device__ __forceinline__ int chamfer_packed(const int* __restrict__ cur, int rw, int c, int gx, int gy, int width,
                                              int height) {
  const int self = cur[c];
  int out = self;
  int best = self == kNoneP ? 0x7fffffff : sq(pk_x(self)) + sq(pk_y(self));
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      if (dx == 0 && dy == 0) continue;
      if (kBorder) {
        const int nx = gx + dx, ny = gy + dy;
        if (nx < 0 || nx >= width || ny < 0 || ny >= height) continue;
      }
      const int n = cur[c + dy * rw + dx];
      if (n == kNoneP) continue;
      const int cxo = dx + pk_x(n), cyo = dy + pk_y(n);
      const int d = sq(cxo) + sq(cyo);
      if (d < best) {
        best = d;
        out = pk(cxo, cyo);
      }
    }
  }
  return out;
}

__host__ __device__ constexpr int sparse_words(int radius) { return (kTW + 2 * radius + 31) / 32; }
static size_t sparse_smem(int radius) {
  const int rw = kTW + 2 * radius, rh = kTH + 2 * radius, cells = rw * rh, nw = sparse_words(radius);
  return sizeof(int) * (3 * static_cast<size_t>(cells) + 4 * static_cast<size_t>(rh) * nw + rh + 32);
}

struct SparseTile {
  const int* cur = nullptr;       // final packed source offsets per region cell
  const uint32_t* list = nullptr; // candidate cells, (cy << 16) | cx
  int n = 0;
};

// The region of the 64x16 tile blockIdx.x (as chamfer_tile) with the sparse
// passes. Returns false when the tile has nothing to propagate.
__device__ __forceinline__ bool sparse_tile(int width, int height, const uint8_t* __restrict__ valid, int in_row0,
                                            int in_rows, int radius, int out_row0, int out_rows, int* sm,
                                            SparseTile& st) {
  const int rw = kTW + 2 * radius, rh = kTH + 2 * radius, cells = rw * rh, nw = sparse_words(radius);
  int* cur = sm;
  int* nxt = sm + cells;
  uint32_t* list = reinterpret_cast<uint32_t*>(sm + 2 * cells);
  uint32_t* vw = reinterpret_cast<uint32_t*>(sm + 3 * cells);  // [rh][nw] valid bits
  uint32_t* iw = vw + rh * nw;                                 // in-image bits
  uint32_t* hw = iw + rh * nw;                                 // horizontally dilated valid bits
  uint32_t* cw = hw + rh * nw;                                 // candidate bits
  int* rowoff = reinterpret_cast<int*>(cw + rh * nw);          // [rh + 1]
  const int tiles_x = (width + kTW - 1) / kTW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x0 = tx * kTW - radius, y0 = out_row0 + ty * kTH - radius;
  const int in_end = in_row0 + in_rows, out_end = out_row0 + out_rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // valid / in-image bit rows of the region (cell lx of row ly = bit lx % 32
  // of word lx / 32); the chamfer state is initialised only for work tiles
  int any_valid = 0, any_hole = 0;
  if (radius <= kWordLoadMaxR) {
    // 4 mask bytes per lane: lane k holds cells xa + 4k .. xa + 4k + 3 of the
    // row (xa = x0 rounded down to 4), one warp-wide load per region row
    const int xa = x0 & ~3, sh = x0 - xa;
    for (int ly = warp; ly < rh; ly += nwarps) {
      const int gy = y0 + ly;
      const bool rowok = gy >= in_row0 && gy < in_end && gy >= 0 && gy < height;
      uint32_t word = 0;
      const int gx = xa + 4 * lane;
      if (rowok && gx < x0 + rw && gx + 4 > x0) {
        const uint8_t* rp = valid + static_cast<int64_t>(gy - in_row0) * width;
        if (gx >= 0 && gx + 4 <= width && (reinterpret_cast<uintptr_t>(rp + gx) & 3) == 0) {
          word = __ldg(reinterpret_cast<const uint32_t*>(rp + gx));
        } else {
          for (int b = 0; b < 4; ++b) {
            const int x = gx + b;
            if (x >= 0 && x < width && rp[x]) word |= 0xffu << (8 * b);
          }
        }
      }
      const unsigned b0 = __ballot_sync(0xffffffffu, word & 0xffu), b1 = __ballot_sync(0xffffffffu, word & 0xff00u),
                     b2 = __ballot_sync(0xffffffffu, word & 0xff0000u),
                     b3 = __ballot_sync(0xffffffffu, word & 0xff000000u);
      auto spread = [](uint32_t x) {  // bit k -> bit 4k (k < 8)
        x = (x | x << 12) & 0x000f000fu;
        x = (x | x << 6) & 0x03030303u;
        return (x | x << 3) & 0x11111111u;
      };
      auto rword = [&](int w) -> uint32_t {  // bits xa + 32w .. of the row
        if (w >= 4) return 0u;
        const int s8 = 8 * w;
        return spread(b0 >> s8 & 0xffu) | spread(b1 >> s8 & 0xffu) << 1 | spread(b2 >> s8 & 0xffu) << 2 |
               spread(b3 >> s8 & 0xffu) << 3;
      };
      if (lane < nw) {
        const int j = lane;
        uint32_t v = __funnelshift_r(rword(j), rword(j + 1), sh);
        // in-region / in-image columns of this word
        const int c0 = 32 * j, gx0 = x0 + c0;
        const int lo = max(0, -gx0), hi = min(32, min(width - gx0, rw - c0));
        uint32_t im = 0;
        if (gy >= 0 && gy < height && hi > lo) im = (hi - lo == 32 ? 0xffffffffu : ((1u << (hi - lo)) - 1u)) << lo;
        const int rl = min(32, rw - c0);
        const uint32_t inreg = rl >= 32 ? 0xffffffffu : (rl > 0 ? (1u << rl) - 1u : 0u);
        v &= inreg;
        vw[ly * nw + j] = v;
        iw[ly * nw + j] = im;
        any_valid |= v != 0;
        if (ly >= radius && ly < radius + kTH && gy < out_end) {
          // output columns: [radius, radius + kTW) of the region, inside the image
          const int olo = max(0, radius - c0), ohi = min(32, min(radius + kTW - c0, width - gx0));
          if (ohi > olo) {
            const uint32_t om = (ohi - olo == 32 ? 0xffffffffu : ((1u << (ohi - olo)) - 1u)) << olo;
            any_hole |= (~v & om) != 0;
          }
        }
      }
    }
  } else {
    for (int ly = warp; ly < rh; ly += nwarps)
      for (int j = 0; j < nw; ++j) {
        const int lx = 32 * j + lane, gx = x0 + lx, gy = y0 + ly;
        const bool inreg = lx < rw;
        const bool inimg = inreg && gx >= 0 && gx < width && gy >= 0 && gy < height;
        const bool v =
            inimg && gy >= in_row0 && gy < in_end && valid[static_cast<int64_t>(gy - in_row0) * width + gx];
        const unsigned vb = __ballot_sync(0xffffffffu, v), ib = __ballot_sync(0xffffffffu, inimg);
        if (lane == 0) {
          vw[ly * nw + j] = vb;
          iw[ly * nw + j] = ib;
        }
        any_valid |= v;
        any_hole |= inreg && !v && lx >= radius && lx < radius + kTW && ly >= radius && ly < radius + kTH &&
                    gx < width && gy < out_end;
      }
  }
  const bool work = __syncthreads_or(any_valid) && __syncthreads_or(any_hole);
  if (!work) return false;
  for (int ly = warp; ly < rh; ly += nwarps)
    for (int lx = lane; lx < rw; lx += 32) {
      const int c = ly * rw + lx;
      const int v = (vw[ly * nw + (lx >> 5)] >> (lx & 31) & 1u) ? 0 : kNoneP;
      cur[c] = v;
      nxt[c] = v;
    }
  // horizontal dilation by r: bit k of word j <- bits k-r .. k+r of the row
  for (int e = threadIdx.x; e < rh * nw; e += blockDim.x) {
    const int ly = e / nw, j = e - ly * nw;
    const uint32_t* row = vw + ly * nw;
    const uint32_t a = j > 0 ? row[j - 1] : 0u, b = row[j], c = j + 1 < nw ? row[j + 1] : 0u;
    uint32_t acc = b;
    for (int sh = 1; sh <= radius; ++sh) acc |= __funnelshift_r(b, c, sh) | __funnelshift_l(a, b, sh);
    hw[e] = acc;
  }
  __syncthreads();
  for (int ly = warp; ly < rh; ly += nwarps) {
    int cnt = 0;
    if (lane < nw) {
      uint32_t acc = 0;
      const int lo = max(0, ly - radius), hi = min(rh - 1, ly + radius);
      for (int y = lo; y <= hi; ++y) acc |= hw[y * nw + lane];
      acc &= ~vw[ly * nw + lane] & iw[ly * nw + lane];
      cw[ly * nw + lane] = acc;
      cnt = __popc(acc);
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (lane == 0) rowoff[ly + 1] = cnt;
  }
  __syncthreads();
  if (warp == 0) {  // inclusive scan of the row counts
    int carry = 0;
    for (int base = 0; base < rh; base += 32) {
      int v = base + lane < rh ? rowoff[base + lane + 1] : 0;
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += t;
      }
      if (base + lane < rh) rowoff[base + lane + 1] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) rowoff[0] = 0;
  }
  __syncthreads();
  for (int ly = warp; ly < rh; ly += nwarps) {
    int o = rowoff[ly];
    for (int j = 0; j < nw; ++j) {
      const uint32_t bits = cw[ly * nw + j];
      if (bits >> lane & 1u)
        list[o + __popc(bits & ((1u << lane) - 1u))] = (static_cast<uint32_t>(ly) << 16) | (32 * j + lane);
      o += __popc(bits);
    }
  }
  const int n = rowoff[rh];
  __syncthreads();
  const bool interior = x0 >= 0 && x0 + rw <= width && y0 >= 0 && y0 + rh <= height;
  for (int pass = 1; pass <= radius; ++pass) {
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const uint32_t le = list[e];
      const int cx = le & 0xffff, cy = le >> 16;
      if (cx < pass || cx >= rw - pass || cy < pass || cy >= rh - pass) continue;
      const int c = cy * rw + cx;
      nxt[c] = interior ? chamfer_packed<false>(cur, rw, c, x0 + cx, y0 + cy, width, height)
                        : chamfer_packed<true>(cur, rw, c, x0 + cx, y0 + cy, width, height);
    }
    __syncthreads();
    int* t = cur;
    cur = nxt;
    nxt = t;
  }
  st.cur = cur;
  st.list = list;
  st.n = n;
  return true;
}

// k_dilate_fused for radius <= 32: every tile is first copied (16-byte moves
// when aligned), then the listed output cells with a source are overwritten.
__global__ void __launch_bounds__(256) k_dilate_sparse(int width, int height, int channels,
                                                       const uint8_t* __restrict__ map_in,
                                                       const uint8_t* __restrict__ valid, int in_row0, int in_rows,
                                                       int radius, OutSet outs, int out_row0, int out_rows) {
  extern __shared__ int smi[];
  const int rw = kTW + 2 * radius;
  const int tiles_x = (width + kTW - 1) / kTW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int out_end = out_row0 + out_rows;
  SparseTile st;
  const bool work = sparse_tile(width, height, valid, in_row0, in_rows, radius, out_row0, out_rows, smi, st);
  const int gx0 = tx * kTW, gy0 = out_row0 + ty * kTH;
  const int64_t row_bytes = static_cast<int64_t>(width) * channels;
  bool copied = false;
  if (gx0 + kTW <= width && gy0 + kTH <= out_end) {
    const uint8_t* src0 = map_in + (static_cast<int64_t>(gy0 - in_row0) * width + gx0) * channels;
    const int64_t dst_off = (static_cast<int64_t>(gy0 - outs.row0) * width + gx0) * channels;
    const int vec_per_row = kTW * channels / 16;
    bool aligned = kTW * channels % 16 == 0 && row_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src0) & 15) == 0;
    for (int k = 0; k < outs.n; ++k) aligned = aligned && (reinterpret_cast<uintptr_t>(outs.p[k] + dst_off) & 15) == 0;
    if (aligned) {
      for (int c = threadIdx.x; c < vec_per_row * kTH; c += blockDim.x) {
        const int r = c / vec_per_row, k = c % vec_per_row;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src0 + r * row_bytes) + k);
        for (int o = 0; o < outs.n; ++o) reinterpret_cast<uint4*>(outs.p[o] + dst_off + r * row_bytes)[k] = v;
      }
      copied = true;
    }
  }
  if (!copied) {
    for (int c = threadIdx.x; c < kTW * kTH; c += blockDim.x) {
      const int lx = c % kTW, ly = c / kTW;
      const int gx = gx0 + lx, gy = gy0 + ly;
      if (gx >= width || gy >= out_end) continue;
      const uint8_t* src = map_in + (static_cast<int64_t>(gy - in_row0) * width + gx) * channels;
      const int64_t doff = (static_cast<int64_t>(gy - outs.row0) * width + gx) * channels;
      for (int o = 0; o < outs.n; ++o)
        for (int ch = 0; ch < channels; ++ch) outs.p[o][doff + ch] = src[ch];
    }
  }
  if (!work) return;
  __syncthreads();  // the fixups below overwrite copies made by other threads
  for (int e = threadIdx.x; e < st.n; e += blockDim.x) {
    const uint32_t le = st.list[e];
    const int cx = le & 0xffff, cy = le >> 16;
    const int lx = cx - radius, ly = cy - radius;
    if (lx < 0 || lx >= kTW || ly < 0 || ly >= kTH) continue;
    const int gx = gx0 + lx, gy = gy0 + ly;
    if (gx >= width || gy >= out_end) continue;
    const int v = st.cur[cy * rw + cx];
    if (v == kNoneP) continue;
    const uint8_t* src =
        map_in + (static_cast<int64_t>(gy + pk_y(v) - in_row0) * width + gx + pk_x(v)) * channels;
    const int64_t doff = (static_cast<int64_t>(gy - outs.row0) * width + gx) * channels;
    for (int o = 0; o < outs.n; ++o)
      for (int ch = 0; ch < channels; ++ch) outs.p[o][doff + ch] = src[ch];
  }
}

// Dilation resolved before the transfer (fused bake, full atlas): the sources
// depend only on the valid mask, so each gutter texel (invalid, with a source
// after r passes) is either given its final colour now - the source is a
// valid unreliable texel, whose raw colour is the constant (128,128,255) - or
// linked into its source query's list (dep_head[slot] -> dep_next[texel] ->
// ...), which the transfer's epilogue walks to store the query's colour into
// every texel that copies it. Valid texels carry bit 1 in `valid` when they
// are queries; qslot maps a query texel to its list slot.
__global__ void __launch_bounds__(256) k_dilate_links(int width, int height, const uint8_t* __restrict__ valid,
                                                      int radius, const int* __restrict__ qslot,
                                                      int* __restrict__ dep_head, int* __restrict__ dep_next,
                                                      uint8_t* __restrict__ rgb,
                                                      const uint8_t* __restrict__ tile_state, int fmt) {
  extern __shared__ int smi[];
  const int rw = kTW + 2 * radius;
  const int tiles_x = (width + kTW - 1) / kTW;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  if (tile_state && radius <= 16) {
    // the raster's 16x16 tile classes: skip output tiles whose four raster
    // tiles are all valid (no hole), or whose halo's raster tiles hold no
    // valid texel (nothing to propagate)
    __shared__ int skip;
    if (threadIdx.x == 0) {
      const int rtx = (width + 15) / 16, rty = (height + 15) / 16;
      bool full = true, empty = true;
      for (int y = ty - 1; y <= ty + 1; ++y)
        for (int x = 4 * tx - 1; x <= 4 * tx + 4; ++x) {
          if (y < 0 || y >= rty || x < 0 || x >= rtx) continue;
          const uint8_t st = tile_state[y * rtx + x];
          empty = empty && st == 0;
          if (y == ty && x >= 4 * tx && x < 4 * tx + 4) full = full && st == 2;
        }
      skip = full || empty;
    }
    __syncthreads();
    if (skip) return;
  }
  SparseTile st;
  if (!sparse_tile(width, height, valid, 0, height, radius, 0, height, smi, st)) return;
  for (int e = threadIdx.x; e < st.n; e += blockDim.x) {
    const uint32_t le = st.list[e];
    const int cx = le & 0xffff, cy = le >> 16;
    const int lx = cx - radius, ly = cy - radius;
    if (lx < 0 || lx >= kTW || ly < 0 || ly >= kTH) continue;
    const int gx = tx * kTW + lx, gy = ty * kTH + ly;
    if (gx >= width || gy >= height) continue;
    const int v = st.cur[cy * rw + cx];
    if (v == kNoneP) continue;
    const int64_t t = static_cast<int64_t>(gy) * width + gx;
    const int64_t src = static_cast<int64_t>(gy + pk_y(v)) * width + (gx + pk_x(v));
    if (valid[src] & 2) {
      const int slot = qslot[src];
      if (slot >= 0) dep_next[t] = atomicExch(&dep_head[slot], static_cast<int>(t));
    } else {
      px_store(rgb, t, fmt, px_neutral(fmt));
    }
  }
}

// ---- global multi-pass fallback (large radius) ----------------------------
__global__ void k_dilate_init(int width, int rows, const uint8_t* __restrict__ valid,
                              int32_t* __restrict__ sx, int32_t* __restrict__ sy,
                              long long* __restrict__ d2, int in_row0) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(width) * rows) return;
  const bool v = valid[i] != 0;
  sx[i] = v ? static_cast<int32_t>(i % width) : 0;
  sy[i] = v ? static_cast<int32_t>(i / width) + in_row0 : 0;
  d2[i] = v ? 0 : 0x7fffffffffffffffll;
}

__global__ void k_dilate_pass(int width, int height, int rows, int in_row0,
                              const int32_t* __restrict__ sx, const int32_t* __restrict__ sy,
                              const long long* __restrict__ d2, int32_t* __restrict__ nsx,
                              int32_t* __restrict__ nsy, long long* __restrict__ nd2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(width) * rows) return;
  const int x = static_cast<int>(i % width), ly = static_cast<int>(i / width), y = ly + in_row0;
  long long best = d2[i];
  int32_t bx = sx[i], by = sy[i];
  if (best != 0) {
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (dx == 0 && dy == 0) continue;
        const int nx = x + dx, ny = y + dy;
        if (nx < 0 || nx >= width || ny < 0 || ny >= height) continue;
        if (ny < in_row0 || ny >= in_row0 + rows) continue;
        const int64_t n = static_cast<int64_t>(ny - in_row0) * width + nx;
        if (d2[n] == 0x7fffffffffffffffll) continue;
        const long long ddx = x - sx[n], ddy = y - sy[n];
        const long long d = ddx * ddx + ddy * ddy;
        if (d < best) {
          best = d;
          bx = sx[n];
          by = sy[n];
        }
      }
  }
  nd2[i] = best;
  nsx[i] = bx;
  nsy[i] = by;
}

__global__ void k_dilate_copy(int width, int channels, const uint8_t* __restrict__ map_in,
                              const uint8_t* __restrict__ valid, int in_row0,
                              const int32_t* __restrict__ sx, const int32_t* __restrict__ sy,
                              const long long* __restrict__ d2, uint8_t* __restrict__ map_out,
                              int out_row0, int out_rows) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(width) * out_rows) return;
  const int x = static_cast<int>(i % width), y = static_cast<int>(i / width) + out_row0;
  const int64_t si = static_cast<int64_t>(y - in_row0) * width + x;
  int64_t src = si;
  if (!valid[si] && d2[si] != 0x7fffffffffffffffll)
    src = static_cast<int64_t>(sy[si] - in_row0) * width + sx[si];
  for (int c = 0; c < channels; ++c) map_out[i * channels + c] = map_in[src * channels + c];
}

}  // namespace

static size_t dilate_smem(int radius) {
  return static_cast<size_t>(4) * (kTW + 2 * radius) * (kTH + 2 * radius) * sizeof(int16_t);
}

bool dilate_links_supported(int radius) { return radius > 0 && radius <= kSparseMaxR; }

void dilate_links(Ctx& ctx, cudaStream_t s, int res, const uint8_t* valid, int radius, const int* qslot,
                  int* dep_head, int* dep_next, uint8_t* rgb, const uint8_t* tile_state, int fmt) {
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  MFB_CUDA_TRY(cudaGetDevice(&dev));
  if (!((attr_set.load(std::memory_order_acquire) >> (dev & 63)) & 1ull)) {
    MFB_CUDA_TRY(cudaFuncSetAttribute(k_dilate_links, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MFB_CUDA_TRY(cudaFuncSetAttribute(k_dilate_sparse, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set.fetch_or(1ull << (dev & 63), std::memory_order_acq_rel);
  }
  const int tiles = ((res + kTW - 1) / kTW) * ((res + kTH - 1) / kTH);
  k_dilate_links<<<tiles, 256, sparse_smem(radius), s>>>(res, res, valid, radius, qslot, dep_head, dep_next, rgb,
                                                            tile_state, fmt);
  ctx.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void dilate_seams_to(Ctx& ctx, cudaStream_t s, int width, int height, int channels, const uint8_t* map_in,
                     const uint8_t* valid, int in_row0, int in_rows, int radius, const OutSet& outs, int out_row0,
                     int out_rows) {
  if (out_rows <= 0 || width <= 0 || outs.n <= 0) return;
  const int64_t out_bytes = static_cast<int64_t>(width) * out_rows * channels;
  const int64_t dst_off = static_cast<int64_t>(out_row0 - outs.row0) * width * channels;
  if (radius == 0) {
    for (int k = 0; k < outs.n; ++k)
      MFB_CUDA_TRY(cudaMemcpyAsync(outs.p[k] + dst_off,
                                   map_in + static_cast<int64_t>(out_row0 - in_row0) * width * channels,
                                   out_bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  const size_t smem = dilate_smem(radius);
  if (radius <= 64 && smem <= 200 * 1024) {
    // the attribute is per device: one bit per device, set once each
    static std::atomic<unsigned long long> attr_set{0};
    int dev = 0;
    MFB_CUDA_TRY(cudaGetDevice(&dev));
    if (!((attr_set.load(std::memory_order_acquire) >> (dev & 63)) & 1ull)) {
      MFB_CUDA_TRY(cudaFuncSetAttribute(k_dilate_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
      MFB_CUDA_TRY(cudaFuncSetAttribute(k_dilate_sparse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        200 * 1024));
      attr_set.fetch_or(1ull << (dev & 63), std::memory_order_acq_rel);
    }
    const int tiles = ((width + kTW - 1) / kTW) * ((out_rows + kTH - 1) / kTH);
    // MFB_DILATE_SPARSE=0: dense passes over the whole region (A/B)
    static const bool sparse = [] {
      const char* e = std::getenv("MFB_DILATE_SPARSE");
      return !(e && e[0] == '0');
    }();
    if (sparse && radius <= kSparseMaxR)
      k_dilate_sparse<<<tiles, 256, sparse_smem(radius), s>>>(width, height, channels, map_in, valid, in_row0,
                                                              in_rows, radius, outs, out_row0, out_rows);
    else
      k_dilate_fused<<<tiles, 256, smem, s>>>(width, height, channels, map_in, valid, in_row0, in_rows,
                                              radius, outs, out_row0, out_rows);
    ctx.count_launch();
    MFB_CUDA_TRY(cudaGetLastError());
    return;
  }
  const int64_t n = static_cast<int64_t>(width) * in_rows;
  auto* sx = ctx.buf<int32_t>("dil.sx", n);
  auto* sy = ctx.buf<int32_t>("dil.sy", n);
  auto* d2 = ctx.buf<long long>("dil.d2", n);
  auto* nsx = ctx.buf<int32_t>("dil.nsx", n);
  auto* nsy = ctx.buf<int32_t>("dil.nsy", n);
  auto* nd2 = ctx.buf<long long>("dil.nd2", n);
  const int T = 256;
  k_dilate_init<<<div_up(n, T), T, 0, s>>>(width, in_rows, valid, sx, sy, d2, in_row0);
  for (int p = 0; p < radius; ++p) {
    k_dilate_pass<<<div_up(n, T), T, 0, s>>>(width, height, in_rows, in_row0, sx, sy, d2, nsx, nsy, nd2);
    std::swap(sx, nsx);
    std::swap(sy, nsy);
    std::swap(d2, nd2);
  }
  for (int k = 0; k < outs.n; ++k)
    k_dilate_copy<<<div_up(static_cast<int64_t>(width) * out_rows, T), T, 0, s>>>(
        width, channels, map_in, valid, in_row0, sx, sy, d2, outs.p[k] + dst_off, out_row0, out_rows);
  ctx.count_launch(radius + 1 + outs.n);
  MFB_CUDA_TRY(cudaGetLastError());
}

void dilate_seams(Ctx& ctx, cudaStream_t s, int width, int height, int channels,
                  const uint8_t* map_in, const uint8_t* valid, int in_row0, int in_rows,
                  int radius, uint8_t* map_out, int out_row0, int out_rows) {
  OutSet one;
  one.p[0] = map_out;
  one.n = 1;
  one.row0 = out_row0;
  dilate_seams_to(ctx, s, width, height, channels, map_in, valid, in_row0, in_rows, radius, one, out_row0,
                  out_rows);
}

}  // namespace mfb
