// bake.cuh — internal interfaces between the libmfbake translation units.
//
// HBM layout:
//   DevMesh   : the reference's arrays verbatim (f64 positions AoS, i32 faces,
//               optional f64 normals, f64 uv pool, i32 face_uvs).
//   GBufDev   : the reference G-buffer layout (gbuffer.h:17-30): four f32x3
//               AoS planes + two u8 planes, row-major, v down; a row slab
//               [row0, row0 + rows) of the full res x res atlas.
//   Lbvh      : 64-byte binary nodes with both child boxes stored in the
//               parent (fp32, rounded outward), child refs >= 0 = node,
//               < 0 = leaf range of <= kLeafMax Morton-ordered triangles;
//               80-byte triangle records (f64 vertices + face id) in leaf order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

struct mf_ctx;

namespace mfb {

// ---------------------------------------------------------------- context
class HostPool;  // host_pool.h

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;      // second stream: dense-mesh work overlaps the lowpoly work
  cudaStream_t aux = nullptr;       // third stream: lowpoly wedge frames overlap its reliability pass
  cudaStream_t side2 = nullptr;     // LBVH helper: triangle repack alongside the hierarchy emission
  cudaStream_t aux2 = nullptr;      // lowpoly reliability pass alongside the raster setup and binning
  cudaEvent_t setup_done = nullptr, join4 = nullptr;
  cudaStream_t lowhi = nullptr;     // the bake's lowpoly branch, high priority (the main stream is the caller's)
  cudaStream_t dn = nullptr;        // dense vertex normals (needed only by the transfer's encode), low priority
  cudaEvent_t lowfork = nullptr, lowjoin = nullptr;
  cudaEvent_t lfork = nullptr, ljoin = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, fork2 = nullptr, join2 = nullptr, join3 = nullptr;
  cudaEvent_t hi_ready = nullptr;   // host entry point: dense mesh uploaded and validated
  cudaEvent_t dfork = nullptr, djoin = nullptr;  // host entry point: dense phase side -> aux -> side
  cudaEvent_t up_fork = nullptr, up_join = nullptr;  // split H2D of one mesh over two streams
  // staged (pageable) dense upload: the host pool's chunk DMAs go to these two
  // streams, which no captured bake graph touches (a capture of the lowpoly
  // branch runs while the pool is still enqueueing)
  cudaStream_t up1 = nullptr, up2 = nullptr;
  cudaEvent_t up1_done = nullptr, up2_done = nullptr;
  bool timing = false;
  bool capturing = false;  // a graph capture of this context's streams is open
  int64_t launches = 0;
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::unordered_map<std::string, Buf> scratch;
  std::unordered_map<std::string, Buf> pinned;
  // CUB temp storage, one slot per stream (main, side, aux, aux2, side2): concurrent
  // branches of the bake must not share it
  void* cub_tmp[7] = {};  // main, side, aux, aux2, side2, lowhi, dn
  size_t cub_tmp_bytes[7] = {};
  int64_t bin_capacity = 0;         // raster tile-bin capacity hint (grows on overflow)
  int fmt = MF_ATLAS_RGB8;          // atlas encoding of the fused bake in progress (MF_ATLAS_*)

  // Grow-only named device scratch (never shrinks; freed with the context).
  void* buf(const std::string& name, size_t bytes);
  template <typename T>
  T* buf(const std::string& name, size_t count) {
    return static_cast<T*>(buf(name, count * sizeof(T) + 16));
  }
  void* host_buf(const std::string& name, size_t bytes);
  void* cub_temp(size_t bytes, cudaStream_t s);
  void sync_all();  // drain every stream of the context
  void count_launch(int n = 1) { launches += n; }
  // Byte fill as a kernel (capi.cu). Inside the bake's captured graphs
  // memset nodes run on the copy engine one after another, each a few us
  // apart, and delayed the lowpoly branch's start by ~35 us (r02 CUPTI
  // timeline); a fill kernel runs beside the other branches' kernels.
  void fill(void* p, int value, size_t bytes, cudaStream_t s);

  // Every scratch (re)allocation bumps the generation: a captured CUDA graph
  // is replayed only while the buffers it references are unchanged.
  uint64_t alloc_gen = 0;
  // Persistent timing events (graph-capturable: never destroyed mid-flight).
  std::vector<cudaEvent_t> ev_pool;
  int wait_value_probe = 0;  // cuStreamWaitValue32 on this device: 0 untested, 1 usable, -1 not
  cudaEvent_t pool_event(int i);
  // Captured fused bake (see capi.cu bake_dev).
  cudaGraphExec_t bake_exec = nullptr;
  std::vector<char> bake_key, bake_prev_key;
  uint64_t bake_gen = 0, bake_prev_gen = ~0ull;
  // Captured phases of the host-buffer bake (capi.cu bake_host_overlapped):
  // the first call with a key runs eagerly, the second captures, later ones
  // replay while no scratch buffer was reallocated.
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    std::vector<char> key, prev_key;
    uint64_t gen = 0, prev_gen = ~0ull;
  };
  GraphSlot g_low, g_dense;
  void invalidate_graphs();  // drop every captured graph and capture key
  // host worker threads staging pageable caller buffers (created on first use)
  HostPool* pool = nullptr;
  HostPool& host_pool();
  ~Ctx();
};

// ---------------------------------------------------------------- meshes
struct DevMesh {
  const double* pos = nullptr;   // V x 3
  const int32_t* faces = nullptr;  // F x 3
  const double* nrm = nullptr;   // V x 3 or null
  const double* uvs = nullptr;   // U x 2 or null
  const int32_t* fuv = nullptr;  // F x 3 or null
  int nv = 0, nf = 0, nu = 0;
  bool has_normals() const { return nrm != nullptr && nv > 0; }
  bool has_uvs() const { return fuv != nullptr && uvs != nullptr && nu > 0; }
};

// ---------------------------------------------------------------- G-buffer
struct GBufDev {
  int res = 0;
  int row0 = 0, rows = 0;  // stored slab of atlas rows
  float* pos = nullptr;    // rows*res*3
  float* nrm = nullptr;
  float* tan = nullptr;
  float* bit = nullptr;
  uint8_t* valid = nullptr;  // rows*res
  uint8_t* rel = nullptr;
  int64_t texels() const { return static_cast<int64_t>(rows) * res; }
};

// ---------------------------------------------------------------- LBVH
constexpr int kLeafMax = 4;     // reference leaf size (bvh.cpp:13)
// LBVH leaf-range cap used by default: results do not depend on the tree, and
// 3 measured ~3% faster than 4 in the config-B walk (2: -2.5%, 4: 0, BVH4: +3%).
constexpr int kLeafMaxDefault = 3;
constexpr int kMaxFaces = 1 << 27;  // leaf refs encode first < 2^27 (leaf_ref)
// Traversal stacks (one entry per level at most). Karras emission over
// (30-bit Morton, index) keys: along a root-to-leaf path the split deltas
// strictly increase, and they range over the 30 Morton bits plus the
// ceil(log2 F) <= 27 index bits, so depth <= 30 + 27 + 1 (lbvh_layout rejects
// F >= kMaxFaces).
constexpr int kStackMax = 64;
static_assert(kStackMax >= 30 + 27 + 1, "traversal stack must cover the deepest Karras tree");

// Child boxes interleaved per coordinate, (left, right) pairs: each pair is
// one f32x2 register pair after the node load, so the transfer walk bounds
// both children with packed FADD2.RM / FFMA2.RM (query.cu box_lb2).
struct alignas(16) BNode {
  float4 a;  // L.min.x R.min.x L.min.y R.min.y
  float4 b;  // L.min.z R.min.z L.max.x R.max.x
  float4 c;  // L.max.y R.max.y L.max.z R.max.z
  int4 d;    // left ref, right ref, range first, range count
};
// float index of coordinate k (0..2 min xyz, 3..5 max xyz) of child `side`
__host__ __device__ __forceinline__ int bnode_coord(int side, int k) { return 2 * k + side; }
static_assert(sizeof(BNode) == 64, "node must be one 64-byte line segment");

struct alignas(16) BTri {
  double v[9];  // the reference's f64 vertices, gathered in leaf order
  int32_t face;
  int32_t pad;
};
static_assert(sizeof(BTri) == 80, "triangle record is 5 x 16 B");

// Per-triangle fp32 box (rounded outward), leaf order: mn.xyz mx.x | mx.yz pad pad.
struct alignas(16) TBox {
  float4 a, b;
};

// Leaf range reference: ~(first << 4 | count), count <= kLeafCountMax
// (first < 2^27 triangles).
constexpr int kLeafCountMax = 15;
__host__ __device__ __forceinline__ int32_t leaf_ref(int first, int count) {
  return ~((first << 4) | count);
}
__host__ __device__ __forceinline__ void leaf_decode(int32_t ref, int& first, int& count) {
  const int32_t r = ~ref;
  first = r >> 4;
  count = r & 15;
}


// Per-triangle fp32 containment planes, leaf order (built only for wide
// leaves, Lbvh::tplane): a unit normal n with the slab lo <= n.x <= hi and,
// per edge, an in-plane outward unit vector m with the half-space m.x <= o,
// every one holding all three vertices (bounds evaluated in f64 from the
// rounded fp32 n / m, then rounded outward). Hence for any point q
// dist(q, T)^2 >= max(0, lo - n.q, n.q - hi)^2 + max(0, max_e m_e.q - o_e)^2
// up to the fp32 evaluation error and the rounded vectors' 1e-7 departure from
// unit length / orthogonality, both covered by the caller's slack.
constexpr int kPlaneLeafMin = 4;  // leaf caps from which the pre-test is built
// internal nodes up to this many triangles get an LPlane (config E per bake:
// caps 64 / 128 / 256 / 1024 / 4096 / 16384 measured 34.8 / 32.1 / 30.6 /
// 29.3 / 29.4 / 30.2 ms - the build is O(F log cap), the walk gains flatten)
constexpr int kNodePlaneMax = 1024;
struct alignas(16) TPlane {
  float4 m0, m1, m2;  // (m_e, o_e)
  float4 n;           // (n, lo)
  float4 hi;          // (hi, -, -, -)
};

// Per-leaf oriented box (built with TPlane): an orthonormal fp32 frame (n the
// leaf's area-weighted normal, u in its plane, v = n x u) with the ranges
// [lo, hi], [umin, umax], [vmin, vmax] that hold every vertex of the leaf's
// triangles (f64 from the rounded directions, rounded outward). Indexed by
// the leaf's first triangle. dist(q, leaf)^2 >= the sum of the three squared
// range excesses, less the same slack as TPlane: a leaf whose bound already
// fails is skipped without touching its triangles.
struct alignas(32) LPlane {
  float n[3], lo, hi, u[3];
  float umin, umax, v[3], vmin, vmax, pad;
};
static_assert(sizeof(LPlane) == 64, "leaf record is two 32-byte loads");

struct Lbvh {
  TPlane* tplane = nullptr;  // device, leaf order, or null (see TPlane)
  LPlane* lplane = nullptr;  // device, by leaf first triangle, or null (see LPlane)
  // the same oriented box per internal node whose range holds at most
  // kNodePlaneMax triangles (a zero record, which never prunes, above that)
  LPlane* nplane = nullptr;
  int n_tris = 0;
  int n_nodes = 0;          // internal nodes (n_tris - 1), root = node 0 when n_tris > 1
  BNode* nodes = nullptr;   // device
  BTri* tris = nullptr;     // device, leaf order
  TBox* tbox = nullptr;     // device, leaf order
  int32_t root_ref = 0;     // 0 (internal root) or a leaf ref when n_tris <= kLeafMax... see build
  int leaf_max = kLeafMaxDefault;  // leaf-range cap the build used
  float root_box[6];        // host copy not needed for traversal; kept for export
  float* root_box_dev = nullptr;
  // [min c, max c, max |coord|] as ordered-int doubles (device); the
  // traversal derives its f64 error slack from max |coord|.
  const unsigned long long* scene_acc = nullptr;
};

// Build into buffers owned by `owner` scratch names prefixed with `tag`.
// leaf_hint: leaf-range size cap (0 = kLeafMaxDefault); MFB_LEAF_MAX overrides.
// vflags (nullable, device): the mesh was uploaded without its validation
// pass; the build checks validateMesh's conditions itself (bit 0 non-finite
// coordinate, bit 1 face index out of range; bad indices zeroed in place).
void lbvh_build(Ctx& ctx, cudaStream_t s, const DevMesh& m, Lbvh& out, const std::string& tag, int leaf_hint = 0,
                int* vflags = nullptr);
// The descriptor lbvh_build fills (device buffers by scratch name), without
// launching anything: used when a captured build is replayed.
void lbvh_layout(Ctx& ctx, const DevMesh& m, Lbvh& out, const std::string& tag, int leaf_hint = 0);
int lbvh_leaf_max(int leaf_hint);

// ---------------------------------------------------------------- lowpoly prep + raster
// computeVertexNormals (mesh.cpp:24-35) followed, when `renorm`, by the
// 1e-20 re-normalisation of tangent.cpp:26-31 / gbuffer.cpp:201-206. If the
// mesh carries normals, they are copied and re-normalised instead.
void vertex_normals(Ctx& ctx, cudaStream_t s, const DevMesh& m, double* out, bool renorm,
                    const std::string& tag);

// Everything rasterizeGBuffer needs before the texel loop: wedge frames
// (tangent.cpp:22-82), reliable flags (gbuffer.cpp:31-83) and per-face
// raster setup. Returns the device pointer of the face-setup array.
struct RasterPlan {
  void* faces = nullptr;   // RasterFace[nf]
  void* attrs = nullptr;   // AttrFace[nf]
  int nf = 0;
  int res = 0;
  cudaEvent_t pending[2] = {nullptr, nullptr};  // side branches raster_gbuffer joins before the texel kernel
  // set by the cooperative prep, which also bins the faces into tiles
  bool binned = false;
  const int* tile_start = nullptr;
  const int* bins = nullptr;
  int capacity = 0;
};
// Wedge frames + reliable flags run as ONE cooperative kernel
// (k_lowpoly_prep) on the aux stream (MFB_COOP_PREP=0: separate kernels on
// aux / aux2); the UV setup and, with `bin` (the rows raster_gbuffer will
// cover, its flags and the counters it would reset), the tile binning run
// on `s`. raster_gbuffer joins the side branch before the interpolation
// (split raster) or before the texel kernel.
#ifndef MFB_COOP_PREP
#define MFB_COOP_PREP 1
#endif
struct PrepBinning {
  int row0 = 0, rows = 0;
  int* flags = nullptr;           // raster flags: [1] bin overflow, [2] bin total
  int* zero4 = nullptr;           // fused query-list counters to reset, or null
  int64_t* row_counts = nullptr;  // per-row valid counts to reset (mf_coverage_rows), or null
};
void prepare_lowpoly(Ctx& ctx, cudaStream_t s, const DevMesh& lo, int res, RasterPlan& plan,
                     const PrepBinning* bin = nullptr);
// Frames only (for mf_wedge_tangents): F x 3 x {T, B, N} x 3 doubles.
void wedge_frames(Ctx& ctx, cudaStream_t s, const DevMesh& lo, double* frames_out);

// Compacted closest-point queries (valid and reliable texels), in 8x4 texel
// blocks so each warp's 32 queries are spatial neighbours.
struct QueryList {
  float4* qpos = nullptr;  // x, y, z (the G-buffer's f32 position), w = slab texel index (int bits)
  float* qtbn = nullptr;   // 9 floats per query: tangent, bitangent, normal (f32, as stored)
  int* count = nullptr;    // device counters: [0] queries, [3] the transfer's batch cursor (reset by the producer)
  int capacity = 0;
};

// Fused-bake raster outputs: instead of the full G-buffer, the raster writes
// the valid mask (g.valid), the raw map for every non-query texel
// (background (128,128,128) / unreliable (128,128,255), gbuffer.cpp:212-227)
// and the query records; debug planes get -1/-2 for invalid/unreliable.
struct RasterFused {
  uint8_t* rgb = nullptr;
  int fmt = MF_ATLAS_RGB8;  // atlas encoding of rgb (MF_ATLAS_*)
  QueryList q;
  int32_t* dbg_face = nullptr;
  double* dbg_ts = nullptr;
  unsigned long long* valid_count = nullptr;  // N_v accumulator (optional)
  int2* pend = nullptr;  // split raster: (slab texel, face) per query, interpolated by k_interp
  // dilation resolved before the transfer (dilate_links): with qslot set, the
  // split raster marks query texels with bit 1 of the valid byte, records
  // their list slot in qslot (slab texel -> slot) and resets dep_head[slot]
  int* qslot = nullptr;
  int* dep_head = nullptr;
  // row-band completion (BandSync): queries per band of band_rows slab rows
  int* band_tot = nullptr;
  int band_rows = 0;
  cudaEvent_t cover_done = nullptr;  // recorded after the coverage/compaction kernel (split raster)
  uint8_t* tile_state = nullptr;  // per 16x16 raster tile: 0 no valid texel, 1 mixed, 2 all valid
};
// True when raster_gbuffer fills RasterFused::qslot / dep_head (split raster,
// single-pass query list).
bool raster_links_supported();

// Tile-binned rasteriser over rows [g.row0, g.row0 + g.rows). Device flags:
// flags[0] = 1 when a texel is claimed twice (AtlasOverlap); flags[1] = 1
// when the tile bins overflowed (re-run after setting ctx.bin_capacity to
// flags[2], the exact bin total). Never synchronises. With `fused` the
// G-buffer planes other than `valid` are not written (see RasterFused).
void raster_gbuffer(Ctx& ctx, cudaStream_t s, const DevMesh& lo, const RasterPlan& plan,
                    GBufDev& g, int* flags_dev, int64_t* row_counts_dev,
                    const RasterFused* fused = nullptr);

// Builds the query list (and the raw map / debug codes of non-query texels)
// from a full G-buffer slab (the mf_transfer_normals entry point).
void gbuffer_queries(Ctx& ctx, cudaStream_t s, const GBufDev& g, const RasterFused& out);

// ---------------------------------------------------------------- queries
// Row-band completion of the fused bake's atlas, for a download that overlaps
// the transfer (host-buffer entry point): the raster counts each band's
// queries (tot), the transfer's warps count finished ones (done); a band's
// rows are final once it and its neighbours are done (dilation sources lie
// within radius <= rows rows), and the warp that completes the last of them
// sets ready[band] = 1, which a copy stream waits on (cuStreamWaitValue32).
struct BandSync {
  int* tot = nullptr;    // [nb] queries per band (raster)
  int* done = nullptr;   // [nb] finished queries per band (transfer)
  int* nbr = nullptr;    // [nb] completed bands among {b-1, b, b+1}
  int* ready = nullptr;  // [nb] 1 once band b's rows are final
  int rows = 0, nb = 0, res = 0;
};
constexpr int kMaxBands = 64;
// Completes bands with no query (one CTA, after the raster).
void band_init(Ctx& ctx, cudaStream_t s, const BandSync& bs);

struct TransferArgs {
  QueryList q;
  int res = 0;
  int slab_row0 = 0;                // absolute atlas row of slab row 0
  const double* hi_positions = nullptr;
  const double* hi_normals = nullptr;
  const int32_t* hi_faces = nullptr;
  double max_dist = 0.0;
  uint8_t* rgb = nullptr;           // raw map slab (indexed by the query's slab texel)
  int fmt = MF_ATLAS_RGB8;          // its encoding (MF_ATLAS_*)
  int32_t* dbg_face = nullptr;
  double* dbg_ts = nullptr;
  unsigned long long* counters = nullptr;  // [queries, hits]
  // dilation links (dilate_links): the epilogue also stores each query's
  // colour into every texel of its list dep_head[slot] -> dep_next[texel]
  const int* dep_head = nullptr;
  const int* dep_next = nullptr;
  BandSync bands;  // optional (bands.done != nullptr)
};
void transfer_normals(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const TransferArgs& a);

void closest_within(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* q, int64_t n,
                    double max_dist, int32_t* face, double* dist_sq, double* point, double* bary);
// sampleSdf (signfield/watertight.cpp:29-38) for n points: unbounded closest
// distance through the LBVH, sign from the trilinear signed field.
void sample_sdf(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* pts, int64_t n, int res,
                const double origin[3], double voxel, const float* field, double* out);
// bounds(mesh) (core/mesh.cpp:12-16) into out6 = min xyz, max xyz (synchronises).
void vertex_bounds(Ctx& ctx, cudaStream_t s, const DevMesh& m, double* out6);
// markSurfaceBand's voxel sweep (signfield/sign_grid.cpp:56-66) over a res^3 grid.
void surface_band(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, int res, const double origin[3], double h,
                  double truncation, double band_world, uint8_t* labels, float* dist);
// Ortho pixel-ray views (renderView, render/raster.cpp:12-102): cams7 = per
// view direction xyz, up xyz, halfExtent. Optional outputs: per-face won-pixel
// counters (castVisibility), per-view face / depth / position / normal images.
void render_views(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* cams7, int nviews, int res, int cull,
                  unsigned long long* hits, int32_t* face_img, float* depth_img, float* pos_img, float* nrm_img,
                  const int32_t* faces, const double* vnormals);
// castVisibility's counts by the reference's own face-order rasteriser on the
// device (z-buffer of atomicMax keys), views in z-buffer-sized passes.
void raster_visibility(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* cams7, int nviews, int res,
                       unsigned long long* hits);
// fibonacciCameras (render/camera.cpp:38-55) into cams7 (host).
void fibonacci_cameras(int count, double half_extent, double* cams7);
// out = positions - center; returns max |out| (synchronises).
double center_mesh(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double center[3], double* out);
void raycast_first(Ctx& ctx, cudaStream_t s, const Lbvh& bvh, const double* o, const double* d,
                   int64_t n, double tmin, double tmax, int32_t* face, double* t, double* u,
                   double* v);
void closest_brute(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* q, int64_t n, int32_t* face,
                   double* dist_sq, double* point, double* bary);
void raycast_brute(Ctx& ctx, cudaStream_t s, const DevMesh& m, const double* o, const double* d, int64_t n,
                   double tmin, double tmax, int32_t* face, double* t, double* u, double* v);

// ---------------------------------------------------------------- dilation
// Destinations of the dilation's output rows: buffer k holds image rows from
// row0 on. With several buffers every output row is stored into each - the
// sharded bake's atlas all-gather done by the producing kernel itself over
// peer (NVLink) memory (mf_bake_normal_map_dev_publish).
constexpr int kMaxPublish = 8;
struct OutSet {
  uint8_t* p[kMaxPublish] = {};
  int n = 0;
  int row0 = 0;
};
void dilate_seams_to(Ctx& ctx, cudaStream_t s, int width, int height, int channels, const uint8_t* map_in,
                     const uint8_t* valid, int in_row0, int in_rows, int radius, const OutSet& outs, int out_row0,
                     int out_rows);
// dilateSeams over a slab: input map rows [in_row0, in_row0 + in_rows) of a
// width x height x channels image with the matching valid slab; outputs rows
// [out_row0, out_row0 + out_rows) (which must lie `radius` rows inside the
// input slab unless at the image border).
// Dilation resolved before the transfer over a full res x res atlas (see
// k_dilate_links): gutter texels whose source is a valid unreliable texel get
// their colour in `rgb` now, the others are linked to their source query.
bool dilate_links_supported(int radius);
void dilate_links(Ctx& ctx, cudaStream_t s, int res, const uint8_t* valid, int radius, const int* qslot,
                  int* dep_head, int* dep_next, uint8_t* rgb, const uint8_t* tile_state = nullptr,
                  int fmt = MF_ATLAS_RGB8);
void dilate_seams(Ctx& ctx, cudaStream_t s, int width, int height, int channels,
                  const uint8_t* map_in, const uint8_t* valid, int in_row0, int in_rows,
                  int radius, uint8_t* map_out, int out_row0, int out_rows);

// ---------------------------------------------------------------- sort / scan (sort.cu)
// Stable LSD sort of 30-bit Morton keys + face ids in three 10-bit onesweep
// passes. hist: the 3 x 1024 digit histograms of the keys (built by the
// Morton kernel); status: sort_status_words(n) words zeroed before the sort;
// counters: 3 tile counters zeroed before the sort. Result in keys_alt /
// vals_alt.
struct SortArgs {
  uint32_t *keys = nullptr, *vals = nullptr, *keys_alt = nullptr, *vals_alt = nullptr;
  int n = 0;
  const int* hist = nullptr;
  uint32_t* status = nullptr;
  int* counters = nullptr;
};
int64_t sort_status_words(int n);
void radix_sort_morton30(Ctx& ctx, cudaStream_t s, const SortArgs& a);
// Exclusive prefix sum of n int32 (single pass, decoupled look-back).
void scan_exclusive(Ctx& ctx, cudaStream_t s, const int* in, int* out, int n, const std::string& tag);

// ---------------------------------------------------------------- texfuse
// Device-resident consumers of the G-buffer: proj/src/texfuse/fuse.cpp and
// mips.cpp (texfuse.cu). Images are row-major interleaved f32 (ImageF).
constexpr int kTfMaxMips = 24;
struct TfCamera {  // OrthoCamera (render/camera.h:12-38) with right() precomputed
  double dir[3], up[3], right[3], he;
  int res;
};
TfCamera tf_camera(const double* cam7, int res);
// buildMips' level sizes (mips.cpp:104-110): returns the chain length;
// lw/lh/off need kTfMaxMips + 1 entries; off[n] = total floats.
int tf_mip_layout(int w, int h, int c, int levels, int* lw, int* lh, int64_t* off);
void tf_edge_mask(Ctx& ctx, cudaStream_t s, int w, int h, const float* pos, const int32_t* face, double limit2,
                  uint8_t* mask);
int tf_build_mips(Ctx& ctx, cudaStream_t s, int w, int h, int c, const float* base, int levels, float sharpen,
                  float* chain, const std::string& tag);
void tf_valid_bounds(Ctx& ctx, cudaStream_t s, int64_t n, const float* pos, const uint8_t* valid, unsigned* b6);
void tf_backproject(Ctx& ctx, cudaStream_t s, int gres, const float* pos, const uint8_t* valid, const unsigned* b6,
                    const TfCamera& cam, int channels, int n_mips, const float* chain, const uint8_t* mask,
                    float* color, uint8_t* sampled);
void tf_incidence(Ctx& ctx, cudaStream_t s, int gres, const float* pos, const float* nrm, const uint8_t* valid,
                  const TfCamera& cam, const float* depth, double tolerance, float* out);
void tf_blend(Ctx& ctx, cudaStream_t s, int k, int64_t n, int c, const float* colors, const uint8_t* sampled,
              const float* inc, const double* priors_host, double alpha, double epsilon, float* out,
              uint8_t* filled);

}  // namespace mfb
