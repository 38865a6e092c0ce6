/*
 * mfbake.h — C ABI of the B200 normal-bake library (libmfbake.so).
 *
 * This is the drop-in boundary for the reference's bake hot path
 * (meshforge, /root/reference/proj). Every entry point below replaces one
 * reference interface; the file:line it replaces is cited next to it. The
 * C++ API in include/meshforge/ (source-compatible with the reference's
 * proj/include/meshforge) is implemented on top of these calls, and the
 * Python bindings (paper_2605_26137_b200/capi.py) bind them with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross the ABI, and
 *     no exception ever does.
 *   - Return value: 0 on success; 1 + (meshforge ErrorCode) for the
 *     reference's own errors (proj/include/meshforge/core/error.h:8-21), so
 *     MF_ERR(EmptyMesh) == 1 ...; negative values for device/runtime failures.
 *     mf_last_error() returns a thread-local message for the last failure.
 *   - Host buffers are caller-owned and laid out exactly as the reference's
 *     std::vector<Eigen::...>::data(): Vector3d = 3 x f64, Vector3f = 3 x f32,
 *     Vector3i = 3 x i32, Vector2d = 2 x f64, ImageU8 = row-major interleaved.
 *   - Device memory is owned by an mf_ctx (one CUDA stream) or by handles
 *     created from it. One context is single-threaded; distinct contexts may
 *     be driven from distinct threads concurrently.
 *   - "_dev" entry points take device pointers (inputs already resident in
 *     HBM); everything else takes host pointers and performs the copies.
 */
#ifndef MFBAKE_H_
#define MFBAKE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MF_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------- */
/* Reference error codes, offset by one (error.h:8-21 enum order). */
enum {
  MF_OK = 0,
  MF_ERR_EMPTY_MESH = 1,        /* ErrorCode::EmptyMesh */
  MF_ERR_INVALID_GEOMETRY = 2,  /* ErrorCode::InvalidGeometry */
  MF_ERR_OUT_OF_BOUNDS = 3,
  MF_ERR_EMPTY_SURFACE = 4,
  MF_ERR_ALL_HIDDEN = 5,
  MF_ERR_CHART_FAILURE = 6,
  MF_ERR_PACK_OVERFLOW = 7,
  MF_ERR_ATLAS_OVERLAP = 8,     /* ErrorCode::AtlasOverlap */
  MF_ERR_SHAPE_MISMATCH = 9,    /* ErrorCode::ShapeMismatch */
  MF_ERR_NOTHING_TO_INPAINT = 10,
  MF_ERR_EXPORT_MISMATCH = 11,
  MF_ERR_INVALID_CONFIG = 12,   /* ErrorCode::InvalidConfig */
  MF_ERR_IO = 13,               /* ErrorCode::IoError */
  /* Runtime failures (no reference equivalent; the C++ wrapper maps them to
   * Error(IoError, ...), a non-validation error, CLI exit code 3). */
  MF_ERR_CUDA = -1,
  MF_ERR_OUT_OF_MEMORY = -2,
  MF_ERR_BAD_ARGUMENT = -3,
  MF_ERR_NO_DEVICE = -4
};

/* ---- mesh view ---------------------------------------------------------- */
/* Non-owning view of meshforge::TriangleMesh (core/mesh.h:15-26).
 * hasNormals() == (normals != NULL && n_vertices > 0);
 * hasUvs()     == (face_uvs != NULL && n_uvs > 0). */
typedef struct mf_mesh_view {
  const double* positions;  /* n_vertices x 3 */
  int32_t n_vertices;
  const int32_t* faces;     /* n_faces x 3 */
  int32_t n_faces;
  const double* normals;    /* nullable, n_vertices x 3 */
  const double* uvs;        /* nullable, n_uvs x 2 */
  int32_t n_uvs;
  const int32_t* face_uvs;  /* nullable, n_faces x 3 */
} mf_mesh_view;

/* Per-call measurements filled by the bake entry points (all optional). */
typedef struct mf_bake_stats {
  int64_t valid_texels;   /* N_v: texels whose centre lies in a UV triangle */
  int64_t queries;        /* N_q: valid and reliable texels (closest-point queries) */
  int64_t hits;           /* queries that found a surface within maxDist */
  int32_t bvh_nodes;      /* internal LBVH nodes of the dense tree (F - 1, binary Karras tree) */
  int32_t bvh_depth;      /* 0: the bake does not measure it (mf_bvh_info reports a tree's depth) */
  /* device time per stage in milliseconds (CUDA events on the ctx stream);
   * only filled when mf_ctx_set_timing(ctx, 1) was called. */
  float ms_upload;        /* H2D of the meshes (host entry points only) */
  float ms_prepare;       /* normals, wedge tangents, reliability, setup */
  float ms_bvh;           /* LBVH build (Morton, sort, emit, refit, repack) */
  float ms_raster;        /* G-buffer rasterisation */
  float ms_transfer;      /* closest-point transfer + RGB8 encode */
  float ms_dilate;        /* seam dilation: the dilation-links kernel of the fused full-atlas
                           * bake (its copies ride on the transfer), else the dilation pass */
  float ms_download;      /* D2H of the result (host entry points only) */
  float ms_total;
} mf_bake_stats;

typedef struct mf_ctx mf_ctx;    /* device context: device + stream + scratch */
typedef struct mf_mesh mf_mesh;  /* device-resident mesh (+ cached derived data) */
typedef struct mf_bvh mf_bvh;    /* device-resident LBVH over an mf_mesh */

/* ---- library / context -------------------------------------------------- */
const char* mf_version(void);
int mf_abi_version(void);
const char* mf_last_error(void);
/* stream: a cudaStream_t (nullable: the context creates its own). */
int mf_ctx_create(int device, void* stream, mf_ctx** out);
void mf_ctx_destroy(mf_ctx* ctx);
int mf_ctx_synchronize(mf_ctx* ctx);
int mf_ctx_set_timing(mf_ctx* ctx, int enabled);
/* Number of kernels this context has launched since creation. */
int64_t mf_ctx_launch_count(const mf_ctx* ctx);

/* ---- device-resident meshes -------------------------------------------- */
/* Validates (validateMesh, core/mesh.cpp:37-48) and uploads. */
int mf_mesh_upload(mf_ctx* ctx, const mf_mesh_view* mesh, mf_mesh** out);
void mf_mesh_destroy(mf_mesh* mesh);

/* ---- reference-shaped entry points (host buffers) ----------------------- */
/* rasterizeGBuffer (bake/gbuffer.h:65, gbuffer.cpp:92-191).
 * Outputs: pos/nrm/tan/bit res*res*3 f32, valid/reliable res*res u8. */
int mf_raster_gbuffer(mf_ctx* ctx, const mf_mesh_view* lowpoly, int resolution, float* position,
                      float* normal, float* tangent, float* bitangent, uint8_t* valid,
                      uint8_t* reliable);

/* transferNormals (bake/gbuffer.h:72-73, gbuffer.cpp:193-252).
 * valid == NULL or resolution < 1 means an empty G-buffer (InvalidConfig). */
int mf_transfer_normals(mf_ctx* ctx, int resolution, const float* position, const float* normal,
                        const float* tangent, const float* bitangent, const uint8_t* valid,
                        const uint8_t* reliable, const mf_mesh_view* highpoly,
                        double bbox_diagonal, double max_distance_fraction, uint8_t* rgb_out);

/* dilateSeams (bake/gbuffer.h:79, gbuffer.cpp:254-322). The map is
 * width x height x channels; the G-buffer mask is gbuffer_res^2. */
int mf_dilate_seams(mf_ctx* ctx, int width, int height, int channels, const uint8_t* map_in,
                    int gbuffer_res, const uint8_t* valid, int radius, uint8_t* map_out);

/* The fused bake: dilateSeams(transferNormals(rasterizeGBuffer(lo,res), hi,
 * diag, frac), g, radius) (test_bake.cpp:205-206) with the G-buffer kept in
 * HBM. rgb_out res*res*3 host. dbg_face (nullable, res*res i32): -1 invalid,
 * -2 unreliable, -3 miss, >=0 hit face. dbg_ts (nullable, res*res*3 f64): the
 * normalised tangent-space vector before encoding (0 where not encoded). */
int mf_bake_normal_map(mf_ctx* ctx, const mf_mesh_view* lowpoly, const mf_mesh_view* highpoly,
                       int resolution, double bbox_diagonal, double max_distance_fraction,
                       int radius, uint8_t* rgb_out, int32_t* dbg_face, double* dbg_ts,
                       mf_bake_stats* stats);

/* Atlas encodings of the fused bake (north_star item 4). RGB8 is the
 * reference's ImageU8(res, res, 3) (gbuffer.cpp:212, encodeChannel :85-88).
 * RGBA8: the same three bytes plus alpha 255, 4 bytes per texel. RG16: the
 * normalised tangent-space x, y as unorm16 round((v + 1) / 2 * 65535),
 * clamped, little-endian x then y (z = sqrt(1 - x^2 - y^2) on decode);
 * background and neutral texels both store (32768, 32768). Dilation copies
 * whole pixels, as dilateSeams does (gbuffer.cpp:311-318). */
enum { MF_ATLAS_RGB8 = 0, MF_ATLAS_RGBA8 = 1, MF_ATLAS_RG16 = 2 };

/* mf_bake_normal_map with an atlas encoding: out holds res*res*bpp bytes,
 * bpp = 3 (RGB8) or 4 (RGBA8, RG16). format RGB8 is mf_bake_normal_map. */
int mf_bake_normal_map_ex(mf_ctx* ctx, const mf_mesh_view* lowpoly, const mf_mesh_view* highpoly,
                          int resolution, double bbox_diagonal, double max_distance_fraction,
                          int radius, int format, void* out, mf_bake_stats* stats);

/* Same bake over device-resident meshes into a device buffer, for rows
 * [row_begin, row_end) of the atlas (0, res for the whole map). rgb_dev holds
 * (row_end - row_begin) * res * 3 bytes. Rows outside the range are still
 * rasterised/transferred within the dilation halo so the slab is exact. */
int mf_bake_normal_map_dev(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int resolution,
                           double bbox_diagonal, double max_distance_fraction, int radius,
                           int row_begin, int row_end, uint8_t* rgb_dev, mf_bake_stats* stats);
/* mf_bake_normal_map_dev with an atlas encoding (MF_ATLAS_*): out_dev holds
 * (row_end - row_begin) * res * bpp bytes (4-byte aligned for bpp 4). */
int mf_bake_normal_map_dev_ex(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int resolution,
                              double bbox_diagonal, double max_distance_fraction, int radius,
                              int row_begin, int row_end, int format, void* out_dev, mf_bake_stats* stats);

/* Per-row valid-texel counts (res int64 on the host) from a coverage
 * pre-pass; used to balance row shards by N_v. */
int mf_coverage_rows(mf_ctx* ctx, mf_mesh* lowpoly, int resolution, int64_t* row_counts);

/* ---- BVH (spatial/bvh.h:30-69) ----------------------------------------- */
/* Bvh::Bvh (bvh.cpp:48-61): validates and builds an LBVH on the device.
 * The mesh must outlive the tree, as in the reference (bvh.h:27). The tree
 * owns its arrays, query scratch and stream: it may outlive `ctx`, and its
 * queries are safe from several host threads at once (they serialise on a
 * per-tree lock), as the reference's const queries are (bvh.h:28). */
int mf_bvh_build(mf_ctx* ctx, mf_mesh* mesh, mf_bvh** out);
void mf_bvh_destroy(mf_bvh* bvh);
/* Stream the tree's queries run on (null = the tree's own stream). Default:
 * the building context's stream if the caller supplied it at mf_ctx_create,
 * else the tree's own. Device-pointer inputs must be ready on that stream. */
int mf_bvh_set_stream(mf_bvh* bvh, void* stream);
/* Node count, leaf count, max depth. */
int mf_bvh_info(const mf_bvh* bvh, int32_t* nodes, int32_t* leaves, int32_t* depth);
/* Export in the reference's Node layout (bvh.h:32-39): per node
 * box min/max (6 f64), left, right, first, count (4 i32); plus faceOrder. */
int mf_bvh_export(mf_bvh* bvh, double* boxes, int32_t* links, int32_t* face_order);

/* Bvh::closestPointWithin (bvh.cpp:151-176); max_distance = +inf gives
 * closestPoint (bvh.cpp:147-149). Host arrays of n queries. Outputs:
 * face (-1 = none), dist_sq (+inf when none), point[3], bary[3]. */
int mf_bvh_closest_within(mf_bvh* bvh, const double* queries, int64_t n, double max_distance,
                          int32_t* face, double* dist_sq, double* point, double* bary);
/* Device-pointer variant of the above. */
int mf_bvh_closest_within_dev(mf_bvh* bvh, const double* queries_dev, int64_t n,
                              double max_distance, int32_t* face_dev, double* dist_sq_dev,
                              double* point_dev, double* bary_dev);

/* Bvh::raycastFirst (bvh.cpp:100-140): nearest hit with tmin <= t <= tmax,
 * ties to the lower face. face -1 = miss (t = +inf). */
int mf_bvh_raycast_first(mf_bvh* bvh, const double* origins, const double* dirs, int64_t n,
                         double tmin, double tmax, int32_t* face, double* t, double* u, double* v);
int mf_bvh_raycast_first_dev(mf_bvh* bvh, const double* origins_dev, const double* dirs_dev,
                             int64_t n, double tmin, double tmax, int32_t* face_dev,
                             double* t_dev, double* u_dev, double* v_dev);

/* ---- multi-GPU: the sharded atlas gathered by the producing kernel ------ */
/* CUDA IPC export of the device allocation that holds dev_ptr: a 64-byte
 * handle plus dev_ptr's byte offset inside it (caching allocators hand out
 * interior pointers). */
int mf_ipc_export(const void* dev_ptr, uint8_t* handle64, uint64_t* offset);
/* Opens a handle exported by another process on this node (peer GPU over
 * NVLink, or the same GPU) into a device pointer usable by this context's
 * kernels; closed by mf_ipc_close or with the context. */
int mf_ipc_open(mf_ctx* ctx, const uint8_t* handle64, uint64_t offset, void** dev_ptr);
int mf_ipc_close(mf_ctx* ctx, void* dev_ptr);
/* mf_bake_normal_map_dev for rows [row_begin, row_end) whose dilation kernel
 * stores every output row straight into each of the n_dst (1..8) full
 * res x res x 3 atlases - this rank's own and its peers' (mf_ipc_open) - at
 * its row index: the atlas all-gather of the row-sharded bake
 * happens inside the producing kernel over peer memory instead of a separate
 * collective. The caller synchronises ranks (a host barrier after this call
 * returns) before reading its atlas. */
int mf_bake_normal_map_dev_publish(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int resolution,
                                   double bbox_diagonal, double max_distance_fraction, int radius, int row_begin,
                                   int row_end, void* const* dst_atlases, int n_dst, mf_bake_stats* stats);

/* ---- bulk closest-point callers ------------------------ */
/* markSurfaceBand (signfield/sign_grid.cpp:23-69, sign_grid.h:14-50) over the
 * mesh `bvh` was built on: grid parameters exactly as the reference derives
 * them (auto-fit cube with dilate_radius + 3 voxels of margin, or the cube
 * `domain` = min xyz, max xyz when non-null), then one bounded closest-point
 * query per voxel centre. Outputs (x fastest, res^3 each): labels 0 = Unknown,
 * 1 = SurfaceBand (VoxelLabel); distance f32 (truncation where no surface is
 * within it). grid_out (nullable, 5 f64): origin xyz, voxelSize, truncation.
 * Errors as the reference: InvalidConfig (resolution < 8, dilate_radius < 0,
 * resolution too small for the margin), OutOfBounds (mesh not inside the grid
 * with 2 voxels of margin). */
int mf_surface_band(mf_bvh* bvh, int resolution, double band_voxels, int dilate_radius, const double* domain,
                    uint8_t* labels, float* distance, double* grid_out);
/* Device-pointer outputs (labels_dev, distance_dev). */
int mf_surface_band_dev(mf_bvh* bvh, int resolution, double band_voxels, int dilate_radius, const double* domain,
                        uint8_t* labels_dev, float* distance_dev, double* grid_out);

/* sampleSdf (signfield/watertight.cpp:29-38, watertight.h:25-28) for n points
 * against the tree of the watertight mesh: values[i] = sign * distance, the
 * distance of the unbounded closest point (closestPoint, bvh.cpp:147-149),
 * the sign that of sampleSignedField (sign_grid.cpp:239-264): the trilinear
 * interpolation of `field` (grid_res^3 f32, x fastest, voxel centres at
 * grid_origin + (i + 0.5) * voxel_size), -1 where it is < 0, else +1. */
int mf_sample_sdf(mf_bvh* bvh, int grid_res, const double* grid_origin, double voxel_size, const float* field,
                  const double* points, int64_t n, double* values);
int mf_sample_sdf_dev(mf_bvh* bvh, int grid_res, const double* grid_origin, double voxel_size, const float* field_dev,
                      const double* points_dev, int64_t n, double* values_dev);

/* ---- ortho ray-cast views ------------------------------ */
/* fibonacciCameras (render/camera.cpp:38-55): count x 7 f64 per camera =
 * direction xyz, up xyz, halfExtent. Host-only helper (no device). */
int mf_fibonacci_cameras(int count, double half_extent, double* cameras);
/* renderView (render/raster.cpp:12-102) for n_views cameras (n x 7 as above)
 * at resolution^2 pixels each, one pixel ray per thread through the LBVH of
 * `mesh` (built per call). Per view, row-major: face i32 (-1 background),
 * depth f32 (+inf background), position f32x3, normal f32x3 (interpolated
 * `vertex_normals`, V x 3 f64; zero when null). backface_cull != 0 is
 * RasterOptions::backfaceCull (raster.h:29-33). Any output may be null. */
int mf_render_views(mf_ctx* ctx, const mf_mesh_view* mesh, const double* cameras, int n_views, int resolution,
                    const double* vertex_normals, int backface_cull, int32_t* face, float* depth, float* position,
                    float* normal);
/* castVisibility (visibility/visibility.cpp:13-59): the mesh centred on its
 * bounds, `viewpoints` fibonacci cameras of half extent 1.04 x its bounding
 * radius, resolution^2 pixel rays each; hits[f] = pixels face f won over all
 * views, state[f] = FaceVisibility (0 Hidden, 1 Visible). state may be null.
 * Errors: EmptyMesh / InvalidGeometry (validateMesh), InvalidConfig
 * (viewpoints or resolution <= 0). */
int mf_cast_visibility(mf_ctx* ctx, const mf_mesh_view* mesh, int viewpoints, int resolution, int64_t* hits,
                       uint8_t* state);

/* raycastFirstBrute / closestPointBrute (bvh.cpp:178-189): O(faces) per
 * query with the same tie rules, one CTA per query on the device. */
int mf_closest_point_brute(mf_ctx* ctx, const mf_mesh_view* mesh, const double* queries, int64_t n,
                           int32_t* face, double* dist_sq, double* point, double* bary);
int mf_raycast_first_brute(mf_ctx* ctx, const mf_mesh_view* mesh, const double* origins,
                           const double* dirs, int64_t n, double tmin, double tmax, int32_t* face,
                           double* t, double* u, double* v);

/* ---- texfuse: device-resident G-buffer consumers -------- */
/* The texture-fusion steps of proj/src/texfuse (fuse.h:15-138, mips.h:17-18).
 * Images are ImageF: row-major interleaved f32. A camera is 7 f64 (direction
 * xyz, up xyz, halfExtent; OrthoCamera, render/camera.h:12-38) plus the view
 * resolution passed beside it. The G-buffer planes are the reference layout
 * (mf_raster_gbuffer). Errors follow the reference's checks: InvalidConfig /
 * ShapeMismatch as 1 + ErrorCode. */
typedef struct mf_fuse_options {  /* FuseOptions + BlendOptions (fuse.h:83-86, 122-130) */
  double edge_threshold;   /* 0.02 */
  double depth_tolerance;  /* 0.005 */
  int32_t mip_levels;      /* 6 */
  float sharpen_strength;  /* 0.2 */
  double alpha;            /* 4.0 */
  double epsilon;          /* 1e-8 */
} mf_fuse_options;
void mf_fuse_options_default(mf_fuse_options* options);
/* buildMips' chain length and total f32 count (levels concatenated, each
 * halving rounding up, stopping at 1x1; mips.cpp:96-112). */
int64_t mf_mip_chain_floats(int width, int height, int channels, int levels, int* n_levels);
/* edgeMask (fuse.cpp:66-101) of a rendered view: position w*h*3 f32, face w*h i32. */
int mf_edge_mask(mf_ctx* ctx, int width, int height, const float* position, const int32_t* face,
                 double bbox_diagonal, double threshold, uint8_t* mask);
/* buildMips (mips.cpp:96-112): chain = mf_mip_chain_floats(...) f32, level 0 = base. */
int mf_build_mips(mf_ctx* ctx, int width, int height, int channels, const float* base, int levels, float sharpen,
                  float* chain, int* n_levels);
/* backprojectView (fuse.cpp:103-186): mips = the view's chain (n_mips levels,
 * level 0 view_res^2 x channels), mask view_res^2; outputs gres^2 x channels
 * f32 colour and gres^2 sampled flags. */
int mf_backproject_view(mf_ctx* ctx, int gres, const float* position, const uint8_t* valid, const double* camera,
                        int view_res, int channels, int n_mips, const float* mips, const uint8_t* mask, float* color,
                        uint8_t* sampled);
/* incidenceMap (fuse.cpp:188-221): depth view_res^2 f32; out gres^2 f32. */
int mf_incidence_map(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                     const double* camera, int view_res, const float* depth, double bbox_diagonal,
                     double depth_tolerance, float* out);
/* blendViews (fuse.cpp:223-280): n_views partial atlases (colors n x w*h*ch,
 * sampled n x w*h), incidence n x w*h, priors n; out w*h*ch f32 + filled. */
int mf_blend_views(mf_ctx* ctx, int n_views, int width, int height, int channels, const float* colors,
                   const uint8_t* sampled, const float* incidence, const double* priors, double alpha, double epsilon,
                   float* color, uint8_t* filled);
/* fuseViews (fuse.cpp:292-326) up to the blend (the reference's inpainting
 * step, fuse.h:110, is declared but never defined by it): per view edgeMask,
 * buildMips, backprojectView, incidenceMap, then blendViews. cameras n x 7
 * (host); view_position n x vres^2 x 3, view_face n x vres^2, view_depth n x
 * vres^2, colors n x vres^2 x channels; priors n (host). options NULL =
 * defaults. Host-buffer form: */
int mf_fuse_views(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                  int n_views, const double* cameras, int view_res, const float* view_position,
                  const int32_t* view_face, const float* view_depth, int channels, const float* colors,
                  const double* priors, double bbox_diagonal, const mf_fuse_options* options, float* color,
                  uint8_t* filled);
/* Same with every image a device pointer (G-buffer, views, colours and
 * outputs resident in HBM; cameras and priors stay host arrays). */
int mf_fuse_views_dev(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                      int n_views, const double* cameras, int view_res, const float* view_position,
                      const int32_t* view_face, const float* view_depth, int channels, const float* colors,
                      const double* priors, double bbox_diagonal, const mf_fuse_options* options, float* color,
                      uint8_t* filled);
/* rasterizeGBuffer into device buffers (the G-buffer the texfuse calls
 * consume without leaving HBM): planes res*res*3 f32, masks res*res u8. */
int mf_raster_gbuffer_dev(mf_ctx* ctx, mf_mesh* lowpoly, int resolution, float* position, float* normal,
                          float* tangent, float* bitangent, uint8_t* valid, uint8_t* reliable);

/* ---- lowpoly helpers ----------------------------------------------------- */
/* computeWedgeTangents (bake/tangent.cpp:22-82): frames n_faces x 3 corners x
 * {tangent, bitangent, normal} x 3 f64 (= std::array<TangentFrame,3>). */
int mf_wedge_tangents(mf_ctx* ctx, const mf_mesh_view* mesh, double* frames);
/* computeVertexNormals (core/mesh.cpp:24-35): n_vertices x 3 f64. */
int mf_vertex_normals(mf_ctx* ctx, const mf_mesh_view* mesh, double* normals);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* MFBAKE_H_ */
