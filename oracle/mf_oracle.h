/*
 * oracle/mf_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference bake path (meshforge), used as the
 * parity checker for the CUDA library. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product path (libmfbake.so) never does.
 *
 * Every function cites the reference file:line it restates. Parity pin: the
 * restatement is checked bit-for-bit against the reference's own translation
 * units (oracle/_ref, built by oracle/Makefile) and against the committed
 * golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Status codes and the mesh view are those of include/mfbake.h.
 */
#ifndef MF_ORACLE_H_
#define MF_ORACLE_H_

#include <stdint.h>

#include "mfbake.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* core/mesh.cpp:24-35 */
int orc_vertex_normals(const mf_mesh_view* m, double* normals);
/* bake/tangent.cpp:22-82; frames: F x 3 corners x {T, B, N} x 3 */
int orc_wedge_tangents(const mf_mesh_view* m, double* frames);
/* bake/gbuffer.cpp:31-83 (anonymous reliableFaces) */
int orc_reliable_faces(const mf_mesh_view* m, uint8_t* reliable);
/* bake/gbuffer.cpp:92-191 */
int orc_raster_gbuffer(const mf_mesh_view* lo, int res, float* pos, float* nrm, float* tan,
                       float* bit, uint8_t* valid, uint8_t* reliable);
/* bake/gbuffer.cpp:193-252; dbg_face/dbg_ts nullable (as mf_bake_normal_map);
 * threads <= 0 means one per hardware thread. */
int orc_transfer_normals(int res, const float* pos, const float* nrm, const float* tan,
                         const float* bit, const uint8_t* valid, const uint8_t* reliable,
                         const mf_mesh_view* hi, double diag, double frac, uint8_t* rgb,
                         int32_t* dbg_face, double* dbg_ts, int threads);
/* bake/gbuffer.cpp:254-322 */
int orc_dilate_seams(int w, int h, int c, const uint8_t* map_in, int gres, const uint8_t* valid,
                     int radius, uint8_t* out);
/* test_bake.cpp:205-206 composition; rgb_raw (nullable) = before dilation. */
int orc_bake(const mf_mesh_view* lo, const mf_mesh_view* hi, int res, double diag, double frac,
             int radius, uint8_t* rgb, uint8_t* rgb_raw, int32_t* dbg_face, double* dbg_ts,
             int threads, int64_t* n_valid, int64_t* n_queries);

/* spatial/bvh.cpp:147-189: closestPointWithin (brute = closestPointBrute). */
int orc_closest_within(const mf_mesh_view* m, const double* q, int64_t n, double max_dist,
                       int brute, int threads, int32_t* face, double* dist_sq, double* point,
                       double* bary);
/* spatial/bvh.cpp:100-140, 178-183: raycastFirst (brute = raycastFirstBrute). */
int orc_raycast_first(const mf_mesh_view* m, const double* o, const double* d, int64_t n,
                      double tmin, double tmax, int brute, int threads, int32_t* face, double* t,
                      double* u, double* v);

/* signfield/sign_grid.cpp:23-69 markSurfaceBand: labels (0 Unknown, 1 SurfaceBand) and
 * f32 distances, res^3 x-fastest; grid_out = origin xyz, voxelSize, truncation. */
int orc_surface_band(const mf_mesh_view* m, int res, double band_voxels, int dilate, const double* domain,
                     int threads, uint8_t* labels, float* dist, double* grid_out);

/* render/camera.cpp:38-55, render/raster.cpp:12-102, visibility/visibility.cpp:13-59 */
void orc_fibonacci_cameras(int count, double half_extent, double* cams7);
int orc_render_views(const mf_mesh_view* m, const double* cams7, int n_views, int res, const double* vn, int cull,
                     int32_t* face, float* depth, float* pos, float* nrm);
int orc_cast_visibility(const mf_mesh_view* m, int viewpoints, int res, int64_t* hits);

#ifdef __cplusplus
}
#endif

#endif /* MF_ORACLE_H_ */
