/*
 * oracle/mf_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU parity checker.
 *
 * A plain-C restatement of the reference bake path (meshforge). Each function
 * follows the cited reference lines with the same floating-point operation
 * order: 3-term dot products are evaluated as
 * (a0*b0 + a1*b1) + a2*b2, linear combinations left to right per component,
 * no FMA contraction (-ffp-contract=off), IEEE division and sqrt.
 *
 * Never linked into or called by the product library.
 */
#define _GNU_SOURCE
#include "mf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---- errors --------------------------------------------------------------- */
static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ---- small vector helpers (Eigen order, see header) ----------------------- */
typedef struct { double v[3]; } d3;
static inline d3 mk3(double x, double y, double z) { d3 r = {{x, y, z}}; return r; }
static inline d3 ld3(const double* p) { return mk3(p[0], p[1], p[2]); }
static inline d3 add3(d3 a, d3 b) { return mk3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static inline d3 sub3(d3 a, d3 b) { return mk3(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static inline d3 scl3(double s, d3 a) { return mk3(s * a.v[0], s * a.v[1], s * a.v[2]); }
static inline d3 mul3(d3 a, double s) { return mk3(a.v[0] * s, a.v[1] * s, a.v[2] * s); }
static inline d3 div3(d3 a, double s) { return mk3(a.v[0] / s, a.v[1] / s, a.v[2] / s); }
static inline double dot3(d3 a, d3 b) { return a.v[0] * b.v[0] + a.v[1] * b.v[1] + a.v[2] * b.v[2]; }
static inline double sqn3(d3 a) { return dot3(a, a); }
static inline double nrm3(d3 a) { return sqrt(sqn3(a)); }
static inline d3 cross3(d3 a, d3 b) {
  return mk3(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2],
             a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static inline double cross2(double ax, double ay, double bx, double by) { return ax * by - ay * bx; }

static int hw_threads(int threads) {
  if (threads > 0) return threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* ---- parallel-for (core/parallel.h:19-43: fixed chunks, atomic cursor) ---- */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
  int64_t next, end, chunk;
  range_fn fn;
  void* ctx;
  pthread_mutex_t mu;
} pf_state;
static void* pf_worker(void* arg) {
  pf_state* s = (pf_state*)arg;
  for (;;) {
    pthread_mutex_lock(&s->mu);
    int64_t lo = s->next;
    s->next += s->chunk;
    pthread_mutex_unlock(&s->mu);
    if (lo >= s->end) return NULL;
    int64_t hi = lo + s->chunk < s->end ? lo + s->chunk : s->end;
    s->fn(s->ctx, lo, hi);
  }
}
static void parallel_for(int64_t n, int64_t chunk, int threads, range_fn fn, void* ctx) {
  if (n <= 0) return;
  threads = hw_threads(threads);
  if (threads <= 1 || n <= chunk) {
    fn(ctx, 0, n);
    return;
  }
  pf_state s;
  s.next = 0;
  s.end = n;
  s.chunk = chunk;
  s.fn = fn;
  s.ctx = ctx;
  pthread_mutex_init(&s.mu, NULL);
  int spawn = (int)((n + chunk - 1) / chunk);
  if (spawn > threads) spawn = threads;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)spawn);
  for (int i = 1; i < spawn; ++i) pthread_create(&th[i], NULL, pf_worker, &s);
  pf_worker(&s);
  for (int i = 1; i < spawn; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&s.mu);
}

/* ---- mesh helpers ---------------------------------------------------------- */
static inline d3 P(const mf_mesh_view* m, int i) { return ld3(m->positions + 3 * (size_t)i); }
static inline int FV(const mf_mesh_view* m, int f, int k) { return m->faces[3 * (size_t)f + k]; }
static inline int has_normals(const mf_mesh_view* m) { return m->normals && m->n_vertices > 0; }
static inline int has_uvs(const mf_mesh_view* m) { return m->face_uvs && m->uvs && m->n_uvs > 0; }

/* core/mesh.cpp:37-48 */
static int validate_mesh(const mf_mesh_view* m) {
  if (!m || m->n_faces <= 0) return fail(MF_ERR_EMPTY_MESH, "EmptyMesh: mesh has no faces");
  for (int64_t i = 0; i < 3 * (int64_t)m->n_vertices; ++i)
    if (!isfinite(m->positions[i]))
      return fail(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: non-finite vertex coordinate");
  for (int64_t i = 0; i < 3 * (int64_t)m->n_faces; ++i)
    if (m->faces[i] < 0 || m->faces[i] >= m->n_vertices)
      return fail(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: face index out of range");
  return 0;
}

/* core/mesh.h:28-31 faceAreaVector */
static d3 face_area_vector(const mf_mesh_view* m, int f) {
  d3 p0 = P(m, FV(m, f, 0)), p1 = P(m, FV(m, f, 1)), p2 = P(m, FV(m, f, 2));
  return scl3(0.5, cross3(sub3(p1, p0), sub3(p2, p0)));
}

/* core/mesh.cpp:24-35 */
int orc_vertex_normals(const mf_mesh_view* m, double* out) {
  memset(out, 0, sizeof(double) * 3 * (size_t)m->n_vertices);
  for (int f = 0; f < m->n_faces; ++f) {
    d3 an = face_area_vector(m, f);
    for (int k = 0; k < 3; ++k) {
      double* n = out + 3 * (size_t)FV(m, f, k);
      n[0] = n[0] + an.v[0];
      n[1] = n[1] + an.v[1];
      n[2] = n[2] + an.v[2];
    }
  }
  for (int v = 0; v < m->n_vertices; ++v) {
    d3 n = ld3(out + 3 * (size_t)v);
    double len = nrm3(n);
    if (len > 0) {
      n = div3(n, len);
      memcpy(out + 3 * (size_t)v, n.v, 24);
    }
  }
  return 0;
}

/* normals as used by tangent.cpp:26-31 / gbuffer.cpp:201-206 */
static double* unit_normals(const mf_mesh_view* m) {
  double* n = (double*)malloc(sizeof(double) * 3 * (size_t)(m->n_vertices > 0 ? m->n_vertices : 1));
  if (has_normals(m)) memcpy(n, m->normals, sizeof(double) * 3 * (size_t)m->n_vertices);
  else orc_vertex_normals(m, n);
  for (int v = 0; v < m->n_vertices; ++v) {
    d3 x = ld3(n + 3 * (size_t)v);
    double len = nrm3(x);
    if (len > 1e-20) {
      x = div3(x, len);
      memcpy(n + 3 * (size_t)v, x.v, 24);
    }
  }
  return n;
}

/* bake/tangent.cpp:11-20 */
static d3 any_perpendicular(d3 n) {
  int s = 0;
  for (int k = 1; k < 3; ++k)
    if (fabs(n.v[k]) < fabs(n.v[s])) s = k;
  d3 axis = mk3(0, 0, 0);
  axis.v[s] = 1.0;
  d3 p = cross3(axis, n);
  double len = nrm3(p);
  return len > 1e-20 ? div3(p, len) : mk3(1, 0, 0);
}

/* open-addressing map (v<<32 | uv) -> accumulated tangent, insertion keeps
 * the face-order summation of tangent.cpp:40-63 */
typedef struct {
  uint64_t* keys;
  d3* vals;
  uint8_t* used;
  size_t cap;
} wedge_map;
static size_t wm_slot(const wedge_map* wm, uint64_t key) {
  uint64_t h = key * 0x9E3779B97F4A7C15ull;
  size_t i = (size_t)(h >> 17) & (wm->cap - 1);
  while (wm->used[i] && wm->keys[i] != key) i = (i + 1) & (wm->cap - 1);
  return i;
}

/* bake/tangent.cpp:22-82 */
int orc_wedge_tangents(const mf_mesh_view* m, double* frames) {
  if (!has_uvs(m))
    return fail(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: tangent frames require a UV-mapped mesh");
  double* normals = unit_normals(m);
  wedge_map wm;
  wm.cap = 1;
  while (wm.cap < 6 * (size_t)m->n_faces + 16) wm.cap <<= 1;
  wm.keys = (uint64_t*)calloc(wm.cap, 8);
  wm.vals = (d3*)calloc(wm.cap, sizeof(d3));
  wm.used = (uint8_t*)calloc(wm.cap, 1);
  for (int f = 0; f < m->n_faces; ++f) {
    const int* tri = m->faces + 3 * (size_t)f;
    const int* uvt = m->face_uvs + 3 * (size_t)f;
    d3 p0 = P(m, tri[0]), p1 = P(m, tri[1]), p2 = P(m, tri[2]);
    const double* u0 = m->uvs + 2 * (size_t)uvt[0];
    const double* u1 = m->uvs + 2 * (size_t)uvt[1];
    const double* u2 = m->uvs + 2 * (size_t)uvt[2];
    double d1x = u1[0] - u0[0], d1y = u1[1] - u0[1];
    double d2x = u2[0] - u0[0], d2y = u2[1] - u0[1];
    double det = d1x * d2y - d2x * d1y;
    if (fabs(det) < 1e-20) continue;
    d3 ft = div3(sub3(mul3(sub3(p1, p0), d2y), mul3(sub3(p2, p0), d1y)), det);
    for (int k = 0; k < 3; ++k) {
      d3 self = P(m, tri[k]);
      d3 ea = sub3(P(m, tri[(k + 1) % 3]), self);
      d3 eb = sub3(P(m, tri[(k + 2) % 3]), self);
      double la = nrm3(ea), lb = nrm3(eb);
      if (la < 1e-20 || lb < 1e-20) continue;
      double c = dot3(ea, eb) / (la * lb);
      if (c < -1.0) c = -1.0;
      if (c > 1.0) c = 1.0;
      double angle = acos(c);
      uint64_t key = ((uint64_t)(uint32_t)tri[k] << 32) | (uint32_t)uvt[k];
      size_t s = wm_slot(&wm, key);
      if (!wm.used[s]) {
        wm.used[s] = 1;
        wm.keys[s] = key;
        wm.vals[s] = mk3(0, 0, 0);
      }
      wm.vals[s] = add3(wm.vals[s], scl3(angle, ft));
    }
  }
  for (int f = 0; f < m->n_faces; ++f) {
    for (int k = 0; k < 3; ++k) {
      int v = FV(m, f, k);
      d3 N = ld3(normals + 3 * (size_t)v);
      if (nrm3(N) < 1e-20) N = mk3(0, 0, 1);
      d3 t = mk3(0, 0, 0);
      uint64_t key = ((uint64_t)(uint32_t)v << 32) | (uint32_t)m->face_uvs[3 * (size_t)f + k];
      size_t s = wm_slot(&wm, key);
      if (wm.used[s]) t = wm.vals[s];
      t = sub3(t, mul3(N, dot3(N, t)));
      double len = nrm3(t);
      d3 T = len > 1e-12 ? div3(t, len) : any_perpendicular(N);
      d3 B = cross3(N, T);
      double* o = frames + ((size_t)f * 3 + k) * 9;
      memcpy(o, T.v, 24);
      memcpy(o + 3, B.v, 24);
      memcpy(o + 6, N.v, 24);
    }
  }
  free(wm.keys);
  free(wm.vals);
  free(wm.used);
  free(normals);
  return 0;
}

/* ---- reliableFaces, bake/gbuffer.cpp:31-83 -------------------------------- */
static int uf_find(int* parent, int x) {
  while (parent[x] != x) x = parent[x] = parent[parent[x]];
  return x;
}
static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
int orc_reliable_faces(const mf_mesh_view* m, uint8_t* reliable) {
  const int nf = m->n_faces, nu = m->n_uvs;
  int* parent = (int*)malloc(sizeof(int) * (size_t)nu);
  for (int i = 0; i < nu; ++i) parent[i] = i;
  for (int f = 0; f < nf; ++f) {
    const int* t = m->face_uvs + 3 * (size_t)f;
    for (int e = 1; e <= 2; ++e) {
      int a = uf_find(parent, t[0]), b = uf_find(parent, t[e]);
      if (a != b) parent[a > b ? a : b] = a < b ? a : b;
    }
  }
  double* uvArea = (double*)malloc(sizeof(double) * (size_t)nf);
  double* ratio = (double*)malloc(sizeof(double) * (size_t)nf);
  int* island = (int*)malloc(sizeof(int) * (size_t)nf);
  int* count = (int*)calloc((size_t)nu + 1, sizeof(int));
  uint8_t* has_ratio = (uint8_t*)calloc((size_t)nf, 1);
  for (int f = 0; f < nf; ++f) {
    const int* t = m->face_uvs + 3 * (size_t)f;
    const double* a = m->uvs + 2 * (size_t)t[0];
    const double* b = m->uvs + 2 * (size_t)t[1];
    const double* c = m->uvs + 2 * (size_t)t[2];
    uvArea[f] = 0.5 * fabs(cross2(b[0] - a[0], b[1] - a[1], c[0] - a[0], c[1] - a[1]));
    island[f] = uf_find(parent, t[0]);
    ratio[f] = -1.0;
    const double surf = nrm3(face_area_vector(m, f));
    if (surf > 1e-20) {
      ratio[f] = uvArea[f] / surf;
      has_ratio[f] = 1;
      count[island[f]]++;
    }
  }
  /* per-island sample lists (face order), median = element size/2 of the
   * sorted list (== std::nth_element at begin + size/2, gbuffer.cpp:69-71) */
  int* start = (int*)malloc(sizeof(int) * ((size_t)nu + 1));
  start[0] = 0;
  for (int i = 0; i < nu; ++i) start[i + 1] = start[i] + count[i];
  double* samples = (double*)malloc(sizeof(double) * (size_t)(start[nu] > 0 ? start[nu] : 1));
  int* fillp = (int*)calloc((size_t)nu, sizeof(int));
  for (int f = 0; f < nf; ++f)
    if (has_ratio[f]) samples[start[island[f]] + fillp[island[f]]++] = ratio[f];
  double* median = (double*)calloc((size_t)nu, sizeof(double));
  for (int i = 0; i < nu; ++i) {
    int n = count[i];
    if (!n) continue;
    qsort(samples + start[i], (size_t)n, sizeof(double), cmp_double);
    median[i] = samples[start[i] + n / 2];
  }
  for (int f = 0; f < nf; ++f) {
    reliable[f] = 0;
    if (uvArea[f] < 1e-8) continue;
    if (ratio[f] < 0.0) continue;
    const double md = median[island[f]];
    if (ratio[f] > 100.0 * md || 100.0 * ratio[f] < md) continue;
    reliable[f] = 1;
  }
  free(parent);
  free(uvArea);
  free(ratio);
  free(island);
  free(count);
  free(start);
  free(samples);
  free(fillp);
  free(median);
  free(has_ratio);
  return 0;
}

/* ---- rasterizeGBuffer, bake/gbuffer.cpp:92-191 ----------------------------- */
static inline int owns_boundary(double dx, double dy) {
  if (dy != 0.0) return dy > 0.0;
  return dx < 0.0;
}

int orc_raster_gbuffer(const mf_mesh_view* lo, int res, float* pos, float* nrm, float* tan,
                       float* bit, uint8_t* valid, uint8_t* rel) {
  int rc = validate_mesh(lo);
  if (rc) return rc;
  if (!has_uvs(lo))
    return fail(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: atlas rasterization needs a UV-mapped mesh");
  if (res < 1) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: resolution must be >= 1");
  const int nf = lo->n_faces;
  double* frames = (double*)malloc(sizeof(double) * 27 * (size_t)nf);
  orc_wedge_tangents(lo, frames);
  uint8_t* reliable = (uint8_t*)malloc((size_t)nf);
  orc_reliable_faces(lo, reliable);

  const size_t texels = (size_t)res * res;
  memset(pos, 0, texels * 12);
  memset(nrm, 0, texels * 12);
  memset(tan, 0, texels * 12);
  memset(bit, 0, texels * 12);
  memset(valid, 0, texels);
  memset(rel, 0, texels);
  int* owner = (int*)malloc(sizeof(int) * texels);
  for (size_t i = 0; i < texels; ++i) owner[i] = -1;

  const double R = res;
  rc = 0;
  for (int f = 0; f < nf && !rc; ++f) {
    const int* uvt = lo->face_uvs + 3 * (size_t)f;
    double p[3][2];
    for (int k = 0; k < 3; ++k) {
      p[k][0] = lo->uvs[2 * (size_t)uvt[k]] * R;
      p[k][1] = lo->uvs[2 * (size_t)uvt[k] + 1] * R;
    }
    const double doubled =
        cross2(p[1][0] - p[0][0], p[1][1] - p[0][1], p[2][0] - p[0][0], p[2][1] - p[0][1]);
    if (doubled == 0.0) continue;
    const double orient = doubled > 0.0 ? 1.0 : -1.0;
    double ox[3], oy[3], dx[3], dy[3], sg[3];
    for (int k = 0; k < 3; ++k) {
      const int i0 = uvt[k], i1 = uvt[(k + 1) % 3];
      const int l = i0 < i1 ? i0 : i1, h = i0 < i1 ? i1 : i0;
      if (l == h) {
        sg[k] = 0.0;
        continue;
      }
      ox[k] = lo->uvs[2 * (size_t)l] * R;
      oy[k] = lo->uvs[2 * (size_t)l + 1] * R;
      dx[k] = lo->uvs[2 * (size_t)h] * R - ox[k];
      dy[k] = lo->uvs[2 * (size_t)h + 1] * R - oy[k];
      sg[k] = (i0 == l ? 1.0 : -1.0) * orient;
    }
    if (sg[0] == 0.0 || sg[1] == 0.0 || sg[2] == 0.0) continue;
    double lbx = p[0][0], lby = p[0][1], hbx = p[0][0], hby = p[0][1];
    for (int k = 1; k < 3; ++k) {
      lbx = p[k][0] < lbx ? p[k][0] : lbx;
      lby = p[k][1] < lby ? p[k][1] : lby;
      hbx = hbx < p[k][0] ? p[k][0] : hbx;
      hby = hby < p[k][1] ? p[k][1] : hby;
    }
    int x0 = (int)floor(lbx - 0.5), y0 = (int)floor(lby - 0.5);
    int x1 = (int)ceil(hbx - 0.5), y1 = (int)ceil(hby - 0.5);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > res - 1) x1 = res - 1;
    if (y1 > res - 1) y1 = res - 1;
    const double* fr = frames + (size_t)f * 27; /* [k][T,B,N][3] */
    const int* tri = lo->faces + 3 * (size_t)f;
    for (int y = y0; y <= y1 && !rc; ++y) {
      for (int x = x0; x <= x1; ++x) {
        const double cx = x + 0.5, cy = y + 0.5;
        int inside = 1;
        for (int k = 0; k < 3 && inside; ++k) {
          const double e = sg[k] * cross2(dx[k], dy[k], cx - ox[k], cy - oy[k]);
          if (e < 0.0 || (e == 0.0 && !owns_boundary(sg[k] * dx[k], sg[k] * dy[k]))) inside = 0;
        }
        if (!inside) continue;
        const size_t t = (size_t)y * res + x;
        if (owner[t] >= 0) {
          rc = fail(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
          break;
        }
        owner[t] = f;
        const double w0 = cross2(p[2][0] - p[1][0], p[2][1] - p[1][1], cx - p[1][0], cy - p[1][1]) / doubled;
        const double w1 = cross2(p[0][0] - p[2][0], p[0][1] - p[2][1], cx - p[2][0], cy - p[2][1]) / doubled;
        const double w2 = cross2(p[1][0] - p[0][0], p[1][1] - p[0][1], cx - p[0][0], cy - p[0][1]) / doubled;
        d3 ps = add3(add3(scl3(w0, P(lo, tri[0])), scl3(w1, P(lo, tri[1]))), scl3(w2, P(lo, tri[2])));
        d3 N0 = ld3(fr + 6), N1 = ld3(fr + 9 + 6), N2 = ld3(fr + 18 + 6);
        d3 T0 = ld3(fr), T1 = ld3(fr + 9), T2 = ld3(fr + 18);
        d3 n = add3(add3(scl3(w0, N0), scl3(w1, N1)), scl3(w2, N2));
        const double nLen = nrm3(n);
        n = nLen > 1e-12 ? div3(n, nLen) : N0;
        d3 tg = add3(add3(scl3(w0, T0), scl3(w1, T1)), scl3(w2, T2));
        tg = sub3(tg, mul3(n, dot3(n, tg)));
        const double tLen = nrm3(tg);
        tg = tLen > 1e-12 ? div3(tg, tLen) : any_perpendicular(n);
        d3 b = cross3(n, tg);
        for (int c = 0; c < 3; ++c) {
          pos[3 * t + c] = (float)ps.v[c];
          nrm[3 * t + c] = (float)n.v[c];
          tan[3 * t + c] = (float)tg.v[c];
          bit[3 * t + c] = (float)b.v[c];
        }
        valid[t] = 1;
        rel[t] = reliable[f];
      }
    }
  }
  free(owner);
  free(frames);
  free(reliable);
  return rc;
}

/* ---- median-split BVH, spatial/bvh.cpp:13-98 ------------------------------- */
typedef struct {
  double mn[3], mx[3];
  int left, right, first, count;
} bnode;
typedef struct {
  const mf_mesh_view* m;
  bnode* nodes;
  int n_nodes, cap;
  int* order;
  double* cen;
} bvh_t;

static inline int cen_less(const double* cen, int axis, int a, int b) {
  double ca = cen[3 * (size_t)a + axis], cb = cen[3 * (size_t)b + axis];
  return ca < cb || (ca == cb && a < b);
}
/* quickselect: after the call, v[k] holds the k-th element of the total
 * order (c[axis], face) with smaller ones before it (std::nth_element
 * contract, bvh.cpp:87-91). */
static void select_kth(int* v, int lo, int hi, int k, const double* cen, int axis) {
  while (hi - lo > 1) {
    int mid = lo + (hi - lo) / 2;
    int a = v[lo], b = v[mid], c = v[hi - 1], piv;
    if (cen_less(cen, axis, a, b)) piv = cen_less(cen, axis, b, c) ? b : (cen_less(cen, axis, a, c) ? c : a);
    else piv = cen_less(cen, axis, a, c) ? a : (cen_less(cen, axis, b, c) ? c : b);
    int i = lo, j = hi - 1;
    while (i <= j) {
      while (cen_less(cen, axis, v[i], piv)) ++i;
      while (cen_less(cen, axis, piv, v[j])) --j;
      if (i <= j) {
        int t = v[i];
        v[i] = v[j];
        v[j] = t;
        ++i;
        --j;
      }
    }
    if (k <= j) hi = j + 1;
    else if (k >= i) lo = i;
    else return;
  }
}

static int bvh_build_rec(bvh_t* b, int begin, int end, int depth) {
  if (b->n_nodes == b->cap) {
    b->cap *= 2;
    b->nodes = (bnode*)realloc(b->nodes, sizeof(bnode) * (size_t)b->cap);
  }
  int ni = b->n_nodes++;
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  double cmn[3] = {INFINITY, INFINITY, INFINITY}, cmx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = begin; i < end; ++i) {
    int f = b->order[i];
    for (int k = 0; k < 3; ++k) {
      const double* p = b->m->positions + 3 * (size_t)FV(b->m, f, k);
      for (int c = 0; c < 3; ++c) {
        mn[c] = p[c] < mn[c] ? p[c] : mn[c];
        mx[c] = mx[c] < p[c] ? p[c] : mx[c];
      }
    }
    const double* cc = b->cen + 3 * (size_t)f;
    for (int c = 0; c < 3; ++c) {
      cmn[c] = cc[c] < cmn[c] ? cc[c] : cmn[c];
      cmx[c] = cmx[c] < cc[c] ? cc[c] : cmx[c];
    }
  }
  bnode* nd = &b->nodes[ni];
  memcpy(nd->mn, mn, 24);
  memcpy(nd->mx, mx, 24);
  nd->left = nd->right = -1;
  nd->first = 0;
  nd->count = 0;
  int count = end - begin;
  if (count <= 4 || depth >= 64) {
    nd->first = begin;
    nd->count = count;
    return ni;
  }
  double ext[3] = {cmx[0] - cmn[0], cmx[1] - cmn[1], cmx[2] - cmn[2]};
  int axis = 0;
  for (int c = 1; c < 3; ++c)
    if (ext[c] > ext[axis]) axis = c;
  int mid = begin + count / 2;
  select_kth(b->order, begin, end, mid, b->cen, axis);
  int l = bvh_build_rec(b, begin, mid, depth + 1);
  int r = bvh_build_rec(b, mid, end, depth + 1);
  b->nodes[ni].left = l;
  b->nodes[ni].right = r;
  return ni;
}

static void bvh_build(bvh_t* b, const mf_mesh_view* m) {
  b->m = m;
  const int n = m->n_faces;
  b->order = (int*)malloc(sizeof(int) * (size_t)n);
  b->cen = (double*)malloc(sizeof(double) * 3 * (size_t)n);
  for (int f = 0; f < n; ++f) {
    b->order[f] = f;
    d3 c = div3(add3(add3(P(m, FV(m, f, 0)), P(m, FV(m, f, 1))), P(m, FV(m, f, 2))), 3.0);
    memcpy(b->cen + 3 * (size_t)f, c.v, 24);
  }
  b->cap = 2 * n / 4 + 2;
  b->nodes = (bnode*)malloc(sizeof(bnode) * (size_t)b->cap);
  b->n_nodes = 0;
  bvh_build_rec(b, 0, n, 0);
}
static void bvh_free(bvh_t* b) {
  free(b->order);
  free(b->cen);
  free(b->nodes);
}

/* core/aabb.h:38-41 */
static inline double box_dist_sq(const bnode* nd, d3 p) {
  d3 d;
  for (int c = 0; c < 3; ++c) {
    double a = nd->mn[c] - p.v[c], b = p.v[c] - nd->mx[c];
    double m = a < b ? b : a;
    d.v[c] = m < 0.0 ? 0.0 : m;
  }
  return sqn3(d);
}

/* spatial/tri_geom.h:37-95 */
static d3 closest_point_triangle(d3 p, d3 a, d3 b, d3 c, d3* bary) {
  d3 ab = sub3(b, a), ac = sub3(c, a), ap = sub3(p, a);
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    *bary = mk3(1, 0, 0);
    return a;
  }
  d3 bp = sub3(p, b);
  double d3_ = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3_ >= 0.0 && d4 <= d3_) {
    *bary = mk3(0, 1, 0);
    return b;
  }
  double vc = d1 * d4 - d3_ * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3_ <= 0.0) {
    double w = d1 / (d1 - d3_);
    *bary = mk3(1.0 - w, w, 0);
    return add3(a, scl3(w, ab));
  }
  d3 cp = sub3(p, c);
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) {
    *bary = mk3(0, 0, 1);
    return c;
  }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    *bary = mk3(1.0 - w, 0, w);
    return add3(a, scl3(w, ac));
  }
  double va = d3_ * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3_) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3_) / ((d4 - d3_) + (d5 - d6));
    *bary = mk3(0, 1.0 - w, w);
    return add3(b, scl3(w, sub3(c, b)));
  }
  double denom = 1.0 / (va + vb + vc);
  double wb = vb * denom, wc = vc * denom;
  *bary = mk3(1.0 - wb - wc, wb, wc);
  return add3(add3(a, mul3(ab, wb)), mul3(ac, wc));
}

typedef struct {
  int face;
  double dist_sq;
  d3 point, bary;
} surf_pt;

/* spatial/bvh.cpp:36-44 testFaceClosest + :21-23 improves */
static inline void test_face_closest(const mf_mesh_view* m, int f, d3 q, surf_pt* best) {
  d3 bary;
  d3 pt = closest_point_triangle(q, P(m, FV(m, f, 0)), P(m, FV(m, f, 1)), P(m, FV(m, f, 2)), &bary);
  double ds = sqn3(sub3(pt, q));
  if (ds < best->dist_sq || (ds == best->dist_sq && f < best->face)) {
    best->face = f;
    best->dist_sq = ds;
    best->point = pt;
    best->bary = bary;
  }
}

typedef struct {
  double d;
  int i;
} heap_e;
static inline int he_less(heap_e a, heap_e b) { return a.d < b.d || (a.d == b.d && a.i < b.i); }

/* spatial/bvh.cpp:151-176 best-first bounded closest point */
static surf_pt bvh_closest_within(const bvh_t* b, d3 q, double max_dist, heap_e** heap_buf,
                                  int* heap_cap) {
  surf_pt best;
  best.face = -1;
  best.dist_sq = isinf(max_dist) ? max_dist : max_dist * max_dist;
  best.point = mk3(0, 0, 0);
  best.bary = mk3(0, 0, 0);
  heap_e* h = *heap_buf;
  int n = 0;
  h[n++] = (heap_e){box_dist_sq(&b->nodes[0], q), 0};
  while (n > 0) {
    heap_e top = h[0];
    h[0] = h[--n];
    for (int i = 0;;) { /* sift down */
      int l = 2 * i + 1, r = l + 1, s = i;
      if (l < n && he_less(h[l], h[s])) s = l;
      if (r < n && he_less(h[r], h[s])) s = r;
      if (s == i) break;
      heap_e t = h[i];
      h[i] = h[s];
      h[s] = t;
      i = s;
    }
    if (top.d > best.dist_sq) break;
    const bnode* nd = &b->nodes[top.i];
    if (nd->count > 0) {
      for (int i = 0; i < nd->count; ++i) test_face_closest(b->m, b->order[nd->first + i], q, &best);
      continue;
    }
    int kids[2] = {nd->left, nd->right};
    for (int c = 0; c < 2; ++c) {
      if (n + 1 > *heap_cap) {
        *heap_cap *= 2;
        *heap_buf = h = (heap_e*)realloc(h, sizeof(heap_e) * (size_t)*heap_cap);
      }
      heap_e e = {box_dist_sq(&b->nodes[kids[c]], q), kids[c]};
      int i = n++;
      h[i] = e;
      while (i > 0) { /* sift up */
        int p = (i - 1) / 2;
        if (!he_less(h[i], h[p])) break;
        heap_e t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
      }
    }
  }
  if (best.face < 0) best.dist_sq = INFINITY;
  return best;
}

/* ---- transferNormals, bake/gbuffer.cpp:193-252 ----------------------------- */
static inline uint8_t encode_channel(double v) {
  long q = lround((v + 1.0) * 0.5 * 255.0);
  return (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q));
}

typedef struct {
  int res;
  const float *pos, *nrm, *tan, *bit;
  const uint8_t *valid, *rel;
  const mf_mesh_view* hi;
  const double* hiN;
  const bvh_t* bvh;
  double max_dist;
  uint8_t* rgb;
  int32_t* dbg_face;
  double* dbg_ts;
} xfer_ctx;

static void xfer_range(void* vctx, int64_t lo, int64_t hi) {
  xfer_ctx* c = (xfer_ctx*)vctx;
  int cap = 256;
  heap_e* heap = (heap_e*)malloc(sizeof(heap_e) * (size_t)cap);
  for (int64_t t = lo; t < hi; ++t) {
    int32_t face = -1;
    double ts3[3] = {0, 0, 0};
    if (!c->valid[t]) goto done;
    uint8_t* px = c->rgb + 3 * t;
    if (!c->rel[t]) {
      face = -2;
      px[0] = 128, px[1] = 128, px[2] = 255;
      goto done;
    }
    d3 q = mk3((double)c->pos[3 * t], (double)c->pos[3 * t + 1], (double)c->pos[3 * t + 2]);
    surf_pt hit = bvh_closest_within(c->bvh, q, c->max_dist, &heap, &cap);
    if (hit.face < 0) {
      face = -3;
      px[0] = 128, px[1] = 128, px[2] = 255;
      goto done;
    }
    face = hit.face;
    {
      const int* tri = c->hi->faces + 3 * (size_t)hit.face;
      d3 n = add3(add3(scl3(hit.bary.v[0], ld3(c->hiN + 3 * (size_t)tri[0])),
                       scl3(hit.bary.v[1], ld3(c->hiN + 3 * (size_t)tri[1]))),
                  scl3(hit.bary.v[2], ld3(c->hiN + 3 * (size_t)tri[2])));
      d3 T = mk3(c->tan[3 * t], c->tan[3 * t + 1], c->tan[3 * t + 2]);
      d3 B = mk3(c->bit[3 * t], c->bit[3 * t + 1], c->bit[3 * t + 2]);
      d3 N = mk3(c->nrm[3 * t], c->nrm[3 * t + 1], c->nrm[3 * t + 2]);
      d3 ts = mk3(dot3(n, T), dot3(n, B), dot3(n, N));
      double len = nrm3(ts);
      if (len < 1e-12) {
        px[0] = 128, px[1] = 128, px[2] = 255;
        goto done;
      }
      ts = div3(ts, len);
      for (int k = 0; k < 3; ++k) {
        px[k] = encode_channel(ts.v[k]);
        ts3[k] = ts.v[k];
      }
    }
  done:
    if (c->dbg_face) c->dbg_face[t] = face;
    if (c->dbg_ts) memcpy(c->dbg_ts + 3 * t, ts3, 24);
  }
  free(heap);
}

int orc_transfer_normals(int res, const float* pos, const float* nrm, const float* tan,
                         const float* bit, const uint8_t* valid, const uint8_t* rel,
                         const mf_mesh_view* hi, double diag, double frac, uint8_t* rgb,
                         int32_t* dbg_face, double* dbg_ts, int threads) {
  if (res < 1 || !valid) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: g-buffer is empty");
  int rc = validate_mesh(hi);
  if (rc) return rc;
  if (!(diag > 0.0) || !(frac > 0.0))
    return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: distance filter must be positive");
  double* hiN = unit_normals(hi);
  bvh_t bvh;
  bvh_build(&bvh, hi);
  const int64_t texels = (int64_t)res * res;
  memset(rgb, 128, (size_t)texels * 3);
  xfer_ctx c = {res, pos, nrm, tan, bit, valid, rel, hi, hiN, &bvh, frac * diag, rgb, dbg_face, dbg_ts};
  parallel_for(texels, 4096, threads, xfer_range, &c);
  bvh_free(&bvh);
  free(hiN);
  return 0;
}

/* ---- dilateSeams, bake/gbuffer.cpp:254-322 --------------------------------- */
int orc_dilate_seams(int w, int h, int ch, const uint8_t* map, int gres, const uint8_t* valid,
                     int radius, uint8_t* out) {
  if (radius < 0) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilation radius must be >= 0");
  if (w != gres || h != gres)
    return fail(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: map and g-buffer resolutions differ");
  memcpy(out, map, (size_t)w * h * ch);
  if (radius == 0) return 0;
  const int res = gres;
  const size_t texels = (size_t)res * res;
  const int64_t none = INT64_MAX;
  int32_t* sx = (int32_t*)calloc(texels * 2, sizeof(int32_t));
  int64_t* d2 = (int64_t*)malloc(texels * sizeof(int64_t));
  for (size_t t = 0; t < texels; ++t) {
    d2[t] = none;
    if (valid[t]) {
      sx[2 * t] = (int32_t)(t % res);
      sx[2 * t + 1] = (int32_t)(t / res);
      d2[t] = 0;
    }
  }
  int32_t* nsx = (int32_t*)malloc(texels * 2 * sizeof(int32_t));
  int64_t* nd2 = (int64_t*)malloc(texels * sizeof(int64_t));
  memcpy(nsx, sx, texels * 2 * sizeof(int32_t));
  memcpy(nd2, d2, texels * sizeof(int64_t));
  for (int pass = 0; pass < radius; ++pass) {
    for (int y = 0; y < res; ++y) {
      for (int x = 0; x < res; ++x) {
        const size_t t = (size_t)y * res + x;
        if (d2[t] == 0) continue;
        int64_t best = d2[t];
        int32_t bx = sx[2 * t], by = sx[2 * t + 1];
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy) continue;
            const int nx = x + dx, ny = y + dy;
            if (nx < 0 || nx >= res || ny < 0 || ny >= res) continue;
            const size_t nt = (size_t)ny * res + nx;
            if (d2[nt] == none) continue;
            const int32_t s0 = sx[2 * nt], s1 = sx[2 * nt + 1];
            const int64_t d = (int64_t)(x - s0) * (x - s0) + (int64_t)(y - s1) * (y - s1);
            if (d < best) {
              best = d;
              bx = s0;
              by = s1;
            }
          }
        nd2[t] = best;
        nsx[2 * t] = bx;
        nsx[2 * t + 1] = by;
      }
    }
    int32_t* ts = sx;
    sx = nsx;
    nsx = ts;
    int64_t* td = d2;
    d2 = nd2;
    nd2 = td;
  }
  for (int y = 0; y < res; ++y)
    for (int x = 0; x < res; ++x) {
      const size_t t = (size_t)y * res + x;
      if (valid[t] || d2[t] == none) continue;
      const size_t s = ((size_t)sx[2 * t + 1] * w + sx[2 * t]) * ch;
      for (int c = 0; c < ch; ++c) out[t * ch + c] = map[s + c];
    }
  free(sx);
  free(d2);
  free(nsx);
  free(nd2);
  return 0;
}

int orc_bake(const mf_mesh_view* lo, const mf_mesh_view* hi, int res, double diag, double frac,
             int radius, uint8_t* rgb, uint8_t* rgb_raw, int32_t* dbg_face, double* dbg_ts,
             int threads, int64_t* n_valid, int64_t* n_queries) {
  if (res < 1) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: resolution must be >= 1");
  const size_t texels = (size_t)res * res;
  float* g = (float*)malloc(texels * 12 * 4);
  uint8_t* v = (uint8_t*)malloc(texels * 2);
  uint8_t* raw = rgb_raw ? rgb_raw : (uint8_t*)malloc(texels * 3);
  int rc = orc_raster_gbuffer(lo, res, g, g + texels * 3, g + texels * 6, g + texels * 9, v, v + texels);
  if (!rc)
    rc = orc_transfer_normals(res, g, g + texels * 3, g + texels * 6, g + texels * 9, v, v + texels,
                              hi, diag, frac, raw, dbg_face, dbg_ts, threads);
  if (!rc) rc = orc_dilate_seams(res, res, 3, raw, res, v, radius, rgb);
  if (!rc) {
    int64_t nv = 0, nq = 0;
    for (size_t t = 0; t < texels; ++t) {
      nv += v[t];
      nq += v[t] && v[texels + t];
    }
    if (n_valid) *n_valid = nv;
    if (n_queries) *n_queries = nq;
  }
  free(g);
  free(v);
  if (!rgb_raw) free(raw);
  return rc;
}

/* ---- bulk closest point / ray cast (spatial/bvh.cpp:100-189) --------------- */
typedef struct {
  const mf_mesh_view* m;
  const bvh_t* bvh;
  const double* q;
  double max_dist;
  int brute;
  int32_t* face;
  double *dist_sq, *point, *bary;
} cp_ctx;
static void cp_range(void* vctx, int64_t lo, int64_t hi) {
  cp_ctx* c = (cp_ctx*)vctx;
  int cap = 256;
  heap_e* heap = (heap_e*)malloc(sizeof(heap_e) * (size_t)cap);
  for (int64_t i = lo; i < hi; ++i) {
    d3 q = ld3(c->q + 3 * i);
    surf_pt sp;
    if (c->brute) {
      sp.face = -1;
      sp.dist_sq = INFINITY;
      sp.point = sp.bary = mk3(0, 0, 0);
      for (int f = 0; f < c->m->n_faces; ++f) test_face_closest(c->m, f, q, &sp);
    } else {
      sp = bvh_closest_within(c->bvh, q, c->max_dist, &heap, &cap);
    }
    c->face[i] = sp.face;
    c->dist_sq[i] = sp.dist_sq;
    if (c->point) memcpy(c->point + 3 * i, sp.point.v, 24);
    if (c->bary) memcpy(c->bary + 3 * i, sp.bary.v, 24);
  }
  free(heap);
}
int orc_closest_within(const mf_mesh_view* m, const double* q, int64_t n, double max_dist,
                       int brute, int threads, int32_t* face, double* dist_sq, double* point,
                       double* bary) {
  int rc = validate_mesh(m);
  if (rc) return rc;
  bvh_t bvh;
  bvh_build(&bvh, m);
  cp_ctx c = {m, &bvh, q, max_dist, brute, face, dist_sq, point, bary};
  parallel_for(n, 256, threads, cp_range, &c);
  bvh_free(&bvh);
  return 0;
}

/* spatial/tri_geom.h:14-33 Moller-Trumbore */
static int ray_triangle(d3 o, d3 d, d3 a, d3 b, d3 c, double* t, double* u, double* v) {
  d3 e1 = sub3(b, a), e2 = sub3(c, a);
  d3 pv = cross3(d, e2);
  double det = dot3(e1, pv);
  if (fabs(det) < 1e-9) return 0;
  double inv = 1.0 / det;
  d3 sv = sub3(o, a);
  *u = dot3(sv, pv) * inv;
  if (*u < 0.0 || *u > 1.0) return 0;
  d3 qv = cross3(sv, e1);
  *v = dot3(d, qv) * inv;
  if (*v < 0.0 || *u + *v > 1.0) return 0;
  *t = dot3(e2, qv) * inv;
  return 1;
}
typedef struct {
  int face;
  double t, u, v;
} ray_hit;
/* bvh.cpp:25-34 testFace */
static inline void test_face(const mf_mesh_view* m, int f, d3 o, d3 d, double tmin, double tmax,
                             ray_hit* best) {
  double t, u, v;
  if (ray_triangle(o, d, P(m, FV(m, f, 0)), P(m, FV(m, f, 1)), P(m, FV(m, f, 2)), &t, &u, &v) &&
      t >= tmin && t <= tmax && (t < best->t || (t == best->t && f < best->face))) {
    best->face = f;
    best->t = t;
    best->u = u;
    best->v = v;
  }
}
/* core/aabb.h:45-56 */
static inline int box_ray(const bnode* nd, d3 o, d3 inv, double tmin, double tmax, double* tnear) {
  for (int a = 0; a < 3; ++a) {
    double t0 = (nd->mn[a] - o.v[a]) * inv.v[a];
    double t1 = (nd->mx[a] - o.v[a]) * inv.v[a];
    if (inv.v[a] < 0.0) {
      double s = t0;
      t0 = t1;
      t1 = s;
    }
    tmin = t0 > tmin ? t0 : tmin;
    tmax = t1 < tmax ? t1 : tmax;
    if (tmax < tmin) return 0;
  }
  *tnear = tmin;
  return 1;
}
/* bvh.cpp:100-140 */
static ray_hit bvh_raycast(const bvh_t* b, d3 o, d3 d, double tmin, double tmax) {
  ray_hit best = {-1, INFINITY, 0, 0};
  d3 inv = mk3(1.0 / d.v[0], 1.0 / d.v[1], 1.0 / d.v[2]);
  int stack[66], top = 0;
  stack[top++] = 0;
  while (top > 0) {
    const bnode* nd = &b->nodes[stack[--top]];
    double tn, limit = tmax < best.t ? tmax : best.t;
    if (!box_ray(nd, o, inv, tmin, limit, &tn)) continue;
    if (nd->count > 0) {
      for (int i = 0; i < nd->count; ++i) test_face(b->m, b->order[nd->first + i], o, d, tmin, tmax, &best);
      continue;
    }
    double tl, tr;
    int hl = box_ray(&b->nodes[nd->left], o, inv, tmin, limit, &tl);
    int hr = box_ray(&b->nodes[nd->right], o, inv, tmin, limit, &tr);
    if (hl && hr) {
      if (tl <= tr) {
        stack[top++] = nd->right;
        stack[top++] = nd->left;
      } else {
        stack[top++] = nd->left;
        stack[top++] = nd->right;
      }
    } else if (hl) {
      stack[top++] = nd->left;
    } else if (hr) {
      stack[top++] = nd->right;
    }
  }
  return best;
}
typedef struct {
  const mf_mesh_view* m;
  const bvh_t* bvh;
  const double *o, *d;
  double tmin, tmax;
  int brute;
  int32_t* face;
  double *t, *u, *v;
} rc_ctx;
static void rc_range(void* vctx, int64_t lo, int64_t hi) {
  rc_ctx* c = (rc_ctx*)vctx;
  for (int64_t i = lo; i < hi; ++i) {
    d3 o = ld3(c->o + 3 * i), d = ld3(c->d + 3 * i);
    ray_hit h;
    if (c->brute) {
      h = (ray_hit){-1, INFINITY, 0, 0};
      for (int f = 0; f < c->m->n_faces; ++f) test_face(c->m, f, o, d, c->tmin, c->tmax, &h);
    } else {
      h = bvh_raycast(c->bvh, o, d, c->tmin, c->tmax);
    }
    c->face[i] = h.face;
    c->t[i] = h.t;
    c->u[i] = h.u;
    c->v[i] = h.v;
  }
}
int orc_raycast_first(const mf_mesh_view* m, const double* o, const double* d, int64_t n,
                      double tmin, double tmax, int brute, int threads, int32_t* face, double* t,
                      double* u, double* v) {
  int rc = validate_mesh(m);
  if (rc) return rc;
  bvh_t bvh;
  bvh_build(&bvh, m);
  rc_ctx c = {m, &bvh, o, d, tmin, tmax, brute, face, t, u, v};
  parallel_for(n, 256, threads, rc_range, &c);
  bvh_free(&bvh);
  return 0;
}

/* ---------------------------------------------------------------- surface band
 * signfield/sign_grid.cpp:23-69 markSurfaceBand: grid parameters (:24-52),
 * then closestPointWithin(voxelCenter, truncation) per voxel (:56-66);
 * voxelCenter = origin + voxelSize * (x + 0.5, y + 0.5, z + 0.5)
 * (sign_grid.h:30-32); index x-fastest (:27-29). */
typedef struct {
  const bvh_t* bvh;
  int res;
  double o[3], h, trunc, band;
  uint8_t* labels;
  float* dist;
} band_ctx;
static void band_range(void* vctx, int64_t lo, int64_t hi) {
  band_ctx* c = (band_ctx*)vctx;
  int cap = 256;
  heap_e* heap = (heap_e*)malloc(sizeof(heap_e) * (size_t)cap);
  const int64_t r = c->res;
  for (int64_t i = lo; i < hi; ++i) {
    const int x = (int)(i % r), y = (int)((i / r) % r), z = (int)(i / (r * r));
    d3 q = mk3(c->o[0] + c->h * (x + 0.5), c->o[1] + c->h * (y + 0.5), c->o[2] + c->h * (z + 0.5));
    surf_pt sp = bvh_closest_within(c->bvh, q, c->trunc, &heap, &cap);
    c->labels[i] = 0;
    c->dist[i] = (float)c->trunc;
    if (sp.face >= 0) {
      const double d = sqrt(sp.dist_sq);
      c->dist[i] = (float)d;
      if (d < c->band) c->labels[i] = 1;
    }
  }
  free(heap);
}
int orc_surface_band(const mf_mesh_view* m, int res, double band_voxels, int dilate, const double* domain,
                     int threads, uint8_t* labels, float* dist, double* grid_out) {
  int rc = validate_mesh(m); /* Bvh(mesh) validates (bvh.cpp:48-50) */
  if (rc) return rc;
  if (res < 8) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: grid resolution must be >= 8");
  if (dilate < 0) return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilate radius must be >= 0");
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = 0; v < m->n_vertices; ++v)
    for (int k = 0; k < 3; ++k) {
      const double p = m->positions[3 * v + k];
      mn[k] = p < mn[k] ? p : mn[k];
      mx[k] = mx[k] < p ? p : mx[k];
    }
  const int margin = dilate + 3;
  if (res - 2 * margin < 4)
    return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: grid resolution too small for the dilation margin");
  band_ctx c;
  double ext[3];
  if (domain) {
    for (int k = 0; k < 3; ++k) ext[k] = domain[3 + k] - domain[k];
  } else {
    for (int k = 0; k < 3; ++k) ext[k] = mx[k] - mn[k];
  }
  double e = ext[0];
  for (int k = 1; k < 3; ++k)
    if (ext[k] > e) e = ext[k];
  if (domain) {
    c.h = e / res;
    for (int k = 0; k < 3; ++k) c.o[k] = domain[k];
  } else {
    const double usable = res - 2.0 * margin;
    c.h = e / usable;
    const double half = 0.5 * res * c.h;
    for (int k = 0; k < 3; ++k) c.o[k] = (mn[k] + mx[k]) * 0.5 - half;
  }
  for (int k = 0; k < 3; ++k)
    if (mn[k] < c.o[k] + 2 * c.h || mx[k] > c.o[k] + (res - 2.0) * c.h)
      return fail(MF_ERR_OUT_OF_BOUNDS, "OutOfBounds: mesh does not fit in the grid with 2 voxels of margin");
  c.trunc = (band_voxels + dilate * sqrt(3.0) + 2.0) * c.h;
  c.band = band_voxels * c.h;
  c.res = res;
  c.labels = labels;
  c.dist = dist;
  bvh_t bvh;
  bvh_build(&bvh, m);
  c.bvh = &bvh;
  parallel_for((int64_t)res * res * res, 4096, threads, band_range, &c);
  bvh_free(&bvh);
  if (grid_out) {
    for (int k = 0; k < 3; ++k) grid_out[k] = c.o[k];
    grid_out[3] = c.h;
    grid_out[4] = c.trunc;
  }
  return 0;
}

/* ---------------------------------------------------------------- ortho views
 * render/camera.cpp:38-55 fibonacciCameras -> cams7 (direction, up, halfExtent). */
void orc_fibonacci_cameras(int count, double half_extent, double* cams7) {
  const double golden = M_PI * (3.0 - sqrt(5.0));
  for (int i = 0; i < count; ++i) {
    const double z = 1.0 - 2.0 * (i + 0.5) / count;
    const double r = sqrt(fmax(0.0, 1.0 - z * z));
    const double a = golden * i;
    const d3 dir = mk3(-(r * cos(a)), -(r * sin(a)), -z);
    const d3 ref = fabs(z) < 0.9 ? mk3(0, 0, 1) : mk3(0, 1, 0);
    d3 up = cross3(dir, ref);
    const double z2 = sqn3(up);
    if (z2 > 0.0) up = div3(up, sqrt(z2));
    double* c = cams7 + 7 * i;
    for (int k = 0; k < 3; ++k) {
      c[k] = dir.v[k];
      c[3 + k] = up.v[k];
    }
    c[6] = half_extent;
  }
}

/* render/raster.cpp:12-102 renderView, face by face in index order over the
 * padded pixel box, Moller-Trumbore with the hoisted per-face factors, z-test
 * "replace iff depth > stored" (ties keep the lower face). Outputs nullable
 * except face/depth scratch. */
static void render_view(const mf_mesh_view* m, const double* vn, const double* cam7, int res, int cull,
                        int32_t* face, float* depth, float* pos, float* nrm) {
  const d3 dir = ld3(cam7), up = ld3(cam7 + 3);
  const d3 right = cross3(dir, up);
  const double he = cam7[6];
  const double step = 2.0 * he / res;
  const size_t n = (size_t)res * res;
  for (size_t i = 0; i < n; ++i) {
    face[i] = -1;
    depth[i] = INFINITY;
    if (pos) pos[3 * i] = pos[3 * i + 1] = pos[3 * i + 2] = 0.f;
    if (nrm) nrm[3 * i] = nrm[3 * i + 1] = nrm[3 * i + 2] = 0.f;
  }
  d3* colU = (d3*)malloc(sizeof(d3) * (size_t)res);
  d3* rowV = (d3*)malloc(sizeof(d3) * (size_t)res);
  for (int p = 0; p < res; ++p) {
    const double pu = -he + (p + 0.5) * (2.0 * he / res); /* camera.h:22-27 */
    const double pv = he - (p + 0.5) * (2.0 * he / res);
    colU[p] = scl3(pu, right);
    rowV[p] = scl3(pv, up);
  }
  for (int f = 0; f < m->n_faces; ++f) {
    const int* tri = m->faces + 3 * (size_t)f;
    const d3 a = P(m, tri[0]), b = P(m, tri[1]), c = P(m, tri[2]);
    if (cull && dot3(cross3(sub3(b, a), sub3(c, a)), dir) > 0.0) continue; /* raster.cpp:44 */
    const double u0 = dot3(a, right), u1 = dot3(b, right), u2 = dot3(c, right);
    const double v0 = dot3(a, up), v1 = dot3(b, up), v2 = dot3(c, up);
    const double umin = fmin(u0, fmin(u1, u2)), umax = fmax(u0, fmax(u1, u2));
    const double vmin = fmin(v0, fmin(v1, v2)), vmax = fmax(v0, fmax(v1, v2));
    int pxLo = (int)floor((umin + he) / step - 0.5) - 1;
    int pxHi = (int)ceil((umax + he) / step - 0.5) + 1;
    int pyLo = (int)floor((he - vmax) / step - 0.5) - 1;
    int pyHi = (int)ceil((he - vmin) / step - 0.5) + 1;
    if (pxLo < 0) pxLo = 0;
    if (pyLo < 0) pyLo = 0;
    if (pxHi > res - 1) pxHi = res - 1;
    if (pyHi > res - 1) pyHi = res - 1;
    if (pxLo > pxHi || pyLo > pyHi) continue;
    const d3 e1 = sub3(b, a), e2 = sub3(c, a);
    const d3 pvec = cross3(dir, e2);
    const double det = dot3(e1, pvec);
    if (fabs(det) < 1e-9) continue;
    const double invDet = 1.0 / det;
    for (int py = pyLo; py <= pyHi; ++py)
      for (int px = pxLo; px <= pxHi; ++px) {
        const d3 origin = add3(colU[px], rowV[py]);
        const d3 svec = sub3(origin, a);
        const double bu = dot3(svec, pvec) * invDet;
        if (bu < 0.0 || bu > 1.0) continue;
        const d3 qvec = cross3(svec, e1);
        const double bv = dot3(dir, qvec) * invDet;
        if (bv < 0.0 || bu + bv > 1.0) continue;
        const double t = dot3(e2, qvec) * invDet;
        const float dp = (float)(-t);
        const size_t idx = (size_t)py * res + px;
        if (face[idx] >= 0 && !(dp > depth[idx])) continue;
        face[idx] = f;
        depth[idx] = dp;
        if (pos) {
          const d3 hit = add3(origin, scl3(t, dir));
          for (int k = 0; k < 3; ++k) pos[3 * idx + k] = (float)hit.v[k];
        }
        if (nrm && vn) {
          d3 nn = add3(add3(scl3(1.0 - bu - bv, ld3(vn + 3 * (size_t)tri[0])), scl3(bu, ld3(vn + 3 * (size_t)tri[1]))),
                       scl3(bv, ld3(vn + 3 * (size_t)tri[2])));
          const double len = nrm3(nn);
          if (len > 0) nn = div3(nn, len);
          for (int k = 0; k < 3; ++k) nrm[3 * idx + k] = (float)nn.v[k];
        }
      }
  }
  free(colU);
  free(rowV);
}

int orc_render_views(const mf_mesh_view* m, const double* cams7, int n_views, int res, const double* vn, int cull,
                     int32_t* face, float* depth, float* pos, float* nrm) {
  const size_t n = (size_t)res * res;
  for (int v = 0; v < n_views; ++v)
    render_view(m, vn, cams7 + 7 * v, res, cull, face + v * n, depth + v * n, pos ? pos + 3 * v * n : NULL,
                nrm ? nrm + 3 * v * n : NULL);
  return 0;
}

/* visibility/visibility.cpp:13-59 castVisibility: validate, centre on the
 * bounds, radius = max |p - centre| (1 if 0), fibonacci cameras of half
 * extent radius * 1.04, per view renderView, won pixels per face. */
int orc_cast_visibility(const mf_mesh_view* m, int viewpoints, int res, int64_t* hits) {
  int rc = validate_mesh(m);
  if (rc) return rc;
  if (viewpoints <= 0 || res <= 0)
    return fail(MF_ERR_INVALID_CONFIG, "InvalidConfig: viewpoints and resolution must be positive");
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = 0; v < m->n_vertices; ++v)
    for (int k = 0; k < 3; ++k) {
      const double p = m->positions[3 * v + k];
      mn[k] = p < mn[k] ? p : mn[k];
      mx[k] = mx[k] < p ? p : mx[k];
    }
  const d3 center = mk3((mn[0] + mx[0]) * 0.5, (mn[1] + mx[1]) * 0.5, (mn[2] + mx[2]) * 0.5);
  double* cpos = (double*)malloc(sizeof(double) * 3 * (size_t)m->n_vertices);
  double radius = 0.0;
  for (int v = 0; v < m->n_vertices; ++v) {
    const d3 p = sub3(P(m, v), center);
    memcpy(cpos + 3 * (size_t)v, p.v, 24);
    const double nn = nrm3(p);
    radius = radius < nn ? nn : radius;
  }
  if (radius <= 0.0) radius = 1.0;
  mf_mesh_view cm = *m;
  cm.positions = cpos;
  double* cams = (double*)malloc(sizeof(double) * 7 * (size_t)viewpoints);
  orc_fibonacci_cameras(viewpoints, radius * 1.04, cams);
  const size_t n = (size_t)res * res;
  int32_t* face = (int32_t*)malloc(sizeof(int32_t) * n);
  float* depth = (float*)malloc(sizeof(float) * n);
  memset(hits, 0, sizeof(int64_t) * (size_t)m->n_faces);
  for (int v = 0; v < viewpoints; ++v) {
    render_view(&cm, NULL, cams + 7 * v, res, 0, face, depth, NULL, NULL);
    for (size_t i = 0; i < n; ++i)
      if (face[i] >= 0) ++hits[face[i]];
  }
  free(face);
  free(depth);
  free(cams);
  free(cpos);
  return 0;
}
