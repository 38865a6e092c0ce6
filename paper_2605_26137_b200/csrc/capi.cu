// capi.cu — the extern "C" boundary of libmfbake (include/mfbake.h).
//
// Orchestration of the fused bake (mf_bake_normal_map[_dev]):
//   main stream : prepare_lowpoly (normals, wedge frames, reliability, face
//                 setup) -> raster G-buffer slab            [rasterizeGBuffer]
//   side stream : dense vertex normals -> LBVH build        [transferNormals
//                                                            :201-208]
//   join        : transfer (closest point + encode)         [:215-250]
//                 -> dilation                               [dilateSeams]
// Meshes are validated on the device at upload (validateMesh,
// core/mesh.cpp:37-48, plus face_uvs range); errors are reported in the
// reference's throw order.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "bake.cuh"
#include "host_pool.h"


namespace mfb {

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

void* Ctx::buf(const std::string& name, size_t bytes) {
  Buf& b = scratch[name];
  if (b.bytes < bytes) {
    if (capturing) throw CaptureRealloc{};
    if (b.ptr) {
      // the streams may still use the old buffer; free after they drain
      sync_all();
      MFB_CUDA_TRY(cudaFree(b.ptr));
      b.ptr = nullptr;
    }
    const size_t want = std::max(bytes, b.bytes + b.bytes / 4);
    ++alloc_gen;
    cudaError_t e = cudaMalloc(&b.ptr, want);
    if (e == cudaErrorMemoryAllocation) {
      (void)cudaGetLastError();
      throw std::bad_alloc();
    }
    MFB_CUDA_TRY(e);
    b.bytes = want;
  }
  return b.ptr;
}
void* Ctx::host_buf(const std::string& name, size_t bytes) {
  Buf& b = pinned[name];
  if (b.bytes < bytes) {
    if (capturing) throw CaptureRealloc{};
    if (b.ptr) {
      MFB_CUDA_TRY(cudaStreamSynchronize(stream));
      MFB_CUDA_TRY(cudaFreeHost(b.ptr));
    }
    ++alloc_gen;
    MFB_CUDA_TRY(cudaMallocHost(&b.ptr, bytes));
    b.bytes = bytes;
  }
  return b.ptr;
}
void Ctx::sync_all() {
  MFB_CUDA_TRY(cudaStreamSynchronize(stream));
  if (side) MFB_CUDA_TRY(cudaStreamSynchronize(side));
  if (aux) MFB_CUDA_TRY(cudaStreamSynchronize(aux));
  if (side2) MFB_CUDA_TRY(cudaStreamSynchronize(side2));
  if (aux2) MFB_CUDA_TRY(cudaStreamSynchronize(aux2));
  if (lowhi) MFB_CUDA_TRY(cudaStreamSynchronize(lowhi));
  if (dn) MFB_CUDA_TRY(cudaStreamSynchronize(dn));
  if (up1) MFB_CUDA_TRY(cudaStreamSynchronize(up1));
  if (up2) MFB_CUDA_TRY(cudaStreamSynchronize(up2));
}
void* Ctx::cub_temp(size_t bytes, cudaStream_t s) {
  const int slot = s == side    ? 1
                   : s == aux   ? 2
                   : s == aux2  ? 3
                   : s == side2 ? 4
                   : s == lowhi ? 5
                   : s == dn    ? 6
                                : 0;
  void*& p = cub_tmp[slot];
  size_t& n = cub_tmp_bytes[slot];
  if (n < bytes) {
    if (capturing) throw CaptureRealloc{};
    if (p) {
      sync_all();
      MFB_CUDA_TRY(cudaFree(p));
    }
    const size_t want = std::max<size_t>(bytes, 1 << 20);
    ++alloc_gen;
    MFB_CUDA_TRY(cudaMalloc(&p, want));
    n = want;
  }
  return p;
}
cudaEvent_t Ctx::pool_event(int i) {
  while (static_cast<int>(ev_pool.size()) <= i) {
    cudaEvent_t e;
    MFB_CUDA_TRY(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  return ev_pool[i];
}

namespace {
__global__ void k_fill(uint32_t* __restrict__ w, size_t nw, uint32_t v, uint8_t* __restrict__ tail, int ntail) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nw; i += stride) w[i] = v;
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < ntail) tail[threadIdx.x] = static_cast<uint8_t>(v);
}
// After the transfer: the bake's flags and counters and the dense mesh's
// validation flag stored straight into the pinned host words (UVA: a
// cudaMallocHost pointer is a device pointer), and every band's ready flag
// released - one launch in place of a fill and three small copies, each of
// which costs a copy-engine round trip on the tail of the bake.
__global__ void k_finish(const int* __restrict__ flags, const unsigned long long* __restrict__ counters,
                         const int* __restrict__ dense_vflags, int* hflags, unsigned long long* hcnt,
                         int* dense_hflag, int* ready, int nb) {
  const int t = threadIdx.x;
  if (t < 4) hflags[t] = flags[t];
  else if (t < 8) hcnt[t - 4] = counters[t - 4];
  else if (t == 8 && dense_vflags) *dense_hflag = *dense_vflags;
  for (int b = t; b < nb; b += blockDim.x) ready[b] = 1;
}
}  // namespace

void finish_flags(Ctx& c, cudaStream_t s, const int* flags, const unsigned long long* counters,
                  const int* dense_vflags, int* hflags, unsigned long long* hcnt, int* dense_hflag, int* ready,
                  int nb) {
  k_finish<<<1, 64, 0, s>>>(flags, counters, dense_vflags, hflags, hcnt, dense_hflag, ready, nb);
  c.count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

void Ctx::fill(void* p, int value, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  // scratch buffers are 256-byte aligned: whole words, then the byte tail
  if (reinterpret_cast<uintptr_t>(p) & 3) {
    MFB_CUDA_TRY(cudaMemsetAsync(p, value, bytes, s));
    return;
  }
  const uint32_t b = static_cast<uint8_t>(value);
  const uint32_t v = b | (b << 8) | (b << 16) | (b << 24);
  const size_t nw = bytes / 4;
  const int ntail = static_cast<int>(bytes - 4 * nw);
  const int grid = static_cast<int>(std::min<size_t>(std::max<size_t>(1, (nw + 255) / 256), kNumSMs * 4));
  k_fill<<<grid, 256, 0, s>>>(static_cast<uint32_t*>(p), nw, v, static_cast<uint8_t*>(p) + 4 * nw, ntail);
  count_launch();
  MFB_CUDA_TRY(cudaGetLastError());
}

HostPool& Ctx::host_pool() {
  if (!pool) {
    const unsigned hw = std::thread::hardware_concurrency();
    const char* e = std::getenv("MFB_HOST_THREADS");
    const int want = e ? std::atoi(e) : 0;
    // (MFB_HOST_THREADS overrides) 5 on the 16-core box: pageable e2e at config
    // B 2.08 ms with 5 threads, 2.09-2.17 with 4, 2.12-2.25 with 8, 2.43-2.50
    // with 12-16 (the staging copies contend for host memory bandwidth)
    pool = new HostPool(want > 0 ? want : static_cast<int>(std::min(5u, std::max(2u, hw / 3))));
  }
  return *pool;
}

void Ctx::invalidate_graphs() {
  if (bake_exec) cudaGraphExecDestroy(bake_exec);
  bake_exec = nullptr;
  bake_key.clear();
  bake_prev_key.clear();
  for (GraphSlot* g : {&g_low, &g_dense}) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    g->exec = nullptr;
    g->key.clear();
    g->prev_key.clear();
  }
}

Ctx::~Ctx() {
  cudaSetDevice(device);
  delete pool;  // idle: every entry point waits for its pool job
  if (bake_exec) cudaGraphExecDestroy(bake_exec);
  for (GraphSlot* g : {&g_low, &g_dense})
    if (g->exec) cudaGraphExecDestroy(g->exec);
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (stream) cudaStreamSynchronize(stream);
  if (side) cudaStreamSynchronize(side);
  if (aux) cudaStreamSynchronize(aux);
  if (side2) cudaStreamSynchronize(side2);
  if (aux2) cudaStreamSynchronize(aux2);
  if (lowhi) cudaStreamSynchronize(lowhi);
  if (dn) cudaStreamSynchronize(dn);
  if (up1) cudaStreamSynchronize(up1);
  if (up2) cudaStreamSynchronize(up2);
  for (auto& kv : scratch) cudaFree(kv.second.ptr);
  for (auto& kv : pinned) cudaFreeHost(kv.second.ptr);
  for (void* p : cub_tmp)
    if (p) cudaFree(p);
  for (cudaEvent_t e : {fork, join, fork2, join2, join3, hi_ready, dfork, djoin, up_fork, up_join, lfork, ljoin, setup_done, join4, lowfork, lowjoin, up1_done, up2_done})
    if (e) cudaEventDestroy(e);
  if (up1) cudaStreamDestroy(up1);
  if (up2) cudaStreamDestroy(up2);
  if (side) cudaStreamDestroy(side);
  if (aux) cudaStreamDestroy(aux);
  if (side2) cudaStreamDestroy(side2);
  if (aux2) cudaStreamDestroy(aux2);
  if (lowhi) cudaStreamDestroy(lowhi);
  if (dn) cudaStreamDestroy(dn);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

namespace {

// ---------------------------------------------------------------- validation
// flags: 1 = non-finite position, 2 = face index out of range,
//        4 = face_uv index out of range (superset of the reference)
// Out-of-range indices are also replaced by 0 in the device copy (nv, nu > 0
// when a mesh is used): a bake launched before the host has read the flags
// (bake_host_overlapped's speculative dense phase) then never indexes out of
// bounds, and its result is discarded for the validation error.
__global__ void k_validate(const double* __restrict__ pos, int nv, int32_t* __restrict__ faces, int nf,
                           int32_t* __restrict__ fuv, int nu, int* flags) {
  int f = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < 3ll * nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(pos[i])) f |= 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < 3ll * nf;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = faces[i];
    if (v < 0 || v >= nv) {
      f |= 2;
      faces[i] = 0;
    }
    if (fuv) {
      const int u = fuv[i];
      if (u < 0 || u >= nu) {
        f |= 4;
        fuv[i] = 0;
      }
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

}  // namespace
}  // namespace mfb

using namespace mfb;

struct mf_ctx {
  Ctx c;
  std::vector<std::pair<void*, void*>> ipc_bases;  // (user pointer, opened base) of mf_ipc_open
  ~mf_ctx() {
    for (auto& b : ipc_bases) cudaIpcCloseMemHandle(b.second);
  }
};

struct mf_mesh {
  mf_ctx* ctx = nullptr;  // the creating context (not used after creation)
  int device = 0;
  DevMesh m;
  void* mem = nullptr;
  int status = MF_OK;  // validateMesh outcome (reference order)
  std::string status_msg;
  bool uv_index_ok = true;
  bool owns_mem = true;  // false when the arrays live in context scratch
  ~mf_mesh() {
    if (mem && owns_mem) cudaFree(mem);
  }
};

// A built tree owns everything its queries touch: the tree arrays, its own
// query scratch and stream (`store`), and a mutex, so const queries from
// several host threads are safe (bvh.h:28) and the tree outlives the context
// (and host thread) that built it. Queries run on `qstream`: the building
// context's stream when that one was supplied by the caller (so device-input
// queries stay ordered with the caller's work), else the tree's own stream;
// mf_bvh_set_stream overrides it.
struct mf_bvh {
  int device = 0;
  mf_mesh* mesh = nullptr;
  Ctx store;  // owns the tree's device arrays, query scratch and stream
  cudaStream_t qstream = nullptr;
  std::mutex mu;
  Lbvh bvh;
  // host export cache
  bool exported = false;
  std::vector<double> boxes;
  std::vector<int32_t> links, order;
  int32_t leaves = 0, depth = 0;
};

namespace {

// MFB_TRACE=1 prints host-side phase timestamps of the entry points (stderr).
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  const char* what;
  explicit HostTrace(const char* w) : on(std::getenv("MFB_TRACE") != nullptr), what(w) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mfb] %s %-14s +%8.3f ms (t=%8.3f)\n", what, phase,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

int fail(int code, const std::string& msg) {
  set_last_error(msg);
  return code;
}

template <typename F>
int guarded(mf_ctx* ctx, F&& fn) {
  try {
    if (ctx) MFB_CUDA_TRY(cudaSetDevice(ctx->c.device));
    return fn();
  } catch (const ApiError& e) {
    return fail(e.code, e.msg);
  } catch (const CudaFailure& e) {
    return fail(MF_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e.err) + " at " + e.file + ":" +
                                 std::to_string(e.line) + " (" + e.expr + ")");
  } catch (const std::bad_alloc&) {
    return fail(MF_ERR_OUT_OF_MEMORY, "device or host allocation failed");
  } catch (const std::exception& e) {
    return fail(MF_ERR_CUDA, e.what());
  }
}

// guarded() for handles that outlive their context (meshes, trees)
template <typename F>
int guarded_dev(int device, F&& fn) {
  try {
    MFB_CUDA_TRY(cudaSetDevice(device));
    return fn();
  } catch (const ApiError& e) {
    return fail(e.code, e.msg);
  } catch (const CudaFailure& e) {
    return fail(MF_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e.err) + " at " + e.file + ":" +
                                 std::to_string(e.line) + " (" + e.expr + ")");
  } catch (const std::bad_alloc&) {
    return fail(MF_ERR_OUT_OF_MEMORY, "device or host allocation failed");
  } catch (const std::exception& e) {
    return fail(MF_ERR_CUDA, e.what());
  }
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool view_has_uvs(const mf_mesh_view* v) { return v->face_uvs && v->uvs && v->n_uvs > 0; }

// Device layout of an uploaded mesh: validates the view's sizes, allocates
// (scratch or owned) and points mesh->m at the device arrays.
struct MeshLayout {
  double* pos = nullptr;
  int32_t* faces = nullptr;
  double* nrm = nullptr;
  double* uvs = nullptr;
  int32_t* fuv = nullptr;
  int* flags = nullptr;
};
MeshLayout layout_mesh(Ctx& c, const mf_mesh_view* v, mf_mesh* mesh, const char* scratch_tag) {
  if (!v) throw ApiError(MF_ERR_BAD_ARGUMENT, "mesh view is null");
  if (v->n_vertices < 0 || v->n_faces < 0 || v->n_uvs < 0) throw ApiError(MF_ERR_BAD_ARGUMENT, "negative size");
  if ((v->n_vertices > 0 && !v->positions) || (v->n_faces > 0 && !v->faces))
    throw ApiError(MF_ERR_BAD_ARGUMENT, "null positions/faces with non-zero size");
  const bool has_n = v->normals && v->n_vertices > 0;
  const bool has_uv = view_has_uvs(v);
  const size_t bp = align_up(sizeof(double) * 3 * v->n_vertices, 256);
  const size_t bf = align_up(sizeof(int32_t) * 3 * v->n_faces, 256);
  const size_t bn = has_n ? bp : 0;
  const size_t bu = has_uv ? align_up(sizeof(double) * 2 * v->n_uvs, 256) : 0;
  const size_t bfu = has_uv ? bf : 0;
  const size_t total = bp + bf + bn + bu + bfu + 256;
  if (mesh->mem && mesh->owns_mem) cudaFree(mesh->mem);
  mesh->mem = nullptr;
  if (scratch_tag) {
    mesh->mem = c.buf(scratch_tag, total);
    mesh->owns_mem = false;
  } else {
    cudaError_t e = cudaMalloc(&mesh->mem, total);
    if (e == cudaErrorMemoryAllocation) {
      (void)cudaGetLastError();
      throw std::bad_alloc();
    }
    MFB_CUDA_TRY(e);
    mesh->owns_mem = true;
  }
  char* p = static_cast<char*>(mesh->mem);
  MeshLayout L;
  L.pos = reinterpret_cast<double*>(p);
  L.faces = reinterpret_cast<int32_t*>(p + bp);
  L.nrm = has_n ? reinterpret_cast<double*>(p + bp + bf) : nullptr;
  L.uvs = has_uv ? reinterpret_cast<double*>(p + bp + bf + bn) : nullptr;
  L.fuv = has_uv ? reinterpret_cast<int32_t*>(p + bp + bf + bn + bu) : nullptr;
  L.flags = reinterpret_cast<int*>(p + total - 256);
  DevMesh m;
  m.nv = v->n_vertices;
  m.nf = v->n_faces;
  m.nu = has_uv ? v->n_uvs : 0;
  m.pos = L.pos;
  m.faces = L.faces;
  m.nrm = L.nrm;
  m.uvs = L.uvs;
  m.fuv = L.fuv;
  mesh->m = m;
  return L;
}

// Enqueues the H2D copies (positions and faces unless `staged`: a staged
// upload already enqueued them) and the device validation of `v` on `s`;
// the validation flags land in `*hflag` (pinned host memory) when `s`
// reaches them. finish_upload() turns them into the mesh status after the
// caller has synchronised.
// defer: no validation pass and no flag read-back here: the caller's LBVH
// build checks the mesh itself (lbvh_build's vflags = L.flags, zeroed here)
// and reads the flags back after it.
void copy_validate_async(Ctx& c, cudaStream_t s, const mf_mesh_view* v, const MeshLayout& L, DevMesh& m,
                         int* hflag, cudaStream_t s2 = nullptr, bool staged = false, bool defer = false) {
  // with s2, the face indices travel on a second stream concurrently with
  // the positions (two H2D streams measured 25 -> 32 GB/s on the box)
  if (!staged) {
    if (s2) {
      MFB_CUDA_TRY(cudaEventRecord(c.up_fork, s));
      MFB_CUDA_TRY(cudaStreamWaitEvent(s2, c.up_fork, 0));
    }
    if (m.nv) MFB_CUDA_TRY(cudaMemcpyAsync(L.pos, v->positions, sizeof(double) * 3 * m.nv, cudaMemcpyHostToDevice, s));
    if (m.nf)
      MFB_CUDA_TRY(cudaMemcpyAsync(L.faces, v->faces, sizeof(int32_t) * 3 * m.nf, cudaMemcpyHostToDevice, s2 ? s2 : s));
  }
  if (s2) {
    MFB_CUDA_TRY(cudaEventRecord(c.up_join, s2));
    MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.up_join, 0));
  }
  if (L.nrm) MFB_CUDA_TRY(cudaMemcpyAsync(L.nrm, v->normals, sizeof(double) * 3 * m.nv, cudaMemcpyHostToDevice, s));
  if (L.uvs) {
    MFB_CUDA_TRY(cudaMemcpyAsync(L.uvs, v->uvs, sizeof(double) * 2 * m.nu, cudaMemcpyHostToDevice, s));
    MFB_CUDA_TRY(cudaMemcpyAsync(L.fuv, v->face_uvs, sizeof(int32_t) * 3 * m.nf, cudaMemcpyHostToDevice, s));
  }
  c.fill(L.flags, 0, sizeof(int), s);
  if (defer) return;
  const int64_t work = std::max<int64_t>(3ll * m.nv, 3ll * m.nf);
  if (work > 0) {
    const int grid = static_cast<int>(std::min<int64_t>(div_up(work, 256), kNumSMs * 16));
    k_validate<<<grid, 256, 0, s>>>(L.pos, m.nv, L.faces, m.nf, L.fuv, m.nu, L.flags);
    c.count_launch();
    MFB_CUDA_TRY(cudaGetLastError());
  }
  MFB_CUDA_TRY(cudaMemcpyAsync(hflag, L.flags, sizeof(int), cudaMemcpyDeviceToHost, s));
}

void upload_mesh_async(Ctx& c, cudaStream_t s, const mf_mesh_view* v, mf_mesh* mesh, const char* scratch_tag,
                       int* hflag, cudaStream_t s2 = nullptr) {
  const MeshLayout L = layout_mesh(c, v, mesh, scratch_tag);
  copy_validate_async(c, s, v, L, mesh->m, hflag, s2);
}

// Pageable host -> device through the context's pinned staging buffer: the
// context's host pool copies 1 MiB chunks into it and enqueues each chunk's
// DMA on the piece's stream right behind the copy, so host copies overlap
// the DMAs (a pageable cudaMemcpyAsync runs both serially on the calling
// thread). Returns once the job is started; c.host_pool().wait() ends it,
// after which every chunk's DMA is enqueued.
struct H2DPiece {
  void* dst;
  const void* src;
  size_t bytes;
  cudaStream_t s;
};
void staged_h2d_start(Ctx& c, const std::vector<H2DPiece>& pieces, const char* tag) {
  struct Chunk {
    char* dst;
    const char* src;
    size_t len, soff;
    cudaStream_t s;
  };
#ifndef MFB_STAGE_CHUNK_KB
#define MFB_STAGE_CHUNK_KB 1024
#endif
  constexpr size_t kChunk = static_cast<size_t>(MFB_STAGE_CHUNK_KB) << 10;
  auto chunks = std::make_shared<std::vector<Chunk>>();
  size_t total = 0;
  for (const H2DPiece& p : pieces) {
    for (size_t off = 0; off < p.bytes; off += kChunk) {
      const size_t len = std::min(kChunk, p.bytes - off);
      chunks->push_back({static_cast<char*>(p.dst) + off, static_cast<const char*>(p.src) + off, len, total, p.s});
      total += len;
    }
    total = align_up(total, 256);
  }
  char* stage = static_cast<char*>(c.host_buf(tag, std::max<size_t>(total, 1)));
  // interleave the pieces so both streams' DMAs start early
  std::stable_sort(chunks->begin(), chunks->end(), [&](const Chunk& a, const Chunk& b) {
    auto rank = [&](const Chunk& k) {
      for (const H2DPiece& p : pieces)
        if (k.src >= static_cast<const char*>(p.src) && k.src < static_cast<const char*>(p.src) + p.bytes)
          return static_cast<size_t>(k.src - static_cast<const char*>(p.src));
      return size_t(0);
    };
    return rank(a) < rank(b);
  });
  const int dev = c.device;
  c.host_pool().start(static_cast<int>(chunks->size()), [chunks, stage, dev](int i) {
    thread_local int cur = -1;
    if (cur != dev) {
      MFB_CUDA_TRY(cudaSetDevice(dev));
      cur = dev;
    }
    const Chunk& k = (*chunks)[i];
    std::memcpy(stage + k.soff, k.src, k.len);
    MFB_CUDA_TRY(cudaMemcpyAsync(k.dst, stage + k.soff, k.len, cudaMemcpyHostToDevice, k.s));
  });
}

// validateMesh (core/mesh.cpp:37-48) outcome from the device flags.
void finish_upload(mf_mesh* mesh, int hf) {
  mesh->status = MF_OK;
  mesh->status_msg.clear();
  if (mesh->m.nf == 0) {
    mesh->status = MF_ERR_EMPTY_MESH;
    mesh->status_msg = "EmptyMesh: mesh has no faces";
  } else if (hf & 1) {
    mesh->status = MF_ERR_INVALID_GEOMETRY;
    mesh->status_msg = "InvalidGeometry: non-finite vertex coordinate";
  } else if (hf & 2) {
    mesh->status = MF_ERR_INVALID_GEOMETRY;
    mesh->status_msg = "InvalidGeometry: face index out of range";
  }
  mesh->uv_index_ok = !(hf & 4);
}

// Upload + device validation into `mesh`, synchronously. With a scratch tag
// the arrays live in the context's grow-only scratch (host-buffer entry
// points: no cudaMalloc per call); otherwise the mesh owns a fresh allocation.
void upload_mesh(Ctx& c, cudaStream_t s, const mf_mesh_view* v, mf_mesh* mesh,
                 const char* scratch_tag = nullptr) {
  int* hf = static_cast<int*>(c.host_buf(std::string("upflag.") + (scratch_tag ? scratch_tag : "own"), sizeof(int)));
  upload_mesh_async(c, s, v, mesh, scratch_tag, hf);
  MFB_CUDA_TRY(cudaStreamSynchronize(s));
  finish_upload(mesh, *hf);
}

void check_mesh(const mf_mesh* mesh) {
  if (mesh->status != MF_OK) throw ApiError(mesh->status, mesh->status_msg);
}

// rasterizeGBuffer's precondition order (gbuffer.cpp:93-97).
void check_lowpoly(const mf_mesh* lo, int res) {
  check_mesh(lo);
  if (!lo->m.has_uvs()) throw ApiError(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: atlas rasterization needs a UV-mapped mesh");
  if (res < 1) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: resolution must be >= 1");
  if (!lo->uv_index_ok) throw ApiError(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: face uv index out of range");
}
void check_transfer_cfg(double diag, double frac) {
  if (!(diag > 0.0) || !(frac > 0.0))
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: distance filter must be positive");
}

// Leaf-range cap of the dense LBVH for a bake (result-invariant: only the
// walk's cost depends on it). Small leaves suit queries near the surface, long
// leaves a wide search ball over small triangles: the ball-to-triangle scale is
// taken as maxDistanceFraction x sqrt(F) (triangle size ~ diag / sqrt(F)).
// Measured: configs A-D (ratio 4.5-10) best at 3; config E (ratio 100) 63.8
// -> 49.8 ms from 3 to 11.
int bake_leaf_hint(double frac, int nf) {
  const double r = frac * std::sqrt(static_cast<double>(std::max(nf, 1)));
  if (!(r >= 27.0)) return 3;
  // wide leaves carry the triangle pre-test (Lbvh::tplane); config E (scale
  // 100): caps 11 / 13 / 15 measured 45.8 / 45.0 / 44.3 ms per bake
  return static_cast<int>(std::min(15.0, std::max(4.0, std::round(r / 6.6))));
}

// Stage timing on the context's persistent event pool: mark k records pool
// event base + k (so the marks survive inside a captured graph).
struct Timer {
  Ctx& c;
  int next;
  explicit Timer(Ctx& cc, int base = 0) : c(cc), next(base) {}
  cudaEvent_t mark(cudaStream_t s) {
    if (!c.timing) return nullptr;
    cudaEvent_t e = c.pool_event(next++);
    // inside a stream capture a plain record is only a dependency marker; an
    // external record becomes an event-record node that timestamps on replay
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    MFB_CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusActive) MFB_CUDA_TRY(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
    else MFB_CUDA_TRY(cudaEventRecord(e, s));
    return e;
  }
  static float ms(cudaEvent_t a, cudaEvent_t b) {
    if (!a || !b) return 0.f;
    float v = 0.f;
    if (cudaEventElapsedTime(&v, a, b) != cudaSuccess) {
      (void)cudaGetLastError();
      return 0.f;
    }
    return v;
  }
};

GBufDev gbuf_slab(Ctx& c, int res, int row0, int rows) {
  GBufDev g;
  g.res = res;
  g.row0 = row0;
  g.rows = rows;
  const int64_t n = g.texels();
  g.pos = c.buf<float>("g.pos", 3 * n);
  g.nrm = c.buf<float>("g.nrm", 3 * n);
  g.tan = c.buf<float>("g.tan", 3 * n);
  g.bit = c.buf<float>("g.bit", 3 * n);
  g.valid = c.buf<uint8_t>("g.valid", n);
  g.rel = c.buf<uint8_t>("g.rel", n);
  return g;
}

QueryList query_list(Ctx& c, int64_t capacity) {
  QueryList q;
  q.capacity = static_cast<int>(capacity);
  q.qpos = c.buf<float4>("q.pos", capacity);
  q.qtbn = c.buf<float>("q.tbn", 9 * capacity);
  q.count = c.buf<int>("q.count", 4);  // [0] pass A, [1] pass B
  return q;
}

constexpr int kBandEventBase = 80;  // pool events 80 .. 80 + kMaxBands - 1: band downloads

// Everything the fused bake enqueues; no host synchronisation inside, so
// the same sequence can be captured into a CUDA graph.
// Recorded in this order (the graph-timing path rebuilds them from the pool
// indices): side0 side1 e0 e1 d0 d1 e2 e3 e4 e5. d0/d1 bracket the dilation
// links kernel (empty when the bake dilates after the transfer, e4/e5).
struct BakeMarks {
  cudaEvent_t side0 = nullptr, side1 = nullptr, e0 = nullptr, e1 = nullptr, d0 = nullptr, d1 = nullptr,
              e2 = nullptr, e3 = nullptr, e4 = nullptr, e5 = nullptr;
};

// Runs `body` (work enqueued on `s`, possibly forking/joining other streams)
// through `slot`: eagerly the first time a key is seen, captured into a graph
// on the second identical call, replayed afterwards. A capture during which
// scratch was (re)allocated is discarded (its pointers are stale).
template <class F>
void run_graphed(Ctx& c, Ctx::GraphSlot& slot, cudaStream_t s, const std::vector<char>& key, bool allow, F&& body) {
  if (allow && slot.exec && key == slot.key && c.alloc_gen == slot.gen) {
    MFB_CUDA_TRY(cudaGraphLaunch(slot.exec, s));
    return;
  }
  if (allow && key == slot.prev_key && c.alloc_gen == slot.prev_gen) {
    cudaGraph_t graph = nullptr;
    MFB_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    c.capturing = true;
    try {
      body();
    } catch (const CaptureRealloc&) {  // scratch had to grow: discard, run eagerly
      c.capturing = false;
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      body();
      slot.prev_key = key;
      slot.prev_gen = c.alloc_gen;
      return;
    } catch (...) {
      c.capturing = false;
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    c.capturing = false;
    MFB_CUDA_TRY(cudaStreamEndCapture(s, &graph));
    if (slot.exec) cudaGraphExecDestroy(slot.exec);
    slot.exec = nullptr;
    MFB_CUDA_TRY(cudaGraphInstantiateWithFlags(&slot.exec, graph, cudaGraphInstantiateFlagUseNodePriority));
    cudaGraphDestroy(graph);
    slot.key = key;
    slot.gen = c.alloc_gen;
    MFB_CUDA_TRY(cudaGraphLaunch(slot.exec, s));
    return;
  }
  body();
  slot.prev_key = key;
  slot.prev_gen = c.alloc_gen;
}

template <class T>
std::vector<char> key_bytes(const T& k) {
  return std::vector<char>(reinterpret_cast<const char*>(&k), reinterpret_cast<const char*>(&k) + sizeof(k));
}

// cuStreamWaitValue32 (driver API, resolved at run time: the library does
// not link libcuda). Null when the driver does not provide it.
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<WaitValueFn>(f);
  }();
  return fn;
}
// One probe per context (first host-buffer bake): a wait on a flag that is
// already set, on the copy stream, must succeed - otherwise the bake keeps
// the single download after the transfer.
bool wait_value_usable(Ctx& c) {
  if (c.wait_value_probe != 0) return c.wait_value_probe > 0;
  c.wait_value_probe = -1;
  if (!wait_value_fn() || !c.aux2) return false;
  int* f = c.buf<int>("bake.waitprobe", 1);
  if (cudaMemsetAsync(f, 0x01, sizeof(int), c.aux2) != cudaSuccess) return false;
  if (wait_value_fn()(reinterpret_cast<CUstream>(c.aux2), reinterpret_cast<CUdeviceptr>(f), 1,
                      CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
    (void)cudaGetLastError();
    return false;
  }
  if (cudaStreamSynchronize(c.aux2) != cudaSuccess) return false;
  c.wait_value_probe = 1;
  return true;
}
void stream_wait_value(cudaStream_t s, int* flag) {
  if (wait_value_fn()(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), 1,
                      CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    throw ApiError(MF_ERR_CUDA, "cuStreamWaitValue32 failed");
}

// Bands downloaded in one copy behind the transfer instead of on the band
// stream (MFB_TAIL_BANDS, default 2; never all of them).
int tail_bands(int nb) {
  static const int k = [] {
    const char* e = std::getenv("MFB_TAIL_BANDS");
    return e ? std::max(0, std::atoi(e)) : 2;
  }();
  return std::min(k, nb - 1);
}

// The bake's three phases. enqueue_bake() chains them with a fork/join (the
// captured graph); the host-buffer entry point interleaves its own upload and
// validation wait between them (bake_host_overlapped).
struct BakeEnq {
  Ctx& c;
  const mf_mesh *lo, *hi;
  int res, radius, rb, re, s0, s1;
  double diag, frac;
  uint8_t* rgb_out;
  int bpp = 3;  // bytes per atlas texel (c.fmt)
  bool debug;
  const OutSet* pub = nullptr;  // set: the dilation stores every output row into each buffer
  Timer& tm;
  BakeMarks& mk;
  GBufDev g;
  int* flags = nullptr;
  unsigned long long* counters = nullptr;
  RasterFused fo;
  Lbvh bvh;
  double* hiN = nullptr;
  // host path: the dense mesh's validation runs inside its LBVH build
  // (lbvh_build vflags); its flags are read back into dense_hflag after it
  int* dense_vflags = nullptr;
  int* dense_hflag = nullptr;

  // Dilation resolved before the transfer (full atlas, one output): the
  // raster and transfer write straight into rgb_out, the gutter texels are
  // filled by dilate_links (constant sources) and by the transfer's epilogue
  // (query sources), and no dilation pass follows the transfer.
  bool links = false;
  int* dep_next = nullptr;
  // host-buffer path: row bands of the atlas downloaded while the transfer
  // runs (BandSync); set before low()
  bool band_sync = false;
  BandSync bs;
  int* band_check = nullptr;  // pinned [nb]: ready flags before the release (MFB_BAND_CHECK)
  int band_ev_base = -1;      // >= 0: record pool event base + b after band b's download

  BakeEnq(Ctx& cc, const mf_mesh* l, const mf_mesh* h, int rs, double dg, double fr, int rad, int b0, int b1,
          uint8_t* out, bool dbg, Timer& t, BakeMarks& m, const OutSet* pb = nullptr)
      : c(cc), lo(l), hi(h), res(rs), radius(rad), rb(b0), re(b1), diag(dg), frac(fr), rgb_out(out), debug(dbg),
        pub(pb), tm(t), mk(m) {
    s0 = std::max(0, rb - radius);  // raster/transfer slab with the dilation halo
    s1 = std::min(res, re + radius);
    g.res = res;
    g.row0 = s0;
    g.rows = s1 - s0;
    g.valid = c.buf<uint8_t>("g.valid", g.texels());
    // flags: [0] AtlasOverlap, [1] bin overflow, [2] bin total, [3] query overflow
    flags = c.buf<int>("bake.flags", 4);
    counters = c.buf<unsigned long long>("bake.counters", 4);
    links = !pub && rb == 0 && re == res && dilate_links_supported(radius) && raster_links_supported();
    fo.fmt = c.fmt;
    bpp = atlas_bpp(c.fmt);
    fo.rgb = links ? rgb_out : c.buf<uint8_t>("bake.raw", bpp * g.texels());
    fo.q = query_list(c, g.texels());
    if (links) {
      fo.qslot = c.buf<int>("bake.qslot", g.texels());
      fo.dep_head = c.buf<int>("bake.dephead", g.texels());
      dep_next = c.buf<int>("bake.depnext", g.texels());
      fo.tile_state = c.buf<uint8_t>("bake.tilestate", static_cast<int64_t>(div_up(res, 16)) * div_up(res, 16));
    }
    fo.valid_count = counters + 2;
    if (debug) {
      fo.dbg_face = c.buf<int32_t>("bake.dface", g.texels());
      fo.dbg_ts = c.buf<double>("bake.dts", 3 * g.texels());
    }
  }

  // main stream: lowpoly prep (its wedge frames on the aux stream) + fused
  // raster (valid mask, raw map, query list)
  void low() {
    cudaStream_t m = c.stream;
    c.fill(flags, 0, 4 * sizeof(int), m);
    c.fill(counters, 0, 4 * sizeof(unsigned long long), m);
    // the lowpoly branch on the context's high-priority stream (the caller's
    // stream has whatever priority the caller gave it), joined back to main
    cudaStream_t s = c.lowhi ? c.lowhi : m;
    if (s != m) {
      MFB_CUDA_TRY(cudaEventRecord(c.lowfork, m));
      MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.lowfork, 0));
    }
    if (band_sync) {
      c.fill(bs.tot, 0, 4 * kMaxBands * sizeof(int), s);
      fo.band_tot = bs.tot;
      fo.band_rows = bs.rows;
    }
    mk.e0 = tm.mark(s);
    RasterPlan plan;
    PrepBinning pb;
    pb.row0 = g.row0;
    pb.rows = g.rows;
    pb.flags = flags;
    pb.zero4 = raster_links_supported() ? fo.q.count : nullptr;
    prepare_lowpoly(c, s, lo->m, res, plan, &pb);
    mk.e1 = tm.mark(s);
    // the dilation links run beside the interpolation kernel (both need only
    // the coverage kernel's outputs)
    cudaStream_t ls = links && c.aux2 ? c.aux2 : nullptr;
    fo.cover_done = ls ? c.pool_event(60) : nullptr;
    raster_gbuffer(c, s, lo->m, plan, g, flags, nullptr, &fo);
    cudaStream_t t = ls ? ls : s;
    if (ls) MFB_CUDA_TRY(cudaStreamWaitEvent(ls, fo.cover_done, 0));
    mk.d0 = tm.mark(t);
    if (links) dilate_links(c, t, res, g.valid, radius, fo.qslot, fo.dep_head, dep_next, rgb_out, fo.tile_state,
                             fo.fmt);
    mk.d1 = tm.mark(t);
    if (links) {
      if (band_sync) band_init(c, t, bs);
      if (ls) {
        MFB_CUDA_TRY(cudaEventRecord(c.pool_event(61), ls));
        MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.pool_event(61), 0));
      }
    } else if (band_sync) {
      band_init(c, s, bs);
    }
    mk.e2 = tm.mark(s);
    if (s != m) {
      MFB_CUDA_TRY(cudaEventRecord(c.lowjoin, s));
      MFB_CUDA_TRY(cudaStreamWaitEvent(m, c.lowjoin, 0));
    }
  }

  // dense mesh: LBVH on the side stream; unit vertex normals (needed only by
  // the transfer's encode) on the aux stream, enqueued after low() so they
  // queue behind the lowpoly wedge frames. Both wait for `ready`.
  void dense_bvh(cudaEvent_t ready) {
    cudaStream_t side = c.side;
    MFB_CUDA_TRY(cudaStreamWaitEvent(side, ready, 0));
    mk.side0 = tm.mark(side);
    lbvh_build(c, side, hi->m, bvh, "hi.bvh", bake_leaf_hint(frac, hi->m.nf));
    mk.side1 = tm.mark(side);
    MFB_CUDA_TRY(cudaEventRecord(c.join, side));
  }
  void dense_normals(cudaEvent_t ready) {
    cudaStream_t ns = c.dn ? c.dn : (c.aux ? c.aux : c.side);
    hiN = c.buf<double>("hi.unitN", 3 * static_cast<size_t>(hi->m.nv));
    if (ns != c.side) MFB_CUDA_TRY(cudaStreamWaitEvent(ns, ready, 0));
    vertex_normals(c, ns, hi->m, hiN, true, "hi");
    MFB_CUDA_TRY(cudaEventRecord(c.join3, ns));
  }

  // host-buffer path: the whole dense phase on the side stream (normals on
  // aux, forked and joined back), so it can be captured from `side` alone;
  // then c.join / c.join3 mark its end for tail().
  void dense_side(bool graphs) {
    cudaStream_t side = c.side, ns = c.dn ? c.dn : (c.aux ? c.aux : c.side);
    lbvh_layout(c, hi->m, bvh, "hi.bvh", bake_leaf_hint(frac, hi->m.nf));
    hiN = c.buf<double>("hi.unitN", 3 * static_cast<size_t>(hi->m.nv));
    const int64_t k[] = {reinterpret_cast<int64_t>(hi->m.pos), reinterpret_cast<int64_t>(hi->m.faces),
                         reinterpret_cast<int64_t>(hi->m.nrm), hi->m.nf, hi->m.nv,
                         reinterpret_cast<int64_t>(dense_vflags), reinterpret_cast<int64_t>(dense_hflag)};
    run_graphed(c, c.g_dense, side, key_bytes(k), graphs, [&] {
      MFB_CUDA_TRY(cudaEventRecord(c.dfork, side));
      mk.side0 = tm.mark(side);
      lbvh_build(c, side, hi->m, bvh, "hi.bvh", bake_leaf_hint(frac, hi->m.nf), dense_vflags);
      mk.side1 = tm.mark(side);
      if (ns != side) {
        MFB_CUDA_TRY(cudaStreamWaitEvent(ns, c.dfork, 0));
        vertex_normals(c, ns, hi->m, hiN, true, "hi");
        MFB_CUDA_TRY(cudaEventRecord(c.djoin, ns));
        MFB_CUDA_TRY(cudaStreamWaitEvent(side, c.djoin, 0));
      } else {
        vertex_normals(c, side, hi->m, hiN, true, "hi");
      }
    });
    MFB_CUDA_TRY(cudaEventRecord(c.join, side));
    MFB_CUDA_TRY(cudaEventRecord(c.join3, side));
  }

  // main stream, after both dense branches: transfer + dilation + flags
  // With host_out (host-buffer entry point) and the dilation links, the atlas
  // downloads in row bands on aux2 while the transfer runs (BandSync).
  void tail(int* hflags_pinned, unsigned long long* hcnt_pinned, uint8_t* host_out = nullptr) {
    cudaStream_t s = c.stream;
    MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.join, 0));
    MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.join3, 0));
    mk.e3 = tm.mark(s);
    TransferArgs ta;
    ta.q = fo.q;
    ta.res = res;
    ta.slab_row0 = s0;
    ta.hi_positions = hi->m.pos;
    ta.hi_normals = hiN;
    ta.hi_faces = hi->m.faces;
    ta.max_dist = frac * diag;
    ta.rgb = fo.rgb;
    ta.fmt = fo.fmt;
    ta.dbg_face = fo.dbg_face;
    ta.dbg_ts = fo.dbg_ts;
    ta.counters = counters;
    if (links) {
      ta.dep_head = fo.dep_head;
      ta.dep_next = dep_next;
    }
    cudaStream_t cp = c.aux2 ? c.aux2 : s;
    if (links && band_sync && host_out && cp != s) {
      // each band's download waits (on cp) for its ready flag, set by the
      // transfer's warps; k_finish after the transfer releases every wait
      // regardless (by then every band is final), so no wait outlives it
      ta.bands = bs;
      cudaEvent_t ev = c.pool_event(40);
      MFB_CUDA_TRY(cudaEventRecord(ev, s));
      transfer_normals(c, s, bvh, ta);
      mk.e4 = tm.mark(s);
      // MFB_BAND_CHECK=1 (tests): the flags as the transfer left them, checked
      // by the host after the bake - every band must have been signalled
      // by the counts, not by the release below
      if (band_check) {
        MFB_CUDA_TRY(cudaMemcpyAsync(band_check, bs.ready, bs.nb * sizeof(int), cudaMemcpyDeviceToHost, s));
      }
      // the last bands complete with the transfer itself: one copy on s right
      // behind it (each wait-value node on cp costs ~7 us even when already
      // satisfied, which is what the copies after the transfer paid)
      mk.e5 = tm.mark(s);
      // (k_finish first: it runs while the band stream's last copy still
      // holds the copy engine)
      finish_flags(c, s, flags, counters, dense_vflags, hflags_pinned, hcnt_pinned, dense_hflag, bs.ready, bs.nb);
      const int nstream = bs.nb - tail_bands(bs.nb);
      if (nstream < bs.nb) {
        const int64_t off = static_cast<int64_t>(bpp) * nstream * bs.rows * res;
        MFB_CUDA_TRY(cudaMemcpyAsync(host_out + off, rgb_out + off,
                                     static_cast<int64_t>(bpp) * (res - nstream * bs.rows) * res,
                                     cudaMemcpyDeviceToHost, s));
        if (band_ev_base >= 0)
          for (int b = nstream; b < bs.nb; ++b) MFB_CUDA_TRY(cudaEventRecord(c.pool_event(band_ev_base + b), s));
      }
      MFB_CUDA_TRY(cudaStreamWaitEvent(cp, ev, 0));
      for (int b = 0; b < nstream; ++b) {
        const int r0 = b * bs.rows, r1 = std::min(res, r0 + bs.rows);
        stream_wait_value(cp, bs.ready + b);
        const int64_t off = static_cast<int64_t>(bpp) * r0 * res;
        MFB_CUDA_TRY(cudaMemcpyAsync(host_out + off, rgb_out + off, static_cast<int64_t>(bpp) * (r1 - r0) * res,
                                     cudaMemcpyDeviceToHost, cp));
        if (band_ev_base >= 0) MFB_CUDA_TRY(cudaEventRecord(c.pool_event(band_ev_base + b), cp));
      }
      MFB_CUDA_TRY(cudaEventRecord(c.join4, cp));
      MFB_CUDA_TRY(cudaStreamWaitEvent(s, c.join4, 0));
      return;
    }
    transfer_normals(c, s, bvh, ta);
    mk.e4 = tm.mark(s);
    if (links) {  // the atlas is complete
      mk.e5 = tm.mark(s);
      if (host_out)
        MFB_CUDA_TRY(cudaMemcpyAsync(host_out, rgb_out, static_cast<int64_t>(bpp) * (re - rb) * res,
                                     cudaMemcpyDeviceToHost, s));
    } else {
      if (pub) dilate_seams_to(c, s, res, res, bpp, fo.rgb, g.valid, s0, s1 - s0, radius, *pub, rb, re - rb);
      else dilate_seams(c, s, res, res, bpp, fo.rgb, g.valid, s0, s1 - s0, radius, rgb_out, rb, re - rb);
      mk.e5 = tm.mark(s);
      if (host_out)
        MFB_CUDA_TRY(cudaMemcpyAsync(host_out, rgb_out, static_cast<int64_t>(bpp) * (re - rb) * res,
                                     cudaMemcpyDeviceToHost, s));
    }
    finish_flags(c, s, flags, counters, dense_vflags, hflags_pinned, hcnt_pinned, dense_hflag, nullptr, 0);
  }
};

// Everything the fused bake enqueues; no host synchronisation inside, so
// the same sequence can be captured into a CUDA graph.
void enqueue_bake(Ctx& c, const mf_mesh* lo, const mf_mesh* hi, int res, double diag, double frac, int radius,
                  int rb, int re, uint8_t* rgb_out, bool debug, Timer& tm, BakeMarks& mk, int* hflags_pinned,
                  unsigned long long* hcnt_pinned, const OutSet* pub = nullptr) {
  BakeEnq q(c, lo, hi, res, diag, frac, radius, rb, re, rgb_out, debug, tm, mk, pub);
  MFB_CUDA_TRY(cudaEventRecord(c.fork, c.stream));
  q.dense_bvh(c.fork);
  q.low();
  q.dense_normals(c.fork);
  q.tail(hflags_pinned, hcnt_pinned);
}

// The fused bake over validated device meshes; rows [rb, re) into rgb_out
// (device). The first call with a given shape runs eagerly (allocating
// scratch), the second identical call captures the whole two-stream sequence
// into a CUDA graph, later ones replay it (MFB_GRAPH=0 disables). Debug
// outputs always run eagerly.
void bake_dev(Ctx& c, const mf_mesh* lo, const mf_mesh* hi, int res, double diag, double frac, int radius,
              int rb, int re, uint8_t* rgb_out, int32_t* dbg_face, double* dbg_ts, mf_bake_stats* st,
              Timer& tm, cudaEvent_t t_begin, const OutSet* pub = nullptr) {
  check_lowpoly(lo, res);
  check_mesh(hi);
  check_transfer_cfg(diag, frac);
  if (radius < 0) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilation radius must be >= 0");
  if (rb < 0 || re > res || rb >= re) throw ApiError(MF_ERR_BAD_ARGUMENT, "row range outside the atlas");
  cudaStream_t s = c.stream;
  // debug outputs and stage timing always run eagerly (events inside a graph
  // are not meaningful)
  // MFB_GRAPH_TIMING=1: keep the captured graph when stage timing is on (its
  // marks are event-record nodes), to time the stages as the graph runs them
  static const bool graph_timing = [] {
    const char* e = std::getenv("MFB_GRAPH_TIMING");
    return e && e[0] == '1';
  }();
  const bool debug = dbg_face || dbg_ts || (c.timing && !graph_timing);
  static const bool graphs = [] {
    const char* e = std::getenv("MFB_GRAPH");
    return !(e && e[0] == '0');
  }();
  int* hflags = static_cast<int*>(c.host_buf("bake.hflags", 4 * sizeof(int)));
  auto* hcnt = static_cast<unsigned long long*>(c.host_buf("bake.hcnt", 4 * sizeof(unsigned long long)));
  // graph key: everything baked into the captured sequence
  // (the mesh handles' contents are immutable after upload: the ABI has no
  // call that modifies an mf_mesh in place)
  struct Key {
    const void *lo, *hi, *out, *lo_mem, *hi_mem;
    int lo_nf, lo_nv, lo_nu, hi_nf, hi_nv, res, radius, rb, re, timing, fmt;
    int64_t bin_capacity;
    double diag, frac;
  };
  const int s0 = std::max(0, rb - radius);
  bool force_eager = false;
  for (int attempt = 0;; ++attempt) {
    Key key{};
    key = Key{lo, hi, rgb_out, lo->mem, hi->mem, lo->m.nf, lo->m.nv, lo->m.nu, hi->m.nf, hi->m.nv, res, radius, rb,
              re, c.timing ? 1 : 0, c.fmt, c.bin_capacity, diag, frac};
    std::vector<char> kb(reinterpret_cast<const char*>(&key), reinterpret_cast<const char*>(&key) + sizeof(key));
    if (pub) {  // published bakes are keyed on their destination buffers too
      const char* pb = reinterpret_cast<const char*>(pub);
      kb.insert(kb.end(), pb, pb + sizeof(OutSet));
    }
    HostTrace ht("bake_dev");
    BakeMarks mk;
    Timer t2(c, tm.next);
    if (graphs && !debug && !force_eager && c.bake_exec && kb == c.bake_key && c.alloc_gen == c.bake_gen) {
      MFB_CUDA_TRY(cudaGraphLaunch(c.bake_exec, s));
      // the graph recorded its marks on pool events tm.next .. tm.next + 7 in this order
      if (c.timing) {
        int i = tm.next;
        mk.side0 = c.pool_event(i++);
        mk.side1 = c.pool_event(i++);
        mk.e0 = c.pool_event(i++);
        mk.e1 = c.pool_event(i++);
        mk.d0 = c.pool_event(i++);
        mk.d1 = c.pool_event(i++);
        mk.e2 = c.pool_event(i++);
        mk.e3 = c.pool_event(i++);
        mk.e4 = c.pool_event(i++);
        mk.e5 = c.pool_event(i++);
      }
    } else if (graphs && !debug && !force_eager && kb == c.bake_prev_key && c.alloc_gen == c.bake_prev_gen) {
      // same shape as the previous eager run: every buffer exists -> capture
      cudaGraph_t graph = nullptr;
      bool realloc = false;
      MFB_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      c.capturing = true;
      try {
        enqueue_bake(c, lo, hi, res, diag, frac, radius, rb, re, rgb_out, false, t2, mk, hflags, hcnt, pub);
      } catch (const CaptureRealloc&) {  // scratch had to grow: discard the capture
        realloc = true;
      } catch (...) {
        c.capturing = false;
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      c.capturing = false;
      if (realloc) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        graph = nullptr;
        (void)cudaGetLastError();
      } else {
        MFB_CUDA_TRY(cudaStreamEndCapture(s, &graph));
      }
      if (realloc || c.alloc_gen != c.bake_prev_gen) {  // scratch changed: do not keep it, run eagerly
        if (graph) cudaGraphDestroy(graph);
        enqueue_bake(c, lo, hi, res, diag, frac, radius, rb, re, rgb_out, false, t2, mk, hflags, hcnt, pub);
        c.bake_prev_gen = c.alloc_gen;
      } else {
        if (c.bake_exec) cudaGraphExecDestroy(c.bake_exec);
        c.bake_exec = nullptr;
        MFB_CUDA_TRY(cudaGraphInstantiateWithFlags(&c.bake_exec, graph, cudaGraphInstantiateFlagUseNodePriority));
        cudaGraphDestroy(graph);
        c.bake_key = kb;
        c.bake_gen = c.alloc_gen;
        MFB_CUDA_TRY(cudaGraphLaunch(c.bake_exec, s));
        }
    } else {
      enqueue_bake(c, lo, hi, res, diag, frac, radius, rb, re, rgb_out, dbg_face || dbg_ts, t2, mk, hflags, hcnt,
                   pub);
      c.bake_prev_key = kb;
      c.bake_prev_gen = c.alloc_gen;
    }
    ht.mark("enqueued");
    if (dbg_face || dbg_ts) {
      if (dbg_face)
        MFB_CUDA_TRY(cudaMemcpyAsync(dbg_face, c.buf<int32_t>("bake.dface", 1) + static_cast<int64_t>(rb - s0) * res,
                                     sizeof(int32_t) * static_cast<int64_t>(re - rb) * res, cudaMemcpyDeviceToHost, s));
      if (dbg_ts)
        MFB_CUDA_TRY(cudaMemcpyAsync(dbg_ts, c.buf<double>("bake.dts", 1) + 3 * static_cast<int64_t>(rb - s0) * res,
                                     sizeof(double) * 3 * static_cast<int64_t>(re - rb) * res, cudaMemcpyDeviceToHost,
                                     s));
    }
    MFB_CUDA_TRY(cudaStreamSynchronize(s));
    ht.mark("synced");
    if (hflags[1] && attempt == 0) {  // tile bins overflowed: rerun eagerly with the exact capacity
      c.bin_capacity = static_cast<int64_t>(hflags[2]) + 1;
      c.invalidate_graphs();
      force_eager = true;
      continue;
    }
    if (hflags[1] || hflags[3]) throw ApiError(MF_ERR_CUDA, "internal capacity overflow");
    if (hflags[0]) throw ApiError(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
    if (st) {
      st->queries = static_cast<int64_t>(hcnt[0] - hcnt[3]);  // less the dead records (unreliable texels)
      st->hits = static_cast<int64_t>(hcnt[1]);
      st->valid_texels = static_cast<int64_t>(hcnt[2]);
      st->bvh_nodes = hi->m.nf > 1 ? hi->m.nf - 1 : 0;
      st->bvh_depth = 0;
      if (c.timing && std::getenv("MFB_TRACE_MARKS")) {  // diagnostic: mark offsets from the bake start
        const cudaEvent_t t0e = t_begin ? t_begin : mk.e0;
        std::fprintf(stderr, "[mfb marks] side0 %.3f side1 %.3f e0 %.3f e1 %.3f e2 %.3f e3 %.3f e4 %.3f e5 %.3f\n",
                     Timer::ms(t0e, mk.side0), Timer::ms(t0e, mk.side1), Timer::ms(t0e, mk.e0),
                     Timer::ms(t0e, mk.e1), Timer::ms(t0e, mk.e2), Timer::ms(t0e, mk.e3), Timer::ms(t0e, mk.e4),
                     Timer::ms(t0e, mk.e5));
      }
      if (c.timing) {
        st->ms_prepare = Timer::ms(mk.e0, mk.e1);
        st->ms_raster = Timer::ms(mk.e1, mk.e2);
        st->ms_bvh = Timer::ms(mk.side0, mk.side1);
        st->ms_transfer = Timer::ms(mk.e3, mk.e4);
        // the dilation links kernel (fused full-atlas bake) or the dilation after the transfer
        st->ms_dilate = Timer::ms(mk.d0, mk.d1) + Timer::ms(mk.e4, mk.e5);
        st->ms_total = Timer::ms(t_begin ? t_begin : mk.e0, mk.e5);
      }
    }
    return;
  }
}

// True when [p, p + bytes) is page-locked host memory (its H2D copy is a
// truly asynchronous DMA; a pageable source blocks the calling thread).
bool host_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// mf_bake_normal_map without debug outputs. The dense mesh's H2D copy and
// device validation run on the side stream while the lowpoly is uploaded,
// validated, prepared and rasterised on the main stream; the host waits for
// the dense validation flag only after the lowpoly work is queued, then
// queues the LBVH / dense normals and the transfer. Errors keep the
// reference's order: lowpoly checks (gbuffer.cpp:93-97), AtlasOverlap
// (:157-159), then transferNormals' checks (:195-199), then dilateSeams' (:255).
void bake_host_overlapped(Ctx& c, mf_ctx* owner, const mf_mesh_view* lv, const mf_mesh_view* hv, int res,
                          double diag, double frac, int radius, uint8_t* rgb_out, mf_bake_stats* st) {
  HostTrace ht("bake_host");
  cudaStream_t s = c.stream;
  mf_mesh lo, hi;
  lo.ctx = hi.ctx = owner;
  int* hup = static_cast<int*>(c.host_buf("bake.upflags", 2 * sizeof(int)));
  int* hflags = static_cast<int*>(c.host_buf("bake.hflags", 4 * sizeof(int)));
  auto* hcnt = static_cast<unsigned long long*>(c.host_buf("bake.hcnt", 4 * sizeof(unsigned long long)));
  Timer tm(c, 0);
  cudaEvent_t t0 = tm.mark(s);
  if (!hv) throw ApiError(MF_ERR_BAD_ARGUMENT, "mesh view is null");
  // The lowpoly's copy goes first: H2D copies share one copy engine in
  // submission order, so the (small) lowpoly must not queue behind the
  // dense mesh. Pinned dense arrays are then submitted before the host waits
  // for the lowpoly flags; pageable ones would block this thread, so they go
  // after the lowpoly work is queued.
  const bool early = host_pinned(hv->positions) && host_pinned(hv->faces) && host_pinned(hv->normals);
  MFB_CUDA_TRY(cudaEventRecord(c.fork, s));  // the caller's earlier work on the ctx stream
  // Pageable dense arrays (a drop-in caller's std::vectors) are staged
  // through the context's pinned buffer by its host pool, starting now: the
  // chunk copies and their DMAs run while this thread uploads and checks the
  // lowpoly and queues its work.
  const bool staged = !early && hv->n_vertices > 0 && hv->n_faces > 0 && c.up1;
  struct PoolGuard {
    Ctx& c;
    bool on = false;
    void wait() {
      if (on) {
        on = false;
        c.host_pool().wait();
      }
    }
    ~PoolGuard() {
      try {
        wait();
      } catch (...) {
      }
    }
  } pool_job{c};
  MeshLayout hiL;
  if (staged) {
    MFB_CUDA_TRY(cudaStreamWaitEvent(c.up1, c.fork, 0));
    MFB_CUDA_TRY(cudaStreamWaitEvent(c.up2, c.fork, 0));
    hiL = layout_mesh(c, hv, &hi, "up.hi");
    staged_h2d_start(c,
                     {{hiL.pos, hv->positions, sizeof(double) * 3 * static_cast<size_t>(hv->n_vertices), c.up1},
                      {hiL.faces, hv->faces, sizeof(int32_t) * 3 * static_cast<size_t>(hv->n_faces), c.up2}},
                     "stage.hi");
    pool_job.on = true;
  }
  // Speculative dense phase (below): its validation is folded into the LBVH
  // build (k_bounds / k_morton), so no validation pass and no flag read-back
  // sit between the dense upload and the build
  const bool spec = hv->n_faces > 0 && hv->n_vertices > 0 && diag > 0.0 && frac > 0.0 && radius >= 0;
  auto upload_hi = [&] {
    MFB_CUDA_TRY(cudaStreamWaitEvent(c.side, c.fork, 0));
    if (staged) {
      pool_job.wait();  // every chunk's DMA is enqueued
      MFB_CUDA_TRY(cudaEventRecord(c.up1_done, c.up1));
      MFB_CUDA_TRY(cudaEventRecord(c.up2_done, c.up2));
      MFB_CUDA_TRY(cudaStreamWaitEvent(c.side, c.up1_done, 0));
      MFB_CUDA_TRY(cudaStreamWaitEvent(c.side, c.up2_done, 0));
      copy_validate_async(c, c.side, hv, hiL, hi.m, hup + 1, nullptr, true, spec);
    } else {
      hiL = layout_mesh(c, hv, &hi, "up.hi");
      copy_validate_async(c, c.side, hv, hiL, hi.m, hup + 1, c.aux ? c.aux : nullptr, false, spec);
    }
    MFB_CUDA_TRY(cudaEventRecord(c.hi_ready, c.side));
  };
  auto drain = [&] {
    try {
      pool_job.wait();
    } catch (...) {
    }
    c.sync_all();
  };
  try {
    ht.mark("entry");
    upload_mesh_async(c, s, lv, &lo, "up.lo", hup);
    ht.mark("lowpoly queued");
    if (early) upload_hi();
    ht.mark("dense upload q");
    MFB_CUDA_TRY(cudaStreamSynchronize(s));
    ht.mark("lowpoly synced");
    finish_upload(&lo, hup[0]);
    check_lowpoly(&lo, res);
    ht.mark("lowpoly checked");
    if (!rgb_out) throw ApiError(MF_ERR_BAD_ARGUMENT, "rgb_out is null");
  } catch (...) {
    drain();
    throw;
  }
  const int bpp = atlas_bpp(c.fmt);
  uint8_t* drgb = c.buf<uint8_t>("bake.rgb", bpp * static_cast<int64_t>(res) * res);
  BakeMarks mk;
  Timer tmb(c, 8);
  BakeEnq q(c, &lo, &hi, res, diag, frac, radius, 0, res, drgb, false, tmb, mk);
  // A pageable rgb_out gets the atlas through pinned staging: its row bands
  // are copied out by the host pool as their DMAs land.
  const bool stage_out = !host_pinned(rgb_out);
  uint8_t* host_dst = stage_out ? static_cast<uint8_t*>(c.host_buf("stage.rgb", bpp * static_cast<size_t>(res) * res))
                                : rgb_out;
  if (q.links && wait_value_usable(c)) {
    q.band_sync = true;
    int* bb = c.buf<int>("bake.bands", 4 * kMaxBands);
    q.bs.tot = bb;
    q.bs.done = bb + kMaxBands;
    q.bs.nbr = bb + 2 * kMaxBands;
    q.bs.ready = bb + 3 * kMaxBands;
    q.bs.res = res;
    // ~32 bands (64 rows at 2048^2): the copy left after the transfer is one
    // small band (16 or 64 bands measured 15-19 us slower end to end). Each
    // band's wait + copy costs the band stream ~11 us whatever its size, so
    // small atlases (a short transfer) get bands of >= kMinBandBytes: at
    // 512^2, 32 bands of 24 KB queued ~320 us of band copies behind a 96 us
    // transfer (config A end to end 0.69 ms)
    constexpr int band_div = 32;
    constexpr int64_t kMinBandBytes = 256 << 10;
    const int64_t row_bytes = static_cast<int64_t>(atlas_bpp(c.fmt)) * res;
    const int min_rows = static_cast<int>(std::min<int64_t>(res, div_up(kMinBandBytes, row_bytes)));
    q.bs.rows = std::max({(div_up(res, band_div) + 15) / 16 * 16, (min_rows + 15) / 16 * 16, (radius + 15) / 16 * 16});
    q.bs.nb = div_up(res, q.bs.rows);
    const char* chk = std::getenv("MFB_BAND_CHECK");
    if (chk && chk[0] == '1') q.band_check = static_cast<int*>(c.host_buf("bake.bandcheck", kMaxBands * sizeof(int)));
    if (stage_out) q.band_ev_base = kBandEventBase;
  }
  static const bool graphs = [] {
    const char* e = std::getenv("MFB_GRAPH");
    return !(e && e[0] == '0');
  }();
  static const bool graph_timing = [] {
    const char* e = std::getenv("MFB_GRAPH_TIMING");
    return e && e[0] == '1';
  }();
  const bool use_graphs = graphs && (!c.timing || graph_timing);
  {
    const int64_t k[] = {reinterpret_cast<int64_t>(lo.m.pos), reinterpret_cast<int64_t>(lo.m.faces),
                         reinterpret_cast<int64_t>(lo.m.nrm), reinterpret_cast<int64_t>(lo.m.uvs),
                         reinterpret_cast<int64_t>(lo.m.fuv), lo.m.nf, lo.m.nv, lo.m.nu, res, c.bin_capacity,
                         q.band_sync ? 1 : 0, radius, c.fmt};
    run_graphed(c, c.g_low, s, key_bytes(k), use_graphs, [&] { q.low(); });
  }
  ht.mark("low queued");
  if (!early) upload_hi();
  // Speculative dense phase: the LBVH / normals / transfer are queued right
  // behind the dense upload and its validation (which zeroes out-of-range
  // indices in the device copy), without a host round trip on the critical
  // path; the validation outcome is read after the bake, in the reference's
  // error order.
  if (spec) {
    hi.status = MF_OK;  // provisional until the flags are read
    q.dense_vflags = hiL.flags;
    q.dense_hflag = hup + 1;
  } else {
    MFB_CUDA_TRY(cudaEventSynchronize(c.hi_ready));
    finish_upload(&hi, hup[1]);
  }
  if (!spec && (hi.status != MF_OK || !(diag > 0.0) || !(frac > 0.0) || radius < 0)) {
    // raster errors precede transferNormals' checks: finish the raster first
    MFB_CUDA_TRY(cudaMemcpyAsync(hflags, q.flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
    drain();
    if (hflags[0]) throw ApiError(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
    check_mesh(&hi);
    check_transfer_cfg(diag, frac);
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilation radius must be >= 0");
  }
  q.dense_side(use_graphs);
  ht.mark("dense queued");
  cudaEvent_t t2 = tm.mark(s);
  q.tail(hflags, hcnt, host_dst);
  ht.mark("tail queued");
  const int64_t row_bytes = static_cast<int64_t>(bpp) * res;
  if (stage_out && q.band_sync) {
    const int dev = c.device, nb = q.bs.nb, rows = q.bs.rows;
    std::vector<cudaEvent_t> ev(nb);
    for (int b = 0; b < nb; ++b) ev[b] = c.pool_event(kBandEventBase + b);
    c.host_pool().start(nb, [=](int b) {
      thread_local int cur = -1;
      if (cur != dev) {
        MFB_CUDA_TRY(cudaSetDevice(dev));
        cur = dev;
      }
      MFB_CUDA_TRY(cudaEventSynchronize(ev[b]));
      const int r0 = b * rows, r1 = std::min(res, r0 + rows);
      std::memcpy(rgb_out + r0 * row_bytes, host_dst + r0 * row_bytes, (r1 - r0) * row_bytes);
    });
    pool_job.on = true;
  }
  cudaEvent_t t3 = tm.mark(s);
  MFB_CUDA_TRY(cudaStreamSynchronize(s));
  ht.mark("synced");
  if (stage_out) {
    if (q.band_sync) {
      pool_job.wait();
    } else {
      constexpr int kRows = 64;
      c.host_pool().run(static_cast<int>(div_up(res, kRows)), [=](int b) {
        const int r0 = b * kRows, r1 = std::min(res, r0 + kRows);
        std::memcpy(rgb_out + r0 * row_bytes, host_dst + r0 * row_bytes, (r1 - r0) * row_bytes);
      });
    }
  }
  if (spec) {
    finish_upload(&hi, hup[1]);
    if (hi.status != MF_OK) {
      if (hflags[0]) throw ApiError(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
      check_mesh(&hi);
    }
  }
  if (hflags[1] || hflags[3]) {
    // tile bins overflowed on this shape: the device-mesh path re-runs with
    // the exact capacity (and keeps it for later calls)
    if (hflags[1]) c.bin_capacity = static_cast<int64_t>(hflags[2]) + 1;
    c.invalidate_graphs();
    Timer tr(c, 8);
    bake_dev(c, &lo, &hi, res, diag, frac, radius, 0, res, drgb, nullptr, nullptr, st, tr, nullptr);
    MFB_CUDA_TRY(cudaMemcpyAsync(rgb_out, drgb, bpp * static_cast<int64_t>(res) * res, cudaMemcpyDeviceToHost, s));
    MFB_CUDA_TRY(cudaStreamSynchronize(s));
    return;
  }
  if (hflags[0]) throw ApiError(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
  if (q.band_check)
    for (int b = 0; b < q.bs.nb; ++b)
      if (q.band_check[b] != 1)
        throw ApiError(MF_ERR_CUDA, "band sync: row band " + std::to_string(b) + " was not signalled by the transfer");
  if (st) {
    st->queries = static_cast<int64_t>(hcnt[0] - hcnt[3]);  // less the dead records (unreliable texels)
    st->hits = static_cast<int64_t>(hcnt[1]);
    st->valid_texels = static_cast<int64_t>(hcnt[2]);
    st->bvh_nodes = hi.m.nf > 1 ? hi.m.nf - 1 : 0;
    st->bvh_depth = 0;
    if (c.timing && std::getenv("MFB_TRACE_MARKS")) {
      std::fprintf(stderr,
                   "[mfb host marks] e0 %.3f e1 %.3f e2 %.3f side0 %.3f side1 %.3f e3 %.3f e4 %.3f e5 %.3f "
                   "dl0 %.3f dl1 %.3f\n",
                   Timer::ms(t0, mk.e0), Timer::ms(t0, mk.e1), Timer::ms(t0, mk.e2), Timer::ms(t0, mk.side0),
                   Timer::ms(t0, mk.side1), Timer::ms(t0, mk.e3), Timer::ms(t0, mk.e4), Timer::ms(t0, mk.e5),
                   Timer::ms(t0, t2), Timer::ms(t0, t3));
    }
    if (c.timing) {
      st->ms_upload = Timer::ms(t0, mk.e0);
      st->ms_prepare = Timer::ms(mk.e0, mk.e1);
      st->ms_raster = Timer::ms(mk.e1, mk.e2);
      st->ms_bvh = Timer::ms(mk.side0, mk.side1);
      st->ms_transfer = Timer::ms(mk.e3, mk.e4);
      st->ms_dilate = Timer::ms(mk.d0, mk.d1) + Timer::ms(mk.e4, mk.e5);
      st->ms_download = Timer::ms(t2, t3);
      st->ms_total = Timer::ms(t0, t3);
    }
  }
}

thread_local std::vector<std::unique_ptr<mf_mesh>> g_tmp_meshes;

}  // namespace

extern "C" {

const char* mf_version(void) { return "mfbake-b200 0.1.0 (sm_100a)"; }
int mf_abi_version(void) { return MF_ABI_VERSION; }
const char* mf_last_error(void) { return g_last_error.c_str(); }

int mf_ctx_create(int device, void* stream, mf_ctx** out) {
  if (!out) return fail(MF_ERR_BAD_ARGUMENT, "out is null");
  *out = nullptr;
  return guarded(nullptr, [&]() -> int {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      (void)cudaGetLastError();
      return fail(MF_ERR_NO_DEVICE, "no CUDA device available");
    }
    if (device < 0 || device >= n) return fail(MF_ERR_NO_DEVICE, "device ordinal out of range");
    MFB_CUDA_TRY(cudaSetDevice(device));
    auto ctx = std::make_unique<mf_ctx>();
    ctx->c.device = device;
    if (stream) {
      ctx->c.stream = static_cast<cudaStream_t>(stream);
    } else {
      MFB_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
      ctx->c.own_stream = true;
    }
    // the dense LBVH branch is the bake's longest pre-transfer chain: its
    // streams get the higher priority so the lowpoly branches fill in around it
    int lo_prio = 0, hi_prio = 0;
    MFB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    // The lowpoly branch streams (wedge frames, reliability, raster) are high
    // priority as well as the LBVH's; the dense normals stay low. With the
    // segment-tree LBVH the lowpoly branch is the longer chain: 1.431 ->
    // 1.401 ms (with the refit climb it was the reverse: 1.52 vs 1.505 ms).
    // Three levels: the lowpoly branch on top, the LBVH one below, the dense
    // vertex normals (needed only by the transfer's encode) lowest. Measured
    // with per-step events: 1.428 ms per bake vs 1.437 (LBVH above the
    // lowpoly branch; r02s: 1.433 vs 1.430) and 1.455-1.465 with the normals
    // at the lowpoly level. With equal priorities the coverage kernel's 16k
    // CTAs (queued first) held the SMs while the LBVH waited ~70-100 us. The
    // pre-transfer phase is bound by the branches' total work, so priorities
    // move it by ~2% at most.
    const int mid_prio = std::min(lo_prio, hi_prio + 1);
    const int lbvh_prio = mid_prio, low_prio = hi_prio;
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.side, cudaStreamNonBlocking, lbvh_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.aux, cudaStreamNonBlocking, low_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.side2, cudaStreamNonBlocking, lbvh_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.aux2, cudaStreamNonBlocking, low_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.lowhi, cudaStreamNonBlocking, low_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.dn, cudaStreamNonBlocking, lo_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.up1, cudaStreamNonBlocking, hi_prio));
    MFB_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->c.up2, cudaStreamNonBlocking, hi_prio));
    for (cudaEvent_t* e : {&ctx->c.fork, &ctx->c.join, &ctx->c.fork2, &ctx->c.join2, &ctx->c.join3, &ctx->c.hi_ready,
                            &ctx->c.dfork, &ctx->c.djoin, &ctx->c.up_fork, &ctx->c.up_join, &ctx->c.lfork,
                            &ctx->c.ljoin, &ctx->c.setup_done, &ctx->c.join4, &ctx->c.lowfork,
                            &ctx->c.lowjoin, &ctx->c.up1_done, &ctx->c.up2_done})
      MFB_CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    *out = ctx.release();
    return MF_OK;
  });
}

void mf_ctx_destroy(mf_ctx* ctx) { delete ctx; }

int mf_ctx_synchronize(mf_ctx* ctx) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    ctx->c.sync_all();
    return MF_OK;
  });
}

int mf_ctx_set_timing(mf_ctx* ctx, int enabled) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  ctx->c.timing = enabled != 0;
  return MF_OK;
}

int64_t mf_ctx_launch_count(const mf_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int mf_mesh_upload(mf_ctx* ctx, const mf_mesh_view* view, mf_mesh** out) {
  if (!ctx || !out) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded(ctx, [&]() -> int {
    auto mesh = std::make_unique<mf_mesh>();
    mesh->ctx = ctx;
    mesh->device = ctx->c.device;
    upload_mesh(ctx->c, ctx->c.stream, view, mesh.get());
    *out = mesh.release();
    return MF_OK;
  });
}

void mf_mesh_destroy(mf_mesh* mesh) {
  if (mesh) cudaSetDevice(mesh->device);
  delete mesh;
}

// rasterizeGBuffer into the slab buffers of g (full atlas); retries once
// with the exact tile-bin capacity when the bins overflowed.
static void raster_full(Ctx& c, const mf_mesh& lo, GBufDev& g) {
  int* flags = c.buf<int>("bake.flags", 4);
  for (int attempt = 0;; ++attempt) {
    MFB_CUDA_TRY(cudaMemsetAsync(flags, 0, 4 * sizeof(int), c.stream));
    RasterPlan plan;
    PrepBinning pb;
    pb.row0 = g.row0;
    pb.rows = g.rows;
    pb.flags = flags;
    prepare_lowpoly(c, c.stream, lo.m, g.res, plan, &pb);
    raster_gbuffer(c, c.stream, lo.m, plan, g, flags, nullptr);
    int hf[4] = {0, 0, 0, 0};
    MFB_CUDA_TRY(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (hf[1] && attempt == 0) {
      c.bin_capacity = static_cast<int64_t>(hf[2]) + 1;
      continue;
    }
    if (hf[1]) throw ApiError(MF_ERR_CUDA, "internal capacity overflow");
    if (hf[0]) throw ApiError(MF_ERR_ATLAS_OVERLAP, "AtlasOverlap: texel claimed by two UV triangles");
    break;
  }
}

int mf_raster_gbuffer(mf_ctx* ctx, const mf_mesh_view* lowpoly, int res, float* position, float* normal,
                      float* tangent, float* bitangent, uint8_t* valid, uint8_t* reliable) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh lo;
    lo.ctx = ctx;
    upload_mesh(c, c.stream, lowpoly, &lo, "up.lo");
    check_lowpoly(&lo, res);
    if (!position || !normal || !tangent || !bitangent || !valid || !reliable)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null G-buffer output");
    GBufDev g = gbuf_slab(c, res, 0, res);
    raster_full(c, lo, g);
    const int64_t n = g.texels();
    MFB_CUDA_TRY(cudaMemcpyAsync(position, g.pos, 12 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(normal, g.nrm, 12 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(tangent, g.tan, 12 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(bitangent, g.bit, 12 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(valid, g.valid, n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(reliable, g.rel, n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_raster_gbuffer_dev(mf_ctx* ctx, mf_mesh* lowpoly, int res, float* position, float* normal, float* tangent,
                          float* bitangent, uint8_t* valid, uint8_t* reliable) {
  if (!ctx || !lowpoly) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_lowpoly(lowpoly, res);
    if (!position || !normal || !tangent || !bitangent || !valid || !reliable)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null G-buffer output");
    GBufDev g;
    g.res = res;
    g.row0 = 0;
    g.rows = res;
    g.pos = position;
    g.nrm = normal;
    g.tan = tangent;
    g.bit = bitangent;
    g.valid = valid;
    g.rel = reliable;
    raster_full(c, *lowpoly, g);
    return MF_OK;
  });
}

int mf_transfer_normals(mf_ctx* ctx, int res, const float* position, const float* normal, const float* tangent,
                        const float* bitangent, const uint8_t* valid, const uint8_t* reliable,
                        const mf_mesh_view* highpoly, double bbox_diagonal, double max_distance_fraction,
                        uint8_t* rgb_out) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    if (res < 1 || !valid) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: g-buffer is empty");
    mf_mesh hi;
    hi.ctx = ctx;
    upload_mesh(c, c.stream, highpoly, &hi, "up.hi");
    check_mesh(&hi);
    check_transfer_cfg(bbox_diagonal, max_distance_fraction);
    if (!position || !normal || !tangent || !bitangent || !reliable || !rgb_out)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null G-buffer input or output");
    GBufDev g = gbuf_slab(c, res, 0, res);
    const int64_t n = g.texels();
    MFB_CUDA_TRY(cudaMemcpyAsync(g.pos, position, 12 * n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(g.nrm, normal, 12 * n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(g.tan, tangent, 12 * n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(g.bit, bitangent, 12 * n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(g.valid, valid, n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(g.rel, reliable, n, cudaMemcpyHostToDevice, c.stream));
    double* hiN = c.buf<double>("hi.unitN", 3 * static_cast<size_t>(hi.m.nv));
    vertex_normals(c, c.stream, hi.m, hiN, true, "hi");
    Lbvh bvh;
    lbvh_build(c, c.stream, hi.m, bvh, "hi.bvh", bake_leaf_hint(max_distance_fraction, hi.m.nf));
    RasterFused fo;
    fo.rgb = c.buf<uint8_t>("bake.raw", 3 * n);
    fo.q = query_list(c, n);
    gbuffer_queries(c, c.stream, g, fo);
    TransferArgs ta;
    ta.q = fo.q;
    ta.res = res;
    ta.slab_row0 = 0;
    ta.hi_positions = hi.m.pos;
    ta.hi_normals = hiN;
    ta.hi_faces = hi.m.faces;
    ta.max_dist = max_distance_fraction * bbox_diagonal;
    ta.rgb = fo.rgb;
    transfer_normals(c, c.stream, bvh, ta);
    uint8_t* raw = fo.rgb;
    MFB_CUDA_TRY(cudaMemcpyAsync(rgb_out, raw, 3 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_dilate_seams(mf_ctx* ctx, int width, int height, int channels, const uint8_t* map_in, int gres,
                    const uint8_t* valid, int radius, uint8_t* map_out) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    if (radius < 0) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilation radius must be >= 0");
    if (width != gres || height != gres)
      throw ApiError(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: map and g-buffer resolutions differ");
    if (channels < 1 || !map_in || !map_out || (gres > 0 && !valid))
      throw ApiError(MF_ERR_BAD_ARGUMENT, "bad map arguments");
    const int64_t n = static_cast<int64_t>(width) * height;
    if (n == 0) return MF_OK;
    uint8_t* din = c.buf<uint8_t>("dil.in", n * channels);
    uint8_t* dout = c.buf<uint8_t>("dil.out", n * channels);
    uint8_t* dval = c.buf<uint8_t>("dil.valid", n);
    MFB_CUDA_TRY(cudaMemcpyAsync(din, map_in, n * channels, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(dval, valid, n, cudaMemcpyHostToDevice, c.stream));
    dilate_seams(c, c.stream, width, height, channels, din, dval, 0, height, radius, dout, 0, height);
    MFB_CUDA_TRY(cudaMemcpyAsync(map_out, dout, n * channels, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

// The atlas encoding of one bake call (Ctx::fmt), restored when the call ends.
struct FmtScope {
  Ctx& c;
  int saved;
  FmtScope(Ctx& cc, int fmt) : c(cc), saved(cc.fmt) {
    if (fmt != MF_ATLAS_RGB8 && fmt != MF_ATLAS_RGBA8 && fmt != MF_ATLAS_RG16)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "unknown atlas format");
    c.fmt = fmt;
  }
  ~FmtScope() { c.fmt = saved; }
};

static int bake_host_call(mf_ctx* ctx, const mf_mesh_view* lowpoly, const mf_mesh_view* highpoly, int res,
                          double bbox_diagonal, double max_distance_fraction, int radius, int fmt, uint8_t* rgb_out,
                          int32_t* dbg_face, double* dbg_ts, mf_bake_stats* stats) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    FmtScope fs(c, fmt);
    const int bpp = atlas_bpp(fmt);
    // debug outputs take the sequential upload -> bake -> download path
    if (!dbg_face && !dbg_ts) {
      mf_bake_stats local{};
      bake_host_overlapped(c, ctx, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius, rgb_out,
                           &local);
      if (stats) *stats = local;
      return MF_OK;
    }
    HostTrace ht("bake_host");
    Timer tm(c, 0);  // host marks use pool events 0..3; bake_dev's start at 8
    Timer tmb(c, 8);
    cudaEvent_t t0 = tm.mark(c.stream);
    mf_mesh lo, hi;
    lo.ctx = hi.ctx = ctx;
    upload_mesh(c, c.stream, lowpoly, &lo, "up.lo");
    ht.mark("upload lo");
    // reference order: lowpoly checks precede the highpoly's (gbuffer.cpp:93-97 then :195-199)
    check_lowpoly(&lo, res);
    upload_mesh(c, c.stream, highpoly, &hi, "up.hi");
    ht.mark("upload hi");
    cudaEvent_t t1 = tm.mark(c.stream);
    if (!rgb_out) throw ApiError(MF_ERR_BAD_ARGUMENT, "rgb_out is null");
    uint8_t* drgb = c.buf<uint8_t>("bake.rgb", bpp * static_cast<int64_t>(res) * res);
    mf_bake_stats local{};
    bake_dev(c, &lo, &hi, res, bbox_diagonal, max_distance_fraction, radius, 0, res, drgb, dbg_face, dbg_ts,
             &local, tmb, t1);
    ht.mark("bake_dev");
    cudaEvent_t t2 = tm.mark(c.stream);
    MFB_CUDA_TRY(cudaMemcpyAsync(rgb_out, drgb, bpp * static_cast<int64_t>(res) * res, cudaMemcpyDeviceToHost,
                                 c.stream));
    cudaEvent_t t3 = tm.mark(c.stream);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    ht.mark("download+sync");
    if (stats) {
      *stats = local;
      if (c.timing) {
        stats->ms_upload = Timer::ms(t0, t1);
        stats->ms_download = Timer::ms(t2, t3);
        stats->ms_total = Timer::ms(t0, t3);
      }
    }
    ht.mark("stats");
    return MF_OK;
  });
}

int mf_bake_normal_map(mf_ctx* ctx, const mf_mesh_view* lowpoly, const mf_mesh_view* highpoly, int res,
                       double bbox_diagonal, double max_distance_fraction, int radius, uint8_t* rgb_out,
                       int32_t* dbg_face, double* dbg_ts, mf_bake_stats* stats) {
  return bake_host_call(ctx, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius, MF_ATLAS_RGB8,
                        rgb_out, dbg_face, dbg_ts, stats);
}

int mf_bake_normal_map_ex(mf_ctx* ctx, const mf_mesh_view* lowpoly, const mf_mesh_view* highpoly, int res,
                          double bbox_diagonal, double max_distance_fraction, int radius, int format, void* out,
                          mf_bake_stats* stats) {
  return bake_host_call(ctx, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius, format,
                        static_cast<uint8_t*>(out), nullptr, nullptr, stats);
}

int mf_bake_normal_map_dev(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int res, double bbox_diagonal,
                           double max_distance_fraction, int radius, int row_begin, int row_end, uint8_t* rgb_dev,
                           mf_bake_stats* stats) {
  return mf_bake_normal_map_dev_ex(ctx, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius,
                                   row_begin, row_end, MF_ATLAS_RGB8, rgb_dev, stats);
}

int mf_bake_normal_map_dev_ex(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int res, double bbox_diagonal,
                              double max_distance_fraction, int radius, int row_begin, int row_end, int format,
                              void* out_dev, mf_bake_stats* stats) {
  uint8_t* rgb_dev = static_cast<uint8_t*>(out_dev);
  if (!ctx || !lowpoly || !highpoly || !rgb_dev) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    FmtScope fs(ctx->c, format);
    if (format != MF_ATLAS_RGB8 && (reinterpret_cast<uintptr_t>(rgb_dev) & 3))
      throw ApiError(MF_ERR_BAD_ARGUMENT, "4-byte atlas formats need a 4-byte aligned buffer");
    Timer tm(ctx->c, 8);
    mf_bake_stats local{};
    bake_dev(ctx->c, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius, row_begin, row_end,
             rgb_dev, nullptr, nullptr, &local, tm, nullptr);
    if (stats) *stats = local;
    return MF_OK;
  });
}

int mf_coverage_rows(mf_ctx* ctx, mf_mesh* lowpoly, int res, int64_t* row_counts) {
  if (!ctx || !lowpoly || !row_counts) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_lowpoly(lowpoly, res);
    GBufDev g = gbuf_slab(c, res, 0, res);
    int* flags = c.buf<int>("bake.flags", 4);
    int64_t* rows = c.buf<int64_t>("cov.rows", res);
    MFB_CUDA_TRY(cudaMemsetAsync(flags, 0, 4 * sizeof(int), c.stream));
    RasterPlan plan;
    PrepBinning pb;
    pb.row0 = g.row0;
    pb.rows = g.rows;
    pb.flags = flags;
    pb.row_counts = rows;
    prepare_lowpoly(c, c.stream, lowpoly->m, res, plan, &pb);
    raster_gbuffer(c, c.stream, lowpoly->m, plan, g, flags, rows);
    MFB_CUDA_TRY(cudaMemcpyAsync(row_counts, rows, sizeof(int64_t) * res, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

// ---------------------------------------------------------------- BVH API
int mf_bvh_build(mf_ctx* ctx, mf_mesh* mesh, mf_bvh** out) {
  if (!ctx || !mesh || !out) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  *out = nullptr;
  return guarded(ctx, [&]() -> int {
    check_mesh(mesh);  // Bvh::Bvh calls validateMesh (bvh.cpp:49)
    auto b = std::make_unique<mf_bvh>();
    b->device = ctx->c.device;
    b->mesh = mesh;
    b->store.device = ctx->c.device;
    MFB_CUDA_TRY(cudaStreamCreateWithFlags(&b->store.stream, cudaStreamNonBlocking));
    b->store.own_stream = true;
    b->qstream = ctx->c.own_stream ? b->store.stream : ctx->c.stream;
    lbvh_build(ctx->c, ctx->c.stream, mesh->m, b->bvh, "bvh");
    // move the persistent arrays out of the context scratch into the handle
    const int nn = std::max(b->bvh.n_nodes, 1);
    BNode* nodes = b->store.buf<BNode>("nodes", nn);
    BTri* tris = b->store.buf<BTri>("tris", b->bvh.n_tris);
    TBox* tbox = b->store.buf<TBox>("tbox", b->bvh.n_tris);
    MFB_CUDA_TRY(cudaMemcpyAsync(tbox, b->bvh.tbox, sizeof(TBox) * b->bvh.n_tris, cudaMemcpyDeviceToDevice, ctx->c.stream));
    auto* acc = b->store.buf<unsigned long long>("acc", 8);
    MFB_CUDA_TRY(cudaMemcpyAsync(nodes, b->bvh.nodes, sizeof(BNode) * nn, cudaMemcpyDeviceToDevice, ctx->c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(tris, b->bvh.tris, sizeof(BTri) * b->bvh.n_tris, cudaMemcpyDeviceToDevice, ctx->c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(acc, b->bvh.scene_acc, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToDevice,
                                 ctx->c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(b->bvh.root_box, b->bvh.root_box_dev, sizeof(float) * 6, cudaMemcpyDeviceToHost,
                                 ctx->c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(ctx->c.stream));
    b->bvh.nodes = nodes;
    b->bvh.tris = tris;
    b->bvh.tbox = tbox;
    b->bvh.scene_acc = acc;
    b->bvh.root_box_dev = nullptr;
    *out = b.release();
    return MF_OK;
  });
}

void mf_bvh_destroy(mf_bvh* bvh) {
  if (bvh) cudaSetDevice(bvh->device);
  delete bvh;
}

int mf_bvh_set_stream(mf_bvh* bvh, void* stream) {
  if (!bvh) return fail(MF_ERR_BAD_ARGUMENT, "bvh is null");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    MFB_CUDA_TRY(cudaStreamSynchronize(bvh->qstream));
    bvh->qstream = stream ? static_cast<cudaStream_t>(stream) : bvh->store.stream;
    return MF_OK;
  });
}

namespace {
void export_bvh(mf_bvh* b) {
  if (b->exported) return;
  const Lbvh& t = b->bvh;
  std::vector<BNode> nodes(std::max(t.n_nodes, 1));
  std::vector<BTri> tris(t.n_tris);
  if (t.n_nodes > 0)
    MFB_CUDA_TRY(cudaMemcpy(nodes.data(), t.nodes, sizeof(BNode) * t.n_nodes, cudaMemcpyDeviceToHost));
  MFB_CUDA_TRY(cudaMemcpy(tris.data(), t.tris, sizeof(BTri) * t.n_tris, cudaMemcpyDeviceToHost));
  b->order.resize(t.n_tris);
  for (int i = 0; i < t.n_tris; ++i) b->order[i] = tris[i].face;
  // DFS pre-order (root = 0), mirroring the reference's node numbering (bvh.cpp:65-66)
  struct Item {
    int32_t ref;
    float box[6];
    int parent, side, depth;
  };
  std::vector<Item> stack;
  Item root{t.root_ref, {t.root_box[0], t.root_box[1], t.root_box[2], t.root_box[3], t.root_box[4], t.root_box[5]},
            -1, 0, 0};
  stack.push_back(root);
  b->boxes.clear();
  b->links.clear();
  b->leaves = 0;
  b->depth = 0;
  while (!stack.empty()) {
    Item it = stack.back();
    stack.pop_back();
    const int idx = static_cast<int>(b->links.size() / 4);
    for (int k = 0; k < 6; ++k) b->boxes.push_back(it.box[k]);
    b->links.insert(b->links.end(), {-1, -1, 0, 0});
    if (it.parent >= 0) b->links[4 * it.parent + it.side] = idx;
    b->depth = std::max(b->depth, it.depth);
    if (it.ref < 0) {
      int first, count;
      leaf_decode(it.ref, first, count);
      b->links[4 * idx + 2] = first;
      b->links[4 * idx + 3] = count;
      ++b->leaves;
      continue;
    }
    const BNode& n = nodes[it.ref];
    const float* f = reinterpret_cast<const float*>(&n);
    Item l{n.d.x, {f[0], f[2], f[4], f[6], f[8], f[10]}, idx, 0, it.depth + 1};  // bnode_coord(0, k)
    Item r{n.d.y, {f[1], f[3], f[5], f[7], f[9], f[11]}, idx, 1, it.depth + 1};  // bnode_coord(1, k)
    stack.push_back(r);  // left is visited (and numbered) first
    stack.push_back(l);
  }
  b->exported = true;
}
}  // namespace

int mf_bvh_info(const mf_bvh* bvh, int32_t* nodes, int32_t* leaves, int32_t* depth) {
  if (!bvh) return fail(MF_ERR_BAD_ARGUMENT, "bvh is null");
  mf_bvh* b = const_cast<mf_bvh*>(bvh);
  return guarded_dev(b->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(b->mu);
    export_bvh(b);
    if (nodes) *nodes = static_cast<int32_t>(b->links.size() / 4);
    if (leaves) *leaves = b->leaves;
    if (depth) *depth = b->depth;
    return MF_OK;
  });
}

int mf_bvh_export(mf_bvh* bvh, double* boxes, int32_t* links, int32_t* face_order) {
  if (!bvh) return fail(MF_ERR_BAD_ARGUMENT, "bvh is null");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    export_bvh(bvh);
    if (boxes) std::memcpy(boxes, bvh->boxes.data(), sizeof(double) * bvh->boxes.size());
    if (links) std::memcpy(links, bvh->links.data(), sizeof(int32_t) * bvh->links.size());
    if (face_order) std::memcpy(face_order, bvh->order.data(), sizeof(int32_t) * bvh->order.size());
    return MF_OK;
  });
}

int mf_bvh_closest_within_dev(mf_bvh* bvh, const double* q, int64_t n, double max_distance, int32_t* face,
                              double* dist_sq, double* point, double* bary) {
  if (!bvh || (n > 0 && (!q || !face || !dist_sq))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    closest_within(c, qs, bvh->bvh, q, n, max_distance, face, dist_sq, point, bary);
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    return MF_OK;
  });
}

int mf_bvh_closest_within(mf_bvh* bvh, const double* q, int64_t n, double max_distance, int32_t* face,
                          double* dist_sq, double* point, double* bary) {
  if (!bvh || (n > 0 && (!q || !face || !dist_sq))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    if (n <= 0) return MF_OK;
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    double* dq = c.buf<double>("cp.q", 3 * n);
    int32_t* df = c.buf<int32_t>("cp.f", n);
    double* dd = c.buf<double>("cp.d", n);
    double* dp = c.buf<double>("cp.p", 3 * n);
    double* db = c.buf<double>("cp.b", 3 * n);
    MFB_CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, qs));
    closest_within(c, qs, bvh->bvh, dq, n, max_distance, df, dd, dp, db);
    MFB_CUDA_TRY(cudaMemcpyAsync(face, df, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(dist_sq, dd, sizeof(double) * n, cudaMemcpyDeviceToHost, qs));
    if (point) MFB_CUDA_TRY(cudaMemcpyAsync(point, dp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, qs));
    if (bary) MFB_CUDA_TRY(cudaMemcpyAsync(bary, db, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    return MF_OK;
  });
}

int mf_sample_sdf_dev(mf_bvh* bvh, int grid_res, const double* grid_origin, double voxel_size, const float* field_dev,
                      const double* points_dev, int64_t n, double* values_dev) {
  if (!bvh || !grid_origin || (n > 0 && (!field_dev || !points_dev || !values_dev)))
    return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    if (grid_res < 2 || !(voxel_size > 0.0))
      throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: the signed field needs res >= 2 and voxelSize > 0");
    std::lock_guard<std::mutex> lk(bvh->mu);
    sample_sdf(bvh->store, bvh->qstream, bvh->bvh, points_dev, n, grid_res, grid_origin, voxel_size, field_dev,
               values_dev);
    MFB_CUDA_TRY(cudaStreamSynchronize(bvh->qstream));
    return MF_OK;
  });
}

int mf_sample_sdf(mf_bvh* bvh, int grid_res, const double* grid_origin, double voxel_size, const float* field,
                  const double* points, int64_t n, double* values) {
  if (!bvh || !grid_origin || (n > 0 && (!field || !points || !values)))
    return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    if (grid_res < 2 || !(voxel_size > 0.0))
      throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: the signed field needs res >= 2 and voxelSize > 0");
    if (n <= 0) return MF_OK;
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    const int64_t cells = static_cast<int64_t>(grid_res) * grid_res * grid_res;
    double* dq = c.buf<double>("sdf.q", 3 * n);
    float* dfield = c.buf<float>("sdf.field", cells);
    double* dv = c.buf<double>("sdf.v", n);
    MFB_CUDA_TRY(cudaMemcpyAsync(dq, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(dfield, field, sizeof(float) * cells, cudaMemcpyHostToDevice, qs));
    sample_sdf(c, qs, bvh->bvh, dq, n, grid_res, grid_origin, voxel_size, dfield, dv);
    MFB_CUDA_TRY(cudaMemcpyAsync(values, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    return MF_OK;
  });
}

int mf_bvh_raycast_first_dev(mf_bvh* bvh, const double* o, const double* d, int64_t n, double tmin, double tmax,
                             int32_t* face, double* t, double* u, double* v) {
  if (!bvh || (n > 0 && (!o || !d || !face || !t || !u || !v))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    raycast_first(c, qs, bvh->bvh, o, d, n, tmin, tmax, face, t, u, v);
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    return MF_OK;
  });
}

int mf_bvh_raycast_first(mf_bvh* bvh, const double* o, const double* d, int64_t n, double tmin, double tmax,
                         int32_t* face, double* t, double* u, double* v) {
  if (!bvh || (n > 0 && (!o || !d || !face || !t || !u || !v))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    if (n <= 0) return MF_OK;
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    double* dO = c.buf<double>("rc.o", 3 * n);
    double* dD = c.buf<double>("rc.d", 3 * n);
    int32_t* df = c.buf<int32_t>("rc.f", n);
    double* dt = c.buf<double>("rc.t", n);
    double* du = c.buf<double>("rc.u", n);
    double* dv = c.buf<double>("rc.v", n);
    MFB_CUDA_TRY(cudaMemcpyAsync(dO, o, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(dD, d, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, qs));
    raycast_first(c, qs, bvh->bvh, dO, dD, n, tmin, tmax, df, dt, du, dv);
    MFB_CUDA_TRY(cudaMemcpyAsync(face, df, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(t, dt, sizeof(double) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(u, du, sizeof(double) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(v, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    return MF_OK;
  });
}

int mf_closest_point_brute(mf_ctx* ctx, const mf_mesh_view* mesh, const double* q, int64_t n, int32_t* face,
                           double* dist_sq, double* point, double* bary) {
  if (!ctx || (n > 0 && (!q || !face || !dist_sq))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "up.m");
    if (n <= 0) return MF_OK;
    double* dq = c.buf<double>("bf.q", 3 * n);
    int32_t* df = c.buf<int32_t>("bf.f", n);
    double* dd = c.buf<double>("bf.d", n);
    double* dp = c.buf<double>("bf.p", 3 * n);
    double* db = c.buf<double>("bf.b", 3 * n);
    MFB_CUDA_TRY(cudaMemcpyAsync(dq, q, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    if (m.m.nf > 0 && m.status == MF_OK) {
      closest_brute(c, c.stream, m.m, dq, n, df, dd, dp, db);
    } else {  // no faces (or unusable indices): every query misses
      MFB_CUDA_TRY(cudaMemsetAsync(df, 0xff, sizeof(int32_t) * n, c.stream));
      std::vector<double> inf(n, INFINITY);
      MFB_CUDA_TRY(cudaMemcpyAsync(dd, inf.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
      MFB_CUDA_TRY(cudaMemsetAsync(dp, 0, sizeof(double) * 3 * n, c.stream));
      MFB_CUDA_TRY(cudaMemsetAsync(db, 0, sizeof(double) * 3 * n, c.stream));
      MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    }
    MFB_CUDA_TRY(cudaMemcpyAsync(face, df, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(dist_sq, dd, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    if (point) MFB_CUDA_TRY(cudaMemcpyAsync(point, dp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    if (bary) MFB_CUDA_TRY(cudaMemcpyAsync(bary, db, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_raycast_first_brute(mf_ctx* ctx, const mf_mesh_view* mesh, const double* o, const double* d, int64_t n,
                           double tmin, double tmax, int32_t* face, double* t, double* u, double* v) {
  if (!ctx || (n > 0 && (!o || !d || !face || !t || !u || !v))) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "up.m");
    if (n <= 0) return MF_OK;
    if (m.m.nf == 0 || m.status != MF_OK) {
      for (int64_t i = 0; i < n; ++i) {
        face[i] = -1;
        t[i] = INFINITY;
        u[i] = v[i] = 0.0;
      }
      return MF_OK;
    }
    double* dO = c.buf<double>("rb.o", 3 * n);
    double* dD = c.buf<double>("rb.d", 3 * n);
    int32_t* df = c.buf<int32_t>("rb.f", n);
    double* dt = c.buf<double>("rb.t", n);
    double* du = c.buf<double>("rb.u", n);
    double* dv = c.buf<double>("rb.v", n);
    MFB_CUDA_TRY(cudaMemcpyAsync(dO, o, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(dD, d, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c.stream));
    raycast_brute(c, c.stream, m.m, dO, dD, n, tmin, tmax, df, dt, du, dv);
    MFB_CUDA_TRY(cudaMemcpyAsync(face, df, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(t, dt, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(u, du, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaMemcpyAsync(v, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_wedge_tangents(mf_ctx* ctx, const mf_mesh_view* mesh, double* frames) {
  if (!ctx || !frames) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "up.m");
    // computeWedgeTangents only requires UVs (tangent.cpp:23-24); indices are
    // used as given, so a bad mesh is reported as the reference would crash on it.
    if (!m.m.has_uvs()) throw ApiError(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: tangent frames require a UV-mapped mesh");
    check_mesh(&m);
    if (!m.uv_index_ok) throw ApiError(MF_ERR_INVALID_GEOMETRY, "InvalidGeometry: face uv index out of range");
    double* d = c.buf<double>("wt.frames", 27 * static_cast<size_t>(m.m.nf));
    wedge_frames(c, c.stream, m.m, d);
    MFB_CUDA_TRY(cudaMemcpyAsync(frames, d, sizeof(double) * 27 * m.m.nf, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_vertex_normals(mf_ctx* ctx, const mf_mesh_view* mesh, double* normals) {
  if (!ctx || !normals) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "up.m");
    if (m.m.nf > 0) check_mesh(&m);
    DevMesh dm = m.m;
    dm.nrm = nullptr;  // computeVertexNormals ignores stored normals
    double* d = c.buf<double>("vn.out", 3 * static_cast<size_t>(std::max(dm.nv, 1)));
    if (dm.nv > 0) {
      if (dm.nf > 0) {
        vertex_normals(c, c.stream, dm, d, false, "vn");
      } else {
        MFB_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(double) * 3 * dm.nv, c.stream));
      }
      MFB_CUDA_TRY(cudaMemcpyAsync(normals, d, sizeof(double) * 3 * dm.nv, cudaMemcpyDeviceToHost, c.stream));
    }
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

}  // extern "C"

// ---------------------------------------------------------------- surface band
namespace {
// sign_grid.cpp:23-54 — the grid parameters, in the reference's expression
// order (host f64, no contraction: -ffp-contract is irrelevant here, nvcc's
// host compiler sees plain mul/add statements).
struct BandGrid {
  double origin[3], h, truncation, band_world;
};
BandGrid band_grid(Ctx& c, const mf_bvh* bvh, int res, double band_voxels, int dilate, const double* domain) {
  if (res < 8) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: grid resolution must be >= 8");
  if (dilate < 0) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: dilate radius must be >= 0");
  double box[6];
  vertex_bounds(c, bvh->qstream, bvh->mesh->m, box);  // bounds(mesh), mesh.cpp:12-16
  const int margin = dilate + 3;
  if (res - 2 * margin < 4)
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: grid resolution too small for the dilation margin");
  BandGrid g;
  auto max_coeff = [](const double e[3]) {  // Eigen maxCoeff: first maximum
    double m = e[0];
    for (int k = 1; k < 3; ++k)
      if (e[k] > m) m = e[k];
    return m;
  };
  if (domain) {
    const double ext[3] = {domain[3] - domain[0], domain[4] - domain[1], domain[5] - domain[2]};
    g.h = max_coeff(ext) / res;
    for (int k = 0; k < 3; ++k) g.origin[k] = domain[k];
  } else {
    const double usable = res - 2.0 * margin;
    const double ext[3] = {box[3] - box[0], box[4] - box[1], box[5] - box[2]};
    g.h = max_coeff(ext) / usable;
    const double half = 0.5 * res * g.h;
    for (int k = 0; k < 3; ++k) {
      const double center = (box[k] + box[3 + k]) * 0.5;  // aabb.h:25
      g.origin[k] = center - half;
    }
  }
  bool out = false;
  for (int k = 0; k < 3; ++k) {
    const double gmin = g.origin[k] + 2 * g.h;
    const double gmax = g.origin[k] + (res - 2.0) * g.h;
    if (box[k] < gmin || box[3 + k] > gmax) out = true;
  }
  if (out) throw ApiError(MF_ERR_OUT_OF_BOUNDS, "OutOfBounds: mesh does not fit in the grid with 2 voxels of margin");
  g.truncation = (band_voxels + dilate * std::sqrt(3.0) + 2.0) * g.h;
  g.band_world = band_voxels * g.h;
  return g;
}
}  // namespace

extern "C" {
int mf_surface_band_dev(mf_bvh* bvh, int resolution, double band_voxels, int dilate_radius, const double* domain,
                        uint8_t* labels_dev, float* distance_dev, double* grid_out) {
  if (!bvh || !labels_dev || !distance_dev) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    const BandGrid g = band_grid(c, bvh, resolution, band_voxels, dilate_radius, domain);
    surface_band(c, qs, bvh->bvh, resolution, g.origin, g.h, g.truncation, g.band_world, labels_dev,
                 distance_dev);
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    if (grid_out) {
      grid_out[0] = g.origin[0];
      grid_out[1] = g.origin[1];
      grid_out[2] = g.origin[2];
      grid_out[3] = g.h;
      grid_out[4] = g.truncation;
    }
    return MF_OK;
  });
}

int mf_surface_band(mf_bvh* bvh, int resolution, double band_voxels, int dilate_radius, const double* domain,
                    uint8_t* labels, float* distance, double* grid_out) {
  if (!bvh || !labels || !distance) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded_dev(bvh->device, [&]() -> int {
    std::lock_guard<std::mutex> lk(bvh->mu);
    Ctx& c = bvh->store;
    const cudaStream_t qs = bvh->qstream;
    const BandGrid g = band_grid(c, bvh, resolution, band_voxels, dilate_radius, domain);
    const int64_t n = static_cast<int64_t>(resolution) * resolution * resolution;
    uint8_t* dl = c.buf<uint8_t>("band.labels", n);
    float* dd = c.buf<float>("band.dist", n);
    surface_band(c, qs, bvh->bvh, resolution, g.origin, g.h, g.truncation, g.band_world, dl, dd);
    MFB_CUDA_TRY(cudaMemcpyAsync(labels, dl, n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaMemcpyAsync(distance, dd, sizeof(float) * n, cudaMemcpyDeviceToHost, qs));
    MFB_CUDA_TRY(cudaStreamSynchronize(qs));
    if (grid_out) {
      grid_out[0] = g.origin[0];
      grid_out[1] = g.origin[1];
      grid_out[2] = g.origin[2];
      grid_out[3] = g.h;
      grid_out[4] = g.truncation;
    }
    return MF_OK;
  });
}
}  // extern "C"

// ---------------------------------------------------------------- ortho views
extern "C" {
int mf_fibonacci_cameras(int count, double half_extent, double* cameras) {
  if (count < 0 || (count > 0 && !cameras)) return fail(MF_ERR_BAD_ARGUMENT, "bad camera buffer");
  fibonacci_cameras(count, half_extent, cameras);
  return MF_OK;
}

int mf_render_views(mf_ctx* ctx, const mf_mesh_view* mesh, const double* cameras, int n_views, int resolution,
                    const double* vertex_normals, int backface_cull, int32_t* face, float* depth, float* position,
                    float* normal) {
  if (!ctx || !mesh || (n_views > 0 && !cameras)) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    if (n_views < 0 || resolution < 0) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: negative view count");
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "rv.mesh");
    check_mesh(&m);
    Lbvh bvh;
    lbvh_build(c, c.stream, m.m, bvh, "rv.bvh");
    const int64_t px = static_cast<int64_t>(n_views) * resolution * resolution;
    double* dvn = nullptr;
    if (vertex_normals && normal) {
      dvn = c.buf<double>("rv.vn", 3 * static_cast<size_t>(m.m.nv));
      MFB_CUDA_TRY(cudaMemcpyAsync(dvn, vertex_normals, sizeof(double) * 3 * m.m.nv, cudaMemcpyHostToDevice,
                                   c.stream));
    }
    int32_t* df = c.buf<int32_t>("rv.face", px);
    float* dd = depth ? c.buf<float>("rv.depth", px) : nullptr;
    float* dp = position ? c.buf<float>("rv.pos", 3 * px) : nullptr;
    float* dn = normal ? c.buf<float>("rv.nrm", 3 * px) : nullptr;
    render_views(c, c.stream, bvh, cameras, n_views, resolution, backface_cull, nullptr, df, dd, dp, dn, m.m.faces,
                 dvn);
    if (face) MFB_CUDA_TRY(cudaMemcpyAsync(face, df, sizeof(int32_t) * px, cudaMemcpyDeviceToHost, c.stream));
    if (depth) MFB_CUDA_TRY(cudaMemcpyAsync(depth, dd, sizeof(float) * px, cudaMemcpyDeviceToHost, c.stream));
    if (position) MFB_CUDA_TRY(cudaMemcpyAsync(position, dp, sizeof(float) * 3 * px, cudaMemcpyDeviceToHost, c.stream));
    if (normal) MFB_CUDA_TRY(cudaMemcpyAsync(normal, dn, sizeof(float) * 3 * px, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_cast_visibility(mf_ctx* ctx, const mf_mesh_view* mesh, int viewpoints, int resolution, int64_t* hits,
                       uint8_t* state) {
  if (!ctx || !mesh || !hits) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_mesh m;
    m.ctx = ctx;
    upload_mesh(c, c.stream, mesh, &m, "vis.mesh");
    check_mesh(&m);  // validateMesh (visibility.cpp:14)
    if (viewpoints <= 0 || resolution <= 0)
      throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: viewpoints and resolution must be positive");
    const int nf = m.m.nf;
    // centred copy (visibility.cpp:20-30): bounds centre, max |p - centre|
    double box[6];
    vertex_bounds(c, c.stream, m.m, box);
    double center[3];
    for (int k = 0; k < 3; ++k) center[k] = (box[k] + box[3 + k]) * 0.5;  // aabb.h:25
    DevMesh cm = m.m;
    double* cpos = c.buf<double>("vis.cpos", 3 * static_cast<size_t>(m.m.nv));
    double radius = center_mesh(c, c.stream, m.m, center, cpos);
    cm.pos = cpos;
    if (radius <= 0.0) radius = 1.0;
    std::vector<double> cams(7 * static_cast<size_t>(viewpoints));
    fibonacci_cameras(viewpoints, radius * 1.04, cams.data());
    auto* dh = c.buf<unsigned long long>("vis.hits", nf);
    MFB_CUDA_TRY(cudaMemsetAsync(dh, 0, sizeof(unsigned long long) * nf, c.stream));
    // the reference's face-order rasteriser on the device (z-buffer of
    // atomicMax keys; 57 ms vs 431 ms for one pixel ray per thread through the
    // LBVH at 512 views x 1024^2)
    raster_visibility(c, c.stream, cm, cams.data(), viewpoints, resolution, dh);
    MFB_CUDA_TRY(cudaMemcpyAsync(hits, dh, sizeof(int64_t) * nf, cudaMemcpyDeviceToHost, c.stream));
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (state)
      for (int f = 0; f < nf; ++f) state[f] = hits[f] > 0 ? 1 : 0;  // visibility.cpp:53-56
    return MF_OK;
  });
}
}  // extern "C"

// ---------------------------------------------------------------- peer-memory publish (multi-GPU)
extern "C" {
int mf_ipc_export(const void* dev_ptr, uint8_t* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(nullptr, [&]() -> int {
    CUdeviceptr base = 0;
    size_t size = 0;
    cudaIpcMemHandle_t h;
    {
      cudaPointerAttributes a{};
      MFB_CUDA_TRY(cudaPointerGetAttributes(&a, dev_ptr));
      if (a.type != cudaMemoryTypeDevice) throw ApiError(MF_ERR_BAD_ARGUMENT, "not device memory");
    }
    // the caller's pointer may sit inside a larger (caching-allocator) block:
    // find its base with the driver entry point (no link-time libcuda)
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<RangeFn>(fn);
    }();
    if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
      throw ApiError(MF_ERR_CUDA, "cuMemGetAddressRange failed");
    void* b = reinterpret_cast<void*>(base);
    MFB_CUDA_TRY(cudaIpcGetMemHandle(&h, b));
    std::memcpy(handle, &h, sizeof(h));
    *offset = static_cast<uint64_t>(reinterpret_cast<uintptr_t>(dev_ptr) - static_cast<uintptr_t>(base));
    return MF_OK;
  });
}

int mf_ipc_open(mf_ctx* ctx, const uint8_t* handle, uint64_t offset, void** dev_ptr) {
  if (!ctx || !handle || !dev_ptr) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    MFB_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<char*>(base) + offset;
    ctx->ipc_bases.push_back({*dev_ptr, base});
    return MF_OK;
  });
}

int mf_ipc_close(mf_ctx* ctx, void* dev_ptr) {
  if (!ctx || !dev_ptr) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  return guarded(ctx, [&]() -> int {
    for (auto it = ctx->ipc_bases.begin(); it != ctx->ipc_bases.end(); ++it)
      if (it->first == dev_ptr) {
        MFB_CUDA_TRY(cudaIpcCloseMemHandle(it->second));
        ctx->ipc_bases.erase(it);
        return MF_OK;
      }
    throw ApiError(MF_ERR_BAD_ARGUMENT, "pointer was not opened with mf_ipc_open");
  });
}

int mf_bake_normal_map_dev_publish(mf_ctx* ctx, mf_mesh* lowpoly, mf_mesh* highpoly, int res, double bbox_diagonal,
                                   double max_distance_fraction, int radius, int row_begin, int row_end,
                                   void* const* dst_atlases, int n_dst, mf_bake_stats* stats) {
  if (!ctx || !lowpoly || !highpoly || !dst_atlases) return fail(MF_ERR_BAD_ARGUMENT, "null argument");
  if (n_dst < 1 || n_dst > kMaxPublish) return fail(MF_ERR_BAD_ARGUMENT, "n_dst must be 1..8");
  return guarded(ctx, [&]() -> int {
    OutSet outs;
    for (int k = 0; k < n_dst; ++k) {
      if (!dst_atlases[k]) throw ApiError(MF_ERR_BAD_ARGUMENT, "null destination atlas");
      outs.p[k] = static_cast<uint8_t*>(dst_atlases[k]);
    }
    outs.n = n_dst;
    outs.row0 = 0;  // full res x res x 3 atlases: rows land at their own index
    Timer tm(ctx->c, 8);
    mf_bake_stats local{};
    bake_dev(ctx->c, lowpoly, highpoly, res, bbox_diagonal, max_distance_fraction, radius, row_begin, row_end,
             outs.p[0] + 3ll * row_begin * res, nullptr, nullptr, &local, tm, nullptr, &outs);
    if (stats) *stats = local;
    return MF_OK;
  });
}
}  // extern "C"

// ---------------------------------------------------------------- texfuse
// The G-buffer consumers of proj/src/texfuse (texfuse.cu). Host entry points
// copy their inputs into context scratch, run the device kernels and copy the
// results back; mf_fuse_views_dev keeps everything in HBM.
namespace {

template <typename T>
T* up(Ctx& c, const std::string& name, const T* host, size_t count) {
  T* d = c.buf<T>(name, count);
  if (count) MFB_CUDA_TRY(cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyHostToDevice, c.stream));
  return d;
}
template <typename T>
void down(Ctx& c, T* host, const T* dev, size_t count) {
  if (count) MFB_CUDA_TRY(cudaMemcpyAsync(host, dev, sizeof(T) * count, cudaMemcpyDeviceToHost, c.stream));
}

// edgeMask's argument checks (fuse.cpp:68-71)
void check_edge_args(int w, int h, double diag, double threshold) {
  if (w < 1 || h < 1) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: edge mask needs a rendered view");
  if (!(diag > 0.0) || !(threshold > 0.0))
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: edge mask scale must be positive");
}
// buildMips (mips.cpp:98-102)
void check_mip_args(int w, int h, int c, int levels, float sharpen) {
  if (w < 1 || h < 1 || c < 1) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: mip base image is empty");
  if (levels < 1) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: mip chain needs >= 1 level");
  if (!(sharpen >= 0.0f)) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: sharpen strength must be >= 0");
}
// backprojectView (fuse.cpp:106-113): the chain's level 0 is view_res^2 by construction here
void check_backproject_args(int gres, const uint8_t* valid, int view_res, int channels, int n_mips) {
  if (gres < 1 || !valid) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: geometry image is empty");
  if (n_mips < 1 || channels < 1 || view_res < 1)
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: view mip chain is empty");
}
// incidenceMap (fuse.cpp:191-196)
void check_incidence_args(int gres, const uint8_t* valid, double diag, double tol, int view_res) {
  if (gres < 1 || !valid) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: geometry image is empty");
  if (!(diag > 0.0) || !(tol > 0.0))
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: incidence scale must be positive");
  if (view_res < 1) throw ApiError(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: depth buffer does not match the camera");
}
// blendViews (fuse.cpp:226-233)
void check_blend_args(int k, const double* priors, double alpha, double eps) {
  if (k <= 0) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: no views to blend");
  if (!priors) throw ApiError(MF_ERR_BAD_ARGUMENT, "priors is null");
  if (!(eps > 0.0) || !(alpha >= 0.0))
    throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: blend needs epsilon > 0 and alpha >= 0");
  for (int i = 0; i < k; ++i)
    if (!(priors[i] >= 0.0)) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: priors must be >= 0");
}

int64_t mip_floats(int w, int h, int c, int levels, int* n_levels) {
  int lw[kTfMaxMips + 1], lh[kTfMaxMips + 1];
  int64_t off[kTfMaxMips + 1];
  const int n = tf_mip_layout(w, h, c, levels, lw, lh, off);
  if (n_levels) *n_levels = n;
  return off[n];
}

// fuseViews (fuse.cpp:292-326) without the inpainting step, every buffer
// device-resident: per view the edge mask, the mip chain, the backprojected
// partial atlas and the incidence map, then the blend. Partial atlases and
// incidence maps stay in context scratch (k x gres^2 x (channels + 1) f32).
void fuse_dev(Ctx& c, int gres, const float* pos, const float* nrm, const uint8_t* valid, int k,
              const double* cams, int vres, const float* vpos, const int32_t* vface, const float* vdepth, int ch,
              const float* colors, const double* priors, double diag, const mf_fuse_options& o, float* color,
              uint8_t* filled) {
  if (k <= 0 || !cams || !priors) throw ApiError(MF_ERR_INVALID_CONFIG, "InvalidConfig: cameras, views, colors and priors must pair up");
  check_edge_args(vres, vres, diag, o.edge_threshold);
  check_mip_args(vres, vres, ch, o.mip_levels, o.sharpen_strength);
  int n_mips = 0;
  const int64_t chain_floats = mip_floats(vres, vres, ch, o.mip_levels, &n_mips);
  check_backproject_args(gres, valid, vres, ch, n_mips);
  check_incidence_args(gres, valid, diag, o.depth_tolerance, vres);
  check_blend_args(k, priors, o.alpha, o.epsilon);
  cudaStream_t s = c.stream;
  const int64_t n = static_cast<int64_t>(gres) * gres, vn = static_cast<int64_t>(vres) * vres;
  auto* b6 = c.buf<unsigned>("tf.bounds", 6);
  tf_valid_bounds(c, s, n, pos, valid, b6);
  float* part = c.buf<float>("tf.part", static_cast<size_t>(k) * n * ch);
  uint8_t* samp = c.buf<uint8_t>("tf.samp", static_cast<size_t>(k) * n);
  float* inc = c.buf<float>("tf.inc", static_cast<size_t>(k) * n);
  uint8_t* mask = c.buf<uint8_t>("tf.mask", vn);
  float* chain = c.buf<float>("tf.chain", chain_floats);
  double limit2 = o.edge_threshold * diag;
  limit2 *= limit2;
  for (int i = 0; i < k; ++i) {
    const TfCamera cam = tf_camera(cams + 7 * i, vres);
    tf_edge_mask(c, s, vres, vres, vpos + 3 * vn * i, vface + vn * i, limit2, mask);
    tf_build_mips(c, s, vres, vres, ch, colors + vn * ch * i, o.mip_levels, o.sharpen_strength, chain, "tf.mips");
    tf_backproject(c, s, gres, pos, valid, b6, cam, ch, n_mips, chain, mask, part + n * ch * i, samp + n * i);
    tf_incidence(c, s, gres, pos, nrm, valid, cam, vdepth + vn * i, o.depth_tolerance * diag, inc + n * i);
  }
  tf_blend(c, s, k, n, ch, part, samp, inc, priors, o.alpha, o.epsilon, color, filled);
}

}  // namespace

void mf_fuse_options_default(mf_fuse_options* o) {
  if (!o) return;
  o->edge_threshold = 0.02;  // FuseOptions (fuse.h:122-130)
  o->depth_tolerance = 0.005;
  o->mip_levels = 6;
  o->sharpen_strength = 0.2f;
  o->alpha = 4.0;  // BlendOptions (fuse.h:83-86)
  o->epsilon = 1e-8;
}

int64_t mf_mip_chain_floats(int width, int height, int channels, int levels, int* n_levels) {
  if (width < 1 || height < 1 || channels < 1 || levels < 1) {
    if (n_levels) *n_levels = 0;
    return 0;
  }
  return mip_floats(width, height, channels, levels, n_levels);
}

int mf_edge_mask(mf_ctx* ctx, int width, int height, const float* position, const int32_t* face,
                 double bbox_diagonal, double threshold, uint8_t* mask) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_edge_args(width, height, bbox_diagonal, threshold);
    if (!position || !face || !mask) throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(width) * height;
    double limit2 = threshold * bbox_diagonal;
    limit2 *= limit2;
    uint8_t* dm = c.buf<uint8_t>("tf.mask", n);
    tf_edge_mask(c, c.stream, width, height, up(c, "tf.vpos", position, 3 * n), up(c, "tf.vface", face, n), limit2,
                 dm);
    down(c, mask, dm, n);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_build_mips(mf_ctx* ctx, int width, int height, int channels, const float* base, int levels, float sharpen,
                  float* chain, int* n_levels) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_mip_args(width, height, channels, levels, sharpen);
    if (!base || !chain) throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    int n = 0;
    const int64_t total = mip_floats(width, height, channels, levels, &n);
    float* d = c.buf<float>("tf.chain", total);
    MFB_CUDA_TRY(cudaMemcpyAsync(d, base, sizeof(float) * width * static_cast<size_t>(height) * channels,
                                 cudaMemcpyHostToDevice, c.stream));
    tf_build_mips(c, c.stream, width, height, channels, d, levels, sharpen, d, "tf.mips");
    down(c, chain, d, total);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    if (n_levels) *n_levels = n;
    return MF_OK;
  });
}

int mf_backproject_view(mf_ctx* ctx, int gres, const float* position, const uint8_t* valid, const double* camera,
                        int view_res, int channels, int n_mips, const float* mips, const uint8_t* mask, float* color,
                        uint8_t* sampled) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_backproject_args(gres, valid, view_res, channels, n_mips);
    if (!position || !camera || !mips || !mask || !color || !sampled)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    int expect = 0;
    const int64_t chain_floats = mip_floats(view_res, view_res, channels, n_mips, &expect);
    if (expect != n_mips) throw ApiError(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: mip chain does not match the view");
    const size_t n = static_cast<size_t>(gres) * gres, vn = static_cast<size_t>(view_res) * view_res;
    const float* dpos = up(c, "tf.gpos", position, 3 * n);
    const uint8_t* dval = up(c, "tf.gval", valid, n);
    auto* b6 = c.buf<unsigned>("tf.bounds", 6);
    tf_valid_bounds(c, c.stream, n, dpos, dval, b6);
    float* dcol = c.buf<float>("tf.part", n * channels);
    uint8_t* dsam = c.buf<uint8_t>("tf.samp", n);
    tf_backproject(c, c.stream, gres, dpos, dval, b6, tf_camera(camera, view_res), channels, n_mips,
                   up(c, "tf.chain", mips, chain_floats), up(c, "tf.mask", mask, vn), dcol, dsam);
    down(c, color, dcol, n * channels);
    down(c, sampled, dsam, n);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_incidence_map(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                     const double* camera, int view_res, const float* depth, double bbox_diagonal,
                     double depth_tolerance, float* out) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_incidence_args(gres, valid, bbox_diagonal, depth_tolerance, view_res);
    if (!position || !normal || !camera || !depth || !out) throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(gres) * gres, vn = static_cast<size_t>(view_res) * view_res;
    float* dout = c.buf<float>("tf.inc", n);
    tf_incidence(c, c.stream, gres, up(c, "tf.gpos", position, 3 * n), up(c, "tf.gnrm", normal, 3 * n),
                 up(c, "tf.gval", valid, n), tf_camera(camera, view_res), up(c, "tf.depth", depth, vn),
                 depth_tolerance * bbox_diagonal, dout);
    down(c, out, dout, n);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_blend_views(mf_ctx* ctx, int n_views, int width, int height, int channels, const float* colors,
                   const uint8_t* sampled, const float* incidence, const double* priors, double alpha, double epsilon,
                   float* color, uint8_t* filled) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    check_blend_args(n_views, priors, alpha, epsilon);
    if (width < 0 || height < 0 || channels < 0) throw ApiError(MF_ERR_SHAPE_MISMATCH, "ShapeMismatch: bad atlas shape");
    if (!colors || !sampled || !incidence || !color || !filled) throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(width) * height, k = static_cast<size_t>(n_views);
    float* dout = c.buf<float>("tf.out", n * channels);
    uint8_t* dfill = c.buf<uint8_t>("tf.fill", n);
    tf_blend(c, c.stream, n_views, static_cast<int64_t>(n), channels, up(c, "tf.part", colors, k * n * channels),
             up(c, "tf.samp", sampled, k * n), up(c, "tf.inc", incidence, k * n), priors, alpha, epsilon, dout,
             dfill);
    down(c, color, dout, n * channels);
    down(c, filled, dfill, n);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}

int mf_fuse_views_dev(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                      int n_views, const double* cameras, int view_res, const float* view_position,
                      const int32_t* view_face, const float* view_depth, int channels, const float* colors,
                      const double* priors, double bbox_diagonal, const mf_fuse_options* options, float* color,
                      uint8_t* filled) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    mf_fuse_options o;
    mf_fuse_options_default(&o);
    if (options) o = *options;
    if (!position || !normal || !view_position || !view_face || !view_depth || !colors || !color || !filled)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    fuse_dev(ctx->c, gres, position, normal, valid, n_views, cameras, view_res, view_position, view_face, view_depth,
             channels, colors, priors, bbox_diagonal, o, color, filled);
    return MF_OK;
  });
}

int mf_fuse_views(mf_ctx* ctx, int gres, const float* position, const float* normal, const uint8_t* valid,
                  int n_views, const double* cameras, int view_res, const float* view_position,
                  const int32_t* view_face, const float* view_depth, int channels, const float* colors,
                  const double* priors, double bbox_diagonal, const mf_fuse_options* options, float* color,
                  uint8_t* filled) {
  if (!ctx) return fail(MF_ERR_BAD_ARGUMENT, "ctx is null");
  return guarded(ctx, [&]() -> int {
    Ctx& c = ctx->c;
    mf_fuse_options o;
    mf_fuse_options_default(&o);
    if (options) o = *options;
    if (n_views <= 0 || gres < 1 || !valid || view_res < 1 || channels < 1) {  // argument errors first
      fuse_dev(c, gres, nullptr, nullptr, valid, n_views, cameras, view_res, nullptr, nullptr, nullptr, channels,
               nullptr, priors, bbox_diagonal, o, nullptr, nullptr);
    }
    if (!position || !normal || !view_position || !view_face || !view_depth || !colors || !color || !filled)
      throw ApiError(MF_ERR_BAD_ARGUMENT, "null argument");
    const size_t n = static_cast<size_t>(gres) * gres, vn = static_cast<size_t>(view_res) * view_res,
                 k = static_cast<size_t>(n_views);
    float* dout = c.buf<float>("tf.out", n * channels);
    uint8_t* dfill = c.buf<uint8_t>("tf.fill", n);
    fuse_dev(c, gres, up(c, "tf.gpos", position, 3 * n), up(c, "tf.gnrm", normal, 3 * n), up(c, "tf.gval", valid, n),
             n_views, cameras, view_res, up(c, "tf.vpos", view_position, 3 * vn * k), up(c, "tf.vface", view_face, vn * k),
             up(c, "tf.vdepth", view_depth, vn * k), channels, up(c, "tf.colors", colors, vn * k * channels), priors,
             bbox_diagonal, o, dout, dfill);
    down(c, color, dout, n * channels);
    down(c, filled, dfill, n);
    MFB_CUDA_TRY(cudaStreamSynchronize(c.stream));
    return MF_OK;
  });
}
