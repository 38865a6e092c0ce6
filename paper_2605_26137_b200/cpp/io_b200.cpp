// io_b200.cpp — the formats either side of the bake:
// OBJ ingest / export (io/obj_io.cpp), PNG encode / decode (io/png_io.cpp)
// and the raw f32 raster / grid files (io/raster_io.cpp), host C++.
//
// readObj: the whole file is read once and parsed on all host threads over
// line-aligned chunks. Pass 1 counts v / vt / vn / f records per chunk; a
// prefix over chunks gives every record its slot and the element counts in
// force at each line (negative OBJ indices resolve against them, exactly as
// the reference's sequential reader does); pass 2 parses into place. Numbers
// are read with std::from_chars (correctly rounded, like istream's strtod).
// The first error in file order wins, as in the reference.
//
// PNG: chunks written directly over zlib. Rows are filtered adaptively
// (minimum sum of absolute filtered bytes over the five PNG filters, libpng's
// heuristic) in parallel, then row bands are deflated in parallel as one zlib
// stream: raw deflate per band primed with the previous band's last 32 KiB,
// sync-flushed, Adler-32 combined (the pigz construction).
#include <zlib.h>

#include <algorithm>
#include <array>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "meshforge/core/error.h"
#include "meshforge/io/obj_io.h"
#include "meshforge/io/png_io.h"
#include "meshforge/io/raster_io.h"

namespace meshforge {
namespace {

// ------------------------------------------------------------------ files
std::vector<char> slurp(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw Error(ErrorCode::IoError, "cannot open " + path);
  std::vector<char> buf;
  long n = -1;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
  }
  if (n >= 0) {  // regular file: one read into the final buffer
    buf.resize(static_cast<size_t>(n));
    const size_t got = n ? std::fread(buf.data(), 1, buf.size(), f) : 0;
    buf.resize(got);
  } else {  // pipes and the like
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  }
  std::fclose(f);
  return buf;
}

void spill(const std::string& path, const void* data, size_t bytes) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Error(ErrorCode::IoError, "cannot write " + path);
  const size_t put = bytes ? std::fwrite(data, 1, bytes, f) : 0;
  const bool ok = std::fclose(f) == 0 && put == bytes;
  if (!ok) throw Error(ErrorCode::IoError, "failed writing " + path);
}

int workers(size_t units, size_t min_per_worker) {
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<int>(std::max<size_t>(1, std::min(hw, units / std::max<size_t>(1, min_per_worker))));
}

template <class F>
void run_parallel(int n, F&& fn) {
  if (n <= 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> ts;
  ts.reserve(n);
  for (int i = 0; i < n; ++i) ts.emplace_back([&, i] { fn(i); });
  for (auto& t : ts) t.join();
}

// ------------------------------------------------------------------ OBJ
inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

struct Cursor {
  const char* p;
  const char* end;
  void skip() {
    while (p < end && is_space(*p)) ++p;
  }
  std::string_view token() {  // istream >> std::string
    skip();
    const char* b = p;
    while (p < end && !is_space(*p)) ++p;
    return {b, static_cast<size_t>(p - b)};
  }
  // istream >> double: leading blanks, optional '+', the longest number;
  // a failed extraction gives 0 and fails the rest of the line
  bool number(double& v, bool& failed) {
    if (failed) return false;
    skip();
    const char* b = p;
    if (b < end && *b == '+') ++b;
    const auto r = std::from_chars(b, end, v);
    if (r.ec == std::errc::result_out_of_range) {  // strtod saturates
      v = (b < end && *b == '-') ? -std::numeric_limits<double>::infinity()
                                 : std::numeric_limits<double>::infinity();
      p = r.ptr;
      return true;
    }
    if (r.ec != std::errc()) {
      v = 0.0;
      failed = true;
      return false;
    }
    p = r.ptr;
    return true;
  }
};

enum : int { kNone = 0, kV, kVt, kVn, kF };

int line_kind(std::string_view tag) {
  if (tag == "v") return kV;
  if (tag == "vt") return kVt;
  if (tag == "vn") return kVn;
  if (tag == "f") return kF;
  return kNone;
}

// obj_io.cpp:17-33: "v", "v/vt", "v/vt/vn", "v//vn"; absent or unparsable fields stay 0
void parse_corner(std::string_view t, int& v, int& vt, int& vn) {
  int* slot[3] = {&v, &vt, &vn};
  v = vt = vn = 0;
  size_t pos = 0;
  for (int field = 0; field < 3; ++field) {
    const size_t next = t.find('/', pos);
    const std::string_view part = t.substr(pos, next == std::string_view::npos ? std::string_view::npos : next - pos);
    if (!part.empty()) std::from_chars(part.data(), part.data() + part.size(), *slot[field]);
    if (next == std::string_view::npos) break;
    pos = next + 1;
  }
}

struct ObjCounts {
  int64_t v = 0, vt = 0, vn = 0, tris = 0;
};

struct ObjError {
  int64_t at = std::numeric_limits<int64_t>::max();  // byte offset of the failing line
  ErrorCode code = ErrorCode::InvalidGeometry;
  std::string msg;
  void set(int64_t pos, ErrorCode c, std::string m) {
    if (pos < at) {
      at = pos;
      code = c;
      msg = std::move(m);
    }
  }
};

// obj_io.cpp:35-41
bool resolve(int raw, int64_t count, int& out) {
  const int64_t idx = raw > 0 ? static_cast<int64_t>(raw) - 1 : count + raw;
  if (idx < 0 || idx >= count) return false;
  out = static_cast<int>(idx);
  return true;
}

template <class F>
void for_lines(const char* b, const char* e, F&& fn) {
  while (b < e) {
    const char* nl = static_cast<const char*>(std::memchr(b, '\n', static_cast<size_t>(e - b)));
    const char* le = nl ? nl : e;
    if (le > b && *b != '#') fn(b, le);  // empty and '#' lines skipped (obj_io.cpp:58)
    b = nl ? nl + 1 : e;
  }
}

}  // namespace

TriangleMesh readObj(const std::string& path) {
  const std::vector<char> text = slurp(path);
  const char* base = text.data();
  const size_t n = text.size();
  const int nt = workers(n, size_t{1} << 20);
  std::vector<size_t> cut(nt + 1, n);
  cut[0] = 0;
  for (int i = 1; i < nt; ++i) {
    size_t c = std::max(cut[i - 1], n * i / nt);
    while (c < n && base[c - 1] != '\n') ++c;
    cut[i] = c;
  }
  // pass 1: counts per chunk
  std::vector<ObjCounts> cnt(nt);
  run_parallel(nt, [&](int t) {
    ObjCounts& k = cnt[t];
    for_lines(base + cut[t], base + cut[t + 1], [&](const char* b, const char* e) {
      Cursor c{b, e};
      switch (line_kind(c.token())) {
        case kV: ++k.v; break;
        case kVt: ++k.vt; break;
        case kVn: ++k.vn; break;
        case kF: {
          int64_t corners = 0;
          while (!c.token().empty()) ++corners;
          if (corners >= 3) k.tris += corners - 2;
          break;
        }
        default: break;
      }
    });
  });
  std::vector<ObjCounts> off(nt + 1);
  for (int t = 0; t < nt; ++t) {
    off[t + 1].v = off[t].v + cnt[t].v;
    off[t + 1].vt = off[t].vt + cnt[t].vt;
    off[t + 1].vn = off[t].vn + cnt[t].vn;
    off[t + 1].tris = off[t].tris + cnt[t].tris;
  }
  const ObjCounts total = off[nt];
  if (total.tris > std::numeric_limits<int>::max() || total.v > std::numeric_limits<int>::max())
    throw Error(ErrorCode::InvalidGeometry, "obj too large");
  TriangleMesh mesh;
  mesh.positions.resize(total.v);
  mesh.uvs.resize(total.vt);
  std::vector<Eigen::Vector3d> normal_pool(total.vn);
  mesh.faces.resize(total.tris);
  std::vector<std::array<int, 3>> tri_uv(total.tris), tri_vn(total.tris);
  std::vector<ObjError> errs(nt);
  // pass 2: parse into place
  run_parallel(nt, [&](int t) {
    ObjCounts at = off[t];
    ObjError& err = errs[t];
    std::vector<std::array<int, 3>> corners;
    for_lines(base + cut[t], base + cut[t + 1], [&](const char* b, const char* e) {
      if (err.at != std::numeric_limits<int64_t>::max()) return;  // this chunk already failed
      Cursor c{b, e};
      const int kind = line_kind(c.token());
      bool failed = false;
      if (kind == kV || kind == kVn) {
        double x = 0, y = 0, z = 0;
        c.number(x, failed);
        c.number(y, failed);
        c.number(z, failed);
        if (kind == kV) mesh.positions[at.v++] = Eigen::Vector3d(x, y, z);
        else normal_pool[at.vn++] = Eigen::Vector3d(x, y, z);
      } else if (kind == kVt) {
        double u = 0, v = 0;
        c.number(u, failed);
        c.number(v, failed);
        mesh.uvs[at.vt++] = Eigen::Vector2d(u, v);
      } else if (kind == kF) {
        corners.clear();
        for (std::string_view tok = c.token(); !tok.empty(); tok = c.token()) {
          int v, vt, vn;
          parse_corner(tok, v, vt, vn);
          std::array<int, 3> r{-1, -1, -1};
          if (!resolve(v, at.v, r[0])) {
            err.set(b - base, ErrorCode::InvalidGeometry, "obj vertex index out of range");
            return;
          }
          if (vt != 0 && !resolve(vt, at.vt, r[1])) {
            err.set(b - base, ErrorCode::InvalidGeometry, "obj uv index out of range");
            return;
          }
          if (vn != 0 && !resolve(vn, at.vn, r[2])) {
            err.set(b - base, ErrorCode::InvalidGeometry, "obj normal index out of range");
            return;
          }
          corners.push_back(r);
        }
        if (corners.size() < 3) {
          err.set(b - base, ErrorCode::InvalidGeometry, "obj face with fewer than 3 corners");
          return;
        }
        for (size_t k = 2; k < corners.size(); ++k) {  // fan (obj_io.cpp:87-99)
          const auto& a = corners[0];
          const auto& p = corners[k - 1];
          const auto& q = corners[k];
          mesh.faces[at.tris] = Eigen::Vector3i(a[0], p[0], q[0]);
          tri_uv[at.tris] = {a[1], p[1], q[1]};
          tri_vn[at.tris] = {a[2], p[2], q[2]};
          ++at.tris;
        }
      }
    });
  });
  const ObjError* first = nullptr;
  for (const ObjError& e : errs)
    if (e.at != std::numeric_limits<int64_t>::max() && (!first || e.at < first->at)) first = &e;
  if (first) throw Error(first->code, first->msg);

  // uv sets only when every corner has one (obj_io.cpp:103-106)
  bool all_uv = true, all_vn = true;
  for (int64_t f = 0; f < total.tris && (all_uv || all_vn); ++f) {
    all_uv = all_uv && tri_uv[f][0] >= 0 && tri_uv[f][1] >= 0 && tri_uv[f][2] >= 0;
    all_vn = all_vn && tri_vn[f][0] >= 0 && tri_vn[f][1] >= 0 && tri_vn[f][2] >= 0;
  }
  if (all_uv) {  // (with no faces the reference keeps the uv pool too)
    mesh.faceUvs.resize(total.tris);
    for (int64_t f = 0; f < total.tris; ++f) mesh.faceUvs[f] = Eigen::Vector3i(tri_uv[f][0], tri_uv[f][1], tri_uv[f][2]);
  } else {
    mesh.uvs.clear();
  }
  // per-vertex normals only when every corner references one and each
  // vertex always names the same one (obj_io.cpp:108-128)
  if (all_vn && total.tris > 0) {
    std::vector<int> vnorm(mesh.positions.size(), -1);
    bool consistent = true;
    for (int64_t f = 0; f < total.tris && consistent; ++f)
      for (int k = 0; k < 3; ++k) {
        int& slot = vnorm[mesh.faces[f][k]];
        if (slot < 0) slot = tri_vn[f][k];
        else if (slot != tri_vn[f][k]) {
          consistent = false;
          break;
        }
      }
    if (consistent) {
      mesh.normals.assign(mesh.positions.size(), Eigen::Vector3d::UnitZ());
      for (size_t v = 0; v < mesh.positions.size(); ++v)
        if (vnorm[v] >= 0) mesh.normals[v] = normal_pool[vnorm[v]];
    }
  }
  if (mesh.positions.empty()) throw Error(ErrorCode::EmptyMesh, "obj has no vertices: " + path);
  return mesh;
}

namespace {
// "%.17g" (std::ostream with precision max_digits10, obj_io.cpp:141)
inline char* put_double(char* o, double v) {
  return std::to_chars(o, o + 32, v, std::chars_format::general, std::numeric_limits<double>::max_digits10).ptr;
}
inline char* put_int(char* o, int v) { return std::to_chars(o, o + 12, v).ptr; }
}  // namespace

void writeObj(const std::string& path, const TriangleMesh& mesh) {
  // obj_io.cpp:138-165 record by record; records formatted in parallel blocks
  const bool uv = mesh.hasUvs(), nrm = mesh.hasNormals();
  const size_t nv = mesh.positions.size(), nu = mesh.uvs.size(), nn = mesh.normals.size(), nf = mesh.faces.size();
  const size_t records = nv + nu + nn + nf;
  const int nt = workers(records, 1 << 16);
  std::vector<std::string> parts(nt);
  run_parallel(nt, [&](int t) {
    const size_t lo = records * t / nt, hi = records * (t + 1) / nt;
    std::string& s = parts[t];
    s.resize((hi - lo) * 80 + 64);
    char* o = s.data();
    for (size_t r = lo; r < hi; ++r) {
      if (r < nv) {
        const auto& p = mesh.positions[r];
        std::memcpy(o, "v ", 2);
        o = put_double(o + 2, p.x());
        *o++ = ' ';
        o = put_double(o, p.y());
        *o++ = ' ';
        o = put_double(o, p.z());
      } else if (r < nv + nu) {
        const auto& q = mesh.uvs[r - nv];
        std::memcpy(o, "vt ", 3);
        o = put_double(o + 3, q.x());
        *o++ = ' ';
        o = put_double(o, q.y());
      } else if (r < nv + nu + nn) {
        const auto& q = mesh.normals[r - nv - nu];
        std::memcpy(o, "vn ", 3);
        o = put_double(o + 3, q.x());
        *o++ = ' ';
        o = put_double(o, q.y());
        *o++ = ' ';
        o = put_double(o, q.z());
      } else {
        const size_t f = r - nv - nu - nn;
        *o++ = 'f';
        for (int k = 0; k < 3; ++k) {
          const int v = mesh.faces[f][k] + 1;
          *o++ = ' ';
          o = put_int(o, v);
          if (uv) {
            *o++ = '/';
            o = put_int(o, mesh.faceUvs[f][k] + 1);
            if (nrm) {
              *o++ = '/';
              o = put_int(o, v);
            }
          } else if (nrm) {
            *o++ = '/';
            *o++ = '/';
            o = put_int(o, v);
          }
        }
      }
      *o++ = '\n';
    }
    s.resize(static_cast<size_t>(o - s.data()));
  });
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw Error(ErrorCode::IoError, "cannot write " + path);
  bool ok = true;
  for (const auto& s : parts) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
  ok = std::fclose(f) == 0 && ok;
  if (!ok) throw Error(ErrorCode::IoError, "failed writing " + path);
}

// ------------------------------------------------------------------ PNG
namespace {

constexpr uint8_t kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

void put_be32(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(static_cast<uint8_t>(v >> 24));
  o.push_back(static_cast<uint8_t>(v >> 16));
  o.push_back(static_cast<uint8_t>(v >> 8));
  o.push_back(static_cast<uint8_t>(v));
}
uint32_t get_be32(const uint8_t* p) {
  return (static_cast<uint32_t>(p[0]) << 24) | (static_cast<uint32_t>(p[1]) << 16) |
         (static_cast<uint32_t>(p[2]) << 8) | p[3];
}
void put_chunk(std::vector<uint8_t>& o, const char* type, const uint8_t* data, size_t len) {
  put_be32(o, static_cast<uint32_t>(len));
  const size_t at = o.size();
  o.insert(o.end(), type, type + 4);
  if (len) o.insert(o.end(), data, data + len);
  put_be32(o, static_cast<uint32_t>(crc32(0L, o.data() + at, static_cast<uInt>(len + 4))));
}

inline uint8_t paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return static_cast<uint8_t>(pa <= pb && pa <= pc ? a : (pb <= pc ? b : c));
}

// One filtered row (filter byte + bytes): the filter with the least sum of
// |signed byte| wins (libpng's adaptive heuristic).
void filter_row(const uint8_t* cur, const uint8_t* prev, size_t len, int bpp, uint8_t* out,
                std::vector<uint8_t>& buf) {
  buf.resize(5 * len);
  uint64_t best = ~0ull;
  int pick = 0;
  for (int ft = 0; ft < 5; ++ft) {
    uint8_t* d = buf.data() + ft * len;
    uint64_t sum = 0;
    for (size_t i = 0; i < len; ++i) {
      const int a = i >= static_cast<size_t>(bpp) ? cur[i - bpp] : 0;
      const int b = prev ? prev[i] : 0;
      const int c = (prev && i >= static_cast<size_t>(bpp)) ? prev[i - bpp] : 0;
      uint8_t v = cur[i];
      switch (ft) {
        case 1: v = static_cast<uint8_t>(cur[i] - a); break;
        case 2: v = static_cast<uint8_t>(cur[i] - b); break;
        case 3: v = static_cast<uint8_t>(cur[i] - ((a + b) >> 1)); break;
        case 4: v = static_cast<uint8_t>(cur[i] - paeth(a, b, c)); break;
        default: break;
      }
      d[i] = v;
      sum += static_cast<uint64_t>(std::abs(static_cast<int>(static_cast<int8_t>(v))));
    }
    if (sum < best) {
      best = sum;
      pick = ft;
    }
  }
  out[0] = static_cast<uint8_t>(pick);
  std::memcpy(out + 1, buf.data() + pick * len, len);
}

}  // namespace

std::vector<std::uint8_t> encodePng(const ImageU8& image) {
  if (image.empty() || (image.channels != 1 && image.channels != 3))
    throw Error(ErrorCode::IoError, "png writer requires non-empty gray or rgb image");
  const int w = image.width, h = image.height, ch = image.channels;
  const size_t row = static_cast<size_t>(w) * ch, stride = row + 1;
  std::vector<uint8_t> filtered(stride * h);
  const int nt = workers(filtered.size(), size_t{1} << 18);
  run_parallel(nt, [&](int t) {
    std::vector<uint8_t> scratch;
    for (int y = h * t / nt; y < h * (t + 1) / nt; ++y)
      filter_row(image.data.data() + y * row, y ? image.data.data() + (y - 1) * row : nullptr, row, ch,
                 filtered.data() + y * stride, scratch);
  });
  // one zlib stream: header, raw-deflate bands (primed with the previous
  // band's tail, sync-flushed), final block, Adler-32 of all filtered bytes
  const size_t total = filtered.size();
  const int nb = workers(total, size_t{1} << 20);
  std::vector<std::vector<uint8_t>> band(nb);
  std::vector<uLong> adl(nb);
  std::vector<size_t> lo(nb + 1);
  for (int b = 0; b <= nb; ++b) lo[b] = total * b / nb;
  bool ok = true;
  run_parallel(nb, [&](int b) {
    z_stream z{};
    if (deflateInit2(&z, Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, 8, Z_DEFAULT_STRATEGY) != Z_OK) {
      ok = false;
      return;
    }
    if (b > 0) {
      const size_t dict = std::min<size_t>(32768, lo[b]);
      deflateSetDictionary(&z, filtered.data() + lo[b] - dict, static_cast<uInt>(dict));
    }
    const size_t len = lo[b + 1] - lo[b];
    band[b].resize(deflateBound(&z, static_cast<uLong>(len)) + 16);
    z.next_in = filtered.data() + lo[b];
    z.avail_in = static_cast<uInt>(len);
    z.next_out = band[b].data();
    z.avail_out = static_cast<uInt>(band[b].size());
    const int r = deflate(&z, b == nb - 1 ? Z_FINISH : Z_SYNC_FLUSH);
    if (r != (b == nb - 1 ? Z_STREAM_END : Z_OK)) ok = false;
    band[b].resize(band[b].size() - z.avail_out);
    deflateEnd(&z);
    adl[b] = adler32(adler32(0L, Z_NULL, 0), filtered.data() + lo[b], static_cast<uInt>(len));
  });
  if (!ok) throw Error(ErrorCode::IoError, "png encode failed");
  uLong a = adler32(0L, Z_NULL, 0);
  for (int b = 0; b < nb; ++b) a = adler32_combine(a, adl[b], static_cast<z_off_t>(lo[b + 1] - lo[b]));
  std::vector<uint8_t> idat{0x78, 0x9c};
  for (const auto& v : band) idat.insert(idat.end(), v.begin(), v.end());
  put_be32(idat, static_cast<uint32_t>(a));

  std::vector<uint8_t> out(kSig, kSig + 8);
  uint8_t ihdr[13];
  const uint32_t dims[2] = {static_cast<uint32_t>(w), static_cast<uint32_t>(h)};
  for (int k = 0; k < 2; ++k)
    for (int i = 0; i < 4; ++i) ihdr[4 * k + i] = static_cast<uint8_t>(dims[k] >> (24 - 8 * i));
  ihdr[8] = 8;                   // bit depth
  ihdr[9] = ch == 1 ? 0 : 2;     // gray / RGB
  ihdr[10] = ihdr[11] = ihdr[12] = 0;
  put_chunk(out, "IHDR", ihdr, 13);
  for (size_t at = 0; at < idat.size(); at += size_t{1} << 20)
    put_chunk(out, "IDAT", idat.data() + at, std::min(idat.size() - at, size_t{1} << 20));
  put_chunk(out, "IEND", nullptr, 0);
  return out;
}

ImageU8 decodePng(const std::uint8_t* bytes, std::size_t size) {
  auto fail = [] { return Error(ErrorCode::IoError, "png decode failed"); };
  if (!bytes || size < 8 || std::memcmp(bytes, kSig, 8) != 0) throw fail();
  uint32_t w = 0, h = 0;
  int depth = 0, ctype = -1, interlace = 0;
  std::vector<uint8_t> idat, plte;
  bool seen_end = false;
  for (size_t p = 8; p + 12 <= size && !seen_end;) {
    const uint32_t len = get_be32(bytes + p);
    if (p + 12 + static_cast<size_t>(len) > size) throw fail();
    const uint8_t* type = bytes + p + 4;
    const uint8_t* data = bytes + p + 8;
    if (crc32(crc32(0L, Z_NULL, 0), type, len + 4) != get_be32(data + len)) throw fail();
    if (!std::memcmp(type, "IHDR", 4) && len == 13) {
      w = get_be32(data);
      h = get_be32(data + 4);
      depth = data[8];
      ctype = data[9];
      interlace = data[12];
    } else if (!std::memcmp(type, "PLTE", 4)) {
      plte.assign(data, data + len);
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      seen_end = true;
    }
    p += 12 + static_cast<size_t>(len);
  }
  static const int kSamples[7] = {1, 0, 3, 1, 2, 0, 4};
  if (w == 0 || h == 0 || ctype < 0 || ctype > 6 || kSamples[ctype] == 0 || interlace != 0) throw fail();
  if (!(depth == 1 || depth == 2 || depth == 4 || depth == 8 || depth == 16)) throw fail();
  if ((ctype == 2 || ctype == 4 || ctype == 6) && depth < 8) throw fail();
  if (ctype == 3 && (depth > 8 || plte.empty())) throw fail();
  const int spp = kSamples[ctype];
  const size_t bits = static_cast<size_t>(w) * spp * depth;
  const size_t row = (bits + 7) / 8;
  const int bpp = std::max(1, spp * depth / 8);
  std::vector<uint8_t> raw((row + 1) * h);
  uLongf got = static_cast<uLongf>(raw.size());
  if (uncompress(raw.data(), &got, idat.data(), static_cast<uLong>(idat.size())) != Z_OK || got != raw.size())
    throw fail();
  // unfilter in place
  for (uint32_t y = 0; y < h; ++y) {
    uint8_t* r = raw.data() + y * (row + 1);
    const uint8_t ft = r[0];
    uint8_t* cur = r + 1;
    const uint8_t* prev = y ? raw.data() + (y - 1) * (row + 1) + 1 : nullptr;
    for (size_t i = 0; i < row; ++i) {
      const int a = i >= static_cast<size_t>(bpp) ? cur[i - bpp] : 0;
      const int b = prev ? prev[i] : 0;
      const int c = (prev && i >= static_cast<size_t>(bpp)) ? prev[i - bpp] : 0;
      switch (ft) {
        case 0: break;
        case 1: cur[i] = static_cast<uint8_t>(cur[i] + a); break;
        case 2: cur[i] = static_cast<uint8_t>(cur[i] + b); break;
        case 3: cur[i] = static_cast<uint8_t>(cur[i] + ((a + b) >> 1)); break;
        case 4: cur[i] = static_cast<uint8_t>(cur[i] + paeth(a, b, c)); break;
        default: throw fail();
      }
    }
  }
  // libpng's read transforms of the reference (png_io.cpp:57-66): 16 -> 8
  // bits (high byte), palette -> RGB, low-depth gray -> 8 bits, alpha stripped
  const int out_ch = (ctype == 0 || ctype == 4) ? 1 : 3;
  ImageU8 img(static_cast<int>(w), static_cast<int>(h), out_ch);
  for (uint32_t y = 0; y < h; ++y) {
    const uint8_t* src = raw.data() + y * (row + 1) + 1;
    for (uint32_t x = 0; x < w; ++x) {
      auto sample = [&](int s) -> int {  // 8-bit sample s of pixel x
        if (depth == 16) return src[(static_cast<size_t>(x) * spp + s) * 2];
        if (depth == 8) return src[static_cast<size_t>(x) * spp + s];
        const size_t bit = static_cast<size_t>(x) * depth;
        const int v = (src[bit / 8] >> (8 - depth - static_cast<int>(bit % 8))) & ((1 << depth) - 1);
        return ctype == 3 ? v : v * (255 / ((1 << depth) - 1));
      };
      uint8_t* dst = &img.at(static_cast<int>(x), static_cast<int>(y));
      if (ctype == 3) {
        const size_t e = static_cast<size_t>(sample(0)) * 3;
        if (e + 3 > plte.size()) throw fail();
        dst[0] = plte[e];
        dst[1] = plte[e + 1];
        dst[2] = plte[e + 2];
      } else if (out_ch == 1) {
        dst[0] = static_cast<uint8_t>(sample(0));
      } else {
        for (int k = 0; k < 3; ++k) dst[k] = static_cast<uint8_t>(sample(k));
      }
    }
  }
  return img;
}

void writePng(const std::string& path, const ImageU8& image) {
  const std::vector<uint8_t> bytes = encodePng(image);
  spill(path, bytes.data(), bytes.size());
}

ImageU8 readPng(const std::string& path) {
  const std::vector<char> bytes = slurp(path);
  if (bytes.empty()) throw Error(ErrorCode::IoError, "empty png file " + path);
  return decodePng(reinterpret_cast<const uint8_t*>(bytes.data()), bytes.size());
}

// ------------------------------------------------------------------ raw f32 files
void writeRasterF32(const std::string& path, const ImageF& image) {
  if (image.empty()) throw Error(ErrorCode::IoError, "refusing to write empty raster " + path);
  std::vector<char> buf(16 + image.data.size() * sizeof(float));
  const std::int32_t hdr[4] = {kRasterMagic, image.width, image.height, image.channels};
  std::memcpy(buf.data(), hdr, 16);
  std::memcpy(buf.data() + 16, image.data.data(), image.data.size() * sizeof(float));
  spill(path, buf.data(), buf.size());
}

ImageF readRasterF32(const std::string& path) {
  const std::vector<char> b = slurp(path);
  std::int32_t hdr[4];
  if (b.size() < sizeof(hdr)) throw Error(ErrorCode::IoError, "truncated file " + path);
  std::memcpy(hdr, b.data(), sizeof(hdr));
  if (hdr[0] != kRasterMagic) throw Error(ErrorCode::IoError, "bad raster magic in " + path);
  if (hdr[1] <= 0 || hdr[2] <= 0 || hdr[3] <= 0 || hdr[3] > 16)
    throw Error(ErrorCode::IoError, "bad raster dimensions in " + path);
  ImageF img(hdr[1], hdr[2], hdr[3]);
  const size_t bytes = img.data.size() * sizeof(float);
  if (b.size() < sizeof(hdr) + bytes) throw Error(ErrorCode::IoError, "truncated file " + path);
  std::memcpy(img.data.data(), b.data() + sizeof(hdr), bytes);
  return img;
}

void writeGridF32(const std::string& path, const GridFile& grid) {
  const size_t expected = static_cast<size_t>(grid.nx) * grid.ny * grid.nz;
  if (expected == 0 || grid.values.size() != expected)
    throw Error(ErrorCode::ShapeMismatch, "grid value count does not match dimensions");
  std::vector<char> buf(32 + expected * sizeof(float));
  const std::int32_t hdr[8] = {kGridMagic, kGridVersion, grid.nx, grid.ny, grid.nz, 0, 0, 0};
  std::memcpy(buf.data(), hdr, 32);
  std::memcpy(buf.data() + 32, grid.values.data(), expected * sizeof(float));
  spill(path, buf.data(), buf.size());
}

GridFile readGridF32(const std::string& path) {
  const std::vector<char> b = slurp(path);
  std::int32_t hdr[8];
  if (b.size() < sizeof(hdr)) throw Error(ErrorCode::IoError, "truncated file " + path);
  std::memcpy(hdr, b.data(), sizeof(hdr));
  if (hdr[0] != kGridMagic || hdr[1] != kGridVersion) throw Error(ErrorCode::IoError, "bad grid header in " + path);
  if (hdr[2] <= 0 || hdr[3] <= 0 || hdr[4] <= 0) throw Error(ErrorCode::IoError, "bad grid dimensions in " + path);
  GridFile g;
  g.nx = hdr[2];
  g.ny = hdr[3];
  g.nz = hdr[4];
  g.values.resize(static_cast<size_t>(g.nx) * g.ny * g.nz);
  const size_t bytes = g.values.size() * sizeof(float);
  if (b.size() < sizeof(hdr) + bytes) throw Error(ErrorCode::IoError, "truncated file " + path);
  std::memcpy(g.values.data(), b.data() + sizeof(hdr), bytes);
  return g;
}

}  // namespace meshforge
