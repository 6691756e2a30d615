// Scene ingest and deterministic scene generators (host C++).
//
// These run once per scene, off the frame path. They must nevertheless
// produce exactly the reference's scenes (same vertices, quads, materials,
// camera doubles) because every parity test starts from them:
//   OBJ/MTL/camera parsing  proj/src/scene.cpp:195-454
//   look-at camera          proj/src/scene.cpp:128-158
//   matrix inverse          proj/src/scene.cpp:86-126
//   synthetic scenes        proj/src/synthetic.cpp:27-204
//   quad grouping           proj/src/grouping.cpp:25-177
// The BASELINE.json workloads (stack64k, tiny4m, mixed16m) have no reference
// generator; their recipes are in SURVEY.md 8(d) and DESIGN.md.
#include <algorithm>
#include <array>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <type_traits>
#include <unordered_map>
#include <numeric>
#include <random>
#include <sstream>

#include "veil_internal.hpp"

namespace veil {

Scene::Scene() {}

Scene::~Scene() {
  if (device) release_device_scene(device);
  for (DeviceScene* d : shards)
    if (d) release_device_scene(d);
}

double Scene::degenerate_quad_percent() const {
  if (quads.empty()) return 0.0;
  if (degenerate_version == geometry_version) return degenerate_cache;  // per-frame report
  size_t n = 0;
  for (const veil_quad& q : quads) {
    bool t0 = q.v[0] == q.v[1] || q.v[1] == q.v[2] || q.v[0] == q.v[2];
    bool t1 = q.v[0] == q.v[2] || q.v[2] == q.v[3] || q.v[0] == q.v[3];
    if (t0 || t1) ++n;
  }
  degenerate_cache = 100.0 * double(n) / double(quads.size());
  degenerate_version = geometry_version;
  return degenerate_cache;
}

void validate_camera(const Camera& c, bool extended) {
  if (c.width <= 0 || c.height <= 0)
    throw Error(VEIL_ERR_INVALID_ARG, "viewport dimensions must be positive");
  int mw = extended ? kExtMaxViewport : kMaxViewportWidth;
  int mh = extended ? kExtMaxViewport : kMaxViewportHeight;
  if (c.width > mw || c.height > mh) {
    if (extended)
      throw Error(VEIL_ERR_INVALID_ARG, "viewport exceeds the 16384x16384 extended limit");
    throw Error(VEIL_ERR_INVALID_ARG, "viewport exceeds the 2560x2048 limit");
  }
}

void validate_scene(const Scene& s) {
  validate_camera(s.camera, s.extended);
  for (size_t i = 0; i < s.quads.size(); ++i) {
    for (uint32_t v : s.quads[i].v)
      if (v >= s.vertices.size())
        throw Error(VEIL_ERR_INVALID_ARG, "quad " + std::to_string(i) + " references vertex " +
                                              std::to_string(v) + " out of range");
    if (s.quads[i].material >= s.materials.size())
      throw Error(VEIL_ERR_INVALID_ARG,
                  "quad " + std::to_string(i) + " references material out of range");
  }
  for (const veil_material& m : s.materials)
    if (m.texture >= int(s.textures.size()))
      throw Error(VEIL_ERR_INVALID_ARG, "material references texture out of range");
}

// ------------------------------------------------------------- matrices

namespace {

struct D3 {
  double x, y, z;
};
D3 sub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
D3 crs(D3 a, D3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double dt(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
D3 nrm(D3 a) {
  double l2 = dt(a, a);
  if (l2 <= 0.0) return {0, 0, 0};
  double inv = 1.0 / std::sqrt(l2);
  return {a.x * inv, a.y * inv, a.z * inv};
}

void mat_mul(const double* a, const double* b, double* out) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int k = 0; k < 4; ++k) s += a[i * 4 + k] * b[k * 4 + j];
      out[i * 4 + j] = s;
    }
}

}  // namespace

bool mat4_inverse(const double* in, double* out) {
  double a[4][8];
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 4; ++j) a[i][j] = in[i * 4 + j];
    for (int j = 0; j < 4; ++j) a[i][4 + j] = i == j ? 1.0 : 0.0;
  }
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    for (int r = col + 1; r < 4; ++r)
      if (std::abs(a[r][col]) > std::abs(a[piv][col])) piv = r;
    if (std::abs(a[piv][col]) < 1e-14) return false;
    if (piv != col)
      for (int j = 0; j < 8; ++j) std::swap(a[piv][j], a[col][j]);
    double inv_p = 1.0 / a[col][col];
    for (int j = 0; j < 8; ++j) a[col][j] *= inv_p;
    for (int r = 0; r < 4; ++r) {
      if (r == col) continue;
      double f = a[r][col];
      if (f == 0.0) continue;
      for (int j = 0; j < 8; ++j) a[r][j] -= f * a[col][j];
    }
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) out[i * 4 + j] = a[i][4 + j];
  return true;
}

Camera look_at_camera(const double from_[3], const double at_[3], const double up_[3],
                      double fov_deg, double near_z, double far_z, int width, int height) {
  D3 from{from_[0], from_[1], from_[2]}, at{at_[0], at_[1], at_[2]}, up{up_[0], up_[1], up_[2]};
  D3 fwd = nrm(sub(at, from));
  D3 right = nrm(crs(fwd, up));
  D3 vup = crs(right, fwd);
  double view[16] = {right.x, right.y, right.z, -dt(right, from),
                     vup.x,   vup.y,   vup.z,   -dt(vup, from),
                     -fwd.x,  -fwd.y,  -fwd.z,  dt(fwd, from),
                     0.0,     0.0,     0.0,     1.0};
  double f = 1.0 / std::tan(fov_deg * (3.14159265358979323846 / 180.0) * 0.5);
  double aspect = double(width) / double(height);
  double proj[16] = {0};
  proj[0] = f / aspect;
  proj[5] = f;
  proj[10] = far_z / (near_z - far_z);
  proj[11] = near_z * far_z / (near_z - far_z);
  proj[14] = -1.0;
  Camera c;
  mat_mul(proj, view, c.m);
  c.width = width;
  c.height = height;
  c.has_eye = true;
  c.eye[0] = from.x;
  c.eye[1] = from.y;
  c.eye[2] = from.z;
  return c;
}

// -------------------------------------------------------------- textures

namespace {

Texture texture_from_image(const Image8& img) {
  Texture t;
  TextureLevel base;
  base.width = img.width;
  base.height = img.height;
  base.texels.resize(size_t(img.width) * img.height * 4);
  for (size_t i = 0; i < base.texels.size(); ++i) base.texels[i] = img.rgba[i] / 255.0f;
  t.levels.push_back(std::move(base));
  while (t.levels.back().width > 1 || t.levels.back().height > 1) {
    const TextureLevel& s = t.levels.back();
    TextureLevel n;
    n.width = std::max(1, s.width / 2);
    n.height = std::max(1, s.height / 2);
    n.texels.resize(size_t(n.width) * n.height * 4);
    for (int y = 0; y < n.height; ++y)
      for (int x = 0; x < n.width; ++x) {
        int x0 = std::min(2 * x, s.width - 1), x1 = std::min(2 * x + 1, s.width - 1);
        int y0 = std::min(2 * y, s.height - 1), y1 = std::min(2 * y + 1, s.height - 1);
        for (int c = 0; c < 4; ++c) {
          // (t00 + t10) + t01 + t11, then * 0.25f (reference scene.cpp:180-186)
          float v = s.texels[(size_t(y0) * s.width + x0) * 4 + c] +
                    s.texels[(size_t(y0) * s.width + x1) * 4 + c] +
                    s.texels[(size_t(y1) * s.width + x0) * 4 + c] +
                    s.texels[(size_t(y1) * s.width + x1) * 4 + c];
          n.texels[(size_t(y) * n.width + x) * 4 + c] = v * 0.25f;
        }
      }
    t.levels.push_back(std::move(n));
  }
  return t;
}

// ------------------------------------------------------------ text ingest
//
// OBJ / MTL / camera-config ingest (behaviour of reference scene.cpp:195-454:
// the same scenes, vertex numbering, materials, camera doubles and error
// messages). Files are read whole and scanned line by line with a cursor
// that tokenises on whitespace and reads numbers the way an istream does
// (strtof for floats, strtod for doubles, failing on an incomplete number);
// OBJ directives dispatch through a keyword switch, and each distinct
// (position, uv, normal) corner becomes a vertex, numbered by first use.


[[noreturn]] void parse_error(const std::string& path, int line, const std::string& what) {
  throw Error(VEIL_ERR_PARSE, path + ":" + std::to_string(line) + ": " + what);
}

std::string slurp(const std::string& path, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(VEIL_ERR_IO, std::string("cannot open ") + what + " " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

std::string parent_dir(const std::string& p) {
  const size_t s = p.find_last_of('/');
  return s == std::string::npos ? std::string() : p.substr(0, s);
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

// One line of text with a read position.
class Cursor {
 public:
  Cursor(const char* b, const char* e) : p_(b), e_(e) {}
  void skip_space() {
    while (p_ < e_ && is_space(*p_)) ++p_;
  }
  bool word(std::string* out) {  // next whitespace-delimited token
    skip_space();
    const char* b = p_;
    while (p_ < e_ && !is_space(*p_)) ++p_;
    if (b == p_) return false;
    out->assign(b, p_);
    return true;
  }
  template <typename T>
  bool number(T* out) {  // a decimal number at the cursor; false leaves *out alone
    skip_space();
    const char* b = p_;
    const char* q = p_;
    while (q < e_ && (std::isdigit((unsigned char)*q) || *q == '+' || *q == '-' || *q == '.' || *q == 'e' ||
                      *q == 'E'))
      ++q;
    if (q == b) return false;
    const std::string run(b, q);
    char* end = nullptr;
    T v;
    if constexpr (std::is_same_v<T, float>)
      v = std::strtof(run.c_str(), &end);
    else
      v = std::strtod(run.c_str(), &end);
    if (end != run.c_str() + run.size()) return false;
    p_ = q;
    *out = v;
    return true;
  }

 private:
  const char* p_;
  const char* e_;
};

// Calls fn(line_number, cursor) for every line of text.
template <typename Fn>
void for_each_line(const std::string& text, Fn&& fn) {
  const char* p = text.data();
  const char* end = p + text.size();
  int line_no = 0;
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    const char* le = nl ? nl : end;
    Cursor c(p, le);
    fn(++line_no, c);
    p = nl ? nl + 1 : end;
  }
}

// atoi of a field: optional sign, then digits; anything else ends it.
int leading_int(const std::string& s, size_t b, size_t e) {
  while (b < e && is_space(s[b])) ++b;
  bool neg = false;
  if (b < e && (s[b] == '+' || s[b] == '-')) neg = s[b++] == '-';
  long long v = 0;
  for (; b < e && std::isdigit((unsigned char)s[b]); ++b) v = v * 10 + (s[b] - '0');
  return int(neg ? -v : v);
}

struct Corner {
  int v = 0, vt = 0, vn = 0;  // 1-based or negative OBJ references, 0 = absent
  bool operator==(const Corner& o) const { return v == o.v && vt == o.vt && vn == o.vn; }
};
struct CornerHash {
  size_t operator()(const Corner& c) const {
    uint64_t h = uint64_t(uint32_t(c.v)) * 0x9e3779b97f4a7c15ull;
    h ^= uint64_t(uint32_t(c.vt)) + 0x7f4a7c159e3779b9ull + (h << 6) + (h >> 2);
    h ^= uint64_t(uint32_t(c.vn)) + 0x94d049bb133111ebull + (h << 6) + (h >> 2);
    return size_t(h);
  }
};

// "v", "v/vt", "v/vt/vn" or "v//vn"
Corner parse_corner(const std::string& tok, const std::string& path, int line) {
  Corner c;
  const size_t s1 = tok.find('/');
  if (s1 == std::string::npos) {
    c.v = leading_int(tok, 0, tok.size());
    return c;
  }
  c.v = leading_int(tok, 0, s1);
  const size_t s2 = tok.find('/', s1 + 1);
  if (s2 == std::string::npos) {
    c.vt = leading_int(tok, s1 + 1, tok.size());
    return c;
  }
  c.vt = leading_int(tok, s1 + 1, s2);
  c.vn = leading_int(tok, s2 + 1, tok.size());
  if (c.v == 0) parse_error(path, line, "malformed face vertex '" + tok + "'");
  return c;
}

// An OBJ reference into a list of `count` entries -> 0-based index.
size_t resolve(int ref, size_t count, const std::string& path, int line) {
  const long long i = ref > 0 ? (long long)ref - 1 : (long long)count + ref;
  if (ref == 0 || i < 0 || i >= (long long)count)
    parse_error(path, line, "index " + std::to_string(ref) + " out of range");
  return size_t(i);
}

veil_material default_material() {
  veil_material m{};
  m.base_color[0] = m.base_color[1] = m.base_color[2] = m.base_color[3] = 1.0f;
  m.opacity = 1.0f;
  m.texture = -1;
  m.flags = VEIL_MATERIAL_VERTEX_COLORS | VEIL_MATERIAL_VERTEX_NORMALS;
  return m;
}

// newmtl / Kd / d / map_Kd; anything else is ignored.
void read_mtl(const std::string& path, Scene* s, std::map<std::string, uint32_t>* names) {
  const std::string text = slurp(path, "material file");
  const std::string dir = parent_dir(path);
  veil_material* cur = nullptr;
  std::string key, arg;
  for_each_line(text, [&](int line, Cursor& c) {
    if (!c.word(&key) || key[0] == '#') return;
    if (key == "newmtl") {
      arg.clear();
      c.word(&arg);
      (*names)[arg] = uint32_t(s->materials.size());
      s->materials.push_back(default_material());
      s->material_names.push_back(arg);
      cur = &s->materials.back();
      return;
    }
    if (!cur) return;
    if (key == "Kd") {
      for (int k = 0; k < 3 && c.number(&cur->base_color[k]); ++k) {
      }
    } else if (key == "d") {
      c.number(&cur->opacity);
      if (cur->opacity < 0.0f || cur->opacity > 1.0f) parse_error(path, line, "dissolve outside [0,1]");
    } else if (key == "map_Kd") {
      arg.clear();
      c.word(&arg);
      if (!dir.empty()) arg = dir + "/" + arg;
      s->textures.push_back(texture_from_image(read_png(arg)));
      cur->texture = int(s->textures.size()) - 1;
      cur->flags |= VEIL_MATERIAL_UVS;
    }
  });
}

enum class Directive { kOther, kPosition, kNormal, kTexcoord, kFace, kUseMtl, kMtlLib };

Directive directive(const std::string& k) {
  switch (k.size()) {
    case 1:
      return k[0] == 'v' ? Directive::kPosition : k[0] == 'f' ? Directive::kFace : Directive::kOther;
    case 2:
      return k == "vn" ? Directive::kNormal : k == "vt" ? Directive::kTexcoord : Directive::kOther;
    case 6:
      return k == "usemtl" ? Directive::kUseMtl : k == "mtllib" ? Directive::kMtlLib : Directive::kOther;
    default:
      return Directive::kOther;
  }
}

// The OBJ attribute pools and the corner -> vertex numbering of one load.
struct ObjBuilder {
  Scene* s;
  const std::string& path;
  std::vector<std::array<float, 3>> positions, normals;
  std::vector<std::array<float, 4>> colours;
  std::vector<std::array<float, 2>> texcoords;
  std::unordered_map<Corner, uint32_t, CornerHash> numbering;

  uint32_t vertex(const Corner& c, int line) {
    auto hit = numbering.find(c);
    if (hit != numbering.end()) return hit->second;
    veil_vertex v{};
    const size_t pi = resolve(c.v, positions.size(), path, line);
    std::copy(positions[pi].begin(), positions[pi].end(), v.position);
    std::copy(colours[pi].begin(), colours[pi].end(), v.color);
    if (c.vt) {
      const auto& t = texcoords[resolve(c.vt, texcoords.size(), path, line)];
      v.uv[0] = t[0];
      v.uv[1] = t[1];
      s->flags |= VEIL_SCENE_HAS_UVS;
    }
    if (c.vn) {
      // unit normal in float (reference math.hpp:80-85 normalize)
      const auto& n = normals[resolve(c.vn, normals.size(), path, line)];
      const float len2 = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
      const float inv = len2 <= 0.0f ? 0.0f : 1.0f / std::sqrt(len2);
      for (int k = 0; k < 3; ++k) v.normal[k] = len2 <= 0.0f ? 0.0f : n[k] * inv;
      s->flags |= VEIL_SCENE_HAS_NORMALS;
    }
    const uint32_t id = uint32_t(s->vertices.size());
    s->vertices.push_back(v);
    numbering.emplace(c, id);
    return id;
  }
};

void add_default_material(Scene* s) {
  if (!s->materials.empty()) return;
  s->materials.push_back(default_material());
  s->material_names.push_back("default");
}

}  // namespace

Camera load_camera_file(const std::string& path) {
  const std::string text = slurp(path, "camera config");
  Camera cam;
  bool have_matrix = false, have_look = false;
  double from[3] = {0, 0, 5}, at[3] = {0, 0, 0}, up[3] = {0, 1, 0};
  double fov = 60.0, nz = 0.1, fz = 100.0;
  // "key = values" lines: the key loses its blanks; lines without '=' or
  // starting with '#' are skipped
  int line_no = 0;
  size_t pos = 0;
  while (pos < text.size()) {
    size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) nl = text.size();
    const std::string row = text.substr(pos, nl - pos);
    pos = nl + 1;
    ++line_no;
    const size_t eq = row.find('=');
    if (row.empty() || row[0] == '#' || eq == std::string::npos) continue;
    std::string key;
    for (size_t i = 0; i < eq; ++i)
      if (row[i] != ' ' && row[i] != '\t') key += row[i];
    Cursor c(row.data() + eq + 1, row.data() + row.size());
    auto take = [&](int n, double* out) {
      for (int i = 0; i < n; ++i)
        if (!c.number(&out[i])) parse_error(path, line_no, "expected " + std::to_string(n) + " numbers");
    };
    double v[16];
    if (key == "view_projection") {
      take(16, v);
      std::copy(v, v + 16, cam.m);
      have_matrix = true;
    } else if (key == "width" || key == "height") {
      take(1, v);
      (key == "width" ? cam.width : cam.height) = int(v[0]);
    } else if (key == "eye") {
      take(3, cam.eye);
      cam.has_eye = true;
    } else if (key == "look_from" || key == "look_at") {
      take(3, key == "look_from" ? from : at);
      have_look = true;
    } else if (key == "up") {
      take(3, up);
    } else if (key == "fov_deg" || key == "near" || key == "far") {
      take(1, key == "fov_deg" ? &fov : key == "near" ? &nz : &fz);
    } else {
      parse_error(path, line_no, "unknown camera key '" + key + "'");
    }
  }
  if (have_look && !have_matrix) {
    // the friendly form: a look-at camera; an explicit eye still wins
    Camera look = look_at_camera(from, at, up, fov, nz, fz, cam.width, cam.height);
    if (cam.has_eye) std::copy(cam.eye, cam.eye + 3, look.eye);
    cam = look;
  }
  validate_camera(cam, false);
  return cam;
}

void load_obj_scene(Scene* s, const std::string& mesh, const std::string& mtl,
                    const std::string& cam) {
  const std::string text = slurp(mesh, "mesh file");
  const std::string dir = parent_dir(mesh);
  std::map<std::string, uint32_t> names;
  if (!mtl.empty()) read_mtl(mtl, s, &names);
  ObjBuilder ob{s, mesh, {}, {}, {}, {}, {}};
  uint32_t material = 0;
  std::string key, tok;
  std::vector<Corner> face;
  for_each_line(text, [&](int line, Cursor& c) {
    if (!c.word(&key) || key[0] == '#') return;
    switch (directive(key)) {
      case Directive::kPosition: {
        std::array<float, 3> p;
        if (!(c.number(&p[0]) && c.number(&p[1]) && c.number(&p[2]))) parse_error(mesh, line, "malformed vertex");
        std::array<float, 4> col = {1.0f, 1.0f, 1.0f, 1.0f};
        float rgb[3];
        if (c.number(&rgb[0]) && c.number(&rgb[1]) && c.number(&rgb[2])) {  // optional vertex colour
          std::copy(rgb, rgb + 3, col.begin());
          s->flags |= VEIL_SCENE_HAS_COLORS;
        }
        ob.positions.push_back(p);
        ob.colours.push_back(col);
        break;
      }
      case Directive::kNormal: {
        std::array<float, 3> n;
        if (!(c.number(&n[0]) && c.number(&n[1]) && c.number(&n[2]))) parse_error(mesh, line, "malformed normal");
        ob.normals.push_back(n);
        break;
      }
      case Directive::kTexcoord: {
        std::array<float, 2> t;
        if (!(c.number(&t[0]) && c.number(&t[1]))) parse_error(mesh, line, "malformed texcoord");
        ob.texcoords.push_back(t);
        break;
      }
      case Directive::kFace: {
        face.clear();
        while (c.word(&tok)) face.push_back(parse_corner(tok, mesh, line));
        if (face.size() != 3 && face.size() != 4)
          parse_error(mesh, line, "unsupported face arity " + std::to_string(face.size()));
        add_default_material(s);
        veil_quad q{};
        q.material = material;
        for (size_t i = 0; i < face.size(); ++i) q.v[i] = ob.vertex(face[i], line);
        if (face.size() == 3) q.v[3] = q.v[2];  // a triangle is a quad with v3 == v2
        s->quads.push_back(q);
        break;
      }
      case Directive::kUseMtl: {
        tok.clear();
        c.word(&tok);
        const auto it = names.find(tok);
        if (it != names.end()) {
          material = it->second;
        } else {  // unknown names select the default material
          add_default_material(s);
          material = 0;
        }
        break;
      }
      case Directive::kMtlLib:
        if (mtl.empty()) {
          tok.clear();
          c.word(&tok);
          read_mtl(dir.empty() ? tok : dir + "/" + tok, s, &names);
        }
        break;
      case Directive::kOther:
        break;
    }
  });
  add_default_material(s);
  if (!cam.empty()) s->camera = load_camera_file(cam);
  validate_scene(*s);
}

// -------------------------------------------------- synthetic generators

namespace {

// Seeded uniforms of the reference (synthetic.cpp:29-43).
struct Rng {
  std::mt19937_64 e;
  explicit Rng(uint64_t seed) : e(seed) {}
  double uniform(double lo, double hi) {
    double u = double(e() >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
  }
  int uniform_int(int lo, int hi) { return lo + int(e() % uint64_t(hi - lo + 1)); }
  float channel() { return float(uniform_int(40, 255)) / 255.0f; }
};

struct Builder {
  Scene* s;
  Builder(Scene* sc, int w, int h, const char* mat_name) : s(sc) {
    s->camera = Camera();
    s->camera.width = w;
    s->camera.height = h;
    s->materials.push_back(default_material());
    s->material_names.push_back(mat_name);
    s->flags = VEIL_SCENE_HAS_COLORS | VEIL_SCENE_HAS_NORMALS;
  }
  uint32_t vertex(double x, double y, double z, const float c[4]) {
    veil_vertex v{};
    v.position[0] = float(x);
    v.position[1] = float(y);
    v.position[2] = float(z);
    v.normal[2] = -1.0f;
    for (int k = 0; k < 4; ++k) v.color[k] = c[k];
    s->vertices.push_back(v);
    return uint32_t(s->vertices.size() - 1);
  }
  void quad(const double (*xy)[2], const double* z, const float c[4]) {
    veil_quad q{};
    for (int i = 0; i < 4; ++i) q.v[i] = vertex(xy[i][0], xy[i][1], z[i], c);
    s->quads.push_back(q);
  }
  void triangle(const double (*xy)[2], const double* z, const float c[4]) {
    veil_quad q{};
    for (int i = 0; i < 3; ++i) q.v[i] = vertex(xy[i][0], xy[i][1], z[i], c);
    q.v[3] = q.v[2];
    s->quads.push_back(q);
  }
};

float alpha_grid(Rng& r, float lo, float hi) {
  int a = int(std::lround(lo * 255.0f));
  int b = int(std::lround(hi * 255.0f));
  return float(r.uniform_int(a, b)) / 255.0f;
}

void color3(Rng& r, float c[4]) {
  c[0] = r.channel();
  c[1] = r.channel();
  c[2] = r.channel();
}

const double kFull[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};

}  // namespace

void synthetic_scene(Scene* s, const std::string& kind, uint64_t seed, int width, int height) {
  int w = width > 0 ? width : 512, h = height > 0 ? height : 512;
  Rng rng(seed);
  if (kind == "layered_quads") {  // synthetic.cpp:104-120 (8 layers, alpha 0.6)
    Builder b(s, w, h, "synthetic");
    const int n = 8;
    for (int i = 0; i < n; ++i) {
      double z = 0.2 + 0.6 * double(i) / double(std::max(1, n - 1));
      float alpha = float(std::lround(0.6f * 255.0f)) / 255.0f;
      float c[4];
      color3(rng, c);
      c[3] = alpha;
      double d[4] = {z, z, z, z};
      b.quad(kFull, d, c);
    }
  } else if (kind == "intersecting_shells") {  // synthetic.cpp:122-145 (32 sheets)
    Builder b(s, w, h, "synthetic");
    const int n = 32;
    for (int i = 0; i < n; ++i) {
      double slope = rng.uniform(0.10, 0.30);
      slope = slope * (rng.uniform_int(0, 1) ? 1.0 : -1.0);
      double center = rng.uniform(-0.3, 0.3);
      bool tilt_x = i % 3 != 2;
      float c[4];
      color3(rng, c);
      c[3] = 128.0f / 255.0f;
      double d[4];
      for (int k = 0; k < 4; ++k) {
        double t = tilt_x ? kFull[k][0] : kFull[k][1];
        d[k] = 0.5 + slope * (t - center);
      }
      b.quad(kFull, d, c);
    }
  } else if (kind == "random_soup") {  // synthetic.cpp:147-166 (4000 triangles)
    Builder b(s, w, h, "synthetic");
    for (int i = 0; i < 4000; ++i) {
      double cx = rng.uniform(-0.85, 0.85);
      double cy = rng.uniform(-0.85, 0.85);
      double z = rng.uniform(0.05, 0.95);
      double r = rng.uniform(0.02, 0.12);
      double xy[3][2], d[3];
      for (int k = 0; k < 3; ++k) {
        xy[k][0] = cx + rng.uniform(-r, r);
        xy[k][1] = cy + rng.uniform(-r, r);
        d[k] = z + rng.uniform(-0.01, 0.01);
      }
      float c[4];
      color3(rng, c);
      c[3] = alpha_grid(rng, 0.25f, 0.85f);
      b.triangle(xy, d, c);
    }
  } else if (kind == "dense_bin") {  // synthetic.cpp:168-195
    Builder b(s, w, h, "synthetic");
    double bw = 2.0 * kBinSize / double(w);
    double bh = 2.0 * kBinSize / double(h);
    double x0 = -1.0 + 4 * bw, y0 = -1.0 + 4 * bh;
    auto square = [&](double cx, double cy, double z, double r) {
      double xy[4][2] = {{cx - r, cy - r}, {cx + r, cy - r}, {cx + r, cy + r}, {cx - r, cy + r}};
      double d[4] = {z, z, z, z};
      float c[4];
      color3(rng, c);
      c[3] = alpha_grid(rng, 0.3f, 0.7f);
      b.quad(xy, d, c);
    };
    for (int i = 0; i < 600; ++i) {
      double cx = x0 + rng.uniform(0.2, 0.8) * bw;
      double cy = y0 + rng.uniform(0.2, 0.8) * bh;
      double z = rng.uniform(0.1, 0.9);
      double r = rng.uniform(0.05, 0.15) * bw;
      square(cx, cy, z, r);
    }
    for (int i = 0; i < 60; ++i) {
      double cx = rng.uniform(-0.9, 0.9);
      double cy = rng.uniform(-0.9, 0.9);
      double z = rng.uniform(0.1, 0.9);
      double r = rng.uniform(0.02, 0.06);
      square(cx, cy, z, r);
    }
  } else {
    throw Error(VEIL_ERR_INVALID_ARG, "unknown synthetic scene kind");
  }
}

// ------------------------------------------------- BASELINE.json workloads

namespace {

float grid_channel(std::mt19937_64& e) { return float(e() % 216 + 40) / 255.0f; }

// Jittered grid mesh over NDC [-1,1]^2 with per-vertex depth and colour.
void grid_mesh(Builder& b, std::mt19937_64& e, int nx, int ny) {
  auto U = [&](double lo, double hi) { return lo + (hi - lo) * (double(e() >> 11) * 0x1.0p-53); };
  const double cw = 2.0 / nx, ch = 2.0 / ny;
  uint32_t base = uint32_t(b.s->vertices.size());
  b.s->vertices.reserve(b.s->vertices.size() + size_t(nx + 1) * (ny + 1));
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      double x = -1.0 + cw * i, y = -1.0 + ch * j;
      if (i > 0 && i < nx && j > 0 && j < ny) {
        double jx = U(-0.25, 0.25);
        double jy = U(-0.25, 0.25);
        x += jx * cw;
        y += jy * ch;
      }
      double z = U(0.2, 0.8);
      float c[4];
      c[0] = grid_channel(e);
      c[1] = grid_channel(e);
      c[2] = grid_channel(e);
      c[3] = 128.0f / 255.0f;
      b.vertex(x, y, z, c);
    }
  b.s->quads.reserve(b.s->quads.size() + size_t(nx) * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      veil_quad q{};
      uint32_t v00 = base + uint32_t(j * (nx + 1) + i);
      q.v[0] = v00;
      q.v[1] = v00 + 1;
      q.v[2] = v00 + 1 + uint32_t(nx + 1);
      q.v[3] = v00 + uint32_t(nx + 1);
      b.s->quads.push_back(q);
    }
}

// Axis-aligned translucent quads with half extents U(lo,hi) pixels, constant
// depth per quad (SURVEY.md 8(d), C2 recipe, strictly sequenced draws).
void stacked_quads(Builder& b, std::mt19937_64& e, uint32_t count, double lo, double hi, int w,
                   int h) {
  auto U = [&](double a, double c) { return a + (c - a) * (double(e() >> 11) * 0x1.0p-53); };
  for (uint32_t i = 0; i < count; ++i) {
    double hx_px = U(lo, hi);
    double hy_px = U(lo, hi);
    double cx = U(-1.0, 1.0);
    double cy = U(-1.0, 1.0);
    double z = U(0.05, 0.95);
    float c[4];
    c[0] = grid_channel(e);
    c[1] = grid_channel(e);
    c[2] = grid_channel(e);
    c[3] = float(e() % 151 + 64) / 255.0f;
    double hx = hx_px * 2.0 / w, hy = hy_px * 2.0 / h;
    double xy[4][2] = {{cx - hx, cy - hy}, {cx + hx, cy - hy}, {cx + hx, cy + hy}, {cx - hx, cy + hy}};
    double d[4] = {z, z, z, z};
    b.quad(xy, d, c);
  }
}

}  // namespace

void workload_scene(Scene* s, const std::string& name, uint64_t seed, int width, int height) {
  std::mt19937_64 e(seed);
  if (name == "stack64k") {  // C2
    int w = width > 0 ? width : 1920, h = height > 0 ? height : 1080;
    Builder b(s, w, h, "default");
    s->vertices.reserve(65536 * 4);
    s->quads.reserve(65536);
    stacked_quads(b, e, 65536, 12.0, 20.0, w, h);
  } else if (name == "tiny4m") {  // C4
    int w = width > 0 ? width : 3840, h = height > 0 ? height : 2160;
    Builder b(s, w, h, "default");
    s->extended = true;
    grid_mesh(b, e, 2048, 2048);
  } else if (name == "mixed16m") {  // C5
    int w = width > 0 ? width : 7680, h = height > 0 ? height : 4320;
    Builder b(s, w, h, "default");
    s->extended = true;
    grid_mesh(b, e, 4096, 3840);
    stacked_quads(b, e, 1048576, 4.0, 12.0, w, h);
  } else {
    throw Error(VEIL_ERR_INVALID_ARG, "unknown workload '" + name + "'");
  }
  validate_scene(*s);
}

// ---------------------------------------------------------- quad grouping

double group_quads(Scene* s) {
  struct Tri {
    uint32_t v[3];
    uint32_t mat;
  };
  std::vector<Tri> tris;
  for (const veil_quad& q : s->quads) {
    uint32_t t0[3] = {q.v[0], q.v[1], q.v[2]}, t1[3] = {q.v[0], q.v[2], q.v[3]};
    bool d0 = t0[0] == t0[1] || t0[1] == t0[2] || t0[0] == t0[2];
    bool d1 = t1[0] == t1[1] || t1[1] == t1[2] || t1[0] == t1[2];
    if (!d0 && !d1)
      throw Error(VEIL_ERR_INVALID_ARG,
                  "--group-quads requires a pure triangle mesh (quads already present)");
    if (d0 && d1) continue;
    const uint32_t* live = d0 ? t1 : t0;
    tris.push_back({{live[0], live[1], live[2]}, q.material});
  }
  // Candidates: same-material pairs sharing exactly one edge.
  std::map<std::pair<uint32_t, uint32_t>, std::vector<uint32_t>> by_edge;
  for (uint32_t t = 0; t < tris.size(); ++t) {
    const Tri& tr = tris[t];
    if (tr.v[0] == tr.v[1] || tr.v[1] == tr.v[2] || tr.v[0] == tr.v[2]) continue;
    for (int k = 0; k < 3; ++k) {
      uint32_t a = tr.v[k], b = tr.v[(k + 1) % 3];
      by_edge[{std::min(a, b), std::max(a, b)}].push_back(t);
    }
  }
  std::map<std::pair<uint32_t, uint32_t>, std::pair<int, std::pair<uint32_t, uint32_t>>> shared;
  for (const auto& [edge, ts] : by_edge)
    for (size_t i = 0; i < ts.size(); ++i)
      for (size_t j = i + 1; j < ts.size(); ++j) {
        auto& info = shared[{std::min(ts[i], ts[j]), std::max(ts[i], ts[j])}];
        info.first++;
        info.second = edge;
      }
  struct Cand {
    uint32_t t0, t1, e0, e1;
  };
  std::vector<Cand> cands;
  for (const auto& [pr, info] : shared) {
    if (info.first != 1) continue;
    if (tris[pr.first].mat != tris[pr.second].mat) continue;
    cands.push_back({pr.first, pr.second, info.second.first, info.second.second});
  }
  std::vector<uint32_t> per_tri(tris.size(), 0);
  for (const Cand& c : cands) per_tri[c.t0]++, per_tri[c.t1]++;
  std::vector<uint32_t> order(cands.size());
  std::iota(order.begin(), order.end(), 0);
  auto degree = [&](const Cand& c) { return (per_tri[c.t0] - 1) + (per_tri[c.t1] - 1); };
  std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    uint32_t dx = degree(cands[x]), dy = degree(cands[y]);
    if (dx != dy) return dx < dy;
    if (cands[x].t0 != cands[y].t0) return cands[x].t0 < cands[y].t0;
    return cands[x].t1 < cands[y].t1;
  });
  std::vector<int32_t> pair_of(tris.size(), -1);
  for (uint32_t n : order) {
    const Cand& c = cands[n];
    if (pair_of[c.t0] >= 0 || pair_of[c.t1] >= 0) continue;
    pair_of[c.t0] = int32_t(n);
    pair_of[c.t1] = int32_t(n);
  }
  std::vector<veil_quad> out;
  uint64_t degenerate = 0;
  for (uint32_t t = 0; t < tris.size(); ++t) {
    int32_t n = pair_of[t];
    veil_quad q{};
    if (n >= 0) {
      const Cand& c = cands[n];
      if (c.t0 != t) continue;
      const Tri& a = tris[c.t0];
      const Tri& b = tris[c.t1];
      auto is_shared = [&](uint32_t v) { return v == c.e0 || v == c.e1; };
      int ua = 0, ub = 0;
      while (is_shared(a.v[ua])) ++ua;
      while (is_shared(b.v[ub])) ++ub;
      q.v[0] = a.v[(ua + 2) % 3];
      q.v[1] = a.v[ua];
      q.v[2] = a.v[(ua + 1) % 3];
      q.v[3] = b.v[ub];
      q.material = a.mat;
    } else {
      q.v[0] = tris[t].v[0];
      q.v[1] = tris[t].v[1];
      q.v[2] = tris[t].v[2];
      q.v[3] = tris[t].v[2];
      q.material = tris[t].mat;
      ++degenerate;
    }
    out.push_back(q);
  }
  s->quads = std::move(out);
  s->geometry_version++;
  return s->quads.empty() ? 0.0 : 100.0 * double(degenerate) / double(s->quads.size());
}

}  // namespace veil
