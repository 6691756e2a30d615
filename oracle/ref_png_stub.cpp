// Test infrastructure only (never shipped, never on the product path).
//
// The reference's image.cpp needs libpng, whose headers are absent from this
// image. The oracle build of the reference links this
// file instead: a small zlib PNG reader (8-bit grey / grey+alpha / RGB / RGBA,
// non-interlaced, all five row filters) so the reference can load textured
// OBJ scenes for golden fixtures. Writing PNGs is not needed by the oracle.
#include <zlib.h>

#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "veil/error.hpp"
#include "veil/image.hpp"

namespace veil {

namespace {

uint32_t be32(const uint8_t* p) { return (uint32_t(p[0]) << 24) | (p[1] << 16) | (p[2] << 8) | p[3]; }

int paeth(int a, int b, int c) {
  const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

}  // namespace

Image8 load_png(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error(ErrorCode::io, "cannot open " + path);
  const std::vector<uint8_t> d((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (d.size() < 8 || d[1] != 'P' || d[2] != 'N' || d[3] != 'G')
    throw Error(ErrorCode::parse, "not a PNG: " + path);
  int w = 0, h = 0, depth = 0, ctype = 0, interlace = 0;
  std::vector<uint8_t> idat;
  for (size_t p = 8; p + 8 <= d.size();) {
    const uint32_t len = be32(&d[p]);
    const std::string type(reinterpret_cast<const char*>(&d[p + 4]), 4);
    const uint8_t* body = &d[p + 8];
    if (type == "IHDR") {
      w = int(be32(body)), h = int(be32(body + 4)), depth = body[8], ctype = body[9], interlace = body[12];
    } else if (type == "IDAT") {
      idat.insert(idat.end(), body, body + len);
    } else if (type == "IEND") {
      break;
    }
    p += 12 + len;
  }
  const int ch = ctype == 0 ? 1 : ctype == 4 ? 2 : ctype == 2 ? 3 : ctype == 6 ? 4 : 0;
  if (depth != 8 || ch == 0 || interlace != 0 || w <= 0 || h <= 0)
    throw Error(ErrorCode::parse, "unsupported PNG format: " + path);
  const size_t stride = size_t(w) * ch;
  std::vector<uint8_t> raw((stride + 1) * h);
  uLongf n = raw.size();
  if (uncompress(raw.data(), &n, idat.data(), idat.size()) != Z_OK || n != raw.size())
    throw Error(ErrorCode::parse, "corrupt PNG data: " + path);
  std::vector<uint8_t> px(stride * h);
  for (int y = 0; y < h; ++y) {
    const uint8_t ft = raw[y * (stride + 1)];
    const uint8_t* src = &raw[y * (stride + 1) + 1];
    uint8_t* row = &px[y * stride];
    const uint8_t* up = y ? &px[(y - 1) * stride] : nullptr;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= size_t(ch) ? row[i - ch] : 0, b = up ? up[i] : 0,
                c = (up && i >= size_t(ch)) ? up[i - ch] : 0;
      int v = src[i];
      if (ft == 1) v += a;
      else if (ft == 2) v += b;
      else if (ft == 3) v += (a + b) / 2;
      else if (ft == 4) v += paeth(a, b, c);
      row[i] = uint8_t(v);
    }
  }
  Image8 img(w, h);
  for (size_t i = 0; i < size_t(w) * h; ++i) {
    const uint8_t* s = &px[i * ch];
    uint8_t* o = &img.rgba[i * 4];
    o[0] = s[0];
    o[1] = ch >= 3 ? s[1] : s[0];
    o[2] = ch >= 3 ? s[2] : s[0];
    o[3] = ch == 4 ? s[3] : ch == 2 ? s[1] : 255;
  }
  return img;
}

void save_png(const Image8&, const std::string& path) {
  throw Error(ErrorCode::io, "oracle/_ref build does not write PNGs: " + path);
}

}  // namespace veil
