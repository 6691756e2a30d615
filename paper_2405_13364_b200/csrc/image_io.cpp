// PNG read/write on zlib (libpng is not in this image). Host I/O, off the
// frame path; replaces proj/src/image.cpp:37-108. Reading normalises every
// non-interlaced PNG to 8-bit RGBA with the reference's transform set
// (expand palette/gray/low bit depths, strip 16-bit to the high byte, gray to
// RGB, opaque alpha filler); writing emits 8-bit RGBA.
#include <zlib.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>

#include "veil_internal.hpp"

namespace veil {

namespace {

uint32_t be32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | p[3];
}

void put32(std::vector<uint8_t>& v, uint32_t x) {
  v.push_back(uint8_t(x >> 24));
  v.push_back(uint8_t(x >> 16));
  v.push_back(uint8_t(x >> 8));
  v.push_back(uint8_t(x));
}

void chunk(std::vector<uint8_t>& out, const char* type, const std::vector<uint8_t>& data) {
  put32(out, uint32_t(data.size()));
  size_t start = out.size();
  out.insert(out.end(), type, type + 4);
  out.insert(out.end(), data.begin(), data.end());
  uint32_t crc = uint32_t(crc32(0, out.data() + start, uInt(out.size() - start)));
  put32(out, crc);
}

int paeth(int a, int b, int c) {
  int p = a + b - c;
  int pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  if (pa <= pb && pa <= pc) return a;
  return pb <= pc ? b : c;
}

}  // namespace

Image8 read_png(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(VEIL_ERR_IO, "cannot open " + path);
  std::vector<uint8_t> f((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
  if (f.size() < 8 || std::memcmp(f.data(), sig, 8) != 0)
    throw Error(VEIL_ERR_IO, "not a PNG file: " + path);
  uint32_t w = 0, h = 0;
  int depth = 0, ctype = 0, interlace = 0;
  std::vector<uint8_t> idat, plte, trns;
  size_t pos = 8;
  while (pos + 12 <= f.size()) {
    uint32_t len = be32(&f[pos]);
    if (pos + 12 + len > f.size()) break;
    const char* type = reinterpret_cast<const char*>(&f[pos + 4]);
    const uint8_t* d = &f[pos + 8];
    if (!std::memcmp(type, "IHDR", 4) && len >= 13) {
      w = be32(d);
      h = be32(d + 4);
      depth = d[8];
      ctype = d[9];
      interlace = d[12];
    } else if (!std::memcmp(type, "PLTE", 4)) {
      plte.assign(d, d + len);
    } else if (!std::memcmp(type, "tRNS", 4)) {
      trns.assign(d, d + len);
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), d, d + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      break;
    }
    pos += 12 + len;
  }
  if (w == 0 || h == 0) throw Error(VEIL_ERR_IO, "failed to decode PNG " + path);
  if (interlace) throw Error(VEIL_ERR_IO, "interlaced PNG not supported: " + path);
  int channels = ctype == 0 ? 1 : ctype == 2 ? 3 : ctype == 3 ? 1 : ctype == 4 ? 2 : ctype == 6 ? 4 : 0;
  if (!channels) throw Error(VEIL_ERR_IO, "unsupported PNG color type: " + path);
  size_t bpp_bits = size_t(channels) * depth;
  size_t stride = (size_t(w) * bpp_bits + 7) / 8;
  size_t bpp = std::max<size_t>(1, bpp_bits / 8);
  std::vector<uint8_t> raw(size_t(h) * (stride + 1));
  uLongf raw_len = uLongf(raw.size());
  if (uncompress(raw.data(), &raw_len, idat.data(), uLong(idat.size())) != Z_OK ||
      raw_len != raw.size())
    throw Error(VEIL_ERR_IO, "failed to decode PNG " + path);
  std::vector<uint8_t> px(size_t(h) * stride), prev(stride, 0);
  for (uint32_t y = 0; y < h; ++y) {
    uint8_t ft = raw[size_t(y) * (stride + 1)];
    const uint8_t* src = &raw[size_t(y) * (stride + 1) + 1];
    uint8_t* dst = &px[size_t(y) * stride];
    for (size_t x = 0; x < stride; ++x) {
      int a = x >= bpp ? dst[x - bpp] : 0, b = prev[x], c = x >= bpp ? prev[x - bpp] : 0;
      int v = src[x];
      switch (ft) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) / 2; break;
        case 4: v += paeth(a, b, c); break;
        default: throw Error(VEIL_ERR_IO, "failed to decode PNG " + path);
      }
      dst[x] = uint8_t(v);
    }
    std::memcpy(prev.data(), dst, stride);
  }
  auto sample = [&](const uint8_t* row, uint32_t x, int ch) -> uint32_t {
    size_t idx = size_t(x) * channels + ch;
    if (depth == 16) return row[idx * 2];  // strip_16: high byte
    if (depth == 8) return row[idx];
    size_t bit = idx * depth;
    uint32_t v = (row[bit / 8] >> (8 - depth - bit % 8)) & ((1u << depth) - 1);
    return v;
  };
  Image8 img;
  img.width = int(w);
  img.height = int(h);
  img.rgba.resize(size_t(w) * h * 4);
  for (uint32_t y = 0; y < h; ++y) {
    const uint8_t* row = &px[size_t(y) * stride];
    for (uint32_t x = 0; x < w; ++x) {
      uint8_t* o = &img.rgba[(size_t(y) * w + x) * 4];
      if (ctype == 3) {
        uint32_t i = sample(row, x, 0);
        o[0] = i * 3 + 2 < plte.size() ? plte[i * 3] : 0;
        o[1] = i * 3 + 2 < plte.size() ? plte[i * 3 + 1] : 0;
        o[2] = i * 3 + 2 < plte.size() ? plte[i * 3 + 2] : 0;
        o[3] = i < trns.size() ? trns[i] : 255;
      } else if (ctype == 0 || ctype == 4) {
        uint32_t g = sample(row, x, 0);
        if (depth < 8) g = g * 255 / ((1u << depth) - 1);
        o[0] = o[1] = o[2] = uint8_t(g);
        o[3] = ctype == 4 ? uint8_t(sample(row, x, 1)) : 255;
      } else {
        o[0] = uint8_t(sample(row, x, 0));
        o[1] = uint8_t(sample(row, x, 1));
        o[2] = uint8_t(sample(row, x, 2));
        o[3] = ctype == 6 ? uint8_t(sample(row, x, 3)) : 255;
      }
    }
  }
  return img;
}

void write_png(const Image8& img, const std::string& path) {
  std::vector<uint8_t> raw;
  raw.reserve(size_t(img.height) * (size_t(img.width) * 4 + 1));
  for (int y = 0; y < img.height; ++y) {
    raw.push_back(0);
    const uint8_t* r = img.rgba.data() + size_t(y) * img.width * 4;
    raw.insert(raw.end(), r, r + size_t(img.width) * 4);
  }
  uLongf zlen = compressBound(uLong(raw.size()));
  std::vector<uint8_t> z(zlen);
  if (compress2(z.data(), &zlen, raw.data(), uLong(raw.size()), 6) != Z_OK)
    throw Error(VEIL_ERR_IO, "failed to encode PNG " + path);
  z.resize(zlen);
  std::vector<uint8_t> out = {137, 80, 78, 71, 13, 10, 26, 10};
  std::vector<uint8_t> ihdr;
  put32(ihdr, uint32_t(img.width));
  put32(ihdr, uint32_t(img.height));
  ihdr.insert(ihdr.end(), {8, 6, 0, 0, 0});
  chunk(out, "IHDR", ihdr);
  chunk(out, "IDAT", z);
  chunk(out, "IEND", {});
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw Error(VEIL_ERR_IO, "cannot write " + path);
  size_t n = std::fwrite(out.data(), 1, out.size(), fp);
  std::fclose(fp);
  if (n != out.size()) throw Error(VEIL_ERR_IO, "cannot write " + path);
}

}  // namespace veil
