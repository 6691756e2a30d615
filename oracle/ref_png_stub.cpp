// Test infrastructure only (never shipped, never on the product path).
//
// The reference's image.cpp needs libpng, whose headers are absent from this
// image. The oracle build of the reference links this
// stub instead: PNG I/O is off the frame path,
// so the render results of the reference are unaffected.
#include <string>

#include "veil/error.hpp"
#include "veil/image.hpp"

namespace veil {

Image8 load_png(const std::string& path) {
  throw Error(ErrorCode::io, "oracle/_ref build has no libpng: cannot read " + path);
}

void save_png(const Image8&, const std::string& path) {
  throw Error(ErrorCode::io, "oracle/_ref build has no libpng: cannot write " + path);
}

}  // namespace veil
