// image_io_stub.cpp — TEST INFRASTRUCTURE ONLY. The reference's image_io.cpp needs libpng /
// libjpeg, which this image lacks; dataio.cpp (compiled for its checkpoint PLY and optimizer
// sidecar writers) references these two symbols, so they are stubbed to the reference's own
// "unsupported" error. No image is ever decoded by the oracle.
#include "omnisplat/dataio.hpp"
#include "omnisplat/error.hpp"

namespace omnisplat {

Image load_image(const std::string& path) {
    throw Error(ErrorCode::UnsupportedFormat, "image decoding not built into the oracle: " + path);
}

void save_image(const Image&, const std::string& path) {
    throw Error(ErrorCode::UnsupportedFormat, "image encoding not built into the oracle: " + path);
}

}  // namespace omnisplat
