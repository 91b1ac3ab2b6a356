// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
// The reference's io.cpp needs libpng (png.h is absent in this image), but
// synth.cpp links against four of its functions. Only ring_cameras /
// synth_scene are used from synth.cpp, so these stubs are never executed.
#include <stdexcept>

#include "svr/io.hpp"

namespace svr {
Image load_png(const std::string&) { throw std::runtime_error("io stub: load_png unavailable"); }
void save_png(const Image&, const std::string&) {
    throw std::runtime_error("io stub: save_png unavailable");
}
void save_depth(const Image&, const std::string&) {
    throw std::runtime_error("io stub: save_depth unavailable");
}
void save_cameras(const std::vector<CameraFrame>&, const std::string&) {
    throw std::runtime_error("io stub: save_cameras unavailable");
}
}  // namespace svr
