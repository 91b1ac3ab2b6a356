// svrx.h — SVRX checkpoint codec (io.cpp:229-359), host side.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace svrb {

// std::runtime_error of load_checkpoint / save_checkpoint
struct SvrxError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// std::invalid_argument of to_voxel_index (octree.hpp:47-49, 71-72)
struct SvrxInvalid : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct SvrxScene {
    std::vector<uint64_t> codes;
    std::vector<uint8_t> levels;
    std::vector<uint32_t> corner_index;  // [n][8]
    std::vector<float> density;
    std::vector<float> sh;
    int sh_degree = 3;
    double bounds_center[3] = {0, 0, 0};
    double bounds_size = 1.0;
};

std::string svrx_header(uint64_t n, uint64_t p, int sh_degree, const double* bc, double bs);
std::vector<uint8_t> svrx_encode(const SvrxScene& s);
void svrx_write(const std::string& path, const std::vector<uint8_t>& bytes);
SvrxScene svrx_read(const std::string& path);                   // checks, in io.cpp order
void svrx_validate(const SvrxScene& s, const std::string& path);  // corner-key structure

}  // namespace svrb
