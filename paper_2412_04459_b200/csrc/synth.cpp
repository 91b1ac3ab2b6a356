// synth.cpp — deterministic synthetic fixtures for tests and benchmarks.
//
// Not part of the render path. Produces the benchmark scenes of SURVEY §8(d)
// on hosts where the reference is absent (the GPU box), with the same RNG
// stream as the oracle's generator so both sides see identical scenes:
//   * generator G: level-3 dense grid, random leaf subdivision (pattern of
//     tests/test_raster.cpp:15-28), corner-pool dedup in first-seen order
//     (rebuild_corner_indexing, scene.cpp:8-26), densities U(-4,2.5), SH from
//     tests/test_raster.cpp:29-37;
//   * ring_cameras (synth.cpp:89-118).
// Compiled with -ffp-contract=off so camera poses match the reference bit
// for bit.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "svr_b200.h"

namespace {

thread_local std::string g_err;

constexpr int kMaxLevel = 16;

struct Path {
    uint64_t code;
    int level;
};

uint64_t to_code(uint32_t i, uint32_t j, uint32_t k, int level) {
    uint64_t code = 0;
    for (int n = 0; n < level; ++n) {
        uint64_t bits = 4 * (i & 1) + 2 * (j & 1) + (k & 1);
        code |= bits << (3 * n);
        i >>= 1;
        j >>= 1;
        k >>= 1;
    }
    return code << (3 * (kMaxLevel - level));
}

void to_index(const Path& p, uint32_t& i, uint32_t& j, uint32_t& k) {
    uint64_t c = p.code >> (3 * (kMaxLevel - p.level));
    i = j = k = 0;
    for (int n = 0; n < p.level; ++n) {
        i |= uint32_t((c >> 2) & 1) << n;
        j |= uint32_t((c >> 1) & 1) << n;
        k |= uint32_t(c & 1) << n;
        c >>= 3;
    }
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(T)));
    if (!p) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

struct V3 {
    double x, y, z;
};
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
V3 normalized(V3 v) {
    double n = std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z);
    return n > 0.0 ? V3{v.x / n, v.y / n, v.z / n} : V3{0, 0, 0};
}

}  // namespace

extern "C" {

int svr_synth_random_scene(uint64_t seed, uint64_t target, int max_level, int sh_degree,
                           uint64_t* n_voxels, uint64_t* n_pool, uint64_t** codes,
                           uint8_t** levels, uint32_t** corner_index, float** density,
                           float** sh) {
    try {
        if (max_level < 3 || max_level > kMaxLevel || sh_degree < 0 || sh_degree > 3)
            throw std::invalid_argument("synth: max_level in [3,16], sh_degree in [0,3]");
        if (max_level < 20 && double(target) > std::ldexp(1.0, 3 * max_level))
            throw std::invalid_argument("synth: target exceeds the voxel capacity of max_level");
        std::mt19937_64 rng(seed);
        std::vector<Path> vox;
        vox.reserve(target + 8);
        for (uint32_t i = 0; i < 8; ++i)
            for (uint32_t j = 0; j < 8; ++j)
                for (uint32_t k = 0; k < 8; ++k) vox.push_back({to_code(i, j, k, 3), 3});
        while (vox.size() + 7 <= target) {
            size_t pick = rng() % vox.size();
            if (vox[pick].level >= max_level) continue;
            Path p = vox[pick];
            int shift = 3 * (kMaxLevel - p.level - 1);
            vox[pick] = {p.code, p.level + 1};
            for (uint64_t c = 1; c < 8; ++c) vox.push_back({p.code | (c << shift), p.level + 1});
        }
        const size_t N = vox.size();
        // corner pool, first-seen order over (voxel, corner)
        std::vector<uint32_t> ci(N * 8);
        std::unordered_map<uint64_t, uint32_t> pool_of;
        pool_of.reserve(N * 2);
        uint32_t P = 0;
        for (size_t v = 0; v < N; ++v) {
            uint32_t i, j, k;
            to_index(vox[v], i, j, k);
            uint32_t step = uint32_t(1) << (kMaxLevel - vox[v].level);
            for (uint32_t c = 0; c < 8; ++c) {
                uint64_t x = uint64_t(i + ((c >> 2) & 1)) * step;
                uint64_t y = uint64_t(j + ((c >> 1) & 1)) * step;
                uint64_t z = uint64_t(k + (c & 1)) * step;
                uint64_t key = (x << 34) | (y << 17) | z;
                auto it = pool_of.try_emplace(key, P);
                if (it.second) ++P;
                ci[8 * v + c] = it.first->second;
            }
        }
        std::uniform_real_distribution<double> ud(-4.0, 2.5), uc(0.05, 0.8);
        std::vector<float> dens(P);
        for (auto& d : dens) d = float(ud(rng));
        const int stride = 3 * (sh_degree + 1) * (sh_degree + 1);
        std::vector<float> coeffs(N * stride, 0.0f);
        for (size_t v = 0; v < N; ++v) {
            float* s = coeffs.data() + v * stride;
            for (int ch = 0; ch < 3; ++ch) s[ch] = float(uc(rng) / 0.28209479177387814);
            for (int m = 3; m < stride; ++m) s[m] = float(0.1 * (uc(rng) - 0.4));
        }
        std::vector<uint64_t> cv(N);
        std::vector<uint8_t> lv(N);
        for (size_t v = 0; v < N; ++v) {
            cv[v] = vox[v].code;
            lv[v] = uint8_t(vox[v].level);
        }
        *n_voxels = N;
        *n_pool = P;
        *codes = dup(cv);
        *levels = dup(lv);
        *corner_index = dup(ci);
        *density = dup(dens);
        *sh = dup(coeffs);
        return SVR_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SVR_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVR_ERR_RUNTIME;
    }
}

int svr_ring_camera(int n_views, int index, int width, int height, double distance,
                    double fov_x_deg, svr_camera* out) {
    if (n_views < 1 || index < 0 || index >= n_views || !out) return SVR_ERR_INVALID_ARGUMENT;
    const int i = index;
    double theta = 2.0 * M_PI * i / n_views + 0.1;
    double elev = (i % 2 == 0 ? 0.35 : -0.3) + 0.05 * (i % 3);
    V3 pos{std::cos(elev) * std::cos(theta), std::sin(elev), std::cos(elev) * std::sin(theta)};
    pos = {pos.x * distance, pos.y * distance, pos.z * distance};
    V3 fwd = normalized(V3{-pos.x, -pos.y, -pos.z});
    V3 right = normalized(cross(fwd, V3{0, 1, 0}));
    V3 down = cross(fwd, right);
    out->width = width;
    out->height = height;
    out->fx = 0.5 * width / std::tan(0.5 * fov_x_deg * M_PI / 180.0);
    out->fy = out->fx;
    out->cx = 0.5 * width;
    out->cy = 0.5 * height;
    const double cols[3][3] = {{right.x, right.y, right.z},
                               {down.x, down.y, down.z},
                               {fwd.x, fwd.y, fwd.z}};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out->rot[3 * r + c] = cols[c][r];
    out->pos[0] = pos.x;
    out->pos[1] = pos.y;
    out->pos[2] = pos.z;
    return SVR_OK;
}

}  // extern "C"
