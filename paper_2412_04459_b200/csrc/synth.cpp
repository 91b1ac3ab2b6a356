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
#include <algorithm>
#include <cmath>
#include <queue>
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


// rebuild_corner_indexing (scene.cpp:8-26): corner pool in first-seen order
// over (voxel, corner), then densities U(-4,2.5) per pool entry and SH as
// tests/test_raster.cpp:29-37, drawn from rng in that order.
void emit_scene(const std::vector<Path>& vox, std::mt19937_64& rng, int sh_degree,
                uint64_t* n_voxels, uint64_t* n_pool, uint64_t** codes, uint8_t** levels,
                uint32_t** corner_index, float** density, float** sh) {
    const size_t N = vox.size();
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
}

// ---- init_unbounded (optim.cpp:96-184) ------------------------------------
// Every expression keeps the reference's operand order (geom.hpp, camera.hpp,
// octree.hpp) and the file is built with -ffp-contract=off, so the
// observed/refined decisions — and therefore the voxel set — are identical.
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

struct Bounds {
    V3 center;
    double size;
};

// Camera::project (camera.hpp:33-37) through world_to_cam = rot^T (p - pos).
bool point_observed(V3 p, const std::vector<svr_camera>& cams) {  // optim.cpp:43-50
    for (const svr_camera& c : cams) {
        V3 d = sub(p, V3{c.pos[0], c.pos[1], c.pos[2]});
        const double* m = c.rot;
        V3 q{m[0] * d.x + m[3] * d.y + m[6] * d.z, m[1] * d.x + m[4] * d.y + m[7] * d.z,
             m[2] * d.x + m[5] * d.y + m[8] * d.z};
        double u = c.fx * q.x / q.z + c.cx, v = c.fy * q.y / q.z + c.cy;
        if (q.z > 0 && u >= 0 && u <= c.width && v >= 0 && v <= c.height) return true;
    }
    return false;
}

// voxel_observed (optim.cpp:52-56) over corner_keys/corner_position (octree.hpp:130-146).
bool voxel_observed(const Bounds& b, const Path& p, const std::vector<svr_camera>& cams) {
    uint32_t i, j, k;
    to_index(p, i, j, k);
    uint32_t step = uint32_t(1) << (kMaxLevel - p.level);
    double cell = b.size / double(uint64_t(1) << kMaxLevel);
    V3 lo = sub(b.center, V3{0.5 * b.size, 0.5 * b.size, 0.5 * b.size});
    for (uint32_t c = 0; c < 8; ++c) {
        uint32_t x = (i + ((c >> 2) & 1)) * step, y = (j + ((c >> 1) & 1)) * step,
                 z = (k + (c & 1)) * step;
        if (point_observed(add(lo, V3{cell * x, cell * y, cell * z}), cams)) return true;
    }
    return false;
}

// max_sampling_rate (optim.cpp:69-78) at voxel_geometry (octree.hpp:85-90).
double max_sampling_rate(const Bounds& b, const Path& p, const std::vector<svr_camera>& cams) {
    uint32_t i, j, k;
    to_index(p, i, j, k);
    double size = std::ldexp(b.size, -p.level);
    V3 lo = sub(b.center, V3{0.5 * b.size, 0.5 * b.size, 0.5 * b.size});
    V3 center = add(lo, V3{size * (i + 0.5), size * (j + 0.5), size * (k + 0.5)});
    double best = 0.0;
    for (const svr_camera& c : cams) {
        double z = dot3(sub(center, V3{c.pos[0], c.pos[1], c.pos[2]}),
                        V3{c.rot[2], c.rot[5], c.rot[8]});
        if (z <= 0) continue;
        best = std::max(best, size * c.fx / z);
    }
    return best;
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
        emit_scene(vox, rng, sh_degree, n_voxels, n_pool, codes, levels, corner_index, density,
                   sh);
        return SVR_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SVR_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVR_ERR_RUNTIME;
    }
}

int svr_synth_unbounded_scene(const svr_camera* cams, int n_cams, int init_level,
                              int shell_levels, double bg_ratio, uint64_t seed, int sh_degree,
                              uint64_t* n_voxels, uint64_t* n_pool, uint64_t** codes,
                              uint8_t** levels, uint32_t** corner_index, float** density,
                              float** sh, double* bounds_center, double* bounds_size) {
    try {
        if (!cams || n_cams < 2)
            throw std::invalid_argument("init_unbounded needs at least two cameras");
        if (init_level < 1 || init_level > kMaxLevel)
            throw std::invalid_argument("init_level out of [1,16]");
        if (shell_levels < 1 || shell_levels > kMaxLevel - 2)
            throw std::invalid_argument("shell_levels out of range");
        if (bg_ratio <= 0) throw std::invalid_argument("bg_ratio must be positive");
        if (sh_degree < 0 || sh_degree > 3)
            throw std::invalid_argument("sh_degree out of [0,3]");
        std::vector<svr_camera> cv(cams, cams + n_cams);
        V3 center{0, 0, 0};
        for (const svr_camera& c : cv) center = add(center, V3{c.pos[0], c.pos[1], c.pos[2]});
        center = {center.x / double(n_cams), center.y / double(n_cams), center.z / double(n_cams)};
        std::vector<double> dist;
        for (const svr_camera& c : cv) {
            V3 d = sub(V3{c.pos[0], c.pos[1], c.pos[2]}, center);
            dist.push_back(std::sqrt(dot3(d, d)));
        }
        std::nth_element(dist.begin(), dist.begin() + dist.size() / 2, dist.end());
        double radius = dist[dist.size() / 2];
        if (radius <= 0) throw std::invalid_argument("degenerate camera set: coincident positions");
        Bounds b{center, std::ldexp(2.0 * radius, shell_levels)};

        std::vector<Path> vox;
        int lv_main = shell_levels + init_level;
        if (lv_main > kMaxLevel)
            throw std::invalid_argument("shell_levels + init_level exceeds 16");
        uint32_t half = uint32_t(1) << (lv_main - 1), m = uint32_t(1) << (init_level - 1);
        size_t fg = 0;
        for (uint32_t i = half - m; i < half + m; ++i)
            for (uint32_t j = half - m; j < half + m; ++j)
                for (uint32_t k = half - m; k < half + m; ++k) {
                    Path p{to_code(i, j, k, lv_main), lv_main};
                    if (voxel_observed(b, p, cv)) {
                        vox.push_back(p);
                        ++fg;
                    }
                }
        if (fg == 0) throw std::invalid_argument("no observed voxels in the main region");

        struct ShellVox {
            double rate;
            uint64_t tiebreak;
            Path path;
            bool operator<(const ShellVox& o) const {
                return rate != o.rate ? rate < o.rate : tiebreak > o.tiebreak;
            }
        };
        std::priority_queue<ShellVox> shell;
        auto push_shell = [&](const Path& p) {
            shell.push({max_sampling_rate(b, p, cv), p.code | (uint64_t(p.level) << 48), p});
        };
        for (int s = 1; s <= shell_levels; ++s) {
            int lv = shell_levels - s + 2;
            uint32_t h = uint32_t(1) << (lv - 1);
            for (uint32_t i = h - 2; i < h + 2; ++i)
                for (uint32_t j = h - 2; j < h + 2; ++j)
                    for (uint32_t k = h - 2; k < h + 2; ++k) {
                        bool inner = i >= h - 1 && i < h + 1 && j >= h - 1 && j < h + 1 &&
                                     k >= h - 1 && k < h + 1;
                        if (inner) continue;
                        Path p{to_code(i, j, k, lv), lv};
                        if (voxel_observed(b, p, cv)) push_shell(p);
                    }
        }
        std::vector<Path> bg_done;
        size_t bg = shell.size();
        while (bg < size_t(bg_ratio * double(fg)) && !shell.empty()) {
            ShellVox top = shell.top();
            shell.pop();
            if (top.path.level >= kMaxLevel) {
                bg_done.push_back(top.path);
                continue;
            }
            --bg;
            int shift = 3 * (kMaxLevel - top.path.level - 1);
            for (uint64_t c = 0; c < 8; ++c) {
                Path ch{top.path.code | (c << shift), top.path.level + 1};
                if (voxel_observed(b, ch, cv)) {
                    push_shell(ch);
                    ++bg;
                }
            }
        }
        while (!shell.empty()) {
            bg_done.push_back(shell.top().path);
            shell.pop();
        }
        for (const Path& p : bg_done) vox.push_back(p);
        std::mt19937_64 rng(seed);
        emit_scene(vox, rng, sh_degree, n_voxels, n_pool, codes, levels, corner_index, density,
                   sh);
        bounds_center[0] = b.center.x;
        bounds_center[1] = b.center.y;
        bounds_center[2] = b.center.z;
        *bounds_size = b.size;
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
