// synth.cpp — deterministic synthetic fixtures for tests and benchmarks.
//
// Not part of the render path. Produces the benchmark scenes of SURVEY §8(d)
// on hosts where the reference is absent (the GPU box), with the same RNG
// stream as the oracle's generator so both sides see identical scenes:
//   * generator G: level-3 dense grid, random leaf subdivision (pattern of
//     tests/test_raster.cpp:15-28), corner-pool dedup in first-seen order
//     (rebuild_corner_indexing, scene.cpp:8-26), densities U(-4,2.5), SH from
//     tests/test_raster.cpp:29-37;
//   * the unbounded rig scene of configs 4/5 (the voxel set init_unbounded,
//     optim.cpp:96-184, builds), parameters drawn as for G;
//   * ring_cameras (synth.cpp:89-118).
// Compiled with -ffp-contract=off so camera poses match the reference bit
// for bit.
#include <algorithm>
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

// ---- unbounded-scene fixture (the scene init_unbounded, optim.cpp:96-184,
// builds for a camera rig) ---------------------------------------------------
// A voxel is handled as one packed key, `code | level << 48`; that key is
// also the ordering tie-break of the refinement frontier. The frontier order
// (highest max-sampling-rate first, then smallest key) is a strict total
// order, so the order in which candidates are *inserted* is irrelevant: only
// the main block's enumeration order and the frontier's pop order reach the
// output. The float expressions (camera projection, corner positions, voxel
// centres, rates) are evaluated with the reference geometry's operand order
// and this file is built with -ffp-contract=off, so every observed/refined
// decision — and therefore the voxel list — is bit-identical
// (tests/test_abi_cpu.py::test_unbounded_generator_matches_reference).
constexpr uint64_t kKeyLevelShift = 48;

inline uint64_t pack_key(uint64_t code, int level) {
    return code | (uint64_t(level) << kKeyLevelShift);
}
inline int key_level(uint64_t key) { return int(key >> kKeyLevelShift); }
inline uint64_t key_code(uint64_t key) { return key & ((uint64_t(1) << kKeyLevelShift) - 1); }

class RigView {
  public:
    RigView(const svr_camera* cams, int n, const double centre[3], double extent)
        : cams_(cams, cams + n), extent_(extent) {
        for (int a = 0; a < 3; ++a) lo_[a] = centre[a] - 0.5 * extent;
        cell_ = extent / double(uint64_t(1) << kMaxLevel);
    }

    // any camera sees the point inside its image rectangle, in front of it
    // (Camera::project, camera.hpp:29-35)
    bool sees(const double p[3]) const {
        for (const svr_camera& c : cams_) {
            const double d0 = p[0] - c.pos[0], d1 = p[1] - c.pos[1], d2 = p[2] - c.pos[2];
            const double* r = c.rot;
            const double cx = r[0] * d0 + r[3] * d1 + r[6] * d2;
            const double cy = r[1] * d0 + r[4] * d1 + r[7] * d2;
            const double cz = r[2] * d0 + r[5] * d1 + r[8] * d2;
            const double u = c.fx * cx / cz + c.cx;
            const double v = c.fy * cy / cz + c.cy;
            if (cz > 0 && u >= 0 && u <= c.width && v >= 0 && v <= c.height) return true;
        }
        return false;
    }

    // some corner of the voxel is seen (corner grid of octree.hpp:130-146)
    bool sees_voxel(uint64_t key) const {
        uint32_t ijk[3];
        Path p{key_code(key), key_level(key)};
        to_index(p, ijk[0], ijk[1], ijk[2]);
        const uint32_t step = uint32_t(1) << (kMaxLevel - p.level);
        for (uint32_t corner = 0; corner < 8; ++corner) {
            double q[3];
            for (int a = 0; a < 3; ++a) {
                const uint32_t g = (ijk[a] + ((corner >> (2 - a)) & 1)) * step;
                q[a] = lo_[a] + cell_ * g;
            }
            if (sees(q)) return true;
        }
        return false;
    }

    // largest pixels-per-voxel-size over the cameras in front of the centre
    // (max_sampling_rate, optim.cpp:68-77, at voxel_geometry, octree.hpp:85-90)
    double rate(uint64_t key) const {
        uint32_t ijk[3];
        Path p{key_code(key), key_level(key)};
        to_index(p, ijk[0], ijk[1], ijk[2]);
        const double size = std::ldexp(extent_, -p.level);
        double ctr[3];
        for (int a = 0; a < 3; ++a) ctr[a] = lo_[a] + size * (ijk[a] + 0.5);
        double best = 0.0;
        for (const svr_camera& c : cams_) {
            const double z = (ctr[0] - c.pos[0]) * c.rot[2] + (ctr[1] - c.pos[1]) * c.rot[5] +
                             (ctr[2] - c.pos[2]) * c.rot[8];
            if (z > 0) best = std::max(best, size * c.fx / z);
        }
        return best;
    }

  private:
    std::vector<svr_camera> cams_;
    double lo_[3];
    double cell_;
    double extent_;
};

struct Frontier {
    struct Item {
        double rate;
        uint64_t key;
    };
    // max-heap on rate; among equal rates the smaller key comes out first
    static bool below(const Item& a, const Item& b) {
        if (a.rate != b.rate) return a.rate < b.rate;
        return a.key > b.key;
    }
    std::vector<Item> heap;
    void push(double rate, uint64_t key) {
        heap.push_back({rate, key});
        std::push_heap(heap.begin(), heap.end(), below);
    }
    uint64_t pop() {
        std::pop_heap(heap.begin(), heap.end(), below);
        uint64_t k = heap.back().key;
        heap.pop_back();
        return k;
    }
};

// Voxel list of the unbounded rig scene: the observed cells of the central
// 2^init_level block at level shell_levels + init_level (i, j, k order),
// then the background shells refined coarse-to-fine by sampling rate until
// there are bg_ratio times as many background voxels as foreground ones.
std::vector<Path> unbounded_voxels(const RigView& rig, int init_level, int shell_levels,
                                   double bg_ratio) {
    const int fine = shell_levels + init_level;
    std::vector<Path> out;
    const uint64_t side = uint64_t(1) << init_level;
    const uint32_t first = (uint32_t(1) << (fine - 1)) - (uint32_t(1) << (init_level - 1));
    for (uint64_t n = 0; n < side * side * side; ++n) {
        const uint32_t i = first + uint32_t(n / (side * side));
        const uint32_t j = first + uint32_t((n / side) % side);
        const uint32_t k = first + uint32_t(n % side);
        const uint64_t code = to_code(i, j, k, fine);
        if (rig.sees_voxel(pack_key(code, fine))) out.push_back({code, fine});
    }
    const size_t n_fg = out.size();
    if (n_fg == 0) throw std::invalid_argument("unbounded scene: no camera observes the main block");

    // shell at level lv: the 4x4x4 cells around the scene centre minus the
    // inner 2x2x2 (which the next finer level covers)
    Frontier front;
    for (int lv = 2; lv <= shell_levels + 1; ++lv) {
        const uint32_t c0 = (uint32_t(1) << (lv - 1)) - 2;
        for (uint32_t n = 0; n < 64; ++n) {
            const uint32_t di = n >> 4, dj = (n >> 2) & 3, dk = n & 3;
            if ((di == 1 || di == 2) && (dj == 1 || dj == 2) && (dk == 1 || dk == 2)) continue;
            const uint64_t key = pack_key(to_code(c0 + di, c0 + dj, c0 + dk, lv), lv);
            if (rig.sees_voxel(key)) front.push(rig.rate(key), key);
        }
    }
    const size_t bg_target = size_t(bg_ratio * double(n_fg));
    std::vector<uint64_t> settled;  // background leaves that can no longer split
    while (!front.heap.empty() && front.heap.size() + settled.size() < bg_target) {
        const uint64_t key = front.pop();
        const int lv = key_level(key);
        if (lv >= kMaxLevel) {
            settled.push_back(key);
            continue;
        }
        const int shift = 3 * (kMaxLevel - lv - 1);
        for (uint64_t child = 0; child < 8; ++child) {
            const uint64_t ck = pack_key(key_code(key) | (child << shift), lv + 1);
            if (rig.sees_voxel(ck)) front.push(rig.rate(ck), ck);
        }
    }
    while (!front.heap.empty()) settled.push_back(front.pop());
    for (uint64_t key : settled) out.push_back({key_code(key), key_level(key)});
    return out;
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
            throw std::invalid_argument("unbounded scene: the rig needs two or more cameras");
        if (init_level < 1 || shell_levels < 1 || shell_levels + init_level > kMaxLevel)
            throw std::invalid_argument(
                "unbounded scene: need init_level, shell_levels >= 1 and their sum <= 16");
        if (!(bg_ratio > 0)) throw std::invalid_argument("unbounded scene: bg_ratio must be > 0");
        if (sh_degree < 0 || sh_degree > 3)
            throw std::invalid_argument("unbounded scene: sh_degree must be in [0, 3]");
        // rig centre = mean camera position; main block edge = twice the
        // median camera distance from it; the scene cube is 2^shell_levels
        // main blocks wide
        double centre[3] = {0, 0, 0};
        for (int c = 0; c < n_cams; ++c)
            for (int a = 0; a < 3; ++a) centre[a] += cams[c].pos[a];
        for (int a = 0; a < 3; ++a) centre[a] = centre[a] / double(n_cams);
        std::vector<double> reach(n_cams);
        for (int c = 0; c < n_cams; ++c) {
            const double d0 = cams[c].pos[0] - centre[0], d1 = cams[c].pos[1] - centre[1],
                         d2 = cams[c].pos[2] - centre[2];
            reach[c] = std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        }
        std::nth_element(reach.begin(), reach.begin() + n_cams / 2, reach.end());
        const double radius = reach[n_cams / 2];
        if (!(radius > 0))
            throw std::invalid_argument("unbounded scene: all cameras at one position");
        const double extent = std::ldexp(2.0 * radius, shell_levels);
        RigView rig(cams, n_cams, centre, extent);
        std::vector<Path> vox = unbounded_voxels(rig, init_level, shell_levels, bg_ratio);
        std::mt19937_64 rng(seed);
        emit_scene(vox, rng, sh_degree, n_voxels, n_pool, codes, levels, corner_index, density,
                   sh);
        for (int a = 0; a < 3; ++a) bounds_center[a] = centre[a];
        *bounds_size = extent;
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
