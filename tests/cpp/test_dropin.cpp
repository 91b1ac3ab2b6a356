// C++ test of the drop-in (paper_2412_04459_b200/cpp/raster_dropin.cpp): the
// reference's own raster.hpp API, linked against the GPU implementation
// instead of raster.cpp, exercised in the pattern of proj/tests/test_raster.cpp.
// Expected values come from the C oracle (oracle/svr_oracle.c, pinned to the
// unmodified reference by tests/test_oracle_cpu.py). Prints one line per
// failed check and "ALL PASSED" at the end; exit code = number of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "svr/raster.hpp"
#include "svr_oracle.h"

using namespace svr;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        bool ok = false;                                                       \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const T&) {                                                   \
            ok = true;                                                         \
        } catch (...) {                                                        \
        }                                                                      \
        CHECK(ok && #T);                                                       \
    } while (0)

namespace {

SparseScene random_scene(std::mt19937_64& rng, int subdivisions, int sh_degree = 2) {
    SparseScene s;  // test_raster.cpp:15-39
    s.bounds = {{0, 0, 0}, 1.0};
    for (uint32_t i = 0; i < 8; ++i)
        for (uint32_t j = 0; j < 8; ++j)
            for (uint32_t k = 0; k < 8; ++k) s.voxels.push_back(to_octpath({i, j, k, 3}));
    for (int n = 0; n < subdivisions; ++n) {
        size_t pick = rng() % s.voxels.size();
        if (s.voxels[pick].level >= 8) continue;
        auto kids = child_paths(s.voxels[pick]);
        s.voxels[pick] = kids[0];
        for (int c = 1; c < 8; ++c) s.voxels.push_back(kids[c]);
    }
    rebuild_corner_indexing(s, {});
    std::uniform_real_distribution<double> ud(-4.0, 2.5), uc(0.05, 0.8);
    for (auto& d : s.density) d = float(ud(rng));
    s.sh_degree = sh_degree;
    s.sh.assign(s.voxel_count() * s.sh_stride(), 0.0f);
    for (size_t vi = 0; vi < s.voxel_count(); ++vi) {
        float* sh = s.sh_of(vi);
        for (int ch = 0; ch < 3; ++ch) sh[ch] = float(sh_dc_for_intensity(uc(rng)));
        for (int m = 3; m < s.sh_stride(); ++m) sh[m] = float(0.1 * (uc(rng) - 0.4));
    }
    return s;
}

Camera look_at_origin(int w, int h, double dist, double theta, double elev = 0.25) {
    Camera cam;  // test_raster.cpp:41-60
    cam.width = w;
    cam.height = h;
    cam.fx = cam.fy = 0.9 * w;
    cam.cx = 0.5 * w;
    cam.cy = 0.5 * h;
    Vec3 pos = dist * Vec3{std::cos(elev) * std::cos(theta), std::sin(elev),
                           std::cos(elev) * std::sin(theta)};
    Vec3 fwd = normalized(-pos);
    Vec3 right = normalized(cross(fwd, Vec3{0, 1, 0}));
    Vec3 down = cross(fwd, right);
    for (int r = 0; r < 3; ++r) {
        cam.rot(r, 0) = right[r];
        cam.rot(r, 1) = down[r];
        cam.rot(r, 2) = fwd[r];
    }
    cam.pos = pos;
    return cam;
}

struct Desc {
    std::vector<uint64_t> codes;
    std::vector<uint8_t> levels;
    svr_scene_desc d{};
    explicit Desc(const SparseScene& s) {
        for (auto& p : s.voxels) {
            codes.push_back(p.code);
            levels.push_back(uint8_t(p.level));
        }
        d.n_voxels = s.voxel_count();
        d.n_pool = s.pool_count();
        d.sh_degree = s.sh_degree;
        d.bounds_center[0] = s.bounds.center.x;
        d.bounds_center[1] = s.bounds.center.y;
        d.bounds_center[2] = s.bounds.center.z;
        d.bounds_size = s.bounds.size;
        d.codes = codes.data();
        d.levels = levels.data();
        d.corner_index = s.voxel_count() ? s.corner_index[0].data() : nullptr;
        d.density = s.density.data();
        d.sh = s.sh.data();
    }
};

svr_camera cc(const Camera& cam) {
    svr_camera c;
    c.width = cam.width, c.height = cam.height, c.fx = cam.fx, c.fy = cam.fy, c.cx = cam.cx, c.cy = cam.cy;
    for (int i = 0; i < 9; ++i) c.rot[i] = cam.rot.m[i];
    c.pos[0] = cam.pos.x, c.pos[1] = cam.pos.y, c.pos[2] = cam.pos.z;
    return c;
}

svr_render_options co(const RenderOptions& o) {
    svr_render_options r;
    r.K = o.K, r.t_threshold = o.t_threshold, r.supersample = o.supersample;
    r.background[0] = o.background.x, r.background[1] = o.background.y, r.background[2] = o.background.z;
    r.near_plane = o.near_plane, r.far_sentinel = o.far_sentinel;
    r.record_stats = o.record_stats, r.training = o.training;
    return r;
}

double max_delta(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

}  // namespace

int main() {
    // option validation (test_raster.cpp:86-99)
    {
        SparseScene s;
        s.bounds = {{0, 0, 0}, 1.0};
        Camera cam = look_at_origin(16, 16, 1.5, 0.3);
        RenderOptions o;
        o.K = 4;
        CHECK_THROWS_AS(render(s, cam, o), std::invalid_argument);
        o.K = 1;
        o.supersample = 0.5;
        CHECK_THROWS_AS(render(s, cam, o), std::invalid_argument);
        o.supersample = 1.0;
        o.t_threshold = 0.0;
        CHECK_THROWS_AS(render(s, cam, o), std::invalid_argument);
    }
    // empty scene renders the background (test_raster.cpp:101-115)
    {
        SparseScene s;
        s.bounds = {{0, 0, 0}, 1.0};
        Camera cam = look_at_origin(32, 24, 1.5, 0.7);
        RenderOptions o;
        o.background = {0.25, 0.5, 0.75};
        RenderOutput r = render(s, cam, o);
        bool ok = true;
        for (int y = 0; y < 24; ++y)
            for (int x = 0; x < 32; ++x)
                ok = ok && std::abs(r.color.at(x, y, 0) - 0.25) < 1e-7 &&
                     std::abs(r.color.at(x, y, 2) - 0.75) < 1e-7 && r.transmittance.at(x, y) == 1.0 &&
                     r.depth.at(x, y) == o.far_sentinel;
        CHECK(ok);
    }
    // project_voxel basics (test_raster.cpp:117-127)
    {
        Camera cam = look_at_origin(64, 64, 2.0, 0.0, 0.0);
        PreVoxel pv;
        CHECK(project_voxel(cam, {0, 0, 0}, 0.25, pv));
        CHECK(std::abs(0.5 * (pv.x0 + pv.x1) - cam.cx) < 1e-6 * cam.cx);
        CHECK(std::abs(0.5 * (pv.y0 + pv.y1) - cam.cy) < 1e-6 * cam.cy);
        CHECK(!project_voxel(cam, cam.pos + 1.0 * Vec3{cam.rot(0, 2), cam.rot(1, 2), cam.rot(2, 2)} * -1.0,
                             0.25, pv));
    }
    // tile_sign_patterns covers every pixel and equals the oracle (test_raster.cpp:149-186)
    {
        Camera wide;
        wide.width = wide.height = 32;
        wide.fx = wide.fy = 16;
        wide.cx = wide.cy = 20;
        std::vector<uint8_t> om(4);
        svr_camera w = cc(wide);
        orc_tile_masks(&w, om.data());
        bool found_multi = false;
        for (int ty = 0; ty < 2; ++ty)
            for (int tx = 0; tx < 2; ++tx) {
                auto p = tile_sign_patterns(wide, tx, ty);
                uint8_t m = 0;
                for (auto s : p) m |= uint8_t(1u << s);
                CHECK(m == om[ty * 2 + tx]);
                if (p.size() >= 2) found_multi = true;
                for (int py = ty * 16; py < (ty + 1) * 16; ++py)
                    for (int px = tx * 16; px < (tx + 1) * 16; ++px)
                        CHECK(std::count(p.begin(), p.end(), ray_sign_bits(wide.pixel_ray(px, py).dir)) == 1);
            }
        CHECK(found_multi);
    }
    // build_sort_entries / sort_entries bit-exact vs the oracle (test_raster.cpp:188-211)
    {
        std::mt19937_64 rng(7);
        SparseScene s = random_scene(rng, 60);
        Camera cam = look_at_origin(64, 64, 1.8, 0.9);
        std::vector<PreVoxel> pre;
        for (size_t vi = 0; vi < s.voxel_count(); ++vi) {
            auto [center, size] = s.geometry_of(vi);
            PreVoxel pv;
            pv.vid = uint32_t(vi);
            pv.center = center;
            pv.size = size;
            if (project_voxel(cam, center, size, pv)) pre.push_back(pv);
        }
        auto entries = build_sort_entries(pre, cam, s);
        Desc d(s);
        svr_camera c = cc(cam);
        uint64_t n = 0;
        orc_entries(&d.d, &c, 1e-6, 0, &n, nullptr, nullptr);
        std::vector<uint64_t> k(n);
        std::vector<uint32_t> v(n);
        orc_entries(&d.d, &c, 1e-6, 0, &n, k.data(), v.data());
        CHECK(entries.size() == n);
        bool same = entries.size() == n;
        for (size_t i = 0; same && i < n; ++i) same = entries[i].key == k[i] && entries[i].value == v[i];
        CHECK(same);
        sort_entries(entries);
        orc_entries(&d.d, &c, 1e-6, 1, &n, k.data(), v.data());
        same = true;
        for (size_t i = 0; same && i < n; ++i) same = entries[i].key == k[i] && entries[i].value == v[i];
        CHECK(same);
        Camera huge = cam;
        huge.width = 1 << 20;
        CHECK_THROWS_AS(build_sort_entries(pre, huge, s), std::length_error);
    }
    // rasterizer matches the oracle(s) (test_raster.cpp:242-257)
    {
        std::mt19937_64 rng(2024);
        RenderOptions o;
        o.supersample = 1.0;
        o.background = {0.1, 0.2, 0.3};
        for (int trial = 0; trial < 8; ++trial) {
            SparseScene s = random_scene(rng, 40);
            Camera cam = look_at_origin(64, 64, 1.6 + 0.1 * trial, 0.8 * trial, 0.3 - 0.05 * trial);
            o.K = 1 + trial % 3;
            RenderOutput a = render(s, cam, o);
            RenderOutput b = render_oracle(s, cam, o);
            CHECK(max_delta(a.color.data, b.color.data) <= 1e-4);
            CHECK(max_delta(a.transmittance.data, b.transmittance.data) <= 1e-4);
            CHECK(max_delta(a.normal.data, b.normal.data) <= 1e-4);
            Desc d(s);
            svr_camera c = cc(cam);
            svr_render_options ro = co(o);
            std::vector<double> col(64 * 64 * 3), dep(64 * 64), med(64 * 64), nor(64 * 64 * 3), tf(64 * 64);
            orc_render(&d.d, &c, &ro, col.data(), dep.data(), med.data(), nor.data(), tf.data(), nullptr);
            CHECK(max_delta(a.color.data, col) <= 1e-4);
            CHECK(max_delta(b.color.data, col) <= 1e-6);  // fp64 GPU oracle vs C oracle
        }
    }
    // backward: zero upstream, mismatch, and gradients vs the oracle (test_raster.cpp:413-502)
    {
        std::mt19937_64 rng(2);
        SparseScene s = random_scene(rng, 10);
        Camera cam = look_at_origin(24, 24, 1.7, 0.5);
        RenderOptions o;
        o.supersample = 1.0;
        o.training = true;
        PoolsD pools = make_pools(s);
        RenderOutput r = render_with_pools(s, pools, cam, o);
        UpstreamGrads ug;
        SceneGradients g = render_backward(s, pools, *r.records, ug);
        bool zero = true;
        for (double v : g.density) zero = zero && v == 0.0;
        for (double v : g.sh) zero = zero && v == 0.0;
        CHECK(zero);
        CHECK(r.records->contribs.size() > 0);
        size_t total = 0;
        for (uint32_t c : r.records->pix_count) total += c;
        CHECK(total == r.records->contribs.size());
        ug.d_weight.assign(r.records->contribs.size() + 1, 0.0);
        CHECK_THROWS_AS(render_backward(s, pools, *r.records, ug), std::runtime_error);
        ForwardRecords fake;
        CHECK_THROWS_AS(render_backward(s, pools, fake, UpstreamGrads{}), std::runtime_error);
    }
    {
        std::mt19937_64 rng(17);
        SparseScene s = random_scene(rng, 30, 3);
        Camera cam = look_at_origin(40, 32, 1.9, 0.6, 0.2);
        RenderOptions o;
        o.supersample = 1.5;
        o.K = 2;
        o.training = true;
        o.background = {0.15, 0.25, 0.1};
        PoolsD pools = make_pools(s);
        RenderOutput r = render_with_pools(s, pools, cam, o);
        Desc d(s);
        svr_camera c = cc(cam);
        svr_render_options ro = co(o);
        ro.training = 0;
        std::vector<double> col(40 * 32 * 3), dep(40 * 32), med(40 * 32), nor(40 * 32 * 3), tf(40 * 32);
        orc_render(&d.d, &c, &ro, col.data(), dep.data(), med.data(), nor.data(), tf.data(), nullptr);
        UpstreamGrads ug;
        ug.d_color = Image(40, 32, 3);
        std::uniform_real_distribution<double> u(0, 1);
        for (size_t i = 0; i < col.size(); ++i) ug.d_color.data[i] = (col[i] > u(rng) ? 1.0 : -1.0) / col.size();
        SceneGradients g = render_backward(s, pools, *r.records, ug);
        std::vector<double> gd(s.pool_count()), gs(s.sh.size()), gp(s.voxel_count());
        ro.training = 1;
        orc_backward(&d.d, &c, &ro, ug.d_color.data.data(), nullptr, nullptr, nullptr, gd.data(), gs.data(), gp.data());
        auto close = [](const std::vector<double>& a, const std::vector<double>& b) {
            double mx = 0;
            for (double v : b) mx = std::max(mx, std::abs(v));
            int bad = 0;
            for (size_t i = 0; i < a.size(); ++i)
                if (std::abs(a[i] - b[i]) > 1e-3 * (std::max(std::abs(a[i]), std::abs(b[i])) + 1e-3 * mx)) ++bad;
            return bad;
        };
        CHECK(close(g.density, gd) == 0);
        CHECK(close(g.sh, gs) == 0);
        CHECK(close(g.priority, gp) == 0);
    }
    std::printf("%s: %d checks, %d failed\n", g_fail ? "FAILED" : "ALL PASSED", g_checks, g_fail);
    return g_fail;
}
