// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" shim around the UNMODIFIED reference sources
// (/root/reference/proj/src/{scene,image,raster,losses,...}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libsvr_ref.so. Only tests/, smoke() and
// bench.py's CPU-baseline leg load it, and only as the checker / the timed
// CPU baseline. Nothing here is reachable from the CUDA product path.
//
// Every function maps reference exceptions onto the svr_status codes of
// include/svr_b200.h so the tests can compare error behaviour too.

#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "svr/io.hpp"
#include "svr/losses.hpp"
#include "svr/optim.hpp"
#include "svr/raster.hpp"
#include "svr/synth.hpp"
#include "svr_b200.h"

using namespace svr;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SVR_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SVR_ERR_INVALID_ARGUMENT;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return SVR_ERR_LENGTH;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return SVR_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVR_ERR_RUNTIME;
    }
}

Camera to_cam(const svr_camera* c) {
    Camera cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 9; ++i) cam.rot.m[i] = c->rot[i];
    cam.pos = {c->pos[0], c->pos[1], c->pos[2]};
    return cam;
}

void from_cam(const Camera& cam, svr_camera* c) {
    c->width = cam.width;
    c->height = cam.height;
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->cx = cam.cx;
    c->cy = cam.cy;
    for (int i = 0; i < 9; ++i) c->rot[i] = cam.rot.m[i];
    c->pos[0] = cam.pos.x;
    c->pos[1] = cam.pos.y;
    c->pos[2] = cam.pos.z;
}

RenderOptions to_opts(const svr_render_options* o) {
    RenderOptions r;
    r.K = o->K;
    r.t_threshold = o->t_threshold;
    r.supersample = o->supersample;
    r.background = {o->background[0], o->background[1], o->background[2]};
    r.near_plane = o->near_plane;
    r.far_sentinel = o->far_sentinel;
    r.record_stats = o->record_stats != 0;
    r.training = o->training != 0;
    return r;
}

void copy_img(const Image& img, double* dst) {
    if (dst) std::memcpy(dst, img.data.data(), img.data.size() * sizeof(double));
}

// Public-API preprocess used by the reference tests (test_raster.cpp:68-82).
std::vector<PreVoxel> preprocess_public(const SparseScene& s, const Camera& cam, double near) {
    std::vector<PreVoxel> pre;
    for (size_t vi = 0; vi < s.voxel_count(); ++vi) {
        auto [center, size] = s.geometry_of(vi);
        PreVoxel pv;
        pv.vid = uint32_t(vi);
        pv.center = center;
        pv.size = size;
        if (!project_voxel(cam, center, size, pv, near)) continue;
        pv.V = s.corners_of(vi);
        pv.normal = voxel_normal(pv.V);
        pre.push_back(pv);
    }
    return pre;
}

struct Frame {
    std::shared_ptr<ForwardRecords> rec;
    RenderOutput out;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Generator G, built from the reference's own primitives
// (to_octpath, child_paths, rebuild_corner_indexing) with the RNG pattern of
// tests/test_raster.cpp:15-37 and a voxel-count target instead of a fixed
// subdivision count.
int ref_scene_gen(uint64_t seed, uint64_t target, int max_level, int sh_degree, void** out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        auto* s = new SparseScene;
        s->bounds = {{0, 0, 0}, 1.0};
        for (uint32_t i = 0; i < 8; ++i)
            for (uint32_t j = 0; j < 8; ++j)
                for (uint32_t k = 0; k < 8; ++k) s->voxels.push_back(to_octpath({i, j, k, 3}));
        while (s->voxels.size() + 7 <= target) {
            size_t pick = rng() % s->voxels.size();
            if (s->voxels[pick].level >= max_level) continue;
            auto kids = child_paths(s->voxels[pick]);
            s->voxels[pick] = kids[0];
            for (int c = 1; c < 8; ++c) s->voxels.push_back(kids[c]);
        }
        rebuild_corner_indexing(*s, {});
        std::uniform_real_distribution<double> ud(-4.0, 2.5), uc(0.05, 0.8);
        for (auto& d : s->density) d = float(ud(rng));
        s->sh_degree = sh_degree;
        s->sh.assign(s->voxel_count() * s->sh_stride(), 0.0f);
        for (size_t vi = 0; vi < s->voxel_count(); ++vi) {
            float* sh = s->sh_of(vi);
            for (int ch = 0; ch < 3; ++ch) sh[ch] = float(sh_dc_for_intensity(uc(rng)));
            for (int m = 3; m < s->sh_stride(); ++m) sh[m] = float(0.1 * (uc(rng) - 0.4));
        }
        *out = s;
    });
}

// Config-4/5 scene: the reference's own init_unbounded
// (optim.cpp:96-184), then parameters drawn as generator G from a fresh
// mt19937_64(seed) (density per pool entry, then SH per voxel).
int ref_scene_unbounded(const svr_camera* cams, int n_cams, int init_level, int shell_levels,
                        double bg_ratio, uint64_t seed, int sh_degree, void** out) {
    return guarded([&] {
        std::vector<Camera> cv;
        for (int i = 0; i < n_cams; ++i) cv.push_back(to_cam(&cams[i]));
        TrainConfig cfg;
        cfg.init_level = init_level;
        cfg.shell_levels = shell_levels;
        cfg.bg_ratio = bg_ratio;
        cfg.sh_degree = sh_degree;
        auto* s = new SparseScene(init_unbounded(cv, cfg));
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> ud(-4.0, 2.5), uc(0.05, 0.8);
        for (auto& d : s->density) d = float(ud(rng));
        for (size_t vi = 0; vi < s->voxel_count(); ++vi) {
            float* sh = s->sh_of(vi);
            for (int ch = 0; ch < 3; ++ch) sh[ch] = float(sh_dc_for_intensity(uc(rng)));
            for (int m = 3; m < s->sh_stride(); ++m) sh[m] = float(0.1 * (uc(rng) - 0.4));
        }
        *out = s;
    });
}

void ref_scene_bounds(void* h, double* center, double* size) {
    auto* s = static_cast<SparseScene*>(h);
    center[0] = s->bounds.center.x;
    center[1] = s->bounds.center.y;
    center[2] = s->bounds.center.z;
    *size = s->bounds.size;
}

// Scene from explicit arrays (fixtures built elsewhere).
int ref_scene_make(const svr_scene_desc* d, void** out) {
    return guarded([&] {
        auto* s = new SparseScene;
        s->bounds = {{d->bounds_center[0], d->bounds_center[1], d->bounds_center[2]},
                     d->bounds_size};
        s->voxels.resize(d->n_voxels);
        s->corner_index.resize(d->n_voxels);
        for (uint64_t i = 0; i < d->n_voxels; ++i) {
            s->voxels[i] = {d->codes[i], int(d->levels[i])};
            for (int c = 0; c < 8; ++c) s->corner_index[i][c] = d->corner_index[8 * i + c];
        }
        s->density.assign(d->density, d->density + d->n_pool);
        s->sh_degree = d->sh_degree;
        s->sh.assign(d->sh, d->sh + d->n_voxels * s->sh_stride());
        *out = s;
    });
}

// Rebuild corner indexing with a constant fill (tests like test_raster.cpp:284-309).
int ref_scene_from_paths(const uint64_t* codes, const uint8_t* levels, uint64_t n, float fill,
                         int sh_degree, void** out) {
    return guarded([&] {
        auto* s = new SparseScene;
        s->bounds = {{0, 0, 0}, 1.0};
        for (uint64_t i = 0; i < n; ++i) s->voxels.push_back({codes[i], int(levels[i])});
        rebuild_corner_indexing(*s, {}, fill);
        s->sh_degree = sh_degree;
        s->sh.assign(s->voxel_count() * s->sh_stride(), 0.0f);
        *out = s;
    });
}

void ref_scene_free(void* h) { delete static_cast<SparseScene*>(h); }

// save_checkpoint / load_checkpoint (io.cpp:250-359): the reference's SVRX
// writer and reader, to pin svr_scene_save_svrx / svr_scene_load_svrx.
int ref_save_checkpoint(void* h, const char* path) {
    return guarded([&] { save_checkpoint(*static_cast<SparseScene*>(h), path); });
}

int ref_load_checkpoint(const char* path, void** out) {
    return guarded([&] { *out = new SparseScene(load_checkpoint(path)); });
}


void ref_scene_sizes(void* h, uint64_t* n, uint64_t* p, int* deg) {
    auto* s = static_cast<SparseScene*>(h);
    *n = s->voxel_count();
    *p = s->pool_count();
    *deg = s->sh_degree;
}

void ref_scene_export(void* h, uint64_t* codes, uint8_t* levels, uint32_t* ci, float* dens,
                      float* sh) {
    auto* s = static_cast<SparseScene*>(h);
    for (size_t i = 0; i < s->voxel_count(); ++i) {
        if (codes) codes[i] = s->voxels[i].code;
        if (levels) levels[i] = uint8_t(s->voxels[i].level);
        if (ci)
            for (int c = 0; c < 8; ++c) ci[8 * i + c] = s->corner_index[i][c];
    }
    if (dens) std::memcpy(dens, s->density.data(), s->density.size() * sizeof(float));
    if (sh) std::memcpy(sh, s->sh.data(), s->sh.size() * sizeof(float));
}

void ref_scene_set_params(void* h, const float* dens, const float* sh) {
    auto* s = static_cast<SparseScene*>(h);
    if (dens) std::memcpy(s->density.data(), dens, s->density.size() * sizeof(float));
    if (sh) std::memcpy(s->sh.data(), sh, s->sh.size() * sizeof(float));
}

int ref_ring_camera(int n, int i, int w, int h, double dist, double fov, svr_camera* out) {
    return guarded([&] {
        auto cams = ring_cameras(n, w, h, dist, fov);
        from_cam(cams.at(size_t(i)), out);
    });
}

int ref_scaled_camera(const svr_camera* c, double ss, svr_camera* out) {
    return guarded([&] {
        Camera cam = to_cam(c);
        int sw = int(std::ceil(ss * cam.width)), sh = int(std::ceil(ss * cam.height));
        from_cam(cam.scaled(sw, sh), out);
    });
}

// svr::render / render_oracle; outputs at target resolution (double).
int ref_render(void* h, const svr_camera* c, const svr_render_options* o, int oracle,
               double* color, double* depth, double* median, double* normal, double* tfin,
               double* max_blend) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        RenderOptions opts = to_opts(o);
        opts.training = false;
        RenderOutput r = oracle ? render_oracle(*s, to_cam(c), opts) : render(*s, to_cam(c), opts);
        copy_img(r.color, color);
        copy_img(r.depth, depth);
        copy_img(r.median_depth, median);
        copy_img(r.normal, normal);
        copy_img(r.transmittance, tfin);
        if (max_blend && !r.max_blend_weight.empty())
            std::memcpy(max_blend, r.max_blend_weight.data(),
                        r.max_blend_weight.size() * sizeof(double));
    });
}

// project_voxel over every voxel (geometry_of + project_voxel), on the
// camera given (callers pass the supersampled camera).
int ref_project(void* h, const svr_camera* c, double near, uint8_t* visible, double* aabb,
                int32_t* rect) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        Camera cam = to_cam(c);
        for (size_t vi = 0; vi < s->voxel_count(); ++vi) {
            auto [center, size] = s->geometry_of(vi);
            PreVoxel pv;
            bool ok = project_voxel(cam, center, size, pv, near);
            visible[vi] = ok ? 1 : 0;
            aabb[4 * vi + 0] = ok ? pv.x0 : 0;
            aabb[4 * vi + 1] = ok ? pv.x1 : 0;
            aabb[4 * vi + 2] = ok ? pv.y0 : 0;
            aabb[4 * vi + 3] = ok ? pv.y1 : 0;
            rect[4 * vi + 0] = pv.tx0;
            rect[4 * vi + 1] = pv.tx1;
            rect[4 * vi + 2] = pv.ty0;
            rect[4 * vi + 3] = pv.ty1;
        }
    });
}

int ref_project_one(const svr_camera* c, const double* center, double size, double near,
                    double* aabb, int32_t* rect, int* visible) {
    return guarded([&] {
        PreVoxel pv;
        bool ok = project_voxel(to_cam(c), {center[0], center[1], center[2]}, size, pv, near);
        *visible = ok;
        aabb[0] = pv.x0;
        aabb[1] = pv.x1;
        aabb[2] = pv.y0;
        aabb[3] = pv.y1;
        rect[0] = pv.tx0;
        rect[1] = pv.tx1;
        rect[2] = pv.ty0;
        rect[3] = pv.ty1;
    });
}

int ref_tile_masks(const svr_camera* c, uint8_t* masks) {
    return guarded([&] {
        Camera cam = to_cam(c);
        int ntx = (cam.width + kTileSize - 1) / kTileSize;
        int nty = (cam.height + kTileSize - 1) / kTileSize;
        for (int ty = 0; ty < nty; ++ty)
            for (int tx = 0; tx < ntx; ++tx) {
                uint8_t m = 0;
                for (SignBits sb : tile_sign_patterns(cam, tx, ty)) m |= uint8_t(1u << sb);
                masks[size_t(ty) * ntx + tx] = m;
            }
    });
}

// build_sort_entries (+ sort_entries when sorted != 0) on the given camera.
// Two-phase: keys == NULL returns the count.
int ref_entries(void* h, const svr_camera* c, double near, int sorted, uint64_t* n_out,
                uint64_t* keys, uint32_t* values) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        Camera cam = to_cam(c);
        auto pre = preprocess_public(*s, cam, near);
        auto entries = build_sort_entries(pre, cam, *s);
        if (sorted) sort_entries(entries);
        *n_out = entries.size();
        if (keys)
            for (size_t i = 0; i < entries.size(); ++i) {
                keys[i] = entries[i].key;
                values[i] = entries[i].value;
            }
    });
}

// Entry list of one view held on the reference side, so a large view
// (config 4: ~97M entries) is built once and read back emitted, then sorted.
int ref_entries_begin(void* h, const svr_camera* c, double near, void** out, uint64_t* n_out) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        Camera cam = to_cam(c);
        auto pre = preprocess_public(*s, cam, near);
        auto* e = new std::vector<SortEntry>(build_sort_entries(pre, cam, *s));
        *out = e;
        *n_out = e->size();
    });
}

int ref_entries_copy(void* h, int sort_first, uint64_t* keys, uint32_t* values) {
    return guarded([&] {
        auto* e = static_cast<std::vector<SortEntry>*>(h);
        if (sort_first) sort_entries(*e);
        for (size_t i = 0; i < e->size(); ++i) {
            keys[i] = (*e)[i].key;
            values[i] = (*e)[i].value;
        }
    });
}

void ref_entries_end(void* h) { delete static_cast<std::vector<SortEntry>*>(h); }

int ref_sort_entries(uint64_t n, uint64_t* keys, uint32_t* values) {
    return guarded([&] {
        std::vector<SortEntry> e(n);
        for (uint64_t i = 0; i < n; ++i) e[i] = {keys[i], values[i]};
        sort_entries(e);
        for (uint64_t i = 0; i < n; ++i) {
            keys[i] = e[i].key;
            values[i] = e[i].value;
        }
    });
}

// Training forward. Returns a frame handle holding the ForwardRecords.
int ref_forward_train(void* h, const svr_camera* c, const svr_render_options* o, void** frame,
                      uint64_t* n_pre, uint64_t* n_contribs, double* color, double* depth,
                      double* normal, double* tfin) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        RenderOptions opts = to_opts(o);
        opts.training = true;
        auto* f = new Frame;
        f->out = render_with_pools(*s, make_pools(*s), to_cam(c), opts);
        f->rec = f->out.records;
        *n_pre = f->rec->pre.size();
        *n_contribs = f->rec->contribs.size();
        copy_img(f->out.color, color);
        copy_img(f->out.depth, depth);
        copy_img(f->out.normal, normal);
        copy_img(f->out.transmittance, tfin);
        *frame = f;
    });
}

void ref_frame_free(void* f) { delete static_cast<Frame*>(f); }

void ref_frame_records(void* fh, uint32_t* pre_vids, uint32_t* contrib_pre, double* a, double* b,
                       uint32_t* pix_begin, uint32_t* pix_count, double* ss_tfin) {
    auto* f = static_cast<Frame*>(fh);
    const ForwardRecords& r = *f->rec;
    if (pre_vids)
        for (size_t i = 0; i < r.pre.size(); ++i) pre_vids[i] = r.pre[i].vid;
    for (size_t i = 0; i < r.contribs.size(); ++i) {
        if (contrib_pre) contrib_pre[i] = r.contribs[i].pre;
        if (a) a[i] = r.contribs[i].a;
        if (b) b[i] = r.contribs[i].b;
    }
    if (pix_begin) std::memcpy(pix_begin, r.pix_begin.data(), r.pix_begin.size() * 4);
    if (pix_count) std::memcpy(pix_count, r.pix_count.data(), r.pix_count.size() * 4);
    if (ss_tfin) copy_img(r.ss_tfin, ss_tfin);
}

// The gradient of one optim::train iteration (optim.cpp:433-477): render
// (training) -> mse + lambda_ssim * ssim -> ray_losses -> render_backward.
int ref_train_iteration_grads(void* h, const svr_camera* c, const svr_render_options* o,
                              const double* gt, double lambda_ssim, double w_T, double w_dist,
                              double w_R, double* losses, double* g_density, double* g_sh,
                              double* g_priority) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        RenderOptions opts = to_opts(o);
        opts.training = true;
        PoolsD pools = make_pools(*s);
        RenderOutput out = render_with_pools(*s, pools, to_cam(c), opts);
        Image g(out.color.width, out.color.height, 3);
        std::memcpy(g.data.data(), gt, g.data.size() * sizeof(double));
        UpstreamGrads ug;
        ug.d_color = Image(g.width, g.height, 3);
        losses[0] = mse_loss(out.color, g, 1.0, &ug.d_color);
        losses[1] = ssim_loss(out.color, g, lambda_ssim, &ug.d_color);
        RayLossWeights rw;
        rw.w_T = w_T;
        rw.w_dist = w_dist;
        rw.w_R = w_R;
        RayLossValues rv = ray_losses(*s, *out.records, g, rw, ug);
        losses[2] = rv.l_T;
        losses[3] = rv.l_dist;
        losses[4] = rv.l_R;
        SceneGradients sg = render_backward(*s, pools, *out.records, ug);
        std::memcpy(g_density, sg.density.data(), sg.density.size() * sizeof(double));
        std::memcpy(g_sh, sg.sh.data(), sg.sh.size() * sizeof(double));
        std::memcpy(g_priority, sg.priority.data(), sg.priority.size() * sizeof(double));
    });
}

// mse_loss + ssim_loss (losses.cpp:71-139) of a W x H x 3 image; d (may be
// NULL) receives w_mse * dMSE + w_ssim * d(1 - SSIM).
int ref_image_losses(const double* a, const double* b, int W, int H, double w_mse, double w_ssim,
                     double* out, double* d) {
    return guarded([&] {
        Image ia(W, H, 3), ib(W, H, 3);
        std::memcpy(ia.data.data(), a, ia.data.size() * sizeof(double));
        std::memcpy(ib.data.data(), b, ib.data.size() * sizeof(double));
        Image g(W, H, 3);
        out[0] = mse_loss(ia, ib, w_mse, d ? &g : nullptr);
        out[1] = ssim_loss(ia, ib, w_ssim, d ? &g : nullptr);
        if (d) std::memcpy(d, g.data.data(), g.data.size() * sizeof(double));
    });
}

// adam_step (optim.cpp:322-345) on host arrays: params (float), grads
// (double), moments (double); lr_alt applies where i % period >= n_primary.
int ref_adam_step(float* params, const double* grads, double* m, double* v, uint64_t n,
                  int64_t step_before, double lr, double lr_alt, uint32_t period,
                  uint32_t n_primary, double beta1, double beta2, double eps) {
    return guarded([&] {
        std::vector<float> p(params, params + n);
        std::vector<double> g(grads, grads + n);
        AdamState st;
        st.m.assign(m, m + n);
        st.v.assign(v, v + n);
        st.step = step_before;
        std::function<double(size_t)> lr_of = nullptr;
        if (period)
            lr_of = [&](size_t i) { return (i % period) >= n_primary ? lr_alt : lr; };
        adam_step(p, g, st, lr, lr_of, beta1, beta2, eps);
        std::memcpy(params, p.data(), n * 4);
        std::memcpy(m, st.m.data(), n * 8);
        std::memcpy(v, st.v.data(), n * 8);
    });
}

// prune / subdivide_voxels (optim.cpp:207-298) with their AdaptRemap; the
// remap arrays must hold the new voxel / pool counts (callers over-allocate).
int ref_prune(void* h, const double* stats, double thr, void** out, int64_t* voxel_src,
              int64_t* pool_src, uint64_t* n_vox, uint64_t* n_pool) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        std::vector<double> st(stats, stats + s->voxel_count());
        AdaptRemap rm;
        auto* o = new SparseScene(prune(*s, st, thr, &rm));
        *n_vox = o->voxel_count();
        *n_pool = o->pool_count();
        std::memcpy(voxel_src, rm.voxel_src.data(), rm.voxel_src.size() * 8);
        std::memcpy(pool_src, rm.pool_src.data(), rm.pool_src.size() * 8);
        *out = o;
    });
}

int ref_subdivide(void* h, const uint32_t* sel, uint64_t n_sel, void** out, int64_t* voxel_src,
                  int64_t* pool_src, uint64_t* n_vox, uint64_t* n_pool) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        std::vector<uint32_t> sv(sel, sel + n_sel);
        AdaptRemap rm;
        auto* o = new SparseScene(subdivide_voxels(*s, sv, &rm));
        *n_vox = o->voxel_count();
        *n_pool = o->pool_count();
        std::memcpy(voxel_src, rm.voxel_src.data(), rm.voxel_src.size() * 8);
        std::memcpy(pool_src, rm.pool_src.data(), rm.pool_src.size() * 8);
        *out = o;
    });
}

// ray_losses (losses.cpp:141-238) on a training frame; fresh zero upstream
// buffers sized by the reference itself, copied out (NULL = not wanted).
int ref_frame_ray_losses(void* fh, const double* gt, double w_T, double w_dist, double w_R,
                         double* values, double* d_tfin_ss, double* d_weight,
                         double* d_voxel_color) {
    return guarded([&] {
        auto* f = static_cast<Frame*>(fh);
        const ForwardRecords& r = *f->rec;
        const int W = f->out.color.width, H = f->out.color.height;
        Image g(W, H, 3);
        std::memcpy(g.data.data(), gt, g.data.size() * sizeof(double));
        RayLossWeights w;
        w.w_T = w_T;
        w.w_dist = w_dist;
        w.w_R = w_R;
        UpstreamGrads ug;
        RayLossValues v = ray_losses(SparseScene{}, r, g, w, ug);
        values[0] = v.l_T;
        values[1] = v.l_dist;
        values[2] = v.l_R;
        if (d_tfin_ss && !ug.d_tfin_ss.empty())
            std::memcpy(d_tfin_ss, ug.d_tfin_ss.data(), ug.d_tfin_ss.size() * sizeof(double));
        if (d_weight && !ug.d_weight.empty())
            std::memcpy(d_weight, ug.d_weight.data(), ug.d_weight.size() * sizeof(double));
        if (d_voxel_color)
            for (size_t i = 0; i < ug.d_voxel_color.size(); ++i)
                for (int c = 0; c < 3; ++c) d_voxel_color[3 * i + c] = ug.d_voxel_color[i][c];
    });
}

// render_backward with image-level upstream grads at target resolution.
// Any pointer may be NULL (= empty buffer = zero, raster.hpp:100-110).
int ref_backward(void* h, void* fh, const double* d_color, const double* d_depth,
                 const double* d_normal, const double* d_tfin_ss, const double* d_weight,
                 uint64_t n_weight, const double* d_voxel_color, uint64_t n_vc,
                 double* g_density, double* g_sh, double* g_priority) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        auto* f = static_cast<Frame*>(fh);
        const ForwardRecords& r = *f->rec;
        int W = f->out.color.width, H = f->out.color.height;
        UpstreamGrads ug;
        auto img = [&](const double* p, int ch) {
            Image im;
            if (p) {
                im = Image(W, H, ch);
                std::memcpy(im.data.data(), p, im.data.size() * sizeof(double));
            }
            return im;
        };
        ug.d_color = img(d_color, 3);
        ug.d_depth = img(d_depth, 1);
        ug.d_normal = img(d_normal, 3);
        if (d_tfin_ss)
            ug.d_tfin_ss.assign(d_tfin_ss, d_tfin_ss + size_t(r.ss_cam.width) * r.ss_cam.height);
        if (d_weight) ug.d_weight.assign(d_weight, d_weight + n_weight);
        if (d_voxel_color)
            for (uint64_t i = 0; i < n_vc; ++i)
                ug.d_voxel_color.push_back(
                    {d_voxel_color[3 * i], d_voxel_color[3 * i + 1], d_voxel_color[3 * i + 2]});
        SceneGradients g = render_backward(*s, make_pools(*s), r, ug);
        std::memcpy(g_density, g.density.data(), g.density.size() * sizeof(double));
        std::memcpy(g_sh, g.sh.data(), g.sh.size() * sizeof(double));
        std::memcpy(g_priority, g.priority.data(), g.priority.size() * sizeof(double));
    });
}

// The config-3 training step on the CPU: render(training) -> L1 -> backward.
// L1 is new (no reference), written in the pattern of mse_loss
// (losses.cpp:121-131): L = mean|C-gt|, dL/dC = sign(C-gt)/(3WH).
int ref_train_step_l1(void* h, const svr_camera* c, const svr_render_options* o,
                      const double* gt, double* loss, double* d_color_out, double* g_density,
                      double* g_sh, double* g_priority) {
    return guarded([&] {
        auto* s = static_cast<SparseScene*>(h);
        RenderOptions opts = to_opts(o);
        opts.training = true;
        PoolsD pools = make_pools(*s);
        RenderOutput r = render_with_pools(*s, pools, to_cam(c), opts);
        UpstreamGrads ug;
        ug.d_color = Image(r.color.width, r.color.height, 3);
        const double inv_n = 1.0 / double(r.color.data.size());
        double total = 0.0;
        for (size_t i = 0; i < r.color.data.size(); ++i) {
            double e = r.color.data[i] - gt[i];
            total += std::abs(e);
            ug.d_color.data[i] = (e > 0 ? 1.0 : (e < 0 ? -1.0 : 0.0)) * inv_n;
        }
        *loss = total * inv_n;
        if (d_color_out) copy_img(ug.d_color, d_color_out);
        SceneGradients g = render_backward(*s, pools, *r.records, ug);
        std::memcpy(g_density, g.density.data(), g.density.size() * sizeof(double));
        std::memcpy(g_sh, g.sh.data(), g.sh.size() * sizeof(double));
        std::memcpy(g_priority, g.priority.data(), g.priority.size() * sizeof(double));
    });
}

}  // extern "C"
