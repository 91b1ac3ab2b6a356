// dropin_support.cu — C-ABI pieces that exist so the C++ drop-in
// (paper_2412_04459_b200/cpp/raster_dropin.cpp) can serve the whole of
// raster.hpp:
//   * svr_frame_pre      ForwardRecords::pre (raster.hpp:55-64, 72-82) for a
//                        rendered frame: exact fp64 geometry/AABB, V, colour,
//                        normal of every visible voxel in vid order;
//   * svr_render_oracle  render_oracle (raster.cpp:425-473): per pixel,
//                        intersect every visible voxel, composite the hits in
//                        (entry distance, dir_dep_order) order. fp64 on the
//                        GPU, one thread per pixel, O(hits x voxels) per ray —
//                        a test oracle for small scenes, not a render path.
#include <cuda_runtime.h>

#include <cmath>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {
namespace {

constexpr uint64_t kMask48 = (uint64_t(1) << 48) - 1;

__global__ void frame_pre_kernel(DevCamera cam, uint64_t n, const uint64_t* paths, const int4* rects,
                                 const uint32_t* rank, const float4* records,
                                 const uint32_t* corner_index, const float* density,
                                 const double* bc, double bsize, double near_plane,
                                 svr_pre_voxel* out) {
    uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int4 r = rects[v];
    if (r.y < r.x) return;
    svr_pre_voxel p;
    p.vid = uint32_t(v);
    double center[3], size;
    voxel_geometry(paths[v] & kMask48, int(paths[v] >> 48), bc, bsize, center, &size);
    Projection pr;
    project_voxel(cam, center, size, near_plane, pr);
    for (int i = 0; i < 3; ++i) p.center[i] = center[i];
    p.size = size;
    for (int c = 0; c < 8; ++c) p.V[c] = density[corner_index[8 * v + c]];
    const float4* rec = records + v * kRecordF4;
    p.color[0] = rec[4].x, p.color[1] = rec[4].y, p.color[2] = rec[4].z;
    // density_gradient in double from the exact corner values (field.hpp:132-154)
    double g[3] = {0, 0, 0};
    for (int c = 0; c < 8; ++c) {
        g[0] += 0.25 * p.V[c] * (((c >> 2) & 1) ? 1.0 : -1.0);
        g[1] += 0.25 * p.V[c] * (((c >> 1) & 1) ? 1.0 : -1.0);
        g[2] += 0.25 * p.V[c] * ((c & 1) ? 1.0 : -1.0);
    }
    const double len = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    p.degenerate = len == 0.0;
    for (int i = 0; i < 3; ++i) {
        p.raw[i] = g[i];
        p.normal[i] = len == 0.0 ? 0.0 : g[i] / len;
    }
    p.x0 = pr.x0, p.x1 = pr.x1, p.y0 = pr.y0, p.y1 = pr.y1;
    p.tx0 = pr.tx0, p.tx1 = pr.tx1, p.ty0 = pr.ty0, p.ty1 = pr.ty1;
    out[rank[v]] = p;
}

// Per visible voxel, fp64 data for the oracle: centre, size, V, colour, normal.
struct OracleVoxel {
    double c[3], size, V[8], col[3], n[3];
    uint64_t code;
};

__global__ void oracle_prep_kernel(DevCamera cam, uint64_t n, const uint64_t* paths,
                                   const uint32_t* corner_index, const float* density,
                                   const float* sh, int deg, int stride, const double* bc,
                                   double bsize, double near_plane, OracleVoxel* out,
                                   unsigned int* count) {
    uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    double center[3], size;
    voxel_geometry(paths[v] & kMask48, int(paths[v] >> 48), bc, bsize, center, &size);
    Projection pr;
    if (!project_voxel(cam, center, size, near_plane, pr)) return;
    OracleVoxel o;
    for (int i = 0; i < 3; ++i) o.c[i] = center[i];
    o.size = size;
    o.code = paths[v] & kMask48;
    for (int c = 0; c < 8; ++c) o.V[c] = density[corner_index[8 * v + c]];
    // sh_eval in double (sh.hpp:48-58)
    double d[3] = {center[0] - cam.pos[0], center[1] - cam.pos[1], center[2] - cam.pos[2]};
    double nr = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double x = nr > 0 ? d[0] / nr : 0, y = nr > 0 ? d[1] / nr : 0, z = nr > 0 ? d[2] / nr : 0;
    double b[16] = {0};
    b[0] = 0.28209479177387814;
    if (deg >= 1) {
        b[1] = -0.4886025119029199 * y;
        b[2] = 0.4886025119029199 * z;
        b[3] = -0.4886025119029199 * x;
    }
    if (deg >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        b[4] = 1.0925484305920792 * x * y;
        b[5] = -1.0925484305920792 * y * z;
        b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        b[7] = -1.0925484305920792 * x * z;
        b[8] = 0.5462742152960396 * (xx - yy);
        if (deg >= 3) {
            b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
            b[10] = 2.890611442640554 * x * y * z;
            b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            b[14] = 1.445305721320277 * z * (xx - yy);
            b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
    }
    const int nb = (deg + 1) * (deg + 1);
    for (int ch = 0; ch < 3; ++ch) {
        double s = 0;
        for (int m = 0; m < nb; ++m) s += b[m] * sh[v * stride + 3 * m + ch];
        o.col[ch] = s > 0 ? s : 0;
    }
    double g[3] = {0, 0, 0};
    for (int c = 0; c < 8; ++c) {
        g[0] += 0.25 * o.V[c] * (((c >> 2) & 1) ? 1.0 : -1.0);
        g[1] += 0.25 * o.V[c] * (((c >> 1) & 1) ? 1.0 : -1.0);
        g[2] += 0.25 * o.V[c] * ((c & 1) ? 1.0 : -1.0);
    }
    double len = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    for (int i = 0; i < 3; ++i) o.n[i] = len == 0.0 ? 0.0 : g[i] / len;
    out[atomicAdd(count, 1u)] = o;
}

__device__ bool slab64(const OracleVoxel& v, const double* o, const double* d, double& a, double& b) {
    a = -INFINITY;
    b = INFINITY;
    for (int ax = 0; ax < 3; ++ax) {  // field.hpp:58-69 with std::min/max semantics
        double lo = v.c[ax] - 0.5 * v.size, hi = v.c[ax] + 0.5 * v.size;
        double c0 = (lo - o[ax]) / d[ax], c1 = (hi - o[ax]) / d[ax];
        double mn = (c1 < c0) ? c1 : c0, mx = (c0 < c1) ? c1 : c0;
        a = (a < mn) ? mn : a;
        b = (mx < b) ? mx : b;
    }
    return (a <= b) && (a > 0.0);
}

__device__ double explin64(double x) { return x > 1.1 ? x : exp(x / 1.1 - 1.0 + log(1.1)); }

__global__ void oracle_render_kernel(DevCamera cam, const OracleVoxel* vox, const unsigned int* count,
                                     int K, double thr, double bg0, double bg1, double bg2, double far,
                                     float* color, float* depth, float* median, float* normal,
                                     float* tfin) {
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y;
    if (px >= cam.W) return;
    const unsigned int n = *count;
    double d[3];
    pixel_ray_dir(cam, double(px), double(py), d);
    const uint32_t s = sign_bits(d);
    const uint64_t S = uint64_t(s) * kGroupOnes;
    const double o[3] = {cam.pos[0], cam.pos[1], cam.pos[2]};
    const double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double T = 1.0, col[3] = {0, 0, 0}, nor[3] = {0, 0, 0}, dep = 0.0, med = -1.0;
    int cntc = 0;
    double last_a = -INFINITY;
    uint64_t last_o = 0;
    bool first = true;
    for (;;) {
        int best = -1;
        double ba = INFINITY, bb = 0;
        uint64_t bo = ~uint64_t(0);
        for (unsigned int p = 0; p < n; ++p) {
            double a, b;
            if (!slab64(vox[p], o, d, a, b)) continue;
            const uint64_t ord = vox[p].code ^ S;
            const bool after = first || a > last_a || (a == last_a && ord > last_o);
            const bool before = a < ba || (a == ba && ord < bo);
            if (after && before) {
                best = int(p);
                ba = a;
                bb = b;
                bo = ord;
            }
        }
        if (best < 0) break;
        first = false;
        last_a = ba;
        last_o = bo;
        const OracleVoxel& v = vox[best];
        // CompositeCtx::add (raster.cpp:30-54) in fp64
        const double l = (bb - ba) * dn;
        double sum = 0, sa[3], tk[3];
        const double lo[3] = {v.c[0] - 0.5 * v.size, v.c[1] - 0.5 * v.size, v.c[2] - 0.5 * v.size};
        for (int k = 0; k < K; ++k) {
            const double t = ba + (k + 0.5) / K * (bb - ba);
            double q[3];
            for (int ax = 0; ax < 3; ++ax) q[ax] = (o[ax] + t * d[ax] - lo[ax]) / v.size;
            double val = 0;
            for (int c = 0; c < 8; ++c)
                val += (((c >> 2) & 1) ? q[0] : 1 - q[0]) * (((c >> 1) & 1) ? q[1] : 1 - q[1]) *
                       ((c & 1) ? q[2] : 1 - q[2]) * v.V[c];
            const double act = explin64(val);
            sum += act;
            tk[k] = t;
            sa[k] = 1.0 - exp(-(l / K) * act);
        }
        const double alpha = 1.0 - exp(-(l / K) * sum);
        double dv = 0, Tk = 1;
        for (int k = 0; k < K; ++k) {
            dv += Tk * sa[k] * tk[k];
            Tk *= 1.0 - sa[k];
        }
        for (int i = 0; i < 3; ++i) {
            col[i] += T * alpha * v.col[i];
            nor[i] += T * alpha * v.n[i];
        }
        dep += T * dv;
        if (med < 0.0) {
            double Tf = T;
            for (int k = 0; k < K; ++k) {
                Tf *= 1.0 - sa[k];
                if (Tf < 0.5) {
                    med = tk[k];
                    break;
                }
            }
        }
        T *= 1.0 - alpha;
        ++cntc;
        if (T < thr) break;
    }
    col[0] += T * bg0;
    col[1] += T * bg1;
    col[2] += T * bg2;
    if (cntc == 0) dep = far;
    if (med < 0.0) med = far;
    const uint64_t p = uint64_t(py) * cam.W + px;
    for (int i = 0; i < 3; ++i) {
        color[3 * p + i] = float(col[i]);
        normal[3 * p + i] = float(nor[i]);
    }
    depth[p] = float(dep);
    median[p] = float(med);
    tfin[p] = float(T);
}

}  // namespace
}  // namespace svrb

using namespace svrb;

namespace svrb {
uint64_t frame_visible_count(svr_frame* f);  // capi.cu
int guarded_call(void (*fn)(void*), void* arg);
DevCamera make_dev_camera(const svr_camera& c);
}

extern "C" int svr_frame_pre(svr_frame* f, svr_pre_voxel* out, uint64_t n) {
    struct Arg {
        svr_frame* f;
        svr_pre_voxel* out;
        uint64_t n;
    } arg{f, out, n};
    return guarded_call(
        [](void* p) {
            Arg& a = *static_cast<Arg*>(p);
            svr_frame* f = a.f;
            if (!f || !f->scene) throw Error(SVR_ERR_INVALID_ARGUMENT, "frame has not been rendered");
            SVR_CUDA(cudaSetDevice(f->ctx->device));
            const uint64_t nv = frame_visible_count(f);
            if (a.n != nv) throw Error(SVR_ERR_INVALID_ARGUMENT, "pre size mismatch");
            if (!nv) return;
            cudaStream_t st = f->ctx->stream;
            DevBuf dout, dbc;
            dout.reserve(nv * sizeof(svr_pre_voxel));
            dbc.reserve(3 * sizeof(double));
            SVR_CUDA(cudaMemcpyAsync(dbc.p, f->scene->bounds_center, 24, cudaMemcpyHostToDevice, st));
            const uint64_t N = f->n_voxels;
            frame_pre_kernel<<<unsigned((N + 127) / 128), 128, 0, st>>>(
                f->cam, N, f->scene->paths.as<uint64_t>(), f->rects.as<int4>(),
                f->visible_rank.as<uint32_t>(), f->records.as<float4>(),
                f->scene->corner_index.as<uint32_t>(), f->scene->density.as<float>(),
                dbc.as<double>(), f->scene->bounds_size, f->opts.near_plane,
                dout.as<svr_pre_voxel>());
            SVR_LAUNCH("frame_pre_kernel");
            SVR_CUDA(cudaMemcpyAsync(a.out, dout.p, nv * sizeof(svr_pre_voxel), cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaStreamSynchronize(st));
        },
        &arg);
}

extern "C" int svr_render_oracle(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
                                 const svr_render_options* opts, svr_frame* f) {
    struct Arg {
        svr_ctx* ctx;
        const svr_scene* scene;
        const svr_camera* cam;
        const svr_render_options* opts;
        svr_frame* f;
    } arg{ctx, scene, cam, opts, f};
    return guarded_call(
        [](void* p) {
            Arg& a = *static_cast<Arg*>(p);
            if (!a.ctx || !a.scene || !a.cam || !a.opts || !a.f)
                throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
            if (a.opts->K < 1 || a.opts->K > 3)
                throw Error(SVR_ERR_INVALID_ARGUMENT, "sample count K out of [1,3]");
            SVR_CUDA(cudaSetDevice(a.ctx->device));
            cudaStream_t st = a.ctx->stream;
            const svr_scene* s = a.scene;
            svr_frame* f = a.f;
            const DevCamera cam = make_dev_camera(*a.cam);
            const uint64_t N = s->n_voxels, npx = uint64_t(cam.W) * cam.H;
            DevBuf vox, cnt, dbc;
            vox.reserve(std::max<uint64_t>(N, 1) * sizeof(OracleVoxel));
            cnt.reserve(16);
            dbc.reserve(24);
            SVR_CUDA(cudaMemsetAsync(cnt.p, 0, 16, st));
            SVR_CUDA(cudaMemcpyAsync(dbc.p, s->bounds_center, 24, cudaMemcpyHostToDevice, st));
            if (N)
                oracle_prep_kernel<<<unsigned((N + 127) / 128), 128, 0, st>>>(
                    cam, N, s->paths.as<uint64_t>(), s->corner_index.as<uint32_t>(),
                    s->density.as<float>(), s->sh.as<float>(), s->sh_degree, s->sh_stride,
                    dbc.as<double>(), s->bounds_size, a.opts->near_plane, vox.as<OracleVoxel>(),
                    cnt.as<unsigned int>());
            f->ctx = a.ctx;
            f->scene = s;
            f->opts = *a.opts;
            f->opts.training = 0;
            f->cam = cam;
            f->ss_cam = *a.cam;
            f->W = f->sw = cam.W;
            f->H = f->sh = cam.H;
            f->ntx = cam.ntx;
            f->nty = cam.nty;
            f->n_voxels = N;
            f->n_entries = 0;
            f->has_records = false;
            f->training = false;
            f->n_visible = ~uint64_t(0);
            f->alloc_outputs(npx);
            f->rects.reserve(std::max<uint64_t>(N, 1) * 16);
            dim3 grid(unsigned((cam.W + 63) / 64), unsigned(cam.H));
            oracle_render_kernel<<<grid, 64, 0, st>>>(
                cam, vox.as<OracleVoxel>(), cnt.as<unsigned int>(), a.opts->K, a.opts->t_threshold,
                a.opts->background[0], a.opts->background[1], a.opts->background[2],
                a.opts->far_sentinel, f->out_color, f->out_depth,
                f->out_median, f->out_normal, f->out_tfin);
            SVR_LAUNCH("oracle_render_kernel");
            SVR_CUDA(cudaStreamSynchronize(st));
        },
        &arg);
}
