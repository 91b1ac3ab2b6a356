/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference rasterizer (double precision,
 * single thread), following /root/reference/proj/src/raster.cpp and the
 * headers it inlines. Compiled with -ffp-contract=off (oracle/Makefile) so
 * the fp64 projection and tile-pattern arithmetic round exactly like the
 * reference's x86-64 -O2 build. Only tests/, smoke() and bench.py's CPU
 * leg may load it.
 */
#include "svr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16
#define MAX_LEVEL 16
#define GROUP_ONES 0x249249249249ull
#define AABB_PAD 1e-6
#define KNEE 1.1

typedef struct { double x, y, z; } v3;

static v3 V3(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 add(v3 a, v3 b) { return V3(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return V3(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scale(v3 a, double s) { return V3(a.x * s, a.y * s, a.z * s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static double norm3(v3 a) { return sqrt(dot(a, a)); }
static v3 normalized(v3 a) {  /* geom.hpp:57-60 */
    double n = norm3(a);
    return n > 0.0 ? V3(a.x / n, a.y / n, a.z / n) : V3(0, 0, 0);
}
static double comp(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

/* ------------------------------------------------------------ camera.hpp */
static int tiles_along(int px) { return (px + TILE - 1) / TILE; }

static svr_camera cam_scaled(const svr_camera* c, int nw, int nh) {  /* camera.hpp:38-48 */
    svr_camera s = *c;
    double rx = (double)nw / c->width, ry = (double)nh / c->height;
    s.width = nw; s.height = nh;
    s.fx = c->fx * rx; s.cx = c->cx * rx;
    s.fy = c->fy * ry; s.cy = c->cy * ry;
    return s;
}

static v3 mat_vec(const double* m, v3 v) {  /* geom.hpp:73-76 */
    return V3(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
              m[6] * v.x + m[7] * v.y + m[8] * v.z);
}

static v3 pixel_dir(const svr_camera* c, double px, double py) {  /* camera.hpp:24-27 */
    v3 d = V3((px + 0.5 - c->cx) / c->fx, (py + 0.5 - c->cy) / c->fy, 1.0);
    return mat_vec(c->rot, d);
}

static v3 world_to_cam(const svr_camera* c, v3 p) {  /* camera.hpp:29 */
    double t[9] = {c->rot[0], c->rot[3], c->rot[6], c->rot[1], c->rot[4],
                   c->rot[7], c->rot[2], c->rot[5], c->rot[8]};
    return mat_vec(t, sub(p, V3(c->pos[0], c->pos[1], c->pos[2])));
}

static uint32_t sign_bits(v3 d) {  /* octree.hpp:93-95 */
    return 4u * (d.x < 0.0) + 2u * (d.y < 0.0) + 1u * (d.z < 0.0);
}

/* ------------------------------------------------------------ octree.hpp */
static void geometry(const svr_scene_desc* s, uint64_t vi, v3* center, double* size) {
    int level = s->levels[vi];
    uint64_t code = s->codes[vi] >> (3 * (MAX_LEVEL - level));
    uint32_t i = 0, j = 0, k = 0;
    for (int n = 0; n < level; ++n) {  /* octree.hpp:68-82 */
        i |= (uint32_t)((code & 4) >> 2) << n;
        j |= (uint32_t)((code & 2) >> 1) << n;
        k |= (uint32_t)(code & 1) << n;
        code >>= 3;
    }
    double sz = ldexp(s->bounds_size, -level);  /* octree.hpp:85-90 */
    v3 lo = sub(V3(s->bounds_center[0], s->bounds_center[1], s->bounds_center[2]),
                V3(0.5 * s->bounds_size, 0.5 * s->bounds_size, 0.5 * s->bounds_size));
    *center = add(lo, V3(sz * (i + 0.5), sz * (j + 0.5), sz * (k + 0.5)));
    *size = sz;
}

/* ------------------------------------------------------------ field.hpp / sh.hpp */
static double explin(double x) { return x > KNEE ? x : exp(x / KNEE - 1.0 + log(KNEE)); }
static double explin_deriv(double x) { return x > KNEE ? 1.0 : explin(x) / KNEE; }

static void tri_weights(v3 q, double* w) {
    double wx[2] = {1.0 - q.x, q.x}, wy[2] = {1.0 - q.y, q.y}, wz[2] = {1.0 - q.z, q.z};
    for (int c = 0; c < 8; ++c) w[c] = wx[(c >> 2) & 1] * wy[(c >> 1) & 1] * wz[c & 1];
}

static double trilinear(const double* V, v3 q) {
    double w[8], s = 0.0;
    tri_weights(q, w);
    for (int c = 0; c < 8; ++c) s += w[c] * V[c];
    return s;
}

static int ray_aabb(v3 center, double size, v3 o, v3 d, double* pa, double* pb) {
    double a = -INFINITY, b = INFINITY;
    for (int ax = 0; ax < 3; ++ax) {  /* field.hpp:58-69, std::min/max semantics */
        double lo = comp(center, ax) - 0.5 * size, hi = comp(center, ax) + 0.5 * size;
        double c0 = (lo - comp(o, ax)) / comp(d, ax);
        double c1 = (hi - comp(o, ax)) / comp(d, ax);
        double mn = (c1 < c0) ? c1 : c0, mx = (c0 < c1) ? c1 : c0;
        a = (a < mn) ? mn : a;
        b = (mx < b) ? mx : b;
    }
    *pa = a; *pb = b;
    return (a <= b) && (a > 0.0);
}

typedef struct { int K; double l, alpha; v3 q[8]; double v[8], t[8], sa[8]; } acache;

static double voxel_alpha(const double* V, v3 center, double size, double a, double b, v3 o,
                          v3 d, int K, acache* c) {  /* field.hpp:92-116 */
    double l = (b - a) * norm3(d), sum = 0.0;
    c->K = K; c->l = l;
    v3 lo = sub(center, V3(0.5 * size, 0.5 * size, 0.5 * size));
    for (int k = 0; k < K; ++k) {
        double t = a + (k + 0.5) / K * (b - a);
        v3 q = V3((o.x + t * d.x - lo.x) / size, (o.y + t * d.y - lo.y) / size,
               (o.z + t * d.z - lo.z) / size);
        double v = trilinear(V, q), act = explin(v);
        sum += act;
        c->q[k] = q; c->v[k] = v; c->t[k] = t;
        c->sa[k] = 1.0 - exp(-(l / K) * act);
    }
    c->alpha = 1.0 - exp(-(l / K) * sum);
    return c->alpha;
}

static double voxel_depth(const acache* c) {  /* field.hpp:173-181 */
    double d = 0.0, T = 1.0;
    for (int k = 0; k < c->K; ++k) { d += T * c->sa[k] * c->t[k]; T *= 1.0 - c->sa[k]; }
    return d;
}

static void voxel_depth_backward(const acache* c, double* dd) {  /* field.hpp:184-201 */
    double a1 = c->sa[0], a2 = c->sa[1], a3 = c->sa[2], t1 = c->t[0], t2 = c->t[1], t3 = c->t[2];
    if (c->K == 1) { dd[0] = t1; dd[1] = dd[2] = 0; }
    else if (c->K == 2) { dd[0] = t1 - a2 * t2; dd[1] = t2 - a1 * t2; dd[2] = 0; }
    else {
        dd[0] = t1 + a2 * a3 * t3 - a2 * t2 - a3 * t3;
        dd[1] = t2 + a1 * a3 * t3 - a1 * t2 - a3 * t3;
        dd[2] = t3 + a1 * a2 * t3 - a1 * t3 - a2 * t3;
    }
}

static v3 density_gradient(const double* V) {  /* field.hpp:132-141 */
    v3 g = V3(0, 0, 0);
    for (int c = 0; c < 8; ++c) {
        v3 s = V3(((c >> 2) & 1) ? 1.0 : -1.0, ((c >> 1) & 1) ? 1.0 : -1.0, (c & 1) ? 1.0 : -1.0);
        g = add(g, scale(s, 0.25 * V[c]));
    }
    return g;
}

static int sh_basis(int deg, v3 d, double* b) {  /* sh.hpp:18-45 */
    memset(b, 0, 16 * sizeof(double));
    b[0] = 0.28209479177387814;
    if (deg < 1) return 1;
    double x = d.x, y = d.y, z = d.z, C1 = 0.4886025119029199;
    b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    if (deg < 2) return 4;
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = 1.0925484305920792 * xy; b[5] = -1.0925484305920792 * yz;
    b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy); b[7] = -1.0925484305920792 * xz;
    b[8] = 0.5462742152960396 * (xx - yy);
    if (deg < 3) return 9;
    b[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    b[10] = 2.890611442640554 * xy * z;
    b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    b[14] = 1.445305721320277 * z * (xx - yy);
    b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
    return 16;
}

/* ------------------------------------------------------------ raster.cpp */
typedef struct {
    uint32_t vid;
    v3 center, color, n, raw;
    double size, V[8];
    int degenerate;
    double x0, x1, y0, y1;
    int tx0, tx1, ty0, ty1;
} pre_t;

static int to_int_x86(double f) {  /* cvttsd2si: INT_MIN outside the int32 range */
    return (f > -2147483649.0 && f < 2147483648.0) ? (int)f : (int)0x80000000u;
}
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static int project(const svr_camera* cam, v3 center, double size, double near, pre_t* o) {
    o->tx0 = 0; o->tx1 = -1; o->ty0 = 0; o->ty1 = -1;  /* raster.cpp:72-118 */
    int front = 0, behind = 0;
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (int c = 0; c < 8; ++c) {
        double h = 0.5 * size;
        v3 corner = add(center, V3(((c >> 2) & 1) ? h : -h, ((c >> 1) & 1) ? h : -h, (c & 1) ? h : -h));
        v3 pc = world_to_cam(cam, corner);
        if (pc.z <= near) { behind = 1; continue; }
        front = 1;
        double u = cam->fx * pc.x / pc.z + cam->cx, v = cam->fy * pc.y / pc.z + cam->cy;
        x0 = (u < x0) ? u : x0; x1 = (x1 < u) ? u : x1;
        y0 = (v < y0) ? v : y0; y1 = (y1 < v) ? v : y1;
    }
    if (!front) return 0;
    if (behind) { x0 = 0; x1 = cam->width; y0 = 0; y1 = cam->height; }
    x0 -= AABB_PAD; x1 += AABB_PAD; y0 -= AABB_PAD; y1 += AABB_PAD;
    if (x1 < 0 || y1 < 0 || x0 > cam->width || y0 > cam->height) return 0;
    o->x0 = x0; o->x1 = x1; o->y0 = y0; o->y1 = y1;
    int ntx = tiles_along(cam->width), nty = tiles_along(cam->height);
    o->tx0 = clampi(to_int_x86(floor(x0 / TILE)), 0, ntx - 1);
    o->tx1 = clampi(to_int_x86(floor(x1 / TILE)), 0, ntx - 1);
    o->ty0 = clampi(to_int_x86(floor(y0 / TILE)), 0, nty - 1);
    o->ty1 = clampi(to_int_x86(floor(y1 / TILE)), 0, nty - 1);
    return 1;
}

static uint32_t tile_mask(const svr_camera* cam, int tx, int ty) {  /* raster.cpp:120-142 */
    int px0 = tx * TILE, py0 = ty * TILE;
    int px1 = px0 + TILE - 1 < cam->width - 1 ? px0 + TILE - 1 : cam->width - 1;
    int py1 = py0 + TILE - 1 < cam->height - 1 ? py0 + TILE - 1 : cam->height - 1;
    int neg[3] = {0, 0, 0}, nonneg[3] = {0, 0, 0};
    int ys[2] = {py0, py1}, xs[2] = {px0, px1};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            v3 d = pixel_dir(cam, xs[b], ys[a]);
            for (int ax = 0; ax < 3; ++ax) {
                if (comp(d, ax) < 0.0) neg[ax] = 1; else nonneg[ax] = 1;
            }
        }
    uint32_t m = 0;
    for (uint32_t s = 0; s < 8; ++s) {
        int ok = 1;
        for (int ax = 0; ax < 3; ++ax) {
            int want = (s >> (2 - ax)) & 1;
            if (want ? !neg[ax] : !nonneg[ax]) ok = 0;
        }
        if (ok) m |= 1u << s;
    }
    return m;
}

static pre_t* preprocess(const svr_scene_desc* s, const svr_camera* cam, double near, size_t* n) {
    pre_t* pre = (pre_t*)malloc((s->n_voxels + 1) * sizeof(pre_t));  /* raster.cpp:182-201 */
    int stride = 3 * (s->sh_degree + 1) * (s->sh_degree + 1);
    size_t k = 0;
    v3 pos = V3(cam->pos[0], cam->pos[1], cam->pos[2]);
    for (uint64_t vi = 0; vi < s->n_voxels; ++vi) {
        pre_t p;
        memset(&p, 0, sizeof p);
        p.vid = (uint32_t)vi;
        geometry(s, vi, &p.center, &p.size);
        if (!project(cam, p.center, p.size, near, &p)) continue;
        for (int c = 0; c < 8; ++c) p.V[c] = s->density[s->corner_index[8 * vi + c]];
        double b[16];
        int nb = sh_basis(s->sh_degree, normalized(sub(p.center, pos)), b);
        const float* co = s->sh + vi * stride;
        v3 col = V3(0, 0, 0);
        for (int m = 0; m < nb; ++m) {
            col.x += b[m] * co[3 * m]; col.y += b[m] * co[3 * m + 1]; col.z += b[m] * co[3 * m + 2];
        }
        p.color = V3(col.x > 0 ? col.x : 0, col.y > 0 ? col.y : 0, col.z > 0 ? col.z : 0);
        p.raw = density_gradient(p.V);
        double len = norm3(p.raw);
        p.degenerate = len == 0.0;
        p.n = p.degenerate ? V3(0, 0, 0) : V3(p.raw.x / len, p.raw.y / len, p.raw.z / len);
        pre[k++] = p;
    }
    *n = k;
    return pre;
}

typedef struct { uint64_t key; uint32_t value; } entry_t;

static int cmp_entry(const void* a, const void* b) {  /* raster.cpp:174-178 */
    const entry_t *x = (const entry_t*)a, *y = (const entry_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->value < y->value ? -1 : (x->value > y->value);
}

static entry_t* build_entries(const svr_scene_desc* s, const pre_t* pre, size_t npre,
                              const svr_camera* cam, size_t* n) {
    int ntx = tiles_along(cam->width), nty = tiles_along(cam->height);  /* raster.cpp:144-172 */
    uint8_t* masks = (uint8_t*)malloc((size_t)ntx * nty + 1);
    for (int t = 0; t < ntx * nty; ++t) masks[t] = (uint8_t)tile_mask(cam, t % ntx, t / ntx);
    size_t cnt = 0;
    for (size_t i = 0; i < npre; ++i)
        for (int ty = pre[i].ty0; ty <= pre[i].ty1; ++ty)
            for (int tx = pre[i].tx0; tx <= pre[i].tx1; ++tx)
                cnt += __builtin_popcount(masks[(size_t)ty * ntx + tx]);
    entry_t* e = (entry_t*)malloc((cnt + 1) * sizeof(entry_t));
    size_t k = 0;
    for (size_t i = 0; i < npre; ++i) {
        uint64_t code = s->codes[pre[i].vid];
        for (int ty = pre[i].ty0; ty <= pre[i].ty1; ++ty)
            for (int tx = pre[i].tx0; tx <= pre[i].tx1; ++tx) {
                uint64_t tid = (uint64_t)ty * ntx + tx;
                for (uint32_t sb = 0; sb < 8; ++sb)
                    if (masks[tid] >> sb & 1) {
                        e[k].key = (tid << 48) | (code ^ ((uint64_t)sb * GROUP_ONES));
                        e[k].value = (sb << 29) | pre[i].vid;
                        ++k;
                    }
            }
    }
    free(masks);
    *n = cnt;
    return e;
}

/* AreaResampler (image.cpp:9-60) */
typedef struct { int src, dst; int* ptr; int* idx; double* w; } taps_t;

static taps_t axis_taps(int src, int dst) {
    taps_t t;
    t.src = src; t.dst = dst;
    double scl = (double)src / dst;
    t.ptr = (int*)calloc(dst + 1, sizeof(int));
    t.idx = (int*)malloc(((size_t)src + 2 * dst + 2) * sizeof(int));
    t.w = (double*)malloc(((size_t)src + 2 * dst + 2) * sizeof(double));
    int k = 0;
    for (int d = 0; d < dst; ++d) {
        double lo = d * scl, hi = (d + 1) * scl;
        int s0 = (int)lo, s1 = (int)ceil(hi) - 1;
        if (s1 > src - 1) s1 = src - 1;
        for (int s = s0; s <= s1; ++s) {
            double a = hi < (double)(s + 1) ? hi : (double)(s + 1);
            double b = lo > (double)s ? lo : (double)s;
            if (a - b > 0) { t.idx[k] = s; t.w[k] = (a - b) / scl; ++k; }
        }
        t.ptr[d + 1] = k;
    }
    return t;
}
static void free_taps(taps_t* t) { free(t->ptr); free(t->idx); free(t->w); }

static void downsample(const double* src, int sw, int sh, int ch, double* dst, int W, int H) {
    taps_t tx = axis_taps(sw, W), ty = axis_taps(sh, H);
    double* mid = (double*)calloc((size_t)W * sh * ch, sizeof(double));
    for (int y = 0; y < sh; ++y)
        for (int x = 0; x < W; ++x)
            for (int t = tx.ptr[x]; t < tx.ptr[x + 1]; ++t)
                for (int c = 0; c < ch; ++c)
                    mid[((size_t)y * W + x) * ch + c] += tx.w[t] * src[((size_t)y * sw + tx.idx[t]) * ch + c];
    memset(dst, 0, (size_t)W * H * ch * sizeof(double));
    for (int y = 0; y < H; ++y)
        for (int t = ty.ptr[y]; t < ty.ptr[y + 1]; ++t)
            for (int x = 0; x < W; ++x)
                for (int c = 0; c < ch; ++c)
                    dst[((size_t)y * W + x) * ch + c] += ty.w[t] * mid[((size_t)ty.idx[t] * W + x) * ch + c];
    free(mid); free_taps(&tx); free_taps(&ty);
}

static void adjoint(const double* g, int W, int H, int ch, double* src, int sw, int sh) {
    taps_t tx = axis_taps(sw, W), ty = axis_taps(sh, H);
    double* mid = (double*)calloc((size_t)W * sh * ch, sizeof(double));
    for (int y = 0; y < H; ++y)
        for (int t = ty.ptr[y]; t < ty.ptr[y + 1]; ++t)
            for (int x = 0; x < W; ++x)
                for (int c = 0; c < ch; ++c)
                    mid[((size_t)ty.idx[t] * W + x) * ch + c] += ty.w[t] * g[((size_t)y * W + x) * ch + c];
    memset(src, 0, (size_t)sw * sh * ch * sizeof(double));
    for (int y = 0; y < sh; ++y)
        for (int x = 0; x < W; ++x)
            for (int t = tx.ptr[x]; t < tx.ptr[x + 1]; ++t)
                for (int c = 0; c < ch; ++c)
                    src[((size_t)y * sw + tx.idx[t]) * ch + c] += tx.w[t] * mid[((size_t)y * W + x) * ch + c];
    free(mid); free_taps(&tx); free_taps(&ty);
}

typedef struct { uint32_t pre; double a, b; } contrib_t;

typedef struct {
    svr_camera ss;
    int sw, sh;
    pre_t* pre;
    size_t npre;
    contrib_t* contribs;
    size_t ncontribs, cap;
    uint32_t *pix_begin, *pix_count;
    double *ss_color, *ss_depth, *ss_median, *ss_normal, *ss_tfin;
} fwd_t;

static void push_contrib(fwd_t* f, uint32_t p, double a, double b) {
    if (f->ncontribs == f->cap) {
        f->cap = f->cap ? 2 * f->cap : 1024;
        f->contribs = (contrib_t*)realloc(f->contribs, f->cap * sizeof(contrib_t));
    }
    f->contribs[f->ncontribs].pre = p; f->contribs[f->ncontribs].a = a; f->contribs[f->ncontribs].b = b;
    f->ncontribs++;
}

static void free_fwd(fwd_t* f) {
    free(f->pre); free(f->contribs); free(f->pix_begin); free(f->pix_count);
    free(f->ss_color); free(f->ss_depth); free(f->ss_median); free(f->ss_normal); free(f->ss_tfin);
}

static int validate(const svr_render_options* o) {  /* raster.cpp:207-211 */
    if (o->supersample < 1.0) return SVR_ERR_INVALID_ARGUMENT;
    if (o->K < 1 || o->K > 3) return SVR_ERR_INVALID_ARGUMENT;
    if (o->t_threshold <= 0.0 || o->t_threshold >= 1.0) return SVR_ERR_INVALID_ARGUMENT;
    return SVR_OK;
}

/* render_with_pools at ss resolution (raster.cpp:205-282). */
static int forward(const svr_scene_desc* s, const svr_camera* cam, const svr_render_options* o,
                   int training, double* max_blend, fwd_t* f) {
    int st = validate(o);
    if (st) return st;
    memset(f, 0, sizeof *f);
    f->sw = (int)ceil(o->supersample * cam->width);
    f->sh = (int)ceil(o->supersample * cam->height);
    f->ss = cam_scaled(cam, f->sw, f->sh);
    int ntx = tiles_along(f->sw), nty = tiles_along(f->sh);
    if (s->n_voxels >= (1ull << 29) || (uint64_t)ntx * nty >= (1ull << 16)) return SVR_ERR_LENGTH;
    f->pre = preprocess(s, &f->ss, o->near_plane, &f->npre);
    size_t ne;
    entry_t* e = build_entries(s, f->pre, f->npre, &f->ss, &ne);
    qsort(e, ne, sizeof(entry_t), cmp_entry);
    uint32_t* pre_of = (uint32_t*)malloc((s->n_voxels + 1) * sizeof(uint32_t));
    for (size_t i = 0; i < f->npre; ++i) pre_of[f->pre[i].vid] = (uint32_t)i;
    size_t np = (size_t)f->sw * f->sh;
    f->ss_color = (double*)calloc(np * 3, sizeof(double));
    f->ss_depth = (double*)calloc(np, sizeof(double));
    f->ss_median = (double*)calloc(np, sizeof(double));
    f->ss_normal = (double*)calloc(np * 3, sizeof(double));
    f->ss_tfin = (double*)calloc(np, sizeof(double));
    f->pix_begin = (uint32_t*)calloc(np, sizeof(uint32_t));
    f->pix_count = (uint32_t*)calloc(np, sizeof(uint32_t));
    if (max_blend) memset(max_blend, 0, s->n_voxels * sizeof(double));
    v3 bg = V3(o->background[0], o->background[1], o->background[2]);
    v3 orig = V3(f->ss.pos[0], f->ss.pos[1], f->ss.pos[2]);
    size_t cursor = 0;
    for (int ty = 0; ty < nty; ++ty)
        for (int tx = 0; tx < ntx; ++tx) {
            uint64_t tid = (uint64_t)ty * ntx + tx;
            size_t lo = cursor;
            while (cursor < ne && (e[cursor].key >> 48) == tid) ++cursor;
            size_t hi = cursor;
            int px1 = (tx + 1) * TILE < f->sw ? (tx + 1) * TILE : f->sw;
            int py1 = (ty + 1) * TILE < f->sh ? (ty + 1) * TILE : f->sh;
            for (int py = ty * TILE; py < py1; ++py)
                for (int px = tx * TILE; px < px1; ++px) {
                    v3 d = pixel_dir(&f->ss, px, py);
                    uint32_t sb = sign_bits(d);
                    size_t pix = (size_t)py * f->sw + px;
                    f->pix_begin[pix] = (uint32_t)f->ncontribs;
                    double T = 1.0, depth = 0.0, median = -1.0;
                    v3 col = V3(0, 0, 0), nrm = V3(0, 0, 0);
                    int count = 0;
                    double cx = px + 0.5, cy = py + 0.5;
                    for (size_t k = lo; k < hi; ++k) {  /* CompositeCtx::add, raster.cpp:30-54 */
                        if ((e[k].value >> 29) != sb) continue;
                        uint32_t pi = pre_of[e[k].value & ((1u << 29) - 1)];
                        const pre_t* pv = &f->pre[pi];
                        if (cx < pv->x0 || cx > pv->x1 || cy < pv->y0 || cy > pv->y1) continue;
                        double a, b;
                        if (!ray_aabb(pv->center, pv->size, orig, d, &a, &b)) continue;
                        acache c;
                        double alpha = voxel_alpha(pv->V, pv->center, pv->size, a, b, orig, d, o->K, &c);
                        double dv = voxel_depth(&c);
                        col = add(col, scale(pv->color, T * alpha));
                        nrm = add(nrm, scale(pv->n, T * alpha));
                        depth += T * dv;
                        if (median < 0.0) {
                            double Tf = T;
                            for (int q = 0; q < o->K; ++q) {
                                Tf *= 1.0 - c.sa[q];
                                if (Tf < 0.5) { median = c.t[q]; break; }
                            }
                        }
                        if (max_blend && T * alpha > max_blend[pv->vid]) max_blend[pv->vid] = T * alpha;
                        if (training) push_contrib(f, pi, a, b);
                        T *= 1.0 - alpha;
                        ++count;
                        if (T < o->t_threshold) break;
                    }
                    col = add(col, scale(bg, T));  /* finish, raster.cpp:56-60 */
                    if (count == 0) depth = o->far_sentinel;
                    if (median < 0.0) median = o->far_sentinel;
                    f->pix_count[pix] = (uint32_t)f->ncontribs - f->pix_begin[pix];
                    f->ss_color[3 * pix] = col.x; f->ss_color[3 * pix + 1] = col.y; f->ss_color[3 * pix + 2] = col.z;
                    f->ss_normal[3 * pix] = nrm.x; f->ss_normal[3 * pix + 1] = nrm.y; f->ss_normal[3 * pix + 2] = nrm.z;
                    f->ss_depth[pix] = depth; f->ss_median[pix] = median; f->ss_tfin[pix] = T;
                }
        }
    free(e); free(pre_of);
    return SVR_OK;
}

int orc_tile_masks(const svr_camera* cam, uint8_t* masks) {
    int ntx = tiles_along(cam->width), nty = tiles_along(cam->height);
    for (int t = 0; t < ntx * nty; ++t) masks[t] = (uint8_t)tile_mask(cam, t % ntx, t / ntx);
    return SVR_OK;
}

int orc_project(const svr_scene_desc* s, const svr_camera* cam, double near, uint8_t* visible,
                double* aabb, int32_t* rect) {
    for (uint64_t vi = 0; vi < s->n_voxels; ++vi) {
        pre_t p;
        memset(&p, 0, sizeof p);
        geometry(s, vi, &p.center, &p.size);
        int ok = project(cam, p.center, p.size, near, &p);
        visible[vi] = (uint8_t)ok;
        aabb[4 * vi] = ok ? p.x0 : 0; aabb[4 * vi + 1] = ok ? p.x1 : 0;
        aabb[4 * vi + 2] = ok ? p.y0 : 0; aabb[4 * vi + 3] = ok ? p.y1 : 0;
        rect[4 * vi] = p.tx0; rect[4 * vi + 1] = p.tx1; rect[4 * vi + 2] = p.ty0; rect[4 * vi + 3] = p.ty1;
    }
    return SVR_OK;
}

int orc_entries(const svr_scene_desc* s, const svr_camera* cam, double near, int sorted,
                uint64_t* n_out, uint64_t* keys, uint32_t* values) {
    int ntx = tiles_along(cam->width), nty = tiles_along(cam->height);
    if (s->n_voxels >= (1ull << 29) || (uint64_t)ntx * nty >= (1ull << 16)) return SVR_ERR_LENGTH;
    size_t npre, ne;
    pre_t* pre = preprocess(s, cam, near, &npre);
    entry_t* e = build_entries(s, pre, npre, cam, &ne);
    if (sorted) qsort(e, ne, sizeof(entry_t), cmp_entry);
    *n_out = ne;
    if (keys)
        for (size_t i = 0; i < ne; ++i) { keys[i] = e[i].key; values[i] = e[i].value; }
    free(pre); free(e);
    return SVR_OK;
}

int orc_render(const svr_scene_desc* s, const svr_camera* cam, const svr_render_options* o,
               double* color, double* depth, double* median, double* normal, double* tfin,
               double* max_blend) {
    fwd_t f;
    int st = forward(s, cam, o, 0, o->record_stats ? max_blend : NULL, &f);
    if (st) return st;
    int W = cam->width, H = cam->height;  /* raster.cpp:283-288 */
    downsample(f.ss_color, f.sw, f.sh, 3, color, W, H);
    downsample(f.ss_depth, f.sw, f.sh, 1, depth, W, H);
    downsample(f.ss_median, f.sw, f.sh, 1, median, W, H);
    downsample(f.ss_normal, f.sw, f.sh, 3, normal, W, H);
    downsample(f.ss_tfin, f.sw, f.sh, 1, tfin, W, H);
    free_fwd(&f);
    return SVR_OK;
}

int orc_backward(const svr_scene_desc* s, const svr_camera* cam, const svr_render_options* o,
                 const double* d_color, const double* d_depth, const double* d_normal,
                 const double* d_tfin_ss, double* g_density, double* g_sh, double* g_priority) {
    fwd_t f;
    int st = forward(s, cam, o, 1, NULL, &f);
    if (st) return st;
    const int sw = f.sw, sh = f.sh, W = cam->width, H = cam->height, K = o->K;
    const int stride = 3 * (s->sh_degree + 1) * (s->sh_degree + 1);
    memset(g_density, 0, s->n_pool * sizeof(double));
    memset(g_sh, 0, s->n_voxels * stride * sizeof(double));
    memset(g_priority, 0, s->n_voxels * sizeof(double));
    size_t np = (size_t)sw * sh;
    double* gC = d_color ? (double*)malloc(np * 3 * sizeof(double)) : NULL;  /* raster.cpp:317-324 */
    double* gD = d_depth ? (double*)malloc(np * sizeof(double)) : NULL;
    double* gN = d_normal ? (double*)malloc(np * 3 * sizeof(double)) : NULL;
    if (gC) adjoint(d_color, W, H, 3, gC, sw, sh);
    if (gD) adjoint(d_depth, W, H, 1, gD, sw, sh);
    if (gN) adjoint(d_normal, W, H, 3, gN, sw, sh);
    v3* gc_pre = (v3*)calloc(f.npre + 1, sizeof(v3));
    v3* gn_pre = (v3*)calloc(f.npre + 1, sizeof(v3));
    size_t cap = 16;
    acache* caches = (acache*)malloc(cap * sizeof(acache));
    double *Ts = (double*)malloc(cap * 8), *ds = (double*)malloc(cap * 8), *phis = (double*)malloc(cap * 8);
    v3 bg = V3(o->background[0], o->background[1], o->background[2]);
    v3 orig = V3(f.ss.pos[0], f.ss.pos[1], f.ss.pos[2]);
    for (int py = 0; py < sh; ++py)
        for (int px = 0; px < sw; ++px) {  /* raster.cpp:340-409 */
            size_t pix = (size_t)py * sw + px;
            uint32_t n = f.pix_count[pix];
            if (!n) continue;
            uint32_t base = f.pix_begin[pix];
            v3 d = pixel_dir(&f.ss, px, py);
            v3 gc = gC ? V3(gC[3 * pix], gC[3 * pix + 1], gC[3 * pix + 2]) : V3(0, 0, 0);
            v3 gn = gN ? V3(gN[3 * pix], gN[3 * pix + 1], gN[3 * pix + 2]) : V3(0, 0, 0);
            double gd = gD ? gD[pix] : 0.0, gt = d_tfin_ss ? d_tfin_ss[pix] : 0.0;
            if (n > cap) {
                cap = 2 * n;
                caches = (acache*)realloc(caches, cap * sizeof(acache));
                Ts = (double*)realloc(Ts, cap * 8); ds = (double*)realloc(ds, cap * 8);
                phis = (double*)realloc(phis, cap * 8);
            }
            double T = 1.0;
            for (uint32_t i = 0; i < n; ++i) {
                const contrib_t* c = &f.contribs[base + i];
                const pre_t* pv = &f.pre[c->pre];
                voxel_alpha(pv->V, pv->center, pv->size, c->a, c->b, orig, d, K, &caches[i]);
                ds[i] = voxel_depth(&caches[i]);
                Ts[i] = T;
                T *= 1.0 - caches[i].alpha;
                phis[i] = dot(gc, pv->color) + dot(gn, pv->n);
            }
            double Ra = dot(gc, bg) + gt, Rd = 0.0;
            for (int i = (int)n - 1; i >= 0; --i) {
                const contrib_t* c = &f.contribs[base + i];
                const pre_t* pv = &f.pre[c->pre];
                const acache* ca = &caches[i];
                double alpha = ca->alpha, A = Ts[i] * (phis[i] - Ra - Rd);
                g_priority[pv->vid] += fabs(alpha * A);
                double dd[3];
                voxel_depth_backward(ca, dd);
                for (int k = 0; k < K; ++k) {
                    double others = 1.0;
                    for (int m = 0; m < K; ++m) if (m != k) others *= 1.0 - ca->sa[m];
                    double dAk = A * others + Ts[i] * gd * dd[k];
                    double dv = dAk * (1.0 - ca->sa[k]) * (ca->l / K) * explin_deriv(ca->v[k]);
                    double w[8];
                    tri_weights(ca->q[k], w);
                    for (int c8 = 0; c8 < 8; ++c8)
                        g_density[s->corner_index[8 * (size_t)pv->vid + c8]] += dv * w[c8];
                }
                double wgt = Ts[i] * alpha;
                gc_pre[c->pre] = add(gc_pre[c->pre], scale(gc, wgt));
                gn_pre[c->pre] = add(gn_pre[c->pre], scale(gn, wgt));
                Ra = alpha * phis[i] + (1.0 - alpha) * Ra;
                Rd = ds[i] * gd + (1.0 - alpha) * Rd;
            }
        }
    for (size_t p = 0; p < f.npre; ++p) {  /* raster.cpp:411-421 */
        const pre_t* pv = &f.pre[p];
        v3 dir = normalized(sub(pv->center, orig));
        double b[16];
        int nb = sh_basis(s->sh_degree, dir, b);
        const float* co = s->sh + (size_t)pv->vid * stride;
        v3 raw = V3(0, 0, 0);
        for (int m = 0; m < nb; ++m) {
            raw.x += b[m] * co[3 * m]; raw.y += b[m] * co[3 * m + 1]; raw.z += b[m] * co[3 * m + 2];
        }
        double gx = raw.x > 0 ? gc_pre[p].x : 0, gy = raw.y > 0 ? gc_pre[p].y : 0,
               gz = raw.z > 0 ? gc_pre[p].z : 0;
        double* out = g_sh + (size_t)pv->vid * stride;
        for (int m = 0; m < nb; ++m) { out[3 * m] += b[m] * gx; out[3 * m + 1] += b[m] * gy; out[3 * m + 2] += b[m] * gz; }
        if (!pv->degenerate) {  /* field.hpp:158-170 */
            double len = norm3(pv->raw);
            v3 dn = gn_pre[p];
            v3 g = V3((dn.x - pv->n.x * dot(dn, pv->n)) / len, (dn.y - pv->n.y * dot(dn, pv->n)) / len,
                   (dn.z - pv->n.z * dot(dn, pv->n)) / len);
            for (int c8 = 0; c8 < 8; ++c8) {
                double si = ((c8 >> 2) & 1) ? 1.0 : -1.0, sj = ((c8 >> 1) & 1) ? 1.0 : -1.0,
                       sk = (c8 & 1) ? 1.0 : -1.0;
                g_density[s->corner_index[8 * (size_t)pv->vid + c8]] += 0.25 * (g.x * si + g.y * sj + g.z * sk);
            }
        }
    }
    free(gC); free(gD); free(gN); free(gc_pre); free(gn_pre);
    free(caches); free(Ts); free(ds); free(phis);
    free_fwd(&f);
    return SVR_OK;
}

/* ------------------------------------------------------------ primitive hooks
 * Exported only so tests/test_oracle_cpu.py can pin the restatement against
 * the known-answer vectors of the reference's unit tests
 * (test_octree.cpp, test_field.cpp, test_sh.cpp, test_camera.cpp,
 * test_image.cpp). */
uint64_t orc_t_octpath(uint32_t i, uint32_t j, uint32_t k, int level) {  /* octree.hpp:51-66 */
    uint64_t code = 0;
    for (int n = 0; n < level; ++n) {
        uint64_t bits = 4 * (i & 1) + 2 * (j & 1) + (k & 1);
        code |= bits << (3 * n);
        i >>= 1; j >>= 1; k >>= 1;
    }
    return code << (3 * (MAX_LEVEL - level));
}
uint32_t orc_t_sign_bits(double x, double y, double z) { return sign_bits(V3(x, y, z)); }
uint64_t orc_t_dir_dep_order(uint64_t code, uint32_t s) { return code ^ ((uint64_t)s * GROUP_ONES); }
double orc_t_explin(double x) { return explin(x); }
double orc_t_explin_deriv(double x) { return explin_deriv(x); }
int orc_t_ray_aabb(const double* c, double size, const double* o, const double* d, double* ab) {
    return ray_aabb(V3(c[0], c[1], c[2]), size, V3(o[0], o[1], o[2]), V3(d[0], d[1], d[2]), &ab[0], &ab[1]);
}
double orc_t_voxel_alpha(const double* V, const double* c, double size, const double* o,
                         const double* d, int K) {
    double a, b;
    ray_aabb(V3(c[0], c[1], c[2]), size, V3(o[0], o[1], o[2]), V3(d[0], d[1], d[2]), &a, &b);
    acache ca;
    return voxel_alpha(V, V3(c[0], c[1], c[2]), size, a, b, V3(o[0], o[1], o[2]), V3(d[0], d[1], d[2]), K, &ca);
}
double orc_t_voxel_depth(const double* sa, const double* t, int K) {
    acache c;
    memset(&c, 0, sizeof c);
    c.K = K;
    for (int k = 0; k < K; ++k) { c.sa[k] = sa[k]; c.t[k] = t[k]; }
    return voxel_depth(&c);
}
void orc_t_sh_basis(int deg, double x, double y, double z, double* b) { sh_basis(deg, V3(x, y, z), b); }
void orc_t_pixel_ray(const svr_camera* cam, double px, double py, double* d) {
    v3 r = pixel_dir(cam, px, py);
    d[0] = r.x; d[1] = r.y; d[2] = r.z;
}
void orc_t_downsample(const double* src, int sw, int sh, int ch, double* dst, int W, int H) {
    downsample(src, sw, sh, ch, dst, W, H);
}
void orc_t_adjoint(const double* g, int W, int H, int ch, double* src, int sw, int sh) {
    adjoint(g, W, H, ch, src, sw, sh);
}
