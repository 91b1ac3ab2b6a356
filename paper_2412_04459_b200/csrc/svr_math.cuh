// svr_math.cuh — per-voxel math shared by the sm_100a kernels.
//
// Two precision regimes, as the parity contract demands (SURVEY §7 hard
// part 1, §8(a)):
//   * fp64, bit-exact with the reference's double arithmetic: voxel geometry
//     (octree.hpp:68-90), corner projection + padded AABB + tile rect
//     (raster.cpp:72-118), per-pixel ray direction and sign bits
//     (camera.hpp:24-27, octree.hpp:93-95), tile sign patterns
//     (raster.cpp:120-142). Every operation goes through an explicitly
//     rounded intrinsic (__dadd_rn, __dmul_rn, ...) in the same evaluation
//     order the reference's C++ uses, so no FMA contraction can occur
//     regardless of compiler flags. The host copy (used only by the C++
//     drop-in's camera scaling) compiles the same expressions with
//     -ffp-contract=off.
//   * fp32, tolerance-checked: ray/box slab test, K-point alpha quadrature,
//     depth, SH colour, normals (field.hpp:23-201, sh.hpp:18-83).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define SVR_HD __host__ __device__ __forceinline__
#else
#define SVR_HD inline
#endif

namespace svrb {

constexpr int kTile = 16;
constexpr int kMaxLevel = 16;
constexpr uint64_t kGroupOnes = 0x249249249249ull;  // octree.hpp:19
constexpr double kAabbPad = 1e-6;                     // raster.cpp:11
constexpr float kExplinKnee = 1.1f;                   // field.hpp:19

// Programmatic dependent launch (sm_90+): a frame's kernels are launched
// with programmatic stream serialisation, so the next kernel's CTAs are
// scheduled while the current one drains; every such kernel first waits for
// its predecessor's completion (griddepcontrol.wait) and lets its own
// dependents launch (griddepcontrol.launch_dependents). Both are no-ops for
// a kernel launched without the attribute.
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#else
inline void pdl_enter() {}
#endif

// Live entry count of a deferred-E frame (capacity `cap`, device count
// `*n_dev`). A frame that outgrew its capacity emitted only a prefix of its
// entries (the rest of the buffer holds stale keys of earlier frames), so it
// sorts and composites nothing; the host re-renders it when it is consumed.
SVR_HD uint64_t live_entries(uint64_t cap, const unsigned long long* n_dev) {
    if (!n_dev) return cap;
    const uint64_t d = uint64_t(*n_dev);
    return d > cap ? 0 : d;
}

// ---------------------------------------------------------------- fp64 exact
#if defined(__CUDA_ARCH__)
SVR_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
SVR_HD double dsub(double a, double b) { return __dsub_rn(a, b); }
SVR_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
SVR_HD double ddiv(double a, double b) { return __ddiv_rn(a, b); }
#else
SVR_HD double dadd(double a, double b) { return a + b; }
SVR_HD double dsub(double a, double b) { return a - b; }
SVR_HD double dmul(double a, double b) { return a * b; }
SVR_HD double ddiv(double a, double b) { return a / b; }
#endif

// Camera as the kernels see it (svr::Camera, camera.hpp:13-49).
struct DevCamera {
    int W, H, ntx, nty;
    double fx, fy, cx, cy;
    double rot[9];  // camera-to-world, row-major
    double pos[3];
};

// Mat3 * Vec3 in geom.hpp:73-76 order: (m0*x + m1*y) + m2*z per row.
SVR_HD void mat_vec(const double* m, double x, double y, double z, double* o) {
    o[0] = dadd(dadd(dmul(m[0], x), dmul(m[1], y)), dmul(m[2], z));
    o[1] = dadd(dadd(dmul(m[3], x), dmul(m[4], y)), dmul(m[5], z));
    o[2] = dadd(dadd(dmul(m[6], x), dmul(m[7], y)), dmul(m[8], z));
}

// rot.transposed() * v (camera.hpp:29): row r of the transpose = column r.
SVR_HD void mat_t_vec(const double* m, double x, double y, double z, double* o) {
    o[0] = dadd(dadd(dmul(m[0], x), dmul(m[3], y)), dmul(m[6], z));
    o[1] = dadd(dadd(dmul(m[1], x), dmul(m[4], y)), dmul(m[7], z));
    o[2] = dadd(dadd(dmul(m[2], x), dmul(m[5], y)), dmul(m[8], z));
}

// Camera::pixel_ray direction (camera.hpp:24-27), unnormalised.
SVR_HD void pixel_ray_dir(const DevCamera& c, double px, double py, double* d) {
    double cxd = ddiv(dsub(dadd(px, 0.5), c.cx), c.fx);
    double cyd = ddiv(dsub(dadd(py, 0.5), c.cy), c.fy);
    mat_vec(c.rot, cxd, cyd, 1.0, d);
}

// Side planes of the view frustum through an 8x4 pixel block whose first
// pixel is (wx0, wy0), widened by one pixel on every side: camera-frame
// half-spaces x/z >= a, x/z <= b, y/z >= c, y/z <= d with inward normals
// (1,0,-a), (-1,0,b), (0,1,-c), (0,-1,d), rotated to world (n_w = rot n_c).
SVR_HD void warp_cone_planes(const DevCamera& cam, int wx0, int wy0, float (*cone)[3]) {
    const double a_ = (double(wx0) - 0.5 - cam.cx) / cam.fx, b_ = (double(wx0) + 8.5 - cam.cx) / cam.fx;
    const double c_ = (double(wy0) - 0.5 - cam.cy) / cam.fy, d_ = (double(wy0) + 4.5 - cam.cy) / cam.fy;
    const double nc[4][3] = {{1.0, 0.0, -a_}, {-1.0, 0.0, b_}, {0.0, 1.0, -c_}, {0.0, -1.0, d_}};
    for (int q = 0; q < 4; ++q)
        for (int r = 0; r < 3; ++r)
            cone[q][r] = float(cam.rot[3 * r + 0] * nc[q][0] + cam.rot[3 * r + 1] * nc[q][1] +
                               cam.rot[3 * r + 2] * nc[q][2]);
}

// False iff the camera-relative box [lo.xyz, lo.xyz + lo.w] lies strictly
// outside one of the planes: then no pixel ray of the block can hit it and
// the per-pixel slab test would reject it, so skipping it changes nothing.
// The one-pixel widening dwarfs the fp32 rounding of this test.
SVR_HD bool box_in_cone(const float (*cone)[3], float4 lo) {
    const float eps = 1e-5f * (fabsf(lo.x) + fabsf(lo.y) + fabsf(lo.z) + lo.w);
    bool in = true;
    for (int q = 0; q < 4; ++q) {
        const float vmax = cone[q][0] * lo.x + cone[q][1] * lo.y + cone[q][2] * lo.z +
                           lo.w * (fmaxf(cone[q][0], 0.f) + fmaxf(cone[q][1], 0.f) +
                                   fmaxf(cone[q][2], 0.f));
        if (vmax < -eps) in = false;
    }
    return in;
}

// Frustum culling pays only for entries whose screen AABB is loose.
constexpr float kConeMinArea = 64.0f * 64.0f;  // px^2

// ray_sign_bits (octree.hpp:93-95): bit2 = x<0, bit1 = y<0, bit0 = z<0.
SVR_HD uint32_t sign_bits(const double* d) {
    return 4u * (d[0] < 0.0) + 2u * (d[1] < 0.0) + 1u * (d[2] < 0.0);
}

// int(double) as the reference's x86-64 build executes it (cvttsd2si):
// truncation, and INT_MIN for anything outside the int32 range.
SVR_HD int x86_double_to_int(double f) {
    return (f > -2147483649.0 && f < 2147483648.0) ? int(f) : int(0x80000000u);
}

SVR_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// to_voxel_index (octree.hpp:68-82) + voxel_geometry (octree.hpp:85-90).
// Levels/paths are validated once at upload, so no checks here.
// Every third bit of x (bits 0, 3, ..., 27) packed into bits 0..9.
SVR_HD uint32_t compact_by_3(uint32_t x) {
    x &= 0x09249249u;
    x = (x | (x >> 2)) & 0x030C30C3u;
    x = (x | (x >> 4)) & 0x0300F00Fu;
    x = (x | (x >> 8)) & 0x030000FFu;
    return (x | (x >> 16)) & 0x000003FFu;
}
SVR_HD void voxel_geometry(uint64_t code, int level, const double* bc, double bsize,
                           double* center, double* size) {
    // the path's level digits (i, j, k bits of level n at 3n+2, 3n+1, 3n),
    // de-interleaved with shift-mask steps on two 32-bit halves (10 + 6
    // levels) instead of a loop over the levels
    const uint64_t c = code >> (3 * (kMaxLevel - level));
    const uint32_t lo = uint32_t(c) & 0x3FFFFFFFu, hi = uint32_t(c >> 30);
    const uint32_t i = compact_by_3(lo >> 2) | (compact_by_3(hi >> 2) << 10);
    const uint32_t j = compact_by_3(lo >> 1) | (compact_by_3(hi >> 1) << 10);
    const uint32_t k = compact_by_3(lo) | (compact_by_3(hi) << 10);
    // bsize * 2^-level: a power-of-two scale is exact, as ldexp is
    double s;
#if defined(__CUDA_ARCH__)
    s = dmul(bsize, __longlong_as_double(int64_t(1023 - level) << 52));
#else
    s = ldexp(bsize, -level);
#endif
    double half_root = dmul(0.5, bsize);
    center[0] = dadd(dsub(bc[0], half_root), dmul(s, dadd(double(i), 0.5)));
    center[1] = dadd(dsub(bc[1], half_root), dmul(s, dadd(double(j), 0.5)));
    center[2] = dadd(dsub(bc[2], half_root), dmul(s, dadd(double(k), 0.5)));
    *size = s;
}

struct Projection {
    double x0, x1, y0, y1;
    int tx0, tx1, ty0, ty1;
    bool straddles;  // a corner is at or behind the near plane: AABB = whole image
};

// project_voxel (raster.cpp:72-118), bit-exact. Returns false when culled;
// then tx0=0, tx1=-1, ty0=0, ty1=-1 exactly like a fresh PreVoxel.
SVR_HD bool project_voxel(const DevCamera& cam, const double* center, double size, double near,
                          Projection& out) {
    out.tx0 = 0;
    out.tx1 = -1;
    out.ty0 = 0;
    out.ty1 = -1;
    out.x0 = out.x1 = out.y0 = out.y1 = 0.0;
    out.straddles = false;
    bool any_front = false, any_behind = false;
    const double inf = __builtin_huge_val();
    double x0 = inf, x1 = -inf, y0 = inf, y1 = -inf;
    double h = dmul(0.5, size);
    for (int c = 0; c < 8; ++c) {
        double px = dadd(center[0], ((c >> 2) & 1) ? h : -h);
        double py = dadd(center[1], ((c >> 1) & 1) ? h : -h);
        double pz = dadd(center[2], (c & 1) ? h : -h);
        double pc[3];
        mat_t_vec(cam.rot, dsub(px, cam.pos[0]), dsub(py, cam.pos[1]), dsub(pz, cam.pos[2]), pc);
        if (pc[2] <= near) {
            any_behind = true;
            continue;
        }
        any_front = true;
        double u = dadd(ddiv(dmul(cam.fx, pc[0]), pc[2]), cam.cx);
        double v = dadd(ddiv(dmul(cam.fy, pc[1]), pc[2]), cam.cy);
        x0 = (u < x0) ? u : x0;  // std::min(x0, u)
        x1 = (x1 < u) ? u : x1;  // std::max(x1, u)
        y0 = (v < y0) ? v : y0;
        y1 = (y1 < v) ? v : y1;
    }
    if (!any_front) return false;
    out.straddles = any_behind;
    if (any_behind) {
        x0 = 0;
        x1 = cam.W;
        y0 = 0;
        y1 = cam.H;
    }
    x0 = dsub(x0, kAabbPad);
    x1 = dadd(x1, kAabbPad);
    y0 = dsub(y0, kAabbPad);
    y1 = dadd(y1, kAabbPad);
    if (x1 < 0 || y1 < 0 || x0 > cam.W || y0 > cam.H) return false;
    out.x0 = x0;
    out.x1 = x1;
    out.y0 = y0;
    out.y1 = y1;
    out.tx0 = clampi(x86_double_to_int(floor(ddiv(x0, double(kTile)))), 0, cam.ntx - 1);
    out.tx1 = clampi(x86_double_to_int(floor(ddiv(x1, double(kTile)))), 0, cam.ntx - 1);
    out.ty0 = clampi(x86_double_to_int(floor(ddiv(y0, double(kTile)))), 0, cam.nty - 1);
    out.ty1 = clampi(x86_double_to_int(floor(ddiv(y1, double(kTile)))), 0, cam.nty - 1);
    return true;
}

// Inverse ray-direction component for the fp32 slab tests. ray_aabb
// (field.hpp:58-69) divides in double, where a zero component turns the axis
// into "inside iff lo - o <= 0 < hi - o" (0/0 = NaN falls out of its
// std::min/std::max argument order; either sign of zero). A float 1/0 = inf
// would make lo * inf = NaN and fminf/fmaxf would drop the wrong operand, so
// components that vanish in float get a finite stand-in of 1e30 with the
// double's sign (+ for either zero), which reproduces those cases exactly.
SVR_HD float slab_inv(double d) {
    const float f = float(d);
    if (fabsf(f) >= 1e-30f) return 1.0f / f;
    return d < 0.0 ? -1e30f : 1e30f;
}

// Conservative fp32 pre-test for K1: true only when project_voxel would
// certainly cull the voxel — its bounding sphere (half-diagonal plus a
// rounding margin of 1e-5 of the coordinates' magnitude) lies wholly behind
// the near plane, or wholly in front of it and wholly outside one image side
// widened by a pixel (raster.cpp:104: x1 < 0 || y1 < 0 || x0 > W || y0 > H).
// Anything else takes the exact fp64 path, so the outputs are unchanged.
// The four side-plane normal lengths of surely_culled (per camera).
struct CullNorms {
    float n[4];
};
SVR_HD CullNorms cull_norms(const DevCamera& cam) {
    const float fx = float(cam.fx), fy = float(cam.fy), cx = float(cam.cx), cy = float(cam.cy);
    const float W = float(cam.W), H = float(cam.H);
    auto nrm = [](float a, float b) { return sqrtf(a * a + b * b); };
    return CullNorms{{nrm(fx, cx + 1.f), nrm(-fx, W + 1.f - cx), nrm(fy, cy + 1.f), nrm(-fy, H + 1.f - cy)}};
}
SVR_HD bool surely_culled(const DevCamera& cam, const double* center, double size, double near,
                          const CullNorms& cn) {
    const float c0 = float(center[0] - cam.pos[0]), c1 = float(center[1] - cam.pos[1]),
                c2 = float(center[2] - cam.pos[2]);
    const float px = float(cam.rot[0]) * c0 + float(cam.rot[3]) * c1 + float(cam.rot[6]) * c2;
    const float py = float(cam.rot[1]) * c0 + float(cam.rot[4]) * c1 + float(cam.rot[7]) * c2;
    const float pz = float(cam.rot[2]) * c0 + float(cam.rot[5]) * c1 + float(cam.rot[8]) * c2;
    const float mag = fabsf(c0) + fabsf(c1) + fabsf(c2) + float(size);
    const float r = float(size) * 0.8660255f + 1e-5f * mag;
    const float nr = float(near);
    if (pz + r < nr - 1e-5f * fabsf(nr)) return true;  // every corner behind the near plane
    if (pz - r <= nr + 1e-5f * fabsf(nr)) return false;  // may straddle: whole-image AABB
    // every corner in front: the sphere outside a side plane through the eye
    // (a * q + b * z < 0 over the whole sphere)
    auto outside = [&](float a, float b, float q, float nab) {  // nab = |(a, b)|
        const float d = a * q + b * pz;
        return d + r * nab + 1e-5f * (fabsf(a * q) + fabsf(b * pz)) < 0.f;
    };
    const float fx = float(cam.fx), fy = float(cam.fy), cx = float(cam.cx), cy = float(cam.cy);
    const float W = float(cam.W), H = float(cam.H);
    return outside(fx, cx + 1.f, px, cn.n[0]) ||              // every u < -1
           outside(-fx, W + 1.f - cx, px, cn.n[1]) ||         // every u > W + 1
           outside(fy, cy + 1.f, py, cn.n[2]) ||              // every v < -1
           outside(-fy, H + 1.f - cy, py, cn.n[3]);           // every v > H + 1
}

// True iff no pixel ray of the image can enter the box at t > 0: all eight
// corners lie strictly outside one side plane of the image frustum (planes
// through the camera centre along the image border widened by one pixel;
// a ray point has camera z = t > 0, and the outside of a plane through the
// centre is convex, so the whole box is outside too). Used only to give
// near-plane voxels, whose reference AABB is the whole image
// (raster.cpp:95-101), an empty compositing footprint; their entries are
// still emitted exactly as the reference does.
SVR_HD bool box_outside_image_frustum(const DevCamera& cam, const double* center, double size) {
    const double u0 = (-1.0 - cam.cx) / cam.fx, u1 = (cam.W + 1.0 - cam.cx) / cam.fx;
    const double v0 = (-1.0 - cam.cy) / cam.fy, v1 = (cam.H + 1.0 - cam.cy) / cam.fy;
    const double h = 0.5 * size;
    bool out[4] = {true, true, true, true};
    for (int c = 0; c < 8; ++c) {
        double pc[3];
        mat_t_vec(cam.rot, center[0] + (((c >> 2) & 1) ? h : -h) - cam.pos[0],
                  center[1] + (((c >> 1) & 1) ? h : -h) - cam.pos[1],
                  center[2] + ((c & 1) ? h : -h) - cam.pos[2], pc);
        const double tol = 1e-9 * (fabs(pc[0]) + fabs(pc[1]) + fabs(pc[2]));
        if (pc[0] - u0 * pc[2] >= -tol) out[0] = false;
        if (u1 * pc[2] - pc[0] >= -tol) out[1] = false;
        if (pc[1] - v0 * pc[2] >= -tol) out[2] = false;
        if (v1 * pc[2] - pc[1] >= -tol) out[3] = false;
    }
    return out[0] || out[1] || out[2] || out[3];
}

// tile_sign_patterns (raster.cpp:120-142) as a bitmask over s in [0,8).
SVR_HD uint32_t tile_sign_mask(const DevCamera& cam, int tx, int ty) {
    int px0 = tx * kTile, py0 = ty * kTile;
    int px1 = px0 + kTile - 1 < cam.W - 1 ? px0 + kTile - 1 : cam.W - 1;
    int py1 = py0 + kTile - 1 < cam.H - 1 ? py0 + kTile - 1 : cam.H - 1;
    bool neg[3] = {false, false, false}, nonneg[3] = {false, false, false};
    for (int yi = 0; yi < 2; ++yi)
        for (int xi = 0; xi < 2; ++xi) {
            double d[3];
            pixel_ray_dir(cam, double(xi ? px1 : px0), double(yi ? py1 : py0), d);
            for (int ax = 0; ax < 3; ++ax) (d[ax] < 0.0 ? neg[ax] : nonneg[ax]) = true;
        }
    uint32_t mask = 0;
    for (uint32_t s = 0; s < 8; ++s) {
        bool ok = true;
        for (int ax = 0; ax < 3; ++ax) {
            bool want_neg = (s >> (2 - ax)) & 1;
            if (want_neg ? !neg[ax] : !nonneg[ax]) ok = false;
        }
        if (ok) mask |= 1u << s;
    }
    return mask;
}

// ---------------------------------------------------------------- fp32 field
// explin (field.hpp:23-26) and its derivative (field.hpp:28-31).
#if defined(__CUDA_ARCH__)
// exp(x) as one MUFU.EX2 (flush-to-zero; results are < 1e-38 only where they
// are irrelevant to alpha = 1 - exp(-x) and explin's exponential branch).
__device__ __forceinline__ float fexp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}
#else
inline float fexp(float x) { return expf(x); }
#endif
// alpha = 1 - exp(-x) for x >= 0 (voxel_alpha, field.hpp:92-116). For
// x < 1/32 the difference 1 - exp(-x) would keep only the absolute accuracy
// of exp near 1 (~1e-7), i.e. a large relative error in a small alpha, and
// that error adds up over the hundreds of faint voxels a ray can cross
// (depth = sum T alpha t grows with t). There the series
// x - x^2/2 + x^3/6 - x^4/24 is used (truncation < x^5/120).
SVR_HD float one_minus_exp_neg(float x) {
    const float big = 1.0f - fexp(-x);
    const float small = x * (1.0f - x * (0.5f - x * (1.0f / 6.0f - x * (1.0f / 24.0f))));
    return x < 0.03125f ? small : big;
}

// explin below the knee (field.hpp:23-26): exp(x/1.1 - 1 + ln 1.1)
// = 2^(x * log2(e)/1.1 + log2(1.1/e)), one FFMA + one MUFU.EX2; branch-free
// select. (The constants carry the reference's 1.1/e exactly to fp32: an
// error in them is a uniform relative bias on every optical depth, which
// compounds through T over hundreds of voxels per ray.)
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ float fexp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
#else
inline float fexp2(float x) { return exp2f(x); }
#endif
constexpr float kExplinA = 1.31154096f;   // log2(e) / 1.1
constexpr float kExplinB = -1.30519152f;  // log2(1.1 / e)
SVR_HD float explin(float x) {
    const float e = fexp2(fmaf(x, kExplinA, kExplinB));
    return x > kExplinKnee ? x : e;
}
SVR_HD float explin_deriv(float x) {
    return x > kExplinKnee ? 1.0f : fexp2(fmaf(x, kExplinA, kExplinB)) * (1.0f / 1.1f);
}

// trilinear (field.hpp:33-47), corner order (i<<2)|(j<<1)|k.
SVR_HD float trilinear(const float* V, float qx, float qy, float qz) {
    float wx0 = 1.0f - qx, wy0 = 1.0f - qy, wz0 = 1.0f - qz;
    float a00 = V[0] * wz0 + V[1] * qz;
    float a01 = V[2] * wz0 + V[3] * qz;
    float a10 = V[4] * wz0 + V[5] * qz;
    float a11 = V[6] * wz0 + V[7] * qz;
    float b0 = a00 * wy0 + a01 * qy;
    float b1 = a10 * wy0 + a11 * qy;
    return b0 * wx0 + b1 * qx;
}

// The same interpolant in monomial form, f = c0 + c1 qx + c2 qy + c3 qz +
// c4 qx qy + c5 qx qz + c6 qy qz + c7 qx qy qz: the voxel record carries the
// coefficients (computed once per voxel by K1), so a sample costs 7 FFMA
// instead of 7 lerps.
SVR_HD void trilinear_coeffs(const float* V, float* c) {
    c[0] = V[0];
    c[1] = V[4] - V[0];
    c[2] = V[2] - V[0];
    c[3] = V[1] - V[0];
    c[4] = (V[6] - V[4]) - (V[2] - V[0]);
    c[5] = (V[5] - V[4]) - (V[1] - V[0]);
    c[6] = (V[3] - V[2]) - (V[1] - V[0]);
    c[7] = ((V[7] - V[6]) - (V[5] - V[4])) - ((V[3] - V[2]) - (V[1] - V[0]));
}
// The record stores the coefficients pair-ordered for packed FP32:
//   ca = (c6, c7, c2, c4), cb = (c3, c5, c0, c1)
// so that (t6, t3) = qy * (qz * (c6, c7) + (c2, c4)) + (qz * (c3, c5) + (c0, c1))
// is three FFMA2 on register pairs as they come out of the 16-B loads, and
// f = qx * t3 + t6 one FFMA: each lane rounds exactly like the scalar chain.
SVR_HD void pack_coeffs(const float* c, float4& ca, float4& cb) {
    ca = make_float4(c[6], c[7], c[2], c[4]);
    cb = make_float4(c[3], c[5], c[0], c[1]);
}
SVR_HD void unpack_coeffs(float4 ca, float4 cb, float* c) {
    c[0] = cb.z; c[1] = cb.w; c[2] = ca.z; c[3] = cb.x;
    c[4] = ca.w; c[5] = cb.y; c[6] = ca.x; c[7] = ca.y;
}
SVR_HD float trilinear_poly_s(float4 ca, float4 cb, float qx, float qy, float qz) {
    const float t3 = fmaf(qy, fmaf(qz, ca.y, ca.w), fmaf(qz, cb.y, cb.w));
    const float t6 = fmaf(qy, fmaf(qz, ca.x, ca.z), fmaf(qz, cb.x, cb.z));
    return fmaf(qx, t3, t6);
}
// Corner densities back from the coefficients (epilogue's normal chain).
SVR_HD void trilinear_corners(float4 ca, float4 cb, float* V) {
    float c[8];
    unpack_coeffs(ca, cb, c);
    for (int n = 0; n < 8; ++n) {
        const float i = float((n >> 2) & 1), j = float((n >> 1) & 1), k = float(n & 1);
        V[n] = c[0] + i * c[1] + j * c[2] + k * c[3] + i * j * c[4] + i * k * c[5] + j * k * c[6] +
               i * j * k * c[7];
    }
}

SVR_HD void trilinear_weights(float qx, float qy, float qz, float* w) {
    float wx[2] = {1.0f - qx, qx}, wy[2] = {1.0f - qy, qy}, wz[2] = {1.0f - qz, qz};
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = wx[(c >> 2) & 1] * wy[(c >> 1) & 1] * wz[c & 1];
}

#if defined(__CUDACC__)
// Blackwell packed FP32 (FFMA2 / FMUL2: two IEEE fp32 operations per
// instruction, each rounded exactly like the scalar one). The slab's near and
// far face of an axis share every operand but the face selector, so one
// FFMA2 + one FMUL2 give both: 6 instead of 12 instructions per slab test.
#ifndef SVR_F32X2
#define SVR_F32X2 1
#endif
#ifndef SVR_F32X2_ACC
#define SVR_F32X2_ACC 1
#endif
#ifndef SVR_F32X2_Q
#define SVR_F32X2_Q 1
#endif
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(f32x2 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

#ifndef SVR_F32X2_TRI
#define SVR_F32X2_TRI 1
#endif
// trilinear_poly_s in three FFMA2 + one FFMA (record layout: pack_coeffs).
__device__ __forceinline__ float trilinear_poly(float4 ca, float4 cb, float qx, float qy, float qz) {
#if SVR_F32X2_TRI
    const f32x2 z2 = pk2(qz, qz);
    const f32x2 a = fma2(z2, pk2(ca.x, ca.y), pk2(ca.z, ca.w));
    const f32x2 b = fma2(z2, pk2(cb.x, cb.y), pk2(cb.z, cb.w));
    float t6, t3;
    up2(fma2(pk2(qy, qy), a, b), t6, t3);
    return fmaf(qx, t3, t6);
#else
    return trilinear_poly_s(ca, cb, qx, qy, qz);
#endif
}

struct SlabSel {
    float nx, ny, nz;  // 1 where the inverse direction component is negative
#if SVR_F32X2
    f32x2 px, py, pz;  // (n, 1 - n) per axis: the near and the far face
#endif
};
__device__ __forceinline__ SlabSel slab_sel(float ix, float iy, float iz) {
    SlabSel q;
    q.nx = ix < 0.f ? 1.f : 0.f;
    q.ny = iy < 0.f ? 1.f : 0.f;
    q.nz = iz < 0.f ? 1.f : 0.f;
#if SVR_F32X2
    q.px = pk2(q.nx, 1.f - q.nx);
    q.py = pk2(q.ny, 1.f - q.ny);
    q.pz = pk2(q.nz, 1.f - q.nz);
#endif
    return q;
}
__device__ __forceinline__ void slab_s(float4 lo, float ix, float iy, float iz, const SlabSel& q,
                                       float& ta, float& tb) {
#if SVR_F32X2
    float ax, bx, ay, by, az, bz;
    const f32x2 w = pk2(lo.w, lo.w);
    up2(mul2(fma2(w, q.px, pk2(lo.x, lo.x)), pk2(ix, ix)), ax, bx);
    up2(mul2(fma2(w, q.py, pk2(lo.y, lo.y)), pk2(iy, iy)), ay, by);
    up2(mul2(fma2(w, q.pz, pk2(lo.z, lo.z)), pk2(iz, iz)), az, bz);
#else
    const float ax = fmaf(lo.w, q.nx, lo.x) * ix, bx = fmaf(lo.w, 1.f - q.nx, lo.x) * ix;
    const float ay = fmaf(lo.w, q.ny, lo.y) * iy, by = fmaf(lo.w, 1.f - q.ny, lo.y) * iy;
    const float az = fmaf(lo.w, q.nz, lo.z) * iz, bz = fmaf(lo.w, 1.f - q.nz, lo.z) * iz;
#endif
    ta = fmaxf(fmaxf(ax, ay), az);
    tb = fminf(fminf(bx, by), bz);
}
#endif  // __CUDACC__

// density_gradient + voxel_normal (field.hpp:132-154).
SVR_HD void density_gradient(const float* V, float* g) {
    g[0] = 0.25f * ((V[4] + V[5] + V[6] + V[7]) - (V[0] + V[1] + V[2] + V[3]));
    g[1] = 0.25f * ((V[2] + V[3] + V[6] + V[7]) - (V[0] + V[1] + V[4] + V[5]));
    g[2] = 0.25f * ((V[1] + V[3] + V[5] + V[7]) - (V[0] + V[2] + V[4] + V[6]));
}

SVR_HD void voxel_normal(const float* V, float* n) {
    float g[3];
    density_gradient(V, g);
    float len = sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (len == 0.0f) {
        n[0] = n[1] = n[2] = 0.0f;
        return;
    }
    float inv = 1.0f / len;
    n[0] = g[0] * inv;
    n[1] = g[1] * inv;
    n[2] = g[2] * inv;
}

// voxel_normal_backward (field.hpp:158-170).
SVR_HD void voxel_normal_backward(const float* V, const float* dn, float* gV) {
    float g[3];
    density_gradient(V, g);
    float len = sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (len == 0.0f) {
        for (int c = 0; c < 8; ++c) gV[c] = 0.0f;
        return;
    }
    float inv = 1.0f / len;
    float n[3] = {g[0] * inv, g[1] * inv, g[2] * inv};
    float dot = dn[0] * n[0] + dn[1] * n[1] + dn[2] * n[2];
    float gx = (dn[0] - n[0] * dot) * inv, gy = (dn[1] - n[1] * dot) * inv,
          gz = (dn[2] - n[2] * dot) * inv;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float si = ((c >> 2) & 1) ? 1.0f : -1.0f;
        float sj = ((c >> 1) & 1) ? 1.0f : -1.0f;
        float sk = (c & 1) ? 1.0f : -1.0f;
        gV[c] = 0.25f * (gx * si + gy * sj + gz * sk);
    }
}

// sh_basis (sh.hpp:18-45), 3DGS ordering and constants.
SVR_HD int sh_basis(int degree, float x, float y, float z, float* b) {
    b[0] = 0.28209479177387814f;
    if (degree < 1) return 1;
    const float C1 = 0.4886025119029199f;
    b[1] = -C1 * y;
    b[2] = C1 * z;
    b[3] = -C1 * x;
    if (degree < 2) return 4;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = 1.0925484305920792f * xy;
    b[5] = -1.0925484305920792f * yz;
    b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    b[7] = -1.0925484305920792f * xz;
    b[8] = 0.5462742152960396f * (xx - yy);
    if (degree < 3) return 9;
    b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    b[10] = 2.890611442640554f * xy * z;
    b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
    return 16;
}

}  // namespace svrb
