// backward.cu — gradient path of the rasterizer on sm_100a.
//
//   lift               AreaResampler::adjoint (image.cpp:47-60)
//   l1_loss            new L1 photometric loss (pattern of losses.cpp:121-131)
//   K9 composite_bwd   render_backward per-pixel reverse walk (raster.cpp:340-409)
//   K10 voxel_epilogue sh_eval_backward + voxel_normal_backward per visible voxel
//                      (raster.cpp:411-421, sh.hpp:62-80, field.hpp:158-170)
//
// K9 keeps the reference's division-free recursion (raster.cpp:374-407):
// the forward record pass stored, per contribution, the entry id and the
// transmittance in front of it (T_i), so the reverse walk needs no
// T/(1-alpha). All pixels of a tile walk the tile's entry list backwards in
// lock-step (coherent shared-memory staging, like the forward), so the
// per-entry gradient of the 32 pixels of a warp is reduced with shuffles and
// then through shared memory; one set of global atomics per (tile, entry).
#include <cuda_runtime.h>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {

namespace {


__global__ void lift_kernel(TapTable t, const float* g, int ch, int W, float* out, int sw,
                            int sh) {
    pdl_enter();
    int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= sw || y >= sh) return;
    float acc[3] = {0.f, 0.f, 0.f};
    for (int ty = t.ptr_y[y]; ty < t.ptr_y[y + 1]; ++ty) {
        const int dy = t.idx_y[ty];
        const float wy = t.w_y[ty];
        float mid[3] = {0.f, 0.f, 0.f};
        for (int tx = t.ptr_x[x]; tx < t.ptr_x[x + 1]; ++tx) {
            const float wx = t.w_x[tx];
            const float* s = g + (uint64_t(dy) * W + t.idx_x[tx]) * ch;
            for (int c = 0; c < ch; ++c) mid[c] += wx * s[c];
        }
        for (int c = 0; c < ch; ++c) acc[c] += wy * mid[c];
    }
    for (int c = 0; c < ch; ++c) out[(uint64_t(y) * sw + x) * ch + c] = acc[c];
}

__global__ void l1_kernel(const float* c, const float* gt, uint64_t n, float inv_n, float* d_color,
                          float* loss) {
    pdl_enter();
    float s = 0.f;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        float e = c[i] - gt[i];
        s += fabsf(e);
        d_color[i] = (e > 0.f ? inv_n : (e < 0.f ? -inv_n : 0.f));
    }
    if (!loss) return;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ float s_w[32];
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? s_w[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(loss, s * inv_n);
    }
}

// Sum of v[0..15] over the 32 lanes by recursive halving: each step sends
// half of the remaining values to the partner lane, so 16 values cost 16
// shuffles instead of 80. On return lanes 2q and 2q+1 hold the total of
// component q.
__device__ __forceinline__ float warp_transpose_sum16(float (&v)[16], int lane) {
#pragma unroll
    for (int h = 8, bit = 16; h >= 1; h >>= 1, bit >>= 1) {
        const bool upper = (lane & bit) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = upper ? v[i] : v[i + h];
            const float keep = upper ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
        }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// K9: warp-autonomous reverse walk. Each warp owns the same 8x4 pixel block
// as the forward composite and walks the tile's entry list backwards in
// chunks of 32, visiting only chunks that hold one of its pending
// contributions. Per chunk, the entries that can matter for the block
// (sign pattern, screen AABB, frustum: the forward's own filters) are
// gathered into warp-private shared memory; then the warp repeatedly takes
// the largest pending entry id over its lanes (every lane's contribution
// list is descending) and the lanes whose next contribution it is apply the
// division-free recursion of raster.cpp:374-407. The 15 per-entry sums
// (8 corner densities, colour, normal, priority) are reduced across the warp
// by recursive halving and issued as one vector of global atomics.
#ifndef SVR_BWD_F32X2
#define SVR_BWD_F32X2 0  // packed FP32 in the hit path (bit-identical; measured: no gain, 75 registers)
#endif
#ifndef SVR_BWD_VNEXT
#define SVR_BWD_VNEXT 0  // values of the chunk below loaded while the current one is walked (config 3 0.586 -> 0.609 ms, config 5 2.64 -> 2.68: off)
#endif
#ifndef SVR_BWD_CPASYNC
#define SVR_BWD_CPASYNC 0  // records gathered with cp.async, no register staging (config 3 0.588 -> 0.587 ms, config 5 2.638 -> 2.643: neutral, off)
#endif
#ifndef SVR_BWD_SMEMRED
#define SVR_BWD_SMEMRED 0  // warp reduction through shared memory (config 3 0.589 -> 0.616 ms, config 5 2.66 -> 2.70: off)
#endif
#ifndef SVR_BWD_DIRECT
#define SVR_BWD_DIRECT 12  // at most this many hit lanes: per-lane float4 reductions instead of the shuffle tree (4: 0.588, 8: 0.568, 12: 0.560, 16: 0.569, 32: 1.07 ms on config 3)
#endif
// UPC: per-contribution upstream gradients (d_weight / d_voxel_color, the
// ray losses) present; without them the hit loop carries no checks for them.
template <int K, bool UPC>
#ifndef SVR_BWD_MINB
// CTAs per SM the register allocation targets: 4 (64 registers, no spills)
// for K <= 2 (config 3 K9 0.586 -> 0.573 ms; 3 CTAs at 71-72 registers:
// 0.589), unconstrained for K = 3, which spills at 64
#define SVR_BWD_MINB(K) ((K) <= 2 ? 4 : 1)
#endif
__global__ void __launch_bounds__(256, SVR_BWD_MINB(K)) composite_backward_kernel(DevCamera cam, BackwardArgs a) {
    pdl_enter();
    __shared__ float4 s_rec[8][32][kRecordF4];
    __shared__ float s_cone[8][4][3];
#if SVR_BWD_SMEMRED
    // per warp: 32 rows of 16 sums at a 20-float stride, the upper 16 rows
    // shifted by 16 floats (conflict-free row stores and column loads)
    constexpr int kRedRow = 20;
    __shared__ __align__(16) float s_red[8][32 * kRedRow + 16];
#endif

    const int tile = a.tile_order ? int(a.tile_order[blockIdx.x]) : int(blockIdx.x);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tx = tile % cam.ntx, ty = tile / cam.ntx;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const bool inside = px < cam.W && py < cam.H;
    const uint32_t slot = uint32_t(tile) * 256u + uint32_t((py % kTile) * kTile + (px % kTile));
    const int wx0 = px - (lane & 7), wy0 = py - (lane >> 3);
    const float fx0 = float(wx0) + 0.5f, fx1 = float(wx0) + 7.5f;
    const float fy0 = float(wy0) + 0.5f, fy1 = float(wy0) + 3.5f;

    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const uint32_t my_sign = sign_bits(dd);
    const uint32_t warp_signs = __reduce_or_sync(0xffffffffu, inside ? (1u << my_sign) : 0u);
    const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
    const float ix = slab_inv(dd[0]), iy = slab_inv(dd[1]), iz = slab_inv(dd[2]);
    const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));
#if SVR_BWD_F32X2
    const SlabSel ssel = slab_sel(ix, iy, iz);
#endif
    float (*cone)[3] = s_cone[warp];
    if (lane == 0) warp_cone_planes(cam, wx0, wy0, cone);
    __syncwarp();

    int n = 0;
    uint32_t base = 0;
    float gC[3] = {0.f, 0.f, 0.f}, gN[3] = {0.f, 0.f, 0.f}, gD = 0.f, gT = 0.f;
    if (inside) {
        n = int(a.pix_count[slot]);
        base = a.pix_begin[slot];
        const uint64_t p = uint64_t(py) * cam.W + px;
        if (a.gC) gC[0] = a.gC[3 * p], gC[1] = a.gC[3 * p + 1], gC[2] = a.gC[3 * p + 2];
        if (a.gN) gN[0] = a.gN[3 * p], gN[1] = a.gN[3 * p + 1], gN[2] = a.gN[3 * p + 2];
        if (a.gD) gD = a.gD[p];
        if (a.gT) gT = a.gT[p];
    }
    // pending contributions: (e1, T1) next, (e2, T2) the one after (prefetched)
    // record k of this pixel: compact base + k, or staged k * stride + slot
    const uint64_t rb = a.stage_stride ? slot : base;
    const uint64_t rs = a.stage_stride ? a.stage_stride : 1u;
    int kidx = n - 1;
    int e1 = -1, e2 = -1;
    float T1 = 0.f, T2 = 0.f;
    if (kidx >= 0) e1 = int(a.contrib_entry[rb + kidx * rs]), T1 = a.contrib_T[rb + kidx * rs];
    if (kidx >= 1)
        e2 = int(a.contrib_entry[rb + (kidx - 1) * rs]), T2 = a.contrib_T[rb + (kidx - 1) * rs];
    float Ra = gC[0] * a.bg[0] + gC[1] * a.bg[1] + gC[2] * a.bg[2] + gT;
    float Rd = 0.f;

    const uint2 range = a.ranges[tile];
    constexpr uint32_t kVidMask = (1u << 29) - 1u;
    float4 (*wrec)[kRecordF4] = s_rec[warp];

    int cur = __reduce_max_sync(0xffffffffu, unsigned(e1 + 1)) - 1;
#if SVR_BWD_VNEXT
    // the values of the chunk below the current one, loaded while it is
    // walked (the walk usually moves to the adjacent chunk next)
    uint32_t vn = 0, vn_c0 = 0xffffffffu;
#endif
    while (cur >= 0) {
        // chunk holding `cur`, aligned to the tile's range start
        const uint32_t c0 = range.x + (uint32_t(cur) - range.x) / 32u * 32u;
        const uint32_t e = c0 + lane;
        bool rel = false;
        uint32_t v = 0;
#if SVR_BWD_VNEXT
        const bool have = vn_c0 == c0;
        const uint32_t vh = vn;
        if (c0 >= range.x + 32u) {
            vn_c0 = c0 - 32u;
            vn = __ldg(a.vals + c0 - 32u + lane);
        } else {
            vn_c0 = 0xffffffffu;
        }
#endif
        if (e < range.y && e <= uint32_t(cur)) {
#if SVR_BWD_VNEXT
            v = have ? vh : __ldg(a.vals + e);
#else
            v = __ldg(a.vals + e);
#endif
            const float4 b = __ldg(a.records + uint64_t(v & kVidMask) * kRecordF4 + 1);
            rel = ((warp_signs >> (v >> 29)) & 1u) &&
                  !(fx1 < b.x || fx0 > b.y || fy1 < b.z || fy0 > b.w);
            if (rel && (b.y - b.x) * (b.w - b.z) > kConeMinArea) {
                const float4 lo = __ldg(a.records + uint64_t(v & kVidMask) * kRecordF4);
                rel = box_in_cone(cone, lo);
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, rel);
        if (rel) {
            const int sl = __popc(m & ((1u << lane) - 1u));
            const float4* src = a.records + uint64_t(v & kVidMask) * kRecordF4;
#if SVR_BWD_CPASYNC
#pragma unroll
            for (int k = 0; k < kRecordF4; ++k) {
                const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(&wrec[sl][k]));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + k) : "memory");
            }
#else
#pragma unroll
            for (int k = 0; k < kRecordF4; ++k) wrec[sl][k] = __ldg(src + k);
#endif
        }
#if SVR_BWD_CPASYNC
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
#endif
        __syncwarp();
        while (cur >= int(c0)) {
            const int sl = __popc(m & ((1u << (uint32_t(cur) - c0)) - 1u));
            const bool hit = (e1 == cur);
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.f;
            if (hit) {
                const float4 lo = wrec[sl][0];
                const float inv = wrec[sl][5].w;
#if SVR_BWD_F32X2
                float ta, tb;
                slab_s(lo, ix, iy, iz, ssel, ta, tb);  // packed FP32, same floats
#else
                float t0 = lo.x * ix, t1 = (lo.x + lo.w) * ix;
                float ta = fminf(t0, t1), tb = fmaxf(t0, t1);
                t0 = lo.y * iy;
                t1 = (lo.y + lo.w) * iy;
                ta = fmaxf(ta, fminf(t0, t1));
                tb = fminf(tb, fmaxf(t0, t1));
                t0 = lo.z * iz;
                t1 = (lo.z + lo.w) * iz;
                ta = fmaxf(ta, fminf(t0, t1));
                tb = fminf(tb, fmaxf(t0, t1));
#endif
                const float4 va = wrec[sl][2], vb = wrec[sl][3];
                const float seg = tb - ta;
                const float lk = seg * dnorm * (1.0f / K);
                float sa[K], tk[K], vk[K], qk[K][3];
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    tk[k] = ta + ((k + 0.5f) / K) * seg;
#if SVR_BWD_F32X2
                    up2(mul2(fma2(pk2(tk[k], tk[k]), pk2(dx, dy), pk2(-lo.x, -lo.y)), pk2(inv, inv)), qk[k][0],
                        qk[k][1]);
#else
                    qk[k][0] = (tk[k] * dx - lo.x) * inv;
                    qk[k][1] = (tk[k] * dy - lo.y) * inv;
#endif
                    qk[k][2] = (tk[k] * dz - lo.z) * inv;
                    vk[k] = trilinear_poly(va, vb, qk[k][0], qk[k][1], qk[k][2]);
                    const float act = explin(vk[k]);
                    sum += act;
                    sa[k] = one_minus_exp_neg(lk * act);
                }
                const float alpha = (K == 1) ? sa[0] : one_minus_exp_neg(lk * sum);
                float dvox = 0.f, Tk = 1.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dvox += Tk * sa[k] * tk[k];
                    Tk *= 1.0f - sa[k];
                }
                const float Ti = T1;
                const float4 col = wrec[sl][4], nor = wrec[sl][5];
                const float gw = (UPC && a.d_weight) ? a.d_weight[base + kidx] : 0.f;
                const float phi = gC[0] * col.x + gC[1] * col.y + gC[2] * col.z + gN[0] * nor.x +
                                  gN[1] * nor.y + gN[2] * nor.z + gw;
                const float A = Ti * (phi - Ra - Rd);  // dL/dalpha_i (raster.cpp:383)
                acc[14] = fabsf(alpha * A);
                // voxel_depth_backward (field.hpp:184-201)
                float ddk[K];
                if constexpr (K == 1) {
                    ddk[0] = tk[0];
                } else if constexpr (K == 2) {
                    ddk[0] = tk[0] - sa[1] * tk[1];
                    ddk[1] = tk[1] - sa[0] * tk[1];
                } else {
                    ddk[0] = tk[0] + sa[1] * sa[2] * tk[2] - sa[1] * tk[1] - sa[2] * tk[2];
                    ddk[1] = tk[1] + sa[0] * sa[2] * tk[2] - sa[0] * tk[1] - sa[2] * tk[2];
                    ddk[2] = tk[2] + sa[0] * sa[1] * tk[2] - sa[0] * tk[2] - sa[1] * tk[2];
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    float others = 1.f;
#pragma unroll
                    for (int mm = 0; mm < K; ++mm)
                        if (mm != k) others *= 1.0f - sa[mm];
                    const float dAk = A * others + Ti * gD * ddk[k];
                    const float dv = dAk * (1.0f - sa[k]) * lk * explin_deriv(vk[k]);
#if SVR_BWD_F32X2
                    {  // corners (2j, 2j+1) differ only in the z weight: FMUL2 / FFMA2 pairs
                        const float wx[2] = {1.0f - qk[k][0], qk[k][0]}, wy[2] = {1.0f - qk[k][1], qk[k][1]};
                        const f32x2 wz = pk2(1.0f - qk[k][2], qk[k][2]), dd = pk2(dv, dv);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float wxy = wx[(j >> 1) & 1] * wy[j & 1];
                            const f32x2 a2 = fma2(dd, mul2(pk2(wxy, wxy), wz), pk2(acc[2 * j], acc[2 * j + 1]));
                            up2(a2, acc[2 * j], acc[2 * j + 1]);
                        }
                    }
#else
                    float w[8];
                    trilinear_weights(qk[k][0], qk[k][1], qk[k][2], w);
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[c] += dv * w[c];
#endif
                }
                const float wgt = Ti * alpha;
                acc[8] = wgt * gC[0];
                acc[9] = wgt * gC[1];
                acc[10] = wgt * gC[2];
                if (UPC && a.d_voxel_color) {
                    const float* vc = a.d_voxel_color + 3ull * (base + kidx);
                    acc[8] += vc[0];
                    acc[9] += vc[1];
                    acc[10] += vc[2];
                }
                acc[11] = wgt * gN[0];
                acc[12] = wgt * gN[1];
                acc[13] = wgt * gN[2];
                Ra = alpha * phi + (1.0f - alpha) * Ra;
                Rd = dvox * gD + (1.0f - alpha) * Rd;
                // advance this pixel's list; prefetch the one after
                --kidx;
                e1 = e2;
                T1 = T2;
                if (kidx >= 1) {
                    e2 = int(a.contrib_entry[rb + (kidx - 1) * rs]);
                    T2 = a.contrib_T[rb + (kidx - 1) * rs];
                } else {
                    e2 = -1;
                }
            }
            const uint32_t vid = __float_as_uint(wrec[sl][4].w);
            const uint32_t hm = __ballot_sync(0xffffffffu, hit);
            float4* gv = reinterpret_cast<float4*>(a.g_vox + 16ull * vid);
            if (__popc(hm) <= SVR_BWD_DIRECT) {
                // few pixels: each one adds its own 15 values (no 31-shuffle
                // reduction) as four float4 reductions into the voxel's record
                if (hit) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        atomicAdd(gv + j, make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]));
                }
            } else {
                // component q ends on lanes 2q, 2q+1; lanes 8j gather q = 4j..4j+3
#if SVR_BWD_SMEMRED
                // through shared memory: each lane stores its 16 values as a
                // row (4 x STS.128), lane (q, h) sums component q over rows
                // 16h..16h+15 (16 LDS with immediate offsets) and one shuffle
                // joins the halves: ~40 instructions instead of the 62 of the
                // shuffle transpose (16 SHFL + 30 SEL + 16 FADD)
                float* red = s_red[warp];
                float4* row = reinterpret_cast<float4*>(red + kRedRow * lane + (lane >> 4) * 16);
#pragma unroll
                for (int j = 0; j < 4; ++j) row[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
                __syncwarp();
                const float* col = red + (lane >> 1) + (lane & 1) * (16 * kRedRow + 16);
                float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    p0 += col[(j + 0) * kRedRow];
                    p1 += col[(j + 1) * kRedRow];
                    p2 += col[(j + 2) * kRedRow];
                    p3 += col[(j + 3) * kRedRow];
                }
                const float half = (p0 + p1) + (p2 + p3);
                const float tot = half + __shfl_xor_sync(0xffffffffu, half, 1);
                __syncwarp();  // rows are rewritten by the next entry
#else
                const float tot = warp_transpose_sum16(acc, lane);
#endif
                const float t1 = __shfl_down_sync(0xffffffffu, tot, 2);
                const float t2 = __shfl_down_sync(0xffffffffu, tot, 4);
                const float t3 = __shfl_down_sync(0xffffffffu, tot, 6);
                if ((lane & 7) == 0) atomicAdd(gv + (lane >> 3), make_float4(tot, t1, t2, t3));
            }
            cur = __reduce_max_sync(0xffffffffu, unsigned(e1 + 1)) - 1;
        }
        __syncwarp();
    }
}

// ray_losses (losses.cpp:141-238). A group of L = 8 lanes per supersampled
// pixel (4 pixels per warp: a pixel has a few dozen contributions, so a
// whole warp per pixel left most lanes idle; 8 lanes: 264 -> 277 it/s on
// config 3i): its contributions are contiguous in the compact (reference)
// order, so lane k handles contribution chunk*L + k and the upstream
// gradient reads/writes are coalesced per group. w = T_i * alpha_i is
// recomputed from the voxel record exactly as the forward composited it
// (fp32 slab + quadrature); m = (a + b) / 2 and l = b - a come from the same
// slab. L_dist's prefix sums are segmented shuffle scans carried across
// chunks; its suffix half is a second pass in reverse over (w, m) kept in
// scratch, like the reference's two loops.
template <int L>
__device__ __forceinline__ float group_incl_scan_f(float v, int lane, unsigned gmask) {
#pragma unroll
    for (int o = 1; o < L; o <<= 1) {
        const float n = __shfl_up_sync(gmask, v, o, L);
        if (lane >= o) v += n;
    }
    return v;
}

// L_T (losses.cpp:163-174): one thread per supersampled pixel.
__global__ void __launch_bounds__(256) ray_loss_T_kernel(RayLossArgs a, uint64_t npix) {
    pdl_enter();
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const double inv_rays = 1.0 / double(npix);
    float lT = 0.f;
    if (p < npix) {
        const float eps = 1e-6f;
        const float T = a.tfin[p];
        const float Tc = fminf(fmaxf(T, eps), 1.0f - eps);
        const float l0 = logf(Tc), l1 = logf(1.0f - Tc);
        lT = -(Tc * l0 + (1.0f - Tc) * l1);
        if (T > eps && T < 1.0f - eps && a.d_tfin_ss) a.d_tfin_ss[p] += float(a.w_T * inv_rays) * (l1 - l0);
    }
    for (int o = 16; o > 0; o >>= 1) lT += __shfl_xor_sync(0xffffffffu, lT, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(a.sums, double(lT) * inv_rays);
}

template <int K, int L>
__global__ void __launch_bounds__(256) ray_losses_kernel(DevCamera cam, RayLossArgs a) {
    pdl_enter();
    // L lanes per pixel: grid (ceil(W / (256 / L)), H); group g of block
    // (bx, y) owns pixel ((256 / L) bx + g, y)
    const int lane = threadIdx.x & (L - 1);
    const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (threadIdx.x & 31 & ~(L - 1)));
    const int px = int(blockIdx.x) * (256 / L) + int(threadIdx.x / L), py = int(blockIdx.y);
    const uint64_t npix = uint64_t(cam.W) * cam.H;
    const double inv_rays = 1.0 / double(npix);
    float lT = 0.f, ldist = 0.f, lR = 0.f;
    if (px < cam.W) {
        const uint32_t tile = uint32_t(py / kTile) * cam.ntx + uint32_t(px / kTile);
        const uint32_t slot = tile * 256u + uint32_t((py % kTile) * kTile + (px % kTile));
        const uint32_t n = a.pix_count[slot];
        if (n > 0 && (a.w_dist != 0.0 || a.w_R != 0.0)) {
            const uint32_t base = a.pix_begin[slot];
            double dd[3];
            pixel_ray_dir(cam, double(px), double(py), dd);
            const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
            const float ix = slab_inv(dd[0]), iy = slab_inv(dd[1]), iz = slab_inv(dd[2]);
            const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));
            float g[3] = {0.f, 0.f, 0.f};
            if (a.w_R != 0.0) {
                const int gx = min(a.gt_w - 1, px * a.gt_w / cam.W);
                const int gy = min(a.gt_h - 1, py * a.gt_h / cam.H);
                const float* gp = a.gt + (uint64_t(gy) * a.gt_w + gx) * 3;
                g[0] = gp[0], g[1] = gp[1], g[2] = gp[2];
            }
            constexpr uint32_t kVidMask = (1u << 29) - 1u;
            const float wd = float(a.w_dist * inv_rays);
            float Wc = 0.f, Sc = 0.f;  // prefix carries across chunks
            for (uint32_t c0 = 0; c0 < n; c0 += L) {
                const uint32_t i = c0 + lane;
                const bool on = i < n;
                float w = 0.f, m = 0.f, dl = 0.f, gdw = 0.f;
                float err = 0.f, e0 = 0.f, e1 = 0.f, e2 = 0.f;
                if (on) {
                    const uint64_t at = a.stage_stride ? uint64_t(i) * a.stage_stride + slot : uint64_t(base) + i;
                    const uint32_t e = a.contrib_entry[at];
                    const float T = a.contrib_T[at];
                    const float4* rec = a.records + uint64_t(__ldg(a.vals + e) & kVidMask) * kRecordF4;
                    const float4 lo = __ldg(rec);
                    const float inv = __ldg(rec + 5).w;
                    float t0 = lo.x * ix, t1 = (lo.x + lo.w) * ix;
                    float ta = fminf(t0, t1), tb = fmaxf(t0, t1);
                    t0 = lo.y * iy;
                    t1 = (lo.y + lo.w) * iy;
                    ta = fmaxf(ta, fminf(t0, t1));
                    tb = fminf(tb, fmaxf(t0, t1));
                    t0 = lo.z * iz;
                    t1 = (lo.z + lo.w) * iz;
                    ta = fmaxf(ta, fminf(t0, t1));
                    tb = fminf(tb, fmaxf(t0, t1));
                    const float4 va = __ldg(rec + 2), vb = __ldg(rec + 3);
                    const float seg = tb - ta;
                    const float lk = seg * dnorm * (1.0f / K);
                    float sum = 0.f, sa0 = 0.f;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const float tk = ta + ((k + 0.5f) / K) * seg;
                        const float act = explin(trilinear_poly(va, vb, (tk * dx - lo.x) * inv,
                                                                (tk * dy - lo.y) * inv,
                                                                (tk * dz - lo.z) * inv));
                        sum += act;
                        if (K == 1) sa0 = one_minus_exp_neg(lk * act);
                    }
                    const float alpha = (K == 1) ? sa0 : one_minus_exp_neg(lk * sum);
                    w = T * alpha;
                    m = 0.5f * (ta + tb);
                    dl = tb - ta;
                    if (a.w_R != 0.0) {
                        const float4 col = __ldg(rec + 4);
                        e0 = col.x - g[0], e1 = col.y - g[1], e2 = col.z - g[2];
                        err = e0 * e0 + e1 * e1 + e2 * e2;
                    }
                }
                if (a.w_dist != 0.0) {
                    const float wi = group_incl_scan_f<L>(w, lane, gmask);
                    const float si = group_incl_scan_f<L>(w * m, lane, gmask);
                    const float Wpre = Wc + wi - w, Spre = Sc + si - w * m;
                    if (on) {
                        ldist += 2.f * w * (m * Wpre - Spre) + w * w * dl * (1.0f / 3.0f);
                        gdw = wd * (2.f * (m * Wpre - Spre) + 2.f * w * dl * (1.0f / 3.0f));
                        a.scratch[base + i] = make_float2(w, m);
                    }
                    Wc += __shfl_sync(gmask, wi, L - 1, L);
                    Sc += __shfl_sync(gmask, si, L - 1, L);
                }
                if (on) {
                    if (a.w_R != 0.0) {
                        lR += w * err;
                        gdw += float(a.w_R * inv_rays) * err;
                        const float sc = float(a.w_R * 2.0 * inv_rays) * w;
                        float* dvc = a.d_voxel_color + 3ull * (base + i);
                        dvc[0] += sc * e0;
                        dvc[1] += sc * e1;
                        dvc[2] += sc * e2;
                    }
                    a.d_weight[base + i] += gdw;
                }
            }
            if (a.w_dist != 0.0) {  // suffix half of d|m_i - m_j|, chunks in reverse
                float Wsc = 0.f, Ssc = 0.f;
                const uint32_t last = (n - 1) / L * L;
                for (int c0 = int(last); c0 >= 0; c0 -= L) {
                    const uint32_t i = uint32_t(c0) + (L - 1) - lane;  // reversed lane order
                    const bool on = i < n;
                    float2 wm = make_float2(0.f, 0.f);
                    if (on) wm = a.scratch[base + i];
                    const float wi = group_incl_scan_f<L>(wm.x, lane, gmask);
                    const float si = group_incl_scan_f<L>(wm.x * wm.y, lane, gmask);
                    const float Wsuf = Wsc + wi - wm.x, Ssuf = Ssc + si - wm.x * wm.y;
                    if (on) a.d_weight[base + i] += wd * (2.f * (Ssuf - wm.y * Wsuf));
                    Wsc += __shfl_sync(gmask, wi, L - 1, L);
                    Ssc += __shfl_sync(gmask, si, L - 1, L);
                }
            }
        }
    }
    // block sums -> one double atomic per value per block
    __shared__ float s_red[3][8];
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lT += __shfl_xor_sync(0xffffffffu, lT, o);
        ldist += __shfl_xor_sync(0xffffffffu, ldist, o);
        lR += __shfl_xor_sync(0xffffffffu, lR, o);
    }
    if ((threadIdx.x & 31) == 0) s_red[0][warp] = lT, s_red[1][warp] = ldist, s_red[2][warp] = lR;
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += s_red[threadIdx.x][w];
        atomicAdd(a.sums + threadIdx.x, t * inv_rays);
    }
}

// ---- mse_loss + ssim_loss (losses.cpp:71-139) ------------------------------
// Valid-mode separable 11-tap Gaussian blurs of a, b, a^2, b^2, ab (row
// pass, then column pass fused with the SSIM map and its three gradient
// maps), then the exact adjoint blur (column, then row) of those maps, as
// blur_valid / blur_adjoint do. fp32 storage, fp64 where sums meet.
constexpr float kSsimC1 = 0.01f * 0.01f, kSsimC2 = 0.03f * 0.03f;

__global__ void ssim_rows_kernel(ImageLossArgs a) {
    pdl_enter();
    const int Wv = a.W - 10;
    const uint64_t n = uint64_t(Wv) * a.H * 3;
    double sq = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % 3), x = int((i / 3) % Wv), y = int(i / (3ull * Wv));
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const uint64_t j = (uint64_t(y) * a.W + x + k) * 3 + c;
            const float va = a.a[j], vb = a.b[j], w = a.kern[k];
            s0 += w * va;
            s1 += w * vb;
            s2 += w * (va * va);
            s3 += w * (vb * vb);
            s4 += w * (va * vb);
        }
        a.mid[i] = s0;
        a.mid[n + i] = s1;
        a.mid[2 * n + i] = s2;
        a.mid[3 * n + i] = s3;
        a.mid[4 * n + i] = s4;
    }
    // MSE over the full image rides along (grid-stride over W*H*3)
    const uint64_t nf = uint64_t(a.W) * a.H * 3;
    const double inv_n = 1.0 / double(nf);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nf;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double e = double(a.a[i]) - double(a.b[i]);
        sq += e * e;
        if (a.d_a && a.w_mse != 0.0) a.d_a[i] += float(a.w_mse * 2.0 * e * inv_n);
    }
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(a.sums, sq);
}

__global__ void ssim_cols_kernel(ImageLossArgs a) {
    pdl_enter();
    const int Wv = a.W - 10, Hv = a.H - 10;
    const uint64_t nmid = uint64_t(Wv) * a.H * 3, nv = uint64_t(Wv) * Hv * 3;
    const double g = -a.w_ssim / double(nv);  // dL/dmean of ssim_loss: -weight
    double tot = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % 3), x = int((i / 3) % Wv), y = int(i / (3ull * Wv));
        float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const uint64_t j = (uint64_t(y + k) * Wv + x) * 3 + c;
#pragma unroll
            for (int q = 0; q < 5; ++q) m[q] += a.kern[k] * a.mid[q * nmid + j];
        }
        const double ma = m[0], mb = m[1];
        const double va = m[2] - ma * ma, vb = m[3] - mb * mb, cab = m[4] - ma * mb;
        const double n1 = 2.0 * ma * mb + kSsimC1, n2 = 2.0 * cab + kSsimC2;
        const double d1 = ma * ma + mb * mb + kSsimC1, d2 = va + vb + kSsimC2;
        const double sv = (n1 * n2) / (d1 * d2);
        tot += sv;
        if (a.d_a) {
            const double ds_dmu = 2.0 * mb * n2 / (d1 * d2) - 2.0 * ma * sv / d1;
            const double ds_dva = -sv / d2;
            const double ds_dcab = 2.0 * n1 / (d1 * d2);
            a.maps[i] = float(g * (ds_dmu - 2.0 * ma * ds_dva - mb * ds_dcab));
            a.maps[nv + i] = float(g * ds_dva);
            a.maps[2 * nv + i] = float(g * ds_dcab);
        }
    }
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(a.sums + 1, tot);
}

// blur_adjoint (losses.cpp:47-61), column half: valid maps -> (W-10) x H
__global__ void ssim_adj_cols_kernel(ImageLossArgs a) {
    pdl_enter();
    const int Wv = a.W - 10, Hv = a.H - 10;
    const uint64_t nv = uint64_t(Wv) * Hv * 3, n = uint64_t(Wv) * a.H * 3;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % 3), x = int((i / 3) % Wv), y = int(i / (3ull * Wv));
        float s[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const int yy = y - k;  // output row yy + k == y
            if (yy < 0 || yy >= Hv) continue;
            const uint64_t j = (uint64_t(yy) * Wv + x) * 3 + c;
#pragma unroll
            for (int q = 0; q < 3; ++q) s[q] += a.kern[k] * a.maps[q * nv + j];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) a.adj[q * n + i] = s[q];
    }
}

// row half of the adjoint, then d_a += g1 + 2 a g2 + b g3 (losses.cpp:110-115)
__global__ void ssim_adj_rows_kernel(ImageLossArgs a) {
    pdl_enter();
    const int Wv = a.W - 10;
    const uint64_t nm = uint64_t(Wv) * a.H * 3, n = uint64_t(a.W) * a.H * 3;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const int c = int(i % 3), x = int((i / 3) % a.W), y = int(i / (3ull * a.W));
        float s[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const int xx = x - k;
            if (xx < 0 || xx >= Wv) continue;
            const uint64_t j = (uint64_t(y) * Wv + xx) * 3 + c;
#pragma unroll
            for (int q = 0; q < 3; ++q) s[q] += a.kern[k] * a.adj[q * nm + j];
        }
        a.d_a[i] += s[0] + 2.0f * a.a[i] * s[1] + a.b[i] * s[2];
    }
}

// adam_step (optim.cpp:322-345): HBM-bound elementwise update, grid-stride.
// Every double operation is explicitly rounded (no FMA contraction) in the
// reference's order, so params match std::vector<float> updates exactly.
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
    pdl_enter();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double g = double(a.grads[i]);
        if (isnan(g)) {
            atomicOr(a.nan_flag, 1u);
            continue;
        }
        const double m = __dadd_rn(__dmul_rn(a.beta1, a.m[i]), __dmul_rn(__dsub_rn(1.0, a.beta1), g));
        const double v = __dadd_rn(__dmul_rn(a.beta2, a.v[i]),
                                   __dmul_rn(__dmul_rn(__dsub_rn(1.0, a.beta2), g), g));
        a.m[i] = m;
        a.v[i] = v;
        const double mhat = __ddiv_rn(m, a.bc1), vhat = __ddiv_rn(v, a.bc2);
        const double lr = (a.period && (i % a.period) >= a.n_primary) ? a.lr_alt : a.lr;
        const double step = __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), a.eps));
        a.params[i] = float(__dsub_rn(double(a.params[i]), step));
    }
}

// K10: 16 lanes per voxel, lane m owns SH basis function m, so the SH rows
// (3(d+1)^2 floats per voxel) are read and written as contiguous runs, and
// component m of K9's per-voxel record (8 corner densities, colour, normal,
// priority). The clamp mask (sh.hpp:66-74) comes from K1's clamped colour;
// lanes 0..7 add the normal chain (field.hpp:158-170) to
// their corner and issue the voxel's 8 pool atomics. Voxels outside `pre`
// leave at once (their group only zeroes SH gradients when not accumulating).
// The loads of one voxel's epilogue, issued together before any use: the
// kernel is latency-bound (ncu: 20 of 28 cycles per instruction waiting on
// L1TEX), so every independent load goes out in one round trip instead of
// rects -> record -> colour -> corner index -> priority in sequence.
struct EpiLoads {
    float gvm;      // K9's record, component m
    float4 d;       // sh_eval direction
    float4 rgb;     // K1's clamped colour (clamp mask)
    uint32_t ci;    // corner index m (lanes 0..7)
    float pr;       // priority (lane 14)
    float o0, o1, o2;  // SH gradients so far (accumulating backward)
};

__device__ __forceinline__ EpiLoads epilogue_load(const EpilogueArgs& a, uint64_t v, int m) {
    const int nb = (a.sh_degree + 1) * (a.sh_degree + 1);
    EpiLoads L;
    L.gvm = a.g_vox[16 * v + m];
    L.d = __ldg(a.view_dir + v);
    L.rgb = a.sh ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(a.records + v * kRecordF4 + 4);
    L.ci = m < 8 ? __ldg(a.corner_index + 8 * v + m) : 0u;
    L.pr = m == 14 ? a.g_priority[v] : 0.f;
    L.o0 = L.o1 = L.o2 = 0.f;
    if (a.accumulate && m < nb) {
        const float* o = a.g_sh + v * uint64_t(a.sh_stride) + 3 * m;
        L.o0 = o[0], L.o1 = o[1], L.o2 = o[2];
    }
    return L;
}

// Corner m's share of the normal chain (field.hpp:158-170).
__device__ __forceinline__ float normal_chain(const float4* rec, float dn0, float dn1, float dn2, int m) {
    const float dn[3] = {dn0, dn1, dn2};
    float V[8];
    trilinear_corners(rec[2], rec[3], V);
    float gV[8];
    voxel_normal_backward(V, dn, gV);
    float g = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) g = (m == c) ? gV[c] : g;
    return g;
}

// One visible voxel (all 16 lanes of its group present).
__device__ __forceinline__ void epilogue_visible(const EpilogueArgs& a, uint64_t v, int m, unsigned gmask,
                                                 const EpiLoads& L) {
    const int nb = (a.sh_degree + 1) * (a.sh_degree + 1);
    float* gsh = a.g_sh + v * uint64_t(a.sh_stride);
    // K9's record of this voxel: lane m holds component m (coalesced 64 B);
    // consumed here and left zero for the next backward
    const float gvm = L.gvm;
    // sh_eval direction exactly as K1 used it (raster.cpp:195-196): the
    // forward colour and this clamp mask see identical floats
    float b[16] = {};  // lanes m >= (d+1)^2 read zeros, not stale registers
    sh_basis(a.sh_degree, L.d.x, L.d.y, L.d.z, b);
    float bm = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) bm = (m == i) ? b[i] : bm;
    // The clamp mask (sh.hpp:72-74) is raw > 0 per channel, i.e. the
    // forward's clamped colour max(0, raw) > 0: read from K1's record (16 B,
    // one sector for the 16 lanes) instead of re-evaluating the SH sum from
    // the coefficients (192 B per voxel), and exactly the clamp the forward
    // applied.
    float4 rgb = L.rgb;
    if (a.sh) {
        // the pools changed since the forward (svr_scene_set_params): the
        // reference's mask reads the pools it is given (raster.cpp:414), so
        // evaluate raw from the current coefficients, reduced over the lanes
        float c0 = 0.f, c1 = 0.f, c2 = 0.f;
        if (m < nb) {
            const float* co = a.sh + v * uint64_t(a.sh_stride) + 3 * m;
            c0 = co[0], c1 = co[1], c2 = co[2];
        }
        float r0 = bm * c0, r1 = bm * c1, r2 = bm * c2;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            r0 += __shfl_xor_sync(gmask, r0, o, 16);
            r1 += __shfl_xor_sync(gmask, r1, o, 16);
            r2 += __shfl_xor_sync(gmask, r2, o, 16);
        }
        rgb = make_float4(r0, r1, r2, 0.f);
    }
    const float gc0 = __shfl_sync(gmask, gvm, 8, 16), gc1 = __shfl_sync(gmask, gvm, 9, 16),
                gc2 = __shfl_sync(gmask, gvm, 10, 16);
    const float dn0 = __shfl_sync(gmask, gvm, 11, 16), dn1 = __shfl_sync(gmask, gvm, 12, 16),
                dn2 = __shfl_sync(gmask, gvm, 13, 16);
    // reset the record only now: a store right behind the load of the same
    // address stalls the thread until the load returns (0.84 vs 0.16 ms)
    a.g_vox[16 * v + m] = 0.f;
    const float g0 = rgb.x > 0.f ? gc0 : 0.f;
    const float g1 = rgb.y > 0.f ? gc1 : 0.f;
    const float g2 = rgb.z > 0.f ? gc2 : 0.f;
    if (m < nb) {
        float* o = gsh + 3 * m;
        if (a.accumulate) {
            o[0] = L.o0 + bm * g0;
            o[1] = L.o1 + bm * g1;
            o[2] = L.o2 + bm * g2;
        } else {
            o[0] = bm * g0;
            o[1] = bm * g1;
            o[2] = bm * g2;
        }
    }
    if (m == 14) a.g_priority[v] = L.pr + gvm;
    if (m >= 8) return;
    // corner m: the compositing sum plus the normal chain (field.hpp:158-170)
    float gd = gvm;
    if (dn0 != 0.f || dn1 != 0.f || dn2 != 0.f) gd += normal_chain(a.records + v * kRecordF4, dn0, dn1, dn2, m);
    if (gd != 0.f) atomicAdd(a.g_density + L.ci, gd);
}

#ifndef SVR_EPI_VPG
#define SVR_EPI_VPG 1  // voxels per group with all loads issued first (2 / 4: config 3 epilogue 167 -> 203-229 us)
#endif
#ifndef SVR_EPI_MINB
#define SVR_EPI_MINB 6  // 40 registers (loads hoisted: config 3 epilogue 199 -> 167 us; 8 CTAs/32 registers spill)
#endif
__global__ void __launch_bounds__(256, SVR_EPI_MINB) voxel_epilogue_kernel(EpilogueArgs a) {
    pdl_enter();
    const int m = threadIdx.x & 15;
    const unsigned gmask = 0xffffu << (threadIdx.x & 16);  // this voxel's 16 lanes
    if (a.list) {  // training frames: K1's list of the voxels in `pre`, grid-stride
        const uint64_t nl = *a.n_list;
        for (uint64_t i = uint64_t(blockIdx.x) * 16u + (threadIdx.x >> 4); i < nl;
             i += uint64_t(gridDim.x) * 16u) {
            const uint64_t v = __ldg(a.list + i);
            epilogue_visible(a, v, m, gmask, epilogue_load(a, v, m));
        }
        return;
    }
    // SVR_EPI_VPG voxels per 16-lane group, all their loads issued before
    // the first one is processed; the record loads go out with the `pre`
    // rectangle (98 % of config-3 voxels are visible; an invisible voxel's
    // record is zero and unused)
    constexpr int G = SVR_EPI_VPG;
    const uint64_t v0 = uint64_t(blockIdx.x) * (16u * G) + (threadIdx.x >> 4);
    int4 r[G];
    EpiLoads L[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const uint64_t v = v0 + 16u * j;
        r[j] = v < a.n ? a.rects[v] : make_int4(0, -1, 0, -1);
        if (v < a.n) L[j] = epilogue_load(a, v, m);
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const uint64_t v = v0 + 16u * j;
        if (v >= a.n) continue;
        if (!(r[j].y >= r[j].x)) {  // not in `pre`: no gradient
            if (!a.accumulate)
                for (int i = m; i < a.sh_stride; i += 16) a.g_sh[v * uint64_t(a.sh_stride) + i] = 0.f;
            continue;
        }
        epilogue_visible(a, v, m, gmask, L[j]);
    }
}

inline unsigned blocks_for(uint64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

void launch_lift(const TapTable& t, const float* g, int channels, int W, float* out, int sw,
                 int sh, cudaStream_t st) {
    dim3 grid(blocks_for(sw, 128), sh);
    launch_pdl(lift_kernel, grid, 128, 0, st, t, g, channels, W, out, sw, sh);
    SVR_LAUNCH("lift_kernel");
}

void launch_l1_loss(const float* color, const float* gt, uint64_t n, float* d_color, float* loss,
                    cudaStream_t st) {
    if (loss) SVR_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), st));
    unsigned blocks = unsigned(std::min<uint64_t>(blocks_for(n, 256), 148 * 8));
    launch_pdl(l1_kernel, blocks, 256, 0, st, color, gt, n, 1.0f / float(n), d_color, loss);
    SVR_LAUNCH("l1_kernel");
}

void launch_composite_backward(const DevCamera& cam, const BackwardArgs& a, cudaStream_t st) {
    const unsigned ntiles = unsigned(cam.ntx * cam.nty);
    const bool upc = a.d_weight || a.d_voxel_color;
    switch (a.K) {
        case 1:
            if (upc) launch_pdl(composite_backward_kernel<1, true>, ntiles, 256, 0, st, cam, a);
            else launch_pdl(composite_backward_kernel<1, false>, ntiles, 256, 0, st, cam, a);
            break;
        case 2:
            if (upc) launch_pdl(composite_backward_kernel<2, true>, ntiles, 256, 0, st, cam, a);
            else launch_pdl(composite_backward_kernel<2, false>, ntiles, 256, 0, st, cam, a);
            break;
        case 3:
            if (upc) launch_pdl(composite_backward_kernel<3, true>, ntiles, 256, 0, st, cam, a);
            else launch_pdl(composite_backward_kernel<3, false>, ntiles, 256, 0, st, cam, a);
            break;
        default:
            throw Error(SVR_ERR_INVALID_ARGUMENT, "rasterizer sample count K must be in {1,2,3}");
    }
    SVR_LAUNCH("composite_backward_kernel");
}

void launch_ray_losses(const DevCamera& cam, const RayLossArgs& a, cudaStream_t st) {
    const uint64_t npix = uint64_t(cam.W) * cam.H;
    if (a.w_T != 0.0) {
        launch_pdl(ray_loss_T_kernel, unsigned((npix + 255) / 256), 256, 0, st, a, npix);
        SVR_LAUNCH("ray_loss_T_kernel");
    }
    if (a.w_dist == 0.0 && a.w_R == 0.0) return;
#ifndef SVR_RL_LANES
#define SVR_RL_LANES 8
#endif
    constexpr int L = SVR_RL_LANES;  // lanes per pixel
    const dim3 grid(unsigned((cam.W + 256 / L - 1) / (256 / L)), unsigned(cam.H));
    switch (a.K) {
        case 1: launch_pdl(ray_losses_kernel<1, L>, grid, 256, 0, st, cam, a); break;
        case 2: launch_pdl(ray_losses_kernel<2, L>, grid, 256, 0, st, cam, a); break;
        case 3: launch_pdl(ray_losses_kernel<3, L>, grid, 256, 0, st, cam, a); break;
        default: throw Error(SVR_ERR_INVALID_ARGUMENT, "rasterizer sample count K must be in {1,2,3}");
    }
    SVR_LAUNCH("ray_losses_kernel");
}

void launch_image_losses(const ImageLossArgs& a, cudaStream_t st) {
    const unsigned g = 148 * 8;
    launch_pdl(ssim_rows_kernel, g, 256, 0, st, a);
    SVR_LAUNCH("ssim_rows_kernel");
    launch_pdl(ssim_cols_kernel, g, 256, 0, st, a);
    SVR_LAUNCH("ssim_cols_kernel");
    if (!a.d_a || a.w_ssim == 0.0) return;
    launch_pdl(ssim_adj_cols_kernel, g, 256, 0, st, a);
    SVR_LAUNCH("ssim_adj_cols_kernel");
    launch_pdl(ssim_adj_rows_kernel, g, 256, 0, st, a);
    SVR_LAUNCH("ssim_adj_rows_kernel");
}

void launch_adam(const AdamArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    const unsigned blocks = unsigned(std::min<uint64_t>(blocks_for(a.n, 256), 148 * 16));
    launch_pdl(adam_kernel, blocks, 256, 0, st, a);
    SVR_LAUNCH("adam_kernel");
}

void launch_voxel_epilogue(const DevCamera& cam, const EpilogueArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    // with K1's visible list: a persistent grid (the list length lives on the device)
    launch_pdl(voxel_epilogue_kernel, a.list ? 148u * 16u : blocks_for(a.n, 16 * SVR_EPI_VPG), 256, 0, st, a);
    (void)cam;
    SVR_LAUNCH("voxel_epilogue_kernel");
}

}  // namespace svrb
