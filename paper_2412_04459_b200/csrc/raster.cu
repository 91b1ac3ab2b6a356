// raster.cu — forward path of the sparse-voxel rasterizer on sm_100a.
//
// Kernel map (reference → kernel):
//   K2 tile_setup      tile_sign_patterns (raster.cpp:120-142) for every tile
//                      + summed-area table of per-tile pattern counts
//   K1 preprocess      preprocess (raster.cpp:182-201): geometry_of, project_voxel
//                      (fp64 exact), density gather, sh_eval, voxel_normal; writes
//                      the 112-B voxel record and the voxel's entry count
//   K4 duplicate       build_sort_entries (raster.cpp:144-172) emission loop
//   K6 tile_ranges     the cursor scan of raster.cpp:238-245
//   K7 composite       tile loop raster.cpp:238-281 + CompositeCtx (17-61)
//   K8 downsample      AreaResampler::downsample (image.cpp:31-45)
#include <cuda_runtime.h>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {

namespace {

constexpr uint64_t kCodeMask48 = (uint64_t(1) << 48) - 1;

// ------------------------------------------------------------------- K2
__global__ void __launch_bounds__(1024) tile_setup_kernel(DevCamera cam, uint8_t* masks,
                                                          uint32_t* sat, FrameStatus* status) {
    const int ntx = cam.ntx, nty = cam.nty, ntiles = ntx * nty;
    const int sw = ntx + 1;
    __shared__ unsigned int s_or;
    if (threadIdx.x == 0) s_or = 0;
    __syncthreads();
    unsigned int local_or = 0;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        int tx = t % ntx, ty = t / ntx;
        uint32_t m = tile_sign_mask(cam, tx, ty);
        masks[t] = uint8_t(m);
        local_or |= m;
        sat[(ty + 1) * sw + tx + 1] = __popc(m);
    }
    for (int i = threadIdx.x; i < sw; i += blockDim.x) sat[i] = 0;
    for (int i = threadIdx.x; i <= nty; i += blockDim.x) sat[i * sw] = 0;
    atomicOr(&s_or, local_or);
    __syncthreads();
    for (int r = threadIdx.x + 1; r <= nty; r += blockDim.x) {
        uint32_t run = 0;
        for (int c = 1; c <= ntx; ++c) {
            run += sat[r * sw + c];
            sat[r * sw + c] = run;
        }
    }
    __syncthreads();
    for (int c = threadIdx.x + 1; c <= ntx; c += blockDim.x) {
        uint32_t run = 0;
        for (int r = 1; r <= nty; ++r) {
            run += sat[r * sw + c];
            sat[r * sw + c] = run;
        }
    }
    if (threadIdx.x == 0 && status) status->pattern_or = s_or;
}

__global__ void tile_masks_kernel(DevCamera cam, uint8_t* masks) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cam.ntx * cam.nty) return;
    masks[t] = uint8_t(tile_sign_mask(cam, t % cam.ntx, t / cam.ntx));
}

__device__ __forceinline__ uint32_t sat_rect(const uint32_t* sat, int ntx, int tx0, int tx1, int ty0,
                                             int ty1) {
    const int sw = ntx + 1;
    return sat[(ty1 + 1) * sw + tx1 + 1] - sat[ty0 * sw + tx1 + 1] - sat[(ty1 + 1) * sw + tx0] +
           sat[ty0 * sw + tx0];
}

// ------------------------------------------------------------------- K1
__global__ void __launch_bounds__(256) preprocess_kernel(DevCamera cam, PreprocessArgs a) {
    uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= a.n) return;
    const uint64_t path = a.paths[v];
    double center[3], size;
    voxel_geometry(path & kCodeMask48, int(path >> 48), a.bc, a.bsize, center, &size);
    Projection pr;
    bool vis = project_voxel(cam, center, size, a.near_plane, pr);
    a.rects[v] = make_int4(pr.tx0, pr.tx1, pr.ty0, pr.ty1);
    if (a.aabb) a.aabb[v] = make_double4(pr.x0, pr.x1, pr.y0, pr.y1);
    if (!vis) {
        a.counts[v] = 0;
        return;
    }
    a.counts[v] = sat_rect(a.tile_sat, cam.ntx, pr.tx0, pr.tx1, pr.ty0, pr.ty1);

    // Geometry relative to the camera, rounded once from the exact doubles.
    const double h = dmul(0.5, size);
    float4 r0, r1, r2, r3, r4, r5, r6;
    r0.x = float(dsub(dsub(center[0], h), cam.pos[0]));
    r0.y = float(dsub(dsub(center[1], h), cam.pos[1]));
    r0.z = float(dsub(dsub(center[2], h), cam.pos[2]));
    r0.w = float(1.0 / size);
    r1.x = float(dsub(dadd(center[0], h), cam.pos[0]));
    r1.y = float(dsub(dadd(center[1], h), cam.pos[1]));
    r1.z = float(dsub(dadd(center[2], h), cam.pos[2]));
    r1.w = __uint_as_float(uint32_t(v));
    // Screen AABB, rounded outward so the fp32 test is a superset.
    r2 = make_float4(__double2float_rd(pr.x0), __double2float_ru(pr.x1),
                     __double2float_rd(pr.y0), __double2float_ru(pr.y1));
    const uint4* ci4 = reinterpret_cast<const uint4*>(a.corner_index + 8 * v);
    uint4 c0 = ci4[0], c1 = ci4[1];
    float V[8] = {a.density[c0.x], a.density[c0.y], a.density[c0.z], a.density[c0.w],
                  a.density[c1.x], a.density[c1.y], a.density[c1.z], a.density[c1.w]};
    r3 = make_float4(V[0], V[1], V[2], V[3]);
    r4 = make_float4(V[4], V[5], V[6], V[7]);
    // sh_eval(normalized(center - cam.pos)) (raster.cpp:195-196, sh.hpp:48-58)
    double dx = dsub(center[0], cam.pos[0]), dy = dsub(center[1], cam.pos[1]),
           dz = dsub(center[2], cam.pos[2]);
    double nrm = sqrt(dx * dx + dy * dy + dz * dz);
    float ux = 0.f, uy = 0.f, uz = 0.f;
    if (nrm > 0.0) {
        ux = float(dx / nrm);
        uy = float(dy / nrm);
        uz = float(dz / nrm);
    }
    float b[16];
    int nb = sh_basis(a.sh_degree, ux, uy, uz, b);
    const float* co = a.sh + v * uint64_t(a.sh_stride);
    float cr = 0.f, cg = 0.f, cb = 0.f;
    for (int m = 0; m < nb; ++m) {
        cr += b[m] * co[3 * m + 0];
        cg += b[m] * co[3 * m + 1];
        cb += b[m] * co[3 * m + 2];
    }
    r5 = make_float4(fmaxf(0.f, cr), fmaxf(0.f, cg), fmaxf(0.f, cb), 0.f);
    float n[3];
    voxel_normal(V, n);
    r6 = make_float4(n[0], n[1], n[2], 0.f);
    float4* rec = a.records + v * kRecordF4;
    rec[0] = r0;
    rec[1] = r1;
    rec[2] = r2;
    rec[3] = r3;
    rec[4] = r4;
    rec[5] = r5;
    rec[6] = r6;
}

// ------------------------------------------------------------------- K4
__global__ void __launch_bounds__(256) duplicate_kernel(DevCamera cam, uint64_t n,
                                                        const uint64_t* paths, const int4* rects,
                                                        const uint8_t* masks,
                                                        const uint32_t* counts,
                                                        const uint32_t* offsets, uint64_t* keys,
                                                        uint32_t* vals) {
    uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n || counts[v] == 0) return;
    const uint64_t code = paths[v] & kCodeMask48;
    const int4 r = rects[v];
    uint32_t o = offsets[v];
    for (int ty = r.z; ty <= r.w; ++ty)
        for (int tx = r.x; tx <= r.y; ++tx) {
            uint64_t tid = uint64_t(ty) * cam.ntx + tx;
            uint32_t m = masks[tid];
            while (m) {
                uint32_t s = __ffs(m) - 1;
                m &= m - 1;
                keys[o] = (tid << 48) | (code ^ (uint64_t(s) * kGroupOnes));
                vals[o] = (s << 29) | uint32_t(v);
                ++o;
            }
        }
}

// Same emission for an explicit `pre` list (svr_build_sort_entries).
__global__ void duplicate_list_kernel(DevCamera cam, uint64_t n, const uint32_t* vids,
                                      const uint64_t* codes, const int4* rects,
                                      const uint8_t* masks, const uint32_t* offsets,
                                      uint64_t* keys, uint32_t* vals) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t code = codes[i];
    const int4 r = rects[i];
    uint32_t o = offsets[i];
    for (int ty = r.z; ty <= r.w; ++ty)
        for (int tx = r.x; tx <= r.y; ++tx) {
            uint64_t tid = uint64_t(ty) * cam.ntx + tx;
            uint32_t m = masks[tid];
            while (m) {
                uint32_t s = __ffs(m) - 1;
                m &= m - 1;
                keys[o] = (tid << 48) | (code ^ (uint64_t(s) * kGroupOnes));
                vals[o] = (s << 29) | vids[i];
                ++o;
            }
        }
}

__global__ void entry_counts_kernel(DevCamera cam, uint64_t n, const int4* rects,
                                    const uint32_t* sat, uint32_t* counts) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 r = rects[i];
    counts[i] = (r.y < r.x || r.w < r.z) ? 0u : sat_rect(sat, cam.ntx, r.x, r.y, r.z, r.w);
}

// ------------------------------------------------------------------- K6
__global__ void tile_ranges_kernel(const uint64_t* keys, uint64_t n, uint2* ranges) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t t = uint32_t(keys[i] >> 48);
    if (i == 0 || uint32_t(keys[i - 1] >> 48) != t) ranges[t].x = uint32_t(i);
    if (i == n - 1 || uint32_t(keys[i + 1] >> 48) != t) ranges[t].y = uint32_t(i + 1);
}

// ------------------------------------------------------------------- K7
// One CTA per 16x16 tile, one thread per pixel. Voxel records of a batch of
// 256 entries are staged in shared memory (one 112-B record per thread,
// SoA by float4 slot so every read in the inner loop is a broadcast), the
// batch is walked front to back with exactly CompositeCtx::add's arithmetic
// in fp32, and the CTA exits as soon as every pixel terminated
// (__syncthreads_count as the block-wide vote).
template <int K, bool RECORD>
__global__ void __launch_bounds__(256) composite_kernel(DevCamera cam, CompositeArgs a) {
    __shared__ float4 s_rec[kRecordF4][256];
    __shared__ uint32_t s_sign[256];

    const int tile = blockIdx.x;
    const int tx = tile % cam.ntx, ty = tile / cam.ntx;
    const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < cam.W && py < cam.H;

    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const uint32_t my_sign = sign_bits(dd);
    const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
    const float ix = 1.0f / dx, iy = 1.0f / dy, iz = 1.0f / dz;
    const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));
    const float pcx = float(px) + 0.5f, pcy = float(py) + 0.5f;

    float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f, nx = 0.f, ny = 0.f, nz = 0.f, depth = 0.f;
    float median = -1.0f;
    uint32_t cnt = 0;
    bool done = !inside;
    const uint32_t slot = uint32_t(tile) * 256u + threadIdx.x;
    uint32_t rec_base = 0;
    if (RECORD) rec_base = inside ? a.pix_begin[slot] : 0u;

    const uint2 range = a.ranges[tile];
    const float thr = a.t_threshold;
    for (uint32_t start = range.x; start < range.y; start += 256) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t idx = start + threadIdx.x;
        if (idx < range.y) {
            uint32_t val = a.vals[idx];
            uint32_t vid = val & ((1u << 29) - 1u);
            s_sign[threadIdx.x] = val >> 29;
            const float4* rec = a.records + uint64_t(vid) * kRecordF4;
#pragma unroll
            for (int k = 0; k < kRecordF4; ++k) s_rec[k][threadIdx.x] = __ldg(rec + k);
        }
        __syncthreads();
        const int nb = int(min(256u, range.y - start));
        if (!done) {
            for (int j = 0; j < nb; ++j) {
                if (s_sign[j] != my_sign) continue;
                const float4 bb = s_rec[2][j];
                if (pcx < bb.x || pcx > bb.y || pcy < bb.z || pcy > bb.w) continue;
                const float4 lo = s_rec[0][j], hi = s_rec[1][j];
                float t0 = lo.x * ix, t1 = hi.x * ix;
                float ta = fminf(t0, t1), tb = fmaxf(t0, t1);
                t0 = lo.y * iy;
                t1 = hi.y * iy;
                ta = fmaxf(ta, fminf(t0, t1));
                tb = fminf(tb, fmaxf(t0, t1));
                t0 = lo.z * iz;
                t1 = hi.z * iz;
                ta = fmaxf(ta, fminf(t0, t1));
                tb = fminf(tb, fmaxf(t0, t1));
                if (!(ta <= tb && ta > 0.0f)) continue;
                // voxel_alpha (field.hpp:92-116), K-point midpoint quadrature
                const float4 va = s_rec[3][j], vb = s_rec[4][j];
                const float V[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
                const float seg = tb - ta;
                const float lk = seg * dnorm * (1.0f / K);
                float sa[K], tk[K];
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    tk[k] = ta + ((k + 0.5f) / K) * seg;
                    const float qx = (tk[k] * dx - lo.x) * lo.w;
                    const float qy = (tk[k] * dy - lo.y) * lo.w;
                    const float qz = (tk[k] * dz - lo.z) * lo.w;
                    const float act = explin(trilinear(V, qx, qy, qz));
                    sum += act;
                    sa[k] = 1.0f - fexp(-lk * act);
                }
                const float alpha = (K == 1) ? sa[0] : 1.0f - fexp(-lk * sum);
                // voxel_depth (field.hpp:173-181)
                float dvox = 0.f, Tk = 1.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dvox += Tk * sa[k] * tk[k];
                    Tk *= 1.0f - sa[k];
                }
                if (median < 0.0f) {
                    float Tf = T;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        Tf *= 1.0f - sa[k];
                        if (Tf < 0.5f) {
                            median = tk[k];
                            break;
                        }
                    }
                }
                const float w = T * alpha;
                if (!RECORD) {
                    const float4 col = s_rec[5][j], nor = s_rec[6][j];
                    cr += w * col.x;
                    cg += w * col.y;
                    cb += w * col.z;
                    nx += w * nor.x;
                    ny += w * nor.y;
                    nz += w * nor.z;
                    depth += T * dvox;
                    if (a.max_blend) atomicMax(a.max_blend + __float_as_uint(hi.w), __float_as_uint(w));
                } else {
                    a.contrib_entry[rec_base + cnt] = start + j;
                    a.contrib_T[rec_base + cnt] = T;
                }
                T *= 1.0f - alpha;
                ++cnt;
                if (T < thr) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (RECORD || !inside) return;
    // CompositeCtx::finish (raster.cpp:56-60)
    cr += T * a.bg[0];
    cg += T * a.bg[1];
    cb += T * a.bg[2];
    if (cnt == 0) depth = a.far_sentinel;
    if (median < 0.0f) median = a.far_sentinel;
    const uint64_t p = uint64_t(py) * cam.W + px;
    a.color[3 * p + 0] = cr;
    a.color[3 * p + 1] = cg;
    a.color[3 * p + 2] = cb;
    a.normal[3 * p + 0] = nx;
    a.normal[3 * p + 1] = ny;
    a.normal[3 * p + 2] = nz;
    a.depth[p] = depth;
    a.median[p] = median;
    a.tfin[p] = T;
    if (a.pix_count) a.pix_count[slot] = cnt;
}

// ------------------------------------------------------------------- K8
__global__ void downsample_kernel(TapTable t, const float* src, int ch, int sw, float* dst, int W,
                                  int H) {
    int x = blockIdx.x * blockDim.x + threadIdx.x;
    int y = blockIdx.y;
    if (x >= W || y >= H) return;
    float acc[3] = {0.f, 0.f, 0.f};
    for (int ty = t.ptr_y[y]; ty < t.ptr_y[y + 1]; ++ty) {
        const int sy = t.idx_y[ty];
        const float wy = t.w_y[ty];
        float mid[3] = {0.f, 0.f, 0.f};
        for (int tx = t.ptr_x[x]; tx < t.ptr_x[x + 1]; ++tx) {
            const float wx = t.w_x[tx];
            const float* s = src + (uint64_t(sy) * sw + t.idx_x[tx]) * ch;
            for (int c = 0; c < ch; ++c) mid[c] += wx * s[c];
        }
        for (int c = 0; c < ch; ++c) acc[c] += wy * mid[c];
    }
    for (int c = 0; c < ch; ++c) dst[(uint64_t(y) * W + x) * ch + c] = acc[c];
}

__global__ void tile_to_image_kernel(const uint32_t* tm, uint32_t* img, int sw, int sh, int ntx) {
    int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= sw || y >= sh) return;
    int tile = (y / kTile) * ntx + x / kTile;
    img[uint64_t(y) * sw + x] = tm[uint64_t(tile) * 256 + (y % kTile) * kTile + (x % kTile)];
}

__global__ void visible_flags_kernel(const int4* rects, uint64_t n, uint32_t* flags) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int4 r = rects[i];
    flags[i] = (r.y >= r.x) ? 1u : 0u;
}

// Re-derives each contribution's segment with the composite kernel's own
// fp32 slab test, widened to double for ForwardRecords::contribs.
__global__ void __launch_bounds__(256) contrib_segments_kernel(
    DevCamera cam, const uint2* ranges, const uint32_t* vals, const float4* records,
    const uint32_t* pix_count, const uint32_t* pix_begin, const uint32_t* contrib_entry,
    const uint32_t* pre_rank, uint32_t* contrib_pre, double* oa, double* ob) {
    const int tile = blockIdx.x;
    const int tx = tile % cam.ntx, ty = tile / cam.ntx;
    const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
    if (px >= cam.W || py >= cam.H) return;
    const uint32_t slot = uint32_t(tile) * 256u + threadIdx.x;
    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const float ix = 1.0f / float(dd[0]), iy = 1.0f / float(dd[1]), iz = 1.0f / float(dd[2]);
    const uint32_t n = pix_count[slot], base = pix_begin[slot];
    for (uint32_t c = 0; c < n; ++c) {
        uint32_t e = contrib_entry[base + c];
        uint32_t vid = vals[e] & ((1u << 29) - 1u);
        const float4 lo = records[uint64_t(vid) * kRecordF4 + 0];
        const float4 hi = records[uint64_t(vid) * kRecordF4 + 1];
        float t0 = lo.x * ix, t1 = hi.x * ix;
        float ta = fminf(t0, t1), tb = fmaxf(t0, t1);
        t0 = lo.y * iy;
        t1 = hi.y * iy;
        ta = fmaxf(ta, fminf(t0, t1));
        tb = fminf(tb, fmaxf(t0, t1));
        t0 = lo.z * iz;
        t1 = hi.z * iz;
        ta = fmaxf(ta, fminf(t0, t1));
        tb = fminf(tb, fmaxf(t0, t1));
        contrib_pre[base + c] = pre_rank[vid];
        oa[base + c] = ta;
        ob[base + c] = tb;
    }
}

__global__ void project_batch_kernel(DevCamera cam, uint64_t n, const double* centers,
                                     const double* sizes, double near_plane, uint8_t* visible,
                                     double* aabb, int* rect) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Projection pr;
    bool vis = project_voxel(cam, centers + 3 * i, sizes[i], near_plane, pr);
    visible[i] = vis ? 1 : 0;
    aabb[4 * i + 0] = pr.x0;
    aabb[4 * i + 1] = pr.x1;
    aabb[4 * i + 2] = pr.y0;
    aabb[4 * i + 3] = pr.y1;
    rect[4 * i + 0] = pr.tx0;
    rect[4 * i + 1] = pr.tx1;
    rect[4 * i + 2] = pr.ty0;
    rect[4 * i + 3] = pr.ty1;
}

inline unsigned blocks_for(uint64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

void launch_tile_setup(const DevCamera& cam, uint8_t* masks, uint32_t* sat, FrameStatus* status,
                       cudaStream_t st) {
    tile_setup_kernel<<<1, 1024, 0, st>>>(cam, masks, sat, status);
    SVR_LAUNCH("tile_setup_kernel");
}

void launch_tile_masks_only(const DevCamera& cam, uint8_t* masks, cudaStream_t st) {
    int n = cam.ntx * cam.nty;
    tile_masks_kernel<<<blocks_for(n, 256), 256, 0, st>>>(cam, masks);
    SVR_LAUNCH("tile_masks_kernel");
}

void launch_preprocess(const DevCamera& cam, const PreprocessArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    preprocess_kernel<<<blocks_for(a.n, 256), 256, 0, st>>>(cam, a);
    SVR_LAUNCH("preprocess_kernel");
}

void launch_duplicate(const DevCamera& cam, uint64_t n, const uint64_t* paths, const int4* rects,
                      const uint8_t* masks, const uint32_t* counts, const uint32_t* offsets,
                      uint64_t* keys, uint32_t* vals, cudaStream_t st) {
    if (n == 0) return;
    duplicate_kernel<<<blocks_for(n, 256), 256, 0, st>>>(cam, n, paths, rects, masks, counts,
                                                         offsets, keys, vals);
    SVR_LAUNCH("duplicate_kernel");
}

void launch_duplicate_list(const DevCamera& cam, uint64_t n, const uint32_t* vids,
                           const uint64_t* codes, const int4* rects, const uint8_t* masks,
                           const uint32_t* offsets, uint64_t* keys, uint32_t* vals,
                           cudaStream_t st) {
    if (n == 0) return;
    duplicate_list_kernel<<<blocks_for(n, 256), 256, 0, st>>>(cam, n, vids, codes, rects, masks,
                                                              offsets, keys, vals);
    SVR_LAUNCH("duplicate_list_kernel");
}

void launch_entry_counts(const DevCamera& cam, uint64_t n, const int4* rects,
                         const uint32_t* sat, uint32_t* counts, cudaStream_t st) {
    if (n == 0) return;
    entry_counts_kernel<<<blocks_for(n, 256), 256, 0, st>>>(cam, n, rects, sat, counts);
    SVR_LAUNCH("entry_counts_kernel");
}

void launch_tile_ranges(const uint64_t* keys, uint64_t n, uint2* ranges, int ntiles,
                        cudaStream_t st) {
    SVR_CUDA(cudaMemsetAsync(ranges, 0, size_t(ntiles) * sizeof(uint2), st));
    if (n == 0) return;
    tile_ranges_kernel<<<blocks_for(n, 256), 256, 0, st>>>(keys, n, ranges);
    SVR_LAUNCH("tile_ranges_kernel");
}

void launch_composite(const DevCamera& cam, const CompositeArgs& a, bool record_pass,
                      cudaStream_t st) {
    const unsigned ntiles = unsigned(cam.ntx * cam.nty);
#define SVR_COMPOSITE_CASE(KK)                                                        \
    case KK:                                                                          \
        if (record_pass)                                                              \
            composite_kernel<KK, true><<<ntiles, 256, 0, st>>>(cam, a);              \
        else                                                                          \
            composite_kernel<KK, false><<<ntiles, 256, 0, st>>>(cam, a);             \
        break;
    switch (a.K) {
        SVR_COMPOSITE_CASE(1)
        SVR_COMPOSITE_CASE(2)
        SVR_COMPOSITE_CASE(3)
        default:
            throw Error(SVR_ERR_INVALID_ARGUMENT, "rasterizer sample count K must be in {1,2,3}");
    }
#undef SVR_COMPOSITE_CASE
    SVR_LAUNCH("composite_kernel");
}

void launch_downsample(const TapTable& t, const float* src, int channels, int sw, float* dst,
                       int W, int H, cudaStream_t st) {
    dim3 grid(blocks_for(W, 128), H);
    downsample_kernel<<<grid, 128, 0, st>>>(t, src, channels, sw, dst, W, H);
    SVR_LAUNCH("downsample_kernel");
}

void launch_tile_to_image_u32(const uint32_t* tm, uint32_t* img, int sw, int sh, int ntx,
                              cudaStream_t st) {
    dim3 grid(blocks_for(sw, 128), sh);
    tile_to_image_kernel<<<grid, 128, 0, st>>>(tm, img, sw, sh, ntx);
    SVR_LAUNCH("tile_to_image_kernel");
}

void launch_visible_flags(const int4* rects, uint64_t n, uint32_t* flags, cudaStream_t st) {
    if (n == 0) return;
    visible_flags_kernel<<<blocks_for(n, 256), 256, 0, st>>>(rects, n, flags);
    SVR_LAUNCH("visible_flags_kernel");
}

void launch_contrib_segments(const DevCamera& cam, const uint2* ranges, const uint32_t* vals,
                             const float4* records, const uint32_t* pix_count,
                             const uint32_t* pix_begin, const uint32_t* contrib_entry,
                             const uint32_t* pre_rank, uint32_t* contrib_pre, double* a,
                             double* b, int ntiles, cudaStream_t st) {
    contrib_segments_kernel<<<ntiles, 256, 0, st>>>(cam, ranges, vals, records, pix_count,
                                                    pix_begin, contrib_entry, pre_rank,
                                                    contrib_pre, a, b);
    SVR_LAUNCH("contrib_segments_kernel");
}

void launch_project_batch(const DevCamera& cam, uint64_t n, const double* centers,
                          const double* sizes, double near_plane, uint8_t* visible,
                          double* aabb, int* rect, cudaStream_t st) {
    if (n == 0) return;
    project_batch_kernel<<<blocks_for(n, 128), 128, 0, st>>>(cam, n, centers, sizes, near_plane,
                                                             visible, aabb, rect);
    SVR_LAUNCH("project_batch_kernel");
}

}  // namespace svrb
