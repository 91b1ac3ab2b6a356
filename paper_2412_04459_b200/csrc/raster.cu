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
// Single CTA: per-tile sign-pattern masks (fp64, bit-exact) and the
// summed-area table of their popcounts, built in shared memory (one
// warp-parallel row scan, then column sums), so a voxel's entry count is
// four table reads whatever its tile rectangle (near-plane straddlers cover
// the whole image).
constexpr int kSatSmemMax = 48 * 1024;  // u32 entries that fit the dynamic smem budget

__global__ void __launch_bounds__(1024) tile_setup_kernel(DevCamera cam, uint8_t* masks,
                                                          uint32_t* sat, FrameStatus* status,
                                                          int use_smem, int2* rowspan) {
    pdl_enter();
    extern __shared__ uint32_t s_sat[];
    const int ntx = cam.ntx, nty = cam.nty, ntiles = ntx * nty;
    const int sw = ntx + 1, ncell = sw * (nty + 1);
    // CTA 0: popcount table; CTA 1 + s (rank-ordered emission): table of bit s
    const int b = blockIdx.x;
    sat += size_t(b) * ncell;
    uint32_t* t = use_smem ? s_sat : sat;
    __shared__ unsigned int s_or;
    if (threadIdx.x == 0) s_or = 0;
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) t[i] = 0;
    __syncthreads();
    unsigned int local_or = 0;
    for (int k = threadIdx.x; k < ntiles; k += blockDim.x) {
        const int tx = k % ntx, ty = k / ntx;
        const uint32_t m = masks[k];  // tile_masks_kernel, launched just before
        local_or |= m;
        t[(ty + 1) * sw + tx + 1] = b == 0 ? __popc(m) : ((m >> (b - 1)) & 1u);
    }
    atomicOr(&s_or, local_or);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // row prefix sums: one warp per row, 32 columns at a time
    for (int r = warp + 1; r <= nty; r += nwarps) {
        uint32_t carry = 0;
        for (int c0 = 1; c0 <= ntx; c0 += 32) {
            const int c = c0 + lane;
            uint32_t v = c <= ntx ? t[r * sw + c] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += n;
            }
            if (c <= ntx) t[r * sw + c] = v + carry;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    // column prefix sums: one warp per column, 32 rows at a time (a column's
    // cells are sw words apart, sw odd for even ntx: no bank conflicts)
    for (int c = warp + 1; c <= ntx; c += nwarps) {
        uint32_t carry = 0;
        for (int r0 = 1; r0 <= nty; r0 += 32) {
            const int r = r0 + lane;
            uint32_t v = r <= nty ? t[r * sw + c] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += n;
            }
            if (r <= nty) t[r * sw + c] = v + carry;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    if (use_smem)
        for (int i = threadIdx.x; i < ncell; i += blockDim.x) sat[i] = t[i];
    if (threadIdx.x == 0 && status && b == 0) status->pattern_or = s_or;
    // per-pattern tables: the row span of pattern b-1 (the pattern regions are
    // convex in the image, so a row's tiles with bit s are nearly always one
    // run): {lo, hi}, {1, 0} when empty, {-1, -1} when not one run
    // one warp per row: ballots over 32 tiles at a time give the first and
    // last tile holding pattern b-1 and their count
    if (b > 0 && rowspan)
        for (int ty = warp; ty < nty; ty += nwarps) {
            int lo = ntx, hi = -1, cnt = 0;
            for (int tx0 = 0; tx0 < ntx; tx0 += 32) {
                const int tx = tx0 + lane;
                const unsigned bal =
                    __ballot_sync(0xffffffffu, tx < ntx && ((masks[ty * ntx + tx] >> (b - 1)) & 1u));
                if (bal) {
                    lo = min(lo, tx0 + __ffs(bal) - 1);
                    hi = tx0 + 31 - __clz(bal);
                    cnt += __popc(bal);
                }
            }
            if (lane == 0)
                rowspan[(b - 1) * nty + ty] = cnt == 0 ? make_int2(1, 0)
                                              : cnt == hi - lo + 1 ? make_int2(lo, hi) : make_int2(-1, -1);
        }
}

__global__ void tile_masks_kernel(DevCamera cam, uint8_t* masks) {
    pdl_enter();
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
// 128 threads = 4 warps, one voxel per thread. A conservative fp32 test first
// drops the voxels the exact fp64 projection would certainly cull. For scenes
// whose voxel order is not spatially coherent, that test runs in its own pass
// (precull_kernel) and K1 walks the worklist of survivors (a.order), so a
// warp's lanes are not split between culled and projected voxels. In scene
// order, the 96-B records of the CTA's visible voxels are staged in shared
// memory and written back as contiguous runs.
constexpr int kPreThreads = 128;
#ifndef SVR_PRE_MINB
#define SVR_PRE_MINB 6
#endif

// K1a for scenes stored out of spatial order: voxels the fp32 pre-test
// certainly culls get their (empty) outputs here, in scene order (coalesced);
// the others are appended to a worklist (warp-aggregated) that K1 then
// walks, so its warps carry no culled lanes.
__global__ void __launch_bounds__(256) precull_kernel(DevCamera cam, PreprocessArgs a, uint32_t* work,
                                                      unsigned int* n_work) {
    pdl_enter();
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool keep = false;
    if (v < a.n) {
        const uint64_t path = a.paths[v];
        double center[3], size;
        voxel_geometry(path & kCodeMask48, int(path >> 48), a.bc, a.bsize, center, &size);
        keep = !surely_culled(cam, center, size, a.near_plane, a.cull);
        if (!keep) {
            a.rects[v] = make_int4(0, -1, 0, -1);
            a.counts[v] = 0u;
            if (a.aabb) a.aabb[v] = make_double4(0.0, 0.0, 0.0, 0.0);
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (m == 0) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(n_work, unsigned(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (keep) work[base + __popc(m & ((1u << lane) - 1u))] = uint32_t(v);
}

__global__ void __launch_bounds__(kPreThreads, SVR_PRE_MINB) preprocess_kernel(DevCamera cam, PreprocessArgs a) {
    pdl_enter();
    extern __shared__ float4 smem4[];
    float4* s_rec = smem4;
    const uint64_t v0 = uint64_t(blockIdx.x) * kPreThreads;
    const uint64_t n_items = a.n_order ? uint64_t(*a.n_order) : a.n;  // worklist: live length
    if (v0 >= n_items) return;
    const bool valid = v0 + threadIdx.x < n_items;
    const uint64_t v = a.order ? (valid ? uint64_t(__ldg(a.order + v0 + threadIdx.x)) : a.n)
                               : v0 + threadIdx.x;

    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0, r3 = r0, r4 = r0, r5 = r0;  // r0.w = 0: not visible
    if (valid) {
        const uint64_t path = a.paths[v];
        double center[3], size;
        voxel_geometry(path & kCodeMask48, int(path >> 48), a.bc, a.bsize, center, &size);
        Projection pr;
        bool vis = false;
        if (!a.n_order && surely_culled(cam, center, size, a.near_plane, a.cull)) {
            pr.tx0 = pr.ty0 = 0;  // a fresh PreVoxel, as project_voxel leaves a culled one
            pr.tx1 = pr.ty1 = -1;
            pr.x0 = pr.x1 = pr.y0 = pr.y1 = 0.0;
            pr.straddles = false;
        } else {
            vis = project_voxel(cam, center, size, a.near_plane, pr);
        }
        a.rects[v] = make_int4(pr.tx0, pr.tx1, pr.ty0, pr.ty1);
        if (a.aabb) a.aabb[v] = make_double4(pr.x0, pr.x1, pr.y0, pr.y1);
        a.counts[v] = vis ? sat_rect(a.tile_sat, cam.ntx, pr.tx0, pr.tx1, pr.ty0, pr.ty1) : 0u;
        if (vis) {
            // Geometry relative to the camera, rounded once from the exact doubles.
            const double h = dmul(0.5, size);
            r0.x = float(dsub(dsub(center[0], h), cam.pos[0]));
            r0.y = float(dsub(dsub(center[1], h), cam.pos[1]));
            r0.z = float(dsub(dsub(center[2], h), cam.pos[2]));
            r0.w = float(size);
            // Screen AABB, rounded outward so the fp32 test is a superset;
            // empty for near-plane voxels no image ray can reach (their
            // entries stay; the compositing warps skip them at the AABB test).
            r1 = make_float4(__double2float_rd(pr.x0), __double2float_ru(pr.x1),
                             __double2float_rd(pr.y0), __double2float_ru(pr.y1));
            if (pr.straddles && box_outside_image_frustum(cam, center, size))
                r1 = make_float4(1.f, 0.f, 1.f, 0.f);
            const uint4* ci4 = reinterpret_cast<const uint4*>(a.corner_index + 8 * v);
            const uint4 c0 = __ldg(ci4), c1 = __ldg(ci4 + 1);
            float V[8] = {__ldg(a.density + c0.x), __ldg(a.density + c0.y), __ldg(a.density + c0.z),
                          __ldg(a.density + c0.w), __ldg(a.density + c1.x), __ldg(a.density + c1.y),
                          __ldg(a.density + c1.z), __ldg(a.density + c1.w)};
            float cf[8];
            trilinear_coeffs(V, cf);
            pack_coeffs(cf, r2, r3);
            // sh_eval(normalized(center - cam.pos)) (raster.cpp:195-196, sh.hpp:48-58)
            const double dx = dsub(center[0], cam.pos[0]), dy = dsub(center[1], cam.pos[1]),
                         dz = dsub(center[2], cam.pos[2]);
            const double nrm = sqrt(dx * dx + dy * dy + dz * dz);
            float ux = 0.f, uy = 0.f, uz = 0.f;
            if (nrm > 0.0) {
                ux = float(dx / nrm);
                uy = float(dy / nrm);
                uz = float(dz / nrm);
            }
            if (a.view_dir) a.view_dir[v] = make_float4(ux, uy, uz, 0.f);
            float b[16];
            const int nb = sh_basis(a.sh_degree, ux, uy, uz, b);
            float cr = 0.f, cg = 0.f, cb = 0.f;
            const float* co = a.sh + v * uint64_t(a.sh_stride);
            if (a.sh_stride == 48) {
                // degree 3: 12 aligned 16-B loads of this voxel's 192 B
                const float4* c4 = reinterpret_cast<const float4*>(co);
#pragma unroll
                for (int q = 0; q < 12; ++q) {
                    const float4 t = __ldg(c4 + q);
                    const float e4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int e = 4 * q + j, m = e / 3, ch = e - 3 * (e / 3);
                        const float c = b[m] * e4[j];
                        if (ch == 0) cr += c;
                        else if (ch == 1) cg += c;
                        else cb += c;
                    }
                }
            } else {
                for (int m = 0; m < nb; ++m) {
                    cr += b[m] * __ldg(co + 3 * m + 0);
                    cg += b[m] * __ldg(co + 3 * m + 1);
                    cb += b[m] * __ldg(co + 3 * m + 2);
                }
            }
            r4 = make_float4(fmaxf(0.f, cr), fmaxf(0.f, cg), fmaxf(0.f, cb), __uint_as_float(uint32_t(v)));
            float n[3];
            voxel_normal(V, n);
            r5 = make_float4(n[0], n[1], n[2], float(1.0 / size));
        }
    }
    if (a.vis_list) {  // training frames: list the voxels in `pre` for the epilogue
        const bool in_pre = valid && r0.w > 0.f;
        const unsigned vm = __ballot_sync(0xffffffffu, in_pre);
        if (vm) {
            const int ln = threadIdx.x & 31;
            unsigned base = 0;
            if (ln == __ffs(vm) - 1) base = atomicAdd(a.n_vis_list, unsigned(__popc(vm)));
            base = __shfl_sync(0xffffffffu, base, __ffs(vm) - 1);
            if (in_pre) a.vis_list[base + __popc(vm & ((1u << ln) - 1u))] = uint32_t(v);
        }
    }
    if (a.order) {  // worklist order: each thread stores its own record
        if (valid && r0.w > 0.f) {
            float4* dst = a.records + v * kRecordF4;
            dst[0] = r0;
            dst[1] = r1;
            dst[2] = r2;
            dst[3] = r3;
            dst[4] = r4;
            dst[5] = r5;
        }
        return;
    }
    // Records of visible voxels only (nothing reads the others): staged in
    // shared memory and written back as contiguous runs.
    __shared__ uint8_t s_vis[kPreThreads];
    float4* sr = s_rec + threadIdx.x * kRecordF4;
    sr[0] = r0;
    sr[1] = r1;
    sr[2] = r2;
    sr[3] = r3;
    sr[4] = r4;
    sr[5] = r5;
    const bool my_vis = valid && r0.w > 0.f;  // size > 0 marks a visible voxel's record
    s_vis[threadIdx.x] = my_vis;
    const bool all_vis = __syncthreads_and(my_vis || !valid);
    const int nblk = v0 < a.n ? int(min(uint64_t(kPreThreads), a.n - v0)) : 0;
    float4* dst = a.records + v0 * kRecordF4;
    if (all_vis) {
        for (int i = threadIdx.x; i < nblk * kRecordF4; i += kPreThreads) dst[i] = s_rec[i];
    } else {
        for (int i = threadIdx.x; i < nblk * kRecordF4; i += kPreThreads)
            if (s_vis[i / kRecordF4]) dst[i] = s_rec[i];
    }
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

// Packed variant of K4: one u64 per entry,
//   tile | top 3*Lmax bits of dir_dep_order(code, s) | s | vid,
// whose unsigned order is exactly the reference's (key, value) order
// (the dropped order bits are the sign pattern repeated, raster.cpp:165,
// octree.hpp:99-101). The kernel also accumulates the radix-sort digit
// histograms of every pass, so the sort needs no separate histogram read.
__device__ __forceinline__ uint64_t packed_key(PackedFormat fmt, const uint32_t* __restrict__ rank,
                                               uint64_t n, uint64_t v, uint64_t code, uint64_t tid,
                                               uint32_t sgn) {
    const uint64_t order = fmt.rank_bits
                               ? uint64_t(__ldg(rank + sgn * n + v))
                               : (code ^ (uint64_t(sgn) * kGroupOnes)) >> (48 - 3 * fmt.lmax);
    return (tid << fmt.tile_shift) | (order << (fmt.vb + 3)) | (uint64_t(sgn) << fmt.vb) | v;
}

// Voxels with more than this many entries (large or near-plane footprints,
// which get the whole screen) are emitted by duplicate_big_kernel.
constexpr uint32_t kBigEntries = 128;

__global__ void __launch_bounds__(256) duplicate_packed_kernel(
    DevCamera cam, uint64_t n, const uint64_t* __restrict__ paths, const int4* __restrict__ rects,
    const uint8_t* __restrict__ masks, const uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ offsets, PackedFormat fmt, const uint32_t* __restrict__ rank,
    uint64_t* __restrict__ keys, uint32_t* big, unsigned int* n_big, uint64_t cap) {
    pdl_enter();
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint32_t cnt = counts[v];
    if (cnt == 0) return;
    uint32_t o = offsets[v];
    if (uint64_t(o) + cnt > cap) return;  // deferred-E frame that outgrew its buffers (flagged)
    if (cnt > kBigEntries) {
        big[atomicAdd(n_big, 1u)] = uint32_t(v);
        return;
    }
    const uint64_t code = paths[v] & kCodeMask48;
    const int4 r = rects[v];
    for (int ty = r.z; ty <= r.w; ++ty)
        for (int tx = r.x; tx <= r.y; ++tx) {
            const uint64_t tid = uint64_t(ty) * cam.ntx + tx;
            uint32_t m = masks[tid];
            while (m) {
                const uint32_t sgn = __ffs(m) - 1;
                m &= m - 1;
                keys[o++] = packed_key(fmt, rank, n, v, code, tid, sgn);
            }
        }
}

// One CTA per large voxel (grid-stride over the list): warp w emits rows
// ty0 + w, ty0 + w + 8, ...; a row starts at the voxel's offset plus the
// SAT count of the rect rows above it, and lanes place their tile's
// patterns by a warp prefix sum, so the reference emission order
// (vid, ty, tx, s) is kept exactly.
__global__ void __launch_bounds__(256) duplicate_big_kernel(
    DevCamera cam, uint64_t n, const uint64_t* __restrict__ paths, const int4* __restrict__ rects,
    const uint8_t* __restrict__ masks, const uint32_t* __restrict__ offsets,
    const uint32_t* __restrict__ tile_sat, PackedFormat fmt, const uint32_t* __restrict__ rank,
    uint64_t* __restrict__ keys, const uint32_t* __restrict__ big,
    const unsigned int* __restrict__ n_big) {
    pdl_enter();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nb = *n_big;
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const uint64_t v = big[b];
        const uint64_t code = paths[v] & kCodeMask48;
        const int4 r = rects[v];
        const uint32_t o0 = offsets[v];
        for (int ty = r.z + warp; ty <= r.w; ty += 8) {
            uint32_t o = o0 + (ty > r.z ? sat_rect(tile_sat, cam.ntx, r.x, r.y, r.z, ty - 1) : 0u);
            for (int tx0 = r.x; tx0 <= r.y; tx0 += 32) {
                const int tx = tx0 + lane;
                const uint64_t tid = uint64_t(ty) * cam.ntx + tx;
                uint32_t m = tx <= r.y ? uint32_t(masks[tid]) : 0u;
                const uint32_t c = __popc(m);
                uint32_t incl = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += y;
                }
                uint32_t at = o + incl - c;
                while (m) {
                    const uint32_t sgn = __ffs(m) - 1;
                    m &= m - 1;
                    keys[at++] = packed_key(fmt, rank, n, v, code, tid, sgn);
                }
                o += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
    }
}

// Rank-ordered K4. Every (sign pattern s, voxel v) pair has a scene-constant
// Morton rank r = rank[s*n + v] (build_morton_rank), and the reference's
// within-tile order is ascending r. K4a writes each pair's entry count at
// its rank, pc[r] = #tiles of v's rectangle whose mask holds s (per-pattern
// SATs); an exclusive scan of pc over r gives every pair the offset of its
// entries in RANK order; K4b emits them there. The keys therefore come out
// sorted by everything below the tile bits, and a stable sort on the tile
// bits alone (2 radix passes at 1024^2 instead of 5) yields the reference's
// (tile, key, value) order (raster.cpp:174-178) exactly.
__device__ __forceinline__ uint64_t ranked_key(PackedFormat fmt, uint64_t tid, uint64_t r, uint32_t s,
                                               uint64_t v) {
    return (tid << fmt.tile_shift) | (r << (fmt.vb + 3)) | (uint64_t(s) << fmt.vb) | v;
}

__global__ void __launch_bounds__(256) pair_counts_kernel(
    DevCamera cam, uint64_t n, const uint32_t* __restrict__ counts, const int4* __restrict__ rects,
    const uint32_t* __restrict__ sat, FrameStatus* __restrict__ status,
    const uint32_t* __restrict__ rank, uint32_t* __restrict__ pc, uint32_t* __restrict__ block_sums,
    HugePairs huge) {
    pdl_enter();
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n || counts[v] == 0) return;
    const int ncell = (cam.ntx + 1) * (cam.nty + 1);
    const int4 r = rects[v];
    uint32_t pat = status->pattern_or;
    while (pat) {
        const uint32_t s = __ffs(pat) - 1;
        pat &= pat - 1;
        const uint32_t c = sat_rect(sat + size_t(1 + s) * ncell, cam.ntx, r.x, r.y, r.z, r.w);
        if (!c) continue;
        const uint32_t rk = __ldg(rank + s * n + v);
        if (huge.min && c >= huge.min) {
            const uint32_t slot = atomicAdd(&status->n_huge_pairs, 1u);
            if (huge.divert && slot < huge.cap) {  // merged per tile later, no entries now
                huge.keys[slot] = rk;
                huge.vals[slot] = (s << 29) | uint32_t(v);
                atomicAdd(&status->n_huge_entries, (unsigned long long)c);
                continue;
            }
        }
        pc[rk] = c;
        if (block_sums) {
            // the scan's block sums directly (no reduce pass over the 8n
            // counts): lanes adding to the same rank block combine first
            const uint32_t blk = rk / kScanChunk;
            const unsigned peers = __match_any_sync(__activemask(), blk);
            const uint32_t sum = __reduce_add_sync(peers, c);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(block_sums + blk, sum);
        }
    }
}

// ---- huge pairs: per-tile merge instead of duplicate + sort ----------------
// (1) every listed pair adds its tile rectangle to a per-pattern 2D
// difference array; (2) one CTA integrates them, counts per tile the pairs
// whose pattern the tile holds (exactly the entries the reference emits for
// them there, raster.cpp:155-170), adds the tile's sorted small entries and
// scans the totals into the final tile ranges; (3) per tile, the small keys
// (rank-ordered) and the huge pairs covering the tile (the rank-sorted list,
// filtered) are merged by rank straight into the final value array.
__global__ void huge_cover_kernel(DevCamera cam, HugePairs huge, const uint32_t* __restrict__ vals,
                                  const FrameStatus* __restrict__ status,
                                  const int4* __restrict__ rects, int* __restrict__ diff) {
    pdl_enter();
    const uint32_t nh = min(status->n_huge_pairs, huge.cap);
    const int sw = cam.ntx + 1, ncell = sw * (cam.nty + 1);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const uint32_t pv = vals[i];
        const int4 r = __ldg(rects + (pv & ((1u << 29) - 1u)));
        int* d = diff + size_t(pv >> 29) * ncell;
        atomicAdd(d + r.z * sw + r.x, 1);
        atomicAdd(d + r.z * sw + r.y + 1, -1);
        atomicAdd(d + (r.w + 1) * sw + r.x, -1);
        atomicAdd(d + (r.w + 1) * sw + r.y + 1, 1);
    }
}

constexpr int kMergeThreads = 1024;
__global__ void __launch_bounds__(kMergeThreads) huge_ranges_kernel(
    DevCamera cam, const FrameStatus* __restrict__ status, const uint8_t* __restrict__ masks,
    int* __restrict__ diff, const uint2* __restrict__ small_ranges, uint2* __restrict__ ranges,
    unsigned long long* n_total) {
    pdl_enter();
    __shared__ uint32_t s_cnt[4096];
    __shared__ uint32_t s_warp[kMergeThreads / 32];
    __shared__ int s_d[4225 + 65];  // one pattern's (ntx+1)(nty+1) difference cells
    const int ntiles = cam.ntx * cam.nty, sw = cam.ntx + 1, ncell = sw * (cam.nty + 1);
    for (int t = threadIdx.x; t < ntiles; t += kMergeThreads) s_cnt[t] = 0;
    const uint32_t pat = status->pattern_or;
    const bool fits = ncell <= 4225 + 65;
    for (int s = 0; s < 8; ++s) {
        if (!((pat >> s) & 1u)) continue;
        int* d = fits ? s_d : diff + size_t(s) * ncell;  // integrate in shared memory when it fits
        __syncthreads();
        if (fits)
            for (int i = threadIdx.x; i < ncell; i += kMergeThreads) s_d[i] = diff[size_t(s) * ncell + i];
        __syncthreads();
        for (int y = threadIdx.x; y <= cam.nty; y += kMergeThreads) {  // rows
            int run = 0;
            for (int x = 0; x < sw; ++x) run = (d[y * sw + x] += run);
        }
        __syncthreads();
        for (int x = threadIdx.x; x < sw; x += kMergeThreads) {  // columns
            int run = 0;
            for (int y = 0; y <= cam.nty; ++y) run = (d[y * sw + x] += run);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < ntiles; t += kMergeThreads)
            if ((masks[t] >> s) & 1u) s_cnt[t] += uint32_t(d[(t / cam.ntx) * sw + t % cam.ntx]);
    }
    __syncthreads();
    // totals per tile, exclusive scan over tiles (4 tiles per thread)
    uint32_t tot[4], sum = 0;
    const int t0 = threadIdx.x * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int t = t0 + k;
        uint32_t c = 0;
        if (t < ntiles) {
            const uint2 sr = small_ranges[t];
            c = s_cnt[t] + (sr.y > sr.x ? sr.y - sr.x : 0u);
        }
        tot[k] = c;
        sum += c;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = s_warp[lane];
        uint32_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        s_warp[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = s_warp[warp] + incl - sum;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int t = t0 + k;
        if (t < ntiles) ranges[t] = make_uint2(run, run + tot[k]);
        run += tot[k];
    }
    if (threadIdx.x == kMergeThreads - 1) *n_total = run;
}


// The huge list packed for the merge: {rank, value, tx0 | tx1 << 16,
// ty0 | ty1 << 16}, one 16-B load per pair instead of a key, a value and a
// dependent rectangle gather; twice: in rank order (R) and in (pattern, rank)
// order (S, whose per-pattern runs [sb[s], sb[8 + s]) serve the tile groups
// holding a single sign pattern: 3970 of 4096 tiles in config 4, a quarter
// of the pairs each).
__global__ void huge_pack_kernel(HugePairs huge, const uint64_t* __restrict__ rkeys,
                                 const uint32_t* __restrict__ rvals, const uint64_t* __restrict__ skeys_s,
                                 const uint32_t* __restrict__ svals, const FrameStatus* __restrict__ status,
                                 const int4* __restrict__ rects, uint4* __restrict__ packed_r,
                                 uint4* __restrict__ packed_s, uint32_t* __restrict__ sb) {
    pdl_enter();
    const uint32_t nh = min(status->n_huge_pairs, huge.cap);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nh; j += gridDim.x * blockDim.x) {
        uint32_t pv = rvals[j];
        int4 r = __ldg(rects + (pv & ((1u << 29) - 1u)));
        packed_r[j] = make_uint4(uint32_t(rkeys[j]), pv, uint32_t(r.x) | (uint32_t(r.y) << 16),
                                 uint32_t(r.z) | (uint32_t(r.w) << 16));
        pv = svals[j];
        r = __ldg(rects + (pv & ((1u << 29) - 1u)));
        packed_s[j] = make_uint4(uint32_t(skeys_s[j]), pv, uint32_t(r.x) | (uint32_t(r.y) << 16),
                                 uint32_t(r.z) | (uint32_t(r.w) << 16));
        const uint32_t s = pv >> 29;
        if (j == 0 || (svals[j - 1] >> 29) != s) sb[s] = j;
        if (j + 1 == nh || (svals[j + 1] >> 29) != s) sb[8 + s] = j + 1;
    }
}

// The list tiles [t0, t0 + G) merge from: the pattern's run of S when they
// all hold one and the same sign pattern, else all of R. Single tiles decide
// by their own mask (apos below uses that rule, and the group kernel only
// takes groups whose tiles all hold the same single pattern).
struct MergeList {
    const uint4* p;
    uint32_t lo, hi;
    bool single;
};
__device__ __forceinline__ MergeList merge_list(const DevCamera& cam, int t0, int G, const uint8_t* masks,
                                                const uint4* packed_r, const uint4* packed_s,
                                                const uint32_t* sb, uint32_t nh) {
    const int ntiles = cam.ntx * cam.nty;
    uint32_t pat = 0;
    for (int g = 0; g < G; ++g)
        if (t0 + g < ntiles) pat |= masks[t0 + g];
    if (__popc(pat) == 1) {
        const int s = __ffs(pat) - 1;
        return {packed_s, sb[s], max(sb[s], sb[8 + s]), true};
    }
    return {packed_r, 0u, nh, false};
}

// For every sorted small entry: how many pairs of its tile group's list rank
// below it (its place in that list), one binary search each.
__global__ void huge_apos_kernel(DevCamera cam, const uint64_t* __restrict__ skeys,
                                 const FrameStatus* __restrict__ status, uint64_t cap_small,
                                 PackedFormat fmt, HugePairs huge, const uint8_t* __restrict__ masks,
                                 const uint4* __restrict__ packed_r, const uint4* __restrict__ packed_s,
                                 const uint32_t* __restrict__ sb, uint32_t* __restrict__ apos) {
    pdl_enter();
    const uint64_t n = live_entries(cap_small, &status->n_entries);
    const uint32_t nh = min(status->n_huge_pairs, huge.cap);
    const uint64_t rmask = (uint64_t(1) << fmt.rank_bits) - 1;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = skeys[e];
        const uint32_t ra = uint32_t((k >> (fmt.vb + 3)) & rmask);
        const int tile = int(k >> fmt.tile_shift);
        const MergeList L = merge_list(cam, tile, 1, masks, packed_r, packed_s, sb, nh);
        uint32_t lo = L.lo, hi = L.hi;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&L.p[mid].x) < ra) lo = mid + 1;
            else hi = mid;
        }
        apos[e] = lo - L.lo;
    }
}

// One CTA per group of kMergeTiles consecutive tiles sharing one sign
// pattern (or per single tile otherwise), in steps of kMergeStep listed
// pairs (kMergeK consecutive per thread; the 16-B records serve all the
// group's tiles). Per tile: which pairs cover it (rectangle and the tile's
// sign patterns: exactly the reference's emission rule); block scans give
// each kept pair the kept pairs before it and the small entries ranked below
// it (entries marked at their apos; the step's ones cached in shared memory
// by the tile's warp). Kept pairs and the step's small entries go straight to
// their merged positions.
constexpr int kMergeTiles = 8;   // tiles per CTA (one warp each for the small entries)
constexpr int kMergeK = 8;       // listed pairs per thread per step
constexpr int kMergeStep = 256 * kMergeK;
constexpr int kMergeWin = 128;   // small entries cached per tile and step (the rest: global)

template <int G>
__device__ __forceinline__ void merge_huge_body(
    int t0, DevCamera cam, HugePairs huge, const uint4* __restrict__ packed_r,
    const uint4* __restrict__ packed_s, const uint32_t* __restrict__ sb,
    const FrameStatus* __restrict__ status, const uint8_t* __restrict__ masks,
    const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ apos,
    const uint2* __restrict__ small_ranges, PackedFormat fmt, const uint2* __restrict__ ranges,
    uint32_t* __restrict__ vals, uint64_t cap, const unsigned long long* __restrict__ n_total) {
    __shared__ uint32_t s_tk[G][256];     // per tile: each thread's kept bits | kept before (in warp) << kMergeK
    __shared__ uint32_t s_wk[G][8], s_wm[G][8];  // per warp totals, then exclusive prefixes
    __shared__ uint32_t s_tot[G][2];
    // small entries ranked just below pair c0 + i, 16-bit counters packed in
    // pairs (dynamic shared memory; a counter would need 65536 small entries
    // of one tile ranked between the same two listed pairs to overflow)
    extern __shared__ uint32_t s_mark32[];
    uint16_t(*s_mark)[kMergeStep] = reinterpret_cast<uint16_t(*)[kMergeStep]>(s_mark32);
    __shared__ uint32_t s_mp[G][256];  // marks before each thread's first pair (in its warp)
    __shared__ uint32_t s_wpos[G][kMergeWin], s_wval[G][kMergeWin];  // the step's small entries
    __shared__ uint32_t s_run[G], s_ia[G], s_a0[G], s_na[G], s_ob[G], s_nw[G];
    if (*n_total > cap) return;  // deferred frame that outgrew its buffers: re-rendered
    const int ntiles = cam.ntx * cam.nty;
    // groups of kMergeTiles tiles sharing one sign pattern go to the G =
    // kMergeTiles instance; the tiles of the other groups, one CTA each, to G = 1
    {
        const int grp = (t0 / kMergeTiles) * kMergeTiles;
        const bool uniform = merge_list(cam, grp, kMergeTiles, masks, packed_r, packed_s, sb, 0).single;
        if (uniform != (G == kMergeTiles)) return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto value_of = [&](uint64_t k) {
        return (uint32_t((k >> fmt.vb) & 7u) << 29) | uint32_t(k & ((uint64_t(1) << fmt.vb) - 1));
    };
    uint32_t txs[G], tys[G], tms[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int t = t0 + g;
        const bool live = t < ntiles;
        txs[g] = live ? uint32_t(t % cam.ntx) : 0xffffu;
        tys[g] = live ? uint32_t(t / cam.ntx) : 0xffffu;
        tms[g] = live ? masks[t] : 0u;
    }
    if (threadIdx.x < G) {
        const int t = t0 + threadIdx.x;
        const uint2 sr = t < ntiles ? small_ranges[t] : make_uint2(0, 0);
        s_a0[threadIdx.x] = sr.x;
        s_na[threadIdx.x] = sr.y > sr.x ? sr.y - sr.x : 0u;
        s_ob[threadIdx.x] = t < ntiles ? ranges[t].x : 0u;
        s_run[threadIdx.x] = s_ia[threadIdx.x] = 0;
    }
    const MergeList L = merge_list(cam, t0, G, masks, packed_r, packed_s, sb,
                                   min(status->n_huge_pairs, huge.cap));
    const uint4* __restrict__ packed = L.p + L.lo;
    const uint32_t nh = L.hi - L.lo;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t c0 = 0; c0 < nh; c0 += kMergeStep) {
        for (int i = threadIdx.x; i < G * kMergeStep / 2; i += 256) s_mark32[i] = 0;
        // this thread's pairs (thread-contiguous 128 B)
        uint4 rec[kMergeK];
#pragma unroll
        for (int k = 0; k < kMergeK; ++k) {
            const uint32_t j = c0 + threadIdx.x * kMergeK + k;
            rec[k] = j < nh ? __ldg(packed + j) : make_uint4(0, 0, 0xffffu, 0xffffu);
        }
        __syncthreads();
        // warp w: tile w's small entries ranked inside this step, marked and cached
        if (warp < G) {
            const uint32_t ia = s_ia[warp], na = s_na[warp], a0 = s_a0[warp];
            uint32_t nw = 0;
            for (uint32_t i0 = ia; i0 < na; i0 += 32) {
                const uint32_t i = i0 + lane;
                const uint32_t p = i < na ? apos[a0 + i] : 0xffffffffu;
                const bool in = p < c0 + kMergeStep;
                const uint32_t bin = __ballot_sync(0xffffffffu, in);
                if (in) {
                    const uint32_t q = warp * kMergeStep + (p - c0);
                    atomicAdd(s_mark32 + (q >> 1), 1u << (16 * (q & 1)));
                    const uint32_t at = nw + __popc(bin & lt);
                    if (at < kMergeWin) {
                        s_wpos[warp][at] = p - c0;
                        s_wval[warp][at] = value_of(skeys[a0 + i]);
                    }
                }
                nw += __popc(bin);
                if (bin != 0xffffffffu) break;  // apos is nondecreasing: the rest lie later
            }
            if (lane == 0) s_nw[warp] = nw;
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < G; ++g) {
            uint32_t keep = 0, m = 0;
#pragma unroll
            for (int k = 0; k < kMergeK; ++k) {
                const uint32_t rx0 = rec[k].z & 0xffffu, rx1 = rec[k].z >> 16;
                const uint32_t ry0 = rec[k].w & 0xffffu, ry1 = rec[k].w >> 16;
                const bool in = txs[g] >= rx0 && txs[g] <= rx1 && tys[g] >= ry0 && tys[g] <= ry1 &&
                                ((tms[g] >> (rec[k].y >> 29)) & 1u) &&
                                c0 + threadIdx.x * kMergeK + k < nh;
                keep |= uint32_t(in) << k;
                m += s_mark[g][threadIdx.x * kMergeK + k];
            }
            uint32_t ik = __popc(keep), im = m;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t yk = __shfl_up_sync(0xffffffffu, ik, o);
                const uint32_t ym = __shfl_up_sync(0xffffffffu, im, o);
                if (lane >= o) {
                    ik += yk;
                    im += ym;
                }
            }
            // in-warp exclusive kept count above the kept bits
            s_tk[g][threadIdx.x] = keep | ((ik - __popc(keep)) << kMergeK);
            if (lane == 31) {
                s_wk[g][warp] = ik;
                s_wm[g][warp] = im;
            }
            s_mp[g][threadIdx.x] = im - m;  // marks before this thread's pairs (in its warp)
        }
        __syncthreads();
        if (threadIdx.x < 2 * G) {  // cross-warp exclusive prefixes: kept (tid < G), marks (tid >= G)
            const int g = threadIdx.x % G;
            uint32_t* w = threadIdx.x < G ? s_wk[g] : s_wm[g];
            uint32_t run = 0;
            for (int q = 0; q < 8; ++q) {
                const uint32_t c = w[q];
                w[q] = run;
                run += c;
            }
            s_tot[g][threadIdx.x < G ? 0 : 1] = run;
        }
        __syncthreads();
        // kept pairs: merged position = kept before + small entries ranked below
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint32_t tk = s_tk[g][threadIdx.x];
            uint32_t kb = s_run[g] + s_wk[g][warp] + (tk >> kMergeK);
            uint32_t ab = s_ia[g] + s_wm[g][warp] + s_mp[g][threadIdx.x];
#pragma unroll
            for (int k = 0; k < kMergeK; ++k) {
                ab += s_mark[g][threadIdx.x * kMergeK + k];  // entries ranked below this pair
                if ((tk >> k) & 1u) vals[s_ob[g] + kb++ + ab] = rec[k].y;
            }
        }
        // the step's small entries (warp w, tile w): after the kept pairs ranked below
        if (warp < G) {
            const uint32_t nw = s_nw[warp];
            for (uint32_t q = lane; q < nw; q += 32) {
                uint32_t pl, v;
                if (q < kMergeWin) {
                    pl = s_wpos[warp][q];
                    v = s_wval[warp][q];
                } else {  // more than the cache holds: straight from global memory
                    const uint32_t i = s_ia[warp] + q;
                    pl = apos[s_a0[warp] + i] - c0;
                    v = value_of(skeys[s_a0[warp] + i]);
                }
                const uint32_t th = pl / kMergeK, tw = th >> 5;
                uint32_t kept_before = s_run[warp];
                if (th < 256) {
                    const uint32_t tk = s_tk[warp][th];
                    kept_before += s_wk[warp][tw] + (tk >> kMergeK) +
                                   __popc(tk & ((1u << (pl % kMergeK)) - 1u));
                } else {
                    kept_before += s_tot[warp][0];
                }
                vals[s_ob[warp] + s_ia[warp] + q + kept_before] = v;
            }
        }
        __syncthreads();
        if (threadIdx.x < G) {
            s_run[threadIdx.x] += s_tot[threadIdx.x][0];
            s_ia[threadIdx.x] += s_nw[threadIdx.x];
        }
    }
    __syncthreads();
    for (int g = 0; g < G; ++g)
        for (uint32_t i = s_ia[g] + threadIdx.x; i < s_na[g]; i += 256)
            vals[s_ob[g] + i + s_run[g]] = value_of(skeys[s_a0[g] + i]);
}

// CTAs [0, ntiles): single tiles of the groups without a uniform sign pattern
// (they merge from the longer lists: scheduled first); then one CTA per group.
__global__ void __launch_bounds__(256) merge_huge_kernel(
    DevCamera cam, HugePairs huge, const uint4* __restrict__ packed_r,
    const uint4* __restrict__ packed_s, const uint32_t* __restrict__ sb,
    const FrameStatus* __restrict__ status, const uint8_t* __restrict__ masks,
    const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ apos,
    const uint2* __restrict__ small_ranges, PackedFormat fmt, const uint2* __restrict__ ranges,
    uint32_t* __restrict__ vals, uint64_t cap, const unsigned long long* __restrict__ n_total) {
    pdl_enter();
    const int ntiles = cam.ntx * cam.nty;
    if (int(blockIdx.x) < ntiles)
        merge_huge_body<1>(int(blockIdx.x), cam, huge, packed_r, packed_s, sb, status, masks, skeys, apos,
                           small_ranges, fmt, ranges, vals, cap, n_total);
    else
        merge_huge_body<kMergeTiles>((int(blockIdx.x) - ntiles) * kMergeTiles, cam, huge, packed_r, packed_s,
                                     sb, status, masks, skeys, apos, small_ranges, fmt, ranges, vals, cap,
                                     n_total);
}

__global__ void __launch_bounds__(kScanThreads) duplicate_ranked_kernel(
    DevCamera cam, uint64_t m, const uint32_t* __restrict__ pc, const uint32_t* __restrict__ partial,
    const uint32_t* __restrict__ order, const int4* __restrict__ rects, const uint8_t* __restrict__ masks,
    const int2* __restrict__ rowspan, PackedFormat fmt, uint64_t* __restrict__ keys, uint64_t cap, uint2* big,
    unsigned int* n_big, TileDigits td) {
    pdl_enter();
    __shared__ uint32_t s_warp[kScanThreads / 32 + 1];
    __shared__ uint32_t s_h[2][256];  // the sort's two tile-digit histograms
    if (td.hist) s_h[threadIdx.x >> 8][threadIdx.x & 255] = 0;
    const uint64_t i0 = uint64_t(blockIdx.x) * kScanChunk + uint64_t(threadIdx.x) * 8;
    uint32_t x[8];
    if (i0 + 8 <= m) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(pc + i0));
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(pc + i0) + 1);
        x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = i0 + k < m ? pc[i0 + k] : 0u;
    }
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += x[k];
    // block exclusive scan of the per-thread sums (scan.cu's apply phase)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    }
    __syncthreads();
    uint64_t o = uint64_t(partial[blockIdx.x]) + s_warp[warp] + incl - sum;
    for (int k = 0; k < 8 && sum; ++k) {
        const uint32_t cnt = x[k];
        if (cnt == 0) continue;
        if (o + cnt <= cap) {  // else: deferred-E frame that outgrew its buffers (flagged)
            const uint64_t r = i0 + k;
            if (cnt > kRankedBigMin) {
                big[atomicAdd(n_big, 1u)] = make_uint2(uint32_t(r), uint32_t(o));
            } else {
                const uint32_t ov = __ldg(order + r);
                const uint32_t s = ov >> 29;
                const uint64_t v = ov & ((1u << 29) - 1u);
                const int4 rc = __ldg(rects + v);
                uint64_t at = o;
                for (int ty = rc.z; ty <= rc.w; ++ty) {
                    const int2 sp = __ldg(rowspan + s * cam.nty + ty);
                    if (sp.x >= 0) {  // one run: no mask reads
                        const int a = max(sp.x, rc.x), e = min(sp.y, rc.y);
                        for (int tx = a; tx <= e; ++tx) {
                            const uint32_t t = uint32_t(ty) * cam.ntx + tx;
                            keys[at++] = ranked_key(fmt, t, r, s, v);
                            if (td.hist) atomicAdd(&s_h[0][t & td.m0], 1u);
                        }
                        if (td.hist && td.two && e >= a)  // high digit: one add per 2^b0-aligned segment
                            for (uint32_t t = uint32_t(ty) * cam.ntx + a, t1 = uint32_t(ty) * cam.ntx + e; t <= t1;) {
                                const uint32_t seg_end = min(t1, (((t >> td.b0) + 1) << td.b0) - 1);
                                atomicAdd(&s_h[1][(t >> td.b0) & td.m1], seg_end - t + 1);
                                t = seg_end + 1;
                            }
                    } else {
                        for (int tx = rc.x; tx <= rc.y; ++tx) {
                            const uint32_t t = uint32_t(ty) * cam.ntx + tx;
                            if ((__ldg(masks + t) >> s) & 1u) {
                                keys[at++] = ranked_key(fmt, t, r, s, v);
                                if (td.hist) {
                                    atomicAdd(&s_h[0][t & td.m0], 1u);
                                    if (td.two) atomicAdd(&s_h[1][(t >> td.b0) & td.m1], 1u);
                                }
                            }
                        }
                    }
                }
            }
        }
        o += cnt;
    }
    if (td.hist) {  // the CTA's counts into the sort's global histograms
        __syncthreads();
        const uint32_t c = s_h[threadIdx.x >> 8][threadIdx.x & 255];
        if (c) atomicAdd(td.hist + threadIdx.x, c);
    }
}

// One warp per large pair (grid-stride over the list). Per group of 32 rows,
// lane i takes row ty0 + i: its entry count (the row span clipped to the
// rectangle, or the pattern-s SAT row count for a row that is not one run),
// a warp scan turns the counts into row offsets, then the rows are written
// one after another with the lanes across the columns (coalesced stores).
__global__ void __launch_bounds__(256) duplicate_big_ranked_kernel(
    DevCamera cam, const uint32_t* __restrict__ order, const int4* __restrict__ rects,
    const uint8_t* __restrict__ masks, const uint32_t* __restrict__ sat, const int2* __restrict__ rowspan,
    PackedFormat fmt, uint64_t* __restrict__ keys, const uint2* __restrict__ big,
    const unsigned int* __restrict__ n_big, TileDigits td) {
    pdl_enter();
    __shared__ uint32_t s_h[2][256];
    // low digit of one-run rows as range increments: a difference array over
    // the 2^b0 bins plus a count of whole periods (added to every bin)
    __shared__ int s_d0[257];
    __shared__ uint32_t s_all0, s_wsum[8];
    if (td.hist) {
        s_h[0][threadIdx.x] = 0;
        s_h[1][threadIdx.x] = 0;
        s_d0[threadIdx.x] = 0;
        if (threadIdx.x == 0) s_d0[256] = 0, s_all0 = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const uint32_t nb = *n_big;
    const int ncell = (cam.ntx + 1) * (cam.nty + 1);
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += nwarps) {
        const uint2 e = big[b];
        const uint32_t ov = __ldg(order + e.x);
        const uint32_t s = ov >> 29;
        const uint64_t v = ov & ((1u << 29) - 1u);
        const uint32_t* sat_s = sat + size_t(1 + s) * ncell;
        const int4 rc = __ldg(rects + v);
        uint64_t at = e.y;
        for (int ty0 = rc.z; ty0 <= rc.w; ty0 += 32) {
            const int ty = ty0 + lane;
            int a = 0, len = 0;
            if (ty <= rc.w) {
                const int2 sp = __ldg(rowspan + s * cam.nty + ty);
                if (sp.x >= 0) {
                    a = max(sp.x, rc.x);
                    len = max(0, min(sp.y, rc.y) - a + 1);
                } else {
                    a = -1;  // not one run: ballot over the masks below
                    len = int(sat_rect(sat_s, cam.ntx, rc.x, rc.y, ty, ty));
                }
            }
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (td.hist && a >= 0 && len > 0) {
                const uint32_t t0 = uint32_t(ty) * cam.ntx + uint32_t(a), t1 = t0 + uint32_t(len) - 1;
                // low digit: the row's bins t0 .. t1 (mod 2^b0) as range increments
                const uint32_t P = td.m0 + 1, full = uint32_t(len) >> td.b0, rem = uint32_t(len) & td.m0;
                const uint32_t st = t0 & td.m0;
                if (full) atomicAdd(&s_all0, full);
                if (rem) {
                    atomicAdd(&s_d0[st], 1);
                    if (st + rem <= P) {
                        atomicAdd(&s_d0[st + rem], -1);
                    } else {
                        atomicAdd(&s_d0[0], 1);
                        atomicAdd(&s_d0[st + rem - P], -1);
                    }
                }
                // high digit: one add per 2^b0-aligned segment
                if (td.two)
                    for (uint32_t t = t0; t <= t1;) {
                        const uint32_t seg_end = min(t1, (((t >> td.b0) + 1) << td.b0) - 1);
                        atomicAdd(&s_h[1][(t >> td.b0) & td.m1], seg_end - t + 1);
                        t = seg_end + 1;
                    }
            }
            if (!__any_sync(0xffffffffu, a < 0 && len > 0)) {
                // every row one run: the group's entries as one flat range.
                // Rows of one length and start column (a rectangle inside
                // the pattern's runs, the usual case) give lane q its row by a
                // division; otherwise a binary search over the row prefix sums.
                const int nrows = min(32, rc.w - ty0 + 1);
                const int L0 = __shfl_sync(0xffffffffu, len, 0), A0 = __shfl_sync(0xffffffffu, a, 0);
                const bool uni = L0 > 0 && __all_sync(0xffffffffu, lane >= nrows || (len == L0 && a == A0));
                const float invL = uni ? 1.0f / float(L0) : 0.f;
                for (int e0 = 0; e0 < total; e0 += 32) {
                    const int q = e0 + lane;
                    uint32_t t;
                    if (uni) {
                        int j = int((float(q) + 0.5f) * invL);
                        j -= j * L0 > q;
                        j += (j + 1) * L0 <= q;
                        t = uint32_t(ty0 + j) * cam.ntx + uint32_t(A0 + (q - j * L0));
                    } else {
                        int j = 0;
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1)
                            if (__shfl_sync(0xffffffffu, incl, j + step - 1) <= q) j += step;
                        const int lj = __shfl_sync(0xffffffffu, len, j), aj = __shfl_sync(0xffffffffu, a, j);
                        const int ij = __shfl_sync(0xffffffffu, incl, j);
                        t = uint32_t(ty0 + j) * cam.ntx + aj + (q - (ij - lj));
                    }
                    if (q < total) keys[at + q] = ranked_key(fmt, t, e.x, s, v);
                }
                at += uint64_t(total);
                continue;
            }
            const int nrows = min(32, rc.w - ty0 + 1);
            for (int j = 0; j < nrows; ++j) {
                const int l = __shfl_sync(0xffffffffu, len, j);
                if (l == 0) continue;
                const int aj = __shfl_sync(0xffffffffu, a, j);
                const uint64_t ro = at + uint64_t(__shfl_sync(0xffffffffu, incl, j) - l);
                const uint64_t trow = uint64_t(ty0 + j) * cam.ntx;
                if (aj >= 0) {  // (the row's digits were counted by its lane above)
                    for (int c = lane; c < l; c += 32) keys[ro + c] = ranked_key(fmt, trow + aj + c, e.x, s, v);
                } else {
                    uint64_t w = ro;
                    for (int tx0 = rc.x; tx0 <= rc.y; tx0 += 32) {
                        const int tx = tx0 + lane;
                        const bool hit = tx <= rc.y && ((__ldg(masks + trow + tx) >> s) & 1u);
                        const unsigned bal = __ballot_sync(0xffffffffu, hit);
                        if (hit) {
                            keys[w + __popc(bal & ((1u << lane) - 1u))] = ranked_key(fmt, trow + tx, e.x, s, v);
                            if (td.hist) {
                                const uint32_t t = uint32_t(trow + tx);
                                atomicAdd(&s_h[0][t & td.m0], 1u);
                                if (td.two) atomicAdd(&s_h[1][(t >> td.b0) & td.m1], 1u);
                            }
                        }
                        w += __popc(bal);
                    }
                }
            }
            at += uint64_t(total);
        }
    }
    if (td.hist) {
        __syncthreads();
        // low digit: inclusive scan of the difference array (block scan), plus
        // the whole periods and the per-entry counts of the non-run rows
        int x = s_d0[threadIdx.x];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[threadIdx.x >> 5] = uint32_t(x);
        __syncthreads();
        for (int w = 0; w < int(threadIdx.x >> 5); ++w) x += int(s_wsum[w]);
        const uint32_t c0 = threadIdx.x <= td.m0 ? s_h[0][threadIdx.x] + uint32_t(x) + s_all0 : 0u;
        if (c0) atomicAdd(td.hist + threadIdx.x, c0);
        if (s_h[1][threadIdx.x]) atomicAdd(td.hist + 256 + threadIdx.x, s_h[1][threadIdx.x]);
    }
}

__global__ void rank_keys_kernel(const uint64_t* __restrict__ paths, uint64_t n, uint64_t* keys,
                                 uint32_t* vals) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= 8 * n) return;
    const uint64_t s = i / n, v = i - s * n;
    keys[i] = (paths[v] & kCodeMask48) ^ (s * kGroupOnes);
    vals[i] = uint32_t(s << 29) | uint32_t(v);
}

__global__ void rank_scatter_kernel(const uint32_t* __restrict__ vals, uint64_t n, uint32_t* rank) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= 8 * n) return;
    const uint32_t val = vals[i];
    rank[uint64_t(val >> 29) * n + (val & ((1u << 29) - 1u))] = uint32_t(i);
}

__global__ void tile_ranges_packed_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                          PackedFormat fmt, uint2* ranges, uint32_t* vals,
                                          const unsigned long long* n_dev) {
    pdl_enter();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    n = live_entries(n, n_dev);  // deferred-E frame: the device count decides
    if (i >= n) return;
    const uint64_t k = keys[i];
    const uint32_t t = uint32_t(k >> fmt.tile_shift);
    vals[i] = (uint32_t((k >> fmt.vb) & 7u) << 29) | uint32_t(k & ((uint64_t(1) << fmt.vb) - 1));
    if (i == 0 || uint32_t(keys[i - 1] >> fmt.tile_shift) != t) ranges[t].x = uint32_t(i);
    if (i == n - 1 || uint32_t(keys[i + 1] >> fmt.tile_shift) != t) ranges[t].y = uint32_t(i + 1);
}

__global__ void unpack_entries_kernel(const uint64_t* packed, uint64_t n, PackedFormat fmt,
                                      const uint64_t* paths, uint64_t* keys, uint32_t* vals) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = packed[i];
    const uint64_t vid = k & ((uint64_t(1) << fmt.vb) - 1);
    const uint64_t sgn = (k >> fmt.vb) & 7u;
    const uint64_t tid = k >> fmt.tile_shift;
    vals[i] = uint32_t(sgn << 29) | uint32_t(vid);
    if (fmt.rank_bits) {
        keys[i] = (tid << 48) | ((paths[vid] & kCodeMask48) ^ (sgn * kGroupOnes));
        return;
    }
    const int obits = 3 * fmt.lmax;
    const uint64_t otop = (k >> (fmt.vb + 3)) & ((uint64_t(1) << obits) - 1);
    const uint64_t low = obits < 48 ? ((sgn * kGroupOnes) & ((uint64_t(1) << (48 - obits)) - 1)) : 0;
    keys[i] = (tid << 48) | (obits > 0 ? (otop << (48 - obits)) : 0) | low;
}

// ------------------------------------------------------------------- K6
__global__ void tile_ranges_kernel(const uint64_t* keys, uint64_t n, uint2* ranges) {
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t t = uint32_t(keys[i] >> 48);
    if (i == 0 || uint32_t(keys[i - 1] >> 48) != t) ranges[t].x = uint32_t(i);
    if (i == n - 1 || uint32_t(keys[i + 1] >> 48) != t) ranges[t].y = uint32_t(i + 1);
}

// Longest-processing-time-first tile order for K7: tiles bucketed by
// floor(log2(entries+1)), heaviest bucket first, so the long tiles start in
// the first wave and the kernel tail is made of short ones.
__global__ void __launch_bounds__(1024) tile_order_kernel(uint2* ranges, int ntiles,
                                                          uint32_t* order) {
    pdl_enter();
    __shared__ uint32_t s_cnt[33];
    if (threadIdx.x < 33) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        uint2 r = ranges[t];
        if (r.x > r.y) {  // no entries (value-only sort finish leaves lo > hi)
            r = make_uint2(0u, 0u);
            ranges[t] = r;
        }
        atomicAdd(&s_cnt[31 - __clz(r.y - r.x + 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 31; b >= 0; --b) {
            const uint32_t c = s_cnt[b];
            s_cnt[b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
        const uint2 r = ranges[t];
        order[atomicAdd(&s_cnt[31 - __clz(r.y - r.x + 1)], 1u)] = uint32_t(t);
    }
}

// ------------------------------------------------------------------- K7
// One CTA per 16x16 tile (LPT order), eight warps; each warp owns an 8x4
// pixel block and runs autonomously (no CTA barrier inside the entry loop,
// so a warp whose block sees few voxels never waits for a busy neighbour).
//
// The tile's sorted entry list is consumed in chunks of 32 (one entry per
// lane). Per chunk the warp culls with the reference's own filters lifted to
// its block (sign patterns, screen AABB; a frustum test for loose AABBs) and
// ballots the survivors ("slots"). Their 96-B records are copied into
// warp-private shared memory with cp.async one chunk AHEAD of use (double
// buffer), so the L2 latency of the gather overlaps the compositing of the
// previous chunk.
//
// Compositing a chunk is two-phase:
//   A. every lane tests every slot (sign, AABB, fp32 slab): a bit per slot;
//   B. every lane walks ITS OWN hit bits in entry order and runs the K-point
//      quadrature + CompositeCtx::add only there. All lanes execute the same
//      instructions (they differ in which slot they read), so lane
//      utilisation is set by the busiest pixel of the block, not by how
//      many pixels each voxel covers (~1/3 of the block on config 2).
// The per-pixel set and order of composited voxels is the reference's
// (raster.cpp:17-61, 238-281), and a pixel stops after the voxel that took
// T below the threshold.
__device__ __forceinline__ void pixel_of(const DevCamera& cam, int tile, int tid, int& px, int& py) {
    const int tx = tile % cam.ntx, ty = tile / cam.ntx;
    const int warp = tid >> 5, lane = tid & 31;
    px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
}

#ifndef SVR_CP_CG
#define SVR_CP_CG 1  // plain-render record copies L2-only (.cg): cfg2 composite 312 -> 309 us, cfg4 -0.5 %;
#endif               // the recording modes keep .ca (cfg5 staged composite +1.1 % with .cg)
template <bool CG = false>
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (CG && SVR_CP_CG)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// fp32 slab test of ray_aabb (field.hpp:58-69) against the camera-relative
// box [lo.xyz, lo.xyz + lo.w], with the near/far face of each axis chosen by
// the sign of the inverse direction (n = 1 where it is negative): fma(w, 1, lo)
// rounds exactly like lo + w and fma(w, 0, lo) = lo, so ta/tb are the same
// floats as the min/max form below, three instructions cheaper.
// TMA bulk copies (cp.async.bulk, completion counted on an mbarrier): the
// SVR_BULK=1 variant of the warp path stages each surviving 96-B record with
// ONE bulk copy instead of six 16-B cp.async (measured slower).
#ifndef SVR_BULK
#define SVR_BULK 0
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void slab(float4 lo, float ix, float iy, float iz, float& ta, float& tb) {
    float t0 = lo.x * ix, t1 = (lo.x + lo.w) * ix;
    ta = fminf(t0, t1);
    tb = fmaxf(t0, t1);
    t0 = lo.y * iy;
    t1 = (lo.y + lo.w) * iy;
    ta = fmaxf(ta, fminf(t0, t1));
    tb = fminf(tb, fmaxf(t0, t1));
    t0 = lo.z * iz;
    t1 = (lo.z + lo.w) * iz;
    ta = fmaxf(ta, fminf(t0, t1));
    tb = fminf(tb, fmaxf(t0, t1));
}

constexpr int kCompWarps = 8;
constexpr size_t kCompSmem = size_t(2) * kCompWarps * 32 * kRecordF4 * sizeof(float4);

// MODE 0: plain render; 1: record pass (RECORD); 2: render with per-voxel
// max-blend stats and/or staged training records (their checks compiled in);
// 3: staged training records only (the single-pass training render).
// A warp's staged records: 32 slots x 6 float4. SVR_REC_SOA stores them as
// six planes of 32 (slot stride 16 B), so phase-B lanes reading different
// slots and the cp.async writes of different slots hit distinct banks (the
// 96-B slot stride of the slot-major layout maps 32 slots onto 4 bank groups).
#ifndef SVR_REC_SOA
#define SVR_REC_SOA 1
#endif
#if SVR_REC_SOA
#define WREC(w, slot, k) (w)[(k) * 32 + (slot)]
#else
#define WREC(w, slot, k) (w)[(slot) * kRecordF4 + (k)]
#endif
#if SVR_REC_SOA && SVR_BULK
#error "SVR_BULK copies a record as one contiguous 96-B block: needs SVR_REC_SOA=0"
#endif
#ifndef SVR_PHB_SLABS
#define SVR_PHB_SLABS 1
#endif
#ifndef SVR_COOP_BATCH
#define SVR_COOP_BATCH 1024  // 2048: cfg4 composite 1.55 -> 1.65 ms (spills at 64 registers), cfg5 staged 1.82 -> 1.79
#endif
constexpr int kBatch = SVR_COOP_BATCH;  // entries culled per CTA batch (cooperative path)
static_assert(kBatch == 1024 || kBatch == 2048, "cooperative batch: 1024 or 2048 entries");
using NzWord = std::conditional_t<(kBatch > 1024), unsigned long long, uint32_t>;
constexpr int kSubs = kBatch / 32;  // 32-entry sub-chunks per batch
#ifndef SVR_PHA_UNROLL
#define SVR_PHA_UNROLL 4  // phase-A slab loop unroll factor (2 -> 4: cfg4 composite 1.54 -> 1.52 ms, cfg5 staged -1.1 %, cfg2 neutral; 1: +5 %)
#endif
constexpr int kPhaseAUnroll = SVR_PHA_UNROLL;
#ifndef SVR_COOP_BBPRE
#define SVR_COOP_BBPRE 0  // next batch's AABBs loaded before compositing, culled after (cfg4 1.55 -> 1.66 ms at 3 CTAs/SM, 2.05 at 4 with spills; cfg5 1.81 -> 1.89: off)
#endif
#ifndef SVR_COOP_VPRE
#define SVR_COOP_VPRE 1  // values of the next batch's cull loaded a batch ahead (cfg4 composite 1.68 -> 1.55 ms)
#endif
#ifndef SVR_COOP_BYTES
#define SVR_COOP_BYTES 1  // cull masks as bytes, balloted by the consumer (needs SVR_COOP_NZ): cfg4 composite 1.76 -> 1.67 ms
#endif
#ifndef SVR_COOP_NZ
#define SVR_COOP_NZ 1  // per-warp summary of the sub-chunks with survivors
#endif

// Shared memory of K7 besides the record buffers: the two per-tile paths
// (warp-autonomous below, CTA-cooperative after it) use it in turn.
template <int K, int MODE>
struct CompShared {
    static constexpr bool ENTRY = MODE != 0;  // slots need their entry index
    union {
        struct {
            uint32_t vid[2][kCompWarps][32];
            uint8_t j[2][kCompWarps][32];  // chunk-local entry index of each slot
        } w;
        struct {
#if SVR_COOP_BYTES
            uint8_t mb[2][kSubs][32];  // [batch buf][sub-chunk][entry]: the blocks it survives for
#else
            uint32_t ball[2][kSubs][kCompWarps];  // [batch buf][sub-chunk][warp]
#endif
            NzWord nz[2][kCompWarps];  // [batch buf][warp]: bit = sub-chunk with survivors
            uint8_t sign[2][kCompWarps][32];   // sign pattern of each slot
            uint32_t ent[ENTRY ? 2 : 1][kCompWarps][32];  // entry index of each slot
            uint32_t wsig[kCompWarps];
            uint32_t signwarps[8];
        } c;
    };
    float cone[kCompWarps][4][3];
    uint64_t mbar[SVR_BULK ? kCompWarps : 1][2];  // SVR_BULK: per warp and record buffer
    // pixel centres for phase B (one LDS instead of a per-hit rematerialised
    // copy); the entry-recording modes need the space for c.ent instead
    float2 pc[ENTRY ? 1 : 256];
};

template <int K, int MODE>
__device__ __forceinline__ void composite_tile_warp(const DevCamera& cam, const CompositeArgs& a,
                                                    int tile, CompShared<K, MODE>& sh,
                                                    float4* s_rec_dyn) {
    constexpr bool RECORD = MODE == 1;
    constexpr bool EXTRA = MODE == 2;
    constexpr bool STAGED = MODE == 3;
    constexpr bool PC_SMEM = !CompShared<K, MODE>::ENTRY;
    auto& s_vid = sh.w.vid;
    auto& s_j = sh.w.j;
    auto& s_cone = sh.cone;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int px, py;
    pixel_of(cam, tile, threadIdx.x, px, py);
    const bool inside = px < cam.W && py < cam.H;
    // this warp's 8x4 footprint in pixel-centre coordinates
    const int wx0 = px - (lane & 7), wy0 = py - (lane >> 3);
    const float fx0 = float(wx0) + 0.5f, fx1 = float(wx0) + 7.5f;
    const float fy0 = float(wy0) + 0.5f, fy1 = float(wy0) + 3.5f;

    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const uint32_t my_sign = sign_bits(dd);
    const uint32_t warp_signs = __reduce_or_sync(0xffffffffu, inside ? (1u << my_sign) : 0u);
    const bool one_sign = __popc(warp_signs) <= 1;
    const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
    const float ix = slab_inv(dd[0]), iy = slab_inv(dd[1]), iz = slab_inv(dd[2]);
    const SlabSel ssel = slab_sel(ix, iy, iz);
    const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));
    const float pcx = float(px) + 0.5f, pcy = float(py) + 0.5f;
    if (PC_SMEM) sh.pc[PC_SMEM ? threadIdx.x : 0] = make_float2(pcx, pcy);
    // Frustum of this warp's 8x4 block (warp_cone_planes): skips boxes whose
    // screen AABB is loose, e.g. near-plane voxels, which get the full screen
    // (raster.cpp:95-101), without changing the composited set.
    float (*cone)[3] = s_cone[warp];
    if (lane == 0) warp_cone_planes(cam, wx0, wy0, cone);
#if SVR_BULK
    uint64_t* mbar = sh.mbar[SVR_BULK ? warp : 0];
    if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned phase = 0;  // bit b: parity of buffer b's next completion
    unsigned pend = 0;   // bit b: buffer b has copies in flight
#endif
    __syncwarp();

    float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f, nx = 0.f, ny = 0.f, nz = 0.f, depth = 0.f;
    float median = -1.0f;
    uint32_t cnt = 0;
    bool done = !inside;
    const uint32_t slot = uint32_t(tile) * 256u + uint32_t((py % kTile) * kTile + (px % kTile));
    uint32_t rec_base = 0;
    if (RECORD) rec_base = inside ? a.pix_begin[slot] : 0u;

    const uint2 range = a.ranges[tile];
    const float thr = a.t_threshold;
    constexpr uint32_t kVidMask = (1u << 29) - 1u;
    float4* wrec0 = s_rec_dyn + size_t(warp) * 32 * kRecordF4;
    float4* wrec1 = wrec0 + kCompWarps * 32 * kRecordF4;

    // Cull one chunk (entries c .. c+31, lane = entry) and start the copy of
    // its surviving records into buffer `buf`. Returns the survivor mask.
    auto stage = [&](uint32_t c, uint32_t v, float4 b, int buf) -> uint32_t {
        bool rel = c + lane < range.y && ((warp_signs >> (v >> 29)) & 1u) &&
                   !(fx1 < b.x || fx0 > b.y || fy1 < b.z || fy0 > b.w);
        // frustum test only for entries with a large screen AABB
        const bool wide = rel && (b.y - b.x) * (b.w - b.z) > kConeMinArea;
        if (__any_sync(0xffffffffu, wide) && wide)
            rel = box_in_cone(cone, __ldg(a.records + uint64_t(v & kVidMask) * kRecordF4));
        const uint32_t m = __ballot_sync(0xffffffffu, rel);
        uint32_t* wvid = s_vid[buf][warp];
        const int at = __popc(m & ((1u << lane) - 1u));
        if (rel) {
            wvid[at] = v;
            s_j[buf][warp][at] = uint8_t(lane);
        }
        float4* wrec = buf ? wrec1 : wrec0;
#if SVR_BULK
        if (lane == 0) mbar_arrive_expect(&mbar[buf], unsigned(__popc(m)) * kRecordF4 * 16u);
        if (rel) bulk_g2s(&WREC(wrec, at, 0), a.records + uint64_t(v & kVidMask) * kRecordF4, kRecordF4 * 16u,
                          &mbar[buf]);
        pend |= 1u << buf;
#else
        if (rel) {  // the lane of each surviving entry copies its record
            const float4* src = a.records + uint64_t(v & kVidMask) * kRecordF4;
#pragma unroll
            for (int k = 0; k < kRecordF4; ++k) cp_async16<MODE == 0>(&WREC(wrec, at, k), src + k);
        }
        cp_async_commit();
#endif
        return m;
    };

    // software pipeline: chunk c's records are in flight while chunk c-1 is
    // composited; (v1, b1) describe chunk c+1, v2 chunk c+2.
    uint32_t v0 = 0, v1 = 0, v2 = 0;
    float4 b0 = make_float4(0.f, -1.f, 0.f, -1.f), b1 = b0;
    if (range.x + lane < range.y) {
        v0 = __ldg(a.vals + range.x + lane);
        b0 = __ldg(a.records + uint64_t(v0 & kVidMask) * kRecordF4 + 1);
    }
    if (range.x + 32 + lane < range.y) {
        v1 = __ldg(a.vals + range.x + 32 + lane);
        b1 = __ldg(a.records + uint64_t(v1 & kVidMask) * kRecordF4 + 1);
    }
    if (range.x + 64 + lane < range.y) v2 = __ldg(a.vals + range.x + 64 + lane);
    uint32_t m_cur = range.x < range.y ? stage(range.x, v0, b0, 0) : 0u;
    int buf = 0;

    for (uint32_t c = range.x; c < range.y; c += 32, buf ^= 1) {
        if (__all_sync(0xffffffffu, done)) break;
        // prefetch: AABB of chunk c+2, values of chunk c+3
        float4 b2 = make_float4(0.f, -1.f, 0.f, -1.f);
        uint32_t v3 = 0;
        if (c + 64 + lane < range.y) b2 = __ldg(a.records + uint64_t(v2 & kVidMask) * kRecordF4 + 1);
        if (c + 96 + lane < range.y) v3 = __ldg(a.vals + c + 96 + lane);
        // stage chunk c+1 into the other buffer, then wait for chunk c
        uint32_t m_next = 0;
#if SVR_BULK
        if (c + 32 < range.y) m_next = stage(c + 32, v1, b1, buf ^ 1);
        mbar_wait(&mbar[buf], (phase >> buf) & 1u);  // chunk c's records landed
        phase ^= 1u << buf;
        pend &= ~(1u << buf);
#else
        if (c + 32 < range.y) {
            m_next = stage(c + 32, v1, b1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
#endif
        __syncwarp();

        const int nrel = __popc(m_cur);
        float4* wrec = buf ? wrec1 : wrec0;
        const uint32_t* wvid = s_vid[buf][warp];
        const uint8_t* wj = s_j[buf][warp];
        // Phase A: this lane's slab hits among the slots (the sign-pattern
        // and AABB filters, which rarely reject a slab hit, run in phase B).
        uint32_t hits = 0;
        if (!done) {
#pragma unroll kPhaseAUnroll
            for (int sl = 0; sl < nrel; ++sl) {
                float ta, tb;
                slab_s(WREC(wrec, sl, 0), ix, iy, iz, ssel, ta, tb);
                hits |= uint32_t(ta <= tb && ta > 0.0f) << sl;
            }
        }
        // Phase B: this lane's hits, in entry order.
        while (hits) {
            const int s_ = __ffs(hits) - 1;
            hits &= hits - 1;
            const float4 bb = WREC(wrec, s_, 1);
            const float2 pc = PC_SMEM ? sh.pc[PC_SMEM ? threadIdx.x : 0] : make_float2(pcx, pcy);
            if (!((one_sign || (wvid[s_] >> 29) == my_sign) &&
                  !(pc.x < bb.x || pc.x > bb.y || pc.y < bb.z || pc.y > bb.w)))
                continue;
            const float4 lo = WREC(wrec, s_, 0);
            float ta, tb;
#if SVR_PHB_SLABS
            slab_s(lo, ix, iy, iz, ssel, ta, tb);
#else
            slab(lo, ix, iy, iz, ta, tb);  // same floats as slab_s; needs no per-lane face selectors
#endif
            const float4 va = WREC(wrec, s_, 2), vb = WREC(wrec, s_, 3);
            const float inv = WREC(wrec, s_, 5).w;
            const float seg = tb - ta;
            const float lk = seg * dnorm * (1.0f / K);
            // voxel_alpha (field.hpp:92-116), K-point midpoint quadrature
            float sa[K], tk[K], sum = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                tk[k] = ta + ((k + 0.5f) / K) * seg;
#if SVR_F32X2_Q
                float qx, qy;  // (qx, qy) in one FFMA2 + FMUL2, same roundings
                up2(mul2(fma2(pk2(tk[k], tk[k]), pk2(dx, dy), pk2(-lo.x, -lo.y)), pk2(inv, inv)), qx, qy);
#else
                const float qx = (tk[k] * dx - lo.x) * inv;
                const float qy = (tk[k] * dy - lo.y) * inv;
#endif
                const float qz = (tk[k] * dz - lo.z) * inv;
                const float act = explin(trilinear_poly(va, vb, qx, qy, qz));
                sum += act;
                sa[k] = one_minus_exp_neg(lk * act);
            }
            const float alpha = (K == 1) ? sa[0] : one_minus_exp_neg(lk * sum);
            const uint32_t entry = c + wj[s_];
            if (!RECORD) {
                // voxel_depth (field.hpp:173-181) and the median crossing
                float dv = 0.f, Tk = 1.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dv += Tk * sa[k] * tk[k];
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
                const float4 col = WREC(wrec, s_, 4), nor = WREC(wrec, s_, 5);
#if SVR_F32X2_ACC
                {  // (cr, cg) and (nx, ny) as packed pairs: one FFMA2 each
                    const f32x2 ww = pk2(w, w);
                    f32x2 c2 = fma2(ww, pk2(col.x, col.y), pk2(cr, cg));
                    f32x2 n2 = fma2(ww, pk2(nor.x, nor.y), pk2(nx, ny));
                    up2(c2, cr, cg);
                    up2(n2, nx, ny);
                }
#else
                cr += w * col.x;
                cg += w * col.y;
                nx += w * nor.x;
                ny += w * nor.y;
#endif
                cb += w * col.z;
                nz += w * nor.z;
                depth += T * dv;
                if (EXTRA && a.max_blend) atomicMax(a.max_blend + __float_as_uint(col.w), __float_as_uint(w));
                if (STAGED || (EXTRA && a.stage_entry)) {
                    if (cnt < a.stage_cap) {
                        const uint32_t at = cnt * a.stage_stride + slot;
                        a.stage_entry[at] = entry;
                        a.stage_T[at] = T;
                    } else {
                        *a.overflow = 1u;
                    }
                }
            } else {
                a.contrib_entry[rec_base + cnt] = entry;
                a.contrib_T[rec_base + cnt] = T;
            }
            T *= 1.0f - alpha;
            ++cnt;
            if (T < thr) {
                done = true;
                hits = 0;
            }
        }
        __syncwarp();  // buffer `buf` is restaged two chunks later
        m_cur = m_next;
        v1 = v2;
        b1 = b2;
        v2 = v3;
    }
#if SVR_BULK
    for (int bb = 0; bb < 2; ++bb)  // no copy may outlive the CTA's shared memory
        if ((pend >> bb) & 1u) mbar_wait(&mbar[bb], (phase >> bb) & 1u);
#else
    cp_async_wait<0>();  // no copy may outlive the CTA's shared memory
#endif
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

// K7, CTA-cooperative variant. The tile's entries are culled ONCE per CTA
// instead of once per warp: per batch of 1024 entries every thread loads four
// entries' values and screen AABBs, tests them against the eight 8x4 pixel blocks
// of the tile (footprint overlap, the sign patterns present in each block,
// the block frustum for loose AABBs) and the eight per-block ballots go to
// shared memory. Each warp then walks only its own survivors of the batch
// (a broadcast word per 32 entries, zero for most of them on config 4),
// packing them into groups of up to 32 slots whose 96-B records are copied
// with cp.async while the previous group is composited (phase A slab tests,
// phase B per-lane hits, exactly as in composite_kernel). Warps meet at one
// CTA barrier per batch (a config-2 tile is a single batch, so its warps run
// unsynchronised after the cull); the CTA leaves once every warp is done.

template <int K, int MODE>
__device__ __forceinline__ void composite_tile_coop(const DevCamera& cam, const CompositeArgs& a,
                                                    int tile, CompShared<K, MODE>& sh,
                                                    float4* s_rec_dyn) {
    constexpr bool RECORD = MODE == 1;
    constexpr bool EXTRA = MODE == 2;
    constexpr bool STAGED = MODE == 3;
    constexpr bool ENTRY = CompShared<K, MODE>::ENTRY;
#if SVR_COOP_BYTES
    auto& s_mb = sh.c.mb;
#else
    auto& s_ball = sh.c.ball;
#endif
    auto& s_nz = sh.c.nz;
    auto& s_sign = sh.c.sign;
    auto& s_ent = sh.c.ent;
    auto& s_cone = sh.cone;
    auto& s_wsig = sh.c.wsig;
    auto& s_signwarps = sh.c.signwarps;
    auto& s_pc = sh.pc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int px, py;
    pixel_of(cam, tile, threadIdx.x, px, py);
    const bool inside = px < cam.W && py < cam.H;
    const int wx0 = px - (lane & 7), wy0 = py - (lane >> 3);

    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const uint32_t my_sign = sign_bits(dd);
    const uint32_t warp_signs = __reduce_or_sync(0xffffffffu, inside ? (1u << my_sign) : 0u);
    const bool one_sign = __popc(warp_signs) <= 1;
    const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
    const float ix = slab_inv(dd[0]), iy = slab_inv(dd[1]), iz = slab_inv(dd[2]);
    const SlabSel ssel = slab_sel(ix, iy, iz);
    const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));
    const float pcx = float(px) + 0.5f, pcy = float(py) + 0.5f;
    if (!ENTRY) s_pc[threadIdx.x] = make_float2(pcx, pcy);
    if (lane == 0) {
        warp_cone_planes(cam, wx0, wy0, s_cone[warp]);
        s_wsig[warp] = warp_signs;
    }
    __syncthreads();
    if (threadIdx.x < 8) {  // for each sign pattern, the blocks whose pixels have it
        uint32_t m = 0;
        for (int w = 0; w < kCompWarps; ++w) m |= ((s_wsig[w] >> threadIdx.x) & 1u) << w;
        s_signwarps[threadIdx.x] = m;
    }
    if (threadIdx.x < 2 * kCompWarps) (&s_nz[0][0])[threadIdx.x] = 0;
    __syncthreads();  // s_signwarps before the first cull
    // tile footprint in pixel-centre coordinates: block (bx, by) covers
    // x in [X0 + 8bx + .5, X0 + 8bx + 7.5], y in [Y0 + 4by + .5, Y0 + 4by + 3.5]
    const float X0 = float((tile % cam.ntx) * kTile), Y0 = float((tile / cam.ntx) * kTile);

    float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f, nx = 0.f, ny = 0.f, nz = 0.f, depth = 0.f;
    float median = -1.0f;
    uint32_t cnt = 0;
    bool done = !inside;
    const uint32_t slot = uint32_t(tile) * 256u + uint32_t((py % kTile) * kTile + (px % kTile));
    uint32_t rec_base = 0;
    if (RECORD) rec_base = inside ? a.pix_begin[slot] : 0u;

    const uint2 range = a.ranges[tile];
    const float thr = a.t_threshold;
    constexpr uint32_t kVidMask = (1u << 29) - 1u;
    float4* wrec0 = s_rec_dyn + size_t(warp) * 32 * kRecordF4;

    // Culls entries range.x + kBatch b + 256 r + threadIdx.x (r < 4) into
    // ballot buffer pb: sub-chunk 8 r + warp, one word per target warp.
#if SVR_COOP_VPRE
    // the values of the batch the next produce culls, loaded one batch ahead
    // (its AABB loads then wait on one global round trip, not two)
    uint32_t vpre[kBatch / 256];
    auto load_vals = [&](uint32_t b) {
#pragma unroll
        for (int r = 0; r < kBatch / 256; ++r) {
            const uint32_t idx = range.x + b * kBatch + r * 256 + threadIdx.x;
            vpre[r] = idx < range.y ? __ldg(a.vals + idx) : 0u;
        }
    };
#endif
#if SVR_COOP_BBPRE
    // the next batch's screen AABBs, loaded before the current batch is
    // composited and culled after it (the loads' latency hides behind it)
    float4 bbpre[kBatch / 256];
    auto load_bb = [&](uint32_t b) {
#pragma unroll
        for (int r = 0; r < kBatch / 256; ++r) {
            const uint32_t idx = range.x + b * kBatch + r * 256 + threadIdx.x;
            bbpre[r] = idx < range.y ? __ldg(a.records + uint64_t(vpre[r] & kVidMask) * kRecordF4 + 1)
                                     : make_float4(0.f, -1.f, 0.f, -1.f);
        }
    };
#endif
    auto produce = [&](uint32_t b, int pb) {
#pragma unroll
        for (int r = 0; r < kBatch / 256; ++r) {
            const uint32_t idx = range.x + b * kBatch + r * 256 + threadIdx.x;
            uint32_t m = 0;
            if (idx < range.y) {
#if SVR_COOP_VPRE
                const uint32_t v = vpre[r];
#else
                const uint32_t v = __ldg(a.vals + idx);
#endif
                const float4* rec = a.records + uint64_t(v & kVidMask) * kRecordF4;
#if SVR_COOP_BBPRE
                const float4 bb = bbpre[r];
#else
                const float4 bb = __ldg(rec + 1);
#endif
                const uint32_t xm = (!(X0 + 7.5f < bb.x || X0 + 0.5f > bb.y) ? 0x55u : 0u) |
                                    (!(X0 + 15.5f < bb.x || X0 + 8.5f > bb.y) ? 0xAAu : 0u);
                const uint32_t ym = (!(Y0 + 3.5f < bb.z || Y0 + 0.5f > bb.w) ? 0x03u : 0u) |
                                    (!(Y0 + 7.5f < bb.z || Y0 + 4.5f > bb.w) ? 0x0Cu : 0u) |
                                    (!(Y0 + 11.5f < bb.z || Y0 + 8.5f > bb.w) ? 0x30u : 0u) |
                                    (!(Y0 + 15.5f < bb.z || Y0 + 12.5f > bb.w) ? 0xC0u : 0u);
                m = xm & ym & s_signwarps[v >> 29];
                // frustum of each block only for entries with a large screen AABB
                if (m && (bb.y - bb.x) * (bb.w - bb.z) > kConeMinArea) {
                    const float4 lo = __ldg(rec);
                    for (int w = 0; w < kCompWarps; ++w)
                        if (((m >> w) & 1u) && !box_in_cone(s_cone[w], lo)) m &= ~(1u << w);
                }
            }
#if SVR_COOP_BYTES
            // each entry's 8-bit block mask as a byte; a consuming warp
            // ballots its own bit of the sub-chunks it visits
            s_mb[pb][r * kCompWarps + warp][lane] = uint8_t(m);
            const uint32_t any = __reduce_or_sync(0xffffffffu, m);
            if (lane < kCompWarps && ((any >> lane) & 1u))
                atomicOr(&s_nz[pb][lane], NzWord(1) << (r * kCompWarps + warp));
#else
            uint32_t mine = 0;
#pragma unroll
            for (int w = 0; w < kCompWarps; ++w) {
                const uint32_t bw = __ballot_sync(0xffffffffu, (m >> w) & 1u);
                if (lane == w) mine = bw;
            }
            if (lane < kCompWarps) s_ball[pb][r * kCompWarps + warp][lane] = mine;
#if SVR_COOP_NZ
            if (lane < kCompWarps && mine) atomicOr(&s_nz[pb][lane], 1u << (r * kCompWarps + warp));
#endif
#endif
        }
    };

    // Composites group buffer g (n slots, records landed).
    auto composite_group = [&](int g, int n) {
        float4* wrec = g ? wrec0 + kCompWarps * 32 * kRecordF4 : wrec0;
        const uint8_t* wsg = s_sign[g][warp];
        // Phase A: this lane's slab hits among the slots.
        uint32_t hits = 0;
        if (!done) {
#pragma unroll kPhaseAUnroll
            for (int sl = 0; sl < n; ++sl) {
                float ta, tb;
                slab_s(WREC(wrec, sl, 0), ix, iy, iz, ssel, ta, tb);
                hits |= uint32_t(ta <= tb && ta > 0.0f) << sl;
            }
        }
        // Phase B: this lane's hits, in entry order.
        while (hits) {
            const int s_ = __ffs(hits) - 1;
            hits &= hits - 1;
            const float4 bb = WREC(wrec, s_, 1);
            const float2 pc = ENTRY ? make_float2(pcx, pcy) : s_pc[ENTRY ? 0 : threadIdx.x];
            if (!((one_sign || wsg[s_] == my_sign) &&
                  !(pc.x < bb.x || pc.x > bb.y || pc.y < bb.z || pc.y > bb.w)))
                continue;
            const float4 lo = WREC(wrec, s_, 0);
            float ta, tb;
#if SVR_PHB_SLABS
            slab_s(lo, ix, iy, iz, ssel, ta, tb);
#else
            slab(lo, ix, iy, iz, ta, tb);
#endif
            const float4 va = WREC(wrec, s_, 2), vb = WREC(wrec, s_, 3);
            const float inv = WREC(wrec, s_, 5).w;
            const float seg = tb - ta;
            const float lk = seg * dnorm * (1.0f / K);
            // voxel_alpha (field.hpp:92-116), K-point midpoint quadrature
            float sa[K], tk[K], sum = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                tk[k] = ta + ((k + 0.5f) / K) * seg;
#if SVR_F32X2_Q
                float qx, qy;  // (qx, qy) in one FFMA2 + FMUL2, same roundings
                up2(mul2(fma2(pk2(tk[k], tk[k]), pk2(dx, dy), pk2(-lo.x, -lo.y)), pk2(inv, inv)), qx, qy);
#else
                const float qx = (tk[k] * dx - lo.x) * inv;
                const float qy = (tk[k] * dy - lo.y) * inv;
#endif
                const float qz = (tk[k] * dz - lo.z) * inv;
                const float act = explin(trilinear_poly(va, vb, qx, qy, qz));
                sum += act;
                sa[k] = one_minus_exp_neg(lk * act);
            }
            const float alpha = (K == 1) ? sa[0] : one_minus_exp_neg(lk * sum);
            if (!RECORD) {
                // voxel_depth (field.hpp:173-181) and the median crossing
                float dv = 0.f, Tk = 1.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dv += Tk * sa[k] * tk[k];
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
                const float4 col = WREC(wrec, s_, 4), nor = WREC(wrec, s_, 5);
#if SVR_F32X2_ACC
                {  // (cr, cg) and (nx, ny) as packed pairs: one FFMA2 each
                    const f32x2 ww = pk2(w, w);
                    f32x2 c2 = fma2(ww, pk2(col.x, col.y), pk2(cr, cg));
                    f32x2 n2 = fma2(ww, pk2(nor.x, nor.y), pk2(nx, ny));
                    up2(c2, cr, cg);
                    up2(n2, nx, ny);
                }
#else
                cr += w * col.x;
                cg += w * col.y;
                nx += w * nor.x;
                ny += w * nor.y;
#endif
                cb += w * col.z;
                nz += w * nor.z;
                depth += T * dv;
                if (EXTRA && a.max_blend) atomicMax(a.max_blend + __float_as_uint(col.w), __float_as_uint(w));
                if (STAGED || (EXTRA && a.stage_entry)) {
                    if (cnt < a.stage_cap) {
                        const uint32_t at = cnt * a.stage_stride + slot;
                        a.stage_entry[at] = s_ent[ENTRY ? g : 0][warp][s_];
                        a.stage_T[at] = T;
                    } else {
                        *a.overflow = 1u;
                    }
                }
            } else {
                a.contrib_entry[rec_base + cnt] = s_ent[ENTRY ? g : 0][warp][s_];
                a.contrib_T[rec_base + cnt] = T;
            }
            T *= 1.0f - alpha;
            ++cnt;
            if (T < thr) {
                done = true;
                hits = 0;
            }
        }
    };

    const uint32_t n_entries = range.y > range.x ? range.y - range.x : 0u;
    const uint32_t n_batches = (n_entries + kBatch - 1) / kBatch;
    int g = 0;            // group buffer being filled
    int nfill = 0;        // slots staged into it
    bool pend = false;    // the other buffer holds a full group not yet composited
    bool wdone = __all_sync(0xffffffffu, done);
#if SVR_COOP_BBPRE
    if (n_batches) {
        load_vals(0);
        load_bb(0);
        produce(0, 0);
        if (n_batches > 1) load_vals(1);
    }
#elif SVR_COOP_VPRE
    if (n_batches) {
        load_vals(0);
        produce(0, 0);
        if (n_batches > 1) load_vals(1);
    }
#else
    if (n_batches) produce(0, 0);
#endif
    __syncthreads();
    for (uint32_t b = 0; b < n_batches; ++b) {
        const int pb = b & 1;
#if SVR_COOP_BBPRE
        if (b + 1 < n_batches) load_bb(b + 1);
#else
        if (b + 1 < n_batches) {
            produce(b + 1, pb ^ 1);
#if SVR_COOP_VPRE
            if (b + 2 < n_batches) load_vals(b + 2);
#endif
        }
#endif
        if (!wdone) {
#if SVR_COOP_NZ
            // only the sub-chunks with survivors for this block (the summary
            // is cleared here; its next writers run after the batch barrier)
            NzWord nzm = s_nz[pb][warp];
            __syncwarp();
            if (lane == 0) s_nz[pb][warp] = 0;
            while (nzm) {
                const int sub = (kBatch > 1024 ? __ffsll((long long)nzm) : __ffs(uint32_t(nzm))) - 1;
                nzm &= nzm - 1;
#else
            for (int sub = 0; sub < kSubs; ++sub) {
#endif
#if SVR_COOP_BYTES
                uint32_t ball = __ballot_sync(0xffffffffu, (s_mb[pb][sub][lane] >> warp) & 1u);
#else
                uint32_t ball = s_ball[pb][sub][warp];
#endif
                const uint32_t e0 = range.x + b * kBatch + sub * 32;
                while (ball) {
                    const int take = min(32 - nfill, __popc(ball));
                    // the first `take` survivors (entry order) go to group g
                    const uint32_t part =
                        take == __popc(ball)
                            ? ball
                            : __ballot_sync(0xffffffffu, ((ball >> lane) & 1u) &&
                                                             __popc(ball & ((1u << lane) - 1u)) < take);
                    ball &= ~part;
                    if ((part >> lane) & 1u) {
                        const int at = nfill + __popc(part & ((1u << lane) - 1u));
                        const uint32_t v = __ldg(a.vals + e0 + lane);
                        s_sign[g][warp][at] = uint8_t(v >> 29);
                        if (ENTRY) s_ent[ENTRY ? g : 0][warp][at] = e0 + lane;
                        const float4* src = a.records + uint64_t(v & kVidMask) * kRecordF4;
                        float4* wrec = g ? wrec0 + kCompWarps * 32 * kRecordF4 : wrec0;
#pragma unroll
                        for (int k = 0; k < kRecordF4; ++k) cp_async16<MODE == 0>(&WREC(wrec, at, k), src + k);
                    }
                    nfill += take;
                    if (nfill == 32) {  // group full: composite the previous one meanwhile
                        cp_async_commit();
                        if (pend) {
                            cp_async_wait<1>();
                            __syncwarp();
                            composite_group(g ^ 1, 32);
                            __syncwarp();  // its buffer is restaged next
                        }
                        pend = true;
                        g ^= 1;
                        nfill = 0;
                        wdone = __all_sync(0xffffffffu, done);
                        if (wdone) break;
                    }
                }
                if (wdone) break;
            }
        }
#if SVR_COOP_BBPRE
        if (b + 1 < n_batches) {  // every warp culls, composited or done
            produce(b + 1, pb ^ 1);
            if (b + 2 < n_batches) load_vals(b + 2);
        }
#endif
        // ballot buffer pb is rewritten by the produce two batches on
        if (__syncthreads_and(wdone)) break;
    }
    // drain: the pending full group, then the partial one
    cp_async_commit();
    if (!wdone) {
        if (pend) {
            cp_async_wait<1>();
            __syncwarp();
            composite_group(g ^ 1, 32);
        }
        cp_async_wait<0>();
        __syncwarp();
        if (nfill) composite_group(g, nfill);
    }
    cp_async_wait<0>();  // no copy may outlive the CTA's shared memory
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

// CTAs per SM the register allocation targets: 4 for the plain render (63
// registers; 3 with 75 is 3 % slower), 3 for the recording modes, whose
// extra state spills otherwise (config 3 staged render 316 -> 296 us).
#ifndef SVR_COOP_MINB0
#define SVR_COOP_MINB0 4  // CTAs per SM of the cooperative plain render
#endif
#define SVR_COOP_MINB(MODE) ((MODE) == 0 ? SVR_COOP_MINB0 : 3)
#ifndef SVR_COMP_MINB
#define SVR_COMP_MINB(MODE) ((MODE) == 0 ? 4 : 3)
#endif
// K7: one CTA per tile (LPT order), warp-autonomous or CTA-cooperative
// (launch_composite picks per frame: the cooperative cull pays once tiles
// hold thousands of entries — config 4, ~22K per tile: 3.62 -> 2.11 ms — and
// costs its batch barrier on short lists — config 2, ~430: 0.33 -> 0.38 ms).
template <int K, int MODE>
__global__ void __launch_bounds__(256, SVR_COMP_MINB(MODE)) composite_kernel(DevCamera cam, CompositeArgs a) {
    pdl_enter();
    extern __shared__ float4 s_rec_dyn[];  // [2][8 warps][32 slots][kRecordF4]
    __shared__ CompShared<K, MODE> sh;
    const int tile = a.tile_order ? int(a.tile_order[blockIdx.x]) : int(blockIdx.x);
    composite_tile_warp<K, MODE>(cam, a, tile, sh, s_rec_dyn);
}

template <int K, int MODE>
__global__ void __launch_bounds__(256, SVR_COOP_MINB(MODE)) composite_coop_kernel(DevCamera cam, CompositeArgs a) {
    pdl_enter();
    extern __shared__ float4 s_rec_dyn[];
    __shared__ CompShared<K, MODE> sh;
    const int tile = a.tile_order ? int(a.tile_order[blockIdx.x]) : int(blockIdx.x);
    composite_tile_coop<K, MODE>(cam, a, tile, sh, s_rec_dyn);
}

__global__ void compact_contribs_kernel(const uint32_t* __restrict__ pix_count,
                                        const uint32_t* __restrict__ pix_begin,
                                        const uint32_t* __restrict__ stage_entry,
                                        const float* __restrict__ stage_T, uint32_t stride,
                                        uint32_t* contrib_entry, float* contrib_T) {
    pdl_enter();
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= stride) return;
    const uint32_t n = pix_count[slot], b = pix_begin[slot];
    for (uint32_t k = 0; k < n; ++k) {
        contrib_entry[b + k] = stage_entry[uint64_t(k) * stride + slot];
        contrib_T[b + k] = stage_T[uint64_t(k) * stride + slot];
    }
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
    const float ix = slab_inv(dd[0]), iy = slab_inv(dd[1]), iz = slab_inv(dd[2]);
    const uint32_t n = pix_count[slot], base = pix_begin[slot];
    for (uint32_t c = 0; c < n; ++c) {
        uint32_t e = contrib_entry[base + c];
        uint32_t vid = vals[e] & ((1u << 29) - 1u);
        const float4 lo = records[uint64_t(vid) * kRecordF4 + 0];
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

// Frame summary -> mapped pinned host memory, written by the SM over PCIe:
// no copy-engine transfer, so this read-back never queues behind a large
// asynchronous image download on the copy stream.
__global__ void status_to_host_kernel(const FrameStatus* d, FrameStatus* h, uint64_t cap,
                                      unsigned int* overflow_count) {
    pdl_enter();
    *h = *d;
    if (overflow_count && d->n_entries + d->n_huge_entries > cap) atomicAdd(overflow_count, 1u);
}

inline unsigned blocks_for(uint64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

void launch_status_to_host(const FrameStatus* d, FrameStatus* h, cudaStream_t st, uint64_t cap,
                           unsigned int* overflow_count) {
    launch_pdl(status_to_host_kernel, 1, 1, 0, st, d, h, cap, overflow_count);
    SVR_LAUNCH("status_to_host_kernel");
}

void launch_tile_setup(const DevCamera& cam, uint8_t* masks, uint32_t* sat, FrameStatus* status,
                       cudaStream_t st, int2* rowspan) {
    const int ncell = (cam.ntx + 1) * (cam.nty + 1);
    const int use_smem = ncell <= kSatSmemMax;
    const size_t smem = use_smem ? size_t(ncell) * 4 : 0;
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set))
        SVR_CUDA(cudaFuncSetAttribute(tile_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSatSmemMax * 4));
    // masks: one thread per tile (fp64 corner rays); then the SAT in one CTA
    const int ntiles = cam.ntx * cam.nty;
    launch_pdl(tile_masks_kernel, blocks_for(ntiles, 128), 128, 0, st, cam, masks);
    SVR_LAUNCH("tile_masks_kernel");
    launch_pdl(tile_setup_kernel, rowspan ? 9 : 1, 1024, smem, st, cam, masks, sat, status, use_smem, rowspan);
    SVR_LAUNCH("tile_setup_kernel");
}

void launch_tile_masks_only(const DevCamera& cam, uint8_t* masks, cudaStream_t st) {
    int n = cam.ntx * cam.nty;
    tile_masks_kernel<<<blocks_for(n, 256), 256, 0, st>>>(cam, masks);
    SVR_LAUNCH("tile_masks_kernel");
}

void launch_preprocess(const DevCamera& cam, const PreprocessArgs& args, cudaStream_t st) {
    if (args.n == 0) return;
    PreprocessArgs a = args;
    a.cull = cull_norms(cam);
    const size_t smem = a.order ? 0 : size_t(kPreThreads) * kRecordF4 * 16;
    if (a.n_order) {  // worklist mode: a.order is filled by the pre-cull pass
        launch_pdl(precull_kernel, blocks_for(a.n, 256), 256, 0, st, cam, a, const_cast<uint32_t*>(a.order),
                   const_cast<unsigned int*>(a.n_order));
        SVR_LAUNCH("precull_kernel");
    }
    launch_pdl(preprocess_kernel, blocks_for(a.n, kPreThreads), kPreThreads, smem, st, cam, a);
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

void launch_duplicate_packed(const DevCamera& cam, uint64_t n, const uint64_t* paths,
                             const int4* rects, const uint8_t* masks, const uint32_t* counts,
                             const uint32_t* offsets, PackedFormat fmt, const uint32_t* rank,
                             uint64_t* keys, const uint32_t* tile_sat, uint32_t* big,
                             unsigned int* n_big, cudaStream_t st, uint64_t cap) {
    if (n == 0) return;
    launch_pdl(duplicate_packed_kernel, blocks_for(n, 256), 256, 0, st, cam, n, paths, rects, masks,
               counts, offsets, fmt, rank, keys, big, n_big, cap);
    SVR_LAUNCH("duplicate_packed_kernel");
    launch_pdl(duplicate_big_kernel, 148 * 4, 256, 0, st, cam, n, paths, rects, masks, offsets, tile_sat,
                                                   fmt, rank, keys, big, n_big);
    SVR_LAUNCH("duplicate_big_kernel");
}

void launch_pair_counts(const DevCamera& cam, uint64_t n, const uint32_t* counts, const int4* rects,
                        const uint32_t* sat, FrameStatus* status, const uint32_t* rank,
                        uint32_t* pc, uint32_t* block_sums, cudaStream_t st, const HugePairs& huge) {
    if (n == 0) return;
    SVR_CUDA(cudaMemsetAsync(pc, 0, 8 * n * sizeof(uint32_t), st));
    if (block_sums)
        SVR_CUDA(cudaMemsetAsync(block_sums, 0, (8 * n + kScanChunk - 1) / kScanChunk * sizeof(uint32_t), st));
    if (huge.divert && huge.cap) {  // padding sorts last by rank and by pattern
        SVR_CUDA(cudaMemsetAsync(huge.keys, 0xff, size_t(huge.cap) * 8, st));
        SVR_CUDA(cudaMemsetAsync(huge.vals, 0xff, size_t(huge.cap) * 4, st));
    }
    launch_pdl(pair_counts_kernel, blocks_for(n, 256), 256, 0, st, cam, n, counts, rects, sat, status, rank,
               pc, block_sums, huge);
    SVR_LAUNCH("pair_counts_kernel");
}

void launch_merge_huge(const DevCamera& cam, const HugePairs& huge, const uint64_t* hkeys,
                       const uint32_t* hvals, const uint64_t* skeys_s, const uint32_t* svals_s,
                       const FrameStatus* status, const int4* rects,
                       const uint8_t* masks, const uint64_t* small_keys, const uint2* small_ranges,
                       PackedFormat fmt, int* diff, uint4* packed, uint32_t* apos, uint2* ranges,
                       uint32_t* vals, uint64_t cap, unsigned long long* n_total, cudaStream_t st) {
    const int ntiles = cam.ntx * cam.nty;
    if (ntiles > 4096) throw Error(SVR_ERR_RUNTIME, "huge-pair merge supports at most 4096 tiles");
    const size_t ncell = size_t(cam.ntx + 1) * (cam.nty + 1);
    SVR_CUDA(cudaMemsetAsync(diff, 0, 8 * ncell * sizeof(int), st));
    launch_pdl(huge_cover_kernel, std::max(1u, blocks_for(huge.cap, 256)), 256, 0, st, cam, huge, hvals,
               status, rects, diff);
    SVR_LAUNCH("huge_cover_kernel");
    launch_pdl(huge_ranges_kernel, 1, kMergeThreads, 0, st, cam, status, masks, diff, small_ranges, ranges,
               n_total);
    SVR_LAUNCH("huge_ranges_kernel");
    uint4* packed_s = packed + huge.cap;
    uint32_t* sb = reinterpret_cast<uint32_t*>(packed_s + huge.cap);
    SVR_CUDA(cudaMemsetAsync(sb, 0, 16 * sizeof(uint32_t), st));
    launch_pdl(huge_pack_kernel, std::max(1u, blocks_for(huge.cap, 256)), 256, 0, st, huge, hkeys, hvals,
               skeys_s, svals_s, status, rects, packed, packed_s, sb);
    SVR_LAUNCH("huge_pack_kernel");
    launch_pdl(huge_apos_kernel, 148u * 8u, 256, 0, st, cam, small_keys, status, cap, fmt, huge, masks,
               const_cast<const uint4*>(packed), const_cast<const uint4*>(packed_s),
               const_cast<const uint32_t*>(sb), apos);
    SVR_LAUNCH("huge_apos_kernel");
    constexpr size_t kMergeDyn = size_t(kMergeTiles) * kMergeStep * 2;
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set))
        SVR_CUDA(cudaFuncSetAttribute(merge_huge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kMergeDyn)));
    launch_pdl(merge_huge_kernel, unsigned(ntiles + (ntiles + kMergeTiles - 1) / kMergeTiles), 256, kMergeDyn,
               st, cam, huge, const_cast<const uint4*>(packed), const_cast<const uint4*>(packed_s),
               const_cast<const uint32_t*>(sb), status, masks, small_keys, const_cast<const uint32_t*>(apos),
               small_ranges, fmt, ranges, vals, cap, n_total);
    SVR_LAUNCH("merge_huge_kernel");
}

void launch_duplicate_ranked(const DevCamera& cam, uint64_t n, const uint32_t* pc,
                             const uint32_t* partial, const uint32_t* order, const int4* rects,
                             const uint8_t* masks, const uint32_t* sat, const int2* rowspan,
                             PackedFormat fmt, uint64_t* keys, uint64_t cap, uint2* big,
                             unsigned int* n_big, cudaStream_t st, TileDigits td) {
    if (n == 0) return;
    const uint64_t m = 8 * n;
    launch_pdl(duplicate_ranked_kernel, unsigned((m + kScanChunk - 1) / kScanChunk), kScanThreads, 0, st, cam,
               m, pc, partial, order, rects, masks, rowspan, fmt, keys, cap, big, n_big, td);
    SVR_LAUNCH("duplicate_ranked_kernel");
    launch_pdl(duplicate_big_ranked_kernel, 148 * 8, 256, 0, st, cam, order, rects, masks, sat, rowspan, fmt,
               keys, big, n_big, td);
    SVR_LAUNCH("duplicate_big_ranked_kernel");
}

size_t morton_rank_scratch_bytes(uint64_t n, int lmax) {
    const uint64_t m = 8 * n;
    const int npass = (3 * lmax + 7) / 8;
    return 2 * m * 8 + 2 * m * 4 + 256 + sort_scratch_bytes(m, npass);
}

void build_morton_rank(const uint64_t* paths, uint64_t n, int lmax, uint32_t* rank, uint32_t* order,
                       void* scratch, cudaStream_t st) {
    if (n == 0) return;
    const uint64_t m = 8 * n;
    char* p = static_cast<char*>(scratch);
    uint64_t* k0 = reinterpret_cast<uint64_t*>(p);
    uint64_t* k1 = k0 + m;
    uint32_t* v0 = reinterpret_cast<uint32_t*>(k1 + m);
    uint32_t* v1 = v0 + m;
    void* sort_scratch = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(v1 + m) + 255) &
                                                 ~uintptr_t(255));
    rank_keys_kernel<<<blocks_for(m, 256), 256, 0, st>>>(paths, n, k0, v0);
    SVR_LAUNCH("rank_keys_kernel");
    // (code ^ s*G) differs only in bits [48 - 3*lmax, 48); the pairs are
    // generated in ascending value order, so the stable sort breaks key ties
    // by value exactly as std::sort on (key, value) does.
    RadixPass passes[kMaxRadixPasses];
    int np = 0;
    for (int b = 48 - 3 * lmax; b < 48; b += 8) passes[np++] = {0, b, std::min(8, 48 - b)};
    int out = 0;
    if (np > 0) out = radix_sort_pairs(k0, v0, k1, v1, m, passes, np, sort_scratch, st);
    rank_scatter_kernel<<<blocks_for(m, 256), 256, 0, st>>>(out ? v1 : v0, n, rank);
    SVR_LAUNCH("rank_scatter_kernel");
    if (order) SVR_CUDA(cudaMemcpyAsync(order, out ? v1 : v0, m * 4, cudaMemcpyDeviceToDevice, st));
}

void launch_tile_ranges_packed(const uint64_t* keys, uint64_t n, PackedFormat fmt, uint2* ranges,
                               uint32_t* vals, int ntiles, cudaStream_t st,
                               const unsigned long long* n_dev) {
    SVR_CUDA(cudaMemsetAsync(ranges, 0, size_t(ntiles) * sizeof(uint2), st));
    if (n == 0) return;
    launch_pdl(tile_ranges_packed_kernel, blocks_for(n, 256), 256, 0, st, keys, n, fmt, ranges, vals, n_dev);
    SVR_LAUNCH("tile_ranges_packed_kernel");
}

void launch_unpack_entries(const uint64_t* packed, uint64_t n, PackedFormat fmt,
                           const uint64_t* paths, uint64_t* keys, uint32_t* vals, cudaStream_t st) {
    if (n == 0) return;
    unpack_entries_kernel<<<blocks_for(n, 256), 256, 0, st>>>(packed, n, fmt, paths, keys, vals);
    SVR_LAUNCH("unpack_entries_kernel");
}

void launch_tile_ranges(const uint64_t* keys, uint64_t n, uint2* ranges, int ntiles,
                        cudaStream_t st) {
    SVR_CUDA(cudaMemsetAsync(ranges, 0, size_t(ntiles) * sizeof(uint2), st));
    if (n == 0) return;
    tile_ranges_kernel<<<blocks_for(n, 256), 256, 0, st>>>(keys, n, ranges);
    SVR_LAUNCH("tile_ranges_kernel");
}

void launch_compact_contribs(const uint32_t* pix_count, const uint32_t* pix_begin,
                             const uint32_t* stage_entry, const float* stage_T, uint32_t stride,
                             uint32_t* contrib_entry, float* contrib_T, cudaStream_t st) {
    if (stride == 0) return;
    launch_pdl(compact_contribs_kernel, blocks_for(stride, 256), 256, 0, st, pix_count, pix_begin,
               stage_entry, stage_T, stride, contrib_entry, contrib_T);
    SVR_LAUNCH("compact_contribs_kernel");
}

void launch_tile_order(uint2* ranges, int ntiles, uint32_t* order, cudaStream_t st) {
    launch_pdl(tile_order_kernel, 1, 1024, 0, st, ranges, ntiles, order);
    SVR_LAUNCH("tile_order_kernel");
}

void launch_composite(const DevCamera& cam, const CompositeArgs& a, bool record_pass, bool coop,
                      cudaStream_t st) {
    const unsigned ntiles = unsigned(cam.ntx * cam.nty);
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) {
        for (auto fn : {composite_kernel<1, 0>, composite_kernel<1, 1>, composite_kernel<1, 2>,
                        composite_kernel<1, 3>, composite_kernel<2, 0>, composite_kernel<2, 1>,
                        composite_kernel<2, 2>, composite_kernel<2, 3>, composite_kernel<3, 0>,
                        composite_kernel<3, 1>, composite_kernel<3, 2>, composite_kernel<3, 3>,
                        composite_coop_kernel<1, 0>, composite_coop_kernel<1, 1>,
                        composite_coop_kernel<1, 2>, composite_coop_kernel<1, 3>,
                        composite_coop_kernel<2, 0>, composite_coop_kernel<2, 1>,
                        composite_coop_kernel<2, 2>, composite_coop_kernel<2, 3>,
                        composite_coop_kernel<3, 0>, composite_coop_kernel<3, 1>,
                        composite_coop_kernel<3, 2>, composite_coop_kernel<3, 3>})
            SVR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCompSmem)));
    }
    const int mode = record_pass ? 1 : a.max_blend ? 2 : a.stage_entry ? 3 : 0;
#define SVR_COMPOSITE_LAUNCH(KK, MM)                                                    \
    if (coop)                                                                           \
        launch_pdl(composite_coop_kernel<KK, MM>, ntiles, 256, kCompSmem, st, cam, a); \
    else                                                                                \
        launch_pdl(composite_kernel<KK, MM>, ntiles, 256, kCompSmem, st, cam, a);
#define SVR_COMPOSITE_CASE(KK)                                                          \
    case KK:                                                                            \
        if (mode == 1) {                                                                \
            SVR_COMPOSITE_LAUNCH(KK, 1)                                                 \
        } else if (mode == 2) {                                                         \
            SVR_COMPOSITE_LAUNCH(KK, 2)                                                 \
        } else if (mode == 3) {                                                         \
            SVR_COMPOSITE_LAUNCH(KK, 3)                                                 \
        } else {                                                                        \
            SVR_COMPOSITE_LAUNCH(KK, 0)                                                 \
        }                                                                               \
        break;
    switch (a.K) {
        SVR_COMPOSITE_CASE(1)
        SVR_COMPOSITE_CASE(2)
        SVR_COMPOSITE_CASE(3)
        default:
            throw Error(SVR_ERR_INVALID_ARGUMENT, "rasterizer sample count K must be in {1,2,3}");
    }
#undef SVR_COMPOSITE_CASE
#undef SVR_COMPOSITE_LAUNCH
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
