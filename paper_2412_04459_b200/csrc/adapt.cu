// adapt.cu — scene adaptation on the device:
// prune (optim.cpp:207-234) and subdivide_voxels (optim.cpp:236-298), each
// followed by rebuild_corner_indexing (scene.cpp:8-26), as sort-based passes.
//
// rebuild_corner_indexing assigns pool entries in order of FIRST APPEARANCE
// of a corner lattice key while walking voxels in order and corners 0..7.
// On the device: the 8N keys are stably sorted with their position
// p = 8*voxel + corner; the head of each equal-key run holds the run's
// smallest p; flagging those positions and scanning the flags in position
// order gives every run its pool index; a gather writes corner_index.
// Densities come from the old scene's key -> pool map (binary search in its
// sorted unique keys), from the subdivision's fresh averages, or `fill`.
//
// Fresh subdivision points (optim.cpp:266-281) are the mean of
// trilinear(parent V, q) over every (parent, child, corner) that produces the
// key; the contributions are emitted in the reference's loop order and summed
// sequentially per key after a stable sort, in double, so the float that
// lands in the pool is bit-identical. Remaps (AdaptRemap: voxel_src,
// pool_src) are produced the same way.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {

namespace {

constexpr uint64_t kMask48 = (uint64_t(1) << 48) - 1;

__device__ __forceinline__ void voxel_ijk(uint64_t path, uint32_t& i, uint32_t& j, uint32_t& k,
                                          int& lv) {
    lv = int(path >> 48);
    uint64_t c = (path & kMask48) >> (3 * (kMaxLevel - lv));
    i = j = k = 0;
    for (int n = 0; n < lv; ++n) {  // to_voxel_index (octree.hpp:68-82)
        i |= uint32_t((c >> 2) & 1) << n;
        j |= uint32_t((c >> 1) & 1) << n;
        k |= uint32_t(c & 1) << n;
        c >>= 3;
    }
}

// corner_keys (octree.hpp:130-139) + CornerKey::packed (126)
__device__ __forceinline__ uint64_t corner_key(uint32_t i, uint32_t j, uint32_t k, int lv, int c) {
    const uint32_t step = uint32_t(1) << (kMaxLevel - lv);
    return (uint64_t((i + ((c >> 2) & 1)) * step) << 34) | (uint64_t((j + ((c >> 1) & 1)) * step) << 17) |
           uint64_t((k + (c & 1)) * step);
}

__global__ void corner_keys_kernel(const uint64_t* __restrict__ paths, uint64_t n, uint64_t* keys,
                                   uint32_t* pos) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    uint32_t i, j, k;
    int lv;
    voxel_ijk(paths[v], i, j, k, lv);
    for (int c = 0; c < 8; ++c) {
        keys[8 * v + c] = corner_key(i, j, k, lv, c);
        pos[8 * v + c] = uint32_t(8 * v + c);
    }
}

// heads of equal-key runs of the sorted keys: first-appearance flags by
// position, and run heads in sorted order
__global__ void run_heads_kernel(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ spos,
                                 uint64_t m, uint32_t* first_flag, uint32_t* head) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const bool h = j == 0 || skeys[j] != skeys[j - 1];
    head[j] = h;
    if (h) first_flag[spos[j]] = 1u;
}

// run id g (exclusive scan of heads, minus... computed as incl - 1) ->
// pool index of the run = rank of its first position; corner_index and the
// pool's key per entry
__global__ void assign_pool_kernel(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ spos,
                                   const uint32_t* __restrict__ head, const uint32_t* __restrict__ head_excl,
                                   const uint32_t* __restrict__ first_rank, uint64_t m,
                                   uint32_t* run_pool, uint64_t* pool_key) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m || !head[j]) return;
    const uint32_t g = head_excl[j];
    const uint32_t p = first_rank[spos[j]];
    run_pool[g] = p;
    pool_key[p] = skeys[j];
}

__global__ void scatter_corner_index_kernel(const uint32_t* __restrict__ spos,
                                            const uint32_t* __restrict__ head,
                                            const uint32_t* __restrict__ head_excl,
                                            const uint32_t* __restrict__ run_pool, uint64_t m,
                                            uint32_t* corner_index) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const uint32_t g = head_excl[j] + head[j] - 1;  // inclusive - 1
    corner_index[spos[j]] = run_pool[g];
}

// unique (key, pool) table of a consistent scene: the head of every run
__global__ void unique_keys_kernel(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ spos,
                                   const uint32_t* __restrict__ head, const uint32_t* __restrict__ head_excl,
                                   const uint32_t* __restrict__ corner_index, uint64_t m, uint64_t* ukey,
                                   uint32_t* upool) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m || !head[j]) return;
    const uint32_t g = head_excl[j];
    ukey[g] = skeys[j];
    upool[g] = corner_index[spos[j]];
}

__device__ __forceinline__ int64_t find_key(const uint64_t* __restrict__ ukey, uint64_t nu, uint64_t k) {
    uint64_t lo = 0, hi = nu;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (ukey[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return (lo < nu && ukey[lo] == k) ? int64_t(lo) : -1;
}

// densities + pool_src of the new pool (rebuild_corner_indexing's
// key_density lookup, scene.cpp:18-21; pool_sources, optim.cpp:190-205)
__global__ void pool_density_kernel(const uint64_t* __restrict__ pool_key, uint64_t np,
                                    const uint64_t* __restrict__ old_ukey, const uint32_t* __restrict__ old_upool,
                                    uint64_t n_old_u, const float* __restrict__ old_density,
                                    const uint64_t* __restrict__ fresh_key, const float* __restrict__ fresh_val,
                                    uint64_t n_fresh, float fill, float* density, int64_t* pool_src) {
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= np) return;
    const uint64_t k = pool_key[p];
    const int64_t o = find_key(old_ukey, n_old_u, k);
    if (o >= 0) {
        density[p] = old_density[old_upool[o]];
        pool_src[p] = int64_t(old_upool[o]);
        return;
    }
    pool_src[p] = -1;
    const int64_t f = n_fresh ? find_key(fresh_key, n_fresh, k) : -1;
    density[p] = f >= 0 ? fresh_val[f] : fill;
}

// prune: kept voxels, in order (optim.cpp:219-224)
__global__ void keep_flags_kernel(const float* __restrict__ stat, uint64_t n, double thr, uint32_t* keep) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v < n) keep[v] = double(stat[v]) >= thr;
}

__global__ void compact_voxels_kernel(const uint64_t* __restrict__ paths, const uint32_t* __restrict__ keep,
                                      const uint32_t* __restrict__ at, uint64_t n, uint64_t* out_paths,
                                      int64_t* voxel_src, int64_t* sh_src) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n || !keep[v]) return;
    out_paths[at[v]] = paths[v];
    voxel_src[at[v]] = int64_t(v);
    sh_src[at[v]] = int64_t(v);
}

// subdivide: 8 children in place of each selected voxel (optim.cpp:263-289)
__global__ void subdivide_voxels_kernel(const uint64_t* __restrict__ paths, const uint32_t* __restrict__ sel,
                                        const uint32_t* __restrict__ at, uint64_t n, uint64_t* out_paths,
                                        int64_t* voxel_src, int64_t* sh_src) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const uint64_t o = at[v];
    if (!sel[v]) {
        out_paths[o] = paths[v];
        voxel_src[o] = int64_t(v);
        sh_src[o] = int64_t(v);
        return;
    }
    const int lv = int(paths[v] >> 48);
    const int shift = 3 * (kMaxLevel - lv - 1);  // child_paths (octree.hpp:103-110)
    for (uint64_t c = 0; c < 8; ++c) {
        out_paths[o + c] = ((paths[v] & kMask48) | (c << shift)) | (uint64_t(lv + 1) << 48);
        voxel_src[o + c] = -1;
        sh_src[o + c] = int64_t(v);
    }
}

// fresh points: per selected parent (rank r among the selected, in voxel
// order), child c, corner q -> 64 contributions, in the reference's loop
// order; those whose key already exists are marked invalid (key = ~0)
__global__ void fresh_contribs_kernel(const uint64_t* __restrict__ paths, const uint32_t* __restrict__ sel,
                                      const uint32_t* __restrict__ sel_rank, uint64_t n,
                                      const uint32_t* __restrict__ corner_index,
                                      const float* __restrict__ density,
                                      const uint64_t* __restrict__ old_ukey, uint64_t n_old_u,
                                      uint64_t* keys, uint32_t* order, double* vals) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= n || !sel[v]) return;
    const uint64_t base = uint64_t(sel_rank[v]) * 64;
    uint32_t i, j, k;
    int lv;
    voxel_ijk(paths[v], i, j, k, lv);
    double V[8];
    for (int c = 0; c < 8; ++c) V[c] = double(density[corner_index[8 * v + c]]);  // corners_of
    for (int ch = 0; ch < 8; ++ch) {
        // child voxel index at level lv+1
        const uint32_t ci = (i << 1) | ((ch >> 2) & 1), cj = (j << 1) | ((ch >> 1) & 1),
                       ck = (k << 1) | (ch & 1);
        for (int c = 0; c < 8; ++c) {
            const uint64_t at = base + uint64_t(ch) * 8 + c;
            const uint64_t key = corner_key(ci, cj, ck, lv + 1, c);
            order[at] = uint32_t(at);
            if (find_key(old_ukey, n_old_u, key) >= 0) {
                keys[at] = ~uint64_t(0);
                vals[at] = 0.0;
                continue;
            }
            // child-corner position in the parent's local coordinates
            const double q[3] = {0.5 * double((ci & 1) + ((c >> 2) & 1)),
                                 0.5 * double((cj & 1) + ((c >> 1) & 1)),
                                 0.5 * double((ck & 1) + (c & 1))};
            // trilinear(V, q) in the reference's operation order (field.hpp:33-47)
            const double wx[2] = {__dsub_rn(1.0, q[0]), q[0]}, wy[2] = {__dsub_rn(1.0, q[1]), q[1]},
                         wz[2] = {__dsub_rn(1.0, q[2]), q[2]};
            double s = 0.0;
            for (int cc = 0; cc < 8; ++cc) {
                const double w = __dmul_rn(__dmul_rn(wx[(cc >> 2) & 1], wy[(cc >> 1) & 1]), wz[cc & 1]);
                s = __dadd_rn(s, __dmul_rn(w, V[cc]));
            }
            keys[at] = key;
            vals[at] = s;
        }
    }
}

// per run of equal keys (sorted stably, so in loop order): sequential double
// sum and count -> float(sum / count) (optim.cpp:281)
__global__ void fresh_average_kernel(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ sorder,
                                     const double* __restrict__ vals, const uint32_t* __restrict__ head,
                                     const uint32_t* __restrict__ head_excl, uint64_t m, uint64_t* fkey,
                                     float* fval) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m || !head[j] || skeys[j] == ~uint64_t(0)) return;
    double s = 0.0;
    int cnt = 0;
    for (uint64_t t = j; t < m && skeys[t] == skeys[j]; ++t) {
        s = __dadd_rn(s, vals[sorder[t]]);
        ++cnt;
    }
    const uint32_t g = head_excl[j];
    fkey[g] = skeys[j];
    fval[g] = float(__ddiv_rn(s, double(cnt)));
}

__global__ void gather_sh_kernel(const float* __restrict__ sh, const int64_t* __restrict__ sh_src,
                                 uint64_t n, int stride, float* out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * uint64_t(stride)) return;
    const uint64_t v = i / uint64_t(stride), e = i - v * uint64_t(stride);
    out[i] = sh[uint64_t(sh_src[v]) * stride + e];
}

__global__ void max_level_kernel(const uint64_t* __restrict__ paths, uint64_t n, unsigned int* out) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned int lv = v < n ? unsigned(paths[v] >> 48) : 0u;
    lv = __reduce_max_sync(0xffffffffu, lv);
    if ((threadIdx.x & 31) == 0 && lv) atomicMax(out, lv);
}

inline unsigned blocks_for(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

// Sorted (key, pos) of a key array with run heads and their exclusive scan.
struct SortedKeys {
    DevBuf keys[2], pos[2], head, head_excl;
    uint64_t* skeys = nullptr;
    uint32_t* spos = nullptr;
    uint64_t m = 0, runs = 0;
};

void sort_keys_with_pos(svr_ctx* ctx, SortedKeys& s, uint64_t m, int key_bits, cudaStream_t st) {
    s.m = m;
    RadixPass passes[kMaxRadixPasses];
    int np = 0;
    for (int b = 0; b < key_bits; b += 8) passes[np++] = {0, b, std::min(8, key_bits - b)};
    DevBuf scratch;
    scratch.reserve(sort_scratch_bytes(std::max<uint64_t>(m, 2), np));
    const int out = m > 1 ? radix_sort_pairs(s.keys[0].as<uint64_t>(), s.pos[0].as<uint32_t>(),
                                             s.keys[1].as<uint64_t>(), s.pos[1].as<uint32_t>(), m,
                                             passes, np, scratch.p, st)
                          : 0;
    s.skeys = s.keys[out].as<uint64_t>();
    s.spos = s.pos[out].as<uint32_t>();
    SVR_CUDA(cudaStreamSynchronize(st));  // scratch goes out of scope
    (void)ctx;
}

uint64_t scan_total(svr_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st) {
    DevBuf scratch, tot;
    scratch.reserve(scan_scratch_bytes(std::max<uint64_t>(n, 1)));
    tot.reserve(8);
    SVR_CUDA(cudaMemsetAsync(tot.p, 0, 8, st));
    if (n) exclusive_scan_u32(in, out, n, tot.as<unsigned long long>(), scratch.p, st);
    unsigned long long h = 0;
    SVR_CUDA(cudaMemcpyAsync(&h, tot.p, 8, cudaMemcpyDeviceToHost, st));
    SVR_CUDA(cudaStreamSynchronize(st));
    (void)ctx;
    return h;
}

}  // namespace

void launch_keep_flags(const float* stat, uint64_t n, double thr, uint32_t* keep, cudaStream_t st) {
    keep_flags_kernel<<<blocks_for(n, 256), 256, 0, st>>>(stat, n, thr, keep);
    SVR_LAUNCH("keep_flags_kernel");
}

// The device half of prune / subdivide_voxels. flags: per old voxel, keep
// (prune) or selected (subdivide), device u32. Returns the new scene with
// its AdaptRemap stored on it.
svr_scene* adapt_scene(svr_ctx* ctx, const svr_scene* old, const uint32_t* flags, bool subdivide,
                       float fill) {
    cudaStream_t st = ctx->stream;
    const uint64_t N = old->n_voxels;
    const int stride = old->sh_stride;
    // 1. old key -> pool table (corner_key_to_pool, scene.cpp:28-36)
    SortedKeys ok;
    const uint64_t m_old = 8 * N;
    for (int b = 0; b < 2; ++b) {
        ok.keys[b].reserve(std::max<uint64_t>(m_old, 1) * 8);
        ok.pos[b].reserve(std::max<uint64_t>(m_old, 1) * 4);
    }
    if (N) {
        corner_keys_kernel<<<blocks_for(N, 256), 256, 0, st>>>(old->paths.as<uint64_t>(), N,
                                                               ok.keys[0].as<uint64_t>(), ok.pos[0].as<uint32_t>());
        SVR_LAUNCH("corner_keys_kernel");
    }
    sort_keys_with_pos(ctx, ok, m_old, 51, st);
    ok.head.reserve(std::max<uint64_t>(m_old, 1) * 4);
    ok.head_excl.reserve(std::max<uint64_t>(m_old, 1) * 4);
    DevBuf scratch_first;
    scratch_first.reserve(std::max<uint64_t>(m_old, 1) * 4);
    SVR_CUDA(cudaMemsetAsync(scratch_first.p, 0, std::max<uint64_t>(m_old, 1) * 4, st));
    if (m_old) {
        run_heads_kernel<<<blocks_for(m_old, 256), 256, 0, st>>>(ok.skeys, ok.spos, m_old,
                                                                 scratch_first.as<uint32_t>(), ok.head.as<uint32_t>());
        SVR_LAUNCH("run_heads_kernel");
    }
    const uint64_t n_old_u = scan_total(ctx, ok.head.as<uint32_t>(), ok.head_excl.as<uint32_t>(), m_old, st);
    DevBuf old_ukey, old_upool;
    old_ukey.reserve(std::max<uint64_t>(n_old_u, 1) * 8);
    old_upool.reserve(std::max<uint64_t>(n_old_u, 1) * 4);
    if (m_old) {
        unique_keys_kernel<<<blocks_for(m_old, 256), 256, 0, st>>>(
            ok.skeys, ok.spos, ok.head.as<uint32_t>(), ok.head_excl.as<uint32_t>(),
            old->corner_index.as<uint32_t>(), m_old, old_ukey.as<uint64_t>(), old_upool.as<uint32_t>());
        SVR_LAUNCH("unique_keys_kernel");
    }

    // 2. new voxel list + voxel_src / sh_src
    DevBuf cnt, at;
    cnt.reserve(std::max<uint64_t>(N, 1) * 4);
    at.reserve(std::max<uint64_t>(N, 1) * 4);
    uint64_t N2 = 0;
    DevBuf sel_rank;
    uint64_t n_sel = 0;
    if (subdivide) {
        std::vector<uint32_t> h(N);
        SVR_CUDA(cudaMemcpy(h.data(), flags, N * 4, cudaMemcpyDeviceToHost));
        for (auto& x : h) {
            n_sel += x;
            x = x ? 8u : 1u;
        }
        SVR_CUDA(cudaMemcpy(cnt.p, h.data(), N * 4, cudaMemcpyHostToDevice));
        N2 = scan_total(ctx, cnt.as<uint32_t>(), at.as<uint32_t>(), N, st);
        sel_rank.reserve(std::max<uint64_t>(N, 1) * 4);
        scan_total(ctx, flags, sel_rank.as<uint32_t>(), N, st);
    } else {
        N2 = scan_total(ctx, flags, at.as<uint32_t>(), N, st);
    }
    if (N2 > (uint64_t(1) << 29))  // kMaxVoxelCount (scene.hpp:19), optim.cpp:248-249
        throw Error(SVR_ERR_LENGTH, "subdivision exceeds voxel capacity");
    auto* s = new svr_scene;
    try {
        s->n_voxels = N2;
        s->sh_degree = old->sh_degree;
        s->sh_stride = stride;
        for (int i = 0; i < 3; ++i) s->bounds_center[i] = old->bounds_center[i];
        s->bounds_size = old->bounds_size;
        s->paths.reserve(std::max<uint64_t>(N2, 1) * 8);
        s->voxel_src.reserve(std::max<uint64_t>(N2, 1) * 8);
        DevBuf sh_src;
        sh_src.reserve(std::max<uint64_t>(N2, 1) * 8);
        if (N) {
            if (subdivide)
                subdivide_voxels_kernel<<<blocks_for(N, 256), 256, 0, st>>>(
                    old->paths.as<uint64_t>(), flags, at.as<uint32_t>(), N, s->paths.as<uint64_t>(),
                    s->voxel_src.as<int64_t>(), sh_src.as<int64_t>());
            else
                compact_voxels_kernel<<<blocks_for(N, 256), 256, 0, st>>>(
                    old->paths.as<uint64_t>(), flags, at.as<uint32_t>(), N, s->paths.as<uint64_t>(),
                    s->voxel_src.as<int64_t>(), sh_src.as<int64_t>());
            SVR_LAUNCH("adapt_voxels_kernel");
        }
        // 3. fresh subdivision points
        DevBuf fkey, fval;
        uint64_t n_fresh = 0;
        if (subdivide && n_sel) {
            SortedKeys fk;
            const uint64_t mf = 64 * n_sel;
            for (int b = 0; b < 2; ++b) {
                fk.keys[b].reserve(mf * 8);
                fk.pos[b].reserve(mf * 4);
            }
            DevBuf vals;
            vals.reserve(mf * 8);
            fresh_contribs_kernel<<<blocks_for(N, 128), 128, 0, st>>>(
                old->paths.as<uint64_t>(), flags, sel_rank.as<uint32_t>(), N,
                old->corner_index.as<uint32_t>(), old->density.as<float>(), old_ukey.as<uint64_t>(),
                n_old_u, fk.keys[0].as<uint64_t>(), fk.pos[0].as<uint32_t>(), vals.as<double>());
            SVR_LAUNCH("fresh_contribs_kernel");
            sort_keys_with_pos(ctx, fk, mf, 64, st);
            fk.head.reserve(mf * 4);
            fk.head_excl.reserve(mf * 4);
            DevBuf dummy;
            dummy.reserve(mf * 4);
            SVR_CUDA(cudaMemsetAsync(dummy.p, 0, mf * 4, st));
            run_heads_kernel<<<blocks_for(mf, 256), 256, 0, st>>>(fk.skeys, fk.spos, mf,
                                                                  dummy.as<uint32_t>(), fk.head.as<uint32_t>());
            SVR_LAUNCH("run_heads_kernel");
            n_fresh = scan_total(ctx, fk.head.as<uint32_t>(), fk.head_excl.as<uint32_t>(), mf, st);
            fkey.reserve(std::max<uint64_t>(n_fresh, 1) * 8);
            fval.reserve(std::max<uint64_t>(n_fresh, 1) * 4);
            fresh_average_kernel<<<blocks_for(mf, 256), 256, 0, st>>>(
                fk.skeys, fk.spos, vals.as<double>(), fk.head.as<uint32_t>(), fk.head_excl.as<uint32_t>(),
                mf, fkey.as<uint64_t>(), fval.as<float>());
            SVR_LAUNCH("fresh_average_kernel");
            // the all-ones key of existing points sorts last: drop it
            if (n_fresh) {
                uint64_t lastk = 0;
                SVR_CUDA(cudaMemcpy(&lastk, fk.skeys + mf - 1, 8, cudaMemcpyDeviceToHost));
                if (lastk == ~uint64_t(0)) --n_fresh;
            }
        }
        // 4. rebuild_corner_indexing on the new voxel list
        SortedKeys nk;
        const uint64_t m = 8 * N2;
        for (int b = 0; b < 2; ++b) {
            nk.keys[b].reserve(std::max<uint64_t>(m, 1) * 8);
            nk.pos[b].reserve(std::max<uint64_t>(m, 1) * 4);
        }
        if (N2) {
            corner_keys_kernel<<<blocks_for(N2, 256), 256, 0, st>>>(
                s->paths.as<uint64_t>(), N2, nk.keys[0].as<uint64_t>(), nk.pos[0].as<uint32_t>());
            SVR_LAUNCH("corner_keys_kernel");
        }
        sort_keys_with_pos(ctx, nk, m, 51, st);
        nk.head.reserve(std::max<uint64_t>(m, 1) * 4);
        nk.head_excl.reserve(std::max<uint64_t>(m, 1) * 4);
        DevBuf first, first_rank;
        first.reserve(std::max<uint64_t>(m, 1) * 4);
        first_rank.reserve(std::max<uint64_t>(m, 1) * 4);
        SVR_CUDA(cudaMemsetAsync(first.p, 0, std::max<uint64_t>(m, 1) * 4, st));
        if (m) {
            run_heads_kernel<<<blocks_for(m, 256), 256, 0, st>>>(nk.skeys, nk.spos, m,
                                                                 first.as<uint32_t>(), nk.head.as<uint32_t>());
            SVR_LAUNCH("run_heads_kernel");
        }
        const uint64_t P2 = scan_total(ctx, first.as<uint32_t>(), first_rank.as<uint32_t>(), m, st);
        scan_total(ctx, nk.head.as<uint32_t>(), nk.head_excl.as<uint32_t>(), m, st);
        s->n_pool = P2;
        s->corner_index.reserve(std::max<uint64_t>(N2, 1) * 32);
        s->density.reserve(std::max<uint64_t>(P2, 1) * 4);
        s->pool_src.reserve(std::max<uint64_t>(P2, 1) * 8);
        DevBuf run_pool, pool_key;
        run_pool.reserve(std::max<uint64_t>(P2, 1) * 4);
        pool_key.reserve(std::max<uint64_t>(P2, 1) * 8);
        if (m) {
            assign_pool_kernel<<<blocks_for(m, 256), 256, 0, st>>>(
                nk.skeys, nk.spos, nk.head.as<uint32_t>(), nk.head_excl.as<uint32_t>(),
                first_rank.as<uint32_t>(), m, run_pool.as<uint32_t>(), pool_key.as<uint64_t>());
            SVR_LAUNCH("assign_pool_kernel");
            scatter_corner_index_kernel<<<blocks_for(m, 256), 256, 0, st>>>(
                nk.spos, nk.head.as<uint32_t>(), nk.head_excl.as<uint32_t>(), run_pool.as<uint32_t>(), m,
                s->corner_index.as<uint32_t>());
            SVR_LAUNCH("scatter_corner_index_kernel");
        }
        if (P2) {
            pool_density_kernel<<<blocks_for(P2, 256), 256, 0, st>>>(
                pool_key.as<uint64_t>(), P2, old_ukey.as<uint64_t>(), old_upool.as<uint32_t>(), n_old_u,
                old->density.as<float>(), fkey.as<uint64_t>(), fval.as<float>(), n_fresh, fill,
                s->density.as<float>(), s->pool_src.as<int64_t>());
            SVR_LAUNCH("pool_density_kernel");
        }
        // 5. SH rows, max level, Morton rank table
        s->sh.reserve(std::max<uint64_t>(N2 * stride, 1) * 4);
        if (N2) {
            gather_sh_kernel<<<blocks_for(N2 * stride, 256), 256, 0, st>>>(
                old->sh.as<float>(), sh_src.as<int64_t>(), N2, stride, s->sh.as<float>());
            SVR_LAUNCH("gather_sh_kernel");
        }
        DevBuf ml;
        ml.reserve(4);
        SVR_CUDA(cudaMemsetAsync(ml.p, 0, 4, st));
        if (N2) {
            max_level_kernel<<<blocks_for(N2, 256), 256, 0, st>>>(s->paths.as<uint64_t>(), N2,
                                                                   ml.as<unsigned int>());
            SVR_LAUNCH("max_level_kernel");
        }
        unsigned int hml = 1;
        SVR_CUDA(cudaMemcpyAsync(&hml, ml.p, 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        s->max_level = std::max(1, int(hml));
        if (N2 > 0 && N2 < (uint64_t(1) << 28)) {
            s->morton_rank.reserve(N2 * 8 * 4);
            s->morton_order.reserve(N2 * 8 * 4);
            DevBuf tmp;
            tmp.reserve(morton_rank_scratch_bytes(N2, s->max_level));
            build_morton_rank(s->paths.as<uint64_t>(), N2, s->max_level, s->morton_rank.as<uint32_t>(),
                              s->morton_order.as<uint32_t>(), tmp.p, st);
            SVR_CUDA(cudaStreamSynchronize(st));
            s->rank_bits = 0;
            for (uint64_t x = 8 * N2 - 1; x; x >>= 1) ++s->rank_bits;
        }
        s->has_remap = true;
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

}  // namespace svrb
