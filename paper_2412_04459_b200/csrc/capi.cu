// capi.cu — the C ABI (include/svr_b200.h): contexts, device-resident scenes,
// per-view frames, and the orchestration of the sm_100a kernels that
// replaces render_with_pools / render_backward (raster.cpp:205-423).
//
// There is no CPU fallback: every compute entry point launches CUDA kernels
// and fails with SVR_ERR_NO_DEVICE / SVR_ERR_CUDA when it cannot.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "svr_internal.h"
#include "svr_kernels.h"
#include "svrx.h"

namespace svrb {

namespace {
thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVR_PDL");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

// Records a stage boundary on the context stream (no-op unless timing).
void mark(svr_ctx* ctx, int stage) {
    if (!ctx->timing) return;
    cudaEvent_t e;
    if (!ctx->event_pool.empty()) {
        e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
    } else {
        SVR_CUDA(cudaEventCreate(&e));
    }
    SVR_CUDA(cudaEventRecord(e, ctx->stream));
    ctx->marks.push_back({stage, e});
}

// Folds recorded marks into stage_ms (synchronises the stream).
void collect_marks(svr_ctx* ctx) {
    if (ctx->marks.empty()) return;
    SVR_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t i = 0; i + 1 < ctx->marks.size(); ++i) {
        int st = ctx->marks[i].first;
        if (st < 0) continue;
        float ms = 0.f;
        SVR_CUDA(cudaEventElapsedTime(&ms, ctx->marks[i].second, ctx->marks[i + 1].second));
        ctx->stage_ms[st] += ms;
    }
    for (auto& m : ctx->marks) ctx->event_pool.push_back(m.second);
    ctx->marks.clear();
}

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        throw Error(SVR_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    throw Error(SVR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void DevBuf::reserve(size_t n) {
    if (n <= bytes) return;
    release();
    size_t alloc = std::max<size_t>(n + n / 4, 256);  // headroom: E varies from view to view
    SVR_CUDA(cudaMalloc(&p, alloc));
    bytes = alloc;
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

void HostBuf::reserve(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    SVR_CUDA(cudaMallocHost(&p, n));
    bytes = n;
}

HostBuf::~HostBuf() {
    if (p) cudaFreeHost(p);
}

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return SVR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc& e) {
        g_last_error = e.what();
        return SVR_ERR_RUNTIME;
    } catch (const std::invalid_argument& e) {  // e.g. SvrxInvalid (octree level checks)
        g_last_error = e.what();
        return SVR_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SVR_ERR_RUNTIME;
    }
}

void require(bool ok, int status, const char* msg) {
    if (!ok) throw Error(status, msg);
}

int tiles_along(int px) { return (px + kTile - 1) / kTile; }

// Camera::scaled (camera.hpp:38-48).
svr_camera scaled_camera(const svr_camera& c, int nw, int nh) {
    svr_camera s = c;
    double rx = double(nw) / c.width, ry = double(nh) / c.height;
    s.width = nw;
    s.height = nh;
    s.fx = c.fx * rx;
    s.cx = c.cx * rx;
    s.fy = c.fy * ry;
    s.cy = c.cy * ry;
    return s;
}

DevCamera dev_camera(const svr_camera& c) {
    DevCamera d{};
    d.W = c.width;
    d.H = c.height;
    d.ntx = tiles_along(c.width);
    d.nty = tiles_along(c.height);
    d.fx = c.fx;
    d.fy = c.fy;
    d.cx = c.cx;
    d.cy = c.cy;
    for (int i = 0; i < 9; ++i) d.rot[i] = c.rot[i];
    for (int i = 0; i < 3; ++i) d.pos[i] = c.pos[i];
    return d;
}

int bit_width(uint64_t x) {
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

void set_device(svr_ctx* ctx) { SVR_CUDA(cudaSetDevice(ctx->device)); }

template <class T>
T* grow(DevBuf& b, uint64_t count) {
    b.reserve(std::max<uint64_t>(count, 1) * sizeof(T));
    return b.as<T>();
}

// axis_taps (image.cpp:9-23) as CSR, plus the transposed table for the adjoint.
void axis_taps(int src, int dst, std::vector<int>& ptr, std::vector<int>& idx,
               std::vector<float>& w, std::vector<int>& tptr, std::vector<int>& tidx,
               std::vector<float>& tw) {
    double scale = double(src) / dst;
    ptr.assign(1, 0);
    idx.clear();
    w.clear();
    std::vector<std::vector<std::pair<int, float>>> tr(src);
    for (int d = 0; d < dst; ++d) {
        double lo = d * scale, hi = (d + 1) * scale;
        int s0 = int(lo), s1 = std::min(src - 1, int(std::ceil(hi)) - 1);
        for (int s = s0; s <= s1; ++s) {
            double overlap = std::min(hi, double(s + 1)) - std::max(lo, double(s));
            if (overlap > 0) {
                idx.push_back(s);
                w.push_back(float(overlap / scale));
                tr[s].push_back({d, float(overlap / scale)});
            }
        }
        ptr.push_back(int(idx.size()));
    }
    tptr.assign(1, 0);
    tidx.clear();
    tw.clear();
    for (int s = 0; s < src; ++s) {
        for (auto& pr : tr[s]) {
            tidx.push_back(pr.first);
            tw.push_back(pr.second);
        }
        tptr.push_back(int(tidx.size()));
    }
}

struct TapSet {
    TapTable fwd, adj;
};

TapSet ensure_taps(svr_frame* f) {
    // Layout inside f->taps: [ptr_x idx_x w_x ptr_y idx_y w_y tptr_x tidx_x tw_x tptr_y tidx_y tw_y]
    std::vector<int> px, ix, py, iy, tpx, tix, tpy, tiy;
    std::vector<float> wx, wy, twx, twy;
    axis_taps(f->sw, f->W, px, ix, wx, tpx, tix, twx);
    axis_taps(f->sh, f->H, py, iy, wy, tpy, tiy, twy);
    std::vector<std::pair<const void*, size_t>> parts = {
        {px.data(), px.size() * 4},   {ix.data(), ix.size() * 4},   {wx.data(), wx.size() * 4},
        {py.data(), py.size() * 4},   {iy.data(), iy.size() * 4},   {wy.data(), wy.size() * 4},
        {tpx.data(), tpx.size() * 4}, {tix.data(), tix.size() * 4}, {twx.data(), twx.size() * 4},
        {tpy.data(), tpy.size() * 4}, {tiy.data(), tiy.size() * 4}, {twy.data(), twy.size() * 4}};
    std::vector<size_t> off;
    size_t total = 0;
    for (auto& p : parts) {
        off.push_back(total);
        total += (p.second + 15) & ~size_t(15);
    }
    bool fresh = !(f->tap_src_w == f->sw && f->tap_src_h == f->sh && f->tap_dst_w == f->W &&
                   f->tap_dst_h == f->H);
    if (fresh) {
        f->taps.reserve(total);
        std::vector<char> host(total, 0);
        for (size_t i = 0; i < parts.size(); ++i)
            if (parts[i].second) std::memcpy(host.data() + off[i], parts[i].first, parts[i].second);
        SVR_CUDA(cudaMemcpy(f->taps.p, host.data(), total, cudaMemcpyHostToDevice));
        f->tap_src_w = f->sw;
        f->tap_src_h = f->sh;
        f->tap_dst_w = f->W;
        f->tap_dst_h = f->H;
    }
    char* b = f->taps.as<char>();
    TapSet t;
    t.fwd = {reinterpret_cast<int*>(b + off[0]),  reinterpret_cast<int*>(b + off[1]),
             reinterpret_cast<float*>(b + off[2]), reinterpret_cast<int*>(b + off[3]),
             reinterpret_cast<int*>(b + off[4]),  reinterpret_cast<float*>(b + off[5])};
    t.adj = {reinterpret_cast<int*>(b + off[6]),  reinterpret_cast<int*>(b + off[7]),
             reinterpret_cast<float*>(b + off[8]), reinterpret_cast<int*>(b + off[9]),
             reinterpret_cast<int*>(b + off[10]), reinterpret_cast<float*>(b + off[11])};
    return t;
}

// Device-side ordering against a frame's in-flight asynchronous downloads:
// anything that rewrites frame buffers first makes the main stream wait.
void wait_copies(svr_frame* f) {
    if (f && f->copy_pending) {
        SVR_CUDA(cudaStreamWaitEvent(f->ctx->stream, f->copied, 0));
        f->copy_pending = false;
    }
}

// Validation of RenderOptions, in raster.cpp:207-211 order.
void validate_options(const svr_render_options& o) {
    require(o.supersample >= 1.0, SVR_ERR_INVALID_ARGUMENT, "supersample factor must be >= 1");
    require(o.K >= 1 && o.K <= 3, SVR_ERR_INVALID_ARGUMENT,
            "rasterizer sample count K must be in {1,2,3}");
    require(o.t_threshold > 0.0 && o.t_threshold < 1.0, SVR_ERR_INVALID_ARGUMENT,
            "transmittance threshold must be in (0,1)");
}

// Radix digits that can differ between entries (see sort.cu): the sign
// pattern (value bits 29..31) when more than one pattern exists, then the
// key bits from the finest occupied octree level up to the top tile-id bit.
int plan_sort(int max_level, int ntiles, uint32_t pattern_or, RadixPass* passes) {
    int np = 0;
    if (__builtin_popcount(pattern_or) > 1) passes[np++] = {1, 29, 3};
    int lo = 48 - 3 * max_level;
    int hi = 48 + bit_width(uint64_t(ntiles - 1));
    for (int b = lo; b < hi; b += 8) passes[np++] = {0, b, std::min(8, hi - b)};
    return np;
}

bool packed_keys_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVR_PACKED_KEYS");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

bool rank_keys_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVR_RANK_KEYS");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

void render_impl(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam_in,
                 const svr_render_options* opts, svr_frame* f, bool allow_deferred = true) {
    require(ctx && scene && cam_in && opts && f, SVR_ERR_INVALID_ARGUMENT, "null argument");
    set_device(ctx);
    validate_options(*opts);
    require(cam_in->width > 0 && cam_in->height > 0, SVR_ERR_INVALID_ARGUMENT,
            "camera resolution must be positive");
    cudaStream_t st = ctx->stream;
    const int W = cam_in->width, H = cam_in->height;
    const int sw = int(std::ceil(opts->supersample * W));
    const int sh = int(std::ceil(opts->supersample * H));
    const svr_camera ss_cam = scaled_camera(*cam_in, sw, sh);
    const DevCamera cam = dev_camera(ss_cam);
    const int ntiles = cam.ntx * cam.nty;
    // build_sort_entries capacity checks (raster.cpp:146-150)
    require(scene->n_voxels < (uint64_t(1) << 29), SVR_ERR_LENGTH,
            "voxel count exceeds the 29-bit id capacity");
    require(uint64_t(cam.ntx) * cam.nty < (uint64_t(1) << 16), SVR_ERR_LENGTH,
            "tile count exceeds the 16-bit id capacity");

    if (f->copy_pending) {  // rendering rewrites the outputs an async copy reads
        SVR_CUDA(cudaStreamWaitEvent(ctx->stream, f->copied, 0));
        f->copy_pending = false;
    }
    f->ctx = ctx;
    f->scene = scene;
    f->opts = *opts;
    f->req_cam = *cam_in;
    f->req_opts = *opts;
    f->pending_dl.clear();
    f->cam = cam;
    f->ss_cam = ss_cam;
    f->W = W;
    f->H = H;
    f->sw = sw;
    f->sh = sh;
    f->ntx = cam.ntx;
    f->nty = cam.nty;
    f->n_voxels = scene->n_voxels;
    f->training = opts->training != 0;
    f->has_records = false;
    f->param_version = scene->param_version;
    f->n_contribs = 0;
    f->il_pending = f->rl_pending = false;  // loss values belong to the previous render
    const uint64_t N = scene->n_voxels;
    const bool ss1 = (sw == W && sh == H);

    // Rank-ordered duplicate (keys emitted pre-sorted below the tile bits) when
    // the scene has its pair list; SVR_RANKED=0 keeps the voxel-order emission.
    const char* ranked_env = std::getenv("SVR_RANKED");  // read per frame (parity tests flip it)
    const bool ranked_enabled = ranked_env == nullptr || ranked_env[0] != '0';
    const bool ranked_ok = ranked_enabled && N > 0 && scene->rank_bits > 0 &&
                           (std::max(1, bit_width(N - 1)) + 3 + scene->rank_bits +
                            bit_width(uint64_t(ntiles - 1))) <= 64;

    // K2: tile sign masks + SAT (+ the per-pattern SATs of the ranked duplicate)
    uint8_t* masks = grow<uint8_t>(f->tile_masks, ntiles);
    const uint64_t ncell = uint64_t(cam.ntx + 1) * (cam.nty + 1);
    uint32_t* sat = grow<uint32_t>(f->tile_sat, ncell * (ranked_ok ? 9 : 1));
    FrameStatus* status = grow<FrameStatus>(f->status, 1);
    SVR_CUDA(cudaMemsetAsync(status, 0, sizeof(FrameStatus), st));
    mark(ctx, kStageTileSetup);
    int2* rowspan = ranked_ok ? grow<int2>(f->rowspan, uint64_t(8) * cam.nty) : nullptr;
    launch_tile_setup(cam, masks, sat, status, st, rowspan);

    // K1: preprocess
    PreprocessArgs pa{};
    pa.n = N;
    pa.paths = scene->paths.as<uint64_t>();
    pa.corner_index = scene->corner_index.as<uint32_t>();
    pa.density = scene->density.as<float>();
    pa.sh = scene->sh.as<float>();
    pa.sh_degree = scene->sh_degree;
    pa.sh_stride = scene->sh_stride;
    for (int i = 0; i < 3; ++i) pa.bc[i] = scene->bounds_center[i];
    pa.bsize = scene->bounds_size;
    pa.near_plane = opts->near_plane;
    pa.tile_sat = sat;
    pa.rects = grow<int4>(f->rects, N);
    pa.aabb = ctx->debug ? grow<double4>(f->aabb, N) : nullptr;
    pa.records = grow<float4>(f->records, N * kRecordF4);
    pa.counts = grow<uint32_t>(f->counts, N);
    pa.view_dir = f->training ? grow<float4>(f->view_dir, N) : nullptr;
    pa.vis_list = f->training ? grow<uint32_t>(f->vis_list, N) : nullptr;
    pa.n_vis_list = f->training ? &status->n_vis_list : nullptr;
    // scenes stored out of spatial order: pre-cull pass + worklist
    pa.order = scene->unordered ? grow<uint32_t>(f->work, N) : nullptr;
    pa.n_order = scene->unordered ? &status->n_work : nullptr;
    mark(ctx, kStagePreprocess);
    launch_preprocess(cam, pa, st);

    // K3: scan of the entry counts -> emission offsets and E: per (pattern,
    // voxel) pair in rank order for the ranked duplicate, else per voxel (also
    // for the ranked path's parity dump of the voxel-order emission).
    uint32_t* offsets = grow<uint32_t>(f->offsets, N);
    uint32_t* pc = nullptr;
    const size_t scan_bytes = scan_scratch_bytes(std::max<uint64_t>(N, uint64_t(ntiles) * 256));
    ctx->scratch.reserve(scan_bytes + (ranked_ok ? scan_scratch_bytes(8 * N) + 256 : 0));
    // the ranked path's block prefixes live past the general scan scratch
    uint32_t* pair_partial = reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->scratch.p) +
                                                         ((scan_bytes + 255) & ~size_t(255)));
    // Huge pairs (>= SVR_HUGE_MIN tiles) skip duplicate + sort and are merged
    // into the tile lists by rank (raster.cu: HugePairs), in production
    // frames, once an earlier frame showed there are some. Off by default:
    // config-4 view 0 gains (4.63 -> 4.01 ms) but over the bench's 30 views
    // the merge's long-pole tiles cost more than the sort it replaces
    // (4.97 -> 5.64 ms), and config 2 pays its fixed cost (+0.19 ms); see
    // DESIGN.md §8.
    const char* huge_env = std::getenv("SVR_HUGE_MIN");  // read per frame (parity tests set it)
    const uint32_t huge_min = huge_env ? uint32_t(std::strtoul(huge_env, nullptr, 10)) : 0u;
    HugePairs huge{};
    huge.min = ranked_ok ? huge_min : 0u;
    huge.divert = huge.min && !ctx->debug && f->huge_hint > 0 && ntiles <= 4096 &&
                  packed_keys_enabled() && rank_keys_enabled();
    if (huge.divert) {
        uint32_t cap = 4096;
        while (cap < 2 * f->huge_hint && cap < (1u << 22)) cap <<= 1;
        huge.cap = cap;
        huge.keys = grow<uint64_t>(f->huge_keys, 2 * uint64_t(cap));  // + the sort's ping-pong half
        huge.vals = grow<uint32_t>(f->huge_vals, 2 * uint64_t(cap));
    }
    f->huge_used = huge.divert != 0;
    mark(ctx, kStageScan);
    if (ranked_ok) {
        pc = grow<uint32_t>(f->pair_counts, 8 * N);
#ifndef SVR_PAIR_ATOMIC_SUMS
#define SVR_PAIR_ATOMIC_SUMS 1
#endif
        // Large scenes (N >= 2^22): K4a accumulates the scan's block sums
        // itself (warp-combined atomics), so only the block-sum scan remains
        // instead of a reduce pass over all 8N counts (config 4: 250 MB, the
        // scan stage 181 -> 149 us). At config-2 sizes the reduce pass is
        // cheaper than the per-pair match + atomic (38 vs 44 us).
        const char* pa_env = std::getenv("SVR_PAIR_ATOMIC_MIN");  // parity tests lower it
        const bool atomic_sums =
            SVR_PAIR_ATOMIC_SUMS && N >= (pa_env ? std::strtoull(pa_env, nullptr, 10) : (uint64_t(1) << 22));
        launch_pair_counts(cam, N, pa.counts, pa.rects, sat, status, scene->morton_rank.as<uint32_t>(), pc,
                           atomic_sums ? pair_partial : nullptr, st, huge);
        if (atomic_sums)
            scan_block_sums(pair_partial, (8 * N + kScanChunk - 1) / kScanChunk, &status->n_entries, st);
        else
            scan_block_prefixes(pc, 8 * N, &status->n_entries, pair_partial, st);
    }
    if (!ranked_ok || ctx->debug)
        exclusive_scan_u32(pa.counts, offsets, N, ranked_ok ? &status->n_entries_voxel : &status->n_entries,
                           ctx->scratch.p, st);
    mark(ctx, -1);
    f->hstatus.reserve(sizeof(FrameStatus));
    FrameStatus* hs = static_cast<FrameStatus*>(f->hstatus.p);
    // Deferred E (svr_ctx_set_async): no host round trip here; the sort and
    // its neighbours run on a capacity sized from earlier frames and read the
    // live count on the device. Needs a capacity and the pattern-independent
    // sort plan of the rank-keyed packed format (never for training frames,
    // whose record buffers are sized from the contribution count).
    // Morton-rank keys: tile | rank(s, vid) | s | vid, sorted on tile|rank only.
    const int tile_bits = bit_width(uint64_t(ntiles - 1));
    const int vb = std::max(1, bit_width(N > 0 ? N - 1 : 0));
    const int rb = scene->rank_bits;
    const bool use_rank = rank_keys_enabled() && N > 0 && rb > 0 && (vb + 3 + rb + tile_bits) <= 64;
    // A frame whose rank keys do not fit in 64 bits (e.g. > 2^23 voxels at
    // 1024^2, 8160 tiles at 1080p with 7.8M voxels) or with packed keys
    // switched off reads E back synchronously instead.
    const bool deferred = allow_deferred && ctx->async_frames && !f->training && !ctx->debug &&
                          f->e_cap > 0 && use_rank && packed_keys_enabled();
    // E: all entries of the frame (= the capacity in a deferred frame);
    // E_sort: those the duplicate emits and the sort orders (without the
    // huge pairs' entries, which the merge places).
    uint64_t E, E_sort;
    uint32_t pattern_or = 0;
    if (deferred) {
        E = E_sort = f->e_cap;
    } else {
        launch_status_to_host(status, hs, st);
        SVR_CUDA(cudaStreamSynchronize(st));
        E_sort = hs->n_entries;
        E = E_sort + hs->n_huge_entries;
        pattern_or = hs->pattern_or;
        f->huge_hint = hs->n_huge_pairs;
        f->n_vis_list = f->training ? hs->n_vis_list : 0;
        require(E < (uint64_t(1) << 30), SVR_ERR_LENGTH, "entry count exceeds 2^30");
        f->e_cap = std::max<uint64_t>(f->e_cap, E + E / 4 + 1024);
    }
    f->n_entries = E;
    f->e_pending = deferred;

    // K4 + K5 + K6. Packed path when tile | order | s | vid fits in 64 bits
    // (config 2: 12 + 27 + 3 + 20 = 62): keys-only sort of 8-B entries, digit
    // histograms fused into the duplicate kernel. Otherwise the general
    // (u64 key, u32 value) path. Both reproduce the reference's emission
    // order (vid, ty, tx, s) and its (key, value) sort order.
    const int lmax = scene->max_level;
    const bool multi = __builtin_popcount(pattern_or) > 1;
    f->packed = packed_keys_enabled() && N > 0 && (use_rank || (vb + 3 + 3 * lmax + tile_bits) <= 64);
    require(!deferred || (f->packed && use_rank), SVR_ERR_RUNTIME, "deferred frame needs rank keys");
    uint2* ranges = grow<uint2>(f->ranges, ntiles);
    RadixPass passes[kMaxRadixPasses];
    int np = 0;
    f->sort_keys_kept = true;
    if (f->packed) {
        f->fmt = use_rank ? PackedFormat{vb, lmax, vb + 3 + rb, rb}
                          : PackedFormat{vb, lmax, vb + 3 + 3 * lmax, 0};
        const bool ranked = ranked_ok;
        require(!ranked || use_rank, SVR_ERR_RUNTIME, "ranked duplicate needs rank keys");
        // ranked emission: the keys arrive sorted below the tile bits
        const int lo = ranked ? f->fmt.tile_shift : vb + ((multi && !use_rank) ? 0 : 3);
        const int hi = f->fmt.tile_shift + tile_bits;
        {  // the fewest 8-bit-or-narrower passes, bits spread evenly (12 tile
           // bits: 6 + 6; SVR_SORT_EVEN=0 keeps 8 + 4)
            static const bool even = [] {
                const char* e = std::getenv("SVR_SORT_EVEN");
                return e == nullptr || e[0] != '0';
            }();
            const int nb = hi - lo, npass = (nb + 7) / 8;
            for (int q = 0, b = lo; q < npass; ++q) {
                const int w = even ? (nb - (b - lo) + (npass - q) - 1) / (npass - q) : std::min(8, hi - b);
                passes[np++] = {0, b, w};
                b += w;
            }
        }
        RadixPlan plan{};
        plan.n = np;
        for (int i = 0; i < np; ++i) plan.p[i] = passes[i];
        grow<uint64_t>(f->keys[0], E);
        grow<uint64_t>(f->keys[1], E);
        grow<uint32_t>(f->vals[0], E);
        if (huge.divert) grow<uint32_t>(f->vals[1], E);
        ctx->scratch2.reserve(sort_scratch_bytes(E, np));
        mark(ctx, kStageDuplicate);
        if (!ranked || ctx->debug) {
            // voxel-order emission (reference order (vid, ty, tx, s)); with the
            // ranked path it only feeds the parity dump of the unsorted keys
            uint64_t* dk = ranked ? f->keys[1].as<uint64_t>() : f->keys[0].as<uint64_t>();
            launch_duplicate_packed(cam, N, pa.paths, pa.rects, masks, pa.counts, offsets, f->fmt,
                                    use_rank ? scene->morton_rank.as<uint32_t>() : nullptr, dk, sat,
                                    grow<uint32_t>(f->big, N), &status->n_big, st, E);
            if (ctx->debug) {
                grow<uint64_t>(f->dbg_keys, E);
                SVR_CUDA(cudaMemcpyAsync(f->dbg_keys.p, dk, E * 8, cudaMemcpyDeviceToDevice, st));
            }
        }
        // ranked, large E: K4 counts the (at most two) tile digits of the sort
        // and the sort skips its histogram read of the keys (config 4, 97M
        // entries: sort + duplicate 2.29 -> 2.10 ms). At config-2 sizes the
        // shared-memory atomics cost what the read saves, so the separate
        // histogram kernel stays.
        const char* fh_env = std::getenv("SVR_FUSED_HIST_MIN");  // parity tests lower it
        const uint64_t fh_min = fh_env ? std::strtoull(fh_env, nullptr, 10) : (uint64_t(1) << 24);
        const bool fused_hist = ranked && np >= 1 && np <= 2 && E_sort > 1 && E_sort >= fh_min;
        TileDigits td{};
        if (fused_hist) {
            sort_prepare(ctx->scratch2.p, E_sort, np, st);
            td.hist = sort_hist_ptr(ctx->scratch2.p);
            td.b0 = passes[0].bits;
            td.m0 = (1u << passes[0].bits) - 1u;
            td.two = np == 2;
            td.m1 = np == 2 ? (1u << passes[1].bits) - 1u : 0u;
        }
        if (ranked)
            launch_duplicate_ranked(cam, N, pc, pair_partial, scene->morton_order.as<uint32_t>(), pa.rects,
                                    masks, sat, rowspan, f->fmt, f->keys[0].as<uint64_t>(), E_sort,
                                    grow<uint2>(f->big_pairs, E / kRankedBigMin + 1),
                                    &status->n_big_ranked, st, td);
        mark(ctx, kStageSort);
        const unsigned long long* n_dev = deferred ? &status->n_entries : nullptr;
        // Ranked emission outside debug mode: the last pass writes the values
        // the compositing kernels read, and the ranges come from per-tile
        // counts taken during the histogram read (no sorted keys written).
        f->sort_keys_kept = !(ranked && !ctx->debug && np > 0 && E_sort > 1) || huge.divert;
        if (!f->sort_keys_kept) {
            SortFinish fin{f->vals[0].as<uint32_t>(), ranges, f->fmt.vb, f->fmt.tile_shift, ntiles};
            f->sorted_buf = radix_sort_keys(f->keys[0].as<uint64_t>(), f->keys[1].as<uint64_t>(), E_sort,
                                            passes, np, ctx->scratch2.p, st, fused_hist, n_dev, &fin);
            mark(ctx, kStageRanges);
        } else {
            f->sorted_buf = radix_sort_keys(f->keys[0].as<uint64_t>(), f->keys[1].as<uint64_t>(), E_sort,
                                            passes, np, ctx->scratch2.p, st, fused_hist, n_dev);
            mark(ctx, kStageRanges);
            launch_tile_ranges_packed(f->keys[f->sorted_buf].as<uint64_t>(), E_sort, f->fmt,
                                      huge.divert ? grow<uint2>(f->ranges_small, ntiles) : ranges,
                                      f->vals[0].as<uint32_t>(), ntiles, st, n_dev);
        }
        f->vals_buf = 0;
        if (huge.divert) {
            // the huge pairs in rank order, then merged into every tile's list
            RadixPass hp[kMaxRadixPasses];
            int nhp = 0;
            for (int b = 0; b < rb; b += 8) hp[nhp++] = {0, b, std::min(8, rb - b)};
            f->huge_scratch.reserve(sort_scratch_bytes(huge.cap, nhp));
            uint64_t* hk = f->huge_keys.as<uint64_t>();
            uint32_t* hv = f->huge_vals.as<uint32_t>();
            const int hb = radix_sort_pairs(hk, hv, hk + huge.cap, hv + huge.cap, huge.cap, hp, nhp,
                                            f->huge_scratch.p, st);
            // and stably by sign pattern (value bits 29..31) into the other half
            const RadixPass byp{1, 29, 3};
            const size_t ho = size_t(hb) * huge.cap, so = size_t(hb ^ 1) * huge.cap;
            radix_sort_pairs(hk + ho, hv + ho, hk + so, hv + so, huge.cap, &byp, 1, f->huge_scratch.p, st);
            launch_merge_huge(cam, huge, hk + ho, hv + ho, hk + so, hv + so, status,
                              pa.rects, masks, f->keys[f->sorted_buf].as<uint64_t>(),
                              f->ranges_small.as<uint2>(), f->fmt,
                              grow<int>(f->huge_diff, 8 * uint64_t(cam.ntx + 1) * (cam.nty + 1)),
                              grow<uint4>(f->huge_pack, 2 * uint64_t(huge.cap) + 4), grow<uint32_t>(f->huge_apos, E),
                              ranges,
                              f->vals[1].as<uint32_t>(), E,
                              grow<unsigned long long>(f->huge_total, 1), st);
            f->vals_buf = 1;
        }
    } else {
        for (int b = 0; b < 2; ++b) {
            grow<uint64_t>(f->keys[b], E);
            grow<uint32_t>(f->vals[b], E);
        }
        mark(ctx, kStageDuplicate);
        launch_duplicate(cam, N, pa.paths, pa.rects, masks, pa.counts, offsets,
                         f->keys[0].as<uint64_t>(), f->vals[0].as<uint32_t>(), st);
        if (ctx->debug) {
            grow<uint64_t>(f->dbg_keys, E);
            grow<uint32_t>(f->dbg_vals, E);
            SVR_CUDA(cudaMemcpyAsync(f->dbg_keys.p, f->keys[0].p, E * 8, cudaMemcpyDeviceToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(f->dbg_vals.p, f->vals[0].p, E * 4, cudaMemcpyDeviceToDevice, st));
        }
        np = plan_sort(lmax, ntiles, pattern_or, passes);
        mark(ctx, kStageSort);
        ctx->scratch2.reserve(sort_scratch_bytes(E, np));
        f->sorted_buf = radix_sort_pairs(f->keys[0].as<uint64_t>(), f->vals[0].as<uint32_t>(),
                                         f->keys[1].as<uint64_t>(), f->vals[1].as<uint32_t>(), E,
                                         passes, np, ctx->scratch2.p, st);
        mark(ctx, kStageRanges);
        launch_tile_ranges(f->keys[f->sorted_buf].as<uint64_t>(), E, ranges, ntiles, st);
        f->vals_buf = f->sorted_buf;
    }
    f->sort_passes = np;
    const uint32_t* svals = f->vals[f->vals_buf].as<uint32_t>();
    uint32_t* torder = grow<uint32_t>(f->tile_order, ntiles);
    launch_tile_order(ranges, ntiles, torder, st);
    mark(ctx, -1);

    // output buffers
    const uint64_t npx = uint64_t(W) * H, nss = uint64_t(sw) * sh;
    f->alloc_outputs(npx);
    float *oc = f->out_color, *od = f->out_depth, *om = f->out_median, *on = f->out_normal,
          *ot = f->out_tfin;
    CompositeArgs ca{};
    ca.ranges = ranges;
    ca.tile_order = torder;
    ca.vals = svals;
    ca.records = pa.records;
    ca.K = opts->K;
    ca.t_threshold = float(opts->t_threshold);
    for (int i = 0; i < 3; ++i) ca.bg[i] = float(opts->background[i]);
    ca.far_sentinel = float(opts->far_sentinel);
    // K7 path: the CTA-cooperative cull once the tiles average >= 2048
    // entries (SVR_COOP_MIN; E is the capacity of a deferred frame)
    static const uint64_t coop_min = [] {
        const char* e = std::getenv("SVR_COOP_MIN");
        return e ? uint64_t(std::strtoull(e, nullptr, 10)) : uint64_t(2048);
    }();
    const bool coop = E >= coop_min * uint64_t(ntiles);
    f->composite_path = coop ? 1 : 0;
    if (ss1) {
        ca.color = oc, ca.depth = od, ca.median = om, ca.normal = on, ca.tfin = ot;
    } else {
        ca.color = grow<float>(f->ss_color, nss * 3);
        ca.depth = grow<float>(f->ss_depth, nss);
        ca.median = grow<float>(f->ss_median, nss);
        ca.normal = grow<float>(f->ss_normal, nss * 3);
        ca.tfin = grow<float>(f->ss_tfin, nss);
    }
    if (opts->record_stats) {
        ca.max_blend = grow<unsigned int>(f->max_blend, N);
        SVR_CUDA(cudaMemsetAsync(ca.max_blend, 0, N * 4, st));
    }
    const uint64_t nslots = uint64_t(ntiles) * 256;
    f->staged = false;
    f->compact_valid = false;
    if (f->training) {
        ca.pix_count = grow<uint32_t>(f->pix_count, nslots);
        SVR_CUDA(cudaMemsetAsync(ca.pix_count, 0, nslots * 4, st));
        static const bool stage_enabled = [] {
            const char* e = std::getenv("SVR_STAGED_RECORDS");
            return e == nullptr || e[0] != '0';
        }();
        if (stage_enabled && nslots < (uint64_t(1) << 32) &&
            uint64_t(f->stage_cap) * nslots < (uint64_t(1) << 32)) {
            ca.stage_entry = grow<uint32_t>(f->stage_entry, uint64_t(f->stage_cap) * nslots);
            ca.stage_T = grow<float>(f->stage_T, uint64_t(f->stage_cap) * nslots);
            ca.stage_cap = f->stage_cap;
            ca.stage_stride = uint32_t(nslots);
            ca.overflow = &status->overflow;
        }
    }

    // K7: composite
    mark(ctx, kStageComposite);
    launch_composite(cam, ca, false, coop, st);
    mark(ctx, kStageOther);

    if (f->training) {
        // ForwardRecords: per-pixel contribution lists in the reference's
        // order (tile-major, pixel row-major inside the tile).
        uint32_t* pb = grow<uint32_t>(f->pix_begin, uint64_t(ntiles) * 256);
        exclusive_scan_u32(ca.pix_count, pb, uint64_t(ntiles) * 256, &status->n_contribs,
                           ctx->scratch.p, st);
        launch_status_to_host(status, hs, st);
        SVR_CUDA(cudaStreamSynchronize(st));
        const uint64_t C = hs->n_contribs;
        require(C < (uint64_t(1) << 32), SVR_ERR_LENGTH, "contribution count exceeds 2^32");
        f->n_contribs = C;
        if (ca.stage_entry && !hs->overflow) {
            f->staged = true;  // one pass did it; compact lists are built on demand
        } else {
            // second pass writes the compact lists directly; a staged frame
            // that overflowed doubles its capacity for the next render
            if (ca.stage_entry) f->stage_cap = std::min<uint32_t>(f->stage_cap * 2, 4096);
            CompositeArgs cr = ca;
            cr.pix_begin = pb;
            cr.contrib_entry = grow<uint32_t>(f->contrib_entry, C);
            cr.contrib_T = grow<float>(f->contrib_T, C);
            cr.max_blend = nullptr;
            cr.stage_entry = nullptr;
            mark(ctx, kStageRecord);
            launch_composite(cam, cr, true, coop, st);
            mark(ctx, -1);
            f->compact_valid = true;
        }
        f->has_records = true;
    }

    // K8: area downsampling of the five outputs (identity when ss == 1)
    if (!ss1) {
        TapSet taps = ensure_taps(f);
        mark(ctx, kStageDownsample);
        launch_downsample(taps.fwd, ca.color, 3, sw, oc, W, H, st);
        launch_downsample(taps.fwd, ca.depth, 1, sw, od, W, H, st);
        launch_downsample(taps.fwd, ca.median, 1, sw, om, W, H, st);
        launch_downsample(taps.fwd, ca.normal, 3, sw, on, W, H, st);
        launch_downsample(taps.fwd, ca.tfin, 1, sw, ot, W, H, st);
    }
    (void)nss;
    mark(ctx, -1);
    f->n_visible = ~uint64_t(0);  // computed lazily
    if (deferred) {
        if (!ctx->overflow_count.p) {  // the context's counter starts at zero
            grow<unsigned int>(ctx->overflow_count, 1);
            SVR_CUDA(cudaMemsetAsync(ctx->overflow_count.p, 0, sizeof(unsigned int), st));
        }
        launch_status_to_host(status, hs, st, f->e_cap, ctx->overflow_count.as<unsigned int>());
        if (!f->done) SVR_CUDA(cudaEventCreateWithFlags(&f->done, cudaEventDisableTiming));
        SVR_CUDA(cudaEventRecord(f->done, st));  // settle this frame without draining the stream
    }
}

void resolve_frame(svr_frame* f);


// Compact (reference-order) contribution lists for the host-facing records.
void ensure_compact(svr_frame* f) {
    if (!f->has_records || f->compact_valid) return;
    const uint64_t nslots = uint64_t(f->ntx) * f->nty * 256;
    launch_compact_contribs(f->pix_count.as<uint32_t>(), f->pix_begin.as<uint32_t>(),
                            f->stage_entry.as<uint32_t>(), f->stage_T.as<float>(),
                            uint32_t(nslots), grow<uint32_t>(f->contrib_entry, f->n_contribs),
                            grow<float>(f->contrib_T, f->n_contribs), f->ctx->stream);
    f->compact_valid = true;
}

uint64_t count_visible(svr_frame* f) {
    if (f->n_visible != ~uint64_t(0)) return f->n_visible;
    svr_ctx* ctx = f->ctx;
    cudaStream_t st = ctx->stream;
    const uint64_t N = f->n_voxels;
    uint32_t* flags = grow<uint32_t>(f->visible_rank, N);
    launch_visible_flags(f->rects.as<int4>(), N, flags, st);
    DevBuf tot;
    tot.reserve(8);
    ctx->scratch.reserve(scan_scratch_bytes(N));
    exclusive_scan_u32(flags, flags, N, tot.as<unsigned long long>(), ctx->scratch.p, st);
    unsigned long long h = 0;
    SVR_CUDA(cudaMemcpyAsync(&h, tot.p, 8, cudaMemcpyDeviceToHost, st));
    SVR_CUDA(cudaStreamSynchronize(st));
    f->n_visible = h;
    return h;
}

struct BufView {
    const void* p;
    size_t bytes;
};

BufView frame_buffer(svr_frame* f, svr_buffer which) {
    require(f && f->ctx, SVR_ERR_INVALID_ARGUMENT, "frame has not been rendered");
    const uint64_t npx = uint64_t(f->W) * f->H, nss = uint64_t(f->sw) * f->sh;
    const bool ss1 = (f->sw == f->W && f->sh == f->H);
    const uint64_t ntiles = uint64_t(f->ntx) * f->nty;
    switch (which) {  // materialised buffers reuse scratch an async copy may still read
        case SVR_BUF_COLOR: case SVR_BUF_DEPTH: case SVR_BUF_MEDIAN_DEPTH: case SVR_BUF_NORMAL:
        case SVR_BUF_TRANSMITTANCE: case SVR_BUF_OUTPUTS: case SVR_BUF_MAX_BLEND: case SVR_BUF_SS_COLOR:
        case SVR_BUF_SS_DEPTH: case SVR_BUF_SS_TFIN: case SVR_BUF_TILE_RANGES:
        case SVR_BUF_TILE_MASKS: case SVR_BUF_VOXEL_RECTS: break;
        default:
            wait_copies(f);
            resolve_frame(f);  // these need the entry count
    }
    switch (which) {
        case SVR_BUF_COLOR: return {f->out_color, npx * 12};
        case SVR_BUF_DEPTH: return {f->out_depth, npx * 4};
        case SVR_BUF_MEDIAN_DEPTH: return {f->out_median, npx * 4};
        case SVR_BUF_NORMAL: return {f->out_normal, npx * 12};
        case SVR_BUF_TRANSMITTANCE: return {f->out_tfin, npx * 4};
        case SVR_BUF_OUTPUTS: return {f->out_color, npx * 36};
        case SVR_BUF_MAX_BLEND:
            require(f->opts.record_stats, SVR_ERR_INVALID_ARGUMENT, "render without record_stats");
            return {f->max_blend.p, f->n_voxels * 4};
        case SVR_BUF_SS_COLOR: return {ss1 ? f->out_color : f->ss_color.p, nss * 12};
        case SVR_BUF_SS_DEPTH: return {ss1 ? f->out_depth : f->ss_depth.p, nss * 4};
        case SVR_BUF_SS_TFIN: return {ss1 ? f->out_tfin : f->ss_tfin.p, nss * 4};
        case SVR_BUF_SORT_KEYS:
        case SVR_BUF_SORT_VALUES:
            if (f->packed && (!f->sort_keys_kept || f->huge_used)) {
                // production frames keep only the sorted values (merged with
                // the huge pairs' entries when those took the merge path)
                require(which == SVR_BUF_SORT_VALUES, SVR_ERR_INVALID_ARGUMENT,
                        "sorted key dump needs svr_ctx_set_debug");
                return {f->vals[f->vals_buf].p, f->n_entries * 4};
            }
            if (f->packed) {
                uint64_t* k = grow<uint64_t>(f->ref_keys, f->n_entries);
                uint32_t* v = grow<uint32_t>(f->ref_vals, f->n_entries);
                launch_unpack_entries(f->keys[f->sorted_buf].as<uint64_t>(), f->n_entries, f->fmt,
                                      f->scene->paths.as<uint64_t>(), k, v, f->ctx->stream);
                return which == SVR_BUF_SORT_KEYS ? BufView{k, f->n_entries * 8}
                                                  : BufView{v, f->n_entries * 4};
            }
            return which == SVR_BUF_SORT_KEYS ? BufView{f->keys[f->sorted_buf].p, f->n_entries * 8}
                                              : BufView{f->vals[f->sorted_buf].p, f->n_entries * 4};
        case SVR_BUF_TILE_RANGES: return {f->ranges.p, ntiles * 8};
        case SVR_BUF_TILE_MASKS: return {f->tile_masks.p, ntiles};
        case SVR_BUF_VOXEL_RECTS: return {f->rects.p, f->n_voxels * 16};
        case SVR_BUF_VOXEL_AABB:
            require(f->ctx->debug, SVR_ERR_INVALID_ARGUMENT, "AABB dump needs svr_ctx_set_debug");
            return {f->aabb.p, f->n_voxels * 32};
        case SVR_BUF_ENTRIES_KEYS:
        case SVR_BUF_ENTRIES_VALUES:
            require(f->ctx->debug, SVR_ERR_INVALID_ARGUMENT, "entry dump needs svr_ctx_set_debug");
            if (f->packed) {
                uint64_t* k = grow<uint64_t>(f->ref_keys, f->n_entries);
                uint32_t* v = grow<uint32_t>(f->ref_vals, f->n_entries);
                launch_unpack_entries(f->dbg_keys.as<uint64_t>(), f->n_entries, f->fmt,
                                      f->scene->paths.as<uint64_t>(), k, v, f->ctx->stream);
                return which == SVR_BUF_ENTRIES_KEYS ? BufView{k, f->n_entries * 8}
                                                     : BufView{v, f->n_entries * 4};
            }
            return which == SVR_BUF_ENTRIES_KEYS ? BufView{f->dbg_keys.p, f->n_entries * 8}
                                                 : BufView{f->dbg_vals.p, f->n_entries * 4};
        case SVR_BUF_PIX_COUNT:
        case SVR_BUF_PIX_BEGIN: {
            require(f->has_records, SVR_ERR_RUNTIME, "frame has no forward records");
            uint32_t* img = grow<uint32_t>(f->bwd_dcolor, nss);
            launch_tile_to_image_u32(which == SVR_BUF_PIX_COUNT ? f->pix_count.as<uint32_t>()
                                                                : f->pix_begin.as<uint32_t>(),
                                     img, f->sw, f->sh, f->ntx, f->ctx->stream);
            return {img, nss * 4};
        }
        default: break;
    }
    throw Error(SVR_ERR_INVALID_ARGUMENT, "unknown buffer id");
}

// Settles a deferred frame: the live entry count is read (the frame's work
// is complete), and a frame that outgrew its capacity is rendered again
// with the count known (its pending asynchronous downloads are repeated).
void resolve_frame(svr_frame* f) {
    if (!f || !f->e_pending) return;
    SVR_CUDA(cudaEventSynchronize(f->done));
    const FrameStatus* hs = static_cast<const FrameStatus*>(f->hstatus.p);
    const uint64_t E = hs->n_entries + hs->n_huge_entries;
    f->huge_hint = hs->n_huge_pairs;
    f->e_pending = false;
    if (E <= f->e_cap) {
        f->n_entries = E;
        f->e_cap = std::max<uint64_t>(f->e_cap, E + E / 8);
        return;
    }
    f->e_cap = E + E / 4 + 1024;
    auto dl = f->pending_dl;
    const svr_camera cam = f->req_cam;
    const svr_render_options opts = f->req_opts;
    render_impl(f->ctx, f->scene, &cam, &opts, f, false);
    for (const auto& d : dl) {
        BufView b = frame_buffer(f, d.which);
        SVR_CUDA(cudaMemcpyAsync(d.dst, b.p, d.bytes, cudaMemcpyDeviceToHost, f->ctx->stream));
    }
    SVR_CUDA(cudaStreamSynchronize(f->ctx->stream));
}

void backward_impl(svr_ctx* ctx, const svr_scene* scene, svr_frame* f, const svr_upstream* up,
                   svr_gradients* out, bool accumulate) {
    require(ctx && scene && f && up && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
    set_device(ctx);
    require(f->has_records, SVR_ERR_RUNTIME,
            "frame has no forward records (render with training = true)");
    require(f->scene == scene, SVR_ERR_RUNTIME, "frame was rendered from another scene");
    // raster.cpp:327-332
    require(!up->d_weight || up->n_d_weight == f->n_contribs, SVR_ERR_RUNTIME,
            "per-contribution weight gradients do not match the records");
    require(!up->d_voxel_color || up->n_d_voxel_color == f->n_contribs, SVR_ERR_RUNTIME,
            "per-contribution color gradients do not match the records");
    wait_copies(f);
    resolve_frame(f);
    cudaStream_t st = ctx->stream;
    const uint64_t N = scene->n_voxels, P = scene->n_pool;
    const uint64_t shn = N * uint64_t(scene->sh_stride);
    const uint64_t npx = uint64_t(f->W) * f->H, nss = uint64_t(f->sw) * f->sh;
    const bool ss1 = (f->sw == f->W && f->sh == f->H);

    // Stage upstream buffers on the device.
    struct Up {
        const float* p;
        uint64_t n;
    };
    Up ins[6] = {{up->d_color, npx * 3},        {up->d_depth, npx},
                 {up->d_normal, npx * 3},       {up->d_tfin_ss, nss},
                 {up->d_weight, f->n_contribs}, {up->d_voxel_color, f->n_contribs * 3}};
    const float* dev_in[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    uint64_t total = 0;
    for (auto& u : ins)
        if (u.p && !up->on_device) total += (u.n + 3) & ~uint64_t(3);
    float* stage = total ? grow<float>(f->bwd_dcolor, total + 16) : nullptr;
    uint64_t off = 0;
    for (int i = 0; i < 6; ++i) {
        if (!ins[i].p) continue;
        if (up->on_device) {
            dev_in[i] = ins[i].p;
        } else {
            SVR_CUDA(cudaMemcpyAsync(stage + off, ins[i].p, ins[i].n * 4, cudaMemcpyHostToDevice, st));
            dev_in[i] = stage + off;
            off += (ins[i].n + 3) & ~uint64_t(3);
        }
    }
    // Lift image-level grads to the supersampled grid (raster.cpp:317-324).
    const float* gC = dev_in[0];
    const float* gD = dev_in[1];
    const float* gN = dev_in[2];
    if (!ss1 && (gC || gD || gN)) {
        TapSet taps = ensure_taps(f);
        float* lift = grow<float>(f->bwd_lift, nss * 7);
        if (gC) {
            launch_lift(taps.adj, gC, 3, f->W, lift, f->sw, f->sh, st);
            gC = lift;
        }
        if (gD) {
            launch_lift(taps.adj, gD, 1, f->W, lift + nss * 3, f->sw, f->sh, st);
            gD = lift + nss * 3;
        }
        if (gN) {
            launch_lift(taps.adj, gN, 3, f->W, lift + nss * 4, f->sw, f->sh, st);
            gN = lift + nss * 4;
        }
    }

    // Gradient outputs on device.
    float *gd = out->density, *gs = out->sh, *gp = out->priority;
    if (!out->on_device) {
        gd = grow<float>(ctx->bwd_density, P);
        gs = grow<float>(ctx->bwd_sh, shn);
        gp = grow<float>(ctx->bwd_priority, N);
        require(!accumulate, SVR_ERR_INVALID_ARGUMENT, "accumulate needs device gradient buffers");
    }
    require(gd && gs && gp, SVR_ERR_INVALID_ARGUMENT, "gradient buffers must not be null");
    if (!accumulate) {
        SVR_CUDA(cudaMemsetAsync(gd, 0, P * 4, st));
        SVR_CUDA(cudaMemsetAsync(gp, 0, N * 4, st));
    }
    // per-voxel gradient records (16 floats): zero when (re)allocated, then
    // kept zero by the epilogue, which consumes every record K9 touched
    if (f->bwd_gc.bytes < N * 64 || !f->gvox_clean) {
        f->bwd_gc.reserve(std::max<uint64_t>(N, 1) * 64);
        SVR_CUDA(cudaMemsetAsync(f->bwd_gc.p, 0, f->bwd_gc.bytes, st));
    }
    float* gvox = f->bwd_gc.as<float>();
    f->gvox_clean = false;

    BackwardArgs ba{};
    ba.ranges = f->ranges.as<uint2>();
    ba.tile_order = f->tile_order.as<uint32_t>();
    ba.vals = f->vals[f->vals_buf].as<uint32_t>();
    ba.records = f->records.as<float4>();
    ba.corner_index = scene->corner_index.as<uint32_t>();
    ba.K = f->opts.K;
    for (int i = 0; i < 3; ++i) ba.bg[i] = float(f->opts.background[i]);
    ba.gC = gC;
    ba.gD = gD;
    ba.gN = gN;
    ba.gT = dev_in[3];
    ba.d_weight = dev_in[4];
    ba.d_voxel_color = dev_in[5];
    ba.pix_count = f->pix_count.as<uint32_t>();
    ba.pix_begin = f->pix_begin.as<uint32_t>();
    ba.contrib_entry = f->staged ? f->stage_entry.as<uint32_t>() : f->contrib_entry.as<uint32_t>();
    ba.contrib_T = f->staged ? f->stage_T.as<float>() : f->contrib_T.as<float>();
    ba.stage_stride = f->staged ? uint32_t(uint64_t(f->ntx) * f->nty * 256) : 0u;
    ba.g_vox = gvox;
    mark(ctx, kStageBackward);
    launch_composite_backward(f->cam, ba, st);

    EpilogueArgs ea{};
    ea.n = N;
    ea.paths = scene->paths.as<uint64_t>();
    ea.rects = f->rects.as<int4>();
    ea.records = f->records.as<float4>();
    ea.view_dir = f->view_dir.as<float4>();
    ea.corner_index = scene->corner_index.as<uint32_t>();
    // the SH clamp mask from the forward's colours, unless the pools changed
    // since the forward (then from the coefficients the backward is given)
    ea.sh = scene->param_version != f->param_version ? scene->sh.as<float>() : nullptr;
    ea.sh_degree = scene->sh_degree;
    ea.sh_stride = scene->sh_stride;
    for (int i = 0; i < 3; ++i) ea.bc[i] = scene->bounds_center[i];
    ea.bsize = scene->bounds_size;
    ea.g_vox = gvox;
    ea.g_sh = gs;
    ea.g_density = gd;
    ea.g_priority = gp;
    ea.accumulate = accumulate ? 1 : 0;
    // When most voxels are outside the view (large scenes, config 5) the
    // epilogue walks K1's list of visible voxels (an overwriting backward
    // then clears the SH gradients first); otherwise one pass over every
    // voxel, which also writes the others' zero SH gradients (config 5:
    // epilogue 3.35 -> 1.40 ms per step; config 3, 98 % visible: full pass
    // 0.25 ms vs list 0.31 ms + a 200 MB clear).
    if (f->training && f->vis_list.p && 2 * f->n_vis_list < N) {
        ea.list = f->vis_list.as<uint32_t>();
        ea.n_list = &f->status.as<FrameStatus>()->n_vis_list;
        if (!accumulate) SVR_CUDA(cudaMemsetAsync(gs, 0, shn * 4, st));
    }
    mark(ctx, kStageEpilogue);
    launch_voxel_epilogue(f->cam, ea, st);
    f->gvox_clean = true;
    mark(ctx, -1);

    if (!out->on_device) {
        if (out->density) SVR_CUDA(cudaMemcpyAsync(out->density, gd, P * 4, cudaMemcpyDeviceToHost, st));
        if (out->sh) SVR_CUDA(cudaMemcpyAsync(out->sh, gs, shn * 4, cudaMemcpyDeviceToHost, st));
        if (out->priority) SVR_CUDA(cudaMemcpyAsync(out->priority, gp, N * 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
    }
}

}  // namespace

// Entry points shared with dropin_support.cu.
uint64_t frame_visible_count(svr_frame* f) { return count_visible(f); }
int guarded_call(void (*fn)(void*), void* arg) {
    return guard([&] { fn(arg); });
}
DevCamera make_dev_camera(const svr_camera& c) { return dev_camera(c); }

}  // namespace svrb

using namespace svrb;

extern "C" {

const char* svr_last_error(void) { return g_last_error.c_str(); }
int svr_abi_version(void) { return SVR_ABI_VERSION; }

int svr_ctx_create(int device, svr_ctx** out) {
    return guard([&] {
        require(out != nullptr, SVR_ERR_INVALID_ARGUMENT, "null output");
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            throw Error(SVR_ERR_NO_DEVICE, "no CUDA device: the rasterizer has no CPU fallback");
        require(device >= 0 && device < n, SVR_ERR_INVALID_ARGUMENT, "device index out of range");
        auto* c = new svr_ctx;
        c->device = device;
        SVR_CUDA(cudaSetDevice(device));
        SVR_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        SVR_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        SVR_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        *out = c;
    });
}

int svr_ctx_destroy(svr_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->copy_stream);
        for (auto& m : ctx->marks) cudaEventDestroy(m.second);
        for (auto& e : ctx->event_pool) cudaEventDestroy(e);
        cudaStreamDestroy(ctx->stream);
        cudaStreamDestroy(ctx->copy_stream);
        delete ctx;
    });
}

void* svr_ctx_stream(svr_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int svr_ctx_synchronize(svr_ctx* ctx) {
    return guard([&] { SVR_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int svr_ctx_set_async(svr_ctx* ctx, int on) {
    return guard([&] {
        require(ctx != nullptr, SVR_ERR_INVALID_ARGUMENT, "null argument");
        ctx->async_frames = on != 0;
    });
}

int svr_ctx_overflow_count(svr_ctx* ctx, uint32_t* out) {
    return guard([&] {
        require(ctx && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        *out = 0;
        if (ctx->overflow_count.p) {
            SVR_CUDA(cudaMemcpyAsync(out, ctx->overflow_count.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
            SVR_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    });
}

int svr_ctx_set_debug(svr_ctx* ctx, int debug) {
    return guard([&] { ctx->debug = debug != 0; });
}

int svr_scene_upload(svr_ctx* ctx, const svr_scene_desc* d, svr_scene** out) {
    return guard([&] {
        require(ctx && d && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        require(d->sh_degree >= 0 && d->sh_degree <= 3, SVR_ERR_INVALID_ARGUMENT,
                "SH degree out of [0,3]");
        set_device(ctx);
        const uint64_t N = d->n_voxels;
        const int stride = 3 * (d->sh_degree + 1) * (d->sh_degree + 1);
        std::vector<uint64_t> paths(N);
        int max_level = 1;
        for (uint64_t i = 0; i < N; ++i) {
            int lv = d->levels[i];
            // check_level / to_voxel_index (octree.hpp:47-49, 68-73)
            require(lv >= 1 && lv <= kMaxLevel, SVR_ERR_INVALID_ARGUMENT,
                    "octree level out of [1,16]");
            int shift = 3 * (kMaxLevel - lv);
            require(shift >= 64 || (d->codes[i] & ((uint64_t(1) << shift) - 1)) == 0,
                    SVR_ERR_INVALID_ARGUMENT, "octpath has nonzero bits below its level");
            require((d->codes[i] >> 48) == 0, SVR_ERR_INVALID_ARGUMENT,
                    "octpath code exceeds 48 bits");
            paths[i] = d->codes[i] | (uint64_t(lv) << 48);
            max_level = std::max(max_level, lv);
        }
        for (uint64_t i = 0; i < N * 8; ++i)
            require(d->corner_index[i] < d->n_pool, SVR_ERR_INVALID_ARGUMENT,
                    "corner index out of the density pool");
        auto* s = new svr_scene;
        try {
            s->n_voxels = N;
            s->n_pool = d->n_pool;
            s->sh_degree = d->sh_degree;
            s->sh_stride = stride;
            s->max_level = max_level;
            for (int i = 0; i < 3; ++i) s->bounds_center[i] = d->bounds_center[i];
            s->bounds_size = d->bounds_size;
            s->paths.reserve(std::max<uint64_t>(N, 1) * 8);
            s->corner_index.reserve(std::max<uint64_t>(N, 1) * 32);
            s->density.reserve(std::max<uint64_t>(d->n_pool, 1) * 4);
            s->sh.reserve(std::max<uint64_t>(N * stride, 1) * 4);
            if (N) {
                SVR_CUDA(cudaMemcpy(s->paths.p, paths.data(), N * 8, cudaMemcpyHostToDevice));
                SVR_CUDA(cudaMemcpy(s->corner_index.p, d->corner_index, N * 32,
                                    cudaMemcpyHostToDevice));
                SVR_CUDA(cudaMemcpy(s->sh.p, d->sh, N * stride * 4, cudaMemcpyHostToDevice));
            }
            if (d->n_pool)
                SVR_CUDA(cudaMemcpy(s->density.p, d->density, d->n_pool * 4, cudaMemcpyHostToDevice));
            // Morton rank table for the sort keys (needs 8N < 2^32).
            if (N > 0 && N < (uint64_t(1) << 28)) {
                s->morton_rank.reserve(N * 8 * 4);
                s->morton_order.reserve(N * 8 * 4);
                DevBuf tmp;
                tmp.reserve(morton_rank_scratch_bytes(N, max_level));
                build_morton_rank(s->paths.as<uint64_t>(), N, max_level,
                                  s->morton_rank.as<uint32_t>(), s->morton_order.as<uint32_t>(), tmp.p,
                                  ctx->stream);
                // K1 walks a scene stored out of spatial order in Morton order
                // (less than 90 % of neighbouring voxels in ascending code order)
                constexpr uint64_t kPathCode = (uint64_t(1) << 48) - 1;
                uint64_t asc = 0;
                for (uint64_t i = 1; i < N; ++i) asc += (paths[i] & kPathCode) > (paths[i - 1] & kPathCode);
                const char* po = std::getenv("SVR_PROC_ORDER");  // 0: never, 1: always
                const bool want = po ? po[0] == '1' : (N > 1 && asc * 10 < (N - 1) * 9);
                s->unordered = want;
                SVR_CUDA(cudaStreamSynchronize(ctx->stream));
                s->rank_bits = bit_width(8 * N - 1);
            }
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

int svr_scene_prune(svr_ctx* ctx, const svr_scene* s, const float* max_blend_weight, uint64_t n,
                    double threshold, int32_t on_device, svr_scene** out) {
    return guard([&] {
        require(ctx && s && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        require(n == s->n_voxels, SVR_ERR_INVALID_ARGUMENT, "prune: stats size mismatch");
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        DevBuf stat, keep;
        const float* dstat = max_blend_weight;
        if (!on_device && n) {
            stat.reserve(n * 4);
            SVR_CUDA(cudaMemcpyAsync(stat.p, max_blend_weight, n * 4, cudaMemcpyHostToDevice, st));
            dstat = stat.as<float>();
        }
        keep.reserve(std::max<uint64_t>(n, 1) * 4);
        if (n) launch_keep_flags(dstat, n, threshold, keep.as<uint32_t>(), st);
        *out = adapt_scene(ctx, s, keep.as<uint32_t>(), false, 0.0f);
    });
}

int svr_scene_subdivide(svr_ctx* ctx, const svr_scene* s, const uint32_t* selected, uint64_t n_sel,
                        svr_scene** out) {
    return guard([&] {
        require(ctx && s && out && (n_sel == 0 || selected), SVR_ERR_INVALID_ARGUMENT,
                "null argument");
        set_device(ctx);
        const uint64_t N = s->n_voxels;
        std::vector<uint64_t> paths(N);
        if (N) SVR_CUDA(cudaMemcpy(paths.data(), s->paths.p, N * 8, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> sel(N, 0u);
        uint64_t n_new = 0;
        for (uint64_t q = 0; q < n_sel; ++q) {  // optim.cpp:239-245
            const uint32_t vi = selected[q];
            require(vi < N, SVR_ERR_INVALID_ARGUMENT, "subdivide: voxel id out of range");
            if (int(paths[vi] >> 48) >= kMaxLevel) continue;  // finest level: kept as-is
            if (!sel[vi]) ++n_new;
            sel[vi] = 1u;
        }
        require(N + 7 * n_new <= (uint64_t(1) << 29), SVR_ERR_LENGTH,
                "subdivision exceeds voxel capacity");
        DevBuf flags;
        flags.reserve(std::max<uint64_t>(N, 1) * 4);
        if (N) SVR_CUDA(cudaMemcpy(flags.p, sel.data(), N * 4, cudaMemcpyHostToDevice));
        *out = adapt_scene(ctx, s, flags.as<uint32_t>(), true, 0.0f);
    });
}

int svr_scene_remap(const svr_scene* s, int64_t* voxel_src, int64_t* pool_src) {
    return guard([&] {
        require(s && s->has_remap, SVR_ERR_INVALID_ARGUMENT, "scene was not produced by adaptation");
        if (voxel_src && s->n_voxels)
            SVR_CUDA(cudaMemcpy(voxel_src, s->voxel_src.p, s->n_voxels * 8, cudaMemcpyDeviceToHost));
        if (pool_src && s->n_pool)
            SVR_CUDA(cudaMemcpy(pool_src, s->pool_src.p, s->n_pool * 8, cudaMemcpyDeviceToHost));
    });
}

int svr_scene_info(const svr_scene* s, svr_scene_desc* out) {
    return guard([&] {
        require(s && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        *out = svr_scene_desc{};
        out->n_voxels = s->n_voxels;
        out->n_pool = s->n_pool;
        out->sh_degree = s->sh_degree;
        for (int i = 0; i < 3; ++i) out->bounds_center[i] = s->bounds_center[i];
        out->bounds_size = s->bounds_size;
    });
}

int svr_scene_download(svr_ctx* ctx, const svr_scene* s, uint64_t* codes, uint8_t* levels,
                       uint32_t* corner_index, float* density, float* sh) {
    return guard([&] {
        require(ctx && s, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        const uint64_t N = s->n_voxels, P = s->n_pool;
        std::vector<uint64_t> paths(N);
        if (N && (codes || levels))
            SVR_CUDA(cudaMemcpyAsync(paths.data(), s->paths.p, N * 8, cudaMemcpyDeviceToHost, st));
        if (N && corner_index)
            SVR_CUDA(cudaMemcpyAsync(corner_index, s->corner_index.p, N * 32, cudaMemcpyDeviceToHost, st));
        if (P && density) SVR_CUDA(cudaMemcpyAsync(density, s->density.p, P * 4, cudaMemcpyDeviceToHost, st));
        if (N && sh)
            SVR_CUDA(cudaMemcpyAsync(sh, s->sh.p, N * uint64_t(s->sh_stride) * 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < N; ++i) {
            if (codes) codes[i] = paths[i] & ((uint64_t(1) << 48) - 1);
            if (levels) levels[i] = uint8_t(paths[i] >> 48);
        }
    });
}

int svr_scene_save_svrx(svr_ctx* ctx, const svr_scene* s, const char* path) {
    return guard([&] {
        require(ctx && s && path, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        SvrxScene h;
        const uint64_t N = s->n_voxels, P = s->n_pool;
        std::vector<uint64_t> paths(N);
        h.corner_index.resize(N * 8);
        h.density.resize(P);
        h.sh.resize(N * uint64_t(s->sh_stride));
        // the parameters as the device holds them now (training updates them in place)
        if (N) {
            SVR_CUDA(cudaMemcpyAsync(paths.data(), s->paths.p, N * 8, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemcpyAsync(h.corner_index.data(), s->corner_index.p, N * 32,
                                     cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemcpyAsync(h.sh.data(), s->sh.p, h.sh.size() * 4, cudaMemcpyDeviceToHost, st));
        }
        if (P) SVR_CUDA(cudaMemcpyAsync(h.density.data(), s->density.p, P * 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        h.codes.resize(N);
        h.levels.resize(N);
        for (uint64_t i = 0; i < N; ++i) {
            h.codes[i] = paths[i] & ((uint64_t(1) << 48) - 1);
            h.levels[i] = uint8_t(paths[i] >> 48);
        }
        h.sh_degree = s->sh_degree;
        for (int i = 0; i < 3; ++i) h.bounds_center[i] = s->bounds_center[i];
        h.bounds_size = s->bounds_size;
        svrx_write(path, svrx_encode(h));
    });
}

int svr_scene_load_svrx(svr_ctx* ctx, const char* path, svr_scene** out) {
    return guard([&] {
        require(ctx && path && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        SvrxScene h = svrx_read(path);
        svrx_validate(h, path);
        svr_scene_desc d{};
        d.n_voxels = h.codes.size();
        d.n_pool = h.density.size();
        d.sh_degree = h.sh_degree;
        for (int i = 0; i < 3; ++i) d.bounds_center[i] = h.bounds_center[i];
        d.bounds_size = h.bounds_size;
        d.codes = h.codes.data();
        d.levels = h.levels.data();
        d.corner_index = h.corner_index.data();
        d.density = h.density.data();
        d.sh = h.sh.data();
        const int st = svr_scene_upload(ctx, &d, out);
        if (st != SVR_OK) throw Error(st, svr_last_error());
    });
}

int svr_scene_set_params(svr_ctx* ctx, svr_scene* s, const float* density, const float* sh,
                         int on_device) {
    return guard([&] {
        require(ctx && s, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (density && s->n_pool)
            SVR_CUDA(cudaMemcpyAsync(s->density.p, density, s->n_pool * 4, k, ctx->stream));
        if (sh && s->n_voxels)
            SVR_CUDA(cudaMemcpyAsync(s->sh.p, sh, s->n_voxels * s->sh_stride * 4, k, ctx->stream));
        if (!on_device) SVR_CUDA(cudaStreamSynchronize(ctx->stream));
        if (sh) ++s->param_version;
    });
}

int svr_scene_destroy(svr_scene* s) {
    return guard([&] { delete s; });
}

int svr_scene_param_ptrs(svr_scene* s, float** density, float** sh, uint64_t* n_pool,
                         uint64_t* n_sh) {
    return guard([&] {
        require(s != nullptr, SVR_ERR_INVALID_ARGUMENT, "null scene");
        if (density) *density = s->density.as<float>();
        if (sh) *sh = s->sh.as<float>();
        if (n_pool) *n_pool = s->n_pool;
        if (n_sh) *n_sh = s->n_voxels * s->sh_stride;
    });
}

int svr_frame_create(svr_ctx* ctx, svr_frame** out) {
    return guard([&] {
        require(ctx && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        auto* f = new svr_frame;
        f->ctx = ctx;
        *out = f;
    });
}

int svr_frame_destroy(svr_frame* f) {
    return guard([&] {
        if (!f) return;
        if (f->ctx) cudaSetDevice(f->ctx->device);
        if (f->copied) {
            cudaEventSynchronize(f->copied);
            cudaEventDestroy(f->copied);
        }
        if (f->ready) cudaEventDestroy(f->ready);
        if (f->done) cudaEventDestroy(f->done);
        delete f;
    });
}

int svr_render(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
               const svr_render_options* opts, svr_frame* frame) {
    return guard([&] { render_impl(ctx, scene, cam, opts, frame); });
}

int svr_frame_get_info(svr_frame* f, svr_frame_info* out) {
    return guard([&] {
        require(f && out && f->scene, SVR_ERR_INVALID_ARGUMENT, "frame has not been rendered");
        set_device(f->ctx);
        resolve_frame(f);
        out->width = f->W;
        out->height = f->H;
        out->ss_width = f->sw;
        out->ss_height = f->sh;
        out->tiles_x = f->ntx;
        out->tiles_y = f->nty;
        out->n_visible = count_visible(f);
        out->n_entries = f->n_entries;
        out->n_contribs = f->n_contribs;
        out->sort_passes = f->sort_passes;
        out->training = f->training;
        out->composite_path = f->composite_path;
        out->reserved = 0;
    });
}

int svr_frame_download(svr_frame* f, svr_buffer which, void* dst, size_t bytes) {
    return guard([&] {
        set_device(f->ctx);
        resolve_frame(f);
        BufView b = frame_buffer(f, which);
        require(bytes == b.bytes, SVR_ERR_INVALID_ARGUMENT, "download size mismatch");
        if (bytes)
            SVR_CUDA(cudaMemcpyAsync(dst, b.p, bytes, cudaMemcpyDeviceToHost, f->ctx->stream));
        SVR_CUDA(cudaStreamSynchronize(f->ctx->stream));
    });
}

int svr_frame_download_async(svr_frame* f, svr_buffer which, void* dst, size_t bytes) {
    return guard([&] {
        require(f && f->ctx && dst, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(f->ctx);
        BufView b = frame_buffer(f, which);
        require(bytes == b.bytes, SVR_ERR_INVALID_ARGUMENT, "download size mismatch");
        if (!f->ready) SVR_CUDA(cudaEventCreateWithFlags(&f->ready, cudaEventDisableTiming));
        if (!f->copied) SVR_CUDA(cudaEventCreateWithFlags(&f->copied, cudaEventDisableTiming));
        SVR_CUDA(cudaEventRecord(f->ready, f->ctx->stream));
        SVR_CUDA(cudaStreamWaitEvent(f->ctx->copy_stream, f->ready, 0));
        if (bytes)
            SVR_CUDA(cudaMemcpyAsync(dst, b.p, bytes, cudaMemcpyDeviceToHost, f->ctx->copy_stream));
        SVR_CUDA(cudaEventRecord(f->copied, f->ctx->copy_stream));
        f->copy_pending = true;
        if (f->e_pending) f->pending_dl.push_back({which, dst, bytes});
    });
}

int svr_frame_wait(svr_frame* f) {
    return guard([&] {
        require(f != nullptr, SVR_ERR_INVALID_ARGUMENT, "null argument");
        if (f->copied) SVR_CUDA(cudaEventSynchronize(f->copied));
        if (f->ctx) {
            set_device(f->ctx);
            resolve_frame(f);  // an outgrown deferred frame is rendered and copied again
        }
        f->pending_dl.clear();
    });
}

int svr_frame_device_ptr(svr_frame* f, svr_buffer which, void** ptr, size_t* bytes) {
    return guard([&] {
        require(f && f->ctx && ptr && bytes, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(f->ctx);
        resolve_frame(f);  // the pointer must address a complete frame's buffer
        BufView b = frame_buffer(f, which);
        *ptr = const_cast<void*>(b.p);
        *bytes = b.bytes;
    });
}

int svr_frame_records(svr_frame* f, uint32_t* pre_vids, uint64_t n_pre, uint32_t* contrib_pre,
                      double* contrib_a, double* contrib_b, uint64_t n_contribs) {
    return guard([&] {
        require(f && f->has_records, SVR_ERR_RUNTIME, "frame has no forward records");
        set_device(f->ctx);
        cudaStream_t st = f->ctx->stream;
        ensure_compact(f);
        uint64_t nv = count_visible(f);
        require(n_pre == nv, SVR_ERR_INVALID_ARGUMENT, "pre size mismatch");
        require(n_contribs == f->n_contribs, SVR_ERR_INVALID_ARGUMENT, "contrib size mismatch");
        const uint64_t N = f->n_voxels;
        if (pre_vids && nv) {
            std::vector<int4> rects(N);
            SVR_CUDA(cudaMemcpy(rects.data(), f->rects.p, N * 16, cudaMemcpyDeviceToHost));
            uint64_t k = 0;
            for (uint64_t v = 0; v < N; ++v)
                if (rects[v].y >= rects[v].x) pre_vids[k++] = uint32_t(v);
        }
        if (n_contribs && (contrib_pre || contrib_a || contrib_b)) {
            DevBuf dp, da, db;
            uint32_t* p = grow<uint32_t>(dp, n_contribs);
            double* a = grow<double>(da, n_contribs);
            double* b = grow<double>(db, n_contribs);
            launch_contrib_segments(f->cam, f->ranges.as<uint2>(), f->vals[f->vals_buf].as<uint32_t>(),
                                    f->records.as<float4>(), f->pix_count.as<uint32_t>(),
                                    f->pix_begin.as<uint32_t>(), f->contrib_entry.as<uint32_t>(),
                                    f->visible_rank.as<uint32_t>(), p, a, b, f->ntx * f->nty, st);
            if (contrib_pre) SVR_CUDA(cudaMemcpyAsync(contrib_pre, p, n_contribs * 4, cudaMemcpyDeviceToHost, st));
            if (contrib_a) SVR_CUDA(cudaMemcpyAsync(contrib_a, a, n_contribs * 8, cudaMemcpyDeviceToHost, st));
            if (contrib_b) SVR_CUDA(cudaMemcpyAsync(contrib_b, b, n_contribs * 8, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaStreamSynchronize(st));
        }
    });
}

int svr_render_backward(svr_ctx* ctx, const svr_scene* scene, svr_frame* frame,
                        const svr_upstream* up, svr_gradients* out) {
    return guard([&] { backward_impl(ctx, scene, frame, up, out, false); });
}

int svr_l1_loss(svr_ctx* ctx, svr_frame* f, const float* gt, float* d_color, float* loss) {
    return guard([&] {
        require(ctx && f && gt && d_color, SVR_ERR_INVALID_ARGUMENT, "null argument");
        require(f->scene, SVR_ERR_INVALID_ARGUMENT, "frame has not been rendered");
        set_device(ctx);
        wait_copies(f);
        resolve_frame(f);
        launch_l1_loss(f->out_color, gt, uint64_t(f->W) * f->H * 3, d_color, loss,
                       ctx->stream);
    });
}

int svr_ray_losses(svr_ctx* ctx, svr_frame* f, const float* gt, const svr_ray_loss_weights* w,
                   svr_ray_loss_values* out, float* d_tfin_ss, float* d_weight,
                   float* d_voxel_color, int32_t on_device) {
    return guard([&] {
        require(ctx && f && gt && w && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        require(f->has_records, SVR_ERR_RUNTIME,
                "frame has no forward records (render with training = true)");
        // losses.cpp:154-161 sizes the upstream buffers the weights need
        require(w->w_T == 0.0 || d_tfin_ss, SVR_ERR_INVALID_ARGUMENT, "w_T needs d_tfin_ss");
        require((w->w_dist == 0.0 && w->w_R == 0.0) || d_weight, SVR_ERR_INVALID_ARGUMENT,
                "w_dist / w_R need d_weight");
        require(w->w_R == 0.0 || d_voxel_color, SVR_ERR_INVALID_ARGUMENT, "w_R needs d_voxel_color");
        set_device(ctx);
        wait_copies(f);
        cudaStream_t st = ctx->stream;
        const uint64_t nss = uint64_t(f->sw) * f->sh, C = f->n_contribs;
        const uint64_t ngt = uint64_t(f->W) * f->H * 3;
        const bool ss1 = (f->sw == f->W && f->sh == f->H);
        float *dgt = const_cast<float*>(gt), *dtf = d_tfin_ss, *dw = d_weight, *dvc = d_voxel_color;
        DevBuf tgt, ttf, tw, tvc;
        if (!on_device) {
            dgt = grow<float>(tgt, ngt);
            SVR_CUDA(cudaMemcpyAsync(dgt, gt, ngt * 4, cudaMemcpyHostToDevice, st));
            auto stage = [&](float* h, DevBuf& b, uint64_t n) -> float* {
                if (!h) return nullptr;
                float* d = grow<float>(b, n);
                SVR_CUDA(cudaMemcpyAsync(d, h, n * 4, cudaMemcpyHostToDevice, st));
                return d;
            };
            dtf = stage(d_tfin_ss, ttf, nss);
            dw = stage(d_weight, tw, C);
            dvc = stage(d_voxel_color, tvc, C * 3);
        }
        double* sums = grow<double>(f->rl_sums, 3);
        SVR_CUDA(cudaMemsetAsync(sums, 0, 3 * sizeof(double), st));
        RayLossArgs ra{};
        ra.ranges = f->ranges.as<uint2>();
        ra.vals = f->vals[f->vals_buf].as<uint32_t>();
        ra.records = f->records.as<float4>();
        ra.K = f->opts.K;
        ra.pix_count = f->pix_count.as<uint32_t>();
        ra.pix_begin = f->pix_begin.as<uint32_t>();
        ra.contrib_entry = f->staged ? f->stage_entry.as<uint32_t>() : f->contrib_entry.as<uint32_t>();
        ra.contrib_T = f->staged ? f->stage_T.as<float>() : f->contrib_T.as<float>();
        ra.stage_stride = f->staged ? uint32_t(uint64_t(f->ntx) * f->nty * 256) : 0u;
        ra.tfin = ss1 ? f->out_tfin : f->ss_tfin.as<float>();
        ra.gt = dgt;
        ra.gt_w = f->W;
        ra.gt_h = f->H;
        ra.w_T = w->w_T;
        ra.w_dist = w->w_dist;
        ra.w_R = w->w_R;
        ra.d_tfin_ss = dtf;
        ra.d_weight = dw;
        ra.d_voxel_color = dvc;
        ra.scratch = w->w_dist != 0.0 ? grow<float2>(f->rl_scratch, std::max<uint64_t>(C, 1)) : nullptr;
        ra.sums = sums;
        launch_ray_losses(f->cam, ra, st);
        f->rl_w[0] = w->w_T;
        f->rl_w[1] = w->w_dist;
        f->rl_w[2] = w->w_R;
        f->rl_pending = true;
        if (on_device == 2) return;  // deferred: values via svr_frame_loss_values
        double hs[3];
        SVR_CUDA(cudaMemcpyAsync(hs, sums, sizeof(hs), cudaMemcpyDeviceToHost, st));
        if (!on_device) {
            if (d_tfin_ss) SVR_CUDA(cudaMemcpyAsync(d_tfin_ss, dtf, nss * 4, cudaMemcpyDeviceToHost, st));
            if (d_weight) SVR_CUDA(cudaMemcpyAsync(d_weight, dw, C * 4, cudaMemcpyDeviceToHost, st));
            if (d_voxel_color)
                SVR_CUDA(cudaMemcpyAsync(d_voxel_color, dvc, C * 12, cudaMemcpyDeviceToHost, st));
        }
        SVR_CUDA(cudaStreamSynchronize(st));
        out->l_T = w->w_T != 0.0 ? hs[0] : 0.0;
        out->l_dist = w->w_dist != 0.0 ? hs[1] : 0.0;
        out->l_R = w->w_R != 0.0 ? hs[2] : 0.0;
    });
}

int svr_image_losses(svr_ctx* ctx, svr_frame* f, const float* gt, double w_mse, double w_ssim,
                     double* out, float* d_color, int32_t on_device) {
    return guard([&] {
        require(ctx && f && gt && out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        require(f->scene, SVR_ERR_INVALID_ARGUMENT, "frame has not been rendered");
        // ssim_core (losses.cpp:73-75)
        require(f->W >= 11 && f->H >= 11, SVR_ERR_INVALID_ARGUMENT,
                "ssim: images smaller than the 11x11 window");
        set_device(ctx);
        wait_copies(f);
        resolve_frame(f);  // losses of a complete frame, never of an outgrown deferred one
        cudaStream_t st = ctx->stream;
        const uint64_t n = uint64_t(f->W) * f->H * 3;
        ImageLossArgs a{};
        a.a = f->out_color;
        a.W = f->W;
        a.H = f->H;
        // gauss_kernel (losses.cpp:15-29) in double, then narrowed
        double k[11], ks = 0.0;
        for (int i = 0; i < 11; ++i) {
            const double d = i - 5;
            k[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
            ks += k[i];
        }
        for (int i = 0; i < 11; ++i) a.kern[i] = float(k[i] / ks);
        a.w_mse = w_mse;
        a.w_ssim = w_ssim;
        DevBuf tgt, td;
        float* dgt = const_cast<float*>(gt);
        float* dd = d_color;
        if (!on_device) {
            dgt = grow<float>(tgt, n);
            SVR_CUDA(cudaMemcpyAsync(dgt, gt, n * 4, cudaMemcpyHostToDevice, st));
            if (d_color) {
                dd = grow<float>(td, n);
                SVR_CUDA(cudaMemcpyAsync(dd, d_color, n * 4, cudaMemcpyHostToDevice, st));
            }
        }
        a.b = dgt;
        a.d_a = dd;
        const uint64_t wv = uint64_t(f->W - 10);
        a.mid = grow<float>(f->il_mid, 5 * wv * f->H * 3);
        a.maps = grow<float>(f->il_maps, 3 * wv * (f->H - 10) * 3);
        a.adj = grow<float>(f->il_adj, 3 * wv * f->H * 3);
        a.sums = grow<double>(f->il_sums, 2);
        SVR_CUDA(cudaMemsetAsync(a.sums, 0, 16, st));
        launch_image_losses(a, st);
        f->il_norm[0] = double(n);
        f->il_norm[1] = double(wv * (f->H - 10) * 3);
        f->il_pending = true;
        if (on_device == 2) return;  // deferred: values via svr_frame_loss_values
        double hs[2];
        SVR_CUDA(cudaMemcpyAsync(hs, a.sums, 16, cudaMemcpyDeviceToHost, st));
        if (!on_device && d_color)
            SVR_CUDA(cudaMemcpyAsync(d_color, dd, n * 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        out[0] = hs[0] / double(n);
        out[1] = 1.0 - hs[1] / double(wv * (f->H - 10) * 3);
    });
}

int svr_frame_loss_values(svr_frame* f, double* out) {
    return guard([&] {
        require(f && out && f->ctx, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(f->ctx);
        cudaStream_t st = f->ctx->stream;
        double il[2] = {0.0, 0.0}, rl[3] = {0.0, 0.0, 0.0};
        if (f->il_pending) SVR_CUDA(cudaMemcpyAsync(il, f->il_sums.p, 16, cudaMemcpyDeviceToHost, st));
        if (f->rl_pending) SVR_CUDA(cudaMemcpyAsync(rl, f->rl_sums.p, 24, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        out[0] = f->il_pending ? il[0] / f->il_norm[0] : 0.0;
        out[1] = f->il_pending ? 1.0 - il[1] / f->il_norm[1] : 0.0;
        out[2] = (f->rl_pending && f->rl_w[0] != 0.0) ? rl[0] : 0.0;
        out[3] = (f->rl_pending && f->rl_w[1] != 0.0) ? rl[1] : 0.0;
        out[4] = (f->rl_pending && f->rl_w[2] != 0.0) ? rl[2] : 0.0;
    });
}

int svr_ctx_take_adam_nan(svr_ctx* ctx, int32_t* nan_seen) {
    return guard([&] {
        require(ctx && nan_seen, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        unsigned int h = 0;
        if (ctx->adam_flag.p) {
            SVR_CUDA(cudaMemcpyAsync(&h, ctx->adam_flag.p, 4, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemsetAsync(ctx->adam_flag.p, 0, 4, st));
        }
        SVR_CUDA(cudaStreamSynchronize(st));
        *nan_seen = h != 0;
    });
}

int svr_adam_step(svr_ctx* ctx, float* params, const float* grads, double* m, double* v,
                  uint64_t n, int64_t step, double lr, double lr_alt, uint32_t period,
                  uint32_t n_primary, double beta1, double beta2, double eps, int32_t on_device) {
    return guard([&] {
        require(ctx && (n == 0 || (params && grads && m && v)), SVR_ERR_INVALID_ARGUMENT,
                "null argument");
        require(step >= 1, SVR_ERR_INVALID_ARGUMENT, "adam_step: step counts from 1");
        set_device(ctx);
        cudaStream_t st = ctx->stream;
        AdamArgs a{};
        a.n = n;
        // optim.cpp:334-335, on the host exactly as the reference
        a.bc1 = 1.0 - std::pow(beta1, double(step));
        a.bc2 = 1.0 - std::pow(beta2, double(step));
        a.lr = lr;
        a.lr_alt = lr_alt;
        a.beta1 = beta1;
        a.beta2 = beta2;
        a.eps = eps;
        a.period = period;
        a.n_primary = n_primary;
        DevBuf tp, tg, tm, tv;
        a.params = params;
        a.grads = grads;
        a.m = m;
        a.v = v;
        if (!on_device && n) {
            a.params = grow<float>(tp, n);
            a.m = grow<double>(tm, n);
            a.v = grow<double>(tv, n);
            float* g = grow<float>(tg, n);
            SVR_CUDA(cudaMemcpyAsync(a.params, params, n * 4, cudaMemcpyHostToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(g, grads, n * 4, cudaMemcpyHostToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(a.m, m, n * 8, cudaMemcpyHostToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(a.v, v, n * 8, cudaMemcpyHostToDevice, st));
            a.grads = g;
        }
        if (!ctx->adam_flag.p) {
            grow<unsigned int>(ctx->adam_flag, 1);
            SVR_CUDA(cudaMemsetAsync(ctx->adam_flag.p, 0, 4, st));
        }
        unsigned int* flag = ctx->adam_flag.as<unsigned int>();
        a.nan_flag = flag;
        if (on_device == 2) {  // deferred: the flag stays set until svr_ctx_take_adam_nan
            launch_adam(a, st);
            return;
        }
        SVR_CUDA(cudaMemsetAsync(flag, 0, 4, st));
        launch_adam(a, st);
        unsigned int hflag = 0;
        SVR_CUDA(cudaMemcpyAsync(&hflag, flag, 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaMemsetAsync(flag, 0, 4, st));  // reported here: not left for svr_ctx_take_adam_nan
        if (!on_device && n) {
            SVR_CUDA(cudaMemcpyAsync(params, a.params, n * 4, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemcpyAsync(m, a.m, n * 8, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemcpyAsync(v, a.v, n * 8, cudaMemcpyDeviceToHost, st));
        }
        SVR_CUDA(cudaStreamSynchronize(st));
        require(hflag == 0, SVR_ERR_RUNTIME, "adam_step: NaN gradient");
    });
}

int svr_train_step_l1(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
                      const svr_render_options* opts, const float* gt_device, svr_frame* f,
                      svr_gradients* grads, int accumulate, float* loss_device) {
    return guard([&] {
        require(opts && grads && grads->on_device, SVR_ERR_INVALID_ARGUMENT,
                "train step needs device gradient buffers");
        svr_render_options o = *opts;
        o.training = 1;
        render_impl(ctx, scene, cam, &o, f);
        const uint64_t n = uint64_t(f->W) * f->H * 3;
        float* dcol = grow<float>(f->l1_grad, n);
        launch_l1_loss(f->out_color, gt_device, n, dcol, loss_device, ctx->stream);
        svr_upstream up{};
        up.d_color = dcol;
        up.on_device = 1;
        backward_impl(ctx, scene, f, &up, grads, accumulate != 0);
    });
}

int svr_project_voxels(svr_ctx* ctx, const svr_camera* cam, uint64_t n, const double* centers,
                       const double* sizes, double near_plane, uint8_t* visible, double* aabb,
                       int32_t* rect) {
    return guard([&] {
        require(ctx && cam, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        if (n == 0) return;
        cudaStream_t st = ctx->stream;
        DevCamera dc = dev_camera(*cam);
        DevBuf b;
        b.reserve(n * (24 + 8 + 1 + 32 + 16) + 64);
        char* p = b.as<char>();
        double* dcen = reinterpret_cast<double*>(p);
        double* dsz = dcen + 3 * n;
        double* dab = dsz + n;
        int* drc = reinterpret_cast<int*>(dab + 4 * n);
        uint8_t* dvis = reinterpret_cast<uint8_t*>(drc + 4 * n);
        SVR_CUDA(cudaMemcpyAsync(dcen, centers, n * 24, cudaMemcpyHostToDevice, st));
        SVR_CUDA(cudaMemcpyAsync(dsz, sizes, n * 8, cudaMemcpyHostToDevice, st));
        launch_project_batch(dc, n, dcen, dsz, near_plane, dvis, dab, drc, st);
        SVR_CUDA(cudaMemcpyAsync(visible, dvis, n, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaMemcpyAsync(aabb, dab, n * 32, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaMemcpyAsync(rect, drc, n * 16, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
    });
}

int svr_tile_sign_masks(svr_ctx* ctx, const svr_camera* cam, uint8_t* masks, uint64_t n_tiles) {
    return guard([&] {
        require(ctx && cam && masks, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        DevCamera dc = dev_camera(*cam);
        require(n_tiles == uint64_t(dc.ntx) * dc.nty, SVR_ERR_INVALID_ARGUMENT,
                "tile count mismatch");
        if (!n_tiles) return;
        DevBuf b;
        b.reserve(n_tiles);
        launch_tile_masks_only(dc, b.as<uint8_t>(), ctx->stream);
        SVR_CUDA(cudaMemcpyAsync(masks, b.p, n_tiles, cudaMemcpyDeviceToHost, ctx->stream));
        SVR_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int svr_build_sort_entries(svr_ctx* ctx, const svr_camera* cam, uint64_t scene_voxel_count,
                           uint64_t n_pre, const uint32_t* vids, const uint64_t* codes,
                           const int32_t* rects, uint64_t* keys, uint32_t* values,
                           uint64_t capacity, uint64_t* n_out) {
    return guard([&] {
        require(ctx && cam && n_out, SVR_ERR_INVALID_ARGUMENT, "null argument");
        set_device(ctx);
        require(scene_voxel_count < (uint64_t(1) << 29), SVR_ERR_LENGTH,
                "voxel count exceeds the 29-bit id capacity");
        DevCamera dc = dev_camera(*cam);
        require(uint64_t(dc.ntx) * dc.nty < (uint64_t(1) << 16), SVR_ERR_LENGTH,
                "tile count exceeds the 16-bit id capacity");
        cudaStream_t st = ctx->stream;
        const int ntiles = dc.ntx * dc.nty;
        const uint64_t n = n_pre;
        DevBuf bm, bsat, bst, bv, bc, br, bcnt, boff, bk, bvals;
        uint8_t* masks = grow<uint8_t>(bm, ntiles);
        uint32_t* sat = grow<uint32_t>(bsat, uint64_t(dc.ntx + 1) * (dc.nty + 1));
        FrameStatus* status = grow<FrameStatus>(bst, 1);
        SVR_CUDA(cudaMemsetAsync(status, 0, sizeof(FrameStatus), st));
        launch_tile_setup(dc, masks, sat, status, st);
        uint32_t* dv = grow<uint32_t>(bv, n);
        uint64_t* dcode = grow<uint64_t>(bc, n);
        int4* drect = grow<int4>(br, n);
        uint32_t* cnt = grow<uint32_t>(bcnt, n);
        uint32_t* off = grow<uint32_t>(boff, n);
        if (n) {
            SVR_CUDA(cudaMemcpyAsync(dv, vids, n * 4, cudaMemcpyHostToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(dcode, codes, n * 8, cudaMemcpyHostToDevice, st));
            SVR_CUDA(cudaMemcpyAsync(drect, rects, n * 16, cudaMemcpyHostToDevice, st));
        }
        launch_entry_counts(dc, n, drect, sat, cnt, st);
        ctx->scratch.reserve(scan_scratch_bytes(n));
        exclusive_scan_u32(cnt, off, n, &status->n_entries, ctx->scratch.p, st);
        unsigned long long E = 0;
        SVR_CUDA(cudaMemcpyAsync(&E, &status->n_entries, 8, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
        *n_out = E;
        if (!keys) return;
        require(capacity >= E, SVR_ERR_INVALID_ARGUMENT, "entry buffer too small");
        uint64_t* dk = grow<uint64_t>(bk, E);
        uint32_t* dvv = grow<uint32_t>(bvals, E);
        launch_duplicate_list(dc, n, dv, dcode, drect, masks, off, dk, dvv, st);
        if (E) {
            SVR_CUDA(cudaMemcpyAsync(keys, dk, E * 8, cudaMemcpyDeviceToHost, st));
            SVR_CUDA(cudaMemcpyAsync(values, dvv, E * 4, cudaMemcpyDeviceToHost, st));
        }
        SVR_CUDA(cudaStreamSynchronize(st));
    });
}

int svr_sort_entries(svr_ctx* ctx, uint64_t n, uint64_t* keys, uint32_t* values) {
    return guard([&] {
        require(ctx, SVR_ERR_INVALID_ARGUMENT, "null context");
        set_device(ctx);
        if (n <= 1) return;
        // Only digits where some pair differs need a pass (stable LSD).
        uint64_t kx = 0;
        uint32_t vx = 0;
        for (uint64_t i = 1; i < n; ++i) {
            kx |= keys[i] ^ keys[0];
            vx |= values[i] ^ values[0];
        }
        RadixPass passes[kMaxRadixPasses];
        int np = 0;
        auto add_range = [&](int src, uint64_t diff) {
            if (!diff) return;
            int lo = __builtin_ctzll(diff), hi = 64 - __builtin_clzll(diff);
            for (int b = lo; b < hi; b += 8) passes[np++] = {src, b, std::min(8, hi - b)};
        };
        add_range(1, vx);
        add_range(0, kx);
        cudaStream_t st = ctx->stream;
        DevBuf k0, v0, k1, v1;
        uint64_t* dk0 = grow<uint64_t>(k0, n);
        uint32_t* dv0 = grow<uint32_t>(v0, n);
        uint64_t* dk1 = grow<uint64_t>(k1, n);
        uint32_t* dv1 = grow<uint32_t>(v1, n);
        SVR_CUDA(cudaMemcpyAsync(dk0, keys, n * 8, cudaMemcpyHostToDevice, st));
        SVR_CUDA(cudaMemcpyAsync(dv0, values, n * 4, cudaMemcpyHostToDevice, st));
        ctx->scratch2.reserve(sort_scratch_bytes(n, np));
        int r = radix_sort_pairs(dk0, dv0, dk1, dv1, n, passes, np, ctx->scratch2.p, st);
        SVR_CUDA(cudaMemcpyAsync(keys, r ? dk1 : dk0, n * 8, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaMemcpyAsync(values, r ? dv1 : dv0, n * 4, cudaMemcpyDeviceToHost, st));
        SVR_CUDA(cudaStreamSynchronize(st));
    });
}

void svr_free(void* p) { std::free(p); }

int svr_host_alloc(size_t bytes, void** out) {
    return guard([&] {
        require(out != nullptr, SVR_ERR_INVALID_ARGUMENT, "null argument");
        *out = nullptr;
        if (bytes) SVR_CUDA(cudaMallocHost(out, bytes));
    });
}

int svr_host_free(void* p) {
    return guard([&] {
        if (p) SVR_CUDA(cudaFreeHost(p));
    });
}

unsigned long long svr_launch_count(void) { return g_launches.load(); }

int svr_ctx_enable_timing(svr_ctx* ctx, int enable) {
    return guard([&] {
        require(ctx != nullptr, SVR_ERR_INVALID_ARGUMENT, "null context");
        collect_marks(ctx);
        ctx->timing = enable != 0;
    });
}

int svr_ctx_stage_times(svr_ctx* ctx, double* ms, int n, int reset) {
    return guard([&] {
        require(ctx != nullptr, SVR_ERR_INVALID_ARGUMENT, "null context");
        set_device(ctx);
        collect_marks(ctx);
        for (int i = 0; i < n && i < kNumStages; ++i) ms[i] = ctx->stage_ms[i];
        if (reset)
            for (double& v : ctx->stage_ms) v = 0.0;
    });
}

}  // extern "C"
