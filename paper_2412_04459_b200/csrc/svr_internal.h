// svr_internal.h — host-side objects behind the C ABI (include/svr_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "svr_b200.h"
#include "svr_kernels.h"
#include "svr_math.cuh"

namespace svrb {

// Errors carry the svr_status they map to (and thereby the reference
// exception type the C++ drop-in rethrows).
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void cuda_check(cudaError_t e, const char* what);
void count_launch();

// Frame kernels are launched with programmatic stream serialisation
// (svr_math.cuh: pdl_enter); SVR_PDL=0 turns it off.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...), "cudaLaunchKernelEx");
}
#define SVR_CUDA(x) ::svrb::cuda_check((x), #x)

// Function attributes (the dynamic shared-memory opt-in) are per device:
// true the first time the current device asks through `flags` (one bit per
// device ordinal; concurrent first calls may both see true, and setting an
// attribute twice is harmless).
inline bool first_on_device(std::atomic<uint64_t>& flags) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const uint64_t bit = uint64_t(1) << (dev & 63);
    return (flags.fetch_or(bit) & bit) == 0;
}
#define SVR_LAUNCH(what) (::svrb::count_launch(), ::svrb::cuda_check(cudaGetLastError(), what))

// Stages timed by svr_ctx_stage_times (CUDA events on the context stream).
enum Stage {
    kStageTileSetup = 0,
    kStagePreprocess,
    kStageScan,
    kStageDuplicate,
    kStageSort,
    kStageRanges,
    kStageComposite,
    kStageRecord,
    kStageDownsample,
    kStageBackward,
    kStageEpilogue,
    kStageOther,
    kNumStages
};

// Grow-only device allocation; contents are not preserved across growth.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    void release();
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// Pinned host staging buffer, grow-only.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    ~HostBuf();
};

// adapt.cu: prune / subdivide_voxels on the device (flags: keep / selected).
svr_scene* adapt_scene(svr_ctx* ctx, const svr_scene* old, const uint32_t* flags, bool subdivide,
                       float fill);
void launch_keep_flags(const float* stat, uint64_t n, double thr, uint32_t* keep, cudaStream_t st);

}  // namespace svrb

struct svr_ctx {
    int device = 0;
    bool timing = false;
    std::vector<std::pair<int, cudaEvent_t>> marks;  // stage starting at each event
    std::vector<cudaEvent_t> event_pool;
    double stage_ms[svrb::kNumStages] = {};
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // svr_frame_download_async
    int num_sms = 148;
    bool debug = false;
    svrb::DevBuf scratch;   // sort/scan temporaries
    svrb::DevBuf scratch2;
    svrb::HostBuf pinned;   // small readbacks (mapped: written by status_to_host_kernel)
    svrb::DevBuf adam_flag; // svr_adam_step NaN flag
    bool async_frames = false;  // svr_ctx_set_async: renders skip the mid-frame E read-back
    svrb::DevBuf overflow_count;  // deferred frames whose E outgrew their capacity
    // device gradients of a host-buffer svr_render_backward, kept between
    // calls (config 2: 215 MB that would otherwise be allocated per call)
    svrb::DevBuf bwd_density, bwd_sh, bwd_priority;
    svrb::DevBuf batch_losses;  // per-view L1 losses of svr_train_batch_l1
};

struct svr_scene {
    uint64_t n_voxels = 0, n_pool = 0;
    int sh_degree = 3, sh_stride = 48;
    int max_level = 1;
    double bounds_center[3] = {0, 0, 0};
    double bounds_size = 1.0;
    svrb::DevBuf paths;         // u64: code | level << 48
    svrb::DevBuf corner_index;  // u32 [n][8]
    svrb::DevBuf density;       // f32 [n_pool]
    svrb::DevBuf sh;            // f32 [n][stride]
    svrb::DevBuf morton_rank;   // u32 [8][n]: build_morton_rank (sort keys)
    svrb::DevBuf morton_order;  // u32 [8n]: the (s, vid) pairs in rank order
    bool unordered = false;     // voxels not in spatial order: K1 runs pre-cull + worklist
    uint64_t param_version = 0; // bumped by svr_scene_set_params
    int rank_bits = 0;          // bit width of 8n-1; 0 = no table
    // AdaptRemap of a scene produced by svr_scene_prune / svr_scene_subdivide
    svrb::DevBuf voxel_src, pool_src;  // int64 per voxel / per pool entry
    bool has_remap = false;
};

// Per-view state. Also the device half of svr::ForwardRecords.
struct svr_frame {
    svr_ctx* ctx = nullptr;
    const svr_scene* scene = nullptr;
    svr_render_options opts{};
    svrb::DevCamera cam{};     // supersampled camera actually rendered with
    svr_camera ss_cam{};       // same, ABI form
    int W = 0, H = 0, sw = 0, sh = 0, ntx = 0, nty = 0;
    uint64_t n_voxels = 0;
    uint64_t n_visible = 0, n_entries = 0, n_contribs = 0;
    int sort_passes = 0;
    int composite_path = 0;  // 1: the last render composited CTA-cooperatively
    bool training = false;
    bool has_records = false;
    uint64_t param_version = 0;  // the scene's parameter version when rendered
    // huge-pair merge (raster.cu: HugePairs): last frame's count of huge pairs
    // (the hint that turns the merge on) and its buffers
    uint32_t huge_hint = 0;
    bool huge_used = false;
    svrb::DevBuf huge_keys, huge_vals, huge_scratch, huge_diff, huge_total, huge_pack, huge_apos,
        ranges_small;

    svrb::DevBuf tile_masks, tile_sat, rects, aabb, records, counts, offsets, visible_rank;
    svrb::DevBuf keys[2], vals[2], dbg_keys, dbg_vals, ranges, tile_order, big;
    svrb::DevBuf pair_counts, big_pairs, rowspan;  // rank-ordered duplicate
    svrb::DevBuf work;                             // K1 worklist (unordered scenes)
    svrb::DevBuf vis_list;                         // K1's visible voxels (training frames)
    uint64_t n_vis_list = 0;                       // its length (read with E)
    bool sort_keys_kept = true;  // false: the last sort pass wrote values only
    // the five output images, one allocation in svr_buffer id order (so
    // SVR_BUF_OUTPUTS reads them back with one copy); set by alloc_outputs
    svrb::DevBuf out_all, max_blend;
    float *out_color = nullptr, *out_depth = nullptr, *out_median = nullptr, *out_normal = nullptr,
          *out_tfin = nullptr;
    void alloc_outputs(uint64_t npx) {
        out_all.reserve(npx * 9 * sizeof(float));
        float* b = out_all.as<float>();
        out_color = b;
        out_depth = b + 3 * npx;
        out_median = b + 4 * npx;
        out_normal = b + 5 * npx;
        out_tfin = b + 8 * npx;
    }
    svrb::DevBuf ss_color, ss_depth, ss_median, ss_normal, ss_tfin;
    svrb::DevBuf pix_count, pix_begin, contrib_entry, contrib_T;
    svrb::DevBuf stage_entry, stage_T;  // single-pass training records
    svrb::DevBuf view_dir;              // training: K1's sh_eval directions
    svrb::DevBuf rl_sums, rl_scratch;   // svr_ray_losses
    double rl_w[3] = {0.0, 0.0, 0.0};   // weights of the last ray-loss call (value masking)
    double il_norm[2] = {1.0, 1.0};     // normalisers of the last image-loss call
    bool rl_pending = false, il_pending = false;
    svrb::DevBuf il_mid, il_maps, il_adj, il_sums;  // svr_image_losses
    uint32_t stage_cap = 64;            // per-pixel capacity, doubles on overflow
    bool staged = false;                // records live in stage_* ...
    bool compact_valid = false;         // ... and contrib_* is (not yet) built
    svrb::DevBuf taps;  // resampler tables
    svrb::DevBuf bwd_gc, bwd_gn, bwd_lift, bwd_dcolor, status, l1_grad;  // bwd_gc: K9 per-voxel records
    bool gvox_clean = false;  // bwd_gc all zero (the last backward's epilogue ran)
    int sorted_buf = 0;  // which of keys[]/vals[] holds the sorted list
    int vals_buf = 0;    // which vals[] the compositing kernels read
    bool packed = false; // entries in the packed 64-bit format (PackedFormat)
    svrb::PackedFormat fmt{};
    svrb::DevBuf ref_keys, ref_vals;  // reference-format dumps of packed entries
    int tap_src_w = -1, tap_src_h = -1, tap_dst_w = -1, tap_dst_h = -1;
    int n_taps_x = 0, n_taps_y = 0;
    // asynchronous read-back (svr_frame_download_async)
    cudaEvent_t ready = nullptr;   // main stream reached the copy point
    cudaEvent_t copied = nullptr;  // copy stream finished the downloads
    bool copy_pending = false;
    // deferred-E rendering (svr_ctx_set_async): the entry count is read back
    // only when a result is consumed (svr_frame_wait / download / info)
    svrb::HostBuf hstatus;        // mapped FrameStatus of this frame
    uint64_t e_cap = 0;           // entry capacity a deferred render may use
    bool e_pending = false;       // hstatus not yet checked against e_cap
    cudaEvent_t done = nullptr;   // end of the last deferred render
    svr_camera req_cam{};         // the request, for a re-render on overflow
    svr_render_options req_opts{};
    struct PendingDownload {
        svr_buffer which;
        void* dst;
        size_t bytes;
    };
    std::vector<PendingDownload> pending_dl;  // async downloads since the last wait
};
