/*
 * svr_b200.h — C ABI of the B200-native sparse-voxel rasterizer.
 *
 * This is the drop-in boundary for the render and gradient path of the
 * reference C++ toolkit (`proj/include/svr/raster.hpp:52-141`,
 * `proj/src/raster.cpp`). Every entry point takes plain pointers and sizes;
 * no C++ or torch types cross it. The C++ API of the reference
 * (`svr::render`, `svr::render_with_pools`, `svr::render_backward`,
 * `svr::project_voxel`, `svr::tile_sign_patterns`, `svr::build_sort_entries`,
 * `svr::sort_entries`) is re-implemented on top of this ABI in
 * `paper_2412_04459_b200/cpp/raster_dropin.cpp`; see INTEGRATION.md.
 *
 * Errors: every function returns an svr_status. On failure a thread-local
 * message is available from svr_last_error(). The status codes map 1:1 onto
 * the exception types the reference throws:
 *   SVR_ERR_INVALID_ARGUMENT -> std::invalid_argument (raster.cpp:207-211,
 *                               octree.hpp:47-49/54-55/71-72)
 *   SVR_ERR_LENGTH           -> std::length_error     (raster.cpp:146-150)
 *   SVR_ERR_RUNTIME          -> std::runtime_error    (raster.cpp:329-332)
 * SVR_ERR_CUDA / SVR_ERR_NO_DEVICE have no reference counterpart (the
 * reference never touches a GPU); there is no CPU fallback.
 */
#ifndef SVR_B200_H
#define SVR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVR_ABI_VERSION 1

typedef enum svr_status {
    SVR_OK = 0,
    SVR_ERR_INVALID_ARGUMENT = 1,
    SVR_ERR_LENGTH = 2,
    SVR_ERR_RUNTIME = 3,
    SVR_ERR_CUDA = 4,
    SVR_ERR_NO_DEVICE = 5
} svr_status;

/* Limits of the reference (raster.hpp:18-20, scene.hpp:19, octree.hpp:16). */
#define SVR_TILE_SIZE 16
#define SVR_TILE_ID_BITS 16
#define SVR_VOXEL_ID_BITS 29
#define SVR_MAX_LEVEL 16

typedef struct svr_ctx svr_ctx;     /* one per (host thread, device): stream + arenas */
typedef struct svr_scene svr_scene; /* device-resident SparseScene                     */
typedef struct svr_frame svr_frame; /* device-resident per-view state (ForwardRecords) */

/* svr::Camera (camera.hpp:13-49). rot is the row-major camera-to-world
 * rotation, pos the camera centre. */
typedef struct svr_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double rot[9];
    double pos[3];
} svr_camera;

/* svr::RenderOptions (raster.hpp:22-31). */
typedef struct svr_render_options {
    int32_t K;              /* samples per voxel, 1..3            */
    double t_threshold;     /* early-termination transmittance    */
    double supersample;     /* >= 1                               */
    double background[3];
    double near_plane;
    double far_sentinel;
    int32_t record_stats;   /* per-voxel max blending weight      */
    int32_t training;       /* keep forward records for backward  */
} svr_render_options;

/* svr::SparseScene (scene.hpp:21-46), host arrays. */
typedef struct svr_scene_desc {
    uint64_t n_voxels;
    uint64_t n_pool;
    int32_t sh_degree;               /* 0..3                              */
    double bounds_center[3];
    double bounds_size;
    const uint64_t* codes;           /* OctPath.code, 48-bit left aligned */
    const uint8_t* levels;           /* OctPath.level, 1..16              */
    const uint32_t* corner_index;    /* [n_voxels][8]                     */
    const float* density;            /* [n_pool]                          */
    const float* sh;                 /* [n_voxels][3*(deg+1)^2]           */
} svr_scene_desc;

/* Per-view summary (one device->host read). */
typedef struct svr_frame_info {
    int32_t width, height;        /* target resolution            */
    int32_t ss_width, ss_height;  /* supersampled render grid     */
    int32_t tiles_x, tiles_y;
    uint64_t n_visible;           /* |pre| (raster.cpp:217)       */
    uint64_t n_entries;           /* E   (raster.cpp:218)         */
    uint64_t n_contribs;          /* training only                */
    int32_t sort_passes;          /* radix passes the sort ran    */
    int32_t training;
    int32_t composite_path;       /* 0 warp-autonomous, 1 CTA-cooperative K7 */
    int32_t reserved;
} svr_frame_info;

/* Buffers a frame exposes (svr_frame_download / svr_frame_device_ptr).
 * Images are row-major with interleaved channels, float32, exactly the
 * svr::Image layout (image.hpp:10-26) narrowed to f32. */
typedef enum svr_buffer {
    SVR_BUF_COLOR = 0,         /* W*H*3   f32                            */
    SVR_BUF_DEPTH = 1,         /* W*H     f32                            */
    SVR_BUF_MEDIAN_DEPTH = 2,  /* W*H     f32                            */
    SVR_BUF_NORMAL = 3,        /* W*H*3   f32                            */
    SVR_BUF_TRANSMITTANCE = 4, /* W*H     f32                            */
    SVR_BUF_MAX_BLEND = 5,     /* n_voxels f32 (record_stats)           */
    SVR_BUF_SS_COLOR = 6,      /* sw*sh*3 f32                            */
    SVR_BUF_SS_DEPTH = 7,      /* sw*sh   f32                            */
    SVR_BUF_SS_TFIN = 8,       /* sw*sh   f32                            */
    SVR_BUF_SORT_KEYS = 9,     /* E u64, sorted SortEntry::key           */
    SVR_BUF_SORT_VALUES = 10,  /* E u32, sorted SortEntry::value         */
    SVR_BUF_TILE_RANGES = 11,  /* tiles*2 u32, [lo,hi) per tile          */
    SVR_BUF_TILE_MASKS = 12,   /* tiles u8, bit s set iff pattern s used */
    SVR_BUF_VOXEL_RECTS = 13,  /* n_voxels*4 i32 (tx0,tx1,ty0,ty1); tx1<tx0 => culled */
    SVR_BUF_VOXEL_AABB = 14,   /* n_voxels*4 f64 (x0,x1,y0,y1), exact    */
    SVR_BUF_ENTRIES_KEYS = 15,   /* E u64 in emission order (debug mode) */
    SVR_BUF_ENTRIES_VALUES = 16, /* E u32 in emission order (debug mode) */
    SVR_BUF_PIX_COUNT = 17,    /* sw*sh u32 (training)                   */
    SVR_BUF_PIX_BEGIN = 18,    /* sw*sh u32 (training)                   */
    SVR_BUF_VOXEL_COLOR = 19,  /* n_voxels*3 f32 (visible voxels only)   */
    SVR_BUF_VOXEL_NORMAL = 20, /* n_voxels*3 f32 (visible voxels only)   */
    SVR_BUF_OUTPUTS = 21       /* W*H*9 f32: the five images above, contiguous
                                * in id order (COLOR, DEPTH, MEDIAN_DEPTH,
                                * NORMAL, TRANSMITTANCE): one copy per frame */
} svr_buffer;

/* ---- context ---------------------------------------------------------- */
const char* svr_last_error(void);
int svr_abi_version(void);
int svr_ctx_create(int device, svr_ctx** out);
int svr_ctx_destroy(svr_ctx* ctx);
/* cudaStream_t the context launches on (for event timing by the caller). */
void* svr_ctx_stream(svr_ctx* ctx);
int svr_ctx_synchronize(svr_ctx* ctx);
/* Deferred-E rendering for serving loops: svr_render no longer waits for the
 * entry count mid-frame (the frame is enqueued whole, so back-to-back renders
 * keep the GPU busy); the sort runs on a capacity learned from earlier
 * frames of the same svr_frame and reads the live count on the device. The
 * count is checked when a result is consumed (svr_frame_wait, download,
 * info, backward): a frame that outgrew its capacity is rendered again there
 * (and its asynchronous downloads repeated), so results are always those of
 * a complete frame. Training frames always take the synchronous path.
 * svr_ctx_overflow_count reports how many deferred frames outgrew theirs. */
int svr_ctx_set_async(svr_ctx* ctx, int on);
int svr_ctx_overflow_count(svr_ctx* ctx, uint32_t* out);
/* debug != 0 keeps the pre-sort entry list so it can be dumped bit-exactly. */
int svr_ctx_set_debug(svr_ctx* ctx, int debug);

/* ---- scene ------------------------------------------------------------ */
/* Validates levels/paths like to_voxel_index (octree.hpp:68-82) and uploads. */
int svr_scene_upload(svr_ctx* ctx, const svr_scene_desc* desc, svr_scene** out);
/* Refresh the parameter pools (PoolsD, raster.hpp:47-52) without touching
 * the geometry. on_device != 0: pointers are device pointers. Either may be
 * NULL to keep the current values. */
int svr_scene_set_params(svr_ctx* ctx, svr_scene* scene, const float* density, const float* sh,
                         int on_device);
int svr_scene_destroy(svr_scene* scene);
/* SVRX checkpoints (io.cpp:229-359, save_checkpoint / load_checkpoint): the
 * scene's CURRENT device parameters are written (training updates them in
 * place), and a file is loaded straight into a new device scene. The
 * container is byte-compatible with the reference's; the reader repeats its
 * checks (magic, CRC32, version, header, lengths, corner-key structure) with
 * its std::runtime_error conditions (SVR_ERR_RUNTIME) and the octree level
 * checks' std::invalid_argument (SVR_ERR_INVALID_ARGUMENT). */
int svr_scene_save_svrx(svr_ctx* ctx, const svr_scene* scene, const char* path);
/* Scene adaptation on the device (optim.cpp:207-298 + scene.cpp:8-26):
 * prune keeps the voxels with max_blend_weight >= threshold (n = n_voxels,
 * f32; on_device selects device/host), subdivide replaces each selected
 * voxel (host list, duplicates and level-16 voxels ignored) by its 8
 * children; both rebuild the corner indexing in the reference's
 * first-appearance pool order with its densities (fresh subdivision points:
 * mean of the parents' trilinear values, in double) and return a NEW scene,
 * whose AdaptRemap (voxel_src per voxel, pool_src per pool entry, -1 = new)
 * svr_scene_remap copies out. Errors: invalid_argument (stats size, voxel id
 * out of range), length_error (capacity 2^29). */
int svr_scene_prune(svr_ctx* ctx, const svr_scene* scene, const float* max_blend_weight, uint64_t n,
                    double threshold, int32_t on_device, svr_scene** out);
int svr_scene_subdivide(svr_ctx* ctx, const svr_scene* scene, const uint32_t* selected,
                        uint64_t n_selected, svr_scene** out);
int svr_scene_remap(const svr_scene* scene, int64_t* voxel_src, int64_t* pool_src);
/* Counts, degree and bounds of a device scene (array pointers left NULL). */
int svr_scene_info(const svr_scene* scene, svr_scene_desc* out);
/* Host copies of a device scene's arrays (any pointer may be NULL). */
int svr_scene_download(svr_ctx* ctx, const svr_scene* scene, uint64_t* codes, uint8_t* levels,
                       uint32_t* corner_index, float* density, float* sh);
int svr_scene_load_svrx(svr_ctx* ctx, const char* path, svr_scene** out);
/* Device pointers of the parameter pools (for optimisers living on device). */
int svr_scene_param_ptrs(svr_scene* scene, float** density, float** sh, uint64_t* n_pool,
                         uint64_t* n_sh);

/* ---- forward (raster.cpp:205-301) ------------------------------------- */
int svr_frame_create(svr_ctx* ctx, svr_frame** out);
int svr_frame_destroy(svr_frame* frame);
/* Renders `cam` into `frame` (buffers are reused across calls). Throws the
 * reference's invalid_argument / length_error conditions as status codes. */
int svr_render(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
               const svr_render_options* opts, svr_frame* frame);
int svr_frame_get_info(svr_frame* frame, svr_frame_info* out);
/* Copies a buffer to host memory (synchronous). bytes must match. */
int svr_frame_download(svr_frame* frame, svr_buffer which, void* dst, size_t bytes);
/* Pipelined variant for serving loops: enqueues the copy on the context's
 * copy stream behind the frame's pending work and returns at once. dst
 * (pinned host memory for a truly asynchronous copy) is complete after
 * svr_frame_wait(frame). A later render, backward or download through the
 * same frame waits for the copy on the device, so a caller alternating two
 * frames overlaps frame i's read-back with frame i+1's rendering. */
int svr_frame_download_async(svr_frame* frame, svr_buffer which, void* dst, size_t bytes);
/* Blocks until the frame's asynchronous downloads have landed. */
int svr_frame_wait(svr_frame* frame);
/* Page-locked host memory for svr_frame_download_async destinations (so the
 * copy runs at full PCIe rate and truly asynchronously); free with
 * svr_host_free. */
int svr_host_alloc(size_t bytes, void** out);
int svr_host_free(void* p);
/* Device pointer + size of a buffer (no copy, valid until the next render). */
int svr_frame_device_ptr(svr_frame* frame, svr_buffer which, void** ptr, size_t* bytes);

/* ForwardRecords materialisation (raster.hpp:72-82): visible voxel ids in
 * `pre` order, and per contribution the pre index plus the ray segment. */
int svr_frame_records(svr_frame* frame, uint32_t* pre_vids, uint64_t n_pre,
                      uint32_t* contrib_pre, double* contrib_a, double* contrib_b,
                      uint64_t n_contribs);

/* svr::PreVoxel (raster.hpp:55-64) with VoxelNormal (field.hpp:143-147). */
typedef struct svr_pre_voxel {
    uint32_t vid;
    int32_t degenerate;
    double center[3];
    double size;
    double V[8];
    double color[3];
    double normal[3];
    double raw[3];
    double x0, x1, y0, y1;
    int32_t tx0, tx1, ty0, ty1;
} svr_pre_voxel;

/* ForwardRecords::pre of a rendered frame: every visible voxel in vid order
 * (n = svr_frame_info.n_visible). Geometry and AABB are the exact fp64
 * values; colour and normal come from the fp32 preprocess. */
int svr_frame_pre(svr_frame* frame, svr_pre_voxel* out, uint64_t n);

/* render_oracle (raster.cpp:425-473): brute-force per-ray compositing of
 * every visible voxel in (entry distance, dir_dep_order) order, fp64, no
 * tiles and no supersampling. Fills the frame's five target-resolution
 * images. O(hits x voxels) per pixel: a test oracle for small scenes. */
int svr_render_oracle(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
                      const svr_render_options* opts, svr_frame* frame);

/* ---- backward (raster.cpp:303-423) ------------------------------------ */
typedef struct svr_upstream {
    const float* d_color;        /* W*H*3 or NULL   */
    const float* d_depth;        /* W*H   or NULL   */
    const float* d_normal;       /* W*H*3 or NULL   */
    const float* d_tfin_ss;      /* sw*sh or NULL   */
    const float* d_weight;       /* n_contribs or NULL  */
    const float* d_voxel_color;  /* n_contribs*3 or NULL */
    uint64_t n_d_weight;         /* element counts for the size checks */
    uint64_t n_d_voxel_color;    /* (in Vec3 units)                     */
    int32_t on_device;           /* pointers are device pointers        */
} svr_upstream;

typedef struct svr_gradients {
    float* density;   /* n_pool                */
    float* sh;        /* n_voxels*stride       */
    float* priority;  /* n_voxels              */
    int32_t on_device;
} svr_gradients;

int svr_render_backward(svr_ctx* ctx, const svr_scene* scene, svr_frame* frame,
                        const svr_upstream* up, svr_gradients* out);

/* ray_losses (losses.cpp:141-238) on the device, over the frame's forward
 * records (render with training = 1): transmittance entropy L_T, distortion
 * L_dist and per-voxel colour L_R. gt is the W*H*3 target image (f32); each
 * supersampled ray reads the gt pixel its footprint falls in. The weighted
 * gradients are ACCUMULATED (+=, like UpstreamGrads in the reference) into
 * d_tfin_ss (sw*sh), d_weight (n_contribs) and d_voxel_color (n_contribs*3),
 * which any of may be NULL when its weights are zero. All pointers are
 * device pointers when on_device, else host. Loss values (unweighted, as
 * RayLossValues) go to *out. */
typedef struct svr_ray_loss_weights {
    double w_T, w_dist, w_R;
} svr_ray_loss_weights;
typedef struct svr_ray_loss_values {
    double l_T, l_dist, l_R;
} svr_ray_loss_values;
int svr_ray_losses(svr_ctx* ctx, svr_frame* frame, const float* gt,
                   const svr_ray_loss_weights* weights, svr_ray_loss_values* out,
                   float* d_tfin_ss, float* d_weight, float* d_voxel_color, int32_t on_device);

/* mse_loss + ssim_loss (losses.cpp:71-139) of the frame's rendered colour
 * against gt (W*H*3 f32): out[0] = mean squared error, out[1] = 1 - mean
 * SSIM (11x11 Gaussian window, sigma 1.5, valid mode). d_color (W*H*3) is
 * ACCUMULATED with w_mse * dMSE/dC + w_ssim * d(1 - SSIM)/dC, as the
 * reference's mse_loss(.., w_mse, &d) and ssim_loss(.., w_ssim, &d) do;
 * NULL skips the gradients. Pointers are device pointers when on_device. */
int svr_image_losses(svr_ctx* ctx, svr_frame* frame, const float* gt, double w_mse,
                     double w_ssim, double* out, float* d_color, int32_t on_device);

/* adam_step (optim.cpp:322-345) over a float parameter pool on the device:
 * m, v are the fp64 moment buffers (AdamState, zero-initialised by the
 * caller), `step` the updated step count (state.step after ++), so
 * bc1 = 1 - beta1^step and bc2 = 1 - beta2^step are the reference's. The
 * per-element learning rate is lr, or lr_alt for elements with
 * (i % period) >= n_primary when period > 0 (the reference's SH rule:
 * period = stride, n_primary = 3). Double arithmetic in the reference's
 * order, so the float parameters match it bit for bit given the same
 * gradients. A NaN gradient returns SVR_ERR_RUNTIME (std::runtime_error).
 * All pointers are device pointers when on_device, else host. */
int svr_adam_step(svr_ctx* ctx, float* params, const float* grads, double* m, double* v,
                  uint64_t n, int64_t step, double lr, double lr_alt, uint32_t period,
                  uint32_t n_primary, double beta1, double beta2, double eps, int32_t on_device);

/* Deferred mode (on_device = 2) of svr_ray_losses, svr_image_losses and
 * svr_adam_step: device pointers, nothing is read back and the host does not
 * wait, so a whole training iteration is enqueued without a stall. The loss
 * values of the frame's last svr_image_losses / svr_ray_losses calls are then
 * read with svr_frame_loss_values (out[5] = mse, 1 - ssim, l_T, l_dist, l_R),
 * and a NaN gradient seen by any deferred Adam step since the last check is
 * reported by svr_ctx_take_adam_nan (which clears it). */
int svr_frame_loss_values(svr_frame* frame, double* out);
int svr_ctx_take_adam_nan(svr_ctx* ctx, int32_t* nan_seen);

/* L1 photometric loss on the rendered colour (new; pattern of mse_loss,
 * losses.cpp:121-131): L = mean|C-gt|, dL/dC = sign(C-gt)/(3WH). gt is a
 * device pointer (W*H*3 f32); d_color (device, W*H*3) receives the gradient;
 * loss (device, 1 f32) may be NULL. */
int svr_l1_loss(svr_ctx* ctx, svr_frame* frame, const float* gt, float* d_color, float* loss);

/* One view of the training step: forward(training) -> L1 -> backward,
 * accumulating into device gradient buffers (not cleared when accumulate). */
int svr_train_step_l1(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cam,
                      const svr_render_options* opts, const float* gt_device, svr_frame* frame,
                      svr_gradients* grads, int accumulate, float* loss_device);

/* ---- multi-GPU training step ------------------------------
 * One process per GPU. Rank 0 makes a unique id (svr_comm_unique_id), the
 * caller hands it to every rank by its own means, each rank creates its
 * communicator on its context. svr_train_batch_l1 runs forward -> L1 ->
 * backward over the rank's views (svr_train_step_l1, accumulating into the
 * device gradients; an empty batch contributes zeros), sums the per-view L1
 * losses into *loss_device and, when comm spans more than one rank,
 * all-reduces [density | SH | priority] in place over NCCL (buckets of
 * 64 MiB in one group) on the context stream, then polls NCCL's asynchronous
 * error state. NCCL (libnccl.so.2) is loaded at first use. */
typedef struct svr_comm svr_comm;
int svr_comm_unique_id(uint8_t id[128]);
int svr_comm_create(svr_ctx* ctx, const uint8_t id[128], int rank, int world, svr_comm** out);
int svr_comm_destroy(svr_comm* comm);
/* Registers a device buffer (e.g. the gradients) with the communicator, so
 * NCCL may use NVLS in-switch reduction / zero-copy paths on it. */
int svr_comm_register(svr_comm* comm, void* ptr, size_t bytes);
/* SVR_ERR_RUNTIME (communicator aborted) after an asynchronous NCCL error. */
int svr_comm_check(svr_comm* comm);
int svr_comm_allreduce_gradients(svr_comm* comm, svr_gradients* grads, uint64_t n_pool,
                                 uint64_t n_sh, uint64_t n_vox);
int svr_train_batch_l1(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cams,
                       const float* const* gts_device, int n_views,
                       const svr_render_options* opts, svr_frame* frame, svr_gradients* grads,
                       svr_comm* comm, float* loss_device);

/* ---- pipeline pieces (raster.hpp:115-127), batch form, host buffers ---- */
/* project_voxel (raster.cpp:72-118) for n voxels. visible[i] is 0/1; aabb is
 * (x0,x1,y0,y1) and rect (tx0,tx1,ty0,ty1) per voxel. */
int svr_project_voxels(svr_ctx* ctx, const svr_camera* cam, uint64_t n, const double* centers,
                       const double* sizes, double near_plane, uint8_t* visible, double* aabb,
                       int32_t* rect);
/* tile_sign_patterns (raster.cpp:120-142) for every tile: bitmask per tile. */
int svr_tile_sign_masks(svr_ctx* ctx, const svr_camera* cam, uint8_t* masks, uint64_t n_tiles);
/* build_sort_entries (raster.cpp:144-172): `pre` given as voxel ids, their
 * paths and tile rects. Two-phase: call with keys==NULL to get *n_out. */
int svr_build_sort_entries(svr_ctx* ctx, const svr_camera* cam, uint64_t scene_voxel_count,
                           uint64_t n_pre, const uint32_t* vids, const uint64_t* codes,
                           const int32_t* rects, uint64_t* keys, uint32_t* values,
                           uint64_t capacity, uint64_t* n_out);
/* sort_entries (raster.cpp:174-178): ascending (key, value), in place. */
int svr_sort_entries(svr_ctx* ctx, uint64_t n, uint64_t* keys, uint32_t* values);

/* ---- synthetic fixtures (host utility, not on the render path) -------- */
/* Generator G of SURVEY §8(d): level-3 dense grid, random subdivision to
 * <= max_level until the next split would exceed target, densities
 * U(-4,2.5), SH from the pattern of tests/test_raster.cpp:15-37. Writes
 * host arrays allocated by the library (free with svr_free). */
int svr_synth_random_scene(uint64_t seed, uint64_t target, int max_level, int sh_degree,
                           uint64_t* n_voxels, uint64_t* n_pool, uint64_t** codes,
                           uint8_t** levels, uint32_t** corner_index, float** density,
                           float** sh);
/* init_unbounded (optim.cpp:96-184) for cameras cams[0..n_cams): observed
 * main block at level shell_levels+init_level, coarser shells refined by
 * max sampling rate until bg/fg >= bg_ratio; then the pool is built as
 * rebuild_corner_indexing and parameters drawn as generator G from a fresh
 * mt19937_64(seed) (densities U(-4,2.5), SH as tests/test_raster.cpp:29-37).
 * Also returns the scene bounds (centre, size). Same ownership as above. */
int svr_synth_unbounded_scene(const svr_camera* cams, int n_cams, int init_level,
                              int shell_levels, double bg_ratio, uint64_t seed, int sh_degree,
                              uint64_t* n_voxels, uint64_t* n_pool, uint64_t** codes,
                              uint8_t** levels, uint32_t** corner_index, float** density,
                              float** sh, double* bounds_center, double* bounds_size);
/* ring_cameras (synth.cpp:89-118), camera i of n. */
int svr_ring_camera(int n_views, int index, int width, int height, double distance,
                    double fov_x_deg, svr_camera* out);
void svr_free(void* p);

/* ---- instrumentation ---------------------------------------------------- */
/* Number of kernels this library has launched (process-wide). */
unsigned long long svr_launch_count(void);
/* Per-stage CUDA-event timing on the context stream. Stage order:
 * tile_setup, preprocess, scan, duplicate, sort, ranges, composite,
 * record, downsample, backward, epilogue, other. */
int svr_ctx_enable_timing(svr_ctx* ctx, int enable);
int svr_ctx_stage_times(svr_ctx* ctx, double* ms, int n, int reset);

#ifdef __cplusplus
}
#endif
#endif /* SVR_B200_H */
