// svr_kernels.h — host launchers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "svr_math.cuh"

namespace svrb {

// ---- scan.cu ---------------------------------------------------------------
// Exclusive prefix sum of n u32 values; writes the u64 grand total to
// *total (device). `scratch` must hold scan_scratch_bytes(n).
size_t scan_scratch_bytes(uint64_t n);
// The first two phases only: u32 scratch[b] = exclusive prefix of block b's
// kScanChunk inputs (for kernels that fuse the apply phase, kScanThreads
// threads x 8 consecutive items per block).
constexpr int kScanThreads = 512;
constexpr int kScanChunk = 4096;
void scan_block_prefixes(const uint32_t* in, uint64_t n, unsigned long long* total, void* scratch,
                         cudaStream_t st);
// The second phase alone, over block sums the caller accumulated (u32
// partial[b] = sum of block b's inputs): in place to exclusive prefixes.
void scan_block_sums(uint32_t* partial, uint64_t nb, unsigned long long* total, cudaStream_t st);
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, unsigned long long* total,
                        void* scratch, cudaStream_t st);

// ---- sort.cu ---------------------------------------------------------------
// One LSD digit: bits [shift, shift+bits) of the key (src 0) or value (src 1).
struct RadixPass {
    int src;
    int shift;
    int bits;  // 1..8
};
constexpr int kMaxRadixPasses = 16;
size_t sort_scratch_bytes(uint64_t n, int npasses);
// Stable LSD onesweep sort of (key, value) pairs over the given digits.
// Ping-pongs between buffer 0 and 1; returns the index holding the result.
int radix_sort_pairs(uint64_t* keys0, uint32_t* vals0, uint64_t* keys1, uint32_t* vals1,
                     uint64_t n, const RadixPass* passes, int npasses, void* scratch,
                     cudaStream_t st);
// Keys-only variant. With hist_ready the digit histograms were already
// accumulated into sort_hist_ptr(scratch) (after sort_prepare) by the
// producer of the keys (the fused duplicate kernel).
struct RadixPlan {
    int n;
    RadixPass p[kMaxRadixPasses];
};
uint32_t* sort_hist_ptr(void* scratch);
void sort_prepare(void* scratch, uint64_t n, int npasses, cudaStream_t st);
// n_dev (optional): the live count on the device (<= n, the capacity the
// launch grids are sized for); partitions past it exit at once.
// fin (optional): the last pass writes, instead of keys, the reference value
// (s << 29 | vid) of each packed key (vid = low fin->vb bits, s the next 3)
// into fin->vals, and the tile ranges (tile = key >> fin->tile_shift) into
// fin->ranges from the ends of each partition's tile runs; tiles without
// entries are left with lo > hi (launch_tile_order turns them into [0, 0)).
// The sorted keys are then never written and the range kernel's pass over
// them is gone.
struct SortFinish {
    uint32_t* vals;
    uint2* ranges;
    int vb, tile_shift, ntiles;
};
int radix_sort_keys(uint64_t* keys0, uint64_t* keys1, uint64_t n, const RadixPass* passes,
                    int npasses, void* scratch, cudaStream_t st, bool hist_ready,
                    const unsigned long long* n_dev = nullptr, const SortFinish* fin = nullptr);

// ---- raster.cu -------------------------------------------------------------
struct FrameStatus {          // device -> host summary, one read per frame
    unsigned long long n_entries;
    unsigned int pattern_or;  // OR of all tile sign masks
    unsigned int overflow;    // a pixel exceeded the staged-record capacity
    unsigned long long n_contribs;
    unsigned int n_big;       // voxels handed to the cooperative duplicate
    unsigned int n_big_ranked;  // the same for the rank-ordered duplicate
    unsigned int n_work;        // K1 worklist length (pre-cull pass)
    unsigned int n_vis_list;    // K1's list of visible voxels (training frames)
    unsigned long long n_entries_voxel;  // E from the per-voxel scan (parity dumps of the ranked path)
    unsigned int n_huge_pairs;           // pairs with >= HugePairs::min entries (all of them counted)
    unsigned long long n_huge_entries;   // entries of the pairs diverted to the per-tile merge
};

// Huge (sign pattern, voxel) pairs — a large voxel near a camera inside the
// scene covers hundreds of tiles (config 4: 22K voxels hold 91M of 94M
// entries). With `divert`, pair_counts lists them (rank, value) instead of
// giving them entries to duplicate and sort; after the sort of the other
// entries, merge_huge_kernel interleaves them into every tile's list in rank
// order, producing exactly the sorted values and tile ranges the full sort
// would (raster.cpp:144-178, 238-245).
struct HugePairs {
    uint32_t min;       // entry count from which a pair is huge (0: off)
    int divert;         // list them (else only count them: the next frame's hint)
    uint32_t cap;       // list capacity; pairs past it take the ordinary path
    uint64_t* keys;     // [cap] rank, UINT64_MAX padding
    uint32_t* vals;     // [cap] s << 29 | vid
};

// With rowspan (int2 [8][nty]): also the eight per-sign-pattern SATs at
// sat + (1 + s) * ncell (ncell = (ntx + 1) * (nty + 1)) and each pattern's
// per-row tile run, for the rank-ordered duplicate.
void launch_tile_setup(const DevCamera& cam, uint8_t* masks, uint32_t* sat, FrameStatus* status,
                       cudaStream_t st, int2* rowspan = nullptr);
// Copies the device FrameStatus into host-mapped pinned memory with a kernel.
// With overflow_count: counts frames whose entry total exceeded `cap`.
void launch_status_to_host(const FrameStatus* d, FrameStatus* h, cudaStream_t st,
                           uint64_t cap = ~uint64_t(0), unsigned int* overflow_count = nullptr);

struct PreprocessArgs {
    uint64_t n;
    const uint64_t* paths;
    const uint32_t* corner_index;
    const float* density;
    const float* sh;
    int sh_degree, sh_stride;
    double bc[3];
    double bsize;
    double near_plane;
    const uint32_t* tile_sat;
    int4* rects;
    double4* aabb;  // optional
    float4* records;
    uint32_t* counts;
    float4* view_dir;  // optional (training): unit sh_eval direction per visible voxel
    const uint32_t* order;  // optional: voxel worklist (filled by the pre-cull pass, n voxels of room)
    const unsigned int* n_order;  // with order: its live length on the device (zeroed by the caller)
    uint32_t* vis_list;           // optional: visible voxels appended here (n_vis_list counts them)
    unsigned int* n_vis_list;
    CullNorms cull;               // set by launch_preprocess (cull_norms of the camera)
};
void launch_preprocess(const DevCamera& cam, const PreprocessArgs& a, cudaStream_t st);

void launch_duplicate(const DevCamera& cam, uint64_t n, const uint64_t* paths, const int4* rects,
                      const uint8_t* masks, const uint32_t* counts, const uint32_t* offsets,
                      uint64_t* keys, uint32_t* vals, cudaStream_t st);

void launch_tile_ranges(const uint64_t* keys, uint64_t n, uint2* ranges, int ntiles,
                        cudaStream_t st);

// Packed entry format (when it fits in 64 bits):
//   tile | top 3*Lmax order bits | sign s (3) | vid (vb bits)
// Sorting it keys-only reproduces the reference's (key, value) order.
struct PackedFormat {
    int vb;          // voxel-id bits
    int lmax;        // finest occupied octree level
    int tile_shift;  // vb + 3 + order bits
    int rank_bits;   // >0: order = Morton rank of (s, vid) (scene table); 0: code ^ s*G bits
};
void launch_duplicate_packed(const DevCamera& cam, uint64_t n, const uint64_t* paths,
                             const int4* rects, const uint8_t* masks, const uint32_t* counts,
                             const uint32_t* offsets, PackedFormat fmt, const uint32_t* rank,
                             uint64_t* keys, const uint32_t* tile_sat, uint32_t* big,
                             unsigned int* n_big, cudaStream_t st, uint64_t cap = ~uint64_t(0));
// Direction-aware Morton rank table of a scene: rank[s*n + vid] = position of
// (code_vid ^ s*kGroupOnes, s << 29 | vid) in the ascending order of all 8n
// such pairs, i.e. the reference's within-tile (key, value) order
// (raster.cpp:163-177) as one dense integer. Camera independent.
size_t morton_rank_scratch_bytes(uint64_t n, int lmax);
void build_morton_rank(const uint64_t* paths, uint64_t n, int lmax, uint32_t* rank, uint32_t* order,
                       void* scratch, cudaStream_t st);
// Rank-ordered K4 (needs the per-pattern SATs of launch_tile_setup
// per_pattern, the rank table and the scene's pair list order[r] =
// s << 29 | vid). K4a: pc[rank[s*n + v]] = entries of pair (s, v), 8n u32,
// zeroed here. scan_block_prefixes(pc) -> block prefixes in `partial`. K4b:
// the apply phase of that scan, fused with emission: pair r's entries land
// at its rank-order offset with key tile | r | s | vid, so the keys come out
// sorted below the tile bits. big: E / 128 + 1 uint2 (pairs with more than
// 128 entries, emitted cooperatively).
void launch_pair_counts(const DevCamera& cam, uint64_t n, const uint32_t* counts, const int4* rects,
                        const uint32_t* sat, FrameStatus* status, const uint32_t* rank,
                        uint32_t* pc, uint32_t* block_sums, cudaStream_t st, const HugePairs& huge);
// The huge-pair merge: tile coverage counts of the (rank-sorted) huge list
// and the final tile ranges (small + huge per tile, scanned), then per tile
// the rank-order merge of its small sorted keys with the huge pairs covering
// it into `vals`. diff: int [8][(ntx+1)(nty+1)] scratch; n_total: E.
// huge_*_sorted: the list in rank order; *_s: the same in (pattern, rank)
// order; packed: 2 * cap uint4 + 16 words.
void launch_merge_huge(const DevCamera& cam, const HugePairs& huge, const uint64_t* huge_keys_sorted,
                       const uint32_t* huge_vals_sorted, const uint64_t* skeys_s, const uint32_t* svals_s,
                       const FrameStatus* status,
                       const int4* rects, const uint8_t* masks, const uint64_t* small_keys,
                       const uint2* small_ranges, PackedFormat fmt, int* diff, uint4* packed,
                       uint32_t* apos, uint2* ranges, uint32_t* vals, uint64_t cap,
                       unsigned long long* n_total, cudaStream_t st);
#ifndef SVR_RBIG
#define SVR_RBIG 128
#endif
constexpr uint32_t kRankedBigMin = SVR_RBIG;  // pairs with more entries: one warp each
// Optional: K4 also counts the tile-only sort's digit histograms (the keys'
// tile id t: digit 0 = t & m0, digit 1 = (t >> b0) & m1 when two) into
// hist[2][256] (sort_hist_ptr, after sort_prepare), so the sort skips its
// histogram read of the keys.
struct TileDigits {
    uint32_t* hist;
    uint32_t m0, m1;
    int b0;
    int two;
};
void launch_duplicate_ranked(const DevCamera& cam, uint64_t n, const uint32_t* pc,
                             const uint32_t* partial, const uint32_t* order, const int4* rects,
                             const uint8_t* masks, const uint32_t* sat, const int2* rowspan,
                             PackedFormat fmt, uint64_t* keys, uint64_t cap, uint2* big,
                             unsigned int* n_big, cudaStream_t st, TileDigits td = TileDigits{});
// Tile ranges from packed sorted keys; also writes the reference value
// (s << 29 | vid) per entry for the compositing kernels.
void launch_tile_ranges_packed(const uint64_t* keys, uint64_t n, PackedFormat fmt, uint2* ranges,
                               uint32_t* vals, int ntiles, cudaStream_t st,
                               const unsigned long long* n_dev = nullptr);
// Reference SortEntry (key, value) from packed keys (parity dumps).
void launch_unpack_entries(const uint64_t* packed, uint64_t n, PackedFormat fmt,
                           const uint64_t* paths, uint64_t* keys, uint32_t* vals, cudaStream_t st);

struct CompositeArgs {
    const uint2* ranges;
    const uint32_t* tile_order;  // optional LPT tile schedule
    const uint32_t* vals;
    const float4* records;
    int K;
    float t_threshold;
    float bg[3];
    float far_sentinel;
    float* color;   // sw*sh*3
    float* depth;
    float* median;
    float* normal;
    float* tfin;
    uint32_t* pix_count;        // tile-major [ntiles*256], optional
    unsigned int* max_blend;    // per voxel, optional (float bits)
    // record pass
    const uint32_t* pix_begin;  // tile-major
    uint32_t* contrib_entry;
    float* contrib_T;
    // single-pass training records: contribution k of pixel slot s goes to
    // stage_*[k * stage_stride + s] while k < stage_cap, else *overflow = 1
    uint32_t* stage_entry;
    float* stage_T;
    uint32_t stage_cap, stage_stride;
    unsigned int* overflow;
};
// Staged -> compact (reference order) contribution records.
void launch_compact_contribs(const uint32_t* pix_count, const uint32_t* pix_begin,
                             const uint32_t* stage_entry, const float* stage_T, uint32_t stride,
                             uint32_t* contrib_entry, float* contrib_T, cudaStream_t st);
void launch_composite(const DevCamera& cam, const CompositeArgs& a, bool record_pass, bool coop,
                      cudaStream_t st);
void launch_tile_order(uint2* ranges, int ntiles, uint32_t* order, cudaStream_t st);

// Area resampler (image.cpp:9-45): CSR taps per destination index.
struct TapTable {
    const int* ptr_x;  // dst_w+1
    const int* idx_x;
    const float* w_x;
    const int* ptr_y;  // dst_h+1
    const int* idx_y;
    const float* w_y;
};
// Downsamples `nch` interleaved channel images src (sw x sh) -> dst (W x H).
void launch_downsample(const TapTable& t, const float* src, int channels, int sw, float* dst,
                       int W, int H, cudaStream_t st);

// Gathers tile-major per-pixel values into row-major image order.
void launch_tile_to_image_u32(const uint32_t* tm, uint32_t* img, int sw, int sh, int ntx,
                              cudaStream_t st);

// Visible rank (pre index) per voxel: 1 where rect is non-empty.
void launch_visible_flags(const int4* rects, uint64_t n, uint32_t* flags, cudaStream_t st);

// Contribution segments (a, b) in double for ForwardRecords materialisation.
void launch_contrib_segments(const DevCamera& cam, const uint2* ranges, const uint32_t* vals,
                             const float4* records, const uint32_t* pix_count,
                             const uint32_t* pix_begin, const uint32_t* contrib_entry,
                             const uint32_t* pre_rank, uint32_t* contrib_pre, double* a,
                             double* b, int ntiles, cudaStream_t st);

// ---- backward.cu -----------------------------------------------------------
// Adjoint of the area resampler (image.cpp:47-60); transposed CSR taps.
void launch_lift(const TapTable& transposed, const float* g, int channels, int W, float* out,
                 int sw, int sh, cudaStream_t st);

void launch_l1_loss(const float* color, const float* gt, uint64_t n, float* d_color, float* loss,
                    cudaStream_t st);

// ray_losses (losses.cpp:141-238) over device forward records.
struct RayLossArgs {
    const uint2* ranges;
    const uint32_t* vals;
    const float4* records;
    int K;
    const uint32_t* pix_count;      // tile-major
    const uint32_t* pix_begin;
    const uint32_t* contrib_entry;  // compact, or staged when stage_stride > 0
    const float* contrib_T;
    uint32_t stage_stride;
    const float* tfin;              // ss image, row-major (sw*sh)
    const float* gt;                // W*H*3
    int gt_w, gt_h;
    double w_T, w_dist, w_R;
    float* d_tfin_ss;               // sw*sh, +=
    float* d_weight;                // n_contribs, +=
    float* d_voxel_color;           // n_contribs*3, +=
    float2* scratch;                // n_contribs: (w, m) per contribution
    double* sums;                   // 3: l_T, l_dist, l_R (+=)
};
void launch_ray_losses(const DevCamera& cam, const RayLossArgs& a, cudaStream_t st);

// mse_loss + ssim_loss (losses.cpp:71-139) on W x H x 3 images.
struct ImageLossArgs {
    const float* a;   // rendered colour
    const float* b;   // ground truth
    int W, H;
    float kern[11];   // gauss_kernel (losses.cpp:15-29), normalised in double
    double w_mse, w_ssim;
    float* d_a;       // W*H*3, += (may be null)
    float* mid;       // scratch: 5 x (W-10) x H x 3
    float* maps;      // scratch: 3 x (W-10) x (H-10) x 3 (u1, u2, u3), then reused
    float* adj;       // scratch: 3 x (W-10) x H x 3
    double* sums;     // [0] sum of squared errors, [1] sum of the SSIM map
};
void launch_image_losses(const ImageLossArgs& a, cudaStream_t st);

// adam_step (optim.cpp:322-345), fp64 moments, reference operation order.
struct AdamArgs {
    float* params;
    const float* grads;
    double* m;
    double* v;
    uint64_t n;
    double bc1, bc2, lr, lr_alt, beta1, beta2, eps;
    uint32_t period, n_primary;
    unsigned int* nan_flag;
};
void launch_adam(const AdamArgs& a, cudaStream_t st);

struct BackwardArgs {
    const uint2* ranges;
    const uint32_t* tile_order;  // optional LPT tile schedule (forward's)
    const uint32_t* vals;
    const float4* records;
    const uint32_t* corner_index;
    int K;
    float bg[3];
    const float* gC;  // ss res, optional
    const float* gD;
    const float* gN;
    const float* gT;
    const float* d_weight;       // per contrib, optional
    const float* d_voxel_color;  // per contrib x3, optional
    const uint32_t* pix_count;   // tile-major
    const uint32_t* pix_begin;
    const uint32_t* contrib_entry;  // compact, or staged when stage_stride > 0
    const float* contrib_T;
    uint32_t stage_stride;
    // per voxel x16 (scratch, all zero on entry): 8 corner densities, colour,
    // normal, priority; summed with float4 reductions, consumed (and zeroed
    // again) by the epilogue
    float* g_vox;
};
void launch_composite_backward(const DevCamera& cam, const BackwardArgs& a, cudaStream_t st);

struct EpilogueArgs {
    uint64_t n;
    const uint64_t* paths;
    const int4* rects;
    const float4* records;
    const float4* view_dir;  // K1's sh_eval directions (same floats as the forward)
    const uint32_t* corner_index;
    const float* sh;
    int sh_degree, sh_stride;
    double bc[3];
    double bsize;
    float* g_vox;       // K9's per-voxel sums; read and reset to zero here
    float* g_sh;
    float* g_density;
    float* g_priority;
    int accumulate;
    const uint32_t* list;         // optional: the voxels in `pre` (K1, training frames), any order
    const unsigned int* n_list;   // its length on the device; SH gradients of the others untouched
};
void launch_voxel_epilogue(const DevCamera& cam, const EpilogueArgs& a, cudaStream_t st);

// ---- pieces (batch utilities for the drop-in's pipeline functions) ---------
void launch_project_batch(const DevCamera& cam, uint64_t n, const double* centers,
                          const double* sizes, double near_plane, uint8_t* visible,
                          double* aabb, int* rect, cudaStream_t st);
void launch_tile_masks_only(const DevCamera& cam, uint8_t* masks, cudaStream_t st);
void launch_entry_counts(const DevCamera& cam, uint64_t n, const int4* rects,
                         const uint32_t* sat, uint32_t* counts, cudaStream_t st);
void launch_duplicate_list(const DevCamera& cam, uint64_t n, const uint32_t* vids,
                           const uint64_t* codes, const int4* rects, const uint8_t* masks,
                           const uint32_t* offsets, uint64_t* keys, uint32_t* vals,
                           cudaStream_t st);

// Voxel record (96 B = 6 float4), written by K1, read by K7/K9/K10:
//   [0] lo.xyz (camera-relative min corner), size   [1] screen AABB x0,x1,y0,y1
//   [2] c6,c7,c2,c4   [3] c3,c5,c0,c1  (trilinear_coeffs of the corner densities
//       V0..V7, pair-ordered for FFMA2: pack_coeffs)
//   [4] rgb, vid (bits)   [5] unit normal, 1/size
constexpr int kRecordF4 = 6;

}  // namespace svrb
