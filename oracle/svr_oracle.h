/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * svr_oracle: a plain-C (C11, double precision) restatement of the
 * reference rasterizer's render and gradient path, used as the CPU checker
 * of the CUDA product. Pinned against the unmodified reference
 * (oracle/_ref/libsvr_ref.so) by tests/test_oracle.py and against the
 * committed golden fixtures in tests/golden/.
 */
#ifndef SVR_ORACLE_H
#define SVR_ORACLE_H

#include <stdint.h>

#include "svr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* tile_sign_patterns (raster.cpp:120-142) for every tile, as bitmasks. */
int orc_tile_masks(const svr_camera* cam, uint8_t* masks);

/* geometry_of + project_voxel (raster.cpp:72-118) per voxel on `cam`. */
int orc_project(const svr_scene_desc* s, const svr_camera* cam, double near_plane,
                uint8_t* visible, double* aabb, int32_t* rect);

/* preprocess + build_sort_entries (+ sort_entries) on `cam`; keys == NULL
 * returns the count only. */
int orc_entries(const svr_scene_desc* s, const svr_camera* cam, double near_plane, int sorted,
                uint64_t* n_out, uint64_t* keys, uint32_t* values);

/* render_with_pools (raster.cpp:205-297): images at target resolution. */
int orc_render(const svr_scene_desc* s, const svr_camera* cam, const svr_render_options* o,
               double* color, double* depth, double* median, double* normal, double* tfin,
               double* max_blend);

/* render_with_pools(training) followed by render_backward
 * (raster.cpp:303-423) with image-level upstream gradients (NULL = zero). */
int orc_backward(const svr_scene_desc* s, const svr_camera* cam, const svr_render_options* o,
                 const double* d_color, const double* d_depth, const double* d_normal,
                 const double* d_tfin_ss, double* g_density, double* g_sh, double* g_priority);

#ifdef __cplusplus
}
#endif
#endif
