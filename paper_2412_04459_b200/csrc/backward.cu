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

constexpr int kAcc = 15;  // 8 corner densities + 3 colour + 3 normal + priority

__global__ void lift_kernel(TapTable t, const float* g, int ch, int W, float* out, int sw,
                            int sh) {
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

template <int K>
__global__ void __launch_bounds__(256) composite_backward_kernel(DevCamera cam, BackwardArgs a) {
    __shared__ float4 s_rec[kRecordF4][256];
    __shared__ float s_acc[kAcc][256];
    __shared__ uint32_t s_touch[256];
    __shared__ int s_max_last;

    const int tile = blockIdx.x;
    const int tx = tile % cam.ntx, ty = tile / cam.ntx;
    const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < cam.W && py < cam.H;
    const uint32_t slot = uint32_t(tile) * 256u + threadIdx.x;
    const int lane = threadIdx.x & 31;

    double dd[3];
    pixel_ray_dir(cam, double(px), double(py), dd);
    const float dx = float(dd[0]), dy = float(dd[1]), dz = float(dd[2]);
    const float ix = 1.0f / dx, iy = 1.0f / dy, iz = 1.0f / dz;
    const float dnorm = float(sqrt(dd[0] * dd[0] + dd[1] * dd[1] + dd[2] * dd[2]));

    uint32_t n = 0, base = 0;
    float gC[3] = {0.f, 0.f, 0.f}, gN[3] = {0.f, 0.f, 0.f}, gD = 0.f, gT = 0.f;
    if (inside) {
        n = a.pix_count[slot];
        base = a.pix_begin[slot];
        const uint64_t p = uint64_t(py) * cam.W + px;
        if (a.gC) gC[0] = a.gC[3 * p], gC[1] = a.gC[3 * p + 1], gC[2] = a.gC[3 * p + 2];
        if (a.gN) gN[0] = a.gN[3 * p], gN[1] = a.gN[3 * p + 1], gN[2] = a.gN[3 * p + 2];
        if (a.gD) gD = a.gD[p];
        if (a.gT) gT = a.gT[p];
    }
    int kidx = int(n) - 1;  // next contribution to match, walking backwards
    int next_e = kidx >= 0 ? int(a.contrib_entry[base + kidx]) : -1;
    float Ra = gC[0] * a.bg[0] + gC[1] * a.bg[1] + gC[2] * a.bg[2] + gT;
    float Rd = 0.f;

    if (threadIdx.x == 0) s_max_last = -1;
    for (int i = threadIdx.x; i < kAcc * 256; i += 256) (&s_acc[0][0])[i] = 0.f;
    __syncthreads();
    atomicMax(&s_max_last, next_e);
    __syncthreads();
    const int last = s_max_last;
    const uint2 range = a.ranges[tile];
    if (last < 0) return;

    for (int end = last + 1; end > int(range.x); end -= 256) {
        const int start = max(int(range.x), end - 256);
        const int nb = end - start;
        if (threadIdx.x < nb) {
            const uint32_t vid = a.vals[start + threadIdx.x] & ((1u << 29) - 1u);
            const float4* rec = a.records + uint64_t(vid) * kRecordF4;
#pragma unroll
            for (int k = 0; k < kRecordF4; ++k) s_rec[k][threadIdx.x] = __ldg(rec + k);
        }
        s_touch[threadIdx.x] = 0;
        __syncthreads();
        for (int j = nb - 1; j >= 0; --j) {
            const bool hit = (next_e == start + j);
            if (!__any_sync(0xffffffffu, hit)) continue;
            float acc[kAcc];
#pragma unroll
            for (int q = 0; q < kAcc; ++q) acc[q] = 0.f;
            if (hit) {
                const float4 lo = s_rec[0][j];
                const float inv = s_rec[5][j].w;
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
                const float4 va = s_rec[2][j], vb = s_rec[3][j];
                const float V[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
                const float seg = tb - ta;
                const float lk = seg * dnorm * (1.0f / K);
                float sa[K], tk[K], vk[K], qk[K][3];
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    tk[k] = ta + ((k + 0.5f) / K) * seg;
                    qk[k][0] = (tk[k] * dx - lo.x) * inv;
                    qk[k][1] = (tk[k] * dy - lo.y) * inv;
                    qk[k][2] = (tk[k] * dz - lo.z) * inv;
                    vk[k] = trilinear(V, qk[k][0], qk[k][1], qk[k][2]);
                    const float act = explin(vk[k]);
                    sum += act;
                    sa[k] = 1.0f - fexp(-lk * act);
                }
                const float alpha = (K == 1) ? sa[0] : 1.0f - fexp(-lk * sum);
                float dvox = 0.f, Tk = 1.f;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    dvox += Tk * sa[k] * tk[k];
                    Tk *= 1.0f - sa[k];
                }
                const float Ti = a.contrib_T[base + kidx];
                const float4 col = s_rec[4][j], nor = s_rec[5][j];
                const float gw = a.d_weight ? a.d_weight[base + kidx] : 0.f;
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
                    for (int m = 0; m < K; ++m)
                        if (m != k) others *= 1.0f - sa[m];
                    const float dAk = A * others + Ti * gD * ddk[k];
                    const float dv = dAk * (1.0f - sa[k]) * lk * explin_deriv(vk[k]);
                    float w[8];
                    trilinear_weights(qk[k][0], qk[k][1], qk[k][2], w);
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[c] += dv * w[c];
                }
                const float wgt = Ti * alpha;
                acc[8] = wgt * gC[0];
                acc[9] = wgt * gC[1];
                acc[10] = wgt * gC[2];
                if (a.d_voxel_color) {
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
                --kidx;
                next_e = kidx >= 0 ? int(a.contrib_entry[base + kidx]) : -1;
            }
#pragma unroll
            for (int q = 0; q < kAcc; ++q) {
                float v = acc[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                acc[q] = v;
            }
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < kAcc; ++q) atomicAdd(&s_acc[q][j], acc[q]);
                s_touch[j] = 1;
            }
        }
        __syncthreads();
        // one set of global atomics per touched entry of this batch
        if (threadIdx.x < nb && s_touch[threadIdx.x]) {
            const int j = threadIdx.x;
            const uint32_t vid = __float_as_uint(s_rec[4][j].w);
            const uint4* ci4 = reinterpret_cast<const uint4*>(a.corner_index + 8ull * vid);
            const uint4 c0 = ci4[0], c1 = ci4[1];
            const uint32_t ci[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int c = 0; c < 8; ++c) atomicAdd(a.g_density + ci[c], s_acc[c][j]);
            atomicAdd(a.g_color + 3ull * vid + 0, s_acc[8][j]);
            atomicAdd(a.g_color + 3ull * vid + 1, s_acc[9][j]);
            atomicAdd(a.g_color + 3ull * vid + 2, s_acc[10][j]);
            atomicAdd(a.g_normal + 3ull * vid + 0, s_acc[11][j]);
            atomicAdd(a.g_normal + 3ull * vid + 1, s_acc[12][j]);
            atomicAdd(a.g_normal + 3ull * vid + 2, s_acc[13][j]);
            atomicAdd(a.g_priority + vid, s_acc[14][j]);
#pragma unroll
            for (int q = 0; q < kAcc; ++q) s_acc[q][j] = 0.f;
        }
        if (__syncthreads_count(kidx >= 0) == 0) break;
    }
}

__global__ void __launch_bounds__(256) voxel_epilogue_kernel(DevCamera cam, EpilogueArgs a) {
    const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= a.n) return;
    float* gsh = a.g_sh + v * uint64_t(a.sh_stride);
    const int4 r = a.rects[v];
    if (r.y < r.x) {  // not in `pre`: no gradient
        if (!a.accumulate)
            for (int m = 0; m < a.sh_stride; ++m) gsh[m] = 0.f;
        return;
    }
    const uint64_t path = a.paths[v];
    double center[3], size;
    voxel_geometry(path & ((uint64_t(1) << 48) - 1), int(path >> 48), a.bc, a.bsize, center, &size);
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
    const int nb = sh_basis(a.sh_degree, ux, uy, uz, b);
    const float* co = a.sh + v * uint64_t(a.sh_stride);
    float raw[3] = {0.f, 0.f, 0.f};
    for (int m = 0; m < nb; ++m) {
        raw[0] += b[m] * co[3 * m + 0];
        raw[1] += b[m] * co[3 * m + 1];
        raw[2] += b[m] * co[3 * m + 2];
    }
    const float g0 = raw[0] > 0.f ? a.g_color[3 * v + 0] : 0.f;
    const float g1 = raw[1] > 0.f ? a.g_color[3 * v + 1] : 0.f;
    const float g2 = raw[2] > 0.f ? a.g_color[3 * v + 2] : 0.f;
    for (int m = 0; m < nb; ++m) {
        float o0 = b[m] * g0, o1 = b[m] * g1, o2 = b[m] * g2;
        if (a.accumulate) {
            gsh[3 * m + 0] += o0;
            gsh[3 * m + 1] += o1;
            gsh[3 * m + 2] += o2;
        } else {
            gsh[3 * m + 0] = o0;
            gsh[3 * m + 1] = o1;
            gsh[3 * m + 2] = o2;
        }
    }
    const float4* rec = a.records + v * kRecordF4;
    const float4 va = rec[2], vb = rec[3];
    const float V[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
    const float dn[3] = {a.g_normal[3 * v], a.g_normal[3 * v + 1], a.g_normal[3 * v + 2]};
    if (dn[0] == 0.f && dn[1] == 0.f && dn[2] == 0.f) return;
    float gV[8];
    voxel_normal_backward(V, dn, gV);
    const uint4* ci4 = reinterpret_cast<const uint4*>(a.corner_index + 8 * v);
    const uint4 c0 = ci4[0], c1 = ci4[1];
    const uint32_t ci[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) atomicAdd(a.g_density + ci[c], gV[c]);
}

inline unsigned blocks_for(uint64_t n, int threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

void launch_lift(const TapTable& t, const float* g, int channels, int W, float* out, int sw,
                 int sh, cudaStream_t st) {
    dim3 grid(blocks_for(sw, 128), sh);
    lift_kernel<<<grid, 128, 0, st>>>(t, g, channels, W, out, sw, sh);
    SVR_LAUNCH("lift_kernel");
}

void launch_l1_loss(const float* color, const float* gt, uint64_t n, float* d_color, float* loss,
                    cudaStream_t st) {
    if (loss) SVR_CUDA(cudaMemsetAsync(loss, 0, sizeof(float), st));
    unsigned blocks = unsigned(std::min<uint64_t>(blocks_for(n, 256), 148 * 8));
    l1_kernel<<<blocks, 256, 0, st>>>(color, gt, n, 1.0f / float(n), d_color, loss);
    SVR_LAUNCH("l1_kernel");
}

void launch_composite_backward(const DevCamera& cam, const BackwardArgs& a, cudaStream_t st) {
    const unsigned ntiles = unsigned(cam.ntx * cam.nty);
    switch (a.K) {
        case 1:
            composite_backward_kernel<1><<<ntiles, 256, 0, st>>>(cam, a);
            break;
        case 2:
            composite_backward_kernel<2><<<ntiles, 256, 0, st>>>(cam, a);
            break;
        case 3:
            composite_backward_kernel<3><<<ntiles, 256, 0, st>>>(cam, a);
            break;
        default:
            throw Error(SVR_ERR_INVALID_ARGUMENT, "rasterizer sample count K must be in {1,2,3}");
    }
    SVR_LAUNCH("composite_backward_kernel");
}

void launch_voxel_epilogue(const DevCamera& cam, const EpilogueArgs& a, cudaStream_t st) {
    if (a.n == 0) return;
    voxel_epilogue_kernel<<<blocks_for(a.n, 256), 256, 0, st>>>(cam, a);
    SVR_LAUNCH("voxel_epilogue_kernel");
}

}  // namespace svrb
