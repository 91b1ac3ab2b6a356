// scan.cu — device-wide exclusive prefix sum over u32 (reduce-then-scan).
//
// Used for the per-voxel entry counts (the "key duplication by block-wide
// prefix scan" step that replaces the push_back loop of build_sort_entries,
// raster.cpp:155-170), the visible-voxel rank (`pre` index, raster.cpp:
// 221-223) and the per-pixel contribution counts (ForwardRecords::pix_begin,
// raster.cpp:256-270). HBM-bound: 4 B read twice + 4 B written per element.
#include <cuda_runtime.h>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {

namespace {

constexpr int kThreads = 512;
constexpr int kItems = 8;
constexpr int kChunk = kThreads * kItems;  // 4096 elements per block
static_assert(kChunk == kScanChunk && kThreads == kScanThreads, "svr_kernels.h scan geometry");

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the total too.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(v);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (kThreads / 32) ? s_warp[lane] : 0;
        uint32_t wi = warp_incl_scan(w);
        if (lane < (kThreads / 32)) s_warp[lane] = wi - w;
        if (lane == 31) s_warp[kThreads / 32] = wi;
    }
    __syncthreads();
    total = s_warp[kThreads / 32];
    uint32_t r = s_warp[warp] + incl - v;
    __syncthreads();
    return r;
}

__device__ __forceinline__ void load_items(const uint32_t* in, uint64_t n, uint64_t base,
                                           uint32_t* x) {
    uint64_t i0 = base + uint64_t(threadIdx.x) * kItems;
    if (i0 + kItems <= n && ((reinterpret_cast<uintptr_t>(in + i0) & 15) == 0)) {
        uint4 a = *reinterpret_cast<const uint4*>(in + i0);
        uint4 b = *reinterpret_cast<const uint4*>(in + i0 + 4);
        x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w;
        x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < kItems; ++k) x[k] = (i0 + k < n) ? in[i0 + k] : 0u;
    }
}

__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(const uint32_t* in, uint64_t n,
                                                               uint32_t* partial) {
    pdl_enter();
    __shared__ uint32_t s_warp[kThreads / 32 + 1];
    uint32_t x[kItems];
    load_items(in, n, uint64_t(blockIdx.x) * kChunk, x);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) s += x[k];
    uint32_t total;
    block_excl_scan(s, s_warp, total);
    if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

// Single block: exclusive scan of the block partials (in place), u64 total.
__global__ void __launch_bounds__(kThreads) scan_partials_kernel(uint32_t* partial, uint64_t nb,
                                                                 unsigned long long* total) {
    pdl_enter();
    __shared__ uint32_t s_warp[kThreads / 32 + 1];
    unsigned long long carry = 0;
    for (uint64_t base = 0; base < nb; base += kThreads) {
        uint64_t i = base + threadIdx.x;
        uint32_t v = i < nb ? partial[i] : 0u;
        uint32_t t;
        uint32_t e = block_excl_scan(v, s_warp, t);
        if (i < nb) partial[i] = uint32_t(carry) + e;
        carry += t;
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(kThreads) scan_apply_kernel(const uint32_t* in, uint32_t* out,
                                                              uint64_t n, const uint32_t* partial) {
    pdl_enter();
    __shared__ uint32_t s_warp[kThreads / 32 + 1];
    uint32_t x[kItems];
    const uint64_t base = uint64_t(blockIdx.x) * kChunk;
    load_items(in, n, base, x);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) s += x[k];
    uint32_t t;
    uint32_t run = block_excl_scan(s, s_warp, t) + partial[blockIdx.x];
    uint64_t i0 = base + uint64_t(threadIdx.x) * kItems;
    uint32_t y[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        y[k] = run;
        run += x[k];
    }
    if (i0 + kItems <= n && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
        reinterpret_cast<uint4*>(out + i0)[0] = make_uint4(y[0], y[1], y[2], y[3]);
        reinterpret_cast<uint4*>(out + i0)[1] = make_uint4(y[4], y[5], y[6], y[7]);
    } else {
#pragma unroll
        for (int k = 0; k < kItems; ++k)
            if (i0 + k < n) out[i0 + k] = y[k];
    }
}

}  // namespace

size_t scan_scratch_bytes(uint64_t n) { return ((n + kChunk - 1) / kChunk + 1) * sizeof(uint32_t); }

void scan_block_prefixes(const uint32_t* in, uint64_t n, unsigned long long* total, void* scratch,
                         cudaStream_t st) {
    if (n == 0) {
        SVR_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), st));
        return;
    }
    uint64_t nb = (n + kChunk - 1) / kChunk;
    uint32_t* partial = static_cast<uint32_t*>(scratch);
    launch_pdl(scan_reduce_kernel, unsigned(nb), kThreads, 0, st, in, n, partial);
    SVR_LAUNCH("scan_reduce_kernel");
    launch_pdl(scan_partials_kernel, 1, kThreads, 0, st, partial, nb, total);
    SVR_LAUNCH("scan_partials_kernel");
}

void scan_block_sums(uint32_t* partial, uint64_t nb, unsigned long long* total, cudaStream_t st) {
    if (nb == 0) {
        SVR_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), st));
        return;
    }
    launch_pdl(scan_partials_kernel, 1, kThreads, 0, st, partial, nb, total);
    SVR_LAUNCH("scan_partials_kernel");
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, unsigned long long* total,
                        void* scratch, cudaStream_t st) {
    if (n == 0) {
        SVR_CUDA(cudaMemsetAsync(total, 0, sizeof(unsigned long long), st));
        return;
    }
    uint64_t nb = (n + kChunk - 1) / kChunk;
    uint32_t* partial = static_cast<uint32_t*>(scratch);
    launch_pdl(scan_reduce_kernel, unsigned(nb), kThreads, 0, st, in, n, partial);
    SVR_LAUNCH("scan_reduce_kernel");
    launch_pdl(scan_partials_kernel, 1, kThreads, 0, st, partial, nb, total);
    SVR_LAUNCH("scan_partials_kernel");
    launch_pdl(scan_apply_kernel, unsigned(nb), kThreads, 0, st, in, out, n, partial);
    SVR_LAUNCH("scan_apply_kernel");
}

}  // namespace svrb
