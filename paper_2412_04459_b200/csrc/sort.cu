// sort.cu — hand-written onesweep LSD radix sort of (u64 key, u32 value).
//
// Replaces sort_entries (raster.cpp:174-178, std::sort by (key, value)).
// Design (Adinets & Merrill, "Onesweep", 2022):
//   1. one upsweep kernel builds the digit histograms of ALL passes in a
//      single read of the keys;
//   2. one kernel per pass: each CTA claims a partition via an atomic
//      ticket (forward-progress order), ranks its keys with warp-level
//      match.any multi-split, publishes its per-digit count and resolves its
//      global offset by decoupled look-back over earlier partitions, then
//      scatters through shared memory so global writes are digit-contiguous.
// Each pass reads and writes every pair once (12 B + 12 B). The sort is
// stable, so sorting only the key bits that can differ (the caller decides,
// see capi.cu) reproduces the full (key, value) order exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "svr_internal.h"
#include "svr_kernels.h"

namespace svrb {

namespace {

#ifndef SVR_SORT_EARLY_SCATTER
#define SVR_SORT_EARLY_SCATTER 1
#endif
#ifndef SVR_SORT_LB_PREFETCH
#define SVR_SORT_LB_PREFETCH 0
#endif
#ifndef SVR_SORT_CONST_BITS
#define SVR_SORT_CONST_BITS 1
#endif
#ifndef SVR_SORT_ATOMIC_RANK
#define SVR_SORT_ATOMIC_RANK 1
#endif
constexpr int kRadix = 256;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;
constexpr int kTileKeys = kThreads * kItems;  // 2048 pairs per partition
// keys-only partitions are larger: 3072 keys, so a config-2 pass (1.76M
// keys) is 574 CTAs = one wave of 4 resident CTAs on 148 SMs
#ifndef SVR_SORT_ITEMS
#define SVR_SORT_ITEMS 12  // keys per thread (keys-only): 16 is 7 % faster at 97M keys, 5 % slower at 4.5M
#endif
constexpr int kItemsK = SVR_SORT_ITEMS;
constexpr int kTileKeysK = kThreads * kItemsK;
template <bool PAIRS, int IK = kItemsK>
struct Part {
    static constexpr int items = PAIRS ? kItems : IK;
    static constexpr int keys = kThreads * items;
};
// keys-only passes over at least this many keys use 16 keys per thread
// (fewer partitions to look back over: 7 % faster at 97M keys, 5 % slower at 4.5M)
constexpr uint64_t kLargeSortKeys = uint64_t(1) << 25;
constexpr int kItemsLarge = 16;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

struct PassSpec {
    int n;
    RadixPass p[kMaxRadixPasses];
};

__device__ __forceinline__ uint32_t digit_of(uint64_t k, uint32_t v, RadixPass p) {
    uint64_t w = p.src == 0 ? k : uint64_t(v);
    return uint32_t(w >> p.shift) & ((1u << p.bits) - 1u);
}

__global__ void __launch_bounds__(kThreads) hist_kernel(const uint64_t* keys, const uint32_t* vals,
                                                        uint64_t n, PassSpec spec,
                                                        uint32_t* hist,
                                                        const unsigned long long* n_dev) {
    pdl_enter();
    n = live_entries(n, n_dev);  // deferred-E frame: the device count decides
    __shared__ uint32_t s_hist[kMaxRadixPasses][kRadix];
    for (int i = threadIdx.x; i < spec.n * kRadix; i += kThreads) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * kThreads) {
        uint64_t k = keys[i];
        uint32_t v = vals ? vals[i] : 0u;
        for (int p = 0; p < spec.n; ++p) atomicAdd(&s_hist[p][digit_of(k, v, spec.p[p])], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < spec.n * kRadix; i += kThreads) {
        uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

__global__ void ranges_init_kernel(uint2* ranges, int ntiles) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < ntiles) ranges[t] = make_uint2(0xffffffffu, 0u);
}

// One block per pass: exclusive scan of the 256 digit counts.
__global__ void __launch_bounds__(kRadix) bin_scan_kernel(uint32_t* hist) {
    pdl_enter();
    __shared__ uint32_t s[kRadix];
    uint32_t* h = hist + blockIdx.x * kRadix;
    uint32_t v = h[threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kRadix; o <<= 1) {
        uint32_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
        __syncthreads();
        s[threadIdx.x] += t;
        __syncthreads();
    }
    h[threadIdx.x] = s[threadIdx.x] - v;
}

// Lanes holding the same digit (di < 2^bits, or kRadix for an empty slot).
// BALLOT: one ballot per digit bit instead of match.any — faster in the
// large-sort instantiation (16 keys per thread; config 4 sort 1.51 -> 1.38
// ms), slower at config-2 sizes (0.054 -> 0.067 ms), so only there.
#ifndef SVR_SORT_BALLOT_ALL
#define SVR_SORT_BALLOT_ALL 0
#endif
// BITS > 0: the pass's digit width as a compile-time constant (unrolled
// ballots, constant masks); EMPTY: the warp holds out-of-range slots (only in
// the last partition), whose digit kRadix needs one more ballot.
template <bool BALLOT, int BITS = 0, bool EMPTY = true>
__device__ __forceinline__ uint32_t digit_peers(uint32_t di, int bits) {
    if (!BALLOT) return __match_any_sync(0xffffffffu, di);
    uint32_t peers = 0xffffffffu;
    if constexpr (BITS > 0) {
#pragma unroll
        for (int b = 0; b < BITS; ++b) {
            // lanes whose bit b equals ours: one predicate test, the ballot,
            // a select and one LOP3 (C++ gives ptxas two predicates per bit)
            asm("{\n\t.reg .pred p;\n\t.reg .b32 t, m;\n\t"
                "and.b32 t, %1, %2;\n\t"
                "setp.ne.u32 p, t, 0;\n\t"
                "vote.sync.ballot.b32 t, p, 0xffffffff;\n\t"
                "selp.b32 m, 0, -1, p;\n\t"
                "xor.b32 t, t, m;\n\t"
                "and.b32 %0, %0, t;\n\t}"
                : "+r"(peers)
                : "r"(di), "r"(1u << b));
        }
    } else {
        for (int b = 0; b < bits; ++b) {
            const bool on = (di >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, on);
            peers &= on ? bal : ~bal;
        }
    }
    if (!EMPTY) return peers;
    const bool empty = di >= uint32_t(kRadix);
    const uint32_t bal = __ballot_sync(0xffffffffu, empty);
    return peers & (empty ? bal : ~bal);
}

// Keys-only digit with a compile-time width when BITS > 0.
template <int BITS>
__device__ __forceinline__ uint32_t key_digit(uint64_t k, RadixPass p) {
    const uint32_t mask = BITS > 0 ? (1u << BITS) - 1u : (1u << p.bits) - 1u;
    return uint32_t(k >> p.shift) & mask;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

template <bool PAIRS, int IK = kItemsK, int BITS = 0>
__global__ void __launch_bounds__(kThreads, 4) onesweep_kernel(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint64_t n, RadixPass pass,
    const uint32_t* __restrict__ bin_base, uint32_t* status, uint32_t* ticket,
    const unsigned long long* n_dev, int out_vb, uint2* ranges, int tile_shift) {
    pdl_enter();
    __shared__ uint32_t s_warp_hist[kWarps][kRadix + 1];
    __shared__ uint32_t s_block_excl[kRadix];
    __shared__ uint32_t s_global[kRadix];
    __shared__ uint64_t s_keys[Part<PAIRS, IK>::keys];
    __shared__ uint32_t s_vals[PAIRS ? Part<PAIRS, IK>::keys : 1];
    __shared__ uint32_t s_part;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_part = atomicAdd(ticket, 1u);
    for (int i = threadIdx.x; i < kWarps * (kRadix + 1); i += kThreads)
        (&s_warp_hist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    n = live_entries(n, n_dev);  // deferred-E frame: the device count decides
    const uint64_t base = uint64_t(part) * Part<PAIRS, IK>::keys;
    if (base >= n && part > 0) return;  // past the live count: no later partition looks back here
    const uint64_t wbase = base + uint64_t(warp) * 32 * Part<PAIRS, IK>::items;

    // Digits are recomputed from the key/value when needed (saves registers);
    // out-of-range slots get digit kRadix and are ranked into a discarded bin.
    uint64_t k[Part<PAIRS, IK>::items];
    uint32_t v[PAIRS ? Part<PAIRS, IK>::items : 1], r[Part<PAIRS, IK>::items];
    const uint64_t nvalid = n > wbase ? n - wbase : 0;
    // Slots past the live count (last partition only) take the pass's largest
    // digit: they rank after every real key of that bin in this partition, i.e.
    // at the partition's end (shared positions >= tile_n), and are never
    // written out; no later partition reads this one's status.
    const uint32_t pad_digit = (1u << (BITS > 0 ? BITS : pass.bits)) - 1u;
    auto dig = [&](int i) -> uint32_t {
        if (uint64_t(i) * 32 + lane < nvalid)
            return PAIRS ? digit_of(k[i], v[PAIRS ? i : 0], pass) : key_digit<BITS>(k[i], pass);
        return pad_digit;
    };
#pragma unroll
    for (int i = 0; i < Part<PAIRS, IK>::items; ++i) {
        uint64_t idx = wbase + uint64_t(i) * 32 + lane;
        k[i] = idx < n ? keys_in[idx] : 0ull;
        if (PAIRS) v[PAIRS ? i : 0] = idx < n ? vals_in[idx] : 0u;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t* wh = s_warp_hist[warp];
#if SVR_SORT_ATOMIC_RANK
    // Warp-aggregated shared-memory atomics: the leader of each digit group
    // reserves the group's slots; the items' reservations pipeline instead of
    // serialising on a load/store/syncwarp round trip each.
#pragma unroll
    for (int i = 0; i < Part<PAIRS, IK>::items; ++i) {
        const uint32_t di = dig(i);
        constexpr bool kBallot = !PAIRS && (SVR_SORT_BALLOT_ALL || IK == kItemsLarge);
        const uint32_t peers = digit_peers<kBallot, BITS, false>(di, pass.bits);
        const int leader = __ffs(peers) - 1;
        uint32_t prev = 0;
        if (lane == leader) prev = atomicAdd(&wh[di], uint32_t(__popc(peers)));
        r[i] = __shfl_sync(0xffffffffu, prev, leader) + __popc(peers & lt_mask);
    }
#else
#pragma unroll
    for (int i = 0; i < Part<PAIRS, IK>::items; ++i) {
        const uint32_t di = dig(i);
        uint32_t peers = __match_any_sync(0xffffffffu, di);
        uint32_t below = __popc(peers & lt_mask);
        uint32_t prev = wh[di];
        r[i] = prev + below;
        __syncwarp();
        if (below == 0) wh[di] = prev + __popc(peers);
        __syncwarp();
    }
#endif
    __syncthreads();

    // Per digit: exclusive offsets across warps, block total, block-wide
    // exclusive scan over digits, decoupled look-back for the global base.
    const int dg = threadIdx.x;  // kThreads == kRadix
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        uint32_t t = s_warp_hist[w][dg];
        s_warp_hist[w][dg] = cnt;
        cnt += t;
    }
    // bins past the pass's digit range stay empty: no status, no look-back
    // (a 4-bit pass polls 16 bins per predecessor instead of 256)
    const bool live_bin = dg < (1 << pass.bits);
    uint32_t* my_status = status + uint64_t(part) * kRadix + dg;
    if (live_bin) {
        if (part == 0)
            st_volatile(my_status, kFlagInc | cnt);
        else
            st_volatile(my_status, kFlagAgg | cnt);
    }
    // the predecessor's status, read now and consumed after the scatter: when
    // it is already inclusive the look-back costs no further round trip
    uint32_t pre = 0;
    if (SVR_SORT_LB_PREFETCH && part > 0 && live_bin) pre = ld_volatile(status + uint64_t(part - 1) * kRadix + dg);

    // block-wide exclusive scan of cnt over digits: warp scans, then the
    // eight warp totals (two barriers instead of sixteen)
    __shared__ uint32_t s_wtot[kWarps];
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wtot[warp] = incl;
    __syncthreads();
    uint32_t dbase = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) dbase += w < warp ? s_wtot[w] : 0u;
    const uint32_t block_excl = dbase + incl - cnt;
    s_block_excl[dg] = block_excl;
#if SVR_SORT_EARLY_SCATTER
    // The shared-memory scatter needs only block-local offsets: do it before
    // the look-back, so the (L2-latency-bound) look-back of the live-bin
    // threads overlaps the other warps' scatter instead of idling the CTA.
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Part<PAIRS, IK>::items; ++i) {
        const uint32_t di = dig(i);
        const uint32_t pos = s_block_excl[di] + s_warp_hist[warp][di] + r[i];
        s_keys[pos] = k[i];
        if (PAIRS) s_vals[pos] = v[PAIRS ? i : 0];
    }
#endif

    // Decoupled look-back, four predecessors per round so the dependent
    // L2 round trips overlap; stops at the first inclusive prefix.
    uint32_t excl = 0;
    if (SVR_SORT_LB_PREFETCH && (pre & kFlagInc)) {
        excl = pre & kValMask;
        st_volatile(my_status, kFlagInc | (excl + cnt));
    } else if (part > 0 && live_bin) {
        int64_t p = int64_t(part) - 1;
        while (p >= 0) {
            uint32_t s[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                s[q] = (p - q >= 0) ? ld_volatile(status + uint64_t(p - q) * kRadix + dg) : kFlagInc;
            int q = 0;
            bool stop = false;
            for (; q < 4; ++q) {
                if ((s[q] & ~kValMask) == 0) break;  // not published yet: re-poll from here
                excl += s[q] & kValMask;
                if (s[q] & kFlagInc) {
                    stop = true;
                    break;
                }
            }
            if (stop) break;
            p -= q;
        }
        st_volatile(my_status, kFlagInc | (excl + cnt));
    }
    s_global[dg] = bin_base[dg] + excl - block_excl;
#if !SVR_SORT_EARLY_SCATTER
    __syncthreads();

    // Scatter to shared memory in digit order, then out to global.
#pragma unroll
    for (int i = 0; i < Part<PAIRS, IK>::items; ++i) {
        const uint32_t di = dig(i);
        const uint32_t pos = s_block_excl[di] + s_warp_hist[warp][di] + r[i];
        s_keys[pos] = k[i];
        if (PAIRS) s_vals[pos] = v[PAIRS ? i : 0];
    }
#endif
    __syncthreads();
    const uint32_t tile_n = uint32_t(min(uint64_t(Part<PAIRS, IK>::keys), n - base));
    for (uint32_t pos = threadIdx.x; pos < tile_n; pos += kThreads) {
        uint64_t kk = s_keys[pos];
        uint32_t vv = PAIRS ? s_vals[pos] : 0u;
        uint32_t dd = PAIRS ? digit_of(kk, vv, pass) : key_digit<BITS>(kk, pass);
        uint64_t o = uint64_t(s_global[dd]) + pos;
        if (!PAIRS && out_vb >= 0) {
            // final pass of a packed sort: the reference value only, and the
            // tile ranges from the run ends in this partition (a tile's keys
            // are contiguous in the output, so min of starts / max of ends)
            vals_out[o] = (uint32_t((kk >> out_vb) & 7u) << 29) | uint32_t(kk & ((uint64_t(1) << out_vb) - 1));
            const uint64_t t = kk >> tile_shift;
            bool first, last;
            if (tile_shift >= 32) {  // the tile lies in the high words: 4-B neighbour loads, 32-bit compares
                const uint32_t* s_hi = reinterpret_cast<const uint32_t*>(s_keys) + 1;
                const uint32_t hi = uint32_t(kk >> 32);
                const int hs = tile_shift - 32;
                first = pos == 0 || ((s_hi[2 * (pos - 1)] ^ hi) >> hs) != 0u;
                last = pos + 1 == tile_n || ((s_hi[2 * (pos + 1)] ^ hi) >> hs) != 0u;
            } else {
                first = pos == 0 || (s_keys[pos - 1] >> tile_shift) != t;
                last = pos + 1 == tile_n || (s_keys[pos + 1] >> tile_shift) != t;
            }
            if (first) atomicMin(&ranges[t].x, uint32_t(o));
            if (last) atomicMax(&ranges[t].y, uint32_t(o + 1));
            continue;
        }
        keys_out[o] = kk;
        if (PAIRS) vals_out[o] = vv;
    }
}

// Keys-only pass kernel with the digit width as a compile-time constant
// (the tile bits are split evenly, so 4..7 cover every image up to 2^14 tiles).
template <int IK>
decltype(&onesweep_kernel<false, IK, 0>) pick_onesweep(int bits) {
#if SVR_SORT_CONST_BITS
    switch (bits) {
        case 4: return onesweep_kernel<false, IK, 4>;
        case 5: return onesweep_kernel<false, IK, 5>;
        case 6: return onesweep_kernel<false, IK, 6>;
        case 7: return onesweep_kernel<false, IK, 7>;
        default: break;
    }
#endif
    (void)bits;
    return onesweep_kernel<false, IK, 0>;
}

}  // namespace

size_t sort_scratch_bytes(uint64_t n, int npasses) {
    uint64_t nparts = (n + kTileKeys - 1) / kTileKeys;  // >= keys-only partition count
    return size_t(npasses) * kRadix * 4                     // histograms / bin bases
           + size_t(npasses) * 4 + 64                       // tickets
           + size_t(npasses) * (nparts + 1) * kRadix * 4;   // look-back status per pass
}

int radix_sort_pairs(uint64_t* keys0, uint32_t* vals0, uint64_t* keys1, uint32_t* vals1,
                     uint64_t n, const RadixPass* passes, int npasses, void* scratch,
                     cudaStream_t st) {
    if (n <= 1 || npasses == 0) return 0;
    if (npasses > kMaxRadixPasses) throw Error(SVR_ERR_RUNTIME, "too many radix passes");
    if (n >= (uint64_t(1) << 30))
        throw Error(SVR_ERR_LENGTH, "sort supports fewer than 2^30 entries");
    PassSpec spec{};
    spec.n = npasses;
    for (int i = 0; i < npasses; ++i) spec.p[i] = passes[i];
    uint64_t nparts = (n + kTileKeys - 1) / kTileKeys;
    char* s = static_cast<char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(s);
    uint32_t* tickets = reinterpret_cast<uint32_t*>(s + size_t(npasses) * kRadix * 4);
    uint32_t* status =
        reinterpret_cast<uint32_t*>(s + size_t(npasses) * kRadix * 4 + size_t(npasses) * 4 + 64);
    // one memset clears histograms, tickets and every pass's look-back status
    SVR_CUDA(cudaMemsetAsync(hist, 0, sort_scratch_bytes(n, npasses), st));
    int hist_blocks = int(std::min<uint64_t>((n + kThreads - 1) / kThreads, 148 * 4));
    hist_kernel<<<hist_blocks, kThreads, 0, st>>>(keys0, vals0, n, spec, hist, nullptr);
    SVR_LAUNCH("hist_kernel");
    bin_scan_kernel<<<npasses, kRadix, 0, st>>>(hist);
    SVR_LAUNCH("bin_scan_kernel");
    uint64_t* kin = keys0;
    uint32_t* vin = vals0;
    uint64_t* kout = keys1;
    uint32_t* vout = vals1;
    int cur = 0;
    for (int p = 0; p < npasses; ++p) {
        onesweep_kernel<true><<<unsigned(nparts), kThreads, 0, st>>>(
            kin, vin, kout, vout, n, passes[p], hist + p * kRadix,
            status + size_t(p) * (nparts + 1) * kRadix, tickets + p, nullptr, -1, nullptr, 0);
        SVR_LAUNCH("onesweep_kernel");
        std::swap(kin, kout);
        std::swap(vin, vout);
        cur ^= 1;
    }
    return cur;
}

uint32_t* sort_hist_ptr(void* scratch) { return static_cast<uint32_t*>(scratch); }

void sort_prepare(void* scratch, uint64_t n, int npasses, cudaStream_t st) {
    SVR_CUDA(cudaMemsetAsync(scratch, 0, sort_scratch_bytes(n, npasses), st));
}

int radix_sort_keys(uint64_t* keys0, uint64_t* keys1, uint64_t n, const RadixPass* passes,
                    int npasses, void* scratch, cudaStream_t st, bool hist_ready,
                    const unsigned long long* n_dev, const SortFinish* fin) {
    if (fin) {
        ranges_init_kernel<<<(fin->ntiles + 255) / 256, 256, 0, st>>>(fin->ranges, fin->ntiles);
        SVR_LAUNCH("ranges_init_kernel");
    }
    if (n <= 1 || npasses == 0) return 0;
    if (npasses > kMaxRadixPasses) throw Error(SVR_ERR_RUNTIME, "too many radix passes");
    if (n >= (uint64_t(1) << 30))
        throw Error(SVR_ERR_LENGTH, "sort supports fewer than 2^30 entries");
    for (int i = 0; i < npasses; ++i)
        if (passes[i].src != 0) throw Error(SVR_ERR_RUNTIME, "keys-only sort takes key digits only");
    const uint64_t nparts_alloc = (n + kTileKeys - 1) / kTileKeys;
    const uint64_t nparts = (n + kTileKeysK - 1) / kTileKeysK;
    char* s = static_cast<char*>(scratch);
    uint32_t* hist = reinterpret_cast<uint32_t*>(s);
    uint32_t* tickets = reinterpret_cast<uint32_t*>(s + size_t(npasses) * kRadix * 4);
    uint32_t* status =
        reinterpret_cast<uint32_t*>(s + size_t(npasses) * kRadix * 4 + size_t(npasses) * 4 + 64);
    if (!hist_ready) {
        SVR_CUDA(cudaMemsetAsync(hist, 0, sort_scratch_bytes(n, npasses), st));
        PassSpec spec{};
        spec.n = npasses;
        for (int i = 0; i < npasses; ++i) spec.p[i] = passes[i];
        int hist_blocks = int(std::min<uint64_t>((n + kThreads - 1) / kThreads, 148 * 4));
        launch_pdl(hist_kernel, hist_blocks, kThreads, 0, st, keys0, (const uint32_t*)nullptr, n, spec, hist,
                   n_dev);
        SVR_LAUNCH("hist_kernel");
    }
    launch_pdl(bin_scan_kernel, npasses, kRadix, 0, st, hist);
    SVR_LAUNCH("bin_scan_kernel");
    uint64_t* kin = keys0;
    uint64_t* kout = keys1;
    int cur = 0;
    const char* lk_env = std::getenv("SVR_LARGE_SORT_MIN");  // parity tests lower it
    const bool large = n >= (lk_env ? std::strtoull(lk_env, nullptr, 10) : kLargeSortKeys);
    const uint64_t nparts_run = large ? (n + uint64_t(kThreads) * kItemsLarge - 1) / (uint64_t(kThreads) * kItemsLarge)
                                      : nparts;
    for (int p = 0; p < npasses; ++p) {
        const bool last_fin = fin && p == npasses - 1;
        launch_pdl(large ? pick_onesweep<kItemsLarge>(passes[p].bits) : pick_onesweep<kItemsK>(passes[p].bits),
                   unsigned(nparts_run), kThreads, 0, st, (const uint64_t*)kin,
                   (const uint32_t*)nullptr, kout, last_fin ? fin->vals : (uint32_t*)nullptr, n, passes[p],
                   (const uint32_t*)(hist + p * kRadix), status + size_t(p) * (nparts_alloc + 1) * kRadix,
                   tickets + p, n_dev, last_fin ? fin->vb : -1, last_fin ? fin->ranges : (uint2*)nullptr,
                   last_fin ? fin->tile_shift : 0);
        SVR_LAUNCH("onesweep_kernel");
        std::swap(kin, kout);
        cur ^= 1;
    }
    return cur;
}

}  // namespace svrb
