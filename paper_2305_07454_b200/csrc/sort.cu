// Stable LSD radix sort (u64 keys, u32 values) and a device-wide exclusive scan, written for
// sm_100a without CUB/Thrust (north_star: no library sort as product code).
//
// Per 8-bit digit pass: (1) per-tile digit histograms, (2) digit-major exclusive scan of the
// histograms so tile t's keys of digit d precede tile t+1's (stability), (3) per-tile stable
// ranking with __match_any_sync peer groups and per-warp digit counters in shared memory, then
// scatter. Passes whose digit is constant across all keys are skipped (decided on the host from a
// device-side OR/AND reduction of the keys).
#include "kernels.cuh"
#include "sort_api.cuh"

namespace cvlg {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* in, uint64_t n,
                                                                   uint32_t* partial) {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * kScanThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    s = warp_sum(s);
    __shared__ uint32_t ws[kScanThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
        partial[blockIdx.x] = t;
    }
}

// single CTA: exclusive scan of partial[0..n) in place, total -> *total
__global__ void __launch_bounds__(1024) scan_partials_kernel(uint32_t* partial, uint64_t n,
                                                             uint32_t* total) {
    __shared__ uint32_t sm[1024 / 32 + 1];
    uint32_t carry = 0;
    for (uint64_t base = 0; base < n; base += 1024) {
        const uint64_t idx = base + threadIdx.x;
        const uint32_t v = idx < n ? partial[idx] : 0u;
        uint32_t tot;
        const uint32_t ex = block_exclusive_scan<1024>(v, sm, tot);
        if (idx < n) partial[idx] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const uint32_t* in, uint32_t* out,
                                                                 uint64_t n,
                                                                 const uint32_t* partial) {
    __shared__ uint32_t sm[kScanThreads / 32 + 1];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
    // blocked arrangement: thread t owns items [t*8, t*8+8)
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(threadIdx.x) * kScanItems + i;
        v[i] = idx < n ? in[idx] : 0u;
        s += v[i];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<kScanThreads>(s, sm, tot) + partial[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(threadIdx.x) * kScanItems + i;
        if (idx < n) out[idx] = ex;
        ex += v[i];
    }
}

// ---- radix ----------------------------------------------------------------------------------
constexpr int kRThreads = 256;
constexpr int kRItems = 16;
constexpr int kRTile = kRThreads * kRItems;  // 4096 keys per tile
constexpr int kRWarps = kRThreads / 32;
constexpr int kRWarpKeys = kRTile / kRWarps;  // 512 keys per warp, 16 rounds of 32

__global__ void __launch_bounds__(kRThreads) radix_hist_kernel(const uint64_t* keys, uint64_t n,
                                                               int shift, uint32_t* counts,
                                                               uint32_t n_tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRTile;
#pragma unroll 4
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * kRThreads + threadIdx.x;
        if (idx < n) {
            const uint32_t d = static_cast<uint32_t>(keys[idx] >> shift) & 0xFFu;
            atomicAdd(&h[d], 1u);
        }
    }
    __syncthreads();
    counts[static_cast<uint64_t>(threadIdx.x) * n_tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRThreads) radix_scatter_kernel(
    const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out, uint32_t* vals_out,
    uint64_t n, int shift, const uint32_t* offsets, uint32_t n_tiles) {
    __shared__ uint32_t wc[kRWarps][256];
    __shared__ uint32_t tile_off[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRWarps * 256; i += kRThreads) (&wc[0][0])[i] = 0;
    tile_off[threadIdx.x] = offsets[static_cast<uint64_t>(threadIdx.x) * n_tiles + blockIdx.x];
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kRTile + static_cast<uint64_t>(warp) * kRWarpKeys;
    uint64_t k[kRItems];
    uint32_t v[kRItems];
    uint32_t rank[kRItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * 32 + lane;
        const bool valid = idx < n;
        k[i] = valid ? keys_in[idx] : 0ull;
        v[i] = valid ? vals_in[idx] : 0u;
        const uint32_t d = valid ? (static_cast<uint32_t>(k[i] >> shift) & 0xFFu) : 256u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        uint32_t r = 0;
        if (valid) {
            const uint32_t before = wc[warp][d];
            r = before + __popc(peers & lt);
        }
        __syncwarp();
        if (valid && (peers & lt) == 0) wc[warp][d] += __popc(peers);
        __syncwarp();
        rank[i] = r;
    }
    __syncthreads();
    // exclusive prefix across warps, per digit
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRWarps; ++w) {
            const uint32_t t = wc[w][d];
            wc[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * 32 + lane;
        if (idx < n) {
            const uint32_t d = static_cast<uint32_t>(k[i] >> shift) & 0xFFu;
            const uint64_t pos = static_cast<uint64_t>(tile_off[d]) + wc[warp][d] + rank[i];
            keys_out[pos] = k[i];
            vals_out[pos] = v[i];
        }
    }
}

// ---- one-sweep LSD passes ------------------------------------------------------------------------
// (1) radix_hist8_kernel: global 256-bin histograms of all 8 byte digits in one read of the keys;
// (2) its last block (radix_digit_base_block): per pass, exclusive digit offsets + "digit
//     constant" flags (a digit is constant iff one bin holds every key: the pass is skipped, order
//     unchanged) and the pass plan;
// (3) radix_onesweep_kernel per remaining pass: tiles taken in order from an atomic counter rank
//     their keys (stable, as radix_scatter_kernel), publish per-digit counts, and resolve their
//     per-digit offsets by a decoupled look-back over previous tiles (one 32-bit word per
//     (tile, digit): 2-bit flag | 30-bit count), then scatter. One launch per pass.
constexpr uint32_t kOsAgg = 1u << 30, kOsInc = 2u << 30, kOsMask = (1u << 30) - 1;

// digit offsets + pass plan from the complete histograms (one block: the last histogram block)
// plan[d] for digit d = 1 + (index of the buffer its pass reads: 0 = keys, 1 = alt) when the pass
// runs, 0 when the digit is constant (skipped); plan[8] = buffer holding the result. Decided on
// the device, so the host never waits for the histograms.
__device__ void radix_digit_base_block(const uint32_t* hist, uint64_t n, uint32_t* base,
                                       unsigned long long* constant_mask, int d_begin, int d_end,
                                       uint32_t* plan) {
    __shared__ uint32_t sm[256 / 32 + 1];
    __shared__ unsigned long long cmask;
    if (threadIdx.x == 0) cmask = 0;
    __syncthreads();
    for (int p = 0; p < 8; ++p) {
        const uint32_t v = __ldcg(&hist[p * 256 + threadIdx.x]);
        uint32_t tot;
        base[p * 256 + threadIdx.x] = block_exclusive_scan<256>(v, sm, tot);
        if (v == n) atomicOr(&cmask, 1ull << p);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long c = cmask;
        *constant_mask = c;
        uint32_t cur = 0;
        for (int d = 0; d < 8; ++d) {
            const bool run = d >= d_begin && d < d_end && !((c >> d) & 1);
            plan[d] = run ? 1 + cur : 0;
            if (run) cur ^= 1;
        }
        plan[8] = cur;
    }
}

// global 256-bin histograms of all 8 byte digits in one read; the last block to finish derives
// the digit offsets and the pass plan (no separate launch)
__global__ void __launch_bounds__(256) radix_hist8_kernel(const uint64_t* keys, uint64_t n, uint32_t* hist,
                                                          uint32_t* base, unsigned long long* constant_mask,
                                                          int d_begin, int d_end, uint32_t* plan,
                                                          uint32_t* done) {
    __shared__ uint32_t h[8][256];
    __shared__ bool last;
    for (int i = threadIdx.x; i < 8 * 256; i += 256) (&h[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += static_cast<uint64_t>(gridDim.x) * 256) {
        const uint64_t k = keys[i];
#pragma unroll
        for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 256; i += 256) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    radix_digit_base_block(hist, n, base, constant_mask, d_begin, d_end, plan);
}

// keys/vals <- alt when the result ended in the alternate buffers (plan[8] == 1)
__global__ void radix_result_copy_kernel(uint64_t* keys, uint32_t* vals, const uint64_t* keys_alt,
                                         const uint32_t* vals_alt, uint64_t n, const uint32_t* plan) {
    if (plan[8] == 0) return;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        keys[i] = keys_alt[i];
        vals[i] = vals_alt[i];
    }
}

// tile keys/values staged in shared memory in digit order before the scatter: each digit's keys
// leave the tile as one contiguous run (coalesced stores instead of one sector per key)
constexpr size_t kOsDynSmem = static_cast<size_t>(kRTile) * (8 + 4);

#ifndef CVLG_OS_MINB
#define CVLG_OS_MINB 3
#endif
// (3 CTAs per SM: 85 registers; unbounded, ptxas took 127 and only 2 CTAs fit, leaving the pass
// latency-bound at 23% issue-active)
__global__ void __launch_bounds__(kRThreads, CVLG_OS_MINB) radix_onesweep_kernel(
    uint64_t* keys_a, uint32_t* vals_a, uint64_t* keys_b, uint32_t* vals_b, uint64_t n, int shift,
    const uint32_t* digit_base, uint32_t* status, uint32_t* tile_counter, const uint32_t* plan) {
    const uint32_t pl = plan[shift / 8];
    if (pl == 0) return;  // constant digit: order unchanged, pass skipped
    const uint64_t* keys_in = pl == 1 ? keys_a : keys_b;
    const uint32_t* vals_in = pl == 1 ? vals_a : vals_b;
    uint64_t* keys_out = pl == 1 ? keys_b : keys_a;
    uint32_t* vals_out = pl == 1 ? vals_b : vals_a;
    extern __shared__ __align__(16) uint8_t os_smem[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(os_smem);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kRTile);
    __shared__ uint32_t wc[kRWarps][256];
    __shared__ uint32_t tile_off[256];  // global position of the tile's first key of each digit
    __shared__ uint32_t dstart[256];    // tile-local position of that key
    __shared__ uint32_t scan_sm[kRWarps + 1];
    __shared__ uint32_t s_tile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = threadIdx.x; i < kRWarps * 256; i += kRThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t tile0 = static_cast<uint64_t>(tile) * kRTile;
    const uint64_t base = tile0 + static_cast<uint64_t>(warp) * kRWarpKeys;
    const uint32_t tile_n = static_cast<uint32_t>(n - tile0 < kRTile ? n - tile0 : kRTile);
    uint64_t k[kRItems];
    uint32_t v[kRItems];
    uint32_t rank[kRItems];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * 32 + lane;
        const bool valid = idx < n;
        k[i] = valid ? keys_in[idx] : 0ull;
        v[i] = valid ? vals_in[idx] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * 32 + lane;
        const bool valid = idx < n;
        const uint32_t d = valid ? (static_cast<uint32_t>(k[i] >> shift) & 0xFFu) : 256u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        // the peer group's leader reserves its ranks with one shared-memory atomic; the returned
        // count is not needed before the next item's reservation, so the items of a thread do
        // not form a read-modify-write chain through the counters
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (valid && lane == leader) old = atomicAdd(&wc[warp][d], static_cast<uint32_t>(__popc(peers)));
        rank[i] = __shfl_sync(0xFFFFFFFFu, old, leader) + __popc(peers & lt);
    }
    __syncthreads();
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRWarps; ++w) {
            const uint32_t t = wc[w][d];
            wc[w][d] = run;
            run += t;
        }
        volatile uint32_t* st = status;
        const uint64_t me = static_cast<uint64_t>(tile) * 256 + d;
        uint32_t excl = 0;
        if (tile == 0) {
            st[me] = kOsInc | run;
        } else {
            st[me] = kOsAgg | run;
            for (int64_t t = static_cast<int64_t>(tile) - 1; t >= 0; --t) {
                uint32_t w;
                do {
                    w = st[static_cast<uint64_t>(t) * 256 + d];
                } while ((w & ~kOsMask) == 0);
                excl += w & kOsMask;
                if ((w & ~kOsMask) == kOsInc) break;
            }
            st[me] = kOsInc | (excl + run);
        }
        uint32_t tot;
        const uint32_t ds = block_exclusive_scan<kRThreads>(run, scan_sm, tot);
        dstart[d] = ds;
        tile_off[d] = digit_base[d] + excl;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRItems; ++i) {
        const uint64_t idx = base + static_cast<uint64_t>(i) * 32 + lane;
        if (idx < n) {
            const uint32_t d = static_cast<uint32_t>(k[i] >> shift) & 0xFFu;
            const uint32_t lp = dstart[d] + wc[warp][d] + rank[i];
            sk[lp] = k[i];
            sv[lp] = v[i];
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tile_n; j += kRThreads) {
        const uint64_t key = sk[j];
        const uint32_t d = static_cast<uint32_t>(key >> shift) & 0xFFu;
        const uint64_t pos = static_cast<uint64_t>(tile_off[d]) + (j - dstart[d]);
        keys_out[pos] = key;
        vals_out[pos] = sv[j];
    }
}

__global__ void key_or_and_kernel(const uint64_t* keys, uint64_t n, unsigned long long* acc) {
    uint64_t o = 0, a = ~0ull;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        o |= keys[i];
        a &= keys[i];
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        o |= __shfl_xor_sync(0xFFFFFFFFu, o, s);
        a &= __shfl_xor_sync(0xFFFFFFFFu, a, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&acc[0], o);
        atomicAnd(&acc[1], a);
    }
}

}  // namespace

uint64_t scan_temp_words(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 2; }

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* d_total,
                        uint32_t* d_tmp, cudaStream_t s) {
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 0) {
        if (d_total) cudaMemsetAsync(d_total, 0, 4, s);
        return;
    }
    scan_reduce_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, d_tmp);
    count_launch();
    scan_partials_kernel<<<1, 1024, 0, s>>>(d_tmp, nb, d_total);
    count_launch();
    scan_down_kernel<<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, out, n, d_tmp);
    count_launch();
}

uint64_t radix_temp_bytes(uint64_t n) {
    const uint64_t tiles = (n + kRTile - 1) / kRTile;
    const uint64_t counts = 256 * tiles;
    const uint64_t legacy = (counts + scan_temp_words(counts) + 16) * 4 + 64;
    const uint64_t onesweep = (2 * 8 * 256 + 2 + 8 + 16 + 8 * counts) * 4 + 64;  // hist, base, mask, counters, plan, status
    return std::max(legacy, onesweep);
}

void radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                      uint64_t n, int begin_bit, int end_bit, void* d_tmp, cudaStream_t s,
                      unsigned long long* d_orand, unsigned long long* h_orand, bool* in_alt) {
    if (in_alt) *in_alt = false;
    if (n <= 1 || end_bit <= begin_bit) return;
    if (n < (1ull << 30) && d_orand && h_orand) {  // one-sweep passes, planned on the device
        const uint32_t n_tiles = static_cast<uint32_t>((n + kRTile - 1) / kRTile);
        uint32_t* hist = static_cast<uint32_t*>(d_tmp);
        uint32_t* dbase = hist + 8 * 256;
        unsigned long long* cmask = reinterpret_cast<unsigned long long*>(dbase + 8 * 256);
        uint32_t* counters = reinterpret_cast<uint32_t*>(cmask + 1);  // 8
        uint32_t* plan = counters + 8;                                // 9 (+ pad to 16)
        uint32_t* status = plan + 16;                                 // [digit][n_tiles][256]
        const int d_begin = begin_bit / 8, d_end = std::min(8, (end_bit + 7) / 8);
        uint32_t* done = plan + 15;  // (plan uses 9 of its 16 words)
        cudaMemsetAsync(hist, 0, (2 * 8 * 256 + 2 + 8 + 16) * 4, s);
        cudaMemsetAsync(status + static_cast<uint64_t>(d_begin) * n_tiles * 256, 0,
                        static_cast<uint64_t>(d_end - d_begin) * n_tiles * 256 * 4, s);
        const unsigned hb = static_cast<unsigned>(std::min<uint64_t>((n + 4095) / 4096, 148 * 4));
        radix_hist8_kernel<<<hb, 256, 0, s>>>(keys, n, hist, dbase, cmask, d_begin, d_end, plan, done);
        count_launch();
        per_device(kPdOnesweepAttr, [] {
            cudaFuncSetAttribute(radix_onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kOsDynSmem));
            return 1;
        });
        for (int d = d_begin; d < d_end; ++d) {
            radix_onesweep_kernel<<<n_tiles, kRThreads, kOsDynSmem, s>>>(
                keys, vals, keys_alt, vals_alt, n, 8 * d, dbase + d * 256,
                status + static_cast<uint64_t>(d) * n_tiles * 256, counters + d, plan);
            count_launch();
        }
        if (in_alt && h_orand) {  // the caller swaps buffers instead of a copy pass
            cudaMemcpyAsync(h_orand, plan + 8, 4, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            *in_alt = *reinterpret_cast<const uint32_t*>(h_orand) != 0;
            return;
        }
        radix_result_copy_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8)), 256, 0, s>>>(
            keys, vals, keys_alt, vals_alt, n, plan);
        count_launch();
        return;
    }
    // constant-digit detection
    uint64_t diff = ~0ull;
    if (d_orand && h_orand) {
        const unsigned long long init[2] = {0ull, ~0ull};
        cudaMemcpyAsync(d_orand, init, 16, cudaMemcpyHostToDevice, s);
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 2048));
        key_or_and_kernel<<<blocks, 256, 0, s>>>(keys, n, d_orand);
        count_launch();
        cudaMemcpyAsync(h_orand, d_orand, 16, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        diff = h_orand[0] ^ h_orand[1];
    }
    const uint32_t n_tiles = static_cast<uint32_t>((n + kRTile - 1) / kRTile);
    const uint64_t n_counts = 256ull * n_tiles;
    uint32_t* counts = static_cast<uint32_t*>(d_tmp);
    uint32_t* scan_tmp = counts + n_counts;
    uint64_t* ki = keys;
    uint32_t* vi = vals;
    uint64_t* ko = keys_alt;
    uint32_t* vo = vals_alt;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        if (((diff >> shift) & 0xFFull) == 0) continue;  // digit constant: order unchanged
        radix_hist_kernel<<<n_tiles, kRThreads, 0, s>>>(ki, n, shift, counts, n_tiles);
        count_launch();
        exclusive_scan_u32(counts, counts, n_counts, nullptr, scan_tmp, s);
        radix_scatter_kernel<<<n_tiles, kRThreads, 0, s>>>(ki, vi, ko, vo, n, shift, counts,
                                                           n_tiles);
        count_launch();
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    if (ki != keys) {
        cudaMemcpyAsync(keys, ki, n * 8, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(vals, vi, n * 4, cudaMemcpyDeviceToDevice, s);
    }
}

}  // namespace cvlg
