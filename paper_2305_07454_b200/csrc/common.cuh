// Device utilities shared by the sm_100a kernels: memory-model helpers for decoupled look-back,
// warp/block scans, and the error-code convention of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cvlg {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// Block-wide exclusive scan of one value per thread. `smem` needs NW entries (NW = warps).
// Returns the exclusive prefix; `total` receives the block sum. Contains __syncthreads.
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T& total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < NW ? smem[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < NW) smem[lane] = wi - w;
        if (lane == NW - 1) smem[NW] = wi;
    }
    __syncthreads();
    T res = smem[warp] + inc - v;
    total = smem[NW];
    __syncthreads();
    return res;
}

// Decoupled look-back, single u64 counter, split into publish (as early as possible) and a
// CTA-wide resolve (as late as possible): every thread of the CTA inspects one predecessor, so a
// window of NT tiles is examined per step. flag: 0 = not ready, 1 = aggregate, 2 = inclusive.
struct Lookback1 {
    uint32_t* flag;
    uint64_t* agg;
    uint64_t* inc;
};

__device__ __forceinline__ void lookback1_publish(const Lookback1& st, uint32_t tile, uint64_t a) {
    if (tile == 0) {
        st_relaxed_u64(&st.inc[0], a);
        st_release_u32(&st.flag[0], 2u);
    } else {
        st_relaxed_u64(&st.agg[tile], a);
        st_release_u32(&st.flag[tile], 1u);
    }
}

// All NT threads call. Returns the exclusive prefix of `tile` and publishes its inclusive value.
template <int NT>
__device__ __forceinline__ uint64_t lookback1_resolve(const Lookback1& st, uint32_t tile, uint64_t a,
                                                      uint64_t* smem64 /* NT/32 + 2 */) {
    if (tile == 0) return 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    uint64_t total = 0;
    int64_t j = static_cast<int64_t>(tile) - 1;
    __shared__ int s_stop;
    while (true) {
        const int64_t idx = j - static_cast<int64_t>(threadIdx.x);
        uint32_t f = 2;
        uint64_t v = 0;
        if (idx >= 0) {
            do {
                f = ld_acquire_u32(&st.flag[idx]);
            } while (f == 0);
            v = ld_relaxed_u64(f == 2 ? &st.inc[idx] : &st.agg[idx]);
        }
        // nearest inclusive predecessor = lowest thread index with f == 2
        if (threadIdx.x == 0) s_stop = NT;
        __syncthreads();
        if (f == 2) atomicMin(&s_stop, static_cast<int>(threadIdx.x));
        __syncthreads();
        const int stop = s_stop;
        if (static_cast<int>(threadIdx.x) > stop) v = 0;
        v = warp_sum(v);
        if (lane == 0) smem64[warp] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t s = 0;
            for (int w = 0; w < NW; ++w) s += smem64[w];
            smem64[NW] = s;
        }
        __syncthreads();
        total += smem64[NW];
        __syncthreads();
        if (stop < NT) break;
        j -= NT;
    }
    if (threadIdx.x == 0) {
        st_relaxed_u64(&st.inc[tile], total + a);
        st_release_u32(&st.flag[tile], 2u);
    }
    return total;
}

// CTA-wide look-back without publishing: the exclusive prefix of `tile` over tiles < tile.
// Each thread inspects one predecessor per step (window of NT tiles); warps combine with ballots
// (nearest inclusive predecessor = first lane with flag 2), one barrier per step. `sm` / `smf`
// hold 2 * (NT / 32) entries (double-buffered by step parity); callers separate two calls with a
// barrier. All NT threads call.
template <int NT>
__device__ __forceinline__ uint64_t lookback_exclusive(const Lookback1& st, uint32_t tile, uint64_t* sm,
                                                       uint32_t* smf) {
    if (tile == 0) return 0;
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t total = 0;
    int64_t j = static_cast<int64_t>(tile) - 1;
    for (int step = 0;; ++step) {
        uint64_t* bv = sm + (step & 1) * NW;
        uint32_t* bf = smf + (step & 1) * NW;
        const int64_t idx = j - static_cast<int64_t>(threadIdx.x);
        uint32_t f = 2;
        uint64_t v = 0;
        if (idx >= 0) {
            do {
                f = ld_acquire_u32(&st.flag[idx]);
            } while (f == 0);
            v = ld_relaxed_u64(f == 2 ? &st.inc[idx] : &st.agg[idx]);
        }
        const uint32_t done = __ballot_sync(0xFFFFFFFFu, f == 2);
        const int stop = done ? __ffs(done) - 1 : 32;
        v = warp_sum(lane <= stop ? v : 0ull);
        // per warp: sum up to (and including) its first inclusive lane
        if (lane == 0) {
            bv[warp] = v;
            bf[warp] = done != 0;
        }
        __syncthreads();
        bool stopped = false;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            if (!stopped) total += bv[w];
            stopped = stopped || bf[w];
        }
        if (stopped) break;
        j -= NT;
    }
    return total;
}

__device__ __forceinline__ void lookback_publish_inclusive(const Lookback1& st, uint32_t tile, uint64_t v) {
    st_relaxed_u64(&st.inc[tile], v);
    st_release_u32(&st.flag[tile], 2u);
}

// Decoupled look-back state for a scan over tiles carrying two u64 counters.
// flag: 0 = not ready, 1 = aggregate published, 2 = inclusive prefix published.
struct LookbackState {
    uint32_t* flag;
    uint64_t* agg;  // [2 * tiles]
    uint64_t* inc;  // [2 * tiles]
};

// Called by all threads of warp 0 of the tile's CTA. Returns the exclusive prefix (a, b).
__device__ __forceinline__ void lookback_publish_and_scan(const LookbackState& st, uint32_t tile,
                                                          uint64_t a, uint64_t b, uint64_t& ex_a,
                                                          uint64_t& ex_b) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) {
            st_relaxed_u64(&st.inc[0], a);
            st_relaxed_u64(&st.inc[1], b);
            st_release_u32(&st.flag[0], 2u);
        }
        ex_a = 0;
        ex_b = 0;
        return;
    }
    if (lane == 0) {
        st_relaxed_u64(&st.agg[2 * tile], a);
        st_relaxed_u64(&st.agg[2 * tile + 1], b);
        st_release_u32(&st.flag[tile], 1u);
    }
    uint64_t sa = 0, sb = 0;
    int64_t j = static_cast<int64_t>(tile) - 1;
    while (true) {
        const int64_t idx = j - lane;
        uint32_t f = 2;
        if (idx >= 0) {
            do {
                f = ld_acquire_u32(&st.flag[idx]);
            } while (f == 0);
        }
        uint64_t va = 0, vb = 0;
        if (idx >= 0) {
            const uint64_t* src = (f == 2) ? st.inc : st.agg;
            va = ld_relaxed_u64(&src[2 * idx]);
            vb = ld_relaxed_u64(&src[2 * idx + 1]);
        }
        const uint32_t done = __ballot_sync(0xFFFFFFFFu, f == 2);
        const int stop = done ? (__ffs(done) - 1) : 32;
        if (lane > stop) {
            va = 0;
            vb = 0;
        }
        sa += warp_sum(va);
        sb += warp_sum(vb);
        if (done) break;
        j -= 32;
    }
    if (lane == 0) {
        st_relaxed_u64(&st.inc[2 * tile], sa + a);
        st_relaxed_u64(&st.inc[2 * tile + 1], sb + b);
        st_release_u32(&st.flag[tile], 2u);
    }
    ex_a = sa;
    ex_b = sb;
}

}  // namespace cvlg
