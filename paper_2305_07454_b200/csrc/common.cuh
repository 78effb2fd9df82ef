// Device utilities shared by the sm_100a kernels: relaxed/acquire memory helpers and warp/block
// scans.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cvlg {

constexpr int kWarp = 32;

// Launch facts that live in each device's context (the >48 KB shared-memory opt-in, SM count,
// occupancy): computed once per (device, key) under a lock by `compute`, which runs with that
// device current. Defined in pipeline.cu.
int per_device(int key, int (*compute)());
enum : int { kPdDecodeCtas = 0, kPdSms, kPdFoldPerSm0, kPdFoldPerSm1, kPdOnesweepAttr, kPdCount };

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

}  // namespace cvlg
