// Multi-GPU data plane kernels (route_api.cuh): journey-hash routing of CSV data lines and the
// time-slab partition of the per-cell combine's tuples.
//
// Line routing mirrors the reference's parse-then-route loop (proj/src/aggregate.cpp:418-438):
// the reference parses each line (ingest.cpp:119-157) and pushes the record to
// journey_hash(journey_id) % P (ingest.cpp:287-291). A line's partition depends only on its
// trimmed journey_id field, so it is computed here from the raw bytes; lines the reference would
// reject go wherever the hash of their (possibly empty) id field sends them: the owner counts the
// rejection exactly like a single GPU would, and the counts add up.
//
// Both routing passes stage a 16 KB tile (+ 256 B halo) of one piece in shared memory with 16-byte
// loads, build '\n' and ',' bitmaps by SWAR, and give each thread the lines starting in its 64
// bytes. The count pass sums line bytes per owner; the scatter pass re-derives the same lines,
// turns per-thread byte counts into stream offsets (one multi-owner block scan) and copies each
// line warp-cooperatively (32 consecutive bytes per store instruction) into the owner's stream —
// a peer GPU's receive buffer when the driver hands in peer pointers, so the exchange happens
// inside the scatter (NVLink stores) instead of in a separate all-to-all.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "fastparse.cuh"
#include "route_api.cuh"
#include "sort_api.cuh"

namespace cvlg {
namespace {

constexpr int kRStage = kRouteTile + kRouteHalo + 16;  // staged bytes incl. the alignment lead
constexpr int kRWords = (kRStage + 31) / 32;             // bitmap words
constexpr int kRNW = kRouteThreads / 32;

struct RouteSmem {
    alignas(16) uint8_t buf[kRWords * 32 + 32];
    uint32_t nl[kRWords + 4];
    uint32_t cm[kRWords + 4];
    uint32_t off[kMaxOwners][kRouteThreads];  // per-thread routed bytes, then stream offsets
    uint32_t wsum[kMaxOwners][kRNW];
    uint32_t tot[kMaxOwners];
    unsigned long long lines[kMaxOwners];
    uint32_t piece;
};

// 64 bits of a bitmap starting at bit `pos` (bits past the words read as 0).
__device__ __forceinline__ uint64_t bits64_at(const uint32_t* bm, uint32_t pos) {
    const uint32_t w = pos >> 5, s = pos & 31;
    const uint32_t a = bm[w], b = bm[w + 1], c = bm[w + 2];
    const uint32_t lo = __funnelshift_r(a, b, s), hi = __funnelshift_r(b, c, s);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// First set bit at position >= pos in [pos, limit) of a bitmap; limit if none.
__device__ __forceinline__ uint32_t next_bit(const uint32_t* bm, uint32_t pos, uint32_t limit) {
    while (pos < limit) {
        const uint32_t w = pos >> 5;
        const uint32_t m = bm[w] >> (pos & 31);
        if (m) {
            const uint32_t r = pos + __ffs(m) - 1;
            return r < limit ? r : limit;
        }
        pos = (w + 1) << 5;
    }
    return limit;
}

struct LineInfo {
    uint64_t q;      // absolute start
    uint32_t len;    // bytes to copy: content + '\n' (appended when the piece ends without one)
    uint32_t owner;  // kMaxOwners: not a data line (empty / "\r" only)
};

struct TileCtx {
    const uint8_t* in;
    const uint8_t* buf;
    uint64_t base;   // absolute offset of buf[0]
    uint32_t send;   // staged bytes in buf
    uint64_t pe;     // piece end (absolute)
    int32_t id_col;
    uint32_t n_owners;

    __device__ __forceinline__ uint8_t byte(uint64_t a) const {
        const uint64_t r = a - base;
        return r < send ? buf[r] : in[a];
    }
};

// The line starting at buf position q: its end, whether it is a data line (read_shard,
// ingest.cpp:203-233: one trailing '\r' stripped, empty lines skipped), and the owner of its
// trimmed journey_id field (split_fields / trim, ingest.cpp:31-53).
__device__ LineInfo line_at(const TileCtx& T, const uint32_t* nl, const uint32_t* cm, uint32_t q,
                            uint32_t* error) {
    LineInfo li;
    li.q = T.base + q;
    // line end: first '\n' at or after q, staged bitmap first, then global bytes
    uint32_t e = next_bit(nl, q, T.send);
    uint64_t e_abs = T.base + e;
    if (e == T.send) {
        e_abs = T.base + T.send;
        while (e_abs < T.pe && T.in[e_abs] != '\n') ++e_abs;
    }
    const uint64_t L = e_abs - li.q;  // content bytes (the '\n' excluded)
    if (L + 1 >= (1ull << 31)) {
        atomicExch(error, 1u);
        li.len = 0;
        li.owner = kMaxOwners;
        return li;
    }
    li.len = static_cast<uint32_t>(L + 1);
    if (L == 0 || (L == 1 && T.byte(li.q) == '\r')) {
        li.owner = kMaxOwners;
        return li;
    }
    // the line as parsed: one trailing '\r' removed (next_line, ingest.cpp:208)
    const uint64_t end = T.byte(e_abs - 1) == '\r' ? e_abs - 1 : e_abs;
    // field id_col: after id_col commas
    uint64_t fs = li.q;
    bool present = true;
    for (int32_t k = 0; k < T.id_col; ++k) {
        uint64_t c;
        const uint64_t rel = fs - T.base;
        if (rel < T.send) {
            const uint32_t cb = next_bit(cm, static_cast<uint32_t>(rel), T.send);
            c = T.base + cb;
            if (cb == T.send) {
                c = T.base + T.send;
                while (c < end && T.in[c] != ',') ++c;
            }
        } else {
            c = fs;
            while (c < end && T.in[c] != ',') ++c;
        }
        if (c >= end) {
            present = false;
            break;
        }
        fs = c + 1;
    }
    uint64_t h = 1469598103934665603ull;  // journey_hash (ingest.cpp:287-291) of the trimmed field
    if (present) {
        uint64_t fe;
        const uint64_t rel = fs - T.base;
        if (rel < T.send) {
            const uint32_t cb = next_bit(cm, static_cast<uint32_t>(rel), T.send);
            fe = T.base + cb;
            if (cb == T.send) {
                fe = T.base + T.send;
                while (fe < end && T.in[fe] != ',') ++fe;
            }
        } else {
            fe = fs;
            while (fe < end && T.in[fe] != ',') ++fe;
        }
        if (fe > end) fe = end;
        while (fs < fe && is_trim(T.byte(fs))) ++fs;
        while (fe > fs && is_trim(T.byte(fe - 1))) --fe;
        for (uint64_t a = fs; a < fe; ++a) h = (h ^ T.byte(a)) * 1099511628211ull;
    }
    li.owner = static_cast<uint32_t>(h % T.n_owners);
    return li;
}

template <bool kScatter>
__global__ void __launch_bounds__(kRouteThreads) route_kernel(RouteParams P) {
    __shared__ RouteSmem S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N = P.n_owners;
    if (tid < kMaxOwners) S.lines[tid] = 0;
    for (uint32_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        if (tid == 0) {
            uint32_t lo = 0, hi = P.n_pieces;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) / 2;
                if (P.tile_first[mid] <= t) lo = mid;
                else hi = mid;
            }
            S.piece = lo;
        }
        __syncthreads();
        const uint32_t p = S.piece;
        const uint64_t ps = P.piece_off[p], pe = P.piece_off[p + 1];
        const uint64_t tb = ps + static_cast<uint64_t>(t - P.tile_first[p]) * kRouteTile;
        const uint32_t tlen = static_cast<uint32_t>(pe - tb < kRouteTile ? pe - tb : kRouteTile);
        const uint64_t base = tb & ~15ull;
        const uint32_t lead = static_cast<uint32_t>(tb - base);
        const uint64_t stage_end = tb + kRouteTile + kRouteHalo < pe ? tb + kRouteTile + kRouteHalo : pe;
        const uint32_t send = static_cast<uint32_t>(stage_end - base);

        // ---- stage [base, stage_end) with 16-byte loads; zero the rest of the buffer ------------
        for (uint32_t v = tid; v < kRWords * 2 + 2; v += kRouteThreads) {
            const uint32_t o = v * 16;
            uint4 x = make_uint4(0, 0, 0, 0);
            if (o < send) {
                x = *reinterpret_cast<const uint4*>(P.in + base + o);
                if (o + 16 > send) {
                    uint8_t* b = reinterpret_cast<uint8_t*>(&x);
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (o + k >= send) b[k] = 0;
                }
            }
            *reinterpret_cast<uint4*>(S.buf + o) = x;
        }
        for (int o = tid; o < kMaxOwners * kRouteThreads; o += kRouteThreads) (&S.off[0][0])[o] = 0;
        __syncthreads();
        for (int w = tid; w < kRWords; w += kRouteThreads) {
            const uint32_t* x = reinterpret_cast<const uint32_t*>(S.buf + 32 * w);
            uint32_t xs[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) xs[k] = x[k];
            uint32_t mn, mc;
            class_masks32(xs, mn, mc);
            S.nl[w] = mn;
            S.cm[w] = mc;
        }
        if (tid < 4) {
            S.nl[kRWords + tid] = 0;
            S.cm[kRWords + tid] = 0;
        }
        __syncthreads();

        // ---- line starts in this thread's 64 bytes of the tile ----------------------------------
        TileCtx T{P.in, S.buf, base, send, pe, P.id_col[p], N};
        const uint32_t r0 = 64u * tid;  // tile-relative
        uint64_t starts = 0;
        if (r0 < tlen) {
            const uint32_t q0 = lead + r0;
            if (q0 >= 1) starts = bits64_at(S.nl, q0 - 1);
            else starts = bits64_at(S.nl, 0) << 1;
            if (tid == 0) {
                const bool first = tb == ps;
                const bool s0 = first || (lead ? S.buf[lead - 1] == '\n' : P.in[tb - 1] == '\n');
                starts = (starts & ~1ull) | (s0 ? 1ull : 0ull);
            }
            const uint32_t n = tlen - r0;
            if (n < 64) starts &= (1ull << n) - 1;
        }

        // ---- count pass: bytes per owner ---------------------------------------------------------
        {
            uint64_t m = starts;
            while (m) {
                const int i = __ffsll(static_cast<long long>(m)) - 1;
                m &= m - 1;
                const LineInfo li = line_at(T, S.nl, S.cm, lead + r0 + i, P.error);
                if (li.owner < kMaxOwners) {
                    S.off[li.owner][tid] += li.len;
                    if (!kScatter) atomicAdd(&S.lines[li.owner], 1ull);
                }
            }
        }
        // ---- per-owner block scan: thread offsets within the tile, tile totals --------------------
        for (uint32_t o = 0; o < N; ++o) {
            const uint32_t v = S.off[o][tid];
            const uint32_t inc = warp_inclusive_sum(v);
            if (lane == 31) S.wsum[o][warp] = inc;
            S.off[o][tid] = inc - v;
        }
        __syncthreads();
        if (tid < static_cast<int>(N)) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kRNW; ++w) {
                const uint32_t x = S.wsum[tid][w];
                S.wsum[tid][w] = run;
                run += x;
            }
            S.tot[tid] = run;
        }
        __syncthreads();
        if (!kScatter) {
            if (tid < static_cast<int>(N)) P.tile_bytes[static_cast<uint64_t>(t) * N + tid] = S.tot[tid];
        } else {
            for (uint32_t o = 0; o < N; ++o) S.off[o][tid] += S.wsum[o][warp];
            __syncwarp();
            // ---- scatter: the warp copies its lanes' lines one at a time, 32 bytes per store ------
            uint64_t m = starts;
            bool pending = false;
            LineInfo cur{0, 0, kMaxOwners};
            uint64_t dst = 0;
            while (true) {
                while (!pending && m) {
                    const int i = __ffsll(static_cast<long long>(m)) - 1;
                    m &= m - 1;
                    cur = line_at(T, S.nl, S.cm, lead + r0 + i, P.error);
                    if (cur.owner < kMaxOwners) {
                        const uint32_t o = cur.owner;
                        dst = reinterpret_cast<uint64_t>(P.dst[o]) +
                              P.tile_base[static_cast<uint64_t>(t) * N + o] + S.off[o][tid];
                        S.off[o][tid] += cur.len;
                        pending = true;
                    }
                }
                const uint32_t want = __ballot_sync(0xFFFFFFFFu, pending);
                if (!want) break;
                const int leader = __ffs(want) - 1;
                const uint64_t q = __shfl_sync(0xFFFFFFFFu, cur.q, leader);
                const uint32_t len = __shfl_sync(0xFFFFFFFFu, cur.len, leader);
                uint8_t* d = reinterpret_cast<uint8_t*>(__shfl_sync(0xFFFFFFFFu, dst, leader));
                for (uint32_t k = lane; k < len; k += 32) d[k] = k + 1 < len ? T.byte(q + k) : uint8_t('\n');
                if (lane == leader) pending = false;
            }
        }
        __syncthreads();
    }
    if (!kScatter && P.lines && tid < static_cast<int>(N) && S.lines[tid])
        atomicAdd(&P.lines[tid], S.lines[tid]);
}

// One block per owner: exclusive scan of the tiles' byte counts (u64 carry across chunks).
__global__ void __launch_bounds__(1024) route_scan_kernel(const uint32_t* tile_bytes, uint32_t n_tiles,
                                                          uint32_t N, const uint32_t* tile_first,
                                                          uint32_t n_pieces, const uint64_t* hdr_off,
                                                          uint64_t* tile_base, uint64_t* piece_obase,
                                                          uint64_t* owner_total) {
    __shared__ unsigned long long smem[33];
    const uint32_t o = blockIdx.x;
    unsigned long long carry = 0;
    for (uint32_t c0 = 0; c0 < n_tiles; c0 += 1024) {
        const uint32_t t = c0 + threadIdx.x;
        const unsigned long long v = t < n_tiles ? tile_bytes[static_cast<uint64_t>(t) * N + o] : 0ull;
        unsigned long long total;
        const unsigned long long ex = block_exclusive_scan<1024>(v, smem, total);
        if (t < n_tiles) {
            uint32_t lo = 0, hi = n_pieces;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) / 2;
                if (tile_first[mid] <= t) lo = mid;
                else hi = mid;
            }
            tile_base[static_cast<uint64_t>(t) * N + o] = carry + ex + hdr_off[lo + 1];
            if (tile_first[lo] == t) piece_obase[static_cast<uint64_t>(lo) * N + o] = carry + ex;
        }
        carry += total;
    }
    if (threadIdx.x == 0) owner_total[o] = carry;
}

__global__ void route_headers_kernel(const uint8_t* hdr, const uint64_t* hdr_off, uint32_t n_pieces,
                                     const uint64_t* piece_obase, uint32_t N, uint8_t* const* dst) {
    const uint32_t p = blockIdx.x;
    if (p >= n_pieces) return;
    const uint64_t a = hdr_off[p], len = hdr_off[p + 1] - a;
    for (uint32_t o = 0; o < N; ++o) {
        uint8_t* d = dst[o] + a + piece_obase[static_cast<uint64_t>(p) * N + o];
        for (uint64_t k = threadIdx.x; k < len; k += blockDim.x) d[k] = hdr[a + k];
    }
}

__device__ __forceinline__ uint32_t tuple_owner(uint64_t cell, uint64_t cells_per_t, uint32_t T,
                                                uint32_t N) {
    const uint64_t t = cell / cells_per_t;
    const uint64_t o = t * N / T;
    return static_cast<uint32_t>(o < N ? o : N - 1);
}

__global__ void tuple_count_kernel(const PairTuple* tu, uint64_t n, uint64_t cells_per_t,
                                   uint32_t T, uint32_t N, unsigned long long* counts) {
    __shared__ unsigned long long c[kMaxOwners];
    if (threadIdx.x < kMaxOwners) c[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(&c[tuple_owner(tu[i].cell, cells_per_t, T, N)], 1ull);
    __syncthreads();
    if (threadIdx.x < N && c[threadIdx.x]) atomicAdd(&counts[threadIdx.x], c[threadIdx.x]);
}

__global__ void tuple_scatter_kernel(const PairTuple* tu, uint64_t n, uint64_t cells_per_t,
                                     uint32_t T, uint32_t N, unsigned long long* cursors,
                                     PairTuple* const* dst) {
    const int lane = threadIdx.x & 31;
    for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x);
         i0 < n; i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        PairTuple x{};
        uint32_t o = kMaxOwners;
        if (ok) {
            x = tu[i];
            o = tuple_owner(x.cell, cells_per_t, T, N);
        }
        // warp-aggregated reservation per owner (tuple order within an owner is irrelevant: the
        // owner sorts by (cell, journey key), which is unique)
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, o);
        const int leader = __ffs(peers) - 1;
        unsigned long long b = 0;
        if (ok && lane == leader) b = atomicAdd(&cursors[o], static_cast<unsigned long long>(__popc(peers)));
        b = __shfl_sync(0xFFFFFFFFu, b, leader);
        if (ok) dst[o][b + __popc(peers & ((1u << lane) - 1u))] = x;
    }
}

int sm_count() {
    int d = 0, v = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
}

unsigned route_grid(uint32_t n_tiles) {
    const uint64_t g = static_cast<uint64_t>(per_device(kPdSms, sm_count)) * 4;
    return static_cast<unsigned>(std::min<uint64_t>(g, std::max<uint32_t>(n_tiles, 1)));
}

}  // namespace

void launch_route_count(const RouteParams& p, cudaStream_t s) {
    if (!p.n_tiles) return;
    route_kernel<false><<<route_grid(p.n_tiles), kRouteThreads, 0, s>>>(p);
    count_launch();
}

void launch_route_scatter(const RouteParams& p, cudaStream_t s) {
    if (!p.n_tiles) return;
    route_kernel<true><<<route_grid(p.n_tiles), kRouteThreads, 0, s>>>(p);
    count_launch();
}

void launch_route_scan(const uint32_t* tile_bytes, uint32_t n_tiles, uint32_t n_owners,
                       const uint32_t* tile_first, uint32_t n_pieces, const uint64_t* hdr_off,
                       uint64_t* tile_base, uint64_t* piece_obase, uint64_t* owner_total,
                       cudaStream_t s) {
    route_scan_kernel<<<n_owners, 1024, 0, s>>>(tile_bytes, n_tiles, n_owners, tile_first, n_pieces,
                                                hdr_off, tile_base, piece_obase, owner_total);
    count_launch();
}

void launch_route_headers(const uint8_t* hdr, const uint64_t* hdr_off, uint32_t n_pieces,
                          const uint64_t* piece_obase, uint32_t n_owners, uint8_t* const* dst,
                          cudaStream_t s) {
    if (!n_pieces) return;
    route_headers_kernel<<<n_pieces, 128, 0, s>>>(hdr, hdr_off, n_pieces, piece_obase, n_owners, dst);
    count_launch();
}

void launch_tuple_count(const PairTuple* t, uint64_t n, uint64_t cells_per_t, uint32_t n_batches,
                        uint32_t n_owners, unsigned long long* counts, cudaStream_t s) {
    if (!n) return;
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
    tuple_count_kernel<<<g, 256, 0, s>>>(t, n, cells_per_t, n_batches, n_owners, counts);
    count_launch();
}

void launch_tuple_scatter(const PairTuple* t, uint64_t n, uint64_t cells_per_t, uint32_t n_batches,
                          uint32_t n_owners, unsigned long long* cursors, PairTuple* const* dst,
                          cudaStream_t s) {
    if (!n) return;
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
    tuple_scatter_kernel<<<g, 256, 0, s>>>(t, n, cells_per_t, n_batches, n_owners, cursors, dst);
    count_launch();
}

}  // namespace cvlg
