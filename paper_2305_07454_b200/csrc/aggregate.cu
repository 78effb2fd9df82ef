// Journey dictionary, canonical (journey, timestamp) ordering, dedup, per-(cell, journey) fold
// and the canonical per-cell finalize, for sm_100a.
//
// Reference semantics restated here (proj/src/aggregate.cpp):
//   dedup on (journey, epoch) with min-provenance survivor       :266-291
//   filter_reason on survivors                                   :293-303
//   journey ids -> lexicographic ranks, items sorted (rank, sec)  :305-328
//   cellmap[(g, rank)] += speed in (rank, sec) order              :331-358
//   finalize: sort by (g, journey), fold subtotals in journey order, f32 narrow :161-204
#include <algorithm>
#include <climits>

#include "agg_api.cuh"
#include "kernels.cuh"
#include "sort_api.cuh"

namespace cvlg {

namespace {

constexpr uint64_t kEmpty = ~0ull;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint64_t kDeadPair = ~0ull;  // pair slot vacated by a window reload (compacted away)

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ void cas128(unsigned long long* addr, uint64_t c0, uint64_t c1,
                                       uint64_t v0, uint64_t v1, uint64_t& o0, uint64_t& o1) {
    asm volatile(
        "{\n\t.reg .b128 c, v, d;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(o0), "=l"(o1)
        : "l"(c0), "l"(c1), "l"(v0), "l"(v1), "l"(addr)
        : "memory");
}

__device__ __forceinline__ bool bytes_equal(const uint8_t* a, const uint8_t* b, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i)
        if (a[i] != b[i]) return false;
    return true;
}

__device__ __forceinline__ uint32_t shard_of(const uint64_t* shard_off, uint32_t n_shards,
                                             uint64_t p) {
    uint32_t lo = 0, hi = n_shards;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (shard_off[mid] <= p) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ---- H: dense run-head list from K1's per-tile lists --------------------------------------------
// tiles[t] = (slot base, data lines, head base, heads)
__global__ void tile_field_kernel(const uint4* tiles, uint64_t n, int field, uint32_t* out) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const uint4 v = tiles[t];
    out[t] = field == 0 ? v.x : field == 1 ? v.y : field == 2 ? v.z : v.w;
}

__device__ uint32_t dict_insert_one(const DictParams& D, uint64_t id, ulonglong2 hk);

// heads in tile order (= provenance order for regular tiles); a run ends at the next head of its
// tile or at the tile's last line (runs never cross tiles: a tile's first line is always a head)
// With D.table set, each head's journey id is also inserted into the dictionary on the way
// (hdict at its dense index), so the dense key list is never written or read back.
__global__ void heads_compact_kernel(const uint4* tiles, uint64_t n, const uint32_t* hpos,
                                     const uint32_t* hscr, const uint64_t* hid_scr,
                                     const ulonglong2* hkey_scr, uint32_t* hslot, uint32_t* hend,
                                     uint64_t* hid, ulonglong2* hkey, DictParams D) {
    // one thread per tile (journey-ordered input: a head or two per tile); tiles with many heads
    // (shuffled rows) are copied by the whole warp afterwards
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    uint32_t base = 0;
    if (t < n) {
        v = tiles[t];
        base = hpos[t];
    }
    const bool small = v.w <= 8;
    if (small) {
        for (uint32_t i = 0; i < v.w; ++i) {
            hslot[base + i] = hscr[v.z + i];
            hend[base + i] = i + 1 < v.w ? hscr[v.z + i + 1] : v.x + v.y;
            hid[base + i] = hid_scr[v.z + i];
            if (D.table) D.hdict[base + i] = dict_insert_one(D, hid_scr[v.z + i], hkey_scr[v.z + i]);
            else hkey[base + i] = hkey_scr[v.z + i];
        }
    }
    uint32_t big = __ballot_sync(0xFFFFFFFFu, !small);
    while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const uint32_t x = __shfl_sync(0xFFFFFFFFu, v.x, src), y = __shfl_sync(0xFFFFFFFFu, v.y, src),
                       z = __shfl_sync(0xFFFFFFFFu, v.z, src), w = __shfl_sync(0xFFFFFFFFu, v.w, src);
        const uint32_t bb = __shfl_sync(0xFFFFFFFFu, base, src);
        for (uint32_t i = lane; i < w; i += 32) {
            hslot[bb + i] = hscr[z + i];
            hend[bb + i] = i + 1 < w ? hscr[z + i + 1] : x + y;
            hid[bb + i] = hid_scr[z + i];
            if (D.table) D.hdict[bb + i] = dict_insert_one(D, hid_scr[z + i], hkey_scr[z + i]);
            else hkey[bb + i] = hkey_scr[z + i];
        }
    }
}

// slow path: pack the per-tile slot ranges densely (provenance order), remap the heads
__global__ void densify_kernel(DensifyParams D) {
    const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
    if (t >= D.n_tiles) return;
    const int lane = threadIdx.x & 31;
    const uint4 v = D.tiles[t];
    const uint32_t dst = D.lpos[t];
    long long t_lo = LLONG_MAX, t_hi = LLONG_MIN;  // kept epochs (the slow sort's key range)
    // four rounds of loads in flight before their stores (memory-level parallelism)
    for (uint32_t k0 = lane; k0 < v.y; k0 += 128) {
        int64_t ts[4];
        double sp[4];
        uint32_t cd[4];
        uint64_t lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t k = k0 + 32u * u;
            if (k < v.y) {
                ts[u] = D.ts[v.x + k];
                sp[u] = D.speed[v.x + k];
                cd[u] = D.code[v.x + k];
                lo[u] = D.loff[v.x + k];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t k = k0 + 32u * u;
            if (k < v.y) {
                D.ts_out[dst + k] = ts[u];
                D.speed_out[dst + k] = sp[u];
                D.code_out[dst + k] = cd[u];
                D.loff_out[dst + k] = lo[u];
                if ((cd[u] & kCodeMask) != kCodeRejected) {
                    t_lo = ts[u] < t_lo ? ts[u] : t_lo;
                    t_hi = ts[u] > t_hi ? ts[u] : t_hi;
                }
                if (D.rec_out) {
                    ulonglong2 r;
                    r.x = static_cast<unsigned long long>(__double_as_longlong(sp[u]));
                    r.y = cd[u];
                    D.rec_out[dst + k] = r;
                }
            }
        }
    }
    if (D.ts_mm) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long a = __shfl_xor_sync(0xFFFFFFFFu, t_lo, o), b = __shfl_xor_sync(0xFFFFFFFFu, t_hi, o);
            t_lo = a < t_lo ? a : t_lo;
            t_hi = b > t_hi ? b : t_hi;
        }
        if (lane == 0 && t_lo <= t_hi) {
            atomicMin(&D.ts_mm[0], t_lo);
            atomicMax(&D.ts_mm[1], t_hi);
        }
    }
    if (D.lat) {
        for (uint32_t k = lane; k < v.y; k += 32) {
            D.lat_out[dst + k] = D.lat[v.x + k];
            D.lon_out[dst + k] = D.lon[v.x + k];
        }
    }
    const uint32_t hb = D.hpos[t];
    for (uint32_t i = lane; i < v.w; i += 32) D.hslot_out[hb + i] = dst + (D.hscr[v.z + i] - v.x);
}

// ---- D1: dictionary insert (one thread per run head) -----------------------------------------
// Short ids (<= 15 bytes) are keyed exactly by (bytes 0..7 BE, bytes 8..14 BE << 8 | len);
// longer ids by (FNV-1a high 40 bits | len, offset << 8 | 0xFF) with a byte comparison.
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0u, 0x0123u); }

__device__ uint32_t dict_insert_one(const DictParams& D, uint64_t id, ulonglong2 hk) {
    const uint64_t off = id & ((1ull << 40) - 1);
    const uint32_t len = static_cast<uint32_t>(id >> 40);
    const uint8_t* p = D.csv + off;
    uint64_t e0, e1, slot;
    const bool is_long = len > 15;
    if (hk.y != kNoKey) {  // K1 assembled the key from the staged tile (no CSV gather)
        e0 = hk.x;
        e1 = hk.y;
        slot = mix64(e0 ^ mix64(e1)) & D.mask;
    } else if (!is_long) {
        uint64_t k0 = 0, k1 = 0;
        if (off + 20 <= D.csv_len) {  // 5 aligned words cover bytes [off, off + 16)
            const uint32_t* w = reinterpret_cast<const uint32_t*>(D.csv + (off & ~3ull));
            const uint32_t sh = static_cast<uint32_t>(off & 3) * 8;
            const uint32_t a0 = w[0], a1 = w[1], a2 = w[2], a3 = w[3], a4 = w[4];
            uint32_t b[4] = {__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                             __funnelshift_r(a2, a3, sh), __funnelshift_r(a3, a4, sh)};
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // zero the bytes at index >= len
                const int keep = static_cast<int>(len) - 4 * q;
                b[q] = keep >= 4 ? b[q] : (keep <= 0 ? 0u : (b[q] & (0xFFFFFFFFu >> (8 * (4 - keep)))));
            }
            k0 = (static_cast<uint64_t>(bswap32(b[0])) << 32) | bswap32(b[1]);
            k1 = ((static_cast<uint64_t>(bswap32(b[2])) << 32) | bswap32(b[3])) >> 8;
        } else {
            for (uint32_t i = 0; i < 8; ++i) k0 = (k0 << 8) | (i < len ? p[i] : 0u);
            for (uint32_t i = 8; i < 15; ++i) k1 = (k1 << 8) | (i < len ? p[i] : 0u);
        }
        e0 = k0;
        e1 = (k1 << 8) | len;
        slot = mix64(e0 ^ mix64(e1)) & D.mask;
    } else {
        uint64_t fnv = 1469598103934665603ull;
        for (uint32_t i = 0; i < len; ++i) fnv = (fnv ^ p[i]) * 1099511628211ull;
        e0 = (fnv & ~0xFFFFFFull) | (len & 0xFFFFFFu);
        e1 = (off << 8) | 0xFF;
        slot = mix64(fnv) & D.mask;
    }
    const uint32_t wmax = __reduce_max_sync(__activemask(), len);
    // one atomic per warp, and only while the warp's longest id is longer than what is already
    // recorded: every head of a journey inserts the same id, so the shared maximum is settled by
    // the first warps and later warps only read it (row-shuffled input has a head per line:
    // 1.6M same-address atomics otherwise)
    if (len == wmax && wmax > ld_relaxed_u64(reinterpret_cast<const uint64_t*>(D.max_len))) {
        const uint32_t lanes = __match_any_sync(__activemask(), len);
        if ((threadIdx.x & 31) == __ffs(lanes) - 1) atomicMax(D.max_len, static_cast<unsigned long long>(len));
    }
    const uint64_t max_probe = D.mask < 4096 ? D.mask : 4096;
    for (uint64_t probe = 0;; ++probe) {
        if (probe > max_probe) {  // table too full for this many distinct ids: re-run larger
            atomicOr(D.full, 1u);
            break;
        }
        uint64_t o0, o1;
        // read first: a journey id is inserted by every one of its run heads, and a failing CAS
        // on a hot key is still a serialized read-modify-write at L2. Entries go from empty to
        // their value once (one 128-bit CAS) and never change, so two non-empty halves are
        // consistent; anything else is decided by the CAS itself.
        o1 = ld_relaxed_u64(reinterpret_cast<const uint64_t*>(&D.table[2 * slot + 1]));
        o0 = ld_relaxed_u64(reinterpret_cast<const uint64_t*>(&D.table[2 * slot]));
        if (o0 == kEmpty || o1 == kEmpty)
            cas128(&D.table[2 * slot], kEmpty, kEmpty, e0, e1, o0, o1);
        if (o0 == kEmpty && o1 == kEmpty) break;  // inserted
        if (!is_long) {
            if (o0 == e0 && o1 == e1) break;
        } else if ((o1 & 0xFF) == 0xFF && o0 == e0) {
            if (bytes_equal(D.csv + (o1 >> 8), p, len)) break;
        }
        slot = (slot + 1) & D.mask;
    }
    return static_cast<uint32_t>(slot);
}

__global__ void dict_insert_kernel(DictParams D) {
    const uint64_t h = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (h >= D.n_heads) return;
    D.hdict[h] = dict_insert_one(D, D.hid[h], D.hkey[h]);
}

// ---- D2: occupied slots -> flags for compaction ---------------------------------------------
__global__ void dict_flags_kernel(const unsigned long long* table, uint64_t cap, uint32_t* flags) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= cap) return;
    flags[i] = (table[2 * i] != kEmpty || table[2 * i + 1] != kEmpty) ? 1u : 0u;
}

__global__ void dict_compact_kernel(const uint32_t* flags, const uint32_t* pos, uint64_t cap,
                                    uint32_t* uslot) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= cap || !flags[i]) return;
    uslot[pos[i]] = static_cast<uint32_t>(i);
}

// chunk c (bytes 8c..8c+7, big-endian, zero padded) or the length (c == -1) of unique entry
// perm[i], for the LSD string sort (padded bytes, then length, is std::string order).
__global__ void dict_chunk_kernel(const unsigned long long* table, const uint32_t* uslot,
                                  const uint32_t* perm, uint64_t n, int c, const uint8_t* csv,
                                  uint64_t* keys) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t slot = uslot[perm[i]];
    const uint64_t e0 = table[2 * slot], e1 = table[2 * slot + 1];
    const bool is_long = (e1 & 0xFF) == 0xFF;
    const uint32_t len = is_long ? static_cast<uint32_t>(e0 & 0xFFFFFF) : static_cast<uint32_t>(e1 & 0xFF);
    if (c < 0) {
        keys[i] = len;
        return;
    }
    uint64_t k = 0;
    if (!is_long) {
        if (c == 0) k = e0;
        else if (c == 1) k = (e1 >> 8) << 8;
    } else {
        const uint8_t* p = csv + (e1 >> 8);
        for (uint32_t b = 0; b < 8; ++b) {
            const uint32_t at = 8 * c + b;
            k = (k << 8) | (at < len ? p[at] : 0u);
        }
    }
    keys[i] = k;
}

__global__ void dict_rank_kernel(const uint32_t* uslot, const uint32_t* perm, uint64_t n,
                                 uint32_t* rank_of_slot) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    rank_of_slot[uslot[perm[i]]] = static_cast<uint32_t>(i);
}

__global__ void head_rank_kernel(const uint32_t* hdict, const uint32_t* rank_of_slot, uint64_t n,
                                 uint32_t* hrank) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    hrank[i] = rank_of_slot[hdict[i]];
}

// ---- O1: head sort keys ----------------------------------------------------------------------
__global__ void head_keys_kernel(const uint32_t* hrank, const uint32_t* hslot, const int64_t* ts,
                                 uint64_t n_heads, int64_t ts_min, int tsbits, int mode,
                                 uint64_t* keys, uint32_t* vals) {
    const uint64_t h = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (h >= n_heads) return;
    const uint64_t t = (static_cast<uint64_t>(ts[hslot[h]]) - static_cast<uint64_t>(ts_min));
    // mode 0: (rank << tsbits) | t ; mode 1: t only (then a second pass on rank)
    keys[h] = mode == 0 ? ((static_cast<uint64_t>(hrank[h]) << tsbits) | t) : t;
    vals[h] = static_cast<uint32_t>(h);
}

__global__ void gather_rank_keys_kernel(const uint32_t* rank_src, const uint32_t* vals, uint64_t n,
                                        uint64_t* keys) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    keys[i] = rank_src[vals[i]];
}

// ---- O2: validity of the run-merge order + journey starts ------------------------------------
__global__ void head_order_check_kernel(const uint32_t* perm, const uint32_t* hrank,
                                        const uint32_t* hslot, const uint32_t* hend,
                                        const int64_t* ts, const uint32_t* code, uint64_t n_heads,
                                        uint32_t* jstart, uint32_t* invalid) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n_heads) return;
    const uint32_t h = perm[i];
    const uint32_t r = hrank[h];
    if (i == 0 || hrank[perm[i - 1]] != r) {
        jstart[r] = static_cast<uint32_t>(i);
        return;
    }
    const uint32_t hp = perm[i - 1];
    uint64_t last = hend[hp] - 1;
    while ((code[last] & kCodeMask) == kCodeRejected) --last;  // run head is accepted
    if (!(ts[last] < ts[hslot[h]])) *invalid = 1u;
}

// ---- S: slow path: per-slot journey rank, sort keys ------------------------------------------
__global__ void slot_keys_kernel(const uint32_t* hslot, const uint32_t* hrank, uint64_t n_heads,
                                 const int64_t* ts, const uint32_t* code, uint64_t n_slots,
                                 int64_t ts_min, int tsbits, int mode, uint32_t reject_rank,
                                 uint64_t* keys, uint32_t* vals, uint32_t* srank) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n_slots) return;
    uint32_t r;
    uint64_t t = 0;
    if ((code[i] & kCodeMask) == kCodeRejected || n_heads == 0 || hslot[0] > i) {
        r = reject_rank;  // sorts after every journey and is never folded
    } else {
        uint64_t lo = 0, hi = n_heads;  // run = last head with hslot <= i
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (hslot[mid] <= i) lo = mid;
            else hi = mid;
        }
        r = hrank[lo];
        t = (static_cast<uint64_t>(ts[i]) - static_cast<uint64_t>(ts_min));
    }
    keys[i] = mode == 0 ? ((static_cast<uint64_t>(r) << tsbits) | t) : t;
    vals[i] = static_cast<uint32_t>(i);
    srank[i] = r;
}

// min / max epoch over non-rejected slots (the slow path's combined sort key)
__global__ void ts_range_kernel(const int64_t* ts, const uint32_t* code, uint64_t n, long long* mm) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if ((code[i] & kCodeMask) == kCodeRejected) continue;
        const long long t = ts[i];
        lo = t < lo ? t : lo;
        hi = t > hi ? t : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long a = __shfl_xor_sync(0xFFFFFFFFu, lo, o), b = __shfl_xor_sync(0xFFFFFFFFu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

__global__ void ts_range_init_kernel(long long* mm) {
    mm[0] = LLONG_MAX;
    mm[1] = LLONG_MIN;
}

// Same keys without a search: one thread per run head writes its run's slots (dense layout: a
// run ends at the next head), thread 0 also the slots before the first head (rejected lines).
__global__ void run_keys_kernel(const uint32_t* hslot, const uint32_t* hrank, const uint32_t* hdict,
                                const uint32_t* rank_of_slot, uint64_t n_heads,
                                const int64_t* ts, const uint32_t* code, uint64_t n_slots,
                                int64_t ts_min, int tsbits, int mode, uint32_t reject_rank,
                                uint64_t* keys, uint32_t* vals, uint32_t* srank) {
    const uint64_t h = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (h >= n_heads) return;
    auto put = [&](uint64_t i, uint32_t r) {
        uint64_t t = 0;
        if ((code[i] & kCodeMask) == kCodeRejected) r = reject_rank;
        else t = static_cast<uint64_t>(ts[i]) - static_cast<uint64_t>(ts_min);
        keys[i] = mode == 0 ? ((static_cast<uint64_t>(r) << tsbits) | t) : t;
        vals[i] = static_cast<uint32_t>(i);
        srank[i] = r;
    };
    if (h == 0)
        for (uint64_t i = 0; i < hslot[0]; ++i) put(i, reject_rank);
    const uint64_t end = h + 1 < n_heads ? hslot[h + 1] : n_slots;
    const uint32_t r = hrank ? hrank[h] : rank_of_slot[hdict[h]];
    for (uint64_t i = hslot[h]; i < end; ++i) put(i, r);
}

// journey starts from the sorted keys: the rank is key >> rank_shift (no gather through perm)
__global__ void slot_jstart_kernel(const uint64_t* keys, int rank_shift, uint64_t n, uint32_t* jstart) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = static_cast<uint32_t>(keys[i] >> rank_shift);
    if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> rank_shift) != r) jstart[r] = static_cast<uint32_t>(i);
}

// ---- payload re-parse for the duplicate-conflict check (aggregate.cpp:286) -------------------
__device__ bool parse_at(const FoldParams& P, uint64_t loff, Parsed& pr, const uint8_t*& line) {
    const uint32_t s = shard_of(P.shard_off, P.n_shards, loff);
    const uint64_t s_end = P.shard_off[s + 1];
    uint64_t e = loff;
    while (e < s_end && P.csv[e] != '\n') ++e;
    int32_t len = static_cast<int32_t>(e - loff);
    line = P.csv + loff;
    if (len > 0 && line[len - 1] == '\r') --len;
    return parse_line(line, len, P.cmap[s], pr) == kAccepted;
}

__device__ bool payload_equal(const FoldParams& P, uint64_t la, uint64_t lb) {
    Parsed a, b;
    const uint8_t *pa, *pb;
    if (!parse_at(P, la, a, pa) || !parse_at(P, lb, b, pb)) return false;
    if (!(a.lat == b.lat && a.lon == b.lon && a.speed == b.speed && a.heading == b.heading))
        return false;
    if (a.postal_len != b.postal_len) return false;
    return bytes_equal(pa + a.postal_begin, pb + b.postal_begin, static_cast<uint32_t>(a.postal_len));
}

// records entry point: CvRecord::operator== minus the dedup key (id and time are equal)
__device__ bool payload_equal_rec(const FoldParams& P, uint64_t a, uint64_t b) {
    if (!(P.r_lat[a] == P.r_lat[b] && P.r_lon[a] == P.r_lon[b] && P.r_speed[a] == P.r_speed[b] &&
          P.r_heading[a] == P.r_heading[b]))
        return false;
    const uint64_t pa = P.r_postal[a], pb = P.r_postal[b];
    if ((pa >> 40) != (pb >> 40)) return false;
    return bytes_equal(P.r_postal_arena + (pa & ((1ull << 40) - 1)),
                       P.r_postal_arena + (pb & ((1ull << 40) - 1)), static_cast<uint32_t>(pa >> 40));
}

// ---- F: per-journey fold -----------------------------------------------------------------------
// One LANE per journey (dynamic assignment), so the inherently sequential per-(cell, journey)
// left fold (aggregate.cpp:349-356) runs with every lane busy. Each window the warp stages the
// next kChunk records of all 32 lanes' streams into shared memory with coalesced loads (two
// lanes' chunks per instruction), then every lane walks its own chunk in (rank, ts) order.
// Accumulators live in registers while consecutive records share a cell; on a cell change the
// running (sum, count) is parked in the (cell, journey) hash table and the new cell's is loaded
// (re-entries continue the same fold), so per-(cell, journey) subtotals are exact.
constexpr int kFoldWarps = kFoldThreads / 32;
constexpr int kChunk = 8;        // slow path window (staged through registers: slot indirection)
#ifndef CVLG_FOLD_CHUNK
#define CVLG_FOLD_CHUNK 16
#endif
constexpr int kChunkFast = CVLG_FOLD_CHUNK;  // fast path window (cp.async straight to shared)
static_assert(32 % kChunkFast == 0 && 32 % kChunk == 0, "a window staging round covers 32 / kCh lanes");
#ifndef CVLG_LANE_CELLS
#define CVLG_LANE_CELLS 10
#endif
constexpr int kLaneCellsFast = CVLG_LANE_CELLS;  // per-lane cell table; a journey visits ~9 cells
constexpr int kLaneCellsSlow = 10;  // (slow path also stages slot ids and timestamps: less shared memory left)

constexpr uint64_t kSpillProbes = 512;  // (a full table fails fast; the host re-runs it larger)
constexpr uint32_t kBinSpilled = 0x80000000u;  // t_c flag: this entry's time-bin window spilled

__device__ __forceinline__ uint64_t table_find(const FoldParams& P, uint64_t key, bool insert,
                                               bool& fresh) {
    uint64_t slot = mix64(key) & P.spill_mask;
    fresh = false;
    // probes are bounded (inserts that give up count as overflow: the host re-runs with a larger
    // table), so a lookup that stops at the same bound is still exact
    const uint64_t limit = P.spill_mask < kSpillProbes ? P.spill_mask + 1 : kSpillProbes;
    for (uint64_t probe = 0; probe < limit; ++probe) {
        uint64_t cur = P.spill_key[slot];
        if (cur == kEmpty && insert) {
            cur = atomicCAS(reinterpret_cast<unsigned long long*>(&P.spill_key[slot]), kEmpty, key);
            if (cur == kEmpty) {
                fresh = true;
                return slot;
            }
        }
        if (cur == key) return slot;
        if (cur == kEmpty) return kEmpty;
        slot = (slot + 1) & P.spill_mask;
    }
    return kEmpty;
}

template <bool kSlow>
#ifndef CVLG_FOLD_MINB
#define CVLG_FOLD_MINB 1
#endif
#ifndef CVLG_FOLD_MINB_SLOW
#define CVLG_FOLD_MINB_SLOW 4  // the slow path waits on gathers: 4 CTAs per SM (128 registers)
#endif
__global__ void __launch_bounds__(kFoldWarps * 32, kSlow ? CVLG_FOLD_MINB_SLOW : CVLG_FOLD_MINB)
    fold_lane_kernel(FoldParams P) {
    constexpr int kLaneCells = kSlow ? kLaneCellsSlow : kLaneCellsFast;
    constexpr int kCh = kSlow ? kChunk : kChunkFast;
    __shared__ uint32_t s_code[kFoldWarps][32][kCh + 1];
    __shared__ double s_speed[kFoldWarps][32][kCh + 1];
    __shared__ uint32_t s_slot[kSlow ? kFoldWarps : 1][32][kChunk + 1];
    __shared__ long long s_ts[kSlow ? kFoldWarps : 1][32][kSlow ? kChunk + 1 : 1];
    // per-lane (cell -> running subtotal) table, entry e of lane l at [e][l]
    __shared__ uint32_t t_g[kFoldWarps][kLaneCells][32];
    __shared__ uint32_t t_c[kFoldWarps][kLaneCells][32];
    __shared__ double t_s[kFoldWarps][kLaneCells][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t c_acc = 0, c_oog = 0, c_spd = 0, c_miss = 0, c_unb = 0, c_dup = 0, c_conf = 0,
             c_ovf = 0;

    // first journey: spread over every CTA and warp (lane-major), so a run with fewer journeys
    // than lanes still occupies all SMs; later ones come from the shared counter
    const uint64_t n_lanes = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    // work items are handed out longest first when P.jorder is set (a journey index sorted by
    // record count): the last items any warp picks up are short, so warps do not idle behind one
    // long straggler once the counter runs out
    auto order = [&](uint64_t i) -> uint64_t { return P.jorder && i < P.n_journeys ? P.jorder[i] : i; };
    auto next_journey = [&]() {
        return order(n_lanes + atomicAdd(reinterpret_cast<unsigned long long*>(P.journey_counter), 1ull));
    };
    uint64_t j = order(static_cast<uint64_t>(lane * kFoldWarps + warp) * gridDim.x + blockIdx.x);
    bool active = j < P.n_journeys;
    uint32_t ri = 0, re = 0;    // fast path: remaining runs of the journey, [ri, re) in perm
    // fast path prefetch: the next run of this journey (runs[ri]) and the next journey (its run
    // range and first run), loaded one or more windows before they are needed, so switching runs
    // or journeys never stalls the warp on a dependent global load
    uint2 nrun = make_uint2(0u, 0u);
    uint64_t jn = ~0ull;
    uint32_t jn_ri = 0, jn_re = 0;
    uint2 jn_run = make_uint2(0u, 0u);
    int jstage = 0;  // 0: jn's run range not loaded, 1: first run not loaded, 2: ready
    uint64_t pos = 0, end = 0;  // current stream window: slots (fast) / perm positions (slow)
    uint32_t n_cells = 0;       // entries used in this lane's table
    uint64_t seen = 0;          // bloom filter of the cells this journey visited (new cells skip the search)
    uint32_t cur = 0;           // table entry of the current cell (valid when n_cells > 0)
    uint32_t cur_g = kNone;
    double cur_sum = 0.0;
    uint32_t cur_cnt = 0;
    uint32_t evict = 0;
    bool spilled = false;
    int64_t prev_ts = 0;
    uint64_t surv = 0;
    bool have_prev = false;
    // time-bin windows: entries [0, wstart) belong to closed windows, [wstart, n_cells) to the
    // current one; bins of closed windows are covered by the current segment [seg_lo, cur_tb]
    // (bins rise along a segment) and up to four older segment hulls (lo | hi << 16).
    // Invariants (window mode), which make the fold exact:
    //  * each (cell, journey) subtotal lives in exactly one place: this lane's table, the live
    //    directory block of its bin in the pair list, or the spill table (spilled windows only;
    //    an entry read back from the spill table is marked moved-out there: count 0);
    //  * one bin's table entries are adjacent (a reopened bin first flushes every closed entry),
    //    so a flush writes one directory block per bin and dir[bin] names the only live block;
    //  * reloading a block vacates its pair slots (dead list, compacted after the fold) and
    //    clears dir[bin];
    //  * the reopen test is a superset test: a false positive costs one directory read.
    uint32_t wstart = 0, wlo = 0, cur_tb = kNone, seg_lo = 0;
    uint32_t iv0 = 0xFFFFu, iv1 = 0xFFFFu, iv2 = 0xFFFFu, iv3 = 0xFFFFu;
    const uint64_t dir_row = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * P.n_bins;

    auto start_journey = [&]() {
        cur_g = kNone;
        n_cells = 0;
        seen = 0;
        evict = 0;
        spilled = false;
        have_prev = false;
        wstart = 0;
        cur_tb = kNone;
        iv0 = iv1 = iv2 = iv3 = 0xFFFFu;
        if (kSlow) {
            pos = P.jstart[j];
            end = P.jstart[j + 1];
        } else {
            // (ri, re, first run) come from the prefetch when ready, else are loaded here
            if (jstage == 2) {
                ri = jn_ri;
                re = jn_re;
                pos = jn_run.x;
                end = jn_run.y;
            } else {
                ri = P.jstart[j];
                re = P.jstart[j + 1];
                const uint2 r0 = P.runs[ri];
                pos = r0.x;
                end = r0.y;
            }
            ++ri;
            jstage = 0;
            if (ri < re) {
                nrun = P.runs[ri];
                jn = ~0ull;
            } else {  // last run open: take the next journey now (not earlier: no hoarding)
                jn = next_journey();
            }
        }
    };
    auto spill_store = [&](uint32_t g, double s, uint32_t c) {
        bool fresh;
        const uint64_t t = table_find(P, (static_cast<uint64_t>(g) << 32) | j, true, fresh);
        if (t == kEmpty) {
            ++c_ovf;
            atomicExch(P.abort_flag, 1u);
            return;
        }
        P.spill_sum[t] = s;
        P.spill_cnt[t] = c & ~kBinSpilled;
    };
    // write the whole journey out: appended pairs, or the spill table once it has spilled
    auto flush_journey = [&]() {
        const uint64_t jr = P.jrank ? P.jrank[j] : j;  // (bin-group mode: the group's journey)
        if (cur_g != kNone) {
            t_s[warp][cur][lane] = cur_sum;
            t_c[warp][cur][lane] = cur_cnt;
        }
        if (!spilled) {
            const uint32_t base = n_cells ? atomicAdd(P.pair_count, n_cells) : 0u;
            for (uint32_t e = 0; e < n_cells; ++e) {
                const uint64_t at = static_cast<uint64_t>(base) + e;
                if (at >= P.pair_cap) {
                    ++c_ovf;
                    continue;
                }
                P.pair_key[at] = (static_cast<uint64_t>(t_g[warp][e][lane]) << P.rank_bits) | jr;
                P.pair_sum[at] = t_s[warp][e][lane];
                P.pair_cnt[at] = t_c[warp][e][lane] & ~kBinSpilled;
            }
        } else {
            for (uint32_t e = 0; e < n_cells; ++e)
                spill_store(t_g[warp][e][lane], t_s[warp][e][lane], t_c[warp][e][lane]);
        }
    };
    // closed-window entries [0, upto) -> pair list at `base` (one directory block per time bin,
    // entries of one bin are adjacent in the table), then the rest of the table moves down
    auto flush_closed = [&](uint32_t upto, uint32_t base) {
        const uint64_t jr = j;  // (window mode is never combined with bin groups)
        uint32_t e = 0;
        while (e < upto) {
            const uint32_t tb = t_g[warp][e][lane] / P.drc;
            const uint32_t lo = tb * P.drc;
            uint32_t f = e, flag = 0;
            bool ovf = false;
            do {
                const uint64_t at = static_cast<uint64_t>(base) + f;
                const uint32_t cn = t_c[warp][f][lane];
                flag |= cn & kBinSpilled;
                if (at < P.pair_cap) {
                    P.pair_key[at] = (static_cast<uint64_t>(t_g[warp][f][lane]) << P.rank_bits) | jr;
                    P.pair_sum[at] = t_s[warp][f][lane];
                    P.pair_cnt[at] = cn & ~kBinSpilled;
                } else {
                    ++c_ovf;
                    ovf = true;
                }
                ++f;
            } while (f < upto && t_g[warp][f][lane] - lo < P.drc);
            // a block past the pair list is never published (a reopen would read past the
            // allocation); the attempt is void and re-runs without windows
            if (ovf) atomicExch(P.abort_flag, 1u);
            else P.dir[dir_row + tb] = make_uint4(static_cast<uint32_t>(j), P.epoch, base + e, (f - e) | flag);
            e = f;
        }
        for (uint32_t q = upto; q < n_cells; ++q) {
            t_g[warp][q - upto][lane] = t_g[warp][q][lane];
            t_s[warp][q - upto][lane] = t_s[warp][q][lane];
            t_c[warp][q - upto][lane] = t_c[warp][q][lane];
        }
        n_cells -= upto;
        cur = cur >= upto ? cur - upto : 0;
        wstart = wstart >= upto ? wstart - upto : 0;
    };
    auto in_segments = [&](uint32_t tb) {
        auto in = [&](uint32_t iv) { return tb >= (iv & 0xFFFFu) && tb <= (iv >> 16); };
        return in(iv0) || in(iv1) || in(iv2) || in(iv3);
    };
    auto push_segment = [&](uint32_t lo, uint32_t hi) {
        const uint32_t l3 = min(iv3 & 0xFFFFu, iv2 & 0xFFFFu), h3 = max(iv3 >> 16, iv2 >> 16);
        iv3 = l3 | (h3 << 16);  // oldest two merge into their hull (a superset: still exact-safe)
        iv2 = iv1;
        iv1 = iv0;
        iv0 = lo | (hi << 16);
    };
    // a window of an already-closed bin opened: bring back that bin's flushed block (if any);
    // a bin whose window spilled has more of its subtotals in the spill table: the window
    // continues in spilled state (lookups)
    auto reopen = [&](uint32_t tb) {
        if (n_cells) {  // every entry is closed now: flush them (keeps bins contiguous)
            const uint32_t base = atomicAdd(P.pair_count, n_cells);
            flush_closed(n_cells, base);
        }
        const uint4 d = P.dir[dir_row + tb];
        if (d.x == static_cast<uint32_t>(j) && d.y == P.epoch &&
            static_cast<uint64_t>(d.z) + (d.w & ~kBinSpilled) <= P.pair_cap) {
            const uint32_t cnt = d.w & ~kBinSpilled;
            const uint32_t dl = atomicAdd(P.dead_count, cnt);
            for (uint32_t q = 0; q < cnt; ++q) {
                const uint64_t at = static_cast<uint64_t>(d.z) + q;
                t_g[warp][q][lane] = static_cast<uint32_t>(P.pair_key[at] >> P.rank_bits);
                t_s[warp][q][lane] = P.pair_sum[at];
                t_c[warp][q][lane] = P.pair_cnt[at] | (d.w & kBinSpilled);
                P.pair_key[at] = kDeadPair;
                P.dead_list[dl + q] = static_cast<uint32_t>(at);
            }
            n_cells = cnt;
            spilled = (d.w & kBinSpilled) != 0;
            seen = ~0ull;  // reloaded (or spilled) codes: search for the rest of this window
            P.dir[dir_row + tb] = make_uint4(0u, 0u, 0u, 0u);
        }
        wstart = 0;
    };
    if (active) start_journey();

    uint32_t round = 0;
    while (__any_sync(0xFFFFFFFFu, active)) {
        if ((++round & 31) == 0) {  // a spill insert failed somewhere: this attempt is void, stop
            uint32_t a = 0;
            if (lane == 0) a = *reinterpret_cast<volatile const uint32_t*>(P.abort_flag);
            if (__shfl_sync(0xFFFFFFFFu, a, 0)) break;
        }
        const uint64_t left = end - pos;
        const uint32_t avail = !active ? 0u : (left < kCh ? static_cast<uint32_t>(left) : kCh);
        // ---- stage every lane's next chunk: 32/kCh lane chunks per coalesced access ----------------
        constexpr int kPer = 32 / kCh;
        constexpr int kIt = 32 / kPer;
        const int k = lane % kCh;
        if constexpr (!kSlow) {  // fast path: cp.async global -> shared, every copy in flight at once
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                const int src = it * kPer + lane / kCh;
                const uint64_t p0 = __shfl_sync(0xFFFFFFFFu, pos, src);
                const uint32_t a = __shfl_sync(0xFFFFFFFFu, avail, src);
                if (static_cast<uint32_t>(k) < a) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(&s_code[warp][src][k]))),
                                 "l"(&P.code[p0 + k])
                                 : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                     static_cast<uint32_t>(__cvta_generic_to_shared(&s_speed[warp][src][k]))),
                                 "l"(&P.speed[p0 + k])
                                 : "memory");
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else {  // (all loads first, then the shared stores: every load of the window in flight)
            uint32_t slv[kIt], cv[kIt];
            double sv[kIt];
            long long tv[kIt];
            uint64_t p0s[kIt];
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                const int src = it * kPer + lane / kCh;
                const uint64_t p0 = __shfl_sync(0xFFFFFFFFu, pos, src);
                const uint32_t a = __shfl_sync(0xFFFFFFFFu, avail, src);
                const bool in = static_cast<uint32_t>(k) < a;
                slv[it] = in ? __ldg(&P.perm[p0 + k]) : 0u;
                p0s[it] = p0;
            }
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                const int src = it * kPer + lane / kCh;
                const uint32_t a = __shfl_sync(0xFFFFFFFFu, avail, src);
                const bool in = static_cast<uint32_t>(k) < a;
                if (P.rec) {  // (speed, code) of the slot in one 16-byte gather
                    const ulonglong2 r = in ? __ldg(&P.rec[slv[it]]) : make_ulonglong2(0ull, 0ull);
                    cv[it] = static_cast<uint32_t>(r.y);
                    sv[it] = __longlong_as_double(static_cast<long long>(r.x));
                } else {
                    cv[it] = in ? __ldg(&P.code[slv[it]]) : 0u;
                    sv[it] = in ? __ldg(&P.speed[slv[it]]) : 0.0;
                }
                tv[it] = !in ? 0 : P.skey ? static_cast<long long>(P.skey[p0s[it] + k]) : __ldg(&P.ts[slv[it]]);
            }
#pragma unroll
            for (int it = 0; it < kIt; ++it) {
                const int src = it * kPer + lane / kCh;
                s_code[warp][src][k] = cv[it];
                s_speed[warp][src][k] = sv[it];
                s_slot[warp][src][k] = slv[it];
                s_ts[warp][src][kSlow ? k : 0] = tv[it];
            }
        }
        __syncwarp();
        // ---- pass 1: this lane's chunk in (rank, ts) order: dedup (slow path), filters, and the
        // positions where the accepted records' cell changes (segment starts) -------------------
        uint32_t use = 0, segs = 0;
        {
            uint32_t prev = cur_g;
            for (uint32_t k = 0; k < avail; ++k) {
                const uint32_t code = s_code[warp][lane][k] & kCodeMask;
                if (kSlow) {
                    const uint32_t slot = s_slot[warp][lane][k];
                    const int64_t t = s_ts[warp][lane][kSlow ? k : 0];
                    if (have_prev && t == prev_ts) {  // duplicate key: dropped before filtering
                        ++c_dup;
                        const bool same = P.r_lat ? payload_equal_rec(P, P.loff[slot], P.loff[surv])
                                                  : payload_equal(P, P.loff[slot], P.loff[surv]);
                        if (!same) ++c_conf;
                        continue;
                    }
                    have_prev = true;
                    prev_ts = t;
                    surv = slot;
                }
                if (code >= kCodeFirstSpecial) {
                    if (code == kCodeOutOfGrid) ++c_oog;
                    else if (code == kCodeSpeedCeiling) ++c_spd;
                    else if (code == kCodeMissingField) ++c_miss;
                    else if (code == kCodeUnbinnable) ++c_unb;
                    continue;  // kCodeRejected: counted by decode
                }
                ++c_acc;
                use |= 1u << k;
                if (code != prev) {
                    segs |= 1u << k;
                    prev = code;
                }
            }
        }
        // ---- pass 2: the left fold (aggregate.cpp:349-356). Records before the first segment
        // start continue the current cell; then one warp-wide round per segment index, so every
        // lane's cell switch of that round runs together instead of the warp serializing on each
        // record where any lane switches.
        auto accumulate = [&](uint32_t from, uint32_t to) {
            uint32_t m = use & ((to >= 32 ? 0xFFFFFFFFu : ((1u << to) - 1u)) & ~((1u << from) - 1u));
            while (m) {
                const uint32_t k = __ffs(m) - 1;
                m &= m - 1;
                cur_sum = __dadd_rn(cur_sum, s_speed[warp][lane][k]);  // aggregate.cpp:354
                ++cur_cnt;
            }
        };
        accumulate(0, segs ? static_cast<uint32_t>(__ffs(segs) - 1) : avail);
        while (__any_sync(0xFFFFFFFFu, segs != 0)) {
            if (segs) {
                const uint32_t k0 = __ffs(segs) - 1;
                segs &= segs - 1;
                const uint32_t k1 = segs ? static_cast<uint32_t>(__ffs(segs) - 1) : avail;
                const uint32_t code = s_code[warp][lane][k0] & kCodeMask;
                if (cur_g != kNone) {  // park the current subtotal in its table entry
                    t_s[warp][cur][lane] = cur_sum;
                    t_c[warp][cur][lane] = cur_cnt;
                }
                if (P.win && (cur_tb == kNone || code - wlo >= P.drc)) {  // a new time-bin window
                    const uint32_t tb = code / P.drc;
                    wlo = tb * P.drc;
                    bool again = false;
                    if (cur_tb != kNone) {
                        if (tb < cur_tb) {  // bins fell (midnight, next day): a new segment
                            push_segment(seg_lo, cur_tb);
                            seg_lo = tb;
                        }
                        again = in_segments(tb);
                    } else {
                        seg_lo = tb;
                    }
                    cur_tb = tb;
                    wstart = n_cells;
                    spilled = false;  // (window mode: spilled and the bloom filter are per window:
                    seen = 0;         //  no entry of a fresh window's bin exists anywhere)
                    if (again) reopen(tb);
                }
                const uint64_t bit = 1ull << ((code * 0x9E3779B1u) >> 26);
                const bool maybe_seen = (seen & bit) != 0;
                seen |= bit;
                uint32_t e = n_cells;
                if (maybe_seen) {  // all entries at once: independent loads, no dependent chain
                    uint32_t match = 0;
#pragma unroll
                    for (int q = 0; q < kLaneCells; ++q)
                        match |= (t_g[warp][q][lane] == code ? 1u : 0u) << q;
                    match &= (n_cells >= 32 ? 0xFFFFFFFFu : ((1u << n_cells) - 1u));
                    e = match ? static_cast<uint32_t>(__ffs(match) - 1) : n_cells;
                }
                if (e < n_cells) {
                    cur_sum = t_s[warp][e][lane];
                    cur_cnt = t_c[warp][e][lane];
                } else {
                    if (n_cells == kLaneCells && wstart > 0) {  // room: flush closed windows
                        const uint32_t base = atomicAdd(P.pair_count, wstart);
                        flush_closed(wstart, base);
                    }
                    if (n_cells < kLaneCells) {
                        e = n_cells++;
                    } else {  // table full: move the oldest-assigned entry to the spill table
                        e = evict;
                        evict = (evict + 1) % kLaneCells;
                        spill_store(t_g[warp][e][lane], t_s[warp][e][lane], t_c[warp][e][lane]);
                        spilled = true;
                    }
                    cur_sum = 0.0;
                    cur_cnt = P.win && spilled ? kBinSpilled : 0u;  // (marks the bin's block)
                    if (spilled && maybe_seen) {  // the cell may have been evicted earlier: continue its fold
                        bool fresh;
                        const uint64_t t = table_find(P, (static_cast<uint64_t>(code) << 32) | j,
                                                      false, fresh);
                        if (t != kEmpty && P.spill_cnt[t]) {
                            cur_sum = P.spill_sum[t];
                            cur_cnt |= P.spill_cnt[t];
                            P.spill_cnt[t] = 0;  // moved back out (a later eviction re-fills it)
                        }
                    }
                    t_g[warp][e][lane] = code;
                }
                cur = e;
                cur_g = code;
                accumulate(k0, k1);
            }
        }
        __syncwarp();
        // ---- flush closed windows of nearly full tables, one pair-list reservation per warp ------
        if (P.win) {
            const bool want = active && wstart > 0 && n_cells + P.flush_slack >= kLaneCells;
            if (__any_sync(0xFFFFFFFFu, want)) {
                const uint32_t c = want ? wstart : 0u;
                const uint32_t incl = warp_inclusive_sum(c);
                uint32_t base = 0;
                if (lane == 31) base = atomicAdd(P.pair_count, incl);
                base = __shfl_sync(0xFFFFFFFFu, base, 31);
                if (want) flush_closed(wstart, base + incl - c);
            }
        }
        // ---- advance the stream ----------------------------------------------------------------
        if (!kSlow && active && jn < P.n_journeys) {  // advance the next-journey prefetch
            if (jstage == 0) {
                jn_ri = P.jstart[jn];
                jn_re = P.jstart[jn + 1];
                jstage = 1;
            } else if (jstage == 1) {
                jn_run = P.runs[jn_ri];
                jstage = 2;
            }
        }
        pos += avail;
        if (active && pos >= end) {
            if (!kSlow && ri < re) {
                pos = nrun.x;
                end = nrun.y;
                ++ri;
                if (ri < re) nrun = P.runs[ri];
                else jn = next_journey();
            } else {
                flush_journey();
                if (kSlow) {
                    j = next_journey();
                } else {
                    if (jstage == 1) {  // first run of the prefetched journey not in yet
                        jn_run = P.runs[jn_ri];
                        jstage = 2;
                    }
                    j = jn;
                }
                active = j < P.n_journeys;
                if (active) start_journey();
            }
        }
    }
    unsigned long long vals[8] = {c_acc, c_oog, c_spd, c_miss, c_unb, c_dup, c_conf, c_ovf};
    const int idx[8] = {kStAccepted, kStFiltOutOfGrid, kStFiltSpeed, kStFiltMissing,
                        kStUnbinnable, kStDups, kStConflicts, kStOverflow};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned long long s = warp_sum(vals[k]);
        if (lane == 0 && s) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[idx[k]]), s);
    }
}

// fast path: the runs in perm order as (start, end) slot pairs (one load per run switch)
__global__ void run_list_kernel(const uint32_t* perm, const uint32_t* hslot, const uint32_t* hend,
                                uint64_t n, uint2* runs) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t h = perm[i];
    runs[i] = make_uint2(hslot[h], hend[h]);
}

// ---- bin-group mode (few long journeys) ----------------------------------------------------------
// A (cell, journey) subtotal only ever collects records of the cell's time bin, so the records of
// one (journey, bin) pair form an independent fold: runs are cut where the bin of the accepted
// records changes, the pieces are sorted by (journey, bin, stream order), and every (journey, bin)
// group becomes one lane's work item (its pieces in stream order = the journey's ts order).
__global__ void run_journey_kernel(const uint32_t* jstart, uint64_t J, uint32_t* run_j) {
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (j >= J) return;
    for (uint32_t r = jstart[j]; r < jstart[j + 1]; ++r) run_j[r] = static_cast<uint32_t>(j);
}

// one warp per run: pieces [start, end) with key (journey << (bin_bits + order_bits) | bin <<
// order_bits | run << 9 | piece-in-run). Records before the run's first accepted record belong
// to its first piece (they only count filter stats in the fold).
__global__ void bin_pieces_kernel(const uint2* runs, uint64_t n_runs, const uint32_t* run_j,
                                  const uint32_t* code, uint32_t drc, int bin_bits, int run_bits,
                                  uint64_t* keys, uint32_t* vals, uint2* pieces, uint32_t* counter,
                                  uint64_t cap) {
    const uint64_t r = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (r >= n_runs) return;
    const int lane = threadIdx.x & 31;
    const uint2 run = runs[r];
    const uint64_t jkey = static_cast<uint64_t>(run_j[r]) << (bin_bits + run_bits + 9);
    const int order_bits = run_bits + 9;
    constexpr uint32_t kNoBin = 0xFFFFFFFFu;
    uint32_t cur_bin = kNoBin, start = run.x, n_piece = 0;
    auto emit = [&](uint32_t end) {
        if (lane == 0 && n_piece >= 512) atomicOr(counter + 1, 1u);  // order field overflow: host falls back
        if (lane == 0) {
            const uint32_t at = atomicAdd(counter, 1u);
            if (at < cap) {
                const uint64_t b = cur_bin == kNoBin ? 0u : cur_bin;
                keys[at] = jkey | (b << order_bits) | (r << 9) | n_piece;
                vals[at] = at;
                pieces[at] = make_uint2(start, end);
            }
        }
        ++n_piece;
    };
    for (uint32_t base = run.x; base < run.y; base += 32) {
        const uint32_t i = base + lane;
        const uint32_t c = i < run.y ? (code[i] & kCodeMask) : kCodeRejected;
        const bool acc = c < kCodeFirstSpecial;
        uint32_t x = acc ? c / drc : kNoBin;  // bin of the last accepted record at or before me
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o && x == kNoBin) x = t;
        }
        uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, x, 1);
        if (lane == 0 || prev == kNoBin) prev = cur_bin;
        const uint32_t my = acc ? c / drc : kNoBin;
        uint32_t cut = __ballot_sync(0xFFFFFFFFu, acc && prev != kNoBin && my != prev);
        const uint32_t last = __shfl_sync(0xFFFFFFFFu, x, 31);
        if (cur_bin == kNoBin) {  // the open piece takes the bin of its first accepted record
            const uint32_t first = __ballot_sync(0xFFFFFFFFu, acc);
            if (first) cur_bin = __shfl_sync(0xFFFFFFFFu, my, __ffs(first) - 1);
        }
        while (cut) {
            const int l = __ffs(cut) - 1;
            cut &= cut - 1;
            emit(base + l);
            start = base + l;
            cur_bin = __shfl_sync(0xFFFFFFFFu, my, l);
        }
        if (last != kNoBin) cur_bin = last;
    }
    emit(run.y);
}

// sorted pieces -> runs in group order, flags at group starts
__global__ void bin_groups_kernel(const uint64_t* keys, const uint32_t* vals, const uint2* pieces,
                                  uint64_t n, int order_bits, uint32_t* flags, uint2* runs_out) {
    const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    runs_out[k] = pieces[vals[k]];
    flags[k] = (k == 0 || (keys[k] >> order_bits) != (keys[k - 1] >> order_bits)) ? 1u : 0u;
}

__global__ void bin_group_starts_kernel(const uint64_t* keys, const uint32_t* flags, const uint32_t* pos,
                                        uint64_t n, int order_bits, int bin_bits, uint32_t* gstart,
                                        uint32_t* gj) {
    const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (k >= n || !flags[k]) return;
    gstart[pos[k]] = static_cast<uint32_t>(k);
    gj[pos[k]] = static_cast<uint32_t>(keys[k] >> (order_bits + bin_bits));
}

// longest-first work order: key = ~(records of item j) (ascending = longest first), value = j
__global__ void journey_len_keys_kernel(const uint32_t* jstart, uint64_t n, const uint2* runs,
                                        int runs_mode, uint64_t* keys, uint32_t* vals) {
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (j >= n) return;
    uint64_t len = 0;
    if (runs_mode) {  // fast path: sum of the item's run lengths
        for (uint32_t r = jstart[j]; r < jstart[j + 1]; ++r) len += runs[r].y - runs[r].x;
    } else {
        len = jstart[j + 1] - jstart[j];
    }
    keys[j] = 0xFFFFFFFFull - (len > 0xFFFFFFFFull ? 0xFFFFFFFFull : len);
    vals[j] = static_cast<uint32_t>(j);
}

// spilled journeys' subtotals -> pair list
__global__ void spill_drain_kernel(FoldParams P) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i > P.spill_mask) return;
    const uint64_t k = P.spill_key[i];
    if (k == kEmpty || P.spill_cnt[i] == 0) return;  // (cnt 0: moved back out by its lane)
    const uint32_t pos = atomicAdd(P.pair_count, 1u);
    if (pos >= P.pair_cap) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStOverflow]), 1ull);
        return;
    }
    const uint64_t j = k & 0xFFFFFFFFull;
    P.pair_key[pos] = ((k >> 32) << P.rank_bits) | (P.jrank ? P.jrank[j] : j);
    P.pair_sum[pos] = P.spill_sum[i];
    P.pair_cnt[pos] = P.spill_cnt[i];
}

__global__ void pair_vals_kernel(uint32_t* vals, uint64_t n) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) vals[i] = static_cast<uint32_t>(i);
}

// ---- Z: canonical per-cell fold (finalize_range, aggregate.cpp:161-187) ----------------------
__global__ void finalize_kernel(const uint64_t* keys, const uint32_t* vals, uint64_t n,
                                int rank_bits, const double* pair_sum, const uint32_t* pair_cnt,
                                uint32_t D, uint64_t RC, uint32_t t_base, uint32_t t_rows,
                                uint32_t* planes, uint32_t* raw) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t g = keys[i] >> rank_bits;
    const uint64_t tg = g / (D * RC);
    if (tg < t_base || tg - t_base >= t_rows) return;  // outside the rows this lattice holds
    if (i > 0 && (keys[i - 1] >> rank_bits) == g) return;
    double sum = 0.0;
    uint64_t cnt = 0;
    uint32_t vol = 0;
    for (uint64_t k = i; k < n && (keys[k] >> rank_bits) == g; ++k) {
        sum = __dadd_rn(sum, pair_sum[vals[k]]);  // journey-lexicographic order
        cnt += pair_cnt[vals[k]];
        ++vol;
    }
    const uint64_t t = tg - t_base;
    const uint64_t d = (g / RC) % D;
    const uint64_t rc = g % RC;
    const float mean = __double2float_rn(__ddiv_rn(sum, static_cast<double>(cnt)));
    planes[(t * 8 + d) * RC + rc] = __float_as_uint(mean);
    planes[(t * 8 + 4 + d) * RC + rc] = vol;
    if (raw) raw[(t * 4 + d) * RC + rc] = static_cast<uint32_t>(cnt);
}

// ---- multi-GPU exchange: (cell, local rank) pairs <-> (cell, global journey key) tuples ------
__global__ void rank_slot_kernel(const uint32_t* uslot, const uint32_t* perm, uint64_t n,
                                 uint32_t* rank_slot) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) rank_slot[i] = uslot[perm[i]];
}

// Global journey key = the dictionary's exact inline key (ids <= 15 bytes): (bytes 0..7 BE,
// bytes 8..14 BE << 8 | len) orders exactly like std::string (SURVEY §7 hard part 2).
__global__ void export_pairs_kernel(const uint64_t* pkey, const double* psum, const uint32_t* pcnt,
                                    uint64_t n, int rbits, const uint32_t* rank_slot,
                                    const unsigned long long* table, uint64_t* cell, uint64_t* k0,
                                    uint64_t* k1, double* sum, uint64_t* cnt, uint64_t stride,
                                    const uint32_t* grank, uint32_t* bad) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t key = pkey[i];
    const uint64_t r = rbits ? (key & ((1ull << rbits) - 1)) : 0;
    uint64_t e0, e1;
    if (grank) {  // global lexicographic rank (any id length), merged across GPUs on the host
        e0 = grank[r];
        e1 = 0;
    } else {
        const uint32_t slot = rank_slot[r];
        e0 = table[2 * slot];
        e1 = table[2 * slot + 1];
        if ((e1 & 0xFF) == 0xFF) *bad = 1u;  // id longer than 15 bytes: no exact inline key
    }
    const uint64_t o = i * stride;
    cell[o] = key >> rbits;
    k0[o] = e0;
    k1[o] = e1;
    sum[o] = psum[i];
    cnt[o] = pcnt[i];
}

// Journey ids in local rank order (for the cross-GPU merge of long ids): lengths, then bytes.
__device__ __forceinline__ uint32_t id_len_of(uint64_t e0, uint64_t e1) {
    return (e1 & 0xFF) == 0xFF ? static_cast<uint32_t>(e0 & 0xFFFFFF) : static_cast<uint32_t>(e1 & 0xFF);
}

__global__ void id_len_kernel(const uint32_t* rank_slot, const unsigned long long* table, uint64_t n,
                              uint32_t* len) {
    const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const uint32_t slot = rank_slot[r];
    len[r] = id_len_of(table[2 * slot], table[2 * slot + 1]);
}

__global__ void id_copy_kernel(const uint32_t* rank_slot, const unsigned long long* table,
                               const uint8_t* csv, uint64_t n, const uint32_t* pos, uint8_t* blob) {
    const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (r >= n) return;
    const uint32_t slot = rank_slot[r];
    const uint64_t e0 = table[2 * slot], e1 = table[2 * slot + 1];
    const uint32_t len = id_len_of(e0, e1);
    uint8_t* d = blob + pos[r];
    if ((e1 & 0xFF) == 0xFF) {
        const uint8_t* p = csv + (e1 >> 8);
        for (uint32_t k = 0; k < len; ++k) d[k] = p[k];
    } else {
        for (uint32_t k = 0; k < len; ++k)
            d[k] = static_cast<uint8_t>(k < 8 ? e0 >> (56 - 8 * k) : e1 >> (64 - 8 * (k - 8)));
    }
}

__global__ void gather_u64_kernel(const uint64_t* src, uint64_t stride, const uint32_t* idx,
                                  uint64_t n, uint64_t* dst) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) dst[i] = src[(idx ? idx[i] : i) * stride];
}

__global__ void import_pairs_kernel(const double* sum, const uint64_t* cnt, uint64_t stride,
                                    uint64_t n, double* psum, uint32_t* pcnt) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    psum[i] = sum[i * stride];
    pcnt[i] = static_cast<uint32_t>(cnt[i * stride]);
}

inline unsigned grid_for(uint64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

// ================================ host launchers ================================================
void launch_tile_field(const uint4* tiles, uint64_t n, int field, uint32_t* out, cudaStream_t s) {
    if (!n) return;
    tile_field_kernel<<<grid_for(n, 256), 256, 0, s>>>(tiles, n, field, out);
    count_launch();
}

void launch_heads_compact(const uint4* tiles, uint64_t n, const uint32_t* hpos, const uint32_t* hscr,
                          const uint64_t* hid_scr, const ulonglong2* hkey_scr, uint32_t* hslot,
                          uint32_t* hend, uint64_t* hid, ulonglong2* hkey, cudaStream_t s,
                          const DictParams* dict) {
    if (!n) return;
    DictParams D{};
    if (dict) D = *dict;
    heads_compact_kernel<<<grid_for(n, 256), 256, 0, s>>>(tiles, n, hpos, hscr, hid_scr, hkey_scr, hslot,
                                                          hend, hid, hkey, D);
    count_launch();
}

void launch_ts_range(const int64_t* ts, const uint32_t* code, uint64_t n, long long* mm, cudaStream_t s) {
    ts_range_init_kernel<<<1, 1, 0, s>>>(mm);
    count_launch();
    if (n) {
        ts_range_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8)), 256, 0, s>>>(
            ts, code, n, mm);
        count_launch();
    }
}

void launch_densify(const DensifyParams& d, cudaStream_t s) {
    if (!d.n_tiles) return;
    densify_kernel<<<grid_for(d.n_tiles, 8), 256, 0, s>>>(d);
    count_launch();
}

void launch_dict_insert(const DictParams& d, cudaStream_t s) {
    if (!d.n_heads) return;
    dict_insert_kernel<<<grid_for(d.n_heads, 256), 256, 0, s>>>(d);
    count_launch();
}

void launch_dict_flags(const unsigned long long* table, uint64_t cap, uint32_t* flags,
                       cudaStream_t s) {
    dict_flags_kernel<<<grid_for(cap, 256), 256, 0, s>>>(table, cap, flags);
    count_launch();
}

void launch_dict_compact(const uint32_t* flags, const uint32_t* pos, uint64_t cap, uint32_t* uslot,
                         cudaStream_t s) {
    dict_compact_kernel<<<grid_for(cap, 256), 256, 0, s>>>(flags, pos, cap, uslot);
    count_launch();
}

void launch_dict_chunk(const unsigned long long* table, const uint32_t* uslot, const uint32_t* perm,
                       uint64_t n, int c, const uint8_t* csv, uint64_t* keys, cudaStream_t s) {
    dict_chunk_kernel<<<grid_for(n, 256), 256, 0, s>>>(table, uslot, perm, n, c, csv, keys);
    count_launch();
}

void launch_dict_rank(const uint32_t* uslot, const uint32_t* perm, uint64_t n,
                      uint32_t* rank_of_slot, cudaStream_t s) {
    dict_rank_kernel<<<grid_for(n, 256), 256, 0, s>>>(uslot, perm, n, rank_of_slot);
    count_launch();
}

void launch_head_rank(const uint32_t* hdict, const uint32_t* rank_of_slot, uint64_t n,
                      uint32_t* hrank, cudaStream_t s) {
    head_rank_kernel<<<grid_for(n, 256), 256, 0, s>>>(hdict, rank_of_slot, n, hrank);
    count_launch();
}

void launch_head_keys(const uint32_t* hrank, const uint32_t* hslot, const int64_t* ts,
                      uint64_t n_heads, int64_t ts_min, int tsbits, int mode, uint64_t* keys,
                      uint32_t* vals, cudaStream_t s) {
    head_keys_kernel<<<grid_for(n_heads, 256), 256, 0, s>>>(hrank, hslot, ts, n_heads, ts_min,
                                                            tsbits, mode, keys, vals);
    count_launch();
}

void launch_gather_rank_keys(const uint32_t* rank_src, const uint32_t* vals, uint64_t n,
                             uint64_t* keys, cudaStream_t s) {
    gather_rank_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(rank_src, vals, n, keys);
    count_launch();
}

void launch_head_order_check(const uint32_t* perm, const uint32_t* hrank, const uint32_t* hslot,
                             const uint32_t* hend, const int64_t* ts, const uint32_t* code,
                             uint64_t n_heads, uint32_t* jstart, uint32_t* invalid, cudaStream_t s) {
    head_order_check_kernel<<<grid_for(n_heads, 256), 256, 0, s>>>(perm, hrank, hslot, hend, ts, code,
                                                                   n_heads, jstart, invalid);
    count_launch();
}

void launch_slot_keys(const uint32_t* hslot, const uint32_t* hrank, const uint32_t* hdict,
                      const uint32_t* rank_of_slot, uint64_t n_heads,
                      const int64_t* ts, const uint32_t* code, uint64_t n_slots, int64_t ts_min,
                      int tsbits, int mode, uint32_t reject_rank, uint64_t* keys, uint32_t* vals,
                      uint32_t* srank, cudaStream_t s) {
    if (n_heads == 0) {
        slot_keys_kernel<<<grid_for(n_slots, 256), 256, 0, s>>>(hslot, hrank, n_heads, ts, code,
                                                                n_slots, ts_min, tsbits, mode,
                                                                reject_rank, keys, vals, srank);
    } else {
        run_keys_kernel<<<grid_for(n_heads, 256), 256, 0, s>>>(hslot, hrank, hdict, rank_of_slot, n_heads, ts, code,
                                                               n_slots, ts_min, tsbits, mode,
                                                               reject_rank, keys, vals, srank);
    }
    count_launch();
}

void launch_slot_jstart(const uint64_t* keys, int rank_shift, uint64_t n, uint32_t* jstart,
                        cudaStream_t s) {
    if (!n) return;
    slot_jstart_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, rank_shift, n, jstart);
    count_launch();
}

// one warp per journey at least (the first journeys go lane-major to lane 0 of every warp of the
// grid, so few long journeys spread over every SM instead of filling the lanes of a few warps),
// capped at what is resident at once (journeys are handed out dynamically, so CTAs beyond the
// resident set would find nothing left to do)
unsigned fold_grid(uint64_t n_journeys, bool slow) {
    const int sms = per_device(kPdSms, [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    });
    const int per_sm = slow ? per_device(kPdFoldPerSm1, [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fold_lane_kernel<true>, kFoldWarps * 32, 0);
        return n;
    }) : per_device(kPdFoldPerSm0, [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fold_lane_kernel<false>, kFoldWarps * 32, 0);
        return n;
    });
    const uint64_t cap = static_cast<uint64_t>(sms) * std::max(1, per_sm);
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n_journeys + kFoldWarps - 1) / kFoldWarps, cap)));
}

// live pairs of the tail [n - dead, n) -> src list (any order)
__global__ void pair_tail_live_kernel(const uint64_t* key, uint64_t n, uint64_t dead, uint32_t* src,
                                      uint32_t* counter) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= dead) return;
    const uint64_t at = n - dead + i;
    if (key[at] != kDeadPair) src[atomicAdd(counter, 1u)] = static_cast<uint32_t>(at);
}

// vacated slots of the head [0, n - dead) take the tail's live pairs
__global__ void pair_fill_kernel(uint64_t* key, double* sum, uint32_t* cnt, uint64_t n, uint64_t dead,
                                 const uint32_t* dead_list, const uint32_t* src, uint32_t* counter) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= dead) return;
    const uint32_t at = dead_list[i];
    if (at >= n - dead) return;
    const uint32_t from = src[atomicAdd(counter, 1u)];
    key[at] = key[from];
    sum[at] = sum[from];
    cnt[at] = cnt[from];
}

void launch_pair_compact(uint64_t* key, double* sum, uint32_t* cnt, uint64_t n, uint64_t dead,
                         const uint32_t* dead_list, uint32_t* src_list, uint32_t* counters,
                         cudaStream_t s) {
    if (!dead) return;
    cudaMemsetAsync(counters, 0, 8, s);
    pair_tail_live_kernel<<<grid_for(dead, 256), 256, 0, s>>>(key, n, dead, src_list, counters);
    pair_fill_kernel<<<grid_for(dead, 256), 256, 0, s>>>(key, sum, cnt, n, dead, dead_list, src_list,
                                                         counters + 1);
    count_launch();
    count_launch();
}

void launch_fold(const FoldParams& p, bool slow, cudaStream_t s) {
    if (!slow && p.n_heads && !p.runs_ready) {
        run_list_kernel<<<grid_for(p.n_heads, 256), 256, 0, s>>>(p.perm, p.hslot, p.hend, p.n_heads,
                                                                 const_cast<uint2*>(p.runs));
        count_launch();
    }
    if (p.n_journeys) {
        const unsigned lb = fold_grid(p.n_journeys, slow);
        if (slow) fold_lane_kernel<true><<<lb, kFoldWarps * 32, 0, s>>>(p);
        else fold_lane_kernel<false><<<lb, kFoldWarps * 32, 0, s>>>(p);
        count_launch();
    }
    spill_drain_kernel<<<grid_for(p.spill_mask + 1, 256), 256, 0, s>>>(p);
    count_launch();
}

void launch_run_list(const uint32_t* perm, const uint32_t* hslot, const uint32_t* hend, uint64_t n,
                     uint2* runs, cudaStream_t s) {
    if (!n) return;
    run_list_kernel<<<grid_for(n, 256), 256, 0, s>>>(perm, hslot, hend, n, runs);
    count_launch();
}

void launch_bin_pieces(const uint2* runs, uint64_t n_runs, const uint32_t* jstart, uint64_t J,
                       uint32_t* run_j, const uint32_t* code, uint32_t drc, int bin_bits, int run_bits,
                       uint64_t* keys, uint32_t* vals, uint2* pieces, uint32_t* counter,
                       uint64_t cap, cudaStream_t s) {
    if (!n_runs || !J) return;
    run_journey_kernel<<<grid_for(J, 256), 256, 0, s>>>(jstart, J, run_j);
    bin_pieces_kernel<<<grid_for(n_runs * 32, 256), 256, 0, s>>>(runs, n_runs, run_j, code, drc, bin_bits,
                                                                   run_bits, keys, vals, pieces, counter, cap);
    count_launch();
    count_launch();
}

void launch_bin_groups(const uint64_t* keys, const uint32_t* vals, const uint2* pieces, uint64_t n,
                       int order_bits, int bin_bits, uint32_t* flags, uint2* runs_out, cudaStream_t s) {
    (void)bin_bits;
    if (!n) return;
    bin_groups_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, vals, pieces, n, order_bits, flags, runs_out);
    count_launch();
}

void launch_bin_group_starts(const uint64_t* keys, const uint32_t* flags, const uint32_t* pos,
                             uint64_t n, int order_bits, int bin_bits, uint32_t* gstart,
                             uint32_t* gj, cudaStream_t s) {
    if (!n) return;
    bin_group_starts_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, flags, pos, n, order_bits, bin_bits,
                                                             gstart, gj);
    count_launch();
}

void launch_journey_len_keys(const uint32_t* jstart, uint64_t n, const uint2* runs, int runs_mode,
                             uint64_t* keys, uint32_t* vals, cudaStream_t s) {
    if (!n) return;
    journey_len_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(jstart, n, runs, runs_mode, keys, vals);
    count_launch();
}

void launch_rank_slot(const uint32_t* uslot, const uint32_t* perm, uint64_t n, uint32_t* rank_slot,
                      cudaStream_t s) {
    if (!n) return;
    rank_slot_kernel<<<grid_for(n, 256), 256, 0, s>>>(uslot, perm, n, rank_slot);
    count_launch();
}

void launch_export_pairs(const uint64_t* pkey, const double* psum, const uint32_t* pcnt, uint64_t n,
                         int rbits, const uint32_t* rank_slot, const unsigned long long* table,
                         uint64_t* cell, uint64_t* k0, uint64_t* k1, double* sum, uint64_t* cnt,
                         uint64_t stride, const uint32_t* grank, uint32_t* bad, cudaStream_t s) {
    if (!n) return;
    export_pairs_kernel<<<grid_for(n, 256), 256, 0, s>>>(pkey, psum, pcnt, n, rbits, rank_slot,
                                                         table, cell, k0, k1, sum, cnt, stride,
                                                         grank, bad);
    count_launch();
}

void launch_id_len(const uint32_t* rank_slot, const unsigned long long* table, uint64_t n,
                   uint32_t* len, cudaStream_t s) {
    if (!n) return;
    id_len_kernel<<<grid_for(n, 256), 256, 0, s>>>(rank_slot, table, n, len);
    count_launch();
}

void launch_id_copy(const uint32_t* rank_slot, const unsigned long long* table, const uint8_t* csv,
                    uint64_t n, const uint32_t* pos, uint8_t* blob, cudaStream_t s) {
    if (!n) return;
    id_copy_kernel<<<grid_for(n, 256), 256, 0, s>>>(rank_slot, table, csv, n, pos, blob);
    count_launch();
}

void launch_gather_u64(const uint64_t* src, uint64_t stride, const uint32_t* idx, uint64_t n,
                       uint64_t* dst, cudaStream_t s) {
    if (!n) return;
    gather_u64_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, stride, idx, n, dst);
    count_launch();
}

void launch_import_pairs(const double* sum, const uint64_t* cnt, uint64_t stride, uint64_t n,
                         double* psum, uint32_t* pcnt, cudaStream_t s) {
    if (!n) return;
    import_pairs_kernel<<<grid_for(n, 256), 256, 0, s>>>(sum, cnt, stride, n, psum, pcnt);
    count_launch();
}

void launch_pair_vals(uint32_t* vals, uint64_t n, cudaStream_t s) {
    if (!n) return;
    pair_vals_kernel<<<grid_for(n, 256), 256, 0, s>>>(vals, n);
    count_launch();
}

void launch_finalize(const uint64_t* keys, const uint32_t* vals, uint64_t n, int rank_bits,
                     const double* pair_sum, const uint32_t* pair_cnt, uint32_t D, uint64_t RC,
                     uint32_t t_base, uint32_t t_rows, uint32_t* planes, uint32_t* raw,
                     cudaStream_t s) {
    if (!n) return;
    finalize_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, vals, n, rank_bits, pair_sum, pair_cnt,
                                                     D, RC, t_base, t_rows, planes, raw);
    count_launch();
}

}  // namespace cvlg
