// Journey dictionary, canonical (journey, timestamp) ordering, dedup, per-(cell, journey) fold
// and the canonical per-cell finalize, for sm_100a.
//
// Reference semantics restated here (proj/src/aggregate.cpp):
//   dedup on (journey, epoch) with min-provenance survivor       :266-291
//   filter_reason on survivors                                   :293-303
//   journey ids -> lexicographic ranks, items sorted (rank, sec)  :305-328
//   cellmap[(g, rank)] += speed in (rank, sec) order              :331-358
//   finalize: sort by (g, journey), fold subtotals in journey order, f32 narrow :161-204
#include "agg_api.cuh"
#include "kernels.cuh"
#include "sort_api.cuh"

namespace cvlg {

namespace {

constexpr uint64_t kEmpty = ~0ull;

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

// ---- D1: dictionary insert (one thread per run head) -----------------------------------------
__global__ void dict_insert_kernel(const uint64_t* hk0, const uint64_t* hk1, const uint64_t* hidref,
                                   const uint64_t* hhash, uint64_t n_heads, const uint8_t* csv,
                                   unsigned long long* table, uint64_t mask, uint32_t* hdict,
                                   uint64_t* stats, unsigned long long* max_len) {
    const uint64_t h = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (h >= n_heads) return;
    uint64_t e0, e1, slot;
    const uint64_t k1 = hk1[h];
    const bool is_long = (k1 & 0xFF) == 0xFF;
    uint32_t len;
    uint64_t off = 0;
    if (!is_long) {
        e0 = hk0[h];
        e1 = k1;
        len = static_cast<uint32_t>(k1 & 0xFF);
        slot = mix64(e0 ^ mix64(e1)) & mask;
    } else {
        const uint64_t ref = hidref[h];
        off = ref >> 24;
        len = static_cast<uint32_t>(ref & 0xFFFFFF);
        e0 = (hhash[h] & ~0xFFFFFFull) | len;
        e1 = (off << 8) | 0xFF;
        slot = mix64(hhash[h]) & mask;
    }
    if (len) atomicMax(max_len, static_cast<unsigned long long>(len));
    for (uint64_t probe = 0; probe <= mask; ++probe) {
        uint64_t o0, o1;
        cas128(&table[2 * slot], kEmpty, kEmpty, e0, e1, o0, o1);
        if (o0 == kEmpty && o1 == kEmpty) break;  // inserted
        if (!is_long) {
            if (o0 == e0 && o1 == e1) break;
        } else if ((o1 & 0xFF) == 0xFF && o0 == e0) {
            if (bytes_equal(csv + (o1 >> 8), csv + off, len)) break;
        }
        slot = (slot + 1) & mask;
    }
    hdict[h] = static_cast<uint32_t>(slot);
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
// perm[i], for the LSD string sort.
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
    const uint64_t t = static_cast<uint64_t>(ts[hslot[h]] - ts_min);
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
                                        const uint32_t* hslot, const int64_t* ts, uint64_t n_heads,
                                        uint64_t n_slots, uint32_t* jstart, uint32_t* invalid) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n_heads) return;
    const uint32_t h = perm[i];
    const uint32_t r = hrank[h];
    if (i == 0 || hrank[perm[i - 1]] != r) {
        jstart[r] = static_cast<uint32_t>(i);
        return;
    }
    const uint32_t hp = perm[i - 1];
    const uint64_t end_prev = (hp + 1 < n_heads) ? hslot[hp + 1] : n_slots;
    const int64_t last_prev = ts[end_prev - 1];
    const int64_t first_cur = ts[hslot[h]];
    if (!(last_prev < first_cur)) *invalid = 1u;
}

// ---- S: slow path: per-slot journey rank, sort keys ------------------------------------------
__global__ void slot_keys_kernel(const uint32_t* hslot, const uint32_t* hrank, uint64_t n_heads,
                                 const int64_t* ts, uint64_t n_slots, int64_t ts_min, int tsbits,
                                 int mode, uint64_t* keys, uint32_t* vals, uint32_t* srank) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n_slots) return;
    // run = last head with hslot <= i
    uint64_t lo = 0, hi = n_heads;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (hslot[mid] <= i) lo = mid;
        else hi = mid;
    }
    const uint32_t r = hrank[lo];
    const uint64_t t = static_cast<uint64_t>(ts[i] - ts_min);
    keys[i] = mode == 0 ? ((static_cast<uint64_t>(r) << tsbits) | t) : t;
    vals[i] = static_cast<uint32_t>(i);
    srank[i] = r;
}

__global__ void slot_jstart_kernel(const uint32_t* perm, const uint32_t* srank, uint64_t n,
                                   uint32_t* jstart) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = srank[perm[i]];
    if (i == 0 || srank[perm[i - 1]] != r) jstart[r] = static_cast<uint32_t>(i);
}

// ---- payload re-parse for the duplicate-conflict check (aggregate.cpp:286) -------------------
__device__ bool parse_at(const FoldParams& P, uint64_t loff, Parsed& pr, const uint8_t*& line) {
    uint32_t lo = 0, hi = P.n_shards;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (P.shard_off[mid] <= loff) lo = mid;
        else hi = mid;
    }
    const uint64_t s_end = P.shard_off[lo + 1];
    uint64_t e = loff;
    while (e < s_end && P.csv[e] != '\n') ++e;
    int32_t len = static_cast<int32_t>(e - loff);
    line = P.csv + loff;
    if (len > 0 && line[len - 1] == '\r') --len;
    return parse_line(line, len, P.cmap[lo], pr) == kAccepted;
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

// ---- F: per-journey fold into the (cell, journey) table --------------------------------------
__device__ __forceinline__ uint64_t pair_find_or_insert(const FoldParams& P, uint64_t key,
                                                        bool& fresh) {
    uint64_t slot = mix64(key) & P.pair_mask;
    for (uint64_t probe = 0; probe <= P.pair_mask; ++probe) {
        const unsigned long long old =
            atomicCAS(reinterpret_cast<unsigned long long*>(&P.pair_key[slot]), kEmpty, key);
        if (old == kEmpty) {
            fresh = true;
            return slot;
        }
        if (old == key) {
            fresh = false;
            return slot;
        }
        slot = (slot + 1) & P.pair_mask;
    }
    fresh = false;
    return kEmpty;  // table full (bounded by construction)
}

template <bool kSlow>
__global__ void __launch_bounds__(128) fold_kernel(FoldParams P) {
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    uint32_t c_acc = 0, c_oog = 0, c_spd = 0, c_miss = 0, c_unb = 0, c_dup = 0, c_conf = 0,
             c_ovf = 0;
    if (j < P.n_journeys) {
        const uint64_t rank_bits = static_cast<uint64_t>(j);
        uint32_t cur_code = kCodeOutOfGrid;  // "none"
        uint64_t cur_slot = kEmpty;
        double cur_sum = 0.0;
        uint32_t cur_cnt = 0;
        const uint32_t b = P.jstart[j], e = P.jstart[j + 1];
        int64_t prev_ts = 0;
        uint64_t surv_slot = 0;
        bool have_prev = false;
        // iterate the journey's records in (rank, ts) order
        uint32_t i = b;
        uint64_t run_pos = 0, run_end = 0;
        while (true) {
            uint64_t slot;
            if (kSlow) {
                if (i >= e) break;
                slot = P.perm[i++];
            } else {
                if (run_pos >= run_end) {
                    if (i >= e) break;
                    const uint32_t h = P.perm[i++];
                    run_pos = P.hslot[h];
                    run_end = (h + 1 < P.n_heads) ? P.hslot[h + 1] : P.n_slots;
                }
                slot = run_pos++;
            }
            if (kSlow) {
                const int64_t t = P.ts[slot];
                if (have_prev && t == prev_ts) {
                    ++c_dup;
                    if (!payload_equal(P, P.loff[slot], P.loff[surv_slot])) ++c_conf;
                    continue;
                }
                have_prev = true;
                prev_ts = t;
                surv_slot = slot;
            }
            const uint32_t code = P.code[slot];
            if (code >= kCodeFirstSpecial) {
                if (code == kCodeOutOfGrid) ++c_oog;
                else if (code == kCodeSpeedCeiling) ++c_spd;
                else if (code == kCodeMissingField) ++c_miss;
                else ++c_unb;
                continue;
            }
            ++c_acc;
            const double v = P.speed[slot];
            if (code != cur_code) {
                if (cur_slot != kEmpty) {
                    P.pair_sum[cur_slot] = cur_sum;
                    P.pair_cnt[cur_slot] = cur_cnt;
                }
                bool fresh;
                cur_slot = pair_find_or_insert(P, (static_cast<uint64_t>(code) << 32) | rank_bits, fresh);
                if (cur_slot == kEmpty) {
                    ++c_ovf;
                    cur_code = kCodeOutOfGrid;
                    continue;
                }
                cur_code = code;
                if (fresh) {
                    cur_sum = 0.0;
                    cur_cnt = 0;
                } else {
                    cur_sum = P.pair_sum[cur_slot];
                    cur_cnt = P.pair_cnt[cur_slot];
                }
            }
            cur_sum = __dadd_rn(cur_sum, v);  // left fold in (rank, ts) order (aggregate.cpp:354)
            ++cur_cnt;
        }
        if (cur_slot != kEmpty) {
            P.pair_sum[cur_slot] = cur_sum;
            P.pair_cnt[cur_slot] = cur_cnt;
        }
    }
    unsigned long long v[8] = {c_acc, c_oog, c_spd, c_miss, c_unb, c_dup, c_conf, c_ovf};
    const int idx[8] = {kStAccepted, kStFiltOutOfGrid, kStFiltSpeed, kStFiltMissing,
                        kStUnbinnable, kStDups, kStConflicts, kStOverflow};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned long long s = warp_sum(v[k]);
        if ((threadIdx.x & 31) == 0 && s)
            atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[idx[k]]), s);
    }
}

// ---- P: pairs -> sorted (g, rank) ------------------------------------------------------------
__global__ void pair_flags_kernel(const uint64_t* pair_key, uint64_t cap, uint32_t* flags) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= cap) return;
    flags[i] = pair_key[i] != kEmpty ? 1u : 0u;
}

__global__ void pair_compact_kernel(const uint64_t* pair_key, const uint32_t* flags,
                                    const uint32_t* pos, uint64_t cap, int rank_bits,
                                    uint64_t* keys, uint32_t* vals) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= cap || !flags[i]) return;
    const uint64_t k = pair_key[i];
    const uint64_t g = k >> 32, r = k & 0xFFFFFFFFull;
    keys[pos[i]] = (g << rank_bits) | r;
    vals[pos[i]] = static_cast<uint32_t>(i);
}

// ---- Z: canonical per-cell fold (finalize_range, aggregate.cpp:161-187) ----------------------
__global__ void finalize_kernel(const uint64_t* keys, const uint32_t* vals, uint64_t n,
                                int rank_bits, const double* pair_sum, const uint32_t* pair_cnt,
                                uint32_t D, uint64_t RC, uint32_t* planes, uint32_t* raw) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t g = keys[i] >> rank_bits;
    if (i > 0 && (keys[i - 1] >> rank_bits) == g) return;
    double sum = 0.0;
    uint64_t cnt = 0;
    uint32_t vol = 0;
    for (uint64_t k = i; k < n && (keys[k] >> rank_bits) == g; ++k) {
        sum = __dadd_rn(sum, pair_sum[vals[k]]);  // journey-lexicographic order
        cnt += pair_cnt[vals[k]];
        ++vol;
    }
    const uint64_t t = g / (D * RC);
    const uint64_t d = (g / RC) % D;
    const uint64_t rc = g % RC;
    const float mean = __double2float_rn(__ddiv_rn(sum, static_cast<double>(cnt)));
    planes[(t * 8 + d) * RC + rc] = __float_as_uint(mean);
    planes[(t * 8 + 4 + d) * RC + rc] = vol;
    if (raw) raw[(t * 4 + d) * RC + rc] = static_cast<uint32_t>(cnt);
}

inline unsigned grid_for(uint64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

// ================================ host launchers ================================================
void launch_dict_insert(const DecodeOut& d, uint64_t n_heads, const uint8_t* csv,
                        unsigned long long* table, uint64_t mask, uint32_t* hdict, uint64_t* stats,
                        unsigned long long* max_len, cudaStream_t s) {
    if (!n_heads) return;
    dict_insert_kernel<<<grid_for(n_heads, 256), 256, 0, s>>>(d.hk0, d.hk1, d.hidref, d.hhash,
                                                              n_heads, csv, table, mask, hdict,
                                                              stats, max_len);
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
                             const int64_t* ts, uint64_t n_heads, uint64_t n_slots,
                             uint32_t* jstart, uint32_t* invalid, cudaStream_t s) {
    head_order_check_kernel<<<grid_for(n_heads, 256), 256, 0, s>>>(perm, hrank, hslot, ts,
                                                                   n_heads, n_slots, jstart,
                                                                   invalid);
    count_launch();
}

void launch_slot_keys(const uint32_t* hslot, const uint32_t* hrank, uint64_t n_heads,
                      const int64_t* ts, uint64_t n_slots, int64_t ts_min, int tsbits, int mode,
                      uint64_t* keys, uint32_t* vals, uint32_t* srank, cudaStream_t s) {
    slot_keys_kernel<<<grid_for(n_slots, 256), 256, 0, s>>>(hslot, hrank, n_heads, ts, n_slots,
                                                            ts_min, tsbits, mode, keys, vals,
                                                            srank);
    count_launch();
}

void launch_slot_jstart(const uint32_t* perm, const uint32_t* srank, uint64_t n, uint32_t* jstart,
                        cudaStream_t s) {
    slot_jstart_kernel<<<grid_for(n, 256), 256, 0, s>>>(perm, srank, n, jstart);
    count_launch();
}

void launch_fold(const FoldParams& p, bool slow, cudaStream_t s) {
    if (!p.n_journeys) return;
    if (slow) fold_kernel<true><<<grid_for(p.n_journeys, 128), 128, 0, s>>>(p);
    else fold_kernel<false><<<grid_for(p.n_journeys, 128), 128, 0, s>>>(p);
    count_launch();
}

void launch_pair_flags(const uint64_t* pair_key, uint64_t cap, uint32_t* flags, cudaStream_t s) {
    pair_flags_kernel<<<grid_for(cap, 256), 256, 0, s>>>(pair_key, cap, flags);
    count_launch();
}

void launch_pair_compact(const uint64_t* pair_key, const uint32_t* flags, const uint32_t* pos,
                         uint64_t cap, int rank_bits, uint64_t* keys, uint32_t* vals,
                         cudaStream_t s) {
    pair_compact_kernel<<<grid_for(cap, 256), 256, 0, s>>>(pair_key, flags, pos, cap, rank_bits,
                                                           keys, vals);
    count_launch();
}

void launch_finalize(const uint64_t* keys, const uint32_t* vals, uint64_t n, int rank_bits,
                     const double* pair_sum, const uint32_t* pair_cnt, uint32_t D, uint64_t RC,
                     uint32_t* planes, uint32_t* raw, cudaStream_t s) {
    if (!n) return;
    finalize_kernel<<<grid_for(n, 256), 256, 0, s>>>(keys, vals, n, rank_bits, pair_sum, pair_cnt,
                                                     D, RC, planes, raw);
    count_launch();
}

}  // namespace cvlg
