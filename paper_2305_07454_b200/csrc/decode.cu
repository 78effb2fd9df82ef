// K0 (shard header map) and K1 (tile decode) for sm_100a.
//
// K1 makes a single pass over the concatenated CSV shards in HBM. Each CTA takes one 16 KB tile
// (dynamic tile order, so decoupled look-back always makes progress) and:
//   1. stages tile + 1 KB halo (+16 B before) in shared memory with one TMA bulk copy
//      (cp.async.bulk + mbarrier); edge tiles use bounded vector loads;
//   2. builds '\n' and ',' bitmaps cooperatively (SIMD-within-a-register byte compares);
//   3. lists the DATA lines that start in the tile (non-empty, not a header, good shard) — this
//      needs no parsing, so the tile publishes its line count to the decoupled look-back
//      immediately and learns its global slot base before any record is parsed;
//   4. parses one line per thread: a fast path for plain fields (comma bitmap walk, fixed
//      19-byte timestamp, Clinger decimal conversion), falling back to the general restatement
//      of parse_record_impl (parse.cuh) for anything unusual; then filter + binning (grid.cuh);
//   5. marks run heads (journey id changes or timestamp stops increasing vs. the previous data
//      line) and writes ts / speed / cell code / line offset at slot = base + line index, so
//      consecutive threads write consecutive slots.
// Slots follow byte order; shards are concatenated in lexicographic path order, so slot order
// equals the reference's (shard_rank, line) provenance order (aggregate.cpp:287-289).
#include "kernels.cuh"

namespace cvlg {

namespace {

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                  1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                  1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra.uni DONE%=;\n\t"
        "bra.uni WAIT%=;\n"
        "DONE%=:\n\t}" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// bit i set iff byte i (of 16) equals c4's byte value
__device__ __forceinline__ uint32_t eq_mask16(uint4 v, uint32_t c4) {
    uint32_t m = 0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t eq = __vcmpeq4(w[k], c4) & 0x08040201u;
        m |= ((eq * 0x01010101u) >> 24) << (4 * k);
    }
    return m;
}

// [-]digits[.digits] with <= 19 digits and mantissa <= 2^53: the Clinger case of
// parse_double, computed identically (one correctly rounded IEEE operation). Returns false
// when the general parser must decide (anything else, including trim characters).
__device__ __forceinline__ bool fast_number(const uint8_t* __restrict__ s, uint32_t n, double& v) {
    uint32_t i = 0;
    const bool neg = s[0] == '-';
    if (neg) i = 1;
    uint32_t w32 = 0;  // first 9 digits in 32-bit arithmetic
    uint32_t nd = 0, dot = 0xFFFFFFFFu;
    for (; i < n && nd < 9; ++i) {
        const uint32_t d = static_cast<uint32_t>(s[i]) - '0';
        if (d < 10) {
            w32 = w32 * 10 + d;
            ++nd;
        } else if (d == static_cast<uint32_t>('.' - '0') && dot == 0xFFFFFFFFu) {
            dot = nd;
        } else {
            return false;
        }
    }
    uint64_t w = w32;
    for (; i < n; ++i) {
        const uint32_t d = static_cast<uint32_t>(s[i]) - '0';
        if (d < 10) {
            w = w * 10 + d;
            ++nd;
        } else if (d == static_cast<uint32_t>('.' - '0') && dot == 0xFFFFFFFFu) {
            dot = nd;
        } else {
            return false;
        }
    }
    if (nd == 0 || nd > 19 || w > (1ull << 53)) return false;
    const uint32_t fd = dot == 0xFFFFFFFFu ? 0u : nd - dot;
    const double m = static_cast<double>(w);
    const double r = fd ? __ddiv_rn(m, kPow10[fd]) : m;
    v = neg ? -r : r;
    return true;
}

struct LineOut {
    int64_t ts;
    double lat, lon, speed, heading;
    uint32_t id_rel, id_len;  // tile-relative id span
};

constexpr uint8_t kNeedGeneral = 255;

// Fast path of parse_record_impl for a line entirely staged in shared memory whose required
// fields are all plain: returns kAccepted or kRangeViolation, or kNeedGeneral whenever the
// general restatement (parse_line) has to decide (trim characters, empty/missing fields, bad
// timestamps, non-Clinger numbers, required columns beyond the 8th field).
__device__ __forceinline__ uint8_t fast_parse(const uint8_t* __restrict__ tile,
                                              const uint32_t* __restrict__ cm, uint32_t p,
                                              uint32_t e, const ColumnMap& map, LineOut& o) {
    // positions of the first 8 commas (e when absent)
    uint32_t c[8];
    {
        uint32_t w = p >> 5;
        uint32_t m = cm[w] & (0xFFFFFFFFu << (p & 31));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            while (m == 0 && ((w + 1) << 5) < e) m = cm[++w];
            uint32_t x = e;
            if (m) {
                const uint32_t pos = (w << 5) + (__ffs(m) - 1);
                m &= m - 1;
                if (pos < e) x = pos;
            }
            c[k] = x;
        }
    }
    auto fbeg = [&](int32_t f) -> uint32_t {
        uint32_t b = p;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (f == k + 1) b = c[k] + 1;
        return b;
    };
    auto fend = [&](int32_t f) -> uint32_t {
        uint32_t x = e;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (f == k) x = c[k];
        return x;
    };
    const int32_t cols[6] = {map.journey_id, map.timestamp, map.latitude,
                             map.longitude, map.speed,     map.heading};
    uint32_t fb[6], fe[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        if (cols[k] > 7) return kNeedGeneral;
        fb[k] = fbeg(cols[k]);
        fe[k] = fend(cols[k]);
        // a field that runs into the end of the line without its comma does not exist
        if (fb[k] > e) return kNeedGeneral;
        if (fe[k] <= fb[k]) return kNeedGeneral;  // empty (MissingField) -> general decides
    }
    // id must not need trimming; numbers/timestamp reject trim characters themselves
    if (is_trim(tile[fb[0]]) || is_trim(tile[fe[0] - 1])) return kNeedGeneral;
    if (fe[1] - fb[1] != 19 || !parse_timestamp(tile + fb[1], 19, o.ts)) return kNeedGeneral;
    if (!fast_number(tile + fb[2], fe[2] - fb[2], o.lat) ||
        !fast_number(tile + fb[3], fe[3] - fb[3], o.lon) ||
        !fast_number(tile + fb[4], fe[4] - fb[4], o.speed) ||
        !fast_number(tile + fb[5], fe[5] - fb[5], o.heading))
        return kNeedGeneral;
    if (o.heading == 360.0) o.heading = 0.0;
    o.id_rel = fb[0];
    o.id_len = fe[0] - fb[0];
    if (!(o.lat >= -90.0 && o.lat <= 90.0) || !(o.lon >= -180.0 && o.lon <= 180.0) ||
        !(o.speed >= 0.0) || !(o.heading >= 0.0 && o.heading < 360.0))
        return kRangeViolation;  // fast numbers are always finite
    return kAccepted;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// K0: one thread per shard. Header = first line (ingest.cpp:204-221).
__global__ void parse_headers_kernel(const uint8_t* csv, const uint64_t* shard_off,
                                     uint32_t n_shards, ColumnMap* cmap, uint8_t* good,
                                     uint64_t* stats) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_shards) return;
    const uint64_t b = shard_off[s], e = shard_off[s + 1];
    ColumnMap m;
    if (b == e) {  // empty file: zero rows, no header, no rejection
        good[s] = 0;
        m.journey_id = m.timestamp = m.latitude = m.longitude = m.postal_code = m.speed =
            m.heading = -1;
        m.n_columns = 0;
        cmap[s] = m;
        return;
    }
    uint64_t x = b;
    while (x < e && csv[x] != '\n') ++x;
    uint64_t n = x - b;
    if (n > 0 && csv[b + n - 1] == '\r') --n;
    const bool ok = parse_header(csv + b, static_cast<int64_t>(n), m);
    good[s] = ok ? 1 : 0;
    cmap[s] = m;
    if (!ok) atomicAdd(reinterpret_cast<unsigned long long*>(&stats[kStBadHeader]), 1ull);
}

void launch_parse_headers(const uint8_t* csv, const uint64_t* shard_off, uint32_t n_shards,
                          ColumnMap* cmap, uint8_t* good, uint64_t* stats, cudaStream_t s) {
    if (n_shards == 0) return;
    parse_headers_kernel<<<(n_shards + 127) / 128, 128, 0, s>>>(csv, shard_off, n_shards, cmap,
                                                                 good, stats);
}

// ---------------------------------------------------------------------------------------------
// K1
constexpr int kStage = kPre + kTile + kHalo;
constexpr int kWords = (kTile + kHalo) / 32;
constexpr int kMaxShardsInTile = 32;

__global__ void __launch_bounds__(kDecodeThreads, 4) decode_kernel(DecodeParams P) {
    __shared__ __align__(128) uint8_t buf[kStage];
    __shared__ uint32_t nl[kWords];
    __shared__ uint32_t cm[kWords];
    __shared__ uint32_t starts[kLineCap];  // p_rel | shard_delta << 16
    __shared__ uint32_t scan_smem[kDecodeThreads / 32 + 1];
    __shared__ uint64_t sh_off[kMaxShardsInTile + 2];
    __shared__ uint32_t sh_first, sh_count, sh_overflow, s_tile;
    __shared__ unsigned long long s_base;
    __shared__ __align__(8) uint64_t bar;
    // parsed lines of the current pass (staged until the slot base is known)
    __shared__ long long st_ts[kLineCap];
    __shared__ double st_speed[kLineCap];
    __shared__ uint32_t st_code[kLineCap];
    __shared__ uint32_t st_id[kLineCap];   // tile-relative id start
    __shared__ uint32_t st_len[kLineCap];  // id length | accepted << 31
    __shared__ long long c_ts;
    __shared__ uint32_t c_id, c_len, c_code;
    __shared__ uint32_t s_cnt[8];  // rejects[4], heads, transitions, accepted
    __shared__ uint64_t s_lb[kDecodeThreads / 32 + 2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_tile = atomicAdd(P.tile_counter, 1u);
        mbar_init(&bar, 1);
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= P.tile_end) return;

    const uint64_t tb = static_cast<uint64_t>(tile) * kTile;
    const uint64_t te = min(tb + kTile, P.total_end);
    const uint32_t tlen = static_cast<uint32_t>(te - tb);
    const uint64_t stage_end = min(tb + kTile + kHalo, P.avail_end);
    const uint32_t staged_len = static_cast<uint32_t>(stage_end - tb);  // valid bytes from tb
    const uint8_t* tile_s = buf + kPre;

    // ---- 1. stage bytes --------------------------------------------------------------------
    const bool use_tma = P.aligned16 && tb >= kPre && tb + kTile + kHalo <= P.avail_end;
    if (use_tma) {
        if (tid == 0) {
            mbar_expect_tx(&bar, kStage);
            tma_load_1d(buf, P.csv + tb - kPre, kStage, &bar);
        }
    } else {
        for (int v = tid; v < kStage; v += kDecodeThreads) {
            const int64_t a = static_cast<int64_t>(tb) - kPre + v;
            buf[v] = a < 0 ? uint8_t('\n')
                           : (static_cast<uint64_t>(a) < stage_end ? P.csv[a] : uint8_t(0));
        }
    }
    if (tid == 32) {  // shard containing tb (overlaps the copy)
        uint32_t lo = 0, hi = P.n_shards;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (P.shard_off[mid] <= tb) lo = mid;
            else hi = mid;
        }
        sh_first = lo;
        uint32_t c = 0, s = lo + 1;
        while (s <= P.n_shards && P.shard_off[s] < te && c < kMaxShardsInTile) sh_off[c++] = P.shard_off[s++];
        sh_overflow = (s <= P.n_shards && P.shard_off[s] < te) ? 1u : 0u;
        sh_count = c;
    }
    if (use_tma) mbar_wait(&bar, 0);
    __syncthreads();

    // ---- 2. '\n' and ',' bitmaps over [tb, tb + kTile + kHalo) ---------------------------------
    for (int w = tid; w < kWords; w += kDecodeThreads) {
        const uint4* p = reinterpret_cast<const uint4*>(tile_s + 32 * w);
        const uint4 a = p[0], b = p[1];
        nl[w] = eq_mask16(a, 0x0A0A0A0Au) | (eq_mask16(b, 0x0A0A0A0Au) << 16);
        cm[w] = eq_mask16(a, 0x2C2C2C2Cu) | (eq_mask16(b, 0x2C2C2C2Cu) << 16);
    }
    __syncthreads();

    auto shard_of = [&](uint64_t p) -> uint32_t {
        if (!sh_overflow) {
            uint32_t s = sh_first;
            for (uint32_t k = 0; k < sh_count; ++k)
                if (sh_off[k] <= p) s = sh_first + 1 + k;
            return s;
        }
        uint32_t lo = 0, hi = P.n_shards;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (P.shard_off[mid] <= p) lo = mid;
            else hi = mid;
        }
        return lo;
    };

    // ---- 3. data lines starting in [0, tlen) ----------------------------------------------------
    // thread t owns tile words 2t, 2t+1 (kTile / 32 = 512 words)
    uint32_t smask[2];
    uint32_t my_count = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int w = 2 * tid + k;
        const uint32_t prev_top = (w == 0) ? (buf[kPre - 1] == '\n' ? 1u : 0u) : (nl[w - 1] >> 31);
        uint32_t m = (nl[w] << 1) | prev_top;
        const int lo = 32 * w;
        if (lo >= static_cast<int>(tlen)) m = 0;
        else if (lo + 32 > static_cast<int>(tlen)) m &= (1u << (tlen - lo)) - 1u;
        // keep only data lines: not a shard start (header), good shard, non-empty
        uint32_t keep = m;
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t pr = static_cast<uint32_t>(lo + bit);
            const uint64_t p = tb + pr;
            const uint32_t s = shard_of(p);
            const uint64_t s_end = P.shard_off[s + 1];
            bool data = p != P.shard_off[s] && P.shard_good[s];
            if (data) {
                const uint8_t c0 = tile_s[pr];
                if (c0 == '\n') data = false;
                else if (c0 == '\r' && (p + 1 == s_end || tile_s[pr + 1] == '\n')) data = false;
            }
            if (!data) keep &= ~(1u << bit);
        }
        smask[k] = keep;
        my_count += __popc(keep);
    }
    uint32_t n_data;
    const uint32_t my_off = block_exclusive_scan<kDecodeThreads>(my_count, scan_smem, n_data);

    // ---- publish the tile's line count now; resolve the slot base after parsing ------------------
    if (tid == 0) lookback1_publish(P.lb, tile, n_data);
    if (tid < 8) s_cnt[tid] = 0;
    if (tid == 0) {
        c_len = 0;  // "no previous data line" for the first line of the tile
        c_ts = 0;
        c_id = 0;
        c_code = kCodeRejected;
    }
    uint64_t base = 0;
    bool resolved = false;
    long long ts_min = LLONG_MAX, ts_max = LLONG_MIN;
    uint32_t c_acc = 0;

    for (uint32_t pass_base = 0; pass_base < n_data; pass_base += kLineCap) {
        {
            uint32_t idx = my_off;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                uint32_t m = smask[k];
                while (m) {
                    const int bit = __ffs(m) - 1;
                    m &= m - 1;
                    if (idx >= pass_base && idx < pass_base + kLineCap)
                        starts[idx - pass_base] = static_cast<uint32_t>(32 * (2 * tid + k) + bit);
                    ++idx;
                }
            }
        }
        __syncthreads();
        const uint32_t n_pass = min(static_cast<uint32_t>(kLineCap), n_data - pass_base);
        // ---- 4. parse: one data line per thread, results staged in shared memory -----------------
        for (uint32_t li = tid; li < n_pass; li += kDecodeThreads) {
            uint8_t why;
            LineOut o;
            o.ts = 0;
            o.speed = 0.0;
            o.id_rel = 0;
            o.id_len = 0;
            uint32_t code = kCodeRejected;
            const uint32_t p_rel = starts[li];
            const uint64_t p = tb + p_rel;
            const uint32_t s = shard_of(p);
            const uint64_t s_end = P.shard_off[s + 1];
            // line end: next '\n' at or after p, clamped to the shard end
            uint64_t e = 0;
            bool found = false;
            {
                uint32_t w = p_rel >> 5;
                uint32_t m = nl[w] & (0xFFFFFFFFu << (p_rel & 31));
                while (true) {
                    if (m) {
                        const uint32_t x = 32 * w + (__ffs(m) - 1);
                        if (x < staged_len) {
                            e = tb + x;
                            found = true;
                        }
                        break;
                    }
                    if (++w >= static_cast<uint32_t>(kWords) || 32 * w >= staged_len) break;
                    m = nl[w];
                }
            }
            if (!found) {
                uint64_t x = tb + staged_len;
                while (x < P.avail_end && x < s_end && P.csv[x] != '\n') ++x;
                e = x;
            }
            if (e > s_end) e = s_end;
            const bool in_smem = e <= stage_end;
            const uint8_t* gline = P.csv + p;
            uint32_t len = static_cast<uint32_t>(e - p);
            const uint8_t last = in_smem ? tile_s[p_rel + len - 1] : gline[len - 1];
            if (last == '\r') --len;  // len > 0: empty lines are not data lines
            const ColumnMap map = P.cmap[s];
            why = kNeedGeneral;
            if (in_smem) why = fast_parse(tile_s, cm, p_rel, p_rel + len, map, o);
            if (why == kNeedGeneral) {
                const uint8_t* line = in_smem ? tile_s + p_rel : gline;
                Parsed pr;
                why = parse_line(line, static_cast<int32_t>(len), map, pr);
                if (why == kAccepted) {
                    o.ts = pr.epoch;
                    o.lat = pr.lat;
                    o.lon = pr.lon;
                    o.speed = pr.speed;
                    o.heading = pr.heading;
                    o.id_rel = p_rel + static_cast<uint32_t>(pr.id_begin);
                    o.id_len = static_cast<uint32_t>(pr.id_len);
                }
            }
            if (why == kAccepted) {
                code = cell_code(o.ts, o.lat, o.lon, o.speed, o.heading, P.grid);
                ts_min = min(ts_min, static_cast<long long>(o.ts));
                ts_max = max(ts_max, static_cast<long long>(o.ts));
                ++c_acc;
            } else {
                atomicAdd(&s_cnt[why - 1], 1u);  // rare
            }
            st_ts[li] = o.ts;
            st_speed[li] = o.speed;
            st_code[li] = code;
            st_id[li] = o.id_rel;
            st_len[li] = o.id_len | (why == kAccepted ? 0x80000000u : 0u);
        }
        if (!resolved) {
            // predecessors have had a full parse phase to publish: the walk is short
            base = lookback1_resolve<kDecodeThreads>(P.lb, tile, n_data, s_lb);
            resolved = true;
            if (tid == 0 && base + n_data > P.out.slot_cap)
                atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStOverflow]), 1ull);
        } else {
            __syncthreads();
        }
        const bool fits = base + n_data <= P.out.slot_cap;
        // ---- 5. run heads + coalesced writes ------------------------------------------------------
        uint32_t my_heads = 0, my_trans = 0;
        for (uint32_t k = tid; k < n_pass; k += kDecodeThreads) {
            const uint32_t ln = st_len[k];
            uint32_t code = st_code[k];
            if (ln >> 31) {
                const uint32_t pl = k ? st_len[k - 1] : c_len;
                const long long pts = k ? st_ts[k - 1] : c_ts;
                const uint32_t idl = ln & 0x7FFFFFFFu;
                bool head = true;
                if ((pl >> 31) && (pl & 0x7FFFFFFFu) == idl && pts < st_ts[k]) {
                    const uint32_t pid = k ? st_id[k - 1] : c_id;
                    const uint32_t mid = st_id[k];
                    const uint8_t* pa = (pid + idl <= staged_len) ? tile_s + pid : P.csv + tb + pid;
                    const uint8_t* pb = (mid + idl <= staged_len) ? tile_s + mid : P.csv + tb + mid;
                    bool same = true;
                    for (uint32_t i = 0; i < idl; ++i)
                        if (pa[i] != pb[i]) {
                            same = false;
                            break;
                        }
                    head = !same;
                }
                if (head) {
                    ++my_heads;
                    code |= kHeadBit;
                } else if ((k ? st_code[k - 1] : c_code) != code) {
                    ++my_trans;
                }
            }
            if (fits) {
                const uint64_t slot = base + pass_base + k;
                P.out.ts[slot] = st_ts[k];
                P.out.speed[slot] = st_speed[k];
                P.out.code[slot] = code;
                P.out.loff[slot] = tb + starts[k];
            }
        }
        if (my_heads) atomicAdd(&s_cnt[4], my_heads);
        if (my_trans) atomicAdd(&s_cnt[5], my_trans);
        __syncthreads();
        if (tid == 0) {  // carry the pass's last line
            c_ts = st_ts[n_pass - 1];
            c_id = st_id[n_pass - 1];
            c_len = st_len[n_pass - 1];
            c_code = st_code[n_pass - 1];
        }
        __syncthreads();
    }
    if (!resolved) lookback1_resolve<kDecodeThreads>(P.lb, tile, n_data, s_lb);

    // ---- stats -----------------------------------------------------------------------------------
    if (c_acc) atomicAdd(&s_cnt[6], c_acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ts_min = min(ts_min, __shfl_xor_sync(0xFFFFFFFFu, ts_min, o));
        ts_max = max(ts_max, __shfl_xor_sync(0xFFFFFFFFu, ts_max, o));
    }
    if ((tid & 31) == 0 && ts_min <= ts_max) {
        atomicMin(&P.ts_minmax[0], ts_min);
        atomicMax(&P.ts_minmax[1], ts_max);
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(P.stats);
        if (n_data) atomicAdd(&st[kStRowsRead], static_cast<unsigned long long>(n_data));
        for (int i = 0; i < 4; ++i)
            if (s_cnt[i]) atomicAdd(&st[kStRejBase + i], static_cast<unsigned long long>(s_cnt[i]));
        if (s_cnt[4]) atomicAdd(&st[kStHeads], static_cast<unsigned long long>(s_cnt[4]));
        if (s_cnt[5]) atomicAdd(&st[kStGTransitions], static_cast<unsigned long long>(s_cnt[5]));
        if (s_cnt[6]) atomicAdd(&st[kStParsed], static_cast<unsigned long long>(s_cnt[6]));
    }
}

void launch_decode(const DecodeParams& p, uint32_t n_ctas, cudaStream_t s) {
    if (n_ctas == 0) return;
    decode_kernel<<<n_ctas, kDecodeThreads, 0, s>>>(p);
}

}  // namespace cvlg
