// K0 (shard header map) and K1 (tile decode) for sm_100a.
//
// K1 makes a single pass over the concatenated CSV shards in HBM. Each CTA takes one 16 KB tile
// (dynamic tile order, so decoupled look-back always makes progress) and:
//   1. stages tile + 1 KB halo (+16 B before) in shared memory with one TMA bulk copy
//      (cp.async.bulk + mbarrier); edge tiles use bounded loads;
//   2. builds '\n' and ',' bitmaps cooperatively (SIMD-within-a-register zero-byte detection);
//   3. lists the DATA lines that start in the tile (non-empty, not a header, good shard) — this
//      needs no parsing, so the tile publishes its line count to the decoupled look-back at once
//      and resolves its slot base only after parsing (CTA-wide look-back window);
//   4. parses one line per thread. Fast path: field boundaries from a 96-bit register window of
//      the comma bitmap, the 19-byte timestamp from five 32-bit words, decimals digit by digit
//      from registers (Clinger: one correctly rounded division). Anything unusual (trim
//      characters, missing fields, non-Clinger numbers, non-canonical column maps, long lines)
//      goes to the general restatement of parse_record_impl (parse.cuh); then filter + binning
//      (grid.cuh);
//   5. marks run heads (journey id changes or timestamp stops increasing vs. the previous data
//      line) and writes ts / speed / cell code / line offset at slot = base + line index, so
//      consecutive threads write consecutive slots.
// Slots follow byte order; shards are concatenated in lexicographic path order, so slot order
// equals the reference's (shard_rank, line) provenance order (aggregate.cpp:287-289).
#include <algorithm>

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

// 4-bit mask: bit k set iff byte k of x equals the byte replicated in pat (exact zero-byte test,
// no cross-byte carries), compressed with one multiply.
__device__ __forceinline__ uint32_t eqmask4(uint32_t x, uint32_t pat) {
    const uint32_t t = x ^ pat;
    const uint32_t y = (t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
    const uint32_t z = ~(y | t) & 0x80808080u;
    return ((z >> 7) * 0x10204080u) >> 28;
}

// 32-bit little-endian word holding bytes [off, off + 4) of a 4-byte aligned shared buffer.
__device__ __forceinline__ uint32_t word_at(const uint32_t* w, uint32_t off) {
    const uint32_t i = off >> 2, sh = (off & 3) * 8;
    return __funnelshift_r(w[i], w[i + 1], sh);
}

__device__ __forceinline__ uint32_t byte_of(uint32_t w, uint32_t k) { return (w >> (8 * k)) & 0xFF; }

// Exact "YYYY-MM-DD HH:MM:SS" (datetime.cpp:53-75) from five little-endian words.
__device__ __forceinline__ bool fast_timestamp(const uint32_t* w, uint32_t off, int64_t& out) {
    const uint32_t t0 = word_at(w, off), t1 = word_at(w, off + 4), t2 = word_at(w, off + 8),
                   t3 = word_at(w, off + 12), t4 = word_at(w, off + 16);
    // separators at 4 '-', 7 '-', 10 ' ', 13 ':', 16 ':'
    if ((t1 & 0xFF0000FFu) != 0x2D00002Du || ((t2 >> 16) & 0xFF) != ' ' ||
        ((t3 >> 8) & 0xFF) != ':' || (t4 & 0xFF) != ':')
        return false;
    // the 14 digit positions, separators replaced by '0'
    const uint32_t a = t0, b = (t1 & 0x00FFFF00u) | 0x30000030u,
                   c = (t2 & 0xFF00FFFFu) | 0x00300000u, d = (t3 & 0xFFFF00FFu) | 0x00003000u,
                   e = (t4 & 0x00FFFF00u) | 0x30000030u;
    // byte in '0'..'9'  <=>  high nibble 3 and (byte + 6) keeps high nibble 3
    const uint32_t hi = ((a | b | c | d | e) & 0xC0C0C0C0u) |
                        (((a & b & c & d & e) & 0x30303030u) ^ 0x30303030u);
    const uint32_t lo = ((a + 0x06060606u) | (b + 0x06060606u) | (c + 0x06060606u) |
                         (d + 0x06060606u) | (e + 0x06060606u)) & 0x40404040u;
    if (hi != 0 || lo != 0) return false;
    const uint32_t da = a - 0x30303030u, db = b - 0x30303030u, dc = c - 0x30303030u,
                   dd = d - 0x30303030u, de = e - 0x30303030u;
    const int y = static_cast<int>(byte_of(da, 0) * 1000 + byte_of(da, 1) * 100 + byte_of(da, 2) * 10 +
                                   byte_of(da, 3));
    const int mo = static_cast<int>(byte_of(db, 1) * 10 + byte_of(db, 2));
    const int dy = static_cast<int>(byte_of(dc, 0) * 10 + byte_of(dc, 1));
    const int h = static_cast<int>(byte_of(dc, 3) * 10 + byte_of(dd, 0));
    const int mi = static_cast<int>(byte_of(dd, 2) * 10 + byte_of(dd, 3));
    const int s = static_cast<int>(byte_of(de, 1) * 10 + byte_of(de, 2));
    if (mo < 1 || mo > 12 || dy < 1 || dy > static_cast<int>(days_in_month(y, mo)) || h > 23 ||
        mi > 59 || s > 59)
        return false;
    out = days_from_civil(y, static_cast<unsigned>(mo), static_cast<unsigned>(dy)) * 86400 +
          h * 3600 + mi * 60 + s;
    return true;
}

__constant__ uint32_t kPow10u[9] = {1u, 10u, 100u, 1000u, 10000u, 100000u, 1000000u, 10000000u,
                                    100000000u};

// 4 ASCII digits (first = lowest byte = most significant) -> value
__device__ __forceinline__ uint32_t swar4(uint32_t v) {
    v &= 0x0F0F0F0Fu;
    v = (v * 10u + (v >> 8)) & 0x00FF00FFu;
    return (v * 100u + (v >> 16)) & 0xFFFFu;
}

// all four bytes in '0'..'9' (exact nibble test)
__device__ __forceinline__ bool all_digits4(uint32_t v) {
    return ((v & 0xF0F0F0F0u) | (((v + 0x06060606u) & 0xF0F0F0F0u) >> 4)) == 0x33333333u;
}

// value of the F (1..8) digits at bytes [at, at + F) of the shared buffer; false if any is not a
// digit. Reads the 8 bytes ending at the last digit and forces the leading 8 - F bytes to '0'.
__device__ __forceinline__ bool digits8(const uint32_t* w, uint32_t at, uint32_t F, uint32_t& val) {
    const uint32_t st = at + F - 8;
    uint32_t g0 = word_at(w, st), g1 = word_at(w, st + 4);
    const uint32_t k = 8 - F;  // leading pad bytes
    if (k >= 4) {
        g0 = 0x30303030u;
        const uint32_t m = k == 4 ? 0u : (0xFFFFFFFFu >> (8 * (8 - k)));
        g1 = (g1 & ~m) | (0x30303030u & m);
    } else if (k > 0) {
        const uint32_t m = 0xFFFFFFFFu >> (8 * (4 - k));
        g0 = (g0 & ~m) | (0x30303030u & m);
    }
    if (!all_digits4(g0) || !all_digits4(g1)) return false;
    val = swar4(g0) * 10000u + swar4(g1);
    return true;
}

// [-]I['.'F] with I <= 3 digits and F <= 8 digits (or an integer of <= 8 digits): the Clinger
// case of parse_double computed identically (w < 10^11 exact; one correctly rounded division
// by 10^F). SWAR digit conversion; false -> the general parser decides.
__device__ __forceinline__ bool fast_number(const uint32_t* w, uint32_t off, uint32_t n, double& v) {
    const bool neg = (word_at(w, off) & 0xFF) == '-';
    const uint32_t o = off + (neg ? 1u : 0u);
    const uint32_t m = n - (neg ? 1u : 0u);
    if (n == 0 || m == 0) return false;
    const uint32_t h = word_at(w, o);
    const uint32_t lim = m < 4 ? ((1u << m) - 1u) : 0xFu;
    const uint32_t dm = eqmask4(h, 0x2E2E2E2Eu) & lim;
    uint64_t mant;
    uint32_t fd;
    if (dm == 0) {  // integer
        if (m > 8) return false;
        uint32_t val;
        if (!digits8(w, o, m, val)) return false;
        mant = val;
        fd = 0;
    } else {
        const uint32_t L = __ffs(dm) - 1;  // digits before the dot (0..3)
        const uint32_t F = m - L - 1;      // digits after it
        if (F > 8 || L + F == 0) return false;
        const uint32_t d = h - 0x30303030u;
        const uint32_t b0 = d & 0xFF, b1 = (d >> 8) & 0xFF, b2 = (d >> 16) & 0xFF;
        uint32_t ip = 0;
        if (L >= 1) {
            if (b0 > 9) return false;
            ip = b0;
        }
        if (L >= 2) {
            if (b1 > 9) return false;
            ip = ip * 10 + b1;
        }
        if (L == 3) {
            if (b2 > 9) return false;
            ip = ip * 10 + b2;
        }
        uint32_t fp = 0;
        if (F && !digits8(w, o + L + 1, F, fp)) return false;
        mant = static_cast<uint64_t>(ip) * kPow10u[F] + fp;
        fd = F;
    }
    const double md = static_cast<double>(mant);
    const double r = fd ? __ddiv_rn(md, kPow10[fd]) : md;
    v = neg ? -r : r;
    return true;
}

struct LineOut {
    int64_t ts;
    double lat, lon, speed, heading;
    uint32_t id_rel, id_len;  // tile-relative id span
};

constexpr uint8_t kNeedGeneral = 255;

// Fast path of parse_record_impl for a line [p, e) (tile-relative) entirely staged in shared
// memory whose header is canonical: journey, timestamp, latitude, longitude as fields 0..3,
// then speed, heading as 5, 6 (`postal` = 1: any column at 4) or 4, 5. Returns kAccepted or
// kRangeViolation, or kNeedGeneral whenever the general restatement has to decide.
__device__ __forceinline__ uint8_t fast_parse(const uint8_t* __restrict__ tile,
                                              const uint32_t* __restrict__ cm, uint32_t p,
                                              uint32_t e, int postal, LineOut& o) {
    const uint32_t len = e - p;
    if (len > 95) return kNeedGeneral;
    // 96-bit comma window starting at bit p
    const uint32_t wi = p >> 5, sh = p & 31;
    const uint32_t a = cm[wi], b = cm[wi + 1], c = cm[wi + 2], d = cm[wi + 3];
    uint32_t m0 = __funnelshift_r(a, b, sh), m1 = __funnelshift_r(b, c, sh),
             m2 = __funnelshift_r(c, d, sh);
    if (len < 32) {
        m0 &= (1u << len) - 1u;
        m1 = m2 = 0;
    } else if (len < 64) {
        m1 &= (1u << (len - 32)) - 1u;
        m2 = 0;
    } else {
        m2 &= (1u << (len - 64)) - 1u;
    }
    // first 7 comma positions (relative to p); len when absent
    uint32_t cpos[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        uint32_t pos = len;
        if (m0) {
            pos = __ffs(m0) - 1;
            m0 &= m0 - 1;
        } else if (m1) {
            pos = 32 + __ffs(m1) - 1;
            m1 &= m1 - 1;
        } else if (m2) {
            pos = 64 + __ffs(m2) - 1;
            m2 &= m2 - 1;
        }
        cpos[k] = pos;
    }
    const uint32_t fe_id = cpos[0];
    const uint32_t fb_ts = cpos[0] + 1, fe_ts = cpos[1];
    const uint32_t fb_la = cpos[1] + 1, fe_la = cpos[2];
    const uint32_t fb_lo = cpos[2] + 1, fe_lo = cpos[3];
    const uint32_t fb_sp = postal ? cpos[4] + 1 : cpos[3] + 1;
    const uint32_t fe_sp = postal ? cpos[5] : cpos[4];
    const uint32_t fb_hd = postal ? cpos[5] + 1 : cpos[4] + 1;
    const uint32_t fe_hd = postal ? cpos[6] : cpos[5];
    // every required field must exist and be non-empty (else: general decides MissingField)
    if (fb_hd >= fe_hd || fe_id == 0 || fb_la >= fe_la || fb_lo >= fe_lo || fb_sp >= fe_sp)
        return kNeedGeneral;
    const uint8_t* q = tile + p;
    if (is_trim(q[0]) || is_trim(q[fe_id - 1])) return kNeedGeneral;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(tile - kPre);  // 16 B aligned
    const uint32_t base = p + kPre;
    if (fe_ts - fb_ts != 19 || !fast_timestamp(words, base + fb_ts, o.ts)) return kNeedGeneral;
    if (!fast_number(words, base + fb_la, fe_la - fb_la, o.lat) ||
        !fast_number(words, base + fb_lo, fe_lo - fb_lo, o.lon) ||
        !fast_number(words, base + fb_sp, fe_sp - fb_sp, o.speed) ||
        !fast_number(words, base + fb_hd, fe_hd - fb_hd, o.heading))
        return kNeedGeneral;
    if (o.heading == 360.0) o.heading = 0.0;
    o.id_rel = p;
    o.id_len = fe_id;
    if (!(o.lat >= -90.0 && o.lat <= 90.0) || !(o.lon >= -180.0 && o.lon <= 180.0) ||
        !(o.speed >= 0.0) || !(o.heading >= 0.0 && o.heading < 360.0))
        return kRangeViolation;  // fast numbers are always finite
    return kAccepted;
}

// The general restatement, kept out of line so the hot loop stays small in the I-cache.
__device__ __noinline__ uint8_t general_parse(const uint8_t* line, int32_t len, const ColumnMap& map,
                                              uint32_t p_rel, LineOut& o) {
    Parsed pr;
    const uint8_t why = parse_line(line, len, map, pr);
    if (why == kAccepted) {
        o.ts = pr.epoch;
        o.lat = pr.lat;
        o.lon = pr.lon;
        o.speed = pr.speed;
        o.heading = pr.heading;
        o.id_rel = p_rel + static_cast<uint32_t>(pr.id_begin);
        o.id_len = static_cast<uint32_t>(pr.id_len);
    }
    return why;
}

// 1 / 0: canonical column map with / without a column between longitude and speed; -1: general
__device__ __forceinline__ int canonical_kind(const ColumnMap& m) {
    if (m.journey_id != 0 || m.timestamp != 1 || m.latitude != 2 || m.longitude != 3) return -1;
    if (m.speed == 5 && m.heading == 6) return 1;
    if (m.speed == 4 && m.heading == 5) return 0;
    return -1;
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
// K1: persistent CTAs, static round-robin tiles (CTA c: tiles c, c + G, ...), double-buffered TMA
// prefetch of the next tile while the current one is parsed. Every CTA of the grid is
// co-resident (G <= occupancy x SMs), and a tile only ever waits on smaller tiles, so the
// decoupled look-back cannot deadlock: the smallest unfinished tile is always being processed.
constexpr int kStage = kPre + kTile + kHalo;
constexpr int kStageAlloc = kStage + 112;  // word_at() over-read padding, keeps 16 B alignment
constexpr int kWords = (kTile + kHalo) / 32;
constexpr int kMaxShardsInTile = 32;
constexpr int kDecodeCtasPerSm = 3;

struct DecodeSmem {
    uint8_t buf[2][kStageAlloc];
    uint32_t nl[kWords + 4];
    uint32_t cm[kWords + 4];
    uint32_t starts[kLineCap];
    long long st_ts[kLineCap];
    double st_speed[kLineCap];
    uint32_t st_code[kLineCap];
    uint32_t st_id[kLineCap];   // tile-relative id start
    uint32_t st_len[kLineCap];  // id length | accepted << 31
};

__global__ void __launch_bounds__(kDecodeThreads, kDecodeCtasPerSm) decode_kernel(DecodeParams P,
                                                                                  uint32_t tile_begin) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    DecodeSmem& S = *reinterpret_cast<DecodeSmem*>(smem_raw);
    __shared__ uint32_t scan_smem[kDecodeThreads / 32 + 1];
    __shared__ uint64_t sh_off[kMaxShardsInTile + 2];
    __shared__ uint32_t sh_first, sh_count, sh_overflow;
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ long long c_ts;
    __shared__ uint32_t c_id, c_len, c_code;
    __shared__ uint32_t s_cnt[8];  // rejects[4], heads, transitions, accepted, rows
    __shared__ uint64_t s_lb[kDecodeThreads / 32 + 2];

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    if (tid < 8) s_cnt[tid] = 0;
    __syncthreads();

    auto can_tma = [&](uint32_t t) {
        const uint64_t tb = static_cast<uint64_t>(t) * kTile;
        return P.aligned16 && tb >= kPre && tb + kTile + kHalo <= P.avail_end;
    };
    auto issue = [&](uint32_t t, int b) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[b], kStage);
        tma_load_1d(S.buf[b], P.csv + static_cast<uint64_t>(t) * kTile - kPre, kStage, &bar[b]);
    };
    uint32_t phase0 = 0, phase1 = 0;
    uint32_t c_acc = 0;
    const uint32_t G = gridDim.x;
    uint32_t tile = tile_begin + blockIdx.x;
    if (tid == 0 && tile < P.tile_end && can_tma(tile)) issue(tile, 0);

    for (uint32_t it = 0; tile < P.tile_end; ++it, tile += G) {
        const int b = it & 1;
        const uint32_t nxt = tile + G;
        if (tid == 0 && nxt < P.tile_end && can_tma(nxt)) issue(nxt, b ^ 1);

        const uint64_t tb = static_cast<uint64_t>(tile) * kTile;
        const uint64_t te = min(tb + kTile, P.total_end);
        const uint32_t tlen = static_cast<uint32_t>(te - tb);
        const uint64_t stage_end = min(tb + kTile + kHalo, P.avail_end);
        const uint32_t staged_len = static_cast<uint32_t>(stage_end - tb);  // valid bytes from tb
        uint8_t* bufb = S.buf[b];
        const uint8_t* tile_s = bufb + kPre;

        // ---- 1. stage bytes (prefetched by TMA, or bounded loads for edge tiles) ------------------
        const bool tma = can_tma(tile);
        if (!tma) {
            for (int v = tid; v < kStage; v += kDecodeThreads) {
                const int64_t a = static_cast<int64_t>(tb) - kPre + v;
                bufb[v] = a < 0 ? uint8_t('\n')
                                : (static_cast<uint64_t>(a) < stage_end ? P.csv[a] : uint8_t(0));
            }
        }
        if (tid < kStageAlloc - kStage) bufb[kStage + tid] = 0;
        if (tid >= 128 && tid < 132) {
            S.nl[kWords + (tid & 3)] = 0;
            S.cm[kWords + (tid & 3)] = 0;
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
        if (tid == 0) {
            c_len = 0;  // "no previous data line" for the first line of the tile
            c_ts = 0;
            c_id = 0;
            c_code = kCodeRejected;
        }
        if (tma) {
            if (b == 0) {
                mbar_wait(&bar[0], phase0);
                phase0 ^= 1;
            } else {
                mbar_wait(&bar[1], phase1);
                phase1 ^= 1;
            }
        }
        __syncthreads();

        // ---- 2. '\n' and ',' bitmaps over [tb, tb + kTile + kHalo) -----------------------------
        for (int w = tid; w < kWords; w += kDecodeThreads) {
            const uint4* p = reinterpret_cast<const uint4*>(tile_s + 32 * w);
            const uint4 a = p[0], c = p[1];
            const uint32_t x[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
            uint32_t mn = 0, mc = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                mn |= eqmask4(x[k], 0x0A0A0A0Au) << (4 * k);
                mc |= eqmask4(x[k], 0x2C2C2C2Cu) << (4 * k);
            }
            S.nl[w] = mn;
            S.cm[w] = mc;
        }
        __syncthreads();

        const bool one_shard = !sh_overflow && sh_count == 0;
        auto shard_of = [&](uint64_t p) -> uint32_t {
            if (one_shard) return sh_first;
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

        // ---- 3. data lines starting in [0, tlen) ------------------------------------------------
        // thread t owns tile words 2t, 2t+1 (kTile / 32 = 512 words)
        uint32_t smask[2];
        uint32_t my_count = 0;
        const bool tile_good = one_shard && P.shard_good[sh_first] && tb != P.shard_off[sh_first];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int w = 2 * tid + k;
            const uint32_t prev_top = (w == 0) ? (bufb[kPre - 1] == '\n' ? 1u : 0u) : (S.nl[w - 1] >> 31);
            uint32_t m = (S.nl[w] << 1) | prev_top;
            const int lo = 32 * w;
            if (lo >= static_cast<int>(tlen)) m = 0;
            else if (lo + 32 > static_cast<int>(tlen)) m &= (1u << (tlen - lo)) - 1u;
            m &= ~S.nl[w];  // a start whose first byte is '\n' is an empty line
            uint32_t keep = m;
            uint32_t cand = m;
            while (cand) {
                const int bit = __ffs(cand) - 1;
                cand &= cand - 1;
                const uint32_t pr = static_cast<uint32_t>(lo + bit);
                const uint64_t p = tb + pr;
                bool data;
                uint64_t s_end;
                if (tile_good) {
                    data = true;
                    s_end = P.shard_off[sh_first + 1];
                } else {
                    const uint32_t s = shard_of(p);
                    data = p != P.shard_off[s] && P.shard_good[s];
                    s_end = P.shard_off[s + 1];
                }
                // "\r\n" or "\r<shard end>" is empty after stripping one '\r'
                if (data && tile_s[pr] == '\r' && (p + 1 == s_end || tile_s[pr + 1] == '\n')) data = false;
                if (!data) keep &= ~(1u << bit);
            }
            smask[k] = keep;
            my_count += __popc(keep);
        }
        uint32_t n_data;
        const uint32_t my_off = block_exclusive_scan<kDecodeThreads>(my_count, scan_smem, n_data);

        // ---- publish the tile's line count now; resolve the slot base after parsing --------------
        if (tid == 0) {
            lookback1_publish(P.lb, tile, n_data);
            s_cnt[7] += n_data;
        }
        uint64_t base = 0;
        bool resolved = false;

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
                            S.starts[idx - pass_base] = static_cast<uint32_t>(32 * (2 * tid + k) + bit);
                        ++idx;
                    }
                }
            }
            __syncthreads();
            const uint32_t n_pass = min(static_cast<uint32_t>(kLineCap), n_data - pass_base);
            // ---- 4. parse: one data line per thread, results staged in shared memory -------------
            for (uint32_t li = tid; li < n_pass; li += kDecodeThreads) {
                uint8_t why;
                LineOut o;
                o.ts = 0;
                o.speed = 0.0;
                o.id_rel = 0;
                o.id_len = 0;
                uint32_t code = kCodeRejected;
                const uint32_t p_rel = S.starts[li];
                const uint64_t p = tb + p_rel;
                const uint32_t s = shard_of(p);
                const uint64_t s_end = P.shard_off[s + 1];
                // line end: next '\n' at or after p (within the staged bytes), clamped to the shard end
                uint64_t e = 0;
                bool found = false;
                {
                    uint32_t w = p_rel >> 5;
                    uint32_t m = S.nl[w] & (0xFFFFFFFFu << (p_rel & 31));
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
                        m = S.nl[w];
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
                const int kind = canonical_kind(map);
                if (in_smem && kind >= 0) why = fast_parse(tile_s, S.cm, p_rel, p_rel + len, kind, o);
                if (why == kNeedGeneral)
                    why = general_parse(in_smem ? tile_s + p_rel : gline, static_cast<int32_t>(len), map,
                                        p_rel, o);
                if (why == kAccepted) {
                    code = cell_code(o.ts, o.lat, o.lon, o.speed, o.heading, P.grid);
                    ++c_acc;
                } else {
                    atomicAdd(&s_cnt[why - 1], 1u);  // rare
                }
                S.st_ts[li] = o.ts;
                S.st_speed[li] = o.speed;
                S.st_code[li] = code;
                S.st_id[li] = o.id_rel;
                S.st_len[li] = o.id_len | (why == kAccepted ? 0x80000000u : 0u);
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
            // ---- 5. run heads + coalesced writes --------------------------------------------------
            uint32_t my_heads = 0, my_trans = 0;
            const uint32_t* ws = reinterpret_cast<const uint32_t*>(bufb);
            for (uint32_t k = tid; k < n_pass; k += kDecodeThreads) {
                const uint32_t ln = S.st_len[k];
                uint32_t code = S.st_code[k];
                if (ln >> 31) {
                    const uint32_t pl = k ? S.st_len[k - 1] : c_len;
                    const long long pts = k ? S.st_ts[k - 1] : c_ts;
                    const uint32_t idl = ln & 0x7FFFFFFFu;
                    bool head = true;
                    if ((pl >> 31) && (pl & 0x7FFFFFFFu) == idl && pts < S.st_ts[k]) {
                        const uint32_t pid = k ? S.st_id[k - 1] : c_id;
                        const uint32_t mid = S.st_id[k];
                        bool same = true;
                        if (pid + idl <= staged_len && mid + idl <= staged_len) {
                            for (uint32_t i = 0; i < idl; i += 4) {
                                uint32_t x = word_at(ws, kPre + pid + i) ^ word_at(ws, kPre + mid + i);
                                if (idl - i < 4) x &= (1u << (8 * (idl - i))) - 1u;
                                if (x) {
                                    same = false;
                                    break;
                                }
                            }
                        } else {
                            const uint8_t* pa = (pid + idl <= staged_len) ? tile_s + pid : P.csv + tb + pid;
                            const uint8_t* pb = (mid + idl <= staged_len) ? tile_s + mid : P.csv + tb + mid;
                            for (uint32_t i = 0; i < idl; ++i)
                                if (pa[i] != pb[i]) {
                                    same = false;
                                    break;
                                }
                        }
                        head = !same;
                    }
                    if (head) {
                        ++my_heads;
                        code |= kHeadBit;
                    } else if ((k ? S.st_code[k - 1] : c_code) != code) {
                        ++my_trans;
                    }
                }
                if (fits) {
                    const uint64_t slot = base + pass_base + k;
                    P.out.ts[slot] = S.st_ts[k];
                    P.out.speed[slot] = S.st_speed[k];
                    P.out.code[slot] = code;
                    P.out.loff[slot] = tb + S.starts[k];
                }
            }
            if (my_heads) atomicAdd(&s_cnt[4], my_heads);
            if (my_trans) atomicAdd(&s_cnt[5], my_trans);
            __syncthreads();
            if (tid == 0) {  // carry the pass's last line
                c_ts = S.st_ts[n_pass - 1];
                c_id = S.st_id[n_pass - 1];
                c_len = S.st_len[n_pass - 1];
                c_code = S.st_code[n_pass - 1];
            }
            __syncthreads();
        }
        if (!resolved) lookback1_resolve<kDecodeThreads>(P.lb, tile, n_data, s_lb);
        __syncthreads();  // buffers and per-tile shared state are reused by the next tile
    }

    // ---- stats (once per CTA) ---------------------------------------------------------------------
    const uint32_t acc = warp_sum(c_acc);
    if ((tid & 31) == 0 && acc) atomicAdd(&s_cnt[6], acc);
    __syncthreads();
    if (tid == 0) {
        unsigned long long* st = reinterpret_cast<unsigned long long*>(P.stats);
        if (s_cnt[7]) atomicAdd(&st[kStRowsRead], static_cast<unsigned long long>(s_cnt[7]));
        for (int i = 0; i < 4; ++i)
            if (s_cnt[i]) atomicAdd(&st[kStRejBase + i], static_cast<unsigned long long>(s_cnt[i]));
        if (s_cnt[4]) atomicAdd(&st[kStHeads], static_cast<unsigned long long>(s_cnt[4]));
        if (s_cnt[5]) atomicAdd(&st[kStGTransitions], static_cast<unsigned long long>(s_cnt[5]));
        if (s_cnt[6]) atomicAdd(&st[kStParsed], static_cast<unsigned long long>(s_cnt[6]));
    }
}

void launch_decode(const DecodeParams& p, uint32_t tile_begin, uint32_t n_tiles, cudaStream_t s) {
    if (n_tiles == 0) return;
    static int max_ctas = 0;
    if (!max_ctas) {
        cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(DecodeSmem)));
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel, kDecodeThreads,
                                                      sizeof(DecodeSmem));
        max_ctas = std::max(1, sms * std::max(per_sm, 1));
    }
    const uint32_t ctas = std::min<uint32_t>(n_tiles, static_cast<uint32_t>(max_ctas));
    decode_kernel<<<ctas, kDecodeThreads, sizeof(DecodeSmem), s>>>(p, tile_begin);
}

}  // namespace cvlg
