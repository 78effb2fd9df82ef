// K0 (shard header map) and K1 (tile decode) for sm_100a.
//
// K1 makes a single pass over the concatenated CSV shards in HBM with persistent CTAs (static
// round-robin tiles: CTA c takes tiles c, c + G, ...). Per 16 KB tile a CTA:
//   1. consumes the tile that one TMA bulk copy (cp.async.bulk + mbarrier) prefetched into one
//      of two stage buffers while the previous tile was decoded, and issues the next one;
//   2. builds '\n' and ',' bitmaps cooperatively (SIMD-within-a-register byte compares; thread t
//      owns tile bytes [64t, 64t + 64));
//   3. finds the DATA lines that start in each thread's 64 bytes (non-empty, not a header, good
//      shard) and numbers them with one block-wide scan;
//   4. each thread parses the lines that start in its own bytes (fast path: field ends from the
//      comma bitmap, fastparse.cuh's SWAR timestamp and cached-shape numbers, all checks combined
//      without branches; anything unusual goes to the general restatement of parse_record_impl,
//      parse.cuh), then filter + binning (grid.cuh);
//   5. marks run heads (journey id changes, or the timestamp stops increasing, vs. the previous
//      data line of the tile) and writes the tile's head list from warp ballots, with each
//      head's inline dictionary key.
// Slot space is sparse per tile (tile t owns slots [t * kLineCap, t * kLineCap + lines)), so no
// tile ever waits for another: no cross-tile scan or look-back. Outputs, in provenance order
// (slot = data line; shards are concatenated in lexicographic path order, so slot order equals
// the reference's (shard_rank, line) order, aggregate.cpp:287-289): ts / speed / cell code
// (| head bit) / line offset per slot, the per-tile run-head lists and tiles[t]. Tiles with more
// than kLineCap data lines (pathological short lines) take slots from an overflow region and a
// multi-pass path over a start list.
#include <algorithm>

#include "fastparse.cuh"
#include "kernels.cuh"

namespace cvlg {

namespace {

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

struct LineOut {
    int64_t ts;
    double lat, lon, speed, heading;
    uint32_t id_rel, id_len;  // tile-relative id span
    uint32_t minute;          // minute of day (fast path), kNoMinute when unknown
};

constexpr uint32_t kNoMinute = 0xFFFFFFFFu;
constexpr uint8_t kNeedGeneral = 255;

// Per-thread fast-path state carried across lines: the last validated date and, per numeric
// column, the decimal point position of the previous line.
struct FastState {
    DateCache dc;
    int q[4] = {-1, -1, -1, -1};
};
static_assert(sizeof(FastState) % 8 == 4, "odd word stride: conflict-free per-thread state");

// First ',' at or after tile-relative byte x within the next 32 bytes (comma bitmap `cm`, bit i =
// tile byte i): its position, or x - 1 when there is none (every caller then fails a length test).
__device__ __forceinline__ uint32_t next_comma(const uint32_t* __restrict__ cm, uint32_t x) {
    const uint32_t m = __funnelshift_r(cm[x >> 5], cm[(x >> 5) + 1], x & 31);
    return x + __ffs(m) - 1;
}

// Fast path of parse_record_impl for a line [p, e) (tile-relative) entirely staged in shared
// memory whose header is canonical: journey, timestamp, latitude, longitude as fields 0..3, then
// speed, heading as 5, 6 (`postal` = 1: any column at 4) or 4, 5. True iff every field has the
// canonical shape and the record is in range (then `o` holds the accepted record); false ->
// the general restatement decides (including every rejection). Field ends come from the comma
// bitmap one field at a time (the timestamp is exactly 19 bytes, its separator checked in
// registers); the checks of all fields are combined without branches.
__device__ __forceinline__ bool fast_parse(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ cm,
                                           uint32_t p, uint32_t e, int postal, FastState& fs, LineOut& o) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(buf);
    const uint32_t c0 = next_comma(cm, p);  // journey id [p, c0)
    const uint32_t c1 = c0 + 20;            // timestamp [c0 + 1, c1)
    const uint32_t c2 = next_comma(cm, c1 + 1);
    const uint32_t c3 = next_comma(cm, c2 + 1);
    const uint32_t c4 = next_comma(cm, c3 + 1);
    uint32_t sp_b = c3 + 1, sp_e = c4;
    if (postal) {
        sp_b = c4 + 1;
        sp_e = next_comma(cm, sp_b);
    }
    const uint32_t hd_b = sp_e + 1;
    uint32_t hd_e;
    {
        const uint32_t m = __funnelshift_r(cm[hd_b >> 5], cm[(hd_b >> 5) + 1], hd_b & 31);
        hd_e = m ? min(hd_b + __ffs(m) - 1, e) : e;
    }
    uint32_t sep;
    bool ok = fast_timestamp(w, kPre + c0 + 1, fs.dc, o.ts, o.minute, sep);
    const uint32_t idl = c0 - p;
    ok &= (idl - 1u < 31u) & (sep == 0x2Cu) & (sp_e < e) & (c4 > c3) &
          !trim_byte(buf[kPre + p]) & !trim_byte(buf[kPre + c0 - 1]);
    bool num = fast_number_hit(w, buf, kPre + c1 + 1, kPre + c2, fs.q[0], o.lat);
    num &= fast_number_hit(w, buf, kPre + c2 + 1, kPre + c3, fs.q[1], o.lon);
    num &= fast_number_hit(w, buf, kPre + sp_b, kPre + sp_e, fs.q[2], o.speed);
    num &= fast_number_hit(w, buf, kPre + hd_b, kPre + hd_e, fs.q[3], o.heading);
    if (!num && ok) {  // a column changed shape: fast_number re-learns the point positions
        num = fast_number(w, buf, kPre + c1 + 1, kPre + c2, fs.q[0], o.lat) &&
              fast_number(w, buf, kPre + c2 + 1, kPre + c3, fs.q[1], o.lon) &&
              fast_number(w, buf, kPre + sp_b, kPre + sp_e, fs.q[2], o.speed) &&
              fast_number(w, buf, kPre + hd_b, kPre + hd_e, fs.q[3], o.heading);
    }
    if (o.heading == 360.0) o.heading = 0.0;
    o.id_rel = p;
    o.id_len = idl;
    return ok & num & (o.lat >= -90.0) & (o.lat <= 90.0) & (o.lon >= -180.0) & (o.lon <= 180.0) &
           (o.speed >= 0.0) & (o.heading >= 0.0) & (o.heading < 360.0);
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
        o.minute = kNoMinute;
    }
    return why;
}

// The dictionary key of a run head's journey id (dict_insert's format: bytes 0..7 big-endian,
// then bytes 8..14 big-endian << 8 | length) from the staged tile, for ids of <= 15 bytes whose
// bytes are staged; otherwise .y = kNoKey and dict_insert reads the id from the CSV itself.
__device__ __forceinline__ ulonglong2 head_key(const uint32_t* ws, uint32_t rel, uint32_t len,
                                               uint32_t staged_len) {
    ulonglong2 k;
    k.x = 0;
    k.y = kNoKey;
    if (len <= 15 && rel + len <= staged_len) {
        uint32_t b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            b[q] = word_at(ws, kPre + rel + 4 * q) & ~bytes_from_rt(static_cast<int>(len) - 4 * q);
        auto bs = [](uint32_t x) { return __byte_perm(x, 0u, 0x0123u); };
        k.x = (static_cast<uint64_t>(bs(b[0])) << 32) | bs(b[1]);
        const uint64_t k1 = ((static_cast<uint64_t>(bs(b[2])) << 32) | bs(b[3])) >> 8;
        k.y = (k1 << 8) | len;
    }
    return k;
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
// K1
constexpr int kStage = kPre + kTile + kHalo;
constexpr int kStageAlloc = kStage + 32;  // word over-read padding, keeps 16 B alignment
constexpr int kWords = (kTile + kHalo) / 32;
constexpr int kMaxShardsInTile = 32;
#ifndef CVLG_DECODE_MINB
#define CVLG_DECODE_MINB (4 * 16384 / kTile)
#endif
constexpr int kDecodeCtasPerSm = CVLG_DECODE_MINB;  // 1024 threads per SM at 64 registers
constexpr int kNW = kDecodeThreads / 32;
constexpr int kRounds = (kLineCap + kDecodeThreads - 1) / kDecodeThreads;
constexpr int kHeadWords = kRounds * kNW;  // one ballot word per (round, warp)
static_assert(kHeadWords <= 32, "head ballot words");
static_assert(kTile / 64 == kDecodeThreads, "thread t owns tile words 2t, 2t+1");

struct DecodeSmem {
    uint8_t buf[2][kStageAlloc];
    uint32_t nl[kWords + 4];
    uint32_t cm[kWords + 4];
    uint32_t starts[kLineCap];
    uint32_t id_rel[kLineCap];  // tile-relative id start
    uint32_t id_len[kLineCap];  // id length | accepted << 31
    uint32_t l_code[kLineCap];  // cell code (no head bit)
    uint32_t hbits[kHeadWords];
    alignas(8) long long l_ts[kLineCap];
    alignas(8) uint8_t fs_raw[sizeof(FastState) * kDecodeThreads];  // per-thread fast-path state
};

__global__ void __launch_bounds__(kDecodeThreads, kDecodeCtasPerSm) decode_kernel(DecodeParams P,
                                                                                  uint32_t tile_begin) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    DecodeSmem& S = *reinterpret_cast<DecodeSmem*>(smem_raw);
    __shared__ uint32_t scan_smem[kNW];
    __shared__ uint64_t sh_off[kMaxShardsInTile + 2];
    __shared__ uint32_t sh_first, sh_count, sh_overflow, sh_good;
    __shared__ int sh_kind;
    __shared__ uint32_t sh_send_rel;
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t s_cnt[8];  // rejects[4], heads, transitions, accepted, rows
    __shared__ uint32_t s_inert;
    __shared__ unsigned long long s_ovf[2];
    __shared__ long long c_ts;
    __shared__ uint32_t c_id, c_len, c_code;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    if (tid < 8) s_cnt[tid] = 0;
    if (tid == 8) s_inert = 0;
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

    // the per-thread fast-path state lives in shared memory (frees registers for occupancy)
    FastState& fs = reinterpret_cast<FastState*>(S.fs_raw)[tid];
    fs = FastState();
    uint32_t phases = 0;  // mbarrier phase of buffer b in bit b
    uint32_t c_acc = 0;
    uint32_t tile = tile_begin + blockIdx.x;
    if (tid == 0 && tile < P.tile_end && can_tma(tile)) issue(tile, 0);

    for (uint32_t it = 0; tile < P.tile_end; ++it, tile += gridDim.x) {
        const int b = it & 1;
        const uint32_t nxt = tile + gridDim.x;
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
        if (tid == 32) {  // shards overlapping the tile (overlaps the copy)
            uint32_t lo = 0, hi = P.n_shards;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) / 2;
                if (P.shard_off[mid] <= tb) lo = mid;
                else hi = mid;
            }
            sh_first = lo;
            uint32_t c = 0, s = lo + 1;
            while (s <= P.n_shards && P.shard_off[s] < te && c < kMaxShardsInTile) sh_off[c++] = P.shard_off[s++];
            const uint32_t over = (s <= P.n_shards && P.shard_off[s] < te) ? 1u : 0u;
            sh_overflow = over;
            sh_count = c;
            const bool one = c == 0 && !over;
            sh_kind = one ? canonical_kind(P.cmap[lo]) : -1;
            sh_good = (one && P.shard_good[lo] && tb != P.shard_off[lo]) ? 1u : 0u;
            {
                const uint64_t se = P.shard_off[lo + 1] - tb;
                sh_send_rel = se > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(se);
            }
        }
        if (tma) {
            mbar_wait(&bar[b], (phases >> b) & 1u);
            phases ^= 1u << b;
        }
        __syncthreads();

        // ---- 2. '\n' / ',' bitmaps of this thread's 64 bytes (+ the halo) and its line starts -----
        auto bitmap_word = [&](int w) -> uint32_t {
            const uint4* p = reinterpret_cast<const uint4*>(tile_s + 32 * w);
            const uint4 a = p[0], c = p[1];
            const uint32_t x[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
            uint32_t mn, mc;
            class_masks32(x, mn, mc);
            S.nl[w] = mn;
            S.cm[w] = mc;
            return mn;
        };
        const uint32_t nlw0 = bitmap_word(2 * tid), nlw1 = bitmap_word(2 * tid + 1);
        if (tid < kWords - 2 * kDecodeThreads) bitmap_word(2 * kDecodeThreads + tid);

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

        // data lines starting in [0, tlen): a start follows a '\n' (or the byte before the tile)
        uint32_t smask[2];
        uint32_t my_count = 0;
        const bool tile_good = sh_good != 0;
        {
            const uint8_t before = (tid == 0) ? bufb[kPre - 1] : tile_s[64 * tid - 1];
            uint32_t prev_top = before == '\n' ? 1u : 0u;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int w = 2 * tid + k;
                const uint32_t nlw = k ? nlw1 : nlw0;
                uint32_t m = (nlw << 1) | prev_top;
                prev_top = nlw >> 31;
                const int lo = 32 * w;
                if (lo >= static_cast<int>(tlen)) m = 0;
                else if (lo + 32 > static_cast<int>(tlen)) m &= (1u << (tlen - lo)) - 1u;
                m &= ~nlw;  // a start whose first byte is '\n' is an empty line
                // ("\r\n" lines are empty too: they keep a slot but are made inert in parse_lines)
                uint32_t keep = m;
                if (!tile_good) {
                    uint32_t cand = m;
                    while (cand) {
                        const int bit = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const uint64_t p = tb + static_cast<uint32_t>(lo + bit);
                        const uint32_t s = shard_of(p);
                        if (p == P.shard_off[s] || !P.shard_good[s]) keep &= ~(1u << bit);
                    }
                }
                smask[k] = keep;
                my_count += __popc(keep);
            }
        }
        // block exclusive scan of my_count, one barrier (also publishes the bitmaps)
        const uint32_t inc = warp_inclusive_sum(my_count);
        if (lane == 31) scan_smem[warp] = inc;
        __syncthreads();
        uint32_t n_data, my_off;
        {
            const uint32_t wv = lane < kNW ? scan_smem[lane] : 0u;
            uint32_t wi = wv;
#pragma unroll
            for (int o = 1; o < kNW; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
                if (lane >= o) wi += t;
            }
            n_data = __shfl_sync(0xFFFFFFFFu, wi, kNW - 1);
            my_off = inc - my_count + __shfl_sync(0xFFFFFFFFu, wi - wv, warp);
        }
        if (tid == 0) s_cnt[7] += n_data;

        // ---- line starts of lines [pass_base, pass_base + kLineCap) ------------------------------
        auto write_starts = [&](uint32_t pass_base) {
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
        };
        // ---- 4. parse: one data line per thread, results staged in shared memory -----------------
        // one data line starting at tile byte p_rel: staged results at index li, outputs at slot
        auto parse_one = [&](uint32_t li, uint32_t p_rel, uint64_t slot) {
            {
                LineOut o;
                o.ts = 0;
                o.speed = 0.0;
                o.id_rel = 0;
                o.id_len = 0;
                uint32_t s;
                uint32_t se_rel;  // shard end relative to the tile start (clamped to 32 bits)
                int kind;
                if (one_shard) {
                    s = sh_first;
                    se_rel = sh_send_rel;
                    kind = sh_kind;
                } else {
                    s = shard_of(tb + p_rel);
                    const uint64_t se = P.shard_off[s + 1] - tb;
                    se_rel = se > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(se);
                    kind = canonical_kind(P.cmap[s]);
                }
                // line end (tile-relative): next '\n' at or after p within the staged bytes,
                // clamped to the shard end; a 96-bit window of the newline bitmap covers every line
                // of <= 95 bytes
                uint32_t e_rel = 0;
                bool found = false;
                {
                    const uint32_t w = p_rel >> 5, sh = p_rel & 31;
                    const uint32_t n0 = S.nl[w], n1 = S.nl[w + 1], n2 = S.nl[w + 2], n3 = S.nl[w + 3];
                    const uint32_t m0 = __funnelshift_r(n0, n1, sh), m1 = __funnelshift_r(n1, n2, sh),
                                   m2 = __funnelshift_r(n2, n3, sh);
                    uint32_t x = 0xFFFFFFFFu;
                    if (m0) x = p_rel + __ffs(m0) - 1;
                    else if (m1) x = p_rel + 31 + __ffs(m1);
                    else if (m2) x = p_rel + 63 + __ffs(m2);
                    if (x != 0xFFFFFFFFu) {
                        if (x < staged_len) {
                            e_rel = x;
                            found = true;
                        }
                    } else {
                        for (uint32_t v = w + 3; v < static_cast<uint32_t>(kWords) && 32 * v < staged_len; ++v) {
                            const uint32_t mm = S.nl[v];
                            if (mm) {
                                const uint32_t y = 32 * v + (__ffs(mm) - 1);
                                if (y < staged_len) {
                                    e_rel = y;
                                    found = true;
                                }
                                break;
                            }
                        }
                    }
                }
                if (!found) {  // the line runs past the staged bytes: scan global memory
                    const uint64_t s_end = tb + se_rel;
                    uint64_t x = tb + staged_len;
                    while (x < P.avail_end && x < s_end && P.csv[x] != '\n') ++x;
                    const uint64_t xr = x - tb;
                    e_rel = xr > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(xr);
                }
                if (e_rel > se_rel) e_rel = se_rel;
                const bool in_smem = e_rel <= staged_len;
                const uint8_t* gline = P.csv + tb + p_rel;
                uint32_t len = e_rel - p_rel;
                const uint8_t last = in_smem ? tile_s[p_rel + len - 1] : gline[len - 1];
                if (last == '\r') --len;
                if (len == 0) {  // "\r\n" / "\r<shard end>": empty, not a data line (inert slot)
                    atomicAdd(&s_inert, 1u);  // rare: a shared counter, not a register
                    P.out.ts[slot] = 0;
                    P.out.speed[slot] = 0.0;
                    P.out.loff[slot] = tb + p_rel;
                    S.l_ts[li] = 0;
                    S.l_code[li] = kCodeRejected;
                    S.id_rel[li] = 0;
                    S.id_len[li] = 0;
                    return;
                }
                uint8_t why = kNeedGeneral;
                if (in_smem && kind >= 0 && fast_parse(bufb, S.cm, p_rel, p_rel + len, kind, fs, o)) why = kAccepted;
                if (why == kNeedGeneral) {  // (a separate out-struct: `o` itself never escapes to
                    LineOut og;              //  the out-of-line call, so it stays in registers)
                    og.ts = 0;
                    og.speed = 0.0;
                    og.id_rel = 0;
                    og.id_len = 0;
                    og.minute = kNoMinute;
                    why = general_parse(in_smem ? tile_s + p_rel : gline, static_cast<int32_t>(len), P.cmap[s],
                                        p_rel, og);
                    o = og;
                }
                uint32_t code = kCodeRejected;
                if (why == kAccepted) {
                    const uint32_t t = o.minute != kNoMinute ? time_bin_mod(o.minute, P.grid)
                                                             : time_bin(o.ts, P.grid.min_step);
                    code = cell_code_t(t, o.lat, o.lon, o.speed, o.heading, P.grid);
                    ++c_acc;
                } else {
                    atomicAdd(&s_cnt[why - 1], 1u);  // rare
                }
                P.out.ts[slot] = o.ts;
                P.out.speed[slot] = o.speed;
                P.out.loff[slot] = tb + p_rel;
                if (P.out.lat) {
                    P.out.lat[slot] = why == kAccepted ? o.lat : 0.0;
                    P.out.lon[slot] = why == kAccepted ? o.lon : 0.0;
                }
                S.l_ts[li] = o.ts;
                S.l_code[li] = code;
                S.id_rel[li] = o.id_rel;
                S.id_len[li] = o.id_len | (why == kAccepted ? 0x80000000u : 0u);
            }
        };
        // overflow tiles: lines [pass_base, pass_base + n_pass) from the start list
        auto parse_lines = [&](uint32_t n_pass, uint64_t slot0) {
            for (uint32_t li = tid; li < n_pass; li += kDecodeThreads) parse_one(li, S.starts[li], slot0 + li);
        };

        // ---- 5. run heads: the journey id changes or the timestamp stops increasing --------------
        // Line 0 compares against the carry (c_*; c_len = 0: no previous line -> head). Writes the
        // slot words (cell code | head bit), counts cell transitions inside runs, and calls
        // emit(index, line) for every head, index = rank among this pass's heads. Returns the
        // pass's head count.
        auto mark_heads = [&](uint32_t n_pass, uint64_t slot0, auto&& emit) -> uint32_t {
            const uint32_t* ws = reinterpret_cast<const uint32_t*>(bufb);
            uint32_t my_trans = 0;
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                if (r > 0 && r * kDecodeThreads >= n_pass) {  // (uniform: no line in this round)
                    if (lane == 0) S.hbits[r * kNW + warp] = 0u;
                    continue;
                }
                const uint32_t k = r * kDecodeThreads + tid;
                bool head = false;
                if (k < n_pass) {
                    const uint32_t ln = S.id_len[k];
                    const uint32_t code = S.l_code[k];
                    const uint32_t pl = k ? S.id_len[k - 1] : c_len;
                    const long long pts = k ? S.l_ts[k - 1] : c_ts;
                    const uint32_t idl = ln & 0x7FFFFFFFu;
                    // a continuation needs: both accepted, equal id lengths, rising timestamps and
                    // equal id bytes (compared straight from the staged tile for ids <= 8 bytes)
                    bool cont = (ln >> 31) && pl == ln && pts < S.l_ts[k];
                    if (cont) {
                        const uint32_t pid = k ? S.id_rel[k - 1] : c_id;
                        const uint32_t mid = S.id_rel[k];
                        if (idl <= 8 && pid + 8 <= staged_len && mid + 8 <= staged_len) {
                            const uint32_t m0 = ~bytes_from_rt(static_cast<int>(idl));
                            const uint32_t m1 = ~bytes_from_rt(static_cast<int>(idl) - 4);
                            const uint32_t x0 = word_at(ws, kPre + pid) ^ word_at(ws, kPre + mid);
                            const uint32_t x1 = word_at(ws, kPre + pid + 4) ^ word_at(ws, kPre + mid + 4);
                            cont = ((x0 & m0) | (x1 & m1)) == 0;
                        } else {
                            const uint8_t* pa = (pid + idl <= staged_len) ? tile_s + pid : P.csv + tb + pid;
                            const uint8_t* pb = (mid + idl <= staged_len) ? tile_s + mid : P.csv + tb + mid;
                            for (uint32_t i = 0; i < idl; ++i)
                                if (pa[i] != pb[i]) {
                                    cont = false;
                                    break;
                                }
                        }
                    }
                    head = (ln >> 31) && !cont;  // rejected lines are never heads
                    if (cont && (k ? S.l_code[k - 1] : c_code) != code) ++my_trans;
                    P.out.code[slot0 + k] = head ? (code | kHeadBit) : code;
                }
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, head);
                if (lane == 0) S.hbits[r * kNW + warp] = bal;
            }
            if (my_trans) atomicAdd(&s_cnt[5], my_trans);
            __syncthreads();
            // exclusive prefix of the head words (every warp computes it redundantly)
            const uint32_t cntw = lane < kHeadWords ? __popc(S.hbits[lane]) : 0u;
            const uint32_t incw = warp_inclusive_sum(cntw);
            const uint32_t nh = __shfl_sync(0xFFFFFFFFu, incw, kHeadWords - 1);
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                if (r > 0 && r * kDecodeThreads >= n_pass) break;
                const uint32_t k = r * kDecodeThreads + tid;
                const int wd = r * kNW + warp;
                const uint32_t bits = S.hbits[wd];
                const uint32_t pre = __shfl_sync(0xFFFFFFFFu, incw - cntw, wd);
                if (k < n_pass && ((bits >> lane) & 1u)) emit(pre + __popc(bits & ((1u << lane) - 1u)), k);
            }
            if (tid == 0) s_cnt[4] += nh;
            return nh;
        };

        uint64_t slot0, head0;
        uint32_t heads = 0;
        if (n_data <= static_cast<uint32_t>(kLineCap)) {
            // ---- common case: the tile's own slot range [tile * kLineCap, + n_data) ----------------
            slot0 = static_cast<uint64_t>(tile) * kLineCap;
            head0 = slot0;
            if (tid == 0) c_len = 0;
            // every thread parses the data lines that start in its own 64 bytes (no start list)
            {
                uint64_t m = (static_cast<uint64_t>(smask[1]) << 32) | smask[0];
                uint32_t li = my_off;
                while (m) {
                    const uint32_t bit = static_cast<uint32_t>(__ffsll(static_cast<long long>(m))) - 1u;
                    m &= m - 1;
                    parse_one(li, 64u * tid + bit, slot0 + li);
                    ++li;
                }
            }
            __syncthreads();
            heads = mark_heads(n_data, slot0, [&](uint32_t idx, uint32_t k) {
                P.out.hslot[head0 + idx] = static_cast<uint32_t>(slot0 + k);
                const uint32_t rel = S.id_rel[k], len = S.id_len[k] & 0x7FFFFFFFu;
                P.out.hid[head0 + idx] = (tb + rel) | (static_cast<uint64_t>(len) << 40);
                P.out.hkey[head0 + idx] = head_key(reinterpret_cast<const uint32_t*>(bufb), rel, len, staged_len);
            });
        } else {
            // ---- more than kLineCap lines: slots and heads from the overflow regions --------------
            if (tid == 0) {
                s_ovf[0] = atomicAdd(P.out.ovf_slots, static_cast<unsigned long long>(n_data));
                s_ovf[1] = atomicAdd(P.out.ovf_heads, static_cast<unsigned long long>(n_data));
                c_len = 0;
            }
            __syncthreads();
            const bool fits = s_ovf[0] + n_data <= P.out.ovf_slot_cap && s_ovf[1] + n_data <= P.out.ovf_head_cap;
            slot0 = P.out.reg_slots + s_ovf[0];
            head0 = P.out.reg_slots + s_ovf[1];
            if (!fits) {
                if (tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStOverflow]), 1ull);
            } else {
                for (uint32_t pass_base = 0; pass_base < n_data; pass_base += kLineCap) {
                    const uint32_t n_pass = min(static_cast<uint32_t>(kLineCap), n_data - pass_base);
                    __syncthreads();
                    write_starts(pass_base);
                    __syncthreads();
                    parse_lines(n_pass, slot0 + pass_base);
                    __syncthreads();
                    heads += mark_heads(n_pass, slot0 + pass_base, [&](uint32_t idx, uint32_t k) {
                        P.out.hslot[head0 + heads + idx] = static_cast<uint32_t>(slot0 + pass_base + k);
                        const uint32_t rel = S.id_rel[k], len = S.id_len[k] & 0x7FFFFFFFu;
                        P.out.hid[head0 + heads + idx] = (tb + rel) | (static_cast<uint64_t>(len) << 40);
                        P.out.hkey[head0 + heads + idx] =
                            head_key(reinterpret_cast<const uint32_t*>(bufb), rel, len, staged_len);
                    });
                    __syncthreads();
                    if (tid == 0) {  // carry the pass's last line
                        c_ts = S.l_ts[n_pass - 1];
                        c_id = S.id_rel[n_pass - 1];
                        c_len = S.id_len[n_pass - 1];
                        c_code = S.l_code[n_pass - 1];
                    }
                }
            }
        }
        if (tid == 0) {
            P.out.tiles[tile] = make_uint4(static_cast<uint32_t>(slot0), n_data, static_cast<uint32_t>(head0), heads);
        }
        __syncthreads();  // buffers and per-tile shared state are reused by the next tile
    }

    // ---- stats (once per CTA) ---------------------------------------------------------------------
    const uint32_t acc = warp_sum(c_acc);
    if (lane == 0 && acc) atomicAdd(&s_cnt[6], acc);
    __syncthreads();
    if (tid == 0 && s_inert) {
        s_cnt[7] -= s_inert;
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStInert]), static_cast<unsigned long long>(s_inert));
    }
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
    const int max_ctas = per_device(kPdDecodeCtas, [] {
        cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(DecodeSmem)));
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel, kDecodeThreads,
                                                      sizeof(DecodeSmem));
        return std::max(1, sms * std::max(per_sm, 1));
    });
    const uint32_t ctas = std::min<uint32_t>(n_tiles, static_cast<uint32_t>(max_ctas));
    decode_kernel<<<ctas, kDecodeThreads, sizeof(DecodeSmem), s>>>(p, tile_begin);
}

// ---------------------------------------------------------------------------------------------
// Records entry point: one CTA per tile of kLineCap records (provenance order). Codes come from
// filter_reason (aggregate.cpp:48-56: MissingField for an empty id when drop_missing, then the
// grid filters) and the binning of grid.cpp; run heads are decided exactly as K1 decides them
// (id change or non-increasing timestamp vs. the previous record; the tile's first record is a
// head); thread 0 writes the tile's head list in order.
constexpr int kRecThreads = 128;

__device__ __forceinline__ bool arena_equal(const uint8_t* a, uint64_t ia, uint64_t ib) {
    const uint32_t la = static_cast<uint32_t>(ia >> 40), lb = static_cast<uint32_t>(ib >> 40);
    if (la != lb) return false;
    const uint8_t* pa = a + (ia & ((1ull << 40) - 1));
    const uint8_t* pb = a + (ib & ((1ull << 40) - 1));
    for (uint32_t i = 0; i < la; ++i)
        if (pa[i] != pb[i]) return false;
    return true;
}

__global__ void __launch_bounds__(kRecThreads) records_decode_kernel(RecordsDecodeParams P) {
    __shared__ uint32_t s_code[kLineCap];
    __shared__ long long s_ts[kLineCap];
    __shared__ unsigned long long s_id[kLineCap];
    __shared__ uint8_t s_head[kLineCap];
    __shared__ uint32_t s_trans;
    const uint32_t t = blockIdx.x;
    const uint64_t base = static_cast<uint64_t>(t) * kLineCap;
    const uint32_t cnt = static_cast<uint32_t>(P.n - base < kLineCap ? P.n - base : kLineCap);
    if (threadIdx.x == 0) s_trans = 0;
    for (uint32_t k = threadIdx.x; k < cnt; k += kRecThreads) {
        const uint32_t r = P.perm[base + k];
        const int64_t ts = P.ts[r];
        const uint64_t id = P.id[r];
        uint32_t code;
        if (P.grid.drop_missing && (id >> 40) == 0) code = kCodeMissingField;
        else code = cell_code(ts, P.lat[r], P.lon[r], P.speed[r], P.heading[r], P.grid);
        P.out.ts[base + k] = ts;
        P.out.speed[base + k] = P.speed[r];
        P.out.loff[base + k] = r;
        s_code[k] = code;
        s_ts[k] = ts;
        s_id[k] = id;
    }
    __syncthreads();
    uint32_t trans = 0;
    for (uint32_t k = threadIdx.x; k < cnt; k += kRecThreads) {
        bool head = true;
        if (k > 0 && s_ts[k - 1] < s_ts[k] && arena_equal(P.arena, s_id[k - 1], s_id[k])) head = false;
        if (!head && s_code[k - 1] != s_code[k]) ++trans;
        s_head[k] = head ? 1 : 0;
        P.out.code[base + k] = head ? (s_code[k] | kHeadBit) : s_code[k];
    }
    if (trans) atomicAdd(&s_trans, trans);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t h = 0;
        for (uint32_t k = 0; k < cnt; ++k) {
            if (!s_head[k]) continue;
            const uint64_t id = s_id[k];
            const uint32_t len = static_cast<uint32_t>(id >> 40);
            P.out.hslot[base + h] = static_cast<uint32_t>(base + k);
            P.out.hid[base + h] = id;
            ulonglong2 key;
            key.x = 0;
            key.y = kNoKey;
            if (len <= 15) {  // dict_insert's inline key: bytes 0..7 BE, bytes 8..14 BE << 8 | len
                const uint8_t* q = P.arena + (id & ((1ull << 40) - 1));
                uint64_t k0 = 0, k1 = 0;
                for (uint32_t i = 0; i < 8; ++i) k0 = (k0 << 8) | (i < len ? q[i] : 0u);
                for (uint32_t i = 8; i < 15; ++i) k1 = (k1 << 8) | (i < len ? q[i] : 0u);
                key.x = k0;
                key.y = (k1 << 8) | len;
            }
            P.out.hkey[base + h] = key;
            ++h;
        }
        P.out.tiles[t] = make_uint4(static_cast<uint32_t>(base), cnt, static_cast<uint32_t>(base), h);
        unsigned long long* st = reinterpret_cast<unsigned long long*>(P.stats);
        atomicAdd(&st[kStRowsRead], static_cast<unsigned long long>(cnt));
        atomicAdd(&st[kStParsed], static_cast<unsigned long long>(cnt));
        atomicAdd(&st[kStHeads], static_cast<unsigned long long>(h));
        if (s_trans) atomicAdd(&st[kStGTransitions], static_cast<unsigned long long>(s_trans));
    }
}

void launch_records_decode(const RecordsDecodeParams& p, cudaStream_t s) {
    if (p.n_tiles == 0) return;
    records_decode_kernel<<<p.n_tiles, kRecThreads, 0, s>>>(p);
}

}  // namespace cvlg
