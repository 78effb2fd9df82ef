// K0 (shard header map) and K1 (tile decode) for sm_100a.
//
// K1 is a single pass over the concatenated CSV shards in HBM. Each CTA takes one 16 KB tile
// (dynamic tile order, so decoupled look-back always makes progress), stages tile + halo in
// shared memory with 128-bit loads, builds a '\n' bitmap cooperatively, lists the lines that
// START in the tile, parses one line per thread (ingest.cpp:119-157 semantics via parse.cuh),
// fuses filter + binning (grid.cuh), compacts accepted records in shared memory in line order,
// marks run heads (journey id changes or timestamp stops increasing), and finally publishes
// (accepted, heads) through a decoupled look-back so every record lands at its global ordinal.
// Because shards are concatenated in lexicographic path order, a record's slot order equals the
// reference's (shard_rank, line) provenance order (aggregate.cpp:287-289).
#include "kernels.cuh"

namespace cvlg {

namespace {

struct Staged {
    long long ts;
    double speed;
    uint32_t code;
    uint32_t line_rel;  // line start relative to tile begin
    uint32_t id_rel;    // id start relative to tile begin
    uint32_t id_len;
};

__device__ __forceinline__ uint32_t nl_mask16(uint4 v) {
    // bit i set iff byte i of the 16 bytes is '\n'
    uint32_t m = 0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t eq = __vcmpeq4(w[k], 0x0A0A0A0Au) & 0x08040201u;
        const uint32_t nib = (eq * 0x01010101u) >> 24;  // sum of the 4 selected bits
        m |= nib << (4 * k);
    }
    return m;
}

__device__ __forceinline__ uint64_t fnv1a(const uint8_t* p, uint32_t n) {
    uint64_t h = 1469598103934665603ull;
    for (uint32_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
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
constexpr int kNlWords = (kTile + kHalo) / 32;
constexpr int kMaxShardsInTile = 32;

__global__ void __launch_bounds__(kDecodeThreads) decode_kernel(DecodeParams P) {
    __shared__ __align__(16) uint8_t buf[kStage];
    __shared__ uint32_t nl[kNlWords];
    __shared__ uint16_t starts[kLineCap];
    __shared__ Staged stage[kMaxAccPerTile];
    __shared__ uint32_t scan_smem[kDecodeThreads / 32 + 1];
    __shared__ uint64_t sh_off[kMaxShardsInTile + 2];  // shard starts (sh_first .. ) in tile
    __shared__ uint32_t sh_first, sh_count, sh_overflow;
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_base_acc, s_base_head;
    __shared__ uint8_t head_flag[kMaxAccPerTile];

    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(P.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= P.tile_end) return;

    const uint64_t tb = static_cast<uint64_t>(tile) * kTile;
    const uint64_t te = min(tb + kTile, P.total_end);
    const uint32_t tlen = static_cast<uint32_t>(te - tb);
    // staged bytes: [tb - kPre, tb + kTile + kHalo) clipped to [0, avail_end)
    const uint64_t stage_end = min(tb + kTile + kHalo, P.avail_end);
    const uint32_t staged_len = static_cast<uint32_t>(stage_end - tb);  // valid bytes from tb

    // ---- stage bytes -------------------------------------------------------------------------
    if (P.aligned16) {
        const uint4* src = reinterpret_cast<const uint4*>(P.csv);
        uint4* dst = reinterpret_cast<uint4*>(buf);
        const int64_t base_vec = static_cast<int64_t>(tb / 16) - 1;  // kPre == 16
        for (int v = tid; v < kStage / 16; v += kDecodeThreads) {
            const int64_t gv = base_vec + v;
            const int64_t gb = gv * 16;
            uint4 val;
            if (gb >= 0 && static_cast<uint64_t>(gb + 16) <= stage_end) {
                val = __ldg(src + gv);
            } else {
                union {
                    uint4 v;
                    uint8_t b[16];
                } tmp;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int64_t a = gb + k;
                    tmp.b[k] = a < 0 ? uint8_t('\n')
                                     : (static_cast<uint64_t>(a) < stage_end ? P.csv[a] : uint8_t(0));
                }
                val = tmp.v;
            }
            dst[v] = val;
        }
    } else {
        for (int v = tid; v < kStage; v += kDecodeThreads) {
            const int64_t a = static_cast<int64_t>(tb) - kPre + v;
            buf[v] = a < 0 ? uint8_t('\n')
                           : (static_cast<uint64_t>(a) < stage_end ? P.csv[a] : uint8_t(0));
        }
    }
    if (tid == 0) {
        // shard containing tb: last s with shard_off[s] <= tb
        uint32_t lo = 0, hi = P.n_shards;  // answer in [0, n_shards-1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (P.shard_off[mid] <= tb) lo = mid;
            else hi = mid;
        }
        sh_first = lo;
        uint32_t c = 0;
        uint32_t s = lo + 1;
        while (s <= P.n_shards && P.shard_off[s] < te && c < kMaxShardsInTile) {
            sh_off[c++] = P.shard_off[s];
            ++s;
        }
        sh_overflow = (s <= P.n_shards && P.shard_off[s] < te) ? 1u : 0u;
        sh_count = c;
    }
    __syncthreads();

    // ---- newline bitmap over [tb, tb + kTile + kHalo) ------------------------------------------
    for (int w = tid; w < kNlWords; w += kDecodeThreads) {
        const uint4* p = reinterpret_cast<const uint4*>(buf + kPre + 32 * w);
        nl[w] = nl_mask16(p[0]) | (nl_mask16(p[1]) << 16);
    }
    __syncthreads();

    // ---- line starts in [0, tlen): positions after a '\n' --------------------------------------
    // each thread owns words 2*tid, 2*tid+1 of the tile (kTile/32 = 512 words, 256 threads)
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
        smask[k] = m;
        my_count += __popc(m);
    }
    uint32_t total_starts;
    const uint32_t my_off = block_exclusive_scan<kDecodeThreads>(my_count, scan_smem, total_starts);

    // per-thread stats
    uint32_t c_rows = 0, c_rej[4] = {0, 0, 0, 0}, c_trans = 0;
    long long ts_min = LLONG_MAX, ts_max = LLONG_MIN;
    uint32_t n_acc = 0;  // uniform across the block

    for (uint32_t pass_base = 0; pass_base < total_starts; pass_base += kLineCap) {
        // scatter this pass's starts
        {
            uint32_t idx = my_off;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                uint32_t m = smask[k];
                while (m) {
                    const int bit = __ffs(m) - 1;
                    m &= m - 1;
                    if (idx >= pass_base && idx < pass_base + kLineCap)
                        starts[idx - pass_base] = static_cast<uint16_t>(32 * (2 * tid + k) + bit);
                    ++idx;
                }
            }
        }
        __syncthreads();
        const uint32_t n_pass = min(static_cast<uint32_t>(kLineCap), total_starts - pass_base);
        for (uint32_t r0 = 0; r0 < n_pass; r0 += kDecodeThreads) {
            const uint32_t li = r0 + tid;
            uint32_t accepted = 0;
            Staged rec;
            if (li < n_pass) {
                const uint32_t p_rel = starts[li];
                const uint64_t p = tb + p_rel;
                // shard of p
                uint32_t s;
                if (!sh_overflow) {
                    s = sh_first;
                    for (uint32_t k = 0; k < sh_count; ++k)
                        if (sh_off[k] <= p) s = sh_first + 1 + k;
                } else {
                    uint32_t lo = 0, hi = P.n_shards;
                    while (hi - lo > 1) {
                        const uint32_t mid = (lo + hi) / 2;
                        if (P.shard_off[mid] <= p) lo = mid;
                        else hi = mid;
                    }
                    s = lo;
                }
                const uint64_t s_begin = P.shard_off[s];
                const uint64_t s_end = P.shard_off[s + 1];
                if (p != s_begin && P.shard_good[s]) {
                    // line end: next '\n' at or after p
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
                            if (++w >= static_cast<uint32_t>(kNlWords)) break;
                            if (32 * w >= staged_len) break;
                            m = nl[w];
                        }
                    }
                    if (!found) {
                        uint64_t x = tb + min(staged_len, static_cast<uint32_t>(kTile + kHalo));
                        if (x < p) x = p;
                        while (x < P.avail_end && x < s_end && P.csv[x] != '\n') ++x;
                        e = x;
                    }
                    if (e > s_end) e = s_end;
                    const bool in_smem = e <= stage_end;
                    const uint8_t* line = in_smem ? (buf + kPre + p_rel) : (P.csv + p);
                    int32_t len = static_cast<int32_t>(e - p);
                    if (len > 0 && line[len - 1] == '\r') --len;
                    if (len > 0) {
                        ++c_rows;
                        Parsed pr;
                        const uint8_t why = parse_line(line, len, P.cmap[s], pr);
                        if (why == kAccepted) {
                            accepted = 1;
                            rec.ts = pr.epoch;
                            rec.speed = pr.speed;
                            rec.code = cell_code(pr.epoch, pr.lat, pr.lon, pr.speed, pr.heading,
                                                 P.grid);
                            rec.line_rel = p_rel;
                            rec.id_rel = p_rel + static_cast<uint32_t>(pr.id_begin);
                            rec.id_len = static_cast<uint32_t>(pr.id_len);
                            ts_min = min(ts_min, static_cast<long long>(pr.epoch));
                            ts_max = max(ts_max, static_cast<long long>(pr.epoch));
                        } else {
                            ++c_rej[why - 1];
                        }
                    }
                }
            }
            uint32_t n_round;
            const uint32_t pos = block_exclusive_scan<kDecodeThreads>(accepted, scan_smem, n_round);
            if (accepted && n_acc + pos < static_cast<uint32_t>(kMaxAccPerTile))
                stage[n_acc + pos] = rec;
            n_acc += n_round;
        }
        __syncthreads();
    }
    if (n_acc > static_cast<uint32_t>(kMaxAccPerTile)) {
        // impossible by the 30-byte bound; keep the invariant loud rather than corrupt memory
        if (tid == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStOverflow]), 1ull);
        n_acc = kMaxAccPerTile;
    }
    __syncthreads();

    // ---- run heads --------------------------------------------------------------------------
    uint32_t my_heads = 0;
    for (uint32_t k = tid; k < n_acc; k += kDecodeThreads) {
        uint8_t head = 1;
        if (k > 0) {
            const Staged& a = stage[k - 1];
            const Staged& b = stage[k];
            if (b.ts > a.ts && a.id_len == b.id_len) {
                const uint8_t* pa = (a.id_rel + a.id_len <= staged_len) ? buf + kPre + a.id_rel
                                                                         : P.csv + tb + a.id_rel;
                const uint8_t* pb = (b.id_rel + b.id_len <= staged_len) ? buf + kPre + b.id_rel
                                                                         : P.csv + tb + b.id_rel;
                bool same = true;
                for (uint32_t i = 0; i < a.id_len; ++i)
                    if (pa[i] != pb[i]) {
                        same = false;
                        break;
                    }
                head = same ? 0 : 1;
            }
            if (!head && a.code != b.code) ++c_trans;
        }
        head_flag[k] = head;
        my_heads += head;
    }
    uint32_t n_heads;
    block_exclusive_scan<kDecodeThreads>(my_heads, scan_smem, n_heads);

    // ---- look-back -----------------------------------------------------------------------------
    if (tid < 32) {
        uint64_t ea, eb;
        lookback_publish_and_scan(P.lb, tile, n_acc, n_heads, ea, eb);
        if (tid == 0) {
            s_base_acc = ea;
            s_base_head = eb;
        }
    }
    __syncthreads();
    const uint64_t base_acc = s_base_acc, base_head = s_base_head;
    const bool fits = base_acc + n_acc <= P.out.slot_cap && base_head + n_heads <= P.out.head_cap;
    if (!fits && tid == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStOverflow]), 1ull);

    // ---- write records + heads (line order) ----------------------------------------------------
    uint32_t head_done = 0;
    for (uint32_t r0 = 0; r0 < n_acc; r0 += kDecodeThreads) {
        const uint32_t k = r0 + tid;
        const uint32_t h = (k < n_acc) ? head_flag[k] : 0u;
        uint32_t n_round;
        const uint32_t hpos = block_exclusive_scan<kDecodeThreads>(h, scan_smem, n_round);
        if (k < n_acc && fits) {
            const Staged& s = stage[k];
            const uint64_t slot = base_acc + k;
            P.out.ts[slot] = s.ts;
            P.out.speed[slot] = s.speed;
            P.out.code[slot] = s.code;
            P.out.loff[slot] = tb + s.line_rel;
            if (h) {
                const uint64_t hi = base_head + head_done + hpos;
                const uint8_t* pid = (s.id_rel + s.id_len <= staged_len) ? buf + kPre + s.id_rel
                                                                         : P.csv + tb + s.id_rel;
                uint64_t k0 = 0, k1 = 0;
                const uint32_t n = s.id_len;
                for (uint32_t i = 0; i < 8; ++i) k0 = (k0 << 8) | (i < n ? pid[i] : 0u);
                for (uint32_t i = 8; i < 15; ++i) k1 = (k1 << 8) | (i < n ? pid[i] : 0u);
                k1 = (k1 << 8) | (n <= 15 ? n : 0xFFu);
                P.out.hslot[hi] = static_cast<uint32_t>(slot);
                P.out.hk0[hi] = k0;
                P.out.hk1[hi] = k1;
                P.out.hidref[hi] = ((tb + s.id_rel) << 24) | (n < 0xFFFFFFu ? n : 0xFFFFFFu);
                P.out.hhash[hi] = fnv1a(pid, n);
            }
        }
        head_done += n_round;
    }

    // ---- stats ---------------------------------------------------------------------------------
    unsigned long long v[6] = {c_rows, c_rej[0], c_rej[1], c_rej[2], c_rej[3], c_trans};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const unsigned long long sum = warp_sum(v[i]);
        if ((tid & 31) == 0 && sum) {
            const int idx = (i == 0) ? kStRowsRead : (i == 5 ? kStGTransitions : kStRejBase + i - 1);
            atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[idx]), sum);
        }
    }
    if (tid == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&P.stats[kStParsed]),
                  static_cast<unsigned long long>(n_acc));
    // ts min/max (warp reduce then atomics)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ts_min = min(ts_min, __shfl_xor_sync(0xFFFFFFFFu, ts_min, o));
        ts_max = max(ts_max, __shfl_xor_sync(0xFFFFFFFFu, ts_max, o));
    }
    if ((tid & 31) == 0 && ts_min <= ts_max) {
        atomicMin(&P.ts_minmax[0], ts_min);
        atomicMax(&P.ts_minmax[1], ts_max);
    }
}

void launch_decode(const DecodeParams& p, uint32_t n_ctas, cudaStream_t s) {
    if (n_ctas == 0) return;
    decode_kernel<<<n_ctas, kDecodeThreads, 0, s>>>(p);
}

}  // namespace cvlg
