// Host orchestration of the sm_100a pipeline and the C ABI (include/cvlg.h).
//
//   K0 header map  ->  K1 tile decode (+ filter + bin, look-back compaction)
//   -> journey dictionary (128-bit CAS hash table) -> lexicographic rank (LSD string sort)
//   -> canonical order: run-merge fast path (sort run heads only) or full (rank, ts) radix sort
//   -> per-journey fold into the (cell, journey) table (dedup + conflict check on the slow path)
//   -> (cell, journey) sort -> canonical per-cell fold -> dense [T][8][R][C] lattice.
// Mirrors cvl::run_pipeline (proj/src/aggregate.cpp:401-452); see DESIGN.md for the mapping.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <string_view>
#include <unordered_map>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <fstream>
#include <functional>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cvlg.h"
#include "pipeline_internal.cuh"
#include "agg_api.cuh"
#include "kernels.cuh"
#include "sort_api.cuh"

namespace cvlg {

static std::atomic<uint64_t> g_launches{0};

int per_device(int key, int (*compute)()) {
    constexpr int kMaxDev = 64;
    static std::mutex mu;
    static int cache[kMaxDev][kPdCount];
    static bool have[kMaxDev][kPdCount];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev || key < 0 || key >= kPdCount) return compute();
    std::lock_guard<std::mutex> lock(mu);
    if (!have[dev][key]) {
        cache[dev][key] = compute();
        have[dev][key] = true;
    }
    return cache[dev][key];
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

thread_local std::string t_last_error;

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(CVLG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool DevBuf::ensure(size_t bytes) {
    if (bytes <= cap && p) return false;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    CK(cudaMalloc(&p, want));
    cap = want;
    return true;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

void HostPinned::ensure(size_t bytes) {
    if (bytes <= cap && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 4096);
    CK(cudaHostAlloc(&p, want, cudaHostAllocDefault));
    cap = want;
}
void HostPinned::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
}

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

uint64_t pow2_at_least(uint64_t v) {
    uint64_t p = 1024;
    while (p < v) p <<= 1;
    return p;
}

Dims validate_grid(const cvlg_grid_spec* s) {
    if (!s) fail(CVLG_E_INVALID_ARG, "grid spec is NULL");
    // GridSpec::validate (grid.cpp:47-57), same order and messages
    if (!(s->lat_min < s->lat_max)) fail(CVLG_E_BAD_GRID, "BadGrid: lat_min must be < lat_max");
    if (!(s->lon_min < s->lon_max)) fail(CVLG_E_BAD_GRID, "BadGrid: lon_min must be < lon_max");
    if (!(s->lat_step > 1e-9) || !(s->lon_step > 1e-9))
        fail(CVLG_E_BAD_GRID, "BadGrid: lat_step/lon_step must be > 1e-9");
    if (s->min_step == 0 || 1440 % s->min_step != 0)
        fail(CVLG_E_BAD_GRID, "BadGrid: min_step must divide 1440");
    if (s->dxn_step == 0 || 360 % s->dxn_step != 0)
        fail(CVLG_E_BAD_GRID, "BadGrid: dxn_step must divide 360");
    if (!std::isfinite(s->dxn_offset)) fail(CVLG_E_BAD_GRID, "BadGrid: dxn_offset must be finite");
    Dims d;
    d.T = 1440 / s->min_step;
    d.D = 360 / s->dxn_step;
    d.R = extent_bins(s->lat_min, s->lat_max, s->lat_step);
    d.C = extent_bins(s->lon_min, s->lon_max, s->lon_step);
    d.RC = static_cast<uint64_t>(d.R) * d.C;
    d.cells = static_cast<uint64_t>(d.T) * d.D * d.RC;
    if (d.D > 4)
        fail(CVLG_E_UNSUPPORTED,
             "dxn_step < 90: BatchFrame holds 4 direction planes (aggregate.hpp:52-54); the "
             "reference indexes past them (undefined behaviour)");
    if (d.cells >= kCodeFirstSpecial)
        fail(CVLG_E_UNSUPPORTED, "grid has >= 2^31-16 cells; the device cell code is 31-bit");
    return d;
}

MarkSource marks_of(std::vector<ChunkMark> v) {
    auto st = std::make_shared<std::pair<std::vector<ChunkMark>, size_t>>(std::move(v), 0);
    return [st](ChunkMark& m) {
        if (st->second >= st->first.size()) return false;
        m = st->first[st->second++];
        return true;
    };
}

namespace {

GridParams make_params(const cvlg_grid_spec* s, const cvlg_filter_rules* r, const Dims& d) {
    GridParams g;
    g.lat_min = s->lat_min;
    g.lat_max = s->lat_max;
    g.lon_min = s->lon_min;
    g.lon_max = s->lon_max;
    g.lat_step = s->lat_step;
    g.lon_step = s->lon_step;
    g.dxn_offset = s->dxn_offset;
    g.dxn_step_d = static_cast<double>(s->dxn_step);
    g.min_step = s->min_step;
    g.dxn_step = s->dxn_step;
    g.R = d.R;
    g.C = d.C;
    g.D = d.D;
    g.T = d.T;
    cvlg_filter_rules def;
    cvlg_default_rules(&def);
    const cvlg_filter_rules* rr = r ? r : &def;
    g.require_in_grid = rr->require_in_grid;
    g.drop_missing = rr->drop_missing;
    g.speed_ceiling = rr->speed_ceiling;
    g.t_magic = time_magic(s->min_step);
    set_inverse_steps(g);
    return g;
}

__global__ void iota_kernel(uint32_t* v, uint64_t n) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) v[i] = static_cast<uint32_t>(i);
}

__global__ void set_u32_kernel(uint32_t* p, uint32_t v) { *p = v; }

__global__ void init_run_kernel(uint64_t* stats) {
    const int i = threadIdx.x;
    if (i < kStCount) stats[i] = 0;
}

unsigned blocks_for(uint64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

uint64_t* h_small64(cvlg_context* c) { return static_cast<uint64_t*>(c->h_small.p); }

}  // namespace

cvlg_context* default_context() {
    thread_local cvlg_context* ctx = nullptr;
    if (!ctx) ctx = cvlg_context_create(-1);
    return ctx;
}

void sync(cvlg_context* c) { CK(cudaStreamSynchronize(c->stream)); }

namespace {

// CVLG_TRACE=1: host timestamps of the pipeline phases on stderr (diagnostics only)
struct Tracer {
    bool on = std::getenv("CVLG_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void operator()(const char* what) const {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[cvlg] %9.3f ms  %s\n", ms, what);
    }
};

// NVTX ranges over the host-side phases of a run (named like the reference's stage_seconds,
// aggregate.cpp:370-449): one open range at a time, closed on every exit path.
struct NvtxStages {
    bool open = false;
    void next(const char* name) {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    void end() {
        if (open) nvtxRangePop();
        open = false;
    }
    ~NvtxStages() { end(); }
};

}  // namespace

// The pipeline proper over CSV bytes in HBM. `marks` drive incremental decode while the bytes
// stream in; the last mark must cover everything.
void run_core(cvlg_context* c, const uint8_t* d_csv, const std::vector<uint64_t>& shard_off,
              const ColumnMap* h_cmap, const uint8_t* h_good, uint64_t bad_headers,
              const cvlg_grid_spec* spec, const cvlg_filter_rules* rules, uint32_t* d_planes,
              uint32_t* d_raw, cvlg_stats* out_stats, const MarkSource& next_mark,
              bool partial, const double* feat_stop_speed, const RecordsDecodeParams* records) {
    const bool feat = feat_stop_speed != nullptr;
    if (records && feat) fail(CVLG_E_INVALID_ARG, "features are not available for records input");
    const Dims dims = validate_grid(spec);
    c->csv_in = d_csv;
    const GridParams gp = make_params(spec, rules, dims);
    cudaStream_t s = c->stream;
    const uint32_t n_shards = static_cast<uint32_t>(shard_off.size() - 1);
    const uint64_t total = records ? records->arena_len : shard_off.back();
    // (records input: tiles of kLineCap parsed records, dense)
    const uint64_t n_tiles = records ? (records->n + kLineCap - 1) / kLineCap : (total + kTile - 1) / kTile;
    if (n_tiles >= (1ull << 32)) fail(CVLG_E_UNSUPPORTED, "input larger than 64 TiB");

    c->h_small.ensure(4096);
    uint64_t* hs = h_small64(c);
    uint64_t* d_stats = nullptr;
    const Tracer TRACE;

    CK(cudaEventRecord(c->ev[0], s));
    NvtxStages nvtx;
    nvtx.next("cvlg: parse");
    // ---- setup -----------------------------------------------------------------------------
    c->stats.ensure(kStCount * 8);
    d_stats = c->stats.as<uint64_t>();
    c->shard_off.ensure((n_shards + 1) * 8);
    CK(cudaMemcpyAsync(c->shard_off.p, shard_off.data(), (n_shards + 1) * 8, cudaMemcpyHostToDevice, s));
    c->cmap.ensure(std::max<uint32_t>(n_shards, 1) * sizeof(ColumnMap));
    c->good.ensure(std::max<uint32_t>(n_shards, 1));
    if (h_cmap) {
        CK(cudaMemcpyAsync(c->cmap.p, h_cmap, n_shards * sizeof(ColumnMap), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c->good.p, h_good, n_shards, cudaMemcpyHostToDevice, s));
    }
    c->tiles.ensure(std::max<uint64_t>(n_tiles, 1) * 16);
    c->counter.ensure(16);

    // ---- K1 decode (slot per data line, sparse per-tile slot ranges) -----------------------------
    DecodeParams P;
    P.csv = d_csv;
    P.total_end = total;
    P.shard_off = c->shard_off.as<uint64_t>();
    P.cmap = c->cmap.as<ColumnMap>();
    P.shard_good = c->good.as<uint8_t>();
    P.n_shards = n_shards;
    P.grid = gp;
    P.stats = d_stats;
    P.aligned16 = (reinterpret_cast<uintptr_t>(d_csv) % 16) == 0;
    const uint64_t reg = n_tiles * static_cast<uint64_t>(kLineCap);
    // Tiles with more than kLineCap data lines (lines averaging < 43 bytes) draw slots from an
    // overflow region; sized small first and re-run with the exact demand if it ever fills.
    uint64_t ovf_cap = 4096 + total / 512;
    uint64_t N = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const uint64_t S_all = reg + ovf_cap;
        if (S_all >= (1ull << 32)) fail(CVLG_E_UNSUPPORTED, "input too large for 32-bit slot ids");
        c->ts.ensure(S_all * 8);
        c->speed.ensure(S_all * 8);
        c->code.ensure(S_all * 4);
        c->loff.ensure(S_all * 8);
        c->hscr.ensure(S_all * 4);
        c->hid_scr.ensure(S_all * 8);
        c->hkey_scr.ensure(S_all * 16);
        P.out.ts = c->ts.as<int64_t>();
        P.out.speed = c->speed.as<double>();
        P.out.code = c->code.as<uint32_t>();
        P.out.loff = c->loff.as<uint64_t>();
        P.out.lat = nullptr;
        P.out.lon = nullptr;
        if (feat) {
            c->lat.ensure(S_all * 8);
            c->lon.ensure(S_all * 8);
            P.out.lat = c->lat.as<double>();
            P.out.lon = c->lon.as<double>();
        }
        P.out.hslot = c->hscr.as<uint32_t>();
        P.out.hid = c->hid_scr.as<uint64_t>();
        P.out.hkey = c->hkey_scr.as<ulonglong2>();
        P.out.tiles = c->tiles.as<uint4>();
        P.out.reg_slots = reg;
        P.out.ovf_slots = c->counter.as<unsigned long long>();
        P.out.ovf_heads = c->counter.as<unsigned long long>() + 1;
        P.out.ovf_slot_cap = ovf_cap;
        P.out.ovf_head_cap = ovf_cap;
        init_run_kernel<<<1, 32, 0, s>>>(d_stats);
        count_launch();
        if (records) {  // already-parsed records: fill K1's outputs directly
            RecordsDecodeParams RP = *records;
            RP.n_tiles = static_cast<uint32_t>(n_tiles);
            RP.grid = gp;
            RP.out = P.out;
            RP.stats = d_stats;
            CK(cudaMemsetAsync(c->counter.p, 0, 16, s));
            CK(cudaEventRecord(c->ev_dec0, s));
            launch_records_decode(RP, s);
            count_launch();
        } else {
            if (h_cmap) {
                if (bad_headers) {
                    hs[0] = bad_headers;
                    CK(cudaMemcpyAsync(d_stats + kStBadHeader, hs, 8, cudaMemcpyHostToDevice, s));
                }
            } else {
                launch_parse_headers(d_csv, P.shard_off, n_shards, c->cmap.as<ColumnMap>(),
                                     c->good.as<uint8_t>(), d_stats, s);
                count_launch();
            }
            CK(cudaMemsetAsync(c->counter.p, 0, 16, s));
            CK(cudaEventRecord(c->ev_dec0, s));
            uint64_t tiles_done = 0;
            if (attempt == 0) {
                ChunkMark m;
                while (next_mark(m)) {
                    const bool last = m.avail_end >= total;
                    const uint64_t t_hi =
                        last ? n_tiles : std::min<uint64_t>(m.safe_end / kTile, n_tiles);
                    if (m.ready) CK(cudaStreamWaitEvent(s, m.ready, 0));
                    if (t_hi > tiles_done) {
                        P.avail_end = m.avail_end;
                        P.tile_end = static_cast<uint32_t>(t_hi);
                        launch_decode(P, static_cast<uint32_t>(tiles_done), static_cast<uint32_t>(t_hi - tiles_done), s);
                        count_launch();
                        tiles_done = t_hi;
                    }
                }
                if (tiles_done < n_tiles) fail(CVLG_E_INTERNAL, "input stream ended early");
            } else if (n_tiles) {
                P.avail_end = total;
                P.tile_end = static_cast<uint32_t>(n_tiles);
                launch_decode(P, 0, static_cast<uint32_t>(n_tiles), s);
                count_launch();
            }
        }
        CK(cudaEventRecord(c->ev_dec1, s));
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hs, d_stats, kStCount * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hs + 32, c->counter.p, 16, cudaMemcpyDeviceToHost, s));
        sync(c);
        N = hs[kStRowsRead];
        const uint64_t need = std::max(hs[32], hs[33]);
        if (!hs[kStOverflow] || need <= ovf_cap) break;
        ovf_cap = need;  // exact demand of the overflow tiles
    }
    CK(cudaEventRecord(c->ev[1], s));
    nvtx.next("cvlg: dedup+filter+accumulate");
        TRACE("decode done");
    if (hs[kStOverflow]) fail(CVLG_E_INTERNAL, "decode capacity invariant violated");
    const uint64_t n_parsed = hs[kStParsed];
    const uint64_t hs_inert = hs[kStInert];
    c->last_slots = 0;  // the slot space is sparse (see cvlg_debug_slots)
    c->dbg_tiles = n_tiles;
    c->dbg_lines = N + hs_inert;
    const uint64_t transitions = hs[kStGTransitions];
    const uint64_t H = hs[kStHeads];
    // Order keys use the biased epoch (ts - INT64_MIN: signed order as unsigned); the radix sort
    // skips the digits that are constant across keys, so no ts range reduction is needed.
    const int64_t ts_min = INT64_MIN;
    if (N >= (1ull << 32) - 1) fail(CVLG_E_UNSUPPORTED, ">= 2^32-1 data lines on one device");

    const uint64_t lattice_words = static_cast<uint64_t>(dims.T) * 8 * dims.RC;
    const uint64_t raw_words = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
    if (d_planes) CK(cudaMemsetAsync(d_planes, 0, lattice_words * 4, s));
    if (d_raw) CK(cudaMemsetAsync(d_raw, 0, raw_words * 4, s));

    bool slow = false;
    c->slow_key_ts = false;
    uint64_t J = 0;
    if (n_parsed > 0) {
        c->scal.ensure(128);
        CK(cudaMemsetAsync(c->scal.p, 0, 128, s));
        unsigned long long* d_maxlen = c->scal.as<unsigned long long>();
        uint32_t* d_total = c->scal.as<uint32_t>() + 4;
        unsigned long long* d_orand = c->scal.as<unsigned long long>() + 4;
        unsigned long long* h_orand = reinterpret_cast<unsigned long long*>(hs + 40);
        uint32_t* d_invalid = c->scal.as<uint32_t>() + 12;
        // dictionary capacity: 2x the distinct ids, which are at most H (and usually far fewer:
        // every run head inserts its journey); start at <= 8M entries, grow if a probe chain fills
        // (<= 2M entries = 32 MB first: L2-resident probes; row-shuffled input has a head per line)
        uint64_t dcap = pow2_at_least(2 * std::min<uint64_t>(H, 1ull << 20));
        const uint64_t flag_n = std::max<uint64_t>({pow2_at_least(2 * H), n_tiles + 1, N + 1});
        c->flags.ensure(flag_n * 4 + 16);
        c->pos.ensure(flag_n * 4 + 16);
        c->scan_tmp.ensure(scan_temp_words(flag_n) * 4 + 64);

        // ---- run heads: K1 listed them per tile; dense list in tile order + run ends -------------
        c->hslot.ensure(H * 4 + 4);
        c->hend.ensure(H * 4 + 4);
        c->thpos.ensure(n_tiles * 4 + 4);
        launch_tile_field(c->tiles.as<uint4>(), n_tiles, 3, c->flags.as<uint32_t>(), s);
        exclusive_scan_u32(c->flags.as<uint32_t>(), c->thpos.as<uint32_t>(), n_tiles, nullptr,
                           c->scan_tmp.as<uint32_t>(), s);
        c->hid.ensure(H * 8 + 8);

        // ---- journey dictionary ----------------------------------------------------------------
        c->hdict.ensure(H * 4);
        uint32_t* d_dict_full = c->scal.as<uint32_t>() + 16;
        for (int attempt = 0;; ++attempt) {
            c->dict.ensure(dcap * 16);
            CK(cudaMemsetAsync(c->dict.p, 0xFF, dcap * 16, s));
            CK(cudaMemsetAsync(d_dict_full, 0, 4, s));
            DictParams DP;
            DP.csv = d_csv;
            DP.shard_off = P.shard_off;
            DP.cmap = P.cmap;
            DP.n_shards = n_shards;
            DP.csv_len = total;
            DP.hid = c->hid.as<uint64_t>();
            DP.hkey = nullptr;  // (inserted by heads_compact from K1's per-tile keys)
            DP.n_heads = H;
            DP.table = c->dict.as<unsigned long long>();
            DP.mask = dcap - 1;
            DP.hdict = c->hdict.as<uint32_t>();
            DP.max_len = d_maxlen;
            DP.full = d_dict_full;
            // dense run-head list in tile order + run ends, each head's id inserted on the way
            launch_heads_compact(c->tiles.as<uint4>(), n_tiles, c->thpos.as<uint32_t>(),
                                 c->hscr.as<uint32_t>(), c->hid_scr.as<uint64_t>(),
                                 c->hkey_scr.as<ulonglong2>(), c->hslot.as<uint32_t>(),
                                 c->hend.as<uint32_t>(), c->hid.as<uint64_t>(), nullptr, s, &DP);
            TRACE("dict inserted");
            launch_dict_flags(c->dict.as<unsigned long long>(), dcap, c->flags.as<uint32_t>(), s);
            exclusive_scan_u32(c->flags.as<uint32_t>(), c->pos.as<uint32_t>(), dcap, d_total,
                               c->scan_tmp.as<uint32_t>(), s);
            CK(cudaMemcpyAsync(hs, c->scal.p, 128, cudaMemcpyDeviceToHost, s));
            sync(c);
            if (static_cast<uint32_t*>(static_cast<void*>(hs))[16] == 0) break;
            if (dcap >= pow2_at_least(2 * H)) fail(CVLG_E_INTERNAL, "journey dictionary overflow");
            dcap = pow2_at_least(2 * H);  // a probe chain filled up: exact bound
        }
        const uint64_t max_len = hs[0];
        J = static_cast<uint32_t*>(static_cast<void*>(hs))[4];
        c->uslot.ensure(J * 4);
        if (TRACE.on) {
            char msg[256];
            std::snprintf(msg, sizeof(msg), "dict compacted: N=%llu parsed=%llu H=%llu J=%llu trans=%llu maxlen=%llu",
                          (unsigned long long)N, (unsigned long long)n_parsed, (unsigned long long)H,
                          (unsigned long long)J, (unsigned long long)transitions, (unsigned long long)max_len);
            TRACE(msg);
        }
        launch_dict_compact(c->flags.as<uint32_t>(), c->pos.as<uint32_t>(), dcap,
                            c->uslot.as<uint32_t>(), s);

        // ---- lexicographic rank: LSD over (length, then 8-byte chunks last..first) ----------------
        const uint64_t sort_n = std::max<uint64_t>({J, H, N + hs_inert});
        c->keys.ensure(sort_n * 8);
        c->keys_alt.ensure(sort_n * 8);
        c->vals.ensure(sort_n * 4);
        c->vals_alt.ensure(sort_n * 4);
        c->sort_tmp.ensure(radix_temp_bytes(sort_n));
        iota_kernel<<<blocks_for(J, 256), 256, 0, s>>>(c->vals.as<uint32_t>(), J);
        count_launch();
        const int n_chunks = static_cast<int>((max_len + 7) / 8);
        for (int ch = -1; ch < n_chunks; ++ch) {
            const int cc = ch < 0 ? -1 : n_chunks - 1 - ch;
            launch_dict_chunk(c->dict.as<unsigned long long>(), c->uslot.as<uint32_t>(),
                              c->vals.as<uint32_t>(), J, cc, d_csv, c->keys.as<uint64_t>(), s);
            radix_sort_pairs(c->keys.as<uint64_t>(), c->vals.as<uint32_t>(),
                             c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), J, 0, 64,
                             c->sort_tmp.p, s, d_orand, h_orand);
        }
        c->rank_of_slot.ensure(dcap * 4);
        launch_dict_rank(c->uslot.as<uint32_t>(), c->vals.as<uint32_t>(), J,
                         c->rank_of_slot.as<uint32_t>(), s);
        c->rank_slot.ensure(J * 4 + 4);
        launch_rank_slot(c->uslot.as<uint32_t>(), c->vals.as<uint32_t>(), J,
                         c->rank_slot.as<uint32_t>(), s);
        c->hrank.ensure(H * 4);
        // runs averaging < 4 records (row-shuffled input) go straight to the full sort, whose keys
        // take the rank from (hdict, rank_of_slot) directly: the head rank list is then only
        // needed by the feature table
        const bool pre_slow = H * 4 > n_parsed;
        if (!pre_slow || feat)
            launch_head_rank(c->hdict.as<uint32_t>(), c->rank_of_slot.as<uint32_t>(), H,
                         c->hrank.as<uint32_t>(), s);
        TRACE("dict sorted");

        // ---- canonical order -----------------------------------------------------------------
        const int tsbits = 64;
        TRACE("ranks done");
        c->jstart.ensure((J + 1) * 4);
        c->srank.ensure(sort_n * 4);
        uint32_t* jstart = c->jstart.as<uint32_t>();
        // runs averaging < 4 records (row-shuffled input): the run merge cannot pay, go straight
        // to the full sort (the head sort + order check would cost as much as the sort itself)
        slow = pre_slow;
        if (!slow) {
            const int rbits = bits_for(J - 1);
            const int mode = 1;  // sort by ts, then (stably) by rank
            CK(cudaMemsetAsync(d_invalid, 0, 4, s));
            launch_head_keys(c->hrank.as<uint32_t>(), c->hslot.as<uint32_t>(), c->ts.as<int64_t>(),
                             H, ts_min, tsbits, mode, c->keys.as<uint64_t>(),
                             c->vals.as<uint32_t>(), s);
            radix_sort_pairs(c->keys.as<uint64_t>(), c->vals.as<uint32_t>(),
                             c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), H, 0,
                             mode == 0 ? tsbits + rbits : tsbits, c->sort_tmp.p, s, d_orand, h_orand);
            if (mode == 1) {
                launch_gather_rank_keys(c->hrank.as<uint32_t>(), c->vals.as<uint32_t>(), H,
                                        c->keys.as<uint64_t>(), s);
                radix_sort_pairs(c->keys.as<uint64_t>(), c->vals.as<uint32_t>(),
                                 c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), H, 0,
                                 rbits, c->sort_tmp.p, s, d_orand, h_orand);
            }
            launch_head_order_check(c->vals.as<uint32_t>(), c->hrank.as<uint32_t>(),
                                    c->hslot.as<uint32_t>(), c->hend.as<uint32_t>(),
                                    c->ts.as<int64_t>(), c->code.as<uint32_t>(), H, jstart,
                                    d_invalid, s);
            CK(cudaMemcpyAsync(hs, d_invalid, 4, cudaMemcpyDeviceToHost, s));
            sync(c);
            slow = static_cast<uint32_t*>(static_cast<void*>(hs))[0] != 0;
        }
        if (!slow) {
            set_u32_kernel<<<1, 1, 0, s>>>(jstart + J, static_cast<uint32_t>(H));
            count_launch();
        } else {
            // full (rank, ts) sort of every data line; provenance order breaks ties (stable);
            // rejected lines take rank J and sort after every journey. First the sparse per-tile
            // slot ranges are packed densely in provenance order (heads remapped).
            launch_tile_field(c->tiles.as<uint4>(), n_tiles, 1, c->flags.as<uint32_t>(), s);
            exclusive_scan_u32(c->flags.as<uint32_t>(), c->pos.as<uint32_t>(), n_tiles, nullptr,
                               c->scan_tmp.as<uint32_t>(), s);
            // dense slot count: data lines plus the inert "\r\n" lines that hold slots
            const uint64_t NS = N + hs[kStInert];
            c->ts2.ensure(NS * 8 + 8);
            c->speed2.ensure(NS * 8 + 8);
            c->code2.ensure(NS * 4 + 4);
            c->loff2.ensure(NS * 8 + 8);
            DensifyParams DZ;
            DZ.tiles = c->tiles.as<uint4>();
            DZ.n_tiles = n_tiles;
            DZ.lpos = c->pos.as<uint32_t>();
            DZ.hpos = c->thpos.as<uint32_t>();
            DZ.hscr = c->hscr.as<uint32_t>();
            DZ.ts = c->ts.as<int64_t>();
            DZ.speed = c->speed.as<double>();
            DZ.code = c->code.as<uint32_t>();
            DZ.loff = c->loff.as<uint64_t>();
            DZ.lat = nullptr;
            DZ.lon = nullptr;
            DZ.lat_out = nullptr;
            DZ.lon_out = nullptr;
            if (feat) {
                c->lat2.ensure(NS * 8 + 8);
                c->lon2.ensure(NS * 8 + 8);
                DZ.lat = c->lat.as<double>();
                DZ.lon = c->lon.as<double>();
                DZ.lat_out = c->lat2.as<double>();
                DZ.lon_out = c->lon2.as<double>();
            }
            DZ.ts_out = c->ts2.as<int64_t>();
            DZ.speed_out = c->speed2.as<double>();
            DZ.code_out = c->code2.as<uint32_t>();
            DZ.loff_out = c->loff2.as<uint64_t>();
            c->rec.ensure(NS * 16 + 16);
            DZ.rec_out = c->rec.as<ulonglong2>();
            long long* d_mm = reinterpret_cast<long long*>(c->scal.as<uint32_t>() + 18);
            {
                const long long init[2] = {LLONG_MAX, LLONG_MIN};
                std::memcpy(hs + 48, init, 16);
                CK(cudaMemcpyAsync(d_mm, hs + 48, 16, cudaMemcpyHostToDevice, s));
            }
            DZ.ts_mm = d_mm;
            DZ.hslot_out = c->hslot.as<uint32_t>();
            launch_densify(DZ, s);
            std::swap(c->ts, c->ts2);
            std::swap(c->speed, c->speed2);
            std::swap(c->code, c->code2);
            std::swap(c->loff, c->loff2);
            if (feat) {
                std::swap(c->lat, c->lat2);
                std::swap(c->lon, c->lon2);
            }
            c->last_slots = NS;
            const int rbits = bits_for(J);
            // one sort on (rank << span_bits | ts - ts_lo) when the kept timestamps' span and the
            // rank fit 64 bits (a day: 17 + 17 bits); else ts then (stably) rank
            int64_t key_ts_min = ts_min;
            int key_tsbits = tsbits;
            int mode = 1;
            {
                CK(cudaMemcpyAsync(hs + 48, d_mm, 16, cudaMemcpyDeviceToHost, s));  // (from densify)
                sync(c);
                const int64_t lo = static_cast<int64_t>(hs[48]), hi = static_cast<int64_t>(hs[49]);
                if (lo <= hi) {
                    const uint64_t span = static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo);
                    const int sb = span == 0 ? 1 : bits_for(span);
                    if (sb + rbits <= 64) {
                        mode = 0;
                        key_ts_min = lo;
                        key_tsbits = sb;
                    }
                }
            }
            launch_slot_keys(c->hslot.as<uint32_t>(), (!pre_slow || feat) ? c->hrank.as<uint32_t>() : nullptr,
                             c->hdict.as<uint32_t>(), c->rank_of_slot.as<uint32_t>(), H,
                             c->ts.as<int64_t>(), c->code.as<uint32_t>(), NS, key_ts_min, key_tsbits, mode,
                             static_cast<uint32_t>(J), c->keys.as<uint64_t>(),
                             c->vals.as<uint32_t>(), c->srank.as<uint32_t>(), s);
            bool in_alt = false;  // (a result in the alternate buffers is swapped in, not copied)
            radix_sort_pairs(c->keys.as<uint64_t>(), c->vals.as<uint32_t>(),
                             c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), NS, 0,
                             mode == 0 ? key_tsbits + rbits : key_tsbits, c->sort_tmp.p, s, d_orand,
                             h_orand, &in_alt);
            if (in_alt) {
                std::swap(c->keys, c->keys_alt);
                std::swap(c->vals, c->vals_alt);
            }
            if (mode == 1) {
                launch_gather_rank_keys(c->srank.as<uint32_t>(), c->vals.as<uint32_t>(), NS,
                                        c->keys.as<uint64_t>(), s);
                radix_sort_pairs(c->keys.as<uint64_t>(), c->vals.as<uint32_t>(),
                                 c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), NS, 0,
                                 rbits, c->sort_tmp.p, s, d_orand, h_orand);
            }
            c->slow_key_ts = mode == 0;  // keys hold (rank, ts - lo): the fold's dedup reads them
            // the sorted keys hold (rank << key_tsbits | ts) (mode 0) or the rank (mode 1)
            launch_slot_jstart(c->keys.as<uint64_t>(), mode == 0 ? key_tsbits : 0, NS, jstart, s);
            set_u32_kernel<<<1, 1, 0, s>>>(jstart + J, static_cast<uint32_t>(n_parsed));
            count_launch();
        }
        TRACE(slow ? "order done (slow path)" : "order done (run-merge fast path)");
        CK(cudaEventRecord(c->ev[2], s));

        // ---- per-journey fold ------------------------------------------------------------------
        const int rbits = bits_for(J - 1);
        const uint64_t pair_bound = slow ? n_parsed : std::min<uint64_t>(n_parsed, H + transitions);
        // time-bin windows write a reloaded bin's pairs twice (the first copy is vacated): margin
        const uint64_t pair_room = std::min<uint64_t>(pair_bound + pair_bound / 2 + 1024, 0xFFFFFFF0ull);
        c->pair_key.ensure(pair_room * 8 + 8);
        c->pair_sum.ensure(pair_room * 8 + 8);
        c->pair_cnt.ensure(pair_room * 4 + 4);
        uint32_t* d_pairs = c->scal.as<uint32_t>() + 13;
        FoldParams F;
        F.n_journeys = J;
        F.jstart = jstart;
        F.perm = c->vals.as<uint32_t>();
        F.hslot = c->hslot.as<uint32_t>();
        F.hend = c->hend.as<uint32_t>();
        c->runs.ensure(H * 8 + 8);
        F.runs = c->runs.as<uint2>();

        F.n_heads = H;
        F.ts = c->ts.as<int64_t>();
        F.speed = c->speed.as<double>();
        F.code = c->code.as<uint32_t>();
        F.rec = slow ? c->rec.as<ulonglong2>() : nullptr;
        F.loff = c->loff.as<uint64_t>();
        F.skey = (slow && c->slow_key_ts) ? c->keys.as<uint64_t>() : nullptr;
        F.pair_key = c->pair_key.as<uint64_t>();
        F.pair_sum = c->pair_sum.as<double>();
        F.pair_cnt = c->pair_cnt.as<uint32_t>();
        F.pair_count = d_pairs;
        F.rank_bits = rbits;
        F.journey_counter = c->scal.as<uint64_t>() + 7;
        F.r_lat = records ? records->lat : nullptr;
        F.r_lon = records ? records->lon : nullptr;
        F.r_speed = records ? records->speed : nullptr;
        F.r_heading = records ? records->heading : nullptr;
        F.r_postal = records ? records->postal : nullptr;
        F.r_postal_arena = records ? records->postal_arena : nullptr;
        F.csv = d_csv;
        F.shard_off = P.shard_off;
        F.cmap = P.cmap;
        F.n_shards = n_shards;
        F.stats = d_stats;
        // time-bin windows: a directory row of T entries per fold lane (off when it would not fit
        // comfortably, or when disabled)
        const uint64_t dir_bytes = static_cast<uint64_t>(fold_grid(J, slow)) * kFoldThreads * dims.T * 16;
        const char* wenv = std::getenv("CVLG_FOLD_WINDOWS");
        F.win = (wenv && wenv[0] == '0') ? 0 : (dir_bytes <= (4ull << 30) ? 1 : 0);
        F.drc = static_cast<uint32_t>(dims.D * dims.RC);
        F.n_bins = dims.T;
        F.dir = nullptr;
        F.dead_list = nullptr;
        F.dead_count = c->scal.as<uint32_t>() + 24;
        F.abort_flag = c->scal.as<uint32_t>() + 28;
        // short windows (fine time bins) close often: flush earlier, in bigger batches (measured:
        // slack 5 best at 1-minute bins, 1 at 5-minute bins)
        F.flush_slack = dims.T >= 720 ? 5u : 1u;
        if (F.win) {
            if (c->fold_dir.ensure(dir_bytes)) {
                CK(cudaMemsetAsync(c->fold_dir.p, 0, c->fold_dir.cap, s));
                c->fold_epoch = 0;
            }
            F.dir = c->fold_dir.as<uint4>();
            c->dead.ensure(pair_room * 8 + 8);
            F.dead_list = c->dead.as<uint32_t>();
        }
        // The spill table only holds journeys with more distinct cells than a lane keeps in
        // shared memory (or a window holds); start small and re-run with the exact bound (and
        // without windows) if it ever fills.
        // (windows keep most subtotals out of the spill table unless they are long: few bins)
        // ---- bin-group mode: few journeys for the lanes (each lane would fold one long journey
        // alone): the work items become (journey, time bin) groups of run pieces ------------------
        F.jrank = nullptr;
        F.runs_ready = 0;
        {
            const char* genv = std::getenv("CVLG_FOLD_GROUPS");
            const uint64_t lanes = static_cast<uint64_t>(fold_grid(~0ull >> 1, false)) * kFoldThreads;
            const int jb = bits_for(J), bb = bits_for(dims.T), rb = bits_for(H);
            const bool want = genv ? genv[0] == '1' : J * 8 <= lanes;
            if (!slow && J && H && want && jb + bb + rb + 9 <= 64 && H < (1ull << 32)) {
                const uint64_t cap = H + transitions + 16;
                c->run_j.ensure(H * 4 + 4);
                c->gkeys.ensure(cap * 8);
                c->gkeys_alt.ensure(cap * 8);
                c->gvals.ensure(cap * 4);
                c->gvals_alt.ensure(cap * 4);
                c->gpieces.ensure(cap * 8);
                c->gruns.ensure(cap * 8);
                c->flags.ensure(cap * 4 + 16);
                c->pos.ensure(cap * 4 + 16);
                c->scan_tmp.ensure(scan_temp_words(cap) * 4 + 64);
                c->sort_tmp.ensure(radix_temp_bytes(cap));
                launch_run_list(F.perm, F.hslot, F.hend, H, const_cast<uint2*>(F.runs), s);
                uint32_t* d_cnt = c->scal.as<uint32_t>() + 30;
                CK(cudaMemsetAsync(d_cnt, 0, 8, s));
                launch_bin_pieces(F.runs, H, jstart, J, c->run_j.as<uint32_t>(), F.code, F.drc, bb, rb,
                                  c->gkeys.as<uint64_t>(), c->gvals.as<uint32_t>(),
                                  c->gpieces.as<uint2>(), d_cnt, cap, s);
                CK(cudaMemcpyAsync(hs, d_cnt, 8, cudaMemcpyDeviceToHost, s));
                sync(c);
                const uint64_t n_pieces = static_cast<uint32_t*>(static_cast<void*>(hs))[0];
                const bool order_ovf = static_cast<uint32_t*>(static_cast<void*>(hs))[1] != 0;
                if (n_pieces > cap) fail(CVLG_E_INTERNAL, "bin pieces exceed their bound");
                if (!order_ovf) {
                radix_sort_pairs(c->gkeys.as<uint64_t>(), c->gvals.as<uint32_t>(),
                                 c->gkeys_alt.as<uint64_t>(), c->gvals_alt.as<uint32_t>(), n_pieces, 0,
                                 jb + bb + rb + 9, c->sort_tmp.p, s, d_orand, h_orand);
                launch_bin_groups(c->gkeys.as<uint64_t>(), c->gvals.as<uint32_t>(), c->gpieces.as<uint2>(),
                                  n_pieces, rb + 9, bb, c->flags.as<uint32_t>(), c->gruns.as<uint2>(), s);
                exclusive_scan_u32(c->flags.as<uint32_t>(), c->pos.as<uint32_t>(), n_pieces, d_cnt,
                                   c->scan_tmp.as<uint32_t>(), s);
                CK(cudaMemcpyAsync(hs, d_cnt, 4, cudaMemcpyDeviceToHost, s));
                sync(c);
                const uint64_t G = static_cast<uint32_t*>(static_cast<void*>(hs))[0];
                c->gstart.ensure(G * 4 + 8);
                c->gj.ensure(G * 4 + 4);
                launch_bin_group_starts(c->gkeys.as<uint64_t>(), c->flags.as<uint32_t>(),
                                        c->pos.as<uint32_t>(), n_pieces, rb + 9, bb,
                                        c->gstart.as<uint32_t>(), c->gj.as<uint32_t>(), s);
                set_u32_kernel<<<1, 1, 0, s>>>(c->gstart.as<uint32_t>() + G, static_cast<uint32_t>(n_pieces));
                count_launch();
                F.n_journeys = G;
                F.jstart = c->gstart.as<uint32_t>();
                F.runs = c->gruns.as<uint2>();
                F.runs_ready = 1;
                F.jrank = c->gj.as<uint32_t>();
                F.win = 0;  // one bin per group: nothing to window
                TRACE("fold: bin groups");
                } else {  // a run with > 511 pieces: fold whole journeys (runs are already built)
                    F.runs_ready = 1;
                }
            }
        }
        // ---- longest-first work order (journey mode): sort the work items by record count -------
        F.jorder = nullptr;
        {
            const char* oenv = std::getenv("CVLG_FOLD_ORDER");
            const uint64_t nj = F.n_journeys;
            if (!F.jrank && nj > 1 && !(oenv && oenv[0] == '0')) {
                if (!slow && !F.runs_ready) {
                    launch_run_list(F.perm, F.hslot, F.hend, H, const_cast<uint2*>(F.runs), s);
                    F.runs_ready = 1;
                }
                c->jo_keys.ensure(nj * 8);
                c->jo_keys_alt.ensure(nj * 8);
                c->jo_vals.ensure(nj * 4);
                c->jo_vals_alt.ensure(nj * 4);
                c->sort_tmp.ensure(radix_temp_bytes(nj));
                launch_journey_len_keys(F.jstart, nj, F.runs, slow ? 0 : 1, c->jo_keys.as<uint64_t>(),
                                        c->jo_vals.as<uint32_t>(), s);
                radix_sort_pairs(c->jo_keys.as<uint64_t>(), c->jo_vals.as<uint32_t>(),
                                 c->jo_keys_alt.as<uint64_t>(), c->jo_vals_alt.as<uint32_t>(), nj, 0, 32,
                                 c->sort_tmp.p, s, d_orand, h_orand);
                F.jorder = c->jo_vals.as<uint32_t>();
            }
        }
        uint64_t scap = pow2_at_least(std::max<uint64_t>(F.win ? 1u << 20 : 1u << 18,
                                                         pair_bound / (F.win && dims.T > 48 ? 16 : 2)));
        F.pair_cap = F.win ? pair_room : pair_bound;
        for (int attempt = 0; attempt < 3; ++attempt) {
            if (++c->fold_epoch == 0) {  // directory tags wrapped: clear the stale ones
                if (F.dir) CK(cudaMemsetAsync(c->fold_dir.p, 0, c->fold_dir.cap, s));
                c->fold_epoch = 1;
            }
            F.epoch = c->fold_epoch;
            CK(cudaMemsetAsync(F.dead_count, 0, 4, s));
            CK(cudaMemsetAsync(F.abort_flag, 0, 4, s));
            c->spill_key.ensure(scap * 8);
            c->spill_sum.ensure(scap * 8);
            c->spill_cnt.ensure(scap * 4);
            CK(cudaMemsetAsync(c->spill_key.p, 0xFF, scap * 8, s));
            CK(cudaMemsetAsync(d_pairs, 0, 4, s));
            CK(cudaMemsetAsync(F.journey_counter, 0, 8, s));
            CK(cudaMemsetAsync(d_stats + kStDups, 0, (kStFiltMissing - kStDups + 1) * 8, s));
            CK(cudaMemsetAsync(d_stats + kStUnbinnable, 0, 2 * 8, s));
            F.spill_key = c->spill_key.as<uint64_t>();
            F.spill_sum = c->spill_sum.as<double>();
            F.spill_cnt = c->spill_cnt.as<uint32_t>();
            F.spill_mask = scap - 1;
            launch_fold(F, slow, s);
            CK(cudaMemcpyAsync(hs, d_pairs, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(hs) + 1, F.dead_count, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(hs + 1, d_stats + kStOverflow, 8, cudaMemcpyDeviceToHost, s));
            sync(c);
            if (hs[1] == 0) break;
            const bool pairs_full = reinterpret_cast<uint32_t*>(hs)[0] > F.pair_cap;
            TRACE(pairs_full ? "fold: pair list overflow, re-run without windows"
                             : "fold: spill table overflow, re-run with a larger table");
            scap = pow2_at_least(2 * pair_bound);
            // windows can write more pairs than pair_bound: a retry without them is bounded by it
            // (the last attempt never keeps windows, whatever the previous one overflowed)
            if (pairs_full || attempt >= 1) {
                F.win = 0;
                F.pair_cap = pair_bound;
            }
        }
        const uint64_t n_written = std::min<uint64_t>(reinterpret_cast<uint32_t*>(hs)[0], F.pair_cap);
        const uint64_t n_dead = F.win ? reinterpret_cast<uint32_t*>(hs)[1] : 0;
        if (n_dead) {
            launch_pair_compact(c->pair_key.as<uint64_t>(), c->pair_sum.as<double>(),
                                c->pair_cnt.as<uint32_t>(), n_written, n_dead, F.dead_list,
                                F.dead_list + pair_room, c->scal.as<uint32_t>() + 26, s);
        }
        CK(cudaEventRecord(c->ev[3], s));
        nvtx.next("cvlg: merge+finalize");
        const uint64_t n_pairs = n_written - n_dead;

        if (feat) {  // per-journey features over the fold's record order (features.cu)
            c->f_J = J;
            c->f_cells = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
            c->f_points.ensure(J * 4 + 4);
            c->f_tfirst.ensure(J * 8 + 8);
            c->f_tlast.ensure(J * 8 + 8);
            c->f_len.ensure(J * 8 + 8);
            c->f_step.ensure(J * 8 + 8);
            c->f_vmax.ensure(J * 8 + 8);
            c->f_acc.ensure(J * 8 + 8);
            c->f_dwell.ensure(J * 8 + 8);
            c->f_stops.ensure(J * 4 + 4);
            c->f_id.ensure(J * 8 + 8);
            c->f_first.ensure(J * 4 + 4);
            c->f_cmin.ensure(c->f_cells * 4);
            c->f_cmax.ensure(c->f_cells * 4);
            FeatureParams FP;
            FP.n_journeys = J;
            FP.jstart = jstart;
            FP.perm = c->vals.as<uint32_t>();
            FP.runs = c->runs.as<uint2>();
            FP.slow = slow ? 1 : 0;
            FP.ts = c->ts.as<int64_t>();
            FP.speed = c->speed.as<double>();
            FP.lat = c->lat.as<double>();
            FP.lon = c->lon.as<double>();
            FP.code = c->code.as<uint32_t>();
            FP.stop_speed = *feat_stop_speed;
            FP.D = dims.D;
            FP.RC = dims.RC;
            FP.points = c->f_points.as<uint32_t>();
            FP.t_first = c->f_tfirst.as<int64_t>();
            FP.t_last = c->f_tlast.as<int64_t>();
            FP.length_m = c->f_len.as<double>();
            FP.max_step_m = c->f_step.as<double>();
            FP.max_speed = c->f_vmax.as<double>();
            FP.max_abs_accel = c->f_acc.as<double>();
            FP.dwell_s = c->f_dwell.as<double>();
            FP.stops = c->f_stops.as<uint32_t>();
            FP.cell_min = c->f_cmin.as<uint32_t>();
            FP.cell_max = c->f_cmax.as<uint32_t>();
            launch_journey_features(FP, c->hrank.as<uint32_t>(), H, c->hid.as<uint64_t>(),
                                    c->f_first.as<uint32_t>(), c->f_id.as<uint64_t>(), c->f_cells, s);
        }
        c->part_pairs = n_pairs;
        c->part_rbits = rbits;
        c->part_J = J;
        c->part_long_ids = max_len > 15;
        // ---- (cell, journey) subtotals -> canonical per-cell fold ----------------------------------
        if (!partial) {
        c->keys_alt.ensure(std::max<uint64_t>(n_pairs, sort_n) * 8);
        c->vals.ensure(std::max<uint64_t>(n_pairs, sort_n) * 4);
        c->vals_alt.ensure(std::max<uint64_t>(n_pairs, sort_n) * 4);
        c->sort_tmp.ensure(radix_temp_bytes(std::max<uint64_t>(n_pairs, sort_n)));
        launch_pair_vals(c->vals.as<uint32_t>(), n_pairs, s);
        const int gbits = bits_for(dims.cells - 1);
        radix_sort_pairs(c->pair_key.as<uint64_t>(), c->vals.as<uint32_t>(),
                         c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), n_pairs, 0,
                         gbits + rbits, c->sort_tmp.p, s, d_orand, h_orand);
        CK(cudaEventRecord(c->ev[4], s));
        launch_finalize(c->pair_key.as<uint64_t>(), c->vals.as<uint32_t>(), n_pairs, rbits,
                        c->pair_sum.as<double>(), c->pair_cnt.as<uint32_t>(), dims.D, dims.RC,
                        0, dims.T, d_planes, d_raw, s);
        } else {
            CK(cudaEventRecord(c->ev[4], s));
        }
    } else {
        if (feat) {
            c->f_J = 0;
            c->f_cells = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
            c->f_cmin.ensure(c->f_cells * 4);
            c->f_cmax.ensure(c->f_cells * 4);
            CK(cudaMemsetAsync(c->f_cmin.p, 0, c->f_cells * 4, s));
            CK(cudaMemsetAsync(c->f_cmax.p, 0, c->f_cells * 4, s));
        }
        c->part_pairs = 0;
        c->part_J = 0;
        c->part_long_ids = false;
        CK(cudaEventRecord(c->ev[2], s));
        CK(cudaEventRecord(c->ev[3], s));
        nvtx.next("cvlg: merge+finalize");
        CK(cudaEventRecord(c->ev[4], s));
    }
    CK(cudaEventRecord(c->ev[5], s));
    nvtx.end();
    CK(cudaMemcpyAsync(hs, d_stats, kStCount * 8, cudaMemcpyDeviceToHost, s));
    sync(c);
    CK(cudaGetLastError());
    if (hs[kStOverflow]) fail(CVLG_E_INTERNAL, "aggregation capacity invariant violated");
    // the reference's stages (aggregate.cpp:370-383, 449): parse | dedup+filter+accumulate
    // (dictionary, canonical order, per-journey fold) | merge (the (cell, journey) sort that
    // brings every cell's subtotals together) | finalize
    float ms[4] = {0, 0, 0, 0};
    cudaEventElapsedTime(&ms[0], c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&ms[1], c->ev[1], c->ev[3]);
    cudaEventElapsedTime(&ms[2], c->ev[3], c->ev[4]);
    cudaEventElapsedTime(&ms[3], c->ev[4], c->ev[5]);
    for (int i = 0; i < 4; ++i) c->stage_ms[i] = ms[i];
    cudaEventElapsedTime(&c->stage_ms[4], c->ev_dec0, c->ev_dec1);
    cudaEventElapsedTime(&c->stage_ms[5], c->ev[1], c->ev[2]);
    if (out_stats) {
        cvlg_stats& st = *out_stats;
        std::memset(&st, 0, sizeof(st));
        st.rows_read = hs[kStRowsRead];
        st.parsed = hs[kStParsed];
        st.duplicates_dropped = hs[kStDups];
        st.conflicting_duplicates = hs[kStConflicts];
        st.accepted = hs[kStAccepted];
        for (int i = 0; i < 4; ++i) st.rejected[i] = hs[kStRejBase + i];
        st.rejected[4] = hs[kStBadHeader];
        st.filtered[0] = hs[kStFiltOutOfGrid];
        st.filtered[1] = hs[kStFiltSpeed];
        st.filtered[2] = hs[kStFiltMissing];
        for (int i = 0; i < 4; ++i) st.stage_seconds[i] = ms[i] / 1000.0;
    }
    if (hs[kStUnbinnable])
        fail(CVLG_E_OUT_OF_BOUNDS,
             "OutOfBounds: a kept record lies outside the grid (require_in_grid = false)");
}

namespace {

// Host-side header map for shards whose bytes are in host memory.
void host_headers(const uint8_t* const* bufs, const uint64_t* lens, size_t n,
                  std::vector<ColumnMap>& cmap, std::vector<uint8_t>& good, uint64_t& bad) {
    cmap.resize(n);
    good.resize(n);
    bad = 0;
    for (size_t s = 0; s < n; ++s) {
        ColumnMap m;
        std::memset(&m, 0xFF, sizeof(m));
        m.n_columns = 0;
        if (lens[s] == 0) {
            good[s] = 0;
            cmap[s] = m;
            continue;
        }
        const uint8_t* b = bufs[s];
        const void* nlp = std::memchr(b, '\n', lens[s]);
        uint64_t len = nlp ? static_cast<uint64_t>(static_cast<const uint8_t*>(nlp) - b) : lens[s];
        if (len > 0 && b[len - 1] == '\r') --len;
        const bool ok = parse_header(b, static_cast<int64_t>(len), m);
        good[s] = ok ? 1 : 0;
        cmap[s] = m;
        if (!ok) ++bad;
    }
}

void run_host(cvlg_context* c, const uint8_t* const* bufs, const uint64_t* lens, size_t n,
              const cvlg_grid_spec* spec, const cvlg_filter_rules* rules, uint32_t* planes,
              uint32_t* raw, cvlg_stats* stats, const double* feat_stop_speed = nullptr) {
    const Dims dims = validate_grid(spec);
    std::vector<uint64_t> off(n + 1, 0);
    for (size_t i = 0; i < n; ++i) off[i + 1] = off[i] + lens[i];
    const uint64_t total = off[n];
    std::vector<ColumnMap> cmap;
    std::vector<uint8_t> good;
    uint64_t bad = 0;
    host_headers(bufs, lens, n, cmap, good, bad);
    c->csv.ensure(total + 16);
    c->input_bytes = total;
    uint8_t* d_csv = c->csv.as<uint8_t>();
    // chunked, line-aligned H2D on the copy stream, decode overlapped on the compute stream
    constexpr uint64_t kChunk = 64ull << 20;
    std::vector<ChunkMark> marks;
    size_t ev_i = 0;
    auto next_event = [&]() {
        if (ev_i >= c->chunk_events.size()) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->chunk_events.push_back(e);
        }
        return c->chunk_events[ev_i++];
    };
    // the copy stream must not start before the previous run finished with the buffer
    cudaEvent_t start_ev = next_event();
    CK(cudaEventRecord(start_ev, c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, start_ev, 0));
    uint64_t safe = 0;
    for (size_t sidx = 0; sidx < n; ++sidx) {
        const uint64_t len = lens[sidx];
        for (uint64_t a = 0; a < len; a += kChunk) {
            const uint64_t b = std::min(len, a + kChunk);
            CK(cudaMemcpyAsync(d_csv + off[sidx] + a, bufs[sidx] + a, b - a, cudaMemcpyHostToDevice,
                               c->copy_stream));
            cudaEvent_t e = next_event();
            CK(cudaEventRecord(e, c->copy_stream));
            if (b == len) {
                safe = off[sidx + 1];
            } else {
                // last '\n' in the piece
                const uint8_t* p = bufs[sidx] + a;
                uint64_t k = b - a;
                while (k > 0 && p[k - 1] != '\n') --k;
                if (k > 0) safe = off[sidx] + a + k;
            }
            marks.push_back(ChunkMark{off[sidx] + b, safe, e});
        }
    }
    if (marks.empty()) marks.push_back(ChunkMark{total, total, nullptr});
    uint32_t* d_planes;
    uint32_t* d_raw = nullptr;
    const uint64_t lattice_words = static_cast<uint64_t>(dims.T) * 8 * dims.RC;
    const uint64_t raw_words = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
    c->planes.ensure(lattice_words * 4);
    d_planes = c->planes.as<uint32_t>();
    if (raw) {
        c->raw.ensure(raw_words * 4);
        d_raw = c->raw.as<uint32_t>();
    }
    run_core(c, d_csv, off, cmap.data(), good.data(), bad, spec, rules, d_planes, d_raw, stats,
             marks_of(std::move(marks)), false, feat_stop_speed);
    if (planes)
        CK(cudaMemcpyAsync(planes, d_planes, lattice_words * 4, cudaMemcpyDeviceToHost, c->stream));
    if (raw) CK(cudaMemcpyAsync(raw, d_raw, raw_words * 4, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
}

// Parsed records (run_pipeline_from_records, aggregate.cpp:454-491): provenance ranks from the
// sorted unique shard paths (:464-468), columns and id / postal arenas uploaded by record index,
// a stable device sort by (rank, (uint32) line) gives the slot order, and the pipeline runs from
// its post-parse stages on (records_decode_kernel fills K1's outputs).
void run_records(cvlg_context* c, const cvlg_record* recs, size_t n, const cvlg_grid_spec* spec,
                 const cvlg_filter_rules* rules, uint32_t* planes, uint32_t* raw, cvlg_stats* stats) {
    const Dims dims = validate_grid(spec);
    if (n >= (1ull << 32) - 1) fail(CVLG_E_UNSUPPORTED, ">= 2^32-1 records on one device");
    cudaStream_t s = c->stream;
    // provenance ranks: lexicographic order of the distinct paths
    std::unordered_map<std::string_view, uint32_t> path_ix;
    std::vector<std::string_view> uniq;
    for (size_t i = 0; i < n; ++i) {
        const std::string_view v(recs[i].shard_path ? recs[i].shard_path : "", recs[i].shard_path_len);
        if (path_ix.emplace(v, 0u).second) uniq.push_back(v);
    }
    std::sort(uniq.begin(), uniq.end());
    for (size_t r = 0; r < uniq.size(); ++r) path_ix[uniq[r]] = static_cast<uint32_t>(r);
    std::vector<uint64_t> key(n), id(n), postal(n);
    std::vector<int64_t> ts(n);
    std::vector<double> lat(n), lon(n), speed(n), heading(n);
    uint64_t id_bytes = 0, postal_bytes = 0;
    for (size_t i = 0; i < n; ++i) {
        id_bytes += recs[i].journey_len;
        postal_bytes += recs[i].postal_len;
    }
    if (id_bytes >= (1ull << 40) || postal_bytes >= (1ull << 40)) fail(CVLG_E_UNSUPPORTED, "string arenas too large");
    std::vector<uint8_t> arena(id_bytes + 16), parena(postal_bytes + 16);
    uint64_t ia = 0, pa = 0;
    for (size_t i = 0; i < n; ++i) {
        const cvlg_record& r = recs[i];
        const std::string_view v(r.shard_path ? r.shard_path : "", r.shard_path_len);
        key[i] = (static_cast<uint64_t>(path_ix[v]) << 32) | static_cast<uint32_t>(r.line_number);
        ts[i] = r.epoch_sec;
        lat[i] = r.latitude;
        lon[i] = r.longitude;
        speed[i] = r.speed;
        heading[i] = r.heading;
        if (r.journey_len) std::memcpy(arena.data() + ia, r.journey_id, r.journey_len);
        id[i] = ia | (static_cast<uint64_t>(r.journey_len) << 40);
        ia += r.journey_len;
        if (r.postal_len) std::memcpy(parena.data() + pa, r.postal_code, r.postal_len);
        postal[i] = pa | (static_cast<uint64_t>(r.postal_len) << 40);
        pa += r.postal_len;
    }
    auto up = [&](DevBuf& b, const void* h, size_t bytes) {
        b.ensure(bytes + 16);
        if (bytes) CK(cudaMemcpyAsync(b.p, h, bytes, cudaMemcpyHostToDevice, s));
    };
    up(c->r_keys, key.data(), n * 8);
    up(c->r_ts, ts.data(), n * 8);
    up(c->r_lat, lat.data(), n * 8);
    up(c->r_lon, lon.data(), n * 8);
    up(c->r_speed, speed.data(), n * 8);
    up(c->r_heading, heading.data(), n * 8);
    up(c->r_id, id.data(), n * 8);
    up(c->r_arena, arena.data(), arena.size());
    up(c->r_postal, postal.data(), n * 8);
    up(c->r_parena, parena.data(), parena.size());
    c->r_keys_alt.ensure(n * 8 + 16);
    c->r_perm.ensure(n * 4 + 16);
    c->r_perm_alt.ensure(n * 4 + 16);
    if (n) {
        iota_kernel<<<blocks_for(n, 256), 256, 0, s>>>(c->r_perm.as<uint32_t>(), n);
        count_launch();
        c->scal.ensure(128);
        c->h_small.ensure(4096);
        c->sort_tmp.ensure(radix_temp_bytes(n));
        radix_sort_pairs(c->r_keys.as<uint64_t>(), c->r_perm.as<uint32_t>(), c->r_keys_alt.as<uint64_t>(),
                         c->r_perm_alt.as<uint32_t>(), n, 0, 64, c->sort_tmp.p, s,
                         c->scal.as<unsigned long long>() + 4,
                         reinterpret_cast<unsigned long long*>(h_small64(c) + 40));
    }
    RecordsDecodeParams RP{};
    RP.perm = c->r_perm.as<uint32_t>();
    RP.n = n;
    RP.ts = c->r_ts.as<int64_t>();
    RP.lat = c->r_lat.as<double>();
    RP.lon = c->r_lon.as<double>();
    RP.speed = c->r_speed.as<double>();
    RP.heading = c->r_heading.as<double>();
    RP.id = c->r_id.as<uint64_t>();
    RP.arena = c->r_arena.as<uint8_t>();
    RP.arena_len = id_bytes;
    RP.postal = c->r_postal.as<uint64_t>();
    RP.postal_arena = c->r_parena.as<uint8_t>();
    const uint64_t lattice_words = static_cast<uint64_t>(dims.T) * 8 * dims.RC;
    const uint64_t raw_words = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
    c->planes.ensure(lattice_words * 4);
    uint32_t* d_planes = c->planes.as<uint32_t>();
    uint32_t* d_raw = nullptr;
    if (raw) {
        c->raw.ensure(raw_words * 4);
        d_raw = c->raw.as<uint32_t>();
    }
    std::vector<uint64_t> off{0, id_bytes};
    run_core(c, RP.arena, off, nullptr, nullptr, 0, spec, rules, d_planes, d_raw, stats,
             marks_of({ChunkMark{id_bytes, id_bytes, nullptr}}), false, nullptr, &RP);
    if (planes) CK(cudaMemcpyAsync(planes, d_planes, lattice_words * 4, cudaMemcpyDeviceToHost, s));
    if (raw) CK(cudaMemcpyAsync(raw, d_raw, raw_words * 4, cudaMemcpyDeviceToHost, s));
    sync(c);
}

// Shard files in rank order -> HBM through the bounded pinned ring (read_shard's I/O half,
// ingest.cpp:195-201, threaded like aggregate.cpp:414-443): run_core decodes every tile whose
// lines are resident while later chunks are still on disk / in flight.
void run_files(cvlg_context* c, const char* const* paths, size_t n, const cvlg_grid_spec* spec,
               const cvlg_filter_rules* rules, uint32_t n_threads, uint32_t* planes, uint32_t* raw,
               cvlg_stats* stats) {
    struct Range {  // NVTX: the whole file-to-lattice call (ingest overlaps the parse stage)
        Range() { nvtxRangePushA("cvlg: run_pipeline(files)"); }
        ~Range() { nvtxRangePop(); }
    } range;
    const Dims dims = validate_grid(spec);
    // sizes and header lines (parse_header, ingest.cpp:204-221) before anything streams
    const std::vector<ShardHead> heads = read_shard_heads(paths, n);
    std::vector<uint64_t> off(n + 1, 0);
    std::vector<ColumnMap> cmap(n);
    std::vector<uint8_t> good(n, 0);
    uint64_t bad = 0;
    std::vector<FileRange> ranges;
    for (size_t r = 0; r < n; ++r) {
        off[r + 1] = off[r] + heads[r].len;
        cmap[r] = heads[r].cmap;
        good[r] = heads[r].good ? 1 : 0;
        if (heads[r].bad_header) ++bad;
        if (heads[r].len) ranges.push_back(FileRange{static_cast<uint32_t>(r), 0, heads[r].len, off[r]});
    }
    const uint64_t total = off[n];
    c->csv.ensure(total + 16);
    c->input_bytes = total;
    uint8_t* d_csv = c->csv.as<uint8_t>();
    const uint64_t lattice_words = static_cast<uint64_t>(dims.T) * 8 * dims.RC;
    const uint64_t raw_words = static_cast<uint64_t>(dims.T) * 4 * dims.RC;
    c->planes.ensure(lattice_words * 4);
    uint32_t* d_planes = c->planes.as<uint32_t>();
    uint32_t* d_raw = nullptr;
    if (raw) {
        c->raw.ensure(raw_words * 4);
        d_raw = c->raw.as<uint32_t>();
    }
    RingIngest ring(c, paths, std::move(ranges), d_csv, n_threads);
    const size_t n_chunks = ring.chunks();
    uint64_t safe = 0;
    size_t k_next = 0;
    MarkSource src = [&](ChunkMark& m) -> bool {
        if (k_next >= n_chunks) {
            if (n_chunks == 0 && k_next == 0) {  // empty input: one mark covering nothing
                ++k_next;
                m = ChunkMark{total, total, nullptr};
                return true;
            }
            return false;
        }
        RingChunk ch;
        if (!ring.next(ch)) fail(CVLG_E_INTERNAL, "ingest ring ended early");
        ++k_next;
        const uint64_t g0 = ch.dst, g1 = g0 + ch.len;
        const uint32_t r = static_cast<uint32_t>(std::upper_bound(off.begin(), off.end(), g0) - off.begin() - 1);
        if (g1 == off[r + 1]) {
            safe = g1;  // lines never cross a shard end
        } else if (ch.nl_end) {
            safe = g0 + ch.nl_end;
        }
        m = ChunkMark{g1, safe, ch.copied};
        // the final mark must cover the whole input even when trailing shards are empty
        if (k_next == n_chunks) m.avail_end = total;
        return true;
    };
    run_core(c, d_csv, off, cmap.data(), good.data(), bad, spec, rules, d_planes, d_raw, stats, src,
             false, nullptr);
    ring.stop();
    if (planes)
        CK(cudaMemcpyAsync(planes, d_planes, lattice_words * 4, cudaMemcpyDeviceToHost, c->stream));
    if (raw) CK(cudaMemcpyAsync(raw, d_raw, raw_words * 4, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
}

}  // namespace

std::vector<ShardHead> read_shard_heads(const char* const* paths, size_t n) {
    std::vector<ShardHead> heads(n);
    for (size_t r = 0; r < n; ++r) {
        ShardHead& h = heads[r];
        const int fd = ::open(paths[r], O_RDONLY);
        struct stat st;
        if (fd < 0 || ::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode)) {
            if (fd >= 0) ::close(fd);
            fail(CVLG_E_IO, std::string("Io: cannot open shard ") + paths[r]);
        }
        h.len = static_cast<uint64_t>(st.st_size);
        std::memset(&h.cmap, 0xFF, sizeof(h.cmap));
        h.cmap.n_columns = 0;
        h.data_begin = h.len;
        if (h.len) {
            std::string head;
            char buf[4096];
            uint64_t at = 0;
            size_t nl = std::string::npos;
            while (at < h.len) {
                const ssize_t k = ::pread(fd, buf, sizeof(buf), static_cast<off_t>(at));
                if (k <= 0) break;
                head.append(buf, static_cast<size_t>(k));
                at += static_cast<uint64_t>(k);
                if ((nl = head.find('\n', at - static_cast<uint64_t>(k))) != std::string::npos) break;
            }
            size_t hl = nl == std::string::npos ? head.size() : nl;
            if (nl != std::string::npos) {
                h.data_begin = nl + 1;
                h.header = head.substr(0, nl + 1);
            } else {
                h.header = head + "\n";
            }
            if (hl > 0 && head[hl - 1] == '\r') --hl;
            h.good = parse_header(reinterpret_cast<const uint8_t*>(head.data()), static_cast<int64_t>(hl), h.cmap);
            h.bad_header = !h.good;
        }
        ::close(fd);
    }
    return heads;
}

// ---- RingIngest -------------------------------------------------------------------------------
struct RingIngest::Impl {
    cvlg_context* c;
    const char* const* paths;
    std::vector<FileRange> ranges;
    uint8_t* d_dst;
    // 16 x 6 MB: small enough that the reader threads' stores are still in the host LLC when
    // the copy engine reads them (measured on the B200 host: 4 MB x 16 slots 48.6 GB/s vs
    // 32 MB x 16 slots 38.3 GB/s on c2; c3 e2e 645 (6 MB) / 656 (4 MB) vs 736 ms (32 MB),
    // profiles/r02_ingest_ring_c3.log)
    uint64_t chunk = 6ull << 20;
    int slots = 16;
    struct Chunk {
        size_t range;
        uint64_t off, len, dst;
    };
    std::vector<Chunk> chunks;
    uint8_t* ring = nullptr;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<uint8_t> ready;
    size_t enqueued = 0;  // chunks [0, enqueued) have their copy enqueued
    bool stopping = false;
    std::string err;
    std::atomic<size_t> next_read{0};
    std::vector<std::thread> pool;
    size_t k_next = 0;

    void reader() {
        cudaSetDevice(c->device);
        int fd = -1;
        uint32_t fd_file = 0xFFFFFFFFu;
        for (size_t k = next_read.fetch_add(1); k < chunks.size(); k = next_read.fetch_add(1)) {
            const Chunk& ch = chunks[k];
            const int slot = static_cast<int>(k % slots);
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stopping || k < static_cast<size_t>(slots) || enqueued > k - slots; });
                if (stopping) break;
            }
            if (cudaEventSynchronize(c->ring_events[slot]) != cudaSuccess) {
                std::lock_guard<std::mutex> lk(mu);
                err = "cudaEventSynchronize failed on the ingest ring";
                stopping = true;
                cv.notify_all();
                break;
            }
            const uint32_t file = ranges[ch.range].file;
            if (file != fd_file) {
                if (fd >= 0) ::close(fd);
                fd = ::open(paths[file], O_RDONLY);
                fd_file = file;
            }
            uint8_t* dst = ring + static_cast<uint64_t>(slot) * chunk;
            uint64_t got = 0;
            while (fd >= 0 && got < ch.len) {
                const ssize_t rd = ::pread(fd, dst + got, ch.len - got, static_cast<off_t>(ch.off + got));
                if (rd <= 0) break;
                got += static_cast<uint64_t>(rd);
            }
            std::lock_guard<std::mutex> lk(mu);
            if (got != ch.len) {
                err = std::string("Io: read failure on ") + paths[file];
                stopping = true;
            } else {
                ready[k] = 1;
            }
            cv.notify_all();
            if (stopping) break;
        }
        if (fd >= 0) ::close(fd);
    }
};

RingIngest::RingIngest(cvlg_context* c, const char* const* paths, std::vector<FileRange> ranges,
                       uint8_t* d_dst, unsigned n_threads)
    : impl_(new Impl) {
    Impl& I = *impl_;
    I.c = c;
    I.paths = paths;
    I.ranges = std::move(ranges);
    I.d_dst = d_dst;
    // ring geometry (CVLG_RING_MB / CVLG_RING_SLOTS override: tuning only)
    if (const char* e = std::getenv("CVLG_RING_MB")) I.chunk = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) << 20;
    if (const char* e = std::getenv("CVLG_RING_SLOTS")) I.slots = std::max(2, std::atoi(e));
    for (size_t i = 0; i < I.ranges.size(); ++i) {
        const FileRange& r = I.ranges[i];
        for (uint64_t a = 0; a < r.len; a += I.chunk)
            I.chunks.push_back(Impl::Chunk{i, r.off + a, std::min(I.chunk, r.len - a), r.dst + a});
    }
    const size_t n_chunks = I.chunks.size();
    I.slots = static_cast<int>(std::min<size_t>(I.slots, std::max<size_t>(n_chunks, 2)));
    c->h_ring.ensure(static_cast<uint64_t>(I.slots) * I.chunk);
    while (c->ring_events.size() < static_cast<size_t>(I.slots)) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ring_events.push_back(e);
    }
    I.ring = static_cast<uint8_t*>(c->h_ring.p);
    // the copies must not start before the previous run finished with the device buffer, and
    // no slot may be refilled before its last copy (from a previous run) completed
    cudaEvent_t start_ev = c->ring_events[0];
    CK(cudaEventRecord(start_ev, c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, start_ev, 0));
    for (int k = 0; k < I.slots; ++k) CK(cudaEventRecord(c->ring_events[k], c->copy_stream));
    I.ready.assign(n_chunks, 0);
    // readers: at most 5/8 of the host threads (the caller's thread feeds the copy engine and
    // the decode; 16 readers on 16 cores measured 20-25% slower than 8-12)
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned workers = std::min(n_threads ? n_threads : hw, std::max(2u, hw * 5 / 8));
    if (const char* e = std::getenv("CVLG_RING_READERS")) workers = std::max(1, std::atoi(e));
    workers = static_cast<unsigned>(std::min<size_t>({workers, static_cast<size_t>(I.slots), std::max<size_t>(n_chunks, 1)}));
    for (unsigned w = 0; w < workers && n_chunks; ++w) I.pool.emplace_back([&I] { I.reader(); });
}

size_t RingIngest::chunks() const { return impl_->chunks.size(); }

bool RingIngest::next(RingChunk& out) {
    Impl& I = *impl_;
    if (I.k_next >= I.chunks.size()) return false;
    const size_t k = I.k_next++;
    {
        std::unique_lock<std::mutex> lk(I.mu);
        I.cv.wait(lk, [&] { return I.ready[k] || !I.err.empty(); });
        if (!I.err.empty()) fail(I.err.rfind("Io:", 0) == 0 ? CVLG_E_IO : CVLG_E_CUDA, I.err);
    }
    const Impl::Chunk& ch = I.chunks[k];
    const int slot = static_cast<int>(k % I.slots);
    const uint8_t* src = I.ring + static_cast<uint64_t>(slot) * I.chunk;
    CK(cudaMemcpyAsync(I.d_dst + ch.dst, src, ch.len, cudaMemcpyHostToDevice, I.c->copy_stream));
    CK(cudaEventRecord(I.c->ring_events[slot], I.c->copy_stream));
    // (before the slot is released for refilling)
    const void* nl = memrchr(src, '\n', ch.len);
    const uint64_t nl_end = nl ? static_cast<uint64_t>(static_cast<const uint8_t*>(nl) - src) + 1 : 0;
    {
        std::lock_guard<std::mutex> lk(I.mu);
        I.enqueued = k + 1;
        I.cv.notify_all();
    }
    out = RingChunk{ch.range, ch.off, ch.len, ch.dst, nl_end, I.c->ring_events[slot]};
    return true;
}

void RingIngest::stop() {
    Impl& I = *impl_;
    {
        std::lock_guard<std::mutex> lk(I.mu);
        I.stopping = true;
        I.cv.notify_all();
    }
    for (auto& t : I.pool)
        if (t.joinable()) t.join();
    I.pool.clear();
}

RingIngest::~RingIngest() {
    stop();
    cudaStreamSynchronize(impl_->c->copy_stream);
    delete impl_;
}

void export_tuples(cvlg_context* c, uint64_t* d_cell, uint64_t* d_key0, uint64_t* d_key1,
                   double* d_sum, uint64_t* d_count, uint64_t stride, cudaStream_t s,
                   const uint32_t* d_grank) {
    if (c->part_long_ids && !d_grank)
        fail(CVLG_E_UNSUPPORTED, "multi-GPU combine needs journey ids <= 15 bytes (exact inline keys)");
    const uint64_t n = c->part_pairs;
    if (!n) return;
    c->h_small.ensure(4096);
    uint32_t* d_bad = c->scal.as<uint32_t>() + 15;
    CK(cudaMemsetAsync(d_bad, 0, 4, s));
    launch_export_pairs(c->pair_key.as<uint64_t>(), c->pair_sum.as<double>(), c->pair_cnt.as<uint32_t>(),
                        n, c->part_rbits, c->rank_slot.as<uint32_t>(), c->dict.as<unsigned long long>(),
                        d_cell, d_key0, d_key1, d_sum, d_count, stride, d_grank, d_bad, s);
    uint32_t* hb = static_cast<uint32_t*>(c->h_small.p) + 200;
    CK(cudaMemcpyAsync(hb, d_bad, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (*hb) fail(CVLG_E_UNSUPPORTED, "multi-GPU combine needs journey ids <= 15 bytes (exact inline keys)");
}

void journey_ids(cvlg_context* c, std::vector<uint8_t>& blob, std::vector<uint64_t>& offs) {
    const uint64_t J = c->part_J;
    offs.assign(J + 1, 0);
    blob.clear();
    if (!J) return;
    cudaStream_t s = c->stream;
    c->flags.ensure(J * 4 + 16);
    c->pos.ensure(J * 4 + 16);
    c->scan_tmp.ensure(scan_temp_words(J) * 4 + 64);
    c->scal.ensure(128);
    uint32_t* d_total = c->scal.as<uint32_t>() + 30;
    launch_id_len(c->rank_slot.as<uint32_t>(), c->dict.as<unsigned long long>(), J, c->flags.as<uint32_t>(), s);
    exclusive_scan_u32(c->flags.as<uint32_t>(), c->pos.as<uint32_t>(), J, d_total, c->scan_tmp.as<uint32_t>(), s);
    uint32_t total = 0;
    CK(cudaMemcpyAsync(&total, d_total, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->x_keys.ensure(static_cast<uint64_t>(total) + 16);
    launch_id_copy(c->rank_slot.as<uint32_t>(), c->dict.as<unsigned long long>(), c->csv_in,
                   J, c->pos.as<uint32_t>(), c->x_keys.as<uint8_t>(), s);
    std::vector<uint32_t> pos(J);
    blob.resize(total);
    CK(cudaMemcpyAsync(pos.data(), c->pos.p, J * 4, cudaMemcpyDeviceToHost, s));
    if (total) CK(cudaMemcpyAsync(blob.data(), c->x_keys.p, total, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    for (uint64_t r = 0; r < J; ++r) offs[r] = pos[r];
    offs[J] = total;
}

void finalize_tuples(cvlg_context* c, const uint64_t* d_cell, const uint64_t* d_key0,
                     const uint64_t* d_key1, const double* d_sum, const uint64_t* d_count,
                     uint64_t stride, uint64_t n, const Dims& dims, uint32_t t0, uint32_t t1,
                     uint32_t* d_planes, uint32_t* d_raw, cudaStream_t s) {
    const uint64_t lattice_words = static_cast<uint64_t>(t1 - t0) * 8 * dims.RC;
    const uint64_t raw_words = static_cast<uint64_t>(t1 - t0) * 4 * dims.RC;
    CK(cudaMemsetAsync(d_planes, 0, lattice_words * 4, s));
    if (d_raw) CK(cudaMemsetAsync(d_raw, 0, raw_words * 4, s));
    if (n) {
        if (n >= (1ull << 32)) fail(CVLG_E_UNSUPPORTED, ">= 2^32 (cell, journey) tuples on one device");
        c->h_small.ensure(4096);
        c->scal.ensure(128);
        unsigned long long* d_orand = c->scal.as<unsigned long long>() + 4;
        unsigned long long* h_orand = reinterpret_cast<unsigned long long*>(h_small64(c) + 40);
        c->x_keys.ensure(n * 8);
        c->keys_alt.ensure(n * 8);
        c->vals.ensure(n * 4);
        c->vals_alt.ensure(n * 4);
        c->sort_tmp.ensure(radix_temp_bytes(n));
        c->x_sum.ensure(n * 8);
        c->x_cnt.ensure(n * 4);
        uint64_t* keys = c->x_keys.as<uint64_t>();
        uint32_t* vals = c->vals.as<uint32_t>();
        // stable LSD over (cell, key0, key1): least significant word first; (cell, key) is unique,
        // so the order is the reference's (g, journey) finalize order (aggregate.cpp:161-204)
        launch_gather_u64(d_key1, stride, nullptr, n, keys, s);
        launch_pair_vals(vals, n, s);
        radix_sort_pairs(keys, vals, c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), n, 0, 64,
                         c->sort_tmp.p, s, d_orand, h_orand);
        launch_gather_u64(d_key0, stride, vals, n, keys, s);
        radix_sort_pairs(keys, vals, c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), n, 0, 64,
                         c->sort_tmp.p, s, d_orand, h_orand);
        launch_gather_u64(d_cell, stride, vals, n, keys, s);
        radix_sort_pairs(keys, vals, c->keys_alt.as<uint64_t>(), c->vals_alt.as<uint32_t>(), n, 0,
                         bits_for(dims.cells - 1), c->sort_tmp.p, s, d_orand, h_orand);
        launch_import_pairs(d_sum, d_count, stride, n, c->x_sum.as<double>(), c->x_cnt.as<uint32_t>(), s);
        launch_finalize(keys, vals, n, 0, c->x_sum.as<double>(), c->x_cnt.as<uint32_t>(), dims.D, dims.RC,
                        t0, t1 - t0, d_planes, d_raw, s);
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
}

int guard(const std::function<void()>& fn) {
    try {
        fn();
        return CVLG_OK;
    } catch (const Error& e) {
        t_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        t_last_error = "host allocation failed";
        return CVLG_E_CUDA;
    } catch (const std::exception& e) {
        t_last_error = e.what();
        return CVLG_E_INTERNAL;
    }
}

}  // namespace cvlg

using namespace cvlg;

// ==================================== C ABI =====================================================
extern "C" {

void cvlg_default_grid(cvlg_grid_spec* s) {
    if (!s) return;
    s->lat_min = 36.0;
    s->lat_max = 40.6;
    s->lon_min = -95.8;
    s->lon_max = -89.1;
    s->lat_step = 0.1;
    s->lon_step = 0.1;
    s->min_step = 5;
    s->dxn_step = 90;
    s->dxn_offset = 0.0;
}

void cvlg_default_rules(cvlg_filter_rules* r) {
    if (!r) return;
    r->require_in_grid = 1;
    r->drop_missing = 1;
    r->speed_ceiling = 250.0;
}

int cvlg_grid_dims(const cvlg_grid_spec* spec, uint32_t* T, uint32_t* D, uint32_t* R, uint32_t* C) {
    return guard([&] {
        const Dims d = validate_grid(spec);
        if (T) *T = d.T;
        if (D) *D = d.D;
        if (R) *R = d.R;
        if (C) *C = d.C;
    });
}

cvlg_context* cvlg_context_create(int device) {
    cvlg_context* c = nullptr;
    const int rc = guard([&] {
        int dev = device;
        if (dev < 0) CK(cudaGetDevice(&dev));
        CK(cudaSetDevice(dev));
        c = new cvlg_context();
        c->device = dev;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
        CK(cudaEventCreate(&c->ev_dec0));
        CK(cudaEventCreate(&c->ev_dec1));
    });
    if (rc != CVLG_OK) {
        delete c;
        return nullptr;
    }
    return c;
}

void cvlg_context_destroy(cvlg_context* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->copy_stream);
    DevBuf* bufs[] = {&c->csv,    &c->shard_off, &c->cmap,     &c->good,     &c->counter,
                      &c->stats,  &c->ts,
                      &c->hscr,   &c->hend,      &c->tiles,    &c->thpos,    &c->ts2,
                      &c->hid_scr, &c->hid, &c->hkey_scr, &c->hkey, &c->rec, &c->r_keys, &c->r_keys_alt, &c->r_perm, &c->r_perm_alt, &c->r_ts, &c->r_lat, &c->r_lon, &c->r_speed, &c->r_heading, &c->r_id, &c->r_arena, &c->r_postal, &c->r_parena, &c->run_j, &c->jo_keys, &c->jo_keys_alt, &c->jo_vals, &c->jo_vals_alt, &c->gkeys, &c->gkeys_alt, &c->gvals, &c->gvals_alt, &c->gpieces, &c->gruns, &c->gstart, &c->gj,      &c->runs,     &c->lat,      &c->lon,
                      &c->lat2,    &c->lon2,     &c->f_points, &c->f_tfirst, &c->f_tlast,
                      &c->f_len,   &c->f_step,   &c->f_vmax,   &c->f_acc,    &c->f_dwell,
                      &c->f_stops, &c->f_id,     &c->f_first,  &c->f_cmin,   &c->f_cmax,
                      &c->speed2, &c->code2,     &c->loff2,
                      &c->speed,  &c->code,      &c->loff,     &c->hslot,    &c->spill_key,
                      &c->spill_sum, &c->spill_cnt, &c->dict,     &c->hdict,
                      &c->flags,  &c->pos,       &c->uslot,    &c->rank_of_slot, &c->hrank,
                      &c->scal,   &c->keys,      &c->vals,     &c->keys_alt, &c->vals_alt,
                      &c->sort_tmp, &c->scan_tmp, &c->srank,   &c->jstart,   &c->pair_key,
                      &c->pair_sum, &c->pair_cnt, &c->planes,  &c->raw, &c->rank_slot,
                      &c->x_keys, &c->x_sum, &c->x_cnt, &c->fold_dir, &c->dead,
                      &c->slice, &c->r_tbytes, &c->r_tbase, &c->r_pobase, &c->r_total, &c->r_lines,
                      &c->r_idcol, &c->r_poff, &c->r_tfirst, &c->r_hdr, &c->r_hoff, &c->r_dst,
                      &c->r_err, &c->r_send, &c->tuples, &c->tuples_in, &c->tuples_send,
                      &c->t_counts, &c->t_dst};
    for (DevBuf* b : bufs) b->release();
    c->h_small.release();
    c->h_ring.release();
    for (auto e : c->ring_events) cudaEventDestroy(e);
    for (auto e : c->chunk_events) cudaEventDestroy(e);
    for (auto e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_dec0) cudaEventDestroy(c->ev_dec0);
    if (c->ev_dec1) cudaEventDestroy(c->ev_dec1);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->copy_stream);
    delete c;
}

int cvlg_run_pipeline(cvlg_context* ctx, const char* const* shard_paths, size_t n_shards,
                      const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                      uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                      uint32_t* raw_count, cvlg_stats* stats) {
    return guard([&] {
        validate_grid(spec);
        if (n_partitions == 0) fail(CVLG_E_ZERO_PARTITIONS, "ZeroPartitions: n_partitions must be >= 1");
        if (n_shards && !shard_paths) fail(CVLG_E_INVALID_ARG, "shard_paths is NULL");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        // lexicographic rank of paths (aggregate.cpp:389-397)
        std::vector<size_t> order(n_shards);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            return std::strcmp(shard_paths[a], shard_paths[b]) < 0;
        });
        std::vector<const char*> ranked(n_shards);
        for (size_t r = 0; r < n_shards; ++r) ranked[r] = shard_paths[order[r]];
        run_files(c, ranked.data(), n_shards, spec, rules, n_threads, planes, raw_count, stats);
    });
}

int cvlg_run_pipeline_host(cvlg_context* ctx, const uint8_t* const* shard_bufs,
                           const uint64_t* shard_lens, size_t n_shards,
                           const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                           uint32_t n_partitions, uint32_t* planes, uint32_t* raw_count,
                           cvlg_stats* stats) {
    return guard([&] {
        validate_grid(spec);
        if (n_partitions == 0) fail(CVLG_E_ZERO_PARTITIONS, "ZeroPartitions: n_partitions must be >= 1");
        if (n_shards && (!shard_bufs || !shard_lens)) fail(CVLG_E_INVALID_ARG, "NULL shard arrays");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        run_host(c, shard_bufs, shard_lens, n_shards, spec, rules, planes, raw_count, stats);
    });
}

int cvlg_run_pipeline_records(cvlg_context* ctx, const cvlg_record* records, size_t n,
                              const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                              uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                              uint32_t* raw_count, cvlg_stats* stats) {
    (void)n_threads;
    return guard([&] {
        validate_grid(spec);
        if (n_partitions == 0) fail(CVLG_E_ZERO_PARTITIONS, "ZeroPartitions: n_partitions must be >= 1");
        if (n && !records) fail(CVLG_E_INVALID_ARG, "NULL records");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        run_records(c, records, n, spec, rules, planes, raw_count, stats);
    });
}

int cvlg_run_pipeline_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                             size_t n_shards, const cvlg_grid_spec* spec,
                             const cvlg_filter_rules* rules, uint32_t* d_planes,
                             uint32_t* d_raw_count, cvlg_stats* stats, void* stream) {
    return guard([&] {
        validate_grid(spec);
        if (!shard_offsets || !d_planes) fail(CVLG_E_INVALID_ARG, "NULL argument");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        std::vector<uint64_t> off(shard_offsets, shard_offsets + n_shards + 1);
        if (off[0] != 0) fail(CVLG_E_INVALID_ARG, "shard_offsets[0] must be 0");
        for (size_t i = 0; i < n_shards; ++i)
            if (off[i + 1] < off[i]) fail(CVLG_E_INVALID_ARG, "shard_offsets must be non-decreasing");
        cudaStream_t saved = c->stream;
        if (stream) c->stream = static_cast<cudaStream_t>(stream);
        try {
            run_core(c, d_csv, off, nullptr, nullptr, 0, spec, rules, d_planes, d_raw_count, stats,
                     marks_of({ChunkMark{off.back(), off.back(), nullptr}}));
        } catch (...) {
            c->stream = saved;
            throw;
        }
        c->stream = saved;
    });
}

int cvlg_journey_features_host(cvlg_context* ctx, const uint8_t* const* shard_bufs,
                               const uint64_t* shard_lens, size_t n_shards, const cvlg_grid_spec* spec,
                               const cvlg_filter_rules* rules, double stop_speed, uint32_t* planes,
                               uint32_t* raw_count, cvlg_stats* stats, uint64_t* n_journeys) {
    return guard([&] {
        validate_grid(spec);
        if (n_shards && (!shard_bufs || !shard_lens)) fail(CVLG_E_INVALID_ARG, "NULL shard arrays");
        if (!(stop_speed == stop_speed)) fail(CVLG_E_INVALID_ARG, "stop_speed is NaN");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        run_host(c, shard_bufs, shard_lens, n_shards, spec, rules, planes, raw_count, stats, &stop_speed);
        if (n_journeys) *n_journeys = c->f_J;
    });
}

int cvlg_journey_features_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                                 size_t n_shards, const cvlg_grid_spec* spec,
                                 const cvlg_filter_rules* rules, double stop_speed, uint32_t* d_planes,
                                 uint32_t* d_raw_count, cvlg_stats* stats, uint64_t* n_journeys,
                                 void* stream) {
    return guard([&] {
        validate_grid(spec);
        if (!shard_offsets || !d_planes) fail(CVLG_E_INVALID_ARG, "NULL argument");
        if (!(stop_speed == stop_speed)) fail(CVLG_E_INVALID_ARG, "stop_speed is NaN");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        std::vector<uint64_t> off(shard_offsets, shard_offsets + n_shards + 1);
        if (off[0] != 0) fail(CVLG_E_INVALID_ARG, "shard_offsets[0] must be 0");
        for (size_t i = 0; i < n_shards; ++i)
            if (off[i + 1] < off[i]) fail(CVLG_E_INVALID_ARG, "shard_offsets must be non-decreasing");
        cudaStream_t saved = c->stream;
        if (stream) c->stream = static_cast<cudaStream_t>(stream);
        try {
            run_core(c, d_csv, off, nullptr, nullptr, 0, spec, rules, d_planes, d_raw_count, stats,
                     marks_of({ChunkMark{off.back(), off.back(), nullptr}}), false, &stop_speed);
        } catch (...) {
            c->stream = saved;
            throw;
        }
        c->stream = saved;
        if (n_journeys) *n_journeys = c->f_J;
    });
}

int cvlg_features_copy(cvlg_context* ctx, cvlg_features* out) {
    return guard([&] {
        if (!out) fail(CVLG_E_INVALID_ARG, "NULL argument");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        const uint64_t J = c->f_J;
        out->n_journeys = J;
        auto cp = [&](void* dst, const DevBuf& src, uint64_t bytes) {
            if (dst && bytes) CK(cudaMemcpy(dst, src.p, bytes, cudaMemcpyDeviceToHost));
        };
        cp(out->points, c->f_points, J * 4);
        cp(out->t_first, c->f_tfirst, J * 8);
        cp(out->t_last, c->f_tlast, J * 8);
        cp(out->length_m, c->f_len, J * 8);
        cp(out->max_step_m, c->f_step, J * 8);
        cp(out->max_speed, c->f_vmax, J * 8);
        cp(out->max_abs_accel, c->f_acc, J * 8);
        cp(out->dwell_s, c->f_dwell, J * 8);
        cp(out->stops, c->f_stops, J * 4);
        cp(out->id_span, c->f_id, J * 8);
        cp(out->cell_speed_min, c->f_cmin, c->f_cells * 4);
        cp(out->cell_speed_max, c->f_cmax, c->f_cells * 4);
    });
}

int cvlg_partial_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                        size_t n_shards, const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                        uint64_t* n_pairs, cvlg_stats* stats, void* stream) {
    return guard([&] {
        validate_grid(spec);
        if (!shard_offsets || !n_pairs) fail(CVLG_E_INVALID_ARG, "NULL argument");
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        std::vector<uint64_t> off(shard_offsets, shard_offsets + n_shards + 1);
        if (off[0] != 0) fail(CVLG_E_INVALID_ARG, "shard_offsets[0] must be 0");
        cudaStream_t saved = c->stream;
        if (stream) c->stream = static_cast<cudaStream_t>(stream);
        try {
            run_core(c, d_csv, off, nullptr, nullptr, 0, spec, rules, nullptr, nullptr, stats,
                     marks_of({ChunkMark{off.back(), off.back(), nullptr}}), true);
        } catch (...) {
            c->stream = saved;
            throw;
        }
        c->stream = saved;
        *n_pairs = c->part_pairs;
    });
}

int cvlg_export_pairs(cvlg_context* ctx, uint64_t* d_cell, uint64_t* d_key0, uint64_t* d_key1,
                      double* d_sum, uint64_t* d_count, void* stream) {
    return guard([&] {
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        if (c->part_pairs && (!d_cell || !d_key0 || !d_key1 || !d_sum || !d_count))
            fail(CVLG_E_INVALID_ARG, "NULL argument");
        export_tuples(c, d_cell, d_key0, d_key1, d_sum, d_count, 1,
                      stream ? static_cast<cudaStream_t>(stream) : c->stream, nullptr);
    });
}

int cvlg_finalize_pairs(cvlg_context* ctx, const uint64_t* d_cell, const uint64_t* d_key0,
                        const uint64_t* d_key1, const double* d_sum, const uint64_t* d_count,
                        uint64_t n, const cvlg_grid_spec* spec, uint32_t* d_planes,
                        uint32_t* d_raw_count, void* stream) {
    return guard([&] {
        const Dims dims = validate_grid(spec);
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        if (!d_planes) fail(CVLG_E_INVALID_ARG, "NULL planes");
        CK(cudaSetDevice(c->device));
        finalize_tuples(c, d_cell, d_key0, d_key1, d_sum, d_count, 1, n, dims, 0, dims.T, d_planes,
                        d_raw_count, stream ? static_cast<cudaStream_t>(stream) : c->stream);
    });
}

int cvlg_debug_slots(cvlg_context* ctx, int64_t* ts, double* speed, uint32_t* code, uint64_t* loff,
                     uint64_t cap, uint64_t* n) {
    return guard([&] {
        cvlg_context* c = ctx ? ctx : default_context();
        if (!c) fail(CVLG_E_CUDA, "no CUDA context");
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        if (c->last_slots) {  // dense (full-sort path): slots 0..NS-1 in provenance order
            const uint64_t m = std::min<uint64_t>(cap, c->last_slots);
            if (n) *n = c->last_slots;
            if (!m) return;
            if (ts) CK(cudaMemcpy(ts, c->ts.p, m * 8, cudaMemcpyDeviceToHost));
            if (speed) CK(cudaMemcpy(speed, c->speed.p, m * 8, cudaMemcpyDeviceToHost));
            if (code) CK(cudaMemcpy(code, c->code.p, m * 4, cudaMemcpyDeviceToHost));
            if (loff) CK(cudaMemcpy(loff, c->loff.p, m * 8, cudaMemcpyDeviceToHost));
            return;
        }
        // sparse (run-merge path): tile t's lines are slots [tiles[t].x, + tiles[t].y)
        if (n) *n = c->dbg_lines;
        if (!cap || !c->dbg_tiles) return;
        std::vector<uint4> tiles(c->dbg_tiles);
        CK(cudaMemcpy(tiles.data(), c->tiles.p, c->dbg_tiles * 16, cudaMemcpyDeviceToHost));
        uint64_t at = 0;
        for (const uint4& t : tiles) {
            const uint64_t k = std::min<uint64_t>(t.y, cap > at ? cap - at : 0);
            if (!k) continue;
            if (ts) CK(cudaMemcpy(ts + at, c->ts.as<int64_t>() + t.x, k * 8, cudaMemcpyDeviceToHost));
            if (speed) CK(cudaMemcpy(speed + at, c->speed.as<double>() + t.x, k * 8, cudaMemcpyDeviceToHost));
            if (code) CK(cudaMemcpy(code + at, c->code.as<uint32_t>() + t.x, k * 4, cudaMemcpyDeviceToHost));
            if (loff) CK(cudaMemcpy(loff + at, c->loff.as<uint64_t>() + t.x, k * 8, cudaMemcpyDeviceToHost));
            at += k;
        }
    });
}

int cvlg_write_container(const uint32_t* planes, const cvlg_grid_spec* spec, int32_t day,
                         const char* path, uint64_t* bytes_written) {
    return guard([&] {
        const Dims d = validate_grid(spec);
        if (!planes || !path) fail(CVLG_E_INVALID_ARG, "NULL argument");
        // NonFiniteValue check (lattice_store.cpp:92-95)
        const uint64_t rc = d.RC;
        for (uint32_t t = 0; t < d.T; ++t)
            for (uint64_t i = 0; i < 4 * rc; ++i) {
                const uint32_t u = planes[(static_cast<uint64_t>(t) * 8) * rc + i];
                if ((u & 0x7F800000u) == 0x7F800000u)
                    fail(CVLG_E_NON_FINITE_VALUE,
                         "NonFiniteValue: NaN/Inf in speed plane of batch " + std::to_string(t));
            }
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) fail(CVLG_E_IO, std::string("Io: cannot open ") + path + " for writing");
        uint8_t h[58];
        size_t k = 0;
        auto put = [&](const void* p, size_t n) {
            std::memcpy(h + k, p, n);  // x86-64 / aarch64 hosts are little-endian
            k += n;
        };
        const char magic[4] = {'C', 'V', 'L', '1'};
        const uint16_t version = 1;
        const uint16_t ms = static_cast<uint16_t>(spec->min_step), ds = static_cast<uint16_t>(spec->dxn_step);
        put(magic, 4);
        put(&version, 2);
        put(&spec->lat_min, 8);
        put(&spec->lat_step, 8);
        put(&spec->lon_min, 8);
        put(&spec->lon_step, 8);
        put(&d.R, 4);
        put(&d.C, 4);
        put(&ms, 2);
        put(&ds, 2);
        put(&d.T, 4);
        put(&day, 4);
        out.write(reinterpret_cast<const char*>(h), 58);
        uint64_t written = 58;
        for (uint32_t t = 0; t < d.T; ++t) {
            out.write(reinterpret_cast<const char*>(&t), 4);
            out.write(reinterpret_cast<const char*>(planes + static_cast<uint64_t>(t) * 8 * rc),
                      static_cast<std::streamsize>(8 * rc * 4));
            written += 4 + 8 * rc * 4;
        }
        out.flush();
        if (!out) fail(CVLG_E_IO, std::string("Io: short write to ") + path);
        if (bytes_written) *bytes_written = written;
    });
}

int cvlg_context_input(cvlg_context* ctx, const uint8_t** d_csv, uint64_t* n_bytes) {
    if (!ctx || !d_csv || !n_bytes) return CVLG_E_INVALID_ARG;
    *d_csv = ctx->csv.as<uint8_t>();
    *n_bytes = ctx->input_bytes;
    return CVLG_OK;
}

int cvlg_last_stage_ms(cvlg_context* ctx, float* ms, int n) {
    if (!ctx || !ms) return CVLG_E_INVALID_ARG;
    for (int i = 0; i < n && i < 6; ++i) ms[i] = ctx->stage_ms[i];
    return CVLG_OK;
}

int cvlg_pin_host(void* ptr, size_t bytes) {
    return guard([&] { CK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault)); });
}

int cvlg_unpin_host(void* ptr) {
    return guard([&] { CK(cudaHostUnregister(ptr)); });
}

uint64_t cvlg_launch_count(void) { return launch_count(); }

int cvlg_last_error(char* buf, size_t len) {
    if (!buf || !len) return CVLG_E_INVALID_ARG;
    std::strncpy(buf, t_last_error.c_str(), len - 1);
    buf[len - 1] = 0;
    return CVLG_OK;
}

}  // extern "C"
