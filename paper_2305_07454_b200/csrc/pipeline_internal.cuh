// Host-side internals shared by the single-GPU pipeline (pipeline.cu) and the multi-GPU driver
// (multi.cu): error plumbing, grow-only device/pinned buffers, the per-device context, the pinned
// ingest ring and the pipeline core.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <vector>

#include "../../include/cvlg.h"
#include "kernels.cuh"
#include "parse.cuh"

namespace cvlg {

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define CK(x) ::cvlg::cuda_check((x), #x)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    bool ensure(size_t bytes);  // true when (re)allocated: contents undefined
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void release();
};

struct HostPinned {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes);
    void release();
};

int bits_for(uint64_t v);          // bits needed to represent values 0..v
uint64_t pow2_at_least(uint64_t v);

struct Dims {
    uint32_t T, D, R, C;
    uint64_t RC, cells;
};
Dims validate_grid(const cvlg_grid_spec* s);  // GridSpec::validate (grid.cpp:47-57) + dims

// A chunk of CSV bytes that became resident: decode every tile whose lines are complete.
struct ChunkMark {
    uint64_t avail_end;  // bytes [0, avail_end) resident
    uint64_t safe_end;   // every line starting before safe_end ends before it
    cudaEvent_t ready;   // recorded on the copy stream (nullptr: already resident)
};
// Yields the marks of a run in order (blocking until the next chunk's copy is enqueued); false
// once the input is complete. The last mark yielded covers every byte.
using MarkSource = std::function<bool(ChunkMark&)>;
MarkSource marks_of(std::vector<ChunkMark> v);

// Header line of each shard file (read_shard, ingest.cpp:203-221): column map, validity, the
// header bytes (through its '\n') and the offset of the first data byte.
struct ShardHead {
    uint64_t len = 0;         // file size
    uint64_t data_begin = 0;  // first byte after the header line (== len: no data lines)
    ColumnMap cmap{};
    bool good = false;        // non-empty with a complete header
    bool bad_header = false;  // non-empty with an unusable header (BadHeader rejection)
    std::string header;       // header line bytes including its '\n' (empty if none)
};
std::vector<ShardHead> read_shard_heads(const char* const* paths, size_t n);

}  // namespace cvlg

struct cvlg_context {
    int device = 0;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    bool own_stream = true;
    cvlg::DevBuf csv, shard_off, cmap, good, counter, stats;
    cvlg::DevBuf ts, speed, code, loff, hslot, hscr, hend, tiles, thpos, hid_scr, hid, hkey_scr, hkey, rec, runs;
    cvlg::DevBuf run_j, gkeys, gkeys_alt, gvals, gvals_alt, gpieces, gruns, gstart, gj;  // fold bin groups
    cvlg::DevBuf jo_keys, jo_keys_alt, jo_vals, jo_vals_alt;  // fold work order (longest first)
    cvlg::DevBuf ts2, speed2, code2, loff2;  // dense copies for the slow (full-sort) path
    // per-journey features (cvlg_journey_features_*): lat/lon per slot, outputs per journey / cell
    cvlg::DevBuf lat, lon, lat2, lon2, f_points, f_tfirst, f_tlast, f_len, f_step, f_vmax, f_acc,
        f_dwell, f_stops, f_id, f_first, f_cmin, f_cmax;
    uint64_t f_J = 0, f_cells = 0;
    cvlg::DevBuf dict, hdict, flags, pos, uslot, rank_of_slot, hrank, scal;
    cvlg::DevBuf keys, vals, keys_alt, vals_alt, sort_tmp, scan_tmp, srank, jstart;
    cvlg::DevBuf pair_key, pair_sum, pair_cnt, spill_key, spill_sum, spill_cnt, fold_dir, dead;
    uint32_t fold_epoch = 0;
    bool slow_key_ts = false;
    cvlg::DevBuf planes, raw, rank_slot, x_keys, x_sum, x_cnt;
    // records entry point (cvlg_run_pipeline_records): columns by record index, provenance sort
    cvlg::DevBuf r_keys, r_keys_alt, r_perm, r_perm_alt, r_ts, r_lat, r_lon, r_speed, r_heading, r_id,
        r_arena, r_postal, r_parena;
    // multi-GPU data plane (multi.cu): this GPU's slice of the input, routing state, tuples
    cvlg::DevBuf slice, r_tbytes, r_tbase, r_pobase, r_total, r_lines, r_idcol, r_poff, r_tfirst,
        r_hdr, r_hoff, r_dst, r_err, r_send, tuples, tuples_in, tuples_send, t_counts, t_dst;
    std::vector<uint64_t> r_h_poff, r_h_hoff, r_h_pobase, r_h_total;  // host copies (routing plan)
    std::vector<uint32_t> r_h_tfirst;
    std::vector<cvlg::ColumnMap> r_h_cmap;  // column map of each piece's shard
    uint32_t r_owners = 0;
    uint64_t r_bad_headers = 0;
    uint64_t t_n = 0;                       // tuples exported by the last cvlg_tuples_export
    std::vector<uint64_t> t_h_counts;
    cvlg::HostPinned h_small, h_ring;
    std::vector<cudaEvent_t> ring_events;  // one per ring slot: its last H2D copy
    // last cvlg_partial_device run: pairs kept in pair_key/pair_sum/pair_cnt
    uint64_t part_pairs = 0, part_J = 0, last_slots = 0;
    uint64_t dbg_tiles = 0, dbg_lines = 0;  // decode geometry of the last run (cvlg_debug_slots)
    uint64_t input_bytes = 0;  // bytes of c->csv staged by the last host/file run
    const uint8_t* csv_in = nullptr;  // CSV bytes of the last run (long journey ids point into it)
    cvlg::DevBuf r_grank;             // global journey ranks (multi-GPU combine with long ids)
    int part_rbits = 0;
    bool part_long_ids = false;
    std::vector<cudaEvent_t> chunk_events;
    cudaEvent_t ev[6] = {};
    cudaEvent_t ev_dec0 = nullptr, ev_dec1 = nullptr;
    float stage_ms[6] = {0, 0, 0, 0, 0, 0};
};

namespace cvlg {

cvlg_context* default_context();
void sync(cvlg_context* c);
int guard(const std::function<void()>& fn);

// The pipeline proper over CSV bytes in HBM (see pipeline.cu). `partial` stops after the
// per-(cell, journey) subtotals (kept in the context for cvlg_export_pairs).
void run_core(cvlg_context* c, const uint8_t* d_csv, const std::vector<uint64_t>& shard_off,
              const ColumnMap* h_cmap, const uint8_t* h_good, uint64_t bad_headers,
              const cvlg_grid_spec* spec, const cvlg_filter_rules* rules, uint32_t* d_planes,
              uint32_t* d_raw, cvlg_stats* out_stats, const MarkSource& next_mark,
              bool partial = false, const double* feat_stop_speed = nullptr,
              const RecordsDecodeParams* records = nullptr);

// Per-(cell, journey) subtotals of the last partial run -> (cell, key0, key1, sum, count) with
// exact global journey keys (stride in u64 words between consecutive tuples' fields).
// With d_grank (device, one u32 per local journey rank: its rank in the global lexicographic
// order of all GPUs' ids) the key is (grank, 0) and ids of any length are supported.
void export_tuples(cvlg_context* c, uint64_t* d_cell, uint64_t* d_key0, uint64_t* d_key1,
                   double* d_sum, uint64_t* d_count, uint64_t stride, cudaStream_t s,
                   const uint32_t* d_grank);
// The last partial run's journey ids in local rank order (host): bytes of rank r are
// blob[offs[r], offs[r + 1]).
void journey_ids(cvlg_context* c, std::vector<uint8_t>& blob, std::vector<uint64_t>& offs);
// Global lexicographic ranks of the union of n sorted, pairwise disjoint id lists.
void merge_id_ranks(const std::vector<const std::vector<uint8_t>*>& blobs,
                    const std::vector<const std::vector<uint64_t>*>& offs,
                    std::vector<std::vector<uint32_t>>& ranks);
// Any union of such tuples -> rows [t0, t1) of the dense lattice (d_planes / d_raw hold only
// those rows; cells without tuples are zero, tuples of other rows are ignored), synchronous.
void finalize_tuples(cvlg_context* c, const uint64_t* d_cell, const uint64_t* d_key0,
                     const uint64_t* d_key1, const double* d_sum, const uint64_t* d_count,
                     uint64_t stride, uint64_t n, const Dims& dims, uint32_t t0, uint32_t t1,
                     uint32_t* d_planes, uint32_t* d_raw, cudaStream_t s);

// Byte ranges of files streamed into device memory through the context's bounded pinned ring:
// reader threads pread chunks into ring slots in any order, next() enqueues each chunk's H2D
// copy (copy stream) in order once it is complete, and a slot is refilled only after its copy
// finished. The destructor stops and joins the readers.
struct FileRange {
    uint32_t file;
    uint64_t off, len;  // bytes [off, off + len) of the file
    uint64_t dst;       // destination offset in the device buffer
};
struct RingChunk {
    size_t range;           // index into the ranges
    uint64_t off, len;      // file bytes of this chunk (within the range)
    uint64_t dst;           // destination offset
    uint64_t nl_end;        // 1 + position of the chunk's last '\n' (0: none), chunk-relative
    cudaEvent_t copied;     // recorded after its H2D copy
};
class RingIngest {
public:
    RingIngest(cvlg_context* c, const char* const* paths, std::vector<FileRange> ranges,
               uint8_t* d_dst, unsigned n_threads);
    ~RingIngest();
    bool next(RingChunk& out);  // false once every chunk has been enqueued
    size_t chunks() const;
    void stop();

private:
    struct Impl;
    Impl* impl_;
};

}  // namespace cvlg
