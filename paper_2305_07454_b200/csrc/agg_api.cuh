// Host-side launchers for aggregate.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kernels.cuh"

namespace cvlg {

struct DictParams {
    const uint8_t* csv;
    const uint64_t* shard_off;
    const ColumnMap* cmap;
    uint32_t n_shards;
    uint64_t csv_len;
    const uint64_t* hid;  // [head] id byte offset | length << 40 (from K1)
    const ulonglong2* hkey;  // [head] inline key from K1 (.y == kNoKey: derive from the CSV)
    uint64_t n_heads;
    unsigned long long* table;  // [2 * (mask + 1)]
    uint64_t mask;
    uint32_t* hdict;
    unsigned long long* max_len;
    uint32_t* full;  // set when a probe chain exceeds its bound (host re-runs with more room)
};

constexpr int kFoldThreads = 128;  // fold CTA size (4 warps, one journey per lane)

struct FoldParams {
    // journeys: [jstart[j], jstart[j+1]) indexes `perm`
    uint64_t n_journeys;
    const uint32_t* jstart;
    const uint32_t* perm;   // fast path: sorted run heads; slow path: sorted slots
    const uint32_t* hslot;  // fast path: run start slots
    const uint32_t* hend;   // fast path: run end slots (exclusive)
    const uint2* runs;      // fast path scratch [H]: (start, end) of the runs in perm order
    uint64_t n_heads;
    const int64_t* ts;
    const double* speed;
    const uint32_t* code;
    const ulonglong2* rec;  // slow path (nullable): (speed bits, code) per dense slot, one gather
    const uint64_t* loff;
    // slow path: the sorted (rank << span | ts - lo) keys, aligned with perm (nullable): equal keys
    // within a journey = equal timestamps, read in order instead of gathering ts per slot
    const uint64_t* skey;
    // (cell, journey) subtotals out: key = cell << rank_bits | rank
    uint64_t* pair_key;
    double* pair_sum;
    uint32_t* pair_cnt;
    uint32_t* pair_count;
    uint64_t pair_cap;
    int rank_bits;
    // bin-group mode (few long journeys): the fold's work items are (journey, time bin) groups of
    // run pieces instead of journeys; jrank[g] is the journey rank of group g (nullable: off)
    const uint32_t* jrank;
    const uint32_t* jorder;     // nullable: work items in this order (longest first)
    int runs_ready;             // runs[] already built (bin-group mode): skip run_list_kernel
    uint64_t* journey_counter;  // dynamic journey assignment (zeroed before the fold)
    // (cell, journey) table, key = cell << 32 | rank
    uint64_t* spill_key;
    double* spill_sum;
    uint32_t* spill_cnt;
    uint64_t spill_mask;
    // time-bin windows (0 = off): a (cell, journey) subtotal can only be revisited in a window of
    // the same time bin, so closed windows go straight to the pair list; a later window of an
    // already-closed bin (another day) reloads that bin's block through the per-lane directory
    int win;
    uint32_t drc;             // cells per time bin (D * R * C)
    uint32_t n_bins;          // T
    uint32_t epoch;           // directory tag of this launch (>= 1)
    uint4* dir;               // [lanes][T]: (journey, epoch, pair base, count)
    uint32_t* dead_list;      // pair slots vacated by reloads
    uint32_t* dead_count;
    uint32_t* abort_flag;     // set by a failed spill insert: every warp stops (the host re-runs)
    uint32_t flush_slack;     // chunk-end flush of closed windows once n_cells + slack >= table size
    // records entry point (nullable): payload columns by record index (loff = record index), so
    // the conflict test compares records instead of re-parsing lines
    const double* r_lat;
    const double* r_lon;
    const double* r_speed;
    const double* r_heading;
    const uint64_t* r_postal;
    const uint8_t* r_postal_arena;
    // conflict re-parse
    const uint8_t* csv;
    const uint64_t* shard_off;
    const ColumnMap* cmap;
    uint32_t n_shards;
    uint64_t* stats;
};

// per-journey features (features.cu)
struct FeatureParams {
    uint64_t n_journeys;
    const uint32_t* jstart;
    const uint32_t* perm;  // slow path: sorted dense slots
    const uint2* runs;     // fast path: (start, end) runs in perm order
    int slow;
    const int64_t* ts;
    const double* speed;
    const double* lat;
    const double* lon;
    const uint32_t* code;
    double stop_speed;
    uint64_t D, RC;
    uint32_t* points;
    int64_t* t_first;
    int64_t* t_last;
    double* length_m;
    double* max_step_m;
    double* max_speed;
    double* max_abs_accel;
    double* dwell_s;
    uint32_t* stops;
    uint32_t* cell_min;  // f32 bits [T][4][R][C] (nullable)
    uint32_t* cell_max;
};
void launch_journey_features(const FeatureParams& f, const uint32_t* hrank, uint64_t n_heads,
                             const uint64_t* hid, uint32_t* first_scratch, uint64_t* id_span,
                             uint64_t n_cells_planes, cudaStream_t s);

struct DensifyParams {
    const uint4* tiles;
    uint64_t n_tiles;
    const uint32_t* lpos;  // exclusive scan of tile lines
    const uint32_t* hpos;  // exclusive scan of tile heads
    const uint32_t* hscr;  // K1's per-tile head lists
    const int64_t* ts;
    const double* speed;
    const uint32_t* code;
    const uint64_t* loff;
    const double* lat;  // nullable (features only)
    const double* lon;
    double* lat_out;
    double* lon_out;
    int64_t* ts_out;
    double* speed_out;
    uint32_t* code_out;
    uint64_t* loff_out;
    ulonglong2* rec_out;  // nullable: (speed bits, code) interleaved for the slow fold's gathers
    long long* ts_mm;     // nullable: min / max epoch over non-rejected slots (init LLONG_MAX / MIN)
    uint32_t* hslot_out;
};

void launch_tile_field(const uint4* tiles, uint64_t n, int field, uint32_t* out, cudaStream_t s);
void launch_heads_compact(const uint4* tiles, uint64_t n, const uint32_t* hpos, const uint32_t* hscr,
                          const uint64_t* hid_scr, const ulonglong2* hkey_scr, uint32_t* hslot,
                          uint32_t* hend, uint64_t* hid, ulonglong2* hkey, cudaStream_t s,
                          const DictParams* dict = nullptr);
void launch_densify(const DensifyParams& d, cudaStream_t s);
void launch_ts_range(const int64_t* ts, const uint32_t* code, uint64_t n, long long* mm, cudaStream_t s);
void launch_dict_insert(const DictParams& d, cudaStream_t s);
void launch_journey_len_keys(const uint32_t* jstart, uint64_t n, const uint2* runs, int runs_mode,
                             uint64_t* keys, uint32_t* vals, cudaStream_t s);
// bin-group mode: runs (perm order) -> pieces split at time-bin changes, keyed (journey, bin,
// stream order); after sorting the keys, groups of equal (journey, bin)
void launch_run_list(const uint32_t* perm, const uint32_t* hslot, const uint32_t* hend, uint64_t n,
                     uint2* runs, cudaStream_t s);
void launch_bin_pieces(const uint2* runs, uint64_t n_runs, const uint32_t* jstart, uint64_t J,
                       uint32_t* run_j, const uint32_t* code, uint32_t drc, int bin_bits, int run_bits,
                       uint64_t* keys, uint32_t* vals, uint2* pieces, uint32_t* counter,
                       uint64_t cap, cudaStream_t s);
void launch_bin_groups(const uint64_t* keys, const uint32_t* vals, const uint2* pieces, uint64_t n,
                       int order_bits, int bin_bits, uint32_t* flags, uint2* runs_out, cudaStream_t s);
void launch_bin_group_starts(const uint64_t* keys, const uint32_t* flags, const uint32_t* pos,
                             uint64_t n, int order_bits, int bin_bits, uint32_t* gstart,
                             uint32_t* gj, cudaStream_t s);
void launch_dict_flags(const unsigned long long* table, uint64_t cap, uint32_t* flags,
                       cudaStream_t s);
void launch_dict_compact(const uint32_t* flags, const uint32_t* pos, uint64_t cap, uint32_t* uslot,
                         cudaStream_t s);
void launch_dict_chunk(const unsigned long long* table, const uint32_t* uslot, const uint32_t* perm,
                       uint64_t n, int c, const uint8_t* csv, uint64_t* keys, cudaStream_t s);
void launch_dict_rank(const uint32_t* uslot, const uint32_t* perm, uint64_t n,
                      uint32_t* rank_of_slot, cudaStream_t s);
void launch_head_rank(const uint32_t* hdict, const uint32_t* rank_of_slot, uint64_t n,
                      uint32_t* hrank, cudaStream_t s);
void launch_head_keys(const uint32_t* hrank, const uint32_t* hslot, const int64_t* ts,
                      uint64_t n_heads, int64_t ts_min, int tsbits, int mode, uint64_t* keys,
                      uint32_t* vals, cudaStream_t s);
void launch_gather_rank_keys(const uint32_t* rank_src, const uint32_t* vals, uint64_t n,
                             uint64_t* keys, cudaStream_t s);
void launch_head_order_check(const uint32_t* perm, const uint32_t* hrank, const uint32_t* hslot,
                             const uint32_t* hend, const int64_t* ts, const uint32_t* code,
                             uint64_t n_heads, uint32_t* jstart, uint32_t* invalid, cudaStream_t s);
void launch_slot_keys(const uint32_t* hslot, const uint32_t* hrank, const uint32_t* hdict,
                      const uint32_t* rank_of_slot, uint64_t n_heads,
                      const int64_t* ts, const uint32_t* code, uint64_t n_slots, int64_t ts_min,
                      int tsbits, int mode, uint32_t reject_rank, uint64_t* keys, uint32_t* vals,
                      uint32_t* srank, cudaStream_t s);
// (sorted keys hold the journey rank at bit rank_shift and up; the reject rank sorts last)
void launch_slot_jstart(const uint64_t* keys, int rank_shift, uint64_t n, uint32_t* jstart,
                        cudaStream_t s);
void launch_fold(const FoldParams& p, bool slow, cudaStream_t s);
// CTAs of the (persistent) fold launch: the directory holds one row per lane of this grid
unsigned fold_grid(uint64_t n_journeys, bool slow);
// moves the live pairs of [0, n) over the `dead` vacated slots: the first n - dead stay live
void launch_pair_compact(uint64_t* key, double* sum, uint32_t* cnt, uint64_t n, uint64_t dead,
                         const uint32_t* dead_list, uint32_t* src_list, uint32_t* counters,
                         cudaStream_t s);
void launch_pair_vals(uint32_t* vals, uint64_t n, cudaStream_t s);
void launch_rank_slot(const uint32_t* uslot, const uint32_t* perm, uint64_t n, uint32_t* rank_slot,
                      cudaStream_t s);
void launch_export_pairs(const uint64_t* pkey, const double* psum, const uint32_t* pcnt, uint64_t n,
                         int rbits, const uint32_t* rank_slot, const unsigned long long* table,
                         uint64_t* cell, uint64_t* k0, uint64_t* k1, double* sum, uint64_t* cnt,
                         uint64_t stride, const uint32_t* grank, uint32_t* bad, cudaStream_t s);
// journey ids by local rank: lengths, then the bytes at pos[r] (exclusive scan of the lengths)
void launch_id_len(const uint32_t* rank_slot, const unsigned long long* table, uint64_t n,
                   uint32_t* len, cudaStream_t s);
void launch_id_copy(const uint32_t* rank_slot, const unsigned long long* table, const uint8_t* csv,
                    uint64_t n, const uint32_t* pos, uint8_t* blob, cudaStream_t s);
// dst[i] = src[(idx ? idx[i] : i) * stride]  (stride in u64 words: 1 = SoA column, 5 = PairTuple)
void launch_gather_u64(const uint64_t* src, uint64_t stride, const uint32_t* idx, uint64_t n,
                       uint64_t* dst, cudaStream_t s);
void launch_import_pairs(const double* sum, const uint64_t* cnt, uint64_t stride, uint64_t n,
                         double* psum, uint32_t* pcnt, cudaStream_t s);
void launch_finalize(const uint64_t* keys, const uint32_t* vals, uint64_t n, int rank_bits,
                     const double* pair_sum, const uint32_t* pair_cnt, uint32_t D, uint64_t RC,
                     uint32_t t_base, uint32_t t_rows, uint32_t* planes, uint32_t* raw,
                     cudaStream_t s);

}  // namespace cvlg
