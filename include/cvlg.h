/* cvlg — C ABI of the B200 (sm_100a) connected-vehicle ETL pipeline.
 *
 * Drop-in boundary for the reference pipeline API
 *   std::vector<BatchFrame> cvl::run_pipeline(const SourceManifest&, const GridSpec&,
 *       const FilterRules&, uint32_t n_partitions, uint32_t n_threads, PipelineStats*)
 *   (reference: proj/include/cvl/aggregate.hpp:125-127, impl proj/src/aggregate.cpp:401-452)
 * Plain pointers and sizes only; no C++ or torch types cross this boundary. A C++ shim with the
 * reference's exact signature lives in include/cvlg.hpp; the bindings a reference maintainer would
 * add are shown in INTEGRATION.md.
 *
 * Output lattice (caller-owned, dense, little-endian u32 words):
 *   planes    [T][8][R][C]: channels 0..3 = mean speed N,E,S,W as f32 bit patterns,
 *                           channels 4..7 = distinct-journey volume N,E,S,W
 *             (= BatchFrame::speed / ::volume, aggregate.hpp:46-57; this is also the block
 *              payload of the .cvl1 container, lattice_store.hpp:14-19)
 *   raw_count [T][4][R][C]: raw record counts per direction (BatchFrame::raw_count)
 * Planes are row-major R x C with row 0 at lat_min. T = 1440/min_step, R/C from extent_bins.
 *
 * Errors: every entry point returns 0 on success, otherwise 1 + the ordinal of the reference's
 * cvl::Err (proj/include/cvl/error.hpp:8-26), or one of the CVLG_E_* codes >= 100 for conditions
 * the reference has no code for. cvlg_last_error() returns the message of the calling thread's
 * last failure. Data problems are never errors: they are counted in cvlg_stats, exactly like the
 * reference's PipelineStats (aggregate.hpp:112-121).
 */
#ifndef CVLG_H_
#define CVLG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cvl::Err + 1 (error.hpp:8-26) */
enum cvlg_status {
    CVLG_OK = 0,
    CVLG_E_MISSING_ROOT = 1,
    CVLG_E_BAD_CONFIG = 2,
    CVLG_E_BAD_GRID = 3,
    CVLG_E_ZERO_PARTITIONS = 4,
    CVLG_E_OUT_OF_BOUNDS = 5,
    CVLG_E_COMPONENT_OUT_OF_RANGE = 6,
    CVLG_E_INDEX_OVERFLOW = 7,
    CVLG_E_GRID_MISMATCH = 8,
    CVLG_E_DIMS_MISMATCH = 9,
    CVLG_E_NON_FINITE_VALUE = 10,
    CVLG_E_IO = 11,
    CVLG_E_BAD_MAGIC = 12,
    CVLG_E_VERSION_UNSUPPORTED = 13,
    CVLG_E_TRUNCATED_FILE = 14,
    CVLG_E_BAD_CHANNEL = 15,
    CVLG_E_TASK_FAILED = 16,
    CVLG_E_DIVIDE_BY_ZERO = 17,
    /* conditions without a reference equivalent */
    CVLG_E_CUDA = 100,        /* CUDA runtime failure (no device, OOM, launch failure) */
    CVLG_E_INVALID_ARG = 101, /* null pointer / inconsistent sizes */
    CVLG_E_UNSUPPORTED = 102, /* e.g. > 4 direction bins (reference: UB), > 2^32-5 cells */
    CVLG_E_INTERNAL = 103     /* a capacity invariant was violated (bug) */
};

/* GridSpec, field for field (proj/include/cvl/grid.hpp:21-41). Defaults: 36, 40.6, -95.8,
 * -89.1, 0.1, 0.1, 5, 90, 0.0 (cvlg_default_grid). */
typedef struct cvlg_grid_spec {
    double lat_min, lat_max, lon_min, lon_max, lat_step, lon_step;
    uint32_t min_step, dxn_step;
    double dxn_offset;
} cvlg_grid_spec;

/* FilterRules (proj/include/cvl/aggregate.hpp:16-20). Defaults: 1, 1, 250.0. */
typedef struct cvlg_filter_rules {
    int32_t require_in_grid;
    int32_t drop_missing;
    double speed_ceiling;
} cvlg_filter_rules;

/* PipelineStats (aggregate.hpp:112-121) with the string-keyed maps flattened:
 *   rejected[]: BadTimestamp, BadNumeric, MissingField, RangeViolation, BadHeader
 *   filtered[]: OutOfGrid, SpeedCeiling, MissingField
 *   stage_seconds[]: the reference's stages (aggregate.cpp:370-383, 449), device time from
 *   CUDA events: parse (decode), dedup+filter+accumulate (journey dictionary, canonical order,
 *   per-journey fold), merge ((cell, journey) sort), finalize */
typedef struct cvlg_stats {
    uint64_t rows_read, parsed, duplicates_dropped, conflicting_duplicates, accepted;
    uint64_t rejected[5];
    uint64_t filtered[3];
    double stage_seconds[4];
} cvlg_stats;

typedef struct cvlg_context cvlg_context;

void cvlg_default_grid(cvlg_grid_spec* spec);
void cvlg_default_rules(cvlg_filter_rules* rules);

/* Validates like GridSpec::validate (grid.cpp:47-57) and returns the lattice dimensions
 * T = batches, D = directions, R = rows, C = cols (grid.cpp:18-22, grid.hpp:33-36). */
int cvlg_grid_dims(const cvlg_grid_spec* spec, uint32_t* T, uint32_t* D, uint32_t* R, uint32_t* C);

/* One context per (host thread, device). Holds streams and grow-only HBM/pinned scratch so
 * repeated calls do not allocate. device < 0 selects the current device. NULL on failure. */
cvlg_context* cvlg_context_create(int device);
void cvlg_context_destroy(cvlg_context* ctx);

/* Replaces cvl::run_pipeline (aggregate.hpp:125-127). Shards are read from disk (n_threads
 * reader threads, 0 = hardware concurrency) into pinned memory, ranked by lexicographic path
 * (aggregate.cpp:389-397), streamed to HBM and processed on the GPU. n_partitions is validated
 * (0 -> CVLG_E_ZERO_PARTITIONS) and otherwise cannot change the output: the result is
 * byte-identical for every partition count, like the reference's. planes / raw_count may be
 * NULL. ctx may be NULL (a thread-local default context is used). */
int cvlg_run_pipeline(cvlg_context* ctx, const char* const* shard_paths, size_t n_shards,
                      const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                      uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                      uint32_t* raw_count, cvlg_stats* stats);

/* Same pipeline over shard bytes already in host memory (pinned or pageable), given in rank
 * order (index i = provenance rank i). Host->device copies are chunked, line-aligned and
 * overlapped with decode. */
int cvlg_run_pipeline_host(cvlg_context* ctx, const uint8_t* const* shard_bufs,
                           const uint64_t* shard_lens, size_t n_shards,
                           const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                           uint32_t n_partitions, uint32_t* planes, uint32_t* raw_count,
                           cvlg_stats* stats);

/* Device-resident pipeline: d_csv holds the shards concatenated in rank order (HBM, 16-byte
 * alignment recommended), shard i occupying [shard_offsets[i], shard_offsets[i+1]) with
 * shard_offsets (host array, n_shards + 1 entries) starting at 0. d_planes / d_raw_count are
 * device buffers (d_raw_count may be NULL). Runs on `stream` (cudaStream_t, NULL = the
 * context's stream) and returns after the results are complete. */
int cvlg_run_pipeline_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                             size_t n_shards, const cvlg_grid_spec* spec,
                             const cvlg_filter_rules* rules, uint32_t* d_planes,
                             uint32_t* d_raw_count, cvlg_stats* stats, void* stream);

/* One parsed record with its provenance: cvl::CvRecord + cvl::RecordProvenance
 * (records.hpp:13-32). Strings are borrowed (pointer + length, need not be NUL-terminated). */
typedef struct cvlg_record {
    const char* journey_id;
    uint32_t journey_len;
    uint32_t postal_len;
    const char* postal_code;
    const char* shard_path;
    uint32_t shard_path_len;
    uint32_t reserved;
    int64_t line_number; /* 1-based, header excluded */
    int64_t epoch_sec;
    double latitude, longitude, speed, heading;
} cvlg_record;

/* Replaces cvl::run_pipeline_from_records (aggregate.hpp:130-133, aggregate.cpp:454-491): the
 * same pipeline over records that are already parsed (no parse step and no parse checks: values
 * are taken as they are). Provenance rank = rank of shard_path among the sorted unique paths;
 * the dedup survivor is the record with the minimum (rank, (uint32) line_number); rows_read =
 * parsed = n. Conflicting duplicates compare the full record (id, time, lat, lon, postal code,
 * speed, heading with ==), each non-survivor against the survivor. */
int cvlg_run_pipeline_records(cvlg_context* ctx, const cvlg_record* records, size_t n,
                              const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                              uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                              uint32_t* raw_count, cvlg_stats* stats);

/* ---- multi-GPU building blocks (one process per GPU; journeys sharded by FNV-1a id hash,
 * ingest.cpp:287-301, so every journey lives on exactly one GPU) ---------------------------
 * cvlg_partial_device runs the device-resident pipeline up to the per-(cell, journey) subtotals
 * and keeps them in the context (n_pairs out). cvlg_export_pairs writes them to caller device
 * buffers as (cell, key0, key1, f64 sum, u64 count) with GLOBAL journey keys (exact,
 * order-preserving inline keys; ids longer than 15 bytes -> CVLG_E_UNSUPPORTED).
 * cvlg_finalize_pairs folds any union of such tuples (e.g. after an all-to-all by cell owner)
 * into a lattice: tuples are ordered by (cell, journey key) and folded exactly like the
 * reference's finalize (aggregate.cpp:161-204); cells without tuples are zero. */
int cvlg_partial_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                        size_t n_shards, const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                        uint64_t* n_pairs, cvlg_stats* stats, void* stream);
int cvlg_export_pairs(cvlg_context* ctx, uint64_t* d_cell, uint64_t* d_key0, uint64_t* d_key1,
                      double* d_sum, uint64_t* d_count, void* stream);
int cvlg_finalize_pairs(cvlg_context* ctx, const uint64_t* d_cell, const uint64_t* d_key0,
                        const uint64_t* d_key1, const double* d_sum, const uint64_t* d_count,
                        uint64_t n, const cvlg_grid_spec* spec, uint32_t* d_planes,
                        uint32_t* d_raw_count, void* stream);

/* ---- multi-GPU pipeline, one host thread ---------------------------
 * cvl::run_pipeline over n_gpus GPUs: journeys are sharded by journey_hash(id) % n_gpus
 * (FNV-1a 64, ingest.cpp:287-291), like the reference's partitions (aggregate.cpp:414-443). Each
 * GPU streams a 1/n_gpus byte range of the shards (cut at line boundaries) into HBM, routes every
 * data line to the GPU owning its journey (stores into the peer's HBM over NVLink), aggregates its
 * journeys, and sends (cell, journey key, sum, count) tuples to the GPU owning the cell's time
 * slab, which folds them in the reference's (cell, journey) order. Output and stats are
 * byte-identical to cvlg_run_pipeline for every n_gpus. `devices` lists the CUDA devices (NULL:
 * 0..n_gpus-1); a device may repeat (several shards on one GPU). Journey keys across GPUs are the
 * exact inline ids when every id is <= 15 bytes, else global ranks from a host merge of the
 * GPUs' sorted id lists. */
typedef struct cvlg_multi cvlg_multi;
cvlg_multi* cvlg_multi_create(const int* devices, uint32_t n_gpus);
void cvlg_multi_destroy(cvlg_multi* m);
uint32_t cvlg_multi_size(const cvlg_multi* m);
cvlg_context* cvlg_multi_context(cvlg_multi* m, uint32_t gpu);  /* borrowed */
int cvlg_run_pipeline_multi(cvlg_multi* m, const char* const* shard_paths, size_t n_shards,
                            const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                            uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                            uint32_t* raw_count, cvlg_stats* stats);

/* The same steps for one process per GPU (the caller moves bytes, e.g. NCCL all-to-all):
 *  1. cvlg_route_stage: rank the paths, cut the data lines into n_parts ranges, stream range
 *     `part` into this context's HBM and count the bytes each owner (0..n_parts-1) receives.
 *  2. cvlg_route_plan: bytes of the stream for `owner` and the offsets (within it) of its
 *     n_pieces virtual shards (header line + the piece's lines routed to `owner`).
 *  3. cvlg_route_scatter: writes the streams to d_dst[owner] (device pointers on this device).
 *     The owner concatenates the streams of parts 0..n_parts-1 in order and runs
 *     cvlg_partial_device over them with the virtual shard offsets as shard_offsets; the BadHeader
 *     count (bad_headers, identical on every part) is added once.
 *  4. cvlg_tuples_export: the subtotals of that run as 40-byte (u64 cell, u64 key0, u64 key1,
 *     f64 sum, u64 count) tuples, counted per slab owner (counts[n_owners], owner of a tuple =
 *     t * n_owners / T for its time bin t; cvlg_slab_rows gives each owner's rows [t0, t1)).
 *  5. cvlg_tuples_scatter: writes them to d_dst[owner] (device pointers on this device).
 *  6. cvlg_finalize_tuples: folds received tuples into rows [t0, t1) of the lattice (the
 *     owner's slab; d_planes / d_raw_count hold those rows only). */
int cvlg_route_stage(cvlg_context* ctx, const char* const* shard_paths, size_t n_shards,
                     uint32_t n_parts, uint32_t part, uint32_t n_threads, uint64_t* n_pieces,
                     uint64_t* bad_headers);
/* Re-runs the count of step 1 on the range already in HBM (device-resident measurements). */
int cvlg_route_count(cvlg_context* ctx);
int cvlg_route_plan(cvlg_context* ctx, uint32_t owner, uint64_t* vshard_off, uint64_t* stream_len);
int cvlg_route_scatter(cvlg_context* ctx, uint8_t* const* d_dst, void* stream);
int cvlg_tuples_export(cvlg_context* ctx, const cvlg_grid_spec* spec, uint32_t n_owners,
                       const uint32_t* global_rank, uint64_t* counts, uint64_t* n_tuples);
/* Journey keys across GPUs: with every id <= 15 bytes (cvlg_partial_info long_ids == 0 on every
 * rank) the tuples carry exact inline keys (global_rank NULL). Otherwise every rank exports its
 * sorted ids (cvlg_journey_ids, local rank order; call with NULL buffers for the sizes), the
 * lists are merged (cvlg_merge_id_ranks, host only: ranks[i][r] = global lexicographic rank of
 * list i's id r) and each rank passes its global_rank (host array, one per local journey). */
int cvlg_partial_info(cvlg_context* ctx, uint64_t* n_journeys, uint64_t* n_pairs, int32_t* long_ids);
int cvlg_journey_ids(cvlg_context* ctx, uint8_t* blob, uint64_t blob_cap, uint64_t* offs,
                     uint64_t offs_cap, uint64_t* n_journeys, uint64_t* blob_bytes);
int cvlg_merge_id_ranks(uint32_t n_lists, const uint8_t* const* blobs, const uint64_t* const* offs,
                        const uint64_t* n_ids, uint32_t* const* ranks);
int cvlg_tuples_scatter(cvlg_context* ctx, const cvlg_grid_spec* spec, uint32_t n_owners,
                        void* const* d_dst, void* stream);
int cvlg_finalize_tuples(cvlg_context* ctx, const void* d_tuples, uint64_t n,
                         const cvlg_grid_spec* spec, uint32_t t0, uint32_t t1, uint32_t* d_planes,
                         uint32_t* d_raw_count, void* stream);
int cvlg_slab_rows(uint32_t n_batches, uint32_t n_owners, uint32_t owner, uint32_t* t0, uint32_t* t1);
/* Host only (no GPU needed): the pieces of part `part` of n_parts, as cvlg_route_stage cuts them:
 * (rank of the file in lexicographic path order, byte offset, length), at most `cap` written. */
int cvlg_split_manifest(const char* const* shard_paths, size_t n_shards, uint32_t n_parts,
                        uint32_t part, uint32_t* piece_file, uint64_t* piece_off, uint64_t* piece_len,
                        size_t cap, size_t* n_pieces);

/* ---- per-journey feature table (north_star extension) -----------------
 * NOT IN THE REFERENCE (proj/ has no such function): parity is against this repository's CPU
 * restatement (tests/test_features.py), never against cvl::run_pipeline. Runs the pipeline (the
 * lattice outputs are as cvlg_run_pipeline_host / _device) and, per journey in lexicographic id
 * order, over the records the lattice aggregates in timestamp order: record count, first/last
 * epoch second, haversine trip length and largest step (mean Earth radius 6,371,008.8 m), largest
 * speed, largest |d speed / d t|, dwell seconds (steps with both ends at speed <= stop_speed) and
 * stop episodes; per cell, min / max speed (f32) in [T][4][R][C] (0 where no record). The
 * results stay in the context until cvlg_features_copy. */
typedef struct cvlg_features {
    uint64_t n_journeys;   /* out */
    uint32_t* points;      /* each array: n_journeys entries, host memory; NULL = skip */
    int64_t* t_first;
    int64_t* t_last;
    double* length_m;
    double* max_step_m;
    double* max_speed;
    double* max_abs_accel;
    double* dwell_s;
    uint32_t* stops;
    uint64_t* id_span;     /* journey id bytes in the concatenated shards: offset | length << 40 */
    float* cell_speed_min; /* T * 4 * R * C */
    float* cell_speed_max;
} cvlg_features;

int cvlg_journey_features_host(cvlg_context* ctx, const uint8_t* const* shard_bufs,
                               const uint64_t* shard_lens, size_t n_shards, const cvlg_grid_spec* spec,
                               const cvlg_filter_rules* rules, double stop_speed, uint32_t* planes,
                               uint32_t* raw_count, cvlg_stats* stats, uint64_t* n_journeys);
int cvlg_journey_features_device(cvlg_context* ctx, const uint8_t* d_csv, const uint64_t* shard_offsets,
                                 size_t n_shards, const cvlg_grid_spec* spec,
                                 const cvlg_filter_rules* rules, double stop_speed, uint32_t* d_planes,
                                 uint32_t* d_raw_count, cvlg_stats* stats, uint64_t* n_journeys,
                                 void* stream);
int cvlg_features_copy(cvlg_context* ctx, cvlg_features* out);

/* .cvl1 container writer (lattice_store.cpp:78-134): 58-byte header then T blocks of
 * (u32 t, planes[t]). Byte-identical to the reference for the same frames. */
int cvlg_write_container(const uint32_t* planes, const cvlg_grid_spec* spec, int32_t day,
                         const char* path, uint64_t* bytes_written);

/* Per-stage device milliseconds of the context's last run: parse, dedup+filter+accumulate,
 * merge, finalize (as stage_seconds), then (index 4) the decode kernel alone and (index 5) the
 * dictionary + canonical order part of stage 1. n <= 6. */
int cvlg_last_stage_ms(cvlg_context* ctx, float* ms, int n);

/* Device address and size of the input bytes the context's last cvlg_run_pipeline /
 * cvlg_run_pipeline_host call staged in HBM (shards concatenated in rank order). They stay
 * resident, unchanged, until the next call on the context, so they can be passed back to
 * cvlg_run_pipeline_device (the device-resident measurement of the same input). */
int cvlg_context_input(cvlg_context* ctx, const uint8_t** d_csv, uint64_t* n_bytes);

/* Test hook: the decode output of the context's last run, one entry per data line in provenance
 * order (slot order; "\r\n" lines hold an inert slot): epoch seconds, speed (f64), cell code
 * (grid.cuh: cell index, or 0x7FFFFFFB rejected by parse, 0x7FFFFFFF OutOfGrid, 0x7FFFFFFE
 * SpeedCeiling, 0x7FFFFFFC off-grid with require_in_grid = false; bit 31 = run head) and the
 * line's byte offset in the concatenated input. *n = number of entries, at most cap written. */
int cvlg_debug_slots(cvlg_context* ctx, int64_t* ts, double* speed, uint32_t* code, uint64_t* loff,
                     uint64_t cap, uint64_t* n);

/* Pins / unpins caller memory for faster H2D (cudaHostRegister). */
int cvlg_pin_host(void* ptr, size_t bytes);
int cvlg_unpin_host(void* ptr);

/* Number of CUDA kernels this library has launched in this process. */
uint64_t cvlg_launch_count(void);

/* Copies the calling thread's last error message (NUL-terminated, truncated to len). */
int cvlg_last_error(char* buf, size_t len);

#ifdef __cplusplus
}
#endif

#endif /* CVLG_H_ */
