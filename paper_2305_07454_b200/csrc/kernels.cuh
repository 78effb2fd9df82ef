// Kernel interfaces of the sm_100a CV-ETL path (see DESIGN.md for the data layout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "grid.cuh"
#include "parse.cuh"

namespace cvlg {

// ---- decode (K0 header map, K1 tile decode) -------------------------------------------------
#ifndef CVLG_TILE
#define CVLG_TILE 16384
#endif
constexpr int kTile = CVLG_TILE;  // CSV bytes per decode tile
constexpr int kHalo = 128;    // bytes staged past the tile end (fast-path lines are <= 95 bytes)
constexpr int kPre = 16;      // bytes staged before the tile (previous-byte '\n' test)
constexpr int kDecodeThreads = kTile / 64;        // one thread per 64 tile bytes
constexpr int kLineCap = 352 * kTile / 16384;  // data lines handled per pass over a tile

// Slot word (one per data line): bits 0..30 = cell code (grid.cuh kCode*), bit 31 = run head.
constexpr uint32_t kHeadBit = 0x80000000u;
constexpr uint32_t kCodeMask = 0x7FFFFFFFu;
constexpr unsigned long long kNoKey = ~0ull;  // hkey[].y of heads whose key dict_insert derives itself

// Stats counters in device memory (u64 each).
enum : int {
    kStRowsRead = 0,
    kStRejBase = 1,  // + (reason-1): BadTimestamp, BadNumeric, MissingField, RangeViolation
    kStBadHeader = 5,
    kStParsed = 6,
    kStDups = 7,
    kStConflicts = 8,
    kStAccepted = 9,
    kStFiltOutOfGrid = 10,
    kStFiltSpeed = 11,
    kStFiltMissing = 12,
    kStGTransitions = 13,  // cell changes inside runs seen in decode: bound on (cell, journey) pairs
    kStUnbinnable = 14,    // kept records that would throw OutOfBounds
    kStOverflow = 15,      // capacity overflow (hash tables / slot arrays)
    kStHeads = 16,
    kStInert = 17,         // "\r\n" lines: hold a slot, are not data lines
    kStCount = 18,
};

// Per data line ("slot"). Slot space: tile t owns slots [t * kLineCap, t * kLineCap + lines(t))
// in provenance order (tiles are in byte order, shards in lexicographic path order); a tile with
// more than kLineCap data lines takes a range of the overflow region [reg_slots, ...). Slots past
// a tile's line count are never written and never read. Rejected lines keep their slot with code
// kCodeRejected.
struct DecodeOut {
    int64_t* ts;      // [slot] epoch seconds
    double* speed;    // [slot]
    uint32_t* code;   // [slot] cell code | kHeadBit
    uint64_t* loff;   // [slot] absolute line offset in the CSV buffer
    double* lat;      // [slot] (nullable: only written when per-journey features are requested)
    double* lon;
    uint32_t* hslot;  // [head scratch] run-head slots; tile t's at tiles[t].z + (0 .. tiles[t].w)
    uint64_t* hid;    // [head scratch] journey id span of the head: byte offset | length << 40
    ulonglong2* hkey;  // [head scratch] the dictionary key of ids <= 15 bytes (dict_insert's
                       // format), .y = kNoKey when the id is longer or not staged
    uint4* tiles;     // [tile] (slot base, data lines, head base, heads)
    uint64_t reg_slots;                  // n_tiles * kLineCap
    unsigned long long* ovf_slots;       // overflow-region slot counter (zeroed)
    unsigned long long* ovf_heads;       // overflow-region head counter (zeroed)
    uint64_t ovf_slot_cap, ovf_head_cap;
};

struct DecodeParams {
    const uint8_t* csv;
    uint64_t avail_end;  // bytes [0, avail_end) resident in HBM
    uint64_t total_end;  // total CSV bytes
    const uint64_t* shard_off;  // [n_shards + 1]
    const ColumnMap* cmap;      // [n_shards]
    const uint8_t* shard_good;  // [n_shards]
    uint32_t n_shards;
    uint32_t tile_end;
    GridParams grid;
    DecodeOut out;
    uint64_t* stats;
    int aligned16;
};

void launch_parse_headers(const uint8_t* csv, const uint64_t* shard_off, uint32_t n_shards,
                          ColumnMap* cmap, uint8_t* good, uint64_t* stats, cudaStream_t s);
void launch_decode(const DecodeParams& p, uint32_t tile_begin, uint32_t n_tiles, cudaStream_t s);

// Records entry point (cvlg_run_pipeline_records): already-parsed records, in provenance order
// through perm, fill the same per-slot columns, run heads and tiles as K1 (tiles of kLineCap
// records, dense). Columns are indexed by record; loff[slot] = the record index.
struct RecordsDecodeParams {
    const uint32_t* perm;  // slot order -> record index
    uint64_t n;
    const int64_t* ts;
    const double* lat;
    const double* lon;
    const double* speed;
    const double* heading;
    const uint64_t* id;    // arena offset | length << 40
    const uint8_t* arena;  // journey id bytes
    uint64_t arena_len;
    const uint64_t* postal;       // postal code spans in postal_arena (the fold's conflict test)
    const uint8_t* postal_arena;
    uint32_t n_tiles;
    GridParams grid;
    DecodeOut out;
    uint64_t* stats;
};
void launch_records_decode(const RecordsDecodeParams& p, cudaStream_t s);

}  // namespace cvlg
