// Multi-GPU data plane: routing of CSV data lines to the GPU owning their journey.
//
// The reference routes every parsed record to partition journey_hash(id) % P
// (proj/src/aggregate.cpp:432-438, journey_hash = FNV-1a 64, proj/src/ingest.cpp:287-291) and
// journeys never straddle partitions (aggregate.cpp:372-373). Here the partitions are GPUs and
// the unit that moves is the raw data line: each GPU holds a contiguous 1/N slice of the
// concatenated shards as "pieces" (a shard's data lines, header excluded, possibly cut at line
// boundaries), finds every line, hashes its trimmed journey_id field exactly like the record the
// reference would build from it (ingest.cpp:31-53, 128-143), and copies the line into the owner's
// receive stream. The owner's stream holds, per (source GPU, piece) in provenance order, the
// piece's header line followed by its lines routed there, so it is an ordinary manifest of
// "virtual shards" whose byte order is the reference's (shard_rank, line) provenance order
// (aggregate.cpp:274-276): the single-GPU pipeline runs on it unchanged.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cvlg {

constexpr int kRouteTile = 16384;   // piece bytes per routing tile (tiles never span pieces)
constexpr int kRouteHalo = 256;     // bytes staged past the tile (lines ending there need no global loads)
constexpr int kRouteThreads = 256;  // one thread per 64 tile bytes
constexpr int kMaxOwners = 16;      // GPUs per routing group

struct RouteParams {
    const uint8_t* in;           // the GPU's pieces, concatenated
    const uint64_t* piece_off;   // [n_pieces + 1] piece byte ranges in `in`
    const uint32_t* tile_first;  // [n_pieces + 1] first routing tile of each piece
    const int32_t* id_col;       // [n_pieces] journey_id column of the piece's shard
    uint32_t n_pieces;
    uint32_t n_tiles;
    uint32_t n_owners;
    uint32_t* tile_bytes;        // count pass: [n_tiles][n_owners] bytes routed to each owner
    const uint64_t* tile_base;   // scatter pass: [n_tiles][n_owners] stream offset of the
                                 // tile's first line for each owner (headers included)
    uint8_t* const* dst;         // scatter pass: [n_owners] destination streams (device or peer)
    unsigned long long* lines;   // [n_owners] routed data lines (count pass), nullable
    uint32_t* error;             // set to 1 when a line is >= 2^31 bytes (unsupported)
};

// Count pass: tile_bytes (and lines) for every tile.
void launch_route_count(const RouteParams& p, cudaStream_t s);
// Exclusive scan over tiles per owner (u64) into tile_base, plus the per-piece header offsets
// (hdr_incl[piece] = header bytes of pieces 0..piece) ; owner_total[o] = routed bytes.
// piece_obase[p][o] = routed bytes of pieces before p (the piece's header position is
// hdr_excl[p] + piece_obase[p][o]).
void launch_route_scan(const uint32_t* tile_bytes, uint32_t n_tiles, uint32_t n_owners,
                       const uint32_t* tile_piece_first, uint32_t n_pieces,
                       const uint64_t* hdr_incl, uint64_t* tile_base, uint64_t* piece_obase,
                       uint64_t* owner_total, cudaStream_t s);
// Scatter pass: every kept line to dst[owner] + its stream offset.
void launch_route_scatter(const RouteParams& p, cudaStream_t s);
// Header lines: piece p's header (hdr + hdr_off[p], hdr_len[p] bytes) to every owner's stream at
// hdr_off[p] + piece_obase[p][o] (hdr_off doubles as hdr_excl: headers are stored back to back).
void launch_route_headers(const uint8_t* hdr, const uint64_t* hdr_off, uint32_t n_pieces,
                          const uint64_t* piece_obase, uint32_t n_owners, uint8_t* const* dst,
                          cudaStream_t s);

// (cell, journey key, f64 sum, u64 count) tuples of the per-cell combine, 40 bytes each.
struct PairTuple {
    uint64_t cell, key0, key1;
    double sum;
    uint64_t count;
};
// Tuples to the GPU owning the cell's time bin (contiguous slabs: owner = t * N / T).
void launch_tuple_count(const PairTuple* t, uint64_t n, uint64_t cells_per_t, uint32_t n_batches,
                        uint32_t n_owners, unsigned long long* counts, cudaStream_t s);
void launch_tuple_scatter(const PairTuple* t, uint64_t n, uint64_t cells_per_t, uint32_t n_batches,
                          uint32_t n_owners, unsigned long long* cursors, PairTuple* const* dst,
                          cudaStream_t s);

}  // namespace cvlg
