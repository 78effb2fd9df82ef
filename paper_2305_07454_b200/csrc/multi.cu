// Multi-GPU pipeline: journeys sharded by FNV-1a id hash across GPUs.
//
// The reference parses shards on worker threads and routes every record to partition
// journey_hash(id) % P (proj/src/aggregate.cpp:414-443); partitions own whole journeys
// (aggregate.cpp:372-373), are aggregated independently and merged exactly (:372-378), and the
// merged entries are finalized in (cell, journey id) order (:161-204). Here a partition is a GPU:
//
//   1. split    the shards' data lines (headers excluded) into N contiguous byte ranges cut at line
//               boundaries (host; split_manifest);
//   2. stage    each GPU streams its range from the files through its pinned ring into HBM;
//   3. route    each GPU finds its lines and the owner of each (FNV-1a of the trimmed journey_id
//               % N) and writes every line into the owner's receive stream — directly into the
//               peer GPU's HBM (route.cu), so the exchange is the scatter itself;
//   4. local    each owner runs the single-GPU pipeline over its stream (virtual shards: one per
//               (source GPU, piece), in provenance order) up to the per-(cell, journey) subtotals;
//   5. combine  subtotals leave as (cell, exact journey key, f64 sum, count) tuples to the GPU
//               owning the cell's time slab (peer stores again), which folds them in the
//               reference's (cell, journey) order into its rows of the lattice.
//
// The same steps are exported one by one (cvlg_route_*, cvlg_tuples_*) for one-process-per-GPU
// callers that move the bytes with NCCL (paper_2305_07454_b200/distributed.py).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string_view>
#include <thread>
#include <vector>

#include "../../include/cvlg.h"
#include "pipeline_internal.cuh"
#include "route_api.cuh"
#include "sort_api.cuh"

namespace cvlg {

struct Piece {
    uint32_t file;
    uint64_t off, len;  // data bytes [off, off + len) of the file: complete lines
};

namespace {

// First line boundary at or after data position `pos` of file `path` (a boundary is a position
// whose previous byte is '\n'), bounded by `limit`.
uint64_t next_line_boundary(const char* path, uint64_t pos, uint64_t first, uint64_t limit) {
    if (pos <= first) return first;
    if (pos >= limit) return limit;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) fail(CVLG_E_IO, std::string("Io: cannot open shard ") + path);
    std::vector<char> buf(1 << 16);
    uint64_t at = pos - 1;
    uint64_t found = limit;
    while (at < limit) {
        const uint64_t want = std::min<uint64_t>(buf.size(), limit - at);
        const ssize_t k = ::pread(fd, buf.data(), want, static_cast<off_t>(at));
        if (k <= 0) break;
        const void* nl = std::memchr(buf.data(), '\n', static_cast<size_t>(k));
        if (nl) {
            found = at + static_cast<uint64_t>(static_cast<const char*>(nl) - buf.data()) + 1;
            break;
        }
        at += static_cast<uint64_t>(k);
    }
    ::close(fd);
    return std::min(found, limit);
}

}  // namespace

// The data lines of the good shards (in rank order, headers excluded) as n_parts contiguous
// ranges of about equal bytes, cut at line boundaries.
std::vector<std::vector<Piece>> split_manifest(const char* const* paths, const std::vector<ShardHead>& heads,
                                               uint32_t n_parts) {
    struct Seg {
        uint32_t file;
        uint64_t a, b, g0;
    };
    std::vector<Seg> segs;
    uint64_t D = 0;
    for (size_t r = 0; r < heads.size(); ++r) {
        const ShardHead& h = heads[r];
        if (!h.good || h.data_begin >= h.len) continue;
        segs.push_back(Seg{static_cast<uint32_t>(r), h.data_begin, h.len, D});
        D += h.len - h.data_begin;
    }
    std::vector<uint64_t> cut(n_parts + 1, D);
    cut[0] = 0;
    for (uint32_t k = 1; k < n_parts; ++k) {
        const uint64_t target = static_cast<uint64_t>((static_cast<unsigned __int128>(D) * k) / n_parts);
        uint64_t g = target;
        if (g < D) {
            size_t s = 0;
            while (s + 1 < segs.size() && segs[s + 1].g0 <= g) ++s;
            const Seg& sg = segs[s];
            const uint64_t pos = sg.a + (g - sg.g0);
            g = sg.g0 + (next_line_boundary(paths[sg.file], pos, sg.a, sg.b) - sg.a);
        }
        cut[k] = std::max(cut[k - 1], std::min(g, D));
    }
    std::vector<std::vector<Piece>> parts(n_parts);
    for (uint32_t k = 0; k < n_parts; ++k) {
        for (const Seg& sg : segs) {
            const uint64_t lo = std::max(cut[k], sg.g0), hi = std::min(cut[k + 1], sg.g0 + (sg.b - sg.a));
            if (lo < hi) parts[k].push_back(Piece{sg.file, sg.a + (lo - sg.g0), hi - lo});
        }
    }
    return parts;
}

void route_count(cvlg_context* c);

void merge_id_ranks(const std::vector<const std::vector<uint8_t>*>& blobs,
                    const std::vector<const std::vector<uint64_t>*>& offs,
                    std::vector<std::vector<uint32_t>>& ranks) {
    const size_t n = blobs.size();
    ranks.assign(n, {});
    struct Cur {
        size_t list;
        uint64_t r;
    };
    auto view = [&](const Cur& c) {
        const std::vector<uint64_t>& o = *offs[c.list];
        return std::string_view(reinterpret_cast<const char*>(blobs[c.list]->data()) + o[c.r],
                                o[c.r + 1] - o[c.r]);
    };
    // std::string order = lexicographic unsigned bytes, prefix first (string_view compare)
    auto later = [&](const Cur& a, const Cur& b) { return view(a) > view(b); };
    std::vector<Cur> heap;
    for (size_t i = 0; i < n; ++i) {
        const uint64_t J = offs[i]->size() - 1;
        ranks[i].assign(J, 0);
        if (J) heap.push_back(Cur{i, 0});
    }
    std::make_heap(heap.begin(), heap.end(), later);
    uint64_t g = 0;
    while (!heap.empty()) {
        std::pop_heap(heap.begin(), heap.end(), later);
        Cur c = heap.back();
        heap.pop_back();
        if (g >= 0xFFFFFFFFull) fail(CVLG_E_UNSUPPORTED, ">= 2^32 - 1 journeys");
        ranks[c.list][c.r] = static_cast<uint32_t>(g++);
        if (++c.r + 1 < offs[c.list]->size()) {
            heap.push_back(c);
            std::push_heap(heap.begin(), heap.end(), later);
        }
    }
}

// Step 2 + 3a: stream the pieces into c->slice, find every line's owner, count bytes per
// (tile, owner), scan. The routing plan stays in the context.
void route_stage(cvlg_context* c, const char* const* paths, const std::vector<ShardHead>& heads,
                 const std::vector<Piece>& pieces, uint32_t n_owners, unsigned n_threads) {
    if (n_owners == 0 || n_owners > static_cast<uint32_t>(kMaxOwners))
        fail(CVLG_E_INVALID_ARG, "routing supports 1.." + std::to_string(kMaxOwners) + " GPUs");
    cudaStream_t s = c->stream;
    const uint32_t P = static_cast<uint32_t>(pieces.size());
    const uint32_t N = n_owners;
    c->r_owners = N;
    c->r_h_poff.assign(P + 1, 0);
    c->r_h_hoff.assign(P + 1, 0);
    c->r_h_tfirst.assign(P + 1, 0);
    c->r_h_cmap.resize(P);
    std::vector<int32_t> idcol(P);
    std::string hdr;
    std::vector<FileRange> ranges;
    for (uint32_t p = 0; p < P; ++p) {
        const Piece& pc = pieces[p];
        c->r_h_poff[p + 1] = c->r_h_poff[p] + pc.len;
        const uint64_t tiles = (pc.len + kRouteTile - 1) / kRouteTile;
        if (c->r_h_tfirst[p] + tiles >= (1ull << 32)) fail(CVLG_E_UNSUPPORTED, "input too large for routing");
        c->r_h_tfirst[p + 1] = static_cast<uint32_t>(c->r_h_tfirst[p] + tiles);
        hdr += heads[pc.file].header;
        c->r_h_hoff[p + 1] = hdr.size();
        c->r_h_cmap[p] = heads[pc.file].cmap;
        idcol[p] = heads[pc.file].cmap.journey_id;
        ranges.push_back(FileRange{pc.file, pc.off, pc.len, c->r_h_poff[p]});
    }
    const uint64_t total = c->r_h_poff[P];
    const uint32_t n_tiles = c->r_h_tfirst[P];
    c->slice.ensure(total + 32);
    {
        RingIngest ring(c, paths, std::move(ranges), c->slice.as<uint8_t>(), n_threads);
        RingChunk ch;
        while (ring.next(ch)) {
        }
        ring.stop();
        CK(cudaStreamSynchronize(c->copy_stream));
    }
    c->r_poff.ensure((P + 1) * 8);
    c->r_tfirst.ensure((P + 1) * 4);
    c->r_idcol.ensure(P * 4 + 4);
    c->r_hdr.ensure(hdr.size() + 1);
    c->r_hoff.ensure((P + 1) * 8);
    CK(cudaMemcpy(c->r_poff.p, c->r_h_poff.data(), (P + 1) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->r_tfirst.p, c->r_h_tfirst.data(), (P + 1) * 4, cudaMemcpyHostToDevice));
    if (P) CK(cudaMemcpy(c->r_idcol.p, idcol.data(), P * 4, cudaMemcpyHostToDevice));
    if (!hdr.empty()) CK(cudaMemcpy(c->r_hdr.p, hdr.data(), hdr.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->r_hoff.p, c->r_h_hoff.data(), (P + 1) * 8, cudaMemcpyHostToDevice));
    route_count(c);
}

// Step 3a alone, on the slice already in HBM (device-resident measurements).
void route_count(cvlg_context* c) {
    cudaStream_t s = c->stream;
    const uint32_t P = static_cast<uint32_t>(c->r_h_poff.size() - 1);
    const uint32_t N = c->r_owners;
    const uint32_t n_tiles = c->r_h_tfirst[P];
    c->r_tbytes.ensure(static_cast<uint64_t>(n_tiles) * N * 4 + 4);
    c->r_tbase.ensure(static_cast<uint64_t>(n_tiles) * N * 8 + 8);
    c->r_pobase.ensure(static_cast<uint64_t>(P) * N * 8 + 8);
    c->r_total.ensure(N * 8);
    c->r_lines.ensure(N * 8);
    c->r_err.ensure(4);
    CK(cudaMemsetAsync(c->r_total.p, 0, N * 8, s));
    CK(cudaMemsetAsync(c->r_lines.p, 0, N * 8, s));
    CK(cudaMemsetAsync(c->r_err.p, 0, 4, s));
    RouteParams RP{};
    RP.in = c->slice.as<uint8_t>();
    RP.piece_off = c->r_poff.as<uint64_t>();
    RP.tile_first = c->r_tfirst.as<uint32_t>();
    RP.id_col = c->r_idcol.as<int32_t>();
    RP.n_pieces = P;
    RP.n_tiles = n_tiles;
    RP.n_owners = N;
    RP.tile_bytes = c->r_tbytes.as<uint32_t>();
    RP.lines = c->r_lines.as<unsigned long long>();
    RP.error = c->r_err.as<uint32_t>();
    launch_route_count(RP, s);
    if (n_tiles)
        launch_route_scan(c->r_tbytes.as<uint32_t>(), n_tiles, N, c->r_tfirst.as<uint32_t>(), P,
                          c->r_hoff.as<uint64_t>(), c->r_tbase.as<uint64_t>(), c->r_pobase.as<uint64_t>(),
                          c->r_total.as<uint64_t>(), s);
    c->r_h_pobase.assign(static_cast<size_t>(P) * N, 0);
    c->r_h_total.assign(N, 0);
    uint32_t err = 0;
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (P) CK(cudaMemcpy(c->r_h_pobase.data(), c->r_pobase.p, static_cast<size_t>(P) * N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c->r_h_total.data(), c->r_total.p, N * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&err, c->r_err.p, 4, cudaMemcpyDeviceToHost));
    if (err) fail(CVLG_E_UNSUPPORTED, "a data line of >= 2 GiB cannot be routed");
}

// Bytes of the stream this GPU sends to `owner`, and its virtual shard offsets within it.
uint64_t route_plan(const cvlg_context* c, uint32_t owner, std::vector<uint64_t>* vs) {
    const size_t P = c->r_h_poff.size() - 1;
    const uint32_t N = c->r_owners;
    if (vs) {
        vs->resize(P);
        for (size_t p = 0; p < P; ++p) (*vs)[p] = c->r_h_hoff[p] + c->r_h_pobase[p * N + owner];
    }
    return c->r_h_hoff[P] + c->r_h_total[owner];
}

// Step 3b: headers + lines into dst[o] (device pointers valid on this GPU: local or peer).
void route_scatter(cvlg_context* c, uint8_t* const* dst, cudaStream_t s) {
    const uint32_t P = static_cast<uint32_t>(c->r_h_poff.size() - 1);
    const uint32_t N = c->r_owners;
    c->r_dst.ensure(N * 8);
    CK(cudaMemcpyAsync(c->r_dst.p, dst, N * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    launch_route_headers(c->r_hdr.as<uint8_t>(), c->r_hoff.as<uint64_t>(), P, c->r_pobase.as<uint64_t>(),
                         N, c->r_dst.as<uint8_t* const>(), s);
    RouteParams RP{};
    RP.in = c->slice.as<uint8_t>();
    RP.piece_off = c->r_poff.as<uint64_t>();
    RP.tile_first = c->r_tfirst.as<uint32_t>();
    RP.id_col = c->r_idcol.as<int32_t>();
    RP.n_pieces = P;
    RP.n_tiles = c->r_h_tfirst[P];
    RP.n_owners = N;
    RP.tile_base = c->r_tbase.as<uint64_t>();
    RP.dst = c->r_dst.as<uint8_t* const>();
    RP.error = c->r_err.as<uint32_t>();
    launch_route_scatter(RP, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
}

// Step 5a: the context's subtotals as PairTuples (c->tuples), counted per slab owner.
void tuples_export(cvlg_context* c, const Dims& dims, uint32_t n_owners, cudaStream_t s,
                   const std::vector<uint32_t>* grank) {
    if (n_owners == 0 || n_owners > static_cast<uint32_t>(kMaxOwners))
        fail(CVLG_E_INVALID_ARG, "the combine supports 1.." + std::to_string(kMaxOwners) + " GPUs");
    const uint64_t n = c->part_pairs;
    c->tuples.ensure(n * sizeof(PairTuple) + 64);
    PairTuple* tu = c->tuples.as<PairTuple>();
    const uint32_t* d_grank = nullptr;
    if (grank) {
        c->r_grank.ensure(grank->size() * 4 + 4);
        if (!grank->empty())
            CK(cudaMemcpy(c->r_grank.p, grank->data(), grank->size() * 4, cudaMemcpyHostToDevice));
        d_grank = c->r_grank.as<uint32_t>();
    }
    export_tuples(c, &tu->cell, &tu->key0, &tu->key1, &tu->sum, &tu->count, 5, s, d_grank);
    c->t_n = n;
    c->t_counts.ensure(kMaxOwners * 8);
    CK(cudaMemsetAsync(c->t_counts.p, 0, kMaxOwners * 8, s));
    launch_tuple_count(tu, n, static_cast<uint64_t>(dims.D) * dims.RC, dims.T, n_owners,
                       c->t_counts.as<unsigned long long>(), s);
    c->t_h_counts.assign(n_owners, 0);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(c->t_h_counts.data(), c->t_counts.p, n_owners * 8, cudaMemcpyDeviceToHost));
}

// Step 5b: tuples to dst[o] (device pointers valid on this GPU).
void tuples_scatter(cvlg_context* c, const Dims& dims, uint32_t n_owners, PairTuple* const* dst,
                    cudaStream_t s) {
    c->t_dst.ensure(n_owners * 8);
    CK(cudaMemcpyAsync(c->t_dst.p, dst, n_owners * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(c->t_counts.p, 0, kMaxOwners * 8, s));
    launch_tuple_scatter(c->tuples.as<PairTuple>(), c->t_n, static_cast<uint64_t>(dims.D) * dims.RC,
                         dims.T, n_owners, c->t_counts.as<unsigned long long>(),
                         c->t_dst.as<PairTuple* const>(), s);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
}

// Rows [t0, t1) of the lattice owned by slab owner o of N (owner(t) = t * N / T).
void slab_rows(uint32_t T, uint32_t N, uint32_t o, uint32_t& t0, uint32_t& t1) {
    auto first = [&](uint32_t r) {  // smallest t with t * N / T >= r
        return static_cast<uint32_t>((static_cast<uint64_t>(r) * T + N - 1) / N);
    };
    t0 = std::min(first(o), T);
    t1 = std::min(first(o + 1), T);
}

}  // namespace cvlg

using namespace cvlg;

struct cvlg_multi {
    std::vector<int> devices;
    std::vector<cvlg_context*> ctx;
    bool peer = true;  // every pair of distinct devices has peer access
};

namespace {

// Runs fn(g) on one host thread per GPU (device made current); rethrows the first failure.
void parallel(cvlg_multi* m, const std::function<void(uint32_t)>& fn) {
    const uint32_t N = static_cast<uint32_t>(m->ctx.size());
    std::vector<Error> errs(N, Error{0, ""});
    std::vector<std::thread> th;
    for (uint32_t g = 0; g < N; ++g) {
        th.emplace_back([&, g] {
            try {
                CK(cudaSetDevice(m->ctx[g]->device));
                fn(g);
            } catch (const Error& e) {
                errs[g] = e;
            } catch (const std::bad_alloc&) {
                errs[g] = Error{CVLG_E_CUDA, "host allocation failed"};
            } catch (const std::exception& e) {
                errs[g] = Error{CVLG_E_INTERNAL, e.what()};
            }
        });
    }
    for (auto& t : th) t.join();
    for (const Error& e : errs)
        if (e.code) throw e;
}

void run_multi(cvlg_multi* m, const char* const* paths, size_t n, const cvlg_grid_spec* spec,
               const cvlg_filter_rules* rules, uint32_t n_threads, uint32_t* planes, uint32_t* raw,
               cvlg_stats* stats) {
    const Dims dims = validate_grid(spec);
    const uint32_t N = static_cast<uint32_t>(m->ctx.size());
    const std::vector<ShardHead> heads = read_shard_heads(paths, n);
    uint64_t bad = 0;
    for (const ShardHead& h : heads) bad += h.bad_header ? 1 : 0;
    const auto parts = split_manifest(paths, heads, N);
    const unsigned hw = n_threads ? n_threads : std::max(1u, std::thread::hardware_concurrency());
    const unsigned per_gpu = std::max(1u, hw / N);

    // 2 + 3a: stage and count on every GPU
    parallel(m, [&](uint32_t g) { route_stage(m->ctx[g], paths, heads, parts[g], N, per_gpu); });
    // receive layout: owner o's stream = sources in order, each its pieces in order
    std::vector<std::vector<uint64_t>> base(N, std::vector<uint64_t>(N, 0));
    std::vector<uint64_t> recv(N, 0);
    std::vector<std::vector<uint64_t>> voff(N);  // owner -> virtual shard offsets (+ end)
    std::vector<std::vector<ColumnMap>> vmap(N);
    for (uint32_t o = 0; o < N; ++o) {
        for (uint32_t g = 0; g < N; ++g) {
            std::vector<uint64_t> vs;
            const uint64_t len = route_plan(m->ctx[g], o, &vs);
            base[g][o] = recv[o];
            for (size_t p = 0; p < vs.size(); ++p) {
                voff[o].push_back(recv[o] + vs[p]);
                vmap[o].push_back(m->ctx[g]->r_h_cmap[p]);
            }
            recv[o] += len;
        }
        voff[o].push_back(recv[o]);
    }
    parallel(m, [&](uint32_t o) {
        m->ctx[o]->csv.ensure(recv[o] + 16);
        m->ctx[o]->input_bytes = recv[o];
    });
    // 3b: every GPU writes its lines straight into the owners' receive streams
    parallel(m, [&](uint32_t g) {
        cvlg_context* c = m->ctx[g];
        std::vector<uint8_t*> dst(N);
        std::vector<uint64_t> soff(N + 1, 0);
        for (uint32_t o = 0; o < N; ++o) soff[o + 1] = soff[o] + route_plan(c, o, nullptr);
        const bool direct = m->peer;
        if (!direct) c->r_send.ensure(soff[N] + 16);
        for (uint32_t o = 0; o < N; ++o)
            dst[o] = direct ? m->ctx[o]->csv.as<uint8_t>() + base[g][o] : c->r_send.as<uint8_t>() + soff[o];
        route_scatter(c, dst.data(), c->stream);
        if (!direct) {
            for (uint32_t o = 0; o < N; ++o)
                if (soff[o + 1] > soff[o])
                    CK(cudaMemcpyPeerAsync(m->ctx[o]->csv.as<uint8_t>() + base[g][o], m->ctx[o]->device,
                                           dst[o], c->device, soff[o + 1] - soff[o], c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    });
    // 4: each owner's journeys through the single-GPU pipeline, up to the subtotals
    std::vector<cvlg_stats> st(N);
    parallel(m, [&](uint32_t o) {
        cvlg_context* c = m->ctx[o];
        std::vector<uint8_t> good(vmap[o].size(), 1);
        run_core(c, c->csv.as<uint8_t>(), voff[o], vmap[o].data(), good.data(), 0, spec, rules, nullptr,
                 nullptr, &st[o], marks_of({ChunkMark{recv[o], recv[o], nullptr}}), true);
    });
    // journey keys that order like the ids across GPUs: exact inline keys (ids <= 15 bytes), else
    // global ranks from a merge of every owner's sorted ids
    bool long_ids = false;
    for (uint32_t o = 0; o < N; ++o) long_ids |= m->ctx[o]->part_long_ids;
    std::vector<std::vector<uint32_t>> granks;
    if (long_ids) {
        std::vector<std::vector<uint8_t>> blobs(N);
        std::vector<std::vector<uint64_t>> offs(N);
        parallel(m, [&](uint32_t o) { journey_ids(m->ctx[o], blobs[o], offs[o]); });
        std::vector<const std::vector<uint8_t>*> bp;
        std::vector<const std::vector<uint64_t>*> op;
        for (uint32_t o = 0; o < N; ++o) {
            bp.push_back(&blobs[o]);
            op.push_back(&offs[o]);
        }
        merge_id_ranks(bp, op, granks);
    }
    parallel(m, [&](uint32_t o) {
        tuples_export(m->ctx[o], dims, N, m->ctx[o]->stream, granks.empty() ? nullptr : &granks[o]);
    });
    // 5: tuples to their slab owners, folded there
    std::vector<uint64_t> tin(N, 0);
    std::vector<std::vector<uint64_t>> tbase(N, std::vector<uint64_t>(N, 0));
    for (uint32_t s = 0; s < N; ++s)
        for (uint32_t o = 0; o < N; ++o) {
            tbase[o][s] = tin[s];
            tin[s] += m->ctx[o]->t_h_counts[s];
        }
    parallel(m, [&](uint32_t s) { m->ctx[s]->tuples_in.ensure(tin[s] * sizeof(PairTuple) + 64); });
    parallel(m, [&](uint32_t o) {
        cvlg_context* c = m->ctx[o];
        std::vector<PairTuple*> dst(N);
        std::vector<uint64_t> soff(N + 1, 0);
        for (uint32_t s = 0; s < N; ++s) soff[s + 1] = soff[s] + c->t_h_counts[s];
        if (!m->peer) c->tuples_send.ensure(soff[N] * sizeof(PairTuple) + 64);
        for (uint32_t s = 0; s < N; ++s)
            dst[s] = m->peer ? m->ctx[s]->tuples_in.as<PairTuple>() + tbase[o][s]
                             : c->tuples_send.as<PairTuple>() + soff[s];
        tuples_scatter(c, dims, N, dst.data(), c->stream);
        if (!m->peer) {
            for (uint32_t s = 0; s < N; ++s)
                if (soff[s + 1] > soff[s])
                    CK(cudaMemcpyPeerAsync(m->ctx[s]->tuples_in.as<PairTuple>() + tbase[o][s], m->ctx[s]->device,
                                           dst[s], c->device, (soff[s + 1] - soff[s]) * sizeof(PairTuple),
                                           c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
    });
    const uint64_t rc4 = 4 * dims.RC;
    parallel(m, [&](uint32_t s) {
        cvlg_context* c = m->ctx[s];
        uint32_t t0, t1;
        slab_rows(dims.T, N, s, t0, t1);
        const uint64_t rows = t1 - t0;
        c->planes.ensure(rows * 2 * rc4 * 4 + 4);
        if (raw) c->raw.ensure(rows * rc4 * 4 + 4);
        PairTuple* tu = c->tuples_in.as<PairTuple>();
        finalize_tuples(c, &tu->cell, &tu->key0, &tu->key1, &tu->sum, &tu->count, 5, tin[s], dims, t0, t1,
                        c->planes.as<uint32_t>(), raw ? c->raw.as<uint32_t>() : nullptr, c->stream);
        if (rows) {
            if (planes)
                CK(cudaMemcpyAsync(planes + t0 * 2 * rc4, c->planes.as<uint32_t>(), rows * 2 * rc4 * 4,
                                   cudaMemcpyDeviceToHost, c->stream));
            if (raw)
                CK(cudaMemcpyAsync(raw + t0 * rc4, c->raw.as<uint32_t>(), rows * rc4 * 4,
                                   cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
    });
    if (stats) {
        cvlg_stats& out = *stats;
        std::memset(&out, 0, sizeof(out));
        for (uint32_t o = 0; o < N; ++o) {
            out.rows_read += st[o].rows_read;
            out.parsed += st[o].parsed;
            out.duplicates_dropped += st[o].duplicates_dropped;
            out.conflicting_duplicates += st[o].conflicting_duplicates;
            out.accepted += st[o].accepted;
            for (int i = 0; i < 5; ++i) out.rejected[i] += st[o].rejected[i];
            for (int i = 0; i < 3; ++i) out.filtered[i] += st[o].filtered[i];
            for (int i = 0; i < 4; ++i) out.stage_seconds[i] = std::max(out.stage_seconds[i], st[o].stage_seconds[i]);
        }
        out.rejected[4] += bad;
    }
}

std::vector<const char*> ranked_paths(const char* const* shard_paths, size_t n_shards) {
    std::vector<size_t> order(n_shards);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return std::strcmp(shard_paths[a], shard_paths[b]) < 0; });
    std::vector<const char*> ranked(n_shards);
    for (size_t r = 0; r < n_shards; ++r) ranked[r] = shard_paths[order[r]];
    return ranked;
}

}  // namespace

extern "C" {

cvlg_multi* cvlg_multi_create(const int* devices, uint32_t n_gpus) {
    cvlg_multi* m = nullptr;
    const int rc = guard([&] {
        if (n_gpus == 0 || n_gpus > static_cast<uint32_t>(kMaxOwners))
            fail(CVLG_E_INVALID_ARG, "n_gpus must be 1.." + std::to_string(kMaxOwners));
        m = new cvlg_multi();
        for (uint32_t g = 0; g < n_gpus; ++g) m->devices.push_back(devices ? devices[g] : static_cast<int>(g));
        for (uint32_t g = 0; g < n_gpus; ++g) {
            cvlg_context* c = cvlg_context_create(m->devices[g]);
            if (!c) fail(CVLG_E_CUDA, "cannot create a context on device " + std::to_string(m->devices[g]));
            m->ctx.push_back(c);
        }
        // peer access between every pair of distinct devices (NVLink / NVSwitch): the routing and
        // combine kernels store straight into the peer's buffers
        for (int a : m->devices)
            for (int b : m->devices) {
                if (a == b) continue;
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, a, b));
                if (!ok) {
                    m->peer = false;
                    continue;
                }
                CK(cudaSetDevice(a));
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CK(e);
            }
    });
    if (rc != CVLG_OK) {
        if (m)
            for (cvlg_context* c : m->ctx) cvlg_context_destroy(c);
        delete m;
        return nullptr;
    }
    return m;
}

void cvlg_multi_destroy(cvlg_multi* m) {
    if (!m) return;
    for (cvlg_context* c : m->ctx) cvlg_context_destroy(c);
    delete m;
}

uint32_t cvlg_multi_size(const cvlg_multi* m) { return m ? static_cast<uint32_t>(m->ctx.size()) : 0; }

cvlg_context* cvlg_multi_context(cvlg_multi* m, uint32_t g) {
    return (m && g < m->ctx.size()) ? m->ctx[g] : nullptr;
}

int cvlg_run_pipeline_multi(cvlg_multi* m, const char* const* shard_paths, size_t n_shards,
                            const cvlg_grid_spec* spec, const cvlg_filter_rules* rules,
                            uint32_t n_partitions, uint32_t n_threads, uint32_t* planes,
                            uint32_t* raw_count, cvlg_stats* stats) {
    return guard([&] {
        validate_grid(spec);
        if (n_partitions == 0) fail(CVLG_E_ZERO_PARTITIONS, "ZeroPartitions: n_partitions must be >= 1");
        if (!m) fail(CVLG_E_INVALID_ARG, "multi-GPU handle is NULL");
        if (n_shards && !shard_paths) fail(CVLG_E_INVALID_ARG, "shard_paths is NULL");
        const std::vector<const char*> ranked = ranked_paths(shard_paths, n_shards);
        run_multi(m, ranked.data(), n_shards, spec, rules, n_threads, planes, raw_count, stats);
    });
}

int cvlg_route_stage(cvlg_context* ctx, const char* const* shard_paths, size_t n_shards,
                     uint32_t n_parts, uint32_t part, uint32_t n_threads, uint64_t* n_pieces,
                     uint64_t* bad_headers) {
    return guard([&] {
        if (!ctx) fail(CVLG_E_INVALID_ARG, "context is NULL");
        if (n_shards && !shard_paths) fail(CVLG_E_INVALID_ARG, "shard_paths is NULL");
        if (part >= n_parts) fail(CVLG_E_INVALID_ARG, "part must be < n_parts");
        CK(cudaSetDevice(ctx->device));
        const std::vector<const char*> ranked = ranked_paths(shard_paths, n_shards);
        const std::vector<ShardHead> heads = read_shard_heads(ranked.data(), n_shards);
        uint64_t bad = 0;
        for (const ShardHead& h : heads) bad += h.bad_header ? 1 : 0;
        const auto parts = split_manifest(ranked.data(), heads, n_parts);
        route_stage(ctx, ranked.data(), heads, parts[part], n_parts, n_threads);
        ctx->r_bad_headers = bad;
        if (n_pieces) *n_pieces = parts[part].size();
        if (bad_headers) *bad_headers = bad;
    });
}

int cvlg_route_count(cvlg_context* ctx) {
    return guard([&] {
        if (!ctx || ctx->r_h_poff.empty()) fail(CVLG_E_INVALID_ARG, "no routing stage on this context");
        CK(cudaSetDevice(ctx->device));
        route_count(ctx);
    });
}

int cvlg_route_plan(cvlg_context* ctx, uint32_t owner, uint64_t* vshard_off, uint64_t* stream_len) {
    return guard([&] {
        if (!ctx || ctx->r_h_poff.empty()) fail(CVLG_E_INVALID_ARG, "no routing stage on this context");
        if (owner >= ctx->r_owners) fail(CVLG_E_INVALID_ARG, "owner out of range");
        std::vector<uint64_t> vs;
        const uint64_t len = route_plan(ctx, owner, &vs);
        if (vshard_off && !vs.empty()) std::memcpy(vshard_off, vs.data(), vs.size() * 8);
        if (stream_len) *stream_len = len;
    });
}

int cvlg_route_scatter(cvlg_context* ctx, uint8_t* const* d_dst, void* stream) {
    return guard([&] {
        if (!ctx || ctx->r_h_poff.empty()) fail(CVLG_E_INVALID_ARG, "no routing stage on this context");
        if (!d_dst) fail(CVLG_E_INVALID_ARG, "NULL destinations");
        CK(cudaSetDevice(ctx->device));
        route_scatter(ctx, d_dst, stream ? static_cast<cudaStream_t>(stream) : ctx->stream);
    });
}

int cvlg_partial_info(cvlg_context* ctx, uint64_t* n_journeys, uint64_t* n_pairs, int32_t* long_ids) {
    if (!ctx) return CVLG_E_INVALID_ARG;
    if (n_journeys) *n_journeys = ctx->part_J;
    if (n_pairs) *n_pairs = ctx->part_pairs;
    if (long_ids) *long_ids = ctx->part_long_ids ? 1 : 0;
    return CVLG_OK;
}

int cvlg_journey_ids(cvlg_context* ctx, uint8_t* blob, uint64_t blob_cap, uint64_t* offs,
                     uint64_t offs_cap, uint64_t* n_journeys, uint64_t* blob_bytes) {
    return guard([&] {
        if (!ctx) fail(CVLG_E_INVALID_ARG, "context is NULL");
        CK(cudaSetDevice(ctx->device));
        std::vector<uint8_t> b;
        std::vector<uint64_t> o;
        journey_ids(ctx, b, o);
        if (n_journeys) *n_journeys = o.size() - 1;
        if (blob_bytes) *blob_bytes = b.size();
        if (blob && !b.empty()) std::memcpy(blob, b.data(), std::min<uint64_t>(blob_cap, b.size()));
        if (offs) std::memcpy(offs, o.data(), std::min<uint64_t>(offs_cap, o.size()) * 8);
    });
}

int cvlg_merge_id_ranks(uint32_t n_lists, const uint8_t* const* blobs, const uint64_t* const* offs,
                        const uint64_t* n_ids, uint32_t* const* ranks) {
    return guard([&] {
        std::vector<std::vector<uint8_t>> bv(n_lists);
        std::vector<std::vector<uint64_t>> ov(n_lists);
        std::vector<const std::vector<uint8_t>*> bp;
        std::vector<const std::vector<uint64_t>*> op;
        for (uint32_t i = 0; i < n_lists; ++i) {
            ov[i].assign(offs[i], offs[i] + n_ids[i] + 1);
            bv[i].assign(blobs[i], blobs[i] + ov[i].back());
            bp.push_back(&bv[i]);
            op.push_back(&ov[i]);
        }
        std::vector<std::vector<uint32_t>> r;
        merge_id_ranks(bp, op, r);
        for (uint32_t i = 0; i < n_lists; ++i)
            if (!r[i].empty()) std::memcpy(ranks[i], r[i].data(), r[i].size() * 4);
    });
}

int cvlg_tuples_export(cvlg_context* ctx, const cvlg_grid_spec* spec, uint32_t n_owners,
                       const uint32_t* global_rank, uint64_t* counts, uint64_t* n_tuples) {
    return guard([&] {
        const Dims dims = validate_grid(spec);
        if (!ctx) fail(CVLG_E_INVALID_ARG, "context is NULL");
        CK(cudaSetDevice(ctx->device));
        std::vector<uint32_t> gr;
        if (global_rank) gr.assign(global_rank, global_rank + ctx->part_J);
        tuples_export(ctx, dims, n_owners, ctx->stream, global_rank ? &gr : nullptr);
        if (counts) std::memcpy(counts, ctx->t_h_counts.data(), n_owners * 8);
        if (n_tuples) *n_tuples = ctx->t_n;
    });
}

int cvlg_tuples_scatter(cvlg_context* ctx, const cvlg_grid_spec* spec, uint32_t n_owners,
                        void* const* d_dst, void* stream) {
    return guard([&] {
        const Dims dims = validate_grid(spec);
        if (!ctx) fail(CVLG_E_INVALID_ARG, "context is NULL");
        if (!d_dst) fail(CVLG_E_INVALID_ARG, "NULL destinations");
        if (ctx->t_h_counts.size() != n_owners) fail(CVLG_E_INVALID_ARG, "n_owners differs from cvlg_tuples_export");
        CK(cudaSetDevice(ctx->device));
        tuples_scatter(ctx, dims, n_owners, reinterpret_cast<PairTuple* const*>(d_dst),
                       stream ? static_cast<cudaStream_t>(stream) : ctx->stream);
    });
}

int cvlg_finalize_tuples(cvlg_context* ctx, const void* d_tuples, uint64_t n,
                         const cvlg_grid_spec* spec, uint32_t t0, uint32_t t1, uint32_t* d_planes,
                         uint32_t* d_raw_count, void* stream) {
    return guard([&] {
        const Dims dims = validate_grid(spec);
        if (!ctx) fail(CVLG_E_INVALID_ARG, "context is NULL");
        if (!d_planes || (n && !d_tuples)) fail(CVLG_E_INVALID_ARG, "NULL argument");
        CK(cudaSetDevice(ctx->device));
        const PairTuple* tu = static_cast<const PairTuple*>(d_tuples);
        if (t0 > t1 || t1 > dims.T) fail(CVLG_E_INVALID_ARG, "rows [t0, t1) outside the lattice");
        finalize_tuples(ctx, &tu->cell, &tu->key0, &tu->key1, &tu->sum, &tu->count, 5, n, dims, t0, t1,
                        d_planes, d_raw_count, stream ? static_cast<cudaStream_t>(stream) : ctx->stream);
    });
}

int cvlg_split_manifest(const char* const* shard_paths, size_t n_shards, uint32_t n_parts,
                        uint32_t part, uint32_t* piece_file, uint64_t* piece_off, uint64_t* piece_len,
                        size_t cap, size_t* n_pieces) {
    return guard([&] {
        if (n_shards && !shard_paths) fail(CVLG_E_INVALID_ARG, "shard_paths is NULL");
        if (part >= n_parts) fail(CVLG_E_INVALID_ARG, "part must be < n_parts");
        const std::vector<const char*> ranked = ranked_paths(shard_paths, n_shards);
        const std::vector<ShardHead> heads = read_shard_heads(ranked.data(), n_shards);
        const auto parts = split_manifest(ranked.data(), heads, n_parts);
        const std::vector<Piece>& ps = parts[part];
        if (n_pieces) *n_pieces = ps.size();
        for (size_t i = 0; i < ps.size() && i < cap; ++i) {
            if (piece_file) piece_file[i] = ps[i].file;
            if (piece_off) piece_off[i] = ps[i].off;
            if (piece_len) piece_len[i] = ps[i].len;
        }
    });
}

int cvlg_slab_rows(uint32_t n_batches, uint32_t n_owners, uint32_t owner, uint32_t* t0, uint32_t* t1) {
    if (!n_owners || owner >= n_owners || !t0 || !t1) return CVLG_E_INVALID_ARG;
    slab_rows(n_batches, n_owners, owner, *t0, *t1);
    return CVLG_OK;
}

}  // extern "C"
