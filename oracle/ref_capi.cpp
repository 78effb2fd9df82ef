// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the product path.
//
// A thin C ABI over the *unmodified* reference library (compiled from the sources under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Python tests and the
// bench's cpu_baseline / `--impl reference` arm drive the reference through these entry
// points via ctypes. Nothing here re-implements reference logic; every function forwards to
// the reference's own public API:
//   ref_run_pipeline      -> cvl::run_pipeline            proj/include/cvl/aggregate.hpp:125
//   ref_oracle_pipeline   -> cvl::oracle_pipeline         proj/include/cvl/bench.hpp:53
//   ref_parse_header      -> cvl::parse_header            proj/include/cvl/ingest.hpp:34
//   ref_parse_record      -> cvl::parse_record            proj/include/cvl/ingest.hpp:40
//   ref_generate_day      -> cvl::generate_day            proj/include/cvl/synth.hpp:61
//   ref_generate_day_mt   -> cvl::generate_journey + cvl::csv_header, one host thread per shard
//                            file, rows rendered with generate_day's own format string
//                            (synth.cpp:157-173); byte-identical to ref_generate_day (tested)
//   ref_write_container   -> cvl::write_container         proj/include/cvl/lattice_store.hpp:43
//   ref_bins              -> lat_bin/lon_bin/time_bin/dxn_bin/global_index  grid.hpp:49-56
//   ref_journey_hash      -> cvl::journey_hash            proj/include/cvl/ingest.hpp:68
//   ref_deduplicate       -> cvl::deduplicate             proj/include/cvl/ingest.hpp:63
#include <atomic>
#include <charconv>
#include <cstdio>
#include <filesystem>
#include <thread>
#include <cstdint>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "cvl/aggregate.hpp"
#include "cvl/bench.hpp"
#include "cvl/error.hpp"
#include "cvl/grid.hpp"
#include "cvl/ingest.hpp"
#include "cvl/lattice_store.hpp"
#include "cvl/synth.hpp"

using namespace cvl;

extern "C" {

struct ref_grid {
    double lat_min, lat_max, lon_min, lon_max, lat_step, lon_step;
    uint32_t min_step, dxn_step;
    double dxn_offset;
};

struct ref_rules {
    int32_t require_in_grid;
    int32_t drop_missing;
    double speed_ceiling;
};

// rejected[]: BadTimestamp, BadNumeric, MissingField, RangeViolation, BadHeader
// filtered[]: OutOfGrid, SpeedCeiling, MissingField
struct ref_stats {
    uint64_t rows_read, parsed, duplicates_dropped, conflicting_duplicates, accepted;
    uint64_t rejected[5];
    uint64_t filtered[3];
    double stage_seconds[4];
};

struct ref_record {
    int64_t epoch_sec;
    double latitude, longitude, speed, heading;
    char journey_id[64];
    char postal_code[64];
};
}

namespace {

GridSpec to_spec(const ref_grid* g) {
    GridSpec s;
    s.lat_min = g->lat_min;
    s.lat_max = g->lat_max;
    s.lon_min = g->lon_min;
    s.lon_max = g->lon_max;
    s.lat_step = g->lat_step;
    s.lon_step = g->lon_step;
    s.min_step = g->min_step;
    s.dxn_step = g->dxn_step;
    s.dxn_offset = g->dxn_offset;
    return s;
}

FilterRules to_rules(const ref_rules* r) {
    FilterRules f;
    if (r) {
        f.require_in_grid = r->require_in_grid != 0;
        f.drop_missing = r->drop_missing != 0;
        f.speed_ceiling = r->speed_ceiling;
    }
    return f;
}

int fail_code(const CvlError& e, char* err, size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return 1 + static_cast<int>(e.code());
}

int fail_other(const std::exception& e, char* err, size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return 1000;
}

// frames -> dense planes [T][8][R][C] (speed bits d0..3, volume d0..3) + raw [T][4][R][C]
void frames_to_planes(const std::vector<BatchFrame>& frames, uint32_t* planes, uint32_t* raw) {
    for (size_t t = 0; t < frames.size(); ++t) {
        const BatchFrame& f = frames[t];
        const size_t rc = static_cast<size_t>(f.rows) * f.cols;
        for (uint32_t d = 0; d < 4; ++d) {
            if (planes) {
                std::memcpy(planes + (t * 8 + d) * rc, f.speed[d].data(), rc * 4);
                std::memcpy(planes + (t * 8 + 4 + d) * rc, f.volume[d].data(), rc * 4);
            }
            if (raw) std::memcpy(raw + (t * 4 + d) * rc, f.raw_count[d].data(), rc * 4);
        }
    }
}

std::vector<BatchFrame> planes_to_frames(const uint32_t* planes, const GridSpec& spec) {
    const uint32_t T = spec.batches(), R = spec.rows(), C = spec.cols();
    const size_t rc = static_cast<size_t>(R) * C;
    std::vector<BatchFrame> frames;
    for (uint32_t t = 0; t < T; ++t) {
        BatchFrame f = BatchFrame::zeros(t, spec);
        for (uint32_t d = 0; d < 4; ++d) {
            std::memcpy(f.speed[d].data(), planes + (static_cast<size_t>(t) * 8 + d) * rc, rc * 4);
            std::memcpy(f.volume[d].data(), planes + (static_cast<size_t>(t) * 8 + 4 + d) * rc,
                        rc * 4);
        }
        frames.push_back(std::move(f));
    }
    return frames;
}

void fill_stats(const PipelineStats& st, ref_stats* out) {
    if (!out) return;
    std::memset(out, 0, sizeof(*out));
    out->rows_read = st.rows_read;
    out->parsed = st.parsed;
    out->duplicates_dropped = st.duplicates_dropped;
    out->conflicting_duplicates = st.conflicting_duplicates;
    out->accepted = st.accepted;
    static const char* kRej[5] = {"BadTimestamp", "BadNumeric", "MissingField", "RangeViolation",
                                  "BadHeader"};
    static const char* kFil[3] = {"OutOfGrid", "SpeedCeiling", "MissingField"};
    for (int i = 0; i < 5; ++i) {
        auto it = st.rejected.find(kRej[i]);
        if (it != st.rejected.end()) out->rejected[i] = it->second;
    }
    for (int i = 0; i < 3; ++i) {
        auto it = st.filtered.find(kFil[i]);
        if (it != st.filtered.end()) out->filtered[i] = it->second;
    }
    for (size_t i = 0; i < st.stage_seconds.size() && i < 4; ++i)
        out->stage_seconds[i] = st.stage_seconds[i].second;
}

} // namespace

extern "C" {

int ref_run_pipeline(const char* const* paths, size_t n_paths, const ref_grid* grid,
                     const ref_rules* rules, uint32_t n_partitions, uint32_t n_threads,
                     uint32_t* planes, uint32_t* raw, ref_stats* stats, char* err, size_t errlen) {
    try {
        SourceManifest m;
        for (size_t i = 0; i < n_paths; ++i) m.shard_paths.emplace_back(paths[i]);
        PipelineStats st;
        const GridSpec spec = to_spec(grid);
        const auto frames = run_pipeline(m, spec, to_rules(rules), n_partitions, n_threads, &st);
        frames_to_planes(frames, planes, raw);
        fill_stats(st, stats);
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

// one parsed record with provenance (layout = cvlg_record in include/cvlg.h)
struct ref_record_prov {
    const char* journey_id;
    uint32_t journey_len;
    uint32_t postal_len;
    const char* postal_code;
    const char* shard_path;
    uint32_t shard_path_len;
    uint32_t reserved;
    int64_t line_number;
    int64_t epoch_sec;
    double latitude, longitude, speed, heading;
};

// -> cvl::run_pipeline_from_records (aggregate.hpp:130-133)
int ref_run_pipeline_from_records(const ref_record_prov* recs, size_t n, const ref_grid* grid,
                                  const ref_rules* rules, uint32_t n_partitions, uint32_t n_threads,
                                  uint32_t* planes, uint32_t* raw, ref_stats* stats, char* err,
                                  size_t errlen) {
    try {
        std::vector<std::pair<CvRecord, RecordProvenance>> records;
        records.reserve(n);
        for (size_t i = 0; i < n; ++i) {
            const ref_record_prov& r = recs[i];
            CvRecord rec;
            rec.journey_id.assign(r.journey_id ? r.journey_id : "", r.journey_len);
            rec.timestamp.epoch_sec = r.epoch_sec;
            rec.latitude = r.latitude;
            rec.longitude = r.longitude;
            rec.postal_code.assign(r.postal_code ? r.postal_code : "", r.postal_len);
            rec.speed = r.speed;
            rec.heading = r.heading;
            RecordProvenance prov;
            prov.shard_path.assign(r.shard_path ? r.shard_path : "", r.shard_path_len);
            prov.line_number = r.line_number;
            records.emplace_back(std::move(rec), std::move(prov));
        }
        PipelineStats st;
        const auto frames = run_pipeline_from_records(records, to_spec(grid), to_rules(rules),
                                                      n_partitions, n_threads, &st);
        frames_to_planes(frames, planes, raw);
        fill_stats(st, stats);
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

int ref_oracle_pipeline(const char* const* paths, size_t n_paths, const ref_grid* grid,
                        const ref_rules* rules, uint32_t* planes, uint32_t* raw, char* err,
                        size_t errlen) {
    try {
        std::vector<std::pair<CvRecord, RecordProvenance>> records;
        for (size_t i = 0; i < n_paths; ++i) {
            ShardData shard = read_shard(paths[i]);
            for (size_t k = 0; k < shard.records.size(); ++k)
                records.emplace_back(std::move(shard.records[k]),
                                     RecordProvenance{paths[i], shard.line_numbers[k]});
        }
        const auto frames = oracle_pipeline(records, to_spec(grid), to_rules(rules));
        frames_to_planes(frames, planes, raw);
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

// cols[8] = journey_id, timestamp, latitude, longitude, postal_code, speed, heading, n_columns
int ref_parse_header(const char* line, size_t len, int32_t* cols) {
    const auto m = parse_header(std::string_view(line, len));
    if (!m) return 0;
    cols[0] = m->journey_id;
    cols[1] = m->timestamp;
    cols[2] = m->latitude;
    cols[3] = m->longitude;
    cols[4] = m->postal_code;
    cols[5] = m->speed;
    cols[6] = m->heading;
    cols[7] = m->n_columns;
    return 1;
}

// returns -1 when accepted (out filled), else the ParseReason ordinal
int ref_parse_record(const char* line, size_t len, const int32_t* cols, ref_record* out) {
    ColumnMap m;
    m.journey_id = cols[0];
    m.timestamp = cols[1];
    m.latitude = cols[2];
    m.longitude = cols[3];
    m.postal_code = cols[4];
    m.speed = cols[5];
    m.heading = cols[6];
    m.n_columns = cols[7];
    const ParseResult r = parse_record(std::string_view(line, len), m);
    if (const auto* rej = std::get_if<ParseRejection>(&r)) return static_cast<int>(rej->reason);
    const CvRecord& rec = std::get<CvRecord>(r);
    if (out) {
        out->epoch_sec = rec.timestamp.epoch_sec;
        out->latitude = rec.latitude;
        out->longitude = rec.longitude;
        out->speed = rec.speed;
        out->heading = rec.heading;
        std::strncpy(out->journey_id, rec.journey_id.c_str(), sizeof(out->journey_id) - 1);
        out->journey_id[sizeof(out->journey_id) - 1] = 0;
        std::strncpy(out->postal_code, rec.postal_code.c_str(), sizeof(out->postal_code) - 1);
        out->postal_code[sizeof(out->postal_code) - 1] = 0;
    }
    return -1;
}

int ref_generate_day(uint64_t seed, uint32_t n_journeys, uint32_t n_shards, double sample_period,
                     double mean_duration, const char* day, const char* out_dir,
                     const double* bbox /* lat_min, lat_max, lon_min, lon_max or NULL */,
                     uint64_t* total_rows, char* err, size_t errlen) {
    try {
        SynthConfig cfg;
        cfg.seed = seed;
        cfg.n_journeys = n_journeys;
        cfg.n_shards = n_shards;
        cfg.sample_period = sample_period;
        cfg.mean_duration = mean_duration;
        cfg.day = day;
        cfg.out_dir = out_dir;
        if (bbox) {
            cfg.lat_min = bbox[0];
            cfg.lat_max = bbox[1];
            cfg.lon_min = bbox[2];
            cfg.lon_max = bbox[3];
        }
        const SourceManifest m = generate_day(cfg);
        if (total_rows) *total_rows = m.total_rows;
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

int ref_generate_day_mt(uint64_t seed, uint32_t n_journeys, uint32_t n_shards, double sample_period,
                        double mean_duration, const char* day, const char* out_dir,
                        uint32_t n_threads, uint64_t* total_rows, char* err, size_t errlen) {
    try {
        SynthConfig cfg;
        cfg.seed = seed;
        cfg.n_journeys = n_journeys;
        cfg.n_shards = n_shards;
        cfg.sample_period = sample_period;
        cfg.mean_duration = mean_duration;
        cfg.day = day;
        cfg.out_dir = out_dir;
        if (cfg.n_shards == 0) fail(Err::BadConfig, "n_shards must be >= 1");
        std::filesystem::create_directories(cfg.out_dir);
        const std::string header = csv_header();
        std::atomic<uint32_t> next{0};
        std::atomic<uint64_t> rows{0};
        std::atomic<bool> bad{false};
        std::string first_err;
        std::mutex mu;
        auto work = [&] {
            std::vector<char> buf;
            buf.reserve(64u << 20);
            char line[256];
            for (uint32_t s = next.fetch_add(1); s < cfg.n_shards && !bad; s = next.fetch_add(1)) {
                try {
                    char name[32];
                    std::snprintf(name, sizeof(name), "shard_%04u.csv", s);
                    const std::string path = (std::filesystem::path(cfg.out_dir) / name).string();
                    std::FILE* f = std::fopen(path.c_str(), "wb");
                    if (!f) fail(Err::Io, "cannot open " + path + " for writing");
                    buf.assign(header.begin(), header.end());
                    buf.push_back('\n');
                    uint64_t local = 0;
                    for (uint32_t j = s; j < cfg.n_journeys; j += cfg.n_shards) {
                        for (const CvRecord& rec : generate_journey(j, cfg)) {
                            const int k = std::snprintf(line, sizeof(line), "%s,%s,%.6f,%.6f,%s,%.2f,%.2f\n",
                                                        rec.journey_id.c_str(), rec.timestamp.to_string().c_str(),
                                                        rec.latitude, rec.longitude, rec.postal_code.c_str(),
                                                        rec.speed, rec.heading);
                            buf.insert(buf.end(), line, line + k);
                            ++local;
                        }
                        if (buf.size() > (48u << 20)) {
                            if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) fail(Err::Io, "short write to " + path);
                            buf.clear();
                        }
                    }
                    if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f) != buf.size())
                        fail(Err::Io, "short write to " + path);
                    if (std::fclose(f) != 0) fail(Err::Io, "short write to " + path);
                    rows += local;
                } catch (const std::exception& e) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (first_err.empty()) first_err = e.what();
                    bad = true;
                }
            }
        };
        const uint32_t nt = std::max<uint32_t>(1, std::min<uint32_t>(n_threads ? n_threads : std::thread::hardware_concurrency(), cfg.n_shards));
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < nt; ++t) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        if (bad) throw std::runtime_error(first_err);
        if (total_rows) *total_rows = rows.load();
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

int ref_write_container(const uint32_t* planes, const ref_grid* grid, int32_t day,
                        const char* path, uint64_t* written, char* err, size_t errlen) {
    try {
        const GridSpec spec = to_spec(grid);
        const uint64_t n = write_container(planes_to_frames(planes, spec), spec, day, path);
        if (written) *written = n;
        return 0;
    } catch (const CvlError& e) {
        return fail_code(e, err, errlen);
    } catch (const std::exception& e) {
        return fail_other(e, err, errlen);
    }
}

// which: 0 lat_bin(x) 1 lon_bin(x) 2 time_bin(epoch) 3 dxn_bin(x) 4 rows 5 cols 6 validate
// For global_index use ref_global_index.
int ref_bins(const ref_grid* grid, int which, double x, int64_t epoch, uint64_t* out) {
    try {
        const GridSpec spec = to_spec(grid);
        switch (which) {
        case 0: *out = lat_bin(x, spec); break;
        case 1: *out = lon_bin(x, spec); break;
        case 2: *out = time_bin(Timestamp{epoch}, spec); break;
        case 3: *out = dxn_bin(x, spec); break;
        case 4: *out = spec.rows(); break;
        case 5: *out = spec.cols(); break;
        case 6: spec.validate(); *out = 0; break;
        default: return 1000;
        }
        return 0;
    } catch (const CvlError& e) {
        return 1 + static_cast<int>(e.code());
    }
}

int ref_global_index(const ref_grid* grid, uint32_t t, uint32_t d, uint32_t r, uint32_t c,
                     uint64_t* out) {
    try {
        *out = global_index(CellIndex{t, d, r, c}, to_spec(grid));
        return 0;
    } catch (const CvlError& e) {
        return 1 + static_cast<int>(e.code());
    }
}

int ref_timestamp_parse(const char* text, size_t len, int64_t* out) {
    const auto ts = Timestamp::parse(std::string_view(text, len));
    if (!ts) return 0;
    *out = ts->epoch_sec;
    return 1;
}

// parse_double (ingest.cpp:66-72) is file-local in the reference; it is exactly this call of the
// libstdc++ std::from_chars the reference links against.
int ref_from_chars(const char* s, size_t len, double* out) {
    if (len == 0) return 0;
    auto [ptr, ec] = std::from_chars(s, s + len, *out);
    return ec == std::errc() && ptr == s + len;
}

uint64_t ref_journey_hash(const char* id, size_t len) {
    return journey_hash(std::string_view(id, len));
}

// Reads the shards like the reference does and returns dedup survivors' (journey, epoch)
// keys in deduplicate()'s output order (journey-id lexicographic, then timestamp).
// ids: caller buffer of n_max * 64 bytes; epochs: n_max.
int64_t ref_deduplicate(const char* const* paths, size_t n_paths, char* ids, int64_t* epochs,
                        double* speeds, int64_t n_max, uint64_t* conflicts) {
    try {
        std::vector<std::pair<CvRecord, RecordProvenance>> records;
        for (size_t i = 0; i < n_paths; ++i) {
            ShardData shard = read_shard(paths[i]);
            for (size_t k = 0; k < shard.records.size(); ++k)
                records.emplace_back(std::move(shard.records[k]),
                                     RecordProvenance{paths[i], shard.line_numbers[k]});
        }
        const auto out = deduplicate(std::move(records), conflicts);
        const int64_t n = static_cast<int64_t>(out.size());
        for (int64_t i = 0; i < n && i < n_max; ++i) {
            std::strncpy(ids + i * 64, out[i].journey_id.c_str(), 63);
            ids[i * 64 + 63] = 0;
            epochs[i] = out[i].timestamp.epoch_sec;
            speeds[i] = out[i].speed;
        }
        return n;
    } catch (...) {
        return -1;
    }
}

} // extern "C"
