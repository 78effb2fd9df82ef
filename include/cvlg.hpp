// C++ shim over the cvlg C ABI with the reference pipeline's exact signature.
//
// Drop-in for   std::vector<cvl::BatchFrame> cvl::run_pipeline(const SourceManifest&,
//                   const GridSpec&, const FilterRules&, uint32_t n_partitions,
//                   uint32_t n_threads = 0, PipelineStats* stats = nullptr)
//               (reference: proj/include/cvl/aggregate.hpp:125-127)
//
// When the reference headers are on the include path (cvl/aggregate.hpp), this defines
// cvl::gpu::run_pipeline over the reference's own types, so a caller such as cmd_process
// (proj/src/cli.cpp:206) or process_day (proj/python/bindings.cpp:149) switches with a one-line
// change: `run_pipeline(...)` -> `gpu::run_pipeline(...)`. Errors are rethrown as
// cvl::CvlError with the same cvl::Err code. Without the reference headers it defines standalone
// mirror types in namespace cvlg with the same fields.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "cvlg.h"

namespace cvlg_detail {

inline std::string last_error() {
    char buf[1024];
    cvlg_last_error(buf, sizeof(buf));
    return buf;
}

template <class Spec>
cvlg_grid_spec to_c(const Spec& s) {
    cvlg_grid_spec g;
    g.lat_min = s.lat_min;
    g.lat_max = s.lat_max;
    g.lon_min = s.lon_min;
    g.lon_max = s.lon_max;
    g.lat_step = s.lat_step;
    g.lon_step = s.lon_step;
    g.min_step = s.min_step;
    g.dxn_step = s.dxn_step;
    g.dxn_offset = s.dxn_offset;
    return g;
}

template <class Rules>
cvlg_filter_rules to_c_rules(const Rules& r) {
    cvlg_filter_rules f;
    f.require_in_grid = r.require_in_grid ? 1 : 0;
    f.drop_missing = r.drop_missing ? 1 : 0;
    f.speed_ceiling = r.speed_ceiling;
    return f;
}

// Dense [T][8][R][C] + [T][4][R][C] -> BatchFrame list (aggregate.hpp:46-57 layout).
template <class Frame>
std::vector<Frame> to_frames(const std::vector<uint32_t>& planes, const std::vector<uint32_t>& raw,
                             uint32_t T, uint32_t R, uint32_t C) {
    const size_t rc = static_cast<size_t>(R) * C;
    std::vector<Frame> frames(T);
    for (uint32_t t = 0; t < T; ++t) {
        Frame& f = frames[t];
        f.t = t;
        f.rows = R;
        f.cols = C;
        for (uint32_t d = 0; d < 4; ++d) {
            f.speed[d].resize(rc);
            f.volume[d].resize(rc);
            f.raw_count[d].resize(rc);
            std::memcpy(f.speed[d].data(), planes.data() + (static_cast<size_t>(t) * 8 + d) * rc, rc * 4);
            std::memcpy(f.volume[d].data(), planes.data() + (static_cast<size_t>(t) * 8 + 4 + d) * rc,
                        rc * 4);
            std::memcpy(f.raw_count[d].data(), raw.data() + (static_cast<size_t>(t) * 4 + d) * rc,
                        rc * 4);
        }
    }
    return frames;
}

template <class Stats>
void fill_stats(const cvlg_stats& s, Stats* out) {
    if (!out) return;
    static const char* kRej[5] = {"BadTimestamp", "BadNumeric", "MissingField", "RangeViolation",
                                  "BadHeader"};
    static const char* kFil[3] = {"OutOfGrid", "SpeedCeiling", "MissingField"};
    static const char* kStage[4] = {"parse", "dedup+filter+accumulate", "merge", "finalize"};
    out->rows_read += s.rows_read;
    out->parsed += s.parsed;
    out->duplicates_dropped += s.duplicates_dropped;
    out->conflicting_duplicates += s.conflicting_duplicates;
    out->accepted += s.accepted;
    for (int i = 0; i < 5; ++i)
        if (s.rejected[i]) out->rejected[kRej[i]] += s.rejected[i];
    for (int i = 0; i < 3; ++i) out->filtered[kFil[i]] += s.filtered[i];
    for (int i = 0; i < 4; ++i) out->stage_seconds.emplace_back(kStage[i], s.stage_seconds[i]);
}

// Generic implementation over any reference-shaped types.
template <class Frame, class Manifest, class Spec, class Rules, class Stats, class Raise>
std::vector<Frame> run_pipeline_impl(const Manifest& manifest, const Spec& spec, const Rules& rules,
                                     uint32_t n_partitions, uint32_t n_threads, Stats* stats,
                                     Raise raise) {
    const cvlg_grid_spec g = to_c(spec);
    const cvlg_filter_rules f = to_c_rules(rules);
    uint32_t T = 0, D = 0, R = 0, C = 0;
    if (int rc = cvlg_grid_dims(&g, &T, &D, &R, &C)) raise(rc, last_error());
    std::vector<const char*> paths;
    paths.reserve(manifest.shard_paths.size());
    for (const auto& p : manifest.shard_paths) paths.push_back(p.c_str());
    std::vector<uint32_t> planes(static_cast<size_t>(T) * 8 * R * C);
    std::vector<uint32_t> raw(static_cast<size_t>(T) * 4 * R * C);
    cvlg_stats st;
    if (int rc = cvlg_run_pipeline(nullptr, paths.data(), paths.size(), &g, &f, n_partitions,
                                   n_threads, planes.data(), raw.data(), &st))
        raise(rc, last_error());
    fill_stats(st, stats);
    return to_frames<Frame>(planes, raw, T, R, C);
}

// cvl::run_pipeline_from_records over any record type with the reference's field names
// (CvRecord: journey_id, timestamp.epoch_sec, latitude, longitude, postal_code, speed, heading;
// RecordProvenance: shard_path, line_number, records.hpp:13-32)
template <class Frame, class Records, class Spec, class Rules, class Stats, class Raise>
std::vector<Frame> run_records_impl(const Records& records, const Spec& spec, const Rules& rules,
                                    uint32_t n_partitions, uint32_t n_threads, Stats* stats,
                                    Raise raise) {
    const cvlg_grid_spec g = to_c(spec);
    const cvlg_filter_rules f = to_c_rules(rules);
    uint32_t T = 0, D = 0, R = 0, C = 0;
    if (int rc = cvlg_grid_dims(&g, &T, &D, &R, &C)) raise(rc, last_error());
    std::vector<cvlg_record> recs(records.size());
    for (size_t i = 0; i < records.size(); ++i) {
        const auto& rec = records[i].first;
        const auto& prov = records[i].second;
        cvlg_record& r = recs[i];
        r.journey_id = rec.journey_id.data();
        r.journey_len = static_cast<uint32_t>(rec.journey_id.size());
        r.postal_code = rec.postal_code.data();
        r.postal_len = static_cast<uint32_t>(rec.postal_code.size());
        r.shard_path = prov.shard_path.data();
        r.shard_path_len = static_cast<uint32_t>(prov.shard_path.size());
        r.reserved = 0;
        r.line_number = prov.line_number;
        r.epoch_sec = rec.timestamp.epoch_sec;
        r.latitude = rec.latitude;
        r.longitude = rec.longitude;
        r.speed = rec.speed;
        r.heading = rec.heading;
    }
    std::vector<uint32_t> planes(static_cast<size_t>(T) * 8 * R * C);
    std::vector<uint32_t> raw(static_cast<size_t>(T) * 4 * R * C);
    cvlg_stats st;
    if (int rc = cvlg_run_pipeline_records(nullptr, recs.data(), recs.size(), &g, &f, n_partitions,
                                           n_threads, planes.data(), raw.data(), &st))
        raise(rc, last_error());
    fill_stats(st, stats);
    return to_frames<Frame>(planes, raw, T, R, C);
}

}  // namespace cvlg_detail

#if defined(__has_include)
#if __has_include("cvl/aggregate.hpp")
#include "cvl/aggregate.hpp"
#include "cvl/error.hpp"
#define CVLG_HAVE_REFERENCE_TYPES 1
#endif
#endif

#ifdef CVLG_HAVE_REFERENCE_TYPES
namespace cvl {
namespace gpu {

// Same contract as cvl::run_pipeline (aggregate.hpp:125-127); runs on the current CUDA device.
inline std::vector<BatchFrame> run_pipeline(const SourceManifest& manifest, const GridSpec& spec,
                                            const FilterRules& rules, uint32_t n_partitions,
                                            uint32_t n_threads = 0, PipelineStats* stats = nullptr) {
    return cvlg_detail::run_pipeline_impl<BatchFrame>(
        manifest, spec, rules, n_partitions, n_threads, stats,
        [](int rc, const std::string& msg) {
            if (rc >= 1 && rc <= 17) throw CvlError(static_cast<Err>(rc - 1), msg);
            throw std::runtime_error("cvlg: " + msg);
        });
}

// Same contract as cvl::run_pipeline_from_records (aggregate.hpp:130-133).
inline std::vector<BatchFrame> run_pipeline_from_records(
    const std::vector<std::pair<CvRecord, RecordProvenance>>& records, const GridSpec& spec,
    const FilterRules& rules, uint32_t n_partitions, uint32_t n_threads = 0,
    PipelineStats* stats = nullptr) {
    return cvlg_detail::run_records_impl<BatchFrame>(
        records, spec, rules, n_partitions, n_threads, stats,
        [](int rc, const std::string& msg) {
            if (rc >= 1 && rc <= 17) throw CvlError(static_cast<Err>(rc - 1), msg);
            throw std::runtime_error("cvlg: " + msg);
        });
}

}  // namespace gpu
}  // namespace cvl
#else
#include <array>
#include <map>

namespace cvlg {

// Standalone mirrors of the reference types (grid.hpp:21-41, aggregate.hpp:16-121,
// records.hpp:48-58, error.hpp:30-39).
struct GridSpec {
    double lat_min = 36.0, lat_max = 40.6, lon_min = -95.8, lon_max = -89.1;
    double lat_step = 0.1, lon_step = 0.1;
    uint32_t min_step = 5, dxn_step = 90;
    double dxn_offset = 0.0;
};
struct FilterRules {
    bool require_in_grid = true;
    double speed_ceiling = 250.0;
    bool drop_missing = true;
};
struct SourceManifest {
    std::vector<std::string> shard_paths;
};
struct BatchFrame {
    uint32_t t = 0, rows = 0, cols = 0;
    std::array<std::vector<float>, 4> speed;
    std::array<std::vector<uint32_t>, 4> volume;
    std::array<std::vector<uint32_t>, 4> raw_count;
};
struct PipelineStats {
    uint64_t rows_read = 0, parsed = 0, duplicates_dropped = 0, conflicting_duplicates = 0,
             accepted = 0;
    std::map<std::string, uint64_t> rejected, filtered;
    std::vector<std::pair<std::string, double>> stage_seconds;
};
class CvlError : public std::runtime_error {
public:
    CvlError(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const { return code_; }  // cvlg_status (= cvl::Err + 1)

private:
    int code_;
};

inline std::vector<BatchFrame> run_pipeline(const SourceManifest& manifest, const GridSpec& spec,
                                            const FilterRules& rules, uint32_t n_partitions,
                                            uint32_t n_threads = 0, PipelineStats* stats = nullptr) {
    return cvlg_detail::run_pipeline_impl<BatchFrame>(
        manifest, spec, rules, n_partitions, n_threads, stats,
        [](int rc, const std::string& msg) { throw CvlError(rc, msg); });
}

}  // namespace cvlg
#endif
