// TEST INFRASTRUCTURE: demonstrates the drop-in boundary with the reference's OWN types.
// Compiled against /root/reference/proj/include and linked with the reference objects
// (oracle/_ref/*.o) plus libcvlg.so. For the shard files given on the command line it runs
//   cvl::run_pipeline        (reference, CPU)  and
//   cvl::gpu::run_pipeline   (include/cvlg.hpp over the C ABI, sm_100a)
// with identical arguments, then compares BatchFrame::bitwise_equal + raw counts + stats and
// the bytes of cvl::write_container for both. Exit code 0 = identical.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "cvl/aggregate.hpp"
#include "cvl/ingest.hpp"
#include "cvl/lattice_store.hpp"
#include "cvlg.hpp"

static std::vector<char> slurp(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: dropin <lat_step> <shard.csv>...\n");
        return 2;
    }
    cvl::SourceManifest m;
    for (int i = 2; i < argc; ++i) m.shard_paths.push_back(argv[i]);
    cvl::GridSpec spec;
    spec.lat_step = spec.lon_step = std::stod(argv[1]);
    cvl::FilterRules rules;
    cvl::PipelineStats a, b;
    const auto ref = cvl::run_pipeline(m, spec, rules, 4, 1, &a);
    const auto gpu = cvl::gpu::run_pipeline(m, spec, rules, 4, 1, &b);
    if (ref.size() != gpu.size()) return 10;
    for (size_t t = 0; t < ref.size(); ++t) {
        if (!ref[t].bitwise_equal(gpu[t])) return 11;
        for (int d = 0; d < 4; ++d)
            if (ref[t].raw_count[d] != gpu[t].raw_count[d]) return 12;
    }
    if (a.rows_read != b.rows_read || a.parsed != b.parsed || a.accepted != b.accepted ||
        a.duplicates_dropped != b.duplicates_dropped ||
        a.conflicting_duplicates != b.conflicting_duplicates || a.rejected != b.rejected ||
        a.filtered != b.filtered)
        return 13;
    cvl::write_container(ref, spec, 18756, "/tmp/cvlg_dropin_ref.cvl1");
    cvl::write_container(gpu, spec, 18756, "/tmp/cvlg_dropin_gpu.cvl1");
    if (slurp("/tmp/cvlg_dropin_ref.cvl1") != slurp("/tmp/cvlg_dropin_gpu.cvl1")) return 14;
    // error mapping: BadGrid surfaces as cvl::CvlError(Err::BadGrid)
    cvl::GridSpec bad = spec;
    bad.min_step = 7;
    try {
        cvl::gpu::run_pipeline(m, bad, rules, 1);
        return 15;
    } catch (const cvl::CvlError& e) {
        if (e.code() != cvl::Err::BadGrid) return 16;
    }
    // the secondary boundary: cvl::run_pipeline_from_records over the same shards' records
    std::vector<std::pair<cvl::CvRecord, cvl::RecordProvenance>> recs;
    for (const auto& path : m.shard_paths) {
        cvl::ShardData sd = cvl::read_shard(path);
        for (size_t k = 0; k < sd.records.size(); ++k)
            recs.emplace_back(std::move(sd.records[k]), cvl::RecordProvenance{path, sd.line_numbers[k]});
    }
    cvl::PipelineStats ra, rb;
    const auto rref = cvl::run_pipeline_from_records(recs, spec, rules, 3, 1, &ra);
    const auto rgpu = cvl::gpu::run_pipeline_from_records(recs, spec, rules, 3, 1, &rb);
    if (rref.size() != rgpu.size()) return 17;
    for (size_t t = 0; t < rref.size(); ++t) {
        if (!rref[t].bitwise_equal(rgpu[t])) return 18;
        for (int d = 0; d < 4; ++d)
            if (rref[t].raw_count[d] != rgpu[t].raw_count[d]) return 19;
    }
    if (ra.rows_read != rb.rows_read || ra.accepted != rb.accepted || ra.filtered != rb.filtered) return 20;
    std::printf("drop-in identical: %zu frames, %llu records\n", gpu.size(),
                static_cast<unsigned long long>(b.accepted));
    return 0;
}
