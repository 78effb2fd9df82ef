// Per-journey feature table and per-cell speed extremes (north_star extension).
//
// NOT IN THE REFERENCE: proj/ has no haversine, dwell or acceleration code, so parity is against
// this repo's own CPU restatement (tests/test_features.py), never against cvl::run_pipeline.
//
// Record set: exactly the records the lattice aggregates (aggregate.cpp:293-358): accepted by
// parse_record_impl, first of each (journey, epoch) duplicate group in provenance order, passing
// filter_reason. Order: each journey's records by timestamp (the canonical (rank, ts) order of
// the fold). One thread per journey walks them sequentially (exact, deterministic):
//   points        number of records
//   t_first/last  first / last epoch second
//   length_m      sum of haversine step distances (mean Earth radius 6,371,008.8 m) in ts order
//   max_step_m    largest step distance
//   max_speed     largest reported speed
//   max_abs_accel largest |speed_k - speed_{k-1}| / (t_k - t_{k-1}) (speed units per second)
//   dwell_s       sum of (t_k - t_{k-1}) over steps whose both ends have speed <= stop_speed
//   stops         number of stop episodes (maximal runs of records with speed <= stop_speed)
// Per cell: min / max of the records' speeds narrowed to f32 (order independent: atomics on the
// f32 bit patterns, which order like the values for non-negative speeds).
#include "agg_api.cuh"
#include "kernels.cuh"
#include "sort_api.cuh"

namespace cvlg {

namespace {

constexpr double kEarthRadiusM = 6371008.8;
constexpr double kDegToRad = 0.017453292519943295;  // pi / 180

__device__ __forceinline__ double haversine_m(double la1, double lo1, double la2, double lo2) {
    const double p1 = la1 * kDegToRad, p2 = la2 * kDegToRad;
    const double dp = (la2 - la1) * kDegToRad, dl = (lo2 - lo1) * kDegToRad;
    const double s1 = sin(0.5 * dp), s2 = sin(0.5 * dl);
    const double a = s1 * s1 + cos(p1) * cos(p2) * s2 * s2;
    return 2.0 * kEarthRadiusM * asin(sqrt(fmin(1.0, a)));
}

__global__ void __launch_bounds__(128) journey_features_kernel(FeatureParams F) {
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (j >= F.n_journeys) return;
    uint32_t points = 0, stops = 0;
    int64_t t_first = 0, t_last = 0, prev_ts = 0;
    double length = 0.0, max_step = 0.0, max_speed = 0.0, max_acc = 0.0, dwell = 0.0;
    double p_lat = 0.0, p_lon = 0.0, p_speed = 0.0;
    bool p_stopped = false, have_prev_any = false;
    int64_t prev_any_ts = 0;
    auto visit = [&](uint32_t slot) {
        const uint32_t code = F.code[slot] & kCodeMask;
        if (code == kCodeRejected) return;
        const int64_t t = F.ts[slot];
        if (F.slow) {  // duplicate (journey, epoch): dropped before filtering (aggregate.cpp:276)
            if (have_prev_any && t == prev_any_ts) return;
            have_prev_any = true;
            prev_any_ts = t;
        }
        if (code >= kCodeFirstSpecial) return;  // filtered
        const double la = F.lat[slot], lo = F.lon[slot], sp = F.speed[slot];
        const bool stopped = sp <= F.stop_speed;
        if (points == 0) {
            t_first = t;
            if (stopped) ++stops;
        } else {
            const double dt = static_cast<double>(t - prev_ts);
            const double step = haversine_m(p_lat, p_lon, la, lo);
            length += step;
            max_step = fmax(max_step, step);
            max_acc = fmax(max_acc, fabs(sp - p_speed) / dt);
            if (stopped && p_stopped) dwell += dt;
            if (stopped && !p_stopped) ++stops;
        }
        max_speed = fmax(max_speed, sp);
        ++points;
        t_last = t;
        prev_ts = t;
        p_lat = la;
        p_lon = lo;
        p_speed = sp;
        p_stopped = stopped;
        if (F.cell_min) {
            const uint32_t g = code;
            const uint64_t tt = g / (F.D * F.RC), d = (g / F.RC) % F.D, rc = g % F.RC;
            const uint64_t at = (tt * 4 + d) * F.RC + rc;
            const float f = __double2float_rn(sp);
            const uint32_t bits = f == 0.0f ? 0u : __float_as_uint(f);  // -0 -> +0
            atomicMin(&F.cell_min[at], bits);
            atomicMax(&F.cell_max[at], bits);
        }
    };
    const uint32_t a = F.jstart[j], b = F.jstart[j + 1];
    if (F.slow) {
        for (uint32_t p = a; p < b; ++p) visit(F.perm[p]);
    } else {
        for (uint32_t r = a; r < b; ++r) {
            const uint2 run = F.runs[r];
            for (uint32_t p = run.x; p < run.y; ++p) visit(p);
        }
    }
    F.points[j] = points;
    F.t_first[j] = t_first;
    F.t_last[j] = t_last;
    F.length_m[j] = length;
    F.max_step_m[j] = max_step;
    F.max_speed[j] = max_speed;
    F.max_abs_accel[j] = max_acc;
    F.dwell_s[j] = dwell;
    F.stops[j] = stops;
}

// first head (in provenance order) of every journey -> its id span in the CSV buffer
__global__ void journey_first_head_kernel(const uint32_t* hrank, uint64_t n_heads, uint32_t* first) {
    const uint64_t h = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (h < n_heads) atomicMin(&first[hrank[h]], static_cast<uint32_t>(h));
}

__global__ void journey_id_kernel(const uint32_t* first, const uint64_t* hid, uint64_t n, uint64_t* id_span) {
    const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (j < n) id_span[j] = hid[first[j]];
}

// cells nobody visited keep the +inf sentinel of the min plane: report 0 like the lattice
__global__ void cell_min_fix_kernel(uint32_t* cell_min, uint64_t n) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n && cell_min[i] == 0x7F800000u) cell_min[i] = 0u;
}

__global__ void fill_u32_kernel(uint32_t* p, uint64_t n, uint32_t v) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = v;
}

inline unsigned blocks(uint64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

void launch_journey_features(const FeatureParams& f, const uint32_t* hrank, uint64_t n_heads,
                             const uint64_t* hid, uint32_t* first_scratch, uint64_t* id_span,
                             uint64_t n_cells_planes, cudaStream_t s) {
    if (f.cell_min && n_cells_planes) {
        fill_u32_kernel<<<blocks(n_cells_planes, 256), 256, 0, s>>>(f.cell_min, n_cells_planes, 0x7F800000u);
        count_launch();
        cudaMemsetAsync(f.cell_max, 0, n_cells_planes * 4, s);
    }
    if (f.n_journeys) {
        journey_features_kernel<<<blocks(f.n_journeys, 128), 128, 0, s>>>(f);
        count_launch();
        cudaMemsetAsync(first_scratch, 0xFF, f.n_journeys * 4, s);
        journey_first_head_kernel<<<blocks(n_heads, 256), 256, 0, s>>>(hrank, n_heads, first_scratch);
        count_launch();
        journey_id_kernel<<<blocks(f.n_journeys, 256), 256, 0, s>>>(first_scratch, hid, f.n_journeys, id_span);
        count_launch();
    }
    if (f.cell_min && n_cells_planes) {
        cell_min_fix_kernel<<<blocks(n_cells_planes, 256), 256, 0, s>>>(f.cell_min, n_cells_planes);
        count_launch();
    }
}

}  // namespace cvlg
