// Per-journey feature table and per-cell speed extremes (north_star extension).
//
// NOT IN THE REFERENCE: proj/ has no haversine, dwell or acceleration code, so parity is against
// this repo's own CPU restatement (tests/test_features.py), never against cvl::run_pipeline.
//
// Record set: exactly the records the lattice aggregates (aggregate.cpp:293-358): accepted by
// parse_record_impl, first of each (journey, epoch) duplicate group in provenance order, passing
// filter_reason. Order: each journey's records by timestamp (the canonical (rank, ts) order of
// the fold). One warp per journey walks them in 32-record chunks (coalesced loads; the link to the
// previous kept record by ballot/shuffle; per-lane partial sums reduced in a fixed order at the
// end, so the result is deterministic):
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

#include <algorithm>

namespace cvlg {

namespace {

constexpr double kEarthRadiusM = 6371008.8;
constexpr double kDegToRad = 0.017453292519943295;  // pi / 180

// One WARP per journey (segmented warp scans): the journey's records are consumed 32 at a time
// (coalesced: consecutive slots of a run, or consecutive perm entries on the full-sort path).
// Each lane finds the previous kept record of its own record from a ballot of "kept" lanes
// (shuffle within the chunk, else the carry of the previous chunk), so every step quantity is
// computed in parallel; per-lane partials are reduced at the end. Counts, epoch seconds, maxima
// and dwell (sums of integral seconds) are exact in any order; length_m sums ~1e3 steps in a
// lane-then-tree order (the restatement's sequential order agrees to ~1e-14 relative).
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}

__global__ void __launch_bounds__(256) journey_features_kernel(FeatureParams F) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t n_warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
         j < F.n_journeys; j += n_warps) {
        // carry: the last kept record before the current chunk, the last non-rejected epoch
        bool c_have = false, c_any = false;
        int64_t c_ts = 0, c_any_ts = 0, t_first = 0;
        double c_lat = 0.0, c_lon = 0.0, c_cos = 0.0, c_speed = 0.0;
        bool c_stopped = false;
        uint32_t points = 0, stops = 0;
        double length = 0.0, max_step = 0.0, max_speed = 0.0, max_acc = 0.0, dwell = 0.0;
        int64_t t_last = 0;
        auto chunk = [&](uint32_t slot, bool valid) {
            const uint32_t code = valid ? (F.code[slot] & kCodeMask) : kCodeRejected;
            const bool nonrej = code != kCodeRejected;
            const int64_t t = nonrej ? F.ts[slot] : 0;
            bool dup = false;
            if (F.slow) {  // duplicate (journey, epoch): dropped before filtering (aggregate.cpp:276)
                const uint32_t nb = __ballot_sync(0xFFFFFFFFu, nonrej);
                const uint32_t below = nb & lt;
                const int src = below ? 31 - __clz(below) : lane;
                const int64_t pt = __shfl_sync(0xFFFFFFFFu, t, src);
                dup = nonrej && (below ? pt == t : (c_any && c_any_ts == t));
                if (nb) {
                    c_any_ts = __shfl_sync(0xFFFFFFFFu, t, 31 - __clz(nb));
                    c_any = true;
                }
            }
            const bool kept = nonrej && !dup && code < kCodeFirstSpecial;
            const uint32_t kb = __ballot_sync(0xFFFFFFFFu, kept);
            if (!kb) return;
            double la = 0.0, lo = 0.0, sp = 0.0, cl = 0.0;
            if (kept) {
                la = F.lat[slot];
                lo = F.lon[slot];
                sp = F.speed[slot];
                cl = cos(la * kDegToRad);
            }
            const bool stopped = sp <= F.stop_speed;
            const uint32_t below = kb & lt;
            const int src = below ? 31 - __clz(below) : lane;
            const int64_t pt = __shfl_sync(0xFFFFFFFFu, t, src);
            const double pla = __shfl_sync(0xFFFFFFFFu, la, src), plo = __shfl_sync(0xFFFFFFFFu, lo, src);
            const double pcl = __shfl_sync(0xFFFFFFFFu, cl, src), psp = __shfl_sync(0xFFFFFFFFu, sp, src);
            const bool pst = __shfl_sync(0xFFFFFFFFu, stopped, src);
            if (kept) {
                const bool has_prev = below != 0 || c_have;
                if (has_prev) {
                    const int64_t p_t = below ? pt : c_ts;
                    const double p_la = below ? pla : c_lat, p_lo = below ? plo : c_lon;
                    const double p_cl = below ? pcl : c_cos, p_sp = below ? psp : c_speed;
                    const bool p_st = below ? pst : c_stopped;
                    const double dt = static_cast<double>(t - p_t);
                    const double s1 = sin(0.5 * (la - p_la) * kDegToRad), s2 = sin(0.5 * (lo - p_lo) * kDegToRad);
                    const double a = s1 * s1 + p_cl * cl * s2 * s2;
                    const double step = 2.0 * kEarthRadiusM * asin(sqrt(fmin(1.0, a)));
                    length += step;
                    max_step = fmax(max_step, step);
                    max_acc = fmax(max_acc, fabs(sp - p_sp) / dt);
                    if (stopped && p_st) dwell += dt;
                    if (stopped && !p_st) ++stops;
                } else {
                    t_first = t;
                    if (stopped) ++stops;
                }
                max_speed = fmax(max_speed, sp);
                ++points;
                if (F.cell_min) {
                    const uint64_t tt = code / (F.D * F.RC), d = (code / F.RC) % F.D, rc = code % F.RC;
                    const uint64_t at = (tt * 4 + d) * F.RC + rc;
                    const float f = __double2float_rn(sp);
                    const uint32_t bits = f == 0.0f ? 0u : __float_as_uint(f);  // -0 -> +0
                    atomicMin(&F.cell_min[at], bits);
                    atomicMax(&F.cell_max[at], bits);
                }
            }
            // carry = the chunk's last kept record
            const int hi = 31 - __clz(kb);
            if (!c_have) t_first = __shfl_sync(0xFFFFFFFFu, t, __ffs(kb) - 1);
            c_ts = __shfl_sync(0xFFFFFFFFu, t, hi);
            c_lat = __shfl_sync(0xFFFFFFFFu, la, hi);
            c_lon = __shfl_sync(0xFFFFFFFFu, lo, hi);
            c_cos = __shfl_sync(0xFFFFFFFFu, cl, hi);
            c_speed = __shfl_sync(0xFFFFFFFFu, sp, hi);
            c_stopped = __shfl_sync(0xFFFFFFFFu, stopped, hi);
            c_have = true;
            t_last = c_ts;
        };
        const uint32_t a0 = F.jstart[j], a1 = F.jstart[j + 1];
        if (F.slow) {
            for (uint32_t base = a0; base < a1; base += 32) {
                const uint32_t p = base + lane;
                chunk(p < a1 ? F.perm[p] : 0u, p < a1);
            }
        } else {
            for (uint32_t r = a0; r < a1; ++r) {
                const uint2 run = F.runs[r];
                for (uint32_t base = run.x; base < run.y; base += 32) chunk(base + lane, base + lane < run.y);
            }
        }
        const uint32_t pts = __reduce_add_sync(0xFFFFFFFFu, points);
        const uint32_t stp = __reduce_add_sync(0xFFFFFFFFu, stops);
        length = warp_sum_d(length);
        dwell = warp_sum_d(dwell);
        max_step = warp_max_d(max_step);
        max_speed = warp_max_d(max_speed);
        max_acc = warp_max_d(max_acc);
        if (lane == 0) {
            F.points[j] = pts;
            F.t_first[j] = t_first;
            F.t_last[j] = t_last;
            F.length_m[j] = length;
            F.max_step_m[j] = max_step;
            F.max_speed[j] = max_speed;
            F.max_abs_accel[j] = max_acc;
            F.dwell_s[j] = dwell;
            F.stops[j] = stp;
        }
    }
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
        const unsigned nb = static_cast<unsigned>(std::min<uint64_t>((f.n_journeys + 7) / 8, 148ull * 8));
        journey_features_kernel<<<nb, 256, 0, s>>>(f);
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
