// Filter + spatio-temporal binning, restated from the reference:
//   snap_to_integer   proj/src/grid.cpp:10-14
//   extent_bins       proj/src/grid.cpp:18-22   (host side: grid dims)
//   linear_bin        proj/src/grid.cpp:26-36
//   time_bin          proj/src/grid.cpp:69-71 (+ Timestamp::minute_of_day datetime.cpp:97-107)
//   dxn_bin           proj/src/grid.cpp:73-81
//   global_index      proj/src/grid.cpp:83-90
//   filter_reason     proj/src/aggregate.cpp:48-56
// All arithmetic is IEEE binary64 with explicit round-to-nearest intrinsics on the device so
// no FMA contraction can change a bin edge.
#pragma once
#include "parse.cuh"

namespace cvlg {

// Per-record cell code (31 bits; bit 31 of the slot word is the run-head flag).
// Values >= kCodeFirstSpecial are not cells, so grids must have < 2^31 - 16 cells.
enum : uint32_t {
    kCodeOutOfGrid = 0x7FFFFFFFu,     // filtered: OutOfGrid
    kCodeSpeedCeiling = 0x7FFFFFFEu,  // filtered: SpeedCeiling
    kCodeMissingField = 0x7FFFFFFDu,  // filtered: MissingField (empty id; unreachable after parse)
    kCodeUnbinnable = 0x7FFFFFFCu,    // require_in_grid=false and off-grid: OutOfBounds if kept
    kCodeRejected = 0x7FFFFFFBu,      // data line rejected by parse (counted in decode)
    kCodeFirstSpecial = 0x7FFFFFF0u,
};

struct GridParams {
    double lat_min, lat_max, lon_min, lon_max, lat_step, lon_step, dxn_offset, dxn_step_d;
    double speed_ceiling;
    uint32_t min_step, dxn_step, R, C, D, T;
    int32_t require_in_grid, drop_missing;
    uint32_t t_magic;  // ceil(2^32 / min_step) (min_step > 1): minute / min_step = umulhi(minute, t_magic)
    double inv_lat_step, inv_lon_step, inv_dxn_step;  // RN(1 / step): the binning fast path
};

// RN(1 / step) for the binning fast path (host side, once per run)
inline void set_inverse_steps(GridParams& g) {
    g.inv_lat_step = 1.0 / g.lat_step;
    g.inv_lon_step = 1.0 / g.lon_step;
    g.inv_dxn_step = 1.0 / g.dxn_step_d;
}

// ceil(2^32 / min_step): exact quotient for every minute of day (minute * min_step < 2^32 / 2^11)
inline uint32_t time_magic(uint32_t min_step) {
    return min_step > 1 ? static_cast<uint32_t>(((1ull << 32) + min_step - 1) / min_step) : 0u;
}

// time_bin from the minute of day (0..1439) of the parsed timestamp (grid.cpp:69-71)
CVLG_HD uint32_t time_bin_mod(uint32_t minute, const GridParams& g) {
    if (g.min_step <= 1) return minute;
#if defined(__CUDA_ARCH__)
    return __umulhi(minute, g.t_magic);
#else
    return static_cast<uint32_t>((static_cast<uint64_t>(minute) * g.t_magic) >> 32);
#endif
}

CVLG_HD double d_abs(double x) { return bits_dbl(dbl_bits(x) & 0x7FFFFFFFFFFFFFFFull); }

CVLG_HD double d_rint(double x) {
#if defined(__CUDA_ARCH__)
    return rint(x);
#else
    return nearbyint(x);
#endif
}

CVLG_HD double snap_to_integer(double q) {
    const double r = d_rint(q);
    const double ar = d_abs(r);
    const double m = ar > 1.0 ? ar : 1.0;  // fmax(1, |r|); r is never NaN here
    if (d_abs(d_sub(q, r)) <= d_mul(1e-9, m)) return r;
    return q;
}

CVLG_HD uint32_t extent_bins(double lo, double hi, double step) {
    const double q = snap_to_integer(d_div(d_sub(hi, lo), step));
    const double n = ceil(q);
    return n < 1.0 ? 1u : static_cast<uint32_t>(n);
}

// floor(snap_to_integer(d / step)) for d >= 0, computed first as qa = RN(d * RN(1/step)).
// |qa - RN(d / step)| <= 3 * 2^-53 * (d / step) (< 3.4e-10 for quotients below 1e6), so when qa is
// more than 4e-9 * max(1, |rint(qa)|) from every integer, no integer lies between qa and the
// exact quotient and snap_to_integer (tolerance 1e-9 * max(1, |r|)) leaves the quotient alone:
// floor(qa) is the exact bin. Otherwise (near a bin edge, or huge quotients) the exact division
// and snap of grid.cpp decide.
CVLG_HD double snapped_floor(double d, double step, double inv) {
    const double qa = d_mul(d, inv);
    const double r = d_rint(qa);
    const double ar = d_abs(r);
    const double m = ar > 1.0 ? ar : 1.0;
    if (qa < 1e6 && d_abs(d_sub(qa, r)) > d_mul(4e-9, m)) return floor(qa);
    return floor(snap_to_integer(d_div(d, step)));
}

// precondition: lo <= x <= hi (checked by the caller)
CVLG_HD uint32_t linear_bin(double x, double lo, double step, uint32_t n) {
    const double q = snap_to_integer(d_div(d_sub(x, lo), step));
    double b = floor(q);
    if (b < 0.0) b = 0.0;
    const double last = static_cast<double>(n - 1);
    if (b > last) b = last;
    return static_cast<uint32_t>(b);
}

CVLG_HD uint32_t linear_bin_fast(double x, double lo, double step, double inv, uint32_t n) {
    double b = snapped_floor(d_sub(x, lo), step, inv);
    if (b < 0.0) b = 0.0;
    const double last = static_cast<double>(n - 1);
    if (b > last) b = last;
    return static_cast<uint32_t>(b);
}

CVLG_HD uint32_t time_bin(int64_t epoch, uint32_t min_step) {
    int64_t day = epoch / 86400;
    if (epoch % 86400 < 0) --day;
    const int64_t sod = epoch - day * 86400;
    return static_cast<uint32_t>(sod / 60) / min_step;
}

CVLG_HD double d_fmod360(double h) {
    if (h >= 0.0 && h < 360.0) return h;  // fmod(h, 360) == h exactly in this range
    return fmod(h, 360.0);
}

CVLG_HD uint32_t dxn_bin(double heading, const GridParams& g) {
    double h = d_add(heading, g.dxn_offset);
    h = d_fmod360(h);
    if (h < 0.0) h = d_add(h, 360.0);
    const uint32_t d = static_cast<uint32_t>(snapped_floor(h, g.dxn_step_d, g.inv_dxn_step));
    return d >= g.D ? d - g.D : d;  // == d % D: h <= 360 so q <= 360 / dxn_step = D
}

// filter_reason + binning for one accepted record with time bin t -> cell code.
CVLG_HD uint32_t cell_code_t(uint32_t t, double lat, double lon, double speed, double heading,
                             const GridParams& g) {
    const bool in_grid = lat >= g.lat_min && lat <= g.lat_max && lon >= g.lon_min && lon <= g.lon_max;
    if (g.require_in_grid && !in_grid) return kCodeOutOfGrid;
    if (speed > g.speed_ceiling) return kCodeSpeedCeiling;
    if (!in_grid) return kCodeUnbinnable;
    const uint32_t d = dxn_bin(heading, g);
    const uint32_t r = linear_bin_fast(lat, g.lat_min, g.lat_step, g.inv_lat_step, g.R);
    const uint32_t c = linear_bin_fast(lon, g.lon_min, g.lon_step, g.inv_lon_step, g.C);
    return ((t * g.D + d) * g.R + r) * g.C + c;
}

CVLG_HD uint32_t cell_code(int64_t epoch, double lat, double lon, double speed, double heading,
                           const GridParams& g) {
    return cell_code_t(time_bin(epoch, g.min_step), lat, lon, speed, heading, g);
}

}  // namespace cvlg
