// TEST INFRASTRUCTURE: compiles the product's device decode headers (parse.cuh, grid.cuh) for
// the host so their exact logic can be fuzzed on CPU against the reference (oracle/_ref) without
// a GPU. The GPU tests then confirm the sm_100a build of the same code agrees.
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../paper_2305_07454_b200/csrc/grid.cuh"
#include "../../paper_2305_07454_b200/csrc/parse.cuh"
#include "../../paper_2305_07454_b200/csrc/fastparse.cuh"

extern "C" {

struct hp_record {
    int64_t epoch_sec;
    double latitude, longitude, speed, heading;
    int32_t id_begin, id_len, postal_begin, postal_len;
};

// returns -1 when accepted, else the reference ParseReason ordinal (records.hpp:34-40)
int hp_parse_record(const char* line, int32_t len, const int32_t* cols, hp_record* out) {
    cvlg::ColumnMap m;
    std::memcpy(&m, cols, sizeof(m));
    cvlg::Parsed p;
    const uint8_t why = cvlg::parse_line(reinterpret_cast<const uint8_t*>(line), len, m, p);
    if (why != cvlg::kAccepted) return why - 1;
    if (out) {
        out->epoch_sec = p.epoch;
        out->latitude = p.lat;
        out->longitude = p.lon;
        out->speed = p.speed;
        out->heading = p.heading;
        out->id_begin = p.id_begin;
        out->id_len = p.id_len;
        out->postal_begin = p.postal_begin;
        out->postal_len = p.postal_len;
    }
    return -1;
}

int hp_parse_header(const char* line, int32_t len, int32_t* cols) {
    cvlg::ColumnMap m;
    const bool ok = cvlg::parse_header(reinterpret_cast<const uint8_t*>(line), len, m);
    std::memcpy(cols, &m, sizeof(m));
    return ok ? 1 : 0;
}

// 1 = accepted (value in *out), 0 = BadNumeric
int hp_parse_double(const char* s, int32_t len, double* out) {
    double v = 0;
    const bool ok = cvlg::parse_double(reinterpret_cast<const uint8_t*>(s), len, v);
    if (ok) *out = v;
    return ok ? 1 : 0;
}

int hp_parse_timestamp(const char* s, int32_t len, int64_t* out) {
    int64_t v = 0;
    const bool ok = cvlg::parse_timestamp(reinterpret_cast<const uint8_t*>(s), len, v);
    if (ok) *out = v;
    return ok ? 1 : 0;
}

// grid: lat_min, lat_max, lon_min, lon_max, lat_step, lon_step, dxn_offset; ints: min_step,
// dxn_step; rules: require_in_grid, speed_ceiling
uint32_t hp_cell_code(const double* gd, const uint32_t* gi, int32_t require_in_grid,
                      double speed_ceiling, int64_t epoch, double lat, double lon, double speed,
                      double heading) {
    cvlg::GridParams g;
    g.lat_min = gd[0];
    g.lat_max = gd[1];
    g.lon_min = gd[2];
    g.lon_max = gd[3];
    g.lat_step = gd[4];
    g.lon_step = gd[5];
    g.dxn_offset = gd[6];
    g.min_step = gi[0];
    g.dxn_step = gi[1];
    g.dxn_step_d = static_cast<double>(gi[1]);
    g.R = cvlg::extent_bins(g.lat_min, g.lat_max, g.lat_step);
    g.C = cvlg::extent_bins(g.lon_min, g.lon_max, g.lon_step);
    g.D = 360 / gi[1];
    g.T = 1440 / gi[0];
    g.require_in_grid = require_in_grid;
    g.drop_missing = 1;
    g.speed_ceiling = speed_ceiling;
    g.t_magic = cvlg::time_magic(g.min_step);
    cvlg::set_inverse_steps(g);
    return cvlg::cell_code(epoch, lat, lon, speed, heading, g);
}

uint32_t hp_extent_bins(double lo, double hi, double step) { return cvlg::extent_bins(lo, hi, step); }

// binning fast path (snapped_floor) against the exact division + snap, over random quotients
// concentrated around bin edges, for the given steps; returns mismatches
uint64_t hp_fuzz_snapped_floor(uint64_t seed, uint64_t count, const double* steps, int n_steps) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 11;
    auto rnd = [&]() {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return x;
    };
    uint64_t bad = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const double step = steps[rnd() % n_steps];
        const double inv = 1.0 / step;
        const double k = static_cast<double>(rnd() % 5000);
        double d;
        switch (rnd() % 4) {
            case 0: d = k * step; break;                                     // on an edge
            case 1: d = k * step + (static_cast<double>(rnd() % 2001) - 1000.0) * 1e-12; break;
            case 2: d = k * step * (1.0 + (static_cast<double>(rnd() % 2001) - 1000.0) * 1e-15); break;
            default: d = (static_cast<double>(rnd() >> 11) / 9007199254740992.0) * 5000.0 * step;
        }
        if (d < 0) d = 0;
        const double fast = cvlg::snapped_floor(d, step, inv);
        const double exact = floor(cvlg::snap_to_integer(d / step));
        if (fast != exact) ++bad;
    }
    return bad;
}

// ---- K1 fast path (fastparse.cuh) -------------------------------------------------------------
// The field is placed at buffer offset 40 + shift (shift 0..3 exercises every word alignment),
// preceded by `pre` (the previous field's bytes) and followed by ','. Returns 1 and the value
// when the fast path decides, 0 when it defers to the general parser.
static int fast_number_at(const char* s, int32_t len, int shift, int qguess, const char* pre, double* out) {
    if (len > 64) return 0;  // the fast path only takes fields of <= 12 bytes
    alignas(16) uint8_t buf[128];
    std::memset(buf, 'x', sizeof(buf));
    const int at = 40 + shift;
    const int pl = static_cast<int>(std::strlen(pre));
    std::memcpy(buf + at - pl, pre, pl);
    std::memcpy(buf + at, s, len);
    buf[at + len] = ',';
    int q = qguess;
    double v = 0;
    const bool ok = cvlg::fast_number(reinterpret_cast<const uint32_t*>(buf), buf, at, at + len, q, v);
    if (ok) *out = v;
    return ok ? 1 : 0;
}

int hp_fast_number(const char* s, int32_t len, int shift, int qguess, double* out) {
    return fast_number_at(s, len, shift, qguess, "-37.5,", out);
}

// 1 + minute of day in *minute when the fast path decides, 0 otherwise. `cache` (3 words + day)
// starts at 1970-01-01 when null.
int hp_fast_timestamp(const char* s, int32_t len, int shift, int64_t* ts, uint32_t* minute) {
    if (len != 19) return 0;
    alignas(16) uint8_t buf[96];
    std::memset(buf, ',', sizeof(buf));
    std::memcpy(buf + 32 + shift, s, len);
    static thread_local cvlg::DateCache dc;
    int64_t t = 0;
    uint32_t m = 0;
    const bool ok = cvlg::fast_timestamp(reinterpret_cast<const uint32_t*>(buf), 32 + shift, dc, t, m);
    if (ok) {
        *ts = t;
        *minute = m;
    }
    return ok ? 1 : 0;
}

uint32_t hp_time_bin_mod(uint32_t minute, uint32_t min_step) {
    cvlg::GridParams g;
    g.min_step = min_step;
    g.t_magic = cvlg::time_magic(min_step);
    return cvlg::time_bin_mod(minute, g);
}

uint32_t hp_time_bin(int64_t epoch, uint32_t min_step) { return cvlg::time_bin(epoch, min_step); }

// x / 10^k through the fast path's Markstein division (k in 1..8)
double hp_div_pow10(double x, int k) { return cvlg::div_pow10(x, k); }

// class_masks32 over random 32-byte blocks (biased towards '\n', ',' and bytes differing from
// them in one bit) against a byte loop; returns the number of mismatching blocks
uint64_t hp_check_class_masks(uint64_t seed, uint64_t count) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 3;
    auto rnd = [&]() {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return x;
    };
    const uint8_t pool[] = {'\n', ',', 0x0B, 0x08, 0x2D, 0x2E, 0x8A, 0xAC, 0x0A ^ 0x80, 0x00, 0xFF, 'a', '0', '9', 0x7F, 0x80};
    uint64_t bad = 0;
    for (uint64_t it = 0; it < count; ++it) {
        uint8_t b[32];
        for (int i = 0; i < 32; ++i) b[i] = (rnd() % 3) ? pool[rnd() % sizeof(pool)] : static_cast<uint8_t>(rnd());
        uint32_t w[8];
        std::memcpy(w, b, 32);
        uint32_t mn = 0, mc = 0, en = 0, ec = 0;
        cvlg::class_masks32(w, mn, mc);
        for (int i = 0; i < 32; ++i) {
            if (b[i] == '\n') en |= 1u << i;
            if (b[i] == ',') ec |= 1u << i;
        }
        if (mn != en || mc != ec) ++bad;
    }
    return bad;
}

// Bulk differential fuzz of fast_number against parse_double over random numeric strings
// (shapes: [-]I.F with I 0..4 digits, F 0..9 digits, integers, junk bytes, '.', '-', '+',
// spaces, exponents). Counts cases where the fast path decided; returns the number of
// disagreements (fast accepted but the value or acceptance differs) and copies the first one.
uint64_t hp_fuzz_fast_number(uint64_t seed, uint64_t count, uint64_t* decided, char* first_bad) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    auto rnd = [&]() {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return x;
    };
    const char junk[] = "0123456789.-+ eE\tx,";
    uint64_t bad = 0, dec = 0;
    char s[32];
    for (uint64_t i = 0; i < count; ++i) {
        int n = 0;
        const uint64_t r = rnd();
        const int shape = r % 8;
        if (shape < 5) {  // [-]I.F
            if (rnd() % 3 == 0) s[n++] = '-';
            const int I = rnd() % 5, F = rnd() % 10;
            for (int k = 0; k < I; ++k) s[n++] = '0' + rnd() % 10;
            if (shape != 4) s[n++] = '.';
            for (int k = 0; k < F; ++k) s[n++] = '0' + rnd() % 10;
        } else {  // junk-ish
            const int L = 1 + rnd() % 13;
            for (int k = 0; k < L; ++k) s[n++] = junk[rnd() % (sizeof(junk) - 1)];
        }
        if (n == 0) continue;
        s[n] = 0;
        double vf = 0, vg = 0;
        const int qg = static_cast<int>(rnd() % 10) - 1;
        const int f = fast_number_at(s, n, static_cast<int>(rnd() % 4), qg == 0 ? -1 : qg + 3, "12.5,", &vf);
        if (!f) continue;
        ++dec;
        const bool g = cvlg::parse_double(reinterpret_cast<const uint8_t*>(s), n, vg);
        if (!g || cvlg::dbl_bits(vf) != cvlg::dbl_bits(vg)) {
            if (!bad) std::memcpy(first_bad, s, n + 1);
            ++bad;
        }
    }
    *decided = dec;
    return bad;
}

// Bulk differential fuzz of fast_timestamp against parse_timestamp: random valid and corrupted
// timestamps across years 0000..9999, month/day edges (leap years), and hour/minute/second edges.
uint64_t hp_fuzz_fast_timestamp(uint64_t seed, uint64_t count, uint64_t* decided, char* first_bad) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 7;
    auto rnd = [&]() {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return x;
    };
    uint64_t bad = 0, dec = 0;
    char s[24];
    cvlg::DateCache dc;
    for (uint64_t i = 0; i < count; ++i) {
        const int y = (rnd() % 4 == 0) ? static_cast<int>(rnd() % 10000) : 1995 + static_cast<int>(rnd() % 40);
        const int mo = static_cast<int>(rnd() % 14), d = static_cast<int>(rnd() % 33);
        const int h = static_cast<int>(rnd() % 26), mi = static_cast<int>(rnd() % 62), se = static_cast<int>(rnd() % 62);
        std::snprintf(s, sizeof(s), "%04d-%02d-%02d %02d:%02d:%02d", y, mo, d, h, mi, se);
        if (rnd() % 8 == 0) s[rnd() % 19] = "0123456789-: xT/"[rnd() % 16];
        alignas(16) uint8_t buf[96];
        std::memset(buf, ',', sizeof(buf));
        const int at = 32 + static_cast<int>(rnd() % 4);
        std::memcpy(buf + at, s, 19);
        int64_t tf = 0, tg = 0;
        uint32_t mf = 0;
        if (!cvlg::fast_timestamp(reinterpret_cast<const uint32_t*>(buf), at, dc, tf, mf)) continue;
        ++dec;
        const bool g = cvlg::parse_timestamp(reinterpret_cast<const uint8_t*>(s), 19, tg);
        int64_t day = tg / 86400;
        if (tg % 86400 < 0) --day;
        const int64_t mod = (tg - day * 86400) / 60;
        if (!g || tf != tg || static_cast<int64_t>(mf) != mod) {
            if (!bad) std::memcpy(first_bad, s, 20);
            ++bad;
        }
    }
    *decided = dec;
    return bad;
}


// fast_number_hit (the cached-shape path of K1) against parse_double: same string shapes as
// hp_fuzz_fast_number; the cached point index is the true one (right-aligned window) half of
// the time, random otherwise. Returns disagreements (hit accepted, value or acceptance differs).
uint64_t hp_fuzz_fast_number_hit(uint64_t seed, uint64_t count, uint64_t* decided, char* first_bad) {
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 5;
    auto rnd = [&]() {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        return x;
    };
    const char junk[] = "0123456789.-+ eE\tx,";
    uint64_t bad = 0, dec = 0;
    char s[32];
    for (uint64_t i = 0; i < count; ++i) {
        int n = 0;
        const uint64_t r = rnd();
        const int shape = r % 8;
        if (shape < 5) {
            if (rnd() % 3 == 0) s[n++] = '-';
            const int I = rnd() % 5, F = rnd() % 10;
            for (int k = 0; k < I; ++k) s[n++] = '0' + rnd() % 10;
            if (shape != 4) s[n++] = '.';
            for (int k = 0; k < F; ++k) s[n++] = '0' + rnd() % 10;
        } else {
            const int L = 1 + rnd() % 13;
            for (int k = 0; k < L; ++k) s[n++] = junk[rnd() % (sizeof(junk) - 1)];
        }
        if (n == 0) continue;
        s[n] = 0;
        int q = static_cast<int>(rnd() % 14) - 1;
        if (rnd() & 1) {
            const char* d = static_cast<const char*>(std::memchr(s, '.', n));
            q = d ? 12 - (n - static_cast<int>(d - s)) : -1;
        }
        alignas(16) uint8_t buf[128];
        std::memset(buf, 'x', sizeof(buf));
        const int at = 40 + static_cast<int>(rnd() % 4);
        std::memcpy(buf + at - 5, "12.5,", 5);
        std::memcpy(buf + at, s, n);
        buf[at + n] = ',';
        double vf = 0, vg = 0;
        if (!cvlg::fast_number_hit(reinterpret_cast<const uint32_t*>(buf), buf, at, at + n, q, vf)) continue;
        ++dec;
        const bool g = cvlg::parse_double(reinterpret_cast<const uint8_t*>(s), n, vg);
        if (!g || cvlg::dbl_bits(vf) != cvlg::dbl_bits(vg)) {
            if (!bad) std::memcpy(first_bad, s, n + 1);
            ++bad;
        }
    }
    *decided = dec;
    return bad;
}

}  // extern "C"
