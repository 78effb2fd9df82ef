// TEST INFRASTRUCTURE: compiles the product's device decode headers (parse.cuh, grid.cuh) for
// the host so their exact logic can be fuzzed on CPU against the reference (oracle/_ref) without
// a GPU. The GPU tests then confirm the sm_100a build of the same code agrees.
#include <cstdint>
#include <cstring>

#include "../../paper_2305_07454_b200/csrc/grid.cuh"
#include "../../paper_2305_07454_b200/csrc/parse.cuh"

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
    return cvlg::cell_code(epoch, lat, lon, speed, heading, g);
}

uint32_t hp_extent_bins(double lo, double hi, double step) { return cvlg::extent_bins(lo, hi, step); }

}  // extern "C"
