// Threaded in-memory synthetic-day generator, byte-identical to the reference generator
// generate_day (proj/src/synth.cpp:145-181; SynthRng :17-38, journey_seed :44-48,
// step_journey :77-101, generate_journey :103-143). Bench/test input tooling:
// journeys are independent substreams, so they are generated in parallel and concatenated in
// the reference's shard order (journey j -> shard j % n_shards, ascending j).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "parse.cuh"

namespace {

struct Rng {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double gauss(double sigma) {
        double u1;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        const double u2 = uniform();
        return sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
    }
};

struct Cfg {
    uint64_t seed;
    double lat_min, lat_max, lon_min, lon_max, sample_period, mean_duration, speed_min, speed_max,
        heading_sigma;
    int64_t day_start;
};

double wrap_heading(double h) {
    h = std::fmod(h, 360.0);
    if (h < 0.0) h += 360.0;
    return h;
}

double reflect(double x, double lo, double hi, bool& bounced) {
    if (x < lo) {
        x = lo + (lo - x);
        bounced = true;
    }
    if (x > hi) {
        x = hi - (x - hi);
        bounced = true;
    }
    return std::clamp(x, lo, hi);
}

void civil_from_days(int64_t z, int& year, unsigned& month, unsigned& day) {
    z += 719468;
    const int64_t era = (z >= 0 ? z : z - 146096) / 146097;
    const unsigned doe = static_cast<unsigned>(z - era * 146097);
    const unsigned yoe = (doe - doe / 1460 + doe / 36524 - doe / 146096) / 365;
    const int64_t y = static_cast<int64_t>(yoe) + era * 400;
    const unsigned doy = doe - (365 * yoe + yoe / 4 - yoe / 100);
    const unsigned mp = (5 * doy + 2) / 153;
    day = doy - (153 * mp + 2) / 5 + 1;
    month = mp + (mp < 10 ? 3 : -9);
    year = static_cast<int>(y + (month <= 2));
}

// Appends journey `j`'s CSV rows to `out`; returns the row count.
uint64_t gen_journey(uint32_t j, const Cfg& c, std::string& out) {
    Rng mix{c.seed ^ (0xa0761d6478bd642full + j)};
    mix.next();
    Rng rng{mix.next()};
    constexpr double kEdge = 1e-6, kDeg = 4.0e-6;
    double time_sec = rng.uniform(0.0, 86400.0);
    double lat = rng.uniform(c.lat_min + kEdge, c.lat_max - kEdge);
    double lon = rng.uniform(c.lon_min + kEdge, c.lon_max - kEdge);
    double speed = rng.uniform(c.speed_min, c.speed_max);
    double heading = rng.uniform(0.0, 360.0);
    const double duration = c.mean_duration * rng.uniform(0.3, 1.7);
    const uint64_t steps = static_cast<uint64_t>(duration / c.sample_period);
    char id[24];
    std::snprintf(id, sizeof(id), "j%06u", j);
    const double start = time_sec;
    char line[256];
    uint64_t rows = 0;
    for (uint64_t k = 0; k <= steps; ++k) {
        time_sec = start + static_cast<double>(k) * c.sample_period;
        if (time_sec >= 86400.0) break;
        const int64_t epoch = c.day_start + static_cast<int64_t>(time_sec);
        int64_t dn = epoch / 86400;
        if (epoch % 86400 < 0) --dn;
        const int sod = static_cast<int>(epoch - dn * 86400);
        int y;
        unsigned mo, d;
        civil_from_days(dn, y, mo, d);
        const int n = std::snprintf(line, sizeof(line),
                                    "%s,%04d-%02u-%02u %02d:%02d:%02d,%.6f,%.6f,65101,%.2f,%.2f\n",
                                    id, y, mo, d, sod / 3600, (sod / 60) % 60, sod % 60, lat, lon,
                                    speed, heading);
        out.append(line, static_cast<size_t>(n));
        ++rows;
        // step_journey (synth.cpp:77-101)
        const double nh = wrap_heading(heading + rng.gauss(c.heading_sigma));
        const double target = c.speed_min + 0.6 * (c.speed_max - c.speed_min);
        double ns = speed + 0.05 * (target - speed) + rng.gauss(1.5);
        ns = std::clamp(ns, c.speed_min, c.speed_max);
        const double rad = nh * std::numbers::pi / 180.0;
        const double dist = ns * c.sample_period * kDeg;
        double nlat = lat + dist * std::cos(rad);
        double nlon = lon + dist * std::sin(rad);
        bool bl = false, bo = false;
        nlat = reflect(nlat, c.lat_min + kEdge, c.lat_max - kEdge, bl);
        nlon = reflect(nlon, c.lon_min + kEdge, c.lon_max - kEdge, bo);
        double fh = nh;
        if (bl) fh = wrap_heading(180.0 - fh);
        if (bo) fh = wrap_heading(360.0 - fh);
        heading = fh;
        speed = ns;
        lat = nlat;
        lon = nlon;
    }
    return rows;
}

}  // namespace

extern "C" {

// Generates the shards of one synthetic day in memory. On return, shard s occupies
// out[offsets[s], offsets[s+1]) (header line included). Two-phase: call with out == NULL to get
// the total size in *offsets[n_shards] (generation runs once; results are cached per call pair
// via the `scratch` handle). Simpler contract used here: the caller passes a capacity; returns
// -1 if too small (with offsets[n_shards] = required bytes).
int64_t cvlg_synth_day_owned(uint64_t seed, uint32_t n_journeys, uint32_t n_shards,
                             double sample_period, double mean_duration, int32_t day_number,
                             const double* bbox, uint32_t n_threads, uint32_t owner_mod,
                             uint32_t owner_rem, uint8_t* out, uint64_t capacity,
                             uint64_t* offsets, uint64_t* total_rows);

int64_t cvlg_synth_day(uint64_t seed, uint32_t n_journeys, uint32_t n_shards, double sample_period,
                       double mean_duration, int32_t day_number, const double* bbox,
                       uint32_t n_threads, uint8_t* out, uint64_t capacity, uint64_t* offsets,
                       uint64_t* total_rows) {
    return cvlg_synth_day_owned(seed, n_journeys, n_shards, sample_period, mean_duration,
                                day_number, bbox, n_threads, 1, 0, out, capacity, offsets,
                                total_rows);
}

// Same day, restricted to the journeys a multi-GPU rank owns: FNV-1a(id) % owner_mod ==
// owner_rem (ingest.cpp:287-301). Journey j stays in shard j % n_shards.
int64_t cvlg_synth_day_owned(uint64_t seed, uint32_t n_journeys, uint32_t n_shards,
                             double sample_period, double mean_duration, int32_t day_number,
                             const double* bbox, uint32_t n_threads, uint32_t owner_mod,
                             uint32_t owner_rem, uint8_t* out, uint64_t capacity,
                             uint64_t* offsets, uint64_t* total_rows) {
    if (n_shards == 0 || !(sample_period > 0.0) || !offsets) return -2;
    Cfg c;
    c.seed = seed;
    c.lat_min = bbox ? bbox[0] : 36.0;
    c.lat_max = bbox ? bbox[1] : 40.6;
    c.lon_min = bbox ? bbox[2] : -95.8;
    c.lon_max = bbox ? bbox[3] : -89.1;
    c.sample_period = sample_period;
    c.mean_duration = mean_duration;
    c.speed_min = 0.0;
    c.speed_max = 130.0;
    c.heading_sigma = 6.0;
    c.day_start = static_cast<int64_t>(day_number) * 86400;
    const unsigned workers = n_threads ? n_threads : std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::string> text(n_journeys);
    std::vector<uint64_t> rows(n_journeys, 0);
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < workers; ++w)
        pool.emplace_back([&] {
            for (uint32_t j = next.fetch_add(64); j < n_journeys; j = next.fetch_add(64))
                for (uint32_t k = j; k < std::min(n_journeys, j + 64); ++k) {
                    if (owner_mod > 1) {
                        char id[24];
                        const int n = std::snprintf(id, sizeof(id), "j%06u", k);
                        uint64_t h = 1469598103934665603ull;
                        for (int i = 0; i < n; ++i)
                            h = (h ^ static_cast<unsigned char>(id[i])) * 1099511628211ull;
                        if (h % owner_mod != owner_rem) continue;
                    }
                    text[k].reserve(static_cast<size_t>(mean_duration / sample_period * 2.0 * 70));
                    rows[k] = gen_journey(k, c, text[k]);
                }
        });
    for (auto& t : pool) t.join();
    static const char kHeader[] = "Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading\n";
    const uint64_t hlen = sizeof(kHeader) - 1;
    uint64_t total = 0, nrows = 0;
    offsets[0] = 0;
    for (uint32_t s = 0; s < n_shards; ++s) {
        uint64_t sz = hlen;
        for (uint32_t j = s; j < n_journeys; j += n_shards) sz += text[j].size();
        total += sz;
        offsets[s + 1] = total;
    }
    for (uint32_t j = 0; j < n_journeys; ++j) nrows += rows[j];
    if (total_rows) *total_rows = nrows;
    if (!out || capacity < total) return -1;
    // parallel copy per shard
    std::vector<std::thread> cp;
    std::atomic<uint32_t> ns{0};
    for (unsigned w = 0; w < std::min<unsigned>(workers, n_shards); ++w)
        cp.emplace_back([&] {
            for (uint32_t s = ns.fetch_add(1); s < n_shards; s = ns.fetch_add(1)) {
                uint8_t* p = out + offsets[s];
                std::memcpy(p, kHeader, hlen);
                p += hlen;
                for (uint32_t j = s; j < n_journeys; j += n_shards) {
                    std::memcpy(p, text[j].data(), text[j].size());
                    p += text[j].size();
                }
            }
        });
    for (auto& t : cp) t.join();
    return static_cast<int64_t>(total);
}

// The same day written straight to shard files `out_dir/shard_%04u.csv` (generate_day's names,
// synth.cpp:157-160) with one host thread per file at a time: memory stays bounded by one
// journey batch per thread, so c3-sized days (34 GB) never sit in host memory at once.
// Returns the total bytes written, or < 0 (-3: I/O failure).
int64_t cvlg_synth_write_day(uint64_t seed, uint32_t n_journeys, uint32_t n_shards,
                             double sample_period, double mean_duration, int32_t day_number,
                             uint32_t n_threads, const char* out_dir, uint64_t* total_rows) {
    if (n_shards == 0 || !(sample_period > 0.0) || !out_dir) return -2;
    Cfg c;
    c.seed = seed;
    c.lat_min = 36.0;
    c.lat_max = 40.6;
    c.lon_min = -95.8;
    c.lon_max = -89.1;
    c.sample_period = sample_period;
    c.mean_duration = mean_duration;
    c.speed_min = 0.0;
    c.speed_max = 130.0;
    c.heading_sigma = 6.0;
    c.day_start = static_cast<int64_t>(day_number) * 86400;
    static const char kHeader[] = "Journey Id,Timestamp,Latitude,Longitude,Postal Code,Speed,Heading\n";
    const unsigned workers = std::min<unsigned>(
        n_threads ? n_threads : std::max(1u, std::thread::hardware_concurrency()), n_shards);
    std::atomic<uint32_t> next{0};
    std::atomic<uint64_t> rows{0}, bytes{0};
    std::atomic<bool> bad{false};
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < workers; ++w)
        pool.emplace_back([&] {
            std::string buf;
            buf.reserve(72u << 20);
            for (uint32_t s = next.fetch_add(1); s < n_shards && !bad; s = next.fetch_add(1)) {
                char path[4096];
                std::snprintf(path, sizeof(path), "%s/shard_%04u.csv", out_dir, s);
                std::FILE* f = std::fopen(path, "wb");
                if (!f) {
                    bad = true;
                    break;
                }
                buf.assign(kHeader, sizeof(kHeader) - 1);
                uint64_t r = 0, b = 0;
                for (uint32_t j = s; j < n_journeys; j += n_shards) {
                    r += gen_journey(j, c, buf);
                    if (buf.size() > (64u << 20)) {
                        if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) bad = true;
                        b += buf.size();
                        buf.clear();
                    }
                }
                if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) bad = true;
                b += buf.size();
                if (std::fclose(f) != 0) bad = true;
                rows += r;
                bytes += b;
            }
        });
    for (auto& t : pool) t.join();
    if (bad) return -3;
    if (total_rows) *total_rows = rows.load();
    return static_cast<int64_t>(bytes.load());
}

// Adversarial variant of a generated day: every data row of the input shards
// (each shard = header line + rows) shuffled with a seeded Fisher-Yates permutation and dealt
// round-robin to n_out shards, each starting with `header`. Returns bytes written, or < 0.
int64_t cvlg_shuffle_rows(const uint8_t* blob, const uint64_t* offs, uint32_t n_in, uint64_t seed,
                          const char* header, uint32_t n_out, uint8_t* out, uint64_t cap,
                          uint64_t* out_offs) {
    if (!blob || !offs || !out || !out_offs || !header || n_out == 0) return -1;
    std::vector<std::pair<uint64_t, uint32_t>> rows;  // (offset, length without '\n')
    for (uint32_t s = 0; s < n_in; ++s) {
        uint64_t p = offs[s];
        const uint64_t e = offs[s + 1];
        while (p < e && blob[p] != '\n') ++p;  // skip the header line
        ++p;
        while (p < e) {
            uint64_t q = p;
            while (q < e && blob[q] != '\n') ++q;
            if (q > p) rows.emplace_back(p, static_cast<uint32_t>(q - p));
            p = q + 1;
        }
    }
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 0x2545F4914F6CDD1Dull;
    for (uint64_t i = rows.size(); i > 1; --i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        std::swap(rows[i - 1], rows[x % i]);
    }
    const uint64_t hl = std::strlen(header);
    uint64_t w = 0;
    for (uint32_t o = 0; o < n_out; ++o) {
        out_offs[o] = w;
        if (w + hl + 1 > cap) return -2;
        std::memcpy(out + w, header, hl);
        w += hl;
        out[w++] = '\n';
        for (uint64_t i = o; i < rows.size(); i += n_out) {
            const auto& r = rows[i];
            if (w + r.second + 1 > cap) return -2;
            std::memcpy(out + w, blob + r.first, r.second);
            w += r.second;
            out[w++] = '\n';
        }
    }
    out_offs[n_out] = w;
    return static_cast<int64_t>(w);
}

}  // extern "C"
