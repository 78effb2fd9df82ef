// Record decode primitives shared by the sm_100a decode kernel and (compiled for the host) by the
// CPU-side conformance harness in tests/native. Everything here is a from-scratch restatement of
// the reference's decode semantics:
//   trim / split_fields        proj/src/ingest.cpp:31-53
//   parse_header/normalize     proj/src/ingest.cpp:56-64, 97-115
//   parse_double (from_chars)  proj/src/ingest.cpp:66-72  (libstdc++ 13 std::from_chars(double),
//                              i.e. the fast_float grammar + correctly rounded result, with
//                              ERANGE reported for non-zero inputs rounding to 0 and for +-inf)
//   Timestamp::parse           proj/src/datetime.cpp:53-75, days_from_civil :10-17
//   parse_record_impl          proj/src/ingest.cpp:119-157
// Decimal->binary conversion: exact Clinger fast path, else an exact big-integer comparison
// against the halfway points of candidate doubles (slow path; never taken by %.6f/%.2f data).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CVLG_HD __host__ __device__ __forceinline__
#define CVLG_HD_NOINLINE static __host__ __device__ __noinline__
#else
#define CVLG_HD static inline
#define CVLG_HD_NOINLINE static
#endif

#if !defined(__CUDA_ARCH__)
#include <math.h>
#include <string.h>
#endif

namespace cvlg {

// Parse outcome codes. kAccepted = 0; the rest are ParseReason ordinal + 1
// (records.hpp:34-40: BadTimestamp, BadNumeric, MissingField, RangeViolation, BadHeader).
enum : uint8_t {
    kAccepted = 0,
    kBadTimestamp = 1,
    kBadNumeric = 2,
    kMissingField = 3,
    kRangeViolation = 4,
};

// Column indices resolved from a shard header (ingest.hpp:18-32).
struct ColumnMap {
    int32_t journey_id, timestamp, latitude, longitude, postal_code, speed, heading, n_columns;
};

CVLG_HD bool is_digit(uint8_t c) { return static_cast<uint8_t>(c - '0') < 10; }
CVLG_HD bool is_trim(uint8_t c) { return c == ' ' || c == '\t' || c == '\r'; }

// ---------------------------------------------------------------------------------------------
// IEEE helpers that behave identically on host and device.
CVLG_HD uint64_t dbl_bits(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
CVLG_HD double bits_dbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
CVLG_HD double d_div(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
CVLG_HD double d_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
CVLG_HD double d_add(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
CVLG_HD double d_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}

// Exact powers of ten representable in binary64 (10^0 .. 10^22).
CVLG_HD double exact_pow10(int k) {
    double p = 1.0;
    // small loop (k <= 22): exact at every step since all intermediate values are exact
    double base = 10.0;
    while (k) {
        if (k & 1) p = d_mul(p, base);
        base = d_mul(base, base);
        k >>= 1;
    }
    return p;
}

// ---------------------------------------------------------------------------------------------
// Timestamp (datetime.cpp:10-17, 34-40, 53-75)
CVLG_HD int64_t days_from_civil(int y, unsigned m, unsigned d) {
    y -= m <= 2;
    const int64_t era = (y >= 0 ? y : y - 399) / 400;
    const unsigned yoe = static_cast<unsigned>(y - era * 400);
    const unsigned doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
    const unsigned doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
    return era * 146097 + static_cast<int64_t>(doe) - 719468;
}

CVLG_HD unsigned days_in_month(int y, unsigned m) {
    const bool leap = (y % 4 == 0) && (y % 100 != 0 || y % 400 == 0);
    if (m == 2) return leap ? 29u : 28u;
    return (m == 4 || m == 6 || m == 9 || m == 11) ? 30u : 31u;
}

CVLG_HD int two_digits(const uint8_t* s, bool& ok) {
    ok = ok && is_digit(s[0]) && is_digit(s[1]);
    return (s[0] - '0') * 10 + (s[1] - '0');
}

// Exact "YYYY-MM-DD HH:MM:SS" (19 bytes) -> epoch seconds (naive local).
CVLG_HD bool parse_timestamp(const uint8_t* s, int n, int64_t& out) {
    if (n != 19 || s[4] != '-' || s[7] != '-' || s[10] != ' ' || s[13] != ':' || s[16] != ':')
        return false;
    bool ok = true;
    const int y = two_digits(s, ok) * 100 + two_digits(s + 2, ok);
    const int mo = two_digits(s + 5, ok);
    const int d = two_digits(s + 8, ok);
    const int h = two_digits(s + 11, ok);
    const int mi = two_digits(s + 14, ok);
    const int sec = two_digits(s + 17, ok);
    if (!ok) return false;
    if (mo < 1 || mo > 12) return false;
    if (d < 1 || d > static_cast<int>(days_in_month(y, static_cast<unsigned>(mo)))) return false;
    if (h > 23 || mi > 59 || sec > 59) return false;
    const int64_t days = days_from_civil(y, static_cast<unsigned>(mo), static_cast<unsigned>(d));
    out = days * 86400 + h * 3600 + mi * 60 + sec;
    return true;
}

// ---------------------------------------------------------------------------------------------
// Exact big-integer slow path for decimal -> binary64 (correct rounding, ties-to-even).
// Only reached when the Clinger fast path cannot prove exactness (> 15-16 significant digits,
// |exponent| > 22, subnormals, overflow/underflow candidates).
struct BigInt {
    static constexpr int kLimbs = 128;  // 4096 bits: enough for 800 digits * 5^1142 scalings
    uint32_t limb[kLimbs];
    int n;  // used limbs
};

CVLG_HD void big_set(BigInt& a, uint64_t v) {
    a.limb[0] = static_cast<uint32_t>(v);
    a.limb[1] = static_cast<uint32_t>(v >> 32);
    a.n = a.limb[1] ? 2 : (a.limb[0] ? 1 : 0);
}

CVLG_HD void big_mul_add(BigInt& a, uint32_t m, uint32_t add) {
    uint64_t carry = add;
    for (int i = 0; i < a.n; ++i) {
        const uint64_t t = static_cast<uint64_t>(a.limb[i]) * m + carry;
        a.limb[i] = static_cast<uint32_t>(t);
        carry = t >> 32;
    }
    if (carry && a.n < BigInt::kLimbs) a.limb[a.n++] = static_cast<uint32_t>(carry);
}

CVLG_HD void big_mul_pow5(BigInt& a, int k) {
    while (k >= 13) {
        big_mul_add(a, 1220703125u, 0);  // 5^13
        k -= 13;
    }
    uint32_t m = 1;
    while (k-- > 0) m *= 5;
    if (m != 1) big_mul_add(a, m, 0);
}

CVLG_HD void big_shl(BigInt& a, int s) {
    if (a.n == 0 || s == 0) return;
    const int words = s >> 5, bits = s & 31;
    int n = a.n + words + 1;
    if (n > BigInt::kLimbs) n = BigInt::kLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int src = i - words;
        uint32_t hi = (src >= 0 && src < a.n) ? a.limb[src] : 0;
        uint32_t lo = (src - 1 >= 0 && src - 1 < a.n) ? a.limb[src - 1] : 0;
        a.limb[i] = bits ? ((hi << bits) | (lo >> (32 - bits))) : hi;
    }
    a.n = n;
    while (a.n > 0 && a.limb[a.n - 1] == 0) --a.n;
}

CVLG_HD int big_cmp(const BigInt& a, const BigInt& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.limb[i] != b.limb[i]) return a.limb[i] < b.limb[i] ? -1 : 1;
    return 0;
}

// Significant-digit view of a validated decimal: digits come from the integer span then the
// fraction span, with leading zeros removed. value = 0.d1d2...dn * 10^(lead+1)
struct DecimalDigits {
    const uint8_t* ip;
    int ilen;
    const uint8_t* fp;
    int flen;
    int64_t exp10;  // explicit exponent
};

// compare D = digits(dd) vs H * 2^k, H < 2^55. Returns -1/0/1. `sticky` means D has extra
// non-zero digits beyond those folded in (strictly greater than the folded value).
CVLG_HD_NOINLINE int cmp_decimal_halfway(const uint8_t* digs, int nd, int64_t p, bool sticky,
                                          uint64_t H, int64_t k) {
    BigInt A, B;
    big_set(A, 0);
    A.n = 0;
    // A = d (nd digits, 9 at a time)
    int i = 0;
    while (i < nd) {
        uint32_t chunk = 0, mul = 1;
        int take = nd - i < 9 ? nd - i : 9;
        for (int t = 0; t < take; ++t) {
            chunk = chunk * 10 + (digs[i + t] - '0');
            mul *= 10;
        }
        if (A.n == 0) {
            big_set(A, chunk);
        } else {
            big_mul_add(A, mul, chunk);
        }
        i += take;
    }
    big_set(B, H);
    if (p >= 0) {
        big_mul_pow5(A, static_cast<int>(p));
        const int64_t s = p - k;
        if (s >= 0) big_shl(A, static_cast<int>(s));
        else big_shl(B, static_cast<int>(-s));
    } else {
        big_mul_pow5(B, static_cast<int>(-p));
        const int64_t s = k - p;
        if (s >= 0) big_shl(B, static_cast<int>(s));
        else big_shl(A, static_cast<int>(-s));
    }
    int c = big_cmp(A, B);
    if (c == 0 && sticky) c = 1;
    return c;
}

// Decompose a positive finite double into M * 2^E (M integer incl. hidden bit).
CVLG_HD void dbl_decompose(double x, uint64_t& M, int64_t& E) {
    const uint64_t u = dbl_bits(x);
    const int be = static_cast<int>((u >> 52) & 0x7FF);
    const uint64_t frac = u & ((1ull << 52) - 1);
    if (be == 0) {
        M = frac;
        E = -1074;
    } else {
        M = frac | (1ull << 52);
        E = be - 1075;
    }
}

// Correctly rounded positive value of the significant digits `digs` (nd <= kMaxDigits, leading
// digit non-zero) times 10^p; `sticky` = more non-zero digits were dropped. Returns +inf on
// overflow and 0.0 on underflow.
CVLG_HD_NOINLINE double slow_decimal_to_double(const uint8_t* digs, int nd, int64_t p, bool sticky) {
    const int64_t lead = p + nd - 1;
    if (lead < -325) return 0.0;
    if (lead > 309) return bits_dbl(0x7FF0000000000000ull);
    // approximate: first up to 19 digits
    uint64_t w = 0;
    int take = nd < 19 ? nd : 19;
    for (int i = 0; i < take; ++i) w = w * 10 + (digs[i] - '0');
    int64_t q = p + (nd - take);
    double approx = static_cast<double>(w);
    // scale by 10^q in steps that stay within range
    while (q > 0) {
        const int s = q > 22 ? 22 : static_cast<int>(q);
        approx = d_mul(approx, exact_pow10(s));
        q -= s;
    }
    while (q < 0) {
        const int s = q < -22 ? 22 : static_cast<int>(-q);
        approx = d_div(approx, exact_pow10(s));
        q += s;
    }
    uint64_t ub = dbl_bits(approx);
    if (ub >= 0x7FF0000000000000ull) ub = 0x7FEFFFFFFFFFFFFFull;  // DBL_MAX
    if (ub == 0) ub = 1;                                           // min subnormal
    for (int iter = 0; iter < 4096; ++iter) {
        uint64_t M;
        int64_t E;
        dbl_decompose(bits_dbl(ub), M, E);
        // halfway to the next double up: (2M+1) * 2^(E-1)
        const int c_hi = cmp_decimal_halfway(digs, nd, p, sticky, 2 * M + 1, E - 1);
        if (c_hi > 0 || (c_hi == 0 && (M & 1))) {
            ++ub;
            if (ub >= 0x7FF0000000000000ull) return bits_dbl(0x7FF0000000000000ull);
            continue;
        }
        // halfway to the next double down
        if (ub == 1) {
            // between 0 and the min subnormal: halfway = 2^-1075 = 1 * 2^-1075
            const int c_lo = cmp_decimal_halfway(digs, nd, p, sticky, 1, -1075);
            if (c_lo < 0 || c_lo == 0) return 0.0;  // tie -> even (0)
            return bits_dbl(ub);
        }
        uint64_t Mp;
        int64_t Ep;
        dbl_decompose(bits_dbl(ub - 1), Mp, Ep);
        const int c_lo = cmp_decimal_halfway(digs, nd, p, sticky, 2 * Mp + 1, Ep - 1);
        if (c_lo < 0) {
            --ub;
            continue;
        }
        if (c_lo == 0) {
            // exact tie between prev and this: pick the even mantissa
            if (M & 1) --ub;
            return bits_dbl(ub);
        }
        return bits_dbl(ub);
    }
    return bits_dbl(ub);
}

CVLG_HD uint8_t lower(uint8_t c) { return (c >= 'A' && c <= 'Z') ? static_cast<uint8_t>(c + 32) : c; }

// from_chars "nan" / "nan(n-char-seq)" / "inf" / "infinity" (case-insensitive, optional '-')
// covering the WHOLE field. Value only matters as "non-finite" downstream.
CVLG_HD bool parse_infnan(const uint8_t* s, int n, double& out) {
    int i = 0;
    bool neg = false;
    if (i < n && s[i] == '-') {
        neg = true;
        ++i;
    }
    if (n - i < 3) return false;
    if (lower(s[i]) == 'n' && lower(s[i + 1]) == 'a' && lower(s[i + 2]) == 'n') {
        int end = i + 3;
        if (end != n && s[end] == '(') {
            for (int j = end + 1; j < n; ++j) {
                const uint8_t c = s[j];
                if (c == ')') {
                    end = j + 1;
                    break;
                }
                if (!((c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || is_digit(c) || c == '_'))
                    break;
            }
        }
        if (end != n) return false;
        out = bits_dbl(neg ? 0xFFF8000000000000ull : 0x7FF8000000000000ull);
        return true;
    }
    if (lower(s[i]) == 'i' && lower(s[i + 1]) == 'n' && lower(s[i + 2]) == 'f') {
        int end = i + 3;
        if (n - i >= 8 && lower(s[i + 3]) == 'i' && lower(s[i + 4]) == 'n' &&
            lower(s[i + 5]) == 'i' && lower(s[i + 6]) == 't' && lower(s[i + 7]) == 'y')
            end = i + 8;
        if (end != n) return false;
        out = bits_dbl(neg ? 0xFFF0000000000000ull : 0x7FF0000000000000ull);
        return true;
    }
    return false;
}

// Gather up to kMaxDigits significant digits into `buf`. Returns count; sets sticky/p.
static constexpr int kMaxDigits = 800;

CVLG_HD_NOINLINE double parse_double_slow(const uint8_t* ip, int ilen, const uint8_t* fp, int flen,
                                          int64_t exp10, bool& is_zero) {
    uint8_t buf[kMaxDigits];
    int nd = 0;
    bool sticky = false;
    bool started = false;
    int64_t frac_used = 0;  // fraction digits consumed into buf (or skipped as leading zeros)
    int64_t int_dropped = 0;
    for (int i = 0; i < ilen; ++i) {
        const uint8_t c = ip[i];
        if (!started && c == '0') continue;
        started = true;
        if (nd < kMaxDigits) buf[nd++] = c;
        else {
            ++int_dropped;
            if (c != '0') sticky = true;
        }
    }
    for (int i = 0; i < flen; ++i) {
        const uint8_t c = fp[i];
        if (!started && c == '0') {
            ++frac_used;
            continue;
        }
        started = true;
        if (nd < kMaxDigits) {
            buf[nd++] = c;
            ++frac_used;
        } else if (c != '0') {
            sticky = true;
        }
    }
    if (nd == 0) {
        is_zero = true;
        return 0.0;
    }
    is_zero = false;
    // value = int(buf) * 10^(exp10 + int_dropped - frac_used)
    const int64_t p = exp10 + int_dropped - frac_used;
    return slow_decimal_to_double(buf, nd, p, sticky);
}

// std::from_chars(first, last, double) with parse_double's full-consumption rule
// (ingest.cpp:66-72). Returns false for BadNumeric (invalid, partial, or ERANGE).
CVLG_HD bool parse_double(const uint8_t* s, int n, double& out) {
    if (n <= 0) return false;
    int i = 0;
    bool neg = false;
    if (s[0] == '-') {
        neg = true;
        i = 1;
        if (i == n) return false;
        if (!is_digit(s[i]) && s[i] != '.') return parse_infnan(s, n, out);
    }
    const int int_begin = i;
    uint64_t w = 0;
    while (i < n && is_digit(s[i])) {
        w = w * 10 + (s[i] - '0');  // may wrap for > 19 digits; then `many` below
        ++i;
    }
    const int int_len = i - int_begin;
    int frac_begin = i, frac_len = 0;
    if (i < n && s[i] == '.') {
        ++i;
        frac_begin = i;
        while (i < n && is_digit(s[i])) {
            w = w * 10 + (s[i] - '0');
            ++i;
        }
        frac_len = i - frac_begin;
    }
    if (int_len + frac_len == 0) return parse_infnan(s, n, out);
    int64_t exp_number = 0;
    if (i < n && (s[i] == 'e' || s[i] == 'E')) {
        int j = i + 1;
        bool neg_exp = false;
        if (j < n && s[j] == '-') {
            neg_exp = true;
            ++j;
        } else if (j < n && s[j] == '+') {
            ++j;
        }
        if (j < n && is_digit(s[j])) {
            while (j < n && is_digit(s[j])) {
                if (exp_number < 0x10000000) exp_number = 10 * exp_number + (s[j] - '0');
                ++j;
            }
            if (neg_exp) exp_number = -exp_number;
            i = j;
        }
        // else: 'e' not consumed -> partial match -> rejected below
    }
    if (i != n) return false;  // from_chars stopped early: parse_double requires ptr == last

    // significant digit count (leading zeros do not count)
    int sig = int_len + frac_len;
    {
        int k = int_begin;
        const int stop_int = int_begin + int_len;
        while (k < stop_int && s[k] == '0') {
            --sig;
            ++k;
        }
        if (k == stop_int) {
            int f = frac_begin;
            const int stop_f = frac_begin + frac_len;
            while (f < stop_f && s[f] == '0') {
                --sig;
                ++f;
            }
        }
    }
    double v;
    if (sig == 0) {
        v = 0.0;  // exact zero: never ERANGE
    } else {
        const int64_t p = exp_number - frac_len;
        if (sig <= 19 && w <= (1ull << 53) && p >= -22 && p <= 22) {
            // Clinger: both operands exact, one correctly rounded IEEE operation
            const double m = static_cast<double>(w);
            v = p < 0 ? d_div(m, exact_pow10(static_cast<int>(-p)))
                      : d_mul(m, exact_pow10(static_cast<int>(p)));
        } else {
            bool is_zero = false;
            v = parse_double_slow(s + int_begin, int_len, s + frac_begin, frac_len, exp_number,
                                  is_zero);
            if (!is_zero) {
                const uint64_t b = dbl_bits(v);
                if (b == 0 || b == 0x7FF0000000000000ull) return false;  // ERANGE
            }
        }
    }
    out = neg ? -v : v;
    return true;
}

// ---------------------------------------------------------------------------------------------
// Header mapping (ingest.cpp:56-64, 97-115). `line` excludes the trailing '\n' and one '\r'.
CVLG_HD bool parse_header(const uint8_t* line, int64_t n, ColumnMap& map) {
    map.journey_id = map.timestamp = map.latitude = map.longitude = -1;
    map.postal_code = map.speed = map.heading = -1;
    int32_t field = 0;
    // normalized name buffer; names longer than 10 chars cannot match
    uint8_t nb[12];
    int nl = 0;
    bool over = false;
    for (int64_t i = 0; i <= n; ++i) {
        if (i == n || line[i] == ',') {
            int which = -1;
            if (!over) {
                auto eq = [&](const char* lit) {
                    int k = 0;
                    for (; lit[k]; ++k)
                        if (k >= nl || nb[k] != static_cast<uint8_t>(lit[k])) return false;
                    return k == nl;
                };
                if (eq("journeyid")) which = 0;
                else if (eq("timestamp")) which = 1;
                else if (eq("latitude")) which = 2;
                else if (eq("longitude")) which = 3;
                else if (eq("postalcode") || eq("zipcode")) which = 4;
                else if (eq("speed")) which = 5;
                else if (eq("heading")) which = 6;
            }
            switch (which) {
            case 0: map.journey_id = field; break;
            case 1: map.timestamp = field; break;
            case 2: map.latitude = field; break;
            case 3: map.longitude = field; break;
            case 4: map.postal_code = field; break;
            case 5: map.speed = field; break;
            case 6: map.heading = field; break;
            default: break;
            }
            ++field;
            nl = 0;
            over = false;
            continue;
        }
        const uint8_t c = line[i];
        if (c == ' ' || c == '_' || c == '-' || c == '\t' || c == '\r') continue;
        if (nl < 11) nb[nl++] = lower(c);
        else over = true;
    }
    map.n_columns = field;
    return map.journey_id >= 0 && map.timestamp >= 0 && map.latitude >= 0 && map.longitude >= 0 &&
           map.speed >= 0 && map.heading >= 0;
}

// A parsed record (only what the aggregation path consumes, plus the payload fields that the
// duplicate-conflict check compares, aggregate.cpp:286).
struct Parsed {
    int64_t epoch;
    double lat, lon, speed, heading;
    int32_t id_begin, id_len;          // offsets into the line
    int32_t postal_begin, postal_len;  // offsets into the line (len 0 when absent)
};

// parse_record_impl (ingest.cpp:119-157). `line` excludes '\n' and one trailing '\r'.
CVLG_HD uint8_t parse_line(const uint8_t* line, int32_t n, const ColumnMap& cm, Parsed& r) {
    // field spans for the 7 mapped columns
    int32_t fb[7], fe[7];
    for (int k = 0; k < 7; ++k) fb[k] = fe[k] = 0;
    const int32_t want[7] = {cm.journey_id, cm.timestamp, cm.latitude, cm.longitude,
                             cm.postal_code, cm.speed, cm.heading};
    int32_t field = 0, start = 0;
    for (int32_t i = 0; i <= n; ++i) {
        if (i == n || line[i] == ',') {
            int32_t b = start, e = i;
            while (b < e && is_trim(line[b])) ++b;
            while (e > b && is_trim(line[e - 1])) --e;
#pragma unroll
            for (int k = 0; k < 7; ++k)
                if (want[k] == field) {
                    fb[k] = b;
                    fe[k] = e;
                }
            ++field;
            start = i + 1;
        }
    }
    // journey, ts, lat, lon, speed, heading must be non-empty (ingest.cpp:135-137)
    if (fe[0] == fb[0] || fe[1] == fb[1] || fe[2] == fb[2] || fe[3] == fb[3] || fe[5] == fb[5] ||
        fe[6] == fb[6])
        return kMissingField;
    if (!parse_timestamp(line + fb[1], fe[1] - fb[1], r.epoch)) return kBadTimestamp;
    if (!parse_double(line + fb[2], fe[2] - fb[2], r.lat) ||
        !parse_double(line + fb[3], fe[3] - fb[3], r.lon) ||
        !parse_double(line + fb[5], fe[5] - fb[5], r.speed) ||
        !parse_double(line + fb[6], fe[6] - fb[6], r.heading))
        return kBadNumeric;
    if (r.heading == 360.0) r.heading = 0.0;  // canonical wrap
    const bool speed_finite = (dbl_bits(r.speed) & 0x7FF0000000000000ull) != 0x7FF0000000000000ull;
    if (!(r.lat >= -90.0 && r.lat <= 90.0) || !(r.lon >= -180.0 && r.lon <= 180.0) ||
        !(r.speed >= 0.0) || !speed_finite || !(r.heading >= 0.0 && r.heading < 360.0))
        return kRangeViolation;
    r.id_begin = fb[0];
    r.id_len = fe[0] - fb[0];
    r.postal_begin = fb[4];
    r.postal_len = fe[4] - fb[4];
    return kAccepted;
}

}  // namespace cvlg
