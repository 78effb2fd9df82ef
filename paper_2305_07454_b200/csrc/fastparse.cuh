// Fast path of parse_record_impl (ingest.cpp:119-157) for K1 decode: SWAR field parsing over a
// line staged in a 16-byte aligned shared-memory buffer. Every function returns false whenever
// it cannot prove that its answer equals the general restatement (parse.cuh) — the caller then
// runs parse_line — so the fast path only ever changes speed, never results.
//
// Portable (host + device) so tests/native/hostparse.cpp fuzzes this exact code on the CPU
// against the reference parser.
//
//   timestamp  datetime.cpp:53-75   19 bytes, date part cached per thread (rows of a trace share
//                                   a calendar day), time part from two byte permutes
//   numbers    ingest.cpp:66-72     std::from_chars(double) for [-]digits[.digits] fields of at
//                                   most 12 bytes: the dot is dropped with two funnel shifts, the
//                                   12 digits are converted with 4-digit SWAR, and the value
//                                   10*M / 10^(F+1) is correctly rounded by Markstein's
//                                   reciprocal correction (exact: the mantissa < 2^53 and 10^k
//                                   is exact, i.e. Clinger's fast path)
#pragma once
#include "parse.cuh"

namespace cvlg {

// ---- portable intrinsics -----------------------------------------------------------------------
CVLG_HD uint32_t fs_r(uint32_t lo, uint32_t hi, uint32_t sh) {  // (hi:lo >> (sh & 31))
#if defined(__CUDA_ARCH__)
    return __funnelshift_r(lo, hi, sh);
#else
    sh &= 31;
    return static_cast<uint32_t>(((static_cast<uint64_t>(hi) << 32) | lo) >> sh);
#endif
}
CVLG_HD uint32_t fs_rc(uint32_t lo, uint32_t hi, uint32_t sh) {  // (hi:lo >> min(sh, 32))
#if defined(__CUDA_ARCH__)
    return __funnelshift_rc(lo, hi, sh);
#else
    if (sh > 32) sh = 32;
    return static_cast<uint32_t>(((static_cast<uint64_t>(hi) << 32) | lo) >> sh);
#endif
}
CVLG_HD uint32_t fs_l(uint32_t lo, uint32_t hi, uint32_t sh) {  // high word of (hi:lo << (sh & 31))
#if defined(__CUDA_ARCH__)
    return __funnelshift_l(lo, hi, sh);
#else
    sh &= 31;
    return static_cast<uint32_t>((((static_cast<uint64_t>(hi) << 32) | lo) << sh) >> 32);
#endif
}
CVLG_HD int clz32(uint32_t x) {
#if defined(__CUDA_ARCH__)
    return __clz(x);
#else
    return x ? __builtin_clz(x) : 32;
#endif
}
CVLG_HD uint32_t bperm(uint32_t x, uint32_t y, uint32_t s) {  // __byte_perm without modes
#if defined(__CUDA_ARCH__)
    return __byte_perm(x, y, s);
#else
    const uint64_t v = (static_cast<uint64_t>(y) << 32) | x;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= static_cast<uint32_t>((v >> (8 * ((s >> (4 * i)) & 7))) & 0xFF) << (8 * i);
    return r;
#endif
}
CVLG_HD double fma_rn(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

// 0x80 in every byte of x equal to the byte replicated in pat (exact, no cross-byte carries)
CVLG_HD uint32_t eqflags(uint32_t x, uint32_t pat) {
    const uint32_t t = x ^ pat;
    return ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;
}

// bytes [off, off + 4) of a 4-byte aligned buffer, little endian
CVLG_HD uint32_t word_at(const uint32_t* w, uint32_t off) {
    return fs_r(w[off >> 2], w[(off >> 2) + 1], (off & 3) * 8);
}

// every byte of a, b, c in '0'..'9' (high nibble 3 and low nibble <= 9; +6 never carries out of a
// byte whose high nibble is 3, and any other byte already fails the high-nibble test)
CVLG_HD bool digits3(uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t hi = ((a | b | c) & 0xC0C0C0C0u) | (((a & b & c) & 0x30303030u) ^ 0x30303030u);
    const uint32_t lo = ((a + 0x06060606u) | (b + 0x06060606u) | (c + 0x06060606u)) & 0x40404040u;
    return (hi | lo) == 0;
}

// 4 ASCII digits (lowest byte = most significant) -> value
CVLG_HD uint32_t swar4(uint32_t v) {
    v &= 0x0F0F0F0Fu;
    v = (v * 10u + (v >> 8)) & 0x00FF00FFu;
    return (v * 100u + (v >> 16)) & 0xFFFFu;
}

constexpr double pow10c(int k) { return k == 0 ? 1.0 : 10.0 * pow10c(k - 1); }  // exact, k <= 22

// mask of the bytes at index >= t of a word (t may be <= 0 or >= 4)
CVLG_HD uint32_t bytes_from_rt(int t) {
    const int sh = 32 - 8 * t;
    return fs_rc(0u, 0xFFFFFFFFu, static_cast<uint32_t>(sh < 0 ? 0 : sh));
}

// keep bytes at index >= t of r, replace the others with '0'
CVLG_HD uint32_t keep_from(uint32_t r, int t) {
    const uint32_t m = bytes_from_rt(t);
    return (r & m) | (0x30303030u & ~m);
}

// 10^k and RN(10^-k), k = 0..8 (k = 0: the integer case divides by 1, exactly)
#if defined(__CUDA_ARCH__)
static __constant__ double kFpPow10[9] = {pow10c(0), pow10c(1), pow10c(2), pow10c(3), pow10c(4),
                                          pow10c(5), pow10c(6), pow10c(7), pow10c(8)};
static __constant__ double kFpInv10[9] = {1.0 / pow10c(0), 1.0 / pow10c(1), 1.0 / pow10c(2),
                                          1.0 / pow10c(3), 1.0 / pow10c(4), 1.0 / pow10c(5),
                                          1.0 / pow10c(6), 1.0 / pow10c(7), 1.0 / pow10c(8)};
#else
static const double kFpPow10[9] = {pow10c(0), pow10c(1), pow10c(2), pow10c(3), pow10c(4),
                                   pow10c(5), pow10c(6), pow10c(7), pow10c(8)};
static const double kFpInv10[9] = {1.0 / pow10c(0), 1.0 / pow10c(1), 1.0 / pow10c(2),
                                   1.0 / pow10c(3), 1.0 / pow10c(4), 1.0 / pow10c(5),
                                   1.0 / pow10c(6), 1.0 / pow10c(7), 1.0 / pow10c(8)};
#endif

// x / 10^k correctly rounded for exact integers 0 <= x < 2^53, 0 <= k <= 8: q0 = RN(x * RN(10^-k))
// is within an ulp, the residual is exact (FMA), and one correction rounds correctly
// (Markstein). Checked bit-equal to IEEE division over 4.8e9 cases (tests/test_fastparse.py).
CVLG_HD double div_pow10(double x, int k) {
    const double p = kFpPow10[k], r = kFpInv10[k];
    const double q0 = d_mul(x, r);
    const double res = fma_rn(-q0, p, x);
    return fma_rn(res, r, q0);
}

// std::from_chars(double) on field [b, e) (buffer offsets, kPre bytes of readable padding before
// the first field) for [-]digits[.digits] of at most 12 bytes. `qguess` carries the point
// position (in the 12-byte window right-aligned at e) of this column from the previous line.
//   short path (<= 8 digits, point in the last 8 bytes): bytes up to the point move up one
//     position over it, so the last two words hold the digits M right-aligned; x = M / 10^F.
//   long path (<= 11 digits): bytes after the point move down one position ('0' enters at 11),
//     so the three words read V = 10 M; x = V / 10^(F+1). Without a point nothing moves.
// Both divide an exact integer by an exact power of ten with correct rounding (div_pow10).
CVLG_HD bool fast_number(const uint32_t* w, const uint8_t* buf, uint32_t b, uint32_t e, int& qguess,
                         double& v) {
    const uint32_t n = e - b;
    if (n - 1u > 11u) return false;  // 1..12 bytes
    const bool neg = buf[b] == '-';
    const uint32_t o = e - 12, i = o >> 2, sh = (o & 3) * 8;
    const uint32_t x0 = w[i], x1 = w[i + 1], x2 = w[i + 2], x3 = w[i + 3];
    const uint32_t a0 = fs_r(x0, x1, sh), a1 = fs_r(x1, x2, sh), a2 = fs_r(x2, x3, sh);
    const int s = 12 - static_cast<int>(n) + (neg ? 1 : 0);  // first byte after the sign
    int q = qguess;
    const bool hit = q >= s && q >= 4 && buf[o + q] == '.';
    if (!hit) {  // rightmost point among the field's bytes in the last 8 (else -1)
        const uint32_t z1 = eqflags(a1, 0x2E2E2E2Eu) & bytes_from_rt(s - 4);
        const uint32_t z2 = eqflags(a2, 0x2E2E2E2Eu) & bytes_from_rt(s - 8);
        q = z2 ? 8 + ((31 - clz32(z2)) >> 3) : (z1 ? 4 + ((31 - clz32(z1)) >> 3) : -1);
        qguess = q;
    }
    const int D = static_cast<int>(n) - (neg ? 1 : 0) - (q >= 0 ? 1 : 0);  // digits (if one point)
    if (D <= 0) return false;
    if (D <= 8) {
        // the last 8 bytes as one 64-bit string (byte 0 = window position 4)
        const uint64_t a = (static_cast<uint64_t>(a2) << 32) | a1;
        uint64_t r = a;
        if (q >= 0) {  // bytes at positions <= q take the byte below them
            const uint64_t sft = (a << 8) | (a0 >> 24);
            const uint64_t keep_hi = q >= 11 ? 0ull : (~0ull << (8 * (q - 3)));  // positions > q
            r = (a & keep_hi) | (sft & ~keep_hi);
        }
        const uint64_t dig = ~0ull << (8 * (8 - D));  // digits occupy [12 - D, 12)
        r = (r & dig) | (0x3030303030303030ull & ~dig);
        const uint32_t r1 = static_cast<uint32_t>(r), r2 = static_cast<uint32_t>(r >> 32);
        if (!digits3(r1, r2, 0x30303030u)) return false;
        const double x = div_pow10(static_cast<double>(swar4(r1) * 10000u + swar4(r2)), q >= 0 ? 11 - q : 0);
        v = neg ? -x : x;
        return true;
    }
    const uint32_t r0 = keep_from(a0, s);
    uint32_t r1 = keep_from(a1, s - 4);
    uint32_t r2 = keep_from(a2, s - 8);
    const int qe = q < 0 ? 12 : q;  // (a point before byte 4 stays in place and fails below)
    const uint32_t s0 = fs_r(r0, r1, 8), s1 = fs_r(r1, r2, 8), s2 = (r2 >> 8) | 0x30000000u;
    const uint32_t m0 = bytes_from_rt(qe), m1 = bytes_from_rt(qe - 4), m2 = bytes_from_rt(qe - 8);
    const uint32_t t0 = (s0 & m0) | (r0 & ~m0);
    r1 = (s1 & m1) | (r1 & ~m1);
    r2 = (s2 & m2) | (r2 & ~m2);
    if (!digits3(t0, r1, r2)) return false;
    const uint64_t V = static_cast<uint64_t>(swar4(t0)) * 100000000ull + (swar4(r1) * 10000u + swar4(r2));
    const double x = div_pow10(static_cast<double>(V), 12 - qe);  // V exact: < 10^12
    v = neg ? -x : x;
    return true;
}

// 4 validated ASCII digits (byte 0 = most significant) -> value, plus `acc`: two 16x8-bit dot
// products on the device (IDP, the FMA pipe) instead of the ALU-pipe swar4 chain. The '0' bias
// (48 * 1111) is folded into the accumulator.
CVLG_HD uint32_t dig4_acc(uint32_t r, uint32_t acc) {
#if defined(__CUDA_ARCH__)
    return __dp2a_hi(0x0001000Au, r, __dp2a_lo(0x006403E8u, r, acc - 53328u));
#else
    return acc + swar4(r);
#endif
}

// std::from_chars(double) on field [b, e) (buffer offsets) for the shape the previous line of
// this column had: [-]digits.digits with the point at window index q (the 12-byte window is
// right-aligned at e, so q = 11 - fraction digits) and at most 8 digits. Branch-free: the
// caller combines the verdicts of all fields; false -> fast_number (which re-learns q) decides.
// Bytes at window positions <= q move up one position (dropping the point), positions before
// the first digit become '0', and the 8-digit string M is converted exactly; x = M / 10^(11-q)
// correctly rounded (div_pow10: M < 10^8 is exact, Clinger's fast path).
CVLG_HD bool fast_number_hit(const uint32_t* w, const uint8_t* buf, uint32_t b, uint32_t e, int q,
                             double& v) {
    const uint32_t n = e - b;
    const uint32_t o = e - 12, i = o >> 2, sh = (o & 3) * 8;
    const uint32_t x0 = w[i], x1 = w[i + 1], x2 = w[i + 2], x3 = w[i + 3];
    const uint32_t a0 = fs_r(x0, x1, sh), a1 = fs_r(x1, x2, sh), a2 = fs_r(x2, x3, sh);
    const uint32_t neg = buf[b] == '-' ? 1u : 0u;
    const int D = static_cast<int>(n) - static_cast<int>(neg) - 1;  // digits (one point)
    const int s = 12 - static_cast<int>(n) + static_cast<int>(neg);  // first byte after the sign
    const uint32_t pt = fs_r(q < 8 ? a1 : a2, a2, static_cast<uint32_t>(8 * q)) & 0xFFu;
    // drop the point: positions <= q take the byte below them
    const uint32_t s1 = fs_l(a0, a1, 8), s2 = fs_l(a1, a2, 8);
    const uint32_t k1 = bytes_from_rt(q - 3), k2 = bytes_from_rt(q - 7);
    uint32_t r1 = (a1 & k1) | (s1 & ~k1);
    uint32_t r2 = (a2 & k2) | (s2 & ~k2);
    // digits occupy [12 - D, 12): everything before becomes '0'
    const uint32_t d1 = bytes_from_rt(8 - D), d2 = bytes_from_rt(4 - D);
    r1 = (r1 & d1) | (0x30303030u & ~d1);
    r2 = (r2 & d2) | (0x30303030u & ~d2);
    const bool ok = (n <= 12u) & (D >= 1) & (D <= 8) & (q >= 4) & (q >= s) & (pt == 0x2Eu) &
                    digits3(r1, r2, 0x30303030u);
    const uint32_t M = dig4_acc(r2, dig4_acc(r1, 0u) * 10000u);
    const double x = div_pow10(static_cast<double>(M), (11 - q) & 7);
    v = bits_dbl(dbl_bits(x) | (static_cast<uint64_t>(neg) << 63));
    return ok;
}

// Trim byte of split_fields (ingest.cpp:31-39): ' ', '\t', '\r' (one range test + bit test)
CVLG_HD bool trim_byte(uint32_t c) {
    const uint32_t t = c - 9u;
    return t < 24u && ((0x800011u >> t) & 1u);
}

// '\n' and ',' flags of 32 staged bytes (words x[0..7], little endian) -> two 32-bit masks, bit i
// = byte i. Per byte class the exact zero-byte test costs 3 operations (the 0x7F mask of x is
// shared; the class bytes have bit 7 clear). Flags of two words are merged into one word
// ((a >> 4) | b: bits 8j+3 and 8j+7) and gathered into its top byte by one multiply: byte j of
// word a moves to bit 24 + j and byte j of word b to bit 28 + j (every partial product lands on
// a distinct bit, so nothing carries into the top byte); byte permutes assemble the masks.
CVLG_HD void class_masks32(const uint32_t* x, uint32_t& mn, uint32_t& mc) {
    uint32_t rn[4], rc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t xa = x[2 * k], xb = x[2 * k + 1];
        const uint32_t ma = xa & 0x7F7F7F7Fu, mb = xb & 0x7F7F7F7Fu;
        const uint32_t na = ~(((ma ^ 0x0A0A0A0Au) + 0x7F7F7F7Fu) | xa) & 0x80808080u;
        const uint32_t nb = ~(((mb ^ 0x0A0A0A0Au) + 0x7F7F7F7Fu) | xb) & 0x80808080u;
        const uint32_t ca = ~(((ma ^ 0x2C2C2C2Cu) + 0x7F7F7F7Fu) | xa) & 0x80808080u;
        const uint32_t cb = ~(((mb ^ 0x2C2C2C2Cu) + 0x7F7F7F7Fu) | xb) & 0x80808080u;
        rn[k] = ((na >> 4) | nb) * 0x204081u;
        rc[k] = ((ca >> 4) | cb) * 0x204081u;
    }
    mn = bperm(bperm(rn[0], rn[1], 0x0073u), bperm(rn[2], rn[3], 0x0073u), 0x5410u);
    mc = bperm(bperm(rc[0], rc[1], 0x0073u), bperm(rc[2], rc[3], 0x0073u), 0x5410u);
}

// Per-thread cache of the last validated calendar date ("YYYY-MM-DD" bytes -> days * 86400).
// Starts at 1970-01-01 (a valid date), so a cache hit always means validated bytes.
struct DateCache {
    uint32_t k0 = 0x30373931u;  // "1970"
    uint32_t k1 = 0x2D31302Du;  // "-01-"
    uint32_t k2 = 0x3130u;      // "01"
    // days * 86400 as two words: 4-byte alignment keeps FastState at an odd word count (9), so
    // the per-thread states in shared memory fall on distinct banks
    uint32_t ds_lo = 0, ds_hi = 0;
};

CVLG_HD int64_t day_sec(const DateCache& dc) {
    return static_cast<int64_t>((static_cast<uint64_t>(dc.ds_hi) << 32) | dc.ds_lo);
}

// validates "YYYY-MM-DD" (datetime.cpp:53-61: month 1..12, day 1..days_in_month) and fills the
// cache; false -> the general parser decides
CVLG_HD bool date_refill(uint32_t t0, uint32_t t1, uint32_t t2, DateCache& dc) {
    if ((t1 & 0xFF0000FFu) != 0x2D00002Du) return false;
    const uint32_t mm = bperm(t1, 0x30303030u, 0x4421u);  // M M 0 0
    const uint32_t dd = bperm(t2, 0x30303030u, 0x4410u);  // D D 0 0
    if (!digits3(t0, mm, dd)) return false;
    const int y = static_cast<int>(swar4(t0));
    const int mo = static_cast<int>(swar4(mm) / 100u);
    const int d = static_cast<int>(swar4(dd) / 100u);
    if (mo < 1 || mo > 12 || d < 1 || d > static_cast<int>(days_in_month(y, static_cast<unsigned>(mo))))
        return false;
    dc.k0 = t0;
    dc.k1 = t1;
    dc.k2 = t2 & 0xFFFFu;
    const int64_t ds = days_from_civil(y, static_cast<unsigned>(mo), static_cast<unsigned>(d)) * 86400;
    dc.ds_lo = static_cast<uint32_t>(static_cast<uint64_t>(ds));
    dc.ds_hi = static_cast<uint32_t>(static_cast<uint64_t>(ds) >> 32);
    return true;
}

// Timestamp::parse (datetime.cpp:65-75) of the 19 bytes at buffer offset off: epoch seconds and
// minute of day (the time_bin input, grid.cpp:69-71). `next` receives the byte after the 19
// (the field separator the caller expects). Branch-free except for the date-cache refill.
CVLG_HD bool fast_timestamp(const uint32_t* w, uint32_t off, DateCache& dc, int64_t& ts, uint32_t& mod,
                            uint32_t& next) {
    const uint32_t i = off >> 2, sh = (off & 3) * 8;
    const uint32_t a0 = w[i], a1 = w[i + 1], a2 = w[i + 2], a3 = w[i + 3], a4 = w[i + 4], a5 = w[i + 5];
    const uint32_t t0 = fs_r(a0, a1, sh), t1 = fs_r(a1, a2, sh), t2 = fs_r(a2, a3, sh),
                   t3 = fs_r(a3, a4, sh), t4 = fs_r(a4, a5, sh);
    next = t4 >> 24;
    if (t0 != dc.k0 || t1 != dc.k1 || (t2 & 0xFFFFu) != dc.k2)
        if (!date_refill(t0, t1, t2, dc)) return false;
    const uint32_t hm = bperm(t2, t3, 0x7643u);             // H H M M
    const uint32_t ss = bperm(t4, 0x30303030u, 0x4421u);    // S S 0 0
    const uint32_t dh = hm & 0x0F0F0F0Fu;
    const uint32_t p = dh * 10u + (dh >> 8);  // byte 0: HH, byte 2: MM
    const uint32_t h = p & 0xFFu, mi = (p >> 16) & 0xFFu;
    const uint32_t s = (ss & 0xFu) * 10u + ((ss >> 8) & 0xFu);
    // ' ' at 10, ':' at 13 and 16, digits, 0..23:0..59:0..59
    const bool ok = ((t2 & 0x00FF0000u) == 0x00200000u) & ((t3 & 0x0000FF00u) == 0x00003A00u) &
                    ((t4 & 0xFFu) == 0x3Au) & digits3(hm, ss, 0x30303030u) & (h <= 23) & (mi <= 59) &
                    (s <= 59);
    mod = h * 60u + mi;
    ts = day_sec(dc) + static_cast<int64_t>(mod * 60u + s);
    return ok;
}

CVLG_HD bool fast_timestamp(const uint32_t* w, uint32_t off, DateCache& dc, int64_t& ts, uint32_t& mod) {
    uint32_t next;
    return fast_timestamp(w, off, dc, ts, mod, next);
}

}  // namespace cvlg
