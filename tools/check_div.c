#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
// q0 = RN(x*r), res = fma(-q0, d, x), q1 = fma(res, r, q0) with r = RN(1/d), d = 10^k; check == x/d
int main(int argc, char** argv) {
  uint64_t lim = strtoull(argv[1], 0, 10);
  long bad = 0, tot = 0;
  for (int k = 1; k <= 8; ++k) {
    double d = 1; for (int i = 0; i < k; ++i) d *= 10;
    double r = 1.0 / d;
    for (uint64_t v = 0; v < lim; ++v) {
      double x = (double)v;
      double q0 = x * r;
      double res = fma(-q0, d, x);
      double q1 = fma(res, r, q0);
      if (q1 != x / d) { if (bad < 10) printf("bad k=%d v=%llu\n", k, (unsigned long long)v); ++bad; }
      ++tot;
    }
    // random 12-digit values
    uint64_t s = 88172645463325252ull;
    for (long i = 0; i < 200000000; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      uint64_t v = s % 1000000000000ull;
      double x = (double)v;
      double q0 = x * r; double res = fma(-q0, d, x); double q1 = fma(res, r, q0);
      if (q1 != x / d) { if (bad < 10) printf("bad k=%d v=%llu\n", k, (unsigned long long)v); ++bad; }
      ++tot;
    }
  }
  printf("checked %ld bad %ld\n", tot, bad);
  return 0;
}
