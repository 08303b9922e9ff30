/* The row update (k_rows.inc.cuh, rows_mma_block) evaluates g / h_rr of Eq 11-13
 * as q0 = g * ri, r = fma(-q0, h, g), q = fma(r, ri, q0) with ri = 1 / h correctly rounded
 * once per pass.  Markstein's theorem says q is the correctly rounded quotient in
 * round-to-nearest (no overflow / underflow).  This program checks the identity bit for bit
 * against IEEE division on 2e7 random pairs over 120 binades of g and 80 of h, a quarter of
 * them with all-ones significands of h and a quarter with h a power of two.
 * Exit status 0 = no mismatch.  Built and run by tests/test_division_identity.py. */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ULL;
static uint64_t nx(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rnd(int emin, int emax) {
  uint64_t m = nx() & ((1ULL << 52) - 1);
  int e = emin + (int)(nx() % (uint64_t)(emax - emin + 1));
  uint64_t bits = ((uint64_t)(e + 1023) << 52) | m;
  double x; memcpy(&x, &bits, 8);
  return (nx() & 1) ? -x : x;
}
int main(int argc, char **argv) {
  long n = 20000000, bad = 0;
  for (long i = 0; i < n; i++) {
    double g = rnd(-60, 60), h = fabs(rnd(-40, 40));
    if (i % 4 == 1) { uint64_t b; memcpy(&b, &h, 8); b |= (1ULL << 52) - 1; memcpy(&h, &b, 8); }  /* all-ones significand */
    if (i % 4 == 2) { uint64_t b; memcpy(&b, &h, 8); b &= ~((1ULL << 52) - 1); memcpy(&h, &b, 8); } /* power of two */
    const double ri = 1.0 / h, q0 = g * ri, r = fma(-q0, h, g), q = fma(r, ri, q0);
    if (q != g / h) { if (bad < 5) printf("mismatch g=%a h=%a q=%a ref=%a\n", g, h, q, g / h); bad++; }
  }
  printf("%ld of %ld differ\n", bad, n);
  return bad != 0;
}
