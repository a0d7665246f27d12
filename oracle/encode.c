/*
 * oracle/encode.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * The one loop of the oracle that is too slow in numpy: "round(.) denotes
 * rounding to the nearest MXFP value" (§2.1, Eq. 1, line 43-45),
 * written as a brute-force nearest-code search.  For every scaled input
 * v = X_j / s (already exact, computed by the caller in fp64) it scans ALL
 * finite non-negative codes of the element format and keeps the one whose
 * value is nearest to |v|; on an exact tie it keeps the code whose least
 * significant bit is 0 (ties-to-even, reading R4).  The sign bit is
 * the sign bit of v (sign-preserving zero, reading R6).  Values
 * beyond q_max therefore land on q_max (saturation, reading R5) because q_max
 * is the nearest finite code.
 *
 * The code-value table (mag_vals[c] for magnitude code c, NAN for non-finite
 * codes) is built by the caller from the bit-field definition in
 * oracle/formats.py; this file knows nothing about formats.
 * Shares no code with the CUDA path.
 */
#include <math.h>
#include <stdint.h>

void orc_encode_nearest(const double *v, int64_t n, const double *mag_vals,
                        int n_mag, int sign_bit, uint8_t *codes_out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs(v[i]);
    int best = -1;
    double best_q = 0.0;
    for (int c = 0; c < n_mag; ++c) {
      double q = mag_vals[c];
      if (isnan(q)) continue; /* non-finite code: never produced */
      if (best < 0) { best = c; best_q = q; continue; }
      /* |a - q| vs |a - best_q| decided exactly through the midpoint of the two
       * code values (exact in fp64: both have <= 4 significant bits), so no
       * rounding of a difference can fake a tie for large |v|. */
      double mid = 0.5 * (q + best_q);
      int closer = (q > best_q) ? (a > mid) : (a < mid);
      int tie = (a == mid);
      if (closer || (tie && (c & 1) == 0 && (best & 1) == 1)) { best = c; best_q = q; }
    }
    uint8_t code = (uint8_t)best;
    if (signbit(v[i])) code |= (uint8_t)(1u << sign_bit);
    codes_out[i] = code;
  }
}
