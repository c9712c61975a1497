/*
 * oracle/lift.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 * Z_2 -> Z_T lifting by EXHAUSTIVE enumeration ("assigns +-1 signs to
 * non-zero coefficients while preserving Brent equation validity"): every sign
 * pattern of the nonzero coefficients, with the first nonzero of each row's u and v
 * fixed to +1 (PAPER:429's rescaling, which loses no solution up to equivalence), is
 * checked with or_verify.  For small instances only (<= 30 free signs).
 * Returns 1 and the first lift found (enumeration order: free sign k = bit k of the
 * counter, bit set = -1), 0 if none exists, -1 if too many free signs.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

int or_lift_exhaustive(int m, int n, int p, const int8_t *z2, int rank, int8_t *out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, l, e, nfree = 0, found = 0;
    int *pos = (int *)malloc(sizeof(int) * (size_t)rank * width + 1);
    uint64_t cnt, total;
    int8_t *cand = (int8_t *)malloc((size_t)rank * width + 1);
    for (l = 0; l < rank; l++) {
        int first_u = 1, first_v = 1;
        for (e = 0; e < width; e++) {
            if (!z2[l * width + e]) continue;
            if (e < mn && first_u) { first_u = 0; continue; }
            if (e >= mn && e < mn + np && first_v) { first_v = 0; continue; }
            pos[nfree++] = l * width + e;
        }
    }
    if (nfree > 30) { free(pos); free(cand); return -1; }
    total = 1ull << nfree;
    for (cnt = 0; cnt < total && !found; cnt++) {
        int k;
        int32_t ff[3];
        memcpy(cand, z2, (size_t)rank * width);
        for (k = 0; k < nfree; k++)
            if ((cnt >> k) & 1) cand[pos[k]] = -1;
        if (or_verify(m, n, p, OR_RING_ZT, cand, rank, ff) == 0) {
            memcpy(out, cand, (size_t)rank * width);
            found = 1;
        }
    }
    free(pos);
    free(cand);
    return found;
}
