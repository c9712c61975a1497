/*
 * oracle/meta.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The meta operators of PAPER:243-262 (section 3.3.2) written from their
 * definitions, on int8 coefficient rows [u(mn) | v(np) | w(pm)] with the C^T
 * layout of R2.  Readings (R25-R30):
 *   transpose  (m,n,p) -> (p,n,m): C = AB  <=>  C^T = B^T A^T
 *   rotate     (m,n,p) -> (n,p,m): the cyclic symmetry of the matmul tensor,
 *              (u, v, w) -> (v, w, u) with the same flattened indices
 *   swap sizes (m,n,p) -> (m,p,n) = rotate(rotate(transpose))
 *   project    (m,n,p) -> (m,n,p-1): drop the last column of B and of
 *              C, then remove terms with a zero factor
 *   extend     (m,n,p:r) -> (m,n,p+1 : r+mn): append a naive (m,n,1)
 *              scheme for the new last column, rows ordered by (i, j)
 *   merge      (m,n,p1:r1) + (m,n,p2:r2) -> (m,n,p1+p2 : r1+r2):
 *              B = [B1 | B2], C = [C1 | C2]; rows of the first scheme first
 *   double     merge with itself
 *   product    (m1,n1,p1:r1) x (m2,n2,p2:r2) -> (m1m2, n1n2, p1p2 : r1r2)
 *              (PAPER:253): Kronecker products, block index i = i1*m2 + i2 (etc.),
 *              row l = l1*r2 + l2
 * Outputs are not sign-normalised.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

#define UIDX(i, j, n) ((i) * (n) + (j))            /* a_ij */
#define VIDX(j, k, p) ((j) * (p) + (k))            /* b_jk */
#define WIDX(k, i, m) ((k) * (m) + (i))            /* c_ik, C^T order */

static int fmt_ok(int m, int n, int p)
{
    return m >= 1 && n >= 1 && p >= 1 && m * n <= OR_MAXLEN && n * p <= OR_MAXLEN && p * m <= OR_MAXLEN;
}

int or_meta_transpose(int m, int n, int p, const int8_t *in, int rank, int8_t *out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, l, i, j, k;
    /* new format (M,N,P) = (p,n,m): A' = B^T (p x n), B' = A^T (n x m), C' = C^T (p x m) */
    int M = p, N = n, P = m;
    if (!fmt_ok(m, n, p)) return -2;
    for (l = 0; l < rank; l++) {
        const int8_t *u = in + (size_t)l * width, *v = u + mn, *w = v + np;
        int8_t *uo = out + (size_t)l * width, *vo = uo + M * N, *wo = vo + N * P;
        for (i = 0; i < m; i++)
            for (j = 0; j < n; j++) vo[VIDX(j, i, P)] = u[UIDX(i, j, n)];      /* B'_{j i} = A_{i j} */
        for (j = 0; j < n; j++)
            for (k = 0; k < p; k++) uo[UIDX(k, j, N)] = v[VIDX(j, k, p)];      /* A'_{k j} = B_{j k} */
        for (i = 0; i < m; i++)
            for (k = 0; k < p; k++) wo[WIDX(i, k, M)] = w[WIDX(k, i, m)];      /* C'_{k i} = C_{i k} */
    }
    return 0;
}

int or_meta_rotate(int m, int n, int p, const int8_t *in, int rank, int8_t *out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, l;
    if (!fmt_ok(m, n, p)) return -2;
    for (l = 0; l < rank; l++) {
        const int8_t *u = in + (size_t)l * width, *v = u + mn, *w = v + np;
        int8_t *o = out + (size_t)l * width;
        memcpy(o, v, (size_t)np);               /* u' = v, format (n,p,m) */
        memcpy(o + np, w, (size_t)pm);          /* v' = w */
        memcpy(o + np + pm, u, (size_t)mn);     /* w' = u */
    }
    return 0;
}

int or_meta_swap_sizes(int m, int n, int p, const int8_t *in, int rank, int8_t *out)
{
    int width = m * n + n * p + p * m, rc;
    int8_t *t1 = (int8_t *)malloc((size_t)rank * width + 1), *t2 = (int8_t *)malloc((size_t)rank * width + 1);
    rc = or_meta_transpose(m, n, p, in, rank, t1);        /* (p,n,m) */
    if (rc == 0) rc = or_meta_rotate(p, n, m, t1, rank, t2);   /* (n,m,p) */
    if (rc == 0) rc = or_meta_rotate(n, m, p, t2, rank, out);  /* (m,p,n) */
    free(t1);
    free(t2);
    return rc;
}

static int row_zero_factor(const int8_t *row, int a, int b, int c)
{
    int e, z;
    for (z = 1, e = 0; e < a; e++) if (row[e]) z = 0;
    if (z) return 1;
    for (z = 1, e = 0; e < b; e++) if (row[a + e]) z = 0;
    if (z) return 1;
    for (z = 1, e = 0; e < c; e++) if (row[a + b + e]) z = 0;
    return z;
}

int or_meta_project(int m, int n, int p, const int8_t *in, int rank, int8_t *out, int *rank_out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm;
    int P = p - 1, nw = mn + n * P + P * m, l, i, j, k, o = 0;
    if (p < 2 || !fmt_ok(m, n, p)) return -2;
    for (l = 0; l < rank; l++) {
        const int8_t *u = in + (size_t)l * width, *v = u + mn, *w = v + np;
        int8_t *uo = out + (size_t)o * nw, *vo = uo + mn, *wo = vo + n * P;
        memcpy(uo, u, (size_t)mn);
        for (j = 0; j < n; j++)
            for (k = 0; k < P; k++) vo[VIDX(j, k, P)] = v[VIDX(j, k, p)];
        for (k = 0; k < P; k++)
            for (i = 0; i < m; i++) wo[WIDX(k, i, m)] = w[WIDX(k, i, m)];
        if (!row_zero_factor(uo, mn, n * P, P * m)) o++;
    }
    *rank_out = o;
    return 0;
}

int or_meta_extend(int m, int n, int p, const int8_t *in, int rank, int8_t *out, int *rank_out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm;
    int P = p + 1, nw = mn + n * P + P * m, l, i, j, k;
    if (!fmt_ok(m, n, P)) return -2;
    memset(out, 0, (size_t)(rank + mn) * nw);
    for (l = 0; l < rank; l++) {
        const int8_t *u = in + (size_t)l * width, *v = u + mn, *w = v + np;
        int8_t *uo = out + (size_t)l * nw, *vo = uo + mn, *wo = vo + n * P;
        memcpy(uo, u, (size_t)mn);
        for (j = 0; j < n; j++)
            for (k = 0; k < p; k++) vo[VIDX(j, k, P)] = v[VIDX(j, k, p)];
        for (k = 0; k < p; k++)
            for (i = 0; i < m; i++) wo[WIDX(k, i, m)] = w[WIDX(k, i, m)];
    }
    for (i = 0; i < m; i++)
        for (j = 0; j < n; j++) {
            int8_t *uo = out + (size_t)(rank + i * n + j) * nw, *vo = uo + mn, *wo = vo + n * P;
            uo[UIDX(i, j, n)] = 1;                 /* a_ij * b_jp -> c_ip */
            vo[VIDX(j, p, P)] = 1;
            wo[WIDX(p, i, m)] = 1;
        }
    *rank_out = rank + mn;
    return 0;
}

int or_meta_merge(int m, int n, int p1, int p2, const int8_t *a, int ra, const int8_t *b, int rb, int8_t *out)
{
    int P = p1 + p2, mn = m * n, nw = mn + n * P + P * m, l, i, j, k;
    int w1 = mn + n * p1 + p1 * m, w2 = mn + n * p2 + p2 * m;
    if (!fmt_ok(m, n, p1) || !fmt_ok(m, n, p2) || !fmt_ok(m, n, P)) return -2;
    memset(out, 0, (size_t)(ra + rb) * nw);
    for (l = 0; l < ra + rb; l++) {
        const int first = l < ra;
        const int pp = first ? p1 : p2, off = first ? 0 : p1;
        const int8_t *u = first ? a + (size_t)l * w1 : b + (size_t)(l - ra) * w2;
        const int8_t *v = u + mn, *w = v + n * pp;
        int8_t *uo = out + (size_t)l * nw, *vo = uo + mn, *wo = vo + n * P;
        memcpy(uo, u, (size_t)mn);
        for (j = 0; j < n; j++)
            for (k = 0; k < pp; k++) vo[VIDX(j, off + k, P)] = v[VIDX(j, k, pp)];
        for (k = 0; k < pp; k++)
            for (i = 0; i < m; i++) wo[WIDX(off + k, i, m)] = w[WIDX(k, i, m)];
    }
    return 0;
}

int or_meta_product(int m1, int n1, int p1, const int8_t *a, int ra, int m2, int n2, int p2, const int8_t *b,
                    int rb, int8_t *out)
{
    int M = m1 * m2, N = n1 * n2, P = p1 * p2, nw = M * N + N * P + P * M;
    int wa = m1 * n1 + n1 * p1 + p1 * m1, wb = m2 * n2 + n2 * p2 + p2 * m2;
    int l1, l2, i1, i2, j1, j2, k1, k2;
    if (!fmt_ok(m1, n1, p1) || !fmt_ok(m2, n2, p2) || !fmt_ok(M, N, P)) return -2;
    memset(out, 0, (size_t)ra * rb * nw);
    for (l1 = 0; l1 < ra; l1++)
        for (l2 = 0; l2 < rb; l2++) {
            const int8_t *ua = a + (size_t)l1 * wa, *va = ua + m1 * n1, *wa_ = va + n1 * p1;
            const int8_t *ub = b + (size_t)l2 * wb, *vb = ub + m2 * n2, *wb_ = vb + n2 * p2;
            int8_t *uo = out + (size_t)(l1 * rb + l2) * nw, *vo = uo + M * N, *wo = vo + N * P;
            for (i1 = 0; i1 < m1; i1++) for (i2 = 0; i2 < m2; i2++)
                for (j1 = 0; j1 < n1; j1++) for (j2 = 0; j2 < n2; j2++)
                    uo[UIDX(i1 * m2 + i2, j1 * n2 + j2, N)] =
                        (int8_t)(ua[UIDX(i1, j1, n1)] * ub[UIDX(i2, j2, n2)]);
            for (j1 = 0; j1 < n1; j1++) for (j2 = 0; j2 < n2; j2++)
                for (k1 = 0; k1 < p1; k1++) for (k2 = 0; k2 < p2; k2++)
                    vo[VIDX(j1 * n2 + j2, k1 * p2 + k2, P)] =
                        (int8_t)(va[VIDX(j1, k1, p1)] * vb[VIDX(j2, k2, p2)]);
            for (k1 = 0; k1 < p1; k1++) for (k2 = 0; k2 < p2; k2++)
                for (i1 = 0; i1 < m1; i1++) for (i2 = 0; i2 < m2; i2++)
                    wo[WIDX(k1 * p2 + k2, i1 * m2 + i2, M)] =
                        (int8_t)(wa_[WIDX(k1, i1, m1)] * wb_[WIDX(k2, i2, m2)]);
        }
    return 0;
}

/* ---------- Alg. 2 Resize, reading R31 ----------
   Decisions from Philox blocks 0x100 and 0x101 of counter (round lo, round hi,
   walker id, block) under key `seed`: x0 < 2^31 -> swap sizes; x1 picks the best
   scheme to try to merge with (same m, n); if not merged and x2 < thr_resize, x3
   picks project (< 0.05) / product with the best picked by y0 (< 0.55) / double
   (< 0.85) / extend.  A result violating R1, max(m,n,p) <= 16
    or r_cap leaves the scheme unchanged.  op_out: bit 0 swapped,
   bits 1.. = 1 merge, 2 project, 3 product, 4 double, 5 extend (0 none). */
static int fits(int m, int n, int p, int rank, int r_cap)
{
    return fmt_ok(m, n, p) && m <= 16 && n <= 16 && p <= 16 && rank >= 1 && rank <= r_cap;
}

static uint32_t uni(uint32_t x, uint32_t n) { return (uint32_t)(((uint64_t)x * n) >> 32); }

int or_resize(int *m, int *n, int *p, int8_t *coeffs, int *rank, int r_cap, int nbest, const int32_t *bfmt,
              const int32_t *brank, const int8_t *const *bcoeffs, uint32_t thr_resize, uint64_t seed,
              uint64_t round, uint64_t walker_id, int *op_out)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t c0[4] = {(uint32_t)round, (uint32_t)(round >> 32), (uint32_t)walker_id, 0x100};
    uint32_t c1[4] = {(uint32_t)round, (uint32_t)(round >> 32), (uint32_t)walker_id, 0x101};
    uint32_t x[4], y[4];
    int M = *m, N = *n, P = *p, r = *rank, op = 0, merged = 0;
    int8_t *tmp = (int8_t *)malloc((size_t)(r_cap + 1) * 3 * OR_MAXLEN + 64);
    or_philox4x32_10(c0, key, x);
    or_philox4x32_10(c1, key, y);
    if (x[0] < 0x80000000u) {
        or_meta_swap_sizes(M, N, P, coeffs, r, tmp);
        memcpy(coeffs, tmp, (size_t)r * (M * N + N * P + P * M));
        { int t = N; N = P; P = t; }
        op |= 1;
    }
    if (nbest > 0) {
        int b = (int)uni(x[1], (uint32_t)nbest);
        if (bfmt[3 * b] == M && bfmt[3 * b + 1] == N && fits(M, N, P + bfmt[3 * b + 2], r + brank[b], r_cap)) {
            or_meta_merge(M, N, P, bfmt[3 * b + 2], coeffs, r, bcoeffs[b], brank[b], tmp);
            P += bfmt[3 * b + 2];
            r += brank[b];
            memcpy(coeffs, tmp, (size_t)r * (M * N + N * P + P * M));
            merged = 1;
            op |= 1 << 1;
        }
    }
    if (!merged && x[2] < thr_resize) {
        uint32_t q = x[3];
        if (q < 214748364u) {                        /* 5% project */
            int nr = 0;
            if (P >= 2 && fits(M, N, P - 1, 1, r_cap)) {
                or_meta_project(M, N, P, coeffs, r, tmp, &nr);
                if (nr >= 1) {
                    P -= 1;
                    r = nr;
                    memcpy(coeffs, tmp, (size_t)r * (M * N + N * P + P * M));
                    op |= 2 << 1;
                }
            }
        } else if (q < 2362232012u) {               /* 50% product with a best scheme */
            if (nbest > 0) {
                int b = (int)uni(y[0], (uint32_t)nbest);
                int m2 = bfmt[3 * b], n2 = bfmt[3 * b + 1], p2 = bfmt[3 * b + 2];
                if (fits(M * m2, N * n2, P * p2, r * brank[b], r_cap)) {
                    int8_t *big = (int8_t *)malloc((size_t)r * brank[b] * 3 * OR_MAXLEN + 64);
                    or_meta_product(M, N, P, coeffs, r, m2, n2, p2, bcoeffs[b], brank[b], big);
                    M *= m2; N *= n2; P *= p2; r *= brank[b];
                    memcpy(coeffs, big, (size_t)r * (M * N + N * P + P * M));
                    free(big);
                    op |= 3 << 1;
                }
            }
        } else if (q < 3650722201u) {               /* 30% double */
            if (fits(M, N, 2 * P, 2 * r, r_cap)) {
                or_meta_merge(M, N, P, P, coeffs, r, coeffs, r, tmp);
                P *= 2;
                r *= 2;
                memcpy(coeffs, tmp, (size_t)r * (M * N + N * P + P * M));
                op |= 4 << 1;
            }
        } else {                                     /* 15% extend */
            int nr = 0;
            if (fits(M, N, P + 1, r + M * N, r_cap)) {
                or_meta_extend(M, N, P, coeffs, r, tmp, &nr);
                P += 1;
                r = nr;
                memcpy(coeffs, tmp, (size_t)r * (M * N + N * P + P * M));
                op |= 5 << 1;
            }
        }
    }
    free(tmp);
    *m = M; *n = N; *p = P; *rank = r;
    if (op_out) *op_out = op;
    return 0;
}
