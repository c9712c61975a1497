/*
 * oracle/scheme.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Schemes as plain int8 rows [u(mn) | v(np) | w(pm)]:
 *   u index a = i*n + j   (coefficient of a_ij)
 *   v index b = j*p + k   (coefficient of b_jk)
 *   w index c = k*m + i   (C^T layout)
 * (reading R2; pinned by T1: the printed (2,2,3:11) scheme verifies only so).
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

static int in_domain(int ring, int x)
{
    if (ring == OR_RING_Z2) return x == 0 || x == 1;
    return x >= -1 && x <= 1;
}

/* Brent equations, PAPER:112-119 (Eq. 1) in the C^T form of PAPER:121-125
   (reading R7):  for every (a,b,c)
       sum_l u_l[a] * v_l[b] * w_l[c]  ==  T(a,b,c),
   T(a,b,c) = 1 iff a = i*n+j, b = j*p+k, c = k*m+i for some (i,j,k), else 0.
   Z_T: exact integer sum.  Z_2: the sum modulo 2.
   Returns 0 on pass, 1 on fail (first failing (a,b,c) in lexicographic order
   written to first_fail), -1 bad arguments, -3 coefficient out of ring. */
int or_verify(int m, int n, int p, int ring, const int8_t *coeffs, int rank,
              int32_t first_fail[3])
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm;
    int a, b, c, l;
    if (first_fail) { first_fail[0] = first_fail[1] = first_fail[2] = -1; }
    if (m < 1 || n < 1 || p < 1 || mn > OR_MAXLEN || np > OR_MAXLEN || pm > OR_MAXLEN ||
        rank < 0 || (rank > 0 && !coeffs))
        return -1;
    for (l = 0; l < rank * width; l++)
        if (!in_domain(ring, coeffs[l])) return -3;
    for (a = 0; a < mn; a++) {
        int i = a / n, j = a % n;
        for (b = 0; b < np; b++) {
            int j2 = b / p, k = b % p;
            for (c = 0; c < pm; c++) {
                int k2 = c / m, i2 = c % m;
                int target = (j == j2 && k == k2 && i == i2) ? 1 : 0;
                long sum = 0;
                int ok;
                for (l = 0; l < rank; l++) {
                    const int8_t *row = coeffs + (size_t)l * width;
                    sum += (long)row[a] * row[mn + b] * row[mn + np + c];
                }
                if (ring == OR_RING_Z2) ok = ((sum % 2 + 2) % 2) == target;
                else ok = (sum == target);
                if (!ok) {
                    if (first_fail) { first_fail[0] = a; first_fail[1] = b; first_fail[2] = c; }
                    return 1;
                }
            }
        }
    }
    return 0;
}

/* Naive additive complexity: nonzero coefficients - 2r - m*p. */
int or_additions(int m, int n, int p, const int8_t *coeffs, int rank)
{
    int width = m * n + n * p + p * m, nnz = 0, l;
    for (l = 0; l < rank * width; l++) nnz += coeffs[l] != 0;
    return nnz - 2 * rank - m * p;
}

/* Sign-symmetry breaking, PAPER:429 and the worked example PAPER:431-505, per
   row (reading R6): if the first nonzero of u is negative, negate u and w; then,
   if the first nonzero of v is negative, negate v and w. */
static int first_nonzero(const int8_t *x, int len)
{
    int e;
    for (e = 0; e < len; e++) if (x[e] != 0) return x[e];
    return 0;
}

void or_normalize_rows(int m, int n, int p, int8_t *coeffs, int rank)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, l, e;
    for (l = 0; l < rank; l++) {
        int8_t *u = coeffs + (size_t)l * width, *v = u + mn, *w = v + np;
        if (first_nonzero(u, mn) < 0) {
            for (e = 0; e < mn; e++) u[e] = (int8_t)-u[e];
            for (e = 0; e < pm; e++) w[e] = (int8_t)-w[e];
        }
        if (first_nonzero(v, np) < 0) {
            for (e = 0; e < np; e++) v[e] = (int8_t)-v[e];
            for (e = 0; e < pm; e++) w[e] = (int8_t)-w[e];
        }
    }
}

/* Naive scheme ("generating naive implementations"): one row per
   product a_ij * b_jk contributing to c_ik, rows ordered l = (i*n + j)*p + k. */
int or_naive(int m, int n, int p, int8_t *coeffs_out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, i, j, k;
    memset(coeffs_out, 0, (size_t)m * n * p * width);
    for (i = 0; i < m; i++)
        for (j = 0; j < n; j++)
            for (k = 0; k < p; k++) {
                int8_t *row = coeffs_out + (size_t)((i * n + j) * p + k) * width;
                row[i * n + j] = 1;
                row[mn + j * p + k] = 1;
                row[mn + np + k * m + i] = 1;
            }
    return m * n * p;
}

/* Rank over Q of a small integer matrix (Bareiss fraction-free elimination). */
int or_matrix_rank(const int8_t *a, int rows, int cols)
{
    long long M[64][64];
    int r, c, rank = 0, i, j;
    long long prev = 1;
    if (rows > 64 || cols > 64) return -1;
    for (r = 0; r < rows; r++)
        for (c = 0; c < cols; c++) M[r][c] = a[r * cols + c];
    for (c = 0; c < cols && rank < rows; c++) {
        int piv = -1;
        for (r = rank; r < rows; r++) if (M[r][c] != 0) { piv = r; break; }
        if (piv < 0) continue;
        if (piv != rank)
            for (j = 0; j < cols; j++) { long long t = M[piv][j]; M[piv][j] = M[rank][j]; M[rank][j] = t; }
        for (i = rank + 1; i < rows; i++) {
            for (j = c + 1; j < cols; j++)
                M[i][j] = (M[rank][c] * M[i][j] - M[i][c] * M[rank][j]) / prev;
            M[i][c] = 0;
        }
        prev = M[rank][c];
        rank++;
    }
    return rank;
}

/* Type invariant: sum_l X^rank U_l Y^rank V_l Z^rank W_l, with
   U_l an m x n matrix, V_l n x p, W_l p x m (the C^T layout: w[k*m+i] at (k,i)). */
int or_type_invariant(int m, int n, int p, const int8_t *coeffs, int rank, int32_t *out)
{
    int mn = m * n, np = n * p, pm = p * m, width = mn + np + pm, l;
    for (l = 0; l < rank; l++) {
        const int8_t *row = coeffs + (size_t)l * width;
        int ru = or_matrix_rank(row, m, n);
        int rv = or_matrix_rank(row + mn, n, p);
        int rw = or_matrix_rank(row + mn + np, p, m);
        if (ru < 0 || rv < 0 || rw < 0) return -1;
        out[(ru * 65 + rv) * 65 + rw] += 1;
    }
    (void)pm;
    return 0;
}

/* Symmetrised polynomial: f(x,y,z) = sum_{pi in S_3} pi( sum_{i=1}^r
 * x^{rank U_i} y^{rank V_i} z^{rank W_i} ).  Written term by term: each term i and each
 * of the six permutations pi of (x, y, z) adds one monomial.  out[(a*65+b)*65+c] +=. */
int or_sym_invariant(int m, int n, int p, const int8_t *coeffs, int rank, int32_t *out)
{
    static const int perms[6][3] = {{0,1,2},{0,2,1},{1,0,2},{1,2,0},{2,0,1},{2,1,0}};
    int mn = m * n, np = n * p, width = mn + np + p * m, l, q;
    for (l = 0; l < rank; l++) {
        const int8_t *row = coeffs + (size_t)l * width;
        int e[3];
        e[0] = or_matrix_rank(row, m, n);             /* exponent of x: rank U_i */
        e[1] = or_matrix_rank(row + mn, n, p);        /* exponent of y: rank V_i */
        e[2] = or_matrix_rank(row + mn + np, p, m);   /* exponent of z: rank W_i */
        if (e[0] < 0 || e[1] < 0 || e[2] < 0) return -1;
        for (q = 0; q < 6; q++) {
            /* pi maps the variables (x, y, z) -> (pi x, pi y, pi z): the exponent of
               variable k after pi is the exponent of the variable pi sent to k */
            int f[3];
            f[perms[q][0]] = e[0];
            f[perms[q][1]] = e[1];
            f[perms[q][2]] = e[2];
            out[(f[0] * 65 + f[1]) * 65 + f[2]] += 1;
        }
    }
    return 0;
}
