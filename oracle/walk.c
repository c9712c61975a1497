/*
 * oracle/walk.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * The RandomWalk of PAPER:297-335 (Algorithm 1) on one scheme, with the moves of
 * PAPER:205-241 (flip, plus, split, reduction, expand), the sign convention of
 * PAPER:426-509, and the readings R8-R23 of DESIGN.md ("Readings") where the
 * paper is silent.  Plain int8 coefficients; every step rebuilds the flip
 * candidate list from scratch (O(r^2)); nothing is incremental, nothing fused.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

enum { RU = 0, RV = 1, RW = 2 };

#define FAC(w, l, X) ((w)->rows + ((size_t)(l) * 3 + (X)) * OR_MAXLEN)
#define BFAC(w, l, X) ((w)->best + ((size_t)(l) * 3 + (X)) * OR_MAXLEN)
#define FNV_PRIME 0x100000001b3ULL
#define DIGEST_INIT 0xcbf29ce484222325ULL

/* step-event flags folded into the digest */
enum { EV_FLIP_OK = 1, EV_FALLBACK = 2, EV_ACCEPT = 4, EV_STRICT = 8, EV_REDUCE = 16,
       EV_PEXPAND = 32, EV_EXPANDED = 64 };

typedef struct { int X, i, j, sigma; } cand_t;

/* ---------- ternary vectors as int8 arrays (the definition of Z_T / Z_2) ---------- */

static int is_zero(const int8_t *x, int len)
{
    int e;
    for (e = 0; e < len; e++) if (x[e] != 0) return 0;
    return 1;
}

static int vec_eq(const int8_t *a, const int8_t *b, int len)
{
    return memcmp(a, b, (size_t)len) == 0;
}

/* a = -b with a != 0 (R4: the zero vector is "equal", never "negated") */
static int vec_negeq(const int8_t *a, const int8_t *b, int len)
{
    int e;
    if (is_zero(a, len)) return 0;
    for (e = 0; e < len; e++) if (a[e] != -b[e]) return 0;
    return 1;
}

/* out = a + sigma*b.  Z_T: valid iff every entry stays in {-1,0,1} (PAPER:197-199,
   "ternary safety").  Z_2: addition = subtraction = XOR. */
static int vec_add(int ring, int8_t *out, const int8_t *a, const int8_t *b, int sigma, int len)
{
    int e, valid = 1;
    for (e = 0; e < len; e++) {
        int s;
        if (ring == OR_RING_Z2) s = (a[e] + b[e]) & 1;
        else {
            s = a[e] + sigma * b[e];
            if (s < -1 || s > 1) valid = 0;
        }
        out[e] = (int8_t)s;
    }
    return valid;
}

static void vec_neg(int8_t *x, int len)
{
    int e;
    for (e = 0; e < len; e++) x[e] = (int8_t)-x[e];
}

static int first_nonzero(const int8_t *x, int len)
{
    int e;
    for (e = 0; e < len; e++) if (x[e] != 0) return x[e];
    return 0;
}

/* PAPER:429 / R6: per row, first nonzero of u and of v made positive, w absorbs
   the sign (alpha u x beta v x gamma w with alpha*beta*gamma = 1).  Z_T only. */
static void normalize_factors(int ring, int8_t *u, int8_t *v, int8_t *w, const int *len)
{
    if (ring != OR_RING_ZT) return;
    if (first_nonzero(u, len[RU]) < 0) { vec_neg(u, len[RU]); vec_neg(w, len[RW]); }
    if (first_nonzero(v, len[RV]) < 0) { vec_neg(v, len[RV]); vec_neg(w, len[RW]); }
}

static void normalize_row(or_walker *w, int l)
{
    normalize_factors(w->ring, FAC(w, l, RU), FAC(w, l, RV), FAC(w, l, RW), w->len);
}

static int row_has_zero(or_walker *w, int l)
{
    return is_zero(FAC(w, l, RU), w->len[RU]) || is_zero(FAC(w, l, RV), w->len[RV]) ||
           is_zero(FAC(w, l, RW), w->len[RW]);
}

static void copy_row(or_walker *w, int dst, int src)
{
    memmove(FAC(w, dst, 0), FAC(w, src, 0), 3 * OR_MAXLEN);
}

static uint32_t word(const or_walker *w, uint64_t seed, int slot)
{
    return or_word(seed, w->step, w->walker_id, slot);
}

/* R9: uniform integer in [0, n) from one 32-bit word */
static uint32_t uniform(uint32_t x, uint32_t n)
{
    return (uint32_t)(((uint64_t)x * n) >> 32);
}

/* ---------- R10: canonical flip-candidate list ---------- */
/* A flip needs two terms sharing a factor, in any role
   (PAPER:241).  U and V compare by equality (normalised nonzero vectors are never
   negatives of each other); W also by negation.
   Order: role X = U, V, W; then i; then j > i. */
static int build_candidates(or_walker *w, cand_t *C)
{
    int X, i, j, n = 0;
    for (X = 0; X < 3; X++)
        for (i = 0; i < w->r; i++) {
            const int8_t *xi = FAC(w, i, X);
            if (is_zero(xi, w->len[X])) continue;
            for (j = i + 1; j < w->r; j++) {
                const int8_t *xj = FAC(w, j, X);
                if (vec_eq(xi, xj, w->len[X])) {
                    C[n].X = X; C[n].i = i; C[n].j = j; C[n].sigma = 1; n++;
                } else if (X == RW && w->ring == OR_RING_ZT && vec_negeq(xi, xj, w->len[X])) {
                    C[n].X = X; C[n].i = i; C[n].j = j; C[n].sigma = -1; n++;
                }
            }
        }
    return n;
}

/* roles (Y,Z) moved by a flip on shared role X, before the e-swap (R11) */
static void flip_roles(int X, int e, int *Y, int *Z)
{
    if (X == RU) { *Y = RV; *Z = RW; }
    else if (X == RV) { *Y = RW; *Z = RU; }
    else { *Y = RU; *Z = RV; }
    if (e) { int t = *Y; *Y = *Z; *Z = t; }
}

/* One flip move on candidate c with variant (d,e) -- PAPER:208-215 applied to
   the role permutation picked by e and the term order picked by d (R11):
       x (x) y_a (x) z_a + s x (x) y_b (x) z_b
     = x (x) (y_a + s y_b) (x) z_a + s x (x) y_b (x) (z_b - z_a)
   Returns 1 and commits (then normalises rows alpha, beta) iff both new factors
   stay in Z_T. */
static int flip_move(or_walker *w, const cand_t *c, int d, int e, int nonzero, int *alpha, int *beta)
{
    int Y, Z, al, be;
    int8_t ny[OR_MAXLEN], nz[OR_MAXLEN];
    flip_roles(c->X, e, &Y, &Z);
    al = d ? c->j : c->i;
    be = d ? c->i : c->j;
    if (!vec_add(w->ring, ny, FAC(w, al, Y), FAC(w, be, Y), c->sigma, w->len[Y])) return 0;
    if (!vec_add(w->ring, nz, FAC(w, be, Z), FAC(w, al, Z), -1, w->len[Z])) return 0;
    if (nonzero && (is_zero(ny, w->len[Y]) || is_zero(nz, w->len[Z]))) return 0;   /* R24 */
    memcpy(FAC(w, al, Y), ny, (size_t)w->len[Y]);
    memcpy(FAC(w, be, Z), nz, (size_t)w->len[Z]);
    normalize_row(w, al);
    normalize_row(w, be);
    *alpha = al;
    *beta = be;
    return 1;
}

/* R11 try_flip: up to K uniform draws over 4|C| (candidate x 2 orders x 2 role
   swaps); the list is not rebuilt between draws. */
static int try_flip(or_walker *w, const cand_t *C, int nC, uint64_t seed, const or_params *prm,
                    int nonzero, int *alpha, int *beta, int *draws)
{
    uint32_t a;
    *draws = 0;
    if (nC == 0) return 0;
    for (a = 0; a < prm->k_flip; a++) {
        int slot = a == 0 ? 0 : 7 + (int)a;
        uint32_t k = uniform(word(w, seed, slot), 4u * (uint32_t)nC);
        (*draws)++;
        if (flip_move(w, &C[k >> 2], (int)(k & 1), (int)((k >> 1) & 1), nonzero, alpha, beta)) return 1;
    }
    return 0;
}

/* ---------- R14 remove with worklist remapping ---------- */
static void remove_row(or_walker *w, int h, int *wl, int *nwl)
{
    int last = w->r - 1, k, n = 0;
    for (k = 0; k < *nwl; k++) if (wl[k] != h) wl[n++] = wl[k];
    *nwl = n;
    if (h != last) {
        copy_row(w, h, last);
        for (k = 0; k < *nwl; k++) if (wl[k] == last) wl[k] = h;
    }
    w->r--;
}

/* ---------- R13 reducible(i,j): two shared factors (any role
   permutation PAPER:241).  Role pairs (A,B,C) tried in the order (U,V,W),
   (U,W,V), (V,W,U); need x_A[i] = x_A[j] and x_B[i] = s x_B[j] (s = -1 allowed
   only for B = W in Z_T); merged x_C = x_C[i] + s x_C[j] must be valid.  The
   merged row is row i with C replaced, then normalised. ---------- */
static int reducible(or_walker *w, int i, int j, int8_t merged[3][OR_MAXLEN])
{
    static const int PAIRS[3][3] = {{RU, RV, RW}, {RU, RW, RV}, {RV, RW, RU}};
    int q;
    for (q = 0; q < 3; q++) {
        int A = PAIRS[q][0], B = PAIRS[q][1], Cr = PAIRS[q][2], sigma, X;
        int8_t nc[OR_MAXLEN];
        if (!vec_eq(FAC(w, i, A), FAC(w, j, A), w->len[A])) continue;
        if (vec_eq(FAC(w, i, B), FAC(w, j, B), w->len[B])) sigma = 1;
        else if (B == RW && w->ring == OR_RING_ZT && vec_negeq(FAC(w, i, B), FAC(w, j, B), w->len[B]))
            sigma = -1;
        else continue;
        if (!vec_add(w->ring, nc, FAC(w, i, Cr), FAC(w, j, Cr), sigma, w->len[Cr])) continue;
        for (X = 0; X < 3; X++) {
            memset(merged[X], 0, OR_MAXLEN);
            memcpy(merged[X], FAC(w, i, X), (size_t)w->len[X]);
        }
        memcpy(merged[Cr], nc, (size_t)w->len[Cr]);
        normalize_factors(w->ring, merged[RU], merged[RV], merged[RW], w->len);
        return 1;
    }
    return 0;
}

static void put_row(or_walker *w, int l, int8_t merged[3][OR_MAXLEN])
{
    int X;
    for (X = 0; X < 3; X++) memcpy(FAC(w, l, X), merged[X], OR_MAXLEN);
}

/* ---------- R12 local reduction after a successful flip ("flip with reduction
   edge checking") ---------- */
static void local_reduce(or_walker *w, int a, int b)
{
    int wl[8], nwl = 2;
    wl[0] = a; wl[1] = b;
    while (nwl > 0) {
        int t = wl[0], k, j;
        for (k = 1; k < nwl; k++) wl[k - 1] = wl[k];
        nwl--;
        if (t >= w->r) continue;
        if (row_has_zero(w, t)) {
            remove_row(w, t, wl, &nwl);
            w->cnt[OR_C_ZERO_REMOVED]++;
            continue;
        }
        for (j = 0; j < w->r; j++) {
            int8_t merged[3][OR_MAXLEN];
            int lo, hi;
            if (j == t) continue;
            if (!reducible(w, t, j, merged)) continue;
            lo = t < j ? t : j;
            hi = t < j ? j : t;
            put_row(w, lo, merged);
            remove_row(w, hi, wl, &nwl);
            w->cnt[OR_C_MERGES]++;
            if (row_has_zero(w, lo)) {
                remove_row(w, lo, wl, &nwl);
                w->cnt[OR_C_ZERO_REMOVED]++;
            } else {
                for (k = nwl; k > 0; k--) wl[k] = wl[k - 1];
                wl[0] = lo;
                nwl++;
            }
            break;
        }
    }
}

/* ---------- R15 reduce_all (Alg.1 "scheme.reduce()") ---------- */
static void reduce_all(or_walker *w)
{
    int changed = 1;
    while (changed) {
        int l, i, j, none = 0;
        changed = 0;
        for (l = 0; l < w->r; l++)
            if (row_has_zero(w, l)) {
                remove_row(w, l, NULL, &none);
                w->cnt[OR_C_ZERO_REMOVED]++;
                changed = 1;
                break;
            }
        if (changed) continue;
        for (i = 0; i < w->r && !changed; i++)
            for (j = i + 1; j < w->r; j++) {
                int8_t merged[3][OR_MAXLEN];
                if (!reducible(w, i, j, merged)) continue;
                put_row(w, i, merged);
                remove_row(w, j, NULL, &none);
                w->cnt[OR_C_MERGES]++;
                if (row_has_zero(w, i)) {
                    remove_row(w, i, NULL, &none);
                    w->cnt[OR_C_ZERO_REMOVED]++;
                }
                changed = 1;
                break;
            }
    }
}

/* ---------- R16 expand = fair coin {plus, split} ---------- */
static const int PERM[6][3] = {{RU, RV, RW}, {RU, RW, RV}, {RV, RU, RW},
                               {RV, RW, RU}, {RW, RU, RV}, {RW, RV, RU}};

static int distinct(int ring, const int8_t *a, const int8_t *b, int len, int role)
{
    if (vec_eq(a, b, len)) return 0;
    if (ring == OR_RING_ZT && vec_negeq(a, b, len)) return 0;
    (void)role;
    return 1;
}

int or_apply_expand(or_walker *w, int plus, int i, int j, int perm)
{
    int A = PERM[perm][0], B = PERM[perm][1], Cr = PERM[perm][2], r = w->r;
    int8_t ai[OR_MAXLEN], aj[OR_MAXLEN], bi[OR_MAXLEN], bj[OR_MAXLEN], ci[OR_MAXLEN], cj[OR_MAXLEN];
    int8_t t1[OR_MAXLEN], t2[OR_MAXLEN], t3[OR_MAXLEN];
    int la = w->len[A], lb = w->len[B], lc = w->len[Cr];
    if (r < 2 || r + 1 > w->R || i == j || i < 0 || j < 0 || i >= r || j >= r) return 0;
    memcpy(ai, FAC(w, i, A), OR_MAXLEN); memcpy(aj, FAC(w, j, A), OR_MAXLEN);
    memcpy(bi, FAC(w, i, B), OR_MAXLEN); memcpy(bj, FAC(w, j, B), OR_MAXLEN);
    memcpy(ci, FAC(w, i, Cr), OR_MAXLEN); memcpy(cj, FAC(w, j, Cr), OR_MAXLEN);
    if (plus) {
        /* u_i(x)v_i(x)w_i + u_j(x)v_j(x)w_j ->
           u_i(x)(v_i+v_j)(x)w_i + u_i(x)v_j(x)(w_j-w_i) + (u_j-u_i)(x)v_j(x)w_j,
           needs u_i != u_j, v_i != v_j, w_i != w_j */
        if (!distinct(w->ring, ai, aj, la, A) || !distinct(w->ring, bi, bj, lb, B) ||
            !distinct(w->ring, ci, cj, lc, Cr))
            return 0;
        memset(t1, 0, OR_MAXLEN); memset(t2, 0, OR_MAXLEN); memset(t3, 0, OR_MAXLEN);
        if (!vec_add(w->ring, t1, bi, bj, 1, lb)) return 0;   /* v_i + v_j */
        if (!vec_add(w->ring, t2, cj, ci, -1, lc)) return 0;  /* w_j - w_i */
        if (!vec_add(w->ring, t3, aj, ai, -1, la)) return 0;  /* u_j - u_i */
        memcpy(FAC(w, i, B), t1, OR_MAXLEN);                  /* row i: (u_i, v_i+v_j, w_i) */
        memcpy(FAC(w, j, A), ai, OR_MAXLEN);                  /* row j: (u_i, v_j, w_j-w_i) */
        memcpy(FAC(w, j, Cr), t2, OR_MAXLEN);
        memcpy(FAC(w, r, A), t3, OR_MAXLEN);                  /* row r: (u_j-u_i, v_j, w_j) */
        memcpy(FAC(w, r, B), bj, OR_MAXLEN);
        memcpy(FAC(w, r, Cr), cj, OR_MAXLEN);
    } else {
        /* -> u_j(x)v_i(x)w_i + u_j(x)v_j(x)w_j + (u_i-u_j)(x)v_i(x)w_i,
           needs u_i != u_j */
        if (!distinct(w->ring, ai, aj, la, A)) return 0;
        memset(t3, 0, OR_MAXLEN);
        if (!vec_add(w->ring, t3, ai, aj, -1, la)) return 0;  /* u_i - u_j */
        memcpy(FAC(w, i, A), aj, OR_MAXLEN);                  /* row i: (u_j, v_i, w_i) */
        memcpy(FAC(w, r, A), t3, OR_MAXLEN);                  /* row r: (u_i-u_j, v_i, w_i) */
        memcpy(FAC(w, r, B), bi, OR_MAXLEN);
        memcpy(FAC(w, r, Cr), ci, OR_MAXLEN);
    }
    normalize_row(w, i);
    normalize_row(w, j);
    normalize_row(w, r);
    w->r = r + 1;
    return 1;
}

static int expand(or_walker *w, uint64_t seed)
{
    int plus, i, j, perm;
    if (w->r < 2 || w->r + 1 > w->R) return 0;
    plus = word(w, seed, 4) < 0x80000000u;
    i = (int)uniform(word(w, seed, 5), (uint32_t)w->r);
    j = (int)uniform(word(w, seed, 6), (uint32_t)(w->r - 1));
    if (j >= i) j++;
    perm = (int)uniform(word(w, seed, 7), 6u);
    return or_apply_expand(w, plus, i, j, perm);
}

/* ---------- helpers ---------- */
static void rows_to_coeffs(const or_walker *w, const int8_t *rows, int rank, int8_t *out)
{
    int width = w->len[0] + w->len[1] + w->len[2], l, X;
    for (l = 0; l < rank; l++) {
        int8_t *dst = out + (size_t)l * width;
        for (X = 0; X < 3; X++) {
            memcpy(dst, rows + ((size_t)l * 3 + X) * OR_MAXLEN, (size_t)w->len[X]);
            dst += w->len[X];
        }
    }
}

static void digest_mix(or_walker *w, uint64_t ev)
{
    w->digest = (w->digest ^ ev) * FNV_PRIME;
    w->digest ^= w->digest >> 32;
}

/* naive additions of the first `rank` rows of a row array */
static int rows_additions(const or_walker *w, const int8_t *rows, int rank)
{
    int l, X, e, nnz = 0;
    for (l = 0; l < rank; l++)
        for (X = 0; X < 3; X++)
            for (e = 0; e < w->len[X]; e++) nnz += rows[((size_t)l * 3 + X) * OR_MAXLEN + e] != 0;
    return nnz - 2 * rank - w->m * w->p;
}

/* ---------- R24: one step of naive-complexity minimisation ----------
   Random flips without reduction edges: try_flip (R11) where a draw is also
   rejected if a new factor is zero; no local reduction, no reduce_all, no expand.
   After a flip, the best scheme is replaced if (rank, additions) is smaller, or
   equal with the 1% plateau acceptance (PAPER:310-313 applied to additions). */
static void complexity_step(or_walker *w, uint64_t seed, const or_params *prm, cand_t *C, int8_t *vbuf)
{
    int nC, ok, alpha = 0, beta = 0, draws = 0;
    uint32_t flags = 0;
    uint64_t ev;
    nC = build_candidates(w, C);
    ok = try_flip(w, C, nC, seed, prm, 1, &alpha, &beta, &draws);
    w->cnt[OR_C_DRAWS] += (uint64_t)draws;
    if (!ok) {
        w->cnt[OR_C_FLIP_FAIL]++;
        alpha = beta = 0;
    } else {
        int adds = rows_additions(w, w->rows, w->r);
        int better = w->r < w->best_r || (w->r == w->best_r && adds < w->best_adds);
        w->cnt[OR_C_FLIPS]++;
        flags |= EV_FLIP_OK;
        if (better || (w->r == w->best_r && adds == w->best_adds && word(w, seed, 1) < prm->thr_accept_eq)) {
            w->best_r = w->r;
            w->best_adds = adds;
            memcpy(w->best, w->rows, (size_t)w->r * 3 * OR_MAXLEN);
            w->cnt[OR_C_BEST_COPIES]++;
            flags |= EV_ACCEPT;
            if (better) {
                int32_t ff[3];
                flags |= EV_STRICT;
                w->cnt[OR_C_IMPROVEMENTS]++;
                rows_to_coeffs(w, w->best, w->best_r, vbuf);
                if (or_verify(w->m, w->n, w->p, w->ring, vbuf, w->best_r, ff) != 0)
                    w->cnt[OR_C_VERIFY_FAIL]++;
            }
        }
    }
    ev = (uint64_t)(uint32_t)w->r | ((uint64_t)(uint32_t)(w->best_adds & 1023) << 10) |
         ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) | ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
    digest_mix(w, ev);
    w->cnt[OR_C_STEPS]++;
    w->step++;
}

/* ---------- R17: one Alg.1 iteration ---------- */
static void walk_step(or_walker *w, uint64_t seed, const or_params *prm, cand_t *C, int8_t *vbuf)
{
    int nC, ok, alpha = 0, beta = 0, draws = 0;
    uint32_t flags = 0;
    uint64_t ev;
    nC = build_candidates(w, C);
    ok = try_flip(w, C, nC, seed, prm, 0, &alpha, &beta, &draws);
    w->cnt[OR_C_DRAWS] += (uint64_t)draws;
    if (!ok) {
        /* if not try_flip: expand; continue */
        int e = expand(w, seed);
        w->cnt[OR_C_FLIP_FAIL]++;
        w->cnt[e ? OR_C_EXPAND_OK : OR_C_EXPAND_REJECT]++;
        flags |= EV_FALLBACK | (e ? EV_EXPANDED : 0);
        alpha = beta = 0;
    } else {
        w->cnt[OR_C_FLIPS]++;
        flags |= EV_FLIP_OK;
        local_reduce(w, alpha, beta);                                   /* R12 */
        /* PAPER:310-313 */
        if (w->r < w->best_r || (w->r == w->best_r && word(w, seed, 1) < prm->thr_accept_eq)) {
            int strict = w->r < w->best_r;
            w->best_r = w->r;
            w->best_adds = rows_additions(w, w->rows, w->r);
            memcpy(w->best, w->rows, (size_t)w->r * 3 * OR_MAXLEN);
            w->cnt[OR_C_BEST_COPIES]++;
            flags |= EV_ACCEPT;
            if (strict) {
                int32_t ff[3];
                flags |= EV_STRICT;
                w->cnt[OR_C_IMPROVEMENTS]++;
                rows_to_coeffs(w, w->best, w->best_r, vbuf);            /* R19 */
                if (or_verify(w->m, w->n, w->p, w->ring, vbuf, w->best_r, ff) != 0)
                    w->cnt[OR_C_VERIFY_FAIL]++;
            }
        }
        /* PAPER:315-317 */
        if (word(w, seed, 2) < prm->thr_reduce) {
            w->cnt[OR_C_REDUCE_CALLS]++;
            flags |= EV_REDUCE;
            reduce_all(w);
        }
        /* PAPER:319-321 */
        if (word(w, seed, 3) < prm->thr_expand && w->r <= w->best_r + prm->expand_slack) {
            int e = expand(w, seed);
            flags |= EV_PEXPAND | (e ? EV_EXPANDED : 0);
            w->cnt[e ? OR_C_EXPAND_OK : OR_C_EXPAND_REJECT]++;
        }
    }
    ev = (uint64_t)(uint32_t)w->r | ((uint64_t)(uint32_t)w->best_r << 10) | ((uint64_t)flags << 20) |
         ((uint64_t)alpha << 32) | ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
    digest_mix(w, ev);
    w->cnt[OR_C_STEPS]++;
    w->step++;
}

/* ---------- public ---------- */
int or_walker_init(or_walker *w, int m, int n, int p, int ring, int R, uint64_t walker_id)
{
    memset(w, 0, sizeof(*w));
    if (m < 1 || n < 1 || p < 1 || m * n > OR_MAXLEN || n * p > OR_MAXLEN || p * m > OR_MAXLEN ||
        R < 1 || R > 512 || (ring != OR_RING_ZT && ring != OR_RING_Z2))
        return -1;
    w->m = m; w->n = n; w->p = p; w->ring = ring; w->R = R;
    w->len[0] = m * n; w->len[1] = n * p; w->len[2] = p * m;
    w->walker_id = walker_id;
    w->rows = (int8_t *)calloc((size_t)(R + 1) * 3 * OR_MAXLEN, 1);
    w->best = (int8_t *)calloc((size_t)(R + 1) * 3 * OR_MAXLEN, 1);
    if (!w->rows || !w->best) return -1;
    return 0;
}

void or_walker_free(or_walker *w)
{
    free(w->rows);
    free(w->best);
    w->rows = w->best = NULL;
}

static int load_rows(or_walker *w, const int8_t *coeffs, int rank)
{
    int width = w->len[0] + w->len[1] + w->len[2], l, X, e;
    if (rank < 1 || rank > w->R) return -2;
    for (l = 0; l < rank * width; l++) {
        int x = coeffs[l];
        if (w->ring == OR_RING_Z2 ? (x != 0 && x != 1) : (x < -1 || x > 1)) return -3;
    }
    memset(w->rows, 0, (size_t)(w->R + 1) * 3 * OR_MAXLEN);
    for (l = 0; l < rank; l++) {
        const int8_t *src = coeffs + (size_t)l * width;
        for (X = 0; X < 3; X++) {
            for (e = 0; e < w->len[X]; e++) FAC(w, l, X)[e] = src[e];
            src += w->len[X];
        }
    }
    w->r = rank;
    for (l = 0; l < rank; l++) {
        if (row_has_zero(w, l)) return -1;   /* seeds carry no zero factors (R5) */
        normalize_row(w, l);
    }
    return 0;
}

/* a seeded scheme is normalised and is the walker's
   initial best (rank assessment). */
int or_seed_rows(or_walker *w, const int8_t *coeffs, int rank)
{
    int rc;
    int32_t ff[3];
    if (or_verify(w->m, w->n, w->p, w->ring, coeffs, rank, ff) != 0) return -4;
    rc = load_rows(w, coeffs, rank);
    if (rc) return rc;
    memcpy(w->best, w->rows, (size_t)(w->R + 1) * 3 * OR_MAXLEN);
    w->best_r = w->r;
    w->best_adds = rows_additions(w, w->rows, w->r);
    w->step = 0;
    w->digest = DIGEST_INIT;
    memset(w->cnt, 0, sizeof(w->cnt));
    return 0;
}

int or_seed_naive(or_walker *w)
{
    int rank = w->m * w->n * w->p, rc;
    int8_t *c;
    if (rank > w->R) return -2;
    c = (int8_t *)malloc((size_t)rank * (w->len[0] + w->len[1] + w->len[2]));
    or_naive(w->m, w->n, w->p, c);
    rc = or_seed_rows(w, c, rank);
    free(c);
    return rc;
}

void or_walk(or_walker *w, uint64_t steps, uint64_t seed, const or_params *prm)
{
    uint64_t s;
    size_t maxc = (size_t)3 * w->R * (w->R + 1) / 2 + 1;
    cand_t *C = (cand_t *)malloc(maxc * sizeof(cand_t));
    int8_t *vbuf = (int8_t *)malloc((size_t)(w->R + 1) * (w->len[0] + w->len[1] + w->len[2]));
    for (s = 0; s < steps; s++) {
        if (prm->mode == 1) complexity_step(w, seed, prm, C, vbuf);
        else walk_step(w, seed, prm, C, vbuf);
    }
    free(C);
    free(vbuf);
}

int or_get_rows(const or_walker *w, int which, int8_t *coeffs_out)
{
    int rank = which ? w->best_r : w->r;
    rows_to_coeffs(w, which ? w->best : w->rows, rank, coeffs_out);
    return rank;
}

/* R23 restart: re-seed from a pool scheme; step counter and counters continue. */
void or_restart(or_walker *w, const int8_t *coeffs, int rank)
{
    if (load_rows(w, coeffs, rank) != 0) return;
    memcpy(w->best, w->rows, (size_t)(w->R + 1) * 3 * OR_MAXLEN);
    w->best_r = w->r;
    w->best_adds = rows_additions(w, w->rows, w->r);
    digest_mix(w, 0xA5A5000000000000ULL | (uint64_t)(uint32_t)rank);
}

int or_count_candidates(or_walker *w)
{
    size_t maxc = (size_t)3 * w->R * (w->R + 1) / 2 + 1;
    cand_t *C = (cand_t *)malloc(maxc * sizeof(cand_t));
    int n = build_candidates(w, C);
    free(C);
    return n;
}

int or_get_candidate(or_walker *w, int idx, int32_t out[4])
{
    size_t maxc = (size_t)3 * w->R * (w->R + 1) / 2 + 1;
    cand_t *C = (cand_t *)malloc(maxc * sizeof(cand_t));
    int n = build_candidates(w, C);
    if (idx < 0 || idx >= n) { free(C); return -1; }
    out[0] = C[idx].X; out[1] = C[idx].i; out[2] = C[idx].j; out[3] = C[idx].sigma;
    free(C);
    return 0;
}

int or_apply_flip(or_walker *w, int cand, int d, int e)
{
    size_t maxc = (size_t)3 * w->R * (w->R + 1) / 2 + 1;
    cand_t *C = (cand_t *)malloc(maxc * sizeof(cand_t));
    int n = build_candidates(w, C), a, b, ok = 0;
    if (cand >= 0 && cand < n) ok = flip_move(w, &C[cand], d, e, 0, &a, &b);
    free(C);
    return ok;
}

void or_reduce_all_public(or_walker *w) { reduce_all(w); }
void or_local_reduce_public(or_walker *w, int a, int b) { local_reduce(w, a, b); }

int or_run_walkers(int m, int n, int p, int ring, int R, int64_t count, uint64_t id_base,
                   const uint64_t *ids, const int8_t *seed_coeffs, int seed_rank, uint64_t steps, uint64_t seed,
                   const or_params *prm, int threads,
                   int32_t *r_out, int32_t *best_r_out, uint64_t *digest_out,
                   uint64_t *cnt_out, int8_t *rows_out, int8_t *best_out)
{
    int64_t k;
    int width = m * n + n * p + p * m, err = 0;
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads) reduction(| : err)
    for (k = 0; k < count; k++) {
        or_walker w;
        int rc = or_walker_init(&w, m, n, p, ring, R, ids ? ids[k] : id_base + (uint64_t)k);
        if (rc == 0) rc = seed_rank > 0 ? or_seed_rows(&w, seed_coeffs, seed_rank) : or_seed_naive(&w);
        if (rc != 0) { err |= 1; or_walker_free(&w); continue; }
        or_walk(&w, steps, seed, prm);
        if (r_out) r_out[k] = w.r;
        if (best_r_out) best_r_out[k] = w.best_r;
        if (digest_out) digest_out[k] = w.digest;
        if (cnt_out) memcpy(cnt_out + k * OR_NCNT, w.cnt, sizeof(w.cnt));
        if (rows_out) {
            memset(rows_out + (size_t)k * R * width, 0, (size_t)R * width);
            or_get_rows(&w, 0, rows_out + (size_t)k * R * width);
        }
        if (best_out) {
            memset(best_out + (size_t)k * R * width, 0, (size_t)R * width);
            or_get_rows(&w, 1, best_out + (size_t)k * R * width);
        }
        or_walker_free(&w);
    }
    return err ? -1 : 0;
}
