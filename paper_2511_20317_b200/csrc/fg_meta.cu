// fg_meta.cu -- host-side meta operators of PAPER:243-262 (section 3.3.2) on bit
// planes: transpose, rotate, swap sizes, project, extend, merge, double, product.
// They orchestrate between walks (north star: "pool-level meta operations stay in
// plain host C orchestration outside the hot path"); readings R25-R30 in DESIGN.md.
// Each operator is a fixed permutation / scatter of factor bits (an index map built
// once per call) applied to the digit and sign words of every row; the product is
// a Kronecker product of set bits.  Independent of oracle/meta.c.
#include <algorithm>
#include <array>
#include <cstring>
#include <vector>
#include "fg_internal.h"

namespace {

struct Sch {                         // one scheme as bit planes, format (m, n, p)
    int m, n, p;
    std::vector<uint64_t> d[3], s[3];    // per role, one word per row
    int rank() const { return (int)d[0].size(); }
    int len(int X) const { return X == 0 ? m * n : (X == 1 ? n * p : p * m); }
};

bool fmt_ok(int m, int n, int p)
{
    return m >= 1 && n >= 1 && p >= 1 && m * n <= 64 && n * p <= 64 && p * m <= 64;
}

int load(int m, int n, int p, int ring, const int8_t *in, int rank, Sch &o)
{
    if (!fmt_ok(m, n, p)) return FG_E_CAPACITY;
    if (rank < 0 || (rank > 0 && !in)) return FG_E_ARG;
    o.m = m; o.n = n; o.p = p;
    const int w = m * n + n * p + p * m;
    for (int X = 0; X < 3; ++X) { o.d[X].assign(rank, 0); o.s[X].assign(rank, 0); }
    for (int l = 0; l < rank; ++l) {
        int off = 0;
        for (int X = 0; X < 3; ++X) {
            for (int e = 0; e < o.len(X); ++e) {
                const int v = in[(size_t)l * w + off + e];
                if (v == 0) continue;
                if (v == 1) o.d[X][l] |= 1ull << e;
                else if (v == -1 && ring == FG_ZT) { o.d[X][l] |= 1ull << e; o.s[X][l] |= 1ull << e; }
                else return FG_E_DOMAIN;
            }
            off += o.len(X);
        }
    }
    return FG_OK;
}

void store(const Sch &a, int8_t *out)
{
    const int w = a.m * a.n + a.n * a.p + a.p * a.m;
    for (int l = 0; l < a.rank(); ++l) {
        int off = 0;
        for (int X = 0; X < 3; ++X) {
            for (int e = 0; e < a.len(X); ++e)
                out[(size_t)l * w + off + e] = ((a.d[X][l] >> e) & 1) ? (((a.s[X][l] >> e) & 1) ? -1 : 1) : 0;
            off += a.len(X);
        }
    }
}

// out bit map[e] <- in bit e (map[e] < 0: dropped)
uint64_t scatter(uint64_t x, const std::vector<int> &map)
{
    uint64_t o = 0;
    for (uint64_t t = x; t; t &= t - 1) {
        const int e = __builtin_ctzll(t);
        if (map[e] >= 0) o |= 1ull << map[e];
    }
    return o;
}

// role `dst` of b <- role `src` of a through the bit map
void remap(const Sch &a, int src, Sch &b, int dst, const std::vector<int> &map)
{
    b.d[dst].resize(a.rank());
    b.s[dst].resize(a.rank());
    for (int l = 0; l < a.rank(); ++l) {
        b.d[dst][l] = scatter(a.d[src][l], map);
        b.s[dst][l] = scatter(a.s[src][l], map);
    }
}

// transpose: C = AB <=> C^T = B^T A^T, (m,n,p) -> (p,n,m)
Sch transpose(const Sch &a)
{
    const int m = a.m, n = a.n, p = a.p;
    Sch b;
    b.m = p; b.n = n; b.p = m;
    std::vector<int> mu(m * n), mv(n * p), mw(p * m);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) mu[i * n + j] = j * m + i;      // A_ij -> B'_ji (B' is n x m)
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < p; ++k) mv[j * p + k] = k * n + j;      // B_jk -> A'_kj (A' is p x n)
    for (int k = 0; k < p; ++k)
        for (int i = 0; i < m; ++i) mw[k * m + i] = i * p + k;      // c_ik -> c'_ki, stored C'^T
    remap(a, 1, b, 0, mv);
    remap(a, 0, b, 1, mu);
    remap(a, 2, b, 2, mw);
    return b;
}

// cyclic symmetry: (u, v, w) -> (v, w, u), (m,n,p) -> (n,p,m), bit positions unchanged
Sch rotate(const Sch &a)
{
    Sch b;
    b.m = a.n; b.n = a.p; b.p = a.m;
    b.d[0] = a.d[1]; b.s[0] = a.s[1];
    b.d[1] = a.d[2]; b.s[1] = a.s[2];
    b.d[2] = a.d[0]; b.s[2] = a.s[0];
    return b;
}

// B, C column k of a (p columns) -> column off + k of P columns
void columns(const Sch &a, int P, int off, Sch &b)
{
    const int m = a.m, n = a.n, p = a.p;
    std::vector<int> mv(n * p), mw(p * m);
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < p; ++k) mv[j * p + k] = (off + k) < P ? j * P + off + k : -1;
    for (int k = 0; k < p; ++k)
        for (int i = 0; i < m; ++i) mw[k * m + i] = (off + k) < P ? (off + k) * m + i : -1;
    b.d[0] = a.d[0]; b.s[0] = a.s[0];
    remap(a, 1, b, 1, mv);
    remap(a, 2, b, 2, mw);
}

void append(Sch &a, const Sch &b)
{
    for (int X = 0; X < 3; ++X) {
        a.d[X].insert(a.d[X].end(), b.d[X].begin(), b.d[X].end());
        a.s[X].insert(a.s[X].end(), b.s[X].begin(), b.s[X].end());
    }
}

}  // namespace

extern "C" {

int fg_meta_transpose(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out)
{
    Sch a;
    int rc = load(m, n, p, ring, in, rank, a);
    if (rc != FG_OK) return rc;
    if (!out) return FG_E_ARG;
    store(transpose(a), out);
    return FG_OK;
}

int fg_meta_rotate(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out)
{
    Sch a;
    int rc = load(m, n, p, ring, in, rank, a);
    if (rc != FG_OK) return rc;
    if (!out) return FG_E_ARG;
    store(rotate(a), out);
    return FG_OK;
}

int fg_meta_swap_sizes(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out)
{
    Sch a;
    int rc = load(m, n, p, ring, in, rank, a);
    if (rc != FG_OK) return rc;
    if (!out) return FG_E_ARG;
    store(rotate(rotate(transpose(a))), out);   // (m,n,p) -> (p,n,m) -> (n,m,p) -> (m,p,n)
    return FG_OK;
}

int fg_meta_project(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out, int *rank_out)
{
    Sch a;
    if (p < 2) return FG_E_ARG;
    int rc = load(m, n, p, ring, in, rank, a);
    if (rc != FG_OK) return rc;
    if (!out || !rank_out) return FG_E_ARG;
    Sch b;
    b.m = m; b.n = n; b.p = p - 1;
    columns(a, p - 1, 0, b);                    // the last column of B and C is dropped
    Sch c;
    c.m = m; c.n = n; c.p = p - 1;
    for (int l = 0; l < b.rank(); ++l) {        // terms with a zero factor vanish
        if (!b.d[0][l] || !b.d[1][l] || !b.d[2][l]) continue;
        for (int X = 0; X < 3; ++X) { c.d[X].push_back(b.d[X][l]); c.s[X].push_back(b.s[X][l]); }
    }
    store(c, out);
    *rank_out = c.rank();
    return FG_OK;
}

int fg_meta_extend(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out, int *rank_out)
{
    Sch a;
    if (!fmt_ok(m, n, p + 1)) return FG_E_CAPACITY;
    int rc = load(m, n, p, ring, in, rank, a);
    if (rc != FG_OK) return rc;
    if (!out || !rank_out) return FG_E_ARG;
    Sch b;
    b.m = m; b.n = n; b.p = p + 1;
    columns(a, p + 1, 0, b);
    Sch nv;                                       // naive (m,n,1) for the new column p
    nv.m = m; nv.n = n; nv.p = p + 1;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            nv.d[0].push_back(1ull << (i * n + j)); nv.s[0].push_back(0);
            nv.d[1].push_back(1ull << (j * (p + 1) + p)); nv.s[1].push_back(0);
            nv.d[2].push_back(1ull << (p * m + i)); nv.s[2].push_back(0);
        }
    append(b, nv);
    store(b, out);
    *rank_out = b.rank();
    return FG_OK;
}

int fg_meta_merge(int m, int n, int p1, int p2, int ring, const int8_t *a_in, int ra, const int8_t *b_in, int rb,
                  int8_t *out)
{
    if (!fmt_ok(m, n, p1 + p2)) return FG_E_CAPACITY;
    Sch a, b;
    int rc = load(m, n, p1, ring, a_in, ra, a);
    if (rc == FG_OK) rc = load(m, n, p2, ring, b_in, rb, b);
    if (rc != FG_OK) return rc;
    if (!out) return FG_E_ARG;
    const int P = p1 + p2;
    Sch x, y;
    x.m = y.m = m; x.n = y.n = n; x.p = y.p = P;
    columns(a, P, 0, x);                          // C1 = A B1 in columns 0 .. p1-1
    columns(b, P, p1, y);                         // C2 = A B2 in columns p1 .. P-1
    append(x, y);
    store(x, out);
    return FG_OK;
}

int fg_meta_double(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out)
{
    return fg_meta_merge(m, n, p, p, ring, in, rank, in, rank, out);
}

int fg_meta_product(int m1, int n1, int p1, const int8_t *a_in, int ra, int m2, int n2, int p2, const int8_t *b_in,
                    int rb, int ring, int8_t *out)
{
    const int M = m1 * m2, N = n1 * n2, P = p1 * p2;
    if (!fmt_ok(M, N, P)) return FG_E_CAPACITY;
    Sch a, b;
    int rc = load(m1, n1, p1, ring, a_in, ra, a);
    if (rc == FG_OK) rc = load(m2, n2, p2, ring, b_in, rb, b);
    if (rc != FG_OK) return rc;
    if (!out) return FG_E_ARG;
    // Kronecker index of (outer element e1 of a's factor, inner element e2 of b's)
    auto kidx = [&](int X, int e1, int e2) {
        int r1, c1, r2, c2, rows2, cols, cols1, cols2;
        if (X == 0) { cols1 = n1; cols2 = n2; rows2 = m2; cols = N; }
        else if (X == 1) { cols1 = p1; cols2 = p2; rows2 = n2; cols = P; }
        else { cols1 = m1; cols2 = m2; rows2 = p2; cols = M; }
        r1 = e1 / cols1; c1 = e1 % cols1; r2 = e2 / cols2; c2 = e2 % cols2;
        return (r1 * rows2 + r2) * cols + (c1 * cols2 + c2);
    };
    Sch c;
    c.m = M; c.n = N; c.p = P;
    for (int l1 = 0; l1 < ra; ++l1)
        for (int l2 = 0; l2 < rb; ++l2)
            for (int X = 0; X < 3; ++X) {
                uint64_t d = 0, s = 0;
                for (uint64_t t1 = a.d[X][l1]; t1; t1 &= t1 - 1) {
                    const int e1 = __builtin_ctzll(t1);
                    for (uint64_t t2 = b.d[X][l2]; t2; t2 &= t2 - 1) {
                        const int e2 = __builtin_ctzll(t2);
                        const int E = kidx(X, e1, e2);
                        d |= 1ull << E;
                        if (ring == FG_ZT && (((a.s[X][l1] >> e1) ^ (b.s[X][l2] >> e2)) & 1)) s |= 1ull << E;
                    }
                }
                c.d[X].push_back(d);
                c.s[X].push_back(s);
            }
    store(c, out);
    return FG_OK;
}

// ---- Alg. 2 Resize, reading R31 ----
static void philox_host(uint32_t c[4], uint32_t k0, uint32_t k1, uint32_t o[4])
{
    uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
    for (int i = 0; i < 10; ++i) {
        if (i) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t a = (uint64_t)0xD2511F53u * x0, b = (uint64_t)0xCD9E8D57u * x2;
        const uint32_t n0 = (uint32_t)(b >> 32) ^ x1 ^ k0, n2 = (uint32_t)(a >> 32) ^ x3 ^ k1;
        x0 = n0; x1 = (uint32_t)b; x2 = n2; x3 = (uint32_t)a;
    }
    o[0] = x0; o[1] = x1; o[2] = x2; o[3] = x3;
}

static bool envelope(int m, int n, int p, int rank, int r_cap)
{
    return fmt_ok(m, n, p) && m <= 16 && n <= 16 && p <= 16 && rank >= 1 && rank <= r_cap;
}

int fg_resize(int *m, int *n, int *p, int ring, int8_t *coeffs, int *rank, int r_cap, int nbest,
              const int32_t *bfmt, const int32_t *brank, const int8_t *const *bcoeffs, uint32_t thr_resize,
              uint64_t seed, uint64_t round, uint64_t walker_id, int *op_out)
{
    if (!m || !n || !p || !coeffs || !rank || r_cap < 1 || nbest < 0 || (nbest > 0 && (!bfmt || !brank || !bcoeffs)))
        return FG_E_ARG;
    Sch a;
    int rc = load(*m, *n, *p, ring, coeffs, *rank, a);
    if (rc != FG_OK) return rc;
    uint32_t c0[4] = {(uint32_t)round, (uint32_t)(round >> 32), (uint32_t)walker_id, 0x100u};
    uint32_t c1[4] = {(uint32_t)round, (uint32_t)(round >> 32), (uint32_t)walker_id, 0x101u};
    uint32_t x[4], y[4];
    philox_host(c0, (uint32_t)seed, (uint32_t)(seed >> 32), x);
    philox_host(c1, (uint32_t)seed, (uint32_t)(seed >> 32), y);
    auto pick = [&](uint32_t w) { return (int)(((uint64_t)w * (uint32_t)nbest) >> 32); };
    int op = 0;
    if (x[0] < 0x80000000u) { a = rotate(rotate(transpose(a))); op |= 1; }       // swap sizes
    bool merged = false;
    if (nbest > 0) {
        const int b = pick(x[1]);
        if (bfmt[3 * b] == a.m && bfmt[3 * b + 1] == a.n &&
            envelope(a.m, a.n, a.p + bfmt[3 * b + 2], a.rank() + brank[b], r_cap)) {
            Sch bb;
            rc = load(bfmt[3 * b], bfmt[3 * b + 1], bfmt[3 * b + 2], ring, bcoeffs[b], brank[b], bb);
            if (rc != FG_OK) return rc;
            const int P = a.p + bb.p;
            Sch x1, y1;
            x1.m = y1.m = a.m; x1.n = y1.n = a.n; x1.p = y1.p = P;
            columns(a, P, 0, x1);
            columns(bb, P, a.p, y1);
            append(x1, y1);
            a = x1;
            merged = true;
            op |= 1 << 1;
        }
    }
    if (!merged && x[2] < thr_resize) {
        const uint32_t q = x[3];
        if (q < 214748364u) {                                   // 5% project
            if (a.p >= 2 && envelope(a.m, a.n, a.p - 1, 1, r_cap)) {
                Sch b;
                b.m = a.m; b.n = a.n; b.p = a.p - 1;
                columns(a, a.p - 1, 0, b);
                Sch c;
                c.m = b.m; c.n = b.n; c.p = b.p;
                for (int l = 0; l < b.rank(); ++l) {
                    if (!b.d[0][l] || !b.d[1][l] || !b.d[2][l]) continue;
                    for (int X = 0; X < 3; ++X) { c.d[X].push_back(b.d[X][l]); c.s[X].push_back(b.s[X][l]); }
                }
                if (c.rank() >= 1) { a = c; op |= 2 << 1; }
            }
        } else if (q < 2362232012u) {                           // 50% product with a best scheme
            if (nbest > 0) {
                const int b = pick(y[0]);
                const int m2 = bfmt[3 * b], n2 = bfmt[3 * b + 1], p2 = bfmt[3 * b + 2];
                if (envelope(a.m * m2, a.n * n2, a.p * p2, a.rank() * brank[b], r_cap)) {
                    std::vector<int8_t> cur((size_t)a.rank() * (a.m * a.n + a.n * a.p + a.p * a.m));
                    store(a, cur.data());
                    const int M = a.m * m2, N = a.n * n2, P = a.p * p2, R = a.rank() * brank[b];
                    std::vector<int8_t> outv((size_t)R * (M * N + N * P + P * M));
                    rc = fg_meta_product(a.m, a.n, a.p, cur.data(), a.rank(), m2, n2, p2, bcoeffs[b], brank[b], ring,
                                         outv.data());
                    if (rc != FG_OK) return rc;
                    rc = load(M, N, P, ring, outv.data(), R, a);
                    if (rc != FG_OK) return rc;
                    op |= 3 << 1;
                }
            }
        } else if (q < 3650722201u) {                           // 30% double
            if (envelope(a.m, a.n, 2 * a.p, 2 * a.rank(), r_cap)) {
                const int P = 2 * a.p;
                Sch x1, y1;
                x1.m = y1.m = a.m; x1.n = y1.n = a.n; x1.p = y1.p = P;
                columns(a, P, 0, x1);
                columns(a, P, a.p, y1);
                append(x1, y1);
                a = x1;
                op |= 4 << 1;
            }
        } else {                                                // 15% extend
            if (envelope(a.m, a.n, a.p + 1, a.rank() + a.m * a.n, r_cap)) {
                Sch b;
                b.m = a.m; b.n = a.n; b.p = a.p + 1;
                columns(a, a.p + 1, 0, b);
                for (int i = 0; i < a.m; ++i)
                    for (int j = 0; j < a.n; ++j) {
                        b.d[0].push_back(1ull << (i * a.n + j)); b.s[0].push_back(0);
                        b.d[1].push_back(1ull << (j * (a.p + 1) + a.p)); b.s[1].push_back(0);
                        b.d[2].push_back(1ull << (a.p * a.m + i)); b.s[2].push_back(0);
                    }
                a = b;
                op |= 5 << 1;
            }
        }
    }
    store(a, coeffs);
    *m = a.m; *n = a.n; *p = a.p; *rank = a.rank();
    if (op_out) *op_out = op;
    return FG_OK;
}

// ---- isotropy invariants and a canonical key for pool dedup ----
// Rank over Q of a factor matrix, computed over GF(2^31 - 1): every minor of a
// ternary matrix with rows*cols <= 64 has order <= 8, so |minor| <= 8^4 (Hadamard)
// < 2^31 - 1 and the modular rank equals the rational one.
static int rank_mod_p(const int8_t *a, int rows, int cols)
{
    const int64_t P = 2147483647;
    int64_t M[64][64];
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) M[r][c] = ((int64_t)a[r * cols + c] % P + P) % P;
    auto inv = [&](int64_t x) {           // Fermat inverse
        int64_t res = 1, b = x, e = P - 2;
        while (e) { if (e & 1) res = res * b % P; b = b * b % P; e >>= 1; }
        return res;
    };
    int rank = 0;
    for (int c = 0; c < cols && rank < rows; ++c) {
        int piv = -1;
        for (int r = rank; r < rows; ++r) if (M[r][c]) { piv = r; break; }
        if (piv < 0) continue;
        for (int k = 0; k < cols; ++k) std::swap(M[piv][k], M[rank][k]);
        const int64_t iv = inv(M[rank][c]);
        for (int r = rank + 1; r < rows; ++r) {
            if (!M[r][c]) continue;
            const int64_t f = M[r][c] * iv % P;
            for (int k = c; k < cols; ++k) M[r][k] = ((M[r][k] - f * M[rank][k]) % P + P) % P;
        }
        rank++;
    }
    return rank;
}

int fg_type_invariant(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int32_t *counts,
                      int32_t rank_sums[3])
{
    Sch a;
    int rc = load(m, n, p, ring, coeffs, rank, a);
    if (rc != FG_OK) return rc;
    if (!counts || !rank_sums) return FG_E_ARG;
    memset(counts, 0, sizeof(int32_t) * 65 * 65 * 65);
    rank_sums[0] = rank_sums[1] = rank_sums[2] = 0;
    const int dims[3][2] = {{m, n}, {n, p}, {p, m}};    // U: m x n, V: n x p, W: p x m (C^T)
    int8_t buf[64];
    for (int l = 0; l < rank; ++l) {
        int rk[3];
        for (int X = 0; X < 3; ++X) {
            const int len = dims[X][0] * dims[X][1];
            for (int e = 0; e < len; ++e)
                buf[e] = ((a.d[X][l] >> e) & 1) ? (((a.s[X][l] >> e) & 1) ? -1 : 1) : 0;
            rk[X] = rank_mod_p(buf, dims[X][0], dims[X][1]);
            rank_sums[X] += rk[X];
        }
        counts[(rk[0] * 65 + rk[1]) * 65 + rk[2]] += 1;
    }
    return FG_OK;
}

// symmetrised polynomial: f = sum over pi in S_3 of pi applied to the
// type polynomial, i.e. every term (ru, rv, rw) contributes one monomial per permutation
int fg_sym_invariant(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int32_t *sym)
{
    if (!sym) return FG_E_ARG;
    std::vector<int32_t> counts((size_t)65 * 65 * 65);
    int32_t sums[3];
    int rc = fg_type_invariant(m, n, p, ring, coeffs, rank, counts.data(), sums);
    if (rc != FG_OK) return rc;
    memset(sym, 0, sizeof(int32_t) * 65 * 65 * 65);
    static const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int a = 0; a <= 8; ++a)            // factor ranks are <= min(dims) <= 8 (R1: mn <= 64)
        for (int b = 0; b <= 8; ++b)
            for (int c = 0; c <= 8; ++c) {
                const int32_t k = counts[(a * 65 + b) * 65 + c];
                if (!k) continue;
                const int e[3] = {a, b, c};
                for (const auto &q : perm) sym[(e[q[0]] * 65 + e[q[1]]) * 65 + e[q[2]]] += k;
            }
    return FG_OK;
}

// canonical key: rows sign-normalised (Z_T), sorted, hashed (FNV-1a over the words);
// equal schemes up to row order and the sign rescaling of PAPER:429 share a key
int fg_scheme_key(int m, int n, int p, int ring, const int8_t *coeffs, int rank, uint64_t *key)
{
    Sch a;
    int rc = load(m, n, p, ring, coeffs, rank, a);
    if (rc != FG_OK) return rc;
    if (!key) return FG_E_ARG;
    std::vector<std::array<uint64_t, 6>> rows(rank);
    for (int l = 0; l < rank; ++l) {
        uint64_t ud = a.d[0][l], us = a.s[0][l], vd = a.d[1][l], vs = a.s[1][l], wd = a.d[2][l], ws = a.s[2][l];
        if (ring == FG_ZT) {
            if (us & (ud & (0 - ud))) { us ^= ud; ws ^= wd; }
            if (vs & (vd & (0 - vd))) { vs ^= vd; ws ^= wd; }
        }
        rows[l] = {ud, us, vd, vs, wd, ws};
    }
    std::sort(rows.begin(), rows.end());
    uint64_t h = 0xcbf29ce484222325ULL ^ ((uint64_t)m << 48 | (uint64_t)n << 32 | (uint64_t)p << 16 | (uint64_t)ring);
    for (const auto &r : rows)
        for (uint64_t x : r) { h ^= x; h *= 0x100000001b3ULL; }
    *key = h;
    return FG_OK;
}

}  // extern "C"
