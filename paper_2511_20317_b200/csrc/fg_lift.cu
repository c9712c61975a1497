// fg_lift.cu -- Z_2 -> Z_T lifting (section 3.10.1; SPEC:578-630 for
// the search shape), host only.  The paper assigns +-1 signs to the nonzero
// coefficients of a Z_2 scheme with a CP solver (OR-Tools) so that the Brent
// equations hold over the integers; here a native exhaustive search does it
// (reading R32 in DESIGN.md):
//   - unknowns: the sign of every nonzero coefficient, except the first nonzero of
//     each row's u and v, pinned to +1 (the alpha*beta*gamma = 1 rescaling of
//     no solution is lost up to that equivalence);
//   - with sign = (-1)^x, a term's sign is the XOR of its (up to three) bits, and an
//     equation sum_l(term) = T with k terms needs exactly (k - T) / 2 negative terms:
//     the XOR of its term bits is fixed, a LINEAR constraint over GF(2) (it is the whole
//     constraint when k <= 2).  Gaussian elimination of all of them leaves the free
//     variables; every other variable is an affine function of them;
//   - a depth-first search over the free variables evaluates each term as soon as its
//     bits are determined and prunes an equation as soon as |T - known sum| exceeds its
//     number of unknown terms;
//   - the search is exhaustive (FG_E_INVALID_SCHEME = no lift exists) within a node
//     budget (FG_E_STATE = budget exhausted, not a proof).
#include <algorithm>
#include <cstring>
#include <vector>
#include "fg_internal.h"

namespace {

struct Lift {
    int m, n, p, rank, mn, np, pm;
    std::vector<uint64_t> u, v, w;          // Z_2 digits per row
    // variables
    struct Var { int row, role, elem; };
    std::vector<Var> vars;
    std::vector<int> sign_u, sign_v, sign_w;   // per row x element: -1/+1, 0 unknown (flattened)
    // terms: (row, a, b, c) with the equation id and the index of the variable completing it
    struct Term { int row, a, b, c, eq; };
    std::vector<Term> terms;
    std::vector<std::vector<int>> completes;   // variable -> terms it completes
    std::vector<int> eq_target, eq_sum, eq_unknown;
    int64_t nodes = 0, budget = 0;

    int &su(int l, int a) { return sign_u[l * 64 + a]; }
    int &sv(int l, int b) { return sign_v[l * 64 + b]; }
    int &sw(int l, int c) { return sign_w[l * 64 + c]; }

    bool assign(size_t k, int val, std::vector<int> &touched)
    {
        const Var &x = vars[k];
        (x.role == 0 ? su(x.row, x.elem) : x.role == 1 ? sv(x.row, x.elem) : sw(x.row, x.elem)) = val;
        bool ok = true;
        for (int t : completes[k]) {
            const Term &tm = terms[t];
            const int val_t = su(tm.row, tm.a) * sv(tm.row, tm.b) * sw(tm.row, tm.c);
            eq_sum[tm.eq] += val_t;
            eq_unknown[tm.eq] -= 1;
            touched.push_back(t);
            const int gap = eq_target[tm.eq] - eq_sum[tm.eq];
            if (gap > eq_unknown[tm.eq] || -gap > eq_unknown[tm.eq]) ok = false;
        }
        return ok;
    }
    void undo(size_t k, const std::vector<int> &touched)
    {
        for (int t : touched) {
            const Term &tm = terms[t];
            eq_sum[tm.eq] -= su(tm.row, tm.a) * sv(tm.row, tm.b) * sw(tm.row, tm.c);
            eq_unknown[tm.eq] += 1;
        }
        const Var &x = vars[k];
        (x.role == 0 ? su(x.row, x.elem) : x.role == 1 ? sv(x.row, x.elem) : sw(x.row, x.elem)) = 0;
    }
    // 1 solved, 0 exhausted, -1 budget (plain search in variable order)
    int dfs(size_t k)
    {
        if (k == vars.size()) return 1;
        if (++nodes > budget) return -1;
        for (int val : {+1, -1}) {
            std::vector<int> touched;
            if (assign(k, val, touched)) {
                const int r = dfs(k + 1);
                if (r != 0) return r;
            }
            undo(k, touched);
        }
        return 0;
    }
    // ---- GF(2)-reduced search (used when the system is small enough to eliminate densely) ----
    int nw = 0;                                   // 64-bit words per row of the linear system
    std::vector<std::vector<uint64_t>> rows_;     // reduced rows: bits 0..V-1 coefficients, bit V constant
    std::vector<int> piv_row;                     // variable -> reduced row it pivots, -1 free
    std::vector<int> free_vars;                   // free variables in search order
    std::vector<int> det_time;                    // variable -> free-order position it is known at (-1: start)
    std::vector<std::vector<int>> det_at;         // position -> variables determined there (-1 stored at slot 0 of +1)
    std::vector<std::vector<int>> term_at;        // position -> terms completed there
    std::vector<uint64_t> xbits;                  // current assignment (one bit per variable)
    std::vector<int> term_vars;                   // term -> up to 3 variable ids (-1 pinned), flattened x3

    int var_bit(int v) const { return (int)((xbits[v >> 6] >> (v & 63)) & 1u); }
    void set_bit(int v, int b) { xbits[v >> 6] = (xbits[v >> 6] & ~(1ull << (v & 63))) | ((uint64_t)(b & 1) << (v & 63)); }
    int eval_pivot(int v) const
    {
        const std::vector<uint64_t> &rw = rows_[piv_row[v]];
        const int V = (int)vars.size();
        int acc = (int)((rw[V >> 6] >> (V & 63)) & 1u);
        for (int i = 0; i < nw; ++i) {
            uint64_t m = rw[i];
            if (i == (v >> 6)) m &= ~(1ull << (v & 63));
            if (i == (V >> 6)) m &= (V & 63) ? ((1ull << (V & 63)) - 1) : 0ull;
            acc ^= __builtin_popcountll(m & xbits[i]) & 1;
        }
        return acc;
    }
    int term_sign(int t) const
    {
        int b = 0;
        for (int q = 0; q < 3; ++q) {
            const int v = term_vars[3 * t + q];
            if (v >= 0) b ^= var_bit(v);
        }
        return b ? -1 : +1;
    }
    // apply the variables and terms of position i; false if an equation became infeasible
    bool apply(int i, std::vector<int> &done_terms)
    {
        for (int v : det_at[i + 1]) set_bit(v, eval_pivot(v));
        bool ok = true;
        for (int t : term_at[i + 1]) {
            const int e = terms[t].eq;
            eq_sum[e] += term_sign(t);
            eq_unknown[e] -= 1;
            done_terms.push_back(t);
            const int gap = eq_target[e] - eq_sum[e];
            if (gap > eq_unknown[e] || -gap > eq_unknown[e]) ok = false;
        }
        return ok;
    }
    void unapply(const std::vector<int> &done_terms)
    {
        for (int t : done_terms) {
            const int e = terms[t].eq;
            eq_sum[e] -= term_sign(t);
            eq_unknown[e] += 1;
        }
    }
    int dfs2(size_t k)
    {
        if (k == free_vars.size()) return 1;
        if (++nodes > budget) return -1;
        for (int b : {0, 1}) {
            set_bit(free_vars[k], b);
            std::vector<int> done;
            if (apply((int)k, done)) {
                const int r = dfs2(k + 1);
                if (r != 0) return r;
            }
            unapply(done);
        }
        return 0;
    }
    // build the reduced system; false if it is inconsistent (no lift)
    bool reduce_gf2(const std::vector<std::vector<int>> &eq_terms)
    {
        const int V = (int)vars.size();
        nw = (V + 1 + 63) / 64;
        std::vector<std::vector<uint64_t>> sys;
        for (size_t e = 0; e < eq_terms.size(); ++e) {
            std::vector<uint64_t> rw(nw, 0);
            const int k = (int)eq_terms[e].size();
            const int neg = (k - eq_target[e]) / 2;
            for (int t : eq_terms[e])
                for (int q = 0; q < 3; ++q) {
                    const int v = term_vars[3 * t + q];
                    if (v >= 0) rw[v >> 6] ^= 1ull << (v & 63);
                }
            if (neg & 1) rw[V >> 6] ^= 1ull << (V & 63);
            sys.push_back(std::move(rw));
        }
        piv_row.assign(V, -1);
        int rank_ = 0;
        for (int v = 0; v < V && rank_ < (int)sys.size(); ++v) {
            int sel = -1;
            for (size_t r = rank_; r < sys.size(); ++r)
                if ((sys[r][v >> 6] >> (v & 63)) & 1u) { sel = (int)r; break; }
            if (sel < 0) continue;
            std::swap(sys[rank_], sys[sel]);
            for (size_t r = 0; r < sys.size(); ++r)
                if ((int)r != rank_ && ((sys[r][v >> 6] >> (v & 63)) & 1u))
                    for (int i = 0; i < nw; ++i) sys[r][i] ^= sys[rank_][i];
            piv_row[v] = rank_;
            rank_++;
        }
        // rows beyond the rank are 0 = constant: inconsistent if the constant is 1
        for (size_t r = rank_; r < sys.size(); ++r)
            if ((sys[r][V >> 6] >> (V & 63)) & 1u) return false;
        sys.resize(rank_);
        rows_.swap(sys);
        free_vars.clear();
        for (int v = 0; v < V; ++v)
            if (piv_row[v] < 0) free_vars.push_back(v);
        std::vector<int> pos(V, -1);
        for (size_t i = 0; i < free_vars.size(); ++i) pos[free_vars[i]] = (int)i;
        det_time.assign(V, -1);
        det_at.assign(free_vars.size() + 1, {});
        for (int v = 0; v < V; ++v) {
            if (piv_row[v] < 0) { det_time[v] = pos[v]; continue; }
            int tmax = -1;
            const std::vector<uint64_t> &rw = rows_[piv_row[v]];
            for (int f : free_vars)
                if ((rw[f >> 6] >> (f & 63)) & 1u) tmax = std::max(tmax, pos[f]);
            det_time[v] = tmax;
            det_at[tmax + 1].push_back(v);
        }
        term_at.assign(free_vars.size() + 1, {});
        for (size_t t = 0; t < terms.size(); ++t) {
            int tmax = -1;
            for (int q = 0; q < 3; ++q) {
                const int v = term_vars[3 * t + q];
                if (v >= 0) tmax = std::max(tmax, det_time[v]);
            }
            term_at[tmax + 1].push_back((int)t);
        }
        xbits.assign(nw, 0);
        return true;
    }
};

}  // namespace

extern "C" int fg_lift(int m, int n, int p, const int8_t *z2, int rank, int64_t node_budget, int8_t *out,
                       int64_t *nodes_used)
{
    if (m < 1 || n < 1 || p < 1 || m * n > 64 || n * p > 64 || p * m > 64) return FG_E_CAPACITY;
    if (!z2 || !out || rank < 1 || node_budget < 1) return FG_E_ARG;
    Lift L;
    L.m = m; L.n = n; L.p = p; L.rank = rank;
    L.mn = m * n; L.np = n * p; L.pm = p * m;
    const int width = L.mn + L.np + L.pm;
    L.u.assign(rank, 0); L.v.assign(rank, 0); L.w.assign(rank, 0);
    for (int l = 0; l < rank; ++l)
        for (int e = 0; e < width; ++e) {
            const int x = z2[(size_t)l * width + e];
            if (x != 0 && x != 1) return FG_E_DOMAIN;
            if (!x) continue;
            if (e < L.mn) L.u[l] |= 1ull << e;
            else if (e < L.mn + L.np) L.v[l] |= 1ull << (e - L.mn);
            else L.w[l] |= 1ull << (e - L.mn - L.np);
        }
    L.sign_u.assign(rank * 64, 0); L.sign_v.assign(rank * 64, 0); L.sign_w.assign(rank * 64, 0);
    for (int l = 0; l < rank; ++l) {
        if (!L.u[l] || !L.v[l] || !L.w[l]) return FG_E_DOMAIN;
        for (uint64_t t = L.u[l]; t; t &= t - 1) {
            const int e = __builtin_ctzll(t);
            if (t == L.u[l]) L.su(l, e) = 1; else L.vars.push_back({l, 0, e});
        }
        for (uint64_t t = L.v[l]; t; t &= t - 1) {
            const int e = __builtin_ctzll(t);
            if (t == L.v[l]) L.sv(l, e) = 1; else L.vars.push_back({l, 1, e});
        }
        for (uint64_t t = L.w[l]; t; t &= t - 1) L.vars.push_back({l, 2, __builtin_ctzll(t)});
    }
    // equations over the (a,b,c) that occur in some term; the others must have T = 0
    std::vector<int> eq_index((size_t)L.mn * L.np * L.pm, -1);
    auto target = [&](int a, int b, int c) {
        const int i = a / n, j = a % n, j2 = b / p, k = b % p, k2 = c / m, i2 = c % m;
        return (j == j2 && k == k2 && i == i2) ? 1 : 0;
    };
    // variable completing a term: the last in variable order among its signs
    std::vector<int> var_of((size_t)rank * 3 * 64, -1);
    for (size_t k = 0; k < L.vars.size(); ++k)
        var_of[((size_t)L.vars[k].row * 3 + L.vars[k].role) * 64 + L.vars[k].elem] = (int)k;
    L.completes.assign(L.vars.size(), {});
    std::vector<int> pinned_terms_eq;   // terms with all signs pinned (no variable)
    for (int l = 0; l < rank; ++l)
        for (uint64_t ta = L.u[l]; ta; ta &= ta - 1)
            for (uint64_t tb = L.v[l]; tb; tb &= tb - 1)
                for (uint64_t tc = L.w[l]; tc; tc &= tc - 1) {
                    const int a = __builtin_ctzll(ta), b = __builtin_ctzll(tb), c = __builtin_ctzll(tc);
                    const size_t key = ((size_t)a * L.np + b) * L.pm + c;
                    if (eq_index[key] < 0) {
                        eq_index[key] = (int)L.eq_target.size();
                        L.eq_target.push_back(target(a, b, c));
                        L.eq_sum.push_back(0);
                        L.eq_unknown.push_back(0);
                    }
                    const int eq = eq_index[key];
                    L.eq_unknown[eq] += 1;
                    int last = std::max(var_of[((size_t)l * 3 + 0) * 64 + a],
                                        std::max(var_of[((size_t)l * 3 + 1) * 64 + b], var_of[((size_t)l * 3 + 2) * 64 + c]));
                    L.terms.push_back({l, a, b, c, eq});
                    L.completes[last].push_back((int)L.terms.size() - 1);   // w is never pinned: last >= 0
                    L.term_vars.push_back(var_of[((size_t)l * 3 + 0) * 64 + a]);
                    L.term_vars.push_back(var_of[((size_t)l * 3 + 1) * 64 + b]);
                    L.term_vars.push_back(var_of[((size_t)l * 3 + 2) * 64 + c]);
                }
    // every equation with T = 1 must have a term (else no lift, and no mod-2 validity)
    for (int a = 0; a < L.mn; ++a)
        for (int b = 0; b < L.np; ++b)
            for (int c = 0; c < L.pm; ++c)
                if (target(a, b, c) && eq_index[((size_t)a * L.np + b) * L.pm + c] < 0) return FG_E_INVALID_SCHEME;
    for (size_t e = 0; e < L.eq_target.size(); ++e)
        if (((L.eq_unknown[e] - L.eq_target[e]) & 1) != 0) return FG_E_INVALID_SCHEME;   // not valid mod 2
    L.budget = node_budget;
    // the GF(2)-reduced search when the dense system fits (about 64 MB), else the plain one
    const size_t V = L.vars.size(), E = L.eq_target.size();
    int res;
    if (V <= 8192 && E * ((V + 64) / 64) <= ((size_t)8 << 20)) {
        std::vector<std::vector<int>> eq_terms(E);
        for (size_t t = 0; t < L.terms.size(); ++t) eq_terms[L.terms[t].eq].push_back((int)t);
        if (!L.reduce_gf2(eq_terms)) {
            res = 0;
        } else {
            std::vector<int> done;
            res = L.apply(-1, done) ? L.dfs2(0) : 0;
        }
        if (res == 1)
            for (size_t k = 0; k < V; ++k) {
                const auto &x = L.vars[k];
                const int sg = L.var_bit((int)k) ? -1 : +1;
                (x.role == 0 ? L.su(x.row, x.elem) : x.role == 1 ? L.sv(x.row, x.elem) : L.sw(x.row, x.elem)) = sg;
            }
    } else {
        res = L.dfs(0);
    }
    if (nodes_used) *nodes_used = L.nodes;
    if (res < 0) return FG_E_STATE;
    if (res == 0) return FG_E_INVALID_SCHEME;
    for (int l = 0; l < rank; ++l)
        for (int e = 0; e < width; ++e) {
            const int x = z2[(size_t)l * width + e];
            int s = 0;
            if (x) s = e < L.mn ? L.su(l, e) : (e < L.mn + L.np ? L.sv(l, e - L.mn) : L.sw(l, e - L.mn - L.np));
            out[(size_t)l * width + e] = (int8_t)s;
        }
    return FG_OK;
}
