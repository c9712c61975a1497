// fg_walk_wl.cuh -- the RandomWalk kernel (Algorithm 1) for walkers
// with 33..512 rows and wide factors (configs C4 and C5: (5,5,5) R = 160 with 25-element
// factors, (4,5,12) / (5,6,10) / (6,7,9) R = 256 / 320 / 416 with up to 63 elements).
// ONE WALKER PER WARP with LINKED CLASSES, rows round-robin over the lanes.
//
// Why: walk_wm (fg_walk_multi.cuh) finds the second row of every draw with a compare
// sweep over all rows and keeps per-row class counts in registers (local memory for
// NS > 8); walk_ql's quad mapping keeps linked class lists but needs 8 walkers' state
// per warp, which does not fit shared memory for R >= 160 two-word factors.  Here one
// walker per warp keeps, per row l (lane l % 32, word l / 32):
//   fac[X][l]  factor X (U and V sign-normalised; W up to sign)
//   nxh[X][l]  the next row of l's class in role X (1023 = none)
//   wsb        the signs of the w factors, one bit per row (the stored W key is the
//              positive form, W classes are "equal up to sign")
//   lc[l]      later counts of the three classes, 10 bits each (R10)
//   tw[w]      per 32-row word the sum of its rows' later counts, 3 x 21-bit fields of a u64
//              (U | V << 21 | W << 42: the draw's prefix scan adds them as they are)
// so a draw (R11) is a lookup in the per-step prefix of the word totals, one warp scan
// of the word's later counts and `hops` next-pointer steps, and a flip commit is ONE
// compare pass over the rows
// for both changed factors (they are in different roles, so the two class updates
// commute) that also gives R12's exact skip test (does a touched row share two
// factors with another row?), as in walk_ql.  The class structure (nx, lc, tw and the
// candidate totals) survives between launches in an HBM image (WalkArgs::wl_img).
//
// Same readings (R8-R23), draw order and digest as the oracle and the other kernels;
// parity: tests/test_gpu_parity.py, tests/test_gpu_fullsize.py, tests/test_gpu_fuzz.py.
#pragma once
#include <cstdlib>
#include <type_traits>
#include "fg_device.cuh"

namespace fgwl {
using namespace fgd;

constexpr int NIL = 1023;
constexpr int PXT = 16, PXS = 6;               // Philox table: 16 steps x 6 words (draw 0, Bernoulli
                                               // flags, block 2 = draws 1-4): 384 B, so (6,7,9) walkers fit
                                               // 9 per SM (8 with a 32-step table)
#ifndef WL_DRAWS
#define WL_DRAWS 4                             // flip draws evaluated at once (lane groups of 32 / WL_DRAWS): 4 measured best (2: -1..-13 %, 8: -3..-13 %)
#endif
constexpr int IMG_SCALARS = 8;                 // nCU, nCV, nCW, dset lo, dset hi, nD, dover, r

// class image per walker (HBM): nxh (3 RM u16), lc (RM), tw (32), wsb (16), scalars
__host__ __device__ constexpr int img_words(int nwd) { return 48 * nwd + 32 * nwd + 32 + 16 + IMG_SCALARS; }

__device__ __forceinline__ uint32_t below_in(int l, int w)      // bits of word w for rows < l
{
    const int b = l - 32 * w;
    return b <= 0 ? 0u : (b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u));
}
__device__ __forceinline__ uint32_t above_in(int l, int w)      // bits of word w for rows > l
{
    const int b = l - 32 * w;
    return b < 0 ? 0xFFFFFFFFu : (b >= 31 ? 0u : ~((2u << b) - 1u));
}
__device__ __forceinline__ uint32_t setf(uint32_t x, int X, int v)
{
    return (x & ~(1023u << (10 * X))) | ((uint32_t)v << (10 * X));
}
__device__ __forceinline__ int getf(uint32_t x, int X) { return (int)((x >> (10 * X)) & 1023u); }

// one walker's shared-memory state
template <class P> struct WS {
    typename P::F *fac;   // [3][RM]
    uint16_t *nxh;        // [3][RM]
    uint32_t *lc;         // [RM]
    uint32_t *wsb;        // [16]
    uint32_t *tw;         // [32] = 16 u64: U | V << 21 | W << 42 per word
    int nwd, RM;
    __device__ __forceinline__ typename P::F key(int X, int l) const { return fac[X * RM + l]; }
    __device__ __forceinline__ int nxt(int X, int l) const { return (int)nxh[X * RM + l]; }
    __device__ __forceinline__ void set_nxt(int X, int l, int v) const { nxh[X * RM + l] = (uint16_t)v; }
    __device__ __forceinline__ uint32_t wsg(int l) const { return (wsb[l >> 5] >> (l & 31)) & 1u; }
    __device__ __forceinline__ void set_wsg(int l, uint32_t v) const      // lane 0
    {
        wsb[l >> 5] = (wsb[l >> 5] & ~(1u << (l & 31))) | ((v & 1u) << (l & 31));
    }
    __device__ __forceinline__ typename P::F full(int X, int l) const
    {
        const typename P::F k = key(X, l);
        return (X == 2 && wsg(l)) ? P::neg(k) : k;
    }
    __device__ __forceinline__ Row<P> row(int l) const
    {
        Row<P> o;
        o.u = key(0, l);
        o.v = key(1, l);
        o.w = full(2, l);
        return o;
    }
    // word total of role X (lane 0 only)
    __device__ __forceinline__ void tw_add(int w, int X, int d) const
    {
        // (a negative d wraps modulo 2^64 and subtracts from its field only: fields stay >= 0)
        reinterpret_cast<unsigned long long *>(tw)[w] += (unsigned long long)(long long)d << (21 * X);
    }
};

// Row t's role-X key goes from o to k (a zero key is in no class, R10: zero factors
// never pair): one compare pass over the live rows (< r), then the class list, the
// later counts and the word totals are relinked.  Returns the change of the role's
// candidate-pair count.  Whole warp; rare paths only (the flip commit has its own
// fused two-change pass in the kernel).
template <class P>
__device__ __noinline__ int key_change(WS<P> s, int r, int t, int X, typename P::F o, typename P::F k)
{
    typedef typename P::F F;
    const int lane = threadIdx.x & 31;
    const bool zo = P::zero(o), zk = P::zero(k);
    int pO = NIL, sO = NIL, pK = NIL, sK = NIL, aK = 0, tO = 0, tK = 0;
    const F *fx = s.fac + X * s.RM;
#pragma unroll 1
    for (int w = 0; w < ((r + 31) >> 5); ++w) {        // live words only
        const int l = 32 * w + lane;
        const F x = fx[l];
        const bool live = l < r && l != t;
        const bool eo = live && !zo && P::eq(x, o);
        const bool ek = live && !zk && P::eq(x, k);
        const uint32_t mO = __ballot_sync(FULL, eo), mK = __ballot_sync(FULL, ek);
        if ((mO | mK) == 0u) continue;
        if (l < t && eo != ek) s.lc[l] += ek ? (1u << (10 * X)) : (0u - (1u << (10 * X)));
        const uint32_t bl = below_in(t, w), ab = above_in(t, w);
        if (mO & bl) pO = 32 * w + 31 - __clz(mO & bl);
        if ((mO & ab) && sO == NIL) sO = 32 * w + __ffs(mO & ab) - 1;
        if (mK & bl) pK = 32 * w + 31 - __clz(mK & bl);
        if ((mK & ab) && sK == NIL) sK = 32 * w + __ffs(mK & ab) - 1;
        aK += __popc(mK & ab);
        tO += __popc(mO);
        tK += __popc(mK);
        const int d = __popc(mK & bl) - __popc(mO & bl);
        if (lane == 0 && d) s.tw_add(w, X, d);
    }
    __syncwarp();
    if (lane == 0) {
        if (pO != NIL) s.set_nxt(X, pO, sO);
        if (pK != NIL) s.set_nxt(X, pK, t);
        s.set_nxt(X, t, sK);
        const int old = getf(s.lc[t], X);
        s.lc[t] = setf(s.lc[t], X, aK);
        s.tw_add(t >> 5, X, aK - old);
        s.fac[X * s.RM + t] = k;
    }
    __syncwarp();
    return tK - tO;
}

struct D3 { int d0, d1, d2; };

// Row l becomes nr (a normalised row): a class update for every role whose key changes
// (all three if `fresh`: l is a new row, in no class yet), and the W sign bit.
template <class P>
__device__ __noinline__ D3 set_row(WS<P> s, int r, int l, Row<P> nr, bool fresh)
{
    const int lane = threadIdx.x & 31;
    D3 d = {0, 0, 0};
    if (fresh) {
        if (lane == 0) { s.set_nxt(0, l, NIL); s.set_nxt(1, l, NIL); s.set_nxt(2, l, NIL); s.lc[l] = 0u; }
        __syncwarp();
    }
#pragma unroll 1
    for (int X = 0; X < 3; ++X) {
        const typename P::F k = X == 0 ? nr.u : (X == 1 ? nr.v : P::abs(nr.w));
        typename P::F o = s.key(X, l);
        if (fresh) o = P::make(0, 0);
        if (!fresh && P::eq(o, k)) continue;
        const int v = key_change<P>(s, r, l, X, o, k);
        d.d0 += X == 0 ? v : 0;
        d.d1 += X == 1 ? v : 0;
        d.d2 += X == 2 ? v : 0;
    }
    if (lane == 0) s.set_wsg(l, P::first_neg(nr.w) ? 1u : 0u);
    __syncwarp();
    return d;
}

template <class P> struct Found { int j; Row<P> mg; };

// The first row l >= lmin, l != t (ascending) with reducible(row t, row l) (R13), and
// the merged row (row t as base); j = -1 if none.  Candidates share two factor keys
// with row t (W up to sign, zero keys included: the oracle compares zero factors as
// equal); each is checked exactly.  Whole warp.
template <class P>
__device__ __noinline__ Found<P> first_reducible(WS<P> s, int r, int t, int lmin)
{
    typedef typename P::F F;
    const int lane = threadIdx.x & 31;
    const Row<P> rt = s.row(t);
    const F k0 = s.key(0, t), k1 = s.key(1, t), k2 = s.key(2, t);
    Found<P> out;
    out.j = -1;
    out.mg = rt;
#pragma unroll 1
    for (int w = 0; w < ((r + 31) >> 5); ++w) {
        const int l = 32 * w + lane;
        const int c = (int)P::eq(s.key(0, l), k0) + (int)P::eq(s.key(1, l), k1) + (int)P::eq(s.key(2, l), k2);
        uint32_t m = __ballot_sync(FULL, l < r && l != t && l >= lmin && c >= 2);
        while (m) {
            const int j = 32 * w + __ffs(m) - 1;
            m &= m - 1u;
            Row<P> mg;
            if (reducible<P>(rt, s.row(j), mg)) {
                out.j = j;
                out.mg = mg;
                return out;
            }
        }
    }
    return out;
}

// Debug only (FG_DBG bit 0): rebuild the class structure from the rows and compare.
// Returns 0 if consistent, else a code.
template <class P>
__device__ __noinline__ uint32_t check_structure(WS<P> s, int r, uint32_t nCU, uint32_t nCV, uint32_t nCW)
{
    const int lane = threadIdx.x & 31;
    uint32_t bad = 0;
    uint32_t tot[3] = {0, 0, 0};
    for (int X = 0; X < 3; ++X) {
        for (int w = 0; w < s.nwd; ++w) {
            const int l = 32 * w + lane;
            int cnt = 0, first = NIL;
            if (l < r) {
                const typename P::F k = s.key(X, l);
                if (!P::zero(k))
                    for (int j = l + 1; j < r; ++j)
                        if (P::eq(s.key(X, j), k)) { if (first == NIL) first = j; cnt++; }
                if (getf(s.lc[l], X) != cnt) bad |= 1u;
                if (s.nxt(X, l) != first) bad |= 2u;
            }
            const int sum = __reduce_add_sync(FULL, (uint32_t)cnt);
            const uint32_t t = (uint32_t)(reinterpret_cast<const unsigned long long *>(s.tw)[w] >> (21 * X)) & 0x1FFFFFu;
            if ((uint32_t)sum != t) bad |= 4u;
            tot[X] += (uint32_t)sum;
        }
    }
    if (tot[0] != nCU || tot[1] != nCV || tot[2] != nCW) bad |= 8u;
    return __reduce_or_sync(FULL, bad);
}

template <class P, int MINB, bool CM>
__global__ void __launch_bounds__(32, MINB) walk_wl(WalkArgs a, int nwd)
{
    typedef typename P::F F;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int RM = 32 * nwd;
    WS<P> s;
    s.fac = reinterpret_cast<F *>(smraw);
    s.lc = reinterpret_cast<uint32_t *>(s.fac + 3 * RM);
    s.tw = s.lc + RM;
    s.wsb = s.tw + 32;
    uint32_t *px = s.wsb + 16;                                 // Philox table [PXT][PXS]
    uint32_t *rc = px + PXT * PXS;                             // 8 rare counters
    s.nxh = reinterpret_cast<uint16_t *>(rc + 8);
    s.nwd = nwd;
    s.RM = RM;
    const int lane = threadIdx.x;
    const int R = a.R;
    const uint64_t seed = a.seed;
    const uint32_t kf = a.k_flip;
    const int IMGW = img_words(nwd);

    auto grab = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.work_counter, 1ull);
        return (int64_t)__shfl_sync(FULL, v, 0);
    };

#pragma unroll 1
    for (int64_t wk = grab(); wk < a.num_walkers; wk = grab()) {
        // ---------------- load the walker ----------------
        const uint64_t *cp = a.cur + (size_t)wk * FG_PLANES * R;
        uint64_t *bw = a.best + (size_t)wk * FG_PLANES * R;
        fg_whdr *hp = a.hdr + wk;
        int r = hp->r;
        int best = hp->best_r;
        uint64_t step = hp->step;
        uint64_t digest = hp->digest;
        int best_adds = hp->best_adds;
        const uint32_t wid = (uint32_t)(a.id_base + wk);
#pragma unroll 1
        for (int l = lane; l < RM; l += 32) {
            F u = P::make(0, 0), v = u, w = u;
            if (l < r) {
                u = P::make(cp[0 * R + l], cp[1 * R + l]);
                v = P::make(cp[2 * R + l], cp[3 * R + l]);
                w = P::make(cp[4 * R + l], cp[5 * R + l]);
            }
            s.fac[l] = u;
            s.fac[RM + l] = v;
            s.fac[2 * RM + l] = P::abs(w);
            s.set_nxt(0, l, NIL); s.set_nxt(1, l, NIL); s.set_nxt(2, l, NIL);
            s.lc[l] = 0u;
            const uint32_t sg = __ballot_sync(FULL, P::first_neg(w));
            if (lane == 0) s.wsb[l >> 5] = sg;
        }
        if (lane < 8) rc[lane] = 0;
        s.tw[lane] = 0;
        __syncwarp();
        uint32_t nCU = 0, nCV = 0, nCW = 0;
        // R15 dirty set D (<= 6 rows, 10 bits each): only rows changed by expands since
        // the last clean scan can be in a reducible pair (flips are cleaned by R12)
        uint64_t dset = 0;
        int nD = 0;
        bool dover = true;
        uint32_t *img = a.wl_img ? a.wl_img + (size_t)wk * IMGW : nullptr;
        const bool resume = img != nullptr && a.img_valid && (int)img[IMGW - 1] == r;
        if (resume) {
            const uint32_t *nxi = img, *lci = img + 3 * RM / 2, *twi = lci + RM;
#pragma unroll 1
            for (int k = lane; k < 3 * RM / 2; k += 32) reinterpret_cast<uint32_t *>(s.nxh)[k] = nxi[k];
#pragma unroll 1
            for (int l = lane; l < RM; l += 32) s.lc[l] = lci[l];
            s.tw[lane] = twi[lane];
            if (lane < 16) s.wsb[lane] = twi[32 + lane];
            const uint32_t *sc = twi + 48;
            nCU = sc[0]; nCV = sc[1]; nCW = sc[2];
            dset = (uint64_t)sc[3] | ((uint64_t)sc[4] << 32);
            nD = (int)sc[5];
            dover = sc[6] != 0u;
        } else {
            // class links and later counts from the rows: O(r^2 / 32) per lane
#pragma unroll 1
            for (int X = 0; X < 3; ++X) {
#pragma unroll 1
                for (int w = 0; w < nwd; ++w) {
                    const int l = 32 * w + lane;
                    int cnt = 0, first = NIL;
                    if (l < r) {
                        const F k = s.key(X, l);
                        if (!P::zero(k)) {
#pragma unroll 1
                            for (int j = l + 1; j < r; ++j)
                                if (P::eq(s.key(X, j), k)) { if (first == NIL) first = j; cnt++; }
                        }
                    }
                    s.set_nxt(X, l, first);
                    s.lc[l] = setf(s.lc[l], X, cnt);
                    const uint32_t sum = __reduce_add_sync(FULL, (uint32_t)cnt);
                    if (lane == 0) s.tw_add(w, X, (int)sum);
                    nCU += X == 0 ? sum : 0u;
                    nCV += X == 1 ? sum : 0u;
                    nCW += X == 2 ? sum : 0u;
                }
            }
        }
        __syncwarp();

        uint32_t c_draws = 0, c_flips = 0, c_red = 0;
        enum { RC_EOK = 0, RC_EREJ, RC_MERGE, RC_ZERO, RC_COPY, RC_IMPR };
        auto bump = [&](int k, uint32_t v) { if (lane == 0) rc[k] += v; };
        auto addC = [&](D3 d) {
            nCU += (uint32_t)d.d0;
            nCV += (uint32_t)d.d1;
            nCW += (uint32_t)d.d2;
        };
        auto d_add = [&](int x) {
            if (dover) return;
            for (int k = 0; k < nD; ++k)
                if ((int)((dset >> (10 * k)) & 1023u) == x) return;
            if (nD == 6) { dover = true; return; }
            dset |= (uint64_t)x << (10 * nD);
            nD++;
        };
        // R14 remove(h) with the 2-entry worklist (entries == h dropped, r-1 -> h): h
        // leaves its classes; row r-1 leaves its classes and re-enters them as row h
        auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) {
            const int last = r - 1;
            const Row<P> lastrow = s.row(last);
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                const int t = k == 0 ? h : last;
                if (k == 1 && h == last) break;
#pragma unroll 1
                for (int X = 0; X < 3; ++X) {
                    const int v = key_change<P>(s, r, t, X, s.key(X, t), P::make(0, 0));
                    nCU += X == 0 ? (uint32_t)v : 0u;
                    nCV += X == 1 ? (uint32_t)v : 0u;
                    nCW += X == 2 ? (uint32_t)v : 0u;
                }
            }
            r--;
            if (h != last) addC(set_row<P>(s, r, h, lastrow, true));
            int n2 = 0, x0 = 0, x1 = 0;
            if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
            if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
            wl0 = x0; wl1 = x1; nwl = n2;
            if (h != last) {
                if (nwl >= 1 && wl0 == last) wl0 = h;
                if (nwl >= 2 && wl1 == last) wl1 = h;
            }
            uint64_t nd = 0;
            int n = 0;
            for (int k = 0; k < nD; ++k) {
                int x = (int)((dset >> (10 * k)) & 1023u);
                if (x == h) continue;
                if (x == last) x = h;
                nd |= (uint64_t)x << (10 * n);
                n++;
            }
            dset = nd;
            nD = n;
        };
        auto row_zero = [&](int l) {
            return P::zero(s.key(0, l)) || P::zero(s.key(1, l)) || P::zero(s.key(2, l));
        };

        // R12: exact worklist reduction after a flip touching rows a0, b0
        auto local_reduce = [&](int a0, int b0) {
            int wl0 = a0, wl1 = b0, nwl = 2;
            while (nwl > 0) {
                const int t = wl0;
                wl0 = wl1;
                nwl--;
                if (t >= r) continue;
                if (row_zero(t)) {
                    remove_row(t, wl0, wl1, nwl);
                    bump(RC_ZERO, 1);
                    continue;
                }
                const Found<P> f = first_reducible<P>(s, r, t, 0);
                if (f.j < 0) continue;
                const int lo = t < f.j ? t : f.j, hi = t < f.j ? f.j : t;
                addC(set_row<P>(s, r, lo, f.mg, false));
                bump(RC_MERGE, 1);
                remove_row(hi, wl0, wl1, nwl);
                if (has_zero(f.mg)) {
                    remove_row(lo, wl0, wl1, nwl);
                    bump(RC_ZERO, 1);
                } else {
                    wl1 = wl0;
                    wl0 = lo;
                    nwl++;
                }
            }
        };

        // R15: reduce_all, exact (lexicographic first reducible pair)
        auto reduce_all = [&]() {
#pragma unroll 1
            for (;;) {
                int zfirst = -1;
#pragma unroll 1
                for (int w = 0; w < ((r + 31) >> 5) && zfirst < 0; ++w) {
                    const int l = 32 * w + lane;
                    const uint32_t m = __ballot_sync(FULL, l < r && row_zero(l));
                    if (m) zfirst = 32 * w + __ffs(m) - 1;
                }
                if (zfirst >= 0) {
                    int n0 = 0, x0 = 0, x1 = 0;
                    remove_row(zfirst, x0, x1, n0);
                    bump(RC_ZERO, 1);
                    continue;
                }
                int bi = -1, bj = -1;
                if (dover) {
#pragma unroll 1
                    for (int i = 0; i + 1 < r && bi < 0; ++i) {
                        const Found<P> f = first_reducible<P>(s, r, i, i + 1);
                        if (f.j >= 0) { bi = i; bj = f.j; }
                    }
                } else {
                    int bestkey = 0x7fffffff;
#pragma unroll 1
                    for (int k = 0; k < nD; ++k) {
                        const int d = (int)((dset >> (10 * k)) & 1023u);
                        const Found<P> f = first_reducible<P>(s, r, d, 0);
                        if (f.j >= 0) {
                            const int kk = (f.j < d ? f.j : d) * 1024 + (f.j < d ? d : f.j);
                            bestkey = kk < bestkey ? kk : bestkey;
                        }
                    }
                    if (bestkey != 0x7fffffff) { bi = bestkey >> 10; bj = bestkey & 1023; }
                }
                if (bi < 0) {
                    dset = 0;
                    nD = 0;
                    dover = false;
                    break;
                }
                // merged = reducible(row i, row j) with row i as base (R15)
                Row<P> mg = s.row(bi);
                reducible<P>(s.row(bi), s.row(bj), mg);
                addC(set_row<P>(s, r, bi, mg, false));
                bump(RC_MERGE, 1);
                int n0 = 0, x0 = 0, x1 = 0;
                remove_row(bj, x0, x1, n0);
                if (has_zero(mg)) {
                    remove_row(bi, x0, x1, n0);
                    bump(RC_ZERO, 1);
                } else {
                    d_add(bi);
                }
            }
        };

        // R16 expand (plus / split), words from Philox block 1 of this step
        auto expand = [&]() -> bool {
            if (r < 2 || r + 1 > R) return false;
            uint32_t b0, b1, b2, b3;
            philox_block(seed, step, wid, 1u, b0, b1, b2, b3);
            const bool plus = b0 < 0x80000000u;
            const int i = (int)__umulhi(b1, (uint32_t)r);
            int j = (int)__umulhi(b2, (uint32_t)(r - 1));
            j += (j >= i);
            const int perm = (int)__umulhi(b3, 6u);
            // PERM = (U,V,W),(U,W,V),(V,U,W),(V,W,U),(W,U,V),(W,V,U)
            const int A = perm >> 1;
            const int B = (1161 >> (2 * perm)) & 3;
            const int Cr = 3 - A - B;
            const Row<P> ri = s.row(i), rj = s.row(j);
            const F ai = get(ri, A), aj = get(rj, A), bi_ = get(ri, B), bj_ = get(rj, B);
            const F ci = get(ri, Cr), cj = get(rj, Cr);
            bool ok = true;
            Row<P> ni = ri, nj = rj, nr = ri;
            if (plus) {
                if (!distinct<P>(ai, aj) || !distinct<P>(bi_, bj_) || !distinct<P>(ci, cj)) return false;
                const F t1 = P::add(bi_, bj_, ok);      // v_i + v_j
                const F t2 = P::sub(cj, ci, ok);        // w_j - w_i
                const F t3 = P::sub(aj, ai, ok);        // u_j - u_i
                if (!ok) return false;
                set(ni, B, t1, true);
                set(nj, A, ai, true);
                set(nj, Cr, t2, true);
                set(nr, A, t3, true);
                set(nr, B, bj_, true);
                set(nr, Cr, cj, true);
            } else {
                if (!distinct<P>(ai, aj)) return false;
                const F t3 = P::sub(ai, aj, ok);        // u_i - u_j
                if (!ok) return false;
                set(ni, A, aj, true);
                set(nr, A, t3, true);
                set(nr, B, bi_, true);
                set(nr, Cr, ci, true);
            }
            normalize<P>(ni);
            normalize<P>(nj);
            normalize<P>(nr);
            const int rold = r;
            addC(set_row<P>(s, r, i, ni, false));
            addC(set_row<P>(s, r, j, nj, false));
            addC(set_row<P>(s, r, rold, nr, true));
            r++;
            d_add(i);
            d_add(j);
            d_add(rold);
            return true;
        };

        // copy of the current rows to an HBM scheme image (best / verify queue): rows < n
        // (n >= r; zeros for r <= t < n)
        auto store_rows = [&](uint64_t *dst, int n) {
#pragma unroll 1
            for (int t = lane; t < n; t += 32) {
                const bool lv = t < r;
                const F u = s.key(0, t), v = s.key(1, t), w = s.full(2, t);
                dst[0 * R + t] = lv ? P::dig(u) : 0;
                dst[1 * R + t] = lv ? P::sgn(u) : 0;
                dst[2 * R + t] = lv ? P::dig(v) : 0;
                dst[3 * R + t] = lv ? P::sgn(v) : 0;
                dst[4 * R + t] = lv ? P::dig(w) : 0;
                dst[5 * R + t] = lv ? P::sgn(w) : 0;
            }
        };
        // a strict improvement goes to the verify queue (rank rows only)
        auto enqueue = [&](uint32_t &flags) {
            flags |= 8u;
            bump(RC_IMPR, 1);
            unsigned slot = 0;
            if (lane == 0) slot = atomicAdd(a.q_count, 1u);
            slot = __shfl_sync(FULL, slot, 0);
            if (slot < a.q_cap) {
                store_rows(a.q_planes + (size_t)slot * FG_PLANES * R, r);
                if (lane == 0) {
                    fg_qmeta qm;
                    qm.walker = wk; qm.step = step; qm.rank = r; qm.ok = -1;
                    qm.ff[0] = qm.ff[1] = qm.ff[2] = -1; qm.pad = 0;
                    a.q_meta[slot] = qm;
                }
            } else if (lane == 0) {
                atomicAdd(a.q_overflow, 1u);
                hp->pad |= 1;
            }
        };
        auto nnz_all = [&]() -> int {
            int v = 0;
#pragma unroll 1
            for (int l = lane; l < r; l += 32) v += P::popd(s.key(0, l)) + P::popd(s.key(1, l)) + P::popd(s.key(2, l));
            return (int)__reduce_add_sync(FULL, (uint32_t)v);
        };

        // R24 (complexity mode, CM: WalkArgs::mode == 1): flips only, best by (rank, naive additions);
        // flips skip R12 there, so the dirty set no longer covers every reducible pair
        int nnz_cur = 0;
        if (CM) {
            nnz_cur = nnz_all();
            dover = true;
        }

        int boff = PXT;
        const uint32_t nsteps = (uint32_t)a.steps;
#pragma unroll 1
        for (uint32_t it = 0; it < nsteps; ++it, ++step, ++boff) {
            if (boff == PXT) {
                // Philox (R8) of the next 16 steps, one block per lane: lane L < 16 block 0 of
                // step + L (draw 0 + the Bernoulli words), lane 16 + L block 2 (draws 1-4)
                uint32_t o0, o1, o2, o3;
                const int L = lane & 15;
                philox_block(seed, step + L, wid, lane < 16 ? 0u : 2u, o0, o1, o2, o3);
                if (lane < 16) {
                    px[L * PXS + 0] = o0;
                    px[L * PXS + 1] = (o1 < a.thr_eq ? 1u : 0u) | (o2 < a.thr_reduce ? 2u : 0u) |
                                      (o3 < a.thr_expand ? 4u : 0u);
                } else {
                    px[L * PXS + 2] = o0; px[L * PXS + 3] = o1;
                    px[L * PXS + 4] = o2; px[L * PXS + 5] = o3;
                }
                __syncwarp();
                boff = 0;
            }
            const uint32_t *pw = px + boff * PXS;
            const uint32_t bern = pw[1];
            uint32_t flags = 0;
            int alpha = 0, beta = 0, draws = 0;
            bool ok = false;
            const uint32_t nU = nCU, nV = nCV, nW = nCW;
            const uint32_t nC = nU + nV + nW;
            int fY = 0, fZ = 0;
            F fny = P::make(0, 0), fnz = fny;

            // ---- R11 try_flip: draws over 4|C| (R9), ND at a time: lane group g (GL lanes)
            // evaluates draw ND*t + g; the first valid one in draw order is the one the
            // sequential loop commits (draws are addressed, not consumed) ----
            if (nC) {
                constexpr int ND = WL_DRAWS, GL = 32 / ND;
                constexpr int WPL = (16 + GL - 1) / GL;           // prefix words per lane (nwd <= 16)
                constexpr int RPL = 32 / GL;                       // rows of the word per lane
                const unsigned gmask = GL == 32 ? FULL : ((1u << GL) - 1u);
                const int grp = lane / GL, gl = lane % GL, gb = grp * GL;
                // prefix of the word totals, once per step (the list is not rebuilt between
                // draws), 3 x 21-bit fields: lane gl of each group holds words WPL*gl ...
                uint64_t winc[WPL];
                uint64_t lsum = 0;
#pragma unroll
                for (int q = 0; q < WPL; ++q) {
                    const int w = WPL * gl + q;
                    uint64_t tv = 0;
                    if (w < nwd) {
                        tv = reinterpret_cast<const unsigned long long *>(s.tw)[w];
                    }
                    lsum += tv;
                    winc[q] = lsum;                                // within-lane inclusive
                }
                uint64_t linc = lsum;
#pragma unroll
                for (int o = 1; o < GL; o <<= 1) {
                    const uint64_t t = __shfl_up_sync(FULL, linc, o, GL);
                    if (gl >= o) linc += t;
                }
                const uint64_t lexc = linc - lsum;                  // words before WPL*gl
#pragma unroll
                for (int q = 0; q < WPL; ++q) winc[q] += lexc;
                uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, cb = 0xFFFFFFFFu;
#pragma unroll 1
                for (uint32_t at = 0; at < kf; at += ND) {
                    const uint32_t a2 = at + (uint32_t)grp;             // this group's draw
                    uint32_t x;
                    if (a2 == 0) x = pw[0];
                    else if (a2 <= 4) x = pw[1 + a2];
                    else {
                        const uint32_t slot = 7 + a2, blk = slot >> 2;
                        if (blk != cb) {
                            philox_block(seed, step, wid, blk, e0, e1, e2, e3);
                            cb = blk;
                        }
                        const uint32_t ws = slot & 3;
                        x = ws == 0 ? e0 : (ws == 1 ? e1 : (ws == 2 ? e2 : e3));
                    }
                    const uint32_t k = __umulhi(x, 4u * nC);
                    const uint32_t idx = k >> 2;
                    const int d = k & 1, e = (k >> 1) & 1;
                    const uint32_t g1 = idx >= nU, g2 = idx >= nU + nV;
                    const int X = (int)(g1 + g2);
                    const uint32_t qq = idx - (g1 ? nU : 0u) - (g2 ? nV : 0u);
                    // the word holding row i: the first word whose inclusive prefix exceeds qq
                    const int sh = 21 * X;
                    int qf = WPL;
#pragma unroll
                    for (int q = WPL - 1; q >= 0; --q)
                        if (WPL * gl + q < nwd && ((uint32_t)(winc[q] >> sh) & 0x1FFFFFu) > qq) qf = q;
                    const int Lw = __ffs((__ballot_sync(FULL, qf < WPL) >> gb) & gmask) - 1;
                    const int qsel = __shfl_sync(FULL, qf, gb | Lw);
                    const int wsel = WPL * Lw + qsel;
                    // prefix before word wsel: lane Lw's inclusive sum of its words before qsel
                    uint64_t wexc = lexc;
#pragma unroll
                    for (int q = 0; q < WPL; ++q)
                        if (q < qf && q < WPL) wexc = winc[q];
                    wexc = __shfl_sync(FULL, qsel == 0 ? lexc : wexc, gb | Lw);
                    // (lane Lw: qf == qsel, so wexc is the inclusive sum of word qsel-1)
                    const uint32_t q1 = qq - ((uint32_t)(wexc >> sh) & 0x1FFFFFu);
                    // row i inside the word: lane gl holds rows RPL*gl ... of word wsel
                    uint32_t lv[RPL];
                    uint32_t rsum = 0;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        const int lw = 32 * wsel + RPL * gl + q;
                        lv[q] = lw < r ? (uint32_t)getf(s.lc[lw], X) : 0u;
                        rsum += lv[q];
                    }
                    uint32_t rinc = rsum;
#pragma unroll
                    for (int o = 1; o < GL; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(FULL, rinc, o, GL);
                        if (gl >= o) rinc += t;
                    }
                    const uint32_t rexc = rinc - rsum;                  // later counts before row RPL*gl
                    const int Lr = __ffs((__ballot_sync(FULL, rinc > q1) >> gb) & gmask) - 1;
                    // within lane Lr's rows: the first row whose running sum exceeds q1
                    uint32_t run = rexc;
                    int qr = RPL - 1;
                    uint32_t accr = rexc;
#pragma unroll
                    for (int q = RPL - 1; q >= 0; --q) {
                        uint32_t before = rexc;
#pragma unroll
                        for (int q2 = 0; q2 < q; ++q2) before += lv[q2];
                        if (before + lv[q] > q1) { qr = q; accr = before; }
                    }
                    (void)run;
                    const int rq = __shfl_sync(FULL, qr, gb | Lr);
                    const uint32_t acc = __shfl_sync(FULL, accr, gb | Lr);
                    const int i = 32 * wsel + RPL * Lr + rq;
                    // j: the (q1 - acc)-th later member of row i's X class
                    const uint16_t *nxX = s.nxh + X * RM;
                    int j = i;
#pragma unroll 1
                    for (uint32_t hops = q1 - acc + 1; hops; --hops) j = nxX[j];
                    const int al = d ? j : i, be = d ? i : j;
                    // (Y,Z) = (V,W) / (W,U) / (U,V) for X = U / V / W, swapped if e
                    const unsigned yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
                    const int Y = yz & 3, Z = yz >> 2;
                    const uint32_t sga = s.wsg(al), sgb = s.wsg(be);
                    const bool sneg = P::RING == FG_ZT && X == 2 && sga != sgb;
                    bool v = a2 < kf;
                    const F ya = s.key(Y, al), yb = s.key(Y, be), za = s.key(Z, al), zb = s.key(Z, be);
                    // the actual w carries its sign bit (stored up to sign)
                    const F yaF = P::sel(Y == 2 && sga, P::neg(ya), ya);
                    const F ybF = P::sel(Y == 2 && sgb, P::neg(yb), yb);
                    const F zaF = P::sel(Z == 2 && sga, P::neg(za), za);
                    const F zbF = P::sel(Z == 2 && sgb, P::neg(zb), zb);
                    const F ny = P::add(yaF, P::sel(sneg, P::neg(ybF), ybF), v);   // y_a + s y_b
                    const F nz = P::sub(zbF, zaF, v);                              // z_b - z_a
                    // R24: no reduction edges -> a draw making a factor zero is rejected
                    if (CM) v = v && !P::zero(ny) && !P::zero(nz);
                    const uint32_t vb = __ballot_sync(FULL, v);
                    if (!vb) {
                        draws += (kf - at) < (uint32_t)ND ? (int)(kf - at) : ND;
                        continue;
                    }
                    const int win = (__ffs(vb) - 1) / GL;              // the earliest valid draw
                    const int src = win * GL;
                    draws += win + 1;
                    alpha = __shfl_sync(FULL, al, src);
                    beta = __shfl_sync(FULL, be, src);
                    fY = __shfl_sync(FULL, Y, src);
                    fZ = __shfl_sync(FULL, Z, src);
                    fny = P::shfl(ny, src);
                    fnz = P::shfl(nz, src);
                    ok = true;
                    break;
                }
            }
            c_draws += draws;

            bool need_local = false;
            if (ok) {
                // ---- commit (A4/A5): row alpha's Y := ny, row beta's Z := nz, R6 per row:
                // only the changed factor can be first-negative; w absorbs the sign ----
                const int fX = 3 - fY - fZ;
                const bool fa = P::first_neg(fny), fb = P::first_neg(fnz);
                const F kY = fY == 2 ? P::abs(fny) : P::sel(fa, P::neg(fny), fny);
                const F kZ = fZ == 2 ? P::abs(fnz) : P::sel(fb, P::neg(fnz), fnz);
                const uint32_t sa = fY == 2 ? (uint32_t)fa : (s.wsg(alpha) ^ (uint32_t)fa);
                const uint32_t sb = fZ == 2 ? (uint32_t)fb : (s.wsg(beta) ^ (uint32_t)fb);
                const F oY = s.key(fY, alpha), oZ = s.key(fZ, beta);
                if (CM) nnz_cur += P::popd(kY) + P::popd(kZ) - P::popd(oY) - P::popd(oZ);
                // R12 test keys: alpha after the commit = (AX, kY, AZ), beta = (AX, BY, kZ)
                // (alpha and beta share the X key: they are in one X class)
                const F AX = s.key(fX, alpha), AZ = s.key(fZ, alpha), BY = s.key(fY, beta);
                const bool zY = P::zero(kY), zZ = P::zero(kZ);
                const F *pX = s.fac + fX * RM, *pY = s.fac + fY * RM, *pZ = s.fac + fZ * RM;
                // fused compare pass: class updates of (alpha, Y) and (beta, Z) + R12 test
                int pO0 = NIL, sO0 = NIL, pK0 = NIL, sK0 = NIL, aK0 = 0, tD0 = 0;
                int pO1 = NIL, sO1 = NIL, pK1 = NIL, sK1 = NIL, aK1 = 0, tD1 = 0;
                bool hit = false;
                // two words per iteration for the 16-byte layouts (ILP at ~2 resident warps
                // per scheduler: +2 % on C5); one for P32 (-2 % on C4, scripts/gpu_r02_ab.sh)
                constexpr int PASS_UNROLL = sizeof(F) > 8 ? 2 : 1;
#pragma unroll PASS_UNROLL
                for (int w = 0; w < ((r + 31) >> 5); ++w) {        // live words only
                    const int l = 32 * w + lane;
                    const F xX = pX[l], xY = pY[l], xZ = pZ[l];
                    const bool la = l < r && l != alpha, lb = l < r && l != beta;
                    const bool yO = P::eq(xY, oY), yK = P::eq(xY, kY), yB = P::eq(xY, BY);
                    const bool zO = P::eq(xZ, oZ), zK = P::eq(xZ, kZ), zA = P::eq(xZ, AZ);
                    const bool xA = P::eq(xX, AX);
                    // two shared factors with alpha (yK, zA, xA) or with beta (yB, zK, xA)
                    const bool two = (yK && (zA || xA)) || (zA && xA) || (yB && (zK || xA)) || (zK && xA);
                    hit = hit || (la && lb && two);
                    const uint32_t mO0 = __ballot_sync(FULL, la && yO), mK0 = __ballot_sync(FULL, la && yK);
                    const uint32_t mO1 = __ballot_sync(FULL, lb && zO), mK1 = __ballot_sync(FULL, lb && zK);
                    if ((mO0 | mK0 | mO1 | mK1) == 0u) continue;
                    uint32_t dl = 0;
                    if (l < alpha && la && yO != yK) dl += yK ? (1u << (10 * fY)) : (0u - (1u << (10 * fY)));
                    if (l < beta && lb && zO != zK) dl += zK ? (1u << (10 * fZ)) : (0u - (1u << (10 * fZ)));
                    if (dl) s.lc[l] += dl;
                    {
                        const uint32_t bl = below_in(alpha, w), ab = above_in(alpha, w);
                        if (mO0 & bl) pO0 = 32 * w + 31 - __clz(mO0 & bl);
                        if ((mO0 & ab) && sO0 == NIL) sO0 = 32 * w + __ffs(mO0 & ab) - 1;
                        if (mK0 & bl) pK0 = 32 * w + 31 - __clz(mK0 & bl);
                        if ((mK0 & ab) && sK0 == NIL) sK0 = 32 * w + __ffs(mK0 & ab) - 1;
                        aK0 += __popc(mK0 & ab);
                        tD0 += __popc(mK0) - __popc(mO0);
                        const int dw = __popc(mK0 & bl) - __popc(mO0 & bl);
                        if (lane == 0 && dw) s.tw_add(w, fY, dw);
                    }
                    {
                        const uint32_t bl = below_in(beta, w), ab = above_in(beta, w);
                        if (mO1 & bl) pO1 = 32 * w + 31 - __clz(mO1 & bl);
                        if ((mO1 & ab) && sO1 == NIL) sO1 = 32 * w + __ffs(mO1 & ab) - 1;
                        if (mK1 & bl) pK1 = 32 * w + 31 - __clz(mK1 & bl);
                        if ((mK1 & ab) && sK1 == NIL) sK1 = 32 * w + __ffs(mK1 & ab) - 1;
                        aK1 += __popc(mK1 & ab);
                        tD1 += __popc(mK1) - __popc(mO1);
                        const int dw = __popc(mK1 & bl) - __popc(mO1 & bl);
                        if (lane == 0 && dw) s.tw_add(w, fZ, dw);
                    }
                }
                hit = __any_sync(FULL, hit);
                __syncwarp();
                if (lane == 0) {
                    // (alpha, Y) and (beta, Z): different roles, disjoint fields
                    if (pO0 != NIL) s.set_nxt(fY, pO0, sO0);
                    if (pK0 != NIL) s.set_nxt(fY, pK0, alpha);
                    s.set_nxt(fY, alpha, sK0);
                    const int old0 = getf(s.lc[alpha], fY);
                    s.lc[alpha] = setf(s.lc[alpha], fY, aK0);
                    s.tw_add(alpha >> 5, fY, aK0 - old0);
                    s.fac[fY * RM + alpha] = kY;
                    if (pO1 != NIL) s.set_nxt(fZ, pO1, sO1);
                    if (pK1 != NIL) s.set_nxt(fZ, pK1, beta);
                    s.set_nxt(fZ, beta, sK1);
                    const int old1 = getf(s.lc[beta], fZ);
                    s.lc[beta] = setf(s.lc[beta], fZ, aK1);
                    s.tw_add(beta >> 5, fZ, aK1 - old1);
                    s.fac[fZ * RM + beta] = kZ;
                    s.set_wsg(alpha, sa);
                    s.set_wsg(beta, sb);
                }
                __syncwarp();
                nCU += (fY == 0 ? (uint32_t)tD0 : 0u) + (fZ == 0 ? (uint32_t)tD1 : 0u);
                nCV += (fY == 1 ? (uint32_t)tD0 : 0u) + (fZ == 1 ? (uint32_t)tD1 : 0u);
                nCW += (fY == 2 ? (uint32_t)tD0 : 0u) + (fZ == 2 ? (uint32_t)tD1 : 0u);
                // the pair itself: X shared, plus Y (kY vs BY) or Z (AZ vs kZ)
                need_local = zY || zZ || hit || P::eq(kY, BY) || P::eq(AZ, kZ);
            }

            uint32_t exp_flag = 0;
            if (CM) {
                // ---- R24 step: flips only; best by (rank, naive additions) ----
                if (ok) {
                    c_flips++;
                    flags |= 1u;
                    const int adds = nnz_cur - 2 * r - a.mp;
                    const bool better = r < best || (r == best && adds < best_adds);
                    if (better || (r == best && adds == best_adds && (bern & 1u))) {
                        store_rows(bw, r > best ? r : best);
                        best = r;
                        best_adds = adds;
                        bump(RC_COPY, 1);
                        flags |= 4u;
                        if (better) enqueue(flags);
                    }
                }
            } else if (!ok) {
                // expand; continue
                exp_flag = 2u;
            } else {
                c_flips++;
                flags |= 1u;
                // ---- R12 local reduction (exact; skipped when no touched row can reduce) ----
                if (need_local) local_reduce(alpha, beta);
                // ---- PAPER:310-313 acceptance ----
                const bool strict = r < best;
                if (strict || (r == best && (bern & 1u))) {
                    store_rows(bw, best);           // rows >= the previous best rank are zero
                    best = r;
                    best_adds = nnz_all() - 2 * r - a.mp;
                    bump(RC_COPY, 1);
                    flags |= 4u;
                    if (strict) enqueue(flags);
                }
                // ---- PAPER:315-317 reduce (R15) ----
                if (bern & 2u) {
                    c_red++;
                    flags |= 16u;
                    if (dover || nD > 0) reduce_all();
                }
                // ---- PAPER:319-321 expand ----
                if ((bern & 4u) && r <= best + a.slack) exp_flag = 32u;
            }
            if (exp_flag) {
                const bool ex = expand();
                flags |= exp_flag | (ex ? 64u : 0u);
                bump(RC_EOK, ex);
                bump(RC_EREJ, !ex);
            }
            const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)(CM ? (best_adds & 1023) : best) << 10) | ((uint64_t)flags << 20) |
                                ((uint64_t)alpha << 32) | ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
            digest = (digest ^ ev) * 0x100000001b3ULL;
            digest ^= digest >> 32;
            if (a.dbg & 1u) {
                const uint32_t bad = check_structure<P>(s, r, nCU, nCV, nCW);
                if (bad && lane == 0 && atomicCAS(a.dbgbuf, 0u, bad) == 0u) {
                    a.dbgbuf[1] = (uint32_t)wk; a.dbgbuf[2] = (uint32_t)step; a.dbgbuf[3] = flags;
                    a.dbgbuf[4] = (uint32_t)r; a.dbgbuf[5] = (uint32_t)alpha; a.dbgbuf[6] = (uint32_t)beta;
                    a.dbgbuf[7] = (uint32_t)(fY | (fZ << 4)); a.dbgbuf[8] = nCU + nCV + nCW;
                    a.dbgbuf[9] = (uint32_t)draws;
                }
            }
            __syncwarp();
        }

        // ---------------- store the walker and its class image ----------------
        store_rows(a.cur + (size_t)wk * FG_PLANES * R, R);
        if (img) {
            uint32_t *nxi = img, *lci = img + 3 * RM / 2, *twi = lci + RM;
#pragma unroll 1
            for (int k = lane; k < 3 * RM / 2; k += 32) nxi[k] = reinterpret_cast<const uint32_t *>(s.nxh)[k];
#pragma unroll 1
            for (int l = lane; l < RM; l += 32) lci[l] = s.lc[l];
            twi[lane] = s.tw[lane];
            if (lane < 16) twi[32 + lane] = s.wsb[lane];
            if (lane == 0) {
                uint32_t *sc = twi + 48;
                sc[0] = nCU; sc[1] = nCV; sc[2] = nCW;
                sc[3] = (uint32_t)dset; sc[4] = (uint32_t)(dset >> 32);
                sc[5] = (uint32_t)nD; sc[6] = dover ? 1u : 0u;
                sc[7] = (uint32_t)r;
            }
        }
        int nnz = 0;
        for (int t = lane; t < best; t += 32)
            nnz += __popcll(bw[0 * R + t]) + __popcll(bw[2 * R + t]) + __popcll(bw[4 * R + t]);
        const int tot_nnz = __reduce_add_sync(FULL, nnz);
        __syncwarp();
        if (lane == 0) {
            hp->r = r;
            hp->best_r = best;
            hp->step = step;
            hp->digest = digest;
            hp->best_adds = best_adds;
            hp->cnt[FG_CNT_STEPS] += a.steps;
            hp->cnt[FG_CNT_DRAWS] += c_draws;
            hp->cnt[FG_CNT_FLIPS] += c_flips;
            hp->cnt[FG_CNT_FLIP_FAIL] += a.steps - c_flips;
            hp->cnt[FG_CNT_EXPAND_OK] += rc[RC_EOK];
            hp->cnt[FG_CNT_EXPAND_REJECT] += rc[RC_EREJ];
            hp->cnt[FG_CNT_MERGES] += rc[RC_MERGE];
            hp->cnt[FG_CNT_ZERO_REMOVED] += rc[RC_ZERO];
            hp->cnt[FG_CNT_BEST_COPIES] += rc[RC_COPY];
            hp->cnt[FG_CNT_IMPROVEMENTS] += rc[RC_IMPR];
            hp->cnt[FG_CNT_REDUCE_CALLS] += c_red;
            int adds = tot_nnz - 2 * best - a.mp;
            if (adds < 0) adds = 0;
            atomicMin(a.best_key, ((unsigned long long)best << 54) | ((unsigned long long)adds << 36) |
                                      (unsigned long long)wk);
        }
        __syncwarp();
    }
}

// shared memory per warp: factors, lc, word totals (32), sign bits (16), Philox table,
// counters, next arrays (3 x RM u16)
template <class P> size_t wl_smem(int nwd)
{
    return (size_t)3 * 32 * nwd * sizeof(typename P::F) + 32 * nwd * 4 + 32 * 4 + 16 * 4 + PXT * PXS * 4 + 8 * 4 +
           3 * 32 * nwd * 2;
}

template <class P, int MINB, bool CM = false>
cudaError_t launch_wl_m(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    const int nwd = (a.R + 31) / 32;
    if (nwd > 16) return cudaErrorInvalidValue;
    const size_t smem = wl_smem<P>(nwd);
    cudaError_t e = cudaFuncSetAttribute(walk_wl<P, MINB, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_wl<P, MINB, CM>, 32, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    int64_t blocks = (int64_t)num_sms * bps;
    if (blocks > a.num_walkers) blocks = a.num_walkers;
    walk_wl<P, MINB, CM><<<(unsigned)blocks, 32, smem, st>>>(a, nwd);
    return cudaGetLastError();
}

// register budget (resident warps per SM the compiler must allow).  Measured
// (scripts/gpu_r02_minb2.sh, gpu_r02_minb3.sh, profiles/r02_ab_wl_minb.txt): P32 (C4, register
// limited) runs best with 18 warps' worth (113 registers; 96 spills more, 128 loses warps);
// the 16-byte layouts are shared-memory limited, so the budget follows the warps that fit:
// 14 for (4,5,12) (14 fit), 11 for (5,6,10) and (6,7,9) (11 / 9 fit): +2 ... +5 % over 128
// registers.  FG_WL_MINB overrides (A/B).
template <class P>
cudaError_t launch_wl(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    // R24 runs with the largest register budget (not a throughput path)
    if (a.mode == 1) return launch_wl_m<P, 11, true>(a, num_sms, st);
    const char *ev = getenv("FG_WL_MINB");
    int mb = ev ? atoi(ev) : 0;
    if (mb == 0) {
        if (std::is_same<P, P32>::value) {
            mb = 18;
        } else if (sizeof(typename P::F) > 8) {
            int dev = 0, per_sm = 0, reserve = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            cudaDeviceGetAttribute(&reserve, cudaDevAttrReservedSharedMemoryPerBlock, dev);
            const int fit = per_sm / (int)(wl_smem<P>((a.R + 31) / 32) + reserve);
            mb = fit >= 16 ? 16 : (fit >= 14 ? 14 : 11);
        } else {
            mb = 16;
        }
    }
    if (mb == 11) return launch_wl_m<P, 11>(a, num_sms, st);
    if (mb == 14) return launch_wl_m<P, 14>(a, num_sms, st);
    if (mb == 18) return launch_wl_m<P, 18>(a, num_sms, st);
    if (mb == 20) return launch_wl_m<P, 20>(a, num_sms, st);
    return launch_wl_m<P, 16>(a, num_sms, st);
}

}  // namespace fgwl
