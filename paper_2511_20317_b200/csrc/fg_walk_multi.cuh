// fg_walk_multi.cu -- the RandomWalk kernel (Algorithm 1) for
// walkers with 33..512 rows (configs C3-C5: (4,4,4) R=96, (5,5,5) R=160,
// (4,5,12)/(5,6,10)/(6,7,9) R=256/320/416).  ONE WALKER PER WARP, rows in shared
// memory; lane L owns rows L*NS .. L*NS+NS-1 ("blocked", so a lane's local prefix
// plus one warp scan gives the canonical (role, row) order of R10), stored at
// physical index slot*32 + L (bank-conflict free when lanes sweep their rows).
//
// Instead of the R<=32 kernel's equality masks (R bits per row), each lane keeps
// per row and role the number of LATER rows in the same class (U, V equal; W equal
// up to sign), packed 3 x 10 bits.  Every change of a factor / removal / appended
// row updates these counts exactly with one broadcast + compare sweep (O(R/32) per
// lane), so a step costs O(R/32) instead of the oracle's O(R^2):
//   - prefix: lane sums + one 64-bit warp scan (3 x 21-bit fields);
//   - each draw (R11, sequential): ballot for the owning lane, lane-local slot
//     search, then j by one compare sweep against x_i + warp scan + nth bit;
//   - R12 (exact skip): rows alpha, beta against all rows for "two shared factors";
//   - R15 reduce_all: only rows touched by expands since the last clean scan can be
//     in a reducible pair (flips are cleaned by R12), so the exact lexicographic
//     search scans that small dirty set D (or all rows if D overflows);
//   - expand (R16), acceptance, verify queue, digest as in fg_walk.cu.
#pragma once
#include "fg_device.cuh"

using namespace fgd;

#define PXS 9

namespace fgwm {

template <class P, int NS, bool CM>
__global__ void __launch_bounds__(32) walk_wm(WalkArgs a)
{
    typedef typename P::F F;
    extern __shared__ __align__(16) unsigned char smraw[];
    F *sf = reinterpret_cast<F *>(smraw);                    // [3][NS*32]
    uint32_t *px = reinterpret_cast<uint32_t *>(sf + 3 * NS * 32);
    uint32_t *rc = px + 32 * PXS;                            // 8 rare counters
    const int lane = threadIdx.x;
    const int R = a.R;
    const uint64_t seed = a.seed;
    const uint32_t kf = a.k_flip;
    constexpr int PLANE = NS * 32;
    // per-row slot loops: fully unrolled up to 8 slots; rolled above (the class counts then
    // live in local memory) -- the fully unrolled kernel for NS = 13 is 39k instructions
    // and stalls on instruction fetch
    constexpr int UNS = NS > 8 ? 1 : NS;

    auto grab = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.work_counter, 1ull);
        return (int64_t)__shfl_sync(FULL, v, 0);
    };
    // physical slot of row l, (l % NS) * 32 + l / NS, from a per-CTA table (a division by
    // the constant NS costs ~5 instructions on every dynamic row access)
    unsigned short *phtab = reinterpret_cast<unsigned short *>(rc + 8);
    for (int t = lane; t < NS * 32; t += 32) phtab[t] = (unsigned short)((t % NS) * 32 + t / NS);
    __syncwarp();
    auto ph = [&](int l) { return (int)phtab[l]; };
    auto fat = [&](int X, int l) -> F { return sf[X * PLANE + ph(l)]; };
    auto own = [&](int X, int s) -> F { return sf[X * PLANE + s * 32 + lane]; };

    for (int64_t wk = grab(); wk < a.num_walkers; wk = grab()) {
        // ---------------- load walker ----------------
        const uint64_t *cp = a.cur + (size_t)wk * FG_PLANES * R;
        uint64_t *bw = a.best + (size_t)wk * FG_PLANES * R;
        for (int t = lane; t < PLANE; t += 32) {
            F u = P::make(0, 0), v = u, w = u;
            if (t < R) {
                u = P::make(cp[0 * R + t], cp[1 * R + t]);
                v = P::make(cp[2 * R + t], cp[3 * R + t]);
                w = P::make(cp[4 * R + t], cp[5 * R + t]);
            }
            sf[0 * PLANE + ph(t)] = u;
            sf[1 * PLANE + ph(t)] = v;
            sf[2 * PLANE + ph(t)] = w;
        }
        if (lane < 8) rc[lane] = 0;
        __syncwarp();
        fg_whdr *hp = a.hdr + wk;
        int r = hp->r;
        int best = hp->best_r;
        uint64_t step = hp->step;
        uint64_t digest = hp->digest;
        int best_adds = hp->best_adds;
        const uint32_t wid = (uint32_t)(a.id_base + wk);
        constexpr bool cmode = CM;               // R24: naive-complexity minimisation
        uint32_t c_draws = 0, c_flips = 0, c_red = 0;
        enum { RC_EOK = 0, RC_EREJ, RC_MERGE, RC_ZERO, RC_COPY, RC_IMPR };
        auto bump = [&](int k, uint32_t v) { if (lane == 0) rc[k] += v; };

        // ---------------- class counts (R10) ----------------
        uint32_t cnt[NS];
        // bits of the (row l) x (factor triple b) class relation, roles U | V<<10 | W<<20
        auto cls3 = [&](int s, F bu, F bv, F bw_, F nbw, bool zu, bool zv, bool zw) -> uint32_t {
            const uint32_t mu = !zu && P::eq(own(0, s), bu);
            const uint32_t mv = !zv && P::eq(own(1, s), bv);
            const F xw = own(2, s);
            const uint32_t mw = !zw && (P::eq(xw, bw_) || P::eq(xw, nbw));
            return mu | (mv << 10) | (mw << 20);
        };
        // cnt[l] += sign * rel(row l, t-content) for l < t
        auto pair_update = [&](int t, F bu, F bv, F bw_, int sign) {
            const F nbw = P::neg(bw_);
            const bool zu = P::zero(bu), zv = P::zero(bv), zw = P::zero(bw_);
#pragma unroll UNS
            for (int s = 0; s < NS; ++s) {
                const int l = lane * NS + s;
                if (l < t) {
                    const uint32_t b = cls3(s, bu, bv, bw_, nbw, zu, zv, zw);
                    cnt[s] = sign > 0 ? cnt[s] + b : cnt[s] - b;
                }
            }
        };
        // cnt[t] = #{ j > t, j < r : rel(row j, t-content) } per role
        auto count_above = [&](int t, F bu, F bv, F bw_) {
            const F nbw = P::neg(bw_);
            const bool zu = P::zero(bu), zv = P::zero(bv), zw = P::zero(bw_);
            uint32_t acc = 0;
#pragma unroll UNS
            for (int s = 0; s < NS; ++s) {
                const int l = lane * NS + s;
                if (l > t && l < r) acc += cls3(s, bu, bv, bw_, nbw, zu, zv, zw);
            }
            acc = (uint32_t)__reduce_add_sync(FULL, acc & 1023u) |
                  ((uint32_t)__reduce_add_sync(FULL, (acc >> 10) & 1023u) << 10) |
                  ((uint32_t)__reduce_add_sync(FULL, acc >> 20) << 20);
#pragma unroll UNS
            for (int s = 0; s < NS; ++s)
                if (lane * NS + s == t) cnt[s] = acc;
        };
        auto set_cnt = [&](int t, uint32_t v) {
#pragma unroll UNS
            for (int s = 0; s < NS; ++s)
                if (lane * NS + s == t) cnt[s] = v;
        };
        auto recount = [&]() {
#pragma unroll UNS
            for (int s = 0; s < NS; ++s) cnt[s] = 0;
            for (int t = 1; t < r; ++t) pair_update(t, fat(0, t), fat(1, t), fat(2, t), +1);
        };
        // change factor X of row t from its current value to nv (exact count update)
        auto change_factor = [&](int t, int X, F nv) {
            const F ov = fat(X, t);
            const F no = P::neg(ov), nn = P::neg(nv);
            const bool zo = P::zero(ov), zn = P::zero(nv);
            const bool classdiff = X == 2 ? !P::eq(P::abs(ov), P::abs(nv)) : !P::eq(ov, nv);
            if (classdiff || zo != zn) {
                uint32_t above = 0;
#pragma unroll UNS
                for (int s = 0; s < NS; ++s) {
                    const int l = lane * NS + s;
                    const F x = own(X, s);
                    const uint32_t mo = !zo && (P::eq(x, ov) || (X == 2 && P::eq(x, no)));
                    const uint32_t mn = !zn && (P::eq(x, nv) || (X == 2 && P::eq(x, nn)));
                    if (l < t) cnt[s] = cnt[s] + ((mn - mo) << (10 * X));
                    above += (l > t && l < r) ? mn : 0u;
                }
                const uint32_t tot = (uint32_t)__reduce_add_sync(FULL, above);
#pragma unroll UNS
                for (int s = 0; s < NS; ++s)
                    if (lane * NS + s == t) cnt[s] = (cnt[s] & ~(1023u << (10 * X))) | (tot << (10 * X));
            }
            __syncwarp();
            if (lane == 0) sf[X * PLANE + ph(t)] = nv;
            __syncwarp();
        };

        // ---------------- dirty set D for R15 (<= 6 rows, 10 bits each) ----------------
        uint64_t dset = 0;
        int nD = 0;
        bool dover = true;          // unknown at load: first reduce_all scans everything
        auto d_add = [&](int x) {
            if (dover) return;
            for (int k = 0; k < nD; ++k)
                if ((int)((dset >> (10 * k)) & 1023u) == x) return;
            if (nD == 6) { dover = true; return; }
            dset |= (uint64_t)x << (10 * nD);
            nD++;
        };

        // R14 remove(h) with optional worklist (entries == h dropped, r-1 -> h)
        auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) {
            const int last = r - 1;
            const F lu = fat(0, last), lv = fat(1, last), lw = fat(2, last);
            pair_update(last, lu, lv, lw, -1);
            if (h != last) {
                pair_update(h, fat(0, h), fat(1, h), fat(2, h), -1);
                __syncwarp();
                if (lane == 0) {
                    sf[0 * PLANE + ph(h)] = lu;
                    sf[1 * PLANE + ph(h)] = lv;
                    sf[2 * PLANE + ph(h)] = lw;
                }
                __syncwarp();
                r--;
                pair_update(h, lu, lv, lw, +1);
                count_above(h, lu, lv, lw);
            } else {
                r--;
            }
            set_cnt(last, 0u);
            int n2 = 0, x0 = 0, x1 = 0;
            if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
            if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
            wl0 = x0; wl1 = x1; nwl = n2;
            if (h != last) {
                if (nwl >= 1 && wl0 == last) wl0 = h;
                if (nwl >= 2 && wl1 == last) wl1 = h;
            }
            // D: drop h, remap last -> h
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
        auto row_at = [&](int l) { Row<P> o; o.u = fat(0, l); o.v = fat(1, l); o.w = fat(2, l); return o; };
        auto put_row = [&](int t, const Row<P> &nr) {
            change_factor(t, 0, nr.u);
            change_factor(t, 1, nr.v);
            change_factor(t, 2, nr.w);
        };
        // after a flip only factor X of row t can change class (normalisation negates
        // the changed factor and w, whose class is sign-free); other factors of t may
        // change sign only: plain stores
        auto put_flip_row = [&](int t, int X, const Row<P> &nr) {
            change_factor(t, X, get(nr, X));
            if (lane == 0) {
                const int pt = ph(t);
                if (X != 0) sf[0 * PLANE + pt] = nr.u;
                if (X != 1) sf[1 * PLANE + pt] = nr.v;
                if (X != 2) sf[2 * PLANE + pt] = nr.w;
            }
            __syncwarp();
        };
        auto append_row = [&](const Row<P> &nr) {
            const int t = r;
            __syncwarp();
            if (lane == 0) {
                sf[0 * PLANE + ph(t)] = nr.u;
                sf[1 * PLANE + ph(t)] = nr.v;
                sf[2 * PLANE + ph(t)] = nr.w;
            }
            __syncwarp();
            pair_update(t, nr.u, nr.v, nr.w, +1);
            set_cnt(t, 0u);
            r++;
        };
        // first row l != t (ascending) with reducible(row t, row l) exact; -1 if none
        auto first_reducible = [&](const Row<P> &rt, int t, int lmin, Row<P> &merged) -> int {
            int found = 0x7fffffff;
            Row<P> mg = rt;
#pragma unroll UNS
            for (int s = 0; s < NS; ++s) {
                const int l = lane * NS + s;
                if (l < r && l != t && l >= lmin && found == 0x7fffffff) {
                    Row<P> rl;
                    rl.u = own(0, s); rl.v = own(1, s); rl.w = own(2, s);
                    if (reducible<P>(rt, rl, mg)) found = l;
                }
            }
            const int j = __reduce_min_sync(FULL, found);
            if (j == 0x7fffffff) return -1;
            const int src = j / NS;
            merged.u = P::shfl(mg.u, src);
            merged.v = P::shfl(mg.v, src);
            merged.w = P::shfl(mg.w, src);
            return j;
        };

        // R12: exact worklist reduction after a flip touching rows a0, b0
        auto slow_local_reduce = [&](int a0, int b0) {
            int wl0 = a0, wl1 = b0, nwl = 2;
            while (nwl > 0) {
                const int t = wl0;
                wl0 = wl1;
                nwl--;
                if (t >= r) continue;
                const Row<P> rt = row_at(t);
                if (has_zero(rt)) {
                    remove_row(t, wl0, wl1, nwl);
                    bump(RC_ZERO, 1);
                    continue;
                }
                Row<P> mg;
                const int j = first_reducible(rt, t, 0, mg);
                if (j < 0) continue;
                const int lo = t < j ? t : j, hi = t < j ? j : t;
                put_row(lo, mg);
                bump(RC_MERGE, 1);
                remove_row(hi, wl0, wl1, nwl);
                if (has_zero(mg)) {
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
        auto slow_reduce_all = [&]() {
            for (;;) {
                int zfirst = 0x7fffffff;
#pragma unroll UNS
                for (int s = 0; s < NS; ++s) {
                    const int l = lane * NS + s;
                    if (l < r && zfirst == 0x7fffffff &&
                        (P::zero(own(0, s)) || P::zero(own(1, s)) || P::zero(own(2, s))))
                        zfirst = l;
                }
                zfirst = __reduce_min_sync(FULL, zfirst);
                if (zfirst != 0x7fffffff) {
                    int n0 = 0, x0 = 0, x1 = 0;
                    remove_row(zfirst, x0, x1, n0);
                    bump(RC_ZERO, 1);
                    continue;
                }
                int bi = -1, bj = -1;
                if (dover) {
                    for (int i = 0; i + 1 < r && bi < 0; ++i) {
                        Row<P> mg;
                        const int j = first_reducible(row_at(i), i, i + 1, mg);
                        if (j >= 0) { bi = i; bj = j; }
                    }
                } else {
                    int bestkey = 0x7fffffff;
                    for (int k = 0; k < nD; ++k) {
                        const int d = (int)((dset >> (10 * k)) & 1023u);
                        const Row<P> rd = row_at(d);
                        int key = 0x7fffffff;
#pragma unroll UNS
                        for (int s = 0; s < NS; ++s) {
                            const int l = lane * NS + s;
                            if (l < r && l != d) {
                                Row<P> rl, mg;
                                rl.u = own(0, s); rl.v = own(1, s); rl.w = own(2, s);
                                if (reducible<P>(rd, rl, mg)) {
                                    const int kk = (l < d ? l : d) * 1024 + (l < d ? d : l);
                                    key = kk < key ? kk : key;
                                }
                            }
                        }
                        key = __reduce_min_sync(FULL, key);
                        bestkey = key < bestkey ? key : bestkey;
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
                Row<P> mg = row_at(bi);
                const Row<P> ri = mg, rj = row_at(bj);
                reducible<P>(ri, rj, mg);
                put_row(bi, mg);
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
            const int A = perm >> 1;
            const int B = (1161 >> (2 * perm)) & 3;
            const int Cr = 3 - A - B;
            const Row<P> ri = row_at(i), rj = row_at(j);
            const F ai = get(ri, A), aj = get(rj, A), bi_ = get(ri, B), bj_ = get(rj, B);
            const F ci = get(ri, Cr), cj = get(rj, Cr);
            bool ok = true;
            Row<P> ni = ri, nj = rj, nr = ri;
            if (plus) {
                if (!distinct<P>(ai, aj) || !distinct<P>(bi_, bj_) || !distinct<P>(ci, cj)) return false;
                const F t1 = P::add(bi_, bj_, ok);
                const F t2 = P::sub(cj, ci, ok);
                const F t3 = P::sub(aj, ai, ok);
                if (!ok) return false;
                set(ni, B, t1, true);
                set(nj, A, ai, true);
                set(nj, Cr, t2, true);
                set(nr, A, t3, true);
                set(nr, B, bj_, true);
                set(nr, Cr, cj, true);
            } else {
                if (!distinct<P>(ai, aj)) return false;
                const F t3 = P::sub(ai, aj, ok);
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
            put_row(i, ni);
            put_row(j, nj);
            append_row(nr);
            d_add(i);
            d_add(j);
            d_add(rold);
            return true;
        };

        // copy of the current rows to an HBM scheme image (best / verify queue)
        auto store_rows = [&](uint64_t *dst) {
            for (int t = lane; t < R; t += 32) {
                const bool lv = t < r;
                const F u = fat(0, t), v = fat(1, t), w = fat(2, t);
                dst[0 * R + t] = lv ? P::dig(u) : 0;
                dst[1 * R + t] = lv ? P::sgn(u) : 0;
                dst[2 * R + t] = lv ? P::dig(v) : 0;
                dst[3 * R + t] = lv ? P::sgn(v) : 0;
                dst[4 * R + t] = lv ? P::dig(w) : 0;
                dst[5 * R + t] = lv ? P::sgn(w) : 0;
            }
        };

        auto nnz_all = [&]() -> int {
            int v = 0;
#pragma unroll UNS
            for (int s = 0; s < NS; ++s)
                if (lane * NS + s < r) v += P::popd(own(0, s)) + P::popd(own(1, s)) + P::popd(own(2, s));
            return __reduce_add_sync(FULL, v);
        };
        auto popr = [&](const Row<P> &x) { return P::popd(x.u) + P::popd(x.v) + P::popd(x.w); };
        recount();
        int nnz_cur = nnz_all();
        int boff = 32;
        const uint32_t nsteps = (uint32_t)a.steps;
        for (uint32_t it = 0; it < nsteps; ++it, ++step, ++boff) {
            if (boff == 32) {
                uint32_t o0, o1, o2, o3;
                philox_block(seed, step + lane, wid, 0u, o0, o1, o2, o3);
                px[lane * PXS + 0] = o0;
                px[lane * PXS + 1] = (o1 < a.thr_eq ? 1u : 0u) | (o2 < a.thr_reduce ? 2u : 0u) |
                                     (o3 < a.thr_expand ? 4u : 0u);
                philox_block(seed, step + lane, wid, 2u, o0, o1, o2, o3);
                px[lane * PXS + 4] = o0; px[lane * PXS + 5] = o1;
                px[lane * PXS + 6] = o2; px[lane * PXS + 7] = o3;
                __syncwarp();
                boff = 0;
            }
            const uint32_t *pw = px + boff * PXS;
            const uint32_t bern = pw[1];
            uint32_t flags = 0;
            int alpha = 0, beta = 0, draws = 0;
            bool ok = false;

            // ---- R10 counts: lane sums (3 x 21 bits) + warp scan ----
            uint64_t lsum = 0;
#pragma unroll UNS
            for (int s = 0; s < NS; ++s)
                lsum += (uint64_t)(cnt[s] & 1023u) | ((uint64_t)((cnt[s] >> 10) & 1023u) << 21) |
                        ((uint64_t)(cnt[s] >> 20) << 42);
            uint64_t incl = lsum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            const uint64_t tot = __shfl_sync(FULL, incl, 31);
            const uint32_t nU = (uint32_t)(tot & 0x1fffffu), nV = (uint32_t)((tot >> 21) & 0x1fffffu);
            const uint32_t nW = (uint32_t)(tot >> 42);
            const uint32_t nC = nU + nV + nW;
            const uint64_t excl = incl - lsum;

            // ---- R11 try_flip (draws sequential; each O(R/32) per lane) ----
            if (nC) {
                uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;
                for (uint32_t at = 0; at < kf; ++at) {
                    uint32_t x;
                    if (at == 0) x = pw[0];
                    else if (at <= 4) x = pw[3 + at];
                    else {
                        const uint32_t slot = 7 + at;
                        if ((slot & 3) == 0) philox_block(seed, step, wid, slot >> 2, e0, e1, e2, e3);
                        const uint32_t ws = slot & 3;
                        x = ws == 0 ? e0 : (ws == 1 ? e1 : (ws == 2 ? e2 : e3));
                    }
                    draws++;
                    const uint32_t k = __umulhi(x, 4u * nC);
                    const uint32_t idx = k >> 2;
                    const int d = k & 1, e = (k >> 1) & 1;
                    const uint32_t g1 = idx >= nU, g2 = idx >= nU + nV;
                    const int X = (int)(g1 + g2);
                    const uint32_t qq = idx - (g1 ? nU : 0u) - (g2 ? nV : 0u);
                    const int sh = 21 * X;
                    // owner lane of row i, then the slot inside it
                    const uint32_t inX = (uint32_t)((incl >> sh) & 0x1fffffu);
                    const int L = __ffs(__ballot_sync(FULL, inX > qq)) - 1;
                    const uint32_t q1 = qq - (uint32_t)((__shfl_sync(FULL, excl, L) >> sh) & 0x1fffffu);
                    int sl = 0;
                    uint32_t q2 = 0, cum = 0;
                    bool found = false;
#pragma unroll UNS
                    for (int s = 0; s < NS; ++s) {
                        const uint32_t f = (cnt[s] >> (10 * X)) & 1023u;
                        if (!found && cum + f > q1) { found = true; sl = s; q2 = q1 - cum; }
                        cum += f;
                    }
                    sl = __shfl_sync(FULL, sl, L);
                    q2 = __shfl_sync(FULL, q2, L);
                    const int i = L * NS + sl;
                    // j: the q2-th row after i in the class of x_X[i]
                    const F xi = fat(X, i);
                    const F nxi = P::neg(xi);
                    uint32_t bits = 0;
#pragma unroll UNS
                    for (int s = 0; s < NS; ++s) {
                        const int l = lane * NS + s;
                        const F xl = own(X, s);
                        const bool m = l > i && l < r && (P::eq(xl, xi) || (X == 2 && P::eq(xl, nxi)));
                        bits |= (uint32_t)m << s;
                    }
                    const uint32_t cb = __popc(bits);
                    uint32_t ex = cb;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(FULL, ex, o);
                        if (lane >= o) ex += t;
                    }
                    ex -= cb;
                    const int M = __ffs(__ballot_sync(FULL, ex <= q2 && q2 < ex + cb)) - 1;
                    uint32_t bm = bits;
                    const uint32_t tt = q2 - ex;     // garbage (large) off lane M: bounded below
                    bm = tt > 0 ? (bm & (bm - 1u)) : bm;
                    bm = tt > 1 ? (bm & (bm - 1u)) : bm;
                    for (uint32_t z = 2; z < tt && z < NS; ++z) bm &= bm - 1u;
                    const int jsl = __shfl_sync(FULL, __ffs(bm) - 1, M);
                    const int j = M * NS + jsl;
                    const int al = d ? j : i, be = d ? i : j;
                    const unsigned yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
                    const int Y = yz & 3, Z = yz >> 2;
                    const Row<P> ra = row_at(al), rb = row_at(be);
                    const bool sneg = P::RING == FG_ZT && X == 2 && !P::eq(ra.w, rb.w);
                    bool v = true;
                    const F yb = get(rb, Y);
                    const F ny = P::add(get(ra, Y), P::sel(sneg, P::neg(yb), yb), v);
                    const F nz = P::sub(get(rb, Z), get(ra, Z), v);
                    // R24: no reduction edges -> a draw making a factor zero is rejected
                    if (cmode) v = v && !P::zero(ny) && !P::zero(nz);
                    if (!v) continue;
                    Row<P> na = ra, nb = rb;
                    set(na, Y, ny, true);
                    set(nb, Z, nz, true);
                    normalize<P>(na);
                    normalize<P>(nb);
                    put_flip_row(al, Y, na);
                    put_flip_row(be, Z, nb);
                    if (cmode) nnz_cur += popr(na) + popr(nb) - popr(ra) - popr(rb);
                    alpha = al;
                    beta = be;
                    ok = true;
                    break;
                }
            }
            c_draws += draws;

            if (cmode) {
                // ---- R24 step: flips only; best by (rank, naive additions) ----
                if (ok) {
                    c_flips++;
                    flags |= 1u;
                    const int adds = nnz_cur - 2 * r - a.mp;
                    const bool better = r < best || (r == best && adds < best_adds);
                    if (better || (r == best && adds == best_adds && (bern & 1u))) {
                        best = r;
                        best_adds = adds;
                        bump(RC_COPY, 1);
                        flags |= 4u;
                        store_rows(bw);
                        if (better) {
                            flags |= 8u;
                            bump(RC_IMPR, 1);
                            unsigned slot = 0;
                            if (lane == 0) slot = atomicAdd(a.q_count, 1u);
                            slot = __shfl_sync(FULL, slot, 0);
                            if (slot < a.q_cap) {
                                store_rows(a.q_planes + (size_t)slot * FG_PLANES * R);
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
                        }
                    }
                }
            }
            // expand (R16) runs last on both paths: one inlined copy
            uint32_t exp_flag = 0;
            if (cmode) {
            } else if (!ok) {
                // expand; continue
                exp_flag = 2u;
            } else {
                c_flips++;
                flags |= 1u;
                // ---- R12 exact skip: touched rows sharing two factors with any row ----
                {
                    const Row<P> ra = row_at(alpha), rb = row_at(beta);
                    const F nwa = P::neg(ra.w), nwb = P::neg(rb.w);
                    bool need = has_zero(ra) || has_zero(rb);
                    bool hit = false;
#pragma unroll UNS
                    for (int s = 0; s < NS; ++s) {
                        const int l = lane * NS + s;
                        if (l < r) {
                            const F xu = own(0, s), xv = own(1, s), xw = own(2, s);
                            const int ca = (int)P::eq(xu, ra.u) + (int)P::eq(xv, ra.v) +
                                           (int)(P::eq(xw, ra.w) || P::eq(xw, nwa));
                            const int cb2 = (int)P::eq(xu, rb.u) + (int)P::eq(xv, rb.v) +
                                            (int)(P::eq(xw, rb.w) || P::eq(xw, nwb));
                            hit |= (l != alpha && ca >= 2) || (l != beta && cb2 >= 2);
                        }
                    }
                    need |= __any_sync(FULL, hit);
                    if (need) slow_local_reduce(alpha, beta);
                }
                // ---- PAPER:310-313 acceptance ----
                bool acc = r < best;
                if (!acc && r == best) acc = bern & 1u;
                if (acc) {
                    const bool strict = r < best;
                    best = r;
                    best_adds = nnz_all() - 2 * r - a.mp;
                    bump(RC_COPY, 1);
                    flags |= 4u;
                    store_rows(bw);
                    if (strict) {
                        flags |= 8u;
                        bump(RC_IMPR, 1);
                        unsigned slot = 0;
                        if (lane == 0) slot = atomicAdd(a.q_count, 1u);
                        slot = __shfl_sync(FULL, slot, 0);
                        if (slot < a.q_cap) {
                            store_rows(a.q_planes + (size_t)slot * FG_PLANES * R);
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
                    }
                }
                // ---- PAPER:315-317 reduce (R15) ----
                if (bern & 2u) {
                    c_red++;
                    flags |= 16u;
                    if (dover || nD > 0) slow_reduce_all();
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
            const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)(cmode ? (best_adds & 1023) : best) << 10) |
                                ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) |
                                ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
            digest = (digest ^ ev) * 0x100000001b3ULL;
            digest ^= digest >> 32;
            __syncwarp();
        }

        // ---------------- store walker ----------------
        store_rows(a.cur + (size_t)wk * FG_PLANES * R);
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
            const unsigned long long key = ((unsigned long long)best << 54) |
                                           ((unsigned long long)adds << 36) | (unsigned long long)wk;
            atomicMin(a.best_key, key);
        }
        __syncwarp();
    }
}

template <class P, int NS, bool CM>
cudaError_t launch_wm_m(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    const size_t smem = 3 * NS * 32 * sizeof(typename P::F) + 32 * PXS * 4 + 8 * 4 + NS * 32 * 2;
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_wm<P, NS, CM>, 32, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    int64_t blocks = (int64_t)num_sms * bps;
    if (blocks > a.num_walkers) blocks = a.num_walkers;
    walk_wm<P, NS, CM><<<(unsigned)blocks, 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <class P, int NS>
cudaError_t launch_wm(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    return a.mode == 1 ? launch_wm_m<P, NS, true>(a, num_sms, st) : launch_wm_m<P, NS, false>(a, num_sms, st);
}

}  // namespace fgwm
