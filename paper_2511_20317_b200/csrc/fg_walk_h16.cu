// fg_walk_h16.cu -- the RandomWalk kernel (Algorithm 1) for walkers
// with at most 32 rows, TWO WALKERS PER WARP: half-warp h (16 lanes) runs walker
// 2g+h, lane k of the half holds rows k and 16+k ("slots" 0 and 1).
//
// Same algorithm, readings and digest as fg_walk.cu (one walker per warp); what
// changes is the mapping.  The one-walker kernel spends most of its issue slots on
// per-walker work that is identical on every lane (draw evaluation, Philox, the
// Alg. 1 tail) and is ALU-pipe bound (profiles/r01_ncu_walk_v5.txt); here one warp
// instruction serves two walkers for all of that, and only the per-row work (class
// masks, counts) doubles per lane.
//   - per-half shared memory mirrors the row keys, the class masks and the row
//     prefix, so a draw reads any row / mask / prefix with one LDS;
//   - draws 0..4 are evaluated lane-parallel in each half (lane k = draw k), 5..15 on
//     demand; the ballot of each half picks its first valid draw (R11);
//   - rare paths (merges, removals, expand, acceptance copies) run divergently per
//     half with half-warp masks.
#include "fg_device.cuh"

using namespace fgd;

#define H16_THREADS 128
#define H16_WARPS (H16_THREADS / 32)
#define PXS 9
#ifndef H16_MINB
#define H16_MINB 6
#endif

namespace {

__device__ __forceinline__ int nth_bit16(uint32_t x, uint32_t t)
{
    x = t > 0 ? (x & (x - 1u)) : x;
    x = t > 1 ? (x & (x - 1u)) : x;
    x = t > 2 ? (x & (x - 1u)) : x;
    for (uint32_t k = 3; k < t && k < 32; ++k) x &= x - 1u;
    return __ffs(x) - 1;
}

template <class P> struct Ev {
    int info;                  // al | be << 8 | Y << 16 | Z << 18
    typename P::F ny, nz;
};

template <class P>
__global__ void __launch_bounds__(H16_THREADS, H16_MINB) walk_h16(WalkArgs a)
{
    typedef typename P::F F;
    __shared__ F sR_all[H16_WARPS][2][3][32];          // row keys   [half][role][row]
    __shared__ uint32_t sM_all[H16_WARPS][2][3][32];   // class masks
    __shared__ uint32_t sP_all[H16_WARPS][2][32];      // inclusive prefix per row (3 x 10 bits)
    __shared__ uint32_t px_all[H16_WARPS][2][32 * PXS];
    __shared__ uint32_t rc_all[H16_WARPS][2][8];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, k = lane & 15, hb = h << 4;
    const unsigned hm = 0xffffu << hb;
    F(*sR)[32] = sR_all[wib][h];
    uint32_t(*sM)[32] = sM_all[wib][h];
    uint32_t *sP = sP_all[wib][h];
    uint32_t *px = px_all[wib][h];
    uint32_t *rc = rc_all[wib][h];
    const int R = a.R;
    const uint64_t seed = a.seed;
    const uint32_t kf = a.k_flip;
    const unsigned ab0 = ~((2u << k) - 1u), ab1 = ~((2u << (16 + k)) - 1u);   // rows above k, 16+k
    const unsigned prm = h ? 0x7632u : 0x5410u;       // half-h bits of two ballots -> 32-row mask

    for (;;) {
        unsigned long long g = 0;
        if (lane == 0) g = atomicAdd(a.work_counter, 2ull);
        g = __shfl_sync(FULL, g, 0);
        if ((int64_t)g >= a.num_walkers) break;
        const int64_t wk = (int64_t)g + h;
        const bool act = wk < a.num_walkers;

        // ---------------- load (rows k and 16+k of this half's walker) ----------------
        const uint64_t *cp = a.cur + (size_t)(act ? wk : 0) * FG_PLANES * R;
        uint64_t *bw = a.best + (size_t)(act ? wk : 0) * FG_PLANES * R;
        Row<P> row0, row1;
        row0.u = row0.v = row0.w = P::make(0, 0);
        row1 = row0;
        if (act && k < R) {
            row0.u = P::make(cp[0 * R + k], cp[1 * R + k]);
            row0.v = P::make(cp[2 * R + k], cp[3 * R + k]);
            row0.w = P::make(cp[4 * R + k], cp[5 * R + k]);
        }
        if (act && 16 + k < R) {
            row1.u = P::make(cp[0 * R + 16 + k], cp[1 * R + 16 + k]);
            row1.v = P::make(cp[2 * R + 16 + k], cp[3 * R + 16 + k]);
            row1.w = P::make(cp[4 * R + 16 + k], cp[5 * R + 16 + k]);
        }
        sR[0][k] = row0.u; sR[1][k] = row0.v; sR[2][k] = row0.w;
        sR[0][16 + k] = row1.u; sR[1][16 + k] = row1.v; sR[2][16 + k] = row1.w;
        if (k < 8) rc[k] = 0;
        fg_whdr *hp = a.hdr + (act ? wk : 0);
        int r = act ? hp->r : 0;
        int best = act ? hp->best_r : 0;
        uint64_t step = act ? hp->step : 0;
        uint64_t digest = act ? hp->digest : 0;
        int best_adds = act ? hp->best_adds : 0;
        const uint32_t wid = (uint32_t)(a.id_base + (act ? wk : 0));
        uint32_t c_draws = 0, c_flips = 0, c_red = 0;
        enum { RC_EOK = 0, RC_EREJ, RC_MERGE, RC_ZERO, RC_COPY, RC_IMPR };
        auto bump = [&](int i, uint32_t v) { if (k == 0) rc[i] += v; };
        __syncwarp();

        unsigned mU0 = 0, mV0 = 0, mW0 = 0, mU1 = 0, mV1 = 0, mW1 = 0;
        F wA0 = P::abs(row0.w), wA1 = P::abs(row1.w);
        auto store_masks = [&]() {
            sM[0][k] = mU0; sM[1][k] = mV0; sM[2][k] = mW0;
            sM[0][16 + k] = mU1; sM[1][16 + k] = mV1; sM[2][16 + k] = mW1;
        };
        // all class masks of this half from the row mirror (no collectives: safe
        // under half divergence)
        auto full_masks = [&]() {
            wA0 = P::abs(row0.w);
            wA1 = P::abs(row1.w);
            const bool l0 = k < r, l1 = 16 + k < r;
            mU0 = mV0 = mW0 = mU1 = mV1 = mW1 = 0;
#pragma unroll 4
            for (int t = 0; t < 32; ++t) {
                const bool tl = t < r;
                const F tu = sR[0][t], tv = sR[1][t], ta = P::abs(sR[2][t]);
                const unsigned bt = 1u << t;
                mU0 |= (tl && l0 && P::eq(row0.u, tu)) ? bt : 0u;
                mV0 |= (tl && l0 && P::eq(row0.v, tv)) ? bt : 0u;
                mW0 |= (tl && l0 && P::eq(wA0, ta)) ? bt : 0u;
                mU1 |= (tl && l1 && P::eq(row1.u, tu)) ? bt : 0u;
                mV1 |= (tl && l1 && P::eq(row1.v, tv)) ? bt : 0u;
                mW1 |= (tl && l1 && P::eq(wA1, ta)) ? bt : 0u;
            }
            store_masks();
        };

        // ---------------- rare paths ----------------
        // The WHOLE warp works on one half's walker: lane l holds row l (read from and
        // written back to that half's mirror), so every collective is full-warp and the
        // code is the one-walker-per-warp routine of fg_walk.cu.  which: 0 = R12 local
        // reduction of rows (ta, tb), 1 = R15 reduce_all, 2 = R16 expand.  Returns the
        // walker's new rank.
        auto rare = [&](int hs, int which, int ta, int tb, int &ei, int &ej) -> int {
            F(*S)[32] = sR_all[wib][hs];
            uint32_t *RC = rc_all[wib][hs];
            int rr = __shfl_sync(FULL, r, hs << 4);
            const uint64_t stp = __shfl_sync(FULL, step, hs << 4);
            const uint32_t wd = __shfl_sync(FULL, wid, hs << 4);
            const unsigned lanebit = 1u << lane;
            const unsigned above = ~((lanebit << 1) - 1u);
            auto bumpr = [&](int i, uint32_t v) { if (lane == 0) RC[i] += v; };
            Row<P> row;
            row.u = S[0][lane]; row.v = S[1][lane]; row.w = S[2][lane];
            __syncwarp();
            auto remove_row = [&](int hh, int &wl0, int &wl1, int &nwl) {
                const int last = rr - 1;
                int n2 = 0, x0 = 0, x1 = 0;
                if (nwl >= 1 && wl0 != hh) { x0 = wl0; n2 = 1; }
                if (nwl >= 2 && wl1 != hh) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
                wl0 = x0; wl1 = x1; nwl = n2;
                if (hh != last) {
                    const Row<P> mv = shfl_row<P>(row, last);
                    if (lane == hh) row = mv;
                    if (nwl >= 1 && wl0 == last) wl0 = hh;
                    if (nwl >= 2 && wl1 == last) wl1 = hh;
                }
                rr--;
            };
            if (which == 0) {
                // R12: exact worklist reduction after a flip touching rows ta, tb
                int wl0 = ta, wl1 = tb, nwl = 2;
                while (nwl > 0) {
                    const int t = wl0;
                    wl0 = wl1;
                    nwl--;
                    if (t >= rr) continue;
                    const Row<P> rt = shfl_row<P>(row, t);
                    if (has_zero(rt)) {
                        remove_row(t, wl0, wl1, nwl);
                        bumpr(RC_ZERO, 1);
                        continue;
                    }
                    Row<P> merged = row;
                    const bool red = lane < rr && lane != t && reducible<P>(rt, row, merged);
                    const unsigned bal = __ballot_sync(FULL, red);
                    if (!bal) continue;
                    const int j = __ffs(bal) - 1;
                    const int lo = t < j ? t : j, hi = t < j ? j : t;
                    const Row<P> mg = shfl_row<P>(merged, j);
                    if (lane == lo) row = mg;
                    bumpr(RC_MERGE, 1);
                    remove_row(hi, wl0, wl1, nwl);
                    if (has_zero(mg)) {
                        remove_row(lo, wl0, wl1, nwl);
                        bumpr(RC_ZERO, 1);
                    } else {
                        wl1 = wl0;
                        wl0 = lo;
                        nwl++;
                    }
                }
            } else if (which == 1) {
                // R15: reduce_all, exact lexicographic
                for (;;) {
                    const unsigned bz = __ballot_sync(FULL, lane < rr && has_zero(row));
                    if (bz) {
                        int n0 = 0, x0 = 0, x1 = 0;
                        remove_row(__ffs(bz) - 1, x0, x1, n0);
                        bumpr(RC_ZERO, 1);
                        continue;
                    }
                    const unsigned act_ = rr >= 32 ? FULL : ((1u << rr) - 1u);
                    const unsigned mu = P::match(row.u) & act_, mv = P::match(row.v) & act_;
                    const unsigned mw = P::match(P::abs(row.w)) & act_;
                    const unsigned two = ((mu & mv) | (mu & mw) | (mv & mw)) & above;
                    unsigned cand = __ballot_sync(FULL, lane < rr && two != 0);
                    bool merged_any = false;
                    while (cand) {
                        const int i = __ffs(cand) - 1;
                        cand &= cand - 1;
                        const Row<P> ri = shfl_row<P>(row, i);
                        Row<P> merged = row;
                        const bool red = lane < rr && lane > i && reducible<P>(ri, row, merged);
                        const unsigned bal = __ballot_sync(FULL, red);
                        if (!bal) continue;
                        const int j = __ffs(bal) - 1;
                        const Row<P> mg = shfl_row<P>(merged, j);
                        if (lane == i) row = mg;
                        bumpr(RC_MERGE, 1);
                        int n0 = 0, x0 = 0, x1 = 0;
                        remove_row(j, x0, x1, n0);
                        if (has_zero(mg)) {
                            remove_row(i, x0, x1, n0);
                            bumpr(RC_ZERO, 1);
                        }
                        merged_any = true;
                        break;
                    }
                    if (!merged_any) break;
                }
            } else {
                // R16 expand (plus / split), words from Philox block 1 of this step
                bool done = false;
                if (rr >= 2 && rr + 1 <= R) {
                    uint32_t b0, b1, b2, b3;
                    philox_block(seed, stp, wd, 1u, b0, b1, b2, b3);
                    const bool plus = b0 < 0x80000000u;
                    const int i = (int)__umulhi(b1, (uint32_t)rr);
                    int j = (int)__umulhi(b2, (uint32_t)(rr - 1));
                    j += (j >= i);
                    const int perm = (int)__umulhi(b3, 6u);
                    const int A = perm >> 1;
                    const int B = (1161 >> (2 * perm)) & 3;
                    const int Cr = 3 - A - B;
                    const Row<P> ri = shfl_row<P>(row, i), rj = shfl_row<P>(row, j);
                    const F ai = get(ri, A), aj = get(rj, A), bi = get(ri, B), bj = get(rj, B);
                    const F ci = get(ri, Cr), cj = get(rj, Cr);
                    bool ok = true;
                    if (plus) {
                        if (distinct<P>(ai, aj) && distinct<P>(bi, bj) && distinct<P>(ci, cj)) {
                            const F t1 = P::add(bi, bj, ok);
                            const F t2 = P::sub(cj, ci, ok);
                            const F t3 = P::sub(aj, ai, ok);
                            if (ok) {
                                set(row, B, t1, lane == i);
                                set(row, A, ai, lane == j);
                                set(row, Cr, t2, lane == j);
                                set(row, A, t3, lane == rr);
                                set(row, B, bj, lane == rr);
                                set(row, Cr, cj, lane == rr);
                                done = true;
                            }
                        }
                    } else if (distinct<P>(ai, aj)) {
                        const F t3 = P::sub(ai, aj, ok);
                        if (ok) {
                            set(row, A, aj, lane == i);
                            set(row, A, t3, lane == rr);
                            set(row, B, bi, lane == rr);
                            set(row, Cr, ci, lane == rr);
                            done = true;
                        }
                    }
                    if (done) {
                        if (lane == i || lane == j || lane == rr) normalize<P>(row);
                        rr++;
                        ei = i;
                        ej = j;
                    }
                }
                bumpr(done ? RC_EOK : RC_EREJ, 1);
            }
            __syncwarp();
            S[0][lane] = row.u; S[1][lane] = row.v; S[2][lane] = row.w;
            __syncwarp();
            return rr;
        };
        // incremental class masks after row t of half hs changed (all lanes call;
        // lanes of half hs apply): bit t of every live row's masks, full masks of t
        auto upd_row = [&](int hs, int t) {
            const bool mine = h == hs;
            const bool l0 = k < r, l1 = 16 + k < r;
            const F tu = sR[0][t], tv = sR[1][t], ta = P::abs(sR[2][t]);
            const bool u0 = l0 && P::eq(row0.u, tu), v0 = l0 && P::eq(row0.v, tv), w0 = l0 && P::eq(wA0, ta);
            const bool u1 = l1 && P::eq(row1.u, tu), v1 = l1 && P::eq(row1.v, tv), w1 = l1 && P::eq(wA1, ta);
            const unsigned MU = __byte_perm(__ballot_sync(FULL, u0), __ballot_sync(FULL, u1), prm);
            const unsigned MV = __byte_perm(__ballot_sync(FULL, v0), __ballot_sync(FULL, v1), prm);
            const unsigned MW = __byte_perm(__ballot_sync(FULL, w0), __ballot_sync(FULL, w1), prm);
            if (mine) {
                const unsigned bt = 1u << t;
                mU0 = (mU0 & ~bt) | (u0 ? bt : 0u); mV0 = (mV0 & ~bt) | (v0 ? bt : 0u); mW0 = (mW0 & ~bt) | (w0 ? bt : 0u);
                mU1 = (mU1 & ~bt) | (u1 ? bt : 0u); mV1 = (mV1 & ~bt) | (v1 ? bt : 0u); mW1 = (mW1 & ~bt) | (w1 ? bt : 0u);
                if (k == (t & 15)) {
                    if (t >> 4) { mU1 = MU; mV1 = MV; mW1 = MW; }
                    else { mU0 = MU; mV0 = MV; mW0 = MW; }
                }
            }
        };
        // this half reloads its rows from its mirror and rebuilds its masks
        auto reload = [&]() {
            row0.u = sR[0][k]; row0.v = sR[1][k]; row0.w = sR[2][k];
            row1.u = sR[0][16 + k]; row1.v = sR[1][16 + k]; row1.w = sR[2][16 + k];
            full_masks();
        };
        auto store_rows = [&](uint64_t *dst) {
            if (k < R) {
                const bool lv = k < r;
                dst[0 * R + k] = lv ? P::dig(row0.u) : 0; dst[1 * R + k] = lv ? P::sgn(row0.u) : 0;
                dst[2 * R + k] = lv ? P::dig(row0.v) : 0; dst[3 * R + k] = lv ? P::sgn(row0.v) : 0;
                dst[4 * R + k] = lv ? P::dig(row0.w) : 0; dst[5 * R + k] = lv ? P::sgn(row0.w) : 0;
            }
            if (16 + k < R) {
                const int l = 16 + k;
                const bool lv = l < r;
                dst[0 * R + l] = lv ? P::dig(row1.u) : 0; dst[1 * R + l] = lv ? P::sgn(row1.u) : 0;
                dst[2 * R + l] = lv ? P::dig(row1.v) : 0; dst[3 * R + l] = lv ? P::sgn(row1.v) : 0;
                dst[4 * R + l] = lv ? P::dig(row1.w) : 0; dst[5 * R + l] = lv ? P::sgn(row1.w) : 0;
            }
        };

        full_masks();
        __syncwarp();
        int boff = 32;
        const uint32_t nsteps = (uint32_t)a.steps;      // both halves step in lockstep

        for (uint32_t it = 0; it < nsteps; ++it, ++step, ++boff) {
            if (boff == 32) {
                // lane k of the half: Philox blocks 0 and 2 of steps 2k, 2k+1 of the batch
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int st = 2 * k + q;
                    uint32_t o0, o1, o2, o3;
                    philox_block(seed, step + st, wid, 0u, o0, o1, o2, o3);
                    px[st * PXS + 0] = o0;
                    px[st * PXS + 1] = (o1 < a.thr_eq ? 1u : 0u) | (o2 < a.thr_reduce ? 2u : 0u) |
                                       (o3 < a.thr_expand ? 4u : 0u);
                    philox_block(seed, step + st, wid, 2u, o0, o1, o2, o3);
                    px[st * PXS + 4] = o0; px[st * PXS + 5] = o1;
                    px[st * PXS + 6] = o2; px[st * PXS + 7] = o3;
                }
                __syncwarp();
                boff = 0;
            }
            const uint32_t *pw = px + boff * PXS;
            const uint32_t bern = pw[1];
            uint32_t flags = 0;
            int alpha = 0, beta = 0;

            // ---- R10: counts of rows k, 16+k; row-order prefix (16-lane scan of both slots) ----
            const bool live0 = k < r, live1 = 16 + k < r;
            const unsigned c0 = live0 ? ((unsigned)__popc(mU0 & ab0) | ((unsigned)__popc(mV0 & ab0) << 10) |
                                         ((unsigned)__popc(mW0 & ab0) << 20)) : 0u;
            const unsigned c1 = live1 ? ((unsigned)__popc(mU1 & ab1) | ((unsigned)__popc(mV1 & ab1) << 10) |
                                         ((unsigned)__popc(mW1 & ab1) << 20)) : 0u;
            uint64_t sc = (uint64_t)c0 | ((uint64_t)c1 << 32);
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const uint64_t t = __shfl_up_sync(FULL, sc, o, 16);
                if (k >= o) sc += t;
            }
            const unsigned tot0 = __shfl_sync(FULL, (unsigned)sc, 15, 16);
            const unsigned pre1 = tot0 + (unsigned)(sc >> 32);
            sP[k] = (unsigned)sc;
            sP[16 + k] = pre1;
            const unsigned tot = __shfl_sync(FULL, pre1, 15, 16);
            const unsigned nU = tot & 1023u, nV = (tot >> 10) & 1023u, nW = tot >> 20;
            const unsigned nC = act ? nU + nV + nW : 0u;
            __syncwarp();

            // ---- R11: draw evaluation, lane k = draw (base + k) of this half's walker ----
            auto eval = [&](uint32_t x, Ev<P> &E) -> bool {
                const uint32_t kk = __umulhi(x, 4u * nC);
                const uint32_t idx = kk >> 2;
                const int d = kk & 1, e = (kk >> 1) & 1;
                const uint32_t g1 = idx >= nU, g2 = idx >= nU + nV;
                const int X = (int)(g1 + g2);
                const uint32_t qq = idx - (g1 ? nU : 0u) - (g2 ? nV : 0u);
                const int sh = 10 * X;
                const unsigned fm = 1023u << sh, qs = qq << sh;
                int i = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) i |= ((sP[i | (st - 1)] & fm) <= qs) ? st : 0;
                const unsigned ex = i ? ((sP[(i - 1) & 31] >> sh) & 1023u) : 0u;
                const unsigned mm = sM[X][i] & ~((2u << i) - 1u);
                const int j = nth_bit16(mm, qq - ex);
                if ((a.dbg & 32u) && (j < 0 || j > 31) && k < 5 && nC > 0) {
                    if (atomicCAS(a.dbgbuf, 0u, 1u) == 0u) {
                        a.dbgbuf[1] = i; a.dbgbuf[2] = qq; a.dbgbuf[3] = ex; a.dbgbuf[4] = mm;
                        a.dbgbuf[5] = X; a.dbgbuf[6] = nC; a.dbgbuf[7] = sP[i]; a.dbgbuf[8] = lane;
                        a.dbgbuf[9] = (uint32_t)step;
                    }
                }
                const int al = d ? j : i, be = d ? i : j;
                const unsigned yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
                const int Y = yz & 3, Z = yz >> 2;
                const F ya = sR[Y][al], yb = sR[Y][be], za = sR[Z][al], zb = sR[Z][be];
                const bool sneg = P::RING == FG_ZT && X == 2 && !P::eq(sR[2][al], sR[2][be]);
                bool v = true;
                E.ny = P::add(ya, P::sel(sneg, P::neg(yb), yb), v);
                E.nz = P::sub(zb, za, v);
                E.info = al | (be << 8) | (Y << 16) | (Z << 18);
                return v;
            };
            Ev<P> E;
            const uint32_t na = kf < 5 ? kf : 5u;
            const uint32_t xa = pw[k == 0 ? 0 : (k < 5 ? 3 + k : 0)];
            unsigned wh = (__ballot_sync(FULL, eval(xa, E) && (uint32_t)k < na && nC > 0) >> hb) & 0xffffu;
            int base = 0;
            const bool needB = !(a.dbg & 16u) && wh == 0 && nC > 0 && kf > 5;
            if (__any_sync(FULL, needB)) {
                // draws 5..15 of this step: slots 12..22 = Philox blocks 3,4,5
                uint32_t o0, o1, o2, o3;
                philox_block(seed, step, wid, 3u + (k < 3 ? k : 0), o0, o1, o2, o3);
                const int att = 5 + k;
                const int src = hb + (((att + 7 - 12) >> 2) & 3), w = (att + 7) & 3;
                const uint32_t w0 = __shfl_sync(FULL, o0, src), w1 = __shfl_sync(FULL, o1, src);
                const uint32_t w2 = __shfl_sync(FULL, o2, src), w3 = __shfl_sync(FULL, o3, src);
                const uint32_t xb = w == 0 ? w0 : (w == 1 ? w1 : (w == 2 ? w2 : w3));
                Ev<P> EB;
                const unsigned whb = (__ballot_sync(FULL, eval(xb, EB) && att < (int)kf && nC > 0) >> hb) & 0xffffu;
                if (needB) { wh = whb; base = 5; E = EB; }
            }
            const bool okh = wh != 0;
            const int draws = okh ? base + __ffs(wh) : (nC ? (int)kf : 0);
            c_draws += draws;

            // ---- commit the winning draw (all lanes; predicated per half) ----
            const int src = hb + (okh ? __ffs(wh) - 1 : 0);
            const int info = __shfl_sync(FULL, E.info, src);
            const F ny = P::shfl(E.ny, src);
            const F nz = P::shfl(E.nz, src);
            if (okh) { alpha = info & 255; beta = (info >> 8) & 255; }
            const int Y = (info >> 16) & 3, Z = (info >> 18) & 3;
            const bool pa0 = okh && k == (alpha & 15) && (alpha >> 4) == 0;
            const bool pa1 = okh && k == (alpha & 15) && (alpha >> 4) == 1;
            const bool pb0 = okh && k == (beta & 15) && (beta >> 4) == 0;
            const bool pb1 = okh && k == (beta & 15) && (beta >> 4) == 1;
            set(row0, Y, ny, pa0);
            set(row0, Z, nz, pb0);
            set(row1, Y, ny, pa1);
            set(row1, Z, nz, pb1);
            if (pa0 || pb0) {
                normalize<P>(row0);
                wA0 = P::abs(row0.w);
                sR[0][k] = row0.u; sR[1][k] = row0.v; sR[2][k] = row0.w;
            }
            if (pa1 || pb1) {
                normalize<P>(row1);
                wA1 = P::abs(row1.w);
                sR[0][16 + k] = row1.u; sR[1][16 + k] = row1.v; sR[2][16 + k] = row1.w;
            }
            __syncwarp();
            // ---- incremental class masks for rows alpha, beta ----
            {
                const F au = sR[0][alpha], av = sR[1][alpha], aw = P::abs(sR[2][alpha]);
                const F bu = sR[0][beta], bv = sR[1][beta], bwk = P::abs(sR[2][beta]);
                const bool ua0 = live0 && P::eq(row0.u, au), ub0 = live0 && P::eq(row0.u, bu);
                const bool va0 = live0 && P::eq(row0.v, av), vb0 = live0 && P::eq(row0.v, bv);
                const bool wa0 = live0 && P::eq(wA0, aw), wb0 = live0 && P::eq(wA0, bwk);
                const bool ua1 = live1 && P::eq(row1.u, au), ub1 = live1 && P::eq(row1.u, bu);
                const bool va1 = live1 && P::eq(row1.v, av), vb1 = live1 && P::eq(row1.v, bv);
                const bool wa1 = live1 && P::eq(wA1, aw), wb1 = live1 && P::eq(wA1, bwk);
                const unsigned MUa = __byte_perm(__ballot_sync(FULL, ua0), __ballot_sync(FULL, ua1), prm);
                const unsigned MUb = __byte_perm(__ballot_sync(FULL, ub0), __ballot_sync(FULL, ub1), prm);
                const unsigned MVa = __byte_perm(__ballot_sync(FULL, va0), __ballot_sync(FULL, va1), prm);
                const unsigned MVb = __byte_perm(__ballot_sync(FULL, vb0), __ballot_sync(FULL, vb1), prm);
                const unsigned MWa = __byte_perm(__ballot_sync(FULL, wa0), __ballot_sync(FULL, wa1), prm);
                const unsigned MWb = __byte_perm(__ballot_sync(FULL, wb0), __ballot_sync(FULL, wb1), prm);
                if (okh) {
                    const unsigned keep = ~((1u << alpha) | (1u << beta));
                    const unsigned ba = 1u << alpha, bb = 1u << beta;
                    mU0 = (mU0 & keep) | (ua0 ? ba : 0u) | (ub0 ? bb : 0u);
                    mV0 = (mV0 & keep) | (va0 ? ba : 0u) | (vb0 ? bb : 0u);
                    mW0 = (mW0 & keep) | (wa0 ? ba : 0u) | (wb0 ? bb : 0u);
                    mU1 = (mU1 & keep) | (ua1 ? ba : 0u) | (ub1 ? bb : 0u);
                    mV1 = (mV1 & keep) | (va1 ? ba : 0u) | (vb1 ? bb : 0u);
                    mW1 = (mW1 & keep) | (wa1 ? ba : 0u) | (wb1 ? bb : 0u);
                }
                if (pa0) { mU0 = MUa; mV0 = MVa; mW0 = MWa; }
                if (pb0) { mU0 = MUb; mV0 = MVb; mW0 = MWb; }
                if (pa1) { mU1 = MUa; mV1 = MVa; mW1 = MWa; }
                if (pb1) { mU1 = MUb; mV1 = MVb; mW1 = MWb; }
                store_masks();
            }
            c_flips += okh;
            flags |= okh ? 1u : 0u;
            // ---- R12 local reduction (exact skip) ----
            {
                const unsigned two0 = ((mU0 & mV0) | (mU0 & mW0) | (mV0 & mW0)) & ~(1u << k);
                const unsigned two1 = ((mU1 & mV1) | (mU1 & mW1) | (mV1 & mW1)) & ~(1u << (16 + k));
                const bool cnd = ((pa0 || pb0) && (has_zero(row0) || two0 != 0)) ||
                                 ((pa1 || pb1) && (has_zero(row1) || two1 != 0));
                const bool needL = (__ballot_sync(FULL, cnd) & hm) != 0;
                const unsigned nl = (a.dbg & 1u) ? 0u : __ballot_sync(FULL, needL);
                if (nl) {
#pragma unroll 1
                    for (int hs = 0; hs < 2; ++hs) {
                        if (!(nl & (1u << (hs << 4)))) continue;
                        const int ta = __shfl_sync(FULL, alpha, hs << 4), tb = __shfl_sync(FULL, beta, hs << 4);
                        int e0, e1;
                        const int nr = rare(hs, 0, ta, tb, e0, e1);
                        if (h == hs) { r = nr; reload(); }
                        __syncwarp();
                    }
                }
            }
            // ---- PAPER:310-313 acceptance ----
            {
                const bool acc = !(a.dbg & 8u) && okh && (r < best || (r == best && (bern & 1u)));
                if (__any_sync(FULL, acc)) {
                    const bool strict = acc && r < best;
                    unsigned slot = 0;
                    if (k == 0 && strict) slot = atomicAdd(a.q_count, 1u);
                    slot = __shfl_sync(FULL, slot, hb);
                    int nz = 0;
                    if (acc) {
                        nz = (k < r ? P::popd(row0.u) + P::popd(row0.v) + P::popd(row0.w) : 0) +
                             (16 + k < r ? P::popd(row1.u) + P::popd(row1.v) + P::popd(row1.w) : 0);
                    }
#pragma unroll
                    for (int o = 8; o >= 1; o >>= 1) nz += __shfl_xor_sync(FULL, nz, o, 16);
                    if (acc) {
                        best = r;
                        best_adds = nz - 2 * r - a.mp;
                        bump(RC_COPY, 1);
                        flags |= 4u;
                        store_rows(bw);
                        if (strict) {
                            flags |= 8u;
                            bump(RC_IMPR, 1);
                            if (slot < a.q_cap) {
                                store_rows(a.q_planes + (size_t)slot * FG_PLANES * R);
                                if (k == 0) {
                                    fg_qmeta qm;
                                    qm.walker = wk; qm.step = step; qm.rank = r; qm.ok = -1;
                                    qm.ff[0] = qm.ff[1] = qm.ff[2] = -1; qm.pad = 0;
                                    a.q_meta[slot] = qm;
                                }
                            } else if (k == 0) {
                                atomicAdd(a.q_overflow, 1u);
                                hp->pad |= 1;
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            // ---- PAPER:315-317 reduce (R15) ----
            {
                const bool red = okh && (bern & 2u);
                c_red += red;
                flags |= red ? 16u : 0u;
                const unsigned two0 = ((mU0 & mV0) | (mU0 & mW0) | (mV0 & mW0)) & ~(1u << k);
                const unsigned two1 = ((mU1 & mV1) | (mU1 & mW1) | (mV1 & mW1)) & ~(1u << (16 + k));
                const bool cnd = (two0 | two1) != 0;   // dead rows have empty masks; R12 left no zero factor
                const unsigned bR = __ballot_sync(FULL, cnd);        // every lane votes (no short circuit)
                const bool needR = red && (bR & hm) != 0;
                const unsigned nrm = (a.dbg & 2u) ? 0u : __ballot_sync(FULL, needR);
                if (nrm) {
#pragma unroll 1
                    for (int hs = 0; hs < 2; ++hs) {
                        if (!(nrm & (1u << (hs << 4)))) continue;
                        int e0, e1;
                        const int nr = rare(hs, 1, 0, 0, e0, e1);
                        if (h == hs) { r = nr; reload(); }
                        __syncwarp();
                    }
                }
            }
            // ---- expand: PAPER:305-307 fallback, or PAPER:319-321 with p_expand ----
            {
                const bool fb = act && !okh;
                const bool pe = okh && (bern & 4u) && r <= best + a.slack;
                const unsigned nx = (a.dbg & 4u) ? 0u : __ballot_sync(FULL, fb || pe);
                if (nx) {
#pragma unroll 1
                    for (int hs = 0; hs < 2; ++hs) {
                        if (!(nx & (1u << (hs << 4)))) continue;
                        int ei = 0, ej = 0;
                        const int rold = __shfl_sync(FULL, r, hs << 4);
                        const int nr = rare(hs, 2, 0, 0, ei, ej);
                        const bool ex = nr != rold;
                        if (h == hs) {
                            flags |= (fb ? 2u : 32u) | (ex ? 64u : 0u);
                            if (ex) {
                                r = nr;
                                row0.u = sR[0][k]; row0.v = sR[1][k]; row0.w = sR[2][k];
                                row1.u = sR[0][16 + k]; row1.v = sR[1][16 + k]; row1.w = sR[2][16 + k];
                                wA0 = P::abs(row0.w);
                                wA1 = P::abs(row1.w);
                            }
                        }
                        if (ex) {
                            // incremental masks for the two changed rows and the new row
                            upd_row(hs, ei);
                            upd_row(hs, ej);
                            upd_row(hs, rold);
                            if (h == hs) store_masks();
                        }
                        __syncwarp();
                    }
                }
            }
            const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)best << 10) |
                                ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) |
                                ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
            digest = (digest ^ ev) * 0x100000001b3ULL;
            digest ^= digest >> 32;
        }

        // ---------------- store both walkers ----------------
        if (act) store_rows(a.cur + (size_t)wk * FG_PLANES * R);
        int nnz = 0;
        if (act && k < best) nnz += __popcll(bw[0 * R + k]) + __popcll(bw[2 * R + k]) + __popcll(bw[4 * R + k]);
        if (act && 16 + k < best)
            nnz += __popcll(bw[0 * R + 16 + k]) + __popcll(bw[2 * R + 16 + k]) + __popcll(bw[4 * R + 16 + k]);
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) nnz += __shfl_xor_sync(FULL, nnz, o, 16);
        __syncwarp();
        if (act && k == 0) {
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
            int adds = nnz - 2 * best - a.mp;
            if (adds < 0) adds = 0;
            atomicMin(a.best_key, ((unsigned long long)best << 54) | ((unsigned long long)adds << 36) |
                                      (unsigned long long)wk);
        }
        __syncwarp();
    }
}

template <class P>
cudaError_t launch_h16(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_h16<P>, H16_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    int64_t blocks = (int64_t)num_sms * bps;
    const int64_t need = (a.num_walkers + 2 * H16_WARPS - 1) / (2 * H16_WARPS);
    if (blocks > need) blocks = need;
    walk_h16<P><<<(unsigned)blocks, H16_THREADS, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t fg_launch_walk_h16(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_H16_P16: return launch_h16<P16>(a, num_sms, st);
    case FG_K_H16_P32: return launch_h16<P32>(a, num_sms, st);
    case FG_K_H16_Z2: return launch_h16<PZ2>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
