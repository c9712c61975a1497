// fg_walk.cu -- the RandomWalk kernel (Algorithm 1) for walkers
// with at most 32 rows: ONE WALKER PER WARP, row l of the scheme in lane l's
// registers, every step's control flow warp-uniform and (on the hot path)
// branch-free.
//
// Per step (reading R17):
//   - Philox words (R8): lane L computes blocks 0 and 2 of step s0+L once per 32
//     steps into a per-warp shared-memory table; a step reads its words with LDS.
//   - flip candidates (R10): each lane keeps the masks of rows equal to its u, its
//     v and its w up to sign (mU, mV, mWp); |C| and the prefix over (role, i) come
//     from popc + one packed warp scan.
//   - try_flip (R11): the first five draws are evaluated LANE-PARALLEL (lane a =
//     draw a: binary search of the prefix, nth-set-bit for j, row fetch by SHFL,
//     LOP3 ternary add/sub with validity); a ballot picks the first valid draw,
//     exactly the draw the sequential loop would commit.  Draws 5..15 (rare) run
//     the same way from on-demand Philox blocks 3-5.
//   - the masks are then updated for the two touched rows only (SHFL + compare +
//     ballot); MATCH.ANY (10x the cost of SHFL on sm_100, tools/microbench) is
//     used only after the rare structural changes (merges, removals, expand).
//   - local reduction check (R12), acceptance, reduce_all (R15,
//     exact skip through the masks), expand (R16).
// Independent of oracle/; parity is checked by tests/test_gpu_parity.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "fg_device.cuh"

using namespace fgd;

#define W32_THREADS 128
#define W32_WARPS (W32_THREADS / 32)
#define PXS 9                        // words per step in the Philox table (8 + 1 pad)
#ifndef W32_MINB
#define W32_MINB 8
#endif

namespace {

// position of the t-th (0-based) set bit of x; x has more than t set bits.  t is
// almost always 0..2 (flip classes are small), so three predicated clears and a
// find-first cover it; larger t takes a short loop.
__device__ __forceinline__ int nth_bit(uint32_t x, uint32_t t)
{
    x = t > 0 ? (x & (x - 1u)) : x;
    x = t > 1 ? (x & (x - 1u)) : x;
    x = t > 2 ? (x & (x - 1u)) : x;
    for (uint32_t k = 3; k < t; ++k) x &= x - 1u;
    return __ffs(x) - 1;
}

template <class P, bool CM>
__global__ void __launch_bounds__(W32_THREADS, W32_MINB) walk_w32(WalkArgs a)
{
    typedef typename P::F F;
    __shared__ uint32_t px_all[W32_WARPS][32 * PXS];
    __shared__ uint32_t rc_all[W32_WARPS][8];     // rare counters (lane 0 updates)
    uint32_t *px = px_all[threadIdx.x >> 5];
    uint32_t *rc = rc_all[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned lanebit = 1u << lane;
    const unsigned above = ~((lanebit << 1) - 1u);          // lanes > this one
    const int R = a.R;
    const uint64_t seed = a.seed;
    const uint32_t kf = a.k_flip;

    // dynamic walker queue: warps that finish early take more walkers
    auto grab = [&]() -> int64_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(a.work_counter, 1ull);
        return (int64_t)__shfl_sync(FULL, v, 0);
    };
    for (int64_t wk = grab(); wk < a.num_walkers; wk = grab()) {
        // ---------------- load walker (coalesced: plane q of rows 0..31) ----------------
        const uint64_t *cp = a.cur + (size_t)wk * FG_PLANES * R;
        uint64_t *bw = a.best + (size_t)wk * FG_PLANES * R;
        Row<P> row;
        row.u = row.v = row.w = P::make(0, 0);
        if (lane < R) {
            row.u = P::make(cp[0 * R + lane], cp[1 * R + lane]);
            row.v = P::make(cp[2 * R + lane], cp[3 * R + lane]);
            row.w = P::make(cp[4 * R + lane], cp[5 * R + lane]);
        }
        fg_whdr *hp = a.hdr + wk;
        int r = hp->r;
        int best = hp->best_r;
        uint64_t step = hp->step;
        uint64_t digest = hp->digest;
        int best_adds = hp->best_adds;
        const uint32_t wid = (uint32_t)(a.id_base + wk);
        constexpr bool cmode = CM;               // R24: naive-complexity minimisation
        // nnz of the current scheme (additions = nnz - 2r - mp), tracked in R24 mode
        int nnz_cur = CM ? __reduce_add_sync(FULL, lane < r ? P::popd(row.u) + P::popd(row.v) + P::popd(row.w) : 0) : 0;

        uint32_t c_draws = 0, c_flips = 0, c_red = 0;
        if (lane < 8) rc[lane] = 0;
        __syncwarp();
        enum { RC_EOK = 0, RC_EREJ, RC_MERGE, RC_ZERO, RC_COPY, RC_IMPR };
        auto bump = [&](int k, uint32_t v) { if (lane == 0) rc[k] += v; };

        // masks of live lanes holding the same u / v / w-up-to-sign as this lane
        unsigned mU = 0, mV = 0, mWp = 0;
        F wA = P::abs(row.w);                 // this lane's w up to sign (cached)
        auto compute_masks = [&]() {
            const unsigned act = r >= 32 ? FULL : ((1u << r) - 1u);
            wA = P::abs(row.w);
            mU = P::match(row.u) & act;
            mV = P::match(row.v) & act;
            mWp = P::match(wA) & act;
        };
        // incremental update after rows ta != tb changed (all other rows unchanged)
        auto update_masks2 = [&](int ta, int tb) {
            if (lane == ta || lane == tb) wA = P::abs(row.w);
            const F ua_ = P::shfl(row.u, ta), ub_ = P::shfl(row.u, tb);
            const F va_ = P::shfl(row.v, ta), vb_ = P::shfl(row.v, tb);
            const F wa_k = P::shfl(wA, ta), wb_k = P::shfl(wA, tb);
            const bool live = lane < r;
            const bool ua = live && P::eq(row.u, ua_), ub = live && P::eq(row.u, ub_);
            const bool va = live && P::eq(row.v, va_), vb = live && P::eq(row.v, vb_);
            const bool wa_ = live && P::eq(wA, wa_k), wb_ = live && P::eq(wA, wb_k);
            const unsigned keep = ~((1u << ta) | (1u << tb));
            mU = (mU & keep) | ((unsigned)ua << ta) | ((unsigned)ub << tb);
            mV = (mV & keep) | ((unsigned)va << ta) | ((unsigned)vb << tb);
            mWp = (mWp & keep) | ((unsigned)wa_ << ta) | ((unsigned)wb_ << tb);
            const unsigned bua = __ballot_sync(FULL, ua), bub = __ballot_sync(FULL, ub);
            const unsigned bva = __ballot_sync(FULL, va), bvb = __ballot_sync(FULL, vb);
            const unsigned bwa = __ballot_sync(FULL, wa_), bwb = __ballot_sync(FULL, wb_);
            if (lane == ta) { mU = bua; mV = bva; mWp = bwa; }
            if (lane == tb) { mU = bub; mV = bvb; mWp = bwb; }
        };

        // R14 remove(h) with the 2-entry worklist (entries == h dropped, r-1 -> h)
        auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) {
            const int last = r - 1;
            int n2 = 0, x0 = 0, x1 = 0;
            if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
            if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
            wl0 = x0; wl1 = x1; nwl = n2;
            if (h != last) {
                const Row<P> mv = shfl_row<P>(row, last);
                if (lane == h) row = mv;
                if (nwl >= 1 && wl0 == last) wl0 = h;
                if (nwl >= 2 && wl1 == last) wl1 = h;
            }
            r--;
        };

        // R12: exact worklist reduction after a flip touching rows a0, b0
        auto slow_local_reduce = [&](int a0, int b0) {
            int wl0 = a0, wl1 = b0, nwl = 2;
            while (nwl > 0) {
                const int t = wl0;
                wl0 = wl1;
                nwl--;
                if (t >= r) continue;
                const Row<P> rt = shfl_row<P>(row, t);
                if (has_zero(rt)) {
                    remove_row(t, wl0, wl1, nwl);
                    bump(RC_ZERO, 1);
                    continue;
                }
                Row<P> merged = row;
                const bool red = lane < r && lane != t && reducible<P>(rt, row, merged);
                const unsigned bal = __ballot_sync(FULL, red);
                if (!bal) continue;
                const int j = __ffs(bal) - 1;
                const int lo = t < j ? t : j, hi = t < j ? j : t;
                const Row<P> mg = shfl_row<P>(merged, j);
                if (lane == lo) row = mg;
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

        // R15: reduce_all, exact
        auto slow_reduce_all = [&]() {
            for (;;) {
                const unsigned bz = __ballot_sync(FULL, lane < r && has_zero(row));
                if (bz) {
                    int n0 = 0, x0 = 0, x1 = 0;
                    remove_row(__ffs(bz) - 1, x0, x1, n0);
                    bump(RC_ZERO, 1);
                    continue;
                }
                compute_masks();
                const unsigned two = ((mU & mV) | (mU & mWp) | (mV & mWp)) & above;
                unsigned cand = __ballot_sync(FULL, lane < r && two != 0);
                bool merged_any = false;
                while (cand) {
                    const int i = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const Row<P> ri = shfl_row<P>(row, i);
                    Row<P> merged = row;
                    const bool red = lane < r && lane > i && reducible<P>(ri, row, merged);
                    const unsigned bal = __ballot_sync(FULL, red);
                    if (!bal) continue;
                    const int j = __ffs(bal) - 1;
                    const Row<P> mg = shfl_row<P>(merged, j);
                    if (lane == i) row = mg;
                    bump(RC_MERGE, 1);
                    int n0 = 0, x0 = 0, x1 = 0;
                    remove_row(j, x0, x1, n0);
                    if (has_zero(mg)) {
                        remove_row(i, x0, x1, n0);
                        bump(RC_ZERO, 1);
                    }
                    merged_any = true;
                    break;
                }
                if (!merged_any) break;
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
            const Row<P> ri = shfl_row<P>(row, i);
            const Row<P> rj = shfl_row<P>(row, j);
            const F ai = get(ri, A), aj = get(rj, A), bi = get(ri, B), bj = get(rj, B);
            const F ci = get(ri, Cr), cj = get(rj, Cr);
            bool ok = true;
            if (plus) {
                if (!distinct<P>(ai, aj) || !distinct<P>(bi, bj) ||
                    !distinct<P>(ci, cj))
                    return false;
                const F t1 = P::add(bi, bj, ok);      // v_i + v_j
                const F t2 = P::sub(cj, ci, ok);      // w_j - w_i
                const F t3 = P::sub(aj, ai, ok);      // u_j - u_i
                if (!ok) return false;
                set(row, B, t1, lane == i);
                set(row, A, ai, lane == j);
                set(row, Cr, t2, lane == j);
                set(row, A, t3, lane == r);
                set(row, B, bj, lane == r);
                set(row, Cr, cj, lane == r);
            } else {
                if (!distinct<P>(ai, aj)) return false;
                const F t3 = P::sub(ai, aj, ok);      // u_i - u_j
                if (!ok) return false;
                set(row, A, aj, lane == i);
                set(row, A, t3, lane == r);
                set(row, B, bi, lane == r);
                set(row, Cr, ci, lane == r);
            }
            if (lane == i || lane == j || lane == r) normalize<P>(row);
            r++;
            compute_masks();
            return true;
        };

        // best copy to HBM and the R19 verify queue
        auto store_rows = [&](uint64_t *dst) {
            if (lane < R) {
                const bool lv = lane < r;
                dst[0 * R + lane] = lv ? P::dig(row.u) : 0;
                dst[1 * R + lane] = lv ? P::sgn(row.u) : 0;
                dst[2 * R + lane] = lv ? P::dig(row.v) : 0;
                dst[3 * R + lane] = lv ? P::sgn(row.v) : 0;
                dst[4 * R + lane] = lv ? P::dig(row.w) : 0;
                dst[5 * R + lane] = lv ? P::sgn(row.w) : 0;
            }
        };
        auto store_best = [&]() { store_rows(bw); };
        auto enqueue_verify = [&]() {
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
        };

        compute_masks();
        int boff = 32;

        const uint32_t nsteps = (uint32_t)a.steps;        // host chunks launches below 2^31 steps
        for (uint32_t it = 0; it < nsteps; ++it, ++step, ++boff) {
            if (boff == 32) {
                // lane L: Philox blocks 0 and 2 of step (step + L) -> px[L*9 + 0..7]
                uint32_t o0, o1, o2, o3;
                philox_block(seed, step + lane, wid, 0u, o0, o1, o2, o3);
                // word 0 = draw 0; the three Bernoulli draws of the step pre-decided (R9)
                px[lane * PXS + 0] = o0;
                px[lane * PXS + 1] = (o1 < a.thr_eq ? 1u : 0u) | (o2 < a.thr_reduce ? 2u : 0u) |
                                     (o3 < a.thr_expand ? 4u : 0u);
                philox_block(seed, step + lane, wid, 2u, o0, o1, o2, o3);
                px[lane * PXS + 4] = o0; px[lane * PXS + 5] = o1;
                px[lane * PXS + 6] = o2; px[lane * PXS + 7] = o3;
                __syncwarp();
                boff = 0;
            }
            const uint32_t *pw = px + boff * PXS;     // [draw 0, Bernoulli flags, -, -, draws 1..4]
            const uint32_t bern = pw[1];
            uint32_t flags = 0;
            int alpha = 0, beta = 0, draws = 0;
            bool ok = false;

            // ---- R10 candidate counts + prefix (packed 3 x 10 bits) ----
            const bool live = lane < r;
            const unsigned cnt = live ? ((unsigned)__popc(mU & above) |
                                         ((unsigned)__popc(mV & above) << 10) |
                                         ((unsigned)__popc(mWp & above) << 20))
                                      : 0u;
            unsigned incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned tot = __shfl_sync(FULL, incl, 31);
            const unsigned nU = tot & 1023u, nV = (tot >> 10) & 1023u, nW = tot >> 20;
            const unsigned nC = nU + nV + nW;
            const unsigned excl = incl - cnt;

            // ---- R11 try_flip: draw `att` evaluated by this lane with word x ----
            int e_al = 0, e_be = 0, e_Y = 0, e_Z = 0;
            F e_ny, e_nz;
            auto eval = [&](uint32_t x) -> bool {
                const uint32_t k = __umulhi(x, 4u * nC);
                const uint32_t idx = k >> 2;
                const int d = k & 1, e = (k >> 1) & 1;
                const uint32_t g1 = idx >= nU, g2 = idx >= nU + nV;
                const int X = (int)(g1 + g2);
                const uint32_t qq = idx - (g1 ? nU : 0u) - (g2 ? nV : 0u);
                const int sh = 10 * X;
                const unsigned fm = 1023u << sh, qs = qq << sh;   // compare fields in place
                int i = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const unsigned v = __shfl_sync(FULL, incl, i | (st - 1)) & fm;
                    i |= (v <= qs) ? st : 0;
                }
                const unsigned ex_i = (__shfl_sync(FULL, excl, i) >> sh) & 1023u;
                const unsigned mu_i = __shfl_sync(FULL, mU, i);
                const unsigned mv_i = __shfl_sync(FULL, mV, i);
                const unsigned mw_i = __shfl_sync(FULL, mWp, i);
                const unsigned mm = ((X & 2) ? mw_i : ((X & 1) ? mv_i : mu_i)) & ~((2u << i) - 1u);
                const int j = nth_bit(mm, qq - ex_i);
                const int al = d ? j : i, be = d ? i : j;
                // (Y,Z) = (V,W) / (W,U) / (U,V) for X = U / V / W, swapped if e:
                // nibble 2X+e of 0x148269 holds Y | Z << 2
                const unsigned yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
                const int Y = yz & 3, Z = yz >> 2;
                const Row<P> ra = shfl_row<P>(row, al);
                const Row<P> rb = shfl_row<P>(row, be);
                // sigma = -1 iff the shared factor is W and the two are negatives
                const bool sneg = P::RING == FG_ZT && X == 2 && !P::eq(ra.w, rb.w);
                bool v = true;
                const F yb = get(rb, Y);
                e_ny = P::add(get(ra, Y), P::sel(sneg, P::neg(yb), yb), v);     // y_a + s y_b
                e_nz = P::sub(get(rb, Z), get(ra, Z), v);              // z_b - z_a
                e_al = al; e_be = be; e_Y = Y; e_Z = Z;
                // R24: no reduction edges -> a draw making a factor zero is rejected
                if (cmode) v = v && !P::zero(e_ny) && !P::zero(e_nz);
                return v;
            };

            if (nC) {
                // draws 0..4: lane a evaluates draw a (words: block 0 word 0, block 2 words 0..3)
                const int na = kf < 5 ? (int)kf : 5;
                const uint32_t x = pw[lane == 0 ? 0 : (lane < 5 ? 3 + lane : 0)];
                unsigned win = __ballot_sync(FULL, eval(x) && lane < na);
                int base = 0;
                // draws 5..K-1, 32 per round: lane L evaluates draw base + L (slot 7 + draw,
                // Philox block slot >> 2 computed per lane)
#pragma unroll 1
                for (int b5 = 5; !win && b5 < (int)kf; b5 += 32) {
                    uint32_t o0, o1, o2, o3;
                    const int att = b5 + lane;
                    const uint32_t slot = 7u + (uint32_t)att;
                    philox_block(seed, step, wid, slot >> 2, o0, o1, o2, o3);
                    const uint32_t w = slot & 3u;
                    const uint32_t xb = w == 0 ? o0 : (w == 1 ? o1 : (w == 2 ? o2 : o3));
                    win = __ballot_sync(FULL, eval(xb) && att < (int)kf);
                    base = b5;
                    draws = b5;
                }
                if (win) {
                    const int src = __ffs(win) - 1;
                    draws = base + src + 1;
                    const unsigned info = __shfl_sync(FULL, (unsigned)(e_al | (e_be << 8) | (e_Y << 16) | (e_Z << 18)), src);
                    const F ny = P::shfl(e_ny, src);
                    const F nz = P::shfl(e_nz, src);
                    alpha = info & 255;
                    beta = (info >> 8) & 255;
                    const bool touched = lane == alpha || lane == beta;
                    const int pold = touched ? P::popd(row.u) + P::popd(row.v) + P::popd(row.w) : 0;
                    set(row, (info >> 16) & 3, ny, lane == alpha);
                    set(row, (info >> 18) & 3, nz, lane == beta);
                    if (touched) normalize<P>(row);
                    if (cmode) {
                        const int pnew = touched ? P::popd(row.u) + P::popd(row.v) + P::popd(row.w) : 0;
                        nnz_cur += __reduce_add_sync(FULL, pnew - pold);
                    }
                    ok = true;
                } else {
                    draws = kf;
                }
            }
            c_draws += draws;

            if (cmode) {
                // ---- R24 step: flips only; best by (rank, naive additions) ----
                if (ok) {
                    c_flips++;
                    flags |= 1u;
                    update_masks2(alpha, beta);
                    const int adds = nnz_cur - 2 * r - a.mp;
                    const bool better = r < best || (r == best && adds < best_adds);
                    if (better || (r == best && adds == best_adds && (bern & 1u))) {
                        best = r;
                        best_adds = adds;
                        bump(RC_COPY, 1);
                        flags |= 4u;
                        store_best();
                        if (better) {
                            flags |= 8u;
                            bump(RC_IMPR, 1);
                            enqueue_verify();
                        }
                    }
                }
            } else if (!ok) {
                // expand; continue
                const bool ex = expand();
                bump(RC_EOK, ex);
                bump(RC_EREJ, !ex);
                flags |= 2u | (ex ? 64u : 0u);
            } else {
                c_flips++;
                flags |= 1u;
                update_masks2(alpha, beta);
                // ---- R12 local reduction (exact skip) ----
                {
                    const unsigned two = ((mU & mV) | (mU & mWp) | (mV & mWp)) & ~lanebit;
                    const bool need = (lane == alpha || lane == beta) && (has_zero(row) || two != 0);
                    if (__any_sync(FULL, need)) {
                        slow_local_reduce(alpha, beta);
                        compute_masks();
                    }
                }
                // ---- PAPER:310-313 acceptance ----
                bool acc = r < best;
                if (!acc && r == best) acc = bern & 1u;
                if (acc) {
                    const bool strict = r < best;
                    best = r;
                    best_adds = __reduce_add_sync(FULL, lane < r ? P::popd(row.u) + P::popd(row.v) + P::popd(row.w) : 0) -
                                2 * r - a.mp;
                    bump(RC_COPY, 1);
                    flags |= 4u;
                    store_best();
                    if (strict) {
                        flags |= 8u;
                        bump(RC_IMPR, 1);
                        enqueue_verify();
                    }
                }
                // ---- PAPER:315-317 reduce (R15) ----
                if (bern & 2u) {
                    c_red++;
                    flags |= 16u;
                    const unsigned two = ((mU & mV) | (mU & mWp) | (mV & mWp)) & ~lanebit;
                    if (__any_sync(FULL, lane < r && (has_zero(row) || two != 0))) {
                        slow_reduce_all();
                        compute_masks();
                    }
                }
                // ---- PAPER:319-321 expand ----
                if ((bern & 4u) && r <= best + a.slack) {
                    const bool ex = expand();
                    flags |= 32u | (ex ? 64u : 0u);
                    bump(RC_EOK, ex);
                    bump(RC_EREJ, !ex);
                }
            }
            // ---- digest ----
            const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)(cmode ? (best_adds & 1023) : best) << 10) |
                                ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) |
                                ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
            digest = (digest ^ ev) * 0x100000001b3ULL;
            digest ^= digest >> 32;
            __syncwarp();
        }

        // ---------------- store walker ----------------
        uint64_t *cw = a.cur + (size_t)wk * FG_PLANES * R;
        if (lane < R) {
            cw[0 * R + lane] = P::dig(row.u); cw[1 * R + lane] = P::sgn(row.u);
            cw[2 * R + lane] = P::dig(row.v); cw[3 * R + lane] = P::sgn(row.v);
            cw[4 * R + lane] = P::dig(row.w); cw[5 * R + lane] = P::sgn(row.w);
        }
        // naive additions of the best -> local best key (R20); each lane
        // re-reads the best row it wrote itself
        const int nnz = lane < best ? (__popcll(bw[0 * R + lane]) + __popcll(bw[2 * R + lane]) +
                                       __popcll(bw[4 * R + lane]))
                                    : 0;
        const int tot_nnz = __reduce_add_sync(FULL, nnz);
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
                                           ((unsigned long long)adds << 36) |
                                           (unsigned long long)wk;
            atomicMin(a.best_key, key);
        }
        __syncwarp();
    }
}

template <class P, bool CM>
cudaError_t launch_w32_m(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_w32<P, CM>, W32_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    const int64_t wpb = W32_WARPS;
    // persistent: every resident warp pulls walkers from the queue
    int64_t blocks = (int64_t)num_sms * bps;
    const int64_t need = (a.num_walkers + wpb - 1) / wpb;
    if (blocks > need) blocks = need;
    walk_w32<P, CM><<<(unsigned)blocks, W32_THREADS, 0, st>>>(a);
    return cudaGetLastError();
}

template <class P>
cudaError_t launch_w32(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    return a.mode == 1 ? launch_w32_m<P, true>(a, num_sms, st) : launch_w32_m<P, false>(a, num_sms, st);
}

}  // namespace

// R <= 32: one-word factors (Z_T <= 16 elements, Z_2 <= 32) run one walker per
// quad (fg_walk_q4.cu); Z_T with 17..32 elements runs this file's one walker per
// warp.  33 <= R <= 512: the multi-row kernel (fg_walk_multi.cu) with the narrowest
// factor layout that fits.  FG_WALK_KERNEL=w32 forces the one-walker-per-warp kernel
// for R <= 32 (parity-exact; DESIGN.md section 4 compares the mappings; the
// one-walker-per-thread and two-walkers-per-warp variants measured there were
// removed from the build in round 2 and live in the git history).
int fg_pick_kernel(int ring, int maxlen, int R)
{
    if (R <= 32) {
        if (maxlen > 32) return FG_K_NONE;
        const char *env = getenv("FG_WALK_KERNEL");
        const bool w32 = env && strcmp(env, "w32") == 0;
        if (ring == FG_ZT) {
            if (maxlen > 16) return FG_K_W32_ZT_K32;
            return w32 ? FG_K_W32_ZT_K16 : FG_K_Q4_P16;
        }
        return w32 ? FG_K_W32_Z2_K32 : FG_K_Q4_Z2;
    }
    // 33 <= R <= 128, one-word factors: the linked-class quad kernel (fg_walk_ql.cu),
    // faster than walk_wm on (4,4,4) Z_T and Z_2 (profiles/r01_bench_multi.txt);
    // FG_WALK_KERNEL=wm forces the one-walker-per-warp multi-row kernel.
    // Everything else with 33 <= R <= 512 (wide factors or R > 128: configs C4, C5) runs
    // the linked-class one-walker-per-warp kernel (fg_walk_wl.cuh);
    // FG_WALK_KERNEL=wm forces the round-1 multi-row kernel, =wl forces walk_wl also
    // where walk_ql is the default.
    const char *env = getenv("FG_WALK_KERNEL");
    const bool wm = env && strcmp(env, "wm") == 0;
    const bool wl = env && strcmp(env, "wl") == 0;
    if (R <= 128 && !wm && !wl) {
        if (ring == FG_ZT && maxlen <= 16) return FG_K_QL_P16;
        if (ring == FG_Z2 && maxlen <= 32) return FG_K_QL_Z2;
    }
    if (wm || R > 512) return fg_multi_kind(ring, maxlen, R);
    if (ring == FG_ZT) return maxlen <= 16 ? FG_K_WL_P16 : (maxlen <= 32 ? FG_K_WL_P32 : FG_K_WL_P64);
    return maxlen <= 32 ? FG_K_WL_Z2 : FG_K_WL_Z64;
}

int fg_kind_for_mode(int kind)
{
    switch (kind) {
    case FG_K_QL_P16: return FG_K_WL_P16;
    case FG_K_QL_Z2: return FG_K_WL_Z2;
    default: return kind;
    }
}

const char *fg_kernel_kind_name(int kind)
{
    switch (kind) {
    case FG_K_W32_ZT_K16: return "walk_w32<P16>";
    case FG_K_W32_ZT_K32: return "walk_w32<P32>";
    case FG_K_W32_Z2_K32: return "walk_w32<PZ2>";
    case FG_K_WM_P16: return "walk_wm<P16>";
    case FG_K_WM_P32: return "walk_wm<P32>";
    case FG_K_WM_P64: return "walk_wm<P64>";
    case FG_K_WM_Z2: return "walk_wm<PZ2>";
    case FG_K_WM_Z64: return "walk_wm<PZ64>";
    case FG_K_Q4_P16: return "walk_q4<P16>";
    case FG_K_Q4_Z2: return "walk_q4<PZ2>";
    case FG_K_QL_P16: return "walk_ql<P16>";
    case FG_K_QL_Z2: return "walk_ql<PZ2>";
    case FG_K_WL_P16: return "walk_wl<P16>";
    case FG_K_WL_P32: return "walk_wl<P32>";
    case FG_K_WL_P64: return "walk_wl<P64>";
    case FG_K_WL_Z2: return "walk_wl<PZ2>";
    case FG_K_WL_Z64: return "walk_wl<PZ64>";
    default: return "none";
    }
}

cudaError_t fg_launch_walk(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_W32_ZT_K16: return launch_w32<P16>(a, num_sms, st);
    case FG_K_W32_ZT_K32: return launch_w32<P32>(a, num_sms, st);
    case FG_K_W32_Z2_K32: return launch_w32<PZ2>(a, num_sms, st);
    case FG_K_Q4_P16:
    case FG_K_Q4_Z2: return fg_launch_walk_q4(kind, a, num_sms, st);
    case FG_K_QL_P16:
    case FG_K_QL_Z2: return fg_launch_walk_ql(kind, a, num_sms, st);
    case FG_K_WL_P16:
    case FG_K_WL_P32:
    case FG_K_WL_P64:
    case FG_K_WL_Z2:
    case FG_K_WL_Z64: return fg_launch_walk_wl(kind, a, num_sms, st);
    default: return fg_launch_walk_multi(kind, fg_multi_ns(a.R), a, num_sms, st);
    }
}
