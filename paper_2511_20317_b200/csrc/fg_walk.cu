// fg_walk.cu -- the RandomWalk kernel (Algorithm 1) for walkers
// with at most 32 rows: ONE WALKER PER WARP, row l of the scheme in lane l's
// registers, every step's control flow warp-uniform.
//
// Per step (reading R17):
//   - Philox words: lane L precomputes blocks 0 and 2 of step s0+L for 32 steps,
//     fetched with SHFL; blocks 1 and 3-5 on demand (R8).
//   - flip candidates (R10): MATCH.ANY over the packed (digits, signs) key of each
//     role gives each lane the set of rows sharing its factor; |C| and the k-th
//     candidate come from popc + one warp prefix scan + a ballot (no O(r^2) list).
//   - try_flip (R11): two SHFLs exchange the factors, LOP3 ternary add/sub with
//     the fused validity vote, per-lane sign normalisation.
//   - local reduction check (R12): refreshed match masks; the exact (rare) worklist
//     path runs only if a touched row has a zero factor or shares two factors.
//   - acceptance, reduce_all (R15, exact skip via the masks),
//     expand (R16) with row broadcasts.
// Independent of oracle/; parity is checked by tests/test_gpu_parity.py.
#include <cstdio>
#include "fg_device.cuh"

using namespace fgd;

#define W32_THREADS 128

namespace {

template <int RING, typename T, bool K16>
__global__ void __launch_bounds__(W32_THREADS) walk_w32(WalkArgs a)
{
    const int lane = threadIdx.x & 31;
    const unsigned lanebit = 1u << lane;
    const unsigned above = ~((lanebit << 1) - 1u);          // lanes > this one
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int R = a.R;
    const uint64_t seed = a.seed;

    for (int64_t wk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wk < a.num_walkers;
         wk += nwarps) {
        // ---------------- load walker (coalesced: plane q of rows 0..31) ----------------
        const uint64_t *cp = a.cur + (size_t)wk * FG_PLANES * R;
        const uint64_t *bp = a.best + (size_t)wk * FG_PLANES * R;
        Row<T> row, brow;
        row.u.d = row.u.s = row.v.d = row.v.s = row.w.d = row.w.s = 0;
        brow = row;
        if (lane < R) {
            row.u.d = (T)cp[0 * R + lane]; row.u.s = (T)cp[1 * R + lane];
            row.v.d = (T)cp[2 * R + lane]; row.v.s = (T)cp[3 * R + lane];
            row.w.d = (T)cp[4 * R + lane]; row.w.s = (T)cp[5 * R + lane];
            brow.u.d = (T)bp[0 * R + lane]; brow.u.s = (T)bp[1 * R + lane];
            brow.v.d = (T)bp[2 * R + lane]; brow.v.s = (T)bp[3 * R + lane];
            brow.w.d = (T)bp[4 * R + lane]; brow.w.s = (T)bp[5 * R + lane];
        }
        fg_whdr *hp = a.hdr + wk;
        int r = hp->r;
        int best = hp->best_r;
        uint64_t step = hp->step;
        uint64_t digest = hp->digest;
        const uint32_t wid = (uint32_t)(a.id_base + wk);

        uint32_t c_draws = 0, c_flips = 0, c_eok = 0, c_erej = 0, c_merge = 0, c_zero = 0,
                 c_copy = 0, c_impr = 0, c_red = 0;

        unsigned mU = 0, mV = 0, mW = 0, mWp = 0;
        bool masks_ok = false;
        auto compute_masks = [&]() {
            const unsigned act = r >= 32 ? FULL : ((1u << r) - 1u);
            mU = match<RING, T, K16>(row.u) & act;
            mV = match<RING, T, K16>(row.v) & act;
            mW = match<RING, T, K16>(row.w) & act;
            if (RING == FG_ZT) {
                // W up to sign: key of the sign-normalised w
                Tv<T> wa = row.w;
                const T nw = (wa.s & (wa.d & (T)(0 - wa.d))) ? ~(T)0 : (T)0;
                wa.s ^= wa.d & nw;
                mWp = match<RING, T, K16>(wa) & act;
            } else {
                mWp = mW;
            }
            masks_ok = true;
        };

        // R14 remove(h) with the 2-entry worklist (entries == h dropped, r-1 -> h)
        auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) {
            const int last = r - 1;
            int n2 = 0, x0 = 0, x1 = 0;
            if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
            if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
            wl0 = x0; wl1 = x1; nwl = n2;
            if (h != last) {
                const Row<T> mv = shfl_row<RING, T, K16>(row, last);
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
                const Row<T> rt = shfl_row<RING, T, K16>(row, t);
                if (has_zero(rt)) {
                    remove_row(t, wl0, wl1, nwl);
                    c_zero++;
                    continue;
                }
                Row<T> merged = row;
                const bool red = lane < r && lane != t && reducible<RING, T>(rt, row, merged);
                const unsigned bal = __ballot_sync(FULL, red);
                if (!bal) continue;
                const int j = __ffs(bal) - 1;
                const int lo = t < j ? t : j, hi = t < j ? j : t;
                const Row<T> mg = shfl_row<RING, T, K16>(merged, j);
                if (lane == lo) row = mg;
                c_merge++;
                remove_row(hi, wl0, wl1, nwl);
                if (has_zero(mg)) {
                    remove_row(lo, wl0, wl1, nwl);
                    c_zero++;
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
                    c_zero++;
                    continue;
                }
                compute_masks();
                const unsigned two = ((mU & mV) | (mU & mWp) | (mV & mWp)) & above;
                unsigned cand = __ballot_sync(FULL, lane < r && two != 0);
                bool merged_any = false;
                while (cand) {
                    const int i = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const Row<T> ri = shfl_row<RING, T, K16>(row, i);
                    Row<T> merged = row;
                    const bool red = lane < r && lane > i && reducible<RING, T>(ri, row, merged);
                    const unsigned bal = __ballot_sync(FULL, red);
                    if (!bal) continue;
                    const int j = __ffs(bal) - 1;
                    const Row<T> mg = shfl_row<RING, T, K16>(merged, j);
                    if (lane == i) row = mg;
                    c_merge++;
                    int n0 = 0, x0 = 0, x1 = 0;
                    remove_row(j, x0, x1, n0);
                    if (has_zero(mg)) {
                        remove_row(i, x0, x1, n0);
                        c_zero++;
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
            const Tv<T> fa = get(row, A), fb = get(row, B), fc = get(row, Cr);
            const Tv<T> ai = shfl<T, K16>(fa, i), aj = shfl<T, K16>(fa, j);
            bool ok = true;
            if (plus) {
                const Tv<T> bi = shfl<T, K16>(fb, i), bj = shfl<T, K16>(fb, j);
                const Tv<T> ci = shfl<T, K16>(fc, i), cj = shfl<T, K16>(fc, j);
                if (!distinct<RING, T>(ai, aj) || !distinct<RING, T>(bi, bj) ||
                    !distinct<RING, T>(ci, cj))
                    return false;
                const Tv<T> t1 = add<RING, T>(bi, bj, ok);      // v_i + v_j
                const Tv<T> t2 = sub<RING, T>(cj, ci, ok);      // w_j - w_i
                const Tv<T> t3 = sub<RING, T>(aj, ai, ok);      // u_j - u_i
                if (!ok) return false;
                set(row, B, t1, lane == i);
                set(row, A, ai, lane == j);
                set(row, Cr, t2, lane == j);
                set(row, A, t3, lane == r);
                set(row, B, bj, lane == r);
                set(row, Cr, cj, lane == r);
            } else {
                if (!distinct<RING, T>(ai, aj)) return false;
                const Tv<T> bi = shfl<T, K16>(fb, i), ci = shfl<T, K16>(fc, i);
                const Tv<T> t3 = sub<RING, T>(ai, aj, ok);      // u_i - u_j
                if (!ok) return false;
                set(row, A, aj, lane == i);
                set(row, A, t3, lane == r);
                set(row, B, bi, lane == r);
                set(row, Cr, ci, lane == r);
            }
            if (lane == i || lane == j || lane == r) normalize<RING, T>(row);
            r++;
            masks_ok = false;
            return true;
        };

        uint32_t p0 = 0, p1 = 0, p2 = 0, p3 = 0, q0 = 0, q1 = 0, q2 = 0, q3 = 0;
        int boff = 32;

        for (uint64_t it = 0; it < a.steps; ++it, ++step, ++boff) {
            if (boff == 32) {
                // lane L: Philox blocks 0 and 2 of step (step + L)
                philox_block(seed, step + lane, wid, 0u, p0, p1, p2, p3);
                philox_block(seed, step + lane, wid, 2u, q0, q1, q2, q3);
                boff = 0;
            }
            if (!masks_ok) compute_masks();
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

            // ---- R11 try_flip ----
            if (nC) {
                uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;   // blocks 3..5 on demand
                const uint32_t kf = a.k_flip;
                for (uint32_t at = 0; at < kf; ++at) {
                    uint32_t x;
                    if (at == 0) {
                        x = __shfl_sync(FULL, p0, boff);
                    } else if (at <= 4) {
                        const uint32_t qs = at == 1 ? q0 : (at == 2 ? q1 : (at == 3 ? q2 : q3));
                        x = __shfl_sync(FULL, qs, boff);
                    } else {
                        const uint32_t slot = 7 + at;
                        if ((slot & 3) == 0 || at == 5)
                            philox_block(seed, step, wid, slot >> 2, e0, e1, e2, e3);
                        const uint32_t wsel = slot & 3;
                        x = wsel == 0 ? e0 : (wsel == 1 ? e1 : (wsel == 2 ? e2 : e3));
                    }
                    draws++;
                    const uint32_t k = __umulhi(x, 4u * nC);
                    const uint32_t idx = k >> 2;
                    const int d = k & 1, e = (k >> 1) & 1;
                    int X;
                    uint32_t qq;
                    if (idx < nU) { X = 0; qq = idx; }
                    else if (idx < nU + nV) { X = 1; qq = idx - nU; }
                    else { X = 2; qq = idx - nU - nV; }
                    const int sh = 10 * X;
                    const unsigned inX = (incl >> sh) & 1023u;
                    const int i = __ffs(__ballot_sync(FULL, inX > qq)) - 1;
                    unsigned info = 0;
                    if (lane == i) {
                        unsigned t = qq - (inX - ((cnt >> sh) & 1023u));
                        unsigned mm = (X == 0 ? mU : (X == 1 ? mV : mWp)) & above;
                        for (; t; --t) mm &= mm - 1u;
                        const int j = __ffs(mm) - 1;
                        const unsigned ng = (RING == FG_ZT && X == 2) ? (((mW >> j) & 1u) ^ 1u) : 0u;
                        info = (unsigned)j | (ng << 8);
                    }
                    info = __shfl_sync(FULL, info, i);
                    const int j = info & 255;
                    const bool sneg = (info >> 8) != 0;
                    const int al = d ? j : i, be = d ? i : j;
                    int Y, Z;
                    if (X == 0) { Y = 1; Z = 2; } else if (X == 1) { Y = 2; Z = 0; } else { Y = 0; Z = 1; }
                    if (e) { const int tt = Y; Y = Z; Z = tt; }
                    const Tv<T> fy = get(row, Y), fz = get(row, Z);
                    const Tv<T> recv = shfl<T, K16>(lane == be ? fy : fz, lane == al ? be : al);
                    bool va = true, vb = true;
                    const Tv<T> ny = add<RING, T>(fy, sneg ? neg(recv) : recv, va);  // y_a + s y_b
                    const Tv<T> nz = sub<RING, T>(fz, recv, vb);                      // z_b - z_a
                    const bool bad = (lane == al && !va) || (lane == be && !vb);
                    if (__any_sync(FULL, bad)) continue;
                    set(row, Y, ny, lane == al);
                    set(row, Z, nz, lane == be);
                    if (lane == al || lane == be) normalize<RING, T>(row);
                    alpha = al;
                    beta = be;
                    ok = true;
                    break;
                }
            }
            c_draws += draws;

            if (!ok) {
                // expand; continue
                const bool ex = expand();
                c_eok += ex;
                c_erej += !ex;
                flags |= 2u | (ex ? 64u : 0u);
            } else {
                c_flips++;
                flags |= 1u;
                compute_masks();
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
                if (!acc && r == best) acc = __shfl_sync(FULL, p1, boff) < a.thr_eq;
                if (acc) {
                    const bool strict = r < best;
                    best = r;
                    brow = row;
                    c_copy++;
                    flags |= 4u;
                    if (strict) {
                        flags |= 8u;
                        c_impr++;
                        // R19: enqueue for the batched Brent verifier
                        unsigned slot = 0;
                        if (lane == 0) slot = atomicAdd(a.q_count, 1u);
                        slot = __shfl_sync(FULL, slot, 0);
                        if (slot < a.q_cap) {
                            uint64_t *qp = a.q_planes + (size_t)slot * FG_PLANES * R;
                            if (lane < R) {
                                const bool lv = lane < r;
                                qp[0 * R + lane] = lv ? (uint64_t)row.u.d : 0;
                                qp[1 * R + lane] = lv ? (uint64_t)row.u.s : 0;
                                qp[2 * R + lane] = lv ? (uint64_t)row.v.d : 0;
                                qp[3 * R + lane] = lv ? (uint64_t)row.v.s : 0;
                                qp[4 * R + lane] = lv ? (uint64_t)row.w.d : 0;
                                qp[5 * R + lane] = lv ? (uint64_t)row.w.s : 0;
                            }
                            if (lane == 0) {
                                fg_qmeta qm;
                                qm.walker = wk; qm.step = step; qm.rank = r; qm.ok = -1;
                                qm.ff[0] = qm.ff[1] = qm.ff[2] = -1; qm.pad = 0;
                                a.q_meta[slot] = qm;
                            }
                        } else if (lane == 0) {
                            atomicAdd(a.q_overflow, 1u);
                        }
                    }
                }
                // ---- PAPER:315-317 reduce (R15) ----
                if (__shfl_sync(FULL, p2, boff) < a.thr_reduce) {
                    c_red++;
                    flags |= 16u;
                    const unsigned two = ((mU & mV) | (mU & mWp) | (mV & mWp)) & ~lanebit;
                    if (__any_sync(FULL, lane < r && (has_zero(row) || two != 0))) {
                        slow_reduce_all();
                        compute_masks();
                    }
                }
                // ---- PAPER:319-321 expand ----
                if (__shfl_sync(FULL, p3, boff) < a.thr_expand && r <= best + a.slack) {
                    const bool ex = expand();
                    flags |= 32u | (ex ? 64u : 0u);
                    c_eok += ex;
                    c_erej += !ex;
                }
            }
            // ---- digest ----
            const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)best << 10) |
                                ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) |
                                ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
            digest = (digest ^ ev) * 0x100000001b3ULL;
            digest ^= digest >> 32;
        }

        // ---------------- store walker ----------------
        uint64_t *cw = a.cur + (size_t)wk * FG_PLANES * R;
        uint64_t *bw = a.best + (size_t)wk * FG_PLANES * R;
        if (lane < R) {
            cw[0 * R + lane] = (uint64_t)row.u.d; cw[1 * R + lane] = (uint64_t)row.u.s;
            cw[2 * R + lane] = (uint64_t)row.v.d; cw[3 * R + lane] = (uint64_t)row.v.s;
            cw[4 * R + lane] = (uint64_t)row.w.d; cw[5 * R + lane] = (uint64_t)row.w.s;
            bw[0 * R + lane] = (uint64_t)brow.u.d; bw[1 * R + lane] = (uint64_t)brow.u.s;
            bw[2 * R + lane] = (uint64_t)brow.v.d; bw[3 * R + lane] = (uint64_t)brow.v.s;
            bw[4 * R + lane] = (uint64_t)brow.w.d; bw[5 * R + lane] = (uint64_t)brow.w.s;
        }
        // naive additions of the best -> local best key (R20)
        const int nnz = lane < best ? (__popcll((uint64_t)brow.u.d) + __popcll((uint64_t)brow.v.d) +
                                       __popcll((uint64_t)brow.w.d))
                                    : 0;
        const int tot_nnz = __reduce_add_sync(FULL, nnz);
        if (lane == 0) {
            hp->r = r;
            hp->best_r = best;
            hp->step = step;
            hp->digest = digest;
            hp->cnt[FG_CNT_STEPS] += a.steps;
            hp->cnt[FG_CNT_DRAWS] += c_draws;
            hp->cnt[FG_CNT_FLIPS] += c_flips;
            hp->cnt[FG_CNT_FLIP_FAIL] += a.steps - c_flips;
            hp->cnt[FG_CNT_EXPAND_OK] += c_eok;
            hp->cnt[FG_CNT_EXPAND_REJECT] += c_erej;
            hp->cnt[FG_CNT_MERGES] += c_merge;
            hp->cnt[FG_CNT_ZERO_REMOVED] += c_zero;
            hp->cnt[FG_CNT_BEST_COPIES] += c_copy;
            hp->cnt[FG_CNT_IMPROVEMENTS] += c_impr;
            hp->cnt[FG_CNT_REDUCE_CALLS] += c_red;
            int adds = tot_nnz - 2 * best - a.mp;
            if (adds < 0) adds = 0;
            const unsigned long long key = ((unsigned long long)best << 54) |
                                           ((unsigned long long)adds << 36) |
                                           (unsigned long long)wk;
            atomicMin(a.best_key, key);
        }
    }
}

template <int RING, typename T, bool K16>
cudaError_t launch_w32(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_w32<RING, T, K16>,
                                                                  W32_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    const int64_t wpb = W32_THREADS / 32;
    const int64_t max_warps = (int64_t)num_sms * bps * wpb;
    // even static partition: every warp runs exactly k walkers (or k-1)
    const int64_t k = (a.num_walkers + max_warps - 1) / max_warps;
    const int64_t nwarps = (a.num_walkers + k - 1) / k;
    const int64_t blocks = (nwarps + wpb - 1) / wpb;
    walk_w32<RING, T, K16><<<(unsigned)blocks, W32_THREADS, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

// R <= 32 implies every factor has <= 32 elements (the matmul tensor's rank is at
// least max(mn, np, pm)), so the warp kernel only needs 32-bit factor words.
int fg_pick_kernel(int ring, int maxlen, int R)
{
    if (R > 32 || maxlen > 32) return FG_K_NONE;
    if (ring == FG_ZT) return maxlen <= 16 ? FG_K_W32_ZT_K16 : FG_K_W32_ZT_K32;
    return FG_K_W32_Z2_K32;
}

const char *fg_kernel_kind_name(int kind)
{
    switch (kind) {
    case FG_K_W32_ZT_K16: return "walk_w32<ZT,u32,key32>";
    case FG_K_W32_ZT_K32: return "walk_w32<ZT,u32,key64>";
    case FG_K_W32_Z2_K32: return "walk_w32<Z2,u32>";
    default: return "none";
    }
}

cudaError_t fg_launch_walk(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_W32_ZT_K16: return launch_w32<FG_ZT, uint32_t, true>(a, num_sms, st);
    case FG_K_W32_ZT_K32: return launch_w32<FG_ZT, uint32_t, false>(a, num_sms, st);
    case FG_K_W32_Z2_K32: return launch_w32<FG_Z2, uint32_t, false>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
