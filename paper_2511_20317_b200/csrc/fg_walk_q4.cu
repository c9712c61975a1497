// fg_walk_q4.cu -- the RandomWalk kernel (Algorithm 1) for walkers
// with at most 32 rows and one-word factors (Z_T <= 16 elements, Z_2 <= 32):
// ONE WALKER PER QUAD (4 lanes), 8 walkers per warp.
//
// Why: the one-walker-per-warp kernel (fg_walk.cu) replicates per-walker scalar
// work on 32 lanes (~420 warp instructions per walker-step); one walker per thread
// (walk_t1, 90; removed in round 2, see git history) leaves a single warp per scheduler at the C2 population
// (16384 walkers = 512 warps on 592 SMSPs, 22% issue, profiles/r01_ncu_walk_t1.txt)
// and lets the slowest of 32 walkers set every loop's trip count (~6 flip draws per
// step for 2 on average).  A quad is the middle: 4x the warps, and the quad splits
// the walker's parallel work:
//   - Philox (R8): lane 0 computes block 0 (draw 0 + the three Bernoulli words),
//     lanes 1 and 3 block 2 (draws 1-4), lane 2 block 3 (draws 5-8) -- one block time
//     per step covers two draw rounds;
//   - try_flip (R11): lane q evaluates draw 4t+q in round t; the quad ballot picks the
//     first valid draw, exactly the draw the sequential loop commits (1.07 rounds per
//     walker on average instead of 2 draws);
//   - class-mask passes, the initial mask build, best copies and the HBM loads and
//     stores are split by row ownership: lane q owns rows l with l % 4 == q.
// Every per-walker scalar (r, best, the step, digest, candidate totals, wneg,
// counters) is replicated in the 4 lanes and evolves identically, so the quad's
// control flow is uniform.  The main path (Philox broadcast, row prefix, draw rounds,
// flip commit) is run by every quad of the warp with full-warp collectives; the rare
// paths (merges, removals, expand) use quad-mask collectives.
//
// Shared memory: per warp a region of T1-style slots with stride 8 (walker w of the
// warp at word slot*8 + w): a slot access by the 4 lanes of a quad (rows l = q mod 4,
// slots 3l+X / l) lands in banks 8*((3q+X) mod 4) + w (resp. 8*q + w) and a
// broadcast read of any slot in bank 8*(slot mod 4) + w -- conflict-free both ways.
// Smem writes are done by the owning lane only; __syncwarp(quad) separates a write
// phase from the next cross-lane read.
//
// Same readings, draw order and digest as fg_walk.cu / the oracle; parity:
// tests/test_gpu_parity.py, tests/test_gpu_kernels.py, tests/test_gpu_fuzz.py.
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "fg_device.cuh"

using namespace fgd;

#define Q4_THREADS 32
#define Q4_WARPS (Q4_THREADS / 32)
// 128 registers = 4 warps per SMSP (the register file is split per SMSP), 16 per SM; a
// __maxnreg__ cap measured +4 % on C2 over __launch_bounds__(32, 14/16), which ptxas also
// compiled to 128 registers but with spills in the Z_2 / R24 instantiations
// (profiles/r02_ab_q4_chunks.txt)
#ifndef Q4_MAXNREG
#define Q4_MAXNREG 128
#endif
#ifndef Q4_ORDER
#define Q4_ORDER 0             // chunked tasks: 0 = completion order (ready queue), 1 = chunk-major
#endif
#ifndef Q4_SPIN_MAX
#define Q4_SPIN_MAX 16384      // a warp waiting for its next chunk sleeps 256 ns, doubling up to this
                               // (256 fixed: -1.4 % on C2 Z_T, spare warps polling take issue slots)
#endif

namespace {

enum : int { SF = 0, SMK = 96, SL = 192, SP = 224, SB = 256, Q4_SLOTS = 352 };

// position of the t-th (0-based) set bit of x; t is almost always 0..2 (flip classes
// are small): predicated clears, a loop only beyond
__device__ __forceinline__ int nth_bit_q4(uint32_t x, uint32_t t)
{
    x = t > 0 ? (x & (x - 1u)) : x;
    x = t > 1 ? (x & (x - 1u)) : x;
    x = t > 2 ? (x & (x - 1u)) : x;
    for (uint32_t k = 3; k < t; ++k) x &= x - 1u;
    return __ffs(x) - 1;
}

template <class P, bool CM>
__global__ void __maxnreg__(Q4_MAXNREG) walk_q4(WalkArgs a)
{
    typedef typename P::F F;
    static_assert(sizeof(F) == 4, "one-word factor layouts only");
    __shared__ uint32_t smem[Q4_WARPS][Q4_SLOTS * 8];
    const int lane = threadIdx.x & 31;
    const int q = lane & 3;
    const int qb = lane & 28;
    const unsigned qm = 0xFu << qb;
    uint32_t *const S = smem[threadIdx.x >> 5] + (lane >> 2);
    // Tasks.  Unchunked (a.chunks == 1): one warp per group of 8 walkers, the whole launch.
    // Chunked: (group, step chunk) tasks over persistent warps.  The first n_groups tasks
    // are the groups' chunk 0; every later task is the next chunk of the group that
    // completed a chunk earliest (a ready queue filled in completion order), so groups
    // migrate between the 3- and 4-warp schedulers of a population that is not a
    // multiple of the scheduler count and all finish together.
    const int64_t n_groups = (a.num_walkers + 7) / 8;
    const bool chunked = a.chunks > 1;
    const uint64_t n_tasks = chunked ? (uint64_t)n_groups * a.chunks : 0;
#pragma unroll 1
    for (int pass = 0;; ++pass) {
    int64_t grp;
    uint32_t chunk = 0;
    if (!chunked) {
        if (pass > 0) break;
        grp = (int64_t)blockIdx.x * Q4_WARPS + (threadIdx.x >> 5);
    } else {
        unsigned long long k = 0;
        uint32_t g1 = 0, ch = 0;
        if (lane == 0) {
            k = atomicAdd(a.work_counter, 1ull);
            if (k < n_tasks) {
                if (k < (unsigned long long)n_groups) {
                    g1 = (uint32_t)k + 1u;
                } else if (Q4_ORDER == 1) {
                    // chunk-major: chunk k / n_groups of group k % n_groups, after its predecessor
                    g1 = (uint32_t)(k % (unsigned long long)n_groups) + 1u;
                    ch = (uint32_t)(k / (unsigned long long)n_groups);
                    for (uint32_t ns = 256; *(volatile uint32_t *)(a.task_done + (g1 - 1u)) < ch;
                         ns = ns < Q4_SPIN_MAX ? 2 * ns : ns)
                        __nanosleep(ns);
                    __threadfence();
                } else {
                    for (uint32_t ns = 256; (g1 = *(volatile uint32_t *)(a.ring + (k - n_groups))) == 0u;
                         ns = ns < Q4_SPIN_MAX ? 2 * ns : ns)
                        __nanosleep(ns);
                    __threadfence();
                    ch = *(volatile uint32_t *)(a.task_done + (g1 - 1u));
                }
            }
        }
        k = __shfl_sync(FULL, k, 0);
        if (k >= n_tasks) break;
        grp = (int64_t)__shfl_sync(FULL, g1, 0) - 1;
        chunk = __shfl_sync(FULL, ch, 0);
        __threadfence();
    }
    const bool last_chunk = chunk + 1 >= (chunked ? a.chunks : 1u);
    const uint64_t done_steps = (uint64_t)chunk * a.chunk_steps;
    const uint64_t left = done_steps >= a.steps ? 0 : a.steps - done_steps;
    const uint32_t nsteps_task = (uint32_t)(!chunked ? a.steps : (last_chunk ? left : (left < a.chunk_steps ? left : a.chunk_steps)));
    const int64_t wk_raw = grp * 8 + (lane >> 2);
    // a quad past the last walker stays in the warp (r = 0, no stores) so the main
    // loop's full-warp collectives see every lane
    const bool valid = wk_raw < a.num_walkers;
    const int64_t wk = valid ? wk_raw : 0;

#define FK(l, X) S[(SF + (l) * 3 + (X)) * 8]
#define MK(l, X) S[(SMK + (l) * 3 + (X)) * 8]
#define LK(l) S[(SL + (l)) * 8]
#define PK(l) S[(SP + (l)) * 8]
#define BK(l, X) S[(SB + (l) * 3 + (X)) * 8]

    auto qsync = [&]() { __syncwarp(qm); };
    auto qor = [&](uint32_t v) {
        v |= __shfl_xor_sync(qm, v, 1);
        v |= __shfl_xor_sync(qm, v, 2);
        return v;
    };
    auto qsum = [&](int v) {
        v += __shfl_xor_sync(qm, v, 1);
        v += __shfl_xor_sync(qm, v, 2);
        return v;
    };
    auto qbcast = [&](uint32_t v, int src) { return __shfl_sync(qm, v, qb | src); };
    const uint32_t own = 0x11111111u << q;    // rows this lane owns
    auto owner = [&](int l) -> bool { return (l & 3) == q; };

    const int R = a.R;
    const uint64_t seed = a.seed;
    const uint32_t kf = a.k_flip;
    const uint32_t wid = (uint32_t)(a.id_base + wk);
    fg_whdr *hp = a.hdr + wk;
    const uint64_t *cp = a.cur + (size_t)wk * FG_PLANES * R;
    uint64_t *bw = a.best + (size_t)wk * FG_PLANES * R;

    int r = valid ? hp->r : 0;
    int best = valid ? hp->best_r : 0;
    uint64_t step = hp->step;
    uint64_t digest = hp->digest;
    int best_adds = hp->best_adds;

    // ---------------- load the walker and its best (own rows) ----------------
    // chunk 0 from the plane layout; later chunks restore the shared-memory image and the
    // scalars the previous chunk of this launch saved (ql_img)
    constexpr int IMGQ = Q4_SLOTS + 8;
    uint32_t *const img = a.ql_img ? a.ql_img + (size_t)wk * IMGQ : nullptr;
    const bool resume = chunk > 0 && img != nullptr;
    uint32_t wneg = 0, bwneg = 0;
    int nnz_cur = 0;
    uint32_t nCp = 0;
    bool maybe = true;     // R15: a full reduce_all may find work
    bool bdirty = false;   // best rows changed in this launch
    if (resume && valid) {
#pragma unroll 1
        for (int k = q; k < Q4_SLOTS; k += 4) S[k * 8] = img[k];
        wneg = img[Q4_SLOTS];
        bwneg = img[Q4_SLOTS + 1];
        nnz_cur = (int)img[Q4_SLOTS + 2];
        nCp = img[Q4_SLOTS + 3];
        maybe = img[Q4_SLOTS + 4] != 0u;
        bdirty = img[Q4_SLOTS + 5] != 0u;
    }
    qsync();
#pragma unroll 1
    for (int l = q; l < 32 && !resume; l += 4) {
        F u = 0, v = 0, w = 0, bu = 0, bv = 0, bwv = 0;
        if (l < R) {
            if (l < r) {
                u = P::make(cp[0 * R + l], cp[1 * R + l]);
                v = P::make(cp[2 * R + l], cp[3 * R + l]);
                w = P::make(cp[4 * R + l], cp[5 * R + l]);
            }
            if (l < best) {
                bu = P::make(bw[0 * R + l], bw[1 * R + l]);
                bv = P::make(bw[2 * R + l], bw[3 * R + l]);
                bwv = P::make(bw[4 * R + l], bw[5 * R + l]);
            }
        }
        nnz_cur += l < r ? P::popd(u) + P::popd(v) + P::popd(w) : 0;
        wneg |= (uint32_t)P::first_neg(w) << l;
        bwneg |= (uint32_t)P::first_neg(bwv) << l;
        FK(l, 0) = u; FK(l, 1) = v; FK(l, 2) = P::abs(w);
        BK(l, 0) = bu; BK(l, 1) = bv; BK(l, 2) = P::abs(bwv);
    }
    if (!resume) {
        wneg = qor(wneg);
        bwneg = qor(bwneg);
        nnz_cur = qsum(nnz_cur);
    }
    qsync();
    auto live_mask = [&]() -> uint32_t { return r >= 32 ? FULL : ((1u << r) - 1u); };
    auto above_of = [](int l) -> uint32_t { return ~((2u << l) - 1u); };

    // class masks and later counts of own rows from scratch (once per launch)
    if (!resume) {
        const uint32_t live = live_mask();
        uint32_t part = 0;
#pragma unroll 1
        for (int l = q; l < 32; l += 4) {
            uint32_t lc = 0;
#pragma unroll
            for (int X = 0; X < 3; ++X) {
                const uint32_t key = FK(l, X);
                uint32_t m = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) m |= (FK(j, X) == key) ? (1u << j) : 0u;
                m = l < r ? (m & live) : 0u;
                MK(l, X) = m;
                lc |= (uint32_t)__popc(m & above_of(l)) << (10 * X);
            }
            LK(l) = lc;
            part += lc;
        }
        nCp = (uint32_t)qsum((int)part);
        qsync();
    }

    auto fac = [&](int l, int X) -> F {
        const F k = FK(l, X);
        return (X == 2 && ((wneg >> l) & 1u)) ? P::neg(k) : k;
    };
    auto read_row = [&](int l) -> Row<P> {
        Row<P> x;
        x.u = FK(l, 0);
        x.v = FK(l, 1);
        const F k = FK(l, 2);
        x.w = ((wneg >> l) & 1u) ? P::neg(k) : k;
        return x;
    };
    auto two_of = [&](int l) -> uint32_t {
        const uint32_t mu = MK(l, 0), mv = MK(l, 1), mw = MK(l, 2);
        return ((mu & mv) | (mu & mw) | (mv & mw)) & ~(1u << l);
    };
    auto row_zero = [&](int l) -> bool { return P::zero(FK(l, 0)) || P::zero(FK(l, 1)) || P::zero(FK(l, 2)); };

    // row l's X key becomes `key` (fresh: l was not in any X class).  Collective over
    // the quad (wtag false) or the whole warp (wtag true: every quad calls it, `act`
    // says whether this quad's update is real).
    auto set_class = [&](auto wtag, int l, int X, uint32_t key, bool fresh, bool act) {
        constexpr bool WARP = decltype(wtag)::value;
        const unsigned msk = WARP ? FULL : qm;
        const uint32_t bl = 1u << l;
        const uint32_t mo = (act && !fresh) ? (MK(l, X) & ~bl) : 0u;
        __syncwarp(msk);                           // old state of row l read by all
        if (act && owner(l)) FK(l, X) = key;
        uint32_t mn = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = 4 * k + q;
            mn |= (FK(j, X) == key) ? (1u << j) : 0u;
        }
        mn |= __shfl_xor_sync(msk, mn, 1);
        mn |= __shfl_xor_sync(msk, mn, 2);
        mn = act ? (mn & live_mask() & ~bl) : 0u;
        const int sh = 10 * X;
        const uint32_t one = 1u << sh;
        for (uint32_t t = (mo | mn) & own; t; t &= t - 1u) {
            const int m = __ffs(t) - 1;
            const bool was = (mo >> m) & 1u;
            const uint32_t mk = MK(m, X);
            MK(m, X) = was ? (mk & ~bl) : (mk | bl);
            if (m < l) LK(m) += was ? (0u - one) : one;
        }
        if (act) {
            const uint32_t ab = above_of(l);
            if (owner(l)) {
                MK(l, X) = mn | bl;
                LK(l) += (uint32_t)(__popc(mn & ab) - __popc(mo & ab)) << sh;
            }
            nCp += (uint32_t)(__popc(mn) - __popc(mo)) << sh;
        }
        __syncwarp(msk);
    };
    // store a whole (normalised) row; only changed keys pay a class update.  Collective.
    auto write_row = [&](int l, const Row<P> &x, bool fresh) {
        const F o0 = FK(l, 0), o1 = FK(l, 1), o2 = FK(l, 2);
        if (fresh) {
            qsync();
            if (owner(l)) LK(l) = 0;
        } else {
            nnz_cur -= P::popd(o0) + P::popd(o1) + P::popd(o2);
        }
        nnz_cur += P::popd(x.u) + P::popd(x.v) + P::popd(x.w);
        const F k0 = x.u, k1 = x.v, k2 = P::abs(x.w);
        if (fresh || k0 != o0) set_class(std::false_type{}, l, 0, k0, fresh, true);
        if (fresh || k1 != o1) set_class(std::false_type{}, l, 1, k1, fresh, true);
        if (fresh || k2 != o2) set_class(std::false_type{}, l, 2, k2, fresh, true);
        wneg = (wneg & ~(1u << l)) | ((uint32_t)P::first_neg(x.w) << l);
    };
    // the flip commit (A4/A5): factor Y of row la becomes va and factor Z of row lb
    // becomes vb (actual signs), if `act`.  The rows' other factors are normalised, so
    // only the new factor can trigger PAPER:429 (R6).  The two class updates touch
    // different roles (Y != Z), so they commute and run fused: one pass over the owned
    // rows compares both keys.  Whole-warp collective (every quad calls it).
    auto commit_pair = [&](bool act, int la, int Y, F va, int lb, int Z, F vb) {
        const F olda = FK(la, Y), oldb = FK(lb, Z);
        const bool fna = P::first_neg(va), fnb = P::first_neg(vb);
        const F ka = Y == 2 ? P::abs(va) : (fna ? P::neg(va) : va);
        const F kb = Z == 2 ? P::abs(vb) : (fnb ? P::neg(vb) : vb);
        if (act) {
            nnz_cur += P::popd(va) - P::popd(olda) + P::popd(vb) - P::popd(oldb);
            if (Y == 2) wneg = (wneg & ~(1u << la)) | ((uint32_t)fna << la);
            else wneg ^= (uint32_t)fna << la;
            if (Z == 2) wneg = (wneg & ~(1u << lb)) | ((uint32_t)fnb << lb);
            else wneg ^= (uint32_t)fnb << lb;
        }
        const bool acta = act && ka != olda, actb = act && kb != oldb;
        const uint32_t ba = 1u << la, bb = 1u << lb;
        const uint32_t moa = acta ? (MK(la, Y) & ~ba) : 0u;
        const uint32_t mob = actb ? (MK(lb, Z) & ~bb) : 0u;
        __syncwarp();                              // old state read by all
        if (acta && owner(la)) FK(la, Y) = ka;
        if (actb && owner(lb)) FK(lb, Z) = kb;
        uint32_t mna = 0, mnb = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = 4 * k + q;
            mna |= (FK(j, Y) == ka) ? (1u << j) : 0u;
            mnb |= (FK(j, Z) == kb) ? (1u << j) : 0u;
        }
        mna |= __shfl_xor_sync(FULL, mna, 1);
        mnb |= __shfl_xor_sync(FULL, mnb, 1);
        mna |= __shfl_xor_sync(FULL, mna, 2);
        mnb |= __shfl_xor_sync(FULL, mnb, 2);
        const uint32_t live = live_mask();
        mna = acta ? (mna & live & ~ba) : 0u;
        mnb = actb ? (mnb & live & ~bb) : 0u;
        const uint32_t onea = 1u << (10 * Y), oneb = 1u << (10 * Z);
        for (uint32_t t = (moa | mna) & own; t; t &= t - 1u) {
            const int m = __ffs(t) - 1;
            const bool was = (moa >> m) & 1u;
            const uint32_t mk = MK(m, Y);
            MK(m, Y) = was ? (mk & ~ba) : (mk | ba);
            if (m < la) LK(m) += was ? (0u - onea) : onea;
        }
        for (uint32_t t = (mob | mnb) & own; t; t &= t - 1u) {
            const int m = __ffs(t) - 1;
            const bool was = (mob >> m) & 1u;
            const uint32_t mk = MK(m, Z);
            MK(m, Z) = was ? (mk & ~bb) : (mk | bb);
            if (m < lb) LK(m) += was ? (0u - oneb) : oneb;
        }
        if (acta) {
            const uint32_t ab = above_of(la);
            if (owner(la)) {
                MK(la, Y) = mna | ba;
                LK(la) += (uint32_t)(__popc(mna & ab) - __popc(moa & ab)) << (10 * Y);
            }
            nCp += (uint32_t)(__popc(mna) - __popc(moa)) << (10 * Y);
        }
        if (actb) {
            const uint32_t ab = above_of(lb);
            if (owner(lb)) {
                MK(lb, Z) = mnb | bb;
                LK(lb) += (uint32_t)(__popc(mnb & ab) - __popc(mob & ab)) << (10 * Z);
            }
            nCp += (uint32_t)(__popc(mnb) - __popc(mob)) << (10 * Z);
        }
        __syncwarp();
    };
    auto unlink = [&](int l, int X) {
        const uint32_t bl = 1u << l;
        const uint32_t mo = MK(l, X) & ~bl;
        const uint32_t one = 1u << (10 * X);
        for (uint32_t t = mo & own; t; t &= t - 1u) {
            const int m = __ffs(t) - 1;
            MK(m, X) &= ~bl;
            if (m < l) LK(m) -= one;
        }
        nCp -= (uint32_t)__popc(mo) << (10 * X);
    };
    // R14 remove(h) with the 2-entry worklist (entries == h dropped, r-1 -> h).  Collective.
    auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) {
        const int last = r - 1;
        int n2 = 0, x0 = 0, x1 = 0;
        if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
        if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
        wl0 = x0; wl1 = x1; nwl = n2;
        nnz_cur -= P::popd(FK(h, 0)) + P::popd(FK(h, 1)) + P::popd(FK(h, 2));
        unlink(h, 0); unlink(h, 1); unlink(h, 2);
        qsync();
        if (h != last) {
            const uint32_t bl = 1u << last, bh = 1u << h;
            uint32_t lc = 0;
            F kk[3];
            uint32_t mos[3];
#pragma unroll
            for (int X = 0; X < 3; ++X) {
                kk[X] = FK(last, X);
                mos[X] = MK(last, X) & ~bl;
                lc |= (uint32_t)__popc(mos[X] & above_of(h)) << (10 * X);
            }
            qsync();
#pragma unroll
            for (int X = 0; X < 3; ++X) {
                const uint32_t one = 1u << (10 * X);
                for (uint32_t t = mos[X] & own; t; t &= t - 1u) {
                    const int m = __ffs(t) - 1;
                    MK(m, X) = (MK(m, X) & ~bl) | bh;
                    if (m > h) LK(m) -= one;
                }
                if (owner(h)) {
                    FK(h, X) = kk[X];
                    MK(h, X) = mos[X] | bh;
                }
            }
            if (owner(h)) LK(h) = lc;
            wneg = (wneg & ~bh) | (((wneg >> last) & 1u) << h);
            if (nwl >= 1 && wl0 == last) wl0 = h;
            if (nwl >= 2 && wl1 == last) wl1 = h;
        }
        if (owner(last)) LK(last) = 0;
        wneg &= ~(1u << last);
        r--;
        qsync();
    };

    uint32_t c_draws = 0, c_flips = 0, c_red = 0, c_eok = 0, c_erej = 0, c_merge = 0, c_zero = 0,
             c_copy = 0, c_impr = 0;

    // R12 (local: worklist {a0, b0}) and R15 (global: lexicographic scan) reductions,
    // exact.  One action per iteration -- a zero-row removal or a merge (write the merged
    // row, remove the other, remove the merged one too if it has a zero factor) -- so
    // the class-updating code is inlined once.  Collective over the quad.
    auto reduce_rows = [&](bool local, int a0, int b0) {
        int wl0 = a0, wl1 = b0, nwl = local ? 2 : 0;
        for (;;) {
            int rm0 = -1, rm1 = -1, wr = -1, lo = -1;
            bool push = false;
            Row<P> merged;
            merged.u = merged.v = merged.w = 0;
            if (local) {
                if (nwl == 0) break;
                const int t = wl0;
                wl0 = wl1;
                nwl--;
                if (t >= r) continue;
                if (row_zero(t)) {
                    rm0 = t;
                    c_zero++;
                } else {
                    const Row<P> rt = read_row(t);
                    int j = -1;
                    for (uint32_t c = two_of(t) & live_mask(); c; c &= c - 1u) {
                        const int jj = __ffs(c) - 1;
                        if (reducible<P>(rt, read_row(jj), merged)) { j = jj; break; }
                    }
                    if (j < 0) continue;
                    lo = t < j ? t : j;
                    wr = lo;
                    rm0 = t < j ? j : t;
                    c_merge++;
                    if (has_zero(merged)) { rm1 = lo; c_zero++; } else push = true;
                }
            } else {
                for (int l = 0; l < r; ++l)
                    if (row_zero(l)) { rm0 = l; break; }
                if (rm0 >= 0) {
                    c_zero++;
                } else {
                    for (int i = 0; i < r && wr < 0; ++i) {
                        const uint32_t c0 = two_of(i) & above_of(i) & live_mask();
                        if (!c0) continue;
                        const Row<P> ri = read_row(i);
                        for (uint32_t c = c0; c; c &= c - 1u) {
                            const int j = __ffs(c) - 1;
                            if (!reducible<P>(ri, read_row(j), merged)) continue;
                            wr = i;
                            rm0 = j;
                            break;
                        }
                    }
                    if (wr < 0) break;
                    c_merge++;
                    if (has_zero(merged)) { rm1 = wr; c_zero++; }
                }
            }
            if (wr >= 0) write_row(wr, merged, false);
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                const int h = k == 0 ? rm0 : rm1;
                if (h < 0) break;
                remove_row(h, wl0, wl1, nwl);
            }
            if (push) {
                wl1 = wl0;
                wl0 = lo;
                nwl++;
            }
        }
    };

    // R16 expand (plus / split), words from Philox block 1 of this step.  Collective.
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
        Row<P> ri = read_row(i), rj = read_row(j);
        const F ai = get(ri, A), aj = get(rj, A), bi = get(ri, B), bj = get(rj, B);
        const F ci = get(ri, Cr), cj = get(rj, Cr);
        bool ok = true;
        Row<P> rn;
        rn.u = rn.v = rn.w = 0;
        if (plus) {
            if (!distinct<P>(ai, aj) || !distinct<P>(bi, bj) || !distinct<P>(ci, cj)) return false;
            const F t1 = P::add(bi, bj, ok);      // v_i + v_j
            const F t2 = P::sub(cj, ci, ok);      // w_j - w_i
            const F t3 = P::sub(aj, ai, ok);      // u_j - u_i
            if (!ok) return false;
            set(ri, B, t1, true);
            set(rj, A, ai, true);
            set(rj, Cr, t2, true);
            set(rn, A, t3, true);
            set(rn, B, bj, true);
            set(rn, Cr, cj, true);
            normalize<P>(ri);
            normalize<P>(rj);
            normalize<P>(rn);
            write_row(i, ri, false);
            write_row(j, rj, false);
        } else {
            if (!distinct<P>(ai, aj)) return false;
            const F t3 = P::sub(ai, aj, ok);      // u_i - u_j
            if (!ok) return false;
            set(ri, A, aj, true);
            set(rn, A, t3, true);
            set(rn, B, bi, true);
            set(rn, Cr, ci, true);
            normalize<P>(ri);
            normalize<P>(rn);
            write_row(i, ri, false);
        }
        r++;
        write_row(r - 1, rn, true);
        maybe = true;
        return true;
    };

    // best copy of own rows into shared memory; HBM once per launch
    auto copy_best = [&]() {
        for (int l = q; l < r; l += 4) {
            BK(l, 0) = FK(l, 0);
            BK(l, 1) = FK(l, 1);
            BK(l, 2) = FK(l, 2);
        }
        bwneg = wneg;
        bdirty = true;
    };
    // R19 verify queue entry: the current rows (== the new best), plane layout
    auto enqueue_verify = [&]() {
        unsigned slot = 0;
        if (q == 0) slot = atomicAdd(a.q_count, 1u);
        slot = qbcast(slot, 0);
        if (slot < a.q_cap) {
            uint64_t *dst = a.q_planes + (size_t)slot * FG_PLANES * R;
            for (int l = q; l < R; l += 4) {
                const bool lv = l < r;
                const F u = lv ? FK(l, 0) : 0, v = lv ? FK(l, 1) : 0, w = lv ? fac(l, 2) : 0;
                dst[0 * R + l] = P::dig(u); dst[1 * R + l] = P::sgn(u);
                dst[2 * R + l] = P::dig(v); dst[3 * R + l] = P::sgn(v);
                dst[4 * R + l] = P::dig(w); dst[5 * R + l] = P::sgn(w);
            }
            if (q == 0) {
                fg_qmeta qm_;
                qm_.walker = wk; qm_.step = step; qm_.rank = r; qm_.ok = -1;
                qm_.ff[0] = qm_.ff[1] = qm_.ff[2] = -1; qm_.pad = 0;
                a.q_meta[slot] = qm_;
            }
        } else if (q == 0) {
            atomicAdd(a.q_overflow, 1u);
            hp->pad |= 1;
        }
    };

    const uint32_t nsteps = nsteps_task;              // host chunks launches below 2^31 steps
#pragma unroll 1
    for (uint32_t it = 0; it < nsteps; ++it, ++step) {
        // Philox (R8): lane 0 block 0 (draw 0 + Bernoulli words), lanes 1 and 3 block 2
        // (draws 1-4), lane 2 block 3 (draws 5-8): rounds 0 and 1 need no further block
        uint32_t cb = q == 0 ? 0u : (q == 2 ? 3u : 2u);
        uint32_t c0, c1, c2, c3;
        philox_block(seed, step, wid, cb, c0, c1, c2, c3);
        const uint32_t bern = __shfl_sync(FULL, (c1 < a.thr_eq ? 1u : 0u) | (c2 < a.thr_reduce ? 2u : 0u) |
                                                    (c3 < a.thr_expand ? 4u : 0u), qb);
        uint32_t flags = 0;
        int alpha = 0, beta = 0;
        uint32_t draws = 0;
        bool ok = false;
        const uint32_t nU = nCp & 1023u, nV = (nCp >> 10) & 1023u, nW = nCp >> 20;
        const uint32_t nC = nU + nV + nW;
        int e_Y = 0, e_Z = 0;
        F e_ny = 0, e_nz = 0;
        // R10 row prefix of the later counts (packed 3 x 10 bits), quad scan per row group;
        // every step (a flip almost always changes a class; a branch on it cost 1 %)
        {
            uint32_t base = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t v = LK(4 * k + q);
                uint32_t sc = v;
                uint32_t t = __shfl_up_sync(FULL, sc, 1, 4);
                sc += q >= 1 ? t : 0u;
                t = __shfl_up_sync(FULL, sc, 2, 4);
                sc += q >= 2 ? t : 0u;
                const uint32_t tot = __shfl_sync(FULL, sc, 3, 4);
                PK(4 * k + q) = base + sc - v;
                base += tot;
            }
            __syncwarp();
        }
        // R11 try_flip: round t, lane q evaluates draw 4t+q; every quad of the warp
        // runs the rounds until the last one has its flip (full-warp ballots)
        bool searching = nC != 0;
#pragma unroll 1
        for (uint32_t t = 0; __any_sync(FULL, searching && 4u * t < kf); ++t) {
            const uint32_t att = 4u * t + (uint32_t)q;
            uint32_t x;
            if (t == 0) {
                const uint32_t s1 = __shfl_sync(FULL, c1, qb | 1);      // block 2 word 1
                x = q <= 1 ? c0 : (q == 2 ? s1 : c2);
            } else if (t == 1) {
                const uint32_t s3 = __shfl_sync(FULL, c3, qb | 1);      // block 2 word 3 (draw 4)
                const uint32_t u0 = __shfl_sync(FULL, c0, qb | 2);      // block 3 word 0 (draw 5)
                const uint32_t u2 = __shfl_sync(FULL, c2, qb | 2);      // block 3 word 2 (draw 7)
                x = q == 0 ? s3 : (q == 1 ? u0 : (q == 2 ? c1 : u2));
            } else {
                const uint32_t slot = 7u + att, blk = slot >> 2;
                if (blk != cb) {
                    philox_block(seed, step, wid, blk, c0, c1, c2, c3);
                    cb = blk;
                }
                const uint32_t wsel = slot & 3u;
                x = wsel == 0 ? c0 : (wsel == 1 ? c1 : (wsel == 2 ? c2 : c3));
            }
            // ---- R11 draw: k uniform over 4|C| (R9), candidate k>>2 in (X, i, j) order ----
            const uint32_t k = __umulhi(x, 4u * nC);
            const uint32_t idx = k >> 2;
            const int d = k & 1, e = (k >> 1) & 1;
            const uint32_t g1 = idx >= nU, g2 = idx >= nU + nV;
            const int X = (int)(g1 + g2);
            const uint32_t qq = idx - (g1 ? nU : 0u) - (g2 ? nV : 0u);
            const int sh = 10 * X;
            const uint32_t fm = 1023u << sh, qs = qq << sh;
            // i = the last row with PF_X(i) <= qq (PF is nondecreasing, PF(0) = 0): three
            // levels of independent loads (rows 8/16/24, then +2/+4/+6, then +1) instead of
            // a five-deep dependent binary search
            int i = 8 * (int)(((PK(8) & fm) <= qs) + ((PK(16) & fm) <= qs) + ((PK(24) & fm) <= qs));
            i += 2 * (int)(((PK(i + 2) & fm) <= qs) + ((PK(i + 4) & fm) <= qs) + ((PK(i + 6) & fm) <= qs));
            i += (PK(i + 1) & fm) <= qs ? 1 : 0;
            const uint32_t ex_i = (PK(i) >> sh) & 1023u;
            const uint32_t mm = MK(i, X) & above_of(i);
            const int j = nth_bit_q4(mm, qq - ex_i) & 31;     // (& 31: quads not searching)
            const int al = d ? j : i, be = d ? i : j;
            // (Y,Z) = (V,W) / (W,U) / (U,V) for X = U / V / W, swapped if e
            const uint32_t yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
            const int Y = yz & 3, Z = yz >> 2;
            const bool sneg = P::RING == FG_ZT && X == 2 && (((wneg >> al) ^ (wneg >> be)) & 1u);
            const F yb = fac(be, Y);
            bool v = searching && att < kf;
            const F ny = P::add(fac(al, Y), sneg ? P::neg(yb) : yb, v);   // y_a + s y_b
            const F nz = P::sub(fac(be, Z), fac(al, Z), v);             // z_b - z_a
            // R24: no reduction edges -> a draw making a factor zero is rejected
            if (CM) v = v && !P::zero(ny) && !P::zero(nz);
            const uint32_t bal = (__ballot_sync(FULL, v) >> qb) & 15u;
            const int src = bal ? __ffs(bal) - 1 : 0;
            const uint32_t info = __shfl_sync(FULL, (uint32_t)(al | (be << 8) | (Y << 16) | (Z << 18)), qb | src);
            const F wny = __shfl_sync(FULL, ny, qb | src);
            const F wnz = __shfl_sync(FULL, nz, qb | src);
            if (bal) {
                alpha = info & 255;
                beta = (info >> 8) & 255;
                e_Y = (info >> 16) & 3;
                e_Z = (info >> 18) & 3;
                e_ny = wny;
                e_nz = wnz;
                draws = 4u * t + (uint32_t)src + 1u;
                ok = true;
                searching = false;
            }
        }
        if (nC && !ok) draws = kf;
        c_draws += draws;
        // commit the flip (every quad takes part; `ok` gates the update)
        commit_pair(ok, alpha, e_Y, e_ny, beta, e_Z, e_nz);

        if (CM) {
            // ---- R24 step: flips only; best by (rank, naive additions) ----
            if (ok) {
                c_flips++;
                flags |= 1u;
                const int adds = nnz_cur - 2 * r - a.mp;
                const bool better = r < best || (r == best && adds < best_adds);
                if (better || (r == best && adds == best_adds && (bern & 1u))) {
                    best = r;
                    best_adds = adds;
                    c_copy++;
                    flags |= 4u;
                    copy_best();
                    if (better) {
                        flags |= 8u;
                        c_impr++;
                        enqueue_verify();
                    }
                }
            }
        } else if (!ok) {
            // expand; continue
            const bool ex = expand();
            c_eok += ex;
            c_erej += !ex;
            flags |= 2u | (ex ? 64u : 0u);
            alpha = beta = 0;
        } else {
            c_flips++;
            flags |= 1u;
            // ---- R12 local reduction (exact skip through the masks) ----
            if (P::zero(e_ny) || P::zero(e_nz) || two_of(alpha) || two_of(beta)) reduce_rows(true, alpha, beta);
            // ---- PAPER:310-313 acceptance ----
            const bool strict = r < best;
            if (strict || (r == best && (bern & 1u))) {
                best = r;
                best_adds = nnz_cur - 2 * r - a.mp;
                c_copy++;
                flags |= 4u;
                copy_best();
                if (strict) {
                    flags |= 8u;
                    c_impr++;
                    enqueue_verify();
                }
            }
            // ---- PAPER:315-317 reduce (R15) ----
            if (bern & 2u) {
                c_red++;
                flags |= 16u;
                if (maybe) {
                    reduce_rows(false, 0, 0);
                    maybe = false;
                }
            }
            // ---- PAPER:319-321 expand ----
            if ((bern & 4u) && r <= best + a.slack) {
                const bool ex = expand();
                flags |= 32u | (ex ? 64u : 0u);
                c_eok += ex;
                c_erej += !ex;
            }
        }
        // ---- digest ----
        const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)(CM ? (best_adds & 1023) : best) << 10) |
                            ((uint64_t)flags << 20) | ((uint64_t)alpha << 32) | ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
        digest = (digest ^ ev) * 0x100000001b3ULL;
        digest ^= digest >> 32;
    }

    // ---------------- not the last chunk: save the image for the next one ----------------
    if (!last_chunk && valid) {
        qsync();
#pragma unroll 1
        for (int k = q; k < Q4_SLOTS; k += 4) img[k] = S[k * 8];
        if (q == 0) {
            img[Q4_SLOTS] = wneg;
            img[Q4_SLOTS + 1] = bwneg;
            img[Q4_SLOTS + 2] = (uint32_t)nnz_cur;
            img[Q4_SLOTS + 3] = nCp;
            img[Q4_SLOTS + 4] = maybe ? 1u : 0u;
            img[Q4_SLOTS + 5] = bdirty ? 1u : 0u;
        }
    }
    // ---------------- last chunk: store own rows (and the best if it changed) ----------------
    uint64_t *cw = a.cur + (size_t)wk * FG_PLANES * R;
    int best_nnz = 0;
    for (int l = q; l < R && valid && last_chunk; l += 4) {
        const bool lv = l < r;
        const F u = lv ? FK(l, 0) : 0, v = lv ? FK(l, 1) : 0, w = lv ? fac(l, 2) : 0;
        cw[0 * R + l] = P::dig(u); cw[1 * R + l] = P::sgn(u);
        cw[2 * R + l] = P::dig(v); cw[3 * R + l] = P::sgn(v);
        cw[4 * R + l] = P::dig(w); cw[5 * R + l] = P::sgn(w);
        const bool lb = l < best;
        const F bu = lb ? BK(l, 0) : 0, bv = lb ? BK(l, 1) : 0, bk = lb ? BK(l, 2) : 0;
        const F bwv = ((bwneg >> l) & 1u) ? P::neg(bk) : bk;
        best_nnz += P::popd(bu) + P::popd(bv) + P::popd(bwv);
        if (bdirty) {
            bw[0 * R + l] = P::dig(bu); bw[1 * R + l] = P::sgn(bu);
            bw[2 * R + l] = P::dig(bv); bw[3 * R + l] = P::sgn(bv);
            bw[4 * R + l] = P::dig(bwv); bw[5 * R + l] = P::sgn(bwv);
        }
    }
    best_nnz = qsum(best_nnz);
    if (q == 0 && valid) {
        hp->r = r;
        hp->best_r = best;
        hp->step = step;
        hp->digest = digest;
        hp->best_adds = best_adds;
        hp->cnt[FG_CNT_STEPS] += nsteps_task;
        hp->cnt[FG_CNT_DRAWS] += c_draws;
        hp->cnt[FG_CNT_FLIPS] += c_flips;
        hp->cnt[FG_CNT_FLIP_FAIL] += nsteps_task - c_flips;
        hp->cnt[FG_CNT_EXPAND_OK] += c_eok;
        hp->cnt[FG_CNT_EXPAND_REJECT] += c_erej;
        hp->cnt[FG_CNT_MERGES] += c_merge;
        hp->cnt[FG_CNT_ZERO_REMOVED] += c_zero;
        hp->cnt[FG_CNT_BEST_COPIES] += c_copy;
        hp->cnt[FG_CNT_IMPROVEMENTS] += c_impr;
        hp->cnt[FG_CNT_REDUCE_CALLS] += c_red;
        int adds = best_nnz - 2 * best - a.mp;
        if (adds < 0) adds = 0;
        if (last_chunk)
            atomicMin(a.best_key, ((unsigned long long)best << 54) | ((unsigned long long)adds << 36) |
                                      (unsigned long long)wk);
    }
    // chunk stored: publish the group's next chunk in the ready queue
    if (chunked && !last_chunk) {
        __syncwarp();
        __threadfence();
        if (lane == 0) {
            atomicExch(a.task_done + grp, chunk + 1u);
            __threadfence();
            if (Q4_ORDER == 0) {
                const unsigned long long slot = atomicAdd(a.ring_tail, 1ull);
                atomicExch(a.ring + slot, (uint32_t)grp + 1u);
            }
        }
    }
    __syncwarp();
    }   // task loop
#undef FK
#undef MK
#undef LK
#undef PK
#undef BK
}

template <class P, bool CM>
cudaError_t launch_q4_m(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    const int64_t groups = (a.num_walkers + 7) / 8;
    // all of the unified L1 as shared memory: 1-warp CTAs with 11 KB of static shared memory
    // each would otherwise be capped by the driver's default carveout, not by registers
    static bool carve = false;
    if (!carve) {
        cudaError_t ce = cudaFuncSetAttribute(walk_q4<P, CM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                              (int)cudaSharedmemCarveoutMaxShared);
        if (ce != cudaSuccess) return ce;
        carve = true;
    }
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_q4<P, CM>, Q4_THREADS, 0);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    const int64_t resident = (int64_t)num_sms * bps * Q4_WARPS;     // warps
    WalkArgs b = a;
    // chunked tasks when the population gives every scheduler more than one warp but is
    // not a whole number of warps per scheduler (the C2 case: 2048 warps on 592
    // schedulers); FG_Q4_CHUNKS forces a count (tests, A/B)
    b.chunks = (groups > (int64_t)num_sms * 4 && groups <= resident && a.steps >= 512 && a.ql_img && a.ring) ? 8u : 1u;
    if (const char *ev = getenv("FG_Q4_CHUNKS")) {
        const long k = strtol(ev, nullptr, 10);
        if (k >= 1 && k <= 64 && a.ql_img && a.ring) b.chunks = (uint32_t)k;
    }
    if ((uint64_t)b.chunks > a.steps) b.chunks = a.steps > 0 ? (uint32_t)a.steps : 1u;
    b.chunk_steps = (a.steps + b.chunks - 1) / b.chunks;
    int64_t blocks;
    if (b.chunks > 1) {
        e = cudaMemsetAsync(b.ring, 0, sizeof(uint32_t) * (size_t)(groups * b.chunks), st);
        if (e != cudaSuccess) return e;
        blocks = resident / Q4_WARPS;
        // FG_Q4_SPARE (A/B): warps beyond one per group, default every resident warp
        if (const char *sv = getenv("FG_Q4_SPARE")) {
            const int64_t w = groups + strtol(sv, nullptr, 10);
            if (w >= groups && w < resident) blocks = (w + Q4_WARPS - 1) / Q4_WARPS;
        }
    } else {
        blocks = (groups + Q4_WARPS - 1) / Q4_WARPS;
    }
    if (getenv("FG_DBG_LAUNCH"))
        fprintf(stderr, "walk_q4: %d CTAs/SM, resident %lld warps, groups %lld, chunks %u, grid %lld\n", bps,
                (long long)resident, (long long)groups, b.chunks, (long long)blocks);
    walk_q4<P, CM><<<(unsigned)blocks, Q4_THREADS, 0, st>>>(b);
    return cudaGetLastError();
}

template <class P>
cudaError_t launch_q4(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    return a.mode == 1 ? launch_q4_m<P, true>(a, num_sms, st) : launch_q4_m<P, false>(a, num_sms, st);
}

}  // namespace

cudaError_t fg_launch_walk_q4(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_Q4_P16: return launch_q4<P16>(a, num_sms, st);
    case FG_K_Q4_Z2: return launch_q4<PZ2>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
