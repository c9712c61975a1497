// fg_walk_ql.cu -- the RandomWalk kernel (Algorithm 1) for walkers
// with 33..128 rows and one-word factors (Z_T <= 16 elements, Z_2 <= 32): ONE WALKER
// PER QUAD, like fg_walk_q4.cu, with the flip classes kept as LINKED LISTS.
//
// Why: walk_q4 keeps one class mask per row and role (R bits); at R = 96 that is 3.4 KB
// per walker and 8 walkers per warp would not fit shared memory.  Here every row keeps,
// per role, the next row of its class in row order (bytes), which is all R10/R11 need:
// the t-th later member of row i is t+1 `next` hops, and the later count of a row (the
// length of its `next` chain) is kept explicitly.  A class change is ONE compare pass over
// the rows (split over the quad) against the old and the new key: it gives the old and
// the new neighbours, the members below the row (whose later counts change) and the
// candidate-pair totals, so no `prev` links are stored.  Five words per row (three keys,
// next links + W sign, later counts) put the C3 population (16384 walkers) in one wave
// of 2-warp CTAs (14 warps per SM).
//
// Per walker (shared memory, per warp stride 8 as in walk_q4; lane q owns rows l % 4 == q):
//   F(l,X)  row l's factor X key (W up to sign; the sign is bit 24 of NX(l))
//   NX(l)   next row of l's U / V / W class (bytes 0..2, 0xFF = none)
//   L(l)    later counts, 3 x 10 bits
//   G(g)    later counts before row group g (8 rows): word 0 = U | V << 16, word 1 = W
// R15 (reduce_all) searches partners of the rows in a dirty set D only: flips are cleaned
// by R12, so only rows changed by expands (or global merges) since the last clean scan
// can be in a reducible pair (as in fg_walk_wl.cuh); D overflow or a fresh load falls
// back to the full lexicographic scan.  The best scheme lives in HBM (written on
// acceptance; rows up to the previous best rank only).
//
// Same readings, draw order and digest as fg_walk.cu / the oracle; parity:
// tests/test_gpu_kernels.py, tests/test_gpu_fuzz.py, tests/test_gpu_fullsize.py.
#include <cstdlib>
#include <type_traits>
#include "fg_device.cuh"

using namespace fgd;

#define QL_THREADS 64                  // 2-warp CTAs: one 1 KB CTA reserve per 2 warps
#define QL_MINB 7
#ifndef QL_SPIN_MAX
#define QL_SPIN_MAX 0                  // a warp waiting for a group's previous chunk: 0 = busy poll,
#endif                                 // else sleep 64 ns doubling up to this

namespace {

constexpr int NIL = 0xFF;

template <class P, int NWD>
__global__ void __launch_bounds__(QL_THREADS, QL_MINB) walk_ql(WalkArgs a)
{
    typedef typename P::F F;
    static_assert(sizeof(F) == 4, "one-word factor layouts only");
    constexpr int RM = 32 * NWD;                 // row capacity of this instantiation
    constexpr int NG = RM / 8;                   // row groups of the prefix
    constexpr int S_NX = 3 * RM, S_L = 4 * RM, S_G = 5 * RM;
    constexpr int SLOTS = 5 * RM + 2 * NG;
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int q = lane & 3;
    const int qb = lane & 28;
    const unsigned qm = 0xFu << qb;
    uint32_t *const S = smem + (threadIdx.x >> 5) * SLOTS * 8 + (lane >> 2);
    // Tasks = (walker group of 8, step chunk), handed out chunk-major by an atomic
    // counter to persistent warps: a population of 1.26 waves costs ~1.3 chunk rounds
    // instead of two full waves.  Chunk c of a group starts after chunk c-1 stored the
    // group's state (task_done flag, fenced).  With one chunk this is one task per warp.
    const int64_t n_groups = (a.num_walkers + 7) / 8;
    const uint64_t n_tasks = (uint64_t)n_groups * a.chunks;
#pragma unroll 1
    for (;;) {
    unsigned long long task = 0;
    if (lane == 0) task = atomicAdd(a.work_counter, 1ull);
    task = __shfl_sync(FULL, task, 0);
    if (task >= n_tasks) break;
    const int64_t grp = (int64_t)(task % (uint64_t)n_groups);
    const uint32_t chunk = (uint32_t)(task / (uint64_t)n_groups);
    if (chunk > 0) {
        if (lane == 0)
            for (uint32_t ns = 64; *(volatile uint32_t *)(a.task_done + grp) < chunk;
                 ns = (int)ns < QL_SPIN_MAX ? 2 * ns : ns)
                if (QL_SPIN_MAX) __nanosleep(ns);
        __syncwarp();
        __threadfence();
    }
    const uint64_t done_steps = (uint64_t)chunk * a.chunk_steps;
    const uint64_t left = done_steps >= a.steps ? 0 : a.steps - done_steps;
    const uint32_t nsteps_task = (uint32_t)(left < a.chunk_steps ? left : a.chunk_steps);
    const int64_t wk_raw = grp * 8 + (lane >> 2);
    // a quad past the last walker stays in the warp (r = 0, no stores)
    const bool valid = wk_raw < a.num_walkers;
    const int64_t wk = valid ? wk_raw : 0;

#define FK(l, X) S[(3 * (l) + (X)) * 8]
#define NXW(l) S[(S_NX + (l)) * 8]
#define LK(l) S[(S_L + (l)) * 8]
#define GK(g, h) S[(S_G + 2 * (g) + (h)) * 8]

    auto owner = [&](int l) __attribute__((always_inline)) -> bool { return (l & 3) == q; };
    auto qsync = [&]() __attribute__((always_inline)) { __syncwarp(qm); };
    auto byte_of = [](uint32_t w, int X) __attribute__((always_inline)) -> int { return (int)((w >> (8 * X)) & 0xFFu); };
    auto nxt = [&](int l, int X) __attribute__((always_inline)) -> int { return byte_of(NXW(l), X); };
    auto set_byte = [](uint32_t w, int X, int v) __attribute__((always_inline)) -> uint32_t {
        return (w & ~(0xFFu << (8 * X))) | (((uint32_t)v & 0xFFu) << (8 * X));
    };
    auto below_in = [](int l, int w) __attribute__((always_inline)) -> uint32_t {      // bits of mask word w for rows < l
        const int b = l - 32 * w;
        return b <= 0 ? 0u : (b >= 32 ? 0xFFFFFFFFu : ((1u << b) - 1u));
    };
    auto above_in = [](int l, int w) __attribute__((always_inline)) -> uint32_t {      // bits of mask word w for rows > l
        const int b = l - 32 * w;
        return b < 0 ? 0xFFFFFFFFu : (b >= 31 ? 0u : ~((2u << b) - 1u));
    };

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

    // W sign of row l: bit 24 of NX(l) (the stored W key is up to sign)
    auto wbit = [&](int l) __attribute__((always_inline)) -> uint32_t { return (NXW(l) >> 24) & 1u; };
    auto set_wbit = [&](int l, uint32_t v) __attribute__((always_inline)) {    // owner; caller syncs
        if (owner(l)) NXW(l) = (NXW(l) & 0x00FFFFFFu) | ((v & 1u) << 24);
    };
    auto live_in = [&](int w) __attribute__((always_inline)) -> uint32_t { return below_in(r, w); };

    // ---------------- load the walker ----------------
    // chunk 0 of a launch builds the class structure from the plane layout; a later chunk
    // restores the shared-memory image and scalars the previous chunk saved (ql_img)
    int nnz_cur = 0;
    uint32_t nCU = 0, nCV = 0, nCW = 0;     // flip-candidate pairs per role (R10)
    // R15 dirty set D (<= 6 rows, 8 bits each) and its overflow flag (fresh load: any pair)
    uint64_t dset = 0;
    int nD = 0;
    bool dover = true;
    constexpr int IMG = SLOTS + 7;          // image words per walker
    uint32_t *const img = a.ql_img ? a.ql_img + (size_t)wk * IMG : nullptr;
    const bool resume = chunk > 0 && img != nullptr && valid;
    if (resume) {
#pragma unroll 1
        for (int k = q; k < SLOTS; k += 4) S[k * 8] = img[k];
        nnz_cur = (int)img[SLOTS];
        nCU = img[SLOTS + 1]; nCV = img[SLOTS + 2]; nCW = img[SLOTS + 3];
        dset = (uint64_t)img[SLOTS + 4] | ((uint64_t)img[SLOTS + 5] << 32);
        nD = (int)(img[SLOTS + 6] & 0xFFu);
        dover = (img[SLOTS + 6] >> 8) != 0u;
        qsync();
    }
    uint32_t own_sign = 0;                       // W signs of own rows (bit l / 4)
#pragma unroll 1
    for (int l = q; l < RM && !resume; l += 4) {
        F u = 0, v = 0, w = 0;
        if (l < r) {
            u = P::make(cp[0 * R + l], cp[1 * R + l]);
            v = P::make(cp[2 * R + l], cp[3 * R + l]);
            w = P::make(cp[4 * R + l], cp[5 * R + l]);
        }
        nnz_cur += l < r ? P::popd(u) + P::popd(v) + P::popd(w) : 0;
        own_sign |= (uint32_t)P::first_neg(w) << (l >> 2);
        FK(l, 0) = u; FK(l, 1) = v; FK(l, 2) = P::abs(w);
    }
    if (!resume) {
        nnz_cur += __shfl_xor_sync(qm, nnz_cur, 1);
        nnz_cur += __shfl_xor_sync(qm, nnz_cur, 2);
    }
    qsync();

    // class links and later counts from scratch (chunk 0): own rows
    auto addn = [&](int X, int v) __attribute__((always_inline)) {
        nCU += X == 0 ? (uint32_t)v : 0u;
        nCV += X == 1 ? (uint32_t)v : 0u;
        nCW += X == 2 ? (uint32_t)v : 0u;
    };
    if (!resume) {
        uint32_t pu = 0, pv_ = 0, pw = 0;
#pragma unroll 1
        for (int l = q; l < RM; l += 4) {
            uint32_t nxw = 0xFFFFFFu, lc = 0;
            if (l < r) {
#pragma unroll 1
                for (int X = 0; X < 3; ++X) {
                    const uint32_t key = FK(l, X);
                    int nx = NIL, cnt = 0;
                    for (int j = l + 1; j < r; ++j) {
                        if (FK(j, X) != key) continue;
                        if (nx == NIL) nx = j;
                        cnt++;
                    }
                    nxw = set_byte(nxw, X, nx);
                    lc |= (uint32_t)cnt << (10 * X);
                }
            }
            NXW(l) = nxw | (((own_sign >> (l >> 2)) & 1u) << 24); LK(l) = lc;
            pu += lc & 1023u; pv_ += (lc >> 10) & 1023u; pw += lc >> 20;
        }
        pu += __shfl_xor_sync(qm, pu, 1); pu += __shfl_xor_sync(qm, pu, 2);
        pv_ += __shfl_xor_sync(qm, pv_, 1); pv_ += __shfl_xor_sync(qm, pv_, 2);
        pw += __shfl_xor_sync(qm, pw, 1); pw += __shfl_xor_sync(qm, pw, 2);
        nCU = pu; nCV = pv_; nCW = pw;
        qsync();
    }

    auto fac = [&](int l, int X) __attribute__((always_inline)) -> F {
        const F k = FK(l, X);
        return (X == 2 && wbit(l)) ? P::neg(k) : k;
    };
    auto read_row = [&](int l) __attribute__((always_inline)) -> Row<P> {
        Row<P> x;
        x.u = FK(l, 0);
        x.v = FK(l, 1);
        const F k = FK(l, 2);
        x.w = wbit(l) ? P::neg(k) : k;
        return x;
    };
    auto row_zero = [&](int l) __attribute__((always_inline)) -> bool { return P::zero(FK(l, 0)) || P::zero(FK(l, 1)) || P::zero(FK(l, 2)); };

    // ---- class structure primitives ----
    // rows j (live, != l) of mask word w whose role-X key equals `key`: each lane compares
    // its 8 rows, the quad ORs the four parts (replicated in the quad).  Collective over msk.
    auto cmask = [&](int w, int X, uint32_t key, int l, unsigned msk) __attribute__((always_inline)) -> uint32_t {
        uint32_t mw = 0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int j = 32 * w + 4 * kk + q;
            mw |= (FK(j, X) == key) ? (1u << (4 * kk + q)) : 0u;
        }
        mw |= __shfl_xor_sync(msk, mw, 1);
        mw |= __shfl_xor_sync(msk, mw, 2);
        return mw & live_in(w) & ~(((l >> 5) == w) ? (1u << (l & 31)) : 0u);
    };
    // Row l's X key goes from `okey` to `key` (fresh: l was in no X class): ONE compare
    // pass against both keys gives the old neighbours (pO, sO: relinked), the new ones
    // (pK, sK: l spliced in), the members below l (their later counts lose / gain l) and
    // the change of the role's pair count.  With WARP the same pass also reports whether
    // some row other than l and `excl` shares two factors with row l after the change
    // (R12's skip test: rows compared with l's other two keys).  Writes by owners; the
    // caller syncs before the next cross-lane read.
    auto change_class = [&](auto wtag, int l, int X, uint32_t okey, uint32_t key, bool fresh, bool act, int excl,
                            bool &two) __attribute__((always_inline)) {
        constexpr bool WARP = decltype(wtag)::value;
        const unsigned msk = WARP ? FULL : qm;
        const int O1 = X == 2 ? 0 : X + 1, O2 = X == 0 ? 2 : X - 1;
        const uint32_t k1 = WARP ? FK(l, O1) : 0u, k2 = WARP ? FK(l, O2) : 0u;
        two = false;
        // one mask word (32 rows) per iteration, not unrolled: a compact loop body keeps
        // the instruction stream small (the unrolled 24-row pass missed the i-cache)
        int pO = NIL, sO = NIL, pK = NIL, sK = NIL, nab = 0, tot = 0;
#pragma unroll 1
        for (int w = 0; w < NWD; ++w) {
            uint32_t mk = 0, mo = 0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int j = 32 * w + 4 * kk + q;
                const uint32_t fj = FK(j, X);
                mk |= (fj == key) ? (1u << (4 * kk + q)) : 0u;
                mo |= (fj == okey) ? (1u << (4 * kk + q)) : 0u;
            }
            mk |= __shfl_xor_sync(msk, mk, 1);
            mo |= __shfl_xor_sync(msk, mo, 1);
            mk |= __shfl_xor_sync(msk, mk, 2);
            mo |= __shfl_xor_sync(msk, mo, 2);
            const uint32_t keep = live_in(w) & ~(((l >> 5) == w) ? (1u << (l & 31)) : 0u);
            mk &= keep;
            mo &= fresh ? 0u : keep;
            if (WARP) {
                uint32_t m1 = 0, m2 = 0;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int j = 32 * w + 4 * kk + q;
                    m1 |= (FK(j, O1) == k1) ? (1u << (4 * kk + q)) : 0u;
                    m2 |= (FK(j, O2) == k2) ? (1u << (4 * kk + q)) : 0u;
                }
                m1 |= __shfl_xor_sync(msk, m1, 1);
                m2 |= __shfl_xor_sync(msk, m2, 1);
                m1 |= __shfl_xor_sync(msk, m1, 2);
                m2 |= __shfl_xor_sync(msk, m2, 2);
                const uint32_t ex = ((excl >> 5) == w && excl >= 0) ? (1u << (excl & 31)) : 0u;
                two = two || ((((mk & (m1 | m2)) | (m1 & m2)) & keep & ~ex) != 0u);
            }
            if (act) {
                const uint32_t bl = below_in(l, w), ab = above_in(l, w);
                const uint32_t lo = mk & bl, hi = mk & ab, olo = mo & bl, ohi = mo & ab;
                if (lo) pK = 32 * w + 31 - __clz(lo);
                if (hi && sK == NIL) sK = 32 * w + __ffs(hi) - 1;
                if (olo) pO = 32 * w + 31 - __clz(olo);
                if (ohi && sO == NIL) sO = 32 * w + __ffs(ohi) - 1;
                nab += __popc(hi);
                tot += __popc(mk) - __popc(mo);
                const uint32_t own = 0x11111111u << q;
                for (uint32_t t = lo & ~olo & own; t; t &= t - 1u) LK(32 * w + __ffs(t) - 1) += 1u << (10 * X);
                for (uint32_t t = olo & ~lo & own; t; t &= t - 1u) LK(32 * w + __ffs(t) - 1) -= 1u << (10 * X);
            }
        }
        if (!act) return;
        if (owner(l)) {
            FK(l, X) = key;
            NXW(l) = set_byte(NXW(l), X, sK);
            LK(l) = (LK(l) & ~(1023u << (10 * X))) | ((uint32_t)nab << (10 * X));
        }
        if (pO != NIL && owner(pO)) NXW(pO) = set_byte(NXW(pO), X, sO);
        if (pK != NIL && owner(pK)) NXW(pK) = set_byte(NXW(pK), X, l);
        addn(X, tot);
    };
    // store a whole (normalised) row; only changed keys pay a class update.  Quad.
    auto write_row = [&](int l, const Row<P> &x, bool fresh) __attribute__((always_inline)) {
        const F o0 = FK(l, 0), o1 = FK(l, 1), o2 = FK(l, 2);
        if (fresh) {
            qsync();
            if (owner(l)) { LK(l) = 0; NXW(l) = 0xFFFFFFu; }
        } else {
            nnz_cur -= P::popd(o0) + P::popd(o1) + P::popd(o2);
        }
        nnz_cur += P::popd(x.u) + P::popd(x.v) + P::popd(x.w);
        qsync();
        // one inlined class update, looped over the roles (rare path: code size)
#pragma unroll 1
        for (int X = 0; X < 3; ++X) {
            const F kX = X == 0 ? x.u : (X == 1 ? x.v : P::abs(x.w));
            const F oX = X == 0 ? o0 : (X == 1 ? o1 : o2);
            bool dummy;
            if (fresh || kX != oX) change_class(std::false_type{}, l, X, oX, kX, fresh, true, -1, dummy);
            qsync();
        }
        set_wbit(l, P::first_neg(x.w));
        qsync();
    };
    // the flip commit: factor Y of row l becomes val (actual sign) if `act`; only this
    // factor can trigger PAPER:429 (R6).  Whole-warp collective.
    auto commit_factor = [&](bool act, int l, int Y, F val, int excl, bool &two) __attribute__((always_inline)) {
        const F old = FK(l, Y);
        const bool fn = P::first_neg(val);
        const F key = Y == 2 ? P::abs(val) : (fn ? P::neg(val) : val);
        if (act) {
            nnz_cur += P::popd(val) - P::popd(old);
            set_wbit(l, Y == 2 ? (uint32_t)fn : (wbit(l) ^ (uint32_t)fn));
        }
        change_class(std::true_type{}, l, Y, old, key, false, act && key != old, excl, two);
        __syncwarp();
    };
    // rows j (live, != l, > lmin) sharing two factor keys with row l (W up to sign), as a
    // row mask: one compare pass (quad)
    auto two_mask = [&](int l, int lmin, uint32_t (&cm)[NWD]) {
        const uint32_t u = FK(l, 0), v = FK(l, 1), w_ = FK(l, 2);
#pragma unroll
        for (int w = 0; w < NWD; ++w) {
            uint32_t m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int j = 32 * w + 4 * kk + q;
                const uint32_t bit = 1u << (4 * kk + q);
                m0 |= FK(j, 0) == u ? bit : 0u;
                m1 |= FK(j, 1) == v ? bit : 0u;
                m2 |= FK(j, 2) == w_ ? bit : 0u;
            }
            uint32_t m = (m0 & m1) | (m0 & m2) | (m1 & m2);
            m |= __shfl_xor_sync(qm, m, 1);
            m |= __shfl_xor_sync(qm, m, 2);
            cm[w] = m & live_in(w) & above_in(lmin, w) & ~(((l >> 5) == w) ? (1u << (l & 31)) : 0u);
        }
    };
    auto d_add = [&](int x) __attribute__((always_inline)) {
        if (dover) return;
        for (int k = 0; k < nD; ++k)
            if ((int)((dset >> (8 * k)) & 0xFFu) == x) return;
        if (nD == 6) { dover = true; return; }
        dset |= (uint64_t)x << (8 * nD);
        nD++;
    };

    // R14 remove(h) with the 2-entry worklist (entries == h dropped, r-1 -> h).  Quad.
    auto remove_row = [&](int h, int &wl0, int &wl1, int &nwl) __attribute__((always_inline)) {
        const int last = r - 1;
        int n2 = 0, x0 = 0, x1 = 0;
        if (nwl >= 1 && wl0 != h) { x0 = wl0; n2 = 1; }
        if (nwl >= 2 && wl1 != h) { if (n2 == 0) x0 = wl1; else x1 = wl1; n2++; }
        wl0 = x0; wl1 = x1; nwl = n2;
        nnz_cur -= P::popd(FK(h, 0)) + P::popd(FK(h, 1)) + P::popd(FK(h, 2));
        // h leaves its classes: its neighbours are relinked, the members below it lose a
        // later member (F(h) keeps the old keys until overwritten; the moves exclude h)
#pragma unroll 1
        for (int X = 0; X < 3; ++X) {
            const uint32_t o = FK(h, X);
            int pO = NIL, sO = NIL, tot = 0;
#pragma unroll 1
            for (int w = 0; w < NWD; ++w) {
                const uint32_t m = cmask(w, X, o, h, qm);
                const uint32_t lo = m & below_in(h, w), hi = m & above_in(h, w);
                if (lo) pO = 32 * w + 31 - __clz(lo);
                if (hi && sO == NIL) sO = 32 * w + __ffs(hi) - 1;
                tot += __popc(m);
                for (uint32_t t = lo & (0x11111111u << q); t; t &= t - 1u) LK(32 * w + __ffs(t) - 1) -= 1u << (10 * X);
            }
            if (pO != NIL && owner(pO)) NXW(pO) = set_byte(NXW(pO), X, sO);
            addn(X, -tot);
            qsync();
        }
        if (h != last) {
            // row `last` (the largest live index: the tail of each of its classes) moves
            // to h: in each class it moves down past its members in (h, last), which lose
            // it as a later member; pred / succ = its new neighbours, and the member that
            // pointed to it becomes a tail if it lies above h
            const F k0 = FK(last, 0), k1 = FK(last, 1), k2 = FK(last, 2);
            uint32_t nxw = 0xFFFFFFu, lc = 0;
#pragma unroll 1
            for (int X = 0; X < 3; ++X) {
                const uint32_t key = X == 0 ? k0 : (X == 1 ? k1 : k2);
                int pred = NIL, succ = NIL, tail = NIL, nab = 0;
#pragma unroll 1
                for (int w = 0; w < NWD; ++w) {
                    const uint32_t m = cmask(w, X, key, last, qm) & ~(((h >> 5) == w) ? (1u << (h & 31)) : 0u);
                    const uint32_t lo = m & below_in(h, w), hi = m & above_in(h, w);
                    if (lo) pred = 32 * w + 31 - __clz(lo);
                    if (hi && succ == NIL) succ = 32 * w + __ffs(hi) - 1;
                    if (m) tail = 32 * w + 31 - __clz(m);
                    nab += __popc(hi);
                    for (uint32_t t = hi & (0x11111111u << q); t; t &= t - 1u) LK(32 * w + __ffs(t) - 1) -= 1u << (10 * X);
                }
                if (tail != NIL && tail > h && owner(tail)) NXW(tail) = set_byte(NXW(tail), X, NIL);
                if (pred != NIL && owner(pred)) NXW(pred) = set_byte(NXW(pred), X, h);
                nxw = set_byte(nxw, X, succ);
                lc |= (uint32_t)nab << (10 * X);
                qsync();
            }
            const uint32_t sl = wbit(last);
            qsync();
            if (owner(h)) {
                FK(h, 0) = k0; FK(h, 1) = k1; FK(h, 2) = k2;
                NXW(h) = nxw | (sl << 24); LK(h) = lc;
            }
            if (nwl >= 1 && wl0 == last) wl0 = h;
            if (nwl >= 2 && wl1 == last) wl1 = h;
        }
        // D: entries == h dropped, last -> h
        uint64_t nd = 0;
        int nn = 0;
        for (int k = 0; k < nD; ++k) {
            int x = (int)((dset >> (8 * k)) & 0xFFu);
            if (x == h) continue;
            if (x == last) x = h;
            nd |= (uint64_t)x << (8 * nn);
            nn++;
        }
        dset = nd;
        nD = nn;
        if (owner(last)) LK(last) = 0;
        r--;
        qsync();
    };

    uint32_t c_draws = 0, c_flips = 0, c_red = 0, c_eok = 0, c_erej = 0, c_merge = 0, c_zero = 0,
             c_copy = 0, c_impr = 0;

    // R12 (local: worklist {a0, b0}) and R15 (global: lexicographic scan), exact; one
    // action per iteration so the merge / removal code is inlined once.  Quad.
    auto reduce_rows = [&](bool local, int a0, int b0) __attribute__((always_inline)) {
        int wl0 = a0, wl1 = b0, nwl = local ? 2 : 0;
        for (;;) {
            int rm0 = -1, rm1 = -1, wr = -1, lo = -1;
            bool push = false;
            Row<P> merged;
            merged.u = merged.v = merged.w = 0;
            int ib = 0, ie = 0;                  // rows i whose partners are searched
            if (local) {
                if (nwl == 0) break;
                const int t = wl0;
                wl0 = wl1;
                nwl--;
                if (t >= r) continue;
                if (row_zero(t)) { rm0 = t; c_zero++; } else { ib = t; ie = t + 1; }
            } else {
                for (int l = 0; l < r; ++l)
                    if (row_zero(l)) { rm0 = l; break; }
                // full lexicographic scan only after a load or a D overflow
                if (rm0 >= 0) c_zero++; else if (dover) { ib = 0; ie = r; }
            }
            if (rm0 < 0 && !local && !dover) {
                // R15 over D: the lexicographically first reducible pair involving a dirty
                // row (for a dirty d the first partner j in row order gives its first pair)
                int bk = 0x7fffffff;
#pragma unroll 1
                for (int k = 0; k < nD; ++k) {
                    const int d = (int)((dset >> (8 * k)) & 0xFFu);
                    uint32_t cm[NWD];
                    two_mask(d, -1, cm);
                    const Row<P> rd = read_row(d);
                    bool found = false;
#pragma unroll
                    for (int w = 0; w < NWD; ++w)
                        for (uint32_t c = cm[w]; c && !found; c &= c - 1u) {
                            const int j = 32 * w + __ffs(c) - 1;
                            Row<P> tmp;
                            if (!reducible<P>(rd, read_row(j), tmp)) continue;
                            found = true;
                            const int kk = (j < d ? j : d) * 256 + (j < d ? d : j);
                            bk = kk < bk ? kk : bk;
                        }
                }
                if (bk == 0x7fffffff) break;
                lo = bk >> 8;
                wr = lo;
                rm0 = bk & 255;
                reducible<P>(read_row(lo), read_row(rm0), merged);     // row i as base (R15)
                c_merge++;
                if (has_zero(merged)) { rm1 = lo; c_zero++; }
            } else if (rm0 < 0) {
                // the first (i, j) in (i, j) order with reducible(row i, row j): local over
                // all j != t, global over j > i (R12 / R15); one inlined search
#pragma unroll 1
                for (int i = ib; i < ie && wr < 0; ++i) {
                    uint32_t cm[NWD];
                    two_mask(i, local ? -1 : i, cm);
                    const Row<P> ri = read_row(i);
#pragma unroll
                    for (int w = 0; w < NWD; ++w)
                        for (uint32_t c = cm[w]; c && wr < 0; c &= c - 1u) {
                            const int j = 32 * w + __ffs(c) - 1;
                            if (!reducible<P>(ri, read_row(j), merged)) continue;
                            lo = i < j ? i : j;
                            wr = lo;
                            rm0 = i < j ? j : i;
                        }
                }
                if (wr < 0) {
                    if (local) continue;
                    break;
                }
                c_merge++;
                if (has_zero(merged)) { rm1 = lo; c_zero++; } else push = local;
            }
            if (wr >= 0) write_row(wr, merged, false);
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                const int h = k == 0 ? rm0 : rm1;
                if (h < 0) break;
                remove_row(h, wl0, wl1, nwl);
            }
            if (!local && wr >= 0 && rm1 < 0) d_add(lo);       // the merged row (R15) is dirty
            if (push) {
                wl1 = wl0;
                wl0 = lo;
                nwl++;
            }
        }
    };

    // R16 expand (plus / split), words from Philox block 1 of this step.  Quad.
    auto expand = [&]() __attribute__((always_inline)) -> bool {
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
        }
        // rows i, j (plus only) and the new row r; one inlined write_row
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
            if (t == 1 && !plus) continue;
            if (t == 2) r++;
            const int l = t == 0 ? i : (t == 1 ? j : r - 1);
            Row<P> x;
            x.u = t == 0 ? ri.u : (t == 1 ? rj.u : rn.u);
            x.v = t == 0 ? ri.v : (t == 1 ? rj.v : rn.v);
            x.w = t == 0 ? ri.w : (t == 1 ? rj.w : rn.w);
            write_row(l, x, t == 2);
            d_add(l);
        }
        return true;
    };

    // store the current rows in plane layout (own rows; zeros above r up to R)
    // rows l < n (n >= r; zeros for r <= l < n)
    auto store_rows = [&](uint64_t *dst, int n) __attribute__((always_inline)) {
        for (int l = q; l < n; l += 4) {
            const bool lv = l < r;
            const F u = lv ? FK(l, 0) : 0, v = lv ? FK(l, 1) : 0, w = lv ? fac(l, 2) : 0;
            dst[0 * R + l] = P::dig(u); dst[1 * R + l] = P::sgn(u);
            dst[2 * R + l] = P::dig(v); dst[3 * R + l] = P::sgn(v);
            dst[4 * R + l] = P::dig(w); dst[5 * R + l] = P::sgn(w);
        }
    };
    // R19 verify queue entry: the current rows (== the new best)
    auto enqueue_verify = [&]() __attribute__((always_inline)) {
        unsigned slot = 0;
        if (q == 0) slot = atomicAdd(a.q_count, 1u);
        slot = __shfl_sync(qm, slot, qb);
        if (slot < a.q_cap) {
            store_rows(a.q_planes + (size_t)slot * FG_PLANES * R, r);   // the verifier reads rank rows
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

    const uint32_t nsteps = nsteps_task;
#pragma unroll 1
    for (uint32_t it = 0; it < nsteps; ++it, ++step) {
        // Philox (R8): lane 0 block 0 (draw 0 + Bernoulli words), lanes 1 and 3 block 2
        // (draws 1-4), lane 2 block 3 (draws 5-8)
        uint32_t cb = q == 0 ? 0u : (q == 2 ? 3u : 2u);
        uint32_t c0, c1, c2, c3;
        philox_block(seed, step, wid, cb, c0, c1, c2, c3);
        const uint32_t bern = __shfl_sync(FULL, (c1 < a.thr_eq ? 1u : 0u) | (c2 < a.thr_reduce ? 2u : 0u) |
                                                    (c3 < a.thr_expand ? 4u : 0u), qb);
        uint32_t flags = 0;
        int alpha = 0, beta = 0;
        uint32_t draws = 0;
        bool ok = false;
        const uint32_t nU = nCU, nV = nCV, nW = nCW;
        const uint32_t nC = nU + nV + nW;
        int e_Y = 0, e_Z = 0;
        F e_ny = 0, e_nz = 0;
        // R10 group prefix of the later counts: lane q sums its two rows of group g
        {
            uint32_t bu = 0, bv = 0, bwc = 0;
#pragma unroll 2
            for (int g = 0; g < NG; ++g) {
                uint32_t s2 = LK(8 * g + q) + LK(8 * g + 4 + q);    // fields <= 2 x 127
                s2 += __shfl_xor_sync(FULL, s2, 1);
                s2 += __shfl_xor_sync(FULL, s2, 2);                 // group total, fields <= 1016
                if (q == (g & 3)) {
                    GK(g, 0) = bu | (bv << 16);
                    GK(g, 1) = bwc;
                }
                bu += s2 & 1023u;
                bv += (s2 >> 10) & 1023u;
                bwc += s2 >> 20;
            }
            __syncwarp();
        }
        // R11 try_flip: round t, lane q evaluates draw 4t+q (full-warp ballots)
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
            // group: the last g with G_X(g) <= qq (G nondecreasing, G(0) = 0)
            int g = 0;
#pragma unroll
            for (int st = 8; st >= 1; st >>= 1) {
                if (g + st < NG) {
                    const uint32_t w0 = GK(g + st, 0), w1 = GK(g + st, 1);
                    const uint32_t v = X == 0 ? (w0 & 0xFFFFu) : (X == 1 ? (w0 >> 16) : w1);
                    g += v <= qq ? st : 0;
                }
            }
            const uint32_t g0w = GK(g, 0), g1w = GK(g, 1);
            uint32_t acc = X == 0 ? (g0w & 0xFFFFu) : (X == 1 ? (g0w >> 16) : g1w);
            // row inside the group: accumulate later counts until past qq
            int i = 8 * g;
#pragma unroll 1
            for (int s = 0; s < 8; ++s) {
                const uint32_t lx = (LK(8 * g + s) >> (10 * X)) & 1023u;
                if (acc + lx > qq) { i = 8 * g + s; break; }
                acc += lx;
            }
            // j: the (qq - acc)-th later member of row i's X class
            int j = i;
            for (uint32_t hops = qq - acc + 1; hops; --hops) j = nxt(j, X);
            j = j < RM ? j : 0;                        // (quads not searching: any row)
            const int al = d ? j : i, be = d ? i : j;
            // (Y,Z) = (V,W) / (W,U) / (U,V) for X = U / V / W, swapped if e
            const uint32_t yz = (0x148269u >> (4 * (2 * X + e))) & 15u;
            const int Y = yz & 3, Z = yz >> 2;
            const bool sneg = P::RING == FG_ZT && X == 2 && (wbit(al) ^ wbit(be));
            const F yb = fac(be, Y);
            bool v = searching && att < kf;
            const F ny = P::add(fac(al, Y), sneg ? P::neg(yb) : yb, v);   // y_a + s y_b
            const F nz = P::sub(fac(be, Z), fac(al, Z), v);             // z_b - z_a
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
        // (one inlined commit, looped over the two touched rows: code size)
        bool two_ab = false;            // a touched row shares two factors with another row
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            bool two;
            commit_factor(ok, c ? beta : alpha, c ? e_Z : e_Y, c ? e_nz : e_ny, c ? -1 : beta, two);
            two_ab = two_ab || two;
        }

        if (!ok) {
            // expand; continue
            const bool ex = expand();
            c_eok += ex;
            c_erej += !ex;
            flags |= 2u | (ex ? 64u : 0u);
            alpha = beta = 0;
        } else {
            c_flips++;
            flags |= 1u;
            // ---- R12 local reduction (exact skip), PAPER:310-313 acceptance
            // reduce (R15, exact skip) -- one loop so the reduction code is inlined once ----
            // alpha's test ran before beta's commit and left beta out: the pair itself is
            // checked here (class keys compare W up to sign)
            const int same = (FK(alpha, 0) == FK(beta, 0)) + (FK(alpha, 1) == FK(beta, 1)) +
                             (FK(alpha, 2) == FK(beta, 2));
            const bool need_local = P::zero(e_ny) || P::zero(e_nz) || two_ab || same >= 2;
#pragma unroll 1
            for (int ph = 0; ph < 2; ++ph) {
                const bool run = ph == 0 ? need_local : ((bern & 2u) && (dover || nD > 0));
                if (run) reduce_rows(ph == 0, alpha, beta);
                if (ph == 0) {
                    const bool strict = r < best;
                    if (strict || (r == best && (bern & 1u))) {
                        // rows >= the previous best rank are already zero in HBM
                        store_rows(bw, best);
                        best = r;
                        best_adds = nnz_cur - 2 * r - a.mp;
                        c_copy++;
                        flags |= 4u;
                        if (strict) {
                            flags |= 8u;
                            c_impr++;
                            enqueue_verify();
                        }
                    }
                    if (bern & 2u) {
                        c_red++;
                        flags |= 16u;
                    }
                } else if (run) {
                    dset = 0;                   // reduce_all ran to completion: clean
                    nD = 0;
                    dover = false;
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
        const uint64_t ev = (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)best << 10) | ((uint64_t)flags << 20) |
                            ((uint64_t)alpha << 32) | ((uint64_t)beta << 42) | ((uint64_t)draws << 52);
        digest = (digest ^ ev) * 0x100000001b3ULL;
        digest ^= digest >> 32;
    }

    // ---------------- save the image for the next chunk of this launch ----------------
    if (valid && img && chunk + 1 < a.chunks) {
        qsync();
#pragma unroll 1
        for (int k = q; k < SLOTS; k += 4) img[k] = S[k * 8];
        if (q == 0) {
            img[SLOTS] = (uint32_t)nnz_cur;
            img[SLOTS + 1] = nCU; img[SLOTS + 2] = nCV; img[SLOTS + 3] = nCW;
            img[SLOTS + 4] = (uint32_t)dset; img[SLOTS + 5] = (uint32_t)(dset >> 32);
            img[SLOTS + 6] = (uint32_t)nD | (dover ? 0x100u : 0u);
        }
    }
    // ---------------- last chunk: store own rows; best additions from the best rows ----------------
    // (earlier chunks hand the state over in the image only)
    __syncwarp();
    const bool last_chunk = chunk + 1 >= a.chunks;
    if (valid && last_chunk) store_rows(a.cur + (size_t)wk * FG_PLANES * R, R);
    int best_nnz = 0;
    for (int l = q; l < R && valid && last_chunk; l += 4)
        if (l < best) best_nnz += __popcll(bw[0 * R + l]) + __popcll(bw[2 * R + l]) + __popcll(bw[4 * R + l]);
    best_nnz += __shfl_xor_sync(qm, best_nnz, 1);
    best_nnz += __shfl_xor_sync(qm, best_nnz, 2);
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
    // this group's chunk is stored: release the next chunk
    __syncwarp();
    __threadfence();
    if (lane == 0) atomicExch(a.task_done + grp, chunk + 1);
    __syncwarp();
    }   // task loop
#undef FK
#undef NXW
#undef LK
#undef GK
}

template <class P, int NWD>
cudaError_t launch_ql(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    constexpr int RM = 32 * NWD;
    const size_t smem = (size_t)(5 * RM + 2 * (RM / 8)) * 8 * 4 * (QL_THREADS / 32);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(walk_ql<P, NWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, walk_ql<P, NWD>, QL_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) bps = 1;
    const int64_t resident = (int64_t)num_sms * bps * (QL_THREADS / 32);   // warps
    const int64_t groups = (a.num_walkers + 7) / 8;
    WalkArgs b = a;
    // one wave: one task per warp; more: 8 step chunks per group over persistent warps
    b.chunks = (groups > resident && a.steps >= 64) ? 8u : 1u;
    if (const char *ev = getenv("FG_QL_CHUNKS")) {               // tests: force chunking
        const long k = strtol(ev, nullptr, 10);
        if (k >= 1 && k <= 64) b.chunks = (uint32_t)k;
    }
    if ((uint64_t)b.chunks > a.steps) b.chunks = a.steps > 0 ? (uint32_t)a.steps : 1u;
    b.chunk_steps = (a.steps + b.chunks - 1) / b.chunks;
    const int64_t warps = groups < resident ? groups : resident;
    const int64_t blocks = (warps + QL_THREADS / 32 - 1) / (QL_THREADS / 32);
    walk_ql<P, NWD><<<(unsigned)blocks, QL_THREADS, smem, st>>>(b);
    return cudaGetLastError();
}

template <class P>
cudaError_t launch_ql_r(const WalkArgs &a, int num_sms, cudaStream_t st)
{
    if (a.R <= 64) return launch_ql<P, 2>(a, num_sms, st);
    if (a.R <= 96) return launch_ql<P, 3>(a, num_sms, st);
    return launch_ql<P, 4>(a, num_sms, st);
}

}  // namespace

cudaError_t fg_launch_walk_ql(int kind, const WalkArgs &a, int num_sms, cudaStream_t st)
{
    switch (kind) {
    case FG_K_QL_P16: return launch_ql_r<P16>(a, num_sms, st);
    case FG_K_QL_Z2: return launch_ql_r<PZ2>(a, num_sms, st);
    default: return cudaErrorInvalidValue;
    }
}
