// fg_device.cuh -- device primitives of the walk: bit-sliced ternary vectors
// (PAPER:388-424), sign normalisation, Philox4x32-10 (reading R8).
// Independent of oracle/ (no shared code).
//
// A factor (one of u, v, w of a rank-one term) is a ternary vector of <= 64
// elements held as bit planes (digits = nonzero, signs = negative, signs subset of
// digits).  Three register layouts ("policies"), chosen per format:
//   P16  Z_T, <= 16 elements: ONE u32 key = digits | signs << 16.  Equality is one
//        compare, a shuffle moves a whole factor, the key is the MATCH value.
//   P32  Z_T, <= 32 elements: two u32 words (digits, signs).
//   PZ2  Z_2, <= 32 elements: one u32 word (digits); +,- are XOR.
#pragma once
#include <cstdint>
#include "fg_internal.h"

namespace fgd {

constexpr unsigned FULL = 0xffffffffu;

// ---- Philox4x32-10 (Random123 constants), R8 ----
__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                       uint32_t k0, uint32_t k1, uint32_t &o0, uint32_t &o1,
                                       uint32_t &o2, uint32_t &o3)
{
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        if (i) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// block b of step s of walker wid under key seed: counter (s_lo, s_hi, wid, b)
__device__ __forceinline__ void philox_block(uint64_t seed, uint64_t s, uint32_t wid, uint32_t b,
                                             uint32_t &o0, uint32_t &o1, uint32_t &o2, uint32_t &o3)
{
    philox((uint32_t)s, (uint32_t)(s >> 32), wid, b, (uint32_t)seed, (uint32_t)(seed >> 32),
           o0, o1, o2, o3);
}

// ------------------------------------------------------------------------------
// P16: key = digits | signs << 16
struct P16 {
    typedef uint32_t F;
    static constexpr int RING = FG_ZT;
    static __device__ __forceinline__ F make(uint64_t d, uint64_t s) { return (uint32_t)d | ((uint32_t)s << 16); }
    static __device__ __forceinline__ uint64_t dig(F a) { return a & 0xffffu; }
    static __device__ __forceinline__ uint64_t sgn(F a) { return a >> 16; }
    static __device__ __forceinline__ bool zero(F a) { return (a & 0xffffu) == 0; }
    static __device__ __forceinline__ bool eq(F a, F b) { return a == b; }
    // a == -b, a != 0 (PAPER:421 with zero excluded, R4)
    static __device__ __forceinline__ bool negeq(F a, F b)
    {
        const uint32_t d = a & 0xffffu;
        return d != 0 && (a ^ b) == (d << 16);
    }
    static __device__ __forceinline__ F neg(F a) { return a ^ (a << 16); }
    // first nonzero made positive (the W-up-to-sign key)
    static __device__ __forceinline__ F abs(F a)
    {
        const uint32_t d = a & 0xffffu;
        const uint32_t lb = d & (0u - d);
        return (a & (lb << 16)) ? neg(a) : a;
    }
    static __device__ __forceinline__ bool first_neg(F a)
    {
        const uint32_t d = a & 0xffffu;
        return (a & ((d & (0u - d)) << 16)) != 0;
    }
    // a + b with the ternary-safety flag (signs simplified under s subset d)
    static __device__ __forceinline__ F add(F a, F b, bool &ok)
    {
        const uint32_t x = a ^ b;
        const uint32_t d = x & 0xffffu;
        const uint32_t s = ((a | b) >> 16) & d;
        ok = ok && ((a & b & ~(x >> 16) & 0xffffu) == 0);
        return __byte_perm(d, s, 0x5410);
    }
    static __device__ __forceinline__ F sub(F a, F b, bool &ok) { return add(a, neg(b), ok); }
    static __device__ __forceinline__ F shfl(F a, int src) { return __shfl_sync(FULL, a, src); }
    static __device__ __forceinline__ F shflm(unsigned m, F a, int src) { return __shfl_sync(m, a, src); }
    static __device__ __forceinline__ unsigned match(F a) { return __match_any_sync(FULL, a); }
    static __device__ __forceinline__ F sel(bool p, F a, F b) { return p ? a : b; }
    static __device__ __forceinline__ int popd(F a) { return __popc(a & 0xffffu); }
};

// P32: (digits, signs) in two words
struct P32 {
    struct F { uint32_t d, s; };
    static constexpr int RING = FG_ZT;
    static __device__ __forceinline__ F make(uint64_t d, uint64_t s) { return {(uint32_t)d, (uint32_t)s}; }
    static __device__ __forceinline__ uint64_t dig(F a) { return a.d; }
    static __device__ __forceinline__ uint64_t sgn(F a) { return a.s; }
    static __device__ __forceinline__ bool zero(F a) { return a.d == 0; }
    static __device__ __forceinline__ bool eq(F a, F b) { return a.d == b.d && a.s == b.s; }
    static __device__ __forceinline__ bool negeq(F a, F b) { return a.d == b.d && a.s == (b.d ^ b.s) && a.d != 0; }
    static __device__ __forceinline__ F neg(F a) { return {a.d, a.d ^ a.s}; }
    static __device__ __forceinline__ F abs(F a) { return (a.s & (a.d & (0u - a.d))) ? neg(a) : a; }
    static __device__ __forceinline__ bool first_neg(F a) { return (a.s & (a.d & (0u - a.d))) != 0; }
    static __device__ __forceinline__ F add(F a, F b, bool &ok)
    {
        const uint32_t d = a.d ^ b.d;
        ok = ok && ((a.d & b.d & ~(a.s ^ b.s)) == 0);
        return {d, (a.s | b.s) & d};
    }
    static __device__ __forceinline__ F sub(F a, F b, bool &ok) { return add(a, neg(b), ok); }
    static __device__ __forceinline__ F shfl(F a, int src)
    {
        return {__shfl_sync(FULL, a.d, src), __shfl_sync(FULL, a.s, src)};
    }
    static __device__ __forceinline__ F shflm(unsigned m, F a, int src)
    {
        return {__shfl_sync(m, a.d, src), __shfl_sync(m, a.s, src)};
    }
    static __device__ __forceinline__ unsigned match(F a)
    {
        return __match_any_sync(FULL, (unsigned long long)a.d | ((unsigned long long)a.s << 32));
    }
    static __device__ __forceinline__ F sel(bool p, F a, F b) { return {p ? a.d : b.d, p ? a.s : b.s}; }
    static __device__ __forceinline__ int popd(F a) { return __popc(a.d); }
};

// PZ2: digits only, arithmetic mod 2
struct PZ2 {
    typedef uint32_t F;
    static constexpr int RING = FG_Z2;
    static __device__ __forceinline__ F make(uint64_t d, uint64_t) { return (uint32_t)d; }
    static __device__ __forceinline__ uint64_t dig(F a) { return a; }
    static __device__ __forceinline__ uint64_t sgn(F) { return 0; }
    static __device__ __forceinline__ bool zero(F a) { return a == 0; }
    static __device__ __forceinline__ bool eq(F a, F b) { return a == b; }
    static __device__ __forceinline__ bool negeq(F, F) { return false; }
    static __device__ __forceinline__ F neg(F a) { return a; }
    static __device__ __forceinline__ F abs(F a) { return a; }
    static __device__ __forceinline__ bool first_neg(F) { return false; }
    static __device__ __forceinline__ F add(F a, F b, bool &) { return a ^ b; }
    static __device__ __forceinline__ F sub(F a, F b, bool &) { return a ^ b; }
    static __device__ __forceinline__ F shfl(F a, int src) { return __shfl_sync(FULL, a, src); }
    static __device__ __forceinline__ F shflm(unsigned m, F a, int src) { return __shfl_sync(m, a, src); }
    static __device__ __forceinline__ unsigned match(F a) { return __match_any_sync(FULL, a); }
    static __device__ __forceinline__ F sel(bool p, F a, F b) { return p ? a : b; }
    static __device__ __forceinline__ int popd(F a) { return __popc(a); }
};

// P64: Z_T, <= 64 elements: (digits, signs) as two u64 words
struct P64 {
    struct F { uint64_t d, s; };
    static constexpr int RING = FG_ZT;
    static __device__ __forceinline__ F make(uint64_t d, uint64_t s) { return {d, s}; }
    static __device__ __forceinline__ uint64_t dig(F a) { return a.d; }
    static __device__ __forceinline__ uint64_t sgn(F a) { return a.s; }
    static __device__ __forceinline__ bool zero(F a) { return a.d == 0; }
    static __device__ __forceinline__ bool eq(F a, F b) { return a.d == b.d && a.s == b.s; }
    static __device__ __forceinline__ bool negeq(F a, F b) { return a.d == b.d && a.s == (b.d ^ b.s) && a.d != 0; }
    static __device__ __forceinline__ F neg(F a) { return {a.d, a.d ^ a.s}; }
    static __device__ __forceinline__ F abs(F a) { return (a.s & (a.d & (0ull - a.d))) ? neg(a) : a; }
    static __device__ __forceinline__ bool first_neg(F a) { return (a.s & (a.d & (0ull - a.d))) != 0; }
    static __device__ __forceinline__ F add(F a, F b, bool &ok)
    {
        const uint64_t d = a.d ^ b.d;
        ok = ok && ((a.d & b.d & ~(a.s ^ b.s)) == 0);
        return {d, (a.s | b.s) & d};
    }
    static __device__ __forceinline__ F sub(F a, F b, bool &ok) { return add(a, neg(b), ok); }
    static __device__ __forceinline__ F shfl(F a, int src)
    {
        return {__shfl_sync(FULL, a.d, src), __shfl_sync(FULL, a.s, src)};
    }
    static __device__ __forceinline__ F sel(bool p, F a, F b) { return {p ? a.d : b.d, p ? a.s : b.s}; }
    static __device__ __forceinline__ int popd(F a) { return __popcll(a.d); }
};

// PZ64: Z_2, <= 64 elements
struct PZ64 {
    typedef uint64_t F;
    static constexpr int RING = FG_Z2;
    static __device__ __forceinline__ F make(uint64_t d, uint64_t) { return d; }
    static __device__ __forceinline__ uint64_t dig(F a) { return a; }
    static __device__ __forceinline__ uint64_t sgn(F) { return 0; }
    static __device__ __forceinline__ bool zero(F a) { return a == 0; }
    static __device__ __forceinline__ bool eq(F a, F b) { return a == b; }
    static __device__ __forceinline__ bool negeq(F, F) { return false; }
    static __device__ __forceinline__ F neg(F a) { return a; }
    static __device__ __forceinline__ F abs(F a) { return a; }
    static __device__ __forceinline__ bool first_neg(F) { return false; }
    static __device__ __forceinline__ F add(F a, F b, bool &) { return a ^ b; }
    static __device__ __forceinline__ F sub(F a, F b, bool &) { return a ^ b; }
    static __device__ __forceinline__ F shfl(F a, int src) { return __shfl_sync(FULL, a, src); }
    static __device__ __forceinline__ F sel(bool p, F a, F b) { return p ? a : b; }
    static __device__ __forceinline__ int popd(F a) { return __popcll(a); }
};

template <class P> struct Row { typename P::F u, v, w; };

// role X in {0: U, 1: V, 2: W}, branch-free
template <class P> __device__ __forceinline__ typename P::F get(const Row<P> &r, int X)
{
    return P::sel(X & 2, r.w, P::sel(X & 1, r.v, r.u));
}
template <class P> __device__ __forceinline__ void set(Row<P> &r, int X, typename P::F x, bool pred)
{
    r.u = P::sel(pred && X == 0, x, r.u);
    r.v = P::sel(pred && X == 1, x, r.v);
    r.w = P::sel(pred && X == 2, x, r.w);
}
template <class P> __device__ __forceinline__ bool has_zero(const Row<P> &r)
{
    return P::zero(r.u) || P::zero(r.v) || P::zero(r.w);
}
template <class P> __device__ __forceinline__ bool distinct(typename P::F a, typename P::F b)
{
    return !P::eq(a, b) && !P::negeq(a, b);
}

// PAPER:429 per row (R6): first nonzero of u, then v, made positive; w absorbs.
template <class P> __device__ __forceinline__ void normalize(Row<P> &r)
{
    if (P::RING != FG_ZT) return;
    const bool nu = P::first_neg(r.u);
    r.u = P::sel(nu, P::neg(r.u), r.u);
    r.w = P::sel(nu, P::neg(r.w), r.w);
    const bool nv = P::first_neg(r.v);
    r.v = P::sel(nv, P::neg(r.v), r.v);
    r.w = P::sel(nv, P::neg(r.w), r.w);
}

template <class P> __device__ __forceinline__ Row<P> shfl_row(const Row<P> &r, int src)
{
    Row<P> o;
    o.u = P::shfl(r.u, src);
    o.v = P::shfl(r.v, src);
    o.w = P::shfl(r.w, src);
    return o;
}

// R13 reducible(i, j) with row i = ri, row j = rj; merged = row i with C replaced
// (x_C[i] + sigma x_C[j]), normalised.  Role pairs (A,B,C) in the order
// (U,V,W), (U,W,V), (V,W,U) (PAPER:233-238 under any permutation).
template <class P> __device__ __forceinline__ bool reducible(const Row<P> &ri, const Row<P> &rj, Row<P> &merged)
{
    if (P::eq(ri.u, rj.u) && P::eq(ri.v, rj.v)) {
        bool ok = true;
        const typename P::F c = P::add(ri.w, rj.w, ok);
        if (ok) { merged = ri; merged.w = c; normalize<P>(merged); return true; }
    }
    const int sg = P::eq(ri.w, rj.w) ? 1 : (P::negeq(ri.w, rj.w) ? -1 : 0);
    if (sg && P::eq(ri.u, rj.u)) {
        bool ok = true;
        const typename P::F c = P::add(ri.v, sg > 0 ? rj.v : P::neg(rj.v), ok);
        if (ok) { merged = ri; merged.v = c; normalize<P>(merged); return true; }
    }
    if (sg && P::eq(ri.v, rj.v)) {
        bool ok = true;
        const typename P::F c = P::add(ri.u, sg > 0 ? rj.u : P::neg(rj.u), ok);
        if (ok) { merged = ri; merged.u = c; normalize<P>(merged); return true; }
    }
    return false;
}

}  // namespace fgd
