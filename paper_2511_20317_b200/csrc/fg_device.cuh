// fg_device.cuh -- device primitives of the walk: bit-sliced ternary vectors
// (PAPER:388-424), sign normalisation, Philox4x32-10 (reading R8).
// Independent of oracle/ (no shared code).
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

// ---- ternary vector: (digits, signs), signs subset of digits ----
template <typename T> struct Tv { T d, s; };

template <typename T> __device__ __forceinline__ bool eq(Tv<T> a, Tv<T> b)
{
    return a.d == b.d && a.s == b.s;
}
// a == -b, a != 0 (PAPER:421 with zero excluded, R4)
template <typename T> __device__ __forceinline__ bool negeq(Tv<T> a, Tv<T> b)
{
    return a.d == b.d && a.s == (b.d ^ b.s) && a.d != 0;
}
template <typename T> __device__ __forceinline__ Tv<T> neg(Tv<T> a) { return {a.d, a.d ^ a.s}; }

// a + b with the ternary-safety flag (signs simplified under s subset d)
template <int RING, typename T> __device__ __forceinline__ Tv<T> add(Tv<T> a, Tv<T> b, bool &ok)
{
    const T d = a.d ^ b.d;
    if (RING == FG_Z2) return {d, (T)0};
    ok = ok && ((a.d & b.d & ~(a.s ^ b.s)) == 0);
    return {d, (a.s | b.s) & d};
}
// a - b = a + (-b)
template <int RING, typename T> __device__ __forceinline__ Tv<T> sub(Tv<T> a, Tv<T> b, bool &ok)
{
    if (RING == FG_Z2) return {a.d ^ b.d, (T)0};
    return add<RING, T>(a, neg(b), ok);
}
template <int RING, typename T> __device__ __forceinline__ bool distinct(Tv<T> a, Tv<T> b)
{
    if (eq(a, b)) return false;
    if (RING == FG_ZT && negeq(a, b)) return false;
    return true;
}

template <typename T> struct Row { Tv<T> u, v, w; };

template <typename T> __device__ __forceinline__ Tv<T> get(const Row<T> &r, int X)
{
    Tv<T> o;
    o.d = X == 0 ? r.u.d : (X == 1 ? r.v.d : r.w.d);
    o.s = X == 0 ? r.u.s : (X == 1 ? r.v.s : r.w.s);
    return o;
}
template <typename T> __device__ __forceinline__ void set(Row<T> &r, int X, Tv<T> x, bool pred)
{
    if (pred && X == 0) r.u = x;
    if (pred && X == 1) r.v = x;
    if (pred && X == 2) r.w = x;
}
template <typename T> __device__ __forceinline__ bool has_zero(const Row<T> &r)
{
    return r.u.d == 0 || r.v.d == 0 || r.w.d == 0;
}

// PAPER:429 per row (R6): first nonzero of u, then v, made positive; w absorbs.
// lowbit(d) = d & -d is the first nonzero position.
template <int RING, typename T> __device__ __forceinline__ void normalize(Row<T> &r)
{
    if (RING != FG_ZT) return;
    const T nu = (r.u.s & (r.u.d & (T)(0 - r.u.d))) ? ~(T)0 : (T)0;
    r.u.s ^= r.u.d & nu;
    r.w.s ^= r.w.d & nu;
    const T nv = (r.v.s & (r.v.d & (T)(0 - r.v.d))) ? ~(T)0 : (T)0;
    r.v.s ^= r.v.d & nv;
    r.w.s ^= r.w.d & nv;
}

template <typename T, bool K16> __device__ __forceinline__ Tv<T> shfl(Tv<T> x, int src)
{
    Tv<T> o;
    if constexpr (sizeof(T) == 4 && K16) {
        const uint32_t k = __shfl_sync(FULL, (uint32_t)(x.d | (x.s << 16)), src);
        o.d = k & 0xffffu;
        o.s = k >> 16;
    } else {
        o.d = __shfl_sync(FULL, x.d, src);
        o.s = __shfl_sync(FULL, x.s, src);
    }
    return o;
}
template <int RING, typename T, bool K16> __device__ __forceinline__ Row<T> shfl_row(const Row<T> &r, int src)
{
    Row<T> o;
    if (RING == FG_Z2) {
        o.u.d = __shfl_sync(FULL, r.u.d, src); o.u.s = 0;
        o.v.d = __shfl_sync(FULL, r.v.d, src); o.v.s = 0;
        o.w.d = __shfl_sync(FULL, r.w.d, src); o.w.s = 0;
    } else {
        o.u = shfl<T, K16>(r.u, src);
        o.v = shfl<T, K16>(r.v, src);
        o.w = shfl<T, K16>(r.w, src);
    }
    return o;
}

// lanes holding the same factor value (all 32 lanes participate)
template <int RING, typename T, bool K16> __device__ __forceinline__ unsigned match(Tv<T> x)
{
    if constexpr (sizeof(T) == 4) {
        if (RING == FG_Z2) return __match_any_sync(FULL, (uint32_t)x.d);
        if constexpr (K16) return __match_any_sync(FULL, (uint32_t)(x.d | (x.s << 16)));
        else return __match_any_sync(FULL, (unsigned long long)x.d | ((unsigned long long)x.s << 32));
    } else {
        if (RING == FG_Z2) return __match_any_sync(FULL, (unsigned long long)x.d);
        return __match_any_sync(FULL, (unsigned long long)x.d) &
               __match_any_sync(FULL, (unsigned long long)x.s);
    }
}

// R13 reducible(i, j) with row i = ri, row j = rj; merged = row i with C replaced
// (x_C[i] + sigma x_C[j]), normalised.  Role pairs (A,B,C) in the order
// (U,V,W), (U,W,V), (V,W,U) (PAPER:233-238 under any permutation).
template <int RING, typename T> __device__ __forceinline__ bool reducible(const Row<T> &ri, const Row<T> &rj,
                                                                          Row<T> &merged)
{
    // (U,V,W): u and v shared, w merged (sigma = +1: B = V)
    if (eq(ri.u, rj.u) && eq(ri.v, rj.v)) {
        bool ok = true;
        Tv<T> c = add<RING, T>(ri.w, rj.w, ok);
        if (ok) { merged = ri; merged.w = c; normalize<RING, T>(merged); return true; }
    }
    // (U,W,V): u shared, w shared up to sign, v merged
    if (eq(ri.u, rj.u)) {
        int sg = eq(ri.w, rj.w) ? 1 : ((RING == FG_ZT && negeq(ri.w, rj.w)) ? -1 : 0);
        if (sg) {
            bool ok = true;
            Tv<T> c = add<RING, T>(ri.v, sg > 0 ? rj.v : neg(rj.v), ok);
            if (ok) { merged = ri; merged.v = c; normalize<RING, T>(merged); return true; }
        }
    }
    // (V,W,U): v shared, w shared up to sign, u merged
    if (eq(ri.v, rj.v)) {
        int sg = eq(ri.w, rj.w) ? 1 : ((RING == FG_ZT && negeq(ri.w, rj.w)) ? -1 : 0);
        if (sg) {
            bool ok = true;
            Tv<T> c = add<RING, T>(ri.u, sg > 0 ? rj.u : neg(rj.u), ok);
            if (ok) { merged = ri; merged.u = c; normalize<RING, T>(merged); return true; }
        }
    }
    return false;
}

}  // namespace fgd
