"""ctypes binding of liboracle.so -- TEST INFRASTRUCTURE ONLY (see oracle.h).

Argument marshalling only; every computation is in the C files next to this one.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
SOURCES = ["philox_bits.c", "scheme.c", "walk.c", "meta.c", "lift.c"]
NCNT = 12
CNT_NAMES = ["steps", "draws", "flips", "flip_fail", "expand_ok", "expand_reject", "merges",
             "zero_removed", "best_copies", "improvements", "reduce_calls", "verify_fail"]


def build_oracle(force: bool = False) -> str:
    srcs = [os.path.join(HERE, s) for s in SOURCES]
    deps = srcs + [os.path.join(HERE, "oracle.h")]
    if not force and os.path.exists(ORACLE_SO):
        t = os.path.getmtime(ORACLE_SO)
        if all(os.path.getmtime(s) <= t for s in deps):
            return ORACLE_SO
    cmd = ["gcc", "-O2", "-std=gnu99", "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra",
           "-Wno-unused-parameter", "-o", ORACLE_SO] + srcs
    subprocess.check_call(cmd)
    return ORACLE_SO


class OracleParams(C.Structure):
    _fields_ = [("k_flip", C.c_uint32), ("thr_accept_eq", C.c_uint32),
                ("thr_reduce", C.c_uint32), ("thr_expand", C.c_uint32),
                ("expand_slack", C.c_int32), ("mode", C.c_uint32)]

    @classmethod
    def default(cls, **kw):
        d = dict(k_flip=16, thr_accept_eq=42949672, thr_reduce=2147483648,
                 thr_expand=42949672, expand_slack=2, mode=0)
        d.update(kw)
        return cls(**d)


class _Walker(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("p", C.c_int), ("ring", C.c_int),
                ("R", C.c_int), ("len", C.c_int * 3), ("r", C.c_int), ("best_r", C.c_int),
                ("best_adds", C.c_int),
                ("walker_id", C.c_uint64), ("step", C.c_uint64), ("digest", C.c_uint64),
                ("cnt", C.c_uint64 * NCNT), ("rows", C.c_void_p), ("best", C.c_void_p)]


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Thin wrapper; ``lib`` exposes the raw C functions."""

    def __init__(self):
        build_oracle()
        lib = C.CDLL(ORACLE_SO)
        self.lib = lib
        vp, i32, u64, i64 = C.c_void_p, C.c_int, C.c_uint64, C.c_int64
        lib.or_word.restype = C.c_uint32
        lib.or_word.argtypes = [u64, u64, u64, i32]
        lib.or_philox4x32_10.argtypes = [vp, vp, vp]
        lib.or_bits_batch.argtypes = [i64, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]
        lib.or_verify.argtypes = [i32, i32, i32, i32, vp, i32, vp]
        lib.or_additions.argtypes = [i32, i32, i32, vp, i32]
        lib.or_normalize_rows.argtypes = [i32, i32, i32, vp, i32]
        lib.or_naive.argtypes = [i32, i32, i32, vp]
        lib.or_type_invariant.argtypes = [i32, i32, i32, vp, i32, vp]
        lib.or_sym_invariant.argtypes = [i32, i32, i32, vp, i32, vp]
        lib.or_matrix_rank.argtypes = [vp, i32, i32]
        lib.or_walker_init.argtypes = [vp, i32, i32, i32, i32, i32, u64]
        lib.or_walker_free.argtypes = [vp]
        lib.or_seed_rows.argtypes = [vp, vp, i32]
        lib.or_seed_naive.argtypes = [vp]
        lib.or_walk.argtypes = [vp, u64, u64, vp]
        lib.or_get_rows.argtypes = [vp, i32, vp]
        lib.or_restart.argtypes = [vp, vp, i32]
        lib.or_count_candidates.argtypes = [vp]
        lib.or_get_candidate.argtypes = [vp, i32, vp]
        lib.or_apply_flip.argtypes = [vp, i32, i32, i32]
        lib.or_apply_expand.argtypes = [vp, i32, i32, i32, i32]
        lib.or_reduce_all_public.argtypes = [vp]
        lib.or_local_reduce_public.argtypes = [vp, i32, i32]
        for nm in ("or_meta_transpose", "or_meta_rotate", "or_meta_swap_sizes"):
            getattr(lib, nm).argtypes = [i32, i32, i32, vp, i32, vp]
        lib.or_meta_project.argtypes = [i32, i32, i32, vp, i32, vp, vp]
        lib.or_meta_extend.argtypes = [i32, i32, i32, vp, i32, vp, vp]
        lib.or_meta_merge.argtypes = [i32, i32, i32, i32, vp, i32, vp, i32, vp]
        lib.or_meta_product.argtypes = [i32, i32, i32, vp, i32, i32, i32, i32, vp, i32, vp]
        lib.or_lift_exhaustive.argtypes = [i32, i32, i32, vp, i32, vp]
        lib.or_resize.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, C.c_uint32, u64, u64, u64, vp]
        lib.or_run_walkers.argtypes = [i32, i32, i32, i32, i32, i64, u64, vp, vp, i32, u64, u64,
                                       vp, i32, vp, vp, vp, vp, vp, vp]

    # ---- scalar helpers ----
    def word(self, seed, step, walker_id, slot):
        return self.lib.or_word(seed, step, walker_id, slot)

    def philox(self, ctr, key):
        c = np.asarray(ctr, dtype=np.uint32)
        k = np.asarray(key, dtype=np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        self.lib.or_philox4x32_10(_p(c), _p(k), _p(out))
        return out

    def bits_batch(self, da, sa, db, sb, op):
        n = len(da)
        arrs = [np.ascontiguousarray(x, dtype=np.uint64) for x in (da, sa, db, sb)]
        d = np.zeros(n, np.uint64)
        s = np.zeros(n, np.uint64)
        valid = np.zeros(n, np.int32)
        eq = np.zeros(n, np.int32)
        neg = np.zeros(n, np.int32)
        self.lib.or_bits_batch(n, *[_p(a) for a in arrs], op, _p(d), _p(s), _p(valid), _p(eq),
                               _p(neg))
        return d, s, valid, eq, neg

    # ---- schemes (int8 [rank, mn+np+pm]) ----
    def verify(self, m, n, p, ring, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        ff = np.full(3, -1, np.int32)
        rc = self.lib.or_verify(m, n, p, ring, _p(c), c.shape[0], _p(ff))
        return rc, tuple(int(x) for x in ff)

    def additions(self, m, n, p, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        return self.lib.or_additions(m, n, p, _p(c), c.shape[0])

    def normalize(self, m, n, p, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8).copy()
        self.lib.or_normalize_rows(m, n, p, _p(c), c.shape[0])
        return c

    def naive(self, m, n, p):
        c = np.zeros((m * n * p, m * n + n * p + p * m), np.int8)
        self.lib.or_naive(m, n, p, _p(c))
        return c

    def type_invariant(self, m, n, p, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        out = np.zeros(65 ** 3, np.int32)
        self.lib.or_type_invariant(m, n, p, _p(c), c.shape[0], _p(out))
        res = {}
        for idx in np.nonzero(out)[0]:
            ru, rest = divmod(int(idx), 65 * 65)
            rv, rw = divmod(rest, 65)
            res[(ru, rv, rw)] = int(out[idx])
        return res

    def sym_invariant(self, m, n, p, coeffs):
        """Symmetrised polynomial: {(a, b, c): coefficient of x^a y^b z^c}."""
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        out = np.zeros(65 ** 3, np.int32)
        if self.lib.or_sym_invariant(m, n, p, _p(c), c.shape[0], _p(out)) != 0:
            raise ValueError("or_sym_invariant failed")
        res = {}
        for idx in np.nonzero(out)[0]:
            a, rest = divmod(int(idx), 65 * 65)
            b, cc = divmod(rest, 65)
            res[(a, b, cc)] = int(out[idx])
        return res

    # ---- meta operators: return ((m, n, p), coeffs) ----
    def meta(self, op, fmt, coeffs, fmt2=None, coeffs2=None):
        m, n, p = fmt
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        r = c.shape[0]
        rk = C.c_int(0)
        if op in ("transpose", "rotate", "swap_sizes"):
            nf = {"transpose": (p, n, m), "rotate": (n, p, m), "swap_sizes": (m, p, n)}[op]
            out = np.zeros((r, c.shape[1]), np.int8)
            rc = getattr(self.lib, "or_meta_" + op)(m, n, p, _p(c), r, _p(out))
        elif op == "project":
            nf = (m, n, p - 1)
            out = np.zeros((r, m * n + n * (p - 1) + (p - 1) * m), np.int8)
            rc = self.lib.or_meta_project(m, n, p, _p(c), r, _p(out), C.byref(rk))
            out = out[: rk.value]
        elif op == "extend":
            nf = (m, n, p + 1)
            out = np.zeros((r + m * n, m * n + n * (p + 1) + (p + 1) * m), np.int8)
            rc = self.lib.or_meta_extend(m, n, p, _p(c), r, _p(out), C.byref(rk))
        elif op in ("merge", "double"):
            if op == "double":
                fmt2, coeffs2 = fmt, coeffs
            p2 = fmt2[2]
            c2 = np.ascontiguousarray(coeffs2, dtype=np.int8)
            nf = (m, n, p + p2)
            out = np.zeros((r + c2.shape[0], m * n + n * (p + p2) + (p + p2) * m), np.int8)
            rc = self.lib.or_meta_merge(m, n, p, p2, _p(c), r, _p(c2), c2.shape[0], _p(out))
        elif op == "product":
            m2, n2, p2 = fmt2
            c2 = np.ascontiguousarray(coeffs2, dtype=np.int8)
            M, N, P = m * m2, n * n2, p * p2
            nf = (M, N, P)
            out = np.zeros((r * c2.shape[0], M * N + N * P + P * M), np.int8)
            rc = self.lib.or_meta_product(m, n, p, _p(c), r, m2, n2, p2, _p(c2), c2.shape[0], _p(out))
        else:
            raise ValueError(op)
        if rc != 0:
            raise ValueError(f"or_meta_{op}: {rc}")
        return nf, out

    def resize(self, fmt, coeffs, bests, r_cap, seed, rnd, walker_id, thr_resize=1 << 31):
        m_, n_, p_ = (C.c_int(x) for x in fmt)
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        buf = np.zeros(r_cap * 192 + 64, np.int8)
        buf[: c.size] = c.reshape(-1)
        rk = C.c_int(c.shape[0])
        nb = len(bests)
        bfmt = np.array([b[0] for b in bests], dtype=np.int32).reshape(-1) if nb else np.zeros(3, np.int32)
        brank = np.array([len(b[1]) for b in bests], dtype=np.int32) if nb else np.zeros(1, np.int32)
        keep = [np.ascontiguousarray(b[1], dtype=np.int8) for b in bests]
        ptrs = (C.c_void_p * max(nb, 1))(*[k.ctypes.data for k in keep])
        op = C.c_int(0)
        self.lib.or_resize(C.byref(m_), C.byref(n_), C.byref(p_), _p(buf), C.byref(rk), r_cap, nb,
                           _p(bfmt), _p(brank), C.cast(ptrs, C.c_void_p), thr_resize, seed, rnd,
                           walker_id, C.byref(op))
        nf = (m_.value, n_.value, p_.value)
        w = nf[0] * nf[1] + nf[1] * nf[2] + nf[2] * nf[0]
        return nf, buf[: rk.value * w].reshape(rk.value, w).copy(), op.value

    def lift_exhaustive(self, m, n, p, z2):
        c = np.ascontiguousarray(z2, dtype=np.int8)
        out = np.zeros_like(c)
        rc = self.lib.or_lift_exhaustive(m, n, p, _p(c), c.shape[0], _p(out))
        return rc, (out if rc == 1 else None)

    def matrix_rank(self, a):
        a = np.ascontiguousarray(a, dtype=np.int8)
        return self.lib.or_matrix_rank(_p(a), a.shape[0], a.shape[1])

    # ---- walkers ----
    def walker(self, m, n, p, ring, R, walker_id=0):
        return OracleWalker(self, m, n, p, ring, R, walker_id)

    def run_walkers(self, m, n, p, ring, R, count, id_base, steps, seed, params=None,
                    threads=None, seed_coeffs=None, want_rows=True, ids=None):
        """Walkers with global ids id_base..id_base+count-1 (or the explicit ids)."""
        if ids is not None:
            ids = np.ascontiguousarray(ids, dtype=np.uint64)
            count = len(ids)
        params = params or OracleParams.default()
        threads = threads or os.cpu_count() or 1
        width = m * n + n * p + p * m
        r = np.zeros(count, np.int32)
        br = np.zeros(count, np.int32)
        dg = np.zeros(count, np.uint64)
        cnt = np.zeros((count, NCNT), np.uint64)
        rows = np.zeros((count, R, width), np.int8) if want_rows else None
        best = np.zeros((count, R, width), np.int8) if want_rows else None
        sc = None if seed_coeffs is None else np.ascontiguousarray(seed_coeffs, dtype=np.int8)
        rc = self.lib.or_run_walkers(m, n, p, ring, R, count, id_base, _p(ids), _p(sc),
                                     0 if sc is None else sc.shape[0], steps, seed,
                                     C.byref(params), threads, _p(r), _p(br), _p(dg), _p(cnt),
                                     _p(rows), _p(best))
        if rc != 0:
            raise RuntimeError("or_run_walkers failed")
        return dict(r=r, best_r=br, digest=dg, cnt=cnt, rows=rows, best=best)


class OracleWalker:
    def __init__(self, orc: Oracle, m, n, p, ring, R, walker_id=0):
        self.o = orc
        self.w = _Walker()
        self.m, self.n, self.p, self.ring, self.R = m, n, p, ring, R
        self.width = m * n + n * p + p * m
        rc = orc.lib.or_walker_init(C.byref(self.w), m, n, p, ring, R, walker_id)
        if rc != 0:
            raise ValueError("or_walker_init failed")

    def __del__(self):
        try:
            self.o.lib.or_walker_free(C.byref(self.w))
        except Exception:
            pass

    @property
    def ref(self):
        return C.byref(self.w)

    def seed_naive(self):
        return self.o.lib.or_seed_naive(self.ref)

    def seed_rows(self, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        return self.o.lib.or_seed_rows(self.ref, _p(c), c.shape[0])

    def walk(self, steps, seed, params=None):
        params = params or OracleParams.default()
        self.o.lib.or_walk(self.ref, steps, seed, C.byref(params))

    def rows(self, which=0):
        out = np.zeros((self.R + 1, self.width), np.int8)
        rank = self.o.lib.or_get_rows(self.ref, which, _p(out))
        return out[:rank].copy()

    def restart(self, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        self.o.lib.or_restart(self.ref, _p(c), c.shape[0])

    @property
    def r(self):
        return self.w.r

    @property
    def best_r(self):
        return self.w.best_r

    @property
    def digest(self):
        return self.w.digest

    @property
    def best_adds(self):
        return self.w.best_adds

    @property
    def step(self):
        return self.w.step

    @property
    def cnt(self):
        return np.array(list(self.w.cnt), dtype=np.uint64)

    def count_candidates(self):
        return self.o.lib.or_count_candidates(self.ref)

    def candidate(self, idx):
        out = np.zeros(4, np.int32)
        if self.o.lib.or_get_candidate(self.ref, idx, _p(out)) != 0:
            raise IndexError(idx)
        return tuple(int(x) for x in out)

    def apply_flip(self, cand, d, e):
        return self.o.lib.or_apply_flip(self.ref, cand, d, e)

    def apply_expand(self, plus, i, j, perm):
        return self.o.lib.or_apply_expand(self.ref, plus, i, j, perm)

    def reduce_all(self):
        self.o.lib.or_reduce_all_public(self.ref)

    def local_reduce(self, a, b):
        self.o.lib.or_local_reduce_public(self.ref, a, b)
