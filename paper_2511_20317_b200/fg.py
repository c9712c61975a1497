"""Thin ctypes binding of libfg.so (include/fg.h).  Argument marshalling only:
every step of the walk runs in libfg's CUDA kernels.  There is no CPU fallback:
if libfg.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBFG = os.environ.get("FG_LIBFG") or os.path.join(HERE, "libfg.so")   # override: A/B experiments only

FG_ZT, FG_Z2 = 0, 1
FG_FLAG_COMPLEXITY = 1
FG_NCNT = 12
CNT_NAMES = ["steps", "draws", "flips", "flip_fail", "expand_ok", "expand_reject", "merges",
             "zero_removed", "best_copies", "improvements", "reduce_calls", "verify_fail"]
STAT_NAMES = ["steps", "draws", "flips", "expands", "reductions", "verified", "verify_fail",
              "queue_overflow", "launches", "walk_us", "verify_us", "walk_launches"]
STATUS = {0: "FG_OK", -1: "FG_E_ARG", -2: "FG_E_CAPACITY", -3: "FG_E_DOMAIN",
          -4: "FG_E_INVALID_SCHEME", -5: "FG_E_CUDA", -6: "FG_E_STATE", -7: "FG_E_UNSUPPORTED"}

if not os.path.exists(LIBFG):
    raise ImportError(f"{LIBFG} is missing: build it with __graft_entry__.build() "
                      "(there is no CPU fallback)")

_lib = C.CDLL(LIBFG)


class FgError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.fg_strerror(status).decode()
        super().__init__(f"{where}: {STATUS.get(status, status)} ({msg})")


class fg_params(C.Structure):
    _fields_ = [("k_flip", C.c_uint32), ("thr_accept_eq", C.c_uint32),
                ("thr_reduce", C.c_uint32), ("thr_expand", C.c_uint32),
                ("expand_slack", C.c_int32), ("phase_steps", C.c_uint32),
                ("flags", C.c_uint32)]


_vp, _i32, _i64, _u64, _sz = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_size_t
_sig = {
    "fg_params_default": (None, [_vp]),
    "fg_strerror": (C.c_char_p, [_i32]),
    "fg_create": (_i32, [_i32, _i32, _i32, _i32, _i32, _i64, _i64, _i32, _vp, _vp]),
    "fg_destroy": (None, [_vp]),
    "fg_seed_naive": (_i32, [_vp]),
    "fg_seed_pool": (_i32, [_vp, _vp, _i32, _i64, _i64]),
    "fg_walk": (_i32, [_vp, _u64, _u64, _vp]),
    "fg_load_walkers": (_i32, [_vp, _vp, _vp, _i64, _i64]),
    "fg_verify": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_verify_batch": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fg_best": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "fg_get_walkers": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fg_get_walker": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "fg_record_bytes": (_sz, [_i32]),
    "fg_export_best": (_i32, [_vp, _vp]),
    "fg_import_best": (_i32, [_vp, _vp, _i32]),
    "fg_record_merge": (_i32, [_vp, _i32, _vp]),
    "fg_record_pack": (_i32, [_i32, _i32, _i32, _i32, _i32, _vp, _i32, _i64, _vp]),
    "fg_record_unpack": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fg_restart": (_i32, [_vp, _i32, _vp]),
    "fg_state_bytes": (_sz, [_vp]),
    "fg_save_state": (_i32, [_vp, _vp]),
    "fg_load_state": (_i32, [_vp, _vp]),
    "fg_stats": (_i32, [_vp, _vp]),
    "fg_kernel_name": (C.c_char_p, [_vp]),
    "fg_rank_first_steps": (_i32, [_vp, _i32, _vp]),
    "fg_meta_transpose": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_meta_rotate": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_meta_swap_sizes": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_meta_project": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "fg_meta_extend": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "fg_meta_merge": (_i32, [_i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp]),
    "fg_meta_double": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_meta_product": (_i32, [_i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp]),
    "fg_resize": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _vp, C.c_uint32, _u64,
                          _u64, _u64, _vp]),
    "fg_lift": (_i32, [_i32, _i32, _i32, _vp, _i32, _i64, _vp, _vp]),
    "fg_type_invariant": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "fg_sym_invariant": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
    "fg_scheme_key": (_i32, [_i32, _i32, _i32, _i32, _vp, _i32, _vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a)   # raw address (e.g. a pinned torch tensor's data_ptr())


def _ck(rc, where):
    if rc != 0:
        raise FgError(rc, where)
    return rc


def params_default(**kw) -> fg_params:
    p = fg_params()
    _lib.fg_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def fg_strerror(status: int) -> str:
    return _lib.fg_strerror(status).decode()


def fg_verify(m, n, p, ring, coeffs):
    """Host exact Brent check: returns (status, first_fail)."""
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    ff = np.full(3, -1, np.int32)
    rc = _lib.fg_verify(m, n, p, ring, _p(c), c.shape[0], _p(ff))
    return rc, tuple(int(x) for x in ff)


def fg_record_bytes(r_cap: int) -> int:
    return _lib.fg_record_bytes(r_cap)


def fg_record_pack(m, n, p, ring, r_cap, coeffs, walker_id) -> np.ndarray:
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    rec = np.zeros(fg_record_bytes(r_cap), np.uint8)
    _ck(_lib.fg_record_pack(m, n, p, ring, r_cap, _p(c), c.shape[0], walker_id, _p(rec)),
        "fg_record_pack")
    return rec


def fg_record_unpack(rec: np.ndarray, r_cap: int):
    vals = [C.c_int() for _ in range(7)]
    wid = C.c_int64()
    rec = np.ascontiguousarray(rec, dtype=np.uint8)
    m_, n_, p_, ring_, rank_, adds_ = (C.c_int() for _ in range(6))
    tmp = np.zeros((r_cap, 64 * 3), np.int8)
    _ck(_lib.fg_record_unpack(_p(rec), C.byref(m_), C.byref(n_), C.byref(p_), C.byref(ring_),
                              C.byref(rank_), C.byref(adds_), C.byref(wid), _p(tmp)),
        "fg_record_unpack")
    m, n, p = m_.value, n_.value, p_.value
    width = m * n + n * p + p * m
    flat = tmp.reshape(-1)[: r_cap * width].reshape(r_cap, width)
    del vals
    return dict(m=m, n=n, p=p, ring=ring_.value, rank=rank_.value, additions=adds_.value,
                walker_id=wid.value, coeffs=flat[: rank_.value].copy())


def fg_record_merge(records: np.ndarray, count: int) -> np.ndarray:
    recs = np.ascontiguousarray(records, dtype=np.uint8)
    out = np.zeros(recs.size // count, np.uint8)
    _ck(_lib.fg_record_merge(_p(recs), count, _p(out)), "fg_record_merge")
    return out


def fg_resize(fmt, coeffs, bests, r_cap, seed, rnd, walker_id, ring=FG_ZT, thr_resize=1 << 31):
    """Alg. 2 on one scheme; bests: list of ((m,n,p), coeffs).
    Returns ((m, n, p), coeffs, op)."""
    m_, n_, p_ = (C.c_int(x) for x in fmt)
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    buf = np.zeros(r_cap * 192, np.int8)
    buf[: c.size] = c.reshape(-1)
    rk = C.c_int(c.shape[0])
    nb = len(bests)
    bfmt = np.array([b[0] for b in bests], dtype=np.int32).reshape(-1) if nb else np.zeros(3, np.int32)
    brank = np.array([len(b[1]) for b in bests], dtype=np.int32) if nb else np.zeros(1, np.int32)
    keep = [np.ascontiguousarray(b[1], dtype=np.int8) for b in bests]
    ptrs = (C.c_void_p * max(nb, 1))(*[k.ctypes.data for k in keep])
    op = C.c_int(0)
    _ck(_lib.fg_resize(C.byref(m_), C.byref(n_), C.byref(p_), ring, _p(buf), C.byref(rk), r_cap, nb,
                       _p(bfmt), _p(brank), C.cast(ptrs, C.c_void_p), thr_resize, seed, rnd, walker_id,
                       C.byref(op)), "fg_resize")
    nf = (m_.value, n_.value, p_.value)
    w = nf[0] * nf[1] + nf[1] * nf[2] + nf[2] * nf[0]
    return nf, buf[: rk.value * w].reshape(rk.value, w).copy(), op.value


def fg_lift(m, n, p, z2, node_budget=10_000_000):
    """Z_2 -> Z_T lifting: (status, lifted coeffs or None, nodes)."""
    c = np.ascontiguousarray(z2, dtype=np.int8)
    out = np.zeros_like(c)
    nodes = C.c_int64(0)
    rc = _lib.fg_lift(m, n, p, _p(c), c.shape[0], node_budget, _p(out), C.byref(nodes))
    return rc, (out if rc == 0 else None), nodes.value


def fg_type_invariant(m, n, p, ring, coeffs):
    """({(ru, rv, rw): count}, (sum ru, sum rv, sum rw)) -- PAPER:515-524."""
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    counts = np.zeros(65 ** 3, np.int32)
    sums = np.zeros(3, np.int32)
    _ck(_lib.fg_type_invariant(m, n, p, ring, _p(c), c.shape[0], _p(counts), _p(sums)),
        "fg_type_invariant")
    out = {}
    for idx in np.nonzero(counts)[0]:
        ru, rest = divmod(int(idx), 65 * 65)
        rv, rw = divmod(rest, 65)
        out[(ru, rv, rw)] = int(counts[idx])
    return out, tuple(int(x) for x in sums)


def fg_sym_invariant(m, n, p, ring, coeffs):
    """{(a, b, c): coefficient} of the symmetrised polynomial."""
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    sym = np.zeros(65 ** 3, np.int32)
    _ck(_lib.fg_sym_invariant(m, n, p, ring, _p(c), c.shape[0], _p(sym)), "fg_sym_invariant")
    out = {}
    for idx in np.nonzero(sym)[0]:
        a, rest = divmod(int(idx), 65 * 65)
        b, cc = divmod(rest, 65)
        out[(a, b, cc)] = int(sym[idx])
    return out


def fg_scheme_key(m, n, p, ring, coeffs) -> int:
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    k = C.c_uint64()
    _ck(_lib.fg_scheme_key(m, n, p, ring, _p(c), c.shape[0], C.byref(k)), "fg_scheme_key")
    return k.value


def fg_meta(op, fmt, coeffs, ring=FG_ZT, fmt2=None, coeffs2=None):
    """Meta operator `op` of PAPER:243-262 on a scheme; returns ((m, n, p), coeffs)."""
    m, n, p = fmt
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    r = c.shape[0]
    rk = C.c_int(0)
    w = lambda a, b, d: a * b + b * d + d * a          # noqa: E731
    if op in ("transpose", "rotate", "swap_sizes", "double"):
        nf = {"transpose": (p, n, m), "rotate": (n, p, m), "swap_sizes": (m, p, n),
              "double": (m, n, 2 * p)}[op]
        out = np.zeros((2 * r if op == "double" else r, w(*nf)), np.int8)
        _ck(getattr(_lib, "fg_meta_" + op)(m, n, p, ring, _p(c), r, _p(out)), "fg_meta_" + op)
        return nf, out
    if op in ("project", "extend"):
        nf = (m, n, p - 1) if op == "project" else (m, n, p + 1)
        out = np.zeros((r + (m * n if op == "extend" else 0), w(*nf)), np.int8)
        _ck(getattr(_lib, "fg_meta_" + op)(m, n, p, ring, _p(c), r, _p(out), C.byref(rk)),
            "fg_meta_" + op)
        return nf, out[: rk.value].copy()
    c2 = np.ascontiguousarray(coeffs2, dtype=np.int8)
    if op == "merge":
        nf = (m, n, p + fmt2[2])
        out = np.zeros((r + c2.shape[0], w(*nf)), np.int8)
        _ck(_lib.fg_meta_merge(m, n, p, fmt2[2], ring, _p(c), r, _p(c2), c2.shape[0], _p(out)),
            "fg_meta_merge")
        return nf, out
    if op == "product":
        m2, n2, p2 = fmt2
        nf = (m * m2, n * n2, p * p2)
        out = np.zeros((r * c2.shape[0], w(*nf)), np.int8)
        _ck(_lib.fg_meta_product(m, n, p, _p(c), r, m2, n2, p2, _p(c2), c2.shape[0], ring, _p(out)),
            "fg_meta_product")
        return nf, out
    raise ValueError(op)


class FlipGraph:
    """One fg_ctx: a pool of walkers of one format on one GPU."""

    def __init__(self, m, n, p, ring=FG_ZT, r_cap=32, num_walkers=64, walker_id_base=0,
                 device=0, stream=None):
        self.m, self.n, self.p, self.ring, self.R = m, n, p, ring, r_cap
        self.W = num_walkers
        self.id_base = walker_id_base
        self.width = m * n + n * p + p * m
        ctx = C.c_void_p()
        _ck(_lib.fg_create(m, n, p, ring, r_cap, num_walkers, walker_id_base, device, stream,
                           C.byref(ctx)), "fg_create")
        self.ctx = ctx

    def close(self):
        if getattr(self, "ctx", None) and _lib is not None:   # _lib is None during interpreter shutdown
            _lib.fg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    @property
    def kernel_name(self):
        return _lib.fg_kernel_name(self.ctx).decode()

    def seed_naive(self):
        _ck(_lib.fg_seed_naive(self.ctx), "fg_seed_naive")

    def seed_pool(self, coeffs, w_begin=0, w_end=None):
        c = np.ascontiguousarray(coeffs, dtype=np.int8)
        w_end = self.W if w_end is None else w_end
        _ck(_lib.fg_seed_pool(self.ctx, _p(c), c.shape[0], w_begin, w_end), "fg_seed_pool")

    def load_walkers(self, schemes, w_begin=0):
        """One scheme per walker (list of int8 [rank, width] arrays)."""
        k = len(schemes)
        buf = np.zeros((k, self.R, self.width), np.int8)
        ranks = np.zeros(k, np.int32)
        for i, c in enumerate(schemes):
            buf[i, : len(c)] = c
            ranks[i] = len(c)
        _ck(_lib.fg_load_walkers(self.ctx, _p(buf), _p(ranks), w_begin, k), "fg_load_walkers")

    def walk(self, steps, seed, params: fg_params | None = None):
        _ck(_lib.fg_walk(self.ctx, steps, seed, None if params is None else C.byref(params)),
            "fg_walk")

    def verify_batch(self, coeffs_list):
        k = len(coeffs_list)
        buf = np.zeros((k, self.R, self.width), np.int8)
        ranks = np.zeros(k, np.int32)
        for i, c in enumerate(coeffs_list):
            buf[i, : len(c)] = c
            ranks[i] = len(c)
        ok = np.zeros(k, np.int32)
        ff = np.zeros((k, 3), np.int32)
        _ck(_lib.fg_verify_batch(self.ctx, _p(buf), _p(ranks), k, _p(ok), _p(ff)),
            "fg_verify_batch")
        return ok, ff

    def best(self):
        rank, adds, wid = C.c_int(), C.c_int(), C.c_int64()
        out = np.zeros((self.R, self.width), np.int8)
        _ck(_lib.fg_best(self.ctx, C.byref(rank), C.byref(adds), C.byref(wid), _p(out)), "fg_best")
        return dict(rank=rank.value, additions=adds.value, walker_id=wid.value,
                    coeffs=out[: rank.value].copy())

    def get_walkers(self, w_begin=0, w_end=None, rows=True):
        w_end = self.W if w_end is None else w_end
        k = w_end - w_begin
        r = np.zeros(k, np.int32)
        br = np.zeros(k, np.int32)
        ba = np.zeros(k, np.int32)
        dg = np.zeros(k, np.uint64)
        st = np.zeros(k, np.uint64)
        cnt = np.zeros((k, FG_NCNT), np.uint64)
        cur = np.zeros((k, self.R, self.width), np.int8) if rows else None
        best = np.zeros((k, self.R, self.width), np.int8) if rows else None
        _ck(_lib.fg_get_walkers(self.ctx, w_begin, w_end, _p(r), _p(br), _p(ba), _p(dg), _p(st),
                                _p(cnt), _p(cur), _p(best)), "fg_get_walkers")
        return dict(r=r, best_r=br, best_adds=ba, digest=dg, step=st, cnt=cnt, rows=cur, best=best)

    def record_bytes(self):
        return fg_record_bytes(self.R)

    def export_best(self) -> np.ndarray:
        rec = np.zeros(self.record_bytes(), np.uint8)
        _ck(_lib.fg_export_best(self.ctx, _p(rec)), "fg_export_best")
        return rec

    def import_best(self, records: np.ndarray, count: int):
        recs = np.ascontiguousarray(records, dtype=np.uint8)
        _ck(_lib.fg_import_best(self.ctx, _p(recs), count), "fg_import_best")

    def restart(self, slack: int) -> int:
        n = C.c_int64()
        _ck(_lib.fg_restart(self.ctx, slack, C.byref(n)), "fg_restart")
        return n.value

    def state_bytes(self) -> int:
        return _lib.fg_state_bytes(self.ctx)

    def save_state(self, buf=None):
        """buf: a numpy uint8 array or a raw host address (pinned torch tensor)."""
        if buf is None:
            buf = np.zeros(self.state_bytes(), np.uint8)
        _ck(_lib.fg_save_state(self.ctx, _p(buf)), "fg_save_state")
        return buf

    def load_state(self, buf):
        _ck(_lib.fg_load_state(self.ctx, _p(buf)), "fg_load_state")

    def rank_first_steps(self, max_rank=None) -> np.ndarray:
        """out[k]: first walker step index of a verified strict improvement to rank k
        (0 for the seeded rank, 2^64-1 if never reached)."""
        max_rank = self.R if max_rank is None else max_rank
        out = np.zeros(max_rank + 1, np.uint64)
        _ck(_lib.fg_rank_first_steps(self.ctx, max_rank, _p(out)), "fg_rank_first_steps")
        return out

    def stats(self) -> dict:
        out = np.zeros(12, np.uint64)
        _ck(_lib.fg_stats(self.ctx, _p(out)), "fg_stats")
        return dict(zip(STAT_NAMES, (int(x) for x in out)))
