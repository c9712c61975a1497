"""Independent numpy checks used to pin the oracle (tests only).

These are NOT a second oracle: they are the mathematical facts the oracle must
satisfy, computed in a different way (dense tensors via einsum instead of per-
equation sums; integer vectors instead of the oracle's C code).
"""
import numpy as np


def split(m, n, p, coeffs):
    mn, np_ = m * n, n * p
    c = np.asarray(coeffs, dtype=np.int64)
    return c[:, :mn], c[:, mn:mn + np_], c[:, mn + np_:]


def scheme_tensor(m, n, p, coeffs):
    """sum_l u_l (x) v_l (x) w_l as a dense (mn, np, pm) integer tensor."""
    U, V, W = split(m, n, p, coeffs)
    return np.einsum("la,lb,lc->abc", U, V, W)


def matmul_tensor(m, n, p):
    """The target of PAPER:116/121 in the C^T layout, built from its meaning: the
    scheme must compute c_ik = sum_j a_ij b_jk, so T[a_ij, b_jk, c_(k,i)] = 1."""
    T = np.zeros((m * n, n * p, p * m), dtype=np.int64)
    for i in range(m):
        for j in range(n):
            for k in range(p):
                T[i * n + j, j * p + k, k * m + i] = 1
    return T


def first_failing(m, n, p, coeffs, ring=0):
    D = scheme_tensor(m, n, p, coeffs) - matmul_tensor(m, n, p)
    if ring == 1:
        D = D % 2
    bad = np.argwhere(D != 0)
    return None if len(bad) == 0 else tuple(int(x) for x in bad[0])


def tadd(a, b, sigma=1):
    """Ternary-safe integer a + sigma*b: returns (result, valid)."""
    s = np.asarray(a, np.int64) + sigma * np.asarray(b, np.int64)
    return s, bool(np.all(np.abs(s) <= 1))


def normalize_row(u, v, w):
    """PAPER:429 per row: make the first nonzero of u, then of v, positive; w absorbs."""
    u, v, w = np.array(u), np.array(v), np.array(w)
    nz = np.flatnonzero(u)
    if len(nz) and u[nz[0]] < 0:
        u, w = -u, -w
    nz = np.flatnonzero(v)
    if len(nz) and v[nz[0]] < 0:
        v, w = -v, -w
    return u, v, w


def brute_force_flips(m, n, p, coeffs, ring=0):
    """All flip moves of PAPER:208-215 under any role permutation,
    found by trying every ordered pair of rows and every role assignment, with no
    candidate list: returns a list of (neighbour rows as int64 array, safe)."""
    U, V, W = split(m, n, p, coeffs)
    facs = [U, V, W]
    r = U.shape[0]
    out = []
    for X in range(3):
        for Y in range(3):
            if Y == X:
                continue
            Z = 3 - X - Y
            for a in range(r):
                for b in range(r):
                    if a == b or not np.any(facs[X][a]):
                        continue
                    if np.array_equal(facs[X][a], facs[X][b]):
                        sigma = 1
                    elif ring == 0 and X == 2 and np.array_equal(facs[X][a], -facs[X][b]):
                        sigma = -1
                    else:
                        continue
                    new = [f.copy() for f in facs]
                    ny = facs[Y][a] + sigma * facs[Y][b]
                    nzv = facs[Z][b] - facs[Z][a]
                    if ring == 1:
                        ny, nzv = ny % 2, nzv % 2
                    safe = bool(np.all(np.abs(ny) <= 1) and np.all(np.abs(nzv) <= 1))
                    new[Y][a] = ny
                    new[Z][b] = nzv
                    out.append((np.concatenate(new, axis=1), safe, (X, min(a, b), max(a, b))))
    return out
