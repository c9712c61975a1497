"""Loader for the text fixtures under tests/golden/ (plain parsing, no arithmetic)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_scheme(name):
    """Returns (m, n, p, coeffs int8 [rank, mn+np+pm]) from a golden scheme file."""
    fmt = None
    rank = None
    blocks = {"U": [], "V": [], "W": []}
    cur = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "format":
                fmt = tuple(int(x) for x in tok[1:4])
            elif tok[0] == "rank":
                rank = int(tok[1])
            elif tok[0] in blocks:
                cur = tok[0]
            else:
                blocks[cur].append([int(x) for x in tok])
    m, n, p = fmt
    U = np.array(blocks["U"], dtype=np.int8)
    V = np.array(blocks["V"], dtype=np.int8)
    W = np.array(blocks["W"], dtype=np.int8)
    assert U.shape == (rank, m * n) and V.shape == (rank, n * p) and W.shape == (rank, p * m)
    return m, n, p, np.concatenate([U, V, W], axis=1)


def load_philox_kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                v = [int(x, 16) for x in line.split()]
                rows.append((v[0:4], v[4:6], v[6:10]))
    return rows
