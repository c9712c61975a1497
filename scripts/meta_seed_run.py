"""C5 (4,5,12) walk from a meta-operator seed instead of naive (PAPER:243-262 operators,
PAPER:262 block multiplication with Strassen): Strassen (the paper-printed (2,2,2:7),
tests/golden/sec36_after.txt) -> product with itself (4,4,4:49) -> double (4,4,8:98) ->
merge with (4,4,4:49) (4,4,12:147) -> swap sizes (4,12,4) -> extend (4,12,5:195) -> swap
sizes (4,5,12:195); every intermediate passes the host Brent check.  Then the same long walk
as scripts/long_run.py (R = 256, 9472 walkers).

  python scripts/meta_seed_run.py <seconds> <out.json> [restart_every slack k_flip]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from golden_io import load_scheme  # noqa: E402
from long_run import run  # noqa: E402
from paper_2511_20317_b200 import fg  # noqa: E402


def seed_4512():
    _, _, _, s = load_scheme("sec36_after.txt")
    steps = []
    f, c = fg.fg_meta("product", (2, 2, 2), s, fmt2=(2, 2, 2), coeffs2=s)
    steps.append((f, c.shape[0]))
    f8, c8 = fg.fg_meta("double", f, c)
    steps.append((f8, c8.shape[0]))
    f, c = fg.fg_meta("merge", f8, c8, fmt2=f, coeffs2=c)
    steps.append((f, c.shape[0]))
    f, c = fg.fg_meta("swap_sizes", f, c)
    f, c = fg.fg_meta("extend", f, c)
    steps.append((f, c.shape[0]))
    f, c = fg.fg_meta("swap_sizes", f, c)
    steps.append((f, c.shape[0]))
    assert f == (4, 5, 12) and fg.fg_verify(*f, fg.FG_ZT, c)[0] == 0
    return c, " -> ".join(f"({a},{b},{d}:{r})" for (a, b, d), r in steps)


if __name__ == "__main__":
    budget, out = float(sys.argv[1]), sys.argv[2]
    every = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    slack = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    k_flip = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    c, note = seed_4512()
    print("seed", note, flush=True)
    run("c5_4512_zt", budget, out, every, slack, k_flip, seed_coeffs=c, seed_note="Strassen meta: " + note)
