"""Mutation check of the oracle's pins (run on the dev box, no GPU).

Each mutation is a plausible mistake in oracle/walk.c (a dropped precondition,
a dropped role pair, a reordered Alg. 1 step, a wrong sign).  For each one this
copies oracle/ and tests/ to a scratch directory, applies the edit, rebuilds
liboracle and runs the -m "not gpu" oracle tests; a mutation must make at
least one of them fail ("caught").

    python tools/oracle_mutations.py            # all mutations
    python tools/oracle_mutations.py m3 m4      # selected ones
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_walk.py", "tests/test_oracle_complexity.py",
         "tests/test_oracle_rules.py"]

REDUCE = """        /* PAPER:315-317 */
        if (word(w, seed, 2) < prm->thr_reduce) {
            w->cnt[OR_C_REDUCE_CALLS]++;
            flags |= EV_REDUCE;
            reduce_all(w);
        }
"""
ACCEPT = "        /* PAPER:310-313 */"
EXPAND = """        /* PAPER:319-321 */
        if (word(w, seed, 3) < prm->thr_expand && w->r <= w->best_r + prm->expand_slack) {
            int e = expand(w, seed);
            flags |= EV_PEXPAND | (e ? EV_EXPANDED : 0);
            w->cnt[e ? OR_C_EXPAND_OK : OR_C_EXPAND_REJECT]++;
        }
"""

MUTATIONS = {
    # (i) PAPER:219: plus accepted when only u differs
    "m1_plus_only_u": [("""        if (!distinct(w->ring, ai, aj, la, A) || !distinct(w->ring, bi, bj, lb, B) ||
            !distinct(w->ring, ci, cj, lc, Cr))""", "        if (!distinct(w->ring, ai, aj, la, A))")],
    # (ii) PAPER:241: reducible() ignores the (U,W,V) role pair
    "m2_drop_role_pair_UW": [("""        int8_t nc[OR_MAXLEN];
        if (!vec_eq(FAC(w, i, A)""", """        int8_t nc[OR_MAXLEN];
        if (q == 1) continue;
        if (!vec_eq(FAC(w, i, A)""")],
    # (iii) PAPER:310-317: reduce_all runs before the acceptance test
    "m3_reduce_before_accept": [(REDUCE, ""), (ACCEPT, REDUCE + ACCEPT)],
    # the p_expand gate runs before reduce
    "m4_expand_before_reduce": [(EXPAND, ""), (REDUCE, EXPAND + REDUCE)],
    # split without its precondition
    "m5_split_no_precondition": [("        if (!distinct(w->ring, ai, aj, la, A)) return 0;\n        memset(t3",
                                  "        memset(t3")],
    # PAPER:233-238 under signs: negated W not recognised by reducible()
    "m6_reduce_no_negated_w": [("        else if (B == RW && w->ring == OR_RING_ZT && vec_negeq(FAC(w, i, B), FAC(w, j, B), w->len[B]))\n            sigma = -1;",
                                "        else if (0) sigma = -1;")],
    # the fallback expand after a failed flip is gated like 319
    "m7_fallback_gated": [("        int e = expand(w, seed);\n        w->cnt[OR_C_FLIP_FAIL]++;",
                           "        int e = w->r <= w->best_r + prm->expand_slack ? expand(w, seed) : 0;\n        w->cnt[OR_C_FLIP_FAIL]++;")],
    # plus's second term takes u_j instead of u_i
    "m8_plus_row_j_uj": [("        memcpy(FAC(w, j, A), ai, OR_MAXLEN);", "        memcpy(FAC(w, j, A), aj, OR_MAXLEN);")],
    # R12 local reduction skipped after a flip
    "m9_no_local_reduce": [("        local_reduce(w, alpha, beta);", "        (void)local_reduce;")],
}


def run(name, edits):
    tmp = tempfile.mkdtemp(prefix="mut_" + name + "_")
    shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"))
    shutil.copytree(os.path.join(ROOT, "tests"), os.path.join(tmp, "tests"))
    so = os.path.join(tmp, "oracle", "liboracle.so")
    if os.path.exists(so):
        os.remove(so)
    path = os.path.join(tmp, "oracle", "walk.c")
    src = open(path).read()
    for old, new in edits:
        if old not in src:
            return "EDIT-NOT-APPLICABLE"
        src = src.replace(old, new, 1)
    open(path, "w").write(src)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] + TESTS,
                       cwd=tmp, capture_output=True, text=True, timeout=1800)
    shutil.rmtree(tmp, ignore_errors=True)
    lines = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
    return ("caught by " + lines[0].split()[1]) if r.returncode != 0 else "SURVIVED"


def main():
    names = sys.argv[1:] or list(MUTATIONS)
    bad = 0
    for nm in names:
        res = run(nm, MUTATIONS[nm])
        bad += not res.startswith("caught")
        print(f"{nm:28s} {res}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
