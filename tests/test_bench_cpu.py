"""bench.py's reference arm (the oracle on the host cores) runs without a GPU and
prints the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3",
                          "--ref-seconds", "4"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("(3,3,3)")


def test_ladder_from_first_interpolates_within_phase():
    """Exact time-to-rank: rank <= t is held from the first step index of a verified
    improvement to any rank <= t; its time is interpolated inside that phase."""
    sys.path.insert(0, ROOT)
    from bench import ladder_from_first
    U = (1 << 64) - 1
    first = [U] * 30
    first[27] = 0          # seeded
    first[25] = 149        # phase 0 of S = 100? no: S = 200 -> phase 0
    first[24] = 450        # phase 2
    first[23] = 451
    first[22] = 300        # reached 22 before 24 and 23: rank <= 23, 24 held from step 300
    lad = ladder_from_first(first, [10.0, 20.0, 40.0], 200, 27, seeded_rank=27)
    assert set(lad) == {22, 23, 24, 25, 26}
    assert lad[26] == lad[25] == (150 / 200 * 10.0 / 1000.0, 150)
    t22 = (10.0 + (300 - 200 + 1) / 200 * 20.0) / 1000.0
    assert lad[24] == lad[23] == lad[22] == (t22, 301)
    # a step beyond the timed phases is not reported
    first[21] = 5000
    assert 21 not in ladder_from_first(first, [10.0, 20.0, 40.0], 200, 27, seeded_rank=27)
