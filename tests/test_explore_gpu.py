"""Exploratory search: walk (GPU) + population sync + Resize (Alg. 2) over
several formats.  Every scheme of the population verifies after every round and the
search is deterministic (counter-based RNG end to end)."""
import numpy as np
import pytest

from golden_io import load_scheme
from oracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_20317_b200 import fg as mod
    return mod


def _population():
    orc = Oracle()
    _, _, _, strassen = load_scheme("sec36_after.txt")
    _, _, _, s223 = load_scheme("scheme_2x2x3_r11.txt")
    return ([((2, 2, 2), strassen)] * 12 + [((2, 2, 1), orc.naive(2, 2, 1))] * 8 +
            [((2, 2, 3), s223)] * 12 + [((2, 3, 2), orc.naive(2, 3, 2))] * 8)


def _run(fg):
    import torch
    from paper_2511_20317_b200.explore import Explorer
    ex = Explorer(_population(), seed=77, stream=torch.cuda.current_stream().cuda_stream,
                  thr_resize=3 << 30)
    ops = []
    for _ in range(3):
        ops += ex.round(400)
        for f, c in ex.pop:
            assert fg.fg_verify(*f, 0, c)[0] == 0, f
    return ex, ops


def test_exploratory_rounds_verify_and_are_deterministic(fg):
    ex1, ops1 = _run(fg)
    ex2, ops2 = _run(fg)
    assert ops1 == ops2
    assert [f for f, _ in ex1.pop] == [f for f, _ in ex2.pop]
    assert all(np.array_equal(a[1], b[1]) for a, b in zip(ex1.pop, ex2.pop))
    assert len(ex1.formats()) >= 3 and len(ex1.registry.best) >= 4
    for f, (rank, adds, c) in ex1.registry.best.items():
        assert fg.fg_verify(*f, 0, c)[0] == 0 and len(c) == rank
    assert ex1.registry.best[(2, 2, 2)][0] == 7
    assert {op >> 1 for op in ops1} - {0} != set()          # some resize operations applied
