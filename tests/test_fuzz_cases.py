"""The random-case generator of the GPU suite (tests/fuzz_cases.py) stays inside the ABI's accepted
ranges and keeps covering what it is there for (host-only checks; the cases run under -m gpu)."""
import numpy as np

from tests.fuzz_cases import draw


def test_draws_are_valid_and_cover_the_range():
    rng = np.random.default_rng(7)
    seen_pairs, seen_levels, wide, phases = set(), set(), 0, set()
    for _ in range(400):
        p = draw(rng)
        assert 1 <= p["levels"] <= 12 and p["H"] >= 1 and p["W"] >= 1 and 1 <= p["N"] <= 3
        assert p["nf"] in (1, 3, 5, 7, 9) and (p["nc"] in (1, 3, 5, 7, 9) if p["levels"] > 1 else p["nc"] == 0)
        assert p["n_ph"] in (1, 4) and (p["n_ph"] == 1 or p["levels"] > 1)
        assert p["win"] in (1, 3, 5) and p["noise"] in ("awgn", "signal")
        K = p["n_o"] * p["n_s"] * p["n_c"]
        assert 1 <= K <= 65536
        wide += K > 256
        seen_levels.add(p["levels"])
        phases.add(p["n_ph"])
        if p["levels"] > 1:
            seen_pairs.add((p["nf"], p["nc"]))
    assert seen_levels == {1, 2, 3, 4, 5} and phases == {1, 4} and wide > 0
    assert len(seen_pairs) >= 14  # fine sizes 3..9 x coarse sizes 3..9 (size 1 is in the pair test)


def test_big_draws_are_megapixel_frames():
    rng = np.random.default_rng(3)
    for _ in range(50):
        p = draw(rng, big=True)
        assert 600 <= p["H"] < 1100 and p["W"] >= 1000 and p["N"] in (1, 2)
