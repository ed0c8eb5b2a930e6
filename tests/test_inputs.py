"""The seeded input recipes (fmm_inputs): deterministic, and the paper's Sec. 6.5
distributions 2 / 3 have their small / large blocks where the paper puts them."""
import numpy as np

import fmm_inputs as fi


def test_draws_are_seeded_and_deterministic():
    for dist in ("u(-1,1)", "u(0,1)", "n(0,1)", "skew", "paper2", "paper3"):
        A1, B1 = fi.draw(dist, 16, 16, 16, 5)
        A2, B2 = fi.draw(dist, 16, 16, 16, 5)
        assert np.array_equal(A1, A2) and np.array_equal(B1, B2)
        A3, _ = fi.draw(dist, 16, 16, 16, 6)
        assert not np.array_equal(A1, A3)


def test_paper_distribution_2_blocks():
    n = 64
    A, B = fi.draw("paper2", n, n, n, 1)
    h = n // 2
    assert A[:, :h].min() >= 0 and A[:, :h].max() <= 1 and A[:, :h].max() > 0.5
    assert A[:, h:].max() <= 1.0 / n ** 2          # Uniform(0, 1/N^2) for j > N/2
    assert B[:h, :].max() <= 1.0 / n ** 2          # Uniform(0, 1/N^2) for i < N/2
    assert B[h:, :].max() > 0.5


def test_paper_distribution_3_blocks():
    n = 64
    A, B = fi.draw("paper3", n, n, n, 1)
    h = n // 2
    assert A[:h, h:].max() <= n ** 2 and A[:h, h:].max() > 0.5 * n ** 2  # Uniform(0, N^2)
    assert A[h:, :].max() <= 1 and A[:, :h].max() <= 1
    assert B[:, :h].max() <= 1.0 / n ** 2 and B[:, h:].max() > 0.5
