"""Harness input generators (paper_2405_12866_b200/inputs.py): distributions and structure."""
import numpy as np

from paper_2405_12866_b200 import inputs as I


def test_haar_unitary_and_states_orthonormal_and_deterministic():
    u = I.haar_unitary(I.rng_for(1, 0, 0))
    assert np.abs(u.conj().T @ u - np.eye(4)).max() < 1e-14
    x = I.haar_states(I.rng_for(3, 1, 0), 9, 16)
    assert np.abs(x.conj() @ x.T - np.eye(16)).max() < 1e-13
    x2 = I.haar_states(I.rng_for(3, 1, 0), 9, 16)
    assert np.array_equal(x, x2)
    # Porter-Thomas: |amp|^2 mean 1/N (P:354 columns of a Haar unitary)
    assert abs(np.mean(np.abs(x) ** 2) * 512 - 1) < 1e-12


def test_haar_first_moment():
    """Haar marginal E|U00|^2 = 1/d (SPEC S:59 Monte-Carlo example, d=4)."""
    rng = np.random.default_rng(5)
    v = np.mean([abs(I.haar_unitary(rng)[0, 0]) ** 2 for _ in range(4000)])
    assert abs(v - 0.25) < 0.02


def test_structures():
    bp = I.brick_pairs(9, 60)
    assert bp.shape == (60, 2)
    assert [tuple(p) for p in bp[:8]] == [(0, 1), (2, 3), (4, 5), (6, 7), (1, 2), (3, 4), (5, 6), (7, 8)]
    c4 = I.c4_pairs(12, 150, I.rng_for(4, 4, 0))
    rnd = c4[4::5]
    assert len(rnd) == 30 and all(b - a >= 2 for a, b in rnd)
    brick = np.delete(c4, np.s_[4::5], axis=0)
    assert np.array_equal(brick, I.brick_pairs(12, 120))


def test_problem_targets_consistent():
    p = I.make_problem("c2", init="W", s=3)
    assert p.x.shape == (64, 64) and p.xv.shape == (16, 64) and p.init.shape == (3, 20, 4, 4)
    # y rows are the target circuit applied to x: norms preserved, U unitary
    assert np.abs(np.linalg.norm(p.y, axis=1) - 1).max() < 1e-13
    assert np.abs(p.y.conj() @ p.y.T - np.eye(64)).max() < 1e-12
    g = p.init.reshape(-1, 4, 4)
    assert max(np.abs(a.conj().T @ a - np.eye(4)).max() for a in g) < 1e-13
