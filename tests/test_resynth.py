"""NEXT-4: gate-deletion re-instantiation of partitions.

The host logic (paper_2405_12866_b200/resynth.py) is driven here by the CPU
oracle through a small Context adapter (test infrastructure), and by libqfs in
the -m gpu test.  Pins: the synthetic partitions carry redundancy by
construction (an identity one-qubit gate next to a one-qubit gate on the same
qubit), so exactly those gates can go; CNOTs cannot (entangling); the reduced
block reproduces the original unitary (dense check, n <= 5)."""
import numpy as np
import pytest

import oracle
from paper_2405_12866_b200 import inputs as I
from paper_2405_12866_b200 import resynth as R

PRM = dict(dist_tol=1e-10, diff_tol_r=1e-3, plateau_window=5, min_iter=6, max_iter=150, m_init=4,
           overtrain_ratio=0.1, beta=0.0, stop_on_first=1)


class OracleContext:
    """The qfs.Context methods resynth uses, served by the CPU oracle."""

    def __init__(self, n, pairs):
        self.n, self.pairs, self.kinds = n, np.asarray(pairs, np.int32), None

    def set_gate_kinds(self, kinds):
        self.kinds = np.asarray(kinds, np.int32)

    def set_samples(self, x, y, xv, yv):
        self.s = (x, y, xv, yv)

    def instantiate(self, init, prm):
        x, y, xv, yv = self.s
        return oracle.instantiate(self.n, self.pairs, x, y, xv, yv, init, prm, threads=4, kinds=self.kinds)


def _unitary(block):
    N = 1 << block.n
    return I.apply_circuit_tensor(block.n, block.pairs, block.gates, np.eye(N, dtype=np.complex128))


def _check_report(block, rep, extra):
    assert len(rep.deleted) == extra
    assert rep.block.k == block.k - extra
    assert all(block.kinds[d] == I.GATE_VAR1 for d in rep.deleted)
    assert np.array_equal(rep.block.kinds, block.kinds[rep.kept])
    # the reduced block implements the original partition (up to a global phase)
    u0, u1 = _unitary(block), _unitary(rep.block)
    ov = np.trace(u0.conj().T @ u1) / u0.shape[0]
    assert abs(abs(ov) - 1) < 1e-8
    assert np.linalg.norm(u1 - ov * u0) / np.sqrt(u0.shape[0]) < 1e-4


def test_partitions_for_rank_cover_disjoint():
    for world in (1, 2, 3, 8):
        got = sorted(p for r in range(world) for p in R.partitions_for_rank(11, r, world))
        assert got == list(range(11))
    with pytest.raises(ValueError):
        R.partitions_for_rank(4, 2, 2)


def test_redundant_block_has_the_constructed_redundancy():
    b = R.redundant_block(4, 3, seed=1, extra=2)
    ids = [j for j in range(b.k) if b.kinds[j] == I.GATE_VAR1 and np.allclose(b.gates[j], np.eye(4))]
    assert len(ids) == 2
    keep = [j for j in range(b.k) if j not in ids]
    red = R.Block(b.n, b.pairs[keep], b.kinds[keep], b.gates[keep])
    assert np.abs(_unitary(b) - _unitary(red)).max() < 1e-14


def test_delete_gates_pass_oracle():
    b = R.redundant_block(4, 3, seed=1, extra=2)
    rep = R.delete_gates_pass(b, PRM, starts=2, seed=3, context_factory=OracleContext)
    _check_report(b, rep, 2)


@pytest.mark.gpu
def test_delete_gates_pass_gpu():
    from paper_2405_12866_b200 import build
    build.build()
    b = R.redundant_block(5, 4, seed=2, extra=3)
    rep = R.delete_gates_pass(b, PRM, starts=4, seed=4)
    _check_report(b, rep, 3)


@pytest.mark.gpu
def test_resynth_partitions_threads_match_sequential_gpu():
    """Partitions processed from host threads (shared-context reuse per partition,
    qfs_set_structure) give the same deletions and gates as the sequential pass."""
    from paper_2405_12866_b200 import build
    build.build()
    blocks = [R.redundant_block(4, 3, seed=5, extra=2), R.redundant_block(5, 3, seed=6, extra=2),
              R.redundant_block(4, 4, seed=7, extra=1)]
    seq = R.resynth_partitions(blocks, PRM, workers=1, starts=4)
    par = R.resynth_partitions(blocks, PRM, workers=3, starts=4)
    for (p1, r1), (p2, r2), b in zip(seq, par, blocks):
        assert p1 == p2
        assert r1.deleted == r2.deleted and r1.kept == r2.kept
        assert np.array_equal(r1.block.gates, r2.block.gates)  # deterministic kernels, same inputs
