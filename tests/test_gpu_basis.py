"""QFactor's full-basis inputs without storing them (
qfs_set_samples_basis): training input m is e_m, generated inside the kernels
that read x (first forward pass, gate 0's environment, sweep-end cost).  Parity
with the oracle fed the explicit identity rows (at M = 2^n the sample
cost is the Hilbert-Schmidt cost), and bit-equality with the same sweep on the
stored basis."""
import numpy as np
import pytest

import oracle
from paper_2405_12866_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    from paper_2405_12866_b200 import build, qfs
    build.build()
    return qfs


def _problem(n, k, seed):
    rng = np.random.default_rng(seed)
    pairs = I.brick_pairs(n, k)
    if k > 2:
        pairs[k // 2] = [n - 1, 0]       # a non-adjacent, reversed pair
    target = np.stack([I.haar_unitary(rng) for _ in pairs])
    init = np.stack([np.stack([I.warm_gate(rng, target[j], 0.4) for j in range(k)]) for _ in range(2)])
    return pairs, target, init


@pytest.mark.parametrize("n,k,m", [(3, 4, 8), (5, 10, 32), (5, 10, 12), (8, 16, 256), (8, 16, 40), (6, 2, 64),
                                   (6, 1, 64), (4, 3, 3)])
def test_basis_trace_parity(Q, n, k, m):
    """Implicit basis vs the oracle on explicit identity rows (1e-10), and vs the
    stored basis through the same streamed kernels (bitwise); K = 1 / 2 take the
    no-forward / single-gate-forward paths, m < 2^n a prefix of the basis."""
    pairs, target, init = _problem(n, k, seed=10 * n + k)
    N = 1 << n
    x = np.eye(N, dtype=np.complex128)[:m]
    y = I.apply_circuit_tensor(n, pairs, target, x)
    ctx = Q.Context(n, pairs)
    ctx.set_samples_basis(y)
    gt = ctx.trace_sweeps(init, m, 3)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, m, 3)
    for t in range(3):
        for s in range(2):
            for i in range(k):
                eo = ot["env"][t, i, s]
                assert np.linalg.norm(gt["env"][t, i, s] - eo) <= 1e-10 * np.linalg.norm(eo)
            assert abs(gt["cost"][t, s] - ot["cost"][t, s]) <= 1e-10 * ot["cost"][t, s] + 1e-15
    ref = Q.Context(n, pairs)
    ref.set_path("streamed")
    ref.set_samples(x, y)
    rt = ref.trace_sweeps(init, m, 3)
    assert np.array_equal(gt["gates"], rt["gates"]) and np.array_equal(gt["cost"], rt["cost"])
    # back to stored inputs on the same context
    ctx.set_samples(x, y)
    e1 = ctx.trace_sweeps(init, m, 1)["env"][0]
    assert np.abs(e1 - ot["env"][0]).max() <= 1e-10 * np.abs(ot["env"][0]).max()
    ctx.close()
    ref.close()


def test_basis_qfactor_instantiate(Q):
    """QFactor mode (M = 2^n implicit basis, no validation, single-iteration
    plateau rule P:176) reaches the same termination, sweep count and final cost
    as the oracle."""
    n, k = 7, 21
    pairs, target, init = _problem(n, k, seed=77)
    N = 1 << n
    x = np.eye(N, dtype=np.complex128)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    prm = dict(dist_tol=1e-10, diff_tol_r=1e-3, plateau_window=1, min_iter=6, max_iter=400, m_init=N,
               overtrain_ratio=1e300, beta=0.0, stop_on_first=1)
    ctx = Q.Context(n, pairs)
    ctx.set_samples_basis(y)
    g1, r1, w1 = ctx.instantiate(init, prm)
    g2, r2, w2 = oracle.instantiate(n, pairs, x, y, None, None, init, prm)
    assert w1 == w2 and r1[w1]["term"] == r2[w2]["term"] == "CONVERGED"
    for a, b in zip(r1, r2):
        assert a["term"] == b["term"] and abs(a["sweeps"] - b["sweeps"]) <= 2
    assert r1[w1]["c_train"] <= 1e-10
    ctx.close()


def test_basis_errors(Q):
    pairs = I.brick_pairs(5, 6)
    y = np.eye(32, dtype=np.complex128)
    ctx = Q.Context(5, pairs, nccl_id=Q.nccl_unique_id(), rank=0, world=1, shard_mode=1)
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_samples_basis(y)          # sample mode: rank shards are not a basis prefix
    assert ei.value.status == 1
    ctx.close()
    ctx = Q.Context(5, pairs)
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_samples_basis(np.zeros((64, 32), np.complex128))  # m_pool > 2^n
    assert ei.value.status == 2
    ctx.close()
