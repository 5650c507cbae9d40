"""Oracle pins for multi-qubit blocks (PAPER.md P:57:
QFactor updates "possibly multi-qubit" unitary gates without parameterising
them).  CPU only: each pin checks the oracle's block functions against
something other than themselves — dense Kronecker embeddings built from the
index definition, brute-force probe circuits, LAPACK, closed forms, and the
already-pinned two-qubit oracle.
"""
import numpy as np
import pytest

import oracle as O
from paper_2405_12866_b200 import inputs as I


def dense_block(n, q, g):
    """2^n x 2^n matrix of gate g on qubits q (l = sum_j b(q_j) 2^j) by brute force."""
    a, N = len(q), 1 << n
    D = np.zeros((N, N), complex)
    for col in range(N):
        li = sum(((col >> q[j]) & 1) << j for j in range(a))
        for lo in range(1 << a):
            row = col
            for j in range(a):
                row = (row & ~(1 << q[j])) | (((lo >> j) & 1) << q[j])
            D[row, col] += g[lo, li]
    return D


@pytest.mark.parametrize("q", [[0, 1, 2], [2, 0, 3], [3, 1, 0], [1, 3]])
def test_block_apply_matches_dense_embedding(q):
    n = 4
    rng = np.random.default_rng(len(q) * 10 + q[0])
    g = I.haar_unitary(rng, 1 << len(q))
    st = I.haar_states(rng, n, 5)
    out = O.apply_block(n, len(q), q, g, st)
    ref = (dense_block(n, q, g) @ st.T).T
    assert np.abs(out - ref).max() < 1e-14
    back = O.apply_block(n, len(q), q, g, out, dagger=True)
    assert np.abs(back - st).max() < 1e-14
    # the harness simulator (tensordot) agrees too
    qq = np.zeros((1, 3), np.int32)
    qq[0, :len(q)] = q
    assert np.abs(I.apply_blocks_tensor(n, qq, [len(q)], I.pack_gates([g]), st) - ref).max() < 1e-14


def test_block_environment_matches_probe_circuits():
    """E_i[a][b] = sum_m <y_m| C with gate i replaced by |b><a| |x_m> (reading R4),
    gates before i at their old values and after i at their new ones (R3)."""
    n, k, m = 4, 4, 3
    qubits, arity = I.block_structure(n, k, seed=3)
    rng = np.random.default_rng(7)
    old = [I.haar_unitary(rng, 1 << int(a)) for a in arity]
    tgt = I.pack_gates([I.haar_unitary(rng, 1 << int(a)) for a in arity])
    x = I.haar_states(rng, n, m)
    y = I.apply_blocks_tensor(n, qubits, arity, tgt, x)
    tr = O.trace_sweeps_blocks(n, qubits, arity, I.pack_gates(old)[None], x, y, m, 1)
    new = I.unpack_gates(tr["gates"][0, 0], arity)
    off = I.gate_offsets(arity)
    for i in range(k):
        d = 1 << int(arity[i])
        e_orc = tr["env"][0, off[i]:off[i + 1]].reshape(d, d)  # s = 1: gate-major == per gate
        e_probe = np.zeros((d, d), complex)
        for a in range(d):
            for b in range(d):
                p = np.zeros((d, d), complex)
                p[b, a] = 1.0
                mats = old[:i] + [p] + new[i + 1:]
                cx = I.apply_blocks_tensor(n, qubits, arity, I.pack_gates(mats), x)
                e_probe[a, b] = np.sum(np.conj(y) * cx)
        assert np.abs(e_orc - e_probe).max() < 1e-13 * max(1.0, np.abs(e_probe).max())


def test_block_k1_full_basis_solves_in_one_sweep():
    """K = 1, M = 2^n basis: E = U^dag in local coordinates, the update is G = U
    exactly and the cost is 0 after one sweep (M = 2^n is the full cost)."""
    n = 3
    q = np.array([[1, 2, 0]], np.int32)
    rng = np.random.default_rng(11)
    U = I.haar_unitary(rng, 8)
    x = np.eye(8, dtype=complex)
    y = I.apply_blocks_tensor(n, q, [3], I.pack_gates([U]), x)
    g0 = I.haar_unitary(rng, 8)
    tr = O.trace_sweeps_blocks(n, q, [3], I.pack_gates([g0])[None], x, y, 8, 1)
    g = tr["gates"][0, 0].reshape(8, 8)
    assert np.abs(g - U).max() < 1e-13
    assert tr["cost"][0, 0] < 1e-26
    assert abs(tr["sigma"][0, 0, 0] - 8.0) < 1e-12  # sum sigma of U^dag = d


def test_block_polar_update_optimal_and_matches_lapack():
    rng = np.random.default_rng(5)
    for _ in range(5):
        E = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
        g, ss = O.polar_update_block(E, np.eye(8, dtype=complex))
        assert np.abs(g.conj().T @ g - np.eye(8)).max() < 1e-13
        u, s, vh = np.linalg.svd(E)
        # E = X D Y^dag  ->  G = Y X^dag
        assert np.abs(g - vh.conj().T @ u.conj().T).max() < 1e-12
        assert abs(ss - s.sum()) < 1e-12 * s.sum()
        assert abs(np.trace(E @ g).real - ss) < 1e-12 * s.sum()
        for _ in range(200):
            V = I.haar_unitary(rng, 8)
            assert np.trace(E @ V).real <= ss + 1e-12
    # beta = 1 returns the old gate
    go = I.haar_unitary(rng, 8)
    g, _ = O.polar_update_block(rng.standard_normal((8, 8)) + 0j, go, beta=1.0)
    assert np.abs(g - go).max() < 1e-13


def test_block_sweeps_fixed_point_and_monotone():
    n, k, m = 5, 6, 8
    qubits, arity, tgt, x, y, xv, yv, init = I.block_problem(n, k, s=2, m_pool=m, v=0, init="R")
    # exact initialisation is a fixed point (cost ~ 0, gates unchanged)
    tr = O.trace_sweeps_blocks(n, qubits, arity, tgt[None], x, y, m, 2)
    assert tr["cost"].max() < 1e-26
    assert np.abs(tr["gates"][-1, 0] - tgt).max() < 1e-12
    # random initialisation: c_train never increases from sweep to sweep, and
    # the per-gate monitor 2 - (2/M) sum sigma never increases within a sweep
    tr = O.trace_sweeps_blocks(n, qubits, arity, init, x, y, m, 6)
    c = tr["cost"]
    assert np.all(np.diff(c, axis=0) <= 1e-12)
    mon = 2.0 - 2.0 * tr["sigma"] / m          # [t][k][s], gate K-1 visited first
    assert np.all(np.diff(mon[:, ::-1, :], axis=1) <= 1e-12)
    assert np.all(mon <= 2.0 + 1e-12)


def test_blocks_with_only_pairs_match_the_pair_oracle():
    n, k, m, s = 5, 8, 6, 2
    pairs = I.brick_pairs(n, k)
    qubits = np.zeros((k, 3), np.int32)
    qubits[:, :2] = pairs
    rng = np.random.default_rng(2)
    gates = np.stack([[I.haar_unitary(rng) for _ in range(k)] for _ in range(s)])
    tgt = np.stack([I.haar_unitary(rng) for _ in range(k)])
    x = I.haar_states(rng, n, m)
    y = I.apply_circuit_tensor(n, pairs, tgt, x)
    a = O.trace_sweeps(n, pairs, gates, x, y, m, 3)
    b = O.trace_sweeps_blocks(n, qubits, [2] * k, gates.reshape(s, -1), x, y, m, 3)
    assert np.abs(a["cost"] - b["cost"]).max() < 1e-14
    assert np.abs(a["gates"].reshape(3, s, -1) - b["gates"]).max() < 1e-13


def test_block_instantiate_warm_converges_and_generalises():
    n, k = 5, 6
    qubits, arity, tgt, x, y, xv, yv, init = I.block_problem(n, k, s=2, m_pool=32, v=16, init="W")
    params = dict(dist_tol=1e-8, diff_tol_r=1e-5, plateau_window=5, min_iter=6, max_iter=400, m_init=8,
                  overtrain_ratio=0.1, beta=0.0, stop_on_first=1)
    g, res, win = O.instantiate_blocks(n, qubits, arity, x, y, xv, yv, init, params)
    assert res[win]["term"] == "CONVERGED" and res[win]["c_train"] <= 1e-8
    fresh = np.concatenate([I.haar_states(np.random.default_rng(99 + r), n, 10) for r in range(5)])
    cy = I.apply_blocks_tensor(n, qubits, arity, tgt, fresh)
    cg = I.apply_blocks_tensor(n, qubits, arity, g[win], fresh)
    err = np.sum(np.abs(cy - cg) ** 2, axis=1)
    assert np.mean(err < 1e-8 * 1.1) >= 0.9
