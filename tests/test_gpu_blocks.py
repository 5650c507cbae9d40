"""GPU parity of multi-qubit block circuits (qfs_create_blocks; SURVEY.md §8(f)
NEXT-3) against the CPU oracle's *_blocks functions, on the same seeded inputs.

Tolerances as for pair circuits: E relative 1e-10
(Frobenius, per gate and start), gates 2e-10 where the environment is well
conditioned (sigma_min / sigma_max >= 1e-8), cost 1e-10 c + 1e-15.
"""
import numpy as np
import pytest

import oracle as O
from paper_2405_12866_b200 import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qfs():
    from paper_2405_12866_b200 import build, qfs as Q
    build.build()
    return Q


def _compare(n, qubits, arity, init, x, y, m, sweeps, gpu, orc):
    off = I.gate_offsets(arity)
    s = init.shape[0]
    gsz = int(off[-1])
    worst = dict(env=0.0, gate=0.0, cost=0.0)
    for t in range(sweeps):
        for i in range(len(arity)):
            d = 1 << int(arity[i])
            for st in range(s):
                sl = slice(s * off[i] + st * d * d, s * off[i] + (st + 1) * d * d)
                eg, eo = gpu["env"][t, sl].reshape(d, d), orc["env"][t, sl].reshape(d, d)
                rel = np.linalg.norm(eg - eo) / max(np.linalg.norm(eo), 1e-300)
                worst["env"] = max(worst["env"], rel)
                assert rel <= 1e-10, (t, i, st, rel)
                sv = np.linalg.svd(eo, compute_uv=False)
                if sv[-1] >= 1e-8 * sv[0]:
                    gg = gpu["gates"][t, st, off[i]:off[i + 1]]
                    go = orc["gates"][t, st, off[i]:off[i + 1]]
                    dg = np.linalg.norm(gg - go)
                    worst["gate"] = max(worst["gate"], dg)
                    assert dg <= 2e-10, (t, i, st, dg)
        dc = np.abs(gpu["cost"][t] - orc["cost"][t])
        worst["cost"] = max(worst["cost"], float(dc.max()))
        assert np.all(dc <= 1e-10 * np.abs(orc["cost"][t]) + 1e-15), (t, dc)
    assert gsz == gpu["gates"].shape[-1]
    return worst


@pytest.mark.parametrize("n,k,m,s,init", [(6, 9, 16, 3, "R"), (6, 9, 16, 3, "W"), (9, 12, 24, 4, "R")])
def test_block_trace_parity(qfs, n, k, m, s, init):
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=s, m_pool=m, v=0, init=init)
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_samples(x, y)
    sweeps = 5
    gpu = ctx.trace_sweeps(g0, m, sweeps)
    orc = O.trace_sweeps_blocks(n, qubits, arity, g0, x, y, m, sweeps)
    _compare(n, qubits, arity, g0, x, y, m, sweeps, gpu, orc)
    assert np.abs(gpu["sigma"] - orc["sigma"]).max() <= 1e-9 * np.abs(orc["sigma"]).max()
    ctx.close()


def test_block_k1_full_basis_one_sweep(qfs):
    n = 3
    q = np.array([[2, 0, 1]], np.int32)
    U = I.haar_unitary(np.random.default_rng(3), 8)
    x = np.eye(8, dtype=complex)
    y = I.apply_blocks_tensor(n, q, [3], I.pack_gates([U]), x)
    ctx = qfs.BlockContext(n, q, [3])
    ctx.set_samples(x, y)
    g0 = I.pack_gates([I.haar_unitary(np.random.default_rng(4), 8)])[None]
    tr = ctx.trace_sweeps(g0, 8, 1)
    assert np.abs(tr["gates"][0, 0].reshape(8, 8) - U).max() < 1e-12
    assert tr["cost"][0, 0] < 1e-24
    ctx.close()


def test_block_instantiate_matches_oracle(qfs):
    n, k = 6, 9
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=3, m_pool=64, v=16, init="W")
    params = dict(dist_tol=1e-8, diff_tol_r=1e-5, plateau_window=5, min_iter=6, max_iter=300, m_init=8,
                  overtrain_ratio=0.1, beta=0.0, stop_on_first=1)
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_samples(x, y, xv, yv)
    gg, rg, wg = ctx.instantiate(g0, params)
    go, ro, wo = O.instantiate_blocks(n, qubits, arity, x, y, xv, yv, g0, params)
    assert rg[wg]["term"] == ro[wo]["term"] == "CONVERGED"
    assert wg == wo
    for a, b in zip(rg, ro):
        assert a["term"] == b["term"]
        assert abs(a["sweeps"] - b["sweeps"]) <= 2
        assert a["final_m"] == b["final_m"]
    assert rg[wg]["c_train"] <= 1e-8
    # generalisation of the winner on fresh states
    fresh = I.haar_states(np.random.default_rng(77), n, 32)
    err = np.sum(np.abs(I.apply_blocks_tensor(n, qubits, arity, tgt, fresh) -
                        I.apply_blocks_tensor(n, qubits, arity, gg[wg], fresh)) ** 2, axis=1)
    assert np.mean(err < 1.1e-8) >= 0.9
    ctx.close()


def test_block_validation_cost_matches_oracle(qfs):
    """c_val after a fixed number of sweeps (no stopping rule can fire)."""
    n, k = 6, 7
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=2, m_pool=16, v=16, init="R")
    params = dict(dist_tol=-1.0, diff_tol_r=1e-3, plateau_window=0, min_iter=6, max_iter=3, m_init=16,
                  overtrain_ratio=1e300, beta=0.0, stop_on_first=0)
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_samples(x, y, xv, yv)
    gg, rg, _ = ctx.instantiate(g0, params)
    go, ro, _ = O.instantiate_blocks(n, qubits, arity, x, y, xv, yv, g0, params)
    for a, b in zip(rg, ro):
        assert a["term"] == b["term"] == "MAX_ITER"
        assert abs(a["c_train"] - b["c_train"]) <= 1e-10 * b["c_train"] + 1e-15
        assert abs(a["c_val"] - b["c_val"]) <= 1e-10 * b["c_val"] + 1e-15
    ctx.close()


def test_block_kinds_fixed_three_qubit_block_and_errors(qfs):
    n, k = 5, 6
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=2, m_pool=16, v=0, init="R")
    kinds = np.zeros(k, np.int32)
    j3 = int(np.nonzero(arity == 3)[0][0])
    kinds[j3] = I.GATE_FIXED
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_gate_kinds(kinds)
    ctx.set_samples(x, y)
    gpu = ctx.trace_sweeps(g0, 16, 3)
    orc = O.trace_sweeps_blocks(n, qubits, arity, g0, x, y, 16, 3, kinds=kinds)
    _compare(n, qubits, arity, g0, x, y, 16, 3, gpu, orc)
    off = I.gate_offsets(arity)
    assert np.array_equal(gpu["gates"][-1, :, off[j3]:off[j3 + 1]], g0[:, off[j3]:off[j3 + 1]])
    # a one-qubit slot on a three-qubit block is rejected
    bad = kinds.copy()
    bad[j3] = I.GATE_VAR1
    with pytest.raises(qfs.QfsError):
        ctx.set_gate_kinds(bad)
    # non-unitary initial gates are reported
    g_bad = g0.copy()
    g_bad[0, off[j3]] *= 1.5
    with pytest.raises(qfs.QfsError):
        ctx.trace_sweeps(g_bad, 16, 1)
    ctx.close()
    # bad structures
    with pytest.raises(qfs.QfsError):
        qfs.BlockContext(n, [[0, 0, 1]], [3])
    with pytest.raises(qfs.QfsError):
        qfs.BlockContext(n, [[0, 1, 5]], [3])
    with pytest.raises(qfs.QfsError):
        qfs.BlockContext(n, [[0, 1, 2]], [4])


def test_block_rank_deficient_environment_jacobi_fallback(qfs):
    """M = 2 states at n = 3: every 8x8 environment has rank <= 2, Newton-Schulz
    cannot converge and the Jacobi fallback runs.  Gates are then not unique
    (reading R5): compare costs, and check the gates stay unitary."""
    n = 3
    q = np.array([[0, 1, 2], [2, 0, 1]], np.int32)
    ar = [3, 3]
    rng = np.random.default_rng(8)
    tgt = I.pack_gates([I.haar_unitary(rng, 8) for _ in ar])
    x = I.haar_states(rng, n, 2)
    y = I.apply_blocks_tensor(n, q, ar, tgt, x)
    g0 = I.pack_gates([I.haar_unitary(rng, 8) for _ in ar])[None]
    ctx = qfs.BlockContext(n, q, ar)
    ctx.set_samples(x, y)
    gpu = ctx.trace_sweeps(g0, 2, 1)
    orc = O.trace_sweeps_blocks(n, q, ar, g0, x, y, 2, 1)
    assert abs(gpu["cost"][0, 0] - orc["cost"][0, 0]) <= 1e-10 * orc["cost"][0, 0] + 1e-14
    assert np.abs(gpu["sigma"] - orc["sigma"]).max() <= 1e-10 * np.abs(orc["sigma"]).max()
    for gm in I.unpack_gates(gpu["gates"][0, 0], ar):
        assert np.abs(gm.conj().T @ gm - np.eye(8)).max() < 1e-12
    ctx.close()


def test_block_trace_parity_n12_sampled(qfs):
    """n = 12 (streamed block path at the bench's sizes per start: M = 32, 16 starts,
    K = 24 with 16 three-qubit blocks); the oracle recomputes two sampled starts."""
    n, k, m, s = 12, 24, 32, 16
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=s, m_pool=m, v=0, init="R")
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_samples(x, y)
    gpu = ctx.trace_sweeps(g0, m, 2)
    ctx.close()
    off = I.gate_offsets(arity)
    for st in (0, 11):
        orc = O.trace_sweeps_blocks(n, qubits, arity, g0[st:st + 1], x, y, m, 2)
        for t in range(2):
            assert abs(gpu["cost"][t, st] - orc["cost"][t, 0]) <= 1e-10 * orc["cost"][t, 0] + 1e-15
            for i in range(k):
                d = 1 << int(arity[i])
                eg = gpu["env"][t, s * off[i] + st * d * d: s * off[i] + (st + 1) * d * d]
                eo = orc["env"][t, off[i]:off[i + 1]]
                assert np.linalg.norm(eg - eo) <= 1e-10 * np.linalg.norm(eo)
            assert np.linalg.norm(gpu["gates"][t, st] - orc["gates"][t, 0]) <= 2e-10 * np.sqrt(k)


@pytest.mark.parametrize("n,k,m", [(3, 4, 3), (4, 7, 5), (5, 9, 7), (7, 11, 13)])
def test_block_trace_parity_ragged(qfs, n, k, m):
    """Ragged sample counts (not multiples of a warp or tile), small n, unsorted
    qubit lists; 3 sweeps, costs and environments against the oracle (gates only
    where the environment is well conditioned, as everywhere)."""
    qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=2, m_pool=m, v=0, init="R", seed=30 + n)
    ctx = qfs.BlockContext(n, qubits, arity)
    ctx.set_samples(x, y)
    gpu = ctx.trace_sweeps(g0, m, 3)
    ctx.close()
    orc = O.trace_sweeps_blocks(n, qubits, arity, g0, x, y, m, 3)
    _compare(n, qubits, arity, g0, x, y, m, 3, gpu, orc)
