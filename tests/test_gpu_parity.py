"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (SURVEY.md §8(c) "Parity tolerances"; north_star: 1e-10 relative
in complex128 over the first 5 sweeps):
  E:     ||E_gpu - E_orc||_F <= 1e-10 ||E_orc||_F
  gates: ||G_gpu - G_orc||_F <= 2e-10, only where sigma_4/sigma_1 >= 1e-8 (the
         polar factor is unique there; reading R5) — otherwise costs only
  cost:  |dc| <= 1e-10 c + 1e-15
Inputs are the seeded synthetic configs of paper_2405_12866_b200.inputs.
"""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2405_12866_b200 import inputs as I

pytestmark = pytest.mark.gpu

ENV_TOL, GATE_TOL, COST_TOL = 1e-10, 2e-10, 1e-10


@pytest.fixture(scope="module")
def qfs():
    from paper_2405_12866_b200 import build, qfs as Q
    build.build()
    return Q


PATHS = ["streamed", "auto"]   # auto = cluster-resident whenever the states fit


def _ctx(Q, n, pairs, path="auto", **kw):
    ctx = Q.Context(n, pairs, **kw)
    ctx.set_path(path)
    return ctx


def rand_c(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def unitary(rng):
    return I.haar_unitary(rng)


# ------------------------------------------------------------ kernel ops ----
@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_op_apply_all_pairs(qfs, n):
    rng = np.random.default_rng(n)
    m = 3
    psi = rand_c(rng, (m, 1 << n))
    ctx = _ctx(qfs, n, [[0, 1]])
    for p0 in range(n):
        for p1 in range(n):
            if p0 == p1:
                continue
            g = rand_c(rng, (4, 4))
            for dag in (False, True):
                got = ctx.op_apply(p0, p1, g, psi, dagger=dag)
                want = oracle.apply_gate(n, p0, p1, g, psi, dagger=dag)
                assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()


@pytest.mark.parametrize("n,m", [(2, 1), (4, 3), (7, 5), (11, 2)])
def test_op_environment(qfs, n, m):
    rng = np.random.default_rng(10 + n)
    phi, chi = rand_c(rng, (m, 1 << n)), rand_c(rng, (m, 1 << n))
    ctx = _ctx(qfs, n, [[0, 1]])
    for p0, p1 in [(0, 1), (1, 0), (0, n - 1), (n - 1, n - 2)] if n > 2 else [(0, 1), (1, 0)]:
        got = ctx.op_environment(p0, p1, phi, chi)
        want = oracle.environment(n, p0, p1, phi, chi)
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def _matrices(rng, count):
    out = []
    for t in range(count):
        kind = t % 6
        if kind == 0:
            a = rand_c(rng, (4, 4))
        elif kind == 1:
            a = unitary(rng) @ np.diag([1, 1e-3, 1e-5, 1e-8]) @ unitary(rng)
        elif kind == 2:
            a = rand_c(rng, (4, 2)) @ rand_c(rng, (2, 4))
        elif kind == 3:
            a = unitary(rng) @ np.diag([2, 2, 1, 1]) @ unitary(rng)
        elif kind == 4:
            a = unitary(rng).conj().T * (1 + 1e-3 * rng.standard_normal())
        else:
            a = rand_c(rng, (4, 4)) * 10.0 ** rng.integers(-6, 6)
        out.append(a)
    return np.stack(out)


def test_op_polar_against_oracle(qfs):
    """K3 on 20k seeded random, ill-conditioned, rank-deficient and degenerate 4x4s."""
    rng = np.random.default_rng(123)
    E = _matrices(rng, 20000)
    G0 = np.stack([unitary(rng) for _ in range(len(E))])
    ctx = _ctx(qfs, 2, [[0, 1]])
    for beta in (0.0, 0.3):
        gn, ss = ctx.op_polar(E, G0, beta)
        for i in range(0, len(E), 7):
            go, so = oracle.polar_update(E[i], G0[i], beta)
            ep = (1 - beta) * E[i] + beta * G0[i].conj().T
            sv = np.linalg.svd(ep, compute_uv=False)
            assert abs(ss[i] - so) <= 1e-12 * so
            assert np.abs(gn[i].conj().T @ gn[i] - np.eye(4)).max() < 1e-13
            assert abs(np.trace(ep @ gn[i]).real - sv.sum()) <= 1e-12 * sv[0]
            if sv[-1] / sv[0] >= 1e-8:
                # polar-factor perturbation bound ~ eps * cond (both sides round)
                tol = max(GATE_TOL, 50 * 2.2e-16 * sv[0] / sv[-1])
                assert np.linalg.norm(gn[i] - go) <= tol


# ------------------------------------------------------------- sweep parity --
def _compare_traces(gt, ot, label):
    env_g, env_o = gt["env"], ot["env"]
    T, K, S = env_o.shape[:3]
    worst = dict(env=0.0, gate=0.0, cost=0.0)
    for t in range(T):
        for s in range(S):
            for i in range(K):
                eo = env_o[t, i, s]
                r = np.linalg.norm(env_g[t, i, s] - eo) / np.linalg.norm(eo)
                worst["env"] = max(worst["env"], r)
                assert r <= ENV_TOL, (label, "env", t, i, s, r)
                sv = np.linalg.svd(eo, compute_uv=False)
                if sv[-1] / sv[0] >= 1e-8:
                    d = np.linalg.norm(gt["gates"][t, s, i] - ot["gates"][t, s, i])
                    worst["gate"] = max(worst["gate"], d)
                    assert d <= GATE_TOL, (label, "gate", t, s, i, d)
            co, cg = ot["cost"][t, s], gt["cost"][t, s]
            worst["cost"] = max(worst["cost"], abs(co - cg) / max(co, 1e-300))
            assert abs(co - cg) <= COST_TOL * co + 1e-15, (label, "cost", t, s, co, cg)
    assert np.abs(gt["sigma"] - ot["sigma"]).max() <= 1e-10 * np.abs(ot["sigma"]).max()
    return worst


CASES = [
    # name, init, S, m (None = config m_init), sweeps, K override
    ("c1", "R", 1, None, 5, None),
    ("c2", "R", 32, None, 5, None),
    ("c2", "W", 8, 64, 5, None),
    ("c3", "R", 8, None, 5, None),
    ("c3", "W", 4, 32, 5, None),
    ("c4", "W", 2, None, 3, 40),
    ("c5b", "W", 1, 16, 3, 30),
    ("c5b", "W", 1, 32, 2, 30),   # resident: a 16-CTA cluster (the largest), mbarrier exchange over 16 ranks
]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name,init,s,m,sweeps,k", CASES)
def test_trace_parity(qfs, name, init, s, m, sweeps, k, path):
    p = I.make_problem(name, init=init, s=s, k=k)
    m = m or p.m_init
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, m, sweeps)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, m, sweeps)
    _compare_traces(gt, ot, f"{name}-{init}")


@pytest.mark.parametrize("path", PATHS)
def test_trace_parity_ragged_and_degenerate(qfs, path):
    """Ragged M (odd row counts), reversed / non-adjacent / repeated pairs, K=1, n=2."""
    rng = np.random.default_rng(5)
    for n, pairs, m in [(2, [[0, 1]], 3), (2, [[1, 0], [0, 1], [1, 0]], 4),
                        (5, [[4, 0], [0, 4], [2, 3], [3, 1], [1, 3], [0, 2]], 7),
                        (9, [[8, 0], [1, 2], [2, 1], [5, 7]], 5)]:
        pairs = np.asarray(pairs, np.int32)
        target = np.stack([unitary(rng) for _ in pairs])
        x = I.haar_states(rng, n, m)
        y = I.apply_circuit_tensor(n, pairs, target, x)
        init = np.stack([np.stack([unitary(rng) for _ in pairs]) for _ in range(3)])
        ctx = _ctx(qfs, n, pairs, path)
        ctx.set_samples(x, y)
        gt = ctx.trace_sweeps(init, m, 4)
        ot = oracle.trace_sweeps(n, pairs, init, x, y, m, 4)
        _compare_traces(gt, ot, f"ragged n={n}")


def test_trace_parity_streamed_forward_n14(qfs):
    """n = 14 takes the per-gate streamed forward (no whole row in SMEM)."""
    rng = np.random.default_rng(14)
    n = 14
    pairs = I.brick_pairs(n, 10)
    pairs[3] = [13, 0]
    target = np.stack([unitary(rng) for _ in pairs])
    x = I.haar_states(rng, n, 2)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    xv = I.haar_states(rng, n, 2)
    yv = I.apply_circuit_tensor(n, pairs, target, xv)
    init = np.stack([unitary(rng) for _ in pairs])[None]
    ctx = _ctx(qfs, n, pairs)
    ctx.set_samples(x, y, xv, yv)
    gt = ctx.trace_sweeps(init, 2, 2)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, 2, 2)
    _compare_traces(gt, ot, "n14")
    # controller with validation on the streamed path
    prm = dict(dist_tol=1e-8, diff_tol_r=1e-3, plateau_window=5, min_iter=6, max_iter=3, m_init=2,
               overtrain_ratio=1e300, beta=0.0, stop_on_first=1)
    g1, r1, w1 = ctx.instantiate(init, prm)
    g2, r2, w2 = oracle.instantiate(n, pairs, x, y, xv, yv, init, prm)
    assert abs(r1[0]["c_val"] - r2[0]["c_val"]) <= 1e-10 * r2[0]["c_val"]
    assert abs(r1[0]["c_train"] - r2[0]["c_train"]) <= 1e-10 * r2[0]["c_train"]


def test_full_size_c4_sampled_starts(qfs):
    """C4 at full size (S=16, M=32, K=150, n=12) in the bench's launch shape,
    the first 5 sweeps (north_star), all 16 starts recomputed by the oracle."""
    p = I.make_problem("c4", init="R")
    ctx = _ctx(qfs, p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, p.m_init, 5)
    pick = list(range(16))   # every start (the oracle runs them side by side on the host cores)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init[pick], p.x, p.y, p.m_init, 5, threads=min(16, os.cpu_count() or 1))
    sub = dict(env=gt["env"][:, :, pick], gates=gt["gates"][:, pick], cost=gt["cost"][:, pick],
               sigma=gt["sigma"][:, :, pick])
    _compare_traces(sub, ot, "c4-full")


def _no_stop(m, sweeps, otr=1e300):
    """Controller parameters that run exactly ``sweeps`` sweeps (validation every sweep)."""
    return dict(dist_tol=-1.0, diff_tol_r=1e-3, plateau_window=0, min_iter=10 ** 6, max_iter=sweeps,
                m_init=m, overtrain_ratio=otr, beta=0.0, stop_on_first=0)


def test_full_size_c4_validation_cost_streamed(qfs):
    """c_val on the streamed path's block validation kernel at
    the C4 bench shape (S=16, V=16, K=150): two sampled starts' c_val and
    c_train after 2 controller steps equal the oracle's within 1e-10."""
    p = I.make_problem("c4", init="R")
    ctx = _ctx(qfs, p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    prm = _no_stop(p.m_init, 2, otr=0.1)
    g1, r1, _ = ctx.instantiate(p.init, prm)
    pick = [3, 14]
    g2, r2, _ = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init[pick], prm, threads=2)
    for j, s in enumerate(pick):
        assert abs(r1[s]["c_val"] - r2[j]["c_val"]) <= COST_TOL * r2[j]["c_val"] + 1e-15, (s, r1[s], r2[j])
        assert abs(r1[s]["c_train"] - r2[j]["c_train"]) <= COST_TOL * r2[j]["c_train"] + 1e-15
        assert np.abs(g1[s] - g2[j]).max() <= GATE_TOL


def test_full_size_c5_first_sweeps(qfs):
    """C5 at full size (n=14, K=300, M=64, V=16, S=1; BASELINE.json configs[4]):
    the first 5 sweeps' environments, gates, costs and sigma sums, then c_val /
    c_train after 3 controller steps (the cluster validation kernel at the real
    K, the WIDE backward reduction at the real M) — all against the oracle."""
    p = I.make_problem("c5", init="R", s=1)
    assert (p.n, p.k, p.m_init, p.xv.shape[0]) == (14, 300, 64, 16)
    ctx = _ctx(qfs, p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, p.m_init, 5)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, p.m_init, 5)
    _compare_traces(gt, ot, "c5-full")
    prm = _no_stop(p.m_init, 2)
    g1, r1, _ = ctx.instantiate(p.init, prm)
    g2, r2, _ = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init, prm)
    assert abs(r1[0]["c_val"] - r2[0]["c_val"]) <= COST_TOL * r2[0]["c_val"]
    assert abs(r1[0]["c_train"] - r2[0]["c_train"]) <= COST_TOL * r2[0]["c_train"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name,init,s,m,k", [("c3", "R", 4, 16, None), ("c3", "W", 3, 32, None),
                                             ("c4", "R", 2, 32, 24)])
def test_trace_parity_beta(qfs, name, init, s, m, k, path):
    """beta-regularised update (reading R15): E' = (1 - beta) E +
    beta G_old^dag traced through whole sweeps at beta = 0.3 on both paths."""
    p = I.make_problem(name, init=init, s=s, k=k)
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, m, 4, beta=0.3)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, m, 4, beta=0.3)
    _compare_traces(gt, ot, f"beta-{name}-{init}")


@pytest.mark.parametrize("name", ["c3", "c5c"])
def test_full_size_resident_sampled_starts(qfs, name):
    """C3 and C5c at full size in the bench's launch configuration (auto path =
    cluster-resident, all 64 starts in one launch), the first 5 sweeps of every
    start recomputed by the oracle."""
    p = I.make_problem(name, init="R")
    pick = list(range(p.init.shape[0]))
    ctx = _ctx(qfs, p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, p.m_init, 5)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init[pick], p.x, p.y, p.m_init, 5, threads=min(16, os.cpu_count() or 1))
    sub = dict(env=gt["env"][:, :, pick], gates=gt["gates"][:, pick], cost=gt["cost"][:, pick],
               sigma=gt["sigma"][:, :, pick])
    _compare_traces(sub, ot, f"{name}-full")


@pytest.mark.parametrize("name,init,s,m", [("c3", "R", 8, None), ("c3", "W", 5, 32), ("c2", "R", 3, None)])
def test_trace_parity_resident_pair_kernel(qfs, monkeypatch, name, init, s, m):
    """The two-starts-per-cluster resident kernel (QFS_RES_PAIR=2: one start's
    polar overlapped with the other's passes; measured slower, not the
    default): traces vs the oracle, odd start counts (a pair with one start),
    and the validation cost of an instantiation step vs the default kernel."""
    p = I.make_problem(name, init=init, s=s)
    m = m or p.m_init
    monkeypatch.setenv("QFS_RES_PAIR", "2")            # read when the context is created
    ctx = qfs.Context(p.n, p.pairs)
    monkeypatch.delenv("QFS_RES_PAIR")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, m, 4)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, m, 4)
    _compare_traces(gt, ot, f"{name}-{init}-pair")
    ref = qfs.Context(p.n, p.pairs)
    ref.set_samples(p.x, p.y, p.xv, p.yv)
    prm = dict(p.params, max_iter=3, m_init=m)
    _, r1, _ = ctx.instantiate(p.init, prm)
    _, r2, _ = ref.instantiate(p.init, prm)
    for a, b in zip(r1, r2):
        assert abs(a["c_val"] - b["c_val"]) <= 1e-10 * max(b["c_val"], 1e-300)
        assert abs(a["c_train"] - b["c_train"]) <= 1e-10 * max(b["c_train"], 1e-300) + 1e-15
    ctx.close()
    ref.close()


# ----------------------------------------------------------- instantiation --
def _inst_both(qfs, p, prm, path="auto"):
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    g1, r1, w1 = ctx.instantiate(p.init, prm)
    g2, r2, w2 = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init, prm, threads=8)
    return (g1, r1, w1), (g2, r2, w2)


@pytest.mark.parametrize("path", PATHS)
def test_instantiate_c1_parity(qfs, path):
    """C1 as configured (500 sweeps, plateau off): same termination, sweeps, final cost."""
    p = I.make_problem("c1", init="R")
    (g1, r1, w1), (g2, r2, w2) = _inst_both(qfs, p, dict(p.params), path)
    assert r1[0]["term"] == r2[0]["term"] and r1[0]["sweeps"] == r2[0]["sweeps"]
    assert abs(r1[0]["c_train"] - r2[0]["c_train"]) <= 1e-7 * r2[0]["c_train"] + 1e-14


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name,s", [("c2", 4), ("c3", 2)])
def test_instantiate_warm_converges_and_matches(qfs, name, s, path):
    """Solvable-by-construction targets reach c_train <= 1e-8 on the GPU and the
    controller takes the same decisions as the oracle (termination, restarts,
    final M, sweep count within +-2; SURVEY §8(c) 'parity unpinned' rule)."""
    p = I.make_problem(name, init="W", s=s)
    prm = dict(p.params, max_iter=300)
    (g1, r1, w1), (g2, r2, w2) = _inst_both(qfs, p, prm, path)
    assert r1[w1]["term"] == "CONVERGED" and r1[w1]["c_train"] <= 1e-8
    assert r2[w2]["term"] == "CONVERGED" and r2[w2]["c_train"] <= 1e-8   # the oracle too
    assert w1 == w2
    for a, b in zip(r1, r2):
        assert a["term"] == b["term"] and a["restarts"] == b["restarts"] and a["final_m"] == b["final_m"]
        assert abs(a["sweeps"] - b["sweeps"]) <= 2


@pytest.mark.parametrize("path", PATHS)
def test_instantiate_restart_geometry_gpu(qfs, path):
    """Double-and-restart on the GPU path (C2 random init, per-start ragged M)."""
    p = I.make_problem("c2", init="R", s=6)
    prm = dict(p.params, max_iter=40, stop_on_first=0)
    (g1, r1, w1), (g2, r2, w2) = _inst_both(qfs, p, prm, path)
    assert any(r["restarts"] > 0 for r in r1)
    for a, b in zip(r1, r2):
        assert a["final_m"] == min(p.m_init * 2 ** a["restarts"], 64)
        assert a["term"] == b["term"] and a["restarts"] == b["restarts"]


@pytest.mark.parametrize("path", PATHS)
def test_winner_rule_gpu(qfs, path):
    """Winner rule on the constructed multistarts of the oracle pin
    (tests/test_oracle_pins.py::test_winner_rule_earliest_then_lowest_index):
    the earliest converged start wins over a later one with a lower c_train,
    identical starts tie to the lower index — the same winner and terminations
    as the oracle, with and without stop_on_first."""
    from test_oracle_pins import _winner_problem
    p, a, b = _winner_problem()
    init = np.stack([a, b, b])
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    for sof in (0, 1):
        prm = dict(p.params, max_iter=300, stop_on_first=sof)
        g1, r1, w1 = ctx.instantiate(init, prm)
        g2, r2, w2 = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, init, prm, threads=3)
        assert w1 == w2 == 1
        assert [r["term"] for r in r1] == [r["term"] for r in r2]
        assert r1[1]["sweeps"] == r1[2]["sweeps"] and abs(r1[1]["sweeps"] - r2[1]["sweeps"]) <= 2


@pytest.mark.parametrize("path", PATHS)
def test_deterministic_bitwise(qfs, path):
    p = I.make_problem("c3", init="R", s=8)
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    a = ctx.trace_sweeps(p.init, 16, 2)
    b = ctx.trace_sweeps(p.init, 16, 2)
    assert np.array_equal(a["gates"], b["gates"]) and np.array_equal(a["cost"], b["cost"])


@pytest.mark.parametrize("path", PATHS)
def test_instantiate_pinned_gate_buffers(qfs, path):
    """Pinned (page-locked) init / out gate buffers are read and written by the
    device in place; pageable ones go through the staging buffer: same bits,
    same results, and the caller's input buffer is left unchanged."""
    import torch
    p = I.make_problem("c3", init="R", s=4)
    prm = dict(p.params, max_iter=3)
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    g_pageable, r1, w1 = ctx.instantiate(p.init, prm)
    gin = torch.from_numpy(np.ascontiguousarray(p.init)).pin_memory().numpy()
    gout = torch.empty(tuple(p.init.shape), dtype=torch.complex128, pin_memory=True).numpy()
    _, r2, w2 = ctx.instantiate(gin, prm, out=gout)
    assert np.array_equal(gout, g_pageable) and w1 == w2 and r1 == r2
    assert np.array_equal(gin, p.init)


def test_launch_shape_independence(qfs):
    """A start's sweep does not depend on the batch it runs in beyond summation
    order: 4 starts in one launch (128-thread backward CTAs, 2 per SM, 37 per
    start) vs each start alone (256-thread CTAs, 148 per start, the all-warp
    WIDE reduction), streamed path; both within the oracle tolerances."""
    p = I.make_problem("c4", init="R", s=4, k=14)
    m = 32
    ctx = _ctx(qfs, p.n, p.pairs, "streamed")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    tb = ctx.trace_sweeps(p.init, m, 3)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, m, 3)
    for s in range(4):
        ts = ctx.trace_sweeps(p.init[s:s + 1], m, 3)
        for t in range(3):
            for i in range(p.k):
                eo = ot["env"][t, i, s]
                assert np.linalg.norm(tb["env"][t, i, s] - eo) <= ENV_TOL * np.linalg.norm(eo)
                assert np.linalg.norm(ts["env"][t, i, 0] - eo) <= ENV_TOL * np.linalg.norm(eo)
                assert np.linalg.norm(ts["env"][t, i, 0] - tb["env"][t, i, s]) <= 1e-12 * np.linalg.norm(eo)
            assert abs(ts["cost"][t, 0] - tb["cost"][t, s]) <= 1e-12 * tb["cost"][t, s] + 1e-15
    ctx.close()


def test_errors(qfs):
    from paper_2405_12866_b200.qfs import QfsError
    p = I.make_problem("c1")
    with pytest.raises(QfsError) as ei:
        qfs.Context(3, [[0, 0]])
    assert ei.value.status == 1
    ctx = _ctx(qfs, p.n, p.pairs)
    prm = dict(p.params)
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(p.init, prm)
    assert ei.value.status == 5           # ERR_STATE before set_samples
    ctx.set_samples(p.x, p.y)
    bad = p.init.copy()
    bad[0, 0] *= 1.5
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(bad, prm)
    assert ei.value.status == 3           # ERR_NUMERIC non-unitary gate
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(p.init, dict(prm, m_init=8))
    assert ei.value.status == 2           # ERR_CAPACITY m_init > m_pool
    nanx = p.x.copy()
    nanx[0, 0] = np.nan
    with pytest.raises(QfsError) as ei:
        ctx.set_samples(nanx, p.y)
    assert ei.value.status == 3


# ------------------------------------------------------------- distributed --
def test_sample_sharded_path_single_rank(qfs, monkeypatch):
    """qfs_create_nccl in sample mode with a one-rank communicator and
    QFS_UNFUSED_POLAR=1, so the multi-rank code path runs: per-gate NCCL
    all-reduce of E, separate polar kernel, all-reduced cost and validation
    sums — equal to the oracle and to the fused path."""
    p = I.make_problem("c3", init="W", s=4)
    nid = qfs.nccl_unique_id()
    monkeypatch.setenv("QFS_UNFUSED_POLAR", "1")       # read when the context is created
    ctx = qfs.Context(p.n, p.pairs, nccl_id=nid, rank=0, world=1, shard_mode=1)
    monkeypatch.delenv("QFS_UNFUSED_POLAR")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    fused = qfs.Context(p.n, p.pairs, nccl_id=qfs.nccl_unique_id(), rank=0, world=1, shard_mode=1)
    fused.set_path("streamed")           # same sweep path as the unfused context (never resident)
    fused.set_samples(p.x, p.y, p.xv, p.yv)
    l0, f0 = ctx.launch_count(), fused.launch_count()
    ctx.trace_sweeps(p.init, 32, 1)
    fused.trace_sweeps(p.init, 32, 1)
    # per sweep: K polar launches + K all-reduces of E + 1 of the cost sums
    assert (ctx.launch_count() - l0) - (fused.launch_count() - f0) == 2 * p.k + 1
    fused.close()
    gt = ctx.trace_sweeps(p.init, 32, 3)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, 32, 3)
    _compare_traces(gt, ot, "sample-mode")
    ref = _ctx(qfs, p.n, p.pairs)
    ref.set_samples(p.x, p.y, p.xv, p.yv)
    rt = ref.trace_sweeps(p.init, 32, 3)
    assert np.abs(rt["gates"] - gt["gates"]).max() < 1e-13
    g1, r1, w1 = ctx.instantiate(p.init, dict(p.params, max_iter=200))
    g2, r2, w2 = ref.instantiate(p.init, dict(p.params, max_iter=200))
    assert w1 == w2 and r1[w1]["term"] == "CONVERGED"
    assert [r["sweeps"] for r in r1] == [r["sweeps"] for r in r2]


def test_multistart_dist_path_single_rank(qfs):
    """qfs_create_nccl in multistart mode: per-sweep (any converged, any active)
    NCCL all-reduce in the controller; same decisions as the plain context."""
    p = I.make_problem("c2", init="W", s=4)
    ctx = qfs.Context(p.n, p.pairs, nccl_id=qfs.nccl_unique_id(), rank=0, world=1, shard_mode=0)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    g1, r1, w1 = ctx.instantiate(p.init, dict(p.params, max_iter=300))
    g2, r2, w2 = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init, dict(p.params, max_iter=300))
    assert w1 == w2 and r1[w1]["term"] == "CONVERGED"
    for a, b in zip(r1, r2):
        assert a["term"] == b["term"] and abs(a["sweeps"] - b["sweeps"]) <= 2


def test_resident_path_selection_and_validation(qfs):
    """Forced resident path: runs where the states fit (C3: cluster of 2 CTAs),
    fails with QFS_ERR_CAPACITY where they do not (n = 12, M = 32); its fused
    validation cost equals the oracle's."""
    from paper_2405_12866_b200.qfs import QfsError
    p = I.make_problem("c3", init="W", s=3)
    ctx = _ctx(qfs, p.n, p.pairs, "resident")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    prm = dict(p.params, max_iter=4, min_iter=100)
    g1, r1, w1 = ctx.instantiate(p.init, prm)
    g2, r2, w2 = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init, prm)
    for a, b in zip(r1, r2):
        assert abs(a["c_val"] - b["c_val"]) <= 1e-10 * b["c_val"]
        assert abs(a["c_train"] - b["c_train"]) <= 1e-10 * b["c_train"]
    q = I.make_problem("c4", init="R", s=1, k=8)
    big = _ctx(qfs, q.n, q.pairs, "resident")
    big.set_samples(q.x, q.y, q.xv, q.yv)
    with pytest.raises(QfsError) as ei:
        big.trace_sweeps(q.init, 32, 1)
    assert ei.value.status == 2
    with pytest.raises(QfsError) as ei:
        big.set_path(7)
    assert ei.value.status == 1


@pytest.mark.parametrize("path", PATHS)
def test_appendix_d_basis_vs_haar_training_states(qfs, path):
    """P:458-464 (App. D) on the GPU path: M = 4 computational-basis training
    states with qubit 0 fixed fit the R_z-first circuit without generalising
    (c_val > 0.1), M = 4 Haar states generalise; the Haar run matches the oracle."""
    from test_oracle_pins import _appendix_d_problem
    n, pairs, target, alpha, xb, xh, xv, ys, init, prm = _appendix_d_problem()
    for x, y, generalises in ((xb, ys["b"], False), (xh, ys["h"], True)):
        ctx = _ctx(qfs, n, pairs, path)
        ctx.set_samples(x, y, xv, ys["v"])
        g1, r1, _ = ctx.instantiate(init, prm)
        g2, r2, _ = oracle.instantiate(n, pairs, x, y, xv, ys["v"], init, prm)
        for a, b in zip(r1, r2):
            assert a["term"] == b["term"] == "MAX_ITER"
            if generalises:
                assert a["c_val"] < 1e-4
                assert abs(a["c_val"] - b["c_val"]) <= 1e-3 * b["c_val"] + 1e-12
                assert abs(a["c_train"] - b["c_train"]) <= 1e-3 * b["c_train"] + 1e-14
            else:
                assert a["c_train"] < 1e-5 and a["c_val"] > 0.1


@pytest.mark.parametrize("path", PATHS)
def test_u3_cnot_template_gate_kinds(qfs, path):
    """NEXT-3: the paper's U3 + CNOT templates (Table 1) through qfs_set_gate_kinds:
    one-qubit variable gates (u (x) I, 2x2 polar of the partial-traced
    environment) and fixed CNOTs; 4-sweep traces equal the oracle's, a warm
    instance converges with the CNOTs untouched, bad kinds / non-u(x)I slots fail."""
    from paper_2405_12866_b200.qfs import QfsError
    n, layers = 6, 4
    pairs, kinds, target, x, y, xv, yv, init = I.u3_cnot_problem(n, layers, s=3, m_pool=64, v=16, init="R")
    ctx = _ctx(qfs, n, pairs, path)
    ctx.set_gate_kinds(kinds)
    ctx.set_samples(x, y, xv, yv)
    gt = ctx.trace_sweeps(init, 8, 4)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, 8, 4, kinds=kinds)
    _compare_traces(gt, ot, f"u3cnot-{path}")
    fixed = np.nonzero(kinds == I.GATE_FIXED)[0]
    assert np.array_equal(gt["gates"][:, :, fixed], np.broadcast_to(I.CNOT, gt["gates"][:, :, fixed].shape))
    pw = I.u3_cnot_problem(n, layers, s=4, m_pool=64, v=16, init="W")
    ctx.set_samples(pw[3], pw[4], pw[5], pw[6])
    prm = dict(dist_tol=1e-8, diff_tol_r=1e-3, plateau_window=5, min_iter=6, max_iter=300, m_init=8,
               overtrain_ratio=0.1, beta=0.0, stop_on_first=1)
    g1, r1, w1 = ctx.instantiate(pw[7], prm)
    g2, r2, w2 = oracle.instantiate(n, pairs, pw[3], pw[4], pw[5], pw[6], pw[7], prm, kinds=kinds)
    assert r1[w1]["term"] == "CONVERGED" and r1[w1]["c_train"] <= 1e-8 and w1 == w2
    for a, b in zip(r1, r2):
        assert a["term"] == b["term"] and abs(a["sweeps"] - b["sweeps"]) <= 2
    assert np.array_equal(g1[w1][fixed], np.broadcast_to(I.CNOT, g1[w1][fixed].shape))
    with pytest.raises(QfsError) as ei:
        ctx.set_gate_kinds(np.full(len(kinds), 7))
    assert ei.value.status == 1
    bad = pw[7].copy()
    j = int(np.nonzero(kinds == I.GATE_VAR1)[0][0])
    bad[0, j] = I.haar_unitary(np.random.default_rng(3))   # a general 4x4 in a one-qubit slot
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(bad, prm)
    assert ei.value.status == 3


def test_set_samples_async_queue(qfs):
    """qfs_set_samples_async: queued sets are consumed oldest first by the next
    calls and give the same traces as qfs_set_samples; a third queued set is
    refused (QFS_ERR_STATE); a non-finite queued set fails the consuming call."""
    import torch
    from paper_2405_12866_b200.qfs import QfsError
    p = I.make_problem("c3", init="R", s=2, k=12)
    q = I.make_problem("c3", init="R", s=2, k=12, m_pool=256)
    ref = _ctx(qfs, p.n, p.pairs)
    ref.set_samples(p.x, p.y, p.xv, p.yv)
    want_p = ref.trace_sweeps(p.init, 16, 1)
    ref.set_samples(q.x, q.y, q.xv, q.yv)
    want_q = ref.trace_sweeps(p.init, 16, 1)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hp = [pin(a) for a in (p.x, p.y, p.xv, p.yv)]
    hq = [pin(a) for a in (q.x, q.y, q.xv, q.yv)]
    ctx = _ctx(qfs, p.n, p.pairs)
    for h in (hp, hq):
        ctx.set_samples_async_host_ptr(h[0].shape[0], h[0].data_ptr(), h[1].data_ptr(), h[2].shape[0],
                                       h[2].data_ptr(), h[3].data_ptr())
    with pytest.raises(QfsError) as ei:
        ctx.set_samples_async_host_ptr(hp[0].shape[0], hp[0].data_ptr(), hp[1].data_ptr(), 16,
                                       hp[2].data_ptr(), hp[3].data_ptr())
    assert ei.value.status == 5
    got_p = ctx.trace_sweeps(p.init, 16, 1)
    got_q = ctx.trace_sweeps(p.init, 16, 1)
    assert np.array_equal(got_p["env"], want_p["env"]) and np.array_equal(got_q["env"], want_q["env"])
    bad = pin(p.x)
    bad[0, 0] = float("nan")
    ctx.set_samples_async_host_ptr(bad.shape[0], bad.data_ptr(), hp[1].data_ptr(), 16, hp[2].data_ptr(),
                                   hp[3].data_ptr())
    with pytest.raises(QfsError) as ei:
        ctx.trace_sweeps(p.init, 16, 1)
    assert ei.value.status == 3


@pytest.mark.gpu
def test_set_structure_matches_fresh_context():
    """qfs_set_structure on a used context gives the same traces as a new context
    (smaller and larger gate counts, gate kinds reset)."""
    from paper_2405_12866_b200 import build, qfs
    build.build()
    p = I.make_problem("c2", init="R", s=3)
    ctx = qfs.Context(p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    ctx.trace_sweeps(p.init, p.m_init, 1)
    rng = np.random.default_rng(3)
    for k in (7, p.k + 6):
        pairs = I.brick_pairs(p.n, k)
        g0 = np.stack([[I.haar_unitary(rng) for _ in range(k)] for _ in range(3)])
        ctx.set_structure(pairs)
        a = ctx.trace_sweeps(g0, p.m_init, 2)
        fresh = qfs.Context(p.n, pairs)
        fresh.set_samples(p.x, p.y, p.xv, p.yv)
        b = fresh.trace_sweeps(g0, p.m_init, 2)
        fresh.close()
        assert np.array_equal(a["cost"], b["cost"]) and np.array_equal(a["gates"], b["gates"])
    ctx.close()


@pytest.mark.gpu
def test_set_structure_errors():
    from paper_2405_12866_b200 import build, qfs
    build.build()
    ctx = qfs.Context(4, I.brick_pairs(4, 3))
    with pytest.raises(qfs.QfsError):
        ctx.set_structure(np.array([[0, 0]], np.int32))      # repeated qubit
    with pytest.raises(qfs.QfsError):
        ctx.set_structure(np.array([[0, 4]], np.int32))      # qubit out of range
    ctx.set_structure(np.array([[1, 3], [0, 2]], np.int32))  # valid: accepted
    ctx.close()
    bq, ba = I.block_structure(5, 3)
    bctx = qfs.BlockContext(5, bq, ba)
    with pytest.raises(qfs.QfsError):
        bctx.set_structure(np.array([[0, 1]], np.int32))     # not for block circuits
    bctx.close()


@pytest.mark.parametrize("name,init,s,m,sweeps,k", [("c4", "W", 2, 32, 3, 40), ("c4", "R", 16, 32, 2, None),
                                                    ("c5", "R", 1, 64, 2, 60), ("c3", "R", 4, 16, 3, None),
                                                    ("c2", "W", 4, 48, 3, None)])
def test_trace_parity_bulk_copy_path(qfs, monkeypatch, name, init, s, m, sweeps, k):
    """Perm mode (QFS_BWD_BULK=1): B cache and chi in per-gate
    permuted sample-blocked layouts, the backward tiles moved by cp.async.bulk
    into an mbarrier ring (bwdt_kernel), the forward scattered into the next
    gates' layouts (fwdp_kernel) — equal to the oracle like the default path
    (ragged M = 48: a partial sample block)."""
    monkeypatch.setenv("QFS_BWD_BULK", "1")              # read when the context is created
    p = I.make_problem(name, init=init, s=s, k=k)
    ctx = _ctx(qfs, p.n, p.pairs, "streamed")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, m, sweeps)
    pick = list(range(s)) if s <= 4 else [0, s - 1]
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init[pick], p.x, p.y, m, sweeps, threads=len(pick))
    sub = dict(env=gt["env"][:, :, pick], gates=gt["gates"][:, pick], cost=gt["cost"][:, pick],
               sigma=gt["sigma"][:, :, pick])
    _compare_traces(sub, ot, f"bulk-{name}")
    prm = dict(p.params, max_iter=2, stop_on_first=0, dist_tol=-1.0, plateau_window=0, m_init=m)
    g1, r1, _ = ctx.instantiate(p.init, prm)
    g2, r2, _ = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init[pick], prm, threads=len(pick))
    for j, q in enumerate(pick):
        assert abs(r1[q]["c_train"] - r2[j]["c_train"]) <= COST_TOL * r2[j]["c_train"]


@pytest.mark.parametrize("n,k,m,v", [(16, 14, 32, 8), (18, 10, 16, 4)])
def test_large_n_streamed_with_validation(qfs, n, k, m, v):
    """Beyond the configs: n = 16 (validation on 8-CTA clusters, 1 MB rows) and
    n = 18 (rows too large for a cluster: the streamed per-gate validation +
    distance kernels), brick pairs plus a reversed long-range pair; two traced
    sweeps and the controller's c_val / c_train after two steps vs the oracle."""
    rng = np.random.default_rng(n)
    pairs = I.brick_pairs(n, k)
    pairs[k // 2] = [n - 1, 1]
    target = np.stack([unitary(rng) for _ in pairs])
    x = I.haar_states(rng, n, m)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    xv = I.haar_states(np.random.default_rng(n + 1), n, v)
    yv = I.apply_circuit_tensor(n, pairs, target, xv)
    init = np.stack([I.warm_gate(rng, target[j], 0.3) for j in range(k)])[None]
    ctx = _ctx(qfs, n, pairs)
    ctx.set_samples(x, y, xv, yv)
    gt = ctx.trace_sweeps(init, m, 2)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, m, 2)
    _compare_traces(gt, ot, f"n{n}")
    prm = _no_stop(m, 2)
    g1, r1, _ = ctx.instantiate(init, prm)
    g2, r2, _ = oracle.instantiate(n, pairs, x, y, xv, yv, init, prm)
    assert abs(r1[0]["c_val"] - r2[0]["c_val"]) <= COST_TOL * r2[0]["c_val"] + 1e-15
    assert abs(r1[0]["c_train"] - r2[0]["c_train"]) <= COST_TOL * r2[0]["c_train"] + 1e-15


@pytest.mark.parametrize("path", PATHS)
def test_empty_and_degenerate_calls_leave_context_usable(qfs, path):
    """Empty inputs (no sample rows, no starts, no sweeps, m = 0, max_iter = 0)
    are refused with QFS_ERR_ARG / QFS_ERR_CAPACITY before any device work,
    a zero-sweep trace only reports gate validity, and
    the sample set uploaded before them is still the one the next call uses:
    its traces equal the oracle's (P:112 sweep; include/qfs.h error codes)."""
    from paper_2405_12866_b200.qfs import QfsError
    p = I.make_problem("c1")
    ctx = _ctx(qfs, p.n, p.pairs, path)
    ctx.set_samples(p.x, p.y)
    empty = np.zeros((0, 1 << p.n), np.complex128)
    with pytest.raises(QfsError) as ei:
        ctx.set_samples(empty, empty)              # m_pool = 0
    assert ei.value.status == 1
    with pytest.raises(QfsError) as ei:
        ctx.trace_sweeps(p.init[:0], p.m_init, 2)  # S = 0 starts
    assert ei.value.status == 1
    with pytest.raises(QfsError) as ei:
        ctx.trace_sweeps(p.init, 0, 2)             # m = 0 rows
    assert ei.value.status == 2
    with pytest.raises(QfsError) as ei:
        ctx.trace_sweeps(p.init, p.x.shape[0] + 1, 2)  # m beyond the pool
    assert ei.value.status == 2
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(p.init, dict(p.params, max_iter=0))
    assert ei.value.status == 1
    with pytest.raises(QfsError) as ei:
        ctx.instantiate(p.init, dict(p.params, m_init=0))
    assert ei.value.status == 2
    z = ctx.trace_sweeps(p.init, p.m_init, 0)      # zero sweeps: nothing written
    assert z["cost"].shape == (0, p.init.shape[0])
    m = p.m_init
    gt = ctx.trace_sweeps(p.init, m, 3)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, m, 3)
    _compare_traces(gt, ot, f"after refused calls ({path})")
    ctx.close()
