"""Device-initiated exchange of the environments in sample mode (SURVEY.md
§8(f) NEXT-2; qfs_set_exchange / qfs_create_emulated).

gpurun offers one GPU, and ranks whose kernels wait on one another must not
run as separate launches on one device (B200_PROFILING.md), so the protocol
is exercised with EMULATED ranks: g ranks on one device, each with its own
pool rows m = r (mod g), states and gate copy, all in the same launches; the
last CTA of each rank's reduction stores its partial E into every rank's
mailbox, raises an epoch flag, waits for the others and sums in rank order —
the exact code path of real ranks, whose peer mailboxes are CUDA-IPC mappings
(tests/test_gpu_multi.py runs that with >= 2 GPUs).  E is a sum over samples
(P:121-125), so the result equals the single-rank sweep up to the order of
that sum.
"""
import numpy as np
import pytest

import oracle
from paper_2405_12866_b200 import inputs as I

pytestmark = pytest.mark.gpu

ENV_TOL, GATE_TOL, COST_TOL = 1e-10, 2e-10, 1e-10


@pytest.fixture(scope="module")
def Q():
    from paper_2405_12866_b200 import build, qfs
    build.build()
    return qfs


def _problem(n, k, m_pool, v, seed, init="R"):
    rng = np.random.default_rng(seed)
    pairs = I.brick_pairs(n, k)
    target = np.stack([I.haar_unitary(rng) for _ in pairs])
    x = I.haar_states(rng, n, m_pool)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    xv = I.haar_states(np.random.default_rng(seed + 1), n, v)
    yv = I.apply_circuit_tensor(n, pairs, target, xv)
    if init == "R":
        g0 = np.stack([I.haar_unitary(rng) for _ in pairs])[None]
    else:
        g0 = np.stack([I.warm_gate(rng, target[j], 0.3) for j in range(k)])[None]
    return pairs, x, y, xv, yv, g0


def _check(gt, ot, label):
    T, K = ot["env"].shape[:2]
    for t in range(T):
        for i in range(K):
            eo = ot["env"][t, i, 0]
            r = np.linalg.norm(gt["env"][t, i, 0] - eo) / np.linalg.norm(eo)
            assert r <= ENV_TOL, (label, t, i, r)
            sv = np.linalg.svd(eo, compute_uv=False)
            if sv[-1] / sv[0] >= 1e-8:
                assert np.linalg.norm(gt["gates"][t, 0, i] - ot["gates"][t, 0, i]) <= GATE_TOL, (label, t, i)
        assert abs(gt["cost"][t, 0] - ot["cost"][t, 0]) <= COST_TOL * ot["cost"][t, 0] + 1e-15


@pytest.mark.parametrize("n,k,m,g", [(9, 24, 32, 2), (9, 24, 32, 4), (9, 24, 32, 8), (9, 24, 16, 8),
                                     (12, 20, 64, 4), (14, 16, 64, 8)])
def test_emulated_ranks_trace_parity(Q, n, k, m, g):
    """Traces through the device exchange equal the oracle (1e-10) and the
    single-rank sweep (1e-12), from 2 rows per rank (the LDGSTS kernel) to 16
    (and the WIDE reduction at n = 14)."""
    pairs, x, y, xv, yv, g0 = _problem(n, k, m, 8, seed=n * 100 + g)
    ctx = Q.Context(n, pairs, emulated_ranks=g)
    ctx.set_samples(x, y, xv, yv)
    gt = ctx.trace_sweeps(g0, m, 3)
    ot = oracle.trace_sweeps(n, pairs, g0, x, y, m, 3)
    _check(gt, ot, f"emul-g{g}-n{n}")
    one = Q.Context(n, pairs)
    one.set_path("streamed")
    one.set_samples(x, y, xv, yv)
    rt = one.trace_sweeps(g0, m, 3)
    assert np.abs(gt["gates"] - rt["gates"]).max() <= 1e-12
    assert np.abs(gt["cost"] - rt["cost"]).max() <= 1e-12 * rt["cost"].max()
    ctx.close()
    one.close()


def test_emulated_ranks_instantiate(Q):
    """The controller over emulated ranks (costs summed over the ranks, c_val
    from the full validation set) takes the oracle's decisions on a warm C3
    instance: converged, same restarts / final M, c_val within 1e-9."""
    p = I.make_problem("c3", init="W", s=1, k=60)
    prm = dict(p.params, max_iter=300)
    ctx = Q.Context(p.n, p.pairs, emulated_ranks=4)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    g1, r1, w1 = ctx.instantiate(p.init, prm)
    g2, r2, w2 = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init, prm)
    assert r1[0]["term"] == r2[0]["term"] == "CONVERGED" and r1[0]["c_train"] <= 1e-8
    assert r1[0]["restarts"] == r2[0]["restarts"] and r1[0]["final_m"] == r2[0]["final_m"]
    assert abs(r1[0]["sweeps"] - r2[0]["sweeps"]) <= 2
    # repeated calls reuse the mailboxes (epochs keep increasing): same result
    g3, r3, _ = ctx.instantiate(p.init, prm)
    assert np.array_equal(g1, g3) and r1 == r3
    ctx.close()


def test_exchange_errors(Q):
    pairs = I.brick_pairs(6, 8)
    ctx = Q.Context(6, pairs, emulated_ranks=2)
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_exchange(0)                      # emulated ranks exchange on the device only
    assert ei.value.status == 1
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_exchange(3)
    assert ei.value.status == 1
    x = I.haar_states(np.random.default_rng(1), 6, 8)
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_samples(x[:7], x[:7])            # 7 rows over 2 ranks
    assert ei.value.status == 2
    ctx.set_samples(x, x)
    g0 = np.stack([I.haar_unitary(np.random.default_rng(2)) for _ in pairs])
    with pytest.raises(Q.QfsError) as ei:
        ctx.trace_sweeps(np.stack([g0, g0]), 8, 1)  # one start per call
    assert ei.value.status == 1
    ctx.close()
    with pytest.raises(Q.QfsError):
        Q.Context(6, pairs, emulated_ranks=64)
