"""GPU checks of the library's guards:
buffer re-planning when a structure grows within its allocation, the 32-bit
offset limit of the streamed kernels (clean QFS_ERR_CAPACITY, never silent
wrap-around), and the -DQFS_DEBUG build whose device bounds checks trap on an
out-of-range offset (compute-sanitizer is closed on this pool)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2405_12866_b200 import inputs as I

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def Q():
    from paper_2405_12866_b200 import build, qfs
    build.build()
    return qfs


def test_set_structure_shrink_run_grow_within_alloc(Q):
    """create with K = 10, shrink to 3 and run (gate / state
    buffers now sized for 3), grow to 8 (still within the pair allocation of
    10) and run: the gates, B cache and sigma buffers must be re-planned; the
    traces equal a fresh context's bit for bit."""
    p = I.make_problem("c2", init="R", s=3, k=10)
    ctx = Q.Context(p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    rng = np.random.default_rng(8)
    for path in ("streamed", "auto"):
        ctx.set_path(path)
        for k in (3, 8, 10, 5, 9):
            pairs = I.brick_pairs(p.n, k)
            g0 = np.stack([[I.haar_unitary(rng) for _ in range(k)] for _ in range(3)])
            ctx.set_structure(pairs)
            a = ctx.trace_sweeps(g0, p.m_init, 2)
            fresh = Q.Context(p.n, pairs)
            fresh.set_path(path)
            fresh.set_samples(p.x, p.y, p.xv, p.yv)
            b = fresh.trace_sweeps(g0, p.m_init, 2)
            fresh.close()
            assert np.array_equal(a["cost"], b["cost"]) and np.array_equal(a["gates"], b["gates"])
            assert np.array_equal(a["env"], b["env"]) and np.array_equal(a["sigma"], b["sigma"])
            ga, ra, _ = ctx.instantiate(g0, dict(p.params, max_iter=3))
            gb, rb, _ = oracle.instantiate(p.n, pairs, p.x, p.y, p.xv, p.yv, g0, dict(p.params, max_iter=3))
            for x, y in zip(ra, rb):
                assert abs(x["c_val"] - y["c_val"]) <= 1e-10 * y["c_val"]
    ctx.close()


def test_offsets_guard_n20(Q):
    """n = 20 with a 256-row pool: 2^20 * 256 * 16 B = 4 GiB reaches the 32-bit
    offsets of the streamed kernels -> QFS_ERR_CAPACITY before any byte is read
    (small dummy buffers are passed; the check precedes every copy).  Just
    below the limit (a 4-row pool, M = 4, K = 3) the sweep matches the oracle."""
    n = 20
    pairs = np.array([[0, 19], [5, 6], [19, 3]], np.int32)
    ctx = Q.Context(n, pairs)
    dummy = np.zeros(16, np.complex128)
    ptr = dummy.ctypes.data
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_samples_host_ptr(256, ptr, ptr, 0, 0, 0)
    assert ei.value.status == 2
    with pytest.raises(Q.QfsError) as ei:
        ctx.set_samples_host_ptr(4, ptr, ptr, 256, ptr, ptr)   # validation rows count too
    assert ei.value.status == 2
    rng = np.random.default_rng(20)
    target = np.stack([I.haar_unitary(rng) for _ in pairs])
    x = I.haar_states(rng, n, 4)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    init = np.stack([I.haar_unitary(rng) for _ in pairs])[None]
    ctx.set_samples(x, y)
    gt = ctx.trace_sweeps(init, 4, 1)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, 4, 1)
    for i in range(3):
        eo = ot["env"][0, i, 0]
        assert np.linalg.norm(gt["env"][0, i, 0] - eo) <= 1e-10 * np.linalg.norm(eo)
    assert abs(gt["cost"][0, 0] - ot["cost"][0, 0]) <= 1e-10 * ot["cost"][0, 0]
    ctx.close()


_DEBUG_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2405_12866_b200 import inputs as I, qfs
assert qfs.LIB_PATH.endswith("libqfs_debug.so"), qfs.LIB_PATH
for name, s, k in (("c4", 3, 20), ("c3", 2, 12), ("c5", 1, 12)):
    p = I.make_problem(name, init="R", s=s, k=k)
    ctx = qfs.Context(p.n, p.pairs)
    ctx.set_path("streamed")
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    gt = ctx.trace_sweeps(p.init, p.m_init, 2)
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, p.m_init, 2, threads=s)
    err = np.abs(gt["env"] - ot["env"]).max() / np.abs(ot["env"]).max()
    assert err <= 1e-10, (name, err)
    prm = dict(p.params, max_iter=2, stop_on_first=0, dist_tol=-1.0)
    ctx.instantiate(p.init, prm)
    ctx.close()
print("debug-build ok")
"""


def test_debug_build_bounds_checks():
    """The -DQFS_DEBUG library (device bounds checks on the streamed kernels'
    offsets) runs the streamed sweep of C3 / C4 / C5 shapes, with validation,
    without tripping a check, and agrees with the oracle."""
    from paper_2405_12866_b200 import build
    build.build(debug=True)
    env = dict(os.environ, QFS_LIB="debug")
    r = subprocess.run([sys.executable, "-c", _DEBUG_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "debug-build ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
