"""Small sweeps of every kernel path (streamed and resident sweeps, sample-sharded
polar, gate kinds, validation, unit ops) in one process: a quick all-paths run.
(compute-sanitizer is closed on this GPU pool, so this is not run under it.)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402

build.build()
prm = lambda p, it: dict(p.params, max_iter=it, min_iter=1, stop_on_first=0)
for name, k, s in (("c2", 8, 3), ("c3", 8, 2), ("c4", 6, 2)):
    p = I.make_problem(name, init="R", s=s, k=k)
    for path in ("streamed", "auto"):
        ctx = qfs.Context(p.n, p.pairs)
        ctx.set_path(path)
        ctx.set_samples(p.x, p.y, p.xv, p.yv)
        ctx.trace_sweeps(p.init, p.m_init, 1)
        ctx.instantiate(p.init, prm(p, 2))
        ctx.close()
        print(name, path, "ok", flush=True)
pairs, kinds, target, x, y, xv, yv, init = I.u3_cnot_problem(5, 2, s=2, m_pool=8, v=4)
for path in ("streamed", "auto"):
    ctx = qfs.Context(5, pairs)
    ctx.set_path(path)
    ctx.set_gate_kinds(kinds)
    ctx.set_samples(x, y, xv, yv)
    ctx.trace_sweeps(init, 4, 1)
    ctx.close()
    print("kinds", path, "ok", flush=True)
p = I.make_problem("c3", init="W", s=2, k=6)
ctx = qfs.Context(p.n, p.pairs, nccl_id=qfs.nccl_unique_id(), rank=0, world=1, shard_mode=1)
ctx.set_samples(p.x, p.y, p.xv, p.yv)
ctx.trace_sweeps(p.init, 16, 1)
ctx.close()
print("sample-mode ok", flush=True)
rng = np.random.default_rng(0)
ctx = qfs.Context(6, [[0, 1]])
psi = rng.standard_normal((3, 64)) + 1j * rng.standard_normal((3, 64))
ctx.op_apply(2, 5, I.haar_unitary(rng), psi)
ctx.op_environment(1, 3, psi, psi)
ctx.op_polar(rng.standard_normal((9, 4, 4)) + 0j, np.stack([np.eye(4)] * 9))
ctx.close()
print("unit ops ok", flush=True)
