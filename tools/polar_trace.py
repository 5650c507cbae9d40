"""Diagnostic: per-gate polar path and cost on real sweep environments.  Build
with QFS_NVCC_DEFINES=-DQFS_DIAG_POLAR: the sum-sigma trace then carries
(Jacobi sweeps or 100 for Newton-Schulz) * 1e7 + clock64 cycles of hw_polar."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs
build.build()
CASES = [tuple(a.split(":")) for a in sys.argv[1:]] or [("c4", "R"), ("c3", "R"), ("c3", "W"), ("c2", "R")]
for cfg, init in CASES:
    p = I.make_problem(cfg, init=init)
    ctx = qfs.Context(p.n, p.pairs)
    ctx.set_samples(p.x, p.y, p.xv, p.yv)
    t = ctx.trace_sweeps(p.init, p.m_init, 3, env=False)
    sg = t["sigma"][1:].ravel()           # sweeps 2-3
    kind = np.floor(sg / 1e7)
    cyc = sg - kind * 1e7
    ns = kind == 100
    print(f"{cfg} {init}: NS {ns.mean():.2f} (cycles {cyc[ns].mean() if ns.any() else 0:.0f}), "
          f"Jacobi {1 - ns.mean():.2f} (sweeps {kind[~ns].mean() if (~ns).any() else 0:.1f}, "
          f"cycles {cyc[~ns].mean() if (~ns).any() else 0:.0f})", flush=True)
