"""Time the half-warp Jacobi polar kernel (K3) alone: one launch of `count`
seeded 4x4 environments, through qfs_op_polar (used for ncu captures)."""
import sys
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2405_12866_b200 import build, qfs, inputs as I

build.build()
count = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(1)
E = (rng.standard_normal((count, 4, 4)) + 1j * rng.standard_normal((count, 4, 4)))
G0 = np.stack([I.haar_unitary(rng) for _ in range(count)])
ctx = qfs.Context(2, [[0, 1]])
for _ in range(3):
    g, s = ctx.op_polar(E, G0)
ctx.profile_enable(True)
for _ in range(20):
    g, s = ctx.op_polar(E, G0)
p = ctx.profile_read()["unit_op"]
print(f"polar_batch count={count}: {p['ms'] / p['launches'] * 1e3:.2f} us per launch (CUDA events)")
