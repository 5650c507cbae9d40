"""Fixed vs per-step cost of one qfs_instantiate call (the bench's timed
region) on short-sweep configs: device time (CUDA events on the library
stream) and host wall time for max_iter = 1, 2, 5, 10, 20, 50 steps, three
repeats each, and a least-squares fit  t(steps) = fixed + steps * per_step.

    python tools/step_overhead.py [config ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    build.build()
    for cfg in sys.argv[1:] or ["c3"]:
        p = I.make_problem(cfg, init="R")
        m = p.m_init
        ctx = qfs.Context(p.n, p.pairs)
        ctx.set_samples(p.x, p.y, p.xv, p.yv)
        stream = torch.cuda.ExternalStream(ctx.stream_ptr())
        g, _, _ = ctx.instantiate(p.init, bench.bench_params(3, m))
        pts = []
        for steps in (1, 2, 5, 10, 20, 50):
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                e0.record(stream)
                g, _, _ = ctx.instantiate(g, bench.bench_params(steps, m))
                e1.record(stream)
                e1.synchronize()
                wall = time.perf_counter() - t0
                pts.append((steps, e0.elapsed_time(e1) * 1e-3, wall))
        a = np.array(pts)
        X = np.stack([np.ones(len(a)), a[:, 0]], 1)
        fd, sd = np.linalg.lstsq(X, a[:, 1], rcond=None)[0]
        fw, sw = np.linalg.lstsq(X, a[:, 2], rcond=None)[0]
        print(json.dumps({"config": cfg, "device_fixed_us": round(fd * 1e6, 1), "device_per_step_us": round(sd * 1e6, 1),
                          "wall_fixed_us": round(fw * 1e6, 1), "wall_per_step_us": round(sw * 1e6, 1),
                          "points": [(int(s), round(d * 1e6, 1), round(w * 1e6, 1)) for s, d, w in pts]}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
