"""Per-gate cost of the environment exchange in sample mode (SURVEY.md §8(e),
§8(f) NEXT-2), on ONE B200:

  single   one rank, M rows, the environment reduced on the device (no exchange)
  nccl     qfs_create_nccl(sample mode) with QFS_UNFUSED_POLAR=1 on a one-rank
           communicator: the host-enqueued path of real ranks — per gate a
           partial-E launch, ncclAllReduce of E, a polar launch
  emul-g   qfs_create_emulated(g): g ranks of M/g rows in the same launches,
           device-initiated exchange through mailboxes (the code path of real
           ranks minus NVLink latency)

Times are CUDA events around the backward phase inside the sweep (one event
pair per phase), divided by the gates; the work (M x 2^n amplitude-samples per
gate) is the same in every row.  Writes one JSON line per case.

    python tools/xchg_bench.py [config] [sweeps] > profiles/r2_exchange.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402


def phase(ctx, init, m, sweeps):
    ctx.bench_sweeps(init, m, 2)              # warm-up (graph capture, allocations)
    ctx.profile_enable(True)
    ctx.bench_sweeps(init, m, 2)              # instrumented graph
    ctx.profile_enable(True)
    sec = ctx.bench_sweeps(init, m, sweeps)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    return sec, prof


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    build.build()
    p = I.make_problem(cfg, init="R", s=1)
    m, K = p.m_init, p.k
    cases = [("single", {}), ("nccl", {"nccl": True})] + [(f"emul-{g}", {"g": g}) for g in (2, 4, 8) if m % g == 0]
    for name, o in cases:
        if o.get("nccl"):
            os.environ["QFS_UNFUSED_POLAR"] = "1"
            ctx = qfs.Context(p.n, p.pairs, nccl_id=qfs.nccl_unique_id(), rank=0, world=1, shard_mode=1)
            os.environ.pop("QFS_UNFUSED_POLAR")
        elif "g" in o:
            ctx = qfs.Context(p.n, p.pairs, emulated_ranks=o["g"])
        else:
            ctx = qfs.Context(p.n, p.pairs)
        ctx.set_path("streamed")
        ctx.set_samples(p.x, p.y)
        sec, prof = phase(ctx, p.init, m, sweeps)
        b = prof["bwd"]
        line = {"config": cfg, "case": name, "n": p.n, "k": K, "m": m, "ranks": o.get("g", 1),
                "sweep_ms": round(sec / sweeps * 1e3, 4),
                "bwd_phase_us_per_gate": round(b["ms"] / sweeps / K * 1e3, 3),
                "bwd_launches_per_sweep": b["launches"] // sweeps,
                "start_sweeps_per_s": round(sweeps / sec, 2)}
        print(json.dumps(line), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
