"""Two ranks on two GPUs (skipped on a box with fewer GPUs —
gpurun offers one, so the host logic of the multi-rank paths is covered by
tests/test_parallel_gloo.py on CPU and the one-rank NCCL path by
test_gpu_parity.py::test_sample_sharded_path_single_rank).

* sample mode (qfs_create_nccl mode 1): rank r holds pool / validation rows
  m = r (mod 2); per gate the partial environments are all-reduced.  The
  sweep equals the one-rank sweep within 1e-12 (only the summation order of
  E differs) and the oracle within the parity tolerances.
* multistart mode: each rank runs its starts; results are bitwise identical
  to one rank running the same starts.
* sample mode with the device-initiated exchange (qfs_set_exchange, NEXT-2):
  the ranks' mailboxes mapped over CUDA IPC; identical gate bits on both
  ranks, equal to the NCCL path within 1e-12.
"""
import os
import pickle

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2405_12866_b200 import build, inputs as I, parallel as PL, qfs
    build.build()
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = I.make_problem("c3", init="W", s=3, k=24)
    rows, vrows = PL.sample_rows(p.x.shape[0], rank, world), PL.sample_rows(p.xv.shape[0], rank, world)
    obj = [qfs.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = qfs.Context(p.n, p.pairs, device=rank, nccl_id=obj[0], rank=rank, world=world, shard_mode=1)
    ctx.set_samples(p.x[rows], p.y[rows], p.xv[vrows], p.yv[vrows])
    tr = ctx.trace_sweeps(p.init, 32, 3)
    g, res, win = ctx.instantiate(p.init, dict(p.params, max_iter=200))
    ctx.close()
    # the device-initiated exchange (NEXT-2): peer mailboxes mapped with CUDA IPC
    obj = [qfs.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    dx = qfs.Context(p.n, p.pairs, device=rank, nccl_id=obj[0], rank=rank, world=world, shard_mode=1)
    dx.set_exchange("device")
    dx.set_samples(p.x[rows], p.y[rows], p.xv[vrows], p.yv[vrows])
    trx = dx.trace_sweeps(p.init, 32, 3)
    dx.close()
    # multistart: this rank's slice of 4 starts
    sl = PL.start_slice(4, rank, world)
    q = I.make_problem("c3", init="R", s=4, k=24)
    mc = qfs.Context(q.n, q.pairs, device=rank)
    mc.set_samples(q.x, q.y, q.xv, q.yv)
    mt = mc.trace_sweeps(q.init[sl.start:sl.stop], 16, 2)
    mc.close()
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(dict(tr=tr, trx=trx, res=res, win=win, mt=mt, sl=(sl.start, sl.stop)), f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (gpurun offers 1)")
def test_two_ranks_sample_and_multistart(tmp_path):
    import socket
    import torch.multiprocessing as mp
    import oracle
    from paper_2405_12866_b200 import build, inputs as I, qfs
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r = [pickle.load(open(tmp_path / f"r{k}.pkl", "rb")) for k in range(2)]
    build.build()
    p = I.make_problem("c3", init="W", s=3, k=24)
    one = qfs.Context(p.n, p.pairs)
    one.set_samples(p.x, p.y, p.xv, p.yv)
    ref = one.trace_sweeps(p.init, 32, 3)
    g1, res1, w1 = one.instantiate(p.init, dict(p.params, max_iter=200))
    for k in range(2):   # identical gate bits on both ranks, = one rank within 1e-12
        assert np.array_equal(r[k]["tr"]["gates"], r[0]["tr"]["gates"])
        assert np.abs(r[k]["tr"]["gates"] - ref["gates"]).max() <= 1e-12
        assert np.abs(r[k]["tr"]["cost"] - ref["cost"]).max() <= 1e-12 * ref["cost"].max()
        assert r[k]["win"] == w1 and r[k]["res"][w1]["term"] == "CONVERGED"
        assert abs(r[k]["res"][w1]["c_val"] - res1[w1]["c_val"]) <= 1e-9 * res1[w1]["c_val"]
    ot = oracle.trace_sweeps(p.n, p.pairs, p.init, p.x, p.y, 32, 3)
    assert np.abs(r[0]["tr"]["env"] - ot["env"]).max() <= 1e-10 * np.abs(ot["env"]).max()
    for k in range(2):   # device exchange: identical bits on both ranks, = the NCCL path within 1e-12
        assert np.array_equal(r[k]["trx"]["gates"], r[0]["trx"]["gates"])
        assert np.abs(r[k]["trx"]["gates"] - r[k]["tr"]["gates"]).max() <= 1e-12
        assert np.abs(r[k]["trx"]["env"] - ot["env"]).max() <= 1e-10 * np.abs(ot["env"]).max()
    q = I.make_problem("c3", init="R", s=4, k=24)
    mq = qfs.Context(q.n, q.pairs)
    mq.set_samples(q.x, q.y, q.xv, q.yv)
    for k in range(2):   # multistart: bitwise equal to one rank running the same starts
        a, b = r[k]["sl"]
        want = mq.trace_sweeps(q.init[a:b], 16, 2)
        assert np.array_equal(r[k]["mt"]["gates"], want["gates"])
        assert np.array_equal(r[k]["mt"]["cost"], want["cost"])
