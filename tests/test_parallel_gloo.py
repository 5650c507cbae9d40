"""Multi-process host logic on CPU (gloo, world size 2): multistart sharding,
result gather and winner rule, and the sample-axis all-reduce of partial
environments.  The per-rank compute engine here is the CPU
oracle (tests may use it); in production it is libqfs on each rank's GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2405_12866_b200 import inputs as I
from paper_2405_12866_b200 import parallel as PL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, kind, out_q)
    except Exception as e:  # report instead of hanging the parent
        out_q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, kind, out_q):
    if kind == "multistart":
        p = I.make_problem("c2", init="W", s=6)
        prm = dict(p.params, max_iter=300)

        def engine(init_local, params):
            return oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, init_local, params, threads=2)

        res, gates, win = PL.run_multistart(engine, p.init, prm, rank, world)
        flag = PL.any_flag(rank == 1, world)
        out_q.put((rank, res, gates, win, flag))
    elif kind == "resynth":
        from paper_2405_12866_b200 import resynth as R
        from test_resynth import OracleContext, PRM
        blocks = [R.redundant_block(3, 2, seed=10 + q, extra=1) for q in range(3)]

        def gather(mine):
            objs = [None] * world
            dist.all_gather_object(objs, mine)
            return objs

        rep = R.resynth_partitions(blocks, PRM, rank, world, gather=gather, starts=2,
                                   context_factory=OracleContext)
        out_q.put((rank, [(p_, r.deleted, r.kept) for p_, r in rep]))
    else:
        import torch
        p = I.make_problem("c3", init="R", s=1)
        M = 16
        rows = PL.sample_rows(M, rank, world)
        assert len(rows) == PL.local_prefix(M, world)
        i = 7
        B = oracle.circuit_forward(p.n, p.pairs[:i], p.init[0, :i], p.x[:M])
        chi = p.y[:M].copy()
        for k in range(p.k - 1, i, -1):
            chi = oracle.apply_gate(p.n, int(p.pairs[k][0]), int(p.pairs[k][1]), p.init[0, k], chi, dagger=True)
        pi0, pi1 = int(p.pairs[i][0]), int(p.pairs[i][1])
        part = oracle.environment(p.n, pi0, pi1, B[rows], chi[rows])
        t = torch.from_numpy(np.stack([part.real, part.imag]))
        dist.all_reduce(t)
        full = oracle.environment(p.n, pi0, pi1, B, chi)
        out_q.put((rank, np.abs(t[0].numpy() + 1j * t[1].numpy() - full).max() / np.abs(full).max()))


def _run(kind, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p_ in ps:
        p_.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for o in outs:
        assert not (len(o) == 3 and o[1] == "error"), o
    for p_ in ps:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    return sorted(outs, key=lambda t: t[0])


def test_shard_helpers():
    assert list(PL.start_slice(10, 0, 3)) == [0, 1, 2]
    assert list(PL.start_slice(10, 2, 3)) == [6, 7, 8, 9]
    assert sum(len(PL.start_slice(10, r, 3)) for r in range(3)) == 10
    assert list(PL.sample_rows(8, 1, 2)) == [1, 3, 5, 7]
    with pytest.raises(ValueError):
        PL.local_prefix(6, 4)
    res = [dict(term="PLATEAU", sweeps=9, c_train=0.3), dict(term="CONVERGED", sweeps=12, c_train=1e-9),
           dict(term="CONVERGED", sweeps=10, c_train=2e-9), dict(term="CONVERGED", sweeps=10, c_train=1e-10)]
    assert PL.select_winner(res) == 2
    assert PL.select_winner([dict(term="PLATEAU", sweeps=3, c_train=c) for c in (0.5, 0.2, 0.2)]) == 1


def test_multistart_gloo_matches_single_process():
    outs = _run("multistart")
    (r0, res0, g0, w0, f0), (r1, res1, g1, w1, f1) = outs
    assert w0 == w1 and f0 and f1
    assert np.array_equal(g0, g1)
    p = I.make_problem("c2", init="W", s=6)
    g, res, win = oracle.instantiate(p.n, p.pairs, p.x, p.y, p.xv, p.yv, p.init,
                                     dict(p.params, max_iter=300), threads=4)
    assert w0 == win
    assert res0[win]["term"] == "CONVERGED" and res0[win]["sweeps"] == res[win]["sweeps"]
    assert np.abs(g0[win] - g[win]).max() == 0.0


def test_sample_shard_allreduce_gloo():
    outs = _run("sample")
    for _, err in outs:
        assert err < 1e-13


def test_resynth_partitions_gloo():
    """NEXT-4: partitions spread over two ranks (p mod world), reports gathered
    in partition order, identical on both ranks and equal to one process."""
    from paper_2405_12866_b200 import resynth as R
    from test_resynth import OracleContext, PRM
    outs = _run("resynth")
    (r0, a), (r1, b) = outs
    assert a == b and [t[0] for t in a] == [0, 1, 2]
    blocks = [R.redundant_block(3, 2, seed=10 + q, extra=1) for q in range(3)]
    one = R.resynth_partitions(blocks, PRM, starts=2, context_factory=OracleContext)
    assert [(p_, r.deleted, r.kept) for p_, r in one] == a
