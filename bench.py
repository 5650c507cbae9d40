#!/usr/bin/env python
"""QFactor-Sample instantiation benchmark on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--shard multistart|sample]
                    [--impl reference]

--gpus N (N > 1) outside torchrun re-executes this script under
torch.distributed.run with N processes, one per GPU (NCCL_DEBUG=INFO on
stderr); under torchrun WORLD_SIZE must equal N.

Workload: BASELINE.json config C4 — n = 12 qubits, K = 150
two-qubit blocks (brick wall + seeded random non-adjacent pairs), M = 32
training states, 16 validation states, S = 16 multistarts per GPU, complex128,
seeded synthetic Haar data (the paper's Table-1 partitions are not available).
A "step" is one pass of the whole hot path: one sweep of every start (B-cache
forward, K fused backward/environment/polar launches, sweep-end cost), the
validation forward, and the host controller's decision — i.e. one iteration
of qfs_instantiate with its stopping rules unable to fire.

value  = start-sweeps per second, whole job (sum over ranks / max-over-ranks
         device time).  Multi-GPU, --shard multistart (default): S starts per
         rank (weak scaling, no data-path collective).  --shard sample
         (default config C5, BASELINE.json configs[4]): ONE job's S starts, the
         pool and validation rows m = rank (mod N) on each rank, per-gate NCCL
         all-reduce of the 4x4 environments inside libqfs (qfs_create_nccl
         mode 1; strong scaling).
e2e    = the same metric through the public API from host buffers: every step
         the step's samples are copied from pinned host memory
         (qfs_set_samples_async, queued one step ahead so the copy overlaps the
         previous step) and qfs_instantiate(max_iter=1) runs with host init
         gates in and host gates/results out.
roofline = the dominant kernel (by device time in the timed region): algorithmic
         bytes / CUDA-event duration vs measured HBM copy bandwidth.
cpu_baseline = the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QFactor-Sample sweeps/sec + time-to-solution per instantiation; % HBM/FP64 peak"
UNIT = "start-sweeps/s"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2 (unit count x clock; context)
FP64_DFMA_MEASURED_TFLOPS = 34.195  # profiles/r1_peaks_microbench.json (tools/peaks.cu DFMA loop, all SMs)
L2_RMW_64MIB_GBS = 9209.1  # profiles/r1_peaks_microbench.json (l2loop_64MiB_rmw_gbs)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        """The timed region, host wall clock."""
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sel = self.lines
        if self.window and self.lines:
            t0, t1 = self.window
            sel = [x for x in self.lines if t0 - 0.05 <= x[0] <= t1 + 0.05]
            if not sel:  # region shorter than the sampling period: nearest samples
                sel = sorted(self.lines, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))[:2]
        for _, ln in sel:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def bench_params(max_iter, m_init):
    # stopping rules that cannot fire: every call runs exactly max_iter sweeps
    # (validation still computed every sweep: finite overtrain ratio, M < 2^n)
    return dict(dist_tol=-1.0, diff_tol_r=1e-3, plateau_window=0, min_iter=6, max_iter=int(max_iter),
                m_init=int(m_init), overtrain_ratio=1e300, beta=0.0, stop_on_first=0)


def cpu_oracle_run(prob, m, starts, threads, steps=1):
    """The oracle as it stands: `steps` controller steps (sweep + validation) of
    `starts` starts at fixed M.  Returns (start-sweeps/s, seconds)."""
    import oracle
    oracle.build()
    init = prob.init[:starts]
    prm = bench_params(1, m)
    t0 = time.perf_counter()
    g = init
    for _ in range(steps):
        g, _, _ = oracle.instantiate(prob.n, prob.pairs, prob.x, prob.y, prob.xv, prob.yv, g, prm,
                                     threads=threads)
    dt = time.perf_counter() - t0
    return starts * steps / dt, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def torchrun_cmd(nproc: int, port: int, argv: list) -> list:
    """The launch the driver uses (one process per GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def maybe_relaunch(gpus: int, argv: list):
    """--gpus N > 1 without a torchrun environment: re-exec under torchrun with N
    ranks and return its exit code (None: run in this process)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus and gpus > 1:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={ws}")
        return None
    if gpus <= 1:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")              # NCCL init lines (transport, NVLS) ...
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout keeps the one JSON line
    return subprocess.call(torchrun_cmd(gpus, free_port(), argv), env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, help="c1..c5, c5b, c5c (default c4; c5 with --shard sample)")
    ap.add_argument("--shard", default="multistart", choices=["multistart", "sample"])
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "device"],
                    help="sample mode: per-gate E all-reduce by host-enqueued NCCL or device-initiated (NEXT-2)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="sample mode on ONE GPU with G emulated ranks (device exchange; one start)")
    ap.add_argument("--starts", type=int, default=None,
                    help="multistarts per GPU (default: config S); with --shard sample: starts of the job")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tts", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rc = maybe_relaunch(args.gpus, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    sample = args.shard == "sample" or args.emulate_ranks > 1
    emul = args.emulate_ranks if args.emulate_ranks > 1 else 0
    if emul:
        args.exchange = "device"
    if args.config is None:
        args.config = "c5" if sample else "c4"

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2405_12866_b200 import inputs as I
    cfgd = I.CONFIGS[args.config]
    s_per = args.starts or cfgd["s"]
    # sample mode: one job of s_per starts whose rows are split over the ranks
    s_tot = s_per if sample else s_per * world
    ranks = emul or world                    # sample-mode ranks (emulated: on this one GPU)
    m_loc = cfgd["m_init"] // ranks if sample else cfgd["m_init"]
    if sample and (cfgd["m_init"] % ranks or cfgd["v"] % ranks):
        raise SystemExit(f"--shard sample: M={cfgd['m_init']} and V={cfgd['v']} must be divisible by {ranks}")
    if emul and (world > 1 or s_per != 1):
        raise SystemExit("--emulate-ranks: one process and one start")
    config = {"workload": f"{args.config.upper()}: n={cfgd['n']} K={cfgd['k']} M={cfgd['m_init']} "
                          f"V={cfgd['v']} S={s_per}{'' if sample else '/GPU'} complex128 "
                          f"(BASELINE.json configs[{min(cfgd['cfg'], 5) - 1}])",
              "n": cfgd["n"], "k": cfgd["k"], "m": cfgd["m_init"], "v": cfgd["v"],
              "starts_per_gpu": s_per if not sample else s_per, "starts_total": s_tot,
              "parallelism": ((f"sample: {emul} emulated ranks on 1 GPU (M/rank={m_loc}, device-initiated "
                               f"exchange of E per gate)") if emul else
                              (f"sample x{world} (M/rank={m_loc}, "
                               f"{'device-initiated exchange' if args.exchange == 'device' else 'NCCL all-reduce'}"
                               f" of E per gate)") if sample else f"multistart x{world}"),
              "l2": "inputs larger than L2 (B cache %.1f GB/GPU > 126 MB)" % (
                  (cfgd["k"] - 1) * s_per * m_loc * (16 << cfgd["n"]) / 1e9)}

    if args.impl == "reference":
        # the reference arm is the CPU oracle (no reference code exists for this paper)
        if rank != 0:
            return
        cores = host_cores()
        prob = I.make_problem(args.config, init="R", s=max(cores, 1))
        starts = min(cores, s_per)
        warm = max(1, args.warmup)
        cpu_oracle_run(prob, cfgd["m_init"], starts, cores, steps=warm)  # untimed warm-up steps
        v, dt = cpu_oracle_run(prob, cfgd["m_init"], starts, cores, steps=args.steps)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                "device": "cpu (host cores; the oracle uses no GPU)",
                "steps": args.steps, "warmup": warm, "ms_per_step": dt / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                 "sample": f"{starts} starts x {args.steps} controller steps of {args.config.upper()}"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2405_12866_b200 import build, qfs
    build.build()
    # one process per GPU; QFS_BENCH_PG=gloo is a functional check of the
    # multi-rank path on a box with fewer GPUs (ranks share devices; its
    # numbers are not measurements)
    pg = os.environ.get("QFS_BENCH_PG", "nccl")
    if pg != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if pg == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(pg)

    # seeded synthetic problem; multistart: starts of rank r are [r*S, (r+1)*S)
    # of the seeded stream; sample: every rank runs all S starts on its rows
    prob = I.make_problem(args.config, init="R", s=s_tot)
    init = np.ascontiguousarray(prob.init if sample else prob.init[rank * s_per:(rank + 1) * s_per])
    m = cfgd["m_init"]                      # global M (qfs_instantiate's m_init is global in sample mode)
    from paper_2405_12866_b200 import parallel as PL
    rows = PL.sample_rows(prob.x.shape[0], rank, world) if sample and not emul else slice(None)
    vrows = PL.sample_rows(prob.xv.shape[0], rank, world) if sample and not emul else slice(None)
    lx, ly = np.ascontiguousarray(prob.x[rows]), np.ascontiguousarray(prob.y[rows])
    lxv, lyv = np.ascontiguousarray(prob.xv[vrows]), np.ascontiguousarray(prob.yv[vrows])
    if emul:
        ctx = qfs.Context(prob.n, prob.pairs, device=local, emulated_ranks=emul)
    elif sample:
        # the library owns the NCCL communicator: rank 0's unique id, broadcast over torch.distributed
        obj = [qfs.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        ctx = qfs.Context(prob.n, prob.pairs, device=local, nccl_id=obj[0], rank=rank, world=world, shard_mode=1)
        if args.exchange == "device":
            ctx.set_exchange(1)
    else:
        ctx = qfs.Context(prob.n, prob.pairs, device=local)
    ctx.set_samples(lx, ly, lxv, lyv)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if pg == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- clocks are sampled from before the warm-up (nvidia-smi needs time to start)
    clk = ClockSampler(local).__enter__()
    # ---- warm-up (also captures the CUDA graph of the sweep)
    gates, _, _ = ctx.instantiate(init, bench_params(args.warmup, m))

    # ---- timed region: K steps, device time from CUDA events on the library stream
    l0 = ctx.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th0 = time.time()
    ev0.record(stream)
    gates, res, _ = ctx.instantiate(gates, bench_params(args.steps, m))
    ev1.record(stream)
    ev1.synchronize()
    clk.mark(th0, time.time())
    barrier()
    launches = ctx.launch_count() - l0
    dt = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    value = s_tot * args.steps / dt
    assert all(r["sweeps"] == args.steps for r in res), res
    clock_window = "timed region"
    if time.time() - th0 < 0.5:
        # shorter than a few nvidia-smi periods (C2, C5b): the clocks are sampled
        # over >= 0.5 s of the SAME step repeated right after the timed region
        # (VERDICT r1 hygiene), and the line says so
        tw0 = time.time()
        reps = 0
        while time.time() - tw0 < 0.5:
            ctx.instantiate(gates, bench_params(args.steps, m))
            reps += 1
        clk.mark(tw0, time.time())
        clock_window = f"{reps} repeats of the timed {args.steps} steps right after it ({time.time() - tw0:.2f} s)"

    # ---- per-kernel CUDA-event durations: the same K steps again with one event
    # pair around each phase of the sweep (the run of forward launches, the run
    # of backward launches, ...), recorded as event nodes inside the sweep graph
    # on the library stream; avg launch duration = phase time / launches.
    ctx.profile_enable(True)
    ctx.instantiate(gates, bench_params(2, m))     # capture the instrumented graph
    ctx.profile_enable(True)                       # reset counters, keep the graph
    barrier()
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    gates, _, _ = ctx.instantiate(gates, bench_params(args.steps, m))
    pe1.record(stream)
    pe1.synchronize()
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    clk.__exit__(None, None, None)
    prof_step_ms = pe0.elapsed_time(pe1) / args.steps

    # ---- roofline of the dominant kernel (by device time)
    peak, peak_src = load_peaks()
    dom = max((k for k in prof if prof[k]["launches"] > 0), key=lambda k: prof[k]["ms"])
    pd = prof[dom]
    tot_ms = sum(v["ms"] for v in prof.values())
    achieved = pd["bytes"] / (pd["ms"] * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            traffic = tj.get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    if dom == "resident":
        # cluster-resident sweep: no HBM traffic inside the sweep; bound by the
        # FP64 pipe: SURVEY.md §8(d)'s algorithmic 96 flops per
        # amp-gate (the uncompute's extra 32 and the fused validation are NOT
        # counted; the kernel time includes them) / time, against the measured
        # DFMA peak (tools/peaks.cu; 37.2 = 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz)
        achieved = pd["flops"] / (pd["ms"] * 1e-3) / 1e12
        peak, peak_src = FP64_DFMA_MEASURED_TFLOPS, "measured DFMA loop (profiles/r1_peaks_microbench.json; derived 37.2)"
        bound, unit = "alu", "TFLOP/s"
    else:
        bound, unit = "hbm", "GB/s"
    roofline = {"bound": bound, "kernel": dom, "achieved": round(achieved, 3), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "avg_launch_us": round(pd["ms"] / pd["launches"] * 1e3, 3),
                "bytes_per_launch": pd["bytes"] / pd["launches"], "flops_per_launch": pd["flops"] / pd["launches"],
                "pipe": "fp64" if bound == "alu" else None,
                # the streamed backward's working set (chi + B_i, ~67 MB at C4) is
                # L2-resident in part: its algorithmic bytes against the measured
                # L2 read+write bandwidth at a 64 MiB working set (tools/peaks.cu)
                "l2_rmw_peak_gbs": L2_RMW_64MIB_GBS if bound == "hbm" else None,
                "frac_of_l2_rmw": round(achieved / L2_RMW_64MIB_GBS, 4) if bound == "hbm" else None,
                "note": ("algorithmic bytes per launch exceed the kernel's DRAM bytes (traffic): part of "
                         "its working set (chi) is L2-resident, so frac against HBM can reach 1; "
                         "frac_of_l2_rmw is the L2-side figure (DESIGN.md section 5)")
                if bound == "hbm" and traffic and traffic < pd["bytes"] / pd["launches"] else None,
                "share_of_kernel_time": round(pd["ms"] / tot_ms, 4),
                "profiled_ms_per_step": round(prof_step_ms, 4),
                "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                "gbs": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] > 0 else 0,
                                "tflops": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 3) if v["ms"] > 0 else 0}
                            for k, v in prof.items() if v["launches"] > 0}}

    # ---- e2e: through the public API from pinned host buffers, copies in the timed region
    N = 1 << prob.n
    hx = torch.from_numpy(lx).pin_memory()
    hy = torch.from_numpy(ly).pin_memory()
    hxv = torch.from_numpy(lxv).pin_memory()
    hyv = torch.from_numpy(lyv).pin_memory()
    h2d = (hx.numel() + hy.numel() + hxv.numel() + hyv.numel()) * 16 + init.nbytes
    d2h = init.nbytes + s_per * 32
    g = gates
    e2e_steps = max(3, args.steps)

    def queue_samples():  # qfs_set_samples_async: H2D on the copy stream, consumed by the next call
        ctx.set_samples_async_host_ptr(hx.shape[0], hx.data_ptr(), hy.data_ptr(), hxv.shape[0], hxv.data_ptr(),
                                       hyv.data_ptr())

    # two caller-owned host gate buffers, alternating as input and output (the
    # C ABI's out_gates): no fresh allocation per step
    # pinned (page-locked) like the sample buffers: libqfs reads / writes them in place
    gbuf = [torch.from_numpy(np.ascontiguousarray(g)).pin_memory().numpy(),
            torch.empty(tuple(np.shape(g)), dtype=torch.complex128, pin_memory=True).numpy()]
    for w in range(2):                   # untimed warm-up of the e2e path (staging buffers, graphs)
        queue_samples()
        ctx.instantiate(gbuf[w % 2], bench_params(1, m), out=gbuf[(w + 1) % 2])
    barrier()
    t0 = time.perf_counter()
    queue_samples()                      # step 0's inputs
    for step in range(e2e_steps):
        if step + 1 < e2e_steps:
            queue_samples()              # step t+1's inputs copy while step t runs
        ctx.instantiate(gbuf[step % 2], bench_params(1, m), out=gbuf[(step + 1) % 2])
    barrier()
    e2e_dt = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": s_tot * e2e_steps / e2e_dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
           "note": "bytes per rank" if world > 1 else "single GPU"}

    # ---- time to solution (rank 0): warm-start instance of the same config, real stopping rules
    tts = None
    if (rank == 0 or sample) and not args.no_tts:   # sample mode: a collective call on every rank
        pw = I.make_problem(args.config, init="W", s=s_per)
        prm = dict(pw.params, max_iter=300)
        ctx.set_samples(pw.x[rows], pw.y[rows], pw.xv[vrows], pw.yv[vrows])
        # one warm-up call (allocations and graph shapes of the
        # restarts), then the median of 3 timed calls
        ctx.instantiate(pw.init, prm)
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            gw, rw, ww = ctx.instantiate(pw.init, prm)
            times.append(max_over_ranks(time.perf_counter() - t0) if sample else time.perf_counter() - t0)
        tsec = statistics.median(times)
        tts = {"seconds": round(tsec, 4), "seconds_runs": [round(t, 4) for t in times],
               "sweeps": rw[ww]["sweeps"], "term": rw[ww]["term"],
               "c_train": rw[ww]["c_train"], "final_m": rw[ww]["final_m"], "init": "W (eps=0.3)",
               "success_fraction": sum(r["term"] == "CONVERGED" for r in rw) / len(rw)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cores = host_cores()
        starts = min(cores, s_per)
        v, cdt = cpu_oracle_run(prob, m, starts, cores, steps=1)
        csteps = 1
        if cdt < 0.5:  # short configs: enough steps for about a second of wall time (bounded)
            csteps = int(min(50, max(2, 1.0 / max(cdt, 1e-3))))
            v, cdt = cpu_oracle_run(prob, m, starts, cores, steps=csteps)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{starts} starts x {csteps} controller step(s) (sweep + validation) of "
                         f"{args.config.upper()}, {cdt:.1f} s wall"}
        if cdt / max(1, starts) * cores < 5.0:  # 1-thread figure when it stays short
            v1, dt1 = cpu_oracle_run(prob, m, 1, 1, steps=1)
            cpu["single_thread"] = {"value": v1, "unit": UNIT, "sample": f"1 start x 1 controller step, {dt1:.1f} s"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong" if sample else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
                "cpu_baseline": cpu, "clocks": dict(clk.summary(), window=clock_window), "time_to_solution": tts,
                "amp_gate_updates_per_s": value * m * N * prob.k}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
