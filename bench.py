#!/usr/bin/env python
"""Benchmark of the TEM forward hot path (BASELINE.json metric).

A STEP = one pass of the whole hot path over one synthetic earth model:
edge mass (§2.2) -> batched multi-shift Jacobi-COCG to relative residual
1e-10 for every shifted system (K + s_i M) x_i = f (§3.2 eq:rmj) ->
channel synthesis u(t_j) = sum_i w_i Re(alpha_ij x_i) for all K channels
-> (default) refinement rounds until every channel is converged.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large]
    python bench.py --impl reference      # the CPU oracle arm

metric  : shift-unknown-iterations/s (sum over shifts of COCG iterations x
          free edge unknowns, per second), whole job over all ranks;
          ms_per_step is the wall time to all time channels.
roofline: the COCG passes against measured HBM bandwidth, at the algorithmic
          96 B per shift-unknown-iteration of a complex shift and 48 B of a
          real shift (split scheme; two-sweep 128 / 64 B).
accuracy: default --accuracy channels: the first solve to 1e-11, then one
          round of tem_forward's double-double iterative refinement
          (corrections to a 1e-4 residual reduction; R13), so the
          channel fields meet the north-star bar (relative L2 <= 1e-7 at
          every channel); the line reports the measured per-channel error
          against a much tighter refined solve of the same forward (untimed)
          and the plain 1e-10 solve's time for context.
e2e     : the same step through tem_forward_host with pinned HOST buffers
          (sigma, f uploaded; all channel fields downloaded) each step.
N > 1   : one process per GPU (torchrun).  Default --partition soundings:
          each rank an independent sounding (the transmitter moved by rank)
          -> weak scaling, no data-path collective.  --partition shifts: ONE
          sounding, its shifted systems dealt to the ranks
          (paper_2506_11657_b200.distributed), each rank synthesises its
          partial sum of every channel and one NCCL reduce sums them onto
          rank 0 inside the timed step -> strong scaling (DESIGN.md
          "Multi-GPU").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic HBM bytes per shift-unknown-iteration of each
# COCG scheme (complex fp64, 16 B per value):
#   two_sweep: sweep 1 reads z, p_old, writes p (48); sweep 2 reads p, x, z,
#              writes x, z (80)                                       -> 128
#   split:     pass 1 reads z, p_old, writes p, z (64) and, every second
#              iteration, reads and writes x (+32); pass 2 reads z (16) -> 96
ALG_BYTES_PER_SUI = {"two_sweep": 128, "split": 96}
KERNELS = {"two_sweep": "COCG sweeps k_sweep<1> + k_sweep<2>",
           "split": "split COCG passes k_sweep<3>/<4> (pass 1) + k_delta (pass 2)"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        pw = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": float(np.median(pw)) if pw else None,
                "samples": len(self.rows)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_job(times, work, device=None):
    """Whole-job aggregation across ranks: elapsed times -> MAX over ranks
    (the job ends when the slowest rank ends), work counts -> SUM.  No-op on a
    single process.  Tensors live on `device` (cuda for NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(times), list(work)
    dev = device or ("cuda" if dist.get_backend() == "nccl" else "cpu")
    t = torch.tensor([float(v) for v in times], dtype=torch.float64, device=dev)
    w = torch.tensor([float(v) for v in work], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()], [int(round(v)) for v in w.tolist()]


def _workload_for_rank(name: str, rank: int):
    from workloads import make_workload
    from workloads.configs import loop_source_edges
    wl = make_workload(name)
    if rank:
        # independent sounding per rank: transmitter moved by `rank` cells along x
        xs = sorted({e[1] for e in wl.source if e[0] == 0})
        ys = sorted({e[2] for e in wl.source if e[0] == 0})
        i0, i1 = xs[0] + rank, xs[-1] + 1 + rank
        if i1 >= wl.grid.shape[0]:
            i0, i1 = xs[0] - rank, xs[-1] + 1 - rank
        wl.source = loop_source_edges(i0, i1, ys[0], ys[-1], wl.surface_k)
    return wl


def _poles(args, wl):
    """Shifts/residues: the committed table (data/rational, the inputs the
    parity tests share with the oracle) or the library's own host fit
    (tem_fit_family) for the workload's channels and degree."""
    from paper_2506_11657_b200 import RationalTable
    if args.poles == "fit":
        return RationalTable.fit(wl.times, wl.n_poles)
    return RationalTable.load(args.config)


def _conducting_mask(fw, wl):
    """Free-or-not edges outside the air layer (reading R6): x, y edges on or
    below the surface node plane, z edges below it."""
    nx, ny, nz = wl.grid.shape
    k = np.arange(fw.Nn) // ((nx + 1) * (ny + 1))
    ks = wl.surface_k
    return ~np.concatenate([k > ks, k > ks, k >= ks])


def _alg_bytes(shifts, iters, N, solver, real_arith):
    """Algorithmic HBM bytes of the COCG loops: per shift-iteration of a
    complex shift ALG_BYTES_PER_SUI[solver], of a real shift (real
    arithmetic, split scheme) half of it (8-byte values)."""
    real = (np.asarray(shifts).imag == 0) & real_arith & (solver == "split")
    per = np.where(real, ALG_BYTES_PER_SUI[solver] / 2, ALG_BYTES_PER_SUI[solver])
    return float(np.sum(per * np.asarray(iters, dtype=np.float64)) * N)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2506_11657_b200 import TemForward

    ws, rank, local = _dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product has no CPU path)")
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2506_11657_b200.distributed import forward_partial, reduce_channels, shard_shifts
    by_shift = args.partition == "shifts"
    wl = _workload_for_rank(args.config, 0 if by_shift else rank)
    table = _poles(args, wl)
    idx = shard_shifts(table.shifts, ws)[rank] if by_shift else np.arange(table.n_shift)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz, device=dev)
    if args.solver:
        fw.solver = args.solver
    solver = fw.solver
    refine = args.accuracy == "channels"
    opts = fw.opts(tol=args.tol, maxit=args.maxit, refine=args.refine_rounds if refine else 0,
                   refine_tol=args.refine_tol,
                   channel_tol=args.channel_tol, safety=args.safety)
    real_arith = os.environ.get("TEM_NO_REAL", "0") in ("", "0")
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).to(dev)
    f = torch.from_numpy(fw.source_vector(wl.source)).to(dev)
    S, K = table.residues.shape
    N = fw.n_unknowns
    stream = torch.cuda.current_stream(dev)

    def step():
        u, iters, relres = forward_partial(fw, sigma, f, table, idx, opts=opts)
        if by_shift:
            reduce_channels(u, dst=0)            # the one exchange: sum of partial channels
        st = fw.forward_stats() if len(idx) else {"shift_iterations": 0, "loop_ms": 0.0, "kernel_launches": 0,
                                                  "refine_rounds": 0, "channel_bound": -1.0,
                                                  "initial_shift_iterations": 0, "relres_max": 0.0}
        return u, iters, relres, st

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        u, iters, relres, st = step()
        del u
    barrier()
    sui = 0
    loop_ms = 0.0
    launches = 0
    alg_bytes = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    u_last = None
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            u_last = None
            u, iters, relres, st = step()
            sui += int(st["shift_iterations"]) * N
            loop_ms += st["loop_ms"]
            alg_bytes += _alg_bytes(table.shifts[idx], iters, N, solver, real_arith) if len(idx) else 0.0
            launches += int(st["kernel_launches"]) + (1 if len(idx) else 0)   # + edge mass
            u_last = u
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if not refine:
        assert np.all(relres <= args.tol), relres

    # max over ranks for the time, sums for the work
    (t_max, loop_max), (sui_tot,) = reduce_job([ms, loop_ms], [sui], dev)

    # ---- field accuracy of the timed step (rank 0, one GPU): against a much
    # tighter refined solve of the same forward, outside the timed region
    accuracy = None
    if rank == 0 and ws == 1 and not args.no_accuracy_check:
        cond = torch.from_numpy(_conducting_mask(fw, wl)).to(dev)
        ref_opts = fw.opts(tol=args.tol, maxit=args.maxit, refine=4, refine_tol=1e-8, channel_tol=1e-13,
                           safety=10.0)
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        ur, xr, _, rr_ref = fw.forward(sigma, f, table, opts=ref_opts)
        e3.record(stream)
        torch.cuda.synchronize(dev)
        ref_st = fw.forward_stats()
        del xr
        urn = torch.linalg.vector_norm(ur[:, cond], dim=1)
        err = (torch.linalg.vector_norm((u_last - ur)[:, cond], dim=1) / urn).cpu().numpy()
        mass = fw.edge_mass(sigma)
        mw = mass.sqrt()
        errM = (torch.linalg.vector_norm((u_last - ur) * mw, dim=1) /
                torch.linalg.vector_norm(ur * mw, dim=1)).cpu().numpy()
        accuracy = {
            "max_channel_rel_l2_conducting": float(err.max()),
            "channel_of_max": int(err.argmax()),
            "channels_over_1e-7": int(np.sum(err > 1e-7)),
            "max_channel_rel_M_norm": float(errM.max()),
            "bar": "north star: relative L2 <= 1e-7 at every channel (conducting edges, DESIGN.md R6)",
            "meets_bar": bool(np.all(err <= 1e-7)),
            "library_bound": float(st["channel_bound"]),
            "refine_rounds": int(st["refine_rounds"]),
            "reference": ("same forward, tem_forward refined to channel_tol 1e-13 (refine_tol 1e-8, "
                          f"{int(ref_st['refine_rounds'])} rounds, double-double residual max "
                          f"{float(np.max(rr_ref)):.1e}), {e2.elapsed_time(e3) / 1e3:.1f} s"),
        }
        del ur, mass, mw
        torch.cuda.empty_cache()
    del u_last

    # ---- the unrefined solve at the north-star tolerance, for context (untimed by the contract)
    plain = None
    if rank == 0 and ws == 1 and refine and not args.no_accuracy_check:
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        u0, x0, it0, _ = fw.forward(sigma, f, table, tol=1e-10, maxit=args.maxit)
        e3.record(stream)
        torch.cuda.synchronize(dev)
        plain = {"tol": 1e-10, "ms": e2.elapsed_time(e3), "shift_iterations": int(np.sum(it0)),
                 "note": "fields of this solve miss the channel bar at late channels (DESIGN.md R13)"}
        del u0, x0

    # ---- e2e through the C ABI with pinned host buffers (rank-local, then max)
    e2e = None
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if not args.no_e2e and by_shift:
        # host sigma, f up; partial forward; reduce; u down on rank 0
        sig_h = torch.from_numpy(fw.sigma_layout(wl.sigma)).pin_memory()
        f_h = torch.from_numpy(fw.source_vector(wl.source)).pin_memory()
        u_h = torch.empty((K, fw.n_slots), dtype=torch.float64).pin_memory()
        barrier()
        t0 = time.perf_counter()
        e2e_sui = 0
        for _ in range(e2e_steps):
            sig_d = sig_h.to(dev, non_blocking=True)
            f_d = f_h.to(dev, non_blocking=True)
            u, it_h, _ = forward_partial(fw, sig_d, f_d, table, idx, opts=opts)
            reduce_channels(u, dst=0)
            if rank == 0:
                u_h.copy_(u)
            torch.cuda.synchronize(dev)
            e2e_sui += int(np.sum(it_h)) * N
        barrier()
        e2e_s = time.perf_counter() - t0
        (e2e_s,), (e2e_sui,) = reduce_job([e2e_s], [e2e_sui], dev)
        e2e = {"value": e2e_sui / e2e_s, "unit": "shift-unknown-iterations/s",
               "h2d_bytes_per_step": int(sig_h.numel() * 8 + f_h.numel() * 8),
               "d2h_bytes_per_step": int(u_h.numel() * 8),
               "ms_per_step": 1e3 * e2e_s / e2e_steps, "steps": e2e_steps}
        del u_h
    elif not args.no_e2e:
        sig_h = torch.from_numpy(fw.sigma_layout(wl.sigma)).pin_memory()
        f_h = torch.from_numpy(fw.source_vector(wl.source)).pin_memory()
        u_h = torch.empty((K, fw.n_slots), dtype=torch.float64).pin_memory()
        barrier()
        t0 = time.perf_counter()
        e2e_sui = 0
        for _ in range(e2e_steps):
            _, it_h, _ = fw.forward_host(sig_h.numpy(), f_h.numpy(), table, opts=opts, out=u_h.numpy())
            e2e_sui += int(np.sum(it_h)) * N
        barrier()
        e2e_s = time.perf_counter() - t0
        (e2e_s,), (e2e_sui,) = reduce_job([e2e_s], [e2e_sui], dev)
        e2e = {"value": e2e_sui / e2e_s, "unit": "shift-unknown-iterations/s",
               "h2d_bytes_per_step": int(sig_h.numel() * 8 + f_h.numel() * 8),
               "d2h_bytes_per_step": int(u_h.numel() * 8),
               "ms_per_step": 1e3 * e2e_s / e2e_steps, "steps": e2e_steps,
               "note": "first call allocates the library's cached device workspace (included)"}
        del u_h

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return None

    peak, peak_kind = _peaks()
    achieved = alg_bytes / (loop_ms * 1e-3) / 1e9
    # measured DRAM bytes of one COCG iteration (both passes, all shifts active)
    # from the committed ncu --set full capture, and the algorithmic bytes of it
    traffic, traffic_alg = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(solver, {})
            # the capture is of one workload and family; other runs report no traffic
            if tj.get("workload", "large") == args.config and tj.get("poles", "fit") == args.poles:
                traffic = tj.get("traffic_bytes_per_iteration")
                traffic_alg = tj.get("algorithmic_bytes_per_iteration")
        except Exception:
            traffic = None
    n_real = int(np.sum(table.shifts.imag == 0)) if (real_arith and solver == "split") else 0
    line = {
        "metric": "shift-unknown-iterations/s",
        "value": sui_tot / (t_max * 1e-3),
        "unit": "shift-unknown-iterations/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if by_shift else "weak",
        "vs_baseline": None,
        "dtype": "f64 (complex128 shifts; real shifts in real arithmetic)",
        "data": f"synthetic (seeded earth model, BASELINE {args.config} shape)",
        "config": {"workload": args.config, "unknowns": N, "shifts": S, "real_shifts": n_real, "channels": K,
                   "poles": args.poles, "uniform_error": table.uniform_error,
                   "degree": int(2 * table.is_pair.sum() + (~table.is_pair).sum()),
                   "accuracy": args.accuracy, "tol": args.tol,
                   "refine": ({"refine_tol": args.refine_tol, "channel_tol": args.channel_tol,
                               "max_rounds": args.refine_rounds,
                               "safety": args.safety, "rounds": int(st["refine_rounds"]),
                               "library_bound": float(st["channel_bound"]),
                               "relres_max_dd": float(st["relres_max"]),
                               "first_solve_shift_iterations": int(st["initial_shift_iterations"])}
                              if refine else None),
                   "field_accuracy": accuracy,
                   "plain_solve": plain,
                   "shift_iterations_per_step": int(st["shift_iterations"]),
                   "iterations_per_shift": [int(i) for i in iters],
                   "l2": "inputs larger than L2 (each shift block %.2f GB)" % (fw.n_slots * S * 16 / 1e9),
                   "wall_time_to_all_channels_ms": t_max / args.steps,
                   "cocg_loop_ms_per_step": loop_ms / args.steps,
                   "outside_cocg_ms_per_step": (ms - loop_ms) / args.steps,
                   "outside_cocg_note": ("edge mass, synthesis of all channels (twice with refinement), the "
                                         "double-double residuals, x update and channel norms of the refinement, "
                                         "host control"),
                   "parallelism": (f"{ws} ranks x shifts {[len(p) for p in shard_shifts(table.shifts, ws)]}"
                                   ", NCCL reduce of the channel fields" if by_shift and ws > 1 else
                                   f"{ws} independent soundings" if ws > 1 else "1 GPU")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per COCG iteration (all passes, all shifts active; "
                                     "split: mean of an even and an odd iteration)",
                     "algorithmic_bytes_per_iteration": traffic_alg,
                     "kernel": (f"{KERNELS[solver]}; algorithmic {ALG_BYTES_PER_SUI[solver]} B per SUI of a "
                                f"complex shift, {ALG_BYTES_PER_SUI[solver] // 2} B of a real shift"),
                     "achieved_from": "algorithmic bytes of all COCG solves / their CUDA-event loop time",
                     "solver": solver, "peak_kind": peak_kind},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.cpu_iters, args.poles)
    if ws > 1:
        dist.destroy_process_group()
    return line


def _oracle_table(config: str, poles: str):
    """The family the GPU arm solves, as DATA: `--poles fit` -> the product's
    fit committed by scripts/make_product_fit_tables.py
    (data/rational/<config>_fit.json, checked against a fresh fit by
    tests/test_product_fit.py); `--poles table` -> the oracle's table."""
    from paper_2506_11657_b200 import RationalTable  # table reading only
    return RationalTable.load(f"{config}_fit" if poles == "fit" else config)


def cpu_baseline(config: str, iters: int, poles: str = "fit"):
    """The oracle (oracle/cocg.py, as it stands) on the same workload and the
    same shifted systems: CSR assembly untimed, then `iters` COCG iterations
    of the hardest (smallest |s|) shift, timed.  Bounded sample, scaled to
    SUI/s."""
    from oracle import cocg, yee
    from workloads import make_workload
    wl = make_workload(config)
    table = _oracle_table(config, poles)
    asm = yee.assemble(wl)
    s = table.shifts[np.argmin(np.abs(table.shifts))]
    t0 = time.perf_counter()
    cocg.cocg(asm, complex(s), tol=1e-300, maxit=iters)
    dt = time.perf_counter() - t0
    return {"value": asm.n * iters / dt, "unit": "shift-unknown-iterations/s", "cores": 1,
            "kind": "oracle",
            "sample": f"{config}: {iters} COCG iterations of 1 of {table.n_shift} shifts "
                      f"(N={asm.n}), scipy CSR, single-threaded; assembly untimed"}


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return None
    from oracle import cocg, yee
    from workloads import make_workload
    wl = make_workload(args.config)
    table = _oracle_table(args.config, args.poles)
    asm = yee.assemble(wl)
    s = complex(table.shifts[np.argmin(np.abs(table.shifts))])
    for _ in range(args.warmup):
        cocg.cocg(asm, s, tol=1e-300, maxit=1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cocg.cocg(asm, s, tol=1e-300, maxit=args.cpu_iters)
    dt = time.perf_counter() - t0
    v = asm.n * args.cpu_iters * args.steps / dt
    sample = (f"{args.config}: each step = {args.cpu_iters} COCG iterations of 1 of "
              f"{table.n_shift} shifts (N={asm.n}), scipy CSR, single-threaded")
    return {"impl": "reference", "metric": "shift-unknown-iterations/s", "value": v,
            "unit": "shift-unknown-iterations/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": args.config, "unknowns": asm.n, "shifts": table.n_shift,
                       "real_shifts": int(np.sum(table.shifts.imag == 0)), "channels": int(table.residues.shape[1]),
                       "poles": args.poles, "degree": int(2 * table.is_pair.sum() + (~table.is_pair).sum())},
            "cpu_baseline": {"value": v, "unit": "shift-unknown-iterations/s", "cores": 1,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "shift-unknown-iterations/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--tol", type=float, default=None,
                    help="COCG tolerance of the first solve (default: 1e-11 with --accuracy channels, "
                         "the north-star 1e-10 with --accuracy residual)")
    ap.add_argument("--accuracy", default="channels", choices=["channels", "residual"],
                    help="channels: refine until the channel fields meet the bar (tem_forward, R13); "
                         "residual: one solve to --tol")
    ap.add_argument("--refine-tol", type=float, default=1e-4)
    ap.add_argument("--refine-rounds", type=int, default=1,
                    help="refinement rounds at most (tem_forward max_refine); the library's channel rule "
                         "may stop earlier.  One round (1e-4) after a 1e-11 first solve meets the bar with >= 1.45x "
                         "margin on every BASELINE config (DESIGN.md R13); the line reports the measured error")
    ap.add_argument("--channel-tol", type=float, default=1e-7)
    ap.add_argument("--safety", type=float, default=1.5)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-accuracy-check", action="store_true")
    ap.add_argument("--poles", default="fit", choices=["table", "fit"])
    ap.add_argument("--maxit", type=int, default=200000)
    ap.add_argument("--cpu-iters", type=int, default=8)
    ap.add_argument("--solver", default=None, choices=["split", "two_sweep"],
                    help="COCG scheme (default: the library's, tem_get_solver)")
    ap.add_argument("--partition", default="soundings", choices=["soundings", "shifts"],
                    help="N>1: independent soundings per rank (weak) or one sounding's shifts "
                         "over the ranks + NCCL reduce of the channels (strong)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.tol is None:
        args.tol = 1e-11 if args.accuracy == "channels" else 1e-10
    if args.warmup < 3:
        sys.stderr.write("bench.py: warning: fewer than 3 warm-up steps\n")
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
