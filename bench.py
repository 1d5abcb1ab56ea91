#!/usr/bin/env python
"""Benchmark: lag-block assembly throughput (triangle-pair x lag quadratures/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Workload: BASELINE.json gives no config for its metric, so the bench runs the
largest configuration that fits one GPU, configs[3] (config 4): icosphere
refined 4x (5120 triangles, 2562 P1 dofs), dt = 0.025, N = 160, p = 0,
reference quadrature rules (q_reg 4, q_sing 5, n_rad auto).  A "step" is one
complete assembly of every canonical block position (pair plan with exact
distance bounds, all-lags quadrature, singular reduction, CSR pattern and
compensated gather) from device-resident mesh/tables.  `value` = units / s,
units = admissible (triangle pair, block position) quadratures.  `e2e` is the
same metric through the public API (assemble_system from host arrays, all
blocks copied back to host as CSR).  --config 2 keeps the round-1 workload.

N > 1 (torchrun, one process per GPU; `--gpus N` without torchrun re-launches
itself under torch.distributed.run): SURVEY 8e row-block sharding - each rank
assembles its own test-vertex rows of every block with no communication (strong
scaling over the fixed config); times are the max over ranks; value counts each
global unit once (halo duplicates reported separately).

--impl reference times the REFERENCE package itself (tdbem from oracle/_ref/pkg
or baseline/_ref, never this repo's package): its assemble_subblocks at every
canonical position for a seeded sample of test rows per step, on all host cores
(oracle/reference_arm.py; rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembly triangle-pair x lag quadratures/s"
UNIT = "units/s"


def flops_per_launch(st, p):
    """ALGORITHMIC FP64 flops of the quadrature kernel:
    36 per geometry point + (1 + 160 (p+1)^2) per in-support (unit, point) evaluation."""
    return 36.0 * st["n_geom"] + (1.0 + 160.0 * (p + 1) ** 2) * st["n_in"]


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"tdb_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        import torch

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if os.environ.get("TDB_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, v: float, device) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_traffic(c: int, kernel: str = "k_quad"):
    """DRAM bytes per launch of the dominant quadrature kernel at config c from its committed
    ncu --set full capture, or None."""
    name = f"ncu_quad_cells_cfg{c}.json" if kernel == "k_quad_cells" else f"ncu_quad_cfg{c}.json"
    path = os.path.join(ROOT, "profiles", "r02", name)
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), path
    except (OSError, ValueError):
        return None, None


REF_ROWS = {1: 24, 2: 8, 3: 4, 4: 2, 5: 1}  # sampled test vertices per reference step


def run_reference(args, world, rank):
    """The reference package's own assembly on the host cores (oracle/reference_arm.py)."""
    if rank != 0:
        return 0
    from oracle import reference_arm as RA

    try:
        rs = RA.RowSampler(args.config, args.ref_rows or REF_ROWS[args.config])
    except (ImportError, RuntimeError) as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return 0
    units_full, npos = RA.full_units(args.config)
    got_u, got_s = [], []
    for step in range(args.warmup + args.steps):
        prep = rs.prepare(step)  # pre-warmed bounds of this step's rows (untimed)
        u, secs = rs.step(prep)
        if step >= args.warmup:
            got_u.append(u)
            got_s.append(secs)
    value = float(sum(got_u) / sum(got_s))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(got_s)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8d meshes)",
        "config": {"workload": rs.name, "units_per_step": units_full, "p": 0, "positions": npos},
        "sample_units_per_step": float(np.mean(got_u)),
        "parallelism": f"{rs.workers} host processes (reference per-position pool)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": rs.workers, "kind": "reference",
                         "sample": rs.describe(args.steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_line(c: int):
    """Bounded reference sample for the cpu_baseline key of our own line (rank 0, N = 1)."""
    from oracle import reference_arm as RA

    rs = RA.RowSampler(c, REF_ROWS[c])
    rs.step(rs.prepare(0))  # warm the pool / page cache
    u, secs = rs.step(rs.prepare(1))
    return {"value": u / secs, "unit": UNIT, "cores": rs.workers, "kind": "reference",
            "sample": rs.describe(1), "sample_units": u, "sample_seconds": secs}


def sum_over_ranks(world, v: float, device) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t.item())


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def time_matvec(A, grid, dev, stream, reps=20, rows=None, cols=None):
    """Block-Hessenberg matvec over a block range (incl. the all-gather when sharded): ms per call."""
    import torch

    clo, chi = cols if cols is not None else (1, grid.N)
    x = torch.randn((chi - clo + 1) * (grid.p + 1) * A.M, dtype=torch.float64, device=dev)
    for _ in range(3):
        A.matvec(x, rows=rows, cols=cols)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        A.matvec(x, rows=rows, cols=cols)
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def matvec_roofline(ms, plan, world, dev, hbm, fp64):
    """Algorithmic bytes / flops of one application (canonical CSR bytes, logical flops) vs the
    measured HBM and FP64 peaks; `bound` names the roof the kernel sits closer to."""
    b = sum_over_ranks(world, plan.bytes if hasattr(plan, "bytes") else 0.0, dev)
    f = sum_over_ranks(world, plan.flops if hasattr(plan, "flops") else 0.0, dev)
    gbs = b / (ms * 1e-3) / 1e9 / max(1, world)
    tfs = f / (ms * 1e-3) / 1e12 / max(1, world)
    t_hbm, t_fp = b / (hbm * 1e9) / max(1, world), f / (fp64 * 1e12) / max(1, world)
    return {"ms": ms, "algorithmic_bytes": b, "flops": f, "achieved_GBps": gbs, "frac_hbm_per_gpu": gbs / hbm,
            "achieved_TFLOPs": tfs, "frac_fp64_per_gpu": tfs / fp64,
            "bound": "hbm" if t_hbm >= t_fp else "fp64",
            "roof_ms": max(t_hbm, t_fp) * 1e3, "frac_of_roof": max(t_hbm, t_fp) * 1e3 / ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-rows", type=int, default=0, help="reference arm: sampled test vertices per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's own launch sets WORLD_SIZE)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    world, rank, local = dist_init()
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch

    from paper_1503_07221_b200 import _lib
    from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan
    from paper_1503_07221_b200.block_system import assemble_system, canonical_positions
    from paper_1503_07221_b200.configs import get_config
    from paper_1503_07221_b200.distributed import DistributedBlockHessenbergMatrix, assemble_system_distributed
    from paper_1503_07221_b200.kernel_weights import tables_for

    # one GPU per rank; TDB_BENCH_BACKEND=gloo (plumbing check on a host with fewer GPUs
    # than ranks - not a measurement) maps ranks onto the visible devices
    local_dev = local % max(1, torch.cuda.device_count()) if os.environ.get("TDB_BENCH_BACKEND") == "gloo" else local
    torch.cuda.set_device(local_dev)
    os.environ["TDB_DEVICE"] = str(local_dev)  # libtdb's default context follows the rank's GPU
    dev = torch.device("cuda", local_dev)
    lag_groups = int(os.environ.get("TDB_LAG_GROUPS", "1"))
    cfg = get_config(args.config)
    mesh, grid = cfg.mesh(), cfg.grid()
    tables = tables_for(grid)
    positions = canonical_positions(grid, mesh.diameter)
    plan = build_plan(mesh, grid, tables, positions)
    ctx = _lib.default_context(local_dev)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)

    # device-resident system: inputs uploaded + buffers sized once (untimed).
    # N > 1: SURVEY 8e row-block sharding - this rank assembles its own test-vertex
    # rows of every block (no communication), strong scaling over a fixed config.
    rows_per_rank = None
    A_mv = None
    if world > 1:
        # world = row blocks x lag groups (TDB_LAG_GROUPS, default 1)
        A_mv = assemble_system_distributed(mesh, grid, rank, world, ctx=ctx, tables=tables, lag_groups=lag_groups,
                                           create_only=True)
        rows_per_rank = A_mv.rows_per_rank
        sys_ = A_mv.dev
    else:
        sys_ = DeviceAssembly(mesh, plan, ctx)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # 256 MB > L2
    for _ in range(args.warmup):
        sys_.rerun()
    clocks = ClockSampler(local)
    step_ms, quad_ms, cells_ms_l = [], [], []
    stats = None
    barrier(world)
    torch.cuda.synchronize(dev)
    clocks.start()
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
        barrier(world)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sys_.rerun()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        stats = sys_.stats()
        quad_ms.append(stats["ms_quad"])
        cells_ms_l.append(stats.get("ms_quad_cells", 0.0))
    torch.cuda.synchronize(dev)
    barrier(world)
    clk = clocks.stop()
    ms = max_over_ranks(world, float(np.mean(step_ms)), dev)
    units = int(round(sum_over_ranks(world, float(stats["units_primary"]), dev)))
    units_computed = int(round(sum_over_ranks(world, float(stats["units"]), dev)))
    value = units / (ms * 1e-3)

    # roofline of the dominant kernel, FP64-bound: k_quad_cells (the regular pairs of the
    # grid families) when the system runs it, else k_quad; the quadrature phase as a whole
    # (k_quad_cells + k_quad for the singular cases) is reported next to it
    fl_all = flops_per_launch(stats, grid.p)
    q_ms = float(np.mean(quad_ms))
    peak_meas = _lib.fp64_peak_tflops(ctx, repeats=5)
    cells_ms = float(np.mean(cells_ms_l))
    if cells_ms > 0.0:
        kname = "k_quad_cells"
        k_ms = cells_ms
        rule_pts = len(plan.rules["regular"][2])
        fl = flops_per_launch({"n_geom": stats["pairs_cells"] * rule_pts, "n_in": stats["n_in_cells"]}, grid.p)
        n_in_k, n_geom_k = stats["n_in_cells"], stats["pairs_cells"] * rule_pts
    else:
        kname, k_ms, fl, n_in_k, n_geom_k = "k_quad", q_ms, fl_all, stats["n_in"], stats["n_geom"]
    achieved = fl / (k_ms * 1e-3) / 1e12
    traffic, traffic_src = load_traffic(args.config, kname)
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak_meas, "unit": "TFLOP/s",
                "frac": achieved / peak_meas,
                "peak_source": "measured in-run, best of a DFMA and a DMMA (FP64 tensor core) "
                               "microbenchmark (tdb_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
                "traffic_source": traffic_src,
                "peak_nominal": 37.2, "frac_of_nominal": achieved / 37.2,
                "traffic": traffic if world == 1 else None, "kernel": kname, "kernel_ms": k_ms,
                "kernel_share_of_step": k_ms / float(np.mean(step_ms)),
                "flops_per_launch": fl, "n_in": n_in_k, "n_geom": n_geom_k,
                "quadrature_phase": {"ms": q_ms, "kernels": "k_quad_cells + k_quad" if cells_ms > 0.0 else "k_quad",
                                     "flops": fl_all, "achieved": fl_all / (q_ms * 1e-3) / 1e12,
                                     "frac": fl_all / (q_ms * 1e-3) / 1e12 / peak_meas,
                                     "share_of_step": q_ms / float(np.mean(step_ms)),
                                     "n_in": stats["n_in"], "n_geom": stats["n_geom"]},
                "note": "rank 0's kernel" if world > 1 else "single GPU"}

    # block Hessenberg matvec (the solve's hot op): HBM roofline on algorithmic bytes
    if A_mv is None:
        from paper_1503_07221_b200.block_system import BlockHessenbergMatrix

        A_mv = BlockHessenbergMatrix(grid=grid, M=mesh.num_vertices, diameter=mesh.diameter, _dev=sys_)
    hbm, hbm_src = hbm_peak()
    mv_ms = max_over_ranks(world, time_matvec(A_mv, grid, dev, stream), dev)
    mvp = A_mv._plan((1, grid.N), (1, grid.N)) if world > 1 else A_mv.matvec_plan()
    matvec = matvec_roofline(mv_ms, mvp, world, dev, hbm, peak_meas)
    # the range the recursive preconditioner applies most (92 of ~100 matvecs per outer step
    # at 2(2,10)): a diagonal quarter block
    q = (((grid.N + 1) // 2) + 1) // 2
    q_ms = max_over_ranks(world, time_matvec(A_mv, grid, dev, stream, rows=(1, q), cols=(1, q)), dev)
    qp = A_mv._plan((1, q), (1, q)) if world > 1 else A_mv.matvec_plan((1, q), (1, q))
    matvec["quarter_diagonal"] = dict(matvec_roofline(q_ms, qp, world, dev, hbm, peak_meas), rows=[1, q])
    matvec.update({
        "hbm_peak_GBps": hbm, "peak_source": hbm_src, "fp64_peak_TFLOPs": peak_meas,
        "kernels": "regular lag terms of the inner family: FP64 DMMA lag-band tiles staged by bulk copies "
                   "(k_band_mv + k_band_reduce); boundary terms and the light-cone tie lag: CSR (k_matvec)",
        "includes": ("ncclAllGather of the iterate" if world > 1 else "transposes + CSR SpMM + DMMA tiles"
                     " + ordered reduce")})

    # end to end through the public API (host mesh in, every block back on the host)
    e2e = None
    if not args.no_e2e:
        e2e_ms = []
        h2d = d2h = 0
        for i in range(max(1, min(args.steps, 3)) + 1):
            barrier(world)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            if world > 1:
                B = DistributedBlockHessenbergMatrix(mesh, grid, rows_per_rank, rank, ctx=ctx, tables=tables,
                                                     lag_groups=lag_groups, row_group=A_mv.row_group,
                                                     lag_group=A_mv.lag_group)
                host = [B.dev.family_arrays(f) for f in range(B.dev.num_families)]
            else:
                B = assemble_system(mesh, grid, tables=tables, device=local)
                host = [B._dev.family_arrays(f) for f in range(B._dev.num_families)]
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            if i > 0:  # first call warms the allocator / plan caches
                e2e_ms.append((t1 - t0) * 1e3)
            d2h = sum(a.nbytes + b.nbytes + c.nbytes for a, b, c in host)
            h2d = (mesh.corners.nbytes + mesh.normals.nbytes + mesh.curls.nbytes + mesh.areas.nbytes
                   + mesh.triangles.nbytes + 2 * mesh.triangles.nbytes
                   + sum(f.pack.coeffs.nbytes for f in plan.families)
                   + sum(sum(a.nbytes for a in plan.rules[c]) for c in plan.rules))
            del B, host
        ems = max_over_ranks(world, float(np.mean(e2e_ms)), dev)
        e2e = {"value": units / (ems * 1e-3), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(sum_over_ranks(world, d2h, dev)),
               "path": ("distributed.DistributedBlockHessenbergMatrix" if world > 1 else
                        "block_system.assemble_system") + " (C ABI tdb_system_assemble) + "
                       "tdb_system_copy_family for every family"}

    # FGMRES(50, 2(2,10)) solve, eps = 1e-5, Gaussian-pulse RHS
    solve = None
    if not args.no_solve:
        from paper_1503_07221_b200 import solvers as S
        from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann

        b = assemble_rhs(mesh, grid, gaussian_pulse_neumann(mesh))
        if world > 1:
            S.set_comm(S.TorchDistComm(group=A_mv.row_group))
            bl = torch.as_tensor(A_mv.local_of(b)).to(dev)
        else:
            bl = torch.as_tensor(b).to(dev)
        cfgS = S.SolverConfig(method="fgmres-recursive", restart=50, tol=1e-5, max_iter=2000,
                              recursion_depth=2, inner_iterations=(2, 10))
        # preconditioner setup (untimed in `seconds`, reported as `setup_seconds`): matvec
        # plans of every sub-range + CUDA-graph capture of one preconditioner application
        barrier(world)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        prec = S.recursive_preconditioner(A_mv, cfgS)
        for _ in range(3):
            prec(bl)
        torch.cuda.synchronize(dev)
        t_setup = max_over_ranks(world, time.perf_counter() - t0, dev)
        barrier(world)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        x, hist = S.fgmres(lambda v: A_mv.matvec(v), bl, cfgS, precond=prec)
        torch.cuda.synchronize(dev)
        ts = max_over_ranks(world, time.perf_counter() - t0, dev)
        S.set_comm(None)
        solve = {"method": "FGMRES(50, 2(2,10)) recursive block preconditioner", "tol": 1e-5,
                 "seconds": ts, "setup_seconds": t_setup, "iterations": len(hist),
                 "ms_per_outer_step": 1e3 * ts / max(1, len(hist)),
                 "final_rel_residual": float(hist[-1]),
                 "rhs": "Gaussian-pulse plane wave (sigma 0.2, t0 1.0), assemble_rhs (device, csrc/tdb_rhs.cu)",
                 "note": "x0 = 0, device vectors; setup = sub-range matvec plans + graph capture of the "
                         "preconditioner (reusable across right-hand sides)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(args.config)
        except (ImportError, RuntimeError) as e:
            cpu = {"value": None, "unavailable": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8d meshes)",
            "config": {"workload": cfg.name, "units_per_step": units, "p": grid.p,
                       "positions": len(plan.where)},
            "nnz": stats["nnz_total"],
            "parallelism": (f"{world // lag_groups} row blocks x {lag_groups} lag groups (NCCL all-gather per "
                            f"matvec{', partial-row all-reduce' if lag_groups > 1 else ''})" if world > 1 else "1 GPU"),
            "units_computed_incl_halo": units_computed,
            "l2": "flushed between timed steps (256 MB write)",
            "roofline": roofline,
            "matvec": matvec,
            "solve": solve,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(stats["launches"]) * args.steps,
            "clocks": clk,
            "phases_ms": {k: stats[k] for k in ("ms_plan", "ms_quad", "ms_finalize", "ms_pattern", "ms_total")},
            "units_case": stats["units_case"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
