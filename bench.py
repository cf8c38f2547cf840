#!/usr/bin/env python
"""Benchmark of the LBM stream-collide hot path (BASELINE.json metric: MLUPS
per GPU and whole box, % of the HBM roofline).

    python bench.py [--gpus N --steps K --warmup W] [--config c4|c3|c1|c0|c2]
                    [--dtype f64|f32] [--impl b200|reference]

N > 1: one rank per GPU over NCCL.  Under torchrun (WORLD_SIZE set) the
ranks are the launcher's; `python bench.py --gpus N` without it re-executes
itself under `torch.distributed.run` with N processes (127.0.0.1
rendezvous) and checks that the rank count equals N.  Default workload:
BASELINE config 4 (the weak-scaling config and the north-star case): D3Q19
TRT (magic, omega_e = 1.8) + Guo 1e-6, fp64, 512^3 cells per GPU stacked in
z, periodic x/y channel with NoSlip walls at the global z-min/z-max planes
and a seeded 20 % random-sphere NoSlip obstacle tile per GPU (seed 100+k).

A "step" is one stream_collide over the whole domain.  `value` is whole-box
MLUPS with the state resident in HBM, timed with CUDA events between a
barrier + synchronize on both sides, max over ranks.  `e2e` is the same
metric through the public API with host buffers: one `run_arrays` call per
job (H2D of the initial rho/u, K sweeps, D2H of the final rho/u, all inside
the timed region; on one rank with walls in z the copies overlap the sweeps
as a wavefront over z-plane chunks).
`--impl reference` times the reference algorithm on the host cores: the C
restatement in oracle/ (the reference itself is numpy-only and cannot run
on the GPU box) on a bounded slab of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_CELL = {(19, 8): 304, (19, 4): 152, (27, 4): 216, (27, 8): 432}

CONFIGS = {
    "c4": dict(stencil="D3Q19", cells=(512, 512, 512), per_gpu=True, model=("TRT_magic", 1.8),
               force=1e-6, geometry="tiles", periodic=(True, True, False), init="rest",
               desc="BASELINE config 4: D3Q19 TRT magic(1.8) + Guo 1e-6, 512^3 per GPU, 20% "
                    "sphere tile per GPU (seed 100+k), NoSlip walls at global z-min/max, "
                    "periodic x,y"),
    "c3": dict(stencil="D3Q19", cells=(512, 512, 512), per_gpu=False, model=("TRT_magic", 1.8),
               force=None, geometry=None, periodic=(True, True, True), init="random",
               desc="BASELINE config 3: D3Q19 TRT magic(1.8), fixed 512^3 periodic (strong), "
                    "seeded random rho/u"),
    "c1": dict(stencil="D3Q19", cells=(128, 128, 128), per_gpu=True, model=("TRT_magic", 1.7),
               force=1e-6, geometry="spheres25", periodic=(True, True, False), init="rest",
               desc="BASELINE config 1: D3Q19 TRT magic(1.7) + Guo 1e-6, 128^3, 25% spheres "
                    "r 4-8, NoSlip z walls"),
    "c0": dict(stencil="D3Q19", cells=(64, 64, 64), per_gpu=True, model=("SRT", 1.8),
               force=None, geometry=None, periodic=(True, True, True), init="random",
               desc="BASELINE config 0: D3Q19 SRT 1.8, 64^3 periodic (L2-resident)"),
    "c2": dict(stencil="D3Q27", cells=(256, 256, 256), per_gpu=True, model=("MRT_raw", 1.9, 1.0),
               force=None, geometry="cavity", periodic=(False, False, False), init="rest",
               ubb=(0.05, 0.0, 0.0), dtype="f32",
               desc="BASELINE config 2: D3Q27 raw-moment MRT (shear 1.9, others 1.0), "
                    "256^3 lid-driven cavity, UBB lid (0.05,0,0)"),
}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default=None, choices=["f64", "f32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no extras)")
    return ap.parse_args(argv)


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_command(gpus, argv, port):
    """torch.distributed.run command that runs this script on `gpus` ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
            str(Path(__file__).resolve()), *argv]


def self_launch(args, argv) -> int | None:
    """`--gpus N` (N > 1) outside a launcher: re-run under torchrun with one
    process per GPU and return its exit code (None: run in this process).
    N larger than the visible device count is refused, unless
    LBM_B200_BACKEND=gloo asks for ranks that share GPUs (a single-GPU
    smoke of the multi-rank path)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "b200" and os.environ.get("LBM_B200_BACKEND") != "gloo":
        import torch
        ndev = torch.cuda.device_count()
        if ndev < args.gpus:
            raise SystemExit(f"--gpus {args.gpus}: only {ndev} CUDA device(s) visible")
    cmd = launch_command(args.gpus, argv, free_port())
    print("bench: launching " + " ".join(cmd[1:6]) + " ...", file=sys.stderr, flush=True)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.setdefault("NCCL_DEBUG", "INFO")
    return subprocess.call(cmd, env=env)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in Path(self.path).read_text().strip().splitlines()]
        except OSError:
            rows = []
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- workload
def build(cfg, ctx, dtype, P):
    import torch
    nx, ny, nzc = cfg["cells"]
    n = ctx.n_ranks
    if cfg["per_gpu"]:
        nz_rank, roots = nzc, n
    else:
        if nzc % n:
            raise SystemExit(f"{nzc} z-planes do not split over {n} ranks")
        nz_rank, roots = nzc // n, n
    st = getattr(P, cfg["stencil"])
    forest = P.create_forest(ctx, (0, 0, 0, 1, 1, roots), (1, 1, roots), periodic=cfg["periodic"],
                             cells_per_block=(nx, ny, nz_rank))
    pdf = P.PdfField(forest, st, layout="fzyx", dtype="float64" if dtype == "f64" else "float32")
    handling = None
    geo = cfg["geometry"]
    if geo is not None:
        from paper_1909_13772_b200 import workloads
        h = P.ensure_flags(forest)
        reg = h.registry
        blk = forest.local_blocks()[0]
        lo, hi = forest.cell_box(blk.id)
        ff = blk.data["flags"]
        if geo == "tiles":
            solid = workloads.sphere_mask((nx, ny, nz_rank), 100 + ctx.rank, 4.0, 8.0, 0.20,
                                          (True, True, False))
            if lo[2] == 0:
                solid[0] = True
            if hi[2] == forest.global_cells(0)[2]:
                solid[-1] = True
            code = solid.astype(np.int8)
        elif geo == "spheres25":
            code = workloads.porous_channel_flags((nx, ny, nz_rank), 1, 0.25).astype(np.int8)
        elif geo == "cavity":
            code = workloads.cavity_flags((nx, ny, nz_rank))
        inner = np.full(code.shape, reg["Fluid"], dtype=np.uint32)
        inner[code == 1] = reg["NoSlip"]
        inner[code == 2] = reg["UBB"]
        ff.interior[...] = inner
        handling = P.BoundaryHandling(forest, st, ubb_velocity=cfg.get("ubb", (0.0, 0.0, 0.0)))
        handling.freeze()
    m = cfg["model"]
    if m[0] == "SRT":
        model = P.SRT(m[1])
    elif m[0] == "TRT_magic":
        model = P.TRT.with_magic(m[1])
    else:
        model = P.MRT.raw_moments(st, m[1], m[2])
    force = P.Guo((cfg["force"], 0.0, 0.0)) if cfg["force"] else None
    return forest, pdf, handling, model, force, (nx, ny, nz_rank)


def init_state(cfg, pdf, dims, ctx, P):
    if cfg["init"] == "random":
        from paper_1909_13772_b200 import workloads
        rho, u = workloads.random_rho_u(dims, 1000 + ctx.rank)
        P.fill_equilibrium_arrays(pdf, rho, u)
    else:
        P.fill_equilibrium(pdf)


# -------------------------------------------------------------- reference
def cpu_reference(cfg, steps, warmup, seconds):
    """The reference algorithm on the host cores (C restatement, all threads)
    on a bounded z-slab of the workload.  Returns a cpu_baseline dict."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle
    from paper_1909_13772_b200 import workloads
    nx, ny, nz = cfg["cells"]
    nzs = max(4, min(nz, int(round(4_000_000 / (nx * ny)))))
    st = oracle.STENCILS[cfg["stencil"]]
    X, Y, Z = nx + 2, ny + 2, nzs + 2
    flags = None
    crop = None
    bits = {"Fluid": 1, "NoSlip": 2, "UBB": 4, "Pressure": 8, "Solid": 16}
    geo = cfg["geometry"]
    if geo is not None:
        # the GPU arm's own inputs (bench.build), cropped to the slab
        if geo == "cavity":
            code = workloads.cavity_flags((nx, ny, nzs))
            crop = "cavity of the slab's dims"
        elif geo == "tiles":
            # rank 0's 20 % sphere tile (seed 100), its global z-min wall, and
            # a NoSlip cap on the slab's last plane where the crop cuts it
            code = workloads.sphere_mask((nx, ny, nz), 100, 4.0, 8.0, 0.20,
                                         (True, True, False))[:nzs].astype(np.int8)
            code[0] = code[-1] = 1
            crop = f"planes 0..{nzs - 1} of the GPU's tile (seed 100) + NoSlip cap"
        else:
            code = workloads.porous_channel_flags((nx, ny, nzs), 1, 0.25).astype(np.int8)
            crop = "the GPU's geometry (seed 1)" if nzs == nz else "porous slab (seed 1)"
        flags = np.zeros((Z, Y, X), dtype=np.uint32)
        inner = np.full(code.shape, 1, dtype=np.uint32)
        inner[code == 1] = 2
        inner[code == 2] = 4
        flags[1:-1, 1:-1, 1:-1] = inner
    m = cfg["model"]
    force = (cfg["force"], 0.0, 0.0) if cfg["force"] else None
    if m[0] == "SRT":
        model = oracle.Model("SRT", omega=m[1], force=force)
    elif m[0] == "TRT_magic":
        we, wo = oracle.trt_magic(m[1])
        model = oracle.Model("TRT", omega_e=we, omega_o=wo, force=force)
    else:
        M = oracle.raw_moment_basis_d3q27(st)
        S = np.full(27, m[2])
        S[4:9] = m[1]
        model = oracle.Model("MRT", M=M, Minv=np.linalg.inv(M), S=S, force=force)
    dom = oracle.Domain(st, (nx, ny, nzs), cfg["periodic"], model, flags, bits,
                        ubb_velocity=cfg.get("ubb", (0.0, 0.0, 0.0)))
    rho, u = workloads.random_rho_u((nx, ny, nzs), 1000) if cfg["init"] == "random" else (
        np.ones((nzs, ny, nx)), np.zeros((nzs, ny, nx, 3)))
    full = np.zeros((st.q, Z, Y, X))
    full[:] = st.w[:, None, None, None]
    full[:, 1:-1, 1:-1, 1:-1] = np.moveaxis(oracle.equilibrium(rho, u, st), 3, 0)
    dom.set_full(full)
    dom.run(max(1, warmup))
    done, t0 = 0, time.perf_counter()
    while done < steps and (done < 2 or time.perf_counter() - t0 < seconds):
        dom.run(1)
        done += 1
    dt = time.perf_counter() - t0
    cells = nx * ny * nzs
    threads = int(os.environ.get("OMP_NUM_THREADS", oracle.threads_available()))
    return {"value": cells * done / dt / 1e6, "unit": "MLUPS", "cores": threads, "kind": "port",
            "sample": f"{nx}x{ny}x{nzs} slab of {cfg['desc'].split(':')[0]}"
                      + (f" ({crop})" if geo is not None else "")
                      + f", {done} steps, oracle/lbm_oracle.c (reference op order, OpenMP "
                      f"{threads} threads), fp64",
            "seconds": dt, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "same_inputs": geo in ("tiles", "spheres25") or nzs == nz}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1 per process; the reference arm runs on
    # rank 0 alone and uses every host thread (set before libgomp loads)
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle
    os.environ["OMP_NUM_THREADS"] = str(oracle.threads_available())
    base = cpu_reference(cfg, args.steps, args.warmup, max(args.cpu_seconds, 60.0))
    line = {"impl": "reference", "metric": "MLUPS", "value": base["value"], "unit": "MLUPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["desc"]},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "MLUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- main
def main():
    args = parse_args()
    rc = self_launch(args, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    cfg = CONFIGS[args.config]
    dtype = args.dtype or cfg.get("dtype", "f64")
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    import torch
    import torch.distributed as dist
    import paper_1909_13772_b200 as P
    ctx = P.init_distributed()
    dev = ctx.device
    torch.cuda.set_device(dev)
    n = ctx.n_ranks
    if n != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but {n} rank(s) are running: launch N > 1 "
                         "through torchrun or let bench.py self-launch (no WORLD_SIZE)")
    forest, pdf, handling, model, force, dims = build(cfg, ctx, dtype, P)
    init_state(cfg, pdf, dims, ctx, P)
    lat = pdf.lattice
    q = pdf.stencil.q
    rb = lat.real_bytes
    cells_rank = dims[0] * dims[1] * dims[2]
    cells_total = cells_rank * n

    def sweep(k):
        # k sweeps in one call: one validation pass, then (P = 1) a replayed
        # two-step CUDA graph; bitwise identical to k stream_collide calls
        P.stream_collide_n(pdf, model, k, force=force, handling=handling)

    # >= 4 so the two-step CUDA graph (both parities) is captured before the
    # timed region even when the driver asks for W = 3
    sweep(max(4, args.warmup))
    torch.cuda.synchronize()
    ctx.barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lat.launches
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.synchronize()
        ctx.barrier()
        ev0.record(stream)
        sweep(args.steps)
        lat.join_streams()
        ev1.record(stream)
        torch.cuda.synchronize()
        ctx.barrier()
    launches = lat.launches - launches0
    print(f"bench: rank {ctx.rank}/{n} device {dev} halo "
          f"{getattr(lat._halo, 'kind', None) if n > 1 else 'none (1 rank)'}",
          file=sys.stderr, flush=True)
    ms = ev0.elapsed_time(ev1)
    if n > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = cells_total * args.steps / (ms / 1e3) / 1e6
    peak, peak_src = measured_peaks()
    bpc = BYTES_PER_CELL[(q, rb)]
    achieved = cells_rank * bpc / (ms_step / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_{args.config}_{dtype}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "bytes_per_cell": bpc, "peak_source": peak_src,
            "kernel": "lbm::k_fused (pull + bounce-back + collide, one pass)",
            "per_launch_ms": round(ms_step, 4) if n == 1 else None}

    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = run_e2e(args, cfg, ctx, dtype, P, forest, pdf, handling, model, force, dims)

    cpu = None
    if ctx.rank == 0 and n == 1 and not args.no_cpu_baseline and not args.profile:
        cpu = cpu_reference(cfg, 10_000, 1, args.cpu_seconds)

    if ctx.rank == 0:
        line = {
            "metric": "MLUPS", "value": round(value, 1), "unit": "MLUPS", "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak" if cfg["per_gpu"] else "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": cfg["desc"], "global_cells": [dims[0], dims[1], dims[2] * n],
                       "cells_per_gpu": cells_rank, "parallelism": f"z-slab x{n}",
                       "halo": (getattr(lat._halo, "kind", None) if n > 1 else None),
                       "pdf_storage": "fp64" if rb == 8 else "fp32 (f - w_i), fp32 arithmetic on centred populations",
                       "l2": (f"working set {2 * lat.elems * rb / 1e9:.1f} GB per GPU >> 126 MB L2 "
                              "(no flush needed)" if 2 * lat.elems * rb > 4 * 126e6 else
                              f"working set {2 * lat.elems * rb / 1e6:.0f} MB per GPU: largely "
                              "L2-resident, no roofline claim (correctness config)")},
            "mlups_per_gpu": round(value / n, 1),
            "roofline": roof, "e2e": e2e, "cpu_baseline": cpu,
            "clocks": clk.summary(), "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, cfg, ctx, dtype, P, forest, pdf, handling, model, force, dims):
    """Public-API run with host buffers: pinned rho/u -> device (H2D), K
    sweeps, final rho/u -> pinned host (D2H), all inside the timed region."""
    import torch
    import torch.distributed as dist
    nx, ny, nz = dims
    from paper_1909_13772_b200 import workloads
    rho, u = workloads.random_rho_u(dims, 7 + ctx.rank, rho_sigma=0.0, u_amp=1e-3)
    rho_h = torch.from_numpy(rho).pin_memory()
    u_h = torch.from_numpy(u).pin_memory()
    out = (torch.empty(rho_h.shape, dtype=torch.float64).pin_memory(),
           torch.empty(u_h.shape, dtype=torch.float64).pin_memory())

    def job(steps):
        # one public call: host rho/u in, K sweeps, host rho/u out (pipelined
        # over z-plane chunks where the box allows; else the call sequence)
        P.run_arrays(pdf, model, steps, rho_h, u_h, force=force, handling=handling, out=out)

    # one untimed pass: the device staging buffers of the H2D / D2H come
    # from torch's caching allocator afterwards (steady state of a job loop)
    job(2)
    torch.cuda.synchronize()
    ctx.barrier()
    t0 = time.perf_counter()
    job(args.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if ctx.n_ranks > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=ctx.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    cells = nx * ny * nz
    # where the time goes without the pipeline (an untimed replay of the same
    # job as the call sequence fill_equilibrium_arrays -> K x stream_collide
    # -> macroscopic_arrays, each phase between synchronisations)
    phases = {}
    # (one warm pass first: the sequence uses torch copy / slice kernels that
    # run_arrays does not, and their first launch loads modules)
    P.fill_equilibrium_arrays(pdf, rho_h, u_h)
    P.stream_collide(pdf, model, force=force, handling=handling)
    P.macroscopic_arrays(pdf, force=force, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    P.fill_equilibrium_arrays(pdf, rho_h, u_h)
    torch.cuda.synchronize()
    phases["h2d_fill_ms"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    for _ in range(args.steps):
        P.stream_collide(pdf, model, force=force, handling=handling)
    torch.cuda.synchronize()
    phases["sweeps_ms"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    P.macroscopic_arrays(pdf, force=force, out=out)
    torch.cuda.synchronize()
    phases["moments_d2h_ms"] = (time.perf_counter() - t) * 1e3
    moved = cells * 32
    phases["h2d_gbs"] = moved / (phases["h2d_fill_ms"] * 1e6)
    phases["d2h_gbs"] = moved / (phases["moments_d2h_ms"] * 1e6)
    seq_s = (phases["h2d_fill_ms"] + phases["sweeps_ms"] + phases["moments_d2h_ms"]) / 1e3
    phases["sequence_mlups"] = cells * args.steps / seq_s / 1e6
    pipelined = pdf.lattice.can_pipeline()
    return {"value": round(cells * ctx.n_ranks * args.steps / dt / 1e6, 1), "unit": "MLUPS",
            "h2d_bytes_per_step": int(cells * 32 / args.steps),
            "d2h_bytes_per_step": int(cells * 32 / args.steps),
            "seconds": round(dt, 4),
            "pipelined": pipelined,
            "breakdown": {k: round(v, 2) for k, v in phases.items()},
            "timed": "P.run_arrays: pinned host rho/u -> H2D -> equilibrium -> K sweeps -> "
                     "moments -> D2H into pinned host rho/u, "
                     + ("as a wavefront over z-plane chunks (4, 4, 8, 16, then 32 planes; 4-plane "
                        "tail steps; copies overlap the sweeps), "
                        if pipelined else "as the call sequence (periodic z or several ranks), ")
                     + "wall clock, max over ranks, after one untimed pass of the same job; "
                       "breakdown = the unpipelined call sequence replayed untimed"}


if __name__ == "__main__":
    main()
