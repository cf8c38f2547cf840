"""Probe: where the run_arrays job time goes at K steps (config 4 fp64).
(a) pinned host rho/u as in bench.py, (b) the same job with device-resident
inputs/outputs (no PCIe), (c) host time to enqueue every launch, (d) the
device-resident sweep rate of the same lattice right before/after."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import bench
import paper_1909_13772_b200 as P
from paper_1909_13772_b200 import _lib, workloads

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = bench.CONFIGS["c4"]
ctx = P.init_distributed()
torch.cuda.set_device(0)
forest, pdf, handling, model, force, dims = bench.build(cfg, ctx, "f64", P)
bench.init_state(cfg, pdf, dims, ctx, P)
rho, u = workloads.random_rho_u(dims, 7, rho_sigma=0.0, u_amp=1e-3)
host = (torch.from_numpy(rho).pin_memory(), torch.from_numpy(u).pin_memory())
hout = (torch.empty_like(host[0]).pin_memory(), torch.empty_like(host[1]).pin_memory())
dev = (host[0].cuda(), host[1].cuda())
dout = (torch.empty_like(dev[0]), torch.empty_like(dev[1]))

calls = []
orig = _lib.call


def traced(name, *a):
    r = orig(name, *a)
    calls.append(time.perf_counter())
    return r


def sweeps(k):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    P.stream_collide_n(pdf, model, k, force=force, handling=handling)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def job(src, dst):
    lat = pdf.lattice
    lat_kp = None
    calls.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if src[0].is_cuda:
        # run_arrays takes device arrays through the call sequence; drive the
        # wavefront directly with device staging sources instead
        from paper_1909_13772_b200.lbm import sweep as S
        from paper_1909_13772_b200.lbm.collision import SRT, Guo, kernel_params
        lat, kp, key, masks = S._prepare(pdf, model, force, handling, upload=False)
        kp_m = kernel_params(pdf.stencil, SRT(1.0), force)
        lat.run_job(kp, key, masks, kp_m, src[0], src[1], K, dst, None)
    else:
        P.run_arrays(pdf, model, K, src[0], src[1], force=force, handling=handling, out=dst)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    return (t1 - t0) * 1e3, ((calls[-1] - t0) * 1e3 if calls else None), len(calls)


_lib.call = traced
import paper_1909_13772_b200.device as D
D._lib.call = traced
print(f"sweep (graph) ms/step before: {sweeps(10):.3f}")
for rep in range(3):
    for name, src, dst in (("pinned host", host, hout), ("device", dev, dout)):
        ms, enq, n = job(src, dst)
        print(f"{name:12s} K={K}: job {ms:8.2f} ms  last launch enqueued at {enq:8.2f} ms  "
              f"({n} calls)  -> {dims[0]*dims[1]*dims[2]*K/ms/1e3:8.1f} MLUPS")
print(f"sweep (graph) ms/step after: {sweeps(10):.3f}")


def ranges(width, reps=5):
    """One sweep as nz / width plane-range launches (no graph), ms per sweep."""
    from paper_1909_13772_b200.lbm import sweep as S
    lat, kp, key, masks = S._prepare(pdf, model, force, handling)
    nz = lat.box.nz
    src, dst = lat.buf[lat.cur], lat.buf[1 - lat.cur]
    sp = lat._sp()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for r in range(reps):
        a, b = (src, dst) if r % 2 == 0 else (dst, src)
        for z0 in range(0, nz, width):
            orig("lbm_fused_step_bits", lat.gref, kp.ref, _lib.ptr(a), _lib.ptr(b),
                 _lib.ptr(masks.cellmask), None, None, z0, min(nz, z0 + width), sp)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for w in (512, 128, 64, 32, 16, 8, 4):
    ms = ranges(w)
    print(f"one sweep as {512 // w:3d} launches of {w:3d} planes: {ms:.3f} ms "
          f"(+{(ms - 0) * 1e3 / (512 // w):.1f} us per launch incl. work)")
