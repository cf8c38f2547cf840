"""Probe: cost of the z-slab split and the fused device-side halo on ONE
B200, with ranks as threads sharing the GPU (runtime backend "threads": each
rank has its own streams; the halo is the boundary kernel's peer stores plus
stream-ordered flag words, no kernel ever spins).  Strong: config 3 (512^3
periodic, fixed) on 1 / 2 / 4 slabs - ideal time = the 1-slab time.  Weak:
config 4 tiles stacked in z, 512^3 per rank - ideal time = ranks x the
1-rank time.  The ranks' sweeps are serialised on one device, so this
measures the split + halo overhead, not NVLink.
Usage: python tools/probe/split_probe.py"""
import sys
import threading
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import bench
import paper_1909_13772_b200 as P

STEPS, WARM = 20, 6
_bar = {}


def prog(ctx, cfgname, dtype):
    cfg = bench.CONFIGS[cfgname]
    torch.cuda.set_device(0)
    forest, pdf, handling, model, force, dims = bench.build(cfg, ctx, dtype, P)
    bench.init_state(cfg, pdf, dims, ctx, P)
    P.stream_collide_n(pdf, model, WARM, force=force, handling=handling)
    pdf.lattice.join_streams()
    torch.cuda.synchronize()
    ctx.barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    P.stream_collide_n(pdf, model, STEPS, force=force, handling=handling)
    pdf.lattice.join_streams()
    e1.record(s)
    torch.cuda.synchronize()
    ctx.barrier()
    kind = getattr(pdf.lattice._halo, "kind", None) if ctx.n_ranks > 1 else None
    return e0.elapsed_time(e1) / STEPS, dims, kind


for cfgname, ranks_list in (("c3", (1, 2, 4)), ("c4", (1, 2))):
    base = None
    for n in ranks_list:
        res = P.run(n, prog, cfgname, "f64", backend="threads", device="cuda", timeout=900)
        ms = max(r[0] for r in res)
        dims, kind = res[0][1], res[0][2]
        cells = dims[0] * dims[1] * dims[2] * n
        base = base or ms
        ideal = base if cfgname == "c3" else base * n
        print(f"{cfgname} f64 {n} slab(s) of {dims}: {ms:.3f} ms/step, {cells / ms / 1e3:.0f} MLUPS "
              f"on the one GPU, overhead vs ideal {100 * (ms / ideal - 1):+.1f} %  (halo {kind})",
              flush=True)
        torch.cuda.empty_cache()
