"""Probe: per-window step time over a long sweep loop (does the fused kernel
slow down as the board heats / hits its power cap?).  Usage:
python tools/probe/steady.py CFG DTYPE WINDOWS STEPS_PER_WINDOW"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import pynvml

import bench
import paper_1909_13772_b200 as P

cfgname, dt, nwin, per = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cfg = bench.CONFIGS[cfgname]
ctx = P.init_distributed()
torch.cuda.set_device(0)
forest, pdf, handling, model, force, dims = bench.build(cfg, ctx, dt, P)
bench.init_state(cfg, pdf, dims, ctx, P)
cells = dims[0] * dims[1] * dims[2]
bpc = bench.BYTES_PER_CELL[(pdf.stencil.q, pdf.lattice.real_bytes)]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
P.stream_collide_n(pdf, model, 6, force=force, handling=handling)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(nwin + 1)]
evs[0].record(s)
for w in range(nwin):
    P.stream_collide_n(pdf, model, per, force=force, handling=handling)
    evs[w + 1].record(s)
samples = []
while not evs[-1].query():
    samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetTemperature(h, 0)))
    time.sleep(0.02)
torch.cuda.synchronize()
peak = 6538.6
for w in range(nwin):
    ms = evs[w].elapsed_time(evs[w + 1]) / per
    print(f"{cfgname} {dt} window {w:3d}: {ms:.4f} ms/step  frac {cells * bpc / ms / 1e6 / peak:.4f}")
k = max(1, len(samples) // 8)
for i in range(0, len(samples), k):
    print("clock/power/temp", samples[i])
