"""Stress run_arrays against the call sequence (tests/test_pipeline.py cases)
under perturbed allocator state and a busy side stream; on a mismatch print
where it differs and which readout disagrees with the host formula."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import bench  # noqa: E402
import paper_1909_13772_b200 as P  # noqa: E402
from paper_1909_13772_b200 import workloads  # noqa: E402
from test_pipeline import _host_moments  # noqa: E402

CASES = [("c4", (64, 48, 40), 7, 8), ("c4", (64, 48, 40), 1, 5), ("c4", (64, 48, 40), 30, 6),
         ("c1", (48, 40, 44), 9, 44), ("c1", (48, 40, 44), 4, 1)]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(1)
junk = []
side = torch.cuda.Stream()
bad_total = 0
t0 = time.time()
for it in range(iters):
    for cfgname, cells, steps, chunk in CASES:
        runs = []
        for pipelined in (False, True):
            # perturb: random live allocations filled with noise, a busy side stream
            if rng.random() < 0.5:
                junk.append(torch.randn(int(rng.integers(1, 4_000_000)), device="cuda",
                                        dtype=torch.float64))
            if len(junk) > 8:
                junk.pop(0)
            with torch.cuda.stream(side):
                a = torch.randn(2048, 2048, device="cuda")
                for _ in range(int(rng.integers(0, 6))):
                    a = a @ a.T
                    a = a / a.norm()
            cfg = dict(bench.CONFIGS[cfgname], cells=cells)
            forest, pdf, handling, model, force, dims = bench.build(cfg, P.Context(), "f64", P)
            rho, u = workloads.random_rho_u(dims, 77, rho_sigma=0.01, u_amp=0.02)
            rho_h = torch.from_numpy(rho).pin_memory()
            u_h = torch.from_numpy(u).pin_memory()
            out = (torch.empty(rho_h.shape, dtype=torch.float64).pin_memory(),
                   torch.empty(u_h.shape, dtype=torch.float64).pin_memory())
            if pipelined:
                P.run_arrays(pdf, model, steps, rho_h, u_h, force=force, handling=handling,
                             out=out, chunk_planes=chunk)
            else:
                P.fill_equilibrium_arrays(pdf, rho_h, u_h)
                for _ in range(steps):
                    P.stream_collide(pdf, model, force=force, handling=handling)
                P.macroscopic_arrays(pdf, force=force, out=out)
            first = (out[0].numpy().copy(), out[1].numpy().copy())
            host = _host_moments(pdf, force)
            runs.append((first, host))
            del pdf, forest, handling
        (fa, ha), (fb, hb) = runs
        same = fa[0].tobytes() == fb[0].tobytes() and fa[1].tobytes() == fb[1].tobytes()
        if not same:
            bad_total += 1
            du = (fa[1] != fb[1]).any(-1)
            print(f"it {it} {cfgname} steps {steps} chunk {chunk}: rho diff "
                  f"{int((fa[0] != fb[0]).sum())} u diff cells {int(du.sum())}; "
                  f"R_K equal {ha[0].tobytes() == hb[0].tobytes()}; "
                  f"seq vs host u {int((fa[1] != ha[1]).any(-1).sum())}, "
                  f"job vs host u {int((fb[1] != hb[1]).any(-1).sum())}; "
                  f"planes {np.nonzero(du.any((1, 2)))[0].tolist()[:20]}; "
                  f"max |du| {float(np.abs(fa[1] - fb[1]).max()):.3e}", flush=True)
print(f"{iters} iterations x {len(CASES)} cases: {bad_total} mismatches, "
      f"{time.time() - t0:.1f} s", flush=True)
