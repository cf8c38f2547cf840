"""Where does run_arrays' fused readout (lbm_fused_step_moments) differ from
the call sequence's?  Prints per-component counts of differing u cells,
split by fluid / non-fluid and by plane, for one small config-1 job."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import bench  # noqa: E402
import paper_1909_13772_b200 as P  # noqa: E402
from paper_1909_13772_b200 import workloads  # noqa: E402

cfgname, cells, steps, chunk = sys.argv[1], tuple(int(v) for v in sys.argv[2].split(",")), \
    int(sys.argv[3]), int(sys.argv[4])
runs = []
for pipelined in (False, True):
    cfg = dict(bench.CONFIGS[cfgname], cells=cells)
    ctx = P.Context()
    forest, pdf, handling, model, force, dims = bench.build(cfg, ctx, "f64", P)
    rho, u = workloads.random_rho_u(dims, 77, rho_sigma=0.01, u_amp=0.02)
    rho_h = torch.from_numpy(rho).pin_memory()
    u_h = torch.from_numpy(u).pin_memory()
    out = (torch.empty(rho_h.shape, dtype=torch.float64).pin_memory(),
           torch.empty(u_h.shape, dtype=torch.float64).pin_memory())
    if pipelined:
        P.run_arrays(pdf, model, steps, rho_h, u_h, force=force, handling=handling, out=out,
                     chunk_planes=chunk)
    else:
        P.fill_equilibrium_arrays(pdf, rho_h, u_h)
        for _ in range(steps):
            P.stream_collide(pdf, model, force=force, handling=handling)
        P.macroscopic_arrays(pdf, force=force, out=out)
    kind, dev = pdf.lattice.readout_device()
    masks = pdf.lattice.stream_masks
    cm = masks.cellmask.cpu().numpy().reshape(dims[2], dims[1], dims[0]) if masks is not None \
        and masks.cellmask is not None else None
    runs.append((out[0].numpy().copy(), out[1].numpy().copy(), dev.cpu().numpy(), cm))
(ra, ua, pa, cm), (rb, ub, pb, _) = runs
print("rho equal", ra.tobytes() == rb.tobytes(), "pdf equal", pa.tobytes() == pb.tobytes())
d = ua != ub
print("u differing cells per component", d.reshape(-1, 3).sum(0), "of", ua.size // 3)
if cm is not None:
    fl = (cm & 1).astype(bool)
    dc = d.any(-1)
    print("differing fluid", int((dc & fl).sum()), "non-fluid", int((dc & ~fl).sum()),
          "fluid total", int(fl.sum()))
print("per plane", d.any(-1).sum((1, 2)).tolist())
idx = np.argwhere(d.any(-1))[:5]
for z, y, x in idx:
    print(z, y, x, ua[z, y, x], ub[z, y, x], (ua[z, y, x] - ub[z, y, x]), "mask",
          None if cm is None else hex(int(cm[z, y, x])))
