"""run_arrays (the pipelined host-to-host job) against the call sequence it
replaces: fill_equilibrium_arrays -> K x stream_collide -> macroscopic_arrays
(reference sweep.py:51-183).  The wavefront over z-plane chunks runs the same
kernels in another order, so rho / u and the end state must agree BITWISE,
for every chunk size (1 plane, uneven, the whole box) and step count (1, a
few, more than the chunk count), fp64 and fp32 storage, NoSlip porous tiles
and the D3Q27 UBB cavity; a periodic z axis takes the unpipelined path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lattice(config, dtype, cells):
    import bench
    import paper_1909_13772_b200 as P
    cfg = dict(bench.CONFIGS[config], cells=cells)
    ctx = P.Context()
    forest, pdf, handling, model, force, dims = bench.build(cfg, ctx, dtype, P)
    return P, forest, pdf, handling, model, force, dims


CASES = [
    ("c4", "f64", (64, 48, 40), 7, 8),
    ("c4", "f64", (64, 48, 40), 1, 5),
    ("c4", "f64", (64, 48, 40), 30, 6),     # more steps than chunks: the wavefront drains
    ("c4", "f32", (64, 48, 41), 6, 3),      # fp32: k_fused_z2 on odd plane ranges
    ("c1", "f64", (48, 40, 44), 9, 44),     # one chunk = the whole box
    ("c1", "f64", (48, 40, 44), 4, 1),      # one plane per chunk
    ("c2", "f32", (40, 36, 34), 5, 4),      # D3Q27 factorised MRT + UBB lid (typed links)
    ("c2", "f64", (40, 36, 34), 3, 7),
    ("c3", "f64", (32, 32, 24), 5, 4),      # periodic z: unpipelined fallback
]


@pytest.mark.parametrize("config,dtype,cells,steps,chunk", CASES)
def test_run_arrays_bitwise_vs_call_sequence(config, dtype, cells, steps, chunk):
    import torch
    from paper_1909_13772_b200 import workloads
    runs = []
    for pipelined in (False, True):
        P, forest, pdf, handling, model, force, dims = _lattice(config, dtype, cells)
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
        first = (out[0].numpy().copy(), out[1].numpy().copy())
        # the end state continues exactly like the sequence's
        for _ in range(3):
            P.stream_collide(pdf, model, force=force, handling=handling)
        kind, dev = pdf.lattice.readout_device()
        rho2, u2 = P.macroscopic_arrays(pdf, force=force)
        runs.append((first, dev.cpu().numpy(), rho2.cpu().numpy(), u2.cpu().numpy(),
                     pdf.lattice.steps))
        del pdf, forest, handling
    (a_first, a_pdf, a_rho, a_u, a_steps), (b_first, b_pdf, b_rho, b_u, b_steps) = runs
    assert a_steps == b_steps == steps + 3
    assert a_first[0].tobytes() == b_first[0].tobytes(), "rho after the job"
    assert a_first[1].tobytes() == b_first[1].tobytes(), "u after the job"
    assert a_pdf.tobytes() == b_pdf.tobytes(), "PDFs three sweeps after the job"
    assert a_rho.tobytes() == b_rho.tobytes() and a_u.tobytes() == b_u.tobytes()
    assert np.isfinite(a_first[0]).all()


def test_run_arrays_rejects_wrong_shapes():
    import paper_1909_13772_b200 as P
    from paper_1909_13772_b200.errors import ValidationError
    P_, forest, pdf, handling, model, force, dims = _lattice("c4", "f64", (32, 32, 16))
    nx, ny, nz = dims
    with pytest.raises(ValidationError):
        P.run_arrays(pdf, model, 2, np.ones((nz, ny, nx + 1)), np.zeros((nz, ny, nx, 3)),
                     force=force, handling=handling)
    with pytest.raises(ValidationError):
        P.run_arrays(pdf, model, -1, np.ones((nz, ny, nx)), np.zeros((nz, ny, nx, 3)),
                     force=force, handling=handling)
