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


def _host_moments(pdf, force):
    """rho / u of R_K (the state the readout reads) in numpy, the reference's
    macroscopic() (lbm/collision.py:157-184) op for op: sequential density,
    momentum in index order, u = m (1 / rho) (+ (F / 2) (1 / rho) for Guo)."""
    import paper_1909_13772_b200 as P
    kind, dev = pdf.lattice.readout_device()
    f = dev.cpu().numpy()
    if kind == "full":
        f = f[:, 1:-1, 1:-1, 1:-1]
    c = np.asarray(pdf.stencil.c)
    rho = f[0].copy()
    for i in range(1, f.shape[0]):
        rho = rho + f[i]
    m = np.zeros(rho.shape + (3,))
    for i in range(f.shape[0]):
        for a in range(3):
            if c[i][a]:
                m[..., a] += c[i][a] * f[i]
    inv = (1.0 / rho)[..., None]
    u = m * inv
    if isinstance(force, P.Guo):
        u = u + 0.5 * np.asarray(force.force) * inv
    return rho, u


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
        host = _host_moments(pdf, force)
        m = pdf.lattice.stream_masks
        fluid = (m.cellmask.cpu().numpy() & 1).astype(bool) if m is not None else None
        # the end state continues exactly like the sequence's
        for _ in range(3):
            P.stream_collide(pdf, model, force=force, handling=handling)
        kind, dev = pdf.lattice.readout_device()
        rho2, u2 = P.macroscopic_arrays(pdf, force=force)
        runs.append((first, dev.cpu().numpy(), rho2.cpu().numpy(), u2.cpu().numpy(),
                     pdf.lattice.steps, host, fluid))
        del pdf, forest, handling
    (a_first, a_pdf, a_rho, a_u, a_steps, a_host, fluid), \
        (b_first, b_pdf, b_rho, b_u, b_steps, b_host, _) = runs
    assert a_steps == b_steps == steps + 3
    assert a_host[0].tobytes() == b_host[0].tobytes() and a_host[1].tobytes() == b_host[1].tobytes(), \
        "R_K after the job"
    # both readouts against the reference formula on the host (collision.py:157-184);
    # fp64 NoSlip tiles only (fp32 readouts widen centred populations, and the
    # UBB lid's R_K carries the wall term the host copy of S(G) does not)
    checks = (("call sequence", a_first), ("run_arrays", b_first)) \
        if dtype == "f64" and config in ("c4", "c1") else ()
    for name, first in checks:
        nr = int((first[0] != a_host[0]).sum())
        du = (first[1] != a_host[1]).any(-1)
        nu = int(du.sum())
        where = "" if fluid is None else \
            f" ({int((du & fluid).sum())} fluid, {int((du & ~fluid).sum())} of {int((~fluid).sum())} non-fluid)"
        assert nr == 0 and nu == 0, (
            f"{name}: {nr} rho / {nu} u cells differ from the host readout{where}, "
            f"max |du| {float(np.abs(first[1] - a_host[1]).max()):.3e}")
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
