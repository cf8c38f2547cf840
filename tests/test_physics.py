"""Physics checks of the reference's LBM suite, re-expressed on the GPU path
("reference tests to re-express"; the reference's own are
pkg/tests/test_lbm.py:619-742).  Bitwise parity already pins the kernels
against the reference; these check that the physics they produce is right:

* Poiseuille flow between bounce-back walls converges at second order;
* the body-force parabola between resting walls equals, shifted by the
  frame velocity, the one between UBB walls moving backwards;
* UBB walls at zero velocity are NoSlip walls, bit for bit;
* a moving UBB lid gives the linear Couette profile;
* at the TRT magic parameter the wall sits exactly half-way (the parabola
  is resolution-exact for every even rate);
* a closed box conserves mass.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _P():
    import paper_1909_13772_b200 as P
    return P


def channel(H, model, *, force=0.0, wall="NoSlip", top=None, wall_velocity=(0.0, 0.0, 0.0),
            u0=0.0, steps=100, width=2):
    """D2Q9 channel, periodic in x, walls on the interior rows y = 0 and
    y = H + 1; returns the x-averaged u_x of the H fluid rows after `steps`."""
    P = _P()
    forest = P.create_forest(P.Context(), (0, 0, 0, 1, 1, 1), (1, 1, 1), d=2,
                             periodic=(True, False, False), cells_per_block=(width, H + 2, 1))
    pdf = P.PdfField(forest, P.D2Q9)
    reg = P.ensure_flags(forest).registry
    for block in forest.local_blocks():
        inner = block.data["flags"].interior
        inner[...] = reg["Fluid"]
        inner[0, 0, :] = reg[wall]
        inner[0, -1, :] = reg[top or wall]
    P.fill_equilibrium(pdf, 1.0, (u0, 0.0))
    handling = P.BoundaryHandling(forest, P.D2Q9, ubb_velocity=wall_velocity)
    guo = P.Guo((force, 0.0, 0.0)) if force else None
    P.stream_collide_n(pdf, model, steps, force=guo, handling=handling)
    f = P.gather_slice(forest, "pdf", (0, 0, 0), forest.global_cells(0))[0]
    rho = f.sum(axis=-1)
    ux = (f @ P.D2Q9.cx.astype(np.float64) + 0.5 * force) / rho
    return ux[1:-1].mean(axis=1)


def parabola(H, g, nu):
    """Body-force Poiseuille profile with the walls half a cell outside the
    first / last fluid row."""
    y = np.arange(H) + 0.5
    return g / (2.0 * nu) * y * (H - y)


def settle(H, nu, decades):
    """Steps for the slowest diffusive mode to decay by e^-decades."""
    return int(math.ceil(decades * H * H / (nu * math.pi ** 2)))


def rms_rel(a, b, scale):
    return float(np.sqrt(np.mean((a - b) ** 2))) / scale


def test_poiseuille_converges_at_second_order():
    P = _P()
    omega, u_max = 1.2, 0.01
    nu = (1.0 / omega - 0.5) / 3.0
    err = {}
    for H in (16, 32):
        g = 8.0 * nu * u_max / (H * H)
        prof = channel(H, P.SRT(omega), force=g, steps=settle(H, nu, 10))
        err[H] = rms_rel(prof, parabola(H, g, nu), u_max)
    assert 3.3 <= err[16] / err[32] <= 4.7, err


def test_body_force_equals_moving_walls_in_the_wall_frame():
    P = _P()
    H, omega, u_max = 16, 1.2, 0.01
    nu = (1.0 / omega - 0.5) / 3.0
    g = 8.0 * nu * u_max / (H * H)
    steps = settle(H, nu, 22)
    resting = channel(H, P.SRT(omega), force=g, steps=steps)
    moving = channel(H, P.SRT(omega), force=g, steps=steps, wall="UBB",
                     wall_velocity=(-u_max, 0.0, 0.0), u0=-u_max)
    assert np.max(np.abs(resting - (moving + u_max))) < 1e-10
    assert rms_rel(resting, parabola(H, g, nu), u_max) < 5e-3


def test_ubb_at_rest_is_noslip_bitwise():
    P = _P()
    a = channel(8, P.SRT(1.3), force=1e-5, steps=40)
    b = channel(8, P.SRT(1.3), force=1e-5, steps=40, wall="UBB")
    assert a.tobytes() == b.tobytes()


def test_couette_profile_from_a_moving_lid():
    P = _P()
    H, omega, U = 16, 1.2, 0.02
    nu = (1.0 / omega - 0.5) / 3.0
    prof = channel(H, P.SRT(omega), top="UBB", wall_velocity=(U, 0.0, 0.0),
                   steps=settle(H, nu, 22))
    y = np.arange(H) + 0.5
    assert np.max(np.abs(prof - U * y / H)) / U < 1e-8


def test_trt_magic_puts_the_wall_half_way():
    P = _P()
    H, u_max = 8, 0.01
    errs = []
    for omega_e in (0.6, 1.0, 1.4, 1.8):
        nu = (1.0 / omega_e - 0.5) / 3.0
        g = 8.0 * nu * u_max / (H * H)
        prof = channel(H, P.TRT.with_magic(omega_e), force=g, steps=settle(H, nu, 30))
        errs.append(rms_rel(prof, parabola(H, g, nu), u_max))
    errs = np.array(errs)
    assert (errs < 1e-9).all() or np.ptp(errs) / errs.mean() < 0.10, errs.tolist()


def test_closed_box_conserves_mass():
    """D3Q19 TRT in a NoSlip box from a random start: the fluid cells keep
    their mass to round-off (bounce-back links reflect, never lose)."""
    P = _P()
    n = 12
    forest = P.create_forest(P.Context(), (0, 0, 0, 1, 1, 1), (1, 1, 1),
                             periodic=(False, False, False), cells_per_block=(n, n, n))
    pdf = P.PdfField(forest, P.D3Q19, layout="fzyx")
    reg = P.ensure_flags(forest).registry
    blk = forest.local_blocks()[0]
    flags = blk.data["flags"].interior
    flags[...] = reg["NoSlip"]
    flags[1:-1, 1:-1, 1:-1] = reg["Fluid"]
    P.fill_equilibrium(pdf)
    rng = np.random.default_rng(3)
    rho = 1.0 + 0.01 * rng.standard_normal((n, n, n))
    u = rng.uniform(-0.02, 0.02, (n, n, n, 3))
    inner = pdf.src(blk).interior
    inner[1:-1, 1:-1, 1:-1] = P.equilibrium(rho, u, P.D3Q19)[1:-1, 1:-1, 1:-1]
    handling = P.BoundaryHandling(forest, P.D3Q19)
    fluid = np.zeros((n, n, n), bool)
    fluid[1:-1, 1:-1, 1:-1] = True
    m0 = float(pdf.src(blk).interior[fluid].sum())
    P.stream_collide_n(pdf, P.TRT.with_magic(1.6), 200, handling=handling)
    m1 = float(pdf.src(blk).interior[fluid].sum())
    assert abs(m1 - m0) < 1e-12 * m0
