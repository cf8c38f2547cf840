"""Seeded synthetic inputs of the BASELINE.json configs.

No public dataset is named by the reference or BASELINE.json; these
generators define the inputs (SURVEY.md section 8d "Synthetic inputs").  All
RNG draws run over the *global* grid in (z, y, x) C-order, so inputs do not
depend on the number of ranks.  Pure numpy (host setup, not the hot path).
"""
from __future__ import annotations

import numpy as np


def random_rho_u(dims, seed, rho_sigma=0.01, u_amp=0.05):
    """rho = 1 + sigma N(0,1), u ~ U(-amp, amp)^3 per cell (configs 0 and 3).
    dims = (nx, ny, nz); returns rho (nz, ny, nx), u (nz, ny, nx, 3)."""
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    rho = 1.0 + rho_sigma * rng.standard_normal((nz, ny, nx))
    u = rng.uniform(-u_amp, u_amp, (nz, ny, nx, 3))
    return rho, u


def sphere_mask(dims, seed, rmin, rmax, solid_fraction, periodic=(True, True, False),
                max_spheres=10_000_000):
    """Random porous medium: spheres with centres U[0, n)^3 and radii
    U[rmin, rmax] added until the solid fraction reaches `solid_fraction`
    (config 1: 128^3, radii 4-8, ~25 %).  Periodic axes wrap.  Returns a
    bool array (nz, ny, nx), True = solid."""
    nx, ny, nz = dims
    n = np.array([nx, ny, nz])
    rng = np.random.default_rng(seed)
    solid = np.zeros((nz, ny, nx), dtype=bool)
    target = solid_fraction * solid.size
    count = 0
    for _ in range(max_spheres):
        if count >= target:
            break
        c = rng.uniform(0.0, 1.0, 3) * n
        r = rng.uniform(rmin, rmax)
        lo = np.floor(c - r).astype(int)
        hi = np.ceil(c + r).astype(int) + 1
        idx = []
        for a in range(3):
            ax = np.arange(lo[a], hi[a])
            if periodic[a]:
                ax = ax % n[a]
                ax_c = np.arange(lo[a], hi[a]) + 0.5 - c[a]
            else:
                keep = (ax >= 0) & (ax < n[a])
                ax_c = ax[keep] + 0.5 - c[a]
                ax = ax[keep]
            idx.append((ax, ax_c))
        (ix, dx), (iy, dy), (iz, dz) = idx
        if ix.size == 0 or iy.size == 0 or iz.size == 0:
            continue
        d2 = dz[:, None, None] ** 2 + dy[None, :, None] ** 2 + dx[None, None, :] ** 2
        inside = d2 <= r * r
        sub = solid[np.ix_(iz, iy, ix)]
        new = inside & ~sub
        count += int(new.sum())
        solid[np.ix_(iz, iy, ix)] = sub | inside
    return solid


def porous_channel_flags(dims, seed, solid_fraction=0.25, rmin=4.0, rmax=8.0,
                         walls_z=True, periodic=(True, True, False)):
    """Config 1 geometry: spheres (NoSlip) + NoSlip planes z = 0 and z = nz-1
    (interior planes).  Returns (solid, wall) bool arrays;
    every solid cell is flagged NoSlip, never Solid (boundary.py:83-86)."""
    nx, ny, nz = dims
    solid = sphere_mask(dims, seed, rmin, rmax, solid_fraction, periodic)
    if walls_z:
        solid[0] = True
        solid[nz - 1] = True
    return solid


def tiled_porous_flags(dims_per_tile, tiles, base_seed=100, solid_fraction=0.20, rmin=4.0,
                       rmax=8.0):
    """Config 4 geometry: one independent 20 % sphere tile per GPU stacked in
    z (seed base_seed + k for tile k, so P = 1 is a sub-problem of P = 8),
    NoSlip walls at the global z-min/z-max planes, periodic x, y."""
    nx, ny, nz = dims_per_tile
    parts = [sphere_mask((nx, ny, nz), base_seed + k, rmin, rmax, solid_fraction,
                         (True, True, False)) for k in range(tiles)]
    solid = np.concatenate(parts, axis=0)
    solid[0] = True
    solid[-1] = True
    return solid


def cavity_flags(dims):
    """Config 2 geometry: NoSlip on five faces (interior boundary planes) and a
    UBB lid on the top plane z = nz-1, lid edges UBB (NoSlip first, then the
    lid plane overwritten).  Returns int codes: 0 fluid, 1 NoSlip, 2 UBB."""
    nx, ny, nz = dims
    code = np.zeros((nz, ny, nx), dtype=np.int8)
    code[0] = 1
    code[:, 0] = 1
    code[:, ny - 1] = 1
    code[:, :, 0] = 1
    code[:, :, nx - 1] = 1
    code[nz - 1] = 2
    return code
