"""Test helper: give a (z-invariant) Euler test state a smooth z dependence -- density and
momentum scaled by a z profile, a z velocity added, the internal energy kept -- so that every
z-direction path (plane rings, z chunks, slab halos) is exercised; with the z-invariant vortex
or Sod a misplaced z plane reads identical data and goes unnoticed."""
import numpy as np


def modulate_z(s0, k0=0):
    """s0: skinny [mz][my][mx][5] (modified in place and returned); k0: global index of
    storage plane 0 (z slabs)."""
    z = np.arange(s0.shape[0], dtype=float) + k0
    m = (1.0 + 0.08 * np.sin(0.9 * z + 0.4))[:, None, None]
    w = (0.3 * np.cos(0.6 * z + 0.1))[:, None, None]
    rho0 = s0[..., 0].copy()
    p_int = s0[..., 4] - 0.5 * (s0[..., 1] ** 2 + s0[..., 2] ** 2 + s0[..., 3] ** 2) / rho0
    rho = rho0 * m
    s0[..., 1] *= m
    s0[..., 2] *= m
    s0[..., 3] = rho * w
    s0[..., 0] = rho
    s0[..., 4] = p_int + 0.5 * (s0[..., 1] ** 2 + s0[..., 2] ** 2 + s0[..., 3] ** 2) / rho
    return s0
