"""ced_oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

numpy restatement of the CED step of paper_2211_13295_b200/csrc/ced.cu (Maxwell's equations
in a conducting medium, face-centred D and B by constrained transport, 2D upwind edge
solver, ADER predictor with the conduction source solved by the exponential step), with the
same expression shapes. The only operations that are not plain IEEE arithmetic are exp and
expm1 of the conduction decay, whose CUDA and libm results may differ by an ulp -- the GPU
comparison is therefore held to 1e-13 relative, bitwise wherever sigma = 0.

PARITY UNPINNED: the reference scopes out CED and stiff-source ADER; no
CED code, test or fixture exists under /root/reference. Self-consistency checks live in
tests/test_ced_oracle.py and tests/test_ced_gpu.py (exact plane waves and their convergence,
div B = 0 and div D = 0 for uniform sigma to round-off, electromagnetic energy never
increases, exact decay of a uniform field for any sigma dt, the magnetic-diffusion limit
recovered by the asymptotic-preserving edge dissipation).

Layout: state[6][mz+1][my+1][mx+1] = Dx, Dy, Dz, Bx, By, Bz on the low face of the zone
with the same index; sigma[mz+1][my+1][mx+1] per zone.
"""
from __future__ import annotations

import numpy as np

from oracle.mhd_oracle import (PERIODIC, OUTFLOW, Geom, _ax, _shift, extrap, mc_limiter,  # noqa
                               weno3)

NF = 6


class Params:
    def __init__(self, order, eps=1.0, mu=1.0, cfac_other=1.5, weno_eps=1e-12,
                 w=(0.25, 0.5, 0.25), bc=(PERIODIC, PERIODIC, PERIODIC)):
        self.order, self.eps_, self.mu = order, eps, mu
        self.c = 1.0 / np.sqrt(eps * mu)
        self.cfac_other, self.eps, self.w = cfac_other, weno_eps, w  # (weno3 reads .eps, .w)
        self.bc = bc


def fill_ghosts(s, sigma, g: Geom, bc):
    R, Q, P = g.shape
    ext = (P, Q, R)
    arrays = [(q, s[q]) for q in range(NF)] + ([(NF, sigma)] if sigma is not None else [])
    for q, arr in arrays:
        idx = []
        for d in range(3):
            lo, hi = g.gh, g.gh + g.n[d]
            if q < NF and q % 3 == d and bc[d] == OUTFLOW:
                hi += 1
            c = np.arange(ext[d])
            idx.append(lo + np.mod(c - lo, hi - lo) if bc[d] == PERIODIC else np.clip(c, lo, hi - 1))
        arr[...] = arr[np.ix_(idx[2], idx[1], idx[0])]
    return s


def cell_avg(s, o3):
    w = []
    for q in range(NF):
        d = q % 3
        b0, b1 = s[q], _shift(s[q], d, 1)
        c = 0.5 * (b0 + b1)
        if o3:
            c = c - (1.0 / 24.0) * (((_shift(s[q], d, 2) - b1) - b0) + _shift(s[q], d, -1))
        w.append(c)
    return w


def decay(z):
    z = np.asarray(z, dtype=np.float64)
    ex = np.exp(-z)
    with np.errstate(divide="ignore", invalid="ignore"):
        ph = np.where(z > 0.0, -np.expm1(-z) / np.where(z > 0.0, z, 1.0), 1.0)
    return ex, ph


def maxwell_flux(u, ie, im, A):
    A1, A2 = (A + 1) % 3, (A + 2) % 3
    f = [None] * NF
    zero = 0.0 * u[0]
    f[A] = zero
    f[A1] = u[3 + A2] * im
    f[A2] = -(u[3 + A1] * im)
    f[3 + A] = zero
    f[3 + A1] = -(u[A2] * ie)
    f[3 + A2] = u[A1] * ie
    return f


class Modes:
    pass


def predict(s, sigma, g: Geom, par: Params, dt):
    o3 = par.order == 3
    w = cell_avg(s, o3)
    ring = tuple(slice(g.gh - 1, g.gh + g.n[2 - ax] + 1) for ax in range(3))

    def sh(arr, dd):
        out = arr
        for d in range(3):
            if dd[d]:
                out = _shift(out, d, dd[d])
        return out[ring]

    face = [[None] * NF for _ in range(6)]
    lin = [[None] * NF for _ in range(3)]
    quad = [[None] * NF for _ in range(3)]
    cross = [[None] * NF for _ in range(3)]
    u0 = [w[q][ring] for q in range(NF)]
    for q in range(NF):
        c0 = u0[q]
        for d in range(3):
            e = [0, 0, 0]
            e[d] = 1
            up, um = sh(w[q], e), sh(w[q], [-x for x in e])
            if not o3:
                lin[d][q] = mc_limiter(up - c0, c0 - um, par.cfac_other)
                quad[d][q] = 0.0
            else:
                lin[d][q], quad[d][q] = weno3(sh(w[q], [-2 * x for x in e]), um, c0, up,
                                              sh(w[q], [2 * x for x in e]), par)
            face[2 * d][q] = extrap(c0, +1.0, lin[d][q], quad[d][q], o3)
            face[2 * d + 1][q] = extrap(c0, -1.0, lin[d][q], quad[d][q], o3)
            if o3:
                da = [0, 0, 0]
                db = [0, 0, 0]
                da[d] = 1
                db[(d + 1) % 3] = 1
                pp = sh(w[q], [da[x] + db[x] for x in range(3)])
                pm = sh(w[q], [da[x] - db[x] for x in range(3)])
                mp = sh(w[q], [-da[x] + db[x] for x in range(3)])
                mm = sh(w[q], [-da[x] - db[x] for x in range(3)])
                cross[d][q] = 0.25 * ((pp - pm) - (mp - mm))
    ie, im = 1.0 / par.eps_, 1.0 / par.mu
    idd = [1.0 / g.d[0], 1.0 / g.d[1], 1.0 / g.d[2]]
    ex, ph = decay(sigma[ring] * ie * (0.5 * dt))
    tau = [0.0] * NF
    for p in range(2 if o3 else 1):
        div = None
        for A in range(3):
            ua = [face[2 * A][q] + 0.5 * tau[q] if p else face[2 * A][q] for q in range(NF)]
            ub = [face[2 * A + 1][q] + 0.5 * tau[q] if p else face[2 * A + 1][q]
                  for q in range(NF)]
            fa, fb = maxwell_flux(ua, ie, im, A), maxwell_flux(ub, ie, im, A)
            if A == 0:
                div = [(fa[q] - fb[q]) * idd[0] for q in range(NF)]
            else:
                div = [div[q] + (fa[q] - fb[q]) * idd[A] for q in range(NF)]
        tau = [2.0 * ((ex * u0[q] + ph * (0.5 * dt) * (-div[q])) - u0[q]) for q in range(3)] + \
              [(-dt) * div[q] for q in range(3, NF)]

    def box(v):
        out = np.zeros(g.shape)
        out[ring] = v
        return out
    # ced.cu's 12 edge-midpoint states (spatial part) and tau/2
    m = Modes()
    m.ht = [box(0.5 * tau[q]) for q in range(NF)]
    m.st = [[None] * NF for _ in range(12)]
    for q in range(NF):
        for C in range(3):
            AA, BB = (C + 1) % 3, (C + 2) % 3
            for lb in range(2):
                for la in range(2):
                    xa = 0.5 if la == 0 else -0.5
                    xb = 0.5 if lb == 0 else -0.5
                    v = u0[q] + xa * lin[AA][q] + xb * lin[BB][q]
                    if o3:
                        v = (v + (1.0 / 6.0) * quad[AA][q] + (1.0 / 6.0) * quad[BB][q] +
                             (xa * xb) * cross[AA][q])
                    m.st[4 * C + 2 * lb + la][q] = box(v)
    return m


def edges(m, g: Geom, par: Params, C, sigma):
    AA, BB = (C + 1) % 3, (C + 2) % 3
    sel = [slice(None)] * 3
    for d in range(3):
        sel[_ax(d)] = slice(g.gh, g.gh + g.n[d] + (0 if d == C else 1))
    sel = tuple(sel)
    e = h = dbp = dbm = dap = dam = bbp = bbm = bap = bam = 0.0
    for lb in range(2):
        for la in range(2):
            def z(arr):
                out = arr
                if la == 0:
                    out = _shift(out, AA, -1)
                if lb == 0:
                    out = _shift(out, BB, -1)
                return out[sel]
            u = [z(m.st[4 * C + 2 * lb + la][q]) + z(m.ht[q]) for q in range(NF)]
            e = e + u[C]
            h = h + u[3 + C]
            if la:
                dbp = dbp + u[BB]
                bbp = bbp + u[3 + BB]
            else:
                dbm = dbm + u[BB]
                bbm = bbm + u[3 + BB]
            if lb:
                dap = dap + u[AA]
                bap = bap + u[3 + AA]
            else:
                dam = dam + u[AA]
                bam = bam + u[3 + AA]
    hc = 0.5 * par.c
    E = np.zeros(g.shape)
    H = np.zeros(g.shape)
    # asymptotic-preserving scaling of the upwind dissipation (Jin-Levermore type): with
    # sigma_e the mean conductivity of the four zones, theta = 1 / (1 + sigma_e h / (2 c eps))
    # per direction; theta = 1 (plain upwind) where sigma_e = 0
    sg = 0.0
    for lb in range(2):
        for la in range(2):
            out = sigma
            if la == 0:
                out = _shift(out, AA, -1)
            if lb == 0:
                out = _shift(out, BB, -1)
            sg = sg + out[sel]
    sg = 0.25 * sg
    ta = 1.0 / (1.0 + sg * g.d[AA] / (2.0 * par.c * par.eps_))
    tb = 1.0 / (1.0 + sg * g.d[BB] / (2.0 * par.c * par.eps_))
    E[sel] = 0.25 * e / par.eps_ + hc * ta * (0.5 * bbp - 0.5 * bbm) - hc * tb * (0.5 * bap - 0.5 * bam)
    H[sel] = 0.25 * h / par.mu - hc * ta * (0.5 * dbp - 0.5 * dbm) + hc * tb * (0.5 * dap - 0.5 * dam)
    return E, H


def update(s, sigma, E, H, g: Geom, par: Params, dt):
    cx, cy, cz = dt / g.d[0], dt / g.d[1], dt / g.d[2]
    gh = g.gh
    nx, ny, nz = g.n
    K, J, I = slice(gh, gh + nz), slice(gh, gh + ny), slice(gh, gh + nx)
    I1, J1, K1 = slice(gh, gh + nx + 1), slice(gh, gh + ny + 1), slice(gh, gh + nz + 1)
    ex, ey, ez = E
    hx, hy, hz = H
    ie = 1.0 / par.eps_

    def up(sl_, d, k=1):
        t = list(sl_)
        a = _ax(d)
        t[a] = slice(t[a].start + k, t[a].stop + k)
        return tuple(t)

    def dstep(q, sl_, d, curl):
        e_, p_ = decay(0.5 * (sigma[sl_] + sigma[up(sl_, d, -1)]) * ie * dt)
        s[q][sl_] = e_ * s[q][sl_] + p_ * curl
    sx = (K, J, I1)
    s[3][sx] = s[3][sx] - (cy * (ez[up(sx, 1)] - ez[sx]) - cz * (ey[up(sx, 2)] - ey[sx]))
    dstep(0, sx, 0, cy * (hz[up(sx, 1)] - hz[sx]) - cz * (hy[up(sx, 2)] - hy[sx]))
    sy = (K, J1, I)
    s[4][sy] = s[4][sy] - (cz * (ex[up(sy, 2)] - ex[sy]) - cx * (ez[up(sy, 0)] - ez[sy]))
    dstep(1, sy, 1, cz * (hx[up(sy, 2)] - hx[sy]) - cx * (hz[up(sy, 0)] - hz[sy]))
    sz = (K1, J, I)
    s[5][sz] = s[5][sz] - (cx * (ey[up(sz, 0)] - ey[sz]) - cy * (ex[up(sz, 1)] - ex[sz]))
    dstep(2, sz, 2, cx * (hy[up(sz, 0)] - hy[sz]) - cy * (hx[up(sz, 1)] - hx[sz]))
    return s


def cfl_dt(g: Geom, par: Params, cfl):
    c = par.c
    return cfl / (c / g.d[0] + c / g.d[1] + c / g.d[2])


def max_div(s, g: Geom):
    gh = g.gh
    nx, ny, nz = g.n
    K, J, I = slice(gh, gh + nz), slice(gh, gh + ny), slice(gh, gh + nx)
    out = []
    for base in (3, 0):
        dv = ((s[base][K, J, slice(gh + 1, gh + nx + 1)] - s[base][K, J, I]) / g.d[0] +
              (s[base + 1][K, slice(gh + 1, gh + ny + 1), I] - s[base + 1][K, J, I]) / g.d[1] +
              (s[base + 2][slice(gh + 1, gh + nz + 1), J, I] - s[base + 2][K, J, I]) / g.d[2])
        out.append(float(np.max(np.abs(dv)) * min(g.d)))
    return tuple(out)  # (div B, div D)


def energy(s, g: Geom, par: Params):
    """0.5 (E.D + H.B) summed over the face samples of the active zones (x zone volume)"""
    gh = g.gh
    act = (slice(gh, gh + g.n[2]), slice(gh, gh + g.n[1]), slice(gh, gh + g.n[0]))
    e = sum((s[q][act] ** 2).sum() for q in range(3)) / par.eps_ + \
        sum((s[q][act] ** 2).sum() for q in range(3, 6)) / par.mu
    return 0.5 * e * g.d[0] * g.d[1] * g.d[2]


def step(s, sigma, g: Geom, par: Params, dt):
    fill_ghosts(s, None, g, par.bc)
    m = predict(s, sigma, g, par, dt)
    EH = [edges(m, g, par, C, sigma) for C in range(3)]
    update(s, sigma, [x[0] for x in EH], [x[1] for x in EH], g, par, dt)


def run_steps(s, sigma, g: Geom, par: Params, dt, nsteps, t_final=0.0):
    t = 0.0
    d = min(dt, t_final) if t_final > 0.0 else dt
    n = 0
    for _ in range(nsteps):
        step(s, sigma, g, par, d)
        n += 1
        t = t + d
        if t_final > 0.0:
            rem = t_final - t
            if rem <= 1e-12 * t_final:
                break
            d = rem if dt >= rem else dt
    return t, n
