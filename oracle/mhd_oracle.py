"""mhd_oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

numpy restatement of the ADER-CT ideal-MHD step of paper_2211_13295_b200/csrc/mhd.cu, with
the same expression shapes (IEEE +,-,*,/,sqrt, no contraction), so the CUDA kernels built
with --fmad=false must agree with it to the last bit.

PARITY UNPINNED. The reference is Euler-only: SPEC.md:8 scopes out MHD and SPEC.md:345 the
multidimensional Riemann solvers, and no MHD code, test or fixture exists under
/root/reference. This restatement is builder-authored, so agreement with it proves the CUDA
implementation does what this file says, not that the scheme is right; the scheme is checked
by self-consistency (tests/test_mhd_oracle.py): div B = 0 to round-off, conservation, and
the measured convergence order on the smooth MHD vortex (Balsara 2004).

The ADER structure follows the reference's Euler step (stepper.cpp:49-78): reconstruction
(MC at order 2, reconstruct.cpp:16-28; WENO3 at order 3, reconstruct.hpp:46-73, plus
unlimited central cross terms) of the 8 cell-centred variables (B from the face averages),
the per-zone ADER predictor (predictor.cpp:26-60, one Picard pass at order 3, with the MHD
flux), HLL face fluxes (riemann.hpp:55-86 structure, fast magnetosonic Davis speeds), edge
EMFs from the two-dimensional HLL Riemann solver (UCT-HLL, Londrillo & Del Zanna 2004),
the conservative update (corrector.cpp:72-125 association) and the CT update of the faces.

Layout: state[8][mz+1][my+1][mx+1]; vars 0..4 cell averages (rho, mx, my, mz, E), 5..7 the
face fields Bx, By, Bz on the LOW face of the zone with the same index.
"""
from __future__ import annotations

import numpy as np

PERIODIC, OUTFLOW = 0, 1
NM = 8


class Unphysical(RuntimeError):
    pass


class Geom:
    def __init__(self, nx, ny, nz, order, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
        self.n = (nx, ny, nz)
        self.gh = 2 if order == 2 else 4  # order 3: WENO radius 2 + ring + the B average
        self.order = order
        self.d = tuple((hi[a] - lo[a]) / self.n[a] for a in range(3))
        self.lo = tuple(lo)
        self.shape = (nz + 2 * self.gh + 1, ny + 2 * self.gh + 1, nx + 2 * self.gh + 1)


class Params:
    def __init__(self, order, gamma=5.0 / 3.0, cfac_rho=2.0, cfac_other=1.5, eps=1e-12,
                 w=(0.25, 0.5, 0.25), bc=(PERIODIC, PERIODIC, PERIODIC), face_solver=0):
        self.order, self.gamma, self.face_solver = order, gamma, face_solver
        self.cfac_rho, self.cfac_other, self.eps, self.w = cfac_rho, cfac_other, eps, w
        self.bc = bc


def _ax(d):
    """numpy axis of spatial axis d (arrays are [k][j][i])"""
    return 2 - d


def _shift(a, d, s):
    return np.roll(a, -s, axis=_ax(d))  # a[..., i + s] at index i


def smin(a, b):
    return np.where(b < a, b, a)


def smax(a, b):
    return np.where(a < b, b, a)


# ------------------------------------------------------------------------------ ghosts

def fill_ghosts(s, g: Geom, bc):
    """k_mhd_ghosts: every ghost takes its composed active image (cells [gh, gh+n); the normal
    axis of a face field [gh, gh+n] at outflow, [gh, gh+n) when periodic)."""
    R, Q, P = g.shape
    ext = (P, Q, R)
    for q in range(NM):
        idx = []
        for d in range(3):
            if bc[d] is None or bc[d] < 0:  # caller-filled (z halos of a slab)
                idx.append(np.arange(ext[d]))
                continue
            lo, hi = g.gh, g.gh + g.n[d]
            if q >= 5 and q - 5 == d and bc[d] == OUTFLOW:
                hi += 1
            c = np.arange(ext[d])
            if bc[d] == PERIODIC:
                m = lo + np.mod(c - lo, hi - lo)
            else:
                m = np.clip(c, lo, hi - 1)
            idx.append(m)
        s[q] = s[q][np.ix_(idx[2], idx[1], idx[0])]
    return s


# ----------------------------------------------------------------------------- physics

def prim(c, gamma, check=True):
    rho = c[0]
    if check and not np.all(rho > 0.0):
        raise Unphysical("non-positive density")
    with np.errstate(all="ignore"):
        inv = 1.0 / rho
        u = [c[1] * inv, c[2] * inv, c[3] * inv]
        b2 = c[5] * c[5] + c[6] * c[6] + c[7] * c[7]
        p = (gamma - 1.0) * (c[4] - 0.5 * (c[1] * u[0] + c[2] * u[1] + c[3] * u[2]) - 0.5 * b2)
    if check and not np.all(p > 0.0):
        raise Unphysical("non-positive pressure")
    return rho, u, p, b2, inv


def unphysical(c, gamma):
    """mask of states with rho <= 0 or p <= 0 (NaN counts as unphysical)"""
    rho, u, p, b2, inv = prim(c, gamma, check=False)
    return ~(rho > 0.0) | ~(p > 0.0)


def positive_or_average(u, w, sel_fn, gamma):
    """mhd.cu positive_or_average: states with rho <= 0 or p <= 0 take the zone's cell average
    (w: the 8 cell-centred arrays, sel_fn maps a box array to the states' zones)"""
    bad = unphysical(u, gamma)
    if not np.any(bad):
        return u
    return [np.where(bad, sel_fn(w[q]), u[q]) for q in range(NM)]


def fast_speed(c, pr, gamma, A):
    rho, u, p, b2, inv = pr
    a2 = gamma * p * inv
    bb = b2 * inv
    bn2 = c[5 + A] * c[5 + A] * inv
    s = a2 + bb
    disc = s * s - 4.0 * a2 * bn2
    disc = np.where(disc > 0.0, disc, 0.0)
    return np.sqrt(0.5 * (s + np.sqrt(disc)))


def mhd_flux(c, pr, A):
    rho, u, p, b2, inv = pr
    un = u[A]
    bn = c[5 + A]
    vb = u[0] * c[5] + u[1] * c[6] + u[2] * c[7]
    pt = p + 0.5 * b2
    f = [None] * NM
    f[0] = c[0] * un
    for d in range(3):
        f[1 + d] = c[1 + d] * un - bn * c[5 + d]
    f[1 + A] = f[1 + A] + pt
    f[4] = (c[4] + pt) * un - bn * vb
    for d in range(3):
        f[5 + d] = c[5 + d] * un - bn * u[d]
    return f


def mc_limiter(a, b, cfac):
    m = 0.5 * np.abs(a + b)
    c1 = cfac * np.abs(a)
    c2 = cfac * np.abs(b)
    m = np.where(c1 < m, c1, m)
    m = np.where(c2 < m, c2, m)
    return m * (np.copysign(0.5, a) + np.copysign(0.5, b))


def weno3(s0, s1, s2, s3, s4, par):
    d0, d1, d2, d3 = s1 - s0, s2 - s1, s3 - s2, s4 - s3
    ux_l = 0.5 * (3.0 * d1 - d0)
    uxx_l = 0.5 * (d1 - d0)
    ux_c = 0.5 * (d1 + d2)
    uxx_c = 0.5 * (d2 - d1)
    ux_r = 0.5 * (3.0 * d2 - d3)
    uxx_r = 0.5 * (d3 - d2)
    k2 = 13.0 / 3.0
    is_l = ux_l * ux_l + k2 * uxx_l * uxx_l
    is_c = ux_c * ux_c + k2 * uxx_c * uxx_c
    is_r = ux_r * ux_r + k2 * uxx_r * uxx_r
    el, ec, er = par.eps + is_l, par.eps + is_c, par.eps + is_r
    al = par.w[0] / (el * el)
    ac = par.w[1] / (ec * ec)
    ar = par.w[2] / (er * er)
    inv = 1.0 / (al + ac + ar)
    return ((al * ux_l + ac * ux_c + ar * ux_r) * inv,
            (al * uxx_l + ac * uxx_c + ar * uxx_r) * inv)


def extrap(m0, side, lin, quad, o3):
    v = m0 + side * 0.5 * lin
    if o3:
        v = v + (1.0 / 6.0) * quad
    return v


def cell_vars(s, o3=False):
    """cell-centred 8 variables; B = mean of the face pair (order 2) or, at order 3, the
    fourth-order cell average 1/2 (b[-1/2] + b[+1/2]) - 1/24 (b[+3/2] - b[+1/2] - b[-1/2] +
    b[-3/2]) (the trapezoid's h^2/8 f'' error reduced to the average's h^2/24 f'').
    Indices whose stencil leaves the box are junk."""
    w = [s[q] for q in range(5)]
    for d in range(3):
        b0, b1 = s[5 + d], _shift(s[5 + d], d, 1)
        c = 0.5 * (b0 + b1)
        if o3:
            bm, b2 = _shift(s[5 + d], d, -1), _shift(s[5 + d], d, 2)
            c = c - (1.0 / 24.0) * (((b2 - b1) - b0) + bm)
        w.append(c)
    return w


def divergence(face, h, idd, gamma, bad):
    """predictor.cpp:12-22 with the MHD flux; `bad` accumulates zones with an unphysical
    face state (those zones' tau is zeroed by the caller, as mhd.cu does)"""
    div = None
    for A in range(3):
        a = [face[2 * A][q] + h[q] if h is not None else face[2 * A][q] for q in range(NM)]
        b = [face[2 * A + 1][q] + h[q] if h is not None else face[2 * A + 1][q]
             for q in range(NM)]
        bad |= unphysical(a, gamma) | unphysical(b, gamma)
        with np.errstate(all="ignore"):
            fa = mhd_flux(a, prim(a, gamma, check=False), A)
            fb = mhd_flux(b, prim(b, gamma, check=False), A)
        if A == 0:
            div = [(fa[q] - fb[q]) * idd[0] for q in range(NM)]
        else:
            div = [div[q] + (fa[q] - fb[q]) * idd[A] for q in range(NM)]
    return div


# ------------------------------------------------------------------------------- step

class Modes:
    pass


def predict(s, g: Geom, par: Params, dt):
    """k_mhd_predict on the ring (active -1..n): returns modes dict over the whole box (only
    ring entries are meaningful)."""
    o3 = par.order == 3
    w = cell_vars(s, o3)
    R, Q, P = g.shape
    ring = tuple(slice(g.gh - 1, g.gh + g.n[2 - ax] + 1) for ax in range(3))  # [k][j][i]

    def sh(arr, dd):  # arr shifted by the offset vector dd (per spatial axis)
        out = arr
        for d in range(3):
            if dd[d]:
                out = _shift(out, d, dd[d])
        return out[ring]

    face = [[None] * NM for _ in range(6)]
    lin = [[None] * NM for _ in range(3)]
    quad = [[None] * NM for _ in range(3)]
    cross = [[None] * NM for _ in range(3)]
    u0 = [None] * NM
    for q in range(NM):
        c0 = w[q][ring]
        u0[q] = c0
        for d in range(3):
            e = [0, 0, 0]
            e[d] = 1
            up = sh(w[q], e)
            um = sh(w[q], [-x for x in e])
            if not o3:
                cf = par.cfac_rho if q == 0 else par.cfac_other
                lin[d][q] = mc_limiter(up - c0, c0 - um, cf)
                quad[d][q] = 0.0
            else:
                upp = sh(w[q], [2 * x for x in e])
                umm = sh(w[q], [-2 * x for x in e])
                lin[d][q], quad[d][q] = weno3(umm, um, c0, up, upp, par)
        for d in range(3):
            face[2 * d][q] = extrap(c0, +1.0, lin[d][q], quad[d][q], o3)
            face[2 * d + 1][q] = extrap(c0, -1.0, lin[d][q], quad[d][q], o3)
        if o3:
            for d in range(3):
                da = [0, 0, 0]
                db = [0, 0, 0]
                da[d] = 1
                db[(d + 1) % 3] = 1
                pp = sh(w[q], [da[x] + db[x] for x in range(3)])
                pm = sh(w[q], [da[x] - db[x] for x in range(3)])
                mp = sh(w[q], [-da[x] + db[x] for x in range(3)])
                mm = sh(w[q], [-da[x] - db[x] for x in range(3)])
                cross[d][q] = 0.25 * ((pp - pm) - (mp - mm))
    idd = [1.0 / g.d[0], 1.0 / g.d[1], 1.0 / g.d[2]]
    bad = np.zeros(u0[0].shape, dtype=bool)
    with np.errstate(all="ignore"):
        div = divergence(face, None, idd, par.gamma, bad)
        tau = [(-dt) * div[q] for q in range(NM)]
        if o3:
            h = [0.5 * tau[q] for q in range(NM)]
            div = divergence(face, h, idd, par.gamma, bad)
            tau = [(-dt) * div[q] for q in range(NM)]
    # mhd.cu: an unphysical predictor state zeroes the zone's tau (first order in time)
    tau = [np.where(bad, 0.0, tau[q]) for q in range(NM)]

    def box(v):
        out = np.zeros((R, Q, P))
        out[ring] = v
        return out

    # the 18 solver states of mhd.cu (spatial part; the half-time state adds ht = tau/2):
    # faces s = 2A (+A), 2A+1 (-A); edge midpoints s = 6 + 4C + 2 lb + la at
    # (xa, xb) = (la ? -1/2 : +1/2, lb ? -1/2 : +1/2) in the (C+1, C+2) plane
    m = Modes()
    # cell averages with B = mean of the zone's face pair: the consumers' positivity fallback
    m.w = cell_vars(s, False)
    m.ht = [box(0.5 * tau[q]) for q in range(NM)]
    m.st = [[None] * NM for _ in range(18)]
    for q in range(NM):
        for d in range(3):
            m.st[2 * d][q] = box(face[2 * d][q])
            m.st[2 * d + 1][q] = box(face[2 * d + 1][q])
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
                    m.st[6 + 4 * C + 2 * lb + la][q] = box(v)
    return m


def _hlld_star(u, q, s, d, sm, pts, pt, bn, A):
    """mhd.cu hlld_star: the star state of one side (rho, v[3], b[3], e)"""
    T1, T2 = (A + 1) % 3, (A + 2) % 3
    rho = d / (s - sm)
    den = d * (s - sm) - bn * bn
    degen = np.abs(den) < 1e-8 * pts
    iden = 1.0 / den
    fv = bn * (sm - q[1][A]) * iden
    fb = (d * (s - q[1][A]) - bn * bn) * iden
    v, b = [None] * 3, [None] * 3
    v[A], b[A] = sm, bn
    for T in (T1, T2):
        v[T] = np.where(degen, q[1][T], q[1][T] - u[5 + T] * fv)
        b[T] = np.where(degen, u[5 + T], u[5 + T] * fb)
    vb = q[1][0] * u[5] + q[1][1] * u[6] + q[1][2] * u[7]
    vbs = v[0] * b[0] + v[1] * b[1] + v[2] * b[2]
    e = ((s - q[1][A]) * u[4] - pt * q[1][A] + pts * sm + bn * (vb - vbs)) / (s - sm)
    return rho, v, b, e


def hlld(ul, ur, ql, qr, cl, cr, A):
    """mhd.cu mhd_hlld<A> (Miyoshi & Kusano 2005), vectorised over faces: fluid fluxes"""
    T1, T2 = (A + 1) % 3, (A + 2) % 3
    with np.errstate(divide="ignore", invalid="ignore"):
        bn = ul[5 + A]
        cm = smax(cl, cr)
        sl = smin(ql[1][A], qr[1][A]) - cm
        sr = smax(ql[1][A], qr[1][A]) + cm
        fl, fr = mhd_flux(ul, ql, A), mhd_flux(ur, qr, A)
        ptl = ql[2] + 0.5 * ql[3]
        ptr = qr[2] + 0.5 * qr[3]
        dl = (sl - ql[1][A]) * ul[0]
        dr = (sr - qr[1][A]) * ur[0]
        idn = 1.0 / (dr - dl)
        sm = (dr * qr[1][A] - dl * ql[1][A] - ptr + ptl) * idn
        pts = (dr * ptl - dl * ptr + dl * dr * (qr[1][A] - ql[1][A])) * idn
        L = _hlld_star(ul, ql, sl, dl, sm, pts, ptl, bn, A)
        R = _hlld_star(ur, qr, sr, dr, sm, pts, ptr, bn, A)
        rl, rr = np.sqrt(L[0]), np.sqrt(R[0])
        sal = sm - np.abs(bn) / rl
        sar = sm + np.abs(bn) / rr
        left = sm >= 0.0

        def pick(a, b):
            return np.where(left, a, b)
        Srho, Se = pick(L[0], R[0]), pick(L[3], R[3])
        Sv = [pick(L[1][d], R[1][d]) for d in range(3)]
        Sb = [pick(L[2][d], R[2][d]) for d in range(3)]
        u = [pick(ul[q], ur[q]) for q in range(5)]
        f = [pick(fl[q], fr[q]) for q in range(5)]
        s = pick(sl, sr)
        fs = [None] * 5
        fs[0] = f[0] + s * (Srho - u[0])
        for d in range(3):
            fs[1 + d] = f[1 + d] + s * (Srho * Sv[d] - u[1 + d])
        fs[4] = f[4] + s * (Se - u[4])
        # double-star states
        degen = 0.5 * bn * bn < 1e-8 * pts
        sg = np.where(bn > 0.0, 1.0, -1.0)
        inv = 1.0 / (rl + rr)
        u2, b2 = [None] * 3, [None] * 3
        u2[A], b2[A] = sm, bn
        for T in (T1, T2):
            u2[T] = (rl * L[1][T] + rr * R[1][T] + (R[2][T] - L[2][T]) * sg) * inv
            b2[T] = (rl * R[2][T] + rr * L[2][T] + rl * rr * (R[1][T] - L[1][T]) * sg) * inv
        vb2 = u2[0] * b2[0] + u2[1] * b2[1] + u2[2] * b2[2]
        vbs = Sv[0] * Sb[0] + Sv[1] * Sb[1] + Sv[2] * Sb[2]
        e2 = np.where(left, Se - rl * (vbs - vb2) * sg, Se + rr * (vbs - vb2) * sg)
        u2 = [np.where(degen, Sv[d], u2[d]) for d in range(3)]
        e2 = np.where(degen, Se, e2)
        sa = pick(sal, sar)
        dstar = (left & (sal <= 0.0)) | (~left & (sar >= 0.0))
        for d in range(3):
            fs[1 + d] = np.where(dstar, fs[1 + d] + sa * (Srho * u2[d] - Srho * Sv[d]), fs[1 + d])
        fs[4] = np.where(dstar, fs[4] + sa * (e2 - Se), fs[4])
        return [np.where(sl >= 0.0, fl[q], np.where(sr <= 0.0, fr[q], fs[q])) for q in range(5)]


def face_fluxes(m, g: Geom, par: Params, A):
    """k_mhd_flux<A>: fluid fluxes of the A faces, stored at the zone right of the face;
    valid at faces 0..n_A, active transverse."""
    ul = [_shift(m.st[2 * A][q], A, -1) + _shift(m.ht[q], A, -1) for q in range(NM)]
    ur = [m.st[2 * A + 1][q] + m.ht[q] for q in range(NM)]
    ul = positive_or_average(ul, m.w, lambda x: _shift(x, A, -1), par.gamma)
    ur = positive_or_average(ur, m.w, lambda x: x, par.gamma)
    bn = 0.5 * (ul[5 + A] + ur[5 + A])
    ul[4] = ul[4] + 0.5 * (bn * bn - ul[5 + A] * ul[5 + A])
    ur[4] = ur[4] + 0.5 * (bn * bn - ur[5 + A] * ur[5 + A])
    ul[5 + A] = bn
    ur[5 + A] = bn
    sel = [slice(None)] * 3
    for d in range(3):
        hi = g.gh + g.n[d] + (1 if d == A else 0)
        sel[_ax(d)] = slice(g.gh, hi)
    sel = tuple(sel)
    ul = [x[sel] for x in ul]
    ur = [x[sel] for x in ur]
    ql, qr = prim(ul, par.gamma), prim(ur, par.gamma)
    cl, cr = fast_speed(ul, ql, par.gamma, A), fast_speed(ur, qr, par.gamma, A)
    if par.face_solver == 1:
        out = np.zeros((5,) + g.shape)
        f5 = hlld(ul, ur, ql, qr, cl, cr, A)
        for q in range(5):
            out[q][sel] = f5[q]
        return out
    sl = smin(ql[1][A] - cl, qr[1][A] - cr)
    sr = smax(ql[1][A] + cl, qr[1][A] + cr)
    fl, fr = mhd_flux(ul, ql, A), mhd_flux(ur, qr, A)
    out = np.zeros((5,) + g.shape)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / (sr - sl)
        for q in range(5):
            mid = (sr * fl[q] - sl * fr[q] + sl * sr * (ur[q] - ul[q])) * inv
            out[q][sel] = np.where(sl >= 0.0, fl[q], np.where(sr <= 0.0, fr[q], mid))
    return out


def edge_emf(m, g: Geom, par: Params, C):
    """k_mhd_emf<C>: E_C on the C edges (a, b = C+1, C+2), stored at the zone whose low a and
    low b sides meet there; valid for a in 0..n_a, b in 0..n_b, C in 0..n_C-1."""
    AA, BB = (C + 1) % 3, (C + 2) % 3
    sel = [slice(None)] * 3
    for d in range(3):
        sel[_ax(d)] = slice(g.gh, g.gh + g.n[d] + (0 if d == C else 1))
    sel = tuple(sel)
    ec, ba, bb = {}, {}, {}
    apa = ama = apb = amb = 0.0
    for lb in range(2):
        for la in range(2):
            def z(arr):
                out = arr
                if la == 0:
                    out = _shift(out, AA, -1)
                if lb == 0:
                    out = _shift(out, BB, -1)
                return out[sel]
            u = [z(m.st[6 + 4 * C + 2 * lb + la][q]) + z(m.ht[q]) for q in range(NM)]
            u = positive_or_average(u, m.w, z, par.gamma)
            pr = prim(u, par.gamma)
            vel = pr[1]
            ec[la, lb] = vel[BB] * u[5 + AA] - vel[AA] * u[5 + BB]
            ba[la, lb] = u[5 + AA]
            bb[la, lb] = u[5 + BB]
            cfa = fast_speed(u, pr, par.gamma, AA)
            cfb = fast_speed(u, pr, par.gamma, BB)
            apa = smax(apa, vel[AA] + cfa)
            ama = smax(ama, cfa - vel[AA])
            apb = smax(apb, vel[BB] + cfb)
            amb = smax(amb, cfb - vel[BB])
    ia = 1.0 / (apa + ama)
    ib = 1.0 / (apb + amb)
    wa = (apa * ia, ama * ia)
    wb = (apb * ib, amb * ib)
    e = (wa[0] * wb[0] * ec[0, 0] + wa[1] * wb[0] * ec[1, 0] + wa[0] * wb[1] * ec[0, 1] +
         wa[1] * wb[1] * ec[1, 1])
    jb = 0.5 * (bb[1, 0] + bb[1, 1]) - 0.5 * (bb[0, 0] + bb[0, 1])
    ja = 0.5 * (ba[0, 1] + ba[1, 1]) - 0.5 * (ba[0, 0] + ba[1, 0])
    out = np.zeros(g.shape)
    out[sel] = e + apa * ama * ia * jb - apb * amb * ib * ja
    return out


def update(s, F, E, g: Geom, dt):
    cx, cy, cz = dt / g.d[0], dt / g.d[1], dt / g.d[2]
    gh = g.gh
    nx, ny, nz = g.n
    K, J, I = slice(gh, gh + nz), slice(gh, gh + ny), slice(gh, gh + nx)

    def sl(k, j, i):
        return (k, j, i)
    for q in range(5):
        fx, fy, fz = F[0][q], F[1][q], F[2][q]
        rr = (-cx * (fx[K, J, slice(gh + 1, gh + nx + 1)] - fx[K, J, I])
              - cy * (fy[K, slice(gh + 1, gh + ny + 1), I] - fy[K, J, I])
              - cz * (fz[slice(gh + 1, gh + nz + 1), J, I] - fz[K, J, I]))
        s[q][K, J, I] = s[q][K, J, I] + rr
    ex, ey, ez = E
    I1, J1, K1 = slice(gh, gh + nx + 1), slice(gh, gh + ny + 1), slice(gh, gh + nz + 1)

    def up(sl_, d):  # the same slice shifted by +1 along spatial axis d
        t = list(sl_)
        a = _ax(d)
        t[a] = slice(t[a].start + 1, t[a].stop + 1)
        return tuple(t)
    sx = (K, J, I1)
    s[5][sx] = s[5][sx] - (cy * (ez[up(sx, 1)] - ez[sx]) - cz * (ey[up(sx, 2)] - ey[sx]))
    sy = (K, J1, I)
    s[6][sy] = s[6][sy] - (cz * (ex[up(sy, 2)] - ex[sy]) - cx * (ez[up(sy, 0)] - ez[sy]))
    sz = (K1, J, I)
    s[7][sz] = s[7][sz] - (cx * (ey[up(sz, 0)] - ey[sz]) - cy * (ex[up(sz, 1)] - ex[sz]))
    return s


P_FLOOR = 1.0e-10  # mhd.cu P_FLOOR


def pressure_floor(s, g: Geom, par: Params):
    """mhd.cu zone_dt(floor=true): active zones whose pressure (B = mean of the zone's face
    pair) is <= P_FLOOR get E raised to p = P_FLOOR; returns how many"""
    w = cell_vars(s, False)
    gh = g.gh
    act = (slice(gh, gh + g.n[2]), slice(gh, gh + g.n[1]), slice(gh, gh + g.n[0]))
    u = [x[act] for x in w]
    rho, v, p, b2, inv = prim(u, par.gamma, check=False)
    bad = (rho > 0.0) & ~(p > P_FLOOR)
    if not np.any(bad):
        return 0
    e = (P_FLOOR / (par.gamma - 1.0) + 0.5 * (u[1] * v[0] + u[2] * v[1] + u[3] * v[2])
         + 0.5 * b2)
    s[4][act] = np.where(bad, e, s[4][act])
    return int(np.count_nonzero(bad))


def cfl_dt(s, g: Geom, par: Params, cfl):
    # each zone's own two faces (mean): no ghost face enters, so the estimate is the same
    # under any domain decomposition
    w = cell_vars(s, False)
    gh = g.gh
    act = (slice(gh, gh + g.n[2]), slice(gh, gh + g.n[1]), slice(gh, gh + g.n[0]))
    u = [x[act] for x in w]
    pr = prim(u, par.gamma)
    sx = np.abs(pr[1][0]) + fast_speed(u, pr, par.gamma, 0)
    sy = np.abs(pr[1][1]) + fast_speed(u, pr, par.gamma, 1)
    sz = np.abs(pr[1][2]) + fast_speed(u, pr, par.gamma, 2)
    return float(np.min(cfl / (sx / g.d[0] + sy / g.d[1] + sz / g.d[2])))


def max_divb(s, g: Geom):
    gh = g.gh
    nx, ny, nz = g.n
    K, J, I = slice(gh, gh + nz), slice(gh, gh + ny), slice(gh, gh + nx)
    dv = ((s[5][K, J, slice(gh + 1, gh + nx + 1)] - s[5][K, J, I]) / g.d[0] +
          (s[6][K, slice(gh + 1, gh + ny + 1), I] - s[6][K, J, I]) / g.d[1] +
          (s[7][slice(gh + 1, gh + nz + 1), J, I] - s[7][K, J, I]) / g.d[2])
    return float(np.max(np.abs(dv)) * min(g.d))


def step(s, g: Geom, par: Params, dt, cfl):
    """one ADER-CT step in place; returns dt_next (the CFL min of the new state)"""
    fill_ghosts(s, g, par.bc)
    return compute(s, g, par, dt, cfl)


def compute(s, g: Geom, par: Params, dt, cfl):
    """the step after the ghost fill (hc_mhd_compute): returns this domain's CFL min"""
    m = predict(s, g, par, dt)
    F = [face_fluxes(m, g, par, A) for A in range(3)]
    E = [edge_emf(m, g, par, C) for C in range(3)]
    update(s, F, E, g, dt)
    pressure_floor(s, g, par)
    return cfl_dt(s, g, par, cfl)


def run_steps(s, g: Geom, par: Params, cfl, nsteps, dt0, t_final=0.0):
    """harness.cpp:155-170 loop shape: returns the dt used by each step and the last dt_next"""
    dt, t, dts = dt0, 0.0, []
    for _ in range(nsteps):
        dn = step(s, g, par, dt, cfl)
        dts.append(dt)
        t = t + dt
        if t_final > 0.0:
            rem = t_final - t
            if rem <= 1e-12 * t_final:
                break
            if dn >= rem:
                dn = rem
        dt = dn
    return dts, dt, t
