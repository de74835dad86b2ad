"""Multi-process (gloo, CPU) tests of the z-slab decomposition's host logic: the halo exchange
of paper_2211_13295_b200.slabs and the global dt min, driving the C restatement (oracle/) as
the per-slab compute. World sizes 2 and 4 must reproduce the single-domain run bit for bit
(the reference's decomposition-transparency property, test_transfer.cpp:151-188)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_2211_13295_b200 import slabs


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab_geom(nx, nloc, z0, order, d):
    g = po.Geom()
    g.nx, g.ny, g.nz, g.ghost = nx, nx, nloc, {2: 2, 3: 3}[order]
    g.dx = g.dy = g.dz = d
    g.origin[0], g.origin[1], g.origin[2] = -5.0, -5.0, -5.0 + z0 * d
    return g


def _worker(rank, world, port, order, bc, steps, nx, nzg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        orc = po.Oracle()
        d = 10.0 / nx
        z0, z1 = slabs.slab_range(nzg, rank, world)
        nloc = z1 - z0
        g = slab_geom(nx, nloc, z0, order, d)
        gglob = slab_geom(nx, nzg, 0, order, d)
        full = _full_state(orc, gglob, order, bc)
        gh = g.ghost
        s = np.ascontiguousarray(full[z0:z1 + 2 * gh])  # slab + its ghost planes (refilled)
        cfl = 0.6 if order == 2 else 0.4
        dt_l = orc.initial_dt(g, s, cfl)
        t = torch.tensor([dt_l], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt = float(t.item())
        par = po.make_params(order)
        modal = po.zeros_modal(g, order)
        f = po.zeros_faces(g)
        r = po.zeros_rate(g)
        dts = [dt]
        for _ in range(steps):
            orc.apply_boundary_skinny(g, bc, s)  # x/y passes (+ a local z fill, replaced)
            planes = torch.from_numpy(s.reshape(s.shape[0], -1))
            slabs.exchange_z_halos(planes, gh, nloc, rank, world, bc == po.PERIODIC)
            dn = orc.ader_step(g, par, modal, s, *f, r, dt, cfl)
            t = torch.tensor([dn], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            dt = float(t.item())
            dts.append(dt)
        q.put((rank, s[gh:gh + nloc].copy(), dts))
    finally:
        dist.destroy_process_group()


def run_slabs(world, order, bc, steps, nx=8, nzg=16):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, order, bc, steps, nx, nzg, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    return np.concatenate([x[1] for x in res], axis=0), res[0][2], [x[2] for x in res]


def _full_state(orc, g, order, bc):
    """the problem's IC with a smooth z-dependent density/energy modulation: the vortex and
    Sod are z-invariant, so without it a swapped z halo would go unnoticed"""
    s = orc.init_sod(g) if bc == po.OUTFLOW else orc.init_isentropic_vortex(g, order)
    z = np.arange(s.shape[0], dtype=float)
    mod = 1.0 + 0.05 * np.sin(0.7 * z + 0.3) + 0.02 * np.cos(1.9 * z)
    s[..., 0] *= mod[:, None, None]
    s[..., 4] *= mod[:, None, None]
    return s


def run_single(order, bc, steps, nx=8, nzg=16):
    orc = po.Oracle()
    d = 10.0 / nx
    g = slab_geom(nx, nzg, 0, order, d)
    s = _full_state(orc, g, order, bc)
    cfl = 0.6 if order == 2 else 0.4
    dts = orc.run_steps(g, po.make_params(order), bc, cfl, steps, s, orc.initial_dt(g, s, cfl))
    gh = g.ghost
    return s[gh:gh + nzg], list(dts)


def test_slab_bookkeeping():
    assert slabs.slab_range(16, 1, 2) == (8, 16)
    with pytest.raises(ValueError):
        slabs.slab_range(15, 0, 2)
    assert slabs.neighbours(0, 4, True) == (3, 1)
    assert slabs.neighbours(0, 4, False) == (None, 1)
    assert slabs.neighbours(3, 4, False) == (2, None)


def test_single_rank_exchange_is_the_local_wrap():
    """world 1: the exchange equals the periodic/outflow z pass of apply_boundary."""
    orc = po.Oracle()
    g = slab_geom(6, 6, 0, 2, 10 / 6)
    rng = np.random.default_rng(3)
    for bc in (po.PERIODIC, po.OUTFLOW):
        s = rng.uniform(1, 2, (g.mz, g.my, g.mx, 5))
        ref = s.copy()
        orc.apply_boundary_skinny(g, bc, ref)
        orc.apply_boundary_skinny(g, bc, s)
        s[:g.ghost] = 0
        s[-g.ghost:] = 0
        slabs.exchange_z_halos(torch.from_numpy(s.reshape(g.mz, -1)), g.ghost, g.nz, 0, 1,
                               bc == po.PERIODIC)
        assert (s == ref).all()


@pytest.mark.parametrize("world,order,bc", [(2, 2, po.PERIODIC), (2, 3, po.PERIODIC),
                                            (4, 2, po.OUTFLOW)])
def test_decomposed_run_is_bit_identical(world, order, bc):
    steps = 4
    got, dts, all_dts = run_slabs(world, order, bc, steps)
    want, dts_ref = run_single(order, bc, steps)
    assert (got.view(np.uint64) == want.view(np.uint64)).all()
    assert dts == dts_ref
    assert all(d == dts for d in all_dts)
