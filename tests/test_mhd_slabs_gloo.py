"""Multi-process (gloo, CPU) tests of the MHD z-slab decomposition's host logic
(paper_2211_13295_b200.mhd_slabs): the 8-array halo exchange (cells and face fields, the shared
z-face plane included) and the global dt min, with the numpy restatement (oracle/mhd_oracle.py)
as the per-slab compute. World sizes 2 and 4 must reproduce the single-domain run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mhd_oracle as mo
from paper_2211_13295_b200 import mhd, mhd_slabs


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_geom(nx, nzg, order, z0, z1):
    """mo.Geom of the slab [z0, z1) with the spacings of mhd_slabs.slab_geometry (exactly 1/nx,
    not re-derived per slab)"""
    g = mhd_slabs.slab_geometry(nx, nx, nzg, order, z0, z1)
    G = mo.Geom(nx, nx, z1 - z0, order, (0, 0, g.origin[2]), (1, 1, z1 / nx))
    G.d = (g.dx, g.dy, g.dz)
    return G


def full_state(nx, nzg, order):
    g = mhd_slabs.slab_geometry(nx, nx, nzg, order, 0, nzg)
    return mhd.random_field(g, order, seed=11), oracle_geom(nx, nzg, order, 0, nzg)


def _worker(rank, world, port, order, steps, nx, nzg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        z0, z1 = mhd_slabs.slab_range(nzg, rank, world)
        nloc = z1 - z0
        full, G = full_state(nx, nzg, order)
        g = oracle_geom(nx, nzg, order, z0, z1)
        gh = g.gh
        s = np.ascontiguousarray(full[:, z0:z1 + 2 * gh + 1])
        par = mo.Params(order, bc=(0, 0, None))
        cfl = 0.4
        t = torch.tensor([mo.cfl_dt(s, g, par, cfl)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt = float(t.item())
        dts = [dt]
        for _ in range(steps):
            mo.fill_ghosts(s, g, par.bc)  # x/y
            planes = torch.from_numpy(s.reshape(mo.NM, s.shape[1], -1))
            mhd_slabs.exchange_z_halos(planes, gh, nloc, rank, world)
            t = torch.tensor([mo.compute(s, g, par, dt, cfl)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            dt = float(t.item())
            dts.append(dt)
        q.put((rank, s[:, gh:gh + nloc].copy(), dts))
    finally:
        dist.destroy_process_group()


def run_slabs(world, order, steps, nx=8, nzg=16):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, order, steps, nx, nzg, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    return np.concatenate([x[1] for x in res], axis=1), res[0][2], [x[2] for x in res]


def run_single(order, steps, nx=8, nzg=16):
    s, G = full_state(nx, nzg, order)
    par = mo.Params(order)
    cfl = 0.4
    dt = mo.cfl_dt(s, G, par, cfl)
    dts = [dt]
    for _ in range(steps):
        dt = mo.step(s, G, par, dt, cfl)
        dts.append(dt)
    return s[:, G.gh:G.gh + nzg], dts


def test_single_rank_exchange_is_the_periodic_fill():
    s, G = full_state(6, 8, 3)
    ref = s.copy()
    mo.fill_ghosts(ref, G, (0, 0, 0))
    mo.fill_ghosts(s, G, (0, 0, None))
    gh = G.gh
    s[:, :gh] = 0
    s[:, gh + 8:] = 0
    mhd_slabs.exchange_z_halos(torch.from_numpy(s.reshape(mo.NM, s.shape[1], -1)), gh, 8, 0, 1)
    assert (s == ref).all()


@pytest.mark.parametrize("world,order,nx,nzg", [(2, 2, 8, 16), (2, 3, 8, 16), (4, 2, 8, 16),
                                                 (3, 2, 6, 12), (3, 3, 6, 18)])
def test_decomposed_mhd_run_is_bit_identical(world, order, nx, nzg):
    """(world 3 on 6 x 6 x 12 and 6 x 6 x 18 meshes: spacings 1/6 are not powers of two -- every slab must
    still step with exactly the single domain's dz)"""
    steps = 3
    got, dts, all_dts = run_slabs(world, order, steps, nx=nx, nzg=nzg)
    want, dts_ref = run_single(order, steps, nx=nx, nzg=nzg)
    assert (got.view(np.uint64) == want.view(np.uint64)).all()
    assert dts == dts_ref
    assert all(d == dts for d in all_dts)
