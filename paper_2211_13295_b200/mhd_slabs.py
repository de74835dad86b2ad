"""mhd_slabs -- z-slab decomposition of the MHD (CT) step over the GPUs of a node, one process
per GPU (BASELINE.json config 5: 512^3 MHD on 2/4/8 B200s).

Every rank owns nz_global / world contiguous z planes of a periodic nx x ny x nz_global mesh
in one ``mhd.MhdStepper`` with caller-filled z ghosts (params.bc[2] = -1). Per step:

  1. x/y ghosts of the slab on the device (hc_mhd_fill_ghosts),
  2. z halo exchange with the two neighbours: each of the 8 variable arrays (5 cell averages,
     3 face fields) sends its planes [gh, 2gh+1) down -- they are the lower rank's top ghost
     planes, the +1 being the shared z-face plane on top of that slab -- and its planes
     [nloc, nloc+gh) up -- the upper rank's bottom ghosts; whole padded planes (x/y ghosts
     included), one grouped NCCL send/recv per side,
  3. the step (hc_mhd_compute), the all-reduce (MIN) of the dt_next accumulator (exact), then
     the device t/dt hand-off (hc_mhd_advance).

step(overlap=True) overlaps the exchange (as slabs.py can for the Euler path): it runs on a
second stream while hc_mhd_compute_range prepares the interior planes [gh, nloc - gh - 1),
whose cell-B, predictor, face and edge stencils never reach a z-ghost plane or the shared top
face plane; the two boundary ranges follow once the halos have landed, then hc_mhd_finish
(update + CFL estimate) -- bit-identical to the sequential step, but measured slower than it
at the configs[4] slab size (the default is the sequential step).

The z-face plane shared by two slabs is updated by both ranks from identical inputs, so the
decomposed run is bit-identical to the single-domain run (tests/test_mhd_slabs_gloo.py runs
the exchange over gloo with the numpy restatement as the per-slab compute). Periodic z only.
"""
from __future__ import annotations

import numpy as np

from . import mhd


def slab_range(nz_global: int, rank: int, world: int):
    if nz_global % world:
        raise ValueError("patch split must divide the mesh evenly")
    nloc = nz_global // world
    if nloc < 4:
        raise ValueError("patch must have at least 4 zones per axis")
    return rank * nloc, (rank + 1) * nloc


def exchange_z_halos(planes, gh: int, nloc: int, rank: int, world: int, group=None, p2p=False):
    """planes: torch tensor [NVAR, nloc + 2 gh + 1, plane_elems] viewing the slab's state
    (CPU or CUDA). Fills the z ghosts of every variable from the periodic z neighbours."""
    import torch
    import torch.distributed as dist

    if nloc < gh + 1:  # the lower send (gh + 1 planes incl. the shared face) must be owned
        raise ValueError(f"slab of {nloc} planes is thinner than the {gh + 1}-plane halo")
    lo_send = planes[:, gh:2 * gh + 1]            # -> lower rank's [gh+nloc, 2gh+nloc+1)
    hi_send = planes[:, nloc:nloc + gh]           # -> upper rank's [0, gh)
    lo_ghost = planes[:, 0:gh]
    hi_ghost = planes[:, gh + nloc:2 * gh + nloc + 1]
    if world == 1 and not p2p:  # (p2p: through the process group, to itself)
        lo_ghost.copy_(hi_send.clone())
        hi_ghost.copy_(lo_send.clone())
        return
    below, above = (rank - 1) % world, (rank + 1) % world
    # gloo moves host memory only (multi-rank tests on one GPU): stage through it
    dev = "cpu" if planes.is_cuda and dist.get_backend(group) == "gloo" else planes.device
    rb = torch.empty(lo_ghost.shape, dtype=planes.dtype, device=dev)
    ra = torch.empty(hi_ghost.shape, dtype=planes.dtype, device=dev)
    # posting order "send down, receive from above, send up, receive from below" matches
    # sends and receives per peer even when below == above (world 2)
    ops = [dist.P2POp(dist.isend, lo_send.contiguous().to(dev), below, group),
           dist.P2POp(dist.irecv, ra, above, group),
           dist.P2POp(dist.isend, hi_send.contiguous().to(dev), above, group),
           dist.P2POp(dist.irecv, rb, below, group)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    lo_ghost.copy_(rb)
    hi_ghost.copy_(ra)


def slab_geometry(nx, ny, nz_global, order, z0, z1):
    """Geometry of the z-slab [z0, z1) of the nx x ny x nz_global mesh on [0,1] x [0, ny d] x
    [0, nz_global d], d = 1/nx: the spacings are set to d itself (not re-derived as
    (hi - lo)/n, which is an ulp off for some slabs when n is not a power of two), so every
    rank steps with the single domain's dx, dy, dz and the decomposition stays bit-transparent.
    slab_geometry(nx, ny, nz, order, 0, nz) is the matching single domain."""
    d = 1.0 / nx
    g = mhd.make_geometry(nx, ny, z1 - z0, order, (0.0, 0.0, z0 * d), (1.0, ny * d, z1 * d))
    g.dx = g.dy = g.dz = d
    g.origin[0], g.origin[1], g.origin[2] = 0.0, 0.0, z0 * d
    return g


class MhdSlabDomain:
    """One rank's slab of a periodic nx x ny x nz_global MHD mesh on [0,1]^2 x [0, nz dz]."""

    def __init__(self, nx, ny, nz_global, order, rank=0, world=1, device=0):
        import torch
        self.rank, self.world, self.order = rank, world, order
        self.z0, self.z1 = slab_range(nz_global, rank, world)
        self.nloc = self.z1 - self.z0
        g = slab_geometry(nx, ny, nz_global, order, self.z0, self.z1)
        self.geom = g
        self.st = mhd.MhdStepper(g, mhd.make_params(order, bc=(0, 0, -1), device=device))
        self.stream = torch.cuda.Stream(device=device)
        self.comm = torch.cuda.Stream(device=device)
        self.st.set_stream(self.stream.cuda_stream)
        # (off by default: the split front kernels cost ~5 % on a 512^2 x 64 slab, more than
        # the ~1.5 % an NVLink exchange of the halos takes; tools/nccl_self_bench.py)
        self.overlap = False
        self.collectives = world > 1  # True at N = 1: the NCCL path to itself (testing)

    def initial_state(self):
        return mhd.orszag_tang(self.geom, self.order)

    def _planes(self):
        import torch
        from .slabs import _CudaArray
        ptr, vs, pe = self.st.state_ptr()
        g = self.geom
        return torch.as_tensor(_CudaArray(ptr, (mhd.NM, g.mz + 1, pe)), device="cuda")

    def _acc(self):
        import torch
        from .slabs import _CudaArray
        return torch.as_tensor(_CudaArray(self.st.dt_acc_ptr(), (1,)), device="cuda")

    def initial_dt(self, cfl):
        dt = self.st.cfl_dt(cfl)
        if self.world > 1:
            import torch
            import torch.distributed as dist
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            dt = float(t.item())
        return dt

    def step(self, overlap=None):
        import torch
        if overlap is None:
            overlap = self.overlap
        gh, n = self.geom.ghost, self.nloc
        lo, hi = gh, n - gh - 1  # interior: no stencil reaches a z ghost or the top face
        with torch.cuda.stream(self.stream):
            self.st.fill_ghosts()
            if overlap and hi > lo:
                ready = torch.cuda.Event()
                ready.record(self.stream)
                self.comm.wait_event(ready)
                with torch.cuda.stream(self.comm):
                    exchange_z_halos(self._planes(), gh, n, self.rank, self.world,
                                     p2p=self.collectives)
                    halos = torch.cuda.Event()
                    halos.record(self.comm)
                self.st.compute_range(lo, hi)  # overlaps the exchange
                self.stream.wait_event(halos)
                self.st.compute_range(0, lo)
                self.st.compute_range(hi, n)
                self.st.finish()
            else:
                exchange_z_halos(self._planes(), gh, n, self.rank, self.world,
                                 p2p=self.collectives)
                self.st.compute()
            if self.world > 1 or self.collectives:
                import torch.distributed as dist
                dist.all_reduce(self._acc(), op=dist.ReduceOp.MIN)
            self.st.advance()

    def close(self):
        self.st.close()
