"""slabs -- z-slab decomposition of one mesh over the GPUs of a node (one process per GPU).

The reference decomposes the mesh into patches inside one process and fills their ghosts by
sequential x, y, z sweeps (transfer.cpp:87-150); its global dt is a host min over patches
(transfer.cpp:177-215). Here every rank owns a contiguous range of z planes of a
``nx x ny x nz_global`` mesh in one ``hydro.Stepper``:

  1. x/y ghosts of the rank's active planes are filled on the device (the x and y passes),
  2. the g z-ghost planes are exchanged with the two neighbouring ranks as whole (padded)
     planes -- the z pass copies full x/y planes, ghosts included, so this reproduces the
     reference's corner/edge contents exactly -- with one grouped NCCL send/recv per side,
  3. the fused step runs, its dt_next scalar is all-reduced (MIN, exact), then the device
     advances t/dt.

Steps 2-3 are the only collectives. Periodic wrap in z connects rank 0 and rank N-1; outflow
copies the edge plane locally. The exchange itself is written against torch tensors so the
same code runs over gloo on CPU tensors (tests/test_slabs_gloo.py) and NCCL on device memory.
"""
from __future__ import annotations

import numpy as np

from . import hydro

PERIODIC, OUTFLOW = hydro.PERIODIC, hydro.OUTFLOW


def slab_range(nz_global: int, rank: int, world: int):
    """Active z planes [z0, z1) of `rank` (even split, like make_patch_set's divisibility
    rule, transfer.cpp:19-22)."""
    if nz_global % world:
        raise ValueError("patch split must divide the mesh evenly")
    nloc = nz_global // world
    if nloc < 4:
        raise ValueError("patch must have at least 4 zones per axis")
    return rank * nloc, (rank + 1) * nloc


def neighbours(rank: int, world: int, periodic: bool):
    """(below, above) ranks in z; None where an outflow boundary ends the mesh."""
    below = (rank - 1) % world if (periodic or rank > 0) else None
    above = (rank + 1) % world if (periodic or rank < world - 1) else None
    return below, above


def exchange_z_halos(planes, gh: int, nloc: int, rank: int, world: int, periodic: bool,
                     group=None, p2p=False):
    """Fills the z-ghost planes of a slab in place.

    planes: torch tensor [nloc + 2 gh, plane_elems] (CPU or CUDA) = the slab's storage with
    one row per z plane. Sends the gh lowest active planes down and the gh highest up; the
    receiving side stores them as its top / bottom ghosts. Single rank + periodic is the local
    wrap; outflow ends copy the edge active plane (boundary.cpp:7-10 map_index). p2p: a single
    periodic rank exchanges with itself through the process group (NCCL send/recv to self --
    the N > 1 code path, runnable on one GPU)."""
    import torch
    import torch.distributed as dist

    below, above = neighbours(rank, world, periodic)
    lo_ghost = planes[0:gh]
    hi_ghost = planes[gh + nloc:gh + nloc + gh]
    lo_act = planes[gh:2 * gh]
    hi_act = planes[nloc:nloc + gh]
    if world == 1 and not p2p:
        if periodic:
            lo_ghost.copy_(hi_act)
            hi_ghost.copy_(lo_act)
    else:
        # Message matching is in posting order per peer pair, and at world 2 (periodic) the
        # neighbour below IS the neighbour above: post "send down, receive from above, send
        # up, receive from below" on every rank so the k-th send to a peer always meets that
        # peer's k-th receive (lowest active planes -> its top ghosts, then highest -> its
        # bottom ghosts).
        # The ghost ranges are whole contiguous planes of [z][y][x][5]: NCCL receives straight
        # into them and sends straight from the active planes (no packing, no temporaries).
        ops = []
        bufs = []
        staged = planes.is_cuda and dist.get_backend(group) == "gloo"
        rb = lo_ghost if below is not None else None
        ra = hi_ghost if above is not None else None
        if below is not None:
            ops.append(dist.P2POp(dist.isend, lo_act, below, group))
        if above is not None:
            ops.append(dist.P2POp(dist.irecv, ra, above, group))
            ops.append(dist.P2POp(dist.isend, hi_act, above, group))
            bufs.append((hi_ghost, ra))
        if below is not None:
            ops.append(dist.P2POp(dist.irecv, rb, below, group))
            bufs.append((lo_ghost, rb))
        if staged:  # gloo moves host memory only (testing N>1 on one GPU): stage through it
            ops = [dist.P2POp(op.op, op.tensor.cpu() if op.op is dist.isend else
                              torch.empty(op.tensor.shape, dtype=op.tensor.dtype), op.peer,
                              op.group) for op in ops]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if staged:  # the received host copies land in the ghost planes
            recvs = iter([op.tensor for op in ops if op.op is dist.irecv])
            for dst, _ in bufs:
                dst.copy_(next(recvs))
    if not periodic:
        if below is None:
            lo_ghost.copy_(planes[gh:gh + 1].expand(gh, -1))
        if above is None:
            hi_ghost.copy_(planes[gh + nloc - 1:gh + nloc].expand(gh, -1))


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view stepper memory."""

    def __init__(self, ptr, shape, dtype="<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": dtype,
                                         "data": (ptr, False), "version": 3, "strides": None}


class SlabDomain:
    """One rank's slab of an ``nx x ny x nz_global`` mesh on [-5,5]^2 x [-5, -5 + nz*dz]."""

    def __init__(self, nx, ny, nz_global, order, rank=0, world=1, device=0, exact=True,
                 solver=hydro.HLL, bc=PERIODIC, dx=None, integrator=hydro.ADER, overlap=None,
                 dz=None):
        self.rank, self.world, self.order = rank, world, order
        # overlap: interior planes computed while the z halos are exchanged. Off by default:
        # splitting the fused launch into interior + two boundary ranges costs more than the
        # exchange it hides (512^2 x 64 slab of configs[4]: +13 % vs +0.2 % for the sequential
        # NCCL exchange, tools/nccl_self_bench.py; an NVLink exchange of 2 x 32 MB is ~2 %)
        overlap = False if overlap is None else overlap
        self.overlap = overlap
        self.periodic = bc == PERIODIC
        self.z0, self.z1 = slab_range(nz_global, rank, world)
        self.nloc = self.z1 - self.z0
        d = 10.0 / nx if dx is None else dx
        g = hydro.Geom()
        g.nx, g.ny, g.nz, g.ghost = nx, ny, self.nloc, hydro.ghost_for_order(order)
        g.dx = g.dy = g.dz = d
        if dz is not None:  # e.g. configs[0]: 128 x 128 x 4 on [-5, 5]^3 (dz = 2.5)
            g.dz = dz
        g.origin[0], g.origin[1], g.origin[2] = -5.0, -5.0, -5.0 + self.z0 * g.dz
        # the vortex is columnar (problems.cpp:11-38), so every slab samples the same
        # (x, y) profile as the single-GPU mesh
        self.geom = g
        self.params = hydro.make_params(order, solver)
        self.api = hydro.HostApi()
        # who fills the z ghosts is fixed here: the stepper itself only for a single rank that
        # never overlaps; otherwise every step exchanges them (whatever step()'s overlap says)
        self.owns_z = world == 1 and not overlap
        self.st = hydro.Stepper(g, self.params, bc=(bc, bc, bc if self.owns_z else None),
                                exact=exact, device=device, integrator=integrator)
        # every device op of the step (our kernels, NCCL, events) is ordered on one stream
        import torch
        self.stream = torch.cuda.Stream(device=device)
        self.comm = torch.cuda.Stream(device=device)  # halo exchange, overlapped
        self.st.set_stream(self.stream.cuda_stream)
        # route a single rank's halos and dt all-reduce through the process group too
        # (exercises the NCCL path on one GPU; tools/nccl_self_gpu.py)
        self.collectives = world > 1

    # ---- host side
    def host_shape(self):
        g = self.geom
        return (g.mz, g.my, g.mx, 5)

    def initial_state(self):
        return self.api.init_isentropic_vortex(self.geom, self.order)

    def initial_dt(self, skinny, cfl):
        d = self.api.initial_dt(self.geom, skinny, cfl)
        return self.allreduce_min_host(d)

    def upload(self, skinny):
        self.st.upload(skinny)

    def download(self, out=None):
        return self.st.download(out)

    def set_time(self, t, dt, cfl, t_final=-1.0):
        self.st.set_time(t, dt, cfl, t_final)

    # ---- collectives
    def allreduce_min_host(self, v):
        if self.world == 1:
            return v
        import torch
        import torch.distributed as dist
        with torch.cuda.stream(self.stream):
            t = torch.tensor([v], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def max_over_ranks(self, v):
        if self.world == 1:
            return v
        import torch
        import torch.distributed as dist
        with torch.cuda.stream(self.stream):
            t = torch.tensor([v], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def _planes(self):
        import torch
        st = self.st
        plane = st.my_pad * st.pitch
        arr = _CudaArray(st.state_ptr(), (st.mz, plane))
        return torch.as_tensor(arr, device="cuda")

    def _acc(self):
        import torch
        acc, _ = self.st.dt_ptrs()
        return torch.as_tensor(_CudaArray(acc, (1,)), device="cuda")

    # ---- one step
    def step(self, kernel_events=None, overlap=None):  # noqa: C901
        """One ADER step; kernel_events=(start, end) bracket the fused kernel.

        overlap (default: on for N>1): the interior planes [G, nloc-G), whose stencils never
        reach the z-ghost planes, are computed while the halo exchange runs on a second
        stream; the two boundary ranges follow once the halos have landed."""
        import torch
        s = self.stream
        if overlap is None:
            overlap = self.overlap
        if self.owns_z and kernel_events is None and not overlap:
            self.st.step(1)
            return
        G = self.order  # stencil halo R + 1 (R = 1 at order 2, 2 at order 3)
        # no all-reduce between the last stage and the advance: the stepper closes the step
        # itself (the seam pair folds the advance into its last CTA)
        local = not (self.world > 1 or self.collectives)
        advanced = False
        with torch.cuda.stream(s):
            for k in range(self.st.stages):  # 1 (ADER) or 2/3 RK stages
                self.st.fill_ghosts()
                if kernel_events is not None and k == 0:
                    kernel_events[0].record(s)
                if overlap and not self.owns_z and self.nloc > 2 * G:
                    ready = torch.cuda.Event()
                    ready.record(s)
                    self.comm.wait_event(ready)
                    with torch.cuda.stream(self.comm):
                        exchange_z_halos(self._planes(), self.geom.ghost, self.nloc, self.rank,
                                         self.world, self.periodic, p2p=self.collectives)
                        halos = torch.cuda.Event()
                        halos.record(self.comm)
                    self.st.compute_range(G, self.nloc - G, False)  # overlaps the exchange
                    s.wait_event(halos)
                    self.st.compute_range(0, G, False)
                    self.st.compute_range(self.nloc - G, self.nloc, True)
                else:
                    if not self.owns_z:
                        exchange_z_halos(self._planes(), self.geom.ghost, self.nloc,
                                         self.rank, self.world, self.periodic,
                                         p2p=self.collectives)
                    if local and k == self.st.stages - 1:
                        self.st.compute_step()
                        advanced = True
                    else:
                        self.st.compute()
            if kernel_events is not None:
                kernel_events[1].record(s)
            if self.world > 1 or self.collectives:
                import torch.distributed as dist
                dist.all_reduce(self._acc(), op=dist.ReduceOp.MIN)
            if not advanced:
                self.st.advance()

    def sync(self):
        return self.st.sync()

    @property
    def launches(self):
        return self.st.launches

    def close(self):
        self.st.close()
