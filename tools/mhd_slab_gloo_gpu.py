"""W MHD slab ranks on ONE GPU (gloo, host-staged halos): the 8-array z exchange including the
shared z-face plane, on device state, must reproduce the single-domain MHD stepper bit for bit
(3D random field: every array varies in z). torchrun --nproc-per-node W tools/mhd_slab_gloo_gpu.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import mhd, mhd_slabs  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    n, order, steps = 16, 3, 3
    nzg = n * world
    gfull = mhd.make_geometry(n, n, nzg, order, (0, 0, 0), (1, 1, nzg / n))
    full = mhd.random_field(gfull, order, seed=5)
    for overlap in (True, False):
        check(n, order, steps, nzg, gfull, full, rank, world, overlap)
    dist.destroy_process_group()


def check(n, order, steps, nzg, gfull, full, rank, world, overlap):
    dom = mhd_slabs.MhdSlabDomain(n, n, nzg, order, rank=rank, world=world, device=0)
    gh = dom.geom.ghost
    dom.st.upload(np.ascontiguousarray(full[:, dom.z0:dom.z1 + 2 * gh + 1]))
    dt0 = dom.initial_dt(0.4)
    dom.st.set_time(0.0, dt0, 0.4)
    for _ in range(steps):
        dom.step(overlap=overlap)
    torch.cuda.synchronize()
    mine = np.ascontiguousarray(dom.st.download()[:, gh:gh + dom.nloc])
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        st = mhd.MhdStepper(gfull, mhd.make_params(order))
        st.upload(full)
        assert st.cfl_dt(0.4) == dt0
        st.set_time(0.0, dt0, 0.4)
        st.step(steps)
        ref = st.download()[:, gh:gh + nzg]
        got = np.concatenate(parts, axis=1)
        a = got[:, :, gh:gh + n, gh:gh + n]
        b = ref[:, :, gh:gh + n, gh:gh + n]
        same = bool((a.view(np.uint64) == b.view(np.uint64)).all())
        print(f"mhd world {world} overlap {overlap}: decomposed == single domain: {same}")
        assert same
    dom.close()


if __name__ == "__main__":
    main()
