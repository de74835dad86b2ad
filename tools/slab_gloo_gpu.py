"""Two ranks on ONE GPU (gloo on CUDA tensors where the backend allows it): the z-slab driver
with real device memory -- x/y ghost fill, halo exchange overlapped with the interior-plane
fused launch, all-reduce of the device dt accumulator -- must reproduce the single-domain
stepper bit for bit. Run: torchrun --nproc-per-node 2 tools/slab_gloo_gpu.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import hydro, slabs  # noqa: E402


def modulate(s, k0):
    """z-dependent density/energy modulation of the (z-invariant) vortex, by GLOBAL storage
    plane index, so that a misplaced z halo cannot go unnoticed"""
    z = np.arange(s.shape[0], dtype=float) + k0
    m = 1.0 + 0.05 * np.sin(0.7 * z + 0.3) + 0.02 * np.cos(1.9 * z)
    s[..., 0] *= m[:, None, None]
    s[..., 4] *= m[:, None, None]
    return s


def main():
    dist.init_process_group(os.environ.get("HC_DIST_BACKEND", "gloo"))
    for overlap in (True, False):
        check(overlap)
    dist.destroy_process_group()


def check(overlap):
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    n, order, steps = 24, 3, 4
    dom = slabs.SlabDomain(n, n, n * world, order, rank=rank, world=world, device=0,
                           overlap=overlap)
    gh = dom.geom.ghost
    s0 = modulate(dom.initial_state(), dom.z0)  # local storage plane p = global z0 + p
    dt0 = dom.initial_dt(s0, 0.4)
    dom.upload(s0)
    dom.set_time(0.0, dt0, 0.4)
    for _ in range(steps):
        dom.step()
    torch.cuda.synchronize()
    out = dom.download()
    t = dom.sync()
    mine = np.ascontiguousarray(out[gh:gh + dom.nloc])
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        g = hydro.make_geometry(n, n, n * world, order, (-5, -5, -5), (5, 5, -5 + 10.0 * world))
        api = hydro.HostApi()
        s = modulate(api.init_isentropic_vortex(g, order), 0)
        st = hydro.Stepper(g, hydro.make_params(order))
        st.upload(s)
        st.set_time(0.0, api.initial_dt(g, s, 0.4), 0.4)
        st.step(steps)
        ref = st.download()[gh:gh + n * world]
        got = np.concatenate(parts, axis=0)
        same = bool((got[:, gh:gh + n, gh:gh + n].view(np.uint64) ==
                     ref[:, gh:gh + n, gh:gh + n].view(np.uint64)).all())
        print(f"world {world} overlap {overlap}: decomposed == single domain: {same}; "
              f"t {t[0]} vs {st.sync()[0]}")
        assert same
    dom.close()


if __name__ == "__main__":
    main()
