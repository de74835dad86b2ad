"""The N > 1 communication path over NCCL on the one GPU of this pool: a single rank whose z
halos go through NCCL send/recv to itself and whose dt_next goes through an NCCL all-reduce
(SlabDomain.collectives / MhdSlabDomain.collectives), overlapped with the interior compute,
must reproduce the periodic single-domain steppers bit for bit.
Run: python tools/nccl_self_gpu.py (sets up a world-1 NCCL process group on 127.0.0.1)."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import hydro, mhd, mhd_slabs, slabs  # noqa: E402


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def euler(n=24, order=3, steps=4):
    dom = slabs.SlabDomain(n, n, n, order, world=1, overlap=True)
    dom.collectives = True
    s0 = dom.initial_state()
    from tests.zmod import modulate_z
    modulate_z(s0)
    dom.upload(s0)
    dt0 = dom.initial_dt(s0, 0.4)
    dom.set_time(0.0, dt0, 0.4)
    for _ in range(steps):
        dom.step()
    torch.cuda.synchronize()
    a = dom.download()
    st = hydro.Stepper(dom.geom, dom.params, bc=(0, 0, 0))
    st.upload(s0)
    st.set_time(0.0, dt0, 0.4)
    st.step(steps)
    b = st.download()
    gh = dom.geom.ghost
    act = np.s_[gh:gh + n, gh:gh + n, gh:gh + n]
    same = bool((a[act].view(np.uint64) == b[act].view(np.uint64)).all())
    print(f"euler nccl-self overlap: decomposed == single domain: {same}")
    return same


def mhd_case(n=16, order=3, steps=3):
    dom = mhd_slabs.MhdSlabDomain(n, n, n, order)
    dom.collectives = True
    g = dom.geom
    s0 = mhd.random_field(g, order, seed=3)
    dom.st.upload(s0)
    dt0 = dom.initial_dt(0.4)
    dom.st.set_time(0.0, dt0, 0.4)
    for _ in range(steps):
        dom.step(overlap=True)
    torch.cuda.synchronize()
    a = dom.st.download()
    st = mhd.MhdStepper(g, mhd.make_params(order))
    st.upload(s0)
    st.set_time(0.0, dt0, 0.4)
    st.step(steps)
    b = st.download()
    gh = g.ghost
    act = np.s_[:, gh:gh + n, gh:gh + n, gh:gh + n]
    same = bool((a[act].view(np.uint64) == b[act].view(np.uint64)).all())
    print(f"mhd nccl-self overlap: decomposed == single domain: {same}")
    return same


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    ok = euler() and mhd_case()
    dist.destroy_process_group()
    assert ok


if __name__ == "__main__":
    main()
