"""Cost of the N > 1 step machinery on one GPU (256^3 O3 HLL, FMA build): the plain device
step vs the slab step with the overlapped z-halo exchange and the dt all-reduce going through
NCCL (a rank exchanging with itself: the copies are local, so this measures the split launches,
the NCCL calls and the stream synchronisation, not NVLink). CUDA-event timing, 20 steps.
Run: python tools/nccl_self_bench.py [n]"""
import json
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_13295_b200 import mhd, mhd_slabs, slabs  # noqa: E402


def run(n, collectives, overlap, steps=20, warmup=3, nz=None):
    dom = slabs.SlabDomain(n, n, nz or n, 3, world=1, exact=False, overlap=overlap)
    dom.collectives = collectives
    s0 = dom.initial_state()
    dom.upload(s0)
    dom.set_time(0.0, dom.initial_dt(s0, 0.4), 0.4)
    for _ in range(warmup):
        dom.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dom.stream)
    for _ in range(steps):
        dom.step()
    e1.record(dom.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    dom.close()
    return ms


def run_mhd(n, nz, collectives, overlap, steps=5, warmup=2):
    dom = mhd_slabs.MhdSlabDomain(n, n, nz, 3)
    dom.collectives = collectives
    dom.st.upload(mhd.orszag_tang(dom.geom, 3))
    dom.st.set_time(0.0, dom.initial_dt(0.4), 0.4)
    for _ in range(warmup):
        dom.step(overlap=overlap)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dom.stream)
    for _ in range(steps):
        dom.step(overlap=overlap)
    e1.record(dom.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    dom.close()
    return ms


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    nz = int(sys.argv[2]) if len(sys.argv) > 2 else n  # 512 64: one rank of configs[4] / 8
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        os.environ.setdefault("MASTER_PORT", str(s.getsockname()[1]))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    res = {"n": n, "nz": nz,
           "plain_step_ms": run(n, False, False, nz=nz),
           "overlapped_local_exchange_ms": run(n, False, True, nz=nz),
           "overlapped_nccl_self_ms": run(n, True, True, nz=nz),
           "sequential_nccl_self_ms": run(n, True, False, nz=nz)}
    if len(sys.argv) > 3:  # MHD slab of the same shape
        res["mhd_sequential_nccl_self_ms"] = run_mhd(n, nz, True, False)
        res["mhd_overlapped_nccl_self_ms"] = run_mhd(n, nz, True, True)
    print(json.dumps(res))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
