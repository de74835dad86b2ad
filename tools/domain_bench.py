"""One configs[4] slab (512^2 x 64 planes, O3, FMA build) stepped through the C-ABI multi-GPU
domain on one GPU -- the slab exchanging its z halos with itself (NCCL self send/recv, or peer
copies), sequential or overlapped with the interior planes, or the fused kernels storing the
boundary planes into the ghost planes themselves (store) -- against the plain stepper that
owns every boundary; then the same mesh as two 32-plane slabs on this GPU (peer copies vs
stores between two steppers). ms per step, CUDA-event timed.
Usage: python tools/domain_bench.py [n nz]"""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2211_13295_b200 import hydro  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nz = int(sys.argv[2]) if len(sys.argv) > 2 else 64
order, steps = 3, 20
api = hydro.HostApi()
g = hydro.make_geometry(n, n, nz, order, lo=(-5, -5, -5 * nz / n), hi=(5, 5, 5 * nz / n))
params = hydro.make_params(order)
s0 = api.init_isentropic_vortex(g, order)
dt0 = api.initial_dt(g, s0, 0.4)


def timed(step, sync):
    for _ in range(3):
        step()
    sync()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for _ in range(steps):
        step()
    sync()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps


res = {"mesh": [n, n, nz], "order": order, "build": "fma"}
st = hydro.Stepper(g, params, exact=False)
st.upload(s0)
st.set_time(0.0, dt0, 0.4)
res["stepper_ms"] = timed(lambda: st.step(1), st.sync)
st.close()
for name, tr, ov, devs in (("nccl", hydro.XCHG_NCCL, False, (0,)),
                           ("nccl_overlap", hydro.XCHG_NCCL, True, (0,)),
                           ("peer", hydro.XCHG_PEER, False, (0,)),
                           ("peer_overlap", hydro.XCHG_PEER, True, (0,)),
                           ("store", hydro.XCHG_STORE, False, (0,)),
                           ("two_slabs_peer", hydro.XCHG_PEER, False, (0, 0)),
                           ("two_slabs_store", hydro.XCHG_STORE, False, (0, 0))):
    d = hydro.Domain(g, params, exact=False, transport=tr, overlap=ov, devices=devs)
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.4)
    res[name + "_ms"] = timed(lambda: d.step(1), d.sync)
    d.close()
print(json.dumps(res))
