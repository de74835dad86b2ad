"""Multi-rank z-slab run on ONE GPU: torchrun launches W ranks (gloo, halos staged through host
memory -- this pool has a single device, and NCCL refuses two ranks on one GPU), each with its
own device stepper, the overlapped step (interior planes during the exchange), the device dt
all-reduce. With a z-modulated initial state the gathered result must equal the single-domain
stepper bit for bit (tools/slab_gloo_gpu.py does the run and the comparison)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_slab_run_on_one_gpu(world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.join(ROOT, "tools", "slab_gloo_gpu.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    for ov in (True, False):
        assert f"world {world} overlap {ov}: decomposed == single domain: True" in r.stdout


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_mhd_slab_run_on_one_gpu(world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.join(ROOT, "tools", "mhd_slab_gloo_gpu.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    for ov in (True, False):
        assert f"mhd world {world} overlap {ov}: decomposed == single domain: True" in r.stdout


def test_nccl_self_exchange_on_one_gpu():
    """The NCCL code path itself: one rank whose halos go through NCCL send/recv to itself and
    whose dt_next goes through an NCCL all-reduce, overlapped with the interior planes, equals
    the single-domain steppers bit for bit (Euler and MHD; tools/nccl_self_gpu.py)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "nccl_self_gpu.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "euler nccl-self overlap: decomposed == single domain: True" in r.stdout
    assert "mhd nccl-self overlap: decomposed == single domain: True" in r.stdout
