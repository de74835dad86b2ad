"""The multi-GPU z-slab domain behind the C ABI (csrc/domain.cu, hc_domain_*): the
reference's PatchSet split along z with run_patch_step's exchange and global dt min
(transfer.cpp:17-47, 87-150, 152-216) on NCCL / peer copies. This pool exposes one GPU, so the
decomposed path runs as one slab exchanging its periodic z halos with itself through the same
NCCL calls (send/recv + all-reduce) -- bit-identical to one stepper owning every boundary --
and the outflow ends as local edge-plane copies. tests/c/domain_selftest.c drives the same
ABI from plain C (no Python, no torch)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2211_13295_b200 import hydro
from tests.zmod import modulate_z

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single(g, params, s0, dt0, cfl, steps, exact, integ, bc):
    st = hydro.Stepper(g, params, bc=bc, exact=exact, integrator=integ)
    st.upload(s0)
    st.set_time(0.0, dt0, cfl)
    st.step(steps)
    t, dt, n = st.sync()
    out = st.download()
    kind = st.kernel_info()[0]
    st.close()
    return out, t, dt, n, kind


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("integ", [hydro.ADER, hydro.RK3])
@pytest.mark.parametrize("transport,overlap", [(hydro.XCHG_NCCL, False), (hydro.XCHG_PEER, False),
                                               (hydro.XCHG_NCCL, True), (hydro.XCHG_PEER, True),
                                               (hydro.XCHG_STORE, False)])
def test_domain_self_exchange_bitwise(exact, integ, transport, overlap):
    order, shape, steps = 3, (64, 14, 12), 4
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    params = hydro.make_params(order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    bc = (hydro.PERIODIC,) * 3
    want, t1, dt1, n1, kind = _single(g, params, s0, dt0, 0.4, steps, exact, integ, bc)
    d = hydro.Domain(g, params, bc=bc, exact=exact, integrator=integ, transport=transport,
                     overlap=overlap)
    assert d.nslabs == 1 and d.nz_local == shape[2] and d.kernel == kind
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.4)
    d.step(steps)
    t2, dt2, n2 = d.sync()
    out = want.copy()
    out[g.ghost:-g.ghost] = 0.0
    d.gather(out)
    d.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    assert (out[act].view(np.uint64) == want[act].view(np.uint64)).all()
    assert (t2, dt2, n2) == (t1, dt1, n1)


def test_domain_one_process_per_gpu_api():
    """hc_domain_create (rank 0 of world 1 with an NCCL unique id): the multi-process entry."""
    order, shape, steps = 2, (32, 12, 8), 3
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    params = hydro.make_params(order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.6)
    want, _, dt1, _, _ = _single(g, params, s0, dt0, 0.6, steps, True, hydro.ADER,
                                 (hydro.PERIODIC,) * 3)
    d = hydro.Domain(g, params, exact=True, rank=0, world=1, nccl_id=hydro.nccl_unique_id())
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.6)
    d.step(steps)
    _, dt2, _ = d.sync()
    out = want.copy()
    d.gather(out)
    d.close()
    assert (out.view(np.uint64) == want.view(np.uint64)).all() and dt1 == dt2


def test_domain_outflow_z():
    """Outflow z: the global ends repeat the edge plane (no exchange across them)."""
    order, shape, steps = 3, (32, 10, 9), 3
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    params = hydro.make_params(order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    bc = (hydro.PERIODIC, hydro.PERIODIC, hydro.OUTFLOW)
    want, _, dt1, _, _ = _single(g, params, s0, dt0, 0.4, steps, True, hydro.ADER, bc)
    d = hydro.Domain(g, params, bc=bc, exact=True)
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.4)
    d.step(steps)
    _, dt2, _ = d.sync()
    out = want.copy()
    d.gather(out)
    d.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    assert (out[act].view(np.uint64) == want[act].view(np.uint64)).all() and dt1 == dt2


def test_domain_rejects_bad_split():
    g = hydro.make_geometry(32, 8, 10, 3)
    with pytest.raises(ValueError, match="divide the mesh evenly"):
        hydro.Domain(g, hydro.make_params(3), devices=(0, 0, 0))


def test_domain_c_selftest(tmp_path):
    """The same checks from plain C through include/hydro_cuda.h and libhydro_cuda.so."""
    exe = tmp_path / "domain_selftest"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "domain_selftest.c"),
                    "-L", os.path.join(ROOT, "paper_2211_13295_b200"), "-lhydro_cuda", "-lm",
                    "-o", str(exe)], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2211_13295_b200") + ":" +
               os.environ.get("LD_LIBRARY_PATH", ""))
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("integ", [hydro.ADER, hydro.RK3])
@pytest.mark.parametrize("nslabs,bcz,shape", [(2, hydro.PERIODIC, (64, 14, 16)),
                                              (4, hydro.PERIODIC, (32, 12, 16)),
                                              (2, hydro.OUTFLOW, (32, 10, 12)),
                                              (3, hydro.PERIODIC, (64, 9, 48))])
def test_domain_peer_store_slabs_bitwise(exact, integ, nslabs, bcz, shape):
    """HC_XCHG_STORE: the fused kernels (ring or seam pair) write their boundary planes into
    the neighbour slabs' ghost planes -- several slabs on this one GPU stand in for peers --
    with no exchange step; bit-identical to the single domain, state, t and dt"""
    order, steps = 3, 4
    api = hydro.HostApi()
    g = hydro.make_geometry(*shape, order)
    params = hydro.make_params(order)
    s0 = modulate_z(api.init_isentropic_vortex(g, order))
    dt0 = api.initial_dt(g, s0, 0.4)
    bc = (hydro.PERIODIC, hydro.PERIODIC, bcz)
    want, t1, dt1, n1, _ = _single(g, params, s0, dt0, 0.4, steps, exact, integ, bc)
    d = hydro.Domain(g, params, bc=bc, exact=exact, integrator=integ,
                     transport=hydro.XCHG_STORE, devices=(0,) * nslabs)
    assert d.nslabs == nslabs
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.4)
    d.step(steps)
    t2, dt2, n2 = d.sync()
    out = want.copy()
    out[g.ghost:-g.ghost] = 0.0
    d.gather(out)
    # a second scatter re-primes the halos (peer copies for the first stage again)
    d.scatter(s0)
    d.set_time(0.0, dt0, 0.4)
    d.step(steps)
    out2 = want.copy()
    d.gather(out2)
    d.close()
    gh = g.ghost
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    assert (out[act].view(np.uint64) == want[act].view(np.uint64)).all(), \
        np.abs(out[act] - want[act]).max()
    assert (out2[act].view(np.uint64) == want[act].view(np.uint64)).all()
    assert (t2, dt2, n2) == (t1, dt1, n1)


def test_stepper_set_zpeer_validates():
    """hc_stepper_set_zpeer: rejected when the stepper fills its own z ghosts, or with no
    neighbour at all"""
    import ctypes as C
    lib = hydro.load_library()
    g = hydro.make_geometry(32, 8, 8, 3)
    st = hydro.Stepper(g, hydro.make_params(3))  # owns its z boundary (bc[2] = periodic)
    bufs = (C.c_void_p * 3)()
    nb = C.c_int()
    assert lib.hc_stepper_buffers(st.h, bufs, C.byref(nb)) == 0
    assert lib.hc_stepper_set_zpeer(st.h, bufs, bufs) != 0
    assert lib.hc_stepper_set_zpeer(st.h, None, None) != 0
    st.close()
