"""The reference's OWN test suites (proj/tests, compiled unmodified by oracle/Makefile and
_build.build_shim) -- once against the reference library, and once linked against the drop-in
shim (paper_2211_13295_b200/shim) so every hydro:: hot-path call runs the sm_100a kernels.
The binaries are built where /root/reference exists and shipped in oracle/_ref/."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _exe(name):
    p = os.path.join(REF_DIR, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (needs /root/reference at build time)")
    return p


def _run(exe, timeout, **extra_env):
    env = dict(os.environ, OMP_NUM_THREADS=str(min(8, os.cpu_count() or 1)), **extra_env)
    return subprocess.run([exe], capture_output=True, text=True, timeout=timeout, env=env)


def test_reference_unit_tests_on_the_reference_library():
    r = _run(_exe("unit_tests_ref"), 600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "test cases: 81 | 81 passed" in r.stdout


@pytest.mark.gpu
def test_reference_unit_tests_on_the_gpu_shim():
    """All 81 reference test cases (185k checks, incl. test_parallel_serial.cpp's bitwise
    kernel-vs-hydro::ref comparisons) with the GPU kernels swapped in."""
    r = _run(_exe("unit_tests_gpu"), 1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "test cases: 81 | 81 passed" in r.stdout


_VOLATILE = re.compile(r"informational zones/sec.*|fraction\(O2\)=\S+ fraction\(O3\)=\S+|"
                       r"in [0-9.e+-]+s")


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_gpu_shim():
    """acceptance_main.cpp through the shim must print the same numbers as the reference
    build for the numerical criteria 1-9 (convergence L1 norms and orders, conservation
    drift, decomposition difference, riemann counters...). Criterion 1 fails in the reference
    itself (O2 order 1.678 vs [1.7, 2.4]) and must fail identically here.
    Criterion 10 is a wall-clock property of the CPU pipeline (the predictor's share of the
    step time grows with order); on the GPU the host<->device staging of the per-kernel API
    dominates both orders, so it is reported, not compared."""
    ref = _run(_exe("acceptance_ref"), 1800)
    gpu = _run(_exe("acceptance_gpu"), 1800)
    a = [_VOLATILE.sub("", x) for x in ref.stdout.splitlines() if "criterion" in x]
    b = [_VOLATILE.sub("", x) for x in gpu.stdout.splitlines() if "criterion" in x]
    assert len(a) == 10 and len(b) == 10
    assert a[:9] == b[:9], "\n".join(a + ["---"] + b)
    assert all(x.startswith("[PASS]") for x in b[1:9])


# ---- the reference's driver (transfer.cpp's PatchSet + harness) on the device-resident path:
# the same binaries linked with shim/hydro_gpu_transfer.cpp instead of transfer.cpp, so
# run_patch_step steps a device PatchSet (hc_patchset_*) and the state stays in HBM between
# steps (host copies only at gather_from_patches or when a hydro:: call touches a patch).

@pytest.mark.gpu
def test_reference_unit_tests_on_the_resident_driver():
    """All 81 reference test cases with transfer.cpp replaced too: test_transfer.cpp's
    split invariance, ledger exactness and dt-min checks (which read the patches' modal state
    after run_patch_step) pass against the device PatchSet (default residency: the patches'
    host structures are current after every run_patch_step)."""
    r = _run(_exe("unit_tests_gpu_resident"), 1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "test cases: 81 | 81 passed" in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_resident_driver():
    """Criteria 1-9 print the same numbers as the reference build through the resident
    driver with the state kept in HBM across steps (HYDRO_GPU_RESIDENT=1: the harness's
    run_simulation -> run_patch_step on the device, gather_from_patches the only read)."""
    ref = _run(_exe("acceptance_ref"), 1800)
    gpu = _run(_exe("acceptance_gpu_resident"), 1800, HYDRO_GPU_RESIDENT="1")
    a = [_VOLATILE.sub("", x) for x in ref.stdout.splitlines() if "criterion" in x]
    b = [_VOLATILE.sub("", x) for x in gpu.stdout.splitlines() if "criterion" in x]
    assert len(a) == 10 and len(b) == 10
    assert a[:9] == b[:9], "\n".join(a + ["---"] + b)


@pytest.mark.gpu
def test_reference_run_benchmark_on_the_resident_driver(tmp_path):
    """hydro::run_benchmark (the reference's own harness code) at 64^3 O3 on the resident
    driver: the final U_skinny bit-identical to the reference library's run_benchmark
    (oracle/_ref), and the harness's zones/s far above the staged per-call path."""
    import json

    import numpy as np

    from oracle import pyoracle as po
    if not po.have_reference():
        pytest.skip("oracle/_ref reference library absent")
    n, order, steps = 64, 3, 6
    out = tmp_path / "final.bin"
    r = subprocess.run([_exe("run_benchmark_gpu"), str(n), str(order), str(steps), "1", "0",
                        str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["steps"] == steps
    _, fin_ref, t_ref, _ = po.Reference().run_benchmark(0, order, 0, po.HLL, (n, n, n), steps,
                                                        threads=0, want_state=True)
    got = np.fromfile(out, dtype=np.float64).reshape(fin_ref.shape)
    gh = 3
    act = np.s_[gh:-gh, gh:-gh, gh:-gh]
    assert (got[act].view(np.uint64) == fin_ref[act].view(np.uint64)).all()
    assert res["t_end"] == t_ref
