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


def _run(exe, timeout):
    env = dict(os.environ, OMP_NUM_THREADS=str(min(8, os.cpu_count() or 1)))
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
