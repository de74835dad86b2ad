"""CPU-only checks of the product boundary: the C-ABI library builds, loads, exports every
symbol include/hydro_cuda.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2211_13295_b200 import hydro


def test_library_exports_every_declared_symbol():
    lib = hydro.load_library()
    names = hydro.exported_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.hc_abi_version() == 1


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors against the C compiler's view of include/hydro_cuda.h."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "sizes.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hydro_cuda.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(hc_geom),"
        " sizeof(hc_limiter), sizeof(hc_params), sizeof(hc_stepper_opts),"
        " offsetof(hc_geom, dx), offsetof(hc_params, lim), offsetof(hc_stepper_opts,"
        " integrator)); return 0;}\n")
    exe = tmp_path / "sizes"
    subprocess.run(["/usr/bin/gcc", "-I" + os.path.join(root, "include"), str(src), "-o",
                    str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(hydro.Geom), C.sizeof(hydro.Limiter), C.sizeof(hydro.Params),
            C.sizeof(hydro.StepperOpts), hydro.Geom.dx.offset, hydro.Params.lim.offset,
            hydro.StepperOpts.integrator.offset]
    assert got == want


def test_invalid_geometry_is_rejected_before_any_device_work():
    api = hydro.HostApi()
    g = hydro.make_geometry(4, 4, 4, 2)
    g.nx = 3  # geometry.hpp:58
    s = hydro.zeros_skinny(g)
    with pytest.raises(ValueError, match="at least 4 zones"):
        api.apply_boundary_skinny(g, hydro.PERIODIC, s)
    g = hydro.make_geometry(4, 4, 4, 2)
    m = np.zeros((g.mz, g.my, g.mx, 5, 11))
    with pytest.raises(ValueError, match="ghost width"):
        api.reconstruct_patch_o3(g, m)


@pytest.mark.skipif(hydro.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_a_device():
    api = hydro.HostApi()
    g = hydro.make_geometry(6, 6, 6, 2)
    s = hydro.zeros_skinny(g)
    with pytest.raises(hydro.HydroCudaError):
        api.apply_boundary_skinny(g, hydro.PERIODIC, s)
    with pytest.raises(hydro.HydroCudaError):
        hydro.Stepper(g, hydro.make_params(2))


def test_host_initial_conditions_match_the_oracle():
    """problems.cpp is host code on both sides: bit-identical vortex/sod/constant."""
    from oracle import pyoracle as po
    orc = po.Oracle()
    api = hydro.HostApi()
    for order, n in ((2, (9, 7, 5)), (3, (8, 8, 6))):
        g = hydro.make_geometry(*n, order)
        go = po.make_geometry(*n, order)
        a = api.init_isentropic_vortex(g, order)
        b = orc.init_isentropic_vortex(go, order)
        assert (a.view(np.uint64) == b.view(np.uint64)).all()
        a = api.init_isentropic_vortex(g, order, t=1.25)
        b = orc.init_isentropic_vortex(go, order, t=1.25)
        assert (a.view(np.uint64) == b.view(np.uint64)).all()
    g = hydro.make_geometry(8, 4, 4, 2, (0, 0, 0), (1, 1, 1))
    go = po.make_geometry(8, 4, 4, 2, (0, 0, 0), (1, 1, 1))
    assert (api.init_sod(g) == orc.init_sod(go)).all()
    assert (api.init_constant(g) == orc.init_constant(go)).all()


def test_extension_struct_layouts_match_the_headers(tmp_path):
    """ctypes mirrors of hc_mhd_params / hc_ced_params against include/hydro_{mhd,ced}.h"""
    import os
    import subprocess

    from paper_2211_13295_b200 import ced, mhd
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "sizes_ext.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hydro_mhd.h"\n#include "hydro_ced.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(hc_mhd_params),'
        " offsetof(hc_mhd_params, bc), offsetof(hc_mhd_params, device),"
        " offsetof(hc_mhd_params, face_solver), sizeof(hc_ced_params),"
        " offsetof(hc_ced_params, bc), offsetof(hc_ced_params, device)); return 0;}\n")
    exe = tmp_path / "sizes_ext"
    subprocess.run(["/usr/bin/gcc", "-I" + os.path.join(root, "include"), str(src), "-o",
                    str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(mhd.MhdParams), mhd.MhdParams.bc.offset, mhd.MhdParams.device.offset,
            mhd.MhdParams.face_solver.offset, C.sizeof(ced.CedParams), ced.CedParams.bc.offset, ced.CedParams.device.offset]
    assert got == want


@pytest.mark.skipif(hydro.device_count() > 0, reason="checks the no-GPU behaviour")
def test_extensions_have_no_cpu_fallback():
    from paper_2211_13295_b200 import ced, mhd
    g = mhd.make_geometry(8, 8, 8, 3, (0, 0, 0), (1, 1, 1))
    with pytest.raises(hydro.HydroCudaError):
        mhd.MhdStepper(g, mhd.make_params(3))
    with pytest.raises(hydro.HydroCudaError):
        ced.CedStepper(g, ced.make_params(3))
