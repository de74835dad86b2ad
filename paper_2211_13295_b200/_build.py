"""Builds libhydro_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Every .cu is compiled with --fmad=false (bit-exact vs the reference's -ffp-contract=off
build) except fused_fast.cu, the FMA-contracted instantiation of the fused step.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build_obj")
LIB = os.path.join(PKG, "libhydro_cuda.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin",
                 "/usr/bin/g++", "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v"]
TUNE = ["-DHC_TUNE"] if os.environ.get("HC_TUNE") == "1" else []
# experiment-only macro overrides for the fused instantiations, e.g. HC_NVCC_DEFS="-DSEAM_FIX_MINB=6"
TUNE += os.environ.get("HC_NVCC_DEFS", "").split()
SOURCES = {
    "capi_common.cu": ["--fmad=false"],
    "patch_kernels.cu": ["--fmad=false"],
    "stepper.cu": ["--fmad=false"],
    "fused_exact.cu": ["--fmad=false"] + TUNE,
    "fused_fast.cu": ["--fmad=true"] + TUNE,
    "peak.cu": ["--fmad=true"],
    "mhd.cu": ["--fmad=false"] + TUNE,
    "ced.cu": ["--fmad=false"] + TUNE,
    "domain.cu": ["--fmad=false"],
    "ader4.cu": ["--fmad=true"] + TUNE,
}


def _compile(name, flags, verbose):
    src = os.path.join(CSRC, name)
    import hashlib
    tag = hashlib.sha1(" ".join(COMMON + flags).encode()).hexdigest()[:8]
    obj = os.path.join(BUILD, name.replace(".cu", f".{tag}.o"))
    log = os.path.join(BUILD, name.replace(".cu", ".ptxas.txt"))
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps += [os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    stem = name.replace(".cu", ".")
    for old in os.listdir(BUILD):  # objects of this source under other flag sets
        if old.startswith(stem) and old.endswith(".o") and os.path.join(BUILD, old) != obj:
            os.remove(os.path.join(BUILD, old))
    cmd = [NVCC, "-c", src, "-o", obj] + COMMON + flags
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed for " + name)
    if verbose:
        print(f"[build] {name}")
    return obj


HOST_SOURCES = ["problems_host.cpp"]
CXX = "/usr/bin/g++"
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fopenmp",
            "-I" + os.path.join(ROOT, "include")]


def _compile_host(name, verbose):
    src = os.path.join(CSRC, name)
    obj = os.path.join(BUILD, name.replace(".cpp", ".o"))
    hdr = os.path.join(ROOT, "include", "hydro_cuda.h")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src),
                                                             os.path.getmtime(hdr)):
        return obj
    subprocess.run([CXX, "-c", src, "-o", obj] + CXXFLAGS, check=True)
    if verbose:
        print(f"[build] {name}")
    return obj


def build(verbose=True) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES) + len(HOST_SOURCES)) as ex:
        futs = [ex.submit(_compile, k, v, verbose) for k, v in SOURCES.items()]
        futs += [ex.submit(_compile_host, h, verbose) for h in HOST_SOURCES]
        objs = [f.result() for f in futs]
    stamp = LIB + ".objs"
    listing = "\n".join(objs)
    same_set = os.path.exists(stamp) and open(stamp).read() == listing
    if same_set and os.path.exists(LIB) and \
            os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", "-o", tmp] + ARCH + ["-ccbin", "/usr/bin/g++", "-Xcompiler",
                                                 "-fopenmp"] + objs + ["-ldl"]
    subprocess.run(cmd, check=True)
    shutil.move(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(listing)
    if verbose:
        print(f"[build] {LIB}")
    return LIB


REF = "/root/reference/proj"
REF_FLAGS = ["-std=c++20", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp",
             "-include", "algorithm"]


def build_shim(verbose=True):
    """Links the reference's own unit tests and acceptance suite against the drop-in shim
    (shim/hydro_gpu_shim.cpp -> libhydro_cuda.so) in place of proj/src/{fields,boundary,
    reconstruct,predictor,corrector,stepper}.cpp. Needs /root/reference (build container
    only); the binaries land in oracle/_ref/ (git-ignored, shipped to the GPU box)."""
    if not os.path.isdir(REF):
        return None
    out_dir = os.path.join(ROOT, "oracle", "_ref")
    os.makedirs(out_dir, exist_ok=True)
    kept = [os.path.join(REF, "src", f) for f in
            ("harness.cpp", "problems.cpp", "transfer.cpp", "serial_ref.cpp")]
    shim = os.path.join(PKG, "shim", "hydro_gpu_shim.cpp")
    tests = sorted(os.path.join(REF, "tests", f) for f in os.listdir(os.path.join(REF, "tests"))
                   if f.endswith(".cpp") and f != "acceptance_main.cpp")
    inc = ["-I" + os.path.join(REF, "include"), "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "oracle", "doctest_shim"), "-I" + os.path.join(REF, "tests"),
           "-I" + os.path.join(PKG, "shim")]
    link = ["-L" + PKG, "-l:libhydro_cuda.so", "-Wl,-rpath,$ORIGIN/../../paper_2211_13295_b200"]
    # the device-resident PatchSet driver replaces transfer.cpp too (hydro_gpu_transfer.cpp)
    xfer = os.path.join(PKG, "shim", "hydro_gpu_transfer.cpp")
    kept_res = [k for k in kept if not k.endswith("transfer.cpp")]
    accept = os.path.join(REF, "tests", "acceptance_main.cpp")
    targets = {
        "unit_tests_gpu": tests + kept + [shim],
        "acceptance_gpu": [accept] + kept + [shim],
        "unit_tests_gpu_resident": tests + kept_res + [shim, xfer],
        "acceptance_gpu_resident": [accept] + kept_res + [shim, xfer],
        "run_benchmark_gpu": [os.path.join(PKG, "shim", "run_benchmark_gpu.cpp")] +
                             [k for k in kept_res if not k.endswith("serial_ref.cpp")] +
                             [shim, xfer],
    }
    deps = [shim, xfer, os.path.join(PKG, "shim", "shim_resident.hpp"),
            os.path.join(PKG, "shim", "run_benchmark_gpu.cpp"), LIB]
    for name, srcs in targets.items():
        exe = os.path.join(out_dir, name)
        if os.path.exists(exe) and os.path.getmtime(exe) >= max(os.path.getmtime(d) for d in deps):
            continue
        subprocess.run([CXX] + REF_FLAGS + inc + ["-o", exe] + srcs + link, check=True)
        if verbose:
            print(f"[build] {exe}")
    return out_dir


if __name__ == "__main__":
    build()
