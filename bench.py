#!/usr/bin/env python
"""bench.py -- zone-updates/s of the fused WENO-ADER step on B200 (BASELINE.json metric).

Workload at N=1 (BASELINE.json configs[1], restated as the Euler proxy of SURVEY.md 8(d)):
C2 = 3D Euler isentropic vortex, 256^3, WENO-ADER + HLL, periodic. The reference has no 4th
order (geometry.hpp:13-27), so order 3 is the closest it supports. N>1 (torchrun): weak
scaling, every rank owns a 256^3 z-slab of a 256 x 256 x (256 N) periodic box; z halos go
over NCCL, dt_next is all-reduced (min).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--exact]

The headline is the FMA build (DFMA contraction, ~2-ulp division): within 1e-12 relative L1 of
the reference after 20 steps (the north star allows 1e-10); the bit-exact build (no
contraction, IEEE division, identical bits) is timed on the same workload and reported
beside it as "other_build".

A "step" is one full ADER step (ghost fill + fused kernel + dt hand-off) over the whole
mesh. value = zones x K / (max over ranks of the CUDA-event time of the K steps). The state
(2 x 720 MB per GPU) exceeds the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "zone-updates/sec (M/s) per GPU and 8-GPU box, % of HBM/FP64 roofline"
UNIT = "Mzone-updates/s"


def flops_per_zone(n, order, solver, ny=None, nz=None):
    """Algorithmic FP64 flops per active zone-update of the reference as written (add, sub,
    mul, div, sqrt = 1): F = R(recon+pred) + Phi*face + cross + 70 with
    R = ring zones / active zones ((n+2)/n)^3 on a cube) and Phi = faces / active zones
    (3(n+1)/n on a cube); C1 (128 x 128 x 4) gives 2837."""
    # order 4 (WENO-AO extension, no reference): 15 WENO-AO points x ~135 flops (6 divisions)
    # plus the quartic face extrapolations, counted by hand from the restatement as written
    recon, pred = {2: (120.0, 258.0), 3: (810.0, 543.0), 4: (2265.0, 543.0)}[order]
    face = {2: {1: 168.0, 0: 154.0}, 3: {1: 188.0, 0: 174.0},
            4: {1: 188.0, 0: 174.0}}[order].get(solver, 188.0)
    cross = 60.0 if order == 3 else 0.0
    nx = float(n)
    ny = float(ny or n)
    nz = float(nz or n)
    act = nx * ny * nz
    R = (nx + 2.0) * (ny + 2.0) * (nz + 2.0) / act
    phi = ((nx + 1.0) * ny * nz + nx * (ny + 1.0) * nz + nx * ny * (nz + 1.0)) / act
    return R * (recon + pred) + phi * face + cross + 70.0


def fp64_nominal_tflops(device, max_mhz):
    """Nominal DFMA rate: SMs x 64 FP64 lanes x 2 flop x the maximum SM clock."""
    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return sms * 64 * 2 * max_mhz * 1e6 / 1e12


BYTES_PER_ZONE = 80.0  # read + write U_skinny (5 doubles), SURVEY.md 8(d)


def _clock_proc(device, stop, out):
    """ClockSampler's child process: polls NVML every 2 ms until told to stop (a separate
    process, so the Python GIL of the timing thread cannot starve it)."""
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(device)
    samples, bits = [], 0
    out.put("ready")
    while not stop.is_set():
        try:
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            pass
        time.sleep(0.002)  # (each NVML query takes the driver; launch-bound runs feel it)
    out.put((samples, bits))


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region, from a forked
    child process (NVML only; no CUDA in the child)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device):
        self.device = device
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.proc = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _add_bits(self, r):
        for bit, name in self.REASONS.items():
            if r & bit and bit != 0x1:
                self.reasons.add(name)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self._add_bits(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            pass

    def __enter__(self):
        if self.nv:
            try:
                import multiprocessing as mp
                ctx = mp.get_context("fork")
                self.stop, self.q = ctx.Event(), ctx.Queue()
                self.proc = ctx.Process(target=_clock_proc, args=(self.device, self.stop, self.q),
                                        daemon=True)
                self.proc.start()
                self.q.get(timeout=30)  # sampling before the timed region starts
            except Exception:
                self.proc = None
            self._sample()
        return self

    def __exit__(self, *a):
        if not self.nv:
            return
        self._sample()  # (one more from this process, still under load)
        if self.proc is not None:
            try:
                self.stop.set()
                samples, bits = self.q.get(timeout=30)
                self.samples.extend(samples)
                self._add_bits(bits)
                self.proc.join(timeout=10)
            except Exception:
                pass

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------------ CPU baseline


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def mesh_of(args):
    """(nx, ny, nz) of the workload on one GPU / one CPU run."""
    return (128, 128, 4) if args.workload == "c1" else (args.n, args.n, args.n)


INTEGRATORS = {"ader": 0, "rk2": 2, "rk3": 3}  # IntegratorChoice codes (predictor.hpp:12)


def run_reference_cpu(n, order, steps, threads, integrator=0):
    """The reference's own harness (hydro::run_benchmark, harness.cpp:222-227) from
    oracle/_ref (built from /root/reference/proj/src); zones/s as it computes it
    (harness.cpp:177-180). Falls back to the C restatement (single thread) if absent."""
    # (no OMP_PROC_BIND / OMP_PLACES: binding made the reference 5 % slower on the box,
    # 6.30 vs 6.61 M/s, and the baseline must not be handicapped)
    from oracle import pyoracle as po
    if po.have_reference():
        ref = po.Reference()
        zps, _, _, _ = ref.run_benchmark(0, order, integrator, 1, n, steps, threads=threads)
        return zps, "reference", threads
    if integrator:
        raise RuntimeError("the C restatement fallback times ADER only (oracle/_ref missing)")
    orc = po.Oracle()
    nx, ny, nz = (n, n, n) if isinstance(n, int) else n
    g = po.make_geometry(nx, ny, nz, order)
    s = orc.init_isentropic_vortex(g, order)
    cfl = 0.6 if order == 2 else 0.4
    dt0 = orc.initial_dt(g, s, cfl)
    t0 = time.perf_counter()
    orc.run_steps(g, po.make_params(order), po.PERIODIC, cfl, steps, s, dt0)
    return nx * ny * nz * steps / (time.perf_counter() - t0), "port", 1


def reference_arm(args):
    """--impl reference: the reference's CPU implementation on the host cores, same metric
    and config; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = cpu_threads()
    mesh, order = mesh_of(args), args.order
    zones = mesh[0] * mesh[1] * mesh[2]
    # W warm-up steps (untimed; they also measure the step cost), then up to K timed steps,
    # capped so the timed part stays near 2 minutes of host time
    integ = INTEGRATORS[args.integrator]
    zps1, kind, cores = run_reference_cpu(mesh, order, max(1, args.warmup), threads, integ)
    step_s = zones / zps1
    steps = max(1, min(args.steps, int(120.0 / max(step_s, 1e-3))))
    zps, kind, cores = run_reference_cpu(mesh, order, steps, threads, integ)
    val = zps / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": zones / zps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (isentropic vortex IC)",
        "config": workload_config(args),
        "build": ("the reference's C++ (oracle/_ref: g++ -O3 -march=x86-64-v3 "
                  "-ffp-contract=off -fopenmp, its own sources)")
                 if kind == "reference" else "C restatement (oracle/, single thread)",
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{'x'.join(map(str, mesh))} O{order} HLL "
                                   f"{args.integrator.upper()} vortex, "
                                   f"{steps} timed steps (of K={args.steps} requested, capped "
                                   "at ~120 s) via hydro::run_benchmark on the host cores"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args):
    """The workload, identical in both arms (the build of each arm is the line's "build")."""
    if args.workload == "c1":
        return {
            "workload": ("C1: 2D Euler isentropic vortex 128 x 128 (x 4 z-invariant planes, "
                         "the reference's minimum), WENO-ADER O3 + HLL, periodic, on [-5,5]^3 "
                         "(configs[0], the reference's CPU-runnable case)"),
            "n": [128, 128, 4], "order": args.order, "solver": "hll", "integrator": "ader",
            "problem": "vortex",
            "l2": "state 7.2 MB fits L2: launch/latency-bound (absolute rate only)",
            "parallelism": f"{args.gpus} independent replicas" if args.gpus > 1
            else "single GPU"}
    scheme = (f"WENO-ADER O{args.order}" if args.integrator == "ader" else
              f"WENO O{args.order} + {args.integrator.upper()} (no ADER predictor; the paper's "
              "CFD RK row)")
    return {
        "workload": (f"C2: 3D Euler isentropic vortex {args.n}^3 per GPU, {scheme}"
                     " + HLL, periodic (configs[1]; the reference has no O4, O3 is its closest"
                     "; --order 4 runs the WENO-AO extension)"),
        "n": args.n, "order": args.order, "solver": "hll", "integrator": args.integrator,
        "problem": "vortex",
        "l2": "state 2 x {:.0f} MB per GPU > 126 MB L2 (no flush needed)".format(
            (args.n + 2 * args.order) ** 3 * 40 / 1e6),
        "parallelism": f"z-slab x{args.gpus}" if args.gpus > 1 else "single GPU",
    }


def build_of(args):
    return ("fma (DFMA contraction + ~2-ulp division; <= 7e-16 rel. L1 vs the reference after "
            "5 steps at 256^3, tests/test_fullsize_parity_gpu.py)") if args.fast else \
        "bit-exact (identical to the reference build)"


# ------------------------------------------------------------- extensions (MHD, CED)


def ext_roofline(name, order, n, ms_step, bytes_per_zone, max_mhz):
    """Roofline of an extension step from ALGORITHMIC work: FP64 flops per zone-update counted
    on the numpy restatement as written (tools/count_flops_ext.py -> profiles/r2_ext_flops.json,
    fitted a + b/n + c/n^2) and the compulsory HBM bytes (read + write the state once: MHD 8
    doubles, CED 6 doubles + the conductivity read). Both are per zone-update; the binding roof
    is the larger fraction. `traffic` is the measured DRAM traffic of a whole step
    (tools/ext_traffic.sh -> profiles/r2_ext_traffic.json)."""
    import torch
    zones = n ** 3
    with open(os.path.join(ROOT, "profiles", "r2_ext_flops.json")) as f:
        c = json.load(f)[f"{name}_o{order}"]
    fpz = c["a"] + c["b"] / n + c["c"] / n ** 2
    fsrc = c.get("source", "profiles/r2_ext_flops.json (restatement as written, "
                           "tools/count_flops_ext.py)")
    t = ms_step * 1e-3
    fp = fpz * zones / t / 1e12
    fp_peak = fp64_nominal_tflops(torch.cuda.current_device(), max_mhz or 1965)
    hbm_peak = measured_peaks().get("hbm_gbs", 6650.0)
    hb = bytes_per_zone * zones / t / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r2_ext_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            # (measured at order 3 only)
            traffic = json.load(f).get(name, {}).get("dram_bytes_per_zone") if order == 3 else None
    fp_frac, hb_frac = fp / fp_peak, hb / hbm_peak
    r = {"bound": "fp64" if fp_frac >= hb_frac else "hbm",
         "achieved": fp if fp_frac >= hb_frac else hb,
         "peak": fp_peak if fp_frac >= hb_frac else hbm_peak,
         "unit": "TFLOP/s" if fp_frac >= hb_frac else "GB/s",
         "frac": max(fp_frac, hb_frac),
         "flops_per_zone": fpz, "flops_source": fsrc,
         "fp64": {"achieved": fp, "peak": fp_peak, "unit": "TFLOP/s", "frac": fp_frac,
                  "peak_source": "nominal DFMA rate at the max SM clock"},
         "hbm": {"achieved": hb, "peak": hbm_peak, "unit": "GB/s", "frac": hb_frac,
                 "bytes_per_zone": bytes_per_zone,
                 "bytes_source": "compulsory: read + write the state once per step"},
         "traffic": traffic * zones if traffic else None,
         "traffic_per_zone": traffic,
         "traffic_note": ("measured DRAM bytes of a whole step per zone at 128^3 "
                          "(profiles/r2_ext_traffic.json); vs the compulsory bytes this is the "
                          "unfused design's re-read factor") if traffic else
                         "no capture (tools/ext_traffic.sh)",
         "kernel_ms_per_launch": ms_step}
    return r


# ---------------------------------------------------------------------- MHD (extension)


def bench_mhd(args):
    """BASELINE.json configs[2]: 3D MHD Orszag-Tang (z-invariant initial data on a 3D mesh)
    with constrained transport and the 2D-HLL edge solver, WENO-ADER O3, 384^3 on one GPU.
    No reference counterpart (parity unpinned; checked against oracle/mhd_oracle.py)."""
    import numpy as np
    import torch

    from paper_2211_13295_b200 import mhd, mhd_slabs
    # (order 4 materialises 96 x 8 solver states per zone: 192^3 fits, 384^3 would not)
    n = args.n if args.n != 256 else (192 if args.order == 4 else 384)
    order = args.order
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    cfl = 0.4
    if world > 1:  # weak scaling: n^3 per rank, z-slabs of a periodic n x n x (n world) mesh
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dom = mhd_slabs.MhdSlabDomain(n, n, n * world, order, rank=rank, world=world,
                                      device=local)
        st, g = dom.st, dom.geom
        s0 = dom.initial_state()
        st.upload(s0)
        st.set_time(0.0, dom.initial_dt(cfl), cfl)
        stream, step = dom.stream, dom.step
    else:
        g = mhd.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
        s0 = mhd.orszag_tang(g, order)
        st = mhd.MhdStepper(g, mhd.make_params(order, face_solver=mhd.HLLD if args.mhd_hlld
                                                else mhd.HLL))
        st.upload(s0)
        st.set_time(0.0, st.cfl_dt(cfl), cfl)
        stream = torch.cuda.ExternalStream(st.stream_ptr)

        def step():
            st.step(1)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = st.launches
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
        tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    launches = st.launches - l0
    t, dt, done = st.sync()
    zones = n ** 3 * world
    value = zones * args.steps / (ms * 1e-3) / 1e6
    roofline = ext_roofline("mhd", order, n, ms / args.steps, 128.0, clocks.max_mhz)
    # end to end through the public API with host buffers (H2D state, step, D2H state)
    host = torch.empty(s0.shape, dtype=torch.float64, pin_memory=True).numpy()
    host[...] = s0
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    ee = 2
    for _ in range(ee):
        st.upload(host)
        step()
        st.download(host)
    e2e_s = (time.perf_counter() - h0) / ee
    if world > 1:
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle import mhd_oracle as mo
        cn = 32
        cg = mhd.make_geometry(cn, cn, cn, order, (0, 0, 0), (1, 1, 1))
        cs = mhd.orszag_tang(cg, order)
        G = mo.Geom(cn, cn, cn, order, (0, 0, 0), (1, 1, 1))
        par = mo.Params(order)
        cdt = mo.cfl_dt(cs, G, par, cfl)
        c0 = time.perf_counter()
        mo.run_steps(cs, G, par, cfl, 2, cdt)
        cpu = {"value": cn ** 3 * 2 / (time.perf_counter() - c0) / 1e6, "unit": UNIT,
               "cores": 1, "kind": "port",
               "sample": f"{cn}^3 O{order} Orszag-Tang, 2 steps of the numpy restatement "
                         "oracle/mhd_oracle.py (the reference has no MHD)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Orszag-Tang IC sampled on the host, B from a vector potential)",
        "config": {"workload": f"C3: 3D ideal MHD Orszag-Tang {n}^3, WENO-ADER O{order}, "
                               f"{'HLLD' if args.mhd_hlld else 'HLL'} "
                               "faces + 2D-HLL (UCT) edge EMFs, constrained transport "
                               "(configs[2]; extension, no reference counterpart)",
                   "n": n, "order": order, "build": "bit-exact (--fmad=false)",
                   "l2": "state + modes ~50 GB > L2",
                   "parallelism": f"z-slab x{world} (NCCL halos of 8 arrays)" if world > 1
                   else "single GPU"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": zones / e2e_s / 1e6, "unit": UNIT,  # (all ranks' zones)
                "h2d_bytes_per_step": host.nbytes, "d2h_bytes_per_step": host.nbytes,
                "api": "hc_mhd_upload + hc_mhd_step + hc_mhd_download (host wall clock)"},
        "gpu_launches": launches, "clocks": clocks.summary(),
        "final": {"t": t, "dt_next": dt, "steps_done": done},
    }
    if rank == 0:
        line["final"]["max_divb"] = st.max_divb()
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------- CED (extension)


def bench_ced(args):
    """BASELINE.json configs[3]: 3D CED with stiff conductivity, WENO-ADER O3, 256^3: a plane
    wave crossing a conducting slab with sigma dt = 1e3 (stiff; the exponential step has no
    dt restriction). Extension without a reference counterpart (parity unpinned; checked
    against oracle/ced_oracle.py)."""
    import numpy as np
    import torch

    from paper_2211_13295_b200 import ced
    n, order = args.n, args.order
    torch.cuda.set_device(0)
    g = ced.make_geometry(n, n, n, order, (0, 0, 0), (1, 1, 1))
    st = ced.CedStepper(g, ced.make_params(order))
    s0 = ced.plane_wave(g)
    dt = st.cfl_dt(0.4)
    x = (np.arange(g.mx + 1) - g.ghost + 0.5) * g.dx
    sigma = np.zeros((g.mz + 1, g.my + 1, g.mx + 1))
    sigma[:, :, (x > 0.4) & (x < 0.6)] = 1e3 / dt
    st.upload(s0, sigma)
    st.set_time(0.0, dt)
    stream = torch.cuda.ExternalStream(st.stream_ptr)
    st.step(args.warmup)
    torch.cuda.synchronize()
    l0 = st.launches
    with ClockSampler(0) as clocks:
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = st.launches - l0
    t, _, done = st.sync()
    zones = n ** 3
    divb, divd = st.max_div()
    roofline = ext_roofline("ced", order, n, ms / args.steps, 104.0, clocks.max_mhz)
    # end to end through the public API with host buffers (H2D state + conductivity, step, D2H)
    host = torch.empty(s0.shape, dtype=torch.float64, pin_memory=True).numpy()
    host[...] = s0
    hsig = torch.empty(sigma.shape, dtype=torch.float64, pin_memory=True).numpy()
    hsig[...] = sigma
    h0 = time.perf_counter()
    ee = 2
    for _ in range(ee):
        st.upload(host, hsig)
        st.step(1)
        st.download(host)
    e2e_s = (time.perf_counter() - h0) / ee
    line = {
        "metric": METRIC, "value": zones * args.steps / (ms * 1e-3) / 1e6, "unit": UNIT,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (plane wave, conducting slab sigma dt = 1e3)",
        "config": {"workload": f"C4: 3D CED with stiff conductivity {n}^3, WENO-ADER O{order}, "
                               "CT for D and B, 2D upwind edge solver, exponential conduction "
                               "step (configs[3]; extension, no reference counterpart)",
                   "n": n, "order": order, "build": "bit-exact (--fmad=false)",
                   "parallelism": "single GPU"},
        "roofline": roofline,
        "cpu_baseline": None,
        "e2e": {"value": zones / e2e_s / 1e6, "unit": UNIT,
                "h2d_bytes_per_step": host.nbytes + hsig.nbytes, "d2h_bytes_per_step": host.nbytes,
                "api": "hc_ced_upload + hc_ced_step + hc_ced_download (host wall clock)"},
        "gpu_launches": launches, "clocks": clocks.summary(),
        "final": {"t": t, "steps_done": done, "max_divb": divb, "max_divd": divd},
    }
    st.close()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------- formally fourth-order ADER (extension)


def bench_ader4(args):
    """The formally fourth-order ADER step (csrc/ader4.cu, hc_ader4_*; the paper's O4 row,
    PAPER.md:1514-1525, which the reference -- second order in time -- does not have): 3D Euler
    isentropic vortex n^3, WENO-AO + cross terms, local space-time predictor, HLL at the
    face/time Gauss points. Roofline from the EXECUTED FP64 flops ncu counts per ring zone /
    face / zone (profiles/r2_ader4_flops.json; there is no restatement to count algorithmic
    flops on); the predictor dominates (~98 % of the step)."""
    import torch

    from paper_2211_13295_b200 import hydro
    n = args.n
    torch.cuda.set_device(0)
    api = hydro.HostApi()
    g = hydro.make_geometry(n, n, n, 3)
    s0 = api.init_isentropic_vortex(g, 3)
    st = hydro.Ader4Stepper(g, hydro.make_params(3))
    st.upload(s0)
    cfl = 0.4
    st.set_time(0.0, api.initial_dt(g, s0, cfl), cfl)
    stream = torch.cuda.ExternalStream(st.stream_ptr)
    st.step(args.warmup)
    torch.cuda.synchronize()
    l0 = st.launches
    with ClockSampler(0) as clocks:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st.step(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = st.launches - l0
    t, dt, done = st.sync()
    zones = n ** 3
    with open(os.path.join(ROOT, "profiles", "r2_ader4_flops.json")) as f:
        c = json.load(f)
    fpz = (c["predict_per_ring_zone"] * (n + 2) ** 3 / zones +
           sum(c["flux_per_face"]) * (n + 1) / n + c["update_per_zone"])
    tstep = ms / args.steps * 1e-3
    fp = fpz * zones / tstep / 1e12
    peak = fp64_nominal_tflops(0, clocks.max_mhz or 1965)
    roofline = {"bound": "fp64", "achieved": fp, "peak": peak, "unit": "TFLOP/s",
                "frac": fp / peak, "flops_per_zone": fpz,
                "flops_source": "profiles/r2_ader4_flops.json: EXECUTED FP64 flops "
                                "(DADD + DMUL + 2 DFMA, ncu) of the step's kernels",
                "peak_source": "nominal DFMA rate at the max SM clock",
                "traffic": None, "kernel_ms_per_launch": ms / args.steps}
    host = torch.empty(s0.shape, dtype=torch.float64, pin_memory=True).numpy()
    host[...] = s0
    h0 = time.perf_counter()
    ee = 2
    for _ in range(ee):
        st.upload(host)
        st.step(1)
        st.download(host)
    e2e_s = (time.perf_counter() - h0) / ee
    line = {
        "metric": METRIC, "value": zones * args.steps / (ms * 1e-3) / 1e6, "unit": UNIT,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (isentropic vortex, Gauss-sampled on the host)",
        "config": {"workload": f"O4: 3D Euler isentropic vortex {n}^3, formally fourth-order "
                               "ADER (WENO-AO + cross terms, space-time predictor, Gauss-point "
                               "quadrature) + HLL (the paper's O4 row; extension, the reference "
                               "is second order in time)",
                   "n": n, "order": 4, "build": "FMA-contracted (--fmad=true)",
                   "l2": "state 0.67 GB + face states 4 GB > L2", "parallelism": "single GPU"},
        "roofline": roofline, "cpu_baseline": None,
        "e2e": {"value": zones / e2e_s / 1e6, "unit": UNIT,
                "h2d_bytes_per_step": host.nbytes, "d2h_bytes_per_step": host.nbytes,
                "api": "hc_ader4_upload + hc_ader4_step + hc_ader4_download (host wall clock)"},
        "gpu_launches": launches, "clocks": clocks.summary(),
        "final": {"t": t, "dt_next": dt, "steps_done": done},
    }
    st.close()
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--mhd-hlld", action="store_true",
                    help="--workload mhd with the HLLD face solver (default HLL)")
    ap.add_argument("--integrator", default="ader", choices=list(INTEGRATORS),
                    help="ader (the reference's one-step ADER, the headline) or the reference's "
                         "rk2 / rk3 (stepper.cpp rk_step; the paper's CFD RK row)")
    ap.add_argument("--exact", action="store_true",
                    help="headline the bit-exact build (default: the FMA build, <= 1e-12 rel. L1)")
    ap.add_argument("--fast", action="store_true", help=argparse.SUPPRESS)  # (the default)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only-timed", action="store_true",
                    help="profiling runs (ncu launch lists): warm-up + timed steps only")
    ap.add_argument("--workload", default="euler",
                    choices=["euler", "c1", "mhd", "ced", "ader4"],
                    help="euler: configs[1] (the headline, 256^3); c1: configs[0] (128 x 128 "
                         "x 4, the reference's CPU-runnable case); mhd: configs[2], 3D "
                         "Orszag-Tang with CT + the multidimensional Riemann solver "
                         "(extension, 384^3); ced: configs[3] (extension, 256^3); ader4: the "
                         "formally fourth-order ADER step (extension, 256^3)")
    args = ap.parse_args()
    args.fast = not args.exact
    if args.workload == "c1" and "--steps" not in sys.argv:
        args.steps = 50  # C1 is quoted over 50 steps
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"

    if args.workload == "ced":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable":
                              "the reference has no CED (SPEC.md:8); nothing to run"}))
            return
        bench_ced(args)
        return
    if args.workload == "ader4":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable":
                              "the reference's ADER is second order in time; no O4 step"}))
            return
        bench_ader4(args)
        return
    if args.workload == "mhd":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable":
                              "the reference has no MHD (SPEC.md:8); nothing to run"}))
            return
        bench_mhd(args)
        return
    if args.impl == "reference":
        reference_arm(args)
        return

    import numpy as np
    import torch

    from paper_2211_13295_b200 import hydro, slabs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert world == args.gpus or world == 1, "launch N>1 with torchrun --nproc-per-node N"

    n, order = args.n, args.order
    mesh = mesh_of(args)
    c1 = args.workload == "c1"

    def make_domain(exact):
        if c1:  # configs[0]: one independent replica per rank, the reference's geometry
            return slabs.SlabDomain(128, 128, 4, order, rank=0, world=1, device=local,
                                    exact=exact, dz=2.5)
        return slabs.SlabDomain(n, n, n * world, order, rank=rank, world=world, device=local,
                                exact=exact, integrator=INTEGRATORS[args.integrator])

    def max_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
    dom = make_domain(not args.fast)
    s0 = dom.initial_state()
    cfl = 0.6 if order == 2 else 0.4
    dt0 = dom.initial_dt(s0, cfl)
    dom.upload(s0)
    dom.set_time(0.0, dt0, cfl)

    stream = dom.stream

    def timed(d, clocks=None):
        for _ in range(args.warmup):
            d.step()
        torch.cuda.synchronize()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        l0 = d.launches
        ev0.record(d.stream)
        for k in range(args.steps):
            d.step(kernel_events=kev[k])
        ev1.record(d.stream)
        torch.cuda.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1)
        kern = sum(a.elapsed_time(b) for a, b in kev) / args.steps
        return max_ranks(ms), kern, d.launches - l0

    with ClockSampler(local) as clocks:
        ms_max, kern_ms, launches = timed(dom)
    t, dt, done = dom.sync()

    zones_local = mesh[0] * mesh[1] * mesh[2]
    zones_total = zones_local * world
    value = zones_total * args.steps / (ms_max * 1e-3) / 1e6

    # roofline of the dominant kernel (the fused step), per launch on this rank. Denominator:
    # the nominal DFMA rate at the maximum SM clock (MEASURED_PEAKS.json has no FP64 figure);
    # the in-run DFMA probe (hc_fp64_peak) and the clock it ran at are reported beside it.
    fpz = flops_per_zone(mesh[0], order, 1, mesh[1], mesh[2])
    fpz_source = "SURVEY.md App. A: the reference's ADER step as written (dynamic count)"
    if args.integrator != "ader":  # executed FP64 flops of the RK step's launches (ncu)
        with open(os.path.join(ROOT, "profiles", "r2_rk_flops.json")) as f:
            fpz = json.load(f)[f"{args.integrator}_o{order}"]["flops_per_zone_step"]
        fpz_source = ("profiles/r2_rk_flops.json: EXECUTED FP64 flops (DADD + DMUL + 2 DFMA, "
                      "ncu, 128^3) of one RK step's compute launches, FMA build")
    with ClockSampler(local) as pclk:
        probe_fp64 = hydro.fp64_peak(local)
    max_mhz = clocks.max_mhz or pclk.max_mhz or 1965
    peak_fp64 = fp64_nominal_tflops(local, max_mhz)
    achieved = fpz * zones_local / (kern_ms * 1e-3) / 1e12
    kind = dom.st.kernel_info()[0] if hasattr(dom, "st") else "ring"
    kernel_desc = {
        "seam": "seam_ader_kernel + seam_fix_kernel: the step's compute launches (the "
                "ring-free pair; timed together, CUDA events around them)",
        "persistent": "persist_ader_kernel (opt-in persistent ring-free kernel)",
    }.get(kind, "fused_ader_kernel (ring kernel; CUDA events around the launch)")
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_achieved = BYTES_PER_ZONE * zones_local / (kern_ms * 1e-3) / 1e9
    roofline = {
        "bound": "fp64", "achieved": achieved, "peak": peak_fp64, "unit": "TFLOP/s",
        "frac": achieved / peak_fp64,
        "peak_source": f"nominal DFMA rate (SMs x 64 lanes x 2 flop x {max_mhz} MHz max SM "
                       "clock; MEASURED_PEAKS.json has no FP64 figure)",
        "peak_probe": {"value": probe_fp64, "unit": "TFLOP/s", "clocks": pclk.summary(),
                       "frac": achieved / probe_fp64,
                       "source": "hc_fp64_peak: 16 DFMA chains per thread, 32 warps per SM, "
                                 "best of 10 launches, this process"},
        "flops_per_zone": fpz, "flops_source": fpz_source, "kernel_ms_per_launch": kern_ms,
        "kernel": kernel_desc,
        "traffic": None,
        "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_achieved / hbm_peak, "bytes_per_zone": BYTES_PER_ZONE,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
    }
    # the binding unit's busy fraction from the committed ncu capture of this kernel
    prof = os.path.join(ROOT, "profiles",
                        f"r2_fused_o{order}_{n}_{'fma' if args.fast else 'exact'}.json")
    if not os.path.exists(prof):
        prof = prof.replace("r2_", "r1_")
    if os.path.exists(prof) and args.integrator == "ader":
        with open(prof) as f:
            k0 = json.load(f)["kernels"][0]
        roofline["fp64_pipe_busy_ncu"] = k0.get("fp64_pipe_pct", 0.0) / 100.0
        roofline["fp64_pipe_source"] = (os.path.relpath(prof, ROOT) + " (ncu --set full, "
                                        "sm__pipe_fp64_cycles_active, one launch)")
    traffic = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic) and args.integrator == "ader":
        with open(traffic) as f:
            tj = json.load(f).get(f"n{n}_o{order}_{'fma' if args.fast else 'exact'}")
        if tj:
            roofline["traffic"] = tj["bytes_per_launch"]
            roofline["traffic_per_zone"] = tj["bytes_per_zone"]
            roofline["traffic_source"] = tj["source"]

    if c1:  # launch-bound, fits L2: no HBM / traffic figures apply
        roofline["traffic"] = None
        for k in ("fp64_pipe_busy_ncu", "fp64_pipe_source", "hbm", "traffic_per_zone",
                  "traffic_source"):
            roofline.pop(k, None)
    if args.only_timed:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                              "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": ms_max / args.steps, "kernel_ms_per_launch": kern_ms,
                              "gpu_launches": launches, "note": "--only-timed profiling run"}))
        dom.close()
        return
    # end to end through the public API with HOST buffers: H2D of the step's input from
    # pinned memory, the step, D2H of the result and of dt_next -- the paper's skinny trick
    host = torch.empty(dom.host_shape(), dtype=torch.float64, pin_memory=True).numpy()
    host[...] = s0

    def e2e_step():
        if world == 1 or c1:  # H2D / fused step / D2H pipelined by z-chunks
            dom.st.step_host(host, host, 1 if c1 else args.e2e_chunks)
        else:  # slab: upload, step with the NCCL halo exchange, download
            dom.upload(host)
            dom.step()
            dom.download(host)
        dom.sync()
    e2e_step()  # untimed warm-up: creates the copy streams and events of the pipeline
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = max_ranks(e0.elapsed_time(e1))
    # world 1: step_host moves only the active zones (40 B each) both ways; N>1: whole slabs
    nbytes = zones_local * 40 if (world == 1 or c1) else host.nbytes
    e2e = {"value": zones_total * args.e2e_steps / (e_ms * 1e-3) / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": (nbytes + 16) * world,
           "steps": args.e2e_steps,
           "api": ("hc_stepper_step_host (H2D of the active U_skinny zones, fused step, D2H, "
                   "pipelined in "
                   f"{1 if c1 else args.e2e_chunks} z-chunks) + hc_stepper_sync (dt_next)")
           if (world == 1 or c1) else
                  "per rank: hc_stepper_upload + slab step (NCCL halos) + hc_stepper_download"}

    # the other contraction policy on the same workload (bit-exact build when the headline is
    # the FMA build and vice versa), reported beside the headline
    other = make_domain(args.fast)
    other.upload(s0)
    other.set_time(0.0, dt0, cfl)
    o_ms, o_kern, _ = timed(other)
    other.close()
    other_line = {"build": "bit-exact" if args.fast else "fma",
                  "value": zones_total * args.steps / (o_ms * 1e-3) / 1e6, "unit": UNIT,
                  "ms_per_step": o_ms / args.steps, "kernel_ms_per_launch": o_kern,
                  "roofline_frac": fpz * zones_local / (o_kern * 1e-3) / 1e12 / peak_fp64,
                  "roofline_frac_probe": fpz * zones_local / (o_kern * 1e-3) / 1e12 / probe_fp64}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        c_steps = 10 if c1 else 2
        zps, kind, cores = run_reference_cpu(mesh, order, c_steps, threads)
        cpu = {"value": zps / 1e6, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"{'x'.join(map(str, mesh))} O{order} HLL ADER vortex, {c_steps} steps "
                         "through hydro::run_benchmark (harness wall clock), default OpenMP "
                         "placement"}
        z1, _, _ = run_reference_cpu(128, order, 1, 1)  # also one thread
        cpu["single_thread"] = {"value": z1 / 1e6, "unit": UNIT, "cores": 1,
                                "sample": f"128^3 O{order}, 1 step, 1 thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (isentropic vortex IC sampled on the host, problems.cpp)",
            "config": workload_config(args), "build": build_of(args), "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e, "other_build": other_line, "gpu_launches": launches,
            "clocks": clocks.summary(),
            "final": {"t": t, "dt_next": dt, "steps_done": done},
        }
        print(json.dumps(line), flush=True)
    dom.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
