"""bench.py's reference arm (the reference's CPU implementation, no GPU needed): one JSON line
with the contract's keys, on a tiny mesh."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--n", "16", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_c1_line_matches_our_config_keys():
    """configs[0] through --workload c1: the reference's own 128 x 128 x 4 mesh; the config
    carries the workload only (each arm's build is the line's "build"), so both arms' configs
    compare equal."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "c1", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["n"] == [128, 128, 4] and d["warmup"] == 3
    assert "build" not in d["config"] and "reference" in d["build"]


def test_reference_arm_rk3_and_unavailable_extensions():
    """--integrator rk3 runs the reference's own rk_step on the host (the paper's CFD RK row);
    the extension workloads have no reference arm and say so in one line"""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--n", "16", "--steps", "1", "--warmup", "1", "--integrator", "rk3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["integrator"] == "rk3" and d["value"] > 0
    assert "RK3" in d["cpu_baseline"]["sample"]
    for w in ("mhd", "ced", "ader4"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl",
                            "reference", "--workload", w], capture_output=True, text=True,
                           timeout=120, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
        assert d["impl"] == "reference" and "unavailable" in d
