"""The bench.py JSON contract (the driver parses one line from stdout).

CPU: the reference arm (`--impl reference`) runs the reference's own CPU path
(oracle/_ref) and must print the contract line with impl/cpu_baseline/e2e.
GPU: the B200 arm must print every key the contract names, with a roofline,
an end-to-end measurement, a launch count and sampled clocks.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbmatch_ref.so")):
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_does_not_load_the_product():
    """The reference arm builds its graph with oracle/gen_oracle.cpp: neither the
    product package nor libbmatch_b200.so may be loaded in that process."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbmatch_ref.so")):
        pytest.skip("oracle/_ref not built")
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'C1', '--steps', '1', "
            "'--warmup', '0']; import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'libbmatch_b200' not in maps, 'product library mapped'; "
            "assert not any(m.startswith('paper_1303_1379_b200') for m in sys.modules), 'product imported'; "
            "print('CLEAN', file=sys.stderr)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "CLEAN" in out.stderr, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.strip()][-1])
    assert d["cardinality"] == 99961 and d["parity"]["ok"]


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--config", "C1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["bound"] == "hbm"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["h2d_bytes_per_step"] > 0
    assert e["pageable"]["ms_per_step"] > 0  # the shim's pageable-buffer path, same calls
    gi = e["gpu_init"]  # GPU cheap init inside the timed region
    assert gi["cardinality"] == 99961 and 0 < gi["initial_cardinality"] <= 99961 and gi["ms_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["parity"]["ok"] and d["cardinality"] == 99961
