"""bench.py prints ONE JSON line with the fields the driver reads; checked on the smallest configuration."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *map(str, args)], stdout=subprocess.PIPE,
                       stderr=subprocess.PIPE, timeout=timeout, cwd=ROOT)
    assert p.returncode == 0, p.stderr.decode()[-2000:]
    lines = [l for l in p.stdout.decode().splitlines() if l.strip()]
    assert len(lines) == 1, lines
    return json.loads(lines[0])


def test_reference_arm_line():
    """`--impl reference` times the CPU port on the host cores; no GPU involved."""
    line = run_bench("--impl", "reference", "--config", 1, "--steps", 1, "--warmup", 0)
    assert line["impl"] == "reference" and line["metric"] == "hooi_s_per_iter" and line["unit"] == "s/iter"
    assert line["higher_is_better"] is False and line["value"] > 0 and line["n_gpus"] == 1
    assert line["config"]["workload"].startswith("C1_200x200x200")
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "s/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_b200_arm_line():
    line = run_bench("--config", 1, "--steps", 3, "--warmup", 3)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["metric"] == "hooi_s_per_iter" and line["unit"] == "s/iter" and line["higher_is_better"] is False
    assert line["steps"] == 3 and line["warmup"] == 3 and line["n_gpus"] == 1 and line["dtype"] == "f64"
    assert abs(line["value"] * 1e3 - line["ms_per_step"]) < 1e-9 and line["value"] > 0
    assert line["vs_baseline"] is None and line["data"] == "synthetic"
    assert "workload" in line["config"] and "model" not in line["config"]
    roof = line["roofline"]
    assert set(("bound", "achieved", "peak", "unit", "frac", "traffic")) <= set(roof)
    assert roof["bound"] in ("hbm", "tensor") and roof["unit"] in ("GB/s", "TFLOP/s")
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-12
    cpu = line["cpu_baseline"]
    assert set(("value", "unit", "cores", "kind", "sample")) <= set(cpu) and cpu["kind"] in ("port", "reference")
    assert cpu["parity_first_iteration"]["max_sin_principal_angle"] < 1e-9
    assert cpu["parity_first_iteration"]["core_norm_rel_diff"] < 1e-10
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] >= 8 * 200 ** 3 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0
    assert set(("sm_mhz", "sm_max_mhz", "reasons")) <= set(line["clocks"])
