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
    """`--impl reference` times the CPU port on the host cores; no GPU involved, no product library mapped."""
    line = run_bench("--impl", "reference", "--config", 1, "--steps", 1, "--warmup", 0)
    assert line["impl"] == "reference" and line["metric"] == "hooi_s_per_iter" and line["unit"] == "s/iter"
    assert line["higher_is_better"] is False and line["value"] > 0 and line["n_gpus"] == 1
    assert line["config"]["workload"].startswith("C1_200x200x200")
    assert line["config"] == {"workload": "C1_200x200x200_to_20x20x20", "iterations": 5,
                              "schedule": "jacobi on optimal_tree", "tree": "T(M2(M3(F1)), M1(M3(F2), M2(F3)))",
                              "n_gpus": 1, "grid": [1, 1, 1], "grid_volume_elements": 0, "compare_grid": None}
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "s/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_does_not_map_the_product_library():
    """The reference arm takes tree, grid and input streams from the reference's own headers (oracle/_ref)."""
    code = ("import sys, bench; sys.argv=['bench.py','--impl','reference','--config','1','--steps','1','--warmup','0'];"
            "bench.main(); print('MAPPED' if 'libtuckerplan_b200' in open('/proc/self/maps').read() else 'CLEAN')")
    p = subprocess.run([sys.executable, "-c", code], stdout=subprocess.PIPE, stderr=subprocess.PIPE, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr.decode()[-2000:]
    assert p.stdout.decode().strip().splitlines()[-1] == "CLEAN"


def test_two_ranks_from_a_plain_command_line():
    """`python bench.py --gpus 2` with no WORLD_SIZE must itself become 2 ranks and print n_gpus == 2.  Here on the CPU
    with the contract-test backend (gloo + the tests' NumPy kernels); on a GPU box the same launch path starts one
    NCCL rank per GPU.  Both arms must print the same `config` object for the same (config, N)."""
    env_free = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "1", "--steps", "1",
                        "--warmup", "1", "--backend", "numpy-test"], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                       timeout=900, cwd=ROOT, env=env_free)
    assert p.returncode == 0, p.stderr.decode()[-3000:]
    lines = [l for l in p.stdout.decode().splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, lines
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["n_gpus"] == 2 and line["config"]["grid"] == [1, 1, 2]
    assert line["config"]["grid_volume_elements"] == 160000          # SURVEY.md §8d table, C1 at P = 2
    assert line["metric"] == "hooi_s_per_iter" and line["scaling"] == "strong" and line["value"] > 0
    per_node = line["ttm_tree"]["per_node"]
    assert all("nvlink_bytes_per_gpu" in r for r in per_node)
    # only the two M3 nodes contract the split mode: each GPU ships half of its partial product
    assert sorted(r["nvlink_bytes_per_gpu"] for r in per_node if r["nvlink_bytes_per_gpu"]) == [8 * 80000 / 2] * 2
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["parity_ok"] and len(cpu["parity_per_iteration"]) == 5
    for row in cpu["parity_per_iteration"]:
        assert row["max_sin_principal_angle"] < 1e-9 and row["core_norm_rel_diff"] < 1e-10
    ref = run_bench("--impl", "reference", "--gpus", 2, "--config", 1, "--steps", 1, "--warmup", 0)
    assert ref["n_gpus"] == 2 and ref["config"] == line["config"]


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
    assert cpu["parity_ok"] and len(cpu["parity_per_iteration"]) == 5       # C1: all 5 iterations compared
    for row in cpu["parity_per_iteration"]:
        assert row["max_sin_principal_angle"] < 1e-9 and row["core_norm_rel_diff"] < 1e-10 and row["fit_rel_diff"] < 1e-10
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] >= 8 * 200 ** 3 // 5 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["by_value_every_call"]["h2d_bytes_per_step"] >= 8 * 200 ** 3
    assert e2e["resident_api"]["value"] > 0
    assert len(line["run_from_start"]["per_iteration_ms"]) >= 5
    assert line["config"]["n_gpus"] == 1 and line["config"]["grid"] == [1, 1, 1]
    assert line["gpu_launches"] > 0
    assert set(("sm_mhz", "sm_max_mhz", "reasons")) <= set(line["clocks"])
