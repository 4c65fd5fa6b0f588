"""The command line on the B200 engine (tools/tuckerplan_cli.cpp) and the on-disk formats of
include/tuckerplan/serialize.hpp, checked the way the reference checks its own tool (tests/test_cli.cpp,
tests/test_serialize.cpp) plus the two transcripts its README prints (proj/README.md:63-72 and :122-126)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1707_05594_b200 import hostgen
from paper_1707_05594_b200 import planner as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1707_05594_b200", "lib")


@pytest.fixture(scope="module")
def cli():
    exe = os.path.join(ROOT, "build", "tuckerplan")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tools", "tuckerplan_cli.cpp"), "-o", exe, "-L" + LIBDIR,
                           "-ltuckerplan_b200", "-Wl,-rpath," + LIBDIR])

    def run(*args):
        p = subprocess.run([exe, *map(str, args)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
        return p.returncode, p.stdout.decode()
    return run


def test_readme_plan_transcript(cli):
    """proj/README.md:63-72, all nine lines."""
    code, out = cli("plan", "--L", "672,672,627,16", "--K", "279,279,153,14", "--procs", 32)
    assert code == 0
    assert out.splitlines() == [
        "spec      L672x672x627x16-K279x279x153x14",
        "tree      opt: 3016394906112 MACs over 8 nodes, depth 3",
        "procs     32",
        "static    grid 4x2x4x1, volume 9784331982",
        "dynamic   volume 2751247296, root grid 32x1x1x1",
        "          node 5 [M1] regrids to 1x1x4x8",
        "          node 8 [M1] regrids to 1x1x32x1",
        "selected  dynamic",
    ]


def test_plan_on_one_processor_degenerates(cli):                      # test_cli.cpp:60-69
    code, out = cli("plan", "--L", "6,5,4", "--K", "3,2,2", "--procs", 1, "--format", "json")
    assert code == 0
    plan = json.loads(out)
    assert plan["format"] == "tuckerplan-plan-v1"
    assert plan["static_grid"] == [1, 1, 1] and plan["dynamic_scheme"]["root"] == [1, 1, 1]
    assert plan["static_volume"]["total"] == 0 and plan["dynamic_volume"]["total"] == 0
    assert set(plan) == {"format", "spec", "strategy", "procs", "grid", "tree", "cost", "static_grid", "static_volume",
                         "dynamic_scheme", "dynamic_volume"}


def test_plan_cost_and_tree_round_trip(cli):                          # test_cli.cpp:71-85
    code, out = cli("plan", "--L", "8,6,5,4", "--K", "4,3,2,2", "--tree", "chain-k", "--procs", 4, "--format", "json")
    assert code == 0
    plan = json.loads(out)
    spec = P.ProblemSpec([8, 6, 5, 4], [4, 3, 2, 2])
    tree = P.chain_tree(spec, P.CHAIN_BY_COST)
    assert plan["cost"]["total_macs"] == P.tree_cost(tree, spec).total_macs

    def labels(node):                                                  # serialize.hpp:49-66: 1-based labels
        return (node["label"], [labels(c) for c in node.get("children", [])])

    def expect(t, node):
        kind = t.kind[node]
        name = "T" if kind == P.ROOT else ("M" if kind == P.MODE else "F") + str(t.mode[node] + 1)
        return (name, [expect(t, c) for c in t.children[node]])
    assert labels(plan["tree"]) == expect(tree, 0)
    per = {e["node"]: e["macs"] for e in plan["cost"]["per_node"]}
    cost = P.tree_cost(tree, spec)
    assert per == {i: m for i, m in enumerate(cost.per_node_macs) if m}


def test_plan_reruns_are_byte_identical_and_simulate_replays_them(cli, tmp_path):   # test_cli.cpp:87-130
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert cli("plan", "--L", "24,20,16,8", "--K", "8,6,4,4", "--procs", 16, "--out", a)[0] == 0
    assert cli("plan", "--L", "24,20,16,8", "--K", "8,6,4,4", "--procs", 16, "--out", b)[0] == 0
    body = a.read_bytes()
    assert body and body == b.read_bytes()
    plan = json.loads(body)
    code, out = cli("simulate", "--plan", a, "--format", "json")
    assert code == 0
    led = json.loads(out)
    assert led["total_model_ttm"] + led["total_model_regrid"] == plan["dynamic_volume"]["total"]
    code, out = cli("simulate", "--plan", a, "--grid", "static", "--format", "json")
    assert code == 0
    led = json.loads(out)
    assert led["total_model_ttm"] + led["total_model_regrid"] == plan["static_volume"]["total"]
    assert led["total_model_regrid"] == 0
    # a plan whose scheme was edited by hand is re-costed on load (plan_from_json recomputes the volumes)
    spec = P.ProblemSpec([24, 20, 16, 8], [8, 6, 4, 4])
    tree = P.optimal_tree(spec).tree
    best = P.optimal_static_grid(tree, spec, 16)
    assert plan["static_grid"] == best.grid and plan["static_volume"]["total"] == best.report.total
    dyn = P.optimal_dynamic_scheme(tree, spec, 16)
    assert plan["dynamic_scheme"]["root"] == dyn.scheme.root
    assert {int(k): v for k, v in plan["dynamic_scheme"]["nodes"].items()} == dyn.scheme.node_grids


def test_simulate_traced_agrees_with_the_model(cli):                  # test_cli.cpp:95-108
    code, out = cli("simulate", "--L", "12,10,8", "--K", "4,3,2", "--procs", 8, "--trace", "--format", "json")
    assert code == 0
    led = json.loads(out)
    assert led["traced"] is True
    for node in led["nodes"]:
        assert node["measured_ttm"] == node["model_ttm"]
    spec = P.ProblemSpec([12, 10, 8], [4, 3, 2])
    assert led["total_flops"] == P.tree_cost(P.optimal_tree(spec).tree, spec).total_macs
    # a regridding scheme: the traced owner changes are the reference's (tests/golden/dynamic_golden.json)
    code, out = cli("simulate", "--L", "8,8,8,8,8", "--K", "2,2,2,2,2", "--procs", 2, "--trace", "--format", "json")
    assert code == 0
    led = json.loads(out)
    with open(os.path.join(ROOT, "tests", "golden", "dynamic_golden.json")) as f:
        gold = [c for c in json.load(f) if c.get("tree_name") == "opt" and "scheme" in c and any(c["scheme"]["regrid"])
                and "traced_regrid" in c["scheme"]][0]
    code, out = cli("simulate", "--L", ",".join(map(str, gold["L"])), "--K", ",".join(map(str, gold["K"])), "--procs",
                    gold["procs"], "--trace", "--format", "json")
    assert code == 0
    led = json.loads(out)
    assert [n["node"] for n in led["nodes"]] == gold["scheme"]["nodes"]
    assert [n["measured_regrid"] for n in led["nodes"]] == gold["scheme"]["traced_regrid"]
    assert [n["measured_ttm"] for n in led["nodes"]] == gold["scheme"]["traced_ttm"]
    assert [n["model_regrid"] for n in led["nodes"]] == gold["scheme"]["regrid"]
    # trace mode is guarded (simulate.hpp:25-26, 130-135)
    assert cli("simulate", "--L", "200,200,200", "--K", "20,20,20", "--procs", 2, "--trace")[0] == 1


def test_invalid_inputs_exit_with_one(cli, tmp_path):                 # test_cli.cpp:176-185
    assert cli("plan", "--L", "6,5,4")[0] == 1                        # no --K
    assert cli("plan", "--L", "6,5", "--K", "3,2", "--procs", 7)[0] == 1   # no grid
    assert cli("plan", "--L", "6,5", "--K", "3,2", "--tree", "towers")[0] == 1
    assert cli("plan", "--L", "6,5", "--K", "7,2")[0] == 1            # K above L
    assert cli("plan", "--L", "6x5", "--K", "3,2")[0] == 1            # bad number
    assert cli("simulate", "--plan", "/nonexistent.json")[0] == 1
    assert cli("frobnicate")[0] == 1
    assert cli("--help")[0] == 0
    assert cli("plan", "--help")[0] == 0
    bad = tmp_path / "bad.json"
    bad.write_text('{"L": [6, 5], "K": [3, 2]')                      # truncated JSON
    code, out = cli("plan", "--spec", bad)
    assert code == 1 and "bad JSON" in out
    spec = tmp_path / "spec.json"
    spec.write_text('{ "K": [3, 2],\n  "L": [6, 5] }')
    code, out = cli("plan", "--spec", spec, "--procs", 2)
    assert code == 0 and out.splitlines()[0] == "spec      L6x5-K3x2"
    assert cli("plan", "--spec", spec, "--L", "6,5", "--K", "3,2")[0] == 1   # both sources
    plan = tmp_path / "noscheme.json"
    plan.write_text(json.dumps({"spec": {"L": [6, 5], "K": [3, 2]}, "procs": 1, "grid": "static"}))
    code, out = cli("simulate", "--plan", plan)
    assert code == 1 and "plan file lacks" in out


def test_tensor_file_format(cli, tmp_path):
    """serialize.hpp:191-216: one JSON header line {"dims":[...]} then little-endian doubles in storage order; the
    values are the reference's random_tensor stream (tests/golden/streams_golden.json pins hostgen to it)."""
    path = tmp_path / "t.bin"
    code, out = cli("gen-tensor", "--L", "12,10,8", "--seed", 7, "--out", path)
    assert code == 0 and out == "wrote %s: dims 12x10x8, 960 elements\n" % path
    raw = path.read_bytes()
    header, _, data = raw.partition(b"\n")
    assert header == b'{"dims":[12,10,8]}'
    values = np.frombuffer(data, dtype="<f8")
    assert values.shape == (960,)
    assert np.array_equal(values, hostgen.random_tensor([12, 10, 8], 7).reshape(-1))
    # truncated / headerless files are rejected (serialize.hpp:203-215)
    cut = tmp_path / "cut.bin"
    cut.write_bytes(raw[:-8])
    code, out = cli("hooi", "--tensor", cut, "--K", "4,3,2")
    assert code == 1 and "fewer elements than its header announces" in out
    junk = tmp_path / "junk.bin"
    junk.write_bytes(b"not a header\n" + data)
    code, out = cli("hooi", "--tensor", junk, "--K", "4,3,2")
    assert code == 1 and "does not start with a" in out
    assert cli("hooi", "--K", "4,3,2")[0] == 1                        # neither --tensor nor --L
    assert cli("hooi", "--tensor", path, "--L", "12,10,8", "--K", "4,3,2")[0] == 1


@pytest.mark.gpu
def test_readme_hooi_transcript_through_the_cli(cli, tmp_path, readme_kat):
    """proj/README.md:118-126: gen-tensor | hooi, Gauss-Seidel on the chain tree, on the GPU."""
    path = tmp_path / "t.bin"
    assert cli("gen-tensor", "--L", "12,10,8", "--seed", 7, "--out", path)[0] == 0
    code, out = cli("hooi", "--tensor", path, "--K", "4,3,2", "--sweeps", 4)
    assert code == 0, out
    lines = out.splitlines()
    assert lines[0] == "start: error " + readme_kat["start_error"]
    assert lines[1] == "sweep 1: error %s, tree macs %d, peak live %d" % (
        readme_kat["sweep1_error"], readme_kat["tree_macs"], readme_kat["peak_live"])
    assert [l.split(",")[0] for l in lines[2:]] == ["sweep 2: error 0.918925317677", "sweep 3: error 0.914793110656",
                                                    "sweep 4: error 0.913449730235"]   # oracle, SURVEY §8c


@pytest.mark.gpu
def test_generated_tensor_feeds_the_sweep_runner(cli, tmp_path):       # test_cli.cpp:187-207
    path = tmp_path / "t.bin"
    assert cli("gen-tensor", "--L", "12,10,8", "--seed", 7, "--out", path)[0] == 0
    report_path = tmp_path / "report.json"
    code, out = cli("hooi", "--tensor", path, "--K", "4,3,2", "--sweeps", 3, "--format", "json", "--out", report_path)
    assert code == 0, out
    report = json.loads(out)
    assert json.loads(report_path.read_text()) == report
    assert len(report["sweeps"]) == 3
    prev = 1e300
    for sweep in report["sweeps"]:
        assert sweep["error"] <= prev * (1.0 + 1e-9)
        prev = sweep["error"]
    assert report["final_error"] == prev
    assert report["scheme"] == "gauss-seidel" and report["tree"] == "chain-input"
    assert report["spec"] == {"L": [12, 10, 8], "K": [4, 3, 2]}
    # Jacobi composes with the searched tree; the stats are the planner's
    code, out = cli("hooi", "--L", "20,18,16", "--K", "5,4,3", "--seed", 3, "--scheme", "jacobi", "--sweeps", 2,
                    "--format", "json")
    assert code == 0, out
    report = json.loads(out)
    spec = P.ProblemSpec([20, 18, 16], [5, 4, 3])
    cost = P.tree_cost(P.optimal_tree(spec).tree, spec)
    assert report["tree"] == "opt" and report["sweeps"][0]["tree_macs"] == cost.total_macs
    assert report["sweeps"][0]["peak_live"] == cost.depth + 1
    assert cli("hooi", "--L", "20,18,16", "--K", "5,4,3", "--tree", "opt")[0] == 1   # Gauss-Seidel needs a chain tree


@pytest.mark.gpu
def test_hooi_on_a_processor_grid_through_the_cli(cli, tmp_path):
    """`hooi --procs P` runs the Jacobi sweeps on the grid executor (tp_grid_*; with one GPU the ranks share it) and
    must print the errors of the single-device run; the report names the grid and its model volume."""
    path = tmp_path / "t.bin"
    assert cli("gen-tensor", "--L", "24,20,16", "--seed", 5, "--out", path)[0] == 0
    base = ["hooi", "--tensor", path, "--K", "4,3,2", "--scheme", "jacobi", "--sweeps", 3]
    code, single = cli(*base)
    assert code == 0
    for extra in (["--procs", 2], ["--procs", 4, "--grid", "2x1x2"], ["--procs", 2, "--dynamic"]):
        code, out = cli(*base, *extra)
        assert code == 0, out
        lines = out.splitlines()
        assert lines[1].startswith("grid: %d ranks on 1 device(s), model volume" % extra[1])
        want = [l for l in single.splitlines() if l.startswith("sweep")]
        got = [l for l in lines if l.startswith("sweep")]
        assert len(got) == 3
        for a, b in zip(got, want):
            ea, eb = float(a.split("error ")[1].split(",")[0]), float(b.split("error ")[1].split(",")[0])
            assert abs(ea - eb) < 5e-10 and a.split(",", 1)[1] == b.split(",", 1)[1]
    report = tmp_path / "r.json"
    assert cli(*base, "--procs", 2, "--out", report, "--format", "json")[0] == 0
    data = json.loads(report.read_text())
    assert data["grid"]["procs"] == 2 and data["grid"]["model_volume"] > 0 and "root" in data["grid"]["scheme"]
    assert cli(*base, "--procs", 2, "--scheme", "gauss-seidel")[0] == 1      # the grid runs jacobi only
    assert cli(*base, "--procs", 3, "--grid", "2x1x1")[0] == 1                # grid does not multiply out to P
