#!/usr/bin/env python
"""Regenerates the golden fixtures in this directory from the REFERENCE itself.

Runs only in the build container (needs /root/reference to compile oracle/_ref/ref_tools,
see oracle/Makefile).  The fixtures it writes are committed; the GPU box never needs the
reference.  Usage:  python tests/golden/make_golden.py
"""
import json
import os
import random
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_TOOLS = os.path.join(ROOT, "oracle", "_ref", "ref_tools")


def run(*args):
    return subprocess.check_output([REF_TOOLS, *map(str, args)]).decode()


def plan(L, K, procs=()):
    args = ["plan", ",".join(map(str, L)), ",".join(map(str, K))]
    if procs:
        args.append(",".join(map(str, procs)))
    return json.loads(run(*args))


def main():
    subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle")])
    cases = []
    # the five BASELINE.json configs, P = 1, 2, 4, 8
    for L, K in [([200] * 3, [20] * 3), ([96] * 4, [10] * 4), ([400, 100, 100, 50], [40, 10, 20, 5]),
                 ([48] * 5, [8] * 5), ([1600] * 3, [100] * 3)]:
        cases.append(plan(L, K, (1, 2, 4, 8)))
    # specs the reference's own tests pin (tests/test_trees.cpp:60-77, test_tree_search.cpp:80-88,177-189,
    # test_grids.cpp:106-124, test_engine.cpp:213-227, README.md:65-72)
    cases.append(plan([4, 4, 4], [2, 2, 2], (1, 2, 4, 8)))
    cases.append(plan([6, 5, 4], [3, 2, 2], (1, 2, 4)))
    cases.append(plan([11, 7, 7, 11, 4], [3, 1, 2, 7, 1], (1, 2, 3, 6)))
    cases.append(plan([672, 672, 627, 16], [279, 279, 153, 14], (32,)))
    cases.append(plan([5, 4, 3, 2], [2, 2, 2, 2], (1, 2, 4, 8, 16)))
    cases.append(plan([8, 7, 6], [3, 3, 2], (1, 2, 3, 6, 12)))
    cases.append(plan([12, 10, 8], [4, 3, 2], (1, 2, 4, 8, 24)))
    cases.append(plan([4, 3, 5], [4, 3, 5], (1, 2, 3, 4, 5, 6, 60)))
    cases.append(plan([7], [3], (1, 2, 3)))
    # invalid specs keep their error codes
    cases.append(plan([4, 0, 4], [2, 2, 2]))
    cases.append(plan([4, 4], [5, 2]))
    # seeded random specs, 2..6 modes
    rng = random.Random(1707_05594)
    for _ in range(160):
        n = rng.randint(2, 6)
        L = [rng.randint(1, 40) for _ in range(n)]
        K = [rng.randint(1, l) for l in L]
        procs = sorted({1, rng.choice([2, 3, 4, 6, 8, 12, 16, 24, 32]), rng.choice([2, 4, 8, 9, 10, 27, 64])})
        cases.append(plan(L, K, procs))
    for _ in range(12):  # a few wider ones exercise the split-despite-reuse branch
        n = rng.randint(7, 9)
        L = [rng.randint(2, 12) for _ in range(n)]
        K = [rng.randint(1, l) for l in L]
        cases.append(plan(L, K, (1, 4, 8)))
    psi = {f"{p},{n}": int(run("psi", p, n)) for p in (1, 2, 4, 8, 12, 32, 64, 360, 1024, 2 ** 20)
           for n in (1, 2, 3, 4, 5, 6, 7)}
    blocks = [json.loads(run("blocks", length, parts)) for length, parts in
              [(100, 8), (1600, 8), (10, 3), (7, 7), (5, 1), (13, 4), (48, 5), (96, 7), (1, 1)]]
    with open(os.path.join(HERE, "planner_golden.json"), "w") as f:
        json.dump({"cases": cases, "psi": psi, "blocks": blocks}, f, separators=(",", ":"))

    # per-node grids: optimal_dynamic_scheme (both objectives), scheme volumes, traced reduce-scatter / regrid counts
    def dynamic(L, K, procs, tree):
        return json.loads(run("dynamic", ",".join(map(str, L)), ",".join(map(str, K)), procs, tree))
    dyn = []
    for L, K in [([200] * 3, [20] * 3), ([96] * 4, [10] * 4), ([400, 100, 100, 50], [40, 10, 20, 5]),
                 ([48] * 5, [8] * 5), ([1600] * 3, [100] * 3)]:
        for procs in (2, 4, 8, 16, 32):
            for tree in ("opt", "chain", "balanced"):
                dyn.append(dynamic(L, K, procs, tree))
    dyn.append(dynamic([672, 672, 627, 16], [279, 279, 153, 14], 32, "opt"))
    dyn.append(dynamic([4, 4], [5, 2], 2, "opt"))          # invalid spec keeps its code
    dyn.append(dynamic([5, 4, 3], [1, 1, 1], 2, "opt"))    # no valid grid
    rng = random.Random(554)
    for _ in range(140):   # small enough for the reference's trace mode (<= 1e6 elements, <= 64 procs)
        n = rng.randint(2, 5)
        L = [rng.randint(2, 14) for _ in range(n)]
        K = [rng.randint(1, l) for l in L]
        procs = rng.choice([2, 3, 4, 6, 8, 12, 16])
        dyn.append(dynamic(L, K, procs, rng.choice(["opt", "chain", "chain_by_cost", "balanced"])))
    with open(os.path.join(HERE, "dynamic_golden.json"), "w") as f:
        json.dump(dyn, f, separators=(",", ":"))

    # seeded streams: reference random_tensor + the gaussian stream random_decomposition consumes
    streams = {}
    tmp = "/tmp/_tp_golden.bin"
    for dims, seed in [((12, 10, 8), 7), ((3, 4, 2), 5), ((2, 5, 3, 2), 9), ((4, 3, 5), 21), ((6, 5, 4), 41)]:
        run("tensor", ",".join(map(str, dims)), seed, tmp)
        streams["tensor:%s:%d" % ("x".join(map(str, dims)), seed)] = np.fromfile(tmp).tolist()
    for count, seed in [(12 * 4 + 10 * 3 + 8 * 2, 0), (64, 1), (33, 2 ** 40 + 3)]:
        run("gaussians", count, seed, tmp)
        streams["gaussians:%d:%d" % (count, seed)] = np.fromfile(tmp).tolist()
    os.remove(tmp)
    with open(os.path.join(HERE, "streams_golden.json"), "w") as f:
        json.dump(streams, f)
    # the reference's float known-answer for the path (proj/README.md:122-126)
    with open(os.path.join(HERE, "readme_kat.json"), "w") as f:
        json.dump({"dims": [12, 10, 8], "tensor_seed": 7, "K": [4, 3, 2], "init_seed": 0, "scheme": "gauss_seidel",
                   "tree": "chain-input", "start_error": "0.986423815729", "sweep1_error": "0.940526801758",
                   "tree_macs": 12736, "peak_live": 3, "source": "proj/README.md:122-126"}, f, indent=1)
    print("wrote", len(cases), "planner cases,", len(dyn), "dynamic-grid cases")


if __name__ == "__main__":
    main()
