"""A C++ caller written against the reference's header API, compiled against include/tuckerplan/ of this repo."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1707_05594_b200", "lib")


@pytest.fixture(scope="module")
def dropin():
    exe = os.path.join(ROOT, "build", "dropin")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "dropin.cpp"), "-o", exe, "-L" + LIBDIR,
                           "-ltuckerplan_b200", "-Wl,-rpath," + LIBDIR])
    return exe


def test_planner_through_cpp_headers(dropin):
    out = subprocess.check_output([dropin, "planner"]).decode().splitlines()
    assert out[0] == "chain 576" and out[1] == "opt 448"                      # test_trees.cpp:60-70, test_tree_search.cpp:80-88
    assert out[2] == "grid 1x2x2 vol 80"                                       # test_grids.cpp:117-124
    assert out[3] == "tree T(M2(M3(M4(F1), M1(F4)), M4(M1(F3))), M4(M3(M1(F2))))"
    assert out[4] == "canonical 1 depth 3"
    assert out[5] == "error 1 mode 1"                                          # Errc::k_too_large at mode 1
    assert out[6] == "error 7"                                                 # Errc::no_valid_grid
    assert out[7].startswith("fold 1 ")
    assert out[8] == "dynamic 9437184 regrids 3 static 11010048 again 9437184"   # SURVEY §8d, grid_dynamic.hpp
    assert out[9] == "error 8"                                                 # Errc::missing_assignment


@pytest.mark.gpu
def test_readme_transcript_through_cpp_headers(dropin, readme_kat):
    out = subprocess.check_output([dropin, "hooi"]).decode().splitlines()
    assert out[0] == "start: error " + readme_kat["start_error"]
    assert out[1] == "sweep 1: error %s, tree macs %d, peak live %d" % (
        readme_kat["sweep1_error"], readme_kat["tree_macs"], readme_kat["peak_live"])
    assert out[2].startswith("sweep 2: error 0.918925317677")
    assert out[3].startswith("resident jacobi: error ")
    assert out[4] == "error 11"                                                # Errc::needs_chain_tree


def test_serialize_checks_through_cpp_headers():
    """tests/cpp/serialize_check.cpp restates the reference's tests/test_serialize.cpp (golden strings included)."""
    exe = os.path.join(ROOT, "build", "serialize_check")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "serialize_check.cpp"), "-o", exe, "-L" + LIBDIR,
                           "-ltuckerplan_b200", "-Wl,-rpath," + LIBDIR])
    p = subprocess.run([exe], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    out = p.stdout.decode()
    assert p.returncode == 0, out
    assert [l for l in out.splitlines() if l.startswith("ok ")] == [
        "ok spec", "ok tree labels", "ok tree round trip", "ok tree labels rejected", "ok grid", "ok scheme",
        "ok reports", "ok traced counts", "ok tensor files", "ok json"]


@pytest.mark.gpu
def test_grid_executor_through_cpp_headers(dropin):
    """GridHooi (include/tuckerplan/hooi.hpp -> tp_grid_*): P = 2 and P = 4 virtual ranks on one GPU give the single-
    device engine's subspaces and fit, and ship exactly the volume optimal_static_grid predicted."""
    out = subprocess.check_output([dropin, "grid"]).decode().splitlines()
    assert len(out) == 3, out
    for line, procs in zip(out[:2], (2, 4)):
        words = line.split()
        assert words[0] == "procs" and int(words[1]) == procs
        fields = dict(zip(words[4::2], words[5::2]))
        assert fields["gap_ok"] == "1" and fields["fit_ok"] == "1" and fields["macs_ok"] == "1", line
        assert int(fields["shipped"]) == int(fields["model"]) > 0, line
    assert out[2] == "error 6"                     # Errc::invalid_grid


def test_supported_api_surface_compiles():
    """tests/cpp/surface_check.cpp names every entry point provided under the reference's header names with the
    reference's signature; its header comment lists what is deliberately absent (bench.hpp statistics, the tree
    enumerator, brute_force_dynamic)."""
    exe = os.path.join(ROOT, "build", "surface_check")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O0", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "surface_check.cpp"), "-o", exe, "-L" + LIBDIR,
                           "-ltuckerplan_b200", "-Wl,-rpath," + LIBDIR])
    assert subprocess.run([exe]).returncode == 0
