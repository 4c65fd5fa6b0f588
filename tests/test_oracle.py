"""Pins the oracle (oracle/hooi_oracle.py) to everything the reference's tests hold for the hot path:
the README float transcript, the integer goldens of tests/test_engine.cpp, and its property tests.
Inputs are the reference's own seeded streams (tests/golden/streams_golden.json, written by
oracle/_ref/ref_tools from the reference's random_tensor)."""
import numpy as np
import pytest

from oracle import hooi_oracle as ho
from paper_1707_05594_b200 import hostgen
from paper_1707_05594_b200 import planner as P


def otree(t: P.TtmTree) -> ho.Tree:
    return ho.Tree(t.n_modes, t.kind, t.mode, t.parent)


def test_product_streams_match_reference(streams_golden):
    """tp_random_tensor reproduces reference random_tensor bit for bit; the factor stream is the same draws."""
    for key, want in streams_golden.items():
        what, shape, seed = key.split(":")
        if what == "tensor":
            dims = [int(x) for x in shape.split("x")]
            got = hostgen.random_tensor(dims, int(seed))
            assert got.ravel().tolist() == want
        else:
            got = hostgen.random_tensor([int(shape)], int(seed))
            assert got.ravel().tolist() == want


def test_readme_transcript(streams_golden, readme_kat):
    """proj/README.md:122-126 — the one float known-answer of the path, to all 12 printed digits."""
    t = np.array(streams_golden["tensor:12x10x8:7"]).reshape(12, 10, 8)
    L, K = [12, 10, 8], [4, 3, 2]
    g = np.array(streams_golden["gaussians:94:0"])
    f = ho.orthonormal_from_gaussians(L, K, g)
    core = ho.core_from_factors(t, f)
    assert "%.12f" % ho.reconstruction_error(t, core, f) == readme_kat["start_error"]
    tree = otree(P.chain_tree(P.ProblemSpec(L, K)))
    st = ho.SweepStats()
    core, f = ho.hooi_sweep(t, L, K, f, tree, "gauss_seidel", st)
    assert "%.12f" % ho.reconstruction_error(t, core, f) == readme_kat["sweep1_error"]
    assert st.tree_macs == readme_kat["tree_macs"] and st.peak_live == readme_kat["peak_live"]
    # the product's Householder QR start agrees with the oracle's LAPACK one (same reflector convention)
    mine = hostgen.random_orthonormal_factors(L, K, 0)
    for a, b in zip(mine, f0 := ho.orthonormal_from_gaussians(L, K, g)):
        assert np.max(np.abs(a - b)) < 1e-13
        assert np.max(np.abs(a.T @ a - np.eye(a.shape[1]))) < 1e-12  # test_engine.cpp:190-204


def ttm_naive(t, m, mode):
    """tests/test_engine.cpp:47-63 element-wise oracle."""
    out_dims = list(t.shape)
    out_dims[mode] = m.shape[0]
    out = np.zeros(out_dims)
    for idx in np.ndindex(*out_dims):
        src = list(idx)
        s = 0.0
        for c in range(t.shape[mode]):
            src[mode] = c
            s += m[idx[mode], c] * t[tuple(src)]
        out[idx] = s
    return out


def test_unfold_fold_ttm(streams_golden):
    t = np.array(streams_golden["tensor:3x4x2:5"]).reshape(3, 4, 2)
    for mode in range(3):  # test_engine.cpp:81-97
        m = ho.unfold(t, mode)
        inner = int(np.prod(t.shape[mode + 1:]))
        for idx in np.ndindex(*t.shape):
            a = int(np.ravel_multi_index(idx[:mode], t.shape[:mode])) if mode else 0
            b = int(np.ravel_multi_index(idx[mode + 1:], t.shape[mode + 1:])) if mode < 2 else 0
            assert m[idx[mode], a * inner + b] == t[idx]
    t = np.array(streams_golden["tensor:2x5x3x2:9"]).reshape(2, 5, 3, 2)
    for mode in range(4):  # test_engine.cpp:99-107
        assert np.array_equal(ho.fold(ho.unfold(t, mode), t.shape, mode), t)
    with pytest.raises(ho.OracleError) as e:
        ho.fold(ho.unfold(t, 0), (2, 5, 3, 3), 0)
    assert e.value.code == "shape_mismatch"
    t = np.array(streams_golden["tensor:4x3x5:21"]).reshape(4, 3, 5)
    rng = np.random.default_rng(11)
    for mode in range(3):  # test_engine.cpp:109-125
        for new_len in (1, 2, 6):
            m = rng.standard_normal((new_len, t.shape[mode]))
            assert np.max(np.abs(ho.ttm(t, m, mode) - ttm_naive(t, m, mode))) < 1e-12
    macs = [0]
    ho.ttm(t, np.eye(2, 4), 0, macs)
    ho.ttm(t, np.eye(3), 1, macs)
    assert macs[0] == 2 * 60 + 3 * 60  # test_engine.cpp:127-133
    with pytest.raises(ho.OracleError):
        ho.ttm(t, np.eye(4), 1)


def test_truncated_basis_rules():
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    v, _ = np.linalg.qr(rng.standard_normal((40, 6)))
    m = u @ np.diag([5, 4, 3, 2, 1, 0.5]) @ v.T
    uu = np.linalg.svd(m)[0]
    for k in range(1, 6):  # test_engine.cpp:138-155
        b, deg = ho.leading_left_factors(m, k)
        assert not deg
        assert np.max(np.abs(b.T @ b - np.eye(k))) < 1e-9
        assert ho.projector_gap(b, uu[:, :k]) < 1e-9
    b, _ = ho.leading_left_factors(np.array([[0.0], [-3.0]]), 1)  # test_engine.cpp:157-162
    assert abs(b[0, 0]) < 1e-12 and abs(b[1, 0] - 1) < 1e-12
    a, _ = np.linalg.qr(rng.standard_normal((4, 3)))
    for k in (1, 2, 3):
        assert np.array_equal(ho.leading_left_factors(a, k)[0], ho.leading_left_factors(-a, k)[0])
    d = np.diag([2.0, 1.0, 1.0])  # test_engine.cpp:172-176
    assert not ho.leading_left_factors(d, 1)[1] and ho.leading_left_factors(d, 2)[1]
    for args, code in [((np.eye(3), 0), "bad_argument"), ((np.eye(3), 4), "bad_argument"),
                       ((np.zeros((0, 0)), 1), "shape_mismatch"), ((np.zeros((2049, 1)), 1), "too_large")]:
        with pytest.raises(ho.OracleError) as e:
            ho.leading_left_factors(*args)
        assert e.value.code == code


def test_sweep_integer_goldens(streams_golden):
    """test_engine.cpp:213-242."""
    L, K = [6, 5, 4], [3, 2, 2]
    spec = P.ProblemSpec(L, K)
    t = np.array(streams_golden["tensor:6x5x4:41"]).reshape(6, 5, 4)
    f = hostgen.random_orthonormal_factors(L, K, 1)
    for tree in (P.chain_tree(spec), P.optimal_tree(spec).tree):
        st = ho.SweepStats()
        ho.hooi_sweep(t, L, K, f, otree(tree), "jacobi", st)
        assert st.tree_macs == P.tree_cost(tree, spec).total_macs
        assert st.peak_live <= P.tree_depth(tree) + 1
    st = ho.SweepStats()
    ho.hooi_sweep(t, L, K, f, otree(P.chain_tree(spec)), "gauss_seidel", st)
    assert st.tree_macs == 1296
    assert st.core_macs == 3 * 120 + 2 * 60 + 2 * 24
    with pytest.raises(ho.OracleError) as e:
        ho.hooi_sweep(t, L, K, f, otree(P.balanced_tree(spec)), "gauss_seidel")
    assert e.value.code == "needs_chain_tree"


def test_sweep_properties():
    """test_engine.cpp:206-211, 244-271: exact at K=L; Jacobi subspaces tree-independent; GS monotone."""
    L = [4, 3, 5]
    t = hostgen.random_tensor(L, 13)
    f = hostgen.random_orthonormal_factors(L, L, 5)
    assert ho.reconstruction_error(t, ho.core_from_factors(t, f), f) < 1e-12
    L, K = [8, 7, 6], [3, 3, 2]
    spec = P.ProblemSpec(L, K)
    t = hostgen.random_tensor(L, 77)
    f = hostgen.random_orthonormal_factors(L, K, 2)
    _, on_chain = ho.hooi_sweep(t, L, K, f, otree(P.chain_tree(spec)), "jacobi")
    for tree in (P.balanced_tree(spec), P.optimal_tree(spec).tree):
        _, other = ho.hooi_sweep(t, L, K, f, otree(tree), "jacobi")
        for n in range(3):
            assert ho.projector_gap(on_chain[n], other[n]) < 1e-9
    t = hostgen.random_tensor(L, 55)
    f = hostgen.random_orthonormal_factors(L, K, 4)
    core = ho.core_from_factors(t, f)
    prev = ho.reconstruction_error(t, core, f)
    for _ in range(6):
        core, f = ho.hooi_sweep(t, L, K, f, otree(P.chain_tree(spec)), "gauss_seidel")
        err = ho.reconstruction_error(t, core, f)
        assert err <= prev + 1e-12
        prev = err
