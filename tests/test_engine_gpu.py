"""GPU parity tests: the CUDA engine (through the C ABI) against the oracle on the same seeded inputs.
Mirrors reference tests/test_engine.cpp; bounds are stated next to each check."""
import numpy as np
import pytest

from oracle import hooi_oracle as ho
from paper_1707_05594_b200 import Errc, TuckerplanError, engine as E, hostgen, planner as P, workloads as W

pytestmark = pytest.mark.gpu
EPS = np.finfo(np.float64).eps


def otree(t):
    return ho.Tree(t.n_modes, t.kind, t.mode, t.parent)


def code_of(fn):
    with pytest.raises(TuckerplanError) as e:
        fn()
    return e.value.code


@pytest.fixture(scope="module")
def ctx():
    c = E.Context(0)
    yield c
    c.close()


def ttm_bound(t, m, mode):
    # forward error of a length-L dot product in any summation order is <= L eps sum|m||x|; oracle (BLAS) and
    # DMMA both obey it, so they differ by at most twice that.  sum|m||x| <= L max|m| max|x|.
    L = t.shape[mode]
    return 2 * L * EPS * L * np.max(np.abs(m)) * np.max(np.abs(t)) + 1e-300


TTM_SHAPES = [
    # dims, mode, new_len
    ((4, 3, 5), 0, 1), ((4, 3, 5), 0, 2), ((4, 3, 5), 0, 6), ((4, 3, 5), 1, 1), ((4, 3, 5), 1, 2), ((4, 3, 5), 1, 6),
    ((4, 3, 5), 2, 1), ((4, 3, 5), 2, 2), ((4, 3, 5), 2, 6),            # test_engine.cpp:109-125
    ((1,), 0, 1), ((7,), 0, 3), ((1, 1, 1), 1, 1), ((9, 1), 0, 4), ((1, 9), 1, 4),
    ((37, 41), 0, 5), ((37, 41), 1, 5), ((64, 64, 64), 1, 8), ((64, 64, 64), 0, 8), ((64, 64, 64), 2, 8),
    ((33, 50, 6), 1, 20), ((33, 50, 5), 1, 20), ((33, 50, 2), 1, 20), ((33, 50, 3), 1, 7),   # tiny / odd inner
    ((10, 100, 48), 1, 10), ((10, 96, 100), 1, 10), ((17, 23, 129), 1, 13), ((5, 200, 200), 1, 20),
    ((200, 4000), 0, 20), ((4000, 200), 1, 20), ((4001, 201), 1, 20), ((1000, 50), 1, 5), ((999, 49), 1, 5),
    ((2, 160, 130), 1, 100), ((130, 160), 1, 100), ((160, 2, 70), 0, 100), ((3, 300, 16), 1, 130),
    ((6, 5, 4, 3, 2), 2, 3), ((6, 5, 4, 3, 2), 4, 2), ((6, 5, 4, 3, 2), 0, 6), ((8, 8, 8, 8), 3, 8),
    ((40, 48, 48), 0, 8), ((12, 48, 2304), 1, 8), ((3, 96, 96), 1, 10), ((24, 11, 16), 1, 33), ((3, 70, 10), 1, 70),
]


@pytest.mark.parametrize("dims,mode,new_len", TTM_SHAPES)
def test_ttm_matches_oracle(ctx, dims, mode, new_len):
    seed = (sum(dims) * 31 + mode * 7 + new_len) % 10000
    t = hostgen.random_tensor(dims, seed)
    m = hostgen.random_tensor([new_len, dims[mode]], seed + 1)
    macs = [5]
    got = E.ttm(t, m, mode, macs, ctx=ctx)
    want = ho.ttm(t, m, mode)
    assert got.shape == want.shape
    assert macs[0] == 5 + new_len * t.size                      # exact MAC ledger, accumulating (ttm.hpp:92-94)
    assert np.max(np.abs(got - want)) <= ttm_bound(t, m, mode)
    # and far tighter in the typical case: a few ulps of the result scale
    assert np.max(np.abs(got - want)) <= 64 * EPS * np.sqrt(dims[mode]) * np.max(np.abs(m)) * np.max(np.abs(t))


SPLITK_SHAPES = [
    # dims, mode, new_len: few columns and a contraction of 32..512 (csrc/ttm_splitk_kernels.cu) -- the K = 40 nodes of
    # C3, the second-level nodes of C1 / C2, ragged warp shares of the contraction, odd trailing extents, inner == 1
    # with a ragged last n-tile, one to six m-tiles and more than one K block
    ((400, 1000), 0, 40), ((400, 10, 100, 5), 0, 40), ((20, 200, 200), 2, 20), ((20, 200, 20), 1, 20),
    ((96, 10, 10, 10), 0, 10), ((10, 10, 96, 10), 2, 10), ((13, 77, 9), 1, 11), ((3, 510, 16), 1, 6), ((5, 33, 8), 1, 48),
    ((4001, 201), 1, 20), ((999, 49), 1, 5), ((7, 512, 11), 1, 44), ((1, 32, 8), 1, 1), ((2, 100, 1000), 1, 7),
]


@pytest.mark.parametrize("dims,mode,new_len", SPLITK_SHAPES)
def test_ttm_split_contraction_kernel(ctx, dims, mode, new_len):
    """The small-node kernel adds up to eight partial sums in warp order: equal to the streaming kernels' result and to the
    oracle to a few ulps of the result scale, and bit-identical from run to run."""
    seed = (sum(dims) * 13 + new_len) % 10000
    t = hostgen.random_tensor(dims, seed)
    m = hostgen.random_tensor([new_len, dims[mode]], seed + 1)
    split = E.ttm(t, m, mode, ctx=ctx)
    again = E.ttm(t, m, mode, ctx=ctx)
    E.check(E.lib.tp_set_global_option(3, E.ctypes.c_longlong(0)))   # TP_GLOBAL_OPT_TTM_SPLITK off
    try:
        streamed = E.ttm(t, m, mode, ctx=ctx)
    finally:
        E.check(E.lib.tp_set_global_option(3, E.ctypes.c_longlong(1)))
    assert np.array_equal(split, again)
    want = ho.ttm(t, m, mode)
    scale = EPS * np.sqrt(dims[mode]) * np.max(np.abs(m)) * np.max(np.abs(t))
    assert np.max(np.abs(split - want)) <= 64 * scale
    assert np.max(np.abs(split - streamed)) <= 64 * scale


PACKED_SHAPES = [
    # dims, mode, new_len: trailing extents 2..7 behind the contracted mode, slab counts around the 32-slab tile,
    # ragged last chunks of the contraction, K blocks of one to four m-tiles and more than one K block
    ((33, 50, 5), 1, 20), ((64, 100, 5), 1, 20), ((31, 16, 3), 1, 8), ((97, 34, 7), 1, 9), ((40, 7, 2), 1, 3),
    ((5, 18, 3), 1, 32), ((70, 20, 5), 1, 40), ((3, 6, 4, 10, 3), 3, 5), ((130, 48, 6), 1, 17), ((1, 22, 3), 1, 4),
    ((400, 100, 5), 1, 20),
]


@pytest.mark.parametrize("dims,mode,new_len", PACKED_SHAPES)
def test_ttm_packed_columns_kernel_is_bit_identical_to_the_general_one(ctx, dims, mode, new_len):
    """csrc/ttm_packed_kernels.cu (1 < inner < 8): same sums in the same order as the general kernels."""
    seed = (sum(dims) * 17 + new_len) % 10000
    t = hostgen.random_tensor(dims, seed)
    m = hostgen.random_tensor([new_len, dims[mode]], seed + 1)
    packed = E.ttm(t, m, mode, ctx=ctx)
    E.check(E.lib.tp_set_global_option(2, E.ctypes.c_longlong(0)))   # TP_GLOBAL_OPT_TTM_PACKED off
    try:
        general = E.ttm(t, m, mode, ctx=ctx)
    finally:
        E.check(E.lib.tp_set_global_option(2, E.ctypes.c_longlong(1)))
    assert np.array_equal(packed, general)
    want = ho.ttm(t, m, mode)
    assert np.max(np.abs(packed - want)) <= 64 * EPS * np.sqrt(dims[mode]) * np.max(np.abs(m)) * np.max(np.abs(t))


def test_ttm_linearity_and_identity(ctx):
    """Size-independent properties at a size the oracle would not finish quickly: identity and linearity."""
    dims = (96, 96, 96, 12)
    t = hostgen.random_tensor(dims, 3)
    for mode in range(4):
        eye = np.eye(dims[mode])
        assert np.array_equal(E.ttm(t, eye, mode, ctx=ctx), t)  # multiplying by exact 0/1 is exact
    a = hostgen.random_tensor([10, 96], 4)
    b = hostgen.random_tensor([10, 96], 5)
    lhs = E.ttm(t, a + b, 1, ctx=ctx)
    rhs = E.ttm(t, a, 1, ctx=ctx) + E.ttm(t, b, 1, ctx=ctx)
    assert np.max(np.abs(lhs - rhs)) <= 8 * 96 * EPS * np.max(np.abs(t)) * 4


def test_ttm_error_codes(ctx):
    t = hostgen.random_tensor((4, 3, 5), 2)
    assert code_of(lambda: E.ttm(t, np.eye(4), 1, ctx=ctx)) == Errc.shape_mismatch       # test_engine.cpp:134-135
    assert code_of(lambda: E.ttm(t, np.eye(4), 3, ctx=ctx)) == Errc.bad_mode
    assert code_of(lambda: E.ttm(t, np.eye(4), -1, ctx=ctx)) == Errc.bad_mode
    assert code_of(lambda: E.ttm(t, np.zeros((0, 3)), 1, ctx=ctx)) == Errc.shape_mismatch
    macs = [2 ** 64 - 10]
    assert code_of(lambda: E.ttm(t, np.eye(4), 0, macs, ctx=ctx)) == Errc.overflow


GRAM_SHAPES = [((6, 40), 0), ((40, 6), 1), ((5, 7, 3), 1), ((5, 7, 3), 0), ((5, 7, 3), 2), ((20, 200, 20), 1),
               ((200, 20, 20), 0), ((20, 20, 200), 2), ((10, 130, 33), 1), ((3, 65, 64), 1), ((10, 10, 96, 10), 2),
               ((129, 100), 0), ((100, 129), 1), ((8, 48, 8, 8), 1), ((400, 7, 11), 0), ((2, 2, 2, 2, 50), 4),
               # large leaves: 128 x 128 tiles on the TMA pipeline (>= 448 rows, >= 64 contraction chunks), all three
               # layouts, ragged last tile rows (1..4 live row blocks), ragged contraction ends, exact multiples
               ((3, 450, 400), 1), ((500, 40, 30), 0), ((1100, 452), 1), ((2, 600, 18, 30), 1), ((1040, 640), 1),
               ((4, 482, 262), 1), ((1030, 546), 1), ((2, 770, 520), 1), ((7, 1000, 150), 1),
               # many tile rows (16, 17 with two live rows in the last)
               ((2048, 1100), 0), ((1100, 2050), 1),
               # odd contiguous extent: stays on the 64 x 64 kernel
               ((3, 450, 401), 1), ((1100, 453), 1)]


@pytest.mark.parametrize("dims,mode", GRAM_SHAPES)
def test_gram_matches_oracle(ctx, dims, mode):
    t = hostgen.random_tensor(dims, 17 + mode)
    dt = E.DeviceTensor.upload(ctx, t)
    got = dt.gram(mode)
    dt.free()
    u = ho.unfold(t, mode)
    want = u @ u.T
    cols = u.shape[1]
    assert np.array_equal(got, got.T)                                   # full symmetric storage
    assert np.max(np.abs(got - want)) <= 64 * EPS * np.sqrt(cols) * np.max(np.abs(t)) ** 2 * np.sqrt(cols)


def test_truncated_basis(ctx):
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    v, _ = np.linalg.qr(rng.standard_normal((40, 6)))
    m = u @ np.diag([5, 4, 3, 2, 1, 0.5]) @ v.T
    uu = np.linalg.svd(m)[0]
    for k in range(1, 6):                                               # test_engine.cpp:138-155
        b, deg = E.leading_left_factors(m, k, ctx=ctx)
        assert not deg
        assert np.max(np.abs(b.T @ b - np.eye(k))) < 1e-9
        assert ho.projector_gap(b, uu[:, :k]) < 1e-9
        ob, _ = ho.leading_left_factors(m, k)
        assert np.max(np.abs(b - ob)) < 1e-9                            # same signs as the oracle
    b, _ = E.leading_left_factors(np.array([[0.0], [-3.0]]), 1, ctx=ctx)  # test_engine.cpp:157-162
    assert abs(b[0, 0]) < 1e-12 and abs(b[1, 0] - 1) < 1e-12
    a, _ = np.linalg.qr(rng.standard_normal((4, 3)))
    for k in (1, 2, 3):                                                 # Gram ignores the sign of the data
        assert np.array_equal(E.leading_left_factors(a, k, ctx=ctx)[0], E.leading_left_factors(-a, k, ctx=ctx)[0])
    d = np.diag([2.0, 1.0, 1.0])                                        # test_engine.cpp:172-176
    assert not E.leading_left_factors(d, 1, ctx=ctx)[1]
    assert E.leading_left_factors(d, 2, ctx=ctx)[1]
    eye = np.eye(3)                                                     # test_engine.cpp:178-188
    assert code_of(lambda: E.leading_left_factors(eye, 0, ctx=ctx)) == Errc.bad_argument
    assert code_of(lambda: E.leading_left_factors(eye, 4, ctx=ctx)) == Errc.bad_argument
    assert code_of(lambda: E.leading_left_factors(np.zeros((0, 0)), 1, ctx=ctx)) == Errc.shape_mismatch
    assert code_of(lambda: E.leading_left_factors(np.zeros((2049, 1)), 1, ctx=ctx)) == Errc.too_large


def test_random_start_and_exact_reconstruction(ctx):
    s = P.ProblemSpec([6, 5, 4], [3, 2, 2])                             # test_engine.cpp:190-204
    t = hostgen.random_tensor([6, 5, 4], 31)
    a = E.random_decomposition(t, s, 7, ctx=ctx)
    b = E.random_decomposition(t, s, 7, ctx=ctx)
    assert a.core.shape == (3, 2, 2)
    for n in range(3):
        assert np.max(np.abs(a.factors[n].T @ a.factors[n] - np.eye(s.K[n]))) < 1e-12
        assert np.array_equal(a.factors[n], b.factors[n])
    assert np.array_equal(a.core, b.core)                               # bit-reproducible reruns
    want = ho.core_from_factors(t, a.factors)
    assert np.max(np.abs(a.core - want)) < 1e-13
    s = P.ProblemSpec([4, 3, 5], [4, 3, 5])                             # test_engine.cpp:206-211
    t = hostgen.random_tensor([4, 3, 5], 13)
    d = E.random_decomposition(t, s, 5, ctx=ctx)
    assert E.reconstruction_error(t, d, ctx=ctx) < 1e-12


def test_readme_transcript_on_gpu(ctx, readme_kat):
    """proj/README.md:122-126 through the CUDA engine: Gauss-Seidel on the chain-input tree."""
    L, K = readme_kat["dims"], readme_kat["K"]
    s = P.ProblemSpec(L, K)
    t = hostgen.random_tensor(L, readme_kat["tensor_seed"])
    d = E.random_decomposition(t, s, readme_kat["init_seed"], ctx=ctx)
    assert "%.12f" % E.reconstruction_error(t, d, ctx=ctx) == readme_kat["start_error"]
    st = E.SweepStats()
    d = E.hooi_sweep(t, s, d, P.chain_tree(s), "gauss_seidel", st, ctx=ctx)
    assert "%.12f" % E.reconstruction_error(t, d, ctx=ctx) == readme_kat["sweep1_error"]
    assert st.tree_macs == readme_kat["tree_macs"] and st.peak_live == readme_kat["peak_live"]


def test_sweep_integer_goldens(ctx):
    L, K = [6, 5, 4], [3, 2, 2]                                         # test_engine.cpp:213-227
    s = P.ProblemSpec(L, K)
    t = hostgen.random_tensor(L, 41)
    d = E.random_decomposition(t, s, 1, ctx=ctx)
    for tree in (P.chain_tree(s), P.optimal_tree(s).tree):
        st = E.SweepStats()
        E.hooi_sweep(t, s, d, tree, "jacobi", st, ctx=ctx)
        assert st.tree_macs == P.tree_cost(tree, s).total_macs
    st = E.SweepStats()
    E.hooi_sweep(t, s, d, P.chain_tree(s), "gauss_seidel", st, ctx=ctx)
    assert st.tree_macs == 1296
    assert st.core_macs == 3 * 120 + 2 * 60 + 2 * 24
    s = P.ProblemSpec([5, 4, 3, 2], [2, 2, 2, 2])                       # test_engine.cpp:229-242
    t = hostgen.random_tensor(s.L, 3)
    d = E.random_decomposition(t, s, 9, ctx=ctx)
    cases = [(P.chain_tree(s), "jacobi"), (P.balanced_tree(s), "jacobi"), (P.optimal_tree(s).tree, "jacobi"),
             (P.chain_tree(s), "gauss_seidel")]
    for tree, kind in cases:
        st, ost = E.SweepStats(), ho.SweepStats()
        E.hooi_sweep(t, s, d, tree, kind, st, ctx=ctx)
        ho.hooi_sweep(t, s.L, s.K, d.factors, otree(tree), kind, ost)
        assert st.peak_live <= P.tree_depth(tree) + 1
        assert (st.tree_macs, st.core_macs, st.peak_live) == (ost.tree_macs, ost.core_macs, ost.peak_live)


def test_jacobi_tree_independence_and_gs_monotone(ctx):
    L, K = [8, 7, 6], [3, 3, 2]                                         # test_engine.cpp:244-271
    s = P.ProblemSpec(L, K)
    t = hostgen.random_tensor(L, 77)
    d = E.random_decomposition(t, s, 2, ctx=ctx)
    on_chain = E.hooi_sweep(t, s, d, P.chain_tree(s), "jacobi", ctx=ctx)
    for tree in (P.balanced_tree(s), P.optimal_tree(s).tree):
        other = E.hooi_sweep(t, s, d, tree, "jacobi", ctx=ctx)
        for n in range(3):
            assert ho.projector_gap(on_chain.factors[n], other.factors[n]) < 1e-9
    t = hostgen.random_tensor(L, 55)
    d = E.random_decomposition(t, s, 4, ctx=ctx)
    prev = E.reconstruction_error(t, d, ctx=ctx)
    for _ in range(6):
        d = E.hooi_sweep(t, s, d, P.chain_tree(s), "gauss_seidel", ctx=ctx)
        err = E.reconstruction_error(t, d, ctx=ctx)
        assert err <= prev + 1e-12
        prev = err


def test_sweep_error_codes(ctx):
    s = P.ProblemSpec([5, 4, 3], [2, 2, 2])                             # test_engine.cpp:273-300
    t = hostgen.random_tensor(s.L, 6)
    d = E.random_decomposition(t, s, 8, ctx=ctx)
    assert code_of(lambda: E.hooi_sweep(t, s, d, P.balanced_tree(s), "gauss_seidel", ctx=ctx)) == Errc.needs_chain_tree
    E.hooi_sweep(t, s, d, P.chain_tree(s), "gauss_seidel", ctx=ctx)
    short = E.Decomposition(d.core, d.factors[:-1])
    assert code_of(lambda: E.hooi_sweep(t, s, short, P.chain_tree(s), "jacobi", ctx=ctx)) == Errc.shape_mismatch
    wrong = hostgen.random_tensor([5, 4, 4], 6)
    assert code_of(lambda: E.random_decomposition(wrong, s, 1, ctx=ctx)) == Errc.shape_mismatch
    assert code_of(lambda: E.reconstruction_error(np.zeros((2, 2)), E.Decomposition(None, []), ctx=ctx)) == Errc.zero_tensor
    big = P.ProblemSpec([2049, 2], [2, 2])
    tree = P.optimal_tree(big).tree
    assert code_of(lambda: E.HooiPlan(ctx, big, tree, "jacobi")) == Errc.too_large


def run_both(ctx, cfg, sweeps, kind="jacobi", tree=None):
    """GPU (resident plan) and oracle on the same bits; returns per-sweep comparisons."""
    spec = cfg.spec
    tree = tree or P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, kind)
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    tnorm = ho.frobenius_norm(t)
    assert abs(dt.norm() - tnorm) <= 1e-13 * tnorm
    rows = []
    ocore = None
    for _ in range(sweeps):
        st = plan.sweep(dt)
        ost = ho.SweepStats()
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), kind, ost)
        gf = plan.get_factors()
        gcore = plan.get_core()
        assert (st.tree_macs, st.core_macs, st.peak_live, st.degenerate) == \
               (ost.tree_macs, ost.core_macs, ost.peak_live, ost.degenerate)
        assert not st.degenerate                      # a degenerate cut has no unique subspace to compare
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(gf, of))
        gn, on = np.sqrt(np.sum(gcore * gcore)), np.sqrt(np.sum(ocore * ocore))
        assert abs(plan.core_norm() - gn) <= 1e-13 * gn
        ofit = np.sqrt(max(tnorm ** 2 - on ** 2, 0.0)) / tnorm
        rows.append(dict(angle=angle, core_rel=abs(gn - on) / on, fit_gpu=plan.fit_from_norms(dt), fit_oracle=ofit))
    err_gpu = plan.reconstruction_error(dt)
    err_oracle = ho.reconstruction_error(t, ocore, of)
    plan.close()
    dt.free()
    return rows, err_gpu, err_oracle


SWEEP_CASES = [
    W.scaled_config(1, [40, 40, 40], [6, 6, 6], 3),
    W.scaled_config(2, [20, 20, 20, 20], [4, 4, 4, 4], 3),
    W.scaled_config(3, [40, 20, 20, 10], [8, 3, 5, 2], 3),
    W.scaled_config(4, [10, 10, 10, 10, 10], [3, 3, 3, 3, 3], 3),
    W.scaled_config(5, [130, 130, 130], [20, 20, 20], 2),
    W.scaled_config(3, [33, 17, 9, 5], [5, 2, 3, 1], 2),
]


@pytest.mark.parametrize("cfg", SWEEP_CASES, ids=lambda c: c.name)
def test_sweep_parity_small(ctx, cfg):
    """north_star bar: subspaces up to column sign, core norm and relative fit within 1e-10 relative, stats exact."""
    rows, err_gpu, err_oracle = run_both(ctx, cfg, cfg.iterations)
    for r in rows:
        assert r["angle"] < 1e-9                     # reference kProjectorTol (tolerances.hpp:17)
        assert r["core_rel"] < 1e-10
        assert abs(r["fit_gpu"] - r["fit_oracle"]) <= 1e-10 * max(r["fit_oracle"], 1e-3)
    assert abs(err_gpu - err_oracle) <= 1e-10 * max(err_oracle, 1e-3)


def test_sweep_parity_gauss_seidel(ctx):
    cfg = W.scaled_config(1, [30, 24, 18], [5, 4, 3], 3)
    rows, err_gpu, err_oracle = run_both(ctx, cfg, 3, "gauss_seidel", P.chain_tree(cfg.spec))
    for r in rows:
        assert r["angle"] < 1e-9 and r["core_rel"] < 1e-10
    assert abs(err_gpu - err_oracle) <= 1e-10 * max(err_oracle, 1e-3)


def test_sweep_parity_config1_full(ctx):
    """BASELINE.json configs[0] at full size (200^3 -> 20^3, 5 Jacobi iterations on the optimal tree)."""
    cfg = W.CONFIGS[1]
    rows, err_gpu, err_oracle = run_both(ctx, cfg, cfg.iterations)
    for r in rows:
        assert r["angle"] < 1e-9 and r["core_rel"] < 1e-10
        assert abs(r["fit_gpu"] - r["fit_oracle"]) <= 1e-10 * max(r["fit_oracle"], 1e-3)
    assert abs(err_gpu - err_oracle) <= 1e-10 * max(err_oracle, 1e-3)
    # converged to the noise floor sigma sqrt(|T|) / ||T|| (||X|| = ||G|| ~ sqrt(prod K))
    floor = cfg.sigma * np.sqrt(np.prod(cfg.L)) / np.sqrt(np.prod(cfg.K) + cfg.sigma ** 2 * np.prod(cfg.L))
    assert err_gpu < 1.05 * floor


def test_fast_eigensolve_is_certified_and_matches(ctx):
    """Leaves with L_n >= 256 take the top-k subspace-iteration path; its residual certificate must hold on the
    low-rank-plus-noise workload, and the factors must still be the oracle's (full eigen-decomposition)."""
    cfg = W.scaled_config(5, [768, 720, 704], [24, 20, 16], 3)
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    rejected = []
    ctx.set_option(2, 1)                          # certificate margins on stderr (shown if the test fails)
    for _ in range(cfg.iterations):
        st = plan.sweep(dt)
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi")
        eligible, rej = plan.evd_info()
        rejected.append(rej)
        assert not st.degenerate
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
        gn, on = plan.core_norm(), np.sqrt(np.sum(ocore * ocore))
        assert angle < 1e-9 and abs(gn - on) <= 1e-10 * on
        # individual vectors too (same sign rule), not just the subspace
        for a, b in zip(plan.get_factors(), of):
            assert np.max(np.abs(a - b)) < 1e-7
    ctx.set_option(2, 0)
    assert eligible == 3
    assert rejected[-1] == 0                      # warm-started sweeps are served by the fast path
    # the same sweeps with the fast path off give the same factors to rounding
    plan.set_fast_evd(False)
    plan.set_factors(f0)
    for _ in range(cfg.iterations):
        plan.sweep(dt)
    assert plan.evd_info()[0] == 0
    angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
    assert angle < 1e-9
    plan.close()
    dt.free()


@pytest.mark.parametrize("L,K,sweeps", [
    ([96, 96, 96, 96], [10, 10, 10, 10], 5),      # small leaves: single-launch Cholesky / Jacobi steps, graph replay
    ([200, 60, 45], [21, 9, 5], 5),               # odd block sizes (29, 17, 13)
    ([720, 240, 40], [106, 12, 10], 4),           # block 114 > 112: cuSOLVER potrf / syevd variant for mode 0
])
def test_fast_eigensolve_small_and_wide_blocks(ctx, L, K, sweeps):
    """Every eligible leaf takes the certified top-k path; from the third sweep on the recorded CUDA graph is what
    runs.  Factors must stay the oracle's (full eigen-decomposition) through all of them."""
    cfg = W.scaled_config(5, L, K, sweeps)
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    rejected = []
    for it in range(sweeps):
        st = plan.sweep(dt)
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi")
        eligible, rej = plan.evd_info()
        rejected.append(rej)
        assert not st.degenerate
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
        gn, on = plan.core_norm(), np.sqrt(np.sum(ocore * ocore))
        assert angle < 1e-9 and abs(gn - on) <= 1e-10 * on, (it, angle, rejected)
        for a, b in zip(plan.get_factors(), of):
            assert np.max(np.abs(a - b)) < 1e-7
    assert eligible == len(L)
    assert rejected[-1] == 0 and rejected[-2] == 0
    plan.close()
    dt.free()


def test_fast_eigensolve_falls_back_without_a_gap(ctx):
    """A plain random tensor has no spectral gap: the certificate fails, the full solve takes over, parity holds."""
    L, K = [800, 24, 20], [12, 5, 4]
    spec = P.ProblemSpec(L, K)
    tree = P.optimal_tree(spec).tree
    t = hostgen.random_tensor(L, 99)
    f0 = hostgen.random_orthonormal_factors(L, K, 98)
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    for it in range(3):
        plan.sweep(dt)
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi")
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
        assert angle < 1e-9, (it, angle, plan.evd_info())
        gn, on = plan.core_norm(), np.sqrt(np.sum(ocore * ocore))
        assert abs(gn - on) <= 1e-10 * on
    plan.close()
    dt.free()


CARRY_CASES = [
    ([40, 36, 30], [6, 5, 4]),
    ([20, 18, 16, 14], [4, 3, 3, 2]),
    ([12, 10, 9, 8, 7], [3, 2, 2, 2, 2]),
    ([300, 8], [3, 3]),
]


@pytest.mark.parametrize("L,K", CARRY_CASES, ids=lambda v: "x".join(map(str, v)))
@pytest.mark.parametrize("tree_kind", ["optimal", "chain", "balanced"])
def test_carried_path_is_bit_identical_and_invalidates(ctx, L, K, tree_kind):
    """TP_OPT_CARRY_PATH only removes recomputation: with it on (default) or off, sweeps give the same bits; changing
    the tensor or the factors between sweeps drops the carried products."""
    cfg = W.scaled_config(1, L, K, 4)
    spec = cfg.spec
    tree = {"optimal": lambda: P.optimal_tree(spec).tree, "chain": lambda: P.chain_tree(spec),
            "balanced": lambda: P.balanced_tree(spec)}[tree_kind]()
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)

    def run(carry, fast):
        plan = E.HooiPlan(ctx, spec, tree, "jacobi")
        plan.set_carry_path(carry)
        plan.set_fast_evd(fast)
        plan.set_factors(f0)
        out = []
        for _ in range(4):
            plan.sweep(dt)
            out.append((plan.get_factors(), plan.get_core()))
        plan.close()
        return out

    for fast in (False, True):
        on, off = run(True, fast), run(False, fast)
        for (fa, ca), (fb, cb) in zip(on, off):
            assert all(np.array_equal(a, b) for a, b in zip(fa, fb))
            assert np.array_equal(ca, cb)

    # against the oracle through a change of tensor and a reset of the factors in mid-run
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    t2 = t.copy()
    noise = hostgen.random_tensor(L, 4242)
    for it in range(6):
        if it == 2:                                  # T <- T + 0.05 E on the device and on the host
            dn = E.DeviceTensor.upload(ctx, noise)
            dt.axpby(1.0, 0.05, dn)
            dn.free()
            t2 = t2 + 0.05 * noise
        if it == 4:
            plan.set_factors(f0)
            of = [f.copy() for f in f0]
        plan.sweep(dt)
        ocore, of = ho.hooi_sweep(t2, spec.L, spec.K, of, otree(tree), "jacobi")
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
        gn, on_ = plan.core_norm(), np.sqrt(np.sum(ocore * ocore))
        assert angle < 1e-9 and abs(gn - on_) <= 1e-10 * on_, (it, angle)
        err = plan.reconstruction_error(dt)
        assert abs(err - ho.reconstruction_error(t2, ocore, of)) <= 1e-10 * max(err, 1e-3)
    plan.close()
    dt.free()


@pytest.mark.parametrize("L,K", [([96, 80, 64], [10, 8, 6]), ([40, 36, 30, 24], [5, 4, 4, 3]), ([300, 8], [3, 3]), ([50], [1])],
                         ids=lambda v: "x".join(map(str, v)))
def test_gauss_seidel_with_carried_chain_and_certified_solve(ctx, L, K):
    """Gauss-Seidel (hooi.hpp:206-225) takes the same two shortcuts as Jacobi: the first chain of a sweep is the one
    the previous sweep's core chain computed, and eligible leaves use the certified top-k solve (checked right after
    each leaf, because the next chain multiplies by the new factor).  Bits do not depend on the carried chain; the
    factors stay the oracle's."""
    cfg = W.scaled_config(1, L, K, 4)
    spec = cfg.spec
    tree = P.chain_tree(spec)
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)

    def run(carry):
        plan = E.HooiPlan(ctx, spec, tree, "gauss_seidel")
        plan.set_carry_path(carry)
        plan.set_factors(f0)
        out = []
        for _ in range(4):
            st = plan.sweep(dt)
            out.append((plan.get_factors(), plan.get_core(), st, plan.evd_info()))
        plan.close()
        return out

    on, off = run(True), run(False)
    of = [f.copy() for f in f0]
    for (fa, ca, st, info), (fb, cb, _, _) in zip(on, off):
        assert all(np.array_equal(a, b) for a, b in zip(fa, fb)) and np.array_equal(ca, cb)
        ost = ho.SweepStats()
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "gauss_seidel", ost)
        assert (st.tree_macs, st.core_macs, st.peak_live, st.degenerate) == \
               (ost.tree_macs, ost.core_macs, ost.peak_live, ost.degenerate)
        angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(fa, of))
        gn, on_ = np.sqrt(np.sum(ca * ca)), np.sqrt(np.sum(ocore * ocore))
        assert angle < 1e-9 and abs(gn - on_) <= 1e-10 * on_
    if L == [96, 80, 64]:
        assert on[-1][3] == (3, 0)                 # all three leaves eligible, none redone in the last sweep
    # a change of the tensor between sweeps drops the carried chain
    plan = E.HooiPlan(ctx, spec, tree, "gauss_seidel")
    plan.set_factors(f0)
    plan.sweep(dt)
    noise = hostgen.random_tensor(L, 77)
    dn = E.DeviceTensor.upload(ctx, noise)
    dt.axpby(1.0, 0.1, dn)
    dn.free()
    plan.sweep(dt)
    t2 = t + 0.1 * noise
    of = [f.copy() for f in f0]
    _, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "gauss_seidel")
    ocore, of = ho.hooi_sweep(t2, spec.L, spec.K, of, otree(tree), "gauss_seidel")
    assert max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of)) < 1e-9
    assert abs(plan.core_norm() - np.sqrt(np.sum(ocore * ocore))) <= 1e-10 * np.sqrt(np.sum(ocore * ocore))
    plan.close()
    dt.free()


STREAM_CASES = [
    ([160, 24, 20], [6, 5, 4], "optimal"),          # 3 modes: one root child contracts mode 0, one does not
    ([130, 12, 10, 8], [5, 3, 3, 2], "optimal"),    # ragged last slab (130 rows in slabs of 32)
    ([96, 20, 18], [5, 4, 3], "chain"),             # chain tree: N root children, the first non-mode-0 one streams
    ([64, 30], [4, 4], "optimal"),
    ([200, 16, 14], [7, 4, 3], "balanced"),
]


@pytest.mark.parametrize("L,K,tree_kind", STREAM_CASES, ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
@pytest.mark.parametrize("kind", ["jacobi", "gauss_seidel"])
def test_by_value_call_with_streamed_upload(ctx, monkeypatch, L, K, tree_kind, kind):
    """tp_hooi_sweep_host uploads large tensors in slabs of the first mode and starts the root products on the slabs
    that have arrived.  Forced on here for small tensors; results must be the oracle's, and equal to rounding to the
    whole-tensor upload (the mode-0 root product is then a sum of per-slab partial products)."""
    if kind == "gauss_seidel" and tree_kind != "chain":
        pytest.skip("Gauss-Seidel needs a chain tree")
    cfg = W.scaled_config(1, L, K, 2)
    spec = cfg.spec
    tree = {"optimal": lambda: P.optimal_tree(spec).tree, "chain": lambda: P.chain_tree(spec),
            "balanced": lambda: P.balanced_tree(spec)}[tree_kind]()
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)

    def run(min_bytes):
        ctx.set_option(1, min_bytes)   # TP_CTX_OPT_STREAMED_UPLOAD_MIN_BYTES
        d = E.Decomposition(None, [f.copy() for f in f0])
        stats = E.SweepStats()
        for _ in range(2):
            d = E.hooi_sweep(t, spec, d, tree, kind, stats, ctx=ctx)
        return d, stats

    streamed, st = run(0)
    whole, _ = run(1 << 60)
    ctx.set_option(1, 256 << 20)       # back to the default
    of = [f.copy() for f in f0]
    for _ in range(2):
        ost = ho.SweepStats()
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), kind, ost)
    assert (st.tree_macs, st.core_macs, st.peak_live, st.degenerate) == \
           (ost.tree_macs, ost.core_macs, ost.peak_live, ost.degenerate)
    for d in (streamed, whole):
        assert max(ho.sin_largest_principal_angle(a, b) for a, b in zip(d.factors, of)) < 1e-9
        gn, on = np.sqrt(np.sum(d.core * d.core)), np.sqrt(np.sum(ocore * ocore))
        assert abs(gn - on) <= 1e-10 * on
        assert abs(E.reconstruction_error(t, d, ctx=ctx) - ho.reconstruction_error(t, ocore, of)) <= 1e-10
    for a, b in zip(streamed.factors, whole.factors):
        assert np.max(np.abs(a - b)) < 1e-10
    if kind == "gauss_seidel":                      # nothing is streamed there: same bits
        assert all(np.array_equal(a, b) for a, b in zip(streamed.factors, whole.factors))


def _random_specs(count, seed):
    """Seeded random problems: 2-5 modes, odd and even extents, K_n = 1 allowed, every leaf with full rank
    (K_n <= prod of the other K, else both sides flag a degenerate cut)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.integers(2, 6))
        L = [int(rng.integers(2, 26 if n < 5 else 12)) for _ in range(n)]
        K = [int(rng.integers(1, min(l, 9) + 1)) for l in L]
        if any(K[m] > np.prod([K[j] for j in range(n) if j != m]) for m in range(n)):
            continue
        out.append((L, K, ["optimal", "chain", "chain_by_cost", "balanced"][int(rng.integers(0, 4))],
                    ["jacobi", "gauss_seidel"][int(rng.integers(0, 2))]))
    return out


@pytest.mark.parametrize("L,K,tree_kind,kind", _random_specs(24, 20261020),
                         ids=lambda v: v if isinstance(v, str) else "x".join(map(str, v)))
def test_sweep_parity_random_specs(ctx, L, K, tree_kind, kind):
    """Three sweeps of a seeded random problem on a random tree strategy and schedule, resident plan vs oracle."""
    cfg = W.scaled_config(3, L, K, 3)
    spec = cfg.spec
    if kind == "gauss_seidel" and tree_kind in ("optimal", "balanced"):
        tree_kind = "chain"
    tree = {"optimal": lambda: P.optimal_tree(spec).tree, "chain": lambda: P.chain_tree(spec),
            "chain_by_cost": lambda: P.chain_tree(spec, P.CHAIN_BY_COST), "balanced": lambda: P.balanced_tree(spec)}[tree_kind]()
    rows, err_gpu, err_oracle = run_both(ctx, cfg, 3, kind, tree)
    for r in rows:
        assert r["angle"] < 1e-9 and r["core_rel"] < 1e-10
        assert abs(r["fit_gpu"] - r["fit_oracle"]) <= 1e-10 * max(r["fit_oracle"], 1e-3)
    assert abs(err_gpu - err_oracle) <= 1e-10 * max(err_oracle, 1e-3)


@pytest.mark.parametrize("index", [2, 3, 4])
def test_sweep_parity_full_size_configs(ctx, index):
    """BASELINE.json configs[1..3] at full size, ALL of their 10 Jacobi iterations on the optimal tree, against the
    oracle after every iteration: the cold first sweep, the warm-started certified solves, and (from the third warm
    sweep on) the replayed whole-sweep graph are all inside the compared range."""
    cfg = W.CONFIGS[index]
    rows, err_gpu, err_oracle = run_both(ctx, cfg, cfg.iterations)
    assert len(rows) == 10
    for r in rows:
        assert r["angle"] < 1e-9 and r["core_rel"] < 1e-10
        assert abs(r["fit_gpu"] - r["fit_oracle"]) <= 1e-10 * max(r["fit_oracle"], 1e-3)
    assert abs(err_gpu - err_oracle) <= 1e-10 * max(err_oracle, 1e-3)


def test_config5_full_size_against_oracle(ctx):
    """BASELINE.json configs[4] (1600^3 -> 100^3, 33 GB) against the oracle for three iterations from the start
    factors (5 s of 16-core NumPy each): the third runs on warm-started Ritz vectors, the recorded leaf-solve graphs
    and the carried core chain, i.e. the state the benchmark's timed region is in."""
    import bench as B
    cfg = W.CONFIGS[5]
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    total = int(np.prod(cfg.L, dtype=np.int64))
    host, handle = B.pinned_array(total)
    try:
        dt = B.build_on_gpu(ctx, cfg, host, 16)
        t = host.reshape(cfg.L)
        tnorm2 = float(np.dot(host, host))
        plan = E.HooiPlan(ctx, spec, tree, "jacobi")
        f0 = W.start_factors(cfg)
        plan.set_factors(f0)
        of = [f.copy() for f in f0]
        for it in range(3):
            st = plan.sweep(dt)
            ost = ho.SweepStats()
            ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi", ost)
            assert (st.tree_macs, st.core_macs, st.peak_live, st.degenerate) == \
                   (ost.tree_macs, ost.core_macs, ost.peak_live, ost.degenerate)
            angle = max(ho.sin_largest_principal_angle(a, b) for a, b in zip(plan.get_factors(), of))
            gn, on = plan.core_norm(), float(np.sqrt(np.sum(ocore * ocore)))
            ofit = np.sqrt(max(tnorm2 - on * on, 0.0) / tnorm2)
            assert angle < 1e-9, (it, angle)
            assert abs(gn - on) <= 1e-10 * on, (it, gn, on)
            assert abs(plan.fit_from_norms(dt) - ofit) <= 1e-10 * max(ofit, 1e-3), it
        assert plan.evd_info()[1] == 0          # no leaf had to be redone with the full solve
        plan.close()
        dt.free()
    finally:
        from paper_1707_05594_b200._lib import lib
        lib.tp_host_free(handle)


@pytest.mark.parametrize("cfg", [W.CONFIGS[1], W.scaled_config(2, [40, 36, 32, 28], [6, 5, 4, 3], 8),
                                 W.scaled_config(3, [240, 60, 60, 40], [30, 5, 10, 3], 8)], ids=lambda c: c.name)
def test_visiting_order_of_the_carried_subtree_does_not_change_the_factors(ctx, cfg):
    """TP_GLOBAL_OPT_CARRY_FIRST: a Jacobi sweep gives the same factors whichever subtree is walked first and whichever
    root-to-leaf path is carried (hooi.hpp:9-12: every product uses the start-of-sweep factors) -- bit for bit, since
    every node is still computed by the same kernel from the same operands."""
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    trails = {}
    try:
        for first in (0, 1):
            E.check(E.lib.tp_set_global_option(6, E.ctypes.c_longlong(first)))   # plans created from now on
            plan = E.HooiPlan(ctx, spec, tree, "jacobi")
            plan.set_factors(f0)
            trail = []
            for _ in range(6):
                plan.sweep(dt)
                trail.append((plan.get_factors(), plan.get_core()))
            trails[first] = trail
            plan.close()
    finally:
        E.check(E.lib.tp_set_global_option(6, E.ctypes.c_longlong(2)))
    for i, ((fa, ca), (fb, cb)) in enumerate(zip(trails[0], trails[1])):
        for a, b in zip(fa, fb):
            assert np.array_equal(a, b), i
        # the core is contracted along the carried path, which differs between the two plans: same value to rounding
        assert np.max(np.abs(ca - cb)) <= 1e-12 * np.max(np.abs(ca)), i
    dt.free()


@pytest.mark.parametrize("cfg", [W.CONFIGS[1], W.scaled_config(2, [40, 36, 32, 28], [6, 5, 4, 3], 8),
                                 W.scaled_config(3, [240, 60, 60, 40], [30, 5, 10, 3], 8)], ids=lambda c: c.name)
def test_whole_sweep_graph_is_bit_identical(ctx, cfg):
    """TP_OPT_SWEEP_GRAPH: the steady-state sweep replayed as one CUDA graph launches the same kernels with the same
    arguments as the eager sweep, so factors and core must agree bit for bit, sweep by sweep; and both match the
    oracle."""
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    sweeps = 8
    results = {}
    for mode in (0, 1):
        plan = E.HooiPlan(ctx, spec, tree, "jacobi")
        plan.set_sweep_graph(mode)
        plan.set_factors(f0)
        trail = []
        for _ in range(sweeps):
            st = plan.sweep(dt)
            trail.append((plan.get_factors(), plan.get_core(), st))
        results[mode] = trail
        replayed, one_launch = plan.sweep_info()
        assert replayed == (mode == 1)          # every leaf of these cases is eligible for a capturable fast solve
        if mode == 1:
            # the replayed sweeps report only their total device time
            tm = plan.last_timing()
            assert tm["total_ms"] > 0 and tm["tree_ms"] == 0
        plan.close()
    of = [f.copy() for f in f0]
    for i in range(sweeps):
        (fa, ca, sa), (fb, cb, sb) = results[0][i], results[1][i]
        for a, b in zip(fa, fb):
            assert np.array_equal(a, b), i
        assert np.array_equal(ca, cb), i
        assert (sa.tree_macs, sa.core_macs, sa.peak_live, sa.degenerate) == (sb.tree_macs, sb.core_macs, sb.peak_live, sb.degenerate)
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi", None)
        assert max(ho.sin_largest_principal_angle(a, b) for a, b in zip(fb, of)) < 1e-9
        on = float(np.sqrt(np.sum(ocore * ocore)))
        assert abs(float(np.sqrt(np.sum(cb * cb))) - on) <= 1e-10 * on
    dt.free()


@pytest.mark.parametrize("graph", [0, 1], ids=["eager", "graph"])
@pytest.mark.parametrize("cfg", [W.scaled_config(1, [64, 56, 48], [8, 6, 5], 6),
                                 W.scaled_config(2, [40, 36, 32, 28], [6, 5, 4, 3], 6),
                                 W.scaled_config(4, [24, 24, 24, 22, 20], [3, 3, 2, 2, 2], 6)], ids=lambda c: c.name)
def test_forked_subtrees_are_bit_identical(ctx, cfg, graph):
    """TP_OPT_FORK_SUBTREES: sibling subtrees on streams of their own (one output buffer per node) run the same
    kernels on the same data as the one-stream walk, so factors and core agree bit for bit, sweep by sweep, eager and
    as a replayed graph; repeated runs of the forked walk are bit-identical too (no race between the branches)."""
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    t = W.build_tensor_host(cfg)
    f0 = W.start_factors(cfg)
    dt = E.DeviceTensor.upload(ctx, t)
    sweeps = 6
    trails = []
    for fork in (0, 1, 1):
        plan = E.HooiPlan(ctx, spec, tree, "jacobi")
        plan.set_sweep_graph(graph)
        plan.set_fork_subtrees(fork)
        plan.set_factors(f0)
        trail = []
        for _ in range(sweeps):
            plan.sweep(dt)
            trail.append((plan.get_factors(), plan.get_core()))
        assert plan.sweep_info()[0] == (graph == 1)
        trails.append(trail)
        plan.close()
    for i in range(sweeps):
        for other in trails[1:]:
            for a, b in zip(trails[0][i][0], other[i][0]):
                assert np.array_equal(a, b), i
            assert np.array_equal(trails[0][i][1], other[i][1]), i
    of = [f.copy() for f in f0]
    for i in range(sweeps):
        ocore, of = ho.hooi_sweep(t, spec.L, spec.K, of, otree(tree), "jacobi", None)
    assert max(ho.sin_largest_principal_angle(a, b) for a, b in zip(trails[1][-1][0], of)) < 1e-9
    dt.free()


def test_small_spectral_gap_parity(ctx):
    """A tensor whose mode-0 Gram matrix has lambda_K / lambda_{K+1} - 1 = 1e-6: not degenerate by the reference's
    1e-10 rule, but too close for a residual-only certificate (angle error ~ residual / gap).  The gap-aware
    certificate must hand this leaf to the full eigen-solve, and the factors must still match the oracle."""
    rng = np.random.default_rng(77)
    L, K = [60, 30, 24], [4, 3, 3]
    spec = P.ProblemSpec(L, K)
    tree = P.optimal_tree(spec).tree
    # T = sum_j s_j a_j (x) B_j with orthonormal a_j and orthonormal (flattened) B_j: mode-0 Gram = A diag(s^2) A^T
    a, _ = np.linalg.qr(rng.standard_normal((L[0], 12)))
    bmat, _ = np.linalg.qr(rng.standard_normal((L[1] * L[2], 12)))
    s2 = np.array([9.0, 7.0, 5.0, 3.0, 3.0 * (1 - 1e-6), 1e-2, 1e-2, 1e-3, 1e-3, 1e-3, 1e-4, 1e-4])
    t = np.ascontiguousarray(((a * np.sqrt(s2)) @ bmat.T).reshape(L))
    f0 = hostgen.random_orthonormal_factors(L, K, 5)
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    # start from factors that keep the other modes complete enough for the mode-0 leaf to see the full spectrum
    plan.set_factors(f0)
    of = [f.copy() for f in f0]
    for _ in range(3):
        st = plan.sweep(dt)
        ost = ho.SweepStats()
        ocore, of = ho.hooi_sweep(t, L, K, of, otree(tree), "jacobi", ost)
        assert st.degenerate == ost.degenerate
    gf = plan.get_factors()
    w = np.linalg.eigvalsh(ho.unfold(ho.ttm(ho.ttm(t, of[1].T, 1), of[2].T, 2), 0) @ ho.unfold(ho.ttm(ho.ttm(t, of[1].T, 1), of[2].T, 2), 0).T)[::-1]
    rel_gap = (w[K[0] - 1] - w[K[0]]) / w[0]
    # only meaningful where the projected problem still has the tiny gap; then parity must hold at the bar
    if 1e-9 < rel_gap < 1e-4:
        assert ho.sin_largest_principal_angle(gf[0], of[0]) < 1e-9
    for m in (1, 2):
        assert ho.sin_largest_principal_angle(gf[m], of[m]) < 1e-9
    plan.close()
    dt.free()


def test_config5_full_size_properties(ctx):
    """BASELINE.json configs[4] (1600^3 -> 100^3, 33 GB) is too large for the oracle inside a unit test, so the full
    size is pinned by size-independent properties: TTM linearity on the real tensor, orthonormal factors, the fit
    reaching the noise floor, ||core||^2 + ||residual||^2 = ||T||^2, exact SweepStats, bit-identical reruns."""
    import bench as B
    cfg = W.CONFIGS[5]
    spec = cfg.spec
    tree = P.optimal_tree(spec).tree
    total = int(np.prod(cfg.L, dtype=np.int64))
    host, handle = B.pinned_array(total)
    try:
        dt = B.build_on_gpu(ctx, cfg, host, 16)
        plan = E.HooiPlan(ctx, spec, tree, "jacobi")
        f0 = W.start_factors(cfg)
        runs = []
        for rerun in range(2):
            plan.set_factors(f0)
            for _ in range(2):
                st = plan.sweep(dt)
            runs.append((plan.get_factors(), plan.get_core()))
        assert st.tree_macs == 896000000000 and st.peak_live == 3 and not st.degenerate
        assert st.core_macs == 100 * 1600 ** 3 + 100 * 100 * 1600 ** 2 + 100 * 100 * 100 * 1600
        for a, b in zip(runs[0][0], runs[1][0]):
            assert np.array_equal(a, b)                      # reruns are bit-identical
        assert np.array_equal(runs[0][1], runs[1][1])
        for f, k in zip(runs[0][0], spec.K):
            assert np.max(np.abs(f.T @ f - np.eye(k))) < 1e-12
        fit = plan.fit_from_norms(dt)
        floor = cfg.sigma * np.sqrt(float(total)) / np.sqrt(np.prod(cfg.K) + cfg.sigma ** 2 * float(total))
        assert abs(fit - floor) < 0.02 * floor               # converged to the noise floor (0.0638)
        tn, gn = dt.norm(), plan.core_norm()
        assert abs(fit - np.sqrt(max(tn * tn - gn * gn, 0.0)) / tn) < 1e-12
        # linearity of the mode product on the full tensor: T x_1 (A + B) = T x_1 A + T x_1 B (first slabs compared)
        a = hostgen.random_tensor([5, 1600], 11)
        b = hostgen.random_tensor([5, 1600], 12)
        za, zb, zab = dt.ttm(a, 1), dt.ttm(b, 1), dt.ttm(a + b, 1)
        za.axpby(1.0, 1.0, zb)
        zab.axpby(1.0, -1.0, za)
        assert zab.norm() <= 1e-13 * za.norm()
        for z in (za, zb, zab):
            z.free()
        plan.close()
        dt.free()
    finally:
        from paper_1707_05594_b200._lib import lib
        lib.tp_host_free(handle)


# shapes with enough columns to take the warp-specialised TMA kernel (>= 148 wide tiles), awkward extents included
TMA_SHAPES = [
    ((3, 50, 40000), 1, 5), ((50, 40002), 0, 7), ((40010, 50), 1, 20), ((130, 18, 300), 1, 13),
    ((2, 770, 20000), 1, 24), ((96, 90, 704), 0, 24), ((24, 720, 704), 1, 20), ((24, 20, 704, 60), 2, 16),
    ((2500, 16, 18), 1, 8), ((38000, 34), 1, 10), ((38001, 34), 1, 33), ((5, 36, 9000), 1, 100),
    ((3, 40, 8, 1250), 1, 41), ((4, 17, 10000), 1, 104), ((4, 18, 10000), 1, 110), ((60000, 20), 1, 3),
    # several tiles per persistent CTA
    ((100000, 64), 1, 16), ((3, 64, 70000), 1, 10), ((200000, 32), 1, 5), ((20, 48, 30000), 1, 13), ((300000, 20), 1, 24),
    ((7, 33, 50000), 1, 100),
    # last row tile at most half full (K <= 8 (KT - 1) + 4 for KT = 6, 8, 10, 13), both layouts, ragged extents
    ((40010, 50), 1, 100), ((38001, 34), 1, 97), ((38000, 36), 1, 44), ((60000, 20), 1, 58), ((3, 40, 20000), 1, 75),
    ((30002, 40), 1, 90), ((5, 36, 9002), 1, 99), ((2, 24, 18, 1300), 1, 42),
]


@pytest.mark.parametrize("dims,mode,new_len", TMA_SHAPES)
def test_ttm_tma_path_matches_oracle(ctx, dims, mode, new_len):
    seed = (sum(dims) * 17 + mode * 5 + new_len) % 10000
    t = hostgen.random_tensor(dims, seed)
    m = hostgen.random_tensor([new_len, dims[mode]], seed + 1)
    got = E.ttm(t, m, mode, ctx=ctx)
    want = ho.ttm(t, m, mode)
    bad = np.argwhere(np.abs(got - want) > 64 * EPS * np.sqrt(dims[mode]) * np.max(np.abs(m)) * np.max(np.abs(t)))
    assert bad.size == 0, (len(bad), bad[:5].tolist(), bad[-3:].tolist())


def test_tma_kernel_is_stable_under_concurrent_kernels(ctx):
    """Regression: the warp-specialised TMA kernel reads its stages with generic-proxy loads; without a
    fence.proxy.async before a stage is handed back, a TMA refill could overtake those reads as soon as other
    kernels shared the SMs (stale 128-byte box rows).  Run it beside unrelated fill kernels and compare with the
    cp.async kernel's result."""
    import os
    import torch
    from paper_1707_05594_b200 import distributed as D
    ops = D.GpuOps(ctx)
    big = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    side = torch.cuda.Stream()
    for dims, k in (((276480, 352), 16), ((384, 360, 352), 20)):
        x = hostgen.random_tensor(dims, 1)
        f = np.asfortranarray(hostgen.random_tensor([k, dims[1]], 2).T).reshape(-1, order="F")
        xb, fb = ops.from_host(x), ops.from_host(f)
        E.check(E.lib.tp_set_global_option(1, E.ctypes.c_longlong(0)))   # TP_GLOBAL_OPT_TTM_TMA off
        try:
            ref = ops.to_host(ops.ttm_partial(xb, list(dims), 1, fb, dims[1], 0, k, [0, k]))
        finally:
            E.check(E.lib.tp_set_global_option(1, E.ctypes.c_longlong(1)))
        for _ in range(5):
            ctx.synchronize()
            torch.cuda.synchronize()
            z = ops.ttm_partial(xb, list(dims), 1, fb, dims[1], 0, k, [0, k])
            with torch.cuda.stream(side):
                for _ in range(30):
                    big.zero_()
            got = ops.to_host(z)
            torch.cuda.synchronize()
            assert np.max(np.abs(got - ref)) <= 64 * EPS * np.sqrt(dims[1]) * np.max(np.abs(f)) * np.max(np.abs(x))


@pytest.mark.parametrize("L,K,order", [([40, 36, 32], [6, 5, 4], None), ([40, 36, 32], [6, 5, 4], [2, 0, 1]),
                                       ([20, 18, 16, 14], [4, 3, 3, 2], None), ([64, 48], [5, 5], [1, 0]),
                                       ([9, 8, 7, 6, 5], [3, 2, 2, 2, 2], None)],
                         ids=lambda v: "x".join(map(str, v)) if v is not None else "natural")
def test_sthosvd_start_matches_the_published_algorithm(ctx, L, K, order):
    """tp_sthosvd against the NumPy restatement of sequentially truncated HOSVD (oracle/hooi_oracle.py::sthosvd): same
    subspaces, same core up to rounding, orthonormal factors, the error bound of the method, and a better start for
    HOOI than random factors."""
    cfg = W.scaled_config(3, L, K, 2)
    spec = cfg.spec
    t = W.build_tensor_host(cfg)
    d, deg = E.sthosvd(t, spec, order, ctx=ctx)
    ocore, ofac, odeg = ho.sthosvd(t, K, order)
    assert deg == odeg == False
    for a, b, k in zip(d.factors, ofac, K):
        assert ho.sin_largest_principal_angle(a, b) < 1e-9
        assert np.max(np.abs(a.T @ a - np.eye(k))) < 1e-12
        assert np.max(np.abs(a - b)) < 1e-7                 # same sign rule: the vectors themselves agree
    assert np.max(np.abs(d.core - ocore)) <= 1e-9 * np.max(np.abs(ocore))
    err = E.reconstruction_error(t, d, ctx=ctx)
    assert abs(err - ho.reconstruction_error(t, ocore, ofac)) <= 1e-10
    # resident form: the plan starts from the same factors, and one HOOI sweep from there beats one from random factors
    tree = P.optimal_tree(spec).tree
    dt = E.DeviceTensor.upload(ctx, t)
    plan = E.HooiPlan(ctx, spec, tree, "jacobi")
    plan.init_sthosvd(dt, order)
    for a, b in zip(plan.get_factors(), d.factors):
        assert np.array_equal(a, b)
    assert np.array_equal(plan.get_core(), d.core)
    assert abs(plan.fit_from_norms(dt) - err) < 1e-12
    plan.sweep(dt)
    after_sthosvd = plan.fit_from_norms(dt)
    plan.set_factors(W.start_factors(cfg))
    plan.sweep(dt)
    after_random = plan.fit_from_norms(dt)
    assert after_sthosvd <= err + 1e-12 and after_sthosvd <= after_random + 1e-12
    plan.close()
    dt.free()
    with pytest.raises(TuckerplanError) as bad:
        E.sthosvd(t, spec, [0] * len(L), ctx=ctx)
    assert bad.value.code == Errc.bad_argument
