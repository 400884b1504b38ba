"""Device sweeps vs the reference CPU oracle on identical seeded inputs.

Parity contract: identical ranks; |RSE_gpu - RSE_ref| <= 1e-10
(absolute difference of relative errors); kept-block diagonal | |T_ii|_gpu - |T_ii|_ref |
<= 1e-10 |T_00| for every cut.
"""
import math

import numpy as np
import pytest

from tests.fixtures import cfg1, planted_plus_noise, shifted_hilbert
from tests.replay import replay

pytestmark = pytest.mark.gpu

TOL_RSE = 1e-10
TOL_DIAG = 1e-10


def _check_parity(dev, ref, a, dims, method, ranks=None, eps=None, qlp="early_exit"):
    sweep = "l2r" if method == "ulv" else "r2l"
    res = dev.decompose_device(a, dims, method, sweep, ranks=ranks, eps=eps, qlp=qlp)
    rep = res.report()
    gpu_rse = res.rse(a)
    rr = ref.decompose(a, dims, method, sweep, ranks=ranks, eps=eps or 0.0)
    ref_rse = ref.rse(rr, a, dims)
    assert rep.ranks_chosen == rr.ranks_chosen
    assert abs(gpu_rse - ref_rse) <= TOL_RSE, (gpu_rse, ref_rse)
    cuts = replay(ref, a, dims, method, ranks=ranks, eps=eps)
    for c, (g, r) in enumerate(zip(rep.cuts, cuts)):
        assert g["rank"] == r["rank"]
        scale = r["diag"][0]
        assert np.max(np.abs(g["diag"] - r["diag"])) <= TOL_DIAG * scale, (c, g["diag"], r["diag"])
    return res, rep, rr, gpu_rse, ref_rse


@pytest.mark.parametrize("method", ["urv", "ulv"])
@pytest.mark.parametrize("qlp", ["early_exit", "full"])
def test_cfg1_fixed_rank(dev, ref, method, qlp):
    a, dims, ranks = cfg1(ref)
    _, rep, rr, g, r = _check_parity(dev, ref, a, dims, method, ranks=ranks, qlp=qlp)
    assert rep.ranks_chosen == ranks
    # the reference's TT-SVD check (BASELINE config 1): within 2x of TT-SVD's RSE
    svd = ref.decompose(a, dims, "svd", "l2r", ranks=ranks)
    assert g <= 2.0 * ref.rse(svd, a, dims)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_cfg1_tolerance_wellposed(dev, ref, method):
    a, dims, _ = cfg1(ref)
    _, rep, *_ = _check_parity(dev, ref, a, dims, method, eps=1e-6)
    assert rep.ranks_chosen == [1, 5, 5, 5, 1]


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_planted_order6_fixed(dev, ref, method):
    dims, ranks = [6] * 6, [1, 4, 5, 5, 5, 4, 1]
    a = planted_plus_noise(ref, dims, ranks, 3, 1e-4)
    _check_parity(dev, ref, a, dims, method, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_hilbert_small_tolerance(dev, ref, method):
    dims = [10] * 4
    a = shifted_hilbert(dims)
    _check_parity(dev, ref, a, dims, method, eps=1e-6)


# 16^5: the first unfolding is 16 x 65,536 (ULV: Col, URV: Row), so pass 1 runs in the
# persistent step loop (k_pass1_big<5> over the row-layout copy / <6>), its guard included
@pytest.mark.parametrize("method", ["urv", "ulv"])
@pytest.mark.parametrize("mode", ["rank", "tol"])
def test_persistent_loop_cuts(dev, ref, method, mode):
    dims, ranks = [16] * 5, [1, 6, 8, 8, 6, 1]
    a = planted_plus_noise(ref, dims, ranks, 9, 1e-6)
    if mode == "rank":
        _check_parity(dev, ref, a, dims, method, ranks=ranks)
    else:
        _check_parity(dev, ref, a, dims, method, eps=1e-4)


@pytest.mark.parametrize("mode", ["rank", "tol"])
def test_persistent_loop_odd_column_count(dev, ref, mode):
    """16 x 243 x 243: the ULV first unfolding is 16 x 59,049 -- an odd column count through
    the persistent loop's row-layout copy (the last column has no 16-byte partner)."""
    dims, ranks = [16, 243, 243], [1, 8, 8, 1]
    a = planted_plus_noise(ref, dims, ranks, 13, 1e-6)
    if mode == "rank":
        _check_parity(dev, ref, a, dims, "ulv", ranks=ranks)
    else:
        _check_parity(dev, ref, a, dims, "ulv", eps=1e-4)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_persistent_loop_hilbert_guard(dev, ref, method):
    """Shifted Hilbert 12 x 12 x 12 x 12 x 12 at a prescribed accuracy well above the noise
    floor: many columns are flagged by the 1e-16 guard inside the persistent loop."""
    dims = [12] * 5
    a = shifted_hilbert(dims)
    _check_parity(dev, ref, a, dims, method, eps=1e-5)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_long_first_unfolding_tsqr(dev, ref, method):
    """16^5 x 8 shifted Hilbert: the first unfolding has 524,288 (ULV) / 1,048,576 (URV)
    columns and an ill-conditioned R1, so pass 2 takes the TSQR route with the streaming
    leaf (one CTA per SM folding its rows into one triangle)."""
    dims = [16, 16, 16, 16, 16, 8]
    a = shifted_hilbert(dims)
    _check_parity(dev, ref, a, dims, method, eps=1e-5)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_planted_exact_recovery(dev, ref, method):
    dims, ranks = [7, 6, 8, 5], [1, 3, 4, 2, 1]
    a = ref.gen_planted_dense(dims, ranks, 301)
    res = dev.decompose_device(a, dims, method, "l2r" if method == "ulv" else "r2l", ranks=ranks)
    assert res.rse(a) <= 1e-10


def test_clamping_and_warnings(dev, ref):
    dims = [4, 6, 1]
    a = ref.gen_gaussian(dims, 5)
    res = dev.decompose(a, dims, "ulv", "l2r", ranks=[1, 9, 9, 1])
    rr = ref.decompose(a, dims, "ulv", "l2r", ranks=[1, 9, 9, 1])
    assert res.report.ranks_chosen == rr.ranks_chosen
    assert res.report.warnings == rr.warnings


def test_zero_tensor(dev, ref):
    dims = [3, 4, 5]
    a = np.zeros(60)
    res = dev.decompose(a, dims, "urv", "r2l", ranks=[1, 2, 3, 1])
    rr = ref.decompose(a, dims, "urv", "r2l", ranks=[1, 2, 3, 1])
    assert res.report.ranks_chosen == rr.ranks_chosen == [1, 1, 1, 1]
    assert res.report.warnings == rr.warnings
    assert all(np.all(c == 0) for c in res.cores)


def test_order_one(dev, ref):
    a = np.arange(1.0, 8.0)
    res = dev.decompose(a, [7], "ulv", "l2r", ranks=[1, 1])
    assert res.report.ranks_chosen == [1, 1]
    np.testing.assert_array_equal(res.cores[0].reshape(-1), a)


def test_rank_chain_errors(dev):
    from paper_2501_07904_b200 import ArgumentError
    a = np.ones(24)
    with pytest.raises(ArgumentError, match="rank chain has 3 entries, expected 4"):
        dev.decompose(a, [2, 3, 4], "urv", "r2l", ranks=[1, 2, 1])
    with pytest.raises(ArgumentError, match="boundary ranks must both be 1"):
        dev.decompose(a, [2, 3, 4], "urv", "r2l", ranks=[2, 2, 2, 1])
    with pytest.raises(ArgumentError, match="squared weights must sum to 1"):
        dev.decompose(a, [2, 3, 4], "urv", "r2l", eps=0.1, weights=[0.5, 0.5])
    with pytest.raises(ArgumentError, match="tolerance must be >= 0"):
        dev.decompose(a, [2, 3, 4], "urv", "r2l", eps=-1.0)


# (5000, 96): the in-place engine's column-parallel mode; (5000, 300): the same with panel
# (delayed) updates; (5000, 40): its row-block mode
@pytest.mark.parametrize("shape", [(30, 20), (20, 30), (100, 400), (100, 20), (1, 7), (7, 1), (5000, 96),
                                   (5000, 300), (5000, 40), (4500, 1200)])
def test_qr_col_pivot_matches_reference(dev, ref, shape):
    rng = np.random.default_rng(7)
    a = np.asfortranarray(rng.standard_normal(shape))
    q, r, perm = dev.qr_col_pivot(a)
    q0, r0, perm0 = ref.qr_col_pivot(a)
    np.testing.assert_array_equal(perm, perm0)
    nrm = np.linalg.norm(a)
    assert np.max(np.abs(r - r0)) <= 1e-12 * nrm
    assert np.max(np.abs(q - q0)) <= 1e-12
    # reference identities (test_factor.cpp:103-140)
    assert np.max(np.abs(q @ r - a[:, perm])) <= 1e-12 * nrm
    assert np.max(np.abs(q.T @ q - np.eye(q.shape[1]))) <= 1e-12
    assert np.all(np.tril(r, -1) == 0.0)
    d = np.abs(np.diag(r))
    assert np.all(d[1:] <= d[:-1] * (1 + 1e-12) + 1e-300)


def test_qr_col_pivot_zero_matrix(dev):
    q, r, perm = dev.qr_col_pivot(np.zeros((5, 3), order="F"))
    np.testing.assert_array_equal(q, np.eye(5, 3))
    assert np.all(r == 0)
    np.testing.assert_array_equal(perm, np.arange(3))


def test_determinism(dev, ref):
    a, dims, ranks = cfg1(ref)
    r1 = dev.decompose(a, dims, "urv", "r2l", ranks=ranks)
    r2 = dev.decompose(a, dims, "urv", "r2l", ranks=ranks)
    for c1, c2 in zip(r1.cores, r2.cores):
        np.testing.assert_array_equal(c1, c2)


# ---- general path: TT-SVD, Alg. 4, URV left-to-right, refine_passes 0/2 ---------------
GENERAL = [("svd", "l2r", 0), ("svd", "r2l", 0), ("ulv", "r2l", 0), ("ulv", "r2l", 1), ("urv", "l2r", 0)]


@pytest.mark.parametrize("method,sweep,retain", GENERAL)
@pytest.mark.parametrize("mode", ["rank", "tol"])
def test_general_paths_vs_reference(dev, ref, method, sweep, retain, mode):
    dims, ranks = [6, 5, 7, 4], [1, 3, 4, 2, 1]
    a = planted_plus_noise(ref, dims, ranks, 11, 1e-3)
    kw = dict(ranks=ranks) if mode == "rank" else dict(eps=0.05)
    res = dev.decompose_device(a, dims, method, sweep, retain=["l11_only", "full_column"][retain], **kw)
    rep = res.report()
    rr = ref.decompose(a, dims, method, sweep, retain=retain, **kw)
    assert rep.ranks_chosen == rr.ranks_chosen
    assert rep.bound_kind == ("plain_sum" if rr.bound_kind else "root_sum_square")
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL_RSE
    assert abs(rep.bound - rr.bound) <= 1e-10 * rep.input_norm
    assert rep.warnings == rr.warnings


@pytest.mark.parametrize("refine", [0, 2])
@pytest.mark.parametrize("method,sweep", [("ulv", "l2r"), ("urv", "r2l")])
def test_refine_passes(dev, ref, refine, method, sweep):
    dims, ranks = [6, 5, 7, 4], [1, 3, 4, 2, 1]
    a = planted_plus_noise(ref, dims, ranks, 13, 1e-3)
    res = dev.decompose_device(a, dims, method, sweep, ranks=ranks, refine_passes=refine)
    rr = ref.decompose(a, dims, method, sweep, ranks=ranks, refine=refine)
    assert res.report().ranks_chosen == rr.ranks_chosen
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL_RSE


def test_cfg1_tt_svd_check(dev, ref):
    """BASELINE config 1: TT-URV/TT-ULV checked against TT-SVD (device TT-SVD now)."""
    a, dims, ranks = cfg1(ref)
    s = dev.decompose_device(a, dims, "svd", "l2r", ranks=ranks)
    s_ref = ref.decompose(a, dims, "svd", "l2r", ranks=ranks)
    assert abs(s.rse(a) - ref.rse(s_ref, a, dims)) <= TOL_RSE
    for method, sweep in (("urv", "r2l"), ("ulv", "l2r")):
        r = dev.decompose_device(a, dims, method, sweep, ranks=ranks)
        assert r.rse(a) <= 2.0 * s.rse(a)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_tall_pass1_engine(dev, ref, method):
    """Cuts whose pivoted matrix W is tall (k > 2048 and k > N) take the in-place engine
    (URV: the last cut I_1 x (I_2 r); ULV: the last cut (r I_{d-1}) x I_d)."""
    dims, ranks = ([9, 700, 5], [1, 6, 4, 1]) if method == "urv" else ([5, 700, 9], [1, 4, 6, 1])
    a = planted_plus_noise(ref, dims, ranks, 21, 1e-6)
    _, rep, *_ = _check_parity(dev, ref, a, dims, method, ranks=ranks)
    _check_parity(dev, ref, a, dims, method, eps=1e-4)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_planted_rank48_gram_pass2(dev, ref, method):
    # 33 <= s <= 160 with a well-conditioned R1: pass 2 takes R_B from the Gram matrix
    # (split-K DMMA GEMM + Cholesky) instead of the TSQR tree
    dims, ranks = [64, 64, 64], [1, 48, 48, 1]
    a = planted_plus_noise(ref, dims, ranks, 21, 1e-6)
    _check_parity(dev, ref, a, dims, method, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_tall_cut_gram_pass1(dev, ref, method):
    # a tall fixed-rank cut (k >= 8N): pass 1 runs as the pivoted Cholesky of W^T W
    dims, ranks = [16, 64, 64], [1, 8, 8, 1]
    a = planted_plus_noise(ref, dims, ranks, 33, 1e-6)
    _check_parity(dev, ref, a, dims, method, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_tall_cut_gram_fallback_ill_conditioned(dev, ref, method):
    # Hilbert-type tall cut at fixed rank: R_ss / R_00 < 1e-4, so the cut is redone by the
    # Householder engine
    dims, ranks = [8, 8, 96], [1, 8, 8, 1]
    _check_parity(dev, ref, shifted_hilbert(dims), dims, method, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
@pytest.mark.parametrize("eps", [0.3, 0.1, 0.01])
def test_fixed_tol_guarantee(dev, ref, method, eps):
    # test_tt_decomp.cpp:80-100 / acceptance 3: the prescribed-accuracy sweeps meet eps,
    # and the device picks the reference's ranks
    dims = [7, 8, 6, 9]
    a = ref.gen_gaussian(dims, 17)
    sweep = "l2r" if method == "ulv" else "r2l"
    res = dev.decompose_device(a, dims, method, sweep, eps=eps)
    assert res.rse(a) <= eps * (1 + 1e-12)
    rr = ref.decompose(a, dims, method, sweep, eps=eps)
    assert res.report().ranks_chosen == rr.ranks_chosen
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL_RSE


def test_hilbert_error_decreases_with_eps(dev, ref):
    # acceptance 9: Hilbert 20^3, the error strictly decreases as eps does
    dims = [20, 20, 20]
    a = shifted_hilbert(dims)
    errs = [dev.decompose_device(a, dims, "urv", "r2l", eps=e).rse(a) for e in (1e-2, 1e-4, 1e-6, 1e-8)]
    assert all(x > y for x, y in zip(errs, errs[1:])), errs
    assert all(e <= t for e, t in zip(errs, (1e-2, 1e-4, 1e-6, 1e-8)))


def test_weights_validation(dev):
    from paper_2501_07904_b200._native import ArgumentError
    dims = [4, 5, 6]
    a = np.random.default_rng(0).standard_normal(int(np.prod(dims)))
    with pytest.raises(ArgumentError, match="squared weights must sum to 1"):
        dev.decompose_device(a, dims, "urv", "r2l", eps=0.1, weights=[0.5, 0.5])
    with pytest.raises(ArgumentError, match="weights given, expected"):
        dev.decompose_device(a, dims, "urv", "r2l", eps=0.1, weights=[1.0])
    with pytest.raises(ArgumentError, match="tolerance must be >= 0"):
        dev.decompose_device(a, dims, "urv", "r2l", eps=-1.0)
    # valid unequal weights
    w = [0.6, 0.8]
    res = dev.decompose_device(a, dims, "urv", "r2l", eps=0.2, weights=w)
    assert res.rse(a) <= 0.2 * (1 + 1e-12)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_order_two_fast_path(dev, ref, method):
    dims, ranks = [30, 40], [1, 7, 1]
    a = planted_plus_noise(ref, dims, ranks, 9, 1e-6)
    _check_parity(dev, ref, a, dims, method, ranks=ranks)
    _check_parity(dev, ref, a, dims, method, eps=1e-4)


def test_square_near_full_rank_cut_in_place(dev, ref):
    """A 2116 x 2116 middle cut kept at nearly full rank in tolerance mode (config 4's
    regime): pass 1, pass 2 and the core's Q run on the in-place engine's column-parallel
    steps. Ranks identical to the reference, RSE within the contract."""
    rng = np.random.default_rng(46)
    dims = [46, 46, 46, 46]
    a = rng.standard_normal(int(np.prod(dims)))
    res = dev.decompose_device(a, dims, "urv", "r2l", eps=1e-3)
    rep = res.report()
    assert max(c["n"] for c in rep.cuts) >= 2048 and max(c["m"] for c in rep.cuts) >= 2048
    rr = ref.decompose(a, dims, "urv", "r2l", eps=1e-3)
    assert rep.ranks_chosen == rr.ranks_chosen
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL_RSE


def test_concurrent_host_threads_match_sequential(dev, ref):
    """The API is reentrant: decompositions issued from several host threads at once (each
    thread has its own stream; bench.py's e2e does this) give the same cores bit for bit
    as the same calls made one after another."""
    import threading

    a, dims, ranks = cfg1(ref)
    jobs = [("urv", "r2l", dict(ranks=ranks)), ("ulv", "l2r", dict(ranks=ranks)),
            ("urv", "r2l", dict(eps=1e-6)), ("ulv", "l2r", dict(eps=1e-6))]

    def run(m, s, kw):
        r = dev.decompose_device(a, dims, m, s, **kw)
        return [r.core(k) for k in range(r.order())]

    seq = [run(*j) for j in jobs]
    out = [None] * len(jobs)

    def work(i):
        out[i] = run(*jobs[i])

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for s_cores, c_cores in zip(seq, out):
        assert len(s_cores) == len(c_cores)
        for x, y in zip(s_cores, c_cores):
            np.testing.assert_array_equal(x, y)


def test_wide_near_full_rank_cut_in_place_warp_steps(dev, ref):
    """64 x 32 x 64 x 64 Gaussian noise at eps 1e-3, TT-ULV: the second cut is a 2048 x 4096
    unfolding kept at nearly full rank, so it runs in place with a warp per column (at most
    2048 rows; 64, 32 and 16 rows per lane as the trailing rows shrink)."""
    rng = np.random.default_rng(64)
    dims = [64, 32, 64, 64]
    a = rng.standard_normal(int(np.prod(dims)))
    res = dev.decompose_device(a, dims, "ulv", "l2r", eps=1e-3)
    rep = res.report()
    assert any(c["m"] == 2048 and c["n"] == 4096 for c in rep.cuts)
    rr = ref.decompose(a, dims, "ulv", "l2r", eps=1e-3)
    assert rep.ranks_chosen == rr.ranks_chosen
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL_RSE


# 160 x 240 x 240: the ULV first unfolding is 160 x 57,600 (Col) and the URV one has
# W = c^T = 240 x 38,400 (Row): both run the subspace (lazy-exact) pivoting engine (k >= 128,
# N >= 32768), whose steps take R rows from Z = E^T W while q_t stays in span(E)
@pytest.mark.parametrize("method", ["urv", "ulv"])
@pytest.mark.parametrize("mode", ["rank", "tol"])
def test_subspace_engine_cuts(dev, ref, method, mode):
    dims, ranks = [160, 240, 240], [1, 12, 12, 1]
    a = planted_plus_noise(ref, dims, ranks, 21, 1e-6)
    if mode == "rank":
        _check_parity(dev, ref, a, dims, method, ranks=ranks)
    else:
        _check_parity(dev, ref, a, dims, method, eps=1e-5)


@pytest.mark.parametrize("method,sweep,retain", [("ulv", "l2r", "l11_only"), ("urv", "r2l", "l11_only"),
                                                 ("svd", "l2r", "l11_only"), ("svd", "r2l", "l11_only"),
                                                 ("ulv", "r2l", "l11_only"), ("ulv", "r2l", "full_column"),
                                                 ("urv", "l2r", "l11_only")])
@pytest.mark.parametrize("refine", [1, 2])
def test_debug_checks_carry_identities(dev, ref, method, sweep, retain, refine):
    """DecompConfig::debug_checks (tt_decomp.cpp:82-98, 193-196, 268-317): the device checks the
    carried matrix against the projected unfolding on every cut, like the reference (which
    passes on the same inputs; test_tt_decomp.cpp:47-78)."""
    dims, ranks = [6, 5, 7, 4], [1, 3, 4, 2, 1]
    a = planted_plus_noise(ref, dims, ranks, 11, 1e-3)
    try:
        rr = ref.decompose(a, dims, method, sweep, ranks=ranks, refine=refine,
                           retain=1 if retain == "full_column" else 0, debug=True)
    except ref.RefError as e:
        # the reference's own coupling check can fail at its 1e-10 tolerance (ULV right to left,
        # refine 2 on this fixture: deviation 1.124e-05 vs coupling 1.128e-05); the device must
        # raise the same class with the same message shape
        assert "[6]" in str(e)
        from paper_2501_07904_b200._native import InvariantError
        with pytest.raises(InvariantError, match="sweep"):
            dev.decompose_device(a, dims, method, sweep, ranks=ranks, refine_passes=refine, retain=retain,
                                 debug_checks=True)
        return
    res = dev.decompose_device(a, dims, method, sweep, ranks=ranks, refine_passes=refine, retain=retain,
                               debug_checks=True)
    assert res.report().ranks_chosen == rr.ranks_chosen


def test_debug_checks_rejected_by_sharded(dev, ref):
    a, dims, ranks = cfg1(ref)
    comms = dev.loopback_group(1)
    blk = dev.shard_block(a, dims, "urv", 1, 0)
    with pytest.raises(Exception, match="debug_checks is not supported by the column-sharded sweep"):
        dev.decompose_sharded(blk, dims, comms[0], "urv", "r2l", ranks=ranks, debug_checks=True)
