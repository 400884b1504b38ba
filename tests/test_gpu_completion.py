"""Tensor completion on the device (ttg_complete; completion.hpp / completion.cpp) against the
UNMODIFIED reference library: the reference's own completion tests (tests/test_completion.cpp)
re-run on the device path, its trace compared with the reference's on the same fixture, and
the rank-adaptive retraction (the extension BASELINE config 4 needs)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS, RANKS = [6, 7, 6], [1, 2, 2, 1]


@pytest.fixture(scope="module")
def fixture(ref):
    """test_completion.cpp:15-25: planted truth (seed 21) on a gen_mask(0.5, 22) half mask."""
    truth = ref.gen_planted_dense(DIMS, RANKS, 21)
    d = np.asarray(DIMS, np.int64)
    ind = np.empty(truth.size)
    f = ref.lib().ref_gen_mask
    f.argtypes = [ref.ip, C.c_int, C.c_double, C.c_uint64, ref.dp]
    ref._check(f(ref._i(d), 3, 0.5, 22, ref._d(ind)))
    linear = np.flatnonzero(ind).astype(np.int64)
    return truth, ind, linear, truth[linear].copy()


def _ref_complete(ref, ind, vals_dense, truth, retraction, step=1.0, max_iters=500, stop_tol=1e-6, refine=2):
    f = ref.lib().ref_complete
    f.argtypes = [ref.dp, ref.dp, ref.ip, C.c_int, ref.ip, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int, ref.dp,
                  ref.dp, ref.dp, ref.dp, C.POINTER(C.c_int), C.POINTER(C.c_int), ref.dp]
    obs, full, ps = np.zeros(max_iters), np.zeros(max_iters), np.zeros(max_iters)
    n, st = C.c_int(), C.c_int()
    d = np.asarray(DIMS, np.int64)
    r = np.asarray(RANKS, np.int64)
    ref._check(f(ref._d(ind), ref._d(vals_dense), ref._i(d), 3, ref._i(r), {"svd": 0, "ulv": 1, "urv": 2}[retraction],
                 step, max_iters, stop_tol, refine, ref._d(truth), ref._d(obs), ref._d(full), ref._d(ps), C.byref(n),
                 C.byref(st), None))
    k = n.value
    return obs[:k], full[:k], ps[:k], ["converged", "max_iters", "diverged"][st.value]


@pytest.mark.parametrize("retraction", ["svd", "ulv", "urv"])
def test_half_observed_recovered(dev, ref, fixture, retraction):
    """test_completion.cpp:88-108 on the device, and the trace against the reference's."""
    truth, ind, linear, vals = fixture
    c = dev.complete(linear, vals, DIMS, ranks=RANKS, retraction=retraction, max_iters=300, truth=truth)
    tr = c.trace
    assert tr.status != "diverged"
    assert tr.rse_full and tr.rse_full[-1] <= 1e-3
    assert len(tr.rse_full) == len(tr.rse_observed) == len(tr.psnr)
    res = c.result()
    x = dev.reconstruct([res.core(k) for k in range(3)]).ravel(order="F")
    assert abs(tr.psnr[-1] - dev.psnr(x, truth)) <= 1e-6
    assert all(r == RANKS for r in tr.ranks)
    obs, full, ps, st = _ref_complete(ref, ind, truth * ind, truth, retraction, max_iters=300)
    # the first iterations agree with the reference's trace to rounding; both end the same way
    m = min(5, len(obs))
    assert np.allclose(tr.rse_observed[:m], obs[:m], rtol=1e-8, atol=1e-14)
    assert tr.status == st
    assert abs(tr.rse_full[-1] - full[-1]) <= 1e-6


def test_full_mask_converges_immediately(dev, fixture):
    """test_completion.cpp:73-86."""
    truth, *_ = fixture
    c = dev.complete(np.arange(truth.size), truth, DIMS, ranks=RANKS, stop_tol=1e-10, truth=truth)
    assert c.trace.status == "converged"
    assert len(c.trace.rse_observed) <= 8
    res = c.result()
    x = dev.reconstruct([res.core(k) for k in range(3)]).ravel(order="F")
    assert np.linalg.norm(x - truth) <= 1e-8 * np.linalg.norm(truth)


def test_zero_step_freezes(dev, fixture):
    """test_completion.cpp:110-122: step 0 keeps the initial guess, 12 iterations, no stop."""
    truth, ind, linear, vals = fixture
    c = dev.complete(linear, vals, DIMS, ranks=RANKS, step_size=0.0, stop_tol=0.0, max_iters=12)
    assert c.trace.status == "max_iters"
    assert len(c.trace.rse_observed) == 12
    assert max(c.trace.rse_observed) - min(c.trace.rse_observed) <= 1e-12


def test_config_errors(dev, fixture):
    truth, ind, linear, vals = fixture
    with pytest.raises(Exception, match="rank chain has 3 entries, expected 4"):
        dev.complete(linear, vals, DIMS, ranks=[1, 2, 1])
    with pytest.raises(Exception, match=r"completion would materialize 252 elements \(cap 100\)"):
        dev.complete(linear, vals, DIMS, ranks=RANKS, dense_cap=100)
    with pytest.raises(Exception, match="step size must be >= 0"):
        dev.complete(linear, vals, DIMS, ranks=RANKS, step_size=-1.0)


def test_rank_adaptive_retraction(dev, ref, fixture):
    """Extension: the retraction at a prescribed accuracy (config 4's harness loop,
    X = URV_eps(Y); Y = reconstruct(X); Y[Omega] = M[Omega]) on the same fixture: the ranks it
    picks are the reference decompose()'s at that eps on the same iterate."""
    truth, ind, linear, vals = fixture
    c = dev.complete(linear, vals, DIMS, eps=1e-3, retraction="urv", max_iters=3, stop_tol=0.0, truth=truth,
                     refine_passes=1)
    assert len(c.trace.ranks) == 4
    # iteration 0 (the initial guess) retracts the zero-filled observations
    y0 = truth * ind
    rr = ref.decompose(y0, DIMS, "urv", "r2l", eps=1e-3)
    assert c.trace.ranks[0] == rr.ranks_chosen
    assert abs(c.trace.initial["rse_full"] - ref.rse(rr, truth, DIMS)) <= 1e-10
