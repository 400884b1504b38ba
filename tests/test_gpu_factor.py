"""Device factor-level API (qr_col_pivot, ulv/urv at every refine_passes, svd, truncation)
against the golden fixtures produced by the reference library and against its own
identities (test_factor.cpp)."""
from pathlib import Path

import numpy as np
import pytest

from tests.golden.make_golden import QR_CASES

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD / "factor.npz")


def _utv(dev, a, lower, refine):
    from paper_2501_07904_b200._native import check, lib
    from paper_2501_07904_b200.api import _dptr
    a = np.asfortranarray(a, np.float64)
    m, n = a.shape
    p = min(m, n)
    u, t, v = (np.zeros((m, p), order="F"), np.zeros((p, p), order="F"), np.zeros((n, p), order="F"))
    check(lib().ttg_utv(_dptr(a), m, n, int(lower), int(refine), _dptr(u), _dptr(t), _dptr(v)))
    return u, t, v


def _determined(gold, name):
    """Pivots beyond the numerical rank are decided by rounding noise in the reference
    too; compare the steps whose pivot norm is well above it."""
    d = np.abs(np.diag(gold[f"{name}/r"]))
    if d.size == 0 or d[0] == 0.0:
        return 0
    return int(np.sum(d > 1e-6 * d[0]))


@pytest.mark.parametrize("name", list(QR_CASES))
def test_qr_col_pivot_vs_golden(dev, gold, name):
    a = gold[f"{name}/a"]
    q, r, perm = dev.qr_col_pivot(a)
    nrm = max(np.linalg.norm(a), 1e-300)
    k = _determined(gold, name)
    full = k == min(a.shape)
    kk = len(perm) if full else k
    np.testing.assert_array_equal(perm[:kk], gold[f"{name}/perm"][:kk])
    # rows of R indexed by source column (positions past k are rounding-ordered)
    r_src = r[:k][:, np.argsort(perm)]
    g_src = gold[f"{name}/r"][:k][:, np.argsort(gold[f"{name}/perm"])]
    assert np.max(np.abs(r_src - g_src), initial=0.0) <= 1e-12 * nrm
    assert np.max(np.abs(q[:, :k] - gold[f"{name}/q"][:, :k]), initial=0.0) <= 1e-10
    assert np.max(np.abs(q @ r - a[:, perm])) <= 1e-12 * nrm


@pytest.mark.parametrize("name", [n for n in QR_CASES if not n.startswith("hilbert")])
@pytest.mark.parametrize("lower", [0, 1])
@pytest.mark.parametrize("refine", [0, 1, 2])
def test_utv_vs_golden(dev, gold, name, lower, refine):
    a = gold[f"{name}/a"]
    u, t, v = _utv(dev, a, lower, refine)
    key = f"{name}/utv{lower}{refine}"
    nrm = max(np.linalg.norm(a), 1e-300)
    k = _determined(gold, name)
    # the reference's factors, elementwise over the determined block (same pivots, same
    # reflector signs); rank-deficient tails are rounding-decided in the reference too
    assert np.max(np.abs(t[:k, :k] - gold[key + "/t"][:k, :k]), initial=0.0) <= 1e-11 * nrm
    assert np.max(np.abs(u[:, :k] - gold[key + "/u"][:, :k]), initial=0.0) <= 1e-10
    assert np.max(np.abs(v[:, :k] - gold[key + "/v"][:, :k]), initial=0.0) <= 1e-10
    # test_factor.cpp:213-243: exact triangularity, orthogonality, reconstruction
    assert np.all((np.triu(t, 1) if lower else np.tril(t, -1)) == 0.0)
    assert np.max(np.abs(u.T @ u - np.eye(u.shape[1]))) <= 1e-12
    assert np.max(np.abs(v.T @ v - np.eye(v.shape[1]))) <= 1e-12
    assert np.max(np.abs(u @ t @ v.T - a)) <= 1e-10 * nrm


@pytest.mark.parametrize("shape", [(30, 20), (20, 30), (12, 12), (9, 1)])
def test_svd_vs_reference(dev, ref, shape):
    from paper_2501_07904_b200._native import check, lib
    from paper_2501_07904_b200.api import _dptr
    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.standard_normal(shape))
    m, n = shape
    p = min(m, n)
    u, s, v = np.zeros((m, p), order="F"), np.zeros(p), np.zeros((n, p), order="F")
    check(lib().ttg_svd(_dptr(a), m, n, 60, 1e-14, _dptr(u), _dptr(s), _dptr(v)))
    u0, s0, v0 = np.zeros((m, p), order="F"), np.zeros(p), np.zeros((n, p), order="F")
    assert ref.lib().ref_svd(ref._d(a), m, n, ref._d(u0), ref._d(s0), ref._d(v0)) == 0
    assert np.max(np.abs(s - s0)) <= 1e-12 * s0[0]
    assert np.max(np.abs(np.abs(u.T @ u0) - np.eye(p))) <= 1e-9
    assert np.max(np.abs((u * s) @ v.T - a)) <= 1e-12 * np.linalg.norm(a)


def test_truncation_known_answers(dev):
    """diag(3,2,1) (test_factor.cpp:245-264) through the device truncation."""
    from paper_2501_07904_b200._native import check, lib
    from paper_2501_07904_b200.api import _dptr, _iptr
    import ctypes as C
    eye = np.eye(3, order="F")
    s = np.array([3.0, 2.0, 1.0])
    for eps, want_r, want_res in [(1.5, 2, 1.0), (10.0, 1, np.sqrt(5.0)), (0.0, 3, 0.0)]:
        r, res = C.c_int64(), C.c_double()
        u1, t11, v1 = np.zeros(9), np.zeros(9), np.zeros(9)
        check(lib().ttg_truncate(0, _dptr(eye), _dptr(s), _dptr(eye), 3, 3, 3, 0, eps, C.byref(r), C.byref(res),
                                 _dptr(u1), _dptr(t11), _dptr(v1)))
        assert r.value == want_r and abs(res.value - want_res) < 1e-15
