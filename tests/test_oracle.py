"""CPU tests: pin the oracle before trusting it.

- the plain-C restatement (oracle/liboracle.so) reproduces the committed golden fixtures,
  which were produced by the UNMODIFIED reference library (tests/golden/make_golden.py),
  BITWISE: generators, qr_col_pivot, ulv/urv at refine 0/1/2, every sweep variant;
- the reference library itself (oracle/_ref, when built here) still reproduces them;
- the reference's own known answers and identities (test_factor.cpp) hold for the port.
"""
from pathlib import Path

import numpy as np
import pytest

from tests.golden.make_golden import QR_CASES, SWEEP_CASES

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def port():
    from oracle import port as p
    if not p.available():
        pytest.skip("oracle/liboracle.so not built (make -C oracle oracle)")
    return p


@pytest.fixture(scope="module")
def factor_gold():
    return np.load(GOLD / "factor.npz")


@pytest.fixture(scope="module")
def sweep_gold():
    return np.load(GOLD / "sweeps.npz")


def port_input(port, dims, ranks, seed, rho):
    """The golden inputs, rebuilt with the port's generators (bitwise = reference)."""
    if ranks is None:
        g = np.meshgrid(*[np.arange(1, n + 1, dtype=np.float64) for n in dims], indexing="ij")
        return (1.0 / (sum(g) - (len(dims) - 1))).ravel(order="F")
    a0 = port.reconstruct_flat(port.gen_planted_cores(dims, ranks, seed), dims, ranks)
    if rho == 0.0:
        return a0
    e = port.gen_gaussian(int(np.prod(dims)), seed + 1)
    return a0 + (rho * np.sqrt(port.sum_squares(a0)) / np.sqrt(port.sum_squares(e))) * e


def test_generators_bitwise(port):
    g = np.load(GOLD / "generators.npz")
    np.testing.assert_array_equal(port.gen_gaussian(1000, 7), g["gauss_1000_7"])
    np.testing.assert_array_equal(port.gen_hilbert([5, 6, 7]), g["hilbert_5x6x7"])
    np.testing.assert_array_equal(port.gen_planted_cores([4, 5, 6], [1, 2, 3, 1], 42), g["planted_4x5x6_123_42"])


@pytest.mark.parametrize("name", list(QR_CASES))
def test_qr_col_pivot_bitwise(port, factor_gold, name):
    a = factor_gold[f"{name}/a"]
    q, r, perm = port.qr_col_pivot(a)
    np.testing.assert_array_equal(perm, factor_gold[f"{name}/perm"])
    np.testing.assert_array_equal(q, factor_gold[f"{name}/q"])
    np.testing.assert_array_equal(r, factor_gold[f"{name}/r"])


@pytest.mark.parametrize("name", list(QR_CASES))
@pytest.mark.parametrize("lower", [0, 1])
@pytest.mark.parametrize("refine", [0, 1, 2])
def test_utv_bitwise(port, factor_gold, name, lower, refine):
    a = factor_gold[f"{name}/a"]
    u, t, v = port.utv(a, lower, refine)
    key = f"{name}/utv{lower}{refine}"
    np.testing.assert_array_equal(u, factor_gold[key + "/u"])
    np.testing.assert_array_equal(t, factor_gold[key + "/t"])
    np.testing.assert_array_equal(v, factor_gold[key + "/v"])


@pytest.mark.parametrize("case", SWEEP_CASES, ids=[c[0] for c in SWEEP_CASES])
def test_sweeps_bitwise(port, sweep_gold, case):
    name, dims, ranks, seed, rho, method, sweep, mode, arg, retain = case
    a = port_input(port, dims, ranks, seed, rho)
    s = sweep_gold[f"{name}/sum_a"]
    assert a.sum() == s[0] and np.sqrt(port.sum_squares(a)) == s[1]
    kw = dict(ranks=arg) if mode == "rank" else dict(eps=arg)
    res = port.decompose(a, dims, method, sweep, retain=retain, **kw)
    assert res["ranks_chosen"] == sweep_gold[f"{name}/ranks"].tolist()
    assert res["step_errors"] == sweep_gold[f"{name}/step_errors"].tolist()
    sc = sweep_gold[f"{name}/scalars"]
    assert res["bound"] == sc[0] and res["bound_kind"] == sc[1] and res["input_norm"] == sc[2]
    for k, c in enumerate(res["cores"]):
        np.testing.assert_array_equal(c, sweep_gold[f"{name}/core{k}"])


def test_reference_library_reproduces_golden(factor_gold, sweep_gold):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built here")
    for name in QR_CASES:
        q, r, perm = ref.qr_col_pivot(factor_gold[f"{name}/a"])
        np.testing.assert_array_equal(r, factor_gold[f"{name}/r"])
        np.testing.assert_array_equal(perm, factor_gold[f"{name}/perm"])
    name, dims, ranks, seed, rho, method, sweep, mode, arg, retain = SWEEP_CASES[0]
    a = ref.gen_planted_dense(dims, ranks, seed)
    e = ref.gen_gaussian(dims, seed + 1)
    a = a + (rho * ref.frobenius_norm(a) / ref.frobenius_norm(e)) * e
    res = ref.decompose(a, dims, method, sweep, ranks=arg)
    for k, c in enumerate(res.cores):
        np.testing.assert_array_equal(c, sweep_gold[f"{name}/core{k}"])


def test_truncation_known_answers(port):
    """diag(3,2,1) spectrum (test_factor.cpp:245-264)."""
    eye = np.eye(3, order="F")
    s = np.array([3.0, 2.0, 1.0])
    r, res, *_ = port.truncate(0, eye, s, eye, eps=1.5)
    assert r == 2 and abs(res - 1.0) < 1e-15
    r, res, *_ = port.truncate(0, eye, s, eye, eps=10.0)
    assert r == 1 and abs(res - np.sqrt(5.0)) < 1e-15
    r, res, *_ = port.truncate(0, eye, s, eye, eps=0.0)
    assert r == 3 and res == 0.0


@pytest.mark.parametrize("shape", [(30, 20), (20, 30), (25, 25)])
def test_qr_identities(port, shape):
    """test_factor.cpp:103-140: reconstruction, orthonormality, exact zeros, |R_kk| nonincreasing."""
    rng = np.random.default_rng(3)
    a = np.asfortranarray(rng.standard_normal(shape))
    q, r, perm = port.qr_col_pivot(a)
    nrm = np.linalg.norm(a)
    assert np.max(np.abs(q @ r - a[:, perm])) <= 1e-12 * nrm
    assert np.max(np.abs(q.T @ q - np.eye(q.shape[1]))) <= 1e-12
    assert np.all(np.tril(r, -1) == 0.0)
    d = np.abs(np.diag(r))
    assert np.all(d[1:] <= d[:-1])
