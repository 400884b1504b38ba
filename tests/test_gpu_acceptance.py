"""Acceptance-style properties (tests/acceptance.cpp criteria 1, 4, 5, 6) re-checked on the
device engine over many seeded fixtures, plus parity with the reference on each."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_fixture(ref, trial):
    rng = np.random.default_rng(100 + trial)
    order = 3 + trial % 2
    dims = [int(x) for x in rng.integers(3, 11, size=order)]
    ranks = [1]
    for k in range(1, order):
        feas = min(int(np.prod(dims[:k])), int(np.prod(dims[k:])))
        ranks.append(int(rng.integers(1, min(5, feas) + 1)))
    ranks.append(1)
    a = ref.gen_gaussian(dims, 1000 + trial)
    return a, dims, ranks


@pytest.mark.parametrize("method,sweep", [("ulv", "l2r"), ("urv", "r2l")])
def test_fixed_rank_bound_and_parity_random(dev, ref, method, sweep):
    """Criterion 1: achieved error within the rss bound; plus |dRSE| <= 1e-10 vs the
    reference on every fixture (random Gaussian tensors: the early exit must extend)."""
    worst = 0.0
    for trial in range(60):
        a, dims, ranks = random_fixture(ref, trial)
        res = dev.decompose_device(a, dims, method, sweep, ranks=ranks)
        rep = res.report()
        nrm = ref.frobenius_norm(a)
        achieved = res.rse(a) * nrm
        assert achieved <= rep.bound + 1e-8 * nrm, (trial, achieved, rep.bound)
        rr = ref.decompose(a, dims, method, sweep, ranks=ranks)
        assert rep.ranks_chosen == rr.ranks_chosen
        worst = max(worst, abs(res.rse(a) - ref.rse(rr, a, dims)))
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("method,sweep", [("ulv", "l2r"), ("urv", "r2l"), ("svd", "l2r"), ("svd", "r2l"),
                                          ("ulv", "r2l"), ("urv", "l2r")])
def test_planted_recovery_all_paths(dev, ref, method, sweep):
    """Criterion 4: exactly low-rank inputs recovered to 1e-10 by every sweep path."""
    for trial in range(6):
        rng = np.random.default_rng(300 + trial)
        order = 3 + trial % 2
        dims = [int(x) for x in rng.integers(5, 10, size=order)]
        ranks = [1] + [int(x) for x in rng.integers(2, 5, size=order - 1)] + [1]
        a = ref.gen_planted_dense(dims, ranks, 77 + trial)
        res = dev.decompose_device(a, dims, method, sweep, ranks=ranks)
        assert res.rse(a) <= 1e-10


@pytest.mark.parametrize("method,sweep", [("ulv", "l2r"), ("urv", "r2l"), ("svd", "l2r"), ("svd", "r2l"),
                                          ("ulv", "r2l"), ("urv", "l2r")])
def test_core_orthogonality(dev, ref, method, sweep):
    """Criterion 5: left-orthogonal cores for left-to-right sweeps (and the reversed URV
    route), right-orthogonal cores for right-to-left sweeps, within 1e-12."""
    for trial in range(4):
        rng = np.random.default_rng(400 + trial)
        dims = [int(rng.integers(4, 8)), int(rng.integers(4, 8)), int(rng.integers(4, 8)), int(rng.integers(3, 6))]
        a = ref.gen_gaussian(dims, 500 + trial)
        cores = dev.decompose(a, dims, method, sweep, ranks=[1, 3, 4, 3, 1]).cores
        if sweep == "l2r":
            for c in cores[:-1]:
                g = c.reshape((-1, c.shape[2]), order="F")
                assert np.max(np.abs(g.T @ g - np.eye(g.shape[1]))) <= 1e-12
        else:
            for c in cores[1:]:
                g = c.reshape((c.shape[0], -1), order="F")
                assert np.max(np.abs(g @ g.T - np.eye(g.shape[0]))) <= 1e-12


def test_cpp_dropin_program(dev):
    """A C++ caller written against the reference headers runs on the device engine."""
    import subprocess
    from paper_2501_07904_b200._native import LIB_PATH
    exe = LIB_PATH.parent / "dropin_check"
    assert exe.exists(), "built by __graft_entry__.build()"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


@pytest.mark.parametrize("method,sweep", [("ulv", "l2r"), ("urv", "r2l")])
@pytest.mark.parametrize("mode", ["rank", "tol"])
def test_edge_shapes_random(dev, ref, method, sweep, mode):
    """Ragged and degenerate shapes (modes of size 1, orders 2-6, wide and tall cuts, ranks
    clamped by the shape), both rank modes, against the reference: identical ranks and
    |dRSE| <= 1e-10."""
    rng = np.random.default_rng(7 if mode == "rank" else 8)
    for trial in range(40):
        order = int(rng.integers(2, 7))
        dims = [int(x) for x in rng.integers(1, 9 if order > 4 else 13, size=order)]
        a = ref.gen_gaussian(dims, 5000 + trial)
        if mode == "rank":
            ranks = [1] + [int(rng.integers(1, 7)) for _ in range(order - 1)] + [1]
            kw = dict(ranks=ranks)
        else:
            kw = dict(eps=float(rng.choice([0.5, 0.2, 0.05])))
        res = dev.decompose_device(a, dims, method, sweep, **kw)
        rr = ref.decompose(a, dims, method, sweep, **kw) if mode == "rank" else \
            ref.decompose(a, dims, method, sweep, eps=kw["eps"])
        assert res.report().ranks_chosen == rr.ranks_chosen, (trial, dims, kw)
        assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= 1e-10, (trial, dims, kw)
