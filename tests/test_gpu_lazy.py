"""Candidate (lazy-exact) pivoting for narrow, very wide first cuts (qrcp_wide.cu k_lz_*): the
engine reads only a gathered candidate set S on most steps and replays the skipped rows of R
for every column on a miss, so its pivots and kept factors must be those of the reference's
step-by-step qr_col_pivot (factor.cpp:62-135) on the same input.

W = 24 x 1,048,576 (above the engine's 1M-column threshold): a planted rank-20 tensor with
noise (config 3's structure, smaller) for TT-ULV-L2R (Col W) and TT-URV-R2L (Row W), and a
Hilbert-type tensor (many near-equal residual norms, exact ties across identical columns) at
fixed rank 12. Contract as SURVEY Appendix A: identical ranks, |dRSE| <= 1e-10, kept |T_ii|
within 1e-10 |T_00| on every cut.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _planted(ref, dims, ranks, seed, rho):
    a0 = ref.gen_planted_dense(dims, ranks, seed)
    e = ref.gen_gaussian(dims, seed + 1)
    return a0 + (rho * ref.frobenius_norm(a0) / ref.frobenius_norm(e)) * e


def _hilbert(dims):
    idx = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1]  # first index fastest
    return 1.0 / (idx.sum(axis=0) + 1.0)


def _check(dev, ref, a, dims, method, sweep, ranks):
    res = dev.decompose_device(a, dims, method, sweep, ranks=ranks)
    rep = res.report()
    rr, cuts = ref.sweep_trace(a, dims, method, ranks=ranks)
    assert rep.ranks_chosen == rr.ranks_chosen
    assert abs(res.rse(a) - ref.rse(rr, a, dims)) <= TOL
    # cuts matched by unfolding shape (the two reports order them differently)
    by_shape = {(c["m"], c["n"]): c for c in cuts}
    assert len(by_shape) == len(rep.cuts)
    for dc in rep.cuts:
        gd = by_shape[(dc["m"], dc["n"])]["diag"]
        r = dc["rank"]
        assert np.abs(dc["diag"][:r] - gd[:r]).max() <= TOL * gd[0], (dc["m"], dc["n"])


@pytest.mark.parametrize("method,sweep,dims", [("ulv", "l2r", [24, 1024, 1024]), ("urv", "r2l", [1024, 1024, 24])])
def test_lazy_planted(dev, ref, method, sweep, dims):
    a = _planted(ref, dims, [1, 20, 20, 1], 31, 1e-4)
    _check(dev, ref, a, dims, method, sweep, [1, 20, 20, 1])


@pytest.mark.parametrize("method,sweep,dims", [("ulv", "l2r", [24, 1024, 1024]), ("urv", "r2l", [1024, 1024, 24])])
def test_lazy_hilbert_ties(dev, ref, method, sweep, dims):
    # rank 7: kept diagonals down to ~1e-5 |T_00|, well above the rounding-ordered tail
    a = _hilbert(dims)
    _check(dev, ref, a, dims, method, sweep, [1, 7, 7, 1])


@pytest.mark.parametrize("method,sweep,dims,ranks", [
    ("ulv", "l2r", [8, 32, 32, 32, 32], [1, 8, 20, 20, 20, 1]),
    ("urv", "r2l", [32, 32, 32, 32, 8], [1, 20, 20, 20, 8, 1]),
])
def test_lazy_wide_second_cut(dev, ref, method, sweep, dims, ranks):
    """The warp-per-column variant (32 < k <= 512): the second cut is 256 x 32,768 (Col W for
    ULV, Row W for URV) after a narrow 8 x 4,194,304 first cut."""
    a = _planted(ref, dims, ranks, 41, 1e-4)
    _check(dev, ref, a, dims, method, sweep, ranks)


@pytest.mark.parametrize("method,sweep,dims,ranks", [
    ("ulv", "l2r", [24, 1024, 1024], [1, 20, 20, 1]),
    ("urv", "r2l", [32, 32, 32, 32, 8], [1, 20, 20, 20, 8, 1]),
])
def test_lazy_exact_pass_in_several_sweeps(dev, ref, method, sweep, dims, ranks, monkeypatch):
    """The DMMA exact pass replays at most 24 rows of R per sweep over W and takes another
    sweep for more. TTG_LZ_MFCAP=1 caps a sweep at 8 rows, so the replays of these cuts (up to
    ~12 rows between misses) go through the several-sweeps path; same contract."""
    monkeypatch.setenv("TTG_LZ_MFCAP", "1")
    a = _planted(ref, dims, ranks, 43, 1e-4)
    _check(dev, ref, a, dims, method, sweep, ranks)
