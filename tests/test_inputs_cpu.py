"""CPU tests: the bench/test input generators (paper_2501_07904_b200/inputs.py over
hostgen/inputs.cpp) give BITWISE the buffers of the reference's own generators
(generators.cpp, reconstruct, frobenius_norm), so the full-size golden fixtures computed by
the reference on its generators (tests/golden/full_cfg*.npz) apply to bench.py's inputs."""
import numpy as np
import pytest

from paper_2501_07904_b200 import inputs
from tests.fixtures import planted_plus_noise, shifted_hilbert


def test_u64_stream_matches_reference(ref):
    got = inputs.u64(5, 123)
    lib = ref.lib()
    import ctypes as C
    lib.ref_rng_u64.argtypes = [C.c_uint64, C.c_int64]
    lib.ref_rng_u64.restype = C.c_uint64
    want = [lib.ref_rng_u64(123, k) for k in range(5)]
    assert [int(x) for x in got] == want


@pytest.mark.parametrize("n,seed", [(1, 3), (2, 3), (7, 11), (100_001, 2), (2_000_000, 40)])
def test_gaussian_bitwise(ref, n, seed):
    got = inputs.gaussian(n, seed)
    want = ref.gen_gaussian([n], seed)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 3 * 4096 + 5, 1_000_003])
def test_frobenius_norm_bitwise(ref, n):
    x = inputs.gaussian(n, 9) * 1e-3
    assert inputs.frobenius_norm(x) == ref.frobenius_norm(x)


@pytest.mark.parametrize("dims,ranks,seed,rho", [
    ([20] * 4, [1, 5, 5, 5, 1], 1, 1e-8),
    ([6] * 6, [1, 4, 5, 5, 5, 4, 1], 3, 1e-4),
    ([12, 9, 10], [1, 7, 5, 1], 5, 1e-6),
    ([5, 4], [1, 3, 1], 2, 0.0),
    ([8] * 5, [1, 4, 6, 6, 4, 1], 3, 1e-4),
])
def test_planted_bitwise(ref, dims, ranks, seed, rho):
    got = inputs.planted(dims, ranks, seed, rho)
    want = planted_plus_noise(ref, dims, ranks, seed, rho)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_planted_cores_bitwise(ref):
    dims, ranks = [6, 7, 5], [1, 3, 4, 1]
    cores = inputs.planted_cores(dims, ranks, 7)
    flat = np.concatenate([c.reshape(-1, order="F") for c in cores])
    want = np.empty_like(flat)
    import ctypes as C
    d = np.asarray(dims, np.int64)
    r = np.asarray(ranks, np.int64)
    ref._check(ref.lib().ref_gen_planted_cores(ref._i(d), 3, ref._i(r), 7, ref._d(want)))
    assert np.array_equal(flat, want)


def test_hilbert_shifted():
    for dims in ([32] * 5, [3, 4, 5], [7]):
        assert np.array_equal(inputs.hilbert_shifted(dims), shifted_hilbert(dims))
    assert inputs.hilbert_shifted([32] * 5)[0] == 1.0


def test_config4_mask_count():
    """the survey's mask (Rng(41).uniform() < 0.5 per entry, storage order)
    observes 8,389,438 of the 256^3 entries."""
    m = inputs.bernoulli_mask(256 ** 3, seed=41)
    assert int(m.sum()) == 8_389_438
    assert set(np.unique(m)) == {0.0, 1.0}


def test_config4_volume_recipe():
    """Blob parameters drawn per blob in the order c_x, c_y, c_z, w_x, w_y, w_z, amplitude
    (SURVEY Appendix C); spot-check one voxel against a direct evaluation."""
    n, nb = 16, 3
    v = np.empty(n ** 3)
    inputs.lib().tig_blobs(n, nb, 4, inputs._d(v))
    u = (inputs.u64(7 * nb, 4) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    p = u.reshape(nb, 7)
    c, w, amp = p[:, :3] * n, 4.0 + 28.0 * p[:, 3:6], 0.2 + 0.8 * p[:, 6]
    x, y, z = 5, 11, 2
    want = sum(amp[b] * np.prod([np.exp(-0.5 * ((t - c[b, a]) / w[b, a]) ** 2) for a, t in enumerate((x, y, z))])
               for b in range(nb))
    assert abs(v[x + n * (y + n * z)] - want) <= 1e-14 * abs(want)
