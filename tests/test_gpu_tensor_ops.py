"""Tensor algebra of the drop-in (tensor_ops.hpp, tt.hpp, factor.hpp rank_reveal_diag) on the
device against the UNMODIFIED reference library on the same inputs: mode_product and kron
bitwise (same operation order), reverse_indices / reverse_tt exactly (permutations), psnr and
rank_reveal_diag to rounding."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref_call(ref, name, argtypes):
    import ctypes as C
    f = getattr(ref.lib(), name)
    f.argtypes = argtypes
    return f


@pytest.mark.parametrize("dims,k,rows", [((3, 4, 5), 2, 6), ((7, 3), 1, 2), ((2, 3, 4, 5), 4, 3), ((9,), 1, 4),
                                         ((20, 20, 20), 3, 20)])
def test_mode_product_bitwise(dev, ref, dims, k, rows):
    import ctypes as C
    rng = np.random.default_rng(k + rows)
    x = rng.standard_normal(int(np.prod(dims)))
    m = np.asfortranarray(rng.standard_normal((rows, dims[k - 1])))
    got = dev.mode_product(x.reshape(dims, order="F"), m, k).ravel(order="F")
    want = np.empty_like(got)
    d = np.asarray(dims, np.int64)
    f = _ref_call(ref, "ref_mode_product", [ref.dp, ref.ip, C.c_int, C.c_int, ref.dp, C.c_int64, C.c_int64, ref.dp])
    ref._check(f(ref._d(x), ref._i(d), d.size, k, ref._d(m), rows, dims[k - 1], ref._d(want)))
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_mode_product_errors(dev):
    x = np.zeros((3, 4))
    with pytest.raises(dev.ArgumentError if hasattr(dev, "ArgumentError") else Exception,
                       match="mode-2 product needs 4 columns, matrix has 3"):
        dev.mode_product(x, np.zeros((2, 3)), 2)
    with pytest.raises(Exception, match="mode 3 out of range 1..2"):
        dev.mode_product(x, np.zeros((2, 4)), 3)


def test_kron_bitwise(dev, ref):
    import ctypes as C
    rng = np.random.default_rng(3)
    a = np.asfortranarray(rng.standard_normal((3, 5)))
    b = np.asfortranarray(rng.standard_normal((4, 2)))
    got = dev.kron(a, b)
    want = np.empty((12, 10), order="F")
    f = _ref_call(ref, "ref_kron", [ref.dp, C.c_int64, C.c_int64, ref.dp, C.c_int64, C.c_int64, ref.dp])
    ref._check(f(ref._d(a), 3, 5, ref._d(b), 4, 2, ref._d(want)))
    assert np.array_equal(got, want)


def test_psnr(dev, ref):
    import ctypes as C
    rng = np.random.default_rng(4)
    t = rng.standard_normal((6, 7, 8))
    e = t + 1e-3 * rng.standard_normal(t.shape)
    d = np.asarray(t.shape, np.int64)
    want = C.c_double()
    f = _ref_call(ref, "ref_psnr", [ref.dp, ref.dp, ref.ip, C.c_int, C.POINTER(C.c_double)])
    te, tt = np.ascontiguousarray(e.ravel(order="F")), np.ascontiguousarray(t.ravel(order="F"))
    ref._check(f(ref._d(te), ref._d(tt), ref._i(d), 3, C.byref(want)))
    assert abs(dev.psnr(te, tt) - want.value) <= 1e-10 * abs(want.value)
    assert np.isinf(dev.psnr(tt, tt))


def test_reverse_indices_and_reverse_tt(dev, ref):
    import ctypes as C
    rng = np.random.default_rng(5)
    dims, ranks = [4, 3, 5, 2], [1, 2, 3, 2, 1]
    x = rng.standard_normal(dims)
    got = dev.reverse_indices(x).ravel(order="F")
    want = np.empty_like(got)
    d = np.asarray(dims, np.int64)
    f = _ref_call(ref, "ref_reverse_indices", [ref.dp, ref.ip, C.c_int, ref.dp])
    xf = np.ascontiguousarray(x.ravel(order="F"))
    ref._check(f(ref._d(xf), ref._i(d), 4, ref._d(want)))
    assert np.array_equal(got, want)
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) for k in range(4)]
    rev = dev.reverse_tt(cores)
    flat = np.concatenate([c.ravel(order="F") for c in cores])
    want = np.empty_like(flat)
    r = np.asarray(ranks, np.int64)
    f = _ref_call(ref, "ref_reverse_tt", [ref.dp, ref.ip, ref.ip, C.c_int, ref.dp])
    ref._check(f(ref._d(flat), ref._i(d), ref._i(r), 4, ref._d(want)))
    assert np.array_equal(np.concatenate([c.ravel(order="F") for c in rev]), want)
    # reverse commutes with reconstruct (test_tt.cpp:120-138)
    a = dev.reconstruct(cores)
    b = dev.reconstruct(rev)
    assert np.abs(dev.reverse_indices(a) - b).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("lower", [True, False])
def test_rank_reveal_diag_vs_reference(dev, ref, lower):
    """rank_reveal_diag through the C++ drop-in is exercised by dropin_check; here the same
    quantities from the device SVD of the reference's own factors vs the reference."""
    import ctypes as C
    rng = np.random.default_rng(6)
    a = np.asfortranarray(rng.standard_normal((10, 8)))
    u, t, v = ref.utv(a, lower=lower, refine=1)
    f = _ref_call(ref, "ref_rank_reveal_diag", [ref.dp, ref.dp, ref.dp, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                                C.c_int64, ref.dp])
    for rank in (1, 3, 8):
        want = np.zeros(4)
        ref._check(f(ref._d(u), ref._d(t), ref._d(v), 10, 8, 8, int(lower), rank, ref._d(want)))
        s_t11 = dev.svd(np.asfortranarray(t[:rank, :rank]))[1]
        s_full = dev.svd(np.asfortranarray(t))[1]
        disc = t[rank:, :] if lower else t[:, rank:]
        got = [s_t11[-1], dev.svd(np.asfortranarray(disc))[1][0] if rank < 8 else 0.0, s_full[rank - 1],
               s_full[rank] if rank < 8 else 0.0]
        assert np.allclose(got, want, rtol=1e-12, atol=1e-14 * s_full[0]), (rank, got, want)
