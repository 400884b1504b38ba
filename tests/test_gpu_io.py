"""Files straight to and from the device: a TTUTVTEN tensor streamed into HBM through pinned
chunks, decomposed without a host copy, and the train written as a TTUTVCOR file that is
byte-identical to the reference's write_tt of the same cores."""
import numpy as np
import pytest

from tests.fixtures import cfg1

pytestmark = pytest.mark.gpu


def test_payload_to_device_bitwise(dev, ref, tmp_path):
    import torch
    # 10.5M doubles (84 MB): more than one 64 MB staging chunk, an odd tail
    dims = [7, 1500, 1000]
    a = np.random.default_rng(5).standard_normal(int(np.prod(dims)))
    p = tmp_path / "big.ttt"
    ref.write_tensor(p, a, dims)
    buf = torch.empty(a.size, dtype=torch.float64, device="cuda")
    assert dev.tensor_file_to_device(p, buf.data_ptr(), a.size) == dims
    np.testing.assert_array_equal(buf.cpu().numpy(), a)


@pytest.mark.parametrize("method,sweep", [("urv", "r2l"), ("ulv", "l2r")])
def test_decompose_file_matches_in_memory(dev, ref, tmp_path, method, sweep):
    a, dims, ranks = cfg1(ref)
    p = tmp_path / "cfg1.ttt"
    ref.write_tensor(p, a, dims)
    rf = dev.decompose_file(p, method, sweep, ranks=ranks)
    rm = dev.decompose_device(a, dims, method, sweep, ranks=ranks)
    assert rf.order() == rm.order()
    for k in range(rm.order()):
        np.testing.assert_array_equal(rf.core(k), rm.core(k))
    assert rf.report().ranks_chosen == rm.report().ranks_chosen


def test_write_file_byte_identical_to_reference(dev, ref, tmp_path):
    a, dims, _ = cfg1(ref)
    res = dev.decompose_device(a, dims, "urv", "r2l", eps=1e-6)
    ours, theirs = tmp_path / "ours.ttc", tmp_path / "theirs.ttc"
    dev.write_result_file(res, ours)
    ref.write_tt(theirs, [res.core(k) for k in range(res.order())])
    assert ours.read_bytes() == theirs.read_bytes()


def test_decompose_file_parse_error(dev, tmp_path):
    from paper_2501_07904_b200._native import ParseError
    p = tmp_path / "bad.ttt"
    p.write_bytes(b"NOTATENSOR")
    with pytest.raises(ParseError) as e:
        dev.decompose_file(p, "urv", "r2l", ranks=[1, 2, 1])
    assert e.value.offset == 0 and "bad magic" in e.value.message
