"""Python mirror of the reference's public API (include/ttutv/tt_decomp.hpp, factor.hpp,
tt.hpp), implemented on the device through the C-ABI. Names, argument meaning and error
classes follow the reference so tests read like its own.

Tensors are numpy float64 arrays; an n-d array is taken in the reference's storage order
(first index fastest, i.e. numpy order='F'); a flat array needs ``dims``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._native import ArgumentError, Config, check, lib, require_gpu, c_double_p, c_int64_p

METHODS = {"svd": 0, "ulv": 1, "urv": 2}
SWEEPS = {"l2r": 0, "left_to_right": 0, "r2l": 1, "right_to_left": 1}
RETAIN = {"l11_only": 0, "full_column": 1}
QLP = {"early_exit": 0, "full": 1, "bitwise": 2}


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(c_double_p)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(c_int64_p)


def _flat(a, dims):
    a = np.asarray(a, dtype=np.float64)
    if dims is None:
        dims = a.shape
        a = a.ravel(order="F")
    a = np.ascontiguousarray(a.reshape(-1))
    dims = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    return a, dims


@dataclass
class DecompReport:
    """Mirror of DecompReport (tt_decomp.hpp:49-61) plus per-cut device diagnostics."""
    step_errors: list
    ranks_requested: list
    ranks_chosen: list
    bound: float
    bound_kind: str
    input_norm: float
    wall_time_ms: float
    warnings: list
    achieved_error: Optional[float] = None
    cuts: list = field(default_factory=list)  # dicts: steps, p, rank, extensions, m, n, diag
    # per cut, the discarded mass computed directly (step_errors keep the reference's
    # kept[p] - kept[r] subtraction, factor.cpp:507-510); -1 where not computed
    direct_step_errors: list = field(default_factory=list)


@dataclass
class DecompResult:
    cores: list  # (r_{k-1}, I_k, r_k) arrays, order='F' semantics
    report: DecompReport

    @property
    def ranks(self):
        return [1] + [c.shape[2] for c in self.cores]


class DeviceResult:
    """Owning handle of a ttg_result (cores resident on the device)."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle

    def __del__(self):
        if getattr(self, "_borrowed", False):
            return
        if getattr(self, "h", None):
            try:
                lib().ttg_result_free(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def order(self) -> int:
        return lib().ttg_result_order(self.h)

    def core_dims(self, k: int):
        d = np.zeros(3, np.int64)
        lib().ttg_result_core_dims(self.h, k, _iptr(d))
        return tuple(int(x) for x in d)

    def core(self, k: int) -> np.ndarray:
        dims = self.core_dims(k)
        out = np.empty(int(np.prod(dims)), np.float64)
        check(lib().ttg_result_core_copy(self.h, k, _dptr(out)))
        return out.reshape(dims, order="F")

    def report(self) -> DecompReport:
        d = self.order()
        se = np.zeros(max(d - 1, 0), np.float64)
        rc = np.zeros(d + 1, np.int64)
        rr = np.zeros(d + 1, np.int64)
        b, ni, wt = C.c_double(), C.c_double(), C.c_double()
        bk = C.c_int()
        nreq = lib().ttg_result_report(self.h, _dptr(se), _iptr(rc), _iptr(rr), C.byref(b), C.byref(bk),
                                       C.byref(ni), C.byref(wt))
        warns = [lib().ttg_result_warning(self.h, i).decode() for i in range(lib().ttg_result_warning_count(self.h))]
        cuts = []
        for c in range(max(d - 1, 0)):
            diag = np.zeros(8192, np.float64)
            info = np.zeros(6, np.int64)
            n = lib().ttg_result_cut_diag(self.h, c, _dptr(diag), diag.size, _iptr(info))
            kept = np.zeros(8194, np.float64)
            nk = lib().ttg_result_cut_kept(self.h, c, _dptr(kept), kept.size)
            cuts.append(dict(steps=int(info[0]), p=int(info[1]), rank=int(info[2]), extensions=int(info[3]),
                             m=int(info[4]), n=int(info[5]), diag=diag[:n].copy(),
                             kept=kept[:min(nk, kept.size)].copy()))
        de = np.zeros(max(d - 1, 0), np.float64)
        lib().ttg_result_direct_errors(self.h, _dptr(de))
        return DecompReport(se.tolist(), rr[:nreq].tolist(), rc.tolist(), b.value,
                            "root_sum_square" if bk.value == 0 else "plain_sum", ni.value, wt.value, warns,
                            cuts=cuts, direct_step_errors=de.tolist())

    def rse(self, a, on_device: bool = False) -> float:
        out = C.c_double()
        if on_device:
            check(lib().ttg_result_rse(self.h, C.c_void_p(a), 1, C.byref(out)))
        else:
            a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
            check(lib().ttg_result_rse(self.h, a.ctypes.data_as(C.c_void_p), 0, C.byref(out)))
        return out.value


def _config(method, sweep, ranks, eps, weights, refine_passes, retain, debug_checks, qlp):
    """ttg_config for DecompConfig + FixedRank/FixedTol (tt_decomp.hpp:24-45); the second
    value keeps the arrays it points into alive."""
    cfg = Config()
    cfg.method = METHODS[method]
    cfg.sweep = SWEEPS[sweep]
    keep = []
    if ranks is not None:
        r = np.ascontiguousarray(np.asarray(ranks, dtype=np.int64))
        keep.append(r)
        cfg.fixed_rank = 1
        cfg.ranks = _iptr(r)
        cfg.nranks = int(r.size)
    else:
        cfg.fixed_rank = 0
        cfg.eps = float(eps if eps is not None else 0.0)
    w = np.ascontiguousarray(np.asarray(list(weights), dtype=np.float64))
    keep.append(w)
    cfg.weights = _dptr(w) if w.size else None
    cfg.nweights = int(w.size)
    cfg.refine_passes = int(refine_passes)
    cfg.retain = RETAIN[retain]
    cfg.debug_checks = int(bool(debug_checks))
    cfg.qlp_policy = QLP[qlp]
    return cfg, keep


def decompose_device(a, dims, method="urv", sweep="r2l", ranks=None, eps=None, weights=(), refine_passes=1,
                     retain="l11_only", debug_checks=False, qlp="early_exit", a_is_device_ptr=False) -> DeviceResult:
    """decompose() (tt_decomp.hpp:100) returning the device-resident result handle.

    With ``a_is_device_ptr`` the tensor is read in place from device memory (an integer
    pointer, e.g. ``torch_tensor.data_ptr()``); otherwise it is copied from the host."""
    require_gpu()
    cfg, keep = _config(method, sweep, ranks, eps, weights, refine_passes, retain, debug_checks, qlp)
    dims = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    h = C.c_void_p()
    if a_is_device_ptr or isinstance(a, int):
        # raw pointer: device memory when a_is_device_ptr, else (pinned) host memory
        ptr = C.c_void_p(int(a))
        check(lib().ttg_decompose(ptr, _iptr(dims), int(dims.size), C.byref(cfg), int(bool(a_is_device_ptr)),
                                  C.byref(h)))
    else:
        flat = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
        check(lib().ttg_decompose(flat.ctypes.data_as(C.c_void_p), _iptr(dims), int(dims.size), C.byref(cfg), 0,
                                  C.byref(h)))
    del keep
    return DeviceResult(h)


# ---- files straight to and from the device (io.hpp / io.cpp:139-211) -----------------------

def tensor_file_header(path) -> list:
    """Dims of a TTUTVTEN file (read_tensor's header checks; host only, no device needed)."""
    order = C.c_int()
    dims = np.zeros(255, np.int64)
    check(lib().ttg_tensor_file_header(str(path).encode(), C.byref(order), _iptr(dims)))
    return dims[: order.value].tolist()


def tensor_file_to_device(path, dst_ptr: int, capacity: int) -> list:
    """Stream a TTUTVTEN payload into device memory at dst_ptr (capacity in elements)."""
    require_gpu()
    check(lib().ttg_tensor_file_to_device(str(path).encode(), C.c_void_p(int(dst_ptr)), int(capacity)))
    return tensor_file_header(path)


def decompose_file(path, method="urv", sweep="r2l", ranks=None, eps=None, weights=(), refine_passes=1,
                   retain="l11_only", debug_checks=False, qlp="early_exit") -> DeviceResult:
    """decompose() of the tensor in a TTUTVTEN file, read straight to the device."""
    require_gpu()
    cfg, keep = _config(method, sweep, ranks, eps, weights, refine_passes, retain, debug_checks, qlp)
    h = C.c_void_p()
    check(lib().ttg_decompose_file(str(path).encode(), C.byref(cfg), C.byref(h)))
    del keep
    return DeviceResult(h)


def write_result_file(res: DeviceResult, path) -> None:
    """The result's train as a TTUTVCOR file (byte-identical to the reference's write_tt)."""
    check(lib().ttg_result_write_file(res.h, str(path).encode()))


# ---- multi-GPU (column-sharded first cut) ---------------------------------

class Comm:
    """Owning handle of a ttg_comm endpoint."""

    def __init__(self, handle: C.c_void_p, rank: int, size: int):
        self.h, self.rank, self.size = handle, rank, size

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ttg_comm_free(self.h)
            except TypeError:
                pass
            self.h = None


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    check(lib().ttg_comm_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm(uid: bytes, size: int, rank: int) -> Comm:
    """NCCL communicator over `size` ranks (one process per GPU); `uid` from rank 0's
    nccl_unique_id(), passed to every rank over any side channel (torch.distributed)."""
    require_gpu()
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    h = C.c_void_p()
    check(lib().ttg_comm_nccl_create(buf, int(size), int(rank), C.byref(h)))
    return Comm(h, rank, size)


def loopback_group(size: int) -> list:
    """`size` endpoints sharing this process's GPU; drive each from its own thread."""
    require_gpu()
    hs = (C.c_void_p * size)()
    check(lib().ttg_comm_loopback_create(int(size), hs))
    return [Comm(C.c_void_p(hs[r]), r, size) for r in range(size)]


_HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def callback_comm(allgather, size: int, rank: int) -> Comm:
    """A communicator over a host transport: ``allgather(send: bytes) -> bytes`` must return the
    concatenation of every rank's `send` in rank order (e.g. torch.distributed.all_gather_object
    or all_gather of uint8 tensors over gloo). The engine stages exchanges through host memory."""
    require_gpu()

    def _cb(send, recv, nbytes, _user):
        try:
            out = allgather(C.string_at(send, nbytes))
            if len(out) != nbytes * size:
                return 2
            C.memmove(recv, out, len(out))
            return 0
        except Exception:  # reported to the engine as a failed exchange
            return 1

    fn = _HOST_ALLGATHER(_cb)
    h = C.c_void_p()
    check(lib().ttg_comm_callback_create(int(size), int(rank), C.cast(fn, C.c_void_p), None, C.byref(h)))
    comm = Comm(h, rank, size)
    comm._keep = fn  # the callback must outlive the communicator
    return comm


def shard_range(dims, method: str, size: int, rank: int):
    """(lo, hi, rows, cols): the block of the first unfolding owned by `rank`."""
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    out = np.zeros(4, np.int64)
    check(lib().ttg_shard_range(_iptr(d), int(d.size), METHODS[method], int(size), int(rank), _iptr(out)))
    return tuple(int(x) for x in out)


def shard_block(a, dims, method: str, size: int, rank: int) -> np.ndarray:
    """This rank's block (column-major flat) of a full tensor `a` (host array)."""
    lo, hi, rows, cols = shard_range(dims, method, size, rank)
    flat = np.asarray(a, dtype=np.float64).reshape(-1, order="F")
    if method == "ulv":
        return np.ascontiguousarray(flat[rows * lo:rows * hi])
    m = flat.size // cols
    c = flat.reshape((m, cols), order="F")
    return np.ascontiguousarray(c[lo:hi, :].reshape(-1, order="F"))


def decompose_sharded(a_local, dims, comm: Comm, method="urv", sweep="r2l", ranks=None, eps=None, weights=(),
                      qlp="early_exit", a_is_device_ptr=False, debug_checks=False) -> DeviceResult:
    """Sharded decompose over the ranks of `comm`: `a_local` is this rank's block
    (shard_range / shard_block); every rank gets the whole train."""
    require_gpu()
    cfg, keep = _config(method, sweep, ranks, eps, weights, 1, "l11_only", debug_checks, qlp)
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.int64))
    h = C.c_void_p()
    if a_is_device_ptr or isinstance(a_local, int):
        src, on_dev = C.c_void_p(int(a_local)), int(bool(a_is_device_ptr))
    else:
        flat = np.ascontiguousarray(np.asarray(a_local, dtype=np.float64).reshape(-1))
        keep.append(flat)
        src, on_dev = flat.ctypes.data_as(C.c_void_p), 0
    check(lib().ttg_decompose_sharded(src, _iptr(d), int(d.size), C.byref(cfg), on_dev, comm.h, C.byref(h)))
    del keep
    return DeviceResult(h)


def decompose(a, dims=None, method="urv", sweep="r2l", ranks=None, eps=None, weights=(), refine_passes=1,
              retain="l11_only", debug_checks=False, qlp="early_exit") -> DecompResult:
    """decompose() (tt_decomp.hpp:100): host tensor in, host cores + report out."""
    flat, dims = _flat(a, dims)
    res = decompose_device(flat, dims, method, sweep, ranks, eps, weights, refine_passes, retain, debug_checks, qlp)
    cores = [res.core(k) for k in range(res.order())]
    return DecompResult(cores, res.report())


# The seven named entry points of tt_decomp.hpp:69-97.
def tt_svd(a, dims=None, sweep="l2r", ranks=None, eps=None, weights=(), refine_passes=1):
    return decompose(a, dims, "svd", sweep, ranks, eps, weights, refine_passes)


def tt_ulv_fixed_rank_l2r(a, ranks, dims=None, refine_passes=1, **kw):
    return decompose(a, dims, "ulv", "l2r", ranks=ranks, refine_passes=refine_passes, **kw)


def tt_ulv_fixed_tol_l2r(a, eps, weights=(), dims=None, refine_passes=1, **kw):
    return decompose(a, dims, "ulv", "l2r", eps=eps, weights=weights, refine_passes=refine_passes, **kw)


def tt_urv_fixed_rank_r2l(a, ranks, dims=None, refine_passes=1, **kw):
    return decompose(a, dims, "urv", "r2l", ranks=ranks, refine_passes=refine_passes, **kw)


def tt_urv_fixed_tol_r2l(a, eps, weights=(), dims=None, refine_passes=1, **kw):
    return decompose(a, dims, "urv", "r2l", eps=eps, weights=weights, refine_passes=refine_passes, **kw)


def tt_ulv_fixed_rank_r2l(a, ranks, retain="l11_only", dims=None, refine_passes=1, **kw):
    return decompose(a, dims, "ulv", "r2l", ranks=ranks, retain=retain, refine_passes=refine_passes, **kw)


def left_orthogonal_via_urv(a, dims=None, ranks=None, eps=None, weights=(), refine_passes=1, **kw):
    return decompose(a, dims, "urv", "l2r", ranks=ranks, eps=eps, weights=weights, refine_passes=refine_passes, **kw)


# ---- completion (completion.hpp; BASELINE config 4) ---------------------------------------
@dataclass
class CompletionTrace:
    """IterationTrace (completion.hpp:57-64) plus the rank chain of every iterate
    (ranks[0] = the initial guess) and the initial guess's own errors."""
    ranks: list = field(default_factory=list)
    rse_observed: list = field(default_factory=list)
    rse_full: list = field(default_factory=list)
    psnr: list = field(default_factory=list)
    wall_time_ms: list = field(default_factory=list)
    status: str = "max_iters"
    note: str = ""
    initial: dict = field(default_factory=dict)


class Completion:
    """Owning handle of a ttg_completion: the trace and the final train (on the device)."""

    def __init__(self, handle: C.c_void_p, d: int, has_truth: bool):
        self.h = handle
        n = lib().ttg_completion_iterations(handle)
        obs, full, ps, wall = (np.zeros(max(n, 1)) for _ in range(4))
        init = np.zeros(3)
        lib().ttg_completion_trace(handle, _dptr(obs), _dptr(full), _dptr(ps), _dptr(wall), _dptr(init))
        ranks = []
        buf = np.zeros(d + 1, np.int64)
        for it in range(n + 1):
            if lib().ttg_completion_ranks(handle, it, _iptr(buf)):
                ranks.append(buf.tolist())
        st = lib().ttg_completion_status(handle)
        self.trace = CompletionTrace(ranks, obs[:n].tolist(), full[:n].tolist() if has_truth else [],
                                     ps[:n].tolist() if has_truth else [], wall[:n].tolist(),
                                     ["converged", "max_iters", "diverged"][st],
                                     lib().ttg_completion_note(handle).decode(),
                                     {"rse_observed": init[0], **({"rse_full": init[1], "psnr": init[2]}
                                                                  if has_truth else {})})

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().ttg_completion_free(self.h)
            except TypeError:
                pass
            self.h = None

    def result(self) -> "DeviceResult":
        """The final iterate's train (a view: valid while this handle lives)."""
        r = DeviceResult(C.c_void_p(lib().ttg_completion_result(self.h)))
        r._owner = self
        r._borrowed = True
        return r


def complete(linear, values, dims, ranks=None, eps=None, retraction="svd", step_size=1.0, max_iters=500,
             stop_tol=1e-6, refine_passes=2, dense_cap=10_000_000, truth=None, on_device=False,
             count=None) -> Completion:
    """complete() (completion.hpp:73-75) on the device. ``linear``/``values``: the mask's
    0-based increasing linear indices and observed values (ObservationMask); ``ranks``: the
    fixed-rank chain, or ``eps`` for the rank-adaptive retraction (extension, config 4).
    With ``on_device`` the three array arguments are device pointers (ints) and ``count`` is
    the number of observations."""
    require_gpu()
    from ._native import CompletionConfig
    dims = np.ascontiguousarray(np.asarray(dims, np.int64))
    cfg = CompletionConfig()
    keep = []
    if ranks is not None:
        r = np.ascontiguousarray(np.asarray(ranks, np.int64))
        keep.append(r)
        cfg.ranks, cfg.nranks, cfg.eps = _iptr(r), int(r.size), 0.0
    else:
        cfg.ranks, cfg.nranks, cfg.eps = None, 0, float(eps)
    cfg.retraction = METHODS[retraction]
    cfg.step_size, cfg.max_iters, cfg.stop_tol = float(step_size), int(max_iters), float(stop_tol)
    cfg.refine_passes, cfg.dense_cap = int(refine_passes), int(dense_cap)
    h = C.c_void_p()
    if on_device:
        if count is None:
            raise ArgumentError("on_device completion needs the observation count")
        check(lib().ttg_complete(C.cast(C.c_void_p(int(linear)), c_int64_p), C.cast(C.c_void_p(int(values)),
                                                                                      c_double_p),
                                 int(count), _iptr(dims), int(dims.size), C.byref(cfg),
                                 C.cast(C.c_void_p(int(truth)), c_double_p) if truth else None, 1, C.byref(h)))
    else:
        li = np.ascontiguousarray(np.asarray(linear, np.int64))
        va = np.ascontiguousarray(np.asarray(values, np.float64))
        tr = np.ascontiguousarray(np.asarray(truth, np.float64).reshape(-1)) if truth is not None else None
        check(lib().ttg_complete(_iptr(li), _dptr(va), int(li.size), _iptr(dims), int(dims.size), C.byref(cfg),
                                 _dptr(tr) if tr is not None else None, 0, C.byref(h)))
    del keep
    return Completion(h, int(dims.size), truth is not None)


# ---- factor level (factor.hpp) -------------------------------------------------------
def qr_col_pivot(a: np.ndarray):
    """qr_col_pivot (factor.hpp:19): returns (q m x p, r p x n, perm)."""
    require_gpu()
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    p = min(m, n)
    q = np.zeros((m, p), order="F")
    r = np.zeros((p, n), order="F")
    perm = np.zeros(n, np.int64)
    check(lib().ttg_qr_col_pivot(_dptr(a), m, n, _dptr(q), _dptr(r), _iptr(perm)))
    return q, r, perm


def utv(a: np.ndarray, lower: bool, refine_passes: int = 1):
    """ulv (lower) / urv (factor.hpp:56-57): returns (u m x p, t p x p, v n x p)."""
    require_gpu()
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    p = min(m, n)
    u, t, v = np.zeros((m, p), order="F"), np.zeros((p, p), order="F"), np.zeros((n, p), order="F")
    check(lib().ttg_utv(_dptr(a), m, n, int(bool(lower)), int(refine_passes), _dptr(u), _dptr(t), _dptr(v)))
    return u, t, v


def svd(a: np.ndarray, max_sweeps: int = 60, pair_tol: float = 1e-14):
    """svd (factor.hpp:34): returns (u m x p, s p, v n x p)."""
    require_gpu()
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    p = min(m, n)
    u, s, v = np.zeros((m, p), order="F"), np.zeros(p), np.zeros((n, p), order="F")
    check(lib().ttg_svd(_dptr(a), m, n, int(max_sweeps), float(pair_tol), _dptr(u), _dptr(s), _dptr(v)))
    return u, s, v


def reconstruct(cores: Sequence[np.ndarray], element_cap: int = 100_000_000) -> np.ndarray:
    """reconstruct (tt.hpp:60): dense tensor (order='F' n-d array) from cores."""
    require_gpu()
    dims = np.array([c.shape[1] for c in cores], np.int64)
    ranks = np.array([1] + [c.shape[2] for c in cores], np.int64)
    flat = np.concatenate([np.asarray(c, np.float64).ravel(order="F") for c in cores])
    out = np.empty(int(np.prod(dims)), np.float64)
    check(lib().ttg_reconstruct(_dptr(flat), _iptr(dims), _iptr(ranks), int(dims.size), int(element_cap), _dptr(out)))
    return out.reshape(tuple(dims), order="F")


def frobenius_norm(a) -> float:
    require_gpu()
    a = np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
    out = C.c_double()
    check(lib().ttg_frobenius_norm(a.ctypes.data_as(C.c_void_p), a.size, 0, C.byref(out)))
    return out.value


# ---- tensor algebra (tensor_ops.hpp, tt.hpp) ------------------------------------------
def mode_product(x: np.ndarray, m: np.ndarray, k: int) -> np.ndarray:
    """mode_product (tensor_ops.hpp:21): x (n-d, order='F' semantics) times m (rows x dims[k-1])
    along 1-based mode k; computed on the device in the reference's operation order."""
    require_gpu()
    x = np.asarray(x, np.float64)
    dims = np.array(x.shape, np.int64)
    m = np.asfortranarray(m, dtype=np.float64)
    flat = np.ascontiguousarray(x.ravel(order="F"))
    od = list(x.shape)
    if 1 <= k <= len(od):
        od[k - 1] = m.shape[0]
    out = np.empty(int(np.prod(od)), np.float64)
    check(lib().ttg_mode_product(_dptr(flat), _iptr(dims), int(dims.size), int(k), _dptr(m), m.shape[0], m.shape[1],
                                 _dptr(out)))
    return out.reshape(od, order="F")


def kron(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    require_gpu()
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    out = np.empty((a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]), order="F")
    check(lib().ttg_kron(_dptr(a), a.shape[0], a.shape[1], _dptr(b), b.shape[0], b.shape[1], _dptr(out)))
    return out


def psnr(estimate, truth) -> float:
    require_gpu()
    e = np.ascontiguousarray(np.asarray(estimate, np.float64).reshape(-1))
    t = np.ascontiguousarray(np.asarray(truth, np.float64).reshape(-1))
    if e.size != t.size:
        raise ArgumentError("psnr: shapes differ")
    out = C.c_double()
    check(lib().ttg_psnr(_dptr(e), _dptr(t), t.size, C.byref(out)))
    return out.value


def reverse_indices(x: np.ndarray) -> np.ndarray:
    """reverse_indices (tensor_ops.hpp:37): out(i_d, ..., i_1) = x(i_1, ..., i_d)."""
    require_gpu()
    x = np.asarray(x, np.float64)
    dims = np.array(x.shape, np.int64)
    flat = np.ascontiguousarray(x.ravel(order="F"))
    out = np.empty(flat.size, np.float64)
    check(lib().ttg_reverse_indices(_dptr(flat), _iptr(dims), int(dims.size), _dptr(out)))
    return out.reshape(tuple(reversed(x.shape)), order="F")


def reverse_tt(cores: Sequence[np.ndarray]) -> list:
    """reverse_tt (tt.hpp:63): the cores of the train with the mode order reversed."""
    require_gpu()
    dims = np.array([c.shape[1] for c in cores], np.int64)
    ranks = np.array([1] + [c.shape[2] for c in cores], np.int64)
    flat = np.concatenate([np.asarray(c, np.float64).ravel(order="F") for c in cores])
    out = np.empty_like(flat)
    check(lib().ttg_reverse_tt(_dptr(flat), _iptr(dims), _iptr(ranks), int(dims.size), _dptr(out)))
    res, off = [], 0
    for c in reversed(cores):
        shp = (c.shape[2], c.shape[1], c.shape[0])
        n = int(np.prod(shp))
        res.append(out[off:off + n].reshape(shp, order="F"))
        off += n
    return res


def kernel_launches() -> int:
    return int(lib().ttg_kernel_launches())
