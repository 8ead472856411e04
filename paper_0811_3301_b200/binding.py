"""Thin ctypes binding over libdtwlb.so (include/dtwlb.h).

Argument marshalling only: every step of the method runs in the library's CUDA
kernels.  Names and argument order follow the C ABI.  Tensors are torch tensors
(device memory from PyTorch; the current torch stream is passed as `stream`).
There is no CPU fallback: if the library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os
import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTWLB_LIB") or os.path.join(_HERE, "libdtwlb.so")

STATUS = {0: "OK", 1: "EINVAL", 2: "EUNSUPPORTED", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL"}
KEOGH_ONLY = 1
NO_PREFILTER = 2
NO_CASCADE = 4
NO_STREAM = 8
NO_ABANDON = 16
MAX_K = 1024


class DtwlbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


EXCHANGE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class NnOpts(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_float), ("index_base", ctypes.c_int64), ("query_block", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("exchange", EXCHANGE_FN), ("exchange_user", ctypes.c_void_p),
                ("db_env", ctypes.c_void_p), ("shards", ctypes.c_int32), ("exchange_walk", ctypes.c_int32),
                ("nccl_comm", ctypes.c_void_p)]


class _DeviceArray:
    """__cuda_array_interface__ view of a library-owned float32 device array (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None,
                                         "stream": torch.cuda.current_stream().cuda_stream}


def _exchange_callback(fn):
    """Wrap fn(thr: torch.Tensor) (a float32 CUDA view of the block's thresholds, lowered
    in place) as the C exchange callback of nn_opts."""
    def cb(ptr, count, _user):
        fn(torch.as_tensor(_DeviceArray(ptr, count), device=torch.device("cuda", torch.cuda.current_device())))
    return EXCHANGE_FN(cb)


class NnStats(ctypes.Structure):
    _fields_ = [("pairs", ctypes.c_int64), ("keogh_evaluated", ctypes.c_int64),
                ("improved_evaluated", ctypes.c_int64), ("dtw_evaluated", ctypes.c_int64),
                ("dtw_abandoned", ctypes.c_int64), ("dtw_cells_nominal", ctypes.c_int64),
                ("dtw_cells_computed", ctypes.c_int64), ("ms_envelope", ctypes.c_double),
                ("ms_keogh", ctypes.c_double), ("ms_select", ctypes.c_double),
                ("ms_improved", ctypes.c_double), ("ms_dtw", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("range1_improved", ctypes.c_int64),
                ("range1_dtw", ctypes.c_int64), ("range1_cells", ctypes.c_int64), ("walk_rounds", ctypes.c_int64),
                ("prefilter_evaluated", ctypes.c_int64), ("prefilter_segment", ctypes.c_int32),
                ("reserved_", ctypes.c_int32), ("ms_survivor_kernel", ctypes.c_double),
                ("ms_dtw_kernel", ctypes.c_double), ("survivor_entries", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["lb_envelope", "lb_keogh", "lb_piecewise", "lb_piecewise_sym", "lb_improved", "dtw_band", "nn_search",
           "nn_merge", "dtwlb_last_error", "dtwlb_release_workspace", "dtwlb_get_unique_id", "dtwlb_comm_init",
           "dtwlb_comm_destroy"]

_lib = None


def load():
    """Load libdtwlb.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_0811_3301_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.lb_envelope.argtypes = [vp, i32, i32, vp, vp, i64, vp]
        lib.lb_keogh.argtypes = [vp, vp, i64, i64, i32, i32, vp, vp]
        lib.lb_piecewise.argtypes = [vp, vp, i64, i64, i32, i32, vp, vp]
        lib.lb_improved.argtypes = [vp, vp, vp, i64, i64, i32, i32, i32, vp, vp]
        lib.lb_piecewise_sym.argtypes = [vp, vp, vp, i64, i64, i32, i32, i32, vp, vp]
        lib.dtw_band.argtypes = [vp, vp, i32, i32, i32, vp, i64, vp]
        lib.nn_search.argtypes = [vp, i64, vp, i64, i32, i32, i32, i32, vp, vp,
                                  ctypes.POINTER(NnOpts), ctypes.POINTER(NnStats), vp]
        lib.nn_merge.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp]
        for f in ("lb_envelope", "lb_keogh", "lb_piecewise", "lb_piecewise_sym", "lb_improved", "dtw_band",
                  "nn_search", "nn_merge"):
            getattr(lib, f).restype = ctypes.c_int
        lib.dtwlb_get_unique_id.argtypes = [vp]
        lib.dtwlb_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(ctypes.c_void_p)]
        lib.dtwlb_comm_destroy.argtypes = [vp]
        for f in ("dtwlb_get_unique_id", "dtwlb_comm_init", "dtwlb_comm_destroy"):
            getattr(lib, f).restype = ctypes.c_int
        lib.dtwlb_last_error.restype = ctypes.c_char_p
        lib.dtwlb_last_error.argtypes = []
        lib.dtwlb_release_workspace.restype = None
        _lib = lib
    return _lib


def _check(status: int):
    if status != 0:
        raise DtwlbError(status, load().dtwlb_last_error().decode())


def _stream():
    if not torch.cuda.is_available():
        return None  # the library reports ECUDA itself
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    return t.contiguous()


def lb_envelope(x: torch.Tensor, w: int):
    """U, L = envelope of each row of x [count][n]."""
    x = _dev(x, "x")
    n = x.shape[-1]
    count = x.numel() // n if n else 0
    U = torch.empty_like(x)
    L = torch.empty_like(x)
    _check(load().lb_envelope(x.data_ptr(), n, w, U.data_ptr(), L.data_ptr(), count, _stream()))
    return U, L


def lb_keogh(q_env: torch.Tensor, db: torch.Tensor, p: int) -> torch.Tensor:
    """[Q][N] LB_Keogh_p (rooted); q_env is [2][Q][n] (U block, then L block)."""
    q_env = _dev(q_env, "q_env")
    db = _dev(db, "db")
    Q, n = q_env.shape[1], q_env.shape[2]
    N = db.shape[0]
    out = torch.empty((Q, N), dtype=torch.float32, device=db.device)
    _check(load().lb_keogh(q_env.data_ptr(), db.data_ptr(), Q, N, n, p, out.data_ptr(), _stream()))
    return out


def lb_piecewise(q_env: torch.Tensor, db: torch.Tensor, p: int) -> torch.Tensor:
    """[Q][N] piecewise-sum bound (rooted, outward-rounded); q_env as lb_keogh."""
    q_env = _dev(q_env, "q_env")
    db = _dev(db, "db")
    Q, n = q_env.shape[1], q_env.shape[2]
    N = db.shape[0]
    out = torch.empty((Q, N), dtype=torch.float32, device=db.device)
    _check(load().lb_piecewise(q_env.data_ptr(), db.data_ptr(), Q, N, n, p, out.data_ptr(), _stream()))
    return out


def lb_piecewise_sym(q: torch.Tensor, q_env: torch.Tensor, db: torch.Tensor, w: int, p: int) -> torch.Tensor:
    """[Q][N] symmetric piecewise-sum bound: max of lb_piecewise(x | env y) and (y | env x) (rooted)."""
    q, q_env, db = _dev(q, "q"), _dev(q_env, "q_env"), _dev(db, "db")
    Q, n = q.shape
    N = db.shape[0]
    out = torch.empty((Q, N), dtype=torch.float32, device=db.device)
    _check(load().lb_piecewise_sym(q.data_ptr(), q_env.data_ptr(), db.data_ptr(), Q, N, n, w, p, out.data_ptr(),
                                   _stream()))
    return out


def lb_improved(q: torch.Tensor, q_env: torch.Tensor, db: torch.Tensor, w: int, p: int) -> torch.Tensor:
    """[Q][N] LB_Improved_p (rooted)."""
    q, q_env, db = _dev(q, "q"), _dev(q_env, "q_env"), _dev(db, "db")
    Q, n = q.shape
    N = db.shape[0]
    out = torch.empty((Q, N), dtype=torch.float32, device=db.device)
    _check(load().lb_improved(q.data_ptr(), q_env.data_ptr(), db.data_ptr(), Q, N, n, w, p, out.data_ptr(),
                              _stream()))
    return out


def dtw_band(x: torch.Tensor, y: torch.Tensor, w: int, p: int) -> torch.Tensor:
    """DTW_p(x[r], y[r]) for each row pair (rooted)."""
    x, y = _dev(x, "x"), _dev(y, "y")
    count, n = x.shape
    out = torch.empty(count, dtype=torch.float32, device=x.device)
    _check(load().dtw_band(x.data_ptr(), y.data_ptr(), n, w, p, out.data_ptr(), count, _stream()))
    return out


def _opts(eps, index_base, query_block, keogh_only, prefilter=True, cascade=True, exchange=None, stream=True,
          db_env=None, shards=0, exchange_walk=0, nccl_comm=None, abandon=True):
    o = NnOpts()
    o.nccl_comm = nccl_comm.handle if isinstance(nccl_comm, Communicator) else nccl_comm
    o.shards = shards
    o.exchange_walk = exchange_walk
    if exchange is not None:
        o.exchange = exchange
    o.eps = eps
    o.index_base = index_base
    o.query_block = query_block
    o.flags = (KEOGH_ONLY if keogh_only else 0) | (0 if prefilter else NO_PREFILTER) | \
        (0 if cascade else NO_CASCADE) | (0 if stream else NO_STREAM) | (0 if abandon else NO_ABANDON)
    o.db_env = db_env.data_ptr() if db_env is not None else None
    return o


def nn_search(queries, db, w: int, p: int, k: int, *, eps: float = 1e-3, index_base: int = 0,
              query_block: int = 0, keogh_only: bool = False, prefilter: bool = True, cascade: bool = True,
              stream: bool = True, db_env=None, exchange=None, out=None, shards: int = 0,
              exchange_walk: int = 0, nccl_comm=None, abandon: bool = True, return_stats: bool = False):
    """Exact k-NN under banded DTW_p.  Returns (idx int64 [Q][k], dist float32 [Q][k]).

    queries/db may be CUDA tensors (device path) or host tensors / numpy arrays
    (pinned host path: the library stages them; outputs are then host tensors).
    ``out`` optionally supplies (idx, dist) output tensors.  ``exchange(thr)`` (sharded
    search) is called once per query block after the first range with a float32 CUDA view
    of the block's thresholds, which it may lower in place (e.g. all-reduce MIN across
    shards; every rank must then pass the same ``query_block``).  ``stream=False`` disables the
    few-query streaming bound pass (DTWLB_NO_STREAM).  ``db_env`` optionally supplies the
    database index: a [2][N][n] CUDA tensor holding lb_envelope(db, w) (U block, then L block),
    reused instead of being computed in the call.  ``shards`` (database-sharded search) is the
    number of shards the exchange combines: each shard's best-first seed range is 1/shards of
    the single-database one (speed only); ``exchange_walk`` (0..3) adds that many exchange calls
    inside the last range's DTW walk (after its rounds 2, 4, 6): a block then makes
    1 + exchange_walk calls on every shard.  ``nccl_comm`` (a ``Communicator``) makes the library
    itself min-reduce the thresholds at those points with NCCL, instead of ``exchange``.
    ``abandon=False`` (DTWLB_NO_ABANDON) runs every DTW the bounds pass to its last row (no early
    abandon inside DTW; same k-NN).
    """
    host = not (isinstance(queries, torch.Tensor) and queries.is_cuda)
    if host:
        queries = torch.as_tensor(np.ascontiguousarray(queries, dtype=np.float32)) \
            if not isinstance(queries, torch.Tensor) else queries.contiguous()
        db = torch.as_tensor(np.ascontiguousarray(db, dtype=np.float32)) \
            if not isinstance(db, torch.Tensor) else db.contiguous()
    else:
        queries, db = _dev(queries, "queries"), _dev(db, "db")
    Q, n = queries.shape
    N = db.shape[0]
    if out is None:
        dev = "cpu" if host else queries.device
        idx = torch.empty((Q, k), dtype=torch.int64, device=dev, pin_memory=host)
        dist = torch.empty((Q, k), dtype=torch.float32, device=dev, pin_memory=host)
    else:
        idx, dist = out
    cb = _exchange_callback(exchange) if exchange is not None else None  # kept alive for the call
    if db_env is not None:
        db_env = _dev(db_env, "db_env")
        if tuple(db_env.shape) != (2, N, n):
            raise ValueError(f"db_env must be [2][N][n] = [2][{N}][{n}], got {tuple(db_env.shape)}")
    o = _opts(eps, index_base, query_block, keogh_only, prefilter, cascade, cb, stream, db_env, shards,
              exchange_walk, nccl_comm, abandon)
    st = NnStats()
    _check(load().nn_search(queries.data_ptr(), Q, db.data_ptr(), N, n, w, p, k, idx.data_ptr(),
                            dist.data_ptr(), ctypes.byref(o), ctypes.byref(st) if return_stats else None,
                            _stream()))
    if return_stats:
        return idx, dist, st.as_dict()
    return idx, dist


def nn_merge(in_idx: torch.Tensor, in_dist: torch.Tensor):
    """Merge [G][Q][k] shard lists into the global [Q][k] (k smallest by (dist, idx))."""
    G, Q, k = in_idx.shape
    in_idx = in_idx.contiguous()
    in_dist = _dev(in_dist, "in_dist")
    idx = torch.empty((Q, k), dtype=torch.int64, device=in_idx.device)
    dist = torch.empty((Q, k), dtype=torch.float32, device=in_idx.device)
    _check(load().nn_merge(in_idx.data_ptr(), in_dist.data_ptr(), G, Q, k, idx.data_ptr(), dist.data_ptr(),
                           _stream()))
    return idx, dist


def release_workspace():
    load().dtwlb_release_workspace()


class Communicator:
    """The library's NCCL communicator (dtwlb_comm_init) for the database-sharded search's
    threshold exchange (nn_opts.nccl_comm).  Create it on every rank with the same 128-byte id."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        if len(unique_id) != 128:
            raise ValueError("unique_id must be the 128 bytes of dtwlb_get_unique_id")
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(load().dtwlb_comm_init(buf, nranks, rank, ctypes.byref(h)))
        self.handle = h.value
        self.nranks, self.rank = nranks, rank

    def close(self):
        if self.handle:
            _check(load().dtwlb_comm_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def get_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().dtwlb_get_unique_id(buf))
    return buf.raw
