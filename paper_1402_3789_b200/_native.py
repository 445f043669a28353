"""ctypes binding of libnnm.so (the C ABI declared in include/nnm.h).

The product path has no CPU fallback: if the library is missing, fails to
load, or finds no usable sm_100 device, every compute call raises.  The
library is built in-tree (``python -m paper_1402_3789_b200.build`` or
``__graft_entry__.build()``) so that the exact ``.so`` that ran is the one in
the repository.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnnm.so")

NNM_OK = 0
NNM_E_INVALID = -1
NNM_E_CUDA = -2
NNM_E_UNSUPPORTED = -3
NNM_E_NOMEM = -4
NNM_E_CAPACITY = -5

ABI_VERSION = 4  # include/nnm.h NNM_ABI_VERSION
FLAG_ROUNDS = 1
PATH_NAMES = {0: "none", 1: "boruvka", 2: "rounds"}
STOP_NAMES = {1: "kl1-reached", 2: "no-eligible-pairs", 3: "single-cluster"}

# every symbol include/nnm.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "nnm_abi_version", "nnm_last_error", "nnm_device_count", "nnm_dataset_create",
    "nnm_dataset_create_device", "nnm_dataset_destroy", "nnm_top_p", "nnm_run",
    "nnm_pairwise", "nnm_bv_begin", "nnm_bv_scan", "nnm_bv_round_bound", "nnm_bv_round_phase1",
    "nnm_bv_round_phase2", "nnm_bv_cache_scatter", "nnm_bv_second", "nnm_bv_finish_round",
    "nnm_bv_end", "nnm_measure_fp32_peak", "nnm_tc_probe", "nnm_csv_load", "nnm_csv_fetch",
    "nnm_csv_free", "nnm_first_nonfinite", "nnm_round_log", "nnm_run_multi", "nnm_host_alloc",
    "nnm_host_free",
)


class Constraints(ctypes.Structure):
    _fields_ = [("kl1", ctypes.c_int64), ("kl2", ctypes.c_int64), ("kl3", ctypes.c_int64),
                ("kl4", ctypes.c_int64), ("dmax", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("device", ctypes.c_int32), ("scans", ctypes.c_int64),
                ("pairs_evaluated", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("ambiguous_rows", ctypes.c_int64),
                ("exact_evals", ctypes.c_int64), ("boruvka_rounds", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("pairs_covered", ctypes.c_double),
                ("prep_ms", ctypes.c_double), ("replay_ms", ctypes.c_double),
                ("tc_items", ctypes.c_int64), ("round_rescans", ctypes.c_int64),
                ("replay_gpu_merges", ctypes.c_int64)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["path"] = PATH_NAMES.get(self.path, str(self.path))
        return d


class RoundStat(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int64), ("ms", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("pairs_evaluated", ctypes.c_double), ("items", ctypes.c_int64),
                ("merged", ctypes.c_int64)]


def round_log(handle) -> list:
    """Per-round records of the last nnm_run on a dataset handle (nnm_round_log)."""
    lib = load()
    n = ctypes.c_int64()
    check(lib.nnm_round_log(handle, None, 0, ctypes.byref(n)))
    buf = (RoundStat * max(1, n.value))()
    check(lib.nnm_round_log(handle, buf, n.value, ctypes.byref(n)))
    return [{k: getattr(buf[i], k) for k, _ in RoundStat._fields_} for i in range(n.value)]


MERGE_DTYPE = np.dtype([("round", np.int64), ("root_a", np.int64), ("root_b", np.int64),
                        ("dist", np.float64), ("new_size", np.int64), ("point_a", np.int64),
                        ("point_b", np.int64)])
COUNTER_KEYS = ("round", "selected", "merged", "same_root", "kl2", "kl3", "unprocessed")
COUNTER_DTYPE = np.dtype([(k, np.int64) for k in COUNTER_KEYS])


class NativeError(RuntimeError):
    """libnnm reported a device-side failure."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lib = None
_lock = threading.Lock()


def load():
    """Load libnnm.so or raise; never falls back to a CPU path."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(the NNM path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        lib.nnm_abi_version.restype = ctypes.c_int
        if lib.nnm_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {lib.nnm_abi_version()}, this package needs "
                              f"{ABI_VERSION}: rebuild it with __graft_entry__.build()")
        lib.nnm_last_error.restype = ctypes.c_char_p
        lib.nnm_device_count.argtypes = [P(i32)]
        lib.nnm_dataset_create.argtypes = [vp, i64, i32, i32, P(vp)]
        lib.nnm_dataset_create_device.argtypes = [vp, i64, i32, i32, P(vp)]
        lib.nnm_dataset_destroy.argtypes = [vp]
        lib.nnm_top_p.argtypes = [vp, i32, vp, vp, dbl, i64, i64, i64, vp, vp, vp, P(i64)]
        lib.nnm_run.argtypes = [vp, i32, P(Constraints), i64, i32, vp, P(i64), vp, P(i64), P(i32),
                                vp, i64, P(i64), P(Stats)]
        lib.nnm_pairwise.argtypes = [i32, vp, i64, vp, i64, i32, i32, vp]
        lib.nnm_bv_begin.argtypes = [vp, i32, dbl, P(i64), P(i64)]
        lib.nnm_bv_scan.argtypes = [vp, i64, i64, vp, vp]
        lib.nnm_bv_round_bound.argtypes = [vp, i32, i32, vp, P(i64)]
        lib.nnm_bv_round_phase1.argtypes = [vp, i32, i32, vp, vp, vp]
        lib.nnm_bv_round_phase2.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, P(i64)]
        lib.nnm_bv_cache_scatter.argtypes = [vp]
        lib.nnm_run_multi.argtypes = [vp, i32, i32, P(Constraints), i64, i32, vp, P(i64), vp,
                                      P(i64), P(i32), vp, i64, P(i64), P(Stats)]
        lib.nnm_tc_probe.argtypes = [vp, vp, i64, P(dbl)]
        lib.nnm_csv_load.argtypes = [ctypes.c_char_p, ctypes.c_char, ctypes.c_char_p, i32, P(vp),
                                     P(i64), P(i64), P(i32), P(i64)]
        lib.nnm_csv_fetch.argtypes = [vp, vp, vp, vp]
        lib.nnm_csv_free.argtypes = [vp]
        lib.nnm_first_nonfinite.argtypes = [vp, i64, i32, P(i64)]
        lib.nnm_bv_second.argtypes = [vp, vp, vp, vp, vp]
        lib.nnm_bv_finish_round.argtypes = [vp, vp, vp, P(i64)]
        lib.nnm_bv_end.argtypes = [vp, i64, vp, P(i64), vp, P(i64), P(i32), P(Stats)]
        lib.nnm_measure_fp32_peak.argtypes = [i32, P(dbl)]
        lib.nnm_round_log.argtypes = [vp, vp, i64, P(i64)]
        lib.nnm_host_alloc.argtypes = [i64, P(vp)]
        lib.nnm_host_free.argtypes = [vp]
        for name in EXPORTED:
            if name not in ("nnm_abi_version", "nnm_last_error"):
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
        return lib


def first_nonfinite(values: np.ndarray) -> int:
    """Flat index of the first non-finite element of a C-contiguous float64 array, or -1."""
    lib = load()
    out = ctypes.c_int64(-1)
    check(lib.nnm_first_nonfinite(values.ctypes.data, int(values.size), 0, ctypes.byref(out)))
    return int(out.value)


HOST_OUT_MIN = 1 << 20        # smaller outputs stay ordinary numpy arrays
HOST_OUT_CAP = 8 << 30        # page-locked output bytes alive at once (then ordinary arrays)
_host_out = 0


def _host_release(addr: int, nbytes: int) -> None:
    global _host_out
    with _lock:
        _host_out -= nbytes
    if _lib is not None:
        _lib.nnm_host_free(addr)


def host_empty(count: int, dtype) -> np.ndarray:
    """Uninitialised 1-D output array, page-locked when large (nnm_host_alloc).

    libnnm detects page-locked merge / label outputs and has the GPU lay the records out
    and the copy engine write them (include/nnm.h).  The block returns to libnnm's pool
    when the last view of the array dies.  Falls back to an ordinary array when small,
    when the cap is reached or when no device is present."""
    global _host_out
    dtype = np.dtype(dtype)
    count = int(count)
    nbytes = count * dtype.itemsize
    if nbytes < HOST_OUT_MIN or gpu_count() == 0:
        return np.empty(count, dtype)
    with _lock:
        if _host_out + nbytes > HOST_OUT_CAP:
            return np.empty(count, dtype)
        _host_out += nbytes
    p = ctypes.c_void_p()
    if load().nnm_host_alloc(nbytes, ctypes.byref(p)) != NNM_OK or not p.value:
        with _lock:
            _host_out -= nbytes
        return np.empty(count, dtype)
    buf = (ctypes.c_char * nbytes).from_address(p.value)
    weakref.finalize(buf, _host_release, p.value, nbytes)
    return np.frombuffer(buf, dtype=dtype, count=count)


def check(rc: int) -> None:
    if rc == NNM_OK:
        return
    msg = (load().nnm_last_error() or b"").decode()
    if rc == NNM_E_INVALID:
        from .model import ValidationError

        raise ValidationError(msg)
    raise NativeError(rc, msg)


_gpu_count = None


def gpu_count() -> int:
    """Number of usable sm_100 devices (0 when there is none; cached)."""
    global _gpu_count
    if _gpu_count is None:
        c = ctypes.c_int32(0)
        try:
            _gpu_count = int(c.value) if load().nnm_device_count(ctypes.byref(c)) == NNM_OK else 0
        except ImportError:
            _gpu_count = 0
    return _gpu_count


def default_device() -> int:
    for var in ("NNM_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v:
            return int(v)
    return 0


class DeviceDataset:
    """A dataset resident in HBM (FP64 exact copy + FP32 screening tiles)."""

    def __init__(self, X=None, *, device: int | None = None, device_ptr: int | None = None,
                 n: int | None = None, d: int | None = None):
        lib = load()
        self.device = default_device() if device is None else int(device)
        h = ctypes.c_void_p()
        if device_ptr is not None:
            self.n, self.d = int(n), int(d)
            check(lib.nnm_dataset_create_device(ctypes.c_void_p(device_ptr), self.n, self.d,
                                                self.device, ctypes.byref(h)))
        else:
            X = np.ascontiguousarray(X, dtype=np.float64)
            self.n, self.d = X.shape
            check(lib.nnm_dataset_create(X.ctypes.data, self.n, self.d, self.device,
                                         ctypes.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, lib.nnm_dataset_destroy, h)

    def close(self):
        self._fin()


def device_dataset(dataset) -> DeviceDataset:
    """Per-Dataset cached device copy (Dataset is frozen with read-only arrays,
    so the cache cannot go stale; model.py:29-76)."""
    dd = getattr(dataset, "_device_cache", None)
    dev = default_device()
    if dd is None or dd.device != dev:
        dd = DeviceDataset(dataset.values, device=dev)
        object.__setattr__(dataset, "_device_cache", dd)
    return dd


def load_csv(path: str, *, delimiter: str = ",", id_column=None, threads: int = 0):
    """Native CSV ingestion (nnm_csv_load): returns (values float64 (n, d), ids list or None).
    Raises ValidationError with the reference's messages (dataio.py:49-116)."""
    lib = load()
    if len(delimiter.encode("utf-8")) != 1:
        raise NotImplementedError("native CSV ingestion needs a single-byte delimiter")
    h = ctypes.c_void_p()
    n, d, nid = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    has = ctypes.c_int32()
    idc = None if id_column is None else str(id_column).encode("utf-8")
    check(lib.nnm_csv_load(os.fsencode(path), delimiter.encode("utf-8"), idc, int(threads),
                           ctypes.byref(h), ctypes.byref(n), ctypes.byref(d), ctypes.byref(has),
                           ctypes.byref(nid)))
    try:
        values = np.empty((n.value, d.value), dtype=np.float64)
        ids = None
        if has.value:
            buf = ctypes.create_string_buffer(max(1, nid.value))
            offs = np.empty(n.value + 1, dtype=np.int64)
            check(lib.nnm_csv_fetch(h, values.ctypes.data, buf, offs.ctypes.data))
            raw = buf.raw[: nid.value]
            ids = [raw[offs[i]:offs[i + 1]].decode("utf-8") for i in range(n.value)]
        else:
            check(lib.nnm_csv_fetch(h, values.ctypes.data, None, None))
    finally:
        lib.nnm_csv_free(h)
    return values, ids
