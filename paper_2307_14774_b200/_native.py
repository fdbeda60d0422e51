"""ctypes binding of libspc5_b200.so (the C ABI declared in include/spc5_b200.h).

Loaded on first use of ``lib`` (any entry point of the package that touches
the device); a missing or unloadable library raises ImportError there --
there is no CPU fallback anywhere in this package.  Loading lazily keeps the
host-only helpers (the seeded workload generators, the CSV records) usable
without the CUDA library, e.g. by bench.py's reference arm, which must not
load it.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libspc5_b200.so"

OK, EINVAL, ECURSOR, EINDEX, ECUDA, ENOMEM = range(6)
F32, F64 = 0, 1


class Spc5Info(ctypes.Structure):
    _fields_ = [("num_rows", ctypes.c_int64), ("num_cols", ctypes.c_int64),
                ("num_panels", ctypes.c_int64), ("num_blocks", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("r", ctypes.c_int32), ("vs", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("mask_bytes", ctypes.c_int32),
                ("block_base", ctypes.c_int64), ("num_chunks", ctypes.c_int64),
                ("num_split_chunks", ctypes.c_int64), ("footprint_bytes", ctypes.c_int64)]


_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_int = ctypes.c_int
_H = ctypes.c_void_p  # opaque handle

# name -> argtypes (restype int unless stated)
SIGNATURES = {
    "spc5_version": [],
    "spc5_last_error": [],
    "spc5_last_launch_count": [],
    "spc5_device_count": [ctypes.POINTER(_int)],
    "spc5_convert_csr": [_i64, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _i64, _vp,
                         ctypes.POINTER(_H)],
    "spc5_convert_timing": [_H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_double)],
    "spc5_import": [_i64, _i64, _int, _int, _int, _i64, _i64, _vp, _vp, _vp, _vp, _int, _i64,
                    _vp, ctypes.POINTER(_H)],
    "spc5_info": [_H, ctypes.POINTER(Spc5Info)],
    "spc5_prepare": [_H, _vp],
    "spc5_export": [_H, _vp, _vp, _vp, _vp, _int, _vp],
    "spc5_device_arrays": [_H, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                           ctypes.POINTER(_vp)],
    "spc5_spmv": [_H, _vp, _vp, _int, _vp],
    "spc5_spmv_panels": [_H, _i64, _i64, _vp, _vp, _int, _vp],
    "spc5_spmv_host": [_H, _vp, _vp, _int, _vp],
    "spc5_partition_by_nnz": [_H, _int, _vp, _vp],
    "spc5_block_value_offsets": [_H, _vp, _vp],
    "spc5_validate": [_H, _vp],
    "spc5_to_csr": [_H, _vp, _vp, _vp, _vp],
    "spc5_free": [_H],
    "spc5_csr_exact": [_i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "spc5_gen_stencil27_rowptr": [_i64, _i64, _i64, _vp, _vp],
    "spc5_gen_stencil27_fill": [_i64, _i64, _i64, _int, ctypes.c_uint64, ctypes.c_double, _vp,
                                _vp, _vp, _vp],
    "spc5_gen_stencil27_box_rowptr": [_i64, _i64, _i64, _i64, _vp, _vp],
    "spc5_gen_stencil27_box_fill": [_i64, _i64, _i64, _i64, _int, ctypes.c_uint64,
                                    ctypes.c_double, _vp, _vp, _vp, _vp],
    "spc5_spmv_mirrored": [_H, _vp, _vp, ctypes.c_double, _vp, _int, _i64, _vp],
    "spc5_gen_powerlaw_rowptr": [_i64, _i64, _i64, ctypes.c_uint64, _vp, _int, _vp, _vp],
    "spc5_gen_powerlaw_fill": [_i64, _i64, _i64, _int, ctypes.c_uint64, _vp, _int, _vp, _vp, _vp,
                               _vp],
    "spc5_gen_fem_rowptr": [_i64, _i64, _i64, _vp, _vp],
    "spc5_gen_fem_fill": [_i64, _i64, _i64, _int, ctypes.c_uint64, _vp, _vp, _vp, _vp],
    "spc5_mg_unique_id": [_vp],
    "spc5_mg_init": [_vp, _int, _int, ctypes.POINTER(_vp)],
    "spc5_mg_partition": [_vp, _i64, _int, _int, _vp, _vp],
    "spc5_mg_shard": [_vp, _H, _vp],
    "spc5_mg_spmv_step": [_vp, _vp, _vp, ctypes.c_double, _vp],
    "spc5_mg_free": [_vp],
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.spc5_last_error.restype = ctypes.c_char_p
    return lib


_lib = None
_lib_lock = threading.Lock()


def load():
    """The loaded library (loads it on the first call)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                _lib = _load()
    return _lib


def __getattr__(name):  # PEP 562: ``nat.lib`` loads on first access
    if name == "lib":
        return load()
    raise AttributeError(name)


class Spc5Error(RuntimeError):
    """CUDA / allocation failure inside the library."""


def check(status: int) -> None:
    """Map a C status to the exception the reference raises."""
    if status == OK:
        return
    msg = load().spc5_last_error().decode("utf-8", "replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status == ECURSOR:
        raise RuntimeError(msg)
    if status == EINDEX:
        raise IndexError(msg)
    raise Spc5Error(msg)


def last_launch_count() -> int:
    return int(load().spc5_last_launch_count())


def device_count() -> int:
    n = ctypes.c_int(0)
    load().spc5_device_count(ctypes.byref(n))
    return int(n.value)
