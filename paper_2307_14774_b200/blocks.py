"""SPC5 beta(r, vs) storage on the GPU: the reference ``spc5.blocks`` surface.

Same names, fields and error behaviour as
/root/reference/pkg/src/spc5/blocks.py, with the data living in HBM:

* ``csr_to_spc5`` (blocks.py:96-143) runs K1 (csrc/convert.cu) and returns a
  device-backed :class:`Spc5Matrix`; its four arrays are fetched to numpy
  lazily, on first attribute access.
* A :class:`Spc5Matrix` built from host arrays (``load_spc5``, user code, or
  fault injection that rewrites a mask in place, cli.py:114-127) is uploaded
  on its next kernel call: writes through the numpy views mark it dirty, so the
  device copy never goes stale (SURVEY 8(b) "Ownership & mutability").
* ``spc5_to_csr`` and ``validate_spc5`` run on the device (csrc/convert.cu,
  csrc/plan.cu).  ``filling_stats``/``footprint_comparison`` are byte
  arithmetic on the counts; ``save_spc5``/``load_spc5`` are file I/O with the
  reference's 60-byte little-endian header (blocks.py:235-272).
"""

from __future__ import annotations

import ctypes
import struct
import weakref
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as nat
from .mmio import CsrMatrix

__all__ = ["Spc5Matrix", "FillingStats", "VALID_R", "VALID_VS", "mask_dtype", "csr_to_spc5",
           "csr_to_spc5_device", "spc5_to_csr", "filling_stats", "footprint_comparison",
           "validate_spc5", "save_spc5", "load_spc5"]

VALID_R = (1, 2, 4, 8)
VALID_VS = (4, 8, 16)
_INDEX_BYTES = 4
_MAGIC = b"SPC5"
_VERSION = 1
_HEAD = "<4sIIIqqBxxxqqq"


def mask_dtype(vs: int) -> np.dtype:
    """u8 for vs <= 8, u16 for vs = 16 (blocks.py:46-48)."""
    return np.dtype(np.uint8) if vs <= 8 else np.dtype(np.uint16)


def _check_shape(r: int, vs: int) -> None:
    if r not in VALID_R:
        raise ValueError(f"r must be one of {VALID_R}, got {r}")
    if vs not in VALID_VS:
        raise ValueError(f"vs must be one of {VALID_VS}, got {vs}")


def torch_stream() -> int:
    """Raw cudaStream_t of torch's current stream (0 when torch has no CUDA)."""
    import torch
    if not torch.cuda.is_available():
        return 0
    return int(torch.cuda.current_stream().cuda_stream)


class _Tracked(np.ndarray):
    """numpy view whose in-place writes mark the owning matrix dirty."""

    def __array_finalize__(self, obj):
        owner = getattr(obj, "_owner", None)
        self._owner = owner if self.base is not None else None

    def _touch(self):
        o = self._owner() if self._owner is not None else None
        if o is not None:
            o._host_dirty = True

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._touch()

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        outs = kwargs.get("out", ())
        for o in outs:
            if isinstance(o, _Tracked):
                o._touch()
        args = [i.view(np.ndarray) if isinstance(i, _Tracked) else i for i in inputs]
        if outs:
            kwargs["out"] = tuple(o.view(np.ndarray) if isinstance(o, _Tracked) else o
                                  for o in outs)
        return getattr(ufunc, method)(*args, **kwargs)


class _Handle:
    """Owns one spc5_matrix_t."""

    def __init__(self, ptr: int):
        self.ptr = ctypes.c_void_p(ptr)
        self.info = nat.Spc5Info()
        nat.check(nat.lib.spc5_info(self.ptr, ctypes.byref(self.info)))

    def refresh(self):
        nat.check(nat.lib.spc5_info(self.ptr, ctypes.byref(self.info)))

    def convert_timing(self) -> dict:
        """Device times (ms) of the K1 conversion that built this matrix."""
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        nat.check(nat.lib.spc5_convert_timing(self.ptr, ctypes.byref(a), ctypes.byref(b),
                                              ctypes.byref(c)))
        return {"k1_count_ms": a.value, "k1_fill_ms": b.value, "plan_ms": c.value}

    def __del__(self):
        try:
            if self.ptr:
                nat.lib.spc5_free(self.ptr)
                self.ptr = ctypes.c_void_p(0)
        except Exception:
            pass


_FIELDS = ("block_rowptr", "block_colidx", "block_masks", "values")


class Spc5Matrix:
    """Block-format matrix (blocks.py:51-78), device resident.

    Constructed like the reference dataclass
    ``Spc5Matrix(num_rows, num_cols, r, vs, block_rowptr, block_colidx,
    block_masks, values)`` from host arrays, or returned device-backed by
    :func:`csr_to_spc5`.
    """

    def __init__(self, num_rows, num_cols, r, vs, block_rowptr=None, block_colidx=None,
                 block_masks=None, values=None, *, _handle: _Handle | None = None,
                 block_base: int = 0):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        self.r = int(r)
        self.vs = int(vs)
        self.block_base = int(block_base)
        self._h = _handle
        self._host = {}
        self._host_dirty = False
        if _handle is None:
            for name, arr in zip(_FIELDS, (block_rowptr, block_colidx, block_masks, values)):
                setattr(self, name, arr)

    # ---- fields ------------------------------------------------------------
    def _get(self, name):
        if name not in self._host:
            if self._h is None:
                return None
            self._fetch()
        return self._host[name]

    def _set(self, name, arr):
        arr = np.asarray(arr)
        t = arr.view(_Tracked)
        t._owner = weakref.ref(self)
        self._host[name] = t
        self._host_dirty = True

    def _fetch(self):
        info = self._h.info
        mdt = mask_dtype(self.vs)
        vdt = np.float64 if info.precision == nat.F64 else np.float32
        rp = np.empty(info.num_panels + 1, np.int64)
        ci = np.empty(info.num_blocks, np.uint32)
        mk = np.empty(info.num_blocks * info.r, mdt)
        va = np.empty(info.nnz, vdt)
        nat.check(nat.lib.spc5_export(self._h.ptr, rp.ctypes.data, ci.ctypes.data,
                                      mk.ctypes.data, va.ctypes.data, 1, torch_stream()))
        dirty = self._host_dirty
        for name, arr in zip(_FIELDS, (rp, ci, mk, va)):
            self._set(name, arr)
        self._host_dirty = dirty

    block_rowptr = property(lambda s: s._get("block_rowptr"),
                            lambda s, v: s._set("block_rowptr", v))
    block_colidx = property(lambda s: s._get("block_colidx"),
                            lambda s, v: s._set("block_colidx", v))
    block_masks = property(lambda s: s._get("block_masks"),
                           lambda s, v: s._set("block_masks", v))
    values = property(lambda s: s._get("values"), lambda s, v: s._set("values", v))

    @property
    def num_panels(self) -> int:
        if self._h is not None and not self._host_dirty:
            return int(self._h.info.num_panels)
        return len(self.block_rowptr) - 1

    @property
    def num_blocks(self) -> int:
        if self._h is not None and not self._host_dirty:
            return int(self._h.info.num_blocks)
        return len(self.block_colidx)

    @property
    def nnz(self) -> int:
        if self._h is not None and not self._host_dirty:
            return int(self._h.info.nnz)
        return len(self.values)

    @property
    def dtype(self) -> np.dtype:
        if self._h is not None and not self._host_dirty:
            return np.dtype(np.float64 if self._h.info.precision == nat.F64 else np.float32)
        return self.values.dtype

    @property
    def precision(self) -> str:
        return "f32" if self.dtype == np.float32 else "f64"

    def __repr__(self):
        return (f"Spc5Matrix({self.num_rows}x{self.num_cols}, beta({self.r},{self.vs}), "
                f"{self.precision}, nb={self.num_blocks}, nnz={self.nnz})")

    # ---- device side -------------------------------------------------------
    def handle(self, stream: int | None = None) -> _Handle:
        """The device handle, (re-)uploading host arrays when they changed."""
        if self._h is None or self._host_dirty:
            self._h = _import_host(self, torch_stream() if stream is None else stream)
            self._host_dirty = False
        return self._h

    @property
    def device_resident(self) -> bool:
        return self._h is not None and not self._host_dirty

    def footprint_bytes(self) -> int:
        return filling_stats(self).footprint_bytes


def as_spc5(s) -> Spc5Matrix:
    """Accept our matrix or any object with the reference Spc5Matrix fields."""
    if isinstance(s, Spc5Matrix):
        return s
    return Spc5Matrix(s.num_rows, s.num_cols, s.r, s.vs, s.block_rowptr, s.block_colidx,
                      s.block_masks, s.values)


def _import_host(s: Spc5Matrix, stream: int) -> _Handle:
    _check_shape(s.r, s.vs)
    rp = np.ascontiguousarray(s.block_rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(s.block_colidx)
    if ci.size and (ci.min() < 0 or ci.max() > 0xFFFFFFFF):
        raise ValueError("block_colidx out of uint32 range")
    ci = ci.astype(np.uint32, copy=False)
    mk = np.ascontiguousarray(s.block_masks)
    mdt = mask_dtype(s.vs)
    if mk.size and int(mk.max()) >> (8 * mdt.itemsize):
        raise ValueError("mask has bits beyond vs")
    mk = mk.astype(mdt, copy=False)
    va = np.ascontiguousarray(s.values)
    if va.dtype not in (np.float32, np.float64):
        raise ValueError("values must be float32 or float64")
    num_panels = (s.num_rows + s.r - 1) // s.r
    if len(rp) != num_panels + 1:
        raise ValueError("block_rowptr length does not match panel count")
    if len(mk) != len(ci) * s.r:
        raise ValueError("mask array length must be num_blocks * r")
    out = ctypes.c_void_p()
    nat.check(nat.lib.spc5_import(s.num_rows, s.num_cols, s.r, s.vs,
                                  nat.F64 if va.dtype == np.float64 else nat.F32,
                                  len(ci), len(va), rp.ctypes.data, ci.ctypes.data,
                                  mk.ctypes.data, va.ctypes.data, 1, s.block_base, stream,
                                  ctypes.byref(out)))
    return _Handle(out.value)


# ---- conversion ------------------------------------------------------------

def csr_to_spc5_device(num_rows: int, num_cols: int, row_ptr, col_idx, values, r: int, vs: int,
                       block_base: int = 0) -> Spc5Matrix:
    """K1 on device CSR arrays (torch CUDA tensors int64 / int32 / f32|f64)."""
    _check_shape(r, vs)
    import torch
    if values.dtype == torch.float64:
        prec = nat.F64
    elif values.dtype == torch.float32:
        prec = nat.F32
    else:
        raise ValueError("values must be float32 or float64")
    row_ptr = row_ptr.contiguous()
    col_idx = col_idx.contiguous()
    values = values.contiguous()
    if row_ptr.dtype != torch.int64 or col_idx.dtype != torch.int32:
        raise ValueError("row_ptr must be int64 and col_idx int32")
    if row_ptr.numel() != num_rows + 1:
        raise ValueError("row_ptr must have num_rows + 1 entries")
    out = ctypes.c_void_p()
    nat.check(nat.lib.spc5_convert_csr(num_rows, num_cols, values.numel(), prec, r, vs,
                                       row_ptr.data_ptr(), col_idx.data_ptr(),
                                       values.data_ptr(), block_base, torch_stream(),
                                       ctypes.byref(out)))
    return Spc5Matrix(num_rows, num_cols, r, vs, _handle=_Handle(out.value),
                      block_base=block_base)


def csr_to_spc5(m, r: int, vs: int, block_base: int = 0) -> Spc5Matrix:
    """Convert CSR to beta(r, vs) on the GPU; bit-exact with blocks.py:96-143."""
    _check_shape(r, vs)
    import torch
    if m.values.dtype not in (np.float32, np.float64):
        raise ValueError("values must be float32 or float64")
    dev = torch.device("cuda", torch.cuda.current_device())
    rp = torch.from_numpy(np.ascontiguousarray(m.row_ptr, dtype=np.int64)).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(m.col_idx, dtype=np.int32)).to(dev)
    va = torch.from_numpy(np.ascontiguousarray(m.values)).to(dev)
    s = csr_to_spc5_device(int(m.num_rows), int(m.num_cols), rp, ci, va, r, vs, block_base)
    del rp, ci, va
    return s


def spc5_to_csr(s) -> CsrMatrix:
    """Invert the block conversion on the device (blocks.py:146-168)."""
    import torch
    s = as_spc5(s)
    h = s.handle()
    info = h.info
    dev = torch.device("cuda", torch.cuda.current_device())
    vdt = torch.float64 if info.precision == nat.F64 else torch.float32
    rp = torch.empty(s.num_rows + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(max(info.nnz, 1), dtype=torch.int32, device=dev)
    va = torch.empty(max(info.nnz, 1), dtype=vdt, device=dev)
    nat.check(nat.lib.spc5_to_csr(h.ptr, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                  torch_stream()))
    torch.cuda.current_stream().synchronize()
    n = info.nnz
    return CsrMatrix(s.num_rows, s.num_cols, rp.cpu().numpy(), ci[:n].cpu().numpy(),
                     va[:n].cpu().numpy())


# ---- statistics / checks / cache --------------------------------------------

@dataclass
class FillingStats:
    num_blocks: int
    avg_nnz_per_block: float
    filling: float
    footprint_bytes: int


def filling_stats(s) -> FillingStats:
    """Block count, mean entries per block, filling, bytes (blocks.py:176-189)."""
    nb, nnz = s.num_blocks, s.nnz
    capacity = nb * s.r * s.vs
    itemsize = 4 if s.precision == "f32" else 8
    footprint = (nnz * itemsize + nb * _INDEX_BYTES + nb * s.r * mask_dtype(s.vs).itemsize
                 + (s.num_panels + 1) * _INDEX_BYTES)
    return FillingStats(num_blocks=nb, avg_nnz_per_block=nnz / nb if nb else 0.0,
                        filling=nnz / capacity if capacity else 0.0, footprint_bytes=footprint)


def footprint_comparison(m, r: int, vs: int) -> tuple[int, int]:
    """(csr_bytes, spc5_bytes) with 4-byte indices (blocks.py:192-198)."""
    csr_bytes = ((m.num_rows + 1) * _INDEX_BYTES + m.nnz * _INDEX_BYTES
                 + m.nnz * m.values.dtype.itemsize)
    return csr_bytes, filling_stats(csr_to_spc5(m, r, vs)).footprint_bytes


def validate_spc5(s) -> None:
    """Structural invariants on the device; ValueError with the reference's message."""
    _check_shape(s.r, s.vs)
    s = as_spc5(s)
    if not s.device_resident:
        if len(s.block_rowptr) != (s.num_rows + s.r - 1) // s.r + 1:
            raise ValueError("block_rowptr length does not match panel count")
        if len(s.block_masks) != len(s.block_colidx) * s.r:
            raise ValueError("mask array length must be num_blocks * r")
    nat.check(nat.lib.spc5_validate(s.handle().ptr, torch_stream()))


def save_spc5(s, path) -> None:
    """Little-endian binary cache, the reference layout (blocks.py:235-248)."""
    header = struct.pack(_HEAD, _MAGIC, _VERSION, s.r, s.vs, s.num_rows, s.num_cols,
                         0 if s.precision == "f32" else 1, s.nnz, s.num_blocks, s.num_panels)
    mdt = "<u1" if s.vs <= 8 else "<u2"
    vdt = "<f4" if s.precision == "f32" else "<f8"
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.asarray(s.block_rowptr).astype("<u4").tobytes())
        fh.write(np.asarray(s.block_colidx).astype("<u4").tobytes())
        fh.write(np.asarray(s.block_masks).astype(mdt).tobytes())
        fh.write(np.asarray(s.values).astype(vdt).tobytes())


def load_spc5(path) -> Spc5Matrix:
    """Read a file written by :func:`save_spc5` bit-exactly (blocks.py:251-272)."""
    raw = Path(path).read_bytes()
    magic, version, r, vs, num_rows, num_cols, prec, nnz, nb, npanels = \
        struct.unpack_from(_HEAD, raw)
    if magic != _MAGIC:
        raise ValueError(f"not a block-matrix cache file: bad magic {magic!r}")
    if version != _VERSION:
        raise ValueError(f"unsupported cache version {version}")
    mdt = np.dtype("<u1") if vs <= 8 else np.dtype("<u2")
    vdt = np.dtype("<f4") if prec == 0 else np.dtype("<f8")
    off = struct.calcsize(_HEAD)
    rowptr = np.frombuffer(raw, "<u4", npanels + 1, off).astype(np.int64)
    off += (npanels + 1) * 4
    colidx = np.frombuffer(raw, "<u4", nb, off).copy()
    off += nb * 4
    masks = np.frombuffer(raw, mdt, nb * r, off).copy()
    off += nb * r * mdt.itemsize
    values = np.frombuffer(raw, vdt, nnz, off).astype(vdt.newbyteorder("="))
    return Spc5Matrix(num_rows, num_cols, r, vs, rowptr, colidx, masks, values)


# ---- per-rank shard files -------------------------------------
# The reference cache (blocks.py:235-272) stores block_rowptr as u4 and knows
# nothing about shards: the 400^3 matrices have > 2^32 / 8 blocks per format
# on few ranks and are only ever held as row-panel shards.  Version 2 keeps
# the reference's array order and little-endian layout, widens block_rowptr to
# i8 and records where the shard sits in the global matrix.
_SHARD_VERSION = 2
_SHARD_HEAD = "<4sIIIqqBxxxqqq" + "qqqii"  # v1 header + global_rows, row_lo, block_base, rank, world
_IO_CHUNK = 1 << 26  # elements per write/read call (bounded host staging)


def save_spc5_shard(s, path, *, global_rows: int, row_lo: int, rank: int, world: int) -> None:
    """Write rank `rank`'s row-panel shard (rows [row_lo, row_lo + s.num_rows) of a
    global_rows-row matrix, its blocks numbered from s.block_base)."""
    s = as_spc5(s)
    header = struct.pack(_SHARD_HEAD, _MAGIC, _SHARD_VERSION, s.r, s.vs, s.num_rows, s.num_cols,
                         0 if s.precision == "f32" else 1, s.nnz, s.num_blocks, s.num_panels,
                         int(global_rows), int(row_lo), int(s.block_base), int(rank), int(world))
    mdt = "<u1" if s.vs <= 8 else "<u2"
    vdt = "<f4" if s.precision == "f32" else "<f8"
    with open(path, "wb") as fh:
        fh.write(header)
        for arr, dt in ((s.block_rowptr, "<i8"), (s.block_colidx, "<u4"), (s.block_masks, mdt),
                        (s.values, vdt)):
            a = np.asarray(arr)
            for i in range(0, a.size, _IO_CHUNK):
                fh.write(a[i:i + _IO_CHUNK].astype(dt, copy=False).tobytes())


def load_spc5_shard(path):
    """Read a shard file: (Spc5Matrix with its block_base, metadata dict)."""
    hs = struct.calcsize(_SHARD_HEAD)
    with open(path, "rb") as fh:
        head = fh.read(hs)
        if len(head) < hs:
            raise ValueError("truncated shard file")
        (magic, version, r, vs, num_rows, num_cols, prec, nnz, nb, npanels, global_rows, row_lo,
         block_base, rank, world) = struct.unpack(_SHARD_HEAD, head)
        if magic != _MAGIC:
            raise ValueError(f"not a block-matrix cache file: bad magic {magic!r}")
        if version != _SHARD_VERSION:
            raise ValueError(f"unsupported shard cache version {version}")
        mdt = np.dtype("<u1") if vs <= 8 else np.dtype("<u2")
        vdt = np.dtype("<f4") if prec == 0 else np.dtype("<f8")

        def read(dt, count):
            out = np.fromfile(fh, dtype=dt, count=count)
            if out.size != count:
                raise ValueError("truncated shard file")
            return out
        rowptr = read(np.dtype("<i8"), npanels + 1)
        colidx = read(np.dtype("<u4"), nb)
        masks = read(mdt, nb * r)
        values = read(vdt, nnz)
    s = Spc5Matrix(num_rows, num_cols, r, vs, rowptr, colidx, masks, values, block_base=block_base)
    return s, {"global_rows": global_rows, "row_lo": row_lo, "rank": rank, "world": world}
