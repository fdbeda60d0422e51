"""Loaders for the golden fixtures in tests/golden/ (made by make_golden.py from the reference)."""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@dataclass
class Csr:
    """Duck-typed CsrMatrix (reference mmio.py:84-100 field names)."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def precision(self) -> str:
        return "f32" if self.values.dtype == np.float32 else "f64"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@lru_cache(maxsize=None)
def expected_small() -> dict:
    return json.loads((GOLDEN / "expected_small.json").read_text())


@lru_cache(maxsize=None)
def _inputs():
    with np.load(GOLDEN / "inputs_small.npz") as z:
        return {k: z[k] for k in z.files}


def small_case(name: str) -> Csr:
    a = _inputs()
    nr, nc = (int(v) for v in a[f"{name}__shape"])
    return Csr(nr, nc, a[f"{name}__row_ptr"].copy(), a[f"{name}__col_idx"].copy(),
               a[f"{name}__values"].copy())


def small_case_names() -> list[str]:
    return list(expected_small()["cases"].keys())


def case_x(name: str, m) -> np.ndarray:
    idx = expected_small()["cases"][name]["index"]
    return np.random.default_rng(100 + idx).uniform(-1, 1, m.num_cols).astype(m.values.dtype)


@lru_cache(maxsize=None)
def config1() -> dict:
    return json.loads((GOLDEN / "config1.json").read_text())


@lru_cache(maxsize=None)
def stencil() -> dict:
    return json.loads((GOLDEN / "stencil.json").read_text())


def fmt_keys(rec: dict):
    for key, f in rec["formats"].items():
        r, vs = (int(v) for v in key.split(","))
        yield r, vs, f
