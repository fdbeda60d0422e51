"""Seeded synthetic workloads for the five BASELINE.json configs.

No public matrix suite is used (SuiteSparse is absent offline); these
generators stand in with the shapes, sizes and value distributions that
BASELINE.json names.  Host versions (numpy) live here; the device versions
(``spc5_gen_stencil27_*``, ``spc5_gen_powerlaw_*``, ``spc5_gen_fem_*`` in
csrc/aux.cu) produce bit-identical CSR arrays so a row slice generated on the
host checks a slice of a device-generated matrix (the sliced oracle, SURVEY.md
8(c)).  Column sampling is stratified with integer arithmetic only (distinct
and sorted by construction, no transcendental functions on either side), and
the lognormal row lengths of config 3 come from a quantile table made here
once and handed to the device.

Values are position keyed, ``v(i, j) = 2*u(i, j) - 1`` with
``u = (splitmix64((i << 32) ^ j ^ seedmix) >> 11) * 2**-53`` -- the scheme the
reference uses for ``make_dense`` (mmio.py:304-322) -- so any row range can be
regenerated without materialising the matrix.  The stencil diagonal is 27
(BASELINE config 2; config 5 leaves it open and uses the same choice).
"""

from __future__ import annotations

import numpy as np

from .mmio import CsrMatrix, dtype_for, make_random, mix64

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MATRIX_SEED = 0
X_SEED = 1

# (dz, dy, dx) in lexicographic order => columns ascend within a row
STENCIL27 = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def seed_mix(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return mix64(np.array([np.uint64(seed) + GOLDEN], dtype=np.uint64))[0]


def keyed_uniform(i: np.ndarray, j: np.ndarray, seed: int) -> np.ndarray:
    """U(-1, 1) in float64, a pure function of (i, j, seed)."""
    key = (np.asarray(i, np.uint64) << np.uint64(32)) ^ np.asarray(j, np.uint64) ^ seed_mix(seed)
    u = (mix64(key) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0


def stencil27_rows(n: int, lo: int, hi: int, precision: str = "f64", seed: int = MATRIX_SEED,
                   diag: float = 27.0, nz: int | None = None) -> CsrMatrix:
    """Rows [lo, hi) of the 27-point stencil on an n x n x nz grid (nz = n: the
    n^3 cube), row = (z*n + y)*n + x.

    Returned as a CSR with ``hi - lo`` rows and ``n*n*nz`` columns; the full
    matrix is ``stencil27_rows(n, 0, n**3)``.  Twin of csrc/aux.cu stencil_*
    (``spc5_gen_stencil27[_box]_*``).
    """
    dtype = dtype_for(precision)
    nz = n if nz is None else nz
    N = n * n * nz
    lo, hi = max(0, lo), min(N, hi)
    i = np.arange(lo, hi, dtype=np.int64)
    z, y, x = i // (n * n), (i // n) % n, i % n
    cols = np.empty((len(i), 27), dtype=np.int64)
    valid = np.empty((len(i), 27), dtype=bool)
    for k, (dz, dy, dx) in enumerate(STENCIL27):
        valid[:, k] = ((z + dz >= 0) & (z + dz < nz) & (y + dy >= 0) & (y + dy < n)
                       & (x + dx >= 0) & (x + dx < n))
        cols[:, k] = i + dz * n * n + dy * n + dx
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(len(i) + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    rows_flat = np.broadcast_to(i[:, None], cols.shape)[valid]
    cols_flat = cols[valid]
    vals = keyed_uniform(rows_flat, cols_flat, seed)
    vals[rows_flat == cols_flat] = diag
    return CsrMatrix(len(i), N, row_ptr, cols_flat.astype(np.int32), vals.astype(dtype))


def stencil27(n: int, precision: str = "f64", seed: int = MATRIX_SEED) -> CsrMatrix:
    return stencil27_rows(n, 0, n ** 3, precision, seed)


def stencil27_nnz(n: int) -> int:
    return (3 * n - 2) ** 3


def x_vector(num_cols: int, precision: str = "f64", seed: int = X_SEED) -> np.ndarray:
    """x ~ U(-1, 1) drawn like the reference harness does (bench.py:168-169)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=num_cols).astype(dtype_for(precision))


def config1(seed: int = MATRIX_SEED) -> CsrMatrix:
    """BASELINE config 1: make_random(8192, 8192, 16, 0.0, seed), f64 (use as-is)."""
    return make_random(8192, 8192, 16, 0.0, seed, "f64")


# ---------------------------------------------------------------- config 3
PL_N = 4_194_304
PL_WINDOW = 4096
PL_TABLE_BITS = 12
PL_SALT = np.uint64(0x5BD1E995)


def powerlaw_len_table(bits: int = PL_TABLE_BITS, mean: float = 16.0, sigma: float = 1.5,
                       max_len: int = 8192) -> np.ndarray:
    """Row lengths: 2^bits quantiles of lognormal(mean, sigma), rounded, clipped to [1, max_len]."""
    from scipy.special import ndtri
    k = 1 << bits
    q = (np.arange(k, dtype=np.float64) + 0.5) / k
    mu = np.log(mean) - sigma * sigma / 2.0
    return np.clip(np.rint(np.exp(mu + sigma * ndtri(q))), 1, max_len).astype(np.int32)


def _pl_key(seedmix, i: int, s, tag: int) -> np.ndarray:
    s = np.asarray(s, dtype=np.uint64)
    return mix64(seedmix ^ (np.uint64(i) << np.uint64(24)) ^ (s << np.uint64(2)) ^ np.uint64(tag))


def _strata(lo: int, width: int, k: int, key: np.ndarray) -> np.ndarray:
    s = np.arange(k, dtype=np.int64)
    a = lo + s * width // k
    b = lo + (s + 1) * width // k
    return a + (key % (b - a).astype(np.uint64)).astype(np.int64)


def powerlaw_rows(lo: int, hi: int, n: int = PL_N, precision: str = "f32",
                  seed: int = MATRIX_SEED, table: np.ndarray | None = None) -> CsrMatrix:
    """Rows [lo, hi) of the config-3 power-law matrix (twin of csrc/aux.cu powerlaw_*).

    Row i: length from the quantile table, 80 % of the columns stratified over
    i +- 4096, the rest stratified over [0, n), merged without duplicates;
    values U(-1, 1) keyed by (i, j).
    """
    table = powerlaw_len_table() if table is None else table
    bits = int(np.log2(len(table)))
    seedmix = seed_mix(seed) ^ PL_SALT
    cols, ptr = [], [0]
    for i in range(lo, hi):
        ln = int(table[int(_pl_key(seedmix, i, 0, 0)) >> (64 - bits)])
        lo_w, hi_w = max(0, i - PL_WINDOW), min(n - 1, i + PL_WINDOW)
        w = hi_w - lo_w + 1
        k_loc = min((4 * ln + 2) // 5, w)
        k_uni = min(ln - k_loc, n)
        loc = _strata(lo_w, w, k_loc, _pl_key(seedmix, i, np.arange(k_loc), 1))
        uni = _strata(0, n, k_uni, _pl_key(seedmix, i, np.arange(k_uni), 2))
        c = np.union1d(loc, uni)
        cols.append(c)
        ptr.append(ptr[-1] + len(c))
    col = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    row_ptr = np.asarray(ptr, dtype=np.int64)
    rows = np.repeat(np.arange(lo, hi, dtype=np.int64), np.diff(row_ptr))
    vals = keyed_uniform(rows, col, seed).astype(dtype_for(precision))
    return CsrMatrix(hi - lo, n, row_ptr, col.astype(np.int32), vals)


# ---------------------------------------------------------------- config 4
FEM_NODES = 262_144
FEM_WINDOW = 2048
FEM_NBR = 26
SQRT3 = 1.7320508075688772


def fem_neighbours(q: int, nodes: int = FEM_NODES, seed: int = MATRIX_SEED) -> np.ndarray:
    """The 26 nodes coupled to node q: stratified over q +- 2048, q excluded, ascending."""
    lo_w = max(0, q - FEM_WINDOW)
    w = min(nodes - 1, q + FEM_WINDOW) - lo_w
    p = _strata(lo_w, w, FEM_NBR, _pl_key(seed_mix(seed) ^ PL_SALT, q, np.arange(FEM_NBR), 3))
    return np.where(p >= q, p + 1, p)


def fem_rows(lo: int, hi: int, nodes: int = FEM_NODES, precision: str = "f64",
             seed: int = MATRIX_SEED) -> CsrMatrix:
    """Rows [lo, hi) of the config-4 FEM-like matrix (twin of csrc/aux.cu fem_*).

    Row 3q+d holds the dense 3x3 blocks of node q and its 26 neighbours
    (81 entries); values sqrt(3) * (u1 + u2 + u3 + u4 - 2), u_k chained
    splitmix64 uniforms keyed by (row, col).
    """
    cols = []
    for i in range(lo, hi):
        q = i // 3
        nodes_q = np.union1d(fem_neighbours(q, nodes, seed), [q])
        cols.append((3 * nodes_q[:, None] + np.arange(3)[None, :]).ravel())
    col = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    row_ptr = np.arange(hi - lo + 1, dtype=np.int64) * 3 * (FEM_NBR + 1)
    rows = np.repeat(np.arange(lo, hi, dtype=np.int64), 3 * (FEM_NBR + 1))
    key = (rows.astype(np.uint64) << np.uint64(32)) ^ col.astype(np.uint64) ^ seed_mix(seed)
    h = mix64(key)
    acc = np.zeros(len(col), dtype=np.float64)
    with np.errstate(over="ignore"):
        for _ in range(4):
            acc += (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            h = mix64(h + GOLDEN)
    vals = ((acc - 2.0) * SQRT3).astype(dtype_for(precision))
    return CsrMatrix(hi - lo, 3 * nodes, row_ptr, col.astype(np.int32), vals)


# Config descriptors used by bench.py and the tests.  ``formats`` are (r, vs).
CONFIGS = {
    1: dict(name="random8192_16perrow_f64", precision="f64", formats=[(1, 8)]),
    2: dict(name="stencil27_128cubed_f64", precision="f64", n=128,
            formats=[(1, 8), (2, 8), (4, 8), (8, 8)]),
    3: dict(name="powerlaw_4M_f32", precision="f32", gen="powerlaw", rows=PL_N, cols=PL_N,
            formats=[(1, 16), (2, 16), (4, 16)]),
    4: dict(name="fem_786K_f64", precision="f64", gen="fem", rows=3 * FEM_NODES,
            cols=3 * FEM_NODES, formats=[(4, 8), (8, 8)]),
    5: dict(name="stencil27_400cubed", precision="f64", n=400,
            formats=[(1, 8), (2, 8), (4, 8), (8, 8)]),
    # the fp32 halves of configs 2 and 5 (BASELINE config 5 names both precisions)
    6: dict(name="stencil27_128cubed_f32", precision="f32", n=128,
            formats=[(1, 16), (2, 16), (4, 16), (8, 16)]),
    7: dict(name="stencil27_400cubed_f32", precision="f32", n=400,
            formats=[(1, 16), (2, 16), (4, 16), (8, 16)]),
}


# ---------------------------------------------------------------- device twins
def _gen_args(cfg):
    gen = cfg.get("gen", "stencil")
    nz = cfg.get("nz", cfg.get("n"))  # stencil box depth (weak scaling: n * ranks)
    return gen, nz


def device_rowptr(cfg, lo: int, hi: int):
    """Row pointers (int64[hi-lo+1], device) of rows [lo, hi) of a config's
    matrix, from the device generator alone -- no columns or values (the
    partition needs only these)."""
    import torch

    from . import _native as nat
    gen, nz = _gen_args(cfg)
    rp = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
    if gen == "stencil":
        nat.check(nat.lib.spc5_gen_stencil27_box_rowptr(cfg["n"], nz, lo, hi, rp.data_ptr(), 0))
    elif gen == "powerlaw":
        table = torch.from_numpy(powerlaw_len_table()).to("cuda")
        nat.check(nat.lib.spc5_gen_powerlaw_rowptr(PL_N, lo, hi, MATRIX_SEED, table.data_ptr(),
                                                   PL_TABLE_BITS, rp.data_ptr(), 0))
    else:
        nat.check(nat.lib.spc5_gen_fem_rowptr(cfg["rows"] // 3, lo, hi, rp.data_ptr(), 0))
    return rp


def device_rows(cfg, lo: int, hi: int, rp=None):
    """Device CSR (row_ptr, col_idx, values) of rows [lo, hi) of a config's
    matrix (stencil / power-law / FEM): the twins of stencil27_rows /
    powerlaw_rows / fem_rows, bit for bit."""
    import torch

    from . import _native as nat
    gen, nz = _gen_args(cfg)
    prec = cfg["precision"]
    tdt = torch.float64 if prec == "f64" else torch.float32
    pc = nat.F64 if prec == "f64" else nat.F32
    if rp is None:
        rp = device_rowptr(cfg, lo, hi)
    nnz = int(rp[-1])
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    va = torch.empty(max(nnz, 1), dtype=tdt, device="cuda")
    if gen == "stencil":
        nat.check(nat.lib.spc5_gen_stencil27_box_fill(cfg["n"], nz, lo, hi, pc, MATRIX_SEED,
                                                      27.0, rp.data_ptr(), ci.data_ptr(),
                                                      va.data_ptr(), 0))
    elif gen == "powerlaw":
        table = torch.from_numpy(powerlaw_len_table()).to("cuda")
        nat.check(nat.lib.spc5_gen_powerlaw_fill(PL_N, lo, hi, pc, MATRIX_SEED,
                                                 table.data_ptr(), PL_TABLE_BITS, rp.data_ptr(),
                                                 ci.data_ptr(), va.data_ptr(), 0))
    else:
        nat.check(nat.lib.spc5_gen_fem_fill(cfg["rows"] // 3, lo, hi, pc, MATRIX_SEED,
                                            rp.data_ptr(), ci.data_ptr(), va.data_ptr(), 0))
    torch.cuda.synchronize()
    return rp, ci[:nnz], va[:nnz]


def host_rows(cfg, lo: int, hi: int) -> CsrMatrix:
    """Host CSR of rows [lo, hi) of a config's matrix (numpy generators)."""
    gen, nz = _gen_args(cfg)
    if gen == "stencil":
        return stencil27_rows(cfg["n"], lo, hi, cfg["precision"], nz=nz)
    if gen == "powerlaw":
        return powerlaw_rows(lo, hi, precision=cfg["precision"])
    return fem_rows(lo, hi, precision=cfg["precision"])


def config_shape(cfg) -> tuple[int, int]:
    """(num_rows, num_cols) of a config's matrix."""
    if "n" in cfg:
        n = cfg["n"] ** 2 * cfg.get("nz", cfg["n"])
        return n, n
    if "rows" in cfg:
        return cfg["rows"], cfg["cols"]
    return 8192, 8192
