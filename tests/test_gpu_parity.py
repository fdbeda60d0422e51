"""GPU parity: the CUDA path (through the C ABI) against the pinned oracle.

Bar (BASELINE.json north_star): conversion bit-exact with the reference;
y within |dy_i| <= tol * sum_j |a_ij x_j| of the reference scalar path with
tol = 1e-12 (f64) / 1e-5 (f32); the reference's own VERIFY_FACTOR budget
against the exact oracle (kernels.py:284-312) must pass too.
"""

import numpy as np
import pytest

from golden_io import (Csr, case_x, config1, digest, expected_small, fmt_keys, small_case,
                       small_case_names, stencil)
from oracle import oracle

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


@pytest.fixture(scope="module")
def spc5(cuda_device):
    import paper_2307_14774_b200 as pkg
    return pkg


def assert_close(m, y, y_ref, x, label=""):
    _, abs_ref = oracle.csr_reference(m, x)
    err = oracle.relative_error(y[:m.num_rows], y_ref[:m.num_rows], abs_ref)
    tol = TOL["f32" if m.values.dtype == np.float32 else "f64"]
    assert err.size == 0 or float(err.max()) <= tol, f"{label}: max rel err {err.max():.3g}"
    scaled = oracle.scaled_error(m, y, x)
    assert scaled.size == 0 or float(scaled.max()) <= oracle.VERIFY_FACTOR, label


# ---------------------------------------------------------------- conversion
@pytest.mark.parametrize("name", small_case_names())
def test_convert_small_bit_exact(spc5, name):
    m = small_case(name)
    rec = expected_small()["cases"][name]
    for r, vs, f in fmt_keys(rec):
        s = spc5.csr_to_spc5(m, r, vs)
        assert s.num_blocks == f["num_blocks"], (name, r, vs)
        assert digest(s.block_rowptr) == f["rowptr"], (name, r, vs)
        assert digest(s.block_colidx) == f["colidx"], (name, r, vs)
        assert digest(s.block_masks) == f["masks"], (name, r, vs)
        assert digest(s.values) == f["values"], (name, r, vs)
        assert spc5.filling_stats(s).footprint_bytes == f["footprint_bytes"]


def test_hand_matrix_known_answers(spc5):
    m = small_case("hand")
    s = spc5.csr_to_spc5(m, 2, 4)
    assert s.block_rowptr.tolist() == [0, 2, 3]
    assert s.block_colidx.tolist() == [0, 6, 6]
    assert s.block_masks.tolist() == [0b1101, 0b0010, 0b0001, 0, 0, 0b0011]
    assert s.values.tolist() == [1, 2, 3, 5, 4, 6, 7]
    for r, vs in ((1, 4), (2, 4), (4, 8), (8, 16)):
        y = np.zeros(4)
        spc5.spmv_spc5_vector(spc5.csr_to_spc5(m, r, vs), np.ones(8), y, spc5.KernelConfig())
        assert y.tolist() == [10, 5, 0, 13]


def test_edge_blocks(spc5):
    m = small_case("edge")
    y = np.zeros(2)
    spc5.spmv_spc5_vector(spc5.csr_to_spc5(m, 2, 8), np.array([9.0, 9, 9, 1, 2]), y,
                          spc5.KernelConfig())
    assert y.tolist() == [5.0, 6.0]


def test_config1_bit_exact(spc5):
    from paper_2307_14774_b200.workloads import config1 as gen1, x_vector
    c1 = config1()
    m = gen1(c1["seed"])
    x = x_vector(8192, "f64", c1["x_seed"])
    for r, vs, f in fmt_keys(c1):
        s = spc5.csr_to_spc5(m, r, vs)
        assert (digest(s.block_rowptr), digest(s.block_colidx), digest(s.block_masks),
                digest(s.values)) == (f["rowptr"], f["colidx"], f["masks"], f["values"])
        part = spc5.partition_by_nnz(s, 8).ranges
        assert part == [tuple(t) for t in f["partition"]["8"]]
        y = np.zeros(8192)
        spc5.spmv_spc5_scalar(s, x, y)
        y_ref = np.zeros(8192)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
        assert digest(y_ref) == f["y_scalar"]
        assert_close(m, y, y_ref, x, f"config1 {r},{vs}")


def test_stencil_bit_exact(spc5):
    from paper_2307_14774_b200.workloads import stencil27, x_vector
    for key, rec in stencil()["cases"].items():
        m = stencil27(rec["n"], rec["precision"])
        x = x_vector(m.num_cols, rec["precision"])
        for r, vs, f in fmt_keys(rec):
            s = spc5.csr_to_spc5(m, r, vs)
            assert (digest(s.block_rowptr), digest(s.block_colidx), digest(s.block_masks),
                    digest(s.values)) == (f["rowptr"], f["colidx"], f["masks"], f["values"])
            y = np.zeros(m.num_rows, m.values.dtype)
            spc5.spmv_spc5_scalar(s, x, y)
            y_ref = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
            assert digest(y_ref) == f["y_scalar"]
            assert_close(m, y, y_ref, x, f"{key} {r},{vs}")


# ---------------------------------------------------------------- SpMV
@pytest.mark.parametrize("name", small_case_names())
def test_spmv_small_vs_oracle(spc5, name):
    m = small_case(name)
    x = case_x(name, m)
    rec = expected_small()["cases"][name]
    for r, vs, f in fmt_keys(rec):
        s = spc5.csr_to_spc5(m, r, vs)
        y = np.zeros(m.num_rows, m.values.dtype)
        spc5.spmv_spc5_scalar(s, x, y)
        y_ref = np.zeros(m.num_rows, m.values.dtype)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
        assert digest(y_ref) == f["y_scalar"]
        assert_close(m, y, y_ref, x, f"{name} {r},{vs}")
        for w, ranges in f["partition"].items():
            assert spc5.partition_by_nnz(s, int(w)).ranges == [tuple(t) for t in ranges]


@pytest.mark.parametrize("name", ["longrows", "longrows_f32", "tall", "rand05", "rand17"])
def test_spmv_repeatable_bitwise(spc5, name):
    """Every format: repeated products are bitwise identical (catches races on
    y rows and carry slots between lanes, warps and chunks)."""
    m = small_case(name)
    x = case_x(name, m)
    for r, vs, _ in fmt_keys(expected_small()["cases"][name]):
        s = spc5.csr_to_spc5(m, r, vs)
        y0 = spc5.spmv(s, x)
        for _ in range(6):
            assert spc5.spmv(s, x).tobytes() == y0.tobytes(), (name, r, vs)


def test_lane_per_panel_split_chunks(spc5, monkeypatch):
    """Lane-per-panel mode on split pieces of long panels (carry slots from that
    mode), forced with the SPC5_LPR_SPLIT plan knob: same tolerance, repeatable."""
    monkeypatch.setenv("SPC5_LPR_SPLIT", "1")
    for name in ("longrows", "longrows_f32", "tall", "rand05"):
        m = small_case(name)
        x = case_x(name, m)
        for r, vs, _ in fmt_keys(expected_small()["cases"][name]):
            s = spc5.csr_to_spc5(m, r, vs)
            y = spc5.spmv(s, x)
            y_ref = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
            assert_close(m, y, y_ref, x, f"{name} {r},{vs} lpr-split")
            assert spc5.spmv(s, x).tobytes() == y.tobytes()


def test_identity_exact_and_cancellation(spc5):
    m = small_case("identity32")
    x = np.random.default_rng(3).uniform(-1, 1, 32)
    y = spc5.spmv(spc5.csr_to_spc5(m, 1, 8), x)
    assert y.tobytes() == x.tobytes()
    m = small_case("cancel")
    s = spc5.csr_to_spc5(m, 1, 4)
    y = np.zeros(1)
    spc5.spmv_spc5_scalar(s, np.ones(3), y)
    assert abs(y[0] - 1.0) <= 8 * 3 * np.finfo(float).eps * 2e16
    rep = spc5.verify_against_oracle(m, 1, 4, spc5.KernelConfig(), trials=3, seed=3)
    assert rep.passed, str(rep)


def test_verify_against_oracle_configs(spc5):
    for name in ("dense16", "tall", "longrows", "rand03", "longrows_f32", "dense16_f32"):
        m = small_case(name)
        prec = "f32" if m.values.dtype == np.float32 else "f64"
        for r, vs in ((1, 8), (2, 16), (4, 4), (8, 8)):
            for strat in ("scalar", "compact", "expand"):
                cfg = spc5.KernelConfig(strategy=strat, precision=prec)
                rep = spc5.verify_against_oracle(m, r, vs, cfg, trials=2, seed=11)
                assert rep.passed, (name, r, vs, str(rep))


def test_accumulate_and_overwrite(spc5):
    m = small_case("tall")
    x = case_x("tall", m)
    s = spc5.csr_to_spc5(m, 4, 8)
    once = np.zeros(m.num_rows)
    spc5.spmv_spc5_vector(s, x, once, spc5.KernelConfig())
    twice = np.full(m.num_rows, 0.0)
    spc5.spmv_spc5_vector(s, x, twice, spc5.KernelConfig())
    spc5.spmv_spc5_vector(s, x, twice, spc5.KernelConfig())
    assert np.allclose(twice, 2 * once, rtol=1e-14, atol=0)
    y = np.full(m.num_rows, np.nan)
    spc5.spmv(s, x, y)
    assert y.tobytes() == once.tobytes()


def test_empty_panels_overwrite(spc5):
    # rows with no entries (and >32 consecutive empty panels) must come back 0 in y = A.x
    n = 4000
    keep = np.arange(0, n, 97)
    counts = np.zeros(n, np.int64)
    counts[keep] = 3
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rp[1:])
    cols = np.concatenate([np.array([i % 50, 100 + i % 7, 300 + i % 11]) for i in keep])
    m = Csr(n, 400, rp, cols.astype(np.int32),
            np.random.default_rng(1).uniform(-1, 1, len(cols)))
    x = np.random.default_rng(2).uniform(-1, 1, 400)
    for r, vs in ((1, 8), (2, 4), (8, 16)):
        s = spc5.csr_to_spc5(m, r, vs)
        y = np.full(n, 7.0)
        spc5.spmv(s, x, y)
        y_ref = np.zeros(n)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
        assert_close(m, y, y_ref, x, f"sparse-rows {r},{vs}")


def giant_row_matrix(precision="f64"):
    # row 3 spans ~9000 blocks at vs=4 (> kSplit = 2048): exercises split chunks + fixup
    rng = np.random.default_rng(5)
    n, ncols = 40, 60000
    rows = []
    for i in range(n):
        if i == 3:
            c = np.arange(0, ncols, 6)
        elif i == 17:
            c = np.arange(5, ncols, 13)
        else:
            c = np.sort(rng.choice(ncols, size=int(rng.integers(0, 40)), replace=False))
        rows.append(c)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum([len(c) for c in rows], out=rp[1:])
    cols = np.concatenate(rows).astype(np.int32)
    dt = np.float64 if precision == "f64" else np.float32
    return Csr(n, ncols, rp, cols, rng.uniform(-1, 1, len(cols)).astype(dt))


def test_giant_panels_split_and_fixup(spc5):
    for prec in ("f64", "f32"):
        m = giant_row_matrix(prec)
        x = np.random.default_rng(9).uniform(-1, 1, m.num_cols).astype(m.values.dtype)
        for r, vs in ((1, 4), (2, 8), (4, 16)):
            s = spc5.csr_to_spc5(m, r, vs)
            ref = oracle.csr_to_spc5(m, r, vs)
            assert np.array_equal(s.block_colidx, ref.block_colidx)
            assert np.array_equal(s.block_masks, ref.block_masks)
            assert s.values.tobytes() == ref.values.tobytes()
            y = np.zeros(m.num_rows, m.values.dtype)
            spc5.spmv_spc5_scalar(s, x, y)
            y_ref = np.zeros(m.num_rows, m.values.dtype)
            oracle.spmv_spc5_scalar(ref, x, y_ref)
            assert_close(m, y, y_ref, x, f"giant {prec} {r},{vs}")
            for w in (2, 3, 5, 8):
                yp = np.zeros(m.num_rows, m.values.dtype)
                spc5.spmv_parallel(s, x, yp, spc5.KernelConfig(precision=prec), w)
                assert yp.tobytes() == y.tobytes(), (prec, r, vs, w)


def _parallel_cases():
    from paper_2307_14774_b200.workloads import fem_rows, powerlaw_rows
    for name in ("tall", "longrows", "rand07", "dense16", "lastpanel"):
        m = small_case(name)
        yield name, m, case_x(name, m)
    # irregular rows (balanced-lane-range chunks) and dense 3x3 blocks
    for name, m in (("powerlaw", powerlaw_rows(1000, 1400, precision="f64")),
                    ("fem", fem_rows(3000, 3300))):
        yield name, m, np.random.default_rng(7).uniform(-1, 1, m.num_cols)


@pytest.mark.parametrize("lpr_split", [False, True])
def test_parallel_bitwise_equal(spc5, lpr_split, monkeypatch):
    if lpr_split:
        monkeypatch.setenv("SPC5_LPR_SPLIT", "1")
    for name, m, x in _parallel_cases():
        prec = "f32" if m.values.dtype == np.float32 else "f64"
        for r in (1, 2, 4, 8):
            s = spc5.csr_to_spc5(m, r, 8)
            expect = np.zeros(m.num_rows, m.values.dtype)
            spc5.spmv_spc5_vector(s, x, expect, spc5.KernelConfig(precision=prec))
            for w in (1, 2, 3, 4, 7, 8):
                y = np.zeros(m.num_rows, m.values.dtype)
                res = spc5.spmv_parallel(s, x, y, spc5.KernelConfig(precision=prec), w)
                assert y.tobytes() == expect.tobytes(), (name, r, w)
                assert res.flops == 2 * m.nnz and res.y is y


def test_row_panel_shards_bitwise(spc5):
    """Each rank converts only its rows (block_base = global block offset): the
    shard's blocks equal the full matrix's slice bit for bit, y to rounding."""
    from paper_2307_14774_b200.workloads import stencil27_rows, x_vector
    n = 20
    full = stencil27_rows(n, 0, n ** 3)
    x = x_vector(full.num_cols)
    for r in (1, 2, 4, 8):
        s = spc5.csr_to_spc5(full, r, 8)
        y_full = spc5.spmv(s, x)
        for P in (2, 3, 4, 8):
            for lo, hi in spc5.partition_by_nnz(s, P).ranges:
                if hi == lo:
                    continue
                rows = stencil27_rows(n, lo * r, min(hi * r, n ** 3))
                base = int(s.block_rowptr[lo])
                sh = spc5.csr_to_spc5(rows, r, 8, block_base=base)
                assert np.array_equal(sh.block_colidx,
                                      s.block_colidx[base:int(s.block_rowptr[hi])])
                y = spc5.spmv(sh, x)
                # same value up to the association of the per-panel sums: chunks at a
                # shard edge may run lane-per-panel where the full run went lane-per-block
                ref = y_full[lo * r:min(hi * r, n ** 3)]
                _, absr = oracle.csr_reference(rows, x)
                assert float(oracle.relative_error(y, ref, absr).max()) <= 1e-15, (r, P, lo)


# ---------------------------------------------------------------- errors
def test_corrupted_mask_raises_and_verify_reports(spc5):
    m = small_case("tall")
    s = spc5.csr_to_spc5(m, 1, 8)
    masks = s.block_masks
    i = int(np.flatnonzero(masks != 0xFF)[0])
    mask = int(masks[i])
    unset = next(k for k in range(8) if not (mask >> k) & 1)
    masks[i] = mask | (1 << unset)  # popcount now exceeds nnz (in-place, like the reference test)
    with pytest.raises((RuntimeError, ValueError, IndexError)):
        spc5.spmv_spc5_vector(s, np.ones(m.num_cols), np.zeros(m.num_rows), spc5.KernelConfig())
    # moved bit: popcount preserved, result wrong -> failed verification, not a crash
    m = spc5.make_random(20, 40, 5, 0.6, seed=4)
    s = spc5.csr_to_spc5(m, 1, 8)
    pc = spc5.mask_popcounts(s.block_masks)
    slot = int(np.flatnonzero((pc >= 1) & (pc < 8))[0])
    mask = int(s.block_masks[slot])
    sb = next(k for k in range(8) if (mask >> k) & 1)
    ub = next(k for k in range(8) if not (mask >> k) & 1)
    s.block_masks[slot] = mask ^ (1 << sb) ^ (1 << ub)
    rep = spc5.verify_against_oracle(m, 1, 8, spc5.KernelConfig(), trials=1, seed=5, spc5=s)
    assert not rep.passed and rep.worst_row >= 0


def test_argument_errors(spc5):
    m = small_case("hand")
    s = spc5.csr_to_spc5(m, 1, 4)
    with pytest.raises(ValueError):
        spc5.csr_to_spc5(m, 3, 4)
    with pytest.raises(ValueError, match="f32"):
        spc5.spmv_spc5_vector(s, np.ones(8), np.zeros(4), spc5.KernelConfig(precision="f32"))
    with pytest.raises(ValueError):
        spc5.spmv_spc5_vector(s, np.ones(8), np.zeros(4), spc5.KernelConfig(strategy="scalar"))
    with pytest.raises(ValueError):
        spc5.spmv_spc5_scalar(s, np.ones(4), np.zeros(4))
    bad = Csr(1, 8, np.array([0, 2], np.int64), np.array([5, 3], np.int32), np.ones(2))
    with pytest.raises(ValueError):
        spc5.csr_to_spc5(bad, 1, 8)


# ---------------------------------------------------------------- aux
def test_to_csr_validate_roundtrip(spc5):
    for name in ("hand", "rand11", "longrows_f32", "empty", "lastpanel"):
        m = small_case(name)
        for r, vs in ((1, 4), (4, 8), (8, 16)):
            s = spc5.csr_to_spc5(m, r, vs)
            spc5.validate_spc5(s)
            back = spc5.spc5_to_csr(s)
            assert np.array_equal(back.row_ptr, m.row_ptr)
            assert np.array_equal(back.col_idx, m.col_idx)
            assert back.values.tobytes() == m.values.tobytes()
    s = spc5.csr_to_spc5(small_case("tall"), 2, 8)
    s.block_colidx[5] = s.block_colidx[4]
    with pytest.raises(ValueError):
        spc5.validate_spc5(s)


def test_device_generator_matches_host(spc5):
    import torch
    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.workloads import stencil27_rows
    n, lo, hi = 20, 1234, 5678
    for prec, tdt in (("f64", torch.float64), ("f32", torch.float32)):
        host = stencil27_rows(n, lo, hi, prec)
        rp = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_rowptr(n, lo, hi, rp.data_ptr(), 0))
        nnz = int(rp[-1])
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        va = torch.empty(nnz, dtype=tdt, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_fill(n, lo, hi, 0 if prec == "f32" else 1, 0, 27.0,
                                                  rp.data_ptr(), ci.data_ptr(), va.data_ptr(), 0))
        torch.cuda.synchronize()
        assert np.array_equal(rp.cpu().numpy(), host.row_ptr)
        assert np.array_equal(ci.cpu().numpy(), host.col_idx)
        assert va.cpu().numpy().tobytes() == host.values.tobytes()


def test_csr_reference_gpu_matches_oracle(spc5):
    for name in ("cancel", "rand00", "longrows", "longrows_f32", "dense16_f32"):
        m = small_case(name)
        x = case_x(name, m)
        y, a = spc5.csr_reference(m, x)
        y2, a2 = oracle.csr_reference(m, x)
        assert np.array_equal(y, y2), name
        assert np.allclose(a, a2, rtol=1e-15, atol=0), name


def test_save_load_device_roundtrip(spc5, tmp_path):
    m = small_case("rand05")
    for r, vs in ((1, 4), (2, 8), (4, 16)):
        s = spc5.csr_to_spc5(m, r, vs)
        spc5.save_spc5(s, tmp_path / "c.spc5")
        t = spc5.load_spc5(tmp_path / "c.spc5")
        x = case_x("rand05", m)
        assert spc5.spmv(t, x).tobytes() == spc5.spmv(s, x).tobytes()


# ---------------------------------------------------------------- full size
@pytest.mark.slow
def test_config2_full_size(spc5):
    """BASELINE config 2 (stencil 128^3, f64, 55.7M nnz): every format bit-exact
    against the oracle conversion, y within tolerance of the oracle scalar path."""
    import torch
    from paper_2307_14774_b200.workloads import stencil27, stencil27_nnz, x_vector
    n = 128
    m = stencil27(n)
    assert m.nnz == stencil27_nnz(n)
    x = x_vector(m.num_cols)
    _, abs_ref = oracle.csr_reference(m, x)
    for r in (1, 2, 4, 8):
        ref = oracle.csr_to_spc5(m, r, 8)
        s = spc5.csr_to_spc5(m, r, 8)
        expect_nb = (n // r) * (3 * n - 2) ** 2 * (1 if r + 2 <= 8 else 2)
        assert s.num_blocks == ref.num_blocks == expect_nb
        for f in ("block_rowptr", "block_colidx", "block_masks", "values"):
            assert np.array_equal(getattr(s, f), getattr(ref, f)), (r, f)
        y = spc5.spmv(s, x)
        y_ref = np.zeros(m.num_rows)
        oracle.spmv_spc5_scalar(ref, x, y_ref, threads=oracle.threads())
        err = oracle.relative_error(y, y_ref, abs_ref)
        assert float(err.max()) <= 1e-12, (r, float(err.max()))
        del s
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- configs 3 and 4
def _device_rows(gen, lo, hi, prec):
    """Rows [lo, hi) of config 3 ('powerlaw') or 4 ('fem') from the device generator."""
    import torch
    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.workloads import FEM_NODES, PL_N, PL_TABLE_BITS, powerlaw_len_table
    tdt = torch.float64 if prec == "f64" else torch.float32
    pc = 1 if prec == "f64" else 0
    rp = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
    table = torch.from_numpy(powerlaw_len_table()).to("cuda")
    if gen == "powerlaw":
        nat.check(nat.lib.spc5_gen_powerlaw_rowptr(PL_N, lo, hi, 0, table.data_ptr(),
                                                   PL_TABLE_BITS, rp.data_ptr(), 0))
    else:
        nat.check(nat.lib.spc5_gen_fem_rowptr(FEM_NODES, lo, hi, rp.data_ptr(), 0))
    nnz = int(rp[-1])
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    va = torch.empty(max(nnz, 1), dtype=tdt, device="cuda")
    if gen == "powerlaw":
        nat.check(nat.lib.spc5_gen_powerlaw_fill(PL_N, lo, hi, pc, 0, table.data_ptr(),
                                                 PL_TABLE_BITS, rp.data_ptr(), ci.data_ptr(),
                                                 va.data_ptr(), 0))
    else:
        nat.check(nat.lib.spc5_gen_fem_fill(FEM_NODES, lo, hi, pc, 0, rp.data_ptr(),
                                            ci.data_ptr(), va.data_ptr(), 0))
    torch.cuda.synchronize()
    return rp, ci[:nnz], va[:nnz]


@pytest.mark.parametrize("gen,prec,lo,hi", [
    ("powerlaw", "f32", 0, 3000), ("powerlaw", "f32", 2_000_000, 2_001_500),
    ("powerlaw", "f32", 4_194_304 - 1500, 4_194_304), ("powerlaw", "f64", 777, 1777),
    ("fem", "f64", 0, 1500), ("fem", "f64", 400_000, 401_000),
    ("fem", "f64", 786_432 - 1200, 786_432), ("fem", "f32", 12_345, 13_345)])
def test_config34_device_generator_matches_host(spc5, gen, prec, lo, hi):
    from paper_2307_14774_b200.workloads import fem_rows, powerlaw_rows
    host = (powerlaw_rows if gen == "powerlaw" else fem_rows)(lo, hi, precision=prec)
    rp, ci, va = _device_rows(gen, lo, hi, prec)
    assert np.array_equal(rp.cpu().numpy(), host.row_ptr)
    assert np.array_equal(ci.cpu().numpy(), host.col_idx)
    assert va.cpu().numpy().tobytes() == host.values.tobytes()


def _full_config_parity(spc5, cfg_id):
    """A BASELINE config at full size: device-generated CSR, every format's
    conversion bit-exact against the oracle, y within tolerance of the oracle
    scalar path and inside the VERIFY_FACTOR budget of the exact sums."""
    import torch
    from paper_2307_14774_b200.mmio import CsrMatrix
    from paper_2307_14774_b200.workloads import CONFIGS, x_vector
    cfg = CONFIGS[cfg_id]
    prec = cfg["precision"]
    rp, ci, va = _device_rows(cfg["gen"], 0, cfg["rows"], prec)
    m = CsrMatrix(cfg["rows"], cfg["cols"], rp.cpu().numpy(), ci.cpu().numpy(), va.cpu().numpy())
    del rp, ci, va
    x = x_vector(m.num_cols, prec)
    _, abs_ref = oracle.csr_reference(m, x)
    for r, vs in cfg["formats"]:
        ref = oracle.csr_to_spc5(m, r, vs)
        s = spc5.csr_to_spc5(m, r, vs)
        for f in ("block_rowptr", "block_colidx", "block_masks", "values"):
            assert np.array_equal(getattr(s, f), getattr(ref, f)), (r, vs, f)
        y = spc5.spmv(s, x)
        y_ref = np.zeros(m.num_rows, dtype=x.dtype)
        oracle.spmv_spc5_scalar(ref, x, y_ref, threads=oracle.threads())
        err = oracle.relative_error(y, y_ref, abs_ref)
        assert float(err.max()) <= TOL[prec], (r, vs, float(err.max()))
        scaled = oracle.scaled_error(m, y, x)
        assert float(scaled.max()) <= oracle.VERIFY_FACTOR, (r, vs)
        del s
        torch.cuda.empty_cache()


@pytest.mark.slow
def test_config3_full_size(spc5):
    """BASELINE config 3: power-law 4,194,304^2, f32, beta(1|2|4, 16)."""
    _full_config_parity(spc5, 3)


@pytest.mark.slow
def test_config4_full_size(spc5):
    """BASELINE config 4: FEM-like 786,432^2 with dense 3x3 blocks, f64, beta(4|8, 8)."""
    _full_config_parity(spc5, 4)


# ---------------------------------------------------------------- fused exchange (iterated products)
def test_spmv_mirrored_peer_stores(spc5):
    """spc5_spmv_mirrored: y = scale*A.x and every row mirrored into each peer
    buffer at row0 + row (here two plain device buffers stand in for peers)."""
    import ctypes
    import torch
    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.blocks import torch_stream
    for name in ("longrows", "tall", "rand05"):
        m = small_case(name)
        x = torch.from_numpy(case_x(name, m)).cuda()
        for r, vs in ((1, 8), (2, 4), (4, 16), (8, 8)):
            s = spc5.csr_to_spc5(m, r, vs)
            y = spc5.spmv(s, x)
            row0 = 37
            peers = [torch.full((m.num_rows + 100,), -7.0, dtype=x.dtype, device="cuda")
                     for _ in range(2)]
            arr = (ctypes.c_void_p * 2)(*[p.data_ptr() for p in peers])
            ym = torch.empty_like(y)
            nat.check(nat.lib.spc5_spmv_mirrored(s.handle().ptr, x.data_ptr(), ym.data_ptr(),
                                                 0.25, arr, 2, row0, torch_stream()))
            torch.cuda.synchronize()
            assert torch.equal(ym, y * 0.25), (name, r, vs)
            for p in peers:
                assert torch.equal(p[row0:row0 + m.num_rows], ym), (name, r, vs)
                assert bool((p[:row0] == -7.0).all()) and bool((p[row0 + m.num_rows:] == -7.0).all())


def test_fused_iteration_single_rank(spc5):
    """iterate_products_fused on a one-rank NCCL group (symmetric memory): the
    same x as the all-gather form, bit for bit."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2307_14774_b200.distributed import (iterate_products, iterate_products_fused,
                                                   shard_layout)
    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.blocks import torch_stream
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        from paper_2307_14774_b200.workloads import stencil27
        m_sq = stencil27(12)  # square: x <- A.x iterates
        x0 = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m_sq.num_cols)).cuda()
        for r, vs in ((1, 8), (4, 8)):
            s = spc5.csr_to_spc5(m_sq, r, vs)
            h = s.handle()
            layout = shard_layout(m_sq.row_ptr, r, 1)

            def local(xf, yout, h=h):
                nat.check(nat.lib.spc5_spmv(h.ptr, xf.data_ptr(), yout.data_ptr(), 0,
                                            torch_stream()))

            xa = iterate_products(x0, 5, layout, 0, 1, local, 1.0 / 64.0)
            xb = iterate_products_fused(x0, 5, layout, 0, 1, h, 1.0 / 64.0)
            torch.cuda.synchronize()
            assert torch.equal(xa, xb), (r, vs)
    finally:
        dist.destroy_process_group()


# ------------------------------------------ lane-per-panel-row step variants
def _banded(n, offsets, dtype, seed):
    """Rows with one fixed column pattern i + offsets (clipped): uniform panels,
    so every chunk runs in lane-per-panel-row mode."""
    rng = np.random.default_rng(seed)
    rows = [np.array([i + o for o in offsets if 0 <= i + o < n], np.int32) for i in range(n)]
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows)
    va = rng.uniform(-1, 1, len(ci)).astype(dtype)
    return Csr(n, n, rp, ci, va)


@pytest.mark.parametrize("pattern", [
    (-1, 0, 1),                      # stencil-like groups: pair slots 3+0 / 2+1 / 1+2
    (-40, -17, 0, 9, 33),            # one bit per block: pair slots of 1-2
    tuple(range(-7, 8)),             # dense rows: slot counts > 4 (batched dispatch)
    (0,),                            # one block per panel row: G-way lane splits
    (-300, -3, -2, -1, 0, 1, 2, 5, 6, 7, 250),  # mixed: 1-5 bits per block
])
def test_lane_per_panel_row_steps(spc5, pattern):
    """The v2 lane-per-panel-row steps (own-row masks, packed counts scanned
    over the row lanes, pair slots for r = 8, 16-bit fields for vs = 16)
    against the oracle for every (r, vs) in both precisions; repeatable."""
    for dtype in (np.float64, np.float32):
        m = _banded(6000, pattern, dtype, seed=len(pattern))
        x = np.random.default_rng(7).uniform(-1, 1, m.num_cols).astype(dtype)
        for r in (1, 2, 4, 8):
            for vs in (4, 8, 16):
                s = spc5.csr_to_spc5(m, r, vs)
                y = spc5.spmv(s, x)
                y_ref = np.zeros(m.num_rows, dtype)
                oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, vs), x, y_ref)
                assert_close(m, y, y_ref, x, f"{pattern} {np.dtype(dtype).name} {r},{vs}")
                assert spc5.spmv(s, x).tobytes() == y.tobytes()


def test_stencil_box_generator_matches_host(spc5):
    """The weak-scaling box (n x n x nz, bench.py --gpus N): device rows ==
    host twin rows, including slab edges whose columns reach the next slab."""
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.workloads import stencil27_rows
    n, nz = 10, 30
    for prec, (lo, hi) in (("f64", (0, 300)), ("f32", (900, 1300)), ("f64", (2650, 3000))):
        host = stencil27_rows(n, lo, hi, prec, nz=nz)
        rp = torch.empty(hi - lo + 1, dtype=torch.int64, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_box_rowptr(n, nz, lo, hi, rp.data_ptr(), 0))
        nnz = int(rp[-1])
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        va = torch.empty(nnz, dtype=torch.float64 if prec == "f64" else torch.float32,
                         device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_box_fill(n, nz, lo, hi, 1 if prec == "f64" else 0,
                                                      0, 27.0, rp.data_ptr(), ci.data_ptr(),
                                                      va.data_ptr(), 0))
        torch.cuda.synchronize()
        assert np.array_equal(rp.cpu().numpy(), host.row_ptr)
        assert np.array_equal(ci.cpu().numpy(), host.col_idx)
        assert va.cpu().numpy().tobytes() == host.values.tobytes()


def test_mostly_empty_rows(spc5):
    """One entry every 97 rows (empty panels everywhere, < 1 block per panel):
    the plan's chunk-boundary search stays bounded and y matches the oracle."""
    n = 200_000
    rows = np.arange(0, n, 97)
    rp = np.zeros(n + 1, np.int64)
    rp[rows + 1] = 1
    rp = np.cumsum(rp)
    ci = (rows * 7 % n).astype(np.int32)
    va = np.random.default_rng(0).uniform(-1, 1, len(ci))
    m = Csr(n, n, rp, ci, va)
    x = np.random.default_rng(1).uniform(-1, 1, n)
    for r in (1, 2, 4, 8):
        s = spc5.csr_to_spc5(m, r, 8)
        y = spc5.spmv(s, x)
        y_ref = np.zeros(n)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, r, 8), x, y_ref)
        assert y.tobytes() == y_ref.tobytes(), r  # one product per row: exact
