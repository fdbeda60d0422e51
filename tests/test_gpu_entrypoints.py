"""GPU entry points beside the product: validate_spc5's invariants with the
reference's messages (blocks.py:201-232), block_value_offsets and
footprint_comparison against the reference's outputs (tests/golden/), and the
timing harness with the reference's test_bench.py semantics (run_bench
validates before timing and refuses on failure, bench.py:153-184)."""

import numpy as np
import pytest

from golden_io import Csr, digest, expected_small, fmt_keys, small_case, small_case_names

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def spc5(cuda_device):
    import paper_2307_14774_b200 as pkg
    return pkg


def _hand_b24(spc5):
    """The reference's hand matrix in beta(2,4) as host arrays (tests/test_blocks.py:30-36):
    rowptr [0,2,3], colidx [0,6,6], masks [0b1101,0b0010,0b0001,0,0,0b0011], values 1..7."""
    return dict(num_rows=4, num_cols=8, r=2, vs=4,
                block_rowptr=np.array([0, 2, 3], np.int64),
                block_colidx=np.array([0, 6, 6], np.uint32),
                block_masks=np.array([0b1101, 0b0010, 0b0001, 0, 0, 0b0011], np.uint8),
                values=np.arange(1.0, 8.0))


# (how the arrays are corrupted, the message validate_spc5 raises, blocks.py:201-232)
CORRUPTIONS = [
    ("rowptr_len", "block_rowptr length does not match panel count"),
    ("rowptr_dec", "block_rowptr must be non-decreasing and start at 0"),
    ("rowptr_start", "block_rowptr must be non-decreasing and start at 0"),
    ("rowptr_cover", "block_rowptr does not cover all blocks"),
    ("mask_len", "mask array length must be num_blocks * r"),
    ("bits_beyond_vs", "mask has bits beyond vs"),
    ("popcount", "sum of mask popcounts differs from NNZ"),
    ("anchor", "block without an entry at its anchor column"),
    ("colidx_order", "panel 0: block columns not strictly increasing"),
    ("past_last_col", "set mask bit maps past the last column"),
]


def _corrupt(d, how):
    d = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d.items()}
    if how == "rowptr_len":
        d["block_rowptr"] = np.array([0, 2, 3, 3], np.int64)
    elif how == "rowptr_dec":
        d["block_rowptr"] = np.array([0, 3, 2], np.int64)
    elif how == "rowptr_start":
        d["block_rowptr"] = np.array([1, 2, 3], np.int64)
    elif how == "rowptr_cover":
        d["block_rowptr"] = np.array([0, 2, 2], np.int64)
    elif how == "mask_len":
        d["block_masks"] = d["block_masks"][:5]
    elif how == "bits_beyond_vs":
        d["block_masks"][1] |= 0b10000  # bit 4 of a vs = 4 mask
    elif how == "popcount":
        d["block_masks"][5] = 0b0111
    elif how == "anchor":  # same popcount, no entry at block 0's anchor column
        d["block_masks"][0] = 0b1110
    elif how == "colidx_order":
        d["block_colidx"] = np.array([6, 0, 6], np.uint32)
    elif how == "past_last_col":
        d["block_colidx"] = np.array([0, 6, 7], np.uint32)  # bit 1 of block 2 -> column 8
    return d


def test_validate_accepts_valid(spc5):
    d = _hand_b24(spc5)
    spc5.validate_spc5(spc5.Spc5Matrix(**d))
    m = small_case("hand")
    for r in (1, 2, 4, 8):
        for vs in (4, 8, 16):
            spc5.validate_spc5(spc5.csr_to_spc5(m, r, vs))


@pytest.mark.parametrize("how,msg", CORRUPTIONS)
def test_validate_invariants_reference_messages(spc5, how, msg):
    d = _corrupt(_hand_b24(spc5), how)
    with pytest.raises(ValueError) as e:
        spc5.validate_spc5(spc5.Spc5Matrix(**d))
    assert str(e.value) == msg


@pytest.mark.parametrize("name", small_case_names())
def test_block_value_offsets_golden(spc5, name):
    m = small_case(name)
    rec = expected_small()["cases"][name]
    for r, vs, f in fmt_keys(rec):
        s = spc5.csr_to_spc5(m, r, vs)
        off = spc5.block_value_offsets(s)
        assert digest(off.astype(np.int64)) == f["offsets"], (name, r, vs)
        assert int(off[-1]) == m.nnz
        if "offsets_list" in f:
            assert off.tolist() == f["offsets_list"]


@pytest.mark.parametrize("name", ["hand", "edge", "tall", "rand03", "rand11", "longrows"])
def test_footprint_comparison_golden(spc5, name):
    m = small_case(name)
    rec = expected_small()["cases"][name]
    for r, vs, f in fmt_keys(rec):
        assert list(spc5.footprint_comparison(m, r, vs)) == f["footprint_comparison"], (r, vs)


# ---- harness (the reference's tests/test_bench.py semantics) ------------------
def test_run_bench_identity(spc5):
    m = spc5.make_identity(256)
    rec = spc5.run_bench("identity:256", m, 1, 8, spc5.KernelConfig(), reps=5, warmup=1)
    assert rec.reps == 5 and rec.median_seconds > 0
    assert rec.gflops == 2 * 256 / rec.median_seconds / 1e9
    assert rec.nnz == 256


def test_run_bench_grid_cardinality(spc5):
    m = spc5.make_random(32, 32, 4, 0.5, seed=1)
    records = [spc5.run_bench("m", m, 1, 8, spc5.KernelConfig(strategy=st, reduction=rd),
                              reps=2, warmup=1)
               for st in ("expand", "compact") for rd in ("hsum", "multi")]
    assert len({(r.strategy, r.reduction) for r in records}) == 4


def test_run_bench_refuses_on_failed_validation(spc5, monkeypatch):
    import paper_2307_14774_b200.harness as harness

    def always_fail(*args, **kwargs):
        return spc5.VerifyReport(passed=False, max_scaled_error=99.0, threshold=8.0,
                                 worst_row=3, worst_trial=0, trials=1)

    monkeypatch.setattr(harness, "verify_against_oracle", always_fail)
    with pytest.raises(spc5.ValidationError, match="worst row 3"):
        spc5.run_bench("m", spc5.make_identity(8), 1, 8, spc5.KernelConfig(), reps=1, warmup=0)


def test_run_bench_refuses_corrupted_conversion(spc5, monkeypatch):
    """A conversion that drops a mask bit must not be timed (bench.py:163-167)."""
    import paper_2307_14774_b200.harness as harness
    real = harness.csr_to_spc5

    def broken(m, r, vs):
        s = real(m, r, vs)
        d = dict(num_rows=s.num_rows, num_cols=s.num_cols, r=s.r, vs=s.vs,
                 block_rowptr=s.block_rowptr.copy(), block_colidx=s.block_colidx.copy(),
                 block_masks=s.block_masks.copy(), values=s.values.copy())
        d["values"][0] += 1.0  # wrong matrix: the product disagrees with the oracle
        return spc5.Spc5Matrix(**d)

    monkeypatch.setattr(harness, "csr_to_spc5", broken)
    with pytest.raises(spc5.ValidationError):
        spc5.run_bench("m", spc5.make_random(64, 64, 4, 0.5, seed=3), 2, 8, spc5.KernelConfig(),
                       reps=1, warmup=0)


def test_run_kernel_parallel_dispatch(spc5):
    m = spc5.make_random(64, 64, 4, 0.5, seed=2)
    s = spc5.csr_to_spc5(m, 2, 8)
    x = np.ones(64)
    y1 = np.zeros(64)
    spc5.run_kernel(s, x, y1, spc5.KernelConfig(), workers=1)
    y4 = np.zeros(64)
    res = spc5.run_kernel(s, x, y4, spc5.KernelConfig(), workers=4)
    assert y1.tobytes() == y4.tobytes()
    assert res.elapsed >= 0 and res.flops == 2 * m.nnz


def test_time_device_spmv(spc5):
    from paper_2307_14774_b200.harness import time_device_spmv
    s = spc5.csr_to_spc5(spc5.make_random(4096, 4096, 16, 0.5, seed=4), 4, 8)
    t = time_device_spmv(s, reps=5, warmup=2)
    assert len(t) == 5 and all(v > 0 for v in t)


def test_csr_type_duck(spc5):
    """Any object with the CsrMatrix fields converts (reference mmio.py:84-100 names)."""
    m = small_case("hand")
    s = spc5.csr_to_spc5(Csr(m.num_rows, m.num_cols, m.row_ptr, m.col_idx, m.values), 2, 4)
    assert s.block_colidx.tolist() == [0, 6, 6]


def test_spmv_csr_matches_sequential_rows(spc5):
    """spmv_csr (kernels.py:106-118): y[i] += row_i . x, within the package
    tolerance of the oracle's sequential CSR sums, for both precisions."""
    from golden_io import case_x, small_case
    from oracle import oracle
    from test_gpu_parity import assert_close
    for name in ("hand", "rand05", "longrows", "longrows_f32", "tall"):
        m = small_case(name)
        x = case_x(name, m)
        y = np.zeros(m.num_rows, m.values.dtype)
        spc5.spmv_csr(m, x, y)
        y_ref = np.zeros(m.num_rows, m.values.dtype)
        oracle.spmv_spc5_scalar(oracle.csr_to_spc5(m, 1, 8), x, y_ref)  # r = 1: CSR row order
        assert_close(m, y, y_ref, x, f"spmv_csr {name}")
        again = y.copy()
        spc5.spmv_csr(m, x, again)  # accumulates
        assert np.allclose(again, 2 * y, rtol=1e-5 if m.values.dtype == np.float32 else 1e-12, atol=0)
    with pytest.raises(ValueError):
        spc5.spmv_csr(small_case("hand"), np.zeros(1), np.zeros(10))


def test_shard_cache_files_roundtrip(spc5, tmp_path):
    """Per-rank shard files: each rank's converted rows written
    with i8 row pointers and shard metadata, read back bit for bit, and the
    reloaded shards' products equal the live shards' bit for bit."""
    from paper_2307_14774_b200.workloads import stencil27_rows, x_vector
    from paper_2307_14774_b200.distributed import shard_layout
    n = 16
    full = stencil27_rows(n, 0, n ** 3)
    x = x_vector(full.num_cols)
    for prec_rows, r, vs in ((full, 2, 8), (full, 8, 8)):
        world = 3
        layout = shard_layout(full.row_ptr, r, world)
        whole = spc5.csr_to_spc5(full, r, vs)
        for rank in range(world):
            lo, hi = layout.rows(rank)
            base = int(whole.block_rowptr[layout.panel_ranges[rank][0]])
            sh = spc5.csr_to_spc5(stencil27_rows(n, lo, hi), r, vs, block_base=base)
            path = tmp_path / f"shard_{r}_{rank}.spc5"
            spc5.save_spc5_shard(sh, path, global_rows=n ** 3, row_lo=lo, rank=rank, world=world)
            back, meta = spc5.load_spc5_shard(path)
            assert meta == {"global_rows": n ** 3, "row_lo": lo, "rank": rank, "world": world}
            assert back.block_base == base and back.block_rowptr.dtype == np.int64
            for f in ("block_rowptr", "block_colidx", "block_masks", "values"):
                assert np.asarray(getattr(back, f)).tobytes() == np.asarray(getattr(sh, f)).tobytes(), f
            assert spc5.spmv(back, x).tobytes() == spc5.spmv(sh, x).tobytes()
    bad = tmp_path / "bad.spc5"
    bad.write_bytes(b"XXXX" + bytes(100))
    with pytest.raises(ValueError):
        spc5.load_spc5_shard(bad)


def test_cli_bench_device_cuda(spc5, tmp_path, capsys):
    """`python -m paper_2307_14774_b200 bench --device cuda` (cli.py:155-185 on the
    GPU): one line and one CSV v1 record per (format, config), readable by
    read_records, plus the roofline companion; a non-cuda device is refused."""
    from paper_2307_14774_b200.__main__ import main
    out = tmp_path / "bench.csv"
    rc = main(["bench", "--device", "cuda", "--matrix", "random:600,700,12,0.5,3", "--format",
               "b1,b4", "--strategy", "scalar,expand", "--reps", "3", "--warmup", "1", "--out",
               str(out)])
    assert rc == 0
    lines = [ln for ln in capsys.readouterr().out.splitlines() if ln.startswith("random:")]
    assert len(lines) == 4 and all("roofline=" in ln for ln in lines)
    recs = spc5.read_records(out)
    assert [(q.r, q.strategy) for q in recs] == [(1, "scalar"), (1, "expand"), (4, "scalar"), (4, "expand")]
    assert all(q.gflops > 0 and q.matrix == "random:600,700,12,0.5,3" for q in recs)
    assert (tmp_path / "bench.scatter.csv").exists() and (tmp_path / "bench.gpu.csv").exists()
    rc = main(["bench", "--device", "cuda", "--matrix", "config:2:0-4096", "--format", "b2",
               "--reps", "2", "--warmup", "1"])
    assert rc == 0
    assert main(["bench", "--device", "cpu", "--matrix", "dense:8"]) == 2


def test_large_pageable_host_buffers_are_staged(spc5):
    """x / y of >= 8 MB in ordinary (pageable) numpy arrays go through the
    library's pinned staging buffers with a host thread team
    (spc5_spmv_host): the result is bitwise the pinned-buffer call's, for
    y = A.x and for the accumulating entry point."""
    import torch
    n = 1_300_000
    rng = np.random.default_rng(21)
    off = np.array([-3, 0, 1, 7, 1000])
    ci = (np.arange(n)[:, None] + off[None, :])
    ci = np.sort(np.clip(ci, 0, n - 1), axis=1)
    keep = np.ones_like(ci, dtype=bool)
    keep[:, 1:] = ci[:, 1:] != ci[:, :-1]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(keep.sum(axis=1), out=rp[1:])
    m = Csr(n, n, rp, ci[keep].astype(np.int32), rng.uniform(-1, 1, int(keep.sum())))
    x = rng.uniform(-1, 1, n)
    for r in (1, 4):
        s = spc5.csr_to_spc5(m, r, 8)
        xp = torch.empty(n, dtype=torch.float64, pin_memory=True)
        xp.numpy()[:] = x
        yp = torch.empty(n, dtype=torch.float64, pin_memory=True)
        spc5.spmv(s, xp.numpy(), yp.numpy())
        y = spc5.spmv(s, x)  # pageable in, pageable out
        assert y.tobytes() == yp.numpy().tobytes(), r
        y_mixed = np.empty(n)
        spc5.spmv(s, xp.numpy(), y_mixed)  # pinned in, pageable out
        assert y_mixed.tobytes() == y.tobytes()
        acc = np.full(n, 0.5)
        spc5.spmv_spc5_scalar(s, x, acc)  # accumulate: y is read from and written to pageable memory
        accp = torch.full((n,), 0.5, dtype=torch.float64).pin_memory()
        spc5.spmv_spc5_scalar(s, xp.numpy(), accp.numpy())
        assert acc.tobytes() == accp.numpy().tobytes()


def test_cli_stats_verify_fit(spc5, tmp_path, capsys):
    """The other reference CLI commands on the GPU functions: `stats`
    (cli.py:81-111), `verify` with the mask fault injection (cli.py:114-152: a
    clean matrix passes every config, a corrupted mask fails) and `fit`
    (cli.py:188-199) over records written by `bench`."""
    from paper_2307_14774_b200.__main__ import main
    assert main(["stats", "--matrix", "dense:32", "--matrix", "random:500,600,9,0.5,1",
                 "--format", "b1,b8"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].split()[:4] == ["matrix", "dim", "nnz", "nnz/row"]
    assert out[1].startswith("dense:32") and "100%|100%" in out[1]
    assert out[2].startswith("random:500,600,9,0.5,1") and "500x600" in out[2]
    spec = "random:400,400,11,0.4,5"
    assert main(["verify", "--matrix", spec, "--format", "b2,b4", "--trials", "2"]) == 0
    ok = [ln for ln in capsys.readouterr().out.splitlines() if ln.startswith(spec)]
    assert len(ok) == 2 * 12 and all("pass" in ln.lower() or "ok" in ln.lower() for ln in ok), ok[:2]
    assert main(["verify", "--matrix", spec, "--format", "b2", "--strategy", "expand",
                 "--reduction", "hsum", "--xload", "partial", "--inject-mask-corruption", "7"]) == 1
    records = []
    for i, n in enumerate((300, 600, 900, 1200, 1500, 1800)):
        out_csv = tmp_path / f"r{i}.csv"
        assert main(["bench", "--matrix", f"random:{n},{n},10,0.5,{i}", "--format", "b1",
                     "--reps", "2", "--warmup", "1", "--out", str(out_csv)]) == 0
        records += spc5.read_records(out_csv)
    merged = tmp_path / "all.csv"
    spc5.write_records(merged, records)
    capsys.readouterr()
    assert main(["fit", str(merged), "--min-records", "5"]) == 0
    assert "cost/block" in capsys.readouterr().out
    assert main(["fit", str(merged), "--min-records", "50"]) == 2
