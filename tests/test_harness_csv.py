"""Harness integration, CPU: the CSV v1 records, the scatter
companion, the GPU companion and the per-block cost fit keep the reference's
contracts (bench.py:43-248; its tests/test_bench.py checks the same)."""

import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2307_14774_b200 import (CSV_VERSION_LINE, BenchRecord, InsufficientDataError,
                                   fit_cost_model, read_records, spearman_rank_correlation,
                                   write_records, write_scatter)
from paper_2307_14774_b200.harness import GpuRecord, write_gpu_records

# the reference's v1 column order (bench.py:54-70, 82)
V1_COLUMNS = ["matrix", "precision", "r", "vs", "strategy", "reduction", "x_load", "workers",
              "reps", "median_seconds", "gflops", "filling", "num_blocks"]


def _rec(i, r=1, vs=8, prec="f64", nb=None, t=None):
    nb = nb if nb is not None else 1000 * (i + 1)
    t = t if t is not None else 2e-9 * nb
    return BenchRecord(matrix=f"m{i}", precision=prec, r=r, vs=vs, strategy="compact",
                       reduction="hsum", x_load="partial", workers=1, reps=10,
                       median_seconds=t, gflops=0.1 * (i + 1) / 3.0, filling=1.0 / 3.0 + i,
                       num_blocks=nb)


def test_csv_round_trip_is_field_identical(tmp_path):
    recs = [_rec(i) for i in range(4)]
    p = tmp_path / "b.csv"
    write_records(p, recs)
    lines = p.read_text().splitlines()
    assert lines[0] == CSV_VERSION_LINE
    assert lines[1].split(",") == V1_COLUMNS
    assert read_records(p) == recs


def test_csv_rejects_foreign_header_and_short_rows(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text(CSV_VERSION_LINE + "\nmatrix,r\nx,1\n")
    with pytest.raises(ValueError):
        read_records(p)
    write_records(p, [_rec(0)])
    p.write_text(p.read_text() + "m9,f64,1\n")
    with pytest.raises(ValueError):
        read_records(p)


def test_scatter_companion(tmp_path):
    recs = [_rec(i, r=2, vs=4) for i in range(3)]
    p = tmp_path / "s.csv"
    write_scatter(p, recs)
    lines = p.read_text().splitlines()
    assert lines[0] == "# spc5 bench scatter v1"
    row = lines[2].split(",")
    assert float(row[4]) == recs[0].avg_nnz_per_block and float(row[5]) == recs[0].gflops


def test_gpu_companion(tmp_path):
    g = GpuRecord(matrix="m", r=1, vs=8, device="cuda:0", median_us=100.5, alg_bytes=581278148,
                  achieved_gbs=5783.9, peak_gbs=6468.6, roofline_frac=0.894)
    p = tmp_path / "g.csv"
    write_gpu_records(p, [g])
    lines = p.read_text().splitlines()
    assert lines[0] == "# spc5 bench gpu v1"
    assert lines[2].split(",")[5] == "581278148"


def test_cost_fit_constant_per_block_cost():
    recs = [_rec(i) for i in range(6)]  # t = 2 ns * nb exactly
    fit = fit_cost_model(recs)[(1, 8, "f64")]
    assert fit.cost_per_block_seconds == pytest.approx(2e-9, rel=1e-12)
    assert fit.r_squared == pytest.approx(1.0) and fit.constant_cost


def test_cost_fit_groups_and_insufficient_data():
    recs = [_rec(i) for i in range(5)] + [_rec(i, r=4) for i in range(2)]
    with pytest.raises(InsufficientDataError, match="r=4 vs=8 f64"):
        fit_cost_model(recs)
    noisy = [_rec(i, t=1e-6 * ((-1) ** i) + 1e-5) for i in range(6)]
    assert not fit_cost_model(noisy)[(1, 8, "f64")].constant_cost


def test_spearman_with_ties():
    assert spearman_rank_correlation([1, 2, 3, 4], [10, 20, 30, 40]) == pytest.approx(1.0)
    assert spearman_rank_correlation([1, 2, 3, 4], [4, 3, 2, 1]) == pytest.approx(-1.0)
    a, b = [1, 2, 2, 3], [1, 3, 2, 4]
    ra = np.array([0, 1.5, 1.5, 3]) - 1.5
    rb = np.array([0, 2, 1, 3]) - 1.5
    want = float(ra @ rb / np.sqrt((ra @ ra) * (rb @ rb)))
    assert spearman_rank_correlation(a, b) == pytest.approx(want)
    assert spearman_rank_correlation([1, 1, 1], [1, 2, 3]) == 0.0


REF_SRC = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not mounted (GPU box)")
def test_reference_reads_our_csv_and_we_read_its(tmp_path):
    sys.path.insert(0, str(REF_SRC))
    try:
        ref = importlib.import_module("spc5.bench")
    finally:
        sys.path.remove(str(REF_SRC))
    recs = [_rec(i) for i in range(6)]
    ours = tmp_path / "ours.csv"
    write_records(ours, recs)
    got = ref.read_records(ours)
    assert [tuple(vars(g).values()) for g in got] == [tuple(vars(r).values()) for r in recs]
    theirs = tmp_path / "theirs.csv"
    ref.write_records(theirs, got)
    assert theirs.read_text() == ours.read_text()
    assert read_records(theirs) == recs
    fr = ref.fit_cost_model(got)[(1, 8, "f64")]
    fo = fit_cost_model(recs)[(1, 8, "f64")]
    assert fr.cost_per_block_seconds == fo.cost_per_block_seconds
    assert fr.r_squared == fo.r_squared
