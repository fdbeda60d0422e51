#!/usr/bin/env python
"""SPC5 beta(r,c) SpMV benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

Workload (N=1 default): BASELINE config 2 -- fp64 27-point stencil on a 128^3
grid (2,097,152 rows, 55,742,968 nnz, position-keyed U(-1,1) values, diagonal
27, x ~ U(-1,1) seed 1), in all four formats beta(1,8), beta(2,8), beta(4,8),
beta(8,8).  One step = y_f = A_f . x for the four formats (device-resident
inputs, one K2 launch each).  Inputs (0.5-0.6 GB per format) are larger than
the 126 MB L2, so no flush is needed between steps; x (16.8 MB) stays L2
resident by design.

metric  GFLOP/s = sum_f 2*nnz / t (bench.py:183 of the reference).
roofline  HBM: algorithmic bytes per launch = filling_stats(s).footprint_bytes
          + 8*num_cols (x) + 8*num_rows (y), over the mean
          CUDA-event launch time of the SpMV kernel; peak = MEASURED_PEAKS.json.
e2e     the same products through the public API (paper_2307_14774_b200.spmv)
        on pinned host numpy buffers: H2D x + kernel + D2H y per format.
cpu_baseline  the C restatement of the reference scalar kernel
        (oracle/spc5_oracle.c, kernels.py:121-143) on all host threads.

N > 1 (torchrun): weak scaling by default -- the stencil on an
128 x 128 x (128 N) box, split into nnz-balanced row-panel shards
(partition_by_nnz), i.e. one 128^3 cube of rows per GPU; each rank converts
only its rows and one step is one product per format with x replicated and no
data-path collective.  --scaling strong splits the config's one matrix (the
default for config 5, BASELINE's multi-GPU config).  The iterated form x <-
A.x with the y-slices all-gathered over NCCL is reported beside
it.  --impl reference runs the CPU port on rank 0 only; the other ranks exit 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
def build_matrices(cfg_id: int, formats, rank_rows=None):
    """Device-generate the config's CSR (or a row slice) and convert to each format."""
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200 import csr_to_spc5, csr_to_spc5_device
    from paper_2307_14774_b200.workloads import CONFIGS, config1
    cfg = CONFIGS[cfg_id]
    prec = cfg["precision"]
    mats = {}
    if cfg_id == 1:
        m = config1()
        for (r, vs) in formats:
            mats[(r, vs)] = csr_to_spc5(m, r, vs)
        return mats, m.num_rows, m.num_cols
    tdt = torch.float64 if prec == "f64" else torch.float32
    pcode = 1 if prec == "f64" else 0
    if cfg.get("gen") in ("powerlaw", "fem"):
        from paper_2307_14774_b200.workloads import PL_TABLE_BITS, powerlaw_len_table
        N, C = cfg["rows"], cfg["cols"]
        table = torch.from_numpy(powerlaw_len_table()).to("cuda")
        rp = torch.empty(N + 1, dtype=torch.int64, device="cuda")
        if cfg["gen"] == "powerlaw":
            nat.check(nat.lib.spc5_gen_powerlaw_rowptr(N, 0, N, 0, table.data_ptr(), PL_TABLE_BITS,
                                                       rp.data_ptr(), 0))
        else:
            nat.check(nat.lib.spc5_gen_fem_rowptr(N // 3, 0, N, rp.data_ptr(), 0))
        nnz = int(rp[-1])
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        va = torch.empty(nnz, dtype=tdt, device="cuda")
        if cfg["gen"] == "powerlaw":
            nat.check(nat.lib.spc5_gen_powerlaw_fill(N, 0, N, pcode, 0, table.data_ptr(),
                                                     PL_TABLE_BITS, rp.data_ptr(), ci.data_ptr(),
                                                     va.data_ptr(), 0))
        else:
            nat.check(nat.lib.spc5_gen_fem_fill(N // 3, 0, N, pcode, 0, rp.data_ptr(),
                                                ci.data_ptr(), va.data_ptr(), 0))
        torch.cuda.synchronize()
        for (r, vs) in formats:
            mats[(r, vs)] = csr_to_spc5_device(N, C, rp, ci, va, r, vs)
        del rp, ci, va
        torch.cuda.empty_cache()
        return mats, N, C
    if "n" not in cfg:
        raise SystemExit(f"config {cfg_id} generator not available in this build")
    n = cfg["n"]
    N = n ** 3
    for (r, vs) in formats:
        lo, hi, base = (0, N, 0) if rank_rows is None else rank_rows(r)
        rows = hi - lo
        rp = torch.empty(rows + 1, dtype=torch.int64, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_rowptr(n, lo, hi, rp.data_ptr(), 0))
        nnz = int(rp[-1])
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        va = torch.empty(nnz, dtype=tdt, device="cuda")
        nat.check(nat.lib.spc5_gen_stencil27_fill(n, lo, hi, pcode, 0, 27.0,
                                                  rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                                  0))
        torch.cuda.synchronize()
        mats[(r, vs)] = csr_to_spc5_device(rows, N, rp, ci, va, r, vs, block_base=base)
        del rp, ci, va
        torch.cuda.empty_cache()
    return mats, N, N


def alg_bytes(s, vb: int) -> int:
    from paper_2307_14774_b200 import filling_stats
    return filling_stats(s).footprint_bytes + vb * s.num_cols + vb * s.num_rows


def fmt_key(r, vs):
    return f"b({r},{vs})"


# ----------------------------------------------------------------------------- GPU validation
def gpu_validate(s, x_t, cfg_id, n_rows):
    """Refuse to time a wrong kernel (bench.py:163-167): VERIFY_FACTOR budget vs the
    GPU exact oracle (csr_reference on device CSR regenerated for the check)."""
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200.blocks import torch_stream
    y = torch.empty(s.num_rows, dtype=x_t.dtype, device="cuda")
    nat.check(nat.lib.spc5_spmv(s.handle().ptr, x_t.data_ptr(), y.data_ptr(), 0, torch_stream()))
    # exact reference from the matrix's own CSR (device spc5_to_csr keeps it on the GPU)
    h = s.handle()
    nnz = h.info.nnz
    rp = torch.empty(s.num_rows + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    va = torch.empty(max(nnz, 1), dtype=x_t.dtype, device="cuda")
    nat.check(nat.lib.spc5_to_csr(h.ptr, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                  torch_stream()))
    ye = torch.empty(s.num_rows, dtype=torch.float64, device="cuda")
    ya = torch.empty(s.num_rows, dtype=torch.float64, device="cuda")
    nat.check(nat.lib.spc5_csr_exact(s.num_rows, 1 if x_t.dtype == torch.float64 else 0,
                                     rp.data_ptr(), ci.data_ptr(), va.data_ptr(), x_t.data_ptr(),
                                     ye.data_ptr(), ya.data_ptr(), torch_stream()))
    eps = torch.finfo(x_t.dtype).eps
    nnz_row = (rp[1:] - rp[:-1]).clamp(min=1).to(torch.float64)
    floor = 1e-300 if x_t.dtype == torch.float64 else 1e-30
    scaled = (y.to(torch.float64) - ye).abs() / (nnz_row * eps * ya + floor)
    rel = ((y.to(torch.float64) - ye).abs() / ya.clamp(min=1e-300)).max().item()
    worst = scaled.max().item() if scaled.numel() else 0.0
    del rp, ci, va, ye, ya, y
    torch.cuda.empty_cache()
    if worst > 8.0:
        raise SystemExit(f"validation failed: max scaled error {worst} > 8")
    return worst, rel


# ----------------------------------------------------------------------------- CPU legs
def cpu_product_sample(cfg_id, formats, budget_s=15.0, threads=None):
    """Time the oracle port of the reference scalar kernel on host threads.

    Returns (gflops, cores, sample description, per-format y for parity)."""
    from oracle import oracle
    from paper_2307_14774_b200.workloads import (CONFIGS, config1, fem_rows, powerlaw_rows,
                                                 stencil27, stencil27_rows, x_vector)
    cfg = CONFIGS[cfg_id]
    # configs 1-2: the whole matrix; 3-5: the first rows (~4 M nnz, a multiple of
    # every r): conversion and product are panel-local, so the slice's y is
    # the full product's y[:hi] (SURVEY 8(c) sliced oracle)
    if cfg_id == 1:
        m = config1()
    elif cfg_id == 2:
        m = stencil27(cfg["n"], cfg["precision"])
    elif cfg.get("gen") == "powerlaw":
        m = powerlaw_rows(0, 262_144)
    elif cfg.get("gen") == "fem":
        m = fem_rows(0, 49_152)
    else:
        m = stencil27_rows(cfg["n"], 0, 147_456, cfg["precision"])
    x = x_vector(m.num_cols, cfg["precision"])
    threads = threads or oracle.threads()
    flops, secs, reps_total, ys = 0.0, 0.0, 0, {}
    per_fmt_budget = budget_s / len(formats)
    for (r, vs) in formats:
        s = oracle.csr_to_spc5(m, r, vs)
        run = oracle.ScalarRunner(s, x, threads)
        run.run()  # warm-up (page faults, thread pool); also the parity vector
        ys[(r, vs)] = run.y().copy()
        t_f, reps = 0.0, 0
        while t_f < per_fmt_budget and reps < 200:
            t0 = time.perf_counter()
            run.run()
            t_f += time.perf_counter() - t0
            reps += 1
        flops += 2.0 * m.nnz * reps
        secs += t_f
        reps_total += reps
    what = "full products" if cfg_id <= 2 else f"products of rows [0, {m.num_rows})"
    sample = (f"config {cfg_id}: {what}, {reps_total} total over formats "
              f"{[fmt_key(*f) for f in formats]}, C port of kernels.py:121-143, "
              f"{threads} OpenMP threads")
    return flops / secs / 1e9, threads, sample, ys, m, x


def reference_arm(args, formats):
    """--impl reference: the CPU port of the reference path, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    from paper_2307_14774_b200.workloads import CONFIGS, config1, stencil27, x_vector
    cfg = CONFIGS[args.config]
    m = config1() if args.config == 1 else stencil27(cfg["n"], cfg["precision"])
    x = x_vector(m.num_cols, cfg["precision"])
    threads = oracle.threads()
    mats = {f: oracle.csr_to_spc5(m, *f) for f in formats}
    # one step = a bounded sample: the same fraction of every format's panels
    runners = [oracle.ScalarRunner(mats[f], x, threads) for f in formats]
    for rn in runners:
        rn.run()
    t0 = time.perf_counter()
    for rn in runners:
        rn.run()
    full = time.perf_counter() - t0
    del runners
    frac = min(1.0, 0.25 / max(full, 1e-9))

    def sub(s, lo, hi):
        b0, b1 = int(s.block_rowptr[lo]), int(s.block_rowptr[hi])
        off = oracle.block_value_offsets(s)
        v0, v1 = int(off[b0]), int(off[b1])
        return oracle.OracleSpc5(min(hi * s.r, s.num_rows) - lo * s.r, s.num_cols, s.r, s.vs,
                                 s.block_rowptr[lo:hi + 1] - b0, s.block_colidx[b0:b1],
                                 s.block_masks[b0 * s.r:b1 * s.r], s.values[v0:v1])
    samples = []
    for f in formats:
        s = mats[f]
        hi = max(1, int(s.num_panels * frac))
        samples.append(oracle.ScalarRunner(sub(s, 0, hi), x, threads))
    nnz_step = sum(sm.s.nnz for sm in samples)
    for _ in range(args.warmup):
        for sm in samples:
            sm.run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for sm in samples:
            sm.run()
    el = time.perf_counter() - t0
    val = 2.0 * nnz_step * args.steps / el / 1e9
    sample = (f"{frac:.3f} of the panels of each of {[fmt_key(*f) for f in formats]} per step "
              f"({nnz_step} nnz/step), C port of the reference scalar kernel (kernels.py:121-143)")
    line = {"impl": "reference", "metric": "SpMV GFLOP/s (2*nnz/t)", "value": val,
            "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": CONFIGS[args.config]["precision"], "data": "synthetic",
            "config": {"workload": CONFIGS[args.config]["name"],
                       "formats": [fmt_key(*f) for f in formats]},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def ours_single(args, formats):
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200 import spmv
    from paper_2307_14774_b200.blocks import torch_stream
    from paper_2307_14774_b200.workloads import CONFIGS, x_vector

    cfgd = CONFIGS[args.config]
    prec = cfgd["precision"]
    vb = 8 if prec == "f64" else 4
    tdt = torch.float64 if prec == "f64" else torch.float32
    t_conv = time.perf_counter()
    mats, num_rows, num_cols = build_matrices(args.config, formats)
    torch.cuda.synchronize()
    t_conv = time.perf_counter() - t_conv
    x_np = x_vector(num_cols, prec)
    x = torch.from_numpy(x_np).to("cuda")
    ys = {f: torch.empty(num_rows, dtype=tdt, device="cuda") for f in formats}
    validation = {fmt_key(*f): gpu_validate(mats[f], x, args.config, num_rows) for f in formats}
    handles = {f: mats[f].handle().ptr for f in formats}
    st = torch_stream()
    stream = torch.cuda.current_stream()

    def run(f, n, stream_handle=None):
        sh = st if stream_handle is None else stream_handle
        launches = 0
        for _ in range(n):
            nat.check(nat.lib.spc5_spmv(handles[f], x.data_ptr(), ys[f].data_ptr(), 0, sh))
            launches += nat.last_launch_count()
        return launches

    for _ in range(args.warmup):
        for f in formats:
            run(f, 1)
    torch.cuda.synchronize()
    # latency-bound configs (config 1: 1.9 MB, L2-resident): the K launches of
    # a format are captured once in a CUDA graph and replayed, so the timed
    # region measures the kernels, not the Python launch loop
    graphs, graph_launches = {}, {}
    if args.config == 1:
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        for f in formats:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                graph_launches[f] = run(f, args.steps, int(cap.cuda_stream))
            graphs[f] = g
        torch.cuda.synchronize()
        for f in formats:  # warm replay
            graphs[f].replay()
        torch.cuda.synchronize()
    # timed region: the K products of each format back to back (K steps of one
    # product per format), one event pair per format bracketing its K launches
    ev = [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
          for _ in formats]
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for i, f in enumerate(formats):
        ev[i][0].record(stream)
        if f in graphs:
            graphs[f].replay()
            launches += graph_launches[f]
        else:
            launches += run(f, args.steps)
        ev[i][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    elapsed = e0.elapsed_time(e1) * 1e-3
    per = {f: [ev[i][0].elapsed_time(ev[i][1]) * 1e-3 / args.steps] for i, f in enumerate(formats)}
    flops_step = sum(2.0 * mats[f].nnz for f in formats)
    value = flops_step * args.steps / elapsed / 1e9
    peak, peak_kind = peaks()
    fmts = {}
    tot_bytes, tot_time = 0.0, 0.0
    for f in formats:
        t = statistics.mean(per[f])
        b = alg_bytes(mats[f], vb)
        tot_bytes += b
        tot_time += t
        fmts[fmt_key(*f)] = {"us": t * 1e6, "gflops": 2.0 * mats[f].nnz / t / 1e9,
                             "alg_bytes": b, "gbs": b / t / 1e9, "frac": b / t / 1e9 / peak,
                             "nnz": mats[f].nnz, "num_blocks": mats[f].num_blocks,
                             "max_scaled_err": validation[fmt_key(*f)][0]}
    achieved = tot_bytes / tot_time / 1e9
    # traffic: DRAM bytes per K2 launch from the committed ncu --set full capture
    # (mean over the format launches, like alg_bytes_per_launch below)
    traffic, traffic_fmt = None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tr = json.loads(tf.read_text()).get(f"config{args.config}")
        if tr and tr.get("per_launch_bytes"):
            traffic_fmt = tr["per_launch_bytes"]
            traffic = sum(traffic_fmt.values()) / len(traffic_fmt)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "alg_bytes_per_launch": tot_bytes / len(formats),
                "traffic_per_launch_by_kernel": traffic_fmt,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
                "alg_bytes_per_step": tot_bytes,
                "kernel": "spc5::spmv_kernel (K2), mean launch time per format (CUDA events around its K launches)"}

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        xp = torch.empty(num_cols, dtype=tdt, pin_memory=True)
        xp.numpy()[:] = x_np
        yp = {f: torch.empty(num_rows, dtype=tdt, pin_memory=True) for f in formats}
        for _ in range(max(1, min(args.warmup, 3))):
            for f in formats:
                spmv(mats[f], xp.numpy(), yp[f].numpy())
        e2e_steps = max(3, min(args.steps, 50))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            for f in formats:
                spmv(mats[f], xp.numpy(), yp[f].numpy())
        el = time.perf_counter() - t0
        for f in formats:  # the e2e result is the device result
            assert torch.equal(yp[f].to("cuda"), ys[f]), "e2e result differs from device result"
        e2e = {"value": flops_step * e2e_steps / el / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": vb * num_cols * len(formats),
               "d2h_bytes_per_step": vb * num_rows * len(formats), "steps": e2e_steps,
               "path": "paper_2307_14774_b200.spmv(numpy pinned) -> spc5_spmv_host"}

    # ---- CPU baseline (oracle port of the reference scalar kernel), rank 0, N=1
    cpu = None
    if not args.no_cpu_baseline:
        del_mats = None
        gfl, cores, sample, cpu_ys, m_host, x_host = cpu_product_sample(args.config, formats,
                                                                          budget_s=12.0)
        from oracle import oracle
        _, abs_ref = oracle.csr_reference(m_host, x_host)
        parity = {}
        for f in formats:
            err = oracle.relative_error(ys[f].cpu().numpy()[:m_host.num_rows], cpu_ys[f],
                                        abs_ref)
            parity[fmt_key(*f)] = float(err.max())
        cpu = {"value": gfl, "unit": "GFLOP/s", "cores": cores, "kind": "port",
               "sample": sample, "max_rel_err_gpu_vs_cpu": parity}

    line = {"metric": "SpMV GFLOP/s (2*nnz/t)", "value": value, "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            # --gpus N runs one n^3 cube of rows per GPU for config 2 (weak)
            "scaling": args.scaling, "vs_baseline": None, "dtype": prec,
            "data": "synthetic",
            "config": {"workload": cfgd["name"], "formats": [fmt_key(*f) for f in formats],
                       "num_rows": num_rows,
                       "nnz": mats[formats[0]].nnz,
                       "step": "y_f = A_f.x for every format, device-resident x/y",
                       "order": "the K products of each format run back to back"
                                + (" (replayed from one CUDA graph per format)" if graphs else ""),
                       "l2": "inputs larger than L2 (no flush); x L2-resident by design",
                       "conversion_s": t_conv},
            "roofline": roofline, "formats": fmts, "gpu_launches": launches,
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--formats", default=None, help="e.g. 1,8;2,8")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: weak = one n^3 stencil cube per GPU (default, config 2); "
                         "strong = the config's one matrix split over the GPUs (config 5)")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "weak" if args.config in (2, 6) else "strong"
    if args.warmup < 3:
        args.warmup = 3
    from paper_2307_14774_b200.workloads import CONFIGS
    formats = CONFIGS[args.config]["formats"]
    if args.formats:
        formats = [tuple(int(v) for v in f.split(",")) for f in args.formats.split(";")]
    if args.impl == "reference":
        reference_arm(args, formats)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2307_14774_b200.distributed import bench_distributed
        bench_distributed(args, formats)
        return
    import torch
    torch.cuda.set_device(0)
    ours_single(args, formats)


if __name__ == "__main__":
    main()
