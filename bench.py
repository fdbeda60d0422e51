#!/usr/bin/env python
"""SPC5 beta(r,c) SpMV benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

Workload (default, N=1): BASELINE config 5 -- the fp64 27-point stencil on a
400^3 grid (64,000,000 rows, 1,719,374,392 nnz, position-keyed U(-1,1)
values, diagonal 27, x ~ U(-1,1) seed 1), in all four formats beta(1,8),
beta(2,8), beta(4,8), beta(8,8).  One step = y_f = A_f . x for the four
formats (device-resident inputs, one K2 launch each).  Each format's arrays
(16-18 GB) are ~130x the 126 MB L2, so no flush is needed between steps.
Conversion (K1) and the validation run before the timed region.

metric  GFLOP/s = sum_f 2*nnz / t (bench.py:183 of the reference).
roofline  HBM: algorithmic bytes per launch = filling_stats(s).footprint_bytes
          + 8*num_cols (x) + 8*num_rows (y), over the mean
          CUDA-event launch time of the SpMV kernel; peak = MEASURED_PEAKS.json.
e2e     the same products through the public API (paper_2307_14774_b200.spmv)
        on pinned host numpy buffers: H2D x + kernel + D2H y per format.
cpu_baseline  the C restatement of the reference scalar kernel
        (oracle/spc5_oracle.c, kernels.py:121-143) on all host threads, over
        a stated row slice of the same matrix (products are panel-local).
validation  before timing, every format's y is checked against exact
        double-double row sums of the GENERATOR's CSR (not a CSR rebuilt from
        the converted matrix), with the reference's VERIFY_FACTOR budget
        (bench.py:163-167: refuse to time a wrong kernel).

N > 1 (torchrun): strong scaling by default -- the config's one matrix split
into nnz-balanced row-panel shards (partition_by_nnz); each rank converts only
its rows and one step is one product per format with x replicated (no
data-path collective).  The iterated form x <- A.x with the y-slices
all-gathered over NCCL (BASELINE config 5's 100 products) is reported beside
it.  --scaling weak runs one 128^3 stencil cube per GPU instead (config 2/6).
--impl reference runs the CPU port of the reference kernel on rank 0 only
(the other ranks exit 0) over the same row slice as cpu_baseline; it never
loads the CUDA library.
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
DEFAULT_CONFIG = 5


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
def fmt_key(r, vs):
    return f"b({r},{vs})"


def config_dict(cfg_id: int, formats, world: int = 1, scaling: str = "strong") -> dict:
    """The `config` object of the JSON line -- identical in both arms."""
    from paper_2307_14774_b200.workloads import CONFIGS, config_shape
    cfg = CONFIGS[cfg_id]
    rows, cols = config_shape(cfg)
    d = {"workload": cfg["name"], "formats": [fmt_key(*f) for f in formats],
         "num_rows": rows, "num_cols": cols, "precision": cfg["precision"],
         "step": "y_f = A_f.x for every format (one product per format)",
         "l2": "per-format matrix arrays larger than the 126 MB L2 (no flush needed)"
               if cfg_id != 1 else "L2-resident (1.9 MB; latency-bound, reported as such)",
         "seeds": {"matrix": 0, "x": 1}}
    if world > 1:
        d["parallelism"] = f"row-panel shards x{world} (partition_by_nnz), {scaling} scaling"
    return d


def cpu_sample_rows(cfg_id: int):
    """Row slice [lo, hi) of the config's matrix that the CPU legs run (a
    multiple of every r; conversion and product are panel-local, so the
    slice's y equals rows [lo, hi) of the full product -- SURVEY 8(c))."""
    from paper_2307_14774_b200.workloads import CONFIGS, config_shape
    cfg = CONFIGS[cfg_id]
    n, _ = config_shape(cfg)
    if cfg_id in (1, 2, 6):
        return 0, n                      # the whole matrix
    if cfg.get("gen") == "powerlaw":
        return 0, 262_144
    if cfg.get("gen") == "fem":
        return 0, 49_152
    mid = (n // 2) // 8 * 8               # 400^3: one interior slab of 2^20 rows
    return mid, mid + (1 << 20)


def host_sample(cfg_id: int):
    """(host CSR of the CPU sample rows, lo, hi, x) -- no CUDA involved."""
    from paper_2307_14774_b200.workloads import CONFIGS, config1, host_rows, x_vector
    cfg = CONFIGS[cfg_id]
    lo, hi = cpu_sample_rows(cfg_id)
    m = config1() if cfg_id == 1 else host_rows(cfg, lo, hi)
    x = x_vector(m.num_cols, cfg["precision"])
    return m, lo, hi, x


def build_matrices(cfg_id: int, formats, validate: bool = True):
    """Generate the config's CSR on the device once, convert it to every format
    (K1) and validate each format's product against exact row sums of that
    generator CSR.  Returns (mats, num_rows, num_cols, x, validation, conv_s)."""
    import torch

    from paper_2307_14774_b200 import _native as nat
    from paper_2307_14774_b200 import csr_to_spc5_device
    from paper_2307_14774_b200.blocks import torch_stream
    from paper_2307_14774_b200.workloads import CONFIGS, config1, device_rows, x_vector
    cfg = CONFIGS[cfg_id]
    prec = cfg["precision"]
    tdt = torch.float64 if prec == "f64" else torch.float32
    if cfg_id == 1:
        m = config1()
        N, C = m.num_rows, m.num_cols
        rp = torch.from_numpy(m.row_ptr).cuda()
        ci = torch.from_numpy(m.col_idx).cuda()
        va = torch.from_numpy(m.values).cuda()
    else:
        from paper_2307_14774_b200.workloads import config_shape
        N, C = config_shape(cfg)
        rp, ci, va = device_rows(cfg, 0, N)
    x_np = x_vector(C, prec)
    x = torch.from_numpy(x_np).to("cuda")
    # exact reference of the generator's CSR (double-double row sums, kernels.py:233-250)
    ye = ya = None
    if validate:
        ye = torch.empty(N, dtype=torch.float64, device="cuda")
        ya = torch.empty(N, dtype=torch.float64, device="cuda")
        nat.check(nat.lib.spc5_csr_exact(N, nat.F64 if prec == "f64" else nat.F32,
                                         rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                         x.data_ptr(), ye.data_ptr(), ya.data_ptr(),
                                         torch_stream()))
        nnz_row = (rp[1:] - rp[:-1]).clamp(min=1).to(torch.float64)
    mats, validation, conv = {}, {}, 0.0
    for f in formats:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = csr_to_spc5_device(N, C, rp, ci, va, *f)
        torch.cuda.synchronize()
        conv += time.perf_counter() - t0
        mats[f] = s
        if validate:
            y = torch.empty(N, dtype=tdt, device="cuda")
            nat.check(nat.lib.spc5_spmv(s.handle().ptr, x.data_ptr(), y.data_ptr(), 0,
                                        torch_stream()))
            eps = torch.finfo(tdt).eps
            floor = 1e-300 if prec == "f64" else 1e-30
            d = (y.to(torch.float64) - ye).abs()
            worst = (d / (nnz_row * eps * ya + floor)).max().item()
            rel = (d / ya.clamp(min=1e-300)).max().item()
            del y, d
            if worst > 8.0:  # VERIFY_FACTOR, kernels.py:43-44
                raise SystemExit(f"validation failed for {fmt_key(*f)}: max scaled error "
                                 f"{worst} > 8 (refusing to time, bench.py:163-167)")
            validation[fmt_key(*f)] = {"max_scaled_err": worst, "max_rel_err_sum_abs": rel}
    del rp, ci, va, ye, ya
    torch.cuda.empty_cache()
    return mats, N, C, x, x_np, validation, conv


def alg_bytes(s, vb: int) -> int:
    from paper_2307_14774_b200 import filling_stats
    return filling_stats(s).footprint_bytes + vb * s.num_cols + vb * s.num_rows


def committed_traffic(cfg_id: int):
    """DRAM bytes per K2 launch from a committed ncu --set full capture
    (profiles/traffic.json), with its source; None when absent."""
    tf = ROOT / "profiles" / "traffic.json"
    if not tf.exists():
        return None, None, None
    tr = json.loads(tf.read_text()).get(f"config{cfg_id}")
    if not tr or not tr.get("per_launch_bytes"):
        return None, None, None
    per = tr["per_launch_bytes"]
    return sum(per.values()) / len(per), per, tr.get("note")


# ----------------------------------------------------------------------------- CPU legs
def cpu_product_sample(cfg_id, formats, budget_s=15.0, threads=None):
    """Time the oracle port of the reference scalar kernel on host threads over
    the config's CPU sample rows.  Returns (gflops, cores, sample, ys, lo, hi, m, x)."""
    from oracle import oracle
    m, lo, hi, x = host_sample(cfg_id)
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
    sample = (f"config {cfg_id}: rows [{lo}, {hi}) ({m.nnz} nnz per format), {reps_total} "
              f"products over formats {[fmt_key(*f) for f in formats]}, C port of "
              f"kernels.py:121-143 (oracle/spc5_oracle.c), {threads} OpenMP threads")
    return flops / secs / 1e9, threads, sample, ys, lo, hi, m, x


def reference_arm(args, formats):
    """--impl reference: the CPU port of the reference path, rank 0 only.

    The reference is pure Python + numpy (no native code to compile); its
    scalar kernel (kernels.py:121-143) restated in C (oracle/spc5_oracle.c)
    runs on all host threads.  One step = one product per format over the
    config's CPU sample rows (a bounded sample of the same matrix).  This arm
    imports only the host-side workload generators; libspc5_b200.so is never
    loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    from paper_2307_14774_b200.workloads import CONFIGS
    m, lo, hi, x = host_sample(args.config)
    threads = oracle.threads()
    runners = [oracle.ScalarRunner(oracle.csr_to_spc5(m, *f), x, threads) for f in formats]
    for _ in range(args.warmup):
        for rn in runners:
            rn.run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for rn in runners:
            rn.run()
    el = time.perf_counter() - t0
    nnz_step = m.nnz * len(formats)
    val = 2.0 * nnz_step * args.steps / el / 1e9
    sample = (f"rows [{lo}, {hi}) of the config-{args.config} matrix ({m.nnz} nnz) in each of "
              f"{[fmt_key(*f) for f in formats]} per step, C port of the reference scalar "
              f"kernel (kernels.py:121-143), {threads} OpenMP threads")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {"impl": "reference", "metric": "SpMV GFLOP/s (2*nnz/t)", "value": val,
            "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": CONFIGS[args.config]["precision"], "data": "synthetic",
            "config": config_dict(args.config, formats, world, args.scaling),
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
    from paper_2307_14774_b200.workloads import CONFIGS

    cfgd = CONFIGS[args.config]
    prec = cfgd["precision"]
    vb = 8 if prec == "f64" else 4
    tdt = torch.float64 if prec == "f64" else torch.float32
    t_setup = time.perf_counter()
    mats, num_rows, num_cols, x, x_np, validation, t_conv = build_matrices(args.config, formats)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    ys = {f: torch.empty(num_rows, dtype=tdt, device="cuda") for f in formats}
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
    per = {f: ev[i][0].elapsed_time(ev[i][1]) * 1e-3 / args.steps for i, f in enumerate(formats)}
    flops_step = sum(2.0 * mats[f].nnz for f in formats)
    value = flops_step * args.steps / elapsed / 1e9
    peak, peak_kind = peaks()
    fmts = {}
    tot_bytes, tot_time = 0.0, 0.0
    for f in formats:
        t = per[f]
        b = alg_bytes(mats[f], vb)
        tot_bytes += b
        tot_time += t
        # K1 (conversion) device time and its algorithmic bytes: the CSR read by
        # each pass (count: row_ptr + col_idx; fill: row_ptr + col_idx + values)
        # plus the SPC5 arrays written
        ct = mats[f].handle().convert_timing()
        nnz, nb = mats[f].nnz, mats[f].num_blocks
        k1_bytes = (2 * (8 * num_rows + 4 * nnz) + vb * nnz          # CSR in, both passes
                    + 8 * (mats[f].num_panels + 1) + 4 * nb           # rowptr, colidx out
                    + nb * f[0] * (1 if f[1] <= 8 else 2) + vb * nnz)  # masks, values out
        k1_ms = ct["k1_count_ms"] + ct["k1_fill_ms"]
        conv = {"k1_ms": k1_ms, "k1_count_ms": ct["k1_count_ms"], "k1_fill_ms": ct["k1_fill_ms"],
                "plan_ms": ct["plan_ms"], "k1_alg_bytes": k1_bytes,
                "k1_gbs": k1_bytes / k1_ms / 1e6 if k1_ms > 0 else None,
                "k1_frac": k1_bytes / k1_ms / 1e6 / peak if k1_ms > 0 else None}
        fmts[fmt_key(*f)] = {"us": t * 1e6, "gflops": 2.0 * mats[f].nnz / t / 1e9,
                             "conversion": conv,
                             "alg_bytes": b, "gbs": b / t / 1e9, "frac": b / t / 1e9 / peak,
                             "nnz": mats[f].nnz, "num_blocks": mats[f].num_blocks,
                             **validation.get(fmt_key(*f), {})}
    achieved = tot_bytes / tot_time / 1e9
    traffic, traffic_fmt, traffic_note = committed_traffic(args.config)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_note and f"committed profile: {traffic_note}",
                "alg_bytes_per_launch": tot_bytes / len(formats),
                "traffic_per_launch_by_kernel": traffic_fmt,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                if peak_kind == "measured" else "fallback (B200_PROFILING.md)",
                "alg_bytes_per_step": tot_bytes,
                "kernel": "spc5::spmv_kernel (K2), mean launch time per format "
                          "(CUDA events around its K launches)"}

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
        del yp
        # the same call on ordinary (pageable) numpy arrays, as a drop-in caller of
        # kernels.py:119-129 would pass them: the copies stage through the driver
        pg_steps = max(2, min(e2e_steps, 5))
        x_pg = np.array(x_np, copy=True)
        y_pg = {f: np.empty(num_rows, dtype=x_np.dtype) for f in formats}
        for f in formats:
            spmv(mats[f], x_pg, y_pg[f])
        t0 = time.perf_counter()
        for _ in range(pg_steps):
            for f in formats:
                spmv(mats[f], x_pg, y_pg[f])
        el_pg = time.perf_counter() - t0
        for f in formats:
            assert np.array_equal(y_pg[f], ys[f].cpu().numpy()), "pageable e2e result differs"
        del y_pg
        e2e = {"value": flops_step * e2e_steps / el / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": vb * num_cols * len(formats),
               "d2h_bytes_per_step": vb * num_rows * len(formats), "steps": e2e_steps,
               "path": "paper_2307_14774_b200.spmv(numpy pinned) -> spc5_spmv_host",
               "pageable": {"value": flops_step * pg_steps / el_pg / 1e9, "unit": "GFLOP/s",
                            "steps": pg_steps,
                            "path": "the same call on pageable numpy arrays"}}

    # ---- CPU baseline (oracle port of the reference scalar kernel), rank 0, N=1
    cpu = None
    if not args.no_cpu_baseline:
        gfl, cores, sample, cpu_ys, lo, hi, m_host, x_host = cpu_product_sample(
            args.config, formats, budget_s=12.0)
        from oracle import oracle
        _, abs_ref = oracle.csr_reference(m_host, x_host)
        parity = {}
        for f in formats:
            err = oracle.relative_error(ys[f][lo:hi].cpu().numpy(), cpu_ys[f], abs_ref)
            parity[fmt_key(*f)] = float(err.max())
        cpu = {"value": gfl, "unit": "GFLOP/s", "cores": cores, "kind": "port",
               "sample": sample, "max_rel_err_gpu_vs_cpu": parity}

    line = {"metric": "SpMV GFLOP/s (2*nnz/t)", "value": value, "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": prec,
            "data": "synthetic",
            "config": config_dict(args.config, formats),
            "matrix": {"nnz": mats[formats[0]].nnz,
                       "order": "the K products of each format run back to back"
                                + (" (replayed from one CUDA graph per format)" if graphs else ""),
                       "conversion_s": t_conv, "setup_s": t_setup},
            "roofline": roofline, "formats": fmts, "gpu_launches": launches,
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--formats", default=None, help="e.g. 1,8;2,8")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--iters", type=int, default=100,
                    help="N > 1: products of the iterated (all-gather) form per format")
    ap.add_argument("--fused", action="store_true",
                    help="N > 1: also time the exchange fused into K2 (NVLink peer stores); "
                         "off by default at N > 1 because it has only run on one-rank groups")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = the config's one matrix split over the GPUs "
                         "(default); weak = one n^3 stencil cube of rows per GPU")
    args = ap.parse_args()
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
