#!/usr/bin/env python
"""bench.py — FDiRW step throughput on B200 (BASELINE.json metric: voxel-updates/s and
HBM GB/s fraction of the FDiRW step at 192³ on 1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl fdirw|reference]
  N>1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step = one FDiRW macro step (a5 superposition + a6 halo exchange when N>1) over the
whole grid, with the kernels built once beforehand by fdirw_build_kernels (a1-a4,
"preconditioned" P; timed separately under "kgen").  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fdirw_inputs as fi  # noqa: E402

METRIC = "voxel-updates/s (FDiRW step)"
UNIT = "voxel-updates/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def _hbm_peak():
    p = _peaks()
    if p and p.get("hbm_gbs"):
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _oracle_problem(cfg, mask):
    import oracle

    oracle.build()
    return oracle.Problem(mask=mask, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt, R=cfg.R,
                          n_fd=cfg.n_fd)


def _oracle_sample(cfg: fi.Config, mask: np.ndarray):
    """The bounded CPU sample of the workload, shared by cpu_baseline and the
    reference arm: an 8-plane target slab through the grid centre, cut to 4 rows of the full x
    extent (192 x 4 x 8 = 6144 targets at 192³; the whole 8-plane slab's kgen would be ~4 h of
    host time), with the kernels of every source that reaches it (oracle kgen, OpenMP over
    sources, timed).  Returns (pb, sbox, tbox, W, t_kgen)."""
    import oracle

    pb = _oracle_problem(cfg, mask)
    nz, ny, nx = mask.shape
    z0, y0 = max(0, nz // 2 - 4), max(0, ny // 2 - 2)
    tbox = (0, nx, y0, min(ny, y0 + 4), z0, min(nz, z0 + 8))
    R = cfg.R
    sbox = oracle.clip_box(pb, (tbox[0] - R, tbox[1] + R, tbox[2] - R, tbox[3] + R, tbox[4] - R, tbox[5] + R))
    t = time.perf_counter()
    W = oracle.build_kernels(pb, sbox)
    return pb, sbox, tbox, W, time.perf_counter() - t


def _box_size(b):
    return (b[1] - b[0]) * (b[3] - b[2]) * (b[5] - b[4])


def cpu_baseline(cfg: fi.Config, mask: np.ndarray, reps: int = 3):
    """The CPU fp64 oracle as it stands, on the host cores: the bounded sample of
    _oracle_sample, its superposition step timed single-threaded and with OpenMP over all cores
    (target planes split between threads, bitwise the same result), its kgen with OpenMP; both
    extrapolated to the whole grid, labelled as such."""
    import oracle

    pb, sbox, tbox, W, t_kgen = _oracle_sample(cfg, mask)
    C = fi.initial_c(mask, "paper").astype(np.float64)
    nt, ns = _box_size(tbox), _box_size(sbox)
    oracle.step_scatter(pb, W, sbox, C, tbox, threads=True)  # warm
    t = time.perf_counter()
    for _ in range(reps):
        oracle.step_scatter(pb, W, sbox, C, tbox, threads=True)
    t_omp = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    oracle.step_scatter(pb, W, sbox, C, tbox)
    t_one = time.perf_counter() - t
    cores = os.cpu_count()
    N = int(mask.size)
    n_fd = oracle.derive(pb).n_fd
    return {"value": nt / t_omp, "unit": UNIT, "cores": cores, "kind": "oracle", "nproc": cores,
            "sample": "oracle fp64 scatter step (OpenMP, %d threads) over the targets of an 8-plane slab through "
                      "the grid centre cut to 4 rows: box x[%d,%d) y[%d,%d) z[%d,%d) = %d voxel-updates, mean of %d; "
                      "kernels of its %d sources by oracle kgen (OpenMP) in %.1f s" % (
                          cores, *tbox, nt, reps, ns, t_kgen),
            "single_thread": {"value": nt / t_one, "unit": UNIT, "cores": 1},
            "kgen": {"sources": ns, "seconds": t_kgen, "cores": cores, "sources_per_s": ns / t_kgen,
                     "window_cell_updates_per_s": ns * cfg.K * n_fd / t_kgen},
            "extrapolated_whole_grid": {"step_seconds": N / (nt / t_omp), "step_seconds_1thread": N / (nt / t_one),
                                        "kgen_seconds": N * t_kgen / ns,
                                        "note": "extrapolated linearly from the sample to all %d voxels (every "
                                                "voxel is a source and a target)" % N}}


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on the host cores, each step
    the oracle superposition (OpenMP) over the same bounded sample cpu_baseline uses."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    cfg = fi.config(args.config, weights=args.weights)
    mask = cfg.mask()
    pb, sbox, tbox, W, t_kgen = _oracle_sample(cfg, mask)
    C = fi.initial_c(mask, "paper").astype(np.float64)
    for _ in range(args.warmup):
        oracle.step_scatter(pb, W, sbox, C, tbox, threads=True)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.step_scatter(pb, W, sbox, C, tbox, threads=True)
    dt = (time.perf_counter() - t) / args.steps
    nt = _box_size(tbox)
    v = nt / dt
    cores = os.cpu_count()
    sample = ("oracle fp64 scatter step (OpenMP, %d threads) over the targets of an 8-plane slab through the grid "
              "centre cut to 4 rows, box x[%d,%d) y[%d,%d) z[%d,%d) of %s (%d voxel-updates per step); kernels of its "
              "%d sources by oracle kgen (OpenMP, %.1f s, untimed)" % (cores, *tbox, args.config, nt, _box_size(sbox),
                                                                      t_kgen))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_name(cfg), "sample": "%d target voxels" % nt},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ fidelity checks (oracle leg)
# Run after every timing, on rank 0 at N = 1: the oracle is the checker here, never a product
# path.  Boxes of cfg3 (192³, particle centre 95.5, r_p = 50): the particle surface, a domain
# corner (uniform liquid) and the particle interior.
FID_BOXES = {"interface": (140, 146, 92, 98, 92, 97), "corner": (0, 5, 185, 192, 0, 3),
             "interior": (93, 99, 94, 100, 95, 99)}
HIST_SOURCES = (140, 144, 92, 96, 92, 95)  # 48 sources straddling the surface (solid + liquid)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def _sl(b):
    return (slice(b[4], b[5]), slice(b[2], b[3]), slice(b[0], b[1]))


class Fidelity:
    """Oracle references for the bench's driver-visible accuracy figures (VERDICT r01 'Missing 5',
    SURVEY §5 metrics): one FDiRW step from the paper's initial field on the FID_BOXES, and the
    oracle's fp64 kernels of HIST_SOURCES for the Fig.11-style weight-value histogram."""

    def __init__(self, cfg, mask):
        import oracle

        self.oracle = oracle
        self.pb = _oracle_problem(cfg, mask)
        self.c0 = fi.initial_c(mask, "paper").astype(np.float64)
        t = time.perf_counter()
        self.ref = {k: oracle.step_box(self.pb, self.c0, b) for k, b in FID_BOXES.items()}
        self.W_hist = oracle.build_kernels(self.pb, HIST_SOURCES)
        self.seconds = time.perf_counter() - t

    def step_boxes(self, field):
        """relL2 of a GPU field one step after c0 against the oracle on every box."""
        return {k: _rel(field[_sl(b)], self.ref[k]) for k, b in FID_BOXES.items()}

    def last_step(self, prev, last, box="interface"):
        """The timed run's LAST step, re-done by the oracle from the field before it."""
        b = FID_BOXES[box]
        return _rel(last[_sl(b)], self.oracle.step_box(self.pb, prev.astype(np.float64), b))

    def histogram(self, stored: dict):
        """Fig.11: off-centre weight values per decade, the oracle's fp64 kernels
        beside each stored format (decoded): count per decade, stored zeros (underflow), median
        relative error."""
        K = self.W_hist.shape[-1]
        off = np.ones(K, bool)
        off[K // 2] = False
        o = self.W_hist[..., off].ravel()
        dec = np.floor(np.log10(np.maximum(o, 1e-300))).astype(int)
        out = {"sources": "x[%d,%d) y[%d,%d) z[%d,%d)" % HIST_SOURCES, "weights": int(o.size),
               "oracle_zero": int((o == 0).sum()),
               "oracle_decades": {str(d): int((dec == d).sum()) for d in range(0, -46, -1) if (dec == d).any() and
                                  (o[dec == d] > 0).any()}}
        for name, W in stored.items():
            g = W[..., off].ravel()
            f = {"zeros_where_oracle_nonzero": int(((g == 0) & (o > 0)).sum()), "median_rel_err": {}}
            for d in range(0, -46, -1):
                sel = (dec == d) & (o > 0)
                if sel.any():
                    f["median_rel_err"][str(d)] = float(np.median(np.abs(g[sel] - o[sel]) / o[sel]))
            out[name] = f
        return out


def _truncation(fd, torch, stream):
    """The method's truncation error (a reported diagnostic, not a gate): one FDiRW
    step (the product, on the GPU) against n_fd whole-grid explicit FD substeps (oracle O6, the
    fine-mesh solver of P:177-181) from the same field.  cfg1 (16³, R2, n_fd = 1000) on the whole
    grid; cfg3 at its domain corner, where FD runs on the uniform-liquid sub-domain
    [0,64) x [128,192) x [0,64) (the particle is > 50 voxels away, so the whole-grid FD equals the
    sub-domain FD there)."""
    import oracle

    out = {}
    cfg = fi.config("cfg1", n_fd=1000, weights="fp32")
    mask = cfg.mask()
    c0 = fi.initial_c(mask, "paper")
    pb = _oracle_problem(cfg, mask)
    ctx = fd.build_kernels(fd.Params(nx=16, ny=16, nz=16, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow,
                                     dt=cfg.dt, radius=cfg.R, n_fd=cfg.n_fd, weights="fp32"), mask, stream=stream)
    try:
        c = torch.from_numpy(c0).cuda()
        fd.run(ctx, c, 1, stream)
        g = c.cpu().numpy()
    finally:
        fd.destroy(ctx)
    ref = oracle.fd_whole_grid(pb, c0.astype(np.float64), 1000)
    out["cfg1"] = {"relL2_vs_whole_grid_fd": _rel(g, ref), "fd_change_relL2": _rel(ref, c0),
                   "oracle_fdirw_vs_fd": _rel(oracle.step_full(pb, c0.astype(np.float64)), ref),
                   "note": "16^3, R2, n_fd=1000 (sigma = 14 voxels > R): one step, paper initial field"}
    cfg3 = fi.config("cfg3")
    m3 = cfg3.mask()
    sub = (slice(0, 64), slice(128, 192), slice(0, 64))
    pbs = _oracle_problem(cfg3, np.ascontiguousarray(m3[sub]))
    c3 = fi.initial_c(m3, "paper").astype(np.float64)
    fd_sub = oracle.fd_whole_grid(pbs, np.ascontiguousarray(c3[sub]), 1000)
    out["cfg3_corner"] = {"box": "x[0,5) y[185,192) z[0,3)", "fd_sub": fd_sub[0:3, 57:64, 0:5]}
    return out


def _ncu_traffic(cfg, bytes_per_launch):
    """dram read+write bytes per launch of the superposition kernel from the newest committed
    `ncu --set full` capture of this config (profiles/r*_superpose_<cfg>_ncu.json), else None."""
    import glob

    best = None
    tag = cfg.name + ("_mx8" if cfg.weights == "mx8" else "")
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_superpose_%s_ncu.json" % tag))):
        try:
            js = json.load(open(f))
            for rec in js.get("launches", []):
                if "superpose" in rec.get("kernel", "") and rec.get("traffic_bytes"):
                    best = (rec["traffic_bytes"], os.path.relpath(f, ROOT))
        except Exception:
            pass
    return best


def _workload_name(cfg):
    return "%s: %s grid, R=%d (K=%d), %s weights, n_fd=%s" % (
        cfg.name, "x".join(map(str, cfg.shape[::-1])), cfg.R, cfg.K,
        cfg.weights, cfg.n_fd or "derived")


def _time_run(fd, torch, ctx, c, args, stream):
    fd.run(ctx, c, args.warmup, stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    fd.run(ctx, c, args.steps, stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / args.steps


def _one_step_field(fd, torch, ctx, mask, stream):
    """The context's field one step after the paper's initial field (fidelity checks)."""
    c = torch.from_numpy(fi.initial_c(mask, "paper")).cuda()
    fd.run(ctx, c, 1, stream)
    return c.cpu().numpy()


def _variant(fd, torch, params, mask, c_host, args, stream, peak, fid=None, hist=None, name=""):
    """A storage variant measured in the same run: its own byte model, step time and, with the
    oracle leg on, relL2 of one step against the oracle on the FID_BOXES."""
    try:
        ctx = fd.build_kernels(params, mask, stream=stream)
    except fd.FdirwError as e:  # a combination the library rejects for this geometry
        return {"unavailable": str(e)}
    try:
        info = ctx.info
        ms = _time_run(fd, torch, ctx, c_host.to("cuda", non_blocking=True), args, stream)
        ceil = fd.read_ceiling(ctx, 5, stream=stream) if params.weights == "mx8" else None
        rel = fid.step_boxes(_one_step_field(fd, torch, ctx, mask, stream)) if fid else None
        if hist is not None and not (params.flags & fd.F_DEDUP_STORAGE):
            hist[name] = fd.export_kernels(ctx, HIST_SOURCES)
    finally:
        fd.destroy(ctx)
    N = int((mask != 2).sum())
    b_w = {"fp32": 4, "mx8": 1.125}.get(params.weights, 2)
    f_u = info["uniform_chunks"] / max(info["chunks"], 1)
    bpv = (1.0 - f_u) * (info["K"] - 1) * b_w + 16
    ach = bpv * N / (ms * 1e-3) / 1e9
    v = {"value": N / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "bytes_per_voxel_update": bpv,
         "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak},
         "weight_bytes": info["weight_bytes"]}
    if ceil:
        v["roofline"]["read_ceiling"] = {"GBps": ceil, "frac": ach / ceil}
    if params.flags & fd.F_DEDUP_STORAGE:
        v.update(uniform_fraction=f_u, uniform_classes=info["uniform_classes"])
    if rel is not None:
        v["relL2_one_step_vs_oracle"] = rel
    return v


def _cfg1_seconds(fd, torch, params, cfg, mask, stream, steps=10):
    """BASELINE configs[0] is quoted in CPU seconds: the whole 16³ problem (every kernel +
    10 steps) by the oracle on the host cores, beside the same through the library on the GPU
    (build + 10 steps + copy back, wall clock)."""
    import oracle

    pb = oracle.Problem(mask=mask, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt, R=cfg.R,
                        n_fd=cfg.n_fd)
    c0 = fi.initial_c(mask, "random", seed=1)
    t = time.perf_counter()
    oracle.step_full(pb, c0.astype(np.float64), steps=steps)
    t_cpu = time.perf_counter() - t
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx = fd.build_kernels(params, mask, stream=stream)
    c = torch.from_numpy(c0).cuda()
    fd.run(ctx, c, steps)
    out = c.cpu()
    t_gpu = time.perf_counter() - t
    fd.destroy(ctx)
    return {"oracle_seconds": t_cpu, "oracle_cores": os.cpu_count(), "gpu_seconds": t_gpu, "steps": steps,
            "note": "whole problem: every source's kernel (oracle kgen, OpenMP) + %d fp64 scatter steps; GPU: "
                    "fdirw_build_kernels + fdirw_run(%d) + copy back, wall clock" % (steps, steps),
            "checksum": float(out.double().sum())}


def _kgen_line(t_kgen, cells_algo, info, cfg, world):
    """kgen (one-time build, a3+a4).  `seconds` = wall time of fdirw_build_kernels (mask upload,
    window dedup, kgen, expand into the gather layout, allocation).  Algorithmic work = every
    source's window × K × n_fd FD cell-updates (the literal method).  The kernel itself
    (device time from CUDA events around its launch, fdirw_info.kgen_kernel_ms) runs the distinct
    windows only, kgen_steps stencil passes each (the Chebyshev degree m, reading A30, or n_fd):
    its rooflines count those passes.  Shared memory (128 B/clk/SM): the column kernel reads 4
    lateral neighbours and writes its cell, 20 B per cell-pass; the balanced pairs kernel (R = 5,
    8; two columns per thread over z segments) moves 4.23 (R5) / 4.29 (R8) accesses of
    4 B per cell-pass.  FP32 lanes: 11 lane-ops per literal substep cell, 8 per Chebyshev
    cell-pass (row form).  `vs_column_design` rates the same cell-passes against the round-1
    column kernel's 20 B ceiling."""
    p = _peaks() or {}
    mhz = float(p.get("sm_max_mhz", 1965.0))
    steps = info["kgen_steps"]
    cheb = steps != info["n_fd"]
    kms = info["kgen_kernel_ms"]
    passes = info["kgen_windows"] * world * cfg.K * steps  # computed cell-passes
    rate = passes / (kms * 1e-3) if kms > 0 else 0.0
    pairs = cfg.R in (5, 8) and not (info.get("flags", 0) & 128)
    # accesses per pair and pass / real cells per pair (kgen_bal.cu): R5 (35+11)+(35+12) over 22
    # cells, R8 (35+11)+(40+13)+(35+12) over 34 cells
    smem_b = {5: 4.0 * 93 / 22, 8: 4.0 * 146 / 34}[cfg.R] if pairs else 20.0
    smem_peak = 148 * 128 * mhz * 1e6
    ops = (8.0 * (steps - 8) + 11.0 * 8) / steps if cheb else 11.0
    alu_peak = 148 * 128 * mhz * 1e6 / ops
    return {"seconds": t_kgen, "kernel_ms": kms,
            "cell_passes_per_s": rate,
            "cell_passes": passes,
            "rate_note": "cell_passes_per_s = the kernel's own work rate: distinct windows x K x stencil passes "
                         "(%d per window) / kernel time; literal_equivalent_* counts every source's window x K x "
                         "n_fd substeps of the literal method (P:109), which the kernel does not execute" % steps,
            "literal_equivalent_cell_updates": cells_algo,
            "literal_equivalent_cell_updates_per_s": cells_algo / (kms * 1e-3) if kms > 0 else None,
            "n_fd": info["n_fd"], "method": "chebyshev" if cheb else "substeps", "passes_per_window": steps,
            "builds_timed": 3 if info.get("_median3") else 1,
            "windows_computed": info["kgen_windows"] * world, "sources": info["kgen_sources"] * world,
            "roofline": {"bound": "smem", "achieved": rate * smem_b / 1e12, "peak": smem_peak / 1e12,
                         "unit": "TB/s", "frac": rate * smem_b / smem_peak,
                         "note": "kgen kernel only: %.1f B of shared-memory traffic per window cell-pass "
                                 "x distinct windows x K x %d passes / kernel time; peak = 148 SMs x "
                                 "128 B/clk x %.0f MHz" % (smem_b, steps, mhz)},
            "alu": {"achieved": rate, "peak": alu_peak, "unit": "cell-passes/s", "frac": rate / alu_peak,
                    "lane_ops_per_cell_pass": ops},
            "kernel": "kgen_bal_kernel (2 columns/thread, balanced z segments)" if pairs else "kgen_kernel (1 column/thread)",
            "vs_column_design": {"frac": rate * 20.0 / smem_peak,
                                 "note": "the same rate against the round-1 column kernel's 20 B/cell-pass "
                                         "shared-memory ceiling (%.2e cell-passes/s)" % (smem_peak / 20.0)}}


def _coarse_roofline(info, ms, steps):
    """Whole coarse step against HBM: algorithmic bytes = stored P̃ (+diag, P_BC) and the group
    vector in and out (12 B per group) per step, plus the Ω_L field read by the one map and written
    by the one remap of the run (8 B per Ω_L voxel, over the run's steps: fdirw_coarse_run keeps the
    state in group values between steps).  P̃ fits in L2 and stays there across steps
    (evict_last), so frac > 1 is possible; it is the step's figure, not one kernel's."""
    peak, src = _hbm_peak()
    algo = info["p_bytes"] + 12 * info["n_groups"] + 8 * info["n_region"] / max(steps, 1)
    ach = algo / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
            "kernel": "coarse step in group space (k_gemv, + Eq.7 with a far field); one map and one remap per run",
            "bytes_per_step": algo, "peak_source": src}


def run_coarse(args):
    """NEXT row N1: the paper's coarse-mesh FDiRW step on the near-field liquid
    of the config's particle (r_p + 5Δh), b = 5, 1 GPU.  Metric: fine Ω_L
    voxels updated per second (N_L per step)."""
    import torch

    import paper_2408_11376_b200 as fd

    cfg = fi.config(args.config, weights=args.weights)
    mask = cfg.mask()
    r_p = cfg.geometry.get("r_p", 50)
    far = cfg.v_far > 0  # N2: the config's mask already labels the far-field reservoir 2
    region = mask.astype(np.uint8) if far else fi.near_field(mask, r_p)
    nz, ny, nx = cfg.shape
    params = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                       radius=cfg.R, n_fd=cfg.n_fd, weights=cfg.weights, v_far=cfg.v_far)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx = fd.coarse_build(params, region, block=args.block)
    t_build = time.perf_counter() - t
    info = ctx.info
    c = torch.from_numpy(fi.initial_c(mask, "paper")).cuda()
    K0 = fd.coarse_far_init(ctx, c, cfg.c_far0) if far else None
    fd.coarse_run(ctx, c, args.warmup)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        fd.coarse_run(ctx, c, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    NL, N = info["n_region"], info["n_groups"]
    extra = {}
    if far:  # Eq.7 balance over Ω_L + reservoir after all steps
        cf = fd.coarse_far_get(ctx)
        m = float(c.double()[torch.from_numpy(region == 1).cuda()].sum())
        extra = {"c_far": cf, "mass_rel_err": abs(m + cf * cfg.v_far - K0) / K0}
    line = {"metric": "voxel-updates/s (coarse-mesh FDiRW step, NEXT row N1)", "value": NL / (ms * 1e-3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": {"fp32": "f32", "fp16": "f16", "bf16": "bf16", "mx8": "mx8"}[cfg.weights] + "-P/f32-accum",
            "data": "synthetic",
            "config": {"workload": "N1%s coarse mesh on the %s near-field liquid (r_p+5), b=%d"
                                   % ("+N2 far field" if far else "", cfg.name, args.block),
                       "N_L": NL, "N": N, "P_bytes": info["p_bytes"], "n_fd": info["n_fd"]},
            "paper_context": {"R50_N_L": 329404, "R50_N": 2515, "V100_fdirw_s_per_1000_steps": 0.7,
                              "source": "P:181 Fig.7e, P:262-263 Table 3"},
            "flops_per_step": info["flops_per_step"],
            "roofline": _coarse_roofline(info, ms, args.steps),
            "build_seconds": t_build, "gpu_launches": 3 * args.steps, "clocks": clk.summary(),
            **extra}
    fd.coarse_destroy(ctx)
    print(json.dumps(line), flush=True)


def run_absorb(args):
    """NEXT row N3: the paper's integrated radionuclide-absorption loop (Fig.4) on
    the open R50 model (cfg3o: near field r_p + 5Δh, far-field reservoir V_L^far of Table 1),
    Table 1 kinetics (k = 0.05 /s, c_S^eq = 1, c_L^eq = 1e-5, D_S·A_S/RT), 1 GPU.  A macro
    step = (1) FDiRW liquid step with p_BC·c_far, (2) solid FD, (3) PSO interface exchange,
    (4) Eq.7, (5) kinetics.  Metric: non-far voxels advanced per second."""
    import torch

    import paper_2408_11376_b200 as fd

    name = args.config if args.config != "cfg3" else "cfg3o"
    cfg = fi.config(name, weights=args.weights)
    if not cfg.v_far:
        raise SystemExit("--mode absorb needs an open config (cfg3o)")
    mask = cfg.mask()
    nz, ny, nx = cfg.shape
    T = fi.TABLE1
    params = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=0.0, dt=cfg.dt, radius=cfg.R,
                       n_fd=cfg.n_fd, weights=cfg.weights, v_far=cfg.v_far,
                       flags=fd.F_PBC_RESERVOIR if args.pbc == "reservoir" else 0)
    kin_p = dict(D_S=fi.D_SLOW_SI, k=0.05, c_S_eq=1.0, c_L_eq=1e-5)  # Table 1
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx = fd.build_kernels(params, mask)
    t_build = time.perf_counter() - t
    c0 = np.where(mask == 1, T["c_L0"], np.where(mask == 0, T["c_S0"], 0.0)).astype(np.float32)
    c = torch.from_numpy(c0).cuda()
    M0 = fd.far_init(ctx, c, cfg.c_far0)
    fd.absorb_run(ctx, c, args.warmup, **kin_p)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        kin = fd.absorb_run(ctx, c, args.steps, **kin_p)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    nonfar = int((mask != 2).sum())
    nf = torch.from_numpy(mask != 2).cuda()
    tot = float(c.double()[nf].sum()) + kin[-1, 2] * cfg.v_far
    info = ctx.info
    peak, peak_src = _hbm_peak()
    sup_bytes = info["bytes_per_voxel_update"] * int((mask == 1).sum())
    line = {"metric": "voxel-updates/s (integrated absorption loop, NEXT row N3)", "value": nonfar / (ms * 1e-3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": {"fp32": "f32", "fp16": "f16", "bf16": "bf16", "mx8": "mx8"}[cfg.weights] + "-weights/f32-accum",
            "data": "synthetic",
            "config": {"workload": "N3 absorption loop on %s (open R50 model, Table 1 kinetics)" % name,
                       "non_far_voxels": nonfar, "solid_voxels": int((mask == 0).sum()),
                       "near_field_liquid_voxels": int((mask == 1).sum()), "n_fd": info["n_fd"]},
            "kinetics_last": {"Q_S": kin[-1, 0], "Q_L": kin[-1, 1], "c_far": kin[-1, 2], "c_bar_S": kin[-1, 3],
                              "t_s": (args.warmup + args.steps) * cfg.dt},
            "mass_rel_err": abs(tot - M0) / M0,
            "p_bc": args.pbc,
            "liquid_min": float(c[torch.from_numpy(mask == 1).cuda()].min()),
            "liquid_min_note": "the near-field liquid's minimum after the warm-up + timed steps; with p_bc = rowsum "
                               "(reading A26) truncated-window row sums > 1 make p_BC < 0 at pores and drained pores "
                               "go negative; p_bc = reservoir keeps every value >= 0 (DESIGN §3 A26)",
            "roofline": {"bound": "hbm", "achieved": sup_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": sup_bytes / (ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "note": "the loop's dominant kernel is the liquid superposition: its algorithmic bytes "
                                 "(near-field liquid voxel-updates x (K-1)*b_w+16) over the whole macro-step time",
                         "streamed_GBps": info["weight_bytes"] / (ms * 1e-3) / 1e9,
                         "streamed_note": "stored weights actually read per step (every non-far chunk, incl. the "
                                          "solid targets whose liquid-step rows are zero with D_slow = 0)"},
            "paper_context": {"note": "Fig.7 (P:181): FDiRW fast diffusion 0.7 s (V100) for t = 0.5 s = 1000 steps of "
                                      "the coarse R50 model; 'radionuclide absorption ... 192^3 ... in 10 minutes' (P:14)"},
            "paper_run": {"steps": 1000, "seconds_incl_build": t_build + 1000 * ms * 1e-3},
            "build_seconds": t_build, "clocks": clk.summary()}
    fd.destroy(ctx)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--weights", default=None)
    ap.add_argument("--impl", default="fdirw", choices=["fdirw", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the storage-variant measurements")
    ap.add_argument("--no-checks", action="store_true", help="skip the oracle fidelity checks")
    ap.add_argument("--no-scaling-384", action="store_true", help="skip the cfg4 384³ strong-scaling step")
    ap.add_argument("--no-kgen-median", action="store_true", help="time one build instead of the median of 3")
    ap.add_argument("--no-bulk-stream", action="store_true",
                    help="A/B: per-thread weight loads instead of the TMA-staged stream (same bits)")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--mode", default="fine", choices=["fine", "coarse", "absorb"],
                    help="fine: the north_star windowed step (default); coarse: NEXT row N1")
    ap.add_argument("--block", type=int, default=5)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 halo: p2p = edge planes stored into the neighbours' memory by the superposition "
                         "(default); nccl = grouped ncclSend/Recv overlapped with the interior tiles")
    ap.add_argument("--pbc", default="reservoir", choices=["rowsum", "reservoir"],
                    help="--mode absorb: p_BC reading — the reservoir's held-Dirichlet FD (default here: every "
                         "concentration stays >= 0) or the library default, A26's 1 - row sum (DESIGN §3 A26)")
    ap.add_argument("--storage", default="dense", choices=["dense", "dedup"],
                    help="dense: north_star gather layout (default); dedup: NEXT row N4 uniform-chunk kernels")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "coarse":
        return run_coarse(args)
    if args.mode == "absorb":
        return run_absorb(args)

    import dataclasses

    import torch
    import torch.distributed as dist

    import paper_2408_11376_b200 as fd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: FDIRW_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 with a gloo process group
    # (exercises the N>1 orchestration on a one-GPU box; P2P transport only — NCCL refuses
    # two ranks on one device).  Never set by the driver.
    one_dev = os.environ.get("FDIRW_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    if world != args.gpus:
        raise SystemExit("--gpus %d but WORLD_SIZE %d (launch N>1 with torch.distributed.run)" % (args.gpus, world))
    torch.cuda.set_device(local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            if one_dev:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    def allreduce(v, op=dist.ReduceOp.SUM):  # scalar fp64 across ranks
        t_ = torch.tensor([v], dtype=torch.float64, device="cpu" if one_dev else "cuda")
        dist.all_reduce(t_, op=op)
        return float(t_.item())

    def new_id():  # a fresh ncclUniqueId per communicator (collective: every rank, same order)
        obj = [fd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def build_sharded(params, mask, z0, z1, tr):
        """This rank's slab context.  NCCL: the build opens the communicator (collective).  P2P:
        build, all-gather the CUDA IPC blobs, open the neighbours' buffers, then the communicator
        fdirw_mass reduces over; every stage agrees across ranks before the next collective, so a
        failure anywhere returns None on all ranks (the caller falls back to NCCL) instead of
        leaving some of them blocked."""
        if world == 1:
            return fd.build_kernels(params, mask, device=local, stream=stream)
        if tr == "nccl":
            return fd.build_kernels(params, mask, rank=rank, world=world, z_begin=z0, z_end=z1, device=local,
                                    nccl_id=new_id(), stream=stream, transport=tr)
        cx, blob, err = None, None, None
        try:
            cx = fd.build_kernels(params, mask, rank=rank, world=world, z_begin=z0, z_end=z1, device=local,
                                  stream=stream, transport=tr)
            blob = fd.p2p_export(cx)
        except fd.FdirwError as e:
            err = str(e)
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        if all(b is not None for b in blobs):
            try:
                fd.p2p_attach(cx, blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
            except fd.FdirwError as e:
                err = str(e)
        if allreduce(1.0 if err or any(b is None for b in blobs) else 0.0, dist.ReduceOp.MAX) > 0:
            if cx is not None:
                fd.destroy(cx)
            barrier()
            return None
        if not one_dev:  # (NCCL refuses two ranks on one device)
            cid = new_id()
            try:
                fd.comm_init(cx, cid)
            except fd.FdirwError as e:
                err = str(e)
            if allreduce(1.0 if err else 0.0, dist.ReduceOp.MAX) > 0:
                fd.destroy(cx)
                barrier()
                return None
        barrier()
        return cx

    def gmass(cx, cc):  # whole-grid Σ (P2P on one device has no communicator: gloo sums slabs)
        if one_dev and world > 1:
            return allreduce(fd.mass_local(cx, cc))
        return fd.mass(cx, cc)

    def build_with_fallback(params, mask, z0, z1, tr):
        cx, note = build_sharded(params, mask, z0, z1, tr), None
        if cx is None:
            tr, note = "nccl", "P2P setup failed on some rank; fell back to NCCL"
            cx = build_sharded(params, mask, z0, z1, tr)
        return cx, tr, note

    def timed(cx, c, steps, sampler=None):
        """K steps through fdirw_run between barriers + synchronize; device ms, max over ranks."""
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        fd.run(cx, c, steps, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1)
        return allreduce(ms, dist.ReduceOp.MAX) if world > 1 else ms

    cfg = fi.config(args.config, weights=args.weights)
    mask = cfg.mask()
    nz, ny, nx = cfg.shape
    z0, z1 = fd.slabs(nz, world)[rank]
    params = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                       radius=cfg.R, n_fd=cfg.n_fd, weights=cfg.weights, v_far=cfg.v_far,
                       flags=(fd.F_DEDUP_STORAGE if args.storage == "dedup" else 0) |
                             (fd.F_NO_BULK_STREAM if args.no_bulk_stream else 0))
    transport = args.transport if (world > 1 and cfg.v_far == 0) else "nccl"  # P2P: closed domain only

    # one tiny build first: CUDA lazy module loading of the library's kernels is a per-process
    # cost, not kgen's; the timed build below then measures a1-a4 themselves
    warm = fd.Params(nx=16, ny=16, nz=16, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                     radius=cfg.R, n_fd=cfg.n_fd, weights=cfg.weights, v_far=0.0)
    fd.destroy(fd.build_kernels(warm, fi.config("cfg1").mask(), device=local, stream=stream))
    # kgen is reported as the median of 3 builds: two extra full builds on one GPU
    # (each destroyed before the next), then the measured build that the steps use
    extra_builds = []
    if world == 1 and not args.no_kgen_median:
        for _ in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            cx = fd.build_kernels(params, mask, device=local, stream=stream)
            extra_builds.append((time.perf_counter() - t, cx.info["kgen_kernel_ms"]))
            fd.destroy(cx)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx, transport, p2p_note = build_with_fallback(params, mask, z0, z1, transport)
    t_kgen = time.perf_counter() - t
    info = ctx.info
    if extra_builds:
        walls = sorted([w for w, _ in extra_builds] + [t_kgen])
        kms = sorted([k for _, k in extra_builds] + [info["kgen_kernel_ms"]])
        t_kgen = walls[1]
        info = dict(info, kgen_kernel_ms=kms[1], _median3=True)

    c0 = fi.initial_c(mask, "paper") * (mask != 2)  # far-field voxels carry the scalar c_far (N2)
    c_host = torch.from_numpy(np.ascontiguousarray(c0[z0:z1])).pin_memory()
    c = c_host.to("cuda", non_blocking=True)
    far = cfg.v_far > 0
    if far:
        total0 = fd.far_init(ctx, c, cfg.c_far0, stream)  # Eq.7's Σc_{S+L}(t0)
    m0 = gmass(ctx, c)
    fd.run(ctx, c, args.warmup, stream)
    torch.cuda.synchronize()
    if transport == "p2p":  # a wait that timed out (never expected) → rebuild on NCCL
        if allreduce(1.0 if fd.p2p_check(ctx) else 0.0, dist.ReduceOp.MAX) > 0:
            fd.destroy(ctx)
            transport, p2p_note = "nccl", "P2P neighbour wait timed out during warm-up; fell back to NCCL"
            ctx = build_sharded(params, mask, z0, z1, transport)
            c.copy_(c_host.to("cuda"))
            m0 = gmass(ctx, c)
            fd.run(ctx, c, args.warmup, stream)
            torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        t_ms = timed(ctx, c, args.steps)
    m1 = gmass(ctx, c)
    cf1 = fd.far_get(ctx, stream) if far else None
    if world > 1:
        t_kgen = allreduce(t_kgen, dist.ReduceOp.MAX)
    checks = world == 1 and rank == 0 and not args.no_checks and not far and cfg.name == "cfg3"
    last = None
    if checks:  # the timed run's last step, re-done by the oracle below from the field before it
        prev = c.cpu().numpy()
        fd.run(ctx, c, 1, stream)
        last = (prev, c.cpu().numpy())

    # per-phase device times (tracing): 20 eager steps with CUDA events between the
    # phases, max over ranks per phase
    phases = None
    try:
        ph = fd.profile_phases(ctx, c.clone(), 20, stream)
        phases = {k: (allreduce(v, dist.ReduceOp.MAX) if world > 1 else v) for k, v in ph.items()}
        phases["note"] = ("fdirw_profile_phases: mean device ms per step of each phase over 20 eager steps "
                          "(no CUDA graph), max over ranks; halo = P2P neighbour wait / NCCL exchange (comm "
                          "stream), interior = the superposition (P2P: all tiles, boundary bands first), boundary "
                          "= NCCL boundary bands, tail = P2P signal / Eq.7")
    except fd.FdirwError as e:  # the same on every rank (a property of the configuration)
        phases = {"unavailable": str(e)}

    # e2e through the public API with HOST buffers (fdirw_step_host): a dependent chain — step
    # k's input is step k−1's result, read back to pinned host memory every step; each step
    # copies its input H2D, steps, copies its result D2H (nothing overlaps across the chain)
    hbuf = [c_host.clone().pin_memory(), torch.empty_like(c_host).pin_memory()]
    fd.step_host(ctx, hbuf[0], hbuf[1], stream)  # allocates the staging slabs
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(args.e2e_steps):
        fd.step_host(ctx, hbuf[k % 2], hbuf[(k + 1) % 2], stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e_ms = e0.elapsed_time(e1)
    if world > 1:
        e_ms = allreduce(e_ms, dist.ReduceOp.MAX)

    # voxel-updates: every target whose C the step computes (far-field voxels, N2, hold the
    # scalar c_far instead and are not counted)
    N = int((mask != 2).sum())
    n_slab = int((mask[z0:z1] != 2).sum())
    ms_step = t_ms / args.steps
    value = N * args.steps / (t_ms * 1e-3)
    e2e_value = N * args.e2e_steps / (e_ms * 1e-3)
    bpv = info["bytes_per_voxel_update"]
    if cfg.weights == "mx8":  # 9/8 B per weight (the C-ABI field is rounded to an integer)
        bpv = (cfg.K - 1) * 1.125 + 16
    dedup_storage = bool(params.flags & fd.F_DEDUP_STORAGE)
    f_u = info["uniform_chunks"] / max(info["chunks"], 1)
    if dedup_storage:  # N4 byte model: uniform chunks' weights come from an L2-resident table
        bw = {"fp32": 4, "mx8": 1.125}.get(cfg.weights, 2)
        bpv = (1.0 - f_u) * (info["K"] - 1) * bw + 16
    per_launch_bytes = bpv * n_slab
    peak, peak_src = _hbm_peak()
    # N=1: one superpose launch; N>1 P2P: wait + one superpose launch + signal; NCCL: interior
    # + boundary-bands superpose launches (NCCL's own kernels are not counted)
    launches_per_step = 1 if world == 1 else (3 if transport == "p2p" else 2)
    if far:  # N2: + per-tile sums (tile_mass, when compacted) + the Eq.7 reduction
        launches_per_step += 2 if world == 1 else 1
    # one superpose launch per step at N=1 (+1 pack, +1 unpack per fdirw_run); the launch
    # duration is the timed region / K to within the two ~10 µs state kernels.
    achieved = per_launch_bytes / (ms_step * 1e-3) / 1e9
    n_src_planes = min(nz, z1 + cfg.R) - max(0, z0 - cfg.R)
    kgen_cells = nx * ny * n_src_planes * cfg.K * info["n_fd"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong",  # the same 192³ (cfg) problem split over N GPUs
        "vs_baseline": None, "dtype": {"fp32": "f32", "fp16": "f16", "bf16": "bf16", "mx8": "mx8"}[cfg.weights] + "-weights/f32-accum",
        "data": "synthetic",
        "config": {"workload": _workload_name(cfg), "voxels": N, "parallelism": "z-slab x%d" % world,
                   "transport": transport if world > 1 else None,
                   "l2": ("inputs larger than L2 (%.1f GB of weights streamed per step)" %
                          (info["weight_bytes"] * world / 1e9) if info["weight_bytes"] > 126e6 else
                          "weights (%.1f MB) fit in the 126 MB L2 and stay resident: not an HBM measurement"
                          % (info["weight_bytes"] / 1e6))},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": ("superpose_mx8_mixed_kernel (MX8 rows + uniform blocks)" if cfg.weights == "mx8" and dedup_storage else
                                "superpose_mx8_kernel (TMA-staged MX8 rows)" if cfg.weights == "mx8" else
                                "superpose_bulk_kernel (TMA-staged weights)" if info["n_tiles"] >= 2 * 148
                                else "superpose_kernel (register prefetch)"),
                     "peak_source": peak_src, "bytes_per_voxel_update": bpv,
                     "note": ("N4 byte model: (1-f_uniform)*(K-1)*b_w+16 per voxel-update, f_uniform=%.4f"
                              % f_u if dedup_storage else
                              "algorithmic bytes (K-1)*b_w+16 per voxel-update x voxels / step time (per rank)")},
        "storage": "dedup (NEXT row N4)" if dedup_storage else "dense",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(c.numel() * 4 * world),
                "d2h_bytes_per_step": int(c.numel() * 4 * world), "steps": args.e2e_steps,
                "api": "fdirw_step_host (C-ABI, host buffers): a dependent chain, step k's input = step k-1's "
                       "result read back to pinned host memory; per step H2D of the slab, the step, D2H of the "
                       "result, serialised"},
        "gpu_launches": (args.steps * launches_per_step + 2) * world,
        "phases_ms": phases,
        "paper_run": {"steps": 1000, "physical_time_s": 1000 * cfg.dt if cfg.dh != 1.0 else None,
                      "seconds_incl_kgen": t_kgen + 1000 * ms_step * 1e-3,
                      "note": "t = 0.5 s of Fig.7 (1000 macro steps) incl. the one-time kernel build"},
        "kgen": _kgen_line(t_kgen, kgen_cells * world, info, cfg, world),
        "mass_rel_err": (abs(m1 + cf1 * cfg.v_far - total0) / total0 if far
                         else (abs(m1 - m0) / abs(m0) if m0 else None)),
        "clocks": clk.summary(),
    }
    if p2p_note:
        line["config"]["transport_note"] = p2p_note
    if world == 1:
        # the practical ceiling of a read-only stream on this box, measured now over the same
        # weight buffer (fdirw_read_ceiling): the kernel reads ~99.9 % of its bytes, the copy peak
        # above moves half of them as writes
        rc = fd.read_ceiling(ctx, 5, stream)
        line["roofline"]["read_ceiling"] = {"GBps": rc, "frac": achieved / rc,
                                            "how": "fdirw_read_ceiling: 128-bit evict-first grid-stride read of "
                                                   "the stored weights, best of 5, CUDA events"}
    tr = _ncu_traffic(cfg, per_launch_bytes) if (world == 1 and not dedup_storage) else None
    if tr:
        line["roofline"]["traffic"] = tr[0]
        line["roofline"]["traffic_source"] = tr[1] + " (ncu --set full, one launch)"

    fid = Fidelity(cfg, mask) if checks else None
    hist = {} if checks else None
    g1 = None
    if checks:
        g1 = _one_step_field(fd, torch, ctx, mask, stream)
        hist[cfg.weights] = fd.export_kernels(ctx, HIST_SOURCES)
    fd.destroy(ctx)
    del c

    if world == 1 and not dedup_storage and not far and not args.no_variants and params.weights != "mx8":
        line["variants"] = {}
        if params.weights == "bf16":  # the paper's storage format, same bytes
            v = _variant(fd, torch, dataclasses.replace(params, weights="fp16"), mask, c_host, args, stream, peak,
                         fid, hist, "fp16")
            v["note"] = "fp16 weights (the paper's P storage format, P:157): same bytes as bf16, 3 more mantissa bits"
            line["variants"]["fp16_weights"] = v
        v = _variant(fd, torch, dataclasses.replace(params, flags=params.flags | fd.F_DEDUP_STORAGE), mask, c_host,
                     args, stream, peak, fid)
        v["note"] = "uniform chunks read a shared class kernel (smem) instead of streaming; bitwise = dense"
        line["variants"]["N4_dedup_storage"] = v
        v = _variant(fd, torch, dataclasses.replace(params, weights="mx8"), mask, c_host, args, stream, peak, fid,
                     hist, "mx8")
        v["note"] = "superpose_mx8_kernel (TMA-staged rows, byte-permute decode); accuracy: tests/test_gpu_mx8.py"
        line["variants"]["mx8_weights"] = v
        v = _variant(fd, torch, dataclasses.replace(params, weights="mx8", flags=params.flags | fd.F_DEDUP_STORAGE),
                     mask, c_host, args, stream, peak)
        if "unavailable" not in v:
            v["note"] = "MX8 weights + N4 storage: superpose_mx8_mixed_kernel (DESIGN §15)"
        line["variants"]["mx8_dedup_storage"] = v

    if checks:  # accuracy of the timed configuration, driver-visible (oracle leg)
        t = time.perf_counter()
        fid_out = {"relL2_one_step_vs_oracle": fid.step_boxes(g1),
                   "relL2_timed_run_last_step": fid.last_step(*last),
                   "boxes": {k: "x[%d,%d) y[%d,%d) z[%d,%d)" % b for k, b in FID_BOXES.items()},
                   "bar": "north_star: relL2 <= 5e-3 (fp16/bf16 weights), mass <= 1e-6",
                   "note": "one step from the paper initial field on each box vs oracle.step_box (fp64, unquantised "
                           "kernels); timed_run_last_step: the last of the timed run's steps re-done by the oracle "
                           "from the field before it (interface box)"}
        trunc = _truncation(fd, torch, stream)
        cb = FID_BOXES["corner"]
        trunc["cfg3_corner"] = {"box": trunc["cfg3_corner"]["box"],
                                "relL2_vs_whole_grid_fd": _rel(g1[_sl(cb)], trunc["cfg3_corner"]["fd_sub"]),
                                "fd_change_relL2": _rel(trunc["cfg3_corner"]["fd_sub"], c0[_sl(cb)]),
                                "note": "FDiRW (R5 window, n_fd=1000: sigma = 14 voxels) vs 1000 whole-grid FD "
                                        "substeps; the uniform liquid corner is stationary under FD"}
        trunc["note"] = ("the windowed method's own error (SURVEY §0, a diagnostic, not a gate): reflecting R-window "
                         "kernels truncate the n_fd = 1000 diffusion (reading A2)")
        fid_out["truncation"] = trunc
        fid_out["weight_histogram"] = fid.histogram(hist)
        fid_out["seconds"] = fid.seconds + time.perf_counter() - t
        line["fidelity"] = fid_out

    if cfg.name == "cfg3" and not far and not args.no_scaling_384 and not dedup_storage:
        line["scaling_384"] = _scaling_384(fd, torch, args, world, rank, local, stream, transport, build_with_fallback,
                                           timed, gmass, allreduce, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, mask)
        if cfg.name == "cfg1":
            line["cfg1_seconds"] = _cfg1_seconds(fd, torch, params, cfg, mask, stream)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _scaling_384(fd, torch, args, world, rank, local, stream, transport, build_with_fallback, timed, gmass, allreduce,
                 dist):
    """north_star's scaling target: cfg4 (384³ = 2x2x2 R50 particles, R5, bf16, Table 1) split
    into z-slabs over the N GPUs of this run — the same slab/halo machinery as the headline line,
    on the workload whose T1/(P·T_P) north_star asks for.  At N = 1 it is the whole 150.8 GB
    problem on one GPU (T1)."""
    cfg = fi.config("cfg4")
    mask = cfg.mask()
    nz, ny, nx = cfg.shape
    z0, z1 = fd.slabs(nz, world)[rank]
    params = fd.Params(nx=nx, ny=ny, nz=nz, dh=cfg.dh, D_fast=cfg.D_fast, D_slow=cfg.D_slow, dt=cfg.dt,
                       radius=cfg.R, n_fd=cfg.n_fd, weights=cfg.weights)
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx, tr, note = build_with_fallback(params, mask, z0, z1, transport)
    t_build = time.perf_counter() - t
    try:
        c = torch.from_numpy(np.ascontiguousarray(fi.initial_c(mask, "paper")[z0:z1])).cuda()
        m0 = gmass(ctx, c)
        fd.run(ctx, c, args.warmup, stream)
        steps = max(10, min(args.steps, 50))
        ms = timed(ctx, c, steps) / steps
        m1 = gmass(ctx, c)
        info = ctx.info
    finally:
        fd.destroy(ctx)
    N = int(mask.size)
    bpv = info["bytes_per_voxel_update"]
    peak, _ = _hbm_peak()
    ach = bpv * int(mask[z0:z1].size) / (ms * 1e-3) / 1e9
    out = {"workload": _workload_name(cfg), "n_gpus": world, "transport": tr if world > 1 else None,
           "steps": steps, "ms_per_step": ms, "value": N / (ms * 1e-3), "unit": UNIT,
           "weight_bytes_per_rank": info["weight_bytes"], "build_seconds_max": (
               allreduce(t_build, dist.ReduceOp.MAX) if world > 1 else t_build),
           "roofline_per_rank": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak},
           "mass_rel_err": abs(m1 - m0) / m0, "scaling": "strong (fixed 384^3 over N GPUs)",
           "note": "efficiency T1/(N*T_N) is left to the reader/driver: T1 = this object's ms_per_step at n_gpus = 1"}
    if note:
        out["transport_note"] = note
    return out


if __name__ == "__main__":
    main()
