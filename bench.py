#!/usr/bin/env python
"""Benchmark: row-sharded sketched rSVD on 1..8 B200s (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one full pass of the hot path over the resident input: CountSketch
draw (K1) -> A~ = A S (K2, fused finiteness test) -> Y = A~ Omega ->
q x {shifted CholeskyQR(Y); Z = sum_p A~_p^T Y_p (NCCL); Y = A~ Z} ->
shifted CholeskyQR3 -> ||Q^T Q - I|| check -> B = sum_p Q_p^T A_p (NCCL) ->
fp64 Gram + eigensolver -> U, sigma, V.  Default workload: C5 (BASELINE
configs[4], m = 2^20, n = 2^15, l = 8000, q = 4; A = 128 GiB resident).

value      = device time of one rSVD (ms, max over ranks), inputs resident in HBM.
e2e        = the same through the public API ``paper_2605_09755_b200.rsvd`` with
             the input in pinned host memory (H2D inside the timed region) and
             U, sigma, V copied back (D2H inside).
roofline   = the dominant kernel of the step, measured live with CUDA events.
cpu_baseline / --impl reference = the oracle port (oracle/skp_oracle.py, the
             reference's algorithm on numpy/scipy) on the workload's first
             rows, extrapolated per phase to the full workload; slab_parity
             compares the GPU path with it on that slab.
Inputs (A = 128 GiB at C5, 17 GB at C3) are far larger than the 126 MB L2,
so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "rSVD time/sketch HBM GB/s/power-iter TFLOP/s vs roofline at 1/2/4/8 B200"

# BASELINE.json configs (C4 = Nystrom; C5 needs one full GPU of HBM at l=8000)
CONFIGS = {
    "C1": dict(m=2000, n=1000, l=200, s=8, k=20, r2=30, q=2, dtype="f64", gen="c1"),
    "C2": dict(m=20000, n=10000, l=2000, s=8, k=100, r2=110, q=3, dtype="f32", gen="c2"),
    "C3": dict(m=262144, n=16384, l=4000, s=8, k=500, r2=520, q=3, dtype="f32", gen="c3"),
    # psd Nystrom of the RBF kernel (BASELINE configs[3]; n x n fp32 = 17.2 GB, r2 = k assumed)
    "C4": dict(m=65536, n=65536, l=4096, s=8, k=256, r2=256, q=2, dtype="f32", gen="c4", seed=4,
               nystrom=True),
    # the headline: the largest config that fits one B200 (BASELINE configs[4], l = 8000, q = 4)
    "C5": dict(m=1048576, n=32768, l=8000, s=8, k=1000, r2=1050, q=4, dtype="f32", gen="c5",
               seed=5),
}


_SM_MAX_MHZ = 1965.0


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), \
            d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except Exception:
                self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7
                          for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------ inputs --
def make_input(cfg, row0, rows, device):
    import torch
    from paper_2605_09755_b200 import datagen
    from paper_2605_09755_b200 import _ops
    g = cfg["gen"]
    if g in ("c1", "c2"):
        # host-generated: into 128-byte rows, as the public upload lays it out
        h = (datagen.c1_matrix(1) if g == "c1" else datagen.c2_matrix(2))[row0:row0 + rows]
        t = _ops.empty2d(h.shape[0], h.shape[1], torch.from_numpy(h[:1]).dtype, device)
        t.copy_(torch.from_numpy(h))
        return t
    if g == "c3":
        return datagen.c3_matrix_gpu(3, cfg["m"], cfg["n"], device=device, row0=row0, rows=rows)
    if g == "c5":
        return datagen.c5_matrix_gpu(5, cfg["m"], cfg["n"], device=device, row0=row0, rows=rows)
    raise ValueError(g)


def spec_of(cfg, seed):
    from paper_2605_09755_b200 import RangeFinderSpec
    return RangeFinderSpec(k=cfg["k"], l=cfg["l"], r1=cfg["l"], r2=cfg["r2"], q=cfg["q"], eps=0.5,
                           sketch_kind="countsketch", seed=seed, s=cfg["s"])


def flops_of(cfg):
    m, n, l, r2, q = cfg["m"], cfg["n"], cfg["l"], cfg["r2"], cfg["q"]
    power = (1 + 2 * q) * 2.0 * m * l * r2
    orth = (q + 1) * 2 * (2.0 * m * r2 * r2 + 2.0 * m * r2 * r2)   # 2 passes x (Gram + Y R^-1)
    qta = 2.0 * m * n * r2
    return power, orth, qta


# ---------------------------------------------------------- CPU baseline ----
def workload_slab(cfg, rows: int):
    """The first ``rows`` rows of the workload's own matrix (same generator,
    spectrum and noise as the timed run), as float32/float64 numpy."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    t = make_input(cfg, 0, min(rows, cfg["m"]), dev)
    out = t.cpu().numpy()
    del t
    torch.cuda.empty_cache()
    return out


def cpu_baseline(cfg, sample_rows: int, reps: int = 1, slab=None):
    """Oracle port on a row slab of the workload; phases extrapolated linearly
    in m (except those independent of m: the sketch draw, Omega, the SVD of
    the r2 x n matrix B).  Returns (ms for the full workload, details, Q)."""
    from oracle import skp_oracle as o
    m, n = cfg["m"], cfg["n"]
    a = workload_slab(cfg, sample_rows) if slab is None else slab
    rows = a.shape[0]
    spec = o.Spec(k=cfg["k"], l=cfg["l"], r1=cfg["l"], r2=cfg["r2"], q=cfg["q"],
                  seed=cfg.get("seed", 3), s=cfg["s"])
    best = None
    qb = None
    for _ in range(reps):
        t = {}
        qb = o.range_finder_sketched(a, spec, timings=t)
        t0 = time.perf_counter()
        b = qb.T @ a.astype(np.float64)
        t["qta"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        o.thin_svd(b)
        t["svd"] = time.perf_counter() - t0
        best = t if best is None or sum(t.values()) < sum(best.values()) else best
    scale = m / rows
    linear = ("cast", "apply_right", "power", "orth", "qta")
    full = sum(v * (scale if k in linear else 1.0) for k, v in best.items())
    return full * 1e3, {"phases_s_sample": {k: round(v, 4) for k, v in best.items()},
                        "rows_sampled": rows, "extrapolated_to_m": m,
                        "q_columns_kept": int(qb.shape[1]), "host": host_info()}, (a, qb, spec)


def slab_parity(cfg, a, qb, spec_o):
    """The GPU path (rsvd, as timed) against the oracle on the same slab:
    max relative sigma difference over the top k, and both rel_err values."""
    import torch
    import paper_2605_09755_b200 as skp
    from oracle import skp_oracle as o
    _, so, _ = o.randsvd(a, qb)
    eo = o.proj_rel_error(a, qb)
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = spec_of(cfg, spec_o.seed)
    res, rel = skp.rsvd(torch.from_numpy(a).to(dev), spec, with_error=True)
    k = cfg["k"]
    sg = res.sigma.double().cpu().numpy()
    return {"rows": int(a.shape[0]), "k": k,
            "sigma_max_rel_diff": float(np.max(np.abs(sg[:k] - so[:k]) / so[:k])),
            "sigma_1": [float(sg[0]), float(so[0])],
            "sigma_k": [float(sg[k - 1]), float(so[k - 1])],
            "rel_err": [float(rel), float(eo)],
            "rel_err_rel_diff": float(abs(rel - eo) / eo) if eo > 0 else 0.0,
            "tolerance": {"sigma": 1e-5, "rel_err": 1e-3}}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def host_info() -> dict:
    """The CPU baseline's host: cores, model and the
    numpy / scipy / BLAS the oracle port runs on."""
    import platform
    import scipy
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}".strip()
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": host_threads(), "cpu_model": model,
            "numpy": np.__version__, "scipy": scipy.__version__, "blas": blas}


# --------------------------------------------------------------- the arm ----
_TRAFFIC_WORLD = [1]


def _traffic(config: str, key: str):
    """DRAM bytes per launch of a kernel at a config, from the committed ncu
    --set full capture (profiles/traffic.json, scripts/summarize_ncu.py) --
    single-GPU captures, so only for 1-rank runs."""
    if _TRAFFIC_WORLD[0] != 1:
        return None, None
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as fh:
            tr = json.load(fh)
    except (OSError, ValueError):
        return None, None
    t = tr.get(config, {}).get(key)
    if t is None:
        return None, None
    return t["bytes_per_launch"], "profiles/traffic.json <- " + t["source"]


def _time_launches(fn, reps: int = 5) -> float:
    """Average ms per call of fn on the current stream (CUDA events, warm)."""
    import torch
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2605_09755_b200 as skp
    from paper_2605_09755_b200 import _lib, _ops, distributed as D, power as skp_power
    from paper_2605_09755_b200.sketching import make_sketch, substream

    device = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(device)
    comm = D.TorchComm() if world > 1 else _LocalComm()
    # the committed ncu captures are 1-rank runs of the configs as listed
    _TRAFFIC_WORLD[0] = world if (args.l is None and args.q is None) else 0
    m, n = cfg["m"], cfg["n"]
    row0, rows = D.shard_rows(m, world, rank)
    a = make_input(cfg, row0, rows, device)
    torch.cuda.synchronize()
    spec = spec_of(cfg, seed=cfg.get("seed", 3))

    def barrier():
        if world > 1:
            dist.barrier()

    def step(timings=None, with_error=False):
        # the timed step is the rSVD (range finder + randsvd, with the
        # reference's orthonormality check) as the reference times it; the
        # quality number ||A - QQ^T A|| / ||A|| is evaluated once after the
        # timed loop (it needs ||A||_F, fused into the sketch)
        return D.rsvd_sharded(a, spec, m, comm, timings, with_error=with_error)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = _lib.load().skp_launch_count()
    clk = ClockSampler(device.index)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    phases = {}
    t_start.record()
    for _ in range(args.steps):
        _, sig, _, _ = step(phases)
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    launches = _lib.load().skp_launch_count() - launches0
    _, sig, _, rel = step(None, with_error=True)   # quality check, outside the timed region
    ms = t_start.elapsed_time(t_end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    phases = {k: v / args.steps for k, v in phases.items()}

    # ---- dominant-kernel measurements (live, CUDA events on this stream) ----
    hbm, bf16, bf16_sus, peak_src = load_peaks()
    l, r2, s_ = cfg["l"], cfg["r2"], cfg["s"]
    sk = make_sketch("countsketch", n, l, substream(spec.seed, 0), s=s_, device=device)
    be = _ops.CudaBackend(device, a.dtype)
    # A~ does not fit beside A (C5 at l = 16000 on one GPU): the step ran the
    # blocked range finder (A~ formed twice in row blocks); its kernels are
    # timed here on a row slab and scaled to the step by rows / krows
    blocked = skp_power._atil_blocked(a, spec, be, sk)
    krows = min(rows, 131072) if blocked else rows
    kscale = rows / krows
    ak = a[:krows]
    atil = _ops.empty2d(krows, l, a.dtype, device)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=device)
    # the kernel the range finder runs: K2 v2 (row gather) when it applies, else v1
    v2 = sk.right_permuted(ak, out=atil, nonfinite=nonfinite) is not None

    def run_sketch():   # as in the timed step: the non-finite test, no ||A||_F pass
        if v2:
            sk.right_permuted(ak, out=atil, nonfinite=nonfinite)
        else:
            sk.right(ak, out=atil, nonfinite=nonfinite)
    sketch_ms = _time_launches(run_sketch)
    esz = a.element_size()
    sketch_bytes = krows * n * esz + krows * l * esz + n * s_ * 5 + (l + 1) * 4
    sketch_gbs = sketch_bytes / (sketch_ms * 1e-3) / 1e9
    # ---- the tensor-core kernels of the step, each timed live as the step runs
    # it (operands laid out as in the pipeline: 128-byte padded rows)
    pa = be.prepare(atil, inplace=True)                 # A~ planes (A~ is not reused)
    h3 = isinstance(pa, _ops.SplitH2)
    z = _ops.empty2d(l, r2, a.dtype, device)
    z.normal_()
    omega_like = _ops.empty2d(l, r2, a.dtype, device)
    omega_like.normal_()
    gram_path = h3 and (blocked or be.gram_ok(pa, omega_like, cfg["q"]))
    del omega_like
    tc = bool(_lib.load().skp_has_tcgen05())
    f32 = cfg["dtype"] == "f32"
    kern = {}
    if h3:
        sz = _ops.split_h2(z, trans=True)
        y = _ops.empty2d(krows, r2, a.dtype, device)
        pg_ms = _time_launches(lambda: _ops.gemm_h3(pa, sz, out=y))
        del y
    else:
        y = _ops.empty2d(krows, r2, a.dtype, device)
        pg_ms = _time_launches(lambda: _ops.gemm(atil, z, out=y))
        del y
    kern["power_gemm"] = dict(
        kernel="gemm_h3 Y = A~ W (tcgen05 3xFP16, pre-split A~)" if h3 else "gemm Y = A~ Z",
        ms=pg_ms, flop=2.0 * krows * l * r2, launches=kscale if gram_path else (1 + 2 * cfg["q"]) * kscale,
        key="gemm_h3_nn")
    if gram_path:
        g_ms = _time_launches(lambda: _ops.syrk_h3(pa), reps=3)
        kern["syrk"] = dict(kernel="syrk_h3 G = A~^T A~ (tcgen05 3xFP16, lower-triangle 256x256 "
                                   "tiles, both operands MN-major)",
                            ms=g_ms, flop=1.0 * krows * l * (l + 1), launches=kscale, key="syrk")
    del pa, z, atil, ak        # (ak is a view of a: e2e below frees a)
    torch.cuda.empty_cache()
    # randsvd's B^T = A^T Q with the in-kernel split of A (Q as fp16 planes of Q^T)
    if h3 and tc and f32:
        qp = _ops.empty2d(rows, r2, a.dtype, device)
        qp.normal_()
        qp /= float(np.sqrt(rows))
        sq = _ops.split_h2(qp, trans=True)
        del qp
        e_a = _ops.h2_exponent(a)
        q_ms = _time_launches(lambda: _ops.gemm_h3s_t(a, e_a, sq), reps=2)
        del sq
        kern["qta"] = dict(kernel="gemm_h3s B^T = A^T Q (tcgen05 3xFP16, A split in the kernel)",
                           ms=q_ms, flop=2.0 * rows * n * r2, launches=1, key="gemm_h3s_qta")
        torch.cuda.empty_cache()
    pipe_peak = bf16 if (h3 or not f32) else bf16 / 2.0
    mma_per_mac = 3 if (tc and f32) else 1
    kernels = {}
    for name, kd in kern.items():
        tflops = kd["flop"] / (kd["ms"] * 1e-3) / 1e12
        tr, src = _traffic(args.config, kd["key"])
        kernels[name] = {
            "kernel": kd["kernel"], "bound": "tensor", "ms_per_launch": round(kd["ms"], 4),
            "launches_per_step": round(kd["launches"], 3),
            "share_of_step": round(kd["ms"] * kd["launches"] / ms, 3),
            "algorithmic_flop_per_launch": kd["flop"], "achieved": round(tflops, 2),
            "peak": round(bf16, 1), "unit": "TFLOP/s", "frac": round(tflops / bf16, 4),
            "emulation": {"mma_per_mac": mma_per_mac,
                          "pipe_tflops": round(tflops * mma_per_mac, 2),
                          "pipe_peak": round(pipe_peak, 1),
                          "pipe_frac": round(tflops * mma_per_mac / pipe_peak, 4),
                          "pipe_peak_sustained": round(bf16_sus if pipe_peak == bf16 else bf16_sus / 2, 1),
                          "pipe_frac_sustained": round(
                              tflops * mma_per_mac / (bf16_sus if pipe_peak == bf16 else bf16_sus / 2), 4)},
            "traffic": tr, "traffic_unit": "DRAM bytes per launch (ncu --set full)",
            "traffic_source": src}
    skey = "sketch_gather" if v2 else "sketch_rows"
    s_tr, s_src = _traffic(args.config, skey)
    # K2's real bound is on chip: shared-memory wavefronts (profiles/
    # r02_smem_gather_ceiling.txt: 0.957 per clock per SM, 8.8e12 gathered
    # entries/s at 1.95 GHz).  Work = the m n s gathered entries plus the row
    # ingest into each of the P slice CTAs (P n words per row), in entry units
    P_sl = -(-l // (896 - 96))
    if v2:  # the plan's slice count (even where K2 v3 applies)
        P_sl = int(_lib.load().skp_sketch_gather_plan_fail_offset(l)) // (896 * 4)
    # K2 v3: one row copy feeds two slices (fp32, even slice count, column passes <= 16384 words)
    n_pass = -(-n // 24576)
    v3 = v2 and P_sl % 2 == 0 and -(-n // n_pass) <= 16384
    copies = P_sl // 2 if v3 else P_sl
    onchip_work = krows * (n * s_ + copies * n)
    onchip_ceiling = 148 * 32 * 0.957 * _SM_MAX_MHZ * 1e6
    onchip = {"work_entries": onchip_work, "slices": P_sl, "row_copies": copies,
              "achieved_entries_per_s": round(onchip_work / (sketch_ms * 1e-3), 1),
              "ceiling_entries_per_s": round(onchip_ceiling, 1),
              "frac_onchip": round(onchip_work / (sketch_ms * 1e-3) / onchip_ceiling, 4),
              "ceiling_source": "profiles/r02_smem_gather_ceiling.txt (scripts/micro/smem_gather.cu)"}
    kernels["sketch"] = {
        "kernel": ("sketch_gather_pair (K2 v3, two slices per CTA; one launch here = one call: its column passes x row chunks)" if v3 else "sketch_gather (K2 v2)") if v2
        else "sketch_right (K2 v1)", "bound": "hbm",
        "onchip": onchip,
        "ms_per_launch": round(sketch_ms, 4),
        # (blocked: two passes over A, each timed here on krows rows)
        "launches_per_step": round((2 if blocked else 1) * kscale, 3),
        "share_of_step": round(sketch_ms * (2 if blocked else 1) * kscale / ms, 3),
        "algorithmic_bytes_per_launch": sketch_bytes,
        "achieved": round(sketch_gbs, 1), "peak": hbm, "unit": "GB/s",
        "frac": round(sketch_gbs / hbm, 4), "traffic": s_tr,
        "traffic_unit": "DRAM bytes per launch (ncu --set full)", "traffic_source": s_src}
    dom = max(kernels, key=lambda k: kernels[k]["share_of_step"])
    roof = dict(kernels[dom], name=dom,
                peak_note=f"{peak_src}: HBM {hbm} GB/s; dense bf16 {bf16} TFLOP/s burst, "
                          f"{bf16_sus} sustained (3xFP16 runs kind::f16 at that rate, 3 MMAs "
                          "per useful MAC: 'emulation')")
    power_f, orth_f, qta_f = flops_of(cfg)
    power_tflops = (power_f / world) / (phases.get("power", float("nan")) * 1e-3) / 1e12
    extra = {
        "kernels": kernels,
        "power_path": ("blocked: A~ does not fit beside A, formed twice in row blocks (SYRK "
                       "of each block into G, q l-dimensional steps, each block's rows of A~ W; "
                       f"kernels timed on {krows} rows)" if blocked else
                       "sketch space (one SYRK of A~, q l-dimensional steps, one A~ W)"
                       if gram_path else "products (1 + 2q products with A~)"),
        "power_phase_TFLOP/s_equivalent": round(power_tflops, 2),
    }
    # slab of the workload for the CPU baseline / oracle parity (rank 0)
    slab = a[:min(args.cpu_rows, rows)].cpu().numpy() if rank == 0 else None

    # ---- end to end through the public API from pinned host memory ----------
    e2e = None
    e2e_note = None
    holder = [a]
    del a                     # (also unbinds the closures' cell: _e2e can free it)
    if not args.no_e2e:
        e2e, e2e_note = _e2e(args, holder, spec, m, comm, device, world, barrier, D, skp)
    holder.clear()
    torch.cuda.empty_cache()

    if rank != 0:
        return None, None
    line = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": cfg["dtype"] + (" (products 3xFP16 on tcgen05 kind::f16, fp64 small cores)" if h3
                                 else " (3xTF32 tcgen05)" if tc and f32 else ""),
        "data": "synthetic (seeded, BASELINE config recipe; random-init factors, no dataset)",
        "config": workload_config(args.config, cfg, world),
        "phases_ms": {k: round(v, 3) for k, v in phases.items()},
        "rel_err": rel, "sigma_1": float(sig[0].item()),
        "roofline": roof, **extra,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if e2e_note:
        line["e2e_note"] = e2e_note
    return line, slab


def _e2e(args, holder, spec, m, comm, device, world, barrier, D, skp):
    """e2e through the public API: the input in pinned host memory, H2D inside
    the timed region (streamed behind the sketch) and U, sigma, V copied back.
    Also times the reference's own two-call sequence on one device_matrix
    handle (range_finder_sketched + randsvd, one upload)."""
    import torch
    import torch.distributed as dist
    a = holder[0]
    nbytes = a.numel() * a.element_size()
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    if avail is not None and avail < nbytes + (24 << 30):
        return None, f"host RAM {avail >> 30} GiB < input {nbytes >> 30} GiB + 24 GiB margin"
    host = torch.empty(tuple(a.shape), dtype=a.dtype, pin_memory=True)
    host.copy_(a)
    torch.cuda.synchronize()
    # the device copy of A is released first: the public call allocates its own
    del a
    holder.clear()
    torch.cuda.empty_cache()

    def one():
        if world == 1:
            res = skp.rsvd(host, spec)
            return (res.U.numel() * res.U.element_size() + res.V.numel() * res.V.element_size()
                    + res.sigma.numel() * res.sigma.element_size())
        return _e2e_sharded(host, spec, m, comm, device, D)

    for _ in range(max(1, min(args.warmup, 2))):
        one()
    barrier()
    torch.cuda.synchronize()
    k2 = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    out_b = 0
    for _ in range(k2):
        out_b = one()
    torch.cuda.synchronize()
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / k2
    pair_ms = None
    if world == 1:
        # the drop-in pair: device_matrix(host) -> range_finder_sketched -> randsvd
        def pair():
            h = skp.device_matrix(host)
            qb = skp.range_finder_sketched(h, spec)
            return skp.randsvd(h, qb)
        pair()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pair()
        torch.cuda.synchronize()
        pair_ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        t = torch.tensor([e2e_ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": round(e2e_ms, 3), "unit": "ms",
           "h2d_bytes_per_step": int(nbytes), "d2h_bytes_per_step": int(out_b), "steps": k2,
           "api": "paper_2605_09755_b200.rsvd(pinned host tensor)" if world == 1 else
                  "distributed.rsvd_sharded on the rank's pinned slab"}
    if pair_ms is not None:
        e2e["drop_in_pair_ms"] = round(pair_ms, 3)
        e2e["drop_in_pair_api"] = ("device_matrix(host) -> range_finder_sketched -> randsvd "
                                   "(one upload; Q returned to and re-read from the host)")
    del host
    return e2e, None


class _LocalComm:
    rank, world = 0, 1

    def allreduce_(self, t):
        return t


def _e2e_sharded(host, spec, m, comm, device, D):
    a = host.to(device, non_blocking=True)
    u, s, v, _ = D.rsvd_sharded(a, spec, m, comm)
    from paper_2605_09755_b200 import _convert
    u_h, s_h, v_h = (_convert.download(t, "cpu") for t in (u, s, v))   # pinned host results
    return u_h.numel() * 4 + s_h.numel() * 8 + v_h.numel() * 4


REF_MAX_STEPS, REF_MAX_WARMUP = 5, 1

# ------------------------------------------------------------- C4: Nystrom ----
NYS_SUB = 8192     # CPU baseline / slab parity: the leading principal n' x n' submatrix


def c4_points(cfg):
    from paper_2605_09755_b200 import datagen
    x = datagen.rbf_points(cfg["n"], 16, seed=cfg["seed"])
    return x, datagen.rbf_bandwidth(x, 4096, seed=cfg["seed"])


def nystrom_spec(cfg):
    from paper_2605_09755_b200 import RangeFinderSpec
    return RangeFinderSpec(k=cfg["k"], l=cfg["l"], r1=cfg["l"], r2=cfg["r2"], q=cfg["q"], eps=0.5,
                           seed=cfg["seed"], s=cfg["s"])


def nystrom_rel_err_dev(kmat, c, w):
    """||K - C W^+ C^T||_F / ||K||_F on the device (fp64, row blocks)."""
    import torch
    wp = torch.linalg.pinv(w.double(), hermitian=True)
    right = wp @ c.double().T                       # r2 x n
    num = den = 0.0
    for r0 in range(0, kmat.shape[0], 4096):
        kb = kmat[r0:r0 + 4096].double()
        num += float(((kb - c[r0:r0 + 4096].double() @ right) ** 2).sum())
        den += float((kb ** 2).sum())
    return (num / den) ** 0.5


def cpu_baseline_nystrom(cfg, sub=NYS_SUB):
    """The oracle's literal nystrom_core (fp64, as the reference computes) on
    the leading sub x sub principal block of the workload's own K; phases
    extrapolated to n (K S ~ n^2, S^T C~ and C~ Y ~ n, the l-dimensional core
    not scaled).  The reference's O(n^3) psd eigen-check is not timed (ours
    skips it above n = 1024 too)."""
    from paper_2605_09755_b200 import datagen
    from oracle import skp_oracle as o
    x, h = c4_points(cfg)
    xs = x[:sub]
    sq = (xs * xs).sum(1)
    kmat = np.exp(-np.maximum(sq[:, None] + sq[None, :] - 2.0 * xs @ xs.T, 0.0) / (2 * h * h))
    kmat = np.minimum(kmat, kmat.T).astype(np.float32)
    spec = o.Spec(k=cfg["k"], l=cfg["l"], r1=cfg["l"], r2=cfg["r2"], q=cfg["q"],
                  seed=cfg["seed"], s=cfg["s"])
    t = {}
    c, w = o.nystrom_core(kmat, spec, stabilized=False, timings=t)
    f = cfg["n"] / sub
    full = t["apply_right"] * f * f + (t["left_t"] + t["contract"]) * f + t["core"]
    det = {"phases_s_sample": {k: round(v, 4) for k, v in t.items()},
           "sample": f"leading {sub} x {sub} principal block of the {cfg['n']}-point RBF kernel; "
                     f"K S extrapolated x{f * f:g} (n^2), S^T C~ and C~ Y x{f:g} (n), the "
                     "l-dimensional core not scaled; the reference's O(n^3) psd check not timed",
           "host": host_info()}
    del xs
    return full * 1e3, det, (kmat, spec, c, w)


def nystrom_slab_parity(cfg, kmat, spec_o):
    """nystrom_psd (fp32 sketch, fp64 literal core) on the CPU baseline's
    principal block against the oracle's literal core on the same bytes."""
    import torch
    import paper_2605_09755_b200 as skp
    from oracle import skp_oracle as o
    co, wo = o.nystrom_core(kmat, spec_o, stabilized=False)
    eo = o.nystrom_rel_error(kmat, co, wo)
    dev = torch.device("cuda", torch.cuda.current_device())
    kd = torch.from_numpy(kmat).to(dev)
    res = skp.nystrom_psd(kd, nystrom_spec(cfg))
    e = nystrom_rel_err_dev(kd, res.C, res.W)
    # literal on both sides: the same Y up to rounding, so W's leading
    # eigenvalues are comparable
    wg = np.sort(np.linalg.eigvalsh(res.W.double().cpu().numpy()))[::-1]
    wr = np.sort(np.linalg.eigvalsh(wo))[::-1]
    # |d lambda_i| / (1e-5 |lambda_i| + 1e-7 |lambda_1|): <= 1 passes
    dev_w = np.abs(wg - wr) / (1e-5 * np.abs(wr) + 1e-7 * np.abs(wr[0]))
    return {"n": int(kmat.shape[0]), "rel_err": [e, eo], "rel_err_rel_diff": abs(e - eo) / eo,
            "W_eig_max_dev_over_tol": float(dev_w.max()),
            "tolerance": {"rel_err": 1e-3,
                          "W_eig": "|d lambda_i| <= 1e-5 lambda_i + 1e-7 lambda_1 (fp32 sketch)"}}


def run_nystrom(args, cfg, rank, world, local_rank):
    """C4: psd Nystrom (power.py:258-298) of the 65536-point RBF kernel.  A
    step = the device symmetry check (N = 1; the transposed tiles live on
    other ranks at N > 1) + sketch K S (K2 v2) + W~ = S^T C~ (all-reduced) +
    the l-dimensional core + C = C~ Y, with K resident in HBM."""
    import torch
    import torch.distributed as dist
    import paper_2605_09755_b200 as skp
    from paper_2605_09755_b200 import _lib, _ops, datagen, distributed as D, power
    from paper_2605_09755_b200.sketching import make_sketch, substream
    device = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(device)
    comm = D.TorchComm() if world > 1 else _LocalComm()
    n, l, s_ = cfg["n"], cfg["l"], cfg["s"]
    x, h = c4_points(cfg)
    row0, rows = D.shard_rows(n, world, rank)
    kmat = datagen.rbf_kernel_gpu(x, h, device=device, row0=row0, rows=rows)
    spec = nystrom_spec(cfg)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        if world == 1:
            power._check_psd_dev(kmat)
        return D.nystrom_sharded(kmat, spec, row0, n, comm)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = _lib.load().skp_launch_count()
    clk = ClockSampler(device.index)
    clk.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        c, w = step()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    launches = _lib.load().skp_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rel = nystrom_rel_err_dev(kmat, c, w) if world == 1 else None
    hbm, _, _, _ = load_peaks()
    # the dominant kernel: K2 v2 on the rank's rows of K
    sk = make_sketch("countsketch", n, l, substream(spec.seed, 0), s=s_, device=device)
    # as the step runs it: fp32 K, fp64 accumulation and fp64 C~ (power._nystrom_dev)
    ctil = _ops.empty2d(rows, l, torch.float64, device)
    nonfinite = torch.zeros(1, dtype=torch.int64, device=device)
    v2 = sk.right_permuted(kmat, out=ctil, nonfinite=nonfinite,
                           out_dtype=torch.float64) is not None
    run_sketch = (lambda: sk.right_permuted(kmat, out=ctil, nonfinite=nonfinite,
                                            out_dtype=torch.float64)) if v2 else \
        (lambda: sk.right(kmat.double(), out=ctil, nonfinite=nonfinite))
    sk_ms = _time_launches(run_sketch)
    sk_bytes = rows * n * 4 + rows * l * 8 + n * s_ * 5
    sym_ms = _time_launches(lambda: _ops.sym_check(kmat)) if world == 1 else None
    del ctil
    sk_gbs = sk_bytes / (sk_ms * 1e-3) / 1e9
    roof = {"kernel": "sketch_gather (K2 v2, fp64 accumulation) C~ = K S" if v2 else "sketch_right (K2 v1)",
            "bound": "hbm", "achieved": round(sk_gbs, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(sk_gbs / hbm, 4), "traffic": None,
            "traffic_unit": "DRAM bytes per launch (ncu --set full)",
            "ms_per_launch": round(sk_ms, 4), "algorithmic_bytes_per_launch": sk_bytes,
            "share_of_step": round(sk_ms / ms, 3)}
    extra = {}
    if sym_ms is not None:
        sb = n * n * 4
        extra["sym_check"] = {"ms": round(sym_ms, 4), "GB/s": round(sb / (sym_ms * 1e-3) / 1e9, 1),
                              "frac_hbm": round(sb / (sym_ms * 1e-3) / 1e9 / hbm, 4),
                              "bytes": sb, "share_of_step": round(sym_ms / ms, 3)}
    e2e = None
    if world == 1 and not args.no_e2e:
        host = torch.empty(tuple(kmat.shape), dtype=kmat.dtype, pin_memory=True)
        host.copy_(kmat)
        del kmat
        torch.cuda.empty_cache()
        skp.nystrom_psd(host, spec)
        torch.cuda.synchronize()
        k2 = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(k2):
            res = skp.nystrom_psd(host, spec)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / k2
        e2e = {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": n * n * 4,
               "d2h_bytes_per_step": int(res.C.numel() * 4 + res.W.numel() * 4), "steps": k2,
               "api": "paper_2605_09755_b200.nystrom_psd(pinned host tensor)"}
        del host
    if rank != 0:
        return None, None
    line = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 K; sketch accumulated in fp64, core in fp64 (DMMA), as the reference",
        "data": "synthetic (seeded RBF points, BASELINE config recipe)",
        "config": workload_config(args.config, cfg, world), "rbf_bandwidth_h": round(h, 6),
        "nystrom_rel_err": rel, "roofline": roof, "sketch": dict(roof), **extra,
        "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e,
    }
    return line, None



def workload_config(name: str, cfg: dict, world: int) -> dict:
    """The `config` object of both arms (ours and --impl reference): the
    workload's shape and the descriptive keys, identical for the two."""
    if cfg.get("nystrom"):
        return {"workload": name, **{k: cfg[k] for k in ("n", "l", "s", "k", "r2", "q")},
                "parallelism": f"rows of K sharded x{world} (NCCL allreduce of the l x l W~)",
                "l2": "no flush: K (17.2 GB) is far larger than the 126 MB L2"}
    return {"workload": name, **{k: cfg[k] for k in ("m", "n", "l", "s", "k", "r2", "q")},
            "parallelism": f"rows sharded x{world} (NCCL allreduces: the l x l G once or "
                           "l x r2 per power step, r2 x r2 Grams, r2 x n B^T)",
            "l2": "no flush: A is far larger than the 126 MB L2"}


def run_reference(args, cfg):
    """The reference's CPU path (the oracle port) on the workload's first
    rows.  One sample is a full range finder + randsvd on the slab (C5: ~20 s
    on 16 cores, most of it m-independent: the sketch draw and the SVD of the
    r2 x n matrix B), so at most REF_MAX_STEPS samples (+ REF_MAX_WARMUP) are
    timed and the JSON line states the counts actually run."""
    ncores = host_threads()
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, str(ncores))
    if cfg.get("nystrom"):
        return run_reference_nystrom(args, cfg, ncores)
    slab = workload_slab(cfg, args.cpu_rows)
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    warm = min(args.warmup, REF_MAX_WARMUP)
    vals = []
    det = None
    for i in range(warm + steps):
        v, det, _ = cpu_baseline(cfg, args.cpu_rows, slab=slab)
        if i >= warm:
            vals.append(v)
    val = statistics.median(vals)
    return {
        "metric": METRIC, "impl": "reference", "value": round(val, 1), "unit": "ms",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": round(val, 1), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (numpy/scipy, as the reference computes)",
        "data": "synthetic (the workload's own first rows: same generator, spectrum, noise)",
        "config": workload_config(args.config, cfg, args.gpus),
        "cpu_baseline": {"value": round(val, 1), "unit": "ms", "cores": ncores, "kind": "port",
                         "sample": f"rows 0..{det['rows_sampled']} of the {cfg['m']}-row workload, "
                                   f"m-linear phases extrapolated x{cfg['m'] / det['rows_sampled']:g}"
                                   " (sketch draw, Omega, SVD of B not scaled); median of "
                                   f"{steps} samples",
                         **det},
        "e2e": {"value": round(val, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def run_reference_nystrom(args, cfg, ncores):
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    warm = min(args.warmup, REF_MAX_WARMUP)
    vals, det = [], None
    for i in range(warm + steps):
        v, det, _ = cpu_baseline_nystrom(cfg)
        if i >= warm:
            vals.append(v)
    val = statistics.median(vals)
    return {
        "metric": METRIC, "impl": "reference", "value": round(val, 1), "unit": "ms",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": round(val, 1), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (numpy/scipy, as the reference computes)",
        "data": "synthetic (seeded RBF points, BASELINE config recipe)",
        "config": workload_config(args.config, cfg, args.gpus),
        "cpu_baseline": {"value": round(val, 1), "unit": "ms", "cores": ncores, "kind": "port",
                         **det},
        "e2e": {"value": round(val, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--l", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=None,
                    help="CPU slab rows (default: 4096, or l rounded up to 1024 when l > 4096 "
                         "-- the reference's spec.validate needs l <= rows)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional multi-rank check with ranks sharing a GPU")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.q is not None:
        cfg["q"] = args.q
    if args.l is not None:
        cfg["l"] = args.l
    if args.cpu_rows is None:
        args.cpu_rows = max(4096, -(-cfg["l"] // 1024) * 1024)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return

    import torch
    if world > 1:
        import torch.distributed as dist
        local_rank = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    if cfg.get("nystrom"):
        line, _ = run_nystrom(args, cfg, rank, world, local_rank)
        if line is not None and world == 1 and not args.no_cpu:
            v, det, (kmat, spec_o, _, _) = cpu_baseline_nystrom(cfg)
            line["cpu_baseline"] = {"value": round(v, 1), "unit": "ms", "cores": host_threads(),
                                    "kind": "port", **det}
            line["slab_parity"] = nystrom_slab_parity(cfg, kmat, spec_o)
        if line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    line, slab = run_ours(args, cfg, rank, world, local_rank)
    if line is not None:
        if world == 1 and not args.no_cpu:
            v, det, (a_s, qb_s, spec_o) = cpu_baseline(cfg, args.cpu_rows, slab=slab)
            line["cpu_baseline"] = {
                "value": round(v, 1), "unit": "ms", "cores": host_threads(), "kind": "port",
                "sample": f"rows 0..{det['rows_sampled']} of the {cfg['m']}-row workload, "
                          f"m-linear phases extrapolated x{cfg['m'] / det['rows_sampled']:g} "
                          "(sketch draw, Omega, SVD of B not scaled)", **det}
            line["slab_parity"] = slab_parity(cfg, a_s, qb_s, spec_o)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
