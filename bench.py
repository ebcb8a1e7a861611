#!/usr/bin/env python
"""Benchmark of the box-spline CT hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (default): BASELINE.json config 5 -- a stack of 2048 independent N = 512
slices, 360 angles, 725 detector bins, zeta_blur = 1, 50 CG iterations, sharded in
contiguous slice blocks over the ranks (no collective in the data path).
One step = the whole hot path of SURVEY.md 8(a) over the rank's slices:
  a1+a2 gram_build   (K0 tables + K1 taps)
  a1+a4 set_filter   (K0 back-projection tables + K2 spectrum)
  a5+a6 backproject  (K3 correction filter + K4)
  a7+a8 cg_solve     (K5 three FFT passes + K6 per iteration)
Metric: CG slice-iterations/s = total slices x iterations / step time (max over
ranks), i.e. whole-job throughput of the full step; per-phase times, Gram-build ms
and back-projection Gvox-angle/s are reported beside it.
Inputs: synthetic (synth/device.py), resident in HBM before the timed region;
the 2.1 GB sinogram stack exceeds the 126 MB L2, so no explicit L2 flush is used.
e2e: the same step through bsct_reconstruct_host with pinned HOST buffers
(H2D of the sinograms and D2H of the reconstructions inside the timed region).
--impl reference: the FP64 NumPy oracle (oracle/) on the host cores, on a bounded
sample of the same workload (this tier's reference arm).
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from synth import CONFIGS  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--slices", type=int, default=None, help="total slices (default: the config's)")
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--solver", default="cg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cufft", action="store_true")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--dense-angles", action="store_true",
                    help="only the SURVEY.md 8(d) Gram-build pair (production vs dense-angle build) at this config "
                         "and config 4, one JSON line")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=float(d["hbm_gbs"]), source="measured", sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    bf16_tflops=float(d.get("bf16_tflops", 1590.0)))
    return dict(hbm_gbs=6650.0, source="fallback", sm_max_mhz=1965.0, bf16_tflops=1590.0)


def ncu_traffic(kernel: str, slices: int):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/*/ncu_traffic.json, bytes per slice x slices of this launch), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic.json")))
    for f in reversed(files):  # the newest capture of this kernel
        k = json.load(open(f))["kernels"].get(kernel)
        if k:
            return k["bytes_per_slice"] * slices, os.path.relpath(f, ROOT)
    return None, None


def fp32_peak_tflops(sm_mhz: float, sms: int = 148) -> float:
    """FP32 non-tensor peak: SMs x 128 FP32 lanes x 2 flop (FMA) x clock (B200_PROFILING.md:
    148 SMs, 1965 MHz max; 4 SMSPs x 32 FP32 lanes per SM)."""
    return sms * 128 * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "samples": len(sm),
                "reasons": sorted(reasons)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- CPU oracle sample
# The FP64 oracle (oracle/, as it stands: never tuned) timed on the host cores: Gram taps and
# back projection split over angle blocks in a multiprocessing.Pool(ncores) (both are sums over
# angles), the CG iterations with SciPy's FFT on all cores (workers=-1 in
# oracle.normal.apply_fft).  Bounded samples: a pixel subset of the back projection and a few CG
# iterations, the times extrapolated to the whole slice and the configured iteration count.
def _oracle_gram_block(args):
    g, a0, a1 = args
    from oracle.gram import gram_taps
    return gram_taps(g, a0, a1)


def _oracle_bp_block(args):
    g, sino, a0, a1, k1, k2 = args
    from oracle.backproject import backproject
    sub = dict(g)
    sub["angles"] = np.asarray(g["angles"])[a0:a1]
    return backproject(sub, sino[a0:a1], pixels=(k1, k2))


def oracle_sample(cfg, iters: int, pool, ncores: int, bp_stride: int = 64, cg_iters: int | None = None):
    """One slice of config `cfg` through the oracle: returns (slice-iterations/s of the whole
    per-slice hot path, detail with the per-phase numbers)."""
    from oracle import solvers
    from synth.sinogram import random_sinogram
    g = cfg.geometry()
    n = len(g["angles"])
    sino = random_sinogram(cfg.seed, 1, n, cfg.n_det)[0]  # timing sample: the values do not matter
    nb = max(1, min(ncores, n))
    blocks = [(i * n // nb, (i + 1) * n // nb) for i in range(nb)]
    t0 = time.perf_counter()
    T = sum(pool.map(_oracle_gram_block, [(g, a0, a1) for a0, a1 in blocks]))
    t1 = time.perf_counter()
    N = cfg.N
    idx = np.arange(0, N * N, bp_stride)
    k1, k2 = idx // N, idx % N
    b_s = sum(pool.map(_oracle_bp_block, [(g, sino, a0, a1, k1, k2) for a0, a1 in blocks]))
    t2 = time.perf_counter()
    b = np.zeros((N, N))
    b.flat[idx] = b_s
    k = min(cg_iters or iters, iters)
    solvers.cg(T, b, k)
    t3 = time.perf_counter()
    bp_s = (t2 - t1) * bp_stride
    cg_s = (t3 - t2) * iters / k
    t_slice = (t1 - t0) + bp_s + cg_s
    return iters / t_slice, dict(gram_ms=1e3 * (t1 - t0), bp_s_extrapolated=bp_s,
                                 bp_gvox_angle_s=N * N * n / bp_s / 1e9, cg_s=cg_s,
                                 cg_slice_iter_s=iters / cg_s, wall_s=t3 - t0,
                                 sample=f"config {cfg.index}, 1 slice: Gram over {nb} angle blocks, back projection of "
                                        f"every {bp_stride}th pixel (time x{bp_stride}), {k} of {iters} CG iterations "
                                        f"(time x{iters}/{k})")


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_pool(ncores: int):
    import multiprocessing as mp
    return mp.get_context("spawn").Pool(ncores)


# bounded oracle samples per config (about 2-8 s each on 16 cores): (bp_stride, cg_iters)
ORACLE_SAMPLES = {1: (4, 20), 2: (16, 10), 3: (64, 5), 4: (256, 3), 5: (32, 10)}


# ----------------------------------------------------------------------------- GPU side measurements
def device_ms(fn, reps: int = 20, warm: int = 3) -> float:
    """Median device time of fn() (CUDA events), each call enqueued behind ~1 ms of device work
    (torch.cuda._sleep) so that the events see the device time, not the host-side call cost."""
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def gram_nonzero_pairs(g: dict, dev) -> int:
    """Number of (tap, angle) pairs with |lambda_x <theta_perp, dk>| < W_t / 2 over the whole
    (2N-1)^2 filter: the terms of P:122-129 that are not exactly zero (counted with torch)."""
    import torch
    N, lx, zeta = int(g["N"]), float(g.get("lambda_x", 1.0)), float(g.get("zeta", 0.0))
    d = torch.arange(-(N - 1), N, device=dev, dtype=torch.float64)
    a, b = d[:, None], d[None, :]
    total = 0
    for t in np.asarray(g["angles"], dtype=np.float64):
        c, s_ = np.cos(t), np.sin(t)
        H = lx * (abs(c) + abs(s_)) + zeta
        total += int((torch.abs(lx * (-s_ * a + c * b)) < H).sum())
    return total


GRAM_OPS_PER_TERM = 25  # FP32 ops per nonzero evaluation (argument, piece search, Horner, add)


def gram_pair(bsct, g: dict, dev, fma_peak_tflops: float, hbm_gbs: float) -> dict:
    """SURVEY.md 8(d) Gram-build pair: (i) the production build (exact zeros skipped) as a fraction
    of max(T_compute(nonzero evaluations), T_HBM(tap write)); (ii) the dense-angle build (every
    (tap, angle) pair, BSCT_GRAM_DENSE=1) as an FP32 rate; the FP32-pipe utilisation of (ii)
    comes from ncu (profiles/r02/ncu_gram_dense_*.txt, read here if present)."""
    import glob

    import torch
    N, n = int(g["N"]), len(g["angles"])
    D = 2 * N - 1
    taps = torch.empty((D, D), device=dev)
    ms = device_ms(lambda: bsct.gram_build(g, taps))
    os.environ["BSCT_GRAM_DENSE"] = "1"
    try:
        ms_dense = device_ms(lambda: bsct.gram_build(g, taps), reps=5)
    finally:
        del os.environ["BSCT_GRAM_DENSE"]
    nnz = gram_nonzero_pairs(g, dev)
    t_comp = nnz * GRAM_OPS_PER_TERM / (fma_peak_tflops * 1e12) * 1e3
    t_hbm = 4.0 * D * D / (hbm_gbs * 1e9) * 1e3
    dense_terms = n * D * D
    out = {"N": N, "n_angles": n, "build_ms": ms, "nonzero_pairs": nnz, "dense_pairs": dense_terms,
           "work_ratio_dense_over_nonzero": dense_terms / max(nnz, 1),
           "t_compute_ms": t_comp, "t_hbm_ms": t_hbm,
           "frac_of_max_compute_hbm": max(t_comp, t_hbm) / ms,
           "dense_build_ms": ms_dense,
           "dense_fp32_tflops_algorithmic": dense_terms * GRAM_OPS_PER_TERM / (ms_dense / 1e3) / 1e12,
           "dense_fp32_tflops_executed": 0.5 * dense_terms * GRAM_OPS_PER_TERM / (ms_dense / 1e3) / 1e12,
           "dense_frac_of_fp32_peak_executed": 0.5 * dense_terms * GRAM_OPS_PER_TERM / (ms_dense / 1e3) / 1e12
                                               / fma_peak_tflops,
           "note": "build_ms = K0 tables + K1 taps (device time); FLOP model 25 FP32 ops per nonzero (tap, angle) "
                   "term (SURVEY.md 8(d)); K1 evaluates the half of the taps up to the centre and mirrors "
                   "(G[k] = G[-k]), so the dense mode executes dense_pairs / 2 terms"}
    for mode in ("dense", "production"):  # ncu pipe utilisation (committed capture)
        files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_gram_{mode}_N{N}.json")))
        if files:
            out[f"{mode}_ncu"] = json.load(open(files[-1]))
            out[f"{mode}_ncu"]["source"] = os.path.relpath(files[-1], ROOT)
    del taps
    return out


def per_config_gpu(bsct, dev, B: int = 16) -> dict:
    """configs 1-4 on this GPU: Gram build (device ms), back projection (B slices) Gvox-angle/s and
    CG slice-iterations/s at the config's iteration count, B = 1 and B = 16."""
    import torch
    out = {}
    for ci in (1, 2, 3, 4):
        c = CONFIGS[ci]
        g = c.geometry()
        dt = torch.float64 if c.dtype == "f64" else torch.float32
        N, n, M = c.N, c.n_angles, c.n_det
        taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=dt, device=dev)
        gm = device_ms(lambda: bsct.gram_build(g, taps), reps=10)
        plan = bsct.plan_create(g, taps, max_batch=B)
        gen = torch.Generator(device=dev).manual_seed(ci)
        row = {"N": N, "dtype": c.dtype, "gram_build_ms": gm}
        for nb in (1, B):
            sino = torch.rand((nb, n, M), dtype=dt, device=dev, generator=gen)
            b = torch.empty((nb, N, N), dtype=dt, device=dev)
            x = torch.empty_like(b)
            bp = device_ms(lambda: bsct.backproject(plan, sino, b), reps=5, warm=2)
            cg = device_ms(lambda: bsct.cg_solve(plan, b, x, c.iters), reps=5, warm=2)
            row[f"B{nb}"] = {"bp_ms": bp, "bp_gvox_angle_s": nb * N * N * n / (bp / 1e3) / 1e9,
                             "cg_ms": cg, "cg_slice_iter_s": nb * c.iters / (cg / 1e3),
                             "cg_us_per_slice_iter": 1e3 * cg / (nb * c.iters)}
        out[ci] = row
        del plan, taps
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    iters = args.iters or cfg.iters
    total = args.slices or cfg.n_slices
    ncores = cpu_cores()
    stride, cgk = ORACLE_SAMPLES[args.config]
    stride *= 4  # each step a smaller sample, so that --steps 20 --warmup 5 ends within minutes
    with oracle_pool(ncores) as pool:
        for _ in range(args.warmup):
            oracle_sample(cfg, iters, pool, ncores, bp_stride=stride, cg_iters=cgk)
        vals, det = [], None
        t0 = time.perf_counter()
        for _ in range(args.steps):
            v, det = oracle_sample(cfg, iters, pool, ncores, bp_stride=stride, cg_iters=cgk)
            vals.append(v)
        wall = time.perf_counter() - t0
    v = float(np.median(vals))
    sample = f"1 of {total} slices per step; {det['sample']}; FP64 NumPy/SciPy oracle, {ncores} processes"
    line = {"impl": "reference", "metric": "CG slice-iterations/s (full hot-path step) at N=512",
            "value": v, "unit": "slice-iterations/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total * iters / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"BASELINE.json configs[{args.config}]", "N": cfg.N,
                                            "slices": total, "iters": iters},
            "cpu_baseline": {"value": v, "unit": "slice-iterations/s", "cores": ncores, "kind": "oracle",
                             "sample": sample, "detail": det, "wall_s": wall},
            "e2e": {"value": v, "unit": "slice-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def fma_peak():
    """Measured FP32 FMA peak (tools/fma_peak.cu on this pool's B200, profiles/*/fma_peak.json), else
    148 SMs x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md)."""
    import glob
    fm = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "fma_peak.json")))
    if fm:
        return float(json.load(open(fm[-1]))["fp32_fma_tflops"]), \
            f"measured: {os.path.relpath(fm[-1], ROOT)} (tools/fma_peak.cu, FP32 FMA chains)"
    return fp32_peak_tflops(1965.0), "derived: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md)"


def bp_tensor_core_path(cfg) -> bool:
    """Whether the library takes K4 v4 (tensor cores) for this geometry: the host check of
    bp_tc.cu (every 8 x 16 pixel tile's samples fit the 32-sample window, <= 8 samples per pixel)."""
    if cfg.dtype != "f32" or os.environ.get("BSCT_BP_V3") == "1":
        return False
    lx, ly, z = cfg.lambda_x, cfg.lambda_y, cfg.zeta
    for t in np.asarray(cfg.angles, dtype=np.float64):
        c, s_ = abs(np.cos(t)), abs(np.sin(t))
        span = (lx / ly) * (7 * s_ + 15 * c)
        cw = int(np.ceil(0.5 * (lx * (c + s_) + z + 3 * ly) / ly - 1e-12))
        if int(np.ceil(span)) + 5 + 2 * cw + 1 > 32 or 2 * cw + 1 > 8:
            return False
    return True


def roofline(per: dict, cfg, B: int, clk: dict, peaks: dict):
    """Roofline of the dominant kernel class of one profiled step (library CUDA events around every
    launch on its stream) and the HBM rooflines of the three FFT passes / whole CG iteration."""
    N, n_ang, M = cfg.N, cfg.n_angles, cfg.n_det
    L = 2
    while L < 2 * N - 1:
        L *= 2
    Q = L // 2 + 1
    dom = max(per, key=lambda k: per[k][0])
    vox_angles = B * N * N * n_ang
    # compulsory HBM bytes per launch of the fused CG passes: A reads p, r, x and
    # writes x, p and T1; B reads and writes T1; C reads T1 and reads/writes r (CG mode)
    cg_bytes = {"pass_a": B * (20 * N * N + 8 * Q * N), "pass_b": B * 16 * Q * N,
                "pass_c": B * (8 * Q * N + 8 * N * N)}
    kernels = {}
    for kk in ("pass_a", "pass_b", "pass_c"):
        if kk in per and per[kk][1] > 0:
            ms1 = per[kk][0] / per[kk][1]
            gbs = cg_bytes[kk] / (ms1 / 1e3) / 1e9
            kernels[kk] = {"ms_per_launch": ms1, "bound": "hbm", "achieved_gbs": gbs,
                           "frac_of_measured_hbm": gbs / peaks["hbm_gbs"]}
    # the whole fused CG iteration (normal apply + updates): compulsory bytes / iteration time
    if all(kk in kernels for kk in ("pass_a", "pass_b", "pass_c")):
        it_ms = sum(kernels[kk]["ms_per_launch"] for kk in ("pass_a", "pass_b", "pass_c"))
        it_bytes = sum(cg_bytes[kk] for kk in ("pass_a", "pass_b", "pass_c"))
        kernels["cg_iteration"] = {"ms": it_ms, "bytes": it_bytes, "achieved_gbs": it_bytes / (it_ms / 1e3) / 1e9,
                                   "frac_of_measured_hbm": it_bytes / (it_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                                   "state_floor_bytes": B * 24 * N * N,
                                   "frac_state_floor": B * 24 * N * N / (it_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                                   "note": "north_star: FFT normal-operator apply >= 60% of HBM roofline"}
    rooflines = {}
    peak_fp32, fp32_src = fma_peak()
    if "backproject" in per and per["backproject"][1] > 0:
        ms_launch = per["backproject"][0] / per["backproject"][1]
        # algorithmic FLOP per vox-angle (K4): S_eff samples x (degree-5 Horner = 5 FMA
        # + 1 FMA accumulate) x 2 flop + 2 FMA for k_theta; S_eff = mean support / lambda_y
        w_mean = (4 / np.pi) * cfg.lambda_x + cfg.zeta + 3 * cfg.lambda_y
        flops = vox_angles * (w_mean / cfg.lambda_y * 12.0 + 4.0)
        ach = flops / (ms_launch / 1e3) / 1e12
        tc = bp_tensor_core_path(cfg)
        if tc:
            # K4 v4 (bp_tc.cu): executed tcgen05 work = per (128-pixel tile, 128-slice group, angle)
            # 12 MMAs of 128 x 128 x 8 TF32 (3xTF32 split, K = 32 window); peak = measured bf16 burst
            # x the nominal TF32 / BF16 ratio (1.1 / 2.25 PFLOP/s dense, B200_PROFILING.md)
            tiles = -(-N // 16) * -(-N // 8) * -(-B // 128)
            mma_flops = tiles * n_ang * 12 * 2.0 * 128 * 128 * 8
            tf32_peak = peaks["bf16_tflops"] * 1.1 / 2.25
            tb, tsrc = ncu_traffic("bp_tc_kernel", B)
            rooflines["backproject"] = {
                "kernel": "backproject (K4 v4, tcgen05 kind::tf32)", "bound": "tensor", "traffic": tb,
                "traffic_source": tsrc,
                "achieved": mma_flops / (ms_launch / 1e3) / 1e12, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": mma_flops / (ms_launch / 1e3) / 1e12 / tf32_peak,
                "peak_source": "derived: MEASURED_PEAKS.json bf16_tflops x 1.1/2.25 (nominal TF32/BF16 dense)",
                "ms_per_launch": ms_launch, "algorithmic_tflops": ach,
                "algorithmic_frac_of_fp32_peak": ach / peak_fp32,
                "note": "achieved = executed MMA FLOP (3 TF32 products on the zero-padded 32-sample window); "
                        "algorithmic_tflops = the direct closed-form FLOP (12 S_eff + 4 per vox-angle) / time"}
        else:
            tb, tsrc = ncu_traffic("bp_v3_kernel", B)
            rooflines["backproject"] = {
                "kernel": "backproject (K4 v3)", "bound": "alu", "achieved": ach, "peak": peak_fp32,
                "unit": "TFLOP/s", "frac": ach / peak_fp32, "traffic": tb, "traffic_source": tsrc,
                "peak_source": fp32_src, "ms_per_launch": ms_launch,
                "note": "FLOP = the direct closed-form evaluation (12 S_eff + 4 per vox-angle, DESIGN.md 6)"}
    if "pass_b" in per and per["pass_b"][1] > 0:
        # pass B: forward + inverse column FFTs of length L on Q columns per slice (nominal
        # 5 L log2 L flops each), bound by the FP32 pipe (ncu: FMA pipe ~70%); HBM fraction beside it
        ms_launch = per["pass_b"][0] / per["pass_b"][1]
        fft_flops = B * Q * 2 * 5.0 * L * np.log2(L)
        ach = fft_flops / (ms_launch / 1e3) / 1e12
        tb, tsrc = ncu_traffic("pass_b_1024_kernel", B)
        rooflines["pass_b"] = {"kernel": "pass_b (column FFT x spectrum x inverse FFT)", "bound": "alu",
                               "achieved": ach, "peak": peak_fp32, "unit": "TFLOP/s", "frac": ach / peak_fp32,
                               "peak_source": fp32_src, "ms_per_launch": ms_launch,
                               "hbm_frac": kernels["pass_b"]["frac_of_measured_hbm"] if "pass_b" in kernels else None,
                               "traffic": tb, "traffic_source": tsrc,
                               "note": "FLOP = 2 x 5 L log2 L per column (nominal radix-2 count); the FP32 "
                                       "FMA peak is the same for FFMA and FFMA2 (profiles/r02/fma_peak.json); "
                                       "executed: 916 FP32x2 instructions per column and lane, ncu "
                                       "sm__pipe_fma_cycles_active 69-74% "
                                       "(profiles/r02/v10/ncu_full_summary.txt, ncu_full_summary_pass_b.txt)"}
    for kk, kname in (("pass_a", "cg_pass_a_1024_kernel"), ("pass_c", "cg_pass_c_1024_kernel")):
        if kk in kernels:
            tb, tsrc = ncu_traffic(kname, B)
            rooflines[kk] = {"kernel": kk, "bound": "hbm", "achieved": kernels[kk]["achieved_gbs"],
                             "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": kernels[kk]["frac_of_measured_hbm"],
                             "traffic": tb, "traffic_source": tsrc, "peak_source": peaks["source"],
                             "ms_per_launch": kernels[kk]["ms_per_launch"]}
    # kernel classes within 3% of the longest are a tie (passes A and B at config 5 differ by ~1% and
    # swap places from run to run): report the one further from its roofline
    tied = [k for k in rooflines if k in per and per[k][0] >= 0.97 * per[dom][0]]
    if dom in rooflines and len(tied) > 1:
        dom = min(tied, key=lambda k: rooflines[k]["frac"])
    roof = dict(rooflines.get(dom) or next(iter(rooflines.values())))
    roof["dominant_class"] = dom
    if len(tied) > 1:
        roof["tied_classes"] = tied
    roof["all"] = rooflines
    return roof, kernels


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2005_13471_b200 as bsct
    from synth.device import poisson_log, stack_images

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bsct.load()
    cfg = CONFIGS[args.config]
    iters = args.iters or cfg.iters
    total = args.slices or cfg.n_slices
    lo, hi = rank * total // ws, (rank + 1) * total // ws       # contiguous slice shard
    B = hi - lo
    g = cfg.geometry()
    N, n_ang, M = cfg.N, cfg.n_angles, cfg.n_det
    dev = torch.device("cuda", local)

    # ---- setup (untimed): plan, synthetic inputs resident in HBM
    taps = torch.empty((2 * N - 1, 2 * N - 1), device=dev)
    bsct.gram_build(g, taps)
    plan = bsct.plan_create(g, taps, max_batch=B)
    imgs = stack_images(cfg, list(range(lo, hi)), device=dev)
    sino = torch.empty((B, n_ang, M), device=dev)
    for c0 in range(0, B, 256):
        bsct.forward_project(plan, imgs[c0:c0 + 256], sino[c0:c0 + 256])
    sino = poisson_log(sino, cfg.noise_level, seed=cfg.seed + lo, kappa=1.0).contiguous()
    del imgs
    b = torch.empty((B, N, N), device=dev)
    x = torch.empty((B, N, N), device=dev)
    torch.cuda.synchronize()

    def step():
        """One timed step: the whole hot path over the rank's slices (Gram build, filter
        spectrum, then bsct_reconstruct = correction filter + back projection + solver)."""
        bsct.gram_build(g, taps)
        bsct.plan_set_filter(plan, taps)
        bsct.reconstruct(plan, sino, x, iters, args.solver)

    # launches per step (library counters; gram_build = K0 tables + K1 taps)
    launches = 2
    bsct.plan_set_filter(plan, taps)
    launches += plan.launches
    bsct.reconstruct(plan, sino, x, iters, args.solver)
    launches += plan.launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for k in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    t_step = e0.elapsed_time(e1) / args.steps

    # ---- breakdown (separate, not part of the headline): the same work as sequential phases
    # (no chunk overlap), each kernel launch bracketed by library CUDA events on its stream
    b = torch.empty((B, N, N), device=dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    plan.profile(True)
    evs[0].record()
    bsct.gram_build(g, taps)
    evs[1].record()
    bsct.plan_set_filter(plan, taps)
    evs[2].record()
    bsct.backproject(plan, sino, b)
    evs[3].record()
    bsct.cg_solve(plan, b, x, iters, args.solver)
    evs[4].record()
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    # the solve alone in the library's default schedule (config 5: L2-resident chunks on four
    # streams, one CUDA graph -- what the timed step runs; the profiled solve above uses the plain
    # whole-batch launches, whose kernels the profiler can time one by one)
    bsct.cg_solve(plan, b, x, iters, args.solver)
    ec = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ec[0].record()
    bsct.cg_solve(plan, b, x, iters, args.solver)
    ec[1].record()
    torch.cuda.synchronize()
    cg_sched_ms = ec[0].elapsed_time(ec[1])
    del b
    phases = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(4)])
    if ws > 1:
        tt = torch.tensor([t_step, *phases.tolist()], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, phases = float(tt[0]), tt[1:].cpu().numpy()
    value = total * iters / (t_step / 1e3)

    # ---- end to end through the public host-buffer API
    e2e = None
    if not args.no_e2e:
        sino_h = sino.cpu().pin_memory()
        x_h = torch.empty((B, N, N), dtype=torch.float32).pin_memory()

        def step_e2e():
            bsct.gram_build(g, taps)
            bsct.plan_set_filter(plan, taps)
            bsct.reconstruct_host(plan, sino_h, x_h, iters, args.solver)

        step_e2e()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step_e2e()
        e1.record()
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / args.steps
        if ws > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": total * iters / (te / 1e3), "unit": "slice-iterations/s",
               "h2d_bytes_per_step": int(sino_h.numel() * 4), "d2h_bytes_per_step": int(x_h.numel() * 4),
               "ms_per_step": te}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel class (profiler events inside the timed region)
    peaks = load_peaks()
    per = {k: (ms, cnt) for k, (ms, cnt) in prof.items()}  # one profiled step
    L = plan.L
    Q = L // 2 + 1
    roof, kernels = roofline(per, cfg, B, clk, peaks)
    if "cg_iteration" in kernels:  # the same algorithmic bytes over the default (chunked) schedule's time
        it_b = kernels["cg_iteration"]["bytes"]
        it_ms = cg_sched_ms / iters
        kernels["cg_iteration_chunked"] = {
            "ms": it_ms, "bytes": it_b, "effective_gbs": it_b / (it_ms / 1e3) / 1e9,
            "effective_frac_of_measured_hbm": it_b / (it_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
            "note": "the 3-pass design's compulsory HBM bytes per iteration over the chunked solve's time: the "
                    "chunks keep T1 and the CG vectors L2-resident, so this is an effective rate (actual DRAM "
                    "traffic is far lower), the measure of the schedule against the HBM-bound design"}

    # ---- side by side (comparison only, not a product path): y = G x through cuFFT
    # (torch.fft: rfft2 of the zero-padded L x L slice, * spectrum, irfft2, crop) against
    # bsct_normal_apply (three fused-free FFT passes) on the same 256-slice batch
    cufft = None
    if not args.no_cufft:
        nb = min(256, B)
        xs = x[:nb].contiguous()
        yb = torch.empty_like(xs)
        S = torch.empty((Q, L), device=dev)
        bsct.plan_spectrum(plan, S)
        St = (S.t() * (L * L)).contiguous()              # [L][Q]: rfft2 layout, undo the 1/L^2
        pad = torch.zeros((nb, L, L), device=dev)

        def cufft_apply():
            pad[:, :N, :N] = xs
            return torch.fft.irfft2(torch.fft.rfft2(pad) * St, s=(L, L))[:, :N, :N]

        ref = cufft_apply()
        bsct.normal_apply(plan, xs, yb)
        torch.cuda.synchronize()
        rel = float((ref - yb).norm() / ref.norm())
        ts = {}
        for name, fn in (("bsct_normal_apply", lambda: bsct.normal_apply(plan, xs, yb)), ("cufft", cufft_apply)):
            for _ in range(3):
                fn()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(10):
                fn()
            a1.record()
            torch.cuda.synchronize()
            ts[name] = a0.elapsed_time(a1) / 10
        cufft = {"slices": nb, "bsct_normal_apply_ms": ts["bsct_normal_apply"], "cufft_ms": ts["cufft"],
                 "speedup": ts["cufft"] / ts["bsct_normal_apply"], "rel_l2_diff": rel,
                 "note": "comparison only: torch.fft (cuFFT) rfft2/irfft2 of the padded slice; not used by the product"}
        del pad, St, S, yb, xs

    # ---- config 4 Gram build (side measurement): the full N = 1024,
    # 720-angle filter on one GPU, and the 8 angle shards one rank each would build before
    # the allreduce (the shards run here back to back on one GPU; max over shards reported)
    gram4 = None
    if not args.no_cufft:
        g4 = CONFIGS[4].geometry()
        N4 = CONFIGS[4].N
        t4 = torch.empty((2 * N4 - 1, 2 * N4 - 1), device=dev)
        part = torch.empty_like(t4)

        def timed(fn, reps=5):
            fn()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(reps):
                fn()
            a1.record()
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps

        full_ms = timed(lambda: bsct.gram_build(g4, t4))
        na = len(g4["angles"])
        shard_ms, acc = [], torch.zeros_like(t4)
        for r in range(8):
            lo, hi = r * na // 8, (r + 1) * na // 8
            shard_ms.append(timed(lambda: bsct.gram_build(g4, part, lo, hi)))
            acc += part
        rel = float((acc - t4).norm() / t4.norm())
        gram4 = {"N": N4, "n_angles": na, "full_ms": full_ms, "shard8_ms_max": max(shard_ms),
                 "shard8_sum_rel_diff": rel,
                 "note": "8 angle shards built back to back on one GPU (a rank's compute before the NCCL "
                         "allreduce of the 16.8 MB partial filter, which is not measured here)"}
        del t4, part, acc
        # D6: back projection of one config-4 slice, whole vs 8 angle shards (plans on the
        # sub-geometries); a rank's compute before the 4 MB allreduce of its partial image
        from paper_2005_13471_b200.parallel import angle_shard_geometry
        taps4 = torch.zeros((2 * N4 - 1, 2 * N4 - 1), device=dev)
        taps4[N4 - 1, N4 - 1] = 1.0  # the back projection does not read the filter
        s4 = torch.rand((1, na, CONFIGS[4].n_det), device=dev, generator=torch.Generator(device=dev).manual_seed(4))
        b4 = torch.empty((1, N4, N4), device=dev)
        pl4 = bsct.plan_create(g4, taps4, max_batch=1)
        bp_full = timed(lambda: bsct.backproject(pl4, s4, b4))
        pb4, acc4, bp_shard = torch.empty_like(b4), torch.zeros_like(b4), []
        for r in range(8):
            sub, lo, hi = angle_shard_geometry(g4, 8, r)
            pls = bsct.plan_create(sub, taps4, max_batch=1)
            ss = s4[:, lo:hi].contiguous()
            bp_shard.append(timed(lambda: bsct.backproject(pls, ss, pb4)))
            acc4 += pb4
        gram4["backproject_angle_shards"] = {
            "full_ms": bp_full, "shard8_ms_max": max(bp_shard),
            "shard8_sum_rel_diff": float((acc4 - b4).norm() / b4.norm()),
            "note": "one 1024^2 slice, 720 angles (SURVEY.md D6, parallel.backproject_sharded); the 4 MB "
                    "allreduce is not measured on one GPU"}
        del taps4, s4, b4, pb4, acc4

    # ---- NEXT-1 (side measurement): forward projector H, plain adjoint H^T and one SIRT
    # iteration on 256 of the slices, against one filter-based CG iteration on the same slices
    # -- the per-iteration cost the paper's method avoids (P:4)
    next1 = None
    if not args.no_cufft:
        nb = min(256, B)
        xs = x[:nb].contiguous()
        hs = torch.empty((nb, n_ang, M), device=dev)
        ims = torch.empty((nb, N, N), device=dev)

        def tm(fn, reps=3):
            fn()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(reps):
                fn()
            a1.record()
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / reps

        f_ms = tm(lambda: bsct.forward_project(plan, xs, hs))
        a_ms = tm(lambda: bsct.adjoint_project(plan, sino[:nb], ims))
        s_ms = tm(lambda: bsct.sirt_solve(plan, sino[:nb], ims, 2)) - tm(lambda: bsct.sirt_solve(plan, sino[:nb], ims, 1))
        c_ms = (tm(lambda: bsct.cg_solve(plan, xs, ims, 12)) - tm(lambda: bsct.cg_solve(plan, xs, ims, 2))) / 10
        va = nb * N * N * n_ang
        next1 = {"slices": nb, "forward_ms": f_ms, "forward_gvox_angle_s": va / (f_ms / 1e3) / 1e9,
                 "adjoint_ms": a_ms, "adjoint_gvox_angle_s": va / (a_ms / 1e3) / 1e9,
                 "sirt_iteration_ms": s_ms, "cg_iteration_ms": c_ms, "sirt_over_cg": s_ms / c_ms}
        del hs, ims, xs

    # ---- SURVEY.md 8(d) Gram-build pair (this config's geometry and config 4's) and the per-config
    # GPU numbers (configs 1-4; config 5 is this run)
    gram = None
    pcfg = None
    if not args.no_cufft:
        fpk, _ = fma_peak()
        gram = {f"config{args.config}": gram_pair(bsct, g, dev, fpk, peaks["hbm_gbs"]),
                "config4": gram_pair(bsct, CONFIGS[4].geometry(), dev, fpk, peaks["hbm_gbs"])}
        pcfg = per_config_gpu(bsct, dev)

    cpu = None
    if not args.no_cpu and ws == 1:
        ncores = cpu_cores()
        stride, cgk = ORACLE_SAMPLES[args.config]
        with oracle_pool(ncores) as pool:
            v, det = oracle_sample(cfg, iters, pool, ncores, bp_stride=stride, cg_iters=cgk)
            per_cfg = {}
            for ci in (1, 2, 3, 4):
                c = CONFIGS[ci]
                s_ci, k_ci = ORACLE_SAMPLES[ci]
                _, d = oracle_sample(c, c.iters, pool, ncores, bp_stride=s_ci, cg_iters=k_ci)
                per_cfg[ci] = {k: d[k] for k in ("gram_ms", "bp_gvox_angle_s", "cg_slice_iter_s", "sample")}
            per_cfg[args.config] = {k: det[k] for k in ("gram_ms", "bp_gvox_angle_s", "cg_slice_iter_s", "sample")}
        cpu = {"value": v, "unit": "slice-iterations/s", "cores": ncores, "kind": "oracle",
               "sample": det["sample"] + f"; FP64 NumPy/SciPy oracle as it stands, Pool({ncores}) over angle "
                                         f"blocks, SciPy FFT workers=-1",
               "detail": det, "per_config": per_cfg}

    kernel_ms = {k: round(v[0], 4) for k, v in per.items()}
    line = {
        "metric": "CG slice-iterations/s (full hot-path step) at N=512",
        "value": value, "unit": "slice-iterations/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"BASELINE.json configs[{args.config}]: {total} slices N={N}, {n_ang} angles, "
                               f"{M} bins, zeta={cfg.zeta}, {iters} {args.solver.upper()} iterations",
                   "slices": total, "slices_per_rank": B, "N": N, "iters": iters, "solver": args.solver,
                   "l2": "inputs (sinogram stack) exceed L2; no flush"},
        "phases_ms": {"gram_build": phases[0], "set_filter": phases[1], "backproject": phases[2],
                      "cg_solve": phases[3],
                      "note": "separate profiled step (library events around every launch; the solve as plain "
                              "whole-batch launches); the timed step calls bsct_reconstruct, whose solve runs "
                              "L2-resident chunks on four streams (cg_chunked_ms)"},
        "gram_build_ms": float(phases[0]),
        "gram_build_plus_set_filter_ms": float(phases[0] + phases[1]),
        "gram_pair": gram,
        "per_config_gpu": pcfg,
        "backproj_gvox_angle_s": total * N * N * n_ang / (phases[2] / 1e3) / 1e9,
        "cg_only_slice_iter_s": total * iters / (phases[3] / 1e3),
        "cg_chunked_ms": cg_sched_ms,
        "cg_chunked_slice_iter_s": total * iters / (cg_sched_ms / 1e3),
        "kernel_ms_per_step": kernel_ms,
        "cg_pass_rooflines": kernels,
        "cufft_side_by_side": cufft,
        "gram_config4": gram4,
        "next1_projection_iteration": next1,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "clocks": clk,
    }
    s = json.dumps(line)
    print(s, flush=True)
    if args.json_out:
        open(args.json_out, "w").write(s + "\n")
    if ws > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- configs 1-4: one slice
def run_single(args):
    """BASELINE.json configs 1-4: one 2D slice.  The two angle sums shard over the ranks
    (SURVEY.md 8(e)): each rank builds the Gram filter over its angle range, bsct_gram_build
    (a2), and one NCCL allreduce sums the (2N-1)^2 partial filters (a3, BJ:configs[4]); the
    back projection likewise (D6: each rank back projects its angle range, one allreduce of the
    N^2 partial image).  The filter spectrum and the CG solve of the single slice do not shard
    (replicas).  One step = gram shard + allreduce + set_filter + BP shard + allreduce + CG."""
    import torch
    import torch.distributed as dist

    import paper_2005_13471_b200 as bsct
    from paper_2005_13471_b200.parallel import angle_shard, angle_shard_geometry
    from synth.sinogram import config_sinogram

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bsct.load()
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    iters = args.iters or cfg.iters
    g = cfg.geometry()
    N, n_ang, M = cfg.N, cfg.n_angles, cfg.n_det
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    D = 2 * N - 1
    ga0, ga1 = angle_shard(n_ang, ws, rank)
    sub, ba0, ba1 = angle_shard_geometry(g, ws, rank)
    taps = torch.empty((D, D), dtype=dt, device=dev)
    bsct.gram_build(g, taps)
    plan = bsct.plan_create(g, taps, max_batch=1)
    plan_s = bsct.plan_create(sub, taps, max_batch=1) if ba1 > ba0 else None
    sino_h = torch.from_numpy(config_sinogram(cfg, 0)[None].astype(np.float64 if cfg.dtype == "f64" else np.float32))
    sino = sino_h.to(dev)
    sino_s = sino[:, ba0:ba1].contiguous()
    b = torch.empty((1, N, N), dtype=dt, device=dev)
    x = torch.empty_like(b)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]

    def step(marks=False):
        if marks:
            ev[0].record()
        bsct.gram_build(g, taps, ga0, ga1)  # this rank's angle shard (a2)
        if marks:
            ev[1].record()
        if ws > 1:
            dist.all_reduce(taps, op=dist.ReduceOp.SUM)  # a3 (same stream: ordered after the build)
        if marks:
            ev[2].record()
        bsct.plan_set_filter(plan, taps)  # a1 + a4
        if marks:
            ev[3].record()
        if plan_s is None:
            b.zero_()
        else:
            bsct.backproject(plan_s, sino_s, b)  # a5 + a6 over this rank's angles (D6)
        if marks:
            ev[4].record()
        if ws > 1:
            dist.all_reduce(b, op=dist.ReduceOp.SUM)
        if marks:
            ev[5].record()
        bsct.cg_solve(plan, b, x, iters, args.solver)  # a7 + a8
        if marks:
            ev[6].record()

    for _ in range(max(args.warmup, 3)):
        step()
    # library kernel launches per step: gram_build (K0 + K1), set_filter, back projection, solve
    launches = 2
    bsct.plan_set_filter(plan, taps)
    launches += plan.launches
    if plan_s is not None:
        bsct.backproject(plan_s, sino_s, b)
        launches += plan_s.launches
    bsct.cg_solve(plan, b, x, iters, args.solver)
    launches += plan.launches
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    t_step = e0.elapsed_time(e1) / args.steps
    # phase breakdown: the median of 10 marked steps
    ph = []
    for _ in range(10):
        step(marks=True)
        torch.cuda.synchronize()
        ph.append([ev[i].elapsed_time(ev[i + 1]) for i in range(6)])
    ph = np.median(np.array(ph), axis=0)
    # e2e: the sinogram from pinned host memory and the reconstruction back, inside the timed region
    sino_p = sino_h.pin_memory()
    x_p = torch.empty((1, N, N), dtype=dt).pin_memory()

    def step_e2e():
        sino.copy_(sino_p, non_blocking=True)
        sino_s.copy_(sino[:, ba0:ba1])
        step()
        x_p.copy_(x, non_blocking=True)

    step_e2e()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step_e2e()
    e1.record()
    torch.cuda.synchronize()
    t_e2e = e0.elapsed_time(e1) / args.steps
    tt = torch.tensor([t_step, t_e2e, *ph.tolist()], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step, t_e2e, ph = float(tt[0]), float(tt[1]), tt[2:].cpu().numpy()
    # kernel-class profile of one step (roofline of the dominant class)
    plan.profile(True)
    if plan_s is not None:
        plan_s.profile(True)
    step()
    prof = plan.profile_read()
    if plan_s is not None:
        for k, v in plan_s.profile_read().items():
            prof[k] = (prof.get(k, (0.0, 0))[0] + v[0], prof.get(k, (0.0, 0))[1] + v[1])
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    peaks = load_peaks()
    roof, kernels = roofline(prof, cfg, 1, clk, peaks)
    line = {
        "metric": f"CG slice-iterations/s (full hot-path step) at N={N}",
        "value": iters / (t_step / 1e3), "unit": "slice-iterations/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": f"BASELINE.json configs[{args.config}]: one slice N={N}, {n_ang} angles, {M} bins, "
                               f"lambda_y={cfg.lambda_y}, zeta={cfg.zeta}, {iters} {args.solver.upper()} iterations; "
                               f"Gram build and back projection over {ws} angle shard(s) + NCCL allreduce",
                   "N": N, "iters": iters, "solver": args.solver, "angle_shards": ws,
                   "l2": "single slice: the working set is L2-resident (no flush; the Gram filter is rebuilt every step)"},
        "phases_ms_max_over_ranks": {"gram_shard": ph[0], "gram_allreduce": ph[1], "set_filter": ph[2],
                                     "backproject_shard": ph[3], "bp_allreduce": ph[4], "cg_solve": ph[5]},
        "gram_build_ms": float(ph[0] + ph[1]),
        "kernel_ms_per_step": {k: round(v[0], 4) for k, v in prof.items()},
        "cg_pass_rooflines": kernels,
        "roofline": roof,
        "cpu_baseline": None,
        "e2e": {"value": iters / (t_e2e / 1e3), "unit": "slice-iterations/s",
                "h2d_bytes_per_step": int(sino_p.numel() * sino_p.element_size()),
                "d2h_bytes_per_step": int(x_p.numel() * x_p.element_size()), "ms_per_step": t_e2e},
        "gpu_launches": launches * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if args.json_out:
        open(args.json_out, "w").write(json.dumps(line) + "\n")
    if ws > 1:
        dist.destroy_process_group()


def run_gram_pair(args):
    """bench.py --dense-angles: the Gram-build pair alone."""
    import torch

    import paper_2005_13471_b200 as bsct
    ws, rank, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    bsct.load()
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    fpk, fsrc = fma_peak()
    out = {"metric": "Gram-filter build ms (production) and dense-angle FP32 rate", "fp32_peak_tflops": fpk,
           "fp32_peak_source": fsrc, "hbm_gbs": peaks["hbm_gbs"]}
    for ci in sorted({args.config, 4}):
        if CONFIGS[ci].dtype != "f32":
            continue
        out[f"config{ci}"] = gram_pair(bsct, CONFIGS[ci].geometry(), dev, fpk, peaks["hbm_gbs"])
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.dense_angles:
        run_gram_pair(args)
    elif CONFIGS[args.config].n_slices == 1:
        run_single(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
