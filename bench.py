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
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=float(d["hbm_gbs"]), source="measured", sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)))
    return dict(hbm_gbs=6650.0, source="fallback", sm_max_mhz=1965.0)


def ncu_traffic(kernel: str, slices: int):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/*/ncu_traffic.json, bytes per slice x slices of this launch), else None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_traffic.json")))
    if not files:
        return None, None
    d = json.load(open(files[-1]))
    k = d["kernels"].get(kernel)
    if not k:
        return None, None
    return k["bytes_per_slice"] * slices, os.path.relpath(files[-1], ROOT)


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
def oracle_sample(cfg, iters: int, bp_stride: int = 64, cg_iters: int | None = None):
    """The FP64 oracle (as it stands) on one slice of the workload: Gram taps, back
    projection of every bp_stride-th pixel (time extrapolated x bp_stride), and CG
    iterations with the FFT apply.  Returns (slice-iterations/s, detail)."""
    from oracle import solvers
    from oracle.backproject import backproject
    from oracle.gram import gram_taps
    from synth.sinogram import config_sinogram
    g = cfg.geometry()
    sino = config_sinogram(cfg, 0)
    t0 = time.perf_counter()
    T = gram_taps(g)
    t1 = time.perf_counter()
    N = cfg.N
    idx = np.arange(0, N * N, bp_stride)
    b_s = backproject(g, sino, pixels=(idx // N, idx % N))
    t2 = time.perf_counter()
    b = np.zeros((N, N))
    b.flat[idx] = b_s
    k = cg_iters or iters
    solvers.cg(T, b, k)
    t3 = time.perf_counter()
    t_slice = (t1 - t0) + (t2 - t1) * bp_stride + (t3 - t2) * iters / k
    return iters / t_slice, dict(gram_s=t1 - t0, bp_s_extrapolated=(t2 - t1) * bp_stride,
                                 cg_s=(t3 - t2) * iters / k, wall_s=t3 - t0)


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    iters = args.iters or cfg.iters
    total = args.slices or cfg.n_slices
    for _ in range(args.warmup):
        oracle_sample(cfg, iters, bp_stride=256, cg_iters=5)
    vals, det = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, det = oracle_sample(cfg, iters, bp_stride=256, cg_iters=5)
        vals.append(v)
    wall = time.perf_counter() - t0
    v = float(np.median(vals))
    sample = (f"1 of {total} slices per step: Gram taps, back projection of every 256th pixel "
              f"(time x256), 5 CG iterations (time x{iters}/5); FP64 NumPy/SciPy oracle")
    line = {"impl": "reference", "metric": "CG slice-iterations/s (full hot-path step) at N=512",
            "value": v, "unit": "slice-iterations/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total * iters / v / max(args.gpus, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"BASELINE.json configs[{args.config}]", "N": cfg.N,
                                            "slices": total, "iters": iters},
            "cpu_baseline": {"value": v, "unit": "slice-iterations/s", "cores": cpu_cores(), "kind": "oracle",
                             "sample": sample, "detail": det, "wall_s": wall},
            "e2e": {"value": v, "unit": "slice-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    dom = max(per, key=lambda k: per[k][0])
    L = plan.L
    Q = L // 2 + 1
    vox_angles = B * N * N * n_ang
    # compulsory HBM bytes per launch of the fused CG passes: A reads p, r, x and
    # writes x, p and T1; B reads and writes T1; C reads T1 and reads/writes r (CG mode)
    cg_bytes = {"pass_a": B * (20 * N * N + 8 * Q * N), "pass_b": B * 16 * Q * N,
                "pass_c": B * (8 * Q * N + 8 * N * N),
                "solver_update": B * 4 * N * N * 6, "solver_finish": B * 4 * N * N * 3}
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
                                   "note": "north_star: FFT normal-operator apply >= 60% of HBM roofline"}
    if dom == "backproject":
        # algorithmic FLOP per vox-angle (K4): S_eff samples x (degree-5 Horner = 5 FMA
        # + 1 FMA accumulate) x 2 flop + 2 FMA for k_theta; S_eff = mean support / lambda_y
        w_mean = (4 / np.pi) * cfg.lambda_x + cfg.zeta + 3 * cfg.lambda_y
        flops = vox_angles * (w_mean / cfg.lambda_y * 12.0 + 4.0)
        ms_launch = per[dom][0] / max(per[dom][1], 1)
        ach = flops / (ms_launch / 1e3) / 1e12
        peak, peak_src = fp32_peak_tflops(clk.get("sm_max_mhz") or 1965.0), \
            "derived: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz (B200_PROFILING.md)"
        import glob
        fm = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "fma_peak.json")))
        if fm:  # measured on this pool's B200 by tools/fma_peak.cu
            peak = float(json.load(open(fm[-1]))["fp32_fma_tflops"])
            peak_src = f"measured: {os.path.relpath(fm[-1], ROOT)} (tools/fma_peak.cu, FP32 FMA chains)"
        tb, tsrc = ncu_traffic("bp_v3_kernel", B)
        roof = {"kernel": "backproject (K4)", "bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "traffic": tb, "traffic_source": tsrc,
                "algorithmic_bytes": B * 4 * (n_ang * (M + 50) + N * N),
                "peak_source": peak_src,
                "note": "FLOP = the direct closed-form evaluation (12 S_eff + 4 per vox-angle, DESIGN.md 6); "
                        "K4 v3 evaluates it from per-tile tables and is shared-memory bound (ncu L1/smem 84%)"}
    else:
        # HBM-bound FFT passes: compulsory bytes of the pass per launch (K5)
        byts = cg_bytes.get(dom, 0)
        ms_launch = per[dom][0] / max(per[dom][1], 1)
        ach = byts / (ms_launch / 1e3) / 1e9
        kname = {"pass_a": "cg_pass_a_1024_kernel", "pass_b": "pass_b_1024_kernel",
                 "pass_c": "cg_pass_c_1024_kernel"}.get(dom, dom)
        tb, tsrc = ncu_traffic(kname, B)
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": tb, "traffic_source": tsrc,
                "peak_source": peaks["source"]}

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

    cpu = None
    if not args.no_cpu and ws == 1:
        v, det = oracle_sample(cfg, iters, bp_stride=16, cg_iters=iters)
        cpu = {"value": v, "unit": "slice-iterations/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"1 slice of config {args.config}: Gram taps, back projection of every 16th pixel "
                         f"(time x16), {iters} CG iterations; FP64 NumPy/SciPy oracle as it stands",
               "detail": det}

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
                      "note": "separate profiled step (library events around every launch); the timed step calls bsct_reconstruct"},
        "gram_build_ms": float(phases[0] + phases[1]),
        "backproj_gvox_angle_s": total * N * N * n_ang / (phases[2] / 1e3) / 1e9,
        "cg_only_slice_iter_s": total * iters / (phases[3] / 1e3),
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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
