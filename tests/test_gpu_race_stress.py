"""Race stress in place of compute-sanitizer racecheck/synccheck (closed on this pool:
profiles/r02/compute_sanitizer_closed.log).  A missing barrier or a shared-memory hazard in a
staging ring shows up as run-to-run differences once warp scheduling changes, so every kernel
family with shared-memory staging or block / cluster synchronisation is run repeatedly while a
second stream keeps the SMs busy with unrelated work (different co-residency and issue order
each time) and must reproduce its first result bitwise (R20: fixed reduction orders):

  K0 tables + K1 Gram tiles (levels 0-2 and dense mode; double-buffered record staging),
  K3 + K4 v3 back projection (cp.async ring), K5 warp-FFT passes A/B/C at L = 512, 1024, 2048
  (fused CG, SD, plain apply), generic passes (FP64), K7 forward, NEXT-2 on-chip cluster
  solver (DSMEM), CG resume."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def noise_stream_work(torch, stream, bufs):
    with torch.cuda.stream(stream):
        for _ in range(4):
            bufs[1].copy_(bufs[0])
            torch.mm(bufs[2], bufs[2], out=bufs[3])


def run_family(bsct, torch, N, n, dt, onchip, monkeypatch):
    tdt = torch.float64 if dt == "f64" else torch.float32
    M = int(1.5 * N) | 1
    g = dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n + 0.01, lambda_y=1.0, n_det=M, zeta=1.0)
    gen = torch.Generator(device="cuda").manual_seed(N)
    sino = torch.rand((2, n, M), dtype=tdt, device="cuda", generator=gen)
    monkeypatch.setenv("BSCT_ONCHIP", "1" if onchip else "0")
    monkeypatch.setenv("BSCT_GRAPH", "0")

    def once():
        taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=tdt, device="cuda")
        monkeypatch.setenv("BSCT_GRAM_DENSE", "1")
        bsct.gram_build(g, taps)
        dense = taps.clone()
        monkeypatch.delenv("BSCT_GRAM_DENSE")
        bsct.gram_build(g, taps)
        plan = bsct.plan_create(g, taps, max_batch=2)
        b = torch.empty((2, N, N), dtype=tdt, device="cuda")
        bsct.backproject(plan, sino, b)
        out = [dense, taps, b]
        for sv in ("cg", "sd", "landweber"):
            x = torch.empty_like(b)
            bsct.cg_solve(plan, b, x, 3, sv)
            out.append(x)
        y = torch.empty_like(b)
        bsct.normal_apply(plan, out[-1], y)
        s2 = torch.empty_like(sino)
        bsct.forward_project(plan, y, s2)
        r, p = b.clone(), b.clone()
        xr = torch.zeros_like(b)
        bsct.cg_resume(plan, xr, r, p, 2)
        out += [y, s2, xr, r, p]
        return out

    ref = [t.clone() for t in once()]
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    bufs = [torch.rand((1 << 22,), device="cuda"), torch.empty((1 << 22,), device="cuda"),
            torch.rand((1024, 1024), device="cuda"), torch.empty((1024, 1024), device="cuda")]
    for _ in range(6):
        noise_stream_work(torch, side, bufs)
        got = once()
        torch.cuda.synchronize()
        for a, c in zip(ref, got):
            assert torch.equal(a, c)


@pytest.mark.parametrize("N,n,dt", [(257, 40, "f32"), (513, 24, "f32"), (1025, 16, "f32"), (100, 30, "f32"),
                                    (40, 30, "f64")])
def test_race_stress(cuda_lib, N, n, dt, monkeypatch):
    import torch
    run_family(cuda_lib, torch, N, n, dt, False, monkeypatch)


@pytest.mark.parametrize("N,dt", [(64, "f64"), (200, "f32"), (256, "f32")])
def test_race_stress_onchip(cuda_lib, N, dt, monkeypatch):
    import torch
    run_family(cuda_lib, torch, N, 24, dt, True, monkeypatch)
