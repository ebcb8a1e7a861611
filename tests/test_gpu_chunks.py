"""L2-resident solver chunks on several streams (api.cu, BSCT_CG_CHUNK / BSCT_CHUNK_STREAMS: chunk k
of the batch runs all its iterations on stream k % ns with its own workspace slices, captured into
a CUDA graph).  Slices are independent (one CG per
slice), so a chunked solve must equal the plain one bit for bit -- x, the residual history and the
breakdown flags -- for CG, steepest descent and Landweber, with a ragged last chunk."""
import numpy as np
import pytest

from gpu_util import gpu_plan
from synth import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
@pytest.mark.parametrize("chunk,streams,graph", [("4", "3", "1"), ("3", "4", "1"), ("5", "2", "0"), ("4", "1", "1")])
def test_chunk_streams_bitwise(cuda_lib, monkeypatch, solver, chunk, streams, graph):
    import torch
    cfg = CONFIGS[5]  # N = 512, L = 1024
    g = cfg.geometry()
    N, B, K = cfg.N, 19, 4  # 19 slices: ragged last chunk
    plan, _ = gpu_plan(cuda_lib, g, "f32", max_batch=B)
    torch.manual_seed(3)
    b = torch.rand((B, N, N), device="cuda")
    out = []
    for chunked in (False, True):
        for k in ("BSCT_CG_CHUNK", "BSCT_CHUNK_STREAMS", "BSCT_GRAPH"):
            monkeypatch.delenv(k, raising=False)
        monkeypatch.setenv("BSCT_CG_CHUNK", "0")  # whole batch
        if chunked:
            monkeypatch.setenv("BSCT_CG_CHUNK", chunk)
            monkeypatch.setenv("BSCT_CHUNK_STREAMS", streams)
            monkeypatch.setenv("BSCT_GRAPH", graph)
        for rep in range(2):  # the second call replays the captured graph
            x = torch.full((B, N, N), np.nan, device="cuda")
            hist = torch.zeros((B, K), dtype=torch.float64, device="cuda")
            flags = torch.zeros(B, dtype=torch.int32, device="cuda")
            cuda_lib.cg_solve(plan, b, x, K, solver, resid_hist=hist, flags=flags)
            torch.cuda.synchronize()
            out.append((x.cpu(), hist.cpu(), flags.cpu()))
    for o in out[1:]:
        for a, c in zip(out[0], o):
            assert torch.equal(a, c)
    assert torch.isfinite(out[0][0]).all()


def test_default_chunking_bitwise(cuda_lib, monkeypatch):
    """The default schedule for B >= 24 at L = 1024 (chunks of 3 slices on 4 streams, one CUDA
    graph) against the whole-batch launches, through bsct_reconstruct as the bench calls it."""
    import torch
    cfg = CONFIGS[5]
    g = cfg.geometry()
    N, B, K = cfg.N, 26, 3
    plan, _ = gpu_plan(cuda_lib, g, "f32", max_batch=B)
    torch.manual_seed(6)
    sino = torch.rand((B, cfg.n_angles, cfg.n_det), device="cuda")
    xs = []
    for chunk in (None, "0"):
        if chunk is None:
            monkeypatch.delenv("BSCT_CG_CHUNK", raising=False)
        else:
            monkeypatch.setenv("BSCT_CG_CHUNK", chunk)
        for _ in range(2):
            x = torch.empty((B, N, N), device="cuda")
            hist = torch.zeros((B, K), dtype=torch.float64, device="cuda")
            cuda_lib.reconstruct(plan, sino, x, K, "cg", resid_hist=hist)
            torch.cuda.synchronize()
            xs.append((x.cpu(), hist.cpu()))
    for o in xs[1:]:
        for a, c in zip(xs[0], o):
            assert torch.equal(a, c)
