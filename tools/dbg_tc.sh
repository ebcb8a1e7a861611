cat > /tmp/l2.py <<'PY'
import os, sys, time
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2005_13471_b200 as bsct
from synth import CONFIGS
cfg = CONFIGS[5]; g = cfg.geometry(); N = 512; B = 512
taps = torch.empty((1023, 1023), device="cuda"); bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
b = torch.rand((B, N, N), device="cuda"); x = torch.empty_like(b)
for ch, pe in (("0", "0"), ("16", "0"), ("32", "0"), ("16", "1"), ("24", "1"), ("32", "1"), ("48", "1"), ("64", "1")):
    os.environ["BSCT_CG_CHUNK"] = ch; os.environ["BSCT_L2_PERSIST"] = pe
    bsct.cg_solve(plan, b, x, 10, "cg"); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bsct.cg_solve(plan, b, x, 10, "cg"); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"chunk {ch} persist {pe}: {ms:.2f} ms for {B} slices x 10 it -> {1e3*ms/(B*10):.3f} us/slice-it", flush=True)
PY
BSCT_L2_PERSIST_LOG=1 timeout 600 python /tmp/l2.py 2>&1 | grep -v "^bsct" ; BSCT_L2_PERSIST_LOG=1 BSCT_CG_CHUNK=32 BSCT_L2_PERSIST=1 timeout 100 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2005_13471_b200 as bsct
from synth import CONFIGS
cfg=CONFIGS[5]; g=cfg.geometry(); taps=torch.empty((1023,1023),device='cuda'); bsct.gram_build(g,taps)
plan=bsct.plan_create(g,taps,max_batch=64); b=torch.rand((64,512,512),device='cuda'); x=torch.empty_like(b)
bsct.cg_solve(plan,b,x,2,'cg'); torch.cuda.synchronize()" 2>&1 | grep bsct
