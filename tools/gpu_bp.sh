# K4 v3 parity + timing sweep over slices per CTA
python -m pytest tests/test_gpu_backproject.py -x -q 2>&1 | tail -3
for sb in 1 2 4; do
  BSCT_BP_SB=$sb python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --iters 1 > gpurun_out/bp_sb$sb.json 2>&1
done
BSCT_BP_V2=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --iters 1 > gpurun_out/bp_v2.json 2>&1
for f in gpurun_out/bp_*.json; do echo $f; tail -1 $f | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['phases_ms']['backproject'], d['kernel_ms_per_step']['backproject'])"; done
