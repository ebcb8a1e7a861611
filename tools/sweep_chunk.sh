set -x
BSCT_CG_CHUNK=2 python -m pytest tests/test_gpu_solvers.py -x -q 2>&1 | tail -2
for c in 0 6 10 13 16 24; do
  BSCT_CG_CHUNK=$c python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/sw_$c.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw_$c.json').read().strip().splitlines()[-1]);print($c, d['phases_ms']['cg_solve'], d['kernel_ms_per_step'])"
done
