# CG-path parity + timing (warp pass B vs the generic pass B)
python -m pytest tests/test_gpu_normal.py tests/test_gpu_solvers.py -x -q 2>&1 | tail -3
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/cg_new.json 2>&1
BSCT_PASSB_V1=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/cg_old.json 2>&1
for f in gpurun_out/cg_new.json gpurun_out/cg_old.json; do echo $f; tail -1 $f | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['phases_ms'], d['kernel_ms_per_step'])"; done
