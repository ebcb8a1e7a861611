python -m pytest tests/test_gpu_solvers.py -x -q -k "reconstruct" 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head
for c in 0 128 256 512; do
  BSCT_PIPE_CHUNK=$c python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/pipe_$c.json 2>&1
  echo "chunk $c: $(tail -1 gpurun_out/pipe_$c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value']))")"
done
BSCT_PIPE_PRIO=0 BSCT_PIPE_CHUNK=256 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/pipe_np.json 2>&1
echo "noprio 256: $(tail -1 gpurun_out/pipe_np.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['ms_per_step'],1))")"
