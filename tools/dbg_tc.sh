timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-cufft --json-out gpurun_out/bench_v2.json > gpurun_out/bench_v2.log 2>&1; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_v2.json'))
print(d['value'], d['ms_per_step'], d['phases_ms'], d['kernel_ms_per_step'], d['e2e']['value'], json.dumps(d['roofline'])[:300])"
for ov in 1; do BSCT_PIPE_OVERLAP=$ov BSCT_PIPE_CHUNK=256 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-cufft --no-e2e > gpurun_out/bench_ov.log 2>&1; tail -c 300 gpurun_out/bench_ov.log | head -c 0; python -c "
import json; d=json.loads(open('gpurun_out/bench_ov.log').read().strip().splitlines()[-1]); print('overlap', d['value'], d['ms_per_step'])"; done
