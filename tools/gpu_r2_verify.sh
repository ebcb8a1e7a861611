set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1; echo rc=$? >> gpurun_out/pt_all.log
tail -3 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -5 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --json-out gpurun_out/bench_v6.json > gpurun_out/bench_v6.log 2>&1; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_v6.json'));print(round(d['value']), d['ms_per_step'], d['e2e']['value'], d['clocks'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1})"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu --no-cufft > gpurun_out/bench_tr.log 2>&1; echo torchrun rc=$?
tail -1 gpurun_out/bench_tr.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('torchrun', round(d['value']), d['ms_per_step'], d['n_gpus'])"
