set -x
timeout 600 python bench.py --steps 3 --warmup 3 --json-out gpurun_out/bench_c5.json > gpurun_out/bench_c5.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/bench_c5.log
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench_c4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --config 4 --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_c4_tr.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/bench_c4_tr.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench_ref.log
nproc
