set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; echo rc=$? >> gpurun_out/pt_all.log
tail -3 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --json-out gpurun_out/bench_v4.json > gpurun_out/bench_v4.log 2>&1; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-cufft --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
