set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pt_all.log 2>&1; echo rc=$? >> gpurun_out/pt_all.log
tail -5 gpurun_out/pt_all.log
timeout 300 python bench.py --dense-angles > gpurun_out/dense.log 2>&1; tail -c 600 gpurun_out/dense.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
