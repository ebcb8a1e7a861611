# persistent L = 2048 CG: parity tests, timing, then the solver test files
timeout 900 python -m pytest tests/test_gpu_persist.py -x -q > gpurun_out/pt_persist.log 2>&1; echo rc=$? >> gpurun_out/pt_persist.log
tail -3 gpurun_out/pt_persist.log
timeout 600 python tools/time_persist.py > gpurun_out/time_persist.log 2>&1; echo time rc=$?; cat gpurun_out/time_persist.log | tail -8
timeout 1200 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_solvers_full.py tests/test_gpu_chunks.py -q > gpurun_out/pt_solvers.log 2>&1; echo rc=$? >> gpurun_out/pt_solvers.log
tail -3 gpurun_out/pt_solvers.log
