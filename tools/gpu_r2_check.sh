set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_gram.py tests/test_gpu_solvers_full.py tests/test_gpu_experiments.py -x -q > gpurun_out/pt_new.log 2>&1; echo rc=$? >> gpurun_out/pt_new.log
tail -30 gpurun_out/pt_new.log
timeout 300 python tools/time_gram.py --out gpurun_out/time_gram.jsonl
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_solvers_full.py > gpurun_out/pt_all.log 2>&1; echo rc=$? >> gpurun_out/pt_all.log
tail -5 gpurun_out/pt_all.log
