timeout 1200 python -m pytest tests/test_gpu_backproject.py tests/test_gpu_fullsize.py tests/test_gpu_lambda_x.py tests/test_gpu_race_stress.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -4
timeout 300 python tools/check_bp_tc.py 2048 2>&1 | grep "N="
