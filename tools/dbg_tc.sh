timeout 1200 python -m pytest tests/test_gpu_backproject.py tests/test_gpu_fullsize.py tests/test_gpu_lambda_x.py tests/test_gpu_race_stress.py tests/test_gpu_determinism.py tests/test_gpu_solvers.py -q -x 2>&1 | tail -3
python tools/check_bp_tc.py 128 > gpurun_out/chk.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:bp_tc_kernel -s 1 -c 1 -o gpurun_out/bptc5 python tools/check_bp_tc.py 128 > gpurun_out/chk_ncu.log 2>&1
echo rc=$?
