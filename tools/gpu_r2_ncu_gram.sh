timeout 600 python -m pytest tests/test_gpu_gram.py -q -x 2>&1 | tail -2
python tools/time_gram.py > gpurun_out/tg_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gram_launches.csv python tools/time_gram.py --configs 5,4 --reps 2 --warm 1 > gpurun_out/tg_ncu.log 2>&1
echo rc=$?
cat gpurun_out/tg_plain.log
