CMD="python tools/time_forward.py"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:forward_v3 -c 1 -o gpurun_out/prof_fwd $CMD > gpurun_out/ncu_fwd.log 2>&1
echo rc=$?
