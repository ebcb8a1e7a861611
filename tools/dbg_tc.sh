python tools/pb_probe.py 5 256 4 > gpurun_out/pb.log 2>&1 && cat gpurun_out/pb.log &&
ncu --set full --clock-control none --import-source on -k regex:pass_b_1024 -s 2 -c 1 -o gpurun_out/pb1 python tools/pb_probe.py 5 256 4 > gpurun_out/pb_ncu.log 2>&1
echo rc=$?
