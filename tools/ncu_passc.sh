# ncu --set full of the two pass C kernels (round-1 cg_pass_c_1024_kernel vs the TMA-pipelined one)
P="python tools/l2_probe.py 256 3"
$P > gpurun_out/ncu_pc_plain.log 2>&1 || exit 1
BSCT_PASSC_TMA=0 ncu --set full --clock-control none --import-source on -k regex:"cg_pass_c" -s 3 -c 1 -o gpurun_out/pc_old $P > gpurun_out/ncu_pc_old.log 2>&1; echo rc=$?
BSCT_PASSC_TMA=1 ncu --set full --clock-control none --import-source on -k regex:"cg_pass_c" -s 3 -c 1 -o gpurun_out/pc_tma $P > gpurun_out/ncu_pc_tma.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/pc_old.ncu-rep > gpurun_out/pc_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/pc_tma.ncu-rep | tail -n +2 >> gpurun_out/pc_summary.txt 2>&1
cat gpurun_out/pc_summary.txt
