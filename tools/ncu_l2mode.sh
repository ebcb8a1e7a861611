# ncu --set full of the three L = 1024 FFT passes in the L2-resident chunked schedule (one stream,
# no graph, --cache-control none: each kernel sees the L2 state its predecessor left)
export BSCT_CG_CHUNK=3 BSCT_CHUNK_STREAMS=1 BSCT_GRAPH=0
P="python tools/l2_probe.py 48 6"
$P > gpurun_out/l2m_plain.log 2>&1 || exit 1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"pass_[abc]_1024" -s 30 -c 3 -o gpurun_out/l2m $P > gpurun_out/l2m_ncu.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/l2m.ncu-rep > gpurun_out/l2m_summary.txt 2>&1
cat gpurun_out/l2m_summary.txt
