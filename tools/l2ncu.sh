M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
BSCT_GRAPH=0 BSCT_CG_CHUNK=4 BSCT_CHUNK_STREAMS=4 python tools/l2_probe.py 64 6 && \
BSCT_GRAPH=0 BSCT_CG_CHUNK=4 BSCT_CHUNK_STREAMS=4 ncu --metrics $M --cache-control none --clock-control none -k regex:"pass_" -s 300 -c 60 --csv --log-file gpurun_out/l2_chunk4.csv python tools/l2_probe.py 64 6 > gpurun_out/l2a.log 2>&1; echo rc=$?
ncu --metrics $M --cache-control none --clock-control none -k regex:"pass_" -s 30 -c 9 --csv --log-file gpurun_out/l2_plain.csv python tools/l2_probe.py 256 6 > gpurun_out/l2b.log 2>&1; echo rc=$?
