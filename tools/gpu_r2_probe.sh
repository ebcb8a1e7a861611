timeout 300 python tools/probe_persist.py > gpurun_out/probe_persist.log 2>&1
for v in minb1 ub1; do BSCT_LIB=paper_2005_13471_b200/var/$v.so timeout 300 python tools/probe_persist.py >> gpurun_out/probe_persist.log 2>&1; done
B=16 timeout 300 python tools/probe_persist.py >> gpurun_out/probe_persist.log 2>&1
cat gpurun_out/probe_persist.log
