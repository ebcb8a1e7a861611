# one --set full capture of kernels matching $K (regex), $C launches, on a short bench run
CMD="python bench.py --slices 64 --iters 2 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-2} -c ${C:-1} -o gpurun_out/prof_k ${CMD} > gpurun_out/ncu_k.log 2>&1
echo rc=$?
