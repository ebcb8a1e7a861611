# one --set full capture of the back-projection kernel on a short bench run
CMD="python bench.py --slices 64 --iters 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
BSCT_BP_SB=${SB:-2} $CMD > gpurun_out/ncu_plain.log 2>&1 && \
BSCT_BP_SB=${SB:-2} ncu --set full --clock-control none --import-source on -k regex:bp_v -s 1 -c 1 -o gpurun_out/prof_bp ${CMD} > gpurun_out/ncu_bp.log 2>&1
echo rc=$?
