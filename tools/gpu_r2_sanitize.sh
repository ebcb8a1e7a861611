# usage: bash tools/gpu_r2_sanitize.sh <tool>   (one compute-sanitizer tool per gpurun call)
T=$1
BSCT_GRAPH=0 python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $T --print-limit 50 env BSCT_GRAPH=0 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
echo rc=$?
tail -25 gpurun_out/sanitize_$T.log
