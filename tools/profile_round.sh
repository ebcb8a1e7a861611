# Round evidence: GPU tests, bench line, ncu launch list of the bench, --set full of the top kernels.
# usage: bash tools/profile_round.sh <tag>
T=${1:-r01}
O=gpurun_out/$T; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python bench.py > $O/bench.jsonl 2> $O/bench.err
# launch list (cold-cache, serialised: compare shares) of a shorter bench command
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-cufft"
$CMD > $O/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD2="python bench.py --slices 64 --iters 2 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD2 > $O/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pass_[abc]_1024|correction|gram_taps" -s 4 -c 7 -o $O/prof_full $CMD2 > $O/ncu_full.log 2>&1
echo "full rc=$?"
# K4 separately (its first launches would be skipped above)
ncu --set full --clock-control none --import-source on -k regex:bp_v3 -s 1 -c 1 -o $O/prof_bp $CMD2 > $O/ncu_bp.log 2>&1
echo "bp rc=$?"
# summaries on the box (gpurun copies back at most 64 MiB of gpurun_out/)
python tools/ncu_summary.py $O/prof_full.ncu-rep > $O/ncu_full_summary.txt 2>&1
python tools/ncu_summary.py $O/prof_bp.ncu-rep | tail -n +2 >> $O/ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py $O/prof_full.ncu-rep 64 > $O/ncu_traffic_full.json 2>&1
python tools/ncu_traffic.py $O/prof_bp.ncu-rep 64 > $O/ncu_traffic_bp.json 2>&1
python tools/launch_shares.py $O/launches.csv > $O/launch_shares.txt 2>&1
gzip -f $O/launches.csv
rm -f $O/prof_full.ncu-rep
