# Round-2 evidence: ncu launch list of the bench command (plain whole-batch solver launches: the
# default chunked schedule launches ~100K small kernels per step, too many to replay under ncu) and
# --set full of the top kernels.  bash tools/profile_r02.sh <tag>
T=${1:-r02}
O=gpurun_out/$T; mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-cufft"
BSCT_CG_CHUNK=0 $CMD > $O/plain_launch.log 2>&1 && \
BSCT_CG_CHUNK=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD2="python bench.py --slices 128 --iters 2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-cufft"
BSCT_CG_CHUNK=0 $CMD2 > $O/plain_full.log 2>&1 && \
BSCT_CG_CHUNK=0 ncu --set full --clock-control none --import-source on -k regex:"pass_[abc]_1024|correction|gram_tiles|bp_tc" -s 6 -c 6 -o $O/prof_full $CMD2 > $O/ncu_full.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py $O/prof_full.ncu-rep > $O/ncu_full_summary.txt 2>&1
python tools/ncu_traffic.py $O/prof_full.ncu-rep 128 > $O/ncu_traffic.json 2>&1
python tools/launch_shares.py $O/launches.csv > $O/launch_shares.txt 2>&1
gzip -f $O/launches.csv
rm -f $O/prof_full.ncu-rep
cat $O/launch_shares.txt | head -20
