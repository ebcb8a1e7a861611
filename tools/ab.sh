# A/B timing of library variants under paper_2005_13471_b200/var/: bash tools/ab.sh [bench args]
for so in paper_2005_13471_b200/var/*.so; do
  BSCT_LIB=$so python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu "$@" > gpurun_out/ab.json 2>&1
  echo "$(basename $so) $(tail -1 gpurun_out/ab.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1})")"
done
