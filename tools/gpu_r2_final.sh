# round-2 final evidence at HEAD: GPU tests, smoke, bench (v12), reference arm, ncu launch list
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; echo rc=$? >> gpurun_out/pt_all.log
tail -3 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? | tee -a gpurun_out/smoke.log; tail -5 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 --json-out gpurun_out/bench_v12.json > gpurun_out/bench_v12.log 2>&1; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_v12.json'));print(round(d['value']), d['ms_per_step'], d['e2e']['value'], d['clocks'], d['roofline']['frac'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1})"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_v12.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref_v12.log | cut -c1-400
# (ncu launch list: tools/profile_r02.sh, plain launches -- the chunked schedule has ~100K launches per step)
