# K3 v2 (register-blocked correction filter): bitwise A/B against the previous build, parity tests, bench
set -x
mkdir -p gpurun_out
python tools/k3_hash.py > gpurun_out/k3_new.txt 2>&1; echo rc=$?
BSCT_LIB=paper_2005_13471_b200/var/k3_old.so python tools/k3_hash.py > gpurun_out/k3_old.txt 2>&1; echo rc=$?
cat gpurun_out/k3_new.txt; diff gpurun_out/k3_new.txt gpurun_out/k3_old.txt && echo K3_BITWISE_EQUAL
timeout 1200 python -m pytest tests/test_gpu_backproject.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py tests/test_gpu_race_stress.py -m gpu -q -x > gpurun_out/pt_k3.log 2>&1; echo rc=$?; tail -3 gpurun_out/pt_k3.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/bench_k3.json > gpurun_out/bench_k3.log 2>&1; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_k3.json'));print(round(d['value']), d['ms_per_step'], d['e2e']['value'], d['clocks'], {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 1})"
