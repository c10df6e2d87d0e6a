# fp64 config-3 PGA on the V-free resident carried SVT: parity tests and it/s
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config3 or config1" > gpurun_out/fp64_cfg3_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/fp64_cfg3_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --skip-extras --no-cpu-baseline > gpurun_out/fp64_cfg3_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open('gpurun_out/fp64_cfg3_bench.log').read().strip().splitlines()[-1])
print('pga fp32', d['pga']['value'], 'fp64', d['pga']['fp64'])
PY
