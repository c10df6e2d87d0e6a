# config 1 (fp64 64x64x16): parity tests and it/s
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "config1 or pga or trace or svt" > gpurun_out/cfg1_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/cfg1_tests.log
timeout 300 python tools/experiments/cfg1_breakdown.py > gpurun_out/cfg1_breakdown.txt 2>&1; echo "cfg1 rc=$?"; grep -v Warn gpurun_out/cfg1_breakdown.txt | head -6
