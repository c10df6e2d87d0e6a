# blocked-tier t_svd through the rotation-accumulation kernels: kernel / factor / config tests and timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factors.py tests/test_gpu_complex_carry.py -q -x -p no:cacheprovider > gpurun_out/tsvd_tests.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/tsvd_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config5" > gpurun_out/tsvd_cfg5.log 2>&1; echo "pytest2 rc=$?"; tail -5 gpurun_out/tsvd_cfg5.log
timeout 600 python tools/experiments/tsvd_time.py > gpurun_out/tsvd_time.txt 2>&1; echo "time rc=$?"; cat gpurun_out/tsvd_time.txt
