# packed blocked-Jacobi rounds: kernel / carry / config tests, config-5 and config-4 timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factors.py tests/test_gpu_complex_carry.py -q -p no:cacheprovider > gpurun_out/packed_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/packed_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config5 or config4" > gpurun_out/packed_cfg.log 2>&1; echo "pytest2 rc=$?"; tail -4 gpurun_out/packed_cfg.log
timeout 600 python tools/experiments/tsvd_time.py > gpurun_out/tsvd_time.txt 2>&1; echo "time rc=$?"; cat gpurun_out/tsvd_time.txt
timeout 900 python tools/experiments/cfg4_pga_iters.py 50 2 > gpurun_out/cfg4_pga_iters.txt 2>&1; echo "cfg4 rc=$?"; grep -E 'iterations:|iteration +(10|11|20|30|40|50):|jacobi_block' gpurun_out/cfg4_pga_iters.txt
