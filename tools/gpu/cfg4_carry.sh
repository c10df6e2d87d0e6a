# complex tensor-core GEMM and carried complex SVT tests, then the 50-iteration config-4 PGA timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_complex_carry.py -q -x -p no:cacheprovider > gpurun_out/ccarry_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/ccarry_tests.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm or blocked" > gpurun_out/ckern_tests.log 2>&1; echo "pytest2 rc=$?"; tail -5 gpurun_out/ckern_tests.log
timeout 900 python tools/experiments/cfg4_pga_iters.py ${1:-50} 2 > gpurun_out/cfg4_pga_iters.txt 2>&1; echo "cfg4 rc=$?"; tail -75 gpurun_out/cfg4_pga_iters.txt
