# mode-product tests, blocked-tier SVT timings and one ncu capture of a complex64 1024^2 blocked round
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_factors.py -q -x -k mode_n_product -p no:cacheprovider > gpurun_out/modeprod.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/modeprod.log
timeout 600 python tools/experiments/svd_blocked_prof.py > gpurun_out/blocked_times.txt 2>&1; echo "times rc=$?"; cat gpurun_out/blocked_times.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_block_kernel -s 30 -c 1 -o gpurun_out/blk_c64 \
    python tools/experiments/svd_blocked_prof.py 1024 > gpurun_out/ncu_blk.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/blk_c64.ncu-rep --page raw --csv > gpurun_out/blk_c64_raw.csv 2>/dev/null
ncu -i gpurun_out/blk_c64.ncu-rep --page source --csv > gpurun_out/blk_c64_src.csv 2>/dev/null
ncu -i gpurun_out/blk_c64.ncu-rep --page details > gpurun_out/blk_c64_details.txt 2>/dev/null
