mkdir -p gpurun_out
timeout 300 python tools/experiments/pga_kernel_breakdown.py 120 5 > gpurun_out/pga_breakdown.txt 2>&1; echo "bd rc=$?"
timeout 300 python tools/experiments/pga_iter_timeline.py > gpurun_out/pga_iter_timeline.txt 2>&1; echo "tl rc=$?"
