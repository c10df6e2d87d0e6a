# per-kernel breakdowns of config 4 and config 1 PGA iterations (CUPTI), fused l_product timeline
mkdir -p gpurun_out
timeout 600 python tools/experiments/cfg4_breakdown.py 2 > gpurun_out/cfg4_breakdown.txt 2>&1; echo "cfg4 rc=$?"
timeout 300 python tools/experiments/cfg1_breakdown.py > gpurun_out/cfg1_breakdown.txt 2>&1; echo "cfg1 rc=$?"
timeout 300 python tools/experiments/lprod_fused_time.py > gpurun_out/lprod_fused_timeline.txt 2>&1; echo "lprod rc=$?"
