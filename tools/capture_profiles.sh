#!/bin/bash
# Round profile capture on the GPU box: bench JSON, launch list of a short bench run, and
# ncu --set full captures of the top kernels (each command runs once without ncu first).
set -x
R=${1:-r02}
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/${R}_bench.json 2> gpurun_out/prof/${R}_bench.err
python bench.py --steps 3 --warmup 3 --skip-extras --no-cpu-baseline --pga-iters 60 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-extras --no-cpu-baseline --pga-iters 60 > /dev/null 2>&1
python tools/experiments/lprod_fused_time.py > gpurun_out/prof/${R}_lprod_fused_timeline.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lprod_fused_kernel -s 3 -c 1 -o gpurun_out/prof/${R}_lprod_fused \
    python tools/experiments/lprod_fused_time.py > /dev/null 2>&1
python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jacobi_qr_kernel -s 1 -c 1 \
    -o gpurun_out/prof/${R}_jacobi_qr python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:xform_tile_kernel -c 2 \
    -o gpurun_out/prof/${R}_xform_pga python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1
# config 4: per-iteration times / sweeps of the 50 iterations, then one warm round of the blocked
# Jacobi with rotation accumulation (a cross round of iteration 31's second sweep) and the A0 = G V GEMM
python tools/experiments/cfg4_pga_iters.py 50 2 > gpurun_out/prof/${R}_cfg4_pga_iters.txt 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jacobi_block_kernel -s 100 -c 1 \
    -o gpurun_out/prof/${R}_jacobi_block python tools/experiments/cfg4_pga_iters.py 30 1 ncu > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:tc3_kernel -c 1 -o gpurun_out/prof/${R}_cgemm_tc \
    python tools/experiments/cfg4_pga_iters.py 12 1 ncu > /dev/null 2>&1
python tools/experiments/tsvd_time.py > gpurun_out/prof/${R}_config5_times.txt 2>&1
python tools/experiments/pga_kernel_breakdown.py 120 5 > gpurun_out/prof/${R}_pga_breakdown.txt 2>&1
python tools/experiments/pga_kernel_breakdown.py 120 5 fp64 > gpurun_out/prof/${R}_pga_breakdown_fp64.txt 2>&1
ls -la gpurun_out/prof
# summaries on the box (the .ncu-rep files together exceed what gpurun copies back): markdown,
# raw CSV per report, then drop the reports themselves
P=gpurun_out/prof
python tools/experiments/ncu_summary.py $P/${R}_ncu_summary.md \
    $P/${R}_lprod_fused.ncu-rep:"config-2 l_product, the one-launch persistent tcgen05 kernel (F, G, I tiles)" \
    $P/${R}_jacobi_qr.ncu-rep:"config-3 PGA K3 (Cholesky-preconditioned Jacobi, warm iteration 121; the 296-slice launch of the split batch)" \
    $P/${R}_xform_pga.ncu-rep:"config-3 PGA fused transforms (K1 + K4 prologue, K1' + norms epilogue)" \
    $P/${R}_jacobi_block.ncu-rep:"config-4 PGA, one warm round of the blocked Jacobi with rotation accumulation (complex64 1024x1024, 99 slices x 43 block pairs)" \
    $P/${R}_cgemm_tc.ncu-rep:"config-4 PGA, complex64 GEMM A0 = G V on tcgen05 (real 1024 x 2048 x 2048 per slice, 3xTF32)" \
    --launches $P/${R}_launches.csv:"bench.py --steps 3 --warmup 3 --skip-extras --pga-iters 60"
for f in $P/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
mv $P/${R}_lprod_fused.ncu-rep gpurun_out/ 2>/dev/null; rm -f gpurun_out/prof/*.ncu-rep
du -sh gpurun_out
