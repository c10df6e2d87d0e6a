set -x
P=gpurun_out/prof
mkdir -p $P
python tools/experiments/lprod_fused_time.py > $P/r02_lprod_fused_timeline.txt 2>&1
python tools/experiments/chol_timeline.py > $P/r02_chol_timeline.txt 2>&1
python tools/experiments/pga_kernel_breakdown.py 120 5 > $P/r02_pga_breakdown.txt 2>&1
python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jacobi_qr_kernel -c 1 \
    -o $P/r02_jacobi_qr python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:xform_tile_kernel -c 2 \
    -o $P/r02_xform_pga python tools/experiments/prof_pga_late.py 120 2 > /dev/null 2>&1
python tools/experiments/ncu_summary.py $P/r02_ncu_summary_pga.md \
    $P/r02_jacobi_qr.ncu-rep:"config-3 PGA K3 (Cholesky-preconditioned Jacobi, warm iteration 121)" \
    $P/r02_xform_pga.ncu-rep:"config-3 PGA fused transforms (K1 + K4 prologue, K1' + norms epilogue)"
for f in $P/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
mv $P/r02_jacobi_qr.ncu-rep gpurun_out/ 2>/dev/null; rm -f gpurun_out/prof/*.ncu-rep
