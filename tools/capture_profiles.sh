#!/bin/bash
# Round profile capture on the GPU box: bench JSON, launch list of a short bench run, and
# ncu --set full captures of the top kernels (each command runs once without ncu first).
set -x
R=${1:-r01}
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/${R}_bench.json 2> gpurun_out/prof/${R}_bench.err
python bench.py --steps 3 --warmup 3 --skip-extras --no-cpu-baseline --pga-iters 60 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-extras --no-cpu-baseline --pga-iters 60 > /dev/null 2>&1
python tools/pdl_ab.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc3_kernel -c 3 -o gpurun_out/prof/${R}_tc3 \
    python tools/pdl_ab.py > /dev/null 2>&1
python tools/prof_pga_late.py 120 2 > /dev/null 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:jacobi_qr_kernel -c 1 \
    -o gpurun_out/prof/${R}_jacobi_qr python tools/prof_pga_late.py 120 2 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:xform_tile_kernel -c 2 \
    -o gpurun_out/prof/${R}_xform_pga python tools/prof_pga_late.py 120 2 > /dev/null 2>&1
python tools/svd_blocked_prof.py 1024 > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:jacobi_block_kernel -s 20 -c 1 -o gpurun_out/prof/${R}_jacobi_block \
    python tools/svd_blocked_prof.py 1024 > /dev/null 2>&1
ls -la gpurun_out/prof
