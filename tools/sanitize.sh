#!/bin/bash
# compute-sanitizer passes over the GPU parity / kernel / edge tests (small shapes): memcheck
# (out-of-bounds and misaligned accesses, leaks), racecheck (shared-memory hazards) and
# synccheck (barrier misuse).  Output: gpurun_out/sanitize_*.log
mkdir -p gpurun_out
SAN=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_kernels.py"
timeout 1500 $SAN --tool memcheck --error-exitcode 9 python -m pytest $T -m gpu -x -q -p no:cacheprovider \
    > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck exit $?" >> gpurun_out/sanitize_memcheck.log
timeout 1200 $SAN --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -p no:cacheprovider > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck exit $?" >> gpurun_out/sanitize_racecheck.log
timeout 1200 $SAN --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -x -q \
    -p no:cacheprovider > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck exit $?" >> gpurun_out/sanitize_synccheck.log
tail -3 gpurun_out/sanitize_*.log
