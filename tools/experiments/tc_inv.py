"""Inverse-transform GEMM shape (NT x P output, K = P) on the tcgen05 engine: MN-major vs
K-major A, 3xTF32 vs 1xTF32, with and without epilogue stores (CUDA-graph timed)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
import tc_micro as T  # noqa: E402  (runs its own sweep first)

lib = nat.lib()
for epi in (1, 2):
    lib.ltb_tc_debug_set_epi_mode(epi)
    print("epi_mode", epi)
    for split in (3, 1):
        T.bench(1, 65536, 96, 96, 1, 0, split=split)
        T.bench(1, 65536, 96, 96, 0, 0, split=split)
        T.bench(1, 96, 65536, 96, 0, 0, split=split)
        T.bench(1, 96, 65536, 96, 0, 1, split=split)
lib.ltb_tc_debug_set_epi_mode(1)
