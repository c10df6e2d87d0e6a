"""tcgen05 engine at the l_product shapes with each epilogue mode (CUDA-graph timed)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
sys.argv = [sys.argv[0]]
import tc_micro as T  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402

lib = nat.lib()
for epi in (3, 1, 2):
    lib.ltb_tc_debug_set_epi_mode(epi)
    print("epi_mode", epi)
    T.bench(1, 65536, 96, 96, 1, 0)
    T.bench(1, 96, 65536, 96, 0, 0)
    T.bench(96, 256, 256, 128, 0, 1)
    T.bench(1, 8192, 8192, 1024, 0, 0)
lib.ltb_tc_debug_set_epi_mode(3)
