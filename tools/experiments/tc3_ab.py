"""A/B of the 3xTF32 engines (A split in shared memory vs A staged in TMEM) on the l_product step."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
sys.argv = [sys.argv[0]]
from paper_2202_02870_b200 import _native as nat  # noqa: E402
import tc_micro as T  # noqa: E402
lib = nat.lib()
for v in (0, 1):
    lib.ltb_tc_debug_set_tc3(v)
    print("tc3 =", v)
    T.bench(1, 65536, 96, 96, 1, 0)
    T.bench(1, 96, 65536, 96, 0, 0)
    T.bench(96, 256, 256, 128, 0, 1)
    T.bench(1, 8192, 8192, 1024, 0, 0)
lib.ltb_tc_debug_set_tc3(1)
