"""A/B of the transposed-output epilogue (direct coalesced stores vs smem box + TMA store) on the l_product step."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
from paper_2202_02870_b200 import _native as nat  # noqa: E402
import runpy  # noqa: E402
for v in (0, 1):
    nat.lib().ltb_tc_debug_set_ct_direct(v)
    print("ct_direct =", v)
    runpy.run_path(str(ROOT / "tools" / "xform_ab.py"), run_name="__main__")
