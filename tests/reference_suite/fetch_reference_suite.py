"""Stage the reference's own test modules for a conformance run against the drop-in.

Test infrastructure, not product code.  Copies `pkg/tests/*.py` and the reference's
brute-force btph oracle (`pkg/src/ltensor/btph.py`, which its tests import and which
is out of scope for the build) unchanged from the reference tree into
`tests/reference_suite/_ref/`.  That directory is git-ignored -- no reference source
enters the history -- but not gpurun-ignored, so the staged copies travel to the GPU
box with the built libltb.so; `__graft_entry__.build()` runs this whenever the
reference tree is present.  The reference's `tests/conftest.py` (the `rng` fixture
and `random_shape`, conftest.py:5-12) is not staged: `tests/conftest.py` defines
both identically, and a second module named `conftest` would shadow the build's own
test helpers.  `conftest.py` beside this file aliases `ltensor` to
`paper_2202_02870_b200` so the modules run unmodified ("How the
build reuses this", step 1).
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
DEST = Path(__file__).resolve().parent / "_ref"


def fetch(ref: Path = REF, dest: Path = DEST) -> list[str]:
    if not (ref / "tests").is_dir():
        return []
    dest.mkdir(parents=True, exist_ok=True)
    staged = []
    for src in sorted((ref / "tests").glob("test_*.py")) + [ref / "src" / "ltensor" / "btph.py"]:
        # test_x.py -> test_reference_x.py: unique basenames beside the build's own tests
        name = src.name.replace("test_", "test_reference_", 1) if src.name.startswith("test_") else src.name
        shutil.copyfile(src, dest / name)
        staged.append(name)
    return staged


if __name__ == "__main__":
    names = fetch(Path(sys.argv[1]) if len(sys.argv) > 1 else REF)
    print(f"staged {len(names)} reference modules into {DEST}" if names else "reference tree not found; nothing staged")
