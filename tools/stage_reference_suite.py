"""Stage the reference's own test files for the drop-in harness.

Copies /root/reference/pkg/tests/test_*.py into baseline/_ref/tests/ — the
git-ignored reference area that travels to the GPU box with the snapshot
(it is not committed; /root/reference does not exist on the box).
tests/test_reference_suite.py runs them there with `fempack` aliased to
this package (tests/refsuite/fempack_alias.py).  Called by __graft_entry__.build().
"""

import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref", "tests")


def stage() -> bool:
    if not os.path.isdir(SRC):
        return False
    os.makedirs(DST, exist_ok=True)
    for f in sorted(os.listdir(SRC)):
        if f.endswith(".py"):
            shutil.copyfile(os.path.join(SRC, f), os.path.join(DST, f))
    return True


if __name__ == "__main__":
    ok = stage()
    print(f"staged reference tests into {DST}" if ok else "reference tree absent; nothing staged")
    sys.exit(0)
