"""Install the reference package featlsq into baseline/_ref (git-ignored,
travels to the GPU box with the repo) and copy its own test files next to
it, so the GPU box can (a) import featlsq — the host framework the drop-in
plugs into — and (b) run featlsq's tests unmodified against the drop-in
(tests/test_gpu_reference_suite.py). Nothing here is committed: the
reference sources stay out of the repo's history.

    python scripts/install_reference.py [--force]

Needs /root/reference (this build container); on the GPU box the
prebuilt baseline/_ref is used as is.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(DEST, "featlsq_tests")


def install(force: bool = False) -> str:
    if not os.path.isdir(SRC):
        if os.path.isdir(os.path.join(DEST, "featlsq")):
            return DEST
        raise RuntimeError(f"{SRC} missing and no prebuilt {DEST}")
    if force or not os.path.isdir(os.path.join(DEST, "featlsq")):
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                        "--no-deps", "--find-links", "/opt/wheelhouse", "--upgrade", "--target",
                        DEST, SRC], check=True, capture_output=True)
    os.makedirs(TESTS, exist_ok=True)
    for name in sorted(os.listdir(os.path.join(SRC, "tests"))):
        if name.endswith(".py"):
            shutil.copy2(os.path.join(SRC, "tests", name), os.path.join(TESTS, name))
    return DEST


if __name__ == "__main__":
    print(install(force="--force" in sys.argv))
