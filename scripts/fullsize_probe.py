"""Full-size D-vs-LAPACK-factor LSQR comparison (tests/fullsize.py) for the
named configs; writes gpurun_out/fullsize_<cfg>.json."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2506_17626_b200._featlsq  # noqa: E402,F401
import fullsize  # noqa: E402

if __name__ == "__main__":
    cps = tuple(int(c) for c in os.environ.get("CPS", "100,300,1000,3000,10000").split(","))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for name in sys.argv[1:]:
        out = fullsize.compare(name, cps, log=lambda s: print(s, flush=True))
        with open(os.path.join(ROOT, "gpurun_out", f"fullsize_{name}.json"), "w") as fh:
            json.dump(out, fh, indent=1)
