"""featlsq's TestWaveBaseline experiment (test_acceptance.py WAVE config)
through the drop-in: per-seed error, best iteration, residual, drop fraction."""
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "featlsq_tests"))
import paper_2506_17626_b200  # noqa: E402,F401
from paper_2506_17626_b200 import integrate  # noqa: E402

integrate.enable()
from test_acceptance import WAVE  # noqa: E402
from featlsq.runner import run_experiment  # noqa: E402

t = time.time()
r = run_experiment(WAVE, fd_cache_dir=tempfile.mkdtemp())
print("drop-in wave error_median", r.error_median, flush=True)
for s in r.seeds:
    print(s.seed, s.error, s.best_iteration, s.iterations_run, s.residual_norm, s.drop_fraction, flush=True)
print("time", time.time() - t)
