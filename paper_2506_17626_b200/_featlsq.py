"""The host framework this package drops into: the reference package `featlsq`.

The drop-in replaces featlsq's hot-path stage functions (assembly.py:124,
filtering.py:92/165/169, solvers.py:87) and keeps everything else of
featlsq as it is — its value types (`Domain`, `Decomposition`,
`FeatureBasis`, `ProblemSpec`, `ConstraintRows`, `LinearOperator2`,
`Jet2`), `decompose`, the problem builders, the monitor/result dataclasses,
`make_test_set`/`l1_error` and the exception classes are imported from
featlsq, not restated here. Only value types and host bookkeeping come from
featlsq; none of its numpy/LAPACK compute is called on this package's path.

featlsq is found on `sys.path`, else in `<repo>/baseline/_ref` (the
`pip install --target baseline/_ref <featlsq>` location that
`__graft_entry__.build()` fills and that travels with the repo to the GPU box).
"""

from __future__ import annotations

import os
import sys

_REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "baseline", "_ref")


def _load():
    try:
        import featlsq  # noqa: F401
        return featlsq
    except ImportError:
        pass
    if os.path.isdir(os.path.join(_REF_DIR, "featlsq")):
        sys.path.append(_REF_DIR)
        import featlsq  # noqa: F401
        return featlsq
    raise ImportError(
        "paper_2506_17626_b200 plugs into the featlsq package, which is not importable: "
        "install it (`pip install <featlsq>`) or run `python -c 'import __graft_entry__ as g; "
        f"g.build()'` to install it into {_REF_DIR}")


featlsq = _load()

from featlsq import assembly as ref_assembly  # noqa: E402,F401
from featlsq import basis as ref_basis  # noqa: E402,F401
from featlsq import domains as ref_domains  # noqa: E402,F401
from featlsq import errors as ref_errors  # noqa: E402,F401
from featlsq import jets as ref_jets  # noqa: E402,F401
from featlsq import linalg as ref_linalg  # noqa: E402,F401
from featlsq import problems as ref_problems  # noqa: E402,F401
from featlsq import solvers as ref_solvers  # noqa: E402,F401
