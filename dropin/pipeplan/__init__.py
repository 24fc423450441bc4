"""``import pipeplan`` resolved to the B200 drop-in (one set of types).

Put ``<repo>/dropin`` first on ``sys.path`` (or ``PYTHONPATH``) and every
``import pipeplan`` / ``from pipeplan.X import ...`` of an existing caller —
the reference's CLI, its test-suite, user code — gets this repository's
planning path: the same 77 public names (reference ``pipeplan/__init__.py:96-174``),
the same frozen dataclasses and exception classes, so ``==`` between results
and ``pytest.raises(pipeplan.ValidationError)`` work unchanged.

Hot-path modules (model, cost, ordering, partition, scheduler, planner,
baselines, fileio) are this package's (``paper_2204_10562_b200``, CUDA via
``libpipeplan_b200.so``).  The reference's tooling modules that are out of
scope here (``oracle`` brute force, ``gantt`` SVG, ``cli``) are
loaded from an installed copy of the reference as ``pipeplan.oracle`` etc.,
so their own ``from .cost import ...`` resolve to the drop-in; they are
looked up in ``$PIPEPLAN_REFERENCE_SRC``, then ``<repo>/baseline/_ref/pipeplan``.
Without a reference copy those three names are simply absent.
"""

import importlib.util
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(os.path.dirname(_HERE))
if _REPO not in sys.path:
    sys.path.append(_REPO)

import paper_2204_10562_b200 as _impl  # noqa: E402
from paper_2204_10562_b200 import *  # noqa: E402,F401,F403
from paper_2204_10562_b200.cost import stage_bwd_time, stage_compute_time, stage_fwd_time  # noqa: E402,F401

from . import baselines, cost, fileio, model, ordering, partition, planner, scheduler  # noqa: E402,F401

__version__ = _impl.__version__
IMPLEMENTATION = "paper_2204_10562_b200"


def _reference_dir():
    for d in (os.environ.get("PIPEPLAN_REFERENCE_SRC"), os.path.join(_REPO, "baseline", "_ref", "pipeplan")):
        if d and os.path.isfile(os.path.join(d, "oracle.py")):
            return d
    return None


def _exec_reference(name, namespace):
    """Run the reference's ``<name>.py`` as this package's submodule (its
    relative imports then bind to the drop-in's modules)."""
    d = _reference_dir()
    if d is None:
        raise ImportError(f"pipeplan.{name} is reference tooling (out of scope here); set PIPEPLAN_REFERENCE_SRC "
                          f"or install the reference into baseline/_ref")
    path = os.path.join(d, f"{name}.py")
    namespace["__file__"] = path
    with open(path) as f:
        exec(compile(f.read(), path, "exec"), namespace)


try:
    from . import oracle  # noqa: F401
    from .oracle import (BudgetExceeded, OracleError, OracleLimits, TStarResult, WStarResult,  # noqa: F401
                         brute_force_t_star, brute_force_w_star, enumerate_plans, optimal_schedule, plan_count)
    _oracle = oracle
except ImportError:
    _oracle = None
try:
    from . import gantt  # noqa: F401
    from .gantt import render_trace_svg  # noqa: F401
    _gantt = gantt
except ImportError:
    _gantt = None

__all__ = list(_impl.__all__) + (["BudgetExceeded", "OracleError", "OracleLimits", "TStarResult", "WStarResult",
                                  "brute_force_t_star", "brute_force_w_star", "enumerate_plans",
                                  "optimal_schedule", "plan_count"] if _oracle is not None else []) + \
    (["render_trace_svg"] if _gantt is not None else [])
__all__ = [n for n in __all__ if n not in ("spp_many", "simulate_pe_many", "check_numeric_range")] + \
    ["spp_many", "simulate_pe_many", "check_numeric_range"]

