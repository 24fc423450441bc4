"""pipeplan.baselines → paper_2204_10562_b200.baselines (see pipeplan/__init__.py)."""
import sys as _sys

from paper_2204_10562_b200 import baselines as _m

_sys.modules[__name__] = _m
